# one-launch network kernel: parity tests + batch-1 latency vs the per-block graph
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -15
timeout 300 python tools/net_latency.py --reps 1000
