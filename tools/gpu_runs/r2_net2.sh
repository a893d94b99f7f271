# one-launch network kernel: parity + latency + per-block timeline
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -5
timeout 300 python tools/net_latency.py --reps 1000
timeout 300 python tools/net_trace.py
