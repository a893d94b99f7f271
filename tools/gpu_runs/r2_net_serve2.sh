# server: CTA 0 stages the request's images (no grid barrier before the first block) -- parity + latency
timeout 600 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -2
timeout 300 python tools/net_latency.py --reps 1000 2>&1 | tail -30
