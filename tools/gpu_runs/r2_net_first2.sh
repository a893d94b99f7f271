# one-launch kernel: straight-line first-block rows -- parity + latency + per-block warp-0 clocks
timeout 600 python -m pytest tests/test_gpu_net.py -q > gpurun_out/net_t.log 2>&1; tail -1 gpurun_out/net_t.log
timeout 300 python tools/net_latency.py --reps 1000 2>&1 | tail -2 | python -c "
import sys,json
for line in sys.stdin:
    a,j=line.split(' ',1); d=json.loads(j); print(' ',a,'net kernel',d['net_zero_copy']['kernels_only_us'],'server',d['server']['median_us'], 'eq', d['outputs_equal'])"
timeout 300 python tools/net_trace.py > /dev/null 2>&1; python -c "
import json;d=json.load(open('gpurun_out/net_trace.json'))
for a in d: print(a, d[a].get('warp0_clocks'))"
