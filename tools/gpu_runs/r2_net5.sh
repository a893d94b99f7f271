python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -3
timeout 300 python tools/net_trace.py > /dev/null; python -c "
import json
d=json.load(open('gpurun_out/net_trace.json'))
for a,r in d.items():
  print(a, r['start_spread_ns'], r['copies_issued_med_ns'])
  for k,v in r.items():
    if isinstance(v,dict): print('  ',k, v)
"
timeout 300 python tools/net_latency.py --reps 1000
