python -c "import __graft_entry__ as g; g.build()"
for r in 1 2 4; do echo reps=$r; BNN_NET_REPS=$r timeout 300 python tools/net_trace.py > /dev/null; python -c "
import json
d=json.load(open('gpurun_out/net_trace.json'))
for a,r in d.items():
  print(a, [ (k.split(':')[1][:14], v.get('items_med_ns')) for k,v in r.items() if isinstance(v,dict)], r['fc_out'] if 'fc_out' in r else '')
"; done
