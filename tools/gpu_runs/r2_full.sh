python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; echo rc=$?
tail -2 gpurun_out/r2_gputest.log
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo rc=$?
tail -2 gpurun_out/r2_bench.err
python -c "
import json;d=json.load(open('gpurun_out/r2_bench.json'))
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])
for k,v in d['roofline']['per_op'].items(): print(k, v)
f=d['extra_workloads']['fashion_b65536']; print('fashion', f['value'], f['per_op'])
print(d['latency_b1']['cifar10']['median_us'], d['latency_b1']['fashion']['median_us'])
"
