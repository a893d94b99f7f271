timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/final1_tests.log 2>&1; tail -2 gpurun_out/final1_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final1_bench.json 2> gpurun_out/final1_bench.err
python3 -c "import json; d=json.load(open('gpurun_out/final1_bench.json')); print(d['value'], d['e2e']['value'], d['clocks'], d['latency_b1']['median_us'], d['throughput_plan']['variants'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic_note'][:90])"
