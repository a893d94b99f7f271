timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/full2_tests.log 2>&1; tail -2 gpurun_out/full2_tests.log
timeout 900 python bench.py --save-plan gpurun_out/tput_plan.json > gpurun_out/full2_bench.json 2> gpurun_out/full2_bench.err
python3 -c "import json; d=json.load(open('gpurun_out/full2_bench.json')); print(d['value'], d['e2e']['value'], d['clocks'], d['latency_b1']['median_us'], d['throughput_plan']['variants'], {k: v['ms'] for k, v in d['roofline']['per_op'].items()})"
