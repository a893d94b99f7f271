timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/early2_tests.log 2>&1; tail -1 gpurun_out/early2_tests.log
timeout 300 python tools/determinism.py --reps 10
timeout 900 python bench.py > gpurun_out/early2_bench.json 2> gpurun_out/early2_bench.err
python3 -c "import json; d=json.load(open('gpurun_out/early2_bench.json')); l=d['latency_b1']; print(d['value'], d['e2e']['value'], d['clocks'], l['median_us'], l['kernels_only_us'], l['per_block_us_b1'], d['throughput_plan']['variants'], d['cpu_baseline']['timed_run_parity'])"
