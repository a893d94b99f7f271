timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 500 python bench.py --steps 5 --warmup 3 --latency-reps 300 --cpu-seconds 8 --no-extra > gpurun_out/bench_tc19.json 2> gpurun_out/bench_tc19.err; tail -3 gpurun_out/bench_tc19.err; python -c "import json;d=json.load(open('gpurun_out/bench_tc19.json'));print(d['value'], d['e2e'], d['latency_b1']['median_us'])"
