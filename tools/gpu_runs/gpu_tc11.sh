timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 400 python bench.py --steps 5 --warmup 3 --latency-reps 300 --cpu-seconds 8 --no-e2e > gpurun_out/bench_tc11.json 2> gpurun_out/bench_tc11.err; tail -3 gpurun_out/bench_tc11.err; python -c "import json;d=json.load(open('gpurun_out/bench_tc11.json'));print(d['value'], d['roofline']['per_op'], d['extra_workloads'])"
timeout 300 python tools/tune.py --arch cifar10 --batches 1 --out gpurun_out/tune_b1 2>&1 | tail -30
