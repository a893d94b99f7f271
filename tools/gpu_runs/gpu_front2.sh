timeout 600 python -m pytest tests/test_gpu_front.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --latency-reps 100 --no-cpu --no-e2e > gpurun_out/bench_front2.json 2> gpurun_out/bench_front2.err; tail -3 gpurun_out/bench_front2.err; python -c "
import json;d=json.load(open('gpurun_out/bench_front2.json'));print(d['value'], d['latency_b1']['median_us'], d['clocks']); print({k:v['ms'] for k,v in d['roofline']['per_op'].items()}); print(d['extra_workloads']['fashion_b65536']['value'], d['extra_workloads']['fashion_b65536']['per_op'])"
