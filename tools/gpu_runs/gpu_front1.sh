# fused front end: parity first, then the default bench
timeout 600 python -m pytest tests/test_gpu_front.py -q -x 2>&1 | tail -25
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --latency-reps 300 --cpu-seconds 5 > gpurun_out/bench_front1.json 2> gpurun_out/bench_front1.err; tail -3 gpurun_out/bench_front1.err; python -c "
import json;d=json.load(open('gpurun_out/bench_front1.json'));print(d['value'], d['e2e']['value'], d['latency_b1']['median_us'], d['clocks']); print({k:v['ms'] for k,v in d['roofline']['per_op'].items()}); print(d['extra_workloads']['fashion_b65536']['value'], d['extra_workloads']['fashion_b65536']['per_op'])"
