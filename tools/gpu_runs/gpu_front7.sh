timeout 600 python -m pytest tests/test_gpu_front.py tests/test_gpu_model.py -q -x 2>&1 | grep -E "Error|error|assert|FAIL|passed|failed" | head -20
timeout 600 python bench.py --steps 5 --warmup 3 --latency-reps 100 --no-cpu --no-e2e > gpurun_out/bench_front7.json 2> gpurun_out/bench_front7.err; tail -3 gpurun_out/bench_front7.err; python -c "
import json;d=json.load(open('gpurun_out/bench_front7.json'));print(d['value'], d['latency_b1']['median_us'], d['clocks']); print({k:v['ms'] for k,v in d['roofline']['per_op'].items()}); print(d['extra_workloads']['fashion_b65536']['value'], d['extra_workloads']['fashion_b65536']['per_op'])"
timeout 300 python bench.py --steps 5 --warmup 3 --latency-reps 10 --no-cpu --no-e2e --no-extra --plan tools/plan_l5_halo.json > gpurun_out/bench_l5halo.json 2> gpurun_out/bench_l5halo.err; tail -2 gpurun_out/bench_l5halo.err; python -c "
import json;d=json.load(open('gpurun_out/bench_l5halo.json'));print(d['value'], d['clocks']); print({k:v['ms'] for k,v in d['roofline']['per_op'].items()})"
python tools/front_trace.py 2>&1 | tail -1
