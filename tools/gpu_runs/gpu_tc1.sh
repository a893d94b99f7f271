set -x
timeout 180 python -m pytest tests/test_gpu_layers.py -q -x -k "tensor_engine or glue" 2>&1 | tail -30
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -30
timeout 300 python bench.py --steps 3 --warmup 3 --latency-reps 200 --no-cpu > gpurun_out/bench_tc1.json 2> gpurun_out/bench_tc1.err; tail -5 gpurun_out/bench_tc1.err; cat gpurun_out/bench_tc1.json
