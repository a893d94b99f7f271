timeout 300 python -m pytest tests/test_gpu_layers.py -q -x -k "tensor_engine" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 400 python bench.py --steps 5 --warmup 3 --latency-reps 300 --cpu-seconds 8 > gpurun_out/bench_tc9.json 2> gpurun_out/bench_tc9.err; tail -3 gpurun_out/bench_tc9.err; cat gpurun_out/bench_tc9.json
