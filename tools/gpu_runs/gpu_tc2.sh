timeout 180 python -m pytest tests/test_gpu_layers.py -q -x -k "tensor_engine or glue" 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25
timeout 300 python bench.py --steps 3 --warmup 3 --latency-reps 200 --cpu-seconds 8 > gpurun_out/bench_tc2.json 2> gpurun_out/bench_tc2.err; tail -3 gpurun_out/bench_tc2.err; cat gpurun_out/bench_tc2.json
