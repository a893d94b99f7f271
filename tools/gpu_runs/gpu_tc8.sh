timeout 60 ./tools/desc_shift_test > gpurun_out/desc_shift.json 2>&1; cat gpurun_out/desc_shift.json
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 400 python bench.py --steps 5 --warmup 3 --latency-reps 300 --cpu-seconds 8 > gpurun_out/bench_tc8.json 2> gpurun_out/bench_tc8.err; tail -3 gpurun_out/bench_tc8.err; cat gpurun_out/bench_tc8.json
