timeout 200 python -m pytest tests/test_gpu_layers.py -q -x -k "tensor_engine" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 400 python bench.py --steps 5 --warmup 3 --latency-reps 300 --cpu-seconds 8 > gpurun_out/bench_tc5.json 2> gpurun_out/bench_tc5.err; tail -3 gpurun_out/bench_tc5.err; cat gpurun_out/bench_tc5.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_block|conv_first" -s 8 -c 3 -o gpurun_out/ncu_full_r1c python bench.py --batch 32768 --steps 1 --warmup 1 --no-e2e --no-cpu --latency-reps 2 > gpurun_out/ncu_full_c.log 2>&1; tail -2 gpurun_out/ncu_full_c.log
