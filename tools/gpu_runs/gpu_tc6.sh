timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 400 python bench.py --steps 5 --warmup 3 --latency-reps 300 --cpu-seconds 8 > gpurun_out/bench_tc6.json 2> gpurun_out/bench_tc6.err; tail -3 gpurun_out/bench_tc6.err; cat gpurun_out/bench_tc6.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_block|conv_first" -s 8 -c 3 -o gpurun_out/ncu_full_r1d python bench.py --batch 32768 --steps 1 --warmup 1 --no-e2e --no-cpu --latency-reps 2 > gpurun_out/ncu_full_d.log 2>&1; tail -2 gpurun_out/ncu_full_d.log
