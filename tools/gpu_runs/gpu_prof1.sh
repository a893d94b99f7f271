timeout 300 python -m pytest tests -m gpu -q -x -k "conv_int or traces or calibrated or golden" 2>&1 | tail -3
timeout 400 python bench.py --steps 5 --warmup 3 --latency-reps 300 --cpu-seconds 8 > gpurun_out/bench_tc3.json 2> gpurun_out/bench_tc3.err; tail -3 gpurun_out/bench_tc3.err; cat gpurun_out/bench_tc3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_r1.csv python bench.py --batch 32768 --steps 2 --warmup 1 --no-e2e --no-cpu --latency-reps 5 > gpurun_out/ncu_launch_bench.log 2>&1; tail -3 gpurun_out/ncu_launch_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_block|conv_first" -s 8 -c 6 -o gpurun_out/ncu_full_r1 python bench.py --batch 32768 --steps 1 --warmup 1 --no-e2e --no-cpu --latency-reps 2 > gpurun_out/ncu_full.log 2>&1; tail -5 gpurun_out/ncu_full.log
ls -la gpurun_out/
