# re-entry verification: GPU parity suite, default bench, and the ncu launch list of a bench run
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --latency-reps 500 --cpu-seconds 8 > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err; tail -3 gpurun_out/bench_v.err; cat gpurun_out/bench_v.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b32768.csv python bench.py --batch 32768 --steps 2 --warmup 1 --no-e2e --no-cpu --latency-reps 2 --no-extra > gpurun_out/launches.log 2>&1; tail -2 gpurun_out/launches.log
