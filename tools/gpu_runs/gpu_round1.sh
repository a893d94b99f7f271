set -x
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)"
./tools/microbench > gpurun_out/microbench.json; cat gpurun_out/microbench.json
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt; tail -40 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 --latency-reps 200 --cpu-seconds 10 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
