# the driver's round-end invocations: smoke, torchrun launch at N=1, reference arm
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --latency-reps 50 --no-extra > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; tail -2 gpurun_out/bench_torchrun1.err; head -c 300 gpurun_out/bench_torchrun1.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -2 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
