set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo rc=$?
tail -3 gpurun_out/r2_bench1.err
BNN_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --latency-reps 50 --no-extra --batch 65536 --tune-batch 32768 > gpurun_out/r2_bench_n2.json 2> gpurun_out/r2_bench_n2.err; echo rc=$?
tail -3 gpurun_out/r2_bench_n2.err
