timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-extra > gpurun_out/c2_torchrun.json 2> gpurun_out/c2_torchrun.err; tail -c 300 gpurun_out/c2_torchrun.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/c2_ref.json 2> gpurun_out/c2_ref.err; cat gpurun_out/c2_ref.json | cut -c1-400
