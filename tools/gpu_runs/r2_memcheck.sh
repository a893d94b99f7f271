# compute-sanitizer memcheck over the round-2 GPU tests (one-launch net kernel + server, layout kernels, CLI)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_net.py tests/test_gpu_layers.py tests/test_cli.py -q -x -k "not idle" > gpurun_out/r2_memcheck.log 2>&1; echo rc=$?
tail -4 gpurun_out/r2_memcheck.log
