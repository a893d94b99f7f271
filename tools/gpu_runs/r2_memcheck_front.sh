# compute-sanitizer memcheck + racecheck-free run over the fused front-end tests (loader-written E rows)
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_front.py -q -x > gpurun_out/r2_memcheck_front.log 2>&1; echo rc=$?
tail -4 gpurun_out/r2_memcheck_front.log
