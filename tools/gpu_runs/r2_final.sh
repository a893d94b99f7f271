# end-of-round validation: memcheck of the one-launch kernel tests, then the driver's pair (pytest -m gpu + bench)
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_net.py -q -x -k "not idle" > gpurun_out/r2_memcheck_net_final.log 2>&1; echo memcheck rc=$?
tail -3 gpurun_out/r2_memcheck_net_final.log
bash tools/gpu_runs/r2_full.sh
