timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/full1_tests.log 2>&1; tail -3 gpurun_out/full1_tests.log
