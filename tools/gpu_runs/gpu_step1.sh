set -x
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_layers.py tests/test_gpu_front.py -x -q -m gpu > gpurun_out/step1_tests.log 2>&1; tail -5 gpurun_out/step1_tests.log
timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 2 3 4 --variants '[[1,0,1],[1,0,3]]' > gpurun_out/step1_sweep.json 2> gpurun_out/step1_sweep.err; cat gpurun_out/step1_sweep.json; tail -3 gpurun_out/step1_sweep.err
