timeout 600 python -m pytest tests/test_gpu_model.py -x -q -m gpu -k "batched or variants or calibrated" > gpurun_out/pair1_tests.log 2>&1; tail -25 gpurun_out/pair1_tests.log
timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 3 4 5 6 --variants '[[1,0,1],[1,0,5]]' > gpurun_out/pair1_sweep.json 2>&1
