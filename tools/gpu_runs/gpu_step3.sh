timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_layers.py -x -q -m gpu > gpurun_out/step3_tests.log 2>&1; tail -3 gpurun_out/step3_tests.log
(cd _ab_old && timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 2 3 4 5 --variants '[[1,0,1]]' > ../gpurun_out/step3_old.json 2>&1)
timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 2 3 4 5 --variants '[[1,0,1],[1,0,3]]' > gpurun_out/step3_new.json 2>&1
