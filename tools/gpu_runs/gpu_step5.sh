timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_layers.py -x -q -m gpu > gpurun_out/step5_tests.log 2>&1; tail -2 gpurun_out/step5_tests.log
for b in 2 3; do timeout 300 python tools/tc_trace.py --block $b --batch 32768 --variant "[1,0,$([ $b = 2 ] && echo 3 || echo 1)]" 2>&1 | head -5; done
timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 2 3 4 5 --variants '[[1,0,1],[1,0,3]]' > gpurun_out/step5_new.json 2>&1
