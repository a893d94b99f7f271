timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_layers.py -x -q -m gpu > gpurun_out/split2_tests.log 2>&1; tail -3 gpurun_out/split2_tests.log
V='[[1,0,1],[1,0,3],[1,0,5]]'
timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 2 3 4 5 6 --variants "$V" > gpurun_out/split2_new.json 2>&1
(cd _ab_split && timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 2 3 4 5 6 --variants "$V" > ../gpurun_out/split2_old.json 2>&1)
timeout 300 python tools/tc_trace.py --block 3 --batch 32768 --variant "[1,0,5]" 2>&1 | head -5
