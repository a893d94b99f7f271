timeout 600 python -m pytest tests/test_gpu_model.py -x -q -m gpu -k "batched or variants or calibrated" > gpurun_out/pair2_tests.log 2>&1; tail -3 gpurun_out/pair2_tests.log
timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 3 4 5 6 --variants '[[1,0,5],[1,128,1],[1,128,5]]' > gpurun_out/pair2_sweep.json 2>&1
timeout 300 python tools/tc_trace.py --block 3 --batch 32768 --variant "[1,128,1]" 2>&1 | head -5
