timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_layers.py -x -q -m gpu > gpurun_out/hx1_tests.log 2>&1; tail -2 gpurun_out/hx1_tests.log
timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 2 --variants '[[1,0,3],[1,0,6]]' > gpurun_out/hx1_sweep.json 2>&1
python3 -c "import json; d=json.load(open('gpurun_out/hx1_sweep.json')); print({k.split(':')[0]: {v: d[k][v]['ms'] for v in d[k]} for k in d})"
timeout 300 python tools/tc_trace.py --block 2 --batch 32768 --variant "[1,0,6]" 2>&1 | tail -9 | head -5
