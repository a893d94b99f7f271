timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_layers.py -x -q -m gpu > gpurun_out/ovl1_tests.log 2>&1; tail -2 gpurun_out/ovl1_tests.log
V='[[1,0,3],[1,0,5],[1,0,1]]'
for o in 1 0 1 0; do
BNN_OVL=$o timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 2 3 4 5 --variants "$V" > gpurun_out/ovl1_$o.json 2>&1
python3 -c "import json; d=json.load(open('gpurun_out/ovl1_$o.json')); print('OVL=$o', {k.split(':')[0]: {v: d[k][v]['ms'] for v in d[k]} for k in d})"
done
timeout 300 python tools/tc_trace.py --block 3 --batch 32768 --variant "[1,0,5]" 2>&1 | tail -9 | head -5
