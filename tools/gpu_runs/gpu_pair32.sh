timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_layers.py -x -q -m gpu > gpurun_out/p32_tests.log 2>&1; tail -1 gpurun_out/p32_tests.log
for r in 1 2; do
timeout 300 python tools/layer_sweep.py --arch fashion --batch 65536 --blocks 2 --variants '[[1,0,0],[1,0,5]]' > gpurun_out/p32.json 2>&1
python3 -c "import json; d=json.load(open('gpurun_out/p32.json')); print({k: {v: d[k][v]['ms'] for v in d[k]} for k in d})"
done
