timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_layers.py -x -q -m gpu > gpurun_out/ch1_tests.log 2>&1; tail -1 gpurun_out/ch1_tests.log
for r in 1 2; do
timeout 300 python tools/layer_sweep.py --arch fashion --batch 65536 --variants '[[1,0,0]]' > gpurun_out/ch1_new.json 2>&1
python3 -c "import json; d=json.load(open('gpurun_out/ch1_new.json')); print('new', {k: {v: d[k][v]['ms'] for v in d[k]} for k in d})"
(cd _ab_split && timeout 300 python tools/layer_sweep.py --arch fashion --batch 65536 --variants '[[1,0,0]]' > ../gpurun_out/ch1_old.json 2>&1)
python3 -c "import json; d=json.load(open('gpurun_out/ch1_old.json')); print('old', {k: {v: d[k][v]['ms'] for v in d[k]} for k in d})"
done
