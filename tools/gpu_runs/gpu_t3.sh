cp paper_2301_05126_b200/libbnn.so /tmp/keep.so
for v in base t3 base t3; do
cp alt_libs/libbnn_$v.so paper_2301_05126_b200/libbnn.so
timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 3 4 5 --variants '[[1,0,0]]' > gpurun_out/t3_$v.json 2>&1
python3 -c "import json; d=json.load(open('gpurun_out/t3_$v.json')); print('$v', {k.split(':')[0]: d[k]['[1, 0, 0]']['ms'] for k in d})" 2>&1 | tail -1
done
cp alt_libs/libbnn_t3.so paper_2301_05126_b200/libbnn.so
timeout 600 python -m pytest tests/test_gpu_model.py -x -q -m gpu -k "batched or variants or calibrated" 2>&1 | tail -1
cp /tmp/keep.so paper_2301_05126_b200/libbnn.so
