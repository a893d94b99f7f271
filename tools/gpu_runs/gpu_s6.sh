cp paper_2301_05126_b200/libbnn.so /tmp/keep.so
for v in s5 s6 s5 s6; do
cp alt_libs/libbnn_$v.so paper_2301_05126_b200/libbnn.so
timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 3 4 5 6 --variants '[[1,0,1]]' > gpurun_out/s6_$v.json 2>&1
python3 -c "import json; d=json.load(open('gpurun_out/s6_$v.json')); print('$v', {k.split(':')[0]: {v: d[k][v]['ms'] for v in d[k]} for k in d})"
done
cp /tmp/keep.so paper_2301_05126_b200/libbnn.so
