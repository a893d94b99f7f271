V='[[1,0,3],[1,0,1]]'
cd _ab_split
for lib in old new; do
cp alt/libbnn_$lib.so paper_2301_05126_b200/libbnn.so
timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 2 3 4 5 --variants "$V" > ../gpurun_out/abl5g_$lib.json 2>&1
python3 -c "import json; d=json.load(open('../gpurun_out/abl5g_$lib.json')); print('$lib', {k.split(':')[0]: {v: d[k][v]['ms'] for v in d[k]} for k in d})"
done
