V='[[1,0,3]]'
cd _ab_split
for lib in old new old new; do
cp alt/libbnn_$lib.so paper_2301_05126_b200/libbnn.so
timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 2 --variants "$V" > ../gpurun_out/abl5f_$lib.json 2>&1
python3 -c "import json; d=json.load(open('../gpurun_out/abl5f_$lib.json')); print('$lib', {v: d[k][v]['ms'] for k in d for v in d[k]})"
done
