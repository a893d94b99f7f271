V='[[1,0,3],[1,0,1]]'
for r in 1 2; do
timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 2 --variants "$V" > gpurun_out/abl5_new_$r.json 2>&1
(cd _ab_split && timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 2 --variants "$V" > ../gpurun_out/abl5_old_$r.json 2>&1)
done
BNN_PDL=0 timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 2 --variants "$V" > gpurun_out/abl5_nopdl.json 2>&1
