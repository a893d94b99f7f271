V='[[1,0,3],[1,0,1]]'
(cd _ab_split && timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 2 --variants "$V" > ../gpurun_out/abl5_cf9_1.json 2>&1)
timeout 300 python tools/layer_sweep.py --batch 262144 --blocks 2 --variants "$V" > gpurun_out/abl5_head_3.json 2>&1
