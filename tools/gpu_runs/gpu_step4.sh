timeout 300 python tools/tc_trace.py --block 2 --batch 32768 --variant "[1,0,3]" 2>&1 | head -5
timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 2 3 4 5 --variants '[[1,0,1],[1,0,3]]' > gpurun_out/step4_new.json 2>&1
(cd _ab_old && timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 2 3 4 5 --variants '[[1,0,1]]' > ../gpurun_out/step4_old.json 2>&1)
