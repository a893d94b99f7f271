timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 3 4 5 --variants '[[1,0,5]]' > gpurun_out/split_base.json 2>&1
(cd _ab_split && timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 3 4 5 --variants '[[1,0,5]]' > ../gpurun_out/split_new.json 2>&1)
(cd _ab_split && timeout 300 python tools/tc_trace.py --block 3 --batch 32768 --variant "[1,0,5]" 2>&1 | head -5)
timeout 300 python tools/tc_trace.py --block 3 --batch 32768 --variant "[1,0,5]" 2>&1 | head -5
