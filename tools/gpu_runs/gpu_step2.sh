timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_layers.py tests/test_gpu_front.py -x -q -m gpu > gpurun_out/step2_tests.log 2>&1; tail -3 gpurun_out/step2_tests.log
for r in 1 2; do
(cd _ab_old && timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 2 3 4 5 --variants '[[1,0,1]]' > ../gpurun_out/step2_old_$r.json 2>&1)
timeout 300 python tools/layer_sweep.py --batch 32768 --blocks 2 3 4 5 --variants '[[1,0,1],[1,0,3]]' > gpurun_out/step2_new_$r.json 2>&1
done
timeout 300 python tools/front_time.py > gpurun_out/step2_front_new.txt 2>&1
(cd _ab_old && timeout 300 python tools/front_time.py > ../gpurun_out/step2_front_old.txt 2>&1)
