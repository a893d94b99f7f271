timeout 600 python -m pytest tests/test_gpu_front.py tests/test_gpu_model.py -x -q -m gpu > gpurun_out/epi1_tests.log 2>&1; tail -2 gpurun_out/epi1_tests.log
for r in 1 2; do
echo "new $(timeout 300 python tools/front_time.py 2>&1 | tail -1) | $(timeout 300 python tools/front_time.py --arch fashion --batch 65536 2>&1 | tail -1)"
(cd _ab_split && echo "old $(timeout 300 python tools/front_time.py 2>&1 | tail -1) | $(timeout 300 python tools/front_time.py --arch fashion --batch 65536 2>&1 | tail -1)")
done
