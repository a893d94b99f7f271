cp paper_2301_05126_b200/libbnn.so /tmp/keep.so
for v in base pre base pre; do
cp alt_libs/libbnn_$v.so paper_2301_05126_b200/libbnn.so
echo "$v $(timeout 300 python tools/front_time.py 2>&1 | tail -1) | $(timeout 300 python tools/front_time.py --arch fashion --batch 65536 2>&1 | tail -1)"
done
cp /tmp/keep.so paper_2301_05126_b200/libbnn.so
timeout 600 python -m pytest tests/test_gpu_front.py tests/test_gpu_model.py -x -q -m gpu 2>&1 | tail -1
