cp paper_2301_05126_b200/libbnn.so /tmp/libbnn_orig.so
for v in 0 32 200 0 32 200; do
cp alt_libs/libbnn_sleep$v.so paper_2301_05126_b200/libbnn.so
echo "sleep=$v $(timeout 300 python tools/front_time.py 2>&1 | tail -1) | fashion $(timeout 300 python tools/front_time.py --arch fashion --batch 65536 2>&1 | tail -1)"
done
cp /tmp/libbnn_orig.so paper_2301_05126_b200/libbnn.so
