cp paper_2301_05126_b200/libbnn.so /tmp/keep.so
for v in base early base early; do
cp alt_libs/libbnn_$v.so paper_2301_05126_b200/libbnn.so
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra --no-tune --latency-reps 2000 > gpurun_out/early_$v.json 2>/dev/null
python3 -c "import json; d=json.load(open('gpurun_out/early_$v.json'))['latency_b1']; print('$v', d['median_us'], d['kernels_only_us'], d['per_block_us_b1'])"
done
cp /tmp/keep.so paper_2301_05126_b200/libbnn.so
