timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/pdl1_tests.log 2>&1; tail -2 gpurun_out/pdl1_tests.log
for pdl in 1 0 1; do
BNN_PDL=$pdl timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra > gpurun_out/pdl1_bench_$pdl.json 2>/dev/null
python3 -c "import json; d=json.load(open('gpurun_out/pdl1_bench_$pdl.json')); l=d['latency_b1']; print('PDL=$pdl', d['value'], d['e2e']['value'], l['median_us'], l['kernels_only_us'], l['per_block_us_b1'])"
done
