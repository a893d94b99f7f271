# round-2 evidence: bench line (+ its tuned plan), launch list of the bench's timed steps under that plan,
# ncu --set full of one inference (B = 32,768) under the bench plan, the one-launch net kernel (CIFAR B = 1)
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --save-plan gpurun_out/r2_plan.json > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench rc=$?
K='regex:tc_front|tc_block|tc_pair|tc_halo|conv_|fc_|net_b1'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --plan gpurun_out/r2_plan.json --steps 2 --warmup 1 --no-latency --no-extra --no-calibrated --no-cpu --no-e2e \
  > gpurun_out/r2_launch_bench.log 2>&1; echo launches rc=$?
python tools/ncu_summary.py launches gpurun_out/r2_launches.csv > gpurun_out/r2_launch_shares.md
PLAN=$(python -c "import json;d=json.load(open('gpurun_out/r2_plan.json'));print(json.dumps(d.get('variants', d)))" 2>/dev/null || echo '{"2": [1, 0, 6]}')
echo plan $PLAN
timeout 900 ncu --set full --clock-control none --import-source on -s 21 -c 7 -o gpurun_out/r2_ncu_full \
  python tools/plan_time.py --batch 32768 --reps 1 --plan '{"2": [1, 0, 6]}' > gpurun_out/r2_ncu_full.log 2>&1; echo full rc=$?
python tools/ncu_summary.py full gpurun_out/r2_ncu_full.ncu-rep > gpurun_out/r2_ncu_full.md
python tools/ncu_summary.py traffic gpurun_out/r2_ncu_full.ncu-rep 32768 > gpurun_out/r2_ncu_traffic.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:net_b1 -s 45 -c 1 -o gpurun_out/r2_net_cifar \
  python tools/net_trace.py > /dev/null 2>&1; echo net rc=$?
python tools/ncu_summary.py full gpurun_out/r2_net_cifar.ncu-rep > gpurun_out/r2_ncu_net.md
tail -3 gpurun_out/r2_bench.err
