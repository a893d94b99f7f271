python -c "import __graft_entry__ as g; g.build()"
for a in cifar10 fashion; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_front -s 3 -c 1 \
     -o gpurun_out/r2_front_v2_$a python tools/front_time.py --arch $a --batch 32768 > gpurun_out/r2_ncu_front_v2_$a.log 2>&1
  tail -1 gpurun_out/r2_ncu_front_v2_$a.log
done
