# E-builder store pattern A/B: front tests, front device time, one ncu capture (smem wavefronts)
timeout 600 python -m pytest -x -q tests/test_gpu_front.py 2>&1 | tail -2
for a in cifar10 fashion; do
  timeout 120 python tools/front_time.py --arch $a --batch 65536
done
for a in cifar10 fashion; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_front -s 3 -c 1 \
     -o gpurun_out/r2_front_e_$a python tools/front_time.py --arch $a --batch 32768 > gpurun_out/r2_ncu_front_e_$a.log 2>&1
  tail -1 gpurun_out/r2_ncu_front_e_$a.log
done
