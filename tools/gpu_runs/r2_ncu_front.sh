# ncu full capture (with source) of the fused front-end kernel, CIFAR and fashion, B=32768
for a in cifar10 fashion; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_front -s 3 -c 1 \
     -o gpurun_out/r2_front_$a python tools/front_time.py --arch $a --batch 32768 > gpurun_out/r2_ncu_front_$a.log 2>&1
  tail -3 gpurun_out/r2_ncu_front_$a.log
done
