timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_front -s 3 -c 1 \
     -o gpurun_out/r2_front_v4_fashion python tools/front_time.py --arch fashion --batch 32768 > /dev/null 2>&1
ncu -i gpurun_out/r2_front_v4_fashion.ncu-rep --page source --csv --print-source sass > gpurun_out/src_v4_fashion.csv 2>/dev/null
ls -la gpurun_out/
