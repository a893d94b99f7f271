# fused front end diagnosis: clock64 timelines of CTA 0 (B = 65536, so CTA 0 sees ~443 images), device
# time, and one ncu --set full capture per arch with the SASS source page
python -c "import __graft_entry__ as g; g.build()"
for a in cifar10 fashion; do
  python tools/front_trace.py --arch $a --batch 65536 && python tools/front_trace_view.py gpurun_out/front_trace_$a.npy 40 > gpurun_out/front_trace_$a.txt
  python tools/front_time.py --arch $a --batch 65536
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_front -s 3 -c 1 \
     -o gpurun_out/r2_front_$a python tools/front_time.py --arch $a --batch 32768 > gpurun_out/r2_ncu_front_$a.log 2>&1
  tail -2 gpurun_out/r2_ncu_front_$a.log
done
