# fused front end: clock64 timelines of CTA 0 (both archs) + device time
for a in cifar10 fashion; do
  python tools/front_trace.py --arch $a --batch 1184 && python tools/front_trace_view.py gpurun_out/front_trace_$a.npy 24 > gpurun_out/front_trace_$a.txt
  python tools/front_time.py --arch $a --batch 32768
done
