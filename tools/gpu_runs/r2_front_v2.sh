# redesigned front end: parity (front + model block tests), device time, CTA-0 timeline
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest -x -q tests/test_gpu_front.py tests/test_gpu_model.py 2>&1 | tail -15
for a in cifar10 fashion; do
  timeout 120 python tools/front_time.py --arch $a --batch 65536
  timeout 120 python tools/front_trace.py --arch $a --batch 65536 && python tools/front_trace_view.py gpurun_out/front_trace_$a.npy 30 > gpurun_out/front_trace_v2_$a.txt
done
head -4 gpurun_out/front_trace_v2_*.txt
