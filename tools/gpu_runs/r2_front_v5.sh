timeout 600 python -m pytest -x -q tests/test_gpu_front.py 2>&1 | tail -2
for a in cifar10 fashion; do
  timeout 120 python tools/front_time.py --arch $a --batch 65536
  timeout 120 python tools/front_trace.py --arch $a --batch 65536 > /dev/null && python tools/front_trace_view.py gpurun_out/front_trace_$a.npy > gpurun_out/front_trace_v5_$a.txt
done
cat gpurun_out/front_trace_v5_*.txt
