# A/B: software-pipelined conv_bin taps in the one-launch kernel (in-tree) vs one tap at a time (alt_libs/np0)
timeout 600 python -m pytest tests/test_gpu_net.py -q > gpurun_out/net_t.log 2>&1; tail -1 gpurun_out/net_t.log
for lib in base alt_libs/np0 base alt_libs/np0; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  echo "$lib:"; BNN_LIB=$L timeout 300 python tools/net_latency.py --reps 500 2>&1 | tail -2 | python -c "
import sys,json
for line in sys.stdin:
    a,j=line.split(' ',1); d=json.loads(j); print(' ',a,'net kernel',d['net_zero_copy']['kernels_only_us'],'server',d['server']['median_us'], 'eq', d['outputs_equal'])"
done
