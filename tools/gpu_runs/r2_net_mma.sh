# one-launch kernel: conv_bin units on the warp-level binary MMA (in-tree) vs popc chains (alt_libs/nomma)
timeout 600 python -m pytest tests/test_gpu_net.py -q > gpurun_out/net_mma_t.log 2>&1; tail -1 gpurun_out/net_mma_t.log
for lib in base alt_libs/nomma base alt_libs/nomma; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  echo "$lib:"; BNN_LIB=$L timeout 300 python tools/net_latency.py --reps 500 2>&1 | tail -2 | python -c "
import sys,json
for line in sys.stdin:
    a,j=line.split(' ',1); d=json.loads(j); print(' ',a,'net kernel',d['net_zero_copy']['kernels_only_us'],'server',d['server']['median_us'], 'eq', d['outputs_equal'])"
done
