# A/B: FC_OUT partial sums accumulated by the fc_bin CTAs (in-tree) vs FC_OUT on the last CTA (alt_libs/old)
timeout 600 python -m pytest tests/test_gpu_net.py tests/test_cli.py -q > gpurun_out/net_t.log 2>&1; tail -1 gpurun_out/net_t.log

for lib in base alt_libs/old base alt_libs/old; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  echo "$lib:"; BNN_LIB=$L timeout 300 python tools/net_latency.py --reps 1000 2>&1 | tail -2 | python -c "
import sys,json
for line in sys.stdin:
    a,j=line.split(' ',1); d=json.loads(j); print(' ',a,'net kernel',d['net_zero_copy']['kernels_only_us'],'server',d['server']['median_us'], 'eq', d['outputs_equal'])"
done
