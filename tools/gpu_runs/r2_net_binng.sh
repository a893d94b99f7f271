# A/B: one-launch kernel's conv_bin units: heuristic tap groups (base) vs forced whole positions (bn1) / 3 groups (bn3)
for lib in base alt_libs/bn1 alt_libs/bn3 base alt_libs/bn1 alt_libs/bn3; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  echo "$lib:"; BNN_LIB=$L timeout 300 python tools/net_latency.py --reps 500 2>&1 | tail -2 | python -c "
import sys,json
for line in sys.stdin:
    a,j=line.split(' ',1); d=json.loads(j); print(' ',a,'net kernel',d['net_zero_copy']['kernels_only_us'],'server',d['server']['median_us'])"
done
for lib in alt_libs/bn1 alt_libs/bn3; do BNN_LIB=$lib/libbnn.so timeout 600 python -m pytest tests/test_gpu_net.py -q 2>&1 | tail -1; done
