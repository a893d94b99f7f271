# A/B: number of H buffers (first-layer outputs in flight) in the fused front end
for lib in base alt_libs/h3 alt_libs/h3a42 alt_libs/h4; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  for a in cifar10 fashion; do echo -n "$lib $a: "; BNN_LIB=$L python tools/front_time.py --arch $a --batch 65536 | tail -1; done
done
BNN_LIB=alt_libs/h3/libbnn.so timeout 300 python -m pytest -q -x tests/test_gpu_front.py 2>&1 | tail -1
