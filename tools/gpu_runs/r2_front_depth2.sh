# A/B after the loader change: 5 L1 accumulators / 4 H buffers (alt_libs builds)
for r in 1 2; do
for lib in base alt_libs/a5 alt_libs/h4 alt_libs/a5h4; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  for a in cifar10 fashion; do
    echo -n "$lib $a: "; BNN_LIB=$L python tools/front_time.py --arch $a --batch 65536 | tail -1
  done
done
done
for lib in alt_libs/a5 alt_libs/h4 alt_libs/a5h4; do
  BNN_LIB=$lib/libbnn.so timeout 300 python -m pytest -q -x tests/test_gpu_front.py 2>&1 | tail -1
done
