# A/B: suspend-time-hint waits in the fused front end (BNN_FRONT_SLEEP=1: epilogue/loader waits, =2: all)
for r in 1 2; do
for lib in base alt_libs/s1 alt_libs/s2; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  for a in cifar10 fashion; do
    echo -n "$lib $a: "; BNN_LIB=$L python tools/front_time.py --arch $a --batch 65536 | tail -1
  done
done
done
for lib in alt_libs/s1 alt_libs/s2; do
  BNN_LIB=$lib/libbnn.so timeout 300 python -m pytest -q -x tests/test_gpu_front.py 2>&1 | tail -1
done
