# A/B: accumulator split of the fused front end: ACC2 = 1 (the L2 MMA warp queues at most one tile ahead of
# its epilogue, so first-layer MMAs wait behind fewer second-layer MMAs), ACC1 = 6
for r in 1 2; do
  for lib in base alt_libs/c21 alt_libs/c61; do
    if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
    for a in cifar10 fashion; do
      echo -n "$lib $a: "; BNN_LIB=$L python tools/front_time.py --arch $a --batch 65536 2>&1 | tail -1
    done
  done
done
for lib in alt_libs/c21 alt_libs/c61; do BNN_LIB=$lib/libbnn.so timeout 300 python -m pytest -q -x tests/test_gpu_front.py 2>&1 | tail -1; done
