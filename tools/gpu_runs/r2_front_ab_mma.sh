# A/B: original front kernel + one-block 9-tap MMA issue (in-tree) vs the v5 redesign + the same MMA issue
timeout 600 python -m pytest -x -q tests/test_gpu_front.py 2>&1 | tail -1
BNN_LIB=alt_libs/v5/libbnn.so timeout 600 python -m pytest -x -q tests/test_gpu_front.py 2>&1 | tail -1
for lib in base alt_libs/v5; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  for a in cifar10 fashion; do echo -n "$lib "; BNN_LIB=$L timeout 120 python tools/front_time.py --arch $a --batch 65536; done
done
