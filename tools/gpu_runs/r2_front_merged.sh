# A/B: one MMA issuer for both front-end layers with first-layer priority (in-tree) vs two issuing warps (alt_libs/m0)
timeout 600 python -m pytest -x -q tests/test_gpu_front.py 2>&1 | tail -1
for r in 1 2; do
  for lib in base alt_libs/m0; do
    if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
    for a in cifar10 fashion; do
      echo -n "$lib $a: "; BNN_LIB=$L timeout 120 python tools/front_time.py --arch $a --batch 65536 2>&1 | tail -1
    done
  done
done
