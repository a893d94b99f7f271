# A/B: 16 instead of 8 epilogue warps in the tcgen05 block / pair kernels (alt_libs/e16): per-op times of the tuned plan
P='{"0": [1, 0, 0], "1": [1, 0, 0], "2": [1, 0, 6], "3": [1, 0, 0], "4": [1, 0, 2], "5": [1, 0, 0], "6": [1, 0, 0], "7": [1, 0, 0]}'
for r in 1 2; do
  for lib in base alt_libs/e16; do
    if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
    echo -n "$lib: "; BNN_LIB=$L timeout 300 python tools/plan_time.py --batch 262144 --reps 5 --plan "$P" 2>&1 | tail -1
  done
done
BNN_LIB=alt_libs/e16/libbnn.so timeout 900 python -m pytest tests/test_gpu_model.py -q -x 2>&1 | tail -1
