# A/B: step MMA (D += c) after the last tap instead of first (alt_libs/se) -- L5 HX time + parity
for r in 1 2; do
for lib in base alt_libs/se; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  echo -n "$lib: "; BNN_LIB=$L python tools/plan_time.py --batch 262144 --reps 5 --plan '{"2": [1, 0, 6]}' 2>&1 | tail -1
done
done
BNN_LIB=alt_libs/se/libbnn.so timeout 900 python -m pytest tests/test_gpu_model.py -q -x 2>&1 | tail -1
BNN_LIB=alt_libs/se/libbnn.so python tools/tc_trace.py --block 2 --batch 9472 --variant "[1,0,6]" 2>&1 | head -5
