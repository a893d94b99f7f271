# sensitivity probe of the fused front end: +300 clk in one stage (d1 loader per image, d2 MMA-L1, d3 EPI-L1,
# d4 MMA-L2, d5 EPI-L2 per tile); the stage whose delay moves the total is on the critical path
for lib in base alt_libs/d1 alt_libs/d2 alt_libs/d3 alt_libs/d4 alt_libs/d5 base; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  for a in fashion cifar10; do
    echo -n "$lib "; BNN_LIB=$L timeout 120 python tools/front_time.py --arch $a --batch 65536 2>&1 | tail -1
  done
done
