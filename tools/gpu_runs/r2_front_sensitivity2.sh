# the same probe with __nanosleep(200 ns) (takes no issue slots from co-resident warps): n1 loader, n3 EPI-L1, n5 EPI-L2
for lib in base alt_libs/n1 alt_libs/n3 alt_libs/n5 base; do
  if [ $lib = base ]; then L=""; else L=$lib/libbnn.so; fi
  for a in fashion cifar10; do
    echo -n "$lib "; BNN_LIB=$L timeout 120 python tools/front_time.py --arch $a --batch 65536 2>&1 | tail -1
  done
done
