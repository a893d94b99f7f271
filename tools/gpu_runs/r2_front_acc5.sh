# front end accumulator / E-ring depth A/B (alt builds in alt_libs/)
for r in 1 2; do for a in fashion cifar10; do
  echo "base $a: $(python tools/front_time.py --arch $a --batch 65536)"
  echo "acc1=5,ering=5 $a: $(BNN_LIB=alt_libs/libbnn_a5.so python tools/front_time.py --arch $a --batch 65536)"
  echo "acc2=3 $a: $(BNN_LIB=alt_libs/libbnn_h2.so python tools/front_time.py --arch $a --batch 65536)"
done; done
