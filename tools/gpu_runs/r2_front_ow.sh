# front end: one accumulator waiter per epilogue group (named-barrier sleepers) vs every warp spinning
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_front.py -q -x 2>&1 | tail -1
for r in 1 2; do for a in cifar10 fashion; do
  echo "new $a: $(python tools/front_time.py --arch $a --batch 65536)"
  echo "old $a: $(BNN_LIB=alt_libs/libbnn_ow0.so python tools/front_time.py --arch $a --batch 65536)"
done; done
