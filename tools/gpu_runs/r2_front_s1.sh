# front end: first-layer tiles shared with the second-layer epilogue group (s1 per image), A/B over s1
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_front.py -q -x 2>&1 | tail -1
BNN_FRONT_S1=2 timeout 600 python -m pytest tests/test_gpu_front.py -q -x 2>&1 | tail -1
for a in fashion cifar10; do for s in default 0 1 2 3 4; do
  if [ $s = default ]; then echo "$a s1=default: $(python tools/front_time.py --arch $a --batch 65536)";
  else echo "$a s1=$s: $(BNN_FRONT_S1=$s python tools/front_time.py --arch $a --batch 65536)"; fi
done; done
