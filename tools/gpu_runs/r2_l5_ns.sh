# L5: HX with N = 128 tiles sharing each A load (tile_q 7) vs HX N = 256 (tile_q 6): parity + time
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_model.py -q -x -k "variants or calibrated" 2>&1 | tail -1
for r in 1 2; do
python tools/plan_time.py --batch 262144 --reps 5 --plan '{"2": [1, 0, 6]}' 2>&1 | tail -2
python tools/plan_time.py --batch 262144 --reps 5 --plan '{"2": [1, 0, 7]}' 2>&1 | tail -2
done
python tools/tc_trace.py --block 2 --batch 9472 --variant "[1,0,7]" 2>&1 | head -6
