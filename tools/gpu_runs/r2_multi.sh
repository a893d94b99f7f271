python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/plan_time.py --batch 262144 --reps 5 --plan '{"2": [1, 0, 6]}'
python tools/tc_trace.py --block 2 --batch 9472 --variant "[1,0,6]" 2>&1 | head -5
