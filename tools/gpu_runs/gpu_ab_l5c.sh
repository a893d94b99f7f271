python tools/tc_trace.py --block 2 --batch 32768 --variant "[1,0,3]" 2>&1 | head -5
(cd _ab_split && python tools/tc_trace.py --block 2 --batch 32768 --variant "[1,0,3]" 2>&1 | head -5)
