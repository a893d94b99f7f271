for e in 3 4 5; do BNN_NVCC_FLAGS="-DFRONT_EXP=$e" python -m paper_2301_05126_b200.csrc.build --force > /dev/null 2>&1; echo "exp $e: $(python tools/front_time.py 2>&1 | tail -1)"; done
