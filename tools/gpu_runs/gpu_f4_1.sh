timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "Error|error|assert|FAIL|passed|failed|mismatch" | head -30
