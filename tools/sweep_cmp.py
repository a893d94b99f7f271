"""Compare layer_sweep JSON outputs: python tools/sweep_cmp.py a.json b.json ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception:
        print(f, "ERR", open(f).read()[-800:])
        continue
    print(f, {k.split(":")[0]: {v: d[k][v]["ms"] for v in d[k] if v in ("[1, 0, 0]", "[1, 0, 1]", "[1, 0, 3]")} for k in d})
