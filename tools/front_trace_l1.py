"""Per-tile view of the L1 pipeline in a tools/front_trace.py capture: builder (E tile built),
MMA-L1 (wait E rows / wait accumulator / issued), epilogue-L1, and the loader's per-image stamps."""
import sys

import numpy as np

t = np.load(sys.argv[1]).astype(np.int64)
i0 = int(sys.argv[2]) if len(sys.argv) > 2 else 20
base = t[2][i0][0]
for c in range(i0, i0 + 12):
    m, e = t[2][c], t[3][c]
    print(f"L1 tile {c}: built {e[3]-base:7d} | MMA wait-start {m[0]-base:7d} E-ready {m[3]-base:7d} acc-free {m[1]-base:7d} "
          f"issued {m[2]-base:7d} | EPI wait {e[0]-base:7d} got {e[1]-base:7d} (w11 {t[1][c][3]-base:7d}) done {e[2]-base:7d}")
ld = t[0][:, 3]
ld = ld[ld > 0]
if len(ld) > 1:
    print("loader per-image period med", int(np.median(np.diff(ld))))
b = t[3][:, 3]
b = b[b > 0]
print("builder per-tile period med", int(np.median(np.diff(b))))
