"""Summarise a tools/front_trace.py capture (clock64 timeline of CTA 0 of the fused front end).

roles: 0 MMA-L2, 1 epilogue-L2, 2 MMA-L1, 3 epilogue-L1; stamps (start, ready/loaded, issued/done)."""
import sys
import numpy as np
t = np.load(sys.argv[1]).astype(np.int64)
names = ["MMA-L2", "EPI-L2", "MMA-L1", "EPI-L1a", "BUILD0", "BUILD1", "LOADX", "EPI-L1b"]
t0 = min(int(r[0]) for role in t for r in role if r[0] > 0)
for role in range(len(t)):
    rows = t[role][t[role][:, 0] > 0]
    if not len(rows):
        continue
    wait = rows[:, 1] - rows[:, 0]
    work = rows[:, 2] - rows[:, 1]
    per = np.diff(rows[:, 0])
    print(f"{names[role]:7} items {len(rows):4}  wait med {int(np.median(wait)):6}  work med {int(np.median(work)):6}  "
          f"period med {int(np.median(per)) if len(per) else 0:6}  span {int(rows[-1, 2] - rows[0, 0])}")
show = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for role in range(len(t)):
    rows = t[role][t[role][:, 0] > 0]
    for i, r in enumerate(rows[:show]):
        print(names[role], i, r[0] - t0, r[1] - r[0], r[2] - r[1])
