"""Summarise an ncu source page (SASS) export: instructions / stall samples / shared-memory wavefronts
per image, the mbarrier spin loops, and the hottest address buckets.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_sass_summary.py src.csv --images 32768 [--bucket 0x200] [--top 25]
"""
import argparse
import csv
import re
from collections import OrderedDict

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--images", type=int, default=1)
ap.add_argument("--bucket", type=lambda x: int(x, 0), default=0x200)
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--lines", default="", help="hex address range lo:hi to print line by line")
args = ap.parse_args()
rows = list(csv.reader(open(args.csv)))
h, data = rows[1], rows[2:]
iE, iS = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
iW = h.index("L1 Wavefronts Shared")
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
n = args.images
lines = [(int(r[0], 16), r[1].strip(), int(r[iE] or 0), int(r[iS] or 0), int(r[iW] or 0), r) for r in data]
print(f"instr/img {sum(x[2] for x in lines) / n:.0f}  stall samples {sum(x[3] for x in lines)}  "
      f"smem wavefronts/img {sum(x[4] for x in lines) / n:.0f}")
idx = {a: i for i, (a, *_r) in enumerate(lines)}
spin = 0
for i, (a, t, e, s, w, r) in enumerate(lines):
    m = re.search(r"BRA 0x([0-9a-f]+)", t)
    if m and t.startswith("@!P0"):
        tgt = int(m.group(1), 16)
        if tgt < a and a - tgt < 0x300 and tgt in idx:
            blk = lines[idx[tgt]:i + 1]
            if any("TRYWAIT" in x[1] for x in blk):
                k = sum(x[2] for x in blk)
                spin += k
                print(f"  spin loop @{a & 0xfffff:05x}: {k / n:.0f} instr/img")
print(f"spin total {spin / n:.0f} instr/img")
b = OrderedDict()
for a, t, e, s, w, r in lines:
    k = (a // args.bucket) * args.bucket
    if k not in b:
        b[k] = [0, 0, 0, t[:60]]
    b[k][0] += e
    b[k][1] += s
    b[k][2] += w
print("bucket   instr/img  samples  smem_wf/img  first instruction")
for k, (e, s, w, t) in sorted(b.items(), key=lambda kv: -kv[1][1])[:args.top]:
    print(f"{k & 0xfffff:05x} {e / n:10.0f} {s:8d} {w / n:10.0f}   {t}")
if args.lines:
    lo, hi = (int(x, 16) for x in args.lines.split(":"))
    for a, t, e, s, w, r in lines:
        if lo <= (a & 0xfffff) < hi:
            det = " ".join(f"{c[6:]}={r[h.index(c)]}" for c in stall_cols if r[h.index(c)] not in ("0", ""))
            print(f"{a & 0xfffff:05x} {s:5d} {e / n:7.1f} {t[:64]:64s} {det}")
