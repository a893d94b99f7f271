"""Clock64 timeline of CTA 0 of one tc_block launch (debug instrument): block --block of the CIFAR
model at --batch images, unfused plan.   python tools/tc_trace.py --block 2 --batch 4736"""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2301_05126_b200 import native
from paper_2301_05126_b200.engine import Engine
from paper_2301_05126_b200.synthetic import export_synthetic_model, make_images

ap = argparse.ArgumentParser()
ap.add_argument("--block", type=int, default=2)
ap.add_argument("--batch", type=int, default=148 * 32)
ap.add_argument("--variant", default="", help="JSON [engine, tile_n, tile_q] for the traced block")
args = ap.parse_args()
m = export_synthetic_model("cifar10", 1)
with Engine(device=0) as eng:
    import json
    pm = eng.prepare(m, {args.block: tuple(json.loads(args.variant))} if args.variant else None)
    pm.set_fuse_front(False)
    x = torch.from_numpy(make_images(m, args.batch, 5).astype(np.uint8)).cuda()
    pm.infer(x)
    torch.cuda.synchronize()
    outs, _ = pm.buffers(args.batch, ops=pm.units)
    op = pm.units[args.block]
    src = outs[args.block - 1]
    buf = torch.zeros(4 * 512 * 4, dtype=torch.int64, device="cuda")
    op.launch(pm.lib, src, outs[args.block], None, args.batch, native.stream_handle())
    torch.cuda.synchronize()
    native.check(pm.lib.bnn_tc_trace(native.ptr(buf)))
    op.launch(pm.lib, src, outs[args.block], None, args.batch, native.stream_handle())
    torch.cuda.synchronize()
    native.check(pm.lib.bnn_tc_trace(None))
    t = buf.cpu().numpy().reshape(4, 512, 4).astype(np.int64)
np.save(f"gpurun_out/tc_trace_b{args.block}.npy", t)
names = ["TMA", "MMA-stage", "MMA-tile", "EPI"]
t0 = min(int(r[0]) for role in t for r in role if r[0] > 0)
for role in range(4):
    rows = t[role][t[role][:, 0] > 0]
    if not len(rows):
        continue
    w = rows[:, 1] - rows[:, 0]
    print(f"{names[role]:9} n {len(rows):4} wait med {int(np.median(w)):6} p90 {int(np.percentile(w, 90)):6}"
          + (f" work med {int(np.median(rows[:, 2] - rows[:, 1])):6}" if rows[:, 2].any() else "")
          + f" period med {int(np.median(np.diff(rows[:, 0]))) if len(rows) > 1 else 0}")
rows = t[3][t[3][:, 0] > 0]
if rows[:, 3].any():
    print("EPI drain med", int(np.median(rows[:, 3] - rows[:, 1])), "process med", int(np.median(rows[:, 2] - rows[:, 3])))
for role in range(4):
    rows = t[role][t[role][:, 0] > 0]
    print(names[role], [(int(r[0] - t0), int(r[1] - r[0]), int(r[2] - r[1]) if r[2] else 0) for r in rows[:14]])
