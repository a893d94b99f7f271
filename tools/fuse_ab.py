"""Whole-plan device time with the fused front end on vs off (B images, default tensor plan):
python tools/fuse_ab.py [--arch cifar10|fashion] [--batch N]"""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2301_05126_b200 as P
from paper_2301_05126_b200.engine import Engine

ap = argparse.ArgumentParser()
ap.add_argument("--arch", default="fashion")
ap.add_argument("--batch", type=int, default=65536)
args = ap.parse_args()
m = P.export_synthetic_model(args.arch, 1 if args.arch == "cifar10" else 7)
x = torch.from_numpy(P.make_images(m, args.batch, 3).astype(np.uint8)).cuda()
with Engine(device=0) as eng:
    pm = eng.prepare(m)
    for fuse in (True, False, True, False):
        pm.set_fuse_front(fuse)
        ops = pm.exec_ops(x)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in ops]
        for _ in range(3):
            pm.infer(x)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            pm.infer(x, events=ev)
            torch.cuda.synchronize()
            ts.append([a.elapsed_time(b) for a, b in ev])
        t = np.median(np.array(ts), axis=0)
        print(f"{args.arch} B={args.batch} fuse={fuse}: total {t.sum():.4f} ms  per op " +
              " ".join(f"{o.name}={v:.4f}" for o, v in zip(ops, t)))
