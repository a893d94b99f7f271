"""Device time of the fused front-end launch alone (CUDA events, B images): python tools/front_time.py [--arch] [--batch]"""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2301_05126_b200 as P
from paper_2301_05126_b200 import native
from paper_2301_05126_b200.engine import Engine, FrontOp

ap = argparse.ArgumentParser()
ap.add_argument("--arch", default="cifar10")
ap.add_argument("--batch", type=int, default=32768)
args = ap.parse_args()
m = P.export_synthetic_model(args.arch, 1 if args.arch == "cifar10" else 7)
x = torch.from_numpy(P.make_images(m, args.batch, 3).astype(np.uint8)).cuda()
with Engine(device=0) as eng:
    pm = eng.prepare(m)
    op = pm.ops[0]
    assert isinstance(op, FrontOp)
    outs, _ = pm.buffers(args.batch)
    for _ in range(3):
        op.launch(pm.lib, x, outs[0], None, args.batch, native.stream_handle())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        op.launch(pm.lib, x, outs[0], None, args.batch, native.stream_handle())
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 10
print(f"front {args.arch} B={args.batch}: {ms:.4f} ms  ({ms / args.batch * 1e6:.2f} ns/img)")
