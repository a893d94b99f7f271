"""Clock64 timeline of CTA 0 of the fused front-end kernel (debug instrument; not a benchmark).

    python tools/front_trace.py [--arch cifar10|fashion] [--batch N]
"""
import argparse, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2301_05126_b200 as P
from paper_2301_05126_b200 import native
from paper_2301_05126_b200.engine import Engine, FrontOp

ap = argparse.ArgumentParser()
ap.add_argument("--arch", default="cifar10")
ap.add_argument("--batch", type=int, default=148 * 8)
args = ap.parse_args()
m = P.export_synthetic_model(args.arch, 1 if args.arch == "cifar10" else 7)
imgs = torch.from_numpy(P.make_images(m, args.batch, 3).astype(np.uint8)).cuda()
with Engine(device=0) as eng:
    pm = eng.prepare(m)
    op = pm.ops[0]
    assert isinstance(op, FrontOp)
    pm.infer(imgs)
    torch.cuda.synchronize()
    buf = torch.zeros(8 * 512 * 4, dtype=torch.int64, device="cuda")
    native.check(pm.lib.bnn_tc_front_trace(native.ptr(buf)))
    pm.infer(imgs)
    torch.cuda.synchronize()
    native.check(pm.lib.bnn_tc_front_trace(None))
    t = buf.cpu().numpy().reshape(8, 512, 4).astype(np.int64)
Path("gpurun_out").mkdir(exist_ok=True)
np.save(f"gpurun_out/front_trace_{args.arch}.npy", t)
print("saved", t.shape)
