"""Per-op device times of the fused plan under given variants (CUDA events, B images):
python tools/plan_time.py [--batch 262144] [--plan JSON] [--reps 5]"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2301_05126_b200 as P
from paper_2301_05126_b200.engine import Engine

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=262144)
ap.add_argument("--plan", default="{}")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
m = P.export_synthetic_model("cifar10", 1)
x = torch.from_numpy(P.make_images(m, 4096, 9).astype(np.uint8)).repeat(args.batch // 4096, 1, 1, 1).cuda()
plan = {int(k): tuple(v) for k, v in json.loads(args.plan).items()}
with Engine(device=0) as eng:
    pm = eng.prepare(m, plan)
    for _ in range(3):
        pm.infer(x)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in pm.ops]
          for _ in range(args.reps)]
    torch.cuda.synchronize()
    for k in range(args.reps):
        pm.infer(x, events=ev[k])
    torch.cuda.synchronize()
    ms = [float(np.median([ev[k][i][0].elapsed_time(ev[k][i][1]) for k in range(args.reps)])) for i in range(len(pm.ops))]
    print(json.dumps({"plan": args.plan, "pitch": getattr(pm.ops[0], "pitch", None), "total_ms": round(sum(ms), 3),
                      "ops": {f"{i}:{o.name}": round(t, 4) for i, (o, t) in enumerate(zip(pm.ops, ms))}}))
