"""Race / determinism stress: the same large batch inferred repeatedly under a given plan must give
bit-identical logits every time.   python tools/determinism.py [--reps 10] [--batch 262144]"""
import argparse
import hashlib
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2301_05126_b200 as P
from paper_2301_05126_b200.engine import Engine

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--batch", type=int, default=262144)
ap.add_argument("--plan", default='{"2": [1, 0, 6], "3": [1, 0, 0], "4": [1, 0, 0], "5": [1, 0, 0], "6": [1, 0, 0]}')
args = ap.parse_args()
m = P.export_synthetic_model("cifar10", 1)
x = torch.from_numpy(P.make_images(m, 4096, 9).astype(np.uint8)).repeat(args.batch // 4096, 1, 1, 1).cuda()
plan = {int(k): tuple(v) for k, v in json.loads(args.plan).items()}
digests = set()
with Engine(device=0) as eng:
    pm = eng.prepare(m, plan)
    for _ in range(args.reps):
        logits, preds = pm.infer(x)
        torch.cuda.synchronize()
        digests.add(hashlib.sha256(logits.cpu().numpy().tobytes() + preds.cpu().numpy().tobytes()).hexdigest())
print(json.dumps({"reps": args.reps, "batch": args.batch, "plan": args.plan, "distinct_outputs": len(digests)}))
sys.exit(0 if len(digests) == 1 else 1)
