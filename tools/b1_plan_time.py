"""Batch-1 CUDA-graph latency under given variant plans (zero-copy replay, host wall clock, median of
N replays):  python tools/b1_plan_time.py '<plan JSON>' ['<plan JSON>' ...]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2301_05126_b200 as P
from paper_2301_05126_b200 import tuner
from paper_2301_05126_b200.engine import Engine

m = P.export_synthetic_model("cifar10", 1)
one = P.make_images(m, 1, 45)
with Engine() as eng:
    table = tuner.profile_model(eng, m, one, [1], warmups=2, reps=5)
    base = tuner.select_plan(table, m).variant_map()
    plans = [("tuned", base)]
    for arg in sys.argv[1:]:
        over = {int(k): tuple(v) for k, v in json.loads(arg).items()}
        plans.append((arg, {**base, **over}))
    plans.append(("tuned+fused-front", base))
    for name, plan in plans * 2:
        eng.prepare(m, plan).front_min_batch = 1 if name.endswith("fused-front") else 10 ** 9
        g = eng.graph(m, batch=1, variants=plan, zero_copy=True)
        for _ in range(50):
            g.replay(one)
        ts = []
        for _ in range(1000):
            t0 = time.perf_counter_ns()
            g.replay(one)
            ts.append(time.perf_counter_ns() - t0)
        print(json.dumps({"plan": name, "median_us": round(float(np.median(ts)) / 1e3, 2),
                          "kernels_only_us": round(g.kernels_only_us(), 2)}))
