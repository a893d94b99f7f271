#!/usr/bin/env python
"""Per-block kernel-variant sweep (BASELINE configs[4]): profile_model + select_plan on the GPU.

    python tools/tune.py --arch cifar10 --batches 1 64 4096 --out profiles/r1_tune_cifar10

Writes <out>_table.json (every (block, variant, batch) cell, CUDA-event medians),
<out>_plan.json (plan format v2, bound to the model digest and the device) and
prints a summary of the per-batch winners.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="cifar10", choices=["cifar10", "fashion"])
    ap.add_argument("--batches", type=int, nargs="+", default=[1, 64, 4096])
    ap.add_argument("--warmups", type=int, default=2)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    from paper_2301_05126_b200 import tuner
    from paper_2301_05126_b200.engine import Engine
    from paper_2301_05126_b200.synthetic import export_synthetic_model, make_images

    seed = 1 if args.arch == "cifar10" else 7
    model = export_synthetic_model(args.arch, seed)
    images = make_images(model, min(max(args.batches), 4096), 2026)
    with Engine() as eng:
        table = tuner.profile_model(eng, model, images, args.batches, args.warmups, args.reps)
        plan = tuner.select_plan(table, model)
        per = tuner.per_batch_assignments(table, model)
        pm = eng.prepare(model)
        names = [op.name for op in pm.units]
    summary = {
        "arch": args.arch, "device": table.meta.device, "batches": args.batches,
        "chosen_batch": plan.batch_size, "predicted_ns_per_image": plan.predicted_per_image_ns(),
        "plan": {f"{i}:{names[i]}": list(v) for i, v in plan.variants.items()},
        "per_batch": {str(b): {f"{i}:{names[i]}": list(v) for i, v in a.items()} for b, a in per.items()},
        "per_batch_total_us": {str(b): round(sum(table.get(i, k, b).total_ns for i, k in a.items()) / 1e3, 2)
                               for b, a in per.items()},
    }
    print(json.dumps(summary, indent=1))
    if args.out:
        Path(args.out + "_table.json").write_text(json.dumps(tuner.table_to_doc(table), indent=1) + "\n")
        tuner.save_plan(plan, args.out + "_plan.json")
        Path(args.out + "_summary.json").write_text(json.dumps(summary, indent=1) + "\n")


if __name__ == "__main__":
    main()
