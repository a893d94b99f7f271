"""Time every tensor-engine variant of every block at one batch (device time per launch, CUDA graphs).

    python tools/layer_sweep.py [--arch cifar10] [--batch 32768] [--blocks 2 3]

A focused view of the autotuner's cells (tuner.profile_model) for kernel work: prints
ms per launch and the block's FP4 tensor-rate fraction for each candidate variant.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="cifar10")
    ap.add_argument("--batch", type=int, default=32768)
    ap.add_argument("--blocks", type=int, nargs="*", default=None)
    ap.add_argument("--variants", default="", help='JSON list of [engine, tile_n, tile_q] (default: tuner candidates)')
    args = ap.parse_args()
    import numpy as np

    from paper_2301_05126_b200 import native, tuner
    from paper_2301_05126_b200.engine import Engine
    from paper_2301_05126_b200.synthetic import export_synthetic_model, make_images

    m = export_synthetic_model(args.arch, 1 if args.arch == "cifar10" else 7)
    imgs = make_images(m, 256, 2026)
    extra = [tuple(v) for v in json.loads(args.variants)] if args.variants else None
    if extra:  # time exactly these candidates on tensor-capable blocks
        base = tuner.candidate_variants
        tuner.candidate_variants = lambda op, batch: extra if op.tc_ok() else base(op, batch)
    with Engine() as eng:
        table = tuner.profile_model(eng, m, imgs, [args.batch], warmups=2, reps=3, engines=(native.ENGINE_TC,))
        pm = eng.prepare(m)
        out = {}
        for (blk, key, b), e in sorted(table.entries.items()):
            if args.blocks and blk not in args.blocks:
                continue
            u = pm.units[blk]
            work = sum(u.work_per_image().values()) * b
            ms = e.compute_ns / 1e6
            frac = 2 * work / (ms / 1e3) / 1e12 / 6618.0
            out.setdefault(f"{blk}:{u.name}", {})[str(list(key))] = {"ms": round(ms, 4), "frac_fp4": round(frac, 3)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
