"""Time the CPU port (oracle/np_route.py) against the reference's own ``bnntuner.reference_infer``.

Runs only in the build container, where /root/reference exists (it is imported read-only from
/root/reference/pkg/src).  The GPU box has no reference, so bench.py times the port; this file
records, on one host, how close the port's time is to the reference's on every CPU-baseline
workload (fashion B=1 seed 123, CIFAR B=1 seed 45, fashion B=1,024,
CIFAR B=256 seed 2026; BLAS threads = all cores and 1), and that both give identical logits.

    python tools/cpu_port_calibration.py [--out profiles/r2_cpu_port_vs_reference.json]
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")


def cpu_model() -> str:
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def timeit(fn, calls: int):
    fn()
    ts = []
    for _ in range(calls):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), float(np.min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(REPO / "profiles" / "r2_cpu_port_vs_reference.json"))
    ap.add_argument("--calls", type=int, default=50)
    args = ap.parse_args()
    from threadpoolctl import threadpool_limits

    import bnntuner as R
    from oracle import np_route

    cores = os.cpu_count() or 1
    rows = []
    cases = [("fashion", 7, 1, 123, args.calls), ("cifar10", 1, 1, 45, args.calls),
             ("fashion", 7, 1024, 2026, 3), ("cifar10", 1, 256, 2026, 3)]
    for arch, mseed, batch, iseed, calls in cases:
        model = R.export_synthetic_model(arch, mseed)
        imgs = np.random.default_rng(iseed).integers(0, 256, size=(batch,) + tuple(model.input.shape))
        it = R.IntTensor(imgs.shape, imgs)
        port = np_route.PreparedModel(model)
        ref_l, ref_p = R.reference_infer(model, it)
        pl, pp = port.infer(imgs)
        same = bool(np.array_equal(ref_l.values, pl) and list(ref_p) == pp.tolist())
        for threads in (cores, 1):
            with threadpool_limits(limits=threads, user_api="blas"):
                rmed, rmin = timeit(lambda: R.reference_infer(model, it), calls)
                pmed, pmin = timeit(lambda: port.infer(imgs), calls)
            row = {"arch": arch, "batch": batch, "image_seed": iseed, "blas_threads": threads, "calls": calls,
                   "reference_median_ms": round(rmed * 1e3, 3), "reference_min_ms": round(rmin * 1e3, 3),
                   "port_median_ms": round(pmed * 1e3, 3), "port_min_ms": round(pmin * 1e3, 3),
                   "port_over_reference": round(pmed / rmed, 3), "identical_logits": same}
            print(json.dumps(row), flush=True)
            rows.append(row)
    doc = {"host_cpu": cpu_model(), "cores": cores, "numpy": np.__version__,
           "what": "bnntuner.reference_infer (imported from /root/reference/pkg/src) vs oracle/np_route.py on the "
                   "BASELINE.md section 2 CPU workloads; median/min wall time per call",
           "rows": rows}
    Path(args.out).write_text(json.dumps(doc, indent=1) + "\n")


if __name__ == "__main__":
    main()
