"""Batch-1 request latency: per-block kernel graph vs the one-launch network kernel (NetPlan).

    python tools/net_latency.py [--reps 1000] [--grid 0]

Host wall clock per request (graph replay + stream sync), zero-copy and copy graphs, plus the
device time of the kernels alone; outputs checked equal across the paths."""
import argparse, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2301_05126_b200 as P
from paper_2301_05126_b200.engine import Engine, GraphRunner, NetPlan

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=1000)
ap.add_argument("--grid", type=int, default=0)
args = ap.parse_args()


def lat(g, one, reps):
    for _ in range(50):
        g.replay(one)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        g.replay(one)
        ts.append(time.perf_counter_ns() - t0)
    ts = np.array(ts) / 1e3
    return {"median_us": round(float(np.median(ts)), 2), "p99_us": round(float(np.percentile(ts, 99)), 2),
            "min_us": round(float(ts.min()), 2), "kernels_only_us": round(g.kernels_only_us(200), 2)}


res = {}
with Engine() as eng:
    for arch, seed, iseed in (("fashion", 7, 123), ("cifar10", 1, 45)):
        m = P.export_synthetic_model(arch, seed)
        one = np.random.default_rng(iseed).integers(0, 256, size=(1,) + tuple(m.input.shape)).astype(np.uint8)
        pm = eng.prepare(m)
        r = {}
        outs = {}
        for name, zc, net in (("blocks_zero_copy", True, False), ("net_zero_copy", True, True),
                              ("net_copy", False, True)):
            g = GraphRunner(pm, 1, zero_copy=zc, net=net)
            if net and args.grid:
                g.net.grid = args.grid
            outs[name] = g.replay(one)
            r[name] = lat(g, one, args.reps)
            r[name]["launches"] = g.launches
        with eng.serve(m, batch=1) as srv:
            o = srv.infer(one)
            for _ in range(50):
                srv.infer(one)
            ts = []
            for _ in range(args.reps):
                t0 = time.perf_counter_ns()
                srv.infer(one)
                ts.append(time.perf_counter_ns() - t0)
            ts = np.array(ts) / 1e3
            r["server"] = {"median_us": round(float(np.median(ts)), 2), "p99_us": round(float(np.percentile(ts, 99)), 2),
                           "min_us": round(float(ts.min()), 2), "launches": 0}
            outs["server"] = o
        base = outs["blocks_zero_copy"]
        r["outputs_equal"] = all(np.array_equal(base[0], o[0]) and np.array_equal(base[1], o[1]) for o in outs.values())
        r["net_smem_bytes"] = NetPlan(pm, 1).smem
        res[arch] = r
        print(arch, json.dumps(r), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/net_latency.json").write_text(json.dumps(res, indent=1))
