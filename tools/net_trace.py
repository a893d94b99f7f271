"""Per-block timeline of the one-launch network kernel (globaltimer stamps of every CTA; debug).

    python tools/net_trace.py [--batch 1]

Per block: when the last CTA passed the barrier, median staging (activations + filter wait) and item
time, and when the last CTA finished its items -- all in ns from the first CTA's filter-copy issue."""
import argparse, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2301_05126_b200 as P
from paper_2301_05126_b200 import native
from paper_2301_05126_b200.engine import Engine, NetPlan

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
args = ap.parse_args()
out = {}
with Engine() as eng:
    for arch, seed in (("fashion", 7), ("cifar10", 1)):
        m = P.export_synthetic_model(arch, seed)
        pm = eng.prepare(m)
        net = NetPlan(pm, args.batch)
        x = torch.from_numpy(P.make_images(m, args.batch, 5).astype(np.uint8)).cuda()
        lg = torch.zeros((args.batch, 10), dtype=torch.int32, device="cuda")
        pr = torch.zeros((args.batch,), dtype=torch.int32, device="cuda")
        for _ in range(20):
            net.launch(x, lg, pr)
        G = torch.cuda.get_device_properties(0).multi_processor_count
        buf = torch.zeros((G, 64), dtype=torch.int64, device="cuda")
        native.check(pm.lib.bnn_net_trace(native.ptr(buf)))
        rows = []
        for _ in range(5):
            buf.zero_()
            net.launch(x, lg, pr)
            torch.cuda.synchronize()
            rows.append(buf.cpu().numpy().copy())
        native.check(pm.lib.bnn_net_trace(None))
        t = rows[-1].astype(np.int64)
        t0 = t[:, 0][t[:, 0] > 0].min()
        res = {"start_spread_ns": int(t[:, 0][t[:, 0] > 0].max() - t0),
               "copies_issued_med_ns": int(np.median(t[:, 1] - t[:, 0]))}
        for l in range(len(pm.units)):
            ev = t[:, 2 + 3 * l: 5 + 3 * l]
            ok = ev[:, 0] > 0
            if not ok.any():
                continue
            e = ev[ok] - t0
            blk = {"ctas": int(ok.sum()), "barrier_last_ns": int(e[:, 0].max()), "barrier_first_ns": int(e[:, 0].min())}
            if (e[:, 1] > 0).any():
                blk["stage_med_ns"] = int(np.median(e[:, 1] - e[:, 0]))
                blk["items_med_ns"] = int(np.median(e[:, 2] - e[:, 1]))
            blk["done_last_ns"] = int(e[:, 2].max())
            res[f"{l}:{pm.units[l].name}"] = blk
        clk = {}
        for l in range(min(6, len(pm.units))):
            c = t[:, 40 + 4 * l: 44 + 4 * l]
            ok = (c[:, 0] > 0) & (c[:, 1] > 0)
            if ok.any():
                c = c[ok]
                clk[str(l)] = {"units_clk_med": int(np.median(c[:, 1] - c[:, 0])), "units_clk_max": int((c[:, 1] - c[:, 0]).max()),
                               "sync_clk_med": int(np.median(np.where(c[:, 2] > 0, c[:, 2] - c[:, 1], 0))),
                               "epi_clk_med": int(np.median(np.where(c[:, 3] > c[:, 2], c[:, 3] - np.maximum(c[:, 2], c[:, 1]), 0)))}
        res["warp0_clocks"] = clk
        out[arch] = res
        print(arch, json.dumps(res, indent=1), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/net_trace.json").write_text(json.dumps(out, indent=1))
