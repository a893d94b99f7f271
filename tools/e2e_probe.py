"""Where does Engine.run_model's end-to-end time go?  python tools/e2e_probe.py"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2301_05126_b200 as P
from paper_2301_05126_b200.engine import Engine

m = P.export_synthetic_model("cifar10", 1)
n = 262144
host = torch.from_numpy(P.make_images(m, 4096, 3).astype(np.uint8)).repeat(n // 4096, 1, 1, 1).pin_memory()
with Engine(device=0) as eng:
    pm = eng.prepare(m)
    x = host.cuda()
    pm.infer(x); torch.cuda.synchronize()
    t0 = time.perf_counter(); pm.infer(x); torch.cuda.synchronize(); print("device infer 262144:", (time.perf_counter() - t0) * 1e3, "ms")
    t0 = time.perf_counter(); y = host.cuda(non_blocking=True); torch.cuda.synchronize(); print("H2D 805 MB:", (time.perf_counter() - t0) * 1e3, "ms")
    for bs in (32768, 65536, 131072, 16384, 32768):
        eng.run_model(m, host, batch_size=bs)
        t0 = time.perf_counter(); r = eng.run_model(m, host, batch_size=bs); dt = time.perf_counter() - t0
        print(f"run_model bs={bs}: {dt * 1e3:.1f} ms  -> {n / dt / 1e6:.3f} M img/s; compute sum {sum(r.compute_ns) / 1e6:.1f} ms")
