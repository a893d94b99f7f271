"""HBM roofline of the standalone layout / step / pool kernels (csrc/layout.cu): algorithmic
bytes (input + output, each touched once) / CUDA-event time, against the measured HBM copy bandwidth.

    python tools/layout_bench.py [--batch 2048] [--out profiles/r2_layout_hbm.json]

Shape: CIFAR L2's activation (64 x 32 x 32) over B images -- inputs far larger than L2."""
import argparse, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2301_05126_b200 import native

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8192)
ap.add_argument("--out", default="gpurun_out/layout_hbm.json")
args = ap.parse_args()
B, C, H, W = args.batch, 64, 32, 32
peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {}
hbm = float(peaks.get("hbm_gbs", 6550.0))
lib = native.device_ready(0)
p = native.ptr
st = lambda: native.stream_handle()
dev = "cuda"
n = B * C * H * W
CW = C // 32
bits = torch.randint(-2**31, 2**31 - 1, (B * H * W * CW,), dtype=torch.int32, device=dev)
ref = torch.randint(-2**62, 2**62, ((n + 63) // 64,), dtype=torch.int64, device=dev)
f4 = torch.empty((B * H * W * C // 2,), dtype=torch.uint8, device=dev)
ints = torch.randint(-300, 300, (n,), dtype=torch.int32, device=dev)
thr = torch.randint(-20, 20, (C,), dtype=torch.int32, device=dev)
pos = torch.tensor([0x5555AAAA, 0x0F0F00FF], dtype=torch.int64).to(torch.int32).to(dev)
o_bits = torch.empty_like(bits)
o_ref = torch.empty_like(ref)
o_int = torch.empty((n // 4,), dtype=torch.int32, device=dev)
o_bits_pool = torch.empty((B * (H // 2) * (W // 2) * CW,), dtype=torch.int32, device=dev)
lib.bnn_bits_to_f4(p(bits), B * H * W, C, p(f4), st())
cases = {
    "bnn_bits_ref_to_nhwc": (lambda: lib.bnn_bits_ref_to_nhwc(p(ref), B, C, H, W, p(o_bits), st()), ref.numel() * 8 + bits.numel() * 4),
    "bnn_bits_nhwc_to_ref": (lambda: lib.bnn_bits_nhwc_to_ref(p(bits), B, C, H, W, p(o_ref), st()), bits.numel() * 4 + ref.numel() * 8),
    "bnn_step_ref": (lambda: lib.bnn_step_ref(p(ints), B, C, H * W, p(thr), p(pos), p(o_ref), st()), n * 4 + ref.numel() * 8),
    "bnn_step_nhwc": (lambda: lib.bnn_step_nhwc(p(ints), B, C, H, W, p(thr), p(pos), p(o_bits), st()), n * 4 + bits.numel() * 4),
    "bnn_maxpool_int": (lambda: lib.bnn_maxpool_int(p(ints), B, C, H, W, p(o_int), st()), n * 4 + n),
    "bnn_maxpool_bits_nhwc": (lambda: lib.bnn_maxpool_bits_nhwc(p(bits), B, C, H, W, p(o_bits_pool), st()), bits.numel() * 4 + o_bits_pool.numel() * 4),
    "bnn_bits_to_f4": (lambda: lib.bnn_bits_to_f4(p(bits), B * H * W, C, p(f4), st()), bits.numel() * 4 + f4.numel()),
    "bnn_f4_to_bits": (lambda: lib.bnn_f4_to_bits(p(f4), B * H * W, C, p(o_bits), st()), f4.numel() + bits.numel() * 4),
}
res = {"shape": [B, C, H, W], "hbm_peak_gbs": hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if peaks else "fallback 6550", "kernels": {}}
for name, (fn, nbytes) in cases.items():
    for _ in range(3):
        native.check(fn(), name)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    reps = 10
    for _ in range(reps):
        native.check(fn(), name)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    gbs = nbytes / ms / 1e6
    res["kernels"][name] = {"ms": round(ms, 4), "bytes": int(nbytes), "gb_s": round(gbs, 1), "frac": round(gbs / hbm, 3)}
    print(f"{name:26} {ms:8.4f} ms  {gbs:8.1f} GB/s  {gbs / hbm:.3f} of HBM", flush=True)
Path(args.out).parent.mkdir(parents=True, exist_ok=True)
Path(args.out).write_text(json.dumps(res, indent=1))
