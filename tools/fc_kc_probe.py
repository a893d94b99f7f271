"""Fashion FC (3,136 -> 2,048, + step) at B = 65,536 through bnn_tc_fc: the real length (32-B K chunks)
vs zero-padded lengths whose rows are 64-B / 128-B multiples (larger TMA boxes / K chunks)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2301_05126_b200 import native

lib = native.device_ready(0)
B, M = 65536, 2048
thr = torch.zeros(M, dtype=torch.int32, device="cuda")
pos = torch.full((M // 32,), -1, dtype=torch.int32, device="cuda")
for L in (3136, 3200, 3328, 4096):
    x = torch.randint(0, 256, (B, L // 2), dtype=torch.uint8, device="cuda") & 0x88 | 0x22
    w = torch.randint(0, 256, (M, L // 2), dtype=torch.uint8, device="cuda") & 0x88 | 0x22
    out = torch.empty((B, M // 2), dtype=torch.uint8, device="cuda")
    v = native.Variant.make(1, 0, 0)
    f = lambda: native.check(lib.bnn_tc_fc(native.ptr(x), B, L, native.ptr(w), M, native.ptr(thr), native.ptr(pos), 1,
                                          native.ptr(out), None, None, v, native.stream_handle()))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        f()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"L={L}: {ms:.4f} ms  ({ms * 3136 / L:.4f} ms scaled to 3,136 useful)")
