"""Feasibility probe for split-K at batch 1: latency of one bnn_tc_conv (8x8, K = 512 outputs, pool)
with the full 512 input channels vs 1/8 of them (64), per launch in a chain of 20 graph-captured launches."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2301_05126_b200 import native

lib = native.device_ready(0)
for (C, H, K, pool, tn) in ((512, 8, 512, 1, 64), (64, 8, 512, 1, 64), (256, 16, 256, 1, 64), (32 * 2, 16, 256, 1, 64),
                            (256, 8, 512, 0, 32), (64, 8, 512, 0, 32)):
    B = 1
    x = (torch.randint(0, 256, (B, H, H, C // 2), dtype=torch.uint8, device="cuda") & 0x88) | 0x22
    w = (torch.randint(0, 256, (K, 9 * C // 2), dtype=torch.uint8, device="cuda") & 0x88) | 0x22
    thr = torch.zeros(K, dtype=torch.int32, device="cuda")
    pos = torch.full((K // 32,), -1, dtype=torch.int32, device="cuda")
    out = torch.empty((B * (H // 2 if pool else H) ** 2 * K // 2,), dtype=torch.uint8, device="cuda")
    v = native.Variant.make(1, tn, 0)
    v.flags = native.VARIANT_STATIC_WEIGHTS
    s = torch.cuda.Stream()
    def go():
        native.check(lib.bnn_tc_conv(native.ptr(x), B, C, H, H, native.ptr(w), K, native.ptr(thr), native.ptr(pos), pool, 1,
                                     native.ptr(out), None, v, s.cuda_stream))
    with torch.cuda.stream(s):
        go(); go()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            go()
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        g.replay()
    b.record(); b.synchronize()
    print(f"C={C} H={H} K={K} pool={pool} tile_n={tn}: {a.elapsed_time(b) * 1e3 / 400:.2f} us per launch")
