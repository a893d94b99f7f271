"""Steady-state per-image periods of each fused front-end stage from a tools/front_trace.py capture:
    python tools/front_periods.py gpurun_out/front_trace_fashion.npy T1 T2
roles: 0 MMA-L2 (+ field 3: loader, per image), 1 EPI-L2, 2 MMA-L1, 3 EPI-L1; stamps (start, ready, done)."""
import sys
import numpy as np

t = np.load(sys.argv[1]).astype(np.int64)
T1, T2 = int(sys.argv[2]), int(sys.argv[3])


def per_image(starts, per):
    s = starts[starts > 0]
    n = len(s) // per
    if n < 4:
        return None
    img = s[: n * per].reshape(n, per)[:, 0]
    d = np.diff(img)[n // 4:]  # skip the pipeline fill
    return int(np.median(d))


print("loader  image period", per_image(t[0][:, 3], 1))
print("MMA-L1  image period", per_image(t[2][:, 0], T1), " ready-wait med", int(np.median((t[2][:, 1] - t[2][:, 0])[t[2][:, 0] > 0])))
print("EPI-L1  image period", per_image(t[3][:, 0], T1), " wait med", int(np.median((t[3][:, 1] - t[3][:, 0])[t[3][:, 0] > 0])),
      " work med", int(np.median((t[3][:, 2] - t[3][:, 1])[t[3][:, 0] > 0])))
print("MMA-L2  image period", per_image(t[0][:, 0], T2), " wait med", int(np.median((t[0][:, 1] - t[0][:, 0])[t[0][:, 0] > 0])))
print("EPI-L2  image period", per_image(t[1][:, 0], T2), " wait med", int(np.median((t[1][:, 1] - t[1][:, 0])[t[1][:, 0] > 0])))
# EPI-L1 per image: from its first tile start to the next image's first tile start, split into the tiles and the boundary
s3 = t[3][t[3][:, 0] > 0]
n = len(s3) // T1
if n >= 4:
    r = s3[: n * T1].reshape(n, T1, 4)
    tiles = (r[:, -1, 2] - r[:, 0, 0])[n // 4:]
    gap = (r[1:, 0, 0] - r[:-1, -1, 2])[n // 4:]
    print("EPI-L1  tiles span med", int(np.median(tiles)), " image-boundary gap med", int(np.median(gap)))
