"""Per-tile detail of a tc_trace.py capture: python tools/trace_tiles.py gpurun_out/tc_trace_b3.npy [stages_per_tile] [first_tile]"""
import sys

import numpy as np

t = np.load(sys.argv[1]).astype(np.int64)
spt = int(sys.argv[2]) if len(sys.argv) > 2 else 9
i0 = int(sys.argv[3]) if len(sys.argv) > 3 else 10
base = t[2][i0][0]
for i in range(i0, i0 + 5):
    mt, ep = t[2][i], t[3][i]
    st = t[1][spt * i:spt * i + spt]
    print(f"tile {i}: MMA tempty wait {mt[0]-base}->{mt[1]-base}  stages(start,ready,issued): " +
          " ".join(f"({s[0]-base},{s[1]-s[0]},{s[2]-s[1]})" for s in st))
    print(f"        EPI wait {ep[0]-base}->{ep[1]-base} drained {ep[3]-base} done {ep[2]-base}")
