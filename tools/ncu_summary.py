#!/usr/bin/env python
"""Summarise ncu captures into the markdown tables committed under profiles/.

    python tools/ncu_summary.py full  gpurun_out/x.ncu-rep      # --set full capture -> per-kernel table
    python tools/ncu_summary.py launches gpurun_out/launches.csv # launch list -> per-kernel time shares
    python tools/ncu_summary.py traffic gpurun_out/x.ncu-rep 32768 # per-launch DRAM bytes (bench "traffic")

The full-capture table reports, per profiled launch: duration, DRAM bytes read+written
(the roofline "traffic"), L2 / DRAM throughput, tensor-pipe and issue utilisation.
"""

from __future__ import annotations

import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    ("gpu__time_duration.sum", "ms"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue %"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
    ("sm__cycles_elapsed.avg.per_second", "SM GHz"),
]


def short(name: str) -> str:
    name = re.sub(r"\(CUtensorMap_st.*", "", name)
    name = re.sub(r"\(const unsigned char.*", "", name)
    name = re.sub(r"^void ", "", name)
    return name.replace("bnn::", "")


def full(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    cols = [(hdr.index(m), label, units[hdr.index(m)]) for m, label in FULL_METRICS if m in hdr]
    kn = hdr.index("Kernel Name")
    out = ["| kernel | " + " | ".join(f"{lab} ({u})" if u else lab for _, lab, u in cols) + " |",
           "|---|" + "---|" * len(cols)]
    for r in data:
        out.append("| " + short(r[kn]) + " | " + " | ".join(r[i] for i, _, _ in cols) + " |")
    return "\n".join(out)


def launches(path: str) -> str:
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        try:
            v = float(r[mv].replace(",", ""))
        except ValueError:
            continue
        k = short(r[kn])
        tot[k] += v
        cnt[k] += 1
    grand = sum(tot.values())
    out = ["| kernel | launches | total | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| {k} | {cnt[k]} | {v:.4g} | {v / grand * 100:.1f}% |")
    return "\n".join(out)


def traffic(path: str, images: int) -> dict:
    """Per profiled launch (in order): kernel, ms, DRAM bytes read + written, and per image."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kn = hdr.index("Kernel Name")

    def val(r, m):
        i = hdr.index(m)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1, "us": 1e-3,
                 "ns": 1e-6}.get(units[i], 1)
        return float(r[i].replace(",", "")) * scale

    out = []
    for r in data:
        tot = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        out.append({"kernel": short(r[kn]), "ms": val(r, "gpu__time_duration.sum"), "dram_bytes": tot,
                    "dram_bytes_per_image": tot / images,
                    "tensor_pct": float(r[hdr.index("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")])})
    return {"images_per_launch": images, "launches": out}


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "traffic":
        import json

        print(json.dumps(traffic(path, int(sys.argv[3])), indent=1))
    else:
        print(full(path) if mode == "full" else launches(path))
