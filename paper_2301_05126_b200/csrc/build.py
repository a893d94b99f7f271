"""Build libbnn.so in-tree: nvcc for sm_100a only (no other arch, no JIT cache).

    python -m paper_2301_05126_b200.csrc.build [--force] [--verbose]

Output: paper_2301_05126_b200/libbnn.so (git-ignored; travels to the GPU box
with the gpurun snapshot).  Sources: every *.cu in this directory.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys
from pathlib import Path

CSRC = Path(__file__).resolve().parent
PKG = CSRC.parent
REPO = PKG.parent
# BNN_BUILD_OUT / BNN_BUILD_OBJ: build an experiment variant elsewhere (with BNN_NVCC_FLAGS=-D...)
LIB = Path(os.environ.get("BNN_BUILD_OUT") or PKG / "libbnn.so")
OBJ = Path(os.environ.get("BNN_BUILD_OBJ") or REPO / "build" / "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"] + os.environ.get("BNN_NVCC_FLAGS", "").split()  # extra flags for experiments


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(CSRC.glob("*.cu"))


def headers():
    return sorted(CSRC.glob("*.cuh")) + [REPO / "include" / "bnn.h"]


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    hdr_mtime = max(p.stat().st_mtime for p in headers())
    objs = []
    procs = []
    for src in sources():
        obj = OBJ / (src.stem + ".o")
        objs.append(obj)
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr_mtime):
            cmd = [nvcc(), *ARCH, *FLAGS, "-I", str(REPO / "include"), "-I", str(CSRC), "-c", str(src),
                   "-o", str(obj)]
            if verbose:
                cmd += ["-Xptxas", "-v"]
                print(" ".join(cmd), flush=True)
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if out.strip() and (verbose or p.returncode):
            print(out, file=sys.stderr)
        if p.returncode:
            failed = True
            print(f"nvcc failed on {src.name}", file=sys.stderr)
    if failed:
        raise RuntimeError("libbnn build failed")
    if force or procs or not LIB.exists():
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
        subprocess.run(cmd, check=True)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    print(build(args.force, args.verbose))


if __name__ == "__main__":
    main()
