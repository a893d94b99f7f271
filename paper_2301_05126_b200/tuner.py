"""Per-block kernel-variant autotuner behind the reference's configuration-search API.

The reference searches a layer -> {CPU, X, Y, Z, XY, XZ, YZ, XYZ} mapping
with wall-clock medians (`bnntuner/profiler.py:98-164`, Algorithm 1 in
`bnntuner/mapper.py:64-107`).  On the GPU the analogous decision is, per
fused block, which kernel variant runs it: the integer-pipe popcount kernel
(tile widths) or the tcgen05 FP4 tensor-core kernel (N tile), i.e. "popc vs
MMA", "tile", "threads", "pack width" (bits vs FP4 operand format) of the
north star.  Same entry points, same semantics:

* ``profile_layer`` / ``profile_model``: W discarded warm-ups + R timed reps,
  medians, relative-spread warning (``UnstableMeasurement``), one table cell
  per (block, variant, batch).  Timing is CUDA events on the launching
  stream, so the measurement is the kernel, not Python dispatch.
* ``per_batch_assignments`` / ``select_plan``: greedy per-block argmin at
  every batch, then the batch with the least per-image total (smaller batch
  on ties).  Determinism under timing noise: candidates have a fixed rank and
  a challenger must beat the incumbent by more than ``WIN_MARGIN`` -- the
  reference's host-clock ties made its ``tune`` non-deterministic.

Per-block independence (the reference's exactness argument, mapper.py:1-8)
holds because every producer epilogue can emit either operand format at the
same cost, so a block's choice never constrains its neighbours; each cell is
timed with its input already in the format its engine reads.
"""

from __future__ import annotations

import json
import platform
import time
import warnings
from dataclasses import dataclass, field
from pathlib import Path
from statistics import median

import numpy as np

from . import native
from .errors import BadRange, IncompleteTable, ModelHashMismatch, ParseError, UnsupportedVersion
from .model import model_digest

DEFAULT_WARMUPS = 2
DEFAULT_REPS = 5
SPREAD_WARN = 0.5
WIN_MARGIN = 0.03
MAX_BATCH_EXP = 20
PLAN_FORMAT_VERSION = 2

Variant = native.Variant


class UnstableMeasurement(UserWarning):
    """A profiled cell showed more run-to-run spread than SPREAD_WARN (profiler.py:33-34)."""


@dataclass(frozen=True)
class ProfileEntry:
    """profiler.py:37-47."""

    overhead_ns: float
    compute_ns: float
    reps: int
    spread: float

    @property
    def total_ns(self) -> float:
        return self.overhead_ns + self.compute_ns


@dataclass(frozen=True)
class ProfileMeta:
    model_hash: str
    device: str
    host: str
    timestamp: str
    warmups: int
    reps: int
    batch_sizes: tuple


@dataclass(eq=False)
class ProfileTable:
    """Cells keyed (block index, variant key, batch) -> ProfileEntry (profiler.py:60-91)."""

    entries: dict = field(default_factory=dict)
    candidates: dict = field(default_factory=dict)  # block -> [variant key] in rank order (all batches)
    meta: ProfileMeta | None = None
    by_batch: dict = field(default_factory=dict)  # (block, batch) -> [variant key]: the candidates AT that batch

    def get(self, block: int, key: tuple, batch: int) -> ProfileEntry:
        return self.entries[(block, tuple(key), batch)]

    def candidates_at(self, block: int, batch: int) -> list:
        """Rank-ordered candidates of ``block`` at ``batch`` (some variants are only candidates at
        small batches, e.g. the FC GEMV at batch <= 8)."""
        return self.by_batch.get((block, batch), self.candidates[block])

    def missing_cells(self, batch_sizes) -> list:
        out = []
        for blk in self.candidates:
            for b in batch_sizes:
                for k in self.candidates_at(blk, b):
                    if (blk, tuple(k), b) not in self.entries:
                        out.append((blk, tuple(k), b))
        return out


@dataclass(eq=False)
class ExecPlan:
    """Per-block variant assignment + batch size (mapper.py:25-54), bound to the model digest
    and to the device it was tuned on."""

    model_name: str
    model_hash: str
    batch_size: int
    variants: dict  # block index -> (engine, tile_n, tile_q)
    predicted_total_ns: float | None
    device: str = ""
    workers: int = 1

    def variant_map(self) -> dict:
        return {int(k): tuple(v) for k, v in self.variants.items()}

    def predicted_per_image_ns(self):
        return None if self.predicted_total_ns is None else self.predicted_total_ns / self.batch_size

    def same_mapping(self, other: "ExecPlan") -> bool:
        return (self.model_hash == other.model_hash and self.batch_size == other.batch_size
                and self.variant_map() == other.variant_map())


def batch_sweep(lower_exp: int, upper_exp: int) -> list:
    """Powers of two 2**lo .. 2**hi (mapper.py:57-61; upper bound raised to 2**20 for the GPU)."""
    if not 0 <= lower_exp <= upper_exp <= MAX_BATCH_EXP:
        raise BadRange(f"need 0 <= lower <= upper <= {MAX_BATCH_EXP}, got ({lower_exp}, {upper_exp})")
    return [2 ** e for e in range(lower_exp, upper_exp + 1)]


def candidate_variants(op, batch: int) -> list:
    """Ranked candidate variant keys (engine, tile_n, tile_q) for one fused block."""
    from .engine import POPC, TC

    kind = op.variant_kind
    cands = []
    if kind is None:
        return [(POPC, 0, 0)]
    if op.tc_ok():
        if kind == "conv_bin" and op.step_mma_ok():
            # first = the incumbent a challenger must beat by WIN_MARGIN: the step-in-the-MMA kernel
            # is never slower in principle (one extra MMA per tile instead of an add per channel),
            # and where its geometry applies HX (one pair of halo-along-x TMA boxes per filter row)
            # measured 6-9 % faster still at full batch
            if op.W == 16 and op.C == 64 and op.H % 8 == 0:
                cands += [(TC, 0, 6)]
            cands += [(TC, 0, 3)]
        cands += [(TC, 0, 0), (TC, 128, 0), (TC, 64, 0)]
        if batch <= 64:  # latency-bound: narrower N tiles spread a layer's filters over more SMs
            cands += [(TC, 32, 0)]
        if kind in ("conv_bin", "fc_bin"):
            cands += [(TC, 0, 5)]  # single-CTA kernels where N = 256 tiles would otherwise run on CTA pairs
        if kind == "conv_bin":
            cands += [(TC, 0, 1)]  # per-tap TMA boxes instead of the halo-reuse kernel
            cands += [(TC, 0, 2)]  # halo-reuse kernel even where its M tiling wastes rows

    if kind == "conv_first":
        cands += [(POPC, 0, 0)]
    elif kind == "conv_bin":
        cands += [(POPC, 64, 0), (POPC, 32, 0), (POPC, 128, 0)]
    elif kind == "fc_bin":
        if batch <= 8:
            cands += [(POPC, 0, -1)]
        cands += [(POPC, 64, 0), (POPC, 128, 0)]
    else:
        cands += [(POPC, 0, 0)]
    seen, out = set(), []
    for c in cands:
        if c not in seen:
            seen.add(c)
            out.append(c)
    return out


def host_description() -> str:
    return f"{platform.platform()} / {platform.processor() or 'unknown cpu'}"


# --------------------------------------------------------------------------- measurement


def _median_entry(samples_ns: list, overheads_ns: list | None = None, label: str = "") -> ProfileEntry:
    med = median(samples_ns)
    spread = (max(samples_ns) - min(samples_ns)) / med if med > 0 else 0.0
    if spread > SPREAD_WARN:
        warnings.warn(f"unstable cell {label}: spread {spread:.2f}", UnstableMeasurement, stacklevel=3)
    ovh = float(median(overheads_ns)) if overheads_ns else 0.0
    return ProfileEntry(ovh, float(med), len(samples_ns), float(spread))


def profile_layer(engine, layer, rep_input, config=None, batch_size=None, warmups: int = DEFAULT_WARMUPS,
                  reps: int = DEFAULT_REPS) -> ProfileEntry:
    """Median (overhead, compute) of one single-layer GPU call (profiler.py:98-120)."""
    if reps < 1:
        raise ValueError("reps must be >= 1")
    for _ in range(warmups):
        engine.execute_layer(layer, rep_input, config, batch_size)
    comp, ovh = [], []
    for _ in range(reps):
        r = engine.execute_layer(layer, rep_input, config, batch_size)
        comp.append(r.compute_ns)
        ovh.append(r.overhead_ns)
    tot = [c + o for c, o in zip(comp, ovh)]
    e = _median_entry(tot, None, f"(layer {getattr(layer.kind, 'value', layer.kind)}, batch={batch_size})")
    return ProfileEntry(float(median(ovh)), float(median(comp)), reps, e.spread)


GRAPH_LAUNCHES = 8  # launches captured per timing graph


def _time_block(pm, i, key, x_in, out, B, warmups, reps, stream) -> list:
    """Device time (ns per launch) of block i under variant ``key`` on prepared inputs.

    The launches are captured in a CUDA graph and timed with events around the
    replay, so host-side enqueue latency (ctypes + launch, ~10 us) never enters
    the measurement -- essential at batch 1, where the kernels themselves take a
    few microseconds.  Each rep = one replay of GRAPH_LAUNCHES back-to-back launches.
    """
    torch = pm.torch
    from .engine import TC

    op = pm.units[i]
    saved = (op.variant, op.engine)
    op.variant = native.Variant.make(*key)
    op.engine = TC if key[0] == TC and op.tc_ok() else 0
    try:
        side = torch.cuda.Stream(pm.dev)
        with torch.cuda.stream(side):
            for _ in range(max(1, warmups)):  # also sets kernel attributes outside the capture
                op.launch(pm.lib, x_in, out, None, B, native.stream_handle())
        side.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for _ in range(GRAPH_LAUNCHES):
                op.launch(pm.lib, x_in, out, None, B, native.stream_handle())
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e6 / GRAPH_LAUNCHES)
        del g
        return ts
    finally:
        op.variant, op.engine = saved


def profile_model(engine, model, images, batch_sizes, warmups: int = DEFAULT_WARMUPS,
                  reps: int = DEFAULT_REPS, engines=None) -> ProfileTable:
    """Every (block, candidate variant, batch) cell (profiler.py:123-154).

    The input of block i is the dataset's first ``batch`` images (tiled if the
    dataset is smaller) propagated through blocks 0..i-1 on the GPU, in both
    operand formats, so every candidate is timed on identical data.
    ``engines``: optional subset of engine ids (e.g. ``(native.ENGINE_TC,)``) to
    restrict the candidates -- large-batch throughput tuning skips the popc cells.
    """
    torch = engine.torch
    vals = np.asarray(images.values if hasattr(images, "values") else images)
    if vals.shape[0] < 1:
        raise ValueError("profiling needs a nonempty dataset sample")
    batch_sizes = sorted({int(b) for b in batch_sizes})
    pm = engine.prepare(model, {})
    fuse_saved = pm.fuse_front
    pm.set_fuse_front(False)  # cells are the planning units; their inputs come from the unfused chain
    try:
        table = _profile_cells(engine, pm, model, vals, batch_sizes, warmups, reps, engines)
    finally:
        pm.set_fuse_front(fuse_saved)
    return table


def _profile_cells(engine, pm, model, vals, batch_sizes, warmups, reps, engines=None) -> ProfileTable:
    torch = engine.torch
    table = ProfileTable()
    st = native.stream_handle()
    lib = pm.lib
    with torch.cuda.device(engine.device):
        for B in batch_sizes:
            reps_needed = -(-B // vals.shape[0])
            imgs = np.concatenate([vals] * reps_needed)[:B]
            x = torch.from_numpy(imgs.astype(np.uint8)).to(pm.dev)
            pm.infer(x)
            outs, _ = pm.buffers(B)
            torch.cuda.synchronize()
            for i, op in enumerate(pm.units):
                cands = candidate_variants(op, B)
                if engines is not None:
                    cands = [c for c in cands if c[0] in engines] or cands
                table.by_batch[(i, B)] = [tuple(c) for c in cands]
                # union over the sweep in rank order (batches ascend, so small-batch-only variants keep
                # their rank); selection at batch B only looks at that batch's own list
                merged = table.candidates.setdefault(i, [])
                merged += [tuple(c) for c in cands if tuple(c) not in merged]
                if i == 0:
                    src = {"img": x}
                else:
                    prev = outs[i - 1]
                    src = {pm.units[i - 1].out_fmt: prev}
                    if op.src.kind == "bits":
                        C, H, W = op.src.nhwc_dims()
                        npix = B * H * W
                        if "bits" not in src and C % 32 == 0:
                            t = torch.empty((B, op.src.words_per_image), dtype=torch.int32, device=pm.dev)
                            native.check(lib.bnn_f4_to_bits(native.ptr(prev), npix, C, native.ptr(t), st))
                            src["bits"] = t
                        if "f4" not in src and C % 64 == 0:
                            t = torch.empty((B, op.src.elems_per_image // 2), dtype=torch.uint8, device=pm.dev)
                            native.check(lib.bnn_bits_to_f4(native.ptr(prev), npix, C, native.ptr(t), st))
                            src["f4"] = t
                out = op.out_alloc(torch, B, pm.dev)
                for key in cands:
                    fmt = "img" if i == 0 else ("f4" if key[0] == 1 and op.tc_ok() else "bits")
                    if fmt not in src:
                        continue
                    ts = _time_block(pm, i, key, src[fmt], out, B, warmups, reps, st)
                    table.entries[(i, tuple(key), B)] = _median_entry(ts, None, f"(block {i} {op.name} {key} B={B})")
    table.meta = ProfileMeta(
        model_hash=model_digest(model), device=_device_name(torch, engine.device), host=host_description(),
        timestamp=time.strftime("%Y-%m-%dT%H:%M:%S%z"), warmups=warmups, reps=reps, batch_sizes=tuple(batch_sizes))
    return table


def _device_name(torch, dev) -> str:
    p = torch.cuda.get_device_properties(dev)
    return f"{p.name} ({p.multi_processor_count} SMs, sm_{p.major}{p.minor})"


# --------------------------------------------------------------------------- selection


def _argmin(table: ProfileTable, blk: int, b: int):
    keys = [k for k in table.candidates_at(blk, b) if (blk, tuple(k), b) in table.entries]
    best = keys[0]
    best_t = table.get(blk, best, b).total_ns
    for k in keys[1:]:
        t = table.get(blk, k, b).total_ns
        if t < best_t * (1.0 - WIN_MARGIN):
            best, best_t = k, t
    return tuple(best), best_t


def per_batch_assignments(table: ProfileTable, model=None) -> dict:
    """Winning variant per block at every batch (mapper.py:64-84)."""
    bs = table.meta.batch_sizes
    empty = [(blk, b) for blk in table.candidates for b in bs
             if not any((blk, tuple(k), b) in table.entries for k in table.candidates_at(blk, b))]
    if empty:
        raise IncompleteTable(empty)
    return {b: {blk: _argmin(table, blk, b)[0] for blk in sorted(table.candidates)} for b in bs}


def select_plan(table: ProfileTable, model) -> ExecPlan:
    """Greedy mapping at the per-image-optimal batch (mapper.py:87-107); smaller batch on ties."""
    per = per_batch_assignments(table, model)
    totals = {b: sum(table.get(blk, k, b).total_ns for blk, k in assign.items()) for b, assign in per.items()}
    chosen = min(totals, key=lambda b: (totals[b] / b, b))
    return ExecPlan(model_name=model.name, model_hash=table.meta.model_hash, batch_size=chosen,
                    variants={blk: tuple(k) for blk, k in per[chosen].items()},
                    predicted_total_ns=totals[chosen], device=table.meta.device)


# --------------------------------------------------------------------------- persistence (plan format v2)


def plan_to_doc(plan: ExecPlan) -> dict:
    return {"format_version": PLAN_FORMAT_VERSION, "model_name": plan.model_name, "model_hash": plan.model_hash,
            "batch_size": plan.batch_size, "device": plan.device,
            "predicted_total_ns": plan.predicted_total_ns,
            "variants": {str(k): list(v) for k, v in sorted(plan.variants.items())}}


def save_plan(plan: ExecPlan, path) -> None:
    Path(path).write_text(json.dumps(plan_to_doc(plan), sort_keys=True, indent=2) + "\n")


def load_plan(path, model=None) -> ExecPlan:
    try:
        doc = json.loads(Path(path).read_text())
    except json.JSONDecodeError as e:
        raise ParseError(f"{path}: line {e.lineno}: {e.msg}") from e
    if doc.get("format_version") != PLAN_FORMAT_VERSION:
        raise UnsupportedVersion(f"{path}: format_version {doc.get('format_version')!r}, "
                                 f"expected {PLAN_FORMAT_VERSION}")
    plan = ExecPlan(model_name=doc["model_name"], model_hash=doc["model_hash"], batch_size=int(doc["batch_size"]),
                    variants={int(k): tuple(v) for k, v in doc["variants"].items()},
                    predicted_total_ns=doc.get("predicted_total_ns"), device=doc.get("device", ""))
    if model is not None and model_digest(model) != plan.model_hash:
        raise ModelHashMismatch(f"{path}: plan was tuned for model {plan.model_hash[:12]}, "
                                f"not {model_digest(model)[:12]}")
    return plan


def table_to_doc(table: ProfileTable) -> dict:
    return {
        "format_version": PLAN_FORMAT_VERSION,
        "meta": None if table.meta is None else {**table.meta.__dict__, "batch_sizes": list(table.meta.batch_sizes)},
        "candidates": {str(k): [list(c) for c in v] for k, v in table.candidates.items()},
        "candidates_by_batch": {f"{blk}@{b}": [list(c) for c in v] for (blk, b), v in sorted(table.by_batch.items())},
        "cells": [{"block": blk, "variant": list(key), "batch": b, "overhead_ns": e.overhead_ns,
                   "compute_ns": e.compute_ns, "reps": e.reps, "spread": e.spread}
                  for (blk, key, b), e in sorted(table.entries.items())],
    }
