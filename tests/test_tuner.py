"""Autotuner selection logic on hand-built tables (mirrors the reference's tests/test_mapper.py)."""

import itertools

import numpy as np
import pytest

import paper_2301_05126_b200 as P
from paper_2301_05126_b200 import tuner
from paper_2301_05126_b200.tuner import ExecPlan, ProfileEntry, ProfileMeta, ProfileTable

POPC64, POPC32, TC0 = (0, 64, 0), (0, 32, 0), (1, 0, 0)


def table(cells: dict, candidates: dict, batches) -> ProfileTable:
    t = ProfileTable()
    t.candidates = {k: list(v) for k, v in candidates.items()}
    for (blk, key, b), ns in cells.items():
        t.entries[(blk, key, b)] = ProfileEntry(0.0, float(ns), 5, 0.0)
    t.meta = ProfileMeta("h" * 64, "dev", "host", "now", 2, 5, tuple(batches))
    return t


def test_batch_sweep():
    assert tuner.batch_sweep(0, 3) == [1, 2, 4, 8]
    with pytest.raises(P.BadRange):
        tuner.batch_sweep(3, 2)
    with pytest.raises(P.BadRange):
        tuner.batch_sweep(0, 21)


def test_hand_example_and_per_image_batch_choice(fashion_model):
    cands = {0: [POPC64], 1: [TC0, POPC64], 2: [TC0, POPC64]}
    cells = {
        (0, POPC64, 1): 10, (0, POPC64, 4): 20,
        (1, TC0, 1): 50, (1, POPC64, 1): 30, (1, TC0, 4): 40, (1, POPC64, 4): 90,
        (2, TC0, 1): 5, (2, POPC64, 1): 6, (2, TC0, 4): 8, (2, POPC64, 4): 7.9,
    }
    t = table(cells, cands, [1, 4])
    per = tuner.per_batch_assignments(t)
    assert per[1] == {0: POPC64, 1: POPC64, 2: TC0}
    assert per[4] == {0: POPC64, 1: TC0, 2: TC0}  # 7.9 does not beat 8 by the 3 % margin
    plan = tuner.select_plan(t, fashion_model)
    assert plan.batch_size == 4 and plan.predicted_total_ns == 68.0  # 68/4 = 17 < 45/1


def test_brute_force_optimal_without_margin(fashion_model, monkeypatch):
    monkeypatch.setattr(tuner, "WIN_MARGIN", 0.0)
    rng = np.random.default_rng(0)
    keys = [TC0, POPC64, POPC32]
    for _ in range(50):
        nblk, batches = 4, [1, 2, 8]
        cells = {(blk, k, b): float(rng.integers(1, 1000)) for blk in range(nblk) for k in keys for b in batches}
        t = table(cells, {blk: keys for blk in range(nblk)}, batches)
        plan = tuner.select_plan(t, fashion_model)
        best = min(((sum(cells[(blk, c[blk], b)] for blk in range(nblk)) / b, b)
                    for b in batches for c in itertools.product(keys, repeat=nblk)))
        assert plan.predicted_total_ns / plan.batch_size == best[0]


def test_ties_prefer_rank_then_smaller_batch(fashion_model):
    cands = {0: [TC0, POPC64]}
    t = table({(0, TC0, 1): 10, (0, POPC64, 1): 10, (0, TC0, 2): 20, (0, POPC64, 2): 20}, cands, [1, 2])
    plan = tuner.select_plan(t, fashion_model)
    assert plan.variants == {0: TC0} and plan.batch_size == 1


def test_incomplete_table(fashion_model):
    t = table({(0, TC0, 1): 1.0}, {0: [TC0], 1: [TC0]}, [1])
    with pytest.raises(P.IncompleteTable):
        tuner.select_plan(t, fashion_model)


def test_plan_round_trip_and_digest_binding(tmp_path, fashion_model, cifar_model):
    plan = ExecPlan(fashion_model.name, P.model_digest(fashion_model), 64, {1: TC0, 2: POPC64}, 123.0, "B200")
    path = tmp_path / "plan.json"
    tuner.save_plan(plan, path)
    back = tuner.load_plan(path, fashion_model)
    assert back.same_mapping(plan) and back.variant_map() == {1: TC0, 2: POPC64}
    with pytest.raises(P.ModelHashMismatch):
        tuner.load_plan(path, cifar_model)
    path.write_text(path.read_text().replace('"format_version": 2', '"format_version": 1'))
    with pytest.raises(P.UnsupportedVersion):
        tuner.load_plan(path)


def test_candidate_variants_per_block_shape():
    """The tensor-engine candidates each block type gets (host logic, no GPU): the step-MMA kernel is
    the incumbent for step-eligible binary convs, HX only for 16-px rows of 64 channels, the
    single-CTA alternative for blocks whose N = 256 tiles may run on CTA pairs."""
    from types import SimpleNamespace

    from paper_2301_05126_b200 import tuner

    def conv(C, H, W, step_ok=True):
        return SimpleNamespace(variant_kind="conv_bin", C=C, H=H, W=W, tc_ok=lambda: True,
                               step_mma_ok=lambda: step_ok)

    l5 = tuner.candidate_variants(conv(64, 16, 16), 32768)
    assert l5[:2] == [(1, 0, 6), (1, 0, 3)] and (1, 0, 5) in l5
    l7 = tuner.candidate_variants(conv(256, 16, 16, step_ok=False), 32768)
    assert l7[0] == (1, 0, 0) and (1, 0, 3) not in l7 and (1, 0, 6) not in l7 and (1, 0, 5) in l7
    fashion = tuner.candidate_variants(conv(64, 14, 14), 32768)
    assert fashion[0] == (1, 0, 3) and (1, 0, 6) not in fashion  # 14-px rows: no HX geometry
    fc = tuner.candidate_variants(SimpleNamespace(variant_kind="fc_bin", tc_ok=lambda: True), 4)
    assert (1, 0, 5) in fc and (0, 0, -1) in fc  # small batch keeps the popc GEMV candidate
    assert len(set(l5)) == len(l5)
    assert (1, 32, 0) in tuner.candidate_variants(conv(256, 16, 16, step_ok=False), 1)  # batch 1: narrow N tiles
    assert (1, 32, 0) not in l7


def test_small_batch_only_candidates_are_selectable():
    """candidates are kept per (block, batch) -- a variant offered only at small batches
    (the FC GEMV at batch <= 8) must win there when it is fastest, and is not required elsewhere."""
    GEMV = (0, 0, -1)
    cells = {(0, TC0, 1): 11.3, (0, GEMV, 1): 3.96, (0, TC0, 4096): 100.0, (0, POPC64, 1): 20.0,
             (0, POPC64, 4096): 400.0}
    t = table(cells, {0: [TC0, GEMV, POPC64]}, [1, 4096])
    t.by_batch = {(0, 1): [TC0, GEMV, POPC64], (0, 4096): [TC0, POPC64]}
    per = tuner.per_batch_assignments(t)
    assert per[1][0] == GEMV and per[4096][0] == TC0
    assert t.missing_cells([1, 4096]) == []
    doc = tuner.table_to_doc(t)
    assert doc["candidates_by_batch"]["0@1"] == [list(TC0), list(GEMV), list(POPC64)]
