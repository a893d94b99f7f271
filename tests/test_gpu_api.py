"""The reference-facing engine API on the GPU, against the CPU oracle.

* the criterion-3 matrix (/root/reference/pkg/tests/test_acceptance.py:217-247): both architectures,
  B in {1, 2, 4, 8}, every layer through ``execute_layer`` under every applicable reference
  ``ParallelConfig`` tag AND every kernel variant of its kind, output == the oracle's layer output
  (compared in the reference boundary format, digests of packed words + masks);
* ``layer_forward`` called directly, ``profile_layer`` (backends.py / profiler.py:98-120 entry points);
* ``ExecutionEngine`` positional construction and ``run_model(model, images, [ParallelConfig...], bs)``
  as `bnntuner/cli.py` and `tests/test_backends.py:171-188` call it;
* multi-device ``Engine(devices=[0, 0])``: image sharding invariance (test_backends.py:141-149);
* the empty-dataset report.
"""

import numpy as np
import pytest

from oracle.oracle import Act, digest, from_boundary

pytestmark = pytest.mark.gpu

TC_VARIANTS = [(1, 0, 0), (1, 64, 0), (1, 128, 0), (1, 0, 1), (1, 0, 2), (1, 0, 3), (1, 0, 5), (1, 0, 6)]
POPC_VARIANTS = [(0, 32, 0), (0, 64, 0), (0, 128, 0), (0, 0, -1)]


@pytest.fixture(scope="module")
def P():
    import paper_2301_05126_b200 as P

    return P


def to_ours(P, act: Act):
    if act.kind == "int":
        return P.Activation.of_integer(P.IntTensor(act.vals.shape, act.vals))
    return P.Activation.of_binary(P.BinaryTensor.from_bits(act.bits, act.bits.shape, act.mask))


def models(P, golden):
    from tests.helpers import model_with_steps

    out = []
    for arch, seed in (("fashion", 7), ("cifar10", 1)):
        out.append((f"{arch}-synthetic", P.export_synthetic_model(arch, seed)))
        cal = next(c for c in golden["calibrated"] if c["arch"] == arch)
        out.append((f"{arch}-calibrated", model_with_steps(cal["arch"], cal["seed"], cal["steps"])))
    return out


def test_criterion_3_matrix(P, golden, oracle_mod):
    from paper_2301_05126_b200 import native

    rng = np.random.default_rng(10_003)
    checked = 0
    with P.ExecutionEngine(2, 1, False) as engine:  # the reference's positional signature
        for name, model in models(P, golden):
            for batch in (1, 2, 4, 8):
                imgs = rng.integers(0, 256, (batch,) + tuple(model.input.shape))
                act = Act("int", vals=imgs.astype(np.int32))
                for i, layer in enumerate(model.layers):
                    ref = oracle_mod.layer_forward(layer, act, route="packed")
                    want = digest(ref)
                    inp = to_ours(P, act)
                    kind = layer.kind.value
                    configs = list(P.applicable_configs(layer.kind))
                    if kind in ("conv_bin", "fc_bin", "fc_int_out"):
                        pv = POPC_VARIANTS if kind != "conv_bin" else [v for v in POPC_VARIANTS if v[2] >= 0]
                        configs += [native.Variant.make(*v) for v in TC_VARIANTS + pv]
                    for cfg in configs:
                        timed = engine.execute_layer(layer, inp, cfg, batch)
                        assert digest(from_boundary(timed.output)) == want, (name, i, kind, cfg, batch)
                        assert timed.compute_ns >= 0 and timed.overhead_ns >= 0
                        checked += 1
                    # layer_forward (the module-level API) on the same input
                    assert digest(from_boundary(P.layer_forward(layer, inp))) == want, (name, i, kind)
                    act = ref
    # fashion 9 layers (8 + 1 flatten tag) / CIFAR 18 layers, x2 models x4 batches, + variants
    assert checked > 2000


def test_profile_layer_entry_points(P, golden, oracle_mod):
    from paper_2301_05126_b200 import native

    model = P.export_synthetic_model("fashion", 7)
    rng = np.random.default_rng(4)
    act = Act("int", vals=rng.integers(0, 256, (4,) + tuple(model.input.shape)).astype(np.int32))
    with P.ExecutionEngine(1) as engine:
        for layer in model.layers:
            inp = to_ours(P, act)
            for cfg in (P.applicable_configs(layer.kind)[-1], None):
                e = P.profile_layer(engine, layer, inp, cfg, 4, warmups=1, reps=3)
                assert e.reps == 3 and e.compute_ns >= 0 and e.total_ns > 0
            if layer.kind.value == "conv_bin":
                e = P.profile_layer(engine, layer, inp, native.Variant.make(1, 0, 0), 4, warmups=1, reps=3)
                assert e.compute_ns > 0
                with pytest.raises(P.ShapeMismatch):
                    P.profile_layer(engine, layer, inp, None, 5)
            act = oracle_mod.layer_forward(layer, act, route="packed")
        flat = next(l for l in model.layers if l.kind.value == "flatten")
        inp = P.Activation.of_binary(P.BinaryTensor.from_bits(np.zeros((1,) + flat.in_shape, int), (1,) + flat.in_shape))
        with pytest.raises(P.ConfigNotApplicable):  # backends.py:456-461: flatten is CPU-only
            engine.execute_layer(flat, inp, P.ParallelConfig.X)


def test_run_model_reference_call(P, golden, oracle_mod):
    """ExecutionEngine(workers, window_rows, fuse_transfers).run_model(model, images, assignments, bs)
    exactly as bnntuner/cli.py:206-215 calls it, with the reference's remainder batching."""
    from tests.helpers import model_with_steps

    cal = next(c for c in golden["calibrated"] if c["arch"] == "fashion")
    m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
    imgs = np.random.default_rng(12).integers(0, 256, (10, 1, 28, 28))
    assignments = [P.ParallelConfig.CPU if l.kind.value == "flatten" else P.ParallelConfig.X for l in m.layers]
    want_l, want_p = oracle_mod.infer(m, imgs, route="packed")
    with P.ExecutionEngine(2, 1, True) as engine:
        rep = engine.run_model(m, P.IntTensor(imgs.shape, imgs), assignments, 4)
        assert rep.predictions == want_p.tolist()
        assert np.array_equal(rep.logits, want_l)
        assert len(rep.overhead_ns) == len(rep.compute_ns) == len(m.layers) and rep.wall_ns > 0
        with pytest.raises(P.ShapeMismatch):
            engine.run_model(m, P.IntTensor(imgs.shape, imgs), assignments[:-1], 4)
        with pytest.raises(ValueError):
            engine.run_model(m, P.IntTensor(imgs.shape, imgs), assignments, 0)
        empty = engine.run_model(m, np.zeros((0, 1, 28, 28), np.uint8), assignments, 4)
        assert empty.predictions == [] and empty.logits.shape == (0, 10) and sum(empty.compute_ns) == 0


@pytest.mark.parametrize("arch", ["fashion", "cifar10"])
def test_multi_device_sharding_invariance(P, golden, oracle_mod, arch):
    """Engine(devices=[0, 0]): two shards, two host threads, two pipelines on one GPU -- identical
    logits and predictions to one device and to the oracle (tests/test_backends.py:141-149)."""
    import torch

    from tests.helpers import model_with_steps

    cal = next(c for c in golden["calibrated"] if c["arch"] == arch)
    m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
    n = 1001 if arch == "fashion" else 333  # odd: uneven shards
    imgs = np.random.default_rng(77).integers(0, 256, (n,) + tuple(m.input.shape)).astype(np.uint8)
    want_l, want_p = oracle_mod.infer(m, imgs, route="packed")
    host = torch.from_numpy(imgs).pin_memory()
    with P.Engine(device=0) as one, P.Engine(devices=[0, 0]) as two, P.Engine(devices=[0, 0, 0]) as three:
        r1 = one.run_model(m, host, batch_size=256)
        r2 = two.run_model(m, host, batch_size=256)
        r3 = three.run_model(m, host)
        for r in (r1, r2, r3):
            assert np.array_equal(r.logits, want_l)
            assert r.predictions == want_p.tolist()
        assert len(two._shards) == 2 and len(three._shards) == 3
        # a plan set through prepare() on the multi-device engine reaches every shard
        pm = two.prepare(m, {i: (1, 0, 5) for i in two.prepare(m).tunable_ops()})
        r4 = two.run_model(m, host, batch_size=128)
        assert np.array_equal(r4.logits, want_l)
        assert all(u.variant is None or u.variant.key() == (1, 0, 5) for u in two._shards[1].prepare(m).units
                   if u.variant_kind is not None)
        del pm
