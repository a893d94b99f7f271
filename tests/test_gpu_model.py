"""Whole-model GPU parity: per fused block (int32 sums AND packed bits), logits, predictions.

The shipped synthetic models saturate, so every check here is
made per block and repeated on the calibrated stress models.
"""

import numpy as np
import pytest

from oracle.oracle import Act, digest
from tests.helpers import model_with_steps, trace_images

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["tc", "popc"])
def engine(request):
    from paper_2301_05126_b200.engine import POPC, TC, Engine

    with Engine(default_engine=TC if request.param == "tc" else POPC) as e:
        yield e


def nhwc_to_bits(words: np.ndarray, shape) -> np.ndarray:
    """(B, words_per_image) int32 NHWC bits or (B, elems/2) uint8 FP4 +-1 -> (B, C, H, W) 0/1 (or (B, L))."""
    B = words.shape[0]
    if len(shape) == 1:
        C, H, W = shape[0], 1, 1
    else:
        C, H, W = shape
    if words.dtype == np.uint8:  # FP4: every nibble must be exactly +1 (0x2) or -1 (0xA)
        assert set(np.unique(words & 0xF).tolist()) | set(np.unique(words >> 4).tolist()) <= {0x2, 0xA}
        from paper_2301_05126_b200.prep import unpack_f4

        out = unpack_f4(words.reshape(B, H, W, C // 2)).transpose(0, 3, 1, 2)
        return out.reshape(B, -1) if len(shape) == 1 else out
    cw = (C + 31) // 32
    w = words.view(np.uint32).reshape(B, H, W, cw)
    by = w.view(np.uint8).reshape(B, H, W, cw * 4)
    bits = np.unpackbits(by, axis=-1, bitorder="little")[..., :C]
    out = bits.transpose(0, 3, 1, 2)
    return out.reshape(B, -1) if len(shape) == 1 else out


def run_blocks(engine, model, images, oracle_mod, variants=None):
    """Run the fused plan keeping sums; compare every op with the oracle's per-layer outputs."""
    import torch

    from paper_2301_05126_b200.engine import ConvOp, FcOp, FcOutOp, FrontOp

    pm = engine.prepare(model, variants)
    x = torch.from_numpy(images.astype(np.uint8)).cuda()
    logits, preds = pm.infer(x, keep_sums=True)
    torch.cuda.synchronize()
    ops = pm.exec_ops(x)
    outs, sums = pm.buffers(images.shape[0], keep_sums=True, ops=ops)
    _, _, acts = oracle_mod.infer(model, images, route="packed", keep=True)
    checks = []
    for op, o, s in zip(ops, outs, sums):
        if isinstance(op, FrontOp):  # one launch, two blocks: debug taps give each block's sums and bits
            s1, mid, s2 = s
            checks += [(op.u0, mid, s1), (op.u1, o, s2)]
        else:
            checks.append((op, o, s))
    for op, o, s in checks:
        head, tail = op.layers[0], op.layers[-1]
        if isinstance(op, FcOutOp):
            want = acts[head].vals
            assert np.array_equal(o[0].cpu().numpy(), want), op.name
            continue
        if isinstance(op, (ConvOp, FcOp)) and op.fused_step:
            want_sums = acts[head].vals
            got_sums = s.cpu().numpy().reshape(want_sums.shape)
            assert np.array_equal(got_sums, want_sums), f"{op.name} sums (layer {head})"
        # output activation of the op's last non-flatten layer
        last = max(i for i in op.layers if acts[i] is not None)
        ref = acts[last]
        kinds = [l.kind.value for l in model.layers]
        while kinds[last] == "flatten":
            last -= 1
        ref = acts[last]
        if op.dst.kind == "bits":
            got = nhwc_to_bits(o.cpu().numpy(), op.dst.shape if kinds[last] != "flatten" else op.dst.shape)
            assert np.array_equal(got.reshape(ref.bits.shape), ref.bits), f"{op.name} bits (layer {last})"
        else:
            assert np.array_equal(o.cpu().numpy().reshape(ref.vals.shape), ref.vals), f"{op.name} ints"
    return logits.cpu().numpy(), preds.cpu().numpy()


def test_traces_match_reference(engine, golden, oracle_mod):
    from paper_2301_05126_b200.synthetic import export_synthetic_model

    for tr in golden["traces"]:
        m = export_synthetic_model(tr["arch"], tr["seed"])
        imgs = trace_images(m, tr["img_seed"], tr["batch"])
        logits, preds = run_blocks(engine, m, imgs, oracle_mod)
        assert logits.tolist() == tr["logits"]
        assert preds.tolist() == tr["preds"]


def test_reference_golden_vector(golden):
    import paper_2301_05126_b200 as P

    ref = golden["reference_golden_fashion_seed7"]
    m = P.export_synthetic_model("fashion", 7)
    img = np.random.default_rng(123).integers(0, 256, size=(1, 1, 28, 28))
    logits, preds = P.reference_infer(m, P.IntTensor(img.shape, img))
    assert logits.values.tolist() == [ref["logits"]]
    assert preds == ref["predictions"]


def test_calibrated_models_per_block(engine, golden, oracle_mod):
    for cal in golden["calibrated"]:
        m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
        imgs = trace_images(m, cal["img_seed"], cal["batch"])
        logits, preds = run_blocks(engine, m, imgs, oracle_mod)
        assert logits.tolist() == cal["logits"]
        assert preds.tolist() == cal["preds"]


@pytest.mark.parametrize("arch,batch", [("fashion", 96), ("cifar10", 24), ("fashion", 149), ("cifar10", 149), ("fashion", 297)])
def test_batched_calibrated_vs_oracle(engine, golden, oracle_mod, arch, batch):
    cal = next(c for c in golden["calibrated"] if c["arch"] == arch)
    m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
    imgs = trace_images(m, 4242, batch)
    logits, preds = run_blocks(engine, m, imgs, oracle_mod)
    ol, op = oracle_mod.infer(m, imgs, route="packed")
    assert np.array_equal(logits, ol) and np.array_equal(preds, op)
    assert len({tuple(r) for r in logits.tolist()}) > batch // 4  # informative


def test_variants_do_not_change_results(engine, golden, oracle_mod):
    cal = next(c for c in golden["calibrated"] if c["arch"] == "cifar10")
    m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
    imgs = trace_images(m, 99, 12)
    pm = engine.prepare(m)
    base = None
    for eng, tn, tq in [(0, 32, 0), (0, 64, 0), (0, 128, 0), (0, 256, 0), (1, 0, 0), (1, 64, 0), (1, 128, 0),
                        (1, 256, 0), (1, 0, 1), (1, 256, 1), (1, 0, 3), (1, 64, 3), (1, 128, 3), (1, 256, 3),
                        (1, 0, 5), (1, 256, 5), (1, 0, 6)]:
        var = {i: (eng, tn, tq) for i in pm.tunable_ops()}
        logits, _ = run_blocks(engine, m, imgs, oracle_mod, variants=var)
        if base is None:
            base = logits
        assert np.array_equal(logits, base), (eng, tn, tq, pm.engines())
    engine.prepare(m, {})


def test_run_model_and_graph(engine, golden):
    import paper_2301_05126_b200 as P

    cal = next(c for c in golden["calibrated"] if c["arch"] == "cifar10")
    m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
    imgs = trace_images(m, 7, 10)
    rep = engine.run_model(m, P.IntTensor(imgs.shape, imgs), batch_size=4)  # short last batch
    ref_logits = np.concatenate([engine.run_model(m, imgs[i:i + 1]).logits for i in range(10)])
    assert np.array_equal(rep.logits, ref_logits)
    assert rep.predictions == [int(p) for p in ref_logits.argmax(axis=1)]
    assert len(rep.compute_ns) == len(m.layers) and sum(rep.compute_ns) > 0
    g = engine.graph(m, batch=1)
    gz = engine.graph(m, batch=1, zero_copy=True)  # kernels read/write pinned host memory directly
    for i in range(10):
        lg, pr = g.replay(imgs[i:i + 1])
        assert np.array_equal(lg[0], ref_logits[i]) and pr[0] == rep.predictions[i]
        lz, pz = gz.replay(imgs[i:i + 1])
        assert np.array_equal(lz[0], ref_logits[i]) and pz[0] == rep.predictions[i]


def test_generic_block_patterns(engine, oracle_mod):
    """Sequences outside the fused patterns: binary pool after step, unfused int pool, int flatten + step."""
    import paper_2301_05126_b200 as P
    from paper_2301_05126_b200.model import LayerKind as K, LayerSpec, StepDirection
    from tests.helpers import weights_from_bits

    rng = np.random.default_rng(17)

    def step(shape, lo=-6, hi=6):
        c = shape[0]
        return LayerSpec(K.STEP, shape, shape, thresholds=P.IntTensor((c,), rng.integers(lo, hi, c)),
                         directions=[StepDirection.POS if p else StepDirection.NEG for p in rng.integers(0, 2, c)])

    def conv(kind, c, k, h, w):
        return LayerSpec(kind, (c, h, w), (k, h, w), weights=weights_from_bits(rng.integers(0, 2, (k, c, 3, 3)),
                                                                               (c, 3, 3)))

    layers = [
        conv(K.CONV_INT, 2, 40, 8, 8), step((40, 8, 8), 100, 300),
        LayerSpec(K.MAXPOOL, (40, 8, 8), (40, 4, 4)),                 # binary pool (OR)
        conv(K.CONV_BIN, 40, 36, 4, 4),
        LayerSpec(K.MAXPOOL, (36, 4, 4), (36, 2, 2)), LayerSpec(K.MAXPOOL, (36, 2, 2), (36, 1, 1)),  # two int pools
        LayerSpec(K.FLATTEN, (36, 1, 1), (36,)), step((36,)),         # step on flattened ints
        LayerSpec(K.FC_BIN, (36,), (20,), weights=weights_from_bits(rng.integers(0, 2, (20, 36)), (36,))),
        step((20,)),
        LayerSpec(K.FC_INT_OUT, (20,), (7,), weights=weights_from_bits(rng.integers(0, 2, (7, 20)), (20,))),
    ]
    m = P.ModelSpec("generic", P.InputSpec(2, 8, 8), layers, 7)
    assert P.validate_model(m) == []
    imgs = rng.integers(0, 256, size=(5, 2, 8, 8))
    logits, preds = engine.infer(m, imgs)
    ol, op = oracle_mod.infer(m, imgs)
    assert np.array_equal(logits, ol) and list(preds) == op.tolist()


@pytest.mark.parametrize("tile_n,mode", [(0, 3), (64, 3), (128, 3), (0, 6)])
def test_step_mma_extreme_thresholds(engine, golden, oracle_mod, tile_n, mode):
    """The step folded into one extra MMA (variant tile_q = 3, bnn_step_rows): thresholds at and
    beyond +-(9C + 1), around 0 and random, both directions -- per-block sums and bits vs the oracle."""
    from paper_2301_05126_b200.engine import ConvOp
    from paper_2301_05126_b200.model import LayerKind, LayerSpec, StepDirection
    from paper_2301_05126_b200.tensors import IntTensor

    cal = next(c for c in golden["calibrated"] if c["arch"] == "cifar10")
    m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
    rng = np.random.default_rng(5)
    for i, layer in enumerate(m.layers):
        if layer.kind is LayerKind.STEP and i >= 2 and m.layers[i - 1].kind is LayerKind.CONV_BIN:
            kred = 9 * m.layers[i - 1].in_shape[0]
            thr = np.asarray(layer.thresholds.values, dtype=np.int64).copy()
            n = thr.size
            pick = rng.random(n) < 0.25
            special = rng.choice([-kred - 3, -kred - 1, -kred, -1, 0, 1, kred, kred + 1, kred + 4], n)
            thr[pick] = special[pick]
            dirs = [StepDirection.NEG if rng.random() < 0.3 else d for d in layer.directions]
            m.layers[i] = LayerSpec(LayerKind.STEP, layer.in_shape, layer.out_shape,
                                    thresholds=IntTensor((n,), thr), directions=dirs)
    imgs = trace_images(m, 31, 20)
    pm = engine.prepare(m)
    var = {i: (1, tile_n, mode) for i in pm.tunable_ops()}
    logits, preds = run_blocks(engine, m, imgs, oracle_mod, variants=var)
    if engine.default_engine == 1:
        assert any(isinstance(u, ConvOp) and u.step_mma_ok() for u in engine.prepare(m, var).units)
    ol, op = oracle_mod.infer(m, imgs, route="packed")
    assert np.array_equal(logits, ol) and np.array_equal(preds, op)
    engine.prepare(m, {})
