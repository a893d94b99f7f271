"""The one-launch front end (bnn_tc_front, csrc/tc_front.cu) against the CPU oracle.

conv_int + [maxpool] + step -> conv_bin + [maxpool] + step, with the intermediate
activation in shared memory.  Every check is per block (int32 sums of both convs,
the first block's +-1 output through the debug tap, the second block's output
bits) and bit-exact, over shapes that exercise: 1..4 input channels, odd widths,
tiles that straddle image rows, pooling on either or both blocks, both output
formats, one image per CTA and many images per CTA (persistent loop), and the
calibrated CIFAR / fashion models end to end.
"""

import numpy as np
import pytest

from tests.helpers import weights_from_bits
from tests.test_gpu_model import run_blocks

pytestmark = pytest.mark.gpu


def front_model(rng, C, H, W, pool1, pool2, classes=10):
    import paper_2301_05126_b200 as P
    from paper_2301_05126_b200.model import LayerKind as K, LayerSpec

    def conv(kind, c, k, h, w):
        return LayerSpec(kind, (c, h, w), (k, h, w),
                         weights=weights_from_bits(rng.integers(0, 2, (k, c, 3, 3)), (c, 3, 3)))

    def step(shape):
        c = shape[0]
        return LayerSpec(K.STEP, shape, shape, thresholds=P.IntTensor((c,), np.zeros(c, dtype=np.int64)),
                         directions=[P.StepDirection.POS] * c)

    layers = [conv(K.CONV_INT, C, 64, H, W)]
    h, w = H, W
    if pool1:
        layers.append(LayerSpec(K.MAXPOOL, (64, h, w), (64, h // 2, w // 2)))
        h, w = h // 2, w // 2
    layers.append(step((64, h, w)))
    layers.append(conv(K.CONV_BIN, 64, 64, h, w))
    if pool2:
        layers.append(LayerSpec(K.MAXPOOL, (64, h, w), (64, h // 2, w // 2)))
        h, w = h // 2, w // 2
    layers.append(step((64, h, w)))
    L = 64 * h * w
    layers.append(LayerSpec(K.FLATTEN, (64, h, w), (L,)))
    layers.append(LayerSpec(K.FC_INT_OUT, (L,), (classes,),
                            weights=weights_from_bits(rng.integers(0, 2, (classes, L)), (L,))))
    m = P.ModelSpec("front", P.InputSpec(C, H, W), layers, classes)
    assert P.validate_model(m) == []
    return m


@pytest.fixture(scope="module")
def tc_engine():
    from paper_2301_05126_b200.engine import TC, Engine

    with Engine(default_engine=TC) as e:
        yield e


SHAPES = [  # C, H, W, pool1, pool2, batch
    (3, 32, 32, 0, 1, 5),      # the CIFAR front (conv 3->64, conv 64->64 + pool)
    (1, 28, 28, 1, 1, 4),      # the fashion front (conv + pool, conv + pool)
    (3, 32, 32, 0, 1, 300),    # > #SMs: several images per CTA, both H buffers and all ring stages cycle
    (1, 28, 28, 1, 1, 333),
    (2, 10, 14, 0, 0, 7),      # no pooling: second block writes straight from the tile epilogue
    (4, 12, 6, 1, 0, 9),       # C = 4 (full u32 pixel word); pool on the first block only
    (3, 9, 11, 0, 0, 3),       # odd dims (byte-load loader path)
    (3, 6, 40, 0, 1, 2),       # wide rows: a tile covers < 4 rows
    # C = 1 + pool (the fashion case) at other shapes
    (1, 8, 40, 1, 1, 3),       # bulk-copied image, pool windows straddling tiles and image rows
    (1, 10, 14, 1, 0, 7),      # 140-B image: byte-load (global) loader path
    (1, 14, 6, 1, 0, 200),     # global loader path, several images per CTA
]


@pytest.mark.parametrize("C,H,W,pool1,pool2,batch", SHAPES)
def test_front_blocks_vs_oracle(tc_engine, oracle_mod, C, H, W, pool1, pool2, batch):
    from paper_2301_05126_b200.engine import FrontOp

    rng = np.random.default_rng(1000 + C * 7 + H + W)
    base = front_model(rng, C, H, W, pool1, pool2)
    calib = rng.integers(0, 256, size=(16, C, H, W))
    m = oracle_mod.calibrated_model(base, calib, 5)  # informative thresholds, mixed POS / NEG
    imgs = rng.integers(0, 256, size=(batch, C, H, W))
    pm = tc_engine.prepare(m)
    pm.front_min_batch = 1  # small batches too (the default sends them to the two-kernel path)
    assert isinstance(pm.ops[0], FrontOp), pm.ops[0].name
    logits, preds = run_blocks(tc_engine, m, imgs, oracle_mod)
    ol, op = oracle_mod.infer(m, imgs, route="packed")
    assert np.array_equal(logits, ol) and np.array_equal(preds, op)


@pytest.mark.parametrize("out_fmt", ["bits", "f4"])
def test_front_output_formats(tc_engine, oracle_mod, out_fmt):
    """Both output formats of the second block (bits for a popc consumer, FP4 for a tensor one)."""
    import torch

    from paper_2301_05126_b200.engine import POPC, TC, FrontOp

    rng = np.random.default_rng(77)
    m = oracle_mod.calibrated_model(front_model(rng, 3, 16, 16, 0, 1), rng.integers(0, 256, (8, 3, 16, 16)), 3)
    # the consumer's engine decides the format the front end writes
    pm = tc_engine.prepare(m, {2: (POPC if out_fmt == "bits" else TC, 0, 0)})
    pm.front_min_batch = 1
    assert isinstance(pm.ops[0], FrontOp) and pm.ops[0].out_fmt == out_fmt
    imgs = rng.integers(0, 256, size=(6, 3, 16, 16))
    run_blocks(tc_engine, m, imgs, oracle_mod)
    tc_engine.prepare(m, {})
    del torch


def test_front_matches_unfused(tc_engine, golden, oracle_mod):
    """Fused and unfused plans agree bit for bit on the calibrated CIFAR / fashion models."""
    import torch

    from tests.helpers import model_with_steps, trace_images

    for cal in golden["calibrated"]:
        m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
        imgs = trace_images(m, 31, 200)
        pm = tc_engine.prepare(m)
        x = torch.from_numpy(imgs.astype(np.uint8)).cuda()
        res = []
        for fuse in (True, False):
            pm.set_fuse_front(fuse)
            lg, pr = pm.infer(x)
            res.append((lg.cpu().numpy().copy(), pr.cpu().numpy().copy()))
        pm.set_fuse_front(True)
        assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
