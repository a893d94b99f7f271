"""Large-batch parity under the production (throughput) plans -- the headline configuration's evidence.

At the small batches of test_gpu_model.py every persistent CTA of the tensor kernels runs at most
one tile.  Here the batch forces many tiles per CTA in every kernel (CIFAR B = 8,192: ~55 images per
front-end CTA, ~110 M = 256 tiles per CTA pair in L7; fashion B = 32,768: ~220 images per front-end
CTA), so the persistent loops, the TMEM accumulator hand-back across CTA pairs and the mbarrier
rings wrapping across tiles are all exercised, on the calibrated (informative) models.

Checks, against the CPU oracle (pinned to the reference's own outputs, tests/test_oracle.py):
  * every image's int32 logits and first-max predictions (all B images);
  * every fused block's packed output bits on >= 1,024 sampled images (first, last and random),
    from the PRODUCTION launch (no debug taps);
  * every fused block's int32 pre-activation sums on the same sample, from a second launch with the
    debug taps on (a different kernel instantiation for the front end, so both are run).
The plans: the bench's tuned throughput plan (HX + step MMA on L5, CTA pairs on the N = 256 blocks),
all-default tensor variants, single-CTA kernels, the per-tap step-MMA kernels and the popc engine.
Reference pattern: /root/reference/pkg/tests/test_acceptance.py:217-247 (full model matrix).
"""

import numpy as np
import pytest

from tests.helpers import model_with_steps
from tests.test_gpu_model import nhwc_to_bits

pytestmark = pytest.mark.gpu

# block index -> (engine, tile_n, tile_q); block 2 of CIFAR is L5 (64 -> 256 channels at 16x16)
TUNED_CIFAR = {0: (1, 0, 0), 1: (1, 0, 0), 2: (1, 0, 6), 3: (1, 0, 0), 4: (1, 0, 0), 5: (1, 0, 0), 6: (1, 0, 0),
               7: (1, 0, 0)}
PLANS = {
    "tuned": "tuned",
    "default_tc": (1, 0, 0),
    "single_cta": (1, 0, 5),
    "step_mma": (1, 0, 3),
    "popc": (0, 0, 0),
}
BATCH = {"cifar10": 8192, "fashion": 32768}
_cache: dict = {}


def sample_index(n: int, k: int = 256, seed: int = 11) -> np.ndarray:
    rng = np.random.default_rng(seed)
    idx = np.concatenate([np.arange(k), np.arange(n - k, n), rng.choice(np.arange(k, n - k), 2 * k, False)])
    return np.unique(idx)


def calibrated(golden, arch):
    cal = next(c for c in golden["calibrated"] if c["arch"] == arch)
    return model_with_steps(cal["arch"], cal["seed"], cal["steps"])


def reference(golden, oracle_mod, arch):
    """(model, images, oracle logits, oracle preds, sample idx, oracle per-layer acts on the sample)."""
    if arch not in _cache:
        m = calibrated(golden, arch)
        B = BATCH[arch]
        imgs = np.random.default_rng(90210).integers(0, 256, size=(B,) + tuple(m.input.shape)).astype(np.uint8)
        ol, op = oracle_mod.infer(m, imgs, route="packed")
        idx = sample_index(B)
        _, _, acts = oracle_mod.infer(m, imgs[idx], route="packed", keep=True)
        _cache[arch] = (m, imgs, ol, op, idx, acts)
    return _cache[arch]


def plan_variants(pm, arch, plan):
    if plan == "tuned":
        return dict(TUNED_CIFAR) if arch == "cifar10" else {i: (1, 0, 0) for i in pm.tunable_ops()}
    return {i: plan for i in pm.tunable_ops()}


def _rows(t, sel):
    if t is None:
        return None
    if isinstance(t, (tuple, list)):
        return type(t)(_rows(u, sel) for u in t)
    return t.index_select(0, sel).cpu().numpy()


def checks_for(ops):
    from paper_2301_05126_b200.engine import FrontOp

    for i, op in enumerate(ops):
        if isinstance(op, FrontOp):
            yield i, op.u0, "mid"
            yield i, op.u1, "out"
        else:
            yield i, op, "out"


def compare_blocks(model, ops, outs, sums, acts, tag):
    """outs / sums: per-op CPU arrays of the sampled images (sums None = bits only)."""
    from paper_2301_05126_b200.engine import ConvOp, FcOp, FcOutOp, FrontOp

    kinds = [l.kind.value for l in model.layers]
    for i, op, which in checks_for(ops):
        o, s = outs[i], None if sums is None else sums[i]
        if isinstance(ops[i], FrontOp):
            s1, mid, s2 = s if s is not None else (None, None, None)
            o, s = (mid, s1) if which == "mid" else (o, s2)
            if which == "mid" and mid is None:
                o = None  # the first block's bits leave the CTA only through the debug tap
        head = op.layers[0]
        if isinstance(op, FcOutOp):
            assert np.array_equal(o[0], acts[head].vals), f"{tag}: {op.name} logits"
            continue
        if s is not None and isinstance(op, (ConvOp, FcOp)) and op.fused_step:
            want = acts[head].vals
            assert np.array_equal(s.reshape(want.shape), want), f"{tag}: {op.name} sums (layer {head})"
        if o is None:
            continue
        last = max(j for j in op.layers if acts[j] is not None)
        while kinds[last] == "flatten":
            last -= 1
        ref = acts[last]
        got = nhwc_to_bits(o, op.dst.shape)
        assert np.array_equal(got.reshape(ref.bits.shape), ref.bits), f"{tag}: {op.name} bits (layer {last})"


@pytest.fixture(scope="module")
def engine():
    from paper_2301_05126_b200.engine import Engine

    with Engine(device=0) as e:
        yield e


@pytest.mark.parametrize("plan", list(PLANS))
@pytest.mark.parametrize("arch", ["cifar10", "fashion"])
def test_large_batch_plan_vs_oracle(engine, golden, oracle_mod, arch, plan):
    import torch

    from paper_2301_05126_b200.engine import FrontOp

    m, imgs, ol, op_, idx, acts = reference(golden, oracle_mod, arch)
    B = imgs.shape[0]
    assert len({tuple(r) for r in ol[:4096].tolist()}) > 1000, "the calibrated model must be informative"
    pm = engine.prepare(m, {})
    pm.set_variants(plan_variants(pm, arch, PLANS[plan]))
    x = torch.from_numpy(imgs).cuda()
    sel = torch.from_numpy(idx).cuda()
    ops = pm.exec_ops(x)
    if PLANS[plan] != (0, 0, 0):
        assert isinstance(ops[0], FrontOp) and all(o.engine == 1 for o in ops), pm.engines()
    # production launch: logits / preds of every image, block output bits of the sample
    logits, preds = pm.infer(x)
    torch.cuda.synchronize()
    assert np.array_equal(logits.cpu().numpy(), ol), f"{arch}/{plan}: logits differ from the oracle"
    assert np.array_equal(preds.cpu().numpy(), op_), f"{arch}/{plan}: predictions differ"
    outs, _ = pm.buffers(B, False, ops)
    compare_blocks(m, ops, [_rows(o, sel) for o in outs], None, acts, f"{arch}/{plan}/production")
    # debug-tap launch: int32 sums (and the front end's first-block bits) of the sample
    logits2, _ = pm.infer(x, keep_sums=True)
    torch.cuda.synchronize()
    assert np.array_equal(logits2.cpu().numpy(), ol)
    outs, sums = pm.buffers(B, True, ops)
    compare_blocks(m, ops, [_rows(o, sel) for o in outs], [_rows(s, sel) for s in sums], acts,
                   f"{arch}/{plan}/sums")
    pm.release()
    engine.prepare(m, {})


@pytest.mark.parametrize("arch", ["cifar10", "fashion"])
def test_run_model_e2e_large_batch(engine, golden, oracle_mod, arch):
    """The bench's e2e leg: the public run_model from pinned host memory (pipelined copy stream,
    short first batch, ping-pong device inputs) -- every logit and prediction vs the oracle, with a
    tail batch below one image per SM (the unfused front end then runs)."""
    import torch

    m, imgs, ol, op_, _, _ = reference(golden, oracle_mod, arch)
    bs = 2048
    # run_model's batches: a short first one (bs / 8), then full ones; leave a tail of 100 < 148 images
    n = bs // 8 + ((imgs.shape[0] - bs // 8) // bs - 1) * bs + 100
    host = torch.from_numpy(imgs[:n]).pin_memory()
    rep = engine.run_model(m, host, batch_size=bs)
    assert np.array_equal(rep.logits, ol[:n])
    assert rep.predictions == op_[:n].tolist()
    assert len(rep.compute_ns) == len(m.layers) and sum(rep.compute_ns) > 0
