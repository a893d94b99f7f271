"""GPU single-layer API vs the reference's outputs (golden digests) -- bit-exact."""

import numpy as np
import pytest

from oracle.oracle import Act, digest, from_boundary
from tests.golden import cases
from tests.helpers import binary_from, weights_from_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2301_05126_b200 as P

    return P


def _gpu_case(P, c):
    n = c["name"]
    if n.startswith("conv_bin"):
        x = binary_from(c["x"], c["mask"])
        return P.conv_bin_forward(x, weights_from_bits(c["w"], (c["C"], 3, 3)), c["K"])
    if n.startswith("conv_int"):
        x = P.IntTensor(c["x"].shape, c["x"])
        return P.conv_int_forward(x, weights_from_bits(c["w"], (c["C"], 3, 3)), c["K"])
    if n.startswith("step"):
        return P.step_forward(P.IntTensor(c["x"].shape, c["x"]), P.IntTensor(c["thr"].shape, c["thr"]), c["pos"])
    if n.startswith("pool_int"):
        return P.maxpool_forward(P.Activation.of_integer(P.IntTensor(c["x"].shape, c["x"])))
    if n.startswith("pool_bin"):
        return P.maxpool_forward(P.Activation.of_binary(binary_from(c["bits"])))
    if n.startswith("fc"):
        return P.fc_forward(binary_from(c["x"], c["mask"]), weights_from_bits(c["w"], (c["L"],)))
    raise KeyError(n)


@pytest.mark.parametrize("case", cases.all_cases(), ids=lambda c: c["name"])
def test_layer_case_bit_exact(P, golden, case):
    out = _gpu_case(P, case)
    assert digest(from_boundary(out)) == golden["cases"][case["name"]]


def test_layout_round_trip(P):
    import torch

    from paper_2301_05126_b200 import native

    lib = native.device_ready()
    rng = np.random.default_rng(5)
    for B, C, H, W in [(1, 1, 1, 1), (2, 70, 3, 5), (3, 64, 7, 7), (1, 512, 4, 4), (2, 33, 1, 1)]:
        t = P.BinaryTensor.from_bits(rng.integers(0, 2, size=(B, C, H, W)), (B, C, H, W))
        words = torch.from_numpy(np.asarray(t.words).view(np.int64)).cuda()
        cw = (C + 31) // 32
        nhwc = torch.zeros(B * H * W * cw, dtype=torch.int32, device="cuda")
        back = torch.zeros_like(words)
        st = native.stream_handle()
        native.check(lib.bnn_bits_ref_to_nhwc(words.data_ptr(), B, C, H, W, nhwc.data_ptr(), st))
        native.check(lib.bnn_bits_nhwc_to_ref(nhwc.data_ptr(), B, C, H, W, back.data_ptr(), st))
        assert np.array_equal(back.cpu().numpy().view(np.uint64), np.asarray(t.words))
        # NHWC semantics: bit c%32 of word (pixel, c//32)
        bits = t.value_bits().transpose(0, 2, 3, 1).reshape(-1, C)
        got = nhwc.cpu().numpy().view(np.uint32).reshape(-1, cw)
        for c in range(C):
            assert np.array_equal((got[:, c // 32] >> (c % 32)) & 1, bits[:, c])


def test_xnor_dot_kats(P):
    """tests/test_core.py:62-85 KATs on the device helper."""
    import torch

    from paper_2301_05126_b200 import native

    lib = native.device_ready()
    rng = np.random.default_rng(11)
    vals = [np.ones(8, int), -np.ones(8, int)]
    kats = [(vals[0], vals[0], 8), (vals[0], vals[1], -8)]
    for n in (1, 63, 64, 65, 192):
        a = P.BinaryTensor.from_bits(rng.integers(0, 2, n), (n,), rng.integers(0, 2, n))
        b = P.BinaryTensor.from_bits(rng.integers(0, 2, n), (n,), rng.integers(0, 2, n))
        kats.append((a, b, P.xnor_popcount_dot(a, b)))
    import ctypes

    for a, b, want in kats:
        if not hasattr(a, "words"):
            a, b = P.pack_bits(a, (len(a),)), P.pack_bits(b, (len(b),))
        dev = [torch.from_numpy(np.asarray(x).view(np.int64)).cuda() for x in (a.words, a.valid_mask, b.words,
                                                                               b.valid_mask)]
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        native.check(lib.bnn_xnor_dot(*[d.data_ptr() for d in dev], a.nwords,
                                      ctypes.cast(out.data_ptr(), ctypes.POINTER(ctypes.c_longlong)),
                                      native.stream_handle()))
        assert int(out.item()) == want


def test_conv_variants_agree(P):
    """Every tile_n variant gives the same sums and bits."""
    from paper_2301_05126_b200 import native

    rng = np.random.default_rng(3)
    for (B, C, K, H, W) in [(3, 64, 256, 8, 8), (2, 256, 128, 6, 6), (2, 96, 70, 5, 7)]:
        x = binary_from(rng.integers(0, 2, (B, C, H, W)))
        w = weights_from_bits(rng.integers(0, 2, (K, C, 3, 3)), (C, 3, 3))
        ref = None
        for tn in (32, 64, 128, 256):
            out = P.conv_bin_forward(x, w, K, variant=native.Variant.make(0, tn))
            if ref is None:
                ref = out
            assert out == ref, tn


def test_errors_are_reference_names(P):
    with pytest.raises(P.OddSpatialDim):
        P.maxpool_forward(P.Activation.of_integer(P.IntTensor((1, 1, 3, 3), np.zeros(9))))
    with pytest.raises(P.ShapeMismatch):
        P.conv_bin_forward(binary_from(np.zeros((1, 2, 3, 3), np.uint8)),
                           weights_from_bits(np.zeros((4, 3, 3, 3), np.uint8), (3, 3, 3)), 4)
    with pytest.raises(P.ShapeMismatch):
        P.fc_forward(binary_from(np.zeros((1, 5), np.uint8)), weights_from_bits(np.zeros((2, 6), np.uint8), (6,)))


TC_CASES = [c for c in cases.conv_bin_cases() if c["C"] % 64 == 0 and c["mask"] is None and c["W"] <= 128] + \
    [c for c in cases.fc_cases() if c["L"] % 64 == 0 and c["mask"] is None]


@pytest.mark.parametrize("case", TC_CASES, ids=lambda c: c["name"])
@pytest.mark.parametrize("tile_n,mode", [(0, 0), (64, 0), (256, 0), (0, 1), (128, 1), (0, 2), (256, 2), (256, 5), (256, 6)])
def test_tensor_engine_case_bit_exact(P, golden, case, tile_n, mode):
    """The tcgen05 kind::mxf4 (FP4 +-1) kernels through the layer API (int32 sums) vs the reference.

    mode 0 = halo-reuse kernel where eligible (one TMA halo box, row-shifted descriptors),
    mode 1 = one TMA box per tap, mode 2 = halo-reuse whenever it fits."""
    from paper_2301_05126_b200 import native

    v = native.Variant.make(native.ENGINE_TC, tile_n, mode)
    if case["name"].startswith("conv_bin"):
        x = binary_from(case["x"])
        out = P.conv_bin_forward(x, weights_from_bits(case["w"], (case["C"], 3, 3)), case["K"], variant=v)
    else:
        out = P.fc_forward(binary_from(case["x"]), weights_from_bits(case["w"], (case["L"],)), variant=v)
    assert digest(from_boundary(out)) == golden["cases"][case["name"]]


def test_bits_f4_glue_round_trip(P):
    import torch

    from paper_2301_05126_b200 import native
    from paper_2301_05126_b200.prep import pack_f4

    lib = native.device_ready()
    rng = np.random.default_rng(8)
    for npix, C in [(1, 32), (37, 64), (500, 512)]:
        words = torch.from_numpy(rng.integers(0, 2**32, size=npix * C // 32, dtype=np.uint64).astype(np.uint32)
                                 .view(np.int32)).cuda()
        f4 = torch.zeros(npix * C // 2, dtype=torch.uint8, device="cuda")
        back = torch.zeros_like(words)
        st = native.stream_handle()
        native.check(lib.bnn_bits_to_f4(words.data_ptr(), npix, C, f4.data_ptr(), st))
        native.check(lib.bnn_f4_to_bits(f4.data_ptr(), npix, C, back.data_ptr(), st))
        assert torch.equal(words, back)
        w = words.cpu().numpy().view(np.uint32)
        bits = ((w[:, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(-1)
        assert np.array_equal(f4.cpu().numpy(), pack_f4(bits))
