"""INTEGRATION.md's bnntuner-side binding (integration/bnntuner_gpu.py) is runnable and exact."""

import numpy as np
import pytest

from tests.helpers import weights_from_bits


def test_binding_loads_and_packs_w_cl():
    """CPU: the stub loads libbnn.so and binds; w_cl_u32 is the reference's w_cl (model.py:125-132) in
    32-bit out-channel-minor words."""
    from integration import bnntuner_gpu as G
    from paper_2301_05126_b200.model import LayerKind, LayerSpec

    rng = np.random.default_rng(3)
    C, K = 70, 5
    wb = rng.integers(0, 2, (K, C, 3, 3))
    layer = LayerSpec(LayerKind.CONV_BIN, (C, 4, 4), (K, 4, 4), weights=weights_from_bits(wb, (C, 3, 3)))
    w = G.w_cl_u32(layer)
    assert w.shape == (9, 3, K) and w.dtype == np.uint32
    for k in range(K):
        for c in range(C):
            for t in range(9):
                assert (int(w[t, c // 32, k]) >> (c % 32)) & 1 == wb[k, c, t // 3, t % 3]
    assert G._lib.bnn_conv_bin.argtypes is not None


@pytest.mark.gpu
def test_binding_conv_bin_exact(oracle_mod):
    import paper_2301_05126_b200 as P
    from integration import bnntuner_gpu as G
    from oracle.oracle import Act

    rng = np.random.default_rng(8)
    for B, C, H, W, K in [(2, 64, 8, 8, 32), (3, 70, 5, 7, 17), (1, 256, 16, 16, 64)]:
        wb = rng.integers(0, 2, (K, C, 3, 3))
        layer = P.LayerSpec(P.LayerKind.CONV_BIN, (C, H, W), (K, H, W), weights=weights_from_bits(wb, (C, 3, 3)))
        bits = rng.integers(0, 2, (B, C, H, W))
        x = P.BinaryTensor.from_bits(bits, bits.shape)
        want = oracle_mod.layer_forward(layer, Act("bin", bits=bits.astype(np.uint8)), route="packed").vals
        got = G.conv_bin_forward_gpu(x, G.w_cl_u32(layer), K)
        assert np.array_equal(got, want)
        staged = G.StagedGpuConvBin(layer, P.Activation.of_binary(x), P.Activation, P.IntTensor)
        for item in range(4):  # several WorkItems -> one launch
            staged.run(item)
        out = staged.finish()
        assert np.array_equal(out.integer.values, want)
