"""CPU-side tests: host mirror of the reference vocabulary, device re-layouts, the C-ABI library."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2301_05126_b200 as P
from paper_2301_05126_b200 import prep
from paper_2301_05126_b200.model import LayerKind, LayerSpec, StepDirection
from tests.helpers import weights_from_bits

REPO = Path(__file__).resolve().parents[1]


# ---------------------------------------------------------------- tensors (tests/test_core.py KATs)

def test_pack_kats():
    t = P.pack_bits([1, 1, 1, 1], (4,))
    assert t.words.tolist() == [0b1111]
    t = P.pack_bits([-1, -1], (2,))
    assert t.words.tolist() == [0]
    assert t.valid_mask.tolist() == [0b11]


def test_pack_round_trip_and_canonical():
    rng = np.random.default_rng(1)
    for n in (1, 63, 64, 65, 200):
        v = rng.choice([-1, 1], n)
        t = P.pack_bits(v, (n,))
        assert np.array_equal(t.unpack(), v)
    t = P.BinaryTensor((3,), np.array([0xFF], np.uint64), np.array([0b101], np.uint64))
    assert t.words.tolist() == [0b101] and t.valid_mask.tolist() == [0b101]
    with pytest.raises(P.NonBinaryValue):
        P.pack_bits([1, 0], (2,))
    with pytest.raises(P.LengthMismatch):
        P.pack_bits([1, 1, 1], (2,))


def test_dot_kats():
    a = P.pack_bits([1] * 8, (8,))
    b = P.pack_bits([-1] * 8, (8,))
    assert P.xnor_popcount_dot(a, a) == 8 and P.xnor_popcount_dot(a, b) == -8
    rng = np.random.default_rng(2)
    for _ in range(200):
        n = int(rng.integers(1, 192))
        x, y = rng.integers(0, 2, n), rng.integers(0, 2, n)
        mx, my = rng.integers(0, 2, n), rng.integers(0, 2, n)
        ta, tb = P.BinaryTensor.from_bits(x, (n,), mx), P.BinaryTensor.from_bits(y, (n,), my)
        want = int(((2 * x - 1) * (2 * y - 1) * mx * my).sum())
        assert P.xnor_popcount_dot(ta, tb) == want


# ---------------------------------------------------------------- model vocabulary

def test_synthetic_digests_match_reference(golden):
    for key, want in golden["digests"].items():
        arch, seed = key.rsplit("-", 1)
        assert P.model_digest(P.export_synthetic_model(arch, int(seed))) == want


def test_validate_model_messages(fashion_model):
    assert P.validate_model(fashion_model) == []
    m = P.export_synthetic_model("fashion", 7)
    m.layers = m.layers[1:]
    probs = P.validate_model(m)
    assert "layer 1 must be conv_int, got maxpool" in probs
    m2 = P.export_synthetic_model("cifar10", 1)
    m2.layers = m2.layers[:-1]
    assert any("last layer must be fc_int_out" in p for p in P.validate_model(m2))
    assert P.validate_model(P.ModelSpec("e", P.InputSpec(1, 2, 2), [], 10)) == ["model has no layers"]


def test_layer_display_names(cifar_model):
    names = [P.layer_display_name(l) for l in cifar_model.layers]
    assert names[:5] == ["C64", "S", "C64", "MP16", "S"] and names[-3:] == ["FC1024", "S", "FC1024"]


# ---------------------------------------------------------------- device re-layouts (numpy simulation)

def test_conv_weight_layout():
    rng = np.random.default_rng(4)
    K, C = 5, 70
    wb = rng.integers(0, 2, (K, C, 3, 3))
    layer = LayerSpec(LayerKind.CONV_BIN, (C, 4, 4), (K, 4, 4), weights=weights_from_bits(wb, (C, 3, 3)))
    w = prep.conv_bin_weights(layer)  # (9, CW, K)
    assert w.shape == (9, 3, K) and w.dtype == np.uint32
    for k in range(K):
        for t in range(9):
            for c in range(C):
                assert (w[t, c // 32, k] >> (c % 32)) & 1 == wb[k, c, t // 3, t % 3]
    assert (w[:, 2, :] >> 6).max() == 0  # channels 70..95 are zero padding


def test_fc_flatten_permutation_preserves_dots():
    """Device NHWC order x permuted weights == reference c-major order x reference weights."""
    rng = np.random.default_rng(6)
    for C, H, W in [(64, 7, 7), (40, 3, 2), (512, 4, 4)]:
        L, M = C * H * W, 9
        x = rng.integers(0, 2, (3, C, H, W))
        wb = rng.integers(0, 2, (M, L))
        layer = LayerSpec(LayerKind.FC_BIN, (L,), (M,), weights=weights_from_bits(wb, (L,)))
        wdev, L_, lw = prep.fc_weights(layer, (C, H, W))
        assert L_ == L
        cw = (C + 31) // 32
        xn = np.zeros((3, H, W, cw * 32), np.uint8)
        xn[..., :C] = x.transpose(0, 2, 3, 1)
        xw = prep.pack_u32(xn.reshape(3, H * W * cw * 32))
        pop = np.bitwise_count(xw[:, None, :] ^ wdev.T[None, :, :]).sum(-1)
        got = L - 2 * pop.astype(np.int64)
        want = (2 * x.reshape(3, L) - 1) @ (2 * wb - 1).T
        assert np.array_equal(got, want)


def test_step_params_bits():
    thr, pos = prep.step_params(P.IntTensor((3,), [1, -2, 3]),
                                [StepDirection.POS, StepDirection.NEG, StepDirection.POS])
    assert thr.tolist() == [1, -2, 3] and pos.tolist() == [0b101]


# ---------------------------------------------------------------- the C-ABI library (no GPU needed)

def _header_symbols():
    text = (REPO / "include" / "bnn.h").read_text()
    return sorted(set(re.findall(r"BNN_API[^;(]*?\b(bnn_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2301_05126_b200 import native

    syms = _header_symbols()
    assert len(syms) >= 14
    lib = native.load()
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(native.EXPORTED) == syms
    assert lib.bnn_abi_version() == 7


def test_serve_control_block_layout_matches_header():
    """The resident server's control block (ABI v7): host-written words (request, stop) and device-written
    words (done, status) on separate 128-B lines; the Python side allocates BNN_NET_CTL_WORDS."""
    from paper_2301_05126_b200 import native

    text = (REPO / "include" / "bnn.h").read_text()
    c = {k: int(v) for k, v in re.findall(r"#define (BNN_NET_CTL_\w+) (\d+)", text)}
    assert c["BNN_NET_CTL_WORDS"] == native.NET_CTL_WORDS == 64
    host, dev = (c["BNN_NET_CTL_REQ"], c["BNN_NET_CTL_STOP"]), (c["BNN_NET_CTL_DONE"], c["BNN_NET_CTL_STATUS"])
    assert {w * 4 // 128 for w in host} == {0} and {w * 4 // 128 for w in dev} == {1}
    assert max(dev) < c["BNN_NET_CTL_WORDS"]
    lib = native.load()  # a misaligned control block is refused before any CUDA call
    buf = (ctypes.c_uint32 * 80)()
    off = (-ctypes.addressof(buf)) % 128 + 4
    dummy = (ctypes.c_uint8 * 64)()
    rc = lib.bnn_net_serve_launch(None, 0, 1, ctypes.addressof(dummy), 0, ctypes.addressof(buf) + off,
                                  ctypes.addressof(buf), None, None, 0, 1.0, None)
    assert rc < 0 and "128-B aligned" in native.last_error()


def test_library_reports_argument_errors_without_gpu():
    """Validation happens before any CUDA call: bad dims -> <0 and a message."""
    from paper_2301_05126_b200 import native

    lib = native.load()
    rc = lib.bnn_maxpool_int(None, 1, 1, 3, 3, None, None)
    assert rc < 0 and "even" in native.last_error()
    rc = lib.bnn_conv_bin(None, None, 1, 0, 3, 3, None, 4, None, None, 0, 0, None, None, None, None)
    assert rc < 0 and "bad dims" in native.last_error()


def test_product_does_not_import_oracle():
    for path in (REPO / "paper_2301_05126_b200").rglob("*.py"):
        text = path.read_text()
        assert "import oracle" not in text and "from oracle" not in text, path


def test_native_unavailable_is_loud(tmp_path):
    from paper_2301_05126_b200 import native

    with pytest.raises(P.NativeUnavailable):
        native.load(tmp_path / "missing.so")


def test_front_smem_query_host_only():
    """bnn_tc_front_smem is a pure host function: shapes the one-launch front end accepts."""
    from paper_2301_05126_b200 import native

    lib = native.load()
    assert lib.bnn_tc_front_smem(3, 32, 32, 64, 64, 0, 1) > 0        # CIFAR front
    assert lib.bnn_tc_front_smem(1, 28, 28, 64, 64, 1, 1) > 0        # fashion front
    assert lib.bnn_tc_front_smem(3, 32, 32, 64, 64, 0, 1) <= 227 * 1024
    assert lib.bnn_tc_front_smem(5, 32, 32, 64, 64, 0, 1) == -1      # C > 4 (one byte per channel in a u32 pixel)
    assert lib.bnn_tc_front_smem(3, 32, 32, 128, 64, 0, 1) == -1     # K1 != 64
    assert lib.bnn_tc_front_smem(3, 31, 32, 64, 64, 1, 0) == -1      # odd dims under pooling
    assert lib.bnn_tc_front_smem(3, 256, 256, 64, 64, 0, 0) == -1    # H buffers exceed shared memory


def _net_layers(specs):
    from paper_2301_05126_b200 import native

    arr = (native.NetLayer * len(specs))()
    for d, (kind, C, H, W, K, pool) in zip(arr, specs):
        d.kind, d.C, d.H, d.W, d.K, d.pool = kind, C, H, W, K, pool
        d.w, d.thr, d.pos = 16, 16, 16  # never dereferenced by the host-side planner
    return arr


def test_net_workspace_plan_host_only():
    """bnn_net_workspace validates the block chain and sizes the one-launch kernel on the host (no GPU
    call when the grid is given): CIFAR and fashion chains at batch 1 fit; broken chains are argument errors."""
    import ctypes

    from paper_2301_05126_b200 import native

    lib = native.load()
    F, B_, FC, OUT = native.NET_CONV_FIRST, native.NET_CONV_BIN, native.NET_FC_BIN, native.NET_FC_OUT
    cifar = [(F, 3, 32, 32, 64, 0), (B_, 64, 32, 32, 64, 1), (B_, 64, 16, 16, 256, 0), (B_, 256, 16, 16, 256, 1),
             (B_, 256, 8, 8, 512, 0), (B_, 512, 8, 8, 512, 1), (FC, 8192, 1, 1, 1024, 0), (OUT, 1024, 1, 1, 10, 0)]
    fashion = [(F, 1, 28, 28, 64, 1), (B_, 64, 14, 14, 64, 1), (FC, 3136, 1, 1, 2048, 0), (OUT, 2048, 1, 1, 10, 0)]
    nb, sm = ctypes.c_size_t(0), ctypes.c_size_t(0)
    for chain in (cifar, fashion):
        for B in (1, 8):
            arr = _net_layers(chain)
            assert lib.bnn_net_workspace(arr, len(chain), B, 148, ctypes.byref(nb), ctypes.byref(sm)) == 0, \
                native.last_error()
            assert nb.value > 0 and 0 < sm.value <= 227 * 1024
    bad = list(cifar)
    bad[3] = (B_, 128, 16, 16, 256, 1)  # input channels do not follow the previous block
    assert lib.bnn_net_workspace(_net_layers(bad), len(bad), 1, 148, ctypes.byref(nb), None) < 0
    assert "does not follow" in native.last_error()
    assert lib.bnn_net_workspace(_net_layers(cifar[:-1]), 7, 1, 148, ctypes.byref(nb), None) < 0
    assert "last block" in native.last_error()
    assert lib.bnn_net_workspace(_net_layers(cifar), 8, 4096, 148, ctypes.byref(nb), None) < 0  # smem


def test_fp4_pack_round_trip():
    """The tensor engine's operand format: +1 -> E2M1 0x2, -1 -> 0xA, element 2i in the low nibble."""
    import numpy as np

    from paper_2301_05126_b200.prep import pack_f4, unpack_f4

    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2, size=(5, 64), dtype=np.uint8)
    packed = pack_f4(bits)
    assert packed.shape == (5, 32) and packed.dtype == np.uint8
    assert int(pack_f4(np.array([1, 0], np.uint8))[0]) == 0xA2
    assert np.array_equal(unpack_f4(packed), bits)


def test_step_rows_encode_every_threshold_exactly():
    """bnn_step_rows (host): the FP4 row of each channel, dotted with the constant A block of the
    step MMA, is exactly c = T + 0.5 (POS) / 0.5 - T (NEG) with T clamped to +-(kred + 1)."""
    from paper_2301_05126_b200 import prep

    for kred in (576, 1600, 64):
        thr = np.arange(-kred - 5, kred + 6, dtype=np.int32)
        for pos in (True, False):
            posbits = prep.posbits_from_bool(np.full(thr.size, pos))
            rows = prep.step_rows(thr, posbits, kred)
            assert rows.shape == (thr.size, 32)
            t = np.clip(thr.astype(np.int64), -kred - 1, kred + 1)
            want = t + 0.5 if pos else 0.5 - t
            assert np.array_equal(prep.step_rows_values(rows), want)
            # same decisions as the strict step on every reachable sum (acc = -v for POS rows)
            v = np.arange(-kred, kred + 1, 2)[None, :]
            acc = -v if pos else v
            fires = (acc + prep.step_rows_values(rows)[:, None]) < 0
            ref = (v > thr[:, None]) if pos else (v < thr[:, None])
            assert np.array_equal(fires, ref)
    with pytest.raises(ValueError):
        prep.step_rows(np.array([5000], np.int32), prep.posbits_from_bool([True]), 5000)


# ---------------------------------------------------------------- engine drop-in signature (no GPU needed)

def test_engine_reference_constructor_validation():
    """ExecutionEngine(workers, window_rows, fuse_transfers, clock) -- backends.py:411-420: the same
    positional arguments and ValueErrors, raised before any device is touched."""
    from paper_2301_05126_b200.engine import Engine

    with pytest.raises(ValueError):
        Engine(0)
    with pytest.raises(ValueError):
        Engine(2, 0)
    with pytest.raises(ValueError):
        Engine(device=0, devices=[0])


def test_run_model_assignment_validation(fashion_model):
    """A reference list[ParallelConfig] is validated as backends.py:514-518 does."""
    from paper_2301_05126_b200.engine import Engine
    from paper_2301_05126_b200.model import ParallelConfig as PC

    m = fashion_model
    ok = [PC.CPU if l.kind is LayerKind.FLATTEN else PC.XYZ for l in m.layers]
    assert Engine._resolve_assignments(m, ok) == (None, None)
    with pytest.raises(P.ShapeMismatch):
        Engine._resolve_assignments(m, ok[:-1])
    bad = list(ok)
    bad[[l.kind for l in m.layers].index(LayerKind.FLATTEN)] = PC.X
    with pytest.raises(P.ConfigNotApplicable):
        Engine._resolve_assignments(m, bad)
    with pytest.raises(P.ConfigNotApplicable):
        Engine._resolve_assignments(m, ["W"] * len(m.layers))

    class RefTag:  # the reference's enum members duck-type on .value
        def __init__(self, v):
            self.value = v

    assert Engine._resolve_assignments(m, [RefTag(c.value) for c in ok]) == (None, None)
    assert Engine._resolve_assignments(m, {1: (1, 0, 0)}) == ({1: (1, 0, 0)}, None)
    assert P.applicable_configs(LayerKind.FLATTEN) == (PC.CPU,)
    assert len(P.applicable_configs(LayerKind.CONV_BIN)) == 8


def test_bench_roofline_classification():
    """bench.op_roofline: every fused block against its binding roof -- the CIFAR L7 block is tensor-bound,
    FC_INT_OUT (10 classes, 40 FP4 ops per byte) is HBM-bound; algorithmic bytes = activations in + out."""
    import importlib.util
    from types import SimpleNamespace

    from paper_2301_05126_b200.engine import DevAct

    spec = importlib.util.spec_from_file_location("bench_mod", REPO / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    fp4 = {"tflops": 8600.0, "source": "test", "sm_mhz": 1800}
    l7 = SimpleNamespace(name="conv_bin+pool+step", engine=1, out_fmt="f4",
                         src=DevAct("bits", (256, 16, 16)), dst=DevAct("bits", (256, 8, 8)),
                         work_per_image=lambda: {"bin_mac": 150_994_944})
    out = SimpleNamespace(name="fc_out_argmax", engine=1, out_fmt="bits",
                          src=DevAct("bits", (1024,)), dst=DevAct("int", (10,)),
                          work_per_image=lambda: {"bin_mac": 10_240})
    assert bench.op_bytes(l7) == 256 * 16 * 16 // 2 + 256 * 8 * 8 // 2
    assert bench.op_bytes(out) == 1024 // 2 + 10 * 4 + 4
    r7 = bench.op_roofline(l7, 12.4, 262_144, 1800.0, 148, fp4)
    ro = bench.op_roofline(out, 0.034, 262_144, 1800.0, 148, fp4)
    assert r7["bound"] == "tensor" and 0.5 < r7["frac"] < 1.0
    assert ro["bound"] == "hbm" and ro["unit"] == "GB/s" and 0.3 < ro["frac"] < 1.0
