"""The binding a `bnntuner` maintainer would add as ``bnntuner/_gpu.py``.

Runnable as-is against either package's objects (duck-typed: ``.dims``, ``.words``, ``.weights``,
``.out_channels`` / ``.out_shape``): it binds libbnn.so with ctypes -- no torch types cross the ABI,
device buffers come from torch's allocator only for convenience -- and provides

* ``conv_bin_forward_gpu(inp, w_cl_u32, out_channels)``: the reference's ``conv_bin_forward``
  (`bnntuner/layers.py:104-115`) for a fully valid BinaryTensor, bit-exact;
* ``w_cl_u32(layer)``: the reference's tap-major channel-packed ``w_cl`` (`model.py:125-132`) in the
  32-bit, out-channel-minor order ``bnn_conv_bin`` reads;
* ``StagedGpuConvBin``: the stage -> run -> finish operator of `bnntuner/backends.py:210-256`, to be
  registered as ``_STAGING[LayerKind.CONV_BIN]`` (`backends.py:389-396`).  The reference's workers
  call ``run`` once per WorkItem from several threads; one launch covers the whole layer, so the
  first call launches it and the others return.

Tested by tests/test_integration.py (CPU: the library loads and binds; GPU: bit-exact vs the oracle).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB = Path(os.environ.get("BNN_LIB", Path(__file__).resolve().parents[1] / "paper_2301_05126_b200" / "libbnn.so"))

_lib = ctypes.CDLL(str(LIB))
P, I = ctypes.c_void_p, ctypes.c_int
_lib.bnn_last_error.restype = ctypes.c_char_p
_lib.bnn_init.argtypes = [I]
_lib.bnn_bits_ref_to_nhwc.argtypes = [P, I, I, I, I, P, P]
# bnn_conv_bin(x, mask, B, C, H, W, w, K, thr, posbits, pool, out_fmt, out_nhwc, sums, variant, stream)
_lib.bnn_conv_bin.argtypes = [P, P, I, I, I, I, P, I, P, P, I, I, P, P, P, P]


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(f"libbnn error {rc}: {(_lib.bnn_last_error() or b'').decode()}")


def w_cl_u32(layer) -> np.ndarray:
    """(9, ceil(C/32), K) uint32: bit c%32 of word (tap, c//32, k) = weight bit of filter k, channel c,
    tap dy*3+dx -- the reference's w_cl (model.py:125-132: u64 [K, 9*ceil(C/64)], tap-major) in 32-bit
    words, out-channel-minor."""
    filters = layer.weights
    C = int(filters[0].dims[0])
    K = len(filters)
    cw = (C + 31) // 32
    out = np.zeros((9, cw * 32, K), dtype=np.uint8)
    for k, f in enumerate(filters):
        n = C * 9
        by = np.ascontiguousarray(np.asarray(f.words, dtype="<u8")).view(np.uint8)
        bits = np.unpackbits(by, bitorder="little")[:n].reshape(C, 9)  # (c, tap)
        out[:, :C, k] = bits.T
    words = np.packbits(out.transpose(0, 2, 1), axis=-1, bitorder="little")  # (9, K, cw*4) bytes
    return np.ascontiguousarray(words.view("<u4").transpose(0, 2, 1))  # (9, cw, K)


def conv_bin_forward_gpu(inp, w_cl, out_channels: int, device: int = 0) -> np.ndarray:
    """inp: BinaryTensor (B,C,H,W), fully valid; w_cl: ``w_cl_u32(layer)``.  -> int32 (B,K,H,W),
    == conv_bin_forward(inp, ...).values."""
    import torch

    B, C, H, W = (int(d) for d in inp.dims)
    _check(_lib.bnn_init(device))
    with torch.cuda.device(device):
        words = torch.from_numpy(np.ascontiguousarray(np.asarray(inp.words, dtype="<u8")).view(np.int64)).cuda()
        nhwc = torch.empty(B * H * W * ((C + 31) // 32), dtype=torch.int32, device="cuda")
        w = torch.from_numpy(np.ascontiguousarray(w_cl).view(np.int32)).cuda()
        sums = torch.empty((B, out_channels, H, W), dtype=torch.int32, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        _check(_lib.bnn_bits_ref_to_nhwc(words.data_ptr(), B, C, H, W, nhwc.data_ptr(), st))
        _check(_lib.bnn_conv_bin(nhwc.data_ptr(), None, B, C, H, W, w.data_ptr(), out_channels,
                                 None, None, 0, 0, None, sums.data_ptr(), None, st))
        return sums.cpu().numpy()


class StagedGpuConvBin:
    """stage (__init__) -> run(WorkItem) -> finish() of backends.py:210-256, one launch per layer."""

    def __init__(self, layer, src, activation_cls=None, int_tensor_cls=None):
        self.layer, self.src = layer, src
        self.w = w_cl_u32(layer)  # the reference caches this on the spec (layer.prepared())
        self._lock = threading.Lock()
        self._done = False
        self.out = None
        self._act_cls, self._int_cls = activation_cls, int_tensor_cls

    def run(self, item) -> None:
        with self._lock:
            if not self._done:
                self.out = conv_bin_forward_gpu(self.src.binary, self.w, len(self.layer.weights))
                self._done = True

    def finish(self):
        if self._act_cls is None:
            return self.out
        return self._act_cls.of_integer(self._int_cls(self.out.shape, self.out))
