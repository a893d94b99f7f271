"""ctypes binding of libbnn.so (include/bnn.h) -- the only door to the GPU.

There is deliberately no fallback: if the library or a CUDA device is
missing, every entry point raises ``NativeUnavailable``.  Buffers are torch
CUDA tensors (torch is plumbing here: device memory and streams); calls are
issued on torch's current stream so they compose with torch copies and CUDA
graphs.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import NativeError, NativeUnavailable

import os

# BNN_LIB: an alternative build of the same library (A/B experiments, tools/); default: the in-tree one
LIB_PATH = Path(os.environ.get("BNN_LIB") or Path(__file__).resolve().with_name("libbnn.so"))

P = ctypes.c_void_p
I = ctypes.c_int
LL = ctypes.c_longlong


OUT_BITS, OUT_F4, OUT_LOGITS = 0, 1, 2  # OUT_F4: NHWC FP4 +-1, the tensor engine's operand format
VARIANT_STATIC_WEIGHTS = 1  # bnn_variant.flags (include/bnn.h)
ENGINE_POPC, ENGINE_TC = 0, 1


class Variant(ctypes.Structure):
    """bnn_variant (include/bnn.h): engine 0 = popc, 1 = tensor; tiles."""

    _fields_ = [("engine", I), ("tile_n", I), ("tile_q", I), ("imgs", I), ("step_rows", P), ("flags", I),
                ("reserved", I)]

    @classmethod
    def make(cls, engine: int = 0, tile_n: int = 0, tile_q: int = 0, imgs: int = 0) -> "Variant":
        v = cls()
        v.engine, v.tile_n, v.tile_q, v.imgs = int(engine), int(tile_n), int(tile_q), int(imgs)
        return v

    def key(self) -> tuple:
        return (int(self.engine), int(self.tile_n), int(self.tile_q))

    def __repr__(self) -> str:
        return f"Variant(engine={self.engine}, tile_n={self.tile_n}, tile_q={self.tile_q})"


NET_CONV_FIRST, NET_CONV_BIN, NET_FC_BIN, NET_FC_OUT = 0, 1, 2, 3  # bnn_net_layer.kind
NET_MAX_LAYERS = 16
NET_CTL_WORDS = 64  # bnn_net_serve_* control block (host-written words and device-written words on separate lines)


class NetLayer(ctypes.Structure):
    """bnn_net_layer (include/bnn.h): one fused block of the one-launch network kernel."""

    _fields_ = [("kind", I), ("C", I), ("H", I), ("W", I), ("K", I), ("pool", I), ("w", P), ("thr", P),
                ("pos", P)]


# name -> (restype, argtypes)
_SIGS = {
    "bnn_abi_version": (I, []),
    "bnn_last_error": (ctypes.c_char_p, []),
    "bnn_launch_count": (LL, [I]),
    "bnn_init": (I, [I]),
    "bnn_bits_ref_to_nhwc": (I, [P, I, I, I, I, P, P]),
    "bnn_bits_nhwc_to_ref": (I, [P, I, I, I, I, P, P]),
    "bnn_step_ref": (I, [P, I, I, LL, P, P, P, P]),
    "bnn_step_nhwc": (I, [P, I, I, I, I, P, P, P, P]),
    "bnn_maxpool_int": (I, [P, I, I, I, I, P, P]),
    "bnn_maxpool_bits_nhwc": (I, [P, I, I, I, I, P, P]),
    "bnn_conv_first": (I, [P, I, I, I, I, I, P, I, P, P, I, I, P, P, P]),
    "bnn_conv_bin": (I, [P, P, I, I, I, I, P, I, P, P, I, I, P, P, ctypes.POINTER(Variant), P]),
    "bnn_fc_bin": (I, [P, P, I, I, I, P, I, P, P, I, P, P, ctypes.POINTER(Variant), P]),
    "bnn_fc_out_argmax": (I, [P, I, I, I, P, I, P, P, P]),
    "bnn_tc_conv": (I, [P, I, I, I, I, P, I, P, P, I, I, P, P, ctypes.POINTER(Variant), P]),
    "bnn_tc_first": (I, [P, I, I, I, I, P, I, P, P, I, I, P, P, P]),
    "bnn_tc_fc": (I, [P, I, I, P, I, P, P, I, P, P, P, ctypes.POINTER(Variant), P]),
    "bnn_tc_front": (I, [P, I, I, I, I, P, P, P, I, P, P, P, I, I, I, I, P, P, P, P, P]),
    "bnn_tc_front_smem": (I, [I, I, I, I, I, I, I]),
    "bnn_tc_front_trace": (I, [P]),
    "bnn_tc_trace": (I, [P]),
    "bnn_step_rows": (I, [P, P, I, I, P]),
    "bnn_bits_to_f4": (I, [P, LL, I, P, P]),
    "bnn_f4_to_bits": (I, [P, LL, I, P, P]),
    "bnn_xnor_dot": (I, [P, P, P, P, I, ctypes.POINTER(LL), P]),
    "bnn_net_workspace": (I, [ctypes.POINTER(NetLayer), I, I, I, ctypes.POINTER(ctypes.c_size_t),
                              ctypes.POINTER(ctypes.c_size_t)]),
    "bnn_net_infer": (I, [ctypes.POINTER(NetLayer), I, P, I, I, P, P, P, ctypes.c_size_t, I, P]),
    "bnn_net_prepare": (I, [ctypes.POINTER(NetLayer), I, I, P, ctypes.c_size_t, P]),
    "bnn_net_trace": (I, [P]),
    "bnn_net_serve_launch": (I, [ctypes.POINTER(NetLayer), I, I, P, ctypes.c_size_t, P, P, P, P, I, ctypes.c_double, P]),
    "bnn_net_serve_request": (I, [P, P, ctypes.c_size_t, P, P, P, ctypes.c_size_t, P, P, ctypes.c_size_t,
                                  ctypes.c_double]),
    "bnn_net_serve_stop": (I, [P]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None
_inited: set = set()


def load(path: Path | None = None):
    """Load libbnn.so and bind every entry point (no GPU needed for this step)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise NativeUnavailable(
                f"{p} is missing; build it with `python -m paper_2301_05126_b200.csrc.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    return (load().bnn_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        raise NativeError(rc, f"{what}: {last_error()}" if what else last_error())


def launches(reset: bool = False) -> int:
    return int(load().bnn_launch_count(1 if reset else 0))


def device_ready(device=None):
    """Import torch, check a CUDA device is present and libbnn supports it."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible; libbnn has no CPU fallback")
    lib = load()
    dev = torch.cuda.current_device() if device is None else int(getattr(device, "index", device) or 0)
    if dev not in _inited:
        check(lib.bnn_init(dev), "bnn_init")
        _inited.add(dev)
    return lib


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else int(t.data_ptr())
