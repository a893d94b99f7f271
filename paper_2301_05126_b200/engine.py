"""GPU execution engine: fused-block planner, device buffers, run_model, CUDA graphs.

Counterpart of the reference's ``ExecutionEngine`` (`bnntuner/backends.py:402-543`):
same ``run_model`` / ``execute_layer`` entry points and the same
``RunReport`` / ``TimedResult`` shapes, but each layer runs as a hand-written
sm_100a kernel from libbnn instead of a thread-pool partition, and layers are
fused into blocks:

    conv_int  [+ int maxpool] + step   -> bnn_conv_first   (1 launch)
    conv_bin  [+ int maxpool] + step   -> bnn_conv_bin     (1 launch)
    fc_bin    + step                   -> bnn_fc_bin       (1 launch)
    fc_int_out + argmax                -> bnn_fc_out_argmax (1 launch)

Flatten is free (the next FC's weight columns are permuted at prepare time).
Any other sequence the reference's validator admits (a binary pool after a
step, an unfused int pool, a step on a flattened int activation, ...) falls
back to the standalone GPU kernels -- never to the CPU.

Between blocks activations stay on the device in the NHWC bit layout
(include/bnn.h); only u8 images go in and int32 logits + predictions come out.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import native, prep
from .errors import ConfigNotApplicable, NativeError, ShapeMismatch, ValidationFailed
from .model import LayerKind, applicable_configs, config_of, kind_of, validate_model

# --------------------------------------------------------------------------- reports


@dataclass(frozen=True, eq=False)
class TimedResult:
    """One layer call: output + (overhead, compute) ns (backends.py:131-137).

    overhead = host<->device transfers and boundary re-layout; compute = the
    kernel(s), timed with CUDA events on the launching stream.
    """

    output: object
    overhead_ns: int
    compute_ns: int


@dataclass
class RunReport:
    """Per-layer accumulated times and predictions (backends.py:560-573).

    A fused block's time is booked on its first layer; absorbed layers get 0.
    ``logits`` (int32 (N, classes)) is an addition the reference does not keep.
    """

    predictions: list
    overhead_ns: list
    compute_ns: list
    wall_ns: int
    logits: np.ndarray | None = None

    def accuracy(self, labels) -> float:
        if not labels:
            return 0.0
        return sum(1 for p, t in zip(self.predictions, labels) if p == t) / len(labels)


# --------------------------------------------------------------------------- device activations


@dataclass(frozen=True)
class DevAct:
    """Descriptor of a device activation (per image).

    kind "u8"/"i32img": input images NCHW; "bits": NHWC bits of ``shape``
    (C,H,W) or (L,); "int": NCHW int32 of ``shape``.  ``src`` = the (C,H,W)
    a flattened bit activation came from (drives the FC column permutation).
    """

    kind: str
    shape: tuple
    src: tuple | None = None

    @property
    def words_per_image(self) -> int:
        if len(self.shape) == 1:
            return (self.shape[0] + 31) // 32
        C, H, W = self.shape
        return H * W * ((C + 31) // 32)

    @property
    def elems_per_image(self) -> int:
        return math.prod(self.shape)

    def nhwc_dims(self):
        """(C, H, W) as the kernels see it (1-D = C=L, H=W=1)."""
        if len(self.shape) == 1:
            return (self.shape[0], 1, 1)
        return self.shape

    def fc_src(self):
        """Shape whose flatten order the next FC's weight permutation must follow."""
        if self.src is not None:
            return self.src
        return self.shape


# --------------------------------------------------------------------------- ops

POPC, TC = native.ENGINE_POPC, native.ENGINE_TC


class Op:
    """One launch group of the fused plan.  ``layers`` = reference layer indices covered.

    ``engine``: POPC (bit-packed operands, integer pipe) or TC (FP4 +-1 operands,
    tcgen05 kind::mxf4).  ``out_fmt``: "bits" or "f4" -- whatever the consuming op reads;
    chosen by ``PreparedModel.configure``.
    """

    name = "op"
    variant_kind = None  # block kind for the autotuner, or None if not tunable

    def __init__(self, layers, src: DevAct, dst: DevAct):
        self.layers = list(layers)
        self.src, self.dst = src, dst
        self.variant = None
        self.engine = POPC
        self.out_fmt = "bits"

    def tc_ok(self) -> bool:
        return False

    @property
    def in_fmt(self) -> str:
        return "f4" if self.engine == TC else "bits"

    def out_alloc(self, torch, B, dev):
        if self.dst.kind == "bits":
            if self.out_fmt == "f4":
                return torch.empty((B, self.dst.elems_per_image // 2), dtype=torch.uint8, device=dev)
            return torch.empty((B, self.dst.words_per_image), dtype=torch.int32, device=dev)
        return torch.empty((B, self.dst.elems_per_image), dtype=torch.int32, device=dev)

    def sums_alloc(self, torch, B, dev):
        return None

    def launch(self, lib, x, out, sums, B, stream):
        raise NotImplementedError

    def work_per_image(self) -> dict:
        return {}

    @property
    def fmt_code(self) -> int:
        return native.OUT_F4 if self.out_fmt == "f4" else native.OUT_BITS


def _upload(torch, arr, dev, dtype=None):
    a = np.ascontiguousarray(arr)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    t = torch.from_numpy(a).to(dev)
    return t if dtype is None else t.to(dtype)


def _engine_variant(op):
    """The op's tensor-engine variant as the engine launches it: its filters / thresholds / step rows
    are device tensors uploaded at prepare time, never written by the preceding launch, so the
    kernels may fetch them before their programmatic-dependent-launch wait (BNN_VARIANT_STATIC_WEIGHTS)."""
    v = op.variant
    if v is None:
        v = op._default_variant = getattr(op, "_default_variant", None) or native.Variant.make(TC, 0, 0)
    v.flags = int(v.flags) | native.VARIANT_STATIC_WEIGHTS
    return v


class _StepParams:
    def __init__(self, step_layer, torch, dev):
        self.thr = self.pos = self.flip = self.host = None
        if step_layer is not None:
            t, p = prep.step_params(step_layer.thresholds, step_layer.directions)
            self.host = (t, p)
            self.thr, self.pos = _upload(torch, t, dev), _upload(torch, p, dev)
            # POS flags: the tensor engine's filters are direction-folded when the step is fused
            self.flip = np.array([bool(d) if isinstance(d, (bool, np.bool_)) else prep.is_positive(d)
                                  for d in step_layer.directions], dtype=bool)


class ConvOp(Op):
    def __init__(self, layers, src, dst, conv_layer, step_layer, pool, first, torch, dev):
        super().__init__(layers, src, dst)
        C, H, W = conv_layer.in_shape
        self.C, self.H, self.W, self.K = C, H, W, conv_layer.out_shape[0]
        self.pool, self.first = bool(pool), bool(first)
        self.layer = conv_layer
        self.torch, self.dev = torch, dev
        self.name = ("conv_first" if first else "conv_bin") + ("+pool" if pool else "") + ("+step" if step_layer else "")
        self.variant_kind = "conv_first" if first else "conv_bin"
        if first:
            self.w = _upload(torch, prep.conv_first_weights(conv_layer), dev, torch.int8)
        else:
            self.w = _upload(torch, prep.conv_bin_weights(conv_layer), dev)
        self._w_tc = None
        st = _StepParams(step_layer, torch, dev)
        self.thr, self.pos, self.flip = st.thr, st.pos, st.flip
        self._step_host, self._step_rows = st.host, None
        self.fused_step = step_layer is not None

    def step_mma_ok(self) -> bool:
        """The fused step can enter the accumulator through one extra MMA (bnn_step_rows)."""
        return not self.first and self.fused_step and 9 * self.C <= prep.STEP_ROWS_MAX_KRED

    @property
    def step_rows(self):
        if self._step_rows is None:
            self._step_rows = _upload(self.torch, prep.step_rows(*self._step_host, 9 * self.C), self.dev)
        return self._step_rows

    def tc_ok(self) -> bool:
        if self.first:  # u8 pixels (the model path), one or two K=32 MMAs per tile
            return self.src.kind == "u8" and 9 * self.C <= 64 and self.W <= 128 and self.K <= 256
        return self.C % 64 == 0 and self.W <= 128 and self.K % 32 == 0

    @property
    def w_tc(self):
        if self._w_tc is None:
            self._w_tc = _upload(self.torch, prep.conv_tc_weights(self.layer, self.flip), self.dev)
        return self._w_tc

    def out_alloc(self, torch, B, dev):
        if not self.fused_step:
            return torch.empty((B, self.K * self.H * self.W), dtype=torch.int32, device=dev)
        return super().out_alloc(torch, B, dev)

    def sums_alloc(self, torch, B, dev):
        return torch.empty((B, self.K * self.H * self.W), dtype=torch.int32, device=dev)

    def launch(self, lib, x, out, sums, B, stream):
        p = native.ptr
        if self.fused_step:
            res, sums_out = p(out), p(sums)
        else:
            res, sums_out = None, p(out)
        fmt = self.fmt_code
        if self.first and self.engine == TC and x.element_size() == 1:
            rc = lib.bnn_tc_first(p(x), B, self.C, self.H, self.W, p(self.w), self.K, p(self.thr), p(self.pos),
                                  int(self.pool), fmt, res, sums_out, stream)
        elif self.first:
            rc = lib.bnn_conv_first(p(x), 1 if x.element_size() == 1 else 0, B, self.C, self.H, self.W, p(self.w),
                                    self.K, p(self.thr), p(self.pos), int(self.pool), fmt, res, sums_out, stream)
        elif self.engine == TC:
            v = _engine_variant(self)
            if v.tile_q in (3, 6) and self.step_mma_ok():
                v.step_rows = p(self.step_rows)  # per-tap / HX kernel with the step in the MMA
            rc = lib.bnn_tc_conv(p(x), B, self.C, self.H, self.W, p(self.w_tc), self.K, p(self.thr), p(self.pos),
                                 int(self.pool), fmt, res, sums_out, v, stream)
        else:
            rc = lib.bnn_conv_bin(p(x), None, B, self.C, self.H, self.W, p(self.w), self.K, p(self.thr),
                                  p(self.pos), int(self.pool), fmt, res, sums_out, self.variant, stream)
        native.check(rc, self.name)

    def work_per_image(self) -> dict:
        macs = self.H * self.W * self.K * self.C * 9
        return {"int_mac" if self.first else "bin_mac": macs}


class FcOp(Op):
    def __init__(self, layers, src, dst, fc_layer, step_layer, torch, dev):
        super().__init__(layers, src, dst)
        self.layer = fc_layer
        self.torch, self.dev = torch, dev
        w, self.L, self.LW = prep.fc_weights(fc_layer, src.fc_src())
        self.M = fc_layer.out_shape[0]
        self.w = _upload(torch, w, dev)
        self._w_tc = None
        self.name = "fc_bin" + ("+step" if step_layer else "")
        self.variant_kind = "fc_bin"
        st = _StepParams(step_layer, torch, dev)
        self.thr, self.pos, self.flip = st.thr, st.pos, st.flip
        self.fused_step = step_layer is not None

    def tc_ok(self) -> bool:
        src = self.src.fc_src()
        chans = src[0]
        return chans % 64 == 0 and self.L % 64 == 0 and (self.M % 32 == 0 or not self.fused_step)

    @property
    def w_tc(self):
        if self._w_tc is None:
            self._w_tc = _upload(self.torch, prep.fc_tc_weights(self.layer, self.src.fc_src(), self.flip), self.dev)
        return self._w_tc

    def out_alloc(self, torch, B, dev):
        if not self.fused_step:
            return torch.empty((B, self.M), dtype=torch.int32, device=dev)
        return super().out_alloc(torch, B, dev)

    def sums_alloc(self, torch, B, dev):
        return torch.empty((B, self.M), dtype=torch.int32, device=dev)

    def launch(self, lib, x, out, sums, B, stream):
        p = native.ptr
        if self.fused_step:
            res, sums_out = p(out), p(sums)
        else:
            res, sums_out = None, p(out)
        if self.engine == TC:
            rc = lib.bnn_tc_fc(p(x), B, self.L, p(self.w_tc), self.M, p(self.thr), p(self.pos), self.fmt_code, res,
                               sums_out, None, _engine_variant(self), stream)
        else:
            rc = lib.bnn_fc_bin(p(x), None, B, self.L, self.LW, p(self.w), self.M, p(self.thr), p(self.pos),
                                self.fmt_code, res, sums_out, self.variant, stream)
        native.check(rc, self.name)

    def work_per_image(self) -> dict:
        return {"bin_mac": self.L * self.M}


class FcOutOp(Op):
    name = "fc_out_argmax"
    variant_kind = "fc_out"

    def __init__(self, layers, src, dst, fc_layer, torch, dev):
        super().__init__(layers, src, dst)
        self.layer = fc_layer
        self.torch, self.dev = torch, dev
        w, self.L, self.LW = prep.fc_out_weights(fc_layer, src.fc_src())
        self.M = fc_layer.out_shape[0]
        self.w = _upload(torch, w, dev)
        self._w_tc = None

    def tc_ok(self) -> bool:
        return self.src.fc_src()[0] % 64 == 0 and self.L % 64 == 0 and self.M <= 256

    @property
    def w_tc(self):
        if self._w_tc is None:
            self._w_tc = _upload(self.torch, prep.fc_tc_weights(self.layer, self.src.fc_src()), self.dev)
        return self._w_tc

    def out_alloc(self, torch, B, dev):
        return (torch.empty((B, self.M), dtype=torch.int32, device=dev),
                torch.empty((B,), dtype=torch.int32, device=dev))

    def launch(self, lib, x, out, sums, B, stream):
        logits, preds = out
        p = native.ptr
        if self.engine == TC:
            rc = lib.bnn_tc_fc(p(x), B, self.L, p(self.w_tc), self.M, None, None, native.OUT_LOGITS, p(logits),
                               None, p(preds), _engine_variant(self), stream)
        else:
            rc = lib.bnn_fc_out_argmax(p(x), B, self.L, self.LW, p(self.w), self.M, p(logits), p(preds), stream)
        native.check(rc, self.name)

    def work_per_image(self) -> dict:
        return {"bin_mac": self.L * self.M}


class FrontOp(Op):
    """The first two fused blocks as ONE launch (bnn_tc_front, csrc/tc_front.cu):
    conv_int + step [+ pool]  ->  conv_bin + step [+ pool], the first block's +-1 output kept in
    shared memory.  Wraps the two planning units; their weights / thresholds are reused.
    Replaces ``layer_forward`` calls for layers ``u0.layers + u1.layers`` (layers.py:178-212).
    """

    variant_kind = None

    def __init__(self, u0: "ConvOp", u1: "ConvOp"):
        super().__init__(list(u0.layers) + list(u1.layers), u0.src, u1.dst)
        self.u0, self.u1 = u0, u1
        self.engine = TC
        self.fused_step = True
        self.name = f"front[{u0.name}>{u1.name}]"

    @staticmethod
    def eligible(lib, u0, u1) -> bool:
        return (isinstance(u0, ConvOp) and isinstance(u1, ConvOp) and u0.first and not u1.first
                and u0.fused_step and u1.fused_step and u0.src.kind == "u8" and u0.engine == TC
                and u1.engine == TC and u1.C == u0.K
                and lib.bnn_tc_front_smem(u0.C, u0.H, u0.W, u0.K, u1.K, int(u0.pool), int(u1.pool)) > 0)

    @property
    def out_fmt(self):
        return self.u1.out_fmt

    @out_fmt.setter
    def out_fmt(self, v):  # Op.__init__ assigns a default; the format is the wrapped unit's
        pass

    def sums_alloc(self, torch, B, dev):
        u0, u1 = self.u0, self.u1
        return (torch.empty((B, u0.K * u0.H * u0.W), dtype=torch.int32, device=dev),
                torch.empty((B, u0.dst.elems_per_image // 2), dtype=torch.uint8, device=dev),
                torch.empty((B, u1.K * u1.H * u1.W), dtype=torch.int32, device=dev))

    def launch(self, lib, x, out, sums, B, stream):
        if x.element_size() != 1:
            raise ShapeMismatch("the fused front end reads u8 pixels")
        u0, u1 = self.u0, self.u1
        p = native.ptr
        s1, mid, s2 = sums if sums is not None else (None, None, None)
        rc = lib.bnn_tc_front(p(x), B, u0.C, u0.H, u0.W, p(u0.w), p(u0.thr), p(u0.pos), int(u0.pool), p(u1.w_tc),
                              p(u1.thr), p(u1.pos), int(u1.pool), u0.K, u1.K, self.fmt_code, p(out), p(s1), p(mid),
                              p(s2), stream)
        native.check(rc, self.name)

    def work_per_image(self) -> dict:
        w = dict(self.u0.work_per_image())
        for k, v in self.u1.work_per_image().items():
            w[k] = w.get(k, 0) + v
        return w


class StepOp(Op):
    name = "step"

    def __init__(self, layers, src, dst, step_layer, torch, dev):
        super().__init__(layers, src, dst)
        st = _StepParams(step_layer, torch, dev)
        self.thr, self.pos, self.flip = st.thr, st.pos, st.flip

    def launch(self, lib, x, out, sums, B, stream):
        C, H, W = self.src.nhwc_dims()
        native.check(lib.bnn_step_nhwc(native.ptr(x), B, C, H, W, native.ptr(self.thr), native.ptr(self.pos),
                                       native.ptr(out), stream), self.name)


class PoolOp(Op):
    def __init__(self, layers, src, dst):
        super().__init__(layers, src, dst)
        self.name = "maxpool_bits" if src.kind == "bits" else "maxpool_int"

    def launch(self, lib, x, out, sums, B, stream):
        C, H, W = self.src.shape
        fn = lib.bnn_maxpool_bits_nhwc if self.src.kind == "bits" else lib.bnn_maxpool_int
        native.check(fn(native.ptr(x), B, C, H, W, native.ptr(out), stream), self.name)


class NetPlan:
    """The whole fused plan as ONE launch for batches up to ``max_batch`` (bnn_net_infer,
    csrc/net_b1.cu): the batch-1 latency path.  Grid-wide barriers replace the kernel boundaries
    between blocks, every block's filters are bulk-copied into shared memory at kernel entry, and
    the arithmetic is xor + popcount on the popc engine's NHWC bit words (the same prepared
    filters as ``bnn_conv_first`` / ``bnn_conv_bin`` / ``bnn_fc_bin`` / ``bnn_fc_out_argmax``).
    Covers ``reference_infer`` (layers.py:215-224) for chains of fused blocks
    conv_int [+ pool] + step -> conv_bin [+ pool] + step ... -> fc_bin + step ... -> fc_int_out.
    """

    def __init__(self, pm: "PreparedModel", max_batch: int = 1, grid: int = 0):
        if not NetPlan.eligible(pm):
            raise ConfigNotApplicable("the one-launch network kernel needs conv_int+step, conv_bin+step, "
                                      "fc_bin+step blocks ending in fc_int_out")
        self.pm, self.max_batch, self.grid = pm, int(max_batch), int(grid)
        units = pm.units
        self.layers = (native.NetLayer * len(units))()
        for i, op in enumerate(units):
            d = self.layers[i]
            if isinstance(op, ConvOp):
                d.kind = native.NET_CONV_FIRST if op.first else native.NET_CONV_BIN
                d.C, d.H, d.W, d.K, d.pool = op.C, op.H, op.W, op.K, int(op.pool)
            else:
                d.kind = native.NET_FC_OUT if isinstance(op, FcOutOp) else native.NET_FC_BIN
                d.C, d.H, d.W, d.K, d.pool = op.L, 1, 1, op.M, 0
            d.w = native.ptr(op.w)
            d.thr = native.ptr(getattr(op, "thr", None))
            d.pos = native.ptr(getattr(op, "pos", None))
        nbytes, smem = ctypes.c_size_t(0), ctypes.c_size_t(0)
        native.check(pm.lib.bnn_net_workspace(self.layers, len(units), self.max_batch, self.grid,
                                              ctypes.byref(nbytes), ctypes.byref(smem)), "bnn_net_workspace")
        self.smem = int(smem.value)
        self.ws = pm.torch.empty(int(nbytes.value), dtype=pm.torch.uint8, device=pm.dev)
        self.units = len(units)
        self.prepare()

    def prepare(self):
        """Pack the filters / step constants into the workspace and zero the barrier counter (once per
        plan, and again after a failed launch)."""
        with self.pm.torch.cuda.device(self.pm.dev):
            native.check(self.pm.lib.bnn_net_prepare(self.layers, self.units, self.max_batch, native.ptr(self.ws),
                                                     self.ws.numel(), native.stream_handle()), "bnn_net_prepare")
            self.pm.torch.cuda.current_stream(self.pm.dev).synchronize()

    @staticmethod
    def eligible(pm: "PreparedModel") -> bool:
        u = pm.units
        if len(u) < 2 or len(u) > native.NET_MAX_LAYERS or not isinstance(u[-1], FcOutOp):
            return False
        for i, op in enumerate(u[:-1]):
            if isinstance(op, ConvOp):
                ok = op.fused_step and op.first == (i == 0) and (op.C <= 3 if op.first else True)
            elif isinstance(op, FcOp):
                ok = op.fused_step and i > 0
            else:
                ok = False
            if not ok:
                return False
        return isinstance(u[0], ConvOp) and u[0].first and u[0].src.kind == "u8"

    def launch(self, x, logits, preds, stream=None):
        """x: (B, C, H, W) uint8, device or pinned host (read once over PCIe); logits / preds: device
        or pinned host int32 tensors (written by the kernel directly)."""
        B = int(x.shape[0])
        if B > self.max_batch or B < 1:
            raise ShapeMismatch(f"batch {B} outside 1..{self.max_batch} of this network plan")
        if x.dtype != self.pm.torch.uint8:
            raise ShapeMismatch("the one-launch network kernel reads u8 pixels")
        host = not x.is_cuda
        rc = self.pm.lib.bnn_net_infer(self.layers, self.units, native.ptr(x), int(host), B, native.ptr(logits),
                                       native.ptr(preds), native.ptr(self.ws), self.ws.numel(), self.grid,
                                       native.stream_handle(stream))
        native.check(rc, "bnn_net_infer")


class NetServer:
    """The one-launch network kernel as a resident server for batch-``batch`` requests
    (bnn_net_serve_launch, csrc/net_b1.cu): the kernel stays on every SM with the filters in shared
    memory; a request copies the images into pinned host memory, rings a host-mapped doorbell, spins on
    the completion word and reads the logits / predictions back from pinned memory -- no launch, graph
    or stream synchronisation per request.  It owns the GPU while it runs: ``close()`` (or the context
    manager, or ``idle_s`` seconds without a request) ends it.  ``infer`` is reference_infer
    (layers.py:215-224) for one request."""

    def __init__(self, pm: "PreparedModel", batch: int = 1, idle_s: float = 30.0, timeout_s: float = 5.0):
        torch = pm.torch
        self.pm, self.batch, self.timeout_s = pm, int(batch), float(timeout_s)
        self.net = NetPlan(pm, self.batch)
        shape = (self.batch,) + tuple(pm.model.input.shape)
        self.ctl = torch.zeros(native.NET_CTL_WORDS, dtype=torch.int32).pin_memory()  # page-aligned
        self.h_x = torch.zeros(shape, dtype=torch.uint8).pin_memory()
        self.h_logits = torch.zeros((self.batch, pm.num_classes), dtype=torch.int32).pin_memory()
        self.h_preds = torch.zeros((self.batch,), dtype=torch.int32).pin_memory()
        self.logits = np.zeros((self.batch, pm.num_classes), dtype=np.int32)
        self.preds = np.zeros((self.batch,), dtype=np.int32)
        self.stream = torch.cuda.Stream(pm.dev)
        p = native.ptr
        with torch.cuda.device(pm.dev):
            rc = pm.lib.bnn_net_serve_launch(self.net.layers, self.net.units, self.batch, p(self.net.ws),
                                             self.net.ws.numel(), p(self.ctl), p(self.h_x), p(self.h_logits),
                                             p(self.h_preds), 0, float(idle_s), self.stream.cuda_stream)
        native.check(rc, "bnn_net_serve_launch")
        self.open = True

    def infer(self, images):
        """images: (batch, C, H, W) uint8-valued array -> (logits (batch, classes) int32, preds (batch,) int32)."""
        if not self.open:
            raise NativeError(-2, "NetServer is closed")
        x = np.ascontiguousarray(np.asarray(images.values if hasattr(images, "values") else images,
                                            dtype=np.uint8).reshape(self.h_x.shape))
        p = native.ptr
        rc = self.pm.lib.bnn_net_serve_request(p(self.ctl), x.ctypes.data, x.nbytes, p(self.h_x), p(self.h_logits),
                                               self.logits.ctypes.data, self.logits.nbytes, p(self.h_preds),
                                               self.preds.ctypes.data, self.preds.nbytes, self.timeout_s)
        native.check(rc, "bnn_net_serve_request")
        return self.logits.copy(), self.preds.copy()

    def close(self):
        if self.open:
            self.pm.lib.bnn_net_serve_stop(native.ptr(self.ctl))
            self.stream.synchronize()
            self.open = False

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


# --------------------------------------------------------------------------- planning


def _kinds(model):
    return [kind_of(l) for l in model.layers]


def plan_ops(model, torch, dev) -> list:
    """Greedy fusion of the layer chain into launch groups (see module doc)."""
    layers = model.layers
    kinds = _kinds(model)
    n = len(layers)
    ops = []
    in_kind = "u8"
    act = DevAct(in_kind, tuple(model.input.shape))
    i = 0
    while i < n:
        k = kinds[i]
        L = layers[i]
        if k in (LayerKind.CONV_INT, LayerKind.CONV_BIN):
            j, pool = i + 1, False
            if j < n and kinds[j] is LayerKind.MAXPOOL:
                pool, j = True, j + 1
            if j < n and kinds[j] is LayerKind.STEP:
                Kc, H, W = L.out_shape
                oshape = (Kc, H // 2, W // 2) if pool else (Kc, H, W)
                dst = DevAct("bits", oshape)
                ops.append(ConvOp(range(i, j + 1), act, dst, L, layers[j], pool, k is LayerKind.CONV_INT, torch, dev))
                act, i = dst, j + 1
                continue
            dst = DevAct("int", tuple(L.out_shape))
            ops.append(ConvOp([i], act, dst, L, None, False, k is LayerKind.CONV_INT, torch, dev))
            act, i = dst, i + 1
        elif k is LayerKind.MAXPOOL:
            C, H, W = act.shape
            dst = DevAct(act.kind, (C, H // 2, W // 2))
            ops.append(PoolOp([i], act, dst))
            act, i = dst, i + 1
        elif k is LayerKind.STEP:
            dst = DevAct("bits", act.shape, src=act.src)
            ops.append(StepOp([i], act, dst, L, torch, dev))
            act, i = dst, i + 1
        elif k is LayerKind.FLATTEN:
            length = act.elems_per_image
            src = act.fc_src() if act.kind == "bits" else None
            act = DevAct(act.kind, (length,), src=src)
            if ops:
                ops[-1].layers.append(i)
            i += 1
        elif k is LayerKind.FC_BIN:
            if i + 1 < n and kinds[i + 1] is LayerKind.STEP:
                dst = DevAct("bits", tuple(L.out_shape))
                ops.append(FcOp([i, i + 1], act, dst, L, layers[i + 1], torch, dev))
                act, i = dst, i + 2
            else:
                dst = DevAct("int", tuple(L.out_shape))
                ops.append(FcOp([i], act, dst, L, None, torch, dev))
                act, i = dst, i + 1
        elif k is LayerKind.FC_INT_OUT:
            dst = DevAct("int", tuple(L.out_shape))
            ops.append(FcOutOp([i], act, dst, L, torch, dev))
            act, i = dst, i + 1
        else:  # pragma: no cover
            raise ConfigNotApplicable(f"unsupported layer kind {k}")
    return ops


# --------------------------------------------------------------------------- prepared model


class PreparedModel:
    """Device-resident weights + fused plan for one model on one device."""

    def __init__(self, model, device=None, variants=None, default_engine=None, fuse_front=True):
        import torch

        problems = validate_model(model)
        if problems:
            raise ValidationFailed(problems)
        self.torch = torch
        self.lib = native.device_ready(device)
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        self.model = model
        with torch.cuda.device(self.dev):
            # planning units: one per fused block (the autotuner's cells; variants index these)
            self.units = plan_ops(model, torch, self.dev)
        self.ops = list(self.units)  # what runs: units, with the front pair merged when eligible
        self.num_classes = model.num_classes
        self._bufs: dict = {}
        self.default_engine = TC if default_engine is None else int(default_engine)
        self.fuse_front = bool(fuse_front)
        self.front_min_batch = torch.cuda.get_device_properties(self.dev).multi_processor_count
        self.set_variants(variants)

    # -- variants (autotuner plans) -------------------------------------------------
    def tunable_ops(self):
        return [i for i, op in enumerate(self.units) if op.variant_kind is not None]

    def set_variants(self, variants, default_engine=None):
        """variants: {op index: native.Variant | tuple(engine, tile_n, tile_q)} or None.

        Ops without an explicit variant use ``default_engine`` (TC where the
        tensor engine can run the op, else POPC).  Engines fix the operand
        formats, so every op's output format is then set to what its consumer
        reads, and device buffers are re-allocated.
        """
        if default_engine is None:
            default_engine = self.default_engine
        for op in self.units:
            op.variant = None
            op.engine = TC if (default_engine == TC and op.tc_ok()) else POPC
        for idx, v in (variants or {}).items():
            # an engine-owned copy: the launches below set engine-specific flags on it
            v = native.Variant.make(v.engine, v.tile_n, v.tile_q, v.imgs) if isinstance(v, native.Variant) \
                else native.Variant.make(*v)
            op = self.units[int(idx)]
            op.engine = TC if (v.engine == TC and op.tc_ok()) else POPC
            # a tensor-engine variant the op cannot run falls back to the popc kernel's own default
            op.variant = v if v.engine == op.engine else None
        self._configure_formats()
        self.ops = list(self.units)
        if self.fuse_front and len(self.units) >= 2 and FrontOp.eligible(self.lib, self.units[0], self.units[1]):
            self.ops = [FrontOp(self.units[0], self.units[1])] + self.units[2:]
        self._bufs.clear()

    def set_fuse_front(self, on: bool):
        """Enable/disable the one-launch front end (bnn_tc_front); keeps the current variants."""
        self.fuse_front = bool(on)
        self.set_variants({i: u.variant for i, u in enumerate(self.units) if u.variant is not None})

    def _configure_formats(self):
        for i, op in enumerate(self.units):
            nxt = self.units[i + 1] if i + 1 < len(self.units) else None
            want = nxt.in_fmt if nxt is not None else "bits"
            can_f4 = isinstance(op, (ConvOp, FcOp)) and op.fused_step and op.dst.kind == "bits"
            if want == "f4" and not can_f4:
                # the consumer cannot read this producer's format: fall back to popc for it (with
                # the popc kernel's default variant -- a tensor-engine variant means nothing there)
                nxt.engine = POPC
                if nxt.variant is not None and nxt.variant.engine != POPC:
                    nxt.variant = None
                want = "bits"
            op.out_fmt = want

    def engines(self) -> list:
        return [("tc" if op.engine == TC else "popc") for op in self.ops]

    def exec_ops(self, x=None) -> list:
        """The launch list for input ``x``.

        The fused front end reads u8 pixels only, and runs one image per CTA at a time, so below
        ``front_min_batch`` images (default: one per SM) the two separate kernels, which spread an
        image's tiles over many SMs, are used instead (the batch-1 latency path)."""
        if self.ops and isinstance(self.ops[0], FrontOp) and x is not None:
            if x.element_size() != 1 or int(x.shape[0]) < self.front_min_batch:
                return self.units
        return self.ops

    # -- buffers ----------------------------------------------------------------------
    def buffers(self, B: int, keep_sums: bool = False, ops=None):
        """Per-op output (and debug sums) buffers for batch ``B``.

        A set allocated for a larger batch is reused through leading-dimension views, so a stream
        of batch sizes (run_model's short first / last batches) never allocates in steady state.
        """
        ops = self.ops if ops is None else ops
        unfused = ops is self.units and ops is not self.ops
        key = (B, keep_sums, unfused)
        if key not in self._bufs:
            bigger = [k for k in self._bufs if k[1] == keep_sums and k[2] == unfused and k[0] > B]
            if bigger:
                outs, sums = self._bufs[min(bigger)]

                def view(t):
                    if t is None:
                        return None
                    if isinstance(t, (tuple, list)):
                        return type(t)(view(u) for u in t)
                    return t[:B]

                self._bufs[key] = ([view(o) for o in outs], [view(x) for x in sums])
            else:
                t = self.torch
                outs = [op.out_alloc(t, B, self.dev) for op in ops]
                sums = [op.sums_alloc(t, B, self.dev) if keep_sums else None for op in ops]
                self._bufs[key] = (outs, sums)
        return self._bufs[key]

    def release(self):
        self._bufs.clear()

    # -- the hot path ---------------------------------------------------------------
    def infer(self, x, keep_sums: bool = False, stream=None, events=None, out=None):
        """Run the plan on device images ``x`` ((B,C,H,W) uint8 or int32 CUDA tensor).

        Returns (logits (B, classes) int32, preds (B,) int32): views of
        engine-owned buffers, overwritten by the next call at the same batch size.
        ``events``: optional list of (start, end) torch.cuda.Event per op.
        ``out``: optional (logits, preds) destination for the last block -- e.g. pinned
        host tensors, which the kernel writes through the unified address space
        (zero-copy); ``x`` may likewise be a pinned host tensor.
        """
        B = int(x.shape[0])
        if tuple(x.shape[1:]) != tuple(self.model.input.shape):
            raise ShapeMismatch(f"images {tuple(x.shape)} do not match input {self.model.input.shape}")
        ops = self.exec_ops(x)
        outs, sums = self.buffers(B, keep_sums, ops)
        st = native.stream_handle(stream)
        cur = x
        last = len(ops) - 1
        for i, op in enumerate(ops):
            if events is not None:
                events[i][0].record()
            dst = out if (out is not None and i == last) else outs[i]
            op.launch(self.lib, cur, dst, sums[i], B, st)
            if events is not None:
                events[i][1].record()
            cur = outs[i]
        return out if out is not None else outs[-1]

    def launches_per_batch(self, B: int | None = None) -> int:
        if B is not None and self.ops and isinstance(self.ops[0], FrontOp) and B < self.front_min_batch:
            return len(self.units)
        return len(self.ops)

    def work_per_image(self) -> dict:
        tot: dict = {}
        for op in self.ops:
            for k, v in op.work_per_image().items():
                tot[k] = tot.get(k, 0) + v
        return tot


# --------------------------------------------------------------------------- engine


def _as_pixels(images) -> np.ndarray:
    """IntTensor / ndarray (N,C,H,W) -> uint8 if every pixel is 0..255, else int32."""
    vals = np.asarray(images.values if hasattr(images, "values") else images)
    if vals.dtype == np.uint8:
        return np.ascontiguousarray(vals)
    if vals.size and (vals.min() < 0 or vals.max() > 255):
        return np.ascontiguousarray(vals.astype(np.int32))
    return np.ascontiguousarray(vals.astype(np.uint8))


class Engine:
    """GPU engine with the reference ExecutionEngine's interface (backends.py:402-543).

    ``Engine(workers=None, window_rows=1, fuse_transfers=False, clock=time.perf_counter_ns, *,
    device=None, devices=None, default_engine=None)``; context manager.

    The positional arguments are the reference's (`backends.py:411-420`, called positionally by
    `bnntuner/cli.py:150,206,264`) with the same validation; on the GPU they do not shape the
    computation: ``workers`` is the number of host threads driving devices (default: one per
    device), ``window_rows`` is validated and kept for plan/profile metadata, and
    ``fuse_transfers`` is always in effect (activations never leave the device between layers).

    ``devices``: CUDA device indices.  With more than one, ``run_model`` shards the images by
    contiguous ranges across them: one host thread and one pair of streams per
    device, weights replicated, no collective; only logits and predictions come back, in image
    order.  The same index may repeat (``devices=[0, 0]`` runs two independent shards on one GPU,
    which exercises the sharding logic on a single-GPU box).  ``prepare`` / ``graph`` /
    ``execute_layer`` / ``infer`` of a multi-device engine use ``devices[0]``.
    """

    def __init__(self, workers=None, window_rows=1, fuse_transfers=False, clock=time.perf_counter_ns, *,
                 device=None, devices=None, default_engine=None):
        import torch

        if workers is not None and int(workers) < 1:
            raise ValueError("workers must be >= 1")
        if int(window_rows) < 1:
            raise ValueError("window_rows must be >= 1")
        if device is not None and devices is not None:
            raise ValueError("pass device or devices, not both")
        self.torch = torch
        if devices is None:
            native.device_ready(device)
            devices = [torch.cuda.current_device() if device is None else int(device)]
        devices = [int(d) for d in devices]
        if not devices:
            raise ValueError("devices must not be empty")
        for d in sorted(set(devices)):
            native.device_ready(d)
        self.devices = devices
        self.device = devices[0]
        self.window_rows = int(window_rows)
        self.fuse_transfers = bool(fuse_transfers)
        self.clock = clock
        self.workers = len(devices) if workers is None else int(workers)
        self.default_engine = TC if default_engine is None else int(default_engine)
        self._prepared: dict = {}
        self._staging: dict = {}
        self._shards = None  # per-device engines of a multi-device engine (built on first use)
        self._pool = None

    def close(self):
        self._prepared.clear()
        self._staging.clear()
        if self._shards:
            for e in self._shards:
                e.close()
        self._shards = None
        if self._pool is not None:
            self._pool.shutdown(wait=True)
            self._pool = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    # -- model preparation ------------------------------------------------------------
    def prepare(self, model, variants=None) -> PreparedModel:
        key = id(model)
        pm = self._prepared.get(key)
        if pm is None or pm.model is not model:
            with self.torch.cuda.device(self.device):
                pm = PreparedModel(model, self.device, variants, self.default_engine)
            self._prepared[key] = pm
        elif variants is not None:
            pm.set_variants(variants)
        return pm

    # -- whole model ----------------------------------------------------------------
    @staticmethod
    def _resolve_assignments(model, assignments):
        """(variants, batch size) of a run_model ``assignments`` argument.

        * an autotuner ``ExecPlan``: its per-block variants and batch size;
        * a {block index: variant} dict;
        * the reference's per-layer ``list[ParallelConfig]`` (ours or the reference's enum):
          validated exactly as `backends.py:514-518` does (length -> ShapeMismatch, applicability
          -> ConfigNotApplicable); the engine's current (default or tuned) variants then run it,
          since the CPU/X/Y/Z thread partitions have no meaning on the GPU;
        * None: the current variants.
        """
        if assignments is None:
            return None, None
        if hasattr(assignments, "variant_map"):
            return assignments.variant_map(), assignments.batch_size
        if isinstance(assignments, dict):
            return assignments, None
        tags = list(assignments)
        if len(tags) != len(model.layers):
            raise ShapeMismatch(f"{len(tags)} assignments for {len(model.layers)} layers")
        for layer, tag in zip(model.layers, tags):
            try:
                cfg = config_of(tag)
            except ValueError:
                raise ConfigNotApplicable(f"{tag!r} is not a ParallelConfig") from None
            if cfg not in applicable_configs(layer.kind):
                raise ConfigNotApplicable(f"{cfg.value} not applicable to {kind_of(layer).value}")
        return None, None

    def run_model(self, model, images, assignments=None, batch_size=None, *, keep_logits=True) -> RunReport:
        """Batches of host images through the fused GPU plan (backends.py:506-543).

        ``assignments``: see ``_resolve_assignments``.  ``batch_size`` (default: all images in
        one batch; must be >= 1, ValueError as in the reference).  The last batch may be short;
        an empty image set returns an empty report.

        Pipelined over two streams: while batch i computes, the copy stream uploads
        batch i+1 (ping-pong device input buffers) and downloads batch i-1's logits and
        predictions straight into one pinned host result buffer, so host<->device traffic
        hides behind the kernels.  compute = CUDA-event kernel time per fused block;
        overhead = the part of the wall time not covered by kernels (exposed transfers,
        launch, synchronisation), booked on the first layer.  A multi-device engine runs one
        such pipeline per device on its image shard (``_run_sharded``).
        """
        variants, bs = self._resolve_assignments(model, assignments)
        if batch_size is not None:
            bs = batch_size
        if bs is not None and int(bs) < 1:
            raise ValueError("batch_size must be >= 1")
        host = self._pinned(images)
        n = int(host.shape[0])
        if tuple(host.shape[1:]) != tuple(model.input.shape):
            raise ShapeMismatch(f"images {tuple(host.shape)} do not match input {tuple(model.input.shape)}")
        if n == 0:
            nl = len(model.layers)
            empty = np.empty((0, model.num_classes), dtype=np.int32) if keep_logits else None
            return RunReport([], [0] * nl, [0] * nl, 0, empty)
        if len(self.devices) > 1:
            return self._run_sharded(model, host, variants, bs, keep_logits)
        return self._run_local(model, host, variants, int(bs or n), keep_logits)

    def _pinned(self, images):
        torch = self.torch
        if hasattr(images, "is_pinned"):  # a host torch tensor (pinned once by the caller)
            return images if images.is_pinned() else images.pin_memory()
        return torch.from_numpy(_as_pixels(images)).pin_memory()

    def _shard_engines(self) -> list:
        if self._shards is None:
            from concurrent.futures import ThreadPoolExecutor

            self._shards = [Engine(clock=self.clock, device=d, default_engine=self.default_engine)
                            for d in self.devices]
            self._pool = ThreadPoolExecutor(max_workers=max(self.workers, len(self.devices)))
        return self._shards

    def _run_sharded(self, model, host, variants, bs, keep_logits) -> RunReport:
        """Image sharding over ``self.devices``: contiguous ranges (parallel.shard_bounds), one host
        thread per device, each running the single-device pipeline on its shard; the reports are
        concatenated in image order (predictions, logits) and summed per layer (times)."""
        from .parallel import shard_bounds

        n = int(host.shape[0])
        subs = self._shard_engines()
        if variants is None and id(model) in self._prepared:  # a plan set through self.prepare()
            pm0 = self._prepared[id(model)]
            variants = {i: (u.variant.engine, u.variant.tile_n, u.variant.tile_q, u.variant.imgs)
                        for i, u in enumerate(pm0.units) if u.variant is not None}
        spans = [shard_bounds(n, len(subs), r) for r in range(len(subs))]
        t0 = self.clock()
        futs = [self._pool.submit(e._run_local, model, host[lo:hi], variants, int(bs or (hi - lo) or 1), keep_logits)
                for e, (lo, hi) in zip(subs, spans) if hi > lo]
        reps = [f.result() for f in futs]
        wall = self.clock() - t0
        nl = len(model.layers)
        preds = [p for r in reps for p in r.predictions]
        logits = np.concatenate([r.logits for r in reps]) if keep_logits else None
        ovh = [sum(r.overhead_ns[i] for r in reps) for i in range(nl)]
        comp = [sum(r.compute_ns[i] for r in reps) for i in range(nl)]
        return RunReport(preds, ovh, comp, int(wall), logits)

    def _run_local(self, model, host, variants, bs: int, keep_logits: bool) -> RunReport:
        torch = self.torch
        n = int(host.shape[0])
        pm = self.prepare(model, variants)
        nl = len(model.layers)
        overhead, compute = [0] * nl, [0] * nl
        t_start = self.clock()
        dev = f"cuda:{self.device}"
        with torch.cuda.device(self.device):
            nb = (n + bs - 1) // bs
            nbuf = 2 if nb > 1 else 1
            # staging buffers and the copy stream are reused across calls (pinning host memory and
            # allocating device buffers per call would cost more than the transfers they stage)
            key = (tuple(host.shape[1:]), host.dtype, bs, nbuf, model.num_classes)
            st = self._staging.get(key)
            if st is None:
                st = {"d_in": [torch.empty((bs,) + tuple(host.shape[1:]), dtype=host.dtype, device=dev)
                               for _ in range(nbuf)],
                      "d_out": [(torch.empty((bs, model.num_classes), dtype=torch.int32, device=dev),
                                 torch.empty((bs,), dtype=torch.int32, device=dev)) for _ in range(nbuf)],
                      "copy": torch.cuda.Stream(), "h": None}
                self._staging = {key: st}  # keep only the latest shape
            d_in, d_out, copy = st["d_in"], st["d_out"], st["copy"]
            if st["h"] is None or st["h"][0].shape[0] < n:
                st["h"] = (torch.empty((n, model.num_classes), dtype=torch.int32).pin_memory(),
                           torch.empty((n,), dtype=torch.int32).pin_memory())
            h_logits, h_preds = st["h"][0][:n], st["h"][1][:n]
            comp = torch.cuda.current_stream()
            loaded = [torch.cuda.Event() for _ in range(nbuf)]
            done = [torch.cuda.Event() for _ in range(nbuf)]
            # batch bounds: a short first batch, so the only upload that cannot overlap compute is small
            first = bs // 8 if (nb > 1 and bs >= 2048) else bs
            bounds, lo = [], 0
            while lo < n:
                hi = min(lo + (first if not bounds else bs), n)
                bounds.append((lo, hi))
                lo = hi
            # ... and a short last batch: what runs after the last kernel (its copies back and the host-side
            # collection of its predictions) is then small too
            if len(bounds) > 2 and first < bs and bounds[-1][1] - bounds[-1][0] > first:
                lo, hi = bounds.pop()
                bounds += [(lo, hi - first), (hi - first, hi)]
            nb = len(bounds)
            fetched = [torch.cuda.Event() for _ in range(nb)]
            timed = []  # (launch list, events) per batch: a short batch may run a different launch list
            preds_all: list = []
            logits_all = np.empty((n, model.num_classes), dtype=np.int32) if keep_logits else None

            def upload(i):
                lo, hi = bounds[i]
                k = i % nbuf
                with torch.cuda.stream(copy):
                    if i >= nbuf:
                        copy.wait_event(done[k])  # batch i-2 finished reading this input buffer
                    d_in[k][: hi - lo].copy_(host[lo:hi], non_blocking=True)
                    loaded[k].record(copy)

            def collect(i):
                # host side of batch i, while the GPU works on later batches
                lo, hi = bounds[i]
                fetched[i].synchronize()
                preds_all.extend(h_preds[lo:hi].numpy().tolist())
                if keep_logits:
                    logits_all[lo:hi] = h_logits[lo:hi].numpy()

            upload(0)
            for i in range(nb):
                lo, hi = bounds[i]
                k = i % nbuf
                if i + 1 < nb:
                    upload(i + 1)
                comp.wait_event(loaded[k])
                xb = d_in[k][: hi - lo]
                ops = pm.exec_ops(xb)  # below front_min_batch images the unfused front runs
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in ops]
                lg, pr = d_out[k]
                pm.infer(xb, events=ev, out=(lg[: hi - lo], pr[: hi - lo]))
                done[k].record(comp)
                timed.append((ops, ev))
                with torch.cuda.stream(copy):
                    copy.wait_event(done[k])
                    h_logits[lo:hi].copy_(lg[: hi - lo], non_blocking=True)
                    h_preds[lo:hi].copy_(pr[: hi - lo], non_blocking=True)
                    fetched[i].record(copy)
                if i >= 1:
                    collect(i - 1)
            copy.synchronize()
            comp.synchronize()
            collect(nb - 1)
            for ops, ev in timed:
                for op, (a_, z_) in zip(ops, ev):
                    compute[op.layers[0]] += int(a_.elapsed_time(z_) * 1e6)
        wall = self.clock() - t_start
        overhead[0] = max(0, int(wall) - sum(compute))
        return RunReport(preds_all, overhead, compute, int(wall), logits_all)

    def infer(self, model, images):
        """(logits int32 (N, classes), preds list[int]) for host images, one batch (per device)."""
        rep = self.run_model(model, images)
        return rep.logits, rep.predictions

    # -- single layer -----------------------------------------------------------------
    def execute_layer(self, layer, act, config=None, batch_size=None) -> TimedResult:
        """One layer through the GPU layer API, timed (backends.py:436-448).

        ``config``: a kernel ``native.Variant`` (the tensor or popc engine for conv_bin / fc), a
        reference ``ParallelConfig`` tag (validated for applicability as `backends.py:456-461`
        does; the layer then runs on its default GPU kernel) or None.
        """
        from . import layers as L

        if batch_size is not None and act.batch != batch_size:
            raise ShapeMismatch(f"batch {act.batch} != requested batch_size {batch_size}")
        if tuple(act.sample_shape) != tuple(layer.in_shape):
            raise ShapeMismatch(
                f"{kind_of(layer).value} expects sample shape {tuple(layer.in_shape)}, got {tuple(act.sample_shape)}")
        variant = config
        if config is not None and not isinstance(config, native.Variant):
            if isinstance(config, tuple):
                variant = native.Variant.make(*config)
            else:
                try:
                    cfg = config_of(config)
                except ValueError:
                    raise ConfigNotApplicable(f"{config!r} is not a ParallelConfig or kernel variant") from None
                if cfg not in applicable_configs(layer.kind):
                    raise ConfigNotApplicable(f"{cfg.value} not applicable to {kind_of(layer).value}")
                variant = None
        timer = L.LayerTimer(self.torch)
        t0 = self.clock()
        with self.torch.cuda.device(self.device):
            out = L.layer_forward(layer, act, timer=timer, variant=variant)
        if timer.compute_ns == 0 and timer.overhead_ns == 0:
            # no kernel (flatten is a host-side relabelling, layers.py:149-161): like the reference's
            # CPU path (backends.py:463-468) the whole call is compute
            return TimedResult(out, 0, max(1, int(self.clock() - t0)))
        return TimedResult(out, timer.overhead_ns, timer.compute_ns)

    # -- batch-1 latency path -----------------------------------------------------------
    def serve(self, model, batch: int = 1, idle_s: float = 30.0) -> "NetServer":
        """A resident one-launch server for batch-``batch`` requests (NetServer; the batch-1 latency path)."""
        return NetServer(self.prepare(model), batch, idle_s)

    def graph(self, model, batch: int = 1, variants=None, zero_copy: bool = False, net: bool = False) -> "GraphRunner":
        """CUDA Graph of one request.  ``net``: the whole model as ONE kernel (NetPlan, the batch-1
        latency path) instead of one launch per fused block."""
        return GraphRunner(self.prepare(model, variants), batch, zero_copy, net)


ExecutionEngine = Engine


class GraphRunner:
    """CUDA-Graph replay of H2D(images) -> fused kernels -> D2H(logits, preds).

    The paper's central finding is that per-layer launch/transfer overhead
    dominates small batches; here the whole request is one graph launch.
    """

    def __init__(self, pm: PreparedModel, batch: int = 1, zero_copy: bool = False, net: bool = False):
        """zero_copy: the first kernel reads the pinned host images and the last kernel writes
        logits/preds into pinned host memory directly (unified addressing) -- no copy nodes.
        net: one launch for the whole model (NetPlan) instead of one per fused block."""
        torch = pm.torch
        self.pm, self.batch, self.zero_copy = pm, int(batch), bool(zero_copy)
        self.net = NetPlan(pm, self.batch) if net else None
        shape = (self.batch,) + tuple(pm.model.input.shape)
        self._bufs_ref = pm.buffers(self.batch)  # the graph bakes these pointers in: keep them alive
        with torch.cuda.device(pm.dev):
            self.h_in = torch.zeros(shape, dtype=torch.uint8).pin_memory()
            self.d_in = torch.zeros(shape, dtype=torch.uint8, device=pm.dev)
            self.h_logits = torch.zeros((self.batch, pm.num_classes), dtype=torch.int32).pin_memory()
            self.h_preds = torch.zeros((self.batch,), dtype=torch.int32).pin_memory()
            self.d_logits = torch.zeros((self.batch, pm.num_classes), dtype=torch.int32, device=pm.dev)
            self.d_preds = torch.zeros((self.batch,), dtype=torch.int32, device=pm.dev)
            self.stream = torch.cuda.Stream(pm.dev)
            with torch.cuda.stream(self.stream):
                for _ in range(2):  # warm-up: buffers allocated, smem attributes set
                    self._body()
            self.stream.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self.stream):
                self._body()
        # the launch list this graph replays (unfused front below one image per SM)
        self.ops = ["net"] if self.net is not None else pm.exec_ops(self.d_in)
        self.launches = len(self.ops)
        self._kernels = None

    def kernels_only_us(self, reps: int = 200) -> float:
        """Device time of the fused kernels alone (no H2D/D2H), from a graph of the same plan."""
        torch = self.pm.torch
        if self._kernels is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                if self.net is not None:
                    self.net.launch(self.d_in, self.d_logits, self.d_preds)
                else:
                    self.pm.infer(self.d_in)
            self._kernels = g
        self._kernels.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            self._kernels.replay()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) * 1e3 / reps

    def _body(self):
        if self.net is not None:
            if self.zero_copy:
                self.net.launch(self.h_in, self.h_logits, self.h_preds)
                return
            self.d_in.copy_(self.h_in, non_blocking=True)
            self.net.launch(self.d_in, self.d_logits, self.d_preds)
            self.h_logits.copy_(self.d_logits, non_blocking=True)
            self.h_preds.copy_(self.d_preds, non_blocking=True)
            return
        if self.zero_copy:
            self.pm.infer(self.h_in, out=(self.h_logits, self.h_preds))
            return
        self.d_in.copy_(self.h_in, non_blocking=True)
        logits, preds = self.pm.infer(self.d_in)
        self.h_logits.copy_(logits, non_blocking=True)
        self.h_preds.copy_(preds, non_blocking=True)

    def replay(self, images=None):
        """Run one request; returns (logits (B, classes) int32, preds (B,) int32) numpy copies."""
        if images is not None:
            self.h_in.numpy()[...] = np.asarray(images.values if hasattr(images, "values") else images,
                                                dtype=np.uint8).reshape(self.h_in.shape)
        self.graph.replay()
        self.graph_stream_sync()
        return self.h_logits.numpy().copy(), self.h_preds.numpy().copy()

    def graph_stream_sync(self):
        self.pm.torch.cuda.current_stream(self.pm.dev).synchronize()
