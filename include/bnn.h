/*
 * bnn.h -- C ABI of libbnn, the sm_100a BNN inference kernels.
 *
 * The reference (arXiv 2301.05126's `bnntuner`, pure Python + numpy) has no
 * FFI; these entry points replace the per-layer compute functions that its
 * Python layer API and execution engine call.  Each declaration cites the
 * reference function whose numerics it reproduces (paths relative to
 * /root/reference/pkg/src/bnntuner/).  The Python binding that calls them
 * is paper_2301_05126_b200/native.py (ctypes); INTEGRATION.md shows how a
 * maintainer would bind them from the reference package.
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless named host_*; the caller owns every
 *    buffer; the library never allocates or frees on a hot call.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous, stream-ordered and CUDA-Graph capturable (no sync, no
 *    malloc, no host callbacks).
 *  - Return 0 on success, <0 for an argument error detected before any launch
 *    (message in bnn_last_error(), thread-local), >0 = a cudaError_t.
 *  - Device binary layout ("NHWC bits"): activation (b, c, y, x) is bit c%32
 *    of u32 word [((b*H + y)*W + x)*CW + c/32], CW = ceil(C/32), tail bits 0;
 *    bit 1 = +1, bit 0 = -1 (the reference's value convention, tensors.py:1-8).
 *    1-D activations are NHWC with H = W = 1.
 *  - Reference layout ("ref bits"): the reference's BinaryTensor words, element
 *    i of the row-major (B,C,H,W) flat index is bit i%64 of u64 word i/64
 *    (tensors.py:29-46).
 *  - Device FP4 layout ("NHWC f4"): the tensor-engine operand format, one E2M1
 *    nibble per element, +1 = 0x2, -1 = 0xA (0x0 = padding), same NHWC order, element
 *    c of a pixel in nibble c%2 (low first) of byte c/2; C % 64 == 0.  A binary dot
 *    product is then an exact block-scaled FP4 MMA (tcgen05 kind::mxf4, unit scales).
 *  - Direction bits `posbits`: bit k of u32 word k/32 is 1 for POS (v > T),
 *    0 for NEG (v < T) (model.py:70-74, layers.py:135-146).
 *  - out_fmt: BNN_OUT_BITS (NHWC bits, u32 words) or BNN_OUT_F4 (NHWC FP4 +-1,
 *    needs K % 32 == 0) selects the fused epilogue's output format.
 */
#ifndef BNN_H
#define BNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BNN_ABI_VERSION 7

#if defined(__GNUC__)
#define BNN_API __attribute__((visibility("default")))
#else
#define BNN_API
#endif

#define BNN_OUT_BITS 0
#define BNN_OUT_F4 1

/* Kernel-variant selector (the autotuner's search space; replaces the
 * reference's ParallelConfig X/Y/Z tags, model.py:38-67). */
typedef struct bnn_variant {
    int engine;     /* 0 = popc (integer pipe), 1 = tensor (tcgen05 kind::mxf4 on FP4 +-1) */
    int tile_n;     /* output channels per CTA (multiple of 32) */
    int tile_q;     /* popc: output pixel quads (2x2) per CTA, or batch rows for FC (-1 = GEMV);
                     * tensor conv: 0 = auto, 1 = per-tap TMA boxes, 2 = halo-reuse whenever it fits,
                     * 3 = per-tap TMA boxes (as 1; the engine pairs it with step_rows),
                     * 5 = per-tap TMA boxes on single CTAs, 6 = halo-along-x boxes (two TMA boxes per
                     * filter row for 16-px rows of 64 channels, else as 1; the engine pairs it with
                     * step_rows).  Tensor conv / FC with N = 256 tiles of a
                     * streamed filter bank otherwise run on CTA pairs (cta_group::2, M = 256). */
    int imgs;       /* images per CTA pass (popc conv) */
    /* tensor engine with a fused step: device (K, 32) FP4 step rows from bnn_step_rows -- the
     * threshold constant then enters the accumulator through one extra MMA per tile instead of an
     * add per channel in the epilogue (per-tap kernels; ignored by the halo kernels).  NULL = off. */
    const uint8_t *step_rows;
    int flags;      /* BNN_VARIANT_* bits */
    int reserved;
} bnn_variant;

/* bnn_variant.flags: the filters, thresholds, direction bits and step rows of this call are not
 * written by ANY kernel that may still be in flight on the stream when this call is launched (every
 * libbnn kernel triggers its dependents at entry, so with programmatic dependent launch several
 * earlier launches can still be running, not only the immediately preceding one) -- e.g. weights
 * uploaded and synchronised before the first launch, as the engine does.  The tensor kernels then
 * fetch them before waiting on the preceding grid; activations are always read after. */
#define BNN_VARIANT_STATIC_WEIGHTS 1

BNN_API int bnn_abi_version(void);
BNN_API const char *bnn_last_error(void);
/* number of kernel launches issued by this thread since the last reset */
BNN_API long long bnn_launch_count(int reset);
/* one-time per-device setup (kernel attributes); called lazily by every entry point */
BNN_API int bnn_init(int device);

/* ---- layout conversion (tensors.py:29-52, backends.py:188-207) ---- */
BNN_API int bnn_bits_ref_to_nhwc(const uint64_t *ref_words, int B, int C, int H, int W,
                         uint32_t *nhwc, void *stream);
BNN_API int bnn_bits_nhwc_to_ref(const uint32_t *nhwc, int B, int C, int H, int W,
                         uint64_t *ref_words, void *stream);

/* ---- step_forward (layers.py:135-146) on NCHW int32 ---- */
/* -> reference flat words (u64, nwords = ceil(B*C*S/64)) */
BNN_API int bnn_step_ref(const int32_t *x, int B, int C, long long S, const int32_t *thr,
                 const uint32_t *posbits, uint64_t *ref_words, void *stream);
/* -> NHWC bits */
BNN_API int bnn_step_nhwc(const int32_t *x, int B, int C, int H, int W, const int32_t *thr,
                  const uint32_t *posbits, uint32_t *nhwc, void *stream);

/* ---- maxpool_forward (layers.py:118-132) ---- */
BNN_API int bnn_maxpool_int(const int32_t *x, int B, int C, int H, int W, int32_t *out, void *stream);
BNN_API int bnn_maxpool_bits_nhwc(const uint32_t *x, int B, int C, int H, int W, uint32_t *out, void *stream);

/* ---- conv_int_forward (layers.py:91-101) [+ fused maxpool + step + pack] ----
 * x: (B,C,H,W) u8 (x_is_u8=1) or int32 pixels; w_pm: int8 +-1 (K, C, 3, 3).
 * pool: fuse the 2x2 int max-pool (requires even H, W).
 * out_nhwc: fused step output bits (needs thr/posbits) or NULL.
 * sums_nchw: int32 pre-activations (B,K,H,W) (pre-pool) or NULL. */
BNN_API int bnn_conv_first(const void *x, int x_is_u8, int B, int C, int H, int W, const int8_t *w_pm,
                   int K, const int32_t *thr, const uint32_t *posbits, int pool, int out_fmt,
                   void *out_nhwc, int32_t *sums_nchw, void *stream);

/* ---- conv_bin_forward (layers.py:104-115; packed route backends.py:210-256)
 *      [+ fused maxpool + step + pack] ----
 * x, mask: NHWC bits (mask NULL = fully valid); w: u32 (9, CW, K): word j of tap t=(dy*3+dx)
 * of filter k at w[(t*CW + j)*K + k] -- the reference's tap-major channel-packed w_cl
 * (model.py:125-132) in 32-bit words, transposed so a CTA's channel tile is contiguous. */
BNN_API int bnn_conv_bin(const uint32_t *x, const uint32_t *mask, int B, int C, int H, int W,
                 const uint32_t *w, int K, const int32_t *thr, const uint32_t *posbits, int pool, int out_fmt,
                 void *out_nhwc, int32_t *sums_nchw, const bnn_variant *v, void *stream);

/* ---- fc_forward for FC_BIN (layers.py:164-175; backends.py:288-324) [+ fused step + pack] ----
 * x, mask: (B, LW) u32 rows; w: (LW, M) u32, word j of row m at w[j*M + m] (same bit
 * order as x; the engine permutes columns to the device flatten order).  L = number of
 * real positions per row (the unmasked valid count); LW >= ceil(L/32) words per row
 * (0 = ceil(L/32)); bits beyond the real positions must be 0 in x and w.
 * out_bits: (B, ceil(M/32)) u32 or NULL; sums: (B, M) int32 or NULL. */
BNN_API int bnn_fc_bin(const uint32_t *x, const uint32_t *mask, int B, int L, int LW, const uint32_t *w, int M,
               const int32_t *thr, const uint32_t *posbits, int out_fmt, void *out_bits, int32_t *sums,
               const bnn_variant *v, void *stream);

/* ---- FC_INT_OUT + argmax (layers.py:164-175, :215-224): int32 logits (B, M) and
 *      first-max predictions (B,) int32 (either may be NULL); w: (M, LW) row-major;
 *      L, LW as for bnn_fc_bin ---- */
BNN_API int bnn_fc_out_argmax(const uint32_t *x, int B, int L, int LW, const uint32_t *w, int M,
                      int32_t *logits, int32_t *preds, void *stream);

/* ---- tensor engine (tcgen05.mma kind::mxf4 on FP4 +-1, TMA tap-shifted / halo boxes) ----
 * conv_bin_forward (layers.py:104-115) [+ fused maxpool + step]: x NHWC f4 (B,H,W,C), C % 64 == 0;
 * w FP4 +-1 (K, 9*C) with element (dy*3+dx)*C + c.  Out-of-image taps are TMA zero-fill.
 * Direction folding: when thr/posbits are given (fused step), the filter rows of POS channels must be
 * negated (E2M1 sign flip), so every step is "acc + c < 0" (one add); sums_nchw still reports the
 * reference pre-activations.  Without thresholds (sums only) the filters are used as they are. */
BNN_API int bnn_tc_conv(const uint8_t *x, int B, int C, int H, int W, const uint8_t *w, int K,
                        const int32_t *thr, const uint32_t *posbits, int pool, int out_fmt, void *out,
                        int32_t *sums_nchw, const bnn_variant *v, void *stream);
/* conv_int_forward (layers.py:91-101) [+ fused maxpool + step]: x u8 NCHW pixels (B,C,H,W) with
 * 9*C <= 64, w int8 +-1 (K, C*9) in (c, dy, dx) order, K <= 256.  One tcgen05 kind::i8 MMA
 * (A unsigned) per 128-pixel tile from an im2col row gathered in shared memory. */
BNN_API int bnn_tc_first(const uint8_t *x, int B, int C, int H, int W, const int8_t *w, int K,
                         const int32_t *thr, const uint32_t *posbits, int pool, int out_fmt, void *out,
                         int32_t *sums_nchw, void *stream);
/* The network's front end in ONE launch: conv_int_forward (layers.py:91-101) + step_forward
 * (:135-146) [+ maxpool_forward (:118-132) when pool1] followed by conv_bin_forward (:104-115) + step
 * [+ maxpool when pool2]; the first block's +-1 activation stays in shared memory (never in HBM).
 * x u8 NCHW (B,C,H,W) with C <= 4; w1 int8 +-1 (K1, 9*C) in (c, dy, dx) order (as bnn_tc_first);
 * w2 FP4 +-1 (K2, 9*K1) tap-major, direction-folded (as bnn_tc_conv with a fused step); K1 = K2 = 64.  out: BNN_OUT_BITS / BNN_OUT_F4
 * NHWC of the second block.  Debug taps (each may be NULL): sums1 int32 NCHW (B,K1,H,W) first-conv
 * pre-activations, mid FP4 NHWC first-block output, sums2 int32 NCHW second-conv pre-activations.
 * Replaces the first two reference layer calls of layer_forward (layers.py:178-212) for that pattern. */
BNN_API int bnn_tc_front(const uint8_t *x, int B, int C, int H, int W, const int8_t *w1, const int32_t *thr1,
                         const uint32_t *pos1, int pool1, const uint8_t *w2, const int32_t *thr2,
                         const uint32_t *pos2, int pool2, int K1, int K2, int out_fmt, void *out,
                         int32_t *sums1, uint8_t *mid, int32_t *sums2, void *stream);
/* Shared-memory bytes bnn_tc_front needs for this shape, or -1 if the shape is not supported. */
BNN_API int bnn_tc_front_smem(int C, int H, int W, int K1, int K2, int pool1, int pool2);
/* Debug only: device buffer of 8 x 512 x 4 u64 that the next bnn_tc_front launches fill with a
 * clock64 timeline of CTA 0 (loader / MMA / builder / epilogue events); NULL turns it off. */
BNN_API int bnn_tc_front_trace(unsigned long long *device_buf);
/* Debug only: the same for the next bnn_tc_conv / bnn_tc_fc launches (4 x 512 x 4 u64; NULL = off). */
BNN_API int bnn_tc_trace(unsigned long long *device_buf);
/* fc_forward (layers.py:164-175) [+ step]: x FP4 (B, L), w FP4 (M, L), L % 64 == 0 (direction-folded
 * rows when thresholds are given, as bnn_tc_conv).
 * out_fmt BNN_OUT_BITS / BNN_OUT_F4 with thresholds, or BNN_OUT_LOGITS (2, M <= 128): int32 logits (B, M) in
 * `out` and first-max argmax in `preds` (FC_INT_OUT + reference_infer's argmax, layers.py:215-224). */
#define BNN_OUT_LOGITS 2
BNN_API int bnn_tc_fc(const uint8_t *x, int B, int L, const uint8_t *w, int M, const int32_t *thr,
                      const uint32_t *posbits, int out_fmt, void *out, int32_t *sums, int32_t *preds,
                      const bnn_variant *v, void *stream);

/* Host-side preparation of bnn_variant.step_rows for a fused step (layers.py:135-146) over `kred`
 * accumulated +-1 products: row n (32 bytes = 64 FP4 values, element 2i in the low nibble of byte i)
 * sums, against the constant step A block (6.0 at K positions 0-23 / 32-55, 0.5 at 24-31 / 56-63),
 * to c_n = T_n + 0.5 (POS) or 0.5 - T_n (NEG) with T clamped to [-kred-1, kred+1] (the same
 * decisions) -- so with direction-folded filters the step fires iff acc + c < 0.  thr (K,) int32,
 * posbits ceil(K/32) words, out K*32 bytes, all HOST memory.  Returns 0, or 1 (nothing written) if
 * some c_n is not representable (kred > 1,600). */
BNN_API int bnn_step_rows(const int32_t *thr, const uint32_t *posbits, int K, int kred, uint8_t *out);

/* ---- format glue: NHWC bits <-> NHWC FP4 +-1 (pixels x C channels, C % 32 == 0; HBM-bound) ---- */
BNN_API int bnn_bits_to_f4(const uint32_t *bits, long long npix, int C, uint8_t *out, void *stream);
BNN_API int bnn_f4_to_bits(const uint8_t *x, long long npix, int C, uint32_t *out, void *stream);

/* ---- the whole network for a small batch as ONE launch (the batch-1 latency path) ----
 * reference_infer (layers.py:215-224) over the fused blocks the engine plans: conv_int_forward (:91-101)
 * [+ maxpool (:118-132)] + step (:135-146), conv_bin_forward (:104-115) [+ maxpool] + step, fc_forward
 * FC_BIN + step (:164-175), and FC_INT_OUT + first-max argmax.  One persistent cooperative launch (one
 * CTA per SM), the blocks separated by grid-wide barriers; each CTA's filter slices are bulk-copied into
 * shared memory at kernel entry and the arithmetic is xor + popcount on NHWC bit words (integer pipe).
 * Block descriptions (host array, copied into every launch):
 *   BNN_NET_CONV_FIRST: C, H, W = input image (C <= 3), K outputs, w = int8 +-1 (K, 9*C) in (c, dy, dx)
 *                       order (as bnn_conv_first); must be block 0.
 *   BNN_NET_CONV_BIN:   C, H, W = input (the previous block's output), w = u32 (9, CW, K) (as bnn_conv_bin).
 *   BNN_NET_FC_BIN:     C = L input bits, K = M outputs, w = u32 (LW, M) in the device flatten order (as
 *                       bnn_fc_bin).
 *   BNN_NET_FC_OUT:     C = L, K = classes, w = u32 (M, LW) (as bnn_fc_out_argmax); must be last.
 * thr / pos: the fused step of every block but the last.  pool: 2x2 max-pool before the step (conv).
 * Workspace: device memory of bnn_net_workspace() bytes (for batches up to B), 128-B aligned.
 * bnn_net_prepare() packs every block's filters and step constants into it (32-output-channel slices,
 * each one contiguous bulk copy) and zeroes the barrier counter: call it once, and again whenever the
 * filters change or a launch failed; every launch leaves the counter at zero.
 * bnn_net_infer(): x = u8 NCHW images (B, C, H, W), device memory, or pinned host memory with x_host = 1
 * (read once over PCIe; 16-B aligned).  logits (B, classes) int32 and preds (B,) int32 may be device or
 * mapped pinned host memory (zero-copy); either may be NULL.  grid: CTAs (0 = one per SM); the launch
 * fails if they cannot all be resident.  smem (may be NULL) receives the dynamic shared memory per CTA;
 * a batch whose activations do not fit is an argument error. */
#define BNN_NET_MAX_LAYERS 16
#define BNN_NET_CONV_FIRST 0
#define BNN_NET_CONV_BIN 1
#define BNN_NET_FC_BIN 2
#define BNN_NET_FC_OUT 3
typedef struct bnn_net_layer {
    int kind;       /* BNN_NET_* */
    int C, H, W, K;
    int pool;
    const void *w;
    const int32_t *thr;
    const uint32_t *pos;
} bnn_net_layer;
BNN_API int bnn_net_workspace(const bnn_net_layer *layers, int n, int B, int grid, size_t *bytes, size_t *smem);
BNN_API int bnn_net_prepare(const bnn_net_layer *layers, int n, int B, void *workspace, size_t ws_bytes,
                            void *stream);
BNN_API int bnn_net_infer(const bnn_net_layer *layers, int n, const uint8_t *x, int x_host, int B, int32_t *logits,
                          int32_t *preds, void *workspace, size_t ws_bytes, int grid, void *stream);
/* Persistent serving: the same kernel launched once as a resident server (it occupies every SM until
 * stopped).  The filters stay in shared memory; CTA 0 polls host_ctl[0] (request number) in pinned,
 * mapped host memory; each request reads the B images from host_x, writes host_logits / host_preds and
 * then sets host_ctl[BNN_NET_CTL_DONE] = the request number.  host_ctl = BNN_NET_CTL_WORDS u32 (128-B
 * aligned), zeroed by the caller before the launch: the host-written words (request, stop) and the
 * device-written words (done, status) sit on separate 128-B lines, so the device's polling of the first
 * and the host's spinning on the second do not contend for one line; status = 1 once the server stopped
 * itself after idle_s seconds without a request.  bnn_net_serve_request is HOST code: copy `bytes` of images into host_x, ring the doorbell,
 * spin on the completion word (timeout_s), copy the logits / predictions out; 0, -2 (server stopped),
 * -3 (timeout).  bnn_net_serve_stop asks the kernel to exit; synchronise its stream afterwards.
 * The workspace must come from bnn_net_workspace / bnn_net_prepare for (at least) batch B. */
#define BNN_NET_CTL_WORDS 64  /* control block: 64 u32 */
#define BNN_NET_CTL_REQ 0     /* host -> device: request number (the doorbell) */
#define BNN_NET_CTL_STOP 1    /* host -> device: 1 = exit */
#define BNN_NET_CTL_DONE 32   /* device -> host: number of the last completed request */
#define BNN_NET_CTL_STATUS 33 /* device -> host: 1 = stopped itself (idle timeout) */
BNN_API int bnn_net_serve_launch(const bnn_net_layer *layers, int n, int B, void *workspace, size_t ws_bytes,
                                 unsigned *host_ctl, const uint8_t *host_x, int32_t *host_logits, int32_t *host_preds,
                                 int grid, double idle_s, void *stream);
BNN_API int bnn_net_serve_request(unsigned *host_ctl, const void *images, size_t bytes, void *host_x,
                                  const int32_t *host_logits, int32_t *logits_out, size_t logits_bytes,
                                  const int32_t *host_preds, int32_t *preds_out, size_t preds_bytes, double timeout_s);
BNN_API int bnn_net_serve_stop(unsigned *host_ctl);
/* Debug only: device buffer of (grid x 64) u64 that the next bnn_net_infer launches fill with globaltimer
 * stamps per CTA (0: entry, 1: filter copies issued; block l: 2+3l barrier passed, 3+3l operands staged,
 * 4+3l items done); NULL turns it off. */
BNN_API int bnn_net_trace(unsigned long long *device_buf);

/* ---- xnor_popcount_dot (tensors.py:184-195): out[0] = 2*popc(~(a^b)&m) - popc(m),
 *      m = am & bm, over nwords u64 words ---- */
BNN_API int bnn_xnor_dot(const uint64_t *a, const uint64_t *am, const uint64_t *b, const uint64_t *bm,
                 int nwords, long long *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BNN_H */
