// abi.cu -- the extern "C" surface declared in include/bnn.h.
//
// Every entry point validates its arguments before launching anything
// (returning <0 with a thread-local message, never throwing across the ABI),
// then launches on the caller's stream.  Nothing here allocates, frees or
// synchronises, so every call is CUDA-Graph capturable.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>
#include <vector>

#include "common.cuh"

namespace bnn {

static thread_local char g_err[512] = "";
static thread_local long long g_launches = 0;

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void count_launch() { ++g_launches; }

bool pdl_on() {
    static const bool on = [] {
        const char *e = getenv("BNN_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int after_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
        return (int)e;
    }
    return 0;
}

int allow_smem(const void *func, size_t bytes, const char *name) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        set_error("%s: cudaGetDevice: %s", name, cudaGetErrorString(e));
        return (int)e;
    }
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({func, dev})) return 0;
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, func);
    if (e != cudaSuccess) {
        set_error("%s: cudaFuncGetAttributes: %s", name, cudaGetErrorString(e));
        return (int)e;
    }
    // the opt-in limit covers static + dynamic shared memory
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) {
        set_error("%s: cudaFuncSetAttribute(%zu B smem): %s", name, bytes, cudaGetErrorString(e));
        return (int)e;
    }
    done.insert({func, dev});
    return 0;
}

int ensure_init() { return 0; }

// kernels (conv_popc.cu, fc_popc.cu, layout.cu, conv_tc.cu)
int conv_bin_popc(const uint32_t *, const uint32_t *, int, int, int, int, const uint32_t *, int,
                  const int32_t *, const uint32_t *, int, int, void *, int32_t *, int, cudaStream_t);
int conv_first(const void *, int, int, int, int, int, const int8_t *, int, const int32_t *, const uint32_t *,
               int, int, void *, int32_t *, cudaStream_t);
int fc_bin_popc(const uint32_t *, const uint32_t *, int, int, int, const uint32_t *, int, const int32_t *,
                const uint32_t *, int, void *, int32_t *, int, cudaStream_t);
int tc_conv(const int8_t *, int, int, int, int, const int8_t *, int, const int32_t *, const uint32_t *, int, int,
            void *, int32_t *, int, int, const uint8_t *, int, cudaStream_t);
int tc_fc(const int8_t *, int, int, const int8_t *, int, const int32_t *, const uint32_t *, int, void *, int32_t *,
          int32_t *, int, int, const uint8_t *, int, cudaStream_t);
int tc_first(const uint8_t *, int, int, int, int, const int8_t *, int, const int32_t *, const uint32_t *, int,
             int, void *, int32_t *, cudaStream_t);
int tc_front(const uint8_t *, int, int, int, int, const int8_t *, const int32_t *, const uint32_t *, int,
             const int8_t *, const int32_t *, const uint32_t *, int, int, int, int, void *, int32_t *, int8_t *,
             int32_t *, cudaStream_t);
int tc_front_smem(int, int, int, int, int, int, int);
void tc_front_set_trace(unsigned long long *);
void tc_set_trace(unsigned long long *);
int bits_to_f4(const uint32_t *, long long, int, uint8_t *, cudaStream_t);
int f4_to_bits(const uint8_t *, long long, int, uint32_t *, cudaStream_t);
int fc_out_argmax(const uint32_t *, int, int, int, const uint32_t *, int, int32_t *, int32_t *, cudaStream_t);
int net_workspace(const bnn_net_layer *, int, int, int, size_t *, size_t *);
void net_set_trace(unsigned long long *);
int net_prepare(const bnn_net_layer *, int, int, void *, size_t, cudaStream_t);
int net_serve_launch(const bnn_net_layer *, int, int, void *, size_t, unsigned *, const uint8_t *, int32_t *, int32_t *,
                     int, double, cudaStream_t);
int net_serve_request(unsigned *, const void *, size_t, void *, const int32_t *, int32_t *, size_t, const int32_t *,
                      int32_t *, size_t, double);
int net_serve_stop(unsigned *);
int net_infer(const bnn_net_layer *, int, const uint8_t *, int, int, int32_t *, int32_t *, void *, size_t, int,
              cudaStream_t);
int ref_to_nhwc(const uint64_t *, int, int, int, int, uint32_t *, cudaStream_t);
int nhwc_to_ref(const uint32_t *, int, int, int, int, uint64_t *, cudaStream_t);
int step_ref(const int32_t *, int, int, long long, const int32_t *, const uint32_t *, uint64_t *, cudaStream_t);
int step_nhwc(const int32_t *, int, int, int, int, const int32_t *, const uint32_t *, uint32_t *, cudaStream_t);
int maxpool_int(const int32_t *, int, int, int, int, int32_t *, cudaStream_t);
int maxpool_bits_nhwc(const uint32_t *, int, int, int, int, uint32_t *, cudaStream_t);
int xnor_dot(const uint64_t *, const uint64_t *, const uint64_t *, const uint64_t *, int, long long *,
             cudaStream_t);

}  // namespace bnn

using namespace bnn;

#define BNN_DIMS_OK(B, C, H, W) \
    BNN_REQUIRE((B) >= 0 && (C) >= 1 && (H) >= 1 && (W) >= 1, "bad dims B=%d C=%d H=%d W=%d", B, C, H, W)

extern "C" {

int bnn_abi_version(void) { return BNN_ABI_VERSION; }

const char *bnn_last_error(void) { return g_err; }

long long bnn_launch_count(int reset) {
    const long long n = g_launches;
    if (reset) g_launches = 0;
    return n;
}

int bnn_init(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        set_error("cudaGetDeviceCount: %s", cudaGetErrorString(e));
        return (int)e;
    }
    BNN_REQUIRE(device >= 0 && device < n, "device %d out of range (%d devices)", device, n);
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) {
        set_error("cudaGetDeviceProperties: %s", cudaGetErrorString(e));
        return (int)e;
    }
    BNN_REQUIRE(prop.major == 10 && prop.minor == 0,
                "libbnn is built for sm_100a (B200); device %d is sm_%d%d", device, prop.major, prop.minor);
    return 0;
}

int bnn_bits_ref_to_nhwc(const uint64_t *ref, int B, int C, int H, int W, uint32_t *nhwc, void *stream) {
    BNN_DIMS_OK(B, C, H, W);
    BNN_REQUIRE(ref && nhwc, "null pointer");
    if (B == 0) return 0;
    return ref_to_nhwc(ref, B, C, H, W, nhwc, as_stream(stream));
}

int bnn_bits_nhwc_to_ref(const uint32_t *nhwc, int B, int C, int H, int W, uint64_t *ref, void *stream) {
    BNN_DIMS_OK(B, C, H, W);
    BNN_REQUIRE(ref && nhwc, "null pointer");
    if (B == 0) return 0;
    return nhwc_to_ref(nhwc, B, C, H, W, ref, as_stream(stream));
}

int bnn_step_ref(const int32_t *x, int B, int C, long long S, const int32_t *thr, const uint32_t *posbits,
                 uint64_t *ref, void *stream) {
    BNN_REQUIRE(B >= 0 && C >= 1 && S >= 1, "bad dims B=%d C=%d S=%lld", B, C, S);
    BNN_REQUIRE(x && thr && posbits && ref, "null pointer");
    if (B == 0) return 0;
    return step_ref(x, B, C, S, thr, posbits, ref, as_stream(stream));
}

int bnn_step_nhwc(const int32_t *x, int B, int C, int H, int W, const int32_t *thr, const uint32_t *posbits,
                  uint32_t *nhwc, void *stream) {
    BNN_DIMS_OK(B, C, H, W);
    BNN_REQUIRE(x && thr && posbits && nhwc, "null pointer");
    if (B == 0) return 0;
    return step_nhwc(x, B, C, H, W, thr, posbits, nhwc, as_stream(stream));
}

int bnn_maxpool_int(const int32_t *x, int B, int C, int H, int W, int32_t *out, void *stream) {
    BNN_DIMS_OK(B, C, H, W);
    BNN_REQUIRE(H % 2 == 0 && W % 2 == 0, "maxpool needs even spatial dims, got %dx%d", H, W);
    BNN_REQUIRE(x && out, "null pointer");
    if (B == 0) return 0;
    return maxpool_int(x, B, C, H, W, out, as_stream(stream));
}

int bnn_maxpool_bits_nhwc(const uint32_t *x, int B, int C, int H, int W, uint32_t *out, void *stream) {
    BNN_DIMS_OK(B, C, H, W);
    BNN_REQUIRE(H % 2 == 0 && W % 2 == 0, "maxpool needs even spatial dims, got %dx%d", H, W);
    BNN_REQUIRE(x && out, "null pointer");
    if (B == 0) return 0;
    return maxpool_bits_nhwc(x, B, C, H, W, out, as_stream(stream));
}

#define BNN_FMT_OK(fmt, K)                                                                              \
    BNN_REQUIRE((fmt) == BNN_OUT_BITS || ((fmt) == BNN_OUT_F4 && (K) % 32 == 0), "bad out_fmt %d for K=%d", \
                fmt, K)

int bnn_conv_first(const void *x, int x_is_u8, int B, int C, int H, int W, const int8_t *w_pm, int K,
                   const int32_t *thr, const uint32_t *posbits, int pool, int out_fmt, void *out_nhwc,
                   int32_t *sums, void *stream) {
    BNN_FMT_OK(out_fmt, K);
    BNN_DIMS_OK(B, C, H, W);
    BNN_REQUIRE(K >= 1, "bad K=%d", K);
    BNN_REQUIRE(x && w_pm, "null pointer");
    BNN_REQUIRE(out_nhwc || sums, "conv_int: no output requested");
    BNN_REQUIRE(!out_nhwc || (thr && posbits), "conv_int: fused step needs thresholds and directions");
    BNN_REQUIRE(!pool || (H % 2 == 0 && W % 2 == 0), "maxpool needs even spatial dims, got %dx%d", H, W);
    if (B == 0) return 0;
    return conv_first(x, x_is_u8, B, C, H, W, w_pm, K, thr, posbits, pool, out_fmt, out_nhwc, sums,
                      as_stream(stream));
}

int bnn_conv_bin(const uint32_t *x, const uint32_t *mask, int B, int C, int H, int W, const uint32_t *w, int K,
                 const int32_t *thr, const uint32_t *posbits, int pool, int out_fmt, void *out_nhwc, int32_t *sums,
                 const bnn_variant *v, void *stream) {
    BNN_FMT_OK(out_fmt, K);
    BNN_DIMS_OK(B, C, H, W);
    BNN_REQUIRE(K >= 1, "bad K=%d", K);
    BNN_REQUIRE(x && w, "null pointer");
    BNN_REQUIRE(out_nhwc || sums, "conv_bin: no output requested");
    BNN_REQUIRE(!out_nhwc || (thr && posbits), "conv_bin: fused step needs thresholds and directions");
    BNN_REQUIRE(!pool || (H % 2 == 0 && W % 2 == 0), "maxpool needs even spatial dims, got %dx%d", H, W);
    BNN_REQUIRE(!v || v->engine == 0, "conv_bin: engine %d not available", v ? v->engine : -1);
    if (B == 0) return 0;
    return conv_bin_popc(x, mask, B, C, H, W, w, K, thr, posbits, pool, out_fmt, out_nhwc, sums,
                         v ? v->tile_n : 0, as_stream(stream));
}

int bnn_fc_bin(const uint32_t *x, const uint32_t *mask, int B, int L, int LW, const uint32_t *w, int M,
               const int32_t *thr, const uint32_t *posbits, int out_fmt, void *out_bits, int32_t *sums,
               const bnn_variant *v, void *stream) {
    BNN_FMT_OK(out_fmt, M);
    BNN_REQUIRE(B >= 0 && L >= 1 && M >= 1, "bad dims B=%d L=%d M=%d", B, L, M);
    BNN_REQUIRE(x && w, "null pointer");
    BNN_REQUIRE(out_bits || sums, "fc: no output requested");
    BNN_REQUIRE(!out_bits || (thr && posbits), "fc: fused step needs thresholds and directions");
    BNN_REQUIRE(!v || v->engine == 0, "fc: engine %d not available", v ? v->engine : -1);
    if (B == 0) return 0;
    int tile = v ? v->tile_n : 0;
    if (v && v->tile_q < 0) tile = 0;  // explicit GEMV request
    if (LW <= 0) LW = (L + 31) / 32;
    BNN_REQUIRE(LW >= (L + 31) / 32, "fc: LW=%d words cannot hold L=%d bits", LW, L);
    return fc_bin_popc(x, mask, B, L, LW, w, M, thr, posbits, out_fmt, out_bits, sums, tile, as_stream(stream));
}

int bnn_fc_out_argmax(const uint32_t *x, int B, int L, int LW, const uint32_t *w, int M, int32_t *logits,
                      int32_t *preds, void *stream) {
    BNN_REQUIRE(B >= 0 && L >= 1 && M >= 1, "bad dims B=%d L=%d M=%d", B, L, M);
    BNN_REQUIRE(x && w && (logits || preds), "null pointer");
    if (B == 0) return 0;
    if (LW <= 0) LW = (L + 31) / 32;
    BNN_REQUIRE(LW >= (L + 31) / 32, "fc_out: LW=%d words cannot hold L=%d bits", LW, L);
    return fc_out_argmax(x, B, L, LW, w, M, logits, preds, as_stream(stream));
}

int bnn_tc_conv(const uint8_t *x, int B, int C, int H, int W, const uint8_t *w, int K, const int32_t *thr,
                const uint32_t *posbits, int pool, int out_fmt, void *out, int32_t *sums, const bnn_variant *v,
                void *stream) {
    BNN_DIMS_OK(B, C, H, W);
    BNN_REQUIRE(K >= 1, "bad K=%d", K);
    BNN_REQUIRE(x && w, "null pointer");
    BNN_REQUIRE(out || sums, "tc_conv: no output requested");
    BNN_REQUIRE(!out || (thr && posbits), "tc_conv: fused step needs thresholds and directions");
    BNN_FMT_OK(out_fmt, K);
    BNN_REQUIRE(!pool || (H % 2 == 0 && W % 2 == 0), "maxpool needs even spatial dims, got %dx%d", H, W);
    BNN_REQUIRE(C % 64 == 0, "tensor engine needs C %% 64 == 0 (got %d)", C);
    BNN_REQUIRE(W <= 128, "tensor engine needs W <= 128 (got %d)", W);
    if (B == 0) return 0;
    // variant.tile_q: 0 = auto (halo-reuse kernel when the filter bank fits smem), 1 = per-tap TMA boxes
    return tc_conv(reinterpret_cast<const int8_t *>(x), B, C, H, W, reinterpret_cast<const int8_t *>(w), K, thr,
                   posbits, pool, out_fmt, out, sums, v ? v->tile_n : 0,
                   v ? v->tile_q : 0, v ? v->step_rows : nullptr, v ? v->flags : 0, as_stream(stream));
}

int bnn_tc_first(const uint8_t *x, int B, int C, int H, int W, const int8_t *w, int K, const int32_t *thr,
                 const uint32_t *posbits, int pool, int out_fmt, void *out, int32_t *sums, void *stream) {
    BNN_DIMS_OK(B, C, H, W);
    BNN_REQUIRE(K >= 1, "bad K=%d", K);
    BNN_REQUIRE(x && w, "null pointer");
    BNN_REQUIRE(out || sums, "tc_first: no output requested");
    BNN_REQUIRE(!out || (thr && posbits), "tc_first: fused step needs thresholds and directions");
    BNN_FMT_OK(out_fmt, K);
    BNN_REQUIRE(!pool || (H % 2 == 0 && W % 2 == 0), "maxpool needs even spatial dims, got %dx%d", H, W);
    if (B == 0) return 0;
    return tc_first(x, B, C, H, W, w, K, thr, posbits, pool, out_fmt, out, sums, as_stream(stream));
}

int bnn_tc_front(const uint8_t *x, int B, int C, int H, int W, const int8_t *w1, const int32_t *thr1,
                 const uint32_t *pos1, int pool1, const uint8_t *w2, const int32_t *thr2, const uint32_t *pos2,
                 int pool2, int K1, int K2, int out_fmt, void *out, int32_t *sums1, uint8_t *mid, int32_t *sums2,
                 void *stream) {
    BNN_DIMS_OK(B, C, H, W);
    BNN_REQUIRE(x && w1 && w2 && thr1 && pos1 && thr2 && pos2, "tc_front: null pointer");
    BNN_REQUIRE(out || sums1 || mid || sums2, "tc_front: no output requested");
    BNN_FMT_OK(out_fmt, K2);
    BNN_REQUIRE(tc_front_smem(C, H, W, K1, K2, pool1, pool2) > 0,
                "tc_front: unsupported shape C=%d H=%d W=%d K1=%d K2=%d pool1=%d pool2=%d", C, H, W, K1, K2, pool1,
                pool2);
    if (B == 0) return 0;
    return tc_front(x, B, C, H, W, w1, thr1, pos1, pool1, reinterpret_cast<const int8_t *>(w2), thr2, pos2, pool2, K1,
                    K2, out_fmt, out, sums1, reinterpret_cast<int8_t *>(mid), sums2, as_stream(stream));
}

int bnn_tc_front_smem(int C, int H, int W, int K1, int K2, int pool1, int pool2) {
    return tc_front_smem(C, H, W, K1, K2, pool1, pool2);
}

int bnn_tc_front_trace(unsigned long long *buf) {
    tc_front_set_trace(buf);
    return 0;
}

int bnn_tc_trace(unsigned long long *buf) {
    tc_set_trace(buf);
    return 0;
}

int bnn_tc_fc(const uint8_t *x, int B, int L, const uint8_t *w, int M, const int32_t *thr, const uint32_t *posbits,
              int out_fmt, void *out, int32_t *sums, int32_t *preds, const bnn_variant *v, void *stream) {
    BNN_REQUIRE(B >= 0 && L >= 1 && M >= 1, "bad dims B=%d L=%d M=%d", B, L, M);
    BNN_REQUIRE(x && w, "null pointer");
    BNN_REQUIRE(L % 64 == 0, "tensor engine needs L %% 64 == 0 (got %d)", L);
    if (out_fmt == BNN_OUT_LOGITS) {
        BNN_REQUIRE(M <= 128, "tc logits tile needs M <= 128 (got %d)", M);
        BNN_REQUIRE(out || preds || sums, "tc_fc: no output requested");
    } else {
        BNN_FMT_OK(out_fmt, M);
        BNN_REQUIRE(out || sums, "tc_fc: no output requested");
        BNN_REQUIRE(!out || (thr && posbits), "tc_fc: fused step needs thresholds and directions");
    }
    if (B == 0) return 0;
    int bn = v ? v->tile_n : 0;
    if (out_fmt == BNN_OUT_LOGITS && (bn < M || bn == 0 || bn > 128)) bn = M <= 32 ? 32 : M <= 64 ? 64 : 128;
    return tc_fc(reinterpret_cast<const int8_t *>(x), B, L, reinterpret_cast<const int8_t *>(w), M, thr, posbits,
                 out_fmt, out, sums, preds, bn, v ? v->tile_q : 0, v ? v->step_rows : nullptr, v ? v->flags : 0,
                 as_stream(stream));
}

// Greedy E2M1 fill: magnitudes in halves {0, 1, 2, 3, 4, 6, 8, 12} (codes 0..7) into the given K
// positions of one step row until they sum to `halves`; any remainder below 12 takes <= 2 slots.
static bool fill_e2m1(uint8_t *row, bool coarse, int halves, bool neg) {
    static const int kHalves[8] = {0, 1, 2, 3, 4, 6, 8, 12};
    for (int k = 0; k < 64 && halves > 0; ++k) {
        if (((k & 31) < 24) != coarse) continue;
        int code = 7;
        while (kHalves[code] > halves) --code;
        halves -= kHalves[code];
        row[k >> 1] |= (uint8_t)((code | (neg ? 8 : 0)) << ((k & 1) * 4));
    }
    return halves == 0;
}

int bnn_step_rows(const int32_t *thr, const uint32_t *posbits, int K, int kred, uint8_t *out) {
    BNN_REQUIRE(K >= 1 && kred >= 1, "step_rows: bad K=%d kred=%d", K, kred);
    BNN_REQUIRE(thr && posbits && out, "null pointer");
    std::vector<uint8_t> rows((size_t)K * 32, 0);
    for (int n = 0; n < K; ++n) {
        // T outside [-kred, kred] decides every sum the same way as the clamped value
        const long long t = std::max<long long>(-kred - 1, std::min<long long>(kred + 1, thr[n]));
        const bool pos = (posbits[n >> 5] >> (n & 31)) & 1u;
        const long long c4 = pos ? 4 * t + 2 : 2 - 4 * t;  // 4c, c = T + 0.5 / 0.5 - T
        const long long m4 = c4 < 0 ? -c4 : c4;
        // 4c = 12 * (coarse halves: 6.0 x values) + (fine halves: 0.5 x values)
        uint8_t *row = rows.data() + (size_t)n * 32;
        if (!fill_e2m1(row, true, (int)(m4 / 12), c4 < 0) || !fill_e2m1(row, false, (int)(m4 % 12), c4 < 0)) return 1;
    }
    std::memcpy(out, rows.data(), rows.size());
    return 0;
}

int bnn_bits_to_f4(const uint32_t *bits, long long npix, int C, uint8_t *out, void *stream) {
    BNN_REQUIRE(npix >= 0 && C >= 1 && C % 32 == 0, "bits_to_f4: bad dims npix=%lld C=%d", npix, C);
    BNN_REQUIRE(bits && out, "null pointer");
    if (npix == 0) return 0;
    return bits_to_f4(bits, npix, C, out, as_stream(stream));
}

int bnn_f4_to_bits(const uint8_t *x, long long npix, int C, uint32_t *out, void *stream) {
    BNN_REQUIRE(npix >= 0 && C >= 1 && C % 32 == 0, "f4_to_bits: bad dims npix=%lld C=%d", npix, C);
    BNN_REQUIRE(x && out, "null pointer");
    if (npix == 0) return 0;
    return f4_to_bits(x, npix, C, out, as_stream(stream));
}

int bnn_xnor_dot(const uint64_t *a, const uint64_t *am, const uint64_t *b, const uint64_t *bm, int nwords,
                 long long *out, void *stream) {
    BNN_REQUIRE(nwords >= 0, "bad nwords");
    BNN_REQUIRE(a && am && b && bm && out, "null pointer");
    return xnor_dot(a, am, b, bm, nwords, out, as_stream(stream));
}

int bnn_net_workspace(const bnn_net_layer *layers, int n, int B, int grid, size_t *bytes, size_t *smem) {
    return net_workspace(layers, n, B, grid, bytes, smem);
}

int bnn_net_infer(const bnn_net_layer *layers, int n, const uint8_t *x, int x_host, int B, int32_t *logits,
                  int32_t *preds, void *workspace, size_t ws_bytes, int grid, void *stream) {
    return net_infer(layers, n, x, x_host, B, logits, preds, workspace, ws_bytes, grid, as_stream(stream));
}

int bnn_net_prepare(const bnn_net_layer *layers, int n, int B, void *workspace, size_t ws_bytes, void *stream) {
    return net_prepare(layers, n, B, workspace, ws_bytes, as_stream(stream));
}

int bnn_net_serve_launch(const bnn_net_layer *layers, int n, int B, void *workspace, size_t ws_bytes, unsigned *host_ctl,
                         const uint8_t *host_x, int32_t *host_logits, int32_t *host_preds, int grid, double idle_s,
                         void *stream) {
    return net_serve_launch(layers, n, B, workspace, ws_bytes, host_ctl, host_x, host_logits, host_preds, grid, idle_s,
                            as_stream(stream));
}

int bnn_net_serve_request(unsigned *host_ctl, const void *images, size_t bytes, void *host_x, const int32_t *host_logits,
                          int32_t *logits_out, size_t logits_bytes, const int32_t *host_preds, int32_t *preds_out,
                          size_t preds_bytes, double timeout_s) {
    return net_serve_request(host_ctl, images, bytes, host_x, host_logits, logits_out, logits_bytes, host_preds,
                             preds_out, preds_bytes, timeout_s);
}

int bnn_net_serve_stop(unsigned *host_ctl) { return net_serve_stop(host_ctl); }

int bnn_net_trace(unsigned long long *device_buf) {
    net_set_trace(device_buf);
    return 0;
}

}  // extern "C"
