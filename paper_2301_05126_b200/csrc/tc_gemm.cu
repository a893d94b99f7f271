// tc_gemm.cu -- BNN conv / FC blocks on the 5th-gen tensor cores (tcgen05.mma kind::i8).
//
// The +-1 data are stored int8 (+1 / -1, 0 = padding) in NHWC so a binary
// dot product is an exact int8 x int8 -> int32 MMA.  Implicit GEMM:
//   rows M    = 128 output pixels of a spatial box (BW x BH x BB) or 128 batch rows (FC)
//   cols N    = BN output channels (64/128/256; 32 for logits)
//   reduction = 9 taps x C channels (conv) or L features (FC), K-major, tap-major
// For tap (dy,dx) the A tile is ONE 4-D TMA box load of the NHWC activation at
// coordinates (c0, x0+dx-1, y0+dy-1, b0): out-of-image taps fall outside the
// tensor and TMA zero-fills them, which is exactly the reference's "invalid
// taps contribute nothing" (layers.py:70-80) -- no masks, no correction table.
//
// Warp roles (192 threads): w0 = TMA producer, w1 = TMEM owner + MMA issuer
// (one elected lane), w2..w5 = epilogue (TMEM lane quarter = warp % 4).
// S-stage smem ring with full/empty mbarriers; tcgen05.commit releases stages.
// Epilogue: tcgen05.ld 32x32b.x32 -> strict threshold per channel (layers.py:
// 135-146) -> optional 2x2 pool as OR(POS)/AND(NEG) of thresholded bits via a
// shared-memory exchange -> NHWC bits or int8 +-1 (next tensor layer), or
// int32 logits + first-max argmax (FC_INT_OUT).  Optional int32 NCHW sums.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace bnn {

struct TcArgs {
    int T, CCH, nks;      // taps, channel chunks per tap, k-steps
    int BW, BH, BB;       // box (pixels per tile = BW*BH*BB <= 128)
    int W, H, B;          // logical activation dims (FC: W = H = 1, B = batch)
    int K;                // output channels / neurons
    int ntx, nty;         // tiles along x, y (tiles along b = gridDim.x / (ntx*nty))
    const int32_t *thr;
    const uint32_t *pos;
    int pool, out_fmt;    // out_fmt: 0 = NHWC bits (u32), 1 = NHWC int8 +-1, 2 = logits + argmax
    void *out;
    int32_t *sums;        // NCHW int32 pre-activations (pre-pool) or null
    int32_t *preds;       // out_fmt 2
    uint32_t idesc;       // instruction descriptor
    int a_bytes;          // TMA bytes of one A box
};

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

// Bounded wait: a pipeline bug becomes a trap (cudaErrorLaunchFailure) after ~seconds, never a hung GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t spins = 0;; ++spins) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if (spins > (1u << 26)) __trap();
    }
}

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(smem_addr(dst)),
        "l"(map), "r"(smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_addr(dst)),
        "l"(map), "r"(smem_addr(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}

// K-major operand, rows of `row_bytes` (64 or 128) swizzled, 8-row groups dense.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, int row_bytes) {
    const uint64_t layout = row_bytes == 128 ? 2ull : 4ull;  // SWIZZLE_128B : SWIZZLE_64B
    uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;                              // LBO (unused for swizzled K-major)
    d |= (uint64_t)((8 * row_bytes) >> 4) << 32;         // SBO: one 8-row swizzle atom
    d |= (uint64_t)1 << 46;                              // descriptor version (sm100)
    d |= layout << 61;
    return d;
}

#define TMEM_LD32(taddr, v)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                              \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),         \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),   \
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), \
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])  \
        : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 channel bits -> 32 int8 bytes (+1 for bit 1, -1 for bit 0)
__device__ __forceinline__ void bits_to_pm8(uint32_t bits, uint4 &lo, uint4 &hi) {
    uint32_t w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t spread = (((bits >> (4 * k)) & 0xFu) * 0x00204081u) & 0x01010101u;
        w[k] = ~(spread * 0xFEu);
    }
    lo = make_uint4(w[0], w[1], w[2], w[3]);
    hi = make_uint4(w[4], w[5], w[6], w[7]);
}

// ------------------------------------------------------------------ the kernel
constexpr int kTcThreads = 192;

template <int BN, int KC, int S>
struct TcSmem {
    static constexpr int A_BYTES = 128 * KC;
    static constexpr int B_BYTES = BN * KC;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int BARS = 2 * S + 1;
    static constexpr int BITS_WORDS = 128 * (BN / 32);
    static constexpr int TOTAL = 1024 /*align slack*/ + S * STAGE + BARS * 8 + 16 + BN * 4 + BN / 8 + BITS_WORDS * 4;
};

template <int BN, int KC, int S>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_block_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const TcArgs a) {
    using L = TcSmem<BN, KC, S>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;
    uint8_t *sB = smem + S * L::A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * L::STAGE);
    uint64_t *empty = full + S;
    uint64_t *accum = empty + S;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accum + 1);
    int32_t *s_thr = reinterpret_cast<int32_t *>(tmem_slot + 4);
    uint32_t *s_pos = reinterpret_cast<uint32_t *>(s_thr + BN);
    uint32_t *s_bits = s_pos + BN / 32;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_xy = a.ntx * a.nty;
    const int tb = blockIdx.x / tiles_xy, rem = blockIdx.x % tiles_xy;
    const int x0 = (rem % a.ntx) * a.BW, y0 = (rem / a.ntx) * a.BH, b0 = tb * a.BB;
    const int n0 = blockIdx.y * BN;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accum, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {  // whole warp: allocate BN TMEM columns (power of two >= 32)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                     "r"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp >= 2) {  // epilogue warps stage thresholds / directions for this channel tile
        for (int i = threadIdx.x - 64; i < BN; i += 128) {
            const int k = n0 + i;
            s_thr[i] = (a.thr && k < a.K) ? __ldg(a.thr + k) : 0;
        }
        for (int i = threadIdx.x - 64; i < BN / 32; i += 128) {
            const int k = n0 + i * 32;
            s_pos[i] = (a.pos && k < a.K) ? __ldg(a.pos + (k >> 5)) : 0u;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            for (int ks = 0; ks < a.nks; ++ks) {
                const int s = ks % S, round = ks / S;
                mbar_wait(&empty[s], (round & 1) ^ 1);
                mbar_expect_tx(&full[s], a.a_bytes + L::B_BYTES);
                const int tap = ks / a.CCH, cc = ks % a.CCH;
                const int dx = a.T == 9 ? tap % 3 - 1 : 0, dy = a.T == 9 ? tap / 3 - 1 : 0;
                tma_load_4d(sA + s * L::A_BYTES, &tmA, &full[s], cc * KC, x0 + dx, y0 + dy, b0);
                tma_load_2d(sB + s * L::B_BYTES, &tmB, &full[s], ks * KC, n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            for (int ks = 0; ks < a.nks; ++ks) {
                const int s = ks % S, round = ks / S;
                mbar_wait(&full[s], round & 1);
                tc_fence_after();
                const uint32_t a_base = smem_addr(sA + s * L::A_BYTES);
                const uint32_t b_base = smem_addr(sB + s * L::B_BYTES);
#pragma unroll
                for (int k = 0; k < KC / 32; ++k)
                    umma_i8(tmem_base, umma_desc(a_base + 32 * k, KC), umma_desc(b_base + 32 * k, KC), a.idesc,
                            (ks | k) != 0);
                umma_commit(&empty[s]);
            }
            umma_commit(accum);
        }
        __syncwarp();
    } else {  // ------------------------- epilogue (warps 2..5)
        mbar_wait(accum, 0);
        tc_fence_after();
        const int q = warp & 3;
        const int m = q * 32 + lane;  // tile row == TMEM lane
        const int npix = a.BW * a.BH * a.BB;
        const int bx = m % a.BW, by = (m / a.BW) % a.BH, bb = m / (a.BW * a.BH);
        const int gx = x0 + bx, gy = y0 + by, gb = b0 + bb;
        const bool inb = m < npix && gx < a.W && gy < a.H && gb < a.B;
        const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16);
        const int Ho = a.pool ? a.H / 2 : a.H, Wo = a.pool ? a.W / 2 : a.W;
        const int KW = (a.K + 31) / 32;
        int best = 0, bestv = 0;
#pragma unroll 1
        for (int j = 0; j < BN / 32; ++j) {
            uint32_t v[32];
            TMEM_LD32(trow + j * 32, v);
            tmem_wait_ld();
            const int nb = n0 + j * 32;
            if (a.sums && inb) {
                for (int i = 0; i < 32 && nb + i < a.K; ++i)
                    a.sums[(((long long)gb * a.K + nb + i) * a.H + gy) * a.W + gx] = (int32_t)v[i];
            }
            if (a.out_fmt == 2) {
                if (inb) {
                    int32_t *lg = static_cast<int32_t *>(a.out);
                    for (int i = 0; i < 32 && nb + i < a.K; ++i) {
                        const int val = (int32_t)v[i];
                        if (lg) lg[(long long)gb * a.K + nb + i] = val;
                        if (nb + i == 0 || val > bestv) {  // first max wins ties (np.argmax)
                            best = nb + i;
                            bestv = val;
                        }
                    }
                }
                continue;
            }
            uint32_t bits = 0;
            const uint32_t pw = s_pos[j];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int t = s_thr[j * 32 + i];
                const int val = (int32_t)v[i];
                const bool pos = (pw >> i) & 1u;
                bits |= (uint32_t)(pos ? val > t : val < t) << i;
            }
            if (nb + 32 > a.K) bits &= (nb >= a.K) ? 0u : (0xffffffffu >> (32 - (a.K - nb)));
            if (a.pool) {
                s_bits[m * (BN / 32) + j] = bits;
            } else if (a.out && inb && nb < a.K) {
                const long long pix = ((long long)gb * a.H + gy) * a.W + gx;
                if (a.out_fmt == 0) {
                    static_cast<uint32_t *>(a.out)[pix * KW + (nb >> 5)] = bits;
                } else {
                    uint4 lo, hi;
                    bits_to_pm8(bits, lo, hi);
                    uint4 *dst = reinterpret_cast<uint4 *>(static_cast<int8_t *>(a.out) + pix * a.K + nb);
                    dst[0] = lo;
                    dst[1] = hi;
                }
            }
        }
        if (a.out_fmt == 2) {
            if (inb && a.preds) a.preds[gb] = best;
        } else if (a.pool && a.out) {
            asm volatile("bar.sync 1, 128;" ::: "memory");  // epilogue warps only
            if (inb && !(bx & 1) && !(by & 1)) {
                const long long opix = ((long long)gb * Ho + gy / 2) * Wo + gx / 2;
#pragma unroll 1
                for (int j = 0; j < BN / 32; ++j) {
                    const int nb = n0 + j * 32;
                    if (nb >= a.K) break;
                    const int st = BN / 32;
                    const uint32_t p0 = s_bits[m * st + j], p1 = s_bits[(m + 1) * st + j];
                    const uint32_t p2 = s_bits[(m + a.BW) * st + j], p3 = s_bits[(m + a.BW + 1) * st + j];
                    const uint32_t pw = s_pos[j];
                    const uint32_t bits = ((p0 | p1 | p2 | p3) & pw) | ((p0 & p1 & p2 & p3) & ~pw);
                    if (a.out_fmt == 0) {
                        static_cast<uint32_t *>(a.out)[opix * KW + (nb >> 5)] = bits;
                    } else {
                        uint4 lo, hi;
                        bits_to_pm8(bits, lo, hi);
                        uint4 *dst = reinterpret_cast<uint4 *>(static_cast<int8_t *>(a.out) + opix * a.K + nb);
                        dst[0] = lo;
                        dst[1] = hi;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(BN));
    }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encoder() {
    static std::once_flag once;
    static int status = 0;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) {
            status = e != cudaSuccess ? (int)e : (int)cudaErrorNotSupported;
        } else {
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        }
    });
    if (status) set_error("cuTensorMapEncodeTiled unavailable");
    return status;
}

static int encode_map(CUtensorMap *map, const void *base, int rank, const cuuint64_t *dims, const cuuint64_t *strides,
                      const cuuint32_t *box, int row_bytes) {
    int e = get_encoder();
    if (e) return e;
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUtensorMapSwizzle sw = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, rank, const_cast<void *>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d): rank %d dims %llu,%llu,%llu,%llu box %u,%u,%u,%u", (int)r, rank,
                  (unsigned long long)dims[0], (unsigned long long)(rank > 1 ? dims[1] : 0),
                  (unsigned long long)(rank > 2 ? dims[2] : 0), (unsigned long long)(rank > 3 ? dims[3] : 0), box[0],
                  rank > 1 ? box[1] : 0, rank > 2 ? box[2] : 0, rank > 3 ? box[3] : 0);
        return -2;
    }
    return 0;
}

static uint32_t make_idesc(int M, int N, bool a_signed) {
    uint32_t d = 0;
    d |= 2u << 4;                       // D format: S32
    d |= (a_signed ? 1u : 0u) << 7;     // A: signed / unsigned 8-bit
    d |= 1u << 10;                      // B: signed 8-bit
    d |= (uint32_t)(N >> 3) << 17;      // N
    d |= (uint32_t)(M >> 4) << 24;      // M
    return d;                           // K-major A and B, no negate, dense
}

template <int BN, int KC>
static int launch_tc(const CUtensorMap &ma, const CUtensorMap &mb, TcArgs &a, int tiles, cudaStream_t st) {
    constexpr int S = (KC * (128 + BN) <= 24 * 1024) ? 8 : (KC * (128 + BN) <= 32 * 1024 ? 6 : 4);
    using L = TcSmem<BN, KC, S>;
    auto kern = tc_block_kernel<BN, KC, S>;
    int e = allow_smem(reinterpret_cast<const void *>(kern), L::TOTAL, "tc_block");
    if (e) return e;
    dim3 grid((unsigned)tiles, (unsigned)ceil_div(a.K, BN));
    kern<<<grid, kTcThreads, L::TOTAL, st>>>(ma, mb, a);
    count_launch();
    return after_launch("tc_block");
}

template <int KC>
static int dispatch_bn(int bn, const CUtensorMap &ma, const CUtensorMap &mb, TcArgs &a, int tiles, cudaStream_t st) {
    switch (bn) {
        case 32: return launch_tc<32, KC>(ma, mb, a, tiles, st);
        case 64: return launch_tc<64, KC>(ma, mb, a, tiles, st);
        case 128: return launch_tc<128, KC>(ma, mb, a, tiles, st);
        default: return launch_tc<256, KC>(ma, mb, a, tiles, st);
    }
}

// Shared launcher: x is int8 NHWC (B, H, W, C) with C % 64 == 0; w is int8 (K, T*C) tap-major.
static int tc_run(const int8_t *x, int B, int C, int H, int W, int T, const int8_t *w, int K, const int32_t *thr,
                  const uint32_t *pos, int pool, int out_fmt, void *out, int32_t *sums, int32_t *preds,
                  int bn_req, cudaStream_t st) {
    BNN_REQUIRE(C % 64 == 0, "tensor engine needs C %% 64 == 0 (got %d)", C);
    BNN_REQUIRE(out_fmt != 1 || K % 32 == 0, "int8 output needs K %% 32 == 0 (got %d)", K);
    const int KC = (C % 128 == 0) ? 128 : 64;
    TcArgs a{};
    a.T = T;
    a.CCH = C / KC;
    a.nks = T * a.CCH;
    a.W = W; a.H = H; a.B = B; a.K = K;
    if (T == 9) {
        a.BW = W <= 128 ? W : 128;
        int bh = 128 / a.BW;
        if (bh > H) bh = H;
        if (pool && (bh & 1)) bh -= 1;
        a.BH = bh < 1 ? 1 : bh;
        a.BB = (a.BH == H && a.BW == W) ? 128 / (a.BW * a.BH) : 1;
        if (a.BB > B) a.BB = B;
        BNN_REQUIRE(!pool || (a.BW == W && (a.BH % 2 == 0)), "tc pool tile %dx%d invalid for %dx%d", a.BW, a.BH, W, H);
    } else {
        a.BW = 1; a.BH = 1; a.BB = 128;
    }
    a.ntx = ceil_div(W, a.BW);
    a.nty = ceil_div(H, a.BH);
    const int ntb = ceil_div(B, a.BB);
    a.thr = thr; a.pos = pos; a.pool = pool; a.out_fmt = out_fmt; a.out = out; a.sums = sums; a.preds = preds;
    a.a_bytes = a.BW * a.BH * a.BB * KC;
    int bn = bn_req;
    if (bn != 32 && bn != 64 && bn != 128 && bn != 256) bn = K <= 32 ? 32 : K <= 64 ? 64 : K <= 128 ? 128 : 256;
    if (out_fmt == 2) BNN_REQUIRE(K <= bn, "logits tile needs K <= BN (K=%d)", K);
    a.idesc = make_idesc(128, bn, true);

    CUtensorMap ma, mb;
    const cuuint64_t adims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    const cuuint64_t astr[3] = {(cuuint64_t)C, (cuuint64_t)W * C, (cuuint64_t)H * W * C};
    const cuuint32_t abox[4] = {(cuuint32_t)KC, (cuuint32_t)a.BW, (cuuint32_t)a.BH, (cuuint32_t)a.BB};
    int e = encode_map(&ma, x, 4, adims, astr, abox, KC);
    if (e) return e;
    const cuuint64_t bdims[2] = {(cuuint64_t)T * C, (cuuint64_t)K};
    const cuuint64_t bstr[1] = {(cuuint64_t)T * C};
    const cuuint32_t bbox[2] = {(cuuint32_t)KC, (cuuint32_t)bn};
    e = encode_map(&mb, w, 2, bdims, bstr, bbox, KC);
    if (e) return e;
    const int tiles = a.ntx * a.nty * ntb;
    return KC == 128 ? dispatch_bn<128>(bn, ma, mb, a, tiles, st) : dispatch_bn<64>(bn, ma, mb, a, tiles, st);
}

int tc_conv(const int8_t *x, int B, int C, int H, int W, const int8_t *w, int K, const int32_t *thr,
            const uint32_t *pos, int pool, int out_fmt, void *out, int32_t *sums, int bn, cudaStream_t st) {
    return tc_run(x, B, C, H, W, 9, w, K, thr, pos, pool, out_fmt, out, sums, nullptr, bn, st);
}

int tc_fc(const int8_t *x, int B, int L, const int8_t *w, int M, const int32_t *thr, const uint32_t *pos,
          int out_fmt, void *out, int32_t *sums, int32_t *preds, int bn, cudaStream_t st) {
    return tc_run(x, B, L, 1, 1, 1, w, M, thr, pos, 0, out_fmt, out, sums, preds, bn, st);
}

}  // namespace bnn
