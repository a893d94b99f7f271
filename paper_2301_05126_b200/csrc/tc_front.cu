// tc_front.cu -- the network's front end as ONE persistent tcgen05 kernel:
//
//   conv_int_forward (layers.py:91-101) + step_forward (:135-146) [+ maxpool_forward (:118-132)]
//     -> +-1 int8 activation that NEVER leaves shared memory ->
//   conv_bin_forward (layers.py:104-115) + step [+ maxpool] -> HBM (int8 +-1 or NHWC bits)
//
// Why: the first layer writes the widest activation of the network (CIFAR: 64 ch x 32 x 32 =
// 64 KiB/image int8) and the second conv reads it straight back; fusing them removes that round
// trip (and the first layer's own pipeline), leaving the second conv's MMAs as the bound.
//
// Per image (CTA-persistent over images b = blockIdx.x + j * gridDim.x):
//  * X stage : the image as a pixel-major, zero-padded grid of u32 words (one byte per channel,
//              C <= 4), X[Y*wp1 + X'] = pixel (Y-1, X'-1), wp1 = W + 2; written by the loader warp
//              straight from the u8 NCHW image (double-buffered; borders stay zero).
//  * E tiles : first-layer A operand.  Output pixels are numbered padded-linear, m = y*wp1 + x
//              (x >= W are junk rows).  E row g = Y*wp1 + x = the 16 B (X[g], X[g+1], X[g+2], 0):
//              the three horizontal taps x-1, x, x+1 of padded input row Y (byte dx*4 + c).  Tap row
//              dy of output m is E row m + dy*wp1, so ONE no-swizzle K-major descriptor with
//              LBO = wp1*16 B covers dy = 0,1 in a K=32 MMA and a second covers dy = 2 (+ a junk
//              chunk multiplied by zero weights).  A = unsigned u8, B = signed s8.  Built per
//              128-row tile by two builder warps (3 word loads + one 16-B store per row), 3-deep ring.
//  * H buffer: the first block's +-1 output in the second conv's A layout: SW64 K-major rows of 64 B
//              over the zero-padded (H2+2) x (W2+2) grid, double-buffered across images.  The second
//              conv reads it with the halo trick (tc_gemm.cu: nine row-shifted descriptors).
//  * Epilogue: threshold (branch-free, tc_ptx.cuh) -> H (first block) or -> pool -> HBM (second).
// The MMA warp interleaves the two layers' tiles (L1 of image r with L2 of image r-1, Bresenham
// merge) so the tensor pipe always has second-conv work while first-layer tiles drain.
#include "common.cuh"
#include "tc_ptx.cuh"

#include <algorithm>

namespace bnn {

constexpr int kFrontEpiWarps = 16;                         // 4 TMEM lane quarters x 4 groups of 16 channels
constexpr int kFrontThreads = 128 + 32 * kFrontEpiWarps;  // w0 loader, w1 MMA, w2-3 E builders, epilogue
constexpr int kFrontK = 64;                                // K1 = K2 = 64 channels
constexpr int kERing = 3;                                  // E tile stages
constexpr int kAccBufs = 4;                                // TMEM accumulators per layer (4 x 64 cols each)
constexpr int kMaxRoundTiles = 64;                         // T1 + T2 (the merge order is a 64-bit mask)

struct FrontArgs {
    int B, C, H, W;
    int H2, W2, wp1, wp2, hp2;
    int T1, T2;
    int pool1, pool2, out_fmt;
    const uint8_t *x;
    const int8_t *w1, *w2;
    const int32_t *thr1, *thr2;
    const uint32_t *pos1, *pos2;
    void *out;
    int32_t *sums1, *sums2;
    int8_t *mid;
};

struct FrontSmem {
    uint32_t h_bytes, e_stage, x_bytes, bits1_bytes, bits2_bytes;
    uint32_t off_h, off_w2, off_w1, off_e, off_x, off_bits1, off_bits2, off_misc, total;
    __host__ __device__ static uint32_t up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }
    __host__ __device__ FrontSmem(int C, int H, int W, int pool1, int pool2) {
        const int wp1 = W + 2, H2 = pool1 ? H / 2 : H, W2 = pool1 ? W / 2 : W;
        const int wp2 = W2 + 2, hp2 = H2 + 2;
        h_bytes = up((uint32_t)hp2 * wp2 * 64, 1024);
        e_stage = up((uint32_t)(128 + 3 * wp1) * 16, 1024);
        x_bytes = up((uint32_t)(128 * ((H * wp1 + 127) / 128) + 3 * wp1 + 4) * 4, 128);  // E rows read + 2
        bits1_bytes = pool1 ? up((uint32_t)H * wp1 * 8, 128) : 0;
        bits2_bytes = pool2 ? up((uint32_t)H2 * wp2 * 8, 128) : 0;
        off_h = 0;
        off_w2 = off_h + 2 * h_bytes;       // must follow H: the last tiles' junk rows read past H[1]
        off_w1 = off_w2 + 9 * kFrontK * 64;
        off_e = off_w1 + 4 * kFrontK * 16;  // 4 chunks x 64 rows x 16 B
        off_x = off_e + kERing * e_stage;
        off_bits1 = off_x + 2 * x_bytes;
        off_bits2 = off_bits1 + bits1_bytes;
        off_misc = off_bits2 + bits2_bytes;
        // misc: 2x64 int32 T', 2x16 P words, pos words, 32 mbarriers, tmem slot
        total = off_misc + 2 * kFrontK * 4 + 2 * 16 * 4 + 16 + 32 * 8 + 16;
    }
};

// no-swizzle K-major descriptor with explicit LBO (K direction) and SBO (8-row groups)
__device__ __forceinline__ uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

#define TMEM_LD16(taddr, v)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"    \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),         \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])    \
        : "r"(taddr))

// PRMT in its generic mode: a selector nibble with bit 3 set replicates the sign of the chosen byte
// (the __byte_perm intrinsic only honours the low 3 bits).  -> (sign(a) x 8, sign(b) x 8, ...)
__device__ __forceinline__ uint32_t prmt_sign(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, 0xFB;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// Strict per-channel step of 16 accumulators as BYTE masks (layers.py:135-146), 8 ALU ops per 4 channels:
// with T' = T + pos, "v - T' < 0" is exactly NEG's "v < T" and exactly NOT POS's "v > T", so the
// sign of v - T' (replicated over a byte by PRMT's sign mode) XOR the POS byte mask P is the
// step's fire mask F (0xFF = +1).  tp = T' of the 16 channels, pm = P of the 16 channels.
__device__ __forceinline__ void fire16(const uint32_t (&v)[16], const int4 *tp, const uint4 pm, uint32_t (&F)[4]) {
    const uint32_t P[4] = {pm.x, pm.y, pm.z, pm.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int4 t = tp[k];
        const uint32_t d0 = (uint32_t)((int32_t)v[4 * k] - t.x), d1 = (uint32_t)((int32_t)v[4 * k + 1] - t.y);
        const uint32_t d2 = (uint32_t)((int32_t)v[4 * k + 2] - t.z), d3 = (uint32_t)((int32_t)v[4 * k + 3] - t.w);
        const uint32_t lo = prmt_sign(d0, d1);  // byte0 = sign(d0) x 8, byte1 = sign(d1) x 8
        const uint32_t hi = prmt_sign(d2, d3);
        F[k] = __byte_perm(lo, hi, 0x5410) ^ P[k];
    }
}

// fire masks -> 16 int8 +-1 (0xFF -> 0x01, 0x00 -> 0xFF)
__device__ __forceinline__ uint4 fire_to_pm8(const uint32_t (&F)[4]) {
    return make_uint4(~(F[0] & 0xFEFEFEFEu), ~(F[1] & 0xFEFEFEFEu), ~(F[2] & 0xFEFEFEFEu), ~(F[3] & 0xFEFEFEFEu));
}

// fire masks -> 16 channel bits (byte k of F[j] -> bit 4j + k)
__device__ __forceinline__ uint32_t fire_to_bits(const uint32_t (&F)[4]) {
    uint32_t b = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) b |= (((F[j] & 0x01010101u) * 0x01020408u) >> 24) << (4 * j);
    return b;
}

// 16 channel bits -> 16 int8 +-1 (one 16-B chunk)
__device__ __forceinline__ uint4 bits16_to_pm8(uint32_t bits) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t spread = (((bits >> (4 * k)) & 0xFu) * 0x00204081u) & 0x01010101u;
        w[k] = ~(spread * 0xFEu);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// one 16-B chunk of an SW64 K-major row (absolute-address swizzle: chunk ^= (row >> 1) & 3)
__device__ __forceinline__ void store_sw64_chunk(uint8_t *hbuf, uint32_t row, int chunk, uint4 v) {
    *reinterpret_cast<uint4 *>(hbuf + row * 64 + (((uint32_t)chunk ^ ((row >> 1) & 3u)) << 4)) = v;
}

// Merge order of one full round (L1 tiles of image r, L2 tiles of image r-1): bit k set = item k is
// an L1 tile.  Bresenham over the two tile counts, L1 first on ties.
__device__ __forceinline__ uint64_t round_mask(int T1, int T2) {
    uint64_t m = 0;
    int i1 = 0, i2 = 0;
    for (int k = 0; k < T1 + T2; ++k) {
        const bool l1 = i1 < T1 && (i2 >= T2 || i1 * T2 <= i2 * T1);
        if (l1) {
            m |= 1ull << k;
            ++i1;
        } else {
            ++i2;
        }
    }
    return m;
}

// (y, x) of padded-linear row m = t*128 + m0 for t = 0, 1, ... without a division per tile
struct RowWalker {
    int wp, qd, rm, y0, x0, y, x;
    __device__ RowWalker(int wp_, int m0) : wp(wp_), qd(128 / wp_), rm(128 % wp_), y0(m0 / wp_), x0(m0 % wp_) {
        y = y0;
        x = x0;
    }
    __device__ void at(int t) {
        if (t == 0) {
            y = y0;
            x = x0;
            return;
        }
        x += rm;
        y += qd;
        if (x >= wp) {
            x -= wp;
            ++y;
        }
    }
};

template <int POOL1, int POOL2>
__global__ void __launch_bounds__(kFrontThreads, 1) tc_front_kernel(const FrontArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    const FrontSmem L(a.C, a.H, a.W, POOL1, POOL2);
    uint8_t *sH = smem + L.off_h;
    uint8_t *sW2 = smem + L.off_w2;
    uint8_t *sW1 = smem + L.off_w1;
    uint8_t *sE = smem + L.off_e;
    uint8_t *sX = smem + L.off_x;
    uint16_t *s_bits1 = reinterpret_cast<uint16_t *>(smem + L.off_bits1);  // [row][4 groups of 16 ch]
    uint16_t *s_bits2 = reinterpret_cast<uint16_t *>(smem + L.off_bits2);
    int32_t *s_tp1 = reinterpret_cast<int32_t *>(smem + L.off_misc);  // T' = T + pos per channel
    int32_t *s_tp2 = s_tp1 + kFrontK;
    uint32_t *s_pm1 = reinterpret_cast<uint32_t *>(s_tp2 + kFrontK);  // POS byte masks, 4 channels per word
    uint32_t *s_pm2 = s_pm1 + 16;
    uint32_t *s_pos = s_pm2 + 16;  // [0..1] pos1, [2..3] pos2 (direction bits, for pooling)
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_pos + 4);
    uint64_t *xfull = bars, *xempty = bars + 2;
    uint64_t *efull = bars + 4, *eempty = bars + 4 + kERing;
    uint64_t *hfull = bars + 10, *hempty = bars + 12;
    uint64_t *t1full = bars + 14, *t1empty = t1full + kAccBufs;
    uint64_t *t2full = t1empty + kAccBufs, *t2empty = t2full + kAccBufs;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 31);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int C = a.C, H = a.H, W = a.W, wp1 = a.wp1, wp2 = a.wp2, H2 = a.H2, W2 = a.W2;
    const int n_local = a.B > (int)blockIdx.x ? (a.B - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    const int chw = C * H * W;
    constexpr int kEpiThreads = 32 * kFrontEpiWarps;

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&xfull[i], 32);
            mbar_init(&xempty[i], 2);
            mbar_init(&hfull[i], kFrontEpiWarps);
            mbar_init(&hempty[i], 1);
        }
        for (int i = 0; i < kAccBufs; ++i) {
            mbar_init(&t1full[i], 1);
            mbar_init(&t1empty[i], kFrontEpiWarps);
            mbar_init(&t2full[i], 1);
            mbar_init(&t2empty[i], kFrontEpiWarps);
        }
        for (int i = 0; i < kERing; ++i) {
            mbar_init(&efull[i], 2);
            mbar_init(&eempty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                     "r"(2 * kAccBufs * kFrontK));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // ---- one-time staging: zero H and X (their pad rows/cols stay zero = out-of-image taps contribute
    // 0), second-conv filters in SW64 K-major slabs (one 64x64 slab per tap), first-layer filters in
    // the no-swizzle [chunk dy][n][16 B] layout (byte dx*4 + c), step pairs and directions.
    for (uint32_t i = tid; i < 2 * L.h_bytes / 16; i += kFrontThreads)
        reinterpret_cast<uint4 *>(sH)[i] = make_uint4(0, 0, 0, 0);
    for (uint32_t i = tid; i < 2 * L.x_bytes / 16; i += kFrontThreads)
        reinterpret_cast<uint4 *>(sX)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < 9 * kFrontK * 4; i += kFrontThreads) {
        const int tap = i / (kFrontK * 4), rem = i % (kFrontK * 4), n = rem >> 2, c = rem & 3;
        const uint4 v = *reinterpret_cast<const uint4 *>(a.w2 + (size_t)n * 9 * kFrontK + tap * kFrontK + c * 16);
        *reinterpret_cast<uint4 *>(sW2 + tap * 4096 + n * 64 + ((c ^ ((n >> 1) & 3)) << 4)) = v;
    }
    for (int i = tid; i < 4 * kFrontK; i += kFrontThreads) {
        const int dy = i / kFrontK, n = i % kFrontK;
        uint32_t wd[4] = {0u, 0u, 0u, 0u};
        if (dy < 3) {
            for (int dx = 0; dx < 3; ++dx)
                for (int c = 0; c < C; ++c)
                    wd[dx] |= (uint32_t)(uint8_t)a.w1[(size_t)n * 9 * C + c * 9 + dy * 3 + dx] << (8 * c);
        }
        *reinterpret_cast<uint4 *>(sW1 + dy * 1024 + n * 16) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
    for (int i = tid; i < kFrontK; i += kFrontThreads) {
        const uint32_t p1 = (__ldg(a.pos1 + (i >> 5)) >> (i & 31)) & 1u, p2 = (__ldg(a.pos2 + (i >> 5)) >> (i & 31)) & 1u;
        s_tp1[i] = __ldg(a.thr1 + i) + (int32_t)p1;
        s_tp2[i] = __ldg(a.thr2 + i) + (int32_t)p2;
    }
    for (int i = tid; i < 16; i += kFrontThreads) {
        uint32_t m1 = 0, m2 = 0;
        for (int b = 0; b < 4; ++b) {
            const int c = 4 * i + b;
            m1 |= ((__ldg(a.pos1 + (c >> 5)) >> (c & 31)) & 1u) ? 0xFFu << (8 * b) : 0u;
            m2 |= ((__ldg(a.pos2 + (c >> 5)) >> (c & 31)) & 1u) ? 0xFFu << (8 * b) : 0u;
        }
        s_pm1[i] = m1;
        s_pm2[i] = m2;
    }
    if (tid < 2) {
        s_pos[tid] = __ldg(a.pos1 + tid);
        s_pos[2 + tid] = __ldg(a.pos2 + tid);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint64_t full_round = round_mask(a.T1, a.T2);

    if (warp == 0) {  // ------------------------------------------------ loader: NCHW u8 -> padded u32 pixel grid
        // 4 pixels per lane-step from 32-bit plane loads when rows are word aligned (also keeps
        // zero-copy reads of pinned host images at 4 B per PCIe request), else byte loads
        const bool vec4 = ((W & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 3) == 0);
        const int hw = H * W, gpr = W >> 2;
        for (int j = 0; j < n_local; ++j) {
            const int s = j & 1;
            mbar_wait(&xempty[s], ((j >> 1) & 1) ^ 1);
            const uint8_t *src = a.x + (size_t)(blockIdx.x + (size_t)j * gridDim.x) * chw;
            uint32_t *dst = reinterpret_cast<uint32_t *>(sX + s * L.x_bytes) + wp1 + 1;  // pixel (0, 0)
            if (vec4) {
                for (int gi = lane; gi < H * gpr; gi += 32) {
                    const int iy = gi / gpr, ix = (gi - iy * gpr) * 4;
                    uint32_t pl[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (c < C) pl[c] = __ldg(reinterpret_cast<const uint32_t *>(src + c * hw + iy * W + ix));
                    uint32_t *d = dst + iy * wp1 + ix;
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        d[k] = ((pl[0] >> (8 * k)) & 0xffu) | (((pl[1] >> (8 * k)) & 0xffu) << 8) |
                               (((pl[2] >> (8 * k)) & 0xffu) << 16) | (((pl[3] >> (8 * k)) & 0xffu) << 24);
                }
            } else {
                for (int p = lane; p < hw; p += 32) {
                    const int iy = p / W, ix = p - iy * W;
                    uint32_t v = 0;
                    for (int c = 0; c < C; ++c) v |= (uint32_t)src[c * hw + p] << (8 * c);
                    dst[iy * wp1 + ix] = v;
                }
            }
            mbar_arrive(&xfull[s]);  // release semantics: this lane's stores are visible to the waiters
        }
    } else if (warp == 1) {  // ---------------------------------------- MMA issuer (whole warp, elected lane)
        const uint32_t idesc1 = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(kFrontK >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t idesc2 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kFrontK >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t e_desc0 = desc_noswz(smem_addr(sE), (uint32_t)wp1 * 16, 128);
        const uint64_t w1_desc0 = desc_noswz(smem_addr(sW1), (uint32_t)kFrontK * 16, 128);
        const uint64_t h_desc0 = umma_desc(smem_addr(sH), 64);
        const uint64_t w2_desc0 = umma_desc(smem_addr(sW2), 64);
        uint32_t c1 = 0, c2 = 0, es = 0, epar = 0;
        for (int r = 0; r <= n_local; ++r) {
            const bool has1 = r < n_local, has2 = r >= 1;
            const int items = (has1 ? a.T1 : 0) + (has2 ? a.T2 : 0);
            int i2 = 0;
            for (int k = 0; k < items; ++k) {
                const bool l1 = has1 && (!has2 || ((full_round >> k) & 1ull));
                if (l1) {
                    mbar_wait(&efull[es], epar);
                    const uint32_t acc = c1 % kAccBufs;
                    mbar_wait(&t1empty[acc], ((c1 / kAccBufs) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem_base + acc * kFrontK;
                    const uint64_t ad = e_desc0 + ((es * L.e_stage) >> 4);
                    umma_i8_elect(d, ad, w1_desc0, idesc1, 0);
                    umma_i8_elect(d, ad + ((2u * wp1 * 16) >> 4), w1_desc0 + (2048 >> 4), idesc1, 1);
                    umma_commit_elect(&eempty[es]);
                    umma_commit_elect(&t1full[acc]);
                    if (++es == kERing) {
                        es = 0;
                        epar ^= 1;
                    }
                    ++c1;
                } else {
                    const int jj = r - 1, hb = jj & 1;
                    if (i2 == 0) mbar_wait(&hfull[hb], (jj >> 1) & 1);
                    const uint32_t acc = c2 % kAccBufs;
                    mbar_wait(&t2empty[acc], ((c2 / kAccBufs) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem_base + (kAccBufs + acc) * kFrontK;
                    const uint64_t base = h_desc0 + ((hb * L.h_bytes + (uint32_t)i2 * 128 * 64) >> 4);
#pragma unroll
                    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                        for (int dx = 0; dx < 3; ++dx) {
                            const int tap = dy * 3 + dx;
                            const uint64_t ad = base + (((uint32_t)(dy * wp2 + dx) * 64) >> 4);
                            const uint64_t bd = w2_desc0 + ((tap * 4096) >> 4);
                            umma_i8_elect(d, ad, bd, idesc2, tap != 0);
                            umma_i8_elect(d, ad + 2, bd + 2, idesc2, 1);
                        }
                    umma_commit_elect(&t2full[acc]);
                    ++c2;
                    if (++i2 == a.T2) umma_commit_elect(&hempty[hb]);
                }
            }
        }
        __syncwarp();
    } else if (warp < 4) {  // ---------------------------------------- E builders (64 threads)
        const int bt = tid - 64;
        const int e_rows = 128 + 2 * wp1;  // rows read with non-zero weights
        uint32_t es = 0, epar = 1;
        for (int j = 0; j < n_local; ++j) {
            const int s = j & 1;
            mbar_wait(&xfull[s], (j >> 1) & 1);
            const uint32_t *xg = reinterpret_cast<const uint32_t *>(sX + s * L.x_bytes);
            for (int t = 0; t < a.T1; ++t) {
                mbar_wait(&eempty[es], epar);
                uint4 *stage = reinterpret_cast<uint4 *>(sE + es * L.e_stage);
                const uint32_t *xt = xg + t * 128;
                for (int l = bt; l < e_rows; l += 64) stage[l] = make_uint4(xt[l], xt[l + 1], xt[l + 2], 0u);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&efull[es]);
                if (++es == kERing) {
                    es = 0;
                    epar ^= 1;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&xempty[s]);
        }
    } else {  // -------------------------------------------------------- epilogue (16 warps)
        // warp -> (TMEM lane quarter q = warp % 4 [hardware rule], channel group g of 16)
        const int q = warp & 3, g = (warp - 4) >> 2;
        const int et = tid - 128;
        const int m0 = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const int Ho = POOL2 ? H2 / 2 : H2, Wo = POOL2 ? W2 / 2 : W2;
        RowWalker rw1(wp1, m0), rw2(wp2, m0);
        uint32_t c1 = 0, c2 = 0;
        for (int r = 0; r <= n_local; ++r) {
            const bool has1 = r < n_local, has2 = r >= 1;
            const int items = (has1 ? a.T1 : 0) + (has2 ? a.T2 : 0);
            const long long img1 = (long long)blockIdx.x + (long long)r * gridDim.x;
            const long long img2 = img1 - gridDim.x;
            uint8_t *hb1 = sH + (r & 1) * L.h_bytes;
            if (has1) mbar_wait(&hempty[r & 1], ((r >> 1) & 1) ^ 1);  // L2 of image r-2 done reading H
            if (POOL1 || POOL2) bar_named(1, kEpiThreads);             // previous round's pool passes done
            int i1 = 0, i2 = 0;
            for (int k = 0; k < items; ++k) {
                const bool l1 = has1 && (!has2 || ((full_round >> k) & 1ull));
                const uint32_t cnt = l1 ? c1 : c2;
                const uint32_t acc = cnt % kAccBufs;
                mbar_wait(l1 ? &t1full[acc] : &t2full[acc], (cnt / kAccBufs) & 1);
                tc_fence_after();
                uint32_t v[16];
                TMEM_LD16(tmem_base + ((l1 ? 0u : (uint32_t)kAccBufs) + acc) * kFrontK + g * 16 + lane_off, v);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(l1 ? &t1empty[acc] : &t2empty[acc]);
                if (l1) {
                    const int t = i1++;
                    rw1.at(t);
                    const int m = t * 128 + m0, y = rw1.y, x = rw1.x;
                    const bool row_ok = m < H * wp1;
                    if (a.sums1 && row_ok && x < W) {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            a.sums1[((img1 * kFrontK + g * 16 + i) * H + y) * W + x] = (int32_t)v[i];
                    }
                    uint32_t F[4];
                    fire16(v, reinterpret_cast<const int4 *>(s_tp1) + g * 4, reinterpret_cast<const uint4 *>(s_pm1)[g], F);
                    if (POOL1) {
                        if (row_ok) s_bits1[m * 4 + g] = (uint16_t)fire_to_bits(F);
                    } else if (row_ok) {
                        const uint4 pm = x < W ? fire_to_pm8(F) : make_uint4(0, 0, 0, 0);
                        store_sw64_chunk(hb1, (uint32_t)(m + wp1 + 1), g, pm);
                        if (a.mid && x < W)
                            *reinterpret_cast<uint4 *>(a.mid + ((img1 * H + y) * W + x) * kFrontK + g * 16) = pm;
                    }
                    ++c1;
                    if (i1 == a.T1) {
                        if (POOL1) {  // 2x2 pool of thresholded bits (OR for POS, AND for NEG) -> H
                            bar_named(2, kEpiThreads);
                            for (int p = et; p < H2 * W2 * 4; p += kEpiThreads) {
                                const int pp = p >> 2, gg = p & 3, py = pp / W2, px = pp - py * W2;
                                const int m00 = 2 * py * wp1 + 2 * px;
                                const uint32_t b0 = s_bits1[m00 * 4 + gg], b1 = s_bits1[(m00 + 1) * 4 + gg];
                                const uint32_t b2 = s_bits1[(m00 + wp1) * 4 + gg], b3 = s_bits1[(m00 + wp1 + 1) * 4 + gg];
                                const uint32_t pw = (s_pos[gg >> 1] >> (16 * (gg & 1))) & 0xffffu;
                                const uint32_t pb = ((b0 | b1 | b2 | b3) & pw) | ((b0 & b1 & b2 & b3) & ~pw);
                                const uint4 pm = bits16_to_pm8(pb);
                                store_sw64_chunk(hb1, (uint32_t)((py + 1) * wp2 + px + 1), gg, pm);
                                if (a.mid)
                                    *reinterpret_cast<uint4 *>(a.mid + ((img1 * H2 + py) * W2 + px) * kFrontK + gg * 16) = pm;
                            }
                        }
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&hfull[r & 1]);
                    }
                } else {
                    const int t = i2++;
                    rw2.at(t);
                    const int m = t * 128 + m0, y = rw2.y, x = rw2.x;
                    const bool row_ok = m < H2 * wp2;
                    const bool pix_ok = row_ok && x < W2;
                    if (a.sums2 && pix_ok) {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            a.sums2[((img2 * kFrontK + g * 16 + i) * H2 + y) * W2 + x] = (int32_t)v[i];
                    }
                    uint32_t F[4];
                    fire16(v, reinterpret_cast<const int4 *>(s_tp2) + g * 4, reinterpret_cast<const uint4 *>(s_pm2)[g], F);
                    if (POOL2) {
                        if (row_ok) s_bits2[m * 4 + g] = (uint16_t)fire_to_bits(F);
                    } else if (pix_ok && a.out) {
                        const long long pix = (img2 * H2 + y) * W2 + x;
                        if (a.out_fmt == 0)
                            static_cast<uint16_t *>(a.out)[pix * 4 + g] = (uint16_t)fire_to_bits(F);
                        else
                            *reinterpret_cast<uint4 *>(static_cast<int8_t *>(a.out) + pix * kFrontK + g * 16) =
                                fire_to_pm8(F);
                    }
                    ++c2;
                    if (i2 == a.T2 && POOL2) {
                        bar_named(3, kEpiThreads);
                        for (int p = et; p < Ho * Wo * 4; p += kEpiThreads) {
                            const int pp = p >> 2, gg = p & 3, py = pp / Wo, px = pp - py * Wo;
                            const int m00 = 2 * py * wp2 + 2 * px;
                            const uint32_t b0 = s_bits2[m00 * 4 + gg], b1 = s_bits2[(m00 + 1) * 4 + gg];
                            const uint32_t b2 = s_bits2[(m00 + wp2) * 4 + gg], b3 = s_bits2[(m00 + wp2 + 1) * 4 + gg];
                            const uint32_t pw = (s_pos[2 + (gg >> 1)] >> (16 * (gg & 1))) & 0xffffu;
                            const uint32_t pb = ((b0 | b1 | b2 | b3) & pw) | ((b0 & b1 & b2 & b3) & ~pw);
                            if (!a.out) continue;
                            const long long pix = (img2 * Ho + py) * Wo + px;
                            if (a.out_fmt == 0)
                                static_cast<uint16_t *>(a.out)[pix * 4 + gg] = (uint16_t)pb;
                            else
                                *reinterpret_cast<uint4 *>(static_cast<int8_t *>(a.out) + pix * kFrontK + gg * 16) =
                                    bits16_to_pm8(pb);
                        }
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * kAccBufs * kFrontK));
    }
}

static int front_sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

int tc_front_smem(int C, int H, int W, int K1, int K2, int pool1, int pool2) {
    if (K1 != kFrontK || K2 != kFrontK || C < 1 || C > 4 || H < 1 || W < 1) return -1;
    if ((pool1 && ((H | W) & 1)) || W + 2 > 1024) return -1;
    const int H2 = pool1 ? H / 2 : H, W2 = pool1 ? W / 2 : W;
    if (pool2 && ((H2 | W2) & 1)) return -1;
    if (ceil_div((long long)H * (W + 2), 128) + ceil_div((long long)H2 * (W2 + 2), 128) > kMaxRoundTiles) return -1;
    const FrontSmem L(C, H, W, pool1, pool2);
    const size_t need = (size_t)L.total + 1024;
    return need <= 227 * 1024 ? (int)need : -1;
}

int tc_front(const uint8_t *x, int B, int C, int H, int W, const int8_t *w1, const int32_t *thr1,
             const uint32_t *pos1, int pool1, const int8_t *w2, const int32_t *thr2, const uint32_t *pos2, int pool2,
             int K1, int K2, int out_fmt, void *out, int32_t *sums1, int8_t *mid, int32_t *sums2, cudaStream_t st) {
    const int smem = tc_front_smem(C, H, W, K1, K2, pool1, pool2);
    BNN_REQUIRE(smem > 0, "tc_front: unsupported shape C=%d H=%d W=%d K1=%d K2=%d pool1=%d pool2=%d", C, H, W, K1, K2,
                pool1, pool2);
    BNN_REQUIRE(out_fmt == 0 || out_fmt == 1, "tc_front: out_fmt must be bits (0) or int8 (1)");
    FrontArgs a{};
    a.B = B; a.C = C; a.H = H; a.W = W;
    a.H2 = pool1 ? H / 2 : H;
    a.W2 = pool1 ? W / 2 : W;
    a.wp1 = W + 2;
    a.wp2 = a.W2 + 2;
    a.hp2 = a.H2 + 2;
    a.T1 = ceil_div((long long)H * a.wp1, 128);
    a.T2 = ceil_div((long long)a.H2 * a.wp2, 128);
    a.pool1 = pool1; a.pool2 = pool2; a.out_fmt = out_fmt;
    a.x = x; a.w1 = w1; a.w2 = w2; a.thr1 = thr1; a.thr2 = thr2; a.pos1 = pos1; a.pos2 = pos2;
    a.out = out; a.sums1 = sums1; a.sums2 = sums2; a.mid = mid;
    if (B == 0) return 0;
    const int grid = std::min(B, front_sm_count());
#define BNN_FRONT(P1, P2)                                                                \
    {                                                                                    \
        auto kern = tc_front_kernel<P1, P2>;                                             \
        int e = allow_smem(reinterpret_cast<const void *>(kern), (size_t)smem, "tc_front"); \
        if (e) return e;                                                                 \
        kern<<<grid, kFrontThreads, smem, st>>>(a);                                      \
    }
    if (pool1) {
        if (pool2) BNN_FRONT(1, 1) else BNN_FRONT(1, 0)
    } else {
        if (pool2) BNN_FRONT(0, 1) else BNN_FRONT(0, 0)
    }
#undef BNN_FRONT
    count_launch();
    return after_launch("tc_front");
}

}  // namespace bnn
