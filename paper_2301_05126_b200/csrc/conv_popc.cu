// conv_popc.cu -- fused 3x3 convolution blocks on the integer pipe.
//
//   conv_bin : implicit-GEMM xor-popcount over NHWC channel-packed bits
//              (reference numerics: conv_bin_forward, layers.py:104-115;
//               packed route: backends.py:210-256)
//   conv_first: integer pixels x +-1 filters (conv_int_forward, layers.py:91-101)
//
// Both share one CTA geometry and one fused epilogue:
//   * 256 threads; a thread owns a 2x2 output "quad" x 8 output channels
//     (32 int accumulators).  Lane = quad_lo*4 + cg4: the 4 lanes that hold
//     the 4 byte-slices of one 32-channel output word are adjacent, so the
//     re-pack is two shfl_xor.
//   * a CTA covers QT consecutive quads (row-major over batch x quad-rows x
//     quad-cols) and tile_n output channels.  The padded input images the
//     quad window touches are staged whole in shared memory (zero halo) and
//     the CTA's weight tile is staged once: [tap*CW + j][tile_n].
//   * epilogue: int32 pre-activation -> optional NCHW int32 dump (layer API /
//     parity) -> strict per-channel threshold -> optional 2x2 pool, which on
//     thresholded bits is OR for POS channels and AND for NEG channels
//     (max(v) > T <=> any v > T;  max(v) < T <=> all v < T) -> ballot-free
//     shuffle re-pack into NHWC words.
//   * out-of-image taps contribute nothing (layers.py:70-80): their mask is 0
//     in the LOP3 (x ^ w) & m, and they are excluded from the valid count.
#include <cstdio>

#include "common.cuh"

namespace bnn {

constexpr int kThreads = 256;

struct ConvArgs {
    const void *x;
    const uint32_t *mask;
    int B, C, H, W, CW;
    int He, We;          // H, W rounded up to even
    int QW, QPI;         // quads per row / per image
    long long nquads;    // B * QPI
    const void *w;
    int K, KW;
    const int32_t *thr;
    const uint32_t *pos;
    uint32_t *out;
    int32_t *sums;
    int tile_n, QT, max_imgs;
    int out_fmt;  // 0 = NHWC bits (u32 words), 1 = NHWC FP4 +-1 (tensor-engine input)
};

// 8 channel bits -> 8 int8 bytes (+1 / -1)

// ---------------------------------------------------------------- epilogue
template <bool POOL>
__device__ __forceinline__ void quad_epilogue(const ConvArgs &a, const int (&dot)[4][8], bool active,
                                              int b, int qy, int qx, int k0, int cg4) {
    // k0 = first of this thread's 8 channels
    const int py0 = 2 * qy, px0 = 2 * qx;
    if (a.sums && active) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int k = k0 + c;
            if (k >= a.K) continue;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int py = py0 + (p >> 1), px = px0 + (p & 1);
                if (py < a.H && px < a.W)
                    a.sums[(((long long)b * a.K + k) * a.H + py) * a.W + px] = dot[p][c];
            }
        }
    }
    if (!a.out) return;  // uniform across the CTA
    const int kw = k0 >> 5;
    const bool word_ok = (kw << 5) < a.K;  // tile_n may exceed K: never store past the last word
    if (POOL) {
        uint32_t byte = 0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int k = k0 + c;
            if (active && k < a.K) {
                const int t = __ldg(a.thr + k);
                const bool pos = dir_pos(a.pos, k);
                uint32_t any = 0, all = 1;
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const uint32_t s = step_bit(dot[p][c], t, pos);
                    any |= s;
                    all &= s;
                }
                byte |= (pos ? any : all) << c;
            }
        }
        if (a.out_fmt == 1) {
            if (active && k0 < a.K) {
                const long long opix = ((long long)b * (a.H >> 1) + qy) * (a.W >> 1) + qx;
                *reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(a.out) + (opix * a.K + k0) / 2) =
                    bits8_to_f4(byte);
            }
            return;
        }
        uint32_t word = byte << (cg4 * 8);
        word |= __shfl_xor_sync(0xffffffffu, word, 1);
        word |= __shfl_xor_sync(0xffffffffu, word, 2);
        if (active && word_ok && cg4 == 0)
            a.out[(((long long)b * (a.H >> 1) + qy) * (a.W >> 1) + qx) * a.KW + kw] = word;
    } else {
        uint32_t word[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int k = k0 + c;
            if (active && k < a.K) {
                const int t = __ldg(a.thr + k);
                const bool pos = dir_pos(a.pos, k);
#pragma unroll
                for (int p = 0; p < 4; ++p) word[p] |= step_bit(dot[p][c], t, pos) << c;
            }
        }
        if (a.out_fmt == 1) {
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int py = py0 + (p >> 1), px = px0 + (p & 1);
                if (active && k0 < a.K && py < a.H && px < a.W) {
                    const long long pix = ((long long)b * a.H + py) * a.W + px;
                    *reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(a.out) + (pix * a.K + k0) / 2) =
                        bits8_to_f4(word[p]);
                }
            }
            return;
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            word[p] <<= cg4 * 8;
            word[p] |= __shfl_xor_sync(0xffffffffu, word[p], 1);
            word[p] |= __shfl_xor_sync(0xffffffffu, word[p], 2);
        }
        // lane cg4 stores pixel p == cg4 of the quad
        uint32_t mine = word[0];
#pragma unroll
        for (int p = 1; p < 4; ++p)
            if (cg4 == p) mine = word[p];
        const int py = py0 + (cg4 >> 1), px = px0 + (cg4 & 1);
        if (active && word_ok && py < a.H && px < a.W)
            a.out[(((long long)b * a.H + py) * a.W + px) * a.KW + kw] = mine;
    }
}

// Thread -> (quad, channel group) decode shared by both kernels.
struct QuadPos {
    int lq, cg4, nw;
    long long g;
    int b, qy, qx;
    bool active;
};

__device__ __forceinline__ QuadPos decode_quad(const ConvArgs &a) {
    QuadPos q;
    const int t = threadIdx.x;
    q.cg4 = t & 3;
    const int qlo = (t >> 2) & 7;
    const int warp = t >> 5;
    const int nwt = a.tile_n >> 5;
    q.nw = warp % nwt;
    q.lq = (warp / nwt) * 8 + qlo;
    q.g = (long long)blockIdx.x * a.QT + q.lq;
    q.active = q.g < a.nquads;
    const long long g = q.active ? q.g : 0;
    q.b = (int)(g / a.QPI);
    const int r = (int)(g % a.QPI);
    q.qy = r / a.QW;
    q.qx = r % a.QW;
    return q;
}

// ---------------------------------------------------------------- conv_bin
template <int JV, bool POOL, bool MASKED>
__global__ void __launch_bounds__(kThreads) conv_bin_popc_kernel(const ConvArgs a) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    extern __shared__ __align__(16) uint32_t smem[];
    const int CW = a.CW;
    const int pw = a.We + 2, ph = a.He + 2;
    const long long g0 = (long long)blockIdx.x * a.QT;
    const int b_first = (int)(g0 / a.QPI);
    const long long g_last = min(g0 + a.QT, a.nquads) - 1;
    const int nimg = (int)(g_last / a.QPI) - b_first + 1;
    const int img_words = ph * pw * CW;
    uint32_t *s_x = smem;
    uint32_t *s_m = s_x + (long long)a.max_imgs * img_words;
    uint32_t *s_w = s_m + (MASKED ? (long long)a.max_imgs * img_words : 0);
    const int n_cta = blockIdx.y * a.tile_n;

    // stage padded images (zero halo / zero beyond H,W) -- JV-word granules
    {
        const uint32_t *xg = static_cast<const uint32_t *>(a.x);
        const int gpp = CW / JV;  // granules per pixel
        const int total = nimg * ph * pw * gpp;
        for (int i = threadIdx.x; i < total; i += kThreads) {
            const int jg = i % gpp;
            int rest = i / gpp;
            const int px = rest % pw;
            rest /= pw;
            const int py = rest % ph;
            const int li = rest / ph;
            const int iy = py - 1, ix = px - 1;
            const bool in = iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
            const long long src = ((((long long)(b_first + li) * a.H + iy) * a.W + ix) * CW) + jg * JV;
            const int dst = ((li * ph + py) * pw + px) * CW + jg * JV;
#pragma unroll
            for (int v = 0; v < JV; ++v) {
                s_x[dst + v] = in ? __ldg(xg + src + v) : 0u;
                if (MASKED) s_m[dst + v] = in ? __ldg(a.mask + src + v) : 0u;
            }
        }
        // weight tile [9*CW][tile_n]
        const uint32_t *wg = static_cast<const uint32_t *>(a.w);
        const int rows = 9 * CW;
        for (int i = threadIdx.x; i < rows * a.tile_n; i += kThreads) {
            const int n = i % a.tile_n, r = i / a.tile_n;
            const int k = n_cta + n;
            s_w[i] = k < a.K ? __ldg(wg + (long long)r * a.K + k) : 0u;
        }
    }
    __syncthreads();

    const QuadPos q = decode_quad(a);
    const int li = q.b - b_first;
    const int cgoff = q.nw * 32 + q.cg4 * 8;  // channel offset inside the CTA tile
    int acc[4][8];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[p][c] = 0;
    int valid[4] = {0, 0, 0, 0};

    if (q.active) {
#pragma unroll 1
        for (int t = 0; t < 9; ++t) {
            const int dy = t / 3, dx = t - 3 * (t / 3);
            int off[4];
            uint32_t m[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int py = 2 * q.qy + (p >> 1), px = 2 * q.qx + (p & 1);
                const int iy = py + dy - 1, ix = px + dx - 1;
                const bool ok = iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
                m[p] = ok ? 0xffffffffu : 0u;
                if (!MASKED) valid[p] += ok ? a.C : 0;
                off[p] = ((li * ph + py + dy) * pw + px + dx) * CW;
            }
            const uint32_t *wrow = s_w + (t * CW) * a.tile_n + cgoff;
#pragma unroll 1
            for (int j = 0; j < CW; j += JV) {
                uint32_t xv[4][JV];
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    if constexpr (JV == 4) {
                        const uint4 v4 = *reinterpret_cast<const uint4 *>(s_x + off[p] + j);
                        xv[p][0] = v4.x; xv[p][1] = v4.y; xv[p][2] = v4.z; xv[p][3] = v4.w;
                    } else if constexpr (JV == 2) {
                        const uint2 v2 = *reinterpret_cast<const uint2 *>(s_x + off[p] + j);
                        xv[p][0] = v2.x; xv[p][1] = v2.y;
                    } else {
                        xv[p][0] = s_x[off[p] + j];
                    }
                }
                uint32_t mm[4][JV];
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int v = 0; v < JV; ++v) {
                        if (MASKED) {
                            mm[p][v] = s_m[off[p] + j + v] & m[p];
                            valid[p] += popc(mm[p][v]);
                        } else {
                            mm[p][v] = m[p];
                        }
                    }
#pragma unroll
                for (int v = 0; v < JV; ++v) {
                    const uint4 w0 = *reinterpret_cast<const uint4 *>(wrow + (j + v) * a.tile_n);
                    const uint4 w1 = *reinterpret_cast<const uint4 *>(wrow + (j + v) * a.tile_n + 4);
                    const uint32_t wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                    for (int p = 0; p < 4; ++p)
#pragma unroll
                        for (int c = 0; c < 8; ++c) acc[p][c] += popc(xor_and(xv[p][v], wv[c], mm[p][v]));
                }
            }
        }
    }
    int dot[4][8];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int c = 0; c < 8; ++c) dot[p][c] = valid[p] - 2 * acc[p][c];
    quad_epilogue<POOL>(a, dot, q.active, q.b, q.qy, q.qx, n_cta + cgoff, q.cg4);
}

// ---------------------------------------------------------------- conv_first
template <typename Tin, bool POOL>
__global__ void __launch_bounds__(kThreads) conv_first_kernel(const ConvArgs a) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    extern __shared__ __align__(16) int32_t smem_i[];
    const int C = a.C;
    const int pw = a.We + 2, ph = a.He + 2;
    const long long g0 = (long long)blockIdx.x * a.QT;
    const int b_first = (int)(g0 / a.QPI);
    const long long g_last = min(g0 + a.QT, a.nquads) - 1;
    const int nimg = (int)(g_last / a.QPI) - b_first + 1;
    const int img_elems = C * ph * pw;
    int32_t *s_x = smem_i;
    int32_t *s_w = s_x + a.max_imgs * img_elems;
    const int n_cta = blockIdx.y * a.tile_n;
    {
        const Tin *xg = static_cast<const Tin *>(a.x);
        const int total = nimg * img_elems;
        for (int i = threadIdx.x; i < total; i += kThreads) {
            const int px = i % pw;
            int rest = i / pw;
            const int py = rest % ph;
            rest /= ph;
            const int c = rest % C;
            const int li = rest / C;
            const int iy = py - 1, ix = px - 1;
            const bool in = iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
            s_x[i] = in ? (int32_t)xg[(((long long)(b_first + li) * C + c) * a.H + iy) * a.W + ix] : 0;
        }
        const int8_t *wg = static_cast<const int8_t *>(a.w);
        const int taps = 9 * C;
        for (int i = threadIdx.x; i < taps * a.tile_n; i += kThreads) {
            const int n = i % a.tile_n, r = i / a.tile_n;
            const int k = n_cta + n;
            s_w[i] = k < a.K ? (int32_t)wg[(long long)k * taps + r] : 0;
        }
    }
    __syncthreads();

    const QuadPos q = decode_quad(a);
    const int li = q.b - b_first;
    const int cgoff = q.nw * 32 + q.cg4 * 8;
    int acc[4][8];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[p][c] = 0;
    if (q.active) {
#pragma unroll 1
        for (int ci = 0; ci < C; ++ci) {
            const int32_t *plane = s_x + (li * C + ci) * ph * pw;
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                const int dy = t / 3, dx = t % 3;
                int xv[4];
#pragma unroll
                for (int p = 0; p < 4; ++p)
                    xv[p] = plane[(2 * q.qy + (p >> 1) + dy) * pw + 2 * q.qx + (p & 1) + dx];
                const int32_t *wr = s_w + (ci * 9 + t) * a.tile_n + cgoff;
                const int4 w0 = *reinterpret_cast<const int4 *>(wr);
                const int4 w1 = *reinterpret_cast<const int4 *>(wr + 4);
                const int wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[p][c] += xv[p] * wv[c];
            }
        }
    }
    quad_epilogue<POOL>(a, acc, q.active, q.b, q.qy, q.qx, n_cta + cgoff, q.cg4);
}

// ---------------------------------------------------------------- conv_first, u8 pixels on IDP4A
// Per CTA: stage the padded u8 images, build each output pixel's im2col row once
// (9*C taps in (c, dy, dx) order, 4 per u32, zero-padded), stage the +-1 filters
// as packed s8x4 words, then acc += dp4a(u8x4 pixels, s8x4 weights): 4 MACs per
// instruction instead of 1 IMAD.  Padding taps read the zero halo -> contribute 0.
__device__ __forceinline__ int dp4a_us(uint32_t a_u8x4, uint32_t b_s8x4, int c) {
    int d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a_u8x4), "r"(b_s8x4), "r"(c));
    return d;
}

template <bool POOL>
__global__ void __launch_bounds__(kThreads) conv_first_dp4a_kernel(const ConvArgs a) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    extern __shared__ __align__(16) uint32_t smem_w[];
    const int C = a.C;
    const int taps = 9 * C, TW = (taps + 3) / 4;
    const int pw = a.We + 2, ph = a.He + 2;
    const long long g0 = (long long)blockIdx.x * a.QT;
    const int b_first = (int)(g0 / a.QPI);
    const long long g_last = min(g0 + a.QT, a.nquads) - 1;
    const int nimg = (int)(g_last / a.QPI) - b_first + 1;
    const int img_bytes = C * ph * pw;
    uint32_t *s_w = smem_w;                                  // [TW][tile_n]
    uint32_t *s_col = s_w + TW * a.tile_n;                   // [QT*4][TW]
    uint8_t *s_img = reinterpret_cast<uint8_t *>(s_col + a.QT * 4 * TW);
    const int n_cta = blockIdx.y * a.tile_n;
    {
        const uint8_t *xg = static_cast<const uint8_t *>(a.x);
        for (int i = threadIdx.x; i < nimg * img_bytes; i += kThreads) {
            const int px = i % pw;
            int rest = i / pw;
            const int py = rest % ph;
            rest /= ph;
            const int c = rest % C;
            const int li = rest / C;
            const int iy = py - 1, ix = px - 1;
            const bool in = iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
            s_img[i] = in ? xg[(((long long)(b_first + li) * C + c) * a.H + iy) * a.W + ix] : (uint8_t)0;
        }
        const int8_t *wg = static_cast<const int8_t *>(a.w);
        for (int i = threadIdx.x; i < TW * a.tile_n; i += kThreads) {
            const int n = i % a.tile_n, t4 = i / a.tile_n;
            const int k = n_cta + n;
            uint32_t word = 0;
            if (k < a.K) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int tap = 4 * t4 + q;
                    const uint32_t byte = tap < taps ? (uint8_t)wg[(long long)k * taps + tap] : 0u;
                    word |= byte << (8 * q);
                }
            }
            s_w[i] = word;
        }
    }
    __syncthreads();
    // im2col rows: one thread per CTA pixel
    for (int i = threadIdx.x; i < a.QT * 4; i += kThreads) {
        const long long g = g0 + i / 4;
        const int p = i % 4;
        uint32_t *row = s_col + i * TW;
        if (g >= a.nquads) {
            for (int t4 = 0; t4 < TW; ++t4) row[t4] = 0;
            continue;
        }
        const int bimg = (int)(g / a.QPI), r = (int)(g % a.QPI);
        const int py = 2 * (r / a.QW) + (p >> 1), px = 2 * (r % a.QW) + (p & 1);
        const uint8_t *base = s_img + (bimg - b_first) * img_bytes;
        for (int t4 = 0; t4 < TW; ++t4) {
            uint32_t word = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int tap = 4 * t4 + q;
                if (tap < taps) {
                    const int c = tap / 9, d = tap % 9;
                    word |= (uint32_t)base[(c * ph + py + d / 3) * pw + px + d % 3] << (8 * q);
                }
            }
            row[t4] = word;
        }
    }
    __syncthreads();

    const QuadPos q = decode_quad(a);
    const int cgoff = q.nw * 32 + q.cg4 * 8;
    int acc[4][8];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[p][c] = 0;
    if (q.active) {
        const uint32_t *col = s_col + q.lq * 4 * TW;
#pragma unroll 1
        for (int t4 = 0; t4 < TW; ++t4) {
            uint32_t xv[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) xv[p] = col[p * TW + t4];
            const uint4 w0 = *reinterpret_cast<const uint4 *>(s_w + t4 * a.tile_n + cgoff);
            const uint4 w1 = *reinterpret_cast<const uint4 *>(s_w + t4 * a.tile_n + cgoff + 4);
            const uint32_t wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[p][c] = dp4a_us(xv[p], wv[c], acc[p][c]);
        }
    }
    quad_epilogue<POOL>(a, acc, q.active, q.b, q.qy, q.qx, n_cta + cgoff, q.cg4);
}

// ---------------------------------------------------------------- host side
static int fill_geometry(ConvArgs &a, int tile_n) {
    a.He = a.H + (a.H & 1);
    a.We = a.W + (a.W & 1);
    a.QW = a.We / 2;
    a.QPI = (a.He / 2) * a.QW;
    a.nquads = (long long)a.B * a.QPI;
    a.KW = (a.K + 31) / 32;
    a.tile_n = tile_n;
    a.QT = 8 * (8 / (tile_n / 32));
    a.max_imgs = (int)std::min<long long>(a.B, (a.QT + a.QPI - 1) / a.QPI + 1);
    return 0;
}

static int pick_tile_n(int K, int requested) {
    if (requested == 32 || requested == 64 || requested == 128 || requested == 256) return requested;
    return K <= 32 ? 32 : 64;
}

constexpr size_t kMaxSmem = 227 * 1024;

template <typename Kern>
static int launch_conv(Kern kern, const ConvArgs &a, size_t smem, cudaStream_t st, const char *name) {
    int e = allow_smem(reinterpret_cast<const void *>(kern), kMaxSmem, name);
    if (e) return e;
    dim3 grid((unsigned)ceil_div(a.nquads, a.QT), (unsigned)ceil_div(a.K, a.tile_n));
    launch_kernel(kern, dim3(grid), dim3(kThreads), smem, st, a);
    count_launch();
    return after_launch(name);
}

int conv_bin_popc(const uint32_t *x, const uint32_t *mask, int B, int C, int H, int W, const uint32_t *w,
                  int K, const int32_t *thr, const uint32_t *pos, int pool, int out_fmt, void *out, int32_t *sums,
                  int tile_n_req, cudaStream_t st) {
    ConvArgs a{};
    a.out_fmt = out_fmt;
    a.x = x; a.mask = mask; a.B = B; a.C = C; a.H = H; a.W = W; a.CW = (C + 31) / 32;
    a.w = w; a.K = K; a.thr = thr; a.pos = pos; a.out = static_cast<uint32_t *>(out); a.sums = sums;
    fill_geometry(a, pick_tile_n(K, tile_n_req));
    const size_t img_bytes = (size_t)(a.He + 2) * (a.We + 2) * a.CW * 4;
    size_t smem = img_bytes * a.max_imgs * (mask ? 2 : 1) + (size_t)9 * a.CW * a.tile_n * 4;
    while (smem > kMaxSmem && a.tile_n > 32) {
        fill_geometry(a, a.tile_n / 2);
        smem = img_bytes * a.max_imgs * (mask ? 2 : 1) + (size_t)9 * a.CW * a.tile_n * 4;
    }
    BNN_REQUIRE(smem <= kMaxSmem, "conv_bin: padded image (%dx%dx%d) does not fit shared memory", H, W, C);
    const int jv = (a.CW % 4 == 0) ? 4 : (a.CW % 2 == 0) ? 2 : 1;
#define BNN_CB(JV, P, M) \
    return launch_conv(conv_bin_popc_kernel<JV, P, M>, a, smem, st, "conv_bin_popc")
    const bool m = mask != nullptr;
    if (jv == 4) {
        if (pool) { if (m) BNN_CB(4, true, true); else BNN_CB(4, true, false); }
        else { if (m) BNN_CB(4, false, true); else BNN_CB(4, false, false); }
    } else if (jv == 2) {
        if (pool) { if (m) BNN_CB(2, true, true); else BNN_CB(2, true, false); }
        else { if (m) BNN_CB(2, false, true); else BNN_CB(2, false, false); }
    } else {
        if (pool) { if (m) BNN_CB(1, true, true); else BNN_CB(1, true, false); }
        else { if (m) BNN_CB(1, false, true); else BNN_CB(1, false, false); }
    }
#undef BNN_CB
}

int conv_first(const void *x, int x_is_u8, int B, int C, int H, int W, const int8_t *w, int K,
               const int32_t *thr, const uint32_t *pos, int pool, int out_fmt, void *out, int32_t *sums,
               cudaStream_t st) {
    ConvArgs a{};
    a.out_fmt = out_fmt;
    a.x = x; a.B = B; a.C = C; a.H = H; a.W = W; a.CW = 0;
    a.w = w; a.K = K; a.thr = thr; a.pos = pos; a.out = static_cast<uint32_t *>(out); a.sums = sums;
    fill_geometry(a, K <= 32 ? 32 : 64);
    const size_t img_bytes = (size_t)C * (a.He + 2) * (a.We + 2) * 4;
    size_t smem = img_bytes * a.max_imgs + (size_t)9 * C * a.tile_n * 4;
    BNN_REQUIRE(smem <= kMaxSmem, "conv_int: padded image (%dx%dx%d) does not fit shared memory", H, W, C);
    if (x_is_u8) {
        const size_t tw = (9 * (size_t)C + 3) / 4;
        const size_t smem8 = ((size_t)C * (a.He + 2) * (a.We + 2) * a.max_imgs + 15) / 16 * 16 +
                             tw * a.tile_n * 4 + (size_t)a.QT * 4 * tw * 4;
        if (smem8 <= kMaxSmem) {
            if (pool) return launch_conv(conv_first_dp4a_kernel<true>, a, smem8, st, "conv_first_dp4a");
            return launch_conv(conv_first_dp4a_kernel<false>, a, smem8, st, "conv_first_dp4a");
        }
        if (pool) return launch_conv(conv_first_kernel<uint8_t, true>, a, smem, st, "conv_first");
        return launch_conv(conv_first_kernel<uint8_t, false>, a, smem, st, "conv_first");
    }
    if (pool) return launch_conv(conv_first_kernel<int32_t, true>, a, smem, st, "conv_first");
    return launch_conv(conv_first_kernel<int32_t, false>, a, smem, st, "conv_first");
}

}  // namespace bnn
