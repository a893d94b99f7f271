// fc_popc.cu -- binary fully-connected layers on the integer pipe.
//
//   fc_bin        : out[b,m] = valid - 2*popc((x_b ^ w_m) & mask_b)
//                   (fc_forward, layers.py:164-175; packed twin backends.py:288-324)
//                   fused with the strict step and the 32-neuron re-pack.
//                   Two shapes: a tiled popc GEMM (batch rows x neurons, K chunks
//                   staged in shared memory) and a split-K GEMV for B <= 8.
//   fc_out_argmax : FC_INT_OUT logits + first-max argmax (layers.py:215-224).
#include "common.cuh"

namespace bnn {

struct FcArgs {
    const uint32_t *x, *mask;
    int B, L, LW;
    const uint32_t *w;  // (LW, M)
    int M, MW;
    const int32_t *thr;
    const uint32_t *pos;
    uint32_t *out;
    int32_t *sums;
    int tile_n, RT;
    int out_fmt;  // 0 = bits, 1 = FP4 +-1
};


constexpr int kFcThreads = 256;
constexpr int kKC = 32;       // K chunk (words) staged per iteration
constexpr int kXS = kKC + 4;  // padded row stride of the x tile (bank spread)

template <bool MASKED>
__global__ void __launch_bounds__(kFcThreads) fc_popc_gemm_kernel(const FcArgs a) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *s_x = smem;                       // [RT][kXS]
    uint32_t *s_m = s_x + a.RT * kXS;           // [RT][kXS] (MASKED)
    uint32_t *s_w = s_m + (MASKED ? a.RT * kXS : 0);  // [kKC][tile_n]
    const int t = threadIdx.x;
    const int cg4 = t & 3, rlo = (t >> 2) & 7, warp = t >> 5;
    const int nwt = a.tile_n >> 5;
    const int nw = warp % nwt, rb = warp / nwt;
    const int lrow = (rb * 8 + rlo) * 4;  // first of this thread's 4 rows (CTA-local)
    const long long row0 = (long long)blockIdx.x * a.RT;
    const int n_cta = blockIdx.y * a.tile_n;
    const int cgoff = nw * 32 + cg4 * 8;

    int acc[4][8];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[p][c] = 0;
    int valid[4] = {0, 0, 0, 0};

    for (int k0 = 0; k0 < a.LW; k0 += kKC) {
        for (int i = t; i < a.RT * kKC; i += kFcThreads) {
            const int j = i % kKC, r = i / kKC;
            const long long row = row0 + r;
            const bool ok = row < a.B && k0 + j < a.LW;
            s_x[r * kXS + j] = ok ? __ldg(a.x + row * a.LW + k0 + j) : 0u;
            if (MASKED) s_m[r * kXS + j] = ok ? __ldg(a.mask + row * a.LW + k0 + j) : 0u;
        }
        for (int i = t; i < kKC * a.tile_n; i += kFcThreads) {
            const int n = i % a.tile_n, j = i / a.tile_n;
            const bool ok = n_cta + n < a.M && k0 + j < a.LW;
            s_w[i] = ok ? __ldg(a.w + (long long)(k0 + j) * a.M + n_cta + n) : 0u;
        }
        __syncthreads();
#pragma unroll 2
        for (int j = 0; j < kKC; j += 4) {
            uint32_t xv[4][4], mv[4][4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const uint4 v = *reinterpret_cast<const uint4 *>(s_x + (lrow + p) * kXS + j);
                xv[p][0] = v.x; xv[p][1] = v.y; xv[p][2] = v.z; xv[p][3] = v.w;
                if (MASKED) {
                    const uint4 m = *reinterpret_cast<const uint4 *>(s_m + (lrow + p) * kXS + j);
                    mv[p][0] = m.x; mv[p][1] = m.y; mv[p][2] = m.z; mv[p][3] = m.w;
#pragma unroll
                    for (int v2 = 0; v2 < 4; ++v2) valid[p] += popc(mv[p][v2]);
                } else {
#pragma unroll
                    for (int v2 = 0; v2 < 4; ++v2) mv[p][v2] = 0xffffffffu;
                }
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint4 w0 = *reinterpret_cast<const uint4 *>(s_w + (j + v) * a.tile_n + cgoff);
                const uint4 w1 = *reinterpret_cast<const uint4 *>(s_w + (j + v) * a.tile_n + cgoff + 4);
                const uint32_t wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[p][c] += popc(xor_and(xv[p][v], wv[c], mv[p][v]));
            }
        }
        __syncthreads();
    }

    // epilogue: dot -> sums / step + pack (lane cg4 stores row p == cg4)
    uint32_t word[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int m = n_cta + cgoff + c;
        if (m >= a.M) continue;
        int th = 0;
        bool ps = true;
        if (a.out) {
            th = __ldg(a.thr + m);
            ps = dir_pos(a.pos, m);
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const long long row = row0 + lrow + p;
            const int d = (MASKED ? valid[p] : a.L) - 2 * acc[p][c];
            if (a.sums && row < a.B) a.sums[row * a.M + m] = d;
            word[p] |= step_bit(d, th, ps) << c;
        }
    }
    if (!a.out) return;
    if (a.out_fmt == 1) {
        const int m0 = n_cta + cgoff;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const long long row = row0 + lrow + p;
            if (row < a.B && m0 < a.M)
                *reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(a.out) + (row * a.M + m0) / 2) =
                    bits8_to_f4(word[p]);
        }
        return;
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        word[p] <<= cg4 * 8;
        word[p] |= __shfl_xor_sync(0xffffffffu, word[p], 1);
        word[p] |= __shfl_xor_sync(0xffffffffu, word[p], 2);
    }
    uint32_t mine = word[0];
#pragma unroll
    for (int p = 1; p < 4; ++p)
        if (cg4 == p) mine = word[p];
    const long long row = row0 + lrow + cg4;
    const int kw = (n_cta + nw * 32) >> 5;
    if (row < a.B && kw < a.MW) a.out[row * a.MW + kw] = mine;
}

// Split-K GEMV for small batches: CTA = 32 neurons (lanes) x 8 K-split warps.
template <int NR, bool MASKED>
__global__ void __launch_bounds__(256) fc_popc_gemv_kernel(const FcArgs a, int row0) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    __shared__ int s_acc[8][NR][32];
    __shared__ int s_val[8][NR];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = blockIdx.x * 32 + lane;
    const bool mok = m < a.M;
    const int per = (a.LW + 7) / 8;
    const int j0 = warp * per, j1 = min(a.LW, j0 + per);
    int acc[NR], val[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[r] = val[r] = 0;
    for (int j = j0; j < j1; ++j) {
        const uint32_t wv = mok ? __ldg(a.w + (long long)j * a.M + m) : 0u;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const int row = row0 + r;
            if (row >= a.B) continue;
            const uint32_t xv = __ldg(a.x + (long long)row * a.LW + j);
            if (MASKED) {
                const uint32_t mk = __ldg(a.mask + (long long)row * a.LW + j);
                acc[r] += popc((xv ^ wv) & mk);
                val[r] += popc(mk);
            } else {
                acc[r] += popc(xv ^ wv);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        s_acc[warp][r][lane] = acc[r];
        if (MASKED && lane == 0) s_val[warp][r] = val[r];
    }
    __syncthreads();
    if (warp >= NR) return;
    const int r = warp, row = row0 + r;
    if (row >= a.B) return;
    int tot = 0, vtot = 0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        tot += s_acc[s][r][lane];
        if (MASKED) vtot += s_val[s][r];
    }
    const int d = (MASKED ? vtot : a.L) - 2 * tot;
    if (a.sums && mok) a.sums[(long long)row * a.M + m] = d;
    if (a.out) {
        const uint32_t bit = mok ? step_bit(d, __ldg(a.thr + m), dir_pos(a.pos, m)) : 0u;
        const uint32_t word = __ballot_sync(0xffffffffu, bit);
        if (a.out_fmt == 1) {
            if (lane < 4 && blockIdx.x * 32 + lane * 8 < a.M)
                *reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(a.out) +
                                              ((long long)row * a.M + blockIdx.x * 32 + lane * 8) / 2) =
                    bits8_to_f4((word >> (8 * lane)) & 0xFFu);
        } else if (lane == 0) {
            a.out[(long long)row * a.MW + blockIdx.x] = word;
        }
    }
}

int fc_bin_popc(const uint32_t *x, const uint32_t *mask, int B, int L, int LW, const uint32_t *w, int M,
                const int32_t *thr, const uint32_t *pos, int out_fmt, void *out, int32_t *sums, int tile_n_req,
                cudaStream_t st) {
    FcArgs a{};
    a.out_fmt = out_fmt;
    a.x = x; a.mask = mask; a.B = B; a.L = L; a.LW = LW; a.w = w; a.M = M; a.MW = (M + 31) / 32;
    a.thr = thr; a.pos = pos; a.out = static_cast<uint32_t *>(out); a.sums = sums;
    const bool m = mask != nullptr;
    if (B <= 8 && tile_n_req <= 0) {
        for (int r0 = 0; r0 < B; r0 += 4) {
            dim3 grid((unsigned)ceil_div(M, 32));
            const int nr = B - r0 >= 4 ? 4 : B - r0;
#define BNN_GV(NR)                                                               \
    if (m) launch_kernel(fc_popc_gemv_kernel<NR, true>, dim3(grid), dim3(256), 0, st, a, r0); \
    else launch_kernel(fc_popc_gemv_kernel<NR, false>, dim3(grid), dim3(256), 0, st, a, r0)
            if (nr == 4) { BNN_GV(4); } else if (nr == 3) { BNN_GV(3); }
            else if (nr == 2) { BNN_GV(2); } else { BNN_GV(1); }
#undef BNN_GV
            count_launch();
            int e = after_launch("fc_popc_gemv");
            if (e) return e;
        }
        return 0;
    }
    int tn = tile_n_req == 32 || tile_n_req == 64 || tile_n_req == 128 || tile_n_req == 256 ? tile_n_req : 64;
    a.tile_n = tn;
    a.RT = 4 * 8 * (8 / (tn / 32));
    const size_t smem = (size_t)a.RT * kXS * 4 * (m ? 2 : 1) + (size_t)kKC * tn * 4;
    const void *fn = m ? reinterpret_cast<const void *>(fc_popc_gemm_kernel<true>)
                       : reinterpret_cast<const void *>(fc_popc_gemm_kernel<false>);
    int e = allow_smem(fn, smem, "fc_popc_gemm");
    if (e) return e;
    dim3 grid((unsigned)ceil_div(B, a.RT), (unsigned)ceil_div(M, tn));
    if (m) launch_kernel(fc_popc_gemm_kernel<true>, dim3(grid), dim3(kFcThreads), smem, st, a);
    else launch_kernel(fc_popc_gemm_kernel<false>, dim3(grid), dim3(kFcThreads), smem, st, a);
    count_launch();
    return after_launch("fc_popc_gemm");
}

// ---------------------------------------------------------------- logits + argmax
constexpr int kOutMax = 32;

__global__ void __launch_bounds__(256) fc_out_argmax_kernel(const uint32_t *__restrict__ x, int B, int L,
                                                           int LW, const uint32_t *__restrict__ w, int M,
                                                           int32_t *logits, int32_t *preds) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    extern __shared__ uint32_t s_w[];  // (M, LW)
    for (int i = threadIdx.x; i < M * LW; i += blockDim.x) s_w[i] = __ldg(w + i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    for (long long row = (long long)blockIdx.x * warps + (threadIdx.x >> 5); row < B;
         row += (long long)gridDim.x * warps) {
        const uint32_t *xr = x + row * LW;
        int best = 0, bestv = 0;
        for (int m0 = 0; m0 < M; m0 += kOutMax) {
            int acc[kOutMax];
#pragma unroll
            for (int m = 0; m < kOutMax; ++m) acc[m] = 0;
            for (int j = lane; j < LW; j += 32) {
                const uint32_t xv = __ldg(xr + j);
#pragma unroll
                for (int m = 0; m < kOutMax; ++m)
                    if (m0 + m < M) acc[m] += popc(xv ^ s_w[(m0 + m) * LW + j]);
            }
#pragma unroll
            for (int m = 0; m < kOutMax; ++m) {
                if (m0 + m >= M) break;
                int v = acc[m];
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                const int logit = L - 2 * v;
                if (logits && lane == m) logits[row * M + m0 + m] = logit;
                if (m0 + m == 0 || logit > bestv) {  // first max wins ties (np.argmax)
                    best = m0 + m;
                    bestv = logit;
                }
            }
        }
        if (preds && lane == 0) preds[row] = best;
    }
}

int fc_out_argmax(const uint32_t *x, int B, int L, int LW, const uint32_t *w, int M, int32_t *logits,
                  int32_t *preds, cudaStream_t st) {
    const size_t smem = (size_t)M * LW * 4;
    BNN_REQUIRE(smem <= 200 * 1024, "fc_out: weight tile %dx%d too large", M, L);
    int e = allow_smem(reinterpret_cast<const void *>(fc_out_argmax_kernel), smem, "fc_out_argmax");
    if (e) return e;
    int blocks = ceil_div(B, 8);
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    launch_kernel(fc_out_argmax_kernel, dim3(blocks), dim3(256), smem, st, x, B, L, LW, w, M, logits, preds);
    count_launch();
    return after_launch("fc_out_argmax");
}

}  // namespace bnn
