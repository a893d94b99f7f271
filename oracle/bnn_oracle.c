/*
 * bnn_oracle.c -- CPU restatement of the reference BNN numerics.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs load it (as the checker or the timed CPU baseline).
 *
 * Two independent routes, both restating /root/reference/pkg/src/bnntuner:
 *
 *  (1) "direct" -- the semantic definition of layers.py:70-175: a 3x3
 *      same-padding convolution whose out-of-image taps contribute nothing
 *      (layers.py:70-80), computed here as an int64 scalar sum over unpacked
 *      values (pixels 0..255, or +1/-1/0 for binary data with masked
 *      positions as 0).  Also the 2x2 int max-pool (layers.py:118-132), the
 *      strict per-channel step (layers.py:135-146) and the +-1 dot FC
 *      (layers.py:164-175).  Slow, obviously correct.
 *
 *  (2) "packed" -- the word-parallel route of backends.py:188-256 / :288-324:
 *      channels packed per pixel into u64 words (channel-last), taps gathered
 *      from a zero-padded word grid, dot = valid - 2*popcount((x ^ w) & mask).
 *      Fully valid inputs only (model inference never produces masked
 *      activations, backends.py:140-145).  Fast; OpenMP over images; this is
 *      the timed CPU baseline ("kind": "port").
 *
 * Parity of both routes is pinned against tests/golden/ (vectors produced by
 * running the reference itself, see tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

/* ------------------------------------------------------------------ direct */

/* out[b,k,i,j] = sum_{c,dy,dx valid} w[k,c,dy,dx] * x[b,c,i+dy-1,j+dx-1]
 * x: int32 (B,C,H,W) (masked / invalid positions already 0); w: int8 (K,C,3,3) */
EXPORT void orc_conv3_direct(const int32_t *x, int B, int C, int H, int W,
                             const int8_t *w, int K, int32_t *out, int nthreads) {
    set_threads(nthreads);
    const long hw = (long)H * W;
#pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b) {
        for (int k = 0; k < K; ++k) {
            int64_t *acc = (int64_t *)calloc((size_t)hw, sizeof(int64_t));
            for (int c = 0; c < C; ++c) {
                const int32_t *plane = x + ((long)b * C + c) * hw;
                for (int dy = 0; dy < 3; ++dy) {
                    for (int dx = 0; dx < 3; ++dx) {
                        const int64_t wt = w[(((long)k * C + c) * 3 + dy) * 3 + dx];
                        const int i0 = dy == 0 ? 1 : 0, i1 = dy == 2 ? H - 1 : H;
                        const int j0 = dx == 0 ? 1 : 0, j1 = dx == 2 ? W - 1 : W;
                        for (int i = i0; i < i1; ++i) {
                            const int32_t *src = plane + (long)(i + dy - 1) * W + (dx - 1);
                            int64_t *dst = acc + (long)i * W;
                            for (int j = j0; j < j1; ++j) dst[j] += wt * src[j];
                        }
                    }
                }
            }
            int32_t *o = out + ((long)b * K + k) * hw;
            for (long p = 0; p < hw; ++p) o[p] = (int32_t)acc[p];
            free(acc);
        }
    }
}

/* 2x2 / stride-2 integer max-pool: (N planes of H x W) -> (N planes of H/2 x W/2) */
EXPORT void orc_maxpool_int(const int32_t *x, long nplanes, int H, int W, int32_t *out) {
    const int h2 = H / 2, w2 = W / 2;
    for (long p = 0; p < nplanes; ++p) {
        const int32_t *s = x + p * H * W;
        int32_t *d = out + p * h2 * w2;
        for (int i = 0; i < h2; ++i)
            for (int j = 0; j < w2; ++j) {
                int32_t a = s[(2 * i) * W + 2 * j], b2 = s[(2 * i) * W + 2 * j + 1];
                int32_t c = s[(2 * i + 1) * W + 2 * j], e = s[(2 * i + 1) * W + 2 * j + 1];
                int32_t m = a > b2 ? a : b2;
                m = m > c ? m : c;
                d[i * w2 + j] = m > e ? m : e;
            }
    }
}

/* 2x2 OR-pool on 0/1 bytes (binary max-pool, layers.py:126-129) */
EXPORT void orc_maxpool_bits(const uint8_t *x, long nplanes, int H, int W, uint8_t *out) {
    const int h2 = H / 2, w2 = W / 2;
    for (long p = 0; p < nplanes; ++p) {
        const uint8_t *s = x + p * H * W;
        uint8_t *d = out + p * h2 * w2;
        for (int i = 0; i < h2; ++i)
            for (int j = 0; j < w2; ++j)
                d[i * w2 + j] = (uint8_t)(s[(2 * i) * W + 2 * j] | s[(2 * i) * W + 2 * j + 1] |
                                          s[(2 * i + 1) * W + 2 * j] | s[(2 * i + 1) * W + 2 * j + 1]);
    }
}

/* strict step: bit = v > T (pos) or v < T (neg); x: (B, C, S) int32 -> 0/1 bytes */
EXPORT void orc_step(const int32_t *x, int B, int C, long S, const int32_t *thr,
                     const uint8_t *pos, uint8_t *out) {
    for (int b = 0; b < B; ++b)
        for (int c = 0; c < C; ++c) {
            const int32_t t = thr[c];
            const int up = pos[c] != 0;
            const int32_t *s = x + ((long)b * C + c) * S;
            uint8_t *d = out + ((long)b * C + c) * S;
            for (long i = 0; i < S; ++i) d[i] = (uint8_t)(up ? s[i] > t : s[i] < t);
        }
}

/* +-1 dot FC: x int8 (B,L) in {+1,-1,0}; w int8 (M,L) in {+1,-1} -> int32 (B,M) */
EXPORT void orc_fc_direct(const int8_t *x, int B, int L, const int8_t *w, int M,
                          int32_t *out, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int m = 0; m < M; ++m) {
            int64_t acc = 0;
            const int8_t *xr = x + (long)b * L, *wr = w + (long)m * L;
            for (int l = 0; l < L; ++l) acc += (int64_t)xr[l] * wr[l];
            out[(long)b * M + m] = (int32_t)acc;
        }
}

/* ------------------------------------------------------------------ packed */

/* Binary conv on channel-last packed words (backends.py:188-256).
 * xw: (B, H, W, nwc) u64, channel c at word c/64 bit c%64, tail bits zero;
 * ww: (K, 9, nwc) u64 tap-major (dy, dx) filters (the reference's w_cl, model.py:125-132);
 * out: int32 (B, K, H, W).  dot = valid_bits - 2 * popcount((x ^ w) over valid taps). */
EXPORT void orc_conv3_packed(const uint64_t *xw, int B, int C, int H, int W,
                             const uint64_t *ww, int K, int32_t *out, int nthreads) {
    set_threads(nthreads);
    const int nwc = (C + 63) / 64;
#pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int i = 0; i < H; ++i)
            for (int j = 0; j < W; ++j) {
                const uint64_t *taps[9];
                int valid = 0;
                for (int t = 0; t < 9; ++t) {
                    const int y = i + t / 3 - 1, x = j + t % 3 - 1;
                    if (y >= 0 && y < H && x >= 0 && x < W) {
                        taps[t] = xw + (((long)b * H + y) * W + x) * nwc;
                        valid += C;
                    } else {
                        taps[t] = 0;
                    }
                }
                for (int k = 0; k < K; ++k) {
                    const uint64_t *wk = ww + (long)k * 9 * nwc;
                    int dis = 0;
                    for (int t = 0; t < 9; ++t) {
                        if (!taps[t]) continue;
                        const uint64_t *a = taps[t], *f = wk + t * nwc;
                        for (int q = 0; q < nwc; ++q) dis += __builtin_popcountll(a[q] ^ f[q]);
                    }
                    out[(((long)b * K + k) * H + i) * W + j] = valid - 2 * dis;
                }
            }
}

/* Binary FC on packed rows (backends.py:288-324): x (B, nw) u64, w (M, nw) u64, L bits */
EXPORT void orc_fc_packed(const uint64_t *xw, int B, int L, const uint64_t *ww, int M,
                          int32_t *out, int nthreads) {
    set_threads(nthreads);
    const int nw = (L + 63) / 64;
#pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int m = 0; m < M; ++m) {
            const uint64_t *a = xw + (long)b * nw, *f = ww + (long)m * nw;
            int dis = 0;
            for (int q = 0; q < nw; ++q) dis += __builtin_popcountll(a[q] ^ f[q]);
            out[(long)b * M + m] = L - 2 * dis;
        }
}

/* first-max argmax per row (np.argmax; layers.py:222-224) */
EXPORT void orc_argmax(const int32_t *logits, int B, int N, int32_t *pred) {
    for (int b = 0; b < B; ++b) {
        const int32_t *r = logits + (long)b * N;
        int best = 0;
        for (int n = 1; n < N; ++n)
            if (r[n] > r[best]) best = n;
        pred[b] = best;
    }
}

EXPORT int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
