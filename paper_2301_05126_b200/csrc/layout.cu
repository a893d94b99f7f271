// layout.cu -- boundary conversions and the standalone (unfused) layer kernels.
//
// These serve the single-layer drop-in API (step_forward, maxpool_forward and
// the BinaryTensor <-> device conversions).  The model path never calls them:
// there every step / pool is fused into the producing conv or FC kernel.
//   ref bits  : reference BinaryTensor words, flat (B,C,H,W) index i at u64 word
//               i/64 bit i%64 (tensors.py:29-46)
//   NHWC bits : device layout, channel c of pixel (b,y,x) at u32 word
//               ((b*H+y)*W+x)*CW + c/32, bit c%32
#include "common.cuh"

namespace bnn {

__global__ void ref_to_nhwc_kernel(const uint64_t *__restrict__ ref, int B, int C, int H, int W, int CW,
                                   uint32_t *__restrict__ out) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    const long long n = (long long)B * H * W * CW;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int cw = (int)(i % CW);
        const long long pix = i / CW;
        const int x = (int)(pix % W);
        const int y = (int)((pix / W) % H);
        const long long b = pix / ((long long)W * H);
        uint32_t word = 0;
        for (int bit = 0; bit < 32; ++bit) {
            const int c = cw * 32 + bit;
            if (c >= C) break;
            const long long f = ((b * C + c) * H + y) * W + x;
            word |= (uint32_t)((__ldg(ref + (f >> 6)) >> (f & 63)) & 1ull) << bit;
        }
        out[i] = word;
    }
}

__global__ void nhwc_to_ref_kernel(const uint32_t *__restrict__ in, int B, int C, int H, int W, int CW,
                                   uint64_t *__restrict__ ref) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    const long long total = (long long)B * C * H * W;
    const long long nw = (total + 63) / 64;
    const long long hw = (long long)H * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nw;
         i += (long long)gridDim.x * blockDim.x) {
        uint64_t word = 0;
        for (int bit = 0; bit < 64; ++bit) {
            const long long f = i * 64 + bit;
            if (f >= total) break;
            const long long s = f % hw;
            const long long bc = f / hw;
            const int c = (int)(bc % C);
            const long long b = bc / C;
            const uint32_t v = __ldg(in + (b * hw + s) * CW + (c >> 5));
            word |= (uint64_t)((v >> (c & 31)) & 1u) << bit;
        }
        ref[i] = word;
    }
}

// ---- fast paths (H*W % 32 == 0, sizes in 32-bit range): a warp moves a 32 x 32 bit block --------------
// 32 consecutive pixels x 32 channels of one image.  In the reference layout channel c's 32 pixels are
// one aligned u32 of the flat words (plane c starts at bit (b*C + c)*H*W, a multiple of 32); in NHWC
// pixel p's 32 channels are one word.  Converting is a 32 x 32 bit transpose held one row per lane:
// five shuffle / mask rounds (Hacker's Delight transpose32 across lanes).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int k = 0, j = 16; k < 5; ++k, j >>= 1) {
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j), m = masks[k];
        x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y << j) & ~m));
    }
    return x;  // bit c of lane p = bit p of lane c's input
}

// a warp per (image, 32-pixel block), every channel word of it; consecutive warps take consecutive pixel
// blocks, so the lanes' per-plane reads (ref -> NHWC) or writes (NHWC -> ref) of neighbouring warps share lines
__global__ void ref_to_nhwc_warp_kernel(const uint32_t *__restrict__ ref32, int B, int C, int HW, int CW,
                                        uint32_t *__restrict__ out) {
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31, nsb = HW >> 5, ntask = B * nsb;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntask; t += (gridDim.x * blockDim.x) >> 5) {
        const int b = t / nsb, sb = t - b * nsb;
        uint32_t *o = out + ((size_t)b * HW + sb * 32 + lane) * CW;
        const uint32_t *src = ref32 + (size_t)b * C * nsb + sb;
        for (int cw0 = 0; cw0 < CW; cw0 += 4) {  // four channel words in flight
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = (cw0 + k) * 32 + lane;
                w[k] = (cw0 + k < CW && c < C) ? __ldg(src + (size_t)c * nsb) : 0u;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (cw0 + k < CW) o[cw0 + k] = warp_transpose32(w[k], lane);
        }
    }
}

__global__ void nhwc_to_ref_warp_kernel(const uint32_t *__restrict__ in, int B, int C, int HW, int CW,
                                        uint32_t *__restrict__ ref32) {
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31, nsb = HW >> 5, ntask = B * nsb;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntask; t += (gridDim.x * blockDim.x) >> 5) {
        const int b = t / nsb, sb = t - b * nsb;
        const uint32_t *ip = in + ((size_t)b * HW + sb * 32 + lane) * CW;
        uint32_t *dst = ref32 + (size_t)b * C * nsb + sb;
        for (int cw0 = 0; cw0 < CW; cw0 += 4) {
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) w[k] = cw0 + k < CW ? __ldg(ip + cw0 + k) : 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = (cw0 + k) * 32 + lane;
                const uint32_t tr = warp_transpose32(w[k], lane);
                if (cw0 + k < CW && c < C) dst[(size_t)c * nsb] = tr;
            }
        }
    }
}

// step -> reference flat words when S % 32 == 0: every ballot's 32 elements share one channel, which the
// warp tracks incrementally (no per-element division)
__global__ void step_ref_s32_kernel(const int32_t *__restrict__ x, int C, int S, int total,
                                    const int32_t *__restrict__ thr, const uint32_t *__restrict__ pos,
                                    uint32_t *__restrict__ ref32) {
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int nw32 = total >> 5;  // u32 words, one per ballot
    for (int wb = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; wb < nw32; wb += nwarps * 32) {
        const int e0 = wb * 32;
        int c = (e0 / S) % C, off = e0 % S;
        int t = __ldg(thr + c);
        bool ps = dir_pos(pos, c);
        uint32_t mine = 0;
        const int nr = min(32, nw32 - wb);
        int v[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = r < nr ? __ldg(x + e0 + r * 32 + lane) : 0;  // all loads in flight
#pragma unroll
        for (int r = 0; r < 32; ++r) {
            const uint32_t m = __ballot_sync(0xffffffffu, step_bit(v[r], t, ps));
            if (lane == r) mine = m;
            off += 32;
            if (off == S) {
                off = 0;
                c = c + 1 == C ? 0 : c + 1;
                t = __ldg(thr + c);
                ps = dir_pos(pos, c);
            }
        }
        if (lane < nr) ref32[wb + lane] = mine;
    }
}

// step -> NHWC bits: a thread per pixel, every channel word (reads coalesced across pixels), 32-bit indices
__global__ void step_nhwc_pix_kernel(const int32_t *__restrict__ x, int B, int C, int HW, int CW,
                                     const int32_t *__restrict__ thr, const uint32_t *__restrict__ pos,
                                     uint32_t *__restrict__ out) {
    pdl_trigger();
    pdl_wait();
    const int npix = B * HW;
    for (int pix = blockIdx.x * blockDim.x + threadIdx.x; pix < npix; pix += gridDim.x * blockDim.x) {
        const int b = pix / HW, s = pix - b * HW;
        const int32_t *xp = x + (size_t)b * C * HW + s;
        for (int cw = 0; cw < CW; ++cw) {
            uint32_t word = 0;
            const uint32_t pw = __ldg(pos + cw);
#pragma unroll 8
            for (int bit = 0; bit < 32; ++bit) {
                const int c = cw * 32 + bit;
                if (c < C) word |= step_bit(__ldg(xp + (size_t)c * HW), __ldg(thr + c), (pw >> bit) & 1u) << bit;
            }
            out[(size_t)pix * CW + cw] = word;
        }
    }
}

__global__ void maxpool_int32_kernel(const int32_t *__restrict__ x, int planes, int H, int W, int32_t *__restrict__ out) {
    pdl_trigger();
    pdl_wait();
    const int h2 = H / 2, w2 = W / 2, n = planes * h2 * w2;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int j = i % w2, t = i / w2, r = t % h2, p = t / h2;
        const int2 *s = reinterpret_cast<const int2 *>(x + ((size_t)p * H + 2 * r) * W + 2 * j);  // W even
        const int2 a = __ldg(s), b = __ldg(s + W / 2);
        out[i] = max(max(a.x, a.y), max(b.x, b.y));
    }
}

__global__ void maxpool_bits32_kernel(const uint32_t *__restrict__ x, int B, int H, int W, int CW,
                                      uint32_t *__restrict__ out) {
    pdl_trigger();
    pdl_wait();
    const int h2 = H / 2, w2 = W / 2, n = B * h2 * w2 * CW;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int cw = i % CW, r = i / CW, j = r % w2, t = r / w2, y = t % h2, b = t / h2;
        const uint32_t *s = x + (((size_t)b * H + 2 * y) * W + 2 * j) * CW + cw;
        out[i] = __ldg(s) | __ldg(s + CW) | __ldg(s + (size_t)W * CW) | __ldg(s + (size_t)W * CW + CW);
    }
}

// step to reference flat words: warp handles 32 consecutive u64 words (2048 elements)
__global__ void step_ref_kernel(const int32_t *__restrict__ x, int C, long long S, long long total,
                                const int32_t *__restrict__ thr, const uint32_t *__restrict__ pos,
                                uint64_t *__restrict__ ref) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long nwords = (total + 63) / 64;
    for (long long wb = warp * 32; wb < nwords; wb += nwarps * 32) {
        uint64_t mine = 0;
        for (int r = 0; r < 64; ++r) {
            const long long e = wb * 64 + (long long)r * 32 + lane;
            uint32_t bit = 0;
            if (e < total) {
                const int c = (int)((e / S) % C);
                bit = step_bit(__ldg(x + e), __ldg(thr + c), dir_pos(pos, c));
            }
            const uint32_t half = __ballot_sync(0xffffffffu, bit);
            if (lane == (r >> 1)) mine |= (uint64_t)half << ((r & 1) * 32);
        }
        if (wb + lane < nwords) ref[wb + lane] = mine;
    }
}

__global__ void step_nhwc_kernel(const int32_t *__restrict__ x, int B, int C, int H, int W, int CW,
                                 const int32_t *__restrict__ thr, const uint32_t *__restrict__ pos,
                                 uint32_t *__restrict__ out) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    const long long npix = (long long)B * H * W;
    const long long hw = (long long)H * W;
    const long long n = npix * CW;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long pix = i % npix;  // consecutive threads -> consecutive pixels (coalesced reads)
        const int cw = (int)(i / npix);
        const long long b = pix / hw, s = pix % hw;
        uint32_t word = 0;
        for (int bit = 0; bit < 32; ++bit) {
            const int c = cw * 32 + bit;
            if (c >= C) break;
            word |= step_bit(__ldg(x + (b * C + c) * hw + s), __ldg(thr + c), dir_pos(pos, c)) << bit;
        }
        out[pix * CW + cw] = word;
    }
}

__global__ void maxpool_int_kernel(const int32_t *__restrict__ x, long long planes, int H, int W,
                                   int32_t *__restrict__ out) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    const int h2 = H / 2, w2 = W / 2;
    const long long n = planes * h2 * w2;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(i % w2);
        const int r = (int)((i / w2) % h2);
        const long long p = i / ((long long)w2 * h2);
        const int32_t *s = x + p * H * W + (2 * r) * W + 2 * j;
        out[i] = max(max(__ldg(s), __ldg(s + 1)), max(__ldg(s + W), __ldg(s + W + 1)));
    }
}

// binary 2x2 max-pool = OR of the four channel words (layers.py:126-129)
__global__ void maxpool_bits_nhwc_kernel(const uint32_t *__restrict__ x, int B, int H, int W, int CW,
                                         uint32_t *__restrict__ out) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    const int h2 = H / 2, w2 = W / 2;
    const long long n = (long long)B * h2 * w2 * CW;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int cw = (int)(i % CW);
        long long r = i / CW;
        const int j = (int)(r % w2);
        r /= w2;
        const int y = (int)(r % h2);
        const long long b = r / h2;
        const uint32_t *s = x + ((b * H + 2 * y) * W + 2 * j) * CW + cw;
        out[i] = __ldg(s) | __ldg(s + CW) | __ldg(s + (long long)W * CW) | __ldg(s + (long long)W * CW + CW);
    }
}

__global__ void xnor_dot_kernel(const uint64_t *a, const uint64_t *am, const uint64_t *b, const uint64_t *bm,
                                int n, long long *out) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    __shared__ long long s_agree[32], s_valid[32];
    long long agree = 0, valid = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t m = am[i] & bm[i];
        agree += __popcll(~(a[i] ^ b[i]) & m);
        valid += __popcll(m);
    }
    for (int o = 16; o; o >>= 1) {
        agree += __shfl_xor_sync(0xffffffffu, agree, o);
        valid += __shfl_xor_sync(0xffffffffu, valid, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_agree[threadIdx.x >> 5] = agree;
        s_valid[threadIdx.x >> 5] = valid;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long A = 0, V = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            A += s_agree[w];
            V += s_valid[w];
        }
        out[0] = 2 * A - V;
    }
}

// NHWC bits -> NHWC FP4 +-1 (tensor-engine operand format, common.cuh): 32 channels per word
__global__ void bits_to_f4_kernel(const uint32_t *__restrict__ bits, long long nwords, uint8_t *__restrict__ out) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nwords;
         i += (long long)gridDim.x * blockDim.x)
        reinterpret_cast<uint4 *>(out)[i] = bits_to_f4(__ldg(bits + i));
}

// NHWC FP4 (+1 -> bit 1, anything else -> bit 0) -> NHWC bits
__global__ void f4_to_bits_kernel(const uint8_t *__restrict__ x, long long nwords, uint32_t *__restrict__ out) {
    pdl_trigger();
    pdl_wait();  // every global read below may depend on the previous launch
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nwords;
         i += (long long)gridDim.x * blockDim.x) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(x) + i);
        out[i] = f4_to_bits8(v.x) | (f4_to_bits8(v.y) << 8) | (f4_to_bits8(v.z) << 16) | (f4_to_bits8(v.w) << 24);
    }
}

int bits_to_f4(const uint32_t *bits, long long npix, int C, uint8_t *out, cudaStream_t st);
int f4_to_bits(const uint8_t *x, long long npix, int C, uint32_t *out, cudaStream_t st);

static unsigned grid_for(long long n, int threads = 256) {
    long long g = (n + threads - 1) / threads;
    if (g > 148LL * 32) g = 148LL * 32;
    return (unsigned)(g < 1 ? 1 : g);
}

static bool fits32(long long n) { return n < (1LL << 31) - (1LL << 20); }

int ref_to_nhwc(const uint64_t *ref, int B, int C, int H, int W, uint32_t *out, cudaStream_t st) {
    const int CW = (C + 31) / 32;
    const long long HW = (long long)H * W;
    if (HW % 32 == 0 && fits32((long long)B * HW * CW) && fits32((long long)B * C * HW / 32)) {
        launch_kernel(ref_to_nhwc_warp_kernel, dim3(grid_for((long long)B * HW)), dim3(256), 0, st,
                      reinterpret_cast<const uint32_t *>(ref), B, C, (int)HW, CW, out);
        count_launch();
        return after_launch("ref_to_nhwc");
    }
    launch_kernel(ref_to_nhwc_kernel, dim3(grid_for((long long)B * H * W * CW)), dim3(256), 0, st, ref, B, C, H, W, CW, out);
    count_launch();
    return after_launch("ref_to_nhwc");
}

int nhwc_to_ref(const uint32_t *in, int B, int C, int H, int W, uint64_t *ref, cudaStream_t st) {
    const int CW = (C + 31) / 32;
    const long long nw = ((long long)B * C * H * W + 63) / 64;
    const long long HW = (long long)H * W;
    if (HW % 32 == 0 && fits32((long long)B * HW * CW) && fits32(nw * 2)) {
        uint32_t *ref32 = reinterpret_cast<uint32_t *>(ref);
        const long long n32 = (long long)B * C * HW / 32;
        if (nw * 2 > n32) {  // the last u64's upper half lies past the data: it must read as zero bits
            const cudaError_t e = cudaMemsetAsync(ref32 + n32, 0, 4, st);
            if (e != cudaSuccess) {
                set_error("nhwc_to_ref: memset: %s", cudaGetErrorString(e));
                return (int)e;
            }
        }
        launch_kernel(nhwc_to_ref_warp_kernel, dim3(grid_for((long long)B * HW)), dim3(256), 0, st, in, B, C,
                      (int)HW, CW, ref32);
        count_launch();
        return after_launch("nhwc_to_ref");
    }
    launch_kernel(nhwc_to_ref_kernel, dim3(grid_for(nw)), dim3(256), 0, st, in, B, C, H, W, CW, ref);
    count_launch();
    return after_launch("nhwc_to_ref");
}

int step_ref(const int32_t *x, int B, int C, long long S, const int32_t *thr, const uint32_t *pos,
             uint64_t *ref, cudaStream_t st) {
    const long long total = (long long)B * C * S;
    const long long nwords = (total + 63) / 64;
    if (S % 32 == 0 && fits32(total)) {
        uint32_t *ref32 = reinterpret_cast<uint32_t *>(ref);
        if (nwords * 2 > total / 32) {  // zero upper half of the last u64
            const cudaError_t e = cudaMemsetAsync(ref32 + total / 32, 0, 4, st);
            if (e != cudaSuccess) {
                set_error("step_ref: memset: %s", cudaGetErrorString(e));
                return (int)e;
            }
        }
        launch_kernel(step_ref_s32_kernel, dim3(grid_for(total / 32)), dim3(256), 0, st, x, C, (int)S, (int)total, thr,
                      pos, ref32);
        count_launch();
        return after_launch("step_ref");
    }
    launch_kernel(step_ref_kernel, dim3(grid_for((nwords + 31) / 32 * 32)), dim3(256), 0, st, x, C, S, total, thr, pos, ref);
    count_launch();
    return after_launch("step_ref");
}

int step_nhwc(const int32_t *x, int B, int C, int H, int W, const int32_t *thr, const uint32_t *pos,
              uint32_t *out, cudaStream_t st) {
    const int CW = (C + 31) / 32;
    if (fits32((long long)B * C * H * W)) {
        launch_kernel(step_nhwc_pix_kernel, dim3(grid_for((long long)B * H * W)), dim3(256), 0, st, x, B, C, H * W, CW,
                      thr, pos, out);
        count_launch();
        return after_launch("step_nhwc");
    }
    launch_kernel(step_nhwc_kernel, dim3(grid_for((long long)B * H * W * CW)), dim3(256), 0, st, x, B, C, H, W, CW, thr, pos, out);
    count_launch();
    return after_launch("step_nhwc");
}

int maxpool_int(const int32_t *x, int B, int C, int H, int W, int32_t *out, cudaStream_t st) {
    const long long planes = (long long)B * C;
    if (fits32(planes * H * W) && (reinterpret_cast<uintptr_t>(x) & 7) == 0) {
        launch_kernel(maxpool_int32_kernel, dim3(grid_for(planes * (H / 2) * (W / 2))), dim3(256), 0, st, x, (int)planes,
                      H, W, out);
        count_launch();
        return after_launch("maxpool_int");
    }
    launch_kernel(maxpool_int_kernel, dim3(grid_for(planes * (H / 2) * (W / 2))), dim3(256), 0, st, x, planes, H, W, out);
    count_launch();
    return after_launch("maxpool_int");
}

int maxpool_bits_nhwc(const uint32_t *x, int B, int C, int H, int W, uint32_t *out, cudaStream_t st) {
    const int CW = (C + 31) / 32;
    if (fits32((long long)B * H * W * CW)) {
        launch_kernel(maxpool_bits32_kernel, dim3(grid_for((long long)B * (H / 2) * (W / 2) * CW)), dim3(256), 0, st, x,
                      B, H, W, CW, out);
        count_launch();
        return after_launch("maxpool_bits_nhwc");
    }
    launch_kernel(maxpool_bits_nhwc_kernel, dim3(grid_for((long long)B * (H / 2) * (W / 2) * CW)), dim3(256), 0, st, x, B, H, W, CW,
                                                                                                 out);
    count_launch();
    return after_launch("maxpool_bits_nhwc");
}

int xnor_dot(const uint64_t *a, const uint64_t *am, const uint64_t *b, const uint64_t *bm, int n,
             long long *out, cudaStream_t st) {
    launch_kernel(xnor_dot_kernel, dim3(1), dim3(256), 0, st, a, am, b, bm, n, out);
    count_launch();
    return after_launch("xnor_dot");
}

}  // namespace bnn

namespace bnn {
int bits_to_f4(const uint32_t *bits, long long npix, int C, uint8_t *out, cudaStream_t st) {
    const long long nw = npix * (C / 32);
    launch_kernel(bits_to_f4_kernel, dim3(grid_for(nw)), dim3(256), 0, st, bits, nw, out);
    count_launch();
    return after_launch("bits_to_f4");
}

int f4_to_bits(const uint8_t *x, long long npix, int C, uint32_t *out, cudaStream_t st) {
    const long long nw = npix * (C / 32);
    launch_kernel(f4_to_bits_kernel, dim3(grid_for(nw)), dim3(256), 0, st, x, nw, out);
    count_launch();
    return after_launch("f4_to_bits");
}
}  // namespace bnn
