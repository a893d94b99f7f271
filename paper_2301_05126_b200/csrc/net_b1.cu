// net_b1.cu -- the whole network for a small batch (the batch-1 latency path) as ONE launch.
//
// reference_infer (layers.py:215-224) = conv_int_forward (:91-101) / conv_bin_forward (:104-115)
// [+ maxpool_forward (:118-132)] + step_forward (:135-146) blocks, fc_forward FC_BIN + step, and the
// FC_INT_OUT logits + first-max argmax -- one persistent kernel, one CTA per SM, the blocks separated
// by grid-wide barriers instead of kernel boundaries.
//
// Why: at batch 1 every block is a few microseconds of latency (launch, operand fetch, epilogue,
// drain) around well under a microsecond of arithmetic; the per-kernel chain (8 launches for CIFAR,
// each a tcgen05 pipeline fill) costs ~43 us of device time.  Here a block boundary is one grid
// barrier (a release-add on an L2 counter and an acquire spin), every block's filters and step
// constants are fetched into shared memory by one bulk copy per slice at kernel entry (they are
// static, so all of them are in flight while the first blocks run), and the integer pipe does the
// arithmetic straight out of shared memory (xor + popc on NHWC bit words -- the packed route of
// backends.py:188-324).
//
// At these sizes a warp's work is a latency chain, not a throughput problem, so the layout is chosen
// for few, independent instructions per warp:
//  * each CTA owns one 32-output-channel slice kb (= one NHWC output word) and a contiguous range of
//    output positions (pixels, or 2x2 pool windows); lane = output channel;
//  * the block input is staged with a zero border ((H+2) x (W+2) pixels), so a tap needs no bounds
//    check: for conv_int a zero pixel adds nothing; for conv_bin a zero word xor the filter counts
//    popc(filter word), which the epilogue of the (few) border positions subtracts from a per-slice
//    table of per-tap filter popcounts -- exactly the reference's "out-of-range taps contribute 0"
//    (layers.py:70-80);
//  * every lane's filter words are contiguous (odd 16-B stride across lanes: conflict-free LDS.128),
//    and a pixel's channel words are contiguous, so 4 words = one LDS.128 on each side;
//  * units = (position, group of taps) spread over the CTA's 16 warps; partial sums meet in shared
//    memory (one ATOMS per pixel per unit), then one epilogue per position: the step (strict
//    threshold, POS / NEG), the 2x2 pool on thresholded bits (OR for POS, AND for NEG: max(v) > T <=>
//    any v > T; max(v) < T <=> all v < T) and the re-pack (one ballot = one output word);
//  * the FC_INT_OUT block runs on the CTA that arrives last at the barrier after the FC (no second
//    grid-wide wait), which writes the logits and predictions -- to device memory or, zero-copy,
//    straight into pinned host memory.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace bnn {

constexpr int kNetThreads = 512;
constexpr int kNetWarps = kNetThreads / 32;
constexpr int kNetSlots = 4;          // 32-channel slices a CTA keeps per block
constexpr int kNetEpiWords = 36;      // per slice after the filter words: 32 thresholds, the POS word, pad
constexpr int kNetTraceEvents = 64;

struct NetLayerK {
    int kind;             // BNN_NET_*
    int C, H, W, K, pool;
    int CW;               // conv_bin: input words per pixel; fc: input words per image (LW)
    int KB;               // output words per position, ceil(K / 32)
    int Ho, Wo, npos;     // output positions per image (pooled)
    int R;                // filter words per output channel: conv_first 1 (tap mask), conv_bin 9*CW, fc LW
    int LS;               // conv_bin / fc: words per lane in a slice (>= R, odd multiple of 4)
    int S;                // fc: warps per image
    int ng, tpg;          // conv: tap groups per position (units = positions x ng), taps (or rows) per group
    int per;              // CTAs per slice (KB <= G), else 0: CTA c owns slices c, c + G, ...
    int chunk;            // positions per CTA
    int in_words, out_words;  // per-image stride (words) of the input / output activation buffer (global)
    int in_off, out_off;      // word offsets of the input / output buffers in the activation region
    int out_pad;              // the output has a zero border (the next block is a conv_bin)
    int slice_words;      // words per packed slice (fc_out: M*LW, one slice)
    int epi_off;          // offset of the step constants in a slice
    int smem_off;         // this block's slots in shared memory
    int ptab_off;         // this block's position table (chunk entries) in shared memory
    int most;             // slots per CTA
    const uint32_t *packed;   // slice-major packed filters + step constants (bnn_net_prepare)
};

struct NetArgs {
    NetLayerK L[BNN_NET_MAX_LAYERS];
    int n, B, x_host;
    int reps;  // debug (BNN_NET_REPS): run every block's units this many times (timing experiments)
    const uint8_t *x;
    uint8_t *xstage;
    uint32_t *act;  // every block's output buffer (zero borders set by bnn_net_prepare), image-major
    int img_stride; // words per image in the activation region (all blocks' outputs of one image)
    int32_t *logits, *preds;
    unsigned *ctr;
    int act_off, red_off, bar_off;
    unsigned long long *trace;  // debug: globaltimer stamps [cta][kNetTraceEvents] (bnn_net_trace), or null
    // persistent serving (bnn_net_serve_launch): host-mapped control words {req, done, stop, status}, the
    // device word CTA 0 publishes each request on, and the idle timeout; ctl == null: one inference
    unsigned *ctl, *go;
    unsigned long long idle_ns;
};

// event 0: kernel entry, 1: filter copies issued; per block l: 2 + 3l = barrier passed, 3 + 3l = operands
// staged, 4 + 3l = units done
// fine-grained clock64 stamps of warp 0 (events 40 + 4l + k, blocks l < 6): units start, units done,
// partial sums combined, epilogues done
#define NET_CLK(l, k)                                                                                      \
    do {                                                                                                   \
        if (DBG && a.trace && threadIdx.x == 0 && (l) < 6)                                                 \
            a.trace[(size_t)blockIdx.x * kNetTraceEvents + 40 + 4 * (l) + (k)] = clock64();                \
    } while (0)
#define NET_TRACE(ev)                                                                                      \
    do {                                                                                                   \
        if (a.trace && threadIdx.x == 0 && (ev) < kNetTraceEvents)                                         \
            a.trace[(size_t)blockIdx.x * kNetTraceEvents + (ev)] = global_ns();                            \
    } while (0)

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned *p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release_gpu(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void red_release_gpu(unsigned *p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// grid-wide barrier on monotonic counters striped over kNetCtrSlots L2 lines (target = barriers so far x
// gridDim.x arrivals in total): CTA c arrives on slot c % kNetCtrSlots, so no single line takes all 148
// atomics; lanes 0..kNetCtrSlots-1 of warp 0 poll one slot each and add them up.  Bounded spin.
constexpr int kNetCtrSlots = 8, kNetCtrStride = 32;  // slots 128 B apart
__device__ __forceinline__ void net_grid_sync(unsigned *ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (lane == 0) red_release_gpu(ctr + (blockIdx.x % kNetCtrSlots) * kNetCtrStride, 1u);  // releases the CTA's writes
        __syncwarp();
        uint64_t t0 = 0;
        for (uint32_t spins = 0;; ++spins) {
            const unsigned v = lane < kNetCtrSlots ? ld_acquire_gpu(ctr + lane * kNetCtrStride) : 0u;
            if (__reduce_add_sync(0xffffffffu, v) >= target) break;
            if ((spins & 1023) == 0) {
                const uint64_t now = global_ns();
                if (t0 == 0) t0 = now;
                else if (now - t0 > 4000000000ull) __trap();
            }
        }
    }
    __syncthreads();
}

// number of in-image rows of a 3x3 window centred at y (same padding)
__device__ __forceinline__ int span3(int y, int H) { return min(y + 1, H - 1) - max(y - 1, 0) + 1; }

__device__ __forceinline__ int popc4(uint4 a, uint4 w) {
    return __popc(a.x ^ w.x) + __popc(a.y ^ w.y) + __popc(a.z ^ w.z) + __popc(a.w ^ w.w);
}

// conv_bin taps [t0, t1) of one position for a compile-time channel-word count CW and pixel count NQ
// (1, or 4 for a 2x2 pool window): all of a tap's filter and activation words are loaded first
template <int CW, int NQ>
__device__ __forceinline__ void conv_taps(const uint32_t *ap, const uint32_t *wl, int t0, int t1, int y0, int x0, int Wp,
                                          int (&acc)[4]) {
    for (int t = t0; t < t1; ++t) {
        const int ty = t / 3, tx = t - 3 * ty;
        const uint32_t *wt = wl + t * CW;
        const uint32_t *aq0 = ap + ((y0 + ty) * Wp + x0 + tx) * CW;
        if constexpr (CW % 4 == 0) {
            uint4 w[CW / 4], av[NQ][CW / 4];
#pragma unroll
            for (int i = 0; i < CW / 4; ++i) w[i] = *reinterpret_cast<const uint4 *>(wt + 4 * i);
#pragma unroll
            for (int q = 0; q < NQ; ++q)
#pragma unroll
                for (int i = 0; i < CW / 4; ++i)
                    av[q][i] = *reinterpret_cast<const uint4 *>(aq0 + ((q >> 1) * Wp + (q & 1)) * CW + 4 * i);
#pragma unroll
            for (int q = 0; q < NQ; ++q)
#pragma unroll
                for (int i = 0; i < CW / 4; ++i) acc[q] += popc4(av[q][i], w[i]);
        } else {
            uint32_t w[CW], av[NQ][CW];
#pragma unroll
            for (int i = 0; i < CW; ++i) w[i] = wt[i];
#pragma unroll
            for (int q = 0; q < NQ; ++q)
#pragma unroll
                for (int i = 0; i < CW; ++i) av[q][i] = aq0[((q >> 1) * Wp + (q & 1)) * CW + i];
#pragma unroll
            for (int q = 0; q < NQ; ++q)
#pragma unroll
                for (int i = 0; i < CW; ++i) acc[q] += __popc(av[q][i] ^ w[i]);
        }
    }
}

// step + optional 2x2 pool on thresholded bits + ballot re-pack; lane 0 stores the output word
__device__ __forceinline__ void net_epilogue(const int (&v)[4], int nq, int k, int K, const uint32_t *epi, int lane,
                                             uint32_t *dst) {
    bool fire = false;
    if (k < K) {
        const int t = static_cast<int>(epi[lane]);
        const bool pos = (epi[32] >> lane) & 1u;
        bool any = false, all = true;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < nq) {
                const bool f = pos ? v[q] > t : v[q] < t;
                any |= f;
                all &= f;
            }
        fire = pos ? any : all;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, fire);
    if (lane == 0) *dst = word;
}

// a block's input (every image's in_words at stride img_stride in the activation region) -> shared memory
__device__ __forceinline__ void net_stage(uint32_t *dst, const uint32_t *src, int B, int in_words, int img_stride) {
    const int n4 = in_words / 4;  // in_words is a multiple of 4
    for (int b = 0; b < B; ++b)
        for (int i = threadIdx.x; i < n4; i += kNetThreads)
            reinterpret_cast<uint4 *>(dst + (size_t)b * in_words)[i] =
                __ldcg(reinterpret_cast<const uint4 *>(src + (size_t)b * img_stride) + i);
}

// the conv epilogue of one position: pre-activations from the tap sums (conv_bin: valid taps x C -
// 2 popc, the zero border's popc(filter) taken back at border pixels), then step / pool / re-pack into
// the output word, written into the interior of a zero-bordered buffer when the next block is a conv
__device__ __forceinline__ void net_conv_epilogue(const NetLayerK &Ly, int (&acc)[4], int nq, int y0, int x0, int oy,
                                                  int ox, int kb, int lane, const uint32_t *epi, uint32_t *out) {
    const int H = Ly.H, W = Ly.W;
    if (Ly.kind == BNN_NET_CONV_BIN) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int y = y0 + (q >> 1), x = x0 + (q & 1);
            if (q < nq && (y == 0 || x == 0 || y >= H - 1 || x >= W - 1)) {
                const uint32_t *wpop = epi + kNetEpiWords;
#pragma unroll
                for (int t = 0; t < 9; ++t) {
                    const int iy = y + t / 3 - 1, ix = x + t % 3 - 1;
                    if (iy < 0 || iy >= H || ix < 0 || ix >= W) acc[q] -= (int)wpop[t * 32 + lane];
                }
            }
            acc[q] = span3(y, H) * span3(x, W) * Ly.C - 2 * acc[q];
        }
    }
    const int pad = Ly.out_pad, Wq = Ly.Wo + 2 * pad;
    const size_t o = ((size_t)(oy + pad) * Wq + ox + pad) * Ly.KB + kb;
    net_epilogue(acc, nq, kb * 32 + lane, Ly.K, epi, lane, out + o);
}

// the CTA's slices of block L: first slice, stride, count (shared by the kernel and the host planner)
__host__ __device__ __forceinline__ void cta_slices(const NetLayerK &L, int c, int G, int &first, int &step, int &cnt) {
    if (L.per > 0) {
        first = c / L.per;
        step = L.KB;
        cnt = first < L.KB ? 1 : 0;
    } else {
        first = c;
        step = G;
        cnt = c < L.KB ? (L.KB - c + G - 1) / G : 0;
    }
}

// the CTA's positions [p0, p1) of block L
__host__ __device__ __forceinline__ void cta_positions(const NetLayerK &L, int c, int NP, int &p0, int &p1) {
    p0 = 0;
    p1 = NP;
    if (L.per > 0) {
        p0 = min(NP, (c % L.per) * L.chunk);
        p1 = min(NP, p0 + L.chunk);
    }
}

template <int DBG>
__global__ void __launch_bounds__(kNetThreads, 1) net_b1_kernel(const __grid_constant__ NetArgs args) {
    // the launch table in shared memory: dynamically indexed kernel parameters are constant-cache loads
    __shared__ __align__(16) NetArgs a;
    for (int i = threadIdx.x; i < (int)(sizeof(NetArgs) / 4); i += kNetThreads)
        reinterpret_cast<uint32_t *>(&a)[i] = reinterpret_cast<const uint32_t *>(&args)[i];
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t *wbar = reinterpret_cast<uint64_t *>(sm);  // one per block
    int *s_flag = reinterpret_cast<int *>(wbar + BNN_NET_MAX_LAYERS);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int l = 0; l < BNN_NET_MAX_LAYERS; ++l) mbar_init(&wbar[l], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint8_t *s_stage = sm + a.act_off;
    uint32_t *s_act = reinterpret_cast<uint32_t *>(s_stage);
    int *s_red = reinterpret_cast<int *>(sm + a.red_off);
    const int G = gridDim.x, B = a.B, img_stride = a.img_stride;
    uint32_t *const act = a.act;
    if (DBG) NET_TRACE(0);

    // ---- prologue: this CTA's slices of every block -> shared memory (one bulk copy per slice), and
    //      the CTA's output positions of every conv block as (y0, x0, image) -----------------------------
    if (tid < a.n * kNetSlots) {
        const int l = tid / kNetSlots, s = tid - l * kNetSlots;
        const NetLayerK &Ly = a.L[l];
        int first, step, cnt;
        if (Ly.kind == BNN_NET_FC_OUT) {
            first = 0, step = 1, cnt = 1;
        } else {
            cta_slices(Ly, blockIdx.x, G, first, step, cnt);
        }
        const uint32_t bytes = (uint32_t)Ly.slice_words * 4;
        if (s == 0) mbar_expect_tx(&wbar[l], cnt * bytes);
        if (s < cnt)
            bulk_load(sm + Ly.smem_off + s * bytes, Ly.packed + (size_t)(first + s * step) * Ly.slice_words, bytes,
                      &wbar[l]);
    }
    for (int l = 0; l < a.n; ++l) {
        const NetLayerK &Ly = a.L[l];
        if (Ly.kind != BNN_NET_CONV_FIRST && Ly.kind != BNN_NET_CONV_BIN) continue;
        int p0, p1;
        cta_positions(Ly, blockIdx.x, B * Ly.npos, p0, p1);
        uint32_t *ptab = reinterpret_cast<uint32_t *>(sm + Ly.ptab_off);
        for (int pi = tid; pi < p1 - p0; pi += kNetThreads) {
            const int pg = p0 + pi, b = pg / Ly.npos, p = pg - b * Ly.npos, oy = p / Ly.Wo, ox = p - oy * Ly.Wo;
            ptab[pi] = (uint32_t)oy | ((uint32_t)ox << 8) | ((uint32_t)b << 16);
        }
    }
    if (DBG) NET_TRACE(1);

    for (unsigned req = 1;; ++req) {
    if (a.ctl) {
        // serving: CTA 0 waits for the host's doorbell (or stop / idle timeout), copies the request's images
        // from pinned host memory into the device staging buffer and publishes the request -- one PCIe pass
        // by one CTA and no grid barrier before the first block
        if (blockIdx.x == 0) {
            if (tid == 0) {
                unsigned pub = req;
                const uint64_t t0 = global_ns();
                for (uint32_t spins = 0;; ++spins) {
                    if (ld_acquire_sys(a.ctl + BNN_NET_CTL_REQ) >= req) break;
                    if (*reinterpret_cast<volatile unsigned *>(a.ctl + BNN_NET_CTL_STOP)) {
                        pub = 0xFFFFFFFFu;
                        break;
                    }
                    if ((spins & 255) == 0 && global_ns() - t0 > a.idle_ns) {
                        *reinterpret_cast<volatile unsigned *>(a.ctl + BNN_NET_CTL_STATUS) = 1u;  // expired: the server stopped itself
                        pub = 0xFFFFFFFFu;
                        break;
                    }
                }
                s_flag[2] = (int)pub;
            }
            __syncthreads();
            if ((unsigned)s_flag[2] != 0xFFFFFFFFu) {
                const int nbytes = B * a.L[0].C * a.L[0].H * a.L[0].W;
                for (int i = tid; i < (nbytes >> 4); i += kNetThreads)
                    reinterpret_cast<uint4 *>(a.xstage)[i] = __ldcv(reinterpret_cast<const uint4 *>(a.x) + i);
                for (int i = ((nbytes >> 4) << 4) + tid; i < nbytes; i += kNetThreads) a.xstage[i] = __ldcv(a.x + i);
            }
            __syncthreads();
            // `go` is device memory read only by this grid: gpu scope (the host's images reached this CTA
            // through its system-scope acquire of the doorbell; the staged copy travels with this release)
            if (tid == 0) st_release_gpu(a.go, (unsigned)s_flag[2]);
        }
        if (tid == 0) {
            unsigned g;
            while ((g = ld_acquire_gpu(a.go)) < req) {
            }
            s_flag[1] = g == 0xFFFFFFFFu;
        }
        __syncthreads();
        if (s_flag[1]) return;
    }
    unsigned nbar = 0;
    const uint8_t *xin = a.x;
    if (a.x_host) {  // zero-copy input: one coalesced pass over PCIe into device memory, then a barrier
        if (!a.ctl) {  // (serving: CTA 0 staged the images before publishing the request)
            const long long nbytes = (long long)B * a.L[0].C * a.L[0].H * a.L[0].W;
            const long long n16 = nbytes >> 4;
            const long long gt = (long long)blockIdx.x * kNetThreads + tid, gs = (long long)G * kNetThreads;
            for (long long i = gt; i < n16; i += gs)
                reinterpret_cast<uint4 *>(a.xstage)[i] = reinterpret_cast<const uint4 *>(a.x)[i];
            for (long long i = (n16 << 4) + gt; i < nbytes; i += gs) a.xstage[i] = a.x[i];
            net_grid_sync(a.ctr, (++nbar) * G);
        }
        xin = a.xstage;
    }

    for (int l = 0; l < a.n; ++l) {
        // by value: the fields live in registers (through a reference into shared memory every use would be
        // an LDS the compiler must repeat after each shared-memory store or atomic)
        const NetLayerK Ly = a.L[l];
        const uint32_t *slots = reinterpret_cast<const uint32_t *>(sm + Ly.smem_off);
        const uint32_t *src = act + Ly.in_off;
        if (Ly.kind == BNN_NET_FC_OUT) {
            // ---- FC_INT_OUT + argmax on the CTA that arrives last after the previous block ------
            __syncthreads();
            if (tid == 0) {  // one acq_rel atomic: releases this CTA's FC outputs, acquires everyone's if last
                const unsigned old = atom_add_acq_rel_gpu(a.ctr + kNetCtrSlots * kNetCtrStride, 1u);  // `done` counter
                s_flag[0] = old == (unsigned)G - 1;
            }
            __syncthreads();
            if (!s_flag[0]) break;  // not the last arriver: done with this request
            if (DBG) NET_TRACE(2 + 3 * l);
            net_stage(s_act, src, B, Ly.in_words, img_stride);
            mbar_wait(&wbar[l], 0);
            __syncthreads();
            int *s_logit = s_red;
            const int R = Ly.R;
            for (int m = warp; m < Ly.K; m += kNetWarps)
                for (int b = 0; b < B; ++b) {
                    int acc = 0;
                    for (int r = lane; r < R; r += 32) acc += __popc(s_act[b * Ly.in_words + r] ^ slots[m * R + r]);
#pragma unroll
                    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                    if (lane == 0) s_logit[b * Ly.K + m] = Ly.C - 2 * acc;
                }
            __syncthreads();
            if (a.logits)
                for (int i = tid; i < B * Ly.K; i += kNetThreads) a.logits[i] = s_logit[i];
            if (tid < B && a.preds) {  // first maximum (np.argmax, layers.py:223)
                int best = 0;
                for (int m = 1; m < Ly.K; ++m)
                    if (s_logit[tid * Ly.K + m] > s_logit[tid * Ly.K + best]) best = m;
                a.preds[tid] = best;
            }
            __syncthreads();
            if (DBG) NET_TRACE(4 + 3 * l);
            if (tid == 0) {
                // every other CTA has left this request: reset the barrier counter for the next one, then
                // (serving) ring the host's completion word.  Its system-scope release orders, cumulatively
                // through the barrier above, this CTA's logits / predictions and the resets before it; the
                // next request reaches the other CTAs only through host acquire -> doorbell -> CTA 0 -> `go`
                // (release / acquire all the way), so they see the reset counters.  One inference: the
                // kernel boundary orders everything.
                for (int k = 0; k <= kNetCtrSlots; ++k)  // every barrier slot and the `done` counter
                    reinterpret_cast<volatile unsigned *>(a.ctr)[k * kNetCtrStride] = 0;
                if (a.ctl) st_release_sys(a.ctl + BNN_NET_CTL_DONE, req);
            }
            break;
        }
        if (l > 0) net_grid_sync(a.ctr, (++nbar) * G);
        if (DBG) NET_TRACE(2 + 3 * l);
        uint32_t *out = act + Ly.out_off;
        const int nq = Ly.pool ? 4 : 1, sh = Ly.pool ? 1 : 0;
        const int NP = B * Ly.npos, H = Ly.H, W = Ly.W, Wp = W + 2, CW = Ly.CW;
        int first, step, cnt, p0, p1;
        cta_slices(Ly, blockIdx.x, G, first, step, cnt);
        cta_positions(Ly, blockIdx.x, NP, p0, p1);
        const int np = p1 - p0, ng = Ly.ng;
        // ---- stage this block's input in shared memory: a contiguous copy (a conv_bin input arrives
        //      with its zero border: the producer wrote only the interior of a zeroed buffer) ------------
        if (Ly.kind == BNN_NET_CONV_FIRST) {
            const int nbytes = B * Ly.C * H * W;
            if ((nbytes & 15) == 0) {
                for (int i = tid; i < nbytes / 16; i += kNetThreads)
                    reinterpret_cast<uint4 *>(s_stage)[i] = a.x_host ? __ldcg(reinterpret_cast<const uint4 *>(xin) + i)
                                                                     : __ldg(reinterpret_cast<const uint4 *>(xin) + i);
            } else {
                for (int i = tid; i < nbytes; i += kNetThreads) s_stage[i] = a.x_host ? __ldcg(xin + i) : __ldg(xin + i);
            }
        } else {
            net_stage(s_act, src, B, Ly.in_words, img_stride);
        }
        if (ng > 1)
            for (int i = tid; i < cnt * np * 4 * 32; i += kNetThreads) s_red[i] = 0;
        mbar_wait(&wbar[l], 0);
        __syncthreads();
        if (DBG) NET_TRACE(3 + 3 * l);
        const int R = Ly.R;
        for (int rep = 0; rep < (DBG ? a.reps : 1); ++rep)
        for (int si = 0; si < cnt; ++si) {
            const int kb = first + si * step;
            const uint32_t *slot = slots + si * Ly.slice_words;
            const uint32_t *epi = slot + Ly.epi_off;
            if (Ly.kind == BNN_NET_FC_BIN) {
                // ---- fc_bin + step: S warps per image split the LW words (4-word groups); combine in smem ---
                const int S = Ly.S, gpc = kNetWarps / S, grp = warp / S, sub = warp % S;
                const int rounds = (np + gpc - 1) / gpc;  // uniform across the CTA
                const int ng4 = (R + 3) / 4;
                for (int round = 0; round < rounds; ++round) {
                    const int pg = p0 + grp + round * gpc;
                    const bool active = pg < p1;
                    int acc = 0;
                    if (active) {
                        const uint32_t *ap = s_act + (size_t)pg * Ly.in_words;
                        const uint32_t *wl = slot + lane * Ly.LS;
                        const int r1 = min(R, 4 * ((sub + 1) * ng4 / S));
                        int r = 4 * (sub * ng4 / S), a0 = 0, a1 = 0;
                        for (; r + 8 <= r1; r += 8) {
                            a0 += popc4(*reinterpret_cast<const uint4 *>(ap + r), *reinterpret_cast<const uint4 *>(wl + r));
                            a1 += popc4(*reinterpret_cast<const uint4 *>(ap + r + 4), *reinterpret_cast<const uint4 *>(wl + r + 4));
                        }
                        for (; r < r1; ++r) a0 += __popc(ap[r] ^ wl[r]);
                        acc = a0 + a1;
                    }
                    if (S > 1) {
                        s_red[warp * 32 + lane] = acc;
                        __syncthreads();
                        if (sub == 0 && active)
                            for (int j = 1; j < S; ++j) acc += s_red[(warp + j) * 32 + lane];
                    }
                    if (sub == 0 && active) {
                        const int v[4] = {Ly.C - 2 * acc, 0, 0, 0};  // C = L (tail bits are 0 on both sides)
                        net_epilogue(v, 1, kb * 32 + lane, Ly.K, epi, lane, out + (size_t)pg * img_stride + kb);
                    }
                    if (S > 1) __syncthreads();  // s_red is reused by the next round
                }
                continue;
            }
            // ---- conv: units = (position, tap group) over the warps; with one group per position the
            //      warp finishes the position itself, else partial sums meet in s_acc -------------------------
            const uint32_t *ptab = reinterpret_cast<const uint32_t *>(sm + Ly.ptab_off);
            int *s_acc = s_red + si * np * 4 * 32;
            const int tpg = Ly.tpg;
            NET_CLK(l, 0);
            for (int u = warp; u < np * ng; u += kNetWarps) {
                const int pi = ng == 1 ? u : (ng == 3 ? u / 3 : (ng == 9 ? u / 9 : u / ng)), g = u - pi * ng;
                const uint32_t e = ptab[pi];
                const int oy = e & 0xff, ox = (e >> 8) & 0xff, b = e >> 16;
                const int y0 = oy << sh, x0 = ox << sh;
                int acc[4] = {0, 0, 0, 0};
                if (Ly.kind == BNN_NET_CONV_FIRST) {
                    // u8 pixels x +-1 filters; a group = one channel's filter row (or all 9*C taps when ng == 1)
                    const int rows = ng == 1 ? 3 * Ly.C : 1, r0 = ng == 1 ? 0 : g;
                    const uint32_t wm = slot[lane];
                    // straight-line rows (clamped addresses, zero by select): the loads of several rows issue
                    // back to back instead of one bounds-checked row at a time
#pragma unroll 3
                    for (int rr = r0; rr < r0 + rows; ++rr) {
                        const int c = rr / 3, dy = rr - 3 * c;
                        const uint32_t bits = wm >> (rr * 3);  // bit c*9 + dy*3 + dx
                        const uint8_t *plane = s_stage + ((size_t)b * Ly.C + c) * H * W;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if (q >= nq) continue;
                            const int y = y0 + (q >> 1) + dy - 1, x = x0 + (q & 1) - 1;
                            const bool yok = y >= 0 && y < H;
                            const uint8_t *r = plane + min(max(y, 0), H - 1) * W;
                            const int pl = r[max(x, 0)], pc = r[x + 1], pr = r[min(x + 2, W - 1)];
                            const int v = ((bits & 1u) ? pl : -pl) * (x >= 0) + ((bits & 2u) ? pc : -pc) +
                                          ((bits & 4u) ? pr : -pr) * (x + 2 < W);
                            acc[q] += yok ? v : 0;
                        }
                    }
                } else {
                    const uint32_t *ap = s_act + (size_t)b * Ly.in_words;  // padded image, (H+2) x (W+2) pixels
                    const uint32_t *wl = slot + lane * Ly.LS;
                    const int t0 = g * tpg, t1 = min(9, (g + 1) * tpg);
                    // fully unrolled over the channel words and pixels of a tap for the usual widths: every
                    // load of the tap is issued before its xor / popc (the generic loop serialises them)
                    if (CW == 2) {
                        if (nq == 4) conv_taps<2, 4>(ap, wl, t0, t1, y0, x0, Wp, acc);
                        else conv_taps<2, 1>(ap, wl, t0, t1, y0, x0, Wp, acc);
                    } else if (CW == 8) {
                        if (nq == 4) conv_taps<8, 4>(ap, wl, t0, t1, y0, x0, Wp, acc);
                        else conv_taps<8, 1>(ap, wl, t0, t1, y0, x0, Wp, acc);
                    } else if (CW == 16) {
                        if (nq == 4) conv_taps<16, 4>(ap, wl, t0, t1, y0, x0, Wp, acc);
                        else conv_taps<16, 1>(ap, wl, t0, t1, y0, x0, Wp, acc);
                    } else {
                        for (int t = t0; t < t1; ++t) {
                            const int ty = t / 3, tx = t - 3 * ty;
                            const uint32_t *wt = wl + t * CW;
                            const uint32_t *aq0 = ap + ((y0 + ty) * Wp + x0 + tx) * CW;
                            for (int i = 0; i < CW; ++i) {
                                const uint32_t w1 = wt[i];
#pragma unroll
                                for (int q = 0; q < 4; ++q)
                                    if (q < nq) acc[q] += __popc(aq0[((q >> 1) * Wp + (q & 1)) * CW + i] ^ w1);
                            }
                        }
                    }
                }
                if (ng == 1) {
                    net_conv_epilogue(Ly, acc, nq, y0, x0, oy, ox, kb, lane, epi, out + (size_t)b * img_stride);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (q < nq) atomicAdd(&s_acc[(pi * 4 + q) * 32 + lane], acc[q]);
                }
            }
            NET_CLK(l, 1);
            if (ng > 1) {
                __syncthreads();
                NET_CLK(l, 2);
                for (int pi = warp; pi < np; pi += kNetWarps) {
                    const uint32_t e = ptab[pi];
                    const int oy = e & 0xff, ox = (e >> 8) & 0xff, b = e >> 16;
                    int acc[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[q] = s_acc[(pi * 4 + q) * 32 + lane];
                    net_conv_epilogue(Ly, acc, nq, oy << sh, ox << sh, oy, ox, kb, lane, epi, out + (size_t)b * img_stride);
                }
            }
            NET_CLK(l, 3);
        }
        if (DBG) NET_TRACE(4 + 3 * l);
    }
    if (!a.ctl) return;
    }
}

// ---------------------------------------------------------------- filter packing (bnn_net_prepare)
// slice kb: conv_first: 32 tap masks (bit c*9 + t) + step constants; conv_bin / fc_bin: the 32 lanes'
// filter words, lane-major with LS words per lane, + step constants (32 thresholds, the POS word, 3
// pad) [+ conv_bin: per-tap filter popcounts, wpop[t*32 + lane]]; fc_out: its (M, LW) filters as they are.
__global__ void net_pack_kernel(int kind, int C, int K, int R, int LS, int CW, int KB, int slice_words, int epi_off,
                                const void *w, const int32_t *thr, const uint32_t *pos, uint32_t *packed) {
    const long long n = kind == BNN_NET_FC_OUT ? (long long)slice_words : (long long)KB * slice_words;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        if (kind == BNN_NET_FC_OUT) {
            v = i < (long long)K * R ? static_cast<const uint32_t *>(w)[i] : 0u;
        } else {
            const int kb = (int)(i / slice_words), o = (int)(i - (long long)kb * slice_words);
            if (o < epi_off) {
                if (kind == BNN_NET_CONV_FIRST) {  // int8 +-1 (K, 9*C) -> tap mask, bit c*9 + t
                    const int k = kb * 32 + o;
                    if (k < K) {
                        const int8_t *w8 = static_cast<const int8_t *>(w);
                        for (int j = 0; j < 9 * C; ++j) v |= (uint32_t)(w8[(size_t)k * 9 * C + j] > 0) << j;
                    }
                } else {  // u32 (R, K) (bnn_conv_bin / bnn_fc_bin layouts) -> lane-major
                    const int ln = o / LS, r = o - ln * LS, k = kb * 32 + ln;
                    if (k < K && r < R) v = static_cast<const uint32_t *>(w)[(size_t)r * K + k];
                }
            } else if (o < epi_off + 32) {
                const int k = kb * 32 + (o - epi_off);
                v = k < K ? (uint32_t)thr[k] : 0u;
            } else if (o == epi_off + 32) {
                v = pos[kb];
            } else if (o >= epi_off + kNetEpiWords) {  // conv_bin: per-tap filter popcount of each lane
                const int j = o - epi_off - kNetEpiWords, t = j / 32, k = kb * 32 + (j & 31);
                if (k < K)
                    for (int cw = 0; cw < CW; ++cw)
                        v += __popc(static_cast<const uint32_t *>(w)[(size_t)(t * CW + cw) * K + k]);
            }
        }
        packed[i] = v;
    }
}

// ---------------------------------------------------------------- host side

struct NetPlan {
    NetArgs a;
    size_t smem = 0;
    size_t ws_bytes = 0;
    size_t packed_off[BNN_NET_MAX_LAYERS] = {0};
    size_t ctr_off = 0, xstage_off = 0, act_off = 0, act_bytes = 0;
};

static unsigned long long *g_net_trace = nullptr;

void net_set_trace(unsigned long long *buf) { g_net_trace = buf; }

static int net_sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

static int round4(int v) { return (v + 3) / 4 * 4; }
static size_t up128(size_t v) { return (v + 127) / 128 * 128; }

// validate the block list and derive the kernel's per-block parameters for batch B on G CTAs
static int net_plan(const bnn_net_layer *layers, int n, int B, int G, NetPlan &P) {
    BNN_REQUIRE(layers && n >= 2 && n <= BNN_NET_MAX_LAYERS, "net: 2..%d blocks required (got %d)",
                BNN_NET_MAX_LAYERS, n);
    BNN_REQUIRE(B >= 1 && B < 256, "net: batch must be 1..255");
    BNN_REQUIRE(G >= 1, "net: grid must be >= 1");
    BNN_REQUIRE(layers[0].kind == BNN_NET_CONV_FIRST, "net: the first block must be BNN_NET_CONV_FIRST");
    BNN_REQUIRE(layers[n - 1].kind == BNN_NET_FC_OUT, "net: the last block must be BNN_NET_FC_OUT");
    std::memset(&P.a, 0, sizeof(P.a));
    NetArgs &a = P.a;
    a.n = n;
    a.B = B;
    int prev_c = 0, prev_h = 0, prev_w = 0;
    size_t packed = 0, red_words = (size_t)kNetWarps * 32, stage_bytes = 16, ptab_words = 0, act_words = 0;
    for (int l = 0; l < n; ++l) {
        const bnn_net_layer &s = layers[l];
        NetLayerK &L = a.L[l];
        L.kind = s.kind;
        L.C = s.C;
        L.H = s.H;
        L.W = s.W;
        L.K = s.K;
        L.pool = s.pool;
        const bool conv = s.kind == BNN_NET_CONV_FIRST || s.kind == BNN_NET_CONV_BIN;
        BNN_REQUIRE(conv || s.kind == BNN_NET_FC_BIN || s.kind == BNN_NET_FC_OUT, "net: block %d: unknown kind %d", l,
                    s.kind);
        BNN_REQUIRE(s.K >= 1 && s.C >= 1, "net: block %d: empty shape", l);
        if (conv) {
            BNN_REQUIRE(s.H >= 1 && s.W >= 1 && s.H <= 254 && s.W <= 254, "net: block %d: image of %dx%d", l, s.H, s.W);
            BNN_REQUIRE(!s.pool || ((s.H | s.W) & 1) == 0, "net: block %d: pooling needs even H, W", l);
            L.Ho = s.pool ? s.H / 2 : s.H;
            L.Wo = s.pool ? s.W / 2 : s.W;
            L.npos = L.Ho * L.Wo;
        } else {
            BNN_REQUIRE(!s.pool, "net: block %d: an FC block cannot pool", l);
            L.Ho = L.Wo = L.npos = 1;
        }
        L.KB = (s.K + 31) / 32;
        if (s.kind == BNN_NET_CONV_FIRST) {
            BNN_REQUIRE(l == 0, "net: BNN_NET_CONV_FIRST must be the first block");
            BNN_REQUIRE(s.C <= 3, "net: conv_first supports C <= 3 (9*C filter bits in one word)");
            L.R = 1;
            L.epi_off = 32;
            L.slice_words = 32 + kNetEpiWords;
            stage_bytes = std::max(stage_bytes, (size_t)B * s.C * s.H * s.W);
        } else if (s.kind == BNN_NET_CONV_BIN) {
            BNN_REQUIRE(prev_c == s.C && prev_h == s.H && prev_w == s.W,
                        "net: block %d: input %dx%dx%d does not follow the previous block", l, s.C, s.H, s.W);
            L.CW = (s.C + 31) / 32;
            L.R = 9 * L.CW;
            L.LS = 4 * (((L.R + 3) / 4) | 1);  // odd number of 16-B groups per lane: conflict-free LDS.128
            L.epi_off = 32 * L.LS;
            L.slice_words = L.epi_off + kNetEpiWords + 9 * 32;
        } else {
            const int LW = (s.C + 31) / 32;
            const int have = prev_h * prev_w * ((prev_c + 31) / 32);  // flattened NHWC words (an FC input: H = W = 1)
            BNN_REQUIRE(have == LW, "net: block %d: L = %d bits (%d words) does not match the previous block's %d words",
                        l, s.C, LW, have);
            L.CW = L.R = LW;
            L.LS = 4 * (((L.R + 3) / 4) | 1);
            L.epi_off = 32 * L.LS;
            L.slice_words = s.kind == BNN_NET_FC_OUT ? round4(s.K * L.R) : L.epi_off + kNetEpiWords;
        }
        if (l > 0) {
            const NetLayerK &Pv = a.L[l - 1];
            L.in_words = Pv.out_words;
            L.in_off = Pv.out_off;
            stage_bytes = std::max(stage_bytes, (size_t)B * L.in_words * 4);
        }
        if (s.kind != BNN_NET_FC_OUT) {
            // this block's output buffer; a conv_bin consumer reads it with a zero border of one pixel
            L.out_pad = (l + 1 < n && layers[l + 1].kind == BNN_NET_CONV_BIN) ? 1 : 0;
            L.out_words = round4((L.Ho + 2 * L.out_pad) * (L.Wo + 2 * L.out_pad) * L.KB);
            L.out_off = (int)act_words;
            act_words += (size_t)L.out_words;
            prev_c = s.K;
            prev_h = L.Ho;
            prev_w = L.Wo;
            // CTAs per slice and positions per CTA
            const int NP = B * L.npos;
            if (L.KB <= G) {
                L.per = std::min(G / L.KB, NP);
                L.chunk = (NP + L.per - 1) / L.per;
                L.per = (NP + L.chunk - 1) / L.chunk;  // CTAs actually given positions
            } else {
                L.per = 0;
                L.chunk = NP;
            }
            L.S = 1;
            if (s.kind == BNN_NET_FC_BIN)
                for (int S = kNetWarps; S > 1; S >>= 1)
                    if ((kNetWarps / S) >= L.chunk && S <= (L.R + 3) / 4) {
                        L.S = S;
                        break;
                    }
            if (s.kind == BNN_NET_CONV_FIRST) {
                // a unit = a whole position (all 3*C filter rows): per-row units with partial sums meeting in
                // shared memory were slower even with fewer positions than warps (CIFAR net kernel 41.0 ->
                // 39.5 us); the per-row path (ng = 3*C) stays in the kernel for other plans
                L.ng = 1;
                L.tpg = 3;
            } else if (s.kind == BNN_NET_CONV_BIN) {
                // three tap rows per unit below one position per warp (nine single-tap units were slower:
                // CIFAR 39.4 -> 38.9 us with three, `tools/gpu_runs/r2_net_binng.sh`)
                L.ng = L.chunk >= kNetWarps ? 1 : 3;
                L.tpg = 9 / L.ng;
            }
            if (conv) {
                L.ptab_off = (int)ptab_words;  // words, made absolute below
                ptab_words += round4(L.chunk);
            }
        }
        P.packed_off[l] = packed;
        packed += up128((size_t)(s.kind == BNN_NET_FC_OUT ? 1 : L.KB) * L.slice_words * 4);
    }
    BNN_REQUIRE(layers[n - 1].K <= 4096, "net: at most 4096 classes");
    // shared memory: [mbarriers + flag | position tables | input stage | reduction | every block's slices]
    size_t off = up128(BNN_NET_MAX_LAYERS * 8 + 16);
    for (int l = 0; l < n; ++l)
        if (a.L[l].kind == BNN_NET_CONV_FIRST || a.L[l].kind == BNN_NET_CONV_BIN)
            a.L[l].ptab_off = (int)off + 4 * a.L[l].ptab_off;
    off += up128(ptab_words * 4);
    a.act_off = (int)off;
    off += up128(stage_bytes);
    a.red_off = (int)off;
    for (int l = 0; l < n; ++l) {
        NetLayerK &L = a.L[l];
        int most = 1;
        if (L.kind != BNN_NET_FC_OUT) {
            most = 0;
            for (int c = 0; c < G; ++c) {
                int f, st, cnt;
                cta_slices(L, c, G, f, st, cnt);
                most = std::max(most, cnt);
            }
            BNN_REQUIRE(most <= kNetSlots, "net: block %d needs %d slices per CTA (max %d)", l, most, kNetSlots);
            if (L.ng > 1) red_words = std::max(red_words, (size_t)most * L.chunk * 4 * 32);
        }
        L.most = most;
    }
    off += up128(std::max(red_words * 4, (size_t)B * layers[n - 1].K * 4));
    for (int l = 0; l < n; ++l) {
        NetLayerK &L = a.L[l];
        L.smem_off = (int)off;
        off += up128((size_t)L.most * L.slice_words * 4);
    }
    const size_t limit = 227 * 1024 - sizeof(NetArgs) - 1024;  // the kernel's static copy of the launch table
    BNN_REQUIRE(off <= limit, "net: batch %d needs %zu B of shared memory per CTA (max %zu)", B, off, limit);
    P.smem = off;
    // workspace: [packed slices of every block | counters (2 KB) | every block's output | staged images]
    const size_t img_bytes = (size_t)B * layers[0].C * layers[0].H * layers[0].W;
    // (every offset before the staged images is independent of B: a workspace prepared for a batch
    // serves any smaller batch, and the zero borders stay where the prepare put them)
    P.ctr_off = packed;
    P.act_off = P.ctr_off + 2048;  // barrier slots, `done`, `go`
    a.img_stride = (int)act_words;
    P.act_bytes = up128((size_t)B * act_words * 4);
    P.xstage_off = P.act_off + P.act_bytes;
    P.ws_bytes = P.xstage_off + up128(img_bytes);
    return 0;
}

static int grid_of(int grid) {
    const int sms = net_sm_count();
    return grid > 0 ? std::min(grid, sms) : sms;
}

int net_workspace(const bnn_net_layer *layers, int n, int B, int grid, size_t *bytes, size_t *smem) {
    BNN_REQUIRE(bytes, "net_workspace: null output");
    NetPlan P;
    const int rc = net_plan(layers, n, B, grid > 0 ? grid : net_sm_count(), P);
    if (rc) return rc;
    *bytes = P.ws_bytes;
    if (smem) *smem = P.smem;
    return 0;
}

int net_prepare(const bnn_net_layer *layers, int n, int B, void *ws, size_t ws_bytes, cudaStream_t st) {
    BNN_REQUIRE(ws, "net_prepare: null workspace");
    NetPlan P;
    const int rc = net_plan(layers, n, B, grid_of(0), P);
    if (rc) return rc;
    BNN_REQUIRE(ws_bytes >= P.ws_bytes, "net_prepare: workspace of %zu B < %zu B (bnn_net_workspace)", ws_bytes,
                P.ws_bytes);
    BNN_REQUIRE((reinterpret_cast<uintptr_t>(ws) & 127) == 0, "net_prepare: workspace must be 128-B aligned");
    for (int l = 0; l < n; ++l) {
        const bnn_net_layer &s = layers[l];
        BNN_REQUIRE(s.w, "net_prepare: block %d has no filters", l);
        if (s.kind != BNN_NET_FC_OUT) BNN_REQUIRE(s.thr && s.pos, "net_prepare: block %d needs thresholds", l);
    }
    uint8_t *w8 = static_cast<uint8_t *>(ws);
    for (int l = 0; l < n; ++l) {
        const bnn_net_layer &s = layers[l];
        const NetLayerK &L = P.a.L[l];
        const long long words = (long long)(s.kind == BNN_NET_FC_OUT ? 1 : L.KB) * L.slice_words;
        const int blocks = (int)std::min<long long>((words + 255) / 256, 4096);
        net_pack_kernel<<<blocks, 256, 0, st>>>(s.kind, s.C, s.K, L.R, L.LS, L.CW, L.KB, L.slice_words, L.epi_off,
                                                 s.w, s.thr, s.pos, reinterpret_cast<uint32_t *>(w8 + P.packed_off[l]));
        count_launch();
    }
    // the barrier counter, and every block's output buffer (its zero border is never written again)
    cudaError_t e = cudaMemsetAsync(w8 + P.ctr_off, 0, 2048, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(w8 + P.act_off, 0, P.act_bytes, st);
    if (e != cudaSuccess) {
        set_error("net_prepare: memset: %s", cudaGetErrorString(e));
        return (int)e;
    }
    return after_launch("net_prepare");
}

int net_infer(const bnn_net_layer *layers, int n, const uint8_t *x, int x_host, int B, int32_t *logits,
              int32_t *preds, void *ws, size_t ws_bytes, int grid, cudaStream_t st) {
    BNN_REQUIRE(x && ws, "net_infer: null pointer");
    const int G = grid_of(grid);
    NetPlan P;
    const int rc = net_plan(layers, n, B, G, P);
    if (rc) return rc;
    BNN_REQUIRE(ws_bytes >= P.ws_bytes, "net_infer: workspace of %zu B < %zu B (bnn_net_workspace)", ws_bytes,
                P.ws_bytes);
    BNN_REQUIRE((reinterpret_cast<uintptr_t>(ws) & 127) == 0, "net_infer: workspace must be 128-B aligned");
    BNN_REQUIRE(!x_host || (reinterpret_cast<uintptr_t>(x) & 15) == 0, "net_infer: host images must be 16-B aligned");
    NetArgs &a = P.a;
    uint8_t *w8 = static_cast<uint8_t *>(ws);
    for (int l = 0; l < n; ++l) a.L[l].packed = reinterpret_cast<const uint32_t *>(w8 + P.packed_off[l]);
    a.x = x;
    a.x_host = x_host ? 1 : 0;
    a.ctr = reinterpret_cast<unsigned *>(w8 + P.ctr_off);
    a.xstage = w8 + P.xstage_off;
    a.act = reinterpret_cast<uint32_t *>(w8 + P.act_off);
    a.logits = logits;
    a.preds = preds;
    a.trace = g_net_trace;
    {
        const char *e = getenv("BNN_NET_REPS");
        a.reps = e ? std::max(1, atoi(e)) : 1;
    }
    auto kern = a.trace || a.reps > 1 ? net_b1_kernel<1> : net_b1_kernel<0>;
    int e = allow_smem(reinterpret_cast<const void *>(kern), P.smem, "net_infer");
    if (e) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kNetThreads);
    cfg.dynamicSmemBytes = P.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the grid barriers need it
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a);
    count_launch();
    return after_launch("net_infer");
}

// ---------------------------------------------------------------- persistent serving
// The same kernel as a resident server: weights stay in shared memory, CTA 0 polls a host-mapped doorbell,
// every request runs the whole network on the images in pinned host memory and rings a completion word --
// no launch, no graph, no stream synchronisation per request.
int net_serve_launch(const bnn_net_layer *layers, int n, int B, void *ws, size_t ws_bytes, unsigned *ctl,
                     const uint8_t *x_host, int32_t *logits, int32_t *preds, int grid, double idle_s, cudaStream_t st) {
    BNN_REQUIRE(ws && ctl && x_host, "net_serve_launch: null pointer");
    BNN_REQUIRE((reinterpret_cast<uintptr_t>(ctl) & 127) == 0, "net_serve_launch: control block must be 128-B aligned");
    BNN_REQUIRE(idle_s > 0, "net_serve_launch: idle timeout must be > 0");
    const int G = grid_of(grid);
    NetPlan P;
    const int rc = net_plan(layers, n, B, G, P);
    if (rc) return rc;
    BNN_REQUIRE(ws_bytes >= P.ws_bytes, "net_serve_launch: workspace of %zu B < %zu B", ws_bytes, P.ws_bytes);
    BNN_REQUIRE((reinterpret_cast<uintptr_t>(ws) & 127) == 0, "net_serve_launch: workspace must be 128-B aligned");
    BNN_REQUIRE((reinterpret_cast<uintptr_t>(x_host) & 15) == 0, "net_serve_launch: images must be 16-B aligned");
    NetArgs &a = P.a;
    uint8_t *w8 = static_cast<uint8_t *>(ws);
    for (int l = 0; l < n; ++l) a.L[l].packed = reinterpret_cast<const uint32_t *>(w8 + P.packed_off[l]);
    a.x = x_host;
    a.x_host = 1;
    a.ctr = reinterpret_cast<unsigned *>(w8 + P.ctr_off);
    a.go = reinterpret_cast<unsigned *>(w8 + P.ctr_off) + (kNetCtrSlots + 1) * kNetCtrStride;
    a.xstage = w8 + P.xstage_off;
    a.act = reinterpret_cast<uint32_t *>(w8 + P.act_off);
    a.logits = logits;
    a.preds = preds;
    a.reps = 1;
    a.ctl = ctl;
    a.idle_ns = (unsigned long long)(idle_s * 1e9);
    cudaError_t e = cudaMemsetAsync(a.go, 0, 4, st);
    if (e != cudaSuccess) {
        set_error("net_serve_launch: memset: %s", cudaGetErrorString(e));
        return (int)e;
    }
    auto kern = net_b1_kernel<0>;
    int r = allow_smem(reinterpret_cast<const void *>(kern), P.smem, "net_serve_launch");
    if (r) return r;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kNetThreads);
    cfg.dynamicSmemBytes = P.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a);
    count_launch();
    return after_launch("net_serve_launch");
}

int net_serve_request(unsigned *ctl, const void *images, size_t bytes, void *x_host, const int32_t *logits_host,
                      int32_t *logits_out, size_t logits_bytes, const int32_t *preds_host, int32_t *preds_out,
                      size_t preds_bytes, double timeout_s) {
    BNN_REQUIRE(ctl && images && x_host, "net_serve_request: null pointer");
    if (__atomic_load_n(ctl + BNN_NET_CTL_STATUS, __ATOMIC_ACQUIRE)) {
        set_error("net_serve_request: the server has stopped (idle timeout or stop)");
        return -2;
    }
    std::memcpy(x_host, images, bytes);
    const unsigned req = __atomic_load_n(ctl + BNN_NET_CTL_REQ, __ATOMIC_RELAXED) + 1;
    __atomic_store_n(ctl + BNN_NET_CTL_REQ, req, __ATOMIC_RELEASE);  // the images are visible before the doorbell
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t spins = 0; __atomic_load_n(ctl + BNN_NET_CTL_DONE, __ATOMIC_ACQUIRE) != req; ++spins) {
        if ((spins & 1023) == 0 &&
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
            set_error("net_serve_request: no completion after %.3f s", timeout_s);
            return -3;
        }
    }
    if (logits_out && logits_host) std::memcpy(logits_out, logits_host, logits_bytes);
    if (preds_out && preds_host) std::memcpy(preds_out, preds_host, preds_bytes);
    return 0;
}

int net_serve_stop(unsigned *ctl) {
    BNN_REQUIRE(ctl, "net_serve_stop: null pointer");
    __atomic_store_n(ctl + BNN_NET_CTL_STOP, 1u, __ATOMIC_RELEASE);
    return 0;
}

}  // namespace bnn
