// tc_gemm.cu -- BNN conv / FC blocks on the 5th-gen tensor cores (tcgen05.mma kind::mxf4).
//
// The +-1 data are stored as FP4 E2M1 codes (+1 = 0x2, -1 = 0xA, 0 = padding; two channels per
// byte, NHWC; common.cuh) so a binary dot product is an exact block-scaled FP4 MMA with unit
// scales and fp32 accumulation: K = 64 per instruction from 32 bytes per row -- twice the K of
// the int8 kind for the same shared-memory traffic, and twice its tensor rate.  Implicit GEMM:
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
#include "tc_ptx.cuh"

namespace bnn {

struct TcArgs {
    int T, CCH, nks;      // taps, channel chunks per tap, k-steps
    int BW, BH, BB;       // box (pixels per tile = BW*BH*BB <= 128)
    int W, H, B;          // logical activation dims (FC: W = H = 1, B = batch)
    int K;                // output channels / neurons
    int ntx, nty;         // tiles along x, y
    int n_mtiles;         // spatial (row) tiles = ntx * nty * ceil(B / BB)
    int bres;             // >0: the whole B operand of bres N tiles (nks slabs each) is smem-resident, loaded once per CTA
    const int32_t *thr;
    const uint32_t *pos;
    int pool, out_fmt;    // out_fmt: 0 = NHWC bits (u32), 1 = NHWC FP4 +-1, 2 = logits + argmax
    void *out;
    int32_t *sums;        // NCHW int32 pre-activations (pre-pool) or null
    int32_t *preds;       // out_fmt 2
    uint32_t idesc;       // instruction descriptor
    int a_bytes;          // TMA bytes of one A box
    unsigned long long *trace;  // debug clock64 timeline of CTA 0 (bnn_tc_trace), or null
    int tma_out;          // FP4 output staged in swizzled smem and written by one TMA store per tile
    int out_rows;         // output pixels per tile (128, or 32 after 2x2 pooling)
    int step_mma;         // the step constant enters the accumulator through one extra MMA per tile
    int early_weights;    // filters / thresholds / step rows may be read before the PDL wait (static)
    // ceil(2^32 / d) for d = ntx * nty, ntx, N tiles: tile index -> coordinates by one wide multiply
    // (the producer is a single thread, and four integer divisions per tile cost it ~700 clk)
    uint64_t md_txy, md_ntx, md_nnt;
};

__host__ __device__ inline uint64_t fdiv_magic(uint32_t d) { return ((1ull << 32) + d - 1) / d; }
// n / d for n * d < 2^32 (every tile index here), d >= 1
__device__ __forceinline__ int fdiv(int n, uint64_t magic) { return (int)(((uint64_t)(uint32_t)n * magic) >> 32); }

// Debug timeline of tc_block_kernel, CTA 0: role 0 = TMA producer per stage (wait start, slot free,
// issued), 1 = MMA per stage (wait start, data ready, issued), 2 = MMA per tile (tempty wait start,
// got), 3 = epilogue (warp 2) per tile (wait start, accumulator ready, done).  512 items x 4 stamps.
#define TC_TRACE(role, n, f, val)                                                                       \
    do {                                                                                                \
        if (a.trace && blockIdx.x == 0 && (n) < 512)                                                     \
            a.trace[((size_t)(role) * 512 + (n)) * 4 + (f)] = (unsigned long long)(val);                 \
    } while (0)
static unsigned long long *g_tc_trace = nullptr;

// ------------------------------------------------------------------ the kernel
constexpr int kTcThreads = 320;  // halo kernel: w0 TMA, w1 MMA, w2..w9 epilogue
// tc_block_kernel: w0 TMA, w1 MMA, 16 epilogue warps (4 TMEM lane quarters x 4 column groups) -- the
// epilogue is latency-bound, so more warps in flight (not fewer instructions) is what keeps up
constexpr int kBlkEpiWarps = 8;
constexpr int kBlkThreads = 64 + 32 * kBlkEpiWarps;
constexpr int kMaxK = 4096;  // output channels / neurons staged in smem (thresholds)

// TMEM: accumulators (double-buffered up to BN = 128; a single BN = 256 buffer drained into
// registers at once) followed by 32 scale-factor columns (16 SFA + 16 SFB, all 2^0).
__host__ __device__ constexpr int tmem_pow2(int cols) { return cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512; }

// The step folded into the MMA (TcArgs::step_mma): acc + c, c = T + 0.5 (POS) / 0.5 - T (NEG), is
// produced by the tensor core through one extra K = 64 MMA per tile whose A block is the same for
// every row -- FP4 6.0 in 48 K positions and 0.5 in 16 (bytes 0x77 x 12 + 0x11 x 4 in each 16-B
// half, so the SW32 swizzle cannot move anything) -- and whose B row for channel n holds FP4 values
// summing to c_n = 6 X + 0.5 Y (bnn_step_rows).  The epilogue then only takes signs.
constexpr int kStepA = 128 * 32;

// TPS = K-steps (tap boxes) per pipeline stage: a 32-B chunk is a single K=64 MMA, too little work
// to amortise a barrier round trip, so thin chunks travel three taps per stage (9 taps = 3 stages)
// PAIR: CTA pair (cluster of 2, tcgen05 cta_group::2) -- M = 256 per MMA, each CTA holds its own
// 128 A rows and HALF of the B tile; the pair's tensor cores share both halves.
template <int BN, int KC, int S, int TPS = 1, bool PAIR = false>
struct TcSmem {
    static constexpr int A_BYTES = 128 * KC;  // one box; a stage holds TPS of them
    static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * KC;
    static constexpr int BITS_WORDS = 128 * (BN / 32);
    static constexpr int NACC = BN == 256 ? 1 : 2;
    static constexpr int ACC_COLS = NACC * BN;
    static constexpr int TMEM_COLS = tmem_pow2(ACC_COLS + 32);
    // runtime total: B region = (bres ? nks : S) stages; thresholds = K ints
    // output staging for the TMA-store epilogue: 2 buffers x out_rows x BN/2 bytes (FP4)
    __host__ __device__ static size_t out_bytes(int out_rows) { return (size_t)2 * out_rows * (BN / 2); }
    // step-MMA operands: the constant 128 x 32-B A block + one 32-B step row per output channel
    __host__ __device__ static size_t step_bytes(int n_ntiles) { return (size_t)kStepA + (size_t)n_ntiles * BN * 32; }
    // bres: number of N-tile filter banks kept resident in smem (0 = B streamed per stage)
    static size_t total(int nks, int bres, int K, int out_rows, size_t step = 0) {
        const size_t b_slabs = bres ? (size_t)nks * bres : (size_t)S * TPS;
        const size_t kpad = (size_t)(K + 31) / 32 * 32;
        return 1024 + (size_t)S * TPS * A_BYTES + b_slabs * B_BYTES + (out_rows ? (out_bytes(out_rows) + 1023) / 1024 * 1024 : 0) +
               step + (2 * S + 5) * 8 + 32 + kpad * 8 + kpad / 8 + (size_t)BITS_WORDS * 4 + 16;
    }
};


__device__ __forceinline__ void store_word(const TcArgs &a, long long pix, int nb, uint32_t bits, int KW) {
    if (a.out_fmt == 0)
        static_cast<uint32_t *>(a.out)[pix * KW + (nb >> 5)] = bits;
    else  // FP4: 32 channels = 16 bytes at byte (pix * K + nb) / 2
        *reinterpret_cast<uint4 *>(static_cast<uint8_t *>(a.out) + ((pix * a.K + nb) >> 1)) = bits_to_f4(bits);
}

// pre-activation from an fp32 accumulator: filters of POS channels are direction-folded (negated)
// whenever the layer's step is fused (thresholds given)
__device__ __forceinline__ int32_t unfold_acc(uint32_t acc, bool negated) {
    const int32_t v = (int32_t)__uint_as_float(acc);
    return negated ? -v : v;
}

// One 32-column accumulator chunk of the tc_block epilogue: debug sums, logits + first-max argmax,
// or the step as fire masks -> FP4 / bits (smem for pooling).  A real function (not a lambda) so it
// is always inlined -- an outlined call passes the accumulator array through local memory.
template <int BN>
__device__ __forceinline__ void tc_chunk(const TcArgs &a, uint32_t (&v)[32], int j, int n0, bool inb, bool logits,
                                         long long gb, int gy, int gx, int m_row, int KW, const float *s_c,
                                         const uint32_t *s_pos,
                                         uint32_t *s_bits, int &best, int &bestv, uint8_t *stage) {
        const int nb = n0 + j * 32;
        if (a.sums && inb) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
                if (nb + i < a.K) {
                    const uint32_t acc = a.step_mma ? __float_as_uint(__uint_as_float(v[i]) - s_c[nb + i]) : v[i];
                    a.sums[(((long long)gb * a.K + nb + i) * a.H + gy) * a.W + gx] =
                        unfold_acc(acc, a.thr != nullptr && ((s_pos[(nb + i) >> 5] >> ((nb + i) & 31)) & 1u));
                }
        }
        if (logits) {
            if (inb) {
                int32_t *lg = static_cast<int32_t *>(a.out);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (nb + i >= a.K) break;
                    const int val = (int32_t)__uint_as_float(v[i]);
                    if (lg) lg[(long long)gb * a.K + nb + i] = val;
                    if (nb + i == 0 || val > bestv) {  // first max wins ties (np.argmax)
                        best = nb + i;
                        bestv = val;
                    }
                }
            }
            return;
        }
        if (nb >= a.K) {
            if (a.pool) s_bits[m_row * (BN / 32) + j] = 0u;
            return;
        }
        if (!a.step_mma) step32c(v, s_c + nb);  // else the MMA already added the constant
        if (!a.pool && a.out_fmt == 1) {  // FP4 straight from the signs (K % 32 == 0)
            if (a.tma_out) {  // swizzled staging row of the TMA store (rows beyond the tensor are clipped)
                *reinterpret_cast<uint4 *>(stage + sw_chunk_off((uint32_t)m_row, (uint32_t)j, BN / 2)) = sgn32_f4(v);
                return;
            }
            if (a.out && inb)
                *reinterpret_cast<uint4 *>(static_cast<uint8_t *>(a.out) +
                                           ((((long long)gb * a.H + gy) * a.W + gx) * a.K + nb) / 2) = sgn32_f4(v);
            return;
        }
        uint32_t bits = sgn32_bits(v);
        if (nb + 32 > a.K) bits &= 0xffffffffu >> (32 - (a.K - nb));
        if (a.pool) {
            s_bits[m_row * (BN / 32) + j] = bits;
        } else if (a.out && inb) {
            store_word(a, ((long long)gb * a.H + gy) * a.W + gx, nb, bits, KW);
        }
}

// Persistent, warp-specialised: grid = min(#tiles, #SMs); CTA c handles tiles c, c+grid, ...
// tile t -> (spatial tile m = t / n_ntiles, channel tile n = t % n_ntiles).  The TMA producer
// runs ahead across tile boundaries through an S-stage ring; the MMA warp accumulates tile i
// into TMEM buffer i%2 while the epilogue warps drain buffer (i-1)%2.
// HX (halo along x; 16-pixel rows of 32-B pixels, tiles of 8 rows x 16 px, filters resident): the
// three taps dx = -1, 0, +1 of a filter row dy share ONE pair of TMA boxes -- the left and right
// 8-px halves of the 8 rows, each with its 1-px halo (10 x 8 px, zero-filled outside the image) --
// and are MMA'd from it by row-shifted descriptors.  The M order is then (half, row, px % 8), so
// every 8-row core group starts 10 rows after the previous one (SBO = 320 B) and the epilogue maps
// TMEM lane m to pixel (m >> 3 & 7, (m >> 6) * 8 + m % 8).  480 instead of 1,152 TMA rows per tile:
// the TMA engine's row rate bounded the per-tap kernel on these layers.
template <int BN, int KC, int S, int TPS, bool HX = false>
__global__ void __launch_bounds__(kBlkThreads, 1)
    tc_block_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmS, const TcArgs a) {
    pdl_trigger();
    using L = TcSmem<BN, KC, S, TPS>;
    extern __shared__ uint8_t smem_raw[];
    // align by pointer arithmetic on the __shared__ array so the compiler keeps the shared address
    // space (a uintptr_t round trip turns every smem access into a generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    uint8_t *sA = smem;
    uint8_t *sB = smem + S * TPS * L::A_BYTES;
    const int b_slabs = a.bres ? a.nks * a.bres : S * TPS;
    uint8_t *s_out = sB + (size_t)b_slabs * L::B_BYTES;  // 1024-aligned (A, B slabs are multiples of 1 KB)
    const size_t out_region = a.tma_out ? (L::out_bytes(a.out_rows) + 1023) / 1024 * 1024 : 0;
    const int n_ntiles = (a.K + BN - 1) / BN;
    uint8_t *s_step = s_out + out_region;  // step MMA: constant A block, then the step rows of every N tile
    uint64_t *full = reinterpret_cast<uint64_t *>(s_step + (a.step_mma ? L::step_bytes(n_ntiles) : 0));
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;   // [2]
    uint64_t *tempty = tfull + 2;  // [2]
    uint64_t *bfull = tempty + 2;  // resident-B arrival
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bfull + 1);
    float2 *s_st =
        reinterpret_cast<float2 *>(smem_raw + ((smem_addr(tmem_slot + 1) - smem_addr(smem_raw) + 15u) & ~15u));
    uint32_t *s_pos = reinterpret_cast<uint32_t *>(s_st + (a.K + 31) / 32 * 32);
    uint32_t *s_bits = s_pos + (a.K + 31) / 32;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_xy = a.ntx * a.nty;
    const int total = a.n_mtiles * n_ntiles;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kBlkEpiWarps);  // one arrive per epilogue warp
        }
        mbar_init(bfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                     "r"(L::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // everything above overlaps the previous launch (PDL); every global read comes after the wait --
    // or, when the caller vouches that filters / thresholds / step rows are static (early_weights),
    // only the activation reads do: those operands are then fetched while the predecessor runs
    if (!a.early_weights) pdl_wait();
    if (warp >= 2) {  // all thresholds / direction words of the layer, once per CTA
        const int kpad = (a.K + 31) / 32 * 32;
        for (int i = threadIdx.x - 64; i < kpad / 32; i += 32 * kBlkEpiWarps) s_pos[i] = a.pos ? __ldg(a.pos + i) : 0u;
        for (int i = threadIdx.x - 64; i < kpad; i += 32 * kBlkEpiWarps) {
            const bool ok = a.thr && a.pos && i < a.K;
            // T clamped to +-(kred + 1) decides every sum the same way -- and is what the step rows hold
            const int kred = a.nks * KC * 2;
            reinterpret_cast<float *>(s_st)[i] =
                step_const(ok ? max(-kred - 1, min(kred + 1, __ldg(a.thr + i))) : 0,
                           ok ? ((__ldg(a.pos + (i >> 5)) >> (i & 31)) & 1u) : true);
        }
        if (a.step_mma) {  // the constant A block of the step MMA (read by the tensor core: async proxy)
            for (int i = threadIdx.x - 64; i < kStepA / 16; i += 32 * kBlkEpiWarps)
                reinterpret_cast<uint4 *>(s_step)[i] = make_uint4(0x77777777u, 0x77777777u, 0x77777777u, 0x11111111u);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t tmem_sfa = tmem_base + L::ACC_COLS, tmem_sfb = tmem_sfa + 16;
    if (warp >= 2 && warp < 6) tmem_fill_sf(tmem_sfa, 32, warp);  // unit scales, one lane quarter per warp
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            if (a.bres || a.step_mma) {  // resident operands, loaded once per CTA
                mbar_expect_tx(bfull, (uint32_t)(a.nks * a.bres) * L::B_BYTES + (a.step_mma ? n_ntiles * BN * 32u : 0u));
                // the whole filter bank (every N tile)
                for (int nt = 0; nt < a.bres; ++nt)
                    for (int ks = 0; ks < a.nks; ++ks)
                        tma_load_2d(sB + (nt * a.nks + ks) * L::B_BYTES, &tmB, bfull, ks * KC, nt * BN);
                if (a.step_mma)
                    for (int nt = 0; nt < n_ntiles; ++nt)
                        tma_load_2d(s_step + kStepA + nt * BN * 32, &tmS, bfull, 0, nt * BN);
            }
            if (a.early_weights) pdl_wait();  // the activations come from the predecessor
            // The producer is a single thread: keep its per-stage work to table lookups.
            const uint32_t tx_bytes = HX ? 2u * 10u * 8u * KC : TPS * (a.a_bytes + (a.bres ? 0 : L::B_BYTES));
            uint32_t s = 0, round_par = 1;  // round_par = parity to wait on empty[s]
            int tn = 0;
            int m = blockIdx.x / n_ntiles, nt = blockIdx.x % n_ntiles;
            const int m_step = gridDim.x / n_ntiles, n_step = gridDim.x % n_ntiles;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                const int n0 = nt * BN;
                const int tb = fdiv(m, a.md_txy), rem = m - tb * tiles_xy;
                const int ty = fdiv(rem, a.md_ntx);
                const int x0 = (rem - ty * a.ntx) * a.BW, y0 = ty * a.BH, b0 = tb * a.BB;
                int cc = 0, dx = a.T == 9 ? -1 : 0, dy = a.T == 9 ? -1 : 0;
                for (int ks = 0; ks < a.nks; ks += TPS, ++tn) {
                    TC_TRACE(0, tn, 0, clock64());
                    mbar_wait(&empty[s], round_par);
                    TC_TRACE(0, tn, 1, clock64());
                    mbar_expect_tx(&full[s], tx_bytes);
                    if constexpr (HX) {  // filter row dy: left / right half boxes with their x halo
                        tma_load_4d(sA + s * TPS * L::A_BYTES, &tmA, &full[s], 0, x0 - 1, y0 + dy, b0);
                        tma_load_4d(sA + s * TPS * L::A_BYTES + 80 * KC, &tmA, &full[s], 0, x0 + 7, y0 + dy, b0);
                    }
#pragma unroll
                    for (int tt = 0; tt < TPS; ++tt) {
                        if (!HX) tma_load_4d(sA + (s * TPS + tt) * L::A_BYTES, &tmA, &full[s], cc * KC, x0 + dx, y0 + dy, b0);
                        if (!a.bres) tma_load_2d(sB + (s * TPS + tt) * L::B_BYTES, &tmB, &full[s], (ks + tt) * KC, n0);
                        if (++cc == a.CCH) {  // next tap (dy, dx) in row-major order
                            cc = 0;
                            if (a.T == 9 && ++dx == 2) {
                                dx = -1;
                                ++dy;
                            }
                        }
                    }
                    TC_TRACE(0, tn, 2, clock64());
                    if (++s == S) {
                        s = 0;
                        round_par ^= 1;
                    }
                }
                // advance (m, nt) by gridDim.x tiles without a division per tile
                nt += n_step;
                m += m_step;
                if (nt >= n_ntiles) {
                    nt -= n_ntiles;
                    ++m;
                }
            }
        }
    } else if (warp == 1) {
        {  // ---------------- MMA issuer (whole warp, one elected lane issues)
            if (a.bres || a.step_mma) mbar_wait(bfull, 0);
            uint32_t lt = 0, s = 0, par = 0;
            // descriptors are additive in their start-address field: build once, offset per MMA
            const uint64_t adesc0 = umma_desc(smem_addr(sA), KC), bdesc0 = umma_desc(smem_addr(sB), KC);
            // HX: 8-row groups 10 rows apart (SBO field = 320 B / 16)
            const uint64_t hdesc0 = (adesc0 & ~(0x3FFFull << 32)) | ((uint64_t)((10 * KC) >> 4) << 32);
            const uint64_t sdesc_a = umma_desc(smem_addr(s_step), 32), sdesc_b = umma_desc(smem_addr(s_step + kStepA), 32);
            int tn = 0;
            // N tile of t advanced without a division: an integer modulo on this path sits between
            // the accumulator hand-back and the first MMA of the next tile
            int nt = blockIdx.x % n_ntiles;
            const int nt_step = gridDim.x % n_ntiles;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
                const uint32_t acc = lt % L::NACC, aph = (lt / L::NACC) & 1;
                const uint32_t b_base = a.bres ? (uint32_t)(nt * a.nks) : 0u;  // resident bank of this N tile
                const uint64_t sdesc = sdesc_b + (((uint32_t)nt * BN * 32) >> 4);
                if (lane == 0) TC_TRACE(2, lt, 0, clock64());
                mbar_wait(&tempty[acc], aph ^ 1);
                tc_fence_after();
                if (lane == 0) TC_TRACE(2, lt, 1, clock64());
                const uint32_t tmem_d = tmem_base + acc * BN;
                if (a.step_mma)  // D = c first (its operands are resident); every tap accumulates on top
                    umma_f4_elect(tmem_d, sdesc_a, sdesc, a.idesc, false, tmem_sfa, tmem_sfb);
                if ((nt += nt_step) >= n_ntiles) nt -= n_ntiles;
                for (int ks = 0; ks < a.nks; ks += TPS, ++tn) {
                    if (lane == 0) TC_TRACE(1, tn, 0, clock64());
                    mbar_wait(&full[s], par);
                    tc_fence_after();
                    if (lane == 0) TC_TRACE(1, tn, 1, clock64());
                    {  // TPS boxes x KC / 32 K-chunks of this stage in one issue block; HX: tap dx = row shift
                        const uint64_t a0 = (HX ? hdesc0 : adesc0) + ((s * TPS * L::A_BYTES) >> 4);
                        const uint64_t b0 =
                            bdesc0 + (((a.bres ? b_base + (uint32_t)ks : (uint32_t)(s * TPS)) * L::B_BYTES) >> 4);
                        umma_f4_multi<TPS, KC / 32, HX ? KC / 16 : L::A_BYTES / 16, L::B_BYTES / 16>(
                            tmem_d, a0, b0, a.idesc, a.step_mma || ks != 0, tmem_sfa, tmem_sfb);
                    }
                    umma_commit_elect(&empty[s]);
                    if (lane == 0) TC_TRACE(1, tn, 2, clock64());
                    if (++s == S) {
                        s = 0;
                        par ^= 1;
                    }
                }
                umma_commit_elect(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {  // ------------------------- epilogue (warps 2..9)
        // TMEM lane quarter = warp % 4 (hardware rule); the two warps sharing a quarter split
        // the 32-column chunks round-robin (group g takes chunks g, g + 4, ...).
        constexpr int NG = kBlkEpiWarps / 4;
        const int q = warp & 3, half = (warp - 2) >> 2;  // half = column group 0..NG-1
        const int m_lane = q * 32 + lane;  // TMEM lane
        const int npix = a.BW * a.BH * a.BB;
        // pixel of this lane within the tile, and its row index in pixel order
        const int bx = HX ? ((m_lane >> 6) << 3) + (m_lane & 7) : m_lane % a.BW;
        const int by = HX ? (m_lane >> 3) & 7 : (m_lane / a.BW) % a.BH;
        const int bb = HX ? 0 : m_lane / (a.BW * a.BH);
        const int m_row = HX ? by * 16 + bx : m_lane;
        const int Ho = a.pool ? a.H / 2 : a.H, Wo = a.pool ? a.W / 2 : a.W;
        const int KW = (a.K + 31) / 32;
        const bool logits = a.out_fmt == 2;
        const int j0 = logits ? 0 : half, jstep = logits ? 1 : NG;
        const bool active_warp = !logits || half == 0;
        uint32_t lt = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
            const uint32_t acc = lt % L::NACC, aph = (lt / L::NACC) & 1;
            const int m = fdiv(t, a.md_nnt), n0 = (t - m * n_ntiles) * BN;
            const int tb = fdiv(m, a.md_txy), rem = m - tb * tiles_xy, ty = fdiv(rem, a.md_ntx);
            const int gx = (rem - ty * a.ntx) * a.BW + bx, gy = ty * a.BH + by, gb = tb * a.BB + bb;
            const bool inb = m_row < npix && gx < a.W && gy < a.H && gb < a.B;
            const uint32_t trow = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
            if (threadIdx.x == 64) TC_TRACE(3, lt, 0, clock64());
            mbar_wait(&tfull[acc], aph);
            if (threadIdx.x == 64) TC_TRACE(3, lt, 1, clock64());
            tc_fence_after();
            uint8_t *stage = s_out + (size_t)(lt & 1) * a.out_rows * (BN / 2);
            auto staging_free = [&]() {
                if (a.tma_out && threadIdx.x == 64) tma_store_wait_read<1>();  // this buffer's store (2 tiles ago) read out
                if (a.pool || a.tma_out)
                    asm volatile("bar.sync 1, %0;" ::"n"(32 * kBlkEpiWarps) : "memory");  // exchange / staging free
            };
            int best = 0, bestv = 0;
            // one 32-column chunk: sums, logits + argmax, or step -> bits (smem for pooling) / output
            if constexpr (L::NACC == 1) {
                // single accumulator: drain this warp's columns into registers and release TMEM to the
                // MMA warp before anything else (the MMA of the next tile waits on it), then threshold /
                // store from registers
                constexpr int NCH = BN / 32 >= NG ? BN / 32 / NG : 1;
                uint32_t vv[NCH][32];
#pragma unroll
                for (int c = 0; c < NCH; ++c) TMEM_LD32(trow + (half + NG * c) * 32, vv[c]);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                if (threadIdx.x == 64) TC_TRACE(3, lt, 3, clock64());
                staging_free();
                // Common case as straight-line code over all NCH chunks, so the scheduler can overlap
                // their latencies (the general per-chunk path branches on every mode flag, which
                // serialises the chunks: with 2 epilogue warps per scheduler that is what bounds it)
                const bool fast = !a.sums && !logits && n0 + BN <= a.K && (a.pool || (a.out_fmt == 1 && a.tma_out));
                if (fast) {
                    if (!a.step_mma) {
#pragma unroll
                        for (int c = 0; c < NCH; ++c)
                            step32c(vv[c], reinterpret_cast<const float *>(s_st) + n0 + (half + NG * c) * 32);
                    }
                    if (a.pool) {
#pragma unroll
                        for (int c = 0; c < NCH; ++c) s_bits[m_row * (BN / 32) + half + NG * c] = sgn32_bits(vv[c]);
                    } else {
#pragma unroll
                        for (int c = 0; c < NCH; ++c)
                            *reinterpret_cast<uint4 *>(stage + sw_chunk_off((uint32_t)m_row, (uint32_t)(half + NG * c), BN / 2)) =
                                sgn32_f4(vv[c]);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
                        tc_chunk<BN>(a, vv[c], half + NG * c, n0, inb, logits, gb, gy, gx, m_row, KW,
                                     reinterpret_cast<const float *>(s_st), s_pos, s_bits, best, bestv, stage);
                }
            } else {
                staging_free();
                if (active_warp) {
#pragma unroll 1
                    for (int j = j0; j < BN / 32; j += jstep) {
                        uint32_t v[32];
                        TMEM_LD32(trow + j * 32, v);
                        tmem_wait_ld();
                        tc_chunk<BN>(a, v, j, n0, inb, logits, gb, gy, gx, m_row, KW,
                                     reinterpret_cast<const float *>(s_st), s_pos, s_bits, best, bestv, stage);
                    }
                }
                // accumulator drained: hand TMEM buffer `acc` back to the MMA warp
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
            }
            if (threadIdx.x == 64) TC_TRACE(3, lt, 2, clock64());
            if (logits) {
                if (half == 0 && inb && a.preds) a.preds[gb] = best;
            } else if (a.pool) {
                asm volatile("bar.sync 1, %0;" ::"n"(32 * kBlkEpiWarps) : "memory");  // all rows of the tile written
                if (a.out && inb && !(bx & 1) && !(by & 1)) {
                    const long long opix = ((long long)gb * Ho + gy / 2) * Wo + gx / 2;
                    // pooled pixel index inside the tile (tiles cover whole rows: BW == W)
                    const int prow = ((bb * a.BH + by) / 2) * (a.BW / 2) + bx / 2;
                    const int st = BN / 32;
#pragma unroll 1
                    for (int j = half; j < BN / 32; j += NG) {
                        const int nb = n0 + j * 32;
                        if (nb >= a.K) break;
                        const uint32_t p0 = s_bits[m_row * st + j], p1 = s_bits[(m_row + 1) * st + j];
                        const uint32_t p2 = s_bits[(m_row + a.BW) * st + j], p3 = s_bits[(m_row + a.BW + 1) * st + j];
                        const uint32_t pw = s_pos[nb >> 5];
                        const uint32_t pb = ((p0 | p1 | p2 | p3) & pw) | ((p0 & p1 & p2 & p3) & ~pw);
                        if (a.tma_out)
                            *reinterpret_cast<uint4 *>(stage + sw_chunk_off((uint32_t)prow, (uint32_t)j, BN / 2)) =
                                bits_to_f4(pb);
                        else
                            store_word(a, opix, nb, pb, KW);
                    }
                }
            }
            if (a.tma_out) {  // the whole tile's output: one TMA store from the staging buffer
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 1, %0;" ::"n"(32 * kBlkEpiWarps) : "memory");
                if (threadIdx.x == 64) {
                    const int tb = fdiv(m, a.md_txy), rem = m - tb * tiles_xy;
                    const int y0 = fdiv(rem, a.md_ntx) * a.BH, b0 = tb * a.BB;
                    const long long p0 = a.pool ? ((long long)b0 * Ho + y0 / 2) * Wo : ((long long)b0 * a.H + y0) * a.W;
                    tma_store_2d(&tmO, stage, n0 / 2, (int)p0);
                    tma_store_commit();
                }
            }
        }
    }
    if (a.tma_out && threadIdx.x == 64) tma_store_wait_all();
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(L::TMEM_COLS));
    }
}

// CTA-pair version of tc_block_kernel, launched only with PAIR = true (clusters of 2): the pair is
// the scheduling unit (M tiles 2u and 2u + 1, rank r takes 2u + r), each CTA TMA-loads its own A
// box and HALF of the streamed B tile with completion counted on the leader's full barrier, the
// leader's MMA warp issues tcgen05.mma.cta_group::2 (M = 256) and commits to both CTAs' barriers,
// and the peer's epilogue returns its accumulator through a remote arrive on the leader's tempty.
// The `if constexpr (PAIR)` alternatives keep the body readable next to tc_block_kernel; the
// single-CTA path is NOT taken from here (tc_block_kernel above is measurably faster for it).
template <int BN, int KC, int S, int TPS, bool PAIR>
__global__ void __launch_bounds__(kBlkThreads, 1)
    tc_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmS, const TcArgs a) {
    pdl_trigger();
    using L = TcSmem<BN, KC, S, TPS, PAIR>;
    extern __shared__ uint8_t smem_raw[];
    // align by pointer arithmetic on the __shared__ array so the compiler keeps the shared address
    // space (a uintptr_t round trip turns every smem access into a generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    uint8_t *sA = smem;
    uint8_t *sB = smem + S * TPS * L::A_BYTES;
    const int b_slabs = a.bres ? a.nks * a.bres : S * TPS;
    uint8_t *s_out = sB + (size_t)b_slabs * L::B_BYTES;  // 1024-aligned (A, B slabs are multiples of 1 KB)
    const size_t out_region = a.tma_out ? (L::out_bytes(a.out_rows) + 1023) / 1024 * 1024 : 0;
    const int n_ntiles = (a.K + BN - 1) / BN;
    uint8_t *s_step = s_out + out_region;  // step MMA: constant A block, then the step rows of every N tile
    uint64_t *full = reinterpret_cast<uint64_t *>(s_step + (a.step_mma ? L::step_bytes(n_ntiles) : 0));
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;   // [2]
    uint64_t *tempty = tfull + 2;  // [2]
    uint64_t *bfull = tempty + 2;  // resident-B arrival
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bfull + 1);
    float2 *s_st =
        reinterpret_cast<float2 *>(smem_raw + ((smem_addr(tmem_slot + 1) - smem_addr(smem_raw) + 15u) & ~15u));
    uint32_t *s_pos = reinterpret_cast<uint32_t *>(s_st + (a.K + 31) / 32 * 32);
    uint32_t *s_bits = s_pos + (a.K + 31) / 32;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_xy = a.ntx * a.nty;
    // scheduling unit = one CTA, or one CTA pair owning M tiles (2u, 2u + 1) (rank r takes 2u + r)
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    const int unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int nunits = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    const int total = (PAIR ? (a.n_mtiles + 1) / 2 : a.n_mtiles) * n_ntiles;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], PAIR ? 2 * kBlkEpiWarps : kBlkEpiWarps);  // one arrive per epilogue warp (of both CTAs)
        }
        mbar_init(bfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        if constexpr (PAIR) {  // same warp in both CTAs
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                         "r"(L::TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                         "r"(L::TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    pdl_wait();  // everything above overlaps the previous launch; every global read comes after
    if (warp >= 2) {  // all thresholds / direction words of the layer, once per CTA
        const int kpad = (a.K + 31) / 32 * 32;
        for (int i = threadIdx.x - 64; i < kpad / 32; i += 32 * kBlkEpiWarps) s_pos[i] = a.pos ? __ldg(a.pos + i) : 0u;
        for (int i = threadIdx.x - 64; i < kpad; i += 32 * kBlkEpiWarps) {
            const bool ok = a.thr && a.pos && i < a.K;
            // T clamped to +-(kred + 1) decides every sum the same way -- and is what the step rows hold
            const int kred = a.nks * KC * 2;
            reinterpret_cast<float *>(s_st)[i] =
                step_const(ok ? max(-kred - 1, min(kred + 1, __ldg(a.thr + i))) : 0,
                           ok ? ((__ldg(a.pos + (i >> 5)) >> (i & 31)) & 1u) : true);
        }
        if (a.step_mma) {  // the constant A block of the step MMA (read by the tensor core: async proxy)
            for (int i = threadIdx.x - 64; i < kStepA / 16; i += 32 * kBlkEpiWarps)
                reinterpret_cast<uint4 *>(s_step)[i] = make_uint4(0x77777777u, 0x77777777u, 0x77777777u, 0x11111111u);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t tmem_sfa = tmem_base + L::ACC_COLS, tmem_sfb = tmem_sfa + 16;
    if (warp >= 2 && warp < 6) tmem_fill_sf(tmem_sfa, 32, warp);  // unit scales, one lane quarter per warp
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) cluster_sync();  // the peer's barriers and scale factors are ready
    tc_fence_after();

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            if (a.bres || a.step_mma) {  // resident operands, loaded once per CTA
                mbar_expect_tx(bfull, (uint32_t)(a.nks * a.bres) * L::B_BYTES + (a.step_mma ? n_ntiles * BN * 32u : 0u));
                // the whole filter bank (every N tile)
                for (int nt = 0; nt < a.bres; ++nt)
                    for (int ks = 0; ks < a.nks; ++ks)
                        tma_load_2d(sB + (nt * a.nks + ks) * L::B_BYTES, &tmB, bfull, ks * KC, nt * BN);
                if (a.step_mma)
                    for (int nt = 0; nt < n_ntiles; ++nt)
                        tma_load_2d(s_step + kStepA + nt * BN * 32, &tmS, bfull, 0, nt * BN);
            }
            // The producer is a single thread: keep its per-stage work to table lookups.
            // PAIR: both CTAs' loads complete on the LEADER's full barrier, which expects both
            const uint32_t tx_bytes = (PAIR ? 2 : 1) * TPS * (a.a_bytes + (a.bres ? 0 : L::B_BYTES));
            uint32_t s = 0, round_par = 1;  // round_par = parity to wait on empty[s]
            int tn = 0;
            int m = unit / n_ntiles, nt = unit % n_ntiles;  // m counts the unit's M tiles
            const int m_step = nunits / n_ntiles, n_step = nunits % n_ntiles;
            for (int t = unit; t < total; t += nunits) {
                const int n0 = nt * BN + (PAIR ? (int)rank * (BN / 2) : 0);  // PAIR: this CTA's half of the B tile
                const int mm = PAIR ? 2 * m + (int)rank : m;
                const int tb = fdiv(mm, a.md_txy), rem = mm - tb * tiles_xy;
                const int ty = fdiv(rem, a.md_ntx);
                const int x0 = (rem - ty * a.ntx) * a.BW, y0 = ty * a.BH, b0 = tb * a.BB;
                int cc = 0, dx = a.T == 9 ? -1 : 0, dy = a.T == 9 ? -1 : 0;
                for (int ks = 0; ks < a.nks; ks += TPS, ++tn) {
                    TC_TRACE(0, tn, 0, clock64());
                    mbar_wait(&empty[s], round_par);
                    TC_TRACE(0, tn, 1, clock64());
                    const uint32_t fbar = PAIR ? mapa_shared(&full[s], 0) : 0u;
                    if (!PAIR || rank == 0) mbar_expect_tx(&full[s], tx_bytes);
#pragma unroll
                    for (int tt = 0; tt < TPS; ++tt) {
                        if constexpr (PAIR) {
                            tma_load_4d_pair(sA + (s * TPS + tt) * L::A_BYTES, &tmA, fbar, cc * KC, x0 + dx, y0 + dy, b0);
                            tma_load_2d_pair(sB + (s * TPS + tt) * L::B_BYTES, &tmB, fbar, (ks + tt) * KC, n0);
                        } else {
                            tma_load_4d(sA + (s * TPS + tt) * L::A_BYTES, &tmA, &full[s], cc * KC, x0 + dx, y0 + dy, b0);
                            if (!a.bres) tma_load_2d(sB + (s * TPS + tt) * L::B_BYTES, &tmB, &full[s], (ks + tt) * KC, n0);
                        }
                        if (++cc == a.CCH) {  // next tap (dy, dx) in row-major order
                            cc = 0;
                            if (a.T == 9 && ++dx == 2) {
                                dx = -1;
                                ++dy;
                            }
                        }
                    }
                    TC_TRACE(0, tn, 2, clock64());
                    if (++s == S) {
                        s = 0;
                        round_par ^= 1;
                    }
                }
                // advance (m, nt) by nunits tiles without a division per tile
                nt += n_step;
                m += m_step;
                if (nt >= n_ntiles) {
                    nt -= n_ntiles;
                    ++m;
                }
            }
        }
    } else if (warp == 1) {
        if (!PAIR || rank == 0) {  // ---------------- MMA issuer (whole warp, one elected lane issues; PAIR: leader)
            if (a.bres || a.step_mma) mbar_wait(bfull, 0);
            uint32_t lt = 0, s = 0, par = 0;
            // descriptors are additive in their start-address field: build once, offset per MMA
            const uint64_t adesc0 = umma_desc(smem_addr(sA), KC), bdesc0 = umma_desc(smem_addr(sB), KC);
            const uint64_t sdesc_a = umma_desc(smem_addr(s_step), 32), sdesc_b = umma_desc(smem_addr(s_step + kStepA), 32);
            int tn = 0;
            // N tile of t advanced without a division: an integer modulo on this path sits between
            // the accumulator hand-back and the first MMA of the next tile
            int nt = unit % n_ntiles;
            const int nt_step = nunits % n_ntiles;
            for (int t = unit; t < total; t += nunits, ++lt) {
                const uint32_t acc = lt % L::NACC, aph = (lt / L::NACC) & 1;
                const uint32_t b_base = a.bres ? (uint32_t)(nt * a.nks) : 0u;  // resident bank of this N tile
                const uint64_t sdesc = sdesc_b + (((uint32_t)nt * BN * 32) >> 4);
                if (lane == 0) TC_TRACE(2, lt, 0, clock64());
                mbar_wait(&tempty[acc], aph ^ 1);  // PAIR: both CTAs' epilogues (remote arrivals)
                tc_fence_after();
                if (lane == 0) TC_TRACE(2, lt, 1, clock64());
                const uint32_t tmem_d = tmem_base + acc * BN;
                if (a.step_mma)  // D = c first (its operands are resident); every tap accumulates on top
                    umma_f4_elect(tmem_d, sdesc_a, sdesc, a.idesc, false, tmem_sfa, tmem_sfb);
                if ((nt += nt_step) >= n_ntiles) nt -= n_ntiles;
                for (int ks = 0; ks < a.nks; ks += TPS, ++tn) {
                    if (lane == 0) TC_TRACE(1, tn, 0, clock64());
                    mbar_wait(&full[s], par);
                    tc_fence_after();
                    if (lane == 0) TC_TRACE(1, tn, 1, clock64());
                    {  // TPS boxes x KC / 32 K-chunks of this stage in one issue block
                        const uint64_t a0 = adesc0 + ((s * TPS * L::A_BYTES) >> 4);
                        const uint64_t b0 =
                            bdesc0 + (((a.bres ? b_base + (uint32_t)ks : (uint32_t)(s * TPS)) * L::B_BYTES) >> 4);
                        umma_f4_multi<TPS, KC / 32, L::A_BYTES / 16, L::B_BYTES / 16, PAIR ? 2 : 1>(
                            tmem_d, a0, b0, a.idesc, (PAIR ? false : a.step_mma) || ks != 0, tmem_sfa, tmem_sfb);
                    }
                    if constexpr (PAIR)
                        umma_commit_pair_elect(&empty[s]);  // the stage is free in both CTAs
                    else
                        umma_commit_elect(&empty[s]);
                    if (lane == 0) TC_TRACE(1, tn, 2, clock64());
                    if (++s == S) {
                        s = 0;
                        par ^= 1;
                    }
                }
                if constexpr (PAIR)
                    umma_commit_pair_elect(&tfull[acc]);
                else
                    umma_commit_elect(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {  // ------------------------- epilogue (warps 2..9)
        // TMEM lane quarter = warp % 4 (hardware rule); the two warps sharing a quarter split
        // the 32-column chunks round-robin (group g takes chunks g, g + 4, ...).
        constexpr int NG = kBlkEpiWarps / 4;
        const int q = warp & 3, half = (warp - 2) >> 2;  // half = column group 0..NG-1
        const int m_row = q * 32 + lane;  // tile row == TMEM lane
        const int npix = a.BW * a.BH * a.BB;
        const int bx = m_row % a.BW, by = (m_row / a.BW) % a.BH, bb = m_row / (a.BW * a.BH);
        const int Ho = a.pool ? a.H / 2 : a.H, Wo = a.pool ? a.W / 2 : a.W;
        const int KW = (a.K + 31) / 32;
        const bool logits = a.out_fmt == 2;
        const int j0 = logits ? 0 : half, jstep = logits ? 1 : NG;
        const bool active_warp = !logits || half == 0;
        // PAIR: the accumulator hand-back goes to the leader's barrier
        const uint32_t tempty_leader = PAIR ? mapa_shared(&tempty[0], 0) : 0u;
        auto release_acc = [&](uint32_t acc) {
            if (lane != 0) return;
            if (PAIR && rank != 0)
                mbar_arrive_cluster(tempty_leader + acc * 8u);
            else
                mbar_arrive(&tempty[acc]);
        };
        uint32_t lt = 0;
        for (int t = unit; t < total; t += nunits, ++lt) {
            const uint32_t acc = lt % L::NACC, aph = (lt / L::NACC) & 1;
            const int tq = fdiv(t, a.md_nnt), n0 = (t - tq * n_ntiles) * BN;
            const int m = PAIR ? 2 * tq + (int)rank : tq;
            const int tb = fdiv(m, a.md_txy), rem = m - tb * tiles_xy, ty = fdiv(rem, a.md_ntx);
            const int gx = (rem - ty * a.ntx) * a.BW + bx, gy = ty * a.BH + by, gb = tb * a.BB + bb;
            const bool inb = m_row < npix && gx < a.W && gy < a.H && gb < a.B;
            const uint32_t trow = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
            if (threadIdx.x == 64) TC_TRACE(3, lt, 0, clock64());
            mbar_wait(&tfull[acc], aph);
            if (threadIdx.x == 64) TC_TRACE(3, lt, 1, clock64());
            tc_fence_after();
            uint8_t *stage = s_out + (size_t)(lt & 1) * a.out_rows * (BN / 2);
            auto staging_free = [&]() {
                if (a.tma_out && threadIdx.x == 64) tma_store_wait_read<1>();  // this buffer's store (2 tiles ago) read out
                if (a.pool || a.tma_out)
                    asm volatile("bar.sync 1, %0;" ::"n"(32 * kBlkEpiWarps) : "memory");  // exchange / staging free
            };
            int best = 0, bestv = 0;
            // one 32-column chunk: sums, logits + argmax, or step -> bits (smem for pooling) / output
            if constexpr (L::NACC == 1) {
                // single accumulator: drain this warp's columns into registers and release TMEM to the
                // MMA warp before anything else (the MMA of the next tile waits on it), then threshold /
                // store from registers
                constexpr int NCH = BN / 32 >= NG ? BN / 32 / NG : 1;
                uint32_t vv[NCH][32];
#pragma unroll
                for (int c = 0; c < NCH; ++c) TMEM_LD32(trow + (half + NG * c) * 32, vv[c]);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                release_acc(acc);
                if (threadIdx.x == 64) TC_TRACE(3, lt, 3, clock64());
                staging_free();
                // Common case as straight-line code over all NCH chunks, so the scheduler can overlap
                // their latencies (the general per-chunk path branches on every mode flag, which
                // serialises the chunks: with 2 epilogue warps per scheduler that is what bounds it)
                const bool fast = !a.sums && !logits && n0 + BN <= a.K && (a.pool || (a.out_fmt == 1 && a.tma_out));
                if (fast) {
                    if (!a.step_mma) {
#pragma unroll
                        for (int c = 0; c < NCH; ++c)
                            step32c(vv[c], reinterpret_cast<const float *>(s_st) + n0 + (half + NG * c) * 32);
                    }
                    if (a.pool) {
#pragma unroll
                        for (int c = 0; c < NCH; ++c) s_bits[m_row * (BN / 32) + half + NG * c] = sgn32_bits(vv[c]);
                    } else {
#pragma unroll
                        for (int c = 0; c < NCH; ++c)
                            *reinterpret_cast<uint4 *>(stage + sw_chunk_off((uint32_t)m_row, (uint32_t)(half + NG * c), BN / 2)) =
                                sgn32_f4(vv[c]);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
                        tc_chunk<BN>(a, vv[c], half + NG * c, n0, inb, logits, gb, gy, gx, m_row, KW,
                                     reinterpret_cast<const float *>(s_st), s_pos, s_bits, best, bestv, stage);
                }
            } else {
                staging_free();
                if (active_warp) {
#pragma unroll 1
                    for (int j = j0; j < BN / 32; j += jstep) {
                        uint32_t v[32];
                        TMEM_LD32(trow + j * 32, v);
                        tmem_wait_ld();
                        tc_chunk<BN>(a, v, j, n0, inb, logits, gb, gy, gx, m_row, KW,
                                     reinterpret_cast<const float *>(s_st), s_pos, s_bits, best, bestv, stage);
                    }
                }
                // accumulator drained: hand TMEM buffer `acc` back to the MMA warp
                tc_fence_before();
                __syncwarp();
                release_acc(acc);
            }
            if (threadIdx.x == 64) TC_TRACE(3, lt, 2, clock64());
            if (logits) {
                if (half == 0 && inb && a.preds) a.preds[gb] = best;
            } else if (a.pool) {
                asm volatile("bar.sync 1, %0;" ::"n"(32 * kBlkEpiWarps) : "memory");  // all rows of the tile written
                if (a.out && inb && !(bx & 1) && !(by & 1)) {
                    const long long opix = ((long long)gb * Ho + gy / 2) * Wo + gx / 2;
                    // pooled pixel index inside the tile (tiles cover whole rows: BW == W)
                    const int prow = ((bb * a.BH + by) / 2) * (a.BW / 2) + bx / 2;
                    const int st = BN / 32;
#pragma unroll 1
                    for (int j = half; j < BN / 32; j += NG) {
                        const int nb = n0 + j * 32;
                        if (nb >= a.K) break;
                        const uint32_t p0 = s_bits[m_row * st + j], p1 = s_bits[(m_row + 1) * st + j];
                        const uint32_t p2 = s_bits[(m_row + a.BW) * st + j], p3 = s_bits[(m_row + a.BW + 1) * st + j];
                        const uint32_t pw = s_pos[nb >> 5];
                        const uint32_t pb = ((p0 | p1 | p2 | p3) & pw) | ((p0 & p1 & p2 & p3) & ~pw);
                        if (a.tma_out)
                            *reinterpret_cast<uint4 *>(stage + sw_chunk_off((uint32_t)prow, (uint32_t)j, BN / 2)) =
                                bits_to_f4(pb);
                        else
                            store_word(a, opix, nb, pb, KW);
                    }
                }
            }
            if (a.tma_out) {  // the whole tile's output: one TMA store from the staging buffer
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 1, %0;" ::"n"(32 * kBlkEpiWarps) : "memory");
                if (threadIdx.x == 64) {
                    const int tb = fdiv(m, a.md_txy), rem = m - tb * tiles_xy;
                    const int y0 = fdiv(rem, a.md_ntx) * a.BH, b0 = tb * a.BB;
                    const long long p0 = a.pool ? ((long long)b0 * Ho + y0 / 2) * Wo : ((long long)b0 * a.H + y0) * a.W;
                    tma_store_2d(&tmO, stage, n0 / 2, (int)p0);
                    tma_store_commit();
                }
            }
        }
    }
    if (a.tma_out && threadIdx.x == 64) tma_store_wait_all();
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) cluster_sync();  // no MMA, commit or remote arrive is still in flight to either CTA
    if (warp == 1) {
        tc_fence_after();
        if constexpr (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(L::TMEM_COLS));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(L::TMEM_COLS));
    }
}

// ------------------------------------------------------------------ halo-reuse conv (one TMA box per tile)
// For layers whose filter bank fits in shared memory (resident B), the A operand of all nine
// taps comes from ONE halo box per (tile, channel chunk): (RH+2) input rows x (W+2) columns,
// loaded with the x = -1 / y = -1 corner so TMA zero-fills the borders.  Output pixels are
// numbered in "padded-linear" order m = r*(W+2) + xo (xo = W, W+1 are junk columns), so tap
// (dy,dx) is the same halo buffer read from row m + dy*(W+2) + dx: nine UMMA descriptors whose
// start addresses differ by whole 64/128-B rows (verified exact with base_offset 0 for SW64 and
// SW128 on B200: profiles/r1_desc_shift_test.json).  L2->smem traffic drops ~9x versus one box
// per tap, which is what bounded the 64-channel layers.
template <int BN, int KC, int S, int MB>
struct HaloSmem {
    static constexpr int B_BYTES = BN * KC;
    static constexpr int BITS_WORDS = MB * 128 * (BN / 32);
    static constexpr int NACC = 2 * MB * BN + 32 <= 512 ? 2 : 1;  // + 32 scale-factor columns
    static constexpr int ACC_COLS = NACC * MB * BN;
    static constexpr int TMEM_COLS = tmem_pow2(ACC_COLS + 32);
    __host__ __device__ static size_t a_stage(int wp) { return ((size_t)(MB * 128 + 2 * wp + 2) * KC + 1023) / 1024 * 1024; }
    static size_t total(int nks, int K, int wp) {
        const size_t kpad = (size_t)(K + 31) / 32 * 32;
        return 1024 + (size_t)S * a_stage(wp) + (size_t)nks * B_BYTES + (2 * S + 5) * 8 + 32 + kpad * 8 + kpad / 8 +
               (size_t)BITS_WORDS * 4 + 16;
    }
};

// One 32-column chunk of the halo epilogue (debug sums, step -> bits for pooling / output).
template <int ST>
__device__ __forceinline__ void halo_chunk(const TcArgs &a, uint32_t (&v)[32], int j, bool inb, int b, int gy,
                                           int xo, long long pix, int m_row, int KW, const float *s_c,
                                           const uint32_t *s_pos,
                                           uint32_t *s_bits) {
    const int nb = j * 32;
    if (a.sums && inb) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (nb + i < a.K)
                a.sums[(((long long)b * a.K + nb + i) * a.H + gy) * a.W + xo] =
                    unfold_acc(v[i], a.thr != nullptr && ((s_pos[(nb + i) >> 5] >> ((nb + i) & 31)) & 1u));
    }
    if (nb >= a.K) {
        if (a.pool) s_bits[m_row * ST + j] = 0u;
        return;
    }
    step32c(v, s_c + nb);
    if (!a.pool && a.out_fmt == 1) {
        if (a.out && inb)
            *reinterpret_cast<uint4 *>(static_cast<uint8_t *>(a.out) + ((pix * a.K + nb) >> 1)) = sgn32_f4(v);
        return;
    }
    uint32_t bits = sgn32_bits(v);
    if (nb + 32 > a.K) bits &= 0xffffffffu >> (32 - (a.K - nb));
    if (a.pool)
        s_bits[m_row * ST + j] = bits;
    else if (a.out && inb)
        store_word(a, pix, nb, bits, KW);
}

template <int BN, int KC, int S, int MB>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_halo_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const TcArgs a) {
    pdl_trigger();
    using L = HaloSmem<BN, KC, S, MB>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    const int wp = a.W + 2;
    const int RH = a.BH;
    const uint32_t a_stage = (uint32_t)L::a_stage(wp);
    uint8_t *sA = smem;
    uint8_t *sB = smem + S * a_stage;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + (size_t)a.nks * L::B_BYTES);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint64_t *bfull = tempty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bfull + 1);
    float2 *s_st =
        reinterpret_cast<float2 *>(smem_raw + ((smem_addr(tmem_slot + 1) - smem_addr(smem_raw) + 15u) & ~15u));
    uint32_t *s_pos = reinterpret_cast<uint32_t *>(s_st + (a.K + 31) / 32 * 32);
    uint32_t *s_bits = s_pos + (a.K + 31) / 32;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_per_img = a.nty;
    const int total = a.n_mtiles;  // = B * tiles_per_img (single channel tile: K <= BN)

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8);
        }
        mbar_init(bfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                     "r"(L::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    pdl_wait();  // everything above overlaps the previous launch; every global read comes after
    if (warp >= 2) {
        const int kpad = (a.K + 31) / 32 * 32;
        for (int i = threadIdx.x - 64; i < kpad / 32; i += 256) s_pos[i] = a.pos ? __ldg(a.pos + i) : 0u;
        for (int i = threadIdx.x - 64; i < kpad; i += 256) {
            const bool ok = a.thr && a.pos && i < a.K;
            reinterpret_cast<float *>(s_st)[i] =
                step_const(ok ? __ldg(a.thr + i) : 0, ok ? ((__ldg(a.pos + (i >> 5)) >> (i & 31)) & 1u) : true);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t tmem_sfa = tmem_base + L::ACC_COLS, tmem_sfb = tmem_sfa + 16;
    if (warp >= 2 && warp < 6) tmem_fill_sf(tmem_sfa, 32, warp);  // unit scales, one lane quarter per warp
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t box_bytes = (uint32_t)(RH + 2) * wp * KC;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer: resident filters, then one halo box per (tile, chunk)
            mbar_expect_tx(bfull, (uint32_t)a.nks * L::B_BYTES);
            for (int ks = 0; ks < a.nks; ++ks) tma_load_2d(sB + ks * L::B_BYTES, &tmB, bfull, ks * KC, 0);
            uint32_t s = 0, par = 1;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                const int b = t / tiles_per_img, y0 = (t % tiles_per_img) * RH;
                for (int cc = 0; cc < a.CCH; ++cc) {
                    mbar_wait(&empty[s], par);
                    mbar_expect_tx(&full[s], box_bytes);
                    tma_load_4d(sA + s * a_stage, &tmA, &full[s], cc * KC, -1, y0 - 1, b);
                    if (++s == S) {
                        s = 0;
                        par ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        {  // ---------------- MMA issuer: 9 shifted descriptors per halo stage (whole warp, elected issue)
            mbar_wait(bfull, 0);
            uint32_t lt = 0, s = 0, par = 0;
            const uint64_t adesc0 = umma_desc(smem_addr(sA), KC), bdesc0 = umma_desc(smem_addr(sB), KC);
            const uint32_t row16 = KC >> 4;  // one K-major row in descriptor units
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
                const uint32_t acc = lt % L::NACC, aph = (lt / L::NACC) & 1;
                mbar_wait(&tempty[acc], aph ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * (MB * BN);
                for (int cc = 0; cc < a.CCH; ++cc) {
                    mbar_wait(&full[s], par);
                    tc_fence_after();
                    const uint64_t ad_s = adesc0 + ((s * a_stage) >> 4);
#pragma unroll
                    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                        for (int dx = 0; dx < 3; ++dx) {
                            const int tap = dy * 3 + dx;
                            const uint64_t ad = ad_s + (uint32_t)(dy * wp + dx) * row16;
                            const uint64_t bd = bdesc0 + (((uint32_t)(tap * a.CCH + cc) * L::B_BYTES) >> 4);
#pragma unroll
                            for (int mb = 0; mb < MB; ++mb)
#pragma unroll
                                for (int k = 0; k < KC / 32; ++k)
                                    umma_f4_elect(tmem_d + mb * BN, ad + (uint32_t)mb * 128 * row16 + 2 * k, bd + 2 * k,
                                                  a.idesc, (cc | tap | k) != 0, tmem_sfa, tmem_sfb);
                        }
                    umma_commit_elect(&empty[s]);
                    if (++s == S) {
                        s = 0;
                        par ^= 1;
                    }
                }
                umma_commit_elect(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {  // ------------------------- epilogue (warps 2..9)
        const int q = warp & 3, half = (warp - 2) >> 2;
        // MB == 2: each half takes one 128-row M block (all chunks); MB == 1: halves split the chunks
        const int mb = MB == 2 ? half : 0;
        const int j0 = MB == 2 ? 0 : half, jstep = MB == 2 ? 1 : 2;
        const int m_row = mb * 128 + q * 32 + lane;  // padded-linear tile row
        const int r = m_row / wp, xo = m_row % wp;
        const int Ho = a.pool ? a.H / 2 : a.H, Wo = a.pool ? a.W / 2 : a.W;
        const int KW = (a.K + 31) / 32;
        constexpr int ST = BN / 32;
        uint32_t lt = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
            const uint32_t acc = lt % L::NACC, aph = (lt / L::NACC) & 1;
            const int b = t / tiles_per_img, y0 = (t % tiles_per_img) * RH;
            const int gy = y0 + r;
            const bool inb = r < RH && xo < a.W && gy < a.H;
            const uint32_t trow = tmem_base + acc * (MB * BN) + mb * BN + ((uint32_t)(q * 32) << 16);
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            if (a.pool) asm volatile("bar.sync 1, 256;" ::: "memory");
            const long long pix = ((long long)b * a.H + gy) * a.W + xo;
            if constexpr (L::NACC == 1) {
                // single accumulator: drain this warp's chunks, release TMEM at once, then process
                constexpr int NCH = MB == 2 ? ST : (ST >= 2 ? ST / 2 : 1);
                uint32_t vv[NCH][32];
#pragma unroll
                for (int c = 0; c < NCH; ++c)
                    if (j0 + c * jstep < ST) TMEM_LD32(trow + (j0 + c * jstep) * 32, vv[c]);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
#pragma unroll
                for (int c = 0; c < NCH; ++c)
                    if (j0 + c * jstep < ST)
                        halo_chunk<ST>(a, vv[c], j0 + c * jstep, inb, b, gy, xo, pix, m_row, KW,
                                       reinterpret_cast<const float *>(s_st), s_pos, s_bits);
            } else {
#pragma unroll 1
                for (int j = j0; j < ST; j += jstep) {
                    uint32_t v[32];
                    TMEM_LD32(trow + j * 32, v);
                    tmem_wait_ld();
                    halo_chunk<ST>(a, v, j, inb, b, gy, xo, pix, m_row, KW, reinterpret_cast<const float *>(s_st), s_pos,
                                   s_bits);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
            }
            if (a.pool) {
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (a.out && inb && !(r & 1) && !(xo & 1)) {
                    const long long opix = ((long long)b * Ho + gy / 2) * Wo + xo / 2;
#pragma unroll 1
                    for (int j = j0; j < ST; j += jstep) {
                        const int nb = j * 32;
                        if (nb >= a.K) break;
                        const uint32_t p0 = s_bits[m_row * ST + j], p1 = s_bits[(m_row + 1) * ST + j];
                        const uint32_t p2 = s_bits[(m_row + wp) * ST + j], p3 = s_bits[(m_row + wp + 1) * ST + j];
                        const uint32_t pw = s_pos[nb >> 5];
                        store_word(a, opix, nb, ((p0 | p1 | p2 | p3) & pw) | ((p0 & p1 & p2 & p3) & ~pw), KW);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(L::TMEM_COLS));
    }
}

// ------------------------------------------------------------------ first layer on the tensor cores (design note)
// conv_int_forward (layers.py:91-101): u8 pixels x +-1 filters.  The reduction is only
// 9*C <= 64 taps, so each 128-pixel tile is ONE or two tcgen05.mma kind::i8 (A unsigned u8,
// B signed s8, K = 32 per instruction).  128 gather threads build their pixel's im2col row
// (taps in (c, dy, dx) order, zero-padded; out-of-image taps read the zero halo) in the
// canonical no-swizzle K-major layout ([row/8][k16][row%8][16 B]); the filters are staged
// once per CTA in the same layout.  Epilogue = the tc_block epilogue (threshold, pool, pack).
// ------------------------------------------------------------------ first layer, warp-specialised pipeline
// The phases of consecutive tiles overlap:
//   w0      : halo loader   (u8 NCHW rows -> smem halo stage, SH-deep ring)
//   w1      : TMEM owner + MMA issuer (one or two K=32 kind::i8 MMAs per tile, A unsigned)
//   w2..w5  : im2col gather (thread = tile row; SA-deep ring of A tiles, generic->async proxy fence)
//   w6..w9  : epilogue (TMEM lane quarter = warp % 4; double-buffered accumulator)
constexpr int kFirstWsThreads = 448;  // w0 loader, w1 MMA, w2..5 gather, w6..13 epilogue

template <int NP, int KB, int SH, int SA>
__global__ void __launch_bounds__(kFirstWsThreads, 1) conv_first_ws_kernel(const uint8_t *__restrict__ x,
                                                                            const int8_t *__restrict__ w,
                                                                            const TcArgs a, int C) {
    pdl_trigger();
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    constexpr int ROWB = KB * 32;                 // bytes per im2col row
    constexpr int SBO = 2 * KB * 128;             // no-swizzle K-major: 8-row group stride
    const int taps = 9 * C;
    const int hp = a.BH + 2, wpp = (a.W + 8 + 3) & ~3;
    const int halo_bytes = (a.BB * C * hp * wpp + 15) & ~15;
    uint8_t *sA = smem;                                   // SA x 128 x ROWB
    uint8_t *sB = sA + SA * 128 * ROWB;                   // NP x ROWB
    uint8_t *sH = sB + NP * ROWB;                         // SH halo stages
    uint64_t *hfull = reinterpret_cast<uint64_t *>(sH + SH * halo_bytes);
    uint64_t *hempty = hfull + SH;
    uint64_t *afull = hempty + SH;
    uint64_t *aempty = afull + SA;
    uint64_t *tfull = aempty + SA;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    int2 *s_st = reinterpret_cast<int2 *>(smem_raw + ((smem_addr(tmem_slot + 1) - smem_addr(smem_raw) + 15u) & ~15u));
    uint32_t *s_pos = reinterpret_cast<uint32_t *>(s_st + NP);       // NP/32
    uint32_t *s_bits = s_pos + NP / 32;                              // 128 * NP/32
    int16_t *s_toff = reinterpret_cast<int16_t *>(s_bits + 128 * (NP / 32));
    uint32_t *s_tmask = reinterpret_cast<uint32_t *>(s_toff + 64);
    int4 *s_items =  // halo word-copy items (wordcopy path), 16-B aligned
        reinterpret_cast<int4 *>(smem_raw + ((smem_addr(s_tmask + 16) - smem_addr(smem_raw) + 15u) & ~15u));

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < SH; ++i) {
            mbar_init(&hfull[i], 64);  // per lane: one async (cp.async completion) + one explicit arrival
            mbar_init(&hempty[i], 4);
        }
        for (int i = 0; i < SA; ++i) {
            mbar_init(&afull[i], 4);
            mbar_init(&aempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                     "r"(2 * NP));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    pdl_wait();  // everything above overlaps the previous launch; every global read comes after
    // filters in the no-swizzle K-major layout, thresholds, tap tables, zero halo pads
    for (int i = tid; i < NP * 2 * KB; i += kFirstWsThreads) {
        const int n = i / (2 * KB), h = i % (2 * KB);
        uint32_t wd[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t word = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int tap = h * 16 + q * 4 + b;
                const uint32_t v = (n < a.K && tap < taps) ? (uint8_t)w[(long long)n * taps + tap] : 0u;
                word |= v << (8 * b);
            }
            wd[q] = word;
        }
        *reinterpret_cast<uint4 *>(sB + (n / 8) * SBO + h * 128 + (n % 8) * 16) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
    for (int i = tid; i < NP; i += kFirstWsThreads) {
        const bool ok = a.thr && a.pos && i < a.K;
        s_st[i] = step_pair(ok ? __ldg(a.thr + i) : 0, ok ? ((__ldg(a.pos + (i >> 5)) >> (i & 31)) & 1u) : true);
    }
    for (int i = tid; i < NP / 32; i += kFirstWsThreads) s_pos[i] = (a.pos && i * 32 < a.K) ? __ldg(a.pos + i) : 0u;
    for (int i = tid; i < 64; i += kFirstWsThreads) {
        const int c = i / 9, d = i % 9;
        s_toff[i] = i < taps ? (int16_t)(c * hp * wpp + (d / 3) * wpp + d % 3 + 3) : (int16_t)0;
    }
    for (int i = tid; i < 16; i += kFirstWsThreads) {
        uint32_t mk = 0;
        for (int b = 0; b < 4; ++b) mk |= (4 * i + b < taps ? 0xFFu : 0u) << (8 * b);
        s_tmask[i] = mk;
    }
    for (int i = tid; i < SH * halo_bytes / 4; i += kFirstWsThreads) reinterpret_cast<uint32_t *>(sH)[i] = 0u;
    const int wpr = a.W / 4;
    const int n_items = (a.W & 3) == 0 ? a.BB * C * hp * wpr : 0;
    for (int i = tid; i < n_items; i += kFirstWsThreads) {
        const int r = i / wpr, q4 = i - r * wpr;
        const int yy = r % hp, rc = r / hp;
        const int c = rc % C, ib = rc / C;
        s_items[i] = make_int4(((ib * C + c) * a.H + (yy - 1)) * a.W + 4 * q4, r * wpp + 4 + 4 * q4, yy, ib);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int tiles_xy = a.nty;
    const bool wordcopy = (a.W & 3) == 0;

    if (warp == 0) {  // ---------------- halo loader (whole warp)
        uint32_t s = 0, par = 1;
        for (int t = blockIdx.x; t < a.n_mtiles; t += gridDim.x) {
            const int y0 = (t % tiles_xy) * a.BH, b0 = (t / tiles_xy) * a.BB;
            mbar_wait(&hempty[s], par);
            uint8_t *stage = sH + s * halo_bytes;
            const int nrows = a.BB * C * hp;
            if (wordcopy) {
                // every (row, word) pair issued back to back as 4-byte cp.async; completion is signalled
                // to hfull asynchronously (cp.async.mbarrier.arrive.noinc), so the loader never stalls
                // on memory latency and runs up to SH tiles ahead
                // per-CTA item table: (source offset from the tile base, smem offset, halo row, image)
                const uint8_t *tile_src = x + ((long long)b0 * C * a.H + y0) * a.W;
                for (int i = lane; i < n_items; i += 32) {
                    const int4 it = s_items[i];
                    const int iy = y0 + it.z - 1;
                    uint32_t *dst = reinterpret_cast<uint32_t *>(stage + it.y);
                    if (iy >= 0 && iy < a.H && b0 + it.w < a.B) {
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)),
                                     "l"(tile_src + it.x)
                                     : "memory");
                    } else {
                        *dst = 0u;
                    }
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(&hfull[s]))
                             : "memory");
            } else {
                for (int i = lane; i < nrows * a.W; i += 32) {
                    const int r = i / a.W, col = i - r * a.W;
                    const int yy = r % hp, rc = r / hp;
                    const int c = rc % C, img = b0 + rc / C;
                    const int iy = y0 + yy - 1;
                    const bool ok = iy >= 0 && iy < a.H && img < a.B;
                    stage[r * wpp + 4 + col] = ok ? x[(((long long)img * C + c) * a.H + iy) * a.W + col] : (uint8_t)0;
                }
                mbar_arrive(&hfull[s]);  // stands in for the async arrival of the cp.async path
            }
            mbar_arrive(&hfull[s]);  // each lane releases its own generic (zero) stores
            if (++s == SH) {
                s = 0;
                par ^= 1;
            }
        }
    } else if (warp == 1) {  // ---------------- MMA issuer (whole warp, elected issue)
        {
            const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(NP >> 3) << 17) | ((128u >> 4) << 24);
            const uint64_t adesc0 = make_desc_noswz(smem_addr(sA), SBO), bdesc0 = make_desc_noswz(smem_addr(sB), SBO);
            uint32_t s = 0, par = 0, lt = 0;
            for (int t = blockIdx.x; t < a.n_mtiles; t += gridDim.x, ++lt) {
                const uint32_t acc = lt & 1, aph = (lt >> 1) & 1;
                mbar_wait(&afull[s], par);
                mbar_wait(&tempty[acc], aph ^ 1);
                tc_fence_after();
#pragma unroll
                for (int kb = 0; kb < KB; ++kb)
                    umma_i8_elect(tmem_base + acc * NP, adesc0 + ((s * 128 * ROWB + kb * 256) >> 4),
                                  bdesc0 + ((kb * 256) >> 4), idesc, kb != 0);
                umma_commit_elect(&aempty[s]);
                umma_commit_elect(&tfull[acc]);
                if (++s == SA) {
                    s = 0;
                    par ^= 1;
                }
            }
        }
        __syncwarp();
    } else if (warp < 6) {  // ---------------- im2col gather: thread = tile row
        const int m_row = tid - 64;
        const int bx = m_row % a.BW, by = (m_row / a.BW) % a.BH, bb = m_row / (a.BW * a.BH);
        const int rowoff = (bb * C) * hp * wpp + by * wpp + bx;
        int toff[32 * KB];
        uint32_t tmask[8 * KB];
#pragma unroll
        for (int i = 0; i < 32 * KB; ++i) toff[i] = s_toff[i] + rowoff;
#pragma unroll
        for (int i = 0; i < 8 * KB; ++i) tmask[i] = s_tmask[i];
        uint32_t hs = 0, hpar = 0, as = 0, apar = 1;
        for (int t = blockIdx.x; t < a.n_mtiles; t += gridDim.x) {
            mbar_wait(&hfull[hs], hpar);
            mbar_wait(&aempty[as], apar);
            const uint8_t *stage = sH + hs * halo_bytes;
            uint8_t *arow = sA + as * 128 * ROWB + (m_row / 8) * SBO + (m_row % 8) * 16;
#pragma unroll
            for (int h = 0; h < 2 * KB; ++h) {
                uint32_t wd[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t word = 0;
#pragma unroll
                    for (int b = 0; b < 4; ++b) word |= (uint32_t)stage[toff[h * 16 + q * 4 + b]] << (8 * b);
                    wd[q] = word & tmask[h * 4 + q];
                }
                *reinterpret_cast<uint4 *>(arow + h * 128) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&afull[as]);
                mbar_arrive(&hempty[hs]);
            }
            if (++hs == SH) {
                hs = 0;
                hpar ^= 1;
            }
            if (++as == SA) {
                as = 0;
                apar ^= 1;
            }
        }
    } else {  // ---------------- epilogue (warps 6..13): lane quarter = warp % 4, halves split the chunks
        const int q = warp & 3, half = (warp - 6) >> 2;
        const int m_row = q * 32 + lane;
        const int npix = a.BW * a.BH * a.BB;
        const int bx = m_row % a.BW, by = (m_row / a.BW) % a.BH, bb = m_row / (a.BW * a.BH);
        const int Ho = a.pool ? a.H / 2 : a.H, Wo = a.pool ? a.W / 2 : a.W;
        const int KW = (a.K + 31) / 32;
        uint32_t lt = 0;
        for (int t = blockIdx.x; t < a.n_mtiles; t += gridDim.x, ++lt) {
            const uint32_t acc = lt & 1, aph = (lt >> 1) & 1;
            const int y0 = (t % tiles_xy) * a.BH, b0 = (t / tiles_xy) * a.BB;
            const int gx = bx, gy = y0 + by, gb = b0 + bb;
            const bool inb = m_row < npix && gx < a.W && gy < a.H && gb < a.B;
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            if (a.pool) asm volatile("bar.sync 2, 256;" ::: "memory");
            const uint32_t trow = tmem_base + acc * NP + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
            for (int j = half; j < NP / 32; j += 2) {
                uint32_t v[32];
                TMEM_LD32(trow + j * 32, v);
                tmem_wait_ld();
                const int nb = j * 32;
                if (a.sums && inb) {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (nb + i < a.K) a.sums[(((long long)gb * a.K + nb + i) * a.H + gy) * a.W + gx] = (int32_t)v[i];
                }
                uint32_t bits = 0;
                if (nb < a.K) {
                    bits = threshold32(v, s_st + nb);
                    if (nb + 32 > a.K) bits &= 0xffffffffu >> (32 - (a.K - nb));
                }
                if (a.pool) {
                    s_bits[m_row * (NP / 32) + j] = bits;
                } else if (a.out && inb && nb < a.K) {
                    store_word(a, ((long long)gb * a.H + gy) * a.W + gx, nb, bits, KW);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (a.pool) {
                asm volatile("bar.sync 2, 256;" ::: "memory");
                if (a.out && inb && !(bx & 1) && !(by & 1)) {
                    const long long opix = ((long long)gb * Ho + gy / 2) * Wo + gx / 2;
                    const int st = NP / 32;
                    for (int j = half; j < NP / 32; j += 2) {
                        const int nb = j * 32;
                        if (nb >= a.K) break;
                        const uint32_t p0 = s_bits[m_row * st + j], p1 = s_bits[(m_row + 1) * st + j];
                        const uint32_t p2 = s_bits[(m_row + a.BW) * st + j], p3 = s_bits[(m_row + a.BW + 1) * st + j];
                        const uint32_t pw = s_pos[j];
                        store_word(a, opix, nb, ((p0 | p1 | p2 | p3) & pw) | ((p0 & p1 & p2 & p3) & ~pw), KW);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * NP));
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
    const CUtensorMapSwizzle sw = row_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                    : CU_TENSOR_MAP_SWIZZLE_32B;
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


static int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 148;
    }
    return cached[dev];
}

template <int BN, int KC, int TPS, bool PAIR = false, bool HX = false>
static int launch_tc_s(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mo, const CUtensorMap &ms,
                       TcArgs &a, cudaStream_t st) {
    // stages: ~12-24 KB of A (+ B) in flight per stage, ~60-100 KB of ring
    constexpr int kRing = 160 * 1024;  // A + streamed-B bytes of the ring (worst case: B not resident)
    constexpr int kBRows = PAIR ? BN / 2 : BN;
    constexpr int kStage = TPS * (128 + kBRows) * KC;
    constexpr int S = KC == 32 ? (kRing / kStage > 14 ? 14 : (kRing / kStage < 2 ? 2 : kRing / kStage))
                               : (KC * (128 + kBRows) <= 24 * 1024) ? 7 : (KC * (128 + kBRows) <= 32 * 1024 ? 5 : 4);
    using L = TcSmem<BN, KC, S, TPS, PAIR>;
    constexpr size_t kLimit = 227 * 1024;
    const int n_ntiles = (a.K + BN - 1) / BN;
    a.bres = 0;
    const int orows = a.tma_out ? a.out_rows : 0;
    if (!PAIR && L::total(a.nks, n_ntiles, a.K, orows) <= kLimit) a.bres = n_ntiles;
    if (HX && !a.bres) return 1;  // HX needs the resident filter bank (the caller falls back)
    if (a.tma_out && L::total(a.nks, a.bres, a.K, orows) > kLimit) a.tma_out = 0;  // no room to stage
    // step MMA last: resident filters and the TMA store matter more
    if (a.step_mma && L::total(a.nks, a.bres, a.K, a.tma_out ? orows : 0, L::step_bytes(n_ntiles)) > kLimit) a.step_mma = 0;
    const size_t smem = L::total(a.nks, a.bres, a.K, a.tma_out ? orows : 0, a.step_mma ? L::step_bytes(n_ntiles) : 0);
    BNN_REQUIRE(smem <= kLimit, "tc_block: %zu B of shared memory needed", smem);
    a.md_txy = fdiv_magic((uint32_t)(a.ntx * a.nty));
    a.md_ntx = fdiv_magic((uint32_t)a.ntx);
    a.md_nnt = fdiv_magic((uint32_t)n_ntiles);
    void (*kern)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, TcArgs);
    if constexpr (PAIR)
        kern = tc_pair_kernel<BN, KC, S, TPS, true>;
    else
        kern = tc_block_kernel<BN, KC, S, TPS, HX>;
    int e = allow_smem(reinterpret_cast<const void *>(kern), smem, "tc_block");
    if (e) return e;
    if constexpr (PAIR) {  // clusters of 2 (one TPC): a CTA pair per unit of two M tiles
        const long long units = (long long)((a.n_mtiles + 1) / 2) * n_ntiles;
        const int grid = 2 * (int)std::min<long long>(units, sm_count() / 2);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kBlkThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl_on() ? 2 : 1;
        cudaLaunchKernelEx(&cfg, kern, ma, mb, mo, ms, a);
    } else {
        const long long tiles = (long long)a.n_mtiles * n_ntiles;
        const int grid = (int)std::min<long long>(tiles, sm_count());
        launch_kernel(kern, dim3(grid), dim3(kBlkThreads), smem, st, ma, mb, mo, ms, a);
    }
    count_launch();
    return after_launch("tc_block");
}

template <int BN, int KC>
static int launch_tc(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mo, const CUtensorMap &ms, TcArgs &a,
                     cudaStream_t st) {
    // thin chunks: several K-steps per stage (3 taps of a 64-channel conv; 7 chunks of e.g. the
    // 3,136-feature fashion FC = 49 chunks)
    if (KC == 32 && a.nks % 3 == 0) return launch_tc_s<BN, KC, 3>(ma, mb, mo, ms, a, st);
    if (KC == 32 && a.nks % 7 == 0) return launch_tc_s<BN, KC, 7>(ma, mb, mo, ms, a, st);
    if (KC == 32 && a.nks % 2 == 0) return launch_tc_s<BN, KC, 2>(ma, mb, mo, ms, a, st);
    return launch_tc_s<BN, KC, 1>(ma, mb, mo, ms, a, st);
}

template <int KC>
static int dispatch_bn(int bn, const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mo, const CUtensorMap &ms,
                       TcArgs &a, cudaStream_t st, bool pair, const CUtensorMap *ma_hx = nullptr) {
    if constexpr (KC == 32)
        if (ma_hx && bn == 256) {
            const int r = launch_tc_s<256, 32, 3, false, true>(*ma_hx, mb, mo, ms, a, st);
            if (r != 1) return r;  // 1 = not eligible after all: the per-tap kernel below
        }
    if constexpr (KC >= 64)
        if (pair) return bn == 256 ? launch_tc_s<256, KC, 1, true>(ma, mb, mo, ms, a, st)
                                   : launch_tc_s<128, KC, 1, true>(ma, mb, mo, ms, a, st);
    if constexpr (KC == 32)  // thin chunks (e.g. a 3,136-feature FC): several per stage, as launch_tc
        if (pair && bn == 256) {
            if (a.nks % 7 == 0) return launch_tc_s<256, 32, 7, true>(ma, mb, mo, ms, a, st);
            if (a.nks % 3 == 0) return launch_tc_s<256, 32, 3, true>(ma, mb, mo, ms, a, st);
            if (a.nks % 2 == 0) return launch_tc_s<256, 32, 2, true>(ma, mb, mo, ms, a, st);
            return launch_tc_s<256, 32, 1, true>(ma, mb, mo, ms, a, st);
        }
    switch (bn) {
        case 32: return launch_tc<32, KC>(ma, mb, mo, ms, a, st);
        case 64: return launch_tc<64, KC>(ma, mb, mo, ms, a, st);
        case 128: return launch_tc<128, KC>(ma, mb, mo, ms, a, st);
        default: return launch_tc<256, KC>(ma, mb, mo, ms, a, st);
    }
}

// Halo mode (see tc_halo_kernel).  Returns 1 if the shape is not eligible (caller falls back).
template <int BN, int KC, int MB>
static int launch_halo(const CUtensorMap &mb, const int8_t *x, TcArgs &a, cudaStream_t st) {
    constexpr int S = MB == 2 ? 4 : 3;
    using L = HaloSmem<BN, KC, S, MB>;
    const int wp = a.W + 2;
    const size_t smem = L::total(a.nks, a.K, wp);
    if (smem > 227 * 1024) return 1;
    CUtensorMap ma;
    const cuuint64_t CB = (cuuint64_t)a.CCH * KC;  // bytes per pixel
    const cuuint64_t adims[4] = {CB, (cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)a.B};
    const cuuint64_t astr[3] = {CB, (cuuint64_t)a.W * CB, (cuuint64_t)a.H * a.W * CB};
    const cuuint32_t abox[4] = {(cuuint32_t)KC, (cuuint32_t)wp, (cuuint32_t)(a.BH + 2), 1};
    int e = encode_map(&ma, x, 4, adims, astr, abox, KC);
    if (e) return e;
    auto kern = tc_halo_kernel<BN, KC, S, MB>;
    e = allow_smem(reinterpret_cast<const void *>(kern), smem, "tc_halo");
    if (e) return e;
    const int grid = (int)std::min<long long>(a.n_mtiles, sm_count());
    launch_kernel(kern, dim3(grid), dim3(kTcThreads), smem, st, ma, mb, a);
    count_launch();
    return after_launch("tc_halo");
}

static int try_halo(const int8_t *x, int B, int C, int H, int W, const int8_t *w, int K, int KC, int bn, int pool,
                    TcArgs a, cudaStream_t st, bool force) {
    if (K > bn || W + 2 > 256 || H < 1) return 1;
    const int CB = C / 2;                        // FP4: bytes per pixel
    const size_t b_bytes = (size_t)9 * CB * bn;  // resident filter bank
    if (b_bytes > 150 * 1024) return 1;
    // pick (MB, RH): most valid output pixels per MMA row, RH even when pooling
    const int wp = W + 2;
    int best_mb = 0, best_rh = 0;
    double best_eff = 0;
    for (int mb = 1; mb <= 2; ++mb) {
        if (mb * bn > 256) continue;  // accumulators (single-buffered above 240 columns) + scale factors
        for (int rh = 1; rh <= H && rh * wp <= mb * 128 && rh + 2 <= 256; ++rh) {
            if (pool && (rh & 1)) continue;
            const int tiles = (H + rh - 1) / rh;
            const double eff = (double)H * W / ((double)tiles * mb * 128);
            if (eff > best_eff + 1e-9) {
                best_eff = eff;
                best_mb = mb;
                best_rh = rh;
            }
        }
    }
    // Halo reuse pays when the A operand dominates the traffic (narrow N); for wide N the per-tap
    // kernel's full M tiles win unless the halo tiling wastes little (measured: profiles/).
    if (!best_mb || (!force && (best_eff < 0.45 || (bn > 64 && best_eff < 0.74)))) return 1;
    a.BH = best_rh;
    a.nty = (H + best_rh - 1) / best_rh;
    a.n_mtiles = B * a.nty;
    CUtensorMap mbm;
    const cuuint64_t bdims[2] = {(cuuint64_t)9 * CB, (cuuint64_t)K};
    const cuuint64_t bstr[1] = {(cuuint64_t)9 * CB};
    const cuuint32_t bbox[2] = {(cuuint32_t)KC, (cuuint32_t)bn};
    int e = encode_map(&mbm, w, 2, bdims, bstr, bbox, KC);
    if (e) return e;
#define BNN_HALO(BNV, KCV, MBV) return launch_halo<BNV, KCV, MBV>(mbm, x, a, st)
#define BNN_HALO_KC(KCV)                                  \
    if (best_mb == 1) {                                   \
        if (bn == 32) BNN_HALO(32, KCV, 1);               \
        if (bn == 64) BNN_HALO(64, KCV, 1);               \
        if (bn == 128) BNN_HALO(128, KCV, 1);             \
        BNN_HALO(256, KCV, 1);                            \
    } else {                                              \
        if (bn == 32) BNN_HALO(32, KCV, 2);               \
        if (bn == 64) BNN_HALO(64, KCV, 2);               \
        BNN_HALO(128, KCV, 2);                            \
    }
    if (KC == 32) {
        BNN_HALO_KC(32)
    } else if (KC == 64) {
        BNN_HALO_KC(64)
    } else {
        BNN_HALO_KC(128)
    }
#undef BNN_HALO_KC
#undef BNN_HALO
}

// Shared launcher: x is int8 NHWC (B, H, W, C) with C % 64 == 0; w is int8 (K, T*C) tap-major.
static int tc_run(const int8_t *x, int B, int C, int H, int W, int T, const int8_t *w, int K, const int32_t *thr,
                  const uint32_t *pos, int pool, int out_fmt, void *out, int32_t *sums, int32_t *preds,
                  int bn_req, cudaStream_t st, bool halo_ok = true, bool halo_force = false,
                  const uint8_t *step_rows = nullptr, bool pair_ok = true, bool hx_ok = false, int flags = 0) {
    BNN_REQUIRE(C % 64 == 0, "tensor engine needs C %% 64 == 0 (got %d)", C);
    BNN_REQUIRE(out_fmt != 1 || K % 32 == 0, "FP4 output needs K %% 32 == 0 (got %d)", K);
    const int CB = C / 2;  // FP4 operand bytes per pixel / row
    int KC = (CB % 128 == 0) ? 128 : (CB % 64 == 0) ? 64 : 32;  // bytes per K chunk (swizzle row)
    // FC rows (T == 1) longer than 128 B move in 128-B chunks even when the length is not a multiple:
    // the last chunk runs past the row on both operands and TMA zero-fills the out-of-bounds bytes (FP4
    // 0 x anything = 0), e.g. the fashion FC's 1,568-B rows: 13 chunks of 128 B instead of 49 of 32 B
    if (T == 1 && KC < 128 && CB > 128) KC = 128;
    TcArgs a{};
    a.T = T;
    a.CCH = (CB + KC - 1) / KC;
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
    a.n_mtiles = a.ntx * a.nty * ntb;
    BNN_REQUIRE(K <= kMaxK, "tensor engine supports K <= %d (got %d)", kMaxK, K);
    a.thr = thr; a.pos = pos; a.pool = pool; a.out_fmt = out_fmt; a.out = out; a.sums = sums; a.preds = preds;
    a.a_bytes = a.BW * a.BH * a.BB * KC;
    a.trace = g_tc_trace;
    a.early_weights = (flags & BNN_VARIANT_STATIC_WEIGHTS) != 0;
    int bn = bn_req;
    if (bn != 32 && bn != 64 && bn != 128 && bn != 256) bn = K <= 32 ? 32 : K <= 64 ? 64 : K <= 128 ? 128 : 256;
    if (out_fmt == 2) {
        if (bn < K || bn > 128) bn = K <= 32 ? 32 : K <= 64 ? 64 : 128;
        BNN_REQUIRE(K <= bn, "logits tile needs K <= 128 (K=%d)", K);
    }
    // CTA pairs (M = 256 per MMA, half of each B tile per CTA) when the B operand is streamed:
    // N = 128 / 256 tiles of a filter bank too large to stay resident.  With N = 128 the pair keeps
    // two accumulators per CTA (double-buffered TMEM) at the smem traffic per MAC of a single-CTA
    // N = 256 tile, which has room for one only.
    const bool pair = pair_ok && (bn == 256 || (bn == 128 && KC >= 64)) && out_fmt != 2 && !step_rows &&
                      (size_t)a.nks * bn * KC > (size_t)128 * 1024;
    a.idesc = idesc_f4(128, bn);

    if (T == 9 && halo_ok && out_fmt != 2) {
        const int r = try_halo(x, B, C, H, W, w, K, KC, bn, pool, a, st, halo_force);
        if (r != 1) return r;  // launched (0) or failed with an error; 1 = not eligible
    }
    if (pair) a.idesc = idesc_f4(256, bn);  // M = 256 across the CTA pair (never for the halo kernels)
    CUtensorMap ma, mb;
    const cuuint64_t adims[4] = {(cuuint64_t)CB, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    const cuuint64_t astr[3] = {(cuuint64_t)CB, (cuuint64_t)W * CB, (cuuint64_t)H * W * CB};
    const cuuint32_t abox[4] = {(cuuint32_t)KC, (cuuint32_t)a.BW, (cuuint32_t)a.BH, (cuuint32_t)a.BB};
    int e = encode_map(&ma, x, 4, adims, astr, abox, KC);
    if (e) return e;
    const cuuint64_t bdims[2] = {(cuuint64_t)T * CB, (cuuint64_t)K};
    const cuuint64_t bstr[1] = {(cuuint64_t)T * CB};
    const cuuint32_t bbox[2] = {(cuuint32_t)KC, (cuuint32_t)(pair ? bn / 2 : bn)};
    e = encode_map(&mb, w, 2, bdims, bstr, bbox, KC);
    if (e) return e;
    // TMA-store epilogue for FP4 outputs when every tile maps to consecutive output pixels (tiles
    // span whole image rows: BW == W and H % BH == 0, or FC rows)
    CUtensorMap mo;
    std::memset(&mo, 0, sizeof(mo));
    a.tma_out = 0;
    a.out_rows = pool ? a.BW * a.BH * a.BB / 4 : a.BW * a.BH * a.BB;
    if (out_fmt == 1 && out && (T == 1 || (a.BW == W && H % a.BH == 0)) && a.out_rows >= 8) {
        const int Ho = pool ? H / 2 : H, Wo = pool ? W / 2 : W;
        const cuuint64_t odims[2] = {(cuuint64_t)K / 2, (cuuint64_t)B * Ho * Wo};
        const cuuint64_t ostr[1] = {(cuuint64_t)K / 2};
        const cuuint32_t obox[2] = {(cuuint32_t)bn / 2, (cuuint32_t)a.out_rows};
        if (bn / 2 >= 32 && encode_map(&mo, out, 2, odims, ostr, obox, bn / 2) == 0) a.tma_out = 1;
    }
    // step rows (bnn_step_rows): the threshold constant enters through one extra MMA per tile
    CUtensorMap ms;
    std::memset(&ms, 0, sizeof(ms));
    a.step_mma = 0;
    if (step_rows && thr && pos && out_fmt != 2) {
        const cuuint64_t sdims[2] = {32, (cuuint64_t)K};
        const cuuint64_t sstr[1] = {32};
        const cuuint32_t sbox[2] = {32, (cuuint32_t)bn};
        e = encode_map(&ms, step_rows, 2, sdims, sstr, sbox, 32);
        if (e) return e;
        a.step_mma = 1;
    }
    // HX (halo along x) A boxes for 16-px rows of 32-B pixels (see tc_block_kernel)
    CUtensorMap ma_hx;
    const bool hx = hx_ok && T == 9 && KC == 32 && a.CCH == 1 && W == 16 && a.BW == 16 && a.BH == 8 && a.BB == 1 &&
                    bn == 256 && H % 8 == 0 && out_fmt != 2;
    if (hx) {
        const cuuint32_t hbox[4] = {(cuuint32_t)KC, 10u, 8u, 1u};
        e = encode_map(&ma_hx, x, 4, adims, astr, hbox, KC);
        if (e) return e;
    }
    return KC == 128 ? dispatch_bn<128>(bn, ma, mb, mo, ms, a, st, pair)
                     : KC == 64 ? dispatch_bn<64>(bn, ma, mb, mo, ms, a, st, pair)
                                : dispatch_bn<32>(bn, ma, mb, mo, ms, a, st, pair, hx ? &ma_hx : nullptr);
}

void tc_set_trace(unsigned long long *buf) { g_tc_trace = buf; }

int tc_conv(const int8_t *x, int B, int C, int H, int W, const int8_t *w, int K, const int32_t *thr,
            const uint32_t *pos, int pool, int out_fmt, void *out, int32_t *sums, int bn, int mode,
            const uint8_t *step_rows, int flags, cudaStream_t st) {
    // mode: 0 = auto (halo when its M-tiling efficiency is high enough), 1 = per-tap boxes only,
    // 2 = halo whenever it fits (the autotuner decides)
    // mode 5: per-tap boxes on single CTAs (no CTA pairs); mode 6: halo-along-x boxes (HX) where the
    // shape allows, else per-tap
    return tc_run(x, B, C, H, W, 9, w, K, thr, pos, pool, out_fmt, out, sums, nullptr, bn, st,
                  mode != 1 && mode != 3 && mode != 5 && mode != 6, mode == 2, step_rows, mode != 5 && mode != 6,
                  mode == 6, flags);
}

int tc_fc(const int8_t *x, int B, int L, const int8_t *w, int M, const int32_t *thr, const uint32_t *pos,
          int out_fmt, void *out, int32_t *sums, int32_t *preds, int bn, int mode, const uint8_t *step_rows,
          int flags, cudaStream_t st) {
    return tc_run(x, B, L, 1, 1, 1, w, M, thr, pos, 0, out_fmt, out, sums, preds, bn, st, true, false, step_rows, mode != 5,
                  false, flags);
}

}  // namespace bnn

namespace bnn {
int tc_first(const uint8_t *x, int B, int C, int H, int W, const int8_t *w, int K, const int32_t *thr,
             const uint32_t *pos, int pool, int out_fmt, void *out, int32_t *sums, cudaStream_t st) {
    BNN_REQUIRE(9 * C <= 64, "tensor first layer needs 9*C <= 64 (C=%d)", C);
    BNN_REQUIRE(K <= 256, "tensor first layer needs K <= 256 (K=%d)", K);
    BNN_REQUIRE(W <= 128, "tensor first layer needs W <= 128 (W=%d)", W);
    TcArgs a{};
    a.W = W; a.H = H; a.B = B; a.K = K;
    a.BW = W;
    int bh = 128 / W;
    if (bh > H) bh = H;
    if (pool && (bh & 1)) bh -= 1;
    a.BH = bh < 1 ? 1 : bh;
    a.BB = (a.BH == H) ? 128 / (a.BW * a.BH) : 1;
    if (a.BB > B) a.BB = B;
    if (a.BB < 1) a.BB = 1;
    a.ntx = 1;
    a.nty = ceil_div(H, a.BH);
    a.n_mtiles = a.nty * ceil_div(B, a.BB);
    a.thr = thr; a.pos = pos; a.pool = pool; a.out_fmt = out_fmt; a.out = out; a.sums = sums;
    const int KB = (9 * C + 31) / 32;
    const int np = K <= 32 ? 32 : K <= 64 ? 64 : K <= 128 ? 128 : 256;
    const size_t wpp = (size_t)((W + 8 + 3) & ~3);
    const size_t halo = ((size_t)a.BB * C * (a.BH + 2) * wpp + 15) & ~size_t(15);
    constexpr int SH = 3, SA = 2;
    const size_t n_items = (W % 4 == 0) ? (size_t)a.BB * C * (a.BH + 2) * (W / 4) : 0;
    const size_t smem = 1024 + (size_t)(SA * 128 + np) * KB * 32 + SH * halo + (2 * SH + 2 * SA + 4) * 8 + 32 + np * 8 +
                        np / 8 + 128 * (np / 32) * 4 + 128 + 64 + 16 + 16 + n_items * 16;
#define BNN_FIRST(NP, KBV)                                                                                        \
    {                                                                                                             \
        auto kern = conv_first_ws_kernel<NP, KBV, SH, SA>;                                                        \
        int e = allow_smem(reinterpret_cast<const void *>(kern), smem, "tc_first");                               \
        if (e) return e;                                                                                          \
        int per_sm = 1;                                                                                           \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFirstWsThreads, smem);                      \
        const int grid = (int)std::min<long long>(a.n_mtiles, (long long)sm_count() * (per_sm < 1 ? 1 : per_sm)); \
        launch_kernel(kern, dim3(grid), dim3(kFirstWsThreads), smem, st, x, w, a, C);                             \
    }
    if (KB == 1) {
        if (np == 32) BNN_FIRST(32, 1) else if (np == 64) BNN_FIRST(64, 1) else if (np == 128) BNN_FIRST(128, 1) else BNN_FIRST(256, 1)
    } else {
        if (np == 32) BNN_FIRST(32, 2) else if (np == 64) BNN_FIRST(64, 2) else if (np == 128) BNN_FIRST(128, 2) else BNN_FIRST(256, 2)
    }
#undef BNN_FIRST
    count_launch();
    return after_launch("tc_first");
}
}  // namespace bnn
