// tc_ptx.cuh -- PTX wrappers shared by the tcgen05 kernels (tc_gemm.cu, tc_front.cu):
// mbarriers (bounded waits), TMA loads, tcgen05 mma / commit / ld, UMMA smem descriptors,
// and the branch-free threshold + int8 +-1 expansion used by every epilogue.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace bnn {

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

// Bounded wait: a pipeline bug becomes a trap (cudaErrorLaunchFailure) after ~4 s of wall time,
// never a hung GPU.  (A try_wait suspend-time hint measured slightly slower: profiles/.)
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    uint64_t t0 = 0;
    for (uint32_t spins = 0;; ++spins) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if ((spins & 63) == 0) {
            const uint64_t now = global_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 4000000000ull) __trap();
        }
    }
}

// The same wait with a suspend-time hint: a waiting warp sleeps in the barrier unit until the phase
// completes (or the hint elapses) instead of re-issuing try_wait -- for waits that are usually long
// (epilogue warps waiting for their accumulator), so idle warps do not take issue slots.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    uint64_t t0 = 0;
    for (uint32_t spins = 0;; ++spins) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity), "r"(1000000u)
            : "memory");
        if (done) return;
        if ((spins & 63) == 0) {
            const uint64_t now = global_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 4000000000ull) __trap();
        }
    }
}

// The same wait with acquire at cluster scope: for barriers that CTAs of the cluster arrive on remotely
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    uint64_t t0 = 0;
    for (uint32_t spins = 0;; ++spins) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if ((spins & 63) == 0) {
            const uint64_t now = global_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 4000000000ull) __trap();
        }
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

// 1-D bulk copy global -> shared (size and both addresses 16-B multiples), completion on an mbarrier
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// TMA tensor store (shared -> global, bulk-group completion) and its group bookkeeping
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, const void *src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem_addr(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// byte offset of 16-B chunk `c` of row `r` in a K-major tile of `rb`-byte rows, TMA swizzle pattern
// matching the row width (SW128 / SW64 / SW32; 16-B rows unswizzled)
__device__ __forceinline__ uint32_t sw_chunk_off(uint32_t r, uint32_t c, int rb) {
    const uint32_t x = rb == 128 ? (r & 7u) : rb == 64 ? ((r >> 1) & 3u) : rb == 32 ? ((r >> 2) & 1u) : 0u;
    return r * (uint32_t)rb + ((c ^ x) << 4);
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

// Whole-warp issue helpers: every lane computes the (warp-uniform) descriptors, one elected
// lane issues -- lets the compiler keep descriptor arithmetic in uniform registers instead of
// shuffling them into uniform registers per MMA from a single divergent lane.
__device__ __forceinline__ void umma_i8_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Binary dot products on the FP4 tensor cores: +-1 operands as E2M1 codes, block-scaled MMA with
// every UE8M0 scale = 2^0 (TMEM scale-factor columns filled with 0x7F by tmem_fill_sf), fp32
// accumulation -- exact for |sum| < 2^24.  K = 64 per instruction (32 bytes per operand row).
__device__ __forceinline__ void umma_f4_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate, uint32_t tmem_sfa, uint32_t tmem_sfb) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tmem_sfa), "r"(tmem_sfb));
}

// The 9 taps of a 3x3 binary conv on the halo layout as ONE issue block: a single elect, then nine
// block-scaled K = 64 MMAs whose A descriptors are the tile's base shifted by dy * a_row + 2 * dx
// (16-B units: a_row = 2 * padded row width for 32-B rows) and whose B descriptors step by one
// 64-row x 32-B filter slab (2 KB) per tap.  All descriptor arithmetic is inside the block, so the
// issuing warp spends ~2 instructions per MMA instead of ~15 (R2UR / VOTEU / ELECT per call).
__device__ __forceinline__ void umma_f4_taps9(uint32_t tmem_d, uint64_t a0, uint32_t a_row, uint64_t b0,
                                              uint32_t idesc, uint32_t tmem_sfa, uint32_t tmem_sfb) {
#define BNN_TAP(AOFF, BOFF, ACC)                                                                         \
    "add.s64 a, %1, " AOFF ";\n\tadd.s64 b, %3, " BOFF ";\n\t"                                        \
    "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %4, [%5], [%6], " ACC ";\n\t"
    asm volatile(
        "{\n\t.reg .pred e, p0, p1;\n\t.reg .b64 a, b, r1, r2, r1b, r2b;\n\t"
        "setp.ne.b32 p0, 0, 0;\n\tsetp.eq.b32 p1, 0, 0;\n\t"
        "cvt.u64.u32 r1, %2;\n\tshl.b64 r2, r1, 1;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        BNN_TAP("0", "0", "p0")
        BNN_TAP("2", "128", "p1")
        BNN_TAP("4", "256", "p1")
        "add.s64 r1b, %1, r1;\n\t"
        "add.s64 a, r1b, 0;\n\tadd.s64 b, %3, 384;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %4, [%5], [%6], p1;\n\t"
        "add.s64 a, r1b, 2;\n\tadd.s64 b, %3, 512;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %4, [%5], [%6], p1;\n\t"
        "add.s64 a, r1b, 4;\n\tadd.s64 b, %3, 640;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %4, [%5], [%6], p1;\n\t"
        "add.s64 r2b, %1, r2;\n\t"
        "add.s64 a, r2b, 0;\n\tadd.s64 b, %3, 768;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %4, [%5], [%6], p1;\n\t"
        "add.s64 a, r2b, 2;\n\tadd.s64 b, %3, 896;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %4, [%5], [%6], p1;\n\t"
        "add.s64 a, r2b, 4;\n\tadd.s64 b, %3, 1024;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %4, [%5], [%6], p1;\n\t"
        "}" ::"r"(tmem_d),
        "l"(a0), "r"(a_row), "l"(b0), "r"(idesc), "r"(tmem_sfa), "r"(tmem_sfb));
#undef BNN_TAP
}

// NT x NK block-scaled FP4 MMAs from ONE elect (CG = 1: this CTA; CG = 2: a CTA pair, issued by the
// leader): MMA i = (tt, k) = (i / NK, i % NK) reads A at a0 + tt * ASTEP + 2k and B at
// b0 + tt * BSTEP + 2k (descriptor start-address units of 16 B; k = 32-B K-chunk of a wider row),
// accumulating on top of D except the first when acc0 == 0.  The descriptor offsets are PTX
// immediates, so the issuing warp spends ~3 issue slots per MMA instead of ~15 (a separate elect,
// VOTEU and R2UR of both descriptors per single-MMA call).
template <int NT, int NK, int ASTEP, int BSTEP, int CG = 1>
__device__ __forceinline__ void umma_f4_multi(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint32_t idesc, uint32_t acc0,
                                              uint32_t tmem_sfa, uint32_t tmem_sfb) {
    constexpr int N = NT * NK;
#define OA(i) ((i) / NK * ASTEP + 2 * ((i) % NK))
#define OB(i) ((i) / NK * BSTEP + 2 * ((i) % NK))
    if constexpr (!(N == 1 || N == 2 || N == 3 || N == 4 || N == 7)) {  // other counts: one call per MMA
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const uint32_t acc = i ? 1u : acc0;
            asm volatile(
                "{\n\t.reg .pred e, p;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::%7.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tmem_d),
                "l"(a0 + OA(i)), "l"(b0 + OB(i)), "r"(idesc), "r"(acc), "r"(tmem_sfa), "r"(tmem_sfb), "n"(CG));
        }
    } else if constexpr (CG == 1) {
        if constexpr (N == 1) {
            asm volatile(
                "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a, b;\n\t"
                "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t"
                "}"
                ::"r"(tmem_d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(tmem_sfa), "r"(tmem_sfb));
        } else if constexpr (N == 2) {
            asm volatile(
                "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a, b;\n\t"
                "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t"
                "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "}"
                ::"r"(tmem_d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(tmem_sfa), "r"(tmem_sfb), "n"(OA(1)), "n"(OB(1)));
        } else if constexpr (N == 3) {
            asm volatile(
                "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a, b;\n\t"
                "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t"
                "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "}"
                ::"r"(tmem_d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(tmem_sfa), "r"(tmem_sfb), "n"(OA(1)), "n"(OB(1)), "n"(OA(2)), "n"(OB(2)));
        } else if constexpr (N == 4) {
            asm volatile(
                "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a, b;\n\t"
                "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t"
                "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %11;\n\tadd.s64 b, %2, %12;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "}"
                ::"r"(tmem_d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(tmem_sfa), "r"(tmem_sfb), "n"(OA(1)), "n"(OB(1)), "n"(OA(2)), "n"(OB(2)), "n"(OA(3)), "n"(OB(3)));
        } else if constexpr (N == 7) {
            asm volatile(
                "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a, b;\n\t"
                "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t"
                "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %11;\n\tadd.s64 b, %2, %12;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %13;\n\tadd.s64 b, %2, %14;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %15;\n\tadd.s64 b, %2, %16;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %17;\n\tadd.s64 b, %2, %18;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "}"
                ::"r"(tmem_d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(tmem_sfa), "r"(tmem_sfb), "n"(OA(1)), "n"(OB(1)), "n"(OA(2)), "n"(OB(2)), "n"(OA(3)), "n"(OB(3)), "n"(OA(4)), "n"(OB(4)), "n"(OA(5)), "n"(OB(5)), "n"(OA(6)), "n"(OB(6)));
        }
    } else {
        if constexpr (N == 1) {
            asm volatile(
                "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a, b;\n\t"
                "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t"
                "}"
                ::"r"(tmem_d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(tmem_sfa), "r"(tmem_sfb));
        } else if constexpr (N == 2) {
            asm volatile(
                "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a, b;\n\t"
                "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t"
                "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "}"
                ::"r"(tmem_d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(tmem_sfa), "r"(tmem_sfb), "n"(OA(1)), "n"(OB(1)));
        } else if constexpr (N == 3) {
            asm volatile(
                "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a, b;\n\t"
                "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t"
                "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "}"
                ::"r"(tmem_d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(tmem_sfa), "r"(tmem_sfb), "n"(OA(1)), "n"(OB(1)), "n"(OA(2)), "n"(OB(2)));
        } else if constexpr (N == 4) {
            asm volatile(
                "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a, b;\n\t"
                "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t"
                "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %11;\n\tadd.s64 b, %2, %12;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "}"
                ::"r"(tmem_d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(tmem_sfa), "r"(tmem_sfb), "n"(OA(1)), "n"(OB(1)), "n"(OA(2)), "n"(OB(2)), "n"(OA(3)), "n"(OB(3)));
        } else if constexpr (N == 7) {
            asm volatile(
                "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a, b;\n\t"
                "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 q, 0, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t"
                "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %11;\n\tadd.s64 b, %2, %12;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %13;\n\tadd.s64 b, %2, %14;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %15;\n\tadd.s64 b, %2, %16;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "add.s64 a, %1, %17;\n\tadd.s64 b, %2, %18;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], a, b, %3, [%5], [%6], q;\n\t"
                "}"
                ::"r"(tmem_d), "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(tmem_sfa), "r"(tmem_sfb), "n"(OA(1)), "n"(OB(1)), "n"(OA(2)), "n"(OB(2)), "n"(OA(3)), "n"(OB(3)), "n"(OA(4)), "n"(OB(4)), "n"(OA(5)), "n"(OB(5)), "n"(OA(6)), "n"(OB(6)));
        }
    }
#undef OA
#undef OB
}

// instruction descriptor of kind::mxf4 (block-scaled): A, B = E2M1, scales UE8M0, K-major, K = 64
__host__ __device__ constexpr uint32_t idesc_f4(int M, int N) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}

// Scale-factor columns: every byte 0x7F (UE8M0 2^0) in `ncols` (multiple of 16) TMEM columns from
// `tcol`, for this warp's 32-lane quarter (call from 4 warps with distinct warp % 4).
__device__ __forceinline__ void tmem_fill_sf(uint32_t tcol, int ncols, int warp) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t v = 0x7F7F7F7Fu;
    for (int c = 0; c < ncols; c += 16)
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                tcol + lane_off + c),
            "r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void umma_commit_elect(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}

// K-major operand, rows of `row_bytes` (32, 64 or 128) swizzled, 8-row groups dense.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, int row_bytes) {
    const uint64_t layout = row_bytes == 128 ? 2ull : row_bytes == 64 ? 4ull : 6ull;  // SW128 : SW64 : SW32
    uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;                              // LBO (unused for swizzled K-major)
    d |= (uint64_t)((8 * row_bytes) >> 4) << 32;         // SBO: one 8-row swizzle atom
    d |= (uint64_t)1 << 46;                              // descriptor version (sm100)
    d |= layout << 61;
    return d;
}

// K-major, no swizzle: core matrices of 8 rows x 16 B; LBO = 128 B between K-adjacent core
// matrices, SBO between 8-row groups.
__device__ __forceinline__ uint64_t make_desc_noswz(uint32_t saddr, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)(128 >> 4) << 16;
    d |= (uint64_t)(sbo >> 4) << 32;
    d |= (uint64_t)1 << 46;
    return d;  // layout type 0 = SWIZZLE_NONE
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


// Strict per-channel threshold of 32 accumulators, branch-free (layers.py:135-146):
// POS fires iff v > t <=> t - v < 0; NEG fires iff v < t <=> v - t < 0.  With the per-channel pair
// (sgn, tsg) = POS ? (-1, t) : (+1, -t), d = sgn*v + tsg is negative exactly when the step fires:
// one IMAD + arithmetic shift + LOP3 per channel (the select-based form costs ~4x more issue).
__device__ __forceinline__ uint32_t threshold32(const uint32_t (&v)[32], const int2 *st) {
    // four independent partial words: the OR chain would otherwise serialise 32 dependent LOP3s
    uint32_t part[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i2 = 0; i2 < 16; ++i2) {
        const int4 q = reinterpret_cast<const int4 *>(st)[i2];  // two channels: (sgn, tsg, sgn, tsg)
        const int d0 = q.x * (int32_t)v[2 * i2] + q.y;
        const int d1 = q.z * (int32_t)v[2 * i2 + 1] + q.w;
        part[i2 & 3] |= ((uint32_t)(d0 >> 31) & (1u << (2 * i2))) | ((uint32_t)(d1 >> 31) & (2u << (2 * i2)));
    }
    return (part[0] | part[1]) | (part[2] | part[3]);
}

// ---- step as byte masks (sign-replicating PRMT), shared by the FP4 epilogues ----
// PRMT in its generic mode: a selector nibble with bit 3 set replicates the sign of the chosen byte
// (the __byte_perm intrinsic only honours the low 3 bits).  -> (sign(a) x 8, sign(b) x 8, ...)
__device__ __forceinline__ uint32_t prmt_sign(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, 0xFB;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// 4 folded accumulators -> fire byte mask (0xFF where d < 0, i.e. the step fires)
__device__ __forceinline__ uint32_t fire4(const uint32_t *d) {
    return __byte_perm(prmt_sign(d[0], d[1]), prmt_sign(d[2], d[3]), 0x5410);
}

// fire byte mask -> 4 bits (byte k -> bit k)
__device__ __forceinline__ uint32_t fire_nib(uint32_t f) { return ((f & 0x80808080u) * 0x00204081u) >> 28; }

// two fire byte masks (8 channels) -> 8 FP4 nibbles (fire -> +1 = 0x2, else -1 = 0xA)
__device__ __forceinline__ uint32_t fire8_f4(uint32_t f0, uint32_t f1) {
    uint32_t u0 = f0 & 0x08080808u, u1 = f1 & 0x08080808u;
    u0 |= u0 >> 4;  // byte 0: ch0 bit 3 | ch1 bit 7; byte 2: ch2 | ch3
    u1 |= u1 >> 4;
    return __byte_perm(u0, u1, 0x6420) ^ 0xAAAAAAAAu;
}

// 32 fp32 accumulators -> 8 fire byte masks (channel 4k+i in byte i of F[k]; 0xFF = the step fires):
// d = sgn * v + tsg (one FFMA), the sign replicated over a byte by PRMT -- 1 FFMA + 0.75 PRMT per channel.
__device__ __forceinline__ void fire32f(const uint32_t (&v)[32], const float2 *st, uint32_t (&F)[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const float4 q0 = reinterpret_cast<const float4 *>(st)[2 * k], q1 = reinterpret_cast<const float4 *>(st)[2 * k + 1];
        const uint32_t d0 = __float_as_uint(fmaf(q0.x, __uint_as_float(v[4 * k]), q0.y));
        const uint32_t d1 = __float_as_uint(fmaf(q0.z, __uint_as_float(v[4 * k + 1]), q0.w));
        const uint32_t d2 = __float_as_uint(fmaf(q1.x, __uint_as_float(v[4 * k + 2]), q1.y));
        const uint32_t d3 = __float_as_uint(fmaf(q1.z, __uint_as_float(v[4 * k + 3]), q1.w));
        F[k] = __byte_perm(prmt_sign(d0, d1), prmt_sign(d2, d3), 0x5410);
    }
}

// The same on accumulators of DIRECTION-FOLDED filters (the rows of POS channels negated, so acc =
// -v for POS, +v for NEG): the step is "acc + c < 0" with c = T + 0.5 (POS) / 0.5 - T (NEG) --
// the half makes every comparison strict and exact.  One FADD per channel, and the 32 constants
// are loaded up front (8 x LDS.128) so their latency is paid once per chunk, not per FFMA pair.
__device__ __forceinline__ void fire32c(const uint32_t (&v)[32], const float *c, uint32_t (&F)[8]) {
    float4 cc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) cc[k] = reinterpret_cast<const float4 *>(c)[k];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t d0 = __float_as_uint(__uint_as_float(v[4 * k]) + cc[k].x);
        const uint32_t d1 = __float_as_uint(__uint_as_float(v[4 * k + 1]) + cc[k].y);
        const uint32_t d2 = __float_as_uint(__uint_as_float(v[4 * k + 2]) + cc[k].z);
        const uint32_t d3 = __float_as_uint(__uint_as_float(v[4 * k + 3]) + cc[k].w);
        F[k] = __byte_perm(prmt_sign(d0, d1), prmt_sign(d2, d3), 0x5410);
    }
}

// per-channel constant of fire32c
__device__ __forceinline__ float step_const(int t, bool pos) { return pos ? (float)t + 0.5f : 0.5f - (float)t; }

// ---- step values -> outputs by funnel shifts: one SHF per channel moves the sign bit (the step
// fires iff d < 0) into place; four independent 8-channel chains per 32 channels ----
// d[0..7] -> 8 FP4 nibbles (fired -> +1 = 0x2, else -1 = 0xA; channel i in nibble i)
__device__ __forceinline__ uint32_t sgn8_f4(const uint32_t *d) {
    uint32_t w = 0;
#pragma unroll
    for (int i = 7; i >= 0; --i) w = __funnelshift_l(d[i], w, 4);  // (w << 4) | top nibble of d[i]
    return (w & 0x88888888u) ^ 0xAAAAAAAAu;
}

__device__ __forceinline__ uint4 sgn32_f4(const uint32_t (&d)[32]) {
    return make_uint4(sgn8_f4(d), sgn8_f4(d + 8), sgn8_f4(d + 16), sgn8_f4(d + 24));
}

// d[0..31] -> 32 fire bits (channel i -> bit i)
__device__ __forceinline__ uint32_t sgn32_bits(const uint32_t (&d)[32]) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        w[k] = 0;
#pragma unroll
        for (int i = 7; i >= 0; --i) w[k] = __funnelshift_l(d[8 * k + i], w[k], 1);
    }
    return __byte_perm(__byte_perm(w[0], w[1], 0x0040), __byte_perm(w[2], w[3], 0x0040), 0x5410);
}

// 32 direction-folded accumulators -> step values d = acc + c (in place; see fire32c)
__device__ __forceinline__ void step32c(uint32_t (&v)[32], const float *c) {
    float4 cc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) cc[k] = reinterpret_cast<const float4 *>(c)[k];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        v[4 * k] = __float_as_uint(__uint_as_float(v[4 * k]) + cc[k].x);
        v[4 * k + 1] = __float_as_uint(__uint_as_float(v[4 * k + 1]) + cc[k].y);
        v[4 * k + 2] = __float_as_uint(__uint_as_float(v[4 * k + 2]) + cc[k].z);
        v[4 * k + 3] = __float_as_uint(__uint_as_float(v[4 * k + 3]) + cc[k].w);
    }
}

// 8 fire masks (32 channels) -> 16 bytes of FP4 +-1 / -> 32 channel bits
__device__ __forceinline__ uint4 fires_to_f4(const uint32_t (&F)[8]) {
    return make_uint4(fire8_f4(F[0], F[1]), fire8_f4(F[2], F[3]), fire8_f4(F[4], F[5]), fire8_f4(F[6], F[7]));
}

__device__ __forceinline__ uint32_t fires_to_bits(const uint32_t (&F)[8]) {
    uint32_t b = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) b |= fire_nib(F[k]) << (4 * k);
    return b;
}

__device__ __forceinline__ int2 step_pair(int t, bool pos) { return pos ? make_int2(-1, t) : make_int2(1, -t); }

// The same step on fp32 accumulators of the FP4 MMAs (integer-valued, exact): d = sgn * v + tsg by
// one FFMA per channel (full rate, unlike a float->int conversion), fires iff d < 0.  tsg is built
// from the integer -T so it is never -0.0.
__device__ __forceinline__ float2 step_pair_f(int t, bool pos) {
    return pos ? make_float2(-1.f, (float)t) : make_float2(1.f, (float)(-t));
}

__device__ __forceinline__ uint32_t threshold32f(const uint32_t (&v)[32], const float2 *st) {
    uint32_t part[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i2 = 0; i2 < 16; ++i2) {
        const float4 q = reinterpret_cast<const float4 *>(st)[i2];  // (sgn, tsg, sgn, tsg)
        const float d0 = fmaf(q.x, __uint_as_float(v[2 * i2]), q.y);
        const float d1 = fmaf(q.z, __uint_as_float(v[2 * i2 + 1]), q.w);
        part[i2 & 3] |= ((__float_as_uint(d0) >> 31) << (2 * i2)) | ((__float_as_uint(d1) >> 31) << (2 * i2 + 1));
    }
    return (part[0] | part[1]) | (part[2] | part[3]);
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// ---- CTA pairs (cluster of 2 on one TPC, tcgen05 cta_group::2) ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// shared::cluster address of the same smem variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void *p, uint32_t rank) {
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(smem_addr(p)), "r"(rank));
    return d;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// arrive on an mbarrier of another CTA of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// TMA loads into this CTA's smem whose completion is counted on an mbarrier of either CTA of the pair
// (the leader's): bar is a shared::cluster address
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_addr(dst)),
        "l"(map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void tma_load_4d_pair(void *dst, const CUtensorMap *map, uint32_t bar, int c0, int c1, int c2,
                                                 int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
        "%6}], [%2];" ::"r"(smem_addr(dst)),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

// M = 256 across the pair: issued by the leader CTA only; A rows 0-127 / 128-255 and B rows
// 0..N/2-1 / N/2..N-1 come from the two CTAs' smem at the same offsets, D lands in each CTA's TMEM
__device__ __forceinline__ void umma_f4_pair_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                   uint32_t accumulate, uint32_t tmem_sfa, uint32_t tmem_sfb) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(tmem_sfa), "r"(tmem_sfb));
}

// completion of the pair's MMAs -> one arrive on the mbarrier at this offset in both CTAs
__device__ __forceinline__ void umma_commit_pair_elect(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}" ::"r"(
            smem_addr(bar)),
        "h"((uint16_t)3)
        : "memory");
}

}  // namespace bnn
