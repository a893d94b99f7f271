// desc_shift_test.cu -- does a UMMA smem descriptor whose start address is shifted by whole
// K-major rows (64 B / 128 B) inside a TMA-swizzled tile read the shifted rows correctly, and
// which "matrix base offset" (descriptor bits 49-51) does it need?  Answers the question
// behind the halo-reuse implicit-GEMM conv (one halo tile, 9 tap descriptors).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/desc_shift_test tools/desc_shift_test.cu
//   ./tools/desc_shift_test      -> one JSON line per (row_bytes, base-offset rule)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e_), __LINE__); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

constexpr int ROWS = 256, N = 64, NSHIFT = 8;
__constant__ int kShifts[NSHIFT] = {0, 1, 2, 3, 5, 8, 34, 67};

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, int row_bytes, int rule) {
    const uint64_t layout = row_bytes == 128 ? 2ull : 4ull;
    uint64_t d = (uint64_t)((addr & 0x3FFFF) >> 4);
    d |= 1ull << 16;
    d |= (uint64_t)((8 * row_bytes) >> 4) << 32;
    d |= 1ull << 46;
    uint64_t bo = 0;
    if (rule == 1) bo = (addr >> 7) & 7;
    if (rule == 2) bo = (addr >> 7) & 3;
    if (rule == 3) bo = (addr >> 6) & 7;
    d |= bo << 49;
    d |= layout << 61;
    return d;
}

template <int RB>
__global__ void k_test(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int rule,
                       int32_t *out) {
    extern __shared__ uint8_t raw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    uint8_t *sA = sm;                 // ROWS x RB
    uint8_t *sB = sA + ROWS * RB;     // N x RB
    uint64_t *bar = (uint64_t *)(sB + N * RB);
    uint32_t *slot = (uint32_t *)(bar + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(sa(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = *slot;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"((ROWS + N) * RB));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sa(sA)),
            "l"(&ma), "r"(0), "r"(0), "r"(sa(bar)));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sa(sB)),
            "l"(&mb), "r"(0), "r"(0), "r"(sa(bar)));
    }
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(ok)
                         : "r"(sa(bar)));
    }
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    for (int si = 0; si < NSHIFT; ++si) {
        const int sh = kShifts[si];
        if (threadIdx.x == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int k = 0; k < RB / 32; ++k) {
                const uint64_t ad = desc(sa(sA) + sh * RB + 32 * k, RB, rule);
                const uint64_t bd = desc(sa(sB) + 32 * k, RB, rule == 0 ? 0 : rule);
                const uint32_t acc = k != 0;
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}" ::
                                 "r"(tm),
                             "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(bar + 1)));
        }
        {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                             : "=r"(ok)
                             : "r"(sa(bar + 1)), "r"(si & 1));
        }
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int c = 0; c < N; c += 8) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(tm + ((uint32_t)(warp * 32) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int i = 0; i < 8; ++i) out[((size_t)si * 128 + warp * 32 + lane) * N + c + i] = (int32_t)v[i];
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

static void make_map(CUtensorMap *m, void *p, int rows, int rb) {
    cuuint64_t dims[2] = {(cuuint64_t)rb, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)rb};
    cuuint32_t box[2] = {(cuuint32_t)rb, (cuuint32_t)rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     rb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("{\"error\": \"encode %d\"}\n", (int)r);
        exit(1);
    }
}

template <int RB>
static void run(int rule) {
    std::vector<int8_t> A(ROWS * RB), B(N * RB);
    srand(7 + RB);
    for (auto &x : A) x = (rand() & 1) ? 1 : -1;
    for (auto &x : B) x = (rand() & 1) ? 1 : -1;
    int8_t *dA, *dB;
    int32_t *dO;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dO, NSHIFT * 128 * N * 4));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    CUtensorMap ma, mb;
    make_map(&ma, dA, ROWS, RB);
    make_map(&mb, dB, N, RB);
    const int smem = 1024 + (ROWS + N) * RB + 64;
    CK(cudaFuncSetAttribute(k_test<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_test<RB><<<1, 128, smem>>>(ma, mb, rule, dO);
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> O(NSHIFT * 128 * N);
    CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
    const int shifts[NSHIFT] = {0, 1, 2, 3, 5, 8, 34, 67};
    printf("{\"row_bytes\": %d, \"rule\": %d, \"ok_per_shift\": [", RB, rule);
    for (int si = 0; si < NSHIFT; ++si) {
        long bad = 0;
        for (int r = 0; r < 128; ++r)
            for (int n = 0; n < N; ++n) {
                int ref = 0;
                for (int k = 0; k < RB; ++k) ref += A[(shifts[si] + r) * RB + k] * B[n * RB + k];
                bad += O[((size_t)si * 128 + r) * N + n] != ref;
            }
        printf("%s[%d, %ld]", si ? ", " : "", shifts[si], bad);
    }
    printf("]}\n");
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
}


// MMA issue throughput with an aligned vs row-shifted A descriptor (N = 64, K = 32 per MMA).
template <int RB>
__global__ void k_rate(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int shift,
                       int iters, unsigned long long *cycles) {
    extern __shared__ uint8_t raw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    uint8_t *sA = sm;
    uint8_t *sB = sA + ROWS * RB;
    uint64_t *bar = (uint64_t *)(sB + N * RB);
    uint32_t *slot = (uint32_t *)(bar + 2);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar + 1)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(sa(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = *slot;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"((ROWS + N) * RB));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sa(sA)), "l"(&ma), "r"(0), "r"(0), "r"(sa(bar)));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sa(sB)), "l"(&mb), "r"(0), "r"(0), "r"(sa(bar)));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(sa(bar)));
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int k = 0; k < RB / 32; ++k) {
                const uint64_t ad = desc(sa(sA) + shift * RB + 32 * k, RB, 0);
                const uint64_t bd = desc(sa(sB) + 32 * k, RB, 0);
                const uint32_t acc = 1;
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}" ::
                                 "r"(tm), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(bar + 1)));
        ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(sa(bar + 1)));
        cycles[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}

template <int RB>
static void rate(int shift) {
    std::vector<int8_t> A(ROWS * RB, 1), B(N * RB, 1);
    int8_t *dA, *dB;
    unsigned long long *dc;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dc, 148 * 8));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    CUtensorMap ma, mb;
    make_map(&ma, dA, ROWS, RB);
    make_map(&mb, dB, N, RB);
    const int smem = 1024 + (ROWS + N) * RB + 64;
    CK(cudaFuncSetAttribute(k_rate<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int iters = 4096;
    k_rate<RB><<<148, 128, smem>>>(ma, mb, shift, iters, dc);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> c(148);
    CK(cudaMemcpy(c.data(), dc, 148 * 8, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (auto v : c) avg += (double)v / 148;
    const double mmas = (double)iters * (RB / 32);
    printf("{\"rate_row_bytes\": %d, \"shift\": %d, \"cycles_per_mma_m128_n64_k32\": %.2f}\n", RB, shift, avg / mmas);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dc);
}

int main() {
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    for (int rule = 0; rule < 4; ++rule) {
        run<64>(rule);
        run<128>(rule);
    }
    for (int sh : {0, 1, 2, 3, 4, 8, 34}) {
        rate<64>(sh);
        rate<128>(sh);
    }
    return 0;
}
