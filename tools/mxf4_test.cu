// mxf4_test.cu -- can a binary (+-1) dot product run on the FP4 tensor cores, exactly?
//
// +1 / -1 are exact E2M1 codes (0x2 / 0xA; 0x0 = padding), so a +-1 GEMM is a block-scaled
// tcgen05.mma kind::mxf4 with every UE8M0 scale = 127 (2^0): K = 64 per instruction from 32 bytes
// per row (half the bytes of the int8 path), fp32 accumulation (exact for |sum| < 2^24).
// This test checks, on one CTA:
//   1. numerics: D = A(128 x K) . B(N x K)^T against a CPU integer dot, for SW32 / SW64 / SW128
//      K-major operand layouts and k-steps inside a swizzle atom (descriptor start + 32 B);
//   2. scale factors written with tcgen05.st (0x7F7F7F7F over a TMEM column range) are honoured;
//   3. the issue rate of back-to-back m128nNk64 MMAs (N = 64, 128, 256), vs the int8 kind.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mxf4_test tools/mxf4_test.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                                 \
    do {                                                                      \
        cudaError_t e = (x);                                                  \
        if (e != cudaSuccess) {                                               \
            printf("{\"error\": \"%s at line %d\"}\n", cudaGetErrorString(e), __LINE__); \
            exit(1);                                                          \
        }                                                                     \
    } while (0)

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw(uint32_t a, int row_bytes) {
    // K-major swizzled: SBO = 8 rows x row_bytes; layout 6 = SW32, 4 = SW64, 2 = SW128
    const uint64_t layout = row_bytes == 128 ? 2ull : row_bytes == 64 ? 4ull : 6ull;
    uint64_t d = (uint64_t)((a & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((8 * row_bytes) >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= layout << 61;
    return d;
}

// byte offset of (row, byte) in a K-major swizzled tile with `rb`-byte rows (absolute-address swizzle)
__host__ __device__ inline uint32_t sw_off(uint32_t row, uint32_t byte, int rb) {
    const uint32_t off = row * rb + byte;
    if (rb == 128) return off ^ (((off >> 7) & 7u) << 4);
    if (rb == 64) return off ^ (((off >> 7) & 3u) << 4);
    return off ^ (((off >> 7) & 1u) << 4);  // SW32: 16-B chunk ^= bit 7
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t par) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(saddr(bar)), "r"(par)
                     : "memory");
}

template <int KIND>  // 0 = mxf4 block32, 1 = i8
__global__ void mma_kernel(const uint8_t *A, const uint8_t *Bm, float *D, int N, int kbytes, int rb, int reps,
                           long long *cycles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sA = sm;
    uint8_t *sB = sm + 128 * kbytes;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    // stage A (128 x kbytes) and B (N x kbytes) as rows of rb bytes: K chunk kc of row r at row' = kc*R + r
    for (int i = tid; i < 128 * kbytes; i += blockDim.x) {
        const int r = i / kbytes, b = i % kbytes, kc = b / rb;
        sA[kc * 128 * rb + sw_off(r, b % rb, rb)] = A[i];
    }
    for (int i = tid; i < N * kbytes; i += blockDim.x) {
        const int r = i / kbytes, b = i % kbytes, kc = b / rb;
        sB[kc * N * rb + sw_off(r, b % rb, rb)] = Bm[i];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tslot;
    const uint32_t sfa = tm + 256, sfb = tm + 384;
    {  // scale factors: every byte 0x7F (UE8M0 2^0) over 64 columns from each SF base, all 128 lanes
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t v = 0x7F7F7F7Fu;
        for (int c = 0; c < 64; c += 16) {
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                    sfa + lane_off + c),
                "r"(v));
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                    sfb + lane_off + c),
                "r"(v));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int kstep_bytes = 32;  // K=64 fp4 or K=32 int8: both 32 bytes per row per MMA
    const int steps = kbytes / kstep_bytes;
    if (tid == 0) {
        uint32_t idesc;
        if (KIND == 0)
            idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
        else
            idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        const long long t0 = clock64();
        for (int rep = 0; rep < reps; ++rep) {
            for (int s = 0; s < steps; ++s) {
                const int kc = (s * kstep_bytes) / rb, within = (s * kstep_bytes) % rb;
                const uint64_t ad = desc_sw(saddr(sA + kc * 128 * rb), rb) + (within >> 4);
                const uint64_t bd = desc_sw(saddr(sB + kc * N * rb), rb) + (within >> 4);
                const uint32_t acc = (s | rep) != 0;
                if (KIND == 0)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(tm),
                        "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
                else
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tm),
                        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar))
                     : "memory");
        mbar_wait(&bar, 0);
        cycles[0] = clock64() - t0;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    {  // D (fp32 or s32) -> global, 32 columns at a time
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const int row = (warp & 3) * 32 + (tid & 31);
        for (int c = 0; c < N; c += 8) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(tm + lane_off + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int i = 0; i < 8; ++i) D[row * N + c + i] = KIND == 0 ? __uint_as_float(v[i]) : (float)(int)v[i];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

static int run(int kind, int N, int kbytes, int rb, int reps, bool check) {
    // values: kind 0 -> fp4 nibbles (+1 0x2, -1 0xA, 0 0x0) two per byte; kind 1 -> int8 +-1/0
    const int kel = kind == 0 ? 2 * kbytes : kbytes;
    std::vector<int> va(128 * kel), vb((size_t)N * kel);
    srand(1234 + N + kbytes + rb);
    for (auto &x : va) x = (rand() % 7 == 0) ? 0 : ((rand() & 1) ? 1 : -1);
    for (auto &x : vb) x = (rand() % 9 == 0) ? 0 : ((rand() & 1) ? 1 : -1);
    auto enc4 = [](int v) { return v == 0 ? 0x0 : (v > 0 ? 0x2 : 0xA); };
    std::vector<uint8_t> ha(128 * kbytes), hb((size_t)N * kbytes);
    for (int r = 0; r < 128; ++r)
        for (int b = 0; b < kbytes; ++b)
            ha[r * kbytes + b] = kind == 0 ? (uint8_t)(enc4(va[r * kel + 2 * b]) | (enc4(va[r * kel + 2 * b + 1]) << 4))
                                           : (uint8_t)(int8_t)va[r * kel + b];
    for (int r = 0; r < N; ++r)
        for (int b = 0; b < kbytes; ++b)
            hb[r * kbytes + b] = kind == 0 ? (uint8_t)(enc4(vb[r * kel + 2 * b]) | (enc4(vb[r * kel + 2 * b + 1]) << 4))
                                           : (uint8_t)(int8_t)vb[r * kel + b];
    uint8_t *dA, *dB;
    float *dD;
    long long *dc;
    CK(cudaMalloc(&dA, ha.size()));
    CK(cudaMalloc(&dB, hb.size()));
    CK(cudaMalloc(&dD, 128 * N * 4));
    CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dA, ha.data(), ha.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hb.data(), hb.size(), cudaMemcpyHostToDevice));
    const size_t smem = (size_t)(128 + N) * kbytes + 1024;
    auto kern = kind == 0 ? mma_kernel<0> : mma_kernel<1>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<1, 128, smem>>>(dA, dB, dD, N, kbytes, rb, reps, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> hd(128 * N);
    long long cyc = 0;
    CK(cudaMemcpy(hd.data(), dD, hd.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    long long bad = 0;
    if (check) {
        for (int r = 0; r < 128; ++r)
            for (int n = 0; n < N; ++n) {
                long long s = 0;
                for (int k = 0; k < kel; ++k) s += (long long)va[r * kel + k] * vb[(size_t)n * kel + k];
                if ((double)hd[r * N + n] != (double)(s * reps)) ++bad;
            }
    }
    const int mmas = reps * (kbytes / 32);
    printf("{\"kind\": \"%s\", \"N\": %d, \"K\": %d, \"row_bytes\": %d, \"reps\": %d, \"mismatches\": %lld, "
           "\"cycles_per_mma\": %.2f, \"macs_per_clk\": %.0f}\n",
           kind == 0 ? "mxf4" : "i8", N, kel, rb, reps, bad, (double)cyc / mmas,
           (double)128 * N * (kind == 0 ? 64 : 32) * mmas / cyc);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    cudaFree(dc);
    return bad ? 1 : 0;
}

int main() {
    int fails = 0;
    // numerics: layouts and in-atom k-steps
    fails += run(0, 64, 32, 32, 1, true);
    fails += run(0, 64, 64, 64, 1, true);
    fails += run(0, 64, 128, 128, 1, true);
    fails += run(0, 256, 128, 128, 1, true);
    fails += run(0, 128, 256, 128, 1, true);
    fails += run(0, 64, 96, 32, 1, true);
    // rates (small K resident, many reps)
    for (int n : {64, 128, 256}) {
        run(0, n, 128, 128, 200, true);
        run(1, n, 128, 128, 200, true);
    }
    printf("{\"fails\": %d}\n", fails);
    return 0;
}
