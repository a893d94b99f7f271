// fp4_peak.cu -- measured throughput peak of the instruction the binary layers run on:
// tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32, m128nNk64, +-1 operands as E2M1 codes.
//
// One persistent CTA per SM (148 on B200), operands resident in shared memory (A 128 x 256 FP4,
// B N x 256 FP4, SW128 K-major -- the layout the production kernels' TMA boxes produce), one elected
// lane issuing `iters` x 4 back-to-back MMAs (the four K = 64 steps of the 128-B swizzle atom) into
// one TMEM accumulator, as a GEMM's K loop does.  The whole grid is timed with CUDA events; every
// CTA also records clock64 and %globaltimer at both ends, so the effective SM clock under this load
// is reported next to the rate.  Result: FP4 dense TFLOP/s (2 x MACs) = the roofline denominator of
// bench.py's tensor-engine kernels (a measured, not derived, FP4 peak).
// Data: random +-1 (the BNN workload's operand statistics).  The accumulators of row 0 are checked
// against a host dot product (fp32 accumulation of an exact integer series, relative 1e-4).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2301_05126_b200/csrc \
//        -o tools/fp4_peak tools/fp4_peak.cu
//   tools/fp4_peak [iters_n256]      -> one JSON line per N, then a summary line
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "tc_ptx.cuh"

using namespace bnn;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            printf("{\"error\": \"%s at line %d\"}\n", cudaGetErrorString(e), __LINE__);       \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

constexpr int KB = 128;  // bytes per operand row = K 256 FP4 = one SW128 atom row

__host__ __device__ inline uint32_t sw128(uint32_t row, uint32_t byte) {
    const uint32_t off = row * KB + byte;
    return off ^ (((off >> 7) & 7u) << 4);
}

template <int N>
__global__ void __launch_bounds__(128, 1) peak_kernel(const uint8_t *A, const uint8_t *B, int iters, float *d_row0,
                                                      unsigned long long *tinfo) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = sm, *sB = sm + 128 * KB;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * KB; i += blockDim.x) sA[sw128(i / KB, i % KB)] = A[i];
    for (int i = tid; i < N * KB; i += blockDim.x) sB[sw128(i / KB, i % KB)] = B[i];
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tslot, sfa = tm + 256, sfb = tm + 384;
    tmem_fill_sf(sfa, 64, warp);
    tmem_fill_sf(sfb, 64, warp);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    unsigned long long c0 = 0, g0 = 0;
    if (warp == 0) {
        const uint32_t idesc = idesc_f4(128, N);
        const uint64_t a0 = umma_desc(smem_addr(sA), KB), b0 = umma_desc(smem_addr(sB), KB);
        c0 = clock64();
        g0 = global_ns();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int s = 0; s < 4; ++s)  // K = 64 steps inside the swizzle atom: start address + 32 B
                umma_f4_elect(tm, a0 + 2 * s, b0 + 2 * s, idesc, (it | s) != 0, sfa, sfb);
        }
        umma_commit_elect(&bar);
        mbar_wait(&bar, 0);
        if (tid == 0) {
            tinfo[4 * blockIdx.x + 0] = clock64() - c0;
            tinfo[4 * blockIdx.x + 1] = global_ns() - g0;
            tinfo[4 * blockIdx.x + 2] = g0;
        }
    }
    __syncthreads();
    tc_fence_after();
    if (blockIdx.x == 0 && warp == 0) {  // row 0 = TMEM lane 0: its N accumulators
        for (int c = 0; c < N; c += 8) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(tm + c));
            tmem_wait_ld();
            if (tid == 0)
                for (int i = 0; i < 8; ++i) d_row0[c + i] = __uint_as_float(v[i]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

template <int N>
static bool run(int iters, int sms, double *tflops_out) {
    std::vector<int> va(128 * 256), vb((size_t)N * 256);
    srand(4242 + N);
    for (auto &x : va) x = (rand() & 1) ? 1 : -1;
    for (auto &x : vb) x = (rand() & 1) ? 1 : -1;
    auto enc = [](int v) { return v > 0 ? 0x2 : 0xA; };
    std::vector<uint8_t> ha(128 * KB), hb((size_t)N * KB);
    for (int r = 0; r < 128; ++r)
        for (int b = 0; b < KB; ++b) ha[r * KB + b] = (uint8_t)(enc(va[r * 256 + 2 * b]) | (enc(va[r * 256 + 2 * b + 1]) << 4));
    for (int r = 0; r < N; ++r)
        for (int b = 0; b < KB; ++b) hb[r * KB + b] = (uint8_t)(enc(vb[r * 256 + 2 * b]) | (enc(vb[r * 256 + 2 * b + 1]) << 4));
    uint8_t *dA, *dB;
    float *dD;
    unsigned long long *dt;
    CK(cudaMalloc(&dA, ha.size()));
    CK(cudaMalloc(&dB, hb.size()));
    CK(cudaMalloc(&dD, N * 4));
    CK(cudaMalloc(&dt, (size_t)sms * 4 * 8));
    CK(cudaMemcpy(dA, ha.data(), ha.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hb.data(), hb.size(), cudaMemcpyHostToDevice));
    const int smem = 200 * 1024;  // one CTA per SM
    CK(cudaFuncSetAttribute(peak_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    peak_kernel<N><<<sms, 128, smem>>>(dA, dB, std::max(1, iters / 20), dD, dt);  // warm-up (clocks ramp)
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    std::vector<unsigned long long> ht((size_t)sms * 4);
    double mhz_med = 0;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0));
        peak_kernel<N><<<sms, 128, smem>>>(dA, dB, iters, dD, dt);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) {
            best = ms;
            CK(cudaMemcpy(ht.data(), dt, ht.size() * 8, cudaMemcpyDeviceToHost));
            std::vector<double> mhz(sms);
            for (int i = 0; i < sms; ++i) mhz[i] = (double)ht[4 * i] / (double)ht[4 * i + 1] * 1e3;
            std::sort(mhz.begin(), mhz.end());
            mhz_med = mhz[sms / 2];
        }
    }
    std::vector<float> hd(N);
    CK(cudaMemcpy(hd.data(), dD, N * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int n = 0; n < N; ++n) {
        long long s = 0;
        for (int k = 0; k < 256; ++k) s += (long long)va[k] * vb[(size_t)n * 256 + k];
        const double want = (double)s * iters;
        if (std::fabs(hd[n] - want) > 1e-4 * std::max(1.0, std::fabs(want)) + 1) ++bad;
    }
    const double mmas = (double)sms * iters * 4;
    const double flops = mmas * 2.0 * 128 * N * 64;
    const double tf = flops / (best * 1e-3) / 1e12;
    const double clk_per_mma = (double)ht[0] / ((double)iters * 4);
    printf("{\"N\": %d, \"sms\": %d, \"iters\": %d, \"ms\": %.3f, \"tflops_fp4_dense\": %.1f, \"sm_mhz_effective\": %.0f, "
           "\"clk_per_mma_cta0\": %.1f, \"macs_per_clk_per_sm\": %.0f, \"row0_mismatches\": %d}\n",
           N, sms, iters, best, tf, mhz_med, clk_per_mma, 128.0 * N * 64 / clk_per_mma, bad);
    *tflops_out = tf;
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    cudaFree(dt);
    return bad == 0;
}

// SW32 variant: each K = 64 step reads its own tile of 32-B rows (the front end's H / filter layout):
// A 128 x 32 B and B N x 32 B per MMA, 4 steps from 4 separate tiles.
template <int N>
__global__ void __launch_bounds__(128, 1) peak_kernel_sw32(int iters, unsigned long long *tinfo) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = sm, *sB = sm + 4 * 128 * 32;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (4 * 128 * 32 + 4 * N * 32) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(sm)[i] = ((i * 2654435761u) & 0x88888888u) | 0x22222222u;  // +-1 codes
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tslot, sfa = tm + 256, sfb = tm + 384;
    tmem_fill_sf(sfa, 64, warp);
    tmem_fill_sf(sfb, 64, warp);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        const uint32_t idesc = idesc_f4(128, N);
        const long long c0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int s = 0; s < 4; ++s)
                umma_f4_elect(tm, umma_desc(smem_addr(sA + s * 128 * 32), 32), umma_desc(smem_addr(sB + s * N * 32), 32),
                              idesc, (it | s) != 0, sfa, sfb);
        }
        umma_commit_elect(&bar);
        mbar_wait(&bar, 0);
        if (tid == 0) tinfo[blockIdx.x] = clock64() - c0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

template <int N>
static void run_sw32(int iters, int sms) {
    unsigned long long *dt;
    CK(cudaMalloc(&dt, (size_t)sms * 8));
    const int smem = 200 * 1024;
    CK(cudaFuncSetAttribute(peak_kernel_sw32<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    peak_kernel_sw32<N><<<sms, 128, smem>>>(iters / 10, dt);
    CK(cudaDeviceSynchronize());
    peak_kernel_sw32<N><<<sms, 128, smem>>>(iters, dt);
    CK(cudaDeviceSynchronize());
    unsigned long long c = 0;
    CK(cudaMemcpy(&c, dt, 8, cudaMemcpyDeviceToHost));
    printf("{\"layout\": \"SW32\", \"N\": %d, \"clk_per_mma_cta0\": %.1f, \"macs_per_clk_per_sm\": %.0f}\n", N,
           (double)c / (iters * 4.0), 128.0 * N * 64 * iters * 4.0 / c);
    cudaFree(dt);
}

int main(int argc, char **argv) {
    int iters = argc > 1 ? atoi(argv[1]) : 200000;
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    const int sms = p.multiProcessorCount;
    double t64, t128, t256;
    bool ok = run<64>(iters * 4, sms, &t64);
    ok &= run<128>(iters * 2, sms, &t128);
    ok &= run<256>(iters, sms, &t256);
    if (argc > 2) {
        run_sw32<64>(iters, sms);
        run_sw32<128>(iters, sms);
        run_sw32<256>(iters, sms);
    }
    printf("{\"device\": \"%s\", \"sms\": %d, \"peak_tflops_fp4_dense\": %.1f, \"instruction\": "
           "\"tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 m128n256k64\", \"ok\": %s}\n",
           p.name, sms, std::max(t64, std::max(t128, t256)), ok ? "true" : "false");
    return ok ? 0 : 1;
}
