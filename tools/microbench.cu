// microbench.cu -- per-SM issue rates of the instructions the BNN kernels live on.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
//   ./tools/microbench            (prints one JSON line)
//
// Each kernel runs a dependency-light unrolled loop on every SM (grid = SMs x
// occupancy) and reports operations per SM-clock, measured with clock64() per
// CTA and averaged.  These are the roofline denominators for the integer-pipe
// (popc) kernel family; the tensor-core family uses MEASURED_PEAKS.json.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_popc(uint32_t seed, unsigned long long *cyc, uint32_t *sink) {
    uint32_t a[8], s[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u; s[i] = 0; }
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] += __popc(a[i] ^ (uint32_t)it);   // LOP3 + POPC + IADD
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= s[i];
    if (r == 0x12345678u) sink[0] = r;
    if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
}

__global__ void k_popc_only(uint32_t seed, unsigned long long *cyc, uint32_t *sink) {
    // popc results feed the next popc input: POPC issue-bound with 8 independent chains
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __popc(a[i]) + a[i];
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= a[i];
    if (r == 0x12345678u) sink[0] = r;
    if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
}

__global__ void k_lop3(uint32_t seed, unsigned long long *cyc, uint32_t *sink) {
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u;
    uint32_t b = seed ^ 0x55555555u, c = seed ^ 0x33333333u;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= a[i];
    if (r == 0x12345678u) sink[0] = r;
    if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
}

__global__ void k_dp4a(uint32_t seed, unsigned long long *cyc, uint32_t *sink) {
    int s[8];
    const int a = (int)(seed * (threadIdx.x + 1)), b = (int)(seed ^ 0x01ff01ffu);
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i] = i;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = __dp4a(a + i, b, s[i]);
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    int r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= s[i];
    if (r == 0x12345678) sink[0] = r;
    if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
}

__global__ void k_imma(uint32_t seed, unsigned long long *cyc, uint32_t *sink) {
    // mma.sync m16n8k32 s8 x s8 -> s32, 4 independent accumulators
    uint32_t a0 = seed * (threadIdx.x + 1), a1 = a0 ^ 0x1234u, a2 = a0 + 7, a3 = a0 * 3;
    uint32_t b0 = seed ^ 0x0f0f0f0fu, b1 = b0 + 11;
    int c[4][4] = {};
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    int r = 0;
    for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) r ^= c[i][j];
    if (r == 0x12345678) sink[0] = r;
    if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
}

template <typename K>
static double rate(K kern, int blocks_per_sm, int threads, double ops_per_thread, int sms, unsigned long long *d_cyc,
                   uint32_t *d_sink) {
    const int grid = sms * blocks_per_sm;
    kern<<<grid, threads>>>(12345u, d_cyc, d_sink);  // warm-up
    cudaMemset(d_cyc, 0, 8);
    kern<<<grid, threads>>>(12345u, d_cyc, d_sink);
    cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost);
    const double avg_cyc = (double)cyc / grid;  // cycles per CTA (all CTAs co-resident)
    return ops_per_thread * threads * blocks_per_sm / avg_cyc;  // ops per SM-cycle
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    unsigned long long *d_cyc;
    uint32_t *d_sink;
    CK(cudaMalloc(&d_cyc, 8));
    CK(cudaMalloc(&d_sink, 4));
    const double popc_chain = rate(k_popc, 4, 256, 8.0 * ITERS, sms, d_cyc, d_sink);
    const double popc_only = rate(k_popc_only, 4, 256, 8.0 * ITERS, sms, d_cyc, d_sink);
    const double lop3 = rate(k_lop3, 4, 256, 8.0 * ITERS, sms, d_cyc, d_sink);
    const double dp4a = rate(k_dp4a, 4, 256, 8.0 * ITERS, sms, d_cyc, d_sink);
    // one m16n8k32 = 16*8*32 MAC per warp
    const double imma = rate(k_imma, 4, 256, 4.0 * (ITERS / 4) * 16 * 8 * 32 / 32.0, sms, d_cyc, d_sink);
    printf("{\"sms\": %d, \"popc_xor_add_words_per_sm_clk\": %.2f, \"popc_words_per_sm_clk\": %.2f, "
           "\"lop3_per_sm_clk\": %.2f, \"dp4a_per_sm_clk\": %.2f, \"imma_s8_mac_per_sm_clk\": %.1f}\n",
           sms, popc_chain, popc_only, lop3, dp4a, imma);
    return 0;
}
