// tmem_bench.cu -- throughput of draining TMEM accumulators into registers (tcgen05.ld), per SM.
//
// Question behind it: the fused front end's epilogues (128 x 64 fp32
// accumulators per tile, K = 576 so the MMA part of a tile is short) run at ~1k clk per tile; is
// that the TMEM read bandwidth?  Each CTA (one per SM) allocates 512 columns; W warps (W/4 per TMEM
// lane quarter) repeatedly load `cols` columns per instruction with the 32x32b shape (one 32-bit
// column per register per lane) and wait, sweeping all 512 columns; the result is bytes/clk/SM
// (128 lanes x 4 B per column).  Variants: x8 / x16 / x32 / x64 per instruction, 4 / 8 / 16 warps,
// wait after each load vs after a batch of loads.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2301_05126_b200/csrc \
//        -o tools/tmem_bench tools/tmem_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "tc_ptx.cuh"

using namespace bnn;

template <int X>
__device__ __forceinline__ void ld_cols(uint32_t taddr, uint32_t *v);

template <>
__device__ __forceinline__ void ld_cols<8>(uint32_t t, uint32_t *v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(t));
}
template <>
__device__ __forceinline__ void ld_cols<16>(uint32_t t, uint32_t *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(t));
}
template <>
__device__ __forceinline__ void ld_cols<32>(uint32_t t, uint32_t *v) {
    uint32_t (&a)[32] = *reinterpret_cast<uint32_t (*)[32]>(v);
    TMEM_LD32(t, a);
}

// 16x256b.x8: 16 lanes x 64 columns per warp instruction (the same 4 KB as 32x32b.x32, other lane mapping)
__device__ __forceinline__ void ld_16x256b_x8(uint32_t t, uint32_t *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(t));
}

// warps sweep 16-lane halves x 64-column blocks with 16x256b.x8
__global__ void __launch_bounds__(512, 1) tmem16_kernel(int iters, unsigned long long *cyc, uint32_t *sink) {
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, nw = blockDim.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tslot;
    const int q = warp & 3, grp = warp >> 2, ngrp = nw >> 2;
    uint32_t acc = 0, v[32];
    __syncthreads();
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int h = 0; h < 2; ++h)
            for (int c = grp * 64; c < 512; c += ngrp * 64) {
                ld_16x256b_x8(tm + ((uint32_t)(q * 32 + h * 16) << 16) + c, v);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) acc ^= v[i];
            }
    }
    __syncthreads();
    const long long c1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = c1 - c0;
    if (acc == 0x12345678u) sink[tid] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

static void run16(int warps, int iters) {
    unsigned long long *dc;
    uint32_t *ds;
    cudaMalloc(&dc, 148 * 8);
    cudaMalloc(&ds, 512 * 4);
    tmem16_kernel<<<148, 32 * warps>>>(1, dc, ds);
    cudaDeviceSynchronize();
    tmem16_kernel<<<148, 32 * warps>>>(iters, dc, ds);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)iters * 512 * 128 * 4;
    printf("{\"shape\": \"16x256b.x8\", \"warps\": %d, \"iters\": %d, \"clk\": %llu, \"bytes_per_clk_per_sm\": %.1f, "
           "\"clk_per_128x64_fp32_tile\": %.0f, \"err\": \"%s\"}\n",
           warps, iters, c, bytes / c, 32768.0 / (bytes / c), cudaGetErrorString(e));
    cudaFree(dc);
    cudaFree(ds);
}

template <int X, int BATCH>
__global__ void __launch_bounds__(512, 1) tmem_kernel(int iters, unsigned long long *cyc, uint32_t *sink) {
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, nw = blockDim.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tslot;
    const int q = warp & 3, grp = warp >> 2, ngrp = nw >> 2;  // lane quarter, column group
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint32_t acc = 0;
    uint32_t v[BATCH][X];
    __syncthreads();
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        // this warp's share of the 512 columns: groups interleave by X * BATCH columns
        for (int c = grp * X * BATCH; c < 512; c += ngrp * X * BATCH) {
#pragma unroll
            for (int b = 0; b < BATCH; ++b) ld_cols<X>(tm + lane_off + c + b * X, v[b]);
            tmem_wait_ld();
#pragma unroll
            for (int b = 0; b < BATCH; ++b)
#pragma unroll
                for (int i = 0; i < X; ++i) acc ^= v[b][i];
        }
    }
    __syncthreads();
    const long long c1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = c1 - c0;
    if (acc == 0x12345678u) sink[tid] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

template <int X, int BATCH>
static void run(int warps, int iters) {
    unsigned long long *dc;
    uint32_t *ds;
    cudaMalloc(&dc, 148 * 8);
    cudaMalloc(&ds, 512 * 4);
    tmem_kernel<X, BATCH><<<148, 32 * warps>>>(1, dc, ds);
    cudaDeviceSynchronize();
    tmem_kernel<X, BATCH><<<148, 32 * warps>>>(iters, dc, ds);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)iters * 512 * 128 * 4;  // all 512 columns x 128 lanes x 4 B per iteration
    printf("{\"shape\": \"32x32b.x%d\", \"loads_per_wait\": %d, \"warps\": %d, \"iters\": %d, \"clk\": %llu, "
           "\"bytes_per_clk_per_sm\": %.1f, \"clk_per_128x64_fp32_tile\": %.0f, \"err\": \"%s\"}\n",
           X, BATCH, warps, iters, c, bytes / c, 32768.0 / (bytes / c), cudaGetErrorString(e));
    cudaFree(dc);
    cudaFree(ds);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<8, 1>(w, 2000);
        run<16, 1>(w, 2000);
        run<32, 1>(w, 2000);
        run<32, 2>(w, 2000);
        run<16, 4>(w, 2000);
        run16(w, 2000);
    }
    return 0;
}
