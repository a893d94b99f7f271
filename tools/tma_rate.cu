// TMA box rate for L5's A operand (64-channel FP4 pixels = 32 B, 16x16 images), per SM with all SMs
// loading: the HX boxes the tc_block kernel issues today (two SW32 boxes of 32 B x 10 px x 8 rows per
// filter row, NHWC) against a chunk-planar layout ([img][chunk 16 B][y][x]) whose box rows are 10 px x
// 16 B = 160 contiguous bytes (one box of 16 rows x 2 chunks per filter row, or four of 8 rows).
// Every stage moves 5,120 B; the consumer only waits and frees (no MMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_rate tools/tma_rate.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

constexpr int S = 6, STAGE = 5120;

__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(unsigned b, unsigned par) {
    unsigned done = 0;
    while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(b), "r"(par) : "memory");
}
__device__ __forceinline__ void ld4(unsigned dst, const CUtensorMap *m, unsigned bar, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                 ::"r"(dst), "l"(m), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap map, int B, unsigned long long *clk) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ alignas(8) unsigned long long full[S], empty[S];
    unsigned char *s = smem + ((1024u - (sa(smem) & 1023u)) & 1023u);
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = clock64();
    unsigned st = 0, par = 0;
    if (threadIdx.x == 0) {  // producer
        for (int img = blockIdx.x; img < B; img += gridDim.x)
            for (int t = 0; t < 2; ++t)
                for (int dy = 0; dy < 3; ++dy) {
                    wait(sa(&empty[st]), par ^ 1);
                    const unsigned fb = sa(&full[st]), dst = sa(s + st * STAGE);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(STAGE) : "memory");
                    if (MODE == 0) {  // HX: NHWC, SW32, (32 B, 10 px, 8 rows) x 2 halves
                        ld4(dst, &map, fb, 0, -1, 8 * t + dy - 1, img);
                        ld4(dst + 2560, &map, fb, 0, 7, 8 * t + dy - 1, img);
                    } else if (MODE == 1) {  // planar strip: (80 u16 = 10 px x 16 B, 16 rows, 2 chunks)
                        ld4(dst, &map, fb, (8 * t - 1) * 8, dy - 1, 0, img);
                    } else {  // planar halves per chunk: 4 x (80 u16, 8 rows, 1 chunk)
                        for (int h = 0; h < 2; ++h)
                            for (int c = 0; c < 2; ++c)
                                ld4(dst + (c * 2 + h) * 1280, &map, fb, (8 * h - 1) * 8, 8 * t + dy - 1, c, img);
                    }
                    if (++st == S) { st = 0; par ^= 1; }
                }
    } else if (threadIdx.x == 32) {  // consumer
        for (int img = blockIdx.x; img < B; img += gridDim.x)
            for (int i = 0; i < 6; ++i) {
                wait(sa(&full[st]), par);
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
                if (++st == S) { st = 0; par ^= 1; }
            }
        clk[blockIdx.x] = clock64() - t0;
    }
}

int main() {
    const int B = 148 * 256, W = 16, H = 16;
    unsigned char *d;
    cudaMalloc(&d, (size_t)B * H * W * 32);
    cudaMemset(d, 1, (size_t)B * H * W * 32);
    unsigned long long *clk;
    cudaMalloc(&clk, 148 * 8);
    printf("[");
    for (int mode = 0; mode < 3; ++mode) {
        CUtensorMap map;
        CUresult r;
        if (mode == 0) {
            cuuint64_t dims[4] = {32, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
            cuuint64_t str[3] = {32, (cuuint64_t)W * 32, (cuuint64_t)H * W * 32};
            cuuint32_t box[4] = {32, 10, 8, 1}, es[4] = {1, 1, 1, 1};
            r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                       CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t dims[4] = {(cuuint64_t)W * 8, (cuuint64_t)H, 2, (cuuint64_t)B};
            cuuint64_t str[3] = {(cuuint64_t)W * 16, (cuuint64_t)H * W * 16, (cuuint64_t)2 * H * W * 16};
            cuuint32_t box[4] = {80, mode == 1 ? 16u : 8u, mode == 1 ? 2u : 1u, 1}, es[4] = {1, 1, 1, 1};
            r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("{\"mode\": %d, \"encode\": %d},", mode, (int)r); continue; }
        auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S * STAGE + 1024);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            kern<<<148, 64, S * STAGE + 1024>>>(map, B, clk);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long c[148];
            cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
            unsigned long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
            const double stages = (double)B / 148 * 6;
            if (rep == 2)
                printf("{\"mode\": %d, \"ms\": %.4f, \"clk_per_stage\": %.1f, \"B_per_clk_per_SM\": %.2f, \"err\": \"%s\"}%s\n", mode, ms,
                       mx / stages, STAGE * stages / mx, cudaGetErrorString(cudaGetLastError()), mode < 2 ? "," : "");
        }
    }
    printf("]\n");
    return 0;
}
