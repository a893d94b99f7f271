// Can one TMA box read the two overlapping halves of a zero-padded 18-px row (x' in [0,10) at
// h * 8 px, h = 0, 1) through a 5-D tensor map whose h stride (256 B) is smaller than the x'
// extent (320 B)?   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_overlap_test tools/tma_overlap_test.cu -lcuda
#include <cstdio>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void k(const __grid_constant__ CUtensorMap map, unsigned char *out, int y0) {
    __shared__ alignas(1024) unsigned char s[2 * 8 * 10 * 32];
    __shared__ alignas(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar), ss = (unsigned)__cvta_generic_to_shared(s);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(5120) : "memory");
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                     ::"r"(ss), "l"(&map), "r"(sb), "r"(0), "r"(0), "r"(y0), "r"(0), "r"(0) : "memory");
        unsigned done = 0;
        while (!done)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(sb) : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 5120; i += blockDim.x) out[i] = s[i];
}

int main() {
    const int W = 16, Wp = 18, H = 16, CB = 32;
    unsigned char *h = new unsigned char[H * Wp * CB];
    for (int y = 0; y < H; ++y)
        for (int xp = 0; xp < Wp; ++xp)
            for (int c = 0; c < CB; ++c)
                h[(y * Wp + xp) * CB + c] = (xp == 0 || xp == Wp - 1) ? 0 : (unsigned char)(1 + (y * 16 + (xp - 1)) % 250);
    unsigned char *d, *o;
    cudaMalloc(&d, H * Wp * CB);
    cudaMalloc(&o, 5120);
    cudaMemcpy(d, h, H * Wp * CB, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[5] = {32, 10, (cuuint64_t)H, 2, 1};
    cuuint64_t str[4] = {32, (cuuint64_t)Wp * 32, 8 * 32, (cuuint64_t)H * Wp * 32};
    cuuint32_t box[5] = {32, 10, 8, 2, 1}, es[5] = {1, 1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, d, dims, str, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("{\"encode\": %d", (int)r);
    if (r != CUDA_SUCCESS) { printf("}\n"); return 0; }
    int bad = 0;
    for (int y0 = -1; y0 <= 9; y0 += 10) {
        k<<<1, 128>>>(map, o, y0);
        unsigned char res[5120];
        cudaMemcpy(res, o, 5120, cudaMemcpyDeviceToHost);
        for (int hh = 0; hh < 2; ++hh)
            for (int yy = 0; yy < 8; ++yy)
                for (int xq = 0; xq < 10; ++xq) {
                    const int y = y0 + yy, xp = hh * 8 + xq;
                    const unsigned char want = (y < 0 || y >= H) ? 0 : h[(y * Wp + xp) * CB];
                    if (res[((hh * 8 + yy) * 10 + xq) * 32] != want) ++bad;
                }
    }
    printf(", \"mismatches\": %d, \"err\": \"%s\"}\n", bad, cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
