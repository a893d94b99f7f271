// Does programmatic dependent launch overlap kernels on this box, in a stream and inside a captured
// CUDA graph?  K1 spins ~20 us after triggering its dependents; K2 stamps %globaltimer before and
// after griddepcontrol.wait.   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/pdl_test tools/pdl_test.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k1(unsigned long long *ts) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) ts[0] = now();
    const unsigned long long t0 = now();
    while (now() - t0 < 20000) {}
    if (threadIdx.x == 0) ts[1] = now();
}

__global__ void k2(unsigned long long *ts) {
    if (threadIdx.x == 0) ts[2] = now();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) ts[3] = now();
}

static void launch(cudaStream_t st, unsigned long long *ts, bool pdl) {
    k1<<<1, 32, 0, st>>>(ts);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k2, ts);
}

static void report(const char *what, unsigned long long *ts) {
    unsigned long long h[4];
    cudaMemcpy(h, ts, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"case\": \"%s\", \"k2_start_after_k1_start_ns\": %lld, \"k1_ns\": %lld, \"k2_wait_done_after_k1_end_ns\": %lld}\n",
           what, (long long)(h[2] - h[0]), (long long)(h[1] - h[0]), (long long)(h[3] - h[1]));
}

int main() {
    unsigned long long *ts;
    cudaMalloc(&ts, 64);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int pdl = 0; pdl < 2; ++pdl) {
        launch(st, ts, pdl);
        cudaStreamSynchronize(st);
        launch(st, ts, pdl);
        cudaStreamSynchronize(st);
        report(pdl ? "stream+pdl" : "stream", ts);
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        launch(st, ts, pdl);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        report(pdl ? "graph+pdl" : "graph", ts);
    }
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
