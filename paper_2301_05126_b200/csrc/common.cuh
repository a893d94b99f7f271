// common.cuh -- shared device helpers and host-side status plumbing for libbnn.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bnn.h"

namespace bnn {

// ---- host-side status -------------------------------------------------------
void set_error(const char *fmt, ...);
void count_launch();
int after_launch(const char *what);  // cudaGetLastError -> status code
int ensure_init();                   // bnn_init(current device) once per device
// raise a kernel's dynamic shared-memory limit once per (kernel, device)
int allow_smem(const void *func, size_t bytes, const char *name);

#define BNN_REQUIRE(cond, ...)          \
    do {                                \
        if (!(cond)) {                  \
            ::bnn::set_error(__VA_ARGS__); \
            return -1;                  \
        }                               \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }
inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// ---- programmatic dependent launch (PDL) ------------------------------------------------------
// Every kernel is launched with programmatic stream serialization: it may start while its
// predecessor is still running, does everything that does not read the predecessor's output
// (barrier init, TMEM allocation, filter / threshold loads) and then waits in pdl_wait() for the
// predecessor grid to complete.  Kernels signal pdl_trigger() at entry so the next launch can be
// scheduled at once.  Cuts the per-layer launch + prologue latency of small (batch-1) grids; no
// effect on results.  BNN_PDL=0 in the environment turns it off.
bool pdl_on();

template <typename... KArgs, typename... Args>
inline void launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// wait for the predecessor grid (no-op when launched without PDL)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// let the dependent grid launch (its own pdl_wait still orders every dependent access)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- device helpers -----------------------------------------------------------
__device__ __forceinline__ int popc(uint32_t v) { return __popc(v); }

// xor + AND mask as one LOP3: (a ^ b) & m
__device__ __forceinline__ uint32_t xor_and(uint32_t a, uint32_t b, uint32_t m) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(r) : "r"(a), "r"(b), "r"(m));
    return r;  // 0x28 = (F0 ^ CC) & AA  with a=F0, b=CC, m=AA
}

__device__ __forceinline__ bool dir_pos(const uint32_t *posbits, int k) {
    return (__ldg(posbits + (k >> 5)) >> (k & 31)) & 1u;
}

// ---- FP4 operand format of the tensor engine ----------------------------------------------------
// A +-1 activation or weight is an exact E2M1 code: +1 = 0x2, -1 = 0xA (0x0 = zero padding).  NHWC,
// two channels per byte, channel c in nibble c & 1 of byte c >> 1 -- so a binary dot product is a
// block-scaled tcgen05.mma kind::mxf4 with unit scales (K = 64 per instruction from 32 bytes).
// 8 channel bits (bit i = +1) -> 8 FP4 nibbles (channel i in nibble i): spread then flip.
__device__ __forceinline__ uint32_t bits8_to_f4(uint32_t b) {
    uint32_t s = b & 0xFFu;
    s = (s | (s << 12)) & 0x000F000Fu;
    s = (s | (s << 6)) & 0x03030303u;
    s = (s | (s << 3)) & 0x11111111u;
    return 0xAAAAAAAAu ^ (s << 3);
}

// 32 channel bits -> 32 FP4 nibbles (16 bytes)
__device__ __forceinline__ uint4 bits_to_f4(uint32_t bits) {
    return make_uint4(bits8_to_f4(bits), bits8_to_f4(bits >> 8), bits8_to_f4(bits >> 16), bits8_to_f4(bits >> 24));
}

// 8 FP4 nibbles -> 8 bits (a nibble is +1 iff it is 0x2: sign bit clear and non-zero)
__device__ __forceinline__ uint32_t f4_to_bits8(uint32_t w) {
    const uint32_t pos = ~w & 0x88888888u & ((w & 0x22222222u) << 2);  // bit 4i+3: sign clear & e0 set
    uint32_t s = pos >> 3;                                              // bit 4i
    s = (s | (s >> 3)) & 0x03030303u;
    s = (s | (s >> 6)) & 0x000F000Fu;
    return (s | (s >> 12)) & 0xFFu;
}

// Strict threshold (layers.py:135-146): +1 iff v > T (POS) or v < T (NEG).
__device__ __forceinline__ uint32_t step_bit(int v, int t, bool pos) {
    return pos ? (v > t) : (v < t);
}

}  // namespace bnn
