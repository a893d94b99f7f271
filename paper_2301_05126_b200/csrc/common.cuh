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

// Strict threshold (layers.py:135-146): +1 iff v > T (POS) or v < T (NEG).
__device__ __forceinline__ uint32_t step_bit(int v, int t, bool pos) {
    return pos ? (v > t) : (v < t);
}

}  // namespace bnn
