// common.cuh — shared helpers of the libfdpd.so CUDA path (status, complex math,
// argument checks, twiddle-table cache).  Product code: never includes anything
// from oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <cstdarg>
#include <string>
#include <cmath>
#include <algorithm>

#include "../../include/fdpd.h"

namespace fdpd {

// ---------------------------------------------------------------- status
void set_error(const char* fmt, ...);
int fail_arg(const char* fmt, ...);
int check_launch(const char* what);

#define FD_REQUIRE(cond, ...)                                   \
    do {                                                        \
        if (!(cond)) return ::fdpd::fail_arg(__VA_ARGS__);      \
    } while (0)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }
inline bool is_pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }
inline int ilog2(long long v) { int r = 0; while ((1LL << r) < v) ++r; return r; }

// ---------------------------------------------------------------- complex
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// acc += a * b
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 acc) {
    acc.x = fmaf(a.x, b.x, acc.x);
    acc.x = fmaf(-a.y, b.y, acc.x);
    acc.y = fmaf(a.x, b.y, acc.y);
    acc.y = fmaf(a.y, b.x, acc.y);
    return acc;
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// ---------------------------------------------------------------- twiddles
// Table W[m] = exp(-2 pi i m / N), m = 0..N-1, complex64 rounded from fp64
// sincospi; cached per N (immutable plan data, freed by fd_shutdown()).
const float2* twiddle_table(int N, cudaStream_t stream);

}  // namespace fdpd
