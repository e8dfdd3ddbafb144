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

// sm_100 packed FP32: one FFMA2 instruction does two fp32 FMAs (same rounding as fmaf).
__device__ __forceinline__ unsigned long long f2_pack(float2 a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 f2_unpack(unsigned long long r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
// (a.x*b.x + c.x, a.y*b.y + c.y)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)), "l"(f2_pack(c)));
    return f2_unpack(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(d);
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(d);
}
// complex product with packed FP32 (FMUL2 + FFMA2), rounding identical to cmul()
__device__ __forceinline__ float2 cmul2(float2 a, float2 b) {
    const float2 t = fmul2(make_float2(-a.y, a.y), make_float2(b.y, b.x));
    return ffma2(make_float2(a.x, a.x), b, t);
}
// complex coefficient times real feature, accumulated: acc += a * w
__device__ __forceinline__ float2 cfma_real(float2 a, float w, float2 acc) { return ffma2(a, make_float2(w, w), acc); }
// acc += a * b (complex), as two FFMA2: (a.x, a.x)*(b.x, b.y) + (-b.y, b.x)*(a.y, a.y).
// Written with the broadcast scalar in the second operand of both, so ptxas uses the
// FFMA2 scalar-operand form and the swap / negate-half modifiers on b, with no register-pair
// duplication (the (-a.y, a.y) form cost two MOVs per complex MAC in the GMP loop);
// products and rounding are identical.
__device__ __forceinline__ float2 cfma2(float2 a, float2 b, float2 acc) {
    acc = ffma2(b, make_float2(a.x, a.x), acc);
    return ffma2(make_float2(-b.y, b.x), make_float2(a.y, a.y), acc);
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// ---------------------------------------------------------------- impairments (NEXT f3)
// Counter-based Philox4x32-10 (Salmon et al., SC'11), the generator the oracle implements in
// numpy: counter (idx lo, idx hi, stream, 0), key (key lo, key hi).
struct Impair {
    float clip;            // PA saturation amplitude, 0 = off
    float pa_std;          // PA measurement noise std (CN), 0 = off
    float awgn_std;        // sqrt(N_0) at the UEs, 0 = off
    unsigned key_lo, key_hi;
    long long sym0;        // global index of the batch's first symbol
    int b0, B_total;       // antenna rows of this call within the full array
    // per-symbol channel redraw (NEXT f4): element strides of per-symbol P / h_fd (0 = one
    // realisation for the whole batch) and per-symbol alpha (device, NULL = scalar)
    long long p_stride, h_stride;
    const float* alpha_dev;
    int precoded;          // chain kernels: P is the precoded spectrum X [n_sym][B][N_d]
};
constexpr unsigned STREAM_PA_NOISE = 1, STREAM_AWGN = 2;

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, unsigned k0, unsigned k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const unsigned lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const unsigned lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}
// CN(0, std^2) sample of global index idx (Box-Muller on the first two words, u = (x + 1/2) 2^-32)
__device__ __forceinline__ float2 cgauss(unsigned long long idx, unsigned stream, unsigned k0, unsigned k1,
                                         float std) {
    const uint4 x = philox4x32_10(make_uint4((unsigned)idx, (unsigned)(idx >> 32), stream, 0u), k0, k1);
    const float u1 = ((float)x.x + 0.5f) * 2.3283064365386963e-10f;
    const float u2 = ((float)x.y + 0.5f) * 2.3283064365386963e-10f;
    const float r = sqrtf(-2.f * logf(u1)) * std * 0.70710678118654752f;
    float s, c;
    sincospif(2.f * u2, &s, &c);
    return make_float2(r * c, r * s);
}
// PA saturation (phase kept) then measurement noise, P:202 (order as SPEC pa_forward)
__device__ __forceinline__ float2 pa_impair(float2 y, unsigned long long idx, const Impair& im) {
    if (im.clip > 0.f) {
        const float a2 = fmaf(y.x, y.x, y.y * y.y);
        if (a2 > im.clip * im.clip) y = cscale(y, im.clip / sqrtf(a2));
    }
    if (im.pa_std > 0.f) y = cadd(y, cgauss(idx, STREAM_PA_NOISE, im.key_lo, im.key_hi, im.pa_std));
    return y;
}

// ---------------------------------------------------------------- TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");   // visible to the async (TMA) proxy
}
// Invalidate an mbarrier before its shared memory is reused for anything else (PTX: other
// memory operations on a live mbarrier object are undefined).
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// L2 prefetch of the line holding p (no register, no completion tracking).
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// One-thread bulk copy global -> shared (TMA engine, UBLKCP), completion counted on bar.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ---------------------------------------------------------------- twiddles
// Table W[m] = exp(-2 pi i m / N), m = 0..N-1, complex64 rounded from fp64
// sincospi; cached per N (immutable plan data, freed by fd_shutdown()).
const float2* twiddle_table(int N, cudaStream_t stream);

}  // namespace fdpd
