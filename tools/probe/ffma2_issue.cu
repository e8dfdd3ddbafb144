// Does an FFMA2 leave its second cycle's issue slot to another pipe?  8 warps per SM-quarter
// run N FFMA2 (8 independent chains) interleaved with K integer LOP3/IADD ops per FFMA2 on
// independent registers.  If FFMA2 blocked only the FMA pipe, K = 1 would cost no extra time.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
template <int K, bool PACKED>
__global__ void __launch_bounds__(256) k(const unsigned long long* in, unsigned long long* out, int iters) {
    unsigned long long acc[8];
    unsigned x[8];
    const unsigned long long a = in[threadIdx.x & 7], b = in[8 + (threadIdx.x & 7)];
    for (int i = 0; i < 8; ++i) { acc[i] = in[16 + i] + threadIdx.x; x[i] = threadIdx.x * 7 + i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (PACKED) acc[i] = ffma2(a, acc[i], b);
            else {
                float lo = __uint_as_float((unsigned)acc[i]), hi = __uint_as_float((unsigned)(acc[i] >> 32));
                asm volatile("fma.rn.f32 %0, %1, %0, %2;" : "+f"(lo) : "f"(__uint_as_float((unsigned)a)), "f"(__uint_as_float((unsigned)b)));
                asm volatile("fma.rn.f32 %0, %1, %0, %2;" : "+f"(hi) : "f"(__uint_as_float((unsigned)a)), "f"(__uint_as_float((unsigned)b)));
                acc[i] = ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
            }
#pragma unroll
            for (int k2 = 0; k2 < K; ++k2) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(x[(i + 1) & 7]), "r"(it));
        }
    }
    unsigned long long s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i] + x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int K, bool P>
void run(const char* name) {
    unsigned long long *in, *out;
    cudaMalloc(&in, 4096); cudaMemset(in, 0x3c, 4096);
    const int blocks = 148 * 4, iters = 4096;
    cudaMalloc(&out, blocks * 256 * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0); k<K, P><<<blocks, 256>>>(in, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    // per SMSP: 8 warps (4 CTAs x 8 warps / 4), each iters*8 steps
    const double cyc = best * 1e-3 * 1.965e9, steps = 8.0 * iters * 8;
    printf("%-28s %.3f ms  cycles per (FMA-pair + %d int) per SMSP: %.2f\n", name, best, K, cyc / steps);
}
int main() {
    run<0, true>("FFMA2 only"); run<1, true>("FFMA2 + 1 LOP3"); run<2, true>("FFMA2 + 2 LOP3"); run<3, true>("FFMA2 + 3 LOP3");
    run<0, false>("2 FFMA only"); run<1, false>("2 FFMA + 1 LOP3"); run<2, false>("2 FFMA + 2 LOP3");
    return 0;
}
