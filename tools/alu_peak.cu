// FP32 SIMT throughput microbenchmark (calibrates the "alu" roofline denominator).
// Measures FFMA (3-register form) and FFMA2 (fma.rn.f32x2) throughput per SM per clock with
// 8 independent accumulator chains per thread, operands in registers, all SMs busy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peak tools/alu_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) k_ffma(const float* in, float* out) {
    float a = in[threadIdx.x & 7], b = in[8 + (threadIdx.x & 7)];
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = in[16 + i];
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(a, acc[i], b);
        asm volatile("" : "+f"(a), "+f"(b));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

__global__ void __launch_bounds__(256) k_ffma2(const unsigned long long* in, unsigned long long* out) {
    unsigned long long a = in[threadIdx.x & 7], b = in[8 + (threadIdx.x & 7)];
    unsigned long long acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = in[16 + i];
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = ffma2(a, acc[i], b);
        asm volatile("" : "+l"(a), "+l"(b));
    }
    unsigned long long s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const int blocks = sms * 8, threads = 256;
    float* in;
    float* out;
    cudaMalloc(&in, 64 * sizeof(float));
    cudaMemset(in, 0, 64 * sizeof(float));
    cudaMalloc(&out, (size_t)blocks * threads * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double fmas = (double)blocks * threads * kIters * 8;
    for (int v = 0; v < 2; ++v) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            if (v == 0)
                k_ffma<<<blocks, threads>>>(in, out);
            else
                k_ffma2<<<blocks, threads>>>((const unsigned long long*)in, (unsigned long long*)out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double lanes = v == 0 ? 1.0 : 2.0;  // FMAs per lane per instruction
        const double tflops = 2.0 * fmas * lanes / (best * 1e-3) / 1e12;
        const double per_clk = fmas * lanes / (best * 1e-3) / (clk_khz * 1e3) / sms;
        printf("{\"op\": \"%s\", \"ms\": %.4f, \"tflops\": %.2f, \"fma_per_sm_per_clk_at_max\": %.1f, "
               "\"sms\": %d, \"max_clk_mhz\": %d}\n",
               v == 0 ? "FFMA" : "FFMA2", best, tflops, per_clk, sms, clk_khz / 1000);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(err));
        return 1;
    }
    return 0;
}
