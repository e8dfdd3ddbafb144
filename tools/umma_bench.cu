// tcgen05.mma kind::tf32 issue-rate microbenchmark (M = 128, K = 8 per instruction,
// SWIZZLE_NONE K-major operands): cycles per MMA for back-to-back MMAs into one TMEM
// accumulator, varying N, the A start offset (16-byte shifts, as in the conv kernel's
// tap shifts) and the A LBO.  One CTA per SM, one issuing thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2205_05158_b200/csrc \
//        -o tools/umma_bench tools/umma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tcgen05.cuh"

using namespace fdpd;

template <int N>
__global__ void k_bench(int n_mma, int a_shift16, int a_lbo, int a_sbo, int b_lbo, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 255);
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    if (threadIdx.x < 32) tmem_alloc(&slot, 256);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t base = smem_u32(sm);
        const uint32_t a0 = base + 16u * a_shift16, b0 = base + 96 * 1024;
        const uint32_t idesc = idesc_tf32_m128(N);
        unsigned long long t0 = clock64();
        for (int i = 0; i < n_mma; ++i) {
            const uint32_t k = (i & 3);
            mma_tf32(tmem, umma_desc(a0 + k * 2 * a_lbo, a_lbo, a_sbo), umma_desc(b0 + k * 2 * b_lbo, b_lbo, 128), idesc,
                     i ? 1u : 0u);
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

// The conv kernel's exact MMA sequence for one tile (CINP x N, Wp, PL), repeated n_tiles times.
template <int CINP, int N>
__global__ void k_conv_seq(int n_tiles, int Wp, int PL, unsigned long long* out, int mode, const float4* gsrc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar, done;
    __shared__ volatile int stop;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 255);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&done, 1);
        stop = 0;
    }
    if (threadIdx.x < 32) tmem_alloc(&slot, 256);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    constexpr int G = CINP / 4, KSTEPS = CINP / 8;
    if (threadIdx.x >= 32) {
        // interference: 1 = spin on an mbarrier, 2 = stream 16-byte smem stores, 3 = global loads
        float4 acc = make_float4(0, 0, 0, 0);
        int it = 0;
        if (mode == 1) mbar_wait(&done, 0);
        else if (mode == 2)
            while (!stop) {
                float4* p = reinterpret_cast<float4*>(sm + 180 * 1024) + ((threadIdx.x + 32 * it++) & 1023);
                *p = make_float4(it, 0, 0, 0);
            }
        else if (mode == 3)
            while (!stop) {
                const float4 v = __ldg(gsrc + ((blockIdx.x * 4096 + threadIdx.x + 384 * it++) & ((1 << 22) - 1)));
                acc.x += v.x;
            }
        if (acc.x == 12345.f) out[0] = 0;
    }
    constexpr uint32_t WBYTES = 2u * CINP * N * 4u;
    if (threadIdx.x < 32) {
        const uint32_t base = smem_u32(sm);
        const uint32_t idesc = idesc_tf32_m128(N);
        const uint32_t ab = base + 9 * WBYTES;
        unsigned long long t0 = clock64();
        for (int t = 0; t < n_tiles; ++t) {
            for (int tap = 0; tap < 9; ++tap) {
                const uint32_t wb = base + tap * WBYTES;
                const uint32_t at = ab + (uint32_t)(((tap / 3) * Wp + (tap % 3)) * 16);
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < KSTEPS; ++k) {
                        const uint64_t ahi = umma_desc(at + 2u * k * PL, PL, 128);
                        const uint64_t alo = umma_desc(at + (uint32_t)(G + 2 * k) * PL, PL, 128);
                        const uint64_t bhi = umma_desc(wb + 2u * k * N * 16, N * 16, 128);
                        const uint64_t blo = umma_desc(wb + (uint32_t)CINP * N * 4 + 2u * k * N * 16, N * 16, 128);
                        mma_tf32(tmem, ahi, bhi, idesc, (tap | k) ? 1u : 0u);
                        mma_tf32(tmem, ahi, blo, idesc, 1u);
                        mma_tf32(tmem, alo, bhi, idesc, 1u);
                    }
                }
                __syncwarp();
            }
        }
        if (elect_one()) umma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        if (threadIdx.x == 0) {
            out[blockIdx.x] = t1 - t0;
            stop = 1;
            mbar_arrive(&done);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

template <int CINP, int N>
void run_seq(int Wp, const char* what, int mode = 0) {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int smem = 200 * 1024;
    const int A_px = (128 + 2 * Wp + 2 + 7) & ~7, PL = (A_px + 1) * 16;
    cudaFuncSetAttribute(k_conv_seq<CINP, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int n_tiles = 64;
    float4* g;
    cudaMalloc(&g, (size_t)16 << 22);
    cudaMemset(g, 0, (size_t)16 << 22);
    k_conv_seq<CINP, N><<<148, 416, smem>>>(n_tiles, Wp, PL, d, mode, g);
    k_conv_seq<CINP, N><<<148, 416, smem>>>(n_tiles, Wp, PL, d, mode, g);
    cudaFree(g);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double n_mma = (double)n_tiles * 9 * (CINP / 8) * 3;
    printf("{\"case\": \"%s\", \"mode\": %d, \"CINP\": %d, \"N\": %d, \"cyc_per_tile\": %.0f, \"cyc_per_mma\": %.1f, \"err\": \"%s\"}\n",
           what, mode, CINP, N, avg / n_tiles, avg / n_mma, cudaGetErrorString(e));
    cudaFree(d);
}

template <int N>
void run(int shift, int lbo, int sbo, const char* what) {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int smem = 160 * 1024;
    cudaFuncSetAttribute(k_bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int n_mma = 2048;
    k_bench<N><<<148, 128, smem>>>(n_mma, shift, lbo, sbo, N * 16, d);
    k_bench<N><<<148, 128, smem>>>(n_mma, shift, lbo, sbo, N * 16, d);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("{\"N\": %d, \"a_shift16\": %d, \"a_lbo\": %d, \"a_sbo\": %d, \"case\": \"%s\", \"cyc_per_mma\": %.1f, "
           "\"ideal_cyc\": %.1f, \"err\": \"%s\"}\n",
           N, shift, lbo, sbo, what, avg / n_mma, 128.0 * N / 256.0, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    // canonical: A core matrices 8 rows x 16 B contiguous, SBO = 128, LBO = 2048 (16 groups)
    run<16>(0, 2048, 128, "canonical");
    run<64>(0, 2048, 128, "canonical");
    run<16>(1, 2048, 128, "shift 16 B");
    run<64>(1, 2048, 128, "shift 16 B");
    run<16>(8, 2048, 128, "shift 128 B");
    run<16>(0, 2960, 128, "conv LBO (185 rows)");
    run<64>(3, 4112, 128, "conv LBO (257 rows) + shift");
    run<16>(0, 128, 256, "K chunks adjacent (LBO 128, SBO 256)");
    run<64>(0, 128, 256, "K chunks adjacent (LBO 128, SBO 256)");
    run<32>(0, 2048, 128, "canonical");
    run<128>(0, 2048, 128, "canonical");
    run_seq<16, 16>(27, "conv seq C2 middle");
    run_seq<16, 16>(27, "C2 middle + 12 warps spinning on an mbarrier", 1);
    run_seq<16, 16>(27, "C2 middle + 12 warps storing to smem", 2);
    run_seq<16, 16>(27, "C2 middle + 12 warps loading global", 3);
    run_seq<32, 32>(60, "conv seq C4 middle");
    run_seq<8, 16>(27, "conv seq C2 first");
    return 0;
}
