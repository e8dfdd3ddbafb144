// Where do the two CTAs of a 2-CTA cluster land?  (256 threads, ~104 KB dynamic smem, 2 CTAs/SM.)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2) k(unsigned* out, long long spin) {
    extern __shared__ unsigned char sm[];
    unsigned smid, rank;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        out[2 * blockIdx.x] = smid;
        out[2 * blockIdx.x + 1] = (unsigned)(clock64() & 0xffffffffu);
        sm[0] = 1;
        const long long t0 = clock64();
        while (clock64() - t0 < spin) {}
    }
    __syncthreads();
}
int main() {
    const int n = 2 * 148 * 3;
    unsigned* d;
    cudaMalloc(&d, n * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 104080);
    k<<<n, 256, 104080>>>(d, 200000);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    unsigned* h = new unsigned[2 * n];
    cudaMemcpy(h, d, n * 8, cudaMemcpyDeviceToHost);
    int same = 0;
    for (int c = 0; c < n / 2; ++c) same += h[4 * c] == h[4 * c + 2];
    printf("clusters %d, both CTAs on one SM: %d\n", n / 2, same);
    for (int c = 0; c < 12; ++c) printf("cluster %d: sm %u, %u  (t %u %u)\n", c, h[4 * c], h[4 * c + 2], h[4 * c + 1], h[4 * c + 3]);
    for (int c = 148; c < 156; ++c) printf("cluster %d: sm %u, %u\n", c, h[4 * c], h[4 * c + 2]);
    return 0;
}
