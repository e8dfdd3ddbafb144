// fdcnn_paper.cu — the paper's own FD-CNN head:
// per (symbol, UE) an S x S Re/Im image, N^Conv 3x3 kernels + bias, ReLU, flatten,
// fully connected linear layer to 2 N_d outputs (real parts, then imaginary parts).
//
//  k_paper_conv : one thread per (image, pixel): 18 MACs per kernel, ReLU, writes the
//                 flattened feature row feat[img][c S^2 + r S + col] (fp32, HBM).
//  k_fc_gemm    : feat [M = n_img][K] x W2^T [K][N = 2 N_d] + b2 -> s_tilde.  FP32 SIMT
//                 GEMM: 128 x 128 x 16 tiles, register double buffering of the next
//                 K-slab, 8 x 8 outputs per thread with packed FP32 (FFMA2); the
//                 epilogue adds the bias and scatters the real / imaginary halves into
//                 the complex output.  Tensor cores (TF32) would miss the 2e-5 parity bar.
#include "common.cuh"

namespace fdpd {

__global__ void k_paper_conv(const float2* __restrict__ s, const float* __restrict__ W1, const float* __restrict__ b1,
                             float* __restrict__ feat, long long n_img, int S, int N_d, int n_conv) {
    const long long total = n_img * S * S;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long img = i / (S * S);
        const int px = (int)(i % (S * S));
        const int y = px / S, x = px % S;
        const float2* si = s + img * N_d;
        float re[9], im[9];
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
                const int yy = y + dy - 1, xx = x + dx - 1;
                const int k = yy * S + xx;
                const bool ok = yy >= 0 && yy < S && xx >= 0 && xx < S && k < N_d;
                const float2 z = ok ? si[k] : make_float2(0.f, 0.f);
                re[dy * 3 + dx] = z.x;
                im[dy * 3 + dx] = z.y;
            }
        float* fo = feat + img * (long long)n_conv * S * S + px;
        for (int c = 0; c < n_conv; ++c) {
            const float* w = W1 + c * 18;
            float acc = b1[c];
#pragma unroll
            for (int t = 0; t < 9; ++t) acc = fmaf(w[t], re[t], acc);
#pragma unroll
            for (int t = 0; t < 9; ++t) acc = fmaf(w[9 + t], im[t], acc);
            fo[(long long)c * S * S] = fmaxf(acc, 0.f);
        }
    }
}

constexpr int GM = 128, GN = 128, GK = 16, GT = 256;

// C[m][n] = sum_k A[m][k] B[n][k] + bias[n]; A, B row-major with K contiguous, K % 4 == 0.
// Output column n < N_d -> Re(out[m][n]), else Im(out[m][n - N_d]).
__global__ void __launch_bounds__(GT, 2) k_fc_gemm(const float* __restrict__ A, const float* __restrict__ Bm,
                                                   const float* __restrict__ bias, float2* __restrict__ out, int M,
                                                   int N, int K, int N_d) {
    __shared__ __align__(16) float As[2][GK][GM + 4];
    __shared__ __align__(16) float Bs[2][GK][GN + 4];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int m0 = blockIdx.y * GM, n0 = blockIdx.x * GN;
    // global -> register staging: 2 float4 of A and 2 of B per thread per K-slab
    const int lr = tid >> 2, lk = (tid & 3) * 4;
    float4 ra[2], rb[2];
    auto gload = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int r = lr + 64 * i;
            const int k = k0 + lk;
            const bool kok = k < K;
            ra[i] = (m0 + r < M && kok) ? __ldg(reinterpret_cast<const float4*>(A + (size_t)(m0 + r) * K + k))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
            rb[i] = (n0 + r < N && kok) ? __ldg(reinterpret_cast<const float4*>(Bm + (size_t)(n0 + r) * K + k))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int r = lr + 64 * i;
            As[buf][lk + 0][r] = ra[i].x;
            As[buf][lk + 1][r] = ra[i].y;
            As[buf][lk + 2][r] = ra[i].z;
            As[buf][lk + 3][r] = ra[i].w;
            Bs[buf][lk + 0][r] = rb[i].x;
            Bs[buf][lk + 1][r] = rb[i].y;
            Bs[buf][lk + 2][r] = rb[i].z;
            Bs[buf][lk + 3][r] = rb[i].w;
        }
    };
    float2 acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
    const int nk = (K + GK - 1) / GK;
    gload(0);
    sstore(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) gload((kt + 1) * GK);
#pragma unroll
        for (int kk = 0; kk < GK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8 + 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 8]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 8 + 4]);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                  make_float2(b1.z, b1.w)};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = ffma2(bv[j], make_float2(av[i], av[i]), acc[i][j]);
        }
        if (kt + 1 < nk) sstore(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int m = m0 + ty * 8 + i;
        if (m >= M) continue;
        float* orow = reinterpret_cast<float*>(out + (size_t)m * N_d);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int n = n0 + tx * 8 + 2 * j + h;
                if (n >= N) continue;
                const float v = (h ? acc[i][j].y : acc[i][j].x) + bias[n];
                if (n < N_d) orow[2 * n] = v;
                else orow[2 * (n - N_d) + 1] = v;
            }
    }
}

}  // namespace fdpd

using namespace fdpd;

extern "C" {

size_t fdcnn_paper_workspace_bytes(int n_conv, long long n_sym, int U, int N_d) {
    if (n_conv <= 0 || n_sym <= 0 || U <= 0 || N_d <= 0) return 0;
    int S = 1;
    while (S * S < N_d) ++S;
    const size_t feat = (sizeof(float) * (size_t)n_sym * U * n_conv * S * S + 255) & ~(size_t)255;
    return feat + sizeof(float) * (size_t)2 * N_d * n_conv * S * S;   // + 16-byte aligned copy of W2
}

int fdcnn_paper_forward(const float* params, int n_conv, const void* s_in, void* s_out, void* workspace,
                        size_t workspace_bytes, long long n_sym, int U, int N_d, cudaStream_t stream) {
    FD_REQUIRE(n_conv >= 1 && n_conv <= 64, "fdcnn_paper_forward: n_conv=%d outside [1,64]", n_conv);
    FD_REQUIRE(n_sym >= 0 && U >= 1 && N_d >= 1 && N_d <= (1 << 20), "fdcnn_paper_forward: bad sizes");
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(params && s_in && s_out && workspace, "fdcnn_paper_forward: NULL pointer");
    FD_REQUIRE(s_in != s_out, "fdcnn_paper_forward: s_out must not alias s_in");
    FD_REQUIRE(aligned16(params) && aligned8(s_in) && aligned8(s_out) && aligned16(workspace),
               "fdcnn_paper_forward: misaligned pointer");
    const size_t need = fdcnn_paper_workspace_bytes(n_conv, n_sym, U, N_d);
    FD_REQUIRE(workspace_bytes >= need, "fdcnn_paper_forward: workspace of %zu bytes required", need);
    int S = 1;
    while (S * S < N_d) ++S;
    const int K = n_conv * S * S;
    FD_REQUIRE(K % 4 == 0, "fdcnn_paper_forward: N^Conv * S^2 = %d must be a multiple of 4", K);
    const long long n_img = n_sym * U;
    FD_REQUIRE(n_img <= 0x7fffffffLL, "fdcnn_paper_forward: too many images per call");
    const float* W1 = params;
    const float* b1 = W1 + n_conv * 18;
    const float* W2 = b1 + n_conv;
    const float* b2 = W2 + (size_t)2 * N_d * K;
    float* feat = (float*)workspace;
    // the FC weights sit at an arbitrary float offset of params: copy them to a 16-byte
    // aligned workspace slot so the GEMM can use 128-bit loads
    float* W2a = (float*)((char*)workspace + ((sizeof(float) * (size_t)n_img * K + 255) & ~(size_t)255));
    if (cudaMemcpyAsync(W2a, W2, sizeof(float) * (size_t)2 * N_d * K, cudaMemcpyDeviceToDevice, stream) != cudaSuccess)
        return check_launch("fdcnn_paper_forward (weights)");
    const long long total = n_img * S * S;
    k_paper_conv<<<(unsigned)std::min<long long>((total + 255) / 256, 148LL * 16), 256, 0, stream>>>(
        (const float2*)s_in, W1, b1, feat, n_img, S, N_d, n_conv);
    int rc = check_launch("fdcnn_paper_forward (conv)");
    if (rc) return rc;
    const int M = (int)n_img, N = 2 * N_d;
    dim3 grid((N + GN - 1) / GN, (M + GM - 1) / GM);
    FD_REQUIRE(grid.y <= 65535, "fdcnn_paper_forward: batch too large for one call");
    k_fc_gemm<<<grid, GT, 0, stream>>>(feat, W2a, b2, (float2*)s_out, M, N, K, N_d);
    return check_launch("fdcnn_paper_forward (fc)");
}

}  // extern "C"
