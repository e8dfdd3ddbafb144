// zf.cu — zero-forcing precoder build (Eq. 6; FD channel P:72; alpha P:84,
// reading A12).  Once per channel realisation, off the per-symbol path.
//
// One CTA per data subcarrier j:
//   Hfd = sum_t H_t e^{-2 pi i k_j t / N}      (fp64 accumulate, stored fp32 in smem)
//   G   = Hfd Hfd^H                             (fp64, one warp per (u, v) pair)
//   G   = L L^H (Cholesky, fp64, one warp) ; Linv ; Ginv = Linv^H Linv ; tr_j = ||Linv||_F^2
//   P0  = Hfd^H Ginv                            (rows b0 .. b0 + B_loc)
// then alpha = rho sqrt(B N / sum_j tr_j) (one CTA, fixed-order fp64 sum) and P = alpha P0.
#include "fft.cuh"

namespace fdpd {

__device__ __forceinline__ double2 dcmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 dcmulc(double2 a, double2 b) {   // a * conj(b)
    return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

// Herr != NULL (imperfect CSI): the precoder uses H_est = sqrt(1-eta) H + sqrt(eta) Herr
// while h_fd (the channel the UEs see) is the true H.
__global__ void __launch_bounds__(256) k_zf(const float2* __restrict__ H, int T, int U, int B, int N, int N_d, int b0,
                                            int B_loc, float2* __restrict__ hfd, float2* __restrict__ P,
                                            double* __restrict__ tr, int* __restrict__ flag,
                                            const float2* __restrict__ Herr, double eta) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* G = reinterpret_cast<double2*>(smem_raw);         // [U][U]  (G, then Ginv)
    double2* Lm = G + U * U;                                   // [U][U]  Cholesky factor
    double2* Li = Lm + U * U;                                  // [U][U]  inverse of L
    double2* tw = Li + U * U;                                  // [T]
    float2* Hs = reinterpret_cast<float2*>(tw + T);            // [U][B]
    // batched builds (per-symbol channel redraw, NEXT f4): channel realisation blockIdx.y
    {
        const size_t c = blockIdx.y;
        H += c * T * U * B;
        hfd += c * (size_t)U * B_loc * N_d;
        P += c * (size_t)B_loc * U * N_d;
        tr += c * N_d;
    }
    const int j = blockIdx.x, tid = threadIdx.x, nth = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = nth >> 5;
    const int k = data_to_bin(j, N, N_d);

    for (int t = tid; t < T; t += nth) {
        double s, c;
        sincospi(-2.0 * (double)(((long long)k * t) % N) / (double)N, &s, &c);
        tw[t] = make_double2(c, s);
    }
    __syncthreads();
    const double ce = sqrt(1.0 - eta), se = sqrt(eta);
    for (int i = tid; i < U * B; i += nth) {
        double2 acc = make_double2(0.0, 0.0), ace = make_double2(0.0, 0.0);
        for (int t = 0; t < T; ++t) {
            const float2 h = H[(size_t)t * U * B + i];
            const double2 w = tw[t];
            acc.x += (double)h.x * w.x - (double)h.y * w.y;
            acc.y += (double)h.x * w.y + (double)h.y * w.x;
            if (Herr) {
                const float2 e = Herr[(size_t)t * U * B + i];
                const double ex = ce * h.x + se * e.x, ey = ce * h.y + se * e.y;
                ace.x += ex * w.x - ey * w.y;
                ace.y += ex * w.y + ey * w.x;
            }
        }
        const float2 hf = make_float2((float)acc.x, (float)acc.y);
        Hs[i] = Herr ? make_float2((float)ace.x, (float)ace.y) : hf;
        const int u = i / B, b = i % B;
        if (b >= b0 && b < b0 + B_loc) hfd[((size_t)u * B_loc + (b - b0)) * N_d + j] = hf;
    }
    __syncthreads();
    // Gram (lower triangle), one warp per pair
    const int npair = U * (U + 1) / 2;
    for (int pr = warp; pr < npair; pr += nwarp) {
        int u = 0;
        while ((u + 1) * (u + 2) / 2 <= pr) ++u;
        const int v = pr - u * (u + 1) / 2;
        double2 acc = make_double2(0.0, 0.0);
        for (int b = lane; b < B; b += 32) {
            const float2 a = Hs[u * B + b], c = Hs[v * B + b];
            acc.x += (double)a.x * c.x + (double)a.y * c.y;
            acc.y += (double)a.y * c.x - (double)a.x * c.y;
        }
        for (int o = 16; o > 0; o >>= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        }
        if (lane == 0) {
            G[u * U + v] = acc;
            G[v * U + u] = make_double2(acc.x, -acc.y);
        }
    }
    __syncthreads();
    // Cholesky + triangular inverse in warp 0 (lane = row / column)
    if (warp == 0) {
        for (int i = lane; i < U * U; i += 32) { Lm[i] = make_double2(0.0, 0.0); Li[i] = make_double2(0.0, 0.0); }
        __syncwarp();
        int bad = 0;
        for (int c = 0; c < U; ++c) {
            if (lane == 0) {
                double d = G[c * U + c].x;
                for (int p = 0; p < c; ++p) d -= Lm[c * U + p].x * Lm[c * U + p].x + Lm[c * U + p].y * Lm[c * U + p].y;
                if (!(d > 1e-300)) { bad = 1; d = 1.0; }
                Lm[c * U + c] = make_double2(sqrt(d), 0.0);
            }
            __syncwarp();
            for (int i = c + 1 + lane; i < U; i += 32) {
                double2 s = G[i * U + c];
                for (int p = 0; p < c; ++p) {
                    const double2 q = dcmulc(Lm[i * U + p], Lm[c * U + p]);
                    s.x -= q.x;
                    s.y -= q.y;
                }
                const double inv = 1.0 / Lm[c * U + c].x;
                Lm[i * U + c] = make_double2(s.x * inv, s.y * inv);
            }
            __syncwarp();
        }
        bad = __shfl_sync(0xffffffffu, bad, 0);
        if (bad && lane == 0) atomicExch(flag, 1);
        for (int c = lane; c < U; c += 32) {
            Li[c * U + c] = make_double2(1.0 / Lm[c * U + c].x, 0.0);
            for (int i = c + 1; i < U; ++i) {
                double2 s = make_double2(0.0, 0.0);
                for (int p = c; p < i; ++p) {
                    const double2 q = dcmul(Lm[i * U + p], Li[p * U + c]);
                    s.x += q.x;
                    s.y += q.y;
                }
                const double inv = -1.0 / Lm[i * U + i].x;
                Li[i * U + c] = make_double2(s.x * inv, s.y * inv);
            }
        }
    }
    __syncthreads();
    // Ginv[u][v] = sum_p conj(Li[p][u]) Li[p][v]
    for (int i = tid; i < U * U; i += nth) {
        const int u = i / U, v = i % U;
        double2 s = make_double2(0.0, 0.0);
        for (int p = (u > v ? u : v); p < U; ++p) {
            const double2 q = dcmulc(Li[p * U + v], Li[p * U + u]);
            s.x += q.x;
            s.y += q.y;
        }
        G[i] = s;
    }
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int u = 0; u < U; ++u) t += G[u * U + u].x;
        tr[j] = t;
    }
    // P0[b][u] = sum_v conj(Hfd[v][b]) Ginv[v][u]
    for (int i = tid; i < B_loc * U; i += nth) {
        const int bl = i / U, u = i % U, b = bl + b0;
        double2 s = make_double2(0.0, 0.0);
        for (int v = 0; v < U; ++v) {
            const float2 h = Hs[v * B + b];
            const double2 g = G[v * U + u];
            s.x += (double)h.x * g.x + (double)h.y * g.y;
            s.y += (double)h.x * g.y - (double)h.y * g.x;
        }
        P[((size_t)bl * U + u) * N_d + j] = make_float2((float)s.x, (float)s.y);
    }
}

// Warp-per-subcarrier variant for small U x B (C1-C3, P; per-warp shared slice <= 24 KB):
// the same arithmetic, in the same order, as k_zf (so the results are bit-identical), but
// eight subcarriers per CTA and no CTA-wide barriers — the per-symbol build of NEXT f4
// (--redraw) issues N_d x n_sym of these tiny problems, where k_zf's 256-thread CTAs with
// ten barriers each were mostly idle.
constexpr int ZFW_WARPS = 8;
__host__ __device__ inline size_t zf_warp_smem(int T, int U, int B) {
    return ((sizeof(double2) * (3 * (size_t)U * U + T) + sizeof(float2) * (size_t)U * B) + 15) & ~(size_t)15;
}
__host__ __device__ inline bool zf_taps_fit(int T, int U, int B) {
    return sizeof(double2) * (size_t)T * U * B <= 48 * 1024;
}
__global__ void __launch_bounds__(32 * ZFW_WARPS) k_zf_warp(const float2* __restrict__ H, int T, int U, int B, int N,
                                                          int N_d, int b0, int B_loc, float2* __restrict__ hfd,
                                                          float2* __restrict__ P, double* __restrict__ tr,
                                                          int* __restrict__ flag, const float2* __restrict__ Herr,
                                                          double eta) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = blockIdx.x * ZFW_WARPS + warp;
    unsigned char* base = smem_raw + (size_t)warp * zf_warp_smem(T, U, B);
    // the realisation's taps, converted to fp64 once per CTA and shared by its 8 subcarriers
    // (when they fit: C1, C2, P) — the per-warp float loads + F2F conversions dominated
    double2* Hd = reinterpret_cast<double2*>(smem_raw + (size_t)ZFW_WARPS * zf_warp_smem(T, U, B));
    const bool shared_taps = Herr == nullptr && zf_taps_fit(T, U, B);
    if (shared_taps) {
        const float2* Hc = H + (size_t)blockIdx.y * T * U * B;
        for (int i = threadIdx.x; i < T * U * B; i += blockDim.x) {
            const float2 h = __ldg(Hc + i);
            Hd[i] = make_double2((double)h.x, (double)h.y);
        }
        __syncthreads();
    }
    if (j >= N_d) return;                                   // whole warp; no CTA barriers below
    double2* G = reinterpret_cast<double2*>(base);
    double2* Lm = G + U * U;
    double2* Li = Lm + U * U;
    double2* tw = Li + U * U;
    float2* Hs = reinterpret_cast<float2*>(tw + T);
    {
        const size_t c = blockIdx.y;
        H += c * T * U * B;
        hfd += c * (size_t)U * B_loc * N_d;
        P += c * (size_t)B_loc * U * N_d;
        tr += c * N_d;
    }
    const int k = data_to_bin(j, N, N_d);
    for (int t = lane; t < T; t += 32) {
        double sn, cs;
        sincospi(-2.0 * (double)(((long long)k * t) % N) / (double)N, &sn, &cs);
        tw[t] = make_double2(cs, sn);
    }
    __syncwarp();
    const double ce = sqrt(1.0 - eta), se = sqrt(eta);
    for (int i = lane; i < U * B; i += 32) {
        double2 acc = make_double2(0.0, 0.0), ace = make_double2(0.0, 0.0);
        if (shared_taps) {
            for (int t = 0; t < T; ++t) {
                const double2 h = Hd[(size_t)t * U * B + i];
                const double2 w = tw[t];
                acc.x += h.x * w.x - h.y * w.y;
                acc.y += h.x * w.y + h.y * w.x;
            }
        } else {
            for (int t = 0; t < T; ++t) {
                const float2 h = H[(size_t)t * U * B + i];
                const double2 w = tw[t];
                acc.x += (double)h.x * w.x - (double)h.y * w.y;
                acc.y += (double)h.x * w.y + (double)h.y * w.x;
                if (Herr) {
                    const float2 e = Herr[(size_t)t * U * B + i];
                    const double ex = ce * h.x + se * e.x, ey = ce * h.y + se * e.y;
                    ace.x += ex * w.x - ey * w.y;
                    ace.y += ex * w.y + ey * w.x;
                }
            }
        }
        const float2 hf = make_float2((float)acc.x, (float)acc.y);
        Hs[i] = Herr ? make_float2((float)ace.x, (float)ace.y) : hf;
        const int u = i / B, b = i % B;
        if (b >= b0 && b < b0 + B_loc) hfd[((size_t)u * B_loc + (b - b0)) * N_d + j] = hf;
    }
    __syncwarp();
    const int npair = U * (U + 1) / 2;
    for (int pr = 0; pr < npair; ++pr) {
        int u = 0;
        while ((u + 1) * (u + 2) / 2 <= pr) ++u;
        const int v = pr - u * (u + 1) / 2;
        double2 acc = make_double2(0.0, 0.0);
        for (int b = lane; b < B; b += 32) {
            const float2 a = Hs[u * B + b], c = Hs[v * B + b];
            acc.x += (double)a.x * c.x + (double)a.y * c.y;
            acc.y += (double)a.y * c.x - (double)a.x * c.y;
        }
        for (int o = 16; o > 0; o >>= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        }
        if (lane == 0) {
            G[u * U + v] = acc;
            G[v * U + u] = make_double2(acc.x, -acc.y);
        }
    }
    for (int i = lane; i < U * U; i += 32) { Lm[i] = make_double2(0.0, 0.0); Li[i] = make_double2(0.0, 0.0); }
    __syncwarp();
    int bad = 0;
    for (int c = 0; c < U; ++c) {
        if (lane == 0) {
            double d = G[c * U + c].x;
            for (int p = 0; p < c; ++p) d -= Lm[c * U + p].x * Lm[c * U + p].x + Lm[c * U + p].y * Lm[c * U + p].y;
            if (!(d > 1e-300)) { bad = 1; d = 1.0; }
            Lm[c * U + c] = make_double2(sqrt(d), 0.0);
        }
        __syncwarp();
        for (int i = c + 1 + lane; i < U; i += 32) {
            double2 sv = G[i * U + c];
            for (int p = 0; p < c; ++p) {
                const double2 q = dcmulc(Lm[i * U + p], Lm[c * U + p]);
                sv.x -= q.x;
                sv.y -= q.y;
            }
            const double inv = 1.0 / Lm[c * U + c].x;
            Lm[i * U + c] = make_double2(sv.x * inv, sv.y * inv);
        }
        __syncwarp();
    }
    bad = __shfl_sync(0xffffffffu, bad, 0);
    if (bad && lane == 0) atomicExch(flag, 1);
    for (int c = lane; c < U; c += 32) {
        Li[c * U + c] = make_double2(1.0 / Lm[c * U + c].x, 0.0);
        for (int i = c + 1; i < U; ++i) {
            double2 sv = make_double2(0.0, 0.0);
            for (int p = c; p < i; ++p) {
                const double2 q = dcmul(Lm[i * U + p], Li[p * U + c]);
                sv.x += q.x;
                sv.y += q.y;
            }
            const double inv = -1.0 / Lm[i * U + i].x;
            Li[i * U + c] = make_double2(sv.x * inv, sv.y * inv);
        }
    }
    __syncwarp();
    for (int i = lane; i < U * U; i += 32) {
        const int u = i / U, v = i % U;
        double2 sv = make_double2(0.0, 0.0);
        for (int p = (u > v ? u : v); p < U; ++p) {
            const double2 q = dcmulc(Li[p * U + v], Li[p * U + u]);
            sv.x += q.x;
            sv.y += q.y;
        }
        G[i] = sv;
    }
    __syncwarp();
    if (lane == 0) {
        double t = 0.0;
        for (int u = 0; u < U; ++u) t += G[u * U + u].x;
        tr[j] = t;
    }
    for (int i = lane; i < B_loc * U; i += 32) {
        const int bl = i / U, u = i % U, b = bl + b0;
        double2 sv = make_double2(0.0, 0.0);
        for (int v = 0; v < U; ++v) {
            const float2 h = Hs[v * B + b];
            const double2 g = G[v * U + u];
            sv.x += (double)h.x * g.x + (double)h.y * g.y;
            sv.y += (double)h.x * g.y - (double)h.y * g.x;
        }
        P[((size_t)bl * U + u) * N_d + j] = make_float2((float)sv.x, (float)sv.y);
    }
}

// Launches k_zf_warp where its per-warp slice fits (<= 24 KB), else k_zf.
static void launch_zf_any(const float2* H, int T, int U, int B, int N, int N_d, int b0, int B_loc, float2* hfd,
                          float2* P, double* tr, int* flag, const float2* Herr, double eta, int n_ch, size_t smem_cta,
                          cudaStream_t st) {
    const size_t per_warp = zf_warp_smem(T, U, B);
    if (per_warp <= 24 * 1024) {
        const size_t smem = per_warp * ZFW_WARPS +
                            ((Herr == nullptr && zf_taps_fit(T, U, B)) ? sizeof(double2) * (size_t)T * U * B : 0);
        cudaFuncSetAttribute(k_zf_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_zf_warp<<<dim3((N_d + ZFW_WARPS - 1) / ZFW_WARPS, n_ch), 32 * ZFW_WARPS, smem, st>>>(
            H, T, U, B, N, N_d, b0, B_loc, hfd, P, tr, flag, Herr, eta);
    } else {
        cudaFuncSetAttribute(k_zf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cta);
        k_zf<<<dim3(N_d, n_ch), 256, smem_cta, st>>>(H, T, U, B, N, N_d, b0, B_loc, hfd, P, tr, flag, Herr, eta);
    }
}

// One CTA per channel realisation c: fixed-order fp64 sum of tr_j, alpha_c (A12); also a
// float copy for the slicer when alpha_f != NULL.
__global__ void k_zf_alpha(const double* __restrict__ tr, int N_d, double scale, double rho, double* alpha,
                           float* alpha_f) {
    __shared__ double part[256];
    const int c = blockIdx.x;
    double s = 0.0;
    for (int j = threadIdx.x; j < N_d; j += blockDim.x) s += tr[(size_t)c * N_d + j];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        alpha[c] = rho * sqrt(scale / part[0]);
        if (alpha_f) alpha_f[c] = (float)alpha[c];
    }
}

// P_c *= alpha_c for the n_ch realisations of `per` complex entries each
__global__ void k_scale(float2* __restrict__ P, long long per, int n_ch, const double* __restrict__ alpha) {
    const long long n = per * n_ch;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        P[i] = cscale(P[i], (float)alpha[i / per]);
}

static size_t zf_smem(int T, int U, int B) {
    return sizeof(double2) * (3 * (size_t)U * U + T) + sizeof(float2) * (size_t)U * B;
}

}  // namespace fdpd

using namespace fdpd;

extern "C" {

size_t zf_workspace_bytes(int N_d) { return N_d > 0 ? sizeof(double) * (size_t)N_d + 16 : 0; }

size_t zf_batched_workspace_bytes(int n_ch, int N_d) {
    return (n_ch > 0 && N_d > 0) ? sizeof(double) * ((size_t)n_ch * N_d + n_ch) + 16 : 0;
}

static int zf_validate(const void* h_taps, const void* h_fd, const void* P, const void* workspace, int T, int U, int B,
                       int N_ifft, int N_d, float rho, int b0, int B_loc, size_t& smem) {
    FD_REQUIRE(h_taps && h_fd && P && workspace, "zf_precoder_build: NULL pointer");
    FD_REQUIRE(aligned8(h_taps) && aligned8(h_fd) && aligned8(P) && aligned8(workspace),
               "zf_precoder_build: misaligned pointer");
    FD_REQUIRE(T >= 1 && T <= 4096, "T=%d outside [1,4096]", T);
    FD_REQUIRE(U >= 1 && U <= 64 && U <= B, "U=%d must be in [1, min(64, B)]", U);
    FD_REQUIRE(is_pow2(N_ifft) && N_ifft <= (1 << 24), "N_ifft=%d must be a power of two", N_ifft);
    FD_REQUIRE(N_d >= 2 && N_d % 2 == 0 && N_d <= N_ifft, "N_d=%d must be even and <= N_ifft", N_d);
    FD_REQUIRE(b0 >= 0 && B_loc >= 1 && b0 + B_loc <= B, "antenna range [%d,%d) outside [0,%d)", b0, b0 + B_loc, B);
    FD_REQUIRE(rho > 0.f, "rho must be > 0");
    smem = zf_smem(T, U, B);
    FD_REQUIRE(smem <= 227 * 1024, "U*B too large for one CTA (%zu bytes of shared memory)", smem);
    return FD_OK;
}

int zf_precoder_build(const void* h_taps, int T, int U, int B, int N_ifft, int N_d, float rho, int b0, int B_loc,
                      void* h_fd, void* P, float* alpha, void* workspace, size_t workspace_bytes,
                      cudaStream_t stream) {
    return zf_precoder_build_ex(h_taps, nullptr, 0.f, T, U, B, N_ifft, N_d, rho, b0, B_loc, h_fd, P, alpha, workspace,
                                workspace_bytes, stream);
}

int zf_precoder_build_ex(const void* h_taps, const void* h_err, float eta, int T, int U, int B, int N_ifft, int N_d,
                         float rho, int b0, int B_loc, void* h_fd, void* P, float* alpha, void* workspace,
                         size_t workspace_bytes, cudaStream_t stream) {
    FD_REQUIRE(alpha, "zf_precoder_build: NULL alpha");
    FD_REQUIRE(eta >= 0.f && eta <= 1.f, "zf_precoder_build_ex: eta=%g outside [0,1]", (double)eta);
    FD_REQUIRE(eta == 0.f || (h_err && aligned8(h_err)), "zf_precoder_build_ex: h_err required when eta > 0");
    size_t smem = 0;
    int rc = zf_validate(h_taps, h_fd, P, workspace, T, U, B, N_ifft, N_d, rho, b0, B_loc, smem);
    if (rc) return rc;
    FD_REQUIRE(workspace_bytes >= zf_workspace_bytes(N_d), "zf workspace too small");
    double* tr = (double*)workspace;
    double* dalpha = tr + N_d;
    int* flag = (int*)(dalpha + 1);
    if (cudaMemsetAsync(flag, 0, sizeof(int), stream) != cudaSuccess) return check_launch("zf memset");
    launch_zf_any((const float2*)h_taps, T, U, B, N_ifft, N_d, b0, B_loc, (float2*)h_fd, (float2*)P, tr, flag,
                  eta > 0.f ? (const float2*)h_err : nullptr, (double)eta, 1, smem, stream);
    rc = check_launch("zf_precoder_build");
    if (rc) return rc;
    k_zf_alpha<<<1, 256, 0, stream>>>(tr, N_d, (double)B * (double)N_ifft, (double)rho, dalpha, nullptr);
    const long long nP = (long long)B_loc * U * N_d;
    k_scale<<<(int)std::min<long long>((nP + 255) / 256, 148LL * 8), 256, 0, stream>>>((float2*)P, nP, 1, dalpha);
    rc = check_launch("zf_precoder_build (alpha)");
    if (rc) return rc;
    double a = 0.0;
    int bad = 0;
    if (cudaMemcpyAsync(&a, dalpha, sizeof(double), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
        return check_launch("zf_precoder_build (sync)");
    if (bad) {
        set_error("zf_precoder_build: Gram matrix not positive definite at some subcarrier");
        return FD_ERR_NUMERIC;
    }
    *alpha = (float)a;
    return FD_OK;
}

int zf_precoder_build_batched(const void* h_taps, int n_ch, int T, int U, int B, int N_ifft, int N_d, float rho,
                              int b0, int B_loc, void* h_fd, void* P, float* alpha, int* status, void* workspace,
                              size_t workspace_bytes, cudaStream_t stream) {
    FD_REQUIRE(n_ch >= 0 && n_ch <= 65535, "zf_precoder_build_batched: n_ch=%d outside [0,65535]", n_ch);
    if (n_ch == 0) return FD_OK;
    FD_REQUIRE(alpha != nullptr, "zf_precoder_build_batched: NULL alpha");
    size_t smem = 0;
    int rc = zf_validate(h_taps, h_fd, P, workspace, T, U, B, N_ifft, N_d, rho, b0, B_loc, smem);
    if (rc) return rc;
    FD_REQUIRE(workspace_bytes >= zf_batched_workspace_bytes(n_ch, N_d), "zf batched workspace too small");
    double* tr = (double*)workspace;
    double* dalpha = tr + (size_t)n_ch * N_d;
    int* flag = status ? status : (int*)(dalpha + n_ch);
    if (cudaMemsetAsync(flag, 0, sizeof(int), stream) != cudaSuccess) return check_launch("zf memset");
    launch_zf_any((const float2*)h_taps, T, U, B, N_ifft, N_d, b0, B_loc, (float2*)h_fd, (float2*)P, tr, flag,
                  nullptr, 0.0, n_ch, smem, stream);
    rc = check_launch("zf_precoder_build_batched");
    if (rc) return rc;
    k_zf_alpha<<<n_ch, 256, 0, stream>>>(tr, N_d, (double)B * (double)N_ifft, (double)rho, dalpha, alpha);
    const long long per = (long long)B_loc * U * N_d;
    k_scale<<<(int)std::min<long long>((per * n_ch + 255) / 256, 148LL * 16), 256, 0, stream>>>((float2*)P, per, n_ch,
                                                                                               dalpha);
    return check_launch("zf_precoder_build_batched (alpha)");
}

}  // extern "C"
