// gmp.cuh — per-antenna GMP PA (Eq. 9; reading A13) evaluated on a
// time-domain OFDM symbol staged in shared memory.
//
// Factorisation used on the GPU (same sum as Eq. 9, regrouped per memory tap l):
//     y_m = sum_l u_{m-l} * G_l(m-l),
//     G_l(q) = sum_p a_{p,l} e_q^{(p-1)/2}
//            + sum_{p>=3} sum_g ( b_{p,l,g} e_{q-g}^{(p-1)/2} + c_{p,l,g} e_{q+g}^{(p-1)/2} ),
// with e_q = |u_q|^2 (so |u|^(p-1) = e^((p-1)/2) needs no sqrt for odd p).
// Each thread evaluates RS samples at once so every broadcast coefficient load
// from shared memory feeds 2*RS FMAs; the envelope powers of the 2M+1 window
// slide with l in registers (fully unrolled on compile-time Kp, L, M).
#pragma once

#include "fft.cuh"

namespace fdpd {

constexpr int GMP_MAX_ORDERS = 8;
constexpr int GMP_MAX_L = 15;
constexpr int GMP_MAX_M = 7;

struct GmpDesc {
    int Kp, L, M, n_coef;
    int pw[GMP_MAX_ORDERS];   // (p - 1) / 2 per order
};

// Specialised path: orders = {1, 3, ..., 2 KP - 1}.
template <int KP, int L, int M, int RS>
__device__ __forceinline__ void gmp_group(const float2* __restrict__ usm, const float* __restrict__ esm,
                                          const float2* __restrict__ cf, int N, const int (&m)[RS],
                                          float2 (&out)[RS]) {
    constexpr int W = 2 * M + 1;
    constexpr int NP = KP > 1 ? KP - 1 : 1;
    constexpr int NA = KP * (L + 1);
    constexpr int NB = (KP - 1) * (L + 1) * M;
    const int mask = N - 1;
    float w[RS][W][NP];
#pragma unroll
    for (int r = 0; r < RS; ++r) {
        out[r] = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const float e = esm[(m[r] - M + i) & mask];
            w[r][i][0] = e;
#pragma unroll
            for (int k = 1; k < NP; ++k) w[r][i][k] = w[r][i][k - 1] * e;
        }
    }
#pragma unroll
    for (int l = 0; l <= L; ++l) {
        if (l > 0) {
#pragma unroll
            for (int r = 0; r < RS; ++r) {
#pragma unroll
                for (int i = W - 1; i >= 1; --i)
#pragma unroll
                    for (int k = 0; k < NP; ++k) w[r][i][k] = w[r][i - 1][k];
                const float e = esm[(m[r] - l - M) & mask];
                w[r][0][0] = e;
#pragma unroll
                for (int k = 1; k < NP; ++k) w[r][0][k] = w[r][0][k - 1] * e;
            }
        }
        float2 G[RS];
        const float2 a1 = cf[l];
#pragma unroll
        for (int r = 0; r < RS; ++r) G[r] = a1;
#pragma unroll
        for (int k = 1; k < KP; ++k) {
            const float2 a = cf[k * (L + 1) + l];
#pragma unroll
            for (int r = 0; r < RS; ++r) {
                G[r].x = fmaf(a.x, w[r][M][k - 1], G[r].x);
                G[r].y = fmaf(a.y, w[r][M][k - 1], G[r].y);
            }
        }
#pragma unroll
        for (int k = 1; k < KP; ++k)
#pragma unroll
            for (int g = 1; g <= M; ++g) {
                const float2 bb = cf[NA + ((k - 1) * (L + 1) + l) * M + (g - 1)];
                const float2 cc = cf[NA + NB + ((k - 1) * (L + 1) + l) * M + (g - 1)];
#pragma unroll
                for (int r = 0; r < RS; ++r) {
                    G[r].x = fmaf(bb.x, w[r][M - g][k - 1], G[r].x);
                    G[r].y = fmaf(bb.y, w[r][M - g][k - 1], G[r].y);
                    G[r].x = fmaf(cc.x, w[r][M + g][k - 1], G[r].x);
                    G[r].y = fmaf(cc.y, w[r][M + g][k - 1], G[r].y);
                }
            }
#pragma unroll
        for (int r = 0; r < RS; ++r) {
            const float2 ul = usm[pidx((m[r] - l) & mask)];
            out[r] = cfma(ul, G[r], out[r]);
        }
    }
}

__device__ __forceinline__ float ipow(float e, int n) {
    float r = 1.f;
    for (int i = 0; i < n; ++i) r *= e;
    return r;
}

// Generic path: any odd ascending orders, runtime Kp, L, M.
__device__ __forceinline__ float2 gmp_sample_generic(const float2* __restrict__ usm, const float* __restrict__ esm,
                                                     const float2* __restrict__ cf, int N, int m, const GmpDesc& d) {
    const int mask = N - 1;
    const int NA = d.Kp * (d.L + 1);
    const int NB = (d.Kp - 1) * (d.L + 1) * d.M;
    float2 out = make_float2(0.f, 0.f);
    for (int l = 0; l <= d.L; ++l) {
        const int q = m - l;
        float2 G = make_float2(0.f, 0.f);
        const float e0 = esm[q & mask];
        for (int k = 0; k < d.Kp; ++k) {
            const float2 a = cf[k * (d.L + 1) + l];
            const float p = ipow(e0, d.pw[k]);
            G.x = fmaf(a.x, p, G.x);
            G.y = fmaf(a.y, p, G.y);
        }
        for (int k = 1; k < d.Kp; ++k)
            for (int g = 1; g <= d.M; ++g) {
                const float2 bb = cf[NA + ((k - 1) * (d.L + 1) + l) * d.M + (g - 1)];
                const float2 cc = cf[NA + NB + ((k - 1) * (d.L + 1) + l) * d.M + (g - 1)];
                const float pb = ipow(esm[(q - g) & mask], d.pw[k]);
                const float pc = ipow(esm[(q + g) & mask], d.pw[k]);
                G.x = fmaf(bb.x, pb, G.x);
                G.y = fmaf(bb.y, pb, G.y);
                G.x = fmaf(cc.x, pc, G.x);
                G.y = fmaf(cc.y, pc, G.y);
            }
        out = cfma(usm[pidx(q & mask)], G, out);
    }
    return out;
}

// Evaluate the GMP over the whole staged symbol and stream it to y (global).
// Sample groups: thread handles m_r = i0 + r * (N / RS), i0 = tid, tid + T, ...
// (consecutive threads -> consecutive samples: conflict-free LDS, coalesced STG).
// KP == 0 selects the generic path.
template <int KP, int L, int M, int RS>
__device__ __forceinline__ void gmp_symbol(const float2* __restrict__ usm, const float* __restrict__ esm,
                                           const float2* __restrict__ cf, int N, const GmpDesc& d,
                                           float2* __restrict__ y, int tid, int T) {
    if constexpr (KP > 0) {
        const int stride = N / RS;
        for (int i0 = tid; i0 < stride; i0 += T) {
            // keep the broadcast coefficient loads inside the loop (no hoisting of all
            // n_coef complex values into registers, which would cap occupancy)
            asm volatile("" ::: "memory");
            int m[RS];
            float2 out[RS];
#pragma unroll
            for (int r = 0; r < RS; ++r) m[r] = i0 + r * stride;
            gmp_group<KP, L, M, RS>(usm, esm, cf, N, m, out);
#pragma unroll
            for (int r = 0; r < RS; ++r) y[m[r]] = out[r];
        }
    } else {
        for (int m = tid; m < N; m += T) y[m] = gmp_sample_generic(usm, esm, cf, N, m, d);
    }
}

}  // namespace fdpd
