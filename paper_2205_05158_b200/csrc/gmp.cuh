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

// Shared-memory coefficient layout of the specialised path, per memory tap l
// (STRIDE complex, 16-byte aligned rows): a_{0..KP-1,l} padded to an even count,
// then (b_{k,l,g}, c_{k,l,g}) pairs for k = 1..KP-1, g = 1..M, so one 128-bit
// broadcast load yields two coefficients.
template <int KP, int M>
struct CoefRow {
    static constexpr int KPE = (KP + 1) & ~1;
    static constexpr int STRIDE = KPE + 2 * (KP - 1) * M;
};

// Number of complex slots the coefficient staging needs (>= n_coef for any layout).
__host__ __device__ inline int coef_smem_elems(int Kp, int L, int M) {
    return (L + 1) * (((Kp + 1) & ~1) + 2 * (Kp - 1) * M);
}

// Stage antenna b's coefficients (global, SURVEY §8(b) order) into shared memory:
// the paired layout for the specialised path (KP > 0), a plain copy otherwise.
template <int KP, int L, int M>
__device__ __forceinline__ void stage_coefs(const float2* __restrict__ cg, float2* __restrict__ cs, const GmpDesc& d,
                                            int tid, int T) {
    if constexpr (KP > 0) {
        using Row = CoefRow<KP, M>;
        constexpr int NA = KP * (L + 1);
        constexpr int NB = (KP - 1) * (L + 1) * M;
        for (int i = tid; i < (L + 1) * Row::STRIDE; i += T) {
            const int l = i / Row::STRIDE, o = i % Row::STRIDE;
            int src = -1;
            if (o < Row::KPE) {
                if (o < KP) src = o * (L + 1) + l;
            } else {
                const int o2 = o - Row::KPE, pr = o2 >> 1;
                const int k = pr / M + 1, g = pr % M + 1;
                src = NA + ((k - 1) * (L + 1) + l) * M + (g - 1) + ((o2 & 1) ? NB : 0);
            }
            cs[i] = src >= 0 ? cg[src] : make_float2(0.f, 0.f);
        }
    } else {
        for (int i = tid; i < d.n_coef; i += T) cs[i] = cg[i];
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

// Generic path over the whole staged symbol (pidx layout): any odd ascending orders,
// runtime Kp, L, M; y (global) gets N samples.  (The specialised shapes use the run-based
// evaluation below.)
template <int KP, int L, int M, int RS>
__device__ __forceinline__ void gmp_symbol(const float2* __restrict__ usm, const float* __restrict__ esm,
                                           const float2* __restrict__ cf, int N, const GmpDesc& d,
                                           float2* __restrict__ y, int tid, int T, const Impair* im = nullptr,
                                           unsigned long long nbase = 0) {
    for (int m = tid; m < N; m += T) {
        const float2 o = gmp_sample_generic(usm, esm, cf, N, m, d);
        y[m] = im ? pa_impair(o, nbase + m, *im) : o;
    }
}

// Same as gmp_symbol for a CTA of T = fft_threads threads, but also leaves this thread's
// outputs in `v` in the pass-0 register layout of the N-point FFT (fft.cuh pass_pos): the
// samples a thread evaluates, {tid + T j : j < N/T}, are exactly its pass-0 FFT inputs, so the
// receive DFT starts without a shared-memory round trip.  y may be NULL (waveform not stored).
template <int LOG2N, int KP, int L, int M, int RS>
__device__ __forceinline__ void gmp_symbol_to_fft(const float2* __restrict__ usm, const float* __restrict__ esm,
                                                  const float2* __restrict__ cf, const GmpDesc& d,
                                                  float2* __restrict__ y, int tid,
                                                  float2 (&v)[(1 << LOG2N) / fft_threads<LOG2N>()],
                                                  const Impair* im = nullptr, unsigned long long nbase = 0) {
    constexpr int N = 1 << LOG2N, T = fft_threads<LOG2N>(), VPT = N / T, R0 = pass_radix<LOG2N>(0);
    constexpr int QN = VPT / R0;      // pass-0 butterflies per thread
    // register slot of sample tid + T*j in the pass-0 layout: j = q + QN * r'
    auto slot = [](int j) { return (j % QN) * R0 + (j / QN); };
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int m = tid + T * j;
        float2 o = gmp_sample_generic(usm, esm, cf, N, m, d);
        if (im) o = pa_impair(o, nbase + m, *im);
        if (y) y[m] = o;
        v[slot(j)] = o;
    }
}

}  // namespace fdpd

namespace fdpd {

// =============================================================================
// Run-based specialised GMP (used by the fused kernels).
//
// Each thread evaluates runs of R contiguous samples [R rho, R rho + R).  The
// envelope window e[R rho - L - M, R rho + R - 1 + M] and the input window
// u[R rho - L, R rho + R - 1] are loaded once per run with 128-bit shared-memory
// loads into registers (compile-time indexed), so each e/u value is read once per
// run instead of once per (sample, tap).  u and e live in XOR-swizzled layouts
// (16-byte chunk x -> x ^ ((x >> 3) & (chunks_per_run - 1))), which makes both the
// per-run 128-bit window loads and the contiguous 8-byte relayout stores
// bank-conflict free.  Coefficient rows (CoefRow layout) are broadcast-loaded once
// per (run, tap) and feed R samples.
// =============================================================================
template <int R>
struct RunLayout {
    static constexpr int CPR_U = R / 2;   // 16-byte chunks per run of complex samples
    static constexpr int CPR_E = R / 4;   // 16-byte chunks per run of float envelopes
    __device__ static __forceinline__ int u_chunk(int x) { return x ^ ((x >> 3) & (CPR_U - 1)); }
    __device__ static __forceinline__ int e_chunk(int x) { return CPR_E > 1 ? x ^ ((x >> 3) & (CPR_E - 1)) : x; }
    __device__ static __forceinline__ int u_phys(int m) { return (u_chunk(m >> 1) << 1) | (m & 1); }
    __device__ static __forceinline__ int e_phys(int m) { return (e_chunk(m >> 2) << 2) | (m & 3); }
};

// HALO (cluster-split symbols, chain_cl.cu): this CTA holds one half of the symbol's samples
// (N local); window chunks left of 0 or right of N come from the partner CTA's buffers
// (usw_r / esw_r, distributed shared memory), which hold the other half — for two halves the
// partner is both the left and the right (circular) neighbour.
//
// The memory taps l can be processed in chunks [L0, L1] (gmp_run_taps), each with its own
// envelope and input windows, so the registers hold the windows of one chunk only (see
// gmp_tap_chunk).  The summation order over l (and within each l) is the same either way.
__host__ __device__ constexpr int round_up_pow2(int x, int a) { return (x + a - 1) & ~(a - 1); }

template <int KP, int L, int M, int R, bool HALO, int L0, int L1>
__device__ __forceinline__ void gmp_run_taps(const float2* __restrict__ usw, const float* __restrict__ esw,
                                             const float2* __restrict__ cf, int N, int rho, float2 (&out)[R],
                                             const float2* usw_r, const float* esw_r) {
    using Row = CoefRow<KP, M>;
    using Lay = RunLayout<R>;
    constexpr int NP = KP > 1 ? KP - 1 : 1;
    // window of envelope samples m0 - E_LO .. m0 + E_HI - 1 (16-byte chunks): q = m0 + i - l +- g
    constexpr int E_LO = round_up_pow2(L1 + M, 4);
    constexpr int E_HI = round_up_pow2(R - L0 + M, 4);
    constexpr int E_N = E_LO + E_HI;
    // window of inputs m0 - U_LO .. m0 + U_HI - 1: q = m0 + i - l
    constexpr int U_LO = round_up_pow2(L1, 2);
    constexpr int U_HI = round_up_pow2(R - L0, 2);
    constexpr int U_N = U_LO + U_HI;
    static_assert(E_N > 0 && U_N > 0, "empty GMP window");
    const int m0 = R * rho;
    float ew[NP][E_N];
    {
        const float4* e4 = reinterpret_cast<const float4*>(esw);
        const int xm = N / 4 - 1;
#pragma unroll
        for (int c = 0; c < E_N / 4; ++c) {
            float4 t;
            if constexpr (HALO) {
                const int q = (m0 - E_LO) / 4 + c;
                const float4* src = (q < 0 || q > xm) ? reinterpret_cast<const float4*>(esw_r) : e4;
                t = src[Lay::e_chunk(q & xm)];
            } else {
                t = e4[Lay::e_chunk(((m0 - E_LO) / 4 + c) & xm)];
            }
            ew[0][4 * c + 0] = t.x;
            ew[0][4 * c + 1] = t.y;
            ew[0][4 * c + 2] = t.z;
            ew[0][4 * c + 3] = t.w;
        }
#pragma unroll
        for (int k = 1; k < NP; ++k)
#pragma unroll
            for (int i = 0; i < E_N; ++i) ew[k][i] = ew[k - 1][i] * ew[0][i];
    }
    float2 uw[U_N];
    {
        const float4* u4 = reinterpret_cast<const float4*>(usw);
        const int xm = N / 2 - 1;
#pragma unroll
        for (int c = 0; c < U_N / 2; ++c) {
            float4 t;
            if constexpr (HALO) {
                const int q = (m0 - U_LO) / 2 + c;
                const float4* src = (q < 0 || q > xm) ? reinterpret_cast<const float4*>(usw_r) : u4;
                t = src[Lay::u_chunk(q & xm)];
            } else {
                t = u4[Lay::u_chunk(((m0 - U_LO) / 2 + c) & xm)];
            }
            uw[2 * c] = make_float2(t.x, t.y);
            uw[2 * c + 1] = make_float2(t.z, t.w);
        }
    }
#pragma unroll
    for (int l = L0; l <= L1; ++l) {
        const float4* row = reinterpret_cast<const float4*>(cf + l * Row::STRIDE);
        float2 G[R];
        // window index of q = m0 + i - l + delta is  i - l + delta + E_LO
#pragma unroll
        for (int kk = 0; kk < Row::KPE / 2; ++kk) {
            const float4 q = row[kk];
            const float2 a0 = make_float2(q.x, q.y), a1 = make_float2(q.z, q.w);
#pragma unroll
            for (int i = 0; i < R; ++i) {
                G[i] = (kk == 0) ? a0 : cfma_real(a0, ew[2 * kk - 1][i - l + E_LO], G[i]);
                if (2 * kk + 1 < KP) G[i] = cfma_real(a1, ew[2 * kk][i - l + E_LO], G[i]);
            }
        }
#pragma unroll
        for (int k = 1; k < KP; ++k)
#pragma unroll
            for (int g = 1; g <= M; ++g) {
                const float4 q = row[Row::KPE / 2 + (k - 1) * M + (g - 1)];
                const float2 bb = make_float2(q.x, q.y), cc = make_float2(q.z, q.w);
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    G[i] = cfma_real(bb, ew[k - 1][i - l - g + E_LO], G[i]);
                    G[i] = cfma_real(cc, ew[k - 1][i - l + g + E_LO], G[i]);
                }
            }
#pragma unroll
        for (int i = 0; i < R; ++i) out[i] = cfma2(uw[i - l + U_LO], G[i], out[i]);
    }
}

// Taps per window chunk: all L + 1 at once.  (Two chunks of 4 taps at the C4 / C5 shape
// halved the envelope window held in registers, but recomputing the envelope powers per chunk
// cost more than the spills it removed once the FFT passes parked their inputs in shared memory:
// C5 chain 5.99 ms with one chunk vs 6.16 ms with two; -DFD_GMP_TAP_CHUNK=4 rebuilds the latter.)
#ifndef FD_GMP_TAP_CHUNK
#define FD_GMP_TAP_CHUNK 0
#endif
template <int KP, int L, int M>
__host__ __device__ constexpr int gmp_tap_chunk() { return FD_GMP_TAP_CHUNK > 0 ? FD_GMP_TAP_CHUNK : L + 1; }

template <int KP, int L, int M, int R, bool HALO, int L0>
__device__ __forceinline__ void gmp_run_chunks(const float2* __restrict__ usw, const float* __restrict__ esw,
                                               const float2* __restrict__ cf, int N, int rho, float2 (&out)[R],
                                               const float2* usw_r, const float* esw_r) {
    constexpr int LC = gmp_tap_chunk<KP, L, M>();
    constexpr int L1 = (L0 + LC - 1 < L) ? L0 + LC - 1 : L;
    gmp_run_taps<KP, L, M, R, HALO, L0, L1>(usw, esw, cf, N, rho, out, usw_r, esw_r);
    if constexpr (L1 < L) gmp_run_chunks<KP, L, M, R, HALO, L1 + 1>(usw, esw, cf, N, rho, out, usw_r, esw_r);
}

template <int KP, int L, int M, int R, bool HALO = false>
__device__ __forceinline__ void gmp_run(const float2* __restrict__ usw, const float* __restrict__ esw,
                                        const float2* __restrict__ cf, int N, int rho, float2 (&out)[R],
                                        const float2* usw_r = nullptr, const float* esw_r = nullptr) {
    static_assert(R % 4 == 0, "run length must be a multiple of 4");
#pragma unroll
    for (int i = 0; i < R; ++i) out[i] = make_float2(0.f, 0.f);
    gmp_run_chunks<KP, L, M, R, HALO, 0>(usw, esw, cf, N, rho, out, usw_r, esw_r);
}
// Whole symbol: relayout of the (already scaled) IDFT output held in the FFT buffer
// (pidx layout) into the swizzled u/e layouts, then all runs; y (global) gets R
// contiguous complex per run via 128-bit stores.  usw aliases the FFT buffer.
// ysm (optional): also store the outputs in shared memory in the FFT's pidx layout.
template <int KP, int L, int M, int R, bool YS = false, bool HALO = false>
__device__ __forceinline__ void gmp_runs_symbol(float2* __restrict__ buf, float* __restrict__ esw,
                                                const float2* __restrict__ cf, int N, float2* __restrict__ y,
                                                int tid, int T, float2* __restrict__ ysm = nullptr,
                                                const Impair* im = nullptr, unsigned long long nbase = 0,
                                                const float2* buf_r = nullptr, const float* esw_r = nullptr) {
#pragma unroll 1
    for (int rho = tid; rho < N / R; rho += T) {
        // keep the coefficient-row loads inside the loop (no hoisting into registers)
        asm volatile("" ::: "memory");
        float2 out[R];
        if constexpr (HALO) {
            // Only the first and the last warp-row of runs reach into the partner's half (windows of
            // at most 16 samples to either side): every other row takes the plain evaluation, whose
            // window loads are shared-memory loads at fixed offsets instead of generic loads behind a
            // pointer select per 16-byte chunk (~45 of the run's ~270 non-FFMA2 instructions).  The
            // choice is warp-uniform, and inside [0, N) both paths load the same values.
            const int row0 = (rho - (tid & 31)) * R;              // first sample of this warp-row
            if (row0 < 16 || row0 + 32 * R + 16 > N)
                gmp_run<KP, L, M, R, true>(buf, esw, cf, N, rho, out, buf_r, esw_r);
            else
                gmp_run<KP, L, M, R, false>(buf, esw, cf, N, rho, out);
        } else {
            gmp_run<KP, L, M, R, false>(buf, esw, cf, N, rho, out);
        }
        if (im) {
#pragma unroll
            for (int i = 0; i < R; ++i) out[i] = pa_impair(out[i], nbase + (unsigned long long)(R * rho + i), *im);
        }
        float4* y4 = reinterpret_cast<float4*>(y + (size_t)R * rho);
#pragma unroll
        for (int i = 0; i < R / 2; ++i) y4[i] = make_float4(out[2 * i].x, out[2 * i].y, out[2 * i + 1].x, out[2 * i + 1].y);
        if constexpr (YS) {
#pragma unroll
            for (int i = 0; i < R; ++i) ysm[pidx(R * rho + i)] = out[i];
        }
    }
}

}  // namespace fdpd
