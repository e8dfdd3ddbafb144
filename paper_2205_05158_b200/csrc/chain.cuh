// chain.cuh — the fused per-(symbol, antenna) chain kernel k_chain_tx and its launcher,
// shared by tx.cu (generic instantiations) and tx_pruned.cu (pruned-FFT instantiations).
#pragma once

#include "gmp.cuh"

namespace fdpd {

// ============================================================================ fused chain_tx
// Shared-memory layout of k_chain_tx (byte offsets): FFT buffer / swizzled u | e (or the
// compact precoded spectrum, whichever is larger) | GMP coefficients | optional y copy.
struct ChainSmem {
    int off_e, off_cf, off_y, bytes;
};
__host__ __device__ inline ChainSmem chain_smem(int N, int N_d, const GmpDesc& d, bool ysm) {
    ChainSmem s;
    const int r16 = 15;
    s.off_e = ((int)sizeof(float2) * padded_len(N) + r16) & ~r16;   // 16-B aligned: float4 window loads (N = 16)
    const int e_bytes = ((N * 4 > N_d * 8 ? N * 4 : N_d * 8) + r16) & ~r16;
    s.off_cf = s.off_e + e_bytes;
    s.off_y = s.off_cf + ((8 * coef_smem_elems(d.Kp, d.L, d.M) + r16) & ~r16);
    s.bytes = s.off_y + (ysm ? (int)sizeof(float2) * padded_len(N) : 0);
    return s;
}
// keep a shared-memory copy of y for the receive DFT when it still allows 2 CTAs/SM
template <int LOG2N>
__host__ __device__ constexpr bool chain_ysm() { return LOG2N <= 11; }

// One CTA per (symbol n, antenna b): precode at the data bins straight into the
// pass-0 registers, IDFT in shared memory, 1/sqrt(N) scale + envelope, GMP, stream y.
//
// RX = true (chain_txrx): the PA output also feeds the receive DFT in the same CTA —
// the PA waveform is re-read from this CTA's shared-memory copy (N <= 4096) or through
// L2, transformed, and XPA at the data bins (Eq. 4 input) is written; y is still
// streamed out to HBM as the chain's product.
//
// PZ > 0 (pruned FFT passes, see fft.cuh): the data bins fill only slots r < PZ and
// r >= 16 - PZ of the radix-16 pass whose points are N/16 apart — the IDFT's first pass
// reads at most 4 non-zero inputs per butterfly and (N = 16^k) the receive DFT's last
// pass computes only the outputs at data bins and writes XPA straight from registers.
template <int LOG2N, int KP, int L, int M, int RS, bool RX, int PZ = 0>
__global__ void __launch_bounds__(fft_threads<LOG2N>(), fft_min_blocks<LOG2N>())
    k_chain_tx(const float2* __restrict__ P, const float2* __restrict__ s, const float2* __restrict__ coef,
               float2* __restrict__ y, float2* __restrict__ XPA, const float2* __restrict__ tw, int B, int U,
               int N_d, float sc, GmpDesc d, Impair imp) {
    constexpr int N = 1 << LOG2N, T = fft_threads<LOG2N>(), VPT = N / T;
    static_assert(PZ == 0 || n_passes<LOG2N>() >= 2, "pruned first pass needs a later pass");
    constexpr bool YSM = RX && KP > 0 && chain_ysm<LOG2N>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const ChainSmem lay = chain_smem(N, N_d, d, YSM);
    float2* usm = reinterpret_cast<float2*>(smem_raw);
    float* esm = reinterpret_cast<float*>(smem_raw + lay.off_e);
    float2* cf = reinterpret_cast<float2*>(smem_raw + lay.off_cf);
    float2* ysm = reinterpret_cast<float2*>(smem_raw + lay.off_y);
    const int tid = threadIdx.x;
    const size_t nb = blockIdx.x;
    const int b = (int)(nb % B);
    const size_t n = nb / B;
    // PA clip / measurement noise (NEXT f3), global sample index ((sym0 + n) B_total + b0 + b) N + m
    const bool impaired = imp.clip > 0.f || imp.pa_std > 0.f;
    const Impair* im = impaired ? &imp : nullptr;
    const unsigned long long nbase =
        ((unsigned long long)(imp.sym0 + (long long)n) * imp.B_total + imp.b0 + b) * (unsigned long long)N;
    // precode (Eq. 1) of the data subcarriers into a compact smem spectrum xs (aliases the
    // e region, unused until after the IDFT), with coalesced L2 loads issued 8 at a time.
    // (Measured alternative: staging P_b and s_n with two TMA bulk copies behind an
    // mbarrier was 6% slower on C2 — every thread then waits for the whole 38 KB.)
    float2* xs = reinterpret_cast<float2*>(esm);
    stage_coefs<KP, L, M>(coef + (size_t)b * d.n_coef, cf, d, tid, T);
    const float2* Pb = P + (size_t)n * imp.p_stride + (size_t)b * U * N_d;
    const float2* sn = s + n * U * N_d;
    if constexpr (PZ > 0) {
        // (PZ > 0: the precode is fused into the sparse first IDFT pass below)
    } else if (imp.precoded) {
        // P holds the precoded spectrum X [n_sym][B][N_d] (chain_txrx_pre): one coalesced
        // pass over the symbol-antenna row into xs
        const float2* Xr = P + nb * N_d;
        for (int j = tid; j < N_d; j += T) xs[j] = cscale(__ldg(Xr + j), sc);
    } else {
        // (Measured: a 4-subcarrier x 4-user predicated batch of 32 loads was 3% slower on
        // C2 than this loop — the extra address arithmetic outweighs the fewer round trips.)
        for (int j = tid; j < N_d; j += T) {
            const float2* pp = Pb + j;
            const float2* sp = sn + j;
            float2 acc = make_float2(0.f, 0.f);
            int u = 0;
            for (; u + 4 <= U; u += 4) {   // 8 independent loads in flight
                float2 pv[4], sv[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    pv[k] = __ldg(pp + k * N_d);
                    sv[k] = __ldg(sp + k * N_d);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) acc = cfma(pv[k], sv[k], acc);
                pp += 4 * N_d;
                sp += 4 * N_d;
            }
            for (; u < U; ++u, pp += N_d, sp += N_d) acc = cfma(__ldg(pp), __ldg(sp), acc);
            xs[j] = cscale(acc, sc);   // the IDFT's N^-1/2 on the N_d data bins instead of the N outputs
        }
    }
    if constexpr (PZ == 0) __syncthreads();
    float2 v[VPT];
    const int h = N_d >> 1;
    if constexpr (PZ > 0) {
        // sparse first IDFT pass: slots r = 0, 15 (and 1, 14 for PZ = 2) of each butterfly.
        // The slots of the radix-16 pass partition the data bins, so each thread precodes
        // exactly the (2 PZ) bins its butterflies read, straight into registers: no compact
        // spectrum in shared memory and no barrier between the precode and the first pass.
        static_assert(pass_radix<LOG2N>(0) == 16, "pruned pass 0 needs radix 16");
        constexpr int NB = 2 * PZ;
        const float2* Xr = P + nb * N_d;
#pragma unroll
        for (int q = 0; q < VPT / 16; ++q) {
            const int j = tid + q * T;
            int pos[NB];
            pos[0] = j;
            pos[NB - 1] = j + 15 * (N / 16);
            if constexpr (PZ == 2) {
                pos[1] = j + N / 16;
                pos[2] = j + 14 * (N / 16);
            }
            int jd[NB];
            bool ok[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const bool lo = pos[i] < h, hi = pos[i] >= N - h;
                ok[i] = lo || hi;
                jd[i] = lo ? pos[i] + h : (hi ? pos[i] - (N - h) : 0);
            }
            float2 xb[NB];
            if (imp.precoded) {
#pragma unroll
                for (int i = 0; i < NB; ++i) xb[i] = ok[i] ? cscale(__ldg(Xr + jd[i]), sc) : make_float2(0.f, 0.f);
            } else {
                float2 acc[NB];
#pragma unroll
                for (int i = 0; i < NB; ++i) acc[i] = make_float2(0.f, 0.f);
                for (int u = 0; u < U; u += 2) {   // 2 users x NB bins x 2 operands in flight
                    float2 pv[2][NB], sv[2][NB];
#pragma unroll
                    for (int k = 0; k < 2; ++k)
#pragma unroll
                        for (int i = 0; i < NB; ++i) {
                            const bool o = ok[i] && u + k < U;
                            const int e = (u + k) * N_d + jd[i];
                            pv[k][i] = o ? __ldg(Pb + e) : make_float2(0.f, 0.f);
                            sv[k][i] = o ? __ldg(sn + e) : make_float2(0.f, 0.f);
                        }
#pragma unroll
                    for (int k = 0; k < 2; ++k)
#pragma unroll
                        for (int i = 0; i < NB; ++i) acc[i] = cfma(pv[k][i], sv[k][i], acc[i]);
                }
#pragma unroll
                for (int i = 0; i < NB; ++i) xb[i] = ok[i] ? cscale(acc[i], sc) : make_float2(0.f, 0.f);
            }
            const float2 x0 = xb[0], x15 = xb[NB - 1];
            const float2 x1 = PZ == 2 ? xb[1] : make_float2(0.f, 0.f);
            const float2 x14 = PZ == 2 ? xb[NB - 2] : make_float2(0.f, 0.f);
            float2 X[16];
            dft16_sparse_in<+1, PZ>(x0, x1, x14, x15, X);
#pragma unroll
            for (int r = 0; r < 16; ++r) usm[17 * j + r] = X[r];   // = pidx(16 j + r)
        }
        __syncthreads();
        if constexpr (KP > 0) {
            if constexpr (n_passes<LOG2N>() > 2) fft_run<LOG2N, +1, 1, n_passes<LOG2N>() - 1>(usm, v, tw, tid);
        } else {
            fft_run<LOG2N, +1, 1>(usm, v, tw, tid);
        }
    } else {
        // branch-free pass-0 fill: data bins are [0, N_d/2) and [N - N_d/2, N) (reading A7)
        constexpr int R0 = pass_radix<LOG2N>(0);
#pragma unroll
        for (int q = 0; q < VPT / R0; ++q)
#pragma unroll
            for (int r = 0; r < R0; ++r) {
                const int pos = pass_pos<R0, VPT, T, N>(tid, q, r);
                const bool lo = pos < h, hi = pos >= N - h;
                const int jj = lo ? pos + h : pos - (N - h);
                const float2 t = xs[(lo || hi) ? jj : 0];
                v[q * R0 + r] = (lo || hi) ? t : make_float2(0.f, 0.f);
            }
        if constexpr (KP > 0) {
            if constexpr (n_passes<LOG2N>() > 1) fft_run<LOG2N, +1, 0, n_passes<LOG2N>() - 1>(usm, v, tw, tid);
        } else {
            fft_run<LOG2N, +1>(usm, v, tw, tid);
        }
    }
    if constexpr (KP > 0) {
        // last IDFT pass, storing u and e = |u|^2 straight into the swizzled run layouts of the
        // GMP (no natural-order store + reload + barrier; the N^-1/2 is already in xs)
        using Lay = RunLayout<RS>;
        constexpr int PL_ = n_passes<LOG2N>() - 1;
        constexpr int RL = pass_radix<LOG2N>(PL_), NSL = pass_ns<LOG2N>(PL_);
        constexpr bool FIRST_IS_LAST = PL_ == 0;
        if constexpr (!FIRST_IS_LAST || PZ > 0) {
            // pass-0 data came in registers only when the last pass is pass 0 without pruning
            pass_load_smem<RL, VPT, T, N>(usm, v, tid);
            __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < VPT / RL; ++q) {
            const int j = tid + q * T;
            const int k = j & (NSL - 1);
            if constexpr (NSL > 1) {
                if constexpr (RL == 16) pass_twiddle_tab16<+1>(v, q * RL, k, NSL, tw + tw_pass_off(N, PL_));
                else pass_twiddle<RL, +1>(v, q * RL, k * (N / (NSL * RL)), tw);
            }
            dftR<RL, +1>(v, q * RL);
            const int dd = (j - k) * RL + k;
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                const int i = dd + r * NSL;
                const float2 x = v[q * RL + r];
                usm[Lay::u_phys(i)] = x;
                esm[Lay::e_phys(i)] = fmaf(x.x, x.x, x.y * x.y);
            }
        }
        __syncthreads();
        float2* yo = y + nb * N;
        gmp_runs_symbol<KP, L, M, RS, YSM>(usm, esm, cf, N, yo, tid, T, ysm, im, nbase);
        if constexpr (RX) {
            __syncthreads();   // y of the whole CTA is written (CTA-scope visibility) and u is no longer read
            constexpr int R0 = pass_radix<LOG2N>(0);
#pragma unroll
            for (int q = 0; q < VPT / R0; ++q)
#pragma unroll
                for (int r = 0; r < R0; ++r) {
                    const int pos = pass_pos<R0, VPT, T, N>(tid, q, r);
                    if constexpr (YSM) v[q * R0 + r] = ysm[pidx(pos)];
                    else v[q * R0 + r] = __ldcg(yo + pos);
                }
            float2* xo = XPA + nb * N_d;
            if constexpr (PZ > 0 && LOG2N % 4 == 0) {
                // all but the last pass, then the last radix-16 pass at the data bins only
                constexpr int NPS = n_passes<LOG2N>();
                fft_run<LOG2N, -1, 0, NPS - 1>(usm, v, tw, tid);
                pass_load_smem<16, VPT, T, N>(usm, v, tid);
#pragma unroll
                for (int q = 0; q < VPT / 16; ++q) {
                    const int j = tid + q * T;         // < N/16 = Ns: twiddle step j, outputs j + r N/16
                    pass_twiddle_tab16<-1>(v, q * 16, j, N / 16, tw + tw_pass_off(N, NPS - 1));
                    float2 out[2 * PZ];
                    dft16_sparse_out<-1, PZ>(v, q * 16, out);
#pragma unroll
                    for (int o = 0; o < 2 * PZ; ++o) {
                        const int r = o < PZ ? o : 16 - 2 * PZ + o;
                        const int k = j + r * (N / 16);
                        if (k < h) xo[k + h] = cscale(out[o], sc);
                        else if (k >= N - h) xo[k - (N - h)] = cscale(out[o], sc);
                    }
                }
            } else {
                fft_run<LOG2N, -1>(usm, v, tw, tid);
                for (int j = tid; j < N_d; j += T) xo[j] = cscale(usm[pidx(data_to_bin(j, N, N_d))], sc);
            }
        }
        return;
    }
    for (int i = tid; i < N; i += T) {
        const float2 t = usm[pidx(i)];   // already scaled (xs carries N^-1/2)
        esm[i] = fmaf(t.x, t.x, t.y * t.y);
    }
    __syncthreads();
    if constexpr (!RX) {
        gmp_symbol<KP, L, M, RS>(usm, esm, cf, N, d, y + nb * N, tid, T, im, nbase);
    } else {
        gmp_symbol_to_fft<LOG2N, KP, L, M, RS>(usm, esm, cf, d, y ? y + nb * N : nullptr, tid, v, im, nbase);
        __syncthreads();                       // every lagged read of u is done before the FFT overwrites it
        fft_run<LOG2N, -1>(usm, v, tw, tid);
        float2* xo = XPA + nb * N_d;
        for (int j = tid; j < N_d; j += T) xo[j] = cscale(usm[pidx(data_to_bin(j, N, N_d))], sc);
    }
}

template <typename K>
inline void set_smem(K kernel, size_t bytes) {
    // opt-in above the 48 KB default; idempotent and cheap after the first call
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int LOG2N, int KP, int L, int M, int RS, bool RX, int PZ = 0>
inline int launch_chain_one(const float2* P, const float2* s, const float2* coef, float2* y, float2* XPA,
                            long long n_sym, int B, int U, int N_d, const GmpDesc& d, const Impair& imp,
                            cudaStream_t st) {
    constexpr int N = 1 << LOG2N;
    const float2* tw = twiddle_table(N, st);
    if (!tw) { set_error("twiddle table allocation failed"); return FD_ERR_CUDA; }
    const ChainSmem lay = chain_smem(N, N_d, d, RX && KP > 0 && chain_ysm<LOG2N>());
    const size_t smem = lay.bytes;
    if (smem > 227 * 1024) return fail_arg("chain_tx: shared-memory footprint %zu B too large", smem);
    set_smem(k_chain_tx<LOG2N, KP, L, M, RS, RX, PZ>, smem);
    k_chain_tx<LOG2N, KP, L, M, RS, RX, PZ><<<(unsigned)(n_sym * B), fft_threads<LOG2N>(), smem, st>>>(
        P, s, coef, y, XPA, tw, B, U, N_d, (float)(1.0 / std::sqrt((double)N)), d, imp);
    return check_launch(RX ? "chain_txrx" : "chain_tx");
}


// Cluster-split chain_txrx for N = 8192 / 16384 (chain_cl.cu); returns -1 when it does not apply.
int launch_chain_cluster(int log2n, int variant, const float2* P, const float2* s, const float2* coef, float2* y,
                         float2* XPA, long long n_sym, int B, int U, int N_d, const GmpDesc& d, const Impair& imp,
                         cudaStream_t st);
// Pruned-FFT chain_txrx instantiations (tx_pruned.cu); returns -1 when none matches.
int launch_chain_pruned(int log2n, int variant, int pz, const float2* P, const float2* s, const float2* coef,
                        float2* y, float2* XPA, long long n_sym, int B, int U, int N_d, const GmpDesc& d,
                        const Impair& imp, cudaStream_t st);

}  // namespace fdpd
