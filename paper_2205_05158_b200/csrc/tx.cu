// tx.cu — transmit side of the hot path: precode (Eq. 1), OFDM IDFT (Eq. 2),
// GMP PA (Eq. 9), and the fused chain_tx (one CTA per (symbol, antenna)).
#include "chain.cuh"

namespace fdpd {

// ============================================================================ precode
// X[n][b][j] = sum_u P[b][u][j] s[n][u][j]          (Eq. 1)
// Per data subcarrier j the contraction is a small complex GEMM X_j[n][b] = sum_u s_j[n][u]
// P_j[b][u] (K = U); a thread-per-output kernel re-reads P_b for every symbol and s_n for
// every antenna (U-fold L2 gathers per output, the first version).  Here a CTA
// owns 32 consecutive subcarriers (lane = j: coalesced 256-byte rows) x NT symbols x a range
// of antennas: s_n for its NT symbols is staged once in shared memory ([NT][U][32], reused by
// every antenna), and each thread accumulates NT x BPT outputs, so a P value fetched from L2
// feeds NT symbols and an s value from shared memory BPT antennas.  The u summation order
// (ascending, one complex FMA per term) is the same as the fused chains.
constexpr int PC_NT = 8, PC_BPT = 4, PC_WARPS = 8;
template <int NT, int BPT>
__global__ void __launch_bounds__(32 * PC_WARPS) k_precode_tile(const float2* __restrict__ P, const float2* __restrict__ s,
                                                                float2* __restrict__ X, long long n_sym, int B, int U,
                                                                int N_d, int b_per_cta) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* ssm = reinterpret_cast<float2*>(smem_raw);   // [NT][U][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = blockIdx.y * 32 + lane;
    const bool jok = j < N_d;
    const long long n0 = (long long)blockIdx.x * NT;
    const int nt = (int)min((long long)NT, n_sym - n0);
    for (int e = threadIdx.x; e < NT * U * 32; e += blockDim.x) {
        const int l = e & 31, r = e >> 5, u = r % U, n = r / U;
        const int jj = blockIdx.y * 32 + l;
        ssm[e] = (n < nt && jj < N_d) ? __ldg(s + ((size_t)(n0 + n) * U + u) * N_d + jj) : make_float2(0.f, 0.f);
    }
    __syncthreads();
    const int b_begin = blockIdx.z * b_per_cta, b_end = min(B, b_begin + b_per_cta);
    for (int b0 = b_begin + warp * BPT; b0 < b_end; b0 += PC_WARPS * BPT) {
        float2 acc[NT][BPT];
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int t = 0; t < BPT; ++t) acc[n][t] = make_float2(0.f, 0.f);
        const float2* Pb = P + (size_t)b0 * U * N_d + (jok ? j : 0);
        int u = 0;
        // 4 users x BPT antennas of P in flight per step (the loop is latency-bound otherwise)
        for (; u + 4 <= U; u += 4) {
            float2 pv[4][BPT];
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int t = 0; t < BPT; ++t)
                    pv[q][t] = (b0 + t < b_end) ? __ldg(Pb + ((size_t)t * U + u + q) * N_d) : make_float2(0.f, 0.f);
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const float2 sv = ssm[(n * U + u + q) * 32 + lane];
#pragma unroll
                    for (int t = 0; t < BPT; ++t) acc[n][t] = cfma(pv[q][t], sv, acc[n][t]);
                }
        }
        for (; u < U; ++u) {
            float2 pv[BPT];
#pragma unroll
            for (int t = 0; t < BPT; ++t)
                pv[t] = (b0 + t < b_end) ? __ldg(Pb + ((size_t)t * U + u) * N_d) : make_float2(0.f, 0.f);
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                const float2 sv = ssm[(n * U + u) * 32 + lane];
#pragma unroll
                for (int t = 0; t < BPT; ++t) acc[n][t] = cfma(pv[t], sv, acc[n][t]);
            }
        }
        if (jok) {
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int t = 0; t < BPT; ++t)
                    if (n < nt && b0 + t < b_end) X[((size_t)(n0 + n) * B + b0 + t) * N_d + j] = acc[n][t];
        }
    }
}

// ============================================================================ helpers
template <int LOG2N>
__device__ __forceinline__ void load_spectrum(float2 (&v)[(1 << LOG2N) / fft_threads<LOG2N>()],
                                              const float2* __restrict__ Xnb, int N_d, int tid) {
    constexpr int N = 1 << LOG2N, T = fft_threads<LOG2N>(), VPT = N / T, R0 = pass_radix<LOG2N>(0);
#pragma unroll
    for (int q = 0; q < VPT / R0; ++q)
#pragma unroll
        for (int r = 0; r < R0; ++r) {
            const int jj = bin_to_data(pass_pos<R0, VPT, T, N>(tid, q, r), N, N_d);
            v[q * R0 + r] = jj >= 0 ? __ldg(Xnb + jj) : make_float2(0.f, 0.f);
        }
}

// ============================================================================ OFDM IDFT
// One CTA per (symbol, antenna).  N^-1/2 is applied to the N_d input bins; with PZ > 0 the
// first radix-16 pass is the sparse one (each thread loads exactly the 2 PZ data bins its
// butterflies read, see chain.cuh); the last pass writes its outputs straight to global memory
// (coalesced: for a fixed output slot r the warp's lanes write consecutive samples), so the
// waveform never makes a natural-order round trip through shared memory.
// (4 CTAs per SM up to N = 4096: no GMP state, so 64 registers suffice and the extra CTA
// keeps more of the waveform stores in flight)
template <int LOG2N>
__host__ __device__ constexpr int ofdm_min_blocks() { return LOG2N <= 12 ? 4 : fft_min_blocks<LOG2N>(); }
template <int LOG2N, int PZ>
__global__ void __launch_bounds__(fft_threads<LOG2N>(), ofdm_min_blocks<LOG2N>()) k_ofdm(const float2* __restrict__ X, float2* __restrict__ x,
                                                              const float2* __restrict__ tw, int B, int N_d, float sc) {
    constexpr int N = 1 << LOG2N, T = fft_threads<LOG2N>(), VPT = N / T, NPS = n_passes<LOG2N>();
    static_assert(PZ == 0 || NPS >= 2, "pruned first pass needs a later pass");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* sm = reinterpret_cast<float2*>(smem_raw);
    const int tid = threadIdx.x;
    const size_t nb = blockIdx.x;
    const float2* Xnb = X + nb * N_d;
    const int h = N_d >> 1;
    float2 v[VPT];
    if constexpr (PZ > 0) {
        constexpr int NB = 2 * PZ;
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
            float2 xb[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const bool lo = pos[i] < h, hi = pos[i] >= N - h;
                xb[i] = (lo || hi) ? cscale(__ldg(Xnb + (lo ? pos[i] + h : pos[i] - (N - h))), sc)
                                   : make_float2(0.f, 0.f);
            }
            float2 Y[16];
            dft16_sparse_in<+1, PZ>(xb[0], PZ == 2 ? xb[1] : make_float2(0.f, 0.f),
                                    PZ == 2 ? xb[NB - 2] : make_float2(0.f, 0.f), xb[NB - 1], Y);
#pragma unroll
            for (int r = 0; r < 16; ++r) sm[17 * j + r] = Y[r];   // = pidx(16 j + r)
        }
        __syncthreads();
        if constexpr (NPS > 2) fft_run<LOG2N, +1, 1, NPS - 1>(sm, v, tw, tid);
    } else {
        load_spectrum<LOG2N>(v, Xnb, N_d, tid);
#pragma unroll
        for (int i = 0; i < VPT; ++i) v[i] = cscale(v[i], sc);
        if constexpr (NPS > 1) fft_run<LOG2N, +1, 0, NPS - 1>(sm, v, tw, tid);
    }
    // last pass -> global
    constexpr int PL = NPS - 1, RL = pass_radix<LOG2N>(PL), NSL = pass_ns<LOG2N>(PL);
    if constexpr (PL > 0) pass_load_smem<RL, VPT, T, N>(sm, v, tid);
    float2* xo = x + nb * N;
#pragma unroll
    for (int q = 0; q < VPT / RL; ++q) {
        const int j = tid + q * T;
        const int k = j & (NSL - 1);
        if constexpr (NSL > 1) {
            if constexpr (RL == 16) pass_twiddle_tab16<+1>(v, q * RL, k, NSL, tw + tw_pass_off(N, PL));
            else pass_twiddle<RL, +1>(v, q * RL, k * (N / (NSL * RL)), tw);
        }
        dftR<RL, +1>(v, q * RL);
        const int dd = (j - k) * RL + k;
#pragma unroll
        for (int r = 0; r < RL; ++r) xo[dd + r * NSL] = v[q * RL + r];
    }
}

// ============================================================================ GMP (standalone)
__host__ __device__ inline int gmp_off_e(int N) { return ((int)sizeof(float2) * padded_len(N) + 15) & ~15; }
__host__ __device__ inline int gmp_off_cf(int N) { return (gmp_off_e(N) + (int)sizeof(float) * N + 15) & ~15; }
template <int KP, int L, int M, int RS>
__global__ void __launch_bounds__(256, 2) k_gmp(const float2* __restrict__ x, const float2* __restrict__ coef,
                                             float2* __restrict__ y, int B, int N, GmpDesc d) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // regions 16-byte aligned (float4 window / coefficient loads; padded_len(16) * 8 = 136)
    float2* usm = reinterpret_cast<float2*>(smem_raw);
    float* esm = reinterpret_cast<float*>(smem_raw + gmp_off_e(N));
    float2* cf = reinterpret_cast<float2*>(smem_raw + gmp_off_cf(N));
    const int tid = threadIdx.x, T = blockDim.x;
    const size_t nb = blockIdx.x;
    const int b = (int)(nb % B);
    stage_coefs<KP, L, M>(coef + (size_t)b * d.n_coef, cf, d, tid, T);
    const float2* xi = x + nb * N;
    if constexpr (KP > 0) {
        // run-based evaluation (gmp.cuh, as in the fused chain): u and e = |u|^2 in the
        // swizzled run layouts, runs of 4 samples, 128-bit stores of y
        using Lay = RunLayout<4>;
        for (int i = tid; i < N; i += T) {
            const float2 t = __ldg(xi + i);
            usm[Lay::u_phys(i)] = t;
            esm[Lay::e_phys(i)] = fmaf(t.x, t.x, t.y * t.y);
        }
        __syncthreads();
        gmp_runs_symbol<KP, L, M, 4>(usm, esm, cf, N, y + nb * N, tid, T);
    } else {
        for (int i = tid; i < N; i += T) {
            const float2 t = xi[i];
            usm[pidx(i)] = t;
            esm[i] = fmaf(t.x, t.x, t.y * t.y);
        }
        __syncthreads();
        gmp_symbol<KP, L, M, RS>(usm, esm, cf, N, d, y + nb * N, tid, T);
    }
}

// ============================================================================ host side
static int validate_gmp(const int* orders, int n_orders, int L, int M, int N, GmpDesc& d, int& variant) {
    FD_REQUIRE(orders != nullptr, "orders is NULL");
    FD_REQUIRE(n_orders >= 1 && n_orders <= GMP_MAX_ORDERS, "n_orders=%d outside [1,%d]", n_orders, GMP_MAX_ORDERS);
    FD_REQUIRE(orders[0] == 1, "orders[0]=%d must be 1", orders[0]);
    for (int k = 0; k < n_orders; ++k) {
        FD_REQUIRE(orders[k] >= 1 && (orders[k] & 1), "orders[%d]=%d must be odd", k, orders[k]);
        FD_REQUIRE(k == 0 || orders[k] > orders[k - 1], "orders must be ascending");
        FD_REQUIRE(orders[k] <= 31, "orders[%d]=%d too large", k, orders[k]);
    }
    FD_REQUIRE(L >= 0 && L <= GMP_MAX_L, "L=%d outside [0,%d]", L, GMP_MAX_L);
    FD_REQUIRE(M >= 0 && M <= GMP_MAX_M, "M=%d outside [0,%d]", M, GMP_MAX_M);
    FD_REQUIRE(L + 2 * M < N, "L + 2M = %d must be < N_ifft = %d", L + 2 * M, N);
    d.Kp = n_orders;
    d.L = L;
    d.M = M;
    d.n_coef = n_orders * (L + 1) + 2 * (n_orders - 1) * (L + 1) * M;
    bool consecutive = true;
    for (int k = 0; k < GMP_MAX_ORDERS; ++k) d.pw[k] = k < n_orders ? (orders[k] - 1) / 2 : 0;
    for (int k = 0; k < n_orders; ++k) consecutive &= (orders[k] == 2 * k + 1);
    variant = 0;
    if (consecutive) {
        if (n_orders == 3 && L == 2 && M == 1) variant = 1;
        else if (n_orders == 4 && L == 4 && M == 2) variant = 2;
        else if (n_orders == 5 && L == 6 && M == 3) variant = 3;
        else if (n_orders == 4 && L == 3 && M == 1) variant = 4;   // the paper's PA/DPD shape
    }
    return FD_OK;
}

static int validate_ofdm(long long n_sym, int B, int N_d, int N) {
    FD_REQUIRE(n_sym >= 0, "n_sym=%lld < 0", n_sym);
    FD_REQUIRE(B >= 1, "B=%d < 1", B);
    FD_REQUIRE(is_pow2(N) && N >= 16 && N <= 16384, "N_ifft=%d must be a power of two in [16, 16384]", N);
    FD_REQUIRE(N_d >= 2 && (N_d % 2) == 0 && N_d <= N, "N_d=%d must be even, >= 2 and <= N_ifft", N_d);
    FD_REQUIRE(n_sym * (long long)B <= 0x7fffffffLL, "n_sym*B too large");
    return FD_OK;
}

template <int LOG2N>
static int launch_ofdm(const float2* X, float2* x, long long n_sym, int B, int N_d, cudaStream_t st) {
    constexpr int N = 1 << LOG2N;
    const float2* tw = twiddle_table(N, st);
    if (!tw) { set_error("twiddle table allocation failed"); return FD_ERR_CUDA; }
    const size_t smem = sizeof(float2) * padded_len(N);
    const float sc = (float)(1.0 / std::sqrt((double)N));
    const int pz = LOG2N >= 8 ? prune_slots(N, N_d) : 0;
    auto go = [&](auto kern) {
        set_smem(kern, smem);
        kern<<<(unsigned)(n_sym * B), fft_threads<LOG2N>(), smem, st>>>(X, x, tw, B, N_d, sc);
    };
    if constexpr (LOG2N >= 8) {
        if (pz == 1) go(k_ofdm<LOG2N, 1>);
        else if (pz == 2) go(k_ofdm<LOG2N, 2>);
        else go(k_ofdm<LOG2N, 0>);
    } else {
        go(k_ofdm<LOG2N, 0>);
    }
    return check_launch("ofdm_modulate");
}

template <int KP, int L, int M, int RS>
static int launch_gmp(const float2* x, const float2* coef, float2* y, long long n_sym, int B, int N, const GmpDesc& d,
                      cudaStream_t st) {
    const size_t smem = (size_t)gmp_off_cf(N) + sizeof(float2) * coef_smem_elems(d.Kp, d.L, d.M);
    set_smem(k_gmp<KP, L, M, RS>, smem);
    k_gmp<KP, L, M, RS><<<(unsigned)(n_sym * B), 256, smem, st>>>(x, coef, y, B, N, d);
    return check_launch("gmp_pa");
}

template <int LOG2N, bool RX>
static int launch_chain(int variant, const float2* P, const float2* s, const float2* coef, float2* y, float2* XPA,
                        long long n_sym, int B, int U, int N_d, const GmpDesc& d, const Impair& imp,
                        cudaStream_t st) {
    if (RX) {
        const int rcl = launch_chain_cluster(LOG2N, variant, P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        if (rcl >= 0) return rcl;
        const int pz = prune_slots(1 << LOG2N, N_d);
        if (pz > 0) {
            const int rc = launch_chain_pruned(LOG2N, variant, pz, P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
            if (rc >= 0) return rc;
        }
    }
    switch (variant) {
        case 1: return launch_chain_one<LOG2N, 3, 2, 1, 8, RX>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        case 2: return launch_chain_one<LOG2N, 4, 4, 2, 4, RX>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        case 3: return launch_chain_one<LOG2N, 5, 6, 3, 4, RX>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        case 4: return launch_chain_one<LOG2N, 4, 3, 1, 4, RX>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        default: return launch_chain_one<LOG2N, 0, 0, 0, 1, RX>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
    }
}

#define FD_LOG2N_SWITCH(LOG2, CALL)        \
    switch (LOG2) {                        \
        case 4: { constexpr int LG = 4; return CALL; }   \
        case 5: { constexpr int LG = 5; return CALL; }   \
        case 6: { constexpr int LG = 6; return CALL; }   \
        case 7: { constexpr int LG = 7; return CALL; }   \
        case 8: { constexpr int LG = 8; return CALL; }   \
        case 9: { constexpr int LG = 9; return CALL; }   \
        case 10: { constexpr int LG = 10; return CALL; } \
        case 11: { constexpr int LG = 11; return CALL; } \
        case 12: { constexpr int LG = 12; return CALL; } \
        case 13: { constexpr int LG = 13; return CALL; } \
        case 14: { constexpr int LG = 14; return CALL; } \
        default: return fail_arg("unsupported N_ifft");   \
    }

}  // namespace fdpd

using namespace fdpd;

extern "C" {

}  // extern "C"

// FD_MATH_FP32 path of precode (precode_tc.cu dispatches on `math`)
namespace fdpd {
int precode_simt(const void* P, const void* s, void* X, long long n_sym, int B_loc, int U, int N_d,
                 cudaStream_t stream);
}
int fdpd::precode_simt(const void* P, const void* s, void* X, long long n_sym, int B_loc, int U, int N_d,
                       cudaStream_t stream) {
    FD_REQUIRE(n_sym >= 0 && B_loc >= 1 && U >= 1 && N_d >= 1, "precode: bad sizes");
    const long long total = n_sym * B_loc * (long long)N_d;
    if (total == 0) return FD_OK;
    FD_REQUIRE(P && s && X, "precode: NULL pointer");
    FD_REQUIRE(aligned8(P) && aligned8(s) && aligned8(X), "precode: pointers must be 8-byte aligned");
    FD_REQUIRE(N_d <= 65535 * 32, "precode: N_d=%d too large", N_d);
    const size_t smem = sizeof(float2) * PC_NT * U * 32;
    FD_REQUIRE(smem <= 200 * 1024, "precode: U=%d too large for the staged tile", U);
    // antenna split over grid.z so that even a short batch gives >= ~2 waves of CTAs
    const long long xy = (long long)((N_d + 31) / 32) * ((n_sym + PC_NT - 1) / PC_NT);
    int zc = 1;
    while (xy * zc < 2 * 148 * 4 && B_loc / (zc * 2) >= PC_WARPS * PC_BPT) zc *= 2;
    const int bpc = (B_loc + zc - 1) / zc;
    set_smem(k_precode_tile<PC_NT, PC_BPT>, smem);
    // symbol tiles fastest: the CTAs that share a (subcarrier tile, antenna range) slice of P run
    // together, so P streams from HBM once per call (432 MB at C5) instead of once per symbol tile
    dim3 grid((unsigned)((n_sym + PC_NT - 1) / PC_NT), (N_d + 31) / 32, zc);
    k_precode_tile<PC_NT, PC_BPT><<<grid, 32 * PC_WARPS, smem, stream>>>((const float2*)P, (const float2*)s,
                                                                        (float2*)X, n_sym, B_loc, U, N_d, bpc);
    return check_launch("precode");
}

extern "C" {

int ofdm_modulate(const void* X, void* x, long long n_sym, int B, int N_d, int N_ifft, cudaStream_t stream) {
    int rc = validate_ofdm(n_sym, B, N_d, N_ifft);
    if (rc) return rc;
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(X && x, "ofdm_modulate: NULL pointer");
    FD_REQUIRE(aligned16(X) && aligned16(x), "ofdm_modulate: pointers must be 16-byte aligned");
    const float2* Xp = (const float2*)X;
    float2* xp = (float2*)x;
    FD_LOG2N_SWITCH(ilog2(N_ifft), launch_ofdm<LG>(Xp, xp, n_sym, B, N_d, stream));
}

int gmp_pa(const void* x, const void* coef, void* y, const int* orders, int n_orders, int L, int M, long long n_sym,
           int B, int N_ifft, cudaStream_t stream) {
    FD_REQUIRE(n_sym >= 0 && B >= 1, "gmp_pa: bad sizes");
    FD_REQUIRE(n_sym == 0 || (x && coef && y), "gmp_pa: NULL pointer");
    FD_REQUIRE(n_sym == 0 || x != y, "gmp_pa: y must not alias x");
    FD_REQUIRE(n_sym == 0 || (aligned16(x) && aligned16(y) && aligned8(coef)), "gmp_pa: misaligned pointer");
    FD_REQUIRE(is_pow2(N_ifft) && N_ifft >= 16 && N_ifft <= 16384, "gmp_pa: N_ifft=%d unsupported", N_ifft);
    FD_REQUIRE(n_sym * (long long)B <= 0x7fffffffLL, "gmp_pa: n_sym*B too large");
    GmpDesc d;
    int variant = 0;
    int rc = validate_gmp(orders, n_orders, L, M, N_ifft, d, variant);
    if (rc) return rc;
    if (n_sym == 0) return FD_OK;
    const float2 *xp = (const float2*)x, *cp = (const float2*)coef;
    float2* yp = (float2*)y;
    switch (variant) {
        case 1: return launch_gmp<3, 2, 1, 4>(xp, cp, yp, n_sym, B, N_ifft, d, stream);
        case 2: return launch_gmp<4, 4, 2, 4>(xp, cp, yp, n_sym, B, N_ifft, d, stream);
        case 3: return launch_gmp<5, 6, 3, 2>(xp, cp, yp, n_sym, B, N_ifft, d, stream);
        case 4: return launch_gmp<4, 3, 1, 4>(xp, cp, yp, n_sym, B, N_ifft, d, stream);
        default: return launch_gmp<0, 0, 0, 1>(xp, cp, yp, n_sym, B, N_ifft, d, stream);
    }
}

static Impair to_impair(const fd_impair* pub, int B_loc) {
    Impair im{};
    im.B_total = B_loc;
    if (pub) {
        im.clip = pub->clip;
        im.pa_std = pub->pa_noise_std;
        im.awgn_std = pub->awgn_n0 > 0.f ? sqrtf(pub->awgn_n0) : 0.f;
        im.key_lo = (unsigned)(pub->noise_key & 0xffffffffull);
        im.key_hi = (unsigned)(pub->noise_key >> 32);
        im.sym0 = pub->sym0;
        im.b0 = pub->b0;
        im.B_total = pub->B_total > 0 ? pub->B_total : B_loc;
    }
    return im;
}

static int chain_tx_impl(const void* P, const void* s_tilde, const void* coef, void* y, const int* orders,
                         int n_orders, int L, int M, long long n_sym, int B_loc, int U, int N_d, int N_ifft,
                         const fd_impair* pub, cudaStream_t stream) {
    const Impair imp = to_impair(pub, B_loc);
    FD_REQUIRE(U >= 1 && U <= 1024, "chain_tx: bad U=%d", U);
    int rc = validate_ofdm(n_sym, B_loc, N_d, N_ifft);
    if (rc) return rc;
    GmpDesc d;
    int variant = 0;
    rc = validate_gmp(orders, n_orders, L, M, N_ifft, d, variant);
    if (rc) return rc;
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(P && s_tilde && coef && y, "chain_tx: NULL pointer");
    FD_REQUIRE(aligned16(P) && aligned16(s_tilde) && aligned8(coef) && aligned16(y), "chain_tx: misaligned pointer");
    const float2 *Pp = (const float2*)P, *sp = (const float2*)s_tilde, *cp = (const float2*)coef;
    float2* yp = (float2*)y;
    FD_LOG2N_SWITCH(ilog2(N_ifft),
                    (launch_chain<LG, false>(variant, Pp, sp, cp, yp, nullptr, n_sym, B_loc, U, N_d, d, imp, stream)));
}

static int chain_txrx_impl(const void* P, const void* s_tilde, const void* coef, void* y, void* XPA,
                           const int* orders, int n_orders, int L, int M, long long n_sym, int B_loc, int U, int N_d,
                           int N_ifft, const fd_impair* pub, cudaStream_t stream, bool per_symbol_P = false,
                           bool precoded = false) {
    Impair imp = to_impair(pub, B_loc);
    if (per_symbol_P) imp.p_stride = (long long)B_loc * U * N_d;
    imp.precoded = precoded ? 1 : 0;
    FD_REQUIRE(U >= 1 && U <= 1024, "chain_txrx: bad U=%d", U);
    int rc = validate_ofdm(n_sym, B_loc, N_d, N_ifft);
    if (rc) return rc;
    GmpDesc d;
    int variant = 0;
    rc = validate_gmp(orders, n_orders, L, M, N_ifft, d, variant);
    if (rc) return rc;
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(P && s_tilde && coef && y && XPA, "chain_txrx: NULL pointer");
    FD_REQUIRE(aligned16(P) && aligned16(s_tilde) && aligned8(coef) && aligned8(XPA) && aligned16(y),
               "chain_txrx: misaligned pointer");
    FD_REQUIRE(y != XPA, "chain_txrx: XPA must not alias y");
    const float2 *Pp = (const float2*)P, *sp = (const float2*)s_tilde, *cp = (const float2*)coef;
    float2 *yp = (float2*)y, *xp = (float2*)XPA;
    FD_LOG2N_SWITCH(ilog2(N_ifft),
                    (launch_chain<LG, true>(variant, Pp, sp, cp, yp, xp, n_sym, B_loc, U, N_d, d, imp, stream)));
}

int chain_tx(const void* P, const void* s_tilde, const void* coef, void* y, const int* orders, int n_orders, int L,
             int M, long long n_sym, int B_loc, int U, int N_d, int N_ifft, cudaStream_t stream) {
    return chain_tx_impl(P, s_tilde, coef, y, orders, n_orders, L, M, n_sym, B_loc, U, N_d, N_ifft, nullptr, stream);
}

int chain_txrx(const void* P, const void* s_tilde, const void* coef, void* y, void* XPA, const int* orders,
               int n_orders, int L, int M, long long n_sym, int B_loc, int U, int N_d, int N_ifft,
               cudaStream_t stream) {
    return chain_txrx_impl(P, s_tilde, coef, y, XPA, orders, n_orders, L, M, n_sym, B_loc, U, N_d, N_ifft, nullptr,
                           stream);
}

int chain_txrx_ex(const void* P, const void* s_tilde, const void* coef, void* y, void* XPA, const int* orders,
                  int n_orders, int L, int M, long long n_sym, int B_loc, int U, int N_d, int N_ifft,
                  const fd_impair* imp, cudaStream_t stream) {
    if (imp) {
        FD_REQUIRE(imp->clip >= 0.f && imp->pa_noise_std >= 0.f, "chain_txrx_ex: negative impairment");
        FD_REQUIRE(imp->b0 >= 0 && (imp->B_total == 0 || imp->b0 + B_loc <= imp->B_total), "chain_txrx_ex: bad b0");
    }
    return chain_txrx_impl(P, s_tilde, coef, y, XPA, orders, n_orders, L, M, n_sym, B_loc, U, N_d, N_ifft, imp,
                           stream);
}

int chain_txrx_ps(const void* P_all, const void* s_tilde, const void* coef, void* y, void* XPA, const int* orders,
                  int n_orders, int L, int M, long long n_sym, int B_loc, int U, int N_d, int N_ifft,
                  const fd_impair* imp, cudaStream_t stream) {
    return chain_txrx_impl(P_all, s_tilde, coef, y, XPA, orders, n_orders, L, M, n_sym, B_loc, U, N_d, N_ifft, imp,
                           stream, true);
}

int chain_txrx_pre(const void* X, const void* coef, void* y, void* XPA, const int* orders, int n_orders, int L, int M,
                   long long n_sym, int B_loc, int N_d, int N_ifft, const fd_impair* imp, cudaStream_t stream) {
    // s_tilde is unused on this path; pass X for the non-NULL check
    return chain_txrx_impl(X, X, coef, y, XPA, orders, n_orders, L, M, n_sym, B_loc, 1, N_d, N_ifft, imp, stream,
                           false, true);
}

}  // extern "C"
