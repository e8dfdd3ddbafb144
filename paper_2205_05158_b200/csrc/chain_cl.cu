// chain_cl.cu — the fused chain (precode -> IDFT -> GMP -> receive DFT) with each
// (symbol, antenna) split over a cluster of two CTAs, for the largest transform (N = 16384:
// C4, C5; the N = 8192 instantiations exist and pass parity but measured slower than the
// 256-thread single-CTA kernel).
//
// Why: one CTA per N = 16384 symbol needs ~203 KB of shared memory and 512 threads with
// 128 registers, so an SM holds ONE CTA and its FFT phases (shared-memory / barrier bound)
// and GMP phase (FMA bound) cannot overlap with another CTA's.  Split over two CTAs, each
// holds N/2 samples (~105 KB), and two CTAs of different clusters share an SM.
//
// The split is one radix-2 step across the pair (Cooley-Tukey with N = 2 N_L):
//   IDFT (Eq. 2):  CTA c transforms the bins of parity c, Y_c = IDFT_{N_L}(X[2k' + c]);
//                  x[h N_L + m] = Y_0[m] + (-1)^h W_N^{-m} Y_1[m]       (CTA h, own half)
//                  — Y of the partner is read from its shared memory (DSMEM).
//   GMP (Eq. 9):   CTA h evaluates its half; the L + M samples of lagged / leading window
//                  across either end come from the partner (circular symbol, A13).
//   DFT (Eq. 4):   X[2k' + c] = DFT_{N_L}( (y_0[m] + (-1)^c y_1[m]) W_N^{c m} )[k'],
//                  y_0 / y_1 the two halves of the PA output (re-read through L2).
// With the data bins contiguous around DC (A7) and N_d % 4 == 0, the parity-c data bins are
// again a contiguous-around-DC set of N_d / 2 local bins, with local data index jl <->
// global data index j = 2 jl + c, so the pruned local transforms of chain.cuh apply as is.
#include <cooperative_groups.h>
#include <cuda_bf16.h>

#define FD_FFT_PLAIN_PIDX 1   // see fft.cuh: this kernel is faster with the plain padded indices
#include "chain.cuh"
#include "tcgen05.cuh"

namespace cg = cooperative_groups;

namespace fdpd {

// Cluster barrier with release / acquire at cluster scope (shared::cluster and global accesses of
// the pair are ordered).  cooperative_groups' cluster.sync() adds a GPU-scope fence and an L1
// invalidate (MEMBAR.ALL.GPU + ERRBAR + CCTL.IVALL: ~1.7 % of the CTA's lifetime per call, four
// calls); the only global data exchanged between the pair, y, is re-read with ld.global.cg.
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

#include "gmp_tc.cuh"

// Phase trace (builds with -DFD_TRACE only; tools/chain_trace.py): per CTA the SM id and
// %globaltimer at the phase boundaries.
#ifdef FD_TRACE
__device__ unsigned long long g_trace[65536 * 8];
__device__ __forceinline__ void trace_mark(int slot) {
    if (threadIdx.x == 0 && blockIdx.x < 65536) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace[(size_t)blockIdx.x * 8 + slot] = t;
    }
}
#define FD_TRACE_MARK(i) trace_mark(i)
#else
#define FD_TRACE_MARK(i)
#endif

// TCG: the GMP on the tensor cores (gmp_tc.cuh; the C4 / C5 shape at N_L = 8192 only).
template <int LOG2NL, int KP, int L, int M, int RS, int PZ, bool TCG = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(fft_threads<LOG2NL>(), fft_min_blocks<LOG2NL>())
    k_chain_cl(const float2* __restrict__ P, const float2* __restrict__ s, const float2* __restrict__ coef,
               float2* __restrict__ y, float2* __restrict__ XPA, const float2* __restrict__ tw_l,
               const float2* __restrict__ tw_g, int B, int U, int N_d, float sc, GmpDesc d, Impair imp) {
    constexpr int NL = 1 << LOG2NL, N = 2 * NL, T = fft_threads<LOG2NL>(), VPT = NL / T;
    static_assert(KP > 0, "specialised GMP shapes only");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cl = cg::this_cluster();
    const int c = (int)cl.block_rank();          // bin parity of the IDFT / DFT, half of the samples
    const int NdL = N_d >> 1;                    // local data bins
    const ChainSmem lay = chain_smem(NL, NdL, d, false);
    float2* usm = reinterpret_cast<float2*>(smem_raw);
    float* esm = reinterpret_cast<float*>(smem_raw + lay.off_e);
    float2* cf = reinterpret_cast<float2*>(smem_raw + lay.off_cf);
    const int tid = threadIdx.x;
    const size_t nb = blockIdx.x >> 1;
    const int b = (int)(nb % B);
    const size_t n = nb / B;
    const bool impaired = imp.clip > 0.f || imp.pa_std > 0.f;
    const Impair* im = impaired ? &imp : nullptr;
    const unsigned long long nbase =
        ((unsigned long long)(imp.sym0 + (long long)n) * imp.B_total + imp.b0 + b) * (unsigned long long)N +
        (unsigned long long)c * NL;

#ifdef FD_TRACE
    if (tid == 0 && blockIdx.x < 65536) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_trace[(size_t)blockIdx.x * 8 + 7] = smid;
    }
#endif
    FD_TRACE_MARK(0);
    // ---- precode (Eq. 1) of this CTA's data bins: local jl <-> global j = 2 jl + c
    float2* xs = reinterpret_cast<float2*>(esm);
    if constexpr (!TCG) stage_coefs<KP, L, M>(coef + (size_t)b * d.n_coef, cf, d, tid, T);
    if (imp.precoded) {
        const float2* Xr = P + nb * N_d + c;
        for (int j0 = tid; j0 < NdL; j0 += 8 * T) {      // eight loads in flight per thread
            float2 t[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (j0 + k * T < NdL) t[k] = __ldg(Xr + 2 * (j0 + k * T));
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (j0 + k * T < NdL) xs[j0 + k * T] = t[k];
        }
    } else {
        const float2* Pb = P + (size_t)n * imp.p_stride + (size_t)b * U * N_d + c;
        const float2* sn = s + n * U * N_d + c;
        for (int jl = tid; jl < NdL; jl += T) {
            const float2* pp = Pb + 2 * jl;
            const float2* sp = sn + 2 * jl;
            float2 acc = make_float2(0.f, 0.f);
            int u = 0;
            for (; u + 4 <= U; u += 4) {
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
            xs[jl] = acc;
        }
    }
    __syncthreads();

    FD_TRACE_MARK(1);
    // ---- local IDFT of the parity-c bins -> Y_c in usm (unnormalised)
    float2 v[VPT];
    const int h = NdL >> 1;
    if constexpr (PZ > 0) {
        static_assert(pass_radix<LOG2NL>(0) == 16, "pruned pass 0 needs radix 16");
        auto bin = [&](int pos) {
            const bool lo = pos < h, hi = pos >= NL - h;
            const float2 t = xs[lo ? pos + h : (hi ? pos - (NL - h) : 0)];
            return (lo || hi) ? t : make_float2(0.f, 0.f);
        };
#pragma unroll
        for (int q = 0; q < VPT / 16; ++q) {
            const int j = tid + q * T;
            const float2 x0 = bin(j), x15 = bin(j + 15 * (NL / 16));
            const float2 x1 = PZ == 2 ? bin(j + NL / 16) : make_float2(0.f, 0.f);
            const float2 x14 = PZ == 2 ? bin(j + 14 * (NL / 16)) : make_float2(0.f, 0.f);
            float2 X[16];
            dft16_sparse_in<+1, PZ>(x0, x1, x14, x15, X);
#pragma unroll
            for (int r = 0; r < 16; ++r) usm[pidx(16 * j + r)] = X[r];
        }
        __syncthreads();
        fft_run<LOG2NL, +1, 1>(usm, v, tw_l, tid, reinterpret_cast<float2*>(esm));   // xs (in esm) is dead after pass 0
    } else {
        constexpr int R0 = pass_radix<LOG2NL>(0);
#pragma unroll
        for (int q = 0; q < VPT / R0; ++q)
#pragma unroll
            for (int r = 0; r < R0; ++r) {
                const int pos = pass_pos<R0, VPT, T, NL>(tid, q, r);
                const bool lo = pos < h, hi = pos >= NL - h;
                const int jj = lo ? pos + h : pos - (NL - h);
                const float2 t = xs[(lo || hi) ? jj : 0];
                v[q * R0 + r] = (lo || hi) ? t : make_float2(0.f, 0.f);
            }
        fft_run<LOG2NL, +1>(usm, v, tw_l, tid);
    }

    FD_TRACE_MARK(2);
    // ---- radix-2 combine across the pair: x[c N_L + m] = Y_0[m] + (-1)^c W_N^{-m} Y_1[m]
    cluster_sync_all();                          // both Y complete
    {
        const float2* usm_r = cl.map_shared_rank(usm, c ^ 1);
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const int i = tid + T * j;
            const float2 own = usm[pidx(i)], oth = usm_r[pidx(i)];
            const float2 Y0 = c ? oth : own, Y1 = c ? own : oth;
            const float2 t = cmul(Y1, cconj(__ldg(tw_g + i)));
            v[j] = cscale(c ? csub(Y0, t) : cadd(Y0, t), sc);
        }
    }
    cluster_sync_all();                          // the partner has read our Y
    using Lay = RunLayout<RS>;
    if constexpr (TCG) {
#pragma unroll
        for (int j = 0; j < VPT; ++j) usm[tid + T * j] = v[j];          // natural order
    } else {
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const int i = tid + T * j;
            usm[Lay::u_phys(i)] = v[j];
            esm[Lay::e_phys(i)] = fmaf(v[j].x, v[j].x, v[j].y * v[j].y);
        }
    }
    cluster_sync_all();                          // both halves' u / e staged (GMP halo reads)

    FD_TRACE_MARK(3);
    // ---- GMP on this half; y (global) gets samples [c N_L, (c + 1) N_L)
    float2* yo = y + nb * N;
    if constexpr (TCG) {
        static_assert(T == 256, "gmp_tc_half runs 256 threads");
        // scratch right behind the natural-order u (the padded FFT layout and e are dead here)
        unsigned char* gsm = smem_raw + (size_t)NL * sizeof(float2);
        gmp_tc_half<KP, L, M>(usm, cl.map_shared_rank(usm, c ^ 1), coef + (size_t)b * d.n_coef, d.n_coef, gsm,
                              reinterpret_cast<const unsigned char*>(cl.map_shared_rank(gsm, c ^ 1)), NL,
                              yo + (size_t)c * NL, tid, im, nbase);
    } else {
        gmp_runs_symbol<KP, L, M, RS, false, true>(usm, esm, cf, NL, yo + (size_t)c * NL, tid, T, nullptr, im, nbase,
                                                   cl.map_shared_rank(usm, c ^ 1), cl.map_shared_rank(esm, c ^ 1));
    }
    FD_TRACE_MARK(4);
    cluster_sync_all();   // the partner is done with our u / e, and both halves of y are written (cluster acq/rel)
    FD_TRACE_MARK(5);

    // ---- receive DFT at the parity-c bins: DFT_{N_L}((y_0 + (-1)^c y_1) W_N^{c m})
    {
        constexpr int R0 = pass_radix<LOG2NL>(0);
#pragma unroll
        for (int q = 0; q < VPT / R0; ++q)
#pragma unroll
            for (int r = 0; r < R0; ++r) {
                const int pos = pass_pos<R0, VPT, T, NL>(tid, q, r);
                const float2 y0 = __ldcg(yo + pos), y1 = __ldcg(yo + NL + pos);
                v[q * R0 + r] = c ? cmul(csub(y0, y1), __ldg(tw_g + pos)) : cadd(y0, y1);
            }
    }
    fft_run<LOG2NL, -1>(usm, v, tw_l, tid, reinterpret_cast<float2*>(esm));       // e (esm) is dead after the GMP
    float2* xo = XPA + nb * N_d + c;
    for (int jl = tid; jl < NdL; jl += T) xo[2 * jl] = cscale(usm[pidx(data_to_bin(jl, NL, NdL))], sc);
    FD_TRACE_MARK(6);
}

template <int LOG2NL, int KP, int L, int M, int RS, int PZ, bool TCG = false>
static int launch_cl_one(const float2* P, const float2* s, const float2* coef, float2* y, float2* XPA,
                         long long n_sym, int B, int U, int N_d, const GmpDesc& d, const Impair& imp, cudaStream_t st) {
    constexpr int NL = 1 << LOG2NL;
    const float2* tw_l = twiddle_table(NL, st);
    const float2* tw_g = twiddle_table(2 * NL, st);
    if (!tw_l || !tw_g) { set_error("twiddle table allocation failed"); return FD_ERR_CUDA; }
    ChainSmem lay = chain_smem(NL, N_d / 2, d, false);
    if constexpr (TCG) {
        // GMP phase: natural-order u, then the tensor-core scratch (two CTAs per SM: <= 113 KB)
        const int need = NL * (int)sizeof(float2) + GT_BYTES;
        if (need > lay.bytes) lay.bytes = need;
    }
    if (lay.bytes > 227 * 1024) return fail_arg("chain_cl: shared-memory footprint %d B too large", lay.bytes);
#ifdef FD_TRACE
    if (getenv("FD_OCC1")) lay.bytes = 120 * 1024;   // experiment: one CTA per SM
#endif
    set_smem(k_chain_cl<LOG2NL, KP, L, M, RS, PZ, TCG>, lay.bytes);
    k_chain_cl<LOG2NL, KP, L, M, RS, PZ, TCG><<<(unsigned)(2 * n_sym * B), fft_threads<LOG2NL>(), lay.bytes, st>>>(
        P, s, coef, y, XPA, tw_l, tw_g, B, U, N_d, (float)(1.0 / std::sqrt((double)(2 * NL))), d, imp);
    return check_launch("chain_txrx (cluster split)");
}

// GMP implementation of the cluster chain (fd_set_gmp_path): 0 = auto (= FP32 SIMT: the
// tensor-core GMP is correct but measured slower), 1 = FP32 SIMT, 2 = tensor cores
// where they apply (the C4 / C5 shape at N = 16384).
static int g_gmp_path = 0;

template <int LOG2NL, int PZ>
static int cl_variant(int variant, const float2* P, const float2* s, const float2* coef, float2* y, float2* XPA,
                      long long n_sym, int B, int U, int N_d, const GmpDesc& d, const Impair& imp, cudaStream_t st) {
    switch (variant) {
        case 2: return launch_cl_one<LOG2NL, 4, 4, 2, 4, PZ>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        case 3:
            if constexpr (LOG2NL == 13) {
                if (g_gmp_path == 2)
                    return launch_cl_one<LOG2NL, 5, 6, 3, 4, PZ, true>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
            }
            return launch_cl_one<LOG2NL, 5, 6, 3, 4, PZ>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        default: return -1;
    }
}

static int g_chain_split = 0;   // 0 = auto (cluster split where it applies), 1 = never

int launch_chain_cluster(int log2n, int variant, const float2* P, const float2* s, const float2* coef, float2* y,
                         float2* XPA, long long n_sym, int B, int U, int N_d, const GmpDesc& d, const Impair& imp,
                         cudaStream_t st) {
    // N = 8192 stays on the single-CTA kernel: with 256 threads it already runs two CTAs per SM
    // and measured faster than the split (C3: 7.41 vs 8.10 ms per 512 symbols); N = 16384 splits
    // (C4: 13.83 -> 12.68 ms per 128 symbols, C5: 7.37 -> 6.77 ms per 32).
    if (g_chain_split == 1 || log2n != 14 || N_d % 4 != 0) return -1;
    // two CTAs per (symbol, antenna): the grid must stay within gridDim.x (else the single-CTA kernel)
    if (2 * n_sym * (long long)B > 0x7fffffffLL) return -1;
    const int NL = 1 << (log2n - 1);
    const int pz = prune_slots(NL, N_d / 2);
    if (log2n == 13) {
        if (pz == 1) return cl_variant<12, 1>(variant, P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        if (pz == 2) return cl_variant<12, 2>(variant, P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        return cl_variant<12, 0>(variant, P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
    }
    if (pz == 1) return cl_variant<13, 1>(variant, P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
    if (pz == 2) return cl_variant<13, 2>(variant, P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
    return cl_variant<13, 0>(variant, P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
}

}  // namespace fdpd

#ifdef FD_TRACE
extern "C" int fd_debug_trace_read(void* host, size_t bytes) {
    return cudaMemcpyFromSymbol(host, fdpd::g_trace, bytes) == cudaSuccess ? FD_OK : FD_ERR_CUDA;
}
#endif

extern "C" int fd_set_gmp_path(int mode) {
    FD_REQUIRE(mode >= 0 && mode <= 2, "fd_set_gmp_path: mode=%d (0 = auto, 1 = FP32 SIMT, 2 = tensor cores)", mode);
    fdpd::g_gmp_path = mode;
    return FD_OK;
}

extern "C" int fd_set_chain_split(int mode) {
    FD_REQUIRE(mode == 0 || mode == 1, "fd_set_chain_split: mode=%d (0 = auto, 1 = off)", mode);
    fdpd::g_chain_split = mode;
    return FD_OK;
}
