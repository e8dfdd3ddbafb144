// rx.cu — evaluation side of the hot path: receive DFT at the data bins,
// FD channel sum over antennas (Eqs. 4-5), QAM slicing and SER.
#include "fft.cuh"
#include "tcgen05.cuh"

namespace fdpd {

// ============================================================================ receive DFT
// XPA[n][b][j] = N^-1/2 sum_m y[n][b][m] e^{-2 pi i k_j m / N}
// PZ > 0 (N = 16^k, data bins within the first / last PZ radix-16 output slots): the last
// pass computes only the outputs at data bins and writes XPA from registers (chain.cuh).
template <int LOG2N, int PZ = 0>
__global__ void __launch_bounds__(fft_threads<LOG2N>(), fft_min_blocks<LOG2N>()) k_rx_fft(const float2* __restrict__ y, float2* __restrict__ XPA,
                                                                const float2* __restrict__ tw, int N_d, float sc) {
    constexpr int N = 1 << LOG2N, T = fft_threads<LOG2N>(), VPT = N / T, R0 = pass_radix<LOG2N>(0);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* sm = reinterpret_cast<float2*>(smem_raw);
    const int tid = threadIdx.x;
    const size_t nb = blockIdx.x;
    const float2* yi = y + nb * N;
    float2 v[VPT];
#pragma unroll
    for (int q = 0; q < VPT / R0; ++q)
#pragma unroll
        for (int r = 0; r < R0; ++r) v[q * R0 + r] = __ldg(yi + pass_pos<R0, VPT, T, N>(tid, q, r));
    float2* xo = XPA + nb * N_d;
    if constexpr (PZ > 0) {
        static_assert(LOG2N % 4 == 0 && LOG2N >= 8, "pruned last pass needs N = 16^k");
        constexpr int NPS = n_passes<LOG2N>();
        const int h = N_d >> 1;
        fft_run<LOG2N, -1, 0, NPS - 1>(sm, v, tw, tid);
        pass_load_smem<16, VPT, T, N>(sm, v, tid);
#pragma unroll
        for (int q = 0; q < VPT / 16; ++q) {
            const int j = tid + q * T;
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
        fft_run<LOG2N, -1>(sm, v, tw, tid);
        for (int j = tid; j < N_d; j += T) xo[j] = cscale(sm[pidx(data_to_bin(j, N, N_d))], sc);
    }
}

// ============================================================================ slicer
struct SliceParams {
    float inv_ac;   // 1 / (alpha * c): yhat -> level units
    float inv_c;    // 1 / c (per-symbol alpha: inv_ac = inv_c / alpha_n)
    float thr;      // boundary_eps / c in level units
    int m;          // sqrt(M_qam)
};

__device__ __forceinline__ int slice_axis(float v, const SliceParams& sp, bool& near) {
    const float lim = (float)(sp.m - 1);
    float d = fmaf(2.f, floorf(0.5f * v), 1.f);
    d = fminf(fmaxf(d, -lim), lim);
    const float bnd = 2.f * rintf(0.5f * v);
    near |= (fabsf(v - bnd) < sp.thr) && (fabsf(bnd) <= lim - 1.f);
    return (int)((d + lim) * 0.5f);
}

// Block-reduce (err, near, total) and add to the global int64 counters.
__device__ __forceinline__ void add_counts(long long* counts, int err, int near, int total) {
    __shared__ int s_red[3][32];
    for (int o = 16; o > 0; o >>= 1) {
        err += __shfl_xor_sync(0xffffffffu, err, o);
        near += __shfl_xor_sync(0xffffffffu, near, o);
        total += __shfl_xor_sync(0xffffffffu, total, o);
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    if (lane == 0) { s_red[0][w] = err; s_red[1][w] = near; s_red[2][w] = total; }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long e = 0, n = 0, c = 0;
        for (int i = 0; i < nw; ++i) { e += s_red[0][i]; n += s_red[1][i]; c += s_red[2][i]; }
        if (e) atomicAdd(reinterpret_cast<unsigned long long*>(counts + 0), (unsigned long long)e);
        if (c) atomicAdd(reinterpret_cast<unsigned long long*>(counts + 1), (unsigned long long)c);
        if (n) atomicAdd(reinterpret_cast<unsigned long long*>(counts + 2), (unsigned long long)n);
    }
}

__global__ void k_slice(const float2* __restrict__ yhat, const uint16_t* __restrict__ idx, uint16_t* __restrict__ dec,
                        long long* counts, long long total, SliceParams sp) {
    int err = 0, near = 0, cnt = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const float2 z = yhat[i];
        bool nr = false;
        const int di = slice_axis(z.x * sp.inv_ac, sp, nr);
        const int dq = slice_axis(z.y * sp.inv_ac, sp, nr);
        const int dd = di + sp.m * dq;
        if (dec) dec[i] = (uint16_t)dd;
        err += (dd != (int)idx[i]);
        near += nr;
        ++cnt;
    }
    add_counts(counts, err, near, cnt);
}

// Mode A, owner side of the fused exchange: y_hat = sum over the source ranks' slots, in rank
// order (deterministic), then slicing + SER like k_slice.  recv [ws][total].
__global__ void k_reduce_slots_ser(const float2* __restrict__ recv, int ws, float2* __restrict__ yhat,
                                   const uint16_t* __restrict__ idx, uint16_t* __restrict__ dec, long long* counts,
                                   long long total, SliceParams sp) {
    int err = 0, near = 0, cnt = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        float2 z = __ldcg(recv + i);              // written by other GPUs: not through L1
        for (int r = 1; r < ws; ++r) z = cadd(z, __ldcg(recv + (size_t)r * total + i));
        yhat[i] = z;
        if (idx) {
            bool nr = false;
            const int di = slice_axis(z.x * sp.inv_ac, sp, nr);
            const int dq = slice_axis(z.y * sp.inv_ac, sp, nr);
            const int dd = di + sp.m * dq;
            if (dec) dec[i] = (uint16_t)dd;
            err += (dd != (int)idx[i]);
            near += nr;
            ++cnt;
        }
    }
    if (idx) add_counts(counts, err, near, cnt);
}

#include "combine_tc.cuh"

// Tensor-core channel sum for 9 <= U <= 32 (combine_tc.cuh); process-wide switch
// (fd_set_combine_path): 0 = auto = the FP32 SIMT kernels (measured faster: C5 0.645 vs 0.80 ms
// per 32 symbols, both latency-bound on their loads), 1 = FP32 SIMT, 2 = tensor cores where
// they apply.
static int g_combine_mode = 0;

static bool launch_combine_tc(const float2* XPA, const float2* hfd, float2* yhat, int B, int U, int N_d,
                              long long n_sym, int accumulate, const uint16_t* idx, uint16_t* dec, long long* counts,
                              const SliceParams& sp, bool ser, cudaStream_t st) {
    if (g_combine_mode != 2 || U < 9 || U > 32 || !aligned16(yhat)) return false;
    CtGeom g{};
    g.B = B;
    g.U = U;
    g.UP = U <= 16 ? 16 : 32;
    g.N_d = N_d;
    g.n_sym = n_sym;
    g.n_ntiles = (int)((n_sym + 31) / 32);
    g.nchunks = (B + CT_KB - 1) / CT_KB;
    const int quads = (N_d + 3) / 4;
    const int groups = std::max(1, std::min(quads, (148 + g.n_ntiles - 1) / g.n_ntiles));
    g.qper = (quads + groups - 1) / groups;
    g.n_qgroups = (quads + g.qper - 1) / g.qper;
    const size_t smem = (size_t)CT_NS * CT_STAGE + 8 * (2 * CT_NS + 4) + 16;
    const unsigned grid = (unsigned)(g.n_qgroups * g.n_ntiles);
    if (ser) {
        cudaFuncSetAttribute(k_combine_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_combine_tc<true><<<grid, CT_THREADS, smem, st>>>(XPA, hfd, yhat, accumulate, idx, dec, counts, sp, g);
    } else {
        cudaFuncSetAttribute(k_combine_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_combine_tc<false><<<grid, CT_THREADS, smem, st>>>(XPA, hfd, yhat, accumulate, idx, dec, counts, sp, g);
    }
    return true;
}

// ============================================================================ channel sum (+ slicing)
// yhat[n][u][j] (+)= sum_b h_fd[u][b][j] XPA[n][b][j]     (Eq. 5)
// Thread per (subcarrier j, symbol n), consecutive threads = consecutive j (coalesced rows);
// users outer, antennas inner (the XPA column is re-read per user from L1/L2).  Measured on
// C2: 0.23 ms per 1024 symbols, faster than the user-chunked (0.27 ms) and antenna-split
// shared-memory-reduction (0.37 ms) variants tried.
template <bool SER, bool AWGN, bool PS>
__global__ void __launch_bounds__(128) k_rx_combine(const float2* __restrict__ XPA, const float2* __restrict__ hfd,
                                                    float2* __restrict__ yhat, int B, int U, int N_d, int accumulate,
                                                    const uint16_t* __restrict__ idx, uint16_t* __restrict__ dec,
                                                    long long* counts, SliceParams sp, Impair imp) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t n = blockIdx.y;
    int err = 0, near = 0, cnt = 0;
    if (j < N_d) {
        const float2* X = XPA + n * B * N_d + j;
        const float2* H = hfd + (PS ? n * imp.h_stride : 0) + j;
        for (int u = 0; u < U; ++u) {
            const float2* h = H + (size_t)u * B * N_d;
            float2 acc = make_float2(0.f, 0.f);
            for (int b0 = 0; b0 < B; b0 += 8) {     // 16 independent loads in flight per thread
                float2 hv[8], xv[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool ok = b0 + k < B;
                    hv[k] = ok ? __ldg(h + (size_t)(b0 + k) * N_d) : make_float2(0.f, 0.f);
                    xv[k] = ok ? __ldg(X + (size_t)(b0 + k) * N_d) : make_float2(0.f, 0.f);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) acc = cfma(hv[k], xv[k], acc);
            }
            const size_t o = (n * U + u) * N_d + j;
            if (accumulate) acc = cadd(acc, yhat[o]);
            if constexpr (AWGN)   // AWGN at the UEs, NEXT f3
                acc = cadd(acc, cgauss((unsigned long long)((imp.sym0 + (long long)n) * U + u) * N_d + j, STREAM_AWGN,
                                       imp.key_lo, imp.key_hi, imp.awgn_std));
            yhat[o] = acc;
            if constexpr (SER) {
                bool nr = false;
                const float inv = PS ? sp.inv_c / imp.alpha_dev[n] : sp.inv_ac;
                const int di = slice_axis(acc.x * inv, sp, nr);
                const int dq = slice_axis(acc.y * inv, sp, nr);
                const int dd = di + sp.m * dq;
                if (dec) dec[o] = (uint16_t)dd;
                err += (dd != (int)idx[o]);
                near += nr;
                ++cnt;
            }
        }
    }
    if (SER) add_counts(counts, err, near, cnt);
}

// Register-blocked variant for a single channel realisation: a thread owns subcarrier j of
// NS consecutive symbols and UC users at a time, so each h_fd value fetched from L2 feeds NS
// symbols and each XPA value UC users (the simple kernel above re-reads XPA per user and
// h_fd per symbol: ~4x the L2 traffic).  Same summation order over b as k_rx_combine.
template <bool SER, bool AWGN, int UC, int NS>
__global__ void __launch_bounds__(128) k_rx_combine_blk(const float2* __restrict__ XPA, const float2* __restrict__ hfd,
                                                        float2* __restrict__ yhat, int B, int U, int N_d,
                                                        long long n_sym, int accumulate,
                                                        const uint16_t* __restrict__ idx, uint16_t* __restrict__ dec,
                                                        long long* counts, SliceParams sp, Impair imp) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    // symbols in reverse launch order: the chain kernel wrote the last symbols last, so their
    // XPA rows are still in L2 when the first channel-sum CTAs start
    const long long n0 = (long long)(gridDim.y - 1 - blockIdx.y) * NS;
    int err = 0, near = 0, cnt = 0;
    if (j < N_d) {
        const float2* Xc[NS];
        bool nok[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            nok[s] = n0 + s < n_sym;
            Xc[s] = XPA + (size_t)(nok[s] ? n0 + s : n0) * B * N_d + j;
        }
        for (int u0 = 0; u0 < U; u0 += UC) {
            float2 acc[NS][UC];
#pragma unroll
            for (int s = 0; s < NS; ++s)
#pragma unroll
                for (int c = 0; c < UC; ++c) acc[s][c] = make_float2(0.f, 0.f);
            const float2* H = hfd + (size_t)u0 * B * N_d + j;
            int b = 0;
            // 4 antennas' loads (4 (UC + NS)) in flight before the MACs
            for (; b + 4 <= B; b += 4) {
                float2 hv[4][UC], xv[4][NS];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#pragma unroll
                    for (int c = 0; c < UC; ++c)
                        hv[q][c] = (u0 + c < U) ? __ldg(H + ((size_t)c * B + b + q) * N_d) : make_float2(0.f, 0.f);
#pragma unroll
                    for (int s = 0; s < NS; ++s) xv[q][s] = __ldg(Xc[s] + (size_t)(b + q) * N_d);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int s = 0; s < NS; ++s)
#pragma unroll
                        for (int c = 0; c < UC; ++c) acc[s][c] = cfma(hv[q][c], xv[q][s], acc[s][c]);
            }
            for (; b < B; ++b) {
                float2 hv[UC], xv[NS];
#pragma unroll
                for (int c = 0; c < UC; ++c)
                    hv[c] = (u0 + c < U) ? __ldg(H + ((size_t)c * B + b) * N_d) : make_float2(0.f, 0.f);
#pragma unroll
                for (int s = 0; s < NS; ++s) xv[s] = __ldg(Xc[s] + (size_t)b * N_d);
#pragma unroll
                for (int s = 0; s < NS; ++s)
#pragma unroll
                    for (int c = 0; c < UC; ++c) acc[s][c] = cfma(hv[c], xv[s], acc[s][c]);
            }
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                if (!nok[s]) continue;
                const long long n = n0 + s;
#pragma unroll
                for (int c = 0; c < UC; ++c) {
                    const int u = u0 + c;
                    if (u >= U) continue;
                    const size_t o = ((size_t)n * U + u) * N_d + j;
                    float2 a = acc[s][c];
                    if (accumulate) a = cadd(a, yhat[o]);
                    if constexpr (AWGN)
                        a = cadd(a, cgauss((unsigned long long)((imp.sym0 + n) * U + u) * N_d + j, STREAM_AWGN,
                                           imp.key_lo, imp.key_hi, imp.awgn_std));
                    yhat[o] = a;
                    if constexpr (SER) {
                        bool nr = false;
                        const int di = slice_axis(a.x * sp.inv_ac, sp, nr);
                        const int dq = slice_axis(a.y * sp.inv_ac, sp, nr);
                        const int dd = di + sp.m * dq;
                        if (dec) dec[o] = (uint16_t)dd;
                        err += (dd != (int)idx[o]);
                        near += nr;
                        ++cnt;
                    }
                }
            }
        }
    }
    if (SER) add_counts(counts, err, near, cnt);
}

// Many users (U = 9..32): per subcarrier the channel sum is a small complex GEMM
// yhat_j[n][u] = sum_b X_j[n][b] h_j[u][b] with a long contraction (b < B = 256..512) — the
// register-blocked kernel above re-reads h_fd from L2 for every symbol pair (6.9 GB per 32
// symbols at C5).  Here a CTA owns 32 subcarriers (lane = j) x NT symbols x all users
// (warp w: users w UPT .. w UPT + UPT - 1): X_j for its NT symbols is staged in shared memory
// in chunks of BC antennas and read by all 8 warps, and each thread's h_fd loads (coalesced
// over j) feed NT symbols from registers.  Same summation order over b as k_rx_combine.
//
// Pipeline: both operands are staged in shared memory by 16-byte cp.async copies, CB_A antennas
// per stage (h_fd rows [u][a] and X rows [n][a] of 32 subcarriers = 256 B each), CB_NS stages
// deep, so ~80 KB per CTA are in flight while a stage is consumed and neither HBM nor L2 latency
// reaches the FMAs; one CTA barrier per stage.  (The first version staged X through registers
// between two barriers and loaded h_fd into registers right before use: 0.646 ms per 32 C5
// symbols with the FMA pipe 43 % busy, long-scoreboard stalls on the h_fd loads.)
//
// Wave balance: the full tiles (NT = 8 symbols) fill whole rounds of the resident CTA slots; the
// tiles of the last, partial round are cut into two NT = 4 halves so that round costs about half
// a tile time (C5: 416 tiles on 296 slots = 2 rounds -> 1.5).
// Mode A exchange fused into the channel sum (ue_combine_peer): instead of a local partial
// y_hat that a reduce-scatter then moves, symbol n of the world batch is stored straight into
// the receive buffer of the rank that owns it (peer memory over NVLink, or this rank's own
// buffer): slot `rank` of owner n / nm, local symbol n % nm.
constexpr int CB_MAX_PEERS = 16;
struct PeerOut {
    float2* base[CB_MAX_PEERS];   // receive buffers [ws][nm][U][N_d] of every rank (peer-mapped)
    int ws, rank, nm;             // ws = 0: plain local output
};

constexpr int CB_A = 2;                         // antennas per stage
constexpr int CB_NS = 5;                        // stages
template <int UPT, int NT>
constexpr int combine_stage_elems() { return (8 * UPT + NT) * CB_A * 32; }   // float2 per stage: h_fd then X
template <int UPT>
constexpr int combine_tile_smem() { return CB_NS * combine_stage_elems<UPT, 8>() * (int)sizeof(float2); }

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
    // 16-byte asynchronous copy global -> shared; !ok: zero fill (src-size 0, src not read)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}

template <bool SER, bool AWGN, int UPT, int NT>
__device__ __forceinline__ void combine_tile_body(const float2* __restrict__ XPA, const float2* __restrict__ hfd,
                                                  float2* __restrict__ yhat, int B, int U, int N_d, int jt,
                                                  long long n0, int nt, int accumulate,
                                                  const uint16_t* __restrict__ idx, uint16_t* __restrict__ dec,
                                                  long long* counts, const SliceParams& sp, const Impair& imp,
                                                  float2* sm, const PeerOut& peer) {
    constexpr int UT = 8 * UPT;                 // users of the tile (8 warps)
    constexpr int STAGE = combine_stage_elems<UPT, NT>();
    constexpr int HROWS = UT * CB_A, XROWS = NT * CB_A;     // 256-byte rows per stage
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j0 = jt * 32, j = j0 + lane;
    const bool jok = j < N_d;
    const int u0 = warp * UPT;
    float2 acc[NT][UPT];
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int c = 0; c < UPT; ++c) acc[n][c] = make_float2(0.f, 0.f);
    const int nstages = (B + CB_A - 1) / CB_A;
    // This thread's 16-byte pieces of a stage: piece e = tid + 256 k -> row e / 16, subcarriers
    // pj = j0 + 2 (e % 16), + 1.  With 16 rows per k step the rows of a thread are CB_A-periodic:
    // its antenna a = (tid / 16) % CB_A is fixed and its h_fd user (X symbol) advances by
    // 16 / CB_A per k, so every source is one base pointer plus a constant stride, advanced by
    // CB_A antennas per stage (no index arithmetic in the loop).
    static_assert(16 % CB_A == 0, "antennas per stage must divide 16");
    constexpr int RPK = 16 / CB_A;              // users / symbols per k step
    constexpr int HK = HROWS / 16, XK = (XROWS + 15) / 16;
    const int pj = j0 + 2 * (threadIdx.x & 15);
    const bool pok = pj < N_d;                  // N_d is even: both subcarriers of a piece or none
    const int r0 = threadIdx.x >> 4, pa = r0 % CB_A, pu = r0 / CB_A;
    const float2* hsrc = hfd + ((size_t)pu * B + pa) * N_d + (pok ? pj : 0);
    const float2* xsrc = XPA + ((size_t)(n0 + (pu < nt ? pu : 0)) * B + pa) * N_d + (pok ? pj : 0);
    const size_t hstep = (size_t)RPK * B * N_d;               // elements between a thread's h_fd / X pieces
    const uint32_t sm0 = smem_u32(sm) + 16u * threadIdx.x;    // piece e of stage 0 (h_fd), X pieces behind
    int ibuf = 0, ist = 0;                                    // next stage to issue and its buffer
    auto issue = [&]() {
        if (ist < nstages) {
            const bool aok = pok && ist * CB_A + pa < B;
            const uint32_t d = sm0 + (uint32_t)ibuf * (STAGE * 8);
#pragma unroll
            for (int k = 0; k < HK; ++k) {
                const bool ok = aok && pu + RPK * k < U;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d + 4096u * k),
                             "l"(ok ? hsrc + hstep * k : hfd), "r"(ok ? 16 : 0)
                             : "memory");
            }
#pragma unroll
            for (int k = 0; k < XK; ++k) {
                if (XROWS % 16 != 0 && r0 + 16 * k >= XROWS) break;
                const bool ok = aok && pu + RPK * k < nt;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d + HROWS * 256u + 4096u * k),
                             "l"(ok ? xsrc + hstep * k : XPA), "r"(ok ? 16 : 0)
                             : "memory");
            }
            hsrc += (size_t)CB_A * N_d;
            xsrc += (size_t)CB_A * N_d;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");     // (empty groups keep the count uniform)
        ++ist;
        if (++ibuf == CB_NS) ibuf = 0;
    };
#pragma unroll
    for (int st = 0; st < CB_NS - 1; ++st) issue();
    int cbuf = 0;
    for (int st = 0; st < nstages; ++st) {
        asm volatile("cp.async.wait_group %0;" ::"n"(CB_NS - 2) : "memory");
        __syncthreads();                       // stage st visible; everyone is done with stage st - 1
        issue();                               // stage st + CB_NS - 1 refills the buffer of stage st - 1
        const float2* hs = sm + (size_t)cbuf * STAGE;
        const float2* xs = hs + HROWS * 32;
        if (++cbuf == CB_NS) cbuf = 0;
#pragma unroll
        for (int a = 0; a < CB_A; ++a) {
            float2 hv[UPT];
#pragma unroll
            for (int c = 0; c < UPT; ++c) hv[c] = hs[((u0 + c) * CB_A + a) * 32 + lane];
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                const float2 xv = xs[(n * CB_A + a) * 32 + lane];
#pragma unroll
                for (int c = 0; c < UPT; ++c) acc[n][c] = cfma2(hv[c], xv, acc[n][c]);
            }
        }
    }
    int err = 0, near = 0, cnt = 0;
    if (jok) {
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            if (n >= nt) continue;
#pragma unroll
            for (int c = 0; c < UPT; ++c) {
                const int u = u0 + c;
                if (u >= U) continue;
                const size_t o = ((size_t)(n0 + n) * U + u) * N_d + j;
                float2 a = acc[n][c];
                if constexpr (!SER && !AWGN) {
                    if (peer.ws > 0) {          // the owner's slot for this rank (Mode A, fused exchange)
                        const long long ng = n0 + n;
                        const int owner = (int)(ng / peer.nm);
                        const long long nl = ng - (long long)owner * peer.nm;
                        peer.base[owner][(((size_t)peer.rank * peer.nm + nl) * U + u) * N_d + j] = a;
                        continue;
                    }
                }
                if (accumulate) a = cadd(a, yhat[o]);
                if constexpr (AWGN)
                    a = cadd(a, cgauss((unsigned long long)((imp.sym0 + n0 + n) * U + u) * N_d + j, STREAM_AWGN,
                                       imp.key_lo, imp.key_hi, imp.awgn_std));
                yhat[o] = a;
                if constexpr (SER) {
                    bool nr = false;
                    const int di = slice_axis(a.x * sp.inv_ac, sp, nr);
                    const int dq = slice_axis(a.y * sp.inv_ac, sp, nr);
                    const int dd = di + sp.m * dq;
                    if (dec) dec[o] = (uint16_t)dd;
                    err += (dd != (int)idx[o]);
                    near += nr;
                    ++cnt;
                }
            }
        }
    }
    if (SER) add_counts(counts, err, near, cnt);
}

// Tiles t = jt * ntile_n + i (symbol tiles fastest: the CTAs sharing a subcarrier tile's h_fd
// slice, U x B x 32, run together, so h_fd comes from HBM once per step and from L2 after; the
// last-written symbols first: their XPA rows are still in L2).  CTAs [0, n_full) take whole
// tiles, the rest half tiles (see above).
template <bool SER, bool AWGN, int UPT>
__global__ void __launch_bounds__(256, 2) k_rx_combine_tile(const float2* __restrict__ XPA, const float2* __restrict__ hfd,
                                                            float2* __restrict__ yhat, int B, int U, int N_d,
                                                            long long n_sym, int ntile_n, int n_full, int accumulate,
                                                            const uint16_t* __restrict__ idx, uint16_t* __restrict__ dec,
                                                            long long* counts, SliceParams sp, Impair imp,
                                                            PeerOut peer) {
    extern __shared__ __align__(16) unsigned char cb_smem[];
    float2* xs = reinterpret_cast<float2*>(cb_smem);   // CB_NS stages of (h_fd rows, X rows)
    const int bid = blockIdx.x;
    const bool full = bid < n_full;
    const int t = full ? bid : n_full + ((bid - n_full) >> 1);
    const int half = full ? 0 : ((bid - n_full) & 1);
    const int jt = t / ntile_n;
    const long long n0 = (long long)(ntile_n - 1 - (t - jt * ntile_n)) * 8 + 4 * half;
    if (full) {
        const int nt = (int)min(8LL, n_sym - n0);
        combine_tile_body<SER, AWGN, UPT, 8>(XPA, hfd, yhat, B, U, N_d, jt, n0, nt, accumulate, idx, dec, counts, sp,
                                             imp, xs, peer);
    } else {
        const int nt = (int)min(4LL, n_sym - n0);
        if (nt <= 0) return;
        combine_tile_body<SER, AWGN, UPT, 4>(XPA, hfd, yhat, B, U, N_d, jt, n0, nt, accumulate, idx, dec, counts, sp,
                                             imp, xs, peer);
    }
}

// Resident CTA slots of kern on the current device, cached per kernel (the instantiations share
// one function-pointer type, so the cache is keyed by the pointer); also raises the kernel's
// dynamic shared-memory limit on first use.
template <typename K>
static int combine_slots(K kern, int smem) {
    static const void* keys[16];
    static int vals[16], n = 0;
    for (int i = 0; i < n; ++i)
        if (keys[i] == reinterpret_cast<const void*>(kern)) return vals[i];
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, smem);
    const int v = std::max(1, sms * per);
    if (n < 16) { keys[n] = reinterpret_cast<const void*>(kern); vals[n] = v; ++n; }
    return v;
}

template <bool SER, bool AWGN>
static void launch_combine(const float2* XPA, const float2* hfd, float2* yhat, int B, int U, int N_d, long long n_sym,
                           int accumulate, const uint16_t* idx, uint16_t* dec, long long* counts,
                           const SliceParams& sp, const Impair& imp, cudaStream_t st,
                           const PeerOut& peer = PeerOut{}) {
    if (imp.h_stride == 0 && imp.alpha_dev == nullptr) {
        if (!AWGN && peer.ws == 0 && launch_combine_tc(XPA, hfd, yhat, B, U, N_d, n_sym, accumulate, idx, dec, counts, sp, SER, st))
            return;
        auto go = [&](auto kern, int ns) {
            dim3 g((N_d + 127) / 128, (unsigned)((n_sym + ns - 1) / ns));
            kern<<<g, 128, 0, st>>>(XPA, hfd, yhat, B, U, N_d, n_sym, accumulate, idx, dec, counts, sp, imp);
        };
        auto go_tile = [&](auto kern, int smem) {
            const int slots = combine_slots(kern, smem);
            const int ntile_n = (int)((n_sym + 7) / 8), tiles = ntile_n * ((N_d + 31) / 32);
            // whole rounds as full tiles; a last round filling under ~3/4 of the slots as half tiles
            int n_full = tiles / slots * slots;
            if ((tiles - n_full) * 4 > slots * 3) n_full = tiles;
            const unsigned grid = (unsigned)(n_full + 2 * (tiles - n_full));
            kern<<<grid, 256, smem, st>>>(XPA, hfd, yhat, B, U, N_d, n_sym, ntile_n, n_full, accumulate, idx, dec,
                                          counts, sp, imp, peer);
        };
        if (U <= 2) go(k_rx_combine_blk<SER, AWGN, 2, 4>, 4);
        else if (U <= 4) go(k_rx_combine_blk<SER, AWGN, 4, 4>, 4);
        else if (U <= 8) go(k_rx_combine_blk<SER, AWGN, 8, 2>, 2);
        // (the tile kernel copies 16-byte pieces: XPA / h_fd rows start 16-byte aligned when the
        // bases are, N_d being even)
        else if (U <= 16 && aligned16(XPA) && aligned16(hfd)) go_tile(k_rx_combine_tile<SER, AWGN, 2>, combine_tile_smem<2>());
        else if (U <= 32 && aligned16(XPA) && aligned16(hfd)) go_tile(k_rx_combine_tile<SER, AWGN, 4>, combine_tile_smem<4>());
        else go(k_rx_combine_blk<SER, AWGN, 8, 2>, 2);
        return;
    }
    dim3 grid((N_d + 127) / 128, (unsigned)n_sym);
    if (imp.h_stride != 0 || imp.alpha_dev != nullptr)
        k_rx_combine<SER, AWGN, true><<<grid, 128, 0, st>>>(XPA, hfd, yhat, B, U, N_d, accumulate, idx, dec, counts, sp,
                                                           imp);
    else
        k_rx_combine<SER, AWGN, false><<<grid, 128, 0, st>>>(XPA, hfd, yhat, B, U, N_d, accumulate, idx, dec, counts,
                                                            sp, imp);
}

// ============================================================================ host side
static int validate_slice(int M_qam, float alpha, float eps, SliceParams& sp) {
    int m = 1;
    while (m * m < M_qam) ++m;
    FD_REQUIRE(m * m == M_qam && M_qam >= 4 && M_qam <= 65536, "M_qam=%d must be a square >= 4", M_qam);
    FD_REQUIRE(alpha > 0.f && std::isfinite(alpha), "alpha=%g must be > 0", (double)alpha);
    FD_REQUIRE(eps >= 0.f, "boundary_eps < 0");
    const double c = 1.0 / std::sqrt(2.0 * (M_qam - 1) / 3.0);
    sp.m = m;
    sp.inv_ac = (float)(1.0 / ((double)alpha * c));
    sp.inv_c = (float)(1.0 / c);
    sp.thr = (float)((double)eps / c);
    return FD_OK;
}

template <int LOG2N>
static int launch_rx_fft(const float2* y, float2* XPA, long long n_sym, int B, int N_d, cudaStream_t st) {
    constexpr int N = 1 << LOG2N;
    const float2* tw = twiddle_table(N, st);
    if (!tw) { set_error("twiddle table allocation failed"); return FD_ERR_CUDA; }
    const size_t smem = sizeof(float2) * padded_len(N);
    const float sc = (float)(1.0 / std::sqrt((double)N));
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<(unsigned)(n_sym * B), fft_threads<LOG2N>(), smem, st>>>(y, XPA, tw, N_d, sc);
    };
    if constexpr (LOG2N % 4 == 0 && LOG2N >= 8) {
        const int pz = prune_slots(N, N_d);
        if (pz == 1) go(k_rx_fft<LOG2N, 1>);
        else if (pz == 2) go(k_rx_fft<LOG2N, 2>);
        else go(k_rx_fft<LOG2N, 0>);
    } else {
        go(k_rx_fft<LOG2N, 0>);
    }
    return check_launch("ue_receive (fft)");
}

static int rx_fft(const float2* y, float2* XPA, long long n_sym, int B, int N_d, int N, cudaStream_t st) {
    switch (ilog2(N)) {
        case 4: return launch_rx_fft<4>(y, XPA, n_sym, B, N_d, st);
        case 5: return launch_rx_fft<5>(y, XPA, n_sym, B, N_d, st);
        case 6: return launch_rx_fft<6>(y, XPA, n_sym, B, N_d, st);
        case 7: return launch_rx_fft<7>(y, XPA, n_sym, B, N_d, st);
        case 8: return launch_rx_fft<8>(y, XPA, n_sym, B, N_d, st);
        case 9: return launch_rx_fft<9>(y, XPA, n_sym, B, N_d, st);
        case 10: return launch_rx_fft<10>(y, XPA, n_sym, B, N_d, st);
        case 11: return launch_rx_fft<11>(y, XPA, n_sym, B, N_d, st);
        case 12: return launch_rx_fft<12>(y, XPA, n_sym, B, N_d, st);
        case 13: return launch_rx_fft<13>(y, XPA, n_sym, B, N_d, st);
        case 14: return launch_rx_fft<14>(y, XPA, n_sym, B, N_d, st);
        default: return fail_arg("unsupported N_ifft=%d", N);
    }
}

static int validate_rx(const void* y, const void* h_fd, const void* yhat, const void* ws, size_t ws_bytes,
                       long long n_sym, int B_loc, int U, int N_d, int N) {
    FD_REQUIRE(n_sym >= 0 && B_loc >= 1 && U >= 1, "ue_receive: bad sizes");
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(y && h_fd && yhat, "ue_receive: NULL pointer");
    FD_REQUIRE(aligned16(y) && aligned8(h_fd) && aligned8(yhat), "ue_receive: misaligned pointer");
    FD_REQUIRE(is_pow2(N) && N >= 16 && N <= 16384, "ue_receive: N_ifft=%d unsupported", N);
    FD_REQUIRE(N_d >= 2 && N_d % 2 == 0 && N_d <= N, "ue_receive: N_d=%d must be even and <= N_ifft", N_d);
    FD_REQUIRE(n_sym <= 65535, "ue_receive: n_sym=%lld > 65535 per call (batch it)", n_sym);
    FD_REQUIRE(n_sym * (long long)B_loc <= 0x7fffffffLL, "ue_receive: n_sym*B too large");
    const size_t need = sizeof(float2) * (size_t)n_sym * B_loc * N_d;
    FD_REQUIRE(ws != nullptr && aligned8(ws) && ws_bytes >= need,
               "ue_receive: workspace of %zu bytes required (got %zu)", need, ws_bytes);
    return FD_OK;
}

}  // namespace fdpd

using namespace fdpd;

extern "C" {

size_t ue_receive_workspace_bytes(long long n_sym, int B_loc, int N_d) {
    if (n_sym <= 0 || B_loc <= 0 || N_d <= 0) return 0;
    return sizeof(float2) * (size_t)n_sym * B_loc * N_d;
}

int ue_receive(const void* y, const void* h_fd, void* yhat, void* workspace, size_t workspace_bytes, long long n_sym,
               int B_loc, int U, int N_d, int N_ifft, int accumulate, cudaStream_t stream) {
    int rc = validate_rx(y, h_fd, yhat, workspace, workspace_bytes, n_sym, B_loc, U, N_d, N_ifft);
    if (rc) return rc;
    if (n_sym == 0) return FD_OK;
    float2* XPA = (float2*)workspace;
    rc = rx_fft((const float2*)y, XPA, n_sym, B_loc, N_d, N_ifft, stream);
    if (rc) return rc;
    launch_combine<false, false>(XPA, (const float2*)h_fd, (float2*)yhat, B_loc, U, N_d, n_sym, accumulate, nullptr, nullptr, nullptr, SliceParams{}, Impair{}, stream);
    return check_launch("ue_receive (combine)");
}

int ue_slice_ser(const void* yhat, float alpha, const uint16_t* tx_idx, int M_qam, uint16_t* dec, long long* counts,
                 long long n_sym, int U, int N_d, float boundary_eps, cudaStream_t stream) {
    FD_REQUIRE(n_sym >= 0 && U >= 1 && N_d >= 1, "ue_slice_ser: bad sizes");
    SliceParams sp;
    int rc = validate_slice(M_qam, alpha, boundary_eps, sp);
    if (rc) return rc;
    const long long total = n_sym * U * (long long)N_d;
    if (total == 0) return FD_OK;
    FD_REQUIRE(yhat && tx_idx && counts, "ue_slice_ser: NULL pointer");
    FD_REQUIRE(aligned8(yhat) && aligned8(counts), "ue_slice_ser: misaligned pointer");
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
    k_slice<<<blocks, 256, 0, stream>>>((const float2*)yhat, tx_idx, dec, counts, total, sp);
    return check_launch("ue_slice_ser");
}

int ue_receive_ser(const void* y, const void* h_fd, void* yhat, void* workspace, size_t workspace_bytes, float alpha,
                   const uint16_t* tx_idx, int M_qam, uint16_t* dec, long long* counts, long long n_sym, int B_loc,
                   int U, int N_d, int N_ifft, float boundary_eps, cudaStream_t stream) {
    int rc = validate_rx(y, h_fd, yhat, workspace, workspace_bytes, n_sym, B_loc, U, N_d, N_ifft);
    if (rc) return rc;
    SliceParams sp;
    rc = validate_slice(M_qam, alpha, boundary_eps, sp);
    if (rc) return rc;
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(tx_idx && counts && aligned8(counts), "ue_receive_ser: NULL/misaligned tx_idx or counts");
    float2* XPA = (float2*)workspace;
    rc = rx_fft((const float2*)y, XPA, n_sym, B_loc, N_d, N_ifft, stream);
    if (rc) return rc;
    launch_combine<true, false>(XPA, (const float2*)h_fd, (float2*)yhat, B_loc, U, N_d, n_sym, 0, tx_idx, dec, counts, sp, Impair{}, stream);
    return check_launch("ue_receive_ser (combine)");
}

}  // extern "C"

extern "C" {

int ue_combine(const void* XPA, const void* h_fd, void* yhat, long long n_sym, int B_loc, int U, int N_d,
               int accumulate, cudaStream_t stream) {
    FD_REQUIRE(n_sym >= 0 && n_sym <= 65535 && B_loc >= 1 && U >= 1 && N_d >= 1, "ue_combine: bad sizes");
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(XPA && h_fd && yhat, "ue_combine: NULL pointer");
    FD_REQUIRE(aligned8(XPA) && aligned8(h_fd) && aligned8(yhat), "ue_combine: misaligned pointer");
    launch_combine<false, false>((const float2*)XPA, (const float2*)h_fd, (float2*)yhat, B_loc, U, N_d, n_sym, accumulate, nullptr, nullptr, nullptr, SliceParams{}, Impair{}, stream);
    return check_launch("ue_combine");
}

int ue_combine_peer(const void* XPA, const void* h_fd, void* const* peer_recv, int world, int rank, long long n_sym,
                    int B_loc, int U, int N_d, cudaStream_t stream) {
    FD_REQUIRE(world >= 1 && world <= CB_MAX_PEERS && rank >= 0 && rank < world,
               "ue_combine_peer: world=%d rank=%d (world <= %d)", world, rank, CB_MAX_PEERS);
    FD_REQUIRE(n_sym >= 0 && n_sym <= 65535 && n_sym % world == 0 && B_loc >= 1 && N_d >= 2 && N_d % 2 == 0,
               "ue_combine_peer: bad sizes (n_sym must be a multiple of world, N_d even)");
    FD_REQUIRE(U >= 9 && U <= 32, "ue_combine_peer: U=%d (the fused exchange serves 9 <= U <= 32)", U);
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(XPA && h_fd && peer_recv, "ue_combine_peer: NULL pointer");
    FD_REQUIRE(aligned16(XPA) && aligned16(h_fd), "ue_combine_peer: XPA / h_fd must be 16-byte aligned");
    PeerOut peer{};
    peer.ws = world;
    peer.rank = rank;
    peer.nm = (int)(n_sym / world);
    for (int r = 0; r < world; ++r) {
        FD_REQUIRE(peer_recv[r] && aligned8(peer_recv[r]), "ue_combine_peer: receive buffer of rank %d missing", r);
        peer.base[r] = (float2*)peer_recv[r];
    }
    launch_combine<false, false>((const float2*)XPA, (const float2*)h_fd, nullptr, B_loc, U, N_d, n_sym, 0, nullptr,
                                 nullptr, nullptr, SliceParams{}, Impair{}, stream, peer);
    return check_launch("ue_combine_peer");
}

int ue_reduce_ser(const void* recv, int world, void* yhat, float alpha, const uint16_t* tx_idx, int M_qam,
                  uint16_t* dec, long long* counts, long long n_sym, int U, int N_d, float boundary_eps,
                  cudaStream_t stream) {
    FD_REQUIRE(world >= 1 && world <= CB_MAX_PEERS && n_sym >= 0 && U >= 1 && N_d >= 1, "ue_reduce_ser: bad sizes");
    SliceParams sp{};
    if (tx_idx) {
        int rc = validate_slice(M_qam, alpha, boundary_eps, sp);
        if (rc) return rc;
        FD_REQUIRE(counts && aligned8(counts), "ue_reduce_ser: counts missing");
    }
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(recv && yhat && aligned8(recv) && aligned8(yhat), "ue_reduce_ser: NULL or misaligned pointer");
    const long long total = n_sym * U * N_d;
    const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 16);
    k_reduce_slots_ser<<<blocks, 256, 0, stream>>>((const float2*)recv, world, (float2*)yhat, tx_idx, dec, counts, total,
                                                   sp);
    return check_launch("ue_reduce_ser");
}

int ue_combine_ser(const void* XPA, const void* h_fd, void* yhat, float alpha, const uint16_t* tx_idx, int M_qam,
                   uint16_t* dec, long long* counts, long long n_sym, int B_loc, int U, int N_d, float boundary_eps,
                   cudaStream_t stream) {
    FD_REQUIRE(n_sym >= 0 && n_sym <= 65535 && B_loc >= 1 && U >= 1 && N_d >= 1, "ue_combine_ser: bad sizes");
    SliceParams sp;
    int rc = validate_slice(M_qam, alpha, boundary_eps, sp);
    if (rc) return rc;
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(XPA && h_fd && yhat && tx_idx && counts, "ue_combine_ser: NULL pointer");
    FD_REQUIRE(aligned8(XPA) && aligned8(h_fd) && aligned8(yhat) && aligned8(counts),
               "ue_combine_ser: misaligned pointer");
    launch_combine<true, false>((const float2*)XPA, (const float2*)h_fd, (float2*)yhat, B_loc, U, N_d, n_sym, 0, tx_idx, dec, counts, sp, Impair{}, stream);
    return check_launch("ue_combine_ser");
}

int ue_combine_ser_ex(const void* XPA, const void* h_fd, void* yhat, float alpha, const uint16_t* tx_idx, int M_qam,
                      uint16_t* dec, long long* counts, long long n_sym, int B_loc, int U, int N_d,
                      float boundary_eps, const fd_impair* imp, cudaStream_t stream) {
    FD_REQUIRE(n_sym >= 0 && n_sym <= 65535 && B_loc >= 1 && U >= 1 && N_d >= 1, "ue_combine_ser_ex: bad sizes");
    FD_REQUIRE(!imp || imp->awgn_n0 >= 0.f, "ue_combine_ser_ex: awgn_n0 < 0");
    SliceParams sp;
    int rc = validate_slice(M_qam, alpha, boundary_eps, sp);
    if (rc) return rc;
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(XPA && h_fd && yhat && tx_idx && counts, "ue_combine_ser_ex: NULL pointer");
    FD_REQUIRE(aligned8(XPA) && aligned8(h_fd) && aligned8(yhat) && aligned8(counts),
               "ue_combine_ser_ex: misaligned pointer");
    Impair im{};
    if (imp) {
        im.awgn_std = imp->awgn_n0 > 0.f ? sqrtf(imp->awgn_n0) : 0.f;
        im.key_lo = (unsigned)(imp->noise_key & 0xffffffffull);
        im.key_hi = (unsigned)(imp->noise_key >> 32);
        im.sym0 = imp->sym0;
    }
    if (im.awgn_std > 0.f)
        launch_combine<true, true>((const float2*)XPA, (const float2*)h_fd, (float2*)yhat, B_loc, U, N_d, n_sym, 0, tx_idx, dec, counts, sp, im, stream);
    else
        launch_combine<true, false>((const float2*)XPA, (const float2*)h_fd, (float2*)yhat, B_loc, U, N_d, n_sym, 0, tx_idx, dec, counts, sp, im, stream);
    return check_launch("ue_combine_ser_ex");
}

int ue_combine_ser_ps(const void* XPA, const void* h_fd_all, void* yhat, const float* alpha_dev,
                      const uint16_t* tx_idx, int M_qam, uint16_t* dec, long long* counts, long long n_sym, int B_loc,
                      int U, int N_d, float boundary_eps, const fd_impair* imp, cudaStream_t stream) {
    FD_REQUIRE(n_sym >= 0 && n_sym <= 65535 && B_loc >= 1 && U >= 1 && N_d >= 1, "ue_combine_ser_ps: bad sizes");
    FD_REQUIRE(!imp || imp->awgn_n0 >= 0.f, "ue_combine_ser_ps: awgn_n0 < 0");
    SliceParams sp;
    int rc = validate_slice(M_qam, 1.f, boundary_eps, sp);
    if (rc) return rc;
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(XPA && h_fd_all && yhat && alpha_dev && tx_idx && counts, "ue_combine_ser_ps: NULL pointer");
    FD_REQUIRE(aligned8(XPA) && aligned8(h_fd_all) && aligned8(yhat) && aligned8(counts),
               "ue_combine_ser_ps: misaligned pointer");
    Impair im{};
    if (imp) {
        im.awgn_std = imp->awgn_n0 > 0.f ? sqrtf(imp->awgn_n0) : 0.f;
        im.key_lo = (unsigned)(imp->noise_key & 0xffffffffull);
        im.key_hi = (unsigned)(imp->noise_key >> 32);
        im.sym0 = imp->sym0;
    }
    im.h_stride = (long long)U * B_loc * N_d;
    im.alpha_dev = alpha_dev;
    if (im.awgn_std > 0.f)
        launch_combine<true, true>((const float2*)XPA, (const float2*)h_fd_all, (float2*)yhat, B_loc, U, N_d, n_sym, 0, tx_idx, dec, counts, sp, im, stream);
    else
        launch_combine<true, false>((const float2*)XPA, (const float2*)h_fd_all, (float2*)yhat, B_loc, U, N_d, n_sym, 0, tx_idx, dec, counts, sp, im, stream);
    return check_launch("ue_combine_ser_ps");
}

}  // extern "C"

extern "C" int fd_set_combine_path(int mode) {
    FD_REQUIRE(mode >= 0 && mode <= 2, "fd_set_combine_path: mode=%d (0 = auto, 1 = FP32 SIMT, 2 = tensor cores)",
               mode);
    fdpd::g_combine_mode = mode;
    return FD_OK;
}
