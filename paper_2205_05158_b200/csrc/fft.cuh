// fft.cuh — one-CTA shared-memory Stockham FFT for N = 2^LOG2N <= 16384 points.
//
// Each pass: every thread holds VPT = N/T complex values in registers, performs
// VPT/R radix-R butterflies (R in {2,4,8,16}; radix-16 = 4x4 with internal
// twiddles) and writes them back in Stockham auto-sort order, so the result is
// in natural order without a bit-reversal pass.  Pass twiddles come from a
// fp64-derived complex64 table W[m] = exp(-2 pi i m / N) (L1-resident).
//
// Shared-memory layout: one pad slot per 16 complex (pidx), which makes the
// stride-R stores of the first pass and the stride-16 loads bank-conflict free.
//
// DIR = +1: inverse transform sum_k X_k e^{+2 pi i k m / N} (Eq. 2);
// DIR = -1: forward transform (the receive DFT of Eq. 4).
// No normalisation is applied here; callers apply N^{-1/2}.
#pragma once

#include "common.cuh"

namespace fdpd {

__device__ __forceinline__ int pidx(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_len(int n) { return n + (n >> 4); }
// pidx(i + c) = pidx(i) + pidx_off(c) whenever the low nibbles of i and c do not carry (c a
// multiple of 16, or i a multiple of 16 and c < 16): written out, the padded index of a pass
// position becomes one base per thread plus compile-time offsets — ptxas does not find this by
// itself and spent a LOP3 + LEA.HI + LEA per shared-memory access on it (a fifth of the
// instructions of the Ns = 16 pass).
__host__ __device__ constexpr int pidx_off(int c) { return c + (c >> 4); }
// FD_FFT_PLAIN_PIDX (defined by chain_cl.cu): keep pidx(position) as written.  The cluster-split
// chain measured 1.7 % SLOWER with the base + offset form (C5 5.66 -> 5.76 ms; its FFT phases
// run under the other CTA's GMP, and the different schedule costs more there than the integer
// instructions saved), the single-CTA chains 1.3 - 2.8 % faster (C2 2.74 -> 2.70 ms, C3 6.65 ->
// 6.46 ms).
#ifdef FD_FFT_PLAIN_PIDX
constexpr bool kPidxBase = false;
#else
constexpr bool kPidxBase = true;
#endif

// multiply by DIR * i
template <int DIR>
__device__ __forceinline__ float2 mul_i(float2 a) {
    return DIR > 0 ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// exp(DIR * 2 pi i m / 16) constants, m = 0..15
__device__ __forceinline__ float2 w16(int m, int dir) {
    // cos(2 pi m / 16), sin(2 pi m / 16)
    const float C[16] = {1.0f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                         0.0f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                         -1.0f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f,
                         0.0f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
    const float S[16] = {0.0f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f,
                         1.0f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                         0.0f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                         -1.0f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f};
    return make_float2(C[m & 15], dir > 0 ? S[m & 15] : -S[m & 15]);
}

template <int DIR>
__device__ __forceinline__ void dft2(float2& a, float2& b) {
    float2 t = csub(a, b);
    a = cadd(a, b);
    b = t;
}

template <int DIR>
__device__ __forceinline__ void dft4(float2& x0, float2& x1, float2& x2, float2& x3) {
    // X_k = sum_n x_n W^{nk}, W = exp(DIR 2 pi i / 4) = DIR * i
    float2 a = cadd(x0, x2), b = csub(x0, x2), c = cadd(x1, x3), d = mul_i<DIR>(csub(x1, x3));
    x0 = cadd(a, c);
    x2 = csub(a, c);
    x1 = cadd(b, d);
    x3 = csub(b, d);
}

// In-register DFT of length R on v[off .. off+R), natural order in and out.
template <int R, int DIR, int N_>
__device__ __forceinline__ void dftR(float2 (&v)[N_], int off) {
    if constexpr (R == 2) {
        dft2<DIR>(v[off], v[off + 1]);
    } else if constexpr (R == 4) {
        dft4<DIR>(v[off], v[off + 1], v[off + 2], v[off + 3]);
    } else if constexpr (R == 8) {
        // n = 2 n1 + n2 ; X[k1 + 4 k2]
#pragma unroll
        for (int n2 = 0; n2 < 2; ++n2) dft4<DIR>(v[off + n2], v[off + 2 + n2], v[off + 4 + n2], v[off + 6 + n2]);
        // now A[n2][k1] at v[off + 2 k1 + n2]; twiddle by W8^{n2 k1} = W16^{2 n2 k1}
#pragma unroll
        for (int k1 = 1; k1 < 4; ++k1) v[off + 2 * k1 + 1] = cmul(v[off + 2 * k1 + 1], w16(2 * k1, DIR));
        float2 t[8];
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            float2 a = v[off + 2 * k1], b = v[off + 2 * k1 + 1];
            t[k1] = cadd(a, b);
            t[k1 + 4] = csub(a, b);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) v[off + i] = t[i];
    } else if constexpr (R == 16) {
        // n = 4 n1 + n2 ; X[k1 + 4 k2]
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) dft4<DIR>(v[off + n2], v[off + 4 + n2], v[off + 8 + n2], v[off + 12 + n2]);
        // A[n2][k1] at v[off + 4 k1 + n2]; twiddle W16^{n2 k1}
#pragma unroll
        for (int k1 = 1; k1 < 4; ++k1)
#pragma unroll
            for (int n2 = 1; n2 < 4; ++n2)
                v[off + 4 * k1 + n2] = cmul(v[off + 4 * k1 + n2], w16(n2 * k1, DIR));
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) dft4<DIR>(v[off + 4 * k1], v[off + 4 * k1 + 1], v[off + 4 * k1 + 2], v[off + 4 * k1 + 3]);
        // X[k1 + 4 k2] is at v[off + 4 k1 + k2]: transpose 4x4
        float2 t[16];
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) t[k1 + 4 * k2] = v[off + 4 * k1 + k2];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[off + i] = t[i];
    }
}

// Radix of pass p for N = 2^LOG2N: 16 while >= 4 bits remain, then the remainder.
template <int LOG2N>
__host__ __device__ constexpr int n_passes() { return LOG2N / 4 + (LOG2N % 4 ? 1 : 0); }
template <int LOG2N>
__host__ __device__ constexpr int pass_radix(int p) {
    return (p < LOG2N / 4) ? 16 : (1 << (LOG2N % 4));
}
template <int LOG2N>
__host__ __device__ constexpr int pass_ns(int p) {
    int ns = 1;
    for (int i = 0; i < p; ++i) ns *= pass_radix<LOG2N>(i);
    return ns;
}

// Threads per CTA for an N-point transform: VPT = 16 values/thread up to N = 4096; N = 8192
// with 256 threads (VPT = 32: two CTAs of ~102 KB per SM instead of one 512-thread CTA);
// N = 16384 with 512 threads.
template <int LOG2N>
__host__ __device__ constexpr int fft_threads() { return LOG2N <= 12 ? (1 << LOG2N) / 16 : (LOG2N == 13 ? 256 : 512); }
// resident CTAs per SM requested from ptxas (register cap 65536 / (T * this)).
// (Measured: N/32 threads with 4 CTAs/SM at N = 4096 was 11% slower — register spills.)
template <int LOG2N>
__host__ __device__ constexpr int fft_min_blocks() { return LOG2N <= 12 ? 3 : (LOG2N == 13 ? 2 : 1); }

// Register layout of a pass with radix R: element (q, r), q < VPT/R, r < R, is
// position j + r * (N/R) with j = tid + q * T.
template <int R, int VPT, int T, int N>
__device__ __forceinline__ int pass_pos(int tid, int q, int r) { return tid + q * T + r * (N / R); }

// Shared-memory slot of pass position (q, r) of thread tid; p0 = pidx(tid).
template <int R, int VPT, int T, int N>
__device__ __forceinline__ int pass_slot(int tid, int p0, int q, int r) {
    if constexpr (kPidxBase && T % 16 == 0 && (N / R) % 16 == 0) return p0 + pidx_off(q * T + r * (N / R));
    else return pidx(pass_pos<R, VPT, T, N>(tid, q, r));
}

template <int R, int VPT, int T, int N>
__device__ __forceinline__ void pass_load_smem(const float2* sm, float2 (&v)[VPT], int tid) {
    const int p0 = pidx(tid);
#pragma unroll
    for (int q = 0; q < VPT / R; ++q)
#pragma unroll
        for (int r = 0; r < R; ++r) v[q * R + r] = sm[pass_slot<R, VPT, T, N>(tid, p0, q, r)];
}

// Multiplies v[off + r], r = 1..R-1, by the pass twiddle W^{r step}: the power-of-two
// exponents come from the fp64-derived table (log2 R scattered loads instead of R-1) and
// the rest from at most three complex products (~3 ulp), e.g. W^7 = (W^1 W^2) W^4.
template <int R, int DIR, int VPT>
__device__ __forceinline__ void pass_twiddle(float2 (&v)[VPT], int off, int step, const float2* __restrict__ tw) {
    float2 wp[R];
    wp[0] = make_float2(1.f, 0.f);
#pragma unroll
    for (int p = 1; p < R; p <<= 1) {
        float2 w = __ldg(tw + p * step);
        if (DIR > 0) w.y = -w.y;
        wp[p] = w;
    }
#pragma unroll
    for (int r = 3; r < R; ++r)
        if (r & (r - 1)) wp[r] = cmul(wp[r & (r - 1)], wp[r & -r]);   // r = (r without lowest bit) + lowest bit
#pragma unroll
    for (int r = 1; r < R; ++r) v[off + r] = cmul(v[off + r], wp[r]);
}

// Radix-16 pass twiddles from the per-pass table that follows the N-entry table
// (twiddle_table): entry [(r - 1) Ns + k] = exp(-2 pi i r k / (16 Ns)), fp64-derived.  A
// thread's 15 loads are coalesced across the warp (k = j mod Ns runs over consecutive j) and
// replace 4 loads + 11 derivation products of pass_twiddle.
template <int DIR, int VPT>
__device__ __forceinline__ void pass_twiddle_tab16(float2 (&v)[VPT], int off, int k, int Ns,
                                                   const float2* __restrict__ tab) {
#pragma unroll
    for (int r = 1; r < 16; ++r) {
        float2 w = __ldg(tab + (r - 1) * Ns + k);
        if (DIR > 0) w.y = -w.y;
        v[off + r] = cmul(v[off + r], w);
    }
}

// Offset (in complex entries) of pass P's radix-16 table behind the N-entry table: tables for
// passes p = 1 .. LOG2N/4 - 1 (Ns = 16^p), 15 Ns entries each.
__host__ __device__ constexpr int tw_pass_off(int N, int P) {
    int off = N, ns = 16;
    for (int p = 1; p < P; ++p, ns *= 16) off += 15 * ns;
    return off;
}
__host__ __device__ constexpr int tw_table_len(int N) {
    int len = N, ns = 16;
    while (ns * 16 <= N) { len += 15 * ns; ns *= 16; }   // radix-16 passes with Ns >= 16
    return len;
}

template <int R, int DIR, int VPT, int T, int N, int TWOFF = 0, int Q0 = 0, int Q1 = VPT / R>
__device__ __forceinline__ void pass_compute_store(float2* sm, float2 (&v)[VPT], int Ns, const float2* __restrict__ tw,
                                                   int tid) {
#pragma unroll
    for (int q = Q0; q < Q1; ++q) {
        const int j = tid + q * T;
        const int k = j & (Ns - 1);
        if (R == 16 && TWOFF > 0 && Ns > 1) pass_twiddle_tab16<DIR>(v, q * R, k, Ns, tw + TWOFF);
        else if (Ns > 1) pass_twiddle<R, DIR>(v, q * R, k * (N / (Ns * R)), tw);
        dftR<R, DIR>(v, q * R);
        const int d = (j - k) * R + k;
        // Ns is a compile-time value after inlining: offsets r Ns are multiples of 16 (Ns >= 16),
        // or d is a multiple of 16 and r < 16 (first pass, radix 16)
        if (kPidxBase && ((Ns & 15) == 0 || (Ns == 1 && R == 16))) {
            const int pd = pidx(d);
#pragma unroll
            for (int r = 0; r < R; ++r) sm[pd + pidx_off(r * Ns)] = v[q * R + r];
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) sm[pidx(d + r * Ns)] = v[q * R + r];
        }
    }
}

// Runs passes [P, PEND) — P = 0: after the caller has filled v with the pass-0 input
// layout (pass_pos with R = pass_radix(0)); P > 0: reading the previous pass from sm.
// With PEND = n_passes the transform (unnormalised) is left in sm in natural order.
// Ends with __syncthreads().
//
// scr (optional, T x VPT/2 complex of free shared memory): a pass reads all of its inputs before
// the barrier that precedes its in-place writes, so VPT complex values per thread are live across
// that barrier — 64 registers at VPT = 32 (N = 8192 over 256 threads), which spilled the
// 128-register chain kernel.  With scr the second half of the inputs is parked in shared memory
// (thread-private slots [i][tid], conflict-free) and reloaded after the first half's butterflies.
template <int LOG2N, int DIR, int P = 0, int PEND = n_passes<LOG2N>()>
__device__ __forceinline__ void fft_run(float2* sm, float2 (&v)[(1 << LOG2N) / fft_threads<LOG2N>()],
                                        const float2* __restrict__ tw, int tid, float2* scr = nullptr) {
    constexpr int N = 1 << LOG2N;
    constexpr int T = fft_threads<LOG2N>();
    constexpr int VPT = N / T;
    constexpr int R = pass_radix<LOG2N>(P);
    constexpr int QN = VPT / R;
    constexpr int TWOFF = (R == 16 && P > 0) ? tw_pass_off(N, P) : 0;
    if constexpr (P > 0 && QN >= 2 && QN % 2 == 0) {
        if (scr != nullptr) {
            constexpr int H = VPT / 2;
            // second half: straight from the pass buffer into the parking slots (8 in flight),
            // then the first half into registers
            const int p0 = pidx(tid);
#pragma unroll
            for (int c0 = H; c0 < VPT; c0 += 8) {
                float2 t[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int x = c0 + e;
                    t[e] = sm[pass_slot<R, VPT, T, N>(tid, p0, x / R, x % R)];
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) scr[(c0 + e - H) * T + tid] = t[e];
                asm volatile("" ::: "memory");
            }
#pragma unroll
            for (int x = 0; x < H; ++x) v[x] = sm[pass_slot<R, VPT, T, N>(tid, p0, x / R, x % R)];
            __syncthreads();
            pass_compute_store<R, DIR, VPT, T, N, TWOFF, 0, QN / 2>(sm, v, pass_ns<LOG2N>(P), tw, tid);
#pragma unroll
            for (int i = 0; i < H; ++i) v[H + i] = scr[i * T + tid];
            pass_compute_store<R, DIR, VPT, T, N, TWOFF, QN / 2, QN>(sm, v, pass_ns<LOG2N>(P), tw, tid);
            __syncthreads();
            if constexpr (P + 1 < PEND) fft_run<LOG2N, DIR, P + 1, PEND>(sm, v, tw, tid, scr);
            return;
        }
    }
    if constexpr (P > 0) {
        pass_load_smem<R, VPT, T, N>(sm, v, tid);
        __syncthreads();
    }
    pass_compute_store<R, DIR, VPT, T, N, TWOFF>(sm, v, pass_ns<LOG2N>(P), tw, tid);
    __syncthreads();
    if constexpr (P + 1 < PEND) fft_run<LOG2N, DIR, P + 1, PEND>(sm, v, tw, tid, scr);
}

// ---------------------------------------------------------------- pruned radix-16 passes
// The data subcarriers occupy the first and last h = N_d / 2 bins (reading A7).  When
// h <= N / 8, the radix-16 pass whose 16 points are N/16 apart sees data only in slots
// r < NZ and r >= 16 - NZ, NZ = ceil(h / (N/16)) <= 2: the IDFT's first pass has at most
// 4 non-zero inputs per butterfly and the receive DFT's last pass needs at most 4 of its
// 16 outputs.  Both are computed without the zero / unused arithmetic.

// x * W16^M, W16 = exp(DIR 2 pi i / 16); exact for multiples of 4
template <int DIR, int M>
__device__ __forceinline__ float2 cmul_w16(float2 x) {
    constexpr int m = ((M % 16) + 16) % 16;
    if constexpr (m == 0) return x;
    else if constexpr (m == 4) return mul_i<DIR>(x);
    else if constexpr (m == 8) return make_float2(-x.x, -x.y);
    else if constexpr (m == 12) return mul_i<-DIR>(x);
    else return cmul(x, w16(m, DIR));
}

// sum_{n2} a[n2] (DIR i)^{n2 K2}: one output of a 4-point DFT
template <int DIR, int K2>
__device__ __forceinline__ float2 dft4_out(float2 a0, float2 a1, float2 a2, float2 a3) {
    constexpr int k = K2 & 3;
    if constexpr (k == 0) return cadd(cadd(a0, a2), cadd(a1, a3));
    else if constexpr (k == 2) return csub(cadd(a0, a2), cadd(a1, a3));
    else if constexpr (k == 1) return cadd(csub(a0, a2), mul_i<DIR>(csub(a1, a3)));
    else return csub(csub(a0, a2), mul_i<DIR>(csub(a1, a3)));
}

// 16-point DFT (natural order out) of inputs that are zero except x0 = x[0], x15 = x[15]
// and, for NZ = 2, x1 = x[1], x14 = x[14].  With n = 4 n1 + n2 every n2 column holds one
// non-zero input, so the first 4-point stage is a twiddle: B[n2](k1) = x W16^{n k1}.
template <int DIR, int NZ>
__device__ __forceinline__ void dft16_sparse_in(float2 x0, float2 x1, float2 x14, float2 x15, float2 (&X)[16]) {
#define FDPD_SPARSE_K1(K1)                                                                     \
    {                                                                                          \
        const float2 b0 = x0, b3 = cmul_w16<DIR, 15 * K1>(x15);                               \
        if constexpr (NZ == 2) {                                                               \
            const float2 b1 = cmul_w16<DIR, K1>(x1), b2 = cmul_w16<DIR, 14 * K1>(x14);         \
            X[K1] = dft4_out<DIR, 0>(b0, b1, b2, b3);                                          \
            X[K1 + 4] = dft4_out<DIR, 1>(b0, b1, b2, b3);                                      \
            X[K1 + 8] = dft4_out<DIR, 2>(b0, b1, b2, b3);                                      \
            X[K1 + 12] = dft4_out<DIR, 3>(b0, b1, b2, b3);                                     \
        } else {                                                                               \
            const float2 t = mul_i<DIR>(b3);   /* (DIR i)^{3 k2} b3 for k2 = 1 is -t */          \
            X[K1] = cadd(b0, b3);                                                              \
            X[K1 + 4] = csub(b0, t);                                                           \
            X[K1 + 8] = csub(b0, b3);                                                          \
            X[K1 + 12] = cadd(b0, t);                                                          \
        }                                                                                      \
    }
    FDPD_SPARSE_K1(0)
    FDPD_SPARSE_K1(1)
    FDPD_SPARSE_K1(2)
    FDPD_SPARSE_K1(3)
#undef FDPD_SPARSE_K1
}

// Outputs r < NZ and r >= 16 - NZ of the 16-point DFT of v[off .. off+16) (natural order
// in); v is clobbered.  out[0..NZ) = X[0..NZ), out[NZ..2NZ) = X[16-NZ..16).
template <int DIR, int NZ, int VPT>
__device__ __forceinline__ void dft16_sparse_out(float2 (&v)[VPT], int off, float2 (&out)[2 * NZ]) {
    // n = 4 n1 + n2: 4-point DFTs over n1 -> A[n2][k1] at v[off + 4 k1 + n2]
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<DIR>(v[off + n2], v[off + 4 + n2], v[off + 8 + n2], v[off + 12 + n2]);
    // X[k1 + 4 k2] = sum_{n2} A[n2][k1] W16^{n2 k1} (DIR i)^{n2 k2}
#define FDPD_OUT(K1, K2)                                                                        \
    dft4_out<DIR, K2>(v[off + 4 * K1], cmul_w16<DIR, K1>(v[off + 4 * K1 + 1]),                  \
                      cmul_w16<DIR, 2 * K1>(v[off + 4 * K1 + 2]), cmul_w16<DIR, 3 * K1>(v[off + 4 * K1 + 3]))
    out[0] = FDPD_OUT(0, 0);                          // r = 0
    if constexpr (NZ == 2) {
        out[1] = FDPD_OUT(1, 0);                      // r = 1
        out[2] = FDPD_OUT(2, 3);                      // r = 14
        out[3] = FDPD_OUT(3, 3);                      // r = 15
    } else {
        out[1] = FDPD_OUT(3, 3);                      // r = 15
    }
#undef FDPD_OUT
}

// Data-subcarrier index of IDFT bin k (reading A7), or -1 for a guard bin.
__device__ __forceinline__ int bin_to_data(int k, int N, int N_d) {
    const int h = N_d >> 1;
    if (k < h) return k + h;
    if (k >= N - h) return k - (N - h);
    return -1;
}
__device__ __forceinline__ int data_to_bin(int j, int N, int N_d) {
    const int h = N_d >> 1;
    return j >= h ? j - h : N - h + j;
}

// Number of leading / trailing radix-16 slots holding data bins: ceil(h / (N/16)) for
// h = N_d / 2, or 0 when the pruned passes do not apply (h > N/8 or N < 16).
inline int prune_slots(int N, int N_d) {
    const int h = N_d / 2, w = N / 16;
    if (N < 16 || h < 1) return 0;
    const int nz = (h + w - 1) / w;
    return nz <= 2 ? nz : 0;
}
}  // namespace fdpd
