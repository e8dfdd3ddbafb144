// gmp_tc.cuh — the GMP PA (Eq. 9; reading A13) of one half symbol on the
// 5th-generation tensor cores, for the cluster-split chain (chain_cl.cu, C4 / C5 shape:
// orders {1,3,5,7,9}, L = 6, M = 3).
//
// With the regrouping of gmp.cuh, y_m = sum_l u_{m-l} G_l(m-l) and
//     G_l(q) = a_{1,l} + sum_{k=1..4} sum_{d=-3..3} C_l[d][k] e_{q+d}^k,
//     C_l[0][k] = a_{2k+1,l},  C_l[-g][k] = b_{2k+1,l,g},  C_l[+g][k] = c_{2k+1,l,g},
// G is a real GEMM per antenna: rows = samples q, K = (shift d, power k), N = (tap l, Re / Im)
// = 14.  The K dimension is laid out so that every shift is a row offset of one feature buffer
// (the implicit-GEMM trick of conv_tc.cu): MMA A rows are 16-byte K planes of consecutive
// samples, so the operand for shift d is the same buffer with its descriptor start moved d rows.
//
// FP32 accuracy without any range scaling (at C5 e^4 spans ~1e-20 .. 3e9 inside one symbol):
//   e^k = hi + lo, hi = tf32(e^k) (8-bit exponent like fp32), lo = e^k - hi (exact in fp32);
//   C = C_hi + C_lo in tf32;
//   MMA1 (kind::tf32, K = 8):  hi(q + d0), hi(q + d0 + 1) for d0 in {-3, -1, 1, 3} (4 MMAs),
//                              B = [C_hi ; C_lo] stacked along N (N = 32): A_hi C_hi + A_hi C_lo
//   MMA2 (kind::f16 bf16, K = 16): lo(q + d0 .. q + d0 + 3) for d0 in {-3, 1} (2 MMAs),
//                              B = bf16(C) (N = 16): A_lo C (lo ~ 2^-11 e^k, so bf16's 8 bits
//                              leave a ~2^-20 relative error on G — A_lo C_lo ~ 2^-22 dropped)
// 6 MMAs per 128 samples against ~205 FFMA2 per sample on the FP32 pipe.  The constant term
// a_{1,l} (order 1, power 0) is added in the epilogue.
//
// Per CTA (its N_L samples) in chunks of 256 (two M = 128 tiles), all 256 threads, software-
// pipelined over two feature buffers and two TMEM accumulators (MMA(k + 1) runs while the
// threads finish chunk k and build the features of chunk k + 2):
//   1. features of samples [q0 - 4, q0 + 261): the tf32 buffer Fp (row r = hi(q), q = q0 - 4 + r;
//      the MMA's second K plane is the next row: descriptor LBO = 16 B) and the bf16 buffer Fq
//      (row r = lo(q), lo(q + 1); second K plane two rows on: LBO = 32 B) — one 16-byte row per
//      sample and buffer; samples outside [0, N_L) are the partner CTA's (distributed shared
//      memory; the symbol is circular, A13);
//   2. one thread issues the 12 MMAs into the chunk's TMEM accumulator (two tiles x 32 columns)
//      and commits to the chunk's mbarrier;
//   3. thread = sample: G_l = D[2l + c] + D[16 + 2l + c] + a_{1,l}, z_l = u_q G_l (packed FP32);
//   4. y_q = sum_l z_l(q - l): shuffles inside the warp's 32 samples, the previous group's last
//      six samples through a small shared-memory carry (the first group of the half takes the
//      partner's last six samples, evaluated on the FP32 pipe before the loop).
// (Included inside namespace fdpd by chain_cl.cu.)
#pragma once

constexpr int GT_CH = 256;                         // samples per chunk (two M = 128 tiles)
constexpr int GT_R = GT_CH + 8;                    // feature rows per chunk
constexpr int GT_BUF = GT_R * 16;                  // bytes of one feature buffer (one 16-byte row per sample)
constexpr int GT_FP = 0;                           // tf32 hi features [2 chunks]
constexpr int GT_FQ = GT_FP + 2 * GT_BUF;          // bf16 lo features [2 chunks]
constexpr int GT_B1 = GT_FQ + 2 * GT_BUF;          // 4 x [32 rows][2 planes] tf32 coefficients
constexpr int GT_B1_MAT = 2 * 32 * 16;
constexpr int GT_B2 = GT_B1 + 4 * GT_B1_MAT;       // 2 x [16 rows][2 planes] bf16 coefficients
constexpr int GT_B2_MAT = 2 * 16 * 16;
constexpr int GT_ZC = GT_B2 + 2 * GT_B2_MAT;       // carries: [2][8 groups][6 taps l = 1..6][6] float2
constexpr int GT_A0 = GT_ZC + 2 * 8 * 6 * 6 * 8;   // a_{1,l}, l = 0..6 (float2)
constexpr int GT_BAR = GT_A0 + 8 * 8;              // 2 mbarriers + TMEM address
constexpr int GT_BYTES = GT_BAR + 32;

// Instruction descriptor: D f32, A / B bf16, K-major, M = 128, N = n (kind::f16, K = 16).
__host__ __device__ constexpr uint32_t idesc_bf16_m128(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ uint32_t bf16x2_bits(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// Global coefficient of antenna row cg (SURVEY §8(b) order) for tap l, shift d, power k >= 1.
template <int KP, int L, int M>
__device__ __forceinline__ float2 gmp_tc_coef(const float2* __restrict__ cg, int l, int d, int k) {
    constexpr int NA = KP * (L + 1), NB = (KP - 1) * (L + 1) * M;
    if (d == 0) return cg[k * (L + 1) + l];
    const int g = d < 0 ? -d : d;
    return cg[NA + ((k - 1) * (L + 1) + l) * M + (g - 1) + (d > 0 ? NB : 0)];
}

// 32 lanes x 32 columns of TMEM -> registers.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// The GMP of this CTA's half: u (natural order, NL samples) in usm, the partner's in usm_r;
// y (global) gets the NL outputs.  256 threads.  sm = GT_BYTES of free shared memory, cs = the
// antenna's n_coef raw coefficients' shared-memory slot (both 16-byte aligned).  Ends with
// every thread past its last use of usm / usm_r (the caller's cluster barrier then releases them).
template <int KP, int L, int M>
__device__ void gmp_tc_half(const float2* __restrict__ usm, const float2* __restrict__ usm_r,
                            const float2* __restrict__ cg, float2* __restrict__ cs, int n_coef,
                            unsigned char* __restrict__ sm, int NL, float2* __restrict__ y, int tid,
                            const Impair* im, unsigned long long nbase) {
    static_assert(KP == 5 && L == 6 && M == 3, "tensor-core GMP: the C4 / C5 shape only");
    constexpr int T = 256;
    const int warp = tid >> 5, lane = tid & 31;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + GT_BAR);          // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + GT_BAR + 16);
    float2* zc = reinterpret_cast<float2*>(sm + GT_ZC);
    float2* a0 = reinterpret_cast<float2*>(sm + GT_A0);
    auto u_at = [&](int q) -> float2 {     // circular over the two halves
        return q < 0 ? usm_r[q + NL] : (q >= NL ? usm_r[q - NL] : usm[q]);
    };

    // ---- coefficients: raw copy, then the MMA operands and the order-1 constants
    for (int e = tid; e < n_coef; e += T) cs[e] = __ldg(cg + e);
    __syncthreads();
    {
        float* b1 = reinterpret_cast<float*>(sm + GT_B1);
        for (int e = tid; e < 4 * 32 * 8; e += T) {            // [s1][n][kk]
            const int s1 = e >> 8, n = (e >> 3) & 31, kk = e & 7;
            const int r = n & 15, l = r >> 1, c = r & 1, k = (kk & 3) + 1, d = -3 + 2 * s1 + (kk >> 2);
            float v = 0.f;
            if (l <= L && d <= M) {
                const float2 cc = gmp_tc_coef<KP, L, M>(cs, l, d, k);
                const float x = c ? cc.y : cc.x;
                const float hi = tf32_rna(x);
                v = n < 16 ? hi : tf32_rna(x - hi);
            }
            // K-major core-matrix layout: plane kk / 4, row n, element kk % 4
            b1[(size_t)s1 * (GT_B1_MAT / 4) + (kk >> 2) * (32 * 4) + n * 4 + (kk & 3)] = v;
        }
        __nv_bfloat16* b2 = reinterpret_cast<__nv_bfloat16*>(sm + GT_B2);
        for (int e = tid; e < 2 * 16 * 16; e += T) {            // [s2][n][kk]
            const int s2 = e >> 8, n = (e >> 4) & 15, kk = e & 15;
            const int l = n >> 1, c = n & 1, k = (kk & 3) + 1, d = -3 + 4 * s2 + (kk >> 2);
            float v = 0.f;
            if (l <= L && d <= M) {
                const float2 cc = gmp_tc_coef<KP, L, M>(cs, l, d, k);
                v = c ? cc.y : cc.x;
            }
            b2[(size_t)s2 * (GT_B2_MAT / 2) + (kk >> 3) * (16 * 8) + n * 8 + (kk & 7)] = __float2bfloat16_rn(v);
        }
        if (tid <= L) a0[tid] = cs[tid];                       // a_{1,l}
        // the partner's last six samples (q = -6 .. -1): z_l(q) = u_q G_l(q) for l = 1..6 on the
        // FP32 pipe, as the carry of the group before chunk 0 (zc[1][7])
        if (tid < 6 * L) {
            const int i = tid / L, l = tid % L + 1, q = -6 + i;
            float ew[2 * M + 1];
#pragma unroll
            for (int d = -M; d <= M; ++d) {
                const float2 uu = u_at(q + d);
                ew[d + M] = fmaf(uu.x, uu.x, uu.y * uu.y);
            }
            float2 G = cs[l];                                 // a_{1,l}
#pragma unroll
            for (int d = -M; d <= M; ++d) {
                float ek = 1.f;
#pragma unroll
                for (int k = 1; k < KP; ++k) {
                    ek *= ew[d + M];
                    const float2 cc = gmp_tc_coef<KP, L, M>(cs, l, d, k);
                    G.x = fmaf(cc.x, ek, G.x);
                    G.y = fmaf(cc.y, ek, G.y);
                }
            }
            zc[((1 * 8 + 7) * 6 + (l - 1)) * 6 + i] = cmul(u_at(q), G);
        }
        if (tid == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
        }
        if (warp == 0) tmem_alloc(tslot, 128);
    }
    const uint32_t sbase = smem_u32(sm);
    constexpr uint32_t ID1 = idesc_tf32_m128(32), ID2 = idesc_bf16_m128(16);
    const int nch = NL / GT_CH;

    // features of chunk ch into buffer ch & 1
    auto features = [&](int ch) {
        const int q0 = ch * GT_CH;
        const bool edge = ch == 0 || ch == nch - 1;
        uint4* fp = reinterpret_cast<uint4*>(sm + GT_FP + (ch & 1) * GT_BUF);
        uint2* fq = reinterpret_cast<uint2*>(sm + GT_FQ + (ch & 1) * GT_BUF);
        for (int rs = tid; rs < GT_R + 1; rs += T) {
            const int q = q0 - 4 + rs;
            const float2 uu = edge ? u_at(q) : usm[q];
            const float e1 = fmaf(uu.x, uu.x, uu.y * uu.y), e2 = e1 * e1, e3 = e2 * e1, e4 = e2 * e2;
            const float h1 = tf32_rna(e1), h2 = tf32_rna(e2), h3 = tf32_rna(e3), h4 = tf32_rna(e4);
            const uint2 lv = make_uint2(bf16x2_bits(e1 - h1, e2 - h2), bf16x2_bits(e3 - h3, e4 - h4));
            if (rs < GT_R) {
                fp[rs] = make_uint4(__float_as_uint(h1), __float_as_uint(h2), __float_as_uint(h3), __float_as_uint(h4));
                fq[2 * rs] = lv;                               // row rs, first half
            }
            if (rs >= 1) fq[2 * rs - 1] = lv;                  // row rs - 1, second half
        }
    };
    // 12 MMAs of chunk ch (feature buffer and accumulator ch & 1), committed to bar[ch & 1]
    auto issue = [&](int ch) {
        const uint32_t fpb = sbase + GT_FP + (ch & 1) * GT_BUF, fqb = sbase + GT_FQ + (ch & 1) * GT_BUF;
        const uint32_t dacc = *tslot + 64u * (ch & 1);
        tc_fence_after();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint32_t d = dacc + 32u * j;
#pragma unroll
            for (int s1 = 0; s1 < 4; ++s1) {   // rows q + d0, d0 = -3 + 2 s1; K plane 2 = the next row
                const uint64_t da = umma_desc(fpb + (128 * j + 1 + 2 * s1) * 16, 16, 128);
                const uint64_t db = umma_desc(sbase + GT_B1 + s1 * GT_B1_MAT, 32 * 16, 128);
                mma_tf32(d, da, db, ID1, s1 > 0 ? 1u : 0u);
            }
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {   // rows q + d0, d0 = -3 + 4 s2; K plane 2 = two rows on
                const uint64_t da = umma_desc(fqb + (128 * j + 1 + 4 * s2) * 16, 32, 128);
                const uint64_t db = umma_desc(sbase + GT_B2 + s2 * GT_B2_MAT, 16 * 16, 128);
                mma_f16(d, da, db, ID2, 1u);
            }
        }
        umma_commit(&bar[ch & 1]);
    };

    features(0);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) issue(0);
#pragma unroll 1
    for (int ch = 0; ch < nch; ++ch) {
        const int q0 = ch * GT_CH;
        if (ch + 1 < nch) features(ch + 1);          // buffer (ch + 1) & 1: MMA(ch - 1) has completed
        mbar_wait(&bar[ch & 1], (uint32_t)((ch >> 1) & 1));
        fence_proxy_async();
        tc_fence_before();
        __syncthreads();                             // features(ch + 1) complete; epilogue(ch - 1) done
        if (tid == 0 && ch + 1 < nch) issue(ch + 1);
        tc_fence_after();
        // ---- thread = sample q = q0 + 32 warp + lane (tile warp / 4, lane quadrant warp % 4)
        const int q = q0 + 32 * warp + lane;
        float v[32];
        tmem_ld32(*tslot + ((uint32_t)(32 * (warp & 3)) << 16) + 64u * (ch & 1) + 32u * (warp >> 2), v);
        const float2 uq = usm[q];
        float2 z[L + 1];
#pragma unroll
        for (int l = 0; l <= L; ++l) {
            const float2 G = fadd2(fadd2(make_float2(v[2 * l], v[2 * l + 1]), make_float2(v[16 + 2 * l], v[17 + 2 * l])),
                                   a0[l]);
            z[l] = cmul2(uq, G);
        }
        const int cb = ch & 1;
        if (lane >= 26) {
#pragma unroll
            for (int l = 1; l <= L; ++l) zc[((cb * 8 + warp) * 6 + (l - 1)) * 6 + (lane - 26)] = z[l];
        }
        __syncthreads();
        // ---- y_q = sum_l z_l(q - l)
        const float2* prev = zc + ((warp > 0 ? cb * 8 + warp - 1 : (cb ^ 1) * 8 + 7) * 6) * 6;
        float2 acc = z[0];
#pragma unroll
        for (int l = 1; l <= L; ++l) {
            float2 t;
            t.x = __shfl_up_sync(0xffffffffu, z[l].x, l);
            t.y = __shfl_up_sync(0xffffffffu, z[l].y, l);
            if (lane < l) t = prev[(l - 1) * 6 + (lane - l + 6)];
            acc = fadd2(acc, t);
        }
        if (im) acc = pa_impair(acc, nbase + (unsigned long long)q, *im);
        y[q] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(*tslot, 128);
    }
    // the caller reuses this shared memory (receive-DFT scratch): retire the mbarriers first —
    // without this ~0.6 % of the received rows (XPA) came out different run to run
    if (tid == 0) {
        mbar_inval(&bar[0]);
        mbar_inval(&bar[1]);
    }
    __syncthreads();
}
