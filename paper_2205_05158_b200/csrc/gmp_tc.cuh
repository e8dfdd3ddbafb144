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
// Per CTA (its N_L samples) in chunks of 512 (four M = 128 tiles), all 256 threads, with two
// TMEM accumulators so that the MMAs of chunk k + 1 run under the epilogue of chunk k:
//   1. (after MMA(k) completed) features of chunk k + 1, samples [q0 - 4, q0 + 517): the tf32
//      buffer Fp (row r = hi(q), q = q0 - 4 + r; the MMA's second K plane is the next row:
//      descriptor LBO = 16 B) and the bf16 buffer Fq (row r = lo(q), lo(q + 1); second K plane
//      two rows on: LBO = 32 B) — one 16-byte row per sample and buffer; samples outside
//      [0, N_L) are the partner CTA's (distributed shared memory; the symbol is circular, A13);
//   2. lane 0 of warps 0..3 issues tile j = warp's 6 MMAs of chunk k + 1 into its accumulator and
//      commits (the chunk's mbarrier counts the four commits);
//   3. thread = sample (two 32-sample groups per warp): G_l = D[2l + c] + D[16 + 2l + c] + a_{1,l},
//      z_l = u_q G_l;
//   4. y_q = sum_l z_l(q - l): shuffles inside each group of 32 samples, the previous group's last
//      six samples through a small shared-memory carry (the first group of the half takes the
//      partner's last six samples, evaluated on the FP32 pipe before the loop).
// (Included inside namespace fdpd by chain_cl.cu.)
#pragma once

constexpr int GT_CH = 512;                         // samples per chunk (four M = 128 tiles)
constexpr int GT_TILES = GT_CH / 128;
constexpr int GT_GROUPS = GT_CH / 32;              // 32-sample groups per chunk
constexpr int GT_R = GT_CH + 8;                    // feature rows per chunk
constexpr int GT_BUF = GT_R * 16;                  // bytes of one feature buffer (one 16-byte row per sample)
constexpr int GT_FP = 0;                           // tf32 hi features
constexpr int GT_FQ = GT_FP + GT_BUF;              // bf16 lo features
constexpr int GT_B1 = GT_FQ + GT_BUF;              // 4 x [32 rows][2 planes] tf32 coefficients
constexpr int GT_B1_MAT = 2 * 32 * 16;
constexpr int GT_B2 = GT_B1 + 4 * GT_B1_MAT;       // 2 x [16 rows][2 planes] bf16 coefficients
constexpr int GT_B2_MAT = 2 * 16 * 16;
constexpr int GT_ZC = GT_B2 + 2 * GT_B2_MAT;       // carries: [2][groups][6 taps l = 1..6][6] float2
constexpr int GT_A0 = GT_ZC + 2 * GT_GROUPS * 6 * 6 * 8;   // a_{1,l}, l = 0..6 (float2)
constexpr int GT_BAR = GT_A0 + 8 * 8;              // 2 mbarriers + TMEM address
constexpr int GT_BYTES = GT_BAR + 32;
constexpr int GT_TMEM = 2 * GT_TILES * 32;         // two accumulators x four tiles x 32 columns

// Instruction descriptor: D f32, A / B bf16, K-major, M = 128, N = n (kind::f16, K = 16).
__host__ __device__ constexpr uint32_t idesc_bf16_m128(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// Round a finite fp32 to tf32 (nearest, ties away) with two integer ops (cvt.rna.tf32.f32 also
// checks for inf / NaN: four instructions; the envelope powers and coefficients are finite).
__device__ __forceinline__ float tf32_fin(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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
                            unsigned char* __restrict__ sm, const unsigned char* __restrict__ sm_r, int NL,
                            float2* __restrict__ y, int tid, const Impair* im, unsigned long long nbase) {
    static_assert(KP == 5 && L == 6 && M == 3, "tensor-core GMP: the C4 / C5 shape only");
    constexpr int T = 256;
    const int warp = tid >> 5, lane = tid & 31;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + GT_BAR);          // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + GT_BAR + 16);
    float2* zc = reinterpret_cast<float2*>(sm + GT_ZC);
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
                const float hi = tf32_fin(x);
                v = n < 16 ? hi : tf32_fin(x - hi);
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
        if (tid == 0) {
            mbar_init(&bar[0], GT_TILES);                 // one commit per tile
            mbar_init(&bar[1], GT_TILES);
        }
        if (warp == 0) tmem_alloc(tslot, GT_TMEM);
    }
    const uint32_t sbase = smem_u32(sm);
    constexpr uint32_t ID1 = idesc_tf32_m128(32), ID2 = idesc_bf16_m128(16);
    const int nch = NL / GT_CH;
    uint4* const fp = reinterpret_cast<uint4*>(sm + GT_FP);
    uint2* const fq = reinterpret_cast<uint2*>(sm + GT_FQ);

    // features of chunk ch: sample rs <-> q = q0 - 4 + rs writes Fp row rs, Fq row rs (first
    // half) and Fq row rs - 1 (second half)
    auto feature = [&](int rs, float2 uu) {
        const float e1 = fmaf(uu.x, uu.x, uu.y * uu.y), e2 = e1 * e1, e3 = e2 * e1, e4 = e2 * e2;
        const float h1 = tf32_fin(e1), h2 = tf32_fin(e2), h3 = tf32_fin(e3), h4 = tf32_fin(e4);
        const uint2 lv = make_uint2(bf16x2_bits(e1 - h1, e2 - h2), bf16x2_bits(e3 - h3, e4 - h4));
        if (rs < GT_R) {
            fp[rs] = make_uint4(__float_as_uint(h1), __float_as_uint(h2), __float_as_uint(h3), __float_as_uint(h4));
            fq[2 * rs] = lv;
        }
        if (rs >= 1) fq[2 * rs - 1] = lv;
    };
    auto features = [&](int ch) {
        const int qb = ch * GT_CH - 4;
        if (ch == 0 || ch == nch - 1) {
            for (int rs = tid; rs < GT_R + 1; rs += T) feature(rs, u_at(qb + rs));
        } else {
#pragma unroll
            for (int k = 0; k < GT_CH / T; ++k) feature(tid + k * T, usm[qb + tid + k * T]);
            if (tid < GT_R + 1 - GT_CH) feature(GT_CH + tid, usm[qb + GT_CH + tid]);
        }
    };
    // tile j of chunk ch: 6 MMAs into accumulator (ch & 1), committed to bar[ch & 1]
    auto issue = [&](int ch, int j) {
        const uint32_t d = *tslot + (uint32_t)(GT_TILES * 32) * (ch & 1) + 32u * j;
        tc_fence_after();
#pragma unroll
        for (int s1 = 0; s1 < 4; ++s1) {     // rows q + d0, d0 = -3 + 2 s1; K plane 2 = the next row
            const uint64_t da = umma_desc(sbase + GT_FP + (128 * j + 1 + 2 * s1) * 16, 16, 128);
            const uint64_t db = umma_desc(sbase + GT_B1 + s1 * GT_B1_MAT, 32 * 16, 128);
            mma_tf32(d, da, db, ID1, s1 > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {     // rows q + d0, d0 = -3 + 4 s2; K plane 2 = two rows on
            const uint64_t da = umma_desc(sbase + GT_FQ + (128 * j + 1 + 4 * s2) * 16, 32, 128);
            const uint64_t db = umma_desc(sbase + GT_B2 + s2 * GT_B2_MAT, 16 * 16, 128);
            mma_f16(d, da, db, ID2, 1u);
        }
        umma_commit(&bar[ch & 1]);
    };
    float2 c0[L + 1];
#pragma unroll
    for (int l = 0; l <= L; ++l) c0[l] = cs[l];                  // a_{1,l}

    float2 acc0 = make_float2(0.f, 0.f);   // y of samples 0..5 without the partner's taps (warp 0)
    features(0);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp < GT_TILES && lane == 0) issue(0, warp);
#pragma unroll 1
    for (int ch = 0; ch < nch; ++ch) {
        const int q0 = ch * GT_CH;
        mbar_wait(&bar[ch & 1], (uint32_t)((ch >> 1) & 1));      // MMA(ch) complete: features free
        if (ch + 1 < nch) features(ch + 1);
        fence_proxy_async();
        tc_fence_before();
        __syncthreads();                             // features(ch + 1) complete; epilogue(ch - 1) done
        if (ch + 1 < nch && warp < GT_TILES && lane == 0) issue(ch + 1, warp);
        tc_fence_after();
        // ---- epilogue: groups g = warp and warp + 8 (tile g / 4, TMEM lane quadrant g % 4 = warp % 4)
        const int cb = ch & 1;
        float2 z[2][L + 1];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = warp + 8 * h;
            const int q = q0 + 32 * g + lane;
            float v[32];
            tmem_ld32(*tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(GT_TILES * 32) * cb + 32u * (g >> 2), v);
            const float2 uq = usm[q];
#pragma unroll
            for (int l = 0; l <= L; ++l) {
                const float2 G = make_float2((v[2 * l] + v[16 + 2 * l]) + c0[l].x, (v[2 * l + 1] + v[17 + 2 * l]) + c0[l].y);
                z[h][l] = cmul(uq, G);
            }
            if (lane >= 26) {
#pragma unroll
                for (int l = 1; l <= L; ++l) zc[((cb * GT_GROUPS + g) * 6 + (l - 1)) * 6 + (lane - 26)] = z[h][l];
            }
        }
        tc_fence_before();
        __syncthreads();
        // ---- y_q = sum_l z_l(q - l)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = warp + 8 * h;
            const int q = q0 + 32 * g + lane;
            // the group before group 0 of chunk 0 is the partner's last: its taps are added after
            // the loop (samples 0..5), once the partner has published them
            const bool first = ch == 0 && g == 0;
            const float2* prev = zc + ((g > 0 ? cb * GT_GROUPS + g - 1 : (cb ^ 1) * GT_GROUPS + GT_GROUPS - 1) * 6) * 6;
            float2 acc = z[h][0];
#pragma unroll
            for (int l = 1; l <= L; ++l) {
                float2 t;
                t.x = __shfl_up_sync(0xffffffffu, z[h][l].x, l);
                t.y = __shfl_up_sync(0xffffffffu, z[h][l].y, l);
                if (lane < l) t = first ? make_float2(0.f, 0.f) : prev[(l - 1) * 6 + (lane - l + 6)];
                acc = cadd(acc, t);
            }
            if (first && lane < L) {
                acc0 = acc;
            } else {
                if (im) acc = pa_impair(acc, nbase + (unsigned long long)q, *im);
                y[q] = acc;
            }
        }
    }
    // samples 0..5: the partner's last six samples' taps (its last group's carry, zc[(nch - 1) & 1])
    cluster_sync_all();
    if (warp == 0 && lane < L) {
        const float2* pz = reinterpret_cast<const float2*>(sm_r + GT_ZC) +
                           ((((nch - 1) & 1) * GT_GROUPS + GT_GROUPS - 1) * 6) * 6;
#pragma unroll
        for (int l = 1; l <= L; ++l)
            if (lane < l) acc0 = cadd(acc0, pz[(l - 1) * 6 + (lane - l + 6)]);
        if (im) acc0 = pa_impair(acc0, nbase + (unsigned long long)lane, *im);
        y[lane] = acc0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(*tslot, GT_TMEM);
    }
    // the caller reuses this shared memory (receive-DFT scratch): retire the mbarriers first —
    // without this ~0.6 % of the received rows (XPA) came out different run to run
    if (tid == 0) {
        mbar_inval(&bar[0]);
        mbar_inval(&bar[1]);
    }
    __syncthreads();
}
