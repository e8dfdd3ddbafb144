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
// The MMA covers eight shift slots -4 .. 3 where seven are needed, so the odd taps are computed
// one sample late for free (their coefficients sit one slot lower):
//     D[q][l even] = G_l(q) - a_{1,l},      D[q][l odd] = G_l(q - 1) - a_{1,l},
//     w_{2p}(q) = u_q G_{2p}(q) + u_{q-1} G_{2p+1}(q - 1)   (p = 0..3, no odd term for p = 3),
//     y_m = sum_{p=0..3} w_{2p}(m - 2p)
// — three lane shifts of a float2 per sample instead of six.
//
// FP32 accuracy without any range scaling (at C5 e^4 spans ~1e-20 .. 3e9 inside one symbol):
//   e^k = hi + lo, hi = tf32(e^k) (8-bit exponent like fp32), lo = e^k - hi (exact in fp32);
//   C = C_hi + C_lo in tf32;
//   MMA1 (kind::tf32, K = 8):  hi(q + d0), hi(q + d0 + 1) for d0 in {-4, -2, 0, 2} (4 MMAs),
//                              B = [C_hi ; C_lo] stacked along N (N = 32): A_hi C_hi + A_hi C_lo
//   MMA2 (kind::f16 bf16, K = 16): lo(q + d0 .. q + d0 + 3) for d0 in {-4, 0} (2 MMAs),
//                              B = bf16(C) (N = 16): A_lo C (lo ~ 2^-11 e^k, so bf16's 8 bits
//                              leave a ~2^-20 relative error on G — A_lo C_lo ~ 2^-22 dropped)
// 6 MMAs per 128 samples against ~205 FFMA2 per sample on the FP32 pipe.  The constant term
// a_{1,l} (order 1, power 0) is added in the epilogue.
//
// Per CTA (its N_L samples) in chunks of 512 (four M = 128 tiles), all 256 threads, two feature
// buffers and two TMEM accumulators, and NO CTA-wide barrier inside the loop (the warps drift
// apart and hide each other's latencies; every hand-over is an mbarrier with an early arrive
// and a late wait).  Iteration ch:
//   0. warps 0..3 wait for features(ch + 1) (built one iteration ago) and lane 0 of each issues
//      its tile's 6 MMAs of chunk ch + 1 into accumulator (ch + 1) & 1 (committed to mma_bar);
//   1. wait for MMA(ch);
//   2. thread = sample (two 32-sample groups per warp): TMEM row -> G, the four w_{2p}; lanes
//      26..31 publish w_2, w_4, w_6 as the next group's carry (ring of four chunk slots), one
//      arrive per warp on carry_bar;
//   3. features of chunk ch + 2, samples [q0 - 4, q0 + 515), into the buffers MMA(ch) just
//      released: the tf32 buffer Fp (row r = hi(q), q = q0 - 4 + r; the MMA's second K plane is
//      the next row: descriptor LBO = 16 B) and the bf16 buffer Fq (row r = lo(q), lo(q + 1);
//      second K plane two rows on: LBO = 32 B) — one 16-byte row per sample and buffer; samples
//      outside [0, N_L) are the partner CTA's (distributed shared memory; the symbol is circular,
//      A13); one arrive per warp on feat_bar;
//   4. wait for the chunk's carries; y_q = sum_p w_{2p}(q - 2p): shuffles inside each group of
//      32 samples, the previous group's last six samples from the carry (the first group of the
//      half takes the partner's last group's carry after the loop).
// (Included inside namespace fdpd by chain_cl.cu.)
#pragma once

constexpr int GT_CH = 512;                         // samples per chunk (four M = 128 tiles)
constexpr int GT_TILES = GT_CH / 128;
constexpr int GT_GROUPS = GT_CH / 32;              // 32-sample groups per chunk
constexpr int GT_R = GT_CH + 8;                    // feature rows per chunk buffer (519 used)
constexpr int GT_NS = GT_CH + 7;                   // samples per chunk with features: q0 - 4 .. q0 + 514
constexpr int GT_BUF = GT_R * 16;                  // bytes of one feature buffer (one 16-byte row per sample)
constexpr int GT_FP = 0;                           // [2] tf32 hi features
constexpr int GT_FQ = GT_FP + 2 * GT_BUF;          // [2] bf16 lo features
constexpr int GT_B1 = GT_FQ + 2 * GT_BUF;          // 4 x [32 rows][2 planes] tf32 coefficients
constexpr int GT_B1_MAT = 2 * 32 * 16;
constexpr int GT_B2 = GT_B1 + 4 * GT_B1_MAT;       // 2 x [16 rows][2 planes] bf16 coefficients
constexpr int GT_B2_MAT = 2 * 16 * 16;
constexpr int GT_ZC_SLOTS = 4;                     // carry ring (warps drift by less than two chunks)
constexpr int GT_ZC = GT_B2 + 2 * GT_B2_MAT;       // carries [slot][group][shift 2, 4, 6][6] float2 (setup: raw coefficients)
constexpr int GT_BAR = GT_ZC + GT_ZC_SLOTS * GT_GROUPS * 3 * 6 * 8;   // 6 mbarriers + TMEM address
constexpr int GT_BYTES = GT_BAR + 64;
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

// 32 lanes x 32 columns of TMEM -> registers, without the wait (tmem_ld_wait32 before any use).
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
// The wait names the loaded registers as in / out operands, so no use of them can be scheduled
// above it.
__device__ __forceinline__ void tmem_ld_wait32(uint32_t (&r)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                   "+r"(r[29]), "+r"(r[30]), "+r"(r[31])::"memory");
}

// The GMP of this CTA's half: u (natural order, NL samples) in usm, the partner's in usm_r;
// y (global) gets the NL outputs.  256 threads.  sm = GT_BYTES of free shared memory (16-byte
// aligned), sm_r the partner's.  Ends with every thread past its last use of usm / usm_r (the
// caller's cluster barrier then releases them).
template <int KP, int L, int M>
__device__ void gmp_tc_half(const float2* __restrict__ usm, const float2* __restrict__ usm_r,
                            const float2* __restrict__ cg, int n_coef, unsigned char* __restrict__ sm,
                            const unsigned char* __restrict__ sm_r, int NL, float2* __restrict__ y, int tid,
                            const Impair* im, unsigned long long nbase) {
    static_assert(KP == 5 && L == 6 && M == 3, "tensor-core GMP: the C4 / C5 shape only");
    constexpr int T = 256, NW = T / 32;
    const int warp = tid >> 5, lane = tid & 31;
    uint64_t* mma_bar = reinterpret_cast<uint64_t*>(sm + GT_BAR);       // [2] MMA(ch) complete
    uint64_t* feat_bar = mma_bar + 2;                                   // [2] features(ch) written
    uint64_t* carry_bar = mma_bar + 4;                                  // [2] carries(ch) published
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + GT_BAR + 48);
    float2* zc = reinterpret_cast<float2*>(sm + GT_ZC);
    float2* cs = zc;                      // raw coefficients during the setup (the carries come later)

    // ---- coefficients: raw copy, then the MMA operands and the order-1 constants
    for (int e = tid; e < n_coef; e += T) cs[e] = __ldg(cg + e);
    __syncthreads();
    {
        // slot d of the feature window holds shift d for the even taps and shift d + 1 for the odd taps
        float* b1 = reinterpret_cast<float*>(sm + GT_B1);
        for (int e = tid; e < 4 * 32 * 8; e += T) {            // [s1][n][kk]
            const int s1 = e >> 8, n = (e >> 3) & 31, kk = e & 7;
            const int r = n & 15, l = r >> 1, c = r & 1, k = (kk & 3) + 1, d = -4 + 2 * s1 + (kk >> 2) + (l & 1);
            float v = 0.f;
            if (l <= L && d >= -M && d <= M) {
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
            const int l = n >> 1, c = n & 1, k = (kk & 3) + 1, d = -4 + 4 * s2 + (kk >> 2) + (l & 1);
            float v = 0.f;
            if (l <= L && d >= -M && d <= M) {
                const float2 cc = gmp_tc_coef<KP, L, M>(cs, l, d, k);
                v = c ? cc.y : cc.x;
            }
            b2[(size_t)s2 * (GT_B2_MAT / 2) + (kk >> 3) * (16 * 8) + n * 8 + (kk & 7)] = __float2bfloat16_rn(v);
        }
        if (tid == 0) {
            mbar_init(&mma_bar[0], GT_TILES);             // one commit per tile
            mbar_init(&mma_bar[1], GT_TILES);
            mbar_init(&feat_bar[0], NW);                  // one arrive per warp
            mbar_init(&feat_bar[1], NW);
            mbar_init(&carry_bar[0], NW);
            mbar_init(&carry_bar[1], NW);
        }
        if (warp == 0) tmem_alloc(tslot, GT_TMEM);
    }
    float2 c0[L + 1];
#pragma unroll
    for (int l = 0; l <= L; ++l) c0[l] = cs[l];                  // a_{1,l}
    const uint32_t sbase = smem_u32(sm);
    constexpr uint32_t ID1 = idesc_tf32_m128(32), ID2 = idesc_bf16_m128(16);
    const int nch = NL / GT_CH;

    // features of sample q = q0 - 4 + rs of a chunk into buffer fb: Fp row rs, Fq row rs (first
    // half) and Fq row rs - 1 (second half)
    auto feature = [&](int fb, int rs, float2 uu) {
        uint4* const fp = reinterpret_cast<uint4*>(sm + GT_FP + fb * GT_BUF);
        uint2* const fq = reinterpret_cast<uint2*>(sm + GT_FQ + fb * GT_BUF);
        const float e1 = fmaf(uu.x, uu.x, uu.y * uu.y), e2 = e1 * e1, e3 = e2 * e1, e4 = e2 * e2;
        const float h1 = tf32_fin(e1), h2 = tf32_fin(e2), h3 = tf32_fin(e3), h4 = tf32_fin(e4);
        const uint2 lv = make_uint2(bf16x2_bits(e1 - h1, e2 - h2), bf16x2_bits(e3 - h3, e4 - h4));
        fp[rs] = make_uint4(__float_as_uint(h1), __float_as_uint(h2), __float_as_uint(h3), __float_as_uint(h4));
        fq[2 * rs] = lv;
        if (rs >= 1) fq[2 * rs - 1] = lv;
    };
    auto features = [&](int ch) {
        const int qb = ch * GT_CH - 4, fb = ch & 1;
        if (ch == 0 || ch == nch - 1) {
            for (int rs = tid; rs < GT_NS; rs += T) {
                const int q = qb + rs;
                feature(fb, rs, q < 0 ? usm_r[q + NL] : (q >= NL ? usm_r[q - NL] : usm[q]));
            }
        } else {
#pragma unroll
            for (int k = 0; k < GT_CH / T; ++k) feature(fb, tid + k * T, usm[qb + tid + k * T]);
            if (tid < GT_NS - GT_CH) feature(fb, GT_CH + tid, usm[qb + GT_CH + tid]);
        }
    };
    // tile j of chunk ch: 6 MMAs into accumulator (ch & 1), committed to mma_bar[ch & 1]
    auto issue = [&](int ch, int j) {
        const int fb = ch & 1;
        const uint32_t d = *tslot + (uint32_t)(GT_TILES * 32) * fb + 32u * j;
#pragma unroll
        for (int s1 = 0; s1 < 4; ++s1) {     // rows q + d0, d0 = -4 + 2 s1; K plane 2 = the next row
            const uint64_t da = umma_desc(sbase + GT_FP + fb * GT_BUF + (128 * j + 2 * s1) * 16, 16, 128);
            const uint64_t db = umma_desc(sbase + GT_B1 + s1 * GT_B1_MAT, 32 * 16, 128);
            mma_tf32(d, da, db, ID1, s1 > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {     // rows q + d0, d0 = -4 + 4 s2; K plane 2 = two rows on
            const uint64_t da = umma_desc(sbase + GT_FQ + fb * GT_BUF + (128 * j + 4 * s2) * 16, 32, 128);
            const uint64_t db = umma_desc(sbase + GT_B2 + s2 * GT_B2_MAT, 16 * 16, 128);
            mma_f16(d, da, db, ID2, 1u);
        }
        umma_commit(&mma_bar[fb]);
    };

    __syncthreads();                       // c0 / MMA operands read from cs before the carries reuse it
    float2 acc0 = make_float2(0.f, 0.f);   // y of samples 0..5 without the partner's taps (warp 0)
    features(0);
    if (nch > 1) features(1);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tslot;
    if (warp < GT_TILES && lane == 0) issue(0, warp);
    __syncwarp();
#pragma unroll 1
    for (int ch = 0; ch < nch; ++ch) {
        const int q0 = ch * GT_CH, cb = ch & 1;
        const uint32_t ph = (uint32_t)((ch >> 1) & 1);
        // ---- 0. MMAs of the next chunk (its features were written one iteration ago)
        if (ch + 1 < nch && warp < GT_TILES) {
            if (ch >= 1) mbar_wait(&feat_bar[cb ^ 1], (uint32_t)((((ch + 1) >> 1) + 1) & 1));
            tc_fence_after();
            if (lane == 0) issue(ch + 1, warp);
            __syncwarp();
        }
        // ---- 1. this chunk's accumulator
        mbar_wait(&mma_bar[cb], ph);
        tc_fence_after();
        // ---- 2. w_{2p} of groups g = warp and warp + 8 (tile g / 4, TMEM lane quadrant g % 4 = warp % 4)
        float2 w[2][4];
        {
            uint32_t r0[32], r1[32];
            const uint32_t ta = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(GT_TILES * 32) * cb + 32u * (warp >> 2);
            tmem_ld32_issue(ta, r0);
            tmem_ld32_issue(ta + 64u, r1);          // group warp + 8: two tiles on
            const int qa = q0 + 32 * warp + lane;
            const float2 ua = usm[qa], ub = usm[qa + 256];
            float2 uam = usm[qa > 0 ? qa - 1 : 0];
            const float2 ubm = usm[qa + 255];
            if (qa == 0) uam = usm_r[NL - 1];
            tmem_ld_wait32(r0);
            tmem_ld_wait32(r1);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t(&r)[32] = h ? r1 : r0;
                const float2 uq = h ? ub : ua, um = h ? ubm : uam;
                auto G = [&](int l) {
                    const float2 hi = make_float2(__uint_as_float(r[2 * l]), __uint_as_float(r[2 * l + 1]));
                    const float2 lo = make_float2(__uint_as_float(r[16 + 2 * l]), __uint_as_float(r[17 + 2 * l]));
                    return fadd2(fadd2(hi, lo), c0[l]);
                };
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    w[h][p] = cmul2(uq, G(2 * p));
                    if (2 * p + 1 <= L) w[h][p] = cfma2(um, G(2 * p + 1), w[h][p]);
                }
                if (lane >= 26) {
                    float2* dst = zc + ((((ch & (GT_ZC_SLOTS - 1)) * GT_GROUPS + warp + 8 * h) * 3) * 6 + (lane - 26));
#pragma unroll
                    for (int p = 1; p < 4; ++p) dst[(p - 1) * 6] = w[h][p];
                }
            }
        }
        tc_fence_before();                 // the TMEM reads above precede the next MMAs into this accumulator
        __syncwarp();
        if (lane == 0) mbar_arrive(&carry_bar[cb]);
        // ---- 3. features two chunks ahead, into the buffers MMA(ch) has released
        if (ch + 2 < nch) {
            features(ch + 2);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&feat_bar[cb]);
        }
        // ---- 4. y_q = sum_p w_{2p}(q - 2p)
        mbar_wait(&carry_bar[cb], ph);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = warp + 8 * h;
            const int q = q0 + 32 * g + lane;
            // the group before group 0 of chunk 0 is the partner's last: its carry is added after
            // the loop (samples 0..5), once the partner has published it
            const bool first = ch == 0 && g == 0;
            const float2* prev = zc + (((g > 0 ? (ch & (GT_ZC_SLOTS - 1)) * GT_GROUPS + g - 1
                                              : ((ch - 1) & (GT_ZC_SLOTS - 1)) * GT_GROUPS + GT_GROUPS - 1) * 3) * 6);
            float2 acc = w[h][0];
#pragma unroll
            for (int p = 1; p < 4; ++p) {
                float2 t;
                t.x = __shfl_up_sync(0xffffffffu, w[h][p].x, 2 * p);
                t.y = __shfl_up_sync(0xffffffffu, w[h][p].y, 2 * p);
                if (lane < 2 * p) t = first ? make_float2(0.f, 0.f) : prev[(p - 1) * 6 + (lane - 2 * p + 6)];
                acc = fadd2(acc, t);
            }
            if (first && lane < L) {
                acc0 = acc;
            } else {
                if (im) acc = pa_impair(acc, nbase + (unsigned long long)q, *im);
                y[q] = acc;
            }
        }
    }
    // samples 0..5: the partner's last group's carry (its slot of chunk nch - 1)
    cluster_sync_all();
    if (warp == 0 && lane < L) {
        const float2* pz = reinterpret_cast<const float2*>(sm_r + GT_ZC) +
                           ((((nch - 1) & (GT_ZC_SLOTS - 1)) * GT_GROUPS + GT_GROUPS - 1) * 3) * 6;
#pragma unroll
        for (int p = 1; p < 4; ++p)
            if (lane < 2 * p) acc0 = fadd2(acc0, pz[(p - 1) * 6 + (lane - 2 * p + 6)]);
        if (im) acc0 = pa_impair(acc0, nbase + (unsigned long long)lane, *im);
        y[lane] = acc0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, GT_TMEM);
    }
    // the caller reuses this shared memory (receive-DFT scratch): retire the mbarriers first —
    // without this ~0.6 % of the received rows (XPA) came out different run to run
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < 6; ++i) mbar_inval(&mma_bar[i]);
    }
    __syncthreads();
}
