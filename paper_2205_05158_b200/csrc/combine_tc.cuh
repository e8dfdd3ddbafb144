// combine_tc.cuh — the channel sum of the receive side (Eq. 5) on the 5th-generation
// tensor cores, with the slicing / SER counters fused into the epilogue.  Included by
// rx.cu (needs SliceParams / slice_axis).
//
//   yhat[n][u][j] = sum_b h_fd[u][b][j] XPA[n][b][j]
//
// Per data subcarrier j a complex (n x B) . (B x U) product with a long K = B.  As a real GEMM
// with K = 2B (chunks of KB = 16 antennas, K = 32 real per chunk):
//   A_j[(n,0,h)][k] = [ Re X^h[n][b] | Im X^h[n][b] ]     B_j[(u,h')][k] = [ Re h^h'[u][b] | -Im h^h'[u][b] ]
//   A_j[(n,1,h)][k] = [ Im X^h[n][b] | -Re X^h[n][b] ]
//   D_j[(n,c,h)][(u,h')]:  sum over h, h' = Re (c = 0) / Im (c = 1) of yhat[n][u][j]
// FP32 accuracy: x = hi + lo (TF32 halves) on both operands, the halves stacked along M (rows h)
// and N (columns h'), so one MMA (M = 128 = 32 symbols x Re/Im x hi/lo, N = 2U, K = 8) forms all
// four products; the epilogue sums them in FP32.
//
// Subcarriers go in quads: a stage holds 4 subcarriers x 16 antennas, read as 32-byte sectors
// XPA[n][b][j..j+4) and h_fd[u][b][j..j+4) (the arrays' native layouts, every sector fully used);
// TMEM holds the quad's 4 accumulators (4 x 2U columns) double-buffered across quads.
// Warp roles (mbarrier rings): warps 0-3 epilogue (TMEM lane quadrant: 8 symbols x Re/Im x hi/lo;
// hi/lo and Re/Im combined with two shuffles, one lane per symbol writes yhat[n][u][j..j+4)
// and slices), warps 4-19 producers (one (subcarrier, 4 antennas, symbol / user) item each per
// stage, loads one stage ahead), warp 20 MMA issue.
// (Included inside namespace fdpd, after tcgen05.cuh.)
#pragma once

constexpr int CT_EPI = 4, CT_PROD = 16;
constexpr int CT_MMA_WARP = CT_EPI + CT_PROD;
constexpr int CT_THREADS = 32 * (CT_MMA_WARP + 1);
constexpr int CT_KB = 16;                          // antennas per K chunk
constexpr int CT_PLANES = 2 * CT_KB / 4;           // 16-byte K planes per operand per subcarrier
constexpr int CT_PL_A = (128 + 1) * 16;            // A plane: 128 rows (+1 pad row)
constexpr int CT_PL_B = (64 + 1) * 16;             // B plane: <= 64 rows
constexpr int CT_AJ = CT_PLANES * CT_PL_A + 32;    // per-subcarrier A, stride = 32 mod 128 B:
constexpr int CT_BJ = CT_PLANES * CT_PL_B + 32;    //   the 4 subcarriers' stores spread over the banks
constexpr int CT_STAGE = 4 * CT_AJ + 4 * CT_BJ;
constexpr int CT_NS = 2;                           // shared-memory stages

struct CtGeom {
    int B, U, UP, N_d;                             // UP = U padded to 16 or 32 (N = 2 UP)
    long long n_sym;
    int n_ntiles, qper, n_qgroups, nchunks;
};

__device__ __forceinline__ void ct_split4(float4 x, float4& hi, float4& lo) {
    hi.x = tf32_rna(x.x); lo.x = tf32_rna(x.x - hi.x);
    hi.y = tf32_rna(x.y); lo.y = tf32_rna(x.y - hi.y);
    hi.z = tf32_rna(x.z); lo.z = tf32_rna(x.z - hi.z);
    hi.w = tf32_rna(x.w); lo.w = tf32_rna(x.w - hi.w);
}
__device__ __forceinline__ void ct_ld4(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}
__device__ __forceinline__ float4 ct_neg(float4 x) { return make_float4(-x.x, -x.y, -x.z, -x.w); }

template <bool SER>
__global__ void __launch_bounds__(CT_THREADS, 1)
    k_combine_tc(const float2* __restrict__ XPA, const float2* __restrict__ hfd, float2* __restrict__ yhat,
                 int accumulate, const uint16_t* __restrict__ idx, uint16_t* __restrict__ dec, long long* counts,
                 SliceParams sp, CtGeom g) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)CT_NS * CT_STAGE);
    uint64_t* full = bars;               // [CT_NS]
    uint64_t* empty = bars + CT_NS;      // [CT_NS]
    uint64_t* tfull = empty + CT_NS;     // [2]
    uint64_t* tempty = tfull + 2;        // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    if (tid == 0) {
        for (int i = 0; i < CT_NS; ++i) {
            mbar_init(&full[i], 32 * CT_PROD);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 32 * CT_EPI);
        }
    }
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int qg = blockIdx.x % g.n_qgroups, nt = blockIdx.x / g.n_qgroups;
    const long long n0 = (long long)nt * 32;
    const int nquads_all = (g.N_d + 3) / 4;
    // quads qg, qg + G, qg + 2G, ... (G = n_qgroups): the CTAs running at the same time work on
    // adjacent quads, so the four 32-byte sectors of each 128-byte line of XPA / h_fd are read
    // by four CTAs within a short window and DRAM fetches each line once (a contiguous quad
    // range per CTA re-fetched each line four times: 3.5 GB of DRAM reads per C5 launch
    // against 0.87 GB of data)
    const int nq = qg < nquads_all ? (nquads_all - 1 - qg) / g.n_qgroups + 1 : 0;
    const int n_stages = nq * g.nchunks;
    const int B = g.B, U = g.U, UP = g.UP, N_d = g.N_d;

    if (warp >= CT_EPI && warp < CT_MMA_WARP) {
        // ------------------------------------------------------------ producers
        const int pt = tid - 32 * CT_EPI;
        const int jl = pt & 3, bq = (pt >> 2) & 3, r = pt >> 4;    // subcarrier, antenna quad, symbol / user
        struct Regs {
            float2 x[4], h[4];
        };
        auto load = [&](int i, Regs& R) {
            const int q = qg + (i / g.nchunks) * g.n_qgroups, c = i % g.nchunks;
            const int j = 4 * q + jl, b = c * CT_KB + 4 * bq;
            const long long n = n0 + r;
            const bool jok = j < N_d;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const bool bok = jok && b + t < B;
                R.x[t] = (bok && n < g.n_sym) ? __ldg(XPA + ((size_t)n * B + b + t) * N_d + j) : make_float2(0.f, 0.f);
                R.h[t] = (bok && r < U) ? __ldg(hfd + ((size_t)r * B + b + t) * N_d + j) : make_float2(0.f, 0.f);
            }
        };
        auto store = [&](unsigned char* st, const Regs& R) {
            unsigned char* A = st + (size_t)jl * CT_AJ;
            unsigned char* Bm = st + 4 * (size_t)CT_AJ + (size_t)jl * CT_BJ;
            const float4 re = make_float4(R.x[0].x, R.x[1].x, R.x[2].x, R.x[3].x);
            const float4 im = make_float4(R.x[0].y, R.x[1].y, R.x[2].y, R.x[3].y);
            float4 rh, rl, ih, il;
            ct_split4(re, rh, rl);
            ct_split4(im, ih, il);
            const size_t p0 = (size_t)bq * CT_PL_A, p1 = (size_t)(4 + bq) * CT_PL_A;
            const int row = 4 * r;                               // (n, c, h) = 4 n + 2 c + h
            *reinterpret_cast<float4*>(A + p0 + (row + 0) * 16) = rh;
            *reinterpret_cast<float4*>(A + p1 + (row + 0) * 16) = ih;
            *reinterpret_cast<float4*>(A + p0 + (row + 1) * 16) = rl;
            *reinterpret_cast<float4*>(A + p1 + (row + 1) * 16) = il;
            *reinterpret_cast<float4*>(A + p0 + (row + 2) * 16) = ih;
            *reinterpret_cast<float4*>(A + p1 + (row + 2) * 16) = ct_neg(rh);
            *reinterpret_cast<float4*>(A + p0 + (row + 3) * 16) = il;
            *reinterpret_cast<float4*>(A + p1 + (row + 3) * 16) = ct_neg(rl);
            if (r < UP) {
                const float4 hre = make_float4(R.h[0].x, R.h[1].x, R.h[2].x, R.h[3].x);
                const float4 him = make_float4(-R.h[0].y, -R.h[1].y, -R.h[2].y, -R.h[3].y);
                float4 a, b2;
                const size_t q0 = (size_t)bq * CT_PL_B, q1 = (size_t)(4 + bq) * CT_PL_B;
                ct_split4(hre, a, b2);                           // rows u (hi) and UP + u (lo)
                *reinterpret_cast<float4*>(Bm + q0 + r * 16) = a;
                *reinterpret_cast<float4*>(Bm + q0 + (UP + r) * 16) = b2;
                ct_split4(him, a, b2);
                *reinterpret_cast<float4*>(Bm + q1 + r * 16) = a;
                *reinterpret_cast<float4*>(Bm + q1 + (UP + r) * 16) = b2;
            }
        };
        int buf = 0;
        uint32_t ph = 0;
        Regs RA, RB;
        auto stage = [&](int i, Regs& cur, Regs& nxt) {
            if (i + 1 < n_stages) load(i + 1, nxt);
            if (i >= CT_NS) mbar_wait(&empty[buf], ph ^ 1u);
            store(sm + (size_t)buf * CT_STAGE, cur);
            fence_proxy_async();
            mbar_arrive(&full[buf]);
            if (++buf == CT_NS) { buf = 0; ph ^= 1u; }
        };
        if (n_stages > 0) load(0, RA);
        for (int i = 0; i < n_stages; i += 2) {
            stage(i, RA, RB);
            if (i + 1 < n_stages) stage(i + 1, RB, RA);
        }
    } else if (warp == CT_MMA_WARP) {
        // ------------------------------------------------------------ MMA issue
        const uint32_t base = smem_u32(sm);
        const uint32_t idesc = idesc_tf32_m128(2 * UP);
        int buf = 0;
        uint32_t ph = 0;
        for (int i = 0; i < n_stages; ++i) {
            const int qi = i / g.nchunks, c = i % g.nchunks, slot = qi & 1;
            if (c == 0 && qi >= 2) mbar_wait(&tempty[slot], (uint32_t)(((qi >> 1) - 1) & 1));
            mbar_wait(&full[buf], ph);
            tc_fence_after();
            const uint32_t sb = base + (uint32_t)buf * CT_STAGE;
            if (elect_one()) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const uint64_t da = umma_desc(sb + jj * CT_AJ, CT_PL_A, 128);
                    const uint64_t db = umma_desc(sb + 4 * CT_AJ + jj * CT_BJ, CT_PL_B, 128);
                    const uint32_t d = tmem + (uint32_t)slot * 256 + (uint32_t)jj * 64;
#pragma unroll
                    for (int s = 0; s < CT_PLANES / 2; ++s) {
                        const uint64_t ka = (uint64_t)((2u * s * CT_PL_A) >> 4), kb = (uint64_t)((2u * s * CT_PL_B) >> 4);
                        mma_tf32(d, da + ka, db + kb, idesc, (c | s) != 0 ? 1u : 0u);
                    }
                }
                umma_commit(&empty[buf]);
                if (c == g.nchunks - 1) umma_commit(&tfull[slot]);
            }
            __syncwarp();
            if (++buf == CT_NS) { buf = 0; ph ^= 1u; }
        }
    } else if (warp < CT_EPI) {
        // ------------------------------------------------------------ epilogue
        const int rr = 32 * warp + lane;                 // TMEM lane = row (n, c, h)
        const int nl = rr >> 2, cc = (rr >> 1) & 1, hh = rr & 1;
        const long long n = n0 + nl;
        const bool writer = cc == 0 && hh == 0 && n < g.n_sym;
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
        int err = 0, nnear = 0, cnt = 0;
        for (int qi = 0; qi < nq; ++qi) {
            const int slot = qi & 1;
            mbar_wait(&tfull[slot], (uint32_t)((qi >> 1) & 1));
            tc_fence_after();
            const int j0 = 4 * (qg + qi * g.n_qgroups);
            const bool vec = j0 + 3 < N_d && (N_d & 3) == 0;
#pragma unroll 1
            for (int ug = 0; ug < UP; ug += 4) {
                uint32_t ra[4][4], rb[4][4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    ct_ld4(ta + (uint32_t)slot * 256 + jj * 64 + ug, ra[jj]);            // h' = hi columns
                    ct_ld4(ta + (uint32_t)slot * 256 + jj * 64 + UP + ug, rb[jj]);       // h' = lo columns
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                float v[4][4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                    for (int k = 0; k < 4; ++k) v[jj][k] = __uint_as_float(ra[jj][k]) + __uint_as_float(rb[jj][k]);
                float im[4][4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        v[jj][k] += __shfl_xor_sync(0xffffffffu, v[jj][k], 1);     // + the other half row (h)
                        im[jj][k] = __shfl_xor_sync(0xffffffffu, v[jj][k], 2);     // c = 1 row: Im
                    }
                if (writer) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int u = ug + k;
                        if (u >= U) break;
                        const size_t o = ((size_t)n * U + u) * N_d + j0;
                        float2 y[4];
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) y[jj] = make_float2(v[jj][k], im[jj][k]);
                        if (vec) {
                            float4* p4 = reinterpret_cast<float4*>(yhat + o);
                            if (accumulate) {
                                const float4 a0 = p4[0], a1 = p4[1];
                                y[0].x += a0.x; y[0].y += a0.y; y[1].x += a0.z; y[1].y += a0.w;
                                y[2].x += a1.x; y[2].y += a1.y; y[3].x += a1.z; y[3].y += a1.w;
                            }
                            p4[0] = make_float4(y[0].x, y[0].y, y[1].x, y[1].y);
                            p4[1] = make_float4(y[2].x, y[2].y, y[3].x, y[3].y);
                        } else {
#pragma unroll
                            for (int jj = 0; jj < 4; ++jj) {
                                if (j0 + jj >= N_d) break;
                                if (accumulate) y[jj] = cadd(y[jj], yhat[o + jj]);
                                yhat[o + jj] = y[jj];
                            }
                        }
                        if constexpr (SER) {
#pragma unroll
                            for (int jj = 0; jj < 4; ++jj) {
                                if (j0 + jj >= N_d) break;
                                bool nr = false;
                                const int di = slice_axis(y[jj].x * sp.inv_ac, sp, nr);
                                const int dq = slice_axis(y[jj].y * sp.inv_ac, sp, nr);
                                const int dd = di + sp.m * dq;
                                if (dec) dec[o + jj] = (uint16_t)dd;
                                err += (dd != (int)idx[o + jj]);
                                nnear += nr;
                                ++cnt;
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[slot]);
        }
        if constexpr (SER) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                err += __shfl_xor_sync(0xffffffffu, err, o);
                nnear += __shfl_xor_sync(0xffffffffu, nnear, o);
                cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            }
            if (lane == 0) {
                if (err) atomicAdd(reinterpret_cast<unsigned long long*>(counts + 0), (unsigned long long)err);
                if (cnt) atomicAdd(reinterpret_cast<unsigned long long*>(counts + 1), (unsigned long long)cnt);
                if (nnear) atomicAdd(reinterpret_cast<unsigned long long*>(counts + 2), (unsigned long long)nnear);
            }
        }
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}
