// precode_tc.cu — ZF precoding (Eq. 1) as per-subcarrier complex GEMMs on the
// 5th-generation tensor cores (tcgen05.mma kind::tf32, accumulators in TMEM).
//
//   X[n][b][j] = sum_u P[b][u][j] s[n][u][j]
//
// For one data subcarrier j this is X_j = P_j s_j, a (B x U) . (U x n) complex product.  As a
// real GEMM with K = 2U:
//   A_j[b][k]     = [ Re P[b][u] (k = u) | Im P[b][u] (k = U + u) ]                (M = 128 antennas)
//   Bs_j[(n,0)][k] = [ Re s[n][u] | -Im s[n][u] ]   ->  D[b][(n,0)] = Re X[n][b][j]
//   Bs_j[(n,1)][k] = [ Im s[n][u] |  Re s[n][u] ]   ->  D[b][(n,1)] = Im X[n][b][j]
// (Bs rows are the GEMM's N dimension, both operands K-major in shared memory.)
//
// Precision (SURVEY §8(b) `math`):
//  * FD_MATH_TF32 (HL = 1): one TF32 pass (operands rounded to TF32, FP32 accumulation),
//    the north star's "TF32 tensor-core precoding" variant, parity 2e-3 (BASELINE configs[2]);
//    64 symbols per tile (N = 128).
//  * FD_MATH_FP32_TC (HL = 2): FP32-accurate split TF32.  x = hi + lo, hi = rna_tf32(x),
//    lo = rna_tf32(x - hi); the symbol operand carries both halves as rows (Bs = [s_hi ; s_lo],
//    N = 128 for 32 symbols) and every K step issues A_hi Bs (N = 128) and A_lo Bs_hi (N = 64):
//    D_big = A_hi s_hi, D_small = A_hi s_lo + A_lo s_hi (A_lo s_lo ~ 2^-22 relative dropped),
//    summed in FP32 in the epilogue.  Parity 2e-5 like the FP32 SIMT kernel.
//
// P operand: either the plain layout P [B][U][N_d] (8-byte gathers; the standalone `precode`)
// or the per-subcarrier packed layout Ppk [N_d][B][2U] written once per channel realisation by
// precode_pack (the rows of A_j, contiguous 256-byte rows at U = 32).
//
// CTA = (antenna tile of 128, symbol tile, contiguous range of subcarriers); one pipeline stage
// per subcarrier.  Warp roles (mbarrier rings, no CTA barrier in the loop):
//   warps 0-3   epilogue: TMEM lane quadrant (w % 4) = 32 antennas, all symbols of the tile; per quad of 4 subcarriers held in TMEM, sums big + small
//               and writes X[n][b][j..j+4) as full 32-byte sectors
//   warps 4-19  producers: load P / s for the stage (loads issued before waiting for the
//               buffer), split, store the K-major operands, fence.proxy.async, arrive
//   warp 20     MMA issue (one elected lane), commits to the stage's empty barrier and the TMEM
//               slot's full barrier
// Stages: NS shared-memory buffers; TMEM: one quad of 4 subcarriers x 128 columns (512).
#include "common.cuh"
#include "tcgen05.cuh"

namespace fdpd {

constexpr int PT_EPI = 4, PT_PROD = 16;
constexpr int PT_MMA_WARP = PT_EPI + PT_PROD;
constexpr int PT_THREADS = 32 * (PT_MMA_WARP + 1);
constexpr int PT_ROWS = 128;                 // rows of every operand plane (M = 128, N = 128)
constexpr int PT_PLANE = (PT_ROWS + 1) * 16; // bytes per 16-byte K chunk (4 tf32) plane, +1 row: conflict-free stores
constexpr int PT_SLOTS = 4, PT_COLS = 64;    // subcarriers per TMEM quad, columns per subcarrier (N = 64)

struct PtGeom {
    int U, B, N_d;
    long long n_sym;
    int planes;                // 2U / 4 K planes per operand
    int ns;                    // shared-memory stages
    int stage_bytes;           // A (HL planes sets) + Bs
    int n_btiles, n_ntiles, jper, n_jgroups;
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld4_nowait(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void split4(float4 x, float4& hi, float4& lo) {
    hi.x = tf32_rna(x.x); lo.x = tf32_rna(x.x - hi.x);
    hi.y = tf32_rna(x.y); lo.y = tf32_rna(x.y - hi.y);
    hi.z = tf32_rna(x.z); lo.z = tf32_rna(x.z - hi.z);
    hi.w = tf32_rna(x.w); lo.w = tf32_rna(x.w - hi.w);
}
__device__ __forceinline__ float4 rna4(float4 x) {
    return make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
}

// HL = 1 (TF32) or 2 (split TF32); PACKED: P is Ppk [N_d][B][2U] (else P [B][U][N_d]).
template <int HL, bool PACKED>
__global__ void __launch_bounds__(PT_THREADS, 1)
    k_precode_tc(const float* __restrict__ P, const float2* __restrict__ s, float2* __restrict__ X, PtGeom g) {
    constexpr int NT = 32;                   // symbols per tile (Bs rows 2 NT per hi / lo half)
    constexpr int NPW = NT / (PT_EPI / 4);   // symbols per epilogue warp column group
    extern __shared__ __align__(128) unsigned char sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int plane_set = g.planes * PT_PLANE;             // bytes of one operand (all K planes)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)g.ns * g.stage_bytes);
    uint64_t* full = bars;                   // [ns]
    uint64_t* empty = bars + g.ns;           // [ns]
    uint64_t* tfull = empty + g.ns;          // [2] quad buffers
    uint64_t* tempty = tfull + 2;            // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    if (tid == 0) {
        for (int i = 0; i < g.ns; ++i) {
            mbar_init(&full[i], 32 * PT_PROD);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 32 * PT_EPI);
        }
    }
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // work of this CTA: (antenna tile, symbol tile) fixed, subcarriers [ja, jb)
    int w = blockIdx.x;
    const int jg = w % g.n_jgroups;
    w /= g.n_jgroups;
    const int bt = w % g.n_btiles, nt = w / g.n_btiles;
    const int b0 = bt * PT_ROWS;
    const long long n0 = (long long)nt * NT;
    const int ja = jg * g.jper, jb = min(g.N_d, ja + g.jper);
    const int n_stages = max(0, jb - ja);
    const int U = g.U, B = g.B, N_d = g.N_d;

    if (warp >= PT_EPI && warp < PT_MMA_WARP) {
        // ---------------------------------------------------------------- producers
        // Software-pipelined by one stage: the loads of stage i + 1 are in flight while stage i
        // is split and stored (one stage of loads per thread left the loop latency-bound:
        // 1.9 TB/s at C5, long-scoreboard stalls).
        const int pt = tid - 32 * PT_EPI;
        const int KQ = g.planes;             // 16-byte k-quads per row (= U / 2)
        const int UQ = U >> 2;               // u-quads
        constexpr int MAXA = PACKED ? 4 : 2; // A items per thread at U <= 32 (128 rows x U/2 or U/4 quads)
        constexpr int PA = PACKED ? 1 : 4;   // float2 loads per plain A item
        const int na = PACKED ? PT_ROWS * KQ : PT_ROWS * UQ;
        const int ns_items = NT * UQ;        // symbol items (n, u-quad), <= 1 per thread
        struct Regs {
            float4 av[MAXA];
            float2 pv[MAXA][PA];
            float2 sv[4];
        };
        // per-thread item geometry, fixed over the stages (no integer divisions in the loop)
        constexpr int QSTEP = 32 * PT_PROD;  // item stride between a thread's items
        const int Q = PACKED ? KQ : UQ;      // quads per operand row
        int a_row[MAXA];                     // operand row r of item t (< 0: no item); its quad is
#pragma unroll                               //   it - r Q (a multiply, no division in the loop)
        for (int t = 0; t < MAXA; ++t) {
            const int it = pt + t * QSTEP;
            a_row[t] = it < na ? it / Q : -1;
        }
        auto a_quad = [&](int t) { return pt + t * QSTEP - a_row[t] * Q; };
        const bool s_item = pt < ns_items;
        const int s_u = s_item ? pt % UQ : 0, s_n = s_item ? pt / UQ : 0;
        const bool s_ok = s_item && n0 + s_n < g.n_sym;
        const float2* s_src = s + ((size_t)(n0 + (s_ok ? s_n : 0)) * U + 4 * s_u) * N_d;
        auto load = [&](int j, Regs& R) {
#pragma unroll
            for (int t = 0; t < MAXA; ++t) {
                const int r = a_row[t];
                if (r < 0) break;
                const bool ok = b0 + r < B;
                if constexpr (PACKED) {
                    R.av[t] = ok ? __ldg(reinterpret_cast<const float4*>(P + ((size_t)j * B + b0 + r) * 2 * U) + a_quad(t))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
                } else {
                    const float2* src = reinterpret_cast<const float2*>(P) + ((size_t)(b0 + r) * U + 4 * a_quad(t)) * N_d + j;
#pragma unroll
                    for (int q = 0; q < PA; ++q) R.pv[t][q] = ok ? __ldg(src + (size_t)q * N_d) : make_float2(0.f, 0.f);
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) R.sv[q] = s_ok ? __ldg(s_src + (size_t)q * N_d + j) : make_float2(0.f, 0.f);
        };
        auto store = [&](unsigned char* st, const Regs& R) {
            unsigned char* a_hi = st;
            unsigned char* a_lo = st + plane_set;
            unsigned char* bs = st + (HL == 2 ? 2 : 1) * plane_set;
#pragma unroll
            for (int t = 0; t < MAXA; ++t) {
                const int r = a_row[t];
                if (r < 0) break;
                if constexpr (PACKED) {
                    const size_t off = (size_t)a_quad(t) * PT_PLANE + r * 16;
                    if constexpr (HL == 2) {
                        float4 hi, lo;
                        split4(R.av[t], hi, lo);
                        *reinterpret_cast<float4*>(a_hi + off) = hi;
                        *reinterpret_cast<float4*>(a_lo + off) = lo;
                    } else {
                        *reinterpret_cast<float4*>(a_hi + off) = rna4(R.av[t]);
                    }
                } else {
                    const float4 re = make_float4(R.pv[t][0].x, R.pv[t][1].x, R.pv[t][2].x, R.pv[t][3].x);
                    const float4 im = make_float4(R.pv[t][0].y, R.pv[t][1].y, R.pv[t][2].y, R.pv[t][3].y);
                    const int aq = a_quad(t);
                    const size_t ore = (size_t)aq * PT_PLANE + r * 16, oim = (size_t)(UQ + aq) * PT_PLANE + r * 16;
                    if constexpr (HL == 2) {
                        float4 hi, lo;
                        split4(re, hi, lo);
                        *reinterpret_cast<float4*>(a_hi + ore) = hi;
                        *reinterpret_cast<float4*>(a_lo + ore) = lo;
                        split4(im, hi, lo);
                        *reinterpret_cast<float4*>(a_hi + oim) = hi;
                        *reinterpret_cast<float4*>(a_lo + oim) = lo;
                    } else {
                        *reinterpret_cast<float4*>(a_hi + ore) = rna4(re);
                        *reinterpret_cast<float4*>(a_hi + oim) = rna4(im);
                    }
                }
            }
            if (s_item) {
                const float4 re = make_float4(R.sv[0].x, R.sv[1].x, R.sv[2].x, R.sv[3].x);
                const float4 im = make_float4(R.sv[0].y, R.sv[1].y, R.sv[2].y, R.sv[3].y);
                // row (n, 0): [Re s | -Im s];  row (n, 1): [Im s | Re s]
                const int r0 = 2 * s_n, r1 = 2 * s_n + 1;
                const size_t p1 = (size_t)s_u * PT_PLANE, p2 = (size_t)(UQ + s_u) * PT_PLANE;
                if constexpr (HL == 2) {
                    float4 hi, lo;
                    split4(re, hi, lo);
                    *reinterpret_cast<float4*>(bs + p1 + r0 * 16) = hi;
                    *reinterpret_cast<float4*>(bs + p1 + (64 + r0) * 16) = lo;
                    *reinterpret_cast<float4*>(bs + p2 + r1 * 16) = hi;
                    *reinterpret_cast<float4*>(bs + p2 + (64 + r1) * 16) = lo;
                    split4(im, hi, lo);
                    *reinterpret_cast<float4*>(bs + p1 + r1 * 16) = hi;
                    *reinterpret_cast<float4*>(bs + p1 + (64 + r1) * 16) = lo;
                    *reinterpret_cast<float4*>(bs + p2 + r0 * 16) = make_float4(-hi.x, -hi.y, -hi.z, -hi.w);
                    *reinterpret_cast<float4*>(bs + p2 + (64 + r0) * 16) = make_float4(-lo.x, -lo.y, -lo.z, -lo.w);
                } else {
                    const float4 hre = rna4(re), him = rna4(im);
                    *reinterpret_cast<float4*>(bs + p1 + r0 * 16) = hre;
                    *reinterpret_cast<float4*>(bs + p2 + r0 * 16) = make_float4(-him.x, -him.y, -him.z, -him.w);
                    *reinterpret_cast<float4*>(bs + p1 + r1 * 16) = him;
                    *reinterpret_cast<float4*>(bs + p2 + r1 * 16) = hre;
                }
            }
        };
        int buf = 0;
        uint32_t ph = 0;
        Regs RA, RB;
        auto stage = [&](int i, Regs& cur, Regs& nxt) {
            if (i + 1 < n_stages) load(ja + i + 1, nxt);
            if (i >= g.ns) mbar_wait(&empty[buf], ph ^ 1u);
            store(sm + (size_t)buf * g.stage_bytes, cur);
            fence_proxy_async();
            mbar_arrive(&full[buf]);
            if (++buf == g.ns) { buf = 0; ph ^= 1u; }
        };
        if (n_stages > 0) load(ja, RA);
        for (int i = 0; i < n_stages; i += 2) {
            stage(i, RA, RB);
            if (i + 1 < n_stages) stage(i + 1, RB, RA);
        }
    } else if (warp == PT_MMA_WARP) {
        // ---------------------------------------------------------------- MMA issue
        const uint32_t base = smem_u32(sm);
        constexpr uint32_t ID64 = idesc_tf32_m128(64);
        const int ksteps = g.planes / 2;     // K = 8 per MMA = two 16-byte planes
        int buf = 0;
        uint32_t ph = 0;
        for (int i = 0; i < n_stages; ++i) {
            // TMEM: two quad buffers of 4 subcarriers x 64 columns; the first MMA of quad q waits
            // until the epilogue has drained quad q - 2
            const int slot = i & (PT_SLOTS - 1), q = i / PT_SLOTS, qb = q & 1;
            if (slot == 0 && q >= 2) mbar_wait(&tempty[qb], (uint32_t)(((q >> 1) - 1) & 1));
            mbar_wait(&full[buf], ph);
            tc_fence_after();
            const uint32_t sb = base + (uint32_t)buf * g.stage_bytes;
            const uint64_t dhi = umma_desc(sb, PT_PLANE, 128);
            const uint64_t dlo = umma_desc(sb + plane_set, PT_PLANE, 128);
            const uint64_t dbs = umma_desc(sb + (HL == 2 ? 2 : 1) * plane_set, PT_PLANE, 128);
            const uint64_t dbs_lo = dbs + (uint64_t)((64u * 16u) >> 4);         // rows 64..127: s_lo
            const uint32_t d = tmem + (uint32_t)qb * (PT_SLOTS * PT_COLS) + (uint32_t)slot * PT_COLS;
            if (elect_one()) {
                if constexpr (HL == 2) {
                    // one accumulator: the two small products first, the large A_hi s_hi last, so
                    // the tensor core's round-toward-zero accumulation acts on the full sum only
                    // in the last K steps (bias ~ K/8 ulp of X instead of 3 K/8)
                    for (int k = 0; k < ksteps; ++k) {
                        const uint64_t kadv = (uint64_t)((2u * k * PT_PLANE) >> 4);
                        mma_tf32(d, dlo + kadv, dbs + kadv, ID64, k > 0 ? 1u : 0u);
                        mma_tf32(d, dhi + kadv, dbs_lo + kadv, ID64, 1u);
                    }
                    for (int k = 0; k < ksteps; ++k) {
                        const uint64_t kadv = (uint64_t)((2u * k * PT_PLANE) >> 4);
                        mma_tf32(d, dhi + kadv, dbs + kadv, ID64, 1u);
                    }
                } else {
                    for (int k = 0; k < ksteps; ++k) {
                        const uint64_t kadv = (uint64_t)((2u * k * PT_PLANE) >> 4);
                        mma_tf32(d, dhi + kadv, dbs + kadv, ID64, k > 0 ? 1u : 0u);
                    }
                }
                umma_commit(&empty[buf]);
                if (slot == PT_SLOTS - 1 || i == n_stages - 1) umma_commit(&tfull[qb]);
            }
            __syncwarp();
            if (++buf == g.ns) { buf = 0; ph ^= 1u; }
        }
    } else if (warp < PT_EPI) {
        // ---------------------------------------------------------------- epilogue
        // per quad of 4 subcarriers: for 2 symbols at a time read the 4 slots' (big + small)
        // columns and write X[n][b][j..j+4) as one 32-byte sector per (n, b) (a partially
        // written sector costs a DRAM read-modify-write: measured 1.9x the X bytes with 16-byte runs)
        const int quad = warp & 3, grp = warp >> 2;
        const int b = b0 + quad * 32 + lane;
        const int nb = grp * NPW;            // first symbol (within the tile) of this warp
        const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16);
        for (int q = 0; q * PT_SLOTS < n_stages; ++q) {
            const int cnt = min(PT_SLOTS, n_stages - q * PT_SLOTS);
            const int jfirst = ja + q * PT_SLOTS;
            const int qb = q & 1;
            mbar_wait(&tfull[qb], (uint32_t)((q >> 1) & 1));
            tc_fence_after();
            const bool vec = cnt == 4 && ((N_d & 3) == 0) && ((jfirst & 3) == 0);
#pragma unroll 1
            for (int p = 0; p < NPW / 2; ++p) {
                const int nl = nb + 2 * p;                    // symbols nl, nl + 1 of the tile
                uint32_t r[PT_SLOTS][4];
#pragma unroll
                for (int t = 0; t < PT_SLOTS; ++t)
                    tmem_ld4_nowait(ta + (uint32_t)qb * (PT_SLOTS * PT_COLS) + (uint32_t)t * PT_COLS + 2 * nl, r[t]);
                tmem_wait_ld();
                float v[PT_SLOTS][4];
#pragma unroll
                for (int t = 0; t < PT_SLOTS; ++t)
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[t][e] = __uint_as_float(r[t][e]);
                if (b < B) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {             // v[t][2h], v[t][2h+1] = Re, Im X[nl + h][b][jfirst + t]
                        const long long n = n0 + nl + h;
                        if (n >= g.n_sym) break;
                        float2* dst = X + ((size_t)n * B + b) * N_d + jfirst;
                        if (vec) {
                            reinterpret_cast<float4*>(dst)[0] = make_float4(v[0][2 * h], v[0][2 * h + 1], v[1][2 * h], v[1][2 * h + 1]);
                            reinterpret_cast<float4*>(dst)[1] = make_float4(v[2][2 * h], v[2][2 * h + 1], v[3][2 * h], v[3][2 * h + 1]);
                        } else {
#pragma unroll
                            for (int t = 0; t < PT_SLOTS; ++t)
                                if (t < cnt) dst[t] = make_float2(v[t][2 * h], v[t][2 * h + 1]);
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[qb]);
        }
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// P [B][U][N_d] -> Ppk [N_d][B][2U]: row (j, b) = Re P[b][0..U)[j], Im P[b][0..U)[j] (fp32).
// CTA = (antenna b, 32 subcarriers): coalesced 256-byte reads of P rows, transposed in shared memory.
__global__ void __launch_bounds__(256) k_precode_pack(const float2* __restrict__ P, float* __restrict__ Ppk, int B,
                                                       int U, int N_d) {
    extern __shared__ __align__(16) float2 tile[];          // [U][33]
    const int b = blockIdx.y, j0 = blockIdx.x * 32;
    for (int e = threadIdx.x; e < U * 32; e += blockDim.x) {
        const int u = e >> 5, l = e & 31;
        tile[u * 33 + l] = j0 + l < N_d ? P[((size_t)b * U + u) * N_d + j0 + l] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 2 * U; e += blockDim.x) {
        const int k = e % (2 * U), l = e / (2 * U);
        if (j0 + l >= N_d) continue;
        const float2 v = tile[(k % U) * 33 + l];
        Ppk[((size_t)(j0 + l) * B + b) * 2 * U + k] = k < U ? v.x : v.y;
    }
}

int precode_simt(const void* P, const void* s, void* X, long long n_sym, int B_loc, int U, int N_d,
                 cudaStream_t stream);

static int launch_precode_tc(const void* P, bool packed, const void* s, void* X, long long n_sym, int B, int U,
                             int N_d, int math, cudaStream_t st) {
    FD_REQUIRE(U % 4 == 0 && U <= 32, "precode (tensor cores): U=%d must be a multiple of 4 and <= 32", U);
    FD_REQUIRE(aligned16(P) && aligned8(s) && aligned16(X), "precode (tensor cores): P / X 16-byte, s 8-byte aligned");
    const int HL = math == FD_MATH_TF32 ? 1 : 2;
    const int NT = 32;
    PtGeom g{};
    g.U = U;
    g.B = B;
    g.N_d = N_d;
    g.n_sym = n_sym;
    g.planes = U / 2;
    g.stage_bytes = (HL + 1) * g.planes * PT_PLANE;
    const size_t bar_bytes = 8 * (2 * 8 + 4) + 16;
    const size_t limit = 227 * 1024;
    g.ns = (int)std::min<size_t>(8, (limit - bar_bytes) / (size_t)g.stage_bytes);
    FD_REQUIRE(g.ns >= 2, "precode (tensor cores): U=%d too large", U);
    g.n_btiles = (B + PT_ROWS - 1) / PT_ROWS;
    const long long ntiles = (n_sym + NT - 1) / NT;
    FD_REQUIRE(ntiles * g.n_btiles < 65536, "precode (tensor cores): batch too large");
    g.n_ntiles = (int)ntiles;
    // one wave of persistent CTAs (one per SM: ~200 KB of stages, 512 TMEM columns); subcarrier
    // ranges in multiples of the epilogue's 4-subcarrier quads
    const int quads = (N_d + 3) / 4;
    int jg = std::max(1, (int)std::min<long long>(quads, (148LL + g.n_btiles * ntiles - 1) / (g.n_btiles * ntiles)));
    g.jper = 4 * ((quads + jg - 1) / jg);
    g.n_jgroups = (N_d + g.jper - 1) / g.jper;
    const size_t smem = (size_t)g.ns * g.stage_bytes + bar_bytes;
    const unsigned grid = (unsigned)(g.n_jgroups * g.n_btiles * ntiles);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, PT_THREADS, smem, st>>>((const float*)P, (const float2*)s, (float2*)X, g);
    };
    if (HL == 1) packed ? go(k_precode_tc<1, true>) : go(k_precode_tc<1, false>);
    else packed ? go(k_precode_tc<2, true>) : go(k_precode_tc<2, false>);
    return check_launch("precode (tensor cores)");
}

}  // namespace fdpd

using namespace fdpd;

extern "C" {

int precode(const void* P, const void* s, void* X, long long n_sym, int B_loc, int U, int N_d, int math,
            cudaStream_t stream) {
    FD_REQUIRE(math == FD_MATH_FP32 || math == FD_MATH_TF32 || math == FD_MATH_FP32_TC, "precode: math=%d", math);
    if (math == FD_MATH_FP32) return precode_simt(P, s, X, n_sym, B_loc, U, N_d, stream);
    FD_REQUIRE(n_sym >= 0 && B_loc >= 1 && U >= 1 && N_d >= 1, "precode: bad sizes");
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(P && s && X, "precode: NULL pointer");
    return launch_precode_tc(P, false, s, X, n_sym, B_loc, U, N_d, math, stream);
}

size_t precode_pack_bytes(int B_loc, int U, int N_d) {
    if (B_loc < 1 || U < 1 || N_d < 1) return 0;
    return (size_t)N_d * B_loc * 2 * U * sizeof(float);
}

int precode_pack(const void* P, void* Ppk, int B_loc, int U, int N_d, cudaStream_t stream) {
    FD_REQUIRE(B_loc >= 1 && U >= 1 && N_d >= 1 && B_loc <= 65535, "precode_pack: bad sizes");
    FD_REQUIRE(P && Ppk, "precode_pack: NULL pointer");
    FD_REQUIRE(aligned8(P) && aligned16(Ppk), "precode_pack: P 8-byte, Ppk 16-byte aligned");
    const size_t smem = sizeof(float2) * U * 33;
    FD_REQUIRE(smem <= 200 * 1024, "precode_pack: U=%d too large", U);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_precode_pack, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((N_d + 31) / 32, B_loc);
    k_precode_pack<<<grid, 256, smem, stream>>>((const float2*)P, (float*)Ppk, B_loc, U, N_d);
    return check_launch("precode_pack");
}

int precode_packed(const void* Ppk, const void* s, void* X, long long n_sym, int B_loc, int U, int N_d, int math,
                   cudaStream_t stream) {
    FD_REQUIRE(math == FD_MATH_TF32 || math == FD_MATH_FP32_TC, "precode_packed: math=%d (1 = TF32, 2 = FP32 TC)",
               math);
    FD_REQUIRE(n_sym >= 0 && B_loc >= 1 && U >= 1 && N_d >= 1, "precode_packed: bad sizes");
    if (n_sym == 0) return FD_OK;
    FD_REQUIRE(Ppk && s && X, "precode_packed: NULL pointer");
    return launch_precode_tc(Ppk, true, s, X, n_sym, B_loc, U, N_d, math, stream);
}

}  // extern "C"
