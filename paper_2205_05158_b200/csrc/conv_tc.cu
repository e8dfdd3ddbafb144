// conv_tc.cu — FD-CNN 3x3 "same" convolutions on the 5th-generation tensor cores
// (Eq. 15; BASELINE residual stack, readings A1-A6).
//
// A 3x3 convolution over an S x S image is an implicit GEMM
//     D[q][co] = sum_{tap, ci} A[q + off(tap)][ci] * W[tap][ci][co],
// q a pixel of the zero-haloed (S+2) x (S+2) image and off(tap) = (dy-1)(S+2) + (dx-1).
// Activations live channels-last in the haloed layout act[img][q][C], so the A operand
// of every tap is the SAME shared-memory tile shifted by off(tap) pixels: with the
// K-major no-swizzle descriptor layout (pixel rows 16 B apart, 4 channels per 16 B row,
// channel groups LBO apart) the shift is just the descriptor's start address — no
// im2col copy.  One CTA computes M = 128 consecutive pixels x all output channels per
// tile with tcgen05.mma kind::tf32 (M = 128, N = Cout padded to 16/32/64, K = 8 per
// instruction) into a TMEM accumulator (two, double-buffered across tiles).
//
// FP32 accuracy with TF32 tensor cores (the 2e-5 parity bar): both operands are split
// x = hi + lo with hi = rna_tf32(x), lo = rna_tf32(x - hi).  The weight halves sit side by
// side in N (B = [W_hi | W_lo], N = 2 Cout) and each K step issues two MMAs into one
// accumulator, A_hi [W_hi | W_lo] (N = 2 Cout) and A_lo W_hi (N = Cout, the first half of
// the same B tile): three of the four products (A_lo W_lo ~ 2^-22 relative is dropped),
// summed in the epilogue.  (An SS-mode
// MMA at N <= 64 costs the same ~46 cycles as at N = 16 — it is bound by reading the
// 4 KB A tile from shared memory — so doubling N is free where 3xTF32's third MMA is not.)  Weights are split once per call into a global image laid out exactly as
// the shared-memory B operand, copied in with cp.async.bulk (TMA); activations are split
// by the CTA while staging A.
//
// Layers: IN_MODE 1 reads the complex symbols (2 real channels, padded to K = 8);
// OUT_MODE 0 writes tanh(D + b) channels-last with a zero halo; OUT_MODE 1 (Cout = 2,
// N padded to 16) writes the residual s_out = s_in + D + b on the first N_d pixels.
#include <cstdlib>

#include "common.cuh"
#include "tcgen05.cuh"

namespace fdpd {

constexpr int TC_M = 128;

// Split-fp16 activation layout (ACT16, written by every layer's epilogue in the FP16 mode and
// read by the next layer): per image C/4 planes [c][hl][gq] (K chunk c of CK channels, hi / lo
// half, 8-channel group gq), each PP pixels x 16 bytes (8 fp16 values of x * 2^12) with TC_GLO
// zero guard pixels before pixel 0 and zeros after the last computed pixel.  A K chunk of a
// tile's A operand is then 2 CK / 8 contiguous pixel ranges, one per plane, copied into the
// shared-memory planes with cp.async.bulk as they are (no producer threads, no split).
constexpr int TC_GLO = 8;

struct TcConv {
    int S, Wp, P, N_d;        // image side, haloed side, haloed pixels, symbols per image
    int PP;                   // ACT16 plane length in pixels (guards included)
    int q_begin, q_end;       // computed pixel range [Wp, Wp + S Wp) (rows 1..S)
    int n_tiles;              // tiles per image
    int A_px, PL;             // staged pixels per tile, plane stride in bytes
    int Cin, Cout;            // real channel counts
    long long n_img;
    int ws, na;               // weight ring slots (9 = all taps resident), A buffers
    int off_a, off_bias, off_bar;   // smem byte offsets (weights at 0)
    int tmem_cols;
    int dbg;                  // experiments only (FDPD_TC_DBG): 1 = every TMA A copy reads tile 0 of image 0
};

// Weights W[co][ci][3][3] -> per tap [ci/4][n][4] with n < 2 NP: rows n < NP hold hi(W[n]),
// rows NP + co hold lo(W[co]); zero padded to CINP x NP.  This is exactly the shared-memory
// B operand (K-major, core matrices 8 rows x 4 ci) of one MMA with N = 2 NP, so
//     D[:, co] + D[:, NP + co] = A (W_hi + W_lo)[co].
__global__ void k_tc_weights(const float* __restrict__ W, float* __restrict__ Wg, int Cin, int Cout, int CINP, int NP) {
    const int per_tap = 2 * CINP * NP;
    const int n = 9 * per_tap;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const int tap = e / per_tap;
        int r = e - tap * per_tap;
        const int gq = r / (2 * NP * 4);
        r -= gq * 2 * NP * 4;
        const int row = r >> 2, ci = 4 * gq + (r & 3);
        const int hl = row >= NP, co = row - hl * NP;
        const float w = (co < Cout && ci < Cin) ? W[((size_t)co * Cin + ci) * 9 + tap] : 0.f;
        const float hi = tf32_rna(w);
        Wg[e] = hl ? tf32_rna(w - hi) : hi;
    }
}

// FP16 split (hidden layers, F16 = true): the same three products with fp16 halves (11 significant
// bits each, 22 together, like the TF32 split) on kind::f16, which takes K = 16 per MMA for the
// same 32 operand bytes per row: half the MMAs and half the shared-memory operand reads of the
// TF32 split.  fp16's range is handled by exact power-of-two scales: activations (tanh outputs,
// |x| <= 1) x 2^12, weights x 2^e with max |W| 2^e <= 2^14 (k_w_scale); the epilogue multiplies
// the accumulators by 2^-(12+e) (exact).  Residuals below the fp16 normal range (|x| < 2^-15)
// keep an absolute error <= 2^-37 instead of 2^-22 relative: negligible against the sums.
constexpr float TC_ACT_SCALE = 4096.f;

// tanh for the tensor-core epilogues: tanh x = (e - 1) / (e + 1), e = 2^(2 x log2 e) with
// ex2.approx (relative error ~2^-22) and a fast reciprocal, |x| clamped to 9 (tanh 9 = 1 - 3e-8):
// 6 branch-free instructions against tanhf's ~20 with divergent paths, which bound the epilogue
// warps (measured: tanhf's FFMA / FADD / BSSY / BSYNC were half of the 64 -> 64 layer's warp
// samples).  Error: absolute <= ~2e-7 for every x (e - 1 cancels near 0, where tanh ~ x), i.e.
// below the ~2.4e-7 relative resolution of the split-fp16 activations the next layer reads.
__device__ __forceinline__ float tanh_fast(float x) {
    const float xc = fminf(fmaxf(x, -9.f), 9.f);
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(xc * 2.8853900817779268f));
    return __fdividef(e - 1.f, e + 1.f);
}

// One CTA of 1024 threads, eight independent loads in flight per thread (a 256-thread loop of
// dependent loads took 68 us per 64 -> 64 layer: 2 % of the C5 step, three times per step).
__global__ void __launch_bounds__(1024) k_w_scale(const float* __restrict__ W, int n, float* __restrict__ scale) {
    __shared__ float red[32];
    float mm[8] = {};
    for (int i0 = threadIdx.x; i0 < n; i0 += 8 * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = i0 + k * blockDim.x;
            if (i < n) mm[k] = fmaxf(mm[k], fabsf(__ldg(W + i)));
        }
    }
    float m = fmaxf(fmaxf(fmaxf(mm[0], mm[1]), fmaxf(mm[2], mm[3])), fmaxf(fmaxf(mm[4], mm[5]), fmaxf(mm[6], mm[7])));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) scale[0] = m > 0.f ? exp2f(14.f - ceilf(log2f(m))) : 1.f;
    }
}

// fp16 weights: per tap [ci/8][n][8] with rows n < NP = hi(W[n] s), NP + co = lo(W[co] s).
__global__ void k_tc_weights_f16(const float* __restrict__ W, __half* __restrict__ Wg, int Cin, int Cout, int CINP,
                                 int NP, const float* __restrict__ scale) {
    const int per_tap = 2 * CINP * NP;
    const int n = 9 * per_tap;
    const float sc = scale[0];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const int tap = e / per_tap;
        int r = e - tap * per_tap;
        const int gq = r / (2 * NP * 8);
        r -= gq * 2 * NP * 8;
        const int row = r >> 3, ci = 8 * gq + (r & 7);
        const int hl = row >= NP, co = row - hl * NP;
        const float w = (co < Cout && ci < Cin) ? W[((size_t)co * Cin + ci) * 9 + tap] * sc : 0.f;
        const __half hi = __float2half_rn(w);
        Wg[e] = hl ? __float2half_rn(w - __half2float(hi)) : hi;
    }
}

// Warp roles (no CTA-wide barrier inside the tile loop; mbarrier pipelines between roles):
//   warps 0-7   epilogue: TMEM lane quadrant (w % 4) (pixels 32(w%4)..+31) x column half w / 4
//   warps 8-15  A producers: load, split hi/lo, store one K chunk (CK input channels) of a tile
//   warp 16     MMA issue (descriptors advanced by uniform adds; one elected lane issues)
//   warp 17     weight TMA: all slices resident (loaded once) or a ring of (chunk, tap) slices
// The A operand is staged per K chunk of CK = min(Cin, 32) channels (hi and lo planes), so a
// 64-channel layer keeps two A chunks in flight next to a 5-slot weight ring, where the
// whole-tile A staging (131 KB) left room for one A buffer and two weight slots.  The MMA
// warp does nothing but wait, issue and commit: it is latency-bound on its own instruction
// stream (measured: a ~100-instruction bookkeeping sequence per weight slice dominated the
// MMA warp's samples), so weight loads live in their own warp and each slice carries 8 MMAs.
// Rings: A chunks (na) with a_full (256 arrivals) / a_empty (tcgen05.commit), weight slices
// (ws) with wfull (TMA bytes) / wempty (commit), two TMEM accumulators with acc_full
// (commit) / acc_empty (256 arrivals).
// The first layer (IN_MODE 1: one K step per tap, C_out tanh per pixel) is bound by its
// epilogue's dependent tanh chains at two warps per scheduler, so it runs 16 epilogue warps
// (four column groups per TMEM lane quadrant) where C_out >= 32.
// TMA_A (hidden layers in the FP16 mode): the A operand arrives by cp.async.bulk from the
// ACT16 layout, so one producer warp (one elected lane) replaces the eight load / split warps.
template <int IN_MODE, int NP, bool TMA_A = false>
struct TcRoles {
    static constexpr int EPI = (IN_MODE == 1 && NP >= 32) ? 16 : 8;
    static constexpr int LOAD = TMA_A ? 1 : 8;
    static constexpr int MMA_WARP = EPI + LOAD, W_WARP = MMA_WARP + 1;
    static constexpr int THREADS = 32 * (W_WARP + 1);
    static constexpr int LOAD_THREADS = 32 * LOAD, EPI_THREADS = 32 * EPI;
};

// K chunk = 32 input channels for both precisions: with the fp16 split a 64-channel layer's
// 9 taps x 2 chunks of weights (144 KB) stay resident in shared memory next to two 32 KB A
// chunks (measured: streaming the weight slices from L2 every tile bound the 64 -> 64 layer,
// tensor pipe 35 % busy; 16-channel chunks with four A buffers measured slower, 0.94 vs
// 0.77 ms per C5 layer of 32 symbols); with the TF32 split (288 KB) they are streamed through
// a ring.
__host__ __device__ constexpr int tc_ck(int cinp, bool f16) {
    (void)f16;
    return cinp >= 32 ? 32 : cinp;
}

// OUT_MODE: 0 = tanh, fp32 channels-last; 1 = residual s_out (C_out = 2); 2 = tanh, ACT16.
// IN_MODE 0 with F16 reads ACT16 (TMA); IN_MODE 0 without F16 reads fp32 channels-last.
template <int CINP, int NP, int IN_MODE, int OUT_MODE, bool F16>
__global__ void __launch_bounds__(TcRoles<IN_MODE, NP, IN_MODE == 0 && F16>::THREADS, 1)
    k_conv_tc(const float* __restrict__ act_in, const float2* __restrict__ s_in, const void* __restrict__ Wg,
              const float* __restrict__ bias, const float* __restrict__ wscale, float* __restrict__ act_out,
              float2* __restrict__ s_out, TcConv g) {
    static_assert(!F16 || IN_MODE == 0, "the fp16 split serves the hidden layers");
    constexpr int EB = F16 ? 2 : 4;       // operand bytes per element in shared memory
    constexpr int G = CINP / 4;           // 16-byte fp32 channel groups of a pixel in global memory
    constexpr int CK = tc_ck(CINP, F16);  // input channels per K chunk
    constexpr int NCH = CINP / CK;        // K chunks per tile
    constexpr int GC = CK * EB / 16;      // 16-byte planes per hi / lo of one chunk
    constexpr int KPM = 32 / EB;          // K per MMA: 8 (tf32) or 16 (f16) = 32 bytes per row
    constexpr int KSC = CK / KPM;         // K steps per chunk (two MMAs each: A_hi, A_lo)
    constexpr int NW = 9 * NCH;           // weight slices per tile, order (chunk, tap)
    constexpr uint32_t WCB = (uint32_t)CK * 2 * NP * EB;  // bytes per weight slice
    constexpr uint32_t IDESC = F16 ? idesc_f16_m128(2 * NP) : idesc_tf32_m128(2 * NP);
    // the A_lo MMA reads only the first NP rows of B (W_hi): A_lo W_lo (~2^-22 relative) is
    // dropped and the MMA reads 25 % fewer shared-memory bytes
    constexpr uint32_t IDESC_LO = F16 ? idesc_f16_m128(NP) : idesc_tf32_m128(NP);
    constexpr bool TMA_A = IN_MODE == 0 && F16;
    using Roles = TcRoles<IN_MODE, NP, TMA_A>;
    constexpr int TC_EPI_WARPS = Roles::EPI, TC_LOAD_WARPS = Roles::LOAD;
    constexpr int TC_MMA_WARP = Roles::MMA_WARP, TC_W_WARP = Roles::W_WARP;
    constexpr int TC_LOAD_THREADS = Roles::LOAD_THREADS, TC_EPI_THREADS = Roles::EPI_THREADS;
    extern __shared__ __align__(128) unsigned char sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + g.off_bar);
    uint64_t* acc_full = bars;                 // [2]
    uint64_t* acc_empty = bars + 2;            // [2]
    uint64_t* a_full = bars + 4;               // [na]
    uint64_t* a_empty = a_full + g.na;         // [na]
    uint64_t* wfull = a_empty + g.na;          // [ws]
    uint64_t* wempty = wfull + g.ws;           // [ws]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + g.ws);
    float* bsm = reinterpret_cast<float*>(sm + g.off_bias);
    const uint32_t sm_base = smem_u32(sm);
    const uint32_t abytes = 2u * GC * g.PL;

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], TC_EPI_THREADS);
        }
        for (int i = 0; i < g.na; ++i) {
            mbar_init(&a_full[i], TMA_A ? 1 : TC_LOAD_THREADS);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < g.ws; ++i) {
            mbar_init(&wfull[i], 1);
            mbar_init(&wempty[i], 1);
        }
    }
    if (tid < NP) bsm[tid] = tid < g.Cout ? bias[tid] : 0.f;
    if (tid == NP) bsm[NP] = F16 ? 1.f / (TC_ACT_SCALE * wscale[0]) : 1.f;   // accumulator scale
    if (warp == 0) tmem_alloc(tmem_slot, g.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // 32-bit tile bookkeeping (the host guarantees n_img * n_tiles < 2^31); ring slots and
    // phases advance incrementally (no divisions in the role loops)
    const int total = (int)(g.n_img * g.n_tiles);
    const int my_tiles = total > (int)blockIdx.x ? (total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

    if (warp >= TC_EPI_WARPS && warp < TC_EPI_WARPS + TC_LOAD_WARPS) {
        // ------------------------------------------------------------ A producers
        const int lt = tid - TC_EPI_THREADS;
        int buf = 0, n_staged = 0;
        uint32_t ph = 0;
        int img = (int)blockIdx.x / g.n_tiles, t = (int)blockIdx.x - img * g.n_tiles;
        const int dimg = (int)gridDim.x / g.n_tiles, dt = (int)gridDim.x - dimg * g.n_tiles;
        if constexpr (TMA_A) {
            // one lane: per (tile, K chunk) the chunk's 2 GC planes, A_px pixels each, from ACT16
            const uint4* a16 = reinterpret_cast<const uint4*>(act_in);
            const uint32_t plane_bytes = (uint32_t)g.A_px * 16u;
            for (int i = 0; i < my_tiles; ++i) {
                const int qa = t * TC_M - 1;              // q0 - Wp - 1 with q0 = Wp + t TC_M
                for (int c = 0; c < NCH; ++c, ++n_staged) {
                    if (n_staged >= g.na) mbar_wait(&a_empty[buf], ph ^ 1u);
                    if (elect_one()) {
                        unsigned char* ab = sm + g.off_a + (size_t)buf * abytes;
                        mbar_arrive_expect_tx(&a_full[buf], 2u * GC * plane_bytes);
                        const uint4* src = (g.dbg & 1) ? a16 + (size_t)c * 2 * GC * g.PP + TC_GLO - 1
                                                       : a16 + ((size_t)img * (CINP / 4) + (size_t)c * 2 * GC) * g.PP + TC_GLO + qa;
#pragma unroll
                        for (int pl = 0; pl < 2 * GC; ++pl)
                            tma_bulk_g2s(ab + (size_t)pl * g.PL, src + (size_t)pl * g.PP, plane_bytes, &a_full[buf]);
                    }
                    __syncwarp();
                    if (++buf == g.na) { buf = 0; ph ^= 1u; }
                }
                img += dimg;
                t += dt;
                if (t >= g.n_tiles) { t -= g.n_tiles; ++img; }
            }
        } else
        for (int i = 0; i < my_tiles; ++i) {
            const int q0 = g.q_begin + t * TC_M;
            const int qa = q0 - g.Wp - 1;
            for (int c = 0; c < NCH; ++c, ++n_staged) {
                if (n_staged >= g.na) mbar_wait(&a_empty[buf], ph ^ 1u);
                unsigned char* ab = sm + g.off_a + (size_t)buf * abytes;
                if constexpr (IN_MODE == 0) {
                    const float4* src = reinterpret_cast<const float4*>(act_in + (size_t)img * g.P * CINP) + c * GC;
                    // PB independent 16-byte loads in flight per thread before any split / store
                    constexpr int PB = 8;
                    const int ne = g.A_px * GC;
                    for (int e0 = lt; e0 < ne; e0 += PB * TC_LOAD_THREADS) {
                        float4 x[PB];
#pragma unroll
                        for (int k = 0; k < PB; ++k) {
                            const int e = e0 + k * TC_LOAD_THREADS;
                            const int p = e / GC, gq = e - p * GC;
                            const int pos = qa + p;
                            x[k] = make_float4(0.f, 0.f, 0.f, 0.f);
                            if (e < ne && pos >= 0 && pos < g.P) x[k] = __ldg(src + (size_t)pos * G + gq);
                        }
#pragma unroll
                        for (int k = 0; k < PB; ++k) {
                            const int e = e0 + k * TC_LOAD_THREADS;
                            if (e >= ne) break;
                            const int p = e / GC, gq = e - p * GC;
                            float4 hi, lo;
                            hi.x = tf32_rna(x[k].x); lo.x = tf32_rna(x[k].x - hi.x);
                            hi.y = tf32_rna(x[k].y); lo.y = tf32_rna(x[k].y - hi.y);
                            hi.z = tf32_rna(x[k].z); lo.z = tf32_rna(x[k].z - hi.z);
                            hi.w = tf32_rna(x[k].w); lo.w = tf32_rna(x[k].w - hi.w);
                            *reinterpret_cast<float4*>(ab + (size_t)gq * g.PL + p * 16) = hi;
                            *reinterpret_cast<float4*>(ab + (size_t)(GC + gq) * g.PL + p * 16) = lo;
                        }
                    }
                } else {
                    // symbols: channel 0 = Re, 1 = Im of s[y S + x] (zero beyond N_d and on the halo)
                    const float2* simg = s_in + (size_t)img * g.N_d;
                    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int p = lt; p < g.A_px; p += TC_LOAD_THREADS) {
                        const int pos = qa + p;
                        float2 z = make_float2(0.f, 0.f);
                        if (pos >= 0 && pos < g.P) {
                            const int row = pos / g.Wp;
                            const int y = row - 1, x = pos - row * g.Wp - 1;
                            const int k = y * g.S + x;
                            if (y >= 0 && y < g.S && x >= 0 && x < g.S && k < g.N_d) z = __ldg(simg + k);
                        }
                        const float hx = tf32_rna(z.x), hy = tf32_rna(z.y);
                        *reinterpret_cast<float4*>(ab + p * 16) = make_float4(hx, hy, 0.f, 0.f);
                        *reinterpret_cast<float4*>(ab + (size_t)GC * g.PL + p * 16) =
                            make_float4(tf32_rna(z.x - hx), tf32_rna(z.y - hy), 0.f, 0.f);
#pragma unroll
                        for (int gq = 1; gq < GC; ++gq) {
                            *reinterpret_cast<float4*>(ab + (size_t)gq * g.PL + p * 16) = z4;
                            *reinterpret_cast<float4*>(ab + (size_t)(GC + gq) * g.PL + p * 16) = z4;
                        }
                    }
                }
                fence_proxy_async();                 // generic smem writes -> tensor-core reads
                mbar_arrive(&a_full[buf]);
                if (++buf == g.na) { buf = 0; ph ^= 1u; }
            }
            img += dimg;
            t += dt;
            if (t >= g.n_tiles) { t -= g.n_tiles; ++img; }
        }
    } else if (warp == TC_W_WARP) {
        // ------------------------------------------------------------ weight slices (TMA)
        const int my_slices = NW * my_tiles;
        const bool resident = g.ws == NW;
        const int n_load = resident ? (my_slices > 0 ? NW : 0) : my_slices;
        int lslot = 0, sl = 0;
        uint32_t lph = 0;
        for (int idx = 0; idx < n_load; ++idx) {
            if (idx >= g.ws) mbar_wait(&wempty[lslot], lph ^ 1u);
            if (elect_one()) {
                const int c = sl / 9, tap = sl - 9 * c;
                mbar_arrive_expect_tx(&wfull[lslot], WCB);
                tma_bulk_g2s(sm + (size_t)lslot * WCB,
                             static_cast<const char*>(Wg) + ((size_t)tap * CINP * 2 * NP + (size_t)c * CK * 2 * NP) * EB,
                             WCB, &wfull[lslot]);
            }
            __syncwarp();
            if (++lslot == g.ws) { lslot = 0; lph ^= 1u; }
            if (++sl == NW) sl = 0;
        }
    } else if (warp == TC_MMA_WARP) {
        // ------------------------------------------------------------ MMA issue
        const bool resident = g.ws == NW;
        const uint32_t PL16 = (uint32_t)g.PL >> 4, WP = (uint32_t)g.Wp;
        const uint64_t adesc0 = umma_desc(sm_base + g.off_a, (uint32_t)g.PL, 128);
        const uint64_t wdesc0 = umma_desc(sm_base, 2 * NP * 16, 128);
        int cslot = 0, buf = 0;
        uint32_t cph = 0, aph = 0;
        if (resident) {
            // Resident weights: after the first tile's weight waits, a chunk is one elected lane
            // issuing its 9 taps x KSC x 2 MMAs in a straight line (descriptors = loop-invariant
            // bases + compile-time offsets).  Measured: with a per-tap elect / syncwarp and the
            // per-tap descriptor arithmetic the MMA warp's own instruction stream bound the
            // 64 -> 64 layer (tensor-core smem pipe 64 % busy, the TMA producer waiting for buffers).
            uint64_t toff[9];
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) toff[tap] = (uint64_t)((tap / 3) * WP + (tap % 3));
            for (int i = 0; i < my_tiles; ++i) {
                const int acc = i & 1;
                if (i >= 2) mbar_wait(&acc_empty[acc], (uint32_t)(((i >> 1) - 1) & 1));
                const uint32_t d = tmem + (uint32_t)acc * (4 * NP);
#pragma unroll 1
                for (int c = 0; c < NCH; ++c) {
                    mbar_wait(&a_full[buf], aph);
                    if (i == 0)
                        for (int tap = 0; tap < 9; ++tap) mbar_wait(&wfull[c * 9 + tap], 0u);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint64_t abase = adesc0 + (uint64_t)(((uint32_t)buf * abytes) >> 4);
                        const uint64_t wbase = wdesc0 + (uint64_t)(((uint32_t)(c * 9) * WCB) >> 4);
#pragma unroll
                        for (int tap = 0; tap < 9; ++tap) {
                            const uint64_t at = abase + toff[tap];
                            const uint64_t wb = wbase + (uint64_t)((tap * WCB) >> 4);
                            const uint32_t dt = d + (tap >= 5 ? 2u * NP : 0u);   // tap groups, see below
#pragma unroll
                            for (int k = 0; k < KSC; ++k) {
                                const uint64_t ahi = at + (uint64_t)(2u * k * PL16);
                                const uint64_t alo = ahi + (uint64_t)(GC * PL16);
                                const uint64_t b = wb + (uint64_t)(2 * k * 2 * NP);
                                const uint32_t accum = (c | k) != 0 || (tap != 0 && tap != 5) ? 1u : 0u;
                                if constexpr (F16) {
                                    mma_f16(dt, ahi, b, IDESC, accum);
                                    mma_f16(dt + NP, alo, b, IDESC_LO, 1u);
                                } else {
                                    mma_tf32(dt, ahi, b, IDESC, accum);
                                    mma_tf32(dt + NP, alo, b, IDESC_LO, 1u);
                                }
                            }
                        }
                        umma_commit(&a_empty[buf]);
                        if (c == NCH - 1) umma_commit(&acc_full[acc]);
                    }
                    __syncwarp();
                    if (++buf == g.na) { buf = 0; aph ^= 1u; }
                }
            }
        } else
        for (int i = 0; i < my_tiles; ++i) {
            const int acc = i & 1;
            if (i >= 2) mbar_wait(&acc_empty[acc], (uint32_t)(((i >> 1) - 1) & 1));
            const uint32_t d = tmem + (uint32_t)acc * (4 * NP);   // two tap-group accumulators of 2 NP
#pragma unroll 1
            for (int c = 0; c < NCH; ++c) {
                mbar_wait(&a_full[buf], aph);
                tc_fence_after();
                const uint64_t abase = adesc0 + (uint64_t)(((uint32_t)buf * abytes) >> 4);
#pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                    const uint64_t at = abase + (uint64_t)((tap / 3) * WP + (tap % 3));
                    const int slot = resident ? c * 9 + tap : cslot;
                    if (!resident || i == 0) {   // resident weights: waited for once, at the first tile
                        mbar_wait(&wfull[slot], resident ? 0u : cph);
                        tc_fence_after();
                    }
                    const uint64_t wb = wdesc0 + (uint64_t)(((uint32_t)slot * WCB) >> 4);
                    // taps 0-4 and 5-8 accumulate in separate TMEM accumulators (summed in the
                    // epilogue): with the tensor core's round-toward-zero accumulation the bias
                    // grows with the number of MMAs into one running sum
                    const uint32_t dt = d + (tap >= 5 ? 2u * NP : 0u);
                    if (elect_one()) {
#pragma unroll
                        for (int k = 0; k < KSC; ++k) {
                            const uint64_t ahi = at + (uint64_t)(2u * k * PL16);
                            const uint64_t alo = ahi + (uint64_t)(GC * PL16);
                            const uint64_t b = wb + (uint64_t)(2 * k * 2 * NP);
                            const uint32_t accum = (c | k) != 0 || (tap != 0 && tap != 5) ? 1u : 0u;
                            if constexpr (F16) mma_f16(dt, ahi, b, IDESC, accum);
                            else mma_tf32(dt, ahi, b, IDESC, accum);
                            // A_lo x W_hi (N = NP) into the small-term half (columns NP..2NP, next to
                            // A_hi x W_lo): the tensor core's FP32 accumulation rounds toward zero,
                            // so every MMA into the large A_hi W_hi accumulator adds a bias of ~1/2
                            // ulp of the running sum; keeping the small products out of it halves
                            // that bias (C5: the CNN output's coherent error 1.1e-6 -> see DESIGN)
                            if constexpr (F16) mma_f16(dt + NP, alo, b, IDESC_LO, 1u);
                            else mma_tf32(dt + NP, alo, b, IDESC_LO, 1u);
                        }
                        if (!resident) umma_commit(&wempty[cslot]);
                    }
                    __syncwarp();
                    if (!resident && ++cslot == g.ws) { cslot = 0; cph ^= 1u; }
                }
                if (elect_one()) umma_commit(&a_empty[buf]);
                __syncwarp();
                if (++buf == g.na) { buf = 0; aph ^= 1u; }
            }
            if (elect_one()) umma_commit(&acc_full[acc]);
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ epilogue (warps 0-7)
        // warp w reads TMEM lanes 32 (w % 4) .. + 31 (its pixels) and the column half w / 4
        constexpr int NGRP = TC_EPI_WARPS / 4;    // column groups per TMEM lane quadrant
        const int quad = warp & 3, half = warp >> 2;
        int img = (int)blockIdx.x / g.n_tiles, t = (int)blockIdx.x - img * g.n_tiles;
        const int dimg = (int)gridDim.x / g.n_tiles, dt = (int)gridDim.x - dimg * g.n_tiles;
        for (int i = 0; i < my_tiles; ++i, img += dimg, t += dt) {
            if (t >= g.n_tiles) { t -= g.n_tiles; ++img; }
            const int acc = i & 1;
            mbar_wait(&acc_full[acc], (uint32_t)((i >> 1) & 1));
            tc_fence_after();
            const int pos = g.q_begin + t * TC_M + quad * 32 + lane;
            const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)acc * (4 * NP);
            const int prow = pos / g.Wp, pcol = pos - prow * g.Wp;
            const bool interior = pos < g.q_end && pcol >= 1 && pcol <= g.S;
            const float dscale = bsm[NP];
            if constexpr (OUT_MODE == 2) {
                // ACT16: the next layer's K chunks (CKO channels) -> planes [c][hl][gq] of 8 channels
                constexpr int CKO = tc_ck(NP, true), GCO = CKO / 8, NPL = NP / 4;
                uint4* o = reinterpret_cast<uint4*>(act_out) + (size_t)img * NPL * g.PP + TC_GLO + pos;
                constexpr int HC = NP / NGRP;
#pragma unroll
                for (int c0 = half * HC; c0 < (half + 1) * HC; c0 += 8) {
                    float v[8], w[8], v2[8], w2[8];
                    tmem_ld8(tbase + c0, v);
                    tmem_ld8(tbase + NP + c0, w);
                    tmem_ld8(tbase + 2 * NP + c0, v2);
                    tmem_ld8(tbase + 3 * NP + c0, w2);
                    // halo / pad pixels: x 0 (a multiply, not a per-element branch: the ternary
                    // compiled to a BSSY / BSYNC region with the bias load inside, per element)
                    const float4 b0 = *reinterpret_cast<const float4*>(bsm + c0);
                    const float4 b1 = *reinterpret_cast<const float4*>(bsm + c0 + 4);
                    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                    const float keep = interior ? TC_ACT_SCALE : 0.f;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        v[j] = keep * tanh_fast(((v[j] + v2[j]) + (w[j] + w2[j])) * dscale + bb[j]);
                    uint4 hi, lo;
                    split_f16x2(v[0], v[1], hi.x, lo.x);
                    split_f16x2(v[2], v[3], hi.y, lo.y);
                    split_f16x2(v[4], v[5], hi.z, lo.z);
                    split_f16x2(v[6], v[7], hi.w, lo.w);
                    const int pl = (c0 / CKO) * 2 * GCO + (c0 % CKO) / 8;
                    if (pos < g.q_end) {
                        o[(size_t)pl * g.PP] = hi;
                        o[(size_t)(pl + GCO) * g.PP] = lo;
                    }
                }
                tc_fence_before();
                mbar_arrive(&acc_empty[acc]);
                // guards + halo row 0 (pixels -TC_GLO .. Wp - 1) from the first tile, halo row S + 1
                // and everything after it (pixels q_end .. PP - TC_GLO - 1) from the last tile
                for (int side = 0; side < 2; ++side) {
                    if (t != (side ? g.n_tiles - 1 : 0)) continue;
                    const int a = side ? TC_GLO + g.q_end : 0, len = side ? g.PP - a : TC_GLO + g.Wp;
                    uint4* z = reinterpret_cast<uint4*>(act_out) + (size_t)img * NPL * g.PP + a;
                    for (int e = tid; e < NPL * len; e += TC_EPI_THREADS) {
                        const int pl = e / len;
                        z[(size_t)pl * g.PP + (e - pl * len)] = make_uint4(0u, 0u, 0u, 0u);
                    }
                }
            } else if constexpr (OUT_MODE == 0) {
                float* o = act_out + ((size_t)img * g.P + pos) * NP;
                constexpr int HC = NP / NGRP;         // columns per warp (>= 8)
#pragma unroll
                for (int c0 = half * HC; c0 < (half + 1) * HC; c0 += 8) {
                    float v[8], w[8], v2[8], w2[8];
                    tmem_ld8(tbase + c0, v);               // taps 0-4: A_hi W_hi
                    tmem_ld8(tbase + NP + c0, w);          //           A_hi W_lo + A_lo W_hi
                    tmem_ld8(tbase + 2 * NP + c0, v2);     // taps 5-8
                    tmem_ld8(tbase + 3 * NP + c0, w2);
                    const float4 b0 = *reinterpret_cast<const float4*>(bsm + c0);
                    const float4 b1 = *reinterpret_cast<const float4*>(bsm + c0 + 4);
                    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                    const float keep = interior ? 1.f : 0.f;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        v[j] = keep * tanh_fast(((v[j] + v2[j]) + (w[j] + w2[j])) * dscale + bb[j]);
                    if (pos < g.q_end) {
                        reinterpret_cast<float4*>(o + c0)[0] = make_float4(v[0], v[1], v[2], v[3]);
                        reinterpret_cast<float4*>(o + c0)[1] = make_float4(v[4], v[5], v[6], v[7]);
                    }
                }
                tc_fence_before();
                mbar_arrive(&acc_empty[acc]);
                // the halo rows 0 and S+1 are never computed: zero them from the first / last tile
                for (int side = 0; side < 2; ++side) {
                    if (t != (side ? g.n_tiles - 1 : 0)) continue;
                    float4* z = reinterpret_cast<float4*>(act_out + ((size_t)img * g.P + (side ? g.q_end : 0)) * NP);
                    for (int e = tid; e < g.Wp * NP / 4; e += TC_EPI_THREADS) z[e] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            } else {
                float v[8], w[8], v2[8], w2[8];
                if (half == 0) {
                    tmem_ld8(tbase, v);
                    tmem_ld8(tbase + NP, w);
                    tmem_ld8(tbase + 2 * NP, v2);
                    tmem_ld8(tbase + 3 * NP, w2);
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        v[j] += v2[j];
                        w[j] += w2[j];
                    }
                }
                tc_fence_before();
                mbar_arrive(&acc_empty[acc]);
                const int k = (prow - 1) * g.S + (pcol - 1);
                if (half == 0 && interior && k < g.N_d) {
                    const size_t o = (size_t)img * g.N_d + k;
                    const float2 z = __ldg(s_in + o);
                    s_out[o] = make_float2(z.x + ((v[0] + w[0]) * dscale + bsm[0]), z.y + ((v[1] + w[1]) * dscale + bsm[1]));
                }
            }
        }
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, g.tmem_cols);
    }
}

// Last layer (C_out = 2) on the FP32 pipe.  On the tensor cores this layer paid the full A
// operand read (9 taps x C_in x hi/lo per pixel) for an N = 16 tile of which 2 columns are
// real (1.9 ms of the C5 CNN's 10.9 ms); as a direct convolution it is 2 x 9 x C_in FMAs per
// pixel.  A group of G = C_in / 4 consecutive lanes owns a 4 x 4 block of output pixels, lane
// gq its 4 input channels 4gq..4gq+3: the group's loads of one haloed pixel are G consecutive
// float4 (coalesced; a 6 x 6 haloed window per 16 outputs), each lane accumulates its
// channels' share of the 16 pixels x 2 outputs,
// and the group reduces with shuffles.  Weights sit in shared memory as [j][tap][gq] float2
// (both outputs), conflict-free across the group.  Writes s_out = s_in + out + b on the first
// N_d pixels (A2-A5).
template <int CINP>
__global__ void __launch_bounds__(256) k_conv_out_cl(const float* __restrict__ act, const float* __restrict__ W,
                                                     const float* __restrict__ bias, const float2* __restrict__ s_in,
                                                     float2* __restrict__ s_out, int S, int Cin, int N_d,
                                                     long long n_img) {
    constexpr int G = CINP / 4;           // lanes per pixel block
    __shared__ float2 wsm[4 * 9 * G];     // [j][tap][gq] -> (W[0][4gq+j][tap], W[1][4gq+j][tap])
    for (int e = threadIdx.x; e < 4 * 9 * G; e += blockDim.x) {
        const int gq = e % G, r = e / G, tap = r % 9, j = r / 9, ci = 4 * gq + j;
        wsm[e] = ci < Cin ? make_float2(W[((size_t)0 * Cin + ci) * 9 + tap], W[((size_t)1 * Cin + ci) * 9 + tap])
                          : make_float2(0.f, 0.f);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, gq = lane % G;
    constexpr int BS = 4;                 // output block side
    const int Wp = S + 2, nbx = (S + BS - 1) / BS, nblk = nbx * nbx;
    const long long gi = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / G;   // pixel block
    const bool active = gi < n_img * nblk;
    const long long img = active ? gi / nblk : 0;
    const int blk = active ? (int)(gi - img * nblk) : 0, by = blk / nbx, bx = blk - by * nbx;
    const int y0 = BS * by, x0 = BS * bx;   // output pixel (y0, x0); haloed rows / cols y0 .. y0 + BS + 1
    const float4* a4 = reinterpret_cast<const float4*>(act + (size_t)img * Wp * Wp * CINP) + gq;
    float2 acc[BS * BS];                  // (out 0, out 1) of pixel py * BS + px: one FFMA2 per weight pair
#pragma unroll
    for (int p = 0; p < BS * BS; ++p) acc[p] = make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < BS + 2; ++r) {
        float4 nb[BS + 2];
#pragma unroll
        for (int c = 0; c < BS + 2; ++c) {
            const int yy = y0 + r, xx = x0 + c;
            nb[c] = (active && yy < Wp && xx < Wp) ? __ldg(a4 + ((size_t)yy * Wp + xx) * G)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int py = 0; py < BS; ++py) {
            const int dy = r - py;
            if (dy < 0 || dy > 2) continue;
#pragma unroll
            for (int px = 0; px < BS; ++px)
#pragma unroll
                for (int dx = 0; dx < 3; ++dx) {
                    const float4 q = nb[px + dx];
                    const int tap = dy * 3 + dx;
                    const float2 w0 = wsm[(0 * 9 + tap) * G + gq], w1 = wsm[(1 * 9 + tap) * G + gq];
                    const float2 w2 = wsm[(2 * 9 + tap) * G + gq], w3 = wsm[(3 * 9 + tap) * G + gq];
                    float2 a = acc[py * BS + px];
                    a = cfma_real(w0, q.x, a);
                    a = cfma_real(w1, q.y, a);
                    a = cfma_real(w2, q.z, a);
                    a = cfma_real(w3, q.w, a);
                    acc[py * BS + px] = a;
                }
        }
    }
    // Reduce-scatter over the group's G lanes: at every level a lane hands one half of its pixels to
    // its partner and keeps the other (G - 1 exchanges of float2 per lane pair of levels instead of
    // a full butterfly over all 16 pixels), so each lane ends with the complete sums of 16 / G
    // pixels and writes them itself.  The order of the additions is fixed by the lane layout.
    int base = 0;                          // first pixel this lane still holds
#pragma unroll
    for (int o = G / 2, cnt = BS * BS; o > 0; o >>= 1, cnt >>= 1) {
        const bool hi = (gq & o) != 0;
#pragma unroll
        for (int i = 0; i < BS * BS / 2; ++i) {
            if (i >= cnt / 2) break;
            const float2 send = hi ? acc[i] : acc[i + cnt / 2];
            const float2 keep = hi ? acc[i + cnt / 2] : acc[i];
            float2 recv;
            recv.x = __shfl_xor_sync(0xffffffffu, send.x, o);
            recv.y = __shfl_xor_sync(0xffffffffu, send.y, o);
            acc[i] = fadd2(keep, recv);
        }
        base += hi ? cnt / 2 : 0;
    }
    if (!active) return;
    const float b0 = bias[0], b1 = bias[1];
#pragma unroll
    for (int i = 0; i < BS * BS / G; ++i) {
        const int p = base + i, py = p / BS, px = p - py * BS;
        const int y = y0 + py, x = x0 + px;
        const int k = y * S + x;
        if (y < S && x < S && k < N_d) {
            const size_t o = (size_t)img * N_d + k;
            const float2 z = __ldg(s_in + o);
            s_out[o] = make_float2(z.x + (acc[i].x + b0), z.y + (acc[i].y + b1));
        }
    }
}

// ============================================================================ host side
static int pad_ch(int c) { return c <= 8 ? 8 : (c <= 16 ? 16 : (c <= 32 ? 32 : 64)); }
static int pad_n(int c) { return c <= 16 ? 16 : (c <= 32 ? 32 : 64); }

// Whether every layer of chans maps onto k_conv_tc (first 2 -> C, middle C -> C', last C -> 2,
// C in {16, 32, 64}).
bool tc_supported(const int* chans, int n_layers) {
    if (n_layers < 2 || chans[0] != 2 || chans[n_layers] != 2) return false;
    for (int l = 1; l < n_layers; ++l)
        if (chans[l] != 16 && chans[l] != 32 && chans[l] != 64) return false;
    return true;
}

static TcConv tc_geom(int S, int N_d, int Cin, int Cout, long long n_img) {
    TcConv g{};
    g.S = S;
    g.Wp = S + 2;
    g.P = g.Wp * g.Wp;
    g.N_d = N_d;
    g.q_begin = g.Wp;
    g.q_end = g.Wp + S * g.Wp;
    g.n_tiles = (S * g.Wp + TC_M - 1) / TC_M;
    g.A_px = (TC_M + 2 * g.Wp + 2 + 7) & ~7;
    g.PL = (g.A_px + 1) * 16;   // one spare row: the 4-channel groups of a pixel hit distinct banks
    // ACT16 planes: guards, then every pixel a tile's A range can touch (up to (n_tiles - 1) TC_M + A_px - 2)
    g.PP = (TC_GLO + std::max(g.P, (g.n_tiles - 1) * TC_M + g.A_px) + 8 + 7) & ~7;
    g.Cin = Cin;
    g.Cout = Cout;
    g.n_img = n_img;
    static const int dbg = [] {
        const char* e = getenv("FDPD_TC_DBG");
        return e ? atoi(e) : 0;
    }();
    g.dbg = dbg;
    return g;
}

// smem plan: weight slices (ws slots of CK x 2NP) | A chunk ring (na buffers) | bias |
// barriers.  Order of preference: resident weights with >= 2 A chunks in flight; a weight
// ring of >= 4 slices with >= 2 A chunks; then shallower variants.
static size_t tc_plan(TcConv& g, int CINP, int NP, bool f16) {
    const int EB = f16 ? 2 : 4;
    const int CK = tc_ck(CINP, f16), NW = 9 * (CINP / CK);
    const size_t slice = (size_t)CK * 2 * NP * EB, abuf = 2ull * (CK * EB / 16) * g.PL;
    const size_t limit = 227 * 1024;
    auto bytes_of = [&](int ws, int na, size_t& off_a, size_t& off_bias, size_t& off_bar) {
        off_a = ws * slice;
        off_bias = off_a + na * abuf;
        off_bar = (off_bias + (NP + 4) * 4 + 15) & ~(size_t)15;
        return off_bar + 8 * (4 + 2 * na + 2 * ws) + 16;
    };
    auto take = [&](int ws, int na) -> size_t {
        size_t oa, ob, obar;
        const size_t bytes = bytes_of(ws, na, oa, ob, obar);
        if (bytes > limit) return 0;
        g.ws = ws;
        g.na = na;
        g.off_a = (int)oa;
        g.off_bias = (int)ob;
        g.off_bar = (int)obar;
        int cols = 32;
        while (cols < 8 * NP) cols <<= 1;   // two tiles x two tap-group accumulators of N = 2 NP
        g.tmem_cols = cols;
        return bytes;
    };
    size_t r;
    // experiment switch (FDPD_TC_WRING=<ws>): stream the weights through a ring of ws slices
    // and give the freed shared memory to A buffers
    static const int wring = [] {
        const char* e = getenv("FDPD_TC_WRING");
        return e ? atoi(e) : 0;
    }();
    if (wring > 0 && wring < NW)
        for (int na = 6; na >= 2; --na)
            if ((r = take(wring, na))) return r;
    for (int na = 4; na >= 2; --na)
        if ((r = take(NW, na))) return r;
    for (int na = 4; na >= 2; --na)
        for (int ws = 16; ws >= 4; --ws)
            if (ws < NW && (r = take(ws, na))) return r;
    for (int na = 2; na >= 1; --na) {
        if ((r = take(NW, na))) return r;
        for (int ws = 8; ws >= 2; --ws)
            if (ws < NW && (r = take(ws, na))) return r;
    }
    return 0;
}

template <int CINP, int NP, int IN_MODE, int OUT_MODE, bool F16>
static int launch_tc_na(const TcConv& g, size_t smem, const float* act_in, const float2* s_in, const void* Wg,
                        const float* bias, const float* wscale, float* act_out, float2* s_out, cudaStream_t st) {
    auto kern = k_conv_tc<CINP, NP, IN_MODE, OUT_MODE, F16>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0, dev = 0, nsm = 148;
    constexpr int THREADS = TcRoles<IN_MODE, NP, IN_MODE == 0 && F16>::THREADS;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long tiles = g.n_img * g.n_tiles;
    const long long grid = std::min<long long>(tiles, (long long)nsm * std::max(per_sm, 1));
    kern<<<(unsigned)grid, THREADS, smem, st>>>(act_in, s_in, Wg, bias, wscale, act_out, s_out, g);
    return check_launch("fdcnn_forward (tensor-core conv)");
}

template <int IN_MODE, int OUT_MODE, int CINP, bool F16>
static int launch_tc_n(int NP, const TcConv& g, size_t smem, const float* act_in, const float2* s_in, const void* Wg,
                       const float* bias, const float* wscale, float* act_out, float2* s_out, cudaStream_t st) {
    switch (NP) {
        case 16: return launch_tc_na<CINP, 16, IN_MODE, OUT_MODE, F16>(g, smem, act_in, s_in, Wg, bias, wscale, act_out, s_out, st);
        case 32: return launch_tc_na<CINP, 32, IN_MODE, OUT_MODE, F16>(g, smem, act_in, s_in, Wg, bias, wscale, act_out, s_out, st);
        default: return launch_tc_na<CINP, 64, IN_MODE, OUT_MODE, F16>(g, smem, act_in, s_in, Wg, bias, wscale, act_out, s_out, st);
    }
}

// Hidden-layer operand precision: FP16 split (default) or the TF32 split (fd_set_cnn_tc_precision).
static int g_tc_f16 = 1;

// Workspace: two channels-last haloed activation buffers + the split weights of every layer.
size_t fdcnn_tc_workspace_bytes(const int* chans, int n_layers, long long n_sym, int U, int N_d) {
    int S = 1;
    while (S * S < N_d) ++S;
    // activations: P pixels x C fp32 (TF32 mode) or C / 4 ACT16 planes of PP pixels x 16 B
    const size_t P = (size_t)tc_geom(S, N_d, 2, 2, 1).PP;
    int cmax = 0;
    for (int l = 1; l < n_layers; ++l) cmax = chans[l] > cmax ? chans[l] : cmax;
    const size_t one = (((size_t)n_sym * U * P * cmax * 4) + 255) & ~(size_t)255;
    size_t bytes = (n_layers > 2 ? 2 : 1) * one;
    for (int l = 0; l < n_layers; ++l)
        bytes += (((size_t)9 * 2 * pad_ch(chans[l]) * pad_n(chans[l + 1]) * 4 + 255) & ~(size_t)255) + 256;
    return bytes;
}

int fdcnn_tc_forward(const float* params, const int* chans, int n_layers, const float2* s_in, float2* s_out,
                     void* workspace, long long n_sym, int U, int N_d, cudaStream_t stream) {
    int S = 1;
    while (S * S < N_d) ++S;
    const long long n_img = n_sym * U;
    const size_t P = (size_t)tc_geom(S, N_d, 2, 2, 1).PP;
    int cmax = 0;
    for (int l = 1; l < n_layers; ++l) cmax = chans[l] > cmax ? chans[l] : cmax;
    const size_t one = (((size_t)n_img * P * cmax * 4) + 255) & ~(size_t)255;
    char* ws = static_cast<char*>(workspace);
    float* act[2] = {reinterpret_cast<float*>(ws), reinterpret_cast<float*>(ws + (n_layers > 2 ? one : 0))};
    char* wptr = ws + (n_layers > 2 ? 2 : 1) * one;
    size_t off = 0;
    int rc = FD_OK;
    for (int l = 0; l < n_layers; ++l) {
        const int ci = chans[l], co = chans[l + 1];
        const int CINP = pad_ch(ci), NP = pad_n(co);
        const float* W = params + off;
        const float* b = W + (size_t)co * ci * 9;
        off += (size_t)co * ci * 9 + co;
        const bool first = l == 0, last = l == n_layers - 1;
        const bool f16 = g_tc_f16 && !first && !last;
        void* Wg = wptr;
        const int nw = 9 * 2 * CINP * NP;
        wptr += ((size_t)nw * 4 + 255) & ~(size_t)255;
        float* wscale = reinterpret_cast<float*>(wptr);
        wptr += 256;
        if (f16) {
            k_w_scale<<<1, 1024, 0, stream>>>(W, co * ci * 9, wscale);
            k_tc_weights_f16<<<(nw + 255) / 256, 256, 0, stream>>>(W, static_cast<__half*>(Wg), ci, co, CINP, NP,
                                                                   wscale);
        } else if (!last) {
            k_tc_weights<<<(nw + 255) / 256, 256, 0, stream>>>(W, static_cast<float*>(Wg), ci, co, CINP, NP);
        }
        if ((rc = check_launch("fdcnn_forward (weight split)"))) return rc;
        TcConv g = tc_geom(S, N_d, ci, co, n_img);
        FD_REQUIRE(n_img * g.n_tiles < (1LL << 31), "fdcnn_forward: too many images per call for the tensor-core path");
        const size_t smem = tc_plan(g, CINP, NP, f16);
        if (!smem) return fail_arg("fdcnn_forward: tensor-core plan does not fit shared memory");
        const float* in = first ? nullptr : act[(l - 1) & 1];
        float* out = last ? nullptr : act[l & 1];
        // FP16 mode: every intermediate activation in the ACT16 layout (first layer's epilogue
        // splits, hidden layers stage A by TMA, the last layer reads hi + lo)
        // FP16 mode: the activations between two tensor-core layers are in the ACT16 layout
        // (the producing epilogue splits, the consumer stages A by TMA); the input of the last
        // layer (FP32 direct convolution) stays fp32 channels-last
        const bool next_f16 = g_tc_f16 && l + 1 < n_layers - 1;
        if (first) {
            rc = next_f16 ? launch_tc_n<1, 2, 8, false>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream)
                          : launch_tc_n<1, 0, 8, false>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream);
        } else if (last) {
            // C_out = 2: direct FP32 convolution on the channels-last activations
            const long long nth = n_img * (long long)(((S + 3) / 4) * ((S + 3) / 4)) * (CINP / 4);
            const unsigned blocks = (unsigned)((nth + 255) / 256);
            switch (CINP) {
                case 16: k_conv_out_cl<16><<<blocks, 256, 0, stream>>>(in, W, b, s_in, s_out, S, ci, N_d, n_img); break;
                case 32: k_conv_out_cl<32><<<blocks, 256, 0, stream>>>(in, W, b, s_in, s_out, S, ci, N_d, n_img); break;
                default: k_conv_out_cl<64><<<blocks, 256, 0, stream>>>(in, W, b, s_in, s_out, S, ci, N_d, n_img); break;
            }
            rc = check_launch("fdcnn_forward (last layer)");
        } else {
            if (f16 && next_f16) {
                switch (CINP) {
                    case 16: rc = launch_tc_n<0, 2, 16, true>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream); break;
                    case 32: rc = launch_tc_n<0, 2, 32, true>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream); break;
                    default: rc = launch_tc_n<0, 2, 64, true>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream); break;
                }
            } else if (f16) {
                switch (CINP) {
                    case 16: rc = launch_tc_n<0, 0, 16, true>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream); break;
                    case 32: rc = launch_tc_n<0, 0, 32, true>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream); break;
                    default: rc = launch_tc_n<0, 0, 64, true>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream); break;
                }
            } else {
                switch (CINP) {
                    case 16: rc = launch_tc_n<0, 0, 16, false>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream); break;
                    case 32: rc = launch_tc_n<0, 0, 32, false>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream); break;
                    default: rc = launch_tc_n<0, 0, 64, false>(NP, g, smem, in, s_in, Wg, b, wscale, out, s_out, stream); break;
                }
            }
        }
        if (rc) return rc;
    }
    return FD_OK;
}

}  // namespace fdpd

extern "C" int fd_set_cnn_tc_precision(int mode) {
    FD_REQUIRE(mode == 0 || mode == 1, "fd_set_cnn_tc_precision: mode=%d (0 = FP16 split, 1 = TF32 split)", mode);
    fdpd::g_tc_f16 = mode == 0 ? 1 : 0;
    return FD_OK;
}
