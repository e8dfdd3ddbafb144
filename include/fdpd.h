/*
 * fdpd.h — C ABI of libfdpd.so, the B200 (sm_100a) hot path of the FD-CNN DPD
 * massive MU-MIMO-OFDM downlink chain of arXiv 2205.05158 (PAPER.md = P:n).
 *
 * Conventions for every entry point
 * ---------------------------------
 *  - Array pointers are CUDA DEVICE memory owned by the caller (e.g. torch
 *    tensors), contiguous, 16-byte aligned.  Small shape descriptors (chans,
 *    orders) are HOST int arrays.  "complex64" = interleaved {float re, im}
 *    (== torch.complex64 / std::complex<float>).
 *  - Calls are asynchronous on `stream`, never allocate and never synchronise,
 *    except zf_precoder_build (which returns alpha to the host) and the
 *    fd_chain_* runtime (documented there).
 *  - Errors: FD_ERR_ARG for bad sizes / null or misaligned pointers (nothing is
 *    launched); FD_ERR_NUMERIC when a Gram matrix is not positive definite;
 *    FD_ERR_CUDA for launch/runtime errors.  fd_last_error() returns a
 *    thread-local message for the last non-OK status.
 *  - Subcarrier map (reading A7): data subcarrier j = 0..N_d-1 sits at IDFT bin
 *    k_j = (j - N_d/2) mod N_ifft; guards are zero.
 *  - Threads: reentrant; the library's only state is an immutable per-N_ifft
 *    twiddle-table cache (freed by fd_shutdown()).
 */
#ifndef FDPD_H
#define FDPD_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FD_OK = 0,
    FD_ERR_ARG = 2,      /* bad dims / pointer / alignment (SPEC exit code 2) */
    FD_ERR_NUMERIC = 3,  /* Gram matrix not positive definite (SPEC exit code 3) */
    FD_ERR_CUDA = 4      /* CUDA launch / runtime error */
} fd_status;

/* Thread-local message describing the last non-OK status of this thread. */
const char* fd_last_error(void);
/* ABI version (major*100 + minor). */
int fd_version(void);
/* Release cached plan data (twiddle tables).  Safe to call at any time when no
 * call is in flight. */
void fd_shutdown(void);

/* -------------------------------------------------------------------------
 * a1. FD-CNN forward — P:167-177 (structure, Eq. 15), BASELINE residual conv
 * stack (SURVEY §8(c) readings A1-A6).
 *
 * For each (symbol n, UE u): the N_d-vector s_in[n][u][:] is laid out row-major
 * in an S x S image, S = ceil(sqrt(N_d)), tail zero-padded; channels
 * [Re, Im]; n_layers 3x3 "same" zero-padded cross-correlation layers
 * with bias, tanh after every layer but the last; residual output
 * s_out = s_in + (h[0] + j h[1]) on the first N_d pixels.
 *
 *  params    device float, per layer l: W[co][ci][3][3] then b[co], layers
 *            concatenated (sum_l co*ci*9 + co floats).
 *  chans     HOST int[n_layers+1]; chans[0] = chans[n_layers] = 2; each <= 256.
 *  s_in      device complex64 [n_sym][U][N_d].
 *  s_out     device complex64 [n_sym][U][N_d]; must not alias s_in.
 *  workspace device scratch of >= fdcnn_workspace_bytes(...) bytes (may be NULL
 *            when that returns 0).
 *
 * Implementation choice (process-wide, not thread-safe against concurrent calls):
 * fd_set_cnn_path(FD_CNN_TENSOR or FD_CNN_AUTO) runs every layer as a tensor-core
 * implicit GEMM (tcgen05 kind::tf32 with hi/lo operand splitting, FP32-accurate)
 * when all hidden widths are 16, 32 or 64; FD_CNN_SIMT forces the FP32 SIMT kernels.
 * The workspace size depends on the path: query it after choosing.  Returns
 * FD_ERR_ARG for an unknown path.
 * ------------------------------------------------------------------------- */
enum { FD_CNN_AUTO = 0, FD_CNN_SIMT = 1, FD_CNN_TENSOR = 2 };
int fd_set_cnn_path(int path);
/* Operand precision of the tensor-core hidden layers (process-wide): 0 = FP16 split (default:
 * fp16 hi + lo halves with exact power-of-two scales, kind::f16, K = 16 per MMA), 1 = TF32 split
 * (kind::tf32).  Both keep three of the four hi/lo products (22 significant bits per operand),
 * FP32 accumulation.  FD_ERR_ARG for other modes. */
int fd_set_cnn_tc_precision(int mode);
size_t fdcnn_workspace_bytes(const int* chans, int n_layers, long long n_sym, int U, int N_d);
int fdcnn_forward(const float* params, const int* chans, int n_layers,
                  const void* s_in, void* s_out, void* workspace, size_t workspace_bytes,
                  long long n_sym, int U, int N_d, cudaStream_t stream);

/* a1 (paper head) — the paper's own FD-CNN, P:170-177, P:206:
 * per (symbol, UE) the S x S Re/Im image (as above, L_U = 1), n_conv 3x3 "same" kernels
 * with bias, ReLU, flatten in (kernel, row, column) order, fully connected linear layer
 * to 2 N_d outputs with bias: s_out[j] = out[j] + i out[N_d + j].
 *  params  device float: W1[n_conv][2][3][3], b1[n_conv], W2[2 N_d][n_conv S^2], b2[2 N_d]
 *          (any float offset; W2 is copied to an aligned workspace slot each call).
 *  n_conv * S^2 must be a multiple of 4.  workspace >= fdcnn_paper_workspace_bytes(...). */
size_t fdcnn_paper_workspace_bytes(int n_conv, long long n_sym, int U, int N_d);
int fdcnn_paper_forward(const float* params, int n_conv, const void* s_in, void* s_out,
                        void* workspace, size_t workspace_bytes, long long n_sym, int U, int N_d,
                        cudaStream_t stream);

/* -------------------------------------------------------------------------
 * a2. Zero-forcing precoder build — Eq. (6), FD channel P:72 (A9),
 * power normalisation P:84 (reading A12).  Once per channel realisation.
 *
 *   Hfd_j = sum_t H_t exp(-j 2 pi k_j t / N_ifft)          (U x B)
 *   G_j   = Hfd_j Hfd_j^H ;  P0_j = Hfd_j^H G_j^-1          (B x U)
 *   alpha = rho * sqrt(B * N_ifft / sum_j tr(G_j^-1))        (mean TD |x|^2 = rho^2)
 *   P_j   = alpha * P0_j
 * Gram, Cholesky and inverse in fp64; outputs complex64.
 *
 *  h_taps    device complex64 [T][U][B] (full array, every rank).
 *  b0,B_loc  emit antenna rows [b0, b0+B_loc) only (antenna sharding).
 *  h_fd      device complex64 out [U][B_loc][N_d].
 *  P         device complex64 out [B_loc][U][N_d] (alpha folded in).
 *  alpha     HOST float out.  The call synchronises `stream`.
 *  workspace device scratch >= zf_workspace_bytes(N_d) bytes.
 *  Returns FD_ERR_NUMERIC if any G_j is not numerically positive definite.
 * ------------------------------------------------------------------------- */
size_t zf_workspace_bytes(int N_d);
int zf_precoder_build(const void* h_taps, int T, int U, int B, int N_ifft, int N_d, float rho,
                      int b0, int B_loc, void* h_fd, void* P, float* alpha,
                      void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* -------------------------------------------------------------------------
 * a3. Precode — Eq. (1):  X[n][b][j] = sum_u P[b][u][j] * s[n][u][j].
 *  P [B_loc][U][N_d], s [n_sym][U][N_d] -> X [n_sym][B_loc][N_d], complex64.
 *
 *  math (BASELINE configs[2] "TF32 tensor-core precoding variant"):
 *   FD_MATH_FP32     FP32 SIMT complex FMAs, u summed in ascending order (identical to the
 *                    fused chain prologue); U <= 800 (8 U KB of shared memory).
 *   FD_MATH_TF32     tensor cores (tcgen05.mma kind::tf32): per subcarrier the real GEMM
 *                    [Re P | Im P] (K = 2U) x [[Re s, Im s], [-Im s, Re s]]; operands rounded to
 *                    TF32, FP32 accumulation: relative error ~1e-3 (parity bar 2e-3).
 *   FD_MATH_FP32_TC  tensor cores with FP32-accurate split-TF32 operands (x = hi + lo, three
 *                    products A_hi s_hi + A_hi s_lo + A_lo s_hi): parity bar 2e-5 like FP32.
 *  Tensor-core modes need U % 4 == 0, U <= 32, P and X 16-byte aligned; they gather P with
 *  8-byte loads — the fast form is precode_packed on a precode_pack'ed precoder.
 *  FD_ERR_ARG for bad sizes / NULL / misaligned pointers / unknown math.
 * ------------------------------------------------------------------------- */
enum { FD_MATH_FP32 = 0, FD_MATH_TF32 = 1, FD_MATH_FP32_TC = 2 };
int precode(const void* P, const void* s, void* X,
            long long n_sym, int B_loc, int U, int N_d, int math, cudaStream_t stream);
/* The precoder in the tensor cores' per-subcarrier layout, written once per channel
 * realisation (off the hot path, like zf_precoder_build): Ppk [N_d][B_loc][2U] float with
 * row (j, b) = Re P[b][0..U)[j], Im P[b][0..U)[j] (the A operand rows of subcarrier j, read as
 * contiguous 8U-byte rows).  Same bytes as P.  Ppk 16-byte aligned, precode_pack_bytes() bytes. */
size_t precode_pack_bytes(int B_loc, int U, int N_d);
int precode_pack(const void* P, void* Ppk, int B_loc, int U, int N_d, cudaStream_t stream);
/* precode with a packed precoder; math = FD_MATH_TF32 or FD_MATH_FP32_TC (tensor cores). */
int precode_packed(const void* Ppk, const void* s, void* X, long long n_sym, int B_loc, int U, int N_d,
                   int math, cudaStream_t stream);

/* -------------------------------------------------------------------------
 * a4. OFDM IDFT — Eq. (2) P:54-57 (unitary, guards zero):
 *   x[n][b][m] = N^-1/2 sum_j X[n][b][j] exp(+j 2 pi k_j m / N),  N = N_ifft.
 *  X [n_sym][B][N_d] -> x [n_sym][B][N_ifft], complex64.
 *  N_ifft power of two, 16 <= N_ifft <= 16384, N_d even, N_d <= N_ifft.
 * ------------------------------------------------------------------------- */
int ofdm_modulate(const void* X, void* x, long long n_sym, int B, int N_d, int N_ifft,
                  cudaStream_t stream);

/* -------------------------------------------------------------------------
 * a5. GMP PA — Eq. (9) P:113-122 as the PA f_b of Eq. (7) P:89-93,
 * odd orders p <-> |u|^(p-1), l = 0..L, g = 1..M, circular within the symbol
 * (reading A13):
 *   y_m = sum_p sum_l a_{p,l} u_{m-l} |u_{m-l}|^(p-1)
 *       + sum_{p>=3} sum_l sum_g ( b_{p,l,g} u_{m-l} |u_{m-l-g}|^(p-1)
 *                                + c_{p,l,g} u_{m-l} |u_{m-l+g}|^(p-1) )
 *  x    device complex64 [n_sym][B][N_ifft]; y same shape, must not alias x.
 *  coef device complex64 [B][n_coef], flattened a[p][l]; b[p>=3][l][g]; c[p>=3][l][g];
 *       n_coef = Kp(L+1) + 2(Kp-1)(L+1)M.
 *  orders HOST int[n_orders], odd, ascending, orders[0] = 1, n_orders <= 8;
 *  0 <= L <= 15, 0 <= M <= 7 (M = 0: no cross terms), L + 2M < N_ifft.
 * ------------------------------------------------------------------------- */
int gmp_pa(const void* x, const void* coef, void* y, const int* orders, int n_orders,
           int L, int M, long long n_sym, int B, int N_ifft, cudaStream_t stream);

/* Fused a3 -> a4 -> a5 (one CTA per (symbol, antenna); X and x never touch HBM).
 * Numerically equivalent to precode -> ofdm_modulate -> gmp_pa.
 *  P [B_loc][U][N_d], s_tilde [n_sym][U][N_d], coef [B_loc][n_coef] -> y [n_sym][B_loc][N_ifft]. */
int chain_tx(const void* P, const void* s_tilde, const void* coef, void* y,
             const int* orders, int n_orders, int L, int M,
             long long n_sym, int B_loc, int U, int N_d, int N_ifft, cudaStream_t stream);

/* Fused a3 -> a4 -> a5 -> receive DFT (first half of a6): as chain_tx, and the PA
 * output of each (symbol, antenna) is also transformed in the same CTA:
 *   XPA[n][b][j] = N^-1/2 sum_m y[n][b][m] exp(-j 2 pi k_j m / N)      (Eq. 4, A9)
 *  XPA device complex64 out [n_sym][B_loc][N_d]; y (required) is written exactly as
 *  chain_tx writes it (the receive DFT re-reads this CTA's y through L2).  Feed XPA to
 *  ue_combine(_ser). */
int chain_txrx(const void* P, const void* s_tilde, const void* coef, void* y, void* XPA,
               const int* orders, int n_orders, int L, int M,
               long long n_sym, int B_loc, int U, int N_d, int N_ifft, cudaStream_t stream);

/* -------------------------------------------------------------------------
 * Impairments (all off on the hot path, readings A11/A16).
 * Noise is drawn from the counter-based Philox4x32-10 generator (Salmon et al., SC'11)
 * with counter (global index lo, hi, stream, 0) and key (noise_key lo, hi): stream 1 = PA
 * measurement noise at index ((sym0 + n) B_total + b0 + b) N_ifft + m, stream 2 = AWGN
 * at index ((sym0 + n) U + u) N_d + j; Box-Muller on the first two output words.  Any
 * batch / shard therefore reproduces the same noise as the whole run (and the oracle).
 * ------------------------------------------------------------------------- */
typedef struct fd_impair {
    float clip;                    /* PA saturation amplitude, phase kept; 0 = off */
    float pa_noise_std;            /* PA measurement noise std, CN(0, std^2); 0 = off */
    float awgn_n0;                 /* UE noise variance N_0 per data subcarrier; 0 = off */
    float csi_eta;                 /* imperfect-CSI weight eta, zf_precoder_build_ex only */
    unsigned long long noise_key;  /* Philox key */
    long long sym0;                /* global index of the batch's first OFDM symbol */
    int b0, B_total;               /* antenna rows of this call within the full array (0: B_loc) */
} fd_impair;

/* chain_txrx with the PA clip + measurement noise applied to the PA output (y and XPA). */
int chain_txrx_ex(const void* P, const void* s_tilde, const void* coef, void* y, void* XPA,
                  const int* orders, int n_orders, int L, int M,
                  long long n_sym, int B_loc, int U, int N_d, int N_ifft, const fd_impair* imp,
                  cudaStream_t stream);
/* chain_txrx on an already precoded spectrum X [n_sym][B_loc][N_d] (the output of precode):
 * the split precode -> chain_txrx_pre moves the U-fold L2 gather of P_b and s_n out of the
 * fused kernel's prologue into one bandwidth-bound kernel.  imp nullable. */
/* chain_txrx / chain_txrx_ex / _ps / _pre at N_ifft = 16384 (N_d % 4 == 0, GMP shapes of
 * the configured workloads) split each (symbol, antenna) over a two-CTA cluster (one radix-2
 * step across the pair, DSMEM exchange).  mode 0 = auto (default), 1 = never (single-CTA kernel).
 * Process-wide; returns FD_ERR_ARG for other modes. */
int fd_set_chain_split(int mode);
/* GMP implementation of the cluster-split chain (process-wide): 0 = auto (default; = FP32 SIMT,
 * measured faster), 1 = FP32 SIMT, 2 = the tensor cores where they apply — the C4 / C5 shape (orders {1,3,5,7,9},
 * L = 6, M = 3) at N_ifft = 16384: Eq. 9's feature contraction G_l(q) = sum_{d,k} C_l[d][k]
 * e_{q+d}^k as shifted-row MMAs, tf32 hi + bf16 lo envelope powers against tf32 hi + lo
 * coefficients (FP32-accurate, no range scaling).  FD_ERR_ARG for other modes. */
int fd_set_gmp_path(int mode);
/* Test support: fill the shared memory of every SM with `pattern` (uninitialised shared-memory
 * reads of a later kernel then change its output; tests/test_gpu_guard.py). */
int fd_debug_poison_smem(unsigned pattern, cudaStream_t stream);
/* Native-runtime / binding policy: from this many users a step runs precode -> chain_txrx_pre. */
#define FD_SPLIT_PRECODE_MIN_U 16
int chain_txrx_pre(const void* X, const void* coef, void* y, void* XPA, const int* orders, int n_orders,
                   int L, int M, long long n_sym, int B_loc, int N_d, int N_ifft, const fd_impair* imp,
                   cudaStream_t stream);
/* zf_precoder_build with imperfect CSI: the precoder is built from
 * H_est = sqrt(1 - eta) H + sqrt(eta) H_err while h_fd (the channel the UEs see) is
 * built from H.  h_err device complex64 [T][U][B]; eta in [0, 1]. */
int zf_precoder_build_ex(const void* h_taps, const void* h_err, float eta, int T, int U, int B, int N_ifft,
                         int N_d, float rho, int b0, int B_loc, void* h_fd, void* P, float* alpha,
                         void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* -------------------------------------------------------------------------
 * Per-symbol channel redraw ("block-constant with a coherence time of
 * one OFDM symbol"): one channel realisation per symbol, so the ZF build joins the hot
 * path.  Shapes gain a leading per-realisation dimension n_ch (= n_sym of the batch).
 *
 * zf_precoder_build_batched: n_ch independent zf_precoder_build's (one alpha each, A12),
 *  fully asynchronous.  h_taps [n_ch][T][U][B]; h_fd out [n_ch][U][B_loc][N_d]; P out
 *  [n_ch][B_loc][U][N_d]; alpha DEVICE float out [n_ch]; status DEVICE int (nullable) set
 *  non-zero when some Gram matrix is not positive definite; workspace >=
 *  zf_batched_workspace_bytes(n_ch, N_d); n_ch <= 65535.
 * chain_txrx_ps: chain_txrx with symbol n of the batch precoded by P_all[n] ([n_sym][B_loc][U][N_d]).
 * ue_combine_ser_ps: ue_combine_ser with h_fd_all[n] ([n_sym][U][B_loc][N_d]) and alpha_dev[n].
 * ------------------------------------------------------------------------- */
size_t zf_batched_workspace_bytes(int n_ch, int N_d);
int zf_precoder_build_batched(const void* h_taps, int n_ch, int T, int U, int B, int N_ifft, int N_d, float rho,
                              int b0, int B_loc, void* h_fd, void* P, float* alpha, int* status,
                              void* workspace, size_t workspace_bytes, cudaStream_t stream);
int chain_txrx_ps(const void* P_all, const void* s_tilde, const void* coef, void* y, void* XPA,
                  const int* orders, int n_orders, int L, int M,
                  long long n_sym, int B_loc, int U, int N_d, int N_ifft, const fd_impair* imp,
                  cudaStream_t stream);
int ue_combine_ser_ps(const void* XPA, const void* h_fd_all, void* yhat, const float* alpha_dev,
                      const uint16_t* tx_idx, int M_qam, uint16_t* dec, long long* counts, long long n_sym,
                      int B_loc, int U, int N_d, float boundary_eps, const fd_impair* imp, cudaStream_t stream);

/* -------------------------------------------------------------------------
 * a6. Evaluation — Eqs. (4)-(5) P:67-77 (noiseless, reading A11), SER P:351.
 *
 * ue_receive: XPA[n][b][j] = N^-1/2 sum_m y[n][b][m] exp(-j 2 pi k_j m / N);
 *             yhat[n][u][j] (+)= sum_{b<B_loc} h_fd[u][b][j] * XPA[n][b][j].
 *  y [n_sym][B_loc][N_ifft], h_fd [U][B_loc][N_d] -> yhat [n_sym][U][N_d], complex64.
 *  accumulate != 0 adds into yhat (antenna shards / chunks); 0 overwrites.
 *  workspace >= ue_receive_workspace_bytes(...) bytes (holds XPA).
 *
 * ue_slice_ser: z = yhat / alpha (genie alpha, A17); per-axis nearest odd level
 *  d = clip(2 floor(v/2) + 1, -(m-1), m-1), v = Re|Im z / c, c = (2(M_qam-1)/3)^-1/2;
 *  dec = (d_I + m-1)/2 + m (d_Q + m-1)/2 ; counts[0] += #(dec != tx_idx),
 *  counts[1] += n_sym*U*N_d, counts[2] += #samples within boundary_eps of an
 *  interior boundary.  tx_idx uint16 [n_sym][U][N_d]; dec nullable; counts device
 *  int64[3] (accumulated: the caller zeroes it).
 * ------------------------------------------------------------------------- */
size_t ue_receive_workspace_bytes(long long n_sym, int B_loc, int N_d);
int ue_receive(const void* y, const void* h_fd, void* yhat, void* workspace, size_t workspace_bytes,
               long long n_sym, int B_loc, int U, int N_d, int N_ifft, int accumulate,
               cudaStream_t stream);
int ue_slice_ser(const void* yhat, float alpha, const uint16_t* tx_idx, int M_qam,
                 uint16_t* dec, long long* counts, long long n_sym, int U, int N_d,
                 float boundary_eps, cudaStream_t stream);
/* Second half of ue_receive on an XPA produced by chain_txrx (or ue_receive's FFT):
 *   yhat[n][u][j] (+)= sum_b h_fd[u][b][j] XPA[n][b][j];  n_sym <= 65535 per call. */
int ue_combine(const void* XPA, const void* h_fd, void* yhat, long long n_sym, int B_loc, int U, int N_d,
               int accumulate, cudaStream_t stream);
/* Channel-sum implementation (process-wide): 0 = auto (default) = the FP32 SIMT kernels
 * (measured faster at C4 / C5); 1 = FP32 SIMT; 2 = tensor cores where they apply — 9 <= U <= 32,
 * no AWGN, one channel realisation, 16-byte aligned yhat (tcgen05 kind::tf32, per-subcarrier
 * real GEMM with K = 2 B_loc, FP32-accurate hi/lo split on both operands, four products),
 * else SIMT.  FD_ERR_ARG for other modes. */
int fd_set_combine_path(int mode);
/* Mode A (antenna sharding, BASELINE configs[4]): the channel sum fused with its
 * exchange.  Rank `rank` of `world` holds antenna rows of XPA [n_sym][B_loc][N_d] and h_fd
 * [U][B_loc][N_d] for the WORLD batch of n_sym = world * nm symbols (symbol n belongs to rank
 * n / nm).  Instead of a local partial y_hat that a reduce-scatter then moves, every partial
 * sum sum_{b local} h_fd[u][b][j] XPA[n][b][j] (Eq. 5 over this rank's antennas) is
 * stored by the kernel straight into slot `rank` of the owner's receive buffer:
 *   peer_recv[n / nm][rank][n % nm][u][j]      (each buffer [world][nm][U][N_d] complex64)
 * peer_recv: HOST array of `world` DEVICE pointers, peer-mapped (NVLink P2P / CUDA IPC) or, for
 * r = rank, local; the stores overlap the kernel's math tile by tile.  9 <= U <= 32, N_d even,
 * XPA / h_fd 16-byte aligned (FD_ERR_ARG otherwise: use ue_combine + a reduce-scatter).
 * The caller orders "all ranks' ue_combine_peer done" before ue_reduce_ser (a stream-ordered
 * barrier: no kernel of this library waits on another GPU). */
int ue_combine_peer(const void* XPA, const void* h_fd, void* const* peer_recv, int world, int rank, long long n_sym,
                    int B_loc, int U, int N_d, cudaStream_t stream);
/* Owner side: yhat[n][u][j] = sum_{r < world} recv[r][n][u][j] in rank order (bit-reproducible),
 * then, when tx_idx is not NULL, slicing + SER counters like ue_slice_ser (dec nullable).
 * recv [world][n_sym][U][N_d], yhat [n_sym][U][N_d] (n_sym = this rank's symbols). */
int ue_reduce_ser(const void* recv, int world, void* yhat, float alpha, const uint16_t* tx_idx, int M_qam,
                  uint16_t* dec, long long* counts, long long n_sym, int U, int N_d, float boundary_eps,
                  cudaStream_t stream);
/* ue_combine (accumulate = 0) fused with ue_slice_ser. */
int ue_combine_ser(const void* XPA, const void* h_fd, void* yhat, float alpha, const uint16_t* tx_idx, int M_qam,
                   uint16_t* dec, long long* counts, long long n_sym, int B_loc, int U, int N_d,
                   float boundary_eps, cudaStream_t stream);
/* ue_combine_ser with AWGN (imp->awgn_n0) added to yhat before slicing. */
int ue_combine_ser_ex(const void* XPA, const void* h_fd, void* yhat, float alpha, const uint16_t* tx_idx, int M_qam,
                      uint16_t* dec, long long* counts, long long n_sym, int B_loc, int U, int N_d,
                      float boundary_eps, const fd_impair* imp, cudaStream_t stream);
/* ue_receive (accumulate = 0) then ue_slice_ser, single GPU. */
int ue_receive_ser(const void* y, const void* h_fd, void* yhat, void* workspace, size_t workspace_bytes,
                   float alpha, const uint16_t* tx_idx, int M_qam, uint16_t* dec, long long* counts,
                   long long n_sym, int B_loc, int U, int N_d, int N_ifft, float boundary_eps,
                   cudaStream_t stream);

/* -------------------------------------------------------------------------
 * Native chain runtime: a plan owning the device-resident state of one channel
 * realisation and running the whole hot path per batch of OFDM symbols
 * (a1 -> a3..a5 -> a6 = fdcnn_forward -> chain_txrx -> ue_combine_ser).
 * Unlike the calls above, the plan allocates (cudaMalloc at create) and the host
 * variant synchronises; everything else follows the conventions above.
 * ------------------------------------------------------------------------- */
#define FD_CHAIN_MAX_LAYERS 8
typedef struct fd_chain_desc {
    int U, B, T, N_d, N_ifft, M_qam;
    int n_layers, chans[FD_CHAIN_MAX_LAYERS + 1];   /* FD-CNN (fdcnn_forward) */
    int n_orders, orders[8], L, M;                   /* GMP PA (gmp_pa) */
    float rho;                                       /* TD RMS target for alpha (A12) */
    float boundary_eps;                              /* SER near-boundary band (1e-4) */
    int head;                                        /* 0: residual stack (fdcnn_forward), 1: paper head */
    int n_conv;                                      /* paper head: N^Conv (fdcnn_paper_forward) */
} fd_chain_desc;
typedef struct fd_chain fd_chain;

/* Copies the HOST arrays h_taps [T][U][B] complex64, coef [B][n_coef] complex64 and
 * params (float) to the device, builds the ZF precoder (zf_precoder_build; synchronises)
 * and reserves buffers for batches of up to max_batch symbols.  A step is fdcnn_forward ->
 * chain_txrx (U < FD_SPLIT_PRECODE_MIN_U) or precode -> chain_txrx_pre (the precode on the
 * tensor cores, FD_MATH_FP32_TC on a precode_pack'ed P, where U % 4 == 0 and U <= 32; else
 * FD_MATH_FP32) -> ue_combine_ser. */
int fd_chain_create(fd_chain** out, const fd_chain_desc* desc, const void* h_taps, const void* coef,
                    const float* params, long long max_batch, cudaStream_t stream);
float fd_chain_alpha(const fd_chain* chain);
void fd_chain_destroy(fd_chain* chain);
/* Device buffers: s [n_sym][U][N_d] complex64, tx_idx uint16 same shape, counts device
 * int64[3] accumulated (caller zeroes); yhat optional device [n_sym][U][N_d] output
 * (NULL: plan-owned).  Asynchronous. */
int fd_chain_run_device(fd_chain* chain, const void* s, const uint16_t* tx_idx, long long n_sym,
                        long long* counts, void* yhat, cudaStream_t stream);
/* HOST buffers (pinned for async copies): copies s and tx_idx in, runs the step, copies
 * the three SER counters (errors, total, near) back and synchronises `stream`. */
int fd_chain_run_host(fd_chain* chain, const void* s_host, const uint16_t* tx_idx_host, long long n_sym,
                      long long* counts_host, cudaStream_t stream);

/* HOST QAM index stream (pinned): the transmitter's symbol mapping runs on the device
 * (qam_map), so only the uint16 indices cross PCIe (2 B instead of 10 B per data
 * subcarrier); otherwise identical to fd_chain_run_host. */
int fd_chain_run_host_qam(fd_chain* chain, const uint16_t* tx_idx_host, long long n_sym, long long* counts_host,
                          cudaStream_t stream);

/* a0 QAM mapping (reading A19; "data symbols"): s = (l_I + j l_Q) c_M with
 * m = sqrt(M_qam), I = idx mod m, Q = idx div m, l = 2 I - (m - 1), c_M = (2 (M_qam - 1) / 3)^-1/2
 * evaluated in fp64 and rounded to complex64 (E|s|^2 = 1).  idx device uint16 [count],
 * s device complex64 [count].  FD_ERR_ARG if M_qam is not a square >= 4 or a pointer is NULL. */
int qam_map(const uint16_t* idx, void* s, long long count, int M_qam, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FDPD_H */
