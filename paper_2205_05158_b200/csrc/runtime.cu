// runtime.cu — native chain runtime: a device-resident plan for one channel
// realisation (CNN weights, PA coefficients, ZF precoder, workspaces) and the step
// entry points that run the whole hot path from host or device buffers.
//
// Step = fdcnn_forward -> chain_txrx -> ue_combine_ser (include/fdpd.h); the host
// variant adds the host->device copy of the step's inputs and the device->host copy
// of the SER counters on the same stream (cudaMemcpyAsync, one per buffer).
#include "common.cuh"

#include <new>
#include <vector>

struct fd_chain {
    fd_chain_desc d;
    int n_coef = 0, n_params = 0, N_d_pad = 0;
    long long cap = 0;
    float alpha = 0.f;
    // device buffers owned by the plan
    float2 *h_taps = nullptr, *coef = nullptr, *h_fd = nullptr, *P = nullptr;
    float* params = nullptr;
    float2 *s = nullptr, *s_tilde = nullptr, *y = nullptr, *XPA = nullptr, *yhat = nullptr;
    float2* X = nullptr;   // precoded spectrum [cap][B][N_d] when U >= FD_SPLIT_PRECODE_MIN_U
    float* Ppk = nullptr;  // precode_pack'ed P for the tensor-core precode (split path, U % 4 == 0, U <= 32)
    uint16_t* idx = nullptr;
    long long* counts = nullptr;
    void* ws_cnn = nullptr;
    size_t ws_cnn_bytes = 0;
    void* ws_zf = nullptr;
    // host-input pipelining: a copy stream and per-chunk events (fd_chain_run_host)
    cudaStream_t copy_stream = nullptr;
    static constexpr int kChunks = 4;
    cudaEvent_t ev_in[kChunks] = {}, ev_free = nullptr;
};

namespace fdpd {
__global__ void k_qam_map(const uint16_t* __restrict__ idx, float2* __restrict__ s, long long count, int m,
                          double scale) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        const int v = idx[i];
        const int I = v % m, Q = v / m;
        s[i] = make_float2((float)((double)(2 * I - (m - 1)) * scale), (float)((double)(2 * Q - (m - 1)) * scale));
    }
}
static int launch_qam_map(const uint16_t* idx, float2* s, long long count, int M_qam, cudaStream_t st) {
    int m = 1;
    while (m * m < M_qam) ++m;
    FD_REQUIRE(m * m == M_qam && M_qam >= 4 && M_qam <= 65536, "qam_map: M_qam=%d must be a square >= 4", M_qam);
    if (count == 0) return FD_OK;
    const double scale = std::sqrt(3.0 / (2.0 * (M_qam - 1)));
    const int blocks = (int)std::min<long long>((count + 255) / 256, 148LL * 16);
    k_qam_map<<<blocks, 256, 0, st>>>(idx, s, count, m, scale);
    return check_launch("qam_map");
}
}  // namespace fdpd

namespace {

template <typename T>
int dalloc(T** p, size_t n) {
    if (n == 0) n = 1;
    if (cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)) != cudaSuccess) {
        fdpd::set_error("fd_chain: cudaMalloc of %zu bytes failed", n * sizeof(T));
        return FD_ERR_CUDA;
    }
    return FD_OK;
}

void release(fd_chain* c) {
    if (!c) return;
    void* ptrs[] = {c->h_taps, c->coef, c->h_fd, c->P, c->params, c->s, c->s_tilde, c->y,
                    c->XPA, c->yhat, c->idx, c->counts, c->ws_cnn, c->ws_zf, c->X, c->Ppk};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (cudaEvent_t e : c->ev_in)
        if (e) cudaEventDestroy(e);
    if (c->ev_free) cudaEventDestroy(c->ev_free);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    delete c;
}

int ensure_batch(fd_chain* c, long long n) {
    if (n <= c->cap) return FD_OK;
    const fd_chain_desc& d = c->d;
    void* old[] = {c->s, c->s_tilde, c->y, c->XPA, c->yhat, c->idx, c->ws_cnn, c->X};
    for (void* p : old)
        if (p) cudaFree(p);
    c->s = c->s_tilde = c->y = c->XPA = c->yhat = c->X = nullptr;
    c->idx = nullptr;
    c->ws_cnn = nullptr;
    int rc;
    if ((rc = dalloc(&c->s, (size_t)n * d.U * d.N_d))) return rc;
    if ((rc = dalloc(&c->s_tilde, (size_t)n * d.U * d.N_d))) return rc;
    if ((rc = dalloc(&c->y, (size_t)n * d.B * d.N_ifft))) return rc;
    if ((rc = dalloc(&c->XPA, (size_t)n * d.B * d.N_d))) return rc;
    if ((rc = dalloc(&c->yhat, (size_t)n * d.U * d.N_d))) return rc;
    if (d.U >= FD_SPLIT_PRECODE_MIN_U && (rc = dalloc(&c->X, (size_t)n * d.B * d.N_d))) return rc;
    if ((rc = dalloc(&c->idx, (size_t)n * d.U * d.N_d))) return rc;
    c->ws_cnn_bytes = d.head == 1 ? fdcnn_paper_workspace_bytes(d.n_conv, n, d.U, d.N_d)
                                  : fdcnn_workspace_bytes(d.chans, d.n_layers, n, d.U, d.N_d);
    if (c->ws_cnn_bytes && (rc = dalloc(reinterpret_cast<char**>(&c->ws_cnn), c->ws_cnn_bytes))) return rc;
    c->cap = n;
    return FD_OK;
}

// The step on symbols [s0, s0 + n) of the plan's buffers (s, tx_idx already offset).
int run_chunk(fd_chain* c, const void* s, const uint16_t* tx_idx, long long s0, long long n, long long* counts,
              void* yhat, cudaStream_t stream) {
    if (n == 0) return FD_OK;
    const fd_chain_desc& d = c->d;
    const size_t pu = (size_t)d.U * d.N_d, pb = (size_t)d.B * d.N_d, py = (size_t)d.B * d.N_ifft;
    float2* st = c->s_tilde + s0 * pu;
    int rc = d.head == 1 ? fdcnn_paper_forward(c->params, d.n_conv, s, st, c->ws_cnn, c->ws_cnn_bytes, n, d.U, d.N_d,
                                               stream)
                         : fdcnn_forward(c->params, d.chans, d.n_layers, s, st, c->ws_cnn, c->ws_cnn_bytes, n, d.U,
                                         d.N_d, stream);
    if (rc) return rc;
    float2* XPA = c->XPA + s0 * pb;
    if (c->X) {
        // many users: tiled precode kernel, then the chain on the precoded spectrum
        float2* X = c->X + s0 * pb;
        rc = c->Ppk ? precode_packed(c->Ppk, st, X, n, d.B, d.U, d.N_d, FD_MATH_FP32_TC, stream)
                    : precode(c->P, st, X, n, d.B, d.U, d.N_d, FD_MATH_FP32, stream);
        if (rc) return rc;
        rc = chain_txrx_pre(X, c->coef, c->y + s0 * py, XPA, d.orders, d.n_orders, d.L, d.M, n, d.B, d.N_d, d.N_ifft,
                            nullptr, stream);
    } else {
        rc = chain_txrx(c->P, st, c->coef, c->y + s0 * py, XPA, d.orders, d.n_orders, d.L, d.M, n, d.B, d.U, d.N_d,
                        d.N_ifft, stream);
    }
    if (rc) return rc;
    return ue_combine_ser(XPA, c->h_fd, yhat ? yhat : (void*)(c->yhat + s0 * pu), c->alpha, tx_idx, d.M_qam, nullptr,
                          counts, n, d.B, d.U, d.N_d, d.boundary_eps, stream);
}

}  // namespace

extern "C" {

int fd_chain_create(fd_chain** out, const fd_chain_desc* desc, const void* h_taps, const void* coef,
                    const float* params, long long max_batch, cudaStream_t stream) {
    FD_REQUIRE(out && desc && h_taps && coef && params, "fd_chain_create: NULL pointer");
    *out = nullptr;
    const fd_chain_desc& d = *desc;
    FD_REQUIRE(d.U >= 1 && d.B >= d.U && d.T >= 1 && d.N_d >= 2 && d.N_ifft >= d.N_d, "fd_chain_create: bad sizes");
    FD_REQUIRE(d.n_layers >= 1 && d.n_layers <= FD_CHAIN_MAX_LAYERS, "fd_chain_create: n_layers");
    FD_REQUIRE(d.n_orders >= 1 && d.n_orders <= 8, "fd_chain_create: n_orders");
    FD_REQUIRE(max_batch >= 0, "fd_chain_create: max_batch < 0");
    // ue_combine_ser takes at most 65535 symbols per call and a step runs the whole batch
    FD_REQUIRE(max_batch <= 65535, "fd_chain_create: max_batch=%lld exceeds 65535 symbols per step", max_batch);
    fd_chain* c = new (std::nothrow) fd_chain();
    if (!c) return fdpd::fail_arg("fd_chain_create: out of host memory");
    c->d = d;
    c->n_coef = d.n_orders * (d.L + 1) + 2 * (d.n_orders - 1) * (d.L + 1) * d.M;
    if (d.head == 1) {
        FD_REQUIRE(d.n_conv >= 1, "fd_chain_create: n_conv");
        int S = 1;
        while (S * S < d.N_d) ++S;
        c->n_params = d.n_conv * 19 + 2 * d.N_d * d.n_conv * S * S + 2 * d.N_d;
    } else {
        for (int l = 0; l < d.n_layers; ++l) c->n_params += d.chans[l + 1] * d.chans[l] * 9 + d.chans[l + 1];
    }
    int rc;
    const cudaMemcpyKind h2d = cudaMemcpyHostToDevice;
#define FD_TRY(x)              \
    if ((rc = (x)) != FD_OK) { \
        release(c);            \
        return rc;             \
    }
    FD_TRY(dalloc(&c->h_taps, (size_t)d.T * d.U * d.B));
    FD_TRY(dalloc(&c->coef, (size_t)d.B * c->n_coef));
    FD_TRY(dalloc(&c->params, (size_t)c->n_params));
    FD_TRY(dalloc(&c->h_fd, (size_t)d.U * d.B * d.N_d));
    FD_TRY(dalloc(&c->P, (size_t)d.B * d.U * d.N_d));
    FD_TRY(dalloc(&c->counts, 3));
    FD_TRY(dalloc(reinterpret_cast<char**>(&c->ws_zf), zf_workspace_bytes(d.N_d)));
    if (cudaMemcpyAsync(c->h_taps, h_taps, sizeof(float2) * (size_t)d.T * d.U * d.B, h2d, stream) != cudaSuccess ||
        cudaMemcpyAsync(c->coef, coef, sizeof(float2) * (size_t)d.B * c->n_coef, h2d, stream) != cudaSuccess ||
        cudaMemcpyAsync(c->params, params, sizeof(float) * (size_t)c->n_params, h2d, stream) != cudaSuccess) {
        release(c);
        return fdpd::check_launch("fd_chain_create (upload)");
    }
    // a2: ZF precoder, once per channel realisation (synchronises)
    FD_TRY(zf_precoder_build(c->h_taps, d.T, d.U, d.B, d.N_ifft, d.N_d, d.rho, 0, d.B, c->h_fd, c->P, &c->alpha,
                             c->ws_zf, zf_workspace_bytes(d.N_d), stream));
    // split path: the FP32-accurate tensor-core precode where it applies (same policy as the
    // binding's auto_precode_math), on the precoder packed once per channel realisation
    if (d.U >= FD_SPLIT_PRECODE_MIN_U && d.U % 4 == 0 && d.U <= 32) {
        FD_TRY(dalloc(&c->Ppk, precode_pack_bytes(d.B, d.U, d.N_d) / sizeof(float)));
        FD_TRY(precode_pack(c->P, c->Ppk, d.B, d.U, d.N_d, stream));
    }
    FD_TRY(ensure_batch(c, max_batch));
#undef FD_TRY
    bool ok = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&c->ev_free, cudaEventDisableTiming) == cudaSuccess;
    for (int k = 0; ok && k < fd_chain::kChunks; ++k)
        ok = cudaEventCreateWithFlags(&c->ev_in[k], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        release(c);
        return fdpd::check_launch("fd_chain_create (streams)");
    }
    *out = c;
    return FD_OK;
}

float fd_chain_alpha(const fd_chain* c) { return c ? c->alpha : 0.f; }

void fd_chain_destroy(fd_chain* c) { release(c); }

int fd_chain_run_device(fd_chain* c, const void* s, const uint16_t* tx_idx, long long n_sym, long long* counts,
                        void* yhat, cudaStream_t stream) {
    FD_REQUIRE(c && s && tx_idx && counts, "fd_chain_run_device: NULL pointer");
    FD_REQUIRE(n_sym >= 0 && n_sym <= c->cap, "fd_chain_run_device: n_sym=%lld exceeds the plan's batch %lld", n_sym,
               c->cap);
    return run_chunk(c, s, tx_idx, 0, n_sym, counts, yhat, stream);
}

int fd_chain_run_host(fd_chain* c, const void* s_host, const uint16_t* idx_host, long long n_sym,
                      long long* counts_host, cudaStream_t stream) {
    FD_REQUIRE(c && s_host && idx_host && counts_host, "fd_chain_run_host: NULL pointer");
    FD_REQUIRE(n_sym >= 0 && n_sym <= c->cap, "fd_chain_run_host: n_sym=%lld exceeds the plan's batch %lld", n_sym,
               c->cap);
    const fd_chain_desc& d = c->d;
    // Pipelined over up to kChunks symbol chunks: chunk k's host->device copy (copy stream)
    // overlaps chunk k-1's compute (stream); only the first chunk's copy is exposed.
    const long long per = (size_t)d.U * d.N_d;
    const int chunks = (int)std::max(1LL, std::min<long long>(fd_chain::kChunks, n_sym / 64));
    if (cudaMemsetAsync(c->counts, 0, 3 * sizeof(long long), stream) != cudaSuccess ||
        cudaEventRecord(c->ev_free, stream) != cudaSuccess ||                   // previous step done with c->s
        cudaStreamWaitEvent(c->copy_stream, c->ev_free, 0) != cudaSuccess)
        return fdpd::check_launch("fd_chain_run_host (order)");
    for (int k = 0; k < chunks; ++k) {
        const long long s0 = n_sym * k / chunks, s1 = n_sym * (k + 1) / chunks;
        const size_t off = (size_t)s0 * per, cnt = (size_t)(s1 - s0) * per;
        if (cudaMemcpyAsync(c->s + off, (const float2*)s_host + off, sizeof(float2) * cnt, cudaMemcpyHostToDevice,
                            c->copy_stream) != cudaSuccess ||
            cudaMemcpyAsync(c->idx + off, idx_host + off, sizeof(uint16_t) * cnt, cudaMemcpyHostToDevice,
                            c->copy_stream) != cudaSuccess ||
            cudaEventRecord(c->ev_in[k], c->copy_stream) != cudaSuccess)
            return fdpd::check_launch("fd_chain_run_host (h2d)");
    }
    for (int k = 0; k < chunks; ++k) {
        const long long s0 = n_sym * k / chunks, s1 = n_sym * (k + 1) / chunks;
        if (cudaStreamWaitEvent(stream, c->ev_in[k], 0) != cudaSuccess) return fdpd::check_launch("fd_chain (wait)");
        const int rc = run_chunk(c, c->s + (size_t)s0 * per, c->idx + (size_t)s0 * per, s0, s1 - s0, c->counts,
                                 nullptr, stream);
        if (rc) return rc;
    }
    if (cudaMemcpyAsync(counts_host, c->counts, 3 * sizeof(long long), cudaMemcpyDeviceToHost, stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
        return fdpd::check_launch("fd_chain_run_host (d2h)");
    return FD_OK;
}

int qam_map(const uint16_t* idx, void* s, long long count, int M_qam, cudaStream_t stream) {
    FD_REQUIRE(count >= 0, "qam_map: count < 0");
    FD_REQUIRE(count == 0 || (idx && s), "qam_map: NULL pointer");
    return fdpd::launch_qam_map(idx, (float2*)s, count, M_qam, stream);
}

int fd_chain_run_host_qam(fd_chain* c, const uint16_t* idx_host, long long n_sym, long long* counts_host,
                          cudaStream_t stream) {
    FD_REQUIRE(c && idx_host && counts_host, "fd_chain_run_host_qam: NULL pointer");
    FD_REQUIRE(n_sym >= 0 && n_sym <= c->cap, "fd_chain_run_host_qam: n_sym=%lld exceeds the plan's batch %lld",
               n_sym, c->cap);
    const fd_chain_desc& d = c->d;
    // as fd_chain_run_host, but only the indices cross PCIe (5x fewer bytes), so two chunks
    // suffice to hide the copy and the step keeps full-size launches; each chunk's symbols are
    // mapped on the compute stream after its copy lands
    const long long per = (size_t)d.U * d.N_d;
    const int chunks = (int)std::max(1LL, std::min<long long>(2, n_sym / 64));
    if (cudaMemsetAsync(c->counts, 0, 3 * sizeof(long long), stream) != cudaSuccess ||
        cudaEventRecord(c->ev_free, stream) != cudaSuccess ||
        cudaStreamWaitEvent(c->copy_stream, c->ev_free, 0) != cudaSuccess)
        return fdpd::check_launch("fd_chain_run_host_qam (order)");
    for (int k = 0; k < chunks; ++k) {
        const long long s0 = n_sym * k / chunks, s1 = n_sym * (k + 1) / chunks;
        const size_t off = (size_t)s0 * per, cnt = (size_t)(s1 - s0) * per;
        if (cudaMemcpyAsync(c->idx + off, idx_host + off, sizeof(uint16_t) * cnt, cudaMemcpyHostToDevice,
                            c->copy_stream) != cudaSuccess ||
            cudaEventRecord(c->ev_in[k], c->copy_stream) != cudaSuccess)
            return fdpd::check_launch("fd_chain_run_host_qam (h2d)");
    }
    for (int k = 0; k < chunks; ++k) {
        const long long s0 = n_sym * k / chunks, s1 = n_sym * (k + 1) / chunks;
        const size_t off = (size_t)s0 * per;
        if (cudaStreamWaitEvent(stream, c->ev_in[k], 0) != cudaSuccess)
            return fdpd::check_launch("fd_chain_run_host_qam (wait)");
        int rc = fdpd::launch_qam_map(c->idx + off, c->s + off, (s1 - s0) * per, d.M_qam, stream);
        if (rc) return rc;
        rc = run_chunk(c, c->s + off, c->idx + off, s0, s1 - s0, c->counts, nullptr, stream);
        if (rc) return rc;
    }
    if (cudaMemcpyAsync(counts_host, c->counts, 3 * sizeof(long long), cudaMemcpyDeviceToHost, stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
        return fdpd::check_launch("fd_chain_run_host_qam (d2h)");
    return FD_OK;
}

}  // extern "C"
