// common.cu — status handling and the twiddle-table plan cache.
#include "fft.cuh"

#include <mutex>
#include <map>

namespace fdpd {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
}

int fail_arg(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return FD_ERR_ARG;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return FD_ERR_CUDA;
    }
    return FD_OK;
}

__global__ void k_twiddles(float2* w, int N) {
    int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m < N) {
        double s, c;
        sincospi(-2.0 * (double)m / (double)N, &s, &c);   // exp(-2 pi i m / N) in fp64
        w[m] = make_float2((float)c, (float)s);
    }
}

// per-pass radix-16 tables behind the N-entry table (fft.cuh tw_pass_off)
__global__ void k_twiddles_pass(float2* w, int N) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    int off = N;
    for (long long ns = 16; ns * 16 <= N; ns *= 16) {
        const int len = 15 * (int)ns;
        if (e < len) {
            const int r = e / (int)ns + 1, k = e % (int)ns;
            double s, c;
            sincospi(-2.0 * (double)(r * k) / (double)(16 * ns), &s, &c);
            w[off + e] = make_float2((float)c, (float)s);
            return;
        }
        e -= len;
        off += len;
    }
}

namespace {
struct TwKey { int dev; int N; bool operator<(const TwKey& o) const { return dev != o.dev ? dev < o.dev : N < o.N; } };
std::mutex g_mu;
std::map<TwKey, float2*> g_tw;
}

const float2* twiddle_table(int N, cudaStream_t stream) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_tw.find({dev, N});
    if (it != g_tw.end()) return it->second;
    float2* w = nullptr;
    const int len = tw_table_len(N);
    if (cudaMalloc(&w, sizeof(float2) * (size_t)len) != cudaSuccess) return nullptr;
    k_twiddles<<<(N + 255) / 256, 256, 0, stream>>>(w, N);
    if (len > N) k_twiddles_pass<<<(len - N + 255) / 256, 256, 0, stream>>>(w, N);
    // the table is plan data: make it visible to every stream before first use
    if (cudaStreamSynchronize(stream) != cudaSuccess) { cudaFree(w); return nullptr; }
    g_tw[{dev, N}] = w;
    return w;
}

// Test support: fill the whole shared memory of every SM with a pattern (uninitialised-read
// detection: a kernel whose output changes after this ran reads shared memory it never wrote).
__global__ void k_poison_smem(uint32_t pattern, int words) {
    extern __shared__ uint32_t sw[];
    for (int i = threadIdx.x; i < words; i += blockDim.x) sw[i] = pattern;
}

}  // namespace fdpd

extern "C" {

int fd_debug_poison_smem(unsigned pattern, cudaStream_t stream) {
    const int bytes = 227 * 1024;
    cudaFuncSetAttribute(fdpd::k_poison_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    fdpd::k_poison_smem<<<4 * 148, 1024, bytes, stream>>>(pattern, bytes / 4);
    return fdpd::check_launch("fd_debug_poison_smem");
}

const char* fd_last_error(void) { return fdpd::g_err.c_str(); }

int fd_version(void) { return 100; }

void fd_shutdown(void) {
    std::lock_guard<std::mutex> lk(fdpd::g_mu);
    for (auto& kv : fdpd::g_tw) cudaFree(kv.second);
    fdpd::g_tw.clear();
}

}  // extern "C"
