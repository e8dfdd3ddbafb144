// fdcnn.cu — FD-CNN DPD forward (Eq. 15; BASELINE residual conv stack,
// readings A1-A6): per (symbol, UE) an S x S two-channel image, 3x3 "same" convs
// with tanh, residual output.
//
// Layer kernel: shared-memory-tiled direct convolution.  A CTA owns (image, tile of
// TR rows, group of COG output channels); input channels are staged 8 at a time
// with a one-pixel zero halo, weights are staged transposed W[ci][tap][co] so one
// 128-bit broadcast load feeds 4 output channels x 4 pixels of FMAs.  The first
// layer reads the complex symbols directly (Re/Im channels, row-major, tail zero
// pad); the last layer writes the residual s_out = s_in + out on the first N_d
// pixels.  tanhf is the accurate libdevice routine (no fast-math).
#include "common.cuh"

namespace fdpd {

constexpr int CNN_THREADS = 256;
constexpr int CI_T = 8;     // input channels staged per chunk
constexpr int PX = 4;       // output pixels per thread (along a row)

struct ConvGeom {
    int Cin, Cout, S, N_d, TR, COG, n_rt, n_cg, pxb;
};

// in_mode: 0 = fp32 activations [img][Cin][S][S], 1 = complex symbols [img][N_d] (Cin = 2)
// out_mode: 0 = tanh activations [img][Cout][S][S], 1 = residual complex s_out (Cout = 2)
template <int CO_T, int IN_MODE, int OUT_MODE>
__global__ void __launch_bounds__(CNN_THREADS)
    k_conv(const float* __restrict__ in, const float2* __restrict__ s_in, const float* __restrict__ W,
           const float* __restrict__ bias, float* __restrict__ out, float2* __restrict__ s_out, ConvGeom g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int S = g.S, SP = S + 2, TRP = g.TR + 2;
    float* sin_ = reinterpret_cast<float*>(smem_raw);                 // [CI_T][TRP][SP]
    float* sw = sin_ + CI_T * TRP * SP;                                // [CI_T][9][COG]
    sw = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sw) + 15) & ~uintptr_t(15));

    int blk = blockIdx.x;
    const int cg = blk % g.n_cg;
    blk /= g.n_cg;
    const int rt = blk % g.n_rt;
    const size_t img = blk / g.n_rt;
    const int r0 = rt * g.TR;
    const int co0 = cg * g.COG;
    const int cog = min(g.COG, g.Cout - co0);

    // work item of this thread
    const int n_cob = (cog + CO_T - 1) / CO_T;
    const int item = threadIdx.x;
    const int n_items = g.TR * g.pxb * n_cob;
    const bool active = item < n_items;
    const int cob = item % n_cob;
    const int rest = item / n_cob;
    const int xb = rest % g.pxb;
    const int ry = rest / g.pxb;              // row inside the tile
    const int x0 = xb * PX;
    const int c_lo = cob * CO_T;              // relative to co0

    float acc[PX][CO_T];
#pragma unroll
    for (int p = 0; p < PX; ++p)
#pragma unroll
        for (int c = 0; c < CO_T; ++c) acc[p][c] = 0.f;

    for (int ci0 = 0; ci0 < g.Cin; ci0 += CI_T) {
        const int nci = min(CI_T, g.Cin - ci0);
        // stage inputs with zero halo
        for (int i = threadIdx.x; i < nci * TRP * SP; i += CNN_THREADS) {
            const int c = i / (TRP * SP);
            const int rem = i % (TRP * SP);
            const int yy = rem / SP - 1 + r0;
            const int xx = rem % SP - 1;
            float v = 0.f;
            if (yy >= 0 && yy < S && xx >= 0 && xx < S) {
                if (IN_MODE == 1) {
                    const int k = yy * S + xx;
                    if (k < g.N_d) {
                        const float2 z = s_in[img * g.N_d + k];
                        v = (ci0 + c) == 0 ? z.x : z.y;
                    }
                } else {
                    v = in[((img * g.Cin + ci0 + c) * S + yy) * S + xx];
                }
            }
            sin_[i] = v;
        }
        // stage weights transposed: sw[c][tap][co - co0]
        for (int i = threadIdx.x; i < nci * 9 * g.COG; i += CNN_THREADS) {
            const int c = i / (9 * g.COG);
            const int rem = i % (9 * g.COG);
            const int tap = rem / g.COG;
            const int co = rem % g.COG;
            sw[i] = co < cog ? W[((size_t)(co0 + co) * g.Cin + ci0 + c) * 9 + tap] : 0.f;
        }
        __syncthreads();
        if (active) {
            for (int c = 0; c < nci; ++c) {
                const float* ip = sin_ + (c * TRP + ry) * SP + x0;
                float iv[3][PX + 2];
#pragma unroll
                for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                    for (int dx = 0; dx < PX + 2; ++dx) iv[dy][dx] = (x0 + dx < SP) ? ip[dy * SP + dx] : 0.f;
                const float* wp = sw + c * 9 * g.COG + c_lo;
#pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                    float wv[CO_T];
                    if constexpr (CO_T == 4) {
                        const float4 w4 = *reinterpret_cast<const float4*>(wp + tap * g.COG);
                        wv[0] = w4.x; wv[1] = w4.y; wv[2] = w4.z; wv[3] = w4.w;
                    } else {
#pragma unroll
                        for (int q = 0; q < CO_T; ++q) wv[q] = wp[tap * g.COG + q];
                    }
                    const int dy = tap / 3, dx = tap % 3;
#pragma unroll
                    for (int p = 0; p < PX; ++p)
#pragma unroll
                        for (int q = 0; q < CO_T; ++q) acc[p][q] = fmaf(wv[q], iv[dy][p + dx], acc[p][q]);
                }
            }
        }
        __syncthreads();
    }
    if (!active) return;
    const int y = r0 + ry;
    if (y >= S) return;
#pragma unroll
    for (int p = 0; p < PX; ++p) {
        const int x = x0 + p;
        if (x >= S) continue;
        if constexpr (OUT_MODE == 0) {
#pragma unroll
            for (int q = 0; q < CO_T; ++q) {
                const int co = co0 + c_lo + q;
                if (c_lo + q < cog) out[((img * g.Cout + co) * S + y) * S + x] = tanhf(acc[p][q] + bias[co]);
            }
        } else if constexpr (CO_T >= 2) {
            const int k = y * S + x;
            if (k < g.N_d) {
                const float2 z = s_in[img * g.N_d + k];
                s_out[img * g.N_d + k] = make_float2(z.x + acc[p][0] + bias[0], z.y + acc[p][1] + bias[1]);
            }
        }
    }
}

// output channels per thread; must match dispatch_conv
static int conv_cot(int Cout) { return (Cout >= 4 && Cout % 4 == 0) ? 4 : (Cout % 2 == 0 ? 2 : 1); }

static ConvGeom make_geom(int Cin, int Cout, int S, int N_d) {
    ConvGeom g;
    g.Cin = Cin;
    g.Cout = Cout;
    g.S = S;
    g.N_d = N_d;
    g.pxb = (S + PX - 1) / PX;
    const int co_t = conv_cot(Cout);
    g.COG = Cout >= 16 ? 16 : Cout;
    const int n_cob = g.COG / co_t;
    int tr = CNN_THREADS / (g.pxb * n_cob);
    if (tr < 1) tr = 1;
    if (tr > S) tr = S;
    const int n_rt = (S + tr - 1) / tr;
    g.TR = (S + n_rt - 1) / n_rt;   // balance the row tiles
    g.n_rt = (S + g.TR - 1) / g.TR;
    g.n_cg = (Cout + g.COG - 1) / g.COG;
    return g;
}

static size_t conv_smem(const ConvGeom& g) {
    return sizeof(float) * ((size_t)CI_T * (g.TR + 2) * (g.S + 2) + 4 + (size_t)CI_T * 9 * g.COG);
}

template <int CO_T, int IN_MODE, int OUT_MODE>
static int launch_conv(const ConvGeom& g, long long n_img, const float* in, const float2* s_in, const float* W,
                       const float* b, float* out, float2* s_out, cudaStream_t st) {
    const size_t smem = conv_smem(g);
    cudaFuncSetAttribute(k_conv<CO_T, IN_MODE, OUT_MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long blocks = n_img * g.n_rt * g.n_cg;
    if (blocks > 0x7fffffffLL) return fail_arg("fdcnn_forward: too many images per call");
    k_conv<CO_T, IN_MODE, OUT_MODE><<<(unsigned)blocks, CNN_THREADS, smem, st>>>(in, s_in, W, b, out, s_out, g);
    return check_launch("fdcnn_forward");
}

template <int IN_MODE, int OUT_MODE>
static int dispatch_conv(const ConvGeom& g, long long n_img, const float* in, const float2* s_in, const float* W,
                         const float* b, float* out, float2* s_out, cudaStream_t st) {
    if (g.Cout >= 4 && g.Cout % 4 == 0) return launch_conv<4, IN_MODE, OUT_MODE>(g, n_img, in, s_in, W, b, out, s_out, st);
    if (g.Cout % 2 == 0) return launch_conv<2, IN_MODE, OUT_MODE>(g, n_img, in, s_in, W, b, out, s_out, st);
    return launch_conv<1, IN_MODE, OUT_MODE>(g, n_img, in, s_in, W, b, out, s_out, st);
}

static int fdcnn_validate(const int* chans, int n_layers, long long n_sym, int U, int N_d) {
    FD_REQUIRE(chans != nullptr, "fdcnn_forward: chans is NULL");
    FD_REQUIRE(n_layers >= 1 && n_layers <= 64, "fdcnn_forward: n_layers=%d", n_layers);
    FD_REQUIRE(chans[0] == 2 && chans[n_layers] == 2, "fdcnn_forward: chans must start and end with 2");
    for (int l = 0; l <= n_layers; ++l) FD_REQUIRE(chans[l] >= 1 && chans[l] <= 256, "fdcnn_forward: chans[%d]=%d", l, chans[l]);
    FD_REQUIRE(n_sym >= 0 && U >= 1 && N_d >= 1 && N_d <= (1 << 20), "fdcnn_forward: bad sizes");
    return FD_OK;
}

}  // namespace fdpd

using namespace fdpd;

extern "C" {

size_t fdcnn_workspace_bytes(const int* chans, int n_layers, long long n_sym, int U, int N_d) {
    if (!chans || n_layers < 2 || n_sym <= 0 || U <= 0 || N_d <= 0) return 0;
    int cmax = 0;
    for (int l = 1; l < n_layers; ++l) cmax = chans[l] > cmax ? chans[l] : cmax;
    int S = 1;
    while (S * S < N_d) ++S;
    const size_t one = sizeof(float) * (size_t)n_sym * U * cmax * S * S;
    return n_layers > 2 ? 2 * one : one;
}

int fdcnn_forward(const float* params, const int* chans, int n_layers, const void* s_in, void* s_out, void* workspace,
                  size_t workspace_bytes, long long n_sym, int U, int N_d, cudaStream_t stream) {
    int rc = fdcnn_validate(chans, n_layers, n_sym, U, N_d);
    if (rc) return rc;
    FD_REQUIRE(params && s_in && s_out, "fdcnn_forward: NULL pointer");
    FD_REQUIRE(s_in != s_out, "fdcnn_forward: s_out must not alias s_in");
    FD_REQUIRE(aligned16(params) && aligned8(s_in) && aligned8(s_out), "fdcnn_forward: misaligned pointer");
    const size_t need = fdcnn_workspace_bytes(chans, n_layers, n_sym, U, N_d);
    FD_REQUIRE(need == 0 || (workspace && aligned16(workspace) && workspace_bytes >= need),
               "fdcnn_forward: workspace of %zu bytes required (got %zu)", need, workspace_bytes);
    if (n_sym == 0) return FD_OK;
    int S = 1;
    while (S * S < N_d) ++S;
    const long long n_img = n_sym * U;
    const float2* sin2 = (const float2*)s_in;
    float2* sout2 = (float2*)s_out;
    float* buf[2] = {(float*)workspace, nullptr};
    if (n_layers > 2) {
        int cmax = 0;
        for (int l = 1; l < n_layers; ++l) cmax = chans[l] > cmax ? chans[l] : cmax;
        buf[1] = buf[0] + (size_t)n_img * cmax * S * S;
    }
    size_t off = 0;
    for (int l = 0; l < n_layers; ++l) {
        const int ci = chans[l], co = chans[l + 1];
        const float* W = params + off;
        const float* b = W + (size_t)co * ci * 9;
        off += (size_t)co * ci * 9 + co;
        const ConvGeom g = make_geom(ci, co, S, N_d);
        FD_REQUIRE(conv_smem(g) <= 200 * 1024 && g.pxb * (g.COG / conv_cot(co)) <= CNN_THREADS,
                   "fdcnn_forward: image too large");
        const bool first = l == 0, last = l == n_layers - 1;
        const float* in = first ? nullptr : buf[(l - 1) & 1];
        float* out = last ? nullptr : buf[l & 1];
        if (first && last) rc = dispatch_conv<1, 1>(g, n_img, in, sin2, W, b, out, sout2, stream);
        else if (first) rc = dispatch_conv<1, 0>(g, n_img, in, sin2, W, b, out, sout2, stream);
        else if (last) rc = dispatch_conv<0, 1>(g, n_img, in, sin2, W, b, out, sout2, stream);
        else rc = dispatch_conv<0, 0>(g, n_img, in, sin2, W, b, out, sout2, stream);
        if (rc) return rc;
    }
    return FD_OK;
}

}  // extern "C"
