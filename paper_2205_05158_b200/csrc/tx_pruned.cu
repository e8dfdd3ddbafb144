// tx_pruned.cu — chain_txrx instantiations with the pruned radix-16 FFT passes (chain.cuh,
// fft.cuh) for the transform sizes and GMP shapes of the configured workloads; compiled in
// its own translation unit so the build parallelises.
#include "chain.cuh"

namespace fdpd {

template <int LOG2N, int PZ>
static int pruned_variant(int variant, const float2* P, const float2* s, const float2* coef, float2* y, float2* XPA,
                          long long n_sym, int B, int U, int N_d, const GmpDesc& d, const Impair& imp,
                          cudaStream_t st) {
    switch (variant) {
        case 2: return launch_chain_one<LOG2N, 4, 4, 2, 4, true, PZ>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        case 3: return launch_chain_one<LOG2N, 5, 6, 3, 4, true, PZ>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        case 4: return launch_chain_one<LOG2N, 4, 3, 1, 4, true, PZ>(P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
        default: return -1;
    }
}

int launch_chain_pruned(int log2n, int variant, int pz, const float2* P, const float2* s, const float2* coef,
                        float2* y, float2* XPA, long long n_sym, int B, int U, int N_d, const GmpDesc& d,
                        const Impair& imp, cudaStream_t st) {
#define FD_PRUNED(LG)                                                                                      \
    case LG:                                                                                               \
        return pz == 1 ? pruned_variant<LG, 1>(variant, P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st)   \
                       : pruned_variant<LG, 2>(variant, P, s, coef, y, XPA, n_sym, B, U, N_d, d, imp, st);
    switch (log2n) {
        FD_PRUNED(12)
        FD_PRUNED(13)
        FD_PRUNED(14)
        default: return -1;
    }
#undef FD_PRUNED
}

}  // namespace fdpd
