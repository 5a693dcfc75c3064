// mtgp_v4.cu -- dispatch for the register-resident generator templated on the exponent
// (kernel: mtgp_v4.cuh; instances: mtgp_v4_<mexp>.cu). u32 output; the float kinds of the larger
// exponents use the shared-memory ring (v2), 11213 has its own tuned kernel (v3).
#include "mtgp_v4.cuh"

namespace mtgpb {

bool v4_supports(uint32_t mexp, int kind) {
    return kind == MTGP_U32 && (mexp == 11213 || mexp == 23209 || mexp == 44497);
}

cudaError_t launch_gen4(uint32_t mexp, int kind, int ck_mode, const GenArgs& a, cudaStream_t st) {
    if (a.n_teams == 0) return cudaSuccess;
    if (kind != MTGP_U32) return cudaErrorInvalidValue;
    switch (mexp) {
        case 11213: return launch_gen4_11213(ck_mode, a, st);
        case 23209: return launch_gen4_23209(ck_mode, a, st);
        case 44497: return launch_gen4_44497(ck_mode, a, st);
    }
    return cudaErrorInvalidValue;
}

int gen4_ctas_per_sm(uint32_t mexp, int kind, int ck_mode) {
    if (kind != MTGP_U32) return 0;
    switch (mexp) {
        case 11213: return gen4_ctas_11213(ck_mode);
        case 23209: return gen4_ctas_23209(ck_mode);
        case 44497: return gen4_ctas_44497(ck_mode);
    }
    return 0;
}

}  // namespace mtgpb
