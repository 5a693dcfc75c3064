// mtgp_v4_44497.cu -- gen4_kernel instances for MTGP32-44497 (u32 output; see mtgp_v4.cuh).
#include "mtgp_v4.cuh"

namespace mtgpb {

cudaError_t launch_gen4_44497(int ck_mode, const GenArgs& a, cudaStream_t st) {
    return ck_mode == 2 ? launch4_t<44497, MTGP_U32, 2>(a, st)
         : ck_mode == 1 ? launch4_t<44497, MTGP_U32, 1>(a, st) : launch4_t<44497, MTGP_U32, 0>(a, st);
}

int gen4_ctas_44497(int ck_mode) {
    return ck_mode == 2 ? occ4_t<44497, MTGP_U32, 2>() : ck_mode == 1 ? occ4_t<44497, MTGP_U32, 1>() : occ4_t<44497, MTGP_U32, 0>();
}

}  // namespace mtgpb
