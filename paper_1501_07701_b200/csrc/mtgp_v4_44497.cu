// mtgp_v4_44497.cu -- gen4_kernel instances for MTGP32-44497 (u32 output; see mtgp_v4.cuh).
#include "mtgp_v4.cuh"

namespace mtgpb {

cudaError_t launch_gen4_44497(bool cksum, const GenArgs& a, cudaStream_t st) {
    return cksum ? launch4_t<44497, MTGP_U32, true>(a, st) : launch4_t<44497, MTGP_U32, false>(a, st);
}

int gen4_ctas_44497(bool cksum) { return cksum ? occ4_t<44497, MTGP_U32, true>() : occ4_t<44497, MTGP_U32, false>(); }

}  // namespace mtgpb
