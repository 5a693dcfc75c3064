// mtgp_v4_11213.cu -- gen4_kernel instances for MTGP32-11213 (u32 output; see mtgp_v4.cuh).
#include "mtgp_v4.cuh"

namespace mtgpb {

cudaError_t launch_gen4_11213(bool cksum, const GenArgs& a, cudaStream_t st) {
    return cksum ? launch4_t<11213, MTGP_U32, true>(a, st) : launch4_t<11213, MTGP_U32, false>(a, st);
}

int gen4_ctas_11213(bool cksum) { return cksum ? occ4_t<11213, MTGP_U32, true>() : occ4_t<11213, MTGP_U32, false>(); }

}  // namespace mtgpb
