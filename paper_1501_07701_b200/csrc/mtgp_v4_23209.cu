// mtgp_v4_23209.cu -- gen4_kernel instances for MTGP32-23209 (u32 output; see mtgp_v4.cuh).
#include "mtgp_v4.cuh"

namespace mtgpb {

cudaError_t launch_gen4_23209(bool cksum, const GenArgs& a, cudaStream_t st) {
    return cksum ? launch4_t<23209, MTGP_U32, true>(a, st) : launch4_t<23209, MTGP_U32, false>(a, st);
}

int gen4_ctas_23209(bool cksum) { return cksum ? occ4_t<23209, MTGP_U32, true>() : occ4_t<23209, MTGP_U32, false>(); }

}  // namespace mtgpb
