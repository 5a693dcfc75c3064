// mtgp_mt.cuh -- Engine::mt (the reference's classic MT recurrence) device interface.
#pragma once

#include "mtgp_internal.cuh"

namespace mtgpb {

struct alignas(16) DevMtParams {
    uint32_t n, m, r, a, b, c, u, s, t, l, pad0, pad1;
};

cudaError_t launch_mt_v1(int kind, bool cksum, const DevMtParams* params, uint32_t* win, uint32_t n_sets,
                         uint32_t nmax, void* out, uint64_t L, DevCksum* ck, cudaStream_t st);

}  // namespace mtgpb
