// mtgp_bitmap.cuh -- the predicate-bitmap output of the register-resident team kernels (gen3 and
// mt_gen3; the internal kinds kKindBitmapBit0 / kKindBitmapRange of the fused random-walk and
// gap passes, mtgp_stat.cu).
#pragma once

#include <stdint.h>

#include "mtgp_internal.cuh"

namespace mtgpb {

// A 128-word half-step (lane t holds words 4t..4t+3, the half-step starting at piece word hs)
// becomes its 128 predicate bits in word order. Each lane packs its 4 bits into nibble t % 8 of a word;
// three OR butterflies over 8-lane groups leave bitmap word q (words 32q..32q+31) in lane 8q; the
// word is shifted by the piece's bit offset (funnel with lane 8q - 8's word) and ORed into the
// stream's bitmap (pieces share boundary words, hence atomicOr: one per 32 words). Lane 1 writes
// the fifth, partial word of a shifted half-step. Branch-free up to the store, so the warp stays
// converged for the generator's next shuffles. valid: this lane's words are inside the piece.
template <int KIND>
__device__ __forceinline__ void bitmap_store(uint32_t lane, uint32_t* bm, unsigned long long poff,
                                             const BitmapPred& pred, const uint32_t o[4], uint32_t hs, bool valid) {
    constexpr unsigned kAll = 0xffffffffu;
    uint32_t nib = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const bool h = KIND == kKindBitmapBit0 ? (o[c] & 1u) != 0u : ((o[c] & pred.mask) - pred.lo) <= pred.span_m1;
        nib |= (h ? 1u : 0u) << c;
    }
    uint32_t v = valid ? nib << (4 * (lane & 7u)) : 0u;
    v |= __shfl_xor_sync(kAll, v, 1);
    v |= __shfl_xor_sync(kAll, v, 2);
    v |= __shfl_xor_sync(kAll, v, 4);
    // lanes 8q: v = bitmap word q; prev = word q - 1 (0 for q = 0); lane 1 gets word 3 for the tail
    const uint32_t sh = (uint32_t)(poff & 31u);
    uint32_t prev = __shfl_sync(kAll, v, (lane - 8u) & 31u);
    const uint32_t m3 = __shfl_sync(kAll, v, 24);
    prev = lane < 8 ? 0u : prev;
    const bool lead = (lane & 7u) == 0;
    const uint32_t w = lead ? __funnelshift_l(prev, v, sh) : (lane == 1 ? __funnelshift_l(m3, 0u, sh) : 0u);
    const uint32_t widx = lead ? (lane >> 3) : 4u;
    if (w != 0) atomicOr(bm + ((poff + hs) >> 5) + widx, w);
}

}  // namespace mtgpb
