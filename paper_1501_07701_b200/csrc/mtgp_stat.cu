// mtgp_stat.cu -- device-side statistical tests over generated streams.
//
// The reference runs a campaign cell as run_test(BufferedStream(make_word_source(status, seed)))
// (proj/src/sieve.cpp:156-158): a fresh stream per (status, seed, test), consumed word by word by
// one of four templates (proj/include/twistsieve/stat_tests.hpp:84-309). Here every stream of a
// context is tested at once: the context generates the next C words of all S streams into one
// HBM chunk (its normal generation kernels), a counting kernel folds the chunk into per-stream
// integer counts, and the chunk buffer is reused. Words never leave the GPU; the host only turns
// the final counts into statistic / p-value / class (stat_host.cpp).
//
// Chunk sizes are whole multiples of each test's unit (walks; pairs of L-bit blocks), so the
// fixed-length tests need no state across chunks. The gap test is data-dependent (it reads until
// the n-th gap closes, within a word budget); it carries {hits so far, last hit position} per
// stream and finds hit ordinals with a per-chunk tile scan. Counts are exact integers, so results
// are bit-identical to the reference templates over the same words.
//
// All four kernels read each word once (coalesced) and do O(1) work per word: HBM/L2-read bound,
// cheap next to generation. Roofline note in DESIGN.md §4.5.
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "mtgp_ctx.h"
#include "stat_host.h"

namespace mtgpb {
namespace {

constexpr uint32_t kThreads = 256;
constexpr uint32_t kWarps = kThreads / 32;
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t letter_of(uint32_t w, uint32_t r, uint32_t s) {
    // detail::letter_of (stat_tests.hpp:60-63): the s most significant bits left after dropping r
    return (w >> (32u - r - s)) & ((1u << s) - 1u);
}

__device__ __forceinline__ uint32_t low_mask(uint32_t k) { return k >= 32 ? kFull : ((1u << k) - 1u); }

// popcount of bits [a, e) of a bitmap (bit i of word q is item 32q + i), a < e
__device__ uint32_t range_popc(const uint32_t* bm, uint32_t a, uint32_t e) {
    const uint32_t qa = a >> 5, qe = (e - 1) >> 5, sa = a & 31u;
    if (qa == qe) return __popc((bm[qa] >> sa) & low_mask(e - a));
    uint32_t h = __popc(bm[qa] >> sa);
    for (uint32_t q = qa + 1; q < qe; ++q) h += __popc(bm[q]);
    return h + __popc(bm[qe] & low_mask(((e - 1) & 31u) + 1));
}

// ---------------------------------------------------------------------------------------------
// random walk (stat_tests.hpp:253-309): walk i = words [i l, (i+1) l); H = number of odd words.
// A CTA takes wpt whole walks: bit 0 of its words -> shared bitmap by warp ballots (coalesced
// loads), then one thread per walk popcounts its bit range.
template <bool SMEM_HIST>
__global__ void __launch_bounds__(kThreads) walk_kernel(const uint32_t* __restrict__ w, uint64_t C, uint32_t l,
                                                        uint32_t wpt, uint64_t walk0, uint64_t n,
                                                        unsigned long long* __restrict__ counts) {
    extern __shared__ uint32_t sm[];
    const uint32_t tile_words = wpt * l;
    const uint32_t nbm = (tile_words + 31) / 32;
    uint32_t* bm = sm;
    uint32_t* hist = sm + nbm;
    const uint32_t st = blockIdx.y;
    const uint64_t first_walk = walk0 + (uint64_t)blockIdx.x * wpt;
    if (first_walk >= n) return;
    const uint32_t* src = w + (size_t)st * C + (size_t)blockIdx.x * tile_words;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (SMEM_HIST)
        for (uint32_t i = threadIdx.x; i <= l; i += kThreads) hist[i] = 0;
    for (uint32_t q = warp; q < nbm; q += kWarps) {
        const uint32_t j = q * 32 + lane;
        const uint32_t odd = j < tile_words ? (__ldg(src + j) & 1u) : 0u;
        const uint32_t b = __ballot_sync(kFull, odd);
        if (lane == 0) bm[q] = b;
    }
    __syncthreads();
    unsigned long long* cs = counts + (size_t)st * (l + 1);
    for (uint32_t t = threadIdx.x; t < wpt && first_walk + t < n; t += kThreads) {
        const uint32_t h = range_popc(bm, t * l, t * l + l);
        if (SMEM_HIST)
            atomicAdd(hist + h, 1u);
        else
            atomicAdd(cs + h, 1ull);
    }
    if (SMEM_HIST) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i <= l; i += kThreads)
            if (hist[i]) atomicAdd(cs + i, (unsigned long long)hist[i]);
    }
}

// The same walks from a bit-0 bitmap the generator wrote directly (ctx_generate_bitmap,
// kKindBitmapBit0): the chunk's words never reach HBM. Bit j of a stream's bitmap is word j of
// its chunk; one thread per walk popcounts its l bits.
template <bool SMEM_HIST>
__global__ void __launch_bounds__(kThreads) walk_bm_kernel(const uint32_t* __restrict__ bm, uint64_t bm_stride,
                                                           uint32_t l, uint32_t wpt, uint64_t walk0, uint64_t n,
                                                           unsigned long long* __restrict__ counts) {
    extern __shared__ uint32_t sm[];
    uint32_t* hist = sm;
    const uint32_t st = blockIdx.y;
    const uint64_t first_walk = walk0 + (uint64_t)blockIdx.x * wpt;
    if (first_walk >= n) return;
    const uint32_t* b = bm + (size_t)st * bm_stride;
    if (SMEM_HIST) {
        for (uint32_t i = threadIdx.x; i <= l; i += kThreads) hist[i] = 0;
        __syncthreads();
    }
    unsigned long long* cs = counts + (size_t)st * (l + 1);
    for (uint32_t t = threadIdx.x; t < wpt && first_walk + t < n; t += kThreads) {
        const uint32_t a = (blockIdx.x * wpt + t) * l;
        const uint32_t h = range_popc(b, a, a + l);
        if (SMEM_HIST)
            atomicAdd(hist + h, 1u);
        else
            atomicAdd(cs + h, 1ull);
    }
    if (SMEM_HIST) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i <= l; i += kThreads)
            if (hist[i]) atomicAdd(cs + i, (unsigned long long)hist[i]);
    }
}

// ---------------------------------------------------------------------------------------------
// Hamming-weight independence (stat_tests.hpp:149-208): s-bit letters concatenated MSB first
// into L-bit blocks; blocks (2i, 2i+1) form pair i. A CTA takes ppt whole pairs (tile_words
// words, a multiple of the pair unit 2L/gcd(2L, s)): letters and an exclusive prefix sum of
// their popcounts go to shared memory, then each block's weight is O(1): the partial first
// letter + prefix difference + the partial last letter.
__global__ void __launch_bounds__(kThreads) hamming_kernel(const uint32_t* __restrict__ w, uint64_t C, uint32_t r,
                                                           uint32_t sb, uint32_t L, uint32_t ppt,
                                                           uint32_t tile_words, uint64_t pair0, uint64_t npairs,
                                                           unsigned long long* __restrict__ table) {
    extern __shared__ uint32_t sm[];
    uint32_t* let = sm;               // [tile_words]
    uint32_t* pre = sm + tile_words;  // [tile_words + 1], pre[j] = sum_{i<j} popc(let[i])
    __shared__ uint32_t warp_tot[kWarps];
    __shared__ uint32_t cat[4];
    const uint32_t st = blockIdx.y;
    const uint64_t first_pair = pair0 + (uint64_t)blockIdx.x * ppt;
    if (first_pair >= npairs) return;
    const uint32_t* src = w + (size_t)st * C + (size_t)blockIdx.x * tile_words;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (threadIdx.x < 4) cat[threadIdx.x] = 0;
    for (uint32_t j = threadIdx.x; j < tile_words; j += kThreads) let[j] = letter_of(__ldg(src + j), r, sb);
    __syncthreads();

    // block-wide exclusive scan: warp w owns a contiguous range of 32-word strips; lanes walk a
    // strip side by side (conflict-free shared-memory access), one warp total pass then one
    // scanned pass
    const uint32_t strips = (tile_words + 31) / 32;
    const uint32_t spw = (strips + kWarps - 1) / kWarps;
    const uint32_t s0 = min(warp * spw, strips), s1 = min(s0 + spw, strips);
    uint32_t own = 0;
    for (uint32_t q = s0; q < s1; ++q) {
        const uint32_t j = q * 32 + lane;
        own += j < tile_words ? __popc(let[j]) : 0u;
    }
    for (int d = 16; d > 0; d >>= 1) own += __shfl_xor_sync(kFull, own, d);
    if (lane == 0) warp_tot[warp] = own;
    __syncthreads();
    uint32_t carry = 0;
    for (uint32_t i = 0; i < warp; ++i) carry += warp_tot[i];
    for (uint32_t q = s0; q < s1; ++q) {
        const uint32_t j = q * 32 + lane;
        const uint32_t v = j < tile_words ? __popc(let[j]) : 0u;
        uint32_t incl = v;
        for (uint32_t d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += u;
        }
        if (j < tile_words) pre[j] = carry + incl - v;
        carry += __shfl_sync(kFull, incl, 31);
    }
    if (warp == kWarps - 1 && lane == 0) {
        uint32_t tot = 0;
        for (uint32_t i = 0; i < kWarps; ++i) tot += warp_tot[i];
        pre[tile_words] = tot;
    }
    __syncthreads();

    const uint32_t half = L / 2;
    for (uint32_t pp = threadIdx.x; pp < ppt && first_pair + pp < npairs; pp += kThreads) {
        uint32_t sign[2];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const uint32_t B = (2 * pp + b) * L, E = B + L;  // local bit range [B, E)
            const uint32_t jf = B / sb, of = B - jf * sb;     // first letter, bits already taken
            const uint32_t jl = (E - 1) / sb, eo = E - jl * sb;  // last letter, bits taken from it
            uint32_t wt;
            if (jf == jl)
                wt = __popc((let[jf] >> (sb - eo)) & low_mask(eo - of));
            else
                wt = __popc(let[jf] & low_mask(sb - of)) + (pre[jl] - pre[jf + 1]) + __popc(let[jl] >> (sb - eo));
            sign[b] = wt > half ? 1u : 0u;
        }
        atomicAdd(&cat[sign[0] * 2 + sign[1]], 1u);  // table[first_sign][second_sign]
    }
    __syncthreads();
    if (threadIdx.x < 4 && cat[threadIdx.x])
        atomicAdd(table + (size_t)st * 4 + threadIdx.x, (unsigned long long)cat[threadIdx.x]);
}

// Long blocks (>= 32 letters): one warp per block, no shared-memory scan. Lanes stride the
// block's letters (coalesced loads straight from the chunk), the partial first / last letters
// are masked, popcounts are warp-reduced; the two blocks of a pair run back to back on the
// same warp.
__global__ void __launch_bounds__(kThreads) hamming_warp_kernel(const uint32_t* __restrict__ w, uint64_t C, uint32_t r,
                                                                uint32_t sb, uint32_t L, uint64_t pairs_chunk,
                                                                uint64_t pair0, uint64_t npairs,
                                                                unsigned long long* __restrict__ table) {
    __shared__ uint32_t cat[4];
    const uint32_t st = blockIdx.y;
    const uint32_t* src = w + (size_t)st * C;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (threadIdx.x < 4) cat[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t half = L / 2;
    const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
    for (uint64_t pp = (uint64_t)blockIdx.x * kWarps + warp; pp < pairs_chunk && pair0 + pp < npairs; pp += nwarps) {
        uint32_t sign[2];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const uint64_t B = (2 * pp + b) * (uint64_t)L, E = B + L;  // chunk-local bit range
            const uint32_t jf = (uint32_t)(B / sb), jl = (uint32_t)((E - 1) / sb);  // letters (< C)
            const uint32_t of = (uint32_t)(B - (uint64_t)jf * sb), eo = (uint32_t)(E - (uint64_t)jl * sb);
            // interior letters whole: popc of the letter = popc of the word under the letter mask
            const uint32_t lmask = ((1u << sb) - 1u) << (32u - r - sb);
            uint32_t cnt = 0;
            for (uint32_t j = jf + 1 + lane; j < jl; j += 32) cnt += __popc(__ldg(src + j) & lmask);
            if (lane == 0) {  // the partial first / last letters
                const uint32_t vf = letter_of(__ldg(src + jf), r, sb);
                if (jf == jl) {
                    cnt += __popc((vf >> (sb - eo)) & low_mask(eo - of));
                } else {
                    cnt += __popc(vf & low_mask(sb - of));  // skips the `of` bits the previous block took
                    cnt += __popc(letter_of(__ldg(src + jl), r, sb) >> (sb - eo));  // top eo bits
                }
            }
            for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(kFull, cnt, d);
            sign[b] = cnt > half ? 1u : 0u;
        }
        if (lane == 0) atomicAdd(&cat[sign[0] * 2 + sign[1]], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 4 && cat[threadIdx.x])
        atomicAdd(table + (size_t)st * 4 + threadIdx.x, (unsigned long long)cat[threadIdx.x]);
}

// ---------------------------------------------------------------------------------------------
// Overlapping-pairs collisions (stat_tests.hpp:214-248): cell i = letter(w_i) << s | letter(w_i+1),
// i < n; a collision is a visit to an occupied cell. The count n - |distinct cells| does not
// depend on visiting order, so cells are marked with atomicOr in a per-stream 2^(2s)-bit map.
// The word before the chunk comes from the previous chunk (prev_in / prev_out ping-pong).
__global__ void __launch_bounds__(kThreads) opso_kernel(const uint32_t* __restrict__ w, uint64_t C, uint64_t P,
                                                        uint32_t r, uint32_t sb, uint64_t n,
                                                        uint32_t* __restrict__ bitmap, uint64_t bm_words,
                                                        const uint32_t* __restrict__ prev_in,
                                                        uint32_t* __restrict__ prev_out,
                                                        unsigned long long* __restrict__ coll) {
    const uint32_t st = blockIdx.y;
    const uint32_t* src = w + (size_t)st * C;
    uint32_t* bmp = bitmap + (size_t)st * bm_words;
    uint32_t mine = 0;
    for (uint64_t j = (uint64_t)blockIdx.x * kThreads + threadIdx.x; j < C; j += (uint64_t)gridDim.x * kThreads) {
        const uint32_t cur_w = __ldg(src + j);
        if (j == C - 1) prev_out[st] = cur_w;
        const uint64_t g = P + j;  // global word index; it closes cell g - 1
        if (g == 0 || g - 1 >= n) continue;
        const uint32_t prv_w = j ? __ldg(src + j - 1) : prev_in[st];
        const uint32_t cell = (letter_of(prv_w, r, sb) << sb) | letter_of(cur_w, r, sb);
        const uint32_t bit = 1u << (cell & 31u);
        mine += (atomicOr(bmp + (cell >> 5), bit) & bit) ? 1u : 0u;
    }
    for (int d = 16; d > 0; d >>= 1) mine += __shfl_xor_sync(kFull, mine, d);
    if ((threadIdx.x & 31u) == 0 && mine) atomicAdd(coll + st, (unsigned long long)mine);
}

// ---------------------------------------------------------------------------------------------
// Gap test (stat_tests.hpp:84-138). Hits h_0 < h_1 < ... are the words whose kept bits fall in
// [alpha, beta) (integer thresholds lo <= v < hi); gap k = h_k - h_{k-1} - 1 for k = 1..n goes to
// bin min(gap, tcut). Only words below the budget count (the reference throws StreamExhausted
// when it would read word `budget`). Per chunk: (1) per-tile hit count / first / last,
// (2) per-tile ordinal base from a scan of the earlier tiles plus the stream's carried state,
// then the tile's gaps, (3) per-stream state update.
constexpr uint32_t kGapTile = 4096;                   // words per CTA
constexpr uint32_t kGapGroups = kGapTile / kThreads;  // 32-word groups per warp (16)
#ifndef MTGP_GAP_HIST_CTAS
#define MTGP_GAP_HIST_CTAS 48  // 24: 16.2 ms, 48: 16.1, 96: 16.0 for the fused desk gap (12: 17.5)
#endif
constexpr uint32_t kGapHistCtas = MTGP_GAP_HIST_CTAS;  // histogram CTAs per stream
// histogram pass: 4 warps x 32 lanes, one 32-word group per lane, one 4096-word tile per CTA
// iteration (8 warps with 16 active lanes each measured slower)
constexpr uint32_t kHistThreads = 128, kHistWarps = kHistThreads / 32;
static_assert(kHistWarps * 32 * 32 == kGapTile, "a tile is one CTA iteration");

struct GapTile {
    uint32_t count;
    int32_t first, last;  // CHUNK-local word index of the tile's first / last hit, -1 if none
};

struct GapState {
    unsigned long long hits;  // hits seen so far (h_0 included)
    long long last_hit;       // global index of the last hit, -1 if none
    unsigned long long end;   // global index of h_n once done
    uint32_t done, exhausted;
};

__device__ __forceinline__ uint32_t gap_ballot(const uint32_t* src, uint64_t j, uint64_t g, uint32_t mask, uint64_t lo,
                                               uint64_t hi, uint64_t budget) {
    const uint64_t v = __ldg(src + j) & mask;
    return __ballot_sync(kFull, g < budget && v >= lo && v < hi);
}

__global__ void __launch_bounds__(kThreads) gap_count_kernel(const uint32_t* __restrict__ w, uint64_t C, uint64_t P,
                                                             uint32_t mask, uint64_t lo, uint64_t hi, uint64_t budget,
                                                             const GapState* __restrict__ state,
                                                             GapTile* __restrict__ tiles, uint32_t T,
                                                             uint32_t* __restrict__ hits) {
    __shared__ uint32_t wc[kWarps];
    __shared__ int32_t wf[kWarps], wl[kWarps];
    const uint32_t st = blockIdx.y, tile = blockIdx.x;
    if (state[st].done) {
        if (threadIdx.x == 0) tiles[(size_t)st * T + tile] = GapTile{0, -1, -1};
        return;
    }
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t* src = w + (size_t)st * C;
    const uint32_t base = tile * kGapTile + warp * (kGapGroups * 32);
    uint32_t cnt = 0, mine = 0;
    int32_t first = -1, last = -1;
#pragma unroll
    for (uint32_t g = 0; g < kGapGroups; ++g) {
        const uint32_t j = base + g * 32;
        const uint32_t m = gap_ballot(src, j + lane, P + j + lane, mask, lo, hi, budget);
        if (lane == g) mine = m;
        if (m) {
            cnt += __popc(m);
            if (first < 0) first = (int32_t)(j + __ffs(m) - 1);
            last = (int32_t)(j + 31 - __clz(m));
        }
    }
    // hit bitmap (1 bit per word) for the histogram pass: 64 B per warp, coalesced
    if (lane < kGapGroups) hits[(size_t)st * (C / 32) + base / 32 + lane] = mine;
    if (lane == 0) {
        wc[warp] = cnt;
        wf[warp] = first;
        wl[warp] = last;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        GapTile t{0, -1, -1};
        for (uint32_t i = 0; i < kWarps; ++i) {
            t.count += wc[i];
            if (t.first < 0) t.first = wf[i];
            if (wl[i] >= 0) t.last = wl[i];
        }
        tiles[(size_t)st * T + tile] = t;
    }
}

// The same per-tile summary from a hit bitmap the generator wrote directly (ctx_generate_bitmap,
// kKindBitmapRange: lo <= (word & mask) < hi). One thread per bitmap word (128 per tile); bits at
// or past the word budget are cleared here (in place, for the histogram pass).
constexpr uint32_t kGapBmThreads = kGapTile / 32;  // 128
__global__ void __launch_bounds__(kGapBmThreads) gap_count_bm_kernel(uint32_t* __restrict__ hits, uint64_t C,
                                                                     uint64_t P, uint64_t budget,
                                                                     const GapState* __restrict__ state,
                                                                     GapTile* __restrict__ tiles, uint32_t T) {
    __shared__ uint32_t wc[kGapBmThreads / 32];
    __shared__ int32_t wf[kGapBmThreads / 32], wl[kGapBmThreads / 32];
    const uint32_t st = blockIdx.y, tile = blockIdx.x;
    if (state[st].done) {
        if (threadIdx.x == 0) tiles[(size_t)st * T + tile] = GapTile{0, -1, -1};
        return;
    }
    const uint32_t q = tile * kGapBmThreads + threadIdx.x;  // bitmap word within the stream's chunk
    uint32_t* hw = hits + (size_t)st * (C / 32) + q;
    uint32_t m = *hw;
    const uint64_t g0 = P + 32ull * q;  // stream index of bit 0
    if (g0 + 32 > budget) {
        m = g0 >= budget ? 0u : (m & low_mask((uint32_t)(budget - g0)));
        *hw = m;
    }
    uint32_t cnt = __popc(m);
    int32_t first = m ? (int32_t)(32 * q + __ffs(m) - 1) : -1;
    int32_t last = m ? (int32_t)(32 * q + 31 - __clz(m)) : -1;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        cnt += __shfl_xor_sync(kFull, cnt, s);
        const int32_t f = __shfl_xor_sync(kFull, first, s);
        const int32_t l = __shfl_xor_sync(kFull, last, s);
        if (f >= 0 && (first < 0 || f < first)) first = f;
        if (l > last) last = l;
    }
    const uint32_t warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31u) == 0) {
        wc[warp] = cnt;
        wf[warp] = first;
        wl[warp] = last;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        GapTile t{0, -1, -1};
        for (uint32_t i = 0; i < kGapBmThreads / 32; ++i) {
            t.count += wc[i];
            if (t.first < 0) t.first = wf[i];
            if (wl[i] >= 0) t.last = wl[i];
        }
        tiles[(size_t)st * T + tile] = t;
    }
}

// Per stream: exclusive scan of the chunk's tile counts -> the ordinal of each tile's first hit
// and the hit before it; advances the carried {hits, last_hit} (done is set by gap_update_kernel
// after the histogram pass, which still needs the old value).
struct GapPre {
    unsigned long long ord0;  // ordinal k of the tile's first hit (it is h_k)
    long long prev;           // global index of the hit before it, -1 if none
};

__global__ void __launch_bounds__(kThreads) gap_scan_kernel(const GapTile* __restrict__ tiles, uint32_t T, uint64_t P,
                                                            GapState* __restrict__ state, GapPre* __restrict__ pre) {
    __shared__ unsigned long long wsum[kWarps];
    __shared__ long long wlast[kWarps];
    const uint32_t st = blockIdx.x;
    const GapState g = state[st];
    if (g.done) return;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const GapTile* tl = tiles + (size_t)st * T;
    const uint32_t seg = (T + kThreads - 1) / kThreads;
    const uint32_t t0 = min(threadIdx.x * seg, T), t1 = min(t0 + seg, T);
    unsigned long long sum = 0;
    long long last = -1;  // chunk-local, positions grow with t so max == most recent
    for (uint32_t t = t0; t < t1; ++t) {
        sum += tl[t].count;
        if (tl[t].count) last = tl[t].last;
    }
    unsigned long long isum = sum;
    long long ilast = last;
    for (uint32_t d = 1; d < 32; d <<= 1) {
        const unsigned long long u = __shfl_up_sync(kFull, isum, d);
        const long long v = __shfl_up_sync(kFull, ilast, d);
        if (lane >= d) {
            isum += u;
            ilast = max(ilast, v);
        }
    }
    if (lane == 31) {
        wsum[warp] = isum;
        wlast[warp] = ilast;
    }
    __syncthreads();
    unsigned long long ord = g.hits + isum - sum;
    long long before = -1;
    {
        const long long v = __shfl_up_sync(kFull, ilast, 1);
        before = lane ? v : -1;
    }
    for (uint32_t i = 0; i < warp; ++i) {
        ord += wsum[i];
        before = max(before, wlast[i]);
    }
    long long prev = before >= 0 ? (long long)P + before : g.last_hit;
    for (uint32_t t = t0; t < t1; ++t) {
        pre[(size_t)st * T + t] = GapPre{ord, prev};
        ord += tl[t].count;
        if (tl[t].count) prev = (long long)P + tl[t].last;
    }
    if (threadIdx.x == kThreads - 1) {  // its running values end at the chunk totals
        state[st].hits = ord;
        state[st].last_hit = prev;
    }
}

// Histogram pass: a CTA walks tiles blockIdx.x, +gridDim.x, ... of one stream (from the hit
// bitmap, not the words), so each CTA zeroes and flushes its shared histogram once.
template <bool SMEM_HIST>
__global__ void __launch_bounds__(kHistThreads) gap_hist_kernel(const uint32_t* __restrict__ hits, uint64_t C, uint64_t P,
                                                            const GapState* __restrict__ state,
                                                            const GapTile* __restrict__ tiles,
                                                            const GapPre* __restrict__ pre, uint32_t T, uint64_t n,
                                                            uint32_t tcut, unsigned long long* __restrict__ counts,
                                                            unsigned long long* __restrict__ end_pos) {
    extern __shared__ uint32_t hist[];
    __shared__ uint32_t wc[kHistWarps];
    __shared__ int32_t wl[kHistWarps];
    const uint32_t st = blockIdx.y;
    if (state[st].done) return;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (SMEM_HIST)
        for (uint32_t i = threadIdx.x; i <= tcut; i += kHistThreads) hist[i] = 0;
    unsigned long long* cs = counts + (size_t)st * (tcut + 1);
    bool touched = false;
    for (uint32_t tile = blockIdx.x; tile < T; tile += gridDim.x) {
        if (tiles[(size_t)st * T + tile].count == 0) continue;
        const GapPre tp = pre[(size_t)st * T + tile];
        if (tp.ord0 > n) break;  // ordinals only grow with the tile index
        touched = true;
        const uint32_t base = tile * kGapTile + warp * (32 * 32);
        // lane g owns group g (32 words) of the warp's 1024: its hit mask, the number of hits
        // before it (exclusive scan) and the last hit before it (exclusive max scan)
        const uint32_t m = __ldg(hits + (size_t)st * (C / 32) + base / 32 + lane);
        const uint32_t c = __popc(m);
        const int32_t lst = m ? (int32_t)(base + lane * 32 + 31 - __clz(m)) : -1;
        uint32_t ic = c;
        int32_t il = lst;
        for (uint32_t d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(kFull, ic, d);
            const int32_t v = __shfl_up_sync(kFull, il, d);
            if (lane >= d) {
                ic += u;
                il = max(il, v);
            }
        }
        const uint32_t warp_cnt = __shfl_sync(kFull, ic, 31);
        const int32_t warp_last = __shfl_sync(kFull, il, 31);
        int32_t before = __shfl_up_sync(kFull, il, 1);
        if (lane == 0) before = -1;
        __syncthreads();  // previous tile's readers of wc / wl are done
        if (lane == 0) {
            wc[warp] = warp_cnt;
            wl[warp] = warp_last;
        }
        __syncthreads();
        unsigned long long ord = tp.ord0;
        long long prev = tp.prev;
        for (uint32_t i = 0; i < warp; ++i) {
            ord += wc[i];
            if (wl[i] >= 0) prev = (long long)P + wl[i];
        }
        if (ord > n || !m) continue;
        unsigned long long k = ord + ic - c;  // ordinal of this group's first hit
        long long pv = before >= 0 ? (long long)P + before : prev;
        const long long pos0 = (long long)P + base + lane * 32;
        for (uint32_t mm = m; mm && k <= n; mm &= mm - 1, ++k) {
            const long long pos = pos0 + __ffs(mm) - 1;  // this hit is h_k
            if (k >= 1) {
                const unsigned long long gap = (unsigned long long)(pos - pv - 1);
                const uint32_t bin = gap < tcut ? (uint32_t)gap : tcut;
                if (SMEM_HIST)
                    atomicAdd(hist + bin, 1u);
                else
                    atomicAdd(cs + bin, 1ull);
                if (k == n) end_pos[st] = (unsigned long long)pos;
            }
            pv = pos;
        }
    }
    if (SMEM_HIST && touched) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i <= tcut; i += kHistThreads)
            if (hist[i]) atomicAdd(cs + i, (unsigned long long)hist[i]);
    }
}

__global__ void gap_update_kernel(uint32_t S, uint64_t P, uint64_t C, uint64_t budget, uint64_t n,
                                  const unsigned long long* __restrict__ end_pos, GapState* __restrict__ state) {
    const uint32_t st = blockIdx.x * blockDim.x + threadIdx.x;
    if (st >= S) return;
    GapState g = state[st];
    if (g.done) return;
    if (g.hits >= n + 1) {  // hits already advanced by gap_scan_kernel
        g.done = 1;
        g.end = end_pos[st];
    } else if (P + C >= budget) {
        g.done = 1;
        g.exhausted = 1;
    }
    state[st] = g;
}

// ---------------------------------------------------------------------------------------------
// host driver

// A device sub-buffer of the context's scratch (non-owning).
struct DevBuf {
    void* p = nullptr;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct Failure {
    int code;
};

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Failure{cuda_error(e, what)};
}

// Context-owned scratch slot, grown on demand: a stat run makes no cudaMalloc / cudaFree after
// the first one of its size (cudaFree synchronises the device and can stall for a long time).
void* scratch(mtgp_ctx* ctx, int slot, size_t bytes) {
    if (ctx->scratch_bytes[slot] < bytes) {
        check(cudaStreamSynchronize(ctx->stream), "sync");
        cudaFree(ctx->d_scratch[slot]);
        ctx->d_scratch[slot] = nullptr;
        ctx->scratch_bytes[slot] = 0;
        check(cudaMalloc(&ctx->d_scratch[slot], bytes), "cudaMalloc stat scratch");
        ctx->scratch_bytes[slot] = bytes;
    }
    return ctx->d_scratch[slot];
}

// Carves the chunk buffer and a run's counters out of scratch slot 1.
struct Arena {
    std::vector<std::pair<DevBuf*, size_t>> parts;
    void add(DevBuf& b, size_t bytes) { parts.push_back({&b, (std::max<size_t>(bytes, 16) + 255) & ~size_t(255)}); }
    uint32_t* commit(mtgp_ctx* ctx, size_t chunk_bytes) {
        size_t total = (chunk_bytes + 255) & ~size_t(255);
        for (auto& pb : parts) total += pb.second;
        char* base = static_cast<char*>(scratch(ctx, 1, total));
        size_t off = (chunk_bytes + 255) & ~size_t(255);
        for (auto& pb : parts) {
            pb.first->p = base + off;
            off += pb.second;
        }
        return reinterpret_cast<uint32_t*>(base);
    }
};

// Saves the context's stream state and restores it on scope exit: the stat run consumes the
// streams from their current position but leaves them (and the checksums) untouched. The jump
// planner's annihilator analysis is made up front at the saved window, so it stays valid after
// the restore (an analysis holds for its window and every later one) and is not redone per run.
struct StateGuard {
    mtgp_ctx* ctx;
    void* win;
    std::vector<uint64_t> pos;
    bool cksum;
    explicit StateGuard(mtgp_ctx* c) : ctx(c), pos(c->position), cksum(c->cksum) {
        const size_t bytes = (size_t)ctx->n_sets * ctx->N * 4;
        win = scratch(ctx, 0, bytes);
        check(cudaMemcpyAsync(win, ctx->d_win, bytes, cudaMemcpyDeviceToDevice, ctx->stream), "state copy");
        if (ctx->planner && ctx->planner->v2_supported()) {
            std::string err;
            const void* prm =
                ctx->engine == 1 ? static_cast<const void*>(ctx->d_mt) : static_cast<const void*>(ctx->d_params);
            check(ctx->planner->analyze_now(prm, ctx->d_win, ctx->stream, err), "annihilator analysis");
        }
        ctx->cksum = false;
    }
    ~StateGuard() {
        cudaMemcpyAsync(ctx->d_win, win, (size_t)ctx->n_sets * ctx->N * 4, cudaMemcpyDeviceToDevice, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        ++ctx->state_epoch;  // the window went back: no speculative windows apply
        ctx->position = pos;
        ctx->cksum = cksum;
    }
};

uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }



// Words per stream per chunk: ~2^30 words (4 GB) per chunk over all streams, 2^16..2^24 per
// stream. Big chunks let the generator split streams into jump-ahead pieces across all SMs and
// amortise the per-call planning; the chunk is the stat pass's only large allocation.
uint64_t chunk_target(uint32_t S) {
    const uint64_t c = (1ull << 30) / std::max<uint32_t>(S, 1);
    return std::min<uint64_t>(std::max<uint64_t>(c, 1ull << 16), 1ull << 24);
}

void generate_chunk(mtgp_ctx* ctx, uint32_t* buf, uint64_t C) {
    const int rc = ctx_generate_device(ctx, MTGP_U32, buf, C);
    if (rc) throw Failure{rc};
}

// Bitmap generation is ALU-heavier than word output, so it wants every team slot: while a fused
// pass runs, auto-sized plans (min_piece_words == 0) cut pieces down to 2^19 words.
struct FusedPieces {
    mtgp_ctx* ctx;
    uint64_t saved;
    explicit FusedPieces(mtgp_ctx* c) : ctx(c), saved(c->min_piece_words) {
        if (!saved) ctx->min_piece_words = 1ull << 19;
    }
    ~FusedPieces() { ctx->min_piece_words = saved; }
};

// The generator can write the bit-0 bitmap instead of words: gen3 (MTGP32-11213) and mt_gen3
// (Engine::mt, n = 624) warp teams
bool bitmap_fusable(const mtgp_ctx* ctx, uint64_t C) {
    if (!ctx->planner || !ctx->planner->v2_supported() || C % 4 != 0) return false;
    if (ctx->engine == 0) return ctx->mexp == 11213 && (ctx->kernel == 0 || ctx->kernel == 3);
    // (the bitmap comes from cudaMalloc: any 256-byte aligned address stands in for it)
    return (ctx->kernel == 0 || ctx->kernel == 6) &&
           ctx->planner->mt3_supported(MTGP_U32, C, reinterpret_cast<const void*>(uintptr_t{256}));
}

void launched(mtgp_ctx* ctx, const char* what) {
    check(cudaGetLastError(), what);
    ctx->total_launches += 1;
}

std::vector<uint64_t> fetch(mtgp_ctx* ctx, const DevBuf& b, size_t n) {
    std::vector<uint64_t> h(n);
    check(cudaMemcpyAsync(h.data(), b.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H counts");
    check(cudaStreamSynchronize(ctx->stream), "sync");
    return h;
}

void run_walk(mtgp_ctx* ctx, const mtgp_stat_spec& sp, mtgp_stat_result* res) {
    const uint32_t S = ctx->n_sets, l = sp.l;
    if (l > (1u << 20)) throw std::invalid_argument("walk length l > 2^20 is not supported on the device path");
    const uint32_t wpt = std::max<uint32_t>(1, 8192 / l);
    const uint32_t tile_words = wpt * l;
    uint32_t tpc = (uint32_t)std::max<uint64_t>(2, chunk_target(S) / tile_words);
    tpc += tpc & 1;  // even: C % 4 == 0 (l is even) keeps the register-ring generator eligible
    const uint64_t C = (uint64_t)tpc * tile_words;
    const uint64_t chunks = ceil_div(sp.n, (uint64_t)tpc * wpt);
    const bool smem_hist = l + 1 <= 16384;
    const size_t smem = 4 * ((size_t)(tile_words + 31) / 32 + (smem_hist ? l + 1 : 0));
    DevBuf counts;
    Arena ar;
    ar.add(counts, (size_t)S * (l + 1) * 8);
    if (bitmap_fusable(ctx, C)) {
        // fused: the generator writes only the bit-0 bitmap (1/32 of the chunk's bytes), so the
        // chunk can be 32x longer for the same memory: all walks in one call when they fit in
        // 2^33 words over all streams (1 GB of bitmap). Long calls give every SM 6 CTAs of
        // generator pieces (FusedPieces), amortise the jump-ahead and skip per-chunk launches.
        // walk_bm_kernel indexes the chunk's bits in 32 bits: keep C < 2^32 words per stream
        const uint64_t tpc_max = ((1ull << 32) / tile_words - 1) & ~1ull;
        uint32_t tpc_f = (uint32_t)std::min<uint64_t>(ceil_div(sp.n, wpt),
                                                      std::max<uint64_t>(tpc, (1ull << 33) / S / tile_words));
        tpc_f = std::max<uint32_t>(2, tpc_f + (tpc_f & 1));
        tpc_f = (uint32_t)std::min<uint64_t>(tpc_f, tpc_max);
        const uint64_t C = (uint64_t)tpc_f * tile_words;
        const uint64_t chunks = ceil_div(sp.n, (uint64_t)tpc_f * wpt);
        const uint32_t tpc = tpc_f;
        FusedPieces fp(ctx);
        const uint64_t bm_stride = (C + 31) / 32;
        uint32_t* const bm = ar.commit(ctx, (size_t)S * bm_stride * 4);
        check(cudaMemsetAsync(counts.p, 0, (size_t)S * (l + 1) * 8, ctx->stream), "memset");
        auto kb = smem_hist ? walk_bm_kernel<true> : walk_bm_kernel<false>;
        const size_t smem_b = smem_hist ? 4 * (size_t)(l + 1) : 0;
        check(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b), "smem attribute");
        for (uint64_t c = 0; c < chunks; ++c) {
            check(cudaMemsetAsync(bm, 0, (size_t)S * bm_stride * 4, ctx->stream), "memset bitmap");
            const int rc = ctx_generate_bitmap(ctx, kKindBitmapBit0, bm, C, BitmapPred{});
            if (rc) throw Failure{rc};
            kb<<<dim3(tpc, S), kThreads, smem_b, ctx->stream>>>(bm, bm_stride, l, wpt, c * tpc * wpt, sp.n,
                                                               counts.as<unsigned long long>());
            launched(ctx, "walk bitmap kernel");
        }
        const auto h = fetch(ctx, counts, (size_t)S * (l + 1));
        for (uint32_t s = 0; s < S; ++s) {
            stat::finish(sp, h.data() + (size_t)s * (l + 1), res + s);
            res[s].words_used = stat::words_needed(sp);
        }
        return;
    }
    uint32_t* const wbuf = ar.commit(ctx, (size_t)S * C * 4);
    check(cudaMemsetAsync(counts.p, 0, (size_t)S * (l + 1) * 8, ctx->stream), "memset");
    auto k = smem_hist ? walk_kernel<true> : walk_kernel<false>;
    check(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attribute");
    for (uint64_t c = 0; c < chunks; ++c) {
        generate_chunk(ctx, wbuf, C);
        k<<<dim3(tpc, S), kThreads, smem, ctx->stream>>>(wbuf, C, l, wpt, c * tpc * wpt, sp.n,
                                                         counts.as<unsigned long long>());
        launched(ctx, "walk kernel");
    }
    const auto h = fetch(ctx, counts, (size_t)S * (l + 1));
    for (uint32_t s = 0; s < S; ++s) {
        stat::finish(sp, h.data() + (size_t)s * (l + 1), res + s);
        res[s].words_used = stat::words_needed(sp);
    }
}

uint32_t gcd32(uint32_t a, uint32_t b) {
    while (b) {
        const uint32_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

void run_hamming(mtgp_ctx* ctx, const mtgp_stat_spec& sp, mtgp_stat_result* res) {
    const uint32_t S = ctx->n_sets;
    // a pair of blocks is 2L bits; the smallest span that is whole words AND whole pairs is
    // 2L / g words = s / g pairs, g = gcd(2L, s)
    const uint64_t two_l = 2ull * sp.L;
    const uint32_t g = two_l > 0xFFFFFFFFull ? 1 : gcd32((uint32_t)two_l, sp.s);
    const uint64_t unit = two_l / g;
    if (unit > 8192)
        throw std::invalid_argument("hamming block pair spans more than 8192 words; not supported on the device path");
    const uint32_t units = std::max<uint32_t>(1, 8192 / (uint32_t)unit);
    const uint32_t tile_words = units * (uint32_t)unit;
    const uint32_t ppt = units * (sp.s / g);  // pairs per tile
    uint32_t tpc = (uint32_t)std::max<uint64_t>(4, chunk_target(S) / tile_words);
    tpc = (tpc + 3) & ~3u;  // C % 4 == 0
    const uint64_t C = (uint64_t)tpc * tile_words;
    const uint64_t npairs = sp.n / 2;
    const uint64_t chunks = ceil_div(npairs, (uint64_t)tpc * ppt);
    const size_t smem = 4 * (2 * (size_t)tile_words + 1);
    DevBuf table;
    Arena ar;
    ar.add(table, (size_t)S * 4 * 8);
    uint32_t* const wbuf = ar.commit(ctx, (size_t)S * C * 4);
    check(cudaMemsetAsync(table.p, 0, (size_t)S * 4 * 8, ctx->stream), "memset");
    check(cudaFuncSetAttribute(hamming_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attribute");
    const bool long_blocks = sp.L >= 32u * sp.s;  // >= 32 letters per block: warp per block
    const uint64_t pairs_chunk = (uint64_t)tpc * ppt;
    for (uint64_t c = 0; c < chunks; ++c) {
        generate_chunk(ctx, wbuf, C);
        if (long_blocks) {
            const uint32_t gx = (uint32_t)std::min<uint64_t>(ceil_div(pairs_chunk, kWarps), 1024);
            hamming_warp_kernel<<<dim3(gx, S), kThreads, 0, ctx->stream>>>(wbuf, C, sp.r, sp.s, sp.L, pairs_chunk,
                                                                           c * pairs_chunk, npairs,
                                                                           table.as<unsigned long long>());
        } else {
            hamming_kernel<<<dim3(tpc, S), kThreads, smem, ctx->stream>>>(wbuf, C, sp.r, sp.s, sp.L, ppt,
                                                                          tile_words, c * tpc * ppt, npairs,
                                                                          table.as<unsigned long long>());
        }
        launched(ctx, "hamming kernel");
    }
    const auto h = fetch(ctx, table, (size_t)S * 4);
    for (uint32_t s = 0; s < S; ++s) {
        stat::finish(sp, h.data() + (size_t)s * 4, res + s);
        res[s].words_used = stat::words_needed(sp);
    }
}

void run_opso(mtgp_ctx* ctx, const mtgp_stat_spec& sp, mtgp_stat_result* res) {
    const uint32_t S = ctx->n_sets;
    const uint64_t cells = 1ull << (2 * sp.s);
    const uint64_t bm_words = std::max<uint64_t>(1, cells / 32);
    const uint64_t W = sp.n + 1;
    const uint64_t C = std::min<uint64_t>(chunk_target(S), (W + 3) & ~3ull);
    const uint64_t chunks = ceil_div(W, C);
    DevBuf bitmap, prev, coll;
    Arena ar;
    ar.add(bitmap, (size_t)S * bm_words * 4);
    ar.add(prev, (size_t)S * 2 * 4);
    ar.add(coll, (size_t)S * 8);
    uint32_t* const wbuf = ar.commit(ctx, (size_t)S * C * 4);
    check(cudaMemsetAsync(bitmap.p, 0, (size_t)S * bm_words * 4, ctx->stream), "memset");
    check(cudaMemsetAsync(prev.p, 0, (size_t)S * 2 * 4, ctx->stream), "memset");
    check(cudaMemsetAsync(coll.p, 0, (size_t)S * 8, ctx->stream), "memset");
    const uint32_t gx = (uint32_t)std::min<uint64_t>(ceil_div(C, kThreads), 64);
    for (uint64_t c = 0; c < chunks; ++c) {
        generate_chunk(ctx, wbuf, C);
        uint32_t* carry = prev.as<uint32_t>();
        opso_kernel<<<dim3(gx, S), kThreads, 0, ctx->stream>>>(wbuf, C, c * C, sp.r, sp.s, sp.n,
                                                               bitmap.as<uint32_t>(), bm_words,
                                                               carry + (c & 1) * S, carry + ((c + 1) & 1) * S,
                                                               coll.as<unsigned long long>());
        launched(ctx, "opso kernel");
    }
    const auto h = fetch(ctx, coll, S);
    for (uint32_t s = 0; s < S; ++s) {
        stat::finish(sp, h.data() + s, res + s);
        res[s].words_used = W;
    }
}

void run_gap(mtgp_ctx* ctx, const mtgp_stat_spec& sp, mtgp_stat_result* res) {
    const uint32_t S = ctx->n_sets;
    const stat::GapShape g = stat::gap_shape(sp);
    const uint32_t tcut = (uint32_t)g.tcut;
    const double p = sp.beta - sp.alpha;
    uint64_t C = (chunk_target(S) + kGapTile - 1) / kGapTile * kGapTile;
    // Fused: the generator writes the hit bitmap itself (1/32 of the chunk's bytes), so one call
    // can cover the expected stream length (+5%) up to 2^33 words over all streams, with every SM
    // full of generator pieces (FusedPieces). The 32-bit hit test needs hi - lo >= 1, hi <= 2^32.
    const bool fused = bitmap_fusable(ctx, C) && g.hi > g.lo && g.hi <= (1ull << 32);
    if (fused) {
        const uint64_t want = (uint64_t)((double)(sp.n + 1) / p * 1.05) + kGapTile;
        // tile positions (GapTile.first/last, gap_hist_kernel) are 32-bit signed chunk offsets:
        // keep C <= 2^31 words per stream
        const uint64_t cap = std::min<uint64_t>(std::max<uint64_t>(C, (1ull << 33) / S), 1ull << 31);
        C = (std::min<uint64_t>(std::min<uint64_t>(std::max<uint64_t>(C, want), cap), g.budget + kGapTile - 1) +
             kGapTile - 1) / kGapTile * kGapTile;
    }
    const uint32_t T = (uint32_t)(C / kGapTile);
    const uint64_t max_chunks = ceil_div(g.budget, C);
    const uint64_t expected_chunks = std::max<uint64_t>(1, (uint64_t)((double)(sp.n + 1) / p / (double)C));
    const bool smem_hist = tcut + 1 <= 12288;
    const size_t smem = smem_hist ? 4 * ((size_t)tcut + 1) : 0;
    DevBuf counts, tiles, pre, state, end, hits;
    Arena ar;
    ar.add(hits, (size_t)S * (C / 32) * 4);
    ar.add(counts, (size_t)S * (tcut + 1) * 8);
    ar.add(tiles, (size_t)S * T * sizeof(GapTile));
    ar.add(pre, (size_t)S * T * sizeof(GapPre));
    ar.add(state, (size_t)S * sizeof(GapState));
    ar.add(end, (size_t)S * 8);
    uint32_t* const wbuf = ar.commit(ctx, fused ? 256 : (size_t)S * C * 4);
    FusedPieces fp(ctx);
    if (!fused) ctx->min_piece_words = fp.saved;
    check(cudaMemsetAsync(counts.p, 0, (size_t)S * (tcut + 1) * 8, ctx->stream), "memset");
    std::vector<GapState> hs(S, GapState{0, -1, 0, 0, 0});
    check(cudaMemcpyAsync(state.p, hs.data(), S * sizeof(GapState), cudaMemcpyHostToDevice, ctx->stream), "H2D state");
    auto hk = smem_hist ? gap_hist_kernel<true> : gap_hist_kernel<false>;
    if (smem > 48 * 1024)
        check(cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attribute");
    for (uint64_t c = 0; c < max_chunks; ++c) {
        const uint64_t P = c * C;
        if (fused) {
            check(cudaMemsetAsync(hits.p, 0, (size_t)S * (C / 32) * 4, ctx->stream), "memset hits");
            BitmapPred pred;
            pred.mask = g.mask;
            pred.lo = (uint32_t)g.lo;
            pred.span_m1 = (uint32_t)(g.hi - g.lo - 1);
            const int rc = ctx_generate_bitmap(ctx, kKindBitmapRange, hits.as<uint32_t>(), C, pred);
            if (rc) throw Failure{rc};
            gap_count_bm_kernel<<<dim3(T, S), kGapBmThreads, 0, ctx->stream>>>(
                hits.as<uint32_t>(), C, P, g.budget, state.as<GapState>(), tiles.as<GapTile>(), T);
            launched(ctx, "gap count bitmap kernel");
        } else {
            generate_chunk(ctx, wbuf, C);
            gap_count_kernel<<<dim3(T, S), kThreads, 0, ctx->stream>>>(wbuf, C, P, g.mask, g.lo, g.hi, g.budget,
                                                                       state.as<GapState>(), tiles.as<GapTile>(), T,
                                                                       hits.as<uint32_t>());
            launched(ctx, "gap count kernel");
        }
        gap_scan_kernel<<<S, kThreads, 0, ctx->stream>>>(tiles.as<GapTile>(), T, P, state.as<GapState>(),
                                                         pre.as<GapPre>());
        launched(ctx, "gap scan kernel");
        hk<<<dim3(std::min<uint32_t>(T, kGapHistCtas), S), kHistThreads, smem, ctx->stream>>>(
                                                        hits.as<uint32_t>(), C, P, state.as<GapState>(),
                                                        tiles.as<GapTile>(), pre.as<GapPre>(), T, sp.n, tcut,
                                                        counts.as<unsigned long long>(), end.as<unsigned long long>());
        launched(ctx, "gap hist kernel");
        gap_update_kernel<<<(S + 127) / 128, 128, 0, ctx->stream>>>(S, P, C, g.budget, sp.n,
                                                                    end.as<unsigned long long>(), state.as<GapState>());
        launched(ctx, "gap update kernel");
        // poll for completion around the expected length, sparsely before it
        if (c + 1 >= expected_chunks && ((c + 1 - expected_chunks) % 2 == 0 || c + 1 == max_chunks)) {
            check(cudaMemcpyAsync(hs.data(), state.p, S * sizeof(GapState), cudaMemcpyDeviceToHost, ctx->stream), "D2H state");
            check(cudaStreamSynchronize(ctx->stream), "sync");
            if (std::all_of(hs.begin(), hs.end(), [](const GapState& x) { return x.done != 0; })) break;
        }
    }
    check(cudaMemcpyAsync(hs.data(), state.p, S * sizeof(GapState), cudaMemcpyDeviceToHost, ctx->stream), "D2H state");
    const auto h = fetch(ctx, counts, (size_t)S * (tcut + 1));
    for (uint32_t s = 0; s < S; ++s) {
        res[s] = mtgp_stat_result{};
        if (!hs[s].done || hs[s].exhausted) {
            res[s].error = MTGP_STAT_EXHAUSTED;
            res[s].words_used = g.budget;
            continue;
        }
        stat::finish(sp, h.data() + (size_t)s * (tcut + 1), res + s);
        res[s].words_used = hs[s].end + 1;
    }
}

}  // namespace
}  // namespace mtgpb

extern "C" int mtgp_stat_run(mtgp_ctx* ctx, const mtgp_stat_spec* spec, mtgp_stat_result* results) {
    using namespace mtgpb;
    if (!ctx || !spec || !results) return set_error(MTGP_EINVAL, "null argument");
    try {
        stat::validate(*spec);
    } catch (const std::invalid_argument& e) {
        return set_error(MTGP_EINVAL, "%s", e.what());
    }
    if (ctx->n_sets > 65535) return set_error(MTGP_EINVAL, "stat tests support at most 65535 streams per context");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    std::memset(results, 0, sizeof(mtgp_stat_result) * ctx->n_sets);
    try {
        StateGuard guard(ctx);
        switch (spec->test) {
            case MTGP_STAT_GAP: run_gap(ctx, *spec, results); break;
            case MTGP_STAT_HAMMING_INDEP: run_hamming(ctx, *spec, results); break;
            case MTGP_STAT_COLLISION_OVER: run_opso(ctx, *spec, results); break;
            case MTGP_STAT_RANDOM_WALK: run_walk(ctx, *spec, results); break;
        }
    } catch (const Failure& f) {
        return f.code;
    } catch (const std::invalid_argument& x) {
        return set_error(MTGP_EINVAL, "%s", x.what());
    }
    return MTGP_OK;
}
