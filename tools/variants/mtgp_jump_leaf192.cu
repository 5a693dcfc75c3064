// tools/variants/mtgp_jump_leaf192.cu -- the Karatsuba jump templated on the leaf width (KJ = 12: 384-output
// leaves, KJ = 6: 192-output leaves one level deeper, MTGP_OPT_JUMP 3). Bit-exact (tests passed)
// but slower: 3.49 vs 2.75 ms per C4-44497 call, 1.59 vs 1.32 at 23209 (8-byte loads: 3.2x the
// load instructions per output). Needs the KaraPlan arrays sized for d <= 3 (27 leaves).
// mtgp_jump.cu -- jump-ahead windows by a transposed-Karatsuba middle product (large N).
//
// A jump computes the window at offset o of a stream: y_j = XOR_{i : q_i = 1} x_{i+j}, j < N,
// where q = x^(o - t0) mod P (mtgp_plan.cu) and x is the stream's state-word prefix from the
// reference point t0. jump_flat_kernel (mtgp_v2.cu) does this directly: N * M word operations
// per piece, which at MTGP32-44497 (N = 1391, M = 44497) is 16% of a bench step.
//
// Here the output range is padded to n_out = 384 * 2^d >= N (d = 1 for N <= 768, 2 for
// N <= 1536) and q is cut into B blocks of n_out bits, so y = XOR_b MP(Q_b, x[b n_out ..]),
// MP(a, z)_j = XOR_i a_i z_{i+j} being a middle product of size n_out. Each MP is split d
// times by the transposed Karatsuba identity (for halves a0, a1 of a and z windows Z0, Z1, Z2
// at offsets 0, m/2, m):
//     y_lo = P ^ L,  y_hi = P ^ H,  P = MP(a0 ^ a1, Z1),  L = MP(a0, Z0 ^ Z1),  H = MP(a1, Z1 ^ Z2)
// so one size-n_out product becomes 3^d size-384 "leaf" products instead of 4^d: 0.75x the
// word operations at d = 1, 0.56x at d = 2. Everything is GF(2)-linear, so the leaves are
// summed over the blocks first and recombined once per piece.
//
//   jump_ztrans_kernel  per prefix row (stream): the leaf z vectors of every block, each an
//                       XOR of up to 2^d shifted prefix windows (shared by all pieces of the
//                       stream).
//   jump_qleaf_kernel   per piece: every leaf's q words (XORs of up to 2^d raw q words).
//   jump_leaf_kernel    one warp per (piece, leaf): the flat kernel's inner loop (lane keeps
//                       12 outputs, q walked two bits at a time, warp-uniform branches) over
//                       the leaf's B * 12 q words.
//   jump_combine_kernel per piece: window word j = XOR of the 2^d leaf outputs of its quarter.
#include <algorithm>
#include <vector>

#include "mtgp_jump.cuh"

namespace mtgpb {

#define FULL 0xffffffffu

namespace {

// Leaf geometry for KJ outputs per lane: KH = 32 KJ outputs per warp (384 or 192), z vectors of
// KZ = 2 KH words, KJ q words per leaf block.
template <int KJ>
struct LeafG {
    static constexpr uint32_t KH = 32 * KJ;
    static constexpr uint32_t KZ = 2 * KH;
    static constexpr uint32_t KHQ = KH / 32;
};
#ifndef MTGP_LEAF_WARPS
#define MTGP_LEAF_WARPS 4
#endif
#ifndef MTGP_LEAF_MINB
#define MTGP_LEAF_MINB 7
#endif
// 7 CTAs of 4 warps per SM (72 registers, no spills): 6 CTAs at 76 registers were 13% slower,
// 8 CTAs (64 registers, spilling) the same (profiles/r1_leaf_sweep.jsonl, r1_jump_sweep.jsonl)
constexpr int kLeafWarps = MTGP_LEAF_WARPS;

template <int KJ>
__global__ void jump_ztrans_kernel(const JumpArgs a, const KaraPlan k, uint32_t n_rows, uint4* __restrict__ zbuf) {
    constexpr uint32_t kZ = LeafG<KJ>::KZ;
    // one thread per 4 output words: index over (row, block, leaf, t4)
    const uint64_t per_row = (uint64_t)k.blocks * k.n_leaf * (kZ / 4);
    const uint64_t total = per_row * n_rows;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t row = (uint32_t)(i / per_row);
        const uint32_t r = (uint32_t)(i % per_row);
        const uint32_t t4 = r % (kZ / 4);
        const uint32_t bl = r / (kZ / 4);
        const uint32_t s = bl % k.n_leaf, b = bl / k.n_leaf;
        const uint4* x4 = reinterpret_cast<const uint4*>(a.pre + (size_t)row * a.pre_stride + a.pre_off);
        const uint32_t base = b * k.n_out + 4 * t4;
        uint4 v = make_uint4(0, 0, 0, 0);
        for (uint32_t u = 0; u < k.nz[s]; ++u) {
            const uint4 g = __ldg(x4 + ((base + k.oz[s][u]) >> 2));
            v.x ^= g.x;
            v.y ^= g.y;
            v.z ^= g.z;
            v.w ^= g.w;
        }
        zbuf[i] = v;
    }
}

// Leaf q words of every (job, leaf, block): XORs of up to 2^d raw q words (one thread per word).
template <int KJ>
__global__ void jump_qleaf_kernel(const JumpArgs a, const KaraPlan k, uint32_t* __restrict__ qleaf) {
    constexpr uint32_t kHq = LeafG<KJ>::KHQ;
    const uint64_t per_job = (uint64_t)k.n_leaf * k.blocks * kHq;
    const uint64_t total = per_job * a.n_jobs;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t job = (uint32_t)(i / per_job);
        const uint32_t r = (uint32_t)(i % per_job);
        const uint32_t w = r % kHq, bs = r / kHq;
        const uint32_t b = bs % k.blocks, s = bs / k.blocks;
        const uint32_t* q = a.q + (size_t)a.jobs[job].q * a.q_words;
        uint32_t v = 0;
        for (uint32_t u = 0; u < k.nq[s]; ++u) {
            const uint32_t idx = b * k.blk_qwords + k.oq[s][u] + w;
            if (idx < a.q_words) v ^= __ldg(q + idx);
        }
        qleaf[i] = v;
    }
}

// The KJ + 32 z words a lane reads for one q word: 16-byte loads for KJ = 12 (its first word is a
// multiple of 4), 8-byte loads for KJ = 6 (a multiple of 2).
template <int KJ>
__device__ __forceinline__ void load_w(const uint32_t* z, uint32_t (&w)[KJ + 32]) {
    if constexpr (KJ % 4 == 0) {
        const uint4* z4 = reinterpret_cast<const uint4*>(z);
#pragma unroll
        for (int v = 0; v < (KJ + 32) / 4; ++v) {
            const uint4 g = __ldg(z4 + v);
            w[4 * v] = g.x;
            w[4 * v + 1] = g.y;
            w[4 * v + 2] = g.z;
            w[4 * v + 3] = g.w;
        }
    } else {
        const uint2* z2 = reinterpret_cast<const uint2*>(z);
#pragma unroll
        for (int v = 0; v < (KJ + 32) / 2; ++v) {
            const uint2 g = __ldg(z2 + v);
            w[2 * v] = g.x;
            w[2 * v + 1] = g.y;
        }
    }
}

template <bool DIRECT, int KJ>
__global__ void __launch_bounds__(kLeafWarps * 32, MTGP_LEAF_MINB) jump_leaf_kernel(const JumpArgs a, const KaraPlan k,
                                                                                  const uint32_t* __restrict__ qleaf,
                                                                                  const uint32_t* __restrict__ zbuf,
                                                                                  uint32_t* __restrict__ leaf_out) {
    constexpr uint32_t kH = LeafG<KJ>::KH, kZ = LeafG<KJ>::KZ, kHq = LeafG<KJ>::KHQ;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t unit = blockIdx.x * kLeafWarps + warp;  // (job, leaf, group)
    const uint32_t g = unit % k.groups, js = unit / k.groups;
    const uint32_t job = js / k.n_leaf, s = js % k.n_leaf;
    if (job >= a.n_jobs) return;
    const uint32_t row = a.jobs[job].row;
    const uint32_t jl = KJ * lane;
    // this group's blocks [b0, b1) of the leaf
    const uint32_t per = (k.blocks + k.groups - 1) / k.groups;
    const uint32_t b0 = min(k.blocks, g * per), b1 = min(k.blocks, b0 + per);
    // z vector of block b: d = 0 reads the prefix itself (x[b * KH, b * KH + 2 KH)); d >= 1 the
    // transformed vectors (one per block, n_leaf * KZ words apart)
    const uint32_t* zs;
    uint32_t zstride;
    if (DIRECT) {
        zs = a.pre + (size_t)row * a.pre_stride + a.pre_off + jl;
        zstride = k.n_out;
    } else {
        zs = zbuf + ((size_t)row * k.blocks * k.n_leaf + s) * kZ + jl;
        zstride = k.n_leaf * kZ;
    }
    zs += (size_t)b0 * zstride;
    const uint32_t total = (b1 - b0) * kHq;
    const uint32_t* ql = qleaf + (size_t)js * k.blocks * kHq + b0 * kHq;
    uint32_t acc[KJ];
#pragma unroll
    for (int i = 0; i < KJ; ++i) acc[i] = 0;
    // zb: the current block's z vector; iw: q word within the block
    const uint32_t* zb = zs;
    uint32_t iw = 0;
    for (uint32_t f0 = 0; f0 < total; f0 += 32) {
        const uint32_t qmine = f0 + lane < total ? __ldg(ql + f0 + lane) : 0u;
        const uint32_t nw = min(32u, total - f0);
        for (uint32_t k32 = 0; k32 < nw; ++k32) {
            // the q word as a warp reduction: REDUX writes a uniform register, so the 2-bit pattern
            // dispatch below runs on the uniform datapath (UISETP / ULOP3 / USHF) instead of
            // vector ISETPs and BSSY/BSYNC pairs; with a SHFL the compiler kept it per-lane.
            // Leaf jump 3.12 -> 2.68 ms per C4-44497 call, 1.45 -> 1.28 at 23209, 1.38 -> 1.17
            // for MT19937 (profiles/r2/jump_leaf_uniform_sweep.jsonl)
            const uint32_t qw = __reduce_or_sync(FULL, lane == k32 ? qmine : 0u);
            if (qw != 0) {
                uint32_t w[KJ + 32];
                load_w<KJ>(zb + iw * 32, w);
#pragma unroll
                for (int bb = 0; bb < 32; bb += 2) {
                    const uint32_t pat = (qw >> bb) & 3u;
                    if (pat == 1) {
#pragma unroll
                        for (int i = 0; i < KJ; ++i) acc[i] ^= w[bb + i];
                    } else if (pat == 2) {
#pragma unroll
                        for (int i = 0; i < KJ; ++i) acc[i] ^= w[bb + 1 + i];
                    } else if (pat == 3) {
#pragma unroll
                        for (int i = 0; i < KJ; ++i) acc[i] ^= w[bb + i] ^ w[bb + 1 + i];
                    }
                }
            }
            if (++iw == kHq) {
                iw = 0;
                zb += zstride;
            }
        }
    }
    uint32_t* dst = leaf_out + (size_t)unit * kH + jl;
    if constexpr (KJ % 4 == 0) {
#pragma unroll
        for (int v = 0; v < KJ / 4; ++v)
            reinterpret_cast<uint4*>(dst)[v] = make_uint4(acc[4 * v], acc[4 * v + 1], acc[4 * v + 2], acc[4 * v + 3]);
    } else {
#pragma unroll
        for (int v = 0; v < KJ / 2; ++v) reinterpret_cast<uint2*>(dst)[v] = make_uint2(acc[2 * v], acc[2 * v + 1]);
    }
}

template <int KJ>
__global__ void jump_combine_kernel(const JumpArgs a, const KaraPlan k, uint32_t N, const uint32_t* __restrict__ leaf_out) {
    constexpr uint32_t kH = LeafG<KJ>::KH;
    const uint32_t job = blockIdx.y;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    const JumpJob jb = a.jobs[job];
    const uint32_t c = t / kH, tt = t % kH;
    const uint32_t* lo = leaf_out + (size_t)job * k.n_leaf * k.groups * kH + tt;
    uint32_t v = 0;
    for (uint32_t u = 0; u < k.n_comb; ++u)
        for (uint32_t g = 0; g < k.groups; ++g) v ^= lo[((size_t)k.comb[c][u] * k.groups + g) * kH];
    a.piece_win[(size_t)jb.piece * N + t] = v;
}

template <int KJ>
cudaError_t launch_kara_t(const JumpArgs& a, const KaraPlan& k, uint32_t N, uint32_t n_rows, uint32_t* zbuf,
                          uint32_t* leaf_out, cudaStream_t st) {
    constexpr uint32_t kH = LeafG<KJ>::KH, kZ = LeafG<KJ>::KZ, kHq = LeafG<KJ>::KHQ;
    if (k.depth > 0) {  // d = 0 reads its z windows straight from the prefix
        const uint64_t total = (uint64_t)n_rows * k.blocks * k.n_leaf * (kZ / 4);
        const uint32_t grid = (uint32_t)std::min<uint64_t>((total + 255) / 256, 148u * 16u);
        jump_ztrans_kernel<KJ><<<grid, 256, 0, st>>>(a, k, n_rows, reinterpret_cast<uint4*>(zbuf));
    }
    uint32_t* qleaf = leaf_out + (size_t)a.n_jobs * k.n_leaf * k.groups * kH;
    {
        const uint64_t total = (uint64_t)a.n_jobs * k.n_leaf * k.blocks * kHq;
        const uint32_t grid = (uint32_t)std::min<uint64_t>((total + 255) / 256, 148u * 16u);
        jump_qleaf_kernel<KJ><<<grid, 256, 0, st>>>(a, k, qleaf);
    }
    {
        const uint32_t units = a.n_jobs * k.n_leaf * k.groups;
        auto kern = k.depth == 0 ? jump_leaf_kernel<true, KJ> : jump_leaf_kernel<false, KJ>;
        kern<<<(units + kLeafWarps - 1) / kLeafWarps, kLeafWarps * 32, 0, st>>>(a, k, qleaf, zbuf, leaf_out);
    }
    {
        const dim3 grid((N + 255) / 256, a.n_jobs);
        jump_combine_kernel<KJ><<<grid, 256, 0, st>>>(a, k, N, leaf_out);
    }
    return cudaGetLastError();
}

}  // namespace

bool kara_plan(uint32_t N, uint32_t q_words, int depth_override, KaraPlan& k, uint32_t leaf_j) {
    if (leaf_j != 12 && leaf_j != 6) return false;
    const uint32_t kH = 32 * leaf_j;
    int d = depth_override;
    if (d < 0)
        for (d = 0; d < 3 && (kH << d) < N; ++d) {
        }
    if (d < 0 || d > 3 || (kH << d) < N) return false;
    k = KaraPlan{};
    k.leaf_j = leaf_j;
    k.depth = (uint32_t)d;
    k.n_out = kH << d;
    k.blk_qwords = k.n_out / 32;
    k.blocks = (32 * q_words + k.n_out - 1) / k.n_out;
    // leaves: base-3 digits s_1..s_d (level 1 most significant), P = 0, L = 1, H = 2.
    // Offsets (in words) of the z windows XORed into a leaf's z vector and of the raw q words
    // XORed into its q words; each level halves the size m.
    k.n_leaf = 1;
    for (int i = 0; i < d; ++i) k.n_leaf *= 3;
    for (uint32_t s = 0; s < k.n_leaf; ++s) {
        std::vector<uint32_t> oz{0}, oq{0};
        uint32_t m = k.n_out, rest = s, div = k.n_leaf / 3;
        auto sym = [](std::vector<uint32_t> v) {  // multiset mod 2
            std::sort(v.begin(), v.end());
            std::vector<uint32_t> o;
            for (size_t i = 0; i < v.size();) {
                size_t j = i;
                while (j < v.size() && v[j] == v[i]) ++j;
                if ((j - i) & 1) o.push_back(v[i]);
                i = j;
            }
            return o;
        };
        for (int lev = 0; lev < d; ++lev) {
            const uint32_t dig = rest / div;
            rest %= div;
            div = div ? div / 3 : 0;
            const uint32_t half = m / 2;
            std::vector<uint32_t> nz, nqv;
            if (dig == 0) {  // P = MP(a0 ^ a1, Z1)
                for (uint32_t o : oz) nz.push_back(o + half);
                for (uint32_t o : oq) nqv.push_back(o), nqv.push_back(o + half);
            } else if (dig == 1) {  // L = MP(a0, Z0 ^ Z1)
                for (uint32_t o : oz) nz.push_back(o), nz.push_back(o + half);
                nqv = oq;
            } else {  // H = MP(a1, Z1 ^ Z2)
                for (uint32_t o : oz) nz.push_back(o + half), nz.push_back(o + m);
                for (uint32_t o : oq) nqv.push_back(o + half);
            }
            oz = sym(nz);
            oq = sym(nqv);
            m = half;
        }
        if (oz.size() > 8 || oq.size() > 8) return false;
        k.nz[s] = (uint32_t)oz.size();
        k.nq[s] = (uint32_t)oq.size();
        for (size_t i = 0; i < oz.size(); ++i) k.oz[s][i] = oz[i];
        for (size_t i = 0; i < oq.size(); ++i) k.oq[s][i] = oq[i] / 32;
    }
    // output quarter c (d bits, level 1 most significant): XOR of the leaves whose digit at
    // every level is P or (bit ? H : L)
    k.n_comb = 1u << d;
    for (uint32_t c = 0; c < (1u << d); ++c)
        for (uint32_t pick = 0; pick < (1u << d); ++pick) {
            uint32_t s = 0;
            for (int lev = 0; lev < d; ++lev) {
                const uint32_t bit = (c >> (d - 1 - lev)) & 1u;
                const uint32_t dig = ((pick >> (d - 1 - lev)) & 1u) ? (bit ? 2u : 1u) : 0u;
                s = s * 3 + dig;
            }
            k.comb[c][pick] = s;
        }
    return true;
}

uint32_t kara_prefix_words(const KaraPlan& k) {
    // the last block's windows reach x[(B + 1) n_out - 1]
    return (k.blocks + 1) * k.n_out;
}

size_t kara_zbuf_words(const KaraPlan& k, uint32_t n_rows) {
    return (size_t)n_rows * k.blocks * k.n_leaf * (64 * k.leaf_j);  // z vectors of 2 * 32 * leaf_j words
}
size_t kara_leaf_words(const KaraPlan& k, uint32_t n_jobs) {
    // partial leaf outputs (n_leaf * G * 32 leaf_j words per job), then the leaf q words
    // (n_leaf * B * leaf_j)
    return (size_t)n_jobs * k.n_leaf * ((size_t)k.groups * 32 * k.leaf_j + (size_t)k.blocks * k.leaf_j);
}

uint32_t kara_groups(const KaraPlan& k, uint32_t n_jobs, int num_sms) {
    // MTGP_LEAF_MINB CTAs x 4 warps per SM resident; at least 4 blocks per group
    const uint64_t want = (uint64_t)num_sms * MTGP_LEAF_MINB * kLeafWarps;
    const uint64_t have = std::max<uint64_t>(1, (uint64_t)n_jobs * k.n_leaf);
    const uint32_t g = (uint32_t)std::min<uint64_t>((want + have - 1) / have, std::max<uint32_t>(1, k.blocks / 4));
    return std::max<uint32_t>(1, g);
}

cudaError_t launch_jump_kara(const JumpArgs& a, const KaraPlan& k, uint32_t N, uint32_t n_rows, uint32_t* zbuf,
                             uint32_t* leaf_out, cudaStream_t st) {
    if (a.n_jobs == 0 || n_rows == 0) return cudaSuccess;
    return k.leaf_j == 6 ? launch_kara_t<6>(a, k, N, n_rows, zbuf, leaf_out, st)
                         : launch_kara_t<12>(a, k, N, n_rows, zbuf, leaf_out, st);
}

}  // namespace mtgpb
