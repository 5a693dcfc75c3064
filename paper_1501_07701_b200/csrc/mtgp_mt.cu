// mtgp_mt.cu -- the reference's own generic MT engine (Engine::mt) on the B200.
//
// Reference semantics (proj/src/generator.cpp): seeding :37-52, refill :68-88, temper :7-13,
// next_u32 = temper of the refilled state in order (generator.hpp:33-36). In sequence form,
// with x_0..x_{n-1} the seeded state:
//     y       = (x_i & upper) | (x_{i+1} & lower)          upper = 0xFFFFFFFF << r
//     x_{i+n} = x_{i+m} ^ (y >> 1) ^ (y & 1 ? a : 0)
//     out_i   = temper(x_{i+n})
// Any d <= n - m consecutive new words are independent (x_{i+m} is at distance n - m), so a
// CTA per stream computes d = min(256, n - m) words per pass from a shared-memory ring of
// >= n + d words with one barrier per pass -- the block-per-stream shape of the MTGP paper,
// applied to the reference's recurrence. Tempering (u, s, t, l, b, c are per status) and the
// float conversions are fused; checksums are accumulated like the MTGP kernels.
#include "mtgp_mt.cuh"
#include "mtgp_v2.cuh"

namespace mtgpb {

template <int KIND, bool CK>
__global__ void __launch_bounds__(256) mt_v1_kernel(const DevMtParams* __restrict__ params, uint32_t* __restrict__ win,
                                                   uint32_t nmax, uint32_t ring_mask, void* __restrict__ out,
                                                   uint64_t L, DevCksum* __restrict__ ck) {
    extern __shared__ uint32_t ring[];
    __shared__ unsigned long long s_sum;
    __shared__ unsigned int s_xor;
    const uint32_t set = blockIdx.x;
    const uint32_t t = threadIdx.x;
    const DevMtParams p = params[set];
    const uint32_t n = p.n, m = p.m;
    const uint32_t upper = p.r ? (0xFFFFFFFFu << p.r) : 0xFFFFFFFFu;
    const uint32_t lower = ~upper;
    uint32_t* w = win + (size_t)set * nmax;
    for (uint32_t j = t; j < n; j += blockDim.x) ring[j] = w[j];
    if (t == 0) {
        s_sum = 0;
        s_xor = 0;
    }
    __syncthreads();
    const uint32_t d = min((uint32_t)blockDim.x, n - m);
    uint32_t* o = reinterpret_cast<uint32_t*>(out) + (size_t)set * L;
    unsigned long long sum = 0;
    uint32_t xr = 0;
    for (uint64_t base = 0; base < L; base += d) {
        const uint32_t i = (uint32_t)base + t;
        if (t < d && base + t < L) {
            const uint32_t y = (ring[i & ring_mask] & upper) | (ring[(i + 1) & ring_mask] & lower);
            const uint32_t x = ring[(i + m) & ring_mask] ^ (y >> 1) ^ ((y & 1u) ? p.a : 0u);
            ring[(i + n) & ring_mask] = x;
            uint32_t v = x;
            v ^= v >> p.u;
            v ^= (v << p.s) & p.b;
            v ^= (v << p.t) & p.c;
            v ^= v >> p.l;
            if (KIND == MTGP_F64_01) {
                // Generator::next_f64_01: u32 * 2^-32 (proj/include/twistsieve/generator.hpp:39-41)
                __stcs(reinterpret_cast<double*>(out) + (size_t)set * L + base + t, (double)v * 0x1p-32);
            } else {
                if (KIND != MTGP_U32) {
                    v = (v >> 9) | 0x3F800000u;
                    if (KIND == MTGP_F32_01OC) v = __float_as_uint(2.0f - __uint_as_float(v));
                }
                __stcs(o + base + t, v);
            }
            if (CK) {
                sum += v;
                xr ^= v;
            }
        }
        __syncthreads();
    }
    for (uint32_t j = t; j < n; j += blockDim.x) w[j] = ring[((uint32_t)L + j) & ring_mask];
    if (CK) {
        for (int sft = 16; sft > 0; sft >>= 1) {
            sum += __shfl_xor_sync(0xffffffffu, sum, sft);
            xr ^= __shfl_xor_sync(0xffffffffu, xr, sft);
        }
        if ((t & 31) == 0) {
            atomicAdd(&s_sum, sum);
            atomicXor(&s_xor, xr);
        }
        __syncthreads();
        if (t == 0) {
            atomicAdd(&ck[set].sum64, s_sum);
            atomicXor(&ck[set].xor32, s_xor);
            atomicAdd(&ck[set].words, (unsigned long long)L);
        }
    }
}

template <int KIND, bool CK>
static cudaError_t launch_mt_t(const DevMtParams* params, uint32_t* win, uint32_t n_sets, uint32_t nmax, void* out,
                               uint64_t L, DevCksum* ck, cudaStream_t st) {
    const uint32_t R = next_pow2(nmax + 256);
    const size_t smem = (size_t)R * 4;
    auto k = mt_v1_kernel<KIND, CK>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<n_sets, 256, smem, st>>>(params, win, nmax, R - 1, out, L, ck);
    return cudaGetLastError();
}

cudaError_t launch_mt_v1(int kind, bool cksum, const DevMtParams* params, uint32_t* win, uint32_t n_sets,
                         uint32_t nmax, void* out, uint64_t L, DevCksum* ck, cudaStream_t st) {
    switch (kind * 2 + (cksum ? 1 : 0)) {
        case 0: return launch_mt_t<MTGP_U32, false>(params, win, n_sets, nmax, out, L, ck, st);
        case 1: return launch_mt_t<MTGP_U32, true>(params, win, n_sets, nmax, out, L, ck, st);
        case 2: return launch_mt_t<MTGP_F32_12, false>(params, win, n_sets, nmax, out, L, ck, st);
        case 3: return launch_mt_t<MTGP_F32_12, true>(params, win, n_sets, nmax, out, L, ck, st);
        case 4: return launch_mt_t<MTGP_F32_01OC, false>(params, win, n_sets, nmax, out, L, ck, st);
        case 5: return launch_mt_t<MTGP_F32_01OC, true>(params, win, n_sets, nmax, out, L, ck, st);
        case 6: return launch_mt_t<MTGP_F64_01, false>(params, win, n_sets, nmax, out, L, ck, st);
        case 7: return launch_mt_t<MTGP_F64_01, true>(params, win, n_sets, nmax, out, L, ck, st);
    }
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------------------------
// Jump-ahead support: raw state words (no tempering) of each split stream, from its window.
__global__ void __launch_bounds__(256) mt_prefix_kernel(const DevMtParams* __restrict__ params,
                                                        const uint32_t* __restrict__ win,
                                                        const uint32_t* __restrict__ sets, uint32_t n_stride,
                                                        uint32_t ring_mask, uint32_t* __restrict__ pre, uint32_t len) {
    extern __shared__ uint32_t ring[];
    const uint32_t row = blockIdx.x, t = threadIdx.x;
    const uint32_t set = sets[row];
    const DevMtParams p = params[set];
    const uint32_t n = p.n, m = p.m;
    const uint32_t upper = p.r ? (0xFFFFFFFFu << p.r) : 0xFFFFFFFFu, lower = ~upper;
    const uint32_t* w = win + (size_t)set * n_stride;
    uint32_t* o = pre + (size_t)row * len;
    for (uint32_t j = t; j < n; j += blockDim.x) {
        ring[j] = w[j];
        o[j] = w[j];
    }
    __syncthreads();
    const uint32_t d = min((uint32_t)blockDim.x, n - m);
    for (uint32_t base = 0; base + n < len; base += d) {
        const uint32_t i = base + t;
        if (t < d && i + n < len) {
            const uint32_t y = (ring[i & ring_mask] & upper) | (ring[(i + 1) & ring_mask] & lower);
            const uint32_t x = ring[(i + m) & ring_mask] ^ (y >> 1) ^ ((y & 1u) ? p.a : 0u);
            ring[(i + n) & ring_mask] = x;
            o[i + n] = x;
        }
        __syncthreads();
    }
}

cudaError_t launch_mt_prefix(const DevMtParams* params, const uint32_t* win, const uint32_t* sets, uint32_t n_rows,
                             uint32_t n, uint32_t* pre, uint32_t len, cudaStream_t st) {
    if (n_rows == 0) return cudaSuccess;
    const uint32_t R = next_pow2(n + 256);
    cudaError_t e = cudaFuncSetAttribute(mt_prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(R * 4));
    if (e != cudaSuccess) return e;
    mt_prefix_kernel<<<n_rows, 256, R * 4, st>>>(params, win, sets, n, R - 1, pre, len);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Warp teams over jump-ahead pieces. A warp keeps its piece's state in a private ring of
// R = next_pow2(n + 256) words, MIRRORED (2R words: every new word is also written R slots up),
// so the three reads of a word index without wrap masks. Each step makes D = 32K new words,
// D = min(256, n - m rounded down to 32) (any n - m consecutive words are independent); lane l
// takes words l, l + 32, ..., so ring accesses and HBM stores are coalesced. K is a template
// parameter (1..8): the strip loop unrolls, full steps carry no bounds checks, one __syncwarp
// per step.
template <int KIND, bool CK, int K>
__device__ __forceinline__ void mt_piece(const DevMtParams& p, uint32_t* ring, uint32_t ring_mask, uint32_t n,
                                         uint32_t lane, uint32_t* optr, uint32_t len, unsigned long long& sum,
                                         uint32_t& xr) {
    const uint32_t m = p.m, R = ring_mask + 1;
    const uint32_t upper = p.r ? (0xFFFFFFFFu << p.r) : 0xFFFFFFFFu, lower = ~upper;
    auto word = [&](uint32_t i, bool store) {
        const uint32_t* q = ring + (i & ring_mask);  // q[0], q[1], q[m] stay inside the mirror
        const uint32_t y = (q[0] & upper) | (q[1] & lower);
        const uint32_t x = q[m] ^ (y >> 1) ^ ((y & 1u) ? p.a : 0u);
        const uint32_t w = (i + n) & ring_mask;
        ring[w] = x;
        ring[w + R] = x;
        if (store) {
            uint32_t v = x;  // temper (generator.cpp:7-13)
            v ^= v >> p.u;
            v ^= (v << p.s) & p.b;
            v ^= (v << p.t) & p.c;
            v ^= v >> p.l;
            if (KIND != MTGP_U32) {
                v = (v >> 9) | 0x3F800000u;
                if (KIND == MTGP_F32_01OC) v = __float_as_uint(2.0f - __uint_as_float(v));
            }
            __stcs(optr + i, v);
            if (CK) {
                sum += v;
                xr ^= v;
            }
        }
    };
    constexpr uint32_t D = 32 * K;
    uint32_t base = 0;
    for (; base + D <= len; base += D) {
#pragma unroll
        for (int k = 0; k < K; ++k) word(base + 32 * k + lane, true);
        __syncwarp();
    }
    if (base < len) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t i = base + 32 * k + lane;
            word(i, i < len);
        }
        __syncwarp();
    }
}

// Two consecutive words per lane (64-word strips, D = 64 K2): the pair shares q[1] and the
// address arithmetic, reads (q0, q1) as one LDS.64, writes the pair to the ring as STS.64 when n
// is even (EVEN_N) and to HBM as one STG.64. Needs even piece lengths and 8-byte aligned output
// (L even: the planner cuts pieces at multiples of 4).
template <int KIND, bool CK, int K2, bool EVEN_N>
__device__ __forceinline__ void mt_piece2(const DevMtParams& p, uint32_t* ring, uint32_t ring_mask, uint32_t n,
                                          uint32_t lane, uint32_t* optr, uint32_t len, unsigned long long& sum,
                                          uint32_t& xr) {
    const uint32_t m = p.m, R = ring_mask + 1;
    const uint32_t upper = p.r ? (0xFFFFFFFFu << p.r) : 0xFFFFFFFFu, lower = ~upper;
    auto temper = [&](uint32_t v) {
        v ^= v >> p.u;
        v ^= (v << p.s) & p.b;
        v ^= (v << p.t) & p.c;
        v ^= v >> p.l;
        if (KIND != MTGP_U32) {
            v = (v >> 9) | 0x3F800000u;
            if (KIND == MTGP_F32_01OC) v = __float_as_uint(2.0f - __uint_as_float(v));
        }
        return v;
    };
    auto pair = [&](uint32_t i, bool store) {  // words i, i + 1 (i even)
        const uint32_t* q = ring + (i & ring_mask);
        const uint2 q01 = *reinterpret_cast<const uint2*>(q);
        const uint32_t q2 = q[2], qm0 = q[m], qm1 = q[m + 1];
        const uint32_t y0 = (q01.x & upper) | (q01.y & lower);
        const uint32_t y1 = (q01.y & upper) | (q2 & lower);
        const uint32_t x0 = qm0 ^ (y0 >> 1) ^ ((y0 & 1u) ? p.a : 0u);
        const uint32_t x1 = qm1 ^ (y1 >> 1) ^ ((y1 & 1u) ? p.a : 0u);
        if (EVEN_N) {
            const uint32_t w = (i + n) & ring_mask;  // even: the pair does not wrap
            *reinterpret_cast<uint2*>(ring + w) = make_uint2(x0, x1);
            *reinterpret_cast<uint2*>(ring + w + R) = make_uint2(x0, x1);
        } else {
            const uint32_t w0 = (i + n) & ring_mask, w1 = (i + n + 1) & ring_mask;
            ring[w0] = x0;
            ring[w0 + R] = x0;
            ring[w1] = x1;
            ring[w1 + R] = x1;
        }
        if (store) {
            const uint32_t v0 = temper(x0), v1 = temper(x1);
            __stcs(reinterpret_cast<uint2*>(optr + i), make_uint2(v0, v1));
            if (CK) {
                sum += v0;
                sum += v1;
                xr ^= v0 ^ v1;
            }
        }
    };
    constexpr uint32_t D = 64 * K2;
    uint32_t base = 0;
    for (; base + D <= len; base += D) {
#pragma unroll
        for (int k = 0; k < K2; ++k) pair(base + 64 * k + 2 * lane, true);
        __syncwarp();
    }
    if (base < len) {
#pragma unroll
        for (int k = 0; k < K2; ++k) {
            const uint32_t i = base + 64 * k + 2 * lane;
            pair(i, i < len);  // len is even, so i < len covers both words
        }
        __syncwarp();
    }
}

template <int KIND, bool CK>
__global__ void __launch_bounds__(kWarpsPerCta * 32) mt_gen2_kernel(MtGenArgs a, uint32_t ring_mask) {
    extern __shared__ uint32_t smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t team = blockIdx.x * kWarpsPerCta + warp;
    if (team >= a.n_teams) return;
    const uint32_t R = ring_mask + 1;
    uint32_t* ring = smem + warp * 2 * R;
    const uint32_t n = a.n;
    const TeamWork tw = a.teams[team];
    for (uint32_t pi = tw.first; pi < tw.first + tw.count; ++pi) {
        const Piece pc = a.pieces[pi];
        const DevMtParams p = a.params[pc.set];
        const uint32_t* w0 = a.piece_win[pi];
        for (uint32_t j = lane; j < n; j += 32) ring[j] = ring[j + R] = w0[j];
        __syncwarp();
        uint32_t* optr = reinterpret_cast<uint32_t*>(a.out) + (size_t)pc.set * a.L + pc.offset;
        const uint32_t len = (uint32_t)pc.len;
        unsigned long long sum = 0;
        uint32_t xr = 0;
        const uint32_t k2 = min(4u, (n - p.m) >> 6);  // 64-word strips for the pair path
        if (a.pairs && k2 > 0) {
            const bool even = (n & 1u) == 0;
            switch (k2 * 2 + (even ? 1 : 0)) {
                case 2: mt_piece2<KIND, CK, 1, false>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
                case 3: mt_piece2<KIND, CK, 1, true>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
                case 4: mt_piece2<KIND, CK, 2, false>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
                case 5: mt_piece2<KIND, CK, 2, true>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
                case 6: mt_piece2<KIND, CK, 3, false>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
                case 7: mt_piece2<KIND, CK, 3, true>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
                case 8: mt_piece2<KIND, CK, 4, false>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
                default: mt_piece2<KIND, CK, 4, true>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
            }
        } else switch (min(8u, (n - p.m) >> 5)) {  // K = D / 32
            case 1: mt_piece<KIND, CK, 1>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
            case 2: mt_piece<KIND, CK, 2>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
            case 3: mt_piece<KIND, CK, 3>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
            case 4: mt_piece<KIND, CK, 4>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
            case 5: mt_piece<KIND, CK, 5>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
            case 6: mt_piece<KIND, CK, 6>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
            case 7: mt_piece<KIND, CK, 7>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
            default: mt_piece<KIND, CK, 8>(p, ring, ring_mask, n, lane, optr, len, sum, xr); break;
        }
        if (pc.offset + pc.len == a.L) {  // end window x_len .. x_{len+n-1}
            uint32_t* wout = a.win_out + (size_t)pc.set * n;
            for (uint32_t k = lane; k < n; k += 32) wout[k] = ring[(len + k) & ring_mask];
        }
        if (CK) {
            for (int sft = 16; sft > 0; sft >>= 1) {
                sum += __shfl_xor_sync(0xffffffffu, sum, sft);
                xr ^= __shfl_xor_sync(0xffffffffu, xr, sft);
            }
            if (lane == 0) {
                atomicAdd(&a.ck[pc.set].sum64, sum);
                atomicXor(&a.ck[pc.set].xor32, xr);
                atomicAdd(&a.ck[pc.set].words, (unsigned long long)len);
            }
        }
        __syncwarp();
    }
}

template <int KIND, bool CK>
static cudaError_t launch_mt2_t(const MtGenArgs& a, cudaStream_t st) {
    const uint32_t R = next_pow2(a.n + 256);
    const size_t smem = (size_t)kWarpsPerCta * 2 * R * 4;  // mirrored rings
    auto k = mt_gen2_kernel<KIND, CK>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<(a.n_teams + kWarpsPerCta - 1) / kWarpsPerCta, kWarpsPerCta * 32, smem, st>>>(a, R - 1);
    return cudaGetLastError();
}

template <int KIND, bool CK>
static int occ_mt2_t(uint32_t n) {
    const uint32_t R = next_pow2(n + 256);
    const size_t smem = (size_t)kWarpsPerCta * 2 * R * 4;  // mirrored rings
    auto k = mt_gen2_kernel<KIND, CK>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    int c = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k, kWarpsPerCta * 32, smem) != cudaSuccess) return 0;
    return c;
}

cudaError_t launch_mt_gen2(int kind, bool cksum, const MtGenArgs& a, cudaStream_t st) {
    if (a.n_teams == 0) return cudaSuccess;
    switch (kind * 2 + (cksum ? 1 : 0)) {
        case 0: return launch_mt2_t<MTGP_U32, false>(a, st);
        case 1: return launch_mt2_t<MTGP_U32, true>(a, st);
        case 2: return launch_mt2_t<MTGP_F32_12, false>(a, st);
        case 3: return launch_mt2_t<MTGP_F32_12, true>(a, st);
        case 4: return launch_mt2_t<MTGP_F32_01OC, false>(a, st);
        case 5: return launch_mt2_t<MTGP_F32_01OC, true>(a, st);
    }
    return cudaErrorInvalidValue;
}

int mt_gen2_ctas_per_sm(uint32_t n, int kind, bool cksum) {
    switch (kind * 2 + (cksum ? 1 : 0)) {
        case 0: return occ_mt2_t<MTGP_U32, false>(n);
        case 1: return occ_mt2_t<MTGP_U32, true>(n);
        case 2: return occ_mt2_t<MTGP_F32_12, false>(n);
        case 3: return occ_mt2_t<MTGP_F32_12, true>(n);
        case 4: return occ_mt2_t<MTGP_F32_01OC, false>(n);
        case 5: return occ_mt2_t<MTGP_F32_01OC, true>(n);
    }
    return 0;
}

}  // namespace mtgpb
