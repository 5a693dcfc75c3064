// mtgp_v5.cu -- gen3's register-resident MTGP32-11213 step with eight consecutive words per lane.
//
// gen3 (mtgp_v3.cu) gives lane t words 4t..4t+3 and 128+4t..128+4t+3 of a 256-word step so each
// STG.128 covers 512 contiguous bytes; every operand stream then needs 5 shuffled words per 4
// outputs. Here lane t owns words 8t..8t+7 of the step and writes them with ONE 256-bit
// streaming store (st.global.cs.v8.b32 -> STG.E.EF.ENL2.256, sm_100), so the warp's 1 KiB step is
// one contiguous store and each operand stream needs 9 shuffled words per 8 outputs:
// per step 18 SHFL + 18 SEL + 1 STG instead of 20 + 20 + 2.
//
//   operand x_{256m + 8t + j + off} (A stream off = 0, C stream off = pos - 1), j = 0..8, sits at
//   history position P = 161 + off + 8t + j counted from the start of step m-2 (512 - N = 161).
//   With 161 + off = 8*Q0 + R: component c = (R + j) mod 8, carry e = (R + j) div 8, source lane
//   s = (t + Q0 + e) mod 32, and s sends its step m-1 word when s < Q0 + e, else its step m-2 word.
//   A: Q0 = 20, R = 1. C: Q0 = 20 + pos/8, R = pos mod 8 (eight unrolled variants).
//
// Needs N - pos >= 256 (all 200 cuRAND sets: >= 258), piece offsets and lengths multiples of 8
// words and 32-byte aligned output (the planner cuts at multiples of 8; L % 8 == 0).
#include "mtgp_v2.cuh"

namespace mtgpb {

#define FULL 0xffffffffu

#ifndef MTGP5_MIN_CTAS
#define MTGP5_MIN_CTAS 6
#endif

namespace {

constexpr uint32_t kN5 = 351;

struct V5Ctx {
    uint32_t lane;
    uint32_t mask, sh2, mul1, tblr, tmpr;
    uint32_t srcA0, srcA1, srcC0, srcC1;
    bool pA0, pA1, pC0, pC1;
};

struct H8 {
    uint32_t v[8];
};

__device__ __forceinline__ uint32_t rec5(const V5Ctx& p, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t x = (a & p.mask) ^ b;
    const uint32_t y = x ^ (x * p.mul1) ^ (c >> p.sh2);
    return y ^ __shfl_sync(FULL, p.tblr, y, 16);
}

__device__ __forceinline__ void fold2(uint32_t t1, uint32_t t2, uint32_t& i1, uint32_t& i2) {
    const uint32_t w = __byte_perm(t1, t2, 0x5410) ^ __byte_perm(t1, t2, 0x7632);
    const uint32_t z = w ^ (w >> 8);
    i1 = z;
    i2 = z >> 16;
}

template <int KIND>
__device__ __forceinline__ uint32_t conv5(uint32_t o) {
    if (KIND == MTGP_U32) return o;
    uint32_t v = (o >> 9) | 0x3F800000u;
    if (KIND == MTGP_F32_01OC) v = __float_as_uint(2.0f - __uint_as_float(v));
    return v;
}

// Nine consecutive operand words from the history (old = step m-2, nw = step m-1), residue R.
template <int R>
__device__ __forceinline__ void fetch9(uint32_t W[9], const H8& old, const H8& nw, uint32_t src0, uint32_t src1,
                                       bool p0, bool p1) {
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const int c = (R + j) & 7;
        const int e = (R + j) >> 3;
        const uint32_t send = (e ? p1 : p0) ? nw.v[c] : old.v[c];
        W[j] = __shfl_sync(FULL, send, e ? src1 : src0);
    }
}

__device__ __forceinline__ void st256(uint32_t* dst, const uint32_t o[8]) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(o[0]), "r"(o[1]),
                 "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7])
                 : "memory");
}

// One 256-word step: reads old (m-2) and nw (m-1), writes the new step into `out_h` (which may
// alias `old`: every history word is fetched before any is overwritten).
template <int RC, int KIND, bool CK, bool TAIL>
__device__ __forceinline__ void step5(const V5Ctx& p, H8& old, const H8& nw, uint32_t* optr, uint32_t n,
                                      uint32_t len, uint32_t* win_out, unsigned long long& sum, uint32_t& xr) {
    uint32_t WA[9], WC[9];
    fetch9<1>(WA, old, nw, p.srcA0, p.srcA1, p.pA0, p.pA1);
    fetch9<RC>(WC, old, nw, p.srcC0, p.srcC1, p.pC0, p.pC1);
    uint32_t r[8], o[8], ix[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) r[c] = rec5(p, WA[c], WA[c + 1], WC[c + 1]);
#pragma unroll
    for (int c = 0; c < 8; c += 2) fold2(WC[c], WC[c + 1], ix[c], ix[c + 1]);
#pragma unroll
    for (int c = 0; c < 8; ++c) o[c] = conv5<KIND>(r[c] ^ __shfl_sync(FULL, p.tmpr, ix[c], 16));
    const uint32_t w0 = n + 8 * p.lane;  // piece word of o[0]
    if (!TAIL || w0 < len) {
        st256(optr + w0, o);
        if (CK) {
#pragma unroll
            for (int c = 0; c < 8; ++c) sum += o[c];
            xr ^= o[0] ^ o[1] ^ o[2] ^ o[3] ^ o[4] ^ o[5] ^ o[6] ^ o[7];
        }
    }
    if (TAIL && win_out) {
        // sequence index of r[c] is kN5 + w0 + c; the end window is [len, len + kN5)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint32_t k = kN5 + w0 + c - len;
            if (k < kN5) win_out[k] = r[c];
        }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) old.v[c] = r[c];
}

template <int RC, int KIND, bool CK>
__device__ __forceinline__ void run5(const V5Ctx& p, H8 X, H8 Y, uint32_t* optr, uint32_t len, uint32_t* win_out,
                                     unsigned long long& sum, uint32_t& xr) {
    // ping-pong: even steps read (X = m-2, Y = m-1) and overwrite X; odd steps read (Y, X), overwrite Y
    const uint32_t steps = (len + kStepWords - 1) / kStepWords;
    uint32_t m = 0;
    for (; (m + 2) * kStepWords + kN5 <= len; m += 2) {
        step5<RC, KIND, CK, false>(p, X, Y, optr, m * kStepWords, len, nullptr, sum, xr);
        step5<RC, KIND, CK, false>(p, Y, X, optr, (m + 1) * kStepWords, len, nullptr, sum, xr);
    }
    while (m < steps) {
        step5<RC, KIND, CK, true>(p, X, Y, optr, m * kStepWords, len, win_out, sum, xr);
        if (++m >= steps) break;
        step5<RC, KIND, CK, true>(p, Y, X, optr, m * kStepWords, len, win_out, sum, xr);
        ++m;
    }
}

}  // namespace

template <int KIND, bool CK>
__global__ void __launch_bounds__(kWarpsPerCta * 32, MTGP5_MIN_CTAS) gen5_kernel(GenArgs a) {
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t team = blockIdx.x * kWarpsPerCta + warp;
    if (team >= a.n_teams) return;
    V5Ctx p;
    p.lane = lane;
    p.srcA0 = (lane + 20) & 31;
    p.srcA1 = (lane + 21) & 31;
    p.pA0 = lane < 20;
    p.pA1 = lane < 21;
    const TeamWork tw = a.teams[team];
    for (uint32_t pi = tw.first; pi < tw.first + tw.count; ++pi) {
        const Piece pc = a.pieces[pi];
        const DevParams& prm = a.params[pc.set];
        p.mask = prm.mask;
        p.sh2 = prm.sh2;
        p.mul1 = prm.mul1;
        p.tblr = prm.tbl[lane & 15];
        p.tmpr = prm.tmp[lane & 15];
        const uint32_t pos = prm.pos;
        const uint32_t q0 = 20 + (pos >> 3), q1 = q0 + 1;  // q1 <= 32
        p.srcC0 = (lane + q0) & 31;
        p.srcC1 = (lane + q1) & 31;
        p.pC0 = lane < q0;
        p.pC1 = lane < q1;
        uint32_t* optr = reinterpret_cast<uint32_t*>(a.out) + (size_t)pc.set * a.L + pc.offset;
        const uint32_t len = (uint32_t)pc.len;
        const uint32_t* w0 = a.piece_win[pi];
        // history before step 0: Y = step -1 = x_{95 + 8t + c}; X = step -2 = x_{-161 + 8t + c}
        // (only positions >= 161, i.e. lanes >= 20, are ever read)
        H8 X, Y;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            Y.v[c] = w0[95 + 8 * lane + c];
            const int k = -161 + 8 * (int)lane + c;
            X.v[c] = k >= 0 ? w0[k] : 0u;
        }
        uint32_t* win_out = nullptr;
        if (pc.offset + pc.len == a.L) {
            win_out = a.win_out + (size_t)pc.set * kN5;
            for (uint32_t j = lane; j + len < kN5; j += 32) win_out[j] = w0[len + j];
        }
        unsigned long long sum = 0;
        uint32_t xr = 0;
        switch (pos & 7u) {
            case 0: run5<0, KIND, CK>(p, X, Y, optr, len, win_out, sum, xr); break;
            case 1: run5<1, KIND, CK>(p, X, Y, optr, len, win_out, sum, xr); break;
            case 2: run5<2, KIND, CK>(p, X, Y, optr, len, win_out, sum, xr); break;
            case 3: run5<3, KIND, CK>(p, X, Y, optr, len, win_out, sum, xr); break;
            case 4: run5<4, KIND, CK>(p, X, Y, optr, len, win_out, sum, xr); break;
            case 5: run5<5, KIND, CK>(p, X, Y, optr, len, win_out, sum, xr); break;
            case 6: run5<6, KIND, CK>(p, X, Y, optr, len, win_out, sum, xr); break;
            default: run5<7, KIND, CK>(p, X, Y, optr, len, win_out, sum, xr); break;
        }
        if (CK) {
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                sum += __shfl_xor_sync(FULL, sum, s);
                xr ^= __shfl_xor_sync(FULL, xr, s);
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
static cudaError_t launch5_t(const GenArgs& a, cudaStream_t st) {
    const uint32_t grid = (a.n_teams + kWarpsPerCta - 1) / kWarpsPerCta;
    gen5_kernel<KIND, CK><<<grid, kWarpsPerCta * 32, 0, st>>>(a);
    return cudaGetLastError();
}

template <int KIND, bool CK>
static int occ5_t() {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gen5_kernel<KIND, CK>, kWarpsPerCta * 32, 0) != cudaSuccess)
        return 0;
    return n;
}

cudaError_t launch_gen5(int kind, bool cksum, const GenArgs& a, cudaStream_t st) {
    if (a.n_teams == 0) return cudaSuccess;
    switch (kind * 2 + (cksum ? 1 : 0)) {
        case 0: return launch5_t<MTGP_U32, false>(a, st);
        case 1: return launch5_t<MTGP_U32, true>(a, st);
        case 2: return launch5_t<MTGP_F32_12, false>(a, st);
        case 3: return launch5_t<MTGP_F32_12, true>(a, st);
        case 4: return launch5_t<MTGP_F32_01OC, false>(a, st);
        case 5: return launch5_t<MTGP_F32_01OC, true>(a, st);
    }
    return cudaErrorInvalidValue;
}

int gen5_ctas_per_sm(int kind, bool cksum) {
    switch (kind * 2 + (cksum ? 1 : 0)) {
        case 0: return occ5_t<MTGP_U32, false>();
        case 1: return occ5_t<MTGP_U32, true>();
        case 2: return occ5_t<MTGP_F32_12, false>();
        case 3: return occ5_t<MTGP_F32_12, true>();
        case 4: return occ5_t<MTGP_F32_01OC, false>();
        case 5: return occ5_t<MTGP_F32_01OC, true>();
    }
    return 0;
}

}  // namespace mtgpb
