// mtgp_v4.cuh -- register-resident MTGP32 generation for any state size (gen3's design, templated
// on the Mersenne exponent; used for MTGP32-23209 and -44497).
//
// Same decomposition and step as gen3 (csrc/mtgp_v3.cu): one warp per jump-ahead piece, 256-word
// steps, lane t owns words 4t..4t+3 of each 128-word half-step, two coalesced STG.128 per step,
// tables in registers, every operand word ONE shfl.idx from a fixed source lane of ONE
// SEL-chosen history register. What changes with N:
//
//   K    = ceil(N / 256) steps of history, kept as 2K half-steps H[0..2K) (oldest first);
//   BASE = 256K - N: operand x_{g+off} of the word produced at step position p sits at history
//          position BASE + off + p (counted from the start of step m-K);
//   with BASE + off = 4Q + R, Q = 32a + b: component (R+j) mod 4 of source lane (t+b+e) mod 32,
//          half-step u + a + [source lane < b + e]  (e = carry of R + j).
//   A stream (off = 0): a, b, R fixed by N.  C stream (off = pos - 1): a_C = Q_C / 32 picks the
//          register pair, so it is a template parameter (AC, one variant per value a set's pos can
//          give: 1 for 11213, 4 for 23209, 9 for 44497) next to R_C = (BASE + pos - 1) mod 4.
//   After each step the history shifts by two half-steps; the main loop is unrolled by K so the
//   shift is register renaming (the 2K-entry history returns to its registers after K steps).
//
// Requires N - pos >= 256 for every set (all cuRAND sets; synthetic sets are built that way).
#pragma once

#include <type_traits>
#include "mtgp_v2.cuh"

namespace mtgpb {

// checksum accumulator of MTGP_OPT_CHECKSUM mode CKM (2: the word sum mod 2^32 in 32 bits)
template <int CKM>
using CkAcc4 = typename std::conditional<CKM == 2, uint32_t, unsigned long long>::type;

// Steps per main-loop trip: 0 = K (the history shift is pure register renaming, but the code is
// K times larger); otherwise the shift costs register moves (IMAD.MOV, FMA pipe) at the loop
// back-edge. -1 (default) = per history depth, measured (profiles/r1_v4_unroll_sweep.jsonl):
// K <= 3 (11213, 23209): K; K >= 4 (44497, K = 6): 2 -- full unrolling there spills at the
// 128-register cap and U = 3 is slower than U = 2.
#ifndef MTGP4_UNROLL
#define MTGP4_UNROLL -1
#endif
#ifndef MTGP4_BIG_CTA
#define MTGP4_BIG_CTA 1
#endif
#ifndef MTGP4_MIN_CTAS
#define MTGP4_MIN_CTAS 0  // 0: by history depth (6 / 5 / 4 CTAs for K = 2 / 3 / >= 4)
#endif

namespace {

constexpr uint32_t kFull4 = 0xffffffffu;

template <uint32_t MEXP>
struct S4 {
    static constexpr uint32_t N = MEXP / 32 + 1;
    static constexpr uint32_t K = (N + 255) / 256;   // steps of history
    static constexpr uint32_t H = 2 * K;             // half-steps kept
    static constexpr uint32_t BASE = 256 * K - N;    // history position of x_g for p = 0
    static constexpr uint32_t QA = BASE >> 2, RA = BASE & 3;
    static constexpr uint32_t AA = QA >> 5, BA = QA & 31;
    static constexpr uint32_t AC_MIN = (BASE + 1) >> 7;  // pos >= 2
    static constexpr uint32_t AC_MAX = H - 3;            // pos <= N - 256
    static constexpr int MIN_CTAS = MTGP4_MIN_CTAS ? MTGP4_MIN_CTAS : (K == 2 ? 6 : K == 3 ? 5 : 4);
    static constexpr int kUnroll = MTGP4_UNROLL;
    static constexpr uint32_t U = kUnroll > 0 ? (uint32_t)kUnroll : (kUnroll == 0 || K <= 3) ? K : 2u;  // steps/trip
    // One CTA per SM holding all of the SM's warps (MIN_CTAS x 4): teams are ordered by stream,
    // so a CTA's warps share one or two streams -- one or two C-stream variants per SM instead of
    // one per 4-warp CTA (the variants otherwise thrash the instruction cache).
    static constexpr uint32_t WARPS = MTGP4_BIG_CTA ? 4u * MIN_CTAS : kWarpsPerCta;
};

struct V4Ctx {
    uint32_t lane;
    uint32_t mask, sh1, sh2, mul1, tblr, tmpr;
    uint32_t srcA0, srcA1, srcC0, srcC1;  // source lanes for carry e = 0 / 1
    bool pA0, pA1, pC0, pC1;              // "take the newer half-step of the pair" (source side)
};

__device__ __forceinline__ uint32_t comp(const uint4& g, int c) {
    return c == 0 ? g.x : c == 1 ? g.y : c == 2 ? g.z : g.w;
}

// M3 (curand_mtgp32_kernel.h:137-145): X = (a & mask) ^ b; X ^= X << sh1; Y = X ^ (c >> sh2);
// result Y ^ tbl[Y & 15] (table lookup = shfl over a 16-lane segment)
__device__ __forceinline__ uint32_t rec4(const V4Ctx& p, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t x = (a & p.mask) ^ b;
    const uint32_t y = x ^ (x * p.mul1) ^ (c >> p.sh2);
    return y ^ __shfl_sync(kFull4, p.tblr, y, 16);
}

// tempering indices of two words (see gen3: fold2)
__device__ __forceinline__ void fold(uint32_t t1, uint32_t t2, uint32_t& i1, uint32_t& i2) {
    const uint32_t w = __byte_perm(t1, t2, 0x5410) ^ __byte_perm(t1, t2, 0x7632);
    const uint32_t z = w ^ (w >> 8);
    i1 = z;
    i2 = z >> 16;
}

template <int KIND>
__device__ __forceinline__ uint32_t conv(uint32_t o) {
    if (KIND == MTGP_U32) return o;
    uint32_t v = (o >> 9) | 0x3F800000u;
    if (KIND == MTGP_F32_01OC) v = __float_as_uint(2.0f - __uint_as_float(v));
    return v;
}

// Five consecutive operand words: residue R, register pair (Hs[LO], Hs[LO + 1]).
template <int R, int LO, int NH>
__device__ __forceinline__ void fetch(uint32_t W[5], const uint4 (&Hs)[NH], uint32_t src0, uint32_t src1, bool p0,
                                      bool p1) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int c = (R + j) & 3;
        const int e = (R + j) >> 2;
        const uint32_t send = (e ? p1 : p0) ? comp(Hs[LO + 1], c) : comp(Hs[LO], c);
        W[j] = __shfl_sync(kFull4, send, e ? src1 : src0);
    }
}

template <uint32_t MEXP, int RC, int AC, int KIND, int CKM, bool TAIL>
__device__ __forceinline__ void step4(const V4Ctx& p, const uint4 (&Hs)[S4<MEXP>::H], uint4& n0, uint4& n1,
                                      uint32_t* optr, uint32_t n, uint32_t len, uint32_t* win_out,
                                      CkAcc4<CKM>& sum, uint32_t& xr) {
    using S = S4<MEXP>;
    uint32_t WA[2][5], WC[2][5];
    fetch<S::RA, S::AA, S::H>(WA[0], Hs, p.srcA0, p.srcA1, p.pA0, p.pA1);
    fetch<S::RA, S::AA + 1, S::H>(WA[1], Hs, p.srcA0, p.srcA1, p.pA0, p.pA1);
    fetch<RC, AC, S::H>(WC[0], Hs, p.srcC0, p.srcC1, p.pC0, p.pC1);
    fetch<RC, AC + 1, S::H>(WC[1], Hs, p.srcC0, p.srcC1, p.pC0, p.pC1);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        uint32_t r[4], o[4], ix[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) r[c] = rec4(p, WA[u][c], WA[u][c + 1], WC[u][c + 1]);
        fold(WC[u][0], WC[u][1], ix[0], ix[1]);
        fold(WC[u][2], WC[u][3], ix[2], ix[3]);
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = conv<KIND>(r[c] ^ __shfl_sync(kFull4, p.tmpr, ix[c], 16));
        const uint32_t w0 = n + 128 * u + 4 * p.lane;  // piece word of o[0]
        if (!TAIL || w0 < len) {
            __stcs(reinterpret_cast<uint4*>(optr + w0), make_uint4(o[0], o[1], o[2], o[3]));
            if (CKM == 2) {
                sum = sum + o[0] + o[1];  // 3-input IADD3s, mod 2^32 (MTGP_OPT_CHECKSUM 2)
                sum = sum + o[2] + o[3];
            } else if (CKM == 1) {
#pragma unroll
                for (int c = 0; c < 4; ++c) sum += o[c];
            }
            if (CKM) xr ^= o[0] ^ o[1] ^ o[2] ^ o[3];
        }
        if (TAIL && win_out) {
            // sequence index of r[c] is N + w0 + c; the end window is [len, len + N)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t k = S::N + w0 + c - len;
                if (k < S::N) win_out[k] = r[c];
            }
        }
        (u == 0 ? n0 : n1) = make_uint4(r[0], r[1], r[2], r[3]);
    }
}

template <int NH>
__device__ __forceinline__ void shift2(uint4 (&Hs)[NH], const uint4& n0, const uint4& n1) {
#pragma unroll
    for (int i = 0; i + 2 < NH; ++i) Hs[i] = Hs[i + 2];
    Hs[NH - 2] = n0;
    Hs[NH - 1] = n1;
}

template <uint32_t MEXP, int RC, int AC, int KIND, int CKM>
__device__ __forceinline__ void run4(const V4Ctx& p, uint4 (&Hs)[S4<MEXP>::H], uint32_t* optr, uint32_t len,
                                  uint32_t* win_out, CkAcc4<CKM>& sum, uint32_t& xr) {
    using S = S4<MEXP>;
    const uint32_t steps = (len + kStepWords - 1) / kStepWords;
    // A step at n produces sequence words [N + n, N + n + 256): no store predicate and no end
    // window while n + 256 + N <= len. The main loop runs U such steps per trip; the rest run
    // the predicated tail variant.
    uint32_t m = 0;
    for (; (m + S::U) * kStepWords + S::N <= len; m += S::U) {
#pragma unroll
        for (uint32_t k = 0; k < S::U; ++k) {
            uint4 n0, n1;
            step4<MEXP, RC, AC, KIND, CKM, false>(p, Hs, n0, n1, optr, (m + k) * kStepWords, len, nullptr, sum, xr);
            shift2(Hs, n0, n1);
        }
    }
    for (; m < steps; ++m) {
        uint4 n0, n1;
        step4<MEXP, RC, AC, KIND, CKM, true>(p, Hs, n0, n1, optr, m * kStepWords, len, win_out, sum, xr);
        shift2(Hs, n0, n1);
    }
}

template <uint32_t MEXP, int AC, int KIND, int CKM>
__device__ __forceinline__ void run_rc(int rc, const V4Ctx& p, uint4 (&Hs)[S4<MEXP>::H], uint32_t* optr, uint32_t len,
                                       uint32_t* win_out, CkAcc4<CKM>& sum, uint32_t& xr) {
    switch (rc) {
        case 0: run4<MEXP, 0, AC, KIND, CKM>(p, Hs, optr, len, win_out, sum, xr); break;
        case 1: run4<MEXP, 1, AC, KIND, CKM>(p, Hs, optr, len, win_out, sum, xr); break;
        case 2: run4<MEXP, 2, AC, KIND, CKM>(p, Hs, optr, len, win_out, sum, xr); break;
        default: run4<MEXP, 3, AC, KIND, CKM>(p, Hs, optr, len, win_out, sum, xr); break;
    }
}

template <uint32_t MEXP, int AC, int KIND, int CKM>
__device__ __forceinline__ void run_ac(int ac, int rc, const V4Ctx& p, uint4 (&Hs)[S4<MEXP>::H], uint32_t* optr,
                                       uint32_t len, uint32_t* win_out, CkAcc4<CKM>& sum, uint32_t& xr) {
    if constexpr (AC <= (int)S4<MEXP>::AC_MAX) {
        if (ac == AC)
            run_rc<MEXP, AC, KIND, CKM>(rc, p, Hs, optr, len, win_out, sum, xr);
        else
            run_ac<MEXP, AC + 1, KIND, CKM>(ac, rc, p, Hs, optr, len, win_out, sum, xr);
    }
}

}  // namespace

template <uint32_t MEXP, int KIND, int CKM>
__global__ void __launch_bounds__(S4<MEXP>::WARPS * 32, S4<MEXP>::MIN_CTAS * kWarpsPerCta / S4<MEXP>::WARPS)
    gen4_kernel(GenArgs a) {
    using S = S4<MEXP>;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t team = blockIdx.x * S::WARPS + warp;
    if (team >= a.n_teams) return;
    V4Ctx p;
    p.lane = lane;
    p.srcA0 = (lane + S::BA) & 31;
    p.srcA1 = (lane + S::BA + 1) & 31;
    p.pA0 = lane < S::BA;
    p.pA1 = lane < S::BA + 1;
    const TeamWork tw = a.teams[team];
    for (uint32_t pi = tw.first; pi < tw.first + tw.count; ++pi) {
        const Piece pc = a.pieces[pi];
        const DevParams& prm = a.params[pc.set];
        p.mask = prm.mask;
        p.sh1 = prm.sh1;
        p.sh2 = prm.sh2;
        p.mul1 = prm.mul1;
        p.tblr = prm.tbl[lane & 15];
        p.tmpr = prm.tmp[lane & 15];
        const uint32_t qc = (S::BASE + prm.pos - 1) >> 2;  // C stream: BASE + pos - 1 = 4 qc + rc
        const int rc = (int)((S::BASE + prm.pos - 1) & 3);
        const int ac = (int)(qc >> 5);
        const uint32_t thr0 = qc & 31, thr1 = thr0 + 1;  // in [0, 32]
        p.srcC0 = (lane + thr0) & 31;
        p.srcC1 = (lane + thr1) & 31;
        p.pC0 = lane < thr0;
        p.pC1 = lane < thr1;
        uint32_t* optr = reinterpret_cast<uint32_t*>(a.out) + (size_t)pc.set * a.L + pc.offset;
        const uint32_t len = (uint32_t)pc.len;
        const uint32_t* w0 = a.piece_win[pi];
        // history before step 0: half-step h, lane t, component c holds x_{128h + 4t + c - BASE}
        uint4 Hs[S::H];
#pragma unroll
        for (int h = 0; h < (int)S::H; ++h) {
            uint32_t v[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int k = 128 * h + 4 * (int)lane + c - (int)S::BASE;
                v[c] = k >= 0 ? w0[k] : 0u;
            }
            Hs[h] = make_uint4(v[0], v[1], v[2], v[3]);
        }
        uint32_t* win_out = nullptr;
        if (pc.offset + pc.len == a.L) {
            win_out = a.win_out + (size_t)pc.set * S::N;
            for (uint32_t j = lane; j + len < S::N; j += 32) win_out[j] = w0[len + j];  // pieces shorter than N
        }
        CkAcc4<CKM> sum = 0;
        uint32_t xr = 0;
        run_ac<MEXP, (int)S::AC_MIN, KIND, CKM>(ac, rc, p, Hs, optr, len, win_out, sum, xr);
        if (CKM) {
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                sum += __shfl_xor_sync(kFull4, sum, s);
                xr ^= __shfl_xor_sync(kFull4, xr, s);
            }
            if (lane == 0) {
                atomicAdd(&a.ck[pc.set].sum64, (unsigned long long)sum);
                atomicXor(&a.ck[pc.set].xor32, xr);
                atomicAdd(&a.ck[pc.set].words, (unsigned long long)len);
            }
        }
        __syncwarp();
    }
}

template <uint32_t MEXP, int KIND, int CKM>
static cudaError_t launch4_t(const GenArgs& a, cudaStream_t st) {
    constexpr uint32_t W = S4<MEXP>::WARPS;
    const uint32_t grid = (a.n_teams + W - 1) / W;
    gen4_kernel<MEXP, KIND, CKM><<<grid, W * 32, 0, st>>>(a);
    return cudaGetLastError();
}

template <uint32_t MEXP, int KIND, int CKM>
static int occ4_t() {
    int n = 0;
    constexpr uint32_t W = S4<MEXP>::WARPS;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gen4_kernel<MEXP, KIND, CKM>, W * 32, 0) != cudaSuccess)
        return 0;
    return n * (int)(W / kWarpsPerCta);  // in the planner's unit: resident 4-warp teams groups
}

// Per-exponent entry points (one translation unit each: mtgp_v4_<mexp>.cu), u32 output only.
cudaError_t launch_gen4_11213(int ck_mode, const GenArgs& a, cudaStream_t st);
cudaError_t launch_gen4_23209(int ck_mode, const GenArgs& a, cudaStream_t st);
cudaError_t launch_gen4_44497(int ck_mode, const GenArgs& a, cudaStream_t st);
int gen4_ctas_11213(int ck_mode);
int gen4_ctas_23209(int ck_mode);
int gen4_ctas_44497(int ck_mode);

}  // namespace mtgpb
