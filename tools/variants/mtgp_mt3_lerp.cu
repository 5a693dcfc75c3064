// tools/variants/mtgp_mt3_lerp.cu -- mt_gen3 with MTGP6_LERP (operand select as lo + m*(hi-lo) on the FMA
// pipe): ALU ops per five half-steps 271 -> 223, but 44.1 vs 42.3 M SM cycles per launch
// (profiles/r2/mt_gen3_lerp_sweep.jsonl); not in the product. Copy over csrc/mtgp_mt3.cu to rebuild.
// mtgp_mt3.cu -- register-resident Engine::mt generation (kernel version 6, mt_gen3_kernel):
// gen4's design (csrc/mtgp_v4.cuh) applied to the reference's classic MT recurrence
// (proj/src/generator.cpp:68-88, temper :7-13), for the MT19937 state shape n = 624.
//
// The recurrences have the same operand structure -- MTGP32 reads x_k, x_{k+1}, x_{k+pos}; MT
// reads x_k, x_{k+1}, x_{k+m} -- so the A stream (x_k, x_{k+1}) and the C stream (x_{k+m}) are
// fetched exactly as in gen4: every operand word is ONE shfl.idx from a fixed source lane of ONE
// SEL-chosen history register. What differs:
//   * step = one 128-word half-step (lane t makes words 4t..4t+3, one STG.128): n - m = 227
//     for MT19937, below gen4's 256-word step; any n - m >= 129 works here;
//   * history = H = ceil(n / 128) half-steps (5 for n = 624, 20 registers), BASE = 128 H - n;
//     operand x_{g-n+off} of the word at step position p is history position BASE + off + p;
//   * the C stream's register pair a_C = (BASE + m) / 128 and residue (BASE + m) mod 4 are
//     template parameters (4 x 4 variants for n = 624, one per status m class);
//   * no table lookups: the tempering is four shift/mask steps on the new word itself, the left
//     shifts as IMAD by 2^s / 2^t (FMA pipe), the right shifts and masks on the ALU pipe;
//   * the step loop is unrolled by H, so the history shift is register renaming.
// u32 output; pieces come from the shared planner / jump-ahead (csrc/mtgp_plan.cu), windows in
// the same n-word window model as every other kernel.
#include <algorithm>
#include <type_traits>

#include "mtgp_bitmap.cuh"
#include "mtgp_mt.cuh"
#include "mtgp_v2.cuh"

#ifndef MTGP6_MIN_CTAS
#define MTGP6_MIN_CTAS 5  // 6: 19% more pieces (jumps) for the same cycles
#endif
// Planned CTAs per SM: the checksum-mode-2 and unchecked variants fit 6 (80 registers), but the
// plan keeps 5 so the piece count (jumps) stays that of the 5-CTA layout
#ifndef MTGP6_MAX_CTAS
#define MTGP6_MAX_CTAS 5
#endif
// Right shifts of the tempering on the FMA pipe as IMAD.HI by 2^(32-k): 0 none, 1 the last
// (v >> l), 2 both (v >> u too).
#ifndef MTGP6_SHR_IMAD
#define MTGP6_SHR_IMAD 0
#endif
#ifndef MTGP6_CK_WIDE
#define MTGP6_CK_WIDE 0
#endif
// Operand select on the FMA pipe: send = lo + m * (hi - lo) with per-lane 0/1 multipliers and the
// pair's differences formed by IMAD (lo * -1 + hi): 9 SEL per step -> 8 + 9 IMAD. mt_gen3 is
// ALU-bound alone (LSU data pipe ~43%), unlike gen3, so moving work to the FMA pipe can pay.
#ifndef MTGP6_LERP
#define MTGP6_LERP 0
#endif

namespace mtgpb {

namespace {

// Checksum modes (MTGP_OPT_CHECKSUM): 0 none; 1 sum64 + xor32; 2 sum32 + xor32 (the sum mod 2^32
// in a 32-bit accumulator: one 3-input IADD3 per two words, no carry chain), as in gen3.
template <int CKM>
using CkAcc6 = typename std::conditional<CKM == 2, uint32_t, unsigned long long>::type;

constexpr uint32_t kFull6 = 0xffffffffu;
constexpr uint32_t kHalfWords = 128;

template <uint32_t NW>
struct S6 {
    static constexpr uint32_t N = NW;
    static constexpr uint32_t H = (N + kHalfWords - 1) / kHalfWords;  // half-steps of history
    static constexpr uint32_t BASE = kHalfWords * H - N;               // history position of x_{g-n}, p = 0
    static constexpr uint32_t QA = BASE >> 2, RA = BASE & 3;
    static constexpr uint32_t AA = QA >> 5, BA = QA & 31;
    static constexpr uint32_t AC_MAX = H - 2;  // n - m >= 129
};

struct M6Ctx {
    uint32_t lane;
    uint32_t upper, a, b, c, u, l, mul_s, mul_t, hi_u, hi_l, one;
    uint32_t srcA0, srcA1, srcC0, srcC1;  // source lanes for carry e = 0 / 1
    bool pA0, pA1, pC0, pC1;              // "send the newer half-step of the pair"
    uint32_t mA0, mA1, mC0, mC1;          // the same as 0/1 multipliers (MTGP6_LERP)
    uint32_t neg1;                        // 0xFFFFFFFF, opaque to the compiler
    uint32_t* bm;                         // bitmap kinds: this stream's bitmap,
    unsigned long long poff;              // the piece's first word within the call, the predicate
    BitmapPred pred;
};

__device__ __forceinline__ uint32_t comp6(const uint4& g, int c) {
    return c == 0 ? g.x : c == 1 ? g.y : c == 2 ? g.z : g.w;
}

// v >> k on the ALU pipe, or as the high word of v * 2^(32-k) on the FMA pipe
template <bool IMAD>
__device__ __forceinline__ uint32_t shr6(uint32_t v, uint32_t k, uint32_t hi) {
    if (!IMAD) return v >> k;
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(hi));
    return r;
}

__device__ __forceinline__ uint32_t mad6(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// CNT consecutive operand words: residue R, register pair (Hs[LO], Hs[LO + 1]).
template <int R, int LO, int CNT, int NH>
__device__ __forceinline__ void fetch6(uint32_t* W, const uint4 (&Hs)[NH], uint32_t src0, uint32_t src1, bool p0,
                                       bool p1, uint32_t m0, uint32_t m1, uint32_t neg1) {
#pragma unroll
    for (int j = 0; j < CNT; ++j) {
        const int c = (R + j) & 3;
        const int e = (R + j) >> 2;
        uint32_t send;
        if (MTGP6_LERP) {
            const uint32_t lo = comp6(Hs[LO], c);
            send = mad6(mad6(lo, neg1, comp6(Hs[LO + 1], c)), e ? m1 : m0, lo);  // lo + m (hi - lo)
        } else {
            send = (e ? p1 : p0) ? comp6(Hs[LO + 1], c) : comp6(Hs[LO], c);
        }
        W[j] = __shfl_sync(kFull6, send, e ? src1 : src0);
    }
}

// u32 -> double in [0,1): u * 2^-32 exactly (Generator::next_f64_01, generator.hpp:39-41), as
// (1 + u * 2^-32) - 1: the bit pattern 0x3FF00000:00000000 | u << 20 minus 1.0 (both exact)
__device__ __forceinline__ double u32_to_f64_01(uint32_t u) {
    return __hiloint2double((int)(0x3FF00000u | (u >> 12)), (int)(u << 20)) - 1.0;
}

// One 128-word step at piece word n; dst = this lane's slot of the step's output (16 bytes for
// u32, 32 bytes for f64: KIND = MTGP_U32 / MTGP_F64_01).
template <uint32_t NW, int RC, int AC, int KIND, int CKM, bool TAIL>
__device__ __forceinline__ void step6(const M6Ctx& p, const uint4 (&Hs)[S6<NW>::H], uint4& nw, uint4* dst,
                                      uint32_t n, uint32_t len, uint32_t* win_out, CkAcc6<CKM>& sum,
                                      uint32_t& xr) {
    using S = S6<NW>;
    uint32_t WA[5], WC[4];
    fetch6<S::RA, S::AA, 5, S::H>(WA, Hs, p.srcA0, p.srcA1, p.pA0, p.pA1, p.mA0, p.mA1, p.neg1);
    fetch6<RC, AC, 4, S::H>(WC, Hs, p.srcC0, p.srcC1, p.pC0, p.pC1, p.mC0, p.mC1, p.neg1);
    uint32_t r[4], o[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        // refill (generator.cpp:68-88): y = upper(x_k) | lower(x_{k+1});
        // x_{k+n} = x_{k+m} ^ (y >> 1) ^ (y odd ? a : 0)
        const uint32_t y = (WA[c] & p.upper) | (WA[c + 1] & ~p.upper);  // one LOP3
        uint32_t mag;  // (y & 1) * a as an IMAD (inline PTX: not turned back into ISETP + SEL)
        asm("mul.lo.u32 %0, %1, %2;" : "=r"(mag) : "r"(y & 1u), "r"(p.a));
        r[c] = WC[c] ^ (y >> 1) ^ mag;
        // temper (generator.cpp:7-13)
        uint32_t v = r[c];
        v ^= shr6<MTGP6_SHR_IMAD >= 2>(v, p.u, p.hi_u);
        v ^= (v * p.mul_s) & p.b;
        v ^= (v * p.mul_t) & p.c;
        v ^= shr6<MTGP6_SHR_IMAD >= 1>(v, p.l, p.hi_l);
        o[c] = v;
    }
    const uint32_t w0 = n + 4 * p.lane;  // piece word of o[0]
    if constexpr (KIND >= kKindBitmapBit0) {
        bitmap_store<KIND>(p.lane, p.bm, p.poff, p.pred, o, n, !TAIL || w0 < len);
    } else if (!TAIL || w0 < len) {
        if (KIND == MTGP_F64_01) {
            // one 256-bit streaming store per lane (STG.E.EF.ENL2.256, sm_100): the warp's 1 KiB
            // step in one contiguous instruction instead of two 16-byte-strided STG.128
            asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(u32_to_f64_01(o[0])),
                         "d"(u32_to_f64_01(o[1])), "d"(u32_to_f64_01(o[2])), "d"(u32_to_f64_01(o[3]))
                         : "memory");
        } else {
            __stcs(dst, make_uint4(o[0], o[1], o[2], o[3]));
        }
        if constexpr (CKM == 2) {
            sum = sum + o[0] + o[1];  // 3-input IADD3s, mod 2^32
            sum = sum + o[2] + o[3];
            xr ^= o[0] ^ o[1] ^ o[2] ^ o[3];
        } else if (CKM == 1) {
#if MTGP6_CK_WIDE
            // 64-bit sum on the FMA pipe: IMAD.WIDE.U32 sum = o * 1 + sum (the 1 is opaque)
#pragma unroll
            for (int c = 0; c < 4; ++c) asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(sum) : "r"(o[c]), "r"(p.one));
#else
#pragma unroll
            for (int c = 0; c < 4; ++c) sum += o[c];
#endif
            xr ^= o[0] ^ o[1] ^ o[2] ^ o[3];
        }
    }
    if (TAIL && win_out) {
        // sequence index of r[c] is n_state + w0 + c; the end window is [len, len + n_state)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t k = S::N + w0 + c - len;
            if (k < S::N) win_out[k] = r[c];
        }
    }
    nw = make_uint4(r[0], r[1], r[2], r[3]);
}

template <int NH>
__device__ __forceinline__ void shift1(uint4 (&Hs)[NH], const uint4& nw) {
#pragma unroll
    for (int i = 0; i + 1 < NH; ++i) Hs[i] = Hs[i + 1];
    Hs[NH - 1] = nw;
}

template <uint32_t NW, int RC, int AC, int KIND, int CKM>
__device__ __forceinline__ void run6(const M6Ctx& p, uint4 (&Hs)[S6<NW>::H], uint32_t* optr, uint32_t len,
                                     uint32_t* win_out, CkAcc6<CKM>& sum, uint32_t& xr) {
    using S = S6<NW>;
    const uint32_t steps = (len + kHalfWords - 1) / kHalfWords;
    // A step at n makes sequence words [N + n, N + n + 128): no store predicate and no end
    // window while n + 128 + N <= len. The main loop runs H such steps per trip (the history
    // returns to its registers); the rest run the predicated tail variant.
    uint32_t m = 0;
    constexpr uint32_t V = KIND == MTGP_F64_01 ? 2 : 1;  // 16-byte vectors per lane per step
    uint4* dst = reinterpret_cast<uint4*>(optr) + V * p.lane;  // step m's slot: dst + 32 V m
    for (; (m + S::H) * kHalfWords + S::N <= len; m += S::H, dst += 32 * V * S::H) {
#pragma unroll
        for (uint32_t k = 0; k < S::H; ++k) {
            uint4 nw;
            step6<NW, RC, AC, KIND, CKM, false>(p, Hs, nw, dst + 32 * V * k, (m + k) * kHalfWords, len, nullptr, sum,
                                               xr);
            shift1(Hs, nw);
        }
    }
    for (; m < steps; ++m, dst += 32 * V) {
        uint4 nw;
        step6<NW, RC, AC, KIND, CKM, true>(p, Hs, nw, dst, m * kHalfWords, len, win_out, sum, xr);
        shift1(Hs, nw);
    }
}

template <uint32_t NW, int AC, int KIND, int CKM>
__device__ __forceinline__ void run6_rc(int rc, const M6Ctx& p, uint4 (&Hs)[S6<NW>::H], uint32_t* optr,
                                        uint32_t len, uint32_t* win_out, CkAcc6<CKM>& sum, uint32_t& xr) {
    switch (rc) {
        case 0: run6<NW, 0, AC, KIND, CKM>(p, Hs, optr, len, win_out, sum, xr); break;
        case 1: run6<NW, 1, AC, KIND, CKM>(p, Hs, optr, len, win_out, sum, xr); break;
        case 2: run6<NW, 2, AC, KIND, CKM>(p, Hs, optr, len, win_out, sum, xr); break;
        default: run6<NW, 3, AC, KIND, CKM>(p, Hs, optr, len, win_out, sum, xr); break;
    }
}

template <uint32_t NW, int AC, int KIND, int CKM>
__device__ __forceinline__ void run6_ac(int ac, int rc, const M6Ctx& p, uint4 (&Hs)[S6<NW>::H], uint32_t* optr,
                                        uint32_t len, uint32_t* win_out, CkAcc6<CKM>& sum, uint32_t& xr) {
    if constexpr (AC <= (int)S6<NW>::AC_MAX) {
        if (ac == AC)
            run6_rc<NW, AC, KIND, CKM>(rc, p, Hs, optr, len, win_out, sum, xr);
        else
            run6_ac<NW, AC + 1, KIND, CKM>(ac, rc, p, Hs, optr, len, win_out, sum, xr);
    }
}

}  // namespace

template <uint32_t NW, int KIND, int CKM>
__global__ void __launch_bounds__(kWarpsPerCta * 32, MTGP6_MIN_CTAS) mt_gen3_kernel(MtGenArgs a) {
    using S = S6<NW>;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t team = blockIdx.x * kWarpsPerCta + warp;
    if (team >= a.n_teams) return;
    M6Ctx p;
    p.lane = lane;
    p.srcA0 = (lane + S::BA) & 31;
    p.srcA1 = (lane + S::BA + 1) & 31;
    p.pA0 = lane < S::BA;
    p.pA1 = lane < S::BA + 1;
    p.mA0 = p.pA0;
    p.mA1 = p.pA1;
    const TeamWork tw = a.teams[team];
    for (uint32_t pi = tw.first; pi < tw.first + tw.count; ++pi) {
        const Piece pc = a.pieces[pi];
        const DevMtParams prm = a.params[pc.set];
        p.upper = prm.r ? (0xFFFFFFFFu << prm.r) : 0xFFFFFFFFu;
        p.a = prm.a;
        p.b = prm.b;
        p.c = prm.c;
        p.u = prm.u;
        p.l = prm.l;
        p.mul_s = prm.mul_s;  // 2^s, 2^t from the host: opaque, so the shifts stay IMADs
        p.mul_t = prm.mul_t;
        p.hi_u = 1u << (32 - prm.u);  // u, l in [1, 31]
        p.hi_l = 1u << (32 - prm.l);
        p.one = prm.n / S::N;  // 1, opaque to the compiler
        const uint32_t qc = (S::BASE + prm.m) >> 2;  // C stream: BASE + m = 4 qc + rc
        const int rc = (int)((S::BASE + prm.m) & 3);
        const int ac = (int)(qc >> 5);
        const uint32_t thr0 = qc & 31, thr1 = thr0 + 1;  // in [0, 32]
        p.srcC0 = (lane + thr0) & 31;
        p.srcC1 = (lane + thr1) & 31;
        p.pC0 = lane < thr0;
        p.pC1 = lane < thr1;
        p.mC0 = p.pC0;
        p.mC1 = p.pC1;
        p.neg1 = 0u - p.one;
        // u32 words or doubles (2 words each): stream stride L samples, piece offset in samples
        constexpr uint32_t kW = KIND == MTGP_F64_01 ? 2 : 1;
        uint32_t* optr = reinterpret_cast<uint32_t*>(a.out) + kW * ((size_t)pc.set * a.L + pc.offset);
        if (KIND >= kKindBitmapBit0) {
            p.bm = reinterpret_cast<uint32_t*>(a.out) + (size_t)pc.set * ((a.L + 31) / 32);
            p.poff = pc.offset;
            p.pred = a.pred;
        }
        const uint32_t len = (uint32_t)pc.len;
        const uint32_t* w0 = a.piece_win[pi];
        // history before step 0: half-step h, lane t, component c holds x_{128h + 4t + c - BASE}
        uint4 Hs[S::H];
#pragma unroll
        for (int h = 0; h < (int)S::H; ++h) {
            uint32_t v[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int k = (int)kHalfWords * h + 4 * (int)lane + c - (int)S::BASE;
                v[c] = k >= 0 ? w0[k] : 0u;
            }
            Hs[h] = make_uint4(v[0], v[1], v[2], v[3]);
        }
        uint32_t* win_out = nullptr;
        if (pc.offset + pc.len == a.L) {
            win_out = a.win_out + (size_t)pc.set * S::N;
            for (uint32_t j = lane; j + len < S::N; j += 32) win_out[j] = w0[len + j];  // pieces shorter than n
        }
        CkAcc6<CKM> sum = 0;
        uint32_t xr = 0;
        run6_ac<NW, 0, KIND, CKM>(ac, rc, p, Hs, optr, len, win_out, sum, xr);
        if (CKM) {
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                sum += __shfl_xor_sync(kFull6, sum, s);
                xr ^= __shfl_xor_sync(kFull6, xr, s);
            }
            if (lane == 0) {
                atomicAdd(&a.ck[pc.set].sum64, (unsigned long long)sum);  // mode 2: low half
                atomicXor(&a.ck[pc.set].xor32, xr);
                atomicAdd(&a.ck[pc.set].words, (unsigned long long)len);
            }
        }
        __syncwarp();
    }
}

bool mt_gen3_supports(uint32_t n, uint32_t min_gap, int kind) {
    return (kind == MTGP_U32 || kind == MTGP_F64_01 || kind == kKindBitmapBit0 || kind == kKindBitmapRange) &&
           n == 624 && min_gap >= 129;
}

template <int KIND, int CKM>
static int mt3_occ() {
    int c = 0;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, mt_gen3_kernel<624, KIND, CKM>, kWarpsPerCta * 32, 0) ==
                   cudaSuccess
               ? (KIND >= kKindBitmapBit0 ? c : std::min(c, MTGP6_MAX_CTAS))  // stat passes: as before
               : 0;
}

cudaError_t launch_mt_gen3(uint32_t n, int kind, int ck_mode, const MtGenArgs& a, cudaStream_t st) {
    if (a.n_teams == 0) return cudaSuccess;
    if (n != 624) return cudaErrorInvalidValue;
    const uint32_t grid = (a.n_teams + kWarpsPerCta - 1) / kWarpsPerCta;
    const dim3 block(kWarpsPerCta * 32);
    if (kind == kKindBitmapBit0) {  // no checksums: the words are never output
        mt_gen3_kernel<624, kKindBitmapBit0, 0><<<grid, block, 0, st>>>(a);
        return cudaGetLastError();
    }
    if (kind == kKindBitmapRange) {
        mt_gen3_kernel<624, kKindBitmapRange, 0><<<grid, block, 0, st>>>(a);
        return cudaGetLastError();
    }
    switch ((kind == MTGP_F64_01 ? 3 : kind == MTGP_U32 ? 0 : 6) + ck_mode) {
        case 0: mt_gen3_kernel<624, MTGP_U32, 0><<<grid, block, 0, st>>>(a); break;
        case 1: mt_gen3_kernel<624, MTGP_U32, 1><<<grid, block, 0, st>>>(a); break;
        case 2: mt_gen3_kernel<624, MTGP_U32, 2><<<grid, block, 0, st>>>(a); break;
        case 3: mt_gen3_kernel<624, MTGP_F64_01, 0><<<grid, block, 0, st>>>(a); break;
        case 4: mt_gen3_kernel<624, MTGP_F64_01, 1><<<grid, block, 0, st>>>(a); break;
        case 5: mt_gen3_kernel<624, MTGP_F64_01, 2><<<grid, block, 0, st>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

int mt_gen3_ctas_per_sm(uint32_t n, int kind, int ck_mode) {
    if (n != 624) return 0;
    if (kind == MTGP_U32)
        return ck_mode == 2 ? mt3_occ<MTGP_U32, 2>() : ck_mode ? mt3_occ<MTGP_U32, 1>() : mt3_occ<MTGP_U32, 0>();
    if (kind == MTGP_F64_01)
        return ck_mode == 2 ? mt3_occ<MTGP_F64_01, 2>() : ck_mode ? mt3_occ<MTGP_F64_01, 1>() : mt3_occ<MTGP_F64_01, 0>();
    if (kind == kKindBitmapBit0) return mt3_occ<kKindBitmapBit0, 0>();
    if (kind == kKindBitmapRange) return mt3_occ<kKindBitmapRange, 0>();
    return 0;
}

}  // namespace mtgpb
