// tools/variants/mtgp_v3_lerp_masksel.cu -- gen3 with the round-2 select experiments (MTGP3_LERP: FMA-pipe
// select lo + m*(hi-lo); MTGP3_MASKSEL: LOP3 mask select without predicate ISETPs). Both measured
// no faster (profiles/r2/gen3_lerp_ck_sweep.jsonl, r2/gen3_masksel_sweep.jsonl) and were removed from
// the product kernel; build with VARIANT_SRCS and tools/sweep_variants.sh by copying over csrc/mtgp_v3.cu.
// Original header:
// mtgp_v3.cu -- register-resident MTGP32-11213 generation (no shared memory on the hot path).
//
// Same decomposition as v2 (one warp per jump-ahead piece, 256-word steps, lane t owns words
// 4t..4t+3 and 128+4t..128+4t+3 of a step, two coalesced STG.128), but the state words never
// go to shared memory. Each lane keeps its own newly produced words of the last two steps in
// registers (only 3 of the 4 half-steps are ever read again: 12 live registers), and every
// operand a lane needs is shuffled in from the lane that produced it:
//
//   operand x_{256m + 128u + 4t + j + off}  (A stream: off = 0; C stream: off = pos - 1),
//   j = 0..4, sits at history position P = 161 + off + 128u + 4t + j  (512 - N = 161)
//   counted from the start of step m-2. With 161 + off = 4*Q0 + R (R = residue):
//     component c' = (R + j) mod 4, carry e = (R + j) div 4,
//     source lane  s = (t + Q0 + e) mod 32,
//     half-step    k = 1 + u + [s < thr_e],  thr_e = (Q0 + e) - 32  (in [8, 32]).
//   So every destination word is ONE shfl.idx from a fixed source lane, whose sent value is ONE
//   SEL between two of the lane's history registers. A: Q0 = 40, R = 1 (compile time).
//   C: Q0 = 40 + pos/4, R = pos mod 4 (four unrolled variants; thresholds per piece).
//
// Per 256-word step per warp: 20 operand SHFL + 16 table SHFL + 2 STG.128 (LSU data-pipe
// wavefronts 44, vs 59 for the shared-memory ring of v2).
#include <type_traits>

#include "mtgp_bitmap.cuh"
#include "mtgp_v2.cuh"

namespace mtgpb {

#define FULL 0xffffffffu


// Occupancy target: 6 CTAs x 4 warps per SM (80 registers). The pipe-balance variants that
// measured slower in round 1 (IMAD.HI shifts, FMA-pipe selects and checksums, ...) are kept in
// tools/variants/mtgp_v3_toggles.cu, their sweeps under profiles/r1_v3_*_sweep.jsonl.
constexpr int kMinCtas3 = 6;
// Operand select of the A (bit 0) / C (bit 1) stream on the FMA pipe: send = lo + m * (hi - lo)
// with a per-lane 0/1 multiplier m and the differences hi - lo formed once per half-step pair by
// IMAD (lo * -1 + hi), shared by both streams. One IMAD per fetch instead of one ALU SEL.
#ifndef MTGP3_LERP
#define MTGP3_LERP 0
#endif
// Operand select as one LOP3 with a per-lane all-ones / all-zeros mask register instead of
// SEL on a predicate (bit 0: A stream, bit 1: C stream): the same ALU op count, but the four
// lane predicates no longer have to be rematerialised by ISETPs on every trip.
#ifndef MTGP3_MASKSEL
#define MTGP3_MASKSEL 0
#endif

namespace {

constexpr uint32_t kN = 351;  // MTGP32-11213 state words

// Checksum modes (MTGP_OPT_CHECKSUM): 0 none; 1 sum64 + xor32; 2 sum32 + xor32 -- the sum of the
// emitted words mod 2^32 in a 32-bit accumulator (one 3-input IADD3 per two words, no carry
// chain), reported in the low half of mtgp_cksum.sum64.
template <int CKM>
using CkAcc = typename std::conditional<CKM == 2, uint32_t, unsigned long long>::type;

struct V3Ctx {
    uint32_t lane;
    uint32_t mask, sh2, mul1, tblr, tmpr;
    uint32_t srcA0, srcA1, srcC0, srcC1;  // source lanes for carry e = 0 / 1
    bool pA0, pA1, pC0, pC1;              // "take the newer half-step" predicates
    uint32_t mA0, mA1, mC0, mC1;          // the same as 0/1 multipliers (MTGP3_LERP)
    uint32_t kA0, kA1, kC0, kC1;          // ... and as 0 / ~0 masks (MTGP3_MASKSEL)
    uint32_t neg1;                        // 0xFFFFFFFF, opaque to the compiler
    // bitmap kinds: this stream's bitmap, the piece's first word within the call, the predicate
    uint32_t* bm;
    unsigned long long poff;
    BitmapPred pred;
};

__device__ __forceinline__ uint32_t comp4(const uint4& g, int c) {
    return c == 0 ? g.x : c == 1 ? g.y : c == 2 ? g.z : g.w;
}

__device__ __forceinline__ uint32_t rec3(const V3Ctx& p, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t x = (a & p.mask) ^ b;
    // x << sh1 as an IMAD by 2^sh1 (FMA pipe; the ALU pipe is the busier one)
    const uint32_t y = x ^ (x * p.mul1) ^ (c >> p.sh2);
    return y ^ __shfl_sync(FULL, p.tblr, y, 16);
}

// Tempering indices of two words at once: the XOR of the low nibbles of each word's four bytes.
// Halves are paired with byte permutes so one LOP3/SHF serves both words (6 ALU ops per two
// words instead of 8): w = (t1.lo16 ^ t1.hi16) | (t2.lo16 ^ t2.hi16) << 16; z = w ^ (w >> 8).
__device__ __forceinline__ void fold2(uint32_t t1, uint32_t t2, uint32_t& i1, uint32_t& i2) {
    const uint32_t w = __byte_perm(t1, t2, 0x5410) ^ __byte_perm(t1, t2, 0x7632);
    const uint32_t z = w ^ (w >> 8);
    i1 = z;        // bits [3:0]; shfl.idx over 16-lane segments ignores the rest
    i2 = z >> 16;
}

template <int KIND>
__device__ __forceinline__ uint32_t conv3(uint32_t o) {
    if (KIND == MTGP_U32 || KIND >= kKindBitmapBit0) return o;
    uint32_t v = (o >> 9) | 0x3F800000u;
    if (KIND == MTGP_F32_01OC) v = __float_as_uint(2.0f - __uint_as_float(v));
    return v;
}

// Five consecutive operand words for half-step U from the history half-steps
// h1 = (k=1), h2 = (k=2), h3 = (k=3); residue R; per-carry source lanes / predicates.
// LERP: the select is lo + m * d with d = hi - lo (dU: the differences of this half-step pair).
template <int R, int U, bool LERP, bool MSEL>
__device__ __forceinline__ void fetch5(uint32_t W[5], const uint4& h1, const uint4& h2, const uint4& h3, const uint4& dU,
                                       uint32_t src0, uint32_t src1, bool p0, bool p1, uint32_t m0, uint32_t m1,
                                       uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int c = (R + j) & 3;
        const int e = (R + j) >> 2;
        const uint4& lo = U == 0 ? h1 : h2;  // k = 1 + U
        const uint4& hi = U == 0 ? h2 : h3;  // k = 2 + U
        uint32_t send;
        if (LERP)
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(send) : "r"(comp4(dU, c)), "r"(e ? m1 : m0), "r"(comp4(lo, c)));
        else if (MSEL)  // (hi & k) | (lo & ~k)
            asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(send) : "r"(comp4(hi, c)), "r"(comp4(lo, c)), "r"(e ? k1 : k0));
        else
            send = (e ? p1 : p0) ? comp4(hi, c) : comp4(lo, c);
        W[j] = __shfl_sync(FULL, send, e ? src1 : src0);
    }
}

__device__ __forceinline__ uint32_t diff1(uint32_t hi, uint32_t lo, uint32_t neg1) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(lo), "r"(neg1), "r"(hi));
    return d;
}

__device__ __forceinline__ uint4 diff4(const uint4& hi, const uint4& lo, uint32_t neg1) {
    return make_uint4(diff1(hi.x, lo.x, neg1), diff1(hi.y, lo.y, neg1), diff1(hi.z, lo.z, neg1),
                      diff1(hi.w, lo.w, neg1));
}

// One 256-word step. Reads history (h1: older step's upper half; h2/h3: newer step's halves),
// returns the new step's two halves in n0/n1. Stores outputs when the chunk is inside the piece.
// sp: this lane's 16-byte output slot of the step's first half (piece word n + 4 * lane).
template <int RC, int KIND, int CKM, bool TAIL>
__device__ __forceinline__ void step3(const V3Ctx& p, const uint4& h1, const uint4& h2, const uint4& h3, uint4& n0,
                                      uint4& n1, uint4* sp, uint32_t n, uint32_t len, uint32_t* win_out,
                                      uint32_t win_lo, CkAcc<CKM>& sum, uint32_t& xr) {
    uint32_t WA[2][5], WC[2][5];
    constexpr bool kLerpA = MTGP3_LERP & 1, kLerpC = MTGP3_LERP & 2;
    uint4 d0 = h1, d1 = h2;
    if (kLerpA || kLerpC) {
        d0 = diff4(h2, h1, p.neg1);
        d1 = diff4(h3, h2, p.neg1);
    }
    constexpr bool kMselA = MTGP3_MASKSEL & 1, kMselC = MTGP3_MASKSEL & 2;
    fetch5<1, 0, kLerpA, kMselA>(WA[0], h1, h2, h3, d0, p.srcA0, p.srcA1, p.pA0, p.pA1, p.mA0, p.mA1, p.kA0, p.kA1);
    fetch5<1, 1, kLerpA, kMselA>(WA[1], h1, h2, h3, d1, p.srcA0, p.srcA1, p.pA0, p.pA1, p.mA0, p.mA1, p.kA0, p.kA1);
    fetch5<RC, 0, kLerpC, kMselC>(WC[0], h1, h2, h3, d0, p.srcC0, p.srcC1, p.pC0, p.pC1, p.mC0, p.mC1, p.kC0,
                                  p.kC1);
    fetch5<RC, 1, kLerpC, kMselC>(WC[1], h1, h2, h3, d1, p.srcC0, p.srcC1, p.pC0, p.pC1, p.mC0, p.mC1, p.kC0,
                                  p.kC1);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        uint32_t r[4], o[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) r[c] = rec3(p, WA[u][c], WA[u][c + 1], WC[u][c + 1]);
        uint32_t ix[4];
        fold2(WC[u][0], WC[u][1], ix[0], ix[1]);
        fold2(WC[u][2], WC[u][3], ix[2], ix[3]);
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = conv3<KIND>(r[c] ^ __shfl_sync(FULL, p.tmpr, ix[c], 16));
        const uint32_t w0 = n + 128 * u + 4 * p.lane;  // piece word of o[0]
        if constexpr (KIND >= kKindBitmapBit0) {
            bitmap_store<KIND>(p.lane, p.bm, p.poff, p.pred, o, n + 128 * u, !TAIL || w0 < len);
        } else if (!TAIL || w0 < len) {
            __stcs(sp + 32 * u, make_uint4(o[0], o[1], o[2], o[3]));
            if (CKM == 2) {
                sum = sum + o[0] + o[1];  // 3-input IADD3s, mod 2^32
                sum = sum + o[2] + o[3];
            } else if (CKM == 1) {
#pragma unroll
                for (int c = 0; c < 4; ++c) sum += o[c];
            }
            if (CKM) xr ^= o[0] ^ o[1] ^ o[2] ^ o[3];
        }
        if (TAIL && win_out) {
            // sequence index of r[c] is kN + w0 + c; the end window is [len, len + kN)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t k = kN + w0 + c - win_lo;
                if (k < kN) win_out[k] = r[c];
            }
        }
        if (u == 0)
            n0 = make_uint4(r[0], r[1], r[2], r[3]);
        else
            n1 = make_uint4(r[0], r[1], r[2], r[3]);
    }
}

// Steps per main-loop trip (even: the history ping-pong returns to its registers every 2 steps).
#ifndef MTGP3_UNROLL
#define MTGP3_UNROLL 2
#endif

template <int RC, int KIND, int CKM>
__device__ __forceinline__ void run3(const V3Ctx& p, uint4 X0, uint4 X1, uint4 Y1, uint32_t* optr, uint32_t len,
                                     uint32_t* win_out, CkAcc<CKM>& sum, uint32_t& xr) {
    // ping-pong: even steps read (Y1 | X0, X1) and write Y; odd steps read (X1 | Y0, Y1), write X
    uint4 Y0;
    const uint32_t steps = (len + kStepWords - 1) / kStepWords;
    // A step at n produces sequence words [N + n, N + n + 256). It needs no store predicate and
    // cannot reach the end window [len, len + N) while n + 256 + N <= len: the main loop runs
    // such steps (MTGP3_UNROLL per trip, then pairs) with a running store pointer and a trip
    // count; the (at most three) remaining steps run the predicated tail variant.
    constexpr uint32_t U = MTGP3_UNROLL;
    uint4* sp = reinterpret_cast<uint4*>(optr) + p.lane;
    const uint32_t full = len > kN ? (len - kN) / kStepWords : 0;  // steps without predicates
    uint32_t m = 0;
    if (U > 2) {
        for (uint32_t it = full / U; it; --it, sp += 64 * U, m += U) {
#pragma unroll
            for (uint32_t q = 0; q < U; q += 2) {
                step3<RC, KIND, CKM, false>(p, Y1, X0, X1, Y0, Y1, sp + 64 * q, (m + q) * kStepWords, len, nullptr, len,
                                            sum, xr);
                step3<RC, KIND, CKM, false>(p, X1, Y0, Y1, X0, X1, sp + 64 * q + 64, (m + q + 1) * kStepWords, len,
                                            nullptr, len, sum, xr);
            }
        }
    }
    for (uint32_t it = (full - m) / 2; it; --it, sp += 128, m += 2) {
        step3<RC, KIND, CKM, false>(p, Y1, X0, X1, Y0, Y1, sp, m * kStepWords, len, nullptr, len, sum, xr);
        step3<RC, KIND, CKM, false>(p, X1, Y0, Y1, X0, X1, sp + 64, (m + 1) * kStepWords, len, nullptr, len, sum, xr);
    }
    while (m < steps) {
        step3<RC, KIND, CKM, true>(p, Y1, X0, X1, Y0, Y1, sp, m * kStepWords, len, win_out, len, sum, xr);
        sp += 64;
        if (++m >= steps) break;
        step3<RC, KIND, CKM, true>(p, X1, Y0, Y1, X0, X1, sp, m * kStepWords, len, win_out, len, sum, xr);
        sp += 64;
        ++m;
    }
}

}  // namespace

template <int KIND, int CKM>
__global__ void __launch_bounds__(kWarpsPerCta * 32, kMinCtas3) gen3_kernel(GenArgs a) {
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t team = blockIdx.x * kWarpsPerCta + warp;
    if (team >= a.n_teams) return;
    V3Ctx p;
    p.lane = lane;
    p.srcA0 = (lane + 8) & 31;
    p.srcA1 = (lane + 9) & 31;
    p.pA0 = lane < 8;
    p.pA1 = lane < 9;
    p.mA0 = p.pA0;
    p.mA1 = p.pA1;
    // all-ones when lane < threshold: an arithmetic shift of (lane - thr), opaque to the
    // predicate analysis that would turn the LOP3 back into a SEL
    p.kA0 = (uint32_t)((int32_t)(lane - 8) >> 31);
    p.kA1 = (uint32_t)((int32_t)(lane - 9) >> 31);
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
        const uint32_t thr0 = 8 + (pos >> 2), thr1 = thr0 + 1;  // in [8, 32]
        p.srcC0 = (lane + thr0) & 31;
        p.srcC1 = (lane + thr1) & 31;
        p.pC0 = lane < thr0;
        p.pC1 = lane < thr1;
        p.mC0 = p.pC0;
        p.mC1 = p.pC1;
        p.kC0 = (uint32_t)((int32_t)(lane - thr0) >> 31);
        p.kC1 = (uint32_t)((int32_t)(lane - thr1) >> 31);
        p.neg1 = 0u - prm.one;
        uint32_t* optr = reinterpret_cast<uint32_t*>(a.out) + (size_t)pc.set * a.L + pc.offset;
        if (KIND >= kKindBitmapBit0) {
            p.bm = reinterpret_cast<uint32_t*>(a.out) + (size_t)pc.set * ((a.L + 31) / 32);
            p.poff = pc.offset;
            p.pred = a.pred;
        }
        const uint32_t len = (uint32_t)pc.len;
        const uint32_t* w0 = a.piece_win[pi];
        // history before step 0: X = "step -1" = x_{95+p}, Y.upper = "step -2" upper = x_{-33+4t+c}
        uint4 X0, X1, Y1;
        {
            uint32_t v[12];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                v[c] = w0[95 + 4 * lane + c];
                v[4 + c] = w0[223 + 4 * lane + c];
                const int k = -33 + 4 * (int)lane + c;
                v[8 + c] = k >= 0 ? w0[k] : 0u;
            }
            X0 = make_uint4(v[0], v[1], v[2], v[3]);
            X1 = make_uint4(v[4], v[5], v[6], v[7]);
            Y1 = make_uint4(v[8], v[9], v[10], v[11]);
        }
        uint32_t* win_out = nullptr;
        if (pc.offset + pc.len == a.L) {
            win_out = a.win_out + (size_t)pc.set * kN;
            // window words that are still start-window words (pieces shorter than N)
            for (uint32_t j = lane; j + len < kN; j += 32) win_out[j] = w0[len + j];
        }
        CkAcc<CKM> sum = 0;
        uint32_t xr = 0;
        switch (pos & 3u) {
            case 0: run3<0, KIND, CKM>(p, X0, X1, Y1, optr, len, win_out, sum, xr); break;
            case 1: run3<1, KIND, CKM>(p, X0, X1, Y1, optr, len, win_out, sum, xr); break;
            case 2: run3<2, KIND, CKM>(p, X0, X1, Y1, optr, len, win_out, sum, xr); break;
            default: run3<3, KIND, CKM>(p, X0, X1, Y1, optr, len, win_out, sum, xr); break;
        }
        if (CKM) {
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                sum += __shfl_xor_sync(FULL, sum, s);
                xr ^= __shfl_xor_sync(FULL, xr, s);
            }
            if (lane == 0) {
                // mode 2 adds the piece's sum mod 2^32: only the low half of sum64 is meaningful
                // (mtgp_checksums masks the high half for contexts that ran mode 2)
                atomicAdd(&a.ck[pc.set].sum64, (unsigned long long)sum);
                atomicXor(&a.ck[pc.set].xor32, xr);
                atomicAdd(&a.ck[pc.set].words, (unsigned long long)len);
            }
        }
        __syncwarp();
    }
}

template <int KIND, int CKM>
static cudaError_t launch3_t(const GenArgs& a, cudaStream_t st) {
    const uint32_t grid = (a.n_teams + kWarpsPerCta - 1) / kWarpsPerCta;
    gen3_kernel<KIND, CKM><<<grid, kWarpsPerCta * 32, 0, st>>>(a);
    return cudaGetLastError();
}

template <int KIND, int CKM>
static int occ3_t() {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gen3_kernel<KIND, CKM>, kWarpsPerCta * 32, 0) != cudaSuccess)
        return 0;
    return n;
}

cudaError_t launch_gen3(int kind, int ck_mode, const GenArgs& a, cudaStream_t st) {
    if (a.n_teams == 0) return cudaSuccess;
    switch (kind * 3 + ck_mode) {
        case 0: return launch3_t<MTGP_U32, 0>(a, st);
        case 1: return launch3_t<MTGP_U32, 1>(a, st);
        case 2: return launch3_t<MTGP_U32, 2>(a, st);
        case 3: return launch3_t<MTGP_F32_12, 0>(a, st);
        case 4: return launch3_t<MTGP_F32_12, 1>(a, st);
        case 5: return launch3_t<MTGP_F32_12, 2>(a, st);
        case 6: return launch3_t<MTGP_F32_01OC, 0>(a, st);
        case 7: return launch3_t<MTGP_F32_01OC, 1>(a, st);
        case 8: return launch3_t<MTGP_F32_01OC, 2>(a, st);
    }
    // bitmap kinds carry no checksums (the words are never output)
    if (kind == kKindBitmapBit0) return launch3_t<kKindBitmapBit0, 0>(a, st);
    if (kind == kKindBitmapRange) return launch3_t<kKindBitmapRange, 0>(a, st);
    return cudaErrorInvalidValue;
}

int gen3_ctas_per_sm(int kind, int ck_mode) {
    switch (kind * 3 + ck_mode) {
        case 0: return occ3_t<MTGP_U32, 0>();
        case 1: return occ3_t<MTGP_U32, 1>();
        case 2: return occ3_t<MTGP_U32, 2>();
        case 3: return occ3_t<MTGP_F32_12, 0>();
        case 4: return occ3_t<MTGP_F32_12, 1>();
        case 5: return occ3_t<MTGP_F32_12, 2>();
        case 6: return occ3_t<MTGP_F32_01OC, 0>();
        case 7: return occ3_t<MTGP_F32_01OC, 1>();
        case 8: return occ3_t<MTGP_F32_01OC, 2>();
    }
    if (kind == kKindBitmapBit0) return occ3_t<kKindBitmapBit0, 0>();
    if (kind == kKindBitmapRange) return occ3_t<kKindBitmapRange, 0>();
    return 0;
}

}  // namespace mtgpb
