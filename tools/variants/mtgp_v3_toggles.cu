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
#include "mtgp_bitmap.cuh"
#include "mtgp_v2.cuh"

namespace mtgpb {

#define FULL 0xffffffffu

#ifndef MTGP3_SH2_IMAD
#define MTGP3_SH2_IMAD 0
#endif
#ifndef MTGP3_FOLD_IMAD
#define MTGP3_FOLD_IMAD 0
#endif
#ifndef MTGP3_MIN_CTAS
#define MTGP3_MIN_CTAS 6
#endif
#ifndef MTGP3_FOLD_PAIR
#define MTGP3_FOLD_PAIR 1
#endif
#ifndef MTGP3_CK_WIDE
#define MTGP3_CK_WIDE 0
#endif
// Checksum sum on the FMA pipe without 64-bit adds: within a run of <= 2^16 words per lane, `sum`
// holds two 32-bit accumulators, A = sum(o) mod 2^32 (IMAD) and B = sum(o >> 16) mod 2^32
// (IMAD.HI); then sum(o) = 2^16 B + ((A - (B << 16)) mod 2^32) exactly (the low halves add up to
// less than 2^32). run3 folds them into the 64-bit total every 8192 steps.
#ifndef MTGP3_CK_HILO
#define MTGP3_CK_HILO 0
#endif
// float kinds: the [1,2) conversion as I2F.RZ + FFMA.RZ instead of LEA.HI on the ALU pipe
#ifndef MTGP3_FLT_FMA
#define MTGP3_FLT_FMA 0
#endif
// x << sh1 as a shift on the ALU pipe instead of an IMAD by 2^sh1 on the FMA pipe
#ifndef MTGP3_SH1_SHF
#define MTGP3_SH1_SHF 0
#endif
// Operand select on the FMA pipe: send = hi * m + lo * (1 - m) with a per-lane 0/1 multiplier
// (two IMADs instead of one SEL on the ALU pipe). 0: SEL everywhere, 1: IMAD for the A and C
// streams, 2: A only, 3: C only.
#ifndef MTGP3_SEL_IMAD
#define MTGP3_SEL_IMAD 0
#endif

namespace {

constexpr uint32_t kN = 351;  // MTGP32-11213 state words

struct V3Ctx {
    uint32_t lane;
    uint32_t mask, sh1, sh2, mul1, mulhi2, m16, m24, m23, one, tblr, tmpr;
    uint32_t srcA0, srcA1, srcC0, srcC1;  // source lanes for carry e = 0 / 1
    bool pA0, pA1, pC0, pC1;              // "take the newer half-step" predicates
    uint32_t mA0, mA1, mC0, mC1;          // the same as 0/1 multipliers (MTGP3_SEL_IMAD)
    uint32_t nA0, nA1, nC0, nC1;          // 1 - m
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
#if MTGP3_SH2_IMAD
    const uint32_t cs = __umulhi(c, p.mulhi2);
#else
    const uint32_t cs = c >> p.sh2;
#endif
#if MTGP3_SH1_SHF
    const uint32_t y = x ^ (x << p.sh1) ^ cs;
#else
    const uint32_t y = x ^ (x * p.mul1) ^ cs;
#endif
    return y ^ __shfl_sync(FULL, p.tblr, y, 16);
}

#if !MTGP3_FOLD_PAIR
__device__ __forceinline__ uint32_t temper3(const V3Ctx& p, uint32_t r, uint32_t t) {
#if MTGP3_FOLD_IMAD
    t ^= __umulhi(t, p.m16);
    t ^= __umulhi(t, p.m24);
#else
    t ^= t >> 16;
    t ^= t >> 8;
#endif
    return r ^ __shfl_sync(FULL, p.tmpr, t, 16);
}
#endif

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
__device__ __forceinline__ uint32_t conv3(const V3Ctx& p, uint32_t o) {
    if (KIND == MTGP_U32 || KIND >= kKindBitmapBit0) return o;
#if MTGP3_FLT_FMA
    // (o >> 9) | 0x3F800000 on the FMA pipe, bit-exact: I2F.RZ keeps o's top 24 significant
    // bits (what it drops is below bit 9), and the FFMA.RZ with 1.0 truncates 1 + o * 2^-32 to
    // 23 fraction bits, i.e. 1 + floor(o / 2^9) * 2^-23
    uint32_t v = __float_as_uint(__fmaf_rz(__uint2float_rz(o), 2.3283064365386963e-10f, 1.0f));
#else
    uint32_t v = (o >> 9) | 0x3F800000u;
#endif
    if (KIND == MTGP_F32_01OC) v = __float_as_uint(2.0f - __uint_as_float(v));
    return v;
}

// Five consecutive operand words for half-step U from the history half-steps
// h1 = (k=1), h2 = (k=2), h3 = (k=3); residue R; per-carry source lanes / predicates.
template <int R, int U, bool IMAD_SEL>
__device__ __forceinline__ void fetch5(uint32_t W[5], const uint4& h1, const uint4& h2, const uint4& h3, uint32_t src0,
                                       uint32_t src1, bool p0, bool p1, uint32_t m0, uint32_t m1, uint32_t n0,
                                       uint32_t n1) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int c = (R + j) & 3;
        const int e = (R + j) >> 2;
        const uint4& lo = U == 0 ? h1 : h2;  // k = 1 + U
        const uint4& hi = U == 0 ? h2 : h3;  // k = 2 + U
        uint32_t send;
        if (IMAD_SEL) {
            // inline PTX keeps the compiler from turning the 0/1 products back into a select
            uint32_t t;
            asm("mul.lo.u32 %0, %1, %2;" : "=r"(t) : "r"(comp4(lo, c)), "r"(e ? n1 : n0));
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(send) : "r"(comp4(hi, c)), "r"(e ? m1 : m0), "r"(t));
        } else
            send = (e ? p1 : p0) ? comp4(hi, c) : comp4(lo, c);
        W[j] = __shfl_sync(FULL, send, e ? src1 : src0);
    }
}

// One 256-word step. Reads history (h1: older step's upper half; h2/h3: newer step's halves),
// returns the new step's two halves in n0/n1. Stores outputs when the chunk is inside the piece.
template <int RC, int KIND, bool CK, bool TAIL>
__device__ __forceinline__ void step3(const V3Ctx& p, const uint4& h1, const uint4& h2, const uint4& h3, uint4& n0,
                                      uint4& n1, uint32_t* optr, uint32_t n, uint32_t len, uint32_t* win_out,
                                      uint32_t win_lo, unsigned long long& sum, uint32_t& xr) {
    uint32_t WA[2][5], WC[2][5];
    constexpr bool kImadA = MTGP3_SEL_IMAD == 1 || MTGP3_SEL_IMAD == 2;
    constexpr bool kImadC = MTGP3_SEL_IMAD == 1 || MTGP3_SEL_IMAD == 3;
    fetch5<1, 0, kImadA>(WA[0], h1, h2, h3, p.srcA0, p.srcA1, p.pA0, p.pA1, p.mA0, p.mA1, p.nA0, p.nA1);
    fetch5<1, 1, kImadA>(WA[1], h1, h2, h3, p.srcA0, p.srcA1, p.pA0, p.pA1, p.mA0, p.mA1, p.nA0, p.nA1);
    fetch5<RC, 0, kImadC>(WC[0], h1, h2, h3, p.srcC0, p.srcC1, p.pC0, p.pC1, p.mC0, p.mC1, p.nC0, p.nC1);
    fetch5<RC, 1, kImadC>(WC[1], h1, h2, h3, p.srcC0, p.srcC1, p.pC0, p.pC1, p.mC0, p.mC1, p.nC0, p.nC1);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        uint32_t r[4], o[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) r[c] = rec3(p, WA[u][c], WA[u][c + 1], WC[u][c + 1]);
#if MTGP3_FOLD_PAIR
        uint32_t ix[4];
        fold2(WC[u][0], WC[u][1], ix[0], ix[1]);
        fold2(WC[u][2], WC[u][3], ix[2], ix[3]);
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = conv3<KIND>(p, r[c] ^ __shfl_sync(FULL, p.tmpr, ix[c], 16));
#else
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = conv3<KIND>(p, temper3(p, r[c], WC[u][c]));
#endif
        const uint32_t w0 = n + 128 * u + 4 * p.lane;  // piece word of o[0]
        if constexpr (KIND >= kKindBitmapBit0) {
            bitmap_store<KIND>(p.lane, p.bm, p.poff, p.pred, o, n + 128 * u, !TAIL || w0 < len);
        } else if (!TAIL || w0 < len) {
            __stcs(reinterpret_cast<uint4*>(optr + w0), make_uint4(o[0], o[1], o[2], o[3]));
            if (CK) {
#if MTGP3_CK_HILO
                uint32_t ca = (uint32_t)sum, cb = (uint32_t)(sum >> 32);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(ca) : "r"(o[c]), "r"(p.one));
                    asm("mad.hi.u32 %0, %1, %2, %0;" : "+r"(cb) : "r"(o[c]), "r"(p.m16));
                }
                sum = ((unsigned long long)cb << 32) | ca;
#elif MTGP3_CK_WIDE
                // 64-bit sum on the FMA pipe: IMAD.WIDE.U32 sum = o * one + sum (one is opaque)
#pragma unroll
                for (int c = 0; c < 4; ++c) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(sum) : "r"(o[c]), "r"(p.one));
#else
#pragma unroll
                for (int c = 0; c < 4; ++c) sum += o[c];
#endif
                xr ^= o[0] ^ o[1] ^ o[2] ^ o[3];
            }
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

#if MTGP3_CK_HILO
// packed (A, B) accumulators -> the exact sum of the words they saw
__device__ __forceinline__ unsigned long long hilo_sum(unsigned long long packed) {
    const uint32_t a = (uint32_t)packed, b = (uint32_t)(packed >> 32);
    return ((unsigned long long)b << 16) + (uint32_t)(a - (b << 16));
}
#endif

template <int RC, int KIND, bool CK>
__device__ __forceinline__ void run3(const V3Ctx& p, uint4 X0, uint4 X1, uint4 Y1, uint32_t* optr, uint32_t len,
                                     uint32_t* win_out, unsigned long long& sum, uint32_t& xr) {
    // ping-pong: even steps read (Y1 | X0, X1) and write Y; odd steps read (X1 | Y0, Y1), write X
    uint4 Y0;
    const uint32_t steps = (len + kStepWords - 1) / kStepWords;
    // A step at n produces sequence words [N + n, N + n + 256). It needs no store predicate and
    // cannot reach the end window [len, len + N) while n + 256 + N <= len: the main loop runs
    // pairs of such steps; the (at most three) remaining steps run the predicated tail variant.
    uint32_t m = 0;
#if MTGP3_CK_HILO
    unsigned long long tot = sum;
    sum = 0;
#endif
    for (; (m + 2) * kStepWords + kN <= len; m += 2) {
        step3<RC, KIND, CK, false>(p, Y1, X0, X1, Y0, Y1, optr, m * kStepWords, len, nullptr, len, sum, xr);
        step3<RC, KIND, CK, false>(p, X1, Y0, Y1, X0, X1, optr, (m + 1) * kStepWords, len, nullptr, len, sum, xr);
#if MTGP3_CK_HILO
        if (CK && (m & 8190u) == 8190u) {  // 8192 steps = 2^16 words per lane
            tot += hilo_sum(sum);
            sum = 0;
        }
#endif
    }
#if MTGP3_CK_HILO
    if (CK) {
        tot += hilo_sum(sum);
        sum = 0;
    }
#endif
    while (m < steps) {
        step3<RC, KIND, CK, true>(p, Y1, X0, X1, Y0, Y1, optr, m * kStepWords, len, win_out, len, sum, xr);
        if (++m >= steps) break;
        step3<RC, KIND, CK, true>(p, X1, Y0, Y1, X0, X1, optr, m * kStepWords, len, win_out, len, sum, xr);
        ++m;
    }
#if MTGP3_CK_HILO
    if (CK) sum = tot + hilo_sum(sum);
#endif
}

}  // namespace

template <int KIND, bool CK>
__global__ void __launch_bounds__(kWarpsPerCta * 32, MTGP3_MIN_CTAS) gen3_kernel(GenArgs a) {
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
    p.nA0 = 1u - p.mA0;
    p.nA1 = 1u - p.mA1;
    const TeamWork tw = a.teams[team];
    for (uint32_t pi = tw.first; pi < tw.first + tw.count; ++pi) {
        const Piece pc = a.pieces[pi];
        const DevParams& prm = a.params[pc.set];
        p.mask = prm.mask;
        p.sh1 = prm.sh1;
        p.sh2 = prm.sh2;
        p.mul1 = prm.mul1;
        p.mulhi2 = prm.mulhi2;
        p.m16 = prm.m16;
        p.m24 = prm.m24;
        p.m23 = prm.m23;
        p.one = prm.one;
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
        p.nC0 = 1u - p.mC0;
        p.nC1 = 1u - p.mC1;
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
        unsigned long long sum = 0;
        uint32_t xr = 0;
        switch (pos & 3u) {
            case 0: run3<0, KIND, CK>(p, X0, X1, Y1, optr, len, win_out, sum, xr); break;
            case 1: run3<1, KIND, CK>(p, X0, X1, Y1, optr, len, win_out, sum, xr); break;
            case 2: run3<2, KIND, CK>(p, X0, X1, Y1, optr, len, win_out, sum, xr); break;
            default: run3<3, KIND, CK>(p, X0, X1, Y1, optr, len, win_out, sum, xr); break;
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
static cudaError_t launch3_t(const GenArgs& a, cudaStream_t st) {
    const uint32_t grid = (a.n_teams + kWarpsPerCta - 1) / kWarpsPerCta;
    gen3_kernel<KIND, CK><<<grid, kWarpsPerCta * 32, 0, st>>>(a);
    return cudaGetLastError();
}

template <int KIND, bool CK>
static int occ3_t() {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gen3_kernel<KIND, CK>, kWarpsPerCta * 32, 0) != cudaSuccess)
        return 0;
    return n;
}

cudaError_t launch_gen3(int kind, bool cksum, const GenArgs& a, cudaStream_t st) {
    if (a.n_teams == 0) return cudaSuccess;
    switch (kind * 2 + (cksum ? 1 : 0)) {
        case 0: return launch3_t<MTGP_U32, false>(a, st);
        case 1: return launch3_t<MTGP_U32, true>(a, st);
        case 2: return launch3_t<MTGP_F32_12, false>(a, st);
        case 3: return launch3_t<MTGP_F32_12, true>(a, st);
        case 4: return launch3_t<MTGP_F32_01OC, false>(a, st);
        case 5: return launch3_t<MTGP_F32_01OC, true>(a, st);
    }
    // bitmap kinds carry no checksums (the words are never output)
    if (kind == kKindBitmapBit0) return launch3_t<kKindBitmapBit0, false>(a, st);
    if (kind == kKindBitmapRange) return launch3_t<kKindBitmapRange, false>(a, st);
    return cudaErrorInvalidValue;
}

int gen3_ctas_per_sm(int kind, bool cksum) {
    switch (kind * 2 + (cksum ? 1 : 0)) {
        case 0: return occ3_t<MTGP_U32, false>();
        case 1: return occ3_t<MTGP_U32, true>();
        case 2: return occ3_t<MTGP_F32_12, false>();
        case 3: return occ3_t<MTGP_F32_12, true>();
        case 4: return occ3_t<MTGP_F32_01OC, false>();
        case 5: return occ3_t<MTGP_F32_01OC, true>();
    }
    if (kind == kKindBitmapBit0) return occ3_t<kKindBitmapBit0, false>();
    if (kind == kKindBitmapRange) return occ3_t<kKindBitmapRange, false>();
    return 0;
}

}  // namespace mtgpb
