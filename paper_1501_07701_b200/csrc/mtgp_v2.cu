// mtgp_v2.cu -- the B200 throughput path for MTGP32.
//
// Work decomposition. A call asks for L words of each of S streams. The S*L words are split
// into "pieces" (contiguous ranges of one stream) so that every resident warp on the GPU has the
// same amount of work; a piece that does not start at the stream's current position starts
// from a GF(2) jump-ahead of the stream's state (mtgp_plan.cu computes x^offset mod P on the
// host, jump_flat_kernel below applies it on the device). One WARP ("team") owns a piece at a time
// and keeps the piece's state in a private shared-memory ring; it needs no CTA barrier, only
// __syncwarp between steps.
//
// gen_kernel step (256 words per warp; safe because any d <= N - pos consecutive MTGP words are
// independent): lane t produces words 4t..4t+3 and 128+4t..128+4t+3 of the
// step, so the two output STG.128 of a warp are each 512 contiguous bytes (fully coalesced),
// and the new state words go to the ring with two aligned STS.128. The four ring operands a
// word needs (x[i], x[i+1], x[i+pos], x[i+pos-1]) are read as aligned LDS.128 groups; the
// 1..4 words a lane needs from its neighbour's group come over shfl. The ring phase is chosen
// per piece so that stores are 16-byte aligned in both the ring and global memory; the
// residues of the two read streams are then (-N) mod 4 (compile time) and (pos-1-N) mod 4
// (runtime, dispatched to one of four unrolled variants). The recursion table and the
// tempering table live in registers (lane l holds entry l & 15) and are looked up with
// shfl.idx over 16-lane segments -- no index masking, no shared-memory table traffic.
// Tempering, the float conversions and the checksums are fused into the same pass.
#include <cstdio>

#include "mtgp_v2.cuh"

namespace mtgpb {

#define FULL 0xffffffffu

// Pipe-balance switches (tools/sweep_variants.sh measures them on the B200):
// move a shift onto the FMA pipe (IMAD / IMAD.HI by an opaque power of two) or keep it on the
// ALU pipe (SHF); accumulate sum64 with IMAD.WIDE or IADD3 carry chains; CTAs/SM register target.
#ifndef MTGP_SH1_IMAD
#define MTGP_SH1_IMAD 1
#endif
#ifndef MTGP_SH2_IMAD
#define MTGP_SH2_IMAD 0
#endif
#ifndef MTGP_FOLD_IMAD
#define MTGP_FOLD_IMAD 0
#endif
#ifndef MTGP_CK_WIDE
#define MTGP_CK_WIDE 0
#endif
#ifndef MTGP_MIN_CTAS
#define MTGP_MIN_CTAS 6
#endif

constexpr uint32_t cpow2(uint32_t v) {
    uint32_t r = 1;
    while (r < v) r <<= 1;
    return r;
}

template <uint32_t MEXP>
struct Shape {
    static constexpr uint32_t N = MEXP / 32 + 1;
    static constexpr uint32_t R = cpow2(N + kStepWords + 8);
    static constexpr uint32_t RM = R - 1;
    static constexpr uint32_t RA = (4u - (N & 3u)) & 3u;  // (-N) mod 4
};

uint32_t v2_ring_words(uint32_t mexp) {
    switch (mexp) {
        case 11213: return Shape<11213>::R;
        case 23209: return Shape<23209>::R;
        case 44497: return Shape<44497>::R;
    }
    return 0;
}

bool v2_supports(uint32_t mexp) { return v2_ring_words(mexp) != 0; }

__device__ __forceinline__ uint32_t comp(const uint4& g, int c) {
    return c == 0 ? g.x : c == 1 ? g.y : c == 2 ? g.z : g.w;
}

// ---- shared-window helpers: 32-bit shared addresses, explicit vector accesses ----
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t x) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(x) : "memory");
}
__device__ __forceinline__ uint32_t umulhi(uint32_t a, uint32_t b) { return __umulhi(a, b); }

struct PieceCtx {
    uint32_t rb;   // shared-window byte address of the ring (aligned to its size)
    uint32_t phi;  // slot(x_j) = (j + phi) & RM
    uint32_t lane;
    uint32_t pos, mask, sh1, sh2, mul1, mulhi2, m16, m24, m23, one, tblr, tmpr;
    uint32_t* optr;
};

// para_rec (external pin curand_mtgp32_kernel.h:137-145) with both shifts
// on the FMA pipe (IMAD / IMAD.HI by opaque powers of two) so the ALU pipe only sees LOP3s.
__device__ __forceinline__ uint32_t rec_f(const PieceCtx& p, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t x = (a & p.mask) ^ b;
#if MTGP_SH1_IMAD
    const uint32_t xs = x * p.mul1;
#else
    const uint32_t xs = x << p.sh1;
#endif
#if MTGP_SH2_IMAD
    const uint32_t cs = umulhi(c, p.mulhi2);
#else
    const uint32_t cs = c >> p.sh2;
#endif
    const uint32_t y = x ^ xs ^ cs;
    return y ^ __shfl_sync(FULL, p.tblr, y, 16);
}

// temper (curand_mtgp32_kernel.h:155-162): the index is the XOR of the low nibbles of T's
// four bytes; shfl.idx over a 16-lane segment reads only index bits [3:0].
__device__ __forceinline__ uint32_t temper_f(const PieceCtx& p, uint32_t r, uint32_t t) {
#if MTGP_FOLD_IMAD
    t ^= umulhi(t, p.m16);
    t ^= umulhi(t, p.m24);
#else
    t ^= t >> 16;
    t ^= t >> 8;
#endif
    return r ^ __shfl_sync(FULL, p.tmpr, t, 16);
}

template <int KIND>
__device__ __forceinline__ uint32_t conv_f(const PieceCtx& p, uint32_t o) {
    if (KIND == MTGP_U32) return o;
    uint32_t v = umulhi(o, p.m23) | 0x3F800000u;                               // [1,2)
    if (KIND == MTGP_F32_01OC) v = __float_as_uint(2.0f - __uint_as_float(v));  // (0,1]
    return v;
}

template <bool CK>
__device__ __forceinline__ void ck_add(const PieceCtx& p, unsigned long long& sum, uint32_t v) {
#if MTGP_CK_WIDE
    if (CK) asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(sum) : "r"(v), "r"(p.one));
#else
    if (CK) sum += v;
#endif
}

// Words [n0, n0+cnt) of the piece, one per lane, cnt <= 255 (all independent).
template <uint32_t MEXP, int KIND, bool CK>
__device__ __forceinline__ void scalar_words(const PieceCtx& p, uint32_t n0, uint32_t cnt, unsigned long long& sum,
                                             uint32_t& xr) {
    using S = Shape<MEXP>;
    constexpr uint32_t RMB = S::R * 4 - 1;
    for (uint32_t base = 0; base < cnt; base += 32) {
        const uint32_t n = n0 + base + p.lane;
        const bool act = base + p.lane < cnt;
        const uint32_t nb = (n + p.phi) * 4;
        const uint32_t a = lds32(p.rb + (nb & RMB));
        const uint32_t b = lds32(p.rb + ((nb + 4) & RMB));
        const uint32_t c = lds32(p.rb + ((nb + 4 * p.pos) & RMB));
        const uint32_t t = lds32(p.rb + ((nb + 4 * p.pos - 4) & RMB));
        const uint32_t r = rec_f(p, a, b, c);
        const uint32_t o = conv_f<KIND>(p, temper_f(p, r, t));
        if (act) {
            sts32(p.rb + ((nb + 4 * S::N) & RMB), r);
            __stcs(p.optr + n, o);
            ck_add<CK>(p, sum, o);
            if (CK) xr ^= o;
        }
    }
}

// One full 256-word step starting at piece word n, ring phase Q = step index mod (R/256).
// RC = (pos - 1 - N) mod 4. The piece's ring phase phi = RA - h puts the aligned x_n group
// at slot 256*Q, so the A groups, and -- except in the last phase(s) of the ring period --
// the C groups and the stores, are addressed as (uniform base) + 16*lane + 512*u without any
// wrap masking; only the uniform E groups and the wrapping phases pay for a mask.
template <uint32_t MEXP, int RC, int KIND, bool CK, int Q>
__device__ __forceinline__ void full_step(const PieceCtx& p, uint32_t n, unsigned long long& sum, uint32_t& xr) {
    using S = Shape<MEXP>;
    constexpr int RA = (int)S::RA;
    constexpr uint32_t RB = S::R * 4;  // ring bytes
    constexpr uint32_t RMB = RB - 1;
    constexpr uint32_t qa = 1024u * Q;                       // A group byte base in this phase
    constexpr uint32_t cS4 = 4u * (S::N + RA);               // store offset from the A base
    constexpr uint32_t cCmax4 = 4u * (S::N - 257u + RA);     // largest C offset (pos <= N - 256)
    constexpr bool wrapC = qa + cCmax4 + 1040u > RB;
    constexpr bool wrapS = qa + cS4 + 1024u > RB;
    const uint32_t l16 = 16 * p.lane;
    const uint32_t cC4 = 4u * (p.pos - 1u + RA - RC);
    const uint32_t aA = p.rb + qa + l16;
    const uint4 GA0 = lds128(aA);
    const uint4 GA1 = lds128(aA + 512);
    const uint4 EA = lds128(p.rb + ((qa + 1024u) & RMB));
    uint4 GC0, GC1;
    if (wrapC) {
        GC0 = lds128(p.rb + ((qa + cC4 + l16) & RMB));
        GC1 = lds128(p.rb + ((qa + cC4 + 512u + l16) & RMB));
    } else {
        const uint32_t aC = p.rb + qa + cC4 + l16;
        GC0 = lds128(aC);
        GC1 = lds128(aC + 512);
    }
    const uint4 EC = lds128(p.rb + ((qa + cC4 + 1024u) & RMB));
    const uint32_t nl = (p.lane + 1) & 31;
    const bool l0 = p.lane == 0;

    uint32_t WA[2][5], WC[2][5];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const uint4 g = u ? GA1 : GA0;
        const uint4 gn = u ? EA : GA1;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int c = RA + j;
            if (c < 4) {
                WA[u][j] = comp(g, c);
            } else {
                const uint32_t send = l0 ? comp(gn, c - 4) : comp(g, c - 4);
                WA[u][j] = __shfl_sync(FULL, send, nl);
            }
        }
        const uint4 h = u ? GC1 : GC0;
        const uint4 hn = u ? EC : GC1;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int c = RC + j;
            if (c < 4) {
                WC[u][j] = comp(h, c);
            } else {
                const uint32_t send = l0 ? comp(hn, c - 4) : comp(h, c - 4);
                WC[u][j] = __shfl_sync(FULL, send, nl);
            }
        }
    }

#pragma unroll
    for (int u = 0; u < 2; ++u) {
        uint32_t r[4], o[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            r[c] = rec_f(p, WA[u][c], WA[u][c + 1], WC[u][c + 1]);
            o[c] = conv_f<KIND>(p, temper_f(p, r[c], WC[u][c]));
            ck_add<CK>(p, sum, o[c]);
        }
        if (CK) xr ^= o[0] ^ o[1] ^ o[2] ^ o[3];
        const uint32_t aS = wrapS ? p.rb + ((qa + cS4 + 512u * u + l16) & RMB) : p.rb + qa + cS4 + 512u * u + l16;
        sts128(aS, r[0], r[1], r[2], r[3]);
        __stcs(reinterpret_cast<uint4*>(p.optr + n + 128 * u) + p.lane, make_uint4(o[0], o[1], o[2], o[3]));
    }
}

// Full steps from piece word n (ring phase 0) while a whole step fits before `end`.
template <uint32_t MEXP, int RC, int KIND, bool CK>
__device__ __forceinline__ void run_steps(const PieceCtx& p, uint32_t n, uint64_t end, unsigned long long& sum,
                                          uint32_t& xr) {
    constexpr int U = (int)(Shape<MEXP>::R / kStepWords);
    static_assert(U == 4 || U == 8, "ring period");
    for (;;) {
#define MTGP_STEP(Qv)                                               \
    if (Qv < U) {                                                   \
        if (n + kStepWords > end) return;                           \
        full_step<MEXP, RC, KIND, CK, (Qv < U ? Qv : 0)>(p, n, sum, xr); \
        __syncwarp();                                               \
        n += kStepWords;                                            \
    }
        MTGP_STEP(0) MTGP_STEP(1) MTGP_STEP(2) MTGP_STEP(3) MTGP_STEP(4) MTGP_STEP(5) MTGP_STEP(6) MTGP_STEP(7)
#undef MTGP_STEP
    }
}

template <uint32_t MEXP, int KIND, bool CK>
__global__ void __launch_bounds__(kWarpsPerCta * 32, MTGP_MIN_CTAS) gen_kernel(GenArgs a) {
    using S = Shape<MEXP>;
    extern __shared__ uint4 smem4[];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t team = blockIdx.x * kWarpsPerCta + warp;
    if (team >= a.n_teams) return;
    PieceCtx p;
    {
        // rings are aligned to their size so that (offset & RMB) | base addresses them
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem4);
        const uint32_t rbytes = S::R * 4;
        p.rb = ((base + rbytes - 1) & ~(rbytes - 1)) + warp * rbytes;
    }
    p.lane = lane;
    const TeamWork tw = a.teams[team];
    for (uint32_t pi = tw.first; pi < tw.first + tw.count; ++pi) {
        const Piece pc = a.pieces[pi];
        const DevParams& prm = a.params[pc.set];
        p.pos = prm.pos;
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
        p.optr = reinterpret_cast<uint32_t*>(a.out) + (size_t)pc.set * a.L + pc.offset;
        const uint64_t len = pc.len;
        // head words so that full steps store 16-byte aligned in global memory
        const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(p.optr) >> 2) & 3u);
        const uint32_t hh = (4u - mis) & 3u;
        const uint32_t h = len < hh ? (uint32_t)len : hh;
        // ring phase: slot(x_h) = RA, so the aligned x_n group of every full step sits at a
        // multiple of 256 slots and STS.128 / STG.128 are both 16-byte aligned
        p.phi = (S::RA - h) & S::RM;
        const uint32_t* w0 = a.piece_win[pi];
        for (uint32_t j = lane; j < S::N; j += 32) sts32(p.rb + (((j + p.phi) & S::RM) << 2), w0[j]);
        __syncwarp();
        unsigned long long sum = 0;
        uint32_t xr = 0;
        scalar_words<MEXP, KIND, CK>(p, 0, h, sum, xr);
        __syncwarp();
        const uint64_t full_end = h + ((len - h) / kStepWords) * kStepWords;
        switch ((prm.pos - 1u - S::N) & 3u) {
            case 0: run_steps<MEXP, 0, KIND, CK>(p, h, full_end, sum, xr); break;
            case 1: run_steps<MEXP, 1, KIND, CK>(p, h, full_end, sum, xr); break;
            case 2: run_steps<MEXP, 2, KIND, CK>(p, h, full_end, sum, xr); break;
            default: run_steps<MEXP, 3, KIND, CK>(p, h, full_end, sum, xr); break;
        }
        scalar_words<MEXP, KIND, CK>(p, (uint32_t)full_end, (uint32_t)(len - full_end), sum, xr);
        __syncwarp();
        if (pc.offset + len == a.L) {
            uint32_t* we = a.win_out + (size_t)pc.set * S::N;
            for (uint32_t j = lane; j < S::N; j += 32)
                we[j] = lds32(p.rb + ((((uint32_t)len + j + p.phi) & S::RM) << 2));
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

// ------------------------------------------------------------------------------------------
// prefix: the raw state-word sequence x_0..x_{len-1} of each listed set from its window.
// One CTA per set (the v1 shape); feeds the jump kernel and the host charpoly analysis.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) prefix_kernel(const DevParams* __restrict__ params,
                                                     const uint32_t* __restrict__ win,
                                                     const uint32_t* __restrict__ sets, uint32_t N,
                                                     uint32_t ring_mask, uint32_t* __restrict__ pre,
                                                     uint32_t len) {
    extern __shared__ uint32_t ring[];
    __shared__ uint32_t s_tbl[16];
    const uint32_t row = blockIdx.x;
    const uint32_t set = sets[row];
    const uint32_t t = threadIdx.x;
    const DevParams& p = params[set];
    const uint32_t pos = p.pos, sh1 = p.sh1, sh2 = p.sh2, mask = p.mask;
    const uint32_t* w = win + (size_t)set * N;
    uint32_t* o = pre + (size_t)row * len;
    for (uint32_t j = t; j < N; j += blockDim.x) {
        ring[j] = w[j];
        o[j] = w[j];
    }
    if (t < 16) s_tbl[t] = p.tbl[t];
    __syncthreads();
    const uint32_t d = min((uint32_t)blockDim.x, N - pos);
    for (uint32_t base = 0; base + N < len; base += d) {
        const uint32_t n = base + t;
        if (t < d && n + N < len) {
            uint32_t x = (ring[n & ring_mask] & mask) ^ ring[(n + 1) & ring_mask];
            x ^= x << sh1;
            const uint32_t y = x ^ (ring[(n + pos) & ring_mask] >> sh2);
            const uint32_t r = y ^ s_tbl[y & 15u];
            ring[(n + N) & ring_mask] = r;
            o[n + N] = r;
        }
        __syncthreads();
    }
}

cudaError_t launch_prefix(const DevParams* params, const uint32_t* win, const uint32_t* sets, uint32_t n_rows,
                          uint32_t N, uint32_t* pre, uint32_t len, cudaStream_t st) {
    if (n_rows == 0) return cudaSuccess;
    const uint32_t R = next_pow2(N + 256);
    const size_t smem = (size_t)R * 4;
    cudaError_t e = cudaFuncSetAttribute(prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    prefix_kernel<<<n_rows, 256, smem, st>>>(params, win, sets, N, R - 1, pre, len);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// jump: y_j = XOR_{i : q_i = 1} x_{i+j}, j in [0, N) -- the window at offset o when
// q = x^o mod P (P annihilates the stream; mtgp_plan.cu). One warp per (job, 32*J-output pass),
// any mix of streams per CTA; the (L2-resident) prefix is read through the read-only L1 path
// (the shared-memory-staged predecessor paid a CTA-wide copy per piece and one CTA per SM slot,
// profiles/r1_launches_flatjump.md). Lane l keeps J consecutive j's in registers and walks q two
// bits at a time.
// ------------------------------------------------------------------------------------------
constexpr int kJumpJ = 12;  // outputs per lane per pass (multiple of 4)
constexpr int kJumpFlatWarps = 4;
template <uint32_t MEXP>
__global__ void __launch_bounds__(kJumpFlatWarps * 32) jump_flat_kernel(JumpArgs a) {
    constexpr uint32_t N = MEXP / 32 + 1;
    constexpr int J = kJumpJ;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // one warp per (job, pass): a pass is 32*J consecutive outputs of the job's window, so a
    // 44497 window (4 passes) runs on 4 warps instead of 4 sequential passes of one warp
    constexpr uint32_t kPasses = (N + 32 * J - 1) / (32 * J);
    const uint32_t unit = blockIdx.x * kJumpFlatWarps + warp;
    const uint32_t job = unit / kPasses;
    if (job >= a.n_jobs) return;
    const JumpJob jb = a.jobs[job];
    const uint4* x4 = reinterpret_cast<const uint4*>(a.pre + (size_t)jb.row * a.pre_stride + a.pre_off);
    const uint32_t* q = a.q + (size_t)jb.q * a.q_words;
    uint32_t* dst = a.piece_win + (size_t)jb.piece * N;
    {
        const uint32_t j0 = (unit % kPasses) * 32 * J;
        const uint32_t jl = j0 + J * lane;  // multiple of 4
        uint32_t acc[J];
#pragma unroll
        for (int k = 0; k < J; ++k) acc[k] = 0;
        for (uint32_t iw0 = 0; iw0 < a.q_words; iw0 += 32) {
            const uint32_t qmine = iw0 + lane < a.q_words ? __ldg(q + iw0 + lane) : 0u;
            const uint32_t nw = min(32u, a.q_words - iw0);
            for (uint32_t k32 = 0; k32 < nw; ++k32) {
                const uint32_t qw = __shfl_sync(FULL, qmine, k32);
                if (qw == 0) continue;
                const uint32_t base4 = ((iw0 + k32) * 32 + jl) >> 2;
                uint32_t w[J + 32];
#pragma unroll
                for (int v = 0; v < (J + 32) / 4; ++v) {
                    const uint4 g = __ldg(x4 + base4 + v);
                    w[4 * v] = g.x;
                    w[4 * v + 1] = g.y;
                    w[4 * v + 2] = g.z;
                    w[4 * v + 3] = g.w;
                }
#pragma unroll
                for (int b = 0; b < 32; b += 2) {
                    const uint32_t pat = (qw >> b) & 3u;
                    if (pat == 1) {
#pragma unroll
                        for (int k = 0; k < J; ++k) acc[k] ^= w[b + k];
                    } else if (pat == 2) {
#pragma unroll
                        for (int k = 0; k < J; ++k) acc[k] ^= w[b + 1 + k];
                    } else if (pat == 3) {
#pragma unroll
                        for (int k = 0; k < J; ++k) acc[k] ^= w[b + k] ^ w[b + 1 + k];
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < J; ++k)
            if (jl + k < N) dst[jl + k] = acc[k];
    }
}

// Same kernel with the window length N a runtime argument (Engine::mt: n per status shape).
__global__ void __launch_bounds__(kJumpFlatWarps * 32) jump_flat_rt_kernel(JumpArgs a, uint32_t N) {
    constexpr int J = kJumpJ;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // one warp per (job, pass): a pass is 32*J consecutive outputs of the job's window, so a
    // 44497 window (4 passes) runs on 4 warps instead of 4 sequential passes of one warp
    const uint32_t kPasses = (N + 32 * J - 1) / (32 * J);
    const uint32_t unit = blockIdx.x * kJumpFlatWarps + warp;
    const uint32_t job = unit / kPasses;
    if (job >= a.n_jobs) return;
    const JumpJob jb = a.jobs[job];
    const uint4* x4 = reinterpret_cast<const uint4*>(a.pre + (size_t)jb.row * a.pre_stride + a.pre_off);
    const uint32_t* q = a.q + (size_t)jb.q * a.q_words;
    uint32_t* dst = a.piece_win + (size_t)jb.piece * N;
    {
        const uint32_t j0 = (unit % kPasses) * 32 * J;
        const uint32_t jl = j0 + J * lane;  // multiple of 4
        uint32_t acc[J];
#pragma unroll
        for (int k = 0; k < J; ++k) acc[k] = 0;
        for (uint32_t iw0 = 0; iw0 < a.q_words; iw0 += 32) {
            const uint32_t qmine = iw0 + lane < a.q_words ? __ldg(q + iw0 + lane) : 0u;
            const uint32_t nw = min(32u, a.q_words - iw0);
            for (uint32_t k32 = 0; k32 < nw; ++k32) {
                const uint32_t qw = __shfl_sync(FULL, qmine, k32);
                if (qw == 0) continue;
                const uint32_t base4 = ((iw0 + k32) * 32 + jl) >> 2;
                uint32_t w[J + 32];
#pragma unroll
                for (int v = 0; v < (J + 32) / 4; ++v) {
                    const uint4 g = __ldg(x4 + base4 + v);
                    w[4 * v] = g.x;
                    w[4 * v + 1] = g.y;
                    w[4 * v + 2] = g.z;
                    w[4 * v + 3] = g.w;
                }
#pragma unroll
                for (int b = 0; b < 32; b += 2) {
                    const uint32_t pat = (qw >> b) & 3u;
                    if (pat == 1) {
#pragma unroll
                        for (int k = 0; k < J; ++k) acc[k] ^= w[b + k];
                    } else if (pat == 2) {
#pragma unroll
                        for (int k = 0; k < J; ++k) acc[k] ^= w[b + 1 + k];
                    } else if (pat == 3) {
#pragma unroll
                        for (int k = 0; k < J; ++k) acc[k] ^= w[b + k] ^ w[b + 1 + k];
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < J; ++k)
            if (jl + k < N) dst[jl + k] = acc[k];
    }
}

template <uint32_t MEXP>
static cudaError_t launch_jump_t(const JumpArgs& a, cudaStream_t st) {
    if (a.n_jobs == 0) return cudaSuccess;
    constexpr uint32_t N = MEXP / 32 + 1, kPasses = (N + 32 * kJumpJ - 1) / (32 * kJumpJ);
    const uint32_t units = a.n_jobs * kPasses;
    jump_flat_kernel<MEXP><<<(units + kJumpFlatWarps - 1) / kJumpFlatWarps, kJumpFlatWarps * 32, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_jump_rt(const JumpArgs& a, uint32_t N, cudaStream_t st) {
    if (a.n_jobs == 0) return cudaSuccess;
    const uint32_t passes = (N + 32 * kJumpJ - 1) / (32 * kJumpJ);
    const uint32_t units = a.n_jobs * passes;
    jump_flat_rt_kernel<<<(units + kJumpFlatWarps - 1) / kJumpFlatWarps, kJumpFlatWarps * 32, 0, st>>>(a, N);
    return cudaGetLastError();
}

cudaError_t launch_jump(uint32_t mexp, const JumpArgs& a, uint32_t n_rows, cudaStream_t st) {
    if (n_rows == 0) return cudaSuccess;
    switch (mexp) {
        case 11213: return launch_jump_t<11213>(a, st);
        case 23209: return launch_jump_t<23209>(a, st);
        case 44497: return launch_jump_t<44497>(a, st);
    }
    return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------------------
template <uint32_t MEXP, int KIND, bool CK>
static cudaError_t launch_gen_t(const GenArgs& a, cudaStream_t st) {
    const size_t smem = (size_t)(kWarpsPerCta + 1) * Shape<MEXP>::R * 4;
    auto k = gen_kernel<MEXP, KIND, CK>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const uint32_t grid = (a.n_teams + kWarpsPerCta - 1) / kWarpsPerCta;
    k<<<grid, kWarpsPerCta * 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <uint32_t MEXP, int KIND, bool CK>
static int occ_t() {
    const size_t smem = (size_t)(kWarpsPerCta + 1) * Shape<MEXP>::R * 4;
    auto k = gen_kernel<MEXP, KIND, CK>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kWarpsPerCta * 32, smem) != cudaSuccess) return 0;
    return n;
}

#define MTGP_DISPATCH(MEXP)                                                             \
    switch (kind * 2 + (cksum ? 1 : 0)) {                                               \
        case 0: return FN<MEXP, MTGP_U32, false> ARGS;                                  \
        case 1: return FN<MEXP, MTGP_U32, true> ARGS;                                   \
        case 2: return FN<MEXP, MTGP_F32_12, false> ARGS;                               \
        case 3: return FN<MEXP, MTGP_F32_12, true> ARGS;                                \
        case 4: return FN<MEXP, MTGP_F32_01OC, false> ARGS;                             \
        case 5: return FN<MEXP, MTGP_F32_01OC, true> ARGS;                              \
    }

cudaError_t launch_gen(uint32_t mexp, int kind, bool cksum, const GenArgs& a, cudaStream_t st) {
    if (a.n_teams == 0) return cudaSuccess;
#define FN launch_gen_t
#define ARGS (a, st)
    switch (mexp) {
        case 11213: MTGP_DISPATCH(11213) break;
        case 23209: MTGP_DISPATCH(23209) break;
        case 44497: MTGP_DISPATCH(44497) break;
    }
#undef FN
#undef ARGS
    return cudaErrorInvalidValue;
}

int gen_ctas_per_sm(uint32_t mexp, int kind, bool cksum) {
#define FN occ_t
#define ARGS ()
    switch (mexp) {
        case 11213: MTGP_DISPATCH(11213) break;
        case 23209: MTGP_DISPATCH(23209) break;
        case 44497: MTGP_DISPATCH(44497) break;
    }
#undef FN
#undef ARGS
    return 0;
}

}  // namespace mtgpb
