// mtgp_plan.cu -- v2 planner: piece decomposition, per-set annihilating polynomials, jump
// polynomials, and the prefix -> jump -> generate launch sequence.
//
// Jump-ahead math. The MTGP32 state is the window (x_i & mask, x_{i+1}, ..., x_{i+N-1}); the
// transition F is GF(2)-linear on an mexp-dimensional space, so every bit-sequence of the
// state words is annihilated by the minimal polynomial P of the stream's state (degree
// <= mexp). If q = x^o mod P then x_{o+j} = XOR_i q_i x_{i+j} (exactly for j >= 1, on the live
// bits for j = 0: the low 32N-mexp bits of the oldest word are dead).
// P comes from Berlekamp-Massey over 2*mexp bits of one bit-plane, LCM'd with further
// functionals until it provably annihilates the whole state (checked on all N window words).
// For the certified cuRAND sets P is the irreducible characteristic polynomial of degree 11213.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>

#include "gf2.h"
#include "mtgp_plan.h"
#include "mtgp_jump.cuh"
#include "mtgp_v2.cuh"
#include "sha1.h"

namespace mtgpb {

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

template <class F>
void parallel_for(size_t n, F&& f) {
    const size_t hw = std::max<size_t>(1, std::thread::hardware_concurrency());
    const size_t nt = std::min(n, hw);
    if (nt <= 1) {
        for (size_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<size_t> next{0};
    std::vector<std::thread> th;
    for (size_t t = 0; t < nt; ++t)
        th.emplace_back([&] {
            for (size_t i; (i = next.fetch_add(1)) < n;) f(i);
        });
    for (auto& x : th) x.join();
}

constexpr uint64_t kMaxPieceWords = 1ull << 30;

// Pieces wanted for W words over T resident teams. An explicit minimum piece length is honoured.
// Auto (min_piece == 0): 2^21-word (8 MB) pieces, but at least three 4-warp CTAs per SM when
// that still leaves pieces of >= 2^19 words -- one CTA per SM left 85% of the warps idle on a
// 128 sets x 2^24 request (902 vs 1038 Gsamples/s; profiles/r1_c5_min_piece.jsonl). Small
// requests that would not fill one CTA per SM (a few streams: a GpuWordSource refill) are split
// into about sqrt(W * jump_k) pieces. That minimises W / (P * r) + P * J / G: one warp generates
// r words/s, the whole GPU G, and one jump costs the GPU as much as J generated words.
// jump_k = G / (r J); ~3.8e-3 at 11213, lower where jumps cost more (PlannerImpl::init_jump).
// Only streams of >= 2^19 words per call are split this way: below that one warp finishes in
// less time than the prefix + jump launches take (~0.1 ms). And only once every stream has
// produced 2^25 words: the first split pays the one-off annihilator analysis and jump
// polynomials (13-45 ms, profiles/r1_first_call.jsonl), which a short-lived source (a sieve cell's
// make_word_source, 10^7 words) would not win back.
constexpr uint64_t kLongLivedWords = 1ull << 25;
uint64_t pieces_wanted(uint64_t W, uint64_t L, uint64_t T, uint64_t quantum, uint64_t min_piece, double jump_k,
                       uint64_t words_done) {
    uint64_t w;
    if (min_piece) {
        w = W / min_piece;
    } else {
        w = W >> 21;
        if ((W >> 19) >= 3 * quantum) w = std::max<uint64_t>(w, 3 * quantum);
        if (w < quantum && jump_k > 0 && L >= (1ull << 19) && words_done >= kLongLivedWords)
            w = std::max<uint64_t>(w, std::min<uint64_t>(quantum, (uint64_t)std::sqrt((double)W * jump_k)));
    }
    return std::min<uint64_t>(T, std::max<uint64_t>(1, w));
}

}  // namespace

struct PlannerImpl {
    std::vector<mtgp_params> sets;
    bool mt = false;  // Engine::mt streams
    int num_sms = 148;
    uint32_t M = 0, N = 0, S = 0;
    bool v2 = false;
    uint32_t mt_min_gap = 0;  // Engine::mt: min over statuses of n - m

    // algebra (per set). Polynomials annihilate the state sequence from the reference point
    // x_{t0} on (t0 = N + 8, rounded to 4): degenerate (uncertified) recursions have a
    // pre-period, so the sequence from x_0 need not be annihilated by the minimal polynomial.
    bool analyzed = false;
    bool jumps_ok = false;             // at least one set can be split
    std::vector<int> set_ok;           // per set: annihilator found
    std::vector<std::unique_ptr<gf2::Modulus>> mods;
    uint32_t t0 = 0;

    // cached plan
    uint64_t plan_L = 0;
    uint32_t plan_T = 0;
    uint64_t plan_want = 0;
    bool plan_valid = false;
    std::vector<Piece> pieces;
    std::vector<TeamWork> teams;
    std::vector<uint32_t> jump_rows;  // set index per prefix row
    std::vector<uint32_t> job_off;
    std::vector<JumpJob> jobs;
    uint32_t n_q = 0;
    uint32_t max_jobs_per_row = 0;
    uint32_t q_words = 0;
    uint32_t pre_len = 0;

    // jump algorithm: the Karatsuba middle product (mtgp_jump.cu) for N > 384 unless forced flat
    int jump_mode = 0;
    bool kara_ok = false;
    KaraPlan kara;

    DevBuf d_pieces, d_teams, d_pwin_ptrs, d_pwin, d_q, d_pre, d_rows, d_joboff, d_jobs, d_win_next, d_all_rows,
        d_zbuf, d_leaf;
    uint64_t plan_id = 0;  // bumped by every plan rebuild

    // Speculative next-call jumps (Planner::run). Call k's prefix x_{t0..} also determines every
    // window of call k + 1 (x^(offset + L - t0) mod P instead of x^(offset - t0)), so while call
    // k generates, a side stream computes call k + 1's piece windows into d_pwin_next. Call k + 1
    // waits for them instead of jumping on the critical path. Worth it when the generator
    // leaves SM slots free (few-piece plans: small shards, single streams).
    DevBuf d_q_next, d_pwin_next;
    uint64_t q_next_plan = ~0ull;  // plan_id the d_q_next polynomials belong to
    cudaStream_t side = nullptr;
    cudaEvent_t ev_pre = nullptr, ev_spec = nullptr;
    bool spec_inflight = false;    // ev_spec not yet waited for on the context stream
    bool spec_ready = false;       // d_pwin_next holds the windows of the call after the last run
    uint64_t spec_epoch = 0, spec_plan = 0;

    // Order the context stream after an in-flight speculative jump: it reads d_pre, d_q_next,
    // the job tables and the Karatsuba scratch, which the context stream's next work may rewrite.
    void join(cudaStream_t st) {
        if (spec_inflight) {
            cudaStreamWaitEvent(st, ev_spec, 0);
            spec_inflight = false;
        }
    }

    ~PlannerImpl() {
        if (side) {
            cudaStreamSynchronize(side);
            cudaStreamDestroy(side);
        }
        if (ev_pre) cudaEventDestroy(ev_pre);
        if (ev_spec) cudaEventDestroy(ev_spec);
        for (DevBuf* b : {&d_pieces, &d_teams, &d_pwin_ptrs, &d_pwin, &d_q, &d_pre, &d_rows, &d_joboff, &d_jobs,
                          &d_win_next, &d_all_rows, &d_zbuf, &d_leaf, &d_q_next, &d_pwin_next})
            b->release();
    }
    cudaError_t build_next_q(uint64_t L, cudaStream_t st);
    // d = 0 (N <= 384, i.e. 11213) keeps the flat jump when the jumps fill the GPU: the grouped
    // d = 0 leaf path measured 0.66 vs 0.51 ms per C2 call (profiles/r1_jump_sweep.jsonl)
    double jump_k = 0;  // pieces_wanted's G / (r J) for this shape
    void init_jump() {
        kara_ok = kara_plan(N, (M + 31) / 32, -1, kara);
        // calibrated at 11213 (N M = 3.9e6, direct jump): r ~ 2.4e9 words/s per warp
        // (profiles/r1_single_stream.jsonl), G ~ 1.15e12, J ~ 1.25e5 words
        const double f = !kara_ok || kara.depth == 0 ? 1.0 : kara.depth == 1 ? 0.75 : 0.5625;
        jump_k = 3.8e-3 * (351.0 * 11213.0) / ((double)N * (double)M * f);
    }
    bool use_kara() const { return kara_ok && ((jump_mode == 0 && kara.depth > 0) || jump_mode == 2); }
    uint32_t last_jump_launches = 1;  // kernels the last jump() call launched

    // words the jump kernels read per row (from x_{t0})
    uint32_t prefix_len() const {
        const uint32_t qw = (M + 31) / 32;
        const uint32_t jblk = 32 * 12;
        uint32_t need = 32 * qw + jblk * ((N + jblk - 1) / jblk) + 36;
        if (kara_ok) need = std::max(need, kara_prefix_words(kara) + 36);
        return (need + 31) & ~31u;
    }
    // words the prefix kernel generates per row (x_0 .. ), rows 128-byte aligned
    uint32_t prefix_stride() const { return (t0 + prefix_len() + 31) & ~31u; }

    cudaError_t analyze(const void* params, const uint32_t* win, cudaStream_t st, std::string& err);

    // engine-specific launches: the state-word prefix of rows, and the jump itself
    cudaError_t prefix(const void* params, const uint32_t* win, const uint32_t* rows, uint32_t n_rows, uint32_t* pre,
                       uint32_t len, cudaStream_t st) const {
        return mt ? launch_mt_prefix(static_cast<const DevMtParams*>(params), win, rows, n_rows, N, pre, len, st)
                  : launch_prefix(static_cast<const DevParams*>(params), win, rows, n_rows, N, pre, len, st);
    }
    cudaError_t jump(const JumpArgs& a, uint32_t n_rows, cudaStream_t st) {
        // d = 0 (11213): the flat kernel runs one warp per jump, which is slow in latency when there
        // are few jumps (a single stream: ~0.3 ms for 351 q words). Split the q blocks over >= 3
        // warps per jump then (profiles/r1_single_stream.jsonl); keep the flat kernel when the
        // jumps already fill the GPU (C2: 0.51 vs 0.66 ms, profiles/r1_jump_sweep.jsonl).
        const bool split0 = jump_mode == 0 && kara_ok && kara.depth == 0 && kara_groups(kara, a.n_jobs, num_sms) >= 3;
        // kernels this jump launches: ztrans (d >= 1), qleaf, leaf, combine; or the one flat kernel
        last_jump_launches = (use_kara() || split0) ? (kara.depth > 0 ? 4u : 3u) : 1u;
        if (use_kara() || split0) {
            KaraPlan k = kara;
            k.groups = kara_groups(k, a.n_jobs, num_sms);
            cudaError_t e;
            if (k.depth > 0 && (e = d_zbuf.ensure(4 * kara_zbuf_words(k, n_rows))) != cudaSuccess) return e;
            if ((e = d_leaf.ensure(4 * kara_leaf_words(k, a.n_jobs))) != cudaSuccess) return e;
            return launch_jump_kara(a, k, N, n_rows, d_zbuf.as<uint32_t>(), d_leaf.as<uint32_t>(), st);
        }
        return mt ? launch_jump_rt(a, N, st) : launch_jump(M, a, n_rows, st);
    }
    cudaError_t build_plan(uint64_t L, uint32_t T, uint64_t min_piece, uint64_t words_done, cudaStream_t st,
                           std::string& err);
};

Planner::Planner(const std::vector<mtgp_params>& sets, int num_sms) : impl_(new PlannerImpl) {
    impl_->sets = sets;
    impl_->num_sms = num_sms;
    impl_->S = (uint32_t)sets.size();
    impl_->M = sets[0].mexp;
    impl_->N = state_words(impl_->M);
    impl_->t0 = (impl_->N + 8 + 3) & ~3u;
    impl_->v2 = v2_supports(impl_->M);
    for (const auto& p : sets)
        if (p.pos + kStepWords > impl_->N) impl_->v2 = false;  // needs N - pos >= 256
    impl_->init_jump();
}
Planner::Planner(const std::vector<mtgp_mt_params>& sets, int num_sms) : impl_(new PlannerImpl) {
    impl_->mt = true;
    impl_->num_sms = num_sms;
    impl_->S = (uint32_t)sets.size();
    impl_->M = sets[0].mexp;
    impl_->N = sets[0].n;
    impl_->t0 = (impl_->N + 8 + 3) & ~3u;
    impl_->v2 = true;
    impl_->mt_min_gap = impl_->N;
    for (const auto& p : sets) {
        if (p.mexp != impl_->M || p.n != impl_->N || p.n - p.m < 32) impl_->v2 = false;
        impl_->mt_min_gap = std::min(impl_->mt_min_gap, p.n - p.m);
    }
    impl_->init_jump();
}
void Planner::set_jump_mode(int mode) { impl_->jump_mode = mode; }
Planner::~Planner() = default;

bool Planner::v2_supported() const { return impl_->v2; }
bool Planner::mt3_supported(int kind, uint64_t L, const void* out) const {
    return impl_->mt && impl_->v2 && mt_gen3_supports(impl_->N, impl_->mt_min_gap, kind) && L % 4 == 0 &&
           (reinterpret_cast<uintptr_t>(out) & 15) == 0;
}
void Planner::invalidate() {
    impl_->analyzed = false;
    impl_->jumps_ok = false;
    impl_->plan_valid = false;
    impl_->spec_ready = false;
}

cudaError_t Planner::analyze_now(const void* params, const uint32_t* win, cudaStream_t st, std::string& err) {
    if (!impl_->v2) return cudaSuccess;
    impl_->join(st);
    return impl_->analyze(params, win, st, err);
}

cudaError_t PlannerImpl::analyze(const void* params, const uint32_t* win, cudaStream_t st, std::string& err) {
    if (analyzed) return cudaSuccess;
    const uint32_t len = ((t0 + 2 * M + N + 64) + 31) & ~31u;
    std::vector<uint32_t> rows(S);
    for (uint32_t s = 0; s < S; ++s) rows[s] = s;
    cudaError_t e;
    if ((e = d_all_rows.ensure(S * 4)) != cudaSuccess) return e;
    DevBuf seq;
    if ((e = seq.ensure((size_t)S * len * 4)) != cudaSuccess) return e;
    cudaMemcpyAsync(d_all_rows.p, rows.data(), S * 4, cudaMemcpyHostToDevice, st);
    if ((e = prefix(params, win, d_all_rows.as<uint32_t>(), S, seq.as<uint32_t>(), len, st)) != cudaSuccess) {
        seq.release();
        return e;
    }
    std::vector<uint32_t> h((size_t)S * len);
    e = cudaMemcpyAsync(h.data(), seq.p, h.size() * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    seq.release();
    if (e != cudaSuccess) return e;

    mods.clear();
    mods.resize(S);
    std::vector<int> ok(S, 0);
    parallel_for(S, [&](size_t s) {
        const uint32_t* x = h.data() + s * len + t0;  // reference point x_{t0}
        // Functionals: parities of dense pseudo-random word masks (the LCM over all single-word
        // functionals is the state's annihilator; degenerate uncertified recursions can hide whole
        // components from single bits, e.g. a constant bit 0). Certified sets finish after one.
        uint32_t fmask[24];
        uint64_t sm = 0x4D54475041ull;
        for (auto& m : fmask) {
            sm += 0x9E3779B97F4A7C15ull;
            uint64_t z = (sm ^ (sm >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            m = static_cast<uint32_t>(z ^ (z >> 31)) | 0x80000001u;
        }
        gf2::Poly P;
        bool good = false;
        for (uint32_t fi = 0; fi < sizeof(fmask) / sizeof(fmask[0]) && !good; ++fi) {
            std::vector<uint64_t> bits((2 * (size_t)M + 63) / 64 + 1, 0);
            for (size_t k = 0; k < 2 * (size_t)M; ++k)
                if (__builtin_parity(x[k] & fmask[fi])) bits[k >> 6] |= 1ull << (k & 63);
            gf2::Poly Q = gf2::berlekamp_massey(bits, 2 * (size_t)M);
            if (fi == 0) {
                P = Q;
            } else {
                // P = lcm(P, Q)
                gf2::Poly g = gf2::gcd(P, Q);
                gf2::Poly qq;
                gf2::divmod(Q, g, &qq, nullptr);
                P = gf2::mul(P, qq);
            }
            if (P.degree() > (int)M) break;
            // P annihilates every bit of the whole window at the reference point, hence (by
            // linearity of the transition) every later window
            std::vector<int> idx;
            for (int i = 0; i <= P.degree(); ++i)
                if (P.coeff(i)) idx.push_back(i);
            bool ann = true;
            for (uint32_t j = 0; j < N && ann; ++j) {
                uint32_t acc = 0;
                for (int i : idx) acc ^= x[i + j];
                ann = acc == 0;
            }
            good = ann;
        }
        if (good) {
            mods[s] = std::make_unique<gf2::Modulus>(P);
            ok[s] = 1;
        }
    });
    set_ok = ok;
    jumps_ok = false;
    for (uint32_t s = 0; s < S; ++s)
        if (ok[s]) jumps_ok = true;
    analyzed = true;
    err.clear();  // a set without an annihilator is simply never split (one piece per call)
    return cudaSuccess;
}

cudaError_t PlannerImpl::build_plan(uint64_t L, uint32_t T, uint64_t min_piece, uint64_t words_done,
                                    cudaStream_t st, std::string& err) {
    const uint64_t W = (uint64_t)S * L;
    // Equal work per SM: team counts are whole multiples of (SMs x warps per CTA), so every SM
    // holds the same number of CTAs (a 5-vs-6 CTA split costs ~10% of the makespan).
    const uint64_t quantum = (uint64_t)num_sms * kWarpsPerCta;
    uint64_t want = pieces_wanted(W, L, T, quantum, min_piece, jump_k, words_done);
    if (want >= quantum) want -= want % quantum;
    want = std::max<uint64_t>(want, (W + kMaxPieceWords - 1) / kMaxPieceWords);
    // the plan is a function of (L, T, want) only: min_piece and words_done enter through want
    if (plan_valid && plan_L == L && plan_T == T && plan_want == want) return cudaSuccess;
    plan_valid = false;
    pieces.clear();
    teams.clear();
    if (L > kMaxPieceWords)
        for (uint32_t s = 0; s < S; ++s)
            if (!set_ok[s]) {
                err = "request needs jump-ahead pieces but stream " + std::to_string(s) +
                      " has no annihilating polynomial";
                return cudaSuccess;
            }
    if (want <= S || !jumps_ok || L < 2ull * t0) {
        for (uint32_t s = 0; s < S; ++s) {
            pieces.push_back(Piece{s, -1, 0, L});
            teams.push_back(TeamWork{s, 1});
        }
    } else {
        // Split the concatenation of all streams into `want` equal ranges cut at stream
        // boundaries; cuts are multiples of 8 words (32-byte aligned pieces), never inside a
        // stream that cannot be jumped, and never in (0, t0) of a stream (jumps start at x_{t0}).
        std::vector<uint64_t> cut(want + 1);
        cut[0] = 0;
        cut[want] = W;
        for (uint64_t g = 1; g < want; ++g) {
            uint64_t c = (W * g / want) & ~7ull;
            const uint64_t s = c / L, off = c % L;
            if (off && !set_ok[s]) c = (off < L / 2) ? s * L : (s + 1) * L;
            else if (off && off < t0) c = s * L + t0;
            cut[g] = std::min<uint64_t>(std::max<uint64_t>(c, cut[g - 1]), W);
        }
        for (uint64_t g = 0; g < want; ++g) {
            uint64_t a = cut[g], b = cut[g + 1];
            if (b <= a) continue;
            TeamWork tw{(uint32_t)pieces.size(), 0};
            while (a < b) {
                const uint32_t s = (uint32_t)(a / L);
                const uint64_t off = a % L;
                const uint64_t end = std::min<uint64_t>(b, (uint64_t)(s + 1) * L);
                pieces.push_back(Piece{s, -1, off, end - a});
                tw.count++;
                a = end;
            }
            teams.push_back(tw);
        }
    }
    // jump jobs, grouped by set
    std::map<uint32_t, std::vector<uint32_t>> by_set;
    for (uint32_t i = 0; i < pieces.size(); ++i)
        if (pieces[i].offset) by_set[pieces[i].set].push_back(i);
    jump_rows.clear();
    max_jobs_per_row = 0;
    job_off.assign(1, 0);
    jobs.clear();
    q_words = (M + 31) / 32;
    std::vector<std::pair<uint32_t, uint32_t>> qlist;  // (piece, set)
    for (auto& kv : by_set) {
        jump_rows.push_back(kv.first);
        for (uint32_t pi : kv.second) {
            pieces[pi].jump_idx = (int32_t)qlist.size();
            jobs.push_back(JumpJob{pi, (uint32_t)qlist.size(), (uint32_t)jump_rows.size() - 1});
            qlist.push_back({pi, kv.first});
        }
        job_off.push_back((uint32_t)jobs.size());
        max_jobs_per_row = std::max<uint32_t>(max_jobs_per_row, (uint32_t)kv.second.size());
    }
    n_q = (uint32_t)qlist.size();
    // jump polynomials x^(offset - t0) mod P (relative to the reference point), chained per set
    std::vector<uint32_t> hq((size_t)n_q * q_words, 0);
    std::vector<uint32_t> rows_list(jump_rows);
    parallel_for(rows_list.size(), [&](size_t r) {
        const uint32_t s = rows_list[r];
        const gf2::Modulus& md = *mods[s];
        std::map<uint64_t, gf2::Poly> step_cache;
        gf2::Poly cur;
        uint64_t cur_off = 0;
        bool have = false;
        for (uint32_t jj = job_off[r]; jj < job_off[r + 1]; ++jj) {
            const uint32_t pi = jobs[jj].piece;
            const uint64_t off = pieces[pi].offset - t0;
            if (!have) {
                cur = md.x_pow(off);
                have = true;
            } else {
                const uint64_t d = off - cur_off;
                auto it = step_cache.find(d);
                if (it == step_cache.end()) it = step_cache.emplace(d, md.x_pow(d)).first;
                cur = md.mulmod(cur, it->second);
            }
            cur_off = off;
            uint32_t* dst = hq.data() + (size_t)jobs[jj].q * q_words;
            for (int i = 0; i <= cur.degree(); ++i)
                if (cur.coeff(i)) dst[i >> 5] |= 1u << (i & 31);
        }
    });
    // device copies
    cudaError_t e;
    pre_len = prefix_len();
    if ((e = d_pieces.ensure(sizeof(Piece) * pieces.size())) != cudaSuccess) return e;
    if ((e = d_teams.ensure(sizeof(TeamWork) * teams.size())) != cudaSuccess) return e;
    if ((e = d_pwin_ptrs.ensure(sizeof(uint32_t*) * pieces.size())) != cudaSuccess) return e;
    if ((e = d_pwin.ensure(sizeof(uint32_t) * N * std::max<size_t>(1, pieces.size()))) != cudaSuccess) return e;
    if ((e = d_q.ensure(sizeof(uint32_t) * std::max<size_t>(1, hq.size()))) != cudaSuccess) return e;
    if ((e = d_pre.ensure(sizeof(uint32_t) * (size_t)prefix_stride() * std::max<size_t>(1, jump_rows.size()))) != cudaSuccess) return e;
    if ((e = d_rows.ensure(sizeof(uint32_t) * std::max<size_t>(1, jump_rows.size()))) != cudaSuccess) return e;
    if ((e = d_joboff.ensure(sizeof(uint32_t) * job_off.size())) != cudaSuccess) return e;
    if ((e = d_jobs.ensure(sizeof(JumpJob) * std::max<size_t>(1, jobs.size()))) != cudaSuccess) return e;
    if ((e = d_win_next.ensure(sizeof(uint32_t) * N * S)) != cudaSuccess) return e;
    // Upload on the context stream: a previous call's kernels may still be reading the plan
    // arrays (the context stream is non-blocking, so a legacy-stream cudaMemcpy would not wait
    // for them). From pageable memory the copies are staged before returning, so the host
    // vectors may change afterwards.
    auto up = [&](void* dst, const void* src, size_t bytes) {
        return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st) : cudaSuccess;
    };
    if ((e = up(d_pieces.p, pieces.data(), sizeof(Piece) * pieces.size())) != cudaSuccess ||
        (e = up(d_teams.p, teams.data(), sizeof(TeamWork) * teams.size())) != cudaSuccess ||
        (e = up(d_q.p, hq.data(), sizeof(uint32_t) * hq.size())) != cudaSuccess ||
        (e = up(d_rows.p, jump_rows.data(), sizeof(uint32_t) * jump_rows.size())) != cudaSuccess ||
        (e = up(d_joboff.p, job_off.data(), sizeof(uint32_t) * job_off.size())) != cudaSuccess ||
        (e = up(d_jobs.p, jobs.data(), sizeof(JumpJob) * jobs.size())) != cudaSuccess)
        return e;
    plan_L = L;
    plan_T = T;
    plan_want = want;
    plan_valid = true;
    ++plan_id;
    return cudaGetLastError();
}

// The current plan's jump polynomials for the NEXT call: x^(offset + L - t0) mod P per job
// (the same pieces, one call later), uploaded to d_q_next.
cudaError_t PlannerImpl::build_next_q(uint64_t L, cudaStream_t st) {
    if (q_next_plan == plan_id) return cudaSuccess;
    std::vector<uint32_t> hq((size_t)n_q * q_words, 0);
    std::vector<uint32_t> rows_list(jump_rows);
    parallel_for(rows_list.size(), [&](size_t r) {
        const gf2::Modulus& md = *mods[rows_list[r]];
        gf2::Poly cur;
        uint64_t cur_off = 0;
        bool have = false;
        std::map<uint64_t, gf2::Poly> step_cache;
        for (uint32_t jj = job_off[r]; jj < job_off[r + 1]; ++jj) {
            const uint64_t off = pieces[jobs[jj].piece].offset + L - t0;
            if (!have) {
                cur = md.x_pow(off);
                have = true;
            } else {
                const uint64_t d = off - cur_off;
                auto it = step_cache.find(d);
                if (it == step_cache.end()) it = step_cache.emplace(d, md.x_pow(d)).first;
                cur = md.mulmod(cur, it->second);
            }
            cur_off = off;
            uint32_t* dst = hq.data() + (size_t)jobs[jj].q * q_words;
            for (int i = 0; i <= cur.degree(); ++i)
                if (cur.coeff(i)) dst[i >> 5] |= 1u << (i & 31);
        }
    });
    cudaError_t e;
    if ((e = d_q_next.ensure(sizeof(uint32_t) * std::max<size_t>(1, hq.size()))) != cudaSuccess) return e;
    if (!hq.empty() &&
        (e = cudaMemcpyAsync(d_q_next.p, hq.data(), sizeof(uint32_t) * hq.size(), cudaMemcpyHostToDevice, st)) !=
            cudaSuccess)
        return e;
    q_next_plan = plan_id;
    return cudaSuccess;
}

cudaError_t Planner::run(PlanRun& r, std::string& err) {
    PlannerImpl& I = *impl_;
    if (!I.v2) {
        err = "v2 kernel does not support this parameter shape";
        return cudaSuccess;
    }
    I.join(r.stream);
    // v3 (register-resident ring) serves MTGP32-11213 when every piece starts 16-byte aligned:
    // 16-byte aligned output, L % 4 == 0 (piece offsets are multiples of 4 by construction)
    const bool reg_ok = !I.mt && r.L % 4 == 0 && (reinterpret_cast<uintptr_t>(r.out) & 15) == 0;
    const bool v3_ok = I.M == 11213 && reg_ok;
    const bool bitmap = r.kind >= kKindBitmapBit0;
    const bool v4_ok = v4_supports(I.M, r.kind) && reg_ok;
    // Engine::mt: mt_gen3 (register-resident, version 6) when the shape allows, else mt_gen2
    const bool mt3_ok = mt3_supported(r.kind, r.L, r.out);
    if (I.mt && r.kind == MTGP_F64_01 && !mt3_ok) {
        err = "Engine::mt f64 output on the warp teams needs kernel 6's shape";
        return cudaSuccess;
    }
    if (!I.mt && (r.want_kernel == 5 || r.want_kernel == 6)) {
        err = "kernels 5 and 6 are Engine::mt kernels";
        return cudaSuccess;
    }
    if (r.want_kernel == 6 && !mt3_ok) {
        err = "kernel 6 needs n = 624, n - m >= 129 for every status, u32 output, words_per_stream % 4 == 0 "
              "and 16-byte aligned output";
        return cudaSuccess;
    }
    const bool use_mt3 = mt3_ok && r.want_kernel != 5;
    if (bitmap && (I.mt ? !use_mt3 : (!v3_ok || (r.want_kernel != 0 && r.want_kernel != 3)))) {
        err = "bitmap output needs kernel v3 (mexp 11213) or Engine::mt kernel 6, words_per_stream % 4 == 0";
        return cudaSuccess;
    }
    if (r.want_kernel == 3 && !v3_ok) {
        err = "kernel v3 needs mexp 11213, words_per_stream % 4 == 0 and 16-byte aligned output";
        return cudaSuccess;
    }
    if (r.want_kernel == 4 && !v4_ok) {
        err = "kernel v4 needs mexp 11213/23209/44497, u32 output, words_per_stream % 4 == 0 and 16-byte aligned output";
        return cudaSuccess;
    }
    // auto: v3 for 11213; v4 (the same register-resident design, templated on N) for 23209 and
    // 44497, where it beats the shared-memory ring by 18% / 27% (profiles/r1_v4_sweep.jsonl);
    // v2 for request shapes the register kernels do not take (float kinds, L % 4 != 0, ...)
    const bool use_v3 = v3_ok && (r.want_kernel == 3 || (r.want_kernel == 0 && I.M == 11213));
    const bool use_v4 = !use_v3 && v4_ok && (r.want_kernel == 4 || (r.want_kernel == 0 && I.M != 11213));
    const int ck_mode = r.cksum ? (r.ck32 ? 2 : 1) : 0;
    const int cps = use_mt3  ? mt_gen3_ctas_per_sm(I.N, r.kind, ck_mode)
                    : I.mt   ? mt_gen2_ctas_per_sm(I.N, r.kind, r.cksum)
                    : use_v3 ? gen3_ctas_per_sm(r.kind, ck_mode)
                    : use_v4 ? gen4_ctas_per_sm(I.M, r.kind, ck_mode)
                             : gen_ctas_per_sm(I.M, r.kind, r.cksum);
    if (cps <= 0) {
        err = "generation kernel cannot be resident";
        return cudaSuccess;
    }
    uint32_t T = (uint32_t)(cps * kWarpsPerCta * I.num_sms);
    if (r.max_pieces) T = std::min(T, r.max_pieces);
    const uint64_t W = (uint64_t)I.S * r.L;
    const bool need_jumps =
        pieces_wanted(W, r.L, T, (uint64_t)I.num_sms * kWarpsPerCta, r.min_piece_words, I.jump_k, r.words_done) > I.S ||
                            r.L > kMaxPieceWords;
    cudaError_t e;
    if (need_jumps && !I.analyzed) {
        if ((e = I.analyze(r.params, r.win, r.stream, err)) != cudaSuccess) return e;
        if (!err.empty()) return cudaSuccess;
    }
    if ((e = I.build_plan(r.L, need_jumps ? T : I.S, r.min_piece_words, r.words_done, r.stream, err)) != cudaSuccess)
        return e;
    if (!err.empty()) return cudaSuccess;

    // Speculative jumps: use the windows the previous call computed for this one when nothing
    // touched the state in between (epoch) and the plan is the same; speculate for the next call
    // when the plan has jumps and its teams fill at most a quarter of the generator's warp slots
    // (auto), or always (MTGP_OPT_PREJUMP 2). Measured (profiles/r2/): one long-lived stream in
    // 2^20-word calls 5.3 -> 8.0 G words/s (the jump leaves the critical path and runs on idle
    // SMs); full-occupancy plans (C2-C5, MT19937) within +-1% (the side-stream jump only fills
    // the generator's tail, and slows the generator by what it saves); half-occupancy plans
    // (C5 shards at 4-8 GPUs, 3 of 6 CTAs per SM) 12-20% slower (it competes with the generator).
    const bool has_jumps = !I.jump_rows.empty();
    const bool use_spec = has_jumps && I.spec_ready && r.epoch == I.spec_epoch && I.spec_plan == I.plan_id;
    I.spec_ready = false;
    const bool spec_next = has_jumps && r.prejump != 1 && (r.prejump == 2 || 4 * I.teams.size() <= (size_t)T);
    if (use_spec) std::swap(I.d_pwin, I.d_pwin_next);  // d_pwin_next's windows are complete (join)
    r.prejumped = use_spec;

    // per-piece start-window pointers: jumped pieces -> d_pwin rows; offset-0 pieces -> current window
    std::vector<const uint32_t*> ptrs(I.pieces.size());
    for (size_t i = 0; i < I.pieces.size(); ++i)
        ptrs[i] = I.pieces[i].offset ? I.d_pwin.as<uint32_t>() + (size_t)i * I.N
                                     : r.win + (size_t)I.pieces[i].set * I.N;
    if ((e = cudaMemcpyAsync(I.d_pwin_ptrs.p, ptrs.data(), sizeof(uint32_t*) * ptrs.size(), cudaMemcpyHostToDevice,
                             r.stream)) != cudaSuccess)
        return e;

    size_t j0 = 0, j1 = 0, g0 = 0, g1 = 0;
    JumpArgs ja;
    ja.pre = I.d_pre.as<uint32_t>();
    ja.pre_len = I.pre_len;
    ja.pre_stride = I.prefix_stride();
    ja.pre_off = I.t0;
    ja.set_of = I.d_rows.as<uint32_t>();
    ja.job_off = I.d_joboff.as<uint32_t>();
    ja.jobs = I.d_jobs.as<JumpJob>();
    ja.q = I.d_q.as<uint32_t>();
    ja.q_words = I.q_words;
    ja.piece_win = I.d_pwin.as<uint32_t>();
    ja.max_jobs_per_row = I.max_jobs_per_row;
    ja.n_jobs = (uint32_t)I.jobs.size();
    if (has_jumps && (!use_spec || spec_next)) {
        // this call's prefix x_0.. (needed by this call's jumps, or by the next call's speculation)
        if (r.timing && !use_spec) r.timing->record(r.stream, &j0);
        if ((e = I.prefix(r.params, r.win, I.d_rows.as<uint32_t>(), (uint32_t)I.jump_rows.size(),
                          I.d_pre.as<uint32_t>(), I.prefix_stride(), r.stream)) != cudaSuccess)
            return e;
        r.launches += 1;
    }
    if (has_jumps && !use_spec) {
        if ((e = I.jump(ja, (uint32_t)I.jump_rows.size(), r.stream)) != cudaSuccess) return e;
        if (r.timing) {
            r.timing->record(r.stream, &j1);
            r.timing->jump.push_back({j0, j1});
        }
        r.launches += I.last_jump_launches;
    }
    if (spec_next) {
        // the next call's windows from this call's prefix, on the side stream, overlapping this
        // call's generation (after this call's own jump: they share the Karatsuba scratch)
        if ((e = I.build_next_q(r.L, r.stream)) != cudaSuccess) return e;
        if ((e = I.d_pwin_next.ensure(sizeof(uint32_t) * I.N * std::max<size_t>(1, I.pieces.size()))) != cudaSuccess)
            return e;
        if (!I.side) {
            if ((e = cudaStreamCreateWithFlags(&I.side, cudaStreamNonBlocking)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&I.ev_pre, cudaEventDisableTiming)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&I.ev_spec, cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        if ((e = cudaEventRecord(I.ev_pre, r.stream)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(I.side, I.ev_pre, 0)) != cudaSuccess) return e;
        JumpArgs jn = ja;
        jn.q = I.d_q_next.as<uint32_t>();
        jn.piece_win = I.d_pwin_next.as<uint32_t>();
        if ((e = I.jump(jn, (uint32_t)I.jump_rows.size(), I.side)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(I.ev_spec, I.side)) != cudaSuccess) return e;
        I.spec_inflight = true;
        I.spec_ready = true;
        I.spec_epoch = r.epoch + 1;
        I.spec_plan = I.plan_id;
        r.launches += I.last_jump_launches;
    }
    if (I.mt) {
        MtGenArgs ma;
        ma.params = static_cast<const DevMtParams*>(r.params);
        ma.pieces = I.d_pieces.as<Piece>();
        ma.teams = I.d_teams.as<TeamWork>();
        ma.n_teams = (uint32_t)I.teams.size();
        ma.piece_win = I.d_pwin_ptrs.as<const uint32_t*>();
        ma.win_out = I.d_win_next.as<uint32_t>();
        ma.out = r.out;
        ma.L = r.L;
        ma.ck = r.ck;
        ma.n = I.N;
        ma.pairs = r.L % 2 == 0 && (reinterpret_cast<uintptr_t>(r.out) & 7) == 0;
        ma.pred = r.pred;
        if (r.timing) r.timing->record(r.stream, &g0);
        e = use_mt3 ? launch_mt_gen3(I.N, r.kind, ck_mode, ma, r.stream)
                    : launch_mt_gen2(r.kind, r.cksum, ma, r.stream);
        if (e != cudaSuccess) return e;
        r.version = use_mt3 ? 6 : 5;
    } else {
        GenArgs ga;
        ga.params = static_cast<const DevParams*>(r.params);
        ga.pieces = I.d_pieces.as<Piece>();
        ga.teams = I.d_teams.as<TeamWork>();
        ga.n_teams = (uint32_t)I.teams.size();
        ga.piece_win = I.d_pwin_ptrs.as<const uint32_t*>();
        ga.win_out = I.d_win_next.as<uint32_t>();
        ga.out = r.out;
        ga.L = r.L;
        ga.ck = r.ck;
        ga.pred = r.pred;
        if (r.timing) r.timing->record(r.stream, &g0);
        e = use_v3   ? launch_gen3(r.kind, ck_mode, ga, r.stream)
            : use_v4 ? launch_gen4(I.M, r.kind, ck_mode, ga, r.stream)
                     : launch_gen(I.M, r.kind, r.cksum, ga, r.stream);
        if (e != cudaSuccess) return e;
        r.version = use_v3 ? 3 : use_v4 ? 4 : 2;
    }
    if (r.timing) {
        r.timing->record(r.stream, &g1);
        r.timing->gen.push_back({g0, g1});
    }
    if ((e = cudaMemcpyAsync(r.win, I.d_win_next.p, sizeof(uint32_t) * I.N * I.S, cudaMemcpyDeviceToDevice,
                             r.stream)) != cudaSuccess)
        return e;
    r.launches += 1;
    r.pieces = (uint32_t)I.pieces.size();
    r.warps_per_piece = 1;
    return cudaGetLastError();
}

cudaError_t Planner::charpoly_sha1(const void* params, uint32_t* win, cudaStream_t st,
                                   std::vector<std::string>& out, std::string& err) {
    PlannerImpl& I = *impl_;
    I.join(st);
    cudaError_t e;
    if (!I.analyzed && (e = I.analyze(params, win, st, err)) != cudaSuccess) return e;
    out.assign(I.S, std::string());
    parallel_for(I.S, [&](size_t s) {
        if (!I.set_ok[s]) return;
        const gf2::Poly& P = I.mods[s]->p;
        std::string c(P.degree() + 1, '0');
        for (int i = 0; i <= P.degree(); ++i)
            if (P.coeff(i)) c[i] = '1';
        out[s] = sha1_hex(c);
    });
    return cudaSuccess;
}

cudaError_t Planner::certify(const void* params, uint32_t* win, cudaStream_t st, std::vector<int>& out,
                             std::string& err) {
    PlannerImpl& I = *impl_;
    I.join(st);
    cudaError_t e;
    if (!I.analyzed && (e = I.analyze(params, win, st, err)) != cudaSuccess) return e;
    out.assign(I.S, 0);
    parallel_for(I.S, [&](size_t s) {
        if (!I.set_ok[s]) return;
        const gf2::Poly& P = I.mods[s]->p;
        out[s] = P.degree() == (int)I.M && gf2::is_irreducible(P) ? 1 : 0;
    });
    return cudaSuccess;
}

cudaError_t Planner::skip(const void* params, uint32_t* win, uint64_t words, cudaStream_t st, std::string& err) {
    PlannerImpl& I = *impl_;
    if (I.mt ? !I.v2 : !v2_supports(I.M)) {
        err = "skip (jump-ahead) is implemented for mexp 11213, 23209 and 44497 and uniform Engine::mt shapes";
        return cudaSuccess;
    }
    I.join(st);  // the skip's jump uses the Karatsuba scratch
    I.spec_ready = false;
    cudaError_t e;
    if (!I.analyzed && (e = I.analyze(params, win, st, err)) != cudaSuccess) return e;
    for (uint32_t s = 0; s < I.S; ++s)
        if (!I.set_ok[s]) {
            err = "no annihilating polynomial found for stream " + std::to_string(s);
            return cudaSuccess;
        }
    if (words < I.t0) {
        err = "skip distance below the jump reference offset";
        return cudaSuccess;
    }
    const uint32_t qw = (I.M + 31) / 32;
    std::vector<uint32_t> hq((size_t)I.S * qw, 0);
    parallel_for(I.S, [&](size_t s) {
        gf2::Poly q = I.mods[s]->x_pow(words - I.t0);
        for (int i = 0; i <= q.degree(); ++i)
            if (q.coeff(i)) hq[s * qw + (i >> 5)] |= 1u << (i & 31);
    });
    const uint32_t pre_len = I.prefix_len();
    const uint32_t pre_stride = I.prefix_stride();
    DevBuf pre, q, rows, joff, jobs, out;
    std::vector<uint32_t> hrows(I.S), hoff(I.S + 1);
    std::vector<JumpJob> hjobs(I.S);
    for (uint32_t s = 0; s < I.S; ++s) {
        hrows[s] = s;
        hoff[s] = s;
        hjobs[s] = JumpJob{s, s, s};
    }
    hoff[I.S] = I.S;
    auto cleanup = [&] {
        for (DevBuf* b : {&pre, &q, &rows, &joff, &jobs, &out}) b->release();
    };
    if ((e = pre.ensure((size_t)pre_stride * I.S * 4)) != cudaSuccess || (e = q.ensure(hq.size() * 4)) != cudaSuccess ||
        (e = rows.ensure(I.S * 4)) != cudaSuccess || (e = joff.ensure((I.S + 1) * 4)) != cudaSuccess ||
        (e = jobs.ensure(I.S * sizeof(JumpJob))) != cudaSuccess || (e = out.ensure((size_t)I.S * I.N * 4)) != cudaSuccess) {
        cleanup();
        return e;
    }
    cudaMemcpyAsync(q.p, hq.data(), hq.size() * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(rows.p, hrows.data(), I.S * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(joff.p, hoff.data(), (I.S + 1) * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(jobs.p, hjobs.data(), I.S * sizeof(JumpJob), cudaMemcpyHostToDevice, st);
    e = I.prefix(params, win, rows.as<uint32_t>(), I.S, pre.as<uint32_t>(), pre_stride, st);
    if (e == cudaSuccess) {
        JumpArgs ja;
        ja.pre = pre.as<uint32_t>();
        ja.pre_len = pre_len;
        ja.pre_stride = pre_stride;
        ja.pre_off = I.t0;
        ja.set_of = rows.as<uint32_t>();
        ja.job_off = joff.as<uint32_t>();
        ja.jobs = jobs.as<JumpJob>();
        ja.q = q.as<uint32_t>();
        ja.q_words = qw;
        ja.piece_win = out.as<uint32_t>();
        ja.n_jobs = I.S;
        e = I.jump(ja, I.S, st);
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(win, out.p, (size_t)I.S * I.N * 4, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cleanup();
    return e;
}

}  // namespace mtgpb
