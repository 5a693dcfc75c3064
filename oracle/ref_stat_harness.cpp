// ref_stat_harness.cpp -- extern "C" shim over the UNMODIFIED reference statistical tests and
// parameter-set tooling, compiled with the reference's own sources
// (proj/src/{stat_tests,stats,classify,gf2poly,dynamic_creator}.cpp and the header templates
// proj/include/twistsieve/stat_tests.hpp:83-309) into
// oracle/_ref/libtwistsieve_ref.so by oracle/Makefile. TEST INFRASTRUCTURE ONLY: the checker for
// the device-side stat tests (tests/test_stat_*.py) and the generator of
// tests/golden/stat_reference.json.
//
// Everything goes through the reference's public API: TestSpec / run_test (stat_tests.hpp),
// make_word_source + BufferedStream (word_source.hpp:75-97, the exact campaign cell of
// sieve.cpp:156-158), and the numerics of stats.hpp / classify.hpp.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "twistsieve/classify.hpp"
#include "twistsieve/dynamic_creator.hpp"
#include "twistsieve/gf2poly.hpp"
#include "twistsieve/params.hpp"
#include "twistsieve/stat_tests.hpp"
#include "twistsieve/stats.hpp"
#include "twistsieve/word_source.hpp"

using namespace twistsieve;

extern "C" {

// Same layout as mtgp_stat_spec / mtgp_stat_result in include/mtgp_b200.h.
struct ref_stat_spec {
    int32_t test;  // 0 gap, 1 hamming_indep, 2 collision_over, 3 random_walk
    uint32_t N;
    uint64_t n;
    uint32_t r, s, L, d, l, t;
    double alpha, beta;
};

struct ref_stat_result {
    double statistic, p_value;
    int32_t classification, degenerate, error, pad;
    uint64_t words_used;
};

}  // extern "C"

namespace {

thread_local std::string g_msg;

TestSpec to_spec(const ref_stat_spec& s) {
    static const char* ids[] = {"gap", "hamming_indep", "collision_over", "random_walk"};
    TestSpec t;
    t.test_id = (s.test >= 0 && s.test < 4) ? ids[s.test] : "unknown";
    t.N = s.N;
    t.n = s.n;
    t.r = s.r;
    t.alpha = s.alpha;
    t.beta = s.beta;
    t.s = s.s;
    t.L = s.L;
    t.d = s.d;
    t.l = s.l;
    t.t = s.t;
    return t;
}

// A finite word buffer with the Stream interface the templates take; counts what it hands out.
struct CountingStream {
    const uint32_t* w;
    uint64_t n, pos = 0;
    uint32_t next_u32() {
        if (pos == n) throw StreamExhausted{};
        return w[pos++];
    }
};

void store(const TestResult& r, ref_stat_result* out) {
    out->statistic = r.statistic;
    out->p_value = r.p_value;
    out->classification = static_cast<int32_t>(r.classification);
    out->degenerate = r.degenerate ? 1 : 0;
    out->error = 0;
    out->pad = 0;
}

ParameterizedStatus status_from12(const uint32_t* f) {
    ParameterizedStatus p;
    p.id = static_cast<std::uint16_t>(f[0]);
    p.mexp = f[1];
    p.n = f[2];
    p.m = f[3];
    p.r = f[4];
    p.a = f[5];
    p.temper_b = f[6];
    p.temper_c = f[7];
    p.temper_u = f[8];
    p.temper_s = f[9];
    p.temper_t = f[10];
    p.temper_l = f[11];
    return p;
}

}  // namespace

extern "C" {

const char* ref_stat_last_message(void) { return g_msg.c_str(); }

// run_test over words[0, n_words). Returns 0 ok, 1 std::invalid_argument, 2 StreamExhausted,
// 3 anything else; the message is in ref_stat_last_message().
int ref_stat_run_words(const uint32_t* words, uint64_t n_words, const ref_stat_spec* spec,
                       ref_stat_result* out) {
    std::memset(out, 0, sizeof(*out));
    CountingStream st{words, n_words};
    try {
        const TestResult r = run_test(st, to_spec(*spec));
        store(r, out);
        out->words_used = st.pos;
        return 0;
    } catch (const StreamExhausted& e) {
        g_msg = e.what();
        out->error = 2;
        out->words_used = st.pos;
        return 2;
    } catch (const std::invalid_argument& e) {
        g_msg = e.what();
        out->error = 1;
        return 1;
    } catch (const std::exception& e) {
        g_msg = e.what();
        out->error = 3;
        return 3;
    }
}

// One campaign cell exactly as run_grid runs it (sieve.cpp:156-158): a fresh
// make_word_source(status, seed) behind a BufferedStream. status12 == NULL: mt19937_params().
int ref_stat_run_cell(const uint32_t* status12, uint32_t seed, const ref_stat_spec* spec,
                      ref_stat_result* out) {
    std::memset(out, 0, sizeof(*out));
    try {
        const ParameterizedStatus p = status12 ? status_from12(status12) : mt19937_params();
        auto source = make_word_source(p, seed);
        BufferedStream stream(*source);
        store(run_test(stream, to_spec(*spec)), out);
        return 0;
    } catch (const StreamExhausted& e) {
        g_msg = e.what();
        out->error = 2;
        return 2;
    } catch (const std::invalid_argument& e) {
        g_msg = e.what();
        out->error = 1;
        return 1;
    } catch (const std::exception& e) {
        g_msg = e.what();
        out->error = 3;
        return 3;
    }
}

// The numerics of stats.hpp / classify.hpp. fn: 0 ln_gamma(a), 1 P(a,x=b), 2 Q(a,x=b),
// 3 chi_square_pvalue(a, df=k), 4 poisson_cdf(k, a), 5 poisson_sf(k, a), 6 poisson_pmf(k, a),
// 7 binomial_log_pmf(k, n, a), 8 binomial_upper_tail(k, n, a), 9 classify_pvalue(a).
// Returns 0 ok, 1 std::invalid_argument (message in ref_stat_last_message()).
int ref_stat_math(int fn, double a, double b, uint64_t k, uint64_t n, double* out) {
    try {
        switch (fn) {
            case 0: *out = ln_gamma(a); return 0;
            case 1: *out = regularized_gamma_p(a, b); return 0;
            case 2: *out = regularized_gamma_q(a, b); return 0;
            case 3: *out = chi_square_pvalue(a, static_cast<unsigned>(k)); return 0;
            case 4: *out = poisson_cdf(k, a); return 0;
            case 5: *out = poisson_sf(k, a); return 0;
            case 6: *out = poisson_pmf(k, a); return 0;
            case 7: *out = binomial_log_pmf(k, n, a); return 0;
            case 8: *out = binomial_upper_tail(k, n, a); return 0;
            case 9: *out = static_cast<double>(static_cast<int>(classify_pvalue(a))); return 0;
        }
        g_msg = "unknown function";
        return 1;
    } catch (const std::invalid_argument& e) {
        g_msg = e.what();
        return 1;
    }
}

// Desk-scale specs of the reference (stat_tests.cpp: desk_*_spec), by index 0..3.
int ref_stat_desk_spec(int i, ref_stat_spec* out) {
    std::memset(out, 0, sizeof(*out));
    const auto b = desk_battery();
    if (i < 0 || i >= static_cast<int>(b.size())) return 1;
    const TestSpec& t = b[i];
    static const char* ids[] = {"gap", "hamming_indep", "collision_over", "random_walk"};
    for (int j = 0; j < 4; ++j)
        if (t.test_id == ids[j]) out->test = j;
    out->N = t.N;
    out->n = t.n;
    out->r = t.r;
    out->s = t.s;
    out->L = t.L;
    out->d = t.d;
    out->l = t.l;
    out->t = t.t;
    out->alpha = t.alpha;
    out->beta = t.beta;
    return 0;
}

// gap_expected_counts (stat_tests.cpp): the tcut the gap test uses is size() - 1.
int ref_gap_tcut(const ref_stat_spec* spec, uint64_t* tcut) {
    try {
        *tcut = gap_expected_counts(to_spec(*spec)).size() - 1;
        return 0;
    } catch (const std::invalid_argument& e) {
        g_msg = e.what();
        return 1;
    }
}

}  // extern "C"

extern "C" {

// The reference's is_irreducible (gf2poly.cpp:342-383) on sum_i bits[i] x^i.
// Returns 1 / 0, or -1 if it throws (constant polynomial).
int ref_is_irreducible(const uint8_t* bits, uint64_t n) {
    try {
        return is_irreducible(Gf2Poly::from_coeff_bits(std::span<const std::uint8_t>(bits, n))) ? 1 : 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// poly_digest(probe_minimal_polynomial(Generator(status, seed), mexp)) and its degree
// (dynamic_creator.cpp:9-38). status12 == NULL: mt19937_params().
int ref_mt_probe_digest(const uint32_t* status12, uint32_t seed, char* out41, int* degree) {
    try {
        const ParameterizedStatus p = status12 ? status_from12(status12) : mt19937_params();
        const Gf2Poly poly = probe_minimal_polynomial(Generator(p, seed), p.mexp);
        const std::string d = poly_digest(poly);
        std::memset(out41, 0, 41);
        std::memcpy(out41, d.data(), std::min<size_t>(40, d.size()));
        *degree = poly.degree();
        return 0;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 1;
    }
}

}  // extern "C"

extern "C" {

// The reference's dc_search acceptance test (dynamic_creator.cpp:79-81) on an arbitrary word
// stream: berlekamp_massey over bit 0 of words[0, 2*mexp + 64) (probe_minimal_polynomial,
// :33-38), then degree == mexp && is_irreducible. *irreducible = -1 when the degree differs.
int ref_bit0_certify(const uint32_t* words, uint64_t nwords, uint32_t mexp, int* degree, int* irreducible) {
    const std::size_t nbits = 2 * static_cast<std::size_t>(mexp) + 64;
    if (nwords < nbits) return 1;
    std::vector<std::uint8_t> bits(nbits);
    for (std::size_t k = 0; k < nbits; ++k) bits[k] = static_cast<std::uint8_t>(words[k] & 1u);
    const Gf2Poly poly = berlekamp_massey(bits);
    *degree = poly.degree();
    *irreducible = poly.degree() == static_cast<int>(mexp) ? (is_irreducible(poly) ? 1 : 0) : -1;
    return 0;
}

}  // extern "C"
