// stat_host.cpp -- host half of the device-side statistical tests (include/mtgp_b200.h,
// "Device-side statistical tests").
//
// The numerics restate the reference's proj/src/stats.cpp and classify.cpp: Lanczos ln Gamma
// (g = 7, the published 9-term coefficient set), the series / modified-Lentz continued fraction
// for the regularized incomplete gamma, and the chi-square / Poisson / binomial tails built on
// them. The reference hand-rolls these "so report bytes do not depend on the platform's libm"
// (stats.hpp:9-10); every floating-point operation below is performed in the reference's
// order, so statistic and p-value match it bit for bit (tests/test_stat_cpu.py pins this
// against the reference compiled from its sources).
//
// The per-test finishing (counts -> statistic) restates stat_tests.hpp:84-309 with the counting
// moved to the GPU (csrc/mtgp_stat.cu).
#include "stat_host.h"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

namespace mtgpb::stat {

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kHalfLn2Pi = 0.91893853320467274178;  // ln(2*pi)/2
// Lanczos coefficients for g = 7, n = 9 (the standard published set).
constexpr double kLanczosG7[9] = {0.99999999999980993,  676.5203681218851,    -1259.1392167224028,
                                  771.32342877765313,   -176.61502916214059,  12.507343278686905,
                                  -0.13857109526572012, 9.9843695780195716e-6, 1.5056327351493116e-7};

// exp(-x + a ln x - ln Gamma(a)): the prefactor both expansions share.
double gamma_prefactor(double a, double x) { return std::exp(-x + a * std::log(x) - ln_gamma(a)); }

// P(a, x) by its power series, for x < a + 1 (stats.cpp:20-29).
double p_series(double a, double x) {
    double term = 1.0 / a;
    double sum = term;
    for (int k = 1; k < 10000; ++k) {
        term *= x / (a + k);
        sum += term;
        if (std::fabs(term) < std::fabs(sum) * 1e-16) break;
    }
    return sum * gamma_prefactor(a, x);
}

// Q(a, x) by the modified Lentz continued fraction, for x >= a + 1 (stats.cpp:32-51).
double q_fraction(double a, double x) {
    constexpr double floor_ = 1e-300;
    double b = x + 1.0 - a;
    double c = 1.0 / floor_;
    double d = 1.0 / b;
    double h = d;
    for (int i = 1; i < 10000; ++i) {
        const double an = -static_cast<double>(i) * (static_cast<double>(i) - a);
        b += 2.0;
        d = an * d + b;
        if (std::fabs(d) < floor_) d = floor_;
        c = b + an / c;
        if (std::fabs(c) < floor_) c = floor_;
        d = 1.0 / d;
        const double step = d * c;
        h *= step;
        if (std::fabs(step - 1.0) < 1e-16) break;
    }
    return h * gamma_prefactor(a, x);
}

void check_gamma_args(double a, double x) {
    if (!(a > 0.0) || x < 0.0) throw std::invalid_argument("regularized gamma requires a > 0, x >= 0");
}

void check_lambda(double lambda) {
    if (!(lambda > 0.0)) throw std::invalid_argument("lambda must be > 0");
}

}  // namespace

double ln_gamma(double x) {
    if (!(x > 0.0)) throw std::invalid_argument("ln_gamma requires x > 0");
    if (x < 0.5) return std::log(kPi / std::sin(kPi * x)) - ln_gamma(1.0 - x);  // reflection
    const double z = x - 1.0;
    double series = kLanczosG7[0];
    for (int i = 1; i < 9; ++i) series += kLanczosG7[i] / (z + i);
    const double t = z + 7.5;
    return kHalfLn2Pi + (z + 0.5) * std::log(t) - t + std::log(series);
}

double gamma_p(double a, double x) {
    check_gamma_args(a, x);
    if (x == 0.0) return 0.0;
    return x < a + 1.0 ? p_series(a, x) : 1.0 - q_fraction(a, x);
}

double gamma_q(double a, double x) {
    check_gamma_args(a, x);
    if (x == 0.0) return 1.0;
    return x < a + 1.0 ? 1.0 - p_series(a, x) : q_fraction(a, x);
}

double chi_square_pvalue(double statistic, unsigned df) {
    if (statistic < 0.0) throw std::invalid_argument("negative chi-square statistic");
    if (df < 1) throw std::invalid_argument("chi-square df must be >= 1");
    return gamma_q(0.5 * static_cast<double>(df), 0.5 * statistic);
}

double poisson_cdf(uint64_t k, double lambda) {  // P(X <= k) = Q(k+1, lambda)
    check_lambda(lambda);
    return gamma_q(static_cast<double>(k) + 1.0, lambda);
}

double poisson_sf(uint64_t k, double lambda) {  // P(X >= k) = P(k, lambda), k >= 1
    check_lambda(lambda);
    return k == 0 ? 1.0 : gamma_p(static_cast<double>(k), lambda);
}

double poisson_pmf(uint64_t k, double lambda) {
    check_lambda(lambda);
    const double kf = static_cast<double>(k);
    return std::exp(-lambda + kf * std::log(lambda) - ln_gamma(kf + 1.0));
}

double binomial_log_pmf(uint64_t k, uint64_t n, double p) {
    const double nf = static_cast<double>(n), kf = static_cast<double>(k);
    const double log_choose = ln_gamma(nf + 1.0) - ln_gamma(kf + 1.0) - ln_gamma(nf - kf + 1.0);
    return log_choose + kf * std::log(p) + (nf - kf) * std::log1p(-p);
}

double binomial_upper_tail(uint64_t count, uint64_t n, double p) {
    if (!(p > 0.0) || !(p < 1.0)) throw std::invalid_argument("binomial p must be in (0, 1)");
    if (count > n) throw std::invalid_argument("count must be <= n");
    if (count == 0) return 1.0;
    // first term in log space, then the term ratio (n-k)/(k+1) * p/(1-p) upward
    double term = std::exp(binomial_log_pmf(count, n, p));
    double sum = term;
    const double odds = p / (1.0 - p);
    for (uint64_t k = count; k < n; ++k) {
        term *= static_cast<double>(n - k) / static_cast<double>(k + 1) * odds;
        sum += term;
        if (term < sum * 1e-18) break;
    }
    return std::min(sum, 1.0);
}

int classify_pvalue(double p) {  // classify.cpp:18-24
    if (!(p >= 0.0) || !(p <= 1.0)) throw std::invalid_argument("p-value outside [0, 1]");
    if (p < 1e-10 || p > 1.0 - 1e-10) return MTGP_PCLASS_DISASTROUS;
    if (p < 0.001 || p > 0.999) return MTGP_PCLASS_SUSPECT;
    return MTGP_PCLASS_CORRECT;
}

// ---------------------------------------------------------------------------------------------
// specs

namespace {

// Largest cut t with n(1-p)^(t+1) >= 5 and n p (1-p)^t >= 5, t < 65536 (stat_tests.hpp:93-101).
uint64_t gap_cut(uint64_t n, double p) {
    const double q = 1.0 - p;
    const double nf = static_cast<double>(n);
    uint64_t t = 1;
    while (t < 65536 && nf * std::pow(q, static_cast<double>(t + 1)) >= 5.0 &&
           nf * p * std::pow(q, static_cast<double>(t)) >= 5.0)
        ++t;
    return t;
}

// Binomial(l, 1/2) pmf and the merged tails of the random-walk test (stat_tests.hpp:260-276).
struct WalkCells {
    std::vector<double> pmf;
    uint32_t lo, hi;
    bool ok;
};

WalkCells walk_cells(const mtgp_stat_spec& s) {
    WalkCells w;
    w.pmf.resize(s.l + 1);
    w.pmf[0] = std::ldexp(1.0, -static_cast<int>(s.l));
    for (uint32_t h = 0; h < s.l; ++h)
        w.pmf[h + 1] = w.pmf[h] * static_cast<double>(s.l - h) / static_cast<double>(h + 1);
    const double nf = static_cast<double>(s.n);
    uint32_t lo = 0;
    double cum = w.pmf[0];
    while (lo + 1 < s.l / 2 && !(nf * cum >= 5.0 && nf * w.pmf[lo + 1] >= 5.0)) {
        ++lo;
        cum += w.pmf[lo];
    }
    w.lo = lo;
    w.hi = s.l - lo;
    w.ok = nf * cum >= 5.0 && (lo + 1 > w.hi - 1 || nf * w.pmf[lo + 1] >= 5.0);
    return w;
}

double opso_lambda(const mtgp_stat_spec& s) {
    const uint64_t k = 1ull << (2 * s.s);
    return static_cast<double>(s.n) * static_cast<double>(s.n) / (2.0 * static_cast<double>(k));
}

}  // namespace

void validate(const mtgp_stat_spec& s) {
    // TestSpec::validate (stat_tests.cpp:7-30)
    if (s.n < 1) throw std::invalid_argument("sample size n must be >= 1");
    if (s.r > 31) throw std::invalid_argument("r must be in [0, 31]");
    switch (s.test) {
        case MTGP_STAT_GAP:
            if (!(s.alpha >= 0.0 && s.alpha < s.beta && s.beta <= 1.0))
                throw std::invalid_argument("gap test requires 0 <= alpha < beta <= 1");
            break;
        case MTGP_STAT_HAMMING_INDEP:
            if (s.s < 1 || s.s > 31) throw std::invalid_argument("s must be in [1, 31]");
            if (s.r + s.s > 32) throw std::invalid_argument("r + s must be <= 32");
            if (s.L < 1) throw std::invalid_argument("block length L must be >= 1");
            if (s.d != 0) throw std::invalid_argument("only d = 0 is supported");
            break;
        case MTGP_STAT_COLLISION_OVER:
            if (s.s < 1 || s.s > 14) throw std::invalid_argument("s must be in [1, 14]");
            if (s.r + s.s > 32) throw std::invalid_argument("r + s must be <= 32");
            if (s.t != 0 && s.t != 2 * s.s) throw std::invalid_argument("cell-count exponent t must equal 2*s");
            break;
        case MTGP_STAT_RANDOM_WALK:
            if (s.l < 2 || s.l % 2 != 0) throw std::invalid_argument("walk length l must be even and >= 2");
            break;
        default:
            throw std::invalid_argument("unknown test id: " + std::to_string(s.test));
    }
    // checks each test makes before its first next_u32()
    switch (s.test) {
        case MTGP_STAT_HAMMING_INDEP:  // stat_tests.hpp:154-155
            if (s.n / 2 < 100) throw std::invalid_argument("sample too small");
            break;
        case MTGP_STAT_COLLISION_OVER: {  // stat_tests.hpp:219-222
            const double lambda = opso_lambda(s);
            if (lambda < 1.0 || lambda > 10.0 * static_cast<double>(s.n))
                throw std::invalid_argument("spec out of sparse regime");
            break;
        }
        case MTGP_STAT_RANDOM_WALK:  // stat_tests.hpp:276-277
            if (!walk_cells(s).ok) throw std::invalid_argument("sample too small");
            break;
        default:
            break;
    }
}

uint64_t counts_len(const mtgp_stat_spec& s) {
    switch (s.test) {
        case MTGP_STAT_GAP: return gap_cut(s.n, s.beta - s.alpha) + 1;
        case MTGP_STAT_HAMMING_INDEP: return 4;
        case MTGP_STAT_COLLISION_OVER: return 1;
        case MTGP_STAT_RANDOM_WALK: return static_cast<uint64_t>(s.l) + 1;
    }
    return 0;
}

GapShape gap_shape(const mtgp_stat_spec& s) {
    GapShape g;
    const double p = s.beta - s.alpha;
    g.tcut = gap_cut(s.n, p);
    // stat_tests.hpp:106-107: (n+1)/p * 8 words of headroom, + 4096
    g.budget = static_cast<uint64_t>(static_cast<double>(s.n + 1) / p * 8.0) + 4096;
    const uint32_t kept = 32 - s.r;
    g.mask = s.r == 0 ? 0xFFFFFFFFu : (0xFFFFFFFFu >> s.r);
    // v * 2^-kept is exact, so u >= alpha <=> v >= ceil(alpha 2^kept) and
    // u < beta <=> v < ceil(beta 2^kept) for integer v.
    g.lo = static_cast<uint64_t>(std::ceil(std::ldexp(s.alpha, static_cast<int>(kept))));
    g.hi = static_cast<uint64_t>(std::ceil(std::ldexp(s.beta, static_cast<int>(kept))));
    return g;
}

uint64_t words_needed(const mtgp_stat_spec& s) {
    switch (s.test) {
        case MTGP_STAT_HAMMING_INDEP: {
            const uint64_t bits = (s.n / 2) * 2 * static_cast<uint64_t>(s.L);
            return (bits + s.s - 1) / s.s;
        }
        case MTGP_STAT_COLLISION_OVER: return s.n + 1;
        case MTGP_STAT_RANDOM_WALK: return s.n * static_cast<uint64_t>(s.l);
    }
    return 0;
}

void finish(const mtgp_stat_spec& s, const uint64_t* counts, mtgp_stat_result* out) {
    double statistic = 0.0, pv = 1.0;
    bool degenerate = false;
    switch (s.test) {
        case MTGP_STAT_GAP: {  // stat_tests.hpp:127-137
            const double p = s.beta - s.alpha, q = 1.0 - p;
            const double nf = static_cast<double>(s.n);
            const uint64_t tcut = gap_cut(s.n, p);
            for (uint64_t c = 0; c <= tcut; ++c) {
                const double expected = c < tcut ? nf * p * std::pow(q, static_cast<double>(c))
                                                 : nf * std::pow(q, static_cast<double>(tcut));
                const double diff = static_cast<double>(counts[c]) - expected;
                statistic += diff * diff / expected;
            }
            pv = chi_square_pvalue(statistic, static_cast<unsigned>(tcut));
            break;
        }
        case MTGP_STAT_HAMMING_INDEP: {  // stat_tests.hpp:195-207
            const double a = static_cast<double>(counts[0]), b = static_cast<double>(counts[1]);
            const double c = static_cast<double>(counts[2]), d = static_cast<double>(counts[3]);
            const double row0 = a + b, row1 = c + d, col0 = a + c, col1 = b + d;
            if (row0 == 0 || row1 == 0 || col0 == 0 || col1 == 0) {
                degenerate = true;
                break;  // statistic 0, p = 1
            }
            const double total = row0 + row1;
            const double delta = a * d - b * c;
            statistic = total * delta * delta / (row0 * row1 * col0 * col1);
            pv = chi_square_pvalue(statistic, 1);
            break;
        }
        case MTGP_STAT_COLLISION_OVER: {  // stat_tests.hpp:240-247
            const uint64_t coll = counts[0];
            const double lambda = opso_lambda(s);
            const double atom = poisson_pmf(coll, lambda);
            const double below = coll == 0 ? 0.0 : poisson_cdf(coll - 1, lambda);
            const double above = poisson_sf(coll + 1, lambda);
            const double p_low = below + 0.5 * atom;
            const double p_high = above + 0.5 * atom;
            pv = std::min(1.0, 2.0 * std::min(p_low, p_high));
            statistic = static_cast<double>(coll);
            break;
        }
        case MTGP_STAT_RANDOM_WALK: {  // stat_tests.hpp:286-307
            const WalkCells w = walk_cells(s);
            const double nf = static_cast<double>(s.n);
            double obs_lo = 0, obs_hi = 0, exp_lo = 0, exp_hi = 0;
            for (uint32_t h = 0; h <= w.lo; ++h) {
                obs_lo += static_cast<double>(counts[h]);
                exp_lo += nf * w.pmf[h];
            }
            for (uint32_t h = w.hi; h <= s.l; ++h) {
                obs_hi += static_cast<double>(counts[h]);
                exp_hi += nf * w.pmf[h];
            }
            auto cell = [&](double observed, double expected) {
                const double diff = observed - expected;
                statistic += diff * diff / expected;
            };
            cell(obs_lo, exp_lo);
            unsigned cells = 2;
            for (uint32_t h = w.lo + 1; h < w.hi; ++h, ++cells) cell(static_cast<double>(counts[h]), nf * w.pmf[h]);
            cell(obs_hi, exp_hi);
            pv = chi_square_pvalue(statistic, cells - 1);
            break;
        }
        default:
            throw std::invalid_argument("unknown test id: " + std::to_string(s.test));
    }
    out->statistic = statistic;
    out->p_value = pv;
    out->classification = classify_pvalue(pv);
    out->degenerate = degenerate ? 1 : 0;
}

}  // namespace mtgpb::stat

// ---------------------------------------------------------------------------------------------
// C-ABI (host-only entry points; mtgp_stat_run lives in mtgp_stat.cu)

namespace mtgpb {
int set_error(int code, const char* fmt, ...);
}

namespace {
template <class F>
int guarded(F&& f) {
    try {
        f();
        return MTGP_OK;
    } catch (const std::invalid_argument& e) {
        return mtgpb::set_error(MTGP_EINVAL, "%s", e.what());
    } catch (const std::exception& e) {
        return mtgpb::set_error(MTGP_EINVAL, "%s", e.what());
    }
}
int null_arg() { return mtgpb::set_error(MTGP_EINVAL, "null argument"); }
}  // namespace

extern "C" {

int mtgp_stat_validate(const mtgp_stat_spec* spec) {
    if (!spec) return null_arg();
    return guarded([&] { mtgpb::stat::validate(*spec); });
}

int mtgp_stat_counts_len(const mtgp_stat_spec* spec, uint64_t* n) {
    if (!spec || !n) return null_arg();
    return guarded([&] {
        mtgpb::stat::validate(*spec);
        *n = mtgpb::stat::counts_len(*spec);
    });
}

int mtgp_stat_finish(const mtgp_stat_spec* spec, const uint64_t* counts, uint64_t n_counts,
                     mtgp_stat_result* out) {
    if (!spec || !counts || !out) return null_arg();
    return guarded([&] {
        mtgpb::stat::validate(*spec);
        if (n_counts != mtgpb::stat::counts_len(*spec))
            throw std::invalid_argument("count vector has the wrong length for this spec");
        *out = mtgp_stat_result{};
        mtgpb::stat::finish(*spec, counts, out);
    });
}

int mtgp_ln_gamma(double x, double* out) {
    if (!out) return null_arg();
    return guarded([&] { *out = mtgpb::stat::ln_gamma(x); });
}
int mtgp_gamma_p(double a, double x, double* out) {
    if (!out) return null_arg();
    return guarded([&] { *out = mtgpb::stat::gamma_p(a, x); });
}
int mtgp_gamma_q(double a, double x, double* out) {
    if (!out) return null_arg();
    return guarded([&] { *out = mtgpb::stat::gamma_q(a, x); });
}
int mtgp_chi_square_pvalue(double statistic, uint32_t df, double* out) {
    if (!out) return null_arg();
    return guarded([&] { *out = mtgpb::stat::chi_square_pvalue(statistic, df); });
}
int mtgp_poisson_cdf(uint64_t k, double lambda, double* out) {
    if (!out) return null_arg();
    return guarded([&] { *out = mtgpb::stat::poisson_cdf(k, lambda); });
}
int mtgp_poisson_sf(uint64_t k, double lambda, double* out) {
    if (!out) return null_arg();
    return guarded([&] { *out = mtgpb::stat::poisson_sf(k, lambda); });
}
int mtgp_poisson_pmf(uint64_t k, double lambda, double* out) {
    if (!out) return null_arg();
    return guarded([&] { *out = mtgpb::stat::poisson_pmf(k, lambda); });
}
int mtgp_binomial_log_pmf(uint64_t k, uint64_t n, double p, double* out) {
    if (!out) return null_arg();
    return guarded([&] { *out = mtgpb::stat::binomial_log_pmf(k, n, p); });
}
int mtgp_binomial_upper_tail(uint64_t count, uint64_t n, double p, double* out) {
    if (!out) return null_arg();
    return guarded([&] { *out = mtgpb::stat::binomial_upper_tail(count, n, p); });
}
int mtgp_classify_pvalue(double p, int32_t* out) {
    if (!out) return null_arg();
    return guarded([&] { *out = mtgpb::stat::classify_pvalue(p); });
}

}  // extern "C"
