// stat_host.h -- host half of the device-side statistical tests: spec validation, the numerics,
// and the step from integer counts to (statistic, p-value, class). Private to libmtgp_b200.so.
#pragma once
#include <cstdint>
#include <vector>

#include "mtgp_b200.h"

namespace mtgpb::stat {

// Numerics of proj/include/twistsieve/stats.hpp; std::invalid_argument where the reference
// throws it (same messages).
double ln_gamma(double x);
double gamma_p(double a, double x);
double gamma_q(double a, double x);
double chi_square_pvalue(double statistic, unsigned df);
double poisson_cdf(uint64_t k, double lambda);
double poisson_sf(uint64_t k, double lambda);
double poisson_pmf(uint64_t k, double lambda);
double binomial_log_pmf(uint64_t k, uint64_t n, double p);
double binomial_upper_tail(uint64_t count, uint64_t n, double p);
int classify_pvalue(double p);  // MTGP_PCLASS_*

// TestSpec::validate plus the test's checks that precede any stream read.
void validate(const mtgp_stat_spec& spec);

// Shape of the count vector mtgp_stat_finish takes.
uint64_t counts_len(const mtgp_stat_spec& spec);

// Gap test (stat_tests.hpp:84-138): tail cut, word budget, and the integer form of the
// interval test: lo <= (w & mask) < hi  <=>  alpha <= (w & mask) * 2^-(32-r) < beta.
struct GapShape {
    uint64_t tcut;
    uint64_t budget;
    uint32_t mask;
    uint64_t lo, hi;
};
GapShape gap_shape(const mtgp_stat_spec& spec);

// Words each fixed-length test reads from the stream.
uint64_t words_needed(const mtgp_stat_spec& spec);

// counts -> result (statistic, p-value, class, degenerate); error fields untouched.
void finish(const mtgp_stat_spec& spec, const uint64_t* counts, mtgp_stat_result* out);

}  // namespace mtgpb::stat
