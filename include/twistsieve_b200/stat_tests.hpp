// twistsieve_b200/stat_tests.hpp -- the reference's statistical tests, run on the GPU over
// device-generated streams ("GPU-fed consumers").
//
// Mirrors proj/include/twistsieve/stat_tests.hpp (TestSpec :18-33, TestResult :35-42, desk specs /
// named_spec, run_test :313-319), classify.hpp (PValueClass, classify_pvalue) and the campaign
// grid of proj/include/twistsieve/sieve.hpp (ResultRow, run_grid = sieve.cpp:116-183). The
// reference runs one test per fresh stream on one CPU core; here run_test tests every stream of a
// StreamBatch at once on the GPU (words never leave HBM) and returns what the reference template
// would return for each stream, bit for bit (statistic, p-value, class, degenerate flag).
//
// Errors follow the reference: an invalid spec throws std::invalid_argument with the reference's
// message; a stream that runs out of its word budget (gap test) is reported per stream as
// StreamExhausted's message "insufficient stream" (word_source.hpp:15-17). run_grid records
// both as per-row errors, as run_grid does (sieve.cpp:163-165).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "mtgp_b200.h"
#include "twistsieve_b200/mtgp.hpp"

namespace twistsieve_b200 {

/// classify.hpp:11: [0.001, 0.999] correct; outside suspect; within 1e-10 of 0 or 1 disastrous.
enum class PValueClass { correct = MTGP_PCLASS_CORRECT, suspect = MTGP_PCLASS_SUSPECT, disastrous = MTGP_PCLASS_DISASTROUS };
const char* to_string(PValueClass c);
PValueClass classify_pvalue(double p);

/// stat_tests.hpp:18-33.
struct TestSpec {
    std::string test_id;  // "gap" | "hamming_indep" | "collision_over" | "random_walk"
    std::uint32_t N = 1;
    std::uint64_t n = 0;
    std::uint32_t r = 0;
    double alpha = 0.0;
    double beta = 0.0;
    std::uint32_t s = 0;
    std::uint32_t L = 0;
    std::uint32_t d = 0;
    std::uint32_t l = 0;
    std::uint32_t t = 0;

    void validate() const;  // TestSpec::validate + the test's pre-read checks
    std::string describe() const;
    mtgp_stat_spec to_c() const;
    bool operator==(const TestSpec&) const = default;
};

/// stat_tests.hpp:35-42.
struct TestResult {
    TestSpec spec;
    std::string status_id;
    double statistic = 0.0;
    double p_value = 0.0;
    PValueClass classification = PValueClass::correct;
    bool degenerate = false;
};

TestSpec desk_gap_spec();      // n=1e6 gaps, r=25, [0, 1/32)
TestSpec desk_hamming_spec();  // n=1e5 blocks, r=25, s=5, L=1200
TestSpec desk_opso_spec();     // n=2^15 pairs, s=11, lambda=128
TestSpec desk_walk_spec();     // n=1e5 walks, l=128
std::vector<TestSpec> desk_battery();
TestSpec named_spec(const std::string& name);  // canonical ids + "hamming", "opso", "walk"

/// One stream's outcome: the TestResult, or the per-stream error message.
struct StreamTest {
    TestResult result;
    std::string error;  // "" or "insufficient stream"
    std::uint64_t words_used = 0;
    bool is_error() const { return !error.empty(); }
};

/// run_test(spec) on every stream of `batch` on the GPU, each from its current position; the
/// batch's state and checksums are unchanged afterwards.
std::vector<StreamTest> run_test(StreamBatch& batch, const TestSpec& spec);

/// sieve.hpp ResultRow: one (status, seed, test) cell.
struct ResultRow {
    std::uint32_t status_index = 0;
    std::uint32_t seed_index = 0;
    std::string status_id;
    std::string test_id;
    std::uint32_t seed = 0;
    double statistic = 0.0;
    double p_value = 0.0;
    PValueClass classification = PValueClass::correct;
    bool degenerate = false;
    std::string error;
    bool is_error() const { return !error.empty(); }
};

/// Every (status, seed, test) cell on fresh streams, rows ordered (status, seed, test) like
/// run_grid (sieve.cpp:116-183); all status x seed streams share one GPU context.
std::vector<ResultRow> run_grid(const std::vector<MtStatus>& statuses, const std::vector<std::uint32_t>& seeds,
                                const std::vector<TestSpec>& specs, int device = 0);
std::vector<ResultRow> run_grid(const std::vector<MtgpStatus>& statuses, const std::vector<std::uint32_t>& seeds,
                                const std::vector<TestSpec>& specs, int device = 0);

/// "m<mexp>-id<id>", the reference's status_display_id for Engine::mt (params.cpp:41-48).
std::string status_display_id(const MtStatus& p);

// Numerics of proj/include/twistsieve/stats.hpp (host; std::invalid_argument as the reference).
double ln_gamma(double x);
double regularized_gamma_p(double a, double x);
double regularized_gamma_q(double a, double x);
double chi_square_pvalue(double statistic, unsigned df);
double poisson_cdf(std::uint64_t k, double lambda);
double poisson_sf(std::uint64_t k, double lambda);
double poisson_pmf(std::uint64_t k, double lambda);
double binomial_upper_tail(std::uint64_t count, std::uint64_t n, double p);

}  // namespace twistsieve_b200
