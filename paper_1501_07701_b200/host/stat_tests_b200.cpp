// stat_tests_b200.cpp -- C++ layer of the device-side statistical tests
// (include/twistsieve_b200/stat_tests.hpp) over the C-ABI (mtgp_stat_*, include/mtgp_b200.h).
#include "twistsieve_b200/stat_tests.hpp"

#include <cstdio>

namespace twistsieve_b200 {

namespace {

constexpr const char* kTestIds[] = {"gap", "hamming_indep", "collision_over", "random_walk"};

int test_index(const std::string& id) {
    for (int i = 0; i < 4; ++i)
        if (id == kTestIds[i]) return i;
    return -1;
}

// C-ABI status -> the reference's exception types, message verbatim (campaign rows record
// e.what(), sieve.cpp:163-165).
void raise(int rc) {
    if (rc == MTGP_OK) return;
    if (rc == MTGP_EINVAL) throw std::invalid_argument(mtgp_last_error());
    throw std::runtime_error(mtgp_last_error());
}

TestResult to_result(const TestSpec& spec, const mtgp_stat_result& r) {
    TestResult t;
    t.spec = spec;
    t.statistic = r.statistic;
    t.p_value = r.p_value;
    t.classification = static_cast<PValueClass>(r.classification);
    t.degenerate = r.degenerate != 0;
    return t;
}

template <class Status>
std::vector<ResultRow> grid(const std::vector<Status>& statuses, const std::vector<std::uint32_t>& seeds,
                            const std::vector<TestSpec>& specs, int device) {
    if (statuses.empty()) throw std::invalid_argument("no statuses");
    if (specs.empty()) throw std::invalid_argument("no test specs");
    for (const auto& st : statuses) st.validate();
    std::vector<Status> sts;
    std::vector<std::uint32_t> sds;
    for (const auto& st : statuses)
        for (std::uint32_t seed : seeds) {
            sts.push_back(st);
            sds.push_back(seed);
        }
    StreamBatch batch(sts, sds, device);
    std::vector<std::vector<StreamTest>> per_test;
    for (const auto& spec : specs) {
        try {
            per_test.push_back(run_test(batch, spec));
        } catch (const std::invalid_argument& e) {
            StreamTest err;
            err.result.spec = spec;
            err.error = e.what();
            per_test.emplace_back(sts.size(), err);
        }
    }
    std::vector<ResultRow> rows;
    rows.reserve(sts.size() * specs.size());
    for (std::size_t si = 0; si < statuses.size(); ++si)
        for (std::size_t wi = 0; wi < seeds.size(); ++wi)
            for (std::size_t ti = 0; ti < specs.size(); ++ti) {
                const StreamTest& c = per_test[ti][si * seeds.size() + wi];
                ResultRow row;
                row.status_index = static_cast<std::uint32_t>(si);
                row.seed_index = static_cast<std::uint32_t>(wi);
                row.status_id = status_display_id(statuses[si]);
                row.test_id = specs[ti].test_id;
                row.seed = seeds[wi];
                row.statistic = c.result.statistic;
                row.p_value = c.result.p_value;
                row.classification = c.result.classification;
                row.degenerate = c.result.degenerate;
                row.error = c.error;
                rows.push_back(std::move(row));
            }
    return rows;
}

}  // namespace

const char* to_string(PValueClass c) {
    switch (c) {
        case PValueClass::correct: return "correct";
        case PValueClass::suspect: return "suspect";
        case PValueClass::disastrous: return "disastrous";
    }
    return "correct";
}

PValueClass classify_pvalue(double p) {
    std::int32_t c = 0;
    raise(mtgp_classify_pvalue(p, &c));
    return static_cast<PValueClass>(c);
}

mtgp_stat_spec TestSpec::to_c() const {
    mtgp_stat_spec c{};
    c.test = test_index(test_id);
    c.N = N;
    c.n = n;
    c.r = r;
    c.s = s;
    c.L = L;
    c.d = d;
    c.l = l;
    c.t = t;
    c.alpha = alpha;
    c.beta = beta;
    return c;
}

void TestSpec::validate() const {
    if (test_index(test_id) < 0) throw std::invalid_argument("unknown test id: " + test_id);
    const mtgp_stat_spec c = to_c();
    raise(mtgp_stat_validate(&c));
}

std::string TestSpec::describe() const {  // stat_tests.cpp:32-50
    char buf[160];
    const auto nn = static_cast<unsigned long long>(n);
    if (test_id == "gap")
        std::snprintf(buf, sizeof buf, "gap(n=%llu,r=%u,alpha=%.9g,beta=%.9g)", nn, r, alpha, beta);
    else if (test_id == "hamming_indep")
        std::snprintf(buf, sizeof buf, "hamming_indep(n=%llu,r=%u,s=%u,L=%u,d=%u)", nn, r, s, L, d);
    else if (test_id == "collision_over")
        std::snprintf(buf, sizeof buf, "collision_over(n=%llu,r=%u,s=%u,t=%u)", nn, r, s, t ? t : 2 * s);
    else
        std::snprintf(buf, sizeof buf, "random_walk(n=%llu,r=%u,l=%u)", nn, r, l);
    return buf;
}

TestSpec desk_gap_spec() {
    TestSpec s;
    s.test_id = "gap";
    s.n = 1000000;
    s.r = 25;
    s.alpha = 0.0;
    s.beta = 1.0 / 32.0;
    return s;
}

TestSpec desk_hamming_spec() {
    TestSpec s;
    s.test_id = "hamming_indep";
    s.n = 100000;
    s.r = 25;
    s.s = 5;
    s.L = 1200;
    return s;
}

TestSpec desk_opso_spec() {
    TestSpec s;
    s.test_id = "collision_over";
    s.n = 32768;
    s.s = 11;
    s.t = 22;
    return s;
}

TestSpec desk_walk_spec() {
    TestSpec s;
    s.test_id = "random_walk";
    s.n = 100000;
    s.l = 128;
    return s;
}

std::vector<TestSpec> desk_battery() { return {desk_gap_spec(), desk_hamming_spec(), desk_opso_spec(), desk_walk_spec()}; }

TestSpec named_spec(const std::string& name) {
    if (name == "gap") return desk_gap_spec();
    if (name == "hamming" || name == "hamming_indep") return desk_hamming_spec();
    if (name == "opso" || name == "collision_over") return desk_opso_spec();
    if (name == "walk" || name == "random_walk") return desk_walk_spec();
    throw std::invalid_argument("unknown test name: " + name);
}

std::vector<StreamTest> run_test(StreamBatch& batch, const TestSpec& spec) {
    spec.validate();
    const mtgp_stat_spec c = spec.to_c();
    std::vector<mtgp_stat_result> r(batch.size());
    raise(mtgp_stat_run(batch.handle(), &c, r.data()));
    std::vector<StreamTest> out(batch.size());
    for (std::uint32_t s = 0; s < batch.size(); ++s) {
        out[s].result = to_result(spec, r[s]);
        out[s].words_used = r[s].words_used;
        if (r[s].error == MTGP_STAT_EXHAUSTED) out[s].error = "insufficient stream";
    }
    return out;
}

std::vector<ResultRow> run_grid(const std::vector<MtStatus>& statuses, const std::vector<std::uint32_t>& seeds,
                                const std::vector<TestSpec>& specs, int device) {
    return grid(statuses, seeds, specs, device);
}

std::vector<ResultRow> run_grid(const std::vector<MtgpStatus>& statuses, const std::vector<std::uint32_t>& seeds,
                                const std::vector<TestSpec>& specs, int device) {
    return grid(statuses, seeds, specs, device);
}

std::string status_display_id(const MtStatus& p) { return "m" + std::to_string(p.mexp) + "-id" + std::to_string(p.id); }

double ln_gamma(double x) {
    double v = 0;
    raise(mtgp_ln_gamma(x, &v));
    return v;
}
double regularized_gamma_p(double a, double x) {
    double v = 0;
    raise(mtgp_gamma_p(a, x, &v));
    return v;
}
double regularized_gamma_q(double a, double x) {
    double v = 0;
    raise(mtgp_gamma_q(a, x, &v));
    return v;
}
double chi_square_pvalue(double statistic, unsigned df) {
    double v = 0;
    raise(mtgp_chi_square_pvalue(statistic, df, &v));
    return v;
}
double poisson_cdf(std::uint64_t k, double lambda) {
    double v = 0;
    raise(mtgp_poisson_cdf(k, lambda, &v));
    return v;
}
double poisson_sf(std::uint64_t k, double lambda) {
    double v = 0;
    raise(mtgp_poisson_sf(k, lambda, &v));
    return v;
}
double poisson_pmf(std::uint64_t k, double lambda) {
    double v = 0;
    raise(mtgp_poisson_pmf(k, lambda, &v));
    return v;
}
double binomial_upper_tail(std::uint64_t count, std::uint64_t n, double p) {
    double v = 0;
    raise(mtgp_binomial_upper_tail(count, n, p, &v));
    return v;
}

}  // namespace twistsieve_b200
