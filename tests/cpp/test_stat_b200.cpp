// test_stat_b200.cpp -- C++ tests of the stat-test layer (include/twistsieve_b200/stat_tests.hpp),
// written like the reference's proj/tests/test_stats.cpp with a tiny local CHECK harness (doctest
// is not available). Built and run by tests/test_cpp_layer.py, which flattens
// tests/golden/stat_reference.json (the reference's own results) into <cases.txt>:
//
//   math <fn> <a-hex> <b-hex> <k> <n> <value-hex>
//   case <test_id> <n> <r> <alpha-hex> <beta-hex> <s> <L> <d> <l> <t> <set> <seed> <stat-hex> <p-hex> <class> <degenerate>
//   cell <test_id> <seed> <stat-hex> <p-hex> <class>
//
//   test_stat_b200 <cases.txt> <curand header> [--gpu]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "twistsieve_b200/stat_tests.hpp"

using namespace twistsieve_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        ++g_checks;                                                       \
        if (!(c)) {                                                       \
            ++g_fail;                                                     \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);      \
        }                                                                 \
    } while (0)

template <class F>
static std::string throws_invalid(F&& f) {
    try {
        f();
    } catch (const std::invalid_argument& e) {
        return e.what();
    } catch (...) {
        return "<other exception>";
    }
    return "<no exception>";
}

static double hexd(const std::string& s) { return std::strtod(s.c_str(), nullptr); }

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const bool gpu = argc > 3 && std::strcmp(argv[3], "--gpu") == 0;
    std::ifstream in(argv[1]);
    std::vector<std::vector<std::string>> math, cases, cells;
    for (std::string line; std::getline(in, line);) {
        std::istringstream ss(line);
        std::vector<std::string> f;
        for (std::string w; ss >> w;) f.push_back(w);
        if (f.empty()) continue;
        if (f[0] == "math") math.push_back(f);
        if (f[0] == "case") cases.push_back(f);
        if (f[0] == "cell") cells.push_back(f);
    }
    CHECK(!math.empty() && !cases.empty() && !cells.empty());

    // ---- specs (stat_tests.cpp:52-104) ----
    CHECK(desk_battery().size() == 4);
    CHECK(named_spec("opso") == desk_opso_spec());
    CHECK(named_spec("hamming").describe() == "hamming_indep(n=100000,r=25,s=5,L=1200,d=0)");
    CHECK(desk_gap_spec().describe() == "gap(n=1000000,r=25,alpha=0,beta=0.03125)");
    CHECK(desk_opso_spec().describe() == "collision_over(n=32768,r=0,s=11,t=22)");
    CHECK(throws_invalid([] { named_spec("birthday"); }) == "unknown test name: birthday");
    for (const auto& s : desk_battery()) s.validate();
    {
        TestSpec s = desk_walk_spec();
        s.n = 10;
        CHECK(throws_invalid([&] { s.validate(); }) == "sample too small");
        s = desk_hamming_spec();
        s.d = 1;
        CHECK(throws_invalid([&] { s.validate(); }) == "only d = 0 is supported");
        s = desk_opso_spec();
        s.n = 10;
        CHECK(throws_invalid([&] { s.validate(); }) == "spec out of sparse regime");
        s = desk_gap_spec();
        s.beta = 0.0;
        CHECK(throws_invalid([&] { s.validate(); }) == "gap test requires 0 <= alpha < beta <= 1");
        s.test_id = "nope";
        CHECK(throws_invalid([&] { s.validate(); }) == "unknown test id: nope");
    }

    // ---- classify (classify.cpp:18-24, test_stats.cpp boundary cases) ----
    CHECK(classify_pvalue(0.001) == PValueClass::correct);
    CHECK(classify_pvalue(0.999) == PValueClass::correct);
    CHECK(classify_pvalue(1e-10) == PValueClass::suspect);
    CHECK(classify_pvalue(1.0 - 1e-10) == PValueClass::suspect);
    CHECK(classify_pvalue(0.0) == PValueClass::disastrous);
    CHECK(throws_invalid([] { classify_pvalue(1.5); }) == "p-value outside [0, 1]");
    CHECK(std::string(to_string(PValueClass::suspect)) == "suspect");

    // ---- numerics, bit-exact against the reference's values ----
    int nm = 0;
    for (const auto& f : math) {
        const std::string& fn = f[1];
        const double a = hexd(f[2]), b = hexd(f[3]), want = hexd(f[6]);
        const auto k = std::strtoull(f[4].c_str(), nullptr, 10), n = std::strtoull(f[5].c_str(), nullptr, 10);
        double got = -1;
        if (fn == "ln_gamma") got = ln_gamma(a);
        else if (fn == "gamma_p") got = regularized_gamma_p(a, b);
        else if (fn == "gamma_q") got = regularized_gamma_q(a, b);
        else if (fn == "chi_square_pvalue") got = chi_square_pvalue(a, static_cast<unsigned>(k));
        else if (fn == "poisson_cdf") got = poisson_cdf(k, a);
        else if (fn == "poisson_sf") got = poisson_sf(k, a);
        else if (fn == "poisson_pmf") got = poisson_pmf(k, a);
        else if (fn == "binomial_upper_tail") got = binomial_upper_tail(k, n, a);
        else continue;
        ++nm;
        if (got != want) std::printf("math %s(%s,%s,%s,%s): %a != %a\n", fn.c_str(), f[2].c_str(), f[3].c_str(), f[4].c_str(), f[5].c_str(), got, want);
        CHECK(got == want);
    }
    CHECK(nm > 50);
    CHECK(throws_invalid([] { chi_square_pvalue(-1.0, 3); }) == "negative chi-square statistic");

    if (gpu) {
        // ---- device-side run_test over MTGP32 streams == the reference template over the same words
        const auto sets = curand_mtgp32_11213(argv[2]);
        for (const auto& f : cases) {
            TestSpec s;
            s.test_id = f[1];
            s.n = std::strtoull(f[2].c_str(), nullptr, 10);
            s.r = std::atoi(f[3].c_str());
            s.alpha = hexd(f[4]);
            s.beta = hexd(f[5]);
            s.s = std::atoi(f[6].c_str());
            s.L = std::atoi(f[7].c_str());
            s.d = std::atoi(f[8].c_str());
            s.l = std::atoi(f[9].c_str());
            s.t = std::atoi(f[10].c_str());
            const int set = std::atoi(f[11].c_str());
            const auto seed = static_cast<std::uint32_t>(std::strtoul(f[12].c_str(), nullptr, 10));
            StreamBatch b(std::vector<MtgpStatus>{sets[set]}, {seed});
            const auto r = run_test(b, s);
            CHECK(r.size() == 1 && !r[0].is_error());
            CHECK(r[0].result.statistic == hexd(f[13]));
            CHECK(r[0].result.p_value == hexd(f[14]));
            CHECK(static_cast<int>(r[0].result.classification) == std::atoi(f[15].c_str()));
            CHECK(static_cast<int>(r[0].result.degenerate) == std::atoi(f[16].c_str()));
        }
        // ---- GPU campaign grid == the reference's own campaign cells (MT19937, desk battery)
        std::vector<std::uint32_t> seeds;
        for (const auto& f : cells) {
            const auto seed = static_cast<std::uint32_t>(std::strtoul(f[2].c_str(), nullptr, 10));
            if (seeds.empty() || seeds.back() != seed) seeds.push_back(seed);
        }
        const auto rows = run_grid(std::vector<MtStatus>{mt19937_status()}, seeds, desk_battery());
        CHECK(rows.size() == cells.size());
        for (std::size_t i = 0; i < rows.size() && i < cells.size(); ++i) {
            CHECK(rows[i].test_id == cells[i][1]);
            CHECK(rows[i].status_id == "m19937-id45279");
            CHECK(rows[i].statistic == hexd(cells[i][3]));
            CHECK(rows[i].p_value == hexd(cells[i][4]));
            CHECK(static_cast<int>(rows[i].classification) == std::atoi(cells[i][5].c_str()));
        }
        // verify_digest on the GPU with the reference's MT19937 preset digest (params.cpp:75)
        CHECK(verify_digest(mt19937_status(), "736dbad14b19609ef909097e1b440834727ed02c"));
        CHECK(!verify_digest(mt19937_status(), "0000000000000000000000000000000000000000"));
        {
            StreamBatch b(std::vector<MtgpStatus>{sets[0], sets[1]}, {1u, 2u});
            const auto c = b.certify();
            CHECK(c.size() == 2 && c[0] && c[1]);
        }
        // a spec error becomes an error row in every cell, the rest of the grid still runs
        TestSpec bad = desk_walk_spec();
        bad.n = 10;
        const auto rows2 = run_grid(std::vector<MtStatus>{mt19937_status()}, {1, 2}, {bad, desk_opso_spec()});
        CHECK(rows2.size() == 4 && rows2[0].error == "sample too small" && !rows2[1].is_error());
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
