// test_ref_binding.cpp -- the drop-in COMPILED AGAINST THE REFERENCE: our C++ layer built with
// -DTWISTSIEVE_B200_WITH_REFERENCE (GpuWordSource derives from twistsieve::WordSource) and
// linked with the reference's own compiled sources (oracle/_ref/libtwistsieve_ref.so), feeding
// the reference's BufferedStream (proj/include/twistsieve/word_source.hpp:80-97) and run_test
// (stat_tests.hpp:312-319) -- the sieve's campaign cell (sieve.cpp:156-158) -- with GPU words.
// Built by oracle/Makefile (target `binding`) where /root/reference exists; the binary travels
// to the GPU box in oracle/_ref/. Run by tests/test_ref_binding.py.
//
//   test_ref_binding <mtgp32_11213_curand.json> --cpu   no device: factory dispatch, the
//                                                       reference's validate(), loud failure
//   test_ref_binding <mtgp32_11213_curand.json> --gpu   + words, streams and campaign cells
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "oracle.h"
#include "twistsieve/params.hpp"
#include "twistsieve/stat_tests.hpp"
#include "twistsieve/word_source.hpp"
#include "twistsieve_b200/mtgp.hpp"

namespace ts = twistsieve;
namespace tb = twistsieve_b200;

static int g_fail = 0;
#define CHECK(c)                                                       \
    do {                                                               \
        if (!(c)) {                                                    \
            std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++g_fail;                                                  \
        }                                                              \
    } while (0)

static void test_case(const char* name, const std::function<void()>& f) {
    const int before = g_fail;
    try {
        f();
    } catch (const std::exception& e) {
        std::printf("  EXCEPTION %s\n", e.what());
        ++g_fail;
    }
    std::printf("[%s] %s\n", g_fail == before ? " ok " : "FAIL", name);
}

template <class F>
static std::string what_of(F&& f) {
    try {
        f();
    } catch (const std::invalid_argument& e) {
        return std::string("invalid_argument: ") + e.what();
    } catch (const std::runtime_error& e) {
        return std::string("runtime_error: ") + e.what();
    }
    return "no exception";
}

static std::vector<std::uint32_t> golden_first32(const std::string& raw, int set, std::uint32_t seed) {
    std::string text;
    for (char ch : raw)
        if (ch != ' ' && ch != '\n' && ch != '\r' && ch != '\t') text += ch;
    const std::string key = "\"set\":" + std::to_string(set) + ",\"seed\":" + std::to_string(seed) + ",\"u32\":[";
    const auto i = text.find(key);
    std::vector<std::uint32_t> out;
    if (i == std::string::npos) return out;
    std::stringstream ss(text.substr(i + key.size(), text.find(']', i) - i - key.size()));
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(static_cast<std::uint32_t>(std::stoul(item)));
    return out;
}

// DC-minted status of the reference's dynamic creator (tests/golden/mt_reference.json dc3217_id7)
static ts::ParameterizedStatus dc3217() {
    ts::ParameterizedStatus p;
    p.id = 7;
    p.mexp = 3217;
    p.n = 101;
    p.m = 9;
    p.r = 15;
    p.a = 3980328967u;
    p.temper_b = 882635769u;
    p.temper_c = 3305209961u;
    p.temper_u = 11;
    p.temper_s = 7;
    p.temper_t = 15;
    p.temper_l = 18;
    return p;
}

static bool same_result(const ts::TestResult& a, const ts::TestResult& b) {
    return std::memcmp(&a.statistic, &b.statistic, sizeof(double)) == 0 &&
           std::memcmp(&a.p_value, &b.p_value, sizeof(double)) == 0 && a.classification == b.classification &&
           a.degenerate == b.degenerate;
}

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    std::ifstream gf(argv[1]);
    std::stringstream gs;
    gs << gf.rdbuf();
    const std::string golden = gs.str();
    const bool gpu = std::strcmp(argv[2], "--gpu") == 0;

    test_case("factory: the reference's planted engines stay the reference's sources", [&] {
        const auto c = ts::make_constant_status(9, 0xDEADBEEFu);
        auto src = tb::make_word_source(c, 1);
        std::vector<std::uint32_t> w(16);
        src->fill(w);
        for (auto x : w) CHECK(x == 0xDEADBEEFu);
        const auto l = ts::make_lfsr16_status(3);
        auto a = tb::make_word_source(l, 77);
        auto b = ts::make_word_source(l, 77);
        std::vector<std::uint32_t> x(70000), y(70000);
        a->fill(x);
        b->fill(y);
        CHECK(x == y);
    });

    test_case("factory: an invalid Engine::mt status fails with the reference's own exception", [&] {
        auto bad = ts::mt19937_params();
        bad.m = bad.n;  // violates 1 <= m < n
        const std::string ours = what_of([&] { tb::make_word_source(bad, 5489); });
        const std::string ref = what_of([&] { bad.validate(); });
        CHECK(ours == ref);
        CHECK(ours.rfind("invalid_argument", 0) == 0);
    });

    if (!gpu) {
        test_case("no device: Engine::mt and MTGP32 construction fail loudly (no CPU fallback)", [&] {
            CHECK(what_of([&] { tb::make_word_source(ts::mt19937_params(), 5489); }).rfind("runtime_error", 0) == 0);
            const auto sets = tb::curand_mtgp32_11213();
            CHECK(what_of([&] { tb::make_word_source(sets[0], 1); }).rfind("runtime_error", 0) == 0);
        });
        std::printf("%s\n", g_fail ? "FAILED" : "ALL OK");
        return g_fail ? 1 : 0;
    }

    test_case("Engine::mt: GPU fill() == the reference's MtWordSource, any fill sizes", [&] {
        for (const auto& st : {ts::mt19937_params(), dc3217()}) {
            auto gpu_src = tb::make_word_source(st, 5489);
            ts::MtWordSource ref(st, 5489);
            std::vector<std::uint32_t> x(1 << 20), y(1 << 20);
            std::size_t done = 0;
            for (std::size_t n : {1u, 623u, 624u, 625u, 4096u, 100000u}) {
                gpu_src->fill(std::span<std::uint32_t>(x.data() + done, n));
                done += n;
            }
            gpu_src->fill(std::span<std::uint32_t>(x.data() + done, x.size() - done));
            ref.fill(y);
            CHECK(x == y);
        }
        // the reference's own goldens (proj/tests/test_generator.cpp:11-15)
        auto s = tb::make_word_source(ts::mt19937_params(), 5489);
        std::vector<std::uint32_t> w(3);
        s->fill(w);
        CHECK(w[0] == 3499211612u && w[1] == 581869302u && w[2] == 3890346734u);
    });

    test_case("BufferedStream over the GPU source == over MtWordSource (2^21 words)", [&] {
        auto gpu_src = tb::make_word_source(ts::mt19937_params(), 4357);
        ts::MtWordSource ref(ts::mt19937_params(), 4357);
        ts::BufferedStream a(*gpu_src), b(ref);
        bool same = true;
        for (int i = 0; i < (1 << 21); ++i) same &= a.next_u32() == b.next_u32();
        CHECK(same);
    });

    test_case("campaign cells: run_test(BufferedStream(GPU source)) == the reference's, desk battery", [&] {
        for (const auto& st : {ts::mt19937_params(), dc3217()}) {
            for (std::uint32_t seed : {1u, 4357u}) {
                for (const auto& spec : ts::desk_battery()) {
                    auto gpu_src = tb::make_word_source(st, seed);
                    ts::BufferedStream gs_(*gpu_src);
                    auto mine = ts::run_test(gs_, spec);
                    auto ref_src = ts::make_word_source(st, seed);
                    ts::BufferedStream rs_(*ref_src);
                    auto ref = ts::run_test(rs_, spec);
                    CHECK(same_result(mine, ref));
                    std::printf("  %s seed %u %-15s stat %.6f p %.6f (reference: stat %.6f p %.6f)\n",
                                ts::status_display_id(st).c_str(), seed, spec.test_id.c_str(), mine.statistic,
                                mine.p_value, ref.statistic, ref.p_value);
                }
            }
        }
    });

    test_case("MTGP32 (the MtgpStatus tag): BufferedStream words == cuRAND's known answers", [&] {
        const auto sets = tb::curand_mtgp32_11213();
        for (int set : {0, 7, 199}) {
            auto src = tb::make_word_source(sets[set], 1);
            ts::BufferedStream bs(*src);
            const auto want = golden_first32(golden, set, 1);
            CHECK(want.size() == 32);
            for (std::size_t i = 0; i < want.size(); ++i) CHECK(bs.next_u32() == want[i]);
        }
    });

    test_case("MTGP32 campaign cells == run_test over the oracle's words (VectorStream)", [&] {
        const auto sets = tb::curand_mtgp32_11213();
        const auto& p = sets[3];
        oracle_mtgp_params op{};
        op.mexp = p.mexp;
        op.pos = p.pos;
        op.sh1 = p.sh1;
        op.sh2 = p.sh2;
        op.mask = p.mask;
        std::memcpy(op.tbl, p.tbl, sizeof(op.tbl));
        std::memcpy(op.tmp_tbl, p.tmp_tbl, sizeof(op.tmp_tbl));
        std::memcpy(op.flt_tmp_tbl, p.flt_tmp_tbl, sizeof(op.flt_tmp_tbl));
        static oracle_mtgp g;
        oracle_mtgp_init(&g, &op, 11);
        std::vector<std::uint32_t> words(std::size_t{1} << 26);
        oracle_mtgp_fill(&g, words.data(), words.size(), 0);
        for (const auto& spec : ts::desk_battery()) {
            auto src = tb::make_word_source(p, 11);
            ts::BufferedStream bs(*src);
            auto mine = ts::run_test(bs, spec);
            ts::VectorStream vs(words);
            auto ref = ts::run_test(vs, spec);
            CHECK(same_result(mine, ref));
            std::printf("  mtgp11213-id3 seed 11 %-15s stat %.6f p %.6f\n", spec.test_id.c_str(), mine.statistic,
                        mine.p_value);
        }
    });

    std::printf("%s\n", g_fail ? "FAILED" : "ALL OK");
    return g_fail ? 1 : 0;
}
