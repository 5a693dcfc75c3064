// test_twistsieve_b200.cpp -- C++ tests of the drop-in layer, written like the reference's
// doctest suite (proj/tests/test_generator.cpp) with a tiny local CHECK harness (doctest is not
// available in this image). Built and run by tests/test_cpp_layer.py.
//
//   test_twistsieve_b200 <golden.json-path>          CPU cases (no device needed)
//   test_twistsieve_b200 <golden.json-path> --gpu    + GPU parity cases
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include <atomic>
#include <chrono>
#include <thread>

#include <cuda_runtime.h>

#include "oracle.h"
#include "twistsieve_b200/mtgp.hpp"

using namespace twistsieve_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        ++g_checks;                                                       \
        if (!(c)) {                                                       \
            std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);    \
            ++g_fail;                                                     \
        }                                                                 \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                \
    do {                                        \
        bool thrown_ = false;                   \
        try {                                   \
            (void)(expr);                       \
        } catch (const T&) {                    \
            thrown_ = true;                     \
        } catch (...) {                         \
        }                                       \
        CHECK(thrown_ && #T);                   \
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

// pull "u32": [...] of the first32 case (set, seed) out of the golden JSON without a JSON lib
static std::vector<std::uint32_t> golden_first32(const std::string& raw, int set, std::uint32_t seed) {
    std::string text;  // whitespace-free copy (the fixture is pretty-printed)
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

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::ifstream gf(argv[1]);
    std::stringstream gs;
    gs << gf.rdbuf();
    const std::string golden = gs.str();
    const bool gpu = argc > 2 && std::strcmp(argv[2], "--gpu") == 0;

    std::vector<MtgpStatus> sets;
    test_case("cuRAND MTGP32-11213 table imports and validates", [&] {
        sets = curand_mtgp32_11213();
        CHECK(sets.size() == 200);
        CHECK(sets[0].mexp == 11213 && sets[0].pos == 88 && sets[0].sh1 == 19 && sets[0].sh2 == 5);
        CHECK(sets[0].mask == 0xfff80000u);
        CHECK(sets[0].poly_sha1 == "cbb03faa650dbd1c8cc2910087257ff86f23f218");
        for (const auto& s : sets) s.validate();
        CHECK(status_display_id(sets[7]) == "mtgp11213-id7");
    });

    test_case("status invariants are enforced (cf. test_generator.cpp:105-126)", [&] {
        MtgpStatus p = sets[0];
        CHECK_THROWS_AS([&] { auto q = p; q.mexp = 11214; q.validate(); }(), std::invalid_argument);
        CHECK_THROWS_AS([&] { auto q = p; q.mask = 0; q.validate(); }(), std::invalid_argument);
        CHECK_THROWS_AS([&] { auto q = p; q.sh1 = 0; q.validate(); }(), std::invalid_argument);
        CHECK_THROWS_AS([&] { auto q = p; q.pos = 1; q.validate(); }(), std::invalid_argument);
        CHECK_THROWS_AS([&] { auto q = p; q.tbl[3] ^= 1; q.validate(); }(), std::invalid_argument);
        CHECK_THROWS_AS([&] { auto q = p; q.flt_tmp_tbl[2] ^= 1; q.validate(); }(), std::invalid_argument);
    });

    test_case("synthetic uncertified sets: deterministic, valid, all exponents", [&] {
        for (std::uint32_t mexp : {11213u, 23209u, 44497u}) {
            for (std::uint32_t k = 0; k < 8; ++k) {
                const MtgpStatus a = synthetic_status(mexp, k), b = synthetic_status(mexp, k);
                CHECK(a == b);
                a.validate();
                CHECK(!a.certified);
                CHECK(a.n() - a.pos >= (mexp == 11213 ? 256u : mexp == 23209 ? 512u : 1024u));
            }
        }
    });

    test_case("status file: JSON and key=value, round trip, path:line errors", [&] {
        const auto dir = std::filesystem::temp_directory_path() / "ts_b200_test";
        std::filesystem::create_directories(dir);
        std::vector<StatusRecord> recs = {{sets[3], 17u}, {synthetic_status(44497, 2), std::nullopt}};
        write_status_file(dir / "a.jsonl", recs);
        const auto back = read_status_file(dir / "a.jsonl");
        CHECK(back.size() == 2);
        CHECK(back[0].status == sets[3] && back[0].seed && *back[0].seed == 17u);
        CHECK(back[1].status == recs[1].status && !back[1].seed);
        std::string kv = "id=3 engine=mtgp32 mexp=11213 pos=" + std::to_string(sets[3].pos) +
                         " sh1=0x" + [&] { char b[16]; std::snprintf(b, 16, "%x", sets[3].sh1); return std::string(b); }() +
                         " sh2=" + std::to_string(sets[3].sh2) + " tbl=";
        for (int i = 0; i < 16; ++i) kv += (i ? "," : "") + std::to_string(sets[3].tbl[i]);
        kv += " tmp_tbl=";
        for (int i = 0; i < 16; ++i) kv += (i ? "," : "") + std::to_string(sets[3].tmp_tbl[i]);
        const auto r = status_from_line(kv);
        CHECK(r.status.pos == sets[3].pos && r.status.sh1 == sets[3].sh1);
        CHECK(std::memcmp(r.status.flt_tmp_tbl, sets[3].flt_tmp_tbl, 64) == 0);
        std::ofstream(dir / "bad.jsonl") << "# comment\n\n" << status_to_json_line(recs[0]) << "\nid=1 bogus=3\n";
        bool located = false;
        try {
            read_status_file(dir / "bad.jsonl");
        } catch (const std::runtime_error& e) {
            located = std::string(e.what()).find("bad.jsonl:4: unknown status field: bogus") != std::string::npos;
        }
        CHECK(located);
        // a file written by the Python tooling parses identically
        if (argc > 3) {
            const auto py = read_status_file(argv[3]);
            CHECK(py.size() >= 2 && py[0].status == sets[0] && py[1].status == synthetic_status(23209, 1));
        }
    });

    test_case("golden fixture parses (cuRAND first32 cases)", [&] {
        CHECK(golden_first32(golden, 0, 1).size() == 32);
        CHECK(golden_first32(golden, 0, 1)[0] == 360948779u);
        CHECK(golden_first32(golden, 199, 0xFFFFFFFFu).size() == 32);
    });

    test_case("Engine::mt status invariants (test_generator.cpp:105-126)", [&] {
        MtStatus p = mt19937_status();
        p.validate();
        CHECK_THROWS_AS([&] { auto q = p; q.r = 30; q.validate(); }(), std::invalid_argument);
        CHECK_THROWS_AS([&] { auto q = p; q.id = 7; q.validate(); }(), std::invalid_argument);
        CHECK_THROWS_AS([&] { auto q = p; q.m = q.n; q.validate(); }(), std::invalid_argument);
        CHECK_THROWS_AS([&] { auto q = p; q.mexp = 19936; q.r = 32 * q.n - 19936; q.validate(); }(),
                        std::invalid_argument);
    });

    test_case("splitmix64 / derive_seed (word_source.cpp:18-27)", [&] {
        CHECK(splitmix64(0) == 0xE220A8397B1DCDAFull);
        CHECK(derive_seed(10, 3) == static_cast<std::uint32_t>(splitmix64(13)));
    });

    if (!gpu) {
        test_case("no device: construction fails loudly (no CPU fallback)", [&] {
            CHECK_THROWS_AS(GpuWordSource(sets[0], 1), std::runtime_error);
        });
    } else {
        test_case("GpuWordSource matches the independently sourced cuRAND known answers", [&] {
            for (int set : {0, 1, 7, 199}) {
                for (std::uint32_t seed : {1u, 0u, 5489u, 0xFFFFFFFFu}) {
                    const auto want = golden_first32(golden, set, seed);
                    CHECK(want.size() == 32);
                    GpuWordSource src(sets[set], seed);
                    std::vector<std::uint32_t> got(32);
                    src.fill(got);
                    CHECK(got == want);
                }
            }
        });
        test_case("fill is chunk-size independent; next_u32 / next_f64_01 continue the stream", [&] {
            GpuWordSource a(sets[5], 42, OutputKind::u32, 0, 4096);
            GpuWordSource b(sets[5], 42, OutputKind::u32, 0, 1 << 16);
            std::vector<std::uint32_t> x(100000), y(100000);
            std::size_t done = 0;
            for (std::size_t n : {1u, 7u, 4095u, 4096u, 4097u, 30000u})
                a.fill(std::span<std::uint32_t>(x.data() + done, n)), done += n;
            a.fill(std::span<std::uint32_t>(x.data() + done, x.size() - done));
            b.fill(y);
            CHECK(x == y);
            const std::uint32_t w = a.next_u32();
            GpuWordSource c(sets[5], 42);
            std::vector<std::uint32_t> z(100001);
            c.fill(z);
            CHECK(w == z[100000]);
            const double u = b.next_f64_01();
            CHECK(u == static_cast<double>(z[100000]) * (1.0 / 4294967296.0));
            CHECK(a.position() == 100001);
        });
        test_case("float kinds through the WordSource interface", [&] {
            GpuWordSource f12(sets[0], 1, OutputKind::f32_12), f01(sets[0], 1, OutputKind::f32_01oc);
            std::vector<std::uint32_t> a(4), b(4);
            f12.fill(a);
            f01.fill(b);
            CHECK(a[0] == 0x3f8ac1d2u && a[1] == 0x3fa3ca34u && a[2] == 0x3fc4f5e7u && a[3] == 0x3fc21b32u);
            CHECK(b[0] == 0x3f6a7c5cu && b[1] == 0x3f386b98u && b[2] == 0x3eec2864u && b[3] == 0x3ef79338u);
        });
        test_case("Engine::mt on the GPU matches std::mt19937 (the reference's own oracle, test_generator.cpp:11-25)", [&] {
            GpuWordSource gen(mt19937_status(), 5489);
            CHECK(gen.next_u32() == 3499211612u);
            CHECK(gen.next_u32() == 581869302u);
            CHECK(gen.next_u32() == 3890346734u);
            auto mine = make_word_source(mt19937_status(), 5489);
            std::mt19937 oracle(5489);
            std::vector<std::uint32_t> w(100000);
            mine->fill(w);
            bool eq = true;
            for (auto v : w) eq = eq && v == oracle();
            CHECK(eq);
            // identical seeds give identical outputs (test_generator.cpp:36-40)
            GpuWordSource a(mt19937_status(), 12345), b(mt19937_status(), 12345);
            std::vector<std::uint32_t> x(1000000), y(1000000);
            a.fill(x);
            b.fill(y);
            CHECK(x == y);
        });
        test_case("make_word_source factory + StreamBatch checksums + skip", [&] {
            auto src = make_word_source(sets[0], 1);
            std::vector<std::uint32_t> w(1 << 20);
            src->fill(w);
            std::uint64_t sum = 0;
            std::uint32_t x = 0;
            for (auto v : w) sum += v, x ^= v;
            CHECK(sum == 2251211974485391ull && x == 0x87db016du && w.back() == 1034305667u);
            StreamBatch batch({sets[0], sets[1]}, {1, 1});
            std::vector<std::uint32_t> out(2 * 1000);
            batch.generate_host(OutputKind::u32, out.data(), 1000);
            batch.skip(1u << 20);
            CHECK(batch.position(1) == 1000 + (1u << 20));
            const auto ck = batch.checksums();
            CHECK(ck[0].words == 1000);
        });
        test_case("MultiGpuBatch: set ranges per device, checksums gathered == one context's", [&] {
            std::vector<std::uint32_t> seeds(sets.size());
            for (std::size_t i = 0; i < seeds.size(); ++i) seeds[i] = 1000 + static_cast<std::uint32_t>(i);
            StreamBatch one(sets, seeds);
            const std::uint64_t L = 1 << 16;
            void* d = nullptr;
            CHECK(mtgp_host_alloc(sets.size() * L * 4, &d) == MTGP_OK);  // host output for the reference batch
            one.generate_host(OutputKind::u32, d, L);
            const auto want = one.checksums();
            mtgp_host_free(d);
            for (auto mode : {MultiGpuBatch::Gather::nccl, MultiGpuBatch::Gather::host}) {
                const std::vector<int> devs = mode == MultiGpuBatch::Gather::nccl ? std::vector<int>{0}
                                                                                   : std::vector<int>{0, 0, 0};
                MultiGpuBatch mb(sets, seeds, devs, mode);
                CHECK(mb.nccl() == (mode == MultiGpuBatch::Gather::nccl));
                std::vector<void*> outs;
                for (std::uint32_t r = 0; r < mb.devices(); ++r) {
                    void* o = nullptr;
                    CHECK(cudaMalloc(&o, mb.range(r).second * L * 4) == cudaSuccess);
                    outs.push_back(o);
                }
                mb.generate_device(OutputKind::u32, outs, L);
                const auto got = mb.checksums();
                CHECK(got.size() == want.size());
                bool same = true;
                for (std::size_t i = 0; i < got.size(); ++i)
                    same &= got[i].sum64 == want[i].sum64 && got[i].xor32 == want[i].xor32 && got[i].words == L;
                CHECK(same);
                for (void* o : outs) cudaFree(o);
            }
        });

        // The reference's concurrency model: one generator per worker thread, never shared
        // (the std::thread pool of sieve.cpp:170-177). T host threads each own a
        // make_word_source() stream on the same GPU -- half MTGP32 (certified sets), half
        // Engine::mt (MT19937) -- and read it with the reference's 4096-word BufferedStream
        // fills. Every word is then checked against the oracle (oracle/*.c, test infrastructure).
        for (unsigned T : {8u, 16u}) {
            const std::string name = "threading model: " + std::to_string(T) +
                                     " host threads, one make_word_source() each, 4096-word fills";
            test_case(name.c_str(), [&] {
                const std::size_t W = std::size_t{1} << 24;
                std::vector<std::vector<std::uint32_t>> got(T, std::vector<std::uint32_t>(W));
                std::vector<std::unique_ptr<WordSource>> srcs(T);
                for (unsigned t = 0; t < T; ++t)
                    srcs[t] = (t % 2 == 0) ? make_word_source(sets[t], 100 + t) : make_word_source(mt19937_status(), 5489 + t);
                std::atomic<int> errors{0};
                const auto t0 = std::chrono::steady_clock::now();
                std::vector<std::thread> pool;
                for (unsigned t = 0; t < T; ++t)
                    pool.emplace_back([&, t] {
                        try {
                            for (std::size_t i = 0; i < W; i += 4096)
                                srcs[t]->fill(std::span<std::uint32_t>(got[t].data() + i, 4096));
                        } catch (...) {
                            ++errors;
                        }
                    });
                for (auto& th : pool) th.join();
                const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                CHECK(errors == 0);
                std::atomic<int> bad{0};
                std::vector<std::thread> check;
                for (unsigned t = 0; t < T; ++t)
                    check.emplace_back([&, t] {
                        std::vector<std::uint32_t> ref(W);
                        if (t % 2 == 0) {
                            oracle_mtgp_params op{};
                            op.mexp = sets[t].mexp;
                            op.pos = sets[t].pos;
                            op.sh1 = sets[t].sh1;
                            op.sh2 = sets[t].sh2;
                            op.mask = sets[t].mask;
                            std::memcpy(op.tbl, sets[t].tbl, 64);
                            std::memcpy(op.tmp_tbl, sets[t].tmp_tbl, 64);
                            std::memcpy(op.flt_tmp_tbl, sets[t].flt_tmp_tbl, 64);
                            auto g = std::make_unique<oracle_mtgp>();
                            oracle_mtgp_init(g.get(), &op, 100 + t);
                            oracle_mtgp_fill(g.get(), ref.data(), W, 0);
                        } else {
                            oracle_mt_params mp;
                            oracle_mt19937_params(&mp);
                            auto g = std::make_unique<oracle_mt>();
                            oracle_mt_init(g.get(), &mp, 5489 + t);
                            oracle_mt_fill(g.get(), ref.data(), W);
                        }
                        if (ref != got[t]) ++bad;
                    });
                for (auto& th : check) th.join();
                CHECK(bad == 0);
                std::printf("  THREADS %u: %zu words per thread in 4096-word fills, %.3f s wall, %.3f G words/s "
                            "aggregate, every word == oracle: %s\n",
                            T, W, secs, T * (double)W / secs / 1e9, bad == 0 ? "yes" : "NO");
            });
        }
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
