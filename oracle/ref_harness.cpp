// ref_harness.cpp -- extern "C" shim over the UNMODIFIED reference generator, compiled together
// with the reference's own sources (proj/src/{generator,params,word_source}.cpp) into
// oracle/_ref/libtwistsieve_ref.so by oracle/Makefile. TEST INFRASTRUCTURE ONLY: used by the
// Engine::mt parity tests and by bench.py's reference arm / cpu_baseline leg.
//
// Everything here goes through the reference's public API: ParameterizedStatus
// (proj/include/twistsieve/params.hpp:21-42), mt19937_params() (proj/src/params.cpp:63-77),
// make_word_source() + WordSource::fill() (proj/include/twistsieve/word_source.hpp:21-25,75-76),
// temper/untemper (generator.hpp:17-18).
#include <pthread.h>
#include <sched.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <span>
#include <thread>
#include <vector>

#include "twistsieve/generator.hpp"
#include "twistsieve/params.hpp"
#include "twistsieve/word_source.hpp"

using namespace twistsieve;

namespace {
ParameterizedStatus status_from(const uint32_t* f) {
    // f = {id, mexp, n, m, r, a, b, c, u, s, t, l}
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

// Words [0, n) of the stream (status, seed) through make_word_source + fill. status==NULL: MT19937.
int ref_fill(const uint32_t* status12, uint32_t seed, uint32_t* out, uint64_t n) {
    try {
        const ParameterizedStatus p = status12 ? status_from(status12) : mt19937_params();
        auto src = make_word_source(p, seed);
        src->fill(std::span<std::uint32_t>(out, n));
        return 0;
    } catch (...) {
        return -1;
    }
}

uint32_t ref_temper(uint32_t w) { return temper(w, mt19937_params()); }
uint32_t ref_untemper(uint32_t w) { return untemper(w, mt19937_params()); }

// 0 if the status validates, 1 if validate() throws std::invalid_argument (params.cpp:23-39).
int ref_validate(const uint32_t* status12) {
    try {
        status_from(status12).validate();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

// CPU throughput of the reference bulk path: `threads` independent MT19937 streams (seeds
// seed0 + t), each filling `words_per_thread` words in `fill_words`-word fill() calls into a
// private buffer, one pinned thread per core. Returns wall seconds; *checksum = XOR of all words
// (keeps the work observable).
double ref_bulk_throughput(int threads, uint64_t words_per_thread, uint32_t fill_words,
                           uint32_t seed0, uint64_t* checksum) {
    if (threads < 1) threads = 1;
    std::atomic<int> ready{0};
    std::atomic<bool> go{false};
    std::vector<uint64_t> xs(threads, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            cpu_set_t set;
            CPU_ZERO(&set);
            CPU_SET(t % CPU_SETSIZE, &set);
            pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
            auto src = make_word_source(mt19937_params(), seed0 + static_cast<uint32_t>(t));
            std::vector<uint32_t> buf(fill_words);
            ready.fetch_add(1);
            while (!go.load(std::memory_order_acquire)) {
            }
            uint64_t x = 0;
            for (uint64_t done = 0; done < words_per_thread; done += fill_words) {
                src->fill(std::span<std::uint32_t>(buf.data(), buf.size()));
                x ^= buf[0] ^ buf[buf.size() - 1];
            }
            xs[t] = x;
        });
    }
    while (ready.load() < threads) {
    }
    const auto t0 = std::chrono::steady_clock::now();
    go.store(true, std::memory_order_release);
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    uint64_t x = 0;
    for (auto v : xs) x ^= v;
    if (checksum) *checksum = x;
    return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"

extern "C" {

// Full-volume parity fixture for Engine::mt (tests/golden/make_mt_full_ck.py): MT19937 streams
// seeds seed0 + s, s < n_streams, each produced through the reference's own make_word_source +
// fill() in 2^18-word calls; after every rec_every words (a multiple of 2^18) the cumulative
// sum64 (mod 2^64) and xor32 of the stream's words so far are recorded:
// sums/xors[s * n_rec + k] cover words [0, (k + 1) * rec_every). Threads take whole streams.
// Returns wall seconds, or -1 if rec_every is not a multiple of the fill size.
double ref_cksum_stream(uint32_t seed0, uint32_t n_streams, uint64_t rec_every, uint32_t n_rec, uint64_t* sums,
                        uint32_t* xors, int threads) {
    constexpr uint64_t kFill = 1u << 18;
    if (rec_every % kFill) return -1.0;
    if (threads < 1) threads = 1;
    std::atomic<uint32_t> next{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&] {
            std::vector<uint32_t> buf(kFill);
            for (;;) {
                const uint32_t s = next.fetch_add(1);
                if (s >= n_streams) break;
                auto src = make_word_source(mt19937_params(), seed0 + s);
                uint64_t sum = 0;
                uint32_t x = 0;
                for (uint32_t k = 0; k < n_rec; ++k) {
                    for (uint64_t done = 0; done < rec_every; done += kFill) {
                        src->fill(std::span<std::uint32_t>(buf.data(), buf.size()));
                        for (uint32_t w : buf) {
                            sum += w;
                            x ^= w;
                        }
                    }
                    sums[(size_t)s * n_rec + k] = sum;
                    xors[(size_t)s * n_rec + k] = x;
                }
            }
        });
    }
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"
