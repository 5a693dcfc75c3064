// The reference's concurrency model at steady state: T host threads, each owning one
// make_word_source() stream (MTGP32-11213 certified sets) on one GPU and reading it through the
// reference's 4096-word fills (BufferedStream, word_source.hpp:94). Each stream first consumes
// 2^25 words (context, plan and jump-ahead analysis warm), then every thread reads `words` more
// while the wall clock runs. Prints one JSON line per T.
//   g++ -std=c++20 -O2 -Iinclude tools/threads_bench.cpp -Lpaper_1501_07701_b200 -ltwistsieve_b200 \
//       -lmtgp_b200 -lpthread -Wl,-rpath,'$ORIGIN/../paper_1501_07701_b200' -o tools/threads_bench
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <thread>
#include <vector>

#include "twistsieve_b200/mtgp.hpp"

using namespace twistsieve_b200;

int main(int argc, char** argv) {
    const std::size_t words = argc > 1 ? std::strtoull(argv[1], nullptr, 0) : (std::size_t{1} << 27);
    const auto sets = curand_mtgp32_11213();
    for (unsigned T : {1u, 2u, 4u, 8u, 16u}) {
        std::vector<std::unique_ptr<WordSource>> src(T);
        for (unsigned t = 0; t < T; ++t) src[t] = make_word_source(sets[t], 1000 + t);
        std::atomic<unsigned> ready{0};
        std::atomic<bool> go{false};
        std::vector<std::uint32_t> sink(T, 0);
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                std::vector<std::uint32_t> buf(4096);
                for (std::size_t i = 0; i < (std::size_t{1} << 25); i += buf.size()) src[t]->fill(buf);
                ready.fetch_add(1);
                while (!go.load()) {
                }
                std::uint32_t x = 0;
                for (std::size_t i = 0; i < words; i += buf.size()) {
                    src[t]->fill(buf);
                    x ^= buf[0];
                }
                sink[t] = x;
            });
        while (ready.load() < T) {
        }
        const auto t0 = std::chrono::steady_clock::now();
        go.store(true);
        for (auto& th : pool) th.join();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::uint32_t x = 0;
        for (auto v : sink) x ^= v;
        std::printf("{\"threads\": %u, \"words_per_thread\": %zu, \"fill_words\": 4096, \"seconds\": %.4f, "
                    "\"aggregate_Gwords_s\": %.3f, \"per_thread_Gwords_s\": %.3f, \"check\": %u}\n",
                    T, words, s, T * (double)words / s / 1e9, words / s / 1e9, x);
        std::fflush(stdout);
    }
    return 0;
}
