// Drop-in consumer throughput: twistsieve_b200::GpuWordSource::fill in the reference's fill sizes
// (BufferedStream 4096 words, word_source.hpp:94; the CLI's 1024, cli.cpp:373), one stream, after
// the stream has produced 2^25 words (long-lived), MTGP32-11213 and MT19937. Prints JSON lines.
//   g++ -std=c++20 -O2 -Iinclude tools/word_source_bench.cpp -Lpaper_1501_07701_b200 \
//       -ltwistsieve_b200 -lmtgp_b200 -Wl,-rpath,$PWD/paper_1501_07701_b200 -o /tmp/wsb && /tmp/wsb
#include <chrono>
#include <cstdio>
#include <vector>

#include "twistsieve_b200/mtgp.hpp"

using namespace twistsieve_b200;

template <class Status>
static void run(const char* name, const Status& st, std::size_t span, std::size_t chunk) {
    GpuWordSource src(st, 1u, OutputKind::u32, 0, chunk);
    std::vector<std::uint32_t> buf(span);
    for (std::uint64_t done = 0; done < (1ull << 25); done += span) src.fill(buf);
    const std::uint64_t total = 1ull << 28;
    const auto t0 = std::chrono::steady_clock::now();
    std::uint32_t x = 0;
    for (std::uint64_t done = 0; done < total; done += span) {
        src.fill(buf);
        x ^= buf[0];
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("{\"engine\": \"%s\", \"fill_words\": %zu, \"chunk_words\": %zu, \"words\": %llu, \"Gwords_s\": %.4f, "
                "\"check\": %u}\n",
                name, span, chunk, (unsigned long long)total, total / s / 1e9, x);
}

int main() {
    const MtgpStatus mtgp = curand_mtgp32_11213()[0];
    const MtStatus mt = mt19937_status();
    for (std::size_t chunk : {std::size_t{1} << 17, std::size_t{1} << 18, std::size_t{1} << 19, std::size_t{1} << 20,
                              std::size_t{1} << 22}) {
        for (std::size_t span : {std::size_t{1024}, std::size_t{4096}}) {
            run("mtgp32-11213", mtgp, span, chunk);
            run("mt19937", mt, span, chunk);
        }
    }
    return 0;
}
