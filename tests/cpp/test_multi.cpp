// test_multi.cpp -- host logic of the multi-GPU batch (paper_1501_07701_b200/csrc/mtgp_multi.h),
// no device: the contiguous balanced partition of set IDs and the padded checksum all-gather,
// run through a fake communicator that moves the blocks around a ring the way an all-gather
// algorithm does (rank r's receive buffer is filled block by block from its left neighbour).
// Built and run by tests/test_multi_gpu_cpu.py.
#include <cstdio>
#include <vector>

#include "mtgp_multi.h"

static int g_fail = 0;
#define CHECK(c)                                                       \
    do {                                                               \
        if (!(c)) {                                                    \
            std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++g_fail;                                                  \
        }                                                              \
    } while (0)

struct RingComm final : mtgpb::GatherComm {
    uint32_t w;
    explicit RingComm(uint32_t world) : w(world) {}
    uint32_t world() const override { return w; }
    const char* name() const override { return "ring"; }
    int all_gather(const std::vector<std::vector<uint8_t>>& send, std::vector<uint8_t>& recv0) override {
        const size_t b = send[0].size();
        std::vector<std::vector<uint8_t>> recv(w, std::vector<uint8_t>(b * w));
        for (uint32_t r = 0; r < w; ++r) std::copy(send[r].begin(), send[r].end(), recv[r].begin() + r * b);
        for (uint32_t step = 1; step < w; ++step)  // rank r receives block (r - step) from rank r - 1
            for (uint32_t r = 0; r < w; ++r) {
                const uint32_t left = (r + w - 1) % w, blk = (r + w - step) % w;
                std::copy(recv[left].begin() + blk * b, recv[left].begin() + (blk + 1) * b, recv[r].begin() + blk * b);
            }
        for (uint32_t r = 1; r < w; ++r) CHECK(recv[r] == recv[0]);  // every rank holds everything
        recv0 = recv[0];
        return 0;
    }
};

int main() {
    // partition: contiguous, balanced, covers [0, n) exactly, first n % w ranks one more
    for (uint32_t n : {1u, 5u, 200u, 1024u, 1600u, 1601u})
        for (uint32_t w = 1; w <= 9 && w <= n; ++w) {
            uint32_t next = 0, lo = ~0u, hi = 0;
            for (uint32_t r = 0; r < w; ++r) {
                uint32_t f, c;
                mtgpb::shard_range(n, w, r, &f, &c);
                CHECK(f == next);
                next = f + c;
                lo = c < lo ? c : lo;
                hi = c > hi ? c : hi;
                CHECK(c == n / w + (r < n % w ? 1u : 0u));
            }
            CHECK(next == n && hi - lo <= 1);
        }
    // gather: uneven per-rank counts come back in global set order, pads dropped
    for (uint32_t n : {5u, 200u, 1024u})
        for (uint32_t w : {1u, 2u, 3u, 8u}) {
            std::vector<std::vector<mtgp_cksum>> per(w);
            for (uint32_t r = 0; r < w; ++r) {
                uint32_t f, c;
                mtgpb::shard_range(n, w, r, &f, &c);
                for (uint32_t s = f; s < f + c; ++s)
                    per[r].push_back(mtgp_cksum{0x100000000ull * s + 7, 1000 + s, 0xABC00000u ^ s, 0});
            }
            RingComm comm(w);
            std::vector<mtgp_cksum> all;
            CHECK(mtgpb::gather_checksums(comm, per, all) == 0);
            CHECK(all.size() == n);
            for (uint32_t s = 0; s < all.size(); ++s)
                CHECK(all[s].sum64 == 0x100000000ull * s + 7 && all[s].words == 1000 + s && all[s].xor32 == (0xABC00000u ^ s));
        }
    std::printf("%s\n", g_fail ? "FAILED" : "ALL OK");
    return g_fail ? 1 : 0;
}
