// mtgp_multi.h -- host-side pieces of the multi-GPU batch (no CUDA in this header): the
// contiguous balanced set-ID partition and the padded all-gather of uneven per-rank checksum
// arrays. mtgp_multi.cu uses them with NCCL; tests/cpp/test_multi.cpp with a fake communicator.
//
// The reference's only parallelism is its worker pool over independent statuses
// (proj/src/sieve.cpp:170-177). Here the unit is a device: parameter-set IDs
// [first, first + count) go to device r (shard.status_range), each device
// generates its streams with no collective on the hot path, and the per-stream checksums
// {sum64, words, xor32} are all-gathered once at the end (north_star (5)).
#pragma once

#include <cstdint>
#include <cstring>
#include <vector>

#include "mtgp_b200.h"

namespace mtgpb {

// Set IDs of rank r when n sets are split over w ranks: contiguous, the first n % w ranks one
// more (the same split as paper_1501_07701_b200.shard.status_range).
inline void shard_range(uint32_t n, uint32_t w, uint32_t r, uint32_t* first, uint32_t* count) {
    const uint32_t base = n / w, extra = n % w;
    *first = r * base + (r < extra ? r : extra);
    *count = base + (r < extra ? 1u : 0u);
}

// An all-gather of equal-size byte blocks over `world` ranks: block r comes from rank r, and
// afterwards every rank holds all blocks in rank order. all_gather returns rank 0's result.
struct GatherComm {
    virtual ~GatherComm() = default;
    virtual uint32_t world() const = 0;
    virtual const char* name() const = 0;
    // returns 0, or an MTGP_E* code (message via set_error)
    virtual int all_gather(const std::vector<std::vector<uint8_t>>& send, std::vector<uint8_t>& recv0) = 0;
};

// Uneven per-rank checksum arrays through an equal-block all-gather: pad every rank's block
// to the largest count (zero records), gather, then trim each block to its own count.
inline int gather_checksums(GatherComm& comm, const std::vector<std::vector<mtgp_cksum>>& per_rank,
                            std::vector<mtgp_cksum>& out) {
    const uint32_t w = comm.world();
    if (per_rank.size() != w) return MTGP_EINVAL;
    size_t maxc = 0;
    for (const auto& v : per_rank) maxc = v.size() > maxc ? v.size() : maxc;
    const size_t block = maxc * sizeof(mtgp_cksum);
    std::vector<std::vector<uint8_t>> send(w, std::vector<uint8_t>(block, 0));
    for (uint32_t r = 0; r < w; ++r)
        if (!per_rank[r].empty()) std::memcpy(send[r].data(), per_rank[r].data(), per_rank[r].size() * sizeof(mtgp_cksum));
    std::vector<uint8_t> recv;
    if (block) {
        const int rc = comm.all_gather(send, recv);
        if (rc) return rc;
        if (recv.size() != block * w) return MTGP_ESTATE;
    }
    out.clear();
    for (uint32_t r = 0; r < w; ++r) {
        const mtgp_cksum* b = reinterpret_cast<const mtgp_cksum*>(recv.data() + r * block);
        out.insert(out.end(), b, b + per_rank[r].size());
    }
    return MTGP_OK;
}

}  // namespace mtgpb
