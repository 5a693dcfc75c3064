// mtgp_internal.cuh -- shared definitions of the B200 MTGP32 generator (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "mtgp_b200.h"

namespace mtgpb {

// Device copy of one parameter set. Tables are stored so a warp can hold them in registers
// (lane l keeps tbl[l & 15], tmp[l & 15]) and look them up with one shfl.
struct alignas(16) DevParams {
    uint32_t pos, sh1, sh2, mask;
    // Multipliers that move shifts onto the FMA pipe: x << sh1 == x * mul1,
    // x >> sh2 == umulhi(x, mulhi2), x >> 16 == umulhi(x, m16), x >> 8 == umulhi(x, m24),
    // x >> 9 == umulhi(x, m23). Loaded from memory so the compiler cannot fold them back to SHF.
    uint32_t mul1, mulhi2, m16, m24, m23, one, pad0, pad1;
    uint32_t tbl[16];
    uint32_t tmp[16];
};

// Internal output kinds (not in the ABI) for the device-side stat tests: instead of the words,
// one predicate bit per word into a per-stream bitmap (stride ceil(L / 32) words; bit j of the
// call's words at word j / 32, bit j % 32). Only the register-resident team kernels produce
// them (gen3: MTGP32-11213; mt_gen3: Engine::mt n = 624); the stat passes use words elsewhere.
constexpr int kKindBitmapBit0 = 16;   // word & 1 (random walk)
constexpr int kKindBitmapRange = 17;  // lo <= (word & mask) < hi (gap-test hits)
struct BitmapPred {
    uint32_t mask = 0xFFFFFFFFu;
    uint32_t lo = 0;       // hit: ((word & mask) - lo) mod 2^32 <= span_m1, i.e.
    uint32_t span_m1 = 0;  // lo <= (word & mask) < lo + span_m1 + 1 <= 2^32
};

struct DevCksum {
    unsigned long long sum64;
    unsigned long long words;
    unsigned int xor32;
    unsigned int pad;
};

// One jump-ahead piece of the v2 kernel: `len` words of stream `set` starting `offset` words
// after the set's position at the start of the call. jump_idx < 0: offset == 0, no jump.
struct Piece {
    uint32_t set;
    int32_t jump_idx;
    uint64_t offset;
    uint64_t len;
};

// A team (one or more warps sharing a ring) processes pieces [first, first+count).
struct TeamWork {
    uint32_t first;
    uint32_t count;
};

// Non-blocking kernel timing: event pairs recorded around launches, resolved on demand.
struct EventPool {
    std::vector<cudaEvent_t> ev;
    size_t used = 0;
    std::vector<std::pair<size_t, size_t>> gen, jump;
    cudaEvent_t record(cudaStream_t st, size_t* idx) {
        if (used == ev.size()) {
            cudaEvent_t e = nullptr;
            cudaEventCreate(&e);
            ev.push_back(e);
        }
        *idx = used;
        cudaEventRecord(ev[used], st);
        return ev[used++];
    }
    // Sums elapsed milliseconds of all recorded pairs, then recycles the events.
    cudaError_t resolve(double* gen_ms, uint64_t* gen_n, double* jump_ms, uint64_t* jump_n) {
        if (used) {
            cudaError_t e = cudaEventSynchronize(ev[used - 1]);
            if (e != cudaSuccess) return e;
        }
        for (auto& p : gen) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[p.first], ev[p.second]);
            *gen_ms += ms;
            ++*gen_n;
        }
        for (auto& p : jump) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[p.first], ev[p.second]);
            *jump_ms += ms;
            ++*jump_n;
        }
        gen.clear();
        jump.clear();
        used = 0;
        return cudaSuccess;
    }
    ~EventPool() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};

inline uint32_t state_words(uint32_t mexp) { return mexp / 32 + 1; }

inline uint32_t next_pow2(uint32_t v) {
    uint32_t r = 1;
    while (r < v) r <<= 1;
    return r;
}

// ---- kernel launchers (mtgp_kernels.cu) ----
cudaError_t launch_v1(int kind, bool cksum, const DevParams* params, uint32_t* win, uint32_t n_sets,
                      uint32_t N, void* out, uint64_t L, DevCksum* ck, cudaStream_t st);

}  // namespace mtgpb
