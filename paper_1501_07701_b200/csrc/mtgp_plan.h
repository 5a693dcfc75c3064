// mtgp_plan.h -- v2 launch planner: splits a call's work into jump-ahead pieces, owns the
// per-set characteristic polynomials and jump polynomials, and launches the v2 kernels.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "mtgp_b200.h"
#include "mtgp_internal.cuh"
#include "mtgp_mt.cuh"

namespace mtgpb {

struct PlanRun {
    int kind = 0;
    bool cksum = true;
    bool ck32 = false;             // MTGP_OPT_CHECKSUM 2: kernels that have it keep a 32-bit sum
    const void* params = nullptr;  // DevParams (MTGP32) or DevMtParams (Engine::mt planner)
    uint32_t* win = nullptr;
    DevCksum* ck = nullptr;
    void* out = nullptr;
    uint64_t L = 0;
    cudaStream_t stream = nullptr;
    uint32_t max_pieces = 0;
    uint64_t min_piece_words = 0;  // 0 = auto
    uint64_t words_done = 0;       // words every stream has produced so far (few-stream splitting)
    BitmapPred pred;               // kKindBitmapRange
    EventPool* timing = nullptr;  // non-null: record event pairs around the launches
    int want_kernel = 0;          // 0 auto, 2 force v2, 3 force v3, 4 v4; Engine::mt: 5 mt_gen2, 6 mt_gen3
    int version = 0;              // kernel that ran (2, 3, 4; 5 = Engine::mt warp teams)
    // Speculative next-call jumps (MTGP_OPT_PREJUMP: 0 auto, 1 off, 2 on). epoch: the context's
    // state epoch at this call (bumped by every state change); the speculation made by a call
    // is used by the next one only if it arrives with epoch + 1 and the same plan.
    int prejump = 0;
    uint64_t epoch = 0;
    bool prejumped = false;       // result: this call's piece windows came from the speculation
    // results
    uint64_t launches = 0;        // kernels launched by this call
    uint32_t pieces = 0, warps_per_piece = 0;
};

struct PlannerImpl;

class Planner {
public:
    Planner(const std::vector<mtgp_params>& sets, int num_sms);
    // Engine::mt streams (the reference's recurrence): same pieces and jumps, warp-team MT kernel.
    // Supported when every status has the same mexp and n and n - m >= 32.
    Planner(const std::vector<mtgp_mt_params>& sets, int num_sms);
    ~Planner();
    bool v2_supported() const;
    // Engine::mt: the register-resident team kernel (version 6) takes this request shape
    bool mt3_supported(int kind, uint64_t L, const void* out) const;
    // MTGP_OPT_JUMP: 0 = auto (Karatsuba jump for N > 384), 1 = direct (flat) jump, 2 = split always
    void set_jump_mode(int mode);
    // forget per-stream algebra and cached plans (after a state restore)
    void invalidate();
    // run the per-stream annihilator analysis now, at the current window (no-op if done). An
    // analysis made at window w stays valid for w and every later window of the same streams.
    cudaError_t analyze_now(const void* params, const uint32_t* win, cudaStream_t st, std::string& err);
    cudaError_t run(PlanRun& r, std::string& err);
    cudaError_t skip(const void* params, uint32_t* win, uint64_t words, cudaStream_t st,
                     std::string& err);
    // SHA-1 of each stream's minimal (for certified sets: characteristic) polynomial, printed as
    // '0'/'1' coefficients lowest degree first; empty where none was found.
    cudaError_t charpoly_sha1(const void* params, uint32_t* win, cudaStream_t st,
                              std::vector<std::string>& out, std::string& err);
    // 1 per stream whose minimal polynomial has degree mexp and is irreducible (maximal period)
    cudaError_t certify(const void* params, uint32_t* win, cudaStream_t st, std::vector<int>& out,
                        std::string& err);

private:
    std::unique_ptr<PlannerImpl> impl_;
};

}  // namespace mtgpb
