// mtgp_ctx.h -- the context object behind the C-ABI handle (private to libmtgp_b200.so), shared
// by the API translation units (mtgp_capi.cu, mtgp_stat.cu).
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "mtgp_b200.h"
#include "mtgp_internal.cuh"
#include "mtgp_mt.cuh"
#include "mtgp_plan.h"

using mtgpb::BitmapPred;
using mtgpb::DevCksum;
using mtgpb::DevMtParams;
using mtgpb::DevParams;
using mtgpb::EventPool;
using mtgpb::Planner;

struct mtgp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    bool own_stream = false;
    uint32_t n_sets = 0, N = 0, mexp = 0;
    int engine = 0;  // 0 = MTGP32, 1 = Engine::mt (the reference's classic recurrence)
    std::vector<mtgp_params> sets;
    std::vector<mtgp_mt_params> mt_sets;
    std::vector<uint64_t> position;
    DevMtParams* d_mt = nullptr;

    DevParams* d_params = nullptr;
    uint32_t* d_win = nullptr;
    DevCksum* d_ck = nullptr;

    // options
    bool cksum = true;
    bool ck32 = false;        // MTGP_OPT_CHECKSUM 2 (32-bit sums where the kernel has them)
    bool ck_sum_mod32 = false;  // a mode-2 call ran since the last reset: sum64 is valid mod 2^32
    int kernel = 0;
    int jump_mode = 0;  // MTGP_OPT_JUMP
    int prejump = 0;    // MTGP_OPT_PREJUMP
    // bumped by every change of the stream states (generation, skip, restore, stat passes): the
    // planner's speculative next-call windows are valid only for the very next state
    uint64_t state_epoch = 0;
    BitmapPred bm_pred;  // predicate of kKindBitmapRange (ctx_generate_bitmap)
    uint32_t stage_next = 0;  // host output: the staging buffer the next chunk uses (alternates across calls)
    uint32_t max_pieces = 0;
    uint64_t min_piece_words = 0;  // 0 = auto (pieces_wanted, mtgp_plan.cu)
    bool timing = false;
    uint64_t host_chunk = 1ull << 20;

    // host-output staging
    void* d_stage = nullptr;
    size_t stage_bytes = 0;
    // short-skip scratch (mtgp_skip below 4096 words): kept across calls, grown on demand
    void* d_skip = nullptr;
    size_t skip_bytes = 0;
    // stat-test scratch (slot 0: saved window, slot 1: chunk + counters), kept across
    // mtgp_stat_run calls, grown on demand, freed with the context
    void* d_scratch[2] = {nullptr, nullptr};
    size_t scratch_bytes[2] = {0, 0};
    cudaEvent_t ev_gen[2] = {nullptr, nullptr};
    cudaEvent_t ev_copy[2] = {nullptr, nullptr};

    // timing
    EventPool pool;
    double gen_ms = 0, jump_ms = 0;
    uint64_t gen_launches = 0, jump_launches = 0;
    uint64_t total_launches = 0;  // every kernel this context launched

    // v2 planner / jump-ahead state
    std::unique_ptr<Planner> planner;
    uint32_t last_pieces = 0, last_warps = 0, last_kernel = 0;

    mtgp_ctx() = default;
    mtgp_ctx(const mtgp_ctx&) = delete;
    mtgp_ctx& operator=(const mtgp_ctx&) = delete;
    // Releases whatever was created, so a partially built context (a failed mtgp_ctx_create)
    // does not leak. cudaFree / cudaEventDestroy / cudaStreamDestroy accept null handles.
    ~mtgp_ctx() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        if (copy_stream) cudaStreamSynchronize(copy_stream);
        planner.reset();
        for (void* p : {(void*)d_params, (void*)d_mt, (void*)d_win, (void*)d_ck, d_stage, d_skip, d_scratch[0], d_scratch[1]})
            if (p) cudaFree(p);
        for (int i = 0; i < 2; ++i) {
            if (ev_gen[i]) cudaEventDestroy(ev_gen[i]);
            if (ev_copy[i]) cudaEventDestroy(ev_copy[i]);
        }
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }
};

namespace mtgpb {
// Sets the thread-local mtgp_last_error() message; returns `code`.
int set_error(int code, const char* fmt, ...);
int cuda_error(cudaError_t e, const char* what);
// One device-side generation of L words per stream into device memory `out` (advances positions).
int ctx_generate_device(mtgp_ctx* ctx, int kind, void* out, uint64_t L);
// The same L words per stream, but only one predicate bit per word into `bitmap` (per stream
// ceil(L / 32) words, which the caller zeroes): kKindBitmapBit0 / kKindBitmapRange with `pred`.
// Register-resident warp-team contexts only (gen3, mt_gen3); MTGP_EINVAL elsewhere.
int ctx_generate_bitmap(mtgp_ctx* ctx, int kind, uint32_t* bitmap, uint64_t L, const BitmapPred& pred);
}  // namespace mtgpb
