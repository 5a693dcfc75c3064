// mtgp_mt.cuh -- Engine::mt (the reference's classic MT recurrence) device interface.
#pragma once

#include "mtgp_internal.cuh"

namespace mtgpb {

struct alignas(16) DevMtParams {
    uint32_t n, m, r, a, b, c, u, s, t, l;
    uint32_t mul_s, mul_t;  // 2^s, 2^t: the left shifts of the tempering as IMADs (mt_gen3)
};

cudaError_t launch_mt_v1(int kind, bool cksum, const DevMtParams* params, uint32_t* win, uint32_t n_sets,
                         uint32_t nmax, void* out, uint64_t L, DevCksum* ck, cudaStream_t st);

// Warp-team generation over jump-ahead pieces (the MTGP planner's decomposition applied to the
// reference's recurrence): one warp per team, a per-warp shared-memory ring.
struct MtGenArgs {
    const DevMtParams* params;
    const Piece* pieces;
    const TeamWork* teams;
    uint32_t n_teams;
    const uint32_t* const* piece_win;  // per piece: start window (n words)
    uint32_t* win_out;                 // [n_sets][n] end windows
    void* out;                         // per-stream stride L
    uint64_t L;
    DevCksum* ck;
    uint32_t n;                        // state words (uniform over the context)
    bool pairs = false;                // two words per lane (L even, output 8-byte aligned)
    BitmapPred pred;                   // kKindBitmapRange
};
// raw state words x_0 .. x_{len-1} of each row's stream (x_0..x_{n-1} = its window)
cudaError_t launch_mt_prefix(const DevMtParams* params, const uint32_t* win, const uint32_t* sets, uint32_t n_rows,
                             uint32_t n, uint32_t* pre, uint32_t len, cudaStream_t st);
cudaError_t launch_mt_gen2(int kind, bool cksum, const MtGenArgs& a, cudaStream_t st);
int mt_gen2_ctas_per_sm(uint32_t n, int kind, bool cksum);
// Register-resident warp teams (csrc/mtgp_mt3.cu, kernel version 6): n = 624, every status
// n - m >= 129 (min_gap), u32 or f64 output, L % 4 == 0, 16-byte aligned output.
bool mt_gen3_supports(uint32_t n, uint32_t min_gap, int kind);
cudaError_t launch_mt_gen3(uint32_t n, int kind, int ck_mode, const MtGenArgs& a, cudaStream_t st);  // ck_mode 0/1/2
int mt_gen3_ctas_per_sm(uint32_t n, int kind, int ck_mode);

}  // namespace mtgpb
