// mtgp_v2.cuh -- launch interface of the v2 kernels (mtgp_v2.cu).
#pragma once

#include "mtgp_internal.cuh"

namespace mtgpb {

// Words a v2 team produces per full step (one warp, 8 words per lane).
constexpr uint32_t kStepWords = 256;
constexpr uint32_t kWarpsPerCta = 4;

struct GenArgs {
    const DevParams* params;
    const Piece* pieces;
    const TeamWork* teams;
    uint32_t n_teams;
    const uint32_t* const* piece_win;  // per piece: start window (N words)
    uint32_t* win_out;                 // [n_sets][N] end windows
    void* out;                         // per-stream stride L (bitmap kinds: ceil(L / 32) words)
    uint64_t L;
    DevCksum* ck;
    BitmapPred pred;                   // kKindBitmapRange
};

struct JumpJob {
    uint32_t piece;  // destination: jumped window of this piece
    uint32_t q;      // index of its jump polynomial
    uint32_t row;    // prefix row (the piece's stream)
};

struct JumpArgs {
    const uint32_t* pre;      // [n_jump_sets][pre_len] state-word prefixes
    uint32_t pre_len;         // words staged per row (>= M + N + slack)
    uint32_t pre_stride;      // words between rows
    uint32_t pre_off;         // reference offset t0: the staged sequence starts at x_{t0}
    const uint32_t* set_of;   // [n_jump_sets] set index of each prefix row
    const uint32_t* job_off;  // [n_jump_sets + 1] CSR offsets into jobs
    const JumpJob* jobs;
    const uint32_t* q;        // [n_q][q_words] jump polynomials, bit i = coeff of x^i
    uint32_t q_words;
    uint32_t* piece_win;      // [n_pieces][N]
    uint32_t max_jobs_per_row = 1;
    uint32_t n_jobs = 0;
};

// ring size (words) of one warp team for exponent mexp
uint32_t v2_ring_words(uint32_t mexp);
bool v2_supports(uint32_t mexp);

cudaError_t launch_prefix(const DevParams* params, const uint32_t* win, const uint32_t* sets, uint32_t n_rows,
                          uint32_t N, uint32_t* pre, uint32_t len, cudaStream_t st);
cudaError_t launch_jump(uint32_t mexp, const JumpArgs& a, uint32_t n_jump_sets, cudaStream_t st);
// the same jump with a runtime window length N (Engine::mt)
cudaError_t launch_jump_rt(const JumpArgs& a, uint32_t N, cudaStream_t st);
cudaError_t launch_gen(uint32_t mexp, int kind, bool cksum, const GenArgs& a, cudaStream_t st);
int gen_ctas_per_sm(uint32_t mexp, int kind, bool cksum);
// v3: register-resident ring, MTGP32-11213 only (mtgp_v3.cu). ck_mode: 0 none, 1 sum64 + xor32,
// 2 sum32 + xor32 (MTGP_OPT_CHECKSUM)
cudaError_t launch_gen3(int kind, int ck_mode, const GenArgs& a, cudaStream_t st);
int gen3_ctas_per_sm(int kind, int ck_mode);
// v4: gen3's register-resident design templated on the exponent (csrc/mtgp_v4.cu)
bool v4_supports(uint32_t mexp, int kind);
cudaError_t launch_gen4(uint32_t mexp, int kind, int ck_mode, const GenArgs& a, cudaStream_t st);
int gen4_ctas_per_sm(uint32_t mexp, int kind, int ck_mode);

}  // namespace mtgpb
