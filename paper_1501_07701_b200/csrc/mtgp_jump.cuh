// mtgp_jump.cuh -- jump-ahead by a transposed-Karatsuba middle product (mtgp_jump.cu).
#pragma once

#include "mtgp_v2.cuh"

namespace mtgpb {

// Launch plan of the Karatsuba jump for one window length N (host-built, passed by value).
struct KaraPlan {
    uint32_t depth = 0;       // Karatsuba levels d (0, 1 or 2)
    uint32_t n_out = 0;       // padded output range 384 * 2^d >= N
    uint32_t blocks = 0;      // B: q blocks of n_out bits
    uint32_t blk_qwords = 0;  // n_out / 32
    uint32_t n_leaf = 0;      // 3^d
    uint32_t nz[9], oz[9][4];  // per leaf: prefix-window offsets (words) XORed into its z vector
    uint32_t nq[9], oq[9][4];  // per leaf: raw q word offsets XORed into its q words
    uint32_t n_comb = 0;       // 2^d
    uint32_t comb[4][4];       // per output quarter: the leaves XORed into it
    uint32_t groups = 1;       // G: the blocks are split over G warps per leaf (set per launch)
};

// false: N > 1536 (use the flat jump). depth_override < 0: the smallest d with 384 * 2^d >= N.
bool kara_plan(uint32_t N, uint32_t q_words, int depth_override, KaraPlan& k);
// block groups per leaf so that n_jobs * n_leaf * G warps fill the GPU (64-register leaf kernel)
uint32_t kara_groups(const KaraPlan& k, uint32_t n_jobs, int num_sms);
// prefix words (from x_{t0}) the Karatsuba jump reads
uint32_t kara_prefix_words(const KaraPlan& k);
size_t kara_zbuf_words(const KaraPlan& k, uint32_t n_rows);
size_t kara_leaf_words(const KaraPlan& k, uint32_t n_jobs);  // k.groups must be set
cudaError_t launch_jump_kara(const JumpArgs& a, const KaraPlan& k, uint32_t N, uint32_t n_rows, uint32_t* zbuf,
                             uint32_t* leaf_out, cudaStream_t st);

}  // namespace mtgpb
