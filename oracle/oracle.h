/*
 * oracle.h -- CPU restatement of the generation path. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load liboracle.so. The product (libmtgp_b200.so) never links or calls it.
 *
 * Two engines are restated here, both sequential, one word at a time:
 *
 *  (1) MTGP32 (Saito & Matsumoto; the generator the paper, chooses for
 *      GPUs). The reference artifact does NOT implement it,
 *      so this restatement follows SURVEY.md Appendix A and is pinned against NVIDIA's
 *      cuRAND MTGP32 host/device headers compiled host-side (oracle/curand_pin.cpp,
 *      /usr/local/cuda/include/curand_mtgp32_kernel.h:137-228,
 *      curand_mtgp32_host.h:155-172) -> tests/golden/mtgp32_11213_curand.json.
 *      Parity status: pinned by an external oracle (cuRAND), not by reference tests.
 *
 *  (2) The reference's own generic MT engine, Engine::mt
 *      (proj/src/generator.cpp:7-13 temper, :18-35 untemper, :37-52 seeding,
 *      :68-88 refill; proj/include/twistsieve/generator.hpp:33-41 next_u32/next_f64_01).
 *      Pinned by the reference's own goldens (proj/tests/test_generator.cpp:11-25,67) and by
 *      the reference compiled from its sources into oracle/_ref/ (oracle/Makefile).
 */
#ifndef MTGP_ORACLE_H
#define MTGP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One MTGP32 parameter set; field meaning as curand_mtgp32.h:140-152 (mtgp32_params_fast). */
typedef struct oracle_mtgp_params {
    uint32_t mexp, pos, sh1, sh2;
    uint32_t tbl[16];
    uint32_t tmp_tbl[16];
    uint32_t flt_tmp_tbl[16];
    uint32_t mask;
} oracle_mtgp_params;

/* Sequential MTGP32 generator: a circular buffer of exactly N = mexp/32 + 1 words. */
typedef struct oracle_mtgp {
    oracle_mtgp_params p;
    uint32_t n;       /* N */
    uint32_t idx;     /* slot of x[i], i = words generated so far, mod N */
    uint64_t count;   /* words generated so far */
    uint32_t st[4096];
} oracle_mtgp;

uint32_t oracle_mtgp_n(uint32_t mexp);
/* Appendix A "Init(seed)" (curand_mtgp32_host.h:155-172). Returns 0, or -1 if mexp too large. */
int oracle_mtgp_init(oracle_mtgp* g, const oracle_mtgp_params* p, uint32_t seed);
/* kind: 0 = u32, 1 = f32 [1,2) bit pattern, 2 = f32 (0,1] bit pattern */
void oracle_mtgp_fill(oracle_mtgp* g, uint32_t* out, size_t n, int kind);
/* Advance without output. */
void oracle_mtgp_skip(oracle_mtgp* g, uint64_t n);
/* Copy the current window x[i..i+N-1] (oldest first). */
void oracle_mtgp_window(const oracle_mtgp* g, uint32_t* out);
/* Construct from a raw window x[i..i+N-1] (analogue of Generator::from_state, generator.cpp:54-66). */
int oracle_mtgp_from_window(oracle_mtgp* g, const oracle_mtgp_params* p, const uint32_t* win);

/* Checksums over n words of stream `seed` from position 0, u32 output. */
typedef struct oracle_cksum {
    uint64_t sum64;
    uint32_t xor32;
    uint32_t last;
    uint32_t poly31;  /* h = h*31 + v (mod 2^32) */
    uint32_t pad;
} oracle_cksum;
void oracle_cksum_words(const uint32_t* w, size_t n, oracle_cksum* acc);

/* Multi-threaded bulk fill: one stream per set, `n` words each, out[s*n + j]. Returns seconds. */
double oracle_mtgp_bulk(const oracle_mtgp_params* sets, const uint32_t* seeds, uint32_t n_sets,
                        uint64_t skip, uint64_t n, uint32_t* out, int kind, int threads);

/* Streaming checksums for full-volume parity fixtures: stream s = (sets[s], seeds[s]) from
 * position 0; out[s*n_rec + k] = cumulative checksums of its first (k+1)*rec_every words.
 * Index 0 = u32 words, 1 = f32 [1,2) bit patterns, 2 = f32 (0,1] bit patterns (1, 2 only when
 * flags & 1). flags & 2 forces the one-word-at-a-time form (otherwise 16 steps per AVX-512
 * vector where the CPU has it and N - pos >= 16). No output buffer; threads take one stream at
 * a time. Returns seconds. */
typedef struct oracle_stream_ck {
    uint64_t sum[3];
    uint32_t xr[3];
    uint32_t pad;
} oracle_stream_ck;
double oracle_mtgp_cksum_stream(const oracle_mtgp_params* sets, const uint32_t* seeds, uint32_t n_sets,
                                uint64_t rec_every, uint32_t n_rec, int flags, oracle_stream_ck* out,
                                int threads);

/* CPU baseline of the generation path: every stream seeded and filled `chunk` words at a time
 * into a reused per-thread buffer until it has produced n words (WordSource::fill semantics,
 * word_source.hpp:21-25), streams handed to threads dynamically. Returns seconds. */
double oracle_mtgp_fill_bulk(const oracle_mtgp_params* sets, const uint32_t* seeds, uint32_t n_sets, uint64_t n,
                             uint64_t chunk, int kind, int threads, uint64_t* sink);

/* ---- classic MT, the reference Engine::mt ---- */
typedef struct oracle_mt_params {
    uint32_t mexp, n, m, r, a;
    uint32_t b, c, u, s, t, l;
} oracle_mt_params;

typedef struct oracle_mt {
    oracle_mt_params p;
    uint32_t index;
    uint32_t st[2048];
} oracle_mt;

void oracle_mt19937_params(oracle_mt_params* p);
int oracle_mt_init(oracle_mt* g, const oracle_mt_params* p, uint32_t seed);
uint32_t oracle_mt_temper(uint32_t y, const oracle_mt_params* p);
uint32_t oracle_mt_untemper(uint32_t y, const oracle_mt_params* p);
void oracle_mt_fill(oracle_mt* g, uint32_t* out, size_t n);

/* splitmix64 / derive_seed (word_source.cpp:18-27) */
uint64_t oracle_splitmix64(uint64_t x);
uint32_t oracle_derive_seed(uint64_t source, uint32_t j);

#ifdef __cplusplus
}
#endif
#endif
