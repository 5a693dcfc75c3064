/*
 * mtgp_b200.h -- C-ABI of the B200-native MTGP32 bulk generator (libmtgp_b200.so).
 *
 * This is the drop-in boundary under the reference's generation path. The reference binds
 * its generation path through C++, not an FFI:
 *
 *   class WordSource { virtual void fill(std::span<std::uint32_t> out) = 0; }
 *        proj/include/twistsieve/word_source.hpp:21-25
 *   std::unique_ptr<WordSource> make_word_source(const ParameterizedStatus&, std::uint32_t seed)
 *        proj/include/twistsieve/word_source.hpp:75-76, proj/src/word_source.cpp:5-16
 *   Generator(ParameterizedStatus, seed) / next_u32 / next_f64_01 / from_state
 *        proj/include/twistsieve/generator.hpp:23-52, proj/src/generator.cpp:37-66
 *
 * Each entry point below names the reference interface it replaces. The C++ layer
 * (include/twistsieve_b200/ headers: GpuWordSource : WordSource, make_word_source for
 * Engine::mtgp32) sits on top of these calls; INTEGRATION.md shows the binding.
 *
 * Conventions (mirroring the reference's error behaviour without exceptions across the ABI):
 *   - every function returns MTGP_OK (0) or a positive MTGP_E* code;
 *   - MTGP_EINVAL is what the reference reports as std::invalid_argument
 *     (ParameterizedStatus::validate, proj/src/params.cpp:23-39; generator.cpp:40-41,57-59);
 *   - mtgp_last_error() returns a thread-local message for the last failure on this thread;
 *   - a context is not thread-safe (one per host thread, like one Generator per worker,
 *     SPEC.md:104-105); it owns one CUDA stream and all its device memory.
 *   - There is no CPU fallback: without a usable sm_100 device, mtgp_ctx_create fails with
 *     MTGP_ECUDA.
 *
 * Output layout: per-stream contiguous. A call with words_per_stream = L writes stream s
 * (parameter set s with seed s) at out[s*L, (s+1)*L) and advances every stream by L words,
 * exactly as L successive WordSource::fill() words would (word_source.hpp:31-33).
 */
#ifndef MTGP_B200_H
#define MTGP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MTGP_ABI_VERSION 1

/* status codes */
#define MTGP_OK 0
#define MTGP_EINVAL 1   /* invalid parameter set / argument  (reference: std::invalid_argument) */
#define MTGP_ECUDA 2    /* CUDA runtime failure or no usable device                           */
#define MTGP_ENOMEM 3   /* device or pinned-host allocation failed                            */
#define MTGP_ESTATE 4   /* call not valid in the context's current state                      */

/* output kinds */
#define MTGP_U32 0      /* tempered 32-bit word                                  */
#define MTGP_F32_12 1   /* single float in [1,2): bits (u32 >> 9) | 0x3F800000   */
#define MTGP_F32_01OC 2 /* single float in (0,1]: 2.0f - [1,2) value (exact)     */
#define MTGP_F64_01 3   /* double in [0,1): u32 * 2^-32, draw for draw (Generator::next_f64_01,
                           proj/include/twistsieve/generator.hpp:39-41); 8 bytes per sample */

/*
 * One MTGP32 parameter set. Field meaning follows mtgp32_params_fast
 * (/usr/local/cuda/include/curand_mtgp32.h:140-152); poly_sha1 is not needed on the device.
 * Replaces: the recurrence fields of ParameterizedStatus (proj/include/twistsieve/params.hpp:21-42)
 * for Engine::mtgp32.
 */
typedef struct mtgp_params {
    uint32_t mexp;           /* Mersenne exponent; N = mexp/32 + 1 words of state */
    uint32_t pos;            /* pick-up position, 3 <= pos <= N - 32              */
    uint32_t sh1, sh2;       /* shifts, 1..31                                      */
    uint32_t tbl[16];        /* recursion table (GF(2)-linear in its 4-bit index)  */
    uint32_t tmp_tbl[16];    /* tempering table                                    */
    uint32_t flt_tmp_tbl[16];/* tempering+float table: must equal (tmp>>9)|0x3F800000 */
    uint32_t mask;           /* 0xFFFFFFFF << (32N - mexp)                         */
} mtgp_params;

/* Per-stream checksum accumulated by the generation kernels (order independent). */
typedef struct mtgp_cksum {
    uint64_t sum64;          /* sum of the emitted 32-bit words (float kinds: bit patterns), mod 2^64 */
    uint64_t words;          /* words emitted                                                        */
    uint32_t xor32;          /* XOR of the emitted words                                             */
    uint32_t pad;
} mtgp_cksum;

typedef struct mtgp_ctx mtgp_ctx;

/* Options for mtgp_set_option */
#define MTGP_OPT_CHECKSUM 1        /* accumulate mtgp_cksum in-kernel: 0 off, 1 (default) sum64 +   */
                                   /* xor32, 2 sum32 + xor32 (the word sum mod 2^32, without the   */
                                   /* 64-bit carry chain; after any mode-2 call mtgp_checksums     */
                                   /* reports sum64 mod 2^32 until mtgp_checksums_reset)           */
#define MTGP_OPT_KERNEL 2          /* 0 = auto, 1 = reference-shaped v1 (one CTA per set), 2 = v2 */
                                   /* (shared-memory ring), 3 = v3 (register ring, mexp 11213),   */
                                   /* 4 = v4 (register ring for any supported exponent);          */
                                   /* Engine::mt contexts: 5 = warp teams, shared-memory rings,   */
                                   /* 6 = warp teams, register-resident (n = 624)                 */
#define MTGP_OPT_MAX_PIECES 3      /* cap on jump-ahead pieces per call (0 = auto)                  */
#define MTGP_OPT_MIN_PIECE_WORDS 4 /* minimum words per jump-ahead piece; 0 (default) = auto: 1<<21, */
                                   /* down to 1<<19 to keep >= 3 CTAs per SM busy                  */
#define MTGP_OPT_TIMING 5          /* 0/1: record CUDA events around every generation kernel        */
#define MTGP_OPT_HOST_CHUNK 6      /* words per stream per device chunk when out is host memory     */
#define MTGP_OPT_JUMP 7            /* jump-ahead algorithm: 0 = auto (Karatsuba middle product for  */
                                   /* windows N > 384 words, direct otherwise), 1 = direct always, */
                                   /* 2 = split (Karatsuba, or q blocks over several warps at d=0) */
#define MTGP_OPT_PREJUMP 8         /* speculative next-call jumps: 0 = auto (when the call's plan   */
                                   /* uses <= 1/4 of the generator's warp slots), 1 = off,         */
                                   /* 2 = always. Each call's jump-ahead windows for the NEXT call  */
                                   /* (same length, no state change in between) are computed on a  */
                                   /* side stream while this call generates                         */

/* Library / device info. */
int mtgp_abi_version(void);
const char* mtgp_last_error(void);

/*
 * Validate one parameter set (replaces ParameterizedStatus::validate for Engine::mtgp32,
 * proj/src/params.cpp:23-39): supported shape, mask, shifts, pos window, table linearity,
 * float table identity. MTGP_EINVAL with a message on failure.
 */
int mtgp_validate_params(const mtgp_params* p);

/*
 * Create a context holding n_sets independent streams; stream s uses sets[s] seeded with
 * seeds[s] (MTGP seed expansion, curand_mtgp32_host.h:155-172).
 * Replaces: Generator::Generator(params, seed) (generator.cpp:37-52) and
 * make_word_source(params, seed) (word_source.cpp:5-16), batched over n_sets streams.
 * All sets of one context must share mexp. `stream` is a cudaStream_t to run on, or NULL for
 * a context-owned stream.
 */
int mtgp_ctx_create(mtgp_ctx** out, int device, const mtgp_params* sets, uint32_t n_sets,
                    const uint32_t* seeds, void* stream);
int mtgp_ctx_destroy(mtgp_ctx* ctx);

/* Number of streams, state words per stream (N), current position (words emitted) of stream s. */
int mtgp_ctx_info(const mtgp_ctx* ctx, uint32_t* n_sets, uint32_t* state_words, uint32_t* mexp);
int mtgp_position(const mtgp_ctx* ctx, uint32_t s, uint64_t* words_emitted);
/* The cudaStream_t all of this context's work is enqueued on. */
int mtgp_ctx_stream(const mtgp_ctx* ctx, void** stream);

int mtgp_set_option(mtgp_ctx* ctx, int option, int64_t value);

/*
 * Bulk generation. Writes words_per_stream outputs of every stream, per-stream contiguous,
 * and advances every stream. out_is_device = 1: `out` is device memory on the context's
 * device (the call is asynchronous on the context stream); 0: `out` is host memory (pageable
 * or pinned; the call returns when the data is in `out`).
 * Replaces: WordSource::fill(std::span<uint32_t>) (word_source.hpp:21-25,31-33) for n_sets
 * streams at once; the float kinds extend next_f64_01 (generator.hpp:39-41) with the
 * single-float [1,2) / (0,1] conversions north_star names.
 */
int mtgp_generate(mtgp_ctx* ctx, int kind, void* out, uint64_t words_per_stream, int out_is_device);
int mtgp_generate_u32(mtgp_ctx* ctx, uint32_t* out, uint64_t words_per_stream, int out_is_device);
int mtgp_generate_f32_12(mtgp_ctx* ctx, float* out, uint64_t words_per_stream, int out_is_device);
int mtgp_generate_f32_01oc(mtgp_ctx* ctx, float* out, uint64_t words_per_stream, int out_is_device);
/* mtgp_generate without waiting: host output is complete (and `out` may be read or reused) only
 * after mtgp_sync. With page-locked `out` (mtgp_host_alloc) generation and the device->host copy
 * overlap the caller's work: GpuWordSource refills one buffer while its consumer reads the other. */
int mtgp_generate_async(mtgp_ctx* ctx, int kind, void* out, uint64_t words_per_stream, int out_is_device);

/*
 * Advance every stream by `words` without writing output (GF(2) jump-ahead; cost independent
 * of `words`). No reference equivalent: the reference can only step.
 */
int mtgp_skip(mtgp_ctx* ctx, uint64_t words);

/*
 * State save / restore: the N-word window x[i..i+N-1] of every stream (oldest first; the low
 * 32N-mexp bits of the oldest word are dead) plus its position i.
 * Replaces: SeedStatus {seed, state, index} / Generator::from_state (generator.hpp:11-15,
 * generator.cpp:54-66). windows: n_sets*N words; positions: n_sets (may be NULL on save).
 */
int mtgp_state_save(mtgp_ctx* ctx, uint32_t* windows, uint64_t* positions);
int mtgp_state_restore(mtgp_ctx* ctx, const uint32_t* windows, const uint64_t* positions);

/* Per-stream checksums accumulated since create / reset (n_sets entries). */
int mtgp_checksums(mtgp_ctx* ctx, mtgp_cksum* out);
int mtgp_checksums_reset(mtgp_ctx* ctx);

/* Wait for all work on the context stream. */
int mtgp_sync(mtgp_ctx* ctx);

/*
 * Page-locked host memory for host-output generation (out_is_device = 0): device->host copies
 * into it run at the PCIe rate instead of through the driver's pageable staging (~4x slower for
 * 4 MB refills). Replaces the reference's std::vector fill buffer of BufferedStream
 * (proj/include/twistsieve/word_source.hpp:94) for GpuWordSource. mtgp_host_free(NULL) is a no-op.
 */
int mtgp_host_alloc(size_t bytes, void** out);
int mtgp_host_free(void* p);

/*
 * Timing of the generation kernels (MTGP_OPT_TIMING = 1): total device milliseconds and launch
 * count of the main generation kernel, and of the jump-ahead kernels, since the last reset.
 */
int mtgp_kernel_timing(mtgp_ctx* ctx, double* gen_ms, uint64_t* gen_launches, double* jump_ms,
                       uint64_t* jump_launches);
int mtgp_kernel_timing_reset(mtgp_ctx* ctx);
/* Number of CUDA kernels this context has launched since creation. */
int mtgp_launch_count(const mtgp_ctx* ctx, uint64_t* launches);

/*
 * Characteristic-polynomial digests (replaces verify_digest / poly_digest for the MTGP engine,
 * proj/include/twistsieve/dynamic_creator.hpp:16-51): out receives n_sets NUL-terminated
 * 41-byte hex SHA-1 strings of each stream's minimal polynomial (Berlekamp-Massey over a
 * device-generated prefix), printed as '0'/'1' coefficients lowest degree first -- the form
 * the MTGP tables' poly_sha1 uses (curand_mtgp32.h:140-152). Empty string: none found.
 */
int mtgp_charpoly_sha1(mtgp_ctx* ctx, char* out);

/*
 * Engine::mt -- the reference's own generic MT recurrence on the GPU, bit-exact with
 * Generator/MtWordSource (proj/src/generator.cpp:7-13,37-52,68-88). Field meaning is that of
 * ParameterizedStatus (proj/include/twistsieve/params.hpp:21-42).
 */
typedef struct mtgp_mt_params {
    uint32_t id, mexp, n, m, r, a;
    uint32_t temper_b, temper_c, temper_u, temper_s, temper_t, temper_l;
} mtgp_mt_params;

/* ParameterizedStatus::validate (proj/src/params.cpp:23-39): MTGP_EINVAL with the reference's
   message on a violated invariant. */
int mtgp_mt_validate_params(const mtgp_mt_params* p);

/*
 * Context of n_sets Engine::mt streams (= n_sets make_word_source(status, seed) calls,
 * proj/src/word_source.cpp:5-16). Seeds expand as Generator::Generator (generator.cpp:37-52).
 * Supports mtgp_generate (all kinds; u32 = next_u32 order), state save/restore (window of n
 * words, stride = max n), checksums, positions, mtgp_skip, mtgp_certify,
 * mtgp_mt_charpoly_digest and mtgp_stat_run. When every status has the same mexp and n and
 * n - m >= 32, generation and long skips use the jump-ahead planner with warp teams (kernel
 * version 5 in mtgp_last_plan; version 6, the register-resident team kernel, for n = 624 with
 * every n - m >= 129, u32 or f64 output, words_per_stream % 4 == 0 and 16-byte aligned output);
 * otherwise (and for MTGP_F64_01 outside version 6's shape) one CTA per stream.
 * MTGP_OPT_KERNEL 5 / 6 force the team kernel, 1 the CTA-per-stream one.
 */
int mtgp_mt_ctx_create(mtgp_ctx** out, int device, const mtgp_mt_params* sets, uint32_t n_sets,
                       const uint32_t* seeds, void* stream);

/* Launch plan of the last generation call: pieces (jump-ahead segments), warps per piece and the
   kernel (1 CTA per stream, 2 shared-memory ring, 3 / 4 register ring, 5 Engine::mt warp teams
   with shared-memory rings, 6 Engine::mt register-resident warp teams). */
int mtgp_last_plan(const mtgp_ctx* ctx, uint32_t* pieces, uint32_t* warps_per_piece,
                   uint32_t* kernel_version);

/*
 * Certification (table tooling): out[s] = 1 iff stream s's minimal polynomial,
 * taken from its current state, has degree mexp and is irreducible -- the maximal-period test the
 * reference's dynamic creator accepts a status by (proj/src/dynamic_creator.cpp:79-81,
 * is_irreducible gf2poly.cpp:342-383). MTGP32 and Engine::mt contexts. State is unchanged.
 */
int mtgp_certify(mtgp_ctx* ctx, int32_t* out);

/*
 * Engine::mt contexts: the reference's poly_digest (proj/src/dynamic_creator.cpp:9-31) of each
 * stream's minimal polynomial probed from bit 0 of its next 2*mexp + 64 outputs
 * (probe_minimal_polynomial, :33-38). For a context seeded with kDefaultProbeSeed (1) this is
 * the digest verify_digest compares with ParameterizedStatus::charpoly_digest (:99-103).
 * out: 41 bytes per stream (40 hex digits + NUL). State is unchanged.
 */
int mtgp_mt_charpoly_digest(mtgp_ctx* ctx, char* out);

/* The irreducibility test alone (host): coeff_bits[i] (0/1, one byte per coefficient, the
   reference's Gf2Poly::from_coeff_bits layout) is the coefficient of x^i. MTGP_EINVAL for a
   constant polynomial, like the reference's is_irreducible. */
int mtgp_gf2_is_irreducible(const uint8_t* coeff_bits, uint64_t n, int32_t* out);

/* ------------------------------------------------------------------------------------------
 * Several GPUs in one process (north_star (5)).
 *
 * The reference's only parallelism is a pool of worker threads over independent statuses
 * (proj/src/sieve.cpp:170-177; one generator per worker). mtgp_multi splits
 * n_sets parameter sets into contiguous balanced ID ranges, one per device (mtgp_shard_range),
 * owns one context per device, and runs every generation call with one host thread per device
 * (no collective on the hot path). The per-stream checksums are all-gathered once, over NCCL
 * (ncclCommInitAll + ncclAllGather on the devices' streams; libnccl is dlopen'ed) when it loads
 * and the devices are distinct, else by host concatenation.
 * ------------------------------------------------------------------------------------------ */
typedef struct mtgp_multi mtgp_multi;

/* Set IDs [*first, *first + *count) of `rank` when n_sets are split over `world` ranks: the
   first n_sets % world ranks get one more (the split bench.py's config 5 uses). */
int mtgp_shard_range(uint32_t n_sets, uint32_t world, uint32_t rank, uint32_t* first, uint32_t* count);

/* Contexts for sets[first_r .. first_r + count_r) on devices[r], seeded with the matching seeds.
   gather: 0 = NCCL when possible else host, 1 = NCCL required, 2 = host. */
int mtgp_multi_create(mtgp_multi** out, const int* devices, uint32_t n_devices, const mtgp_params* sets,
                      uint32_t n_sets, const uint32_t* seeds, int gather);
int mtgp_multi_destroy(mtgp_multi* m);
/* *nccl = 1 when the checksum gather runs over NCCL. */
int mtgp_multi_info(const mtgp_multi* m, uint32_t* n_devices, int* nccl);
/* The context of `rank` (options, timing, positions) and its set range. Owned by m. */
int mtgp_multi_context(mtgp_multi* m, uint32_t rank, mtgp_ctx** ctx, uint32_t* first_set, uint32_t* n_sets);
/* words_per_stream words of every stream: device r writes its streams, per-stream contiguous,
   into device memory outs[r] (on devices[r]); one host thread per device; returns when done. */
int mtgp_multi_generate(mtgp_multi* m, int kind, void* const* outs, uint64_t words_per_stream);
/* Per-stream checksums of all n_sets streams in global set order (the gather). */
int mtgp_multi_checksums(mtgp_multi* m, mtgp_cksum* out);

/* ------------------------------------------------------------------------------------------
 * Device-side statistical tests (GPU-fed consumers).
 *
 * The reference runs each campaign cell (status, seed, test) as run_test(BufferedStream over a
 * fresh make_word_source(status, seed)) (proj/src/sieve.cpp:156-158) with the four templates of
 * proj/include/twistsieve/stat_tests.hpp:83-309. mtgp_stat_run does the same for every stream
 * of a context at once: the words are generated and counted on the GPU (they never leave HBM),
 * and the host turns the integer counts into the statistic, p-value and class with a
 * restatement of the reference's numerics (proj/src/stats.cpp, classify.cpp). Counts are
 * bit-exact with the reference templates over the same words, and so are statistic and p-value
 * (same arithmetic in the same order).
 * ------------------------------------------------------------------------------------------ */
#define MTGP_STAT_GAP 0            /* gap_test            stat_tests.hpp:83-138  */
#define MTGP_STAT_HAMMING_INDEP 1  /* hamming_indep_test  stat_tests.hpp:149-208 */
#define MTGP_STAT_COLLISION_OVER 2 /* collision_over_test stat_tests.hpp:214-248 */
#define MTGP_STAT_RANDOM_WALK 3    /* random_walk_test    stat_tests.hpp:253-309 */

/* PValueClass (proj/include/twistsieve/classify.hpp:11) */
#define MTGP_PCLASS_CORRECT 0
#define MTGP_PCLASS_SUSPECT 1
#define MTGP_PCLASS_DISASTROUS 2

/* per-stream result error codes */
#define MTGP_STAT_OK 0
#define MTGP_STAT_EXHAUSTED 2      /* StreamExhausted ("insufficient stream"), word_source.hpp:15-17 */

/* TestSpec (stat_tests.hpp:18-33); `test` replaces the test_id string. */
typedef struct mtgp_stat_spec {
    int32_t test;
    uint32_t N;      /* replication count (kept at 1) */
    uint64_t n;      /* gaps / blocks / pairs / walks */
    uint32_t r, s, L, d, l, t;
    double alpha, beta;
} mtgp_stat_spec;

/* TestResult (stat_tests.hpp:35-42) for one stream, plus the words the test consumed. */
typedef struct mtgp_stat_result {
    double statistic, p_value;
    int32_t classification, degenerate;
    int32_t error;   /* MTGP_STAT_OK or MTGP_STAT_EXHAUSTED (then the other fields are 0) */
    int32_t pad;
    uint64_t words_used;
} mtgp_stat_result;

/* TestSpec::validate (stat_tests.cpp:7-30) plus each test's pre-consumption checks ("sample
   too small", "spec out of sparse regime"); MTGP_EINVAL with the reference's message. */
int mtgp_stat_validate(const mtgp_stat_spec* spec);

/* Runs the test on every stream of ctx, each from the context's current position; results[s]
   for stream s. The context's state and checksums are left unchanged. The context keeps a
   scratch arena for the generated chunks (about 2^32 bytes at any stream count, up to 2^26
   bytes per stream) until it is destroyed. */
int mtgp_stat_run(mtgp_ctx* ctx, const mtgp_stat_spec* spec, mtgp_stat_result* results);

/* The host half alone: result from a test's integer counts. Layout: gap tcut+1 gap-length
   counts; hamming_indep {table[0][0], [0][1], [1][0], [1][1]}; collision_over {collisions};
   random_walk l+1 right-step counts. *n_counts from mtgp_stat_counts_len. */
int mtgp_stat_counts_len(const mtgp_stat_spec* spec, uint64_t* n_counts);
int mtgp_stat_finish(const mtgp_stat_spec* spec, const uint64_t* counts, uint64_t n_counts,
                     mtgp_stat_result* result);

/* The numerics (proj/include/twistsieve/stats.hpp, classify.hpp); MTGP_EINVAL where the
   reference throws std::invalid_argument. */
int mtgp_ln_gamma(double x, double* out);
int mtgp_gamma_p(double a, double x, double* out);
int mtgp_gamma_q(double a, double x, double* out);
int mtgp_chi_square_pvalue(double statistic, uint32_t df, double* out);
int mtgp_poisson_cdf(uint64_t k, double lambda, double* out);
int mtgp_poisson_sf(uint64_t k, double lambda, double* out);
int mtgp_poisson_pmf(uint64_t k, double lambda, double* out);
int mtgp_binomial_log_pmf(uint64_t k, uint64_t n, double p, double* out);
int mtgp_binomial_upper_tail(uint64_t count, uint64_t n, double p, double* out);
int mtgp_classify_pvalue(double p, int32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* MTGP_B200_H */
