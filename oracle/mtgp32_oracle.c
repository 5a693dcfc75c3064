/*
 * mtgp32_oracle.c -- sequential CPU restatement of MTGP32. TEST INFRASTRUCTURE ONLY
 * (see oracle.h for who may call it). Follows SURVEY.md Appendix A; pinned against the
 * cuRAND MTGP32 headers compiled host-side (oracle/curand_pin.cpp).
 *
 * No reference file:line exists for MTGP32 (the reference implements the classic MT
 * recurrence only, proj/src/generator.cpp:68-88). External pins:
 *   seeding   curand_mtgp32_host.h:155-172  (mtgp32_init_state)
 *   recursion curand_mtgp32_kernel.h:137-145 (para_rec)
 *   temper    curand_mtgp32_kernel.h:155-162 (temper)
 *   float     curand_mtgp32_kernel.h:174-183 (temper_single) == (u32 >> 9) | 0x3F800000
 *   stepping  curand_mtgp32_kernel.h:196-228 (curand: word t of a step reads x[t], x[t+1],
 *             x[t+pos], x[t+pos-1] and writes x[t+N])
 */
#include "oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

uint32_t oracle_mtgp_n(uint32_t mexp) { return mexp / 32 + 1; }

int oracle_mtgp_init(oracle_mtgp* g, const oracle_mtgp_params* p, uint32_t seed) {
    const uint32_t n = oracle_mtgp_n(p->mexp);
    if (n < 4 || n > 4096) return -1;
    g->p = *p;
    g->n = n;
    g->idx = 0;
    g->count = 0;
    /* hidden seed and byte fill, then the Knuth initializer XORed in */
    const uint32_t hidden = p->tbl[4] ^ (p->tbl[8] << 16);
    uint32_t c = hidden;
    c += c >> 16;
    c += c >> 8;
    memset(g->st, (int)(c & 0xffu), sizeof(uint32_t) * n);
    g->st[0] = seed;
    g->st[1] = hidden;
    for (uint32_t i = 1; i < n; ++i)
        g->st[i] ^= 1812433253u * (g->st[i - 1] ^ (g->st[i - 1] >> 30)) + i;
    return 0;
}

int oracle_mtgp_from_window(oracle_mtgp* g, const oracle_mtgp_params* p, const uint32_t* win) {
    const uint32_t n = oracle_mtgp_n(p->mexp);
    if (n < 4 || n > 4096) return -1;
    g->p = *p;
    g->n = n;
    g->idx = 0;
    g->count = 0;
    memcpy(g->st, win, sizeof(uint32_t) * n);
    return 0;
}

void oracle_mtgp_window(const oracle_mtgp* g, uint32_t* out) {
    for (uint32_t j = 0; j < g->n; ++j) {
        uint32_t s = g->idx + j;
        if (s >= g->n) s -= g->n;
        out[j] = g->st[s];
    }
}

/* One step: produce x[i+N] into slot i, return the tempered u32 output. */
static inline uint32_t step(oracle_mtgp* g) {
    const uint32_t n = g->n;
    const uint32_t i = g->idx;
    uint32_t i1 = i + 1;            if (i1 >= n) i1 -= n;
    uint32_t ip = i + g->p.pos;     if (ip >= n) ip -= n;
    uint32_t it = i + g->p.pos - 1; if (it >= n) it -= n;
    uint32_t x = (g->st[i] & g->p.mask) ^ g->st[i1];
    x ^= x << g->p.sh1;
    const uint32_t y = x ^ (g->st[ip] >> g->p.sh2);
    const uint32_t r = y ^ g->p.tbl[y & 15u];
    uint32_t t = g->st[it];
    t ^= t >> 16;
    t ^= t >> 8;
    g->st[i] = r;
    g->idx = i1;
    g->count++;
    return r ^ g->p.tmp_tbl[t & 15u];
}

void oracle_mtgp_fill(oracle_mtgp* g, uint32_t* out, size_t n, int kind) {
    for (size_t j = 0; j < n; ++j) {
        const uint32_t u = step(g);
        if (kind == 0) {
            out[j] = u;
        } else {
            uint32_t fb = (u >> 9) | 0x3F800000u;  /* [1,2) */
            if (kind == 2) {                        /* (0,1] = 2 - [1,2), exact (Sterbenz) */
                float f;
                memcpy(&f, &fb, 4);
                f = 2.0f - f;
                memcpy(&fb, &f, 4);
            }
            out[j] = fb;
        }
    }
}

void oracle_mtgp_skip(oracle_mtgp* g, uint64_t n) {
    for (uint64_t j = 0; j < n; ++j) (void)step(g);
}

void oracle_cksum_words(const uint32_t* w, size_t n, oracle_cksum* acc) {
    for (size_t j = 0; j < n; ++j) {
        acc->sum64 += w[j];
        acc->xor32 ^= w[j];
        acc->poly31 = acc->poly31 * 31u + w[j];
        acc->last = w[j];
    }
}

/* ---- multi-threaded bulk (CPU baseline and full-size parity) ---- */
typedef struct bulk_job {
    const oracle_mtgp_params* sets;
    const uint32_t* seeds;
    uint32_t n_sets;
    uint64_t skip, n;
    uint32_t* out;
    int kind;
    int tid, nthreads;
} bulk_job;

static void* bulk_worker(void* arg) {
    bulk_job* j = (bulk_job*)arg;
    oracle_mtgp g;
    for (uint32_t s = (uint32_t)j->tid; s < j->n_sets; s += (uint32_t)j->nthreads) {
        oracle_mtgp_init(&g, &j->sets[s], j->seeds[s]);
        oracle_mtgp_skip(&g, j->skip);
        oracle_mtgp_fill(&g, j->out + (size_t)s * j->n, (size_t)j->n, j->kind);
    }
    return NULL;
}

double oracle_mtgp_bulk(const oracle_mtgp_params* sets, const uint32_t* seeds, uint32_t n_sets,
                        uint64_t skip, uint64_t n, uint32_t* out, int kind, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 1024) threads = 1024;
    pthread_t th[1024];
    bulk_job jobs[1024];
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (bulk_job){sets, seeds, n_sets, skip, n, out, kind, t, threads};
        pthread_create(&th[t], NULL, bulk_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* ---- streaming checksums (full-volume parity fixtures; no output buffer) ----
 * The cumulative {sum64, xor32} of the u32 words (and, with_float, of the [1,2) and (0,1] bit
 * patterns derived from them exactly as oracle_mtgp_fill does), recorded after every rec_every
 * words of every stream. Two forms of the same Appendix-A step:
 *   - ck_scalar: step() above, one word at a time (the reference form);
 *   - ck_avx512: 16 consecutive steps at once. Any d <= N - pos consecutive steps are
 *     independent (SURVEY.md App. A "Parallelism"), so with N - pos >= 16 one 512-bit vector
 *     computes x[i+N .. i+N+16) from x[i .. i+pos+16), all of which earlier vectors produced.
 *     The 16-entry tables are one vpermd each (it reads the low 4 bits of every index lane,
 *     i.e. tbl[y & 15]). The state is a linear buffer of N + B words, slid down every B words.
 * tests/test_oracle.py checks the AVX-512 form against oracle_mtgp_fill word-for-word sums.
 * Sets are handed to threads dynamically (one stream per task). */
typedef struct ck_acc {
    uint64_t su, s12, s01;
    uint32_t xu, x12, x01;
} ck_acc;

static inline void ck_word(ck_acc* a, uint32_t u, int with_float) {
    a->su += u;
    a->xu ^= u;
    if (with_float) {
        const uint32_t fb = (u >> 9) | 0x3F800000u;
        float f;
        memcpy(&f, &fb, 4);
        f = 2.0f - f;
        uint32_t gb;
        memcpy(&gb, &f, 4);
        a->s12 += fb; a->x12 ^= fb;
        a->s01 += gb; a->x01 ^= gb;
    }
}

static void ck_record(oracle_stream_ck* o, const ck_acc* a) {
    o->sum[0] = a->su; o->sum[1] = a->s12; o->sum[2] = a->s01;
    o->xr[0] = a->xu; o->xr[1] = a->x12; o->xr[2] = a->x01;
    o->pad = 0;
}

static void ck_scalar(oracle_mtgp* g, uint64_t rec_every, uint32_t n_rec, int with_float, oracle_stream_ck* out) {
    ck_acc a = {0, 0, 0, 0, 0, 0};
    for (uint32_t k = 0; k < n_rec; ++k) {
        for (uint64_t w = 0; w < rec_every; ++w) ck_word(&a, step(g), with_float);
        ck_record(&out[k], &a);
    }
}

#if defined(__x86_64__)
#include <immintrin.h>
#define CK_B 8192u /* words per slide of the linear buffer */

__attribute__((target("avx512f"))) static uint32_t xor_lanes(__m512i v) {
    uint32_t l[16], r = 0;
    _mm512_storeu_si512((void*)l, v);
    for (int q = 0; q < 16; ++q) r ^= l[q];
    return r;
}

__attribute__((target("avx512f"))) static inline void ck_avx512_t(const oracle_mtgp* g0, uint64_t rec_every,
                                                                 uint32_t n_rec, const int with_float,
                                                                 oracle_stream_ck* out, uint32_t* buf) {
    const uint32_t n = g0->n, pos = g0->p.pos;
    oracle_mtgp_window(g0, buf);
    const __m512i vmask = _mm512_set1_epi32((int)g0->p.mask);
    const __m512i vtbl = _mm512_loadu_si512((const void*)g0->p.tbl);
    const __m512i vtmp = _mm512_loadu_si512((const void*)g0->p.tmp_tbl);
    const __m128i sh1 = _mm_cvtsi32_si128((int)g0->p.sh1), sh2 = _mm_cvtsi32_si128((int)g0->p.sh2);
    const __m512i flt_or = _mm512_set1_epi32(0x3F800000), two = _mm512_castps_si512(_mm512_set1_ps(2.0f));
    __m512i su = _mm512_setzero_si512(), s12 = su, s01 = su, xu = su, x12 = su, x01 = su;
    uint32_t i = 0;  /* buf[i] = x[done - ...]: the oldest window word of the next step */
    for (uint32_t k = 0; k < n_rec; ++k) {
        /* 16 | rec_every is required by the caller, so records fall on vector boundaries */
        for (uint64_t w = 0; w < rec_every; w += 16) {
            if (i == CK_B) {  /* slide: keep the last N words */
                memmove(buf, buf + CK_B, sizeof(uint32_t) * n);
                i = 0;
            }
            const uint32_t* q = buf + i;
            const __m512i a = _mm512_loadu_si512((const void*)q);
            const __m512i b = _mm512_loadu_si512((const void*)(q + 1));
            const __m512i c = _mm512_loadu_si512((const void*)(q + pos));
            __m512i t = _mm512_loadu_si512((const void*)(q + pos - 1));
            __m512i x = _mm512_xor_si512(_mm512_and_si512(a, vmask), b);
            x = _mm512_xor_si512(x, _mm512_sll_epi32(x, sh1));
            const __m512i y = _mm512_xor_si512(x, _mm512_srl_epi32(c, sh2));
            const __m512i r = _mm512_xor_si512(y, _mm512_permutexvar_epi32(y, vtbl));
            t = _mm512_xor_si512(t, _mm512_srli_epi32(t, 16));
            t = _mm512_xor_si512(t, _mm512_srli_epi32(t, 8));
            const __m512i o = _mm512_xor_si512(r, _mm512_permutexvar_epi32(t, vtmp));
            _mm512_storeu_si512((void*)(buf + i + n), r);
            i += 16;
            su = _mm512_add_epi64(su, _mm512_cvtepu32_epi64(_mm512_castsi512_si256(o)));
            su = _mm512_add_epi64(su, _mm512_cvtepu32_epi64(_mm512_extracti64x4_epi64(o, 1)));
            xu = _mm512_xor_si512(xu, o);
            if (with_float) {
                const __m512i f = _mm512_or_si512(_mm512_srli_epi32(o, 9), flt_or);
                const __m512i h =
                    _mm512_castps_si512(_mm512_sub_ps(_mm512_castsi512_ps(two), _mm512_castsi512_ps(f)));
                s12 = _mm512_add_epi64(s12, _mm512_cvtepu32_epi64(_mm512_castsi512_si256(f)));
                s12 = _mm512_add_epi64(s12, _mm512_cvtepu32_epi64(_mm512_extracti64x4_epi64(f, 1)));
                s01 = _mm512_add_epi64(s01, _mm512_cvtepu32_epi64(_mm512_castsi512_si256(h)));
                s01 = _mm512_add_epi64(s01, _mm512_cvtepu32_epi64(_mm512_extracti64x4_epi64(h, 1)));
                x12 = _mm512_xor_si512(x12, f);
                x01 = _mm512_xor_si512(x01, h);
            }
        }
        oracle_stream_ck* rc = &out[k];
        rc->sum[0] = (uint64_t)_mm512_reduce_add_epi64(su);
        rc->sum[1] = (uint64_t)_mm512_reduce_add_epi64(s12);
        rc->sum[2] = (uint64_t)_mm512_reduce_add_epi64(s01);
        rc->xr[0] = xor_lanes(xu);
        rc->xr[1] = xor_lanes(x12);
        rc->xr[2] = xor_lanes(x01);
        rc->pad = 0;
    }
}

__attribute__((target("avx512f"))) static void ck_avx512(const oracle_mtgp* g0, uint64_t rec_every, uint32_t n_rec,
                                                         int with_float, oracle_stream_ck* out) {
    static __thread uint32_t tbuf[4096 + CK_B + 64] __attribute__((aligned(64)));
    uint32_t* buf = tbuf + (16 - g0->n % 16) % 16;  /* the new words' stores are 64-byte aligned */
    if (with_float)
        ck_avx512_t(g0, rec_every, n_rec, 1, out, buf);
    else
        ck_avx512_t(g0, rec_every, n_rec, 0, out, buf);
}
#endif

typedef struct ck_job {
    const oracle_mtgp_params* sets;
    const uint32_t* seeds;
    uint32_t n_sets;
    uint64_t rec_every;
    uint32_t n_rec;
    int with_float, force_scalar;
    oracle_stream_ck* out;
    uint32_t* next;  /* shared task counter */
} ck_job;

static void* ck_worker(void* arg) {
    ck_job* j = (ck_job*)arg;
    oracle_mtgp g;
    for (;;) {
        const uint32_t s = __atomic_fetch_add(j->next, 1u, __ATOMIC_RELAXED);
        if (s >= j->n_sets) break;
        oracle_mtgp_init(&g, &j->sets[s], j->seeds[s]);
        oracle_stream_ck* o = &j->out[(size_t)s * j->n_rec];
#if defined(__x86_64__)
        if (!j->force_scalar && g.n >= g.p.pos + 16 && j->rec_every % 16 == 0 && __builtin_cpu_supports("avx512f")) {
            ck_avx512(&g, j->rec_every, j->n_rec, j->with_float, o);
            continue;
        }
#endif
        ck_scalar(&g, j->rec_every, j->n_rec, j->with_float, o);
    }
    return NULL;
}

double oracle_mtgp_cksum_stream(const oracle_mtgp_params* sets, const uint32_t* seeds, uint32_t n_sets,
                                uint64_t rec_every, uint32_t n_rec, int flags, oracle_stream_ck* out,
                                int threads) {
    if (threads < 1) threads = 1;
    if (threads > 1024) threads = 1024;
    pthread_t th[1024];
    ck_job job = {sets, seeds, n_sets, rec_every, n_rec, flags & 1, (flags >> 1) & 1, out, NULL};
    uint32_t next = 0;
    job.next = &next;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, ck_worker, &job);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* ---- CPU baseline: every stream filled through a reused fill() buffer (WordSource::fill) ----
 * Threads take streams dynamically; each stream is seeded, then filled `chunk` words at a time
 * into the thread's private buffer (word_source.hpp:21-25 semantics: the caller owns the span)
 * until it has produced n words. The buffer's checksum is folded into *sink so no work can be
 * elided. Returns seconds. */
typedef struct fill_job {
    const oracle_mtgp_params* sets;
    const uint32_t* seeds;
    uint32_t n_sets;
    uint64_t n, chunk;
    int kind;
    uint32_t* next;
    uint64_t sink;
} fill_job;

static void* fill_worker(void* arg) {
    fill_job* j = (fill_job*)arg;
    uint32_t* buf = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)j->chunk);
    oracle_mtgp g;
    uint64_t acc = 0;
    for (;;) {
        const uint32_t s = __atomic_fetch_add(j->next, 1u, __ATOMIC_RELAXED);
        if (s >= j->n_sets) break;
        oracle_mtgp_init(&g, &j->sets[s], j->seeds[s]);
        for (uint64_t done = 0; done < j->n; done += j->chunk) {
            const uint64_t c = j->n - done < j->chunk ? j->n - done : j->chunk;
            oracle_mtgp_fill(&g, buf, (size_t)c, j->kind);
            acc += buf[c - 1];
        }
    }
    free(buf);
    __atomic_fetch_add(&j->sink, acc, __ATOMIC_RELAXED);
    return NULL;
}

double oracle_mtgp_fill_bulk(const oracle_mtgp_params* sets, const uint32_t* seeds, uint32_t n_sets, uint64_t n,
                             uint64_t chunk, int kind, int threads, uint64_t* sink) {
    if (threads < 1) threads = 1;
    if (threads > 1024) threads = 1024;
    if (chunk < 1) chunk = 1;
    pthread_t th[1024];
    uint32_t next = 0;
    fill_job job = {sets, seeds, n_sets, n, chunk, kind, &next, 0};
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, fill_worker, &job);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if (sink) *sink = job.sink;
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}
