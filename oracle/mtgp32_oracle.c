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
