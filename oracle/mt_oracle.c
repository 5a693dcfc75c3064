/*
 * mt_oracle.c -- restatement of the reference's generic MT engine (Engine::mt).
 * TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 *   temper        proj/src/generator.cpp:7-13
 *   untemper      proj/src/generator.cpp:18-35
 *   seeding       proj/src/generator.cpp:37-52  (x0 = seed; xi = 1812433253*(x_{i-1}^(x_{i-1}>>30)) + i)
 *   refill        proj/src/generator.cpp:68-88  (three loops; k+m<n, k+m>=n, last word wraps)
 *   next_u32      proj/include/twistsieve/generator.hpp:33-36
 *   mt19937 preset proj/src/params.cpp:63-77
 *   splitmix64 / derive_seed proj/src/word_source.cpp:18-27
 */
#include "oracle.h"

void oracle_mt19937_params(oracle_mt_params* p) {
    p->mexp = 19937;
    p->n = 624;
    p->m = 397;
    p->r = 31;
    p->a = 0x9908B0DFu;
    p->b = 0x9D2C5680u;
    p->c = 0xEFC60000u;
    p->u = 11;
    p->s = 7;
    p->t = 15;
    p->l = 18;
}

uint32_t oracle_mt_temper(uint32_t y, const oracle_mt_params* p) {
    y ^= y >> p->u;
    y ^= (y << p->s) & p->b;
    y ^= (y << p->t) & p->c;
    y ^= y >> p->l;
    return y;
}

static uint32_t undo_right(uint32_t v, uint32_t shift) {
    uint32_t res = v;
    for (uint32_t done = shift; done < 32; done += shift) res = v ^ (res >> shift);
    return res;
}

static uint32_t undo_left(uint32_t v, uint32_t shift, uint32_t mask) {
    uint32_t res = v;
    for (uint32_t done = shift; done < 32; done += shift) res = v ^ ((res << shift) & mask);
    return res;
}

uint32_t oracle_mt_untemper(uint32_t y, const oracle_mt_params* p) {
    y = undo_right(y, p->l);
    y = undo_left(y, p->t, p->c);
    y = undo_left(y, p->s, p->b);
    y = undo_right(y, p->u);
    return y;
}

int oracle_mt_init(oracle_mt* g, const oracle_mt_params* p, uint32_t seed) {
    if (p->n < 2 || p->n > 2048 || p->m < 1 || p->m >= p->n || p->r >= 32) return -1;
    g->p = *p;
    g->st[0] = seed;
    for (uint32_t i = 1; i < p->n; ++i)
        g->st[i] = 1812433253u * (g->st[i - 1] ^ (g->st[i - 1] >> 30)) + i;
    g->index = p->n;
    return 0;
}

static void refill(oracle_mt* g) {
    const uint32_t n = g->p.n, m = g->p.m;
    const uint32_t upper = 0xFFFFFFFFu << g->p.r;
    const uint32_t lower = ~upper;
    const uint32_t a = g->p.a;
    uint32_t* st = g->st;
    uint32_t k = 0;
    for (; k + m < n; ++k) {
        const uint32_t y = (st[k] & upper) | (st[k + 1] & lower);
        st[k] = st[k + m] ^ (y >> 1) ^ ((y & 1u) ? a : 0u);
    }
    for (; k + 1 < n; ++k) {
        const uint32_t y = (st[k] & upper) | (st[k + 1] & lower);
        st[k] = st[k + m - n] ^ (y >> 1) ^ ((y & 1u) ? a : 0u);
    }
    const uint32_t y = (st[n - 1] & upper) | (st[0] & lower);
    st[n - 1] = st[m - 1] ^ (y >> 1) ^ ((y & 1u) ? a : 0u);
    g->index = 0;
}

void oracle_mt_fill(oracle_mt* g, uint32_t* out, size_t n) {
    for (size_t j = 0; j < n; ++j) {
        if (g->index >= g->p.n) refill(g);
        out[j] = oracle_mt_temper(g->st[g->index++], &g->p);
    }
}

uint64_t oracle_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

uint32_t oracle_derive_seed(uint64_t source, uint32_t j) {
    return (uint32_t)oracle_splitmix64(source + j);
}
