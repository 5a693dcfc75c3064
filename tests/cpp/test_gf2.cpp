// test_gf2.cpp -- CPU test of the jump-ahead algebra (csrc/gf2.cpp) against the oracle.
// Built and run by tests/test_jump_cpu.py:
//   g++ -O2 -mpclmul -msse4.1 -I include -I paper_1501_07701_b200/csrc -I oracle
//       tests/cpp/test_gf2.cpp paper_1501_07701_b200/csrc/gf2.cpp oracle/liboracle.so
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <string>

#include "gf2.h"
#include "oracle.h"
#include "sha1.h"

using namespace mtgpb::gf2;

static int fails = 0;
#define CHECK(c)                                                        \
    do {                                                                \
        if (!(c)) {                                                     \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);    \
            ++fails;                                                    \
        }                                                               \
    } while (0)

// Parse one params record from argv-provided file: mexp pos sh1 sh2 tbl[16] tmp[16] mask
static bool read_params(FILE* f, oracle_mtgp_params* p) {
    if (fscanf(f, "%u %u %u %u", &p->mexp, &p->pos, &p->sh1, &p->sh2) != 4) return false;
    for (int i = 0; i < 16; ++i)
        if (fscanf(f, "%u", &p->tbl[i]) != 1) return false;
    for (int i = 0; i < 16; ++i)
        if (fscanf(f, "%u", &p->tmp_tbl[i]) != 1) return false;
    if (fscanf(f, "%u", &p->mask) != 1) return false;
    for (int i = 0; i < 16; ++i) p->flt_tmp_tbl[i] = (p->tmp_tbl[i] >> 9) | 0x3F800000u;
    return true;
}

// state words x_0.. of the sequence (not outputs): x_0..x_{N-1} = window, then generated.
static std::vector<uint32_t> state_sequence(const oracle_mtgp_params* p, uint32_t seed, size_t len) {
    oracle_mtgp g;
    oracle_mtgp_init(&g, p, seed);
    std::vector<uint32_t> x(len);
    oracle_mtgp_window(&g, x.data());
    const uint32_t n = g.n;
    for (size_t j = n; j < len; ++j) {
        uint32_t dummy;
        oracle_mtgp_fill(&g, &dummy, 1, 0);
        // after one step the newest word is the last element of the window
        uint32_t w[4096];
        oracle_mtgp_window(&g, w);
        x[j] = w[n - 1];
    }
    return x;
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::printf("usage: test_gf2 params.txt\n");
        return 2;
    }
    // 1. small algebra identities
    {
        Poly a, b, p;
        a.set(0); a.set(5); a.set(70); a.set(130);
        b.set(1); b.set(64); b.set(99);
        p.set(0); p.set(3); p.set(200);  // x^200 + x^3 + 1
        Modulus md(p);
        Poly q, r;
        divmod(mul(a, b), p, &q, &r);
        CHECK(md.mulmod(a, b) == r);
        CHECK(add(mul(q, p), r) == mul(a, b));
        // x^(e1+e2) = x^e1 x^e2
        CHECK(md.mulmod(md.x_pow(12345), md.x_pow(777)) == md.x_pow(13122));
        // big operands exercise the Karatsuba path
        Poly big1, big2;
        for (int i = 0; i < 9000; i += 7) big1.set(i);
        for (int i = 3; i < 9000; i += 11) big2.set(i);
        Poly m1 = mul(big1, big2);
        // schoolbook check of a few coefficients
        for (int k : {0, 3, 10, 4500, 9000, 17990}) {
            int c = 0;
            for (int i = 0; i <= k; ++i) c ^= big1.coeff(i) & big2.coeff(k - i);
            CHECK(m1.coeff(k) == (bool)c);
        }
    }
    // 1b. Rabin irreducibility (the reference's is_irreducible, gf2poly.cpp:342-383) on known
    //     cases: primitive trinomials of Mersenne exponents, and products of two factors
    {
        auto tri = [](int n, int k) {
            Poly t;
            t.set(0);
            t.set(k);
            t.set(n);
            return t;
        };
        CHECK(is_irreducible(tri(89, 38)));
        CHECK(is_irreducible(tri(127, 1)));
        CHECK(is_irreducible(tri(521, 32)));
        CHECK(is_irreducible(tri(607, 105)));
        CHECK(is_irreducible(tri(1279, 216)));
        CHECK(!is_irreducible(tri(8, 0)));                       // x^8 + 1 = (x + 1)^8
        CHECK(!is_irreducible(mul(tri(89, 38), tri(127, 1))));   // composite, no small factor
        CHECK(!is_irreducible(mul(tri(127, 1), tri(127, 1))));   // a square
        CHECK(!is_irreducible(tri(200, 3)));                     // x^200 + x^3 + 1 has degree 200
        Poly x1;  // x + 1
        x1.set(0);
        x1.set(1);
        CHECK(is_irreducible(x1));
        // the reference digest of x^2 + x + 1 (coefficient count 3, byte 0x07)
        Poly q;
        q.set(0); q.set(1); q.set(2);
        CHECK(reference_digest(q).size() == 40);
    }
    // 2. MTGP sets from the file: charpoly via BM, annihilation, jump = direct generation
    FILE* f = std::fopen(argv[1], "r");
    if (!f) return 2;
    oracle_mtgp_params prm;
    int nset = 0;
    while (read_params(f, &prm)) {
        const uint32_t M = prm.mexp, N = oracle_mtgp_n(M);
        const size_t len = 2 * (size_t)M + N + 64;
        std::vector<uint32_t> x = state_sequence(&prm, 1234 + nset, len);
        std::vector<uint64_t> bits((2 * M + 63) / 64 + 1, 0);
        for (size_t k = 0; k < 2 * (size_t)M; ++k)
            if (x[k + 1] >> 31) bits[k >> 6] |= 1ull << (k & 63);
        Poly P = berlekamp_massey(bits, 2 * (size_t)M);
        std::printf("set %d mexp %u: BM degree %d\n", nset, M, P.degree());
        {
            const auto t0 = std::chrono::steady_clock::now();
            const bool irr = is_irreducible(P);
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            std::printf("  irreducible %d (%.3f s)\n", (int)irr, s);
        }
        {
            std::string coeffs(P.degree() + 1, '0');
            for (int i = 0; i <= P.degree(); ++i)
                if (P.coeff(i)) coeffs[i] = '1';
            std::printf("  digest %s\n", mtgpb::sha1_hex(coeffs).c_str());
        }
        // annihilation on every bit: sum_i P_i x_{i+j} == 0, j>=1 (j=0: live bits only)
        bool ok = true;
        for (uint32_t j = 0; j < N && ok; ++j) {
            uint32_t acc = 0;
            for (int i = 0; i <= P.degree(); ++i)
                if (P.coeff(i)) acc ^= x[i + j];
            if (j == 0) acc &= prm.mask;
            ok = acc == 0;
        }
        std::printf("  annihilates all bits: %d\n", (int)ok);
        if (nset == 0) CHECK(P.degree() == (int)M);
        if (ok) {
            Modulus md(P);
            for (uint64_t o : {(uint64_t)1, (uint64_t)77, (uint64_t)M + 5, (uint64_t)100000, (uint64_t)1234567}) {
                Poly q = md.x_pow(o);
                oracle_mtgp g;
                oracle_mtgp_init(&g, &prm, 1234 + nset);
                oracle_mtgp_skip(&g, o);
                uint32_t want[4096];
                oracle_mtgp_window(&g, want);
                bool eq = true;
                for (uint32_t j = 0; j < N; ++j) {
                    uint32_t acc = 0;
                    for (int i = 0; i <= q.degree(); ++i)
                        if (q.coeff(i)) acc ^= x[i + j];
                    if (j == 0) eq = eq && ((acc ^ want[0]) & prm.mask) == 0;
                    else eq = eq && acc == want[j];
                }
                std::printf("  jump %llu: %s\n", (unsigned long long)o, eq ? "ok" : "MISMATCH");
                CHECK(eq);
            }
        }
        ++nset;
    }
    std::fclose(f);
    std::printf("%s (%d failures)\n", fails ? "FAILED" : "PASSED", fails);
    return fails ? 1 : 0;
}
