// gf2.h -- host-side GF(2)[x] arithmetic for MTGP32 jump-ahead (charpoly + x^o mod P).
//
// The reference has the same building blocks for its classic-MT dynamic creator
// (proj/src/gf2poly.cpp:255-270 poly_pow_mod, :272-340 berlekamp_massey); this is a separate,
// PCLMULQDQ-based implementation sized for degree 11213..44497 polynomials: Barrett reduction
// with two carry-less products instead of shift-and-XOR long division.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace mtgpb {
namespace gf2 {

// Bit i of w[i/64] is the coefficient of x^i.
struct Poly {
    std::vector<uint64_t> w;
    int degree() const;  // -1 for the zero polynomial
    bool coeff(int i) const { return i >= 0 && (size_t)(i >> 6) < w.size() && ((w[i >> 6] >> (i & 63)) & 1); }
    void set(int i) {
        if ((size_t)(i >> 6) >= w.size()) w.resize((i >> 6) + 1, 0);
        w[i >> 6] |= 1ull << (i & 63);
    }
    void trim();
    bool operator==(const Poly& o) const;
};

Poly mul(const Poly& a, const Poly& b);
Poly square(const Poly& a);  // a^2: bit spreading (one carry-less square per word)
Poly add(const Poly& a, const Poly& b);
Poly shift_left(const Poly& a, int k);
// quotient and remainder by long division (O(deg^2/64)); used once per set
void divmod(const Poly& a, const Poly& p, Poly* q, Poly* r);
Poly gcd(Poly a, Poly b);

// Berlekamp-Massey over a bit sequence s[0..n) (bit k of bits[k/64]). Returns the
// characteristic polynomial P (monic, degree = linear complexity L) with
// sum_i P_i s_{i+j} = 0 for all valid j.
Poly berlekamp_massey(const std::vector<uint64_t>& bits, size_t n);

// Barrett context for reduction modulo a fixed P of degree M.
struct Modulus {
    Poly p;
    Poly mu;  // floor(x^(2M) / P)
    int m = 0;
    explicit Modulus(const Poly& p_);
    Poly reduce(const Poly& a) const;  // deg a < 2M
    Poly mulmod(const Poly& a, const Poly& b) const;
    Poly x_pow(uint64_t e) const;  // x^e mod P
    Poly sqrmod(const Poly& a) const { return reduce(square(a)); }
};

// Rabin's test: p of degree d >= 1 is irreducible iff x^(2^d) = x (mod p) and
// gcd(x^(2^(d/q)) - x, p) = 1 for every prime q | d; like the reference's is_irreducible
// (proj/src/gf2poly.cpp:342-383) also at k = 1..20 as a small-factor sieve. Up to d squarings.
bool is_irreducible(const Poly& p);

// The reference's poly_digest (proj/src/dynamic_creator.cpp:9-31): SHA-1 of the coefficient
// count (degree + 1, 0 for the zero polynomial) as 8 little-endian bytes, then the coefficient
// bits as little-endian bytes; lowercase hex.
std::string reference_digest(const Poly& p);

}  // namespace gf2
}  // namespace mtgpb
