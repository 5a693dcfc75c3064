// gf2.cpp -- see gf2.h.
#include "gf2.h"
#include "sha1.h"

#include <algorithm>
#include <cstring>

#if defined(__PCLMUL__)
#include <smmintrin.h>
#include <wmmintrin.h>
#endif

namespace mtgpb {
namespace gf2 {

int Poly::degree() const {
    for (size_t i = w.size(); i-- > 0;)
        if (w[i]) return (int)(i * 64 + 63 - __builtin_clzll(w[i]));
    return -1;
}

void Poly::trim() {
    while (!w.empty() && w.back() == 0) w.pop_back();
}

bool Poly::operator==(const Poly& o) const {
    Poly a = *this, b = o;
    a.trim();
    b.trim();
    return a.w == b.w;
}

static inline void clmul64(uint64_t a, uint64_t b, uint64_t* lo, uint64_t* hi) {
#if defined(__PCLMUL__)
    __m128i r = _mm_clmulepi64_si128(_mm_cvtsi64_si128((long long)a), _mm_cvtsi64_si128((long long)b), 0);
    *lo = (uint64_t)_mm_cvtsi128_si64(r);
    *hi = (uint64_t)_mm_extract_epi64(r, 1);
#else
    uint64_t l = 0, h = 0;
    for (int i = 0; i < 64; ++i)
        if ((b >> i) & 1) {
            l ^= a << i;
            if (i) h ^= a >> (64 - i);
        }
    *lo = l;
    *hi = h;
#endif
}

// r[0..na+nb) = a * b, schoolbook on 64-bit limbs (Karatsuba above a threshold).
static void mul_raw(const uint64_t* a, size_t na, const uint64_t* b, size_t nb, uint64_t* r) {
    std::memset(r, 0, sizeof(uint64_t) * (na + nb));
    if (na >= 64 && nb >= 64 && na == nb && (na & 1) == 0) {
        // one Karatsuba level: (a1 X + a0)(b1 X + b0), X = x^(64h)
        const size_t h = na / 2;
        std::vector<uint64_t> z0(2 * h), z2(2 * h), z1(2 * h), sa(h), sb(h);
        mul_raw(a, h, b, h, z0.data());
        mul_raw(a + h, h, b + h, h, z2.data());
        for (size_t i = 0; i < h; ++i) {
            sa[i] = a[i] ^ a[h + i];
            sb[i] = b[i] ^ b[h + i];
        }
        mul_raw(sa.data(), h, sb.data(), h, z1.data());
        for (size_t i = 0; i < 2 * h; ++i) {
            z1[i] ^= z0[i] ^ z2[i];
            r[i] ^= z0[i];
            r[i + 2 * h] ^= z2[i];
            r[i + h] ^= z1[i];
        }
        return;
    }
    for (size_t i = 0; i < na; ++i) {
        const uint64_t ai = a[i];
        if (!ai) continue;
        for (size_t j = 0; j < nb; ++j) {
            uint64_t lo, hi;
            clmul64(ai, b[j], &lo, &hi);
            r[i + j] ^= lo;
            r[i + j + 1] ^= hi;
        }
    }
}

Poly mul(const Poly& a, const Poly& b) {
    Poly r;
    if (a.w.empty() || b.w.empty()) return r;
    size_t na = a.w.size(), nb = b.w.size();
    if (na == nb && na >= 64 && (na & 1)) {
        // pad to even for the Karatsuba split
        Poly a2 = a, b2 = b;
        a2.w.push_back(0);
        b2.w.push_back(0);
        r.w.resize(2 * (na + 1));
        mul_raw(a2.w.data(), na + 1, b2.w.data(), nb + 1, r.w.data());
    } else {
        r.w.resize(na + nb);
        mul_raw(a.w.data(), na, b.w.data(), nb, r.w.data());
    }
    r.trim();
    return r;
}

Poly square(const Poly& a) {
    Poly r;
    r.w.assign(2 * a.w.size(), 0);
    for (size_t i = 0; i < a.w.size(); ++i) clmul64(a.w[i], a.w[i], &r.w[2 * i], &r.w[2 * i + 1]);
    r.trim();
    return r;
}

Poly add(const Poly& a, const Poly& b) {
    Poly r = a.w.size() >= b.w.size() ? a : b;
    const Poly& s = a.w.size() >= b.w.size() ? b : a;
    for (size_t i = 0; i < s.w.size(); ++i) r.w[i] ^= s.w[i];
    r.trim();
    return r;
}

Poly shift_left(const Poly& a, int k) {
    Poly r;
    if (a.w.empty()) return r;
    const int q = k >> 6, s = k & 63;
    r.w.assign(a.w.size() + q + 1, 0);
    for (size_t i = 0; i < a.w.size(); ++i) {
        r.w[i + q] ^= a.w[i] << s;
        if (s) r.w[i + q + 1] ^= a.w[i] >> (64 - s);
    }
    r.trim();
    return r;
}

static Poly shift_right(const Poly& a, int k) {
    Poly r;
    const int q = k >> 6, s = k & 63;
    if ((int)a.w.size() <= q) return r;
    r.w.assign(a.w.size() - q, 0);
    for (size_t i = 0; i < r.w.size(); ++i) {
        r.w[i] = a.w[i + q] >> s;
        if (s && i + q + 1 < a.w.size()) r.w[i] |= a.w[i + q + 1] << (64 - s);
    }
    r.trim();
    return r;
}

static Poly low_bits(const Poly& a, int k) {
    Poly r = a;
    const size_t words = (size_t)(k + 63) / 64;
    if (r.w.size() > words) r.w.resize(words);
    if ((k & 63) && r.w.size() == words) r.w[words - 1] &= (1ull << (k & 63)) - 1;
    r.trim();
    return r;
}

void divmod(const Poly& a, const Poly& p, Poly* qo, Poly* ro) {
    Poly r = a;
    r.trim();
    const int dp = p.degree();
    Poly q;
    int dr = r.degree();
    while (dr >= dp) {
        const int sft = dr - dp;
        q.set(sft);
        // r ^= p << sft
        const int wq = sft >> 6, s = sft & 63;
        for (size_t i = 0; i < p.w.size(); ++i) {
            r.w[i + wq] ^= p.w[i] << s;
            if (s && i + wq + 1 < r.w.size()) r.w[i + wq + 1] ^= p.w[i] >> (64 - s);
        }
        // find the new degree, scanning down from dr
        int d = dr - 1;
        while (d >= 0 && !r.coeff(d)) {
            if ((d & 63) == 63 && r.w[d >> 6] == 0) {
                d -= 64;
                continue;
            }
            --d;
        }
        dr = d;
    }
    r.trim();
    q.trim();
    if (qo) *qo = q;
    if (ro) *ro = r;
}

Poly gcd(Poly a, Poly b) {
    a.trim();
    b.trim();
    while (!b.w.empty()) {
        Poly r;
        divmod(a, b, nullptr, &r);
        a = std::move(b);
        b = std::move(r);
    }
    return a;
}

Poly berlekamp_massey(const std::vector<uint64_t>& bits, size_t n) {
    // reversed sequence R: bit (n-1-k) of R = s_k, so sum_{i=0..L} c_i s_{t-i} is
    // parity(C & (R >> (n-1-t))).
    const size_t nw = (n + 63) / 64;
    std::vector<uint64_t> R(nw + 2, 0);
    for (size_t k = 0; k < n; ++k)
        if ((bits[k >> 6] >> (k & 63)) & 1) {
            const size_t b = n - 1 - k;
            R[b >> 6] |= 1ull << (b & 63);
        }
    std::vector<uint64_t> C(nw + 2, 0), B(nw + 2, 0), T;
    C[0] = B[0] = 1;
    size_t L = 0;
    size_t m = 1;
    for (size_t t = 0; t < n; ++t) {
        const size_t off = n - 1 - t;
        const size_t q = off >> 6, s = off & 63;
        const size_t cw = L / 64 + 1;
        uint64_t acc = 0;
        for (size_t i = 0; i < cw; ++i) {
            uint64_t rw = R[q + i] >> s;
            if (s && q + i + 1 < R.size()) rw |= R[q + i + 1] << (64 - s);
            acc ^= C[i] & rw;
        }
        const int d = __builtin_parityll(acc);
        if (!d) {
            ++m;
            continue;
        }
        const bool grow = 2 * L <= t;
        if (grow) T = C;
        // C ^= B << m
        const size_t mq = m >> 6, ms = m & 63;
        const size_t bw = std::min(B.size(), C.size() - mq);
        for (size_t i = 0; i < bw; ++i) {
            if (!B[i]) continue;
            C[i + mq] ^= B[i] << ms;
            if (ms && i + mq + 1 < C.size()) C[i + mq + 1] ^= B[i] >> (64 - ms);
        }
        if (grow) {
            L = t + 1 - L;
            B = T;
            m = 1;
        } else {
            ++m;
        }
    }
    // P(x) = x^L C(1/x)
    Poly P;
    P.w.assign(L / 64 + 1, 0);
    for (size_t i = 0; i <= L; ++i)
        if ((C[i >> 6] >> (i & 63)) & 1) {
            const size_t j = L - i;
            P.w[j >> 6] |= 1ull << (j & 63);
        }
    P.trim();
    return P;
}

Modulus::Modulus(const Poly& p_) : p(p_) {
    p.trim();
    m = p.degree();
    Poly x2m;
    x2m.set(2 * m);
    divmod(x2m, p, &mu, nullptr);
}

Poly Modulus::reduce(const Poly& a) const {
    if (a.degree() < m) return a;
    const Poly hi = shift_right(a, m);
    const Poly t = shift_right(mul(hi, mu), m);
    Poly r = add(a, mul(t, p));
    return low_bits(r, m);
}

Poly Modulus::mulmod(const Poly& a, const Poly& b) const { return reduce(mul(a, b)); }

Poly Modulus::x_pow(uint64_t e) const {
    Poly r;
    r.set(0);
    if (e == 0) return r;
    int top = 63 - __builtin_clzll(e);
    for (int b = top; b >= 0; --b) {
        r = reduce(mul(r, r));
        if ((e >> b) & 1) {
            r = shift_left(r, 1);
            if (r.degree() == m) r = add(r, p);
        }
    }
    return r;
}

}  // namespace gf2
}  // namespace mtgpb

namespace mtgpb {
namespace gf2 {

bool is_irreducible(const Poly& p) {
    const int d = p.degree();
    if (d < 1) return false;
    if (d == 1) return true;
    // k = d / q for the distinct primes q | d, plus k = 1..20 as a sieve for small factors
    // (gcd(x^(2^k) - x, p) = 1 for every k < d when p is irreducible, so the answer is unchanged;
    // a reducible p is usually rejected after a few squarings instead of d)
    std::vector<int> checkpoints;
    for (int k = 1; k <= std::min(20, d - 1); ++k) checkpoints.push_back(k);
    int rem = d;
    for (int q = 2; q * q <= rem; ++q)
        if (rem % q == 0) {
            checkpoints.push_back(d / q);
            while (rem % q == 0) rem /= q;
        }
    if (rem > 1) checkpoints.push_back(d / rem);
    std::sort(checkpoints.begin(), checkpoints.end());
    checkpoints.erase(std::unique(checkpoints.begin(), checkpoints.end()), checkpoints.end());
    const Modulus md(p);
    Poly x;
    x.set(1);
    Poly u = md.reduce(x);  // x mod p (d >= 2: x itself)
    size_t next = 0;
    for (int k = 1; k <= d; ++k) {
        u = md.sqrmod(u);  // x^(2^k) mod p
        while (next < checkpoints.size() && checkpoints[next] == k) {
            ++next;
            Poly g = gcd(add(u, x), p);
            g.trim();
            if (g.degree() != 0) return false;
        }
    }
    Poly ux = add(u, x);
    ux.trim();
    return ux.degree() < 0;
}

std::string reference_digest(const Poly& p) {
    const int d = p.degree();
    const uint64_t nbits = d < 0 ? 0 : (uint64_t)d + 1;
    std::string payload(8, '\0');
    for (int i = 0; i < 8; ++i) payload[i] = static_cast<char>((nbits >> (8 * i)) & 0xff);
    const size_t nbytes = d < 0 ? 0 : (size_t)d / 8 + 1;
    for (size_t i = 0; i < nbytes; ++i) payload.push_back(static_cast<char>((p.w[i / 8] >> (8 * (i % 8))) & 0xff));
    return sha1_hex(payload);
}

}  // namespace gf2
}  // namespace mtgpb
