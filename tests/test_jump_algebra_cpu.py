"""CPU check of the identity the Karatsuba jump (csrc/mtgp_jump.cu) rests on: the transposed
Karatsuba split of a GF(2) middle product with 32-bit word coefficients,
    MP(a, z)_j = XOR_i a_i z_{i+j},  y_lo = P ^ L,  y_hi = P ^ H,
    P = MP(a0 ^ a1, Z1),  L = MP(a0, Z0 ^ Z1),  H = MP(a1, Z1 ^ Z2),
and the block decomposition of a long jump polynomial into middle products."""
import numpy as np
import pytest


def _mp(a, z):
    m = len(a)
    y = np.zeros(m, np.uint32)
    for i in range(m):
        if a[i]:
            y ^= z[i:i + m]
    return y


def _kmp(a, z, d):
    m = len(a)
    if d == 0:
        return _mp(a, z)
    h = m // 2
    a0, a1 = a[:h], a[h:]
    z0, z1, z2 = z[0:m - 1], z[h:h + m - 1], z[m:2 * m - 1]
    p = _kmp(a0 ^ a1, z1, d - 1)
    lo = _kmp(a0, z0 ^ z1, d - 1)
    hi = _kmp(a1, z1 ^ z2, d - 1)
    return np.concatenate([p ^ lo, p ^ hi])


@pytest.mark.parametrize("d", [1, 2, 3])
def test_transposed_karatsuba_middle_product(d):
    rng = np.random.default_rng(d)
    m = 12 << d
    a = rng.integers(0, 2, m).astype(np.uint8)
    z = rng.integers(0, 2**32, 2 * m - 1, dtype=np.uint64).astype(np.uint32)
    assert np.array_equal(_kmp(a, z, d), _mp(a, z))


def test_block_decomposition_of_a_jump():
    """y_j = XOR_{i<M} q_i x_{i+j} (j < N) equals the sum over q blocks of size n_out of
    Karatsuba middle products, with N padded to n_out and q padded with zeros."""
    rng = np.random.default_rng(7)
    M, N, d = 700, 90, 2
    n_out = 96
    q = rng.integers(0, 2, M).astype(np.uint8)
    B = -(-M // n_out)
    x = rng.integers(0, 2**32, (B + 1) * n_out, dtype=np.uint64).astype(np.uint32)
    direct = np.zeros(N, np.uint32)
    for i in range(M):
        if q[i]:
            direct ^= x[i:i + N]
    qp = np.zeros(B * n_out, np.uint8)
    qp[:M] = q
    acc = np.zeros(n_out, np.uint32)
    for b in range(B):
        acc ^= _kmp(qp[b * n_out:(b + 1) * n_out], x[b * n_out:b * n_out + 2 * n_out - 1], d)
    assert np.array_equal(acc[:N], direct)
