"""The exact identities the GPU kernels rely on, checked by brute force on small integers (no GPU, no oracle code):
the kernels compute the same residues as the oracle's plain definitions only because these hold.

* Value kernel step 4 as a convolution (bcast_ntt_kernel): the Toeplitz sums
  b_t = sum_{u < nu} src[t + dmax - u] n_u (dmax = nu - 1, t < nt, nsrc = nt + dmax <= 128) are the coefficients
  X^{t + dmax} of the NEGACYCLIC product mod X^128 + 1 of A = sum_j src_j X^j and B = sum_u n_u X^u (no aliasing),
  and that product is the pointwise product of 128-point negacyclic transforms whose psi-powers are the first 128
  entries of the N-point bit-reversed table.
* The integer NTT's Shoup remainder for q = 2^60 - c, c < 2^32: a w - h q = a w + h c - (h << 60) mod 2^64.
"""
import numpy as np
import pytest

Q = 1152921504606584833          # 2^60 - 2^18 + 1 (q_0 of P16), q = 1 mod 2^17
Q40 = 1099510054913              # a 40-bit body prime of P16


def _root(q, order):
    """A primitive `order`-th root of unity mod q (order a power of two dividing q - 1)."""
    for g in range(2, 1000):
        w = pow(g, (q - 1) // order, q)
        if pow(w, order // 2, q) != 1:
            return w
    raise AssertionError("no root")


def _brv(i, bits):
    return int(format(i, "0%db" % bits)[::-1], 2)


def _toeplitz(src, n, nt, q):
    nu = len(n)
    dmax = nu - 1
    return [sum(src[t + dmax - u] * n[u] for u in range(nu) if 0 <= t + dmax - u < len(src)) % q for t in range(nt)]


def _negacyclic(a, b, q, size=128):
    out = [0] * size
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            k = i + j
            if k < size:
                out[k] = (out[k] + x * y) % q
            else:
                out[k - size] = (out[k - size] - x * y) % q
    return out


@pytest.mark.parametrize("q", [Q, Q40])
@pytest.mark.parametrize("nu,nt", [(64, 64), (64, 17), (8, 8), (1, 64), (33, 64)])
def test_toeplitz_is_exact_negacyclic_128(q, nu, nt):
    rng = np.random.default_rng(nu * 1000 + nt)
    dmax = nu - 1
    nsrc = nt + dmax
    assert nsrc <= 128
    src = [int(x) for x in rng.integers(0, q, nsrc, dtype=np.uint64)]
    n = [int(x) for x in rng.integers(0, q, nu, dtype=np.uint64)]
    direct = _toeplitz(src, n, nt, q)
    conv = _negacyclic(src, n, q)
    assert [conv[t + dmax] for t in range(nt)] == direct


def test_negacyclic_128_via_the_n_point_table():
    """The 128-point negacyclic transform with psi' = psi^(N/128) (psi a primitive 2N-th root, N = 2^16) evaluates A at
    the odd powers of psi'; its merged-twiddle table psi'^{brv_7(i)} equals the N-point table psi^{brv_16(i)}, i < 128;
    pointwise products of the evaluations times 128^{-1} after the inverse give the negacyclic product."""
    q, N = Q40, 1 << 16
    psi = _root(q, 2 * N)
    psi7 = pow(psi, N // 128, q)                      # primitive 256-th root
    assert pow(psi7, 128, q) == q - 1
    for i in range(128):
        assert pow(psi, _brv(i, 16), q) == pow(psi7, _brv(i, 7), q)
    rng = np.random.default_rng(5)
    a = [int(x) for x in rng.integers(0, q, 100, dtype=np.uint64)] + [0] * 28
    b = [int(x) for x in rng.integers(0, q, 64, dtype=np.uint64)] + [0] * 64
    ev = lambda p: [sum(c * pow(psi7, (2 * k + 1) * j, q) for j, c in enumerate(p)) % q for k in range(128)]
    ea, eb = ev(a), ev(b)
    prod = [x * y % q for x, y in zip(ea, eb)]
    inv128 = pow(128, q - 2, q)
    back = [sum(prod[k] * pow(psi7, -(2 * k + 1) * j % 256, q) for k in range(128)) * inv128 % q for j in range(128)]
    assert back == _negacyclic(a, b, q)


def test_shoup_remainder_for_q_2_60_minus_c():
    c = (1 << 60) - Q
    assert 0 < c < (1 << 32)
    rng = np.random.default_rng(7)
    m64 = (1 << 64) - 1
    for _ in range(2000):
        a = int(rng.integers(0, 8 * Q, dtype=np.uint64))
        w = int(rng.integers(0, Q, dtype=np.uint64))
        wp = (w << 64) // Q
        h = (a * wp) >> 64
        generic = (a * w - h * Q) & m64
        hl, hh = h & 0xFFFFFFFF, h >> 32
        hc = ((((hh * c) & 0xFFFFFFFF) << 32) + hl * c) & m64
        trick = (a * w + hc - (((hl << 28) & 0xFFFFFFFF) << 32)) & m64
        assert trick == generic
        assert generic == (a * w) % Q + ((a * w) // Q - h) * Q   # the exact Shoup remainder, in [0, 2q)
