"""T0: the oracle pinned against things other than itself (textbook definitions, brute force,
explicit CRT with Python big integers, closed forms, the paper's own numbers).

Each pin is chosen so that a plausible mistake (dropped term, wrong sign, transposed index) fails."""
import numpy as np
import pytest

from oracle import ckks as O

P12 = O.Params("P12")
P13 = O.Params("P13")
P16 = O.Params("P16")


def rand_limbs(mods, N, seed):
    g = np.random.default_rng(seed)
    return np.stack([g.integers(0, q, N, dtype=np.uint64) for q in mods])


# ---------------------------------------------------------------- PRNG
def test_prng_is_textbook_splitmix64():
    # SplitMix64 from state 0: first output 0xE220A8397B1DCDAF (Vigna's reference sequence);
    # second 0x6E789E6AA1B965F4, third 0x06C45D188009454F.
    assert O.prng_draw(0, 0, 0) == 0xE220A8397B1DCDAF
    assert O.prng_draw(0, 0, 1) == 0x6E789E6AA1B965F4
    assert O.prng_draw(0, 0, 2) == 0x06C45D188009454F


def test_samplers_distribution():
    N = 1 << 15
    t = O.sample_ternary(7, O.STREAM_SK, N)
    assert set(np.unique(t)) == {-1, 0, 1}
    assert all(abs(np.mean(t == v) - 1 / 3) < 0.02 for v in (-1, 0, 1))
    e = O.sample_cbd21(7, 99, N)
    assert np.abs(e).max() <= 21 and abs(e.var() - 10.5) < 0.5 and abs(e.mean()) < 0.1
    q = P16.q[3]
    u = O.sample_uniform(7, 5, [q], [3], N)[0].astype(np.float64)
    assert u.max() < q and abs(u.mean() / q - 0.5) < 0.01


# ---------------------------------------------------------------- ring product (C1)
@pytest.mark.parametrize("N", [16, 64, 256, 1024])
def test_ntt_product_equals_schoolbook(N):
    mods = [P16.q[0], P16.q[5], P16.p[2]]
    a, b = rand_limbs(mods, N, 1), rand_limbs(mods, N, 2)
    assert np.array_equal(O.ring_mul(a, b, mods, N), O.ring_mul_schoolbook(a, b, mods, N))


def test_ntt_product_equals_schoolbook_4096():
    mods = [P12.q[1]]
    a, b = rand_limbs(mods, 4096, 3), rand_limbs(mods, 4096, 4)
    assert np.array_equal(O.ring_mul(a, b, mods, 4096), O.ring_mul_schoolbook(a, b, mods, 4096))


def test_schoolbook_negacyclic_small_closed_form():
    # X^{N-1} * X = X^N = -1
    N, q = 8, P16.q[1]
    a = np.zeros((1, N), np.uint64); a[0, N - 1] = 1
    b = np.zeros((1, N), np.uint64); b[0, 1] = 1
    c = O.ring_mul_schoolbook(a, b, [q], N)
    assert c[0, 0] == q - 1 and c[0, 1:].sum() == 0


@pytest.mark.parametrize("N", [8, 32, 64])
def test_ntt_is_evaluation_at_odd_powers_of_psi(N):
    q = P16.q[2]
    psi = O.primitive_root_2n(q, N)
    assert pow(psi, N, q) == q - 1
    a = rand_limbs([q], N, 5)
    A = O.ntt(a, [q], N)[0]
    for j in range(N):
        x = pow(psi, 2 * j + 1, q)
        assert int(A[j]) == sum(int(a[0, i]) * pow(x, i, q) for i in range(N)) % q


def test_ntt_roundtrip_2_16():
    mods = [P16.q[0], P16.q[7]]
    a = rand_limbs(mods, P16.N, 6)
    assert np.array_equal(O.intt(O.ntt(a, mods, P16.N), mods, P16.N), a)


def test_ntt_product_spot_2_16():
    # spot-check coefficient k of the product at N=2^16 against the defining sum
    N, q = P16.N, P16.q[4]
    a, b = rand_limbs([q], N, 7), rand_limbs([q], N, 8)
    c = O.ring_mul(a, b, [q], N)[0]
    A, B = [int(v) for v in a[0]], [int(v) for v in b[0]]
    for k in (0, 1, 12345, N - 1):
        s = sum(A[i] * B[k - i] for i in range(k + 1)) - sum(A[i] * B[k - i + N] for i in range(k + 1, N))
        assert int(c[k]) == s % q


# ---------------------------------------------------------------- automorphisms, slots (C2)
def test_automorph_group_law_and_ring_hom():
    N = 64
    mods = [P16.q[1], P16.q[2]]
    a, b = rand_limbs(mods, N, 9), rand_limbs(mods, N, 10)
    for g, h in [(5, 25), (3, 2 * N - 1), (2 * N - 1, 2 * N - 1)]:
        lhs = O.automorph(O.automorph(a, h, mods, N), g, mods, N)
        assert np.array_equal(lhs, O.automorph(a, g * h % (2 * N), mods, N))
    g = 5 ** 3 % (2 * N)
    assert np.array_equal(O.automorph(O.ring_mul(a, b, mods, N), g, mods, N),
                          O.ring_mul(O.automorph(a, g, mods, N), O.automorph(b, g, mods, N), mods, N))


def test_encode_fft_equals_direct_sum():
    N = 64
    z = np.random.default_rng(11).uniform(-1, 1, N // 2) + 1j * np.random.default_rng(12).uniform(-1, 1, N // 2)
    assert np.array_equal(O.encode_coeffs(z, 2.0 ** 30, N), O.encode_coeffs_direct(z, 2.0 ** 30, N))


def _dec_plain(m_signed, scale, N):
    return O.decode_coeffs([int(v) for v in m_signed], scale, N)


def test_slot_semantics_rotation_conj_i():
    """sigma_{5^r} = LEFT rotation by r (P:154-157 rho(v;r) = (v_r, v_{r+1}, ...)); sigma_{2N-1} = conj;
    X^{N/2} = multiplication by i."""
    N, q = 64, P16.q[0]
    z = np.random.default_rng(13).uniform(-1, 1, N // 2) + 1j * np.random.default_rng(14).uniform(-1, 1, N // 2)
    sc = 2.0 ** 40
    m = O.encode_coeffs(z, sc, N)
    mq = O.from_signed(m, [q], N)

    def dec(x):
        vals, _ = O.crt_lift(x, [q])
        return O.decode_coeffs(vals, sc, N)

    for r in (1, 3, 17):
        got = dec(O.automorph(mq, pow(5, r, 2 * N), [q], N))
        assert np.allclose(got, np.roll(z, -r), atol=1e-9)
    assert np.allclose(dec(O.automorph(mq, 2 * N - 1, [q], N)), np.conj(z), atol=1e-9)
    assert np.allclose(dec(O.mul_monomial_half(mq, [q], N)), 1j * z, atol=1e-9)


def test_encrypt_decrypt_roundtrip_paper_bound():
    """max per-slot abs error ~9e-6 after one encrypt-decode round trip at n=2^14, Delta=2^40,
    40-bit body primes.  Our oracle at n=2^14 (N=2^15) must stay within 1e-5."""
    import copy
    P = copy.copy(P16)
    P.N, P.n = 1 << 15, 1 << 14
    keys = O.Keys(P, 0x5EED, max_level=3)
    z = np.random.default_rng(15).uniform(-1, 1, P.n) + 1j * np.random.default_rng(16).uniform(-1, 1, P.n)
    pt = O.encode(P, z, 2.0 ** 40, 3)
    ct = O.encrypt_sk(P, keys, pt, 0xE1C)
    dec = O.decrypt(P, keys, ct)
    # decrypt(enc(m)) - m is exactly the CBD(21) error
    diff, _ = O.crt_lift(O.psub(dec.m, pt.m, P.q[:3], P.N), P.q[:3])
    assert max(abs(v) for v in diff) <= 21
    err = np.abs(O.decode(P, dec) - z).max()
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")) as f:
        g = json.load(f)["encrypt_decode_max_abs_error"]
    assert err < g["bound_used"] and g["value"] < g["bound_used"]


# ---------------------------------------------------------------- BConv / ModDown / rescale (C4, C5) by explicit CRT
def test_bconv_explicit_crt():
    N = 16
    qin = [P16.q[1], P16.q[2], P16.q[3]]
    qout = [P16.q[0], P16.p[0], P16.p[5]]
    x = rand_limbs(qin, N, 20)
    y = O.bconv(x, qin, qout, N)
    vals, Qj = O.crt_lift(x, qin, centered=False)
    for k in range(N):
        hits = [u for u in range(len(qin)) if all(int(y[t, k]) == (vals[k] + u * Qj) % qt for t, qt in enumerate(qout))]
        assert len(hits) == 1, k


def test_moddown_explicit_crt():
    P, L, N = P13, 5, P13.N
    mods = P.ext_mods(L)
    b = rand_limbs(mods, N, 21)
    out = O.moddown(P, b, L)
    K = 64  # check the first K coefficients by explicit CRT
    bv, _ = O.crt_lift(b[:, :K], mods, centered=False)
    bp, _ = O.crt_lift(b[L:, :K], P.p, centered=False)
    Q = 1
    for q in P.q[:L]:
        Q *= q
    ov, _ = O.crt_lift(out[:, :K], P.q[:L], centered=False)
    ties = 0
    for k in range(K):
        # rounded ModDown: out = round(b / P) (floor or ceil only when b/P sits within 1e-12 of a half-integer)
        lo = bv[k] // P.P
        frac = (bv[k] - lo * P.P) / P.P
        want = lo + (1 if frac >= 0.5 else 0)
        if abs(frac - 0.5) < 1e-12:
            ties += 1
            assert ov[k] in (lo % Q, (lo + 1) % Q)
        else:
            assert ov[k] == want % Q, k
    assert ties <= 1


def test_moddown_rescale_explicit_crt():
    """Merged ModDown + rescale (R-LAZY): out = round(x / (P q_{L-1})) mod Q_{L-1} (ties within 1e-12 aside)."""
    P, L, N = P13, 5, P13.N
    mods = P.ext_mods(L)
    x = rand_limbs(mods, N, 23)
    out = O.moddown_rescale(P, x, L)
    K = 64
    xv, _ = O.crt_lift(x[:, :K], mods, centered=False)
    ov, Q1 = O.crt_lift(out[:, :K], P.q[:L - 1], centered=False)
    D = P.P * P.q[L - 1]
    for k in range(K):
        lo = xv[k] // D
        frac = (xv[k] - lo * D) / D
        if abs(frac - 0.5) < 1e-12:
            assert ov[k] in (lo % Q1, (lo + 1) % Q1)
        else:
            assert ov[k] == (lo + (1 if frac >= 0.5 else 0)) % Q1, k


def test_lazy_hoisted_rotation_equals_rotation_in_value():
    """ModDown of the extended-basis rotation pair decrypts like the ordinary hoisted rotation."""
    keys = O.Keys(P13, 0x5EED, galois=[O.galois_rot(P13, 3)])
    z = np.random.default_rng(33).uniform(-1, 1, P13.n)
    ct = O.encrypt_sk(P13, keys, O.encode(P13, z, 2.0 ** 40, 6), 1)
    e = O.rotate_hoisted_ext(P13, keys, ct, [3])[0]
    md = O.Ct(np.stack([O.moddown(P13, e[c], 6) for c in range(2)]), ct.scale)
    ref = O.rotate_hoisted(P13, keys, ct, [3])[0]
    assert np.array_equal(md.c, ref.c)      # ModDown(P sigma(c0) + b0) == sigma(c0) + ModDown(b0) exactly


def test_rescale_is_round_division():
    P, L, N = P16, 4, 32
    mods = P.q[:L]
    a = rand_limbs(mods, N, 22)
    out = O.rescale_poly(a, mods, N)
    av, _ = O.crt_lift(a, mods, centered=False)
    ov, Q1 = O.crt_lift(out, mods[:-1], centered=False)
    qL = mods[-1]
    for k in range(N):
        assert ov[k] == ((av[k] + qL // 2) // qL) % Q1


# ---------------------------------------------------------------- keys and key switching (C4)
@pytest.fixture(scope="module")
def keys13():
    galois = [O.galois_rot(P13, r) for r in (1, 5)] + [O.galois_conj(P13)]
    return O.Keys(P13, 0x5EED, galois=galois, relin=True)


def test_key_invariant(keys13):
    """ksk_j[0] + ksk_j[1] s - g_j s'  equals e_j with |e_j| <= 21 on every limb."""
    P, N = P13, P13.N
    ML = keys13.max_level
    mods = P.ext_mods(ML)
    g = O.galois_rot(P13, 5)
    sp = O.automorph(keys13.s, g, mods, N)
    for j, k in enumerate(keys13.ksk[g]):
        lo, hi = P.digit(j, ML)
        gfac = [(P.P % t) if lo <= i < hi else 0 for i, t in enumerate(mods)]
        r = O.psub(O.padd(k[0], O.ring_mul(k[1], keys13.s, mods, N), mods, N), O.pmul_scalar(sp, gfac, mods, N), mods, N)
        for l, t in enumerate(mods):
            v = r[l].astype(object)
            v = np.where(v > t // 2, v - t, v)
            assert np.abs(v.astype(np.int64)).max() <= 21


def _noise(P, keys, ct, ref_m, L):
    dec = O.decrypt(P, keys, ct)
    d, _ = O.crt_lift(O.psub(dec.m, ref_m, P.q[:L], P.N), P.q[:L])
    return max(abs(v) for v in d)


@pytest.mark.parametrize("L", [8, 5])
def test_rotation_keyswitch_error_bound(keys13, L):
    """Dec(rot(ct)) - sigma_g(Dec(ct)) is bounded by the ModDown floor error (alpha per coefficient,
    times s: <= alpha*(N+1)) plus the key-noise term, analytic bound 2*alpha*N."""
    P, N = P13, P13.N
    z = np.random.default_rng(30).uniform(-1, 1, P.n)
    pt = O.encode(P, z, 2.0 ** 40, L)
    ct = O.encrypt_sk(P, keys13, pt, 0xE1C)
    m = O.decrypt(P, keys13, ct).m
    for r in (1, 5):
        g = O.galois_rot(P, r)
        rot = O.rotate(P, keys13, ct, r)
        assert _noise(P, keys13, rot, O.automorph(m, g, P.q[:L], N), L) <= 2 * P.alpha * N
        dz = O.decode(P, O.decrypt(P, keys13, rot))
        assert np.abs(dz - np.roll(z, -r)).max() < 1e-6
    hs = O.rotate_hoisted(P, keys13, ct, [1, 5])
    for r, h in zip((1, 5), hs):
        assert _noise(P, keys13, h, O.automorph(m, O.galois_rot(P, r), P.q[:L], N), L) <= 2 * P.alpha * N
    cj = O.conjugate(P, keys13, ct)
    assert _noise(P, keys13, cj, O.automorph(m, 2 * N - 1, P.q[:L], N), L) <= 2 * P.alpha * N


def test_hoisted_differs_in_bits_but_not_in_value(keys13):
    """sigma does not commute bitwise with fast BConv, so hoisted != single in bits."""
    P, L = P13, 8
    z = np.random.default_rng(31).uniform(-1, 1, P.n)
    ct = O.encrypt_sk(P, keys13, O.encode(P, z, 2.0 ** 40, L), 0xE1C)
    a = O.rotate(P, keys13, ct, 1)
    b = O.rotate_hoisted(P, keys13, ct, [1])[0]
    assert not np.array_equal(a.c, b.c)
    assert np.abs(O.decode(P, O.decrypt(P, keys13, a)) - O.decode(P, O.decrypt(P, keys13, b))).max() < 1e-6


def test_tensor_relin_rescale(keys13):
    P, L = P13, 6
    g = np.random.default_rng(32)
    z1, z2 = g.uniform(-1, 1, P.n), g.uniform(-1, 1, P.n)
    c1 = O.encrypt_sk(P, keys13, O.encode(P, z1, 2.0 ** 40, L), 1)
    c2 = O.encrypt_sk(P, keys13, O.encode(P, z2, 2.0 ** 40, L), 2)
    t = O.tensor(P, c1, c2)
    assert np.abs(O.decode(P, O.decrypt(P, keys13, t)) - z1 * z2).max() < 1e-6
    r = O.rescale(P, O.relinearize(P, keys13, t))
    assert r.L == L - 1 and r.scale == 2.0 ** 80 / P.q[L - 1]
    assert np.abs(O.decode(P, O.decrypt(P, keys13, r)) - z1 * z2).max() < 1e-6


def test_errors():
    with pytest.raises(O.OracleError):
        O.add(P13, O.Ct(np.zeros((2, 2, P13.N), np.uint64), 1.0), O.Ct(np.zeros((2, 2, P13.N), np.uint64), 2.0))
    with pytest.raises(O.OracleError):
        O.rescale(P13, O.Ct(np.zeros((2, 1, P13.N), np.uint64), 1.0))
