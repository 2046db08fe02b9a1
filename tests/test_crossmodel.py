"""C11 pins: the pure-Python big-integer cross-model (oracle/crossmodel.py, an independent
implementation at N = 32 written from DESIGN.md's spec) equals the oracle (oracle/ckks.py + oracle.c +
kernels.py) BIT FOR BIT: PRNG and samplers, keys, encryption, every key-switching primitive (single, hoisted,
conj, relin, the extended-basis variants of R-LAZY / R-RELRS), rescale, and the three kernels' schedules
(projection with C = n/m and C < n/m, score with and without Align_r, value, export).  Also: the oracle's
59-bit fixed-point rounding estimate inside o_bconv_round equals exact rational rounding on P16-sized moduli."""
import random

import numpy as np
import pytest

import synth
from oracle import ckks as O
from oracle import crossmodel as X
from oracle import kernels as K

P5 = O.Params("P5")
XP = X.Params("P5")


def to_np(c):
    return np.array(c, dtype=np.uint64)


def to_x(ct):
    return X.Ct([[[int(v) for v in limb] for limb in comp] for comp in ct.c], ct.scale)


def same(xct, oct_, what):
    assert xct.scale == oct_.scale, what
    assert np.array_equal(to_np(xct.c), oct_.c), what


@pytest.fixture(scope="module")
def keys():
    rots = sorted({r % P5.n for r in range(-16, 16) if r % P5.n})
    g = [O.galois_rot(P5, r) for r in rots] + [O.galois_conj(P5)]
    return O.Keys(P5, 0x5EED, galois=g, relin=True), X.Keys(XP, 0x5EED, galois=g, relin=True)


def test_prng_and_samplers_bit_exact():
    for seed, stream in [(0, 0), (0x5EED, X.S_SK), (7, X.s_ksk(37, 2, 1)), (2 ** 63 + 5, X.s_mask(9))]:
        for i in (0, 1, 2, 1000, 2 ** 40):
            assert X.draw(seed, stream, i) == O.prng_draw(seed, stream, i)
    assert X.draw(0, 0, 0) == 0xE220A8397B1DCDAF              # textbook SplitMix64 first output
    q = P5.q[1]
    assert X.uniform(3, 11, q, 4, 32) == [int(v) for v in O.sample_uniform(3, 11, [q], [4], 32)[0]]
    assert X.ternary(3, 11, 32) == [int(v) for v in O.sample_ternary(3, 11, 32)]
    assert X.cbd21(3, 11, 32) == [int(v) for v in O.sample_cbd21(3, 11, 32)]


def test_keys_bit_exact(keys):
    ok, xk = keys
    assert np.array_equal(to_np(xk.s), ok.s)
    for g in list(ok.ksk):
        for j, (b, a) in enumerate(xk.ksk[g]):
            assert np.array_equal(to_np([b, a]), ok.ksk[g][j]), (g, j)


def _ct(keys, L, seed, scale=2.0 ** 40):
    ok, xk = keys
    m = O.encode(P5, synth.complex_slots(P5.n, seed), scale, L)
    oc = O.encrypt_sk(P5, ok, m, seed)
    xc = X.encrypt_sk(XP, xk, [[int(v) for v in limb] for limb in m.m], scale, seed)
    same(xc, oc, "encrypt")
    return oc, xc


@pytest.mark.parametrize("L", [6, 5, 3, 1])
def test_keyswitch_primitives_bit_exact(keys, L):
    ok, xk = keys
    oc, xc = _ct(keys, L, 10 + L)
    for r in (1, -3, 5):
        same(X.rotate(XP, xk, xc, X.galois_rot(XP, r)), O.rotate(P5, ok, oc, r), "rotate %d L=%d" % (r, L))
    steps = [1, 4, -2]
    ext = X.modup(XP, xc.c[1], L)
    for r, oh in zip(steps, O.rotate_hoisted(P5, ok, oc, steps)):
        same(X.rotate(XP, xk, xc, X.galois_rot(XP, r), ext), oh, "hoisted %d" % r)
    same(X.rotate(XP, xk, xc, 2 * XP.N - 1), O.conjugate(P5, ok, oc), "conj")
    # the extended-basis (lazy) rotations and their merged ModDown + rescale (R-LAZY)
    for r, oe in zip(steps, O.rotate_hoisted_ext(P5, ok, oc, steps)):
        xe = X.rotate_ext(XP, xk, xc, X.galois_rot(XP, r), ext)
        assert np.array_equal(to_np(xe), oe)
        if L > 1:
            assert np.array_equal(to_np([X.moddown_rescale(XP, xe[c], L) for c in range(2)]),
                                  np.stack([O.moddown_rescale(P5, oe[c], L) for c in range(2)]))
    if L > 1:
        same(X.rescale(XP, xc), O.rescale(P5, oc), "rescale")


def test_tensor_relin_bit_exact(keys):
    ok, xk = keys
    a, xa = _ct(keys, 5, 1)
    b, xb = _ct(keys, 5, 2)
    ev = X.XEv(XP, xk, 4, None)
    t, xt = O.tensor(P5, a, b), ev.tensor(xa, xb)
    same(xt, t, "tensor")
    same(ev.relin(xt), O.relinearize(P5, ok, t), "relin")
    same(ev.relin_rescale(xt), K.Ev(P5, ok, 4).relin_rescale(t), "relin_rescale (R-RELRS)")


def test_bconv_round_fixed_point_is_exact_rounding():
    """R-MODDOWN's rounding r = round(sum_k v_k / p_k) is a 59-bit fixed-point estimate (oracle.c o_bconv_round,
    crossmodel.hps_round).  On P16's six 60-bit special primes (the ModDown of every key switch) and on
    {q_{L-1}} u P (merged ModDown + rescale): the output is ALWAYS a lift of x mod B (correct key switching either
    way), it is the exact centred residue for random inputs, and it can differ from exact rounding only when
    x / B lies within 2^-55 of 1/2 -- probed with inputs next to B/2."""
    P16 = O.Params("P16")
    rng = random.Random(5)
    N = 512
    for base in (P16.p, [P16.q[7]] + P16.p):
        B = 1
        for t in base:
            B *= t
        xs = [rng.randrange(B) for _ in range(N - 16)]
        xs += [B // 2 + d for d in range(-7, 8)] + [B - 1]
        rows = np.array([[x % t for x in xs] for t in base], dtype=np.uint64)
        outq = P16.q[:6]
        got = O.bconv_round(rows, base, outq, N)
        for k, x in enumerate(xs):
            y = X.centred(x, B)
            lifts = [y, y + B] if y < 0 else [y, y - B]
            near_half = abs(2 * (x % B) - B) * 2 ** 55 < B
            vals = [[int(got[i][k]) for i in range(len(outq))]]
            ok_lifts = [[v % q for q in outq] for v in lifts]
            assert vals[0] in ok_lifts, k
            if not near_half:
                assert vals[0] == ok_lifts[0], k
        # the cross-model's independent re-typing of the same rule agrees word for word
        vs = [[x * pow(B // b, -1, b) % b for b in base] for x in xs]
        for k, x in enumerate(xs):
            yy = sum(v * (B // b) for v, b in zip(vs[k], base)) - X.hps_round(vs[k], base) * B
            assert [yy % q for q in outq] == [int(got[i][k]) for i in range(len(outq))]


# ------------------------------------------------------------------ per-level special-prime count K(L) (DESIGN.md R-KL)
def test_k_of_level_definition_and_classes():
    """P5A6 (alpha = 6, five 60-bit special primes): K(L) is the smallest K with P_K >= 2^16 max_j Q_j(L), and at
    every level the cross-model -- which generates each special-prime class's key from its definition -- equals the
    oracle -- which derives it from the top class's key -- on keys, single / hoisted rotations, conj, relin, the
    merged ModDown + rescale and the projection and value schedules."""
    PA, XA = O.Params("P5A6"), X.Params("P5A6")
    for L in range(1, PA.L_max + 1):
        D = 1
        for i in range(L):
            D *= PA.q[i]
        KL = PA.K(L)
        assert PA.P_of(L) >= D << 16 and (KL == 1 or PA.P_of(L) // PA.p[KL - 1] < D << 16), L
        assert PA.ext_mods(L) == XA.ext(L) and len(PA.ext_mods(L)) == L + KL
    assert len(set(PA.K_of_level)) >= 3
    g = [O.galois_rot(PA, r) for r in (1, 2, -1, 4)] + [O.galois_conj(PA)]
    ok, xk = O.Keys(PA, 7, galois=g, relin=True), X.Keys(XA, 7, galois=g, relin=True)
    for L in range(1, PA.L_max + 1):
        for gg in g + [0]:
            ko, kx = ok.key_at(gg, L), xk.key_at(gg, L)
            for j in range(len(ko)):
                assert np.array_equal(ko[j], to_np(list(kx[j]))), (L, gg, j)
        m = O.encode(PA, synth.complex_slots(PA.n, 50 + L), 2.0 ** 40, L)
        oc = O.encrypt_sk(PA, ok, m, 9)
        xc = X.encrypt_sk(XA, xk, [[int(v) for v in limb] for limb in m.m], 2.0 ** 40, 9)
        same(X.rotate(XA, xk, xc, X.galois_rot(XA, 1)), O.rotate(PA, ok, oc, 1), "rotate L=%d" % L)
        ext = X.modup(XA, xc.c[1], L)
        for r, oh in zip([2, -1], O.rotate_hoisted(PA, ok, oc, [2, -1])):
            same(X.rotate(XA, xk, xc, X.galois_rot(XA, r), ext), oh, "hoisted L=%d" % L)
        same(X.rotate(XA, xk, xc, 2 * XA.N - 1), O.conjugate(PA, ok, oc), "conj L=%d" % L)
        if L > 1:
            oe = O.rotate_hoisted_ext(PA, ok, oc, [4])[0]
            xe = X.rotate_ext(XA, xk, xc, X.galois_rot(XA, 4), ext)
            assert np.array_equal(to_np(xe), oe)
            assert np.array_equal(to_np([X.moddown_rescale(XA, xe[c], L) for c in range(2)]),
                                  np.stack([O.moddown_rescale(PA, oe[c], L) for c in range(2)]))
            xev = X.XEv(XA, xk, 4, None)
            t = O.tensor(PA, oc, oc)
            same(xev.relin_rescale(xev.tensor(xc, xc)), K.Ev(PA, ok, 4).relin_rescale(t), "relin_rescale L=%d" % L)
            # decryption after the key switch stays exact to the noise (the class key is a valid key for P_K(L))
            z = O.decode(PA, O.decrypt(PA, ok, O.rotate(PA, ok, oc, 1)))
            assert np.abs(z - np.roll(synth.complex_slots(PA.n, 50 + L), -1)).max() < 1e-6


# ------------------------------------------------------------------ the kernels' schedules on both arithmetics
def _xw(pt):
    return ([[int(v) for v in limb] for limb in pt.m], pt.scale)


def _pair(keys, m):
    ok, xk = keys
    oev = K.Ev(P5, ok, m)
    xev = X.XEv(XP, xk, m, lambda z, s: O.encode_coeffs(z, s, P5.N))
    return oev, xev


@pytest.mark.parametrize("C", [None, 3])
def test_projection_schedule_bit_exact(keys, C):
    ok, xk = keys
    m, d_in, d_out, L = 4, 10, 7, 6
    plan = K.ProjPlan(P5.n, m, d_in, d_out, C=C, N1=2 if C is None else 1)
    Xm = synth.fixed_point_uniform((m, d_in), 3)
    W = synth.bert_weight((d_in, d_out), 4)
    Lw = plan.weight_level(L)
    pts = {}

    def w(b, p, u, q):
        if (b, p, u, q) not in pts:
            pts[(b, p, u, q)] = O.encode(P5, K.proj_weight_slots(W, plan, b, p, u, q), float(P5.q[Lw - 1]), Lw)
        return pts[(b, p, u, q)]
    xs = [O.encrypt_sk(P5, ok, O.encode(P5, z, 2.0 ** 40, L), 20 + u) for u, z in enumerate(K.proj_inputs(Xm, plan))]
    oev, xev = _pair(keys, m)
    ys = K.projection(oev, plan, xs, w)
    xys = K.projection(xev, plan, [to_x(x) for x in xs], lambda *a: _xw(w(*a)))
    for a, b in zip(xys, ys):
        same(a, b, "projection C=%s" % C)


@pytest.mark.parametrize("H,dh,C", [(2, 2, 4), (2, 3, 3)])
def test_score_schedule_bit_exact(keys, H, dh, C):
    ok, xk = keys
    m, L0 = 4, 6
    plan = K.ScorePlan(P5.n, m, H, dh, C_qk=C, beta=2)
    g = synth.rng(8)
    Qh, Kh = g.uniform(-1, 1, (H, m, dh)), g.uniform(-1, 1, (H, m, dh))
    perm = K.pi_S(H, dh)
    Qp, Kp = np.concatenate(list(Qh), 1)[:, perm], np.concatenate(list(Kh), 1)[:, perm]
    qs = [O.encrypt_sk(P5, ok, O.encode(P5, K.score_qk_slots(Qp, plan, l), 2.0 ** 40, L0), 30 + l) for l in range(plan.B)]
    ks = [O.encrypt_sk(P5, ok, O.encode(P5, K.score_qk_slots(Kp, plan, l), 2.0 ** 40, L0), 40 + l) for l in range(plan.B)]
    oev, xev = _pair(keys, m)
    S = K.score(oev, plan, qs, ks)
    XS = K.score(xev, plan, [to_x(q) for q in qs], [to_x(k) for k in ks])
    for t, (a, b) in enumerate(zip(XS, S)):
        same(a, b, "S_%d aligned=%s" % (t, plan.aligned))
    for a, b in zip(K.score_export(xev, plan, XS), K.score_export(oev, plan, S)):
        same(a, b, "export stream")


def test_value_and_export_schedule_bit_exact(keys):
    ok, xk = keys
    m, H, dh = 4, 2, 2
    plan = K.ValuePlan(P5.n, m, H, dh)
    Ph = synth.attention_probs(H, m, 9)
    Vh = synth.uniform((H, m, dh), 10)
    vs = [O.encrypt_sk(P5, ok, O.encode(P5, K.value_v_slots(Vh, plan, l), 2.0 ** 40, 6), 50 + l) for l in range(plan.B_V)]
    ps = [O.encrypt_sk(P5, ok, O.encode(P5, K.value_p_slots(Ph, plan, l), 2.0 ** 40, 4), 60 + l) for l in range(plan.B_V)]
    oev, xev = _pair(keys, m)
    outs = K.value(oev, plan, ps, vs)
    xouts = K.value(xev, plan, [to_x(p) for p in ps], [to_x(v) for v in vs])
    for a, b in zip(xouts, outs):
        same(a, b, "value")
    om, osh = K.export_c2m(P5, outs[0], 2, 0x3A5C, 3)
    xm, xsh = X.export_c2m(XP, xouts[0], 2, 0x3A5C, 3)
    same(xm, om, "export masked")
    assert np.array_equal(to_np(xsh), osh)
