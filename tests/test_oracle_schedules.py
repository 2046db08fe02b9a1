"""RotFirst_L (Alg A.3), Phi_C (Alg A.4), Align_r (App. A.3) on the oracle, and the fused schedules of
oracle/kernels.py (what the GPU must reproduce bit for bit) against the paper's own unfused order
(oracle/paper_order.py) on the same encrypted inputs: both decrypt to the textbook float64 result within the
2^-20 target and within noise of each other."""
import numpy as np
import pytest

import synth
from oracle import ckks as O
from oracle import kernels as K
from oracle import paper_order as PO

P13 = O.Params("P13")
TOL = 2.0 ** -20


def enc(P, keys, z, L, seed, scale=2.0 ** 40):
    return O.encrypt_sk(P, keys, O.encode(P, z, scale, L), seed)


def dec(P, keys, ct):
    return O.decode(P, O.decrypt(P, keys, ct))


@pytest.fixture(scope="module")
def keys13():
    from tests.test_oracle_kernels import _galois13
    return O.Keys(P13, synth.SEED_KEYS, galois=_galois13(), relin=True)


# ------------------------------------------------------------------ slot-level definitions
def test_rotfirst_spec_toy_slot_level():
    """RotFirst_{L=3, tau=1} on (a, b, c, d) -> (b, c, a, .); slot 3 zero under G21 (the masks zero
    everything at or beyond L)."""
    a, b, c = 1.0, 2.0, 3.0
    assert np.array_equal(K.rotfirst_reference(np.array([a, b, c, 0.0]), 3, 1), [b, c, a, 0.0])
    # the realisation of Alg A.3 (two cyclic rotations, masks a/b) equals the definition for every (L, tau)
    n = 24
    x = np.arange(1.0, n + 1)
    x_zero_tail = x.copy()
    for Ls in (1, 3, 8, 17, 24):
        xz = x_zero_tail.copy()
        xz[Ls:] = 0.0
        for tau in range(-Ls, 2 * Ls):
            t = tau % Ls
            amask = (np.arange(n) < Ls - t).astype(float)
            bmask = ((np.arange(n) >= Ls - t) & (np.arange(n) < Ls)).astype(float)
            alg = np.roll(xz, -t) * amask + np.roll(xz, -((t - Ls) % n)) * bmask
            assert np.array_equal(alg, K.rotfirst_reference(xz, Ls, t)), (Ls, tau)
            # Alg A.3 needs nothing of the input beyond L: the definition ignores it too
            assert np.array_equal(K.rotfirst_reference(x, Ls, t)[:Ls], K.rotfirst_reference(xz, Ls, t)[:Ls])


def test_phi_c_and_align_slot_level():
    """Phi_C^Delta wraps modulo the C active segments (Alg A.4); Align_r brings head phase r back to 0
    (P:1406-1416): position p of the first H segments receives position (p + H - r) mod H."""
    m, Nseg, C = 4, 8, 5
    X = np.arange(m * Nseg, dtype=float).reshape(Nseg, m)          # row s = segment s
    x = X.reshape(-1).copy()
    x[C * m:] = 0
    for d in range(-C, 2 * C):
        got = K.rotfirst_reference(x, C * m, (d % C) * m).reshape(Nseg, m)
        for s in range(C):
            assert np.array_equal(got[s], X[(s + d) % C])
        assert not got[C:].any()
    H = 3
    for r in range(H):
        got = K.rotfirst_reference(x, H * m, (H - r) * m).reshape(Nseg, m)
        for p in range(H):
            assert np.array_equal(got[p], X[(p + H - r) % H])


# ------------------------------------------------------------------ encrypted RotFirst / Phi_C / Align (fused == definition)
@pytest.mark.parametrize("Ls,taus", [(3, [1, 0, 2]), (20, [7, 13]), (16 * 128, [0, 16, 16 * 127]), (48, [16, 32])])
def test_rotfirst_encrypted_matches_definition(keys13, Ls, taus):
    m = 16
    z = synth.complex_slots(P13.n, 7)
    z[Ls:] = 0
    x = enc(P13, keys13, z, 5, 11)
    ev = K.Ev(P13, keys13, m)
    outs = K.RotFirst_hoisted(ev, x, Ls, taus, m)
    for tau, o in zip(taus, outs):
        assert o.L == 4
        got = dec(P13, keys13, o)
        assert np.abs(got - K.rotfirst_reference(z, Ls, tau % Ls)).max() < 2e-6
        ref_po = dec(P13, keys13, PO.rotfirst(ev, x, Ls, tau, m))
        assert np.abs(got - ref_po).max() < 2e-6


# ------------------------------------------------------------------ projection with C < n/m (Phi_C)
def _projection_case(keys, C, d_in, d_out, N1, L=6, m=16, seed=30):
    plan = K.ProjPlan(P13.n, m, d_in, d_out, C=C, N1=N1)
    X = synth.fixed_point_uniform((m, d_in), seed)
    W = synth.bert_weight((d_in, d_out), seed + 1)
    xs = [enc(P13, keys, z, L, synth.seed_enc(u)) for u, z in enumerate(K.proj_inputs(X, plan))]
    Lw = plan.weight_level(L)
    cache = {}

    def w(b, p, u, q):
        if (b, p, u, q) not in cache:
            cache[(b, p, u, q)] = O.encode(P13, K.proj_weight_slots(W, plan, b, p, u, q), float(P13.q[Lw - 1]), Lw)
        return cache[(b, p, u, q)]
    return plan, X, W, xs, w


def _unpack(plan, keys, ys, d_out):
    return np.concatenate([K.seg_column_unpack(dec(P13, keys, y).real, plan.m, plan.C, d_out, b)
                           for b, y in enumerate(ys)], axis=1)


def test_projection_restricted_C_fused_and_paper_order(keys13):
    """P13, m = 16, C = 128 < N_seg = 256: the bank is Phi_C^q and the giant fold Phi_C^{pN1} (RotFirst_{Cm});
    X W within 2^-20 for the fused schedule and for the paper's order; y_b three levels below x (R-PHIC)."""
    plan, X, W, xs, w = _projection_case(keys13, 128, 300, 200, 8)
    assert plan.restricted and (plan.U, plan.B_out, plan.N2) == (2, 2, 16)
    ev = K.Ev(P13, keys13, plan.m)
    ys = K.projection(ev, plan, xs, w)
    assert all(y.L == 3 for y in ys)
    Y = _unpack(plan, keys13, ys, 200)
    ref = X @ W
    assert np.abs(Y - ref).max() / np.abs(ref).max() < TOL
    Yp = _unpack(plan, keys13, PO.projection(K.Ev(P13, keys13, plan.m), plan, xs, w), 200)
    assert np.abs(Yp - ref).max() / np.abs(ref).max() < TOL
    assert np.abs(Y - Yp).max() / np.abs(ref).max() < TOL
    # the output is segment-column packed with zeros beyond C (the RotFirst masks)
    z = dec(P13, keys13, ys[0])
    assert np.abs(z[plan.C * plan.m:]).max() < 1e-6


def test_projection_full_C_fused_vs_paper_order(keys13):
    plan, X, W, xs, w = _projection_case(keys13, None, 400, 300, 8, L=4, seed=40)
    assert not plan.restricted
    ys = K.projection(K.Ev(P13, keys13, plan.m), plan, xs, w)
    yp = PO.projection(K.Ev(P13, keys13, plan.m), plan, xs, w)
    Y, Yp, ref = _unpack(plan, keys13, ys, 300), _unpack(plan, keys13, yp, 300), X @ W
    for got in (Y, Yp):
        assert np.abs(got - ref).max() / np.abs(ref).max() < TOL
    assert np.abs(Y - Yp).max() / np.abs(ref).max() < TOL
    # different rounding points: the bits differ, the values agree
    assert not np.array_equal(ys[0].c, yp[0].c)


# ------------------------------------------------------------------ score with C mod H != 0 (Align_r) and C mod H = 0
def _score_case(keys, H, dh, C, beta, L0, seed):
    m = 16
    plan = K.ScorePlan(P13.n, m, H, dh, C_qk=C, beta=beta)
    g = synth.rng(seed)
    Qh, Kh = g.uniform(-1, 1, (H, m, dh)), g.uniform(-1, 1, (H, m, dh))
    perm = K.pi_S(H, dh)
    Qp = np.concatenate(list(Qh), 1)[:, perm]
    Kp = np.concatenate(list(Kh), 1)[:, perm]
    qs = [enc(P13, keys, K.score_qk_slots(Qp, plan, l), L0, 100 + l) for l in range(plan.B)]
    ks = [enc(P13, keys, K.score_qk_slots(Kp, plan, l), L0, 200 + l) for l in range(plan.B)]
    return plan, Qh, Kh, qs, ks


def _check_scores(keys, plan, S, ref):
    H, m = plan.H, plan.m
    scale = max(np.abs(r).max() for r in ref)
    got = []
    for t in range(len(S)):
        z = dec(P13, keys, S[t])
        assert np.abs(z[:H * m] - ref[t]).max() / scale < TOL, t
        assert np.abs(z[H * m:]).max() / scale < TOL
        got.append(z)
    return got, scale


def test_score_phase_alignment_H3_C8(keys13):
    """H = 3, C = 8 (C mod H != 0): blocks l = 0, 1, 2 carry head phases r = 0, 2, 1; the score
    diagonals are exact after Align_r (fused schedule and paper order) and the export stream is K_min(S)."""
    plan, Qh, Kh, qs, ks = _score_case(keys13, 3, 8, 8, 4, 6, 41)
    assert plan.aligned and plan.phases == [0, 2, 1] and plan.k_route == 3
    ev = K.Ev(P13, keys13, plan.m)
    S = K.score(ev, plan, qs, ks)
    assert S[0].L == 2
    ref = K.score_reference(Qh, Kh)
    got, scale = _check_scores(keys13, plan, S, ref)
    E = K.score_export(ev, plan, S)
    stream = np.concatenate([dec(P13, keys13, e) for e in E])
    want = np.concatenate(ref)
    assert len(E) == plan.n_out and np.abs(stream[:len(want)] - want).max() / scale < TOL
    Sp = PO.score(K.Ev(P13, keys13, plan.m), plan, qs, ks, ts=[0, 5, 7])
    for t, sp in zip([0, 5, 7], Sp):
        zp = dec(P13, keys13, sp)
        assert np.abs(zp[:plan.H * plan.m] - ref[t]).max() / scale < TOL
        assert np.abs(zp - got[t]).max() / scale < TOL


def test_score_and_export_fused_vs_paper_order(keys13):
    plan, Qh, Kh, qs, ks = _score_case(keys13, 4, 8, 16, 4, 6, 40)
    assert not plan.aligned
    ref = K.score_reference(Qh, Kh)
    ev = K.Ev(P13, keys13, plan.m)
    S = K.score(ev, plan, qs, ks)
    evp = K.Ev(P13, keys13, plan.m)
    Sp = PO.score(evp, plan, qs, ks)
    got, scale = _check_scores(keys13, plan, S, ref)
    gotp, _ = _check_scores(keys13, plan, Sp, ref)
    for a, b in zip(got, gotp):
        assert np.abs(a - b).max() / scale < TOL
    E, Ep = K.score_export(ev, plan, S), PO.score_export(evp, plan, Sp)
    for e, ep in zip(E, Ep):
        assert np.abs(dec(P13, keys13, e) - dec(P13, keys13, ep)).max() / scale < TOL
    # the paper's tree routes with sequential single rotations, the build with one hoisted sum per t
    assert evp.ledger["relin"] == ev.ledger["relin"] == plan.m // 2


# ------------------------------------------------------------------ value
def test_value_fused_vs_paper_order(keys13):
    m, H, dh = 16, 4, 8
    plan = K.ValuePlan(P13.n, m, H, dh, H_blk=2)
    Ph = synth.attention_probs(H, m, 41)
    Vh = synth.uniform((H, m, dh), 42)
    vs = [enc(P13, keys13, K.value_v_slots(Vh, plan, l), 6, 300 + l) for l in range(plan.B_V)]
    ps = [enc(P13, keys13, K.value_p_slots(Ph, plan, l), 4, 400 + l) for l in range(plan.B_V)]
    outs = K.value(K.Ev(P13, keys13, m), plan, ps, vs)
    outp = PO.value(K.Ev(P13, keys13, m), plan, ps, vs)
    ref = K.value_reference(Ph, Vh)
    sc = np.abs(ref).max()
    for l, (o, op) in enumerate(zip(outs, outp)):
        a, b = dec(P13, keys13, o).real, dec(P13, keys13, op).real
        assert np.abs(a - b).max() / sc < TOL
        for hh in range(plan.H_blk):
            h = l * plan.H_blk + hh
            for u in range(dh):
                s = hh * plan.seg_stride + u
                assert np.abs(b[s * m:(s + 1) * m] - ref[h][:, u]).max() / sc < TOL
