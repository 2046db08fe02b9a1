"""T3/T4/T5 for the oracle kernels: decrypted outputs against textbook float64 definitions
(projection = X W, score diagonals = brute-force Q K^T, value = P V), slot-level examples, and the
paper's key-switch counts (Table 2) reproduced by running the same schedule in
count-only mode at the paper's own shapes."""
import numpy as np
import pytest

import synth
from oracle import ckks as O
from oracle import kernels as K

P12 = O.Params("P12")
P13 = O.Params("P13")
TOL = 2.0 ** -20   # north_star: 2^-20 relative (||dec - ref||_inf / ||ref||_inf, G28)


def rel_err(got, ref):
    return np.abs(got - ref).max() / np.abs(ref).max()


def enc(P, keys, z, L, seed, scale=2.0 ** 40):
    return O.encrypt_sk(P, keys, O.encode(P, z, scale, L), seed)


def dec(P, keys, ct):
    return O.decode(P, O.decrypt(P, keys, ct))


# ------------------------------------------------------------------ slot-level definitions (SPEC examples)
def test_shift_definitions_toy():
    # m=2, N_seg=2, x=(a,b,c,d): Phi^1 -> (c,d,a,b), Psi^1 -> (b,a,d,c)
    x = np.array([1.0, 2.0, 3.0, 4.0])
    assert np.array_equal(np.roll(x, -1 * 2), [3, 4, 1, 2])                     # rot(x; Delta m)
    Xm = K.mat(x, 2)
    psi = K.vec(np.roll(Xm, -1, axis=0))
    assert np.array_equal(psi, [2, 1, 4, 3])
    assert np.array_equal(K.vec(K.mat(x, 2)), x)


def test_k_min_paper_table4():
    # Table 4: Softmax 6, LN1 3, GELU 12, LN2 3 at n = 16384
    n = 16384
    assert K.k_min(12 * 128 * 128, n) == 6
    assert K.k_min(128 * 768, n) == 3
    assert K.k_min(128 * 3072, n) == 12
    # N_seg=256 at N=2^16, m=128: K_min(S) = 3
    assert K.k_min(12 * 128 * 128, 32768) == 3


def test_pi_S_matches_definition():
    H, dh = 3, 4
    W = np.arange(5 * H * dh).reshape(5, H * dh).astype(float)
    Wp = K.apply_col_perm(W, K.pi_S(H, dh))
    for h in range(H):
        for u in range(dh):
            assert np.array_equal(Wp[:, u * H + h], W[:, h * dh + u])


def test_proj_weight_slots_reconstruct_matmul_in_clear():
    """Slot-level model of C6 without encryption: sum over (u,q) and Phi^{pN1} fold and Re reproduce XW."""
    n, m, d_in, d_out = 64, 4, 40, 20
    plan = K.ProjPlan(n, m, d_in, d_out, N1=4)
    X = synth.uniform((m, d_in), 1)
    W = synth.uniform((d_in, d_out), 2)
    xt = K.proj_inputs(X, plan)
    for b in range(plan.B_out):
        acc = np.zeros(n, complex)
        for p in range(plan.N2):
            c = np.zeros(n, complex)
            for u in range(plan.U):
                for q in range(plan.N1):
                    c += np.roll(xt[u], -q * m) * K.proj_weight_slots(W, plan, b, p, u, q)
            acc += np.roll(c, -p * plan.N1 * m)
        Y = K.seg_column_unpack(acc.real, m, plan.C, d_out, b)
        assert np.allclose(Y, (X @ W)[:, b * plan.C: b * plan.C + Y.shape[1]], atol=1e-12)


# ------------------------------------------------------------------ encrypted kernels
@pytest.fixture(scope="module")
def keys12():
    plan = K.ProjPlan(P12.n, 32, 64, 64, N1=8)
    rots = [q * plan.m for q in range(1, plan.N1)] + [p * plan.N1 * plan.m for p in range(1, plan.N2)]
    return O.Keys(P12, synth.SEED_KEYS, galois=[O.galois_rot(P12, r) for r in rots] + [O.galois_conj(P12)])


def run_projection(P, keys, X, W, plan, L):
    ev = K.Ev(P, keys, plan.m)
    xs = [enc(P, keys, z, L, synth.seed_enc(u)) for u, z in enumerate(K.proj_inputs(X, plan))]
    wcache = {}

    def w(b, p, u, q):
        key = (b, p, u, q)
        if key not in wcache:
            wcache[key] = O.encode(P, K.proj_weight_slots(W, plan, b, p, u, q), float(P.q[L - 1]), L)
        return wcache[key]
    ys = K.projection(ev, plan, xs, w)
    return ev, ys


def test_projection_config1(keys12):
    """Config 1 (BASELINE configs[0]): N=2^12, 3 limbs, 64x64 single-ciphertext diagonal matvec (m=32 rows)."""
    plan = K.ProjPlan(P12.n, 32, 64, 64, N1=8)
    assert (plan.C, plan.U, plan.B_out, plan.N1, plan.N2) == (64, 1, 1, 8, 8)
    X = synth.fixed_point_uniform((32, 64), synth.seed_data(1))
    W = synth.uniform((64, 64), synth.seed_data(1) + 100, -0.125, 0.125)
    ev, ys = run_projection(P12, keys12, X, W, plan, 3)
    assert ys[0].L == 2
    Y = K.seg_column_unpack(dec(P12, keys12, ys[0]).real, 32, 64, 64, 0)
    assert rel_err(Y, X @ W) < TOL
    assert ev.ledger["rot"] == 7 + 7 and ev.ledger["conj"] == 1 and ev.ledger["ptmul"] == 64


def test_projection_identity_input(keys12):
    """X = I gives Y = W."""
    plan = K.ProjPlan(P12.n, 32, 64, 64, N1=8)
    X = np.zeros((32, 64)); X[np.arange(32), np.arange(32)] = 1.0
    W = synth.uniform((64, 64), 5, -0.125, 0.125)
    _, ys = run_projection(P12, keys12, X, W, plan, 3)
    Y = K.seg_column_unpack(dec(P12, keys12, ys[0]).real, 32, 64, 64, 0)
    assert rel_err(Y, (X @ W)) < TOL and np.allclose(Y[:32, :], W[:32, :], atol=1e-5)


@pytest.fixture(scope="module")
def keys13():
    return O.Keys(P13, synth.SEED_KEYS, galois=_galois13(), relin=True)


def _galois13():
    n = P13.n
    steps = set()
    # projection (m=16, N1=8, N2=C/N1)
    for m, N1, C in [(16, 8, 256)]:
        steps |= {q * m for q in range(1, N1)} | {p * N1 * m for p in range(1, C // N1)}
    # score / value (m=16)
    m = 16
    steps |= {t for t in range(-m, m)} | {d * m for d in range(-(m // 2), m // 2)}
    steps |= {j * m for j in range(1, 256)}                      # routing strides
    steps |= {-(o) for o in range(0, n, m)}                     # export offsets (segment aligned)
    return sorted({O.galois_rot(P13, r) for r in steps if r % n}) + [O.galois_conj(P13)]


def test_projection_ragged_two_inputs(keys13):
    """U=2 complexified inputs with G odd, d_out not a multiple of C (ragged tail), N1=8 at N=2^13."""
    plan = K.ProjPlan(P13.n, 16, 600, 300, N1=8)
    assert (plan.C, plan.G, plan.U, plan.B_out) == (256, 3, 2, 2)
    X = synth.fixed_point_uniform((16, 600), 7)
    W = synth.bert_weight((600, 300), 8)
    ev, ys = run_projection(P13, keys13, X, W, plan, 4)
    Y = np.concatenate([K.seg_column_unpack(dec(P13, keys13, y).real, 16, 256, 300, b) for b, y in enumerate(ys)], axis=1)
    assert rel_err(Y, X @ W) < TOL


def test_score_kernel_brute_force(keys13):
    n, m, H, dh = P13.n, 16, 4, 8
    plan = K.ScorePlan(n, m, H, dh, C_qk=16, beta=4)
    assert plan.B == 2 and plan.n_out == 1
    g = synth.rng(40)
    Qh = g.uniform(-1, 1, (H, m, dh)); Kh = g.uniform(-1, 1, (H, m, dh))
    Q = np.concatenate(list(Qh), axis=1); Kk = np.concatenate(list(Kh), axis=1)   # head-major columns
    perm = K.pi_S(H, dh)
    Qp, Kp = Q[:, perm], Kk[:, perm]
    ev = K.Ev(P13, keys13, m)
    L0 = 6
    qs = [enc(P13, keys13, K.score_qk_slots(Qp, plan, l), L0, 100 + l) for l in range(plan.B)]
    ks = [enc(P13, keys13, K.score_qk_slots(Kp, plan, l), L0, 200 + l) for l in range(plan.B)]
    S = K.score(ev, plan, qs, ks)
    ref = K.score_reference(Qh, Kh)
    scale = max(np.abs(r).max() for r in ref)
    for t in range(m // 2):
        got = dec(P13, keys13, S[t])
        assert np.abs(got[:H * m] - ref[t]).max() / scale < TOL
        assert np.abs(got[H * m:]).max() / scale < TOL            # cut(): only the first Hm slots carry data
    E = K.score_export(ev, plan, S)
    assert len(E) == plan.n_out
    stream = np.concatenate([dec(P13, keys13, e) for e in E])
    want = np.concatenate(ref)
    assert np.abs(stream[:len(want)] - want).max() / scale < TOL
    assert ev.ledger["ctmul"] == (m // 2) * plan.B


def test_value_kernel_brute_force(keys13):
    n, m, H, dh = P13.n, 16, 4, 8
    plan = K.ValuePlan(n, m, H, dh, H_blk=2)
    assert plan.B_V == 2
    Ph = synth.attention_probs(H, m, 41)
    Vh = synth.uniform((H, m, dh), 42)
    ev = K.Ev(P13, keys13, m)
    vs = [enc(P13, keys13, K.value_v_slots(Vh, plan, l), 6, 300 + l) for l in range(plan.B_V)]
    ps = [enc(P13, keys13, K.value_p_slots(Ph, plan, l), 4, 400 + l) for l in range(plan.B_V)]
    outs = K.value(ev, plan, ps, vs)
    ref = K.value_reference(Ph, Vh)
    for l, o in enumerate(outs):
        got = dec(P13, keys13, o).real
        for hh in range(plan.H_blk):
            h = l * plan.H_blk + hh
            for u in range(dh):
                s = hh * plan.seg_stride + u
                assert np.abs(got[s * m:(s + 1) * m] - ref[h][:, u]).max() / np.abs(ref).max() < TOL
    assert ev.ledger["rot"] == plan.B_V * (2 + 2 * (m // 2 - 1) + (dh - 1 + m // 2 - 1))


def test_value_identity_attention(keys13):
    """identity attention P = I gives O = V."""
    n, m, H, dh = P13.n, 16, 2, 8
    plan = K.ValuePlan(n, m, H, dh, H_blk=2)
    Ph = np.stack([np.eye(m)] * H)
    Vh = synth.uniform((H, m, dh), 43)
    ev = K.Ev(P13, keys13, m)
    vs = [enc(P13, keys13, K.value_v_slots(Vh, plan, 0), 6, 1)]
    ps = [enc(P13, keys13, K.value_p_slots(Ph, plan, 0), 4, 2)]
    got = dec(P13, keys13, K.value(ev, plan, ps, vs)[0]).real
    for h in range(H):
        for u in range(dh):
            s = h * plan.seg_stride + u
            assert np.abs(got[s * m:(s + 1) * m] - Vh[h][:, u]).max() < 1e-5


def test_export_c2m_shares_reconstruct(keys13):
    """Alg 3: Dec(<m> + r^) + (-r^) == Dec(<m>) (mod Q_conv) exactly; Re/Im carry x and y."""
    P = P13
    x = synth.fixed_point_uniform(P.n, 50)
    y = synth.fixed_point_uniform(P.n, 51)
    cx, cy = enc(P, keys13, x, 5, 1), enc(P, keys13, y, 5, 2)
    ct = O.complexify(P, cx, cy)
    Lc = 2
    masked, share = K.export_c2m(P, ct, Lc, synth.seed_mask(0), 0)
    t0 = O.decrypt(P, keys13, masked).m
    recon = O.padd(t0, share, P.q[:Lc], P.N)
    plain = O.decrypt(P, keys13, O.mod_drop(P, ct, Lc)).m
    assert np.array_equal(recon, plain)
    z = O.decode(P, O.Pt(recon, ct.scale))
    assert np.abs(z.real - x).max() < 1e-6 and np.abs(z.imag - y).max() < 1e-6
    # P0's decryption alone is masked: it differs from the plaintext on (almost) every coefficient
    assert np.mean(t0 == plain) < 1e-3


def test_l_conv_rule():
    """P:872-876 with ell = 43, sigma = 40: under P16 L_conv = 2 (60 + 40 = 100 bits >= 84)."""
    assert K.l_conv(O.Params("P16")) == 2
    assert K.l_conv(O.Params("P16"), ell=43, sigma=40, B_max=2.0 ** 60) is None or K.l_conv(O.Params("P16"), B_max=2.0 ** 60) > 2


# ------------------------------------------------------------------ Table 2 counts (paper's own shapes, count-only)
def test_value_counts_table2():
    """BERT-base, n = 16384, m = 128, d_h = 64, B_V = 6: 1524 rotations and 384 ct-ct products."""
    plan = K.ValuePlan(16384, 128, 12, 64)
    assert plan.B_V == 6
    ev = K.CountEv(16384)
    K.value(ev, plan, [K.FakeCt(4)] * 6, [K.FakeCt(7)] * 6)
    assert ev.ledger["rot"] == 1524
    assert ev.ledger["ctmul"] == 384


def test_score_counts_table2():
    """BERT-base, n = 16384, B = 7, beta = 16, g = 8, m = 128, C = 120: 448 ct-ct products exactly and
    630 rotations within the +-20 % band the paper's unstated caching allows (G23)."""
    plan = K.ScorePlan(16384, 128, 12, 64, C_qk=120, beta=16)
    assert plan.B == 7 and plan.g == 8
    ev = K.CountEv(16384)
    S = K.score(ev, plan, [K.FakeCt(7)] * 7, [K.FakeCt(7)] * 7)
    K.score_export(ev, plan, S)
    assert ev.ledger["ctmul"] == 448
    assert 0.8 * 630 <= ev.ledger["rot"] <= 1.2 * 630
