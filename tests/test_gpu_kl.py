"""GPU parity for the per-level special-prime count K(L) (DESIGN.md R-KL) on P13A8: N = 2^13, alpha = 8 (one digit
at every level), six 60-bit special primes with K(L) = 2, 2, 3, 4, 4, 5, 6, 6 for L = 1..8 -- the same table as
P16's low levels.  Every key-switching primitive at every level, and the three kernels across the levels they
span, equal the oracle on every limb (the oracle's class keys are pinned against the big-int cross-model's
independently generated ones in tests/test_crossmodel.py)."""
import numpy as np
import pytest

import synth
from oracle import ckks as O
from oracle import kernels as K

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2604_09975_b200 import encf as E  # noqa: E402
from tests.gpu_util import assert_ct_equal, dev_ct, install_masks, weights_tensor  # noqa: E402

PA = O.Params("P13A8")
TOL = 2.0 ** -20


@pytest.fixture(scope="module")
def ca():
    return E.Context("P13A8", 0)


@pytest.fixture(scope="module")
def keysa(ca):
    from tests.test_oracle_kernels import _galois13
    g = _galois13()
    return O.Keys(PA, synth.SEED_KEYS, galois=g, relin=True), ca.keygen(synth.SEED_KEYS, galois=g, relin=True)


def test_k_of_level_table(ca):
    assert PA.K_of_level == [2, 2, 3, 4, 4, 5, 6, 6] == ca.K_of_level
    assert [ca.ext_limbs(L) for L in range(1, 9)] == [3, 4, 6, 8, 9, 11, 13, 14]


@pytest.mark.parametrize("L", [8, 6, 5, 4, 3, 2])
def test_keyswitch_every_class_bit_exact(ca, keysa, L):
    ok, gk = keysa
    ct = O.encrypt_sk(PA, ok, O.encode(PA, synth.complex_slots(PA.n, 70 + L), 2.0 ** 40, L), 3)
    d = dev_ct(ca, ct)
    assert_ct_equal(ca, ca.rotate(gk, d, 16), O.rotate(PA, ok, ct, 16), "rotate L=%d K=%d" % (L, PA.K(L)))
    for r, h, ref in zip([1, -3, 32], ca.rotate_hoisted(gk, d, [1, -3, 32]), O.rotate_hoisted(PA, ok, ct, [1, -3, 32])):
        assert_ct_equal(ca, h, ref, "hoisted %d L=%d" % (r, L))
    assert_ct_equal(ca, ca.conjugate(gk, d), O.conjugate(PA, ok, ct), "conj L=%d" % L)
    t = O.tensor(PA, ct, ct)
    assert_ct_equal(ca, ca.relinearize(gk, ca.tensor(d, d)), O.relinearize(PA, ok, t), "relin L=%d" % L)
    z = O.decode(PA, O.decrypt(PA, ok, O.rotate(PA, ok, ct, 16)))
    assert np.abs(z - np.roll(synth.complex_slots(PA.n, 70 + L), -16)).max() < 1e-6


def test_projection_score_value_across_classes_bit_exact(ca, keysa):
    """Projection at L = 5 (K = 4), score from L = 7 (K = 6 banks, K = 5 relin, K = 4 routing / align) and value
    (V at 7, P_fd at 5: Phi bank at K = 4, relin at K = 4)."""
    ok, gk = keysa
    m = 16
    # projection
    plan = E.ProjPlan(ca, m, 300, 200, N1=8)
    oplan = K.ProjPlan(PA.n, m, 300, 200, N1=8)
    X = synth.fixed_point_uniform((m, 300), 81)
    W = synth.bert_weight((300, 200), 82)
    L = 5
    xs = [O.encrypt_sk(PA, ok, O.encode(PA, z, 2.0 ** 40, L), 90 + u) for u, z in enumerate(K.proj_inputs(X, oplan))]
    pts = {}

    def w(b, p, u, q):
        if (b, p, u, q) not in pts:
            pts[(b, p, u, q)] = O.encode(PA, K.proj_weight_slots(W, oplan, b, p, u, q), float(PA.q[L - 1]), L)
        return pts[(b, p, u, q)]
    ys = K.projection(K.Ev(PA, ok, m), oplan, xs, w)
    order = [w(b, p, u, q) for b in range(oplan.B_out) for p in range(oplan.N2) for u in range(oplan.U) for q in range(oplan.N1)]
    got = plan.matmul(gk, [dev_ct(ca, x) for x in xs], weights_tensor(ca, order, L), float(PA.q[L - 1]))
    for b, (g_, r) in enumerate(zip(got, ys)):
        assert_ct_equal(ca, g_, r, "projection y_%d (K(5) = 4)" % b)
    Y = np.concatenate([K.seg_column_unpack(O.decode(PA, O.decrypt(PA, ok, y)).real, m, 256, 200, b) for b, y in enumerate(ys)], 1)
    assert np.abs(Y - X @ W).max() / np.abs(X @ W).max() < TOL
    # score
    H, dh = 4, 8
    ap = E.AttnPlan(ca, m, H, dh, C_qk=16, beta=4)
    sp = K.ScorePlan(PA.n, m, H, dh, C_qk=16, beta=4)
    g = synth.rng(83)
    Qh, Kh = g.uniform(-1, 1, (H, m, dh)), g.uniform(-1, 1, (H, m, dh))
    perm = K.pi_S(H, dh)
    Qp, Kp = np.concatenate(list(Qh), 1)[:, perm], np.concatenate(list(Kh), 1)[:, perm]
    qs = [O.encrypt_sk(PA, ok, O.encode(PA, K.score_qk_slots(Qp, sp, l), 2.0 ** 40, 7), 100 + l) for l in range(sp.B)]
    ks = [O.encrypt_sk(PA, ok, O.encode(PA, K.score_qk_slots(Kp, sp, l), 2.0 ** 40, 7), 200 + l) for l in range(sp.B)]
    ev = K.Ev(PA, ok, m)
    S = K.score(ev, sp, qs, ks)
    Ex = K.score_export(ev, sp, S)
    ca.mask_clear()
    install_masks(ca, ev)
    gS = ap.score(gk, [dev_ct(ca, x) for x in qs], [dev_ct(ca, x) for x in ks])
    for t, (a, b) in enumerate(zip(gS, S)):
        assert_ct_equal(ca, a, b, "S_%d" % t)
    for a, b in zip(ap.export_stream(gk, gS), Ex):
        assert_ct_equal(ca, a, b, "export stream")
    ref = K.score_reference(Qh, Kh)
    scale = max(np.abs(r).max() for r in ref)
    for t in (0, 7):
        assert np.abs(O.decode(PA, O.decrypt(PA, ok, S[t]))[:H * m] - ref[t]).max() / scale < TOL
    # value
    vp = K.ValuePlan(PA.n, m, H, dh, H_blk=2)
    av = E.AttnPlan(ca, m, H, dh, H_blk=2)
    Ph = synth.attention_probs(H, m, 84)
    Vh = synth.uniform((H, m, dh), 85)
    vs = [O.encrypt_sk(PA, ok, O.encode(PA, K.value_v_slots(Vh, vp, l), 2.0 ** 40, 7), 300 + l) for l in range(vp.B_V)]
    ps = [O.encrypt_sk(PA, ok, O.encode(PA, K.value_p_slots(Ph, vp, l), 2.0 ** 44, 5), 400 + l) for l in range(vp.B_V)]
    ev = K.Ev(PA, ok, m)
    outs = K.value(ev, vp, ps, vs)
    ca.mask_clear()
    install_masks(ca, ev)
    for a, b in zip(av.value(gk, [dev_ct(ca, x) for x in ps], [dev_ct(ca, x) for x in vs]), outs):
        assert_ct_equal(ca, a, b, "value")
    refv = K.value_reference(Ph, Vh)
    got = O.decode(PA, O.decrypt(PA, ok, outs[0])).real
    assert np.abs(got[:m] - refv[0][:, 0]).max() / np.abs(refv).max() < TOL
    ca.mask_clear()
