"""GPU parity (through the C ABI) for the round-2 rows: RotFirst_L / Psi as standalone calls, the restricted
projection (C < n/m: Phi_C bank and giant fold, Alg A.4), the score kernel with head-phase alignment
(C mod H != 0: Align_r, App. A.3) and the value kernel's unit-range partials (the multi-GPU partition).  Every
limb of every output equals the oracle's; decryptions meet the 2^-20 target."""
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

P13 = O.Params("P13")
TOL = 2.0 ** -20


@pytest.fixture(scope="module")
def c13():
    return E.Context("P13", 0)


@pytest.fixture(scope="module")
def keys13(c13):
    from tests.test_oracle_kernels import _galois13
    g = _galois13()
    return O.Keys(P13, synth.SEED_KEYS, galois=g, relin=True), c13.keygen(synth.SEED_KEYS, galois=g, relin=True)


def dec(keys, ct):
    return O.decode(P13, O.decrypt(P13, keys, ct))


@pytest.mark.parametrize("Ls,taus", [(3, [1, 0, 2]), (20, [7, 13]), (16 * 128, [0, 16, 16 * 127]), (48, [16, 32])])
def test_rotfirst_bit_exact(c13, keys13, Ls, taus):
    ok, gk = keys13
    m = 16
    z = synth.complex_slots(P13.n, 7)
    z[Ls:] = 0
    x = O.encrypt_sk(P13, ok, O.encode(P13, z, 2.0 ** 40, 5), 11)
    ev = K.Ev(P13, ok, m)
    ref = K.RotFirst_hoisted(ev, x, Ls, taus, m)
    c13.mask_clear()
    install_masks(c13, ev)
    got = c13.rotfirst(gk, dev_ct(c13, x), Ls, taus, m)
    for tau, g, r in zip(taus, got, ref):
        assert_ct_equal(c13, g, r, "RotFirst_%d(%d)" % (Ls, tau))
        assert np.abs(dec(ok, r) - K.rotfirst_reference(z, Ls, tau % Ls)).max() < 2e-6
    c13.mask_clear()


def test_psi_bit_exact(c13, keys13):
    ok, gk = keys13
    m = 16
    x = O.encrypt_sk(P13, ok, O.encode(P13, synth.complex_slots(P13.n, 8), 2.0 ** 40, 4), 12)
    ts = [0, 3, -5, 15]
    ev = K.Ev(P13, ok, m)
    ref = K.Psi_hoisted(ev, x, ts, m, P13.n // m)
    c13.mask_clear()
    install_masks(c13, ev)
    for t, g, r in zip(ts, c13.psi(gk, dev_ct(c13, x), m, ts), ref):
        assert_ct_equal(c13, g, r, "Psi^%d" % t)
    c13.mask_clear()


def test_projection_restricted_C_bit_exact(c13, keys13):
    """P13, m = 16, C = 128 < N_seg = 256 (Phi_C bank + fold, R-PHIC): bit-exact, y_b at L - 3, X W within 2^-20;
    then the same projection split into two unit ranges (extended partials at the bank level) reduces to the
    same bits."""
    ok, gk = keys13
    m, d_in, d_out, L = 16, 300, 200, 6
    plan = E.ProjPlan(c13, m, d_in, d_out, C=128, N1=8)
    oplan = K.ProjPlan(P13.n, m, d_in, d_out, C=128, N1=8)
    assert oplan.restricted and (plan.C, plan.U, plan.B_out, plan.N1, plan.N2) == (128, 2, 2, 8, 16)
    X = synth.fixed_point_uniform((m, d_in), 30)
    W = synth.bert_weight((d_in, d_out), 31)
    Lw = oplan.weight_level(L)
    xs = [O.encrypt_sk(P13, ok, O.encode(P13, z, 2.0 ** 40, L), synth.seed_enc(u)) for u, z in enumerate(K.proj_inputs(X, oplan))]
    pts = {}

    def w(b, p, u, q):
        if (b, p, u, q) not in pts:
            pts[(b, p, u, q)] = O.encode(P13, K.proj_weight_slots(W, oplan, b, p, u, q), float(P13.q[Lw - 1]), Lw)
        return pts[(b, p, u, q)]
    ev = K.Ev(P13, ok, m)
    ys = K.projection(ev, oplan, xs, w)
    order = [w(b, p, u, q) for b in range(oplan.B_out) for p in range(oplan.N2) for u in range(oplan.U) for q in range(oplan.N1)]
    wd = weights_tensor(c13, order, Lw)
    c13.mask_clear()
    install_masks(c13, ev)
    xd = [dev_ct(c13, x) for x in xs]
    got = plan.matmul(gk, xd, wd, float(P13.q[Lw - 1]))
    for b, (g, r) in enumerate(zip(got, ys)):
        assert g.n_limbs == L - 3
        assert_ct_equal(c13, g, r, "restricted projection y_%d" % b)
    Y = np.concatenate([K.seg_column_unpack(dec(ok, y).real, m, 128, d_out, b) for b, y in enumerate(ys)], axis=1)
    assert np.abs(Y - X @ W).max() / np.abs(X @ W).max() < TOL
    units = plan.B_out * plan.N2
    cut = units // 2 + 5
    a = plan.matmul(gk, xd, wd, float(P13.q[Lw - 1]), 0, cut, finalize=False)
    b = plan.matmul(gk, xd, wd, float(P13.q[Lw - 1]), cut, units, finalize=False)
    assert a[-1].n_limbs == Lw + len(P13.p)
    bs = cut // plan.N2
    s = a[bs].data + b[0].data
    c13.mod_reduce_ext(s, 2, Lw)
    a[bs].data = s
    yfin = plan.finalize(gk, a[:bs] + [a[bs]] + b[1:], 0)
    for bb, (g, r) in enumerate(zip(yfin, ys)):
        assert_ct_equal(c13, g, r, "split restricted projection y_%d" % bb)
    c13.mask_clear()


def test_score_phase_alignment_bit_exact(c13, keys13):
    """H = 3, C = 8: phases (0, 2, 1), Align_r per phase; S_t and the export stream bit-exact, S_t at L - 4."""
    ok, gk = keys13
    m, H, dh = 16, 3, 8
    plan = E.AttnPlan(c13, m, H, dh, C_qk=8, beta=4)
    oplan = K.ScorePlan(P13.n, m, H, dh, C_qk=8, beta=4)
    assert oplan.aligned and plan.B == oplan.B == 3
    g = synth.rng(41)
    Qh, Kh = g.uniform(-1, 1, (H, m, dh)), g.uniform(-1, 1, (H, m, dh))
    perm = K.pi_S(H, dh)
    Qp, Kp = np.concatenate(list(Qh), 1)[:, perm], np.concatenate(list(Kh), 1)[:, perm]
    L0 = 6
    qs = [O.encrypt_sk(P13, ok, O.encode(P13, K.score_qk_slots(Qp, oplan, l), 2.0 ** 40, L0), 100 + l) for l in range(oplan.B)]
    ks = [O.encrypt_sk(P13, ok, O.encode(P13, K.score_qk_slots(Kp, oplan, l), 2.0 ** 40, L0), 200 + l) for l in range(oplan.B)]
    ev = K.Ev(P13, ok, m)
    S = K.score(ev, oplan, qs, ks)
    Ex = K.score_export(ev, oplan, S)
    c13.mask_clear()
    install_masks(c13, ev)
    gS = plan.score(gk, [dev_ct(c13, x) for x in qs], [dev_ct(c13, x) for x in ks])
    for t, (a, b) in enumerate(zip(gS, S)):
        assert a.n_limbs == L0 - 4
        assert_ct_equal(c13, a, b, "aligned S_%d" % t)
    for a, b in zip(plan.export_stream(gk, gS), Ex):
        assert_ct_equal(c13, a, b, "aligned export stream")
    ref = K.score_reference(Qh, Kh)
    scale = max(np.abs(r).max() for r in ref)
    for t in (0, 3, 7):
        assert np.abs(dec(ok, S[t])[:H * m] - ref[t]).max() / scale < TOL
    c13.mask_clear()


def test_value_unit_partials_bit_exact(c13, keys13):
    """The value kernel split into three unit ranges that straddle block boundaries: each partial equals the
    oracle's value_partial, and the uint64 sum of the partials of a block + mod-reduce + finalize equals the
    1-GPU value kernel (and the oracle) on every limb."""
    ok, gk = keys13
    m, H, dh = 16, 4, 8
    plan = E.AttnPlan(c13, m, H, dh, H_blk=2)
    oplan = K.ValuePlan(P13.n, m, H, dh, H_blk=2)
    Ph = synth.attention_probs(H, m, 41)
    Vh = synth.uniform((H, m, dh), 42)
    vs = [O.encrypt_sk(P13, ok, O.encode(P13, K.value_v_slots(Vh, oplan, l), 2.0 ** 40, 6), 300 + l) for l in range(oplan.B_V)]
    ps = [O.encrypt_sk(P13, ok, O.encode(P13, K.value_p_slots(Ph, oplan, l), 2.0 ** 40, 4), 400 + l) for l in range(oplan.B_V)]
    ev = K.Ev(P13, ok, m)
    outs = K.value(ev, oplan, ps, vs)
    ranges = [(0, 5), (5, 11), (11, 16)]
    oparts = [K.value_partial(ev, oplan, ps, vs, a, b) for a, b in ranges]
    c13.mask_clear()
    install_masks(c13, ev)
    pd, vd = [dev_ct(c13, x) for x in ps], [dev_ct(c13, x) for x in vs]
    full = plan.value(gk, pd, vd)
    for a, b in zip(full, outs):
        assert_ct_equal(c13, a, b, "value")
    sums = {}
    for (a, b), op in zip(ranges, oparts):
        blocks = plan.value_blocks(a, b)
        assert blocks == sorted(op)
        for l, part in zip(blocks, plan.value_partial(gk, pd, vd, a, b)):
            assert_ct_equal(c13, part, op[l], "value partial %s block %d" % ((a, b), l))
            sums[l] = part.data.clone() if l not in sums else sums[l] + part.data
    o3 = []
    for l in range(plan.B_V):
        c13.mod_reduce(sums[l], 3, ps[0].L - 1)
        o3.append(E.Ciphertext(sums[l], 3, ps[0].L - 1, oparts[0][0].scale, 1))
    for a, b in zip(plan.value_finalize(gk, o3), outs):
        assert_ct_equal(c13, a, b, "value from partials")
    c13.mask_clear()


def test_guards_reject_bad_inputs(c13, keys13):
    """Host-side validation before any launch: n_limbs outside [1, L_max] and misaligned data are refused
    (ENCF_ERR_LEVEL_MISMATCH / ENCF_ERR_ARG), the value level plan is checked (Lv > Lp)."""
    ok, gk = keys13
    x = dev_ct(c13, O.encrypt_sk(P13, ok, O.encode(P13, synth.complex_slots(P13.n, 1), 2.0 ** 40, 3), 1))
    bad = E.Ciphertext(x.data, 2, 70, x.scale, 1)
    with pytest.raises(E.EncfError) as e:
        c13.add(bad, bad)
    assert e.value.code == 4
    mis = E.Ciphertext(torch.empty(2 * 3 * P13.N + 1, dtype=torch.int64, device=c13.device)[1:], 2, 3, x.scale, 1)
    with pytest.raises(E.EncfError) as e:
        c13.add(mis, x)
    assert e.value.code == 1
    plan = E.AttnPlan(c13, 16, 4, 8, H_blk=2)
    p4 = dev_ct(c13, O.encrypt_sk(P13, ok, O.encode(P13, synth.complex_slots(P13.n, 2), 2.0 ** 40, 4), 2))
    with pytest.raises(E.EncfError) as e:
        plan.value(gk, [p4, p4], [p4, p4])             # Lv = Lp: no room for the U bank
    assert e.value.code == 4


def test_diag_mac_large_bank_wide_path(c13, keys13):
    """A projection whose bank has U N1 = 384 ciphertexts: on the 60-bit limb q_0 (128-bit MAC path) the sum of 384
    products exceeds 2^128 without the periodic fold; the output stays bit-exact with the oracle."""
    ok, gk = keys13
    m, d_in, d_out, L = 16, 1300, 40, 2
    plan = E.ProjPlan(c13, m, d_in, d_out, N1=128)
    oplan = K.ProjPlan(P13.n, m, d_in, d_out, N1=128)
    assert (oplan.U, oplan.N1, oplan.N2, oplan.B_out) == (3, 128, 2, 1)
    X = synth.fixed_point_uniform((m, d_in), 60)
    W = synth.bert_weight((d_in, d_out), 61)
    xs = [O.encrypt_sk(P13, ok, O.encode(P13, z, 2.0 ** 40, L), 70 + u) for u, z in enumerate(K.proj_inputs(X, oplan))]
    pts = {}

    def w(b, p, u, q):
        if (b, p, u, q) not in pts:
            pts[(b, p, u, q)] = O.encode(P13, K.proj_weight_slots(W, oplan, b, p, u, q), float(P13.q[L - 1]), L)
        return pts[(b, p, u, q)]
    ys = K.projection(K.Ev(P13, ok, m), oplan, xs, w)
    order = [w(b, p, u, q) for b in range(oplan.B_out) for p in range(oplan.N2) for u in range(oplan.U) for q in range(oplan.N1)]
    got = plan.matmul(gk, [dev_ct(c13, x) for x in xs], weights_tensor(c13, order, L), float(P13.q[L - 1]))
    assert_ct_equal(c13, got[0], ys[0], "projection with a 384-ciphertext bank")


def test_ctx_refuses_digit_counts_beyond_single_redc(tmp_path):
    """(2 dnum + 2) q_max >= 2^64 would overflow the single-REDC key-switch sums: P13's primes with alpha = 1
    (dnum = 8, 18 q_0 > 2^64) are refused at context creation (ENCF_ERR_ARG)."""
    import json
    import os
    d = json.load(open(os.path.join(os.path.dirname(__file__), "..", "params", "p13.json")))
    d["alpha"] = 1
    p = tmp_path / "p13a1.json"
    p.write_text(json.dumps(d))
    with pytest.raises(E.EncfError) as e:
        E.Context(str(p), 0)
    assert e.value.code == 1
