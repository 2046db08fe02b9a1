"""Full-size parity at BASELINE.json's sizes (N = 2^16, P16) in the launch configuration bench.py times.

The GPU runs the whole kernel (every block / every t) exactly as in the bench; the oracle computes a
SAMPLE of the outputs one by one (output block b = 0 of the QKV projection, diagonal pairs t in
{0, 17, 63} of the score kernel, block 0 of the value kernel), which must agree on every limb.  All
other outputs are checked through properties that hold at any size: decryption against the float64
plaintext definition within 2^-20 (north_star; G28)."""
import numpy as np
import pytest

import synth
from oracle import ckks as O
from oracle import kernels as K

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2604_09975_b200 import encf as E  # noqa: E402
from tests.gpu_util import assert_ct_equal, dev_ct, install_masks  # noqa: E402

P = O.Params("P16")
M, D, H, DH = 128, 768, 12, 64
TOL = 2.0 ** -20


@pytest.fixture(scope="module")
def ctx():
    return E.Context("P16", 0)


def _dec(keys, ct):
    return O.decode(P, O.decrypt(P, keys, ct))


def qkv_wbar(WQ, WK, WV, C=256, C_qk=192):
    """Pre-permuted (pi_S, App. A.2) and G8-padded QKV weight, built with the ORACLE's helpers."""
    perm = K.pi_S(H, DH)
    nqk = -(-(H * DH) // C_qk)
    W = np.zeros((D, (2 * nqk + 3) * C))
    for i, Wm in enumerate((K.apply_col_perm(WQ, perm), K.apply_col_perm(WK, perm))):
        for b in range(nqk):
            W[:, (i * nqk + b) * C:(i * nqk + b) * C + C_qk] = Wm[:, b * C_qk:(b + 1) * C_qk]
    W[:, 2 * nqk * C:] = WV
    return W


def test_qkv_projection_config3_block0_bit_exact(ctx):
    """Config 3: X 128x768 -> [Q^pi_S | K^pi_S | V] (11 output blocks), L = 8 -> 7."""
    L = 8
    X = synth.fixed_point_uniform((M, D), synth.seed_data(3))
    Wbar = qkv_wbar(*(synth.bert_weight((D, D), synth.seed_data(3) + i) for i in range(3)))
    plan = E.ProjPlan(ctx, M, D, Wbar.shape[1])
    oplan = K.ProjPlan(P.n, M, D, Wbar.shape[1])
    assert (plan.U, plan.B_out, plan.N1, plan.N2) == (oplan.U, oplan.B_out, oplan.N1, oplan.N2) == (2, 11, 32, 8)
    g_oracle = [O.galois_rot(P, q * M) for q in range(1, oplan.N1)] + \
               [O.galois_rot(P, p * oplan.N1 * M) for p in range(1, oplan.N2)] + [O.galois_conj(P)]
    okeys = O.Keys(P, synth.SEED_KEYS, galois=g_oracle, max_level=L)
    gkeys = ctx.keygen(synth.SEED_KEYS, galois=plan.galois(), max_level=L)
    xs = [O.encrypt_sk(P, okeys, O.encode(P, z, 2.0 ** 40, L), synth.seed_enc(u)) for u, z in enumerate(K.proj_inputs(X, oplan))]
    cache = {}

    def w(b, p, u, q):
        if (b, p, u, q) not in cache:
            cache[(b, p, u, q)] = O.encode(P, K.proj_weight_slots(Wbar, oplan, b, p, u, q), float(P.q[L - 1]), L)
        return cache[(b, p, u, q)]
    ev = K.Ev(P, okeys, M)
    y0 = K.projection_finalize(ev, oplan, K.projection_partial(ev, oplan, xs, w, 0, oplan.N2)[0])
    # device weights: GPU-encoded stream, block 0 replaced by the oracle's encodings (bit-exact inputs)
    wd = plan.encode_weights(Wbar, L)
    n0 = oplan.N2 * oplan.U * oplan.N1
    pts = [w(0, p, u, q) for p in range(oplan.N2) for u in range(oplan.U) for q in range(oplan.N1)]
    blk = torch.from_numpy(np.ascontiguousarray(np.stack([pt.m for pt in pts])).view(np.int64).reshape(-1).copy()).to(ctx.device)
    ctx.poly_to_ntt(blk, n0, L)
    wd[:blk.numel()] = blk
    ys = plan.matmul(gkeys, [dev_ct(ctx, x) for x in xs], wd, float(P.q[L - 1]))
    assert_ct_equal(ctx, ys[0], y0, "QKV y_0 (N=2^16, L=8)")
    Y = X @ Wbar
    for b, y in enumerate(ys):
        got = K.seg_column_unpack(_dec(okeys, O.Ct(ctx.to_host(y), y.scale)).real, M, 256, Wbar.shape[1], b)
        ref = Y[:, b * 256:(b + 1) * 256]
        assert np.abs(got - ref).max() / np.abs(Y).max() < TOL, b


def _score_case(ctx, H, ts, B_nout):
    L = 7
    plan = E.AttnPlan(ctx, M, H, DH, C_qk=192, beta=16)
    oplan = K.ScorePlan(P.n, M, H, DH, C_qk=192, beta=16)
    assert (plan.B, plan.n_out) == (oplan.B, oplan.n_out) == B_nout
    g = synth.rng(synth.seed_data(4) + H)
    Qh = g.uniform(-1, 1, (H, M, DH)) / np.sqrt(8)
    Kh = g.uniform(-1, 1, (H, M, DH)) / np.sqrt(8)
    perm = K.pi_S(H, DH)
    Qp, Kp = np.concatenate(list(Qh), 1)[:, perm], np.concatenate(list(Kh), 1)[:, perm]
    steps = set()
    for s in range(1, oplan.beta):
        steps |= {M - s, -s}           # Psi^{-s}: rot by t' = (-s mod m) = m - s and t' - m = -s
    for tau in [j * oplan.beta for j in range(1, oplan.g // 2)] + [M // 2 + j * oplan.beta for j in range(oplan.g // 2)]:
        steps |= {tau, tau - M}
    for t in ts:
        s = t % oplan.beta
        if s:
            steps |= {s, s - M}
    for k in range(1, oplan.C // H):    # routing shifts Phi^{kH} (hoisted sum, DESIGN.md R-ROUTE)
        steps.add(k * H * M)
    og = sorted({O.galois_rot(P, r) for r in steps if r % P.n})
    okeys = O.Keys(P, synth.SEED_KEYS, galois=og, relin=True, max_level=L)
    gkeys = ctx.keygen(synth.SEED_KEYS, galois=plan.galois(), relin=True, max_level=L)
    qs = [O.encrypt_sk(P, okeys, O.encode(P, K.score_qk_slots(Qp, oplan, l), 2.0 ** 40, L), 100 + l) for l in range(oplan.B)]
    ks = [O.encrypt_sk(P, okeys, O.encode(P, K.score_qk_slots(Kp, oplan, l), 2.0 ** 40, L), 200 + l) for l in range(oplan.B)]
    ev = K.Ev(P, okeys, M)
    S_ref = K.score(ev, oplan, qs, ks, ts=ts)
    ctx.mask_clear()
    install_masks(ctx, ev)
    S = plan.score(gkeys, [dev_ct(ctx, x) for x in qs], [dev_ct(ctx, x) for x in ks])
    for t, ref in zip(ts, S_ref):
        assert_ct_equal(ctx, S[t], ref, "S_%d (N=2^16)" % t)
    ref_diag = K.score_reference(Qh, Kh)
    scale = max(np.abs(r).max() for r in ref_diag)
    for t in range(0, M // 2, 7):
        got = _dec(okeys, O.Ct(ctx.to_host(S[t]), S[t].scale))
        assert np.abs(got[:H * M] - ref_diag[t]).max() / scale < TOL, t
    Ex = plan.export_stream(gkeys, S)
    stream = np.concatenate([_dec(okeys, O.Ct(ctx.to_host(e), e.scale)) for e in Ex])
    want = np.concatenate(ref_diag)
    assert np.abs(stream[:len(want)] - want).max() / scale < TOL
    ctx.mask_clear()


def test_score_config4_sampled_t_bit_exact(ctx):
    """Config 4 score: Q, K in 4 padded blocks (C_qk = 192 of 256 segments = 16 channels x 12 heads), beta = 16,
    L = 7; sampled t in {0, 17, 63} against the oracle, every t against brute force, K_min(S) = 3 exports."""
    _score_case(ctx, H, [0, 17, 63], (4, 3))


def test_score_bert_large_sampled_t_bit_exact(ctx):
    """NEXT-row workload BERT-large (H = 16, d = 1024): the same kernel with a new plan --
    C_qk = 192 = 12 channels x 16 heads (phases 0), B = 6 blocks, K_min(S) = 4 exports."""
    _score_case(ctx, 16, [0, 63], (6, 4))


def test_value_config4_block0_bit_exact(ctx):
    """Config 4 value: H = 12, d_h = 64, H_blk = 4, B_V = 3; V at 7 limbs, P_fd at 5 limbs."""
    plan = E.AttnPlan(ctx, M, H, DH)
    oplan = K.ValuePlan(P.n, M, H, DH)
    assert (plan.H_blk, plan.B_V) == (oplan.H_blk, oplan.B_V) == (4, 3)
    Ph = synth.attention_probs(H, M, synth.seed_data(4) + 1)
    # V ~ U[-1,1] (the /sqrt(8) of SURVEY config 4 bounds the Q/K scores; O = P V is a convex combination
    # of V rows, so its scale is ||V||).  Absolute error floor of this kernel at Delta = 2^40: ~2e-7
    # (DESIGN.md "Precision").
    Vh = synth.uniform((H, M, DH), synth.seed_data(4) + 2)
    half = M // 2
    steps = {half, half - M} | {t for t in range(1, half)} | {t - M for t in range(1, half)}
    steps |= {d * M for d in range(-(DH - 1), half) if d}
    og = sorted({O.galois_rot(P, r) for r in steps if r % P.n})
    okeys = O.Keys(P, synth.SEED_KEYS, galois=og, relin=True, max_level=7)
    gkeys = ctx.keygen(synth.SEED_KEYS, galois=plan.galois(), relin=True, max_level=7)
    vs = [O.encrypt_sk(P, okeys, O.encode(P, K.value_v_slots(Vh, oplan, l), 2.0 ** 40, 7), 300 + l) for l in range(oplan.B_V)]
    # P_fd imported at Delta * 2^7 (DESIGN.md R-PSCALE: softmax entries are ~1/m)
    ps = [O.encrypt_sk(P, okeys, O.encode(P, K.value_p_slots(Ph, oplan, l), 2.0 ** 47, 5), 400 + l) for l in range(oplan.B_V)]
    ev = K.Ev(P, okeys, M)
    o0 = K.value(ev, oplan, ps, vs, blocks=[0])[0]
    ctx.mask_clear()
    install_masks(ctx, ev)
    outs = plan.value(gkeys, [dev_ct(ctx, x) for x in ps], [dev_ct(ctx, x) for x in vs])
    assert_ct_equal(ctx, outs[0], o0, "value o_0 (N=2^16)")
    ref = K.value_reference(Ph, Vh)
    for l, o in enumerate(outs):
        got = _dec(okeys, O.Ct(ctx.to_host(o), o.scale)).real
        for hh in range(oplan.H_blk):
            h = l * oplan.H_blk + hh
            for u in range(0, DH, 9):
                s = hh * oplan.seg_stride + u
                assert np.abs(got[s * M:(s + 1) * M] - ref[h][:, u]).max() / np.abs(ref).max() < TOL, (l, h, u)
    ctx.mask_clear()


def test_gpt2_ff2_projection_config5_block0_bit_exact(ctx):
    """Config 5 (GPT-2 small linear path, m = 256 tokens, N_seg = C = 128): the FF2 projection 3072 -> 768
    at L = 3 (U = 12 complexified inputs, B_out = 6) exactly as bench.py --workload gpt2-linear launches it;
    output block 0 computed by the oracle must agree on every limb, every block must decrypt to X W."""
    L, m, din, dout = 3, 256, 3072, 768
    X = synth.fixed_point_uniform((m, din), synth.seed_data(5) + 300, 0.0, 1.0)
    W = synth.bert_weight((din, dout), synth.seed_data(5) + 15)
    plan = E.ProjPlan(ctx, m, din, dout)
    oplan = K.ProjPlan(P.n, m, din, dout)
    assert (plan.C, plan.U, plan.B_out, plan.N1, plan.N2) == (oplan.C, oplan.U, oplan.B_out, oplan.N1, oplan.N2)
    assert (plan.C, plan.U, plan.B_out) == (128, 12, 6)
    g_oracle = [O.galois_rot(P, q * m) for q in range(1, oplan.N1)] + \
               [O.galois_rot(P, p * oplan.N1 * m) for p in range(1, oplan.N2)] + [O.galois_conj(P)]
    okeys = O.Keys(P, synth.SEED_KEYS, galois=g_oracle, max_level=L)
    gkeys = ctx.keygen(synth.SEED_KEYS, galois=plan.galois(), max_level=L)
    xs = [O.encrypt_sk(P, okeys, O.encode(P, z, 2.0 ** 40, L), synth.seed_enc(u)) for u, z in enumerate(K.proj_inputs(X, oplan))]
    cache = {}

    def w(b, p, u, q):
        if (b, p, u, q) not in cache:
            cache[(b, p, u, q)] = O.encode(P, K.proj_weight_slots(W, oplan, b, p, u, q), float(P.q[L - 1]), L)
        return cache[(b, p, u, q)]
    ev = K.Ev(P, okeys, m)
    y0 = K.projection_finalize(ev, oplan, K.projection_partial(ev, oplan, xs, w, 0, oplan.N2)[0])
    wd = plan.encode_weights(W, L)
    n0 = oplan.N2 * oplan.U * oplan.N1
    pts = [w(0, p, u, q) for p in range(oplan.N2) for u in range(oplan.U) for q in range(oplan.N1)]
    blk = torch.from_numpy(np.ascontiguousarray(np.stack([pt.m for pt in pts])).view(np.int64).reshape(-1).copy()).to(ctx.device)
    ctx.poly_to_ntt(blk, n0, L)
    wd[:blk.numel()] = blk
    ys = plan.matmul(gkeys, [dev_ct(ctx, x) for x in xs], wd, float(P.q[L - 1]))
    assert_ct_equal(ctx, ys[0], y0, "GPT-2 FF2 y_0 (N=2^16, m=256, L=3)")
    Y = X @ W
    for b, y in enumerate(ys):
        got = K.seg_column_unpack(_dec(okeys, O.Ct(ctx.to_host(y), y.scale)).real, m, 128, dout, b)
        ref = Y[:, b * 128:(b + 1) * 128]
        assert np.abs(got - ref).max() / np.abs(Y).max() < TOL, b
