"""T1/T2/T3 on the B200: every limb of every output of the CUDA path (through the C ABI) equals the
oracle's, on seeded inputs; plus decryption tolerances and error codes."""
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
from tests.gpu_util import assert_ct_equal, dev_ct, dev_pt, install_masks, weights_tensor  # noqa: E402

P12, P13, P16 = O.Params("P12"), O.Params("P13"), O.Params("P16")
TOL = 2.0 ** -20


def rnd(mods, N, seed):
    g = np.random.default_rng(seed)
    return np.stack([g.integers(0, q, N, dtype=np.uint64) for q in mods])


@pytest.fixture(scope="module")
def c13():
    return E.Context("P13", 0)


@pytest.fixture(scope="module")
def c16():
    return E.Context("P16", 0)


def galois13():
    from tests.test_oracle_kernels import _galois13
    return _galois13()


@pytest.fixture(scope="module")
def keys13(c13):
    g = galois13()
    return O.Keys(P13, synth.SEED_KEYS, galois=g, relin=True), c13.keygen(synth.SEED_KEYS, galois=g, relin=True)


# ------------------------------------------------------------------ NTT / ring product
@pytest.mark.parametrize("pname", ["P12", "P13", "P16"])
def test_ntt_roundtrip_and_ring_product(pname):
    P = O.Params(pname)
    ctx = E.Context(pname, 0)
    L = min(P.L_max, 6)
    mods = P.q[:L]
    a, b = rnd(mods, P.N, 1), rnd(mods, P.N, 2)
    A = ctx.pt_from_host(a, 1.0)
    assert np.array_equal(ctx.to_host(ctx.from_ntt(ctx.to_ntt(A))), a)
    x = ctx.to_ntt(ctx.ct_from_host(np.stack([a, a]), 1.0))
    y = ctx.ptmul(x, ctx.to_ntt(ctx.pt_from_host(b, 1.0)))
    ref = O.ring_mul(a, b, mods, P.N)
    got = ctx.to_host(y)
    assert np.array_equal(got[0], ref) and np.array_equal(got[1], ref)


@pytest.mark.parametrize("fill", ["max", "mixed"])
def test_ntt_lazy_bounds_extreme_inputs(fill):
    """Worst-case words for the lazy butterfly ranges ([0, 8q) forward, [0, 4q) inverse, approximate-high
    Shoup products): all-(q-1) limbs and alternating 0 / q-1, on the 60-bit q_0 (integer path) and the 40-bit
    limbs, through the ring product against the oracle's schoolbook-pinned ring_mul."""
    P = P16
    ctx = E.Context("P16", 0)
    mods = P.q[:4]
    if fill == "max":
        a = np.stack([np.full(P.N, q - 1, dtype=np.uint64) for q in mods])
    else:
        a = np.stack([np.where(np.arange(P.N) % 2 == 0, 0, q - 1).astype(np.uint64) for q in mods])
    b = a.copy()
    b[:, ::3] = 1
    A = ctx.pt_from_host(a, 1.0)
    assert np.array_equal(ctx.to_host(ctx.from_ntt(ctx.to_ntt(A))), a)
    x = ctx.to_ntt(ctx.ct_from_host(np.stack([a, a]), 1.0))
    y = ctx.ptmul(x, ctx.to_ntt(ctx.pt_from_host(b, 1.0)))
    ref = O.ring_mul(a, b, mods, P.N)
    got = ctx.to_host(y)
    assert np.array_equal(got[0], ref) and np.array_equal(got[1], ref)


# ------------------------------------------------------------------ keys / enc / dec
def test_keys_bit_exact(c13, keys13):
    ok, gk = keys13
    ML = ok.max_level
    nl = ML + len(P13.p)
    sk = gk.export(0).reshape(nl, P13.N)
    assert np.array_equal(sk, ok.s)
    for g in [galois13()[0], 0]:
        kk = gk.export(1, g).reshape(P13.dnum(ML), 2, nl, P13.N)
        for j in range(P13.dnum(ML)):
            assert np.array_equal(kk[j], ok.ksk[g][j]), (g, j)


def test_encrypt_decrypt_bit_exact(c13, keys13):
    ok, gk = keys13
    z = synth.complex_slots(P13.n, 3)
    pt = O.encode(P13, z, 2.0 ** 40, 6)
    ref = O.encrypt_sk(P13, ok, pt, 77)
    got = c13.encrypt(gk, c13.pt_from_host(pt.m, pt.scale), 77)
    assert_ct_equal(c13, got, ref, "encrypt")
    d = c13.decrypt(gk, got)
    assert np.array_equal(c13.to_host(d), O.decrypt(P13, ok, ref).m)


def test_encode_decode_gpu_vs_oracle(c13):
    z = synth.complex_slots(P13.n, 4)
    ref = O.encode_coeffs(z, 2.0 ** 40, P13.N)
    pt = c13.encode(z, 2.0 ** 40, 3)
    got = c13.to_host(pt)
    refq = O.from_signed(ref, P13.q[:3], P13.N)
    diff = np.minimum((got.astype(object) - refq.astype(object)) % np.array(P13.q[:3], dtype=object)[:, None],
                      (refq.astype(object) - got.astype(object)) % np.array(P13.q[:3], dtype=object)[:, None])
    assert int(diff.max()) <= 1             # float64 encode: +-1 per coefficient
    zz = c13.decode(pt)
    assert np.abs(zz - z).max() < 1e-9


# ------------------------------------------------------------------ key switching & friends
@pytest.mark.parametrize("L", [8, 5, 3, 1])
def test_rotations_conj_bit_exact(c13, keys13, L):
    ok, gk = keys13
    z = synth.complex_slots(P13.n, 10 + L)
    ct = O.encrypt_sk(P13, ok, O.encode(P13, z, 2.0 ** 40, L), 5)
    d = dev_ct(c13, ct)
    for r in (1, 16, -3):
        assert_ct_equal(c13, c13.rotate(gk, d, r), O.rotate(P13, ok, ct, r), "rotate %d L=%d" % (r, L))
    steps = [1, 16, 32, -3, 0]
    hs = c13.rotate_hoisted(gk, d, steps)
    for r, h, ref in zip(steps, hs, O.rotate_hoisted(P13, ok, ct, steps)):
        assert_ct_equal(c13, h, ref, "hoisted %d L=%d" % (r, L))
    assert_ct_equal(c13, c13.conjugate(gk, d), O.conjugate(P13, ok, ct), "conj")


def test_decomplexify_batched_bit_exact(c13, keys13):
    """encf_decomplexify (G3): c + conj(c) for a batch of ciphertexts in one conjugation launch
    sequence equals the oracle's add(c, conjugate(c)) on every limb; the scale doubles."""
    ok, gk = keys13
    L = 4
    cts = [O.encrypt_sk(P13, ok, O.encode(P13, synth.complex_slots(P13.n, 40 + i), 2.0 ** 40, L), 60 + i)
           for i in range(3)]
    outs = c13.decomplexify(gk, [dev_ct(c13, ct) for ct in cts])
    for i, (ct, got) in enumerate(zip(cts, outs)):
        ref = O.Ct(O.add(P13, ct, O.conjugate(P13, ok, ct)).c, 2.0 * ct.scale)   # scale x 2 (G3)
        assert_ct_equal(c13, got, ref, "decomplexify %d" % i)


def test_tensor_relin_rescale_bit_exact(c13, keys13):
    ok, gk = keys13
    a = O.encrypt_sk(P13, ok, O.encode(P13, synth.complex_slots(P13.n, 20), 2.0 ** 40, 7), 1)
    b = O.encrypt_sk(P13, ok, O.encode(P13, synth.complex_slots(P13.n, 21), 2.0 ** 40, 7), 2)
    da, db = dev_ct(c13, a), dev_ct(c13, b)
    t = c13.tensor(da, db)
    tr = O.tensor(P13, a, b)
    assert_ct_equal(c13, t, tr, "tensor")
    r = c13.relinearize(gk, t)
    rr = O.relinearize(P13, ok, tr)
    assert_ct_equal(c13, r, rr, "relin")
    assert_ct_equal(c13, c13.rescale(r), O.rescale(P13, rr), "rescale")
    assert_ct_equal(c13, c13.mod_drop(da, 4), O.mod_drop(P13, a, 4), "mod_drop")
    assert_ct_equal(c13, c13.mul_i(da), O.mul_i(P13, a), "mul_i")
    assert_ct_equal(c13, c13.add(da, db), O.add(P13, a, b), "add")
    assert_ct_equal(c13, c13.add(da, db, sub=True), O.sub(P13, a, b), "sub")
    assert_ct_equal(c13, c13.complexify(da, db), O.complexify(P13, a, b), "complexify")
    many = c13.complexify_many([da, db, da], [db, da, da])      # batched (encf_complexify_many)
    for got, (x, y) in zip(many, [(a, b), (b, a), (a, a)]):
        assert_ct_equal(c13, got, O.complexify(P13, x, y), "complexify_many")


def test_keyswitch_P16_top_level(c16):
    """Config 2 shape (L = 24, dnum = 3, alpha = 8): single and hoisted rotations bit-exact."""
    L = 24
    g = [O.galois_rot(P16, r) for r in (128, 256)]
    ok = O.Keys(P16, synth.SEED_KEYS, galois=g)
    gk = c16.keygen(synth.SEED_KEYS, galois=g)
    ct = O.encrypt_sk(P16, ok, O.encode(P16, synth.uniform(P16.n, 60), 2.0 ** 40, L), 9)
    d = dev_ct(c16, ct)
    assert_ct_equal(c16, c16.rotate(gk, d, 128), O.rotate(P16, ok, ct, 128), "rotate P16 L=24")
    for h, ref in zip(c16.rotate_hoisted(gk, d, [128, 256]), O.rotate_hoisted(P16, ok, ct, [128, 256])):
        assert_ct_equal(c16, h, ref, "hoisted P16 L=24")


def test_error_codes(c13, keys13):
    ok, gk = keys13
    a = O.encrypt_sk(P13, ok, O.encode(P13, synth.complex_slots(P13.n, 30), 2.0 ** 40, 2), 1)
    b = O.encrypt_sk(P13, ok, O.encode(P13, synth.complex_slots(P13.n, 31), 2.0 ** 39, 2), 2)
    with pytest.raises(E.EncfError) as e:
        c13.add(dev_ct(c13, a), dev_ct(c13, b))
    assert e.value.code == 3
    one = dev_ct(c13, O.mod_drop(P13, a, 1))
    with pytest.raises(E.EncfError) as e:
        c13.rescale(one)
    assert e.value.code == 5
    with pytest.raises(E.EncfError) as e:
        c13.rotate(gk, dev_ct(c13, a), 12345)
    assert e.value.code == 11
    with pytest.raises(E.EncfError) as e:
        E.AttnPlan(c13, 15, 4, 8)
    assert e.value.code == 7


# ------------------------------------------------------------------ EncFormer kernels
def _proj_case(P, ctx, okeys, gkeys, m, d_in, d_out, N1, L, seed):
    plan = E.ProjPlan(ctx, m, d_in, d_out, N1=N1)
    oplan = K.ProjPlan(P.n, m, d_in, d_out, N1=N1)
    X = synth.fixed_point_uniform((m, d_in), seed)
    W = synth.bert_weight((d_in, d_out), seed + 1)
    xs = [O.encrypt_sk(P, okeys, O.encode(P, z, 2.0 ** 40, L), synth.seed_enc(u)) for u, z in enumerate(K.proj_inputs(X, oplan))]
    pts = {}

    def w(b, p, u, q):
        if (b, p, u, q) not in pts:
            pts[(b, p, u, q)] = O.encode(P, K.proj_weight_slots(W, oplan, b, p, u, q), float(P.q[L - 1]), L)
        return pts[(b, p, u, q)]
    ys = K.projection(K.Ev(P, okeys, m), oplan, xs, w)
    order = [w(b, p, u, q) for b in range(oplan.B_out) for p in range(oplan.N2) for u in range(oplan.U) for q in range(oplan.N1)]
    wd = weights_tensor(ctx, order, L)
    got = plan.matmul(gkeys, [dev_ct(ctx, x) for x in xs], wd, float(P.q[L - 1]))
    for b, (g, r) in enumerate(zip(got, ys)):
        assert_ct_equal(ctx, g, r, "projection y_%d" % b)
    Y = np.concatenate([K.seg_column_unpack(O.decode(P, O.decrypt(P, okeys, y)).real, m, oplan.C, d_out, b) for b, y in enumerate(ys)], axis=1)
    assert np.abs(Y - X @ W).max() / np.abs(X @ W).max() < TOL
    return plan, oplan, xs, wd, ys


def test_projection_config1_bit_exact():
    ctx = E.Context("P12", 0)
    plan = E.ProjPlan(ctx, 32, 64, 64, N1=8)
    g = plan.galois()
    ok, gk = O.Keys(P12, synth.SEED_KEYS, galois=g), ctx.keygen(synth.SEED_KEYS, galois=g)
    _proj_case(P12, ctx, ok, gk, 32, 64, 64, 8, 3, synth.seed_data(1))


def test_projection_ragged_and_unit_split(c13, keys13):
    """U = 2, G odd, ragged d_out; then the same projection split into two unit ranges (the
    multi-GPU partition), partial accumulators summed as uint64 and mod-reduced (C2), then finalised."""
    ok, gk = keys13
    plan, oplan, xs, wd, ys = _proj_case(P13, c13, ok, gk, 16, 600, 300, 8, 4, 70)
    units = plan.B_out * plan.N2
    cut = units // 2 + 3
    xd = [dev_ct(c13, x) for x in xs]
    a = plan.matmul(gk, xd, wd, float(P13.q[3]), 0, cut, finalize=False)
    b = plan.matmul(gk, xd, wd, float(P13.q[3]), cut, units, finalize=False)
    # block containing `cut` is split across the two "ranks": add as uint64 then mod-reduce
    bsplit = cut // plan.N2
    accs = a[:bsplit] + [None] + b[1:]
    s = a[bsplit].data + b[0].data    # int64 storage; q < 2^61 so the sum is exact (extended-basis partials)
    assert a[bsplit].n_limbs == 4 + len(P13.p)
    c13.mod_reduce_ext(s, 2, 4)
    a[bsplit].data = s
    accs[bsplit] = a[bsplit]
    yfin = plan.finalize(gk, accs, 0)
    for bb, (g, r) in enumerate(zip(yfin, ys)):
        assert_ct_equal(c13, g, r, "split projection y_%d" % bb)


def test_score_and_export_bit_exact(c13, keys13):
    ok, gk = keys13
    m, H, dh = 16, 4, 8
    plan = E.AttnPlan(c13, m, H, dh, C_qk=16, beta=4)
    oplan = K.ScorePlan(P13.n, m, H, dh, C_qk=16, beta=4)
    g = synth.rng(40)
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
        assert_ct_equal(c13, a, b, "S_%d" % t)
    gE = plan.export_stream(gk, gS)
    for a, b in zip(gE, Ex):
        assert_ct_equal(c13, a, b, "export stream")
    # t-range split (multi-GPU partition of the score kernel) gives the same S_t
    part = plan.score(gk, [dev_ct(c13, x) for x in qs], [dev_ct(c13, x) for x in ks], 3, 6)
    for t, a in zip(range(3, 6), part):
        assert_ct_equal(c13, a, S[t], "S_%d (range)" % t)
    c13.mask_clear()


def test_value_bit_exact(c13, keys13):
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
    c13.mask_clear()
    install_masks(c13, ev)
    got = plan.value(gk, [dev_ct(c13, x) for x in ps], [dev_ct(c13, x) for x in vs])
    for a, b in zip(got, outs):
        assert_ct_equal(c13, a, b, "value")
    c13.mask_clear()


def test_export_c2m_bit_exact(c13, keys13):
    ok, gk = keys13
    x, y = synth.fixed_point_uniform(P13.n, 50), synth.fixed_point_uniform(P13.n, 51)
    cx = O.encrypt_sk(P13, ok, O.encode(P13, x, 2.0 ** 40, 5), 1)
    cy = O.encrypt_sk(P13, ok, O.encode(P13, y, 2.0 ** 40, 5), 2)
    ref = O.complexify(P13, cx, cy)
    got = c13.complexify(dev_ct(c13, cx), dev_ct(c13, cy))
    assert_ct_equal(c13, got, ref, "complexify")
    Lc = c13.l_conv()
    assert Lc == K.l_conv(P13)
    masked, share = c13.export_c2m(got, Lc, synth.seed_mask(0), 0)
    rm, rs = K.export_c2m(P13, ref, Lc, synth.seed_mask(0), 0)
    assert np.array_equal(c13.to_host(masked, coeff=False), rm.c)
    assert np.array_equal(share.cpu().numpy().view(np.uint64).reshape(Lc, P13.N), rs)


def test_export_c2m_many_bit_exact(c13, keys13):
    """Batched export (encf_export_c2m_many): ciphertext i with stream id 7 + i equals the oracle's export of it."""
    ok, gk = keys13
    cts = [O.encrypt_sk(P13, ok, O.encode(P13, synth.fixed_point_uniform(P13.n, 70 + i), 2.0 ** 40, 4), 80 + i)
           for i in range(3)]
    Lc = c13.l_conv()
    outs = c13.export_c2m_many([dev_ct(c13, ct) for ct in cts], Lc, synth.seed_mask(1), 7)
    for i, (ct, (masked, share)) in enumerate(zip(cts, outs)):
        rm, rs = K.export_c2m(P13, ct, Lc, synth.seed_mask(1), 7 + i)
        assert np.array_equal(c13.to_host(masked, coeff=False), rm.c), i
        assert np.array_equal(share.cpu().numpy().view(np.uint64).reshape(Lc, P13.N), rs), i


def test_m2c_import_bit_exact(c13, keys13):
    """Alg 4 GPU half: Ring2Field local maps and <c> + [[t^]]_1 equal the oracle's on every limb."""
    ok, gk = keys13
    P, L, ell, sig = P13, 5, 43, 40
    rng = np.random.default_rng(70)
    t = O.encode_coeffs(synth.complex_slots(P.n, 71), 2.0 ** 40, P.N)
    from tests.test_oracle_kernels import _simulate_ext
    ext = [_simulate_ext(v, ell + sig, rng) for v in t]
    dev = {}
    for b in (0, 1):
        words = np.array([[e[b] & (2 ** 64 - 1), e[b] >> 64] for e in ext], dtype=np.uint64)
        dev[b] = torch.from_numpy(words.view(np.int64).reshape(-1).copy()).to(c13.device)
    s0 = c13.ring2field_local(dev[0], 0, ell + sig, L)
    s1 = c13.ring2field_local(dev[1], 1, ell + sig, L)
    r0 = K.ring2field_local(P, [e[0] for e in ext], 0, ell + sig, L)
    r1 = K.ring2field_local(P, [e[1] for e in ext], 1, ell + sig, L)
    assert np.array_equal(c13.to_host(s0), r0) and np.array_equal(c13.to_host(s1), r1)
    c = O.encrypt_sk(P, ok, O.Pt(r0, 2.0 ** 40), 5)
    got = c13.import_m2c(dev_ct(c13, c), s1)
    assert_ct_equal(c13, got, K.import_m2c(P, c, O.Pt(r1, 2.0 ** 40)), "import_m2c")
    lift = torch.from_numpy(np.array([[v, 0] for v in rng.integers(0, 2 ** 62, P.N)], dtype=np.uint64).view(np.int64).reshape(-1).copy()).to(c13.device)
    f = c13.field2ring_local(lift, ell).cpu().numpy().view(np.uint64)
    assert np.array_equal(f, K.field2ring_local(lift.cpu().numpy().view(np.uint64).reshape(-1, 2)[:, 0], ell))


def test_fused_qk_projection_bit_exact(c13, keys13):
    """Fused-QK plan (real inputs, complex weights): GPU encoder == oracle encoding, output bit-exact."""
    ok, gk = keys13
    P, m, d, L = P13, 16, 300, 4
    plan = E.ProjPlan(c13, m, d, 256, N1=8, real_input=True)
    oplan = K.ProjPlan(P.n, m, d, 256, N1=8, real_input=True)
    assert (plan.U, plan.B_out, plan.N1, plan.N2) == (oplan.U, oplan.B_out, oplan.N1, oplan.N2)
    X = synth.fixed_point_uniform((m, d), 90)
    WQ, WK = synth.bert_weight((d, 256), 91), synth.bert_weight((d, 256), 92)
    xs = [O.encrypt_sk(P, ok, O.encode(P, z, 2.0 ** 40, L), 20 + g) for g, z in enumerate(K.proj_inputs(X, oplan))]
    pts = {}

    def w(b, p, g, q):
        if (b, p, g, q) not in pts:
            pts[(b, p, g, q)] = O.encode(P, K.proj_weight_slots_fused(WQ, WK, oplan, b, p, g, q), float(P.q[L - 1]), L)
        return pts[(b, p, g, q)]
    ref = K.projection(K.Ev(P, ok, m), oplan, xs, w, decomplexify=False)
    order = [w(b, p, g, q) for b in range(oplan.B_out) for p in range(oplan.N2) for g in range(oplan.U) for q in range(oplan.N1)]
    wd = weights_tensor(c13, order, L)
    wg = plan.encode_weights_complex(WQ, WK, L)
    assert torch.equal(wg, wd)                        # GPU complex-weight encoder == oracle encoding, word for word
    got = plan.matmul(gk, [dev_ct(c13, x) for x in xs], wd, float(P.q[L - 1]))
    for a, r in zip(got, ref):
        assert_ct_equal(c13, a, r, "fused QK")


# ------------------------------------------------------------------ NTT: FP64-pipe path == integer path
def test_ntt_fp64_path_equals_integer_path(monkeypatch):
    """The 40-bit limbs of P16 run the NTT on the FP64 pipe (ntt.cu FpOps); the 60-bit ones on the integer
    Shoup path.  Forcing the integer path everywhere (ENCF_NTT_INT_ONLY) must give the same words, for
    random limbs, all-(q-1) and all-zero limbs, forward and inverse."""
    P = P16
    L = P.L_max
    mods = list(P.q) + list(P.p)
    a = rnd(mods, P.N, 5)
    a[1, :] = mods[1] - 1
    a[2, :] = 0
    ctx_fp = E.Context("P16", 0)
    monkeypatch.setenv("ENCF_NTT_INT_ONLY", "1")
    ctx_int = E.Context("P16", 0)
    monkeypatch.delenv("ENCF_NTT_INT_ONLY")
    nl = L  # ciphertext-basis limbs (q_0..q_23): 23 of them on the FP64 path
    x = a[:nl]
    outs = []
    for ctx in (ctx_fp, ctx_int):
        t = ctx.pt_from_host(x, 1.0)
        ctx.to_ntt(t)
        f = t.data.cpu().numpy().view(np.uint64).reshape(nl, P.N).copy()
        ctx.from_ntt(t)
        b = ctx.to_host(t, coeff=False)
        outs.append((f, b))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], x) and np.array_equal(outs[1][1], x)
    # inverse of NTT-domain words (canonical) on both paths
    for ctx in (ctx_fp, ctx_int):
        t = ctx.pt_from_host(x, 1.0, ntt=1)
        ctx.from_ntt(t)
        outs.append(ctx.to_host(t, coeff=False))
    assert np.array_equal(outs[2], outs[3])


# ------------------------------------------------------------------ GELU pre-evaluation (Alg 5 steps 1-3)
def test_gelu_preeval_bit_exact(c13, keys13):
    """encf_gelu_preeval on two complex inputs at L = 5 (N = 2^13): both candidate ciphertexts F0^C, F1^C
    equal the oracle's on every limb, and decrypt to Eq. B.2 of the real and imaginary channels."""
    ok, gk = keys13
    coef = K.gelu_fit()
    g = synth.rng(91)
    xs_h, refs = [], []
    for i in range(2):
        x0, x1 = g.uniform(-2.7, 2.7, P13.n), g.uniform(-2.7, 2.7, P13.n)
        x = O.encrypt_sk(P13, ok, O.encode(P13, x0 + 1j * x1, 2.0 ** 40, 5), 500 + i)
        xs_h.append((x, x0, x1))
        refs.append(K.gelu_preeval(K.Ev(P13, ok, 16), x, coef))
    f0, f1 = c13.gelu_preeval(gk, [dev_ct(c13, x) for x, _, _ in xs_h], coef)
    a, b, c, d, e = coef
    for i, ((x, x0, x1), (r0, r1)) in enumerate(zip(xs_h, refs)):
        assert_ct_equal(c13, f0[i], r0, "F0^C[%d]" % i)
        assert_ct_equal(c13, f1[i], r1, "F1^C[%d]" % i)
        z = O.decode(P13, O.decrypt(P13, ok, O.Ct(c13.to_host(f1[i]), f1[i].scale)))
        F1 = lambda v: a * v ** 4 + b * v ** 3 + c * v ** 2 + (0.5 + d) * v + e
        assert np.abs(z - (F1(x0) + 1j * F1(x1))).max() < 1e-5


# ------------------------------------------------------------------ w/o-SCP ablation: RMA repack
def test_repack_rma_bit_exact(c13, keys13):
    """encf_repack_rma (App. G) on two ciphertexts at L = 5, m = 16: every limb equals the oracle's."""
    ok, gk = keys13
    g = synth.rng(56)
    xs, refs = [], []
    for i in range(2):
        v = g.uniform(-1, 1, P13.n) + 1j * g.uniform(-1, 1, P13.n)
        x = O.encrypt_sk(P13, ok, O.encode(P13, v, 2.0 ** 40, 5), 600 + i)
        xs.append(x)
        ev = K.Ev(P13, ok, 16)
        refs.append(K.repack_rma(ev, x, 16))
    c13.mask_clear()
    install_masks(c13, ev)
    got = c13.repack_rma(gk, [dev_ct(c13, x) for x in xs], 16)
    for a, b in zip(got, refs):
        assert_ct_equal(c13, a, b, "RMA repack")
    c13.mask_clear()
