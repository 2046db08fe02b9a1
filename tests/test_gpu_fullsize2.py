"""Full-size (N = 2^16, P16) parity for the cases round 1 left decrypt-checked only:
  * the minimal export stream's STRADDLING pieces: with H m = 1536 slots per S_t and n = 32768, S_21 and S_42 are
    split across two output ciphertexts (masks over two slot ranges); every output ciphertext is compared on every
    limb with the oracle's score_export on the same (random) S_t ciphertexts;
  * conj and relinearisation at the top level L = 24 (dnum = 3, the config-2 key-switch shapes);
  * one BERT-large value block (H = 16, B_V = 4: the last block, heads 12..15)."""
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
M, DH = 128, 64
TOL = 2.0 ** -20


@pytest.fixture(scope="module")
def ctx():
    return E.Context("P16", 0)


def _rand_ct(L, seed, scale):
    g = np.random.default_rng(seed)
    return O.Ct(np.stack([np.stack([g.integers(0, q, P.N, dtype=np.uint64) for q in P.q[:L]]) for _ in range(2)]), scale)


def test_export_stream_straddling_pieces_bit_exact(ctx):
    """BERT-base score export (H = 12, m = 128, K_min(S) = 3): all 64 S_t (random ciphertexts at L = 4) packed into
    the stream; the pieces of S_21 (slots 32256..33792) and S_42 (64512..66048) straddle ciphertexts 0|1 and 1|2."""
    H, L = 12, 4
    plan = E.AttnPlan(ctx, M, H, DH, C_qk=192, beta=16)
    oplan = K.ScorePlan(P.n, M, H, DH, C_qk=192, beta=16)
    assert oplan.n_out == plan.n_out == 3
    seg = H * M
    straddle = [t for t in range(M // 2) if (t * seg) // P.n != (t * seg + seg - 1) // P.n]
    assert straddle == [21, 42]
    offs = sorted({(t * seg) % P.n for t in range(M // 2) if (t * seg) % P.n})
    og = sorted({O.galois_rot(P, -o) for o in offs})
    okeys = O.Keys(P, synth.SEED_KEYS, galois=og, max_level=L)
    gkeys = ctx.keygen(synth.SEED_KEYS, galois=og, max_level=L)
    scale = 2.0 ** 40
    S = [_rand_ct(L, 1000 + t, scale) for t in range(M // 2)]
    ev = K.Ev(P, okeys, M)
    ref = K.score_export(ev, oplan, S)
    ctx.mask_clear()
    install_masks(ctx, ev)
    got = plan.export_stream(gkeys, [dev_ct(ctx, s) for s in S])
    for i, (a, b) in enumerate(zip(got, ref)):
        assert_ct_equal(ctx, a, b, "export stream ciphertext %d (N=2^16)" % i)
    ctx.mask_clear()


def test_conj_and_relin_top_level_bit_exact(ctx):
    """L = 24, dnum = 3 (config 2): conjugation and relinearisation (and the rescale after it) bit-exact."""
    L = 24
    g = [O.galois_conj(P)]
    okeys = O.Keys(P, synth.SEED_KEYS, galois=g, relin=True)
    gkeys = ctx.keygen(synth.SEED_KEYS, galois=g, relin=True)
    a = O.encrypt_sk(P, okeys, O.encode(P, synth.complex_slots(P.n, 61), 2.0 ** 40, L), 1)
    b = O.encrypt_sk(P, okeys, O.encode(P, synth.complex_slots(P.n, 62), 2.0 ** 40, L), 2)
    da, db = dev_ct(ctx, a), dev_ct(ctx, b)
    assert_ct_equal(ctx, ctx.conjugate(gkeys, da), O.conjugate(P, okeys, a), "conj L=24")
    t = O.tensor(P, a, b)
    r = O.relinearize(P, okeys, t)
    gr = ctx.relinearize(gkeys, ctx.tensor(da, db))
    assert_ct_equal(ctx, gr, r, "relin L=24")
    assert_ct_equal(ctx, ctx.rescale(gr), O.rescale(P, r), "rescale after relin L=24")


def test_value_bert_large_last_block_bit_exact(ctx):
    """BERT-large value kernel (NEXT row 4): H = 16, H_blk = 4, B_V = 4; block 3 (heads 12..15) bit-exact, every
    block within 2^-20 of P V."""
    H = 16
    plan = E.AttnPlan(ctx, M, H, DH)
    oplan = K.ValuePlan(P.n, M, H, DH)
    assert (plan.H_blk, plan.B_V) == (oplan.H_blk, oplan.B_V) == (4, 4)
    Ph = synth.attention_probs(H, M, synth.seed_data(4) + 11)
    Vh = synth.uniform((H, M, DH), synth.seed_data(4) + 12)
    half = M // 2
    steps = {half, half - M} | {t for t in range(1, half)} | {t - M for t in range(1, half)}
    steps |= {d * M for d in range(-(DH - 1), half) if d}
    og = sorted({O.galois_rot(P, r) for r in steps if r % P.n})
    okeys = O.Keys(P, synth.SEED_KEYS, galois=og, relin=True, max_level=7)
    gkeys = ctx.keygen(synth.SEED_KEYS, galois=plan.galois(), relin=True, max_level=7)
    vs = [O.encrypt_sk(P, okeys, O.encode(P, K.value_v_slots(Vh, oplan, l), 2.0 ** 40, 7), 700 + l) for l in range(oplan.B_V)]
    ps = [O.encrypt_sk(P, okeys, O.encode(P, K.value_p_slots(Ph, oplan, l), 2.0 ** 47, 5), 800 + l) for l in range(oplan.B_V)]
    ev = K.Ev(P, okeys, M)
    o3 = K.value(ev, oplan, ps, vs, blocks=[3])[0]
    ctx.mask_clear()
    install_masks(ctx, ev)
    outs = plan.value(gkeys, [dev_ct(ctx, x) for x in ps], [dev_ct(ctx, x) for x in vs])
    assert_ct_equal(ctx, outs[3], o3, "BERT-large value o_3 (N=2^16)")
    ref = K.value_reference(Ph, Vh)
    for l, o in enumerate(outs):
        got = O.decode(P, O.decrypt(P, okeys, O.Ct(ctx.to_host(o), o.scale))).real
        for hh in range(oplan.H_blk):
            h = l * oplan.H_blk + hh
            for u in range(0, DH, 13):
                s = hh * oplan.seg_stride + u
                assert np.abs(got[s * M:(s + 1) * M] - ref[h][:, u]).max() / np.abs(ref).max() < TOL, (l, h, u)
    ctx.mask_clear()
