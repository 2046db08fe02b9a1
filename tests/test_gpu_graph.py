"""CUDA-graph execution of the hot path (paper_2604_09975_b200.graphs.GraphedStep, the bench's timed
path): a captured step replays to the SAME words as the eager calls, and a replay on new inputs equals
the oracle on those inputs (every limb)."""
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
from paper_2604_09975_b200.graphs import GraphedStep, PipelinedStep  # noqa: E402
from tests.gpu_util import assert_ct_equal, dev_ct, weights_tensor  # noqa: E402

P13 = O.Params("P13")


def test_graph_replay_projection_attention_export():
    ctx = E.Context("P13", 0)
    m, H, dh, d_in, d_out, L = 16, 4, 8, 64, 96, 6
    proj = E.ProjPlan(ctx, m, d_in, d_out, N1=8)
    attn = E.AttnPlan(ctx, m, H, dh, C_qk=16, beta=4)
    galois = sorted(set(proj.galois()) | set(attn.galois()) | {ctx.galois_conj()})
    ok = O.Keys(P13, synth.SEED_KEYS, galois=galois, relin=True)
    gk = ctx.keygen(synth.SEED_KEYS, galois=galois, relin=True)
    oplan = K.ProjPlan(P13.n, m, d_in, d_out, N1=8)
    W = synth.bert_weight((d_in, d_out), 91)
    pts = [O.encode(P13, K.proj_weight_slots(W, oplan, b, p, u, q), float(P13.q[L - 1]), L)
           for b in range(oplan.B_out) for p in range(oplan.N2) for u in range(oplan.U) for q in range(oplan.N1)]
    wd = weights_tensor(ctx, pts, L)

    def inputs(seed):
        X = synth.fixed_point_uniform((m, d_in), seed)
        xs = [O.encrypt_sk(P13, ok, O.encode(P13, z, 2.0 ** 40, L), synth.seed_enc(u) + seed)
              for u, z in enumerate(K.proj_inputs(X, oplan))]
        g = synth.rng(seed + 1)
        qk = [O.encrypt_sk(P13, ok, O.encode(P13, g.uniform(-1, 1, P13.n), 2.0 ** 40, L), 500 + seed + i) for i in range(4)]
        return xs, qk

    def step(inp):
        y = proj.matmul(gk, inp["x"], wd, float(P13.q[L - 1]))
        S = attn.score(gk, inp["q"], inp["k"])
        ex = [ctx.export_c2m(c, 2, 7, i) for i, c in enumerate(attn.export_stream(gk, S))]
        return [(c.data, None) for c in y] + [(a.data, b) for a, b in ex]

    xs0, qk0 = inputs(10)
    d0 = {"x": [dev_ct(ctx, x) for x in xs0], "q": [dev_ct(ctx, c) for c in qk0[:2]], "k": [dev_ct(ctx, c) for c in qk0[2:]]}
    eager0 = [(a.clone(), b.clone() if b is not None else None) for a, b in step(d0)]     # warm-up (mask cache)
    g = GraphedStep(step, d0)
    out = g()
    torch.cuda.synchronize()
    for (a, b), (ea, eb) in zip(out, eager0):
        assert torch.equal(a, ea)
        assert (b is None) or torch.equal(b, eb)
    # new inputs through the static buffers: the replay equals the oracle's projection on them
    xs1, qk1 = inputs(20)
    host = {"x": [dev_ct(ctx, x).data.cpu().pin_memory() for x in xs1],
            "q": [dev_ct(ctx, c).data.cpu().pin_memory() for c in qk1[:2]],
            "k": [dev_ct(ctx, c).data.cpu().pin_memory() for c in qk1[2:]]}
    out1 = g(host)
    torch.cuda.synchronize()
    ys = K.projection(K.Ev(P13, ok, m), oplan, xs1, lambda b, p, u, q: pts[((b * oplan.N2 + p) * oplan.U + u) * oplan.N1 + q])
    for b, y in enumerate(ys):
        got = E.Ciphertext(out1[b][0], 2, L - 1, y.scale, 1)
        assert_ct_equal(ctx, got, y, "graph-replayed projection y_%d" % b)
    # and the eager path on the same new inputs gives the same export words
    d1 = {k: [E.Ciphertext(h.to(ctx.device), 2, L, 2.0 ** 40, 1) for h in v] for k, v in host.items()}
    eager1 = step(d1)
    for (a, b), (ea, eb) in zip(out1, eager1):
        assert torch.equal(a, ea)
        assert (b is None) or torch.equal(b, eb)
    # the pipelined e2e path (bench.py): two graphs on two input sets, copies on side streams; after 4 steps both
    # sets' host copies hold exactly the eager words
    db = {k: [E.Ciphertext(c.data.clone(), c.n_comp, c.n_limbs, c.scale, c.ntt) for c in v] for k, v in d0.items()}
    pipe = PipelinedStep(step, g, db)
    pin = [[(torch.empty(a.shape, dtype=a.dtype, pin_memory=True),
             torch.empty(b.shape, dtype=b.dtype, pin_memory=True) if b is not None else None) for a, b in gg.outputs]
           for gg in pipe.g]
    pipe.run(host, pin, 4)
    torch.cuda.synchronize()
    for hs in pin:
        for (a, b), (ea, eb) in zip(hs, eager1):
            assert torch.equal(a, ea.cpu())
            assert (b is None) or torch.equal(b, eb.cpu())


def test_graph_replays_draw_fresh_export_masks():
    """a captured export must not reuse its one-time pad r^ across replays.  With the (seed, stream id
    base) in a device buffer advanced inside the graph (encf_export_c2m_many_dev), replay k draws the masks of stream
    ids k 2^32 + i: every replay's masked ciphertext and server share equal the oracle's export_c2m with that
    stream id, and two replays differ."""
    ctx = E.Context("P13", 0)
    ok = O.Keys(P13, synth.SEED_KEYS)
    cts = [O.encrypt_sk(P13, ok, O.encode(P13, synth.fixed_point_uniform(P13.n, 30 + i), 2.0 ** 40, 4), 40 + i)
           for i in range(2)]
    d = {"x": [dev_ct(ctx, c) for c in cts]}
    seed = synth.seed_mask(3)
    state = torch.tensor([seed, 0], dtype=torch.int64, device=ctx.device)

    def step(inp):
        ex = ctx.export_c2m_many(inp["x"], 2, state, 0)
        state[1:].add_(1 << 32)
        return [(a.data, b) for a, b in ex]

    step(d)                                   # eager warm-up: epoch 0
    g = GraphedStep(step, d)                  # capture records the launches without running them
    seen = []
    for k in range(1, 3):                     # replays: epochs 1, 2
        out = [(a.clone(), b.clone()) for a, b in g()]
        torch.cuda.synchronize()
        for i, (a, b) in enumerate(out):
            rm, rs = K.export_c2m(P13, cts[i], 2, seed, (k << 32) + i)
            assert np.array_equal(a.cpu().numpy().view(np.uint64).reshape(2, 2, P13.N), rm.c), (k, i)
            assert np.array_equal(b.cpu().numpy().view(np.uint64).reshape(2, P13.N), rs), (k, i)
        seen.append(out)
    assert not torch.equal(seen[0][0][1], seen[1][0][1])
