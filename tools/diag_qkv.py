import sys; sys.path.insert(0, '.')
import numpy as np, torch, synth
from oracle import ckks as O
from oracle import kernels as K
from paper_2604_09975_b200 import encf as E
from tests.test_gpu_fullsize import qkv_wbar, M, D, P
ctx = E.Context("P16", 0)
L = 8
X = synth.fixed_point_uniform((M, D), synth.seed_data(3))
Wbar = qkv_wbar(*(synth.bert_weight((D, D), synth.seed_data(3) + i) for i in range(3)))
plan = E.ProjPlan(ctx, M, D, Wbar.shape[1]); oplan = K.ProjPlan(P.n, M, D, Wbar.shape[1])
okeys = O.Keys(P, synth.SEED_KEYS, galois=[], max_level=L)
gkeys = ctx.keygen(synth.SEED_KEYS, galois=plan.galois(), max_level=L)
# compare GPU-encoded weights with oracle encoding for a few (b,p,u,q)
wd = plan.encode_weights(Wbar, L)
for (b, p, u, q) in [(0, 0, 0, 0), (0, 1, 0, 3), (1, 0, 0, 0), (5, 2, 1, 7), (10, 7, 1, 31)]:
    idx = ((b * oplan.N2 + p) * oplan.U + u) * oplan.N1 + q
    t = wd[idx * L * ctx.N:(idx + 1) * L * ctx.N].clone()
    pt = E.Plaintext(t, L, float(P.q[L - 1]), 1)
    g = ctx.to_host(pt)
    ref = O.encode(P, K.proj_weight_slots(Wbar, oplan, b, p, u, q), float(P.q[L - 1]), L).m
    d = (g.astype(object) - ref.astype(object))
    print((b, p, u, q), 'max |diff| (first limb)', max(abs(int(v)) for v in d[0][:4096]), 'n diff', int((g != ref).sum()))
xs = [O.encrypt_sk(P, okeys, O.encode(P, z, 2.0 ** 40, L), synth.seed_enc(u)) for u, z in enumerate(K.proj_inputs(X, oplan))]
ys = plan.matmul(gkeys, [ctx.to_ntt(ctx.ct_from_host(x.c, x.scale)) for x in xs], wd, float(P.q[L - 1]))
Y = X @ Wbar
for b, y in enumerate(ys):
    got = K.seg_column_unpack(O.decode(P, O.decrypt(P, okeys, O.Ct(ctx.to_host(y), y.scale))).real, M, 256, Wbar.shape[1], b)
    ref = Y[:, b * 256:(b + 1) * 256]
    print(b, 'rel err', np.abs(got - ref).max() / np.abs(Y).max(), 'scale', y.scale)
