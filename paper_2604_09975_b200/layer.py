"""One EncFormer CKKS-linear layer (BERT-shaped) on one GPU or sharded over a process group.

Host plumbing only: every step of the path runs in libencf kernels through the C ABI (encf.py); the collectives
are torch.distributed calls on uint64 words (NCCL over NVLink on a multi-GPU box; gloo in the same-GPU
multi-process tests).  The layer, in order:

  QKV projection -> score kernel (t-range per rank) -> minimal export stream + C2M export -> value kernel
  ((block, t) units per rank) -> decomplexify O -> out-projection -> C2M export -> FF1 -> C2M export -> FF2 -> C2M

Partition (one contiguous range of units per rank, `unit_ranges`):
  * projections: the (b, p) giant-step units.  Each rank holds ONLY its shard of the plaintext-diagonal stream
    (ENCF_PROJ_W_SHARD), builds the (replicated) baby-step bank, MACs its units and folds them into EXTENDED-basis
    partial accumulators acc_b (R-LAZY).  Exchange: one uint64 SUM all-reduce of the [B_out][2][L+K][N]
    partials (exact: world * q < 2^64), encf_mod_reduce_ext, the block owners finalise (decomplexify + rescale),
    one all-gather of the outputs.
  * score: t-ranges (the Q/K banks are rebuilt on every rank); all-gather of S_t; rank 0 packs the minimal export
    stream (K_min(S) ciphertexts).
  * value: (block l, t) units; every rank returns the UNRELINEARISED partial tensor sums of the blocks it touches;
    uint64 SUM all-reduce of [B_V][3][L][N], encf_mod_reduce, the owners relinearise + rescale, all-gather.
  * C2M exports: ciphertext i of a boundary by rank i mod world.
Modular sums are exact and order-free and every other step is a deterministic function of the same inputs, so
the sharded layer is bit-identical to the 1-GPU layer (tests/test_gpu_sharded.py).
"""
from dataclasses import dataclass

import numpy as np
import torch

from . import encf as E
from . import packing as PK


@dataclass
class LayerSpec:
    name: str
    params: str
    m: int
    d: int
    H: int
    d_h: int
    dff: int
    C_qk: int
    beta: int
    L_qkv: int = 8
    L_vp: int = 5
    L_ff: int = 3


BERT_BASE = LayerSpec("bert-base-layer", "P16", 128, 768, 12, 64, 3072, 192, 16)
BERT_LARGE = LayerSpec("bert-large-layer", "P16", 128, 1024, 16, 64, 4096, 192, 16)
TOY = LayerSpec("toy-layer-p13", "P13", 16, 32, 4, 8, 96, 16, 4)          # same level plan, N = 2^13 (tests)


def unit_ranges(units, world):
    """Contiguous, balanced [begin, end) ranges of `units` work items over `world` ranks."""
    base, extra = divmod(units, world)
    out, b = [], 0
    for r in range(world):
        e = b + base + (1 if r < extra else 0)
        out.append((b, e))
        b = e
    return out


class Comm:
    """The collectives the sharded layer uses, over a torch.distributed process group (None: one rank)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist if group is not None or (dist.is_available() and dist.is_initialized()) else None
        self.group = group
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0

    def all_reduce_sum_(self, t):
        """In-place SUM of int64 tensors holding uint64 words (two's-complement wrap == uint64 addition)."""
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def all_gather(self, t):
        """[world * t.shape[0], ...] concatenation of every rank's equally shaped t."""
        if self.world == 1:
            return t
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.cat(parts)

    def max_(self, x, key=None):
        """Max over ranks of a host double (ciphertext scales a rank without outputs cannot compute).  Scales are
        the same at every step, so with `key` the value is exchanged once and cached: later (CUDA-graph captured)
        steps issue no host-synchronising collective."""
        if self.world == 1:
            return x
        cache = self.__dict__.setdefault("_cache", {})
        if key is not None and key in cache:
            return cache[key]
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        v = float(t.item())
        if key is not None:
            cache[key] = v
        return v


def _owned(n, world, rank):
    """Contiguous block range [b0, b1) finalised by `rank` (n blocks over `world` ranks) and the per-rank count."""
    cnt = -(-n // world)
    b0 = min(rank * cnt, n)
    return b0, min(b0 + cnt, n), cnt


class ShardedProjection:
    """A projection plan plus this rank's shard of its weight stream."""

    def __init__(self, ctx, comm, m, d_in, d_out, W, L, seed_scale=None):
        self.ctx, self.comm = ctx, comm
        self.plan = E.ProjPlan(ctx, m, d_in, d_out)
        self.L, self.Lw = L, L           # restricted plans are not used by the layer (C = n/m)
        self.units = self.plan.B_out * self.plan.N2
        self.u0, self.u1 = unit_ranges(self.units, comm.world)[comm.rank]
        full = self.plan.encode_weights(W, self.Lw)
        per_unit = full.numel() // self.units
        self.w = full[self.u0 * per_unit:self.u1 * per_unit].clone() if comm.world > 1 else full
        del full
        self.w_scale = float(ctx.q[self.Lw - 1])

    def galois(self):
        return self.plan.galois()

    def __call__(self, keys, xs):
        ctx, comm, plan = self.ctx, self.comm, self.plan
        if comm.world == 1:
            return plan.matmul(keys, xs, self.w, self.w_scale)
        N = ctx.N
        parts = plan.matmul(keys, xs, self.w, self.w_scale, self.u0, self.u1, finalize=False, w_shard=True)
        b_first = self.u0 // plan.N2
        La = ctx.level_of_ext(parts[0].n_limbs)       # extended partials: La + K(La) limbs (R-LAZY, R-KL)
        K = ctx.K(La)
        wext = 2 * (La + K) * N
        buf = torch.zeros((plan.B_out, wext), dtype=torch.int64, device=ctx.device)
        for i, a in enumerate(parts):
            buf[b_first + i].copy_(a.data[:wext])
        comm.all_reduce_sum_(buf)                                   # exact uint64 SUM of the extended partials
        b0, b1, cnt = _owned(plan.B_out, comm.world, comm.rank)
        Ly = La - 1
        out = torch.zeros((cnt, 2 * Ly * N), dtype=torch.int64, device=ctx.device)
        scale = 0.0
        if b1 > b0:
            own = buf[b0:b1].contiguous()
            ctx.mod_reduce_ext(own, 2 * (b1 - b0), La)
            accs = [E.Ciphertext(own[i], 2, La + K, parts[0].scale, 1) for i in range(b1 - b0)]
            ys = plan.finalize(keys, accs, b0)
            for i, y in enumerate(ys):
                out[i].copy_(y.data[:2 * Ly * N])
            scale = ys[0].scale
        scale = comm.max_(scale, ("proj", id(self)))
        allys = comm.all_gather(out)
        return [E.Ciphertext(allys[r * cnt + i], 2, Ly, scale, 1)
                for r in range(comm.world) for i in range(_owned(plan.B_out, comm.world, r)[1] - _owned(plan.B_out, comm.world, r)[0])]


class ShardedLayer:
    """The layer state of one rank: context, keys, plans, weight shards, synthetic client inputs."""

    def __init__(self, spec, device, comm=None, seed_off=0):
        import synth
        self.spec, self.comm = spec, comm or Comm(None)
        ctx = self.ctx = E.Context(spec.params, device)
        n, m = ctx.n, spec.m
        self.C = n // m
        self.sc = 2.0 ** 40
        d, H, dh, dff = spec.d, spec.H, spec.d_h, spec.dff
        WQ, WK, WV = (synth.bert_weight((d, d), synth.seed_data(3) + i) for i in range(3))
        Wqkv, self.nqk, self.nv = PK.qkv_weight(WQ, WK, WV, H, dh, self.C, spec.C_qk)
        self.qkv = ShardedProjection(ctx, self.comm, m, d, Wqkv.shape[1], Wqkv, spec.L_qkv)
        self.attn = E.AttnPlan(ctx, m, H, dh, C_qk=spec.C_qk, beta=spec.beta)
        self.oproj = ShardedProjection(ctx, self.comm, m, d, d, synth.bert_weight((d, d), synth.seed_data(5) + 3), spec.L_vp - 2)
        self.ff1 = ShardedProjection(ctx, self.comm, m, d, dff, synth.bert_weight((d, dff), synth.seed_data(5) + 4), spec.L_ff)
        self.ff2 = ShardedProjection(ctx, self.comm, m, dff, d, synth.bert_weight((dff, d), synth.seed_data(5) + 5), spec.L_ff)
        galois = set()
        for pr in (self.qkv, self.oproj, self.ff1, self.ff2):
            galois |= set(pr.galois())
        galois |= set(self.attn.galois())
        galois.add(ctx.galois_conj())
        self.keys = ctx.keygen(synth.SEED_KEYS, galois=sorted(galois), relin=True, max_level=spec.L_qkv)
        X = synth.fixed_point_uniform((m, d), synth.seed_data(3) + seed_off)
        P = synth.attention_probs(H, m, synth.seed_data(4) + seed_off)
        X1 = synth.fixed_point_uniform((m, d), synth.seed_data(5) + seed_off)
        X2 = synth.fixed_point_uniform((m, dff), synth.seed_data(6) + seed_off, 0.0, 1.0)
        self.host_inputs = {
            "x": [self._enc(z, spec.L_qkv, 10 + i) for i, z in enumerate(PK.complexified_inputs(X, m, self.C, n))],
            # P_fd at Delta * 2^floor(log2 m) (DESIGN.md R-PSCALE)
            "p": [self._enc(z, spec.L_vp, 20 + i, scale=self.sc * 2.0 ** (m.bit_length() - 1))
                  for i, z in enumerate(PK.folded_diag_blocks(P, m, self.attn.H_blk, self.attn.seg_stride, n))],
            "f1": [self._enc(z, spec.L_ff, 30 + i) for i, z in enumerate(PK.complexified_inputs(X1, m, self.C, n))],
            "f2": [self._enc(z, spec.L_ff, 40 + i) for i, z in enumerate(PK.complexified_inputs(X2, m, self.C, n))],
        }
        self.dev_inputs = {k: [E.Ciphertext(h[0].to(ctx.device), h[1], h[2], h[3], 1) for h in v]
                           for k, v in self.host_inputs.items()}
        self.h2d_bytes = sum(h[0].nbytes for v in self.host_inputs.values() for h in v)
        self.Lconv = ctx.l_conv()
        self.mask_seed = synth.seed_mask(0)
        torch.cuda.synchronize()

    def _enc(self, z, L, seed, scale=None):
        ct = self.ctx.encrypt(self.keys, self.ctx.encode(z, scale or self.sc, L), seed)
        return (ct.data.cpu().pin_memory(), ct.n_comp, ct.n_limbs, ct.scale)

    def _complex_pairs(self, ys):
        out = [self.ctx.complexify(ys[2 * i], ys[2 * i + 1]) for i in range(len(ys) // 2)]
        if len(ys) % 2:
            out.append(ys[-1])
        return out

    MASK_EPOCH = 1 << 32

    def _export(self, cts, sid):
        """C2M export (Alg 3 GPU half) of ciphertext i by rank i mod world, mask stream id epoch 2^32 + sid + i with
        (seed, base) in a DEVICE buffer advanced every step (fresh one-time pads per inference, also under graph
        replay; encf_export_c2m_many_dev)."""
        comm = self.comm
        st = self.__dict__.setdefault("mask_state", {})
        if sid not in st:
            st[sid] = torch.tensor([self.mask_seed, sid], dtype=torch.int64, device=self.ctx.device)
        out = []
        for i in range(len(cts)):
            if i % comm.world == comm.rank:
                sti = st[sid] + torch.tensor([0, i], dtype=torch.int64, device=self.ctx.device)
                out += [(i, r) for r in self.ctx.export_c2m_many([cts[i]], self.Lconv, sti, 0)]
        return out

    def _advance_masks(self):
        for t in self.__dict__.get("mask_state", {}).values():
            t[1:].add_(self.MASK_EPOCH)

    def score(self, Q, K):
        comm, attn, ctx = self.comm, self.attn, self.ctx
        half = attn.m // 2
        if comm.world == 1:
            return attn.score(self.keys, Q, K)
        t0, t1 = unit_ranges(half, comm.world)[comm.rank]
        cnt = -(-half // comm.world)
        S = attn.score(self.keys, Q, K, t0, t1) if t1 > t0 else []
        Ls = Q[0].n_limbs - (4 if attn.C % attn.H else 3)
        N = ctx.N
        buf = torch.zeros((cnt, 2 * Ls * N), dtype=torch.int64, device=ctx.device)
        for i, s in enumerate(S):
            buf[i].copy_(s.data[:2 * Ls * N])
        scale = comm.max_(S[0].scale if S else 0.0, "score")
        allS = comm.all_gather(buf)
        out = []
        for r, (a, b) in enumerate(unit_ranges(half, comm.world)):
            out += [E.Ciphertext(allS[r * cnt + i], 2, Ls, scale, 1) for i in range(b - a)]
        return out

    def value(self, P, V):
        comm, attn, ctx = self.comm, self.attn, self.ctx
        if comm.world == 1:
            return attn.value(self.keys, P, V)
        units = attn.B_V * (attn.m // 2)
        u0, u1 = unit_ranges(units, comm.world)[comm.rank]
        blocks = attn.value_blocks(u0, u1)
        parts = attn.value_partial(self.keys, P, V, u0, u1)
        Lb, N = P[0].n_limbs - 1, ctx.N
        w3 = 3 * Lb * N
        buf = torch.zeros((attn.B_V, w3), dtype=torch.int64, device=ctx.device)
        for l, pr in zip(blocks, parts):
            buf[l].copy_(pr.data[:w3])
        comm.all_reduce_sum_(buf)
        o3_scale = comm.max_(parts[0].scale if parts else 0.0, "value_o3")
        b0, b1, cnt = _owned(attn.B_V, comm.world, comm.rank)
        out = torch.zeros((cnt, 2 * (Lb - 1) * N), dtype=torch.int64, device=ctx.device)
        scale = 0.0
        if b1 > b0:
            own = buf[b0:b1].contiguous()
            ctx.mod_reduce(own, 3 * (b1 - b0), Lb)
            os = attn.value_finalize(self.keys, [E.Ciphertext(own[i], 3, Lb, o3_scale, 1) for i in range(b1 - b0)])
            for i, o in enumerate(os):
                out[i].copy_(o.data[:2 * (Lb - 1) * N])
            scale = os[0].scale
        scale = comm.max_(scale, "value_o")
        allo = comm.all_gather(out)
        res = []
        for r in range(comm.world):
            a, b, _ = _owned(attn.B_V, comm.world, r)
            res += [E.Ciphertext(allo[r * cnt + i], 2, Lb - 1, scale, 1) for i in range(b - a)]
        return res

    def step(self, inp):
        """One sharded pass of the layer.  Returns this rank's exports [(boundary, index, (masked, share))]."""
        ctx, keys = self.ctx, self.keys
        y = self.qkv(keys, inp["x"])
        nqk = self.nqk
        Q, K, V = y[:nqk], y[nqk:2 * nqk], y[2 * nqk:]
        S = self.score(Q, K)
        ex = []
        if self.comm.rank == 0:              # the K_min(S) stream ciphertexts, exported by rank 0
            stream = self.attn.export_stream(keys, S)
            saved, self.comm = self.comm, _OneRank()
            ex += [("score", i, r) for i, r in self._export(stream, 0)]
            self.comm = saved
        O = self.value(inp["p"], V)
        Ore = ctx.decomplexify(keys, O)            # (G11) replicated: B_V conjugations
        yo = self.oproj(keys, self._complex_pairs(Ore))
        ex += [("ln1", i, r) for i, r in self._export(self._complex_pairs(yo), 100)]
        g1 = self.ff1(keys, inp["f1"])
        ex += [("gelu", i, r) for i, r in self._export(self._complex_pairs(g1), 200)]
        g2 = self.ff2(keys, inp["f2"])
        ex += [("ln2", i, r) for i, r in self._export(self._complex_pairs(g2), 300)]
        self.last = {"y_qkv": y, "S": S, "O": O, "yo": yo, "g1": g1, "g2": g2}
        self._advance_masks()
        return ex


class _OneRank:
    """A stand-in communicator of one rank (rank 0 exports the whole score stream)."""
    world, rank = 1, 0
