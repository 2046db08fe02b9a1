"""Multi-process (gloo, world_size 2, CPU) test of the sharded projection's host logic: units are split
across ranks, each rank computes its partial accumulators (the oracle stands in for the GPU compute),
blocks straddling ranks are SUM-reduced as uint64 over the process group and mod-reduced, then
finalised -- the result must be bit-identical to the unsharded projection."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import ckks as O
from oracle import kernels as K
from paper_2604_09975_b200 import parallel as PAR


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    P = O.Params("P12")
    plan = K.ProjPlan(P.n, 32, 64, 130, N1=8)          # B_out = 3, N2 = 8 -> 24 units
    rots = [q * plan.m for q in range(1, plan.N1)] + [p * plan.N1 * plan.m for p in range(1, plan.N2)]
    keys = O.Keys(P, synth.SEED_KEYS, galois=[O.galois_rot(P, r) for r in rots] + [O.galois_conj(P)])
    X = synth.fixed_point_uniform((32, 64), 3)
    W = synth.bert_weight((64, 130), 4)
    L = 3
    xs = [O.encrypt_sk(P, keys, O.encode(P, z, 2.0 ** 40, L), synth.seed_enc(u)) for u, z in enumerate(K.proj_inputs(X, plan))]
    cache = {}

    def w(b, p, u, q):
        if (b, p, u, q) not in cache:
            cache[(b, p, u, q)] = O.encode(P, K.proj_weight_slots(W, plan, b, p, u, q), float(P.q[L - 1]), L)
        return cache[(b, p, u, q)]
    return P, plan, keys, xs, w


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, plan, keys, xs, w = _setup()
    units = plan.B_out * plan.N2
    ranges = PAR.unit_ranges(units, world)
    u0, u1 = ranges[rank]
    ev = K.Ev(P, keys, plan.m)
    accs = K.projection_partial(ev, plan, xs, w, u0, u1)      # {b: ExtCt} extended-basis partials (R-LAZY)
    parts = {b: torch.from_numpy(a.c.view(np.int64).copy()) for b, a in accs.items()}
    PAR.reduce_partial_blocks(parts, ranges, plan.N2, plan.B_out, lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM),
                              torch.zeros_like)
    ys = {}
    for b, t in parts.items():
        if PAR.owner_of_block(b, ranges, plan.N2) != rank:
            continue
        words = t.numpy().view(np.uint64).reshape(accs[b].c.shape)
        mods = np.array(P.ext_mods(accs[b].L), dtype=np.uint64)[None, :, None]
        acc = K.ExtCt(words % mods, accs[b].L, accs[b].scale)   # the modular reduction after the uint64 SUM
        ys[b] = K.projection_finalize(ev, plan, acc).c
    q.put((rank, ys))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_projection_equals_single_rank(world):
    """world = 4: rank 0 touches only block 0 and rank 3 only block 2, so the per-block collectives pair up only
    because every rank joins every straddled block's all-reduce (a rank skipping one mismatched them)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, ys = q.get(timeout=500)
        got.update(ys)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P, plan, keys, xs, w = _setup()
    ref = K.projection(K.Ev(P, keys, plan.m), plan, xs, w)
    assert sorted(got) == list(range(plan.B_out))
    for b in range(plan.B_out):
        assert np.array_equal(got[b], ref[b].c), b


def test_straddled_blocks():
    ranges = PAR.unit_ranges(24, 4)
    assert ranges == [(0, 6), (6, 12), (12, 18), (18, 24)]
    assert PAR.straddled_blocks(ranges, 8, 3) == [0, 1, 2]
    assert [PAR.owner_of_block(b, ranges, 8) for b in range(3)] == [1, 2, 3]
    assert PAR.straddled_blocks(PAR.unit_ranges(24, 3), 8, 3) == []


def test_unit_ranges_cover_and_balance():
    for units in (1, 7, 72, 144):
        for world in (1, 2, 3, 8):
            r = PAR.unit_ranges(units, world)
            assert r[0][0] == 0 and r[-1][1] == units
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [e - s for s, e in r]
            assert max(sizes) - min(sizes) <= 1
