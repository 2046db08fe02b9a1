"""T6: the sharded layer on W ranks equals the 1-rank layer BIT FOR BIT.

W processes share the one visible GPU (the gpurun box has one B200) and talk over the gloo backend with CUDA
tensors, so the test runs the real CUDA data plane and the real collective plumbing of
paper_2604_09975_b200/layer.py (the same code bench.py drives with NCCL across GPUs): projection unit shards with
an extended-basis uint64 all-reduce, score t-ranges with an all-gather, value (block, t) partials with a uint64
all-reduce, owner finalisation and all-gathers, exports by ciphertext index.  Every intermediate (Q/K/V, S_t, O,
out-projection, FF1, FF2) and every exported (masked ciphertext, server share) must equal the single-rank run's."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _snapshot(layer, ex):
    out = {}
    for k, v in layer.last.items():
        out[k] = [(c.data.cpu().numpy().copy(), c.n_comp, c.n_limbs, c.scale) for c in v]
    out["exports"] = {(b, i): (m.data.cpu().numpy().copy(), s.cpu().numpy().copy()) for b, i, (m, s) in ex}
    return out


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_09975_b200 import layer as LY
    layer = LY.ShardedLayer(LY.TOY, 0, LY.Comm(None))
    ex = layer.step(layer.dev_inputs)
    torch.cuda.synchronize()
    q.put((rank, _snapshot(layer, ex)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def single():
    from paper_2604_09975_b200 import layer as LY
    layer = LY.ShardedLayer(LY.TOY, 0)
    ex = layer.step(layer.dev_inputs)
    torch.cuda.synchronize()
    return _snapshot(layer, ex)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_layer_equals_single_rank(single, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=800) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for k in ("y_qkv", "S", "O", "yo", "g1", "g2"):
        for r in range(world):           # replicated after the all-gathers: every rank holds the full outputs
            assert len(res[r][k]) == len(single[k]), (k, r)
            for i, (a, b) in enumerate(zip(res[r][k], single[k])):
                assert a[1:] == b[1:], (k, r, i, a[1:], b[1:])
                assert np.array_equal(a[0], b[0]), "%s[%d] differs on rank %d (world %d)" % (k, i, r, world)
    merged = {}
    for r in range(world):
        merged.update(res[r]["exports"])
    assert set(merged) == set(single["exports"])
    for key, (m, s) in single["exports"].items():
        assert np.array_equal(merged[key][0], m) and np.array_equal(merged[key][1], s), key
