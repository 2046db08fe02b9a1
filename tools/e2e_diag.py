"""Diagnose the pipelined e2e path: time graph A alone, graph B alone, serialized copies, pipelined copies."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2604_09975_b200.graphs import GraphedStep, PipelinedStep  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "layer"
layer = bench.Layer(0, w)
for _ in range(2):
    layer.step(layer.dev_inputs)
torch.cuda.synchronize()
ga = GraphedStep(layer.step, layer.dev_inputs)
inb = {k: [layer.E.Ciphertext(c.data.clone(), c.n_comp, c.n_limbs, c.scale, c.ntt) for c in v] for k, v in layer.dev_inputs.items()}
pipe = PipelinedStep(layer.step, ga, inb)
free, tot = torch.cuda.mem_get_info()
print("mem free %.1f GB of %.1f" % (free / 1e9, tot / 1e9))
host = {k: [h[0] for h in v] for k, v in layer.host_inputs.items()}
pin = [[(torch.empty(m.data.shape, dtype=m.data.dtype, pin_memory=True),
         torch.empty(sh.shape, dtype=sh.dtype, pin_memory=True) if sh is not None else None) for m, sh in g.outputs] for g in pipe.g]


def timeit(fn, n=4):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("graph A alone %.2f ms" % timeit(lambda: pipe.g[0].graph.replay()))
print("graph B alone %.2f ms" % timeit(lambda: pipe.g[1].graph.replay()))
print("A then B %.2f ms per graph" % (timeit(lambda: (pipe.g[0].graph.replay(), pipe.g[1].graph.replay())) / 2))
print("A with H2D+D2H serialized %.2f ms" % timeit(lambda: ga(host)))
print("pipelined %.2f ms per step" % (timeit(lambda: pipe.run(host, pin, 4), n=2) / 4))
