"""Per-phase, per-kernel device time of one BERT-base layer step (eager, every launch bracketed by CUDA events).
Usage: python tools/phase_breakdown.py [layer|bert-large-layer] > gpurun_out/phase_breakdown.json"""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

KERNELS = bench.PROF_KERNELS


def main():
    workload = sys.argv[1] if len(sys.argv) > 1 else "layer"
    layer = bench.Layer(0, workload)
    ctx, keys, inp = layer.ctx, layer.keys, layer.dev_inputs
    for _ in range(2):
        layer.step(inp)
    torch.cuda.synchronize()
    out = {}

    def phase(name, fn):
        ctx.profile("*")
        r = fn()
        torch.cuda.synchronize()
        out[name] = {k: round(v[0], 3) for k, v in ((k, ctx.profile_read(k)) for k in KERNELS) if v[1]}
        ctx.profile(None)
        return r

    y = phase("qkv", lambda: layer.qkv.matmul(keys, inp["x"], layer.w_qkv, layer.wsc_qkv))
    nqk = layer.nqk
    Q, K, V = y[:nqk], y[nqk:2 * nqk], y[2 * nqk:]
    S = phase("score", lambda: layer.attn.score(keys, Q, K))
    phase("score_export", lambda: layer.attn.export_stream(keys, S))
    phase("value", lambda: layer.attn.value(keys, inp["p"], V))
    for k, v in out.items():
        v["_sum"] = round(sum(v.values()), 3)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
