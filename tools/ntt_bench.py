"""NTT throughput microbench through the C ABI: forward+inverse of a batch of limbs at N = 2^16."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2604_09975_b200 import encf as E  # noqa: E402


def run(nlimbs=24, npolys=16, reps=20):
    ctx = E.Context("P16", 0)
    t = torch.randint(0, 1 << 39, (npolys * nlimbs * ctx.N,), dtype=torch.int64, device="cuda")
    for _ in range(3):
        ctx.poly_to_ntt(t, npolys, nlimbs)
        E._chk(E._lib.encf_poly_from_ntt(ctx.h, t.data_ptr(), npolys, nlimbs, E._stream()), "from")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        ctx.poly_to_ntt(t, npolys, nlimbs)
        E._chk(E._lib.encf_poly_from_ntt(ctx.h, t.data_ptr(), npolys, nlimbs, E._stream()), "from")
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    per = ms * 1e3 / (reps * 2 * npolys * nlimbs)
    return per


if __name__ == "__main__":
    print("us per limb-NTT: %.3f" % run())
