"""Helpers shared by the GPU parity tests (oracle <-> library marshalling; no arithmetic)."""
import numpy as np
import torch

from oracle import ckks as O


def dev_ct(ctx, ct):
    return ctx.to_ntt(ctx.ct_from_host(ct.c, ct.scale))


def dev_pt(ctx, pt):
    return ctx.to_ntt(ctx.pt_from_host(pt.m, pt.scale))


def host_ct(ctx, ct):
    return O.Ct(ctx.to_host(ct), ct.scale)


def assert_ct_equal(ctx, got, ref, what=""):
    g = ctx.to_host(got)
    assert g.shape == ref.c.shape, (what, g.shape, ref.c.shape)
    assert got.scale == ref.scale, (what, got.scale, ref.scale)
    if not np.array_equal(g, ref.c):
        bad = np.argwhere(g != ref.c)
        raise AssertionError("%s: %d of %d words differ, first at %s" % (what, len(bad), g.size, bad[0]))


def install_masks(ctx, ev):
    for key, pt in ev.masks.items():
        if key[0] == "ext":
            _, desc, L, m = key
            ctx.mask_put(desc, m, L, pt.m, ext=True)
        else:
            desc, L, m = key
            ctx.mask_put(desc, m, L, pt.m)


def weights_tensor(ctx, pts, L):
    w = torch.from_numpy(np.ascontiguousarray(np.stack([p.m for p in pts])).view(np.int64).reshape(-1).copy()).to(ctx.device)
    ctx.poly_to_ntt(w, len(pts), L)
    return w
