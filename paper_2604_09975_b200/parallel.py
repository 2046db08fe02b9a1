"""Multi-GPU partition of the hot path: host-side plumbing only (no CUDA, no torch import at module
level, so the partition logic is testable with the gloo backend on a CPU host).

* Projection: the (b, p) giant-step units are split into contiguous ranges, one per rank; each rank produces
  extended-basis partial accumulators acc_b for the b it touches; the partials of a block that straddles ranks are
  combined by a uint64 SUM followed by a per-limb modular reduction (encf_mod_reduce_ext) -- exact because
  world_size * q < 2^64 (q < 2^61) -- and finalised (conj + rescale) by the block's owner.  The modular sum is
  order-free, so the result is bit-identical to the 1-GPU run.
* Score: t-ranges; value: (block, t) unit ranges with unrelinearised partials reduced the same way.
The GPU layer (paper_2604_09975_b200/layer.py) reduces one [B_out][...] buffer with a single all-reduce on every rank;
`reduce_partial_blocks` is the per-block variant (every rank joins every straddled block's collective).
"""


def unit_ranges(units, world):
    """Contiguous, balanced [begin, end) ranges of `units` work items over `world` ranks."""
    base, extra = divmod(units, world)
    out, b = [], 0
    for r in range(world):
        e = b + base + (1 if r < extra else 0)
        out.append((b, e))
        b = e
    return out


def blocks_of(u0, u1, N2):
    """Output blocks b touched by units [u0, u1) (row-major over (b, p), N2 units per block)."""
    if u1 <= u0:
        return []
    return list(range(u0 // N2, (u1 - 1) // N2 + 1))


def owner_of_block(b, ranges, N2):
    """The rank that finalises block b: the last rank whose range touches it."""
    own = None
    for r, (u0, u1) in enumerate(ranges):
        if b in blocks_of(u0, u1, N2):
            own = r
    return own


def straddled_blocks(ranges, N2, B_out):
    """Blocks touched by more than one rank (the only ones that need a reduction), in increasing order."""
    return [b for b in range(B_out) if sum(1 for (u0, u1) in ranges if b in blocks_of(u0, u1, N2)) > 1]


def reduce_partial_blocks(partials, ranges, N2, B_out, all_reduce_sum, zeros_like):
    """partials[b] = this rank's partial accumulator words for block b (int64 tensor holding uint64 residues
    < q < 2^61) or absent.  EVERY rank calls all_reduce_sum once per straddled block, in the same order, contributing
    zeros (zeros_like(block_shape_source)) for a block it does not touch -- so the collectives pair up across ranks
    for any world size.  In place for the touched blocks; the caller then applies the modular reduction.  Returns
    the straddled blocks."""
    sb = straddled_blocks(ranges, N2, B_out)
    shape_src = next(iter(partials.values())) if partials else None
    for b in sb:
        if b in partials:
            all_reduce_sum(partials[b])
        else:
            t = zeros_like(shape_src)
            all_reduce_sum(t)
    return sb
