"""Multi-GPU partition of the hot path: host-side plumbing only.

* Projection: the (b, p) giant-step units are split into contiguous ranges, one per rank; each rank
  produces partial accumulators acc_b (level L) for the b it touches; the partials of a block that
  straddles ranks are combined by a uint64 SUM (NCCL all_reduce / reduce) followed by a per-limb
  modular reduction (encf_mod_reduce) -- exact because world_size * q < 2^64 (q < 2^61) -- and
  finalised (conj + rescale) by the block's owner.  The modular sum is order-free, so the result is
  bit-identical to the 1-GPU run.
* Score: t-ranges; value: independent blocks (no reduction needed).
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


def reduce_partial_blocks(partials, ranges, N2, B_out, all_reduce_sum):
    """partials[b] = this rank's partial accumulator words for block b (int64 tensor holding uint64
    residues < q < 2^61) or None.  Every touched block is SUM-reduced across ranks with
    all_reduce_sum(tensor) (in place); the caller then applies the modular reduction.  Returns the
    list of blocks that were reduced."""
    reduced = []
    for b in range(B_out):
        touching = [r for r, (u0, u1) in enumerate(ranges) if b in blocks_of(u0, u1, N2)]
        if len(touching) > 1 and partials.get(b) is not None:
            all_reduce_sum(partials[b])
            reduced.append(b)
    return reduced
