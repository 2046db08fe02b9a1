"""The paper's own, UNFUSED schedules of the three kernels and the export stream.

TEST INFRASTRUCTURE ONLY (see oracle/ckks.py header).

oracle/kernels.py fixes the bits of the B200 build: it keeps rotations in the extended basis Q_L u P and divides
once (R-LAZY), merges relinearisation with its rescale (R-RELRS) and routes by one hoisted rotation sum (R-ROUTE).
Those are exact identities in VALUE but not in bits (each ModDown / rescale rounds).  This module writes every
kernel the way the paper states it -- every rotation ModDown'ed on its own (Alg A.1-A.4 literally: rot, ptmul
with the mask, add, then rescale), relinearise then rescale, routing by the rotate-add tree of P:1441-1449,
decomplexification before the giant fold as in the main text -- over the same oracle CKKS
primitives (oracle/ckks.py), so that tests can show the fused schedules decrypt to the same values within the
noise of the paper's order on the same inputs (tests/test_oracle_schedules.py).

Citations per function.  Readings shared with kernels.py: G7 (routing sign), G9 (Psi^{+t}), R-PSI0, R-MASK.
"""
import numpy as np

from . import ckks as O
from . import kernels as K


def psi(ev, x, t, m, N_seg, seg0=0, nseg=None):
    """Alg A.2 literally: t <- t mod m; rot(x; t) (.) h + rot(x; (t - m) mod n) (.) u, then rescale.
    The two rotations come from one hoisted ModUp and are each ModDown'ed (ordinary hoisted rotations)."""
    t = int(t) % m
    L = x.L
    hd, ud = K.psi_masks(t, m, N_seg, seg0, nseg)
    if t == 0:
        return ev.rescale(ev.ptmul(x, ev.mask(hd, L, m)))
    r1, r2 = ev.rot_hoisted(x, [t, t - m])
    return ev.rescale(ev.add(ev.ptmul(r1, ev.mask(hd, L, m)), ev.ptmul(r2, ev.mask(ud, L, m))))


def rotfirst(ev, x, Ls, tau, m):
    """Alg A.3 literally: tau <- tau mod L; rot(x; tau) (.) a + rot(x; (tau - L) mod n) (.) b, then
    rescale (the rotations ModDown'ed)."""
    tau = int(tau) % Ls
    L = x.L
    (ad, am), bb = K.rotfirst_masks(Ls, tau, m)
    if tau == 0:
        return ev.rescale(ev.ptmul(x, ev.mask(ad, L, am)))
    bd, bm = bb
    r1, r2 = ev.rot_hoisted(x, [tau, tau - Ls])
    return ev.rescale(ev.add(ev.ptmul(r1, ev.mask(ad, L, am)), ev.ptmul(r2, ev.mask(bd, L, bm))))


def projection(ev, plan, xt, w, decomplexify=True):
    """§3.2 in the main text's order:
      x~_q = Phi_C^q(x~)  (a hoisted rotation, or RotFirst_{Cm} when C < N_seg, Alg A.4)
      c~_p = sum_{q,u} x~_q (.) w~_{u,p,q}
      c_p = (c~_p + conj(c~_p)) / 2      (decomplexify EACH giant accumulator; the 1/2 as scale, G3)
      y = sum_p Phi_C^{p N1}(c_p)          (single rotations, each ModDown'ed; RotFirst when C < N_seg)
    then rescale.  Returns y_b for every output block."""
    m, N1 = plan.m, plan.N1
    bank = []
    for u in range(plan.U):
        if plan.restricted:
            bank.append([rotfirst(ev, xt[u], plan.C * m, q * m, m) for q in range(N1)])
        else:
            rots = ev.rot_hoisted(xt[u], [q * m for q in range(1, N1)]) if N1 > 1 else []
            bank.append([xt[u]] + list(rots))
    ys = []
    for b in range(plan.B_out):
        acc = None
        for p in range(plan.N2):
            cts = [bank[u][q] for u in range(plan.U) for q in range(N1)]
            c = ev.mac_ptmul(cts, [w(b, p, u, q) for u in range(plan.U) for q in range(N1)])
            if decomplexify:
                c = ev.scale_mul(ev.add(c, ev.conj(c)), 2.0)
            if plan.restricted:
                y = rotfirst(ev, c, plan.C * m, p * N1 * m, m)
            else:
                y = ev.rot(c, p * N1 * m) if p else c
            acc = y if acc is None else ev.add(acc, y)
        ys.append(ev.rescale(acc))
    return ys


def score(ev, plan, qs, ks, ts=None):
    """§3.3.1 with App. A.3's phase correction:
      Q bank Psi^{-s}, K bank Psi^{j beta}, Psi^{m/2 + j beta}            (Alg A.2 per offset)
      u_t^(r) = sum_{l: l C mod H = r} q_{-s} (x) (k_{j beta} + i k_{m/2 + j beta}), relinearise, rescale
      route: the rotate-add tree of single rotations (sign G7)
      Align_r = RotFirst_{Hm}(., (H - r) m) per phase, summed        (only when C mod H != 0)
      S_t = Psi^{s}(.) restricted to the H head segments             (R-ALIGN)"""
    m, H, beta, g, N_seg = plan.m, plan.H, plan.beta, plan.g, plan.N_seg
    qb = [[psi(ev, qs[l], -s, m, N_seg) for s in range(beta)] for l in range(plan.B)]
    kb = []
    for l in range(plan.B):
        kt = [j * beta for j in range(g // 2)] + [m // 2 + j * beta for j in range(g // 2)]
        kb.append({t: psi(ev, ks[l], t, m, N_seg) for t in kt})
    groups = K.score_phase_groups(plan)
    S = []
    for t in (range(m // 2) if ts is None else ts):
        j, s = t // beta, t % beta
        parts = []
        for r, ls in sorted(groups.items()):
            u = None
            for l in ls:
                prod = ev.tensor(qb[l][s], ev.add(kb[l][j * beta], ev.mul_i(kb[l][m // 2 + j * beta])))
                u = prod if u is None else ev.add(u, prod)
            T = ev.rescale(ev.relin(u))
            T = K.route(ev, T, plan.k_route, H, m, hoisted=False)
            parts.append(rotfirst(ev, T, H * m, (H - r) * m, m) if plan.aligned else T)
        T = parts[0]
        for x in parts[1:]:
            T = ev.add(T, x)
        S.append(psi(ev, T, s, m, N_seg, 0, H))
    return S


def score_export(ev, plan, S):
    """Minimal export stream (R-EXP) with every offset rotation ModDown'ed, the pieces masked, summed
    and rescaled (the paper's ptmul/add/rescale order)."""
    m, H, n = plan.m, plan.H, plan.n
    seg = H * m
    outs = [None] * plan.n_out
    L = S[0].L
    for t, st in enumerate(S):
        start = t * seg
        o = start % n
        r = ev.rot(st, -o) if o else st
        k = start // n
        first = min(seg, n - o)
        pieces = [(k, o, o + first)]
        if first < seg:
            pieces.append((k + 1, 0, seg - first))
        for (ci, a, b) in pieces:
            y = ev.ptmul(r, ev.mask((0, m, a // m, 1, (b - a) // m), L, m))
            outs[ci] = y if outs[ci] is None else ev.add(outs[ci], y)
    return [ev.rescale(x) for x in outs]


def value(ev, plan, ps, vs):
    """§3.3.2 (G9 Psi^{+t}): uu = v - i Psi^{m/2}(v) (one rescale), U bank Psi^t (Alg A.2 each),
    Phi bank of p_fd (hoisted rotations, each ModDown'ed), b_t = sum_u Phi^{t-u}(p) (.) n_u then rescale,
    o = sum_t u_t (x) b_t, relinearise, then rescale."""
    m, N_seg = plan.m, plan.N_seg
    half = m // 2
    outs = []
    for l in range(plan.B_V):
        v, p = vs[l], ps[l]
        Lv = v.L
        rv = ev.rot_hoisted(v, [half, half - m])
        hd, ud = K.psi_masks(half, m, N_seg)
        sh = ev.add(ev.ptmul(rv[0], ev.mask(hd, Lv, m)), ev.ptmul(rv[1], ev.mask(ud, Lv, m)))
        uu = ev.rescale(ev.sub(ev.ptmul(v, ev.mask((0, m, 0, 1, N_seg), Lv, m)), ev.mul_i(sh)))
        ub = [psi(ev, uu, t, m, N_seg) for t in range(half)]
        deltas = [d for d in range(-(plan.d_h - 1), half) if d != 0]
        pb = dict(zip(deltas, ev.rot_hoisted(p, [d * m for d in deltas])))
        pb[0] = p
        Lp = p.L
        o = None
        for t in range(half):
            bt = ev.rescale(ev.mac_ptmul([pb[t - u] for u in range(plan.d_h)],
                                         [ev.mask((0, m, u, plan.seg_stride, plan.H_blk), Lp, m) for u in range(plan.d_h)]))
            ut = ev.mod_drop(ub[t], bt.L) if ub[t].L > bt.L else ub[t]
            prod = ev.tensor(ut, bt)
            o = prod if o is None else ev.add(o, prod)
        outs.append(ev.rescale(ev.relin(o)))
    return outs
