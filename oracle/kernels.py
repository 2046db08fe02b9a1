"""Oracle for the three EncFormer CKKS kernels + the GPU half of the complex C2M export.

TEST INFRASTRUCTURE ONLY (see oracle/ckks.py header).

The kernels are written as schedules over an evaluator `ev` so the same code runs
  * on real ciphertexts (Ev: oracle/ckks.py arithmetic, bit-exact reference for the GPU), and
  * in count-only mode (CountEv) at the paper's own shapes (n = 16384) to pin the key-switch counts
    of Table 2.
Every step cites the passage it follows; the schedule choices where the paper is silent or wrong are
SURVEY.md §8c C6-C9 / G1-G29 and are restated in DESIGN.md "Readings".
"""
from collections import Counter

import numpy as np

from . import ckks as O


# ====================================================================================== packing (slot level)
def mat(x, m):
    """(mat x)_{r,s} = x_{s m + r}."""
    return np.asarray(x).reshape(-1, m).T


def vec(X):
    return np.asarray(X).T.reshape(-1)


def seg_column_pack(X, m, C, g, n):
    """Segment-column packing: segment c < C holds column X[:, gC + c] (zero past d_in)."""
    d = X.shape[1]
    z = np.zeros(n, dtype=np.complex128)
    for c in range(C):
        col = g * C + c
        if col < d:
            z[c * m:(c + 1) * m] = X[:, col]
    return z


def seg_column_unpack(z, m, C, d, b):
    """Inverse for output block b: columns bC .. bC+C-1 (clipped to d)."""
    cols = [z[c * m:(c + 1) * m] for c in range(C) if b * C + c < d]
    return np.stack(cols, axis=1) if cols else np.zeros((m, 0))


def pi_S(H, d_h):
    """Score-friendly column order: pi_S(h,u) = uH + h; returns perm with
    Wpi[:, pi_S(h,u)] = W[:, k(h,u)], k(h,u) = h d_h + u."""
    perm = np.empty(H * d_h, dtype=np.int64)
    for h in range(H):
        for u in range(d_h):
            perm[u * H + h] = h * d_h + u
    return perm


def apply_col_perm(W, perm):
    return W[:, perm]


def k_min(n_entries, n):
    """K_min(x) = ceil(N(x) / 2n)."""
    return -(-int(n_entries) // (2 * int(n)))


# ====================================================================================== masks
def mask_slots(desc, m, n):
    """Mask descriptor (r0, r1, s0, sstride, scount): ones on rows [r0, r1) of segments
    s0 + k*sstride (k < scount), zero elsewhere.  Covers H/U of Alg A.2, e_s / m_c /
    n_u of App. A.3 and the export range masks."""
    r0, r1, s0, ss, sc = desc
    z = np.zeros(n)
    for k in range(sc):
        s = s0 + k * ss
        z[s * m + r0: s * m + r1] = 1.0
    return z


def psi_masks(t, m, N_seg, seg0=0, nseg=None):
    """H and U of Alg A.2 for shift t (already reduced mod m), optionally restricted to
    segments [seg0, seg0+nseg)."""
    nseg = N_seg if nseg is None else nseg
    return (0, m - t, seg0, 1, nseg), (m - t, m, seg0, 1, nseg)


# ====================================================================================== evaluators
class Ev:
    """Real evaluator over the oracle's CKKS (bit-exact reference)."""

    def __init__(self, P, keys, m=None):
        self.P, self.keys = P, keys
        self.ledger = Counter()
        self.masks = {}          # (desc, level, m) -> Pt   (what the schedule used)
        self.m = m

    # -- plaintexts
    def mask(self, desc, L, m=None):
        m = m or self.m
        key = (tuple(desc), L, m)
        if key not in self.masks:
            z = mask_slots(desc, m, self.P.n)
            self.masks[key] = O.encode(self.P, z, float(self.P.q[L - 1]), L)
        return self.masks[key]

    # -- ciphertext ops
    def rot(self, ct, r):
        if int(r) % self.P.n:
            self.ledger["rot"] += 1
        return O.rotate(self.P, self.keys, ct, r)

    def rot_hoisted(self, ct, rs):
        self.ledger["rot"] += sum(1 for r in rs if int(r) % self.P.n)
        self.ledger["modup_hoisted"] += 1
        return O.rotate_hoisted(self.P, self.keys, ct, rs)

    def conj(self, ct):
        self.ledger["conj"] += 1
        return O.conjugate(self.P, self.keys, ct)

    def tensor(self, a, b):
        self.ledger["ctmul"] += 1
        return O.tensor(self.P, a, b)

    def relin(self, ct):
        self.ledger["relin"] += 1
        return O.relinearize(self.P, self.keys, ct)

    def ptmul(self, ct, pt):
        self.ledger["ptmul"] += 1
        return O.ptmul(self.P, ct, pt)

    def add(self, a, b):
        return O.add(self.P, a, b)

    def sub(self, a, b):
        return O.sub(self.P, a, b)

    def mul_i(self, ct):
        return O.mul_i(self.P, ct)

    def rescale(self, ct):
        self.ledger["rescale"] += 1
        return O.rescale(self.P, ct)

    def mod_drop(self, ct, L):
        return O.mod_drop(self.P, ct, L)

    def scale_mul(self, ct, f):
        """Scale bookkeeping only (the 1/2 of decomplexification, G3): no arithmetic."""
        return O.Ct(ct.c, ct.scale * f)

    # -- lazy (extended-basis) operations, DESIGN.md R-LAZY
    def mask_ext(self, desc, L, m=None):
        """The mask plaintext of (desc, L) extended to the special primes (same integer coefficients)."""
        m = m or self.m
        key = ("ext", tuple(desc), L, m)
        if key not in self.masks:
            z = mask_slots(desc, m, self.P.n)
            coeffs = O.encode_coeffs(z, float(self.P.q[L - 1]), self.P.N)
            self.masks[key] = O.Pt(O.from_signed(coeffs, self.P.ext_mods(L), self.P.N), float(self.P.q[L - 1]))
        return self.masks[key]

    def mask_scale(self, L):
        return float(self.P.q[L - 1])

    def rot_hoisted_ext(self, ct, rs):
        self.ledger["rot"] += sum(1 for r in rs if int(r) % self.P.n)
        self.ledger["modup_hoisted"] += 1
        return [ExtCt(c, ct.L, ct.scale) for c in O.rotate_hoisted_ext(self.P, self.keys, ct, rs)]

    def ext_masked_sum(self, xs, pts, scale):
        """sum_i xs[i] (.) pts[i] over Q_L u P (ring products via the oracle NTT; exact)."""
        self.ledger["ptmul"] += len(xs)
        L = xs[0].L
        emods = self.P.ext_mods(L)
        N = self.P.N
        acc = [np.zeros((len(emods), N), np.uint64) for _ in range(2)]
        for x, pt in zip(xs, pts):
            ptn = O.ntt(pt.m, emods, N)
            for c in range(2):
                acc[c] = O.padd(acc[c], O.pmul_pointwise(O.ntt(x.c[c], emods, N), ptn, emods, N), emods, N)
        return ExtCt(np.stack([O.intt(a, emods, N) for a in acc]), L, scale)

    def lift_ext(self, ct):
        """P * ct in the extended basis (exact)."""
        return ExtCt(np.stack([O.lift_P(self.P, ct.c[i], ct.L) for i in range(2)]), ct.L, ct.scale)

    def rot_ext(self, ct, r):
        if int(r) % self.P.n == 0:
            return self.lift_ext(ct)
        self.ledger["rot"] += 1
        return ExtCt(O.rotate_ext(self.P, self.keys, ct, O.galois_rot(self.P, r)), ct.L, ct.scale)

    def conj_ext(self, ct):
        self.ledger["conj"] += 1
        return ExtCt(O.rotate_ext(self.P, self.keys, ct, O.galois_conj(self.P)), ct.L, ct.scale)

    def ext_add(self, a, b):
        if a.scale != b.scale:
            raise O.OracleError("SCALE_MISMATCH")
        em = self.P.ext_mods(a.L)
        return ExtCt(np.stack([O.padd(a.c[i], b.c[i], em, self.P.N) for i in range(2)]), a.L, a.scale)

    def moddown(self, y):
        self.ledger["moddown"] += 1
        return O.Ct(O.moddown_ext(self.P, y.c, y.L), y.scale)

    def moddown_rescale(self, y):
        self.ledger["moddown"] += 1
        self.ledger["rescale"] += 1
        L = y.L
        c = np.stack([O.moddown_rescale(self.P, y.c[i], L) for i in range(2)])
        return O.Ct(c, y.scale / float(self.P.q[L - 1]))

    def relin_rescale(self, ct):
        """rescale(relin(ct)) with ONE rounding (R-RELRS): the relin key switch kept in the extended basis and
        divided by P q_{L-1} at once."""
        self.ledger["relin"] += 1
        return self.moddown_rescale(ExtCt(O.relinearize_ext(self.P, self.keys, ct), ct.L, ct.scale))

    def mac_ptmul(self, cts, pts):
        """sum_i cts[i] (.) pts[i]  (exact modular sum of ring products; evaluated in the oracle's NTT
        domain -- the sum of ring products is unique)."""
        self.ledger["ptmul"] += len(cts)
        P, N = self.P, self.P.N
        L = cts[0].L
        mods = P.q[:L]
        acc = [np.zeros((L, N), np.uint64) for _ in range(2)]
        cache = self.__dict__.setdefault("_ntt_cache", {})
        for ct, pt in zip(cts, pts):
            if ct.L != L or pt.L != L:
                raise O.OracleError("LEVEL_MISMATCH")
            key = id(ct)
            if key not in cache or cache[key][0] is not ct:
                cache[key] = (ct, [O.ntt(ct.c[c], mods, N) for c in range(2)])
            ctn = cache[key][1]
            pkey = ("pt", id(pt))
            if pkey not in cache or cache[pkey][0] is not pt:
                cache[pkey] = (pt, O.ntt(pt.m, mods, N))
            ptn = cache[pkey][1]
            for c in range(2):
                acc[c] = O.padd(acc[c], O.pmul_pointwise(ctn[c], ptn, mods, N), mods, N)
        scale = cts[0].scale * pts[0].scale
        for ct, pt in zip(cts, pts):
            if ct.scale * pt.scale != scale:
                raise O.OracleError("SCALE_MISMATCH")
        return O.Ct(np.stack([O.intt(a, mods, N) for a in acc]), scale)

    def tensor_sum(self, pairs):
        """sum_t a_t (x) b_t without relinearisation (lazy sum; exact)."""
        out = None
        for a, b in pairs:
            t = self.tensor(a, b)
            out = t if out is None else O.add(self.P, out, t)
        return out


class ExtCt:
    """A ciphertext over the extended basis Q_L u P (coefficient form [2][L+K][N]), scale = the scale of
    the message it carries after the pending division by P."""

    def __init__(self, c, L, scale):
        self.c, self.L, self.scale = c, L, float(scale)
        self.ncomp = 2


class FakeCt:
    def __init__(self, L, scale=1.0, ncomp=2):
        self.L, self.scale, self.ncomp = L, scale, ncomp


class CountEv:
    """Count-only evaluator: same schedule, no arithmetic (for the paper's n=16384 count pins)."""

    def __init__(self, n, q_of_level=None, m=None):
        self.n = n
        self.ledger = Counter()
        self.m = m

    def mask(self, desc, L, m=None):
        return FakeCt(L, 1.0, 1)

    def rot(self, ct, r):
        if int(r) % self.n:
            self.ledger["rot"] += 1
        return FakeCt(ct.L, ct.scale)

    def rot_hoisted(self, ct, rs):
        self.ledger["rot"] += sum(1 for r in rs if int(r) % self.n)
        self.ledger["modup_hoisted"] += 1
        return [FakeCt(ct.L, ct.scale) for _ in rs]

    def conj(self, ct):
        self.ledger["conj"] += 1
        return FakeCt(ct.L, ct.scale)

    def tensor(self, a, b):
        self.ledger["ctmul"] += 1
        return FakeCt(a.L, 1.0, 3)

    def relin(self, ct):
        self.ledger["relin"] += 1
        return FakeCt(ct.L, ct.scale)

    def ptmul(self, ct, pt):
        self.ledger["ptmul"] += 1
        return FakeCt(ct.L, ct.scale, ct.ncomp)

    def add(self, a, b):
        return FakeCt(a.L, a.scale, max(a.ncomp, b.ncomp))

    sub = add

    def mul_i(self, ct):
        return ct

    def rescale(self, ct):
        self.ledger["rescale"] += 1
        return FakeCt(ct.L - 1, ct.scale, ct.ncomp)

    def mod_drop(self, ct, L):
        return FakeCt(L, ct.scale, ct.ncomp)

    def scale_mul(self, ct, f):
        return ct

    def mac_ptmul(self, cts, pts):
        self.ledger["ptmul"] += len(cts)
        return FakeCt(cts[0].L, 1.0)

    def mask_ext(self, desc, L, m=None):
        return FakeCt(L, 1.0, 1)

    def mask_scale(self, L):
        return 1.0

    def rot_hoisted_ext(self, ct, rs):
        return self.rot_hoisted(ct, rs)

    def ext_masked_sum(self, xs, pts, scale):
        self.ledger["ptmul"] += len(xs)
        return FakeCt(xs[0].L, scale)

    def moddown_rescale(self, y):
        self.ledger["moddown"] += 1
        self.ledger["rescale"] += 1
        return FakeCt(y.L - 1, y.scale)

    def relin_rescale(self, ct):
        self.ledger["relin"] += 1
        return self.moddown_rescale(FakeCt(ct.L, ct.scale))

    def lift_ext(self, ct):
        return FakeCt(ct.L, ct.scale)

    def rot_ext(self, ct, r):
        if int(r) % self.n:
            self.ledger["rot"] += 1
        return FakeCt(ct.L, ct.scale)

    def conj_ext(self, ct):
        self.ledger["conj"] += 1
        return FakeCt(ct.L, ct.scale)

    def ext_add(self, a, b):
        return FakeCt(a.L, a.scale)

    def moddown(self, y):
        self.ledger["moddown"] += 1
        return FakeCt(y.L, y.scale)

    def tensor_sum(self, pairs):
        for _ in pairs:
            self.ledger["ctmul"] += 1
        return FakeCt(pairs[0][0].L, 1.0, 3)


# ====================================================================================== shifts (App. A.1)
def Phi(ev, x, delta, m):
    """Phi^Delta = rot(x; Delta m)  (Alg A.1)."""
    return ev.rot(x, delta * m)


def Psi_hoisted(ev, x, ts, m, N_seg, seg0=0, nseg=None):
    """Psi^t for every t in ts from ONE hoisted ModUp of x (Alg A.2):
       Psi^t(x) = rot(x; t)(.)h_t + rot(x; (t-m) mod n)(.)u_t, then rescale.
    The two rotations stay in the extended basis Q_L u P (no ModDown), are masked there and then
    divided by P q_{L-1} at once (lazy ModDown merged with the rescale, DESIGN.md R-LAZY).
    t = 0 (mod m) is realised as x(.)h_0 then rescale (no rotation), so every bank entry sits at the
    same level and scale (reading R-PSI0).  Optional segment restriction merges a trailing
    segment mask (used by the score align step)."""
    L = x.L
    tt = [int(t) % m for t in ts]
    steps = []
    for t in tt:
        if t:
            steps += [t, t - m]
    rots = ev.rot_hoisted_ext(x, steps) if steps else []
    out, i = [], 0
    for t in tt:
        hd, ud = psi_masks(t, m, N_seg, seg0, nseg)
        if t == 0:
            out.append(ev.rescale(ev.ptmul(x, ev.mask(hd, L, m))))
        else:
            y = ev.ext_masked_sum([rots[i], rots[i + 1]], [ev.mask_ext(hd, L, m), ev.mask_ext(ud, L, m)], x.scale * ev.mask_scale(L))
            out.append(ev.moddown_rescale(y))
            i += 2
    return out


def slot_range_desc(lo, hi, m):
    """Mask descriptor + row grid of the slot range [lo, hi): the m-row grid when the range is segment
    aligned, else the 1-row grid (every slot its own 'segment')."""
    if lo % m == 0 and hi % m == 0:
        return (0, m, lo // m, 1, (hi - lo) // m), m
    return (0, 1, lo, 1, hi - lo), 1


def rotfirst_masks(Ls, tau, m):
    """a_{L,tau} = 1{0 <= i < L - tau}, b_{L,tau} = 1{L - tau <= i < L}  (Alg A.3 line 2), as
    (descriptor, grid) pairs; b is None for tau = 0."""
    a = slot_range_desc(0, Ls - tau, m)
    b = slot_range_desc(Ls - tau, Ls, m) if tau else None
    return a, b


def rotfirst_reference(x, Ls, tau):
    """Slot-level definition of RotFirst_L(x; tau) (Alg A.3 Ensure, with G21: slots >= L come out zero):
    out[i] = x[(i + tau) mod L] for i < L, 0 otherwise."""
    x = np.asarray(x)
    out = np.zeros_like(x)
    idx = (np.arange(Ls) + tau) % Ls
    out[:Ls] = x[idx]
    return out


def RotFirst_hoisted(ev, x, Ls, taus, m):
    """RotFirst_L(x; tau) for every tau in taus from ONE hoisted ModUp of x (Alg A.3):
        tau <- tau mod L;  y1 = rot(x; tau) (.) a_{L,tau};  y2 = rot(x; (tau - L) mod n) (.) b_{L,tau};  y1 + y2,
    then rescale (the masks are plaintexts at scale q_{L-1}, DESIGN.md R-MASK).  As for Psi (R-LAZY) the two
    rotations stay in Q_L u P, are masked there and divided by P q_{L-1} at once.  tau = 0 is x (.) a_{L,0}
    then rescale (Alg A.3 with rot(x; 0) and an empty b; no key switch), so every output shares one level."""
    L = x.L
    tt = [int(t) % Ls for t in taus]
    steps = []
    for t in tt:
        if t:
            steps += [t, t - Ls]
    rots = ev.rot_hoisted_ext(x, steps) if steps else []
    out, i = [], 0
    for t in tt:
        (ad, am), bb = rotfirst_masks(Ls, t, m)
        if t == 0:
            out.append(ev.rescale(ev.ptmul(x, ev.mask(ad, L, am))))
        else:
            bd, bm = bb
            y = ev.ext_masked_sum([rots[i], rots[i + 1]], [ev.mask_ext(ad, L, am), ev.mask_ext(bd, L, bm)],
                                  x.scale * ev.mask_scale(L))
            out.append(ev.moddown_rescale(y))
            i += 2
    return out


def rotfirst_ext(ev, c, Ls, tau, m):
    """RotFirst_L(c; tau) BEFORE its ModDown and rescale: the extended-basis masked pair
    rot_ext(c, tau) (.) a + rot_ext(c, tau - L) (.) b (both rotations from one hoisted ModUp; tau = 0: P c (.) a).
    Its moddown_rescale is RotFirst_hoisted(c, [tau]); sums of such terms are ModDown'ed once (R-LAZY)."""
    L = c.L
    tau = int(tau) % Ls
    (ad, am), bb = rotfirst_masks(Ls, tau, m)
    sc = c.scale * ev.mask_scale(L)
    if tau == 0:
        return ev.ext_masked_sum([ev.lift_ext(c)], [ev.mask_ext(ad, L, am)], sc)
    r = ev.rot_hoisted_ext(c, [tau, tau - Ls])
    bd, bm = bb
    return ev.ext_masked_sum(r, [ev.mask_ext(ad, L, am), ev.mask_ext(bd, L, bm)], sc)


def Phi_C(ev, x, deltas, C, m, N_seg):
    """Phi_C^Delta (Alg A.4): C <- min(C, N_seg), Delta <- Delta mod C, RotFirst_{Cm}(x; Delta m);
    one hoisted batch over deltas."""
    C = min(C, N_seg)
    return RotFirst_hoisted(ev, x, C * m, [(int(d) % C) * m for d in deltas], m)


def Align(ev, x, H, r, m):
    """Block phase correction Align_r(x) = RotFirst_{Hm}(x, (H - r) m)  (App. A.3)."""
    return RotFirst_hoisted(ev, x, H * m, [(H - r) * m], m)[0]


# ====================================================================================== projection (§3.2, App. A.2)
class ProjPlan:
    """Plan of the shared pt-ct projection Y = X W.
    C = active segments (default N_seg, G4), N1 | C (G5), N2 = C/N1, G = ceil(d_in/C),
    U = ceil(G/2) complexified inputs, B_out = ceil(d_out/C)."""

    def __init__(self, n, m, d_in, d_out, C=None, N1=None, real_input=False):
        self.n, self.m, self.d_in, self.d_out = n, m, d_in, d_out
        self.N_seg = n // m
        self.C = C or self.N_seg
        self.G = -(-d_in // self.C)
        self.real_input = real_input          # fused QK: real inputs, complex weights (G1)
        self.U = self.G if real_input else -(-self.G // 2)
        self.B_out = -(-d_out // self.C)
        if self.C > self.N_seg:
            raise O.OracleError("PLAN_SHAPE: C > n/m")
        if N1 is None:
            N1 = default_n1(self.C, self.B_out, self.U)
        assert self.C % N1 == 0
        self.N1, self.N2 = N1, self.C // N1
        # C < N_seg: the segment shifts wrap modulo the C active segments (Phi_C = RotFirst_{Cm}, Alg A.4); the
        # bank and the giant fold each spend one level (masks), so y_b lands 3 levels below x (reading R-PHIC)
        self.restricted = self.C < self.N_seg

    def weight_level(self, L):
        """Level of the weight plaintexts for inputs at level L (the bank's level)."""
        return L - 1 if self.restricted else L

    def out_levels(self):
        """Levels the projection consumes (input level - output level)."""
        return 3 if self.restricted else 1


def default_n1(C, B_out, U):
    """Power of two dividing C nearest sqrt(B_out*C/U) (minimises key switches)."""
    import math
    target = math.sqrt(B_out * C / U)
    best = 1
    p = 1
    while p <= C:
        if C % p == 0 and abs(math.log2(p) - math.log2(target)) < abs(math.log2(best) - math.log2(target)) - 1e-12:
            best = p
        p *= 2
    return best


def proj_inputs(X, plan):
    """Complexified inputs x~_u = x^(2u) + i x^(2u+1) as slot vectors (real inputs x^(g) for a
    fused-QK plan)."""
    if plan.real_input:
        return [seg_column_pack(X, plan.m, plan.C, g, plan.n) for g in range(plan.U)]
    return [seg_column_pack(X, plan.m, plan.C, 2 * u, plan.n) + 1j * seg_column_pack(X, plan.m, plan.C, 2 * u + 1, plan.n)
            for u in range(plan.U)]


def proj_weight_slots_fused(Wre, Wim, plan, b, p, g, q):
    """Fused-QK weights: w~(c) = Wre[gC + alpha, bC + beta] + i Wim[gC + alpha, bC + beta] so that
    sum_{g,q} Phi^q(x^(g)) (.) w~ folds to X Wre + i X Wim (real part Q, imaginary part K for Wre = W_Q^pi_S,
    Wim = W_K^pi_S)."""
    C, m = plan.C, plan.m
    d_in, d_out = Wre.shape
    z = np.zeros(plan.n, dtype=np.complex128)
    for c in range(C):
        a = (c + q) % C
        be = (c - p * plan.N1) % C
        col, r = b * C + be, g * C + a
        if col < d_out and r < d_in:
            z[c * m:(c + 1) * m] = Wre[r, col] + 1j * Wim[r, col]
    return z


def proj_weight_slots(Wbar, plan, b, p, u, q):
    """w~^(b)_{u,p,q}(c) = Wbar[(2u)C + alpha, bC + beta] - i Wbar[(2u+1)C + alpha, bC + beta],
    alpha = (c+q) mod C, beta = (c - p N1) mod C; constant over the m rows of segment c; zero for
    c >= C and outside d_in x d_out."""
    C, m = plan.C, plan.m
    d_in, d_out = Wbar.shape
    z = np.zeros(plan.n, dtype=np.complex128)
    for c in range(C):
        a = (c + q) % C
        be = (c - p * plan.N1) % C
        col = b * C + be
        if col >= d_out:
            continue
        r0, r1 = (2 * u) * C + a, (2 * u + 1) * C + a
        w = (Wbar[r0, col] if r0 < d_in else 0.0) - 1j * (Wbar[r1, col] if r1 < d_in else 0.0)
        z[c * m:(c + 1) * m] = w
    return z


def proj_weight_index(plan, b, p, u, q):
    """Flat index of plaintext (b,p,u,q) in the [b][p][u][q] weight stream (the ABI layout)."""
    return ((b * plan.N2 + p) * plan.U + u) * plan.N1 + q


def projection_partial(ev, plan, xt, w, u0, u1):
    """C6 steps 1-3 restricted to the giant-step units [u0, u1) (row-major over (b, p)): the bank is
    built in full, c~_{b,p} and acc_b = sum over the range's p of rot(c~_{b,p}, p N1 m) (p = 0 unrotated).
    Returns {b: acc_b}.  Used to pin the multi-rank partition."""
    m, N1 = plan.m, plan.N1
    bank = []
    for u in range(plan.U):
        if plan.restricted:                     # bank[u][q] = Phi_C^q(x~_u) (Alg A.4), one level
            bank.append(Phi_C(ev, xt[u], list(range(N1)), plan.C, m, plan.N_seg))
            continue
        rots = ev.rot_hoisted(xt[u], [q * m for q in range(1, N1)]) if N1 > 1 else []
        bank.append([xt[u]] + list(rots))
    accs = {}
    for un in range(u0, u1):
        b, p = divmod(un, plan.N2)
        cts = [bank[u][q] for u in range(plan.U) for q in range(N1)]
        pts = [w(b, p, u, q) for u in range(plan.U) for q in range(N1)]
        c = ev.mac_ptmul(cts, pts)
        if plan.restricted:                     # Phi_C^{p N1}(c~_{b,p}) = RotFirst_{Cm}(c; p N1 m), masked in Q_L u P
            e = rotfirst_ext(ev, c, plan.C * m, p * N1 * m, m)
        else:
            e = ev.rot_ext(c, p * N1 * m)      # p = 0: P * c (exact lift); p >= 1: rotation without ModDown (R-LAZY)
        accs[b] = e if b not in accs else ev.ext_add(accs[b], e)
    return accs                                 # extended-basis partial accumulators (reduced across ranks as such)


def projection_finalize(ev, plan, acc_ext, decomplexify=True):
    """C6 steps 4-5 on an extended accumulator: acc = ModDown(acc_ext) (one per block, R-LAZY);
    z = acc + conj(acc) (scale x2, G2/G3) formed in Q_L u P and divided by P q_{L-1} at once."""
    acc = ev.moddown_rescale(acc_ext) if plan.restricted else ev.moddown(acc_ext)   # restricted: fold masks' level
    if decomplexify:
        z = ev.ext_add(ev.lift_ext(acc), ev.conj_ext(acc))
        z.scale = acc.scale * 2.0
        return ev.moddown_rescale(z)
    return ev.rescale(acc)


def projection(ev, plan, xt, w, decomplexify=True):
    """C6 (G2/G3):
      1. bank[u][0] = x~_u ; bank[u][q] = HOISTED rot(x~_u, q m), q = 1..N1-1
      2. c~_{b,p} = sum_{u,q} bank[u][q] (.) w~_{b,p,u,q}          (exact modular sum)
      3. acc_b = c~_{b,0} + sum_{p>=1} rot(c~_{b,p}, p N1 m)       (single rotations, summed in Q_L u P and
         ModDown'ed once per block: lazy ModDown, R-LAZY)
      4. z_b = acc_b + conj(acc_b), scale x2  (decomplexify AFTER the fold, G2; the 1/2 is bookkeeping, G3)
      5. y_b = rescale(z_b)                    (4-5 merged: conj kept in Q_L u P, one division by P q_{L-1})
    w(b, p, u, q) -> plaintext.  Returns the B_out outputs y_b."""
    accs = projection_partial(ev, plan, xt, w, 0, plan.B_out * plan.N2)
    return [projection_finalize(ev, plan, accs[b], decomplexify) for b in range(plan.B_out)]


# ====================================================================================== score kernel (§3.3.1, App. A.3)
class ScorePlan:
    """Score kernel plan.  C_qk used segments per block (multiple of H with
    C_qk/H a power of two -> routing tree; G8 padding), beta | m, g = m/beta even."""

    def __init__(self, n, m, H, d_h, C_qk=None, beta=None):
        if m % 2:
            raise O.OracleError("ODD_SEQ")
        self.n, self.m, self.H, self.d_h = n, m, H, d_h
        self.N_seg = n // m
        if C_qk is None:
            C_qk = H
            while C_qk * 2 <= self.N_seg and C_qk < H * d_h:
                C_qk *= 2
        self.C = C_qk
        if not (H <= C_qk <= self.N_seg):
            raise O.OracleError("PLAN_SHAPE: need H <= C_qk <= n/m")
        self.B = -(-(H * d_h) // C_qk)
        # head phase of block l: r_l = l C mod H (App. A.3); C mod H != 0 -> Align_r per phase group
        self.phases = [(l * C_qk) % H for l in range(self.B)]
        self.aligned = any(self.phases)
        self.k_route = -(-C_qk // H)                 # channel groups folded onto the H head segments
        self.beta = beta or default_beta(m)
        self.g = m // self.beta
        assert m % self.beta == 0 and self.g % 2 == 0
        self.n_out = k_min(H * m * m, n)


def default_beta(m):
    b = 1
    while b * b < m:
        b *= 2
    return b


def score_qk_slots(Qp, plan, l):
    """Block l of Q^{pi_S} (or K^{pi_S}) in segment-column packing: segment c holds column l C_qk + c."""
    return seg_column_pack(Qp, plan.m, plan.C, l, plan.n)


def score(ev, plan, qs, ks, ts=None, route_hoisted=True):
    """C7.  Per block l: Q bank Psi^{-s} (s < beta), K bank Psi^{j beta}, Psi^{m/2 + j beta} (j < g/2),
    all hoisted from one ModUp each.  Per t = j beta + s < m/2:
      T_t = sum_l q_{-s} (x) (k_{j beta} + i k_{m/2 + j beta})   lazy tensor sum, ONE relin, rescale (G6)
      route: sum_{j < C/H} Phi^{jH}(x)  (Phi^{c - (c mod H)}, G7; hoisted sum R-ROUTE, or the paper's tree)
      S_t = Psi^{s}(route) restricted to segments [0, H)  (align + e_[0,H) mask merged, one rescale)
    Returns [S_0 .. S_{m/2-1}]."""
    m, H, beta, g, N_seg = plan.m, plan.H, plan.beta, plan.g, plan.N_seg
    qb, kb = [], []
    for l in range(plan.B):
        qb.append(Psi_hoisted(ev, qs[l], [-s for s in range(beta)], m, N_seg))
        kt = [j * beta for j in range(g // 2)] + [m // 2 + j * beta for j in range(g // 2)]
        kk = Psi_hoisted(ev, ks[l], kt, m, N_seg)
        kb.append({t: c for t, c in zip(kt, kk)})
    S = []
    groups = score_phase_groups(plan)
    for t in (range(m // 2) if ts is None else ts):
        j, s = t // beta, t % beta
        routed = {}
        for r, ls in groups.items():          # one lazy tensor sum per head phase (all blocks when C mod H = 0)
            pairs = [(qb[l][s], ev.add(kb[l][j * beta], ev.mul_i(kb[l][m // 2 + j * beta]))) for l in ls]
            T = ev.relin_rescale(ev.tensor_sum(pairs))          # lazy relin merged with the rescale (R-RELRS)
            routed[r] = route(ev, T, plan.k_route, H, m, hoisted=route_hoisted)
        if plan.aligned:
            T = align_sum(ev, routed, H, m)
        else:
            T = routed[0]
        S.append(Psi_hoisted(ev, T, [s], m, N_seg, 0, H)[0])
    return S


def score_phase_groups(plan):
    """{r: [blocks l with l C mod H = r]} (App. A.3 "We sum score contributions by phase")."""
    groups = {}
    for l, r in enumerate(plan.phases):
        groups.setdefault(r, []).append(l)
    return groups


def align_sum(ev, routed, H, m):
    """sum_r Align_r(x_r) = sum_r RotFirst_{Hm}(x_r, (H - r) m)  (applied before combining phases):
    every Align_r kept in Q_L u P (rotfirst_ext; r = 0 is the mask a_{Hm,0} alone), the phase terms summed there
    and divided by P q_{L-1} ONCE (R-LAZY)."""
    acc = None
    for r in sorted(routed):
        e = rotfirst_ext(ev, routed[r], H * m, (H - r) * m, m)
        acc = e if acc is None else ev.ext_add(acc, e)
    return ev.moddown_rescale(acc)


def route(ev, x, k, H, m, hoisted=True):
    """Fold segment c onto c mod H: out[h] = sum_{j<k} x[h + jH] (the paper's sum_c Phi^{c - (c mod H)}
    (x (.) m_c) with the sign of P:397 corrected, G7).  Segments >= H hold garbage and are masked by the
    caller.
    hoisted=True (the build's schedule, DESIGN.md R-ROUTE): the k-1 shifts Phi^{jH} (j = 1..k-1) of the SAME
    x from ONE hoisted ModUp, kept in the extended basis, summed with P x and ModDown'ed ONCE:
        out = ModDown(P x + sum_{j=1}^{k-1} rot_ext(x, j H m)).
    hoisted=False (the paper's schedule): a binary rotate-add, O(log k) sequential single rotations (the
    m log C term of #rot_S)."""
    if hoisted:
        if k == 1:
            return x
        acc = ev.lift_ext(x)
        for r in ev.rot_hoisted_ext(x, [j * H * m for j in range(1, k)]):
            acc = ev.ext_add(acc, r)
        return ev.moddown(acc)
    result, offset, cnt, pw = None, 0, 1, x
    kk = k
    while kk:
        if kk & 1:
            y = Phi(ev, pw, offset * H, m) if offset else pw
            result = y if result is None else ev.add(result, y)
            offset += cnt
        kk >>= 1
        if kk:
            pw = ev.add(pw, Phi(ev, pw, cnt * H, m))
            cnt *= 2
    return result


def score_export(ev, plan, S):
    """Minimal export stream (A20; t-major order S:181): stream slot (t H + h) m + j
    -> ciphertext floor(./n), slot (. mod n).  S_t is rotated right by its offset o (single KS) and
    masked by the slot range(s) it covers in each ciphertext (straddling pieces split by masks; the
    tail is zero).  The rotations are consumed only by these masked sums, so they stay in the extended
    basis Q_L u P (no ModDown; t with o = 0 enters as P S_t) and every output ciphertext is divided by
    P q_{L-1} at once (lazy ModDown merged with the rescale, DESIGN.md R-LAZY / R-EXP).  Returns K_min(S)
    ciphertexts."""
    m, H, n = plan.m, plan.H, plan.n
    seg = H * m
    terms = [[] for _ in range(plan.n_out)]
    for t, st in enumerate(S):
        start = t * seg
        o = start % n
        r = ev.rot_ext(st, -o) if o else ev.lift_ext(st)
        k = start // n
        first = min(seg, n - o)
        pieces = [(k, o, o + first)]
        if first < seg:
            pieces.append((k + 1, 0, seg - first))
        for (ci, a, b) in pieces:
            desc = (0, m, a // m, 1, (b - a) // m)
            terms[ci].append((r, ev.mask_ext(desc, r.L, m)))
    L = S[0].L
    sc = S[0].scale * ev.mask_scale(L)
    return [ev.moddown_rescale(ev.ext_masked_sum([x for x, _ in tt], [p for _, p in tt], sc)) for tt in terms]


def score_reference(Qh, Kh):
    """Brute force: S^h = Q^h (K^h)^T; Re S_t[h m + j] = S^h[j, (j+t) mod m], Im = S^h[j, (j+t+m/2) mod m]."""
    H, m, _ = Qh.shape
    S = np.einsum("hid,hjd->hij", Qh, Kh)
    out = []
    for t in range(m // 2):
        v = np.zeros(H * m, dtype=np.complex128)
        for h in range(H):
            for jj in range(m):
                v[h * m + jj] = S[h, jj, (jj + t) % m] + 1j * S[h, jj, (jj + t + m // 2) % m]
        out.append(v)
    return out


# ====================================================================================== value kernel (§3.3.2, App. A.3)
class ValuePlan:
    """Value kernel plan: head-major V, folded-diagonal P_fd; needs d_h = m/2
    for the folded stream to reshape directly; otherwise H_blk = 1 (G10)."""

    def __init__(self, n, m, H, d_h, H_blk=None):
        if m % 2:
            raise O.OracleError("ODD_SEQ")
        self.n, self.m, self.H, self.d_h = n, m, H, d_h
        self.N_seg = n // m
        if H_blk is None:
            H_blk = self.N_seg // d_h if d_h == m // 2 else 1
        assert H_blk * max(d_h, m // 2) <= self.N_seg
        self.H_blk = H_blk
        self.B_V = -(-H // H_blk)
        self.seg_stride = max(d_h, m // 2)   # segments per local head


def value_v_slots(Vh, plan, l):
    """Head-major V block l: segment h~ d_h + u holds V^(l H_blk + h~)[:, u]."""
    n, m = plan.n, plan.m
    z = np.zeros(n, dtype=np.complex128)
    for hh in range(plan.H_blk):
        h = l * plan.H_blk + hh
        if h >= plan.H:
            continue
        for u in range(plan.d_h):
            s = hh * plan.seg_stride + u
            z[s * m:(s + 1) * m] = Vh[h][:, u]
    return z


def value_p_slots(Ph, plan, l):
    """Folded-diagonal P_fd block l: segment h~ (m/2) + t holds p_t + i p_{t+m/2} of local head h~,
    p_t[j] = P[j, (j+t) mod m]."""
    n, m = plan.n, plan.m
    z = np.zeros(n, dtype=np.complex128)
    jj = np.arange(m)
    for hh in range(plan.H_blk):
        h = l * plan.H_blk + hh
        if h >= plan.H:
            continue
        for t in range(m // 2):
            s = hh * plan.seg_stride + t
            z[s * m:(s + 1) * m] = Ph[h][jj, (jj + t) % m] + 1j * Ph[h][jj, (jj + t + m // 2) % m]
    return z


def value_partial(ev, plan, ps, vs, u0, u1):
    """C8 steps 1-5 for the units (l, t), flattened l (m/2) + t, in [u0, u1) -- the multi-GPU partition of the
    value kernel: {l: o3_l} with o3_l = sum over the range's t of u_t (x) b_t, UNRELINEARISED.  Every
    object of a unit (u_t, the Phi-bank rotations Phi^{t-u}(p), b_t) has the same bits as in the full kernel (each
    hoisted rotation depends only on its input and offset), so summing the partials of a block over a partition of
    its t (exact modular sum) gives the full kernel's relinearisation input.
      1. uu = v (.) e_all - i (rot(v, m/2)(.)h_{m/2} + rot(v, -m/2)(.)u_{m/2}), ONE rescale
      2. U bank: u_t = Psi^{t}(uu) (hoisted; G9: +t)
      3. Phi bank of p_fd: delta in [t_lo - (d_h - 1), t_hi - 1] (hoisted single rotations by delta m)
      4. b_t = sum_u Phi^{t-u}(p_fd) (.) n_u, rescale
      5. sum_t u_t (x) b_t (u_t mod-dropped to b_t's level)"""
    m, N_seg = plan.m, plan.N_seg
    half = m // 2
    out = {}
    for l in range(plan.B_V):
        ta, tb = max(u0 - l * half, 0), min(u1 - l * half, half)
        if ta >= tb:
            continue
        v, p = vs[l], ps[l]
        Lv = v.L
        rv = ev.rot_hoisted(v, [half, half - m])
        hd, ud = psi_masks(half, m, N_seg)
        sh = ev.add(ev.ptmul(rv[0], ev.mask(hd, Lv, m)), ev.ptmul(rv[1], ev.mask(ud, Lv, m)))
        uu = ev.rescale(ev.sub(ev.ptmul(v, ev.mask((0, m, 0, 1, N_seg), Lv, m)), ev.mul_i(sh)))
        ub = dict(zip(range(ta, tb), Psi_hoisted(ev, uu, list(range(ta, tb)), m, N_seg)))
        deltas = [d for d in range(ta - (plan.d_h - 1), tb) if d != 0]
        pb = dict(zip(deltas, ev.rot_hoisted(p, [d * m for d in deltas])))
        pb[0] = p
        Lp = p.L
        pairs = []
        for t in range(ta, tb):
            cts = [pb[t - u] for u in range(plan.d_h)]
            pts = [ev.mask((0, m, u, plan.seg_stride, plan.H_blk), Lp, m) for u in range(plan.d_h)]
            bt = ev.rescale(ev.mac_ptmul(cts, pts))     # sum_u Phi^{t-u}(p) (.) n_u (exact modular sum)
            pairs.append((ev.mod_drop(ub[t], bt.L) if ub[t].L > bt.L else ub[t], bt))
        out[l] = ev.tensor_sum(pairs)
    return out


def value(ev, plan, ps, vs, blocks=None):
    """C8 (P:425-455 with G9: u_t = Psi^{+t} u): value_partial over every unit of the requested blocks, then
    o = ONE relin merged with the rescale (R-RELRS) per block."""
    half = plan.m // 2
    outs = []
    for l in (range(plan.B_V) if blocks is None else blocks):
        o3 = value_partial(ev, plan, ps, vs, l * half, (l + 1) * half)[l]
        outs.append(ev.relin_rescale(o3))          # lazy relin merged with the rescale (R-RELRS)
    return outs


def value_reference(Ph, Vh):
    return np.einsum("hij,hjd->hid", Ph, Vh)


# ====================================================================================== export (Alg 3, GPU half)
def l_conv(P, ell=43, sigma=40, scale=None, B_max=1.0):
    """Modulus trimming: smallest L with log2 Q_L >= ell + sigma + 1 and Q_L/2 > Delta B_max.
    ell = 43, sigma = 40 (G19).  Returns None if no level satisfies it (ENCF_ERR_CONFIG)."""
    import math
    scale = scale if scale is not None else 2.0 ** P.log2_scale
    Q = 1
    for L in range(1, P.L_max + 1):
        Q *= P.q[L - 1]
        if math.log2(Q) >= ell + sigma + 1 and Q / 2 > scale * B_max:
            return L
    return None


def export_c2m(P, ct, L_conv, mask_seed, stream_id):
    """Alg 3 steps 1 (P1 side) with trimming (C9):
      mod-drop to L_conv; r^ uniform mod q_i per limb (coefficient domain, G18) from
      stream mask(stream_id); d = (c0 + r^, c1) goes to P0; the server share is -r^ mod q_i.
    Returns (masked ciphertext, server share [L_conv][N])."""
    if ct.ncomp != 2:
        raise O.OracleError("FORMAT")
    d = O.mod_drop(P, ct, L_conv)
    mods = P.q[:L_conv]
    r = O.sample_uniform(mask_seed, O.stream_mask(stream_id), mods, list(range(L_conv)), P.N)
    c0 = O.padd(d.c[0], r, mods, P.N)
    share = O.pneg(r, mods, P.N)
    return O.Ct(np.stack([c0, d.c[1]]), ct.scale), share


# ====================================================================================== conversions (App. C, Alg 4)
def ring2field_local(P, mprime, party, ell_sigma, L):
    """Ring2Field local map: party 0: m'_0 mod q; party 1: (m'_1 - 2^{ell+sigma}) mod q, per limb
    of Q_L (Python integers in, coefficient-form residues out)."""
    off = (1 << ell_sigma) if party else 0
    return np.stack([np.array([(int(v) - off) % q for v in mprime], dtype=np.uint64) for q in P.q[:L]])


def field2ring_local(share, ell):
    """Field2Ring local map: reduce the lifted share modulo 2^ell."""
    return np.array([int(v) % (1 << ell) for v in share], dtype=np.uint64)


def import_m2c(P, ct, share_pt):
    """Alg 4 step 4: <m> = <c> + [[t^]]_1 (plaintext share added to c0)."""
    mods = P.q[:ct.L]
    return O.Ct(np.stack([O.padd(ct.c[0], share_pt.m, mods, P.N), ct.c[1]]), ct.scale)


# ====================================================================================== GELU pre-evaluation (NEXT row 2)
def gelu_exact(x):
    import math
    return np.array([0.5 * v * (1.0 + math.erf(v / math.sqrt(2.0))) for v in np.asarray(x, dtype=float).ravel()])


def gelu_fit():
    """Coefficients (a, b, c, d, e) of ApproxGELU's mid-range branch a|x|^4 + b|x|^3 + c|x|^2 + d|x| + e + 0.5x
    (Eq. B.1).  The paper uses BOLT's coefficients without printing them; reading R-GELU
    (SPEC's decision): the least-squares quartic in |x| fitted to GELU(x) - 0.5x on [0, 2.7] (2701
    points, numpy lstsq), frozen by this function."""
    t = np.linspace(0.0, 2.7, 2701)
    target = gelu_exact(t) - 0.5 * t
    A = np.stack([t ** 4, t ** 3, t ** 2, t, np.ones_like(t)], axis=1)
    coef, *_ = np.linalg.lstsq(A, target, rcond=None)
    return tuple(float(v) for v in coef)


def approx_gelu(x, coef):
    """Eq. B.1 in float64 (pass-through above 2.7, zero below -2.7, quartic in |x| plus 0.5x inside)."""
    a, b, c, d, e = coef
    x = np.asarray(x, dtype=float)
    ax = np.abs(x)
    mid = a * ax ** 4 + b * ax ** 3 + c * ax ** 2 + d * ax + e + 0.5 * x
    return np.where(x > 2.7, x, np.where(x < -2.7, 0.0, mid))


def const_mul_rescale(ev, ct, c, target):
    """ct x (public constant c), then rescale: c enters as the INTEGER k = round_half_even(c * Delta) on every
    coefficient (a constant plaintext at scale Delta = target q_{L-1} / scale), so the rescaled result
    carries the tracked scale `target` (set exactly; the true scale differs by |k - c Delta| / (c Delta),
    below 2^-30 here; reading R-GELU)."""
    L, N = ct.L, ev.P.N
    delta = target * float(ev.P.q[L - 1]) / ct.scale
    k = int(round(c * delta))
    mods = ev.P.q[:L]
    cc = np.stack([O.pmul_scalar(ct.c[i], [k % q for q in mods], mods, N) for i in range(ct.ncomp)])
    ev.ledger["ptmul"] += 1
    y = ev.rescale(O.Ct(cc, ct.scale))
    return O.Ct(y.c, target)


def add_const(ev, ct, e):
    """ct + e (public constant): E = round_half_even(e * scale) added to the constant coefficient of c0."""
    L = ct.L
    E = int(round(e * ct.scale))
    c = ct.c.copy()
    for i, q in enumerate(ev.P.q[:L]):
        c[0][i][0] = np.uint64((int(c[0][i][0]) + E) % q)
    return O.Ct(c, ct.scale)


def gelu_preeval(ev, x, coef):
    """Alg 5 steps 1-3, the CKKS half of secure GELU with pre-evaluation.
       1. x^(0) = (x + conj x)/2, x^(1) = (x - conj x)/(2i) = i (conj x - x)/2   (the 1/2 is scale bookkeeping, G3)
       2. per j: x^2, x^3 = x^2 x, x^4 = x^2 x^2 (each one tensor + relin + rescale), then
          F0 = a x^4 - b x^3 + c x^2 + (0.5 - d) x + e,  F1 = a x^4 + b x^3 + c x^2 + (0.5 + d) x + e  (Eq. B.2)
          with every term brought to level L-3 and one common scale (const_mul_rescale / mod_drop)
       3. F0^C = F0^(0) + i F0^(1), F1^C = F1^(0) + i F1^(1)   (i = X^{N/2}, exact)
    Input: complex x at level L >= 4.  Returns (F0^C, F1^C) at level L-3."""
    a, b, c, d, e = coef
    L = x.L
    xc = ev.conj(x)
    xs = [ev.scale_mul(ev.add(x, xc), 2.0), ev.scale_mul(ev.mul_i(ev.sub(xc, x)), 2.0)]
    F0, F1 = [], []
    for xj in xs:
        T = xj.scale
        x2 = ev.rescale(ev.relin(ev.tensor(xj, xj)))
        x3 = ev.rescale(ev.relin(ev.tensor(x2, ev.mod_drop(xj, L - 1))))
        x4 = ev.rescale(ev.relin(ev.tensor(x2, x2)))
        A = const_mul_rescale(ev, x4, a, T)
        B = const_mul_rescale(ev, x3, b, T)
        C = ev.mod_drop(const_mul_rescale(ev, x2, c, T), L - 3)
        D0 = ev.mod_drop(const_mul_rescale(ev, xj, 0.5 - d, T), L - 3)
        D1 = ev.mod_drop(const_mul_rescale(ev, xj, 0.5 + d, T), L - 3)
        base = ev.add(A, C)
        F0.append(add_const(ev, ev.add(ev.sub(base, B), D0), e))
        F1.append(add_const(ev, ev.add(ev.add(base, B), D1), e))
    return ev.add(F0[0], ev.mul_i(F0[1])), ev.add(F1[0], ev.mul_i(F1[1]))


# ====================================================================================== w/o-SCP ablation (NEXT row 3)
def rma_bands(m):
    """Row bands of the RMA masks: log2 m contiguous bands of the m rows of every segment; band k is moved
    by the rotation 2^k (reading R-RMA: App. G gives only the RMA form)."""
    K = int(np.log2(m))
    edges = [round(k * m / K) for k in range(K + 1)]
    return [(edges[k], edges[k + 1]) for k in range(K)]


def repack_rma(ev, x, m):
    """Halevi-Shoup rotation-mask-accumulate repack of the w/o-SCP ablation (App. G):
        Repack(v) = sum_{k < log2 m} Rot(v, 2^k) (.) m_k
    with m_k = the rows of band k (rma_bands) in every segment, i.e. out[s m + j] = v[s m + j + 2^{k(j)}].
    log2 m rotations from ONE hoisted ModUp, kept in the extended basis, masked and summed there, ONE merged
    ModDown + rescale (R-LAZY)."""
    K = int(np.log2(m))
    nseg = ev.P.n // m
    rots = ev.rot_hoisted_ext(x, [1 << k for k in range(K)])
    masks = [ev.mask_ext((r0, r1, 0, 1, nseg), x.L, m) for (r0, r1) in rma_bands(m)]
    return ev.moddown_rescale(ev.ext_masked_sum(rots, masks, x.scale * ev.mask_scale(x.L)))


def repack_rma_reference(v, m):
    """The slot map the RMA repack realises (brute force): out[i] = v[(i + 2^{k(i mod m)}) mod n]."""
    n = len(v)
    out = np.empty_like(v)
    band = np.empty(m, dtype=int)
    for k, (r0, r1) in enumerate(rma_bands(m)):
        band[r0:r1] = k
    for i in range(n):
        out[i] = v[(i + (1 << band[i % m])) % n]
    return out
