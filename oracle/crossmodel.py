"""Tiny pure-Python big-integer CKKS model (SURVEY.md §8c C11 "Tiny cross-model"): an INDEPENDENT
implementation of the oracle's arithmetic at N = 16..32, written from DESIGN.md's spec (PRNG streams, sampling,
hybrid key switching, rounded ModDown, SEAL rescale, merged ModDown + rescale) rather than from oracle.c.

TEST INFRASTRUCTURE ONLY (see oracle/ckks.py header).

Nothing here uses numpy arithmetic, the oracle's C library or its NTT: ring products are schoolbook negacyclic
convolutions on Python ints, the rescale is floor((x + q/2) / q) of the explicit CRT value x, ModDown and the
merged ModDown + rescale form the selected representative y of x mod B as ONE big integer (HPS rounding rule of
DESIGN.md R-MODDOWN, whose agreement with exact rounding is pinned separately), and the PRNG is SplitMix64
re-typed in Python.  The
only shared input is DATA: the parameter JSON and the float64 encodings of masks / weights (bit parity is defined
on integer data).  tests/test_crossmodel.py checks that this model and oracle/ckks.py + kernels.py
agree bit for bit on keys, encryptions, every key-switching primitive and the three kernels' schedules.
"""
import json
import os

M64 = (1 << 64) - 1
_PARAMS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "params")


# ------------------------------------------------------------------------------------ PRNG
def draw(seed, stream, index):
    """mix64((seed XOR stream * 0xD1B54A32D192ED03) + (index + 1) * 0x9E3779B97F4A7C15), SplitMix64 finaliser."""
    z = ((seed ^ ((stream * 0xD1B54A32D192ED03) & M64)) + (((index + 1) * 0x9E3779B97F4A7C15) & M64)) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def uniform(seed, stream, q, gid, N):
    """Uniform mod q: ((hi 2^64 + lo) q) >> 128, hi/lo = draws 2(gid N + k), 2(gid N + k) + 1."""
    out = []
    for k in range(N):
        i = 2 * (gid * N + k)
        out.append((((draw(seed, stream, i) << 64) | draw(seed, stream, i + 1)) * q) >> 128)
    return out


def ternary(seed, stream, N):
    return [((draw(seed, stream, k) * 3) >> 64) - 1 for k in range(N)]


def cbd21(seed, stream, N):
    out = []
    for k in range(N):
        u = draw(seed, stream, k)
        out.append(bin(u & 0x1FFFFF).count("1") - bin((u >> 21) & 0x1FFFFF).count("1"))
    return out


S_SK = 1 << 56
S_ENC_A, S_ENC_E = 3 << 56, (3 << 56) | 1


def s_ksk(g, j, comp):
    return (2 << 56) | (g << 16) | (j << 8) | comp


def s_mask(sid):
    return (4 << 56) | sid


# ------------------------------------------------------------------------------------ ring
class Params:
    def __init__(self, name):
        with open(os.path.join(_PARAMS, name.lower() + ".json")) as f:
            d = json.load(f)
        self.N = int(d["N"])
        self.n = self.N // 2
        self.q = [int(x) for x in d["q"]]
        self.p = [int(x) for x in d["p"]]
        self.alpha = int(d["alpha"])
        self.Lmax = len(self.q)
        self.Kl = [int(k) for k in d.get("K_of_level", [len(self.p)] * self.Lmax)]

    def dnum(self, L):
        return -(-L // self.alpha)

    def K(self, L):
        """Special primes of a key switch at level L (DESIGN.md R-KL)."""
        return self.Kl[L - 1]

    def PK(self, L):
        out = 1
        for x in self.p[:self.K(L)]:
            out *= x
        return out

    def ext(self, L):
        return self.q[:L] + self.p[:self.K(L)]

    def gids(self, L):
        return list(range(L)) + [self.Lmax + k for k in range(self.K(L))]


def negacyclic(a, b, q):
    """c_k = sum_{i+j=k} a_i b_j - sum_{i+j=k+N} a_i b_j  (mod q), the ring product of Z_q[X]/(X^N + 1)."""
    N = len(a)
    c = [0] * N
    for i, ai in enumerate(a):
        if ai:
            for j, bj in enumerate(b):
                k = i + j
                if k < N:
                    c[k] += ai * bj
                else:
                    c[k - N] -= ai * bj
    return [x % q for x in c]


def automorph(a, g, q):
    """sigma_g: X^k -> X^{kg mod 2N} with X^N = -1."""
    N = len(a)
    out = [0] * N
    for k, v in enumerate(a):
        e = (k * g) % (2 * N)
        if e < N:
            out[e] = (out[e] + v) % q
        else:
            out[e - N] = (out[e - N] - v) % q
    return out


def padd(a, b, q):
    return [(x + y) % q for x, y in zip(a, b)]


def psub(a, b, q):
    return [(x - y) % q for x, y in zip(a, b)]


def smul(a, s, q):
    return [(x * s) % q for x in a]


def crt(res, mods):
    """x in [0, prod mods) with x = res_i mod mods_i (explicit CRT)."""
    M = 1
    for q in mods:
        M *= q
    x = 0
    for r, q in zip(res, mods):
        Mi = M // q
        x += r * Mi * pow(Mi, -1, q)
    return x % M, M


def centred(x, M):
    """The representative of x mod M in (-M/2, M/2) (M odd: no tie)."""
    x %= M
    return x - M if 2 * x > M else x


# ------------------------------------------------------------------------------------ keys and encryption
class Keys:
    """ksk_{g,j} = (-a_j s + e_j + g_j s', a_j) over Q_max u P, g_j = P on digit j's q-limbs, 0 elsewhere;
    s' = sigma_g(s), or s^2 for g = 0 (relinearisation)."""

    def __init__(self, P, seed, galois=(), relin=False, max_level=None):
        self.P, self.seed = P, seed
        self.ML = max_level or P.Lmax
        N = P.N
        self.s_signed = ternary(seed, S_SK, N)
        mods = P.ext(self.ML)
        self.s = [[v % t for v in self.s_signed] for t in mods]
        self.galois = list(galois) + ([0] if relin else [])
        self._cls = {}
        self.ksk = {g: self._gen(g, P.K(self.ML)) for g in self.galois}

    def _gen(self, g, K):
        """The key of special modulus P_K = p_0..p_{K-1} over Q_ML u P_K, generated from its definition (each class
        K of DESIGN.md R-KL on its own: same streams, so the a_j / e_j draws are shared by construction)."""
        P, ML = self.P, self.ML
        mods = self.P.q[:ML] + self.P.p[:K]
        gids = list(range(ML)) + [P.Lmax + k for k in range(K)]
        PK = 1
        for x in P.p[:K]:
            PK *= x
        s = [[v % t for v in self.s_signed] for t in mods]
        sp = [negacyclic(si, si, t) for si, t in zip(s, mods)] if g == 0 else [automorph(si, g, t) for si, t in zip(s, mods)]
        out = []
        for j in range(P.dnum(ML)):
            lo, hi = j * P.alpha, min((j + 1) * P.alpha, ML)
            e = cbd21(self.seed, s_ksk(g, j, 1), P.N)
            b, a = [], []
            for i, (t, gid) in enumerate(zip(mods, gids)):
                ai = uniform(self.seed, s_ksk(g, j, 0), t, gid, P.N)
                bi = psub([v % t for v in e], negacyclic(ai, s[i], t), t)
                if lo <= i < hi:
                    bi = padd(bi, smul(sp[i], PK % t, t), t)
                b.append(bi)
                a.append(ai)
            out.append((b, a))
        return out

    def s_at(self, L):
        return self.s[:L]

    def key_at(self, g, L):
        ML, K = self.ML, self.P.K(L)
        if (g, K) not in self._cls:
            self._cls[(g, K)] = self.ksk[g] if K == self.P.K(ML) else self._gen(g, K)
        idx = list(range(L)) + list(range(ML, ML + K))
        return [([b[i] for i in idx], [a[i] for i in idx]) for (b, a) in self._cls[(g, K)][: self.P.dnum(L)]]


class Ct:
    def __init__(self, c, scale):
        self.c, self.scale = c, float(scale)      # c: [comp][limb][N] lists of ints

    @property
    def L(self):
        return len(self.c[0])


def encrypt_sk(P, keys, m, scale, seed):
    """c1 = a uniform (stream enc_a, limb ids i), c0 = -a s + e + m."""
    L = len(m)
    e = cbd21(seed, S_ENC_E, P.N)
    c0, c1 = [], []
    for i in range(L):
        q = P.q[i]
        a = uniform(seed, S_ENC_A, q, i, P.N)
        c0.append(padd(psub([v % q for v in e], negacyclic(a, keys.s[i], q), q), m[i], q))
        c1.append(a)
    return Ct([c0, c1], scale)


def decrypt(P, keys, ct):
    L = ct.L
    out = []
    for i in range(L):
        q = P.q[i]
        m = padd(ct.c[0][i], negacyclic(ct.c[1][i], keys.s[i], q), q)
        if len(ct.c) == 3:
            m = padd(m, negacyclic(ct.c[2][i], negacyclic(keys.s[i], keys.s[i], q), q), q)
        out.append(m)
    return out


# ------------------------------------------------------------------------------------ key switching
def modup(P, d, L):
    """Per digit j: inside the digit d~ = d; on every other modulus t of Q_L u P the integer
    sum_i [d_i (Q_j/q_i)^{-1}]_{q_i} (Q_j/q_i) (fast base conversion, no correction) reduced mod t."""
    mods = P.ext(L)
    N = P.N
    out = []
    for j in range(P.dnum(L)):
        lo, hi = j * P.alpha, min((j + 1) * P.alpha, L)
        dq = P.q[lo:hi]
        Qj = 1
        for q in dq:
            Qj *= q
        ints = []
        for k in range(N):
            s = 0
            for i, q in enumerate(dq):
                s += (d[lo + i][k] * pow(Qj // q, -1, q) % q) * (Qj // q)
            ints.append(s)
        ext = []
        for idx, t in enumerate(mods):
            ext.append(list(d[idx]) if lo <= idx < hi else [v % t for v in ints])
        out.append(ext)
    return out


def ks_inner(P, digits, key, L):
    mods = P.ext(L)
    acc = [[[0] * P.N for _ in mods] for _ in range(2)]
    for dj, (kb, ka) in zip(digits, key):
        for i, t in enumerate(mods):
            acc[0][i] = padd(acc[0][i], negacyclic(dj[i], kb[i], t), t)
            acc[1][i] = padd(acc[1][i], negacyclic(dj[i], ka[i], t), t)
    return acc


def hps_round(vs, bm):
    """r = round(sum_k v_k / b_k) as DESIGN.md R-MODDOWN specifies it: each v_k / b_k as the 59-bit fixed-point
    value floor(v_k 2^{s_k} floor(2^{123 - s_k} / b_k) / 2^64), s_k = 63 - bitlen(b_k), summed, + 2^58, >> 59.
    Equals exact rounding unless sum_k v_k / b_k lies within ~2^-56 of a half-integer
    (tests/test_crossmodel.py pins both statements)."""
    f = 0
    for v, b in zip(vs, bm):
        s = 63 - b.bit_length()
        f += ((v << s) * ((1 << (123 - s)) // b)) >> 64
    return (f + (1 << 58)) >> 59


def div_round(x, L, P, base_idx, keep):
    """round(x / B) mod q_i for i < keep, B = prod of the moduli at positions base_idx of Q_L u P (DESIGN.md
    R-MODDOWN): v_k = [x_k (B/b_k)^{-1}]_{b_k}, r = hps_round(v), y = sum_k v_k (B/b_k) - r B as ONE big integer
    (the representative of x mod B that the rounding selects), then (x_i - y) B^{-1} mod q_i."""
    mods = P.ext(L)
    bm = [mods[i] for i in base_idx]
    B = 1
    for t in bm:
        B *= t
    out = [[0] * P.N for _ in range(keep)]
    for k in range(P.N):
        vs = [x[i][k] * pow(B // b, -1, b) % b for i, b in zip(base_idx, bm)]
        y = sum(v * (B // b) for v, b in zip(vs, bm)) - hps_round(vs, bm) * B
        for i in range(keep):
            q = P.q[i]
            out[i][k] = (x[i][k] - y) * pow(B % q, -1, q) % q
    return out


def moddown(P, b, L):
    return div_round(b, L, P, list(range(L, L + P.K(L))), L)


def moddown_rescale(P, x, L):
    return div_round(x, L, P, [L - 1] + list(range(L, L + P.K(L))), L - 1)


def lift_P(P, c, L):
    PK = P.PK(L)
    return [smul(c[i], PK % P.q[i], P.q[i]) for i in range(L)] + [[0] * P.N for _ in range(P.K(L))]


def rotate_ext(P, keys, ct, g, ext=None):
    """(P sigma_g(c0) + b0, b1) over Q_L u P; `ext` = a hoisted ModUp of c1 (sigma applied to its digits), else
    the single key switch's ModUp of sigma_g(c1)."""
    L = ct.L
    mods = P.ext(L)
    c0 = [automorph(ct.c[0][i], g, P.q[i]) for i in range(L)]
    if ext is None:
        d = modup(P, [automorph(ct.c[1][i], g, P.q[i]) for i in range(L)], L)
    else:
        d = [[automorph(dj[i], g, t) for i, t in enumerate(mods)] for dj in ext]
    b0, b1 = ks_inner(P, d, keys.key_at(g, L), L)
    lp = lift_P(P, c0, L)
    return [[padd(b0[i], lp[i], t) for i, t in enumerate(mods)], b1]


def rotate(P, keys, ct, g, ext=None):
    e = rotate_ext(P, keys, ct, g, ext)
    return Ct([moddown(P, e[0], ct.L), moddown(P, e[1], ct.L)], ct.scale)


def galois_rot(P, r):
    return pow(5, r % P.n, 2 * P.N)


def relin_ext(P, keys, ct):
    L = ct.L
    mods = P.ext(L)
    b0, b1 = ks_inner(P, modup(P, ct.c[2], L), keys.key_at(0, L), L)
    l0, l1 = lift_P(P, ct.c[0], L), lift_P(P, ct.c[1], L)
    return [[padd(b0[i], l0[i], t) for i, t in enumerate(mods)], [padd(b1[i], l1[i], t) for i, t in enumerate(mods)]]


def rescale(P, ct):
    """floor((x + floor(q_{L-1}/2)) / q_{L-1}) mod q_i from the explicit CRT value x in [0, Q_L)."""
    L = ct.L
    ql = P.q[L - 1]
    out = []
    for comp in ct.c:
        o = [[0] * P.N for _ in range(L - 1)]
        for k in range(P.N):
            X, _ = crt([comp[i][k] for i in range(L)], P.q[:L])
            v = (X + ql // 2) // ql
            for i in range(L - 1):
                o[i][k] = v % P.q[i]
        out.append(o)
    return Ct(out, ct.scale / float(ql))


# ------------------------------------------------------------------------------------ evaluator for kernels.py
class XExt:
    def __init__(self, c, L, scale):
        self.c, self.L, self.scale, self.ncomp = c, L, float(scale), 2


class XEv:
    """The evaluator interface of oracle/kernels.py (Ev) on the big-int model, so the kernel schedules run on
    independent arithmetic.  Ciphertexts are Ct / XExt (lists of ints)."""

    def __init__(self, P, keys, m, encode_mask):
        from collections import Counter
        self.P, self.keys, self.m = P, keys, m
        self.ledger = Counter()
        self._enc = encode_mask              # (slot vector, scale) -> signed integer coefficients (shared data)
        self._masks = {}

    def _mask_int(self, desc, L, m):
        from . import kernels as K
        key = (tuple(desc), L, m)
        if key not in self._masks:
            self._masks[key] = [int(v) for v in self._enc(K.mask_slots(desc, m, self.P.n), float(self.P.q[L - 1]))]
        return self._masks[key]

    def mask(self, desc, L, m=None):
        ints = self._mask_int(desc, L, m or self.m)
        return ([[v % q for v in ints] for q in self.P.q[:L]], float(self.P.q[L - 1]))

    def mask_ext(self, desc, L, m=None):
        ints = self._mask_int(desc, L, m or self.m)
        return ([[v % t for v in ints] for t in self.P.ext(L)], float(self.P.q[L - 1]))

    def mask_scale(self, L):
        return float(self.P.q[L - 1])

    def _hoist(self, ct):
        return modup(self.P, ct.c[1], ct.L)

    def rot(self, ct, r):
        if r % self.P.n == 0:
            return Ct([list(map(list, c)) for c in ct.c], ct.scale)
        return rotate(self.P, self.keys, ct, galois_rot(self.P, r))

    def rot_hoisted(self, ct, rs):
        ext = self._hoist(ct)
        return [Ct([list(map(list, c)) for c in ct.c], ct.scale) if r % self.P.n == 0 else
                rotate(self.P, self.keys, ct, galois_rot(self.P, r), ext) for r in rs]

    def conj(self, ct):
        return rotate(self.P, self.keys, ct, 2 * self.P.N - 1)

    def tensor(self, a, b):
        L = a.L
        d = [[], [], []]
        for i in range(L):
            q = self.P.q[i]
            a0, a1, b0, b1 = a.c[0][i], a.c[1][i], b.c[0][i], b.c[1][i]
            d[0].append(negacyclic(a0, b0, q))
            d[1].append(padd(negacyclic(a0, b1, q), negacyclic(a1, b0, q), q))
            d[2].append(negacyclic(a1, b1, q))
        return Ct(d, a.scale * b.scale)

    def ptmul(self, ct, pt):
        m, s = pt
        return Ct([[negacyclic(c[i], m[i], self.P.q[i]) for i in range(ct.L)] for c in ct.c], ct.scale * s)

    def add(self, a, b):
        assert a.scale == b.scale and a.L == b.L
        nc = max(len(a.c), len(b.c))
        z = [[0] * self.P.N for _ in range(a.L)]
        out = []
        for c in range(nc):
            x = a.c[c] if c < len(a.c) else z
            y = b.c[c] if c < len(b.c) else z
            out.append([padd(x[i], y[i], self.P.q[i]) for i in range(a.L)])
        return Ct(out, a.scale)

    def sub(self, a, b):
        assert a.scale == b.scale and a.L == b.L
        return Ct([[psub(a.c[c][i], b.c[c][i], self.P.q[i]) for i in range(a.L)] for c in range(len(a.c))], a.scale)

    def mul_i(self, ct):
        h = self.P.N // 2   # X^{N/2} a: coefficient k moves to k + N/2, negated on wrap
        out = []
        for comp in ct.c:
            o = []
            for i, a in enumerate(comp):
                q = self.P.q[i]
                o.append([(-a[k + h]) % q for k in range(h)] + [a[k] for k in range(h)])
            out.append(o)
        return Ct(out, ct.scale)

    def rescale(self, ct):
        return rescale(self.P, ct)

    def mod_drop(self, ct, L):
        return Ct([c[:L] for c in ct.c], ct.scale)

    def scale_mul(self, ct, f):
        return Ct(ct.c, ct.scale * f)

    def rot_hoisted_ext(self, ct, rs):
        ext = self._hoist(ct)
        out = []
        for r in rs:
            if r % self.P.n == 0:
                out.append(self.lift_ext(ct))
            else:
                out.append(XExt(rotate_ext(self.P, self.keys, ct, galois_rot(self.P, r), ext), ct.L, ct.scale))
        return out

    def ext_masked_sum(self, xs, pts, scale):
        L = xs[0].L
        mods = self.P.ext(L)
        acc = [[[0] * self.P.N for _ in mods] for _ in range(2)]
        for x, (pm, _) in zip(xs, pts):
            for c in range(2):
                for i, t in enumerate(mods):
                    acc[c][i] = padd(acc[c][i], negacyclic(x.c[c][i], pm[i], t), t)
        return XExt(acc, L, scale)

    def lift_ext(self, ct):
        return XExt([lift_P(self.P, ct.c[c], ct.L) for c in range(2)], ct.L, ct.scale)

    def rot_ext(self, ct, r):
        if r % self.P.n == 0:
            return self.lift_ext(ct)
        return XExt(rotate_ext(self.P, self.keys, ct, galois_rot(self.P, r)), ct.L, ct.scale)

    def conj_ext(self, ct):
        return XExt(rotate_ext(self.P, self.keys, ct, 2 * self.P.N - 1), ct.L, ct.scale)

    def ext_add(self, a, b):
        assert a.scale == b.scale
        mods = self.P.ext(a.L)
        return XExt([[padd(a.c[c][i], b.c[c][i], t) for i, t in enumerate(mods)] for c in range(2)], a.L, a.scale)

    def moddown(self, y):
        return Ct([moddown(self.P, y.c[c], y.L) for c in range(2)], y.scale)

    def moddown_rescale(self, y):
        return Ct([moddown_rescale(self.P, y.c[c], y.L) for c in range(2)], y.scale / float(self.P.q[y.L - 1]))

    def relin(self, ct):
        e = relin_ext(self.P, self.keys, ct)
        return Ct([moddown(self.P, e[0], ct.L), moddown(self.P, e[1], ct.L)], ct.scale)

    def relin_rescale(self, ct):
        return self.moddown_rescale(XExt(relin_ext(self.P, self.keys, ct), ct.L, ct.scale))

    def mac_ptmul(self, cts, pts):
        out = None
        for ct, pt in zip(cts, pts):
            y = self.ptmul(ct, pt)
            out = y if out is None else self.add(out, y)
        return out

    def tensor_sum(self, pairs):
        out = None
        for a, b in pairs:
            t = self.tensor(a, b)
            out = t if out is None else self.add(out, t)
        return out


def export_c2m(P, ct, L_conv, mask_seed, stream_id):
    """Alg 3 GPU half: mod-drop to L_conv, r^ uniform mod q_i (stream mask(stream_id), limb ids i),
    d = (c0 + r^, c1), share = -r^."""
    c0, c1, share = [], [], []
    for i in range(L_conv):
        q = P.q[i]
        r = uniform(mask_seed, s_mask(stream_id), q, i, P.N)
        c0.append(padd(ct.c[0][i], r, q))
        c1.append(list(ct.c[1][i]))
        share.append([(-v) % q for v in r])
    return Ct([c0, c1], ct.scale), share
