"""CPU CKKS oracle: keygen / encrypt / decrypt / encode / decode / key switching / rescale.

TEST INFRASTRUCTURE ONLY -- only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this module.  It shares no code with the CUDA library.

Everything here is in the COEFFICIENT domain, by definition.  Ring
products go through the oracle's own textbook NTT (oracle.c: o_ntt_fwd), which tests pin against
schoolbook negacyclic convolution (the ring product mod q is unique, so this is a substitution of
a library primitive, not a reordering of the method).  Big-integer constants (CRT, BConv factors,
P^{-1}) are computed with Python ints.

Citations: RNS-CKKS, Galois keys, rot = cyclic LEFT shift,
conj, rescale, ModSwitchToNext, encode/decode.
Readings where the paper is silent (C3 sampling, C4 hybrid key switching, C5 SEAL rescale) are in
DESIGN.md "Readings" (G12-G18).
"""
import ctypes
import json
import os
import subprocess
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
PARAMS_DIR = os.path.join(os.path.dirname(_HERE), "params")


def build_oracle(force=False):
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    build_oracle()
    lib = ctypes.CDLL(_SO)
    u64, i64, p = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p
    sig = {
        "o_mulmod": ([u64, u64, u64], u64),
        "o_powmod": ([u64, u64, u64], u64),
        "o_invmod": ([u64, u64], u64),
        "o_negacyclic_schoolbook": ([u64, i64, p, p, p], None),
        "o_ntt_fwd_batch": ([i64, p, p, i64, p], None),
        "o_ntt_inv_batch": ([i64, p, p, i64, p], None),
        "o_add_batch": ([i64, p, i64, p, p, p], None),
        "o_sub_batch": ([i64, p, i64, p, p, p], None),
        "o_mul_batch": ([i64, p, i64, p, p, p], None),
        "o_mac_batch": ([i64, p, i64, p, p, p], None),
        "o_mul_scalar_batch": ([i64, p, i64, p, p, p], None),
        "o_from_signed_batch": ([i64, p, i64, p, p], None),
        "o_automorph_batch": ([i64, p, i64, u64, p, p], None),
        "o_bconv": ([i64, i64, p, p, p, i64, p, p, p], None),
        "o_bconv_round": ([i64, i64, p, p, p, i64, p, p, p, p, p, p], None),
        "o_rescale": ([i64, p, i64, p, p], None),
        "o_prng_draw": ([u64, u64, u64], u64),
        "o_sample_uniform": ([u64, u64, i64, p, p, i64, p], None),
        "o_sample_ternary": ([u64, u64, i64, p], None),
        "o_sample_cbd21": ([u64, u64, i64, p], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


class _Lib:
    def __init__(self, lib):
        self._lib = lib

    def __getattr__(self, name):
        f = getattr(self._lib, name)

        def call(*args):
            try:
                return f(*args)
            finally:
                _KEEP.clear()
        return call


LIB = _Lib(_load())


_KEEP = []


def _ptr(a):
    """Raw pointer to a C-contiguous array.  The array is kept alive in _KEEP until the next _call()
    returns (temporaries such as _ptr(_u64(...)) must not be freed before the C call runs)."""
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the oracle must be C-contiguous"
    _KEEP.append(a)
    return ctypes.c_void_p(a.ctypes.data)


def _u64(xs):
    return np.ascontiguousarray(np.array([int(x) for x in xs], dtype=np.uint64))


# ------------------------------------------------------------------------------------ PRNG streams
# DESIGN.md "PRNG and streams" (the paper is silent).
STREAM_SK = 0x01 << 56
def stream_ksk(galois, digit, comp):          # comp 0 = a, 1 = e; galois 0 = relinearisation key
    return (0x02 << 56) | (int(galois) << 16) | (int(digit) << 8) | int(comp)
STREAM_ENC_A = (0x03 << 56) | 0
STREAM_ENC_E = (0x03 << 56) | 1
def stream_mask(stream_id):
    return (0x04 << 56) | int(stream_id)


def prng_draw(seed, stream, index):
    return int(LIB.o_prng_draw(seed, stream, index))


# ------------------------------------------------------------------------------------ parameters
class Params:
    """A parameter set (params/*.json): N, body primes q_0..q_{L-1}, special primes p_0..p_{alpha-1}."""

    def __init__(self, name_or_path):
        path = name_or_path if name_or_path.endswith(".json") else os.path.join(PARAMS_DIR, name_or_path.lower() + ".json")
        with open(path) as f:
            d = json.load(f)
        self.name = d["name"]
        self.N = int(d["N"])
        self.n = self.N // 2
        self.q = [int(x) for x in d["q"]]
        self.p = [int(x) for x in d["p"]]
        self.alpha = int(d["alpha"])
        self.L_max = len(self.q)
        self.log2_scale = int(d["log2_scale"])
        self.P = 1                      # the product of ALL special primes (keys are generated for it)
        for pk in self.p:
            self.P *= pk
        # K(L): special primes a key switch at level L extends by (DESIGN.md R-KL; data in the param file, else all)
        self.K_of_level = [int(k) for k in d.get("K_of_level", [len(self.p)] * self.L_max)]

    def dnum(self, L):
        return -(-L // self.alpha)

    def digit(self, j, L):
        return j * self.alpha, min((j + 1) * self.alpha, L)

    def K(self, L):
        return self.K_of_level[L - 1]

    def P_of(self, L):
        """P_{K(L)} = p_0 ... p_{K(L)-1}: the special modulus of a key switch at level L."""
        out = 1
        for pk in self.p[:self.K(L)]:
            out *= pk
        return out

    # global limb ids: q_i -> i ; p_k -> L_max + k  (PRNG index layout and key limb layout)
    def ext_mods(self, L):
        return self.q[:L] + self.p[:self.K(L)]

    def ext_gids(self, L):
        return list(range(L)) + [self.L_max + k for k in range(self.K(L))]

    def psi(self, q):
        return primitive_root_2n(q, self.N)


@lru_cache(maxsize=None)
def primitive_root_2n(q, N):
    """The smallest primitive 2N-th root of unity mod q (psi^N = -1).  Found as g^((q-1)/2N) for the
    first g giving psi^N = -1, then the minimum over all odd powers (the full set of such roots)."""
    assert (q - 1) % (2 * N) == 0
    for g in range(2, 1000):
        r = pow(g, (q - 1) // (2 * N), q)
        if pow(r, N, q) == q - 1:
            break
    else:
        raise ValueError("no root found")
    best, cur, sq = r, r, r * r % q
    for _ in range(N - 1):
        cur = cur * sq % q
        best = min(best, cur)
    return best


# ------------------------------------------------------------------------------------ polynomial ops
def ntt(a, mods, N):
    """Oracle NTT of each limb (in place on a copy): a_j = a(psi^{2j+1})."""
    out = np.ascontiguousarray(a, dtype=np.uint64).copy()
    nl = len(mods)
    LIB.o_ntt_fwd_batch(nl, _ptr(_u64(mods)), _ptr(_u64([primitive_root_2n(q, N) for q in mods])), N, _ptr(out))
    return out


def intt(a, mods, N):
    out = np.ascontiguousarray(a, dtype=np.uint64).copy()
    nl = len(mods)
    LIB.o_ntt_inv_batch(nl, _ptr(_u64(mods)), _ptr(_u64([primitive_root_2n(q, N) for q in mods])), N, _ptr(out))
    return out


def _binop(fn, a, b, mods, N):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.empty_like(a)
    fn(len(mods), _ptr(_u64(mods)), N, _ptr(a), _ptr(b), _ptr(out))
    return out


def padd(a, b, mods, N):
    return _binop(LIB.o_add_batch, a, b, mods, N)


def psub(a, b, mods, N):
    return _binop(LIB.o_sub_batch, a, b, mods, N)


def pmul_pointwise(a, b, mods, N):
    return _binop(LIB.o_mul_batch, a, b, mods, N)


def pneg(a, mods, N):
    return psub(np.zeros_like(a), a, mods, N)


def pmul_scalar(a, scal, mods, N):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty_like(a)
    LIB.o_mul_scalar_batch(len(mods), _ptr(_u64(mods)), N, _ptr(a), _ptr(_u64([s % q for s, q in zip(scal, mods)])), _ptr(out))
    return out


def ring_mul(a, b, mods, N):
    """Ring product per limb, via the oracle NTT (pinned against ring_mul_schoolbook)."""
    return intt(pmul_pointwise(ntt(a, mods, N), ntt(b, mods, N), mods, N), mods, N)


def ring_mul_schoolbook(a, b, mods, N):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.empty_like(a)
    for l, q in enumerate(mods):
        LIB.o_negacyclic_schoolbook(q, N, _ptr(a[l]), _ptr(b[l]), _ptr(out[l]))
    return out


def from_signed(v, mods, N):
    v = np.ascontiguousarray(v, dtype=np.int64)
    out = np.empty((len(mods), N), dtype=np.uint64)
    LIB.o_from_signed_batch(len(mods), _ptr(_u64(mods)), N, _ptr(v), _ptr(out))
    return out


def automorph(a, g, mods, N):
    """sigma_g: X -> X^g on each limb (coefficient domain)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty_like(a)
    LIB.o_automorph_batch(len(mods), _ptr(_u64(mods)), N, int(g) % (2 * N), _ptr(a), _ptr(out))
    return out


def mul_monomial_half(a, mods, N):
    """X^{N/2} * a (negacyclic): (X^{N/2} a)_k = a_{k-N/2} for k >= N/2, -a_{k+N/2} for k < N/2.
    Decodes to i * (slots)  (App. A of SURVEY: X^{N/2} evaluated at zeta^{5^j} is i)."""
    h = N // 2
    out = np.empty_like(a)
    out[:, h:] = a[:, :h]
    out[:, :h] = pneg(np.ascontiguousarray(a[:, h:]), mods, h)
    return out


def bconv(x, qin, qout, N):
    """Fast base conversion without correction (C4): y_t = sum_i [x_i (Q'/q_i)^{-1}]_{q_i} (Q'/q_i) mod t."""
    Qp = 1
    for q in qin:
        Qp *= q
    vfac = [pow(Qp // q, -1, q) for q in qin]
    wfac = [(Qp // qi) % t for qi in qin for t in qout]
    x = np.ascontiguousarray(x, dtype=np.uint64)
    out = np.empty((len(qout), N), dtype=np.uint64)
    LIB.o_bconv(N, len(qin), _ptr(_u64(qin)), _ptr(x), _ptr(_u64(vfac)), len(qout), _ptr(_u64(qout)), _ptr(_u64(wfac)), _ptr(out))
    return out


def bconv_round(x, qin, qout, N):
    """Fast base conversion WITH the rounding correction (DESIGN.md R-MODDOWN): r = round(sum_i v_i/q_i) from a
    59-bit fixed-point estimate; returns the centred residue of x mod Q' = prod(qin) in every target modulus
    (exact unless sum_i v_i/q_i lies within 2^-56 of a half-integer)."""
    Qp = 1
    for q in qin:
        Qp *= q
    vfac = [pow(Qp // q, -1, q) for q in qin]
    wfac = [(Qp // qi) % t for qi in qin for t in qout]
    qprod = [Qp % t for t in qout]
    csh = [63 - q.bit_length() for q in qin]
    cfix = [(1 << (123 - s)) // q for q, s in zip(qin, csh)]
    x = np.ascontiguousarray(x, dtype=np.uint64)
    out = np.empty((len(qout), N), dtype=np.uint64)
    LIB.o_bconv_round(N, len(qin), _ptr(_u64(qin)), _ptr(x), _ptr(_u64(vfac)), len(qout), _ptr(_u64(qout)), _ptr(_u64(wfac)),
                      _ptr(_u64(qprod)), _ptr(_u64(cfix)), _ptr(_u64(csh)), _ptr(out))
    return out


def rescale_poly(a, mods, N):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty((len(mods) - 1, N), dtype=np.uint64)
    LIB.o_rescale(len(mods), _ptr(_u64(mods)), N, _ptr(a), _ptr(out))
    return out


# ------------------------------------------------------------------------------------ sampling
def sample_uniform(seed, stream, mods, gids, N):
    out = np.empty((len(mods), N), dtype=np.uint64)
    LIB.o_sample_uniform(seed, stream, len(mods), _ptr(_u64(mods)), _ptr(np.ascontiguousarray(np.array(gids, dtype=np.int64))), N, _ptr(out))
    return out


def sample_ternary(seed, stream, N):
    out = np.empty(N, dtype=np.int64)
    LIB.o_sample_ternary(seed, stream, N, _ptr(out))
    return out


def sample_cbd21(seed, stream, N):
    out = np.empty(N, dtype=np.int64)
    LIB.o_sample_cbd21(seed, stream, N, _ptr(out))
    return out


# ------------------------------------------------------------------------------------ CRT
def crt_lift(a, mods, centered=True):
    """Explicit CRT: limbs [L][N] -> Python ints in [0,Q) (or centred in (-Q/2, Q/2])."""
    Q = 1
    for q in mods:
        Q *= q
    terms = []
    for q in mods:
        Qi = Q // q
        terms.append((Qi * pow(Qi, -1, q), q))
    N = a.shape[1]
    out = []
    rows = [[int(v) for v in a[l]] for l in range(len(mods))]
    for k in range(N):
        x = 0
        for l, (c, q) in enumerate(terms):
            x += rows[l][k] * c
        x %= Q
        if centered and x > Q // 2:
            x -= Q
        out.append(x)
    return out, Q


# ------------------------------------------------------------------------------------ encode / decode
@lru_cache(maxsize=None)
def _rot_group(N):
    """e_j = 5^j mod 2N for j < n (slot j <-> evaluation point zeta^{5^j}, zeta = e^{i pi/N})."""
    n = N // 2
    e = np.empty(n, dtype=np.int64)
    x = 1
    for j in range(n):
        e[j] = x
        x = x * 5 % (2 * N)
    return e


def encode_coeffs(z, scale, N):
    """Encode: m_k = round_half_even( scale * (2/N) * Re sum_j z_j zeta^{-5^j k} ).
    The sum over j is a length-2N DFT of the vector A with A[5^j mod 2N] = z_j.
    Returns signed int64 coefficients."""
    n = N // 2
    zz = np.zeros(n, dtype=np.complex128)
    zin = np.asarray(z, dtype=np.complex128).reshape(-1)
    zz[:len(zin)] = zin
    z = zz
    A = np.zeros(2 * N, dtype=np.complex128)
    A[_rot_group(N)] = z
    S = np.fft.fft(A)[:N]                       # sum_e A[e] exp(-2 pi i e k / 2N)
    m = np.rint(scale * (2.0 / N) * S.real)     # np.rint rounds half to even
    if np.max(np.abs(m)) >= 2.0 ** 62:
        raise OverflowError("encode: |scale*z| too large for 63-bit coefficients")
    return m.astype(np.int64)


def encode_coeffs_direct(z, scale, N):
    """O(N^2) reference of the same formula (pin for encode_coeffs at small N)."""
    n = N // 2
    e = _rot_group(N)
    k = np.arange(N)
    zeta = np.exp(-1j * np.pi * np.outer(e, k) / N)
    S = (np.asarray(z, dtype=np.complex128)[:, None] * zeta).sum(axis=0)
    return np.rint(scale * (2.0 / N) * S.real).astype(np.int64)


def decode_coeffs(m, scale, N):
    """Decode: z_j = (1/scale) sum_k m_k zeta^{5^j k} for centred integer coefficients m (Python ints ok)."""
    mf = np.array([float(v) for v in m], dtype=np.float64)
    Z = np.fft.ifft(mf, 2 * N) * (2 * N)           # sum_k m_k exp(+2 pi i e k / 2N)
    return Z[_rot_group(N)] / scale


class Pt:
    def __init__(self, m, scale):
        self.m = np.ascontiguousarray(m, dtype=np.uint64)   # [L][N], coefficient domain
        self.scale = float(scale)

    @property
    def L(self):
        return self.m.shape[0]


class Ct:
    def __init__(self, c, scale):
        self.c = np.ascontiguousarray(c, dtype=np.uint64)   # [comp][L][N], coefficient domain
        self.scale = float(scale)

    @property
    def L(self):
        return self.c.shape[1]

    @property
    def ncomp(self):
        return self.c.shape[0]


class OracleError(Exception):
    """Error names follow SPEC (...) / include/encf.h status codes."""


def encode(P, z, scale, L):
    m = encode_coeffs(z, scale, P.N)
    return Pt(from_signed(m, P.q[:L], P.N), scale)


def decode(P, pt, n_limbs=None):
    mods = P.q[:pt.L]
    vals, _ = crt_lift(pt.m if n_limbs is None else pt.m[:n_limbs], mods if n_limbs is None else mods[:n_limbs])
    return decode_coeffs(vals, pt.scale, P.N)


# ------------------------------------------------------------------------------------ keys
class Keys:
    """Secret key and hybrid key-switching keys (paper silent, P:68 only names them).

    ksk_{g,j} = ( -a_j s + e_j + g_j s' , a_j )  mod Q_max * P, with g_j = P mod q_i on digit j's
    q-limbs and 0 on every other limb.  s' = sigma_g(s) (Galois) or s^2 (relin, g = 0).
    Stored coefficient-domain, limbs [q_0..q_{max_level-1}, p_0..p_{alpha-1}]."""

    def __init__(self, P, seed, galois=(), relin=False, max_level=None):
        self.P = P
        self.seed = int(seed)
        self.max_level = max_level or P.L_max
        N = P.N
        self.s_signed = sample_ternary(self.seed, STREAM_SK, N)
        mods = P.ext_mods(self.max_level)
        self.s = from_signed(self.s_signed, mods, N)          # over Q_max * P
        self.ksk = {}
        self._sp = {}
        self._ntt_cache = {}
        targets = list(galois) + ([0] if relin else [])
        for g in targets:
            self.ksk[int(g)] = self._gen(int(g))

    def _gen(self, g):
        P, N = self.P, self.P.N
        ML = self.max_level
        mods, gids = P.ext_mods(ML), P.ext_gids(ML)
        sp = ring_mul(self.s, self.s, mods, N) if g == 0 else automorph(self.s, g, mods, N)
        self._sp[g] = sp
        PK = P.P_of(ML)
        out = []
        for j in range(P.dnum(ML)):
            lo, hi = P.digit(j, ML)
            a = sample_uniform(self.seed, stream_ksk(g, j, 0), mods, gids, N)
            e = from_signed(sample_cbd21(self.seed, stream_ksk(g, j, 1), N), mods, N)
            gfac = [(PK % t) if lo <= i < hi else 0 for i, t in enumerate(mods)]
            b = padd(psub(e, ring_mul(a, self.s, mods, N), mods, N), pmul_scalar(sp, gfac, mods, N), mods, N)
            out.append(np.stack([b, a]))
        return out                     # list over digits of [2][ML+K(ML)][N]

    _sp = None

    def s_at(self, L):
        return np.ascontiguousarray(self.s[:L])

    def key_at(self, g, L):
        """Key for Galois element g at level L: digits j < dnum(L), limbs Q_L u P_{K(L)}.  When L's special-prime
        class K(L) is below the generated class K(ML) (DESIGN.md R-KL) the key of the smaller special modulus
        P_{K(L)} is ksk_j = (-a_j s + e_j + g_j^{(K(L))} s', a_j) with the SAME a_j, e_j restricted to the smaller
        basis: b_j += (P_{K(L)} - P_{K(ML)}) s' on digit j's q-limbs."""
        if g not in self.ksk:
            raise OracleError("MISSING_KEY g=%d" % g)
        ML = self.max_level
        if L > ML:
            raise OracleError("LEVEL_MISMATCH: key generated up to level %d" % ML)
        P = self.P
        ck = (g, L)
        cache = self.__dict__.setdefault("_key_cache", {})
        if ck in cache:
            return cache[ck]
        KL = P.K(L)
        idx = list(range(L)) + list(range(ML, ML + KL))
        out = [np.ascontiguousarray(k[:, idx]) for k in self.ksk[g][: P.dnum(L)]]
        if KL != P.K(ML):
            d = P.P_of(L) - P.P_of(ML)
            for j, kj in enumerate(out):
                lo, hi = P.digit(j, L)
                mods = P.q[lo:hi]
                kj[0][lo:hi] = padd(kj[0][lo:hi], pmul_scalar(self._sp[g][lo:hi], [d % q for q in mods], mods, P.N), mods, P.N)
        cache[ck] = out
        return out


def galois_rot(P, r):
    """Left rotation by r slots is sigma_{5^r mod 2N} (verified by tests)."""
    return pow(5, int(r) % P.n, 2 * P.N)


def galois_conj(P):
    return 2 * P.N - 1


# ------------------------------------------------------------------------------------ enc / dec
def encrypt_sk(P, keys, pt, seed):
    """Secret-key encryption (DESIGN G17): c1 = a (uniform), c0 = -a s + e + m."""
    L, N = pt.L, P.N
    mods = P.q[:L]
    a = sample_uniform(seed, STREAM_ENC_A, mods, list(range(L)), N)
    e = from_signed(sample_cbd21(seed, STREAM_ENC_E, N), mods, N)
    c0 = padd(psub(e, ring_mul(a, keys.s_at(L), mods, N), mods, N), pt.m, mods, N)
    return Ct(np.stack([c0, a]), pt.scale)


def decrypt(P, keys, ct):
    L, N = ct.L, P.N
    mods = P.q[:L]
    s = keys.s_at(L)
    m = padd(ct.c[0], ring_mul(ct.c[1], s, mods, N), mods, N)
    if ct.ncomp == 3:
        m = padd(m, ring_mul(ct.c[2], ring_mul(s, s, mods, N), mods, N), mods, N)
    return Pt(m, ct.scale)


# ------------------------------------------------------------------------------------ key switching (C4)
def modup(P, d, L):
    """ModUp of d (coefficient domain, level L) for every digit j: inside the digit d~ = d, on every other
    modulus t of Q_L u P fast BConv of the digit's limbs.  Returns a list over j of [(L+alpha)][N]."""
    N = P.N
    mods = P.ext_mods(L)
    out = []
    for j in range(P.dnum(L)):
        lo, hi = P.digit(j, L)
        other = [i for i in range(len(mods)) if not lo <= i < hi]
        ext = np.empty((len(mods), N), dtype=np.uint64)
        ext[lo:hi] = d[lo:hi]
        ext[other] = bconv(d[lo:hi], P.q[lo:hi], [mods[i] for i in other], N)
        out.append(ext)
    return out


def ks_inner(P, ext_digits, key, L):
    """(b0, b1) = sum_j d~_j * ksk_j over Q_L u P (ring products via the oracle NTT; the sum is exact)."""
    N = P.N
    mods = P.ext_mods(L)
    acc = [np.zeros((len(mods), N), dtype=np.uint64) for _ in range(2)]
    for j, dj in enumerate(ext_digits):
        djn = ntt(dj, mods, N)
        for c in range(2):
            prod = pmul_pointwise(djn, ntt(key[j][c], mods, N), mods, N)
            acc[c] = padd(acc[c], prod, mods, N)
    return [intt(a, mods, N) for a in acc]


def moddown(P, b, L):
    """ModDown (C4 with DESIGN.md R-MODDOWN): y = the centred residue [b]_P obtained by the rounded fast
    BConv_{P->Q};  out_i = (b_i - y_i) * P^{-1} mod q_i  =  round(b / P)  (SURVEY's floor version leaves
    an error u in [0, K) per coefficient, ~2^-19 relative after a projection -- above the 2^-20 target)."""
    N = P.N
    PK = P.P_of(L)                    # the special modulus of level L (R-KL)
    y = bconv_round(b[L:], P.p[:P.K(L)], P.q[:L], N)
    pinv = [pow(PK % q, -1, q) for q in P.q[:L]]
    return pmul_scalar(psub(b[:L], y, P.q[:L], N), pinv, P.q[:L], N)


def lift_P(P, c, L):
    """P * c in the extended basis Q_L u P (P = P_{K(L)}): (P mod q_i) c_i on the q-limbs, 0 on the p-limbs."""
    N = P.N
    PK = P.P_of(L)
    out = np.zeros((L + P.K(L), N), dtype=np.uint64)
    out[:L] = pmul_scalar(c, [PK % q for q in P.q[:L]], P.q[:L], N)
    return out


def moddown_rescale(P, x, L):
    """Merged ModDown + rescale (DESIGN.md R-LAZY): x over Q_L u P (coefficient form) ->
    round(x / (P q_{L-1})) mod Q_{L-1}, through ONE rounded fast base conversion from the basis
    B' = {q_{L-1}, p_0..p_{K(L)-1}} to Q_{L-1}."""
    N = P.N
    bp = [P.q[L - 1]] + P.p[:P.K(L)]
    rows = np.concatenate([x[L - 1:L], x[L:]])
    y = bconv_round(rows, bp, P.q[:L - 1], N)
    Bp = P.P_of(L) * P.q[L - 1]
    inv = [pow(Bp % q, -1, q) for q in P.q[:L - 1]]
    return pmul_scalar(psub(x[:L - 1], y, P.q[:L - 1], N), inv, P.q[:L - 1], N)


def rotate_hoisted_ext(P, keys, ct, rs):
    """Hoisted rotations WITHOUT ModDown (DESIGN.md R-LAZY): for each r the extended-basis pair
    (P sigma_g(c0) + b0, b1) over Q_L u P, whose ModDown is the ordinary hoisted rotation."""
    L, N = ct.L, P.N
    mods, emods = P.q[:L], P.ext_mods(L)
    ext = modup(P, ct.c[1], L)
    outs = []
    for r in rs:
        g = galois_rot(P, r)
        ext_g = [automorph(dj, g, emods, N) for dj in ext]
        b0, b1 = ks_inner(P, ext_g, keys.key_at(g, L), L)
        c0 = automorph(ct.c[0], g, mods, N)
        outs.append(np.stack([padd(b0, lift_P(P, c0, L), emods, N), b1]))
    return outs


def rotate_ext(P, keys, ct, g):
    """Single (non-hoisted) key switch WITHOUT ModDown: sigma_g then ModUp of sigma_g(c1); returns the
    extended pair (P sigma_g(c0) + b0, b1) over Q_L u P (DESIGN.md R-LAZY)."""
    L, N = ct.L, P.N
    mods, emods = P.q[:L], P.ext_mods(L)
    c0 = automorph(ct.c[0], g, mods, N)
    c1 = automorph(ct.c[1], g, mods, N)
    b0, b1 = ks_inner(P, modup(P, c1, L), keys.key_at(g, L), L)
    return np.stack([padd(b0, lift_P(P, c0, L), emods, N), b1])


def moddown_ext(P, x, L):
    """ModDown of both components of an extended ciphertext [2][L+K][N] -> [2][L][N]."""
    return np.stack([moddown(P, x[c], L) for c in range(2)])


def keyswitch(P, d, key, L):
    b0, b1 = ks_inner(P, modup(P, d, L), key, L)
    return moddown(P, b0, L), moddown(P, b1, L)


def _apply_galois(P, ct, g, keys):
    L, N = ct.L, P.N
    mods = P.q[:L]
    c0 = automorph(ct.c[0], g, mods, N)
    c1 = automorph(ct.c[1], g, mods, N)
    k0, k1 = keyswitch(P, c1, keys.key_at(g, L), L)
    return Ct(np.stack([padd(c0, k0, mods, N), k1]), ct.scale)


def rotate(P, keys, ct, r):
    """Single (non-hoisted) rotation by r slots to the left: sigma_g then KS of sigma_g(c1)."""
    if ct.ncomp != 2:
        raise OracleError("FORMAT: rotate needs a 2-component ciphertext")
    if int(r) % P.n == 0:
        return Ct(ct.c.copy(), ct.scale)        # identity, no key switch
    return _apply_galois(P, ct, galois_rot(P, r), keys)


def conjugate(P, keys, ct):
    return _apply_galois(P, ct, galois_conj(P), keys)


def rotate_hoisted(P, keys, ct, rs):
    """Hoisted batch (C4): ModUp(c1) ONCE, then sigma_g of every extended digit, inner product with the
    key of sigma_g(s), ModDown, plus sigma_g(c0).  Bits differ from `rotate` (sigma does not commute
    bitwise with fast BConv)."""
    L, N = ct.L, P.N
    mods, emods = P.q[:L], P.ext_mods(L)
    ext = modup(P, ct.c[1], L)
    outs = []
    for r in rs:
        if int(r) % P.n == 0:
            outs.append(Ct(ct.c.copy(), ct.scale))
            continue
        g = galois_rot(P, r)
        ext_g = [automorph(dj, g, emods, N) for dj in ext]
        b0, b1 = ks_inner(P, ext_g, keys.key_at(g, L), L)
        c0 = automorph(ct.c[0], g, mods, N)
        outs.append(Ct(np.stack([padd(c0, moddown(P, b0, L), mods, N), moddown(P, b1, L)]), ct.scale))
    return outs


def relinearize(P, keys, ct):
    if ct.ncomp != 3:
        raise OracleError("FORMAT: relinearize needs 3 components")
    L, N = ct.L, P.N
    mods = P.q[:L]
    k0, k1 = keyswitch(P, ct.c[2], keys.key_at(0, L), L)
    return Ct(np.stack([padd(ct.c[0], k0, mods, N), padd(ct.c[1], k1, mods, N)]), ct.scale)


def relinearize_ext(P, keys, ct):
    """Relinearisation WITHOUT its ModDown (DESIGN.md R-RELRS, the R-LAZY idea applied to relin): the extended
    pair (P d0 + b0, P d1 + b1) over Q_L u P, (b0, b1) = the inner product of ModUp(d2) with the relinearisation
    key.  Its ModDown is relinearize(); moddown_rescale() of it is relin followed by rescale, rounded once."""
    if ct.ncomp != 3:
        raise OracleError("FORMAT: relinearize needs 3 components")
    L, N = ct.L, P.N
    emods = P.ext_mods(L)
    b0, b1 = ks_inner(P, modup(P, ct.c[2], L), keys.key_at(0, L), L)
    return np.stack([padd(b0, lift_P(P, ct.c[0], L), emods, N), padd(b1, lift_P(P, ct.c[1], L), emods, N)])


# ------------------------------------------------------------------------------------ arithmetic
def add(P, a, b):
    if a.scale != b.scale:
        raise OracleError("SCALE_MISMATCH")
    if a.L != b.L:
        raise OracleError("LEVEL_MISMATCH")
    nc = max(a.ncomp, b.ncomp)
    mods = P.q[:a.L]
    out = np.zeros((nc, a.L, P.N), dtype=np.uint64)
    for c in range(nc):
        x = a.c[c] if c < a.ncomp else np.zeros_like(a.c[0])
        y = b.c[c] if c < b.ncomp else np.zeros_like(a.c[0])
        out[c] = padd(x, y, mods, P.N)
    return Ct(out, a.scale)


def sub(P, a, b):
    if a.scale != b.scale:
        raise OracleError("SCALE_MISMATCH")
    if a.L != b.L or a.ncomp != b.ncomp:
        raise OracleError("LEVEL_MISMATCH")
    mods = P.q[:a.L]
    return Ct(np.stack([psub(a.c[c], b.c[c], mods, P.N) for c in range(a.ncomp)]), a.scale)


def mul_i(P, ct):
    """x i  ==  multiply by the monomial X^{N/2} (exact, no key, no level)."""
    mods = P.q[:ct.L]
    return Ct(np.stack([mul_monomial_half(ct.c[c], mods, P.N) for c in range(ct.ncomp)]), ct.scale)


def complexify(P, re, im):
    """Boundary wrapper: re + i*im, i = X^{N/2}."""
    return add(P, re, mul_i(P, im))


def ptmul(P, ct, pt):
    """ct (.) pt, no rescale.  Scale = scale_ct * scale_pt."""
    if ct.L != pt.L:
        raise OracleError("LEVEL_MISMATCH")
    mods = P.q[:ct.L]
    ptn = ntt(pt.m, mods, P.N)
    out = np.stack([intt(pmul_pointwise(ntt(ct.c[c], mods, P.N), ptn, mods, P.N), mods, P.N) for c in range(ct.ncomp)])
    return Ct(out, ct.scale * pt.scale)


def tensor(P, a, b):
    """ct x ct without relinearisation: (a0 b0, a0 b1 + a1 b0, a1 b1).  Scale = product."""
    if a.L != b.L:
        raise OracleError("LEVEL_MISMATCH")
    mods, N = P.q[:a.L], P.N
    a0, a1 = ntt(a.c[0], mods, N), ntt(a.c[1], mods, N)
    b0, b1 = ntt(b.c[0], mods, N), ntt(b.c[1], mods, N)
    d0 = pmul_pointwise(a0, b0, mods, N)
    d1 = padd(pmul_pointwise(a0, b1, mods, N), pmul_pointwise(a1, b0, mods, N), mods, N)
    d2 = pmul_pointwise(a1, b1, mods, N)
    return Ct(np.stack([intt(d, mods, N) for d in (d0, d1, d2)]), a.scale * b.scale)


def rescale(P, ct):
    """Divide-and-round by the last prime (C5); scale <- scale / q_last."""
    if ct.L <= 1:
        raise OracleError("LEVEL_EXHAUSTED")
    mods = P.q[:ct.L]
    return Ct(np.stack([rescale_poly(ct.c[c], mods, P.N) for c in range(ct.ncomp)]), ct.scale / float(mods[-1]))


def mod_drop(P, ct, L):
    """ModSwitchToNext repeated: delete the last limbs, scale unchanged."""
    if L < 1 or L > ct.L:
        raise OracleError("LEVEL_MISMATCH")
    return Ct(np.ascontiguousarray(ct.c[:, :L]), ct.scale)
