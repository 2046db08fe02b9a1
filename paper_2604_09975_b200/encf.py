"""Thin Python binding of libencf (include/encf.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch is used for device memory and
streams.  There is no CPU fallback: importing this module on a machine without the built
libencf.so raises, and every call raises EncfError on a non-OK status.
"""
import ctypes
import json
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("ENCF_LIB_OVERRIDE") or os.path.join(_HERE, "libencf.so")   # override: kernel-variant experiments only
PARAMS_DIR = os.path.join(os.path.dirname(_HERE), "params")

if not os.path.exists(_SO):
    raise ImportError("libencf.so is not built (run __graft_entry__.build()); there is no CPU fallback")

_lib = ctypes.CDLL(_SO)
_p, _i32, _u32, _u64, _f64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t


class CT(ctypes.Structure):
    _fields_ = [("data", _p), ("n_comp", _i32), ("n_limbs", _i32), ("scale", _f64), ("ntt", _i32)]


class PT(ctypes.Structure):
    _fields_ = [("data", _p), ("n_limbs", _i32), ("scale", _f64), ("ntt", _i32)]


class Params(ctypes.Structure):
    _fields_ = [("N", _i32), ("L", _i32), ("K", _i32), ("alpha", _i32), ("q", _p), ("p", _p), ("K_of_level", _p)]


class Counters(ctypes.Structure):
    _fields_ = [(n, _u64) for n in ("keyswitch", "modup", "limb_ntt", "ptmul_terms", "ctmul", "kernel_launches", "alg_bytes",
                                       "limb_ntt_fp64")]


class MaskDesc(ctypes.Structure):
    _fields_ = [(n, _i32) for n in ("m", "r0", "r1", "s0", "sstride", "scount", "level", "ext")]


_SIG = {
    "encf_ctx_create": [ctypes.POINTER(Params), ctypes.c_int, ctypes.POINTER(_p)],
    "encf_ctx_destroy": [_p],
    "encf_stats": [_p, ctypes.POINTER(Counters)],
    "encf_stats_reset": [_p],
    "encf_keygen": [_p, _u64, _p, _i32, _u32, _i32, ctypes.POINTER(_p), _p],
    "encf_keys_destroy": [_p],
    "encf_keys_export": [_p, _p, _i32, _u32, _p, _p],
    "encf_keys_size": [_p, _p, _i32, ctypes.POINTER(_sz)],
    "encf_encrypt_sk": [_p, _p, ctypes.POINTER(PT), _u64, ctypes.POINTER(CT), _p],
    "encf_decrypt": [_p, _p, ctypes.POINTER(CT), ctypes.POINTER(PT), _p],
    "encf_encode": [_p, _p, _p, _i32, _i32, _f64, ctypes.POINTER(PT), _p],
    "encf_decode": [_p, ctypes.POINTER(PT), _p, _p, _p],
    "encf_poly_to_ntt": [_p, _p, _i32, _i32, _p],
    "encf_poly_from_ntt": [_p, _p, _i32, _i32, _p],
    "encf_add": [_p, ctypes.POINTER(CT), ctypes.POINTER(CT), ctypes.POINTER(CT), _p],
    "encf_sub": [_p, ctypes.POINTER(CT), ctypes.POINTER(CT), ctypes.POINTER(CT), _p],
    "encf_mul_i": [_p, ctypes.POINTER(CT), ctypes.POINTER(CT), _p],
    "encf_ptmul": [_p, ctypes.POINTER(CT), ctypes.POINTER(PT), ctypes.POINTER(CT), _p],
    "encf_tensor": [_p, ctypes.POINTER(CT), ctypes.POINTER(CT), ctypes.POINTER(CT), _p],
    "encf_relinearize": [_p, _p, ctypes.POINTER(CT), ctypes.POINTER(CT), _p],
    "encf_rotate": [_p, _p, ctypes.POINTER(CT), _i32, ctypes.POINTER(CT), _p],
    "encf_rotate_hoisted": [_p, _p, ctypes.POINTER(CT), _p, _i32, _p, _p],
    "encf_conjugate": [_p, _p, ctypes.POINTER(CT), ctypes.POINTER(CT), _p],
    "encf_decomplexify": [_p, _p, _p, _i32, _p, _p],
    "encf_export_c2m_many": [_p, _p, _i32, _i32, _u64, _u64, _p, _p, _p],
    "encf_export_c2m_many_dev": [_p, _p, _i32, _i32, _p, _p, _p, _p],
    "encf_rescale": [_p, ctypes.POINTER(CT), ctypes.POINTER(CT), _p],
    "encf_mod_drop": [_p, ctypes.POINTER(CT), _i32, ctypes.POINTER(CT), _p],
    "encf_complexify": [_p, ctypes.POINTER(CT), ctypes.POINTER(CT), ctypes.POINTER(CT), _p],
    "encf_complexify_many": [_p, _p, _p, _i32, _p, _p],
    "encf_mask_put": [_p, ctypes.POINTER(MaskDesc), _p],
    "encf_mask_clear": [_p],
    "encf_proj_plan_create": [_p, _i32, _i32, _i32, _i32, _i32, _u32, ctypes.POINTER(_p)],
    "encf_proj_plan_destroy": [_p],
    "encf_proj_plan_info": [_p, _p],
    "encf_proj_galois": [_p, _p, _p, _i32, ctypes.POINTER(_i32)],
    "encf_proj_weights_size": [_p, _i32, ctypes.POINTER(_sz)],
    "encf_proj_encode_weights": [_p, _p, _p, _i32, _p, _p],
    "encf_proj_encode_weights_complex": [_p, _p, _p, _p, _i32, _p, _p],
    "encf_pt_ct_matmul": [_p, _p, _p, _p, _p, _f64, _i32, _i32, _u32, _p, _p],
    "encf_pt_ct_matmul_finalize": [_p, _p, _p, _p, _i32, _i32, _p, _p],
    "encf_attn_plan_create": [_p, _i32, _i32, _i32, _i32, _i32, _i32, ctypes.POINTER(_p)],
    "encf_attn_plan_destroy": [_p],
    "encf_attn_plan_info": [_p, _p],
    "encf_attn_galois": [_p, _p, _p, _i32, ctypes.POINTER(_i32)],
    "encf_ct_ct_attn_score": [_p, _p, _p, _p, _p, _i32, _i32, _p, _p],
    "encf_attn_export_stream": [_p, _p, _p, _p, _p, _p],
    "encf_ct_ct_attn_value": [_p, _p, _p, _p, _p, _p, _p],
    "encf_ct_ct_attn_value_partial": [_p, _p, _p, _p, _p, _i32, _i32, _p, _p],
    "encf_attn_value_finalize": [_p, _p, _p, _i32, _p, _p],
    "encf_rotfirst": [_p, _p, ctypes.POINTER(CT), _i32, _p, _i32, _i32, _p, _p],
    "encf_psi": [_p, _p, ctypes.POINTER(CT), _i32, _p, _i32, _p, _p],
    "encf_l_conv": [_p, _i32, _i32, _f64, _f64, ctypes.POINTER(_i32)],
    "encf_export_c2m": [_p, ctypes.POINTER(CT), _i32, _u64, _u64, ctypes.POINTER(CT), _p, _p],
    "encf_mod_reduce": [_p, _p, _i32, _i32, _p],
    "encf_mod_reduce_ext": [_p, _p, _i32, _i32, _p],
    "encf_ring2field_local": [_p, _p, _i32, _i32, _i32, _p, _p],
    "encf_field2ring_local": [_p, _p, _i32, _p, _p],
    "encf_import_m2c": [_p, ctypes.POINTER(CT), ctypes.POINTER(PT), ctypes.POINTER(CT), _p],
    "encf_gelu_preeval": [_p, _p, _p, ctypes.c_int32, _p, _p, _p, _p],
    "encf_repack_rma": [_p, _p, _p, ctypes.c_int32, ctypes.c_int32, _p, _p],
    "encf_profile_enable": [_p, ctypes.c_char_p],
    "encf_profile_read": [_p, ctypes.c_char_p, ctypes.POINTER(_f64), ctypes.POINTER(_u64), ctypes.POINTER(_u64)],
    "encf_profile_peek": [_p, ctypes.c_char_p, ctypes.POINTER(_f64), ctypes.POINTER(_u64), ctypes.POINTER(_u64)],
}
for _name, _args in _SIG.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = ctypes.c_int
_lib.encf_status_string.restype = ctypes.c_char_p
_lib.encf_status_string.argtypes = [ctypes.c_int]
_lib.encf_last_error.restype = ctypes.c_char_p
_lib.encf_galois_rot.restype = _u32
_lib.encf_galois_rot.argtypes = [_p, _i32]
_lib.encf_galois_conj.restype = _u32
_lib.encf_galois_conj.argtypes = [_p]

PROJ_DECOMPLEXIFY = 1
PROJ_FINALIZE = 2
PROJ_REAL_INPUT = 4
PROJ_W_SHARD = 8
KEY_RELIN = 1


class EncfError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        super().__init__("%s: %s (%s)" % (where, _lib.encf_status_string(code).decode(), _lib.encf_last_error().decode()))


def _chk(code, where):
    if code != 0:
        raise EncfError(code, where)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _u64_host(xs):
    return np.ascontiguousarray(np.array([int(x) for x in xs], dtype=np.uint64))


class Ciphertext:
    """Device ciphertext [comp][limb][N] (torch int64 storage holding uint64 words)."""

    def __init__(self, data, n_comp, n_limbs, scale, ntt):
        self.data, self.n_comp, self.n_limbs, self.scale, self.ntt = data, n_comp, n_limbs, float(scale), int(ntt)

    def _c(self):
        return CT(self.data.data_ptr(), self.n_comp, self.n_limbs, self.scale, self.ntt)

    def _update(self, c):
        N = self.data.numel() // (self.n_comp * self.n_limbs)
        self.n_comp, self.n_limbs, self.scale, self.ntt = c.n_comp, c.n_limbs, c.scale, c.ntt
        if self.data.numel() > self.n_comp * self.n_limbs * N:     # the library wrote fewer limbs than allocated
            self.data = self.data[: self.n_comp * self.n_limbs * N]
        return self

    @property
    def L(self):
        return self.n_limbs


class Plaintext:
    def __init__(self, data, n_limbs, scale, ntt):
        self.data, self.n_limbs, self.scale, self.ntt = data, n_limbs, float(scale), int(ntt)

    def _p(self):
        return PT(self.data.data_ptr(), self.n_limbs, self.scale, self.ntt)


class Context:
    def __init__(self, params="P16", device=0):
        path = params if str(params).endswith(".json") else os.path.join(PARAMS_DIR, str(params).lower() + ".json")
        with open(path) as f:
            d = json.load(f)
        self.N, self.n = int(d["N"]), int(d["N"]) // 2
        self.q = [int(x) for x in d["q"]]
        self.p = [int(x) for x in d["p"]]
        self.alpha = int(d["alpha"])
        self.L = len(self.q)
        self.device = torch.device("cuda", device)
        qa, pa = _u64_host(self.q), _u64_host(self.p)
        # K(L): special primes of a key switch at level L (DESIGN.md R-KL); absent = all at every level
        self.K_of_level = [int(k) for k in d.get("K_of_level", [len(self.p)] * self.L)]
        ka = np.ascontiguousarray(np.array(self.K_of_level, dtype=np.int32))
        self._keep = (qa, pa, ka)
        prm = Params(self.N, self.L, len(self.p), self.alpha, qa.ctypes.data, pa.ctypes.data, ka.ctypes.data)
        h = _p()
        torch.cuda.init()
        _chk(_lib.encf_ctx_create(ctypes.byref(prm), device, ctypes.byref(h)), "ctx_create")
        self.h = h

    def K(self, L):
        """Special primes of a key switch at level L."""
        return self.K_of_level[L - 1]

    def ext_limbs(self, L):
        """Limbs of an extended-basis object at level L (L + K(L))."""
        return L + self.K(L)

    def level_of_ext(self, nl):
        """The level L of an extended-basis object with nl = L + K(L) limbs."""
        for L in range(1, self.L + 1):
            if L + self.K(L) == nl:
                return L
        raise ValueError("no level has %d extended limbs" % nl)

    def close(self):
        if self.h:
            _lib.encf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- memory
    def empty_ct(self, L, n_comp=2, scale=1.0):
        return Ciphertext(torch.empty(n_comp * L * self.N, dtype=torch.int64, device=self.device), n_comp, L, scale, 1)

    def ct_from_host(self, words, scale, ntt=0):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        t = torch.from_numpy(w.view(np.int64).reshape(-1).copy()).to(self.device)
        return Ciphertext(t, w.shape[0], w.shape[1], scale, ntt)

    def pt_from_host(self, words, scale, ntt=0):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        t = torch.from_numpy(w.view(np.int64).reshape(-1).copy()).to(self.device)
        return Plaintext(t, w.shape[0], scale, ntt)

    def to_host(self, obj, coeff=True):
        """Copy to host as uint64 [comp][L][N] (ciphertext) or [L][N] (plaintext), coefficient domain."""
        d = obj.data.clone()
        ncomp = obj.n_comp if isinstance(obj, Ciphertext) else 1
        if coeff and obj.ntt:
            _chk(_lib.encf_poly_from_ntt(self.h, d.data_ptr(), ncomp, obj.n_limbs, _stream()), "from_ntt")
        a = d.cpu().numpy().view(np.uint64)
        return a.reshape(ncomp, obj.n_limbs, self.N) if isinstance(obj, Ciphertext) else a.reshape(obj.n_limbs, self.N)

    def to_ntt(self, obj):
        if not obj.ntt:
            ncomp = obj.n_comp if isinstance(obj, Ciphertext) else 1
            _chk(_lib.encf_poly_to_ntt(self.h, obj.data.data_ptr(), ncomp, obj.n_limbs, _stream()), "to_ntt")
            obj.ntt = 1
        return obj

    def from_ntt(self, obj):
        if obj.ntt:
            ncomp = obj.n_comp if isinstance(obj, Ciphertext) else 1
            _chk(_lib.encf_poly_from_ntt(self.h, obj.data.data_ptr(), ncomp, obj.n_limbs, _stream()), "from_ntt")
            obj.ntt = 0
        return obj

    def poly_to_ntt(self, tensor, n_polys, n_limbs):
        _chk(_lib.encf_poly_to_ntt(self.h, tensor.data_ptr(), n_polys, n_limbs, _stream()), "to_ntt")

    def stats(self):
        c = Counters()
        _chk(_lib.encf_stats(self.h, ctypes.byref(c)), "stats")
        return {n: getattr(c, n) for n, _ in Counters._fields_}

    def stats_reset(self):
        _chk(_lib.encf_stats_reset(self.h), "stats_reset")

    def profile(self, which):
        """which: kernel name to time with CUDA events, "*" for all, None to disable."""
        _chk(_lib.encf_profile_enable(self.h, which.encode() if which else None), "profile_enable")

    def profile_read(self, kernel, keep=False):
        """(ms, launches, algorithmic bytes) of the recorded launches of `kernel`; keep=True: do not forget them
        (graph replays re-record the same events)."""
        ms, n, by = _f64(), _u64(), _u64()
        f = _lib.encf_profile_peek if keep else _lib.encf_profile_read
        _chk(f(self.h, kernel.encode(), ctypes.byref(ms), ctypes.byref(n), ctypes.byref(by)), "profile_read")
        return ms.value, n.value, by.value

    def galois_rot(self, steps):
        return int(_lib.encf_galois_rot(self.h, int(steps)))

    def galois_conj(self):
        return int(_lib.encf_galois_conj(self.h))

    # -------------------------------------------------------------- keys / enc / dec
    def keygen(self, seed, galois=(), relin=False, max_level=None):
        g = np.ascontiguousarray(np.array(sorted(set(int(x) for x in galois)), dtype=np.uint32))
        h = _p()
        _chk(_lib.encf_keygen(self.h, seed, g.ctypes.data if len(g) else None, len(g), KEY_RELIN if relin else 0,
                              max_level or self.L, ctypes.byref(h), _stream()), "keygen")
        return Keys(self, h, max_level or self.L)

    def encrypt(self, keys, pt, seed):
        out = self.empty_ct(pt.n_limbs)
        c = out._c()
        _chk(_lib.encf_encrypt_sk(self.h, keys.h, ctypes.byref(pt._p()), seed, ctypes.byref(c), _stream()), "encrypt")
        return out._update(c)

    def decrypt(self, keys, ct):
        out = Plaintext(torch.empty(ct.n_limbs * self.N, dtype=torch.int64, device=self.device), ct.n_limbs, ct.scale, 1)
        p = out._p()
        _chk(_lib.encf_decrypt(self.h, keys.h, ctypes.byref(ct._c()), ctypes.byref(p), _stream()), "decrypt")
        out.n_limbs, out.scale, out.ntt = p.n_limbs, p.scale, p.ntt
        return out

    def encode(self, z, scale, L):
        z = np.asarray(z, dtype=np.complex128).reshape(-1)
        re, im = np.ascontiguousarray(z.real), np.ascontiguousarray(z.imag)
        out = Plaintext(torch.empty(L * self.N, dtype=torch.int64, device=self.device), L, scale, 1)
        p = out._p()
        _chk(_lib.encf_encode(self.h, re.ctypes.data, im.ctypes.data, len(z), L, float(scale), ctypes.byref(p), _stream()), "encode")
        return out

    def decode(self, pt):
        re, im = np.empty(self.n), np.empty(self.n)
        _chk(_lib.encf_decode(self.h, ctypes.byref(pt._p()), re.ctypes.data, im.ctypes.data, _stream()), "decode")
        return re + 1j * im

    # -------------------------------------------------------------- homomorphic ops
    def add(self, a, b, sub=False):
        out = self.empty_ct(a.n_limbs, a.n_comp)
        c = out._c()
        f = _lib.encf_sub if sub else _lib.encf_add
        _chk(f(self.h, ctypes.byref(a._c()), ctypes.byref(b._c()), ctypes.byref(c), _stream()), "add")
        return out._update(c)

    def mul_i(self, a):
        out = self.empty_ct(a.n_limbs, a.n_comp)
        c = out._c()
        _chk(_lib.encf_mul_i(self.h, ctypes.byref(a._c()), ctypes.byref(c), _stream()), "mul_i")
        return out._update(c)

    def ptmul(self, a, pt):
        out = self.empty_ct(a.n_limbs, a.n_comp)
        c = out._c()
        _chk(_lib.encf_ptmul(self.h, ctypes.byref(a._c()), ctypes.byref(pt._p()), ctypes.byref(c), _stream()), "ptmul")
        return out._update(c)

    def tensor(self, a, b):
        out = self.empty_ct(a.n_limbs, 3)
        c = out._c()
        _chk(_lib.encf_tensor(self.h, ctypes.byref(a._c()), ctypes.byref(b._c()), ctypes.byref(c), _stream()), "tensor")
        return out._update(c)

    def relinearize(self, keys, a):
        out = self.empty_ct(a.n_limbs, 2)
        c = out._c()
        _chk(_lib.encf_relinearize(self.h, keys.h, ctypes.byref(a._c()), ctypes.byref(c), _stream()), "relinearize")
        return out._update(c)

    def rotate(self, keys, a, steps):
        out = self.empty_ct(a.n_limbs, 2)
        c = out._c()
        _chk(_lib.encf_rotate(self.h, keys.h, ctypes.byref(a._c()), int(steps), ctypes.byref(c), _stream()), "rotate")
        return out._update(c)

    def rotate_hoisted(self, keys, a, steps):
        outs = [self.empty_ct(a.n_limbs, 2) for _ in steps]
        arr = (CT * len(steps))(*[o._c() for o in outs])
        st = np.ascontiguousarray(np.array(steps, dtype=np.int32))
        _chk(_lib.encf_rotate_hoisted(self.h, keys.h, ctypes.byref(a._c()), st.ctypes.data, len(steps), ctypes.cast(arr, _p), _stream()), "rotate_hoisted")
        return [o._update(arr[i]) for i, o in enumerate(outs)]

    def rotfirst(self, keys, a, L_slots, taus, m):
        """RotFirst_{L_slots}(a; tau) for every tau (Alg A.3), one hoisted batch; outputs one level down."""
        outs = [self.empty_ct(a.n_limbs - 1, 2) for _ in taus]
        arr = (CT * len(taus))(*[o._c() for o in outs])
        tt = np.ascontiguousarray(np.array(taus, dtype=np.int32))
        _chk(_lib.encf_rotfirst(self.h, keys.h, ctypes.byref(a._c()), L_slots, tt.ctypes.data, len(taus), m,
                                ctypes.cast(arr, _p), _stream()), "rotfirst")
        return [o._update(arr[i]) for i, o in enumerate(outs)]

    def psi(self, keys, a, m, ts):
        """Psi^t(a) for every t (Alg A.2), one hoisted batch; outputs one level down."""
        outs = [self.empty_ct(a.n_limbs - 1, 2) for _ in ts]
        arr = (CT * len(ts))(*[o._c() for o in outs])
        tt = np.ascontiguousarray(np.array(ts, dtype=np.int32))
        _chk(_lib.encf_psi(self.h, keys.h, ctypes.byref(a._c()), m, tt.ctypes.data, len(ts), ctypes.cast(arr, _p), _stream()), "psi")
        return [o._update(arr[i]) for i, o in enumerate(outs)]

    def conjugate(self, keys, a):
        out = self.empty_ct(a.n_limbs, 2)
        c = out._c()
        _chk(_lib.encf_conjugate(self.h, keys.h, ctypes.byref(a._c()), ctypes.byref(c), _stream()), "conjugate")
        return out._update(c)

    def decomplexify(self, keys, cts):
        """[c + conj(c) (scale x 2) for c in cts] in one batched conjugation (encf_decomplexify)."""
        n = len(cts)
        ins = (CT * n)(*[c._c() for c in cts])
        outs_py = [self.empty_ct(c.n_limbs, 2) for c in cts]
        outs = (CT * n)(*[o._c() for o in outs_py])
        _chk(_lib.encf_decomplexify(self.h, keys.h, ctypes.cast(ins, _p), n, ctypes.cast(outs, _p), _stream()), "decomplexify")
        return [o._update(outs[i]) for i, o in enumerate(outs_py)]

    def rescale(self, a):
        out = self.empty_ct(max(a.n_limbs - 1, 1), a.n_comp)
        c = out._c()
        _chk(_lib.encf_rescale(self.h, ctypes.byref(a._c()), ctypes.byref(c), _stream()), "rescale")
        return out._update(c)

    def mod_drop(self, a, L):
        out = self.empty_ct(L, a.n_comp)
        c = out._c()
        _chk(_lib.encf_mod_drop(self.h, ctypes.byref(a._c()), int(L), ctypes.byref(c), _stream()), "mod_drop")
        return out._update(c)

    def complexify(self, re, im):
        out = self.empty_ct(re.n_limbs, 2)
        c = out._c()
        _chk(_lib.encf_complexify(self.h, ctypes.byref(re._c()), ctypes.byref(im._c()), ctypes.byref(c), _stream()), "complexify")
        return out._update(c)

    def complexify_many(self, res, ims):
        """[re + i im for (re, im) in zip(res, ims)] in batched launches (encf_complexify_many)."""
        n = len(res)
        a = (CT * n)(*[x._c() for x in res])
        b = (CT * n)(*[x._c() for x in ims])
        outs_py = [self.empty_ct(x.n_limbs, x.n_comp) for x in res]
        outs = (CT * n)(*[o._c() for o in outs_py])
        _chk(_lib.encf_complexify_many(self.h, ctypes.cast(a, _p), ctypes.cast(b, _p), n, ctypes.cast(outs, _p), _stream()),
             "complexify_many")
        return [o._update(outs[i]) for i, o in enumerate(outs_py)]

    def mask_put(self, desc, m, level, coeffs, ext=False):
        r0, r1, s0, ss, sc = desc
        d = MaskDesc(m, r0, r1, s0, ss, sc, level, 1 if ext else 0)
        w = np.ascontiguousarray(coeffs, dtype=np.uint64)
        _chk(_lib.encf_mask_put(self.h, ctypes.byref(d), w.ctypes.data), "mask_put")

    def mask_clear(self):
        _chk(_lib.encf_mask_clear(self.h), "mask_clear")

    def l_conv(self, ell=43, sigma=40, scale=2.0 ** 40, B_max=1.0):
        out = _i32()
        _chk(_lib.encf_l_conv(self.h, ell, sigma, scale, B_max, ctypes.byref(out)), "l_conv")
        return out.value

    def export_c2m(self, ct, L_conv, mask_seed, stream_id):
        masked = self.empty_ct(L_conv, 2)
        share = torch.empty(L_conv * self.N, dtype=torch.int64, device=self.device)
        c = masked._c()
        _chk(_lib.encf_export_c2m(self.h, ctypes.byref(ct._c()), int(L_conv), int(mask_seed), int(stream_id), ctypes.byref(c),
                                  share.data_ptr(), _stream()), "export_c2m")
        return masked._update(c), share

    def export_c2m_many(self, cts, L_conv, mask_seed, stream_id0):
        """Batched encf_export_c2m: ciphertext i with stream id stream_id0 + i.  Returns [(masked ct, share)]
        as views into two contiguous device buffers.  mask_seed may also be a DEVICE int64 tensor [2] = (seed,
        stream id base) (encf_export_c2m_many_dev: read at run time, so a graph replay sees its current value; then
        stream_id0 is ignored)."""
        n, N = len(cts), self.N
        masked = torch.empty(n * 2 * L_conv * N, dtype=torch.int64, device=self.device)
        shares = torch.empty(n * L_conv * N, dtype=torch.int64, device=self.device)
        ins = (CT * n)(*[c._c() for c in cts])
        if isinstance(mask_seed, torch.Tensor):
            _chk(_lib.encf_export_c2m_many_dev(self.h, ctypes.cast(ins, _p), n, int(L_conv), mask_seed.data_ptr(),
                                               masked.data_ptr(), shares.data_ptr(), _stream()), "export_c2m_many_dev")
        else:
            _chk(_lib.encf_export_c2m_many(self.h, ctypes.cast(ins, _p), n, int(L_conv), int(mask_seed), int(stream_id0),
                                           masked.data_ptr(), shares.data_ptr(), _stream()), "export_c2m_many")
        w = 2 * L_conv * N
        return [(Ciphertext(masked[i * w:(i + 1) * w], 2, L_conv, cts[i].scale, 0), shares[i * L_conv * N:(i + 1) * L_conv * N])
                for i in range(n)]

    def mod_reduce(self, tensor, n_polys, n_limbs):
        _chk(_lib.encf_mod_reduce(self.h, tensor.data_ptr(), n_polys, n_limbs, _stream()), "mod_reduce")

    def ring2field_local(self, mprime_words, party, ell_sigma, L):
        """mprime_words: device int64 tensor [N][2] (lo, hi).  Returns a coefficient-form Plaintext [L][N]."""
        out = Plaintext(torch.empty(L * self.N, dtype=torch.int64, device=self.device), L, 1.0, 0)
        _chk(_lib.encf_ring2field_local(self.h, mprime_words.data_ptr(), party, ell_sigma, L, out.data.data_ptr(), _stream()), "ring2field")
        return out

    def field2ring_local(self, share_words, ell):
        out = torch.empty(self.N, dtype=torch.int64, device=self.device)
        _chk(_lib.encf_field2ring_local(self.h, share_words.data_ptr(), ell, out.data_ptr(), _stream()), "field2ring")
        return out

    def import_m2c(self, ct, share_pt):
        out = self.empty_ct(ct.n_limbs, 2)
        c = out._c()
        _chk(_lib.encf_import_m2c(self.h, ctypes.byref(ct._c()), ctypes.byref(share_pt._p()), ctypes.byref(c), _stream()), "import_m2c")
        return out._update(c)

    def repack_rma(self, keys, xs, m):
        """w/o-SCP ablation: Halevi-Shoup RMA repack of each ciphertext (one level consumed)."""
        outs = [self.empty_ct(x.n_limbs - 1) for x in xs]
        xa = (CT * len(xs))(*[x._c() for x in xs])
        oa = (CT * len(xs))(*[o._c() for o in outs])
        _chk(_lib.encf_repack_rma(self.h, keys.h, ctypes.cast(xa, _p), len(xs), int(m), ctypes.cast(oa, _p), _stream()),
             "repack_rma")
        return [o._update(oa[i]) for i, o in enumerate(outs)]

    def gelu_preeval(self, keys, xs, coef):
        """Alg 5 steps 1-3 on complex ciphertexts xs (one level and scale): returns (F0^C list, F1^C list) at L - 3."""
        L = xs[0].n_limbs
        f0 = [self.empty_ct(L - 3) for _ in xs]
        f1 = [self.empty_ct(L - 3) for _ in xs]
        xa = (CT * len(xs))(*[x._c() for x in xs])
        a0 = (CT * len(xs))(*[o._c() for o in f0])
        a1 = (CT * len(xs))(*[o._c() for o in f1])
        cf = np.ascontiguousarray(np.array(coef, dtype=np.float64))
        _chk(_lib.encf_gelu_preeval(self.h, keys.h, ctypes.cast(xa, _p), len(xs), cf.ctypes.data, ctypes.cast(a0, _p),
                                    ctypes.cast(a1, _p), _stream()), "gelu_preeval")
        return [o._update(a0[i]) for i, o in enumerate(f0)], [o._update(a1[i]) for i, o in enumerate(f1)]

    def mod_reduce_ext(self, tensor, n_polys, L):
        _chk(_lib.encf_mod_reduce_ext(self.h, tensor.data_ptr(), n_polys, L, _stream()), "mod_reduce_ext")


class Keys:
    def __init__(self, ctx, h, max_level):
        self.ctx, self.h, self.max_level = ctx, h, max_level

    def close(self):
        if self.h:
            _lib.encf_keys_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self, which, galois=0):
        sz = _sz()
        _chk(_lib.encf_keys_size(self.ctx.h, self.h, which, ctypes.byref(sz)), "keys_size")
        t = torch.empty(sz.value, dtype=torch.int64, device=self.ctx.device)
        _chk(_lib.encf_keys_export(self.ctx.h, self.h, which, int(galois), t.data_ptr(), _stream()), "keys_export")
        return t.cpu().numpy().view(np.uint64)


class ProjPlan:
    def __init__(self, ctx, m, d_in, d_out, C=0, N1=0, decomplexify=True, real_input=False):
        """real_input=True: fused-QK plan, real inputs x^(g), complex weights, no decomplexify."""
        h = _p()
        flags = PROJ_REAL_INPUT if real_input else (PROJ_DECOMPLEXIFY if decomplexify else 0)
        _chk(_lib.encf_proj_plan_create(ctx.h, m, d_in, d_out, C, N1, flags, ctypes.byref(h)), "proj_plan")
        self.ctx, self.h = ctx, h
        info = np.zeros(7, dtype=np.int32)
        _chk(_lib.encf_proj_plan_info(h, info.ctypes.data), "proj_plan_info")
        self.C, self.G, self.U, self.B_out, self.N1, self.N2, self.n_pt = [int(x) for x in info]
        self.m = m

    def __del__(self):
        try:
            _lib.encf_proj_plan_destroy(self.h)
        except Exception:
            pass

    def galois(self):
        n = _i32()
        buf = np.zeros(4096, dtype=np.uint32)
        _chk(_lib.encf_proj_galois(self.ctx.h, self.h, buf.ctypes.data, len(buf), ctypes.byref(n)), "proj_galois")
        return [int(x) for x in buf[:n.value]]

    def weights_bytes(self, L):
        sz = _sz()
        _chk(_lib.encf_proj_weights_size(self.h, L, ctypes.byref(sz)), "weights_size")
        return sz.value

    def encode_weights(self, Wbar, L):
        W = np.ascontiguousarray(Wbar, dtype=np.float64)
        t = torch.empty(self.weights_bytes(L) // 8, dtype=torch.int64, device=self.ctx.device)
        _chk(_lib.encf_proj_encode_weights(self.ctx.h, self.h, W.ctypes.data, L, t.data_ptr(), _stream()), "encode_weights")
        return t

    def encode_weights_complex(self, Wre, Wim, L):
        Wr = np.ascontiguousarray(Wre, dtype=np.float64)
        Wi = np.ascontiguousarray(Wim, dtype=np.float64) if Wim is not None else None
        t = torch.empty(self.weights_bytes(L) // 8, dtype=torch.int64, device=self.ctx.device)
        _chk(_lib.encf_proj_encode_weights_complex(self.ctx.h, self.h, Wr.ctypes.data, Wi.ctypes.data if Wi is not None else None,
                                                   L, t.data_ptr(), _stream()), "encode_weights_complex")
        return t

    def matmul(self, keys, xs, w, w_scale, unit_begin=0, unit_end=None, finalize=True, w_shard=False):
        """w_shard: `w` holds only the plaintexts of units [unit_begin, unit_end) (ENCF_PROJ_W_SHARD)."""
        units = self.B_out * self.N2
        unit_end = units if unit_end is None else unit_end
        L = xs[0].n_limbs
        fin = finalize and unit_begin == 0 and unit_end == units
        ys = [self.ctx.empty_ct(L - 1 if fin else L + len(self.ctx.p)) for _ in range(self.B_out)]
        xa = (CT * len(xs))(*[x._c() for x in xs])
        ya = (CT * len(ys))(*[y._c() for y in ys])
        flags = (PROJ_FINALIZE if finalize else 0) | (PROJ_W_SHARD if w_shard else 0)
        _chk(_lib.encf_pt_ct_matmul(self.ctx.h, keys.h, self.h, ctypes.cast(xa, _p), w.data_ptr(), float(w_scale), unit_begin,
                                    unit_end, flags, ctypes.cast(ya, _p), _stream()), "pt_ct_matmul")
        b0, b1 = unit_begin // self.N2, (unit_end - 1) // self.N2 + 1
        return [ys[b]._update(ya[b]) for b in range(b0, b1)]

    def finalize(self, keys, accs, b_begin):
        """accs: extended partial accumulators (n_limbs = L + K)."""
        ys = [self.ctx.empty_ct(self.ctx.level_of_ext(a.n_limbs) - 1) for a in accs]
        aa = (CT * len(accs))(*[a._c() for a in accs])
        ya = (CT * len(ys))(*[y._c() for y in ys])
        _chk(_lib.encf_pt_ct_matmul_finalize(self.ctx.h, keys.h, self.h, ctypes.cast(aa, _p), b_begin, b_begin + len(accs),
                                             ctypes.cast(ya, _p), _stream()), "finalize")
        return [y._update(ya[i]) for i, y in enumerate(ys)]


class AttnPlan:
    def __init__(self, ctx, m, H, d_h, C_qk=0, beta=0, H_blk=0):
        h = _p()
        _chk(_lib.encf_attn_plan_create(ctx.h, m, H, d_h, C_qk, beta, H_blk, ctypes.byref(h)), "attn_plan")
        self.ctx, self.h, self.m, self.H, self.d_h = ctx, h, m, H, d_h
        info = np.zeros(8, dtype=np.int32)
        _chk(_lib.encf_attn_plan_info(h, info.ctypes.data), "attn_plan_info")
        self.B, self.beta, self.g, self.n_out, self.H_blk, self.B_V, self.seg_stride, self.C = [int(x) for x in info]

    def __del__(self):
        try:
            _lib.encf_attn_plan_destroy(self.h)
        except Exception:
            pass

    def galois(self):
        n = _i32()
        buf = np.zeros(1 << 16, dtype=np.uint32)
        _chk(_lib.encf_attn_galois(self.ctx.h, self.h, buf.ctypes.data, len(buf), ctypes.byref(n)), "attn_galois")
        return [int(x) for x in buf[:n.value]]

    def score(self, keys, qs, ks, t_begin=0, t_end=None):
        t_end = self.m // 2 if t_end is None else t_end
        L = qs[0].n_limbs
        outs = [self.ctx.empty_ct(L - 3) for _ in range(t_end - t_begin)]
        qa = (CT * len(qs))(*[x._c() for x in qs])
        ka = (CT * len(ks))(*[x._c() for x in ks])
        oa = (CT * len(outs))(*[o._c() for o in outs])
        _chk(_lib.encf_ct_ct_attn_score(self.ctx.h, keys.h, self.h, ctypes.cast(qa, _p), ctypes.cast(ka, _p), t_begin, t_end,
                                        ctypes.cast(oa, _p), _stream()), "attn_score")
        return [o._update(oa[i]) for i, o in enumerate(outs)]

    def export_stream(self, keys, S):
        L = S[0].n_limbs
        outs = [self.ctx.empty_ct(L - 1) for _ in range(self.n_out)]
        sa = (CT * len(S))(*[x._c() for x in S])
        oa = (CT * len(outs))(*[o._c() for o in outs])
        _chk(_lib.encf_attn_export_stream(self.ctx.h, keys.h, self.h, ctypes.cast(sa, _p), ctypes.cast(oa, _p), _stream()), "export_stream")
        return [o._update(oa[i]) for i, o in enumerate(outs)]

    def value(self, keys, ps, vs):
        L = ps[0].n_limbs
        outs = [self.ctx.empty_ct(L - 2) for _ in range(self.B_V)]
        pa = (CT * len(ps))(*[x._c() for x in ps])
        va = (CT * len(vs))(*[x._c() for x in vs])
        oa = (CT * len(outs))(*[o._c() for o in outs])
        _chk(_lib.encf_ct_ct_attn_value(self.ctx.h, keys.h, self.h, ctypes.cast(pa, _p), ctypes.cast(va, _p), ctypes.cast(oa, _p),
                                        _stream()), "attn_value")
        return [o._update(oa[i]) for i, o in enumerate(outs)]

    def value_blocks(self, unit_begin, unit_end):
        """Blocks touched by the value units [unit_begin, unit_end) (units flattened l (m/2) + t)."""
        half = self.m // 2
        return [l for l in range(self.B_V) if max(unit_begin - l * half, 0) < min(unit_end - l * half, half)]

    def value_partial(self, keys, ps, vs, unit_begin, unit_end):
        """Unrelinearised 3-component partial sums of the touched blocks (encf_ct_ct_attn_value_partial)."""
        L = ps[0].n_limbs
        outs = [self.ctx.empty_ct(L - 1, 3) for _ in self.value_blocks(unit_begin, unit_end)]
        pa = (CT * len(ps))(*[x._c() for x in ps])
        va = (CT * len(vs))(*[x._c() for x in vs])
        oa = (CT * len(outs))(*[o._c() for o in outs])
        _chk(_lib.encf_ct_ct_attn_value_partial(self.ctx.h, keys.h, self.h, ctypes.cast(pa, _p), ctypes.cast(va, _p), unit_begin,
                                                unit_end, ctypes.cast(oa, _p), _stream()), "attn_value_partial")
        return [o._update(oa[i]) for i, o in enumerate(outs)]

    def value_finalize(self, keys, o3s):
        outs = [self.ctx.empty_ct(o.n_limbs - 1) for o in o3s]
        ia = (CT * len(o3s))(*[x._c() for x in o3s])
        oa = (CT * len(outs))(*[o._c() for o in outs])
        _chk(_lib.encf_attn_value_finalize(self.ctx.h, keys.h, ctypes.cast(ia, _p), len(o3s), ctypes.cast(oa, _p), _stream()),
             "attn_value_finalize")
        return [o._update(oa[i]) for i, o in enumerate(outs)]


def exported_symbols():
    """Names declared in include/encf.h that this binding resolves (for the CPU load test)."""
    return sorted(list(_SIG) + ["encf_status_string", "encf_last_error", "encf_galois_rot", "encf_galois_conj"])
