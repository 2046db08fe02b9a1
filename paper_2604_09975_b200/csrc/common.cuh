// common.cuh -- device modular arithmetic and shared host helpers of libencf (sm_100a).
//
// 64-bit RNS words, moduli q < 2^61 (params/*.json).  Products use the 64x64->128 multiply of the
// integer pipe (IMAD.WIDE / IMAD.HI); fixed multipliers use Shoup's precomputed quotient
// w' = floor(w 2^64 / q) (one MULHI + two MULLO per product); variable x variable products and lazy
// 128-bit sums use a Barrett reduction with floor(2^128 / q).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;

#define HD __host__ __device__ __forceinline__

HD u64 umulhi(u64 a, u64 b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (u64)(((unsigned __int128)a * b) >> 64);
#endif
}

struct U128 { u64 lo, hi; };

HD void mac128(U128& acc, u64 a, u64 b) {
    u64 lo = a * b, hi = umulhi(a, b);
    u64 s = acc.lo + lo;
    acc.hi += hi + (s < lo);
    acc.lo = s;
}

HD void add128(U128& acc, u64 v) {
    u64 s = acc.lo + v;
    acc.hi += (s < v);
    acc.lo = s;
}

// Barrett: r = x mod q for a full 128-bit x, ratio = floor(2^128 / q) = (rhi, rlo), q < 2^62.
// The quotient estimate floor(x * ratio / 2^128) (low-low partial product dropped) is below the
// true quotient by at most 3, so at most three conditional subtractions follow.
HD u64 barrett128(U128 x, u64 q, u64 rhi, u64 rlo) {
    u64 a = umulhi(x.lo, rlo);
    u64 b_lo = x.lo * rhi, b_hi = umulhi(x.lo, rhi);
    u64 c_lo = x.hi * rlo, c_hi = umulhi(x.hi, rlo);
    u64 t = a + b_lo;
    u64 c1 = (t < a);
    u64 t2 = t + c_lo;
    u64 c2 = (t2 < t);
    u64 quot = x.hi * rhi + b_hi + c_hi + c1 + c2;
    u64 r = x.lo - quot * q;
    if (r >= q) r -= q;
    if (r >= q) r -= q;
    if (r >= q) r -= q;
    return r;
}

HD u64 mulmod_barrett(u64 a, u64 b, u64 q, u64 rhi, u64 rlo) {
    U128 x{a * b, umulhi(a, b)};
    return barrett128(x, q, rhi, rlo);
}

// Montgomery reduction, R = 2^64: T R^{-1} mod q in [0, q) for any 128-bit T < q 2^64, qinv = -q^{-1} mod 2^64.
// T + m q = 0 mod 2^64 for m = T.lo qinv, so (T + m q) / 2^64 = T.hi + mulhi(m, q) + (T.lo != 0) < 2q.
// Used where one factor of every product is a stored constant kept in Montgomery form (w R mod q): key
// limbs and base-conversion matrices.  Two multiplies instead of the ~7 of barrett128.
HD u64 redc128(U128 T, u64 q, u64 qinv) {
    u64 m = T.lo * qinv;
    u64 t = T.hi + umulhi(m, q) + (T.lo != 0 ? 1ull : 0ull);
    return t >= q ? t - q : t;
}

// Shoup: a * w mod q with wp = floor(w 2^64 / q), w < q, any a < 2^64.  Lazy result in [0, 2q).
HD u64 mul_shoup_lazy(u64 a, u64 w, u64 wp, u64 q) {
    u64 h = umulhi(a, wp);
    return a * w - h * q;
}
HD u64 mul_shoup(u64 a, u64 w, u64 wp, u64 q) {
    u64 r = mul_shoup_lazy(a, w, wp, q);
    return r >= q ? r - q : r;
}
HD u64 shoup_pre(u64 w, u64 q) {  // host only in practice
#ifdef __CUDA_ARCH__
    // floor(w * 2^64 / q) via 128-bit division is not available on device; callers precompute.
    return 0;
#else
    return (u64)(((unsigned __int128)w << 64) / q);
#endif
}

HD u64 add_mod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
HD u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

// Per-modulus constants (device table indexed by modulus id: q_0..q_{L-1}, p_0..p_{K-1}).
struct ModConst {
    u64 q;
    u64 rhi, rlo;       // floor(2^128 / q)
    u64 two_q;
    u64 qinv;           // -q^{-1} mod 2^64 (Montgomery)
};

// Host 128-bit helpers.
inline u64 h_mulmod(u64 a, u64 b, u64 q) { return (u64)(((unsigned __int128)a * b) % q); }
inline u64 h_powmod(u64 a, u64 e, u64 q) {
    u64 r = 1 % q; a %= q;
    while (e) { if (e & 1) r = h_mulmod(r, a, q); a = h_mulmod(a, a, q); e >>= 1; }
    return r;
}
inline u64 h_invmod(u64 a, u64 q) { return h_powmod(a % q, q - 2, q); }
inline u64 h_neg_inv64(u64 q) {   // -q^{-1} mod 2^64, q odd (Newton)
    u64 x = q;
    for (int i = 0; i < 6; i++) x *= 2 - q * x;
    return (u64)0 - x;
}
inline u64 h_mont_R(u64 q) { return (u64)(((unsigned __int128)1 << 64) % q); }
inline void h_ratio128(u64 q, u64& rhi, u64& rlo) {
    // floor(2^128 / q) = floor((2^128 - 1) / q) for q not a power of two
    unsigned __int128 all = ~(unsigned __int128)0;
    unsigned __int128 r = all / q;
    rhi = (u64)(r >> 64); rlo = (u64)r;
}

#define MAX_MODS 64
#define MAX_LIMBS 64

// A map from the limbs of a polynomial batch to modulus ids (passed by value to kernels).
struct LimbMap {
    int n;
    unsigned char mod[MAX_LIMBS];
};
