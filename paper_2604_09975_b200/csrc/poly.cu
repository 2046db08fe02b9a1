// poly.cu -- sm_100a kernels for everything that is not an NTT:
//   pointwise add/sub/ptmul, x i (= X^{N/2}), Galois automorphism as an NTT-domain gather,
//   counter-PRNG sampling, fast base conversion (ModUp / ModDown), the key-switching inner
//   product (hoisted: the automorphism is fused into the digit loads), ModDown epilogue, rescale,
//   the lazy ct x ct tensor sum, the fused plaintext-diagonal multiply-accumulate of the
//   projection, masked sums (Psi shifts, broadcasts), export masking, and float64 encode/decode.
// Integer work runs on the IMAD pipe with 64x64->128 products; every kernel is HBM- or IMAD-bound
// (no dense contraction here: DESIGN.md "Why no tensor cores").
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "ctx.cuh"

namespace {

constexpr int TB = 256;

inline int nblocks(size_t work, int per_block = TB, int cap = 148 * 32) {
    size_t b = (work + per_block - 1) / per_block;
    return (int)(b < (size_t)cap ? b : (size_t)cap);
}

__device__ __forceinline__ int brv(int x, int logN) { return (int)(__brev((unsigned)x) >> (32 - logN)); }

// ------------------------------------------------------------------------------------ pointwise
__global__ void add_kernel(const u64* __restrict__ a, const u64* __restrict__ b, u64* __restrict__ out,
                           size_t total, int N, LimbMap m, const ModConst* mod, int sub) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)((i / N) % m.n);
        u64 q = mod[m.mod[limb]].q;
        u64 x = a[i], y = b[i];
        out[i] = sub ? sub_mod(x, y, q) : add_mod(x, y, q);
    }
}

__global__ void mul_kernel(const u64* __restrict__ a, i64 as, const u64* __restrict__ b, i64 bs, u64* __restrict__ out,
                           i64 os, int npolys, int N, LimbMap m, const ModConst* mod) {
    size_t per = (size_t)m.n * N, total = per * npolys;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        size_t p = i / per, r = i % per;
        int limb = (int)(r / N);
        ModConst mc = mod[m.mod[limb]];
        out[p * os + r] = mulmod_barrett(a[p * as + r], b[p * bs + r], mc.q, mc.rhi, mc.rlo);
    }
}

// x i: X^{N/2}(psi^{e}) = psi^{e N/2} = im^{e mod 4}; in bit-reversed order e_i = 2 brv(i) + 1 is
// 1 mod 4 exactly for i < N/2, so the first half is multiplied by im and the second by -im.
__global__ void mul_i_kernel(const u64* __restrict__ a, u64* __restrict__ out, size_t total, int N, LimbMap m,
                             const ModConst* mod, const u64* im, const u64* im_sh) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)((i / N) % m.n), k = (int)(i % N);
        int mi = m.mod[limb];
        u64 q = mod[mi].q;
        u64 r = mul_shoup(a[i], im[mi], im_sh[mi], q);
        if (k >= N / 2) r = r ? q - r : 0;
        out[i] = r;
    }
}

// out_r = a_r +- X^{N/2} b_r for a batch of same-shape ciphertexts (one launch instead of a mul_i and an add per
// pair; the same two modular operations per word as mul_i_kernel followed by add_kernel, so bit-identical).
__global__ void add_i_batch_kernel(AddIBatch B, int n, size_t per, int N, LimbMap m, const ModConst* mod, const u64* im,
                                   const u64* im_sh, int sub) {
    const size_t total = per * n;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / per);
        const size_t j = i - (size_t)r * per;
        const int limb = (int)((j / N) % m.n), k = (int)(j % N);
        const int mi = m.mod[limb];
        const u64 q = mod[mi].q;
        u64 t = mul_shoup(B.b[r][j], im[mi], im_sh[mi], q);
        if (k >= N / 2) t = t ? q - t : 0;
        const u64 x = B.a[r][j];
        B.out[r][j] = sub ? sub_mod(x, t, q) : add_mod(x, t, q);
    }
}

// sigma_g in the NTT domain: out[i] = in[brv(((e_i g mod 2N) - 1) / 2)], e_i = 2 brv(i) + 1.
// Within an aligned block of 2^k indices the sources are a permutation of an aligned block, so warp
// accesses stay inside one 256-byte segment (coalesced gather).
__global__ void automorph_kernel(const u64* __restrict__ in, i64 is, u64* __restrict__ out, i64 os,
                                 int npolys, int nlimbs, int N, int logN, uint32_t g) {
    size_t per = (size_t)nlimbs * N, total = per * npolys;
    const uint32_t mask2n = 2 * N - 1;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        size_t p = i / per, r = i % per;
        size_t limb = r / N;
        int k = (int)(r % N);
        uint32_t e = 2u * (uint32_t)brv(k, logN) + 1u;
        uint32_t e2 = (uint32_t)(((uint64_t)e * g) & mask2n);
        int src = brv((int)((e2 - 1) >> 1), logN);
        out[p * os + limb * N + k] = in[p * is + limb * N + src];
    }
}

// ------------------------------------------------------------------------------------ PRNG
__device__ __forceinline__ u64 prng_draw(u64 seed, u64 stream, u64 index) {
    u64 z = (seed ^ (stream * 0xD1B54A32D192ED03ULL)) + (index + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

struct Gids { int g[MAX_LIMBS]; };

__global__ void sample_uniform_kernel(u64 seed, u64 stream, u64* out, int N, LimbMap m, Gids gids, const ModConst* mod) {
    size_t total = (size_t)m.n * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)(i / N), k = (int)(i % N);
        u64 q = mod[m.mod[limb]].q;
        u64 idx = 2 * ((u64)gids.g[limb] * (u64)N + (u64)k);
        u64 hi = prng_draw(seed, stream, idx), lo = prng_draw(seed, stream, idx + 1);
        // ((hi 2^64 + lo) q) >> 128 = high word of (hi q + ((lo q) >> 64))
        u64 a_lo = hi * q, a_hi = umulhi(hi, q);
        u64 b = umulhi(lo, q);
        u64 s = a_lo + b;
        out[i] = a_hi + (s < a_lo);
    }
}

__global__ void sample_small_kernel(u64 seed, u64 stream, int kind, u64* out, int N, LimbMap m, const ModConst* mod) {
    size_t total = (size_t)m.n * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)(i / N), k = (int)(i % N);
        u64 q = mod[m.mod[limb]].q;
        u64 u = prng_draw(seed, stream, (u64)k);
        i64 v;
        if (kind == 0) v = (i64)umulhi(u, 3) - 1;
        else v = (i64)__popcll(u & 0x1FFFFFULL) - (i64)__popcll((u >> 21) & 0x1FFFFFULL);
        out[i] = v < 0 ? q - (u64)(-v) : (u64)v;
    }
}

__global__ void scalar_mul_kernel(u64* data, int npolys, int N, LimbMap m, const ModConst* mod, const u64* s, const u64* ssh) {
    size_t total = (size_t)npolys * m.n * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)((i / N) % m.n);
        data[i] = mul_shoup(data[i], s[limb], ssh[limb], mod[m.mod[limb]].q);
    }
}

__global__ void add_scalar_kernel(u64* data, int N, LimbMap m, const ModConst* mod, const u64* sc) {
    const size_t total = (size_t)m.n * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int limb = (int)(i / N);
        data[i] = add_mod(data[i], sc[limb], mod[m.mod[limb]].q);
    }
}

__global__ void mod_reduce_kernel(u64* data, size_t total, int N, LimbMap m, const ModConst* mod) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)((i / N) % m.n);
        data[i] = data[i] % mod[m.mod[limb]].q;
    }
}

// ------------------------------------------------------------------------------------ rescale (C5)
// corr_i[k] = ((c_L[k] + h) mod q_L  mod q_i  -  h mod q_i) mod q_i   (coefficient domain)
__global__ void rescale_prep_kernel(const u64* last, i64 ls, u64* corr, int ncomp, int level, int N,
                                    const ModConst* mod, const u64* hmod) {
    int nl = level - 1;
    size_t per = (size_t)nl * N, total = per * ncomp;
    u64 qL = mod[level - 1].q, h = qL / 2;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int c = (int)(i / per);
        size_t r = i % per;
        int limb = (int)(r / N), k = (int)(r % N);
        const ModConst mc = mod[limb];
        u64 lp = add_mod(last[c * ls + k], h, qL);
        corr[i] = sub_mod(barrett128(U128{lp, 0}, mc.q, mc.rhi, mc.rlo), hmod[limb], mc.q);
    }
}

// out_i = (c_i - corr_i) q_L^{-1} mod q_i   (NTT domain; corr already transformed)
__global__ void rescale_finish_kernel(const u64* in, i64 is, const u64* corr, u64* out, i64 os, int ncomp, int level,
                                      int N, const ModConst* mod, const u64* inv, const u64* inv_sh) {
    int nl = level - 1;
    size_t per = (size_t)nl * N, total = per * ncomp;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int c = (int)(i / per);
        size_t r = i % per;
        int limb = (int)(r / N);
        u64 qi = mod[limb].q;
        u64 d = sub_mod(in[c * is + r], corr[i], qi);
        out[c * os + r] = mul_shoup(d, inv[limb], inv_sh[limb], qi);
    }
}

// out_i = (b_i - y_i) P^{-1} (+ add0_i) mod q_i   (NTT domain)
__global__ void moddown_finish_kernel(const u64* __restrict__ b, const u64* __restrict__ y, const u64* __restrict__ add0,
                                      u64* __restrict__ out, int level, int N, const ModConst* __restrict__ mod,
                                      const u64* pinv, const u64* pinv_sh) {
    size_t total = (size_t)level * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)(i / N);
        u64 q = mod[limb].q;
        u64 r = mul_shoup(sub_mod(b[i], y[i], q), pinv[limb], pinv_sh[limb], q);
        if (add0) r = add_mod(r, add0[i], q);
        out[i] = r;
    }
}

// ------------------------------------------------------------------------------------ lazy tensor sum
struct PtrList { const u64* p[64]; };

// out3 = sum_t (a0 b0, a0 b1 + a1 b0, a1 b1) with 128-bit lazy accumulation (reduced every 64 terms).
__global__ void __launch_bounds__(TB) tensor_acc_kernel(const u64* const* __restrict__ A, const u64* const* __restrict__ B,
                                                        int nterms, u64* __restrict__ out, int level, int N,
                                                        const ModConst* __restrict__ mod) {
    const int limb = blockIdx.y;
    const ModConst mc = mod[limb];
    const size_t cs = (size_t)level * N;   // component stride
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const size_t o = (size_t)limb * N + k;
        u64 r0 = 0, r1 = 0, r2 = 0;
        for (int t0 = 0; t0 < nterms; t0 += 64) {
            U128 d0{0, 0}, d1{0, 0}, d2{0, 0};
            int te = min(nterms, t0 + 64);
            for (int t = t0; t < te; t++) {
                const u64* a = A[t];
                const u64* b = B[t];
                u64 a0 = a[o], a1 = a[cs + o], b0 = b[o], b1 = b[cs + o];
                mac128(d0, a0, b0);
                mac128(d1, a0, b1);
                mac128(d1, a1, b0);
                mac128(d2, a1, b1);
            }
            r0 = add_mod(r0, barrett128(d0, mc.q, mc.rhi, mc.rlo), mc.q);
            r1 = add_mod(r1, barrett128(d1, mc.q, mc.rhi, mc.rlo), mc.q);
            r2 = add_mod(r2, barrett128(d2, mc.q, mc.rhi, mc.rlo), mc.q);
        }
        out[o] = r0;
        out[cs + o] = r1;
        out[2 * cs + o] = r2;
    }
}

// out = sum_t ct_t (.) mask_t   (2-component cts [2][level][N], masks [level][N]; lazy 128-bit sums)
__global__ void __launch_bounds__(TB) masked_sum_kernel(const u64* const* __restrict__ C, const u64* const* __restrict__ M,
                                                        int nterms, u64* __restrict__ out, int level, int N,
                                                        const ModConst* __restrict__ mod) {
    const int limb = blockIdx.y;
    const ModConst mc = mod[limb];
    const size_t cs = (size_t)level * N;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const size_t o = (size_t)limb * N + k;
        u64 r0 = 0, r1 = 0;
        for (int t0 = 0; t0 < nterms; t0 += 128) {
            U128 d0{0, 0}, d1{0, 0};
            int te = min(nterms, t0 + 128);
            for (int t = t0; t < te; t++) {
                const u64* c = C[t];
                u64 w = M[t][o];
                mac128(d0, c[o], w);
                mac128(d1, c[cs + o], w);
            }
            r0 = add_mod(r0, barrett128(d0, mc.q, mc.rhi, mc.rlo), mc.q);
            r1 = add_mod(r1, barrett128(d1, mc.q, mc.rhi, mc.rlo), mc.q);
        }
        out[o] = r0;
        out[cs + o] = r1;
    }
}

// ------------------------------------------------------------------------------------ diagonal MAC (projection, C6 step 2)
// acc[unit][c][l][k] = sum_{uq < nbank} bank[uq][c][l][k] * w[unit][uq][l][k]
// A CTA owns a 32-coefficient tile of one limb: the bank tile (nbank x 2 x 32 words) is staged once in
// shared memory and reused by every unit; the plaintext stream is read exactly once with 128-bit loads
// (two coefficients per thread, 16 unit lanes per CTA), accumulators stay in 128-bit registers and are
// reduced once per unit.
constexpr int MAC_T = 32;      // coefficients per CTA tile
constexpr int MAC_TPR = 16;    // threads per tile row (2 coefficients each)
constexpr int MAC_LANES = 16;  // unit lanes per CTA (blockDim = 256)

// Narrow limbs (q < 2^41): both factors split at 20 bits, x = xh 2^20 + xl, and the product formed Karatsuba-
// style from THREE 32x32->64 products (xh yh, xl yl, (xh+xl)(yh+yl)) accumulated in 64 bits without carries
// (each < 2^43, 64 terms < 2^49): 3 IMAD.WIDE per product instead of the ~6 half-rate ops + carry chain of a
// 64x64->128 MAC, so the kernel stays HBM-bound.  The bank tile is pre-split in shared memory.
__device__ __forceinline__ u64 kara_combine(u64 hh, u64 ll, u64 ss, u64 q, u64 rhi, u64 rlo, u64 t40) {
    const u64 mid = ss - hh - ll;                         // = sum (xh yl + xl yh) < 2^48
    U128 acc{ll, 0};
    mac128(acc, hh, t40);                                 // hh * (2^40 mod q)
    add128(acc, mid << 20);                               // mid 2^20 < 2^68: split
    acc.hi += mid >> 44;
    return barrett128(acc, q, rhi, rlo);
}

template <bool NARROW>
__global__ void __launch_bounds__(MAC_TPR * MAC_LANES) diag_mac_kernel(const u64* __restrict__ bank, int nbank,
                                                                       const u64* __restrict__ w, int units, i64 wus,
                                                                       u64* __restrict__ acc, i64 accs, int level, int N,
                                                                       const ModConst* __restrict__ mod, int limb0) {
    extern __shared__ ulonglong2 sb2[];   // wide: [nbank][2][MAC_T / 2] u64 pairs; narrow: [nbank][2][MAC_T] uint2 {h, l}
    u64* sb = (u64*)sb2;
    const int limb = limb0 + blockIdx.y;
    const int k0 = blockIdx.x * MAC_T;
    const ModConst mc = mod[limb];
    constexpr bool narrow = NARROW;
    const size_t cs = (size_t)level * N;
    const size_t bs = 2 * cs;
    const int kp = threadIdx.x % MAC_TPR, lane = threadIdx.x / MAC_TPR;
    const size_t wl = (size_t)limb * N + k0 + 2 * kp;
    const size_t pstride = (size_t)level * N;
    if constexpr (narrow) {
        uint2* sn = (uint2*)sb2;          // [uq][c][kk]
        for (int i = threadIdx.x; i < nbank * 2 * MAC_T; i += blockDim.x) {
            int uq = i / (2 * MAC_T), r = i % (2 * MAC_T);
            int c = r / MAC_T, kk = r % MAC_T;
            const u64 x = bank[(size_t)uq * bs + c * cs + (size_t)limb * N + k0 + kk];
            const uint32_t h = (uint32_t)(x >> 20), l = (uint32_t)(x & 0xFFFFF);
            sn[i] = make_uint2(h, l);
        }
        __syncthreads();
        const u64 t40 = (1ull << 40) % mc.q;
        // software-pipelined stream: the 8 plaintext words of the NEXT (unit, chunk) are in flight while the
        // current chunk is multiplied (keeps ~128 B per thread outstanding -> HBM-bound, not latency-bound)
        // (the host routes a bank size that is not a multiple of 8 to the 128-bit path: no tail checks here)
        const int nch = nbank >> 3, ustride = gridDim.z * MAC_LANES;
        int u = blockIdx.z * MAC_LANES + lane, ch = 0;
        if (u >= units) return;
        const uint4* sbase = (const uint4*)sn + kp;    // {h, l} pairs of coefficients (k, k+1) of this thread
        ulonglong2 cur[8], nxt[8];
#pragma unroll
        for (int t = 0; t < 8; t++) cur[t] = __ldg((const ulonglong2*)(w + (size_t)u * wus + wl + (size_t)t * pstride));
        u64 h00 = 0, l00 = 0, s00 = 0, h01 = 0, l01 = 0, s01 = 0, h10 = 0, l10 = 0, s10 = 0, h11 = 0, l11 = 0, s11 = 0;
        while (true) {
            int nu = u, nc = ch + 1;
            if (nc == nch) { nu = u + ustride; nc = 0; }
            const bool more = nu < units;
            if (more) {
                const u64* wn = w + (size_t)nu * wus + wl + (size_t)(nc * 8) * pstride;
#pragma unroll
                for (int t = 0; t < 8; t++) nxt[t] = __ldg((const ulonglong2*)(wn + (size_t)t * pstride));
            }
            const uint4* sb8 = sbase + (size_t)(ch * 8) * 2 * (MAC_T / 2);
#pragma unroll
            for (int t = 0; t < 8; t++) {
                const uint32_t ah = (uint32_t)(cur[t].x >> 20), al = (uint32_t)(cur[t].x & 0xFFFFF);
                const uint32_t bh = (uint32_t)(cur[t].y >> 20), bl = (uint32_t)(cur[t].y & 0xFFFFF);
                const uint32_t as = ah + al, bsum = bh + bl;
                const uint4 pp = sb8[(t * 2 + 0) * (MAC_T / 2)];   // {h, l} of k, k+1 (component 0)
                const uint4 rr = sb8[(t * 2 + 1) * (MAC_T / 2)];   // component 1
                h00 += (u64)pp.x * ah; l00 += (u64)pp.y * al; s00 += (u64)(pp.x + pp.y) * as;
                h01 += (u64)pp.z * bh; l01 += (u64)pp.w * bl; s01 += (u64)(pp.z + pp.w) * bsum;
                h10 += (u64)rr.x * ah; l10 += (u64)rr.y * al; s10 += (u64)(rr.x + rr.y) * as;
                h11 += (u64)rr.z * bh; l11 += (u64)rr.w * bl; s11 += (u64)(rr.z + rr.w) * bsum;
            }
            if (ch == nch - 1) {
                u64* o = acc + (size_t)u * accs + wl;
                *(ulonglong2*)o = make_ulonglong2(kara_combine(h00, l00, s00, mc.q, mc.rhi, mc.rlo, t40),
                                                  kara_combine(h01, l01, s01, mc.q, mc.rhi, mc.rlo, t40));
                *(ulonglong2*)(o + cs) = make_ulonglong2(kara_combine(h10, l10, s10, mc.q, mc.rhi, mc.rlo, t40),
                                                         kara_combine(h11, l11, s11, mc.q, mc.rhi, mc.rlo, t40));
                h00 = l00 = s00 = h01 = l01 = s01 = h10 = l10 = s10 = h11 = l11 = s11 = 0;
            }
            if (!more) break;
            u = nu; ch = nc;
#pragma unroll
            for (int t = 0; t < 8; t++) cur[t] = nxt[t];
        }
        return;
    }
    for (int i = threadIdx.x; i < nbank * 2 * MAC_T; i += blockDim.x) {
        int uq = i / (2 * MAC_T), r = i % (2 * MAC_T);
        int c = r / MAC_T, kk = r % MAC_T;
        sb[i] = bank[(size_t)uq * bs + c * cs + (size_t)limb * N + k0 + kk];
    }
    __syncthreads();
    for (int u = blockIdx.z * MAC_LANES + lane; u < units; u += gridDim.z * MAC_LANES) {
        const u64* wu = w + (size_t)u * wus + wl;
        U128 a00{0, 0}, a01{0, 0}, a10{0, 0}, a11{0, 0};   // [component][coefficient]
        int uq = 0;
        for (; uq + 8 <= nbank; uq += 8) {
            ulonglong2 x[8];
#pragma unroll
            for (int t = 0; t < 8; t++) x[t] = __ldg((const ulonglong2*)(wu + (size_t)(uq + t) * pstride));
#pragma unroll
            for (int t = 0; t < 8; t++) {
                const ulonglong2 b0 = sb2[(uq + t) * MAC_T + kp];
                const ulonglong2 b1 = sb2[(uq + t) * MAC_T + MAC_T / 2 + kp];
                mac128(a00, b0.x, x[t].x);
                mac128(a01, b0.y, x[t].y);
                mac128(a10, b1.x, x[t].x);
                mac128(a11, b1.y, x[t].y);
            }
            // every 32 products (< 32 q^2 <= 2^127 for q < 2^61) fold the 128-bit sums back below q, so any bank
            // size is exact
            if (((uq + 8) & 31) == 0) {
                a00 = U128{barrett128(a00, mc.q, mc.rhi, mc.rlo), 0}; a01 = U128{barrett128(a01, mc.q, mc.rhi, mc.rlo), 0};
                a10 = U128{barrett128(a10, mc.q, mc.rhi, mc.rlo), 0}; a11 = U128{barrett128(a11, mc.q, mc.rhi, mc.rlo), 0};
            }
        }
        for (; uq < nbank; uq++) {
            const ulonglong2 xx = __ldg((const ulonglong2*)(wu + (size_t)uq * pstride));
            const ulonglong2 b0 = sb2[uq * MAC_T + kp];
            const ulonglong2 b1 = sb2[uq * MAC_T + MAC_T / 2 + kp];
            mac128(a00, b0.x, xx.x);
            mac128(a01, b0.y, xx.y);
            mac128(a10, b1.x, xx.x);
            mac128(a11, b1.y, xx.y);
        }
        u64* o = acc + (size_t)u * accs + wl;
        *(ulonglong2*)o = make_ulonglong2(barrett128(a00, mc.q, mc.rhi, mc.rlo), barrett128(a01, mc.q, mc.rhi, mc.rlo));
        *(ulonglong2*)(o + cs) = make_ulonglong2(barrett128(a10, mc.q, mc.rhi, mc.rlo), barrett128(a11, mc.q, mc.rhi, mc.rlo));
    }
}

// ------------------------------------------------------------------------------------ diagonal MAC, bulk-copy pipeline
// Same arithmetic and output words as diag_mac_kernel; the plaintext stream reaches shared memory through
// cp.async.bulk (the TMA engine, SASS UBLKCP) into a DM_STAGES-deep ring of 32 KB stages guarded by mbarriers, so a
// CTA keeps up to DM_STAGES x 32 KB of HBM reads in flight with no register staging (the register double buffer of
// diag_mac_kernel limited it to 2 CTAs/SM and ~64 KB per SM).  Stage s = (unit group g of 16 units, bank chunk c of 8
// rows): 128 rows of 32 coefficients (256 B each, one bulk copy per row, issued by 128 threads), consumed by the 16
// unit lanes x 16 threads (2 coefficients each) of the CTA; one __syncthreads per stage returns the slot to the ring.
constexpr int DM_ROWS = 8;
constexpr int DM_STAGE_WORDS = MAC_LANES * DM_ROWS * MAC_T;   // 4096 words = 32 KB
constexpr int DM_MAX_STAGES = 5;
#ifndef MAC_KARA
#define MAC_KARA 1   // wide-limb (30-bit split) plaintext MAC: Karatsuba, 3 products; 0: 4 products (A/B)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// One 4-D tensor TMA per stage: the weight stream as the tensor [units][nbank][level][N] (u64) with box
// {32 coefficients, 1 limb, 8 bank rows, 16 units} = 32 KB, landing as [16][8][32] words -- the layout the consumers
// read; out-of-range units / rows are zero-filled (and never consumed).
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
        ::"r"(smem_u32(dst)), "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)) : "memory");
}

template <bool NARROW, int ROWS, int MINB>
__global__ void __launch_bounds__(MAC_TPR * MAC_LANES, MINB) diag_mac_tma_kernel(const __grid_constant__ CUtensorMap tmw,
                                                                             const u64* __restrict__ bank, int nbank,
                                                                             const u64* __restrict__ w, int units, i64 wus,
                                                                             u64* __restrict__ acc, i64 accs, int level, int N,
                                                                             const ModConst* __restrict__ mod, int limb0,
                                                                             int nstages, int fp_split) {
    extern __shared__ __align__(128) u64 dm_sm[];
    const bool fpw = NARROW && fp_split && (threadIdx.x >> 5) >= 4;   // warp-uniform: FP64-pipe warps (narrow limbs)
    constexpr int SW = MAC_LANES * ROWS * MAC_T;                 // words per stage
    u64* stg = dm_sm;                                            // [nstages][16 lanes][8 rows][32 coefficients]
    u64* sb = stg + (size_t)nstages * SW;            // bank tile, layout of diag_mac_kernel
    uint64_t* bars = (uint64_t*)(sb + (size_t)nbank * 2 * MAC_T);
    const int limb = limb0 + blockIdx.y;
    const int k0 = blockIdx.x * MAC_T;
    const ModConst mc = mod[limb];
    const size_t cs = (size_t)level * N, bs = 2 * cs, pstride = (size_t)level * N;
    const int tid = threadIdx.x, kp = tid % MAC_TPR, lane = tid / MAC_TPR;
    if (tid == 0) {
        for (int i = 0; i < nstages; i++) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // bank tile (read once per CTA; L2-resident across the tiles of one launch)
    if constexpr (NARROW) {
        uint2* sn = (uint2*)sb;
        for (int i = tid; i < nbank * 2 * MAC_T; i += blockDim.x) {
            const int uq = i / (2 * MAC_T), r = i % (2 * MAC_T), c = r / MAC_T, kk = r % MAC_T;
            const u64 x = bank[(size_t)uq * bs + c * cs + (size_t)limb * N + k0 + kk];
            sn[i] = make_uint2((uint32_t)(x >> 20), (uint32_t)(x & 0xFFFFF));
        }
    } else {
        // 128-bit limbs (q < 2^60): bank words pre-split at 30 bits, {h, l} per word (see the consumer)
        uint2* sn = (uint2*)sb;
        for (int i = tid; i < nbank * 2 * MAC_T; i += blockDim.x) {
            const int uq = i / (2 * MAC_T), r = i % (2 * MAC_T), c = r / MAC_T, kk = r % MAC_T;
            const u64 x = bank[(size_t)uq * bs + c * cs + (size_t)limb * N + k0 + kk];
            sn[i] = make_uint2((uint32_t)(x >> 30), (uint32_t)(x & 0x3FFFFFFFu));
        }
    }
    __syncthreads();
    const int ngroups = (units + MAC_LANES - 1) / MAC_LANES;
    const int nch = (nbank + ROWS - 1) / ROWS;
    const int mygroups = blockIdx.z < ngroups ? (ngroups - 1 - blockIdx.z) / gridDim.z + 1 : 0;
    const int total = mygroups * nch;
    auto issue = [&](int s) {
        if (tid != 0) return;
        const int g = blockIdx.z + (s / nch) * gridDim.z, c = s % nch;
        const int slot = s % nstages;
        mbar_arrive_expect_tx(&bars[slot], (uint32_t)(SW * 8));      // the full box (OOB zero-filled)
        tma_load_4d(stg + (size_t)slot * SW, &tmw, k0, limb, c * ROWS, g * MAC_LANES, &bars[slot]);
    };
    (void)w; (void)pstride;
    for (int s = 0; s < nstages - 1 && s < total; s++) issue(s);
    const u64 t40 = (1ull << 40) % mc.q;
    u64 h00 = 0, l00 = 0, s00 = 0, h01 = 0, l01 = 0, s01 = 0, h10 = 0, l10 = 0, s10 = 0, h11 = 0, l11 = 0, s11 = 0;
    U128 a00{0, 0}, a01{0, 0}, a10{0, 0}, a11{0, 0};
    for (int s = 0; s < total; s++) {
        if (s + nstages - 1 < total) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads of the slot before its refill
            issue(s + nstages - 1);
        }
        const int slot = s % nstages;
        mbar_wait(&bars[slot], (uint32_t)((s / nstages) & 1));
        const int g = blockIdx.z + (s / nch) * gridDim.z, c = s % nch;
        const int rows = min(ROWS, nbank - c * ROWS);
        const int u = g * MAC_LANES + lane;
        if (u < units) {
            const ulonglong2* xr = (const ulonglong2*)(stg + (size_t)slot * SW + (size_t)lane * ROWS * MAC_T) + kp;
            if constexpr (NARROW) {
                const uint4* sb8 = (const uint4*)sb + kp + (size_t)(c * ROWS) * 2 * (MAC_T / 2);
                auto row = [&](int t) {
                    const ulonglong2 x = xr[t * (MAC_T / 2)];
                    const uint32_t ah = (uint32_t)(x.x >> 20), al = (uint32_t)(x.x & 0xFFFFF);
                    const uint32_t bh = (uint32_t)(x.y >> 20), bl = (uint32_t)(x.y & 0xFFFFF);
                    const uint32_t as = ah + al, bsum = bh + bl;
                    const uint4 pp = sb8[(t * 2 + 0) * (MAC_T / 2)];
                    const uint4 rr = sb8[(t * 2 + 1) * (MAC_T / 2)];
                    h00 += (u64)pp.x * ah; l00 += (u64)pp.y * al; s00 += (u64)(pp.x + pp.y) * as;
                    h01 += (u64)pp.z * bh; l01 += (u64)pp.w * bl; s01 += (u64)(pp.z + pp.w) * bsum;
                    h10 += (u64)rr.x * ah; l10 += (u64)rr.y * al; s10 += (u64)(rr.x + rr.y) * as;
                    h11 += (u64)rr.z * bh; l11 += (u64)rr.w * bl; s11 += (u64)(rr.z + rr.w) * bsum;
                };
                // FP64-pipe copy of the same split products (warps 4-7 when fp_split): pieces < 2^21 + 2^20, products
                // < 2^44, sums of <= 512 products < 2^53 -- exact in doubles, kept in the bits of the same u64 accumulators
                // and converted back before kara_combine, so the words are identical; each SM sub-partition runs one
                // integer-pipe and one FP64-pipe warp of the CTA
                auto row_fp = [&](int t) {
                    auto cvd = [](uint32_t v) -> double {
                        return __dsub_rn(__hiloint2double(0x43300000, (int)v), 4503599627370496.0);
                    };
                    auto acc = [](u64& a, double x, double y) {
                        a = (u64)__double_as_longlong(__fma_rn(x, y, __longlong_as_double((long long)a)));
                    };
                    const ulonglong2 x = xr[t * (MAC_T / 2)];
                    const double ah = cvd((uint32_t)(x.x >> 20)), al = cvd((uint32_t)(x.x & 0xFFFFF));
                    const double bh = cvd((uint32_t)(x.y >> 20)), bl = cvd((uint32_t)(x.y & 0xFFFFF));
                    const double as = __dadd_rn(ah, al), bsum = __dadd_rn(bh, bl);
                    const uint4 pp = sb8[(t * 2 + 0) * (MAC_T / 2)];
                    const uint4 rr = sb8[(t * 2 + 1) * (MAC_T / 2)];
                    const double p0 = cvd(pp.x), p1 = cvd(pp.y), p2 = cvd(pp.z), p3 = cvd(pp.w);
                    const double r0 = cvd(rr.x), r1 = cvd(rr.y), r2 = cvd(rr.z), r3 = cvd(rr.w);
                    acc(h00, p0, ah); acc(l00, p1, al); acc(s00, __dadd_rn(p0, p1), as);
                    acc(h01, p2, bh); acc(l01, p3, bl); acc(s01, __dadd_rn(p2, p3), bsum);
                    acc(h10, r0, ah); acc(l10, r1, al); acc(s10, __dadd_rn(r0, r1), as);
                    acc(h11, r2, bh); acc(l11, r3, bl); acc(s11, __dadd_rn(r2, r3), bsum);
                };
                if (fpw) {
                    if (rows == ROWS) {
#pragma unroll
                        for (int t = 0; t < ROWS; t++) row_fp(t);
                    } else {
                        for (int t = 0; t < rows; t++) row_fp(t);
                    }
                } else if (rows == ROWS) {    // full chunk: no per-row guard in the unrolled body
#pragma unroll
                    for (int t = 0; t < ROWS; t++) row(t);
                } else {
                    for (int t = 0; t < rows; t++) row(t);
                }
            } else {
                // 30-bit split: x = xh 2^30 + xl, b = bh 2^30 + bl (q < 2^60); Karatsuba per product: 3 IMAD.WIDE.U32 into
                // 64-bit sums hh, mm = sum (xh + xl)(bh + bl), ll (MAC_KARA=0: 4 products, md = xh bl + xl bh directly).
                // mm wraps mod 2^64, but md = mm - hh - ll is exact there because md < 16 (2^30 - 1)^2 < 2^64 over the
                // <= ROWS = 8 rows of a chunk; each chunk folds hh 2^60 + md 2^30 + ll into the 128-bit sum
                const uint4* sb8 = (const uint4*)sb + kp + (size_t)(c * ROWS) * 2 * (MAC_T / 2);
                u64 hh00 = 0, md00 = 0, ll00 = 0, hh01 = 0, md01 = 0, ll01 = 0, hh10 = 0, md10 = 0, ll10 = 0, hh11 = 0, md11 = 0,
                    ll11 = 0;
                auto row = [&](int t) {
                    const ulonglong2 x = xr[t * (MAC_T / 2)];
                    const uint32_t ah = (uint32_t)(x.x >> 30), al = (uint32_t)(x.x & 0x3FFFFFFFu);
                    const uint32_t bh = (uint32_t)(x.y >> 30), bl = (uint32_t)(x.y & 0x3FFFFFFFu);
                    const uint4 pp = sb8[(t * 2 + 0) * (MAC_T / 2)];
                    const uint4 rr = sb8[(t * 2 + 1) * (MAC_T / 2)];
#if MAC_KARA
                    const uint32_t as = ah + al, bsum = bh + bl;
                    hh00 += (u64)pp.x * ah; md00 += (u64)(pp.x + pp.y) * as; ll00 += (u64)pp.y * al;
                    hh01 += (u64)pp.z * bh; md01 += (u64)(pp.z + pp.w) * bsum; ll01 += (u64)pp.w * bl;
                    hh10 += (u64)rr.x * ah; md10 += (u64)(rr.x + rr.y) * as; ll10 += (u64)rr.y * al;
                    hh11 += (u64)rr.z * bh; md11 += (u64)(rr.z + rr.w) * bsum; ll11 += (u64)rr.w * bl;
#else
                    hh00 += (u64)pp.x * ah; md00 += (u64)pp.x * al + (u64)pp.y * ah; ll00 += (u64)pp.y * al;
                    hh01 += (u64)pp.z * bh; md01 += (u64)pp.z * bl + (u64)pp.w * bh; ll01 += (u64)pp.w * bl;
                    hh10 += (u64)rr.x * ah; md10 += (u64)rr.x * al + (u64)rr.y * ah; ll10 += (u64)rr.y * al;
                    hh11 += (u64)rr.z * bh; md11 += (u64)rr.z * bl + (u64)rr.w * bh; ll11 += (u64)rr.w * bl;
#endif
                };
                if (rows == ROWS) {
#pragma unroll
                    for (int t = 0; t < ROWS; t++) row(t);
                } else {
                    for (int t = 0; t < rows; t++) row(t);
                }
#if MAC_KARA
                md00 -= hh00 + ll00; md01 -= hh01 + ll01; md10 -= hh10 + ll10; md11 -= hh11 + ll11;
#endif
                auto fold = [](U128& a, u64 hh, u64 md, u64 ll) {
                    add128(a, ll);
                    add128(a, md << 30);
                    a.hi += md >> 34;
                    add128(a, hh << 60);
                    a.hi += hh >> 4;
                };
                fold(a00, hh00, md00, ll00); fold(a01, hh01, md01, ll01);
                fold(a10, hh10, md10, ll10); fold(a11, hh11, md11, ll11);
                if ((((c + 1) * ROWS) & 31) == 0) {     // every 32 products (< 32 q^2 <= 2^127 for q < 2^61): fold below q
                    a00 = U128{barrett128(a00, mc.q, mc.rhi, mc.rlo), 0}; a01 = U128{barrett128(a01, mc.q, mc.rhi, mc.rlo), 0};
                    a10 = U128{barrett128(a10, mc.q, mc.rhi, mc.rlo), 0}; a11 = U128{barrett128(a11, mc.q, mc.rhi, mc.rlo), 0};
                }
            }
            if (c == nch - 1) {
                u64* o = acc + (size_t)u * accs + (size_t)limb * N + k0 + 2 * kp;
                if constexpr (NARROW) {
                    if (fpw) {   // the FP64 warps' sums are exact integers < 2^53 held as double bits
                        auto cv = [](u64& a) { a = (u64)__double2ull_rn(__longlong_as_double((long long)a)); };
                        cv(h00); cv(l00); cv(s00); cv(h01); cv(l01); cv(s01); cv(h10); cv(l10); cv(s10); cv(h11); cv(l11); cv(s11);
                    }
                    *(ulonglong2*)o = make_ulonglong2(kara_combine(h00, l00, s00, mc.q, mc.rhi, mc.rlo, t40),
                                                      kara_combine(h01, l01, s01, mc.q, mc.rhi, mc.rlo, t40));
                    *(ulonglong2*)(o + cs) = make_ulonglong2(kara_combine(h10, l10, s10, mc.q, mc.rhi, mc.rlo, t40),
                                                             kara_combine(h11, l11, s11, mc.q, mc.rhi, mc.rlo, t40));
                    h00 = l00 = s00 = h01 = l01 = s01 = h10 = l10 = s10 = h11 = l11 = s11 = 0;
                } else {
                    *(ulonglong2*)o = make_ulonglong2(barrett128(a00, mc.q, mc.rhi, mc.rlo), barrett128(a01, mc.q, mc.rhi, mc.rlo));
                    *(ulonglong2*)(o + cs) = make_ulonglong2(barrett128(a10, mc.q, mc.rhi, mc.rlo),
                                                             barrett128(a11, mc.q, mc.rhi, mc.rlo));
                    a00 = a01 = a10 = a11 = U128{0, 0};
                }
            }
        }
        __syncthreads();     // every thread is done with this slot: it may be refilled
    }
}

// ------------------------------------------------------------------------------------ export (Alg 3 step 1)
__global__ void export_mask_kernel(u64 seed, u64 stream, u64* c0, u64* share, int level, int N, const ModConst* mod) {
    size_t total = (size_t)level * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)(i / N), k = (int)(i % N);
        u64 q = mod[limb].q;
        u64 idx = 2 * ((u64)limb * (u64)N + (u64)k);
        u64 hi = prng_draw(seed, stream, idx), lo = prng_draw(seed, stream, idx + 1);
        u64 a_lo = hi * q, a_hi = umulhi(hi, q), b = umulhi(lo, q);
        u64 s = a_lo + b;
        u64 r = a_hi + (s < a_lo);
        c0[i] = add_mod(c0[i], r, q);
        share[i] = r ? q - r : 0;
    }
}

// ------------------------------------------------------------------------------------ float64 encode / decode
// S_k = sum_e A[e] exp(sign * 2 pi i e k / 2N): iterative radix-2 FFT of length 2N in global memory
// (preprocessing only: weights and masks are encoded once).
__global__ void fft_bitrev_kernel(double2* a, int n2, int logn2) {
    a += (size_t)blockIdx.y * n2;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += gridDim.x * blockDim.x) {
        int j = (int)(__brev((unsigned)i) >> (32 - logn2));
        if (i < j) { double2 t = a[i]; a[i] = a[j]; a[j] = t; }
    }
}

__global__ void fft_stage_kernel(double2* a, int n2, int len, double sign) {
    a += (size_t)blockIdx.y * n2;
    int half = len / 2;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n2 / 2; b += gridDim.x * blockDim.x) {
        int grp = b / half, j = b % half;
        int i0 = grp * len + j, i1 = i0 + half;
        double s, c;
        sincospi(sign * 2.0 * (double)j / (double)len, &s, &c);
        double2 u = a[i0], v = a[i1];
        double2 t = make_double2(v.x * c - v.y * s, v.x * s + v.y * c);
        a[i0] = make_double2(u.x + t.x, u.y + t.y);
        a[i1] = make_double2(u.x - t.x, u.y - t.y);
    }
}

__global__ void scatter_slots_kernel(const double* re, const double* im, int n_slots, const int* rg, double2* A) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_slots; j += gridDim.x * blockDim.x)
        A[rg[j]] = make_double2(re[j], im ? im[j] : 0.0);
}

__global__ void round_reduce_kernel(const double2* S, double f, int N, int level, const ModConst* mod, u64* out, int* overflow,
                                    LimbMap lm) {
    S += (size_t)blockIdx.y * 2 * N;
    out += (size_t)blockIdx.y * level * N;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        double v = rint(f * S[k].x);   // round half to even
        if (fabs(v) >= 4611686018427387904.0) { *overflow = 1; v = 0; }
        i64 x = (i64)v;
        for (int l = 0; l < level; l++) {
            u64 q = mod[lm.mod[l]].q;
            u64 r = (u64)(x < 0 ? -x : x) % q;
            out[(size_t)l * N + k] = (x < 0 && r) ? q - r : r;
        }
    }
}

__global__ void lift_limb0_kernel(const u64* c, int N, const ModConst* mod, double2* A) {
    u64 q = mod[0].q;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < 2 * N; k += gridDim.x * blockDim.x) {
        double v = 0.0;
        if (k < N) {
            u64 x = c[k];
            v = x > q / 2 ? -(double)(q - x) : (double)x;
        }
        A[k] = make_double2(v, 0.0);
    }
}

__global__ void gather_slots_kernel(const double2* Z, const int* rg, int n, double inv_scale, double* re, double* im) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        double2 z = Z[rg[j]];
        re[j] = z.x * inv_scale;
        im[j] = z.y * inv_scale;
    }
}

void fft2n(encf_ctx& c, double2* A, double sign, cudaStream_t s, int batch = 1) {
    int n2 = 2 * c.N, logn2 = c.logN + 1;
    dim3 g1(nblocks(n2, TB, 512), batch), g2(nblocks(n2 / 2, TB, 256), batch);
    fft_bitrev_kernel<<<g1, TB, 0, s>>>(A, n2, logn2);
    for (int len = 2; len <= n2; len <<= 1) fft_stage_kernel<<<g2, TB, 0, s>>>(A, n2, len, sign);
}

// Projection weight diagonals straight into the FFT input: for plaintext (b,p,u,q) the
// slot r + c m (c < C) holds Wbar[(2u)C + alpha, bC + beta] - i Wbar[(2u+1)C + alpha, bC + beta],
// alpha = (c+q) mod C, beta = (c - p N1) mod C; A[5^j mod 2N] = slot j.
struct WDiag { int b[64], p[64], u[64], q[64]; };
// Wim != nullptr: real-input (fused-QK) plan, w~(c) = Wre[uC + alpha, col] + i Wim[uC + alpha, col].
__global__ void weight_slots_kernel(const double* __restrict__ W, int d_in, int d_out, int C, int N1, int m, WDiag wd,
                                    const int* rg, double2* A, int N, const double* __restrict__ Wim, int real_input) {
    const int bi = blockIdx.y;
    double2* a = A + (size_t)bi * 2 * N;
    const int b = wd.b[bi], p = wd.p[bi], u = wd.u[bi], q = wd.q[bi];
    const int n = N / 2;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        int c = j / m;
        double re = 0.0, im = 0.0;
        if (c < C) {
            int al = (c + q) % C, be = ((c - p * N1) % C + C) % C;
            int col = b * C + be;
            if (col < d_out) {
                if (real_input) {
                    int r0 = u * C + al;
                    if (r0 < d_in) { re = W[(size_t)r0 * d_out + col]; im = Wim ? Wim[(size_t)r0 * d_out + col] : 0.0; }
                } else {
                    int r0 = 2 * u * C + al, r1 = (2 * u + 1) * C + al;
                    if (r0 < d_in) re = W[(size_t)r0 * d_out + col];
                    if (r1 < d_in) im = -W[(size_t)r1 * d_out + col];
                }
            }
        }
        a[rg[j]] = make_double2(re, im);
    }
}

}  // namespace

// ====================================================================================== launchers
#define GRID(total) nblocks((size_t)(total))

void k_add(encf_ctx& c, const u64* a, const u64* b, u64* out, int npolys, const LimbMap& m, bool sub, cudaStream_t s) {
    size_t total = (size_t)npolys * m.n * c.N;
    { int _slot; c.prof_begin("add_kernel", s, 0, _slot);
    add_kernel<<<GRID(total), TB, 0, s>>>(a, b, out, total, c.N, m, c.d_mod, sub ? 1 : 0);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += total * 24;
}

void k_mul(encf_ctx& c, const u64* a, i64 as, const u64* b, i64 bs, u64* out, i64 os, int npolys, const LimbMap& m,
           cudaStream_t s) {
    size_t total = (size_t)npolys * m.n * c.N;
    { int _slot; c.prof_begin("mul_kernel", s, 0, _slot);
    mul_kernel<<<GRID(total), TB, 0, s>>>(a, as, b, bs, out, os, npolys, c.N, m, c.d_mod);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += total * 24;
}

void k_mul_i(encf_ctx& c, const u64* a, u64* out, int npolys, const LimbMap& m, cudaStream_t s) {
    size_t total = (size_t)npolys * m.n * c.N;
    { int _slot; c.prof_begin("mul_i_kernel", s, 0, _slot);
    mul_i_kernel<<<GRID(total), TB, 0, s>>>(a, out, total, c.N, m, c.d_mod, c.d_imag, c.d_imag_sh);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += total * 16;
}

void k_add_i_batch(encf_ctx& c, const AddIBatch& B, int n, int npolys, const LimbMap& m, bool sub, cudaStream_t s) {
    const size_t per = (size_t)npolys * m.n * c.N, total = per * n;
    { int _slot; c.prof_begin("add_i_batch_kernel", s, 0, _slot);
    add_i_batch_kernel<<<GRID(total), TB, 0, s>>>(B, n, per, c.N, m, c.d_mod, c.d_imag, c.d_imag_sh, sub ? 1 : 0);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += total * 24;
}

void k_automorph(encf_ctx& c, const u64* in, i64 is, u64* out, i64 os, int npolys, int nlimbs, uint32_t g, cudaStream_t s) {
    size_t total = (size_t)npolys * nlimbs * c.N;
    { int _slot; c.prof_begin("automorph_kernel", s, 0, _slot);
    automorph_kernel<<<GRID(total), TB, 0, s>>>(in, is, out, os, npolys, nlimbs, c.N, c.logN, g);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += total * 16;
}

void k_copy(const u64* in, u64* out, size_t words, cudaStream_t s) {
    if (words && in != out) CUDA_TRY(cudaMemcpyAsync(out, in, words * 8, cudaMemcpyDeviceToDevice, s));
}

void k_sample_uniform(encf_ctx& c, u64 seed, u64 stream, u64* out, const LimbMap& m, const int* gids, cudaStream_t s) {
    Gids g;
    for (int i = 0; i < m.n; i++) g.g[i] = gids[i];
    { int _slot; c.prof_begin("sample_uniform_kernel", s, 0, _slot);
    sample_uniform_kernel<<<GRID((size_t)m.n * c.N), TB, 0, s>>>(seed, stream, out, c.N, m, g, c.d_mod);
    c.prof_end(_slot, s); }
    c.st_launch++;
}

void k_sample_small(encf_ctx& c, u64 seed, u64 stream, int kind, u64* out, const LimbMap& m, cudaStream_t s) {
    { int _slot; c.prof_begin("sample_small_kernel", s, 0, _slot);
    sample_small_kernel<<<GRID((size_t)m.n * c.N), TB, 0, s>>>(seed, stream, kind, out, c.N, m, c.d_mod);
    c.prof_end(_slot, s); }
    c.st_launch++;
}

// + sc_limb on every (NTT-domain) coefficient of one polynomial: a public constant added to the message
void k_add_scalar(encf_ctx& c, u64* data, const LimbMap& m, const u64* sc, cudaStream_t s) {
    add_scalar_kernel<<<GRID((size_t)m.n * c.N), TB, 0, s>>>(data, c.N, m, c.d_mod, sc);
    c.st_launch++;
    CUDA_TRY(cudaGetLastError());
}

void k_scalar_mul(encf_ctx& c, u64* data, int npolys, const LimbMap& m, const u64* sc, const u64* scs, cudaStream_t s) {
    { int _slot; c.prof_begin("scalar_mul_kernel", s, 0, _slot);
    scalar_mul_kernel<<<GRID((size_t)npolys * m.n * c.N), TB, 0, s>>>(data, npolys, c.N, m, c.d_mod, sc, scs);
    c.prof_end(_slot, s); }
    c.st_launch++;
}

void k_mod_reduce(encf_ctx& c, u64* data, int npolys, const LimbMap& m, cudaStream_t s) {
    size_t total = (size_t)npolys * m.n * c.N;
    { int _slot; c.prof_begin("mod_reduce_kernel", s, 0, _slot);
    mod_reduce_kernel<<<GRID(total), TB, 0, s>>>(data, total, c.N, m, c.d_mod);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += total * 16;
}

void k_rescale_prep(encf_ctx& c, const u64* last, u64* corr, int level, int ncomp, i64 ls, cudaStream_t s) {
    { int _slot; c.prof_begin("rescale_prep_kernel", s, 0, _slot);
    rescale_prep_kernel<<<GRID((size_t)ncomp * (level - 1) * c.N), TB, 0, s>>>(last, ls, corr, ncomp, level, c.N, c.d_mod,
                                                                            c.rescale[level].d_hmod);
    c.prof_end(_slot, s); }
    c.st_launch++;
}

void k_rescale_finish(encf_ctx& c, const u64* in, i64 is, const u64* corr, u64* out, i64 os, int ncomp, int level,
                      cudaStream_t s) {
    const RescaleTab& t = c.rescale[level];
    { int _slot; c.prof_begin("rescale_finish_kernel", s, 0, _slot);
    rescale_finish_kernel<<<GRID((size_t)ncomp * (level - 1) * c.N), TB, 0, s>>>(in, is, corr, out, os, ncomp, level, c.N,
                                                                              c.d_mod, t.d_inv, t.d_inv_sh);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += (size_t)ncomp * (level - 1) * c.N * 24;
}

void k_moddown_finish(encf_ctx& c, const u64* b, const u64* y, const u64* add0, u64* out, int level, const ModDownTab& t,
                      cudaStream_t s) {
    size_t total = (size_t)level * c.N;
    { int _slot; c.prof_begin("moddown_finish_kernel", s, 0, _slot);
    moddown_finish_kernel<<<GRID(total), TB, 0, s>>>(b, y, add0, out, level, c.N, c.d_mod, t.d_pinv, t.d_pinv_sh);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += total * (add0 ? 32 : 24);
}

void k_tensor_acc(encf_ctx& c, const u64* const* A, const u64* const* B, int nterms, u64* out3, int level, cudaStream_t s) {
    dim3 grid((c.N + TB - 1) / TB, level);
    { int _slot; c.prof_begin("tensor_acc_kernel", s, 0, _slot);
    tensor_acc_kernel<<<grid, TB, 0, s>>>(A, B, nterms, out3, level, c.N, c.d_mod);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += (size_t)nterms * 4 * level * c.N * 8 + (size_t)3 * level * c.N * 8;
    c.st_ctmul += nterms;
}

void k_masked_sum(encf_ctx& c, const u64* const* C, const u64* const* M, int nterms, u64* out, int level, cudaStream_t s) {
    dim3 grid((c.N + TB - 1) / TB, level);
    { int _slot; c.prof_begin("masked_sum_kernel", s, 0, _slot);
    masked_sum_kernel<<<grid, TB, 0, s>>>(C, M, nterms, out, level, c.N, c.d_mod);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += (size_t)nterms * 3 * level * c.N * 8 + (size_t)2 * level * c.N * 8;
    c.st_ptmul += nterms;
}

void k_diag_mac(encf_ctx& c, const u64* bank, int nbank, const u64* w, int units, i64 wus, u64* acc, i64 accs, int level,
                cudaStream_t s) {
    size_t smem = (size_t)nbank * 2 * MAC_T * sizeof(u64);   // narrow limbs: pre-split {h, l} uint2 per bank word
    if (nbank > 4096) throw EncfError(ENCF_ERR_PLAN_SHAPE, "diag_mac: more than 4096 bank ciphertexts (64-bit split sums)");
    static const int allow_narrow = std::getenv("ENCF_MAC_WIDE_ONLY") ? 0 : 1;   // experiment switch: 128-bit path everywhere
    static bool attr_set = false;
    if (!attr_set) {
        CUDA_TRY(cudaFuncSetAttribute(diag_mac_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CUDA_TRY(cudaFuncSetAttribute(diag_mac_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_set = true;
    }
    if (smem > 200 * 1024) throw EncfError(ENCF_ERR_PLAN_SHAPE, "diag_mac: bank too large for shared memory");
    int tiles = c.N / MAC_T;
    int zsplit = 1;
    while ((size_t)tiles * level * zsplit < 148 * 8 && zsplit * MAC_LANES < units) zsplit *= 2;
    // limbs [0, nw) on the 128-bit path, [nw, level) (q < 2^41) on the 20-bit Karatsuba path when enabled
    int nw = level;
    if (allow_narrow && nbank % 8 == 0) {
        nw = 0;
        while (nw < level && c.mods[nw] >= (1ull << 41)) nw++;
        for (int i = nw; i < level; i++)
            if (c.mods[i] >= (1ull << 41)) { nw = level; break; }
    }
    // algorithmic bytes: plaintext stream + bank read once + accumulators written once
    const uint64_t bytes = (uint64_t)units * nbank * level * c.N * 8 + (uint64_t)nbank * 2 * level * c.N * 8 +
                           (uint64_t)units * 2 * level * c.N * 8;
    int slot;
    c.prof_begin("diag_mac", s, bytes, slot);
    // Path (ENCF_MAC_VARIANT): "tma2" (default) = tensor-map TMA ring of 32 KB stages at 2 CTAs/SM, "tma1" = 32 KB
    // stages at 1 CTA/SM, "tma3" = 16 KB stages at 3 CTAs/SM, "reg" = register double buffer (diag_mac_kernel, 2 CTAs/SM).
    // Measured on the B200 (BERT layer, profiles/r02_summary.md): tma2 10.3 ms, reg 11.0, tma3 13.2, tma1 14.7; one launch
    // covering the 128-bit and the narrow limbs together (runtime path per CTA, 112 registers) was slower: 12.1 ms.
    // All paths give the same words.
    static const int variant = [] {
        const char* e = std::getenv("ENCF_MAC_VARIANT");
        if (!e) return 2;
        if (!strcmp(e, "reg")) return 0;
        if (!strcmp(e, "tma1")) return 1;
        if (!strcmp(e, "tma2")) return 2;
        if (!strcmp(e, "tma3")) return 3;
        return 0;
    }();
    const size_t bank_b = (size_t)nbank * 2 * MAC_T * 8;
    const int rows = variant == 3 ? 4 : 8;
    const size_t stage_b = (size_t)MAC_LANES * rows * MAC_T * 8;
    const size_t cap = variant == 1 ? 227 * 1024 : variant == 2 ? 113 * 1024 : 75 * 1024;
    // the TMA kernel's 128-bit limbs use a 30-bit split (q < 2^60); larger moduli take the register path
    const int nst = variant && c.max_mod < (1ull << 60) && bank_b + 2 * stage_b + 64 <= cap
                        ? (int)std::min<size_t>(DM_MAX_STAGES, (cap - bank_b - 64) / stage_b) : 0;
    if (nst >= 2) {
        static bool tma_attr = false;
        if (!tma_attr) {
            const int mx = 227 * 1024;
            CUDA_TRY(cudaFuncSetAttribute(diag_mac_tma_kernel<false, 8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            CUDA_TRY(cudaFuncSetAttribute(diag_mac_tma_kernel<true, 8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            CUDA_TRY(cudaFuncSetAttribute(diag_mac_tma_kernel<false, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            CUDA_TRY(cudaFuncSetAttribute(diag_mac_tma_kernel<true, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            CUDA_TRY(cudaFuncSetAttribute(diag_mac_tma_kernel<false, 4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            CUDA_TRY(cudaFuncSetAttribute(diag_mac_tma_kernel<true, 4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
            tma_attr = true;
        }
        const size_t tsm = (size_t)nst * stage_b + bank_b + (size_t)nst * 8;
        const int groups = (units + MAC_LANES - 1) / MAC_LANES;
        int zs = 1;
        const int per_sm = variant == 1 ? 1 : variant;
        while ((size_t)tiles * level * zs < (size_t)148 * per_sm && zs < groups) zs *= 2;
        // the weight stream as a 4-D tensor [units][nbank][level][N] for the TMA engine
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        if (!encode) {
            cudaDriverEntryPointQueryResult qr;
            CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &qr));
            if (qr != cudaDriverEntryPointSuccess || !encode) throw EncfError(ENCF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        }
        CUtensorMap tm;
        const cuuint64_t dims[4] = {(cuuint64_t)c.N, (cuuint64_t)level, (cuuint64_t)nbank, (cuuint64_t)units};
        const cuuint64_t strides[3] = {(cuuint64_t)c.N * 8, (cuuint64_t)level * c.N * 8, (cuuint64_t)wus * 8};
        const cuuint32_t box[4] = {MAC_T, 1, (cuuint32_t)rows, MAC_LANES};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, (void*)w, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            throw EncfError(ENCF_ERR_CUDA, "diag_mac: cuTensorMapEncodeTiled failed");
        auto launch = [&](auto kw, auto kn) {
            if (nw > 0)
                kw<<<dim3(tiles, nw, zs), MAC_TPR * MAC_LANES, tsm, s>>>(tm, bank, nbank, w, units, wus, acc, accs, level, c.N,
                                                                       c.d_mod, 0, nst, 0);
            // narrow limbs: warps 4-7 on the FP64 pipe (exact while nbank <= 512; ENCF_MAC_FP=0: integer pipe only)
            static const int fp_env = [] { const char* e = std::getenv("ENCF_MAC_FP"); return e ? std::atoi(e) : 1; }();
            const int fp_split = fp_env && nbank <= 512 ? 1 : 0;
            if (nw < level)
                kn<<<dim3(tiles, level - nw, zs), MAC_TPR * MAC_LANES, tsm, s>>>(tm, bank, nbank, w, units, wus, acc, accs, level,
                                                                               c.N, c.d_mod, nw, nst, fp_split);
        };
        if (variant == 1) launch(diag_mac_tma_kernel<false, 8, 1>, diag_mac_tma_kernel<true, 8, 1>);
        else if (variant == 2) launch(diag_mac_tma_kernel<false, 8, 2>, diag_mac_tma_kernel<true, 8, 2>);
        else launch(diag_mac_tma_kernel<false, 4, 3>, diag_mac_tma_kernel<true, 4, 3>);
    } else {
        if (nw > 0)
            diag_mac_kernel<false><<<dim3(tiles, nw, zsplit), MAC_TPR * MAC_LANES, smem, s>>>(bank, nbank, w, units, wus, acc, accs,
                                                                                            level, c.N, c.d_mod, 0);
        if (nw < level)
            diag_mac_kernel<true><<<dim3(tiles, level - nw, zsplit), MAC_TPR * MAC_LANES, smem, s>>>(bank, nbank, w, units, wus, acc,
                                                                                                   accs, level, c.N, c.d_mod, nw);
    }
    c.prof_end(slot, s);
    c.st_launch += (nw > 0 ? 1 : 0) + (nw < level ? 1 : 0);   // the 128-bit and the narrow launch
    c.st_bytes += bytes;
    c.st_ptmul += (uint64_t)units * nbank;
}

// The same mask with (seed, stream id base) read from DEVICE memory at run time: a CUDA-graph replay then draws the
// masks of whatever (seed, base) the buffer holds, so a step that advances the base every replay never reuses a
// one-time pad across inferences.  stream = mask(dss[1] + idx).
__global__ void export_mask_dev_kernel(const u64* __restrict__ dss, u64 idx, u64* c0, u64* share, int level, int N,
                                       const ModConst* mod) {
    const u64 seed = dss[0], stream = (0x04ull << 56) | ((dss[1] + idx) & ((1ull << 56) - 1));
    size_t total = (size_t)level * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)(i / N), k = (int)(i % N);
        u64 q = mod[limb].q;
        u64 id = 2 * ((u64)limb * (u64)N + (u64)k);
        u64 hi = prng_draw(seed, stream, id), lo = prng_draw(seed, stream, id + 1);
        u64 a_lo = hi * q, a_hi = umulhi(hi, q), b = umulhi(lo, q);
        u64 s = a_lo + b;
        u64 r = a_hi + (s < a_lo);
        c0[i] = add_mod(c0[i], r, q);
        share[i] = r ? q - r : 0;
    }
}

void k_export_mask_dev(encf_ctx& c, const u64* dss, u64 idx, u64* c0, u64* share, int level, cudaStream_t s) {
    { int _slot; c.prof_begin("export_mask_kernel", s, 0, _slot);
    export_mask_dev_kernel<<<GRID((size_t)level * c.N), TB, 0, s>>>(dss, idx, c0, share, level, c.N, c.d_mod);
    c.prof_end(_slot, s); }
    c.st_launch++;
}

void k_export_mask(encf_ctx& c, u64 seed, u64 stream, u64* c0, u64* share, int level, cudaStream_t s) {
    { int _slot; c.prof_begin("export_mask_kernel", s, 0, _slot);
    export_mask_kernel<<<GRID((size_t)level * c.N), TB, 0, s>>>(seed, stream, c0, share, level, c.N, c.d_mod);
    c.prof_end(_slot, s); }
    c.st_launch++;
}

void k_encode_slots(encf_ctx& c, const double* re, const double* im, int n_slots, double scale, int level, u64* out,
                    cudaStream_t s, const LimbMap* lmap) {
    Scratch sc(s);
    double2* A = (double2*)sc.get((size_t)2 * c.N * 2);
    int* ovf = (int*)sc.get(1);
    CUDA_TRY(cudaMemsetAsync(A, 0, sizeof(double2) * 2 * c.N, s));
    CUDA_TRY(cudaMemsetAsync(ovf, 0, sizeof(int), s));
    { int _slot; c.prof_begin("scatter_slots_kernel", s, 0, _slot);
    scatter_slots_kernel<<<GRID(n_slots), TB, 0, s>>>(re, im, n_slots, c.d_rot_group, A);
    c.prof_end(_slot, s); }
    fft2n(c, A, -1.0, s);
    { int _slot; c.prof_begin("round_reduce_kernel", s, 0, _slot);
    round_reduce_kernel<<<GRID(c.N), TB, 0, s>>>(A, scale * 2.0 / c.N, c.N, lmap ? lmap->n : level, c.d_mod, out, ovf,
                                              lmap ? *lmap : c.qmap(level));
    c.prof_end(_slot, s); }
    int h_ovf = 0;
    CUDA_TRY(cudaMemcpyAsync(&h_ovf, ovf, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (h_ovf) throw EncfError(ENCF_ERR_OVERFLOW, "encode: |coefficient| >= 2^62");
}

void k_encode_weights(encf_ctx& c, const double* dW, int d_in, int d_out, int C, int N1, int m, const int* bs, const int* ps,
                      const int* us, const int* qs, int batch, double scale, int level, u64* out, cudaStream_t s,
                      const double* dWim, int real_input) {
    Scratch sc(s);
    double2* A = (double2*)sc.get((size_t)batch * 2 * c.N * 2);
    int* ovf = (int*)sc.get(1);
    CUDA_TRY(cudaMemsetAsync(A, 0, sizeof(double2) * 2 * c.N * batch, s));
    CUDA_TRY(cudaMemsetAsync(ovf, 0, sizeof(int), s));
    WDiag wd;
    for (int i = 0; i < batch; i++) { wd.b[i] = bs[i]; wd.p[i] = ps[i]; wd.u[i] = us[i]; wd.q[i] = qs[i]; }
    { int _slot; c.prof_begin("weight_slots_kernel", s, 0, _slot);
    weight_slots_kernel<<<dim3(nblocks(c.N / 2, TB, 256), batch), TB, 0, s>>>(dW, d_in, d_out, C, N1, m, wd, c.d_rot_group, A, c.N,
                                                                              dWim, real_input);
    c.prof_end(_slot, s); }
    fft2n(c, A, -1.0, s, batch);
    { int _slot; c.prof_begin("round_reduce_kernel", s, 0, _slot);
    round_reduce_kernel<<<dim3(nblocks(c.N, TB, 256), batch), TB, 0, s>>>(A, scale * 2.0 / c.N, c.N, level, c.d_mod, out, ovf,
                                                                         c.qmap(level));
    c.prof_end(_slot, s); }
    int h_ovf = 0;
    CUDA_TRY(cudaMemcpyAsync(&h_ovf, ovf, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (h_ovf) throw EncfError(ENCF_ERR_OVERFLOW, "encode: |coefficient| >= 2^62");
}

void k_decode_limb0(encf_ctx& c, const u64* coeff0, double scale, double* re, double* im, cudaStream_t s) {
    Scratch sc(s);
    double2* A = (double2*)sc.get((size_t)2 * c.N * 2);
    { int _slot; c.prof_begin("lift_limb0_kernel", s, 0, _slot);
    lift_limb0_kernel<<<GRID(2 * c.N), TB, 0, s>>>(coeff0, c.N, c.d_mod, A);
    c.prof_end(_slot, s); }
    fft2n(c, A, +1.0, s);
    { int _slot; c.prof_begin("gather_slots_kernel", s, 0, _slot);
    gather_slots_kernel<<<GRID(c.N / 2), TB, 0, s>>>(A, c.d_rot_group, c.N / 2, 1.0 / scale, re, im);
    c.prof_end(_slot, s); }
}

// ====================================================================================== batched key switching
// (many independent key switches / rotations / rescales per launch: fills the 148 SMs and removes the
// per-ciphertext launch sequence).  Request tables travel by value as kernel parameters.
namespace {

#ifndef KS_PAIRS_V
#define KS_PAIRS_V 2
#endif
constexpr int KS_PAIRS = KS_PAIRS_V;
#ifndef KS_MINB
#define KS_MINB 2
#endif
__global__ void __launch_bounds__(TB, KS_MINB) ks_inner_batch_kernel(KsInnerBatch B, int dnum, int nl, int key_nl, KeyLimb klm,
                                                            LimbMap em, int N, int logN, const ModConst* __restrict__ mod) {
    // Two coefficients (k, k+1), k even, per thread: the Galois gather maps them to the aligned pair
    // {s, s^1} (brv flips the low bit), so every operand moves with 128-bit loads.
    const int r = blockIdx.z, e = blockIdx.y;
    const u64* __restrict__ ext = B.ext[r];
    const u64* __restrict__ key = B.key[r];
    u64* __restrict__ acc = B.acc[r];
    const uint32_t g = B.gather[r];
    const ModConst mc = mod[em.mod[e]];
    const int kle = klm.kl[e];
    const uint32_t mask2n = 2 * N - 1;
    // KS_PAIRS coefficient pairs per thread (kp, kp + stride, ...): every pair's ext and key loads are issued
    // before the first multiply (the one-pair loop was long_scoreboard-bound at 3.6 TB/s, profiles/r01_ncu_top_kernels_s4.md)
    const int stride = gridDim.x * blockDim.x;
    for (int kp0 = blockIdx.x * blockDim.x + threadIdx.x; 2 * kp0 < N; kp0 += KS_PAIRS * stride) {
        int kk[KS_PAIRS], base[KS_PAIRS], swap[KS_PAIRS];
        bool ok[KS_PAIRS];
#pragma unroll
        for (int p = 0; p < KS_PAIRS; p++) {
            const int k = 2 * (kp0 + p * stride);
            ok[p] = k < N;
            kk[p] = ok[p] ? k : 0;
            base[p] = kk[p];
            swap[p] = 0;
            if (g != 1) {
                uint32_t ee = 2u * (uint32_t)brv(kk[p], logN) + 1u;
                uint32_t e2 = (uint32_t)(((uint64_t)ee * g) & mask2n);
                int src = brv((int)((e2 - 1) >> 1), logN);
                base[p] = src & ~1;
                swap[p] = src & 1;
            }
        }
        U128 a0[KS_PAIRS], a1[KS_PAIRS], b0[KS_PAIRS], b1[KS_PAIRS];
#pragma unroll
        for (int p = 0; p < KS_PAIRS; p++) a0[p] = a1[p] = b0[p] = b1[p] = U128{0, 0};
        for (int j = 0; j < dnum; j++) {
            const u64* kj = key + (size_t)j * 2 * key_nl * N;
            ulonglong2 x[KS_PAIRS], k0[KS_PAIRS], k1[KS_PAIRS];
#pragma unroll
            for (int p = 0; p < KS_PAIRS; p++) {
                x[p] = __ldg((const ulonglong2*)(ext + ((size_t)j * nl + e) * N + base[p]));
                k0[p] = __ldg((const ulonglong2*)(kj + (size_t)kle * N + kk[p]));
                k1[p] = __ldg((const ulonglong2*)(kj + ((size_t)key_nl + kle) * N + kk[p]));
            }
#pragma unroll
            for (int p = 0; p < KS_PAIRS; p++) {
                if (swap[p]) { u64 t = x[p].x; x[p].x = x[p].y; x[p].y = t; }
                mac128(a0[p], x[p].x, k0[p].x);
                mac128(b0[p], x[p].y, k0[p].y);
                mac128(a1[p], x[p].x, k1[p].x);
                mac128(b1[p], x[p].y, k1[p].y);
            }
        }
        // keys are stored in Montgomery form (k R mod q, R = 2^64): one REDC returns sum_j x_j k_j mod q
#pragma unroll
        for (int p = 0; p < KS_PAIRS; p++) {
            if (!ok[p]) continue;
            *(ulonglong2*)(acc + (size_t)e * N + kk[p]) =
                make_ulonglong2(redc128(a0[p], mc.q, mc.qinv), redc128(b0[p], mc.q, mc.qinv));
            *(ulonglong2*)(acc + ((size_t)nl + e) * N + kk[p]) =
                make_ulonglong2(redc128(a1[p], mc.q, mc.qinv), redc128(b1[p], mc.q, mc.qinv));
        }
    }
}

// The same inner product with the operands staged by the TMA engine (ENCF_KS_TMA, default on for N >= 1024): a CTA owns
// an aligned tile of KT = 1024 coefficients of one (request, extended limb).  The Galois gather maps an aligned
// 2^k-block of NTT-domain indices onto ONE aligned 2^k-block (brv keeps the block's low bits of 2 brv(i) + 1 fixed,
// and multiplying by an odd g keeps them fixed), so per digit j three contiguous 8 KB bulk copies (cp.async.bulk,
// SASS UBLKCP) bring the source ext block and the two key tiles into shared memory, all dnum digits issued up front on
// one mbarrier each (up to 72 KB in flight per CTA); the threads then read their permuted pairs from shared memory.
// Same arithmetic and output words as ks_inner_batch_kernel.
constexpr int KT = 1024;
template <int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 3 : 4) ks_inner_tma_kernel(KsInnerBatch B, int dnum, int nl, int key_nl, KeyLimb klm,
                                                                    LimbMap em, int N, int logN, const ModConst* __restrict__ mod,
                                                                    int Lq, const u64* __restrict__ pl,
                                                                    const u64* __restrict__ pl_sh, int lift_slot) {
    // [dnum][3][KT]: ext block, key comp 0, key comp 1 | [lift_slot][KT] the c0 (c1) blocks of a lift | [dnum] mbarriers
    extern __shared__ __align__(128) u64 kt_sm[];
    u64* c0t = kt_sm + (size_t)dnum * 3 * KT;
    u64* c1t = c0t + KT;
    uint64_t* bars = (uint64_t*)(c0t + (size_t)lift_slot * KT);
    const int r = blockIdx.z, e = blockIdx.y;
    const int kb = blockIdx.x * KT;
    const u64* __restrict__ ext = B.ext[r];
    const u64* __restrict__ key = B.key[r];
    const uint32_t g = B.gather[r];
    const u64* __restrict__ c0 = e < Lq ? B.c0[r] : nullptr;    // lift P sigma_{g0}(c0) into component 0 (q-limbs)
    const u64* __restrict__ c1 = c0 ? B.c1[r] : nullptr;        // ... and P sigma_{g0}(c1) into component 1
    const uint32_t g0 = B.g0[r];
    const uint32_t mask2n = 2 * N - 1;
    auto src_of_g = [&](int k, uint32_t gg) -> int {
        if (gg == 1) return k;
        const uint32_t ee = 2u * (uint32_t)brv(k, logN) + 1u;
        const uint32_t e2 = (uint32_t)(((uint64_t)ee * gg) & mask2n);
        return brv((int)((e2 - 1) >> 1), logN);
    };
    auto src_of = [&](int k) -> int { return src_of_g(k, g); };
    const int sb = src_of(kb) & ~(KT - 1);             // the aligned source block of this tile
    const int sb0 = c0 ? src_of_g(kb, g0) & ~(KT - 1) : 0;
    const int kle = klm.kl[e];
    if (threadIdx.x == 0) {
        for (int j = 0; j < dnum; j++) mbar_init(&bars[j], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int j = 0; j < dnum; j++) {
            u64* st = kt_sm + (size_t)j * 3 * KT;
            const u64* kj = key + (size_t)j * 2 * key_nl * N;
            mbar_arrive_expect_tx(&bars[j], (3 + (j == 0 && c0 ? 1 : 0) + (j == 0 && c1 ? 1 : 0)) * KT * 8);
            bulk_g2s(st, ext + ((size_t)j * nl + e) * N + sb, KT * 8, &bars[j]);
            bulk_g2s(st + KT, kj + (size_t)kle * N + kb, KT * 8, &bars[j]);
            bulk_g2s(st + 2 * KT, kj + ((size_t)key_nl + kle) * N + kb, KT * 8, &bars[j]);
            if (j == 0 && c0) bulk_g2s(c0t, c0 + (size_t)e * N + sb0, KT * 8, &bars[0]);
            if (j == 0 && c1) bulk_g2s(c1t, c1 + (size_t)e * N + sb0, KT * 8, &bars[0]);
        }
    }
    __syncthreads();                                    // barrier initialisation visible to every waiting thread
    const ModConst mc = mod[em.mod[e]];
    constexpr int PP = KT / 2 / NT;                     // coefficient pairs per thread
    int kl[PP], sl[PP], sw[PP];
#pragma unroll
    for (int p = 0; p < PP; p++) {
        kl[p] = 2 * (threadIdx.x + p * NT);             // local coefficient (even)
        const int src = src_of(kb + kl[p]);
        sl[p] = (src & ~1) - sb;
        sw[p] = src & 1;
    }
    U128 a0[PP], a1[PP], b0[PP], b1[PP];
#pragma unroll
    for (int p = 0; p < PP; p++) a0[p] = a1[p] = b0[p] = b1[p] = U128{0, 0};
    for (int j = 0; j < dnum; j++) {
        mbar_wait(&bars[j], 0);
        const u64* st = kt_sm + (size_t)j * 3 * KT;
#pragma unroll
        for (int p = 0; p < PP; p++) {
            ulonglong2 x = *(const ulonglong2*)(st + sl[p]);
            const ulonglong2 k0 = *(const ulonglong2*)(st + KT + kl[p]);
            const ulonglong2 k1 = *(const ulonglong2*)(st + 2 * KT + kl[p]);
            if (sw[p]) { u64 t = x.x; x.x = x.y; x.y = t; }
            mac128(a0[p], x.x, k0.x);
            mac128(b0[p], x.y, k0.y);
            mac128(a1[p], x.x, k1.x);
            mac128(b1[p], x.y, k1.y);
        }
    }
    u64* __restrict__ acc = B.acc[r];
    const u64 f = c0 ? pl[e] : 0, fs = c0 ? pl_sh[e] : 0;
#pragma unroll
    for (int p = 0; p < PP; p++) {
        u64 o0 = redc128(a0[p], mc.q, mc.qinv), o1 = redc128(b0[p], mc.q, mc.qinv);
        if (c0) {   // + P sigma_{g0}(c0): the words of k_lift_add over a gathered c0 (add_mod of the Shoup product)
            const int src = src_of_g(kb + kl[p], g0);
            ulonglong2 y = *(const ulonglong2*)(c0t + (src & ~1) - sb0);
            if (src & 1) { const u64 t = y.x; y.x = y.y; y.y = t; }
            o0 = add_mod(o0, mul_shoup(y.x, f, fs, mc.q), mc.q);
            o1 = add_mod(o1, mul_shoup(y.y, f, fs, mc.q), mc.q);
        }
        *(ulonglong2*)(acc + (size_t)e * N + kb + kl[p]) = make_ulonglong2(o0, o1);
        u64 o2 = redc128(a1[p], mc.q, mc.qinv), o3 = redc128(b1[p], mc.q, mc.qinv);
        if (c1) {
            const int src = src_of_g(kb + kl[p], g0);
            ulonglong2 y = *(const ulonglong2*)(c1t + (src & ~1) - sb0);
            if (src & 1) { const u64 t = y.x; y.x = y.y; y.y = t; }
            o2 = add_mod(o2, mul_shoup(y.x, f, fs, mc.q), mc.q);
            o3 = add_mod(o3, mul_shoup(y.y, f, fs, mc.q), mc.q);
        }
        *(ulonglong2*)(acc + ((size_t)nl + e) * N + kb + kl[p]) = make_ulonglong2(o2, o3);
    }
}

// Grouped extended-basis rotation sums (KsGroupBatch): CTA = (tile of KT coefficients, extended limb e, group z); the
// group's requests stream through a two-stage cp.async.bulk ring (per stage: every digit's ext block, both key tiles and,
// on q-limbs, the Galois source block of c0), one request's products are reduced once (REDC) and summed mod q in
// registers, and the group's P x0 lift is added at the end.  The same residues as ks_inner + lift + sum_many_ext.
constexpr int KG_NT = 256, KG_PP = KT / 2 / KG_NT;
__global__ void __launch_bounds__(KG_NT, 2) ks_group_tma_kernel(KsGroupBatch B, int dnum, int nl, int L, int key_nl, KeyLimb klm,
                                                               LimbMap em, int N, int logN, const ModConst* __restrict__ mod,
                                                               const u64* __restrict__ pl, const u64* __restrict__ pl_sh) {
    extern __shared__ __align__(128) u64 kg_sm[];      // [2 stages][3 dnum + 1][KT] | [2] mbarriers
    const int per = 3 * dnum + 1;
    uint64_t* bars = (uint64_t*)(kg_sm + (size_t)2 * per * KT);
    const int z = blockIdx.z, e = blockIdx.y;
    const int kb = blockIdx.x * KT;
    const int r0 = B.start[z], r1 = B.start[z + 1];
    const bool qlimb = e < L;
    const int kle = klm.kl[e];
    const uint32_t mask2n = 2 * N - 1;
    auto src_of_g = [&](int k, uint32_t gg) -> int {
        if (gg == 1) return k;
        const uint32_t ee = 2u * (uint32_t)brv(k, logN) + 1u;
        const uint32_t e2 = (uint32_t)(((uint64_t)ee * gg) & mask2n);
        return brv((int)((e2 - 1) >> 1), logN);
    };
    auto issue = [&](int r) {   // thread 0: request r into stage (r - r0) & 1
        if (r >= r1) return;
        const int slot = (r - r0) & 1;
        u64* st = kg_sm + (size_t)slot * per * KT;
        const u64* c0 = qlimb ? B.c0[r] : nullptr;
        mbar_arrive_expect_tx(&bars[slot], (uint32_t)((3 * dnum + (c0 ? 1 : 0)) * KT * 8));
        for (int j = 0; j < dnum; j++) {
            const u64* kj = B.key[r] + (size_t)j * 2 * key_nl * N;
            bulk_g2s(st + (3 * j) * KT, B.ext[r] + ((size_t)j * nl + e) * N + kb, KT * 8, &bars[slot]);
            bulk_g2s(st + (3 * j + 1) * KT, kj + (size_t)kle * N + kb, KT * 8, &bars[slot]);
            bulk_g2s(st + (3 * j + 2) * KT, kj + ((size_t)key_nl + kle) * N + kb, KT * 8, &bars[slot]);
        }
        if (c0) bulk_g2s(st + (3 * dnum) * KT, c0 + (size_t)e * N + (src_of_g(kb, B.g[r]) & ~(KT - 1)), KT * 8, &bars[slot]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        issue(r0);
        issue(r0 + 1);
    }
    __syncthreads();
    const ModConst mc = mod[em.mod[e]];
    const u64 q = mc.q;
    const u64 f = qlimb ? pl[e] : 0, fs = qlimb ? pl_sh[e] : 0;
    u64 s0[KG_PP][2], s1[KG_PP][2];
#pragma unroll
    for (int p = 0; p < KG_PP; p++) s0[p][0] = s0[p][1] = s1[p][0] = s1[p][1] = 0;
    for (int r = r0; r < r1; r++) {
        const int it = r - r0, slot = it & 1;
        mbar_wait(&bars[slot], (uint32_t)((it >> 1) & 1));
        const u64* st = kg_sm + (size_t)slot * per * KT;
        U128 a0[KG_PP], b0[KG_PP], a1[KG_PP], b1[KG_PP];
#pragma unroll
        for (int p = 0; p < KG_PP; p++) a0[p] = b0[p] = a1[p] = b1[p] = U128{0, 0};
        for (int j = 0; j < dnum; j++) {
#pragma unroll
            for (int p = 0; p < KG_PP; p++) {
                const int kl = 2 * (threadIdx.x + p * KG_NT);
                const ulonglong2 x = *(const ulonglong2*)(st + (3 * j) * KT + kl);
                const ulonglong2 k0 = *(const ulonglong2*)(st + (3 * j + 1) * KT + kl);
                const ulonglong2 k1 = *(const ulonglong2*)(st + (3 * j + 2) * KT + kl);
                mac128(a0[p], x.x, k0.x);
                mac128(b0[p], x.y, k0.y);
                mac128(a1[p], x.x, k1.x);
                mac128(b1[p], x.y, k1.y);
            }
        }
        const bool lift = qlimb && B.c0[r];
        const uint32_t gr = B.g[r];
        const int sb0 = lift ? src_of_g(kb, gr) & ~(KT - 1) : 0;
#pragma unroll
        for (int p = 0; p < KG_PP; p++) {
            u64 o0 = redc128(a0[p], q, mc.qinv), o1 = redc128(b0[p], q, mc.qinv);
            if (lift) {
                const int src = src_of_g(kb + 2 * (threadIdx.x + p * KG_NT), gr);
                ulonglong2 y = *(const ulonglong2*)(st + (3 * dnum) * KT + (src & ~1) - sb0);
                if (src & 1) { const u64 t = y.x; y.x = y.y; y.y = t; }
                o0 = add_mod(o0, mul_shoup(y.x, f, fs, q), q);
                o1 = add_mod(o1, mul_shoup(y.y, f, fs, q), q);
            }
            s0[p][0] = add_mod(s0[p][0], o0, q);
            s0[p][1] = add_mod(s0[p][1], o1, q);
            s1[p][0] = add_mod(s1[p][0], redc128(a1[p], q, mc.qinv), q);
            s1[p][1] = add_mod(s1[p][1], redc128(b1[p], q, mc.qinv), q);
        }
        __syncthreads();                                  // stage consumed by every thread
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(r + 2);
        }
    }
    const u64* x0 = qlimb ? B.x0[z] : nullptr;
    u64* out = B.out[z];
#pragma unroll
    for (int p = 0; p < KG_PP; p++) {
        const int k = kb + 2 * (threadIdx.x + p * KG_NT);
        if (x0) {   // + P x0 (both components; x0 is [2][L][N])
            const ulonglong2 u = __ldg((const ulonglong2*)(x0 + (size_t)e * N + k));
            const ulonglong2 v = __ldg((const ulonglong2*)(x0 + ((size_t)L + e) * N + k));
            s0[p][0] = add_mod(s0[p][0], mul_shoup(u.x, f, fs, q), q);
            s0[p][1] = add_mod(s0[p][1], mul_shoup(u.y, f, fs, q), q);
            s1[p][0] = add_mod(s1[p][0], mul_shoup(v.x, f, fs, q), q);
            s1[p][1] = add_mod(s1[p][1], mul_shoup(v.y, f, fs, q), q);
        }
        *(ulonglong2*)(out + (size_t)e * N + k) = make_ulonglong2(s0[p][0], s0[p][1]);
        *(ulonglong2*)(out + ((size_t)nl + e) * N + k) = make_ulonglong2(s1[p][0], s1[p][1]);
    }
}

// Hoisted rotation SUM (DESIGN.md R-ROUTE) without ModDown, for request r = blockIdx.x (fastest, so the CTAs
// running together share each key tile through L2), coefficient pair tile blockIdx.y, extended limb e = blockIdx.z:
//   acc_0 = sum_i sum_j sigma_{g_i}(ext_j) key_i[j][0] + P (c0 + sum_i sigma_{g_i}(c0))   (P term on q-limbs only)
//   acc_1 = sum_i sum_j sigma_{g_i}(ext_j) key_i[j][1] + P c1
// i.e. P x + sum_i rot_ext(x, g_i) over Q_L u P (oracle kernels.route, hoisted).  Keys are in Montgomery form;
// products are accumulated in 128 bits and REDC'ed every <= 8 products (8 q < 2^64).
__global__ void __launch_bounds__(TB) ks_rotsum_kernel(RotSumBatch B, int nterms, int dnum, int nl, int L, int key_nl,
                                                       KeyLimb klm, LimbMap em, int N, int logN,
                                                       const ModConst* __restrict__ mod, const u64* __restrict__ pl,
                                                       const u64* __restrict__ pl_sh) {
    const int r = blockIdx.x, e = blockIdx.z;
    const int kp = blockIdx.y * blockDim.x + threadIdx.x;
    if (2 * kp >= N) return;
    const int k = 2 * kp;
    const ModConst mc = mod[em.mod[e]];
    const u64 q = mc.q;
    const int kle = klm.kl[e];
    const u64* __restrict__ ext = B.ext[r];
    const u64* __restrict__ c0 = B.c0[r];
    const bool qlimb = e < L;
    const uint32_t mask2n = 2 * N - 1;
    u64 s00 = 0, s01 = 0, s10 = 0, s11 = 0;
    U128 a0{0, 0}, b0{0, 0}, a1{0, 0}, b1{0, 0};
    int cnt = 0;
    u64 cs0 = 0, cs1 = 0;
    if (qlimb) {
        const ulonglong2 v = __ldg((const ulonglong2*)(c0 + (size_t)e * N + k));
        cs0 = v.x; cs1 = v.y;
    }
    for (int i = 0; i < nterms; i++) {
        const uint32_t g = B.g[i];
        const uint32_t ee = 2u * (uint32_t)brv(k, logN) + 1u;
        const uint32_t e2 = (uint32_t)(((uint64_t)ee * g) & mask2n);
        const int src = brv((int)((e2 - 1) >> 1), logN);
        const int base = src & ~1, swap = src & 1;
        const u64* key = B.key[i];
        for (int j = 0; j < dnum; j++) {
            if (cnt + 1 > 8) {
                s00 = add_mod(s00, redc128(a0, q, mc.qinv), q); s01 = add_mod(s01, redc128(b0, q, mc.qinv), q);
                s10 = add_mod(s10, redc128(a1, q, mc.qinv), q); s11 = add_mod(s11, redc128(b1, q, mc.qinv), q);
                a0 = b0 = a1 = b1 = U128{0, 0};
                cnt = 0;
            }
            ulonglong2 x = __ldg((const ulonglong2*)(ext + ((size_t)j * nl + e) * N + base));
            if (swap) { u64 t = x.x; x.x = x.y; x.y = t; }
            const u64* kj = key + (size_t)j * 2 * key_nl * N;
            const ulonglong2 k0 = __ldg((const ulonglong2*)(kj + (size_t)kle * N + k));
            const ulonglong2 k1 = __ldg((const ulonglong2*)(kj + ((size_t)key_nl + kle) * N + k));
            mac128(a0, x.x, k0.x);
            mac128(b0, x.y, k0.y);
            mac128(a1, x.x, k1.x);
            mac128(b1, x.y, k1.y);
            cnt++;
        }
        if (qlimb) {
            ulonglong2 y = __ldg((const ulonglong2*)(c0 + (size_t)e * N + base));
            if (swap) { u64 t = y.x; y.x = y.y; y.y = t; }
            cs0 = add_mod(cs0, y.x, q);
            cs1 = add_mod(cs1, y.y, q);
        }
    }
    s00 = add_mod(s00, redc128(a0, q, mc.qinv), q); s01 = add_mod(s01, redc128(b0, q, mc.qinv), q);
    s10 = add_mod(s10, redc128(a1, q, mc.qinv), q); s11 = add_mod(s11, redc128(b1, q, mc.qinv), q);
    if (qlimb) {
        const u64 p = pl[e], psh = pl_sh[e];
        const ulonglong2 v1 = __ldg((const ulonglong2*)(B.c1[r] + (size_t)e * N + k));
        s00 = add_mod(s00, mul_shoup(cs0, p, psh, q), q);
        s01 = add_mod(s01, mul_shoup(cs1, p, psh, q), q);
        s10 = add_mod(s10, mul_shoup(v1.x, p, psh, q), q);
        s11 = add_mod(s11, mul_shoup(v1.y, p, psh, q), q);
    }
    u64* acc = B.acc[r];
    *(ulonglong2*)(acc + (size_t)e * N + k) = make_ulonglong2(s00, s01);
    *(ulonglong2*)(acc + ((size_t)nl + e) * N + k) = make_ulonglong2(s10, s11);
}

// ks_rotsum_kernel with its operands streamed by the TMA engine (ENCF_ROTSUM_TMA=1, off: measured slower): a CTA owns an aligned tile of RKT
// coefficients of one (request, extended limb); stage (term i, digit j) = the Galois source block of ext (and, for j = 0
// on q-limbs, of c0) plus the two key tiles, RS_NST stages in flight on an mbarrier ring.  Same arithmetic and words.
constexpr int RKT = 512, RS_NT = 128, RS_NST = 4;
__global__ void __launch_bounds__(RS_NT) ks_rotsum_tma_kernel(RotSumBatch B, int nterms, int dnum, int nl, int L, int key_nl,
                                                              KeyLimb klm, LimbMap em, int N, int logN,
                                                              const ModConst* __restrict__ mod, const u64* __restrict__ pl,
                                                              const u64* __restrict__ pl_sh) {
    extern __shared__ __align__(128) u64 rs_sm[];         // [RS_NST][4][RKT] | [RS_NST] mbarriers
    uint64_t* bars = (uint64_t*)(rs_sm + (size_t)RS_NST * 4 * RKT);
    const int r = blockIdx.x, e = blockIdx.z;
    const int kb = blockIdx.y * RKT;
    const bool qlimb = e < L;
    const ModConst mc = mod[em.mod[e]];
    const u64 q = mc.q;
    const int kle = klm.kl[e];
    const u64* __restrict__ ext = B.ext[r];
    const u64* __restrict__ c0 = B.c0[r];
    const uint32_t mask2n = 2 * N - 1;
    auto src_of = [&](int k, uint32_t g) -> int {
        const uint32_t ee = 2u * (uint32_t)brv(k, logN) + 1u;
        const uint32_t e2 = (uint32_t)(((uint64_t)ee * g) & mask2n);
        return brv((int)((e2 - 1) >> 1), logN);
    };
    const int total = nterms * dnum;
    auto issue = [&](int st) {
        if (threadIdx.x != 0) return;
        const int i = st / dnum, j = st % dnum, slot = st % RS_NST;
        const int sb = src_of(kb, B.g[i]) & ~(RKT - 1);
        u64* d = rs_sm + (size_t)slot * 4 * RKT;
        const bool with_c0 = qlimb && j == 0;
        mbar_arrive_expect_tx(&bars[slot], (uint32_t)(with_c0 ? 4 : 3) * RKT * 8);
        const u64* kj = B.key[i] + (size_t)j * 2 * key_nl * N;
        bulk_g2s(d, ext + ((size_t)j * nl + e) * N + sb, RKT * 8, &bars[slot]);
        bulk_g2s(d + RKT, kj + (size_t)kle * N + kb, RKT * 8, &bars[slot]);
        bulk_g2s(d + 2 * RKT, kj + ((size_t)key_nl + kle) * N + kb, RKT * 8, &bars[slot]);
        if (with_c0) bulk_g2s(d + 3 * RKT, c0 + (size_t)e * N + sb, RKT * 8, &bars[slot]);
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < RS_NST; i++) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int st = 0; st < RS_NST - 1 && st < total; st++) issue(st);
    }
    __syncthreads();
    constexpr int PP = RKT / 2 / RS_NT;
    int kl[PP];
    u64 s00[PP], s01[PP], s10[PP], s11[PP], cs0[PP], cs1[PP];
    U128 a0[PP], b0[PP], a1[PP], b1[PP];
#pragma unroll
    for (int p = 0; p < PP; p++) {
        kl[p] = 2 * (threadIdx.x + p * RS_NT);
        s00[p] = s01[p] = s10[p] = s11[p] = 0;
        a0[p] = b0[p] = a1[p] = b1[p] = U128{0, 0};
        cs0[p] = cs1[p] = 0;
        if (qlimb) {
            const ulonglong2 v = __ldg((const ulonglong2*)(c0 + (size_t)e * N + kb + kl[p]));
            cs0[p] = v.x; cs1[p] = v.y;
        }
    }
    int cnt = 0;
    for (int st = 0; st < total; st++) {
        if (st + RS_NST - 1 < total) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(st + RS_NST - 1);
        }
        const int i = st / dnum, j = st % dnum, slot = st % RS_NST;
        const uint32_t g = B.g[i];
        const int sb = src_of(kb, g) & ~(RKT - 1);
        mbar_wait(&bars[slot], (uint32_t)((st / RS_NST) & 1));
        const u64* d = rs_sm + (size_t)slot * 4 * RKT;
        if (cnt + 1 > 8) {      // REDC every <= 8 products (8 q < 2^64)
#pragma unroll
            for (int p = 0; p < PP; p++) {
                s00[p] = add_mod(s00[p], redc128(a0[p], q, mc.qinv), q); s01[p] = add_mod(s01[p], redc128(b0[p], q, mc.qinv), q);
                s10[p] = add_mod(s10[p], redc128(a1[p], q, mc.qinv), q); s11[p] = add_mod(s11[p], redc128(b1[p], q, mc.qinv), q);
                a0[p] = b0[p] = a1[p] = b1[p] = U128{0, 0};
            }
            cnt = 0;
        }
#pragma unroll
        for (int p = 0; p < PP; p++) {
            const int src = src_of(kb + kl[p], g);
            const int sl = (src & ~1) - sb, sw = src & 1;
            ulonglong2 x = *(const ulonglong2*)(d + sl);
            if (sw) { u64 t = x.x; x.x = x.y; x.y = t; }
            const ulonglong2 k0 = *(const ulonglong2*)(d + RKT + kl[p]);
            const ulonglong2 k1 = *(const ulonglong2*)(d + 2 * RKT + kl[p]);
            mac128(a0[p], x.x, k0.x);
            mac128(b0[p], x.y, k0.y);
            mac128(a1[p], x.x, k1.x);
            mac128(b1[p], x.y, k1.y);
            if (qlimb && j == 0) {
                ulonglong2 y = *(const ulonglong2*)(d + 3 * RKT + sl);
                if (sw) { u64 t = y.x; y.x = y.y; y.y = t; }
                cs0[p] = add_mod(cs0[p], y.x, q);
                cs1[p] = add_mod(cs1[p], y.y, q);
            }
        }
        cnt++;
        __syncthreads();            // every thread is done with this slot: it may be refilled
    }
    u64* accp = B.acc[r];
#pragma unroll
    for (int p = 0; p < PP; p++) {
        u64 v00 = add_mod(s00[p], redc128(a0[p], q, mc.qinv), q), v01 = add_mod(s01[p], redc128(b0[p], q, mc.qinv), q);
        u64 v10 = add_mod(s10[p], redc128(a1[p], q, mc.qinv), q), v11 = add_mod(s11[p], redc128(b1[p], q, mc.qinv), q);
        const int k = kb + kl[p];
        if (qlimb) {
            const u64 pe = pl[e], pes = pl_sh[e];
            const ulonglong2 v1 = __ldg((const ulonglong2*)(B.c1[r] + (size_t)e * N + k));
            v00 = add_mod(v00, mul_shoup(cs0[p], pe, pes, q), q);
            v01 = add_mod(v01, mul_shoup(cs1[p], pe, pes, q), q);
            v10 = add_mod(v10, mul_shoup(v1.x, pe, pes, q), q);
            v11 = add_mod(v11, mul_shoup(v1.y, pe, pes, q), q);
        }
        *(ulonglong2*)(accp + (size_t)e * N + k) = make_ulonglong2(v00, v01);
        *(ulonglong2*)(accp + ((size_t)nl + e) * N + k) = make_ulonglong2(v10, v11);
    }
}

// Masked shift Psi^t in the extended basis (DESIGN.md R-LAZY), fused: for request r = blockIdx.x, pair tile
// blockIdx.y, extended limb e = blockIdx.z,
//   out_c = sum_{i<2} mask_i (.) ( sum_j sigma_{g_i}(ext_j) key_i[j][c] + [c == 0] P sigma_{g_i}(c0) )
// = h_t (.) rot_ext(x, t) + u_t (.) rot_ext(x, t - m) without materialising the two rotations.  The masks are
// folded into PRE-MASKED keys (B.key[r][i] = key_i (.) mask_i, Montgomery form, cached per (keys, g, mask)) and
// B.mask[r][i] = (P R) (.) mask_i, so both terms, all digits and the c0 lift accumulate in ONE 128-bit sum per
// output (<= 2 dnum + 2 <= 8 products, 8 q < 2^64) reduced by ONE Montgomery REDC.
__global__ void __launch_bounds__(TB) ks_psi_kernel(PsiBatch B, int dnum, int nl, int L, LimbMap em, int N, int logN,
                                                    const ModConst* __restrict__ mod) {
    const int r = blockIdx.x, e = blockIdx.z;
    const int kp = blockIdx.y * blockDim.x + threadIdx.x;
    if (2 * kp >= N) return;
    const int k = 2 * kp;
    const ModConst mc = mod[em.mod[e]];
    const u64 q = mc.q;
    const u64* __restrict__ ext = B.ext[r];
    const bool qlimb = e < L;
    const uint32_t mask2n = 2 * N - 1;
    U128 A0{0, 0}, B0{0, 0}, A1{0, 0}, B1{0, 0};
    const uint32_t ee = 2u * (uint32_t)brv(k, logN) + 1u;
#pragma unroll
    for (int i = 0; i < 2; i++) {
        const uint32_t g = B.g[r][i];
        const uint32_t e2 = (uint32_t)(((uint64_t)ee * g) & mask2n);
        const int src = brv((int)((e2 - 1) >> 1), logN);
        const int base = src & ~1, swap = src & 1;
        const u64* km = B.key[r][i];
        for (int j = 0; j < dnum; j++) {
            ulonglong2 x = __ldg((const ulonglong2*)(ext + ((size_t)j * nl + e) * N + base));
            if (swap) { u64 t = x.x; x.x = x.y; x.y = t; }
            const u64* kj = km + (size_t)j * 2 * nl * N;
            const ulonglong2 k0 = __ldg((const ulonglong2*)(kj + (size_t)e * N + k));
            const ulonglong2 k1 = __ldg((const ulonglong2*)(kj + ((size_t)nl + e) * N + k));
            mac128(A0, x.x, k0.x);
            mac128(B0, x.y, k0.y);
            mac128(A1, x.x, k1.x);
            mac128(B1, x.y, k1.y);
        }
        if (qlimb) {
            ulonglong2 y = __ldg((const ulonglong2*)(B.c0[r] + (size_t)e * N + base));
            if (swap) { u64 t = y.x; y.x = y.y; y.y = t; }
            const ulonglong2 pm = __ldg((const ulonglong2*)(B.mask[r][i] + (size_t)e * N + k));
            mac128(A0, y.x, pm.x);
            mac128(B0, y.y, pm.y);
        }
    }
    u64* out = B.out[r];
    *(ulonglong2*)(out + (size_t)e * N + k) = make_ulonglong2(redc128(A0, q, mc.qinv), redc128(B0, q, mc.qinv));
    *(ulonglong2*)(out + ((size_t)nl + e) * N + k) = make_ulonglong2(redc128(A1, q, mc.qinv), redc128(B1, q, mc.qinv));
}

// ks_psi_kernel with its operands staged by the TMA engine (ENCF_KS_TMA, as ks_inner_tma_kernel): a CTA owns an aligned
// tile of KT coefficients of one (request, extended limb); for each of the two terms i the Galois source block of ext
// (every digit) and c0, the pre-masked key tiles and the P-mask tile arrive by cp.async.bulk on one mbarrier per term.
// Same arithmetic and output words.
template <int KTP, int NT>
__global__ void __launch_bounds__(NT) ks_psi_tma_kernel(PsiBatch B, int dnum, int nl, int L, LimbMap em, int N, int logN,
                                                       const ModConst* __restrict__ mod) {
    constexpr int KT = KTP;
    extern __shared__ __align__(128) u64 kp_sm[];
    const int r = blockIdx.x, e = blockIdx.z;
    const int kb = blockIdx.y * KT;
    const bool qlimb = e < L;
    const int per = 3 * dnum + (qlimb ? 2 : 0);          // KT-word blocks per term: dnum x (ext, key0, key1) [+ c0, pm]
    uint64_t* bars = (uint64_t*)(kp_sm + (size_t)2 * (3 * dnum + 2) * KT);
    const uint32_t mask2n = 2 * N - 1;
    auto src_of = [&](int k, uint32_t g) -> int {
        const uint32_t ee = 2u * (uint32_t)brv(k, logN) + 1u;
        const uint32_t e2 = (uint32_t)(((uint64_t)ee * g) & mask2n);
        return brv((int)((e2 - 1) >> 1), logN);
    };
    const u64* __restrict__ ext = B.ext[r];
    int sb[2];
#pragma unroll
    for (int i = 0; i < 2; i++) sb[i] = src_of(kb, B.g[r][i]) & ~(KT - 1);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; i++) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 2; i++) {
            u64* st = kp_sm + (size_t)i * (3 * dnum + 2) * KT;
            mbar_arrive_expect_tx(&bars[i], (uint32_t)per * KT * 8);
            const u64* km = B.key[r][i];
            for (int j = 0; j < dnum; j++) {
                const u64* kj = km + (size_t)j * 2 * nl * N;
                bulk_g2s(st + (3 * j) * KT, ext + ((size_t)j * nl + e) * N + sb[i], KT * 8, &bars[i]);
                bulk_g2s(st + (3 * j + 1) * KT, kj + (size_t)e * N + kb, KT * 8, &bars[i]);
                bulk_g2s(st + (3 * j + 2) * KT, kj + ((size_t)nl + e) * N + kb, KT * 8, &bars[i]);
            }
            if (qlimb) {
                bulk_g2s(st + (3 * dnum) * KT, B.c0[r] + (size_t)e * N + sb[i], KT * 8, &bars[i]);
                bulk_g2s(st + (3 * dnum + 1) * KT, B.mask[r][i] + (size_t)e * N + kb, KT * 8, &bars[i]);
            }
        }
    }
    __syncthreads();
    const ModConst mc = mod[em.mod[e]];
    const u64 q = mc.q;
    constexpr int PP = KT / 2 / NT;
    U128 A0[PP], B0[PP], A1[PP], B1[PP];
#pragma unroll
    for (int p = 0; p < PP; p++) A0[p] = B0[p] = A1[p] = B1[p] = U128{0, 0};
#pragma unroll
    for (int i = 0; i < 2; i++) {
        const uint32_t g = B.g[r][i];
        int kl[PP], sl[PP], sw[PP];
#pragma unroll
        for (int p = 0; p < PP; p++) {
            kl[p] = 2 * (threadIdx.x + p * NT);
            const int src = src_of(kb + kl[p], g);
            sl[p] = (src & ~1) - sb[i];
            sw[p] = src & 1;
        }
        mbar_wait(&bars[i], 0);
        const u64* st = kp_sm + (size_t)i * (3 * dnum + 2) * KT;
        for (int j = 0; j < dnum; j++) {
#pragma unroll
            for (int p = 0; p < PP; p++) {
                ulonglong2 x = *(const ulonglong2*)(st + (3 * j) * KT + sl[p]);
                if (sw[p]) { u64 t = x.x; x.x = x.y; x.y = t; }
                const ulonglong2 k0 = *(const ulonglong2*)(st + (3 * j + 1) * KT + kl[p]);
                const ulonglong2 k1 = *(const ulonglong2*)(st + (3 * j + 2) * KT + kl[p]);
                mac128(A0[p], x.x, k0.x);
                mac128(B0[p], x.y, k0.y);
                mac128(A1[p], x.x, k1.x);
                mac128(B1[p], x.y, k1.y);
            }
        }
        if (qlimb) {
#pragma unroll
            for (int p = 0; p < PP; p++) {
                ulonglong2 y = *(const ulonglong2*)(st + (3 * dnum) * KT + sl[p]);
                if (sw[p]) { u64 t = y.x; y.x = y.y; y.y = t; }
                const ulonglong2 pm = *(const ulonglong2*)(st + (3 * dnum + 1) * KT + kl[p]);
                mac128(A0[p], y.x, pm.x);
                mac128(B0[p], y.y, pm.y);
            }
        }
    }
    u64* out = B.out[r];
#pragma unroll
    for (int p = 0; p < PP; p++) {
        const int k = kb + 2 * (threadIdx.x + p * NT);
        *(ulonglong2*)(out + (size_t)e * N + k) = make_ulonglong2(redc128(A0[p], q, mc.qinv), redc128(B0[p], q, mc.qinv));
        *(ulonglong2*)(out + ((size_t)nl + e) * N + k) = make_ulonglong2(redc128(A1[p], q, mc.qinv), redc128(B1[p], q, mc.qinv));
    }
}

// km[j][c][e][k] = key[j][c][kl(e)][k] (.) mask[e][k] mod q_e (the key's Montgomery factor is kept);
// pm[e][k] = PR_e (.) mask[e][k] mod q_e for e < L (PR_e = P R mod q_e).
__global__ void keymask_kernel(const u64* __restrict__ key, int key_nl, const u64* __restrict__ mask, int dnum, int L, int nl,
                               KeyLimb klm, LimbMap em, const u64* __restrict__ pr, u64* __restrict__ out, int N,
                               const ModConst* __restrict__ mod) {
    const size_t total = (size_t)(dnum * 2 + 1) * nl * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % N);
        const size_t row = i / N;
        const int e = (int)(row % nl), jc = (int)(row / nl);
        const ModConst mc = mod[em.mod[e]];
        const u64 m = mask[(size_t)e * N + k];
        if (jc < dnum * 2) {
            const int j = jc >> 1, c = jc & 1;
            const u64 kv = key[((size_t)j * 2 + c) * key_nl * N + (size_t)klm.kl[e] * N + k];
            out[i] = mulmod_barrett(kv, m, mc.q, mc.rhi, mc.rlo);
        } else if (e < L) {
            out[i] = mulmod_barrett(pr[e], m, mc.q, mc.rhi, mc.rlo);
        }
    }
}

// Rotation-mask-accumulate (Halevi-Shoup repack of the w/o-SCP ablation, oracle kernels.repack_rma) without
// ModDown: acc_c = sum_i mask_i (.) ( sum_j sigma_{g_i}(ext_j) key_i[j][c] + [c == 0] P sigma_{g_i}(c0) ).
__global__ void __launch_bounds__(TB) ks_rma_kernel(RotSumBatch B, int nterms, int dnum, int nl, int L, int key_nl,
                                                    KeyLimb klm, LimbMap em, int N, int logN,
                                                    const ModConst* __restrict__ mod, const u64* __restrict__ pl,
                                                    const u64* __restrict__ pl_sh) {
    const int r = blockIdx.x, e = blockIdx.z;
    const int kp = blockIdx.y * blockDim.x + threadIdx.x;
    if (2 * kp >= N) return;
    const int k = 2 * kp;
    const ModConst mc = mod[em.mod[e]];
    const u64 q = mc.q;
    const int kle = klm.kl[e];
    const u64* __restrict__ ext = B.ext[r];
    const bool qlimb = e < L;
    const uint32_t mask2n = 2 * N - 1;
    const uint32_t ee = 2u * (uint32_t)brv(k, logN) + 1u;
    u64 s00 = 0, s01 = 0, s10 = 0, s11 = 0;
    for (int i = 0; i < nterms; i++) {
        const uint32_t e2 = (uint32_t)(((uint64_t)ee * B.g[i]) & mask2n);
        const int src = brv((int)((e2 - 1) >> 1), logN);
        const int base = src & ~1, swap = src & 1;
        const u64* key = B.key[i];
        U128 a0{0, 0}, b0{0, 0}, a1{0, 0}, b1{0, 0};
        for (int j = 0; j < dnum; j++) {
            ulonglong2 x = __ldg((const ulonglong2*)(ext + ((size_t)j * nl + e) * N + base));
            if (swap) { u64 t = x.x; x.x = x.y; x.y = t; }
            const u64* kj = key + (size_t)j * 2 * key_nl * N;
            const ulonglong2 k0 = __ldg((const ulonglong2*)(kj + (size_t)kle * N + k));
            const ulonglong2 k1 = __ldg((const ulonglong2*)(kj + ((size_t)key_nl + kle) * N + k));
            mac128(a0, x.x, k0.x);
            mac128(b0, x.y, k0.y);
            mac128(a1, x.x, k1.x);
            mac128(b1, x.y, k1.y);
        }
        u64 t00 = redc128(a0, q, mc.qinv), t01 = redc128(b0, q, mc.qinv);
        const u64 t10 = redc128(a1, q, mc.qinv), t11 = redc128(b1, q, mc.qinv);
        if (qlimb) {
            ulonglong2 y = __ldg((const ulonglong2*)(B.c0[r] + (size_t)e * N + base));
            if (swap) { u64 t = y.x; y.x = y.y; y.y = t; }
            t00 = add_mod(t00, mul_shoup(y.x, pl[e], pl_sh[e], q), q);
            t01 = add_mod(t01, mul_shoup(y.y, pl[e], pl_sh[e], q), q);
        }
        const ulonglong2 m = __ldg((const ulonglong2*)(B.mask[i] + (size_t)e * N + k));
        s00 = add_mod(s00, mulmod_barrett(t00, m.x, q, mc.rhi, mc.rlo), q);
        s01 = add_mod(s01, mulmod_barrett(t01, m.y, q, mc.rhi, mc.rlo), q);
        s10 = add_mod(s10, mulmod_barrett(t10, m.x, q, mc.rhi, mc.rlo), q);
        s11 = add_mod(s11, mulmod_barrett(t11, m.y, q, mc.rhi, mc.rlo), q);
    }
    u64* acc = B.acc[r];
    *(ulonglong2*)(acc + (size_t)e * N + k) = make_ulonglong2(s00, s01);
    *(ulonglong2*)(acc + ((size_t)nl + e) * N + k) = make_ulonglong2(s10, s11);
}

// out_c = (b_c - y_c) P^{-1} + add_c for request r = blockIdx.z / 2, component c = blockIdx.z % 2.
// b: acc base [r][2][nl][N]; y: [r][2][L][N].
__global__ void moddown_finish_batch_kernel(const u64* __restrict__ acc, const u64* __restrict__ y, OutBatch O, int level,
                                            int nl, int N, const ModConst* __restrict__ mod, const u64* pinv,
                                            const u64* pinv_sh) {
    const int r = blockIdx.z >> 1, c = blockIdx.z & 1;
    const u64* b = acc + ((size_t)r * 2 + c) * nl * N;
    const u64* yy = y + ((size_t)r * 2 + c) * level * N;
    u64* out = O.out[r][c];
    const u64* add = O.add[r][c];
    const size_t total = (size_t)level * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)(i / N);
        u64 q = mod[limb].q;
        u64 v = mul_shoup(sub_mod(b[i], yy[i], q), pinv[limb], pinv_sh[limb], q);
        if (add) v = add_mod(v, add[i], q);
        out[i] = v;
    }
}

// bconv over a batch of polynomials: input poly p at in + p*in_stride, output at out + p*out_stride.
// corr != nullptr: rounded conversion (ModDown, DESIGN.md R-MODDOWN): r = (sum_i umulhi(v_i << s_i, cfix_i) + 2^58) >> 59
// with s_i = 63 - bitlen(q_i), cfix_i = floor(2^(123-s_i) / q_i) (= round(sum_i v_i / q_i), bit-identical to oracle.c
// o_bconv_round); the
// correction -r Q' is folded into the 128-bit accumulator (corr_t = t - Q' mod t).  Templated on the input
// count so no predicated-off multiply is issued.
template <int NIN>
__global__ void __launch_bounds__(TB, 4) bconv_batch_kernel(const u64* __restrict__ in, i64 in_stride, LimbMap im,
                                                            const u64* __restrict__ vfac, const u64* __restrict__ vfac_sh,
                                                            const u64* __restrict__ wfac, LimbMap om, OutPos op,
                                                            u64* __restrict__ out, i64 out_stride, int N,
                                                            const ModConst* __restrict__ mod, const u64* __restrict__ corr,
                                                            const u64* __restrict__ cfix, const u64* __restrict__ csh,
                                                            int pre) {
    // shared: [NIN][nout] wfac | [nout] corr | [nout] q_t | [nout] qinv_t | [NIN] q_i | vf | vfs | cfix | shift | [nout] pos
    // (uniform constants live in shared memory, not in registers: 4 CTAs/SM instead of 2)
    extern __shared__ u64 sw[];
    const int nout = om.n;
    u64* s_corr = sw + NIN * nout;
    u64* s_q = s_corr + nout;
    u64* s_qi = s_q + nout;
    u64* s_in = s_qi + nout;
    u64* s_pos = s_in + 5 * NIN;
    for (int i = threadIdx.x; i < NIN * nout; i += blockDim.x) sw[i] = wfac[i];
    for (int t = threadIdx.x; t < nout; t += blockDim.x) s_pos[t] = (u64)op.pos[t] * (u64)N;
    for (int t = threadIdx.x; t < nout; t += blockDim.x) {
        s_corr[t] = corr ? corr[t] : 0;
        s_q[t] = mod[om.mod[t]].q;
        s_qi[t] = mod[om.mod[t]].qinv;
    }
    for (int i = threadIdx.x; i < NIN; i += blockDim.x) {
        s_in[i] = mod[im.mod[i]].q;
        s_in[NIN + i] = vfac[i];
        s_in[2 * NIN + i] = vfac_sh[i];
        s_in[3 * NIN + i] = corr ? cfix[i] : 0;
        s_in[4 * NIN + i] = corr ? csh[i] : 0;
    }
    __syncthreads();
    in += (size_t)blockIdx.y * in_stride;
    out += (size_t)blockIdx.y * out_stride;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        u64 v[NIN];
#pragma unroll
        for (int i = 0; i < NIN; i++) v[i] = __ldg(in + (size_t)i * N + k);
#pragma unroll
        for (int i = 0; i < NIN; i++) v[i] = pre ? v[i] : mul_shoup(v[i], s_in[NIN + i], s_in[2 * NIN + i], s_in[i]);
        u64 r = 0;
        if (corr) {
            u64 fsum = 0;
#pragma unroll
            for (int i = 0; i < NIN; i++) fsum += umulhi(v[i] << (int)s_in[4 * NIN + i], s_in[3 * NIN + i]);
            r = (fsum + (1ull << 58)) >> 59;
        }
        // 30-bit split (all moduli < 2^60, checked on the host): v = vh 2^30 + vl, w = wh 2^30 + wl, four
        // 32x32->64 products accumulated carry-free in 64 bits (each < 2^60, <= 8 terms), combined once per output
        uint32_t vh[NIN], vl[NIN];
#pragma unroll
        for (int i = 0; i < NIN; i++) { vh[i] = (uint32_t)(v[i] >> 30); vl[i] = (uint32_t)(v[i] & 0x3FFFFFFFu); }
        for (int t = 0; t < nout; t++) {
            u64 hh = 0, hl = 0, lh = 0, ll = 0;
#pragma unroll
            for (int i = 0; i < NIN; i++) {
                const u64 w = sw[i * nout + t];
                const uint32_t wh = (uint32_t)(w >> 30), wlo = (uint32_t)(w & 0x3FFFFFFFu);
                hh += (u64)vh[i] * wh;
                hl += (u64)vh[i] * wlo;
                lh += (u64)vl[i] * wh;
                ll += (u64)vl[i] * wlo;
            }
            U128 acc{ll, 0};
            const u64 mid = hl + lh;                        // < 2^64
            add128(acc, mid << 30);
            acc.hi += mid >> 34;
            add128(acc, hh << 60);
            acc.hi += hh >> 4;
            if (corr) mac128(acc, r, s_corr[t]);
            out[s_pos[t] + k] = redc128(acc, s_q[t], s_qi[t]);   // wfac / corr in Montgomery form
        }
    }
}

// ------------------------------------------------------------------------------------ tensor-core base conversion
// The same conversion on the 5th-generation tensor cores (tcgen05.mma .kind::i8, u8 x u8 -> s32: exact integers).
// With v_i = [x_i vfac_i]_{q_i} split into bytes v_i = sum_a v_i[a] 2^{8a} and the constant matrix
// W'[i][a][t] = 2^{8a} wfac[i][t] mod q_t (wfac in Montgomery form) split into bytes W'[i][a][t][b] (ctx.cu
// bconv_wbytes), one M = 128 coefficients x N = 8 nout x K = 64 bytes MMA pair gives
//   D[k][(t, b)] = sum_{(i, a)} v_i[a](k) W'[i][a][t][b]       (< 64 * 255^2 < 2^22, no overflow)
//   T[t][k] = sum_b D[k][(t, b)] 2^{8b} (+ r corr_t) = (sum_i v_i wfac[i][t] + r corr_t) mod q_t  (T < 2^79 < q_t 2^64)
// and out = REDC(T): bit-identical to bconv_batch_kernel (the same REDC of a congruent 128-bit value < q_t 2^64).
// Operands: A = the tile's v bytes [128 rows][64 B] and B = W' bytes [nb rows][64 B], both K-major in the canonical
// no-swizzle layout ([16-byte K chunk][row][16 B]: SBO = 128 B between 8-row core matrices, LBO = rows x 16 B
// between the two K chunks of one K32 step); D lives in TMEM (lane = coefficient, column = 8 t + b) and is read back
// with tcgen05.ld 32x32b.x8 (one thread per coefficient row).  Inputs beyond NIN are zero rows of B.  Each CTA
// (128 threads) loops over 128-coefficient tiles with the next tile's inputs in flight during the current MMA and
// epilogue.  Microbench + decision: tools/micro/bconv_tc.cu, profiles/r02_summary.md.
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);   // version 1, no swizzle
}

constexpr int BTC_TILE = 128;
#ifndef BTC_LD4
#define BTC_LD4 1   // 0: one TMEM load (8 columns) + wait per output (A/B)
#endif
#ifndef BTC_COMB
#define BTC_COMB 1  // 0: byte planes combined with 64-bit multiply-adds (A/B)
#endif
template <int NIN, bool CORR>
__global__ void __launch_bounds__(BTC_TILE) bconv_tc_kernel(const u64* __restrict__ in, i64 in_stride, LimbMap im,
                                                           const u64* __restrict__ vfac, const u64* __restrict__ vfac_sh,
                                                           const uint8_t* __restrict__ wb, int nb, int tcols, LimbMap om,
                                                           OutPos op, u64* __restrict__ out, i64 out_stride, int N,
                                                           int npolys, const ModConst* __restrict__ mod,
                                                           const u64* __restrict__ corr, const u64* __restrict__ cfix,
                                                           const u64* __restrict__ csh, int pre) {
    extern __shared__ __align__(1024) uint8_t btc_sm[];
    uint8_t* sA = btc_sm;                                   // [4][128][16]
    uint8_t* sB = btc_sm + BTC_TILE * 64;                   // [4][nb][16]
    u64* sq = (u64*)(sB + (size_t)nb * 64);                 // [nout] q_t | qinv_t | corr_t | pos_t * N
    u64* sqi = sq + 32;
    u64* scr = sqi + 32;
    u64* spos = scr + 32;
    uint64_t* mbar = (uint64_t*)(spos + 32);
    uint32_t* tmem_slot = (uint32_t*)(mbar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int nout = om.n;
    for (int i = tid; i < nb * 4; i += BTC_TILE) ((uint4*)sB)[i] = __ldg((const uint4*)wb + i);
    for (int t = tid; t < nout; t += BTC_TILE) {
        sq[t] = mod[om.mod[t]].q;
        sqi[t] = mod[om.mod[t]].qinv;
        scr[t] = CORR ? corr[t] : 0;
        spos[t] = (u64)op.pos[t] * (u64)N;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *tmem_slot;
    u64 qin[NIN], vf[NIN], vfs[NIN], cf[NIN];
    int cs[NIN];
#pragma unroll
    for (int i = 0; i < NIN; i++) {
        qin[i] = mod[im.mod[i]].q;
        vf[i] = vfac[i];
        vfs[i] = vfac_sh[i];
        cf[i] = CORR ? cfix[i] : 0;
        cs[i] = CORR ? (int)csh[i] : 0;
    }
    // instruction descriptor: D s32 (bits 4-5 = 2), A/B u8 (0), K-major, N = nb, M = 128
    const uint32_t idesc = (2u << 4) | ((uint32_t)(nb >> 3) << 17) | ((uint32_t)(BTC_TILE >> 4) << 24);
    const int tpp = N / BTC_TILE, ntiles = tpp * npolys;
    u64 nx[NIN];
    auto load_tile = [&](int tile) {
        if (tile >= ntiles) return;
        const u64* ip = in + (size_t)(tile / tpp) * in_stride + (size_t)(tile % tpp) * BTC_TILE + tid;
#pragma unroll
        for (int i = 0; i < NIN; i++) nx[i] = __ldg(ip + (size_t)i * N);
    };
    load_tile(blockIdx.x);
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int p = tile / tpp, k0 = (tile % tpp) * BTC_TILE;
        u64 r = 0;
        {
            u64 fsum = 0;
#pragma unroll
            for (int i = 0; i < NIN; i++) {
                const u64 v = pre ? nx[i] : mul_shoup(nx[i], vf[i], vfs[i], qin[i]);
                if (CORR) fsum += umulhi(v << cs[i], cf[i]);
                *(u64*)(sA + (i >> 1) * (BTC_TILE * 16) + tid * 16 + (i & 1) * 8) = v;
            }
            if (CORR) r = (fsum + (1ull << 58)) >> 59;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy smem writes -> tensor core
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (tid == 0) {
#pragma unroll
            for (int st = 0; st < 2; st++) {   // K = 64 bytes: two K32 steps of two 16-byte chunks
                const uint64_t da = umma_sdesc(smem_u32(sA) + st * 2 * BTC_TILE * 16, BTC_TILE * 16, 128);
                const uint64_t db = umma_sdesc(smem_u32(sB) + st * 2 * nb * 16, nb * 16, 128);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                    ::"r"(tbase), "l"(da), "l"(db), "r"(idesc), "r"((uint32_t)st) : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
                         : "memory");
        }
        load_tile(tile + gridDim.x);   // next tile's inputs in flight during the MMA and the epilogue
        mbar_wait(mbar, phase);
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        u64* o = out + (size_t)p * out_stride + k0 + tid;
        const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
        auto finish = [&](int t, const uint32_t* d) {
#if BTC_COMB
            // T = sum_b d_b 2^{8b} (d_b < 2^22, T < 2^79) in 32-bit words with shift-adds and carries (ALU pipe), not
            // 64-bit multiply-adds by 2^{8b} (the compiler's IMAD.WIDE on the fmaheavy pipe that bounds this kernel)
            uint32_t w0, w1, w2;
            // byte shifts as PRMT (the shift-adds would be re-fused into IMAD by ptxas)
            asm("{\n\t.reg .u32 A, B, C, D, t, lh, hl, hh;\n\t"
                "prmt.b32 t, %4, 0, 0x2104;\n\tadd.u32 A, %3, t;\n\t"
                "prmt.b32 t, %6, 0, 0x2104;\n\tadd.u32 B, %5, t;\n\t"
                "prmt.b32 t, %8, 0, 0x2104;\n\tadd.u32 C, %7, t;\n\t"
                "prmt.b32 t, %10, 0, 0x2104;\n\tadd.u32 D, %9, t;\n\t"
                "prmt.b32 t, B, 0, 0x1044;\n\tadd.cc.u32 %0, A, t;\n\tprmt.b32 t, B, 0, 0x4432;\n\taddc.u32 lh, t, 0;\n\t"
                "prmt.b32 t, D, 0, 0x1044;\n\tadd.cc.u32 hl, C, t;\n\tprmt.b32 t, D, 0, 0x4432;\n\taddc.u32 hh, t, 0;\n\t"
                "add.cc.u32 %1, lh, hl;\n\taddc.u32 %2, hh, 0;\n\t}"
                : "=r"(w0), "=r"(w1), "=r"(w2)
                : "r"(d[0]), "r"(d[1]), "r"(d[2]), "r"(d[3]), "r"(d[4]), "r"(d[5]), "r"(d[6]), "r"(d[7]));
            U128 T{((u64)w1 << 32) | w0, (u64)w2};
            if (CORR) add128(T, r * scr[t]);   // r <= NIN <= 8 roundings, scr < 2^61: the product fits 64 bits
#else
            const u64 lo4 = (u64)d[0] + ((u64)d[1] << 8) + ((u64)d[2] << 16) + ((u64)d[3] << 24);
            const u64 hi4 = (u64)d[4] + ((u64)d[5] << 8) + ((u64)d[6] << 16) + ((u64)d[7] << 24);
            U128 T{lo4, 0};
            add128(T, hi4 << 32);
            T.hi += hi4 >> 32;
            if (CORR) mac128(T, r, scr[t]);
#endif
            o[spos[t]] = redc128(T, sq[t], sqi[t]);
        };
        int t = 0;
#if BTC_LD4
        // four outputs' 8 partial sums per TMEM load (32 columns) and one wait: the loads' latency is paid once per
        // four outputs instead of once per output (bconv 5.18 -> 5.09 ms per layer)
        for (; t + 4 <= nout; t += 4) {
            uint32_t d[32];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                         "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                         : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                           "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]),
                           "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]),
                           "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
                         : "r"(tl + t * 8));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 4; k++) finish(t + k, d + 8 * k);
        }
#endif
        for (; t < nout; t++) {
            uint32_t d[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
                         : "r"(tl + t * 8));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            finish(t, d);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();               // TMEM and sA are free for the next tile
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(tcols));
}

// Gather-copy: dst + p*dst_stride <- src[p] (words each), optional Galois gather per item (NTT domain).
__global__ void gather_copy_kernel(CopyBatch C, u64* dst, i64 dst_stride, size_t words, int N, int logN) {
    const int p = blockIdx.y;
    const u64* __restrict__ src = C.src[p];
    const uint32_t g = C.g[p];
    u64* d = dst + (size_t)p * dst_stride;
    const uint32_t mask2n = 2 * N - 1;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words; i += (size_t)gridDim.x * blockDim.x) {
        size_t limb = i / N;
        int k = (int)(i % N);
        int s = k;
        if (g != 1) {
            uint32_t e = 2u * (uint32_t)brv(k, logN) + 1u;
            uint32_t e2 = (uint32_t)(((uint64_t)e * g) & mask2n);
            s = brv((int)((e2 - 1) >> 1), logN);
        }
        d[i] = src[limb * N + s];
    }
}

// Same copy, two coefficients (k, k+1), k even, per thread with 128-bit loads/stores: the Galois gather maps them
// to the aligned source pair {s, s^1} (brv flips the lowest bit), as in ks_inner_batch_kernel.
__global__ void gather_copy2_kernel(CopyBatch C, u64* dst, i64 dst_stride, size_t words, int N, int logN) {
    const int p = blockIdx.y;
    const u64* __restrict__ src = C.src[p];
    const uint32_t g = C.g[p];
    u64* d = dst + (size_t)p * dst_stride;
    const uint32_t mask2n = 2 * N - 1;
    const size_t pairs = words / 2;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < pairs; i += (size_t)gridDim.x * blockDim.x) {
        const size_t w = 2 * i;
        const size_t limb = w / N;
        const int k = (int)(w % N);
        int base = k, swap = 0;
        if (g != 1) {
            const uint32_t e = 2u * (uint32_t)brv(k, logN) + 1u;
            const uint32_t e2 = (uint32_t)(((uint64_t)e * g) & mask2n);
            const int sidx = brv((int)((e2 - 1) >> 1), logN);
            base = sidx & ~1;
            swap = sidx & 1;
        }
        ulonglong2 x = __ldg((const ulonglong2*)(src + limb * N + base));
        if (swap) { const u64 t = x.x; x.x = x.y; x.y = t; }
        *(ulonglong2*)(d + w) = x;
    }
}

__global__ void rescale_prep_batch_kernel(const u64* last, u64* corr, int level, int N, const ModConst* mod, const u64* hmod) {
    // corr[p][i][k] = ((last[p][k] + floor(q_{L-1}/2)) mod q_{L-1}) mod q_i - floor(q_{L-1}/2) mod q_i, i < L - 1.  A thread
    // owns two coefficients of one polynomial and writes every target limb: the last limb is read once (was once per
    // target limb), and l mod q_i is l itself when l < q_i (the 60-bit q_0) -- Barrett otherwise
    const int p = blockIdx.y;
    const int nl = level - 1;
    const u64* lp_in = last + (size_t)p * N;
    u64* cr = corr + (size_t)p * nl * N;
    const u64 qL = mod[level - 1].q, h = qL / 2;
    for (int k = 2 * (blockIdx.x * blockDim.x + threadIdx.x); k < N; k += 2 * gridDim.x * blockDim.x) {
        const ulonglong2 x = __ldg((const ulonglong2*)(lp_in + k));
        const u64 l0 = add_mod(x.x, h, qL), l1 = add_mod(x.y, h, qL);
        for (int limb = 0; limb < nl; limb++) {
            const ModConst mc = mod[limb];
            const u64 r0 = l0 < mc.q ? l0 : barrett128(U128{l0, 0}, mc.q, mc.rhi, mc.rlo);
            const u64 r1 = l1 < mc.q ? l1 : barrett128(U128{l1, 0}, mc.q, mc.rhi, mc.rlo);
            *(ulonglong2*)(cr + (size_t)limb * N + k) = make_ulonglong2(sub_mod(r0, hmod[limb], mc.q), sub_mod(r1, hmod[limb], mc.q));
        }
    }
}

__global__ void rescale_finish_batch_kernel(CopyBatch In, const u64* corr, CopyBatch Out, int level, int N,
                                            const ModConst* mod, const u64* inv, const u64* inv_sh) {
    const int p = blockIdx.y;    // polynomial (component) index
    const int nl = level - 1;
    const u64* in = In.src[p];
    u64* out = (u64*)Out.src[p];
    const u64* cr = corr + (size_t)p * nl * N;
    const size_t total = (size_t)nl * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int limb = (int)(i / N);
        u64 qi = mod[limb].q;
        out[i] = mul_shoup(sub_mod(in[i], cr[i], qi), inv[limb], inv_sh[limb], qi);
    }
}

}  // namespace

void k_ks_inner_batch(encf_ctx& c, const KsInnerBatch& B, int nreq, int dnum, int nl, int key_nl, const LimbMap& key_limb_of,
                      cudaStream_t s, const u64* pl, const u64* pl_sh) {
    bool lift = false, lift1 = false;
    for (int i = 0; i < nreq; i++) { lift |= B.c0[i] != nullptr; lift1 |= B.c1[i] != nullptr; }
    const int lslots = lift ? (lift1 ? 2 : 1) : 0;
    if (lift && (!pl || !pl_sh)) throw EncfError(ENCF_ERR_ARG, "ks_inner: c0 lift without its P factors");
    if ((unsigned __int128)dnum * c.max_mod >= ((unsigned __int128)1 << 64))
        throw EncfError(ENCF_ERR_ARG, "ks_inner: dnum * q too large for one Montgomery reduction");
    KeyLimb kl;
    LimbMap em;
    em.n = nl;
    const int Lq = c.level_of_ext(nl);
    for (int e = 0; e < nl; e++) {
        kl.kl[e] = key_limb_of.mod[e];
        em.mod[e] = (unsigned char)(e < Lq ? e : c.L + (e - Lq));
    }
    dim3 grid((c.N / 2 + TB * KS_PAIRS - 1) / (TB * KS_PAIRS), nl, nreq);
    const uint64_t bytes = (uint64_t)nreq * ((uint64_t)dnum * nl * c.N * 8 * 3 + (uint64_t)2 * nl * c.N * 8);
    int slot;
    c.prof_begin("ks_inner", s, bytes, slot);
    static const bool tma = [] { const char* e = std::getenv("ENCF_KS_TMA"); return !e || std::atoi(e) != 0; }();
    if (tma && c.N >= KT && dnum <= 4) {
        const size_t sm = (size_t)dnum * 3 * KT * 8 + (size_t)lslots * KT * 8 + 64;
        static bool attr = false;
        if (!attr) {
            CUDA_TRY(cudaFuncSetAttribute(ks_inner_tma_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 14 * KT * 8 + 64));
            CUDA_TRY(cudaFuncSetAttribute(ks_inner_tma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 14 * KT * 8 + 64));
            attr = true;
        }
        // ENCF_KS_TMA_T=128 (default): 4 coefficient pairs per thread, more CTAs (and bytes in flight) per SM
        // measured (BERT layer): 128 threads x 4 pairs 3.79 ms, 256 threads x 2 pairs 4.61 ms (profiles/r02_summary.md)
        static const int nt = [] { const char* e = std::getenv("ENCF_KS_TMA_T"); return e ? std::atoi(e) : 128; }();
        if (nt == 128)
            ks_inner_tma_kernel<128><<<dim3(c.N / KT, nl, nreq), 128, sm, s>>>(B, dnum, nl, key_nl, kl, em, c.N, c.logN, c.d_mod,
                                                                              Lq, pl, pl_sh, lslots);
        else
            ks_inner_tma_kernel<256><<<dim3(c.N / KT, nl, nreq), 256, sm, s>>>(B, dnum, nl, key_nl, kl, em, c.N, c.logN, c.d_mod,
                                                                              Lq, pl, pl_sh, lslots);
    } else {
        ks_inner_batch_kernel<<<grid, TB, 0, s>>>(B, dnum, nl, key_nl, kl, em, c.N, c.logN, c.d_mod);
        if (lift) {   // register-load variant: the lift as the separate gather + lift_add passes (same words)
            const size_t Lw = (size_t)Lq * c.N;
            u64* c0g = nullptr;
            CUDA_TRY(cudaMallocAsync((void**)&c0g, Lw * nreq * 2 * 8, s));
            CopyBatch cb{}, dst{}, src{};
            int n = 0;
            for (int i = 0; i < nreq; i++) {
                if (!B.c0[i]) continue;
                for (int cc = 0; cc < 2; cc++) {
                    const u64* cp = cc ? B.c1[i] : B.c0[i];
                    if (!cp) continue;
                    cb.src[n] = cp; cb.g[n] = B.g0[i];
                    dst.src[n] = B.acc[i] + (size_t)cc * nl * c.N; dst.g[n] = 1u;
                    src.src[n] = c0g + Lw * n; src.g[n] = 1u;
                    n++;
                }
            }
            k_gather_copy(c, cb, n, c0g, (i64)Lw, Lw, s);
            k_lift_add(c, dst, src, n, Lq, pl, pl_sh, s);
            CUDA_TRY(cudaFreeAsync(c0g, s));
        }
    }
    c.prof_end(slot, s);
    c.st_launch++; c.st_bytes += bytes;
    CUDA_TRY(cudaGetLastError());
}

void k_ks_rotsum(encf_ctx& c, const RotSumBatch& B, int nreq, int nterms, int dnum, int L, int key_nl, cudaStream_t s) {
    if (nterms > RS_TERMS) throw EncfError(ENCF_ERR_ARG, "rotation sum: too many terms");
    const int nl = L + c.Kof(L);
    KeyLimb kl;
    for (int e = 0; e < nl; e++) kl.kl[e] = e < L ? e : (key_nl - c.Kof(L)) + (e - L);
    const LimbMap em = c.extmap(L);
    dim3 grid(nreq, (c.N / 2 + TB - 1) / TB, nl);
    const uint64_t bytes = (uint64_t)nterms * dnum * 2 * nl * c.N * 8 + (uint64_t)nreq * (dnum * nl + 2 * L + 2 * nl) * c.N * 8;
    int slot;
    c.prof_begin("ks_rotsum", s, bytes, slot);
    // ENCF_ROTSUM_TMA=1: the cp.async.bulk ring variant -- measured slower (BERT layer 1.93 -> 3.00 ms: one barrier round
    // per (term, digit) stage of a 512-coefficient tile), so the register-load kernel is the default
    static const bool tma = [] { const char* e = std::getenv("ENCF_ROTSUM_TMA"); return e && std::atoi(e) != 0; }();
    if (tma && c.N >= RKT) {
        const size_t sm = (size_t)RS_NST * 4 * RKT * 8 + RS_NST * 8;
        static bool attr = false;
        if (!attr) {
            CUDA_TRY(cudaFuncSetAttribute(ks_rotsum_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            attr = true;
        }
        ks_rotsum_tma_kernel<<<dim3(nreq, c.N / RKT, nl), RS_NT, sm, s>>>(B, nterms, dnum, nl, L, key_nl, kl, em, c.N, c.logN,
                                                                          c.d_mod, c.moddown[L].d_pl, c.moddown[L].d_pl_sh);
    } else {
        ks_rotsum_kernel<<<grid, TB, 0, s>>>(B, nterms, dnum, nl, L, key_nl, kl, em, c.N, c.logN, c.d_mod, c.moddown[L].d_pl,
                                             c.moddown[L].d_pl_sh);
    }
    c.prof_end(slot, s);
    c.st_launch++; c.st_bytes += bytes;
    CUDA_TRY(cudaGetLastError());
}

void k_ks_psi(encf_ctx& c, const PsiBatch& B, int nreq, int dnum, int L, int key_nl, cudaStream_t s) {
    const int nl = L + c.Kof(L);
    if ((unsigned __int128)(2 * dnum + 2) * c.max_mod >= ((unsigned __int128)1 << 64))
        throw EncfError(ENCF_ERR_ARG, "ks_psi: too many products for one Montgomery reduction");
    const LimbMap em = c.extmap(L);
    dim3 grid(nreq, (c.N / 2 + TB - 1) / TB, nl);
    const uint64_t bytes = (uint64_t)nreq * (2 * dnum * nl + 2 * 2 * dnum * nl + 2 * L + 2 * L + 2 * nl) * c.N * 8;
    int slot;
    c.prof_begin("ks_psi", s, bytes, slot);
    static const bool tma = [] { const char* e = std::getenv("ENCF_KS_TMA"); return !e || std::atoi(e) != 0; }();
    // tile (ENCF_PSI_TILE): 512 coefficients x 128 threads (default) or 1024 x 256
    static const int tile = [] { const char* e = std::getenv("ENCF_PSI_TILE"); return e ? std::atoi(e) : 512; }();
    const size_t sm = (size_t)2 * (3 * dnum + 2) * tile * 8 + 64;
    if (tma && c.N >= tile && sm <= 227 * 1024) {
        static bool attr = false;
        if (!attr) {
            CUDA_TRY(cudaFuncSetAttribute(ks_psi_tma_kernel<1024, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            CUDA_TRY(cudaFuncSetAttribute(ks_psi_tma_kernel<512, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            attr = true;
        }
        if (tile == 1024)
            ks_psi_tma_kernel<1024, 256><<<dim3(nreq, c.N / 1024, nl), 256, sm, s>>>(B, dnum, nl, L, em, c.N, c.logN, c.d_mod);
        else
            ks_psi_tma_kernel<512, 128><<<dim3(nreq, c.N / 512, nl), 128, sm, s>>>(B, dnum, nl, L, em, c.N, c.logN, c.d_mod);
    } else {
        ks_psi_kernel<<<grid, TB, 0, s>>>(B, dnum, nl, L, em, c.N, c.logN, c.d_mod);
    }
    c.prof_end(slot, s);
    c.st_launch++; c.st_bytes += bytes;
    c.st_ptmul += 2 * (uint64_t)nreq;
    (void)key_nl;
    CUDA_TRY(cudaGetLastError());
}

__global__ void key_class_kernel(const u64* __restrict__ full, int nl_full, u64* __restrict__ out, int nl_out, int ML, int dnum,
                                 int alpha, const u64* __restrict__ sp, const u64* __restrict__ dr, int N,
                                 const ModConst* __restrict__ mod) {
    const size_t total = (size_t)dnum * 2 * nl_out * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % N);
        const size_t row = i / N;
        const int e = (int)(row % nl_out), jc = (int)(row / nl_out), j = jc >> 1, comp = jc & 1;
        u64 v = full[((size_t)jc * nl_full + e) * N + k];     // special limb k sits at ML + k in both layouts
        if (comp == 0 && e >= j * alpha && e < min((j + 1) * alpha, ML)) {
            const ModConst mc = mod[e];
            v = add_mod(v, mulmod_barrett(sp[(size_t)e * N + k], dr[e], mc.q, mc.rhi, mc.rlo), mc.q);
        }
        out[i] = v;
    }
}

void k_key_class(encf_ctx& c, const u64* full, int nl_full, u64* out, int nl_out, int ML, int dnum, const u64* sp, const u64* dr,
                 cudaStream_t s) {
    key_class_kernel<<<GRID((size_t)dnum * 2 * nl_out * c.N), TB, 0, s>>>(full, nl_full, out, nl_out, ML, dnum, c.alpha, sp, dr, c.N,
                                                                         c.d_mod);
    c.st_launch++;
    CUDA_TRY(cudaGetLastError());
}

void k_keymask(encf_ctx& c, const u64* key, int key_nl, const u64* mask, int dnum, int L, u64* out, cudaStream_t s) {
    const int nl = L + c.Kof(L);
    KeyLimb kl;
    for (int e = 0; e < nl; e++) kl.kl[e] = e < L ? e : (key_nl - c.Kof(L)) + (e - L);
    const LimbMap em = c.extmap(L);
    std::vector<u64> pr(L);
    for (int i = 0; i < L; i++) {
        const u64 q = c.mods[i];
        u64 P = 1;                                       // P_{K(L)} (R-KL)
        for (int kk = 0; kk < c.Kof(L); kk++) P = h_mulmod(P, c.mods[c.L + kk] % q, q);
        pr[i] = h_mulmod(P, c.mont_R[i], q);
    }
    u64* dpr = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&dpr, L * 8, s));
    CUDA_TRY(cudaMemcpyAsync(dpr, pr.data(), L * 8, cudaMemcpyHostToDevice, s));
    keymask_kernel<<<GRID((size_t)(dnum * 2 + 1) * nl * c.N), TB, 0, s>>>(key, key_nl, mask, dnum, L, nl, kl, em, dpr, out, c.N,
                                                                        c.d_mod);
    CUDA_TRY(cudaFreeAsync(dpr, s));
    c.st_launch++;
    CUDA_TRY(cudaGetLastError());
}

void k_ks_rma(encf_ctx& c, const RotSumBatch& B, int nreq, int nterms, int dnum, int L, int key_nl, cudaStream_t s) {
    if (nterms > RS_TERMS) throw EncfError(ENCF_ERR_ARG, "rma: too many terms");
    const int nl = L + c.Kof(L);
    KeyLimb kl;
    for (int e = 0; e < nl; e++) kl.kl[e] = e < L ? e : (key_nl - c.Kof(L)) + (e - L);
    const LimbMap em = c.extmap(L);
    dim3 grid(nreq, (c.N / 2 + TB - 1) / TB, nl);
    int slot;
    c.prof_begin("ks_rma", s, 0, slot);
    ks_rma_kernel<<<grid, TB, 0, s>>>(B, nterms, dnum, nl, L, key_nl, kl, em, c.N, c.logN, c.d_mod, c.moddown[L].d_pl,
                                      c.moddown[L].d_pl_sh);
    c.prof_end(slot, s);
    c.st_launch++;
    c.st_ptmul += (uint64_t)nreq * nterms;
    CUDA_TRY(cudaGetLastError());
}

void k_moddown_finish_batch(encf_ctx& c, const u64* acc, const u64* y, const OutBatch& O, int nreq, int level, int nl,
                            const ModDownTab& t, cudaStream_t s) {
    dim3 grid(nblocks((size_t)level * c.N, TB, 256), 1, 2 * nreq);
    { int _slot; c.prof_begin("moddown_finish_batch_kernel", s, 0, _slot);
    moddown_finish_batch_kernel<<<grid, TB, 0, s>>>(acc, y, O, level, nl, c.N, c.d_mod, t.d_pinv, t.d_pinv_sh);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += (uint64_t)nreq * 2 * level * c.N * 8 * 4;
}

void k_bconv_batch(encf_ctx& c, const u64* in, i64 in_stride, const LimbMap& im, const u64* vf, const u64* vfs, const u64* wf,
                   const LimbMap& om, u64* out, i64 out_stride, const int* pos, int npolys, cudaStream_t s, const u64* corr,
                   const u64* cfix, const u64* csh, const uint8_t* wb, bool prescaled) {
    const int pre = prescaled ? 1 : 0;
    if (im.n > 16 || im.n < 1) throw EncfError(ENCF_ERR_ARG, "bconv: 1..16 input limbs");
    if (c.max_mod >= (1ull << 60) || im.n > 8) throw EncfError(ENCF_ERR_ARG, "bconv: the 30-bit split needs moduli < 2^60 and <= 8 inputs");
    {   // Montgomery bound of the lazy sum: sum_i q_i + (n_in + 1) <= 2^64 (then T < q_t 2^64)
        unsigned __int128 tot = (unsigned __int128)im.n + 1;
        for (int i = 0; i < im.n; i++) tot += c.mods[im.mod[i]];
        if (tot >> 64) throw EncfError(ENCF_ERR_ARG, "bconv: input moduli too large for the 128-bit lazy sum");
    }
    OutPos op;
    for (int t = 0; t < om.n; t++) op.pos[t] = pos[t];
    static const bool tc = [] { const char* e = std::getenv("ENCF_BCONV_TC"); return !e || std::atoi(e) != 0; }();
    if (tc && wb && om.n <= 32 && c.N % BTC_TILE == 0) {
        const int nb = 8 * ((om.n + 1) & ~1);
        const int tcols = nb <= 32 ? 32 : nb <= 64 ? 64 : nb <= 128 ? 128 : 256;
        const int per_sm = std::min(4, 512 / tcols);   // TMEM: <= 512 columns per SM; smem request caps CTAs per SM
        const size_t need = (size_t)BTC_TILE * 64 + (size_t)nb * 64 + 4 * 32 * 8 + 16;
        const size_t smem_tc = std::max(need, (size_t)(220 * 1024) / per_sm);
        static bool attr = false;
        if (!attr) {
#define A(NI) CUDA_TRY(cudaFuncSetAttribute(bconv_tc_kernel<NI, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)); \
              CUDA_TRY(cudaFuncSetAttribute(bconv_tc_kernel<NI, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            A(1) A(2) A(3) A(4) A(5) A(6) A(7) A(8)
#undef A
            attr = true;
        }
        const int ntiles = c.N / BTC_TILE * npolys;
        const int grid = std::min(ntiles, 148 * per_sm);
        { int _slot; c.prof_begin("bconv_batch_kernel", s, 0, _slot);
        switch (im.n) {
#define B(NI) case NI: if (corr) bconv_tc_kernel<NI, true><<<grid, BTC_TILE, smem_tc, s>>>(in, in_stride, im, vf, vfs, wb, nb, tcols, \
                  om, op, out, out_stride, c.N, npolys, c.d_mod, corr, cfix, csh, pre); \
              else bconv_tc_kernel<NI, false><<<grid, BTC_TILE, smem_tc, s>>>(in, in_stride, im, vf, vfs, wb, nb, tcols, om, op, out, \
                  out_stride, c.N, npolys, c.d_mod, corr, cfix, csh, pre); break;
            B(1) B(2) B(3) B(4) B(5) B(6) B(7) B(8)
#undef B
        }
        c.prof_end(_slot, s); }
        c.st_launch++; c.st_bytes += (uint64_t)npolys * (im.n + om.n) * c.N * 8;
        CUDA_TRY(cudaGetLastError());
        return;
    }
    size_t smem = ((size_t)im.n * om.n + 4 * om.n + 5 * im.n) * sizeof(u64);
    dim3 grid((c.N + TB - 1) / TB, npolys);
    { int _slot; c.prof_begin("bconv_batch_kernel", s, 0, _slot);
    switch (im.n) {
#define B(NI) case NI: bconv_batch_kernel<NI><<<grid, TB, smem, s>>>(in, in_stride, im, vf, vfs, wf, om, op, out, out_stride, c.N, c.d_mod, corr, cfix, csh, pre); break;
        B(1) B(2) B(3) B(4) B(5) B(6) B(7) B(8) B(9) B(10) B(11) B(12) B(13) B(14) B(15) B(16)
#undef B
    }
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += (uint64_t)npolys * (im.n + om.n) * c.N * 8;
    CUDA_TRY(cudaGetLastError());
}

void k_gather_copy(encf_ctx& c, const CopyBatch& C, int n, u64* dst, i64 dst_stride, size_t words, cudaStream_t s) {
    { int _slot; c.prof_begin("gather_copy_kernel", s, 0, _slot);
    bool aligned = (words % 2 == 0) && (dst_stride % 2 == 0) && ((uintptr_t)dst % 16 == 0);
    for (int i = 0; i < n; i++) aligned = aligned && ((uintptr_t)C.src[i] % 16 == 0);
    if (aligned) {
        dim3 grid(nblocks(words / 2, TB, 512), n);
        gather_copy2_kernel<<<grid, TB, 0, s>>>(C, dst, dst_stride, words, c.N, c.logN);
    } else {
        dim3 grid(nblocks(words, TB, 512), n);
        gather_copy_kernel<<<grid, TB, 0, s>>>(C, dst, dst_stride, words, c.N, c.logN);
    }
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += (uint64_t)n * words * 16;
}

void k_rescale_prep_batch(encf_ctx& c, const u64* last, u64* corr, int level, int npolys, cudaStream_t s) {
    dim3 grid(nblocks((size_t)c.N / 2, TB, 256), npolys);
    { int _slot; c.prof_begin("rescale_prep_batch_kernel", s, 0, _slot);
    rescale_prep_batch_kernel<<<grid, TB, 0, s>>>(last, corr, level, c.N, c.d_mod, c.rescale[level].d_hmod);
    c.prof_end(_slot, s); }
    c.st_launch++;
}

void k_rescale_finish_batch(encf_ctx& c, const CopyBatch& In, const u64* corr, const CopyBatch& Out, int level, int npolys,
                            cudaStream_t s) {
    const RescaleTab& t = c.rescale[level];
    dim3 grid(nblocks((size_t)(level - 1) * c.N, TB, 256), npolys);
    { int _slot; c.prof_begin("rescale_finish_batch_kernel", s, 0, _slot);
    rescale_finish_batch_kernel<<<grid, TB, 0, s>>>(In, corr, Out, level, c.N, c.d_mod, t.d_inv, t.d_inv_sh);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += (uint64_t)npolys * (level - 1) * c.N * 8 * 3;
}

// ====================================================================================== batched lazy sums
namespace {

// outs[o] = sum_{t in [off[o], off[o+1])} ct_t (.) mask_t   (mask_t == nullptr: plain add), all
// components, 128-bit lazy accumulation reduced every 128 terms.
__global__ void __launch_bounds__(TB) sum_csr_kernel(const SumDev* __restrict__ terms, const int* __restrict__ off,
                                                     u64* const* __restrict__ outs, int ncomp, int level, int N,
                                                     const ModConst* __restrict__ mod, LimbMap lm) {
    const int o = blockIdx.z, limb = blockIdx.y;
    const ModConst mc = mod[lm.mod[limb]];
    const size_t cs = (size_t)level * N;
    const int t0 = off[o], t1 = off[o + 1];
    u64* out = outs[o];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const size_t idx = (size_t)limb * N + k;
        for (int c = 0; c < ncomp; c++) {
            u64 r = 0;
            for (int ta = t0; ta < t1; ta += 128) {
                U128 acc{0, 0};
                const int tb = min(t1, ta + 128);
                for (int t = ta; t < tb; t++) {
                    const u64* ct = terms[t].ct;
                    const u64* m = terms[t].mask;
                    u64 x = ct[c * cs + idx];
                    if (m) mac128(acc, x, m[idx]);
                    else add128(acc, x);
                }
                r = add_mod(r, barrett128(acc, mc.q, mc.rhi, mc.rlo), mc.q);
            }
            out[c * cs + idx] = r;
        }
    }
}

// Two-component variant: two coefficients per thread (128-bit loads), both components in one pass over the terms
// (one term-descriptor load per term instead of two), and the next term's three loads issued before the current
// term's products (the one-word loop was latency-bound at ~2.5 TB/s).
__global__ void __launch_bounds__(TB) sum_csr2_kernel(const SumDev* __restrict__ terms, const int* __restrict__ off,
                                                      u64* const* __restrict__ outs, int level, int N,
                                                      const ModConst* __restrict__ mod, LimbMap lm) {
    const int o = blockIdx.z, limb = blockIdx.y;
    const ModConst mc = mod[lm.mod[limb]];
    const size_t cs = (size_t)level * N;
    const int t0 = off[o], t1 = off[o + 1];
    u64* out = outs[o];
    for (int kp = blockIdx.x * blockDim.x + threadIdx.x; 2 * kp < N; kp += gridDim.x * blockDim.x) {
        const size_t idx = (size_t)limb * N + 2 * kp;
        u64 r00 = 0, r01 = 0, r10 = 0, r11 = 0;   // [component][coefficient]
        for (int ta = t0; ta < t1; ta += 128) {
            U128 a00{0, 0}, a01{0, 0}, a10{0, 0}, a11{0, 0};
            const int tb = min(t1, ta + 128);
            int t = ta;
            for (; t + 2 <= tb; t += 2) {
                const SumDev d0 = terms[t], d1 = terms[t + 1];
                const ulonglong2 x0 = __ldg((const ulonglong2*)(d0.ct + idx));
                const ulonglong2 y0 = __ldg((const ulonglong2*)(d0.ct + cs + idx));
                const ulonglong2 x1 = __ldg((const ulonglong2*)(d1.ct + idx));
                const ulonglong2 y1 = __ldg((const ulonglong2*)(d1.ct + cs + idx));
                const ulonglong2 m0 = d0.mask ? __ldg((const ulonglong2*)(d0.mask + idx)) : make_ulonglong2(0, 0);
                const ulonglong2 m1 = d1.mask ? __ldg((const ulonglong2*)(d1.mask + idx)) : make_ulonglong2(0, 0);
                if (d0.mask) { mac128(a00, x0.x, m0.x); mac128(a01, x0.y, m0.y); mac128(a10, y0.x, m0.x); mac128(a11, y0.y, m0.y); }
                else { add128(a00, x0.x); add128(a01, x0.y); add128(a10, y0.x); add128(a11, y0.y); }
                if (d1.mask) { mac128(a00, x1.x, m1.x); mac128(a01, x1.y, m1.y); mac128(a10, y1.x, m1.x); mac128(a11, y1.y, m1.y); }
                else { add128(a00, x1.x); add128(a01, x1.y); add128(a10, y1.x); add128(a11, y1.y); }
            }
            if (t < tb) {
                const SumDev d0 = terms[t];
                const ulonglong2 x0 = __ldg((const ulonglong2*)(d0.ct + idx));
                const ulonglong2 y0 = __ldg((const ulonglong2*)(d0.ct + cs + idx));
                if (d0.mask) {
                    const ulonglong2 m0 = __ldg((const ulonglong2*)(d0.mask + idx));
                    mac128(a00, x0.x, m0.x); mac128(a01, x0.y, m0.y); mac128(a10, y0.x, m0.x); mac128(a11, y0.y, m0.y);
                } else { add128(a00, x0.x); add128(a01, x0.y); add128(a10, y0.x); add128(a11, y0.y); }
            }
            r00 = add_mod(r00, barrett128(a00, mc.q, mc.rhi, mc.rlo), mc.q);
            r01 = add_mod(r01, barrett128(a01, mc.q, mc.rhi, mc.rlo), mc.q);
            r10 = add_mod(r10, barrett128(a10, mc.q, mc.rhi, mc.rlo), mc.q);
            r11 = add_mod(r11, barrett128(a11, mc.q, mc.rhi, mc.rlo), mc.q);
        }
        *(ulonglong2*)(out + idx) = make_ulonglong2(r00, r01);
        *(ulonglong2*)(out + cs + idx) = make_ulonglong2(r10, r11);
    }
}

// outs[o] = sum_{t in [off[o], off[o+1])} (a0 b0, a0 b1 + a1 b0, a1 b1)
// Grid (output, coefficient block, limb) with the OUTPUT fastest: the CTAs running together cover one coefficient
// block of every output, so operands shared between outputs (the score kernel's Q/K banks: B (beta + g/2) ciphertexts
// feed all m/2 outputs) are read from HBM about once and re-read from L2.  Karatsuba per pair: a0 b1 + a1 b0 =
// (a0 + a1)(b0 + b1) - a0 b0 - a1 b1, exact in 128 bits over chunks of 16 pairs ((2q)^2 16 < 2^128 for q < 2^61).
// TENSOR_OLD=1 builds the previous kernel (limb-major grid, four products per pair) for A/B.
#ifndef TENSOR_OLD
#define TENSOR_OLD 0
#endif
__global__ void __launch_bounds__(TB) tensor_csr_kernel(const PairDev* __restrict__ pairs, const int* __restrict__ off,
                                                        u64* const* __restrict__ outs, int level, int N,
                                                        const ModConst* __restrict__ mod) {
#if TENSOR_OLD
    const int o = blockIdx.z, limb = blockIdx.y;
#else
    const int o = blockIdx.x, limb = blockIdx.z;
#endif
    const ModConst mc = mod[limb];
    const size_t cs = (size_t)level * N;
    const int t0 = off[o], t1 = off[o + 1];
    u64* out = outs[o];
#if TENSOR_OLD
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
#else
    for (int k = blockIdx.y * blockDim.x + threadIdx.x; k < N; k += gridDim.y * blockDim.x) {
#endif
        const size_t idx = (size_t)limb * N + k;
        u64 r0 = 0, r1 = 0, r2 = 0;
#if TENSOR_OLD
        for (int ta = t0; ta < t1; ta += 64) {
            U128 d0{0, 0}, d1{0, 0}, d2{0, 0};
            const int tb = min(t1, ta + 64);
            for (int t = ta; t < tb; t++) {
                const u64* a = pairs[t].a;
                const u64* b = pairs[t].b;
                u64 a0 = a[idx], a1 = a[pairs[t].as + idx], b0 = b[idx], b1 = b[pairs[t].bs + idx];
                mac128(d0, a0, b0);
                mac128(d1, a0, b1);
                mac128(d1, a1, b0);
                mac128(d2, a1, b1);
            }
#else
        for (int ta = t0; ta < t1; ta += 16) {
            U128 d0{0, 0}, sm{0, 0}, d2{0, 0};
            const int tb = min(t1, ta + 16);
            for (int t = ta; t < tb; t++) {
                const u64* a = pairs[t].a;
                const u64* b = pairs[t].b;
                u64 a0 = a[idx], a1 = a[pairs[t].as + idx], b0 = b[idx], b1 = b[pairs[t].bs + idx];
                mac128(d0, a0, b0);
                mac128(d2, a1, b1);
                mac128(sm, a0 + a1, b0 + b1);
            }
            // d1 = sm - d0 - d2 >= 0 (exact)
            U128 d1 = sm;
            {
                const u64 lo = d1.lo - d0.lo;
                d1.hi = d1.hi - d0.hi - (d1.lo < d0.lo);
                d1.lo = lo;
                const u64 lo2 = d1.lo - d2.lo;
                d1.hi = d1.hi - d2.hi - (d1.lo < d2.lo);
                d1.lo = lo2;
            }
#endif
            r0 = add_mod(r0, barrett128(d0, mc.q, mc.rhi, mc.rlo), mc.q);
            r1 = add_mod(r1, barrett128(d1, mc.q, mc.rhi, mc.rlo), mc.q);
            r2 = add_mod(r2, barrett128(d2, mc.q, mc.rhi, mc.rlo), mc.q);
        }
        out[idx] = r0;
        out[cs + idx] = r1;
        out[2 * cs + idx] = r2;
    }
}

}  // namespace

void k_sum_csr(encf_ctx& c, const SumDev* terms, const int* off, u64* const* outs, int nout, int nterms, int ncomp, int level,
               cudaStream_t s, const LimbMap* lmap) {
    LimbMap lm = lmap ? *lmap : c.qmap(level);
    { int _slot; c.prof_begin("sum_csr_kernel", s, 0, _slot);
    if (ncomp == 2) {
        dim3 grid((c.N / 2 + TB - 1) / TB, level, nout);
        sum_csr2_kernel<<<grid, TB, 0, s>>>(terms, off, outs, level, c.N, c.d_mod, lm);
    } else {
        dim3 grid((c.N + TB - 1) / TB, level, nout);
        sum_csr_kernel<<<grid, TB, 0, s>>>(terms, off, outs, ncomp, level, c.N, c.d_mod, lm);
    }
    c.prof_end(_slot, s); }
    c.st_launch++;
    c.st_bytes += (uint64_t)nterms * ncomp * level * c.N * 8 * 2 + (uint64_t)nout * ncomp * level * c.N * 8;
}

void k_tensor_csr(encf_ctx& c, const PairDev* pairs, const int* off, u64* const* outs, int nout, int nterms, int level,
                  cudaStream_t s) {
#if TENSOR_OLD
    dim3 grid((c.N + TB - 1) / TB, level, nout);
#else
    if (nout > (1 << 30)) throw EncfError(ENCF_ERR_ARG, "tensor: too many outputs");
    dim3 grid(nout, (c.N + TB - 1) / TB, level);
#endif
    { int _slot; c.prof_begin("tensor_csr_kernel", s, 0, _slot);
    tensor_csr_kernel<<<grid, TB, 0, s>>>(pairs, off, outs, level, c.N, c.d_mod);
    c.prof_end(_slot, s); }
    c.st_launch++;
    c.st_bytes += (uint64_t)nterms * 4 * level * c.N * 8 + (uint64_t)nout * 3 * level * c.N * 8;
    c.st_ctmul += nterms;
}

// ====================================================================================== value-kernel broadcast MAC
// b_t = sum_{u < nu} src[t - u] (.) mask_u for t in [t0, t0 + nt), src[delta] = Phi^delta(p_fd) (C8 step 4).
// Coefficient-tiled: the whole delta window (<= 127 ciphertexts x 2 components) and the nu masks of a
// 32-coefficient tile sit in shared memory; every bank word is read from HBM once per launch.
namespace {
constexpr int BC_T = 32;

// One (t group, component) item of the narrow path: b_t = sum_u src[t - u] (.) mask_u for t in [t0, t0 + BC_TR), with the
// 20-bit Karatsuba split of diag_mac_kernel.  Sliding window: stepping u -> u + 1 shifts the TR source words by one
// position, so each step loads one new source word and one mask word (register ring indexed (j - u) mod TR, resolved
// at compile time by unrolling u by TR).  FP = true runs the same split products on the FP64 pipe: pieces < 2^21,
// products < 2^42, sums of <= 64 products < 2^48 -- exact in doubles, so the words are identical.
constexpr int BC_TR = 8;
template <bool FP>
__device__ __forceinline__ void bc_item(const BcastArgs& A, const uint2* ss, const uint2* sk, int kk, int t0, int c, size_t cs,
                                        size_t lo, const ModConst& mc, u64 t40) {
    constexpr int TR = BC_TR;
    using V = typename std::conditional<FP, double, uint32_t>::type;
    using Acc = typename std::conditional<FP, double, u64>::type;
    auto cv = [](uint32_t x) -> V {
        if constexpr (FP) return __dsub_rn(__hiloint2double(0x43300000, (int)x), 4503599627370496.0);
        else return x;
    };
    Acc hh[TR], ll[TR], sum[TR];
#pragma unroll
    for (int jj = 0; jj < TR; jj++) hh[jj] = ll[jj] = sum[jj] = 0;
    // src word of (t0 + jj, u) = ss[(t0 + jj + dmax - u) * 2 BC_T + c BC_T + kk]; indices past the window only occur for
    // t >= nt (never stored) -- clamp them into it
    const uint2* sp = ss + c * BC_T + kk;
    const int dlast = A.nsrc - 1;
    auto src_at = [&](int d) -> uint2 { return sp[(size_t)min(d, dlast) * 2 * BC_T]; };
    V wh[TR], wl[TR], ws[TR];
#pragma unroll
    for (int jj = 0; jj < TR; jj++) {
        const uint2 x = src_at(t0 + jj + A.dmax);
        wh[jj] = cv(x.x); wl[jj] = cv(x.y); ws[jj] = FP ? wh[jj] + wl[jj] : cv(x.x + x.y);
    }
    for (int u0 = 0; u0 < A.nu; u0 += TR) {
#pragma unroll
        for (int du = 0; du < TR; du++) {
            const int u = u0 + du;
            if (u < A.nu) {
                if (u > 0) {   // position 0 of step u enters the slot that held position TR - 1 of step u - 1
                    const uint2 x = src_at(t0 - u + A.dmax);
                    const V h = cv(x.x), l = cv(x.y);
                    const V sv = FP ? h + l : cv(x.x + x.y);
                    const int sl = (TR - du) % TR;
#pragma unroll
                    for (int q = 0; q < TR; q++)
                        if (q == sl) { wh[q] = h; wl[q] = l; ws[q] = sv; }
                }
                const uint2 m = sk[u * BC_T + kk];
                const V mh = cv(m.x), ml = cv(m.y);
                const V ms = FP ? mh + ml : cv(m.x + m.y);
#pragma unroll
                for (int jj = 0; jj < TR; jj++) {
                    const int q = (jj - du + TR) % TR;
                    if constexpr (FP) {
                        hh[jj] = __fma_rn(wh[q], mh, hh[jj]);
                        ll[jj] = __fma_rn(wl[q], ml, ll[jj]);
                        sum[jj] = __fma_rn(ws[q], ms, sum[jj]);
                    } else {
                        hh[jj] += (u64)wh[q] * mh;
                        ll[jj] += (u64)wl[q] * ml;
                        sum[jj] += (u64)ws[q] * ms;
                    }
                }
            }
        }
    }
    const int jmax = min(TR, A.nt - t0);
#pragma unroll
    for (int jj = 0; jj < TR; jj++) {
        if (jj < jmax) {
            u64 h, l, sm;
            if constexpr (FP) { h = (u64)__double2ull_rz(hh[jj]); l = (u64)__double2ull_rz(ll[jj]); sm = (u64)__double2ull_rz(sum[jj]); }
            else { h = hh[jj]; l = ll[jj]; sm = sum[jj]; }
            A.out[t0 + jj][c * cs + lo + kk] = kara_combine(h, l, sm, mc.q, mc.rhi, mc.rlo, t40);
        }
    }
}

__global__ void __launch_bounds__(256) bcast_mac_kernel(BcastArgs A, int level, int N, const ModConst* __restrict__ mod) {
    extern __shared__ u64 sb[];                 // [nsrc][2][BC_T] then [nu][BC_T]  (narrow limbs: uint2 {h, l} per word)
    const int limb = blockIdx.y, k0 = blockIdx.x * BC_T;
    const ModConst mc = mod[limb];
    const bool narrow = mc.q < (1ull << 41);   // 20-bit Karatsuba split (see diag_mac_kernel)
    const size_t cs = (size_t)level * N;
    const size_t lo = (size_t)limb * N + k0;
    u64* sm_src = sb;
    u64* sm_msk = sb + (size_t)A.nsrc * 2 * BC_T;
    for (int i = threadIdx.x; i < A.nsrc * 2 * BC_T; i += blockDim.x) {
        int d = i / (2 * BC_T), r = i % (2 * BC_T);
        int c = r / BC_T, kk = r % BC_T;
        const u64 x = A.src[d][c * cs + lo + kk];
        sm_src[i] = narrow ? ((x >> 20) | ((x & 0xFFFFF) << 32)) : ((x >> 30) | ((x & 0x3FFFFFFFull) << 32));
    }
    for (int i = threadIdx.x; i < A.nu * BC_T; i += blockDim.x) {
        const u64 x = A.mask[i / BC_T][lo + i % BC_T];
        sm_msk[i] = narrow ? ((x >> 20) | ((x & 0xFFFFF) << 32)) : ((x >> 30) | ((x & 0x3FFFFFFFull) << 32));
    }
    __syncthreads();
    const int kk = threadIdx.x % BC_T, w = threadIdx.x / BC_T, nw = blockDim.x / BC_T;
    if (narrow) {
        const u64 t40 = (1ull << 40) % mc.q;
        const uint2* ss = (const uint2*)sm_src;
        const uint2* sk = (const uint2*)sm_msk;
        // register blocking over TR = 8 consecutive t of one component with a SLIDING window (bc_item); every SM
        // sub-partition (warp % 4) holds warps of both pipes
        // An integer-pipe item costs ~1.6x an FP64-pipe item (3 half-rate IMAD.WIDE vs ~3.75 full-rate FP64 ops per
        // product), so FP64 takes ~5/8 of the items: warps 4-7 always, warps 0-3 their second item in every other CTA.
        const int ngrp = (A.nt + BC_TR - 1) / BC_TR;
        const bool fpw = (w >> 2) & 1, odd_cta = (blockIdx.x + blockIdx.y) & 1;
        for (int o = w; o < ngrp * 2; o += nw) {
            const bool fp = fpw || (!odd_cta && o >= nw);
            if (fp) bc_item<true>(A, ss, sk, kk, (o >> 1) * BC_TR, o & 1, cs, lo, mc, t40);
            else bc_item<false>(A, ss, sk, kk, (o >> 1) * BC_TR, o & 1, cs, lo, mc, t40);
        }
        return;
    }
    // 128-bit path (2^41 <= q < 2^60): the same sliding window over TW = 4 consecutive t, words split at 30 bits
    // ({h, l} in shared memory): per product 4 IMAD.WIDE.U32 into 64-bit sums hh, md (= xh ml + xl mh), ll; every 8 u
    // (md < 16 (2^30 - 1)^2 < 2^64) they fold into a 128-bit sum, reduced below q every 32 u (32 q^2 < 2^127)
    constexpr int TW = 4;
    const int ngw = (A.nt + TW - 1) / TW;
    const int dlast = A.nsrc - 1;
    const uint2* ss = (const uint2*)sm_src;
    const uint2* sk = (const uint2*)sm_msk;
    for (int o = w; o < ngw * 2; o += nw) {
        const int t0 = (o >> 1) * TW, c = o & 1;
        U128 acc[TW];
        u64 hh[TW], md[TW], ll[TW];
#pragma unroll
        for (int jj = 0; jj < TW; jj++) { acc[jj] = U128{0, 0}; hh[jj] = md[jj] = ll[jj] = 0; }
        const uint2* sp = ss + c * BC_T + kk;
        auto src_at = [&](int d) -> uint2 { return sp[(size_t)min(d, dlast) * 2 * BC_T]; };
        uint2 win[TW];
#pragma unroll
        for (int jj = 0; jj < TW; jj++) win[jj] = src_at(t0 + jj + A.dmax);
        for (int u0 = 0; u0 < A.nu; u0 += TW) {
#pragma unroll
            for (int du = 0; du < TW; du++) {
                const int u = u0 + du;
                if (u < A.nu) {
                    if (u > 0) {
                        const uint2 x = src_at(t0 - u + A.dmax);
#pragma unroll
                        for (int q = 0; q < TW; q++) if (q == (TW - du) % TW) win[q] = x;
                    }
                    const uint2 m = sk[u * BC_T + kk];
#pragma unroll
                    for (int jj = 0; jj < TW; jj++) {
                        const uint2 x = win[(jj - du + TW) % TW];
                        hh[jj] += (u64)x.x * m.x;
                        md[jj] += (u64)x.x * m.y + (u64)x.y * m.x;
                        ll[jj] += (u64)x.y * m.y;
                    }
                }
            }
            if (((u0 + TW) & 7) == 0 || u0 + TW >= A.nu) {
#pragma unroll
                for (int jj = 0; jj < TW; jj++) {
                    add128(acc[jj], ll[jj]);
                    add128(acc[jj], md[jj] << 30);
                    acc[jj].hi += md[jj] >> 34;
                    add128(acc[jj], hh[jj] << 60);
                    acc[jj].hi += hh[jj] >> 4;
                    hh[jj] = md[jj] = ll[jj] = 0;
                }
            }
            if (((u0 + TW) & 31) == 0) {
#pragma unroll
                for (int jj = 0; jj < TW; jj++) acc[jj] = U128{barrett128(acc[jj], mc.q, mc.rhi, mc.rlo), 0};
            }
        }
        const int jmax = min(TW, A.nt - t0);
#pragma unroll
        for (int jj = 0; jj < TW; jj++)
            if (jj < jmax) A.out[t0 + jj][c * cs + lo + kk] = barrett128(acc[jj], mc.q, mc.rhi, mc.rlo);
    }
}
}  // namespace

void k_bcast_mac(encf_ctx& c, const BcastArgs& A, int level, cudaStream_t s) {
    if (c.max_mod >= (1ull << 60)) throw EncfError(ENCF_ERR_ARG, "bcast_mac: the 30-bit split needs moduli < 2^60");
    const size_t smem = ((size_t)A.nsrc * 2 + A.nu) * BC_T * sizeof(u64);
    static bool attr = false;
    if (!attr) {
        CUDA_TRY(cudaFuncSetAttribute(bcast_mac_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        attr = true;
    }
    if (smem > 220 * 1024) throw EncfError(ENCF_ERR_PLAN_SHAPE, "bcast_mac: window too large");
    dim3 grid(c.N / BC_T, level);
    const uint64_t bytes = ((uint64_t)A.nsrc * 2 + A.nu + (uint64_t)A.nt * 2) * level * c.N * 8;
    int slot;
    c.prof_begin("bcast_mac", s, bytes, slot);
    bcast_mac_kernel<<<grid, 256, smem, s>>>(A, level, c.N, c.d_mod);
    c.prof_end(slot, s);
    c.st_launch++; c.st_bytes += bytes; c.st_ptmul += (uint64_t)A.nt * A.nu;
    CUDA_TRY(cudaGetLastError());
}

// ====================================================================================== lazy key switching helpers
namespace {
__global__ void lift_add_kernel(CopyBatch Dst, CopyBatch Src, int L, int N, const ModConst* __restrict__ mod,
                                const u64* __restrict__ pm, const u64* __restrict__ pm_sh) {
    const int r = blockIdx.y;
    u64* d = (u64*)Dst.src[r];
    const u64* s = Src.src[r];
    const size_t pairs = (size_t)L * N / 2;   // two words per thread, 128-bit accesses (N even, buffers 16-B aligned)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < pairs; i += (size_t)gridDim.x * blockDim.x) {
        const int limb = (int)(2 * i / N);
        const u64 q = mod[limb].q, f = pm[limb], fs = pm_sh[limb];
        ulonglong2 x = ((const ulonglong2*)d)[i];
        const ulonglong2 y = __ldg((const ulonglong2*)s + i);
        x.x = add_mod(x.x, mul_shoup(y.x, f, fs, q), q);
        x.y = add_mod(x.y, mul_shoup(y.y, f, fs, q), q);
        ((ulonglong2*)d)[i] = x;
    }
}
}  // namespace

void k_lift_add(encf_ctx& c, const CopyBatch& dst, const CopyBatch& src, int n, int L, const u64* pm, const u64* pm_sh,
                cudaStream_t s) {
    dim3 grid(nblocks((size_t)L * c.N / 2, TB, 256), n);
    { int _slot; c.prof_begin("lift_add_kernel", s, 0, _slot);
    lift_add_kernel<<<grid, TB, 0, s>>>(dst, src, L, c.N, c.d_mod, pm, pm_sh);
    c.prof_end(_slot, s); }
    c.st_launch++; c.st_bytes += (uint64_t)n * L * c.N * 8 * 3;
}

// ====================================================================================== conversion local maps (App. C)
namespace {
// [[m]]^(q)_b = (m'_b - party 2^{ell+sigma}) mod q_i, m'_b a 128-bit integer (lo, hi) per coefficient.
__global__ void ring2field_kernel(const u64* __restrict__ mp, u64* __restrict__ out, int L, int N, const ModConst* __restrict__ mod,
                                  R2F off) {
    const size_t total = (size_t)L * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int limb = (int)(i / N), k = (int)(i % N);
        const ModConst mc = mod[limb];
        U128 x{mp[2 * (size_t)k], mp[2 * (size_t)k + 1]};
        out[i] = sub_mod(barrett128(x, mc.q, mc.rhi, mc.rlo), off.v[limb], mc.q);
    }
}
__global__ void field2ring_kernel(const u64* __restrict__ sh, u64* __restrict__ out, int N, u64 mask) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) out[k] = sh[2 * (size_t)k] & mask;
}
}  // namespace

void k_ring2field(encf_ctx& c, const u64* mp, u64* out, int L, const R2F& off, cudaStream_t s) {
    { int _slot; c.prof_begin("ring2field_kernel", s, 0, _slot);
    ring2field_kernel<<<GRID((size_t)L * c.N), TB, 0, s>>>(mp, out, L, c.N, c.d_mod, off);
    c.prof_end(_slot, s); }
    c.st_launch++;
}

void k_field2ring(encf_ctx& c, const u64* sh, u64* out, int ell, cudaStream_t s) {
    const u64 mask = ell >= 64 ? ~0ull : ((1ull << ell) - 1);
    { int _slot; c.prof_begin("field2ring_kernel", s, 0, _slot);
    field2ring_kernel<<<GRID((size_t)c.N), TB, 0, s>>>(sh, out, c.N, mask);
    c.prof_end(_slot, s); }
    c.st_launch++;
}

void k_ks_group(encf_ctx& c, const KsGroupBatch& B, int ngrp, int dnum, int L, int key_nl, cudaStream_t s) {
    if (ngrp <= 0) return;
    const int K = c.Kof(L), nl = L + K;
    if ((unsigned __int128)dnum * c.max_mod >= ((unsigned __int128)1 << 64))
        throw EncfError(ENCF_ERR_ARG, "ks_group: dnum * q too large for one Montgomery reduction");
    const size_t sm = (size_t)2 * (3 * dnum + 1) * KT * 8 + 64;
    if (c.N < KT || sm > 227 * 1024) throw EncfError(ENCF_ERR_PLAN_SHAPE, "ks_group: unsupported shape");
    static bool attr = false;
    if (!attr) {
        CUDA_TRY(cudaFuncSetAttribute(ks_group_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr = true;
    }
    KeyLimb kl;
    LimbMap em;
    em.n = nl;
    for (int e = 0; e < nl; e++) {
        kl.kl[e] = e < L ? e : (key_nl - K) + (e - L);
        em.mod[e] = (unsigned char)(e < L ? e : c.L + (e - L));
    }
    const int nreq = B.start[ngrp];
    const uint64_t bytes = (uint64_t)nreq * ((uint64_t)dnum * nl * 3 + L) * c.N * 8 + (uint64_t)ngrp * (2 * nl + 2 * L) * c.N * 8;
    int slot;
    c.prof_begin("ks_inner", s, bytes, slot);
    ks_group_tma_kernel<<<dim3(c.N / KT, nl, ngrp), KG_NT, sm, s>>>(B, dnum, nl, L, key_nl, kl, em, c.N, c.logN, c.d_mod,
                                                                     c.moddown[L].d_pl, c.moddown[L].d_pl_sh);
    c.prof_end(slot, s);
    c.st_launch++; c.st_bytes += bytes; c.st_ks += nreq;
    CUDA_TRY(cudaGetLastError());
}
