/*
 * oracle.c -- plain, slow CPU primitives of the CKKS oracle (EncFormer, arXiv 2604.09975).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library.  It shares no code with the CUDA library
 * (paper_2604_09975_b200/csrc): its own modular arithmetic (every product is
 * (unsigned __int128)a*b % q), its own NTT (textbook iterative Cooley-Tukey in natural order),
 * its own automorphism (coefficient domain, by definition), its own PRNG implementation.
 *
 * Every routine follows a definition written in SURVEY.md §8c (C1-C5), which restates the paper:
 *   ring Z_q[X]/(X^N+1) and RNS, rotations/conj,
 *   rescale / ModSwitchToNext.
 * Where the paper is silent (key switching, sampling, PRNG) the readings are listed in DESIGN.md.
 * OpenMP is used only across independent limbs.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned __int128 u128;

static inline u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static inline u64 addmod(u64 a, u64 b, u64 q) { u128 s = (u128)a + b; return (u64)(s % q); }
static inline u64 submod(u64 a, u64 b, u64 q) { a %= q; b %= q; return a >= b ? a - b : a + (q - b); }

u64 o_mulmod(u64 a, u64 b, u64 q) { return mulmod(a, b, q); }

u64 o_powmod(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod(r, a, q);
        a = mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}

/* q prime: a^{-1} = a^{q-2} (Fermat). */
u64 o_invmod(u64 a, u64 q) { return o_powmod(a, q - 2, q); }

/* ---------------------------------------------------------------- ring product (C1) */

/* Definition of multiplication in Z_q[X]/(X^N+1):
 *   c_k = sum_{i+j=k} a_i b_j  -  sum_{i+j=k+N} a_i b_j   (mod q). */
void o_negacyclic_schoolbook(u64 q, i64 N, const u64* a, const u64* b, u64* c) {
    for (i64 k = 0; k < N; k++) {
        u64 acc = 0;
        for (i64 i = 0; i < N; i++) {
            i64 j = k - i;
            if (j >= 0) acc = addmod(acc, mulmod(a[i], b[j], q), q);
            else        acc = submod(acc, mulmod(a[i], b[j + N], q), q);
        }
        c[k] = acc;
    }
}

static void bitrev_permute(u64* a, i64 N) {
    for (i64 i = 1, j = 0; i < N; i++) {
        i64 bit = N >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) { u64 t = a[i]; a[i] = a[j]; a[j] = t; }
    }
}

/* Cyclic DFT A_j = sum_i a_i w^{ij} (w a primitive N-th root), iterative radix-2 Cooley-Tukey. */
static void cyclic_dft(u64 q, u64 w, i64 N, u64* a) {
    bitrev_permute(a, N);
    for (i64 len = 2; len <= N; len <<= 1) {
        u64 wlen = o_powmod(w, (u64)(N / len), q);
        for (i64 i = 0; i < N; i += len) {
            u64 t = 1;
            for (i64 j = 0; j < len / 2; j++) {
                u64 u = a[i + j];
                u64 v = mulmod(a[i + j + len / 2], t, q);
                a[i + j] = addmod(u, v, q);
                a[i + j + len / 2] = submod(u, v, q);
                t = mulmod(t, wlen, q);
            }
        }
    }
}

/* Oracle NTT (natural order): a_j <- a(psi^{2j+1}) = sum_i a_i psi^{i(2j+1)}, psi a primitive
 * 2N-th root of unity mod q.  Realised as the twist a_i*psi^i followed by a cyclic DFT with psi^2. */
void o_ntt_fwd(u64 q, u64 psi, i64 N, u64* a) {
    u64 t = 1;
    for (i64 i = 0; i < N; i++) { a[i] = mulmod(a[i], t, q); t = mulmod(t, psi, q); }
    cyclic_dft(q, mulmod(psi, psi, q), N, a);
}

/* Inverse of o_ntt_fwd: inverse cyclic DFT, times N^{-1}, untwist by psi^{-i}. */
void o_ntt_inv(u64 q, u64 psi, i64 N, u64* a) {
    u64 psi_inv = o_invmod(psi, q);
    cyclic_dft(q, mulmod(psi_inv, psi_inv, q), N, a);
    u64 n_inv = o_invmod((u64)N % q, q);
    u64 t = n_inv;
    for (i64 i = 0; i < N; i++) { a[i] = mulmod(a[i], t, q); t = mulmod(t, psi_inv, q); }
}

void o_ntt_fwd_batch(i64 nl, const u64* qs, const u64* psis, i64 N, u64* data) {
    #pragma omp parallel for schedule(dynamic)
    for (i64 l = 0; l < nl; l++) o_ntt_fwd(qs[l], psis[l], N, data + l * N);
}

void o_ntt_inv_batch(i64 nl, const u64* qs, const u64* psis, i64 N, u64* data) {
    #pragma omp parallel for schedule(dynamic)
    for (i64 l = 0; l < nl; l++) o_ntt_inv(qs[l], psis[l], N, data + l * N);
}

/* ---------------------------------------------------------------- pointwise (per limb) */

void o_add_batch(i64 nl, const u64* qs, i64 N, const u64* a, const u64* b, u64* out) {
    #pragma omp parallel for
    for (i64 l = 0; l < nl; l++)
        for (i64 k = 0; k < N; k++) out[l * N + k] = addmod(a[l * N + k], b[l * N + k], qs[l]);
}

void o_sub_batch(i64 nl, const u64* qs, i64 N, const u64* a, const u64* b, u64* out) {
    #pragma omp parallel for
    for (i64 l = 0; l < nl; l++)
        for (i64 k = 0; k < N; k++) out[l * N + k] = submod(a[l * N + k], b[l * N + k], qs[l]);
}

void o_mul_batch(i64 nl, const u64* qs, i64 N, const u64* a, const u64* b, u64* out) {
    #pragma omp parallel for
    for (i64 l = 0; l < nl; l++)
        for (i64 k = 0; k < N; k++) out[l * N + k] = mulmod(a[l * N + k], b[l * N + k], qs[l]);
}

/* acc += a*b (mod q), pointwise */
void o_mac_batch(i64 nl, const u64* qs, i64 N, const u64* a, const u64* b, u64* acc) {
    #pragma omp parallel for
    for (i64 l = 0; l < nl; l++)
        for (i64 k = 0; k < N; k++)
            acc[l * N + k] = addmod(acc[l * N + k], mulmod(a[l * N + k], b[l * N + k], qs[l]), qs[l]);
}

/* out = a * s_l (one scalar per limb) */
void o_mul_scalar_batch(i64 nl, const u64* qs, i64 N, const u64* a, const u64* scal, u64* out) {
    #pragma omp parallel for
    for (i64 l = 0; l < nl; l++)
        for (i64 k = 0; k < N; k++) out[l * N + k] = mulmod(a[l * N + k], scal[l] % qs[l], qs[l]);
}

/* Signed integers (|v| < 2^63) into residues per limb. */
void o_from_signed_batch(i64 nl, const u64* qs, i64 N, const i64* v, u64* out) {
    for (i64 l = 0; l < nl; l++)
        for (i64 k = 0; k < N; k++) {
            i64 x = v[k];
            u64 r = (u64)(x < 0 ? -x : x) % qs[l];
            out[l * N + k] = (x < 0 && r) ? qs[l] - r : r;
        }
}

/* ---------------------------------------------------------------- automorphism (C2) */

/* sigma_g : X^k -> X^{k g mod 2N} with X^N = -1, i.e. out[kg mod N] = (+/-) a_k,
 * negated when (k g mod 2N) >= N.  g must be odd.  Coefficient domain, by definition. */
void o_automorph_batch(i64 nl, const u64* qs, i64 N, u64 g, const u64* in, u64* out) {
    u64 two_n = 2 * (u64)N;
    #pragma omp parallel for
    for (i64 l = 0; l < nl; l++)
        for (i64 k = 0; k < N; k++) {
            u64 e = (u64)(((u128)(u64)k * g) % two_n);
            u64 v = in[l * N + k];
            if (e < (u64)N) out[l * N + e] = v;
            else            out[l * N + (e - N)] = v ? qs[l] - v : 0;
        }
}

/* ---------------------------------------------------------------- fast base conversion (C4) */

/* y_t[k] = sum_{i<n_in} [ x_i[k] * vfac_i ]_{q_i} * wfac[i*n_out + t]   (mod t)
 * with vfac_i = (Q'/q_i)^{-1} mod q_i and wfac = (Q'/q_i) mod t computed by the caller (explicit
 * big-integer arithmetic in Python).  No correction term: the result is x + u*Q' with 0 <= u < n_in. */
void o_bconv(i64 N, i64 n_in, const u64* qin, const u64* in, const u64* vfac,
             i64 n_out, const u64* qout, const u64* wfac, u64* out) {
    #pragma omp parallel for
    for (i64 t = 0; t < n_out; t++) {
        u64 qt = qout[t];
        for (i64 k = 0; k < N; k++) {
            u64 acc = 0;
            for (i64 i = 0; i < n_in; i++) {
                u64 v = mulmod(in[i * N + k], vfac[i], qin[i]);
                acc = addmod(acc, mulmod(v, wfac[i * n_out + t] % qt, qt), qt);
            }
            out[t * N + k] = acc;
        }
    }
}

/* Rounded fast base conversion (ModDown with the rounding correction, DESIGN.md R-MODDOWN):
 *   v_i = [x_i * vfac_i]_{q_i};  f_i = floor((v_i << s_i) * cfix_i / 2^64), s_i = 63 - bitlen(q_i),
 *   cfix_i = floor(2^(123 - s_i) / q_i)  (a 59-bit fixed-point estimate of v_i / q_i for any q_i < 2^63);
 *   r = (sum_i f_i + 2^58) >> 59  = round(sum_i v_i / q_i) up to 2^-56;
 *   y_t = sum_i v_i * wfac[i][t] - r * qprod[t]  (mod t),  qprod[t] = Q' mod t.
 * y is the CENTRED residue of x mod Q', so (b - y) / P is round(b / P). */
void o_bconv_round(i64 N, i64 n_in, const u64* qin, const u64* in, const u64* vfac,
                   i64 n_out, const u64* qout, const u64* wfac, const u64* qprod, const u64* cfix, const u64* csh,
                   u64* out) {
    #pragma omp parallel for
    for (i64 t = 0; t < n_out; t++) {
        u64 qt = qout[t];
        for (i64 k = 0; k < N; k++) {
            u64 acc = 0, fsum = 0;
            for (i64 i = 0; i < n_in; i++) {
                u64 v = mulmod(in[i * N + k], vfac[i], qin[i]);
                fsum += (u64)(((u128)(v << csh[i]) * cfix[i]) >> 64);
                acc = addmod(acc, mulmod(v, wfac[i * n_out + t] % qt, qt), qt);
            }
            u64 r = (fsum + (1ULL << 58)) >> 59;
            out[t * N + k] = submod(acc, mulmod(r % qt, qprod[t] % qt, qt), qt);
        }
    }
}

/* ---------------------------------------------------------------- rescale (C5) */

/* SEAL-style divide-and-round by the last prime q_L (coefficient domain):
 *   h = floor(q_L/2);  l' = (c_L + h) mod q_L;
 *   c'_i = (c_i - ((l' mod q_i) - (h mod q_i))) * q_L^{-1}  mod q_i   for i < L.
 * nl = number of input limbs (the last one is dropped). */
void o_rescale(i64 nl, const u64* qs, i64 N, const u64* in, u64* out) {
    u64 qL = qs[nl - 1];
    u64 h = qL / 2;
    const u64* cL = in + (nl - 1) * N;
    #pragma omp parallel for
    for (i64 i = 0; i < nl - 1; i++) {
        u64 qi = qs[i];
        u64 inv = o_invmod(qL % qi, qi);
        for (i64 k = 0; k < N; k++) {
            u64 lp = addmod(cL[k], h, qL);
            u64 corr = submod(lp % qi, h % qi, qi);
            out[i * N + k] = mulmod(submod(in[i * N + k], corr, qi), inv, qi);
        }
    }
}

/* ---------------------------------------------------------------- PRNG and sampling (C3) */

/* Counter-based generator:
 *   draw(seed, stream, index) = mix64( (seed ^ stream*0xD1B54A32D192ED03) + (index+1)*0x9E3779B97F4A7C15 )
 * with mix64 the SplitMix64 finaliser. */
u64 o_prng_draw(u64 seed, u64 stream, u64 index) {
    u64 z = (seed ^ (stream * 0xD1B54A32D192ED03ULL)) + (index + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Uniform mod q for limb with global id gid:  ((hi*2^64 + lo) * q) >> 128,
 * hi = draw(2*(gid*N+k)), lo = draw(2*(gid*N+k)+1). */
void o_sample_uniform(u64 seed, u64 stream, i64 nl, const u64* qs, const i64* gids, i64 N, u64* out) {
    #pragma omp parallel for
    for (i64 l = 0; l < nl; l++)
        for (i64 k = 0; k < N; k++) {
            u64 idx = 2 * ((u64)gids[l] * (u64)N + (u64)k);
            u64 hi = o_prng_draw(seed, stream, idx), lo = o_prng_draw(seed, stream, idx + 1);
            /* (hi*2^64 + lo) * q >> 128 = hi*q + (lo*q >> 64), high word */
            u128 a = (u128)hi * qs[l];
            u128 b = ((u128)lo * qs[l]) >> 64;
            out[l * N + k] = (u64)((a + b) >> 64);
        }
}

/* Ternary: mulhi(u, 3) - 1 in {-1, 0, 1}. */
void o_sample_ternary(u64 seed, u64 stream, i64 N, i64* out) {
    for (i64 k = 0; k < N; k++) {
        u64 u = o_prng_draw(seed, stream, (u64)k);
        out[k] = (i64)(((u128)u * 3) >> 64) - 1;
    }
}

/* Centred binomial eta=21: popcount(u & (2^21-1)) - popcount((u>>21) & (2^21-1)). */
void o_sample_cbd21(u64 seed, u64 stream, i64 N, i64* out) {
    for (i64 k = 0; k < N; k++) {
        u64 u = o_prng_draw(seed, stream, (u64)k);
        out[k] = (i64)__builtin_popcountll(u & 0x1FFFFFULL) - (i64)__builtin_popcountll((u >> 21) & 0x1FFFFFULL);
    }
}
