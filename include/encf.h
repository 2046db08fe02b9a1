/*
 * encf.h -- C ABI of the EncFormer CKKS hot path on B200 (sm_100a).
 *
 * Implements the CKKS linear layers of EncFormer (arXiv 2604.09975): the SCP pt-ct projection
 * (P:253-304), the folded-diagonal score and value kernels
 * and the GPU half of the complex CKKS->MPC conversion (Alg 3, trimming P:863-878),
 * over RNS-CKKS with 64-bit words.
 *
 * CONVENTIONS (apply to every entry point)
 *  - Memory: every ciphertext / plaintext / key / weight buffer passed in is CALLER-OWNED DEVICE
 *    memory (cudaMalloc / torch), unless the argument is documented as "host".  The library owns
 *    only encf_ctx (tables, mask cache, statistics) and encf_keys (key limbs), plus stream-ordered
 *    scratch it allocates and frees internally (cudaMallocAsync on the caller's stream).
 *  - Layout ("interchange"): a ciphertext is [comp][limb][N] uint64 little-endian, limb i reduced
 *    mod q_i in [0, q_i); a plaintext is [limb][N].  Limbs are always the prefix q_0..q_{L-1}.
 *    `ntt` = 0 means coefficient domain (the interchange format), 1 means the library's private
 *    NTT domain (ordering private; convert with encf_poly_to_ntt / encf_poly_from_ntt).  All
 *    homomorphic entry points require ntt = 1 inputs and produce ntt = 1 outputs.
 *  - Streams: `stream` is a cudaStream_t passed as void*; all work is asynchronous on it.
 *  - Validation: argument, level and scale checks run on the host BEFORE any launch and return
 *    synchronously.  Launch errors are returned as ENCF_ERR_CUDA; asynchronous faults surface at
 *    the caller's next synchronisation (and in encf_last_error()).
 *  - Thread safety: a context may be used concurrently from several host threads on different
 *    streams (its tables are immutable after creation; the mask cache is mutex-protected).
 *  - Scales are tracked as doubles: ptmul/ctmul multiply them, rescale divides by q_last,
 *    add/sub require bit-identical scales (ENCF_ERR_SCALE_MISMATCH).
 */
#ifndef ENCF_H
#define ENCF_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ENCF_OK = 0,
    ENCF_ERR_ARG = 1,              /* null pointer, bad size, bad flag */
    ENCF_ERR_LENGTH_MISMATCH = 2,  /* slot vector longer than n */
    ENCF_ERR_SCALE_MISMATCH = 3,   /* add/sub of unequal scales */
    ENCF_ERR_LEVEL_MISMATCH = 4,   /* operands at different levels / level above the key's */
    ENCF_ERR_LEVEL_EXHAUSTED = 5,  /* rescale at one limb */
    ENCF_ERR_PLAN_SHAPE = 6,       /* plan dimensions inconsistent */
    ENCF_ERR_ODD_SEQ = 7,          /* folded-diagonal needs even m */
    ENCF_ERR_FORMAT = 8,           /* wrong component count / domain */
    ENCF_ERR_OVERFLOW = 9,         /* encode value too large */
    ENCF_ERR_CONFIG = 10,          /* L_conv violates P:874-876 */
    ENCF_ERR_MISSING_KEY = 11,     /* Galois / relin key not generated */
    ENCF_ERR_WORKSPACE = 12,
    ENCF_ERR_OOM = 13,
    ENCF_ERR_CUDA = 14
} encf_status;

typedef struct encf_ctx encf_ctx;
typedef struct encf_keys encf_keys;
typedef struct encf_proj_plan encf_proj_plan;
typedef struct encf_attn_plan encf_attn_plan;

/* Ciphertext: data -> [n_comp][n_limbs][N] device uint64. n_comp = 2 (or 3 before relinearisation). */
typedef struct { uint64_t* data; int32_t n_comp; int32_t n_limbs; double scale; int32_t ntt; } encf_ct;
/* Plaintext: data -> [n_limbs][N] device uint64. */
typedef struct { uint64_t* data; int32_t n_limbs; double scale; int32_t ntt; } encf_pt;

/* Parameter set (params/*.json): N a power of two in [2^4, 2^16]; q[0..L-1] body primes, p[0..K-1]
 * special primes, all < 2^61, = 1 mod 2N; alpha = limbs per key-switching digit (hybrid KS).
 * K_of_level (host [L], may be NULL): a key switch at level l extends by the first K_of_level[l-1] special primes
 * (non-decreasing, in [1, K]; DESIGN.md R-KL); NULL = all K at every level.  Extended-basis objects at level l
 * (partial projection accumulators, ext masks) have l + K_of_level[l-1] limbs.  Errors: ARG. */
typedef struct { int32_t N; int32_t L; int32_t K; int32_t alpha; const uint64_t* q; const uint64_t* p;
                 const int32_t* K_of_level; } encf_params;

/* Counters (SURVEY §5 "Tracing"): accumulated since context creation. */
typedef struct {
    uint64_t keyswitch;      /* ModDown pairs (each rotation / conj / relin is one) */
    uint64_t modup;          /* ModUp passes (a hoisted batch counts one) */
    uint64_t limb_ntt;       /* forward + inverse limb transforms launched */
    uint64_t ptmul_terms;    /* plaintext-ciphertext products (fused MAC terms included) */
    uint64_t ctmul;          /* ciphertext tensor products */
    uint64_t kernel_launches;
    uint64_t alg_bytes;      /* algorithmic HBM bytes of the launched kernels */
    uint64_t limb_ntt_fp64;  /* of limb_ntt: transforms of limbs whose modulus runs the FP64-pipe path (q < 2^41) */
} encf_counters;

/* ------------------------------------------------------------------------------------------ context */
/* Builds twiddle / base-conversion / rescale tables on `device`.  Errors: ARG (bad N / primes). */
encf_status encf_ctx_create(const encf_params* params, int device, encf_ctx** out);
encf_status encf_ctx_destroy(encf_ctx* ctx);
const char* encf_status_string(encf_status s);
const char* encf_last_error(void);                 /* thread-local detail of the last failure */
encf_status encf_stats(encf_ctx* ctx, encf_counters* out);
encf_status encf_stats_reset(encf_ctx* ctx);
/* Live kernel timing: while enabled, CUDA events are recorded on the launching stream around every
 * launch of the kernels named in `which` (comma-separated; "*" = every kernel; NULL disables).  Names: "diag_mac",
 * "ks_inner", "ntt" (one fwd/inv transform = a pair of launches) and the *_kernel launchers.
 * encf_profile_read synchronises on those events and returns the summed device time, the launch
 * count and the summed ALGORITHMIC bytes (DESIGN.md §Roofline, 0 where not defined) for `kernel`,
 * then forgets them.  encf_profile_peek returns the same without forgetting: for a stream CAPTURED into a
 * CUDA graph the events are graph nodes re-recorded at every replay, so a peek after each replay reads that
 * replay's launches.  Every entry point of the kernel path is capturable once a warm-up call has filled
 * the mask cache (request tables are then uploaded from a persistent pinned arena). */
encf_status encf_profile_enable(encf_ctx* ctx, const char* which);
encf_status encf_profile_read(encf_ctx* ctx, const char* kernel, double* total_ms, uint64_t* launches, uint64_t* alg_bytes);
encf_status encf_profile_peek(encf_ctx* ctx, const char* kernel, double* total_ms, uint64_t* launches, uint64_t* alg_bytes);

/* ------------------------------------------------------------------------------------------ keys (testing helpers) */
#define ENCF_KEY_RELIN 1u
/* Secret key s (ternary) and hybrid key-switching keys for the Galois elements galois[0..n-1]
 * (5^r mod 2N for a left rotation by r; 2N-1 for conj) and, with ENCF_KEY_RELIN, the
 * relinearisation key (s^2), all drawn from the counter PRNG with `seed`.
 * Keys cover levels <= max_level (limbs q_0..q_{max_level-1}, p_0..p_{K-1}). */
encf_status encf_keygen(encf_ctx* ctx, uint64_t seed, const uint32_t* galois /*host*/, int32_t n_galois,
                        uint32_t flags, int32_t max_level, encf_keys** out, void* stream);
encf_status encf_keys_destroy(encf_keys* keys);
/* Copy key material to device buffer `out` in COEFFICIENT form (interchange): which = 0: secret key
 * [max_level+K][N]; which = 1: ksk of `galois` (0 = relin) [dnum(max_level)][2][max_level+K][N]. */
encf_status encf_keys_export(encf_ctx* ctx, const encf_keys* keys, int32_t which, uint32_t galois,
                             uint64_t* out, void* stream);
encf_status encf_keys_size(encf_ctx* ctx, const encf_keys* keys, int32_t which, size_t* words);
uint32_t encf_galois_rot(encf_ctx* ctx, int32_t steps);   /* 5^(steps mod n) mod 2N */
uint32_t encf_galois_conj(encf_ctx* ctx);                  /* 2N - 1 */

/* Secret-key encryption (DESIGN G17): c1 = a uniform, c0 = -a s + e + m, randomness from `seed`.
 * pt and out may be either domain on input; out is produced in NTT form. */
encf_status encf_encrypt_sk(encf_ctx* ctx, const encf_keys* keys, const encf_pt* pt, uint64_t seed,
                            encf_ct* out, void* stream);
/* m = c0 + c1 s (+ c2 s^2); out->data receives [n_limbs][N] in NTT form. */
encf_status encf_decrypt(encf_ctx* ctx, const encf_keys* keys, const encf_ct* ct, encf_pt* out, void* stream);

/* Encode complex slots (host re/im, n_slots <= n) at `scale` into L limbs (NTT form):
 * m_k = round_half_even(scale (2/N) Re sum_j z_j zeta^{-5^j k}) computed in float64 on the GPU.
 * Errors: LENGTH_MISMATCH, OVERFLOW (|m_k| >= 2^62). */
encf_status encf_encode(encf_ctx* ctx, const double* re, const double* im, int32_t n_slots, int32_t n_limbs,
                        double scale, encf_pt* out, void* stream);
/* Decode (centred lift of limb 0 -- requires |coefficients| < q_0/2 -- then float64 FFT); host re/im [n]. */
encf_status encf_decode(encf_ctx* ctx, const encf_pt* pt, double* re, double* im, void* stream);

/* ------------------------------------------------------------------------------------------ primitives */
/* In-place domain conversion of n_polys consecutive [n_limbs][N] polynomials (limb i mod q_i). */
encf_status encf_poly_to_ntt(encf_ctx* ctx, uint64_t* data, int32_t n_polys, int32_t n_limbs, void* stream);
encf_status encf_poly_from_ntt(encf_ctx* ctx, uint64_t* data, int32_t n_polys, int32_t n_limbs, void* stream);

encf_status encf_add(encf_ctx* ctx, const encf_ct* a, const encf_ct* b, encf_ct* out, void* stream);
encf_status encf_sub(encf_ctx* ctx, const encf_ct* a, const encf_ct* b, encf_ct* out, void* stream);
encf_status encf_mul_i(encf_ctx* ctx, const encf_ct* a, encf_ct* out, void* stream);          /* x X^{N/2} = x i */
encf_status encf_ptmul(encf_ctx* ctx, const encf_ct* a, const encf_pt* w, encf_ct* out, void* stream);
encf_status encf_tensor(encf_ctx* ctx, const encf_ct* a, const encf_ct* b, encf_ct* out3, void* stream);
encf_status encf_relinearize(encf_ctx* ctx, const encf_keys* keys, const encf_ct* in3, encf_ct* out, void* stream);
/* Left rotation by steps[0] (single key switch: sigma_g then ModUp of sigma_g(c1)). n must be 1. */
encf_status encf_rotate(encf_ctx* ctx, const encf_keys* keys, const encf_ct* in, int32_t steps, encf_ct* out, void* stream);
/* Hoisted batch: ONE ModUp of c1, then sigma_g applied to the extended digits for each step (bits
 * differ from encf_rotate by design). outs[i] for steps[i]; steps = 0 mod n copies. */
encf_status encf_rotate_hoisted(encf_ctx* ctx, const encf_keys* keys, const encf_ct* in, const int32_t* steps /*host*/,
                                int32_t n, encf_ct* outs /*host array of n*/, void* stream);
encf_status encf_conjugate(encf_ctx* ctx, const encf_keys* keys, const encf_ct* in, encf_ct* out, void* stream);
/* Decomplexify (DESIGN G3): out[i] = in[i] + conj(in[i]) with scale 2 scale(in[i]) (the 1/2 of
 * (c + conj c)/2 is scale bookkeeping, no level).  n ciphertexts (host array, each 2 components, same level) in
 * one batched conjugation (the single-KS conj of encf_conjugate, bit for bit) + one batched add.  outs: host array
 * of n caller buffers at the input level.  Errors ARG (n < 1), LEVEL_MISMATCH (mixed levels), MISSING_KEY. */
encf_status encf_decomplexify(encf_ctx* ctx, const encf_keys* keys, const encf_ct* in /*host array of n*/, int32_t n,
                              encf_ct* outs /*host array of n*/, void* stream);
/* Divide-and-round by q_{L-1} (SEAL style, C5); out has n_limbs - 1 limbs.  Error LEVEL_EXHAUSTED. */
encf_status encf_rescale(encf_ctx* ctx, const encf_ct* in, encf_ct* out, void* stream);
/* ModSwitchToNext repeated: keep the first n_limbs limbs, scale unchanged. */
encf_status encf_mod_drop(encf_ctx* ctx, const encf_ct* in, int32_t n_limbs, encf_ct* out, void* stream);
/* Boundary wrapper: re + i im. */
encf_status encf_complexify(encf_ctx* ctx, const encf_ct* re, const encf_ct* im, encf_ct* out, void* stream);
/* Batched encf_complexify: out[i] = re[i] + i im[i] (X^{N/2} im[i]) for n pairs (host arrays of n), every input at one
 * level and component count, in ceil(n / 32) launches; the same words as n encf_complexify calls.  Errors: ARG,
 * LEVEL_MISMATCH, SCALE_MISMATCH. */
encf_status encf_complexify_many(encf_ctx* ctx, const encf_ct* re /*host array of n*/, const encf_ct* im /*host array of n*/,
                                 int32_t n, encf_ct* out /*host array of n*/, void* stream);

/* Mask plaintexts (Alg A.2 H/U, App. A.3 e_s / n_u, export ranges): ones on rows [r0,r1) of segments
 * s0 + k*sstride (k < scount) of an m-row segment grid, encoded at scale q_{L-1} at level L.
 * The context caches them; encf_mask_put installs an externally encoded plaintext (host coefficient
 * form [L][N]) for a descriptor -- used by the parity tests to feed the oracle's encodings.  Installing a mask drops
 * the caches derived from it (pre-masked keys of that descriptor, the value kernel's mask spectra); encf_mask_clear
 * drops every mask and every derived cache.  All of them are context-owned device memory. */
typedef struct { int32_t m, r0, r1, s0, sstride, scount, level, ext; } encf_mask_desc;   /* ext = 1: [level + K][N], also reduced mod the special primes (lazy key switching, DESIGN R-LAZY) */
encf_status encf_mask_put(encf_ctx* ctx, const encf_mask_desc* desc, const uint64_t* coeffs /*host [L][N]*/);
encf_status encf_mask_clear(encf_ctx* ctx);

/* ------------------------------------------------------------------------------------------ EncFormer kernels */
#define ENCF_PROJ_DECOMPLEXIFY 1u
/* Fused-QK mode: the G input groups are REAL ciphertexts (U = G, no complexification) and the
 * weights are complex, W~ = Wre + i Wim (e.g. W_Q^pi_S + i W_K^pi_S); the output is Y = X Wre + i X Wim (no
 * decomplexify; incompatible with ENCF_PROJ_DECOMPLEXIFY, G1). */
#define ENCF_PROJ_REAL_INPUT 4u
/* Projection plan: n/m segments, C active (C = 0 -> n/m), N1 | C (0 -> default).  C < n/m makes the
 * plan RESTRICTED: the baby bank is Phi_C^q (RotFirst_{Cm}, Alg A.4) and the giant fold Phi_C^{pN1}, each spending a
 * level, so the weights are encoded at level L - 1 (the bank level) and y_b lands at level L - 3 instead of L - 1
 * (DESIGN.md R-PHIC).  Errors: PLAN_SHAPE (C > n/m, N1 not dividing C, fused-QK with DECOMPLEXIFY). */
encf_status encf_proj_plan_create(encf_ctx* ctx, int32_t m, int32_t d_in, int32_t d_out, int32_t C, int32_t N1,
                                  uint32_t flags, encf_proj_plan** out);
encf_status encf_proj_plan_destroy(encf_proj_plan* plan);
/* Plan shape: out[0..6] = {C, G, U, B_out, N1, N2, n_plaintexts = B_out*N2*U*N1}. */
encf_status encf_proj_plan_info(const encf_proj_plan* plan, int32_t* out7);
/* Galois elements the projection needs (baby q*m, giant p*N1*m, conj): writes up to cap, returns count in *n. */
encf_status encf_proj_galois(encf_ctx* ctx, const encf_proj_plan* plan, uint32_t* out, int32_t cap, int32_t* n);
/* Encode the pre-permuted weight matrix Wbar (host, row-major d_in x d_out doubles) into the
 * diagonal stream w~^(b)_{u,p,q} at level n_limbs, scale q_{n_limbs-1}, NTT form,
 * layout [b][p][u][q][limb][N] (encf_proj_weights_size bytes). */
encf_status encf_proj_weights_size(const encf_proj_plan* plan, int32_t n_limbs, size_t* bytes);
encf_status encf_proj_encode_weights(encf_ctx* ctx, const encf_proj_plan* plan, const double* Wbar /*host*/,
                                     int32_t n_limbs, uint64_t* w_out, void* stream);
/* Real-input plans: w~_{b,p,g,q}(c) = Wre[gC + alpha, bC + beta] + i Wim[gC + alpha, bC + beta] (Wim may be NULL). */
encf_status encf_proj_encode_weights_complex(encf_ctx* ctx, const encf_proj_plan* plan, const double* Wre /*host*/,
                                             const double* Wim /*host or NULL*/, int32_t n_limbs, uint64_t* w_out, void* stream);
/* Y = X W (C6): x[U] complexified inputs (NTT, level L); w_pt the weight stream (NTT form, layout
 * above, level L, scale w_scale).  Units (b,p) in [unit_begin, unit_end) (row-major over b, p).
 * With the full unit range and ENCF_PROJ_FINALIZE, y[b] = rescale(acc_b + conj(acc_b)) (B_out
 * outputs, level L-1).  Without FINALIZE, y[b] receives the partial giant-step sums acc_b of the
 * touched b in the EXTENDED basis Q_L u P (n_limbs = L + K; the giant-step rotations are summed without ModDown,
 * DESIGN.md R-LAZY) for a cross-rank uint64 SUM + encf_mod_reduce_ext, then encf_pt_ct_matmul_finalize. */
#define ENCF_PROJ_FINALIZE 2u
/* w_pt holds only the units [unit_begin, unit_end) (a rank's shard of the weight stream: each GPU keeps
 * 1/world of the plaintext diagonals); without it w_pt is the whole stream and unit u starts at u * U N1 L_w N. */
#define ENCF_PROJ_W_SHARD 8u
encf_status encf_pt_ct_matmul(encf_ctx* ctx, const encf_keys* keys, const encf_proj_plan* plan,
                              const encf_ct* x /*host array [U]*/, const uint64_t* w_pt, double w_scale,
                              int32_t unit_begin, int32_t unit_end, uint32_t flags,
                              encf_ct* y /*host array [B_out]*/, void* stream);
encf_status encf_pt_ct_matmul_finalize(encf_ctx* ctx, const encf_keys* keys, const encf_proj_plan* plan,
                                       const encf_ct* acc, int32_t b_begin, int32_t b_end, encf_ct* y, void* stream);

/* Attention plan: score (C_qk used segments per block, H <= C_qk <= n/m, beta | m with m/beta even) and value
 * (H_blk heads per block).  Errors: ODD_SEQ (odd m), PLAN_SHAPE. */
encf_status encf_attn_plan_create(encf_ctx* ctx, int32_t m, int32_t H, int32_t d_h, int32_t C_qk, int32_t beta,
                                  int32_t H_blk, encf_attn_plan** out);
encf_status encf_attn_plan_destroy(encf_attn_plan* plan);
/* out[0..7] = {B, beta, g, n_out (=K_min(S)), H_blk, B_V, seg_stride, C_qk} */
encf_status encf_attn_plan_info(const encf_attn_plan* plan, int32_t* out8);
encf_status encf_attn_galois(encf_ctx* ctx, const encf_attn_plan* plan, uint32_t* out, int32_t cap, int32_t* n);
/* Score kernel (C7): q[B], k[B] at level L -> s_t[t] for t in [t_begin, t_end), level L-3.  When
 * C_qk mod H != 0 the blocks carry head phases r_l = l C_qk mod H: the lazy tensor sums are formed per
 * phase, routed, aligned by Align_r = RotFirst_{Hm}(., (H - r) m) and summed (one extra level: s_t at L-4). */
encf_status encf_ct_ct_attn_score(encf_ctx* ctx, const encf_keys* keys, const encf_attn_plan* plan,
                                  const encf_ct* q, const encf_ct* k, int32_t t_begin, int32_t t_end,
                                  encf_ct* s_t, void* stream);
/* Minimal export stream (App. A.3): s_t[m/2] -> s_min[K_min(S)] at level L-1 of s_t. */
encf_status encf_attn_export_stream(encf_ctx* ctx, const encf_keys* keys, const encf_attn_plan* plan,
                                    const encf_ct* s_t, encf_ct* s_min, void* stream);
/* Value kernel (C8): p_fd[B_V] (level Lp >= 3), v[B_V] (level Lv >= Lp + 1) -> o[B_V] at
 * level Lp - 2.  Step 4's Phi-broadcast b_t = sum_u Phi^{t-u}(p) (.) n_u runs as negacyclic 128-point convolutions
 * along the window (exact); the first call per (mask set, level) caches the masks' spectra in the context
 * (128 L N words, outside CUDA-graph capture like the masks).  Errors: LEVEL_MISMATCH (level plan), MISSING_KEY. */
encf_status encf_ct_ct_attn_value(encf_ctx* ctx, const encf_keys* keys, const encf_attn_plan* plan,
                                  const encf_ct* p_fd, const encf_ct* v, encf_ct* o, void* stream);
/* Sharded value kernel: units (l, t), flattened l (m/2) + t, in [unit_begin, unit_end).  For every
 * block l the range touches (in increasing l) o3[i] receives the UNRELINEARISED partial sum_{t in range} u_t (x) b_t
 * (3 components, level Lp - 1, caller buffers of 3 (Lp - 1) N words).  Partials of one block from several ranks are
 * summed as uint64 (world_size q < 2^64) + encf_mod_reduce, then encf_attn_value_finalize gives exactly the bits of
 * encf_ct_ct_attn_value.  Errors as encf_ct_ct_attn_value, plus ARG (bad range). */
encf_status encf_ct_ct_attn_value_partial(encf_ctx* ctx, const encf_keys* keys, const encf_attn_plan* plan,
                                          const encf_ct* p_fd, const encf_ct* v, int32_t unit_begin, int32_t unit_end,
                                          encf_ct* o3, void* stream);
/* o[i] = rescale(relin(o3[i])) rounded once (R-RELRS) for n complete 3-component value partials at one level. */
encf_status encf_attn_value_finalize(encf_ctx* ctx, const encf_keys* keys, const encf_ct* o3, int32_t n, encf_ct* o,
                                     void* stream);

/* ------------------------------------------------------------------------------------------ ciphertext shifts (App. A.1) */
/* RotFirst_L(x; tau) for every tau in taus[0..n-1] (Alg A.3; G21: slots >= L come out zero):
 * tau <- tau mod L, rot(x; tau) (.) a_{L,tau} + rot(x; tau - L) (.) b_{L,tau} with a = 1{i < L - tau},
 * b = 1{L - tau <= i < L}, then rescale (masks at scale q_{L-1}); tau = 0 is x (.) a_{L,0}.  One hoisted ModUp,
 * the rotations kept in Q_L u P and divided by P q_{L-1} at once (DESIGN.md R-LAZY).  Phi_C^Delta (Alg A.4) is
 * L = C m, tau = (Delta mod C) m; Align_r is L = H m, tau = (H - r) m.  m: the segment grid used for
 * the mask descriptors of segment-aligned ranges (other ranges use the 1-slot grid).  outs: n caller buffers,
 * level L_in - 1.  Keys: left rotations tau and tau - L.  Errors: ARG, LEVEL_EXHAUSTED, MISSING_KEY. */
encf_status encf_rotfirst(encf_ctx* ctx, const encf_keys* keys, const encf_ct* in, int32_t L_slots, const int32_t* taus /*host*/,
                          int32_t n, int32_t m, encf_ct* outs /*host array of n*/, void* stream);
/* Psi^t(x) for every t in ts[0..n-1] (Alg A.2): rot(x; t) (.) h_t + rot(x; t - m) (.) u_t, rescale;
 * t = 0 mod m is x (.) h_0 (DESIGN.md R-PSI0).  Same conventions as encf_rotfirst; m must divide n. */
encf_status encf_psi(encf_ctx* ctx, const encf_keys* keys, const encf_ct* in, int32_t m, const int32_t* ts /*host*/, int32_t n,
                     encf_ct* outs /*host array of n*/, void* stream);

/* ------------------------------------------------------------------------------------------ export (Alg 3, GPU half) */
/* L_conv rule: smallest L with log2 Q_L >= ell + sigma + 1 and Q_L / 2 > scale * B_max.
 * Error CONFIG if none. */
encf_status encf_l_conv(encf_ctx* ctx, int32_t ell, int32_t sigma, double scale, double B_max, int32_t* L_conv);
/* Mod-drop `in` to L_conv, convert to coefficient form, draw r^ uniform mod q_i (PRNG stream
 * mask(stream_id)), masked = (c0 + r^, c1) [coefficient form, to P0], server_share = -r^ mod q_i
 * [L_conv][N].  masked->data must hold 2*L_conv*N words. */
encf_status encf_export_c2m(encf_ctx* ctx, const encf_ct* in, int32_t L_conv, uint64_t mask_seed, uint64_t stream_id,
                            encf_ct* masked, uint64_t* server_share, void* stream);
/* Batched export (the same steps as encf_export_c2m for each of n ciphertexts of one level): ciphertext i uses
 * stream id stream_id0 + i.  masked: device [n][2][L_conv][N] (coefficient form, caller-owned), shares: device
 * [n][L_conv][N].  One inverse-NTT launch pair for all 2n polynomials.  Errors as encf_export_c2m, plus
 * LEVEL_MISMATCH when the inputs' levels differ. */
encf_status encf_export_c2m_many(encf_ctx* ctx, const encf_ct* in /*host array of n*/, int32_t n, int32_t L_conv,
                                 uint64_t mask_seed, uint64_t stream_id0, uint64_t* masked, uint64_t* shares,
                                 void* stream);
/* encf_export_c2m_many with (mask_seed, stream_id0) read from DEVICE memory d_seed_sid [2] when the kernels run:
 * ciphertext i uses seed d_seed_sid[0] and stream id (d_seed_sid[1] + i) mod 2^56.  A step captured into a CUDA
 * graph that advances d_seed_sid[1] every replay draws fresh masks r^ per inference (a replayed constant seed would
 * reuse the one-time pad: the difference of two masked exports would leak the difference of the messages). */
encf_status encf_export_c2m_many_dev(encf_ctx* ctx, const encf_ct* in /*host array of n*/, int32_t n, int32_t L_conv,
                                     const uint64_t* d_seed_sid /*device [2]*/, uint64_t* masked, uint64_t* shares,
                                     void* stream);
/* ------------------------------------------------------------------------------------------ import (Alg 4, GPU half) */
/* Ring2Field local map (App. C): after Pi_Ext, party b holds m'_b in [0, 2^{ell+sigma}) per
 * coefficient (device [N] little-endian (lo, hi) 64-bit pairs) with m'_0 + m'_1 = 2^{ell+sigma} + cl(m);
 * out[i][k] = m'_0 mod q_i (party 0) or (m'_1 - 2^{ell+sigma}) mod q_i (party 1), i < L (coefficient form). */
encf_status encf_ring2field_local(encf_ctx* ctx, const uint64_t* mprime, int32_t party, int32_t ell_sigma, int32_t L,
                                  uint64_t* out, void* stream);
/* Field2Ring local map (App. C): after the lift to Z_{2^ell'} (device [N] (lo, hi) pairs), each
 * party reduces its share mod 2^ell (ell <= 64): out[k] = lo & (2^ell - 1). */
encf_status encf_field2ring_local(encf_ctx* ctx, const uint64_t* share, int32_t ell, uint64_t* out, void* stream);
/* Alg 4 step 4: P1 outputs <m> = <c> + [[t^]]_1 (c from P0, NTT form; share: plaintext over Q_L in
 * either domain). */
encf_status encf_import_m2c(encf_ctx* ctx, const encf_ct* c, const encf_pt* share, encf_ct* out, void* stream);
/* ------------------------------------------------------------------------------------------ w/o-SCP ablation */
/* Halevi-Shoup rotation-mask-accumulate repack (App. G), used only by the w/o-SCP ablation:
 * out[i] = sum_{k < log2 m} Rot(x[i], 2^k) (.) m_k with m_k = rows [round(k m / log2 m), round((k+1) m / log2 m))
 * of every m-slot segment (DESIGN.md R-RMA), i.e. slot s m + j receives slot s m + j + 2^{k(j)}.  One hoisted
 * ModUp per input, one fused masked inner-product launch, one merged ModDown + rescale: out at level L - 1.
 * Keys: left rotations by 2^k, k < log2 m.  Errors: ARG, PLAN_SHAPE (m not a power of two), LEVEL_EXHAUSTED,
 * LEVEL_MISMATCH, MISSING_KEY. */
encf_status encf_repack_rma(encf_ctx* ctx, const encf_keys* keys, const encf_ct* x, int32_t n, int32_t m, encf_ct* out,
                            void* stream);
/* ------------------------------------------------------------------------------------------ GELU pre-evaluation */
/* Alg 5 steps 1-3, the CKKS half of secure GELU: for each complex x[i] = x^(0) + i x^(1) (level L >= 4,
 * all inputs at one level and scale): x^(0) = (x + conj x)/2, x^(1) = (x - conj x)/(2i) (the 1/2 as scale x 2,
 * G3); per channel x^2, x^3, x^4 (tensor + relin + rescale each) and the Eq. B.2 candidates
 * F0 = a x^4 - b x^3 + c x^2 + (0.5 - d) x + e, F1 = a x^4 + b x^3 + c x^2 + (0.5 + d) x + e with the public
 * coef = {a, b, c, d, e} applied as integers round_half_even(coef * Delta) (DESIGN.md R-GELU);
 * f0[i] = F0^(0) + i F0^(1), f1[i] = F1^(0) + i F1^(1) at level L - 3 (caller buffers, 2 components).
 * Keys: conj + relin.  Errors: ARG, LEVEL_EXHAUSTED (L < 4), LEVEL_MISMATCH / SCALE_MISMATCH (mixed inputs),
 * MISSING_KEY. */
encf_status encf_gelu_preeval(encf_ctx* ctx, const encf_keys* keys, const encf_ct* x, int32_t n, const double* coef,
                              encf_ct* f0, encf_ct* f1, void* stream);

/* After a cross-rank uint64 SUM (C2): reduce n_polys x [n_limbs][N] words mod q_i in place.
 * Valid while the summed value fits in 64 bits (world_size * q < 2^64). */
encf_status encf_mod_reduce(encf_ctx* ctx, uint64_t* data, int32_t n_polys, int32_t n_limbs, void* stream);
/* Same for polynomials over the extended basis [q_0..q_{L-1}, p_0..p_{K-1}] (the partial projection
 * accumulators, which are exchanged across ranks in that basis so the sharded result is bit-identical). */
encf_status encf_mod_reduce_ext(encf_ctx* ctx, uint64_t* data, int32_t n_polys, int32_t L, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ENCF_H */
