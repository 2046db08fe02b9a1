// ctx.cuh -- library context (tables built once per parameter set) and internal launcher API.
#pragma once
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "../../include/encf.h"

struct Status {
    encf_status code;
    std::string msg;
};

void set_last_error(const std::string& s);

#define CUDA_TRY(x)                                                                        \
    do {                                                                                   \
        cudaError_t _e = (x);                                                              \
        if (_e != cudaSuccess) {                                                           \
            set_last_error(std::string(#x) + ": " + cudaGetErrorString(_e));               \
            throw EncfError(ENCF_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e)); \
        }                                                                                  \
    } while (0)

struct EncfError {
    encf_status code;
    std::string msg;
    EncfError(encf_status c, const std::string& m) : code(c), msg(m) {}
};

// A batch of limb polynomials: limb l of poly p lives at base + p*poly_stride + l*N, mod map.mod[l].
struct PolyBatch {
    u64* base;
    i64 poly_stride;
    int npolys;
    LimbMap map;
};

struct NttPostTab { u64* f = nullptr; u64* fsh = nullptr; double* fd = nullptr; };   // per-limb iNTT output factors

struct ModUpTab {         // fast BConv of digit j at level L: digit limbs [lo,hi) -> targets
    int lo, hi;
    LimbMap tgt;          // target modulus ids
    std::vector<int> tgt_pos;   // position of each target inside the extended [Q_L | P] layout
    u64* d_vfac;          // [alpha]      (Q_j/q_i)^{-1} mod q_i
    u64* d_vfac_sh;
    u64* d_wfac;          // [alpha][ntgt] (Q_j/q_i) mod t
    uint8_t* d_wb = nullptr;    // d_wfac as the tensor-core byte matrix (bconv_wbytes), or null
};

struct ModDownTab {       // P -> Q_L
    u64* d_vfac;          // [K]   (P/p_k)^{-1} mod p_k
    u64* d_vfac_sh;
    u64* d_wfac;          // [K][L] (P/p_k) mod q_i
    u64* d_pinv;          // [L]   P^{-1} mod q_i
    u64* d_pinv_sh;
    u64* d_pmod;          // [L]   q_i - (P mod q_i) (rounding correction, DESIGN.md R-MODDOWN)
    u64* d_cfix;          // [K]   floor(2^(123 - s_k) / p_k)
    u64* d_csh;           // [K]   s_k = 63 - bitlen(p_k)
    u64* d_pl;            // [L]   P mod q_i and its Shoup quotient (extended-basis lift, R-LAZY)
    u64* d_pl_sh;
    uint8_t* d_wb = nullptr;    // d_wfac as the tensor-core byte matrix
    NttPostTab post;            // vfac as iNTT output factors (the BConv input then arrives pre-scaled)
};

struct MDRTab {           // merged ModDown + rescale (R-LAZY): basis B' = {q_{L-1}, p_0..p_{K-1}} -> Q_{L-1}
    u64 *d_vfac, *d_vfac_sh, *d_wfac, *d_corr, *d_cfix, *d_csh, *d_inv, *d_inv_sh;
    uint8_t* d_wb = nullptr;    // d_wfac as the tensor-core byte matrix
    NttPostTab post;            // vfac as iNTT output factors
};

struct RescaleTab {       // drop q_{L-1}
    u64* d_inv;           // [L-1] q_{L-1}^{-1} mod q_i
    u64* d_inv_sh;
    u64* d_hmod;          // [L-1] floor(q_{L-1}/2) mod q_i
};

struct MaskKey {
    int m, r0, r1, s0, ss, sc, level, ext;
    bool operator<(const MaskKey& o) const {
        return std::tie(m, r0, r1, s0, ss, sc, level, ext) < std::tie(o.m, o.r0, o.r1, o.s0, o.ss, o.sc, o.level, o.ext);
    }
};

struct KMKey {   // pre-masked key cache entry: (keys object, Galois element, mask descriptor)
    uint64_t keys_id;
    uint32_t g;
    MaskKey mk;
    bool operator<(const KMKey& o) const {
        if (keys_id != o.keys_id) return keys_id < o.keys_id;
        if (g != o.g) return g < o.g;
        return mk < o.mk;
    }
};

struct encf_ctx {
    int device = 0;
    int N = 0, logN = 0, L = 0, K = 0, alpha = 0;
    int s1 = 0, s2 = 0;                 // NTT phase split: N = 2^s1 (rows) x 2^s2 (columns)
    std::vector<u64> mods;              // q_0..q_{L-1}, p_0..p_{K-1}
    u64 max_mod = 0;
    std::vector<u64> mont_R, mont_Rinv; // 2^64 mod q and its inverse, per modulus id
    std::vector<u64> psi;               // chosen primitive 2N-th roots
    ModConst* d_mod = nullptr;          // [L+K]
    u64 *d_psi = nullptr, *d_psi_sh = nullptr, *d_ipsi = nullptr, *d_ipsi_sh = nullptr;   // [L+K][N]
    u64 *d_tw2 = nullptr, *d_itw2 = nullptr;        // [L+K][N][2] interleaved {w, w'} (fwd / inv)
    // FP64-pipe NTT path (ntt.cu) for moduli q < 2^41: twiddles as exact doubles {w, w/q}, per-modulus
    // {q, 1/q, N^-1, N^-1/q}; bit m of fpmask set <=> modulus id m takes the FP64 path
    double *d_twf = nullptr, *d_itwf = nullptr;     // [L+K][N][2]
    double* d_fpc = nullptr;                        // [L+K][4]
    u64 fpmask = 0;
    u64 *d_ninv = nullptr, *d_ninv_sh = nullptr;    // [L+K]
    u64 *d_imag = nullptr, *d_imag_sh = nullptr;    // [L+K]  psi^{N/2} (a 4th root of unity)
    std::vector<std::vector<ModUpTab>> modup;       // [level][digit]
    std::vector<NttPostTab> modup_post;             // [level]: every q-limb's ModUp vfac (its digit's) as iNTT output factors
    std::vector<ModDownTab> moddown;                // [level]
    std::vector<RescaleTab> rescale;                // [level]
    std::vector<MDRTab> mdr;                        // [level] (level >= 2)
    std::vector<void*> allocations;
    std::mutex mu;
    std::map<MaskKey, u64*> masks;      // NTT-form mask plaintexts [level][N]
    std::map<KMKey, u64*> kmasks;       // pre-masked keys (key (.) mask, Montgomery) + P (.) mask, per (keys, g, mask)
    std::map<std::vector<const u64*>, u64*> bhat;   // value-kernel mask spectra (bcast_ntt_table): key = masks + level
    std::vector<int> rot_group;         // 5^j mod 2N (host, for encode)
    int* d_rot_group = nullptr;
    // live kernel timing (encf_profile_*): CUDA events recorded around selected launches
    struct ProfRec { std::string name; cudaEvent_t a, b; uint64_t bytes; };
    bool prof = false, prof_all = false;
    std::string prof_only;
    std::vector<ProfRec> prof_recs;
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t prof_event();
    void prof_begin(const char* name, cudaStream_t s, uint64_t bytes, int& slot);
    void prof_end(int slot, cudaStream_t s);
    // statistics
    std::atomic<uint64_t> st_ks{0}, st_modup{0}, st_ntt{0}, st_ptmul{0}, st_ctmul{0}, st_launch{0}, st_bytes{0}, st_ntt_fp{0};

    std::vector<int> Kl;                // Kl[level] = K(level): special primes of a key switch at that level (R-KL)
    int Kof(int level) const { return Kl[level]; }
    int level_of_ext(int nl) const {    // the level L whose extended basis has nl = L + K(L) limbs (strictly increasing)
        for (int l = 1; l <= L; l++) if (l + Kl[l] == nl) return l;
        throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "no level with this extended limb count");
    }
    int dnum(int level) const { return (level + alpha - 1) / alpha; }
    LimbMap qmap(int level) const {
        LimbMap m; m.n = level;
        for (int i = 0; i < level; i++) m.mod[i] = (unsigned char)i;
        return m;
    }
    LimbMap extmap(int level) const {   // [q_0..q_{level-1}, p_0..p_{K(level)-1}]
        const int Kl_ = Kof(level);
        LimbMap m; m.n = level + Kl_;
        for (int i = 0; i < level; i++) m.mod[i] = (unsigned char)i;
        for (int k = 0; k < Kl_; k++) m.mod[level + k] = (unsigned char)(L + k);
        return m;
    }
    size_t limb_words() const { return (size_t)N; }
    void* dev_alloc(size_t bytes);
    // persistent pinned host arena: request tables uploaded while a stream is being CAPTURED into a CUDA
    // graph must outlive the capture (the memcpy node re-reads them at every replay); freed at destroy.
    std::vector<void*> pinned;
    size_t pin_used = 0, pin_cap = 0;
    void* pinned_persistent(size_t bytes);
};

// key material (device, NTT form)
struct encf_keys {
    uint64_t id = 0;                    // unique per keygen (pre-masked key cache)
    int max_level = 0;
    int dnum = 0;
    u64* sk = nullptr;                  // [max_level + K(max_level)][N]
    std::map<uint32_t, u64*> ksk;       // galois (0 = relin) -> [dnum][2][max_level + K(max_level)][N]
    // keys of the lower special-prime classes K(L) < K(max_level) (R-KL), derived on first use:
    // (galois, K) -> [dnum][2][max_level + K][N]
    std::map<std::pair<uint32_t, int>, u64*> cls;
    std::mutex mu;
    std::vector<void*> allocations;
    int device = 0;
    encf_ctx* ctx = nullptr;            // owner context: its pre-masked key cache entries are evicted at destroy
};

// ------------------------------------------------------------------------------------ scratch
struct Scratch {   // stream-ordered device scratch, freed in the destructor (cudaFreeAsync)
    cudaStream_t s;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t st) : s(st) {}
    u64* get(size_t words) {
        void* p = nullptr;
        cudaError_t e = cudaMallocAsync(&p, words * sizeof(u64), s);
        if (e != cudaSuccess) throw EncfError(ENCF_ERR_OOM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
        ptrs.push_back(p);
        return (u64*)p;
    }
    ~Scratch() { for (void* p : ptrs) cudaFreeAsync(p, s); }
};

// ------------------------------------------------------------------------------------ batched request tables
// (passed BY VALUE as kernel parameters -- CUDA >= 12.1 allows 32 KB of parameters)
constexpr int KS_BATCH = 128;
struct KsInnerBatch {
    const u64* ext[KS_BATCH];
    const u64* key[KS_BATCH];
    u64* acc[KS_BATCH];
    uint32_t gather[KS_BATCH];
    // optional extended-basis lift (R-LAZY rotations kept in Q_L u P): acc_0 += P sigma_{g0}(c0) on the q-limbs, fused
    // into the inner product (k_ks_inner_batch's pl / pl_sh); c0 = nullptr: none
    const u64* c0[KS_BATCH] = {};
    const u64* c1[KS_BATCH] = {};   // optional: acc_1 += P sigma_{g0}(c1) too (the relinearisation's P d1)
    uint32_t g0[KS_BATCH] = {};
};
struct OutBatch {
    u64* out[KS_BATCH][2];
    const u64* add[KS_BATCH][2];
};
constexpr int CP_BATCH = 512;
constexpr int ADDI_BATCH = 32;
struct AddIBatch { const u64* a[ADDI_BATCH]; const u64* b[ADDI_BATCH]; u64* out[ADDI_BATCH]; };
void k_add_i_batch(encf_ctx& c, const AddIBatch& B, int n, int npolys, const LimbMap& m, bool sub, cudaStream_t s);
struct CopyBatch {
    const u64* src[CP_BATCH];
    uint32_t g[CP_BATCH];
};
struct KeyLimb { int kl[MAX_LIMBS]; };
constexpr int RS_TERMS = 32;
struct RotSumBatch {               // hoisted rotation sums (R-ROUTE): per request r, terms i share ModUp(c1_r)
    const u64* ext[KS_BATCH];
    const u64* c0[KS_BATCH];
    const u64* c1[KS_BATCH];
    u64* acc[KS_BATCH];
    const u64* key[RS_TERMS];
    uint32_t g[RS_TERMS];
    const u64* mask[RS_TERMS];     // ks_rma: per-term extended-basis mask (NTT form)
};
struct SumDev { const u64* ct; const u64* mask; };
struct BcastArgs {                 // value-kernel broadcast MAC (C8 step 4)
    const u64* src[128];           // src[i] = Phi^{delta}(p), delta = t0 - dmax + i
    const u64* mask[64];           // n_u, u < nu
    u64* out[64];                  // b_{t0 + t}, t < nt
    int nsrc, nu, nt, dmax;        // dmax = nu - 1
};
struct R2F { u64 v[MAX_LIMBS]; };   // party * 2^{ell+sigma} mod q_i
struct PairDev { const u64* a; const u64* b; i64 as, bs; };   // operands + component strides
struct OutPos { int pos[MAX_LIMBS]; };

// ------------------------------------------------------------------------------------ launchers (ntt.cu)
void ntt_forward(encf_ctx& c, const PolyBatch& b, cudaStream_t s);
// Forward NTT whose last phase writes out_p = (src_p - NTT(y_p)) f (+ add_p) instead of NTT(y_p): the ModDown /
// rescale finish fused into the transform (device tables: per-polynomial src/out/add pointers, per-limb f + Shoup).
struct NttEpilogue { const u64* const* src; u64* const* out; const u64* const* add; const u64* f; const u64* fsh; };
void ntt_forward_epi(encf_ctx& c, const PolyBatch& b, const NttEpilogue* epi, cudaStream_t s);
void ntt_inverse(encf_ctx& c, const PolyBatch& b, cudaStream_t s);
// apply_ninv = false: returns N x (the coefficients); used only in front of the fast base conversions, whose
// vfac constants (ModUp / ModDown / merged ModDown+rescale tables) carry the N^{-1}
// src != nullptr: out-of-place (reads src with b's layout, writes b)
// post != nullptr (with apply_ninv = false): the output is x * post->f[limb] mod q instead of N x (limb = index in b.map)
struct NttPost { const u64* f; const u64* fsh; const double* fd; };
// src_stride: polynomial stride of src (default: b.poly_stride)
void ntt_inverse_scaled(encf_ctx& c, const PolyBatch& b, bool apply_ninv, cudaStream_t s, const u64* src = nullptr,
                        const NttPost* post = nullptr, i64 src_stride = -1);

// ------------------------------------------------------------------------------------ launchers (poly.cu)
void k_add(encf_ctx& c, const u64* a, const u64* b, u64* out, int npolys, const LimbMap& m, bool sub, cudaStream_t s);
void k_mul(encf_ctx& c, const u64* a, i64 a_stride, const u64* b, i64 b_stride, u64* out, i64 o_stride,
           int npolys, const LimbMap& m, cudaStream_t s);
void k_mul_i(encf_ctx& c, const u64* a, u64* out, int npolys, const LimbMap& m, cudaStream_t s);
void k_automorph(encf_ctx& c, const u64* in, i64 in_stride, u64* out, i64 out_stride, int npolys, int nlimbs,
                 uint32_t g, cudaStream_t s);
void k_copy(const u64* in, u64* out, size_t words, cudaStream_t s);
void k_sample_uniform(encf_ctx& c, u64 seed, u64 stream, u64* out, const LimbMap& m, const int* gids, cudaStream_t s);
void k_sample_small(encf_ctx& c, u64 seed, u64 stream, int kind /*0 ternary, 1 cbd21*/, u64* out, const LimbMap& m,
                    cudaStream_t s);
void k_add_scalar(encf_ctx& c, u64* data, const LimbMap& m, const u64* d_scal, cudaStream_t s);
void k_scalar_mul(encf_ctx& c, u64* data, int npolys, const LimbMap& m, const u64* d_scal, const u64* d_scal_sh,
                  cudaStream_t s);
void k_mod_reduce(encf_ctx& c, u64* data, int npolys, const LimbMap& m, cudaStream_t s);
void k_rescale_prep(encf_ctx& c, const u64* last_coeff, u64* corr, int level, int ncomp, i64 last_stride,
                    cudaStream_t s);
void k_rescale_finish(encf_ctx& c, const u64* in, i64 in_stride, const u64* corr, u64* out, i64 out_stride,
                      int ncomp, int level, cudaStream_t s);
void k_moddown_finish(encf_ctx& c, const u64* b, const u64* y, const u64* add0, u64* out, int level,
                      const ModDownTab& t, cudaStream_t s);
void k_tensor_acc(encf_ctx& c, const u64* const* a, const u64* const* b, int nterms, u64* out3, int level,
                  cudaStream_t s);
void k_diag_mac(encf_ctx& c, const u64* bank, int nbank, const u64* w, int units, i64 w_unit_stride,
                u64* acc, i64 acc_stride, int level, cudaStream_t s);
void k_masked_sum(encf_ctx& c, const u64* const* cts, const u64* const* masks, int nterms, u64* out, int level,
                  cudaStream_t s);
void k_export_mask(encf_ctx& c, u64 seed, u64 stream, u64* c0, u64* share, int level, cudaStream_t s);
void k_export_mask_dev(encf_ctx& c, const u64* dss, u64 idx, u64* c0, u64* share, int level, cudaStream_t s);
void k_encode_slots(encf_ctx& c, const double* d_re, const double* d_im, int n_slots, double scale, int level,
                    u64* out, cudaStream_t s, const LimbMap* lmap = nullptr);
void k_encode_weights(encf_ctx& c, const double* dW, int d_in, int d_out, int C, int N1, int m, const int* bs, const int* ps,
                      const int* us, const int* qs, int batch, double scale, int level, u64* out, cudaStream_t s,
                      const double* dWim = nullptr, int real_input = 0);
void k_ks_rotsum(encf_ctx& c, const RotSumBatch& B, int nreq, int nterms, int dnum, int L, int key_nl, cudaStream_t s);
void k_ks_rma(encf_ctx& c, const RotSumBatch& B, int nreq, int nterms, int dnum, int L, int key_nl, cudaStream_t s);
// Grouped extended-basis rotation sums (the projection's giant-step fold, R-LAZY): group g's output
//   out_g = sum_{r in [start[g], start[g+1])} rot_ext(x_r, g_r) + P x0_g   over Q_L u P
// with rot_ext(x_r, g_r) = (sum_j sigma(ext_r,j) key_r,j[0] + P sigma_{g_r}(c0_r), sum_j sigma(ext_r,j) key_r,j[1]) (ext_r the
// ModUp of sigma_{g_r}(c1_r), so no digit gather) and x0_g an optional ciphertext lifted as is (both components, q-limbs)
struct KsGroupBatch {
    const u64* ext[KS_BATCH];
    const u64* key[KS_BATCH];
    const u64* c0[KS_BATCH];
    uint32_t g[KS_BATCH];
    int start[KS_BATCH + 1];
    u64* out[KS_BATCH];            // [2][L+K][N] per group
    const u64* x0[KS_BATCH];       // [2][L][N] or nullptr
};
void k_ks_group(encf_ctx& c, const KsGroupBatch& B, int ngrp, int dnum, int L, int key_nl, cudaStream_t s);
constexpr int PSI_BATCH = 128;
struct PsiBatch {                  // masked shift Psi^t without ModDown: h (.) rot_ext(x, g0) + u (.) rot_ext(x, g1)
    const u64* ext[PSI_BATCH];
    const u64* c0[PSI_BATCH];
    u64* out[PSI_BATCH];
    const u64* key[PSI_BATCH][2];
    const u64* mask[PSI_BATCH][2];
    uint32_t g[PSI_BATCH][2];
};
void k_ks_psi(encf_ctx& c, const PsiBatch& B, int nreq, int dnum, int L, int key_nl, cudaStream_t s);
// pre-masked key of (key of g, ext mask at level L): km [dnum][2][L+K][N] = key (.) m (Montgomery form kept),
// pm [L][N] = (P R mod q) (.) m; one allocation km | pm
// class-K key from the generated key: copy limbs [0, nl_out) of every [digit][comp] and add dr[i] s'_i on digit j's
// q-limbs of component 0 (DESIGN.md R-KL)
void k_key_class(encf_ctx& c, const u64* full, int nl_full, u64* out, int nl_out, int ML, int dnum, const u64* sp, const u64* dr,
                 cudaStream_t s);
void k_keymask(encf_ctx& c, const u64* key, int key_nl, const u64* mask, int dnum, int L, u64* out, cudaStream_t s);
// pl / pl_sh: P mod q_i and its Shoup quotient for the requests' c0 lifts (required when any B.c0 is set)
void k_ks_inner_batch(encf_ctx& c, const KsInnerBatch& B, int nreq, int dnum, int nl, int key_nl, const LimbMap& key_limb_of,
                      cudaStream_t s, const u64* pl = nullptr, const u64* pl_sh = nullptr);
void k_moddown_finish_batch(encf_ctx& c, const u64* acc, const u64* y, const OutBatch& O, int nreq, int level, int nl,
                            const ModDownTab& t, cudaStream_t s);
void k_bconv_batch(encf_ctx& c, const u64* in, i64 in_stride, const LimbMap& im, const u64* vf, const u64* vfs, const u64* wf,
                   const LimbMap& om, u64* out, i64 out_stride, const int* pos, int npolys, cudaStream_t s,
                   const u64* corr = nullptr, const u64* cfix = nullptr, const u64* csh = nullptr,
                   const uint8_t* wb = nullptr,    // wb: byte matrix of wf for the tensor-core path (bconv_wbytes)
                   bool prescaled = false);        // inputs already x vfac mod q_i (iNTT NttPost): skip the scaling
void k_gather_copy(encf_ctx& c, const CopyBatch& C, int n, u64* dst, i64 dst_stride, size_t words, cudaStream_t s);
void k_rescale_prep_batch(encf_ctx& c, const u64* last, u64* corr, int level, int npolys, cudaStream_t s);
void k_rescale_finish_batch(encf_ctx& c, const CopyBatch& In, const u64* corr, const CopyBatch& Out, int level, int npolys,
                            cudaStream_t s);
void k_sum_csr(encf_ctx& c, const SumDev* terms, const int* off, u64* const* outs, int nout, int nterms, int ncomp, int level,
               cudaStream_t s, const LimbMap* lmap = nullptr);
void k_lift_add(encf_ctx& c, const CopyBatch& dst, const CopyBatch& src, int n, int L, const u64* pm, const u64* pm_sh,
                cudaStream_t s);
void k_tensor_csr(encf_ctx& c, const PairDev* pairs, const int* off, u64* const* outs, int nout, int nterms, int level,
                  cudaStream_t s);
void k_bcast_mac(encf_ctx& c, const BcastArgs& A, int level, cudaStream_t s);
// the same outputs through negacyclic 128-point transforms along the window (ntt.cu; needs nsrc <= 128): the masks'
// spectrum table (cached per mask set and level) and the convolution launch
const u64* bcast_ntt_table(encf_ctx& c, const u64* const* masks, int nu, int level, cudaStream_t s);
void k_bcast_ntt(encf_ctx& c, const BcastArgs& A, const u64* bhat, int level, cudaStream_t s);
void k_ring2field(encf_ctx& c, const u64* mp, u64* out, int L, const R2F& off, cudaStream_t s);
void k_field2ring(encf_ctx& c, const u64* sh, u64* out, int ell, cudaStream_t s);
void k_decode_limb0(encf_ctx& c, const u64* coeff_limb0, double scale, double* d_re, double* d_im, cudaStream_t s);

// ------------------------------------------------------------------------------------ ciphertext-level ops (ks.cu)
struct CtView {
    u64* d;
    int ncomp, L;
    double scale;
    u64* comp(int c) const;
};
struct Eval;   // defined in ks.cu
