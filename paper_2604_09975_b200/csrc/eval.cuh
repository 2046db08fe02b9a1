// eval.cuh -- ciphertext-level operations (NTT-domain device ciphertexts) used by the ABI and the
// EncFormer kernels.  Every operation is BATCHED: a list of independent ciphertexts at one level is
// processed by one launch sequence (ModUp / inner product / ModDown / rescale / lazy sums), so the
// grid covers all of them.  Bit-exact schedule contract: SURVEY.md §8c C4/C5 (oracle/ckks.py).
#pragma once
#include <cstring>
#include <vector>
#include "ctx.cuh"

struct DCt {                 // device ciphertext, NTT form, layout [comp][L][N]
    u64* d = nullptr;
    int ncomp = 2, L = 0;
    double scale = 1.0;
    i64 cstride = 0;         // component stride in words (0 -> L * N)
    u64* comp(int c, int N) const { return d + (size_t)c * (cstride ? cstride : (i64)L * N); }
};

// One key switch request: inner product of the (already ModUp'ed) digits `ext` with `key`, with the
// Galois gather `gather` fused into the digit loads, then ModDown; out_c = ModDown(b_c) + add_c.
struct KsReq {
    const u64* ext;
    const u64* key;
    uint32_t gather;
    u64* out0;
    u64* out1;
    const u64* add0;
    const u64* add1;
};

// A lazy sum term: ct (2 or 3 components) times an optional mask plaintext (nullptr = 1).
struct SumTerm {
    const u64* ct;
    const u64* mask;
};

struct Ev {
    encf_ctx& c;
    const encf_keys* keys;
    cudaStream_t s;
    Scratch& sc;
    Ev(encf_ctx& cc, const encf_keys* k, cudaStream_t st, Scratch& scr) : c(cc), keys(k), s(st), sc(scr) {}

    size_t ct_words(int L, int ncomp = 2) const { return (size_t)ncomp * L * c.N; }
    DCt alloc(int L, int ncomp = 2, double scale = 1.0) {
        DCt x; x.d = sc.get(ct_words(L, ncomp)); x.L = L; x.ncomp = ncomp; x.scale = scale; return x;
    }
    std::vector<DCt> alloc_many(int n, int L, int ncomp = 2);

    const u64* key_for(uint32_t g, int L) const;
    uint32_t galois_rot(long steps) const;
    uint32_t galois_conj() const { return 2u * c.N - 1u; }

    // ---- batched key switching core
    // ModUp of polys[i] (NTT form, L limbs), each optionally permuted by gathers[i] first.
    // Returns ext [n][dnum][L+K][N]; ext_stride() words per polynomial.
    u64* modup_many(const std::vector<const u64*>& polys, const std::vector<uint32_t>& gathers, int L);
    size_t ext_stride(int L) const { return (size_t)c.dnum(L) * (L + c.Kof(L)) * c.N; }
    void ks_many(const std::vector<KsReq>& reqs, int L);

    // ---- ciphertext ops (outputs caller-provided; lists must share one level)
    void rotate_many(const std::vector<const DCt*>& ins, const std::vector<uint32_t>& gs, std::vector<DCt>& outs);
    void hoisted_many(const std::vector<const DCt*>& ins, const std::vector<std::vector<uint32_t>>& gs,
                      std::vector<std::vector<DCt>>& outs);
    void relin_many(const std::vector<const DCt*>& ins, std::vector<DCt>& outs);
    void relin_rescale_many(const std::vector<const DCt*>& ins, std::vector<DCt>& outs);   // rescale(relin) rounded once
    void rescale_many(const std::vector<const DCt*>& ins, std::vector<DCt>& outs);
    void sum_many(const std::vector<std::vector<SumTerm>>& terms, int L, int ncomp, std::vector<DCt>& outs,
                  const std::vector<double>& scales);
    void tensor_many(const std::vector<std::vector<std::pair<const DCt*, const DCt*>>>& pairs, std::vector<DCt>& outs);

    // single-item conveniences
    void rotate_galois(const DCt& in, uint32_t g, DCt& out);
    void rotate_hoisted(const DCt& in, const std::vector<uint32_t>& gs, std::vector<DCt>& outs);
    void relin(const DCt& in3, DCt& out);
    void rescale(const DCt& in, DCt& out);
    void add(const DCt& a, const DCt& b, DCt& out, bool sub = false);
    void mul_i(const DCt& a, DCt& out);
    // outs[r] = a[r] +- X^{N/2} b[r] (= add(a, mul_i(b)) bit for bit), batched launches
    void add_i_many(const std::vector<const DCt*>& a, const std::vector<const DCt*>& b, std::vector<DCt>& outs, bool sub = false);
    void ptmul(const DCt& a, const u64* pt, double pt_scale, DCt& out);
    void mod_drop(const DCt& in, int L, DCt& out);
    void copy(const DCt& in, DCt& out);
    void tensor_sum(const std::vector<const DCt*>& A, const std::vector<const DCt*>& B, DCt& out3);
    void masked_sum(const std::vector<const DCt*>& C, const std::vector<const u64*>& M, double m_scale, DCt& out);

    // ---- lazy key switching over the extended basis Q_L u P (DESIGN.md R-LAZY).  An "ext" ciphertext is
    // [2][L+K][N] (NTT form) with .L = L; its ModDown is an ordinary ciphertext.
    std::vector<DCt> alloc_many_ext(int n, int L);
    void hoisted_many_ext(const std::vector<const DCt*>& ins, const std::vector<std::vector<uint32_t>>& gs,
                          std::vector<std::vector<DCt>>& outs);
    void sum_many_ext(const std::vector<std::vector<SumTerm>>& terms, int L, std::vector<DCt>& outs,
                      const std::vector<double>& scales);
    void moddown_rescale_many(const std::vector<DCt>& ins_ext, std::vector<DCt>& outs);   // ins contiguous (alloc_many_ext)
    void moddown_many(const std::vector<DCt>& ins_ext, std::vector<DCt>& outs);           // ins contiguous (alloc_many_ext)
    void rotate_many_ext(const std::vector<const DCt*>& ins, const std::vector<uint32_t>& gs, std::vector<DCt>& outs_ext);
    void lift_many(const std::vector<const DCt*>& ins, std::vector<DCt>& outs_ext);       // P * ct over Q_L u P
    // outs[i] = ModDown(P x_i + sum_{g in gs} rot_ext(x_i, g)): one hoisted ModUp + one ModDown per input (R-ROUTE)
    void rotsum_many(const std::vector<const DCt*>& ins, const std::vector<uint32_t>& gs, std::vector<DCt>& outs);

    // masks
    const u64* mask(int m, int r0, int r1, int s0, int ss, int sc, int level, int ext = 0);
    const u64* mask_ext(int m, int r0, int r1, int s0, int ss, int sc, int level) { return mask(m, r0, r1, s0, ss, sc, level, 1); }
    double mask_scale(int level) const { return (double)c.mods[level - 1]; }
    // cached pre-masked key of Galois element g with the ext mask (m, r0, r1, s0, ss, sc) at level L:
    // returns km ([dnum][2][L+K][N]); *pm = km + dnum*2*(L+K)*N ([L][N], P R (.) mask)
    const u64* keymask(uint32_t g, int m, int r0, int r1, int s0, int ss, int sc, int L, const u64** pm);
    template <class T>
    T* upload(const std::vector<T>& v) {
        // eager: pageable copy (staged by the driver, so v may die at once); under CUDA-graph capture the
        // table is copied into the context's persistent pinned arena, which the memcpy node re-reads at replay
        const size_t bytes = v.size() * sizeof(T);
        u64* d = sc.get((bytes + 7) / 8 + 1);
        if (!bytes) return (T*)d;
        cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
        CUDA_TRY(cudaStreamIsCapturing(s, &st));
        const void* src = v.data();
        if (st == cudaStreamCaptureStatusActive) {
            void* h = c.pinned_persistent(bytes);
            std::memcpy(h, v.data(), bytes);
            src = h;
        }
        CUDA_TRY(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s));
        return (T*)d;
    }
};

void check_scale(double a, double b);
