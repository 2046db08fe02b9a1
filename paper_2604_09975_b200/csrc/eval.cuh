// eval.cuh -- ciphertext-level operations (NTT-domain device ciphertexts) used by the ABI and the
// EncFormer kernels.  Mirrors the schedule contract of SURVEY.md §8c C4/C5 exactly (hybrid key
// switching with fast BConv, floor ModDown, SEAL rescale); bit-exactness against oracle/ is tested.
#pragma once
#include <vector>
#include "ctx.cuh"

struct DCt {                 // device ciphertext, NTT form, layout [comp][L][N]
    u64* d = nullptr;
    int ncomp = 2, L = 0;
    double scale = 1.0;
    u64* comp(int c, int N) const { return d + (size_t)c * L * N; }
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

    const u64* key_for(uint32_t g, int L) const;
    // ModUp of one NTT-form polynomial d (L limbs): returns ext [dnum][L+K][N] NTT form.
    u64* modup(const u64* d_ntt, int L);
    // inner product with key_g (Galois gather g fused, 1 = none) + ModDown of both components;
    // out0 = ModDown(b0) + add0, out1 = ModDown(b1) + add1 (add may be null; may alias out).
    void ks_core(const u64* ext, int L, uint32_t g_gather, const u64* key, u64* out0, u64* out1,
                 const u64* add0, const u64* add1);

    // ciphertext ops (outputs caller-provided in `out`, may alias inputs where noted)
    void rotate_galois(const DCt& in, uint32_t g, DCt& out);                 // single (non-hoisted)
    void rotate_hoisted(const DCt& in, const std::vector<uint32_t>& gs, std::vector<DCt>& outs);
    void relin(const DCt& in3, DCt& out);
    void rescale(const DCt& in, DCt& out);
    void add(const DCt& a, const DCt& b, DCt& out, bool sub = false);
    void mul_i(const DCt& a, DCt& out);
    void ptmul(const DCt& a, const u64* pt, double pt_scale, DCt& out);
    void mod_drop(const DCt& in, int L, DCt& out);
    void copy(const DCt& in, DCt& out);
    // lazy sums
    void tensor_sum(const std::vector<const DCt*>& A, const std::vector<const DCt*>& B, DCt& out3);
    void masked_sum(const std::vector<const DCt*>& C, const std::vector<const u64*>& M, double m_scale, DCt& out);

    uint32_t galois_rot(long steps) const;
    uint32_t galois_conj() const { return 2u * c.N - 1u; }
    // masks
    const u64* mask(int m, int r0, int r1, int s0, int ss, int sc, int level);
    double mask_scale(int level) const { return (double)c.mods[level - 1]; }
    const u64* const* dev_ptrs(const std::vector<const u64*>& v);
};

void check_scale(double a, double b);
