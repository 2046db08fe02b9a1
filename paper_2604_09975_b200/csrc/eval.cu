// eval.cu -- key switching (hybrid, dnum digits), rotations (single and hoisted), conj, relin,
// rescale and the small ciphertext ops, as sequences of the sm_100a kernels of ntt.cu / poly.cu.
#include <cstring>
#include "eval.cuh"

void check_scale(double a, double b) {
    if (!(a == b)) throw EncfError(ENCF_ERR_SCALE_MISMATCH, "operands have different scales");
}

uint32_t Ev::galois_rot(long steps) const {
    long n = c.N / 2;
    long r = ((steps % n) + n) % n;
    u64 g = h_powmod(5, (u64)r, 2 * (u64)c.N);
    return (uint32_t)g;
}

const u64* Ev::key_for(uint32_t g, int L) const {
    if (!keys) throw EncfError(ENCF_ERR_MISSING_KEY, "no keys");
    auto it = keys->ksk.find(g);
    if (it == keys->ksk.end()) throw EncfError(ENCF_ERR_MISSING_KEY, "missing key for galois element " + std::to_string(g));
    if (L > keys->max_level) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "ciphertext level above the key's max_level");
    return it->second;
}

// ModUp (C4): for every digit j, inside the digit d~ = d (NTT limbs copied), elsewhere fast BConv of the
// digit's coefficient-form limbs followed by a forward NTT.
u64* Ev::modup(const u64* d_ntt, int L) {
    const int N = c.N, K = c.K, nl = L + K, dn = c.dnum(L);
    u64* dco = sc.get((size_t)L * N);
    k_copy(d_ntt, dco, (size_t)L * N, s);
    ntt_inverse(c, PolyBatch{dco, 0, 1, c.qmap(L)}, s);
    u64* ext = sc.get((size_t)dn * nl * N);
    LimbMap em = c.extmap(L);
    for (int j = 0; j < dn; j++) {
        const ModUpTab& t = c.modup[L][j];
        u64* ej = ext + (size_t)j * nl * N;
        k_copy(d_ntt + (size_t)t.lo * N, ej + (size_t)t.lo * N, (size_t)(t.hi - t.lo) * N, s);
        LimbMap im;
        im.n = t.hi - t.lo;
        for (int i = 0; i < im.n; i++) im.mod[i] = (unsigned char)(t.lo + i);
        k_bconv(c, dco + (size_t)t.lo * N, im, t.d_vfac, t.d_vfac_sh, t.d_wfac, t.tgt, ej, t.tgt_pos.data(), s);
        // NTT of [0, lo) and [hi, nl)
        if (t.lo > 0) {
            LimbMap m; m.n = t.lo;
            for (int i = 0; i < t.lo; i++) m.mod[i] = em.mod[i];
            ntt_forward(c, PolyBatch{ej, 0, 1, m}, s);
        }
        if (t.hi < nl) {
            LimbMap m; m.n = nl - t.hi;
            for (int i = t.hi; i < nl; i++) m.mod[i - t.hi] = em.mod[i];
            ntt_forward(c, PolyBatch{ej + (size_t)t.hi * N, 0, 1, m}, s);
        }
    }
    c.st_modup++;
    return ext;
}

// Inner product + ModDown (C4): (b0, b1) = sum_j d~_j ksk_j ; out_c = (b_c - fastBConv_{P->Q}([b_c]_P)) P^{-1}.
void Ev::ks_core(const u64* ext, int L, uint32_t gg, const u64* key, u64* out0, u64* out1, const u64* add0,
                 const u64* add1) {
    const int N = c.N, K = c.K, nl = L + K, dn = c.dnum(L);
    const int ML = keys->max_level, key_nl = ML + K;
    u64* acc = sc.get((size_t)2 * nl * N);
    LimbMap klm;   // ext limb -> key limb
    klm.n = nl;
    for (int e = 0; e < nl; e++) klm.mod[e] = (unsigned char)(e < L ? e : ML + (e - L));
    k_ks_inner(c, ext, dn, nl, gg, key, key_nl, klm, acc, s);
    // [b]_P to coefficient form (both components in one batch)
    LimbMap pm; pm.n = K;
    for (int k = 0; k < K; k++) pm.mod[k] = (unsigned char)(c.L + k);
    ntt_inverse(c, PolyBatch{acc + (size_t)L * N, (i64)nl * N, 2, pm}, s);
    u64* y = sc.get((size_t)2 * L * N);
    const ModDownTab& md = c.moddown[L];
    LimbMap qm = c.qmap(L);
    std::vector<int> pos(L);
    for (int i = 0; i < L; i++) pos[i] = i;
    for (int comp = 0; comp < 2; comp++)
        k_bconv(c, acc + (size_t)comp * nl * N + (size_t)L * N, pm, md.d_vfac, md.d_vfac_sh, md.d_wfac, qm,
                y + (size_t)comp * L * N, pos.data(), s);
    ntt_forward(c, PolyBatch{y, (i64)L * N, 2, qm}, s);
    k_moddown_finish(c, acc, y, add0, out0, L, md, s);
    k_moddown_finish(c, acc + (size_t)nl * N, y + (size_t)L * N, add1, out1, L, md, s);
    c.st_ks++;
}

void Ev::rotate_galois(const DCt& in, uint32_t g, DCt& out) {
    if (in.ncomp != 2) throw EncfError(ENCF_ERR_FORMAT, "rotate needs 2 components");
    const int N = c.N, L = in.L;
    const u64* key = key_for(g, L);
    u64* tmp = sc.get((size_t)2 * L * N);
    k_automorph(c, in.d, (i64)L * N, tmp, (i64)L * N, 2, L, g, s);     // sigma_g(c0), sigma_g(c1)
    u64* ext = modup(tmp + (size_t)L * N, L);
    out.L = L; out.ncomp = 2; out.scale = in.scale;
    ks_core(ext, L, 1u, key, out.comp(0, N), out.comp(1, N), tmp, nullptr);
}

void Ev::rotate_hoisted(const DCt& in, const std::vector<uint32_t>& gs, std::vector<DCt>& outs) {
    if (in.ncomp != 2) throw EncfError(ENCF_ERR_FORMAT, "rotate needs 2 components");
    const int N = c.N, L = in.L;
    bool any = false;
    for (uint32_t g : gs) any |= (g != 1u);
    u64* ext = any ? modup(in.comp(1, N), L) : nullptr;
    for (size_t i = 0; i < gs.size(); i++) {
        DCt& o = outs[i];
        o.L = L; o.ncomp = 2; o.scale = in.scale;
        if (gs[i] == 1u) { copy(in, o); continue; }
        const u64* key = key_for(gs[i], L);
        k_automorph(c, in.comp(0, N), 0, o.comp(0, N), 0, 1, L, gs[i], s);
        ks_core(ext, L, gs[i], key, o.comp(0, N), o.comp(1, N), o.comp(0, N), nullptr);
    }
}

void Ev::relin(const DCt& in, DCt& out) {
    if (in.ncomp != 3) throw EncfError(ENCF_ERR_FORMAT, "relinearize needs 3 components");
    const int N = c.N, L = in.L;
    const u64* key = key_for(0u, L);
    u64* ext = modup(in.comp(2, N), L);
    out.L = L; out.ncomp = 2; out.scale = in.scale;
    ks_core(ext, L, 1u, key, out.comp(0, N), out.comp(1, N), in.comp(0, N), in.comp(1, N));
}

// Rescale (C5) in the NTT domain: the last limb to coefficient form, correction per remaining limb,
// forward NTT of the correction, then (c_i - corr_i) q_L^{-1}.
void Ev::rescale(const DCt& in, DCt& out) {
    const int N = c.N, L = in.L, nc = in.ncomp;
    if (L <= 1) throw EncfError(ENCF_ERR_LEVEL_EXHAUSTED, "rescale at one limb");
    u64* last = sc.get((size_t)nc * N);
    for (int comp = 0; comp < nc; comp++) k_copy(in.comp(comp, N) + (size_t)(L - 1) * N, last + (size_t)comp * N, N, s);
    LimbMap lm; lm.n = 1; lm.mod[0] = (unsigned char)(L - 1);
    ntt_inverse(c, PolyBatch{last, (i64)N, nc, lm}, s);
    u64* corr = sc.get((size_t)nc * (L - 1) * N);
    k_rescale_prep(c, last, corr, L, nc, (i64)N, s);
    ntt_forward(c, PolyBatch{corr, (i64)(L - 1) * N, nc, c.qmap(L - 1)}, s);
    k_rescale_finish(c, in.d, (i64)L * N, corr, out.d, (i64)(L - 1) * N, nc, L, s);
    out.L = L - 1; out.ncomp = nc; out.scale = in.scale / (double)c.mods[L - 1];
}

void Ev::add(const DCt& a, const DCt& b, DCt& out, bool sub) {
    check_scale(a.scale, b.scale);
    if (a.L != b.L || a.ncomp != b.ncomp) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "add: level/component mismatch");
    k_add(c, a.d, b.d, out.d, a.ncomp, c.qmap(a.L), sub, s);
    out.L = a.L; out.ncomp = a.ncomp; out.scale = a.scale;
}

void Ev::mul_i(const DCt& a, DCt& out) {
    k_mul_i(c, a.d, out.d, a.ncomp, c.qmap(a.L), s);
    out.L = a.L; out.ncomp = a.ncomp; out.scale = a.scale;
}

void Ev::ptmul(const DCt& a, const u64* pt, double pt_scale, DCt& out) {
    const int N = c.N;
    k_mul(c, a.d, (i64)a.L * N, pt, 0, out.d, (i64)a.L * N, a.ncomp, c.qmap(a.L), s);
    out.L = a.L; out.ncomp = a.ncomp; out.scale = a.scale * pt_scale;
    c.st_ptmul++;
}

void Ev::mod_drop(const DCt& in, int L, DCt& out) {
    if (L < 1 || L > in.L) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "mod_drop: bad level");
    const int N = c.N;
    for (int comp = 0; comp < in.ncomp; comp++) {
        if (out.d + (size_t)comp * L * N != in.d + (size_t)comp * in.L * N)
            CUDA_TRY(cudaMemcpyAsync(out.d + (size_t)comp * L * N, in.d + (size_t)comp * in.L * N, (size_t)L * N * 8,
                                     cudaMemcpyDeviceToDevice, s));
    }
    out.L = L; out.ncomp = in.ncomp; out.scale = in.scale;
}

void Ev::copy(const DCt& in, DCt& out) {
    k_copy(in.d, out.d, ct_words(in.L, in.ncomp), s);
    out.L = in.L; out.ncomp = in.ncomp; out.scale = in.scale;
}

const u64* const* Ev::dev_ptrs(const std::vector<const u64*>& v) {
    u64* d = sc.get(v.size());
    CUDA_TRY(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(u64*), cudaMemcpyHostToDevice, s));
    return (const u64* const*)d;
}

void Ev::tensor_sum(const std::vector<const DCt*>& A, const std::vector<const DCt*>& B, DCt& out3) {
    const int L = A[0]->L;
    double sc0 = A[0]->scale * B[0]->scale;
    std::vector<const u64*> pa, pb;
    for (size_t t = 0; t < A.size(); t++) {
        if (A[t]->L != L || B[t]->L != L) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "tensor: level mismatch");
        check_scale(A[t]->scale * B[t]->scale, sc0);
        pa.push_back(A[t]->d);
        pb.push_back(B[t]->d);
    }
    for (size_t t0 = 0; t0 < pa.size(); t0 += 64) {   // pointer lists of at most 64 entries per launch
        size_t te = std::min(pa.size(), t0 + 64);
        std::vector<const u64*> a(pa.begin() + t0, pa.begin() + te), b(pb.begin() + t0, pb.begin() + te);
        if (t0 == 0) {
            k_tensor_acc(c, dev_ptrs(a), dev_ptrs(b), (int)a.size(), out3.d, L, s);
        } else {
            u64* tmp = sc.get(ct_words(L, 3));
            k_tensor_acc(c, dev_ptrs(a), dev_ptrs(b), (int)a.size(), tmp, L, s);
            k_add(c, out3.d, tmp, out3.d, 3, c.qmap(L), false, s);
        }
    }
    out3.L = L; out3.ncomp = 3; out3.scale = sc0;
}

void Ev::masked_sum(const std::vector<const DCt*>& C, const std::vector<const u64*>& M, double m_scale, DCt& out) {
    const int L = C[0]->L;
    double s0 = C[0]->scale * m_scale;
    std::vector<const u64*> pc;
    for (auto* x : C) {
        if (x->L != L) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "masked_sum: level mismatch");
        check_scale(x->scale * m_scale, s0);
        pc.push_back(x->d);
    }
    k_masked_sum(c, dev_ptrs(pc), dev_ptrs(M), (int)pc.size(), out.d, L, s);
    out.L = L; out.ncomp = 2; out.scale = s0;
}

// Mask plaintexts: cached per (descriptor, level) in NTT form; encoded on the GPU on first use at
// scale q_{level-1}, unless a plaintext was installed with encf_mask_put (parity tests).
const u64* Ev::mask(int m, int r0, int r1, int s0, int ss, int scount, int level) {
    MaskKey key{m, r0, r1, s0, ss, scount, level};
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.masks.find(key);
    if (it != c.masks.end()) return it->second;
    const int N = c.N, n = N / 2;
    std::vector<double> re(n, 0.0);
    for (int k = 0; k < scount; k++) {
        int sg = s0 + k * ss;
        for (int r = r0; r < r1; r++) re[(size_t)sg * m + r] = 1.0;
    }
    u64* pt = nullptr;
    CUDA_TRY(cudaMalloc(&pt, (size_t)level * N * 8));
    Scratch tmp(s);
    double* dre = (double*)tmp.get(n);
    CUDA_TRY(cudaMemcpyAsync(dre, re.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    k_encode_slots(c, dre, nullptr, n, (double)c.mods[level - 1], level, pt, s);
    ntt_forward(c, PolyBatch{pt, 0, 1, c.qmap(level)}, s);
    c.masks[key] = pt;
    return pt;
}
