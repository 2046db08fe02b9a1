// eval.cu -- batched key switching (hybrid, dnum digits, fast BConv, floor ModDown), rotations
// (single and hoisted), conj, relin, rescale and lazy sums as short sequences of sm_100a launches that
// each cover a whole list of ciphertexts.
#include <cstring>
#include "eval.cuh"

void check_scale(double a, double b) {
    if (!(a == b)) throw EncfError(ENCF_ERR_SCALE_MISMATCH, "operands have different scales");
}

uint32_t Ev::galois_rot(long steps) const {
    long n = c.N / 2;
    long r = ((steps % n) + n) % n;
    return (uint32_t)h_powmod(5, (u64)r, 2 * (u64)c.N);
}

// The key of Galois element g (0 = relin) for a key switch at level L: the generated key when L's special-prime
// class K(L) is the top class K(max_level); otherwise the class-K(L) key, derived once and cached (R-KL, oracle
// ckks.Keys.key_at): the same a_j, e_j restricted to Q_max u P_{K(L)} and b_j += (P_{K(L)} - P_{K(max)}) s' on digit
// j's q-limbs, s' = sigma_g(s) or s^2 (NTT domain, Montgomery form kept).
const u64* Ev::key_for(uint32_t g, int L) const {
    if (!keys) throw EncfError(ENCF_ERR_MISSING_KEY, "no keys");
    auto it = keys->ksk.find(g);
    if (it == keys->ksk.end()) throw EncfError(ENCF_ERR_MISSING_KEY, "missing key for galois element " + std::to_string(g));
    if (L > keys->max_level) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "ciphertext level above the key's max_level");
    const int ML = keys->max_level, KM = c.Kof(ML), KL = c.Kof(L);
    if (KL == KM) return it->second;
    encf_keys* kk = const_cast<encf_keys*>(keys);
    std::lock_guard<std::mutex> lk(kk->mu);
    auto f = kk->cls.find({g, KL});
    if (f != kk->cls.end()) return f->second;
    const int N = c.N, dn = c.dnum(ML);
    u64* out = nullptr;
    CUDA_TRY(cudaMalloc(&out, (size_t)dn * 2 * (ML + KL) * N * 8));
    kk->allocations.push_back(out);
    u64* sp = sc.get((size_t)ML * N);
    LimbMap qm = c.qmap(ML);
    if (g == 0u) k_mul(c, keys->sk, 0, keys->sk, 0, sp, 0, 1, qm, s);          // s^2 (NTT domain)
    else k_automorph(c, keys->sk, 0, sp, 0, 1, ML, g % (2u * N), s);           // sigma_g(s)
    std::vector<u64> dr(ML);
    for (int i = 0; i < ML; i++) {
        const u64 q = c.mods[i];
        u64 pl = 1, pm = 1;
        for (int k = 0; k < KM; k++) {
            const u64 pk = c.mods[c.L + k] % q;
            pm = h_mulmod(pm, pk, q);
            if (k < KL) pl = h_mulmod(pl, pk, q);
        }
        dr[i] = h_mulmod(sub_mod(pl, pm, q), c.mont_R[i], q);    // (P_{K(L)} - P_{K(max)}) R mod q_i
    }
    u64* ddr = sc.get(ML);
    CUDA_TRY(cudaMemcpyAsync(ddr, dr.data(), ML * 8, cudaMemcpyHostToDevice, s));   // pageable: staged before return
    k_key_class(c, it->second, ML + KM, out, ML + KL, ML, dn, sp, ddr, s);
    kk->cls[{g, KL}] = out;
    return out;
}

std::vector<DCt> Ev::alloc_many(int n, int L, int ncomp) {
    std::vector<DCt> v(n);
    if (n == 0) return v;
    u64* base = sc.get(ct_words(L, ncomp) * n);
    for (int i = 0; i < n; i++) { v[i].d = base + ct_words(L, ncomp) * i; v[i].L = L; v[i].ncomp = ncomp; }
    return v;
}

// ModUp (C4) of n polynomials: inside digit j, d~ = d (NTT limbs copied); on every other modulus of
// Q_L u P, fast BConv of the digit's coefficient-form limbs, then forward NTT.  One launch sequence for
// all n polynomials.
u64* Ev::modup_many(const std::vector<const u64*>& polys, const std::vector<uint32_t>& gathers, int L) {
    const int N = c.N, K = c.Kof(L), nl = L + K, dn = c.dnum(L), n = (int)polys.size();
    const size_t Lw = (size_t)L * N;
    const size_t es = ext_stride(L);
    u64* ext = sc.get(es * n);
    LimbMap em = c.extmap(L);
    // the inputs' digit limbs (NTT form, Galois-gathered) go straight to their place in ext; the iNTT reads them there
    // (no staging copy of the whole input)
    for (int j = 0; j < dn; j++) {
        const ModUpTab& t = c.modup[L][j];
        for (int i0 = 0; i0 < n; i0 += CP_BATCH) {
            int cnt = std::min(CP_BATCH, n - i0);
            CopyBatch cb;
            for (int i = 0; i < cnt; i++) {
                cb.src[i] = polys[i0 + i] + (size_t)t.lo * N;
                cb.g[i] = gathers.empty() ? 1u : gathers[i0 + i];
            }
            k_gather_copy(c, cb, cnt, ext + es * i0 + (size_t)j * nl * N + (size_t)t.lo * N, (i64)es, (size_t)(t.hi - t.lo) * N, s);
        }
    }
    u64* dco = sc.get(Lw * n);
    for (int j = 0; j < dn; j++) {   // out of place, per digit; the output is x vfac (NttPost), the BConv input
        const ModUpTab& t = c.modup[L][j];
        LimbMap m; m.n = t.hi - t.lo;
        for (int i = 0; i < m.n; i++) m.mod[i] = (unsigned char)(t.lo + i);
        const NttPost post{c.modup_post[L].f + t.lo, c.modup_post[L].fsh + t.lo, c.modup_post[L].fd + 2 * t.lo};
        ntt_inverse_scaled(c, PolyBatch{dco + (size_t)t.lo * N, (i64)Lw, n, m}, false, s,
                           ext + (size_t)j * nl * N + (size_t)t.lo * N, &post, (i64)es);
    }
    for (int j = 0; j < dn; j++) {
        const ModUpTab& t = c.modup[L][j];
        u64* ej = ext + (size_t)j * nl * N;
        LimbMap im;
        im.n = t.hi - t.lo;
        for (int i = 0; i < im.n; i++) im.mod[i] = (unsigned char)(t.lo + i);
        k_bconv_batch(c, dco + (size_t)t.lo * N, (i64)Lw, im, t.d_vfac, t.d_vfac_sh, t.d_wfac, t.tgt, ej, (i64)es,
                      t.tgt_pos.data(), n, s, nullptr, nullptr, nullptr, t.d_wb, true);
        if (t.lo > 0) {
            LimbMap m; m.n = t.lo;
            for (int i = 0; i < t.lo; i++) m.mod[i] = em.mod[i];
            ntt_forward(c, PolyBatch{ej, (i64)es, n, m}, s);
        }
        if (t.hi < nl) {
            LimbMap m; m.n = nl - t.hi;
            for (int i = t.hi; i < nl; i++) m.mod[i - t.hi] = em.mod[i];
            ntt_forward(c, PolyBatch{ej + (size_t)t.hi * N, (i64)es, n, m}, s);
        }
    }
    c.st_modup += n;
    return ext;
}

// Inner product + ModDown (C4 with the rounding correction R-MODDOWN: out = round(b / P)) for a list of
// requests at level L.
void Ev::ks_many(const std::vector<KsReq>& reqs, int L) {
    const int N = c.N, K = c.Kof(L), nl = L + K, dn = c.dnum(L);
    const int ML = keys->max_level, key_nl = ML + K;
    LimbMap klm;
    klm.n = nl;
    for (int e = 0; e < nl; e++) klm.mod[e] = (unsigned char)(e < L ? e : ML + (e - L));
    LimbMap pm; pm.n = K;
    for (int k = 0; k < K; k++) pm.mod[k] = (unsigned char)(c.L + k);
    LimbMap qm = c.qmap(L);
    std::vector<int> pos(L);
    for (int i = 0; i < L; i++) pos[i] = i;
    const ModDownTab& md = c.moddown[L];
    const int n_all = (int)reqs.size();
    for (int r0 = 0; r0 < n_all; r0 += KS_BATCH) {
        const int n = std::min(KS_BATCH, n_all - r0);
        u64* acc = sc.get((size_t)n * 2 * nl * N);
        KsInnerBatch B;
        OutBatch O;
        for (int i = 0; i < n; i++) {
            const KsReq& q = reqs[r0 + i];
            B.ext[i] = q.ext; B.key[i] = q.key; B.gather[i] = q.gather; B.acc[i] = acc + (size_t)i * 2 * nl * N;
            O.out[i][0] = q.out0; O.out[i][1] = q.out1; O.add[i][0] = q.add0; O.add[i][1] = q.add1;
        }
        k_ks_inner_batch(c, B, n, dn, nl, key_nl, klm, s);
        {   // [b]_P x vfac (NttPost): the BConv input
            const NttPost post{md.post.f, md.post.fsh, md.post.fd};
            ntt_inverse_scaled(c, PolyBatch{acc + (size_t)L * N, (i64)nl * N, 2 * n, pm}, false, s, nullptr, &post);
        }
        u64* y = sc.get((size_t)n * 2 * L * N);
        k_bconv_batch(c, acc + (size_t)L * N, (i64)nl * N, pm, md.d_vfac, md.d_vfac_sh, md.d_wfac, qm, y, (i64)L * N,
                      pos.data(), 2 * n, s, md.d_pmod, md.d_cfix, md.d_csh, md.d_wb, true);        // rounded: y = centred [b]_P
        std::vector<const u64*> esrc(2 * n), eadd(2 * n);
        std::vector<u64*> eout(2 * n);
        for (int i = 0; i < n; i++)
            for (int cc = 0; cc < 2; cc++) {
                esrc[2 * i + cc] = acc + ((size_t)i * 2 + cc) * nl * N;
                eout[2 * i + cc] = O.out[i][cc];
                eadd[2 * i + cc] = O.add[i][cc];
            }
        NttEpilogue E{upload(esrc), upload(eout), upload(eadd), md.d_pinv, md.d_pinv_sh};
        ntt_forward_epi(c, PolyBatch{y, (i64)L * N, 2 * n, qm}, &E, s);   // + (b - y) P^{-1} (+ add) fused
        c.st_ks += n;
    }
}

// Single (non-hoisted) rotations: sigma_g(c1) is ModUp'ed (gather fused into the ModUp copy), sigma_g(c0)
// is added in the ModDown epilogue.
void Ev::rotate_many(const std::vector<const DCt*>& ins, const std::vector<uint32_t>& gs, std::vector<DCt>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0]->L;
    std::vector<const u64*> c1;
    std::vector<uint32_t> g1;
    std::vector<int> idx;
    for (int i = 0; i < n; i++) {
        if (ins[i]->L != L || ins[i]->ncomp != 2) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "rotate_many: mixed levels");
        outs[i].L = L; outs[i].ncomp = 2; outs[i].scale = ins[i]->scale; outs[i].cstride = 0;
        if (gs[i] == 1u) { copy(*ins[i], outs[i]); continue; }
        c1.push_back(ins[i]->comp(1, N));
        g1.push_back(gs[i]);
        idx.push_back(i);
    }
    if (idx.empty()) return;
    const int m = (int)idx.size();
    const size_t Lw = (size_t)L * N;
    u64* c0g = sc.get(Lw * m);
    for (int i0 = 0; i0 < m; i0 += CP_BATCH) {
        int cnt = std::min(CP_BATCH, m - i0);
        CopyBatch cb;
        for (int i = 0; i < cnt; i++) { cb.src[i] = ins[idx[i0 + i]]->comp(0, N); cb.g[i] = g1[i0 + i]; }
        k_gather_copy(c, cb, cnt, c0g + Lw * i0, (i64)Lw, Lw, s);
    }
    u64* ext = modup_many(c1, g1, L);
    std::vector<KsReq> reqs(m);
    for (int i = 0; i < m; i++) {
        DCt& o = outs[idx[i]];
        reqs[i] = KsReq{ext + ext_stride(L) * i, key_for(g1[i], L), 1u, o.comp(0, N), o.comp(1, N), c0g + Lw * i, nullptr};
    }
    ks_many(reqs, L);
}

// Hoisted batches: ONE ModUp per input ciphertext, then the Galois gather of each requested element is
// fused into the inner product (SURVEY C4 hoisting; bits differ from rotate_many by design).
void Ev::hoisted_many(const std::vector<const DCt*>& ins, const std::vector<std::vector<uint32_t>>& gs,
                      std::vector<std::vector<DCt>>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0]->L;
    std::vector<const u64*> c1;
    std::vector<int> which;   // ModUp slot per input (-1: no rotation needed)
    for (int i = 0; i < n; i++) {
        if (ins[i]->L != L || ins[i]->ncomp != 2) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "hoisted_many: mixed levels");
        bool any = false;
        for (uint32_t g : gs[i]) any |= (g != 1u);
        which.push_back(any ? (int)c1.size() : -1);
        if (any) c1.push_back(ins[i]->comp(1, N));
    }
    u64* ext = c1.empty() ? nullptr : modup_many(c1, {}, L);
    const size_t Lw = (size_t)L * N;
    // sigma_g(c0) straight into the outputs' component 0 (added in the ModDown epilogue)
    std::vector<KsReq> reqs;
    std::vector<std::pair<const u64*, uint32_t>> c0s;
    std::vector<u64*> c0dst;
    for (int i = 0; i < n; i++) {
        for (size_t k = 0; k < gs[i].size(); k++) {
            DCt& o = outs[i][k];
            o.L = L; o.ncomp = 2; o.scale = ins[i]->scale; o.cstride = 0;
            if (gs[i][k] == 1u) { copy(*ins[i], o); continue; }
            c0s.push_back({ins[i]->comp(0, N), gs[i][k]});
            c0dst.push_back(o.comp(0, N));
            reqs.push_back(KsReq{ext + ext_stride(L) * which[i], key_for(gs[i][k], L), gs[i][k], o.comp(0, N), o.comp(1, N),
                                 o.comp(0, N), nullptr});
        }
    }
    if (reqs.empty()) return;
    // gather-copy c0 into a contiguous scratch then scatter-free: gather into dst pointers one batch at a time
    const int m = (int)c0s.size();
    u64* c0g = sc.get(Lw * m);
    for (int i0 = 0; i0 < m; i0 += CP_BATCH) {
        int cnt = std::min(CP_BATCH, m - i0);
        CopyBatch cb;
        for (int i = 0; i < cnt; i++) { cb.src[i] = c0s[i0 + i].first; cb.g[i] = c0s[i0 + i].second; }
        k_gather_copy(c, cb, cnt, c0g + Lw * i0, (i64)Lw, Lw, s);
    }
    for (int i = 0; i < m; i++) reqs[i].add0 = c0g + Lw * i;
    ks_many(reqs, L);
}

void Ev::relin_many(const std::vector<const DCt*>& ins, std::vector<DCt>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0]->L;
    std::vector<const u64*> d2;
    for (int i = 0; i < n; i++) {
        if (ins[i]->ncomp != 3 || ins[i]->L != L) throw EncfError(ENCF_ERR_FORMAT, "relinearize needs 3 components at one level");
        d2.push_back(ins[i]->comp(2, N));
    }
    const u64* key = key_for(0u, L);
    u64* ext = modup_many(d2, {}, L);
    std::vector<KsReq> reqs(n);
    for (int i = 0; i < n; i++) {
        DCt& o = outs[i];
        o.L = L; o.ncomp = 2; o.scale = ins[i]->scale; o.cstride = 0;
        reqs[i] = KsReq{ext + ext_stride(L) * i, key, 1u, o.comp(0, N), o.comp(1, N), ins[i]->comp(0, N), ins[i]->comp(1, N)};
    }
    ks_many(reqs, L);
}

// Rescale (C5) of a list of ciphertexts at one level: last limbs to coefficient form, correction per
// remaining limb, NTT of the correction, (c_i - corr_i) q_L^{-1}.
void Ev::rescale_many(const std::vector<const DCt*>& ins, std::vector<DCt>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0]->L;
    if (L <= 1) throw EncfError(ENCF_ERR_LEVEL_EXHAUSTED, "rescale at one limb");
    std::vector<const u64*> in_p;
    std::vector<u64*> out_p;
    for (int i = 0; i < n; i++) {
        if (ins[i]->L != L) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "rescale_many: mixed levels");
        outs[i].L = L - 1; outs[i].ncomp = ins[i]->ncomp; outs[i].scale = ins[i]->scale / (double)c.mods[L - 1];
        outs[i].cstride = 0;
        for (int cc = 0; cc < ins[i]->ncomp; cc++) { in_p.push_back(ins[i]->comp(cc, N)); out_p.push_back(outs[i].comp(cc, N)); }
    }
    const int P = (int)in_p.size();
    u64* last = sc.get((size_t)P * N);
    u64* corr = sc.get((size_t)P * (L - 1) * N);
    LimbMap lm; lm.n = 1; lm.mod[0] = (unsigned char)(L - 1);
    for (int p0 = 0; p0 < P; p0 += CP_BATCH) {
        int cnt = std::min(CP_BATCH, P - p0);
        CopyBatch cb;
        for (int i = 0; i < cnt; i++) { cb.src[i] = in_p[p0 + i] + (size_t)(L - 1) * N; cb.g[i] = 1u; }
        k_gather_copy(c, cb, cnt, last + (size_t)p0 * N, (i64)N, (size_t)N, s);
    }
    ntt_inverse(c, PolyBatch{last, (i64)N, P, lm}, s);
    k_rescale_prep_batch(c, last, corr, L, P, s);
    std::vector<const u64*> eadd(P, nullptr);
    const RescaleTab& rt = c.rescale[L];
    NttEpilogue E{upload(in_p), upload(out_p), upload(eadd), rt.d_inv, rt.d_inv_sh};
    ntt_forward_epi(c, PolyBatch{corr, (i64)(L - 1) * N, P, c.qmap(L - 1)}, &E, s);   // (c_i - corr_i) q_L^{-1} fused
}

// outs[o] = sum of terms[o] (each ct times an optional mask), all at level L with ncomp components.
void Ev::sum_many(const std::vector<std::vector<SumTerm>>& terms, int L, int ncomp, std::vector<DCt>& outs,
                  const std::vector<double>& scales) {
    const int n = (int)terms.size();
    if (n == 0) return;
    std::vector<SumDev> t;
    std::vector<int> off{0};
    std::vector<u64*> op;
    for (int o = 0; o < n; o++) {
        for (auto& x : terms[o]) t.push_back(SumDev{x.ct, x.mask});
        off.push_back((int)t.size());
        outs[o].L = L; outs[o].ncomp = ncomp; outs[o].scale = scales[o]; outs[o].cstride = 0;
        op.push_back(outs[o].d);
    }
    for (int o0 = 0; o0 < n; o0 += 32768) {
        int cnt = std::min(32768, n - o0);
        std::vector<int> off2(off.begin() + o0, off.begin() + o0 + cnt + 1);
        std::vector<u64*> op2(op.begin() + o0, op.begin() + o0 + cnt);
        k_sum_csr(c, upload(t), upload(off2), upload(op2), cnt, off2.back() - off2.front(), ncomp, L, s);
    }
}

void Ev::tensor_many(const std::vector<std::vector<std::pair<const DCt*, const DCt*>>>& pairs, std::vector<DCt>& outs) {
    const int n = (int)pairs.size();
    if (n == 0) return;
    const int L = pairs[0][0].first->L;
    std::vector<PairDev> t;
    std::vector<int> off{0};
    std::vector<u64*> op;
    for (int o = 0; o < n; o++) {
        double sc0 = pairs[o][0].first->scale * pairs[o][0].second->scale;
        for (auto& pr : pairs[o]) {
            if (pr.first->L != L || pr.second->L != L) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "tensor: level mismatch");
            if (pr.first->ncomp != 2 || pr.second->ncomp != 2) throw EncfError(ENCF_ERR_FORMAT, "tensor needs 2 components");
            check_scale(pr.first->scale * pr.second->scale, sc0);
            const i64 dflt = (i64)L * c.N;
            t.push_back(PairDev{pr.first->d, pr.second->d, pr.first->cstride ? pr.first->cstride : dflt,
                                pr.second->cstride ? pr.second->cstride : dflt});
        }
        off.push_back((int)t.size());
        outs[o].L = L; outs[o].ncomp = 3; outs[o].scale = sc0; outs[o].cstride = 0;
        op.push_back(outs[o].d);
    }
    k_tensor_csr(c, upload(t), upload(off), upload(op), n, (int)t.size(), L, s);
}

// ------------------------------------------------------------------------------------ single-item ops
void Ev::rotate_galois(const DCt& in, uint32_t g, DCt& out) {
    std::vector<DCt> o{out};
    rotate_many({&in}, {g}, o);
    out = o[0];
}

void Ev::rotate_hoisted(const DCt& in, const std::vector<uint32_t>& gs, std::vector<DCt>& outs) {
    std::vector<std::vector<DCt>> o{outs};
    hoisted_many({&in}, {gs}, o);
    outs = o[0];
}

void Ev::relin(const DCt& in, DCt& out) {
    std::vector<DCt> o{out};
    relin_many({&in}, o);
    out = o[0];
}

void Ev::rescale(const DCt& in, DCt& out) {
    std::vector<DCt> o{out};
    rescale_many({&in}, o);
    out = o[0];
}

void Ev::add(const DCt& a, const DCt& b, DCt& out, bool sub) {
    check_scale(a.scale, b.scale);
    if (a.L != b.L || a.ncomp != b.ncomp) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "add: level/component mismatch");
    k_add(c, a.d, b.d, out.d, a.ncomp, c.qmap(a.L), sub, s);
    out.L = a.L; out.ncomp = a.ncomp; out.scale = a.scale; out.cstride = 0;
}

void Ev::mul_i(const DCt& a, DCt& out) {
    k_mul_i(c, a.d, out.d, a.ncomp, c.qmap(a.L), s);
    out.L = a.L; out.ncomp = a.ncomp; out.scale = a.scale; out.cstride = 0;
}

void Ev::add_i_many(const std::vector<const DCt*>& a, const std::vector<const DCt*>& b, std::vector<DCt>& outs, bool sub) {
    const int n = (int)a.size();
    if ((int)b.size() != n || (int)outs.size() != n) throw EncfError(ENCF_ERR_ARG, "add_i_many: length mismatch");
    if (n == 0) return;
    const int L = a[0]->L, nc = a[0]->ncomp;
    for (int r = 0; r < n; r++) {
        check_scale(a[r]->scale, b[r]->scale);
        for (const DCt* x : {a[r], b[r]})
            if (x->L != L || x->ncomp != nc || (x->cstride != 0 && x->cstride != (i64)L * c.N))
                throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "add_i_many: level/component/layout mismatch");
    }
    for (int r0 = 0; r0 < n; r0 += ADDI_BATCH) {
        const int nb = std::min(ADDI_BATCH, n - r0);
        AddIBatch B;
        for (int r = 0; r < nb; r++) { B.a[r] = a[r0 + r]->d; B.b[r] = b[r0 + r]->d; B.out[r] = outs[r0 + r].d; }
        k_add_i_batch(c, B, nb, nc, c.qmap(L), sub, s);
    }
    for (int r = 0; r < n; r++) {
        outs[r].L = L; outs[r].ncomp = nc; outs[r].scale = a[r]->scale; outs[r].cstride = 0;
    }
}

void Ev::ptmul(const DCt& a, const u64* pt, double pt_scale, DCt& out) {
    const int N = c.N;
    k_mul(c, a.d, (i64)a.L * N, pt, 0, out.d, (i64)a.L * N, a.ncomp, c.qmap(a.L), s);
    out.L = a.L; out.ncomp = a.ncomp; out.scale = a.scale * pt_scale; out.cstride = 0;
    c.st_ptmul++;
}

void Ev::mod_drop(const DCt& in, int L, DCt& out) {
    if (L < 1 || L > in.L) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "mod_drop: bad level");
    const int N = c.N;
    CUDA_TRY(cudaMemcpy2DAsync(out.d, (size_t)L * N * 8, in.d, (size_t)in.L * N * 8, (size_t)L * N * 8, in.ncomp,
                               cudaMemcpyDeviceToDevice, s));
    out.L = L; out.ncomp = in.ncomp; out.scale = in.scale; out.cstride = 0;
}

void Ev::copy(const DCt& in, DCt& out) {
    k_copy(in.d, out.d, ct_words(in.L, in.ncomp), s);
    out.L = in.L; out.ncomp = in.ncomp; out.scale = in.scale; out.cstride = 0;
}

void Ev::tensor_sum(const std::vector<const DCt*>& A, const std::vector<const DCt*>& B, DCt& out3) {
    std::vector<std::pair<const DCt*, const DCt*>> pr;
    for (size_t i = 0; i < A.size(); i++) pr.push_back({A[i], B[i]});
    std::vector<DCt> o{out3};
    tensor_many({pr}, o);
    out3 = o[0];
}

void Ev::masked_sum(const std::vector<const DCt*>& C, const std::vector<const u64*>& M, double m_scale, DCt& out) {
    const int L = C[0]->L;
    double s0 = C[0]->scale * m_scale;
    std::vector<SumTerm> t;
    for (size_t i = 0; i < C.size(); i++) {
        if (C[i]->L != L) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "masked_sum: level mismatch");
        check_scale(C[i]->scale * m_scale, s0);
        t.push_back(SumTerm{C[i]->d, M[i]});
    }
    std::vector<DCt> o{out};
    sum_many({t}, L, 2, o, {s0});
    out = o[0];
}

// ------------------------------------------------------------------------------------ lazy (extended-basis) ops
std::vector<DCt> Ev::alloc_many_ext(int n, int L) {
    std::vector<DCt> v(n);
    if (n == 0) return v;
    const size_t w = (size_t)2 * (L + c.Kof(L)) * c.N;
    u64* base = sc.get(w * n);
    for (int i = 0; i < n; i++) { v[i].d = base + w * i; v[i].L = L; v[i].ncomp = 2; v[i].cstride = (i64)(L + c.Kof(L)) * c.N; }
    return v;
}

// Hoisted rotations kept in the extended basis: (P sigma_g(c0) + b0, b1) over Q_L u P, i.e. the inner
// product without its ModDown plus the lifted sigma_g(c0).
void Ev::hoisted_many_ext(const std::vector<const DCt*>& ins, const std::vector<std::vector<uint32_t>>& gs,
                          std::vector<std::vector<DCt>>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0]->L, K = c.Kof(L), nl = L + K, dn = c.dnum(L);
    std::vector<const u64*> c1;
    for (int i = 0; i < n; i++) {
        if (ins[i]->L != L || ins[i]->ncomp != 2) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "hoisted_many_ext: mixed levels");
        for (uint32_t g : gs[i]) if (g == 1u) throw EncfError(ENCF_ERR_ARG, "hoisted_many_ext: identity rotation");
        c1.push_back(ins[i]->comp(1, N));
    }
    u64* ext = modup_many(c1, {}, L);
    struct R { const u64* ext; const u64* key; uint32_t g; u64* out; const u64* c0; };
    std::vector<R> rq;
    for (int i = 0; i < n; i++)
        for (size_t k = 0; k < gs[i].size(); k++) {
            DCt& o = outs[i][k];
            o.L = L; o.ncomp = 2; o.scale = ins[i]->scale; o.cstride = (i64)nl * N;
            rq.push_back(R{ext + ext_stride(L) * i, key_for(gs[i][k], L), gs[i][k], o.d, ins[i]->comp(0, N)});
        }
    const int m = (int)rq.size();
    const int ML = keys->max_level, key_nl = ML + K;
    LimbMap klm;
    klm.n = nl;
    for (int e2 = 0; e2 < nl; e2++) klm.mod[e2] = (unsigned char)(e2 < L ? e2 : ML + (e2 - L));
    for (int r0 = 0; r0 < m; r0 += KS_BATCH) {
        const int cnt = std::min(KS_BATCH, m - r0);
        KsInnerBatch B;
        for (int i = 0; i < cnt; i++) {
            const R& q = rq[r0 + i];
            B.ext[i] = q.ext; B.key[i] = q.key; B.gather[i] = q.g; B.acc[i] = q.out;
            B.c0[i] = q.c0; B.g0[i] = q.g;   // + P sigma_g(c0) on the q-limbs, fused into the inner product
        }
        k_ks_inner_batch(c, B, cnt, dn, nl, key_nl, klm, s, c.moddown[L].d_pl, c.moddown[L].d_pl_sh);
        c.st_ks += cnt;      // a key switch whose ModDown is deferred (merged into a later moddown_rescale)
    }
}

void Ev::sum_many_ext(const std::vector<std::vector<SumTerm>>& terms, int L, std::vector<DCt>& outs,
                      const std::vector<double>& scales) {
    const int n = (int)terms.size();
    if (n == 0) return;
    std::vector<SumDev> t;
    std::vector<int> off{0};
    std::vector<u64*> op;
    for (int o = 0; o < n; o++) {
        for (auto& x : terms[o]) t.push_back(SumDev{x.ct, x.mask});
        off.push_back((int)t.size());
        outs[o].L = L; outs[o].ncomp = 2; outs[o].scale = scales[o]; outs[o].cstride = (i64)(L + c.Kof(L)) * c.N;
        op.push_back(outs[o].d);
    }
    LimbMap em = c.extmap(L);
    k_sum_csr(c, upload(t), upload(off), upload(op), n, (int)t.size(), 2, L + c.Kof(L), s, &em);
}

// round(x / (P q_{L-1})) mod Q_{L-1} for every extended ciphertext: limbs {q_{L-1}, p_*} to coefficient form,
// ONE rounded fast BConv to Q_{L-1}, forward NTT, (x_i - y_i) (P q_{L-1})^{-1}.
void Ev::moddown_rescale_many(const std::vector<DCt>& ins, std::vector<DCt>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0].L, K = c.Kof(L), nl = L + K;
    if (L < 2) throw EncfError(ENCF_ERR_LEVEL_EXHAUSTED, "moddown_rescale at one limb");
    const size_t w = (size_t)2 * nl * N;
    for (int i = 0; i < n; i++)
        if (ins[i].d != ins[0].d + w * i || ins[i].L != L) throw EncfError(ENCF_ERR_ARG, "moddown_rescale_many: inputs must be contiguous");
    u64* x = ins[0].d;
    LimbMap bm;
    bm.n = K + 1;
    bm.mod[0] = (unsigned char)(L - 1);
    for (int k = 0; k < K; k++) bm.mod[1 + k] = (unsigned char)(c.L + k);
    {
        const NttPost post{c.mdr[L].post.f, c.mdr[L].post.fsh, c.mdr[L].post.fd};   // x vfac: the BConv input
        ntt_inverse_scaled(c, PolyBatch{x + (size_t)(L - 1) * N, (i64)nl * N, 2 * n, bm}, false, s, nullptr, &post);
    }
    const MDRTab& t = c.mdr[L];
    LimbMap qm = c.qmap(L - 1);
    std::vector<int> pos(L - 1);
    for (int i = 0; i < L - 1; i++) pos[i] = i;
    u64* y = sc.get((size_t)n * 2 * (L - 1) * N);
    k_bconv_batch(c, x + (size_t)(L - 1) * N, (i64)nl * N, bm, t.d_vfac, t.d_vfac_sh, t.d_wfac, qm, y, (i64)(L - 1) * N,
                  pos.data(), 2 * n, s, t.d_corr, t.d_cfix, t.d_csh, t.d_wb, true);
    std::vector<const u64*> esrc(2 * n), eadd(2 * n, nullptr);
    std::vector<u64*> eout(2 * n);
    for (int i = 0; i < n; i++) {
        DCt& o = outs[i];
        o.L = L - 1; o.ncomp = 2; o.scale = ins[i].scale / (double)c.mods[L - 1]; o.cstride = 0;
        for (int cc = 0; cc < 2; cc++) {
            esrc[2 * i + cc] = x + w * i + (size_t)cc * nl * N;
            eout[2 * i + cc] = o.comp(cc, N);
        }
    }
    NttEpilogue E{upload(esrc), upload(eout), upload(eadd), t.d_inv, t.d_inv_sh};
    ntt_forward_epi(c, PolyBatch{y, (i64)(L - 1) * N, 2 * n, qm}, &E, s);   // (x - y) (P q_{L-1})^{-1} fused
}

// ModDown of extended ciphertexts (rounded, R-MODDOWN), no rescale.
void Ev::moddown_many(const std::vector<DCt>& ins, std::vector<DCt>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0].L, K = c.Kof(L), nl = L + K;
    const size_t w = (size_t)2 * nl * N;
    for (int i = 0; i < n; i++)
        if (ins[i].d != ins[0].d + w * i || ins[i].L != L) throw EncfError(ENCF_ERR_ARG, "moddown_many: inputs must be contiguous");
    u64* x = ins[0].d;
    LimbMap pm; pm.n = K;
    for (int k = 0; k < K; k++) pm.mod[k] = (unsigned char)(c.L + k);
    LimbMap qm = c.qmap(L);
    std::vector<int> pos(L);
    for (int i = 0; i < L; i++) pos[i] = i;
    const ModDownTab& md = c.moddown[L];
    {
        const NttPost post{md.post.f, md.post.fsh, md.post.fd};   // x vfac: the BConv input
        ntt_inverse_scaled(c, PolyBatch{x + (size_t)L * N, (i64)nl * N, 2 * n, pm}, false, s, nullptr, &post);
    }
    u64* y = sc.get((size_t)n * 2 * L * N);
    k_bconv_batch(c, x + (size_t)L * N, (i64)nl * N, pm, md.d_vfac, md.d_vfac_sh, md.d_wfac, qm, y, (i64)L * N, pos.data(), 2 * n, s,
                  md.d_pmod, md.d_cfix, md.d_csh, md.d_wb, true);
    std::vector<const u64*> esrc(2 * n), eadd(2 * n, nullptr);
    std::vector<u64*> eout(2 * n);
    for (int i = 0; i < n; i++) {
        DCt& o = outs[i];
        o.L = L; o.ncomp = 2; o.scale = ins[i].scale; o.cstride = 0;
        for (int cc = 0; cc < 2; cc++) {
            esrc[2 * i + cc] = x + w * i + (size_t)cc * nl * N;
            eout[2 * i + cc] = o.comp(cc, N);
        }
    }
    NttEpilogue E{upload(esrc), upload(eout), upload(eadd), md.d_pinv, md.d_pinv_sh};
    ntt_forward_epi(c, PolyBatch{y, (i64)L * N, 2 * n, qm}, &E, s);   // (x - y) P^{-1} fused
}

// Single (non-hoisted) key switches without ModDown: (P sigma_g(c0) + b0, b1) over Q_L u P.
void Ev::rotate_many_ext(const std::vector<const DCt*>& ins, const std::vector<uint32_t>& gs, std::vector<DCt>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0]->L, K = c.Kof(L), nl = L + K, dn = c.dnum(L);
    std::vector<const u64*> c1;
    for (int i = 0; i < n; i++) {
        if (ins[i]->L != L || ins[i]->ncomp != 2) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "rotate_many_ext: mixed levels");
        if (gs[i] == 1u) throw EncfError(ENCF_ERR_ARG, "rotate_many_ext: identity rotation (use lift_many)");
        c1.push_back(ins[i]->comp(1, N));
    }
    u64* ext = modup_many(c1, gs, L);                 // ModUp of sigma_g(c1): the gather is fused into the copy
    const int ML = keys->max_level, key_nl = ML + K;
    LimbMap klm;
    klm.n = nl;
    for (int e2 = 0; e2 < nl; e2++) klm.mod[e2] = (unsigned char)(e2 < L ? e2 : ML + (e2 - L));
    for (int r0 = 0; r0 < n; r0 += KS_BATCH) {
        const int cnt = std::min(KS_BATCH, n - r0);
        KsInnerBatch B;
        for (int i = 0; i < cnt; i++) {
            DCt& o = outs[r0 + i];
            o.L = L; o.ncomp = 2; o.scale = ins[r0 + i]->scale; o.cstride = (i64)nl * N;
            B.ext[i] = ext + ext_stride(L) * (r0 + i); B.key[i] = key_for(gs[r0 + i], L); B.gather[i] = 1u; B.acc[i] = o.d;
            B.c0[i] = ins[r0 + i]->comp(0, N); B.g0[i] = gs[r0 + i];   // + P sigma_g(c0), fused into the inner product
        }
        k_ks_inner_batch(c, B, cnt, dn, nl, key_nl, klm, s, c.moddown[L].d_pl, c.moddown[L].d_pl_sh);
        c.st_ks += cnt;
    }
}

void Ev::rotsum_many(const std::vector<const DCt*>& ins, const std::vector<uint32_t>& gs, std::vector<DCt>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0]->L, dn = c.dnum(L);
    std::vector<const u64*> c1;
    for (int i = 0; i < n; i++) {
        if (ins[i]->L != L || ins[i]->ncomp != 2) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "rotsum_many: mixed levels");
        check_scale(ins[i]->scale, ins[0]->scale);
        c1.push_back(ins[i]->comp(1, N));
    }
    for (uint32_t g : gs) if (g == 1u) throw EncfError(ENCF_ERR_ARG, "rotsum_many: identity rotation");
    if ((int)gs.size() > RS_TERMS) throw EncfError(ENCF_ERR_ARG, "rotsum_many: more than RS_TERMS shifts");
    u64* ext = modup_many(c1, {}, L);
    std::vector<DCt> acc = alloc_many_ext(n, L);
    for (int i = 0; i < n; i++) acc[i].scale = ins[i]->scale;
    const int key_nl = keys->max_level + c.Kof(L);
    for (int r0 = 0; r0 < n; r0 += KS_BATCH) {
        const int cnt = std::min(KS_BATCH, n - r0);
        RotSumBatch B;
        for (int i = 0; i < cnt; i++) {
            B.ext[i] = ext + ext_stride(L) * (r0 + i);
            B.c0[i] = ins[r0 + i]->comp(0, N);
            B.c1[i] = ins[r0 + i]->comp(1, N);
            B.acc[i] = acc[r0 + i].d;
        }
        for (size_t t = 0; t < gs.size(); t++) { B.key[t] = key_for(gs[t], L); B.g[t] = gs[t]; }
        k_ks_rotsum(c, B, cnt, (int)gs.size(), dn, L, key_nl, s);
    }
    c.st_ks += (uint64_t)n * gs.size();
    moddown_many(acc, outs);
}

// rescale(relin(ct)) rounded once (R-RELRS; oracle ckks.relinearize_ext + moddown_rescale): the relin key switch
// kept in the extended basis as (P d0 + b0, P d1 + b1), then ONE merged ModDown + rescale.
void Ev::relin_rescale_many(const std::vector<const DCt*>& ins, std::vector<DCt>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0]->L, K = c.Kof(L), nl = L + K, dn = c.dnum(L);
    std::vector<const u64*> d2;
    for (int i = 0; i < n; i++) {
        if (ins[i]->ncomp != 3 || ins[i]->L != L) throw EncfError(ENCF_ERR_FORMAT, "relinearize needs 3 components at one level");
        d2.push_back(ins[i]->comp(2, N));
    }
    const u64* key = key_for(0u, L);
    u64* ext = modup_many(d2, {}, L);
    std::vector<DCt> acc = alloc_many_ext(n, L);
    const int ML = keys->max_level, key_nl = ML + K;
    LimbMap klm;
    klm.n = nl;
    for (int e2 = 0; e2 < nl; e2++) klm.mod[e2] = (unsigned char)(e2 < L ? e2 : ML + (e2 - L));
    for (int r0 = 0; r0 < n; r0 += KS_BATCH) {
        const int cnt = std::min(KS_BATCH, n - r0);
        KsInnerBatch B;
        for (int i = 0; i < cnt; i++) {
            acc[r0 + i].scale = ins[r0 + i]->scale;
            B.ext[i] = ext + ext_stride(L) * (r0 + i); B.key[i] = key; B.gather[i] = 1u; B.acc[i] = acc[r0 + i].d;
            B.c0[i] = ins[r0 + i]->comp(0, N); B.c1[i] = ins[r0 + i]->comp(1, N); B.g0[i] = 1u;   // + P d0, P d1 (fused)
        }
        k_ks_inner_batch(c, B, cnt, dn, nl, key_nl, klm, s, c.moddown[L].d_pl, c.moddown[L].d_pl_sh);
        c.st_ks += cnt;
    }
    moddown_rescale_many(acc, outs);
}

void Ev::lift_many(const std::vector<const DCt*>& ins, std::vector<DCt>& outs) {
    const int n = (int)ins.size();
    if (n == 0) return;
    const int N = c.N, L = ins[0]->L, nl = L + c.Kof(L);
    for (int i = 0; i < n; i++) {
        DCt& o = outs[i];
        o.L = L; o.ncomp = 2; o.scale = ins[i]->scale; o.cstride = (i64)nl * N;
        CUDA_TRY(cudaMemsetAsync(o.d, 0, (size_t)2 * nl * N * 8, s));
    }
    for (int r0 = 0; r0 < 2 * n; r0 += CP_BATCH) {
        const int cnt = std::min(CP_BATCH, 2 * n - r0);
        CopyBatch dst, src;
        for (int i = 0; i < cnt; i++) {
            const int idx = (r0 + i) / 2, comp = (r0 + i) % 2;
            dst.src[i] = outs[idx].comp(comp, N); dst.g[i] = 1u;
            src.src[i] = ins[idx]->comp(comp, N); src.g[i] = 1u;
        }
        k_lift_add(c, dst, src, cnt, L, c.moddown[L].d_pl, c.moddown[L].d_pl_sh, s);
    }
}

// Mask plaintexts: cached per (descriptor, level, ext) in NTT form; encoded on the GPU on first use at
// scale q_{level-1} (ext: the same integer coefficients also reduced mod the special primes), unless a
// plaintext was installed with encf_mask_put (parity tests).
const u64* Ev::mask(int m, int r0, int r1, int s0, int ss, int scount, int level, int ext) {
    MaskKey key{m, r0, r1, s0, ss, scount, level, ext};
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.masks.find(key);
    if (it != c.masks.end()) return it->second;
    const int N = c.N, n = N / 2;
    std::vector<double> re(n, 0.0);
    for (int k = 0; k < scount; k++) {
        int sg = s0 + k * ss;
        for (int r = r0; r < r1; r++) re[(size_t)sg * m + r] = 1.0;
    }
    const LimbMap lm = ext ? c.extmap(level) : c.qmap(level);
    u64* pt = nullptr;
    CUDA_TRY(cudaMalloc(&pt, (size_t)lm.n * N * 8));
    Scratch tmp(s);
    double* dre = (double*)tmp.get(n);
    CUDA_TRY(cudaMemcpyAsync(dre, re.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    k_encode_slots(c, dre, nullptr, n, (double)c.mods[level - 1], level, pt, s, &lm);
    ntt_forward(c, PolyBatch{pt, 0, 1, lm}, s);
    c.masks[key] = pt;
    return pt;
}

const u64* Ev::keymask(uint32_t g, int m, int r0, int r1, int s0, int ss, int sc, int L, const u64** pm) {
    const int nl = L + c.Kof(L), dn = c.dnum(L);
    const size_t kmw = (size_t)dn * 2 * nl * c.N;
    KMKey key{keys->id, g, MaskKey{m, r0, r1, s0, ss, sc, L, 1}};
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.kmasks.find(key);
        if (it != c.kmasks.end()) { *pm = it->second + kmw; return it->second; }
    }
    const u64* mk = mask_ext(m, r0, r1, s0, ss, sc, L);
    const u64* kk = key_for(g, L);
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.kmasks.find(key);          // another thread may have built it meanwhile
    if (it != c.kmasks.end()) { *pm = it->second + kmw; return it->second; }
    u64* buf = nullptr;
    CUDA_TRY(cudaMalloc(&buf, (kmw + (size_t)nl * c.N) * 8));
    k_keymask(c, kk, keys->max_level + c.Kof(L), mk, dn, L, buf, s);
    c.kmasks[key] = buf;
    *pm = buf + kmw;
    return buf;
}
