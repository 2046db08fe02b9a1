// encformer.cu -- the EncFormer CKKS kernels as schedules over the sm_100a primitives:
//   projection (SCP pt-ct matmul),
//   score (folded-diagonal QK^T) + minimal export stream,
//   value (head-major PV),
//   complex C2M export, GPU half (Alg 3; trimming P:863-878).
// The schedules are exactly those of oracle/kernels.py (readings in DESIGN.md);
// the parity tests compare every limb of every output.
#include <cmath>
#include "encformer.cuh"

// ====================================================================================== projection
void proj_plan_init(encf_proj_plan& p, int n, int m, int d_in, int d_out, int C, int N1, uint32_t flags) {
    if (m <= 0 || n % m || d_in <= 0 || d_out <= 0) throw EncfError(ENCF_ERR_PLAN_SHAPE, "bad projection shape");
    p.n = n; p.m = m; p.d_in = d_in; p.d_out = d_out; p.flags = flags;
    p.N_seg = n / m;
    p.C = C > 0 ? C : p.N_seg;
    if (p.C > p.N_seg) throw EncfError(ENCF_ERR_PLAN_SHAPE, "C > n/m");
    p.G = (d_in + p.C - 1) / p.C;
    p.U = (p.G + 1) / 2;
    p.B_out = (d_out + p.C - 1) / p.C;
    if (N1 <= 0) {   // power of two dividing C nearest sqrt(B_out C / U) (G5)
        double target = std::sqrt((double)p.B_out * p.C / p.U);
        int best = 1;
        for (int q = 1; q <= p.C; q *= 2)
            if (p.C % q == 0 && std::fabs(std::log2((double)q) - std::log2(target)) < std::fabs(std::log2((double)best) - std::log2(target)) - 1e-12)
                best = q;
        N1 = best;
    }
    if (p.C % N1) throw EncfError(ENCF_ERR_PLAN_SHAPE, "N1 must divide C");
    p.N1 = N1;
    p.N2 = p.C / N1;
}

std::vector<uint32_t> proj_galois(Ev& ev, const encf_proj_plan& p) {
    std::vector<uint32_t> g;
    for (int q = 1; q < p.N1; q++) g.push_back(ev.galois_rot((long)q * p.m));
    for (int pp = 1; pp < p.N2; pp++) g.push_back(ev.galois_rot((long)pp * p.N1 * p.m));
    g.push_back(ev.galois_conj());
    return g;
}

// C6 steps 1-3 for units [u0, u1) (row-major over (b, p)); writes acc_b (level L) for every touched b
// into accs[b - b_first].  Step 1: hoisted baby-step bank.  Step 2: one fused MAC launch over the
// plaintext stream.  Step 3: giant-step single rotations and adds.
void proj_phase1(Ev& ev, const encf_proj_plan& p, const std::vector<DCt>& x, const u64* w, double w_scale, int u0,
                 int u1, std::vector<DCt>& accs) {
    const int N = ev.c.N, L = x[0].L, U = p.U, N1 = p.N1;
    for (auto& xi : x)
        if (xi.L != L) throw EncfError(ENCF_ERR_LEVEL_MISMATCH, "projection inputs at different levels");
    for (auto& xi : x) check_scale(xi.scale, x[0].scale);
    const size_t ctw = ev.ct_words(L);
    u64* bank = ev.sc.get(ctw * U * N1);
    for (int u = 0; u < U; u++) {
        std::vector<uint32_t> gs;
        std::vector<DCt> outs;
        for (int q = 0; q < N1; q++) {
            DCt o; o.d = bank + ctw * (u * N1 + q); o.L = L;
            outs.push_back(o);
            gs.push_back(q == 0 ? 1u : ev.galois_rot((long)q * p.m));
        }
        ev.rotate_hoisted(x[u], gs, outs);
    }
    const int units = u1 - u0;
    u64* cacc = ev.sc.get(ctw * units);
    const i64 wus = (i64)U * N1 * L * N;
    k_diag_mac(ev.c, bank, U * N1, w + (size_t)u0 * wus, units, wus, cacc, (i64)ctw, L, ev.s);
    const double sc = x[0].scale * w_scale;
    int b_first = u0 / p.N2, b_last = (u1 - 1) / p.N2;
    accs.assign(b_last - b_first + 1, DCt());
    std::vector<bool> init(accs.size(), false);
    DCt tmp = ev.alloc(L);
    for (int un = u0; un < u1; un++) {
        int b = un / p.N2, pp = un % p.N2;
        DCt cu; cu.d = cacc + ctw * (un - u0); cu.L = L; cu.scale = sc;
        DCt& a = accs[b - b_first];
        if (!init[b - b_first]) {
            a = ev.alloc(L, 2, sc);
            if (pp) ev.rotate_galois(cu, ev.galois_rot((long)pp * N1 * p.m), a);
            else ev.copy(cu, a);
            init[b - b_first] = true;
        } else {
            if (pp) { ev.rotate_galois(cu, ev.galois_rot((long)pp * N1 * p.m), tmp); ev.add(a, tmp, a); }
            else ev.add(a, cu, a);
        }
    }
}

// C6 steps 4-5: z = acc + conj(acc) (scale x2, G2/G3), y = rescale(z).
void proj_finalize(Ev& ev, const encf_proj_plan& p, const DCt& acc, DCt& y) {
    DCt z = ev.alloc(acc.L);
    if (p.flags & ENCF_PROJ_DECOMPLEXIFY) {
        ev.rotate_galois(acc, ev.galois_conj(), z);
        ev.add(acc, z, z);
        z.scale = acc.scale * 2.0;
    } else {
        ev.copy(acc, z);
    }
    ev.rescale(z, y);
}

// ====================================================================================== shifts (App. A.1)
// Psi^t for all t in ts from one hoisted ModUp of x (Alg A.2): rot(x,t)(.)h_t + rot(x,t-m)(.)u_t, rescale;
// t = 0: x(.)h_0, rescale.  Optional segment restriction [seg0, seg0+nseg).
void psi_hoisted(Ev& ev, const DCt& x, const std::vector<int>& ts, int m, int N_seg, int seg0, int nseg,
                 std::vector<DCt>& outs) {
    const int L = x.L;
    std::vector<int> tt;
    std::vector<uint32_t> gs;
    for (int t : ts) {
        int r = ((t % m) + m) % m;
        tt.push_back(r);
        if (r) { gs.push_back(ev.galois_rot(r)); gs.push_back(ev.galois_rot(r - m)); }
    }
    std::vector<DCt> rots(gs.size());
    for (auto& r : rots) r = ev.alloc(L);
    if (!gs.empty()) ev.rotate_hoisted(x, gs, rots);
    outs.resize(ts.size());
    size_t i = 0;
    const double ms = ev.mask_scale(L);
    for (size_t k = 0; k < tt.size(); k++) {
        int t = tt[k];
        const u64* hm = ev.mask(m, 0, m - t, seg0, 1, nseg, L);
        DCt y = ev.alloc(L);
        if (t == 0) {
            ev.masked_sum({&x}, {hm}, ms, y);
        } else {
            const u64* um = ev.mask(m, m - t, m, seg0, 1, nseg, L);
            ev.masked_sum({&rots[i], &rots[i + 1]}, {hm, um}, ms, y);
            i += 2;
        }
        outs[k] = ev.alloc(L - 1);
        ev.rescale(y, outs[k]);
    }
}

// ====================================================================================== attention plans
void attn_plan_init(encf_attn_plan& a, int n, int m, int H, int d_h, int C_qk, int beta, int H_blk) {
    if (m % 2) throw EncfError(ENCF_ERR_ODD_SEQ, "folded-diagonal packing needs even m");
    if (m <= 0 || n % m || H <= 0 || d_h <= 0) throw EncfError(ENCF_ERR_PLAN_SHAPE, "bad attention shape");
    a.n = n; a.m = m; a.H = H; a.d_h = d_h;
    a.N_seg = n / m;
    if (C_qk <= 0) {
        C_qk = H;
        while (C_qk * 2 <= a.N_seg && C_qk < H * d_h) C_qk *= 2;
    }
    if (C_qk % H || C_qk > a.N_seg) throw EncfError(ENCF_ERR_PLAN_SHAPE, "C_qk must be a multiple of H and <= n/m");
    a.C = C_qk;
    a.B = (H * d_h + C_qk - 1) / C_qk;
    if (beta <= 0) { beta = 1; while (beta * beta < m) beta *= 2; }
    a.beta = beta;
    if (m % beta || (m / beta) % 2) throw EncfError(ENCF_ERR_PLAN_SHAPE, "beta | m with g = m/beta even");
    a.g = m / beta;
    a.n_out = (int)(((long)H * m * m + 2L * n - 1) / (2L * n));
    a.seg_stride = std::max(d_h, m / 2);
    if (H_blk <= 0) H_blk = (d_h == m / 2) ? a.N_seg / d_h : 1;
    if (H_blk * a.seg_stride > a.N_seg) throw EncfError(ENCF_ERR_PLAN_SHAPE, "H_blk * stride > n/m");
    a.H_blk = H_blk;
    a.B_V = (H + H_blk - 1) / H_blk;
}

std::vector<uint32_t> attn_galois(Ev& ev, const encf_attn_plan& a) {
    std::vector<long> steps;
    const int m = a.m;
    for (int t = 1; t < m; t++) { steps.push_back(t); steps.push_back(t - m); }
    for (int d = -(a.d_h - 1); d < m / 2; d++) steps.push_back((long)d * m);
    for (int k = 1; k <= a.C / a.H; k *= 2) steps.push_back((long)k * a.H * m);
    for (int k = 1; k < a.C / a.H; k++) steps.push_back((long)k * a.H * m);
    const long seg = (long)a.H * m;
    for (int t = 0; t < m / 2; t++) steps.push_back(-((t * seg) % a.n));
    std::vector<uint32_t> g;
    for (long s : steps) {
        uint32_t x = ev.galois_rot(s);
        if (x != 1u && std::find(g.begin(), g.end(), x) == g.end()) g.push_back(x);
    }
    return g;
}

// out[h] = sum_{j<k} x[h + jH] by binary rotate-add (G7; oracle kernels.route).
static DCt route(Ev& ev, const DCt& x, int k, int H, int m) {
    DCt result, pw = x;
    bool have = false;
    int offset = 0, cnt = 1, kk = k;
    DCt tmp = ev.alloc(x.L);
    while (kk) {
        if (kk & 1) {
            DCt y;
            if (offset) { y = ev.alloc(x.L); ev.rotate_galois(pw, ev.galois_rot((long)offset * H * m), y); }
            else y = pw;
            if (!have) { result = ev.alloc(x.L); ev.copy(y, result); have = true; }
            else ev.add(result, y, result);
            offset += cnt;
        }
        kk >>= 1;
        if (kk) {
            DCt npw = ev.alloc(x.L);
            ev.rotate_galois(pw, ev.galois_rot((long)cnt * H * m), tmp);
            ev.add(pw, tmp, npw);
            pw = npw;
            cnt *= 2;
        }
    }
    return result;
}

// ====================================================================================== score (C7)
void score_run(Ev& ev, const encf_attn_plan& a, const std::vector<DCt>& qs, const std::vector<DCt>& ks, int t0, int t1,
               std::vector<DCt>& S) {
    const int m = a.m, H = a.H, beta = a.beta, g = a.g, Ns = a.N_seg;
    std::vector<std::vector<DCt>> qb(a.B);
    std::vector<std::vector<DCt>> kb(a.B);
    std::vector<int> qts, kts;
    for (int s = 0; s < beta; s++) qts.push_back(-s);
    for (int j = 0; j < g / 2; j++) kts.push_back(j * beta);
    for (int j = 0; j < g / 2; j++) kts.push_back(m / 2 + j * beta);
    for (int l = 0; l < a.B; l++) {
        psi_hoisted(ev, qs[l], qts, m, Ns, 0, Ns, qb[l]);
        psi_hoisted(ev, ks[l], kts, m, Ns, 0, Ns, kb[l]);
    }
    const int Lb = qb[0][0].L;
    S.resize(t1 - t0);
    for (int t = t0; t < t1; t++) {
        int j = t / beta, s = t % beta;
        std::vector<DCt> kc(a.B);
        std::vector<const DCt*> A, B;
        for (int l = 0; l < a.B; l++) {
            kc[l] = ev.alloc(Lb);
            DCt im = ev.alloc(Lb);
            ev.mul_i(kb[l][g / 2 + j], im);        // k_{m/2 + j beta}
            ev.add(kb[l][j], im, kc[l]);           // k_{j beta} + i k_{m/2 + j beta}
            A.push_back(&qb[l][s]);
            B.push_back(&kc[l]);
        }
        DCt T3 = ev.alloc(Lb, 3), T2 = ev.alloc(Lb), T = ev.alloc(Lb - 1);
        ev.tensor_sum(A, B, T3);
        ev.relin(T3, T2);
        ev.rescale(T2, T);
        DCt R = route(ev, T, a.C / H, H, m);
        std::vector<DCt> o;
        psi_hoisted(ev, R, {s}, m, Ns, 0, H, o);
        S[t - t0] = o[0];
    }
}

// Minimal export stream (oracle kernels.score_export).
void score_export_run(Ev& ev, const encf_attn_plan& a, const std::vector<DCt>& S, std::vector<DCt>& outs) {
    const int m = a.m, H = a.H, n = a.n;
    const long seg = (long)H * m;
    std::vector<std::vector<const DCt*>> terms(a.n_out);
    std::vector<std::vector<const u64*>> masks(a.n_out);
    std::vector<DCt> rots(S.size());
    const int L = S[0].L;
    for (size_t t = 0; t < S.size(); t++) {
        long start = (long)t * seg;
        long o = start % n;
        if (o) { rots[t] = ev.alloc(L); ev.rotate_galois(S[t], ev.galois_rot(-o), rots[t]); }
        else rots[t] = S[t];
        int k = (int)(start / n);
        long first = std::min(seg, n - o);
        terms[k].push_back(&rots[t]);
        masks[k].push_back(ev.mask(m, 0, m, (int)(o / m), 1, (int)(first / m), L));
        if (first < seg) {
            terms[k + 1].push_back(&rots[t]);
            masks[k + 1].push_back(ev.mask(m, 0, m, 0, 1, (int)((seg - first) / m), L));
        }
    }
    outs.resize(a.n_out);
    for (int k = 0; k < a.n_out; k++) {
        DCt y = ev.alloc(L);
        ev.masked_sum(terms[k], masks[k], ev.mask_scale(L), y);
        outs[k] = ev.alloc(L - 1);
        ev.rescale(y, outs[k]);
    }
}

// ====================================================================================== value (C8)
void value_run(Ev& ev, const encf_attn_plan& a, const std::vector<DCt>& ps, const std::vector<DCt>& vs,
               std::vector<DCt>& outs) {
    const int m = a.m, Ns = a.N_seg, half = m / 2;
    outs.resize(a.B_V);
    for (int l = 0; l < a.B_V; l++) {
        const DCt& v = vs[l];
        const DCt& p = ps[l];
        const int Lv = v.L;
        // 1. uu = v (.) e_all - i (rot(v, m/2)(.)h + rot(v, -m/2)(.)u), one rescale
        std::vector<DCt> rv = {ev.alloc(Lv), ev.alloc(Lv)};
        ev.rotate_hoisted(v, {ev.galois_rot(half), ev.galois_rot(half - m)}, rv);
        const double ms = ev.mask_scale(Lv);
        DCt sh = ev.alloc(Lv), shi = ev.alloc(Lv), ve = ev.alloc(Lv), d = ev.alloc(Lv);
        ev.masked_sum({&rv[0], &rv[1]}, {ev.mask(m, 0, m - half, 0, 1, Ns, Lv), ev.mask(m, m - half, m, 0, 1, Ns, Lv)}, ms, sh);
        ev.masked_sum({&v}, {ev.mask(m, 0, m, 0, 1, Ns, Lv)}, ms, ve);
        ev.mul_i(sh, shi);
        ev.add(ve, shi, d, /*sub=*/true);
        DCt uu = ev.alloc(Lv - 1);
        ev.rescale(d, uu);
        // 2. U bank u_t = Psi^t(uu)
        std::vector<int> ts;
        for (int t = 0; t < half; t++) ts.push_back(t);
        std::vector<DCt> ub;
        psi_hoisted(ev, uu, ts, m, Ns, 0, Ns, ub);
        // 3. Phi bank of p_fd, delta in [-(d_h-1), m/2-1]
        const int dmin = -(a.d_h - 1);
        std::vector<uint32_t> gs;
        for (int dd = dmin; dd < half; dd++) if (dd) gs.push_back(ev.galois_rot((long)dd * m));
        std::vector<DCt> pbv(gs.size());
        for (auto& x : pbv) x = ev.alloc(p.L);
        ev.rotate_hoisted(p, gs, pbv);
        auto pb = [&](int dd) -> const DCt* {
            if (dd == 0) return &p;
            int idx = dd - dmin - (dd > 0 ? 1 : 0);
            return &pbv[idx];
        };
        // 4. b_t = sum_u Phi^{t-u}(p) (.) n_u, rescale
        const int Lp = p.L;
        std::vector<const u64*> nmask(a.d_h);
        for (int u = 0; u < a.d_h; u++) nmask[u] = ev.mask(m, 0, m, u, a.seg_stride, a.H_blk, Lp);
        std::vector<DCt> bt(half);
        for (int t = 0; t < half; t++) {
            std::vector<const DCt*> C;
            for (int u = 0; u < a.d_h; u++) C.push_back(pb(t - u));
            DCt y = ev.alloc(Lp);
            ev.masked_sum(C, nmask, ev.mask_scale(Lp), y);
            bt[t] = ev.alloc(Lp - 1);
            ev.rescale(y, bt[t]);
        }
        // 5. o = sum_t u_t (x) b_t, one relin, rescale
        const int Lb = bt[0].L;
        std::vector<DCt> ud(half);
        std::vector<const DCt*> A, B;
        for (int t = 0; t < half; t++) {
            if (ub[t].L > Lb) { ud[t] = ev.alloc(Lb); ev.mod_drop(ub[t], Lb, ud[t]); }
            else ud[t] = ub[t];
            A.push_back(&ud[t]);
            B.push_back(&bt[t]);
        }
        DCt o3 = ev.alloc(Lb, 3), o2 = ev.alloc(Lb);
        ev.tensor_sum(A, B, o3);
        ev.relin(o3, o2);
        outs[l] = ev.alloc(Lb - 1);
        ev.rescale(o2, outs[l]);
    }
}

// ====================================================================================== export (Alg 3 GPU half)
int l_conv_rule(const encf_ctx& c, int ell, int sigma, double scale, double B_max) {
    double lg = 0.0;
    for (int L = 1; L <= c.L; L++) {
        lg += std::log2((double)c.mods[L - 1]);
        if (lg >= ell + sigma + 1 && std::exp2(lg) / 2 > scale * B_max) return L;
    }
    return -1;
}
