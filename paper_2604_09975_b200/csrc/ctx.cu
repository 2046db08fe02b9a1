// ctx.cu -- context creation: modulus constants, NTT twiddles, base-conversion and rescale tables.
// All constants are computed on the host with exact 128-bit modular arithmetic (no big integers
// are needed: every CRT factor is a product of primes reduced modulo a single prime).
#include <cstring>
#include <cstdlib>
#include "ctx.cuh"

static thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }
const char* encf_last_error_impl() { return g_last_error.c_str(); }

void* encf_ctx::dev_alloc(size_t bytes) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes ? bytes : 8);
    if (e != cudaSuccess) throw EncfError(ENCF_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    allocations.push_back(p);
    return p;
}

static u64* upload(encf_ctx& c, const std::vector<u64>& v) {
    u64* d = (u64*)c.dev_alloc(v.size() * sizeof(u64));
    CUDA_TRY(cudaMemcpy(d, v.data(), v.size() * sizeof(u64), cudaMemcpyHostToDevice));
    return d;
}

// Base-conversion matrix wf ([na][nt], Montgomery form, targets tq) as the byte matrix of the tensor-core path
// (poly.cu bconv_tc_kernel): W'[i][a][t] = 2^{8a} wf[i][t] mod q_t, byte b of it at row n = 8 t + b, K byte kk = 8 i + a,
// in the canonical K-major no-swizzle layout [kk / 16][n][kk % 16]; nb = 8 x (nt rounded up to even) rows, inputs
// i >= na (and the padding target) are zero.  Returns null when the shape does not fit (na > 8 or nt > 32).
static uint8_t* bconv_wbytes(encf_ctx& c, const std::vector<u64>& wf, int na, int nt, const std::vector<u64>& tq) {
    if (na > 8 || nt > 32 || na < 1 || nt < 1) return nullptr;
    const int nb = 8 * ((nt + 1) & ~1);
    std::vector<uint8_t> wb((size_t)nb * 64, 0);
    for (int i = 0; i < na; i++)
        for (int a = 0; a < 8; a++)
            for (int t = 0; t < nt; t++) {
                const u64 wp = h_mulmod(wf[(size_t)i * nt + t], h_powmod(2, 8 * a, tq[t]), tq[t]);
                for (int b = 0; b < 8; b++) {
                    const int n = 8 * t + b, kk = 8 * i + a;
                    wb[(size_t)(kk / 16) * nb * 16 + (size_t)n * 16 + kk % 16] = (uint8_t)(wp >> (8 * b));
                }
            }
    uint8_t* d = (uint8_t*)c.dev_alloc(wb.size());
    CUDA_TRY(cudaMemcpy(d, wb.data(), wb.size(), cudaMemcpyHostToDevice));
    return d;
}

// Per-limb iNTT output factors f (u64 + Shoup quotient + FP64 {f, fl(f/q)}): ntt_inverse_scaled(.., NttPost) multiplies
// its output by them, so the fast base conversion that follows reads [x (Q/q_i)^{-1} N^{-1}]_{q_i} directly.
static NttPostTab make_post(encf_ctx& c, const std::vector<u64>& f, const std::vector<u64>& q) {
    NttPostTab t;
    std::vector<u64> fs(f.size());
    std::vector<double> fd(2 * f.size());
    for (size_t i = 0; i < f.size(); i++) {
        fs[i] = shoup_pre(f[i], q[i]);
        fd[2 * i] = (double)f[i];
        fd[2 * i + 1] = (double)f[i] / (double)q[i];
    }
    t.f = upload(c, f);
    t.fsh = upload(c, fs);
    t.fd = (double*)c.dev_alloc(fd.size() * 8);
    CUDA_TRY(cudaMemcpy(t.fd, fd.data(), fd.size() * 8, cudaMemcpyHostToDevice));
    return t;
}

static int bitrev(int x, int bits) {
    int r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

static bool is_prime_u64(u64 n) {   // deterministic Miller-Rabin for 64-bit
    if (n < 2) return false;
    for (u64 p : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
        if (n % p == 0) return n == p;
    }
    u64 d = n - 1; int r = 0;
    while ((d & 1) == 0) { d >>= 1; r++; }
    for (u64 a : {2ull, 325ull, 9375ull, 28178ull, 450775ull, 9780504ull, 1795265022ull}) {
        u64 x = h_powmod(a % n, d, n);
        if (a % n == 0 || x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int i = 1; i < r; i++) { x = h_mulmod(x, x, n); if (x == n - 1) { comp = false; break; } }
        if (comp) return false;
    }
    return true;
}

// A primitive 2N-th root of unity: g^((q-1)/2N) for the first g with psi^N = -1.
static u64 find_psi(u64 q, int N) {
    for (u64 g = 2; g < 100000; g++) {
        u64 r = h_powmod(g, (q - 1) / (2 * (u64)N), q);
        if (h_powmod(r, (u64)N, q) == q - 1) return r;
    }
    throw EncfError(ENCF_ERR_ARG, "no primitive 2N-th root");
}

static void build(encf_ctx& c, const encf_params* p) {
    c.N = p->N;
    c.logN = 0;
    while ((1 << c.logN) < c.N) c.logN++;
    if ((1 << c.logN) != c.N || c.logN < 4 || c.logN > 16) throw EncfError(ENCF_ERR_ARG, "N must be a power of two in [2^4, 2^16]");
    c.L = p->L; c.K = p->K; c.alpha = p->alpha;
    if (c.L < 1 || c.K < 1 || c.alpha < 1 || c.L + c.K > MAX_MODS || c.alpha > 16)
        throw EncfError(ENCF_ERR_ARG, "bad L/K/alpha");
    // K(L): special primes of a key switch at level L (DESIGN.md R-KL); NULL = all K at every level
    c.Kl.assign(c.L + 1, c.K);
    if (p->K_of_level) {
        for (int l = 1; l <= c.L; l++) {
            const int k = p->K_of_level[l - 1];
            if (k < 1 || k > c.K || (l > 1 && k < c.Kl[l - 1]))
                throw EncfError(ENCF_ERR_ARG, "K_of_level must be non-decreasing in [1, K]");
            c.Kl[l] = k;
        }
    }
    c.Kl[0] = c.Kl[1];
    c.s1 = c.logN / 2;
    c.s2 = c.logN - c.s1;
    c.mods.assign(p->q, p->q + c.L);
    c.mods.insert(c.mods.end(), p->p, p->p + c.K);
    for (u64 q : c.mods) {
        if (q >= (1ull << 61) || (q - 1) % (2 * (u64)c.N) != 0 || !is_prime_u64(q))
            throw EncfError(ENCF_ERR_ARG, "every modulus must be a prime < 2^61 with q = 1 mod 2N");
    }
    const int M = (int)c.mods.size(), N = c.N;
    for (u64 q : c.mods) c.max_mod = std::max(c.max_mod, q);
    {
        // The fused key-switch inner products (ks_inner: dnum products, ks_psi: 2 dnum + 2, ks_rma: dnum per term)
        // sum products below q^2 in 128 bits and reduce ONCE with a Montgomery REDC, which needs the sum < q 2^64,
        // i.e. (2 dnum + 2) q < 2^64 at the top level.  Refuse parameter sets outside that range.
        const unsigned __int128 terms = 2 * (unsigned __int128)((c.L + c.alpha - 1) / c.alpha) + 2;
        if (terms * c.max_mod >= ((unsigned __int128)1 << 64))
            throw EncfError(ENCF_ERR_ARG, "(2 dnum + 2) q_max >= 2^64: digit count too large for the single-REDC inner products");
    }
    for (u64 q : c.mods) {
        c.mont_R.push_back(h_mont_R(q));
        c.mont_Rinv.push_back(h_invmod(h_mont_R(q), q));
    }
    auto mont = [&](u64 w, u64 q) { return h_mulmod(w, h_mont_R(q), q); };   // base-conversion constants in Montgomery form
    std::vector<ModConst> mc(M);
    std::vector<u64> psi(M * (size_t)N), psi_sh(M * (size_t)N), ipsi(M * (size_t)N), ipsi_sh(M * (size_t)N);
    std::vector<u64> ninv(M), ninv_sh(M), im(M), im_sh(M);
    c.psi.resize(M);
    for (int i = 0; i < M; i++) {
        u64 q = c.mods[i];
        mc[i].q = q;
        mc[i].two_q = 2 * q;
        mc[i].qinv = h_neg_inv64(q);
        h_ratio128(q, mc[i].rhi, mc[i].rlo);
        u64 ps = find_psi(q, N), ips = h_invmod(ps, q);
        c.psi[i] = ps;
        // powers psi^k, psi^-k for k < N, then scatter to bit-reversed positions
        std::vector<u64> pw(N), ipw(N);
        pw[0] = 1; ipw[0] = 1;
        for (int k = 1; k < N; k++) { pw[k] = h_mulmod(pw[k - 1], ps, q); ipw[k] = h_mulmod(ipw[k - 1], ips, q); }
        for (int k = 0; k < N; k++) {
            int br = bitrev(k, c.logN);
            size_t o = (size_t)i * N + k;
            psi[o] = pw[br];
            psi_sh[o] = shoup_pre(pw[br], q);
            ipsi[o] = ipw[br];
            ipsi_sh[o] = shoup_pre(ipw[br], q);
        }
        ninv[i] = h_invmod((u64)N % q, q);
        ninv_sh[i] = shoup_pre(ninv[i], q);
        im[i] = h_powmod(ps, (u64)N / 2, q);   // psi^{N/2}: X^{N/2} evaluates to +-im at every NTT point
        im_sh[i] = shoup_pre(im[i], q);
    }
    c.d_mod = (ModConst*)c.dev_alloc(M * sizeof(ModConst));
    CUDA_TRY(cudaMemcpy(c.d_mod, mc.data(), M * sizeof(ModConst), cudaMemcpyHostToDevice));
    c.d_psi = upload(c, psi); c.d_psi_sh = upload(c, psi_sh);
    c.d_ipsi = upload(c, ipsi); c.d_ipsi_sh = upload(c, ipsi_sh);
    {   // interleaved {w, w'} pairs: one 128-bit load per twiddle in the NTT kernels
        std::vector<u64> f(2 * psi.size()), iv(2 * psi.size());
        for (size_t i = 0; i < psi.size(); i++) {
            f[2 * i] = psi[i]; f[2 * i + 1] = psi_sh[i];
            iv[2 * i] = ipsi[i]; iv[2 * i + 1] = ipsi_sh[i];
        }
        c.d_tw2 = upload(c, f);
        c.d_itw2 = upload(c, iv);
        // FP64 path tables (exact integer doubles; w/q rounded to nearest by the host division)
        std::vector<double> ff(2 * psi.size()), fi(2 * psi.size()), fpc(4 * (size_t)M);
        for (size_t i = 0; i < psi.size(); i++) {
            const double q = (double)c.mods[i / N];
            ff[2 * i] = (double)psi[i]; ff[2 * i + 1] = (double)psi[i] / q;
            fi[2 * i] = (double)ipsi[i]; fi[2 * i + 1] = (double)ipsi[i] / q;
        }
        for (int i = 0; i < M; i++) {
            const double q = (double)c.mods[i];
            fpc[4 * i] = q; fpc[4 * i + 1] = 1.0 / q;
            fpc[4 * i + 2] = (double)ninv[i]; fpc[4 * i + 3] = (double)ninv[i] / q;
            if (c.mods[i] < (1ull << 41) && !std::getenv("ENCF_NTT_INT_ONLY")) c.fpmask |= 1ull << i;
        }
        c.d_twf = (double*)c.dev_alloc(ff.size() * 8);
        c.d_itwf = (double*)c.dev_alloc(fi.size() * 8);
        c.d_fpc = (double*)c.dev_alloc(fpc.size() * 8);
        CUDA_TRY(cudaMemcpy(c.d_twf, ff.data(), ff.size() * 8, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(c.d_itwf, fi.data(), fi.size() * 8, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(c.d_fpc, fpc.data(), fpc.size() * 8, cudaMemcpyHostToDevice));
    }
    c.d_ninv = upload(c, ninv); c.d_ninv_sh = upload(c, ninv_sh);
    c.d_imag = upload(c, im); c.d_imag_sh = upload(c, im_sh);

    // ModUp tables per (level, digit) -- SURVEY §8c C4: d~_{j,t} = sum_{i in j} [d_i (Q_j/q_i)^{-1}]_{q_i} (Q_j/q_i) mod t
    c.modup.assign(c.L + 1, {});
    c.moddown.assign(c.L + 1, {});
    c.rescale.assign(c.L + 1, {});
    c.mdr.assign(c.L + 1, {});
    c.modup_post.assign(c.L + 1, {});
    for (int lev = 1; lev <= c.L; lev++) {
        LimbMap ext = c.extmap(lev);
        for (int j = 0; j < c.dnum(lev); j++) {
            ModUpTab t;
            t.lo = j * c.alpha;
            t.hi = std::min((j + 1) * c.alpha, lev);
            t.tgt.n = 0;
            for (int e = 0; e < ext.n; e++) {
                if (e >= t.lo && e < t.hi) continue;
                t.tgt.mod[t.tgt.n++] = ext.mod[e];
                t.tgt_pos.push_back(e);
            }
            int na = t.hi - t.lo;
            std::vector<u64> vf(na), vfs(na), wf((size_t)na * t.tgt.n);
            for (int a = 0; a < na; a++) {
                u64 qi = c.mods[t.lo + a];
                u64 prod = 1;   // Q_j / q_i mod q_i
                for (int b = 0; b < na; b++) if (b != a) prod = h_mulmod(prod, c.mods[t.lo + b] % qi, qi);
                vf[a] = h_mulmod(h_invmod(prod, qi), ninv[t.lo + a], qi);   // x N^{-1}: the iNTT in front skips it
                vfs[a] = shoup_pre(vf[a], qi);
                for (int k = 0; k < t.tgt.n; k++) {
                    u64 tq = c.mods[t.tgt.mod[k]];
                    u64 pr = 1;
                    for (int b = 0; b < na; b++) if (b != a) pr = h_mulmod(pr, c.mods[t.lo + b] % tq, tq);
                    wf[(size_t)a * t.tgt.n + k] = mont(pr, tq);
                }
            }
            t.d_vfac = upload(c, vf); t.d_vfac_sh = upload(c, vfs); t.d_wfac = upload(c, wf);
            {
                std::vector<u64> tq(t.tgt.n);
                for (int k = 0; k < t.tgt.n; k++) tq[k] = c.mods[t.tgt.mod[k]];
                t.d_wb = bconv_wbytes(c, wf, na, t.tgt.n, tq);
            }
            c.modup[lev].push_back(t);
        }
        {   // every q-limb's ModUp input factor (its digit's vfac) for the ModUp iNTT epilogue
            std::vector<u64> f(lev), q(lev);
            for (int j = 0; j < c.dnum(lev); j++) {
                const ModUpTab& t = c.modup[lev][j];
                std::vector<u64> vf(t.hi - t.lo);
                CUDA_TRY(cudaMemcpy(vf.data(), t.d_vfac, vf.size() * 8, cudaMemcpyDeviceToHost));
                for (int a = t.lo; a < t.hi; a++) { f[a] = vf[a - t.lo]; q[a] = c.mods[a]; }
            }
            c.modup_post[lev] = make_post(c, f, q);
        }
        // ModDown: y = fastBConv_{P->Q}([b]_P); out_i = (b_i - y_i) P^{-1} mod q_i, P = P_{K(lev)} (R-KL)
        const int Kl = c.Kof(lev);
        ModDownTab md;
        std::vector<u64> vf(Kl), vfs(Kl), wf((size_t)Kl * lev), pinv(lev), pinvs(lev);
        for (int k = 0; k < Kl; k++) {
            u64 pk = c.mods[c.L + k];
            u64 prod = 1;
            for (int b = 0; b < Kl; b++) if (b != k) prod = h_mulmod(prod, c.mods[c.L + b] % pk, pk);
            vf[k] = h_mulmod(h_invmod(prod, pk), ninv[c.L + k], pk);      // x N^{-1} (iNTT without it)
            vfs[k] = shoup_pre(vf[k], pk);
            for (int i = 0; i < lev; i++) {
                u64 qi = c.mods[i];
                u64 pr = 1;
                for (int b = 0; b < Kl; b++) if (b != k) pr = h_mulmod(pr, c.mods[c.L + b] % qi, qi);
                wf[(size_t)k * lev + i] = mont(pr, qi);
            }
        }
        for (int i = 0; i < lev; i++) {
            u64 qi = c.mods[i], P = 1;
            for (int k = 0; k < Kl; k++) P = h_mulmod(P, c.mods[c.L + k] % qi, qi);
            pinv[i] = h_invmod(P, qi);
            pinvs[i] = shoup_pre(pinv[i], qi);
        }
        md.d_vfac = upload(c, vf); md.d_vfac_sh = upload(c, vfs); md.d_wfac = upload(c, wf);
        md.d_wb = bconv_wbytes(c, wf, Kl, lev, std::vector<u64>(c.mods.begin(), c.mods.begin() + lev));
        md.post = make_post(c, vf, std::vector<u64>(c.mods.begin() + c.L, c.mods.begin() + c.L + Kl));
        md.d_pinv = upload(c, pinv); md.d_pinv_sh = upload(c, pinvs);
        std::vector<u64> pmod(lev);
        for (int i = 0; i < lev; i++) {
            u64 qi = c.mods[i], P = 1;
            for (int k = 0; k < Kl; k++) P = h_mulmod(P, c.mods[c.L + k] % qi, qi);
            pmod[i] = mont(P ? qi - P : 0, qi);      // stored negated: the kernel adds r * (q_i - P mod q_i)
        }
        md.d_pmod = upload(c, pmod);
        std::vector<u64> cfix(Kl), csh(Kl);
        for (int k = 0; k < Kl; k++) {
            u64 pk = c.mods[c.L + k];
            csh[k] = 63 - (64 - __builtin_clzll(pk));
            cfix[k] = (u64)(((unsigned __int128)1 << (123 - csh[k])) / pk);
        }
        md.d_cfix = upload(c, cfix);
        md.d_csh = upload(c, csh);
        std::vector<u64> pl(lev), pls(lev);
        for (int i = 0; i < lev; i++) {
            u64 qi = c.mods[i], P = 1;
            for (int k = 0; k < Kl; k++) P = h_mulmod(P, c.mods[c.L + k] % qi, qi);
            pl[i] = P; pls[i] = shoup_pre(P, qi);
        }
        md.d_pl = upload(c, pl); md.d_pl_sh = upload(c, pls);
        c.moddown[lev] = md;
        // Merged ModDown + rescale (R-LAZY): B' = {q_{lev-1}, p_0..p_{K-1}} -> q_0..q_{lev-2}
        if (lev >= 2) {
            std::vector<u64> bp;
            bp.push_back(c.mods[lev - 1]);
            for (int k = 0; k < Kl; k++) bp.push_back(c.mods[c.L + k]);
            const int nb = (int)bp.size(), nt = lev - 1;
            std::vector<u64> vf(nb), vfs(nb), wf((size_t)nb * nt), corr(nt), cf(nb), cs(nb), inv(nt), invs(nt);
            for (int a = 0; a < nb; a++) {
                u64 ba = bp[a], prod = 1;
                for (int b2 = 0; b2 < nb; b2++) if (b2 != a) prod = h_mulmod(prod, bp[b2] % ba, ba);
                const int mid = a == 0 ? lev - 1 : c.L + (a - 1);
                vf[a] = h_mulmod(h_invmod(prod, ba), ninv[mid], ba); vfs[a] = shoup_pre(vf[a], ba);   // x N^{-1}
                for (int t = 0; t < nt; t++) {
                    u64 qt = c.mods[t], pr = 1;
                    for (int b2 = 0; b2 < nb; b2++) if (b2 != a) pr = h_mulmod(pr, bp[b2] % qt, qt);
                    wf[(size_t)a * nt + t] = mont(pr, qt);
                }
                cs[a] = 63 - (64 - __builtin_clzll(ba));
                cf[a] = (u64)(((unsigned __int128)1 << (123 - cs[a])) / ba);
            }
            for (int t = 0; t < nt; t++) {
                u64 qt = c.mods[t], B = 1;
                for (int b2 = 0; b2 < nb; b2++) B = h_mulmod(B, bp[b2] % qt, qt);
                corr[t] = mont(B ? qt - B : 0, qt);
                inv[t] = h_invmod(B, qt); invs[t] = shoup_pre(inv[t], qt);
            }
            MDRTab mt;
            mt.d_vfac = upload(c, vf); mt.d_vfac_sh = upload(c, vfs); mt.d_wfac = upload(c, wf); mt.d_corr = upload(c, corr);
            mt.d_wb = bconv_wbytes(c, wf, nb, nt, std::vector<u64>(c.mods.begin(), c.mods.begin() + nt));
            mt.post = make_post(c, vf, bp);
            mt.d_cfix = upload(c, cf); mt.d_csh = upload(c, cs); mt.d_inv = upload(c, inv); mt.d_inv_sh = upload(c, invs);
            c.mdr[lev] = mt;
        }
        // Rescale (C5) dropping q_{lev-1}
        if (lev >= 2) {
            RescaleTab rt;
            u64 qL = c.mods[lev - 1], h = qL / 2;
            std::vector<u64> inv(lev - 1), invs(lev - 1), hm(lev - 1);
            for (int i = 0; i < lev - 1; i++) {
                u64 qi = c.mods[i];
                inv[i] = h_invmod(qL % qi, qi);
                invs[i] = shoup_pre(inv[i], qi);
                hm[i] = h % qi;
            }
            rt.d_inv = upload(c, inv); rt.d_inv_sh = upload(c, invs); rt.d_hmod = upload(c, hm);
            c.rescale[lev] = rt;
        }
    }
    // rotation group 5^j mod 2N (encode / decode)
    c.rot_group.resize(N / 2);
    u64 x = 1;
    for (int j = 0; j < N / 2; j++) { c.rot_group[j] = (int)x; x = x * 5 % (2 * (u64)N); }
    c.d_rot_group = (int*)c.dev_alloc(sizeof(int) * (N / 2));
    CUDA_TRY(cudaMemcpy(c.d_rot_group, c.rot_group.data(), sizeof(int) * (N / 2), cudaMemcpyHostToDevice));
}

encf_status ctx_create_impl(const encf_params* params, int device, encf_ctx** out) {
    if (!params || !out || !params->q || !params->p) return ENCF_ERR_ARG;
    encf_ctx* c = new encf_ctx();
    try {
        c->device = device;
        CUDA_TRY(cudaSetDevice(device));
        // keep stream-ordered scratch cached in the device pool across synchronisations (the default
        // release threshold of 0 would unmap and re-map multi-GB scratch at every sync)
        cudaMemPool_t pool;
        CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = ~0ull;
        CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        build(*c, params);
        *out = c;
        return ENCF_OK;
    } catch (const EncfError& e) {
        set_last_error(e.msg);
        for (void* p : c->allocations) cudaFree(p);
        delete c;
        return e.code;
    }
}

encf_status ctx_destroy_impl(encf_ctx* c) {
    if (!c) return ENCF_ERR_ARG;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto& kv : c->masks) cudaFree(kv.second);
    for (auto& kv : c->kmasks) cudaFree(kv.second);
    for (auto& kv : c->bhat) cudaFree(kv.second);
    for (void* p : c->allocations) cudaFree(p);
    for (void* p : c->pinned) cudaFreeHost(p);
    delete c;
    return ENCF_OK;
}

void* encf_ctx::pinned_persistent(size_t bytes) {
    std::lock_guard<std::mutex> lk(mu);
    bytes = (bytes + 255) & ~(size_t)255;
    if (pinned.empty() || pin_used + bytes > pin_cap) {
        const size_t cap = std::max(bytes, (size_t)8 << 20);
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;   // host allocation is legal mid-capture
        CUDA_TRY(cudaThreadExchangeStreamCaptureMode(&mode));
        void* p = nullptr;
        cudaError_t e = cudaHostAlloc(&p, cap, cudaHostAllocDefault);
        CUDA_TRY(cudaThreadExchangeStreamCaptureMode(&mode));
        if (e != cudaSuccess) throw EncfError(ENCF_ERR_OOM, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
        pinned.push_back(p);
        pin_used = 0;
        pin_cap = cap;
    }
    void* r = (char*)pinned.back() + pin_used;
    pin_used += bytes;
    return r;
}

// Under CUDA-graph capture a plain cudaEventRecord only orders the capture; the EXTERNAL flag makes it an
// event-record node that fires at every replay (timing-capable), so captured steps keep their live timing.
static cudaError_t record_event(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaError_t err = cudaStreamIsCapturing(s, &st);
    if (err != cudaSuccess) return err;
    if (st == cudaStreamCaptureStatusActive) return cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    return cudaEventRecord(e, s);
}

cudaEvent_t encf_ctx::prof_event() {
    if (!ev_pool.empty()) { cudaEvent_t e = ev_pool.back(); ev_pool.pop_back(); return e; }
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    return e;
}

void encf_ctx::prof_begin(const char* name, cudaStream_t s, uint64_t bytes, int& slot) {
    slot = -1;
    if (!prof) return;
    if (!prof_all) {   // comma-separated list of kernel names
        const std::string n(name);
        size_t pos = 0;
        bool hit = false;
        while (pos <= prof_only.size()) {
            size_t e = prof_only.find(',', pos);
            if (e == std::string::npos) e = prof_only.size();
            if (prof_only.compare(pos, e - pos, n) == 0 && e - pos == n.size()) { hit = true; break; }
            pos = e + 1;
        }
        if (!hit) return;
    }
    std::lock_guard<std::mutex> lk(mu);
    ProfRec r{name, prof_event(), prof_event(), bytes};
    CUDA_TRY(record_event(r.a, s));
    prof_recs.push_back(r);
    slot = (int)prof_recs.size() - 1;
}

void encf_ctx::prof_end(int slot, cudaStream_t s) {
    if (slot < 0) return;
    std::lock_guard<std::mutex> lk(mu);
    CUDA_TRY(record_event(prof_recs[slot].b, s));
}

extern "C" encf_status encf_profile_enable(encf_ctx* c, const char* which) {
    if (!c) return ENCF_ERR_ARG;
    std::lock_guard<std::mutex> lk(c->mu);
    c->prof = which != nullptr;
    c->prof_all = which && std::string(which) == "*";
    c->prof_only = which ? which : "";
    return ENCF_OK;
}

static encf_status profile_collect(encf_ctx* c, const char* kernel, double* total_ms, uint64_t* launches,
                                   uint64_t* alg_bytes, bool forget) {
    if (!c || !kernel || !total_ms || !launches || !alg_bytes) return ENCF_ERR_ARG;
    try {
        std::lock_guard<std::mutex> lk(c->mu);
        double ms = 0.0;
        uint64_t n = 0, by = 0;
        std::vector<encf_ctx::ProfRec> keep;
        for (auto& r : c->prof_recs) {
            if (r.name != kernel) { keep.push_back(r); continue; }
            CUDA_TRY(cudaEventSynchronize(r.b));
            float t = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
            ms += t; n++; by += r.bytes;
            if (forget) {
                c->ev_pool.push_back(r.a);
                c->ev_pool.push_back(r.b);
            } else {
                keep.push_back(r);
            }
        }
        c->prof_recs = keep;
        *total_ms = ms; *launches = n; *alg_bytes = by;
        return ENCF_OK;
    } catch (const EncfError& e) {
        set_last_error(e.msg);
        return e.code;
    }
}

extern "C" encf_status encf_profile_read(encf_ctx* c, const char* kernel, double* total_ms, uint64_t* launches,
                                         uint64_t* alg_bytes) {
    return profile_collect(c, kernel, total_ms, launches, alg_bytes, true);
}

extern "C" encf_status encf_profile_peek(encf_ctx* c, const char* kernel, double* total_ms, uint64_t* launches,
                                         uint64_t* alg_bytes) {
    return profile_collect(c, kernel, total_ms, launches, alg_bytes, false);
}
