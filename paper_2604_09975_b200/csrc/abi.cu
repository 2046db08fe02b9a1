#include <atomic>
// abi.cu -- extern "C" entry points of libencf (include/encf.h).  Host-side validation happens before
// any launch; C++ exceptions never cross the boundary.
#include <cstring>
#include "encformer.cuh"

encf_status ctx_create_impl(const encf_params* params, int device, encf_ctx** out);
encf_status ctx_destroy_impl(encf_ctx* c);
const char* encf_last_error_impl();

namespace {

template <class F>
encf_status guard(F&& f) {
    try {
        f();
        return ENCF_OK;
    } catch (const EncfError& e) {
        set_last_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return ENCF_ERR_ARG;
    }
}

inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

void need(bool cond, encf_status code, const char* msg) {
    if (!cond) throw EncfError(code, msg);
}

void level_ok(const encf_ctx* c, int L) { need(L >= 1 && L <= c->L, ENCF_ERR_LEVEL_MISMATCH, "n_limbs out of range"); }

// Every ciphertext entering the library is validated here, before any launch: non-null context and data, NTT form,
// 2 or 3 components, 1 <= n_limbs <= L_max (qmap() / the per-level tables are indexed by it), 16-byte aligned
// data (the vectorised kernels use 128-bit accesses).
DCt view(const encf_ctx* ctx, const encf_ct* c) {
    need(ctx != nullptr, ENCF_ERR_ARG, "null context");
    need(c && c->data, ENCF_ERR_ARG, "null ciphertext");
    need(c->ntt == 1, ENCF_ERR_FORMAT, "homomorphic ops need NTT-form ciphertexts (ntt = 1)");
    need(((uintptr_t)c->data & 15) == 0, ENCF_ERR_ARG, "ciphertext data must be 16-byte aligned");
    DCt d;
    d.d = c->data; d.ncomp = c->n_comp; d.L = c->n_limbs; d.scale = c->scale;
    need(d.ncomp == 2 || d.ncomp == 3, ENCF_ERR_FORMAT, "n_comp must be 2 or 3");
    level_ok(ctx, d.L);
    return d;
}

DCt outview(encf_ct* o, int L, int ncomp) {
    need(o && o->data, ENCF_ERR_ARG, "null output");
    need(((uintptr_t)o->data & 15) == 0, ENCF_ERR_ARG, "output data must be 16-byte aligned");
    DCt d; d.d = o->data; d.L = L; d.ncomp = ncomp; return d;
}

void writeback(encf_ct* o, const DCt& d) {
    o->n_comp = d.ncomp; o->n_limbs = d.L; o->scale = d.scale; o->ntt = 1;
}

}  // namespace

extern "C" {

const char* encf_status_string(encf_status s) {
    switch (s) {
        case ENCF_OK: return "ok";
        case ENCF_ERR_ARG: return "invalid argument";
        case ENCF_ERR_LENGTH_MISMATCH: return "length mismatch";
        case ENCF_ERR_SCALE_MISMATCH: return "scale mismatch";
        case ENCF_ERR_LEVEL_MISMATCH: return "level mismatch";
        case ENCF_ERR_LEVEL_EXHAUSTED: return "level exhausted";
        case ENCF_ERR_PLAN_SHAPE: return "plan shape mismatch";
        case ENCF_ERR_ODD_SEQ: return "odd sequence length";
        case ENCF_ERR_FORMAT: return "format mismatch";
        case ENCF_ERR_OVERFLOW: return "overflow";
        case ENCF_ERR_CONFIG: return "configuration violation";
        case ENCF_ERR_MISSING_KEY: return "missing key";
        case ENCF_ERR_WORKSPACE: return "workspace too small";
        case ENCF_ERR_OOM: return "out of memory";
        case ENCF_ERR_CUDA: return "CUDA error";
    }
    return "unknown";
}

const char* encf_last_error(void) { return encf_last_error_impl(); }

encf_status encf_ctx_create(const encf_params* params, int device, encf_ctx** out) { return ctx_create_impl(params, device, out); }
encf_status encf_ctx_destroy(encf_ctx* ctx) { return ctx_destroy_impl(ctx); }

encf_status encf_stats(encf_ctx* c, encf_counters* o) {
    if (!c || !o) return ENCF_ERR_ARG;
    o->keyswitch = c->st_ks; o->modup = c->st_modup; o->limb_ntt = c->st_ntt; o->ptmul_terms = c->st_ptmul;
    o->ctmul = c->st_ctmul; o->kernel_launches = c->st_launch; o->alg_bytes = c->st_bytes; o->limb_ntt_fp64 = c->st_ntt_fp;
    return ENCF_OK;
}

encf_status encf_stats_reset(encf_ctx* c) {
    if (!c) return ENCF_ERR_ARG;
    c->st_ks = 0; c->st_modup = 0; c->st_ntt = 0; c->st_ptmul = 0; c->st_ctmul = 0; c->st_launch = 0; c->st_bytes = 0; c->st_ntt_fp = 0;
    return ENCF_OK;
}

uint32_t encf_galois_rot(encf_ctx* c, int32_t steps) {
    long n = c->N / 2;
    long r = ((steps % n) + n) % n;
    return (uint32_t)h_powmod(5, (u64)r, 2 * (u64)c->N);
}
uint32_t encf_galois_conj(encf_ctx* c) { return 2u * c->N - 1u; }

// ------------------------------------------------------------------------------------ keys
encf_status encf_keygen(encf_ctx* c, uint64_t seed, const uint32_t* galois, int32_t n_galois, uint32_t flags,
                        int32_t max_level, encf_keys** out, void* stream) {
    return guard([&] {
        need(c && out && (n_galois == 0 || galois), ENCF_ERR_ARG, "keygen: null argument");
        level_ok(c, max_level);
        cudaStream_t s = S(stream);
        // keys of the top class K(max_level) (R-KL); lower classes are derived on first use (Ev::key_for)
        const int N = c->N, ML = max_level, K = c->Kof(ML), nl = ML + K;
        encf_keys* k = new encf_keys();
        static std::atomic<uint64_t> next_id{1};
        k->id = next_id++;
        k->max_level = ML;
        k->dnum = c->dnum(ML);
        k->device = c->device;
        k->ctx = c;
        auto alloc = [&](size_t words) { void* p; CUDA_TRY(cudaMalloc(&p, words * 8)); k->allocations.push_back(p); return (u64*)p; };
        LimbMap em = c->extmap(ML);
        std::vector<int> gids(nl);
        for (int i = 0; i < ML; i++) gids[i] = i;
        for (int i = 0; i < K; i++) gids[ML + i] = c->L + i;   // global limb id of p_k = L_max + k
        // secret key (stream 0x01 << 56), ternary
        k->sk = alloc((size_t)nl * N);
        k_sample_small(*c, seed, 0x01ull << 56, 0, k->sk, em, s);
        ntt_forward(*c, PolyBatch{k->sk, 0, 1, em}, s);
        std::vector<uint32_t> targets(galois, galois + n_galois);
        if (flags & ENCF_KEY_RELIN) targets.push_back(0u);
        Scratch sc(s);
        u64* sp = sc.get((size_t)nl * N);
        u64* tmp = sc.get((size_t)nl * N);
        u64* dR = sc.get(nl);
        u64* dRs = sc.get(nl);
        {
            std::vector<u64> r(nl), rs(nl);
            for (int e = 0; e < nl; e++) { u64 q = c->mods[em.mod[e]]; r[e] = c->mont_R[em.mod[e]]; rs[e] = shoup_pre(r[e], q); }
            CUDA_TRY(cudaMemcpyAsync(dR, r.data(), nl * 8, cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(dRs, rs.data(), nl * 8, cudaMemcpyHostToDevice, s));
        }
        for (uint32_t g : targets) {
            need(g == 0u || (g & 1u), ENCF_ERR_ARG, "galois elements must be odd");
            if (k->ksk.count(g)) continue;
            if (g == 0u) k_mul(*c, k->sk, 0, k->sk, 0, sp, 0, 1, em, s);            // s^2
            else k_automorph(*c, k->sk, 0, sp, 0, 1, nl, g % (2u * N), s);          // sigma_g(s)
            u64* key = alloc((size_t)k->dnum * 2 * nl * N);
            for (int j = 0; j < k->dnum; j++) {
                u64* b = key + (size_t)j * 2 * nl * N;
                u64* a = b + (size_t)nl * N;
                u64 st_a = (0x02ull << 56) | ((u64)g << 16) | ((u64)j << 8) | 0ull;
                u64 st_e = (0x02ull << 56) | ((u64)g << 16) | ((u64)j << 8) | 1ull;
                k_sample_uniform(*c, seed, st_a, a, em, gids.data(), s);
                ntt_forward(*c, PolyBatch{a, 0, 1, em}, s);
                k_sample_small(*c, seed, st_e, 1, b, em, s);
                ntt_forward(*c, PolyBatch{b, 0, 1, em}, s);
                k_mul(*c, a, 0, k->sk, 0, tmp, 0, 1, em, s);
                k_add(*c, b, tmp, b, 1, em, true, s);                                // e - a s
                // + g_j s' with g_j = P mod q_i on digit j's q-limbs
                int lo = j * c->alpha, hi = std::min((j + 1) * c->alpha, ML);
                std::vector<u64> pm(hi - lo), pms(hi - lo);
                for (int i = lo; i < hi; i++) {
                    u64 qi = c->mods[i], P = 1;
                    for (int kk = 0; kk < K; kk++) P = h_mulmod(P, c->mods[c->L + kk] % qi, qi);
                    pm[i - lo] = P; pms[i - lo] = shoup_pre(P, qi);
                }
                u64* dp = sc.get(pm.size());
                u64* dps = sc.get(pm.size());
                CUDA_TRY(cudaMemcpyAsync(dp, pm.data(), pm.size() * 8, cudaMemcpyHostToDevice, s));
                CUDA_TRY(cudaMemcpyAsync(dps, pms.data(), pms.size() * 8, cudaMemcpyHostToDevice, s));
                LimbMap dm; dm.n = hi - lo;
                for (int i = lo; i < hi; i++) dm.mod[i - lo] = (unsigned char)i;
                k_copy(sp + (size_t)lo * N, tmp, (size_t)(hi - lo) * N, s);
                k_scalar_mul(*c, tmp, 1, dm, dp, dps, s);
                k_add(*c, b + (size_t)lo * N, tmp, b + (size_t)lo * N, 1, dm, false, s);
            }
            k_scalar_mul(*c, key, k->dnum * 2, em, dR, dRs, s);   // stored in Montgomery form (ks_inner REDC)
            k->ksk[g] = key;
        }
        CUDA_TRY(cudaStreamSynchronize(s));
        *out = k;
    });
}

encf_status encf_keys_destroy(encf_keys* k) {
    if (!k) return ENCF_ERR_ARG;
    cudaSetDevice(k->device);
    cudaDeviceSynchronize();
    if (k->ctx) {   // evict this key set's pre-masked keys from the context cache (they would otherwise leak)
        std::lock_guard<std::mutex> lk(k->ctx->mu);
        for (auto it = k->ctx->kmasks.begin(); it != k->ctx->kmasks.end();) {
            if (it->first.keys_id == k->id) { cudaFree(it->second); it = k->ctx->kmasks.erase(it); }
            else ++it;
        }
    }
    for (void* p : k->allocations) cudaFree(p);
    delete k;
    return ENCF_OK;
}

encf_status encf_keys_size(encf_ctx* c, const encf_keys* k, int32_t which, size_t* words) {
    if (!c || !k || !words) return ENCF_ERR_ARG;
    size_t nl = (size_t)k->max_level + c->Kof(k->max_level);
    *words = which == 0 ? nl * c->N : (size_t)k->dnum * 2 * nl * c->N;
    return ENCF_OK;
}

encf_status encf_keys_export(encf_ctx* c, const encf_keys* k, int32_t which, uint32_t galois, uint64_t* out, void* stream) {
    return guard([&] {
        need(c && k && out, ENCF_ERR_ARG, "keys_export: null argument");
        cudaStream_t s = S(stream);
        const int nl = k->max_level + c->Kof(k->max_level);
        LimbMap em = c->extmap(k->max_level);
        if (which == 0) {
            k_copy(k->sk, out, (size_t)nl * c->N, s);
            ntt_inverse(*c, PolyBatch{out, 0, 1, em}, s);
        } else {
            auto it = k->ksk.find(galois);
            need(it != k->ksk.end(), ENCF_ERR_MISSING_KEY, "keys_export: no such key");
            k_copy(it->second, out, (size_t)k->dnum * 2 * nl * c->N, s);
            {   // out of Montgomery form
                Scratch sc(s);
                u64* dR = sc.get(nl);
                u64* dRs = sc.get(nl);
                std::vector<u64> r(nl), rs(nl);
                for (int e = 0; e < nl; e++) { u64 q = c->mods[em.mod[e]]; r[e] = c->mont_Rinv[em.mod[e]]; rs[e] = shoup_pre(r[e], q); }
                CUDA_TRY(cudaMemcpyAsync(dR, r.data(), nl * 8, cudaMemcpyHostToDevice, s));
                CUDA_TRY(cudaMemcpyAsync(dRs, rs.data(), nl * 8, cudaMemcpyHostToDevice, s));
                k_scalar_mul(*c, out, k->dnum * 2, em, dR, dRs, s);
                CUDA_TRY(cudaStreamSynchronize(s));
            }
            ntt_inverse(*c, PolyBatch{out, (i64)nl * c->N, k->dnum * 2, em}, s);
        }
    });
}

// ------------------------------------------------------------------------------------ enc / dec / encode
encf_status encf_encrypt_sk(encf_ctx* c, const encf_keys* k, const encf_pt* pt, uint64_t seed, encf_ct* out, void* stream) {
    return guard([&] {
        need(c && k && pt && pt->data && out && out->data, ENCF_ERR_ARG, "encrypt: null argument");
        const int L = pt->n_limbs, N = c->N;
        level_ok(c, L);
        need(L <= k->max_level, ENCF_ERR_LEVEL_MISMATCH, "encrypt: level above key");
        cudaStream_t s = S(stream);
        Scratch sc(s);
        LimbMap qm = c->qmap(L);
        u64* c0 = out->data;
        u64* c1 = out->data + (size_t)L * N;
        std::vector<int> gids(L);
        for (int i = 0; i < L; i++) gids[i] = i;
        k_sample_uniform(*c, seed, (0x03ull << 56) | 0ull, c1, qm, gids.data(), s);
        ntt_forward(*c, PolyBatch{c1, 0, 1, qm}, s);
        u64* m = sc.get((size_t)L * N);
        k_copy(pt->data, m, (size_t)L * N, s);
        if (!pt->ntt) ntt_forward(*c, PolyBatch{m, 0, 1, qm}, s);
        u64* e = sc.get((size_t)L * N);
        k_sample_small(*c, seed, (0x03ull << 56) | 1ull, 1, e, qm, s);
        ntt_forward(*c, PolyBatch{e, 0, 1, qm}, s);
        k_mul(*c, c1, 0, k->sk, 0, c0, 0, 1, qm, s);            // a s
        k_add(*c, e, c0, c0, 1, qm, true, s);                   // e - a s
        k_add(*c, c0, m, c0, 1, qm, false, s);                  // + m
        out->n_comp = 2; out->n_limbs = L; out->scale = pt->scale; out->ntt = 1;
    });
}

encf_status encf_decrypt(encf_ctx* c, const encf_keys* k, const encf_ct* ct, encf_pt* out, void* stream) {
    return guard([&] {
        need(c && k && out && out->data, ENCF_ERR_ARG, "decrypt: null argument");
        DCt x = view(c, ct);
        const int L = x.L, N = c->N;
        need(L <= k->max_level, ENCF_ERR_LEVEL_MISMATCH, "decrypt: level above key");
        cudaStream_t s = S(stream);
        Scratch sc(s);
        LimbMap qm = c->qmap(L);
        u64* t = sc.get((size_t)L * N);
        k_mul(*c, x.comp(1, N), 0, k->sk, 0, t, 0, 1, qm, s);
        k_add(*c, x.comp(0, N), t, out->data, 1, qm, false, s);
        if (x.ncomp == 3) {
            u64* s2 = sc.get((size_t)L * N);
            k_mul(*c, k->sk, 0, k->sk, 0, s2, 0, 1, qm, s);
            k_mul(*c, x.comp(2, N), 0, s2, 0, t, 0, 1, qm, s);
            k_add(*c, out->data, t, out->data, 1, qm, false, s);
        }
        out->n_limbs = L; out->scale = x.scale; out->ntt = 1;
    });
}

encf_status encf_encode(encf_ctx* c, const double* re, const double* im, int32_t n_slots, int32_t n_limbs, double scale,
                        encf_pt* out, void* stream) {
    return guard([&] {
        need(c && re && out && out->data, ENCF_ERR_ARG, "encode: null argument");
        need(n_slots >= 0 && n_slots <= c->N / 2, ENCF_ERR_LENGTH_MISMATCH, "encode: more slots than n");
        level_ok(c, n_limbs);
        cudaStream_t s = S(stream);
        Scratch sc(s);
        double* dre = (double*)sc.get(n_slots + 1);
        double* dim = im ? (double*)sc.get(n_slots + 1) : nullptr;
        CUDA_TRY(cudaMemcpyAsync(dre, re, n_slots * sizeof(double), cudaMemcpyHostToDevice, s));
        if (im) CUDA_TRY(cudaMemcpyAsync(dim, im, n_slots * sizeof(double), cudaMemcpyHostToDevice, s));
        k_encode_slots(*c, dre, dim, n_slots, scale, n_limbs, out->data, s);
        ntt_forward(*c, PolyBatch{out->data, 0, 1, c->qmap(n_limbs)}, s);
        out->n_limbs = n_limbs; out->scale = scale; out->ntt = 1;
    });
}

encf_status encf_decode(encf_ctx* c, const encf_pt* pt, double* re, double* im, void* stream) {
    return guard([&] {
        need(c && pt && pt->data && re && im, ENCF_ERR_ARG, "decode: null argument");
        cudaStream_t s = S(stream);
        Scratch sc(s);
        const int N = c->N, n = N / 2;
        u64* l0 = sc.get(N);
        k_copy(pt->data, l0, N, s);
        if (pt->ntt) { LimbMap m; m.n = 1; m.mod[0] = 0; ntt_inverse(*c, PolyBatch{l0, 0, 1, m}, s); }
        double* dre = (double*)sc.get(n);
        double* dim = (double*)sc.get(n);
        k_decode_limb0(*c, l0, pt->scale, dre, dim, s);
        CUDA_TRY(cudaMemcpyAsync(re, dre, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(im, dim, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    });
}

// ------------------------------------------------------------------------------------ primitives
encf_status encf_poly_to_ntt(encf_ctx* c, uint64_t* d, int32_t np, int32_t nl, void* stream) {
    return guard([&] {
        need(c && d && np >= 0, ENCF_ERR_ARG, "to_ntt: bad argument");
        level_ok(c, nl);
        ntt_forward(*c, PolyBatch{d, (i64)nl * c->N, np, c->qmap(nl)}, S(stream));
    });
}

encf_status encf_poly_from_ntt(encf_ctx* c, uint64_t* d, int32_t np, int32_t nl, void* stream) {
    return guard([&] {
        need(c && d && np >= 0, ENCF_ERR_ARG, "from_ntt: bad argument");
        level_ok(c, nl);
        ntt_inverse(*c, PolyBatch{d, (i64)nl * c->N, np, c->qmap(nl)}, S(stream));
    });
}

#define EV_BEGIN(keys)            \
    need(c != nullptr, ENCF_ERR_ARG, "null context"); \
    cudaStream_t s = S(stream);   \
    Scratch sc(s);                \
    Ev ev(*c, keys, s, sc);

encf_status encf_add(encf_ctx* c, const encf_ct* a, const encf_ct* b, encf_ct* out, void* stream) {
    return guard([&] { EV_BEGIN(nullptr); DCt x = view(c, a), y = view(c, b); DCt o = outview(out, x.L, x.ncomp); ev.add(x, y, o); writeback(out, o); });
}
encf_status encf_sub(encf_ctx* c, const encf_ct* a, const encf_ct* b, encf_ct* out, void* stream) {
    return guard([&] { EV_BEGIN(nullptr); DCt x = view(c, a), y = view(c, b); DCt o = outview(out, x.L, x.ncomp); ev.add(x, y, o, true); writeback(out, o); });
}
encf_status encf_mul_i(encf_ctx* c, const encf_ct* a, encf_ct* out, void* stream) {
    return guard([&] { EV_BEGIN(nullptr); DCt x = view(c, a); DCt o = outview(out, x.L, x.ncomp); ev.mul_i(x, o); writeback(out, o); });
}
encf_status encf_ptmul(encf_ctx* c, const encf_ct* a, const encf_pt* w, encf_ct* out, void* stream) {
    return guard([&] {
        EV_BEGIN(nullptr);
        DCt x = view(c, a);
        need(w && w->data && w->ntt == 1, ENCF_ERR_FORMAT, "ptmul needs an NTT-form plaintext");
        need(w->n_limbs == x.L, ENCF_ERR_LEVEL_MISMATCH, "ptmul: level mismatch");
        DCt o = outview(out, x.L, x.ncomp);
        ev.ptmul(x, w->data, w->scale, o);
        writeback(out, o);
    });
}
encf_status encf_tensor(encf_ctx* c, const encf_ct* a, const encf_ct* b, encf_ct* out3, void* stream) {
    return guard([&] {
        EV_BEGIN(nullptr);
        DCt x = view(c, a), y = view(c, b);
        need(x.ncomp == 2 && y.ncomp == 2, ENCF_ERR_FORMAT, "tensor needs 2-component inputs");
        need(x.L == y.L, ENCF_ERR_LEVEL_MISMATCH, "tensor: level mismatch");
        DCt o = outview(out3, x.L, 3);
        ev.tensor_sum({&x}, {&y}, o);
        writeback(out3, o);
    });
}
encf_status encf_relinearize(encf_ctx* c, const encf_keys* k, const encf_ct* in3, encf_ct* out, void* stream) {
    return guard([&] { EV_BEGIN(k); DCt x = view(c, in3); DCt o = outview(out, x.L, 2); ev.relin(x, o); writeback(out, o); });
}
encf_status encf_rotate(encf_ctx* c, const encf_keys* k, const encf_ct* in, int32_t steps, encf_ct* out, void* stream) {
    return guard([&] {
        EV_BEGIN(k);
        DCt x = view(c, in);
        DCt o = outview(out, x.L, 2);
        uint32_t g = ev.galois_rot(steps);
        if (g == 1u) ev.copy(x, o);
        else ev.rotate_galois(x, g, o);
        writeback(out, o);
    });
}
encf_status encf_rotate_hoisted(encf_ctx* c, const encf_keys* k, const encf_ct* in, const int32_t* steps, int32_t n,
                                encf_ct* outs, void* stream) {
    return guard([&] {
        EV_BEGIN(k);
        need(steps && outs && n >= 1, ENCF_ERR_ARG, "rotate_hoisted: bad argument");
        DCt x = view(c, in);
        std::vector<uint32_t> gs;
        std::vector<DCt> os;
        for (int i = 0; i < n; i++) { gs.push_back(ev.galois_rot(steps[i])); os.push_back(outview(&outs[i], x.L, 2)); }
        ev.rotate_hoisted(x, gs, os);
        for (int i = 0; i < n; i++) writeback(&outs[i], os[i]);
    });
}
encf_status encf_conjugate(encf_ctx* c, const encf_keys* k, const encf_ct* in, encf_ct* out, void* stream) {
    return guard([&] { EV_BEGIN(k); DCt x = view(c, in); DCt o = outview(out, x.L, 2); ev.rotate_galois(x, ev.galois_conj(), o); writeback(out, o); });
}
encf_status encf_decomplexify(encf_ctx* c, const encf_keys* k, const encf_ct* in, int32_t n, encf_ct* outs, void* stream) {
    return guard([&] {
        EV_BEGIN(k);
        need(in != nullptr && outs != nullptr && n >= 1, ENCF_ERR_ARG, "decomplexify: n >= 1 ciphertexts");
        std::vector<DCt> xs, cj, os;
        std::vector<const DCt*> xp;
        for (int i = 0; i < n; i++) xs.push_back(view(c, &in[i]));
        for (int i = 0; i < n; i++) {
            need(xs[i].ncomp == 2, ENCF_ERR_FORMAT, "decomplexify: 2-component ciphertexts");
            need(xs[i].L == xs[0].L, ENCF_ERR_LEVEL_MISMATCH, "decomplexify: mixed levels");
            xp.push_back(&xs[i]);
            os.push_back(outview(&outs[i], xs[i].L, 2));
        }
        cj = ev.alloc_many(n, xs[0].L);
        ev.rotate_many(xp, std::vector<uint32_t>(n, ev.galois_conj()), cj);
        for (int i = 0; i < n; i++) {
            ev.add(xs[i], cj[i], os[i]);
            os[i].scale = 2.0 * xs[i].scale;
            writeback(&outs[i], os[i]);
        }
    });
}
encf_status encf_rescale(encf_ctx* c, const encf_ct* in, encf_ct* out, void* stream) {
    return guard([&] { EV_BEGIN(nullptr); DCt x = view(c, in); need(x.L > 1, ENCF_ERR_LEVEL_EXHAUSTED, "rescale at one limb"); DCt o = outview(out, x.L - 1, x.ncomp); ev.rescale(x, o); writeback(out, o); });
}
encf_status encf_mod_drop(encf_ctx* c, const encf_ct* in, int32_t n_limbs, encf_ct* out, void* stream) {
    return guard([&] { EV_BEGIN(nullptr); DCt x = view(c, in); DCt o = outview(out, n_limbs, x.ncomp); ev.mod_drop(x, n_limbs, o); writeback(out, o); });
}
encf_status encf_complexify(encf_ctx* c, const encf_ct* re, const encf_ct* im, encf_ct* out, void* stream) {
    return guard([&] {
        EV_BEGIN(nullptr);
        DCt a = view(c, re), b = view(c, im);
        DCt t = ev.alloc(b.L, b.ncomp);
        ev.mul_i(b, t);
        DCt o = outview(out, a.L, a.ncomp);
        ev.add(a, t, o);
        writeback(out, o);
    });
}

encf_status encf_complexify_many(encf_ctx* c, const encf_ct* re, const encf_ct* im, int32_t n, encf_ct* out, void* stream) {
    return guard([&] {
        EV_BEGIN(nullptr);
        need(re != nullptr && im != nullptr && out != nullptr && n >= 1, ENCF_ERR_ARG, "complexify_many: n >= 1 pairs");
        std::vector<DCt> a, b, o;
        for (int i = 0; i < n; i++) { a.push_back(view(c, &re[i])); b.push_back(view(c, &im[i])); }
        std::vector<const DCt*> ap, bp;
        for (int i = 0; i < n; i++) {
            need(a[i].L == a[0].L && b[i].L == a[0].L && a[i].ncomp == a[0].ncomp && b[i].ncomp == a[0].ncomp,
                 ENCF_ERR_LEVEL_MISMATCH, "complexify_many: every re/im at one level and component count");
            ap.push_back(&a[i]);
            bp.push_back(&b[i]);
            o.push_back(outview(&out[i], a[i].L, a[i].ncomp));
        }
        ev.add_i_many(ap, bp, o);   // re + X^{N/2} im, batched (the words of encf_complexify)
        for (int i = 0; i < n; i++) writeback(&out[i], o[i]);
    });
}

encf_status encf_mask_put(encf_ctx* c, const encf_mask_desc* d, const uint64_t* coeffs) {
    return guard([&] {
        need(c && d && coeffs, ENCF_ERR_ARG, "mask_put: null argument");
        level_ok(c, d->level);
        const int N = c->N, L = d->level;
        const LimbMap lm = d->ext ? c->extmap(L) : c->qmap(L);
        u64* pt = nullptr;
        CUDA_TRY(cudaMalloc(&pt, (size_t)lm.n * N * 8));
        CUDA_TRY(cudaMemcpy(pt, coeffs, (size_t)lm.n * N * 8, cudaMemcpyHostToDevice));
        ntt_forward(*c, PolyBatch{pt, 0, 1, lm}, 0);
        CUDA_TRY(cudaDeviceSynchronize());
        MaskKey key{d->m, d->r0, d->r1, d->s0, d->sstride, d->scount, d->level, d->ext ? 1 : 0};
        std::lock_guard<std::mutex> lk(c->mu);
        auto it = c->masks.find(key);
        if (it != c->masks.end()) cudaFree(it->second);
        c->masks[key] = pt;
        // caches derived from masks go stale: the pre-masked keys of this descriptor, and every value-kernel mask
        // spectrum (keyed by mask addresses, which the allocator may hand out again)
        for (auto k = c->kmasks.begin(); k != c->kmasks.end();) {
            if (!(k->first.mk < key) && !(key < k->first.mk)) { cudaFree(k->second); k = c->kmasks.erase(k); }
            else ++k;
        }
        for (auto& kv : c->bhat) cudaFree(kv.second);
        c->bhat.clear();
    });
}

encf_status encf_mask_clear(encf_ctx* c) {
    if (!c) return ENCF_ERR_ARG;
    cudaDeviceSynchronize();
    std::lock_guard<std::mutex> lk(c->mu);
    for (auto& kv : c->masks) cudaFree(kv.second);
    c->masks.clear();
    for (auto& kv : c->kmasks) cudaFree(kv.second);
    c->kmasks.clear();
    for (auto& kv : c->bhat) cudaFree(kv.second);   // keyed by mask pointers: stale once the masks are gone
    c->bhat.clear();
    return ENCF_OK;
}

// ------------------------------------------------------------------------------------ projection
encf_status encf_proj_plan_create(encf_ctx* c, int32_t m, int32_t d_in, int32_t d_out, int32_t C, int32_t N1, uint32_t flags,
                                  encf_proj_plan** out) {
    return guard([&] {
        need(c && out, ENCF_ERR_ARG, "proj_plan_create: null argument");
        encf_proj_plan* p = new encf_proj_plan();
        try { proj_plan_init(*p, c->N / 2, m, d_in, d_out, C, N1, flags); } catch (...) { delete p; throw; }
        *out = p;
    });
}
encf_status encf_proj_plan_destroy(encf_proj_plan* p) { delete p; return ENCF_OK; }
encf_status encf_proj_plan_info(const encf_proj_plan* p, int32_t* o) {
    if (!p || !o) return ENCF_ERR_ARG;
    o[0] = p->C; o[1] = p->G; o[2] = p->U; o[3] = p->B_out; o[4] = p->N1; o[5] = p->N2; o[6] = p->B_out * p->N2 * p->U * p->N1;
    return ENCF_OK;
}
encf_status encf_proj_galois(encf_ctx* c, const encf_proj_plan* p, uint32_t* out, int32_t cap, int32_t* n) {
    return guard([&] {
        need(c && p && n, ENCF_ERR_ARG, "proj_galois: null argument");
        Scratch sc(0);
        Ev ev(*c, nullptr, 0, sc);
        auto g = proj_galois(ev, *p);
        *n = (int32_t)g.size();
        for (int i = 0; i < (int)g.size() && i < cap && out; i++) out[i] = g[i];
    });
}
encf_status encf_proj_weights_size(const encf_proj_plan* p, int32_t nl, size_t* bytes) {
    if (!p || !bytes) return ENCF_ERR_ARG;
    *bytes = (size_t)p->B_out * p->N2 * p->U * p->N1 * nl * (size_t)(2 * p->n) * 8;
    return ENCF_OK;
}

static void encode_weights_impl(encf_ctx* c, const encf_proj_plan* p, const double* W, const double* Wim, int32_t nl,
                                uint64_t* w_out, cudaStream_t s) {
    need(c && p && W && w_out, ENCF_ERR_ARG, "encode_weights: null argument");
    level_ok(c, nl);
    const int real = (p->flags & ENCF_PROJ_REAL_INPUT) ? 1 : 0;
    need(real || !Wim, ENCF_ERR_ARG, "complex weights need a real-input (fused-QK) plan");
    Scratch sc(s);
    const int N = c->N;
    const double scale = (double)c->mods[nl - 1];
    const size_t wsz = (size_t)p->d_in * p->d_out;
    double* dW = (double*)sc.get(wsz);
    CUDA_TRY(cudaMemcpyAsync(dW, W, wsz * 8, cudaMemcpyHostToDevice, s));
    double* dWi = nullptr;
    if (Wim) {
        dWi = (double*)sc.get(wsz);
        CUDA_TRY(cudaMemcpyAsync(dWi, Wim, wsz * 8, cudaMemcpyHostToDevice, s));
    }
    std::vector<int> bs, ps, us, qs;
    for (int b = 0; b < p->B_out; b++)
        for (int pp = 0; pp < p->N2; pp++)
            for (int u = 0; u < p->U; u++)
                for (int q = 0; q < p->N1; q++) { bs.push_back(b); ps.push_back(pp); us.push_back(u); qs.push_back(q); }
    const int BATCH = 32;
    for (size_t i0 = 0; i0 < bs.size(); i0 += BATCH) {
        int cnt = (int)std::min((size_t)BATCH, bs.size() - i0);
        k_encode_weights(*c, dW, p->d_in, p->d_out, p->C, p->N1, p->m, &bs[i0], &ps[i0], &us[i0], &qs[i0], cnt, scale, nl,
                         w_out + i0 * nl * N, s, dWi, real);
    }
    size_t np = bs.size();
    for (size_t i0 = 0; i0 < np; i0 += 4096) {
        int cnt = (int)std::min((size_t)4096, np - i0);
        ntt_forward(*c, PolyBatch{w_out + i0 * nl * N, (i64)nl * N, cnt, c->qmap(nl)}, s);
    }
}

encf_status encf_proj_encode_weights(encf_ctx* c, const encf_proj_plan* p, const double* W, int32_t nl, uint64_t* w_out,
                                     void* stream) {
    return guard([&] { encode_weights_impl(c, p, W, nullptr, nl, w_out, S(stream)); });
}

encf_status encf_proj_encode_weights_complex(encf_ctx* c, const encf_proj_plan* p, const double* Wre, const double* Wim,
                                             int32_t nl, uint64_t* w_out, void* stream) {
    return guard([&] { encode_weights_impl(c, p, Wre, Wim, nl, w_out, S(stream)); });
}

encf_status encf_pt_ct_matmul(encf_ctx* c, const encf_keys* k, const encf_proj_plan* p, const encf_ct* x, const uint64_t* w,
                              double w_scale, int32_t u0, int32_t u1, uint32_t flags, encf_ct* y, void* stream) {
    return guard([&] {
        need(c && k && p && x && w && y, ENCF_ERR_ARG, "pt_ct_matmul: null argument");
        const int units = p->B_out * p->N2;
        need(0 <= u0 && u0 < u1 && u1 <= units, ENCF_ERR_ARG, "pt_ct_matmul: bad unit range");
        need(p->n == c->N / 2, ENCF_ERR_PLAN_SHAPE, "plan built for another ring");
        EV_BEGIN(k);
        std::vector<DCt> xs;
        for (int u = 0; u < p->U; u++) {
            xs.push_back(view(c, &x[u]));
            need(xs.back().ncomp == 2, ENCF_ERR_FORMAT, "inputs must have 2 components");
        }
        const int L = xs[0].L;
        need(L >= 2, ENCF_ERR_LEVEL_EXHAUSTED, "projection needs two limbs");
        std::vector<DCt> accs;
        const int Lw = p->restricted ? L - 1 : L;
        const size_t wus = (size_t)p->U * p->N1 * Lw * c->N;       // words per (b, p) unit of the weight stream
        const u64* wu = (flags & ENCF_PROJ_W_SHARD) ? w : w + (size_t)u0 * wus;
        proj_phase1(ev, *p, xs, wu, w_scale, u0, u1, accs);
        int b_first = u0 / p->N2;
        bool fin = (flags & ENCF_PROJ_FINALIZE) && u0 == 0 && u1 == units;
        if (fin) {
            std::vector<DCt> ys = ev.alloc_many((int)accs.size(), L - 1);
            proj_finalize_many(ev, *p, accs, ys);
            for (size_t i = 0; i < accs.size(); i++) {
                encf_ct* yo = &y[b_first + i];
                DCt o = outview(yo, L - 1, 2);
                ev.copy(ys[i], o);
                writeback(yo, o);
            }
        } else {   // partial accumulators in the EXTENDED basis at the bank level La (= L, or L - 1 for a restricted
                   // plan): n_limbs = La + K (R-LAZY; reduce with encf_mod_reduce_ext)
            const int La = accs[0].L, Ka = c->Kof(La);
            for (size_t i = 0; i < accs.size(); i++) {
                encf_ct* yo = &y[b_first + i];
                need(yo && yo->data, ENCF_ERR_ARG, "null output");
                k_copy(accs[i].d, yo->data, (size_t)2 * (La + Ka) * c->N, s);
                yo->n_comp = 2; yo->n_limbs = La + Ka; yo->scale = accs[i].scale; yo->ntt = 1;
            }
        }
    });
}

encf_status encf_pt_ct_matmul_finalize(encf_ctx* c, const encf_keys* k, const encf_proj_plan* p, const encf_ct* acc,
                                       int32_t b0, int32_t b1, encf_ct* y, void* stream) {
    return guard([&] {
        need(c && k && p && acc && y && 0 <= b0 && b0 < b1 && b1 <= p->B_out, ENCF_ERR_ARG, "finalize: bad argument");
        EV_BEGIN(k);
        const int L = c->level_of_ext(acc[0].n_limbs);     // extended partials: n_limbs = L + K(L)
        need(L >= 2, ENCF_ERR_LEVEL_MISMATCH, "finalize expects extended accumulators (n_limbs = L + K(L))");
        std::vector<DCt> accs = ev.alloc_many_ext(b1 - b0, L);
        for (int b = b0; b < b1; b++) {
            need(acc[b - b0].n_limbs == L + c->Kof(L) && acc[b - b0].data, ENCF_ERR_LEVEL_MISMATCH, "finalize: mixed accumulators");
            k_copy(acc[b - b0].data, accs[b - b0].d, (size_t)2 * (L + c->Kof(L)) * c->N, s);
            accs[b - b0].scale = acc[b - b0].scale;
        }
        std::vector<DCt> ys = ev.alloc_many(b1 - b0, L - 1);
        proj_finalize_many(ev, *p, accs, ys);
        for (int b = b0; b < b1; b++) {
            DCt o = outview(&y[b - b0], L - 1, 2);
            ev.copy(ys[b - b0], o);
            writeback(&y[b - b0], o);
        }
    });
}

// ------------------------------------------------------------------------------------ attention
encf_status encf_attn_plan_create(encf_ctx* c, int32_t m, int32_t H, int32_t d_h, int32_t C_qk, int32_t beta, int32_t H_blk,
                                  encf_attn_plan** out) {
    return guard([&] {
        need(c && out, ENCF_ERR_ARG, "attn_plan_create: null argument");
        encf_attn_plan* a = new encf_attn_plan();
        try { attn_plan_init(*a, c->N / 2, m, H, d_h, C_qk, beta, H_blk); } catch (...) { delete a; throw; }
        *out = a;
    });
}
encf_status encf_attn_plan_destroy(encf_attn_plan* a) { delete a; return ENCF_OK; }
encf_status encf_attn_plan_info(const encf_attn_plan* a, int32_t* o) {
    if (!a || !o) return ENCF_ERR_ARG;
    o[0] = a->B; o[1] = a->beta; o[2] = a->g; o[3] = a->n_out; o[4] = a->H_blk; o[5] = a->B_V; o[6] = a->seg_stride; o[7] = a->C;
    return ENCF_OK;
}
encf_status encf_attn_galois(encf_ctx* c, const encf_attn_plan* a, uint32_t* out, int32_t cap, int32_t* n) {
    return guard([&] {
        need(c && a && n, ENCF_ERR_ARG, "attn_galois: null argument");
        Scratch sc(0);
        Ev ev(*c, nullptr, 0, sc);
        auto g = attn_galois(ev, *a);
        *n = (int32_t)g.size();
        for (int i = 0; i < (int)g.size() && i < cap && out; i++) out[i] = g[i];
    });
}

encf_status encf_ct_ct_attn_score(encf_ctx* c, const encf_keys* k, const encf_attn_plan* a, const encf_ct* q, const encf_ct* kk,
                                  int32_t t0, int32_t t1, encf_ct* s_t, void* stream) {
    return guard([&] {
        need(c && k && a && q && kk && s_t && 0 <= t0 && t0 < t1 && t1 <= a->m / 2, ENCF_ERR_ARG, "score: bad argument");
        EV_BEGIN(k);
        std::vector<DCt> qs, ks;
        for (int l = 0; l < a->B; l++) { qs.push_back(view(c, &q[l])); ks.push_back(view(c, &kk[l])); }
        std::vector<DCt> S;
        score_run(ev, *a, qs, ks, t0, t1, S);
        for (int t = 0; t < t1 - t0; t++) {
            DCt o = outview(&s_t[t], S[t].L, 2);
            ev.copy(S[t], o);
            writeback(&s_t[t], o);
        }
    });
}

encf_status encf_attn_export_stream(encf_ctx* c, const encf_keys* k, const encf_attn_plan* a, const encf_ct* s_t,
                                    encf_ct* s_min, void* stream) {
    return guard([&] {
        need(c && k && a && s_t && s_min, ENCF_ERR_ARG, "export_stream: null argument");
        EV_BEGIN(k);
        std::vector<DCt> S;
        for (int t = 0; t < a->m / 2; t++) S.push_back(view(c, &s_t[t]));
        std::vector<DCt> outs;
        score_export_run(ev, *a, S, outs);
        for (int i = 0; i < a->n_out; i++) {
            DCt o = outview(&s_min[i], outs[i].L, 2);
            ev.copy(outs[i], o);
            writeback(&s_min[i], o);
        }
    });
}

encf_status encf_ct_ct_attn_value(encf_ctx* c, const encf_keys* k, const encf_attn_plan* a, const encf_ct* p_fd, const encf_ct* v,
                                  encf_ct* o, void* stream) {
    return guard([&] {
        need(c && k && a && p_fd && v && o, ENCF_ERR_ARG, "value: null argument");
        EV_BEGIN(k);
        std::vector<DCt> ps, vs;
        for (int l = 0; l < a->B_V; l++) {
            ps.push_back(view(c, &p_fd[l]));
            vs.push_back(view(c, &v[l]));
            need(vs.back().L >= ps.back().L + 1 && ps.back().L >= 3, ENCF_ERR_LEVEL_MISMATCH, "value: level plan (Lv > Lp >= 3)");
        }
        std::vector<DCt> outs;
        value_run(ev, *a, ps, vs, outs);
        for (int l = 0; l < a->B_V; l++) {
            DCt oo = outview(&o[l], outs[l].L, 2);
            ev.copy(outs[l], oo);
            writeback(&o[l], oo);
        }
    });
}

encf_status encf_ct_ct_attn_value_partial(encf_ctx* c, const encf_keys* k, const encf_attn_plan* a, const encf_ct* p_fd,
                                          const encf_ct* v, int32_t u0, int32_t u1, encf_ct* o3, void* stream) {
    return guard([&] {
        need(c && k && a && p_fd && v && o3, ENCF_ERR_ARG, "value_partial: null argument");
        need(0 <= u0 && u0 < u1 && u1 <= a->B_V * (a->m / 2), ENCF_ERR_ARG, "value_partial: bad unit range");
        EV_BEGIN(k);
        std::vector<DCt> ps, vs;
        for (int l = 0; l < a->B_V; l++) {
            ps.push_back(view(c, &p_fd[l]));
            vs.push_back(view(c, &v[l]));
            need(vs.back().L >= ps.back().L + 1 && ps.back().L >= 3, ENCF_ERR_LEVEL_MISMATCH, "value: level plan (Lv > Lp >= 3)");
        }
        std::vector<int> blocks;
        std::vector<DCt> o3s;
        value_partial_run(ev, *a, ps, vs, u0, u1, blocks, o3s);
        for (size_t i = 0; i < blocks.size(); i++) {
            DCt oo = outview(&o3[i], o3s[i].L, 3);
            ev.copy(o3s[i], oo);
            writeback(&o3[i], oo);
        }
    });
}

encf_status encf_attn_value_finalize(encf_ctx* c, const encf_keys* k, const encf_ct* o3, int32_t n, encf_ct* o, void* stream) {
    return guard([&] {
        need(c && k && o3 && o && n >= 1, ENCF_ERR_ARG, "value_finalize: bad argument");
        EV_BEGIN(k);
        std::vector<DCt> xs;
        for (int i = 0; i < n; i++) {
            xs.push_back(view(c, &o3[i]));
            need(xs.back().ncomp == 3 && xs.back().L == xs[0].L, ENCF_ERR_FORMAT, "value_finalize: 3-component partials at one level");
            need(xs.back().L >= 2, ENCF_ERR_LEVEL_EXHAUSTED, "value_finalize: one limb");
        }
        std::vector<DCt> ys = ev.alloc_many(n, xs[0].L - 1);
        std::vector<const DCt*> xp;
        for (auto& x : xs) xp.push_back(&x);
        ev.relin_rescale_many(xp, ys);
        for (int i = 0; i < n; i++) {
            DCt oo = outview(&o[i], ys[i].L, 2);
            ev.copy(ys[i], oo);
            writeback(&o[i], oo);
        }
    });
}

// ------------------------------------------------------------------------------------ ciphertext shifts (App. A.1)
encf_status encf_rotfirst(encf_ctx* c, const encf_keys* k, const encf_ct* in, int32_t L_slots, const int32_t* taus, int32_t n,
                          int32_t m, encf_ct* outs, void* stream) {
    return guard([&] {
        EV_BEGIN(k);
        need(taus && outs && n >= 1 && m >= 1, ENCF_ERR_ARG, "rotfirst: bad argument");
        need(L_slots >= 1 && L_slots <= c->N / 2, ENCF_ERR_ARG, "rotfirst: L must be in [1, n]");
        DCt x = view(c, in);
        need(x.ncomp == 2, ENCF_ERR_FORMAT, "rotfirst: 2-component input");
        need(x.L >= 2, ENCF_ERR_LEVEL_EXHAUSTED, "rotfirst: needs one level");
        std::vector<ShiftReq> reqs;
        for (int i = 0; i < n; i++) reqs.push_back(rotfirst_req(0, L_slots, taus[i], m));
        std::vector<DCt> os = ev.alloc_many(n, x.L - 1);
        shift_many(ev, {&x}, reqs, os);
        for (int i = 0; i < n; i++) {
            DCt oo = outview(&outs[i], os[i].L, 2);
            ev.copy(os[i], oo);
            writeback(&outs[i], oo);
        }
    });
}

encf_status encf_psi(encf_ctx* c, const encf_keys* k, const encf_ct* in, int32_t m, const int32_t* ts, int32_t n, encf_ct* outs,
                     void* stream) {
    return guard([&] {
        EV_BEGIN(k);
        need(ts && outs && n >= 1 && m >= 1 && (c->N / 2) % m == 0, ENCF_ERR_ARG, "psi: bad argument");
        DCt x = view(c, in);
        need(x.ncomp == 2, ENCF_ERR_FORMAT, "psi: 2-component input");
        need(x.L >= 2, ENCF_ERR_LEVEL_EXHAUSTED, "psi: needs one level");
        std::vector<std::vector<DCt>> os;
        psi_many(ev, {&x}, {std::vector<int>(ts, ts + n)}, m, 0, c->N / 2 / m, os);
        for (int i = 0; i < n; i++) {
            DCt oo = outview(&outs[i], os[0][i].L, 2);
            ev.copy(os[0][i], oo);
            writeback(&outs[i], oo);
        }
    });
}

// ------------------------------------------------------------------------------------ w/o-SCP ablation repack
encf_status encf_repack_rma(encf_ctx* c, const encf_keys* k, const encf_ct* x, int32_t n, int32_t m, encf_ct* out, void* stream) {
    return guard([&] {
        need(c && k && x && out && n > 0, ENCF_ERR_ARG, "repack_rma: null argument");
        EV_BEGIN(k);
        std::vector<DCt> xs;
        for (int i = 0; i < n; i++) xs.push_back(view(c, &x[i]));
        std::vector<DCt> ys;
        repack_rma_run(ev, xs, m, ys);
        for (int i = 0; i < n; i++) {
            DCt o = outview(&out[i], ys[i].L, 2);
            ev.copy(ys[i], o);
            writeback(&out[i], o);
        }
    });
}

// ------------------------------------------------------------------------------------ GELU pre-evaluation
encf_status encf_gelu_preeval(encf_ctx* c, const encf_keys* k, const encf_ct* x, int32_t n, const double* coef, encf_ct* f0,
                              encf_ct* f1, void* stream) {
    return guard([&] {
        need(c && k && x && coef && f0 && f1 && n > 0, ENCF_ERR_ARG, "gelu_preeval: null argument");
        EV_BEGIN(k);
        std::vector<DCt> xs;
        for (int i = 0; i < n; i++) xs.push_back(view(c, &x[i]));
        std::vector<DCt> a, b;
        gelu_preeval_run(ev, xs, coef, a, b);
        for (int i = 0; i < n; i++) {
            DCt oa = outview(&f0[i], a[i].L, 2), ob = outview(&f1[i], b[i].L, 2);
            ev.copy(a[i], oa);
            ev.copy(b[i], ob);
            writeback(&f0[i], oa);
            writeback(&f1[i], ob);
        }
    });
}

// ------------------------------------------------------------------------------------ export
encf_status encf_l_conv(encf_ctx* c, int32_t ell, int32_t sigma, double scale, double B_max, int32_t* L) {
    if (!c || !L) return ENCF_ERR_ARG;
    int r = l_conv_rule(*c, ell, sigma, scale, B_max);
    if (r < 0) { set_last_error("no level satisfies the trimming inequalities (P:874-876)"); return ENCF_ERR_CONFIG; }
    *L = r;
    return ENCF_OK;
}

encf_status encf_export_c2m(encf_ctx* c, const encf_ct* in, int32_t Lc, uint64_t mask_seed, uint64_t stream_id, encf_ct* masked,
                            uint64_t* share, void* stream) {
    return guard([&] {
        need(c && masked && masked->data && share, ENCF_ERR_ARG, "export: null argument");
        DCt x = view(c, in);
        need(x.ncomp == 2, ENCF_ERR_FORMAT, "export needs 2 components");
        need(Lc >= 1 && Lc <= x.L, ENCF_ERR_LEVEL_MISMATCH, "export: L_conv above the ciphertext level");
        need(stream_id < (1ull << 56), ENCF_ERR_ARG, "export: stream_id must be < 2^56");
        cudaStream_t s = S(stream);
        const int N = c->N;
        for (int comp = 0; comp < 2; comp++)
            k_copy(x.comp(comp, N), masked->data + (size_t)comp * Lc * N, (size_t)Lc * N, s);
        ntt_inverse(*c, PolyBatch{masked->data, (i64)Lc * N, 2, c->qmap(Lc)}, s);
        k_export_mask(*c, mask_seed, (0x04ull << 56) | stream_id, masked->data, share, Lc, s);
        masked->n_comp = 2; masked->n_limbs = Lc; masked->scale = x.scale; masked->ntt = 0;
    });
}

static void export_many_impl(encf_ctx* c, const encf_ct* in, int32_t n, int32_t Lc, uint64_t mask_seed, uint64_t stream_id0,
                             const uint64_t* d_seed_sid, uint64_t* masked, uint64_t* shares, void* stream);

encf_status encf_export_c2m_many(encf_ctx* c, const encf_ct* in, int32_t n, int32_t Lc, uint64_t mask_seed, uint64_t stream_id0,
                                 uint64_t* masked, uint64_t* shares, void* stream) {
    return guard([&] {
        need(stream_id0 + (uint64_t)n <= (1ull << 56), ENCF_ERR_ARG, "export_many: stream ids must be < 2^56");
        export_many_impl(c, in, n, Lc, mask_seed, stream_id0, nullptr, masked, shares, stream);
    });
}

encf_status encf_export_c2m_many_dev(encf_ctx* c, const encf_ct* in, int32_t n, int32_t Lc, const uint64_t* d_seed_sid,
                                     uint64_t* masked, uint64_t* shares, void* stream) {
    return guard([&] {
        need(d_seed_sid != nullptr, ENCF_ERR_ARG, "export_many_dev: null seed/stream buffer");
        export_many_impl(c, in, n, Lc, 0, 0, d_seed_sid, masked, shares, stream);
    });
}

static void export_many_impl(encf_ctx* c, const encf_ct* in, int32_t n, int32_t Lc, uint64_t mask_seed, uint64_t stream_id0,
                             const uint64_t* d_seed_sid, uint64_t* masked, uint64_t* shares, void* stream) {
    {
        need(c && in && masked && shares && n >= 1, ENCF_ERR_ARG, "export_many: null argument or n < 1");
        cudaStream_t s = S(stream);
        const int N = c->N;
        const size_t cw = (size_t)2 * Lc * N;
        int L0 = -1;
        for (int i = 0; i < n; i++) {
            DCt x = view(c, &in[i]);
            need(x.ncomp == 2, ENCF_ERR_FORMAT, "export needs 2 components");
            need(Lc >= 1 && Lc <= x.L, ENCF_ERR_LEVEL_MISMATCH, "export: L_conv above the ciphertext level");
            if (L0 < 0) L0 = x.L;
            need(x.L == L0, ENCF_ERR_LEVEL_MISMATCH, "export_many: mixed levels");
            for (int comp = 0; comp < 2; comp++)
                k_copy(x.comp(comp, N), masked + cw * i + (size_t)comp * Lc * N, (size_t)Lc * N, s);
        }
        ntt_inverse(*c, PolyBatch{masked, (i64)Lc * N, 2 * n, c->qmap(Lc)}, s);
        for (int i = 0; i < n; i++) {
            if (d_seed_sid)
                k_export_mask_dev(*c, d_seed_sid, (uint64_t)i, masked + cw * i, shares + (size_t)i * Lc * N, Lc, s);
            else
                k_export_mask(*c, mask_seed, (0x04ull << 56) | (stream_id0 + (uint64_t)i), masked + cw * i,
                              shares + (size_t)i * Lc * N, Lc, s);
        }
    }
}

encf_status encf_ring2field_local(encf_ctx* c, const uint64_t* mp, int32_t party, int32_t ell_sigma, int32_t L, uint64_t* out,
                                  void* stream) {
    return guard([&] {
        need(c && mp && out && (party == 0 || party == 1) && ell_sigma > 0 && ell_sigma < 127, ENCF_ERR_ARG, "ring2field: bad argument");
        level_ok(c, L);
        R2F off;
        for (int i = 0; i < L; i++) {
            u64 q = c->mods[i];
            u64 t = (u64)((((unsigned __int128)1) << ell_sigma) % q);
            off.v[i] = party ? t : 0;
        }
        k_ring2field(*c, mp, out, L, off, S(stream));
    });
}

encf_status encf_field2ring_local(encf_ctx* c, const uint64_t* share, int32_t ell, uint64_t* out, void* stream) {
    return guard([&] {
        need(c && share && out && ell > 0 && ell <= 64, ENCF_ERR_ARG, "field2ring: bad argument");
        k_field2ring(*c, share, out, ell, S(stream));
    });
}

encf_status encf_import_m2c(encf_ctx* c, const encf_ct* ct, const encf_pt* share, encf_ct* out, void* stream) {
    return guard([&] {
        need(c && share && share->data && out && out->data, ENCF_ERR_ARG, "import_m2c: null argument");
        DCt x = view(c, ct);
        need(x.ncomp == 2, ENCF_ERR_FORMAT, "import_m2c needs a 2-component ciphertext");
        need(share->n_limbs == x.L, ENCF_ERR_LEVEL_MISMATCH, "import_m2c: share level != ciphertext level");
        cudaStream_t s = S(stream);
        Scratch sc(s);
        const int N = c->N, L = x.L;
        u64* t = sc.get((size_t)L * N);
        k_copy(share->data, t, (size_t)L * N, s);
        if (!share->ntt) ntt_forward(*c, PolyBatch{t, 0, 1, c->qmap(L)}, s);
        k_add(*c, x.comp(0, N), t, out->data, 1, c->qmap(L), false, s);
        k_copy(x.comp(1, N), out->data + (size_t)L * N, (size_t)L * N, s);
        out->n_comp = 2; out->n_limbs = L; out->scale = x.scale; out->ntt = 1;
    });
}

encf_status encf_mod_reduce_ext(encf_ctx* c, uint64_t* d, int32_t np, int32_t L, void* stream) {
    return guard([&] {
        need(c && d && np >= 0, ENCF_ERR_ARG, "mod_reduce_ext: bad argument");
        level_ok(c, L);
        k_mod_reduce(*c, d, np, c->extmap(L), S(stream));
    });
}

encf_status encf_mod_reduce(encf_ctx* c, uint64_t* d, int32_t np, int32_t nl, void* stream) {
    return guard([&] {
        need(c && d && np >= 0, ENCF_ERR_ARG, "mod_reduce: bad argument");
        level_ok(c, nl);
        k_mod_reduce(*c, d, np, c->qmap(nl), S(stream));
    });
}

}  // extern "C"
