// ntt.cu -- negacyclic NTT / iNTT over 64-bit RNS limbs (the ring isomorphism of P:82) for sm_100a.
//
// Forward: merged-twiddle Cooley-Tukey (bit-reversed output), Harvey lazy butterflies in [0, 4q),
// Shoup twiddles.  Inverse: Gentleman-Sande with psi^{-brv(k)} and a final N^{-1}.
// A limb of N = 2^logN words is split N = R x S (R = 2^s1 rows, S = 2^s2 columns):
//   phase A: the first s1 stages only pair elements of one column (stride S) -> a CTA stages a
//            R x 16 column tile through shared memory (128-byte coalesced row segments);
//   phase B: the last s2 stages stay inside contiguous chunks of S words -> a CTA stages a
//            group of chunks.
// (Inverse runs B then A.)  One launch per phase covers every limb of every polynomial of a batch.
#include "ctx.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kTileElems = 4096;   // 32 KB of shared memory per CTA

struct NttArgs {
    u64* base;
    i64 poly_stride;
    LimbMap map;
    const ModConst* mod;
    const u64* tw;       // psi_brv (fwd) or ipsi_brv (inv): [mods][N]
    const u64* tw_sh;
    const u64* ninv;
    const u64* ninv_sh;
    int N, logN, s1, s2;
};

__device__ __forceinline__ void ct_bfly(u64& X, u64& Y, u64 W, u64 Wp, u64 q, u64 two_q) {
    u64 x = X >= two_q ? X - two_q : X;
    u64 t = mul_shoup_lazy(Y, W, Wp, q);
    X = x + t;
    Y = x - t + two_q;
}

__device__ __forceinline__ void gs_bfly(u64& X, u64& Y, u64 W, u64 Wp, u64 q, u64 two_q) {
    u64 x = X + Y;
    x = x >= two_q ? x - two_q : x;
    u64 t = X - Y + two_q;
    Y = mul_shoup_lazy(t, W, Wp, q);
    X = x;
}

// Phase A (columns).  Forward: stages 0..s1-1.  Inverse: stages s1-1..0, then x N^{-1}, reduce.
template <bool kInverse>
__global__ void __launch_bounds__(kThreads) ntt_cols(NttArgs a) {
    __shared__ u64 sm[kTileElems];
    const int limb = blockIdx.y, poly = blockIdx.z;
    const int mi = a.map.mod[limb];
    const ModConst mc = a.mod[mi];
    const u64 q = mc.q, two_q = 2 * q;
    const int R = 1 << a.s1, S = 1 << a.s2;
    const int CT = S < 16 ? S : 16;
    const int c0 = blockIdx.x * CT;
    u64* g = a.base + (i64)poly * a.poly_stride + (i64)limb * a.N;
    const u64* tw = a.tw + (size_t)mi * a.N;
    const u64* twp = a.tw_sh + (size_t)mi * a.N;
    const int tot = R * CT;
    for (int e = threadIdx.x; e < tot; e += kThreads) {
        int r = e / CT, c = e % CT;
        sm[e] = g[(i64)r * S + c0 + c];
    }
    __syncthreads();
    const int nb = (R / 2) * CT;
    if (!kInverse) {
        for (int st = 0; st < a.s1; st++) {
            const int m = 1 << st, t = R >> (st + 1);
            for (int b = threadIdx.x; b < nb; b += kThreads) {
                int c = b % CT, bb = b / CT;
                int i = bb / t, j = bb % t;
                int r1 = 2 * i * t + j;
                u64 W = __ldg(tw + m + i), Wp = __ldg(twp + m + i);
                ct_bfly(sm[r1 * CT + c], sm[(r1 + t) * CT + c], W, Wp, q, two_q);
            }
            __syncthreads();
        }
    } else {
        for (int st = a.s1 - 1; st >= 0; st--) {
            const int m = 1 << st, t = R >> (st + 1);
            for (int b = threadIdx.x; b < nb; b += kThreads) {
                int c = b % CT, bb = b / CT;
                int i = bb / t, j = bb % t;
                int r1 = 2 * i * t + j;
                u64 W = __ldg(tw + m + i), Wp = __ldg(twp + m + i);
                gs_bfly(sm[r1 * CT + c], sm[(r1 + t) * CT + c], W, Wp, q, two_q);
            }
            __syncthreads();
        }
    }
    const u64 ni = kInverse ? a.ninv[mi] : 0, nip = kInverse ? a.ninv_sh[mi] : 0;
    for (int e = threadIdx.x; e < tot; e += kThreads) {
        int r = e / CT, c = e % CT;
        u64 v = sm[e];
        if (kInverse) v = mul_shoup(v, ni, nip, q);
        g[(i64)r * S + c0 + c] = v;   // forward: lazy [0, 4q) handed to phase B
    }
}

// Phase B (contiguous chunks of S words).  Forward: stages s1..logN-1 then reduce to [0, q).
// Inverse: stages logN-1..s1 (lazy [0, 2q) output handed to phase A).
template <bool kInverse>
__global__ void __launch_bounds__(kThreads) ntt_rows(NttArgs a) {
    __shared__ u64 sm[kTileElems];
    const int limb = blockIdx.y, poly = blockIdx.z;
    const int mi = a.map.mod[limb];
    const ModConst mc = a.mod[mi];
    const u64 q = mc.q, two_q = 2 * q;
    const int S = 1 << a.s2;
    const int G = kTileElems / S < (1 << a.s1) ? kTileElems / S : (1 << a.s1);   // chunks per CTA
    const int ch0 = blockIdx.x * G;
    u64* g = a.base + (i64)poly * a.poly_stride + (i64)limb * a.N + (i64)ch0 * S;
    const u64* tw = a.tw + (size_t)mi * a.N;
    const u64* twp = a.tw_sh + (size_t)mi * a.N;
    const int tot = G * S;
    for (int e = threadIdx.x; e < tot; e += kThreads) sm[e] = g[e];
    __syncthreads();
    const int nb = G * (S / 2);
    if (!kInverse) {
        for (int st = a.s1; st < a.logN; st++) {
            const int m = 1 << st, t = a.N >> (st + 1);
            const int per = S / (2 * t);       // blocks per chunk
            for (int b = threadIdx.x; b < nb; b += kThreads) {
                int ch = b / (S / 2), bb = b % (S / 2);
                int i = bb / t, j = bb % t;
                int y1 = ch * S + 2 * i * t + j;
                int blk = (ch0 + ch) * per + i;
                u64 W = __ldg(tw + m + blk), Wp = __ldg(twp + m + blk);
                ct_bfly(sm[y1], sm[y1 + t], W, Wp, q, two_q);
            }
            __syncthreads();
        }
        for (int e = threadIdx.x; e < tot; e += kThreads) {
            u64 v = sm[e];
            v = v >= two_q ? v - two_q : v;
            v = v >= q ? v - q : v;
            g[e] = v;
        }
    } else {
        for (int st = a.logN - 1; st >= a.s1; st--) {
            const int m = 1 << st, t = a.N >> (st + 1);
            const int per = S / (2 * t);
            for (int b = threadIdx.x; b < nb; b += kThreads) {
                int ch = b / (S / 2), bb = b % (S / 2);
                int i = bb / t, j = bb % t;
                int y1 = ch * S + 2 * i * t + j;
                int blk = (ch0 + ch) * per + i;
                u64 W = __ldg(tw + m + blk), Wp = __ldg(twp + m + blk);
                gs_bfly(sm[y1], sm[y1 + t], W, Wp, q, two_q);
            }
            __syncthreads();
        }
        for (int e = threadIdx.x; e < tot; e += kThreads) g[e] = sm[e];
    }
}

NttArgs make_args(encf_ctx& c, const PolyBatch& b, bool inv) {
    NttArgs a;
    a.base = b.base;
    a.poly_stride = b.poly_stride;
    a.map = b.map;
    a.mod = c.d_mod;
    a.tw = inv ? c.d_ipsi : c.d_psi;
    a.tw_sh = inv ? c.d_ipsi_sh : c.d_psi_sh;
    a.ninv = c.d_ninv;
    a.ninv_sh = c.d_ninv_sh;
    a.N = c.N;
    a.logN = c.logN;
    a.s1 = c.s1;
    a.s2 = c.s2;
    return a;
}

}  // namespace

void ntt_forward(encf_ctx& c, const PolyBatch& b, cudaStream_t s) {
    if (b.npolys <= 0 || b.map.n <= 0) return;
    NttArgs a = make_args(c, b, false);
    const int S = 1 << c.s2, R = 1 << c.s1;
    const int CT = S < 16 ? S : 16;
    dim3 gA(S / CT, b.map.n, b.npolys);
    int G = kTileElems / S < R ? kTileElems / S : R;
    dim3 gB(R / G, b.map.n, b.npolys);
    int slot;
    c.prof_begin("ntt", s, (uint64_t)b.npolys * b.map.n * c.N * 8 * 4, slot);
    ntt_cols<false><<<gA, kThreads, 0, s>>>(a);
    ntt_rows<false><<<gB, kThreads, 0, s>>>(a);
    c.prof_end(slot, s);
    c.st_ntt += (uint64_t)b.npolys * b.map.n;
    c.st_launch += 2;
    c.st_bytes += (uint64_t)b.npolys * b.map.n * c.N * 8 * 4;
    CUDA_TRY(cudaGetLastError());
}

void ntt_inverse(encf_ctx& c, const PolyBatch& b, cudaStream_t s) {
    if (b.npolys <= 0 || b.map.n <= 0) return;
    NttArgs a = make_args(c, b, true);
    const int S = 1 << c.s2, R = 1 << c.s1;
    const int CT = S < 16 ? S : 16;
    dim3 gA(S / CT, b.map.n, b.npolys);
    int G = kTileElems / S < R ? kTileElems / S : R;
    dim3 gB(R / G, b.map.n, b.npolys);
    int slot;
    c.prof_begin("ntt", s, (uint64_t)b.npolys * b.map.n * c.N * 8 * 4, slot);
    ntt_rows<true><<<gB, kThreads, 0, s>>>(a);
    ntt_cols<true><<<gA, kThreads, 0, s>>>(a);
    c.prof_end(slot, s);
    c.st_ntt += (uint64_t)b.npolys * b.map.n;
    c.st_launch += 2;
    c.st_bytes += (uint64_t)b.npolys * b.map.n * c.N * 8 * 4;
    CUDA_TRY(cudaGetLastError());
}
