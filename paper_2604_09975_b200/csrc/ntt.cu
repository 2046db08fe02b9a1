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

// Radix-4 pass over the lines held in shared memory: two consecutive stages (st, st+1) of every
// line at once, 4 elements / 4 butterflies / 3 twiddles per work item, shift-only index math.
// Line l of the tile sits at sm[l * LS + y], y < T = 2^lt.  `st` is the GLOBAL stage of the first of
// the two, `gb0` the global block offset of line l at stage s0 (block index of element y at global
// stage st is (boff(l) << (st - s0)) + (y >> (lt - (st - s0) - 1))).
template <bool kInverse>
__device__ __forceinline__ void radix4_pass(u64* sm, int LS, int nlines, int lt, int s0, int st, const int* boff,
                                            const u64* __restrict__ tw, const u64* __restrict__ twp, u64 q, u64 two_q) {
    const int sl = st - s0;                 // local stage of the first of the two
    const int lgt = lt - sl - 1;            // log2 of span t at stage st
    const int lh = lgt - 1;                 // log2(t/2)
    const int per_line = 1 << (lt - 2);     // work items per line
    const int total = nlines << (lt - 2);
    for (int w = threadIdx.x; w < total; w += blockDim.x) {
        const int l = w >> (lt - 2);
        const int g = w & (per_line - 1);
        const int i = g >> lh;              // block of size 2t at stage st
        const int j = g & ((1 << lh) - 1);
        const int base = l * LS + (i << (lgt + 1)) + j;
        const int h = 1 << lh, t = 1 << lgt;
        const int b1 = (boff[l] << sl) + i;
        const int m1 = 1 << st;
        const int b2 = (boff[l] << (sl + 1)) + 2 * i;
        const int m2 = m1 << 1;
        u64 a0 = sm[base], a1 = sm[base + h], a2 = sm[base + t], a3 = sm[base + t + h];
        const u64 W1 = __ldg(tw + m1 + b1), W1p = __ldg(twp + m1 + b1);
        const u64 Wa = __ldg(tw + m2 + b2), Wap = __ldg(twp + m2 + b2);
        const u64 Wb = __ldg(tw + m2 + b2 + 1), Wbp = __ldg(twp + m2 + b2 + 1);
        if (!kInverse) {
            ct_bfly(a0, a2, W1, W1p, q, two_q);
            ct_bfly(a1, a3, W1, W1p, q, two_q);
            ct_bfly(a0, a1, Wa, Wap, q, two_q);
            ct_bfly(a2, a3, Wb, Wbp, q, two_q);
        } else {
            gs_bfly(a0, a1, Wa, Wap, q, two_q);
            gs_bfly(a2, a3, Wb, Wbp, q, two_q);
            gs_bfly(a0, a2, W1, W1p, q, two_q);
            gs_bfly(a1, a3, W1, W1p, q, two_q);
        }
        sm[base] = a0; sm[base + h] = a1; sm[base + t] = a2; sm[base + t + h] = a3;
    }
}

template <bool kInverse>
__device__ __forceinline__ void radix2_pass(u64* sm, int LS, int nlines, int lt, int s0, int st, const int* boff,
                                            const u64* __restrict__ tw, const u64* __restrict__ twp, u64 q, u64 two_q) {
    const int sl = st - s0;
    const int lgt = lt - sl - 1;
    const int per_line = 1 << (lt - 1);
    const int total = nlines << (lt - 1);
    for (int w = threadIdx.x; w < total; w += blockDim.x) {
        const int l = w >> (lt - 1);
        const int g = w & (per_line - 1);
        const int i = g >> lgt;
        const int j = g & ((1 << lgt) - 1);
        const int base = l * LS + (i << (lgt + 1)) + j;
        const int b = (boff[l] << sl) + i;
        const int m = 1 << st;
        const u64 W = __ldg(tw + m + b), Wp = __ldg(twp + m + b);
        u64 x = sm[base], y = sm[base + (1 << lgt)];
        if (!kInverse) ct_bfly(x, y, W, Wp, q, two_q);
        else gs_bfly(x, y, W, Wp, q, two_q);
        sm[base] = x; sm[base + (1 << lgt)] = y;
    }
}

// Run stages [s0, s0 + lt) of every line (forward ascending, inverse descending) in radix-4 pairs.
template <bool kInverse>
__device__ __forceinline__ void run_stages(u64* sm, int LS, int nlines, int lt, int s0, const int* boff,
                                           const u64* tw, const u64* twp, u64 q, u64 two_q) {
    if (!kInverse) {
        int st = s0;
        for (; st + 1 < s0 + lt; st += 2) {
            radix4_pass<false>(sm, LS, nlines, lt, s0, st, boff, tw, twp, q, two_q);
            __syncthreads();
        }
        if (st < s0 + lt) {
            radix2_pass<false>(sm, LS, nlines, lt, s0, st, boff, tw, twp, q, two_q);
            __syncthreads();
        }
    } else {
        int st = s0 + lt - 1;
        if (lt & 1) {
            radix2_pass<true>(sm, LS, nlines, lt, s0, st, boff, tw, twp, q, two_q);
            __syncthreads();
            st--;
        }
        for (; st - 1 >= s0; st -= 2) {
            radix4_pass<true>(sm, LS, nlines, lt, s0, st - 1, boff, tw, twp, q, two_q);
            __syncthreads();
        }
    }
}

// Phase A (columns).  Forward: stages 0..s1-1.  Inverse: stages s1-1..0, then x N^{-1}, reduce.
// Tile: R = 2^s1 rows x CT columns, loaded with 128-byte row segments, stored transposed in shared
// memory (one padded line per column).
template <bool kInverse>
__global__ void __launch_bounds__(kThreads) ntt_cols(NttArgs a) {
    extern __shared__ u64 sm[];
    __shared__ int boff[64];
    const int limb = blockIdx.y, poly = blockIdx.z;
    const int mi = a.map.mod[limb];
    const ModConst mc = a.mod[mi];
    const u64 q = mc.q, two_q = 2 * q;
    const int R = 1 << a.s1, S = 1 << a.s2;
    const int CT = S < 16 ? S : 16;
    const int lct = CT == 16 ? 4 : (31 - __clz(CT));
    const int LS = R + 1;
    const int c0 = blockIdx.x * CT;
    u64* g = a.base + (i64)poly * a.poly_stride + (i64)limb * a.N;
    const u64* tw = a.tw + (size_t)mi * a.N;
    const u64* twp = a.tw_sh + (size_t)mi * a.N;
    if (threadIdx.x < CT) boff[threadIdx.x] = 0;
    const int tot = R * CT;
    for (int e = threadIdx.x; e < tot; e += kThreads) {
        int r = e >> lct, c = e & (CT - 1);
        sm[c * LS + r] = g[(i64)r * S + c0 + c];
    }
    __syncthreads();
    run_stages<kInverse>(sm, LS, CT, a.s1, 0, boff, tw, twp, q, two_q);
    const u64 ni = kInverse ? a.ninv[mi] : 0, nip = kInverse ? a.ninv_sh[mi] : 0;
    for (int e = threadIdx.x; e < tot; e += kThreads) {
        int r = e >> lct, c = e & (CT - 1);
        u64 v = sm[c * LS + r];
        if (kInverse) v = mul_shoup(v, ni, nip, q);
        g[(i64)r * S + c0 + c] = v;   // forward: lazy [0, 4q) handed to phase B
    }
}

// Phase B (contiguous chunks of S words).  Forward: stages s1..logN-1 then reduce to [0, q).
// Inverse: stages logN-1..s1 (lazy [0, 2q) output handed to phase A).
template <bool kInverse>
__global__ void __launch_bounds__(kThreads) ntt_rows(NttArgs a) {
    extern __shared__ u64 sm[];
    __shared__ int boff[64];
    const int limb = blockIdx.y, poly = blockIdx.z;
    const int mi = a.map.mod[limb];
    const ModConst mc = a.mod[mi];
    const u64 q = mc.q, two_q = 2 * q;
    const int S = 1 << a.s2;
    const int G = kTileElems / S < (1 << a.s1) ? kTileElems / S : (1 << a.s1);   // chunks per CTA
    const int LS = S + 1;
    const int ch0 = blockIdx.x * G;
    u64* g = a.base + (i64)poly * a.poly_stride + (i64)limb * a.N + (i64)ch0 * S;
    const u64* tw = a.tw + (size_t)mi * a.N;
    const u64* twp = a.tw_sh + (size_t)mi * a.N;
    if (threadIdx.x < G) boff[threadIdx.x] = ch0 + threadIdx.x;
    const int tot = G * S;
    for (int e = threadIdx.x; e < tot; e += kThreads) sm[(e >> a.s2) * LS + (e & (S - 1))] = g[e];
    __syncthreads();
    run_stages<kInverse>(sm, LS, G, a.s2, a.s1, boff, tw, twp, q, two_q);
    for (int e = threadIdx.x; e < tot; e += kThreads) {
        u64 v = sm[(e >> a.s2) * LS + (e & (S - 1))];
        if (!kInverse) {
            v = v >= two_q ? v - two_q : v;
            v = v >= q ? v - q : v;
        }
        g[e] = v;
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

size_t smemA(const encf_ctx& c) {
    const int R = 1 << c.s1, S = 1 << c.s2;
    const int CT = S < 16 ? S : 16;
    return (size_t)CT * (R + 1) * sizeof(u64);
}

size_t smemB(const encf_ctx& c) {
    const int R = 1 << c.s1, S = 1 << c.s2;
    const int G = kTileElems / S < R ? kTileElems / S : R;
    return (size_t)G * (S + 1) * sizeof(u64);
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
    ntt_cols<false><<<gA, kThreads, smemA(c), s>>>(a);
    ntt_rows<false><<<gB, kThreads, smemB(c), s>>>(a);
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
    ntt_rows<true><<<gB, kThreads, smemB(c), s>>>(a);
    ntt_cols<true><<<gA, kThreads, smemA(c), s>>>(a);
    c.prof_end(slot, s);
    c.st_ntt += (uint64_t)b.npolys * b.map.n;
    c.st_launch += 2;
    c.st_bytes += (uint64_t)b.npolys * b.map.n * c.N * 8 * 4;
    CUDA_TRY(cudaGetLastError());
}
