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
    const ulonglong2* tw2;   // interleaved {w, w'}: [mods][N]
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

// ---------------------------------------------------------------------------------------------
// Register-resident sub-transforms.  A phase applies LT consecutive stages (global stages
// [s0, s0+LT)) to independent "lines" of T = 2^LT elements.  A line is handled by TPL threads that
// each hold E elements in registers:
//   round A (first EA stages, large spans): thread j holds elements j + TPL*k   (k < E)
//   round B (last EB stages, small spans):  thread j holds elements ((j*G+g) << EB) + k'
// with one shared-memory exchange in between (padded: element x of a line sits at x + x/16, line
// stride LSP = T + T/16 + 1, conflict-free for both mappings and for the transposed column tiles).
template <int LT>
struct Geo {
    static constexpr int EA = (LT + 1) / 2;
    static constexpr int EB = LT - EA;
    static constexpr int E = 1 << EA;
    static constexpr int TPL = 1 << (LT - EA);
    static constexpr int G = 1 << (EA - EB);
    static constexpr int T = 1 << LT;
    static constexpr int LSP = T + T / 16 + 1;
};

__device__ __forceinline__ int pad(int x) { return x + (x >> 4); }

// Round A: local stages 0..EA-1 (forward ascending / inverse descending).  Local block index of the
// pair (k, k+hs) at local stage s is k >> (EA - s); global twiddle index 2^(s0+s) + (boff << s) + blk.
template <int LT, bool INV>
__device__ __forceinline__ void round_a(u64 (&x)[Geo<LT>::E], int s0, int boff, const ulonglong2* __restrict__ tw2,
                                        u64 q, u64 two_q) {
    constexpr int EA = Geo<LT>::EA, E = Geo<LT>::E;
#pragma unroll
    for (int ss = 0; ss < EA; ss++) {
        const int s = INV ? EA - 1 - ss : ss;
        const int hs = E >> (s + 1);
        const int base = (1 << (s0 + s)) + (boff << s);
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k & hs) continue;
            const int idx = base + (k >> (EA - s));
            const ulonglong2 T = __ldg(tw2 + idx);
            if (!INV) ct_bfly(x[k], x[k + hs], T.x, T.y, q, two_q);
            else gs_bfly(x[k], x[k + hs], T.x, T.y, q, two_q);
        }
    }
}

// Round B: local stages EA..LT-1.  Element ((j*G+g) << EB) + k'; block index at local stage EA+r is
// ((j*G+g) << r) + (k' >> (EB - r)).
template <int LT, bool INV>
__device__ __forceinline__ void round_b(u64 (&y)[Geo<LT>::E], int j, int s0, int boff, const ulonglong2* __restrict__ tw2,
                                        u64 q, u64 two_q) {
    constexpr int EA = Geo<LT>::EA, EB = Geo<LT>::EB, G = Geo<LT>::G;
    constexpr int KB = 1 << EB;
#pragma unroll
    for (int rr = 0; rr < EB; rr++) {
        const int r = INV ? EB - 1 - rr : rr;
        const int hs = KB >> (r + 1);
        const int base = (1 << (s0 + EA + r)) + (boff << (EA + r));
#pragma unroll
        for (int g = 0; g < G; g++) {
#pragma unroll
            for (int k = 0; k < KB; k++) {
                if (k & hs) continue;
                const int idx = base + (((j * G + g) << r) + (k >> (EB - r)));
                const ulonglong2 T = __ldg(tw2 + idx);
                if (!INV) ct_bfly(y[g * KB + k], y[g * KB + k + hs], T.x, T.y, q, two_q);
                else gs_bfly(y[g * KB + k], y[g * KB + k + hs], T.x, T.y, q, two_q);
            }
        }
    }
}

template <int LT>
__device__ __forceinline__ void sm_put_a(u64* line, int j, const u64 (&x)[Geo<LT>::E]) {
#pragma unroll
    for (int k = 0; k < Geo<LT>::E; k++) line[pad(j + Geo<LT>::TPL * k)] = x[k];
}
template <int LT>
__device__ __forceinline__ void sm_get_a(const u64* line, int j, u64 (&x)[Geo<LT>::E]) {
#pragma unroll
    for (int k = 0; k < Geo<LT>::E; k++) x[k] = line[pad(j + Geo<LT>::TPL * k)];
}
template <int LT>
__device__ __forceinline__ void sm_put_b(u64* line, int j, const u64 (&y)[Geo<LT>::E]) {
    constexpr int EB = Geo<LT>::EB, G = Geo<LT>::G, KB = 1 << EB;
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
        for (int k = 0; k < KB; k++) line[pad(((j * G + g) << EB) + k)] = y[g * KB + k];
}
template <int LT>
__device__ __forceinline__ void sm_get_b(const u64* line, int j, u64 (&y)[Geo<LT>::E]) {
    constexpr int EB = Geo<LT>::EB, G = Geo<LT>::G, KB = 1 << EB;
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
        for (int k = 0; k < KB; k++) y[g * KB + k] = line[pad(((j * G + g) << EB) + k)];
}

// Phase A (columns of the R x S limb, R = 2^LT rows).  Forward: stages 0..LT-1; inverse: LT-1..0 then
// x N^{-1} and full reduction.  A CTA owns `lines` consecutive columns (128-byte row segments).
#ifndef NTT_MINB
#define NTT_MINB 4
#endif
template <int LT, bool INV>
__global__ void __launch_bounds__(kThreads, NTT_MINB) ntt_cols_r(NttArgs a, int lines) {
    using GG = Geo<LT>;
    extern __shared__ u64 sm[];
    const int limb = blockIdx.y, poly = blockIdx.z;
    const int mi = a.map.mod[limb];
    const u64 q = a.mod[mi].q, two_q = 2 * q;
    const int S = 1 << a.s2;
    const int c0 = blockIdx.x * lines;
    u64* g = a.base + (i64)poly * a.poly_stride + (i64)limb * a.N;
    const ulonglong2* tw2 = a.tw2 + (size_t)mi * a.N;
    const int tot = GG::T * lines;
    const int lgl = 31 - __clz(lines);
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int r = e >> lgl, c = e & (lines - 1);
        sm[c * GG::LSP + pad(r)] = g[(i64)r * S + c0 + c];
    }
    __syncthreads();
    const int l = threadIdx.x / GG::TPL, j = threadIdx.x % GG::TPL;
    u64* line = sm + l * GG::LSP;
    u64 x[GG::E];
    if (!INV) {
        sm_get_a<LT>(line, j, x);
        round_a<LT, false>(x, 0, 0, tw2, q, two_q);
        sm_put_a<LT>(line, j, x);
        __syncthreads();
        sm_get_b<LT>(line, j, x);
        round_b<LT, false>(x, j, 0, 0, tw2, q, two_q);
        sm_put_b<LT>(line, j, x);
    } else {
        sm_get_b<LT>(line, j, x);
        round_b<LT, true>(x, j, 0, 0, tw2, q, two_q);
        sm_put_b<LT>(line, j, x);
        __syncthreads();
        sm_get_a<LT>(line, j, x);
        round_a<LT, true>(x, 0, 0, tw2, q, two_q);
        const u64 ni = a.ninv[mi], nip = a.ninv_sh[mi];
#pragma unroll
        for (int k = 0; k < GG::E; k++) x[k] = mul_shoup(x[k], ni, nip, q);
        sm_put_a<LT>(line, j, x);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int r = e >> lgl, c = e & (lines - 1);
        g[(i64)r * S + c0 + c] = sm[c * GG::LSP + pad(r)];   // forward: lazy [0, 4q) handed to phase B
    }
}

// Phase B (contiguous chunks of S = 2^LT words).  Forward: stages s1..logN-1 then reduce to [0, q);
// the round-A mapping reads the chunk straight from global memory (coalesced).  Inverse: stages
// logN-1..s1, lazy [0, 2q) output written straight from the round-A registers.
template <int LT, bool INV>
__global__ void __launch_bounds__(kThreads, NTT_MINB) ntt_rows_r(NttArgs a, int lines) {
    using GG = Geo<LT>;
    extern __shared__ u64 sm[];
    const int limb = blockIdx.y, poly = blockIdx.z;
    const int mi = a.map.mod[limb];
    const u64 q = a.mod[mi].q, two_q = 2 * q;
    const int ch0 = blockIdx.x * lines;
    u64* g = a.base + (i64)poly * a.poly_stride + (i64)limb * a.N + (i64)ch0 * GG::T;
    const ulonglong2* tw2 = a.tw2 + (size_t)mi * a.N;
    const int l = threadIdx.x / GG::TPL, j = threadIdx.x % GG::TPL;
    u64* line = sm + l * GG::LSP;
    u64* gl = g + (size_t)l * GG::T;
    const int boff = ch0 + l;
    const int tot = GG::T * lines;
    u64 x[GG::E];
    if (!INV) {
#pragma unroll
        for (int k = 0; k < GG::E; k++) x[k] = gl[j + GG::TPL * k];
        round_a<LT, false>(x, a.s1, boff, tw2, q, two_q);
        sm_put_a<LT>(line, j, x);
        __syncthreads();
        sm_get_b<LT>(line, j, x);
        round_b<LT, false>(x, j, a.s1, boff, tw2, q, two_q);
        sm_put_b<LT>(line, j, x);
        __syncthreads();
        for (int e = threadIdx.x; e < tot; e += blockDim.x) {
            u64 v = sm[(e >> LT) * GG::LSP + pad(e & (GG::T - 1))];
            v = v >= two_q ? v - two_q : v;
            v = v >= q ? v - q : v;
            g[e] = v;
        }
    } else {
        for (int e = threadIdx.x; e < tot; e += blockDim.x) sm[(e >> LT) * GG::LSP + pad(e & (GG::T - 1))] = g[e];
        __syncthreads();
        sm_get_b<LT>(line, j, x);
        round_b<LT, true>(x, j, a.s1, boff, tw2, q, two_q);
        sm_put_b<LT>(line, j, x);
        __syncthreads();
        sm_get_a<LT>(line, j, x);
        round_a<LT, true>(x, a.s1, boff, tw2, q, two_q);
#pragma unroll
        for (int k = 0; k < GG::E; k++) gl[j + GG::TPL * k] = x[k];
    }
}

template <bool INV>
void launch_cols(int LT, dim3 grid, int threads, size_t smem, cudaStream_t s, const NttArgs& a, int lines) {
    switch (LT) {
#define C(LTV) case LTV: ntt_cols_r<LTV, INV><<<grid, threads, smem, s>>>(a, lines); break;
        C(2) C(3) C(4) C(5) C(6) C(7) C(8)
#undef C
        default: throw EncfError(ENCF_ERR_ARG, "ntt: unsupported phase size");
    }
}

template <bool INV>
void launch_rows(int LT, dim3 grid, int threads, size_t smem, cudaStream_t s, const NttArgs& a, int lines) {
    switch (LT) {
#define C(LTV) case LTV: ntt_rows_r<LTV, INV><<<grid, threads, smem, s>>>(a, lines); break;
        C(2) C(3) C(4) C(5) C(6) C(7) C(8)
#undef C
        default: throw EncfError(ENCF_ERR_ARG, "ntt: unsupported phase size");
    }
}

struct PhaseCfg { int lines, threads, blocks; size_t smem; };

PhaseCfg phase_cfg(int LT, int avail) {   // avail = number of lines of one limb in this phase
    const int EA = (LT + 1) / 2, TPL = 1 << (LT - EA);
    int lines = kThreads / TPL;
    if (lines > avail) lines = avail;
    const int T = 1 << LT;
    PhaseCfg p;
    p.lines = lines;
    p.threads = lines * TPL;
    p.blocks = avail / lines;
    p.smem = (size_t)lines * (T + T / 16 + 1) * sizeof(u64);
    return p;
}

NttArgs make_args(encf_ctx& c, const PolyBatch& b, bool inv) {
    NttArgs a;
    a.base = b.base;
    a.poly_stride = b.poly_stride;
    a.map = b.map;
    a.mod = c.d_mod;
    a.tw = inv ? c.d_ipsi : c.d_psi;
    a.tw_sh = inv ? c.d_ipsi_sh : c.d_psi_sh;
    a.tw2 = (const ulonglong2*)(inv ? c.d_itw2 : c.d_tw2);
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
    PhaseCfg A = phase_cfg(c.s1, 1 << c.s2), B = phase_cfg(c.s2, 1 << c.s1);
    int slot;
    c.prof_begin("ntt", s, (uint64_t)b.npolys * b.map.n * c.N * 8 * 4, slot);
    launch_cols<false>(c.s1, dim3(A.blocks, b.map.n, b.npolys), A.threads, A.smem, s, a, A.lines);
    launch_rows<false>(c.s2, dim3(B.blocks, b.map.n, b.npolys), B.threads, B.smem, s, a, B.lines);
    c.prof_end(slot, s);
    c.st_ntt += (uint64_t)b.npolys * b.map.n;
    c.st_launch += 2;
    c.st_bytes += (uint64_t)b.npolys * b.map.n * c.N * 8 * 4;
    CUDA_TRY(cudaGetLastError());
}

void ntt_inverse(encf_ctx& c, const PolyBatch& b, cudaStream_t s) {
    if (b.npolys <= 0 || b.map.n <= 0) return;
    NttArgs a = make_args(c, b, true);
    PhaseCfg A = phase_cfg(c.s1, 1 << c.s2), B = phase_cfg(c.s2, 1 << c.s1);
    int slot;
    c.prof_begin("ntt", s, (uint64_t)b.npolys * b.map.n * c.N * 8 * 4, slot);
    launch_rows<true>(c.s2, dim3(B.blocks, b.map.n, b.npolys), B.threads, B.smem, s, a, B.lines);
    launch_cols<true>(c.s1, dim3(A.blocks, b.map.n, b.npolys), A.threads, A.smem, s, a, A.lines);
    c.prof_end(slot, s);
    c.st_ntt += (uint64_t)b.npolys * b.map.n;
    c.st_launch += 2;
    c.st_bytes += (uint64_t)b.npolys * b.map.n * c.N * 8 * 4;
    CUDA_TRY(cudaGetLastError());
}
