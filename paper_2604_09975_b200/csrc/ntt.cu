// ntt.cu -- negacyclic NTT / iNTT over 64-bit RNS limbs (the ring isomorphism of P:82) for sm_100a.
//
// Forward: merged-twiddle Cooley-Tukey (bit-reversed output), Harvey lazy butterflies in [0, 8q),
// Shoup twiddles.  Inverse: Gentleman-Sande with psi^{-brv(k)} and a final N^{-1}.
// A limb of N = 2^logN words is split N = R x S (R = 2^s1 rows, S = 2^s2 columns):
//   phase A: the first s1 stages only pair elements of one column (stride S) -> a CTA stages a
//            R x 16 column tile through shared memory (128-byte coalesced row segments);
//   phase B: the last s2 stages stay inside contiguous chunks of S words -> a CTA stages a
//            group of chunks.
// (Inverse runs B then A.)  One launch per phase covers every limb of every polynomial of a batch.
#include <cstdlib>
#include <type_traits>
#include "ctx.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kTileElems = 4096;   // 32 KB of shared memory per CTA

struct NttArgs {
    u64* base;
    i64 poly_stride;
    const u64* src_base;     // inverse only: the first phase reads from here -> out-of-place transform
    i64 src_stride;          // polynomial stride of src_base (limb stride N, like base)
    LimbMap map;
    const ModConst* mod;
    const u64* tw;       // psi_brv (fwd) or ipsi_brv (inv): [mods][N]
    const u64* tw_sh;
    const ulonglong2* tw2;   // interleaved {w, w'}: [mods][N]
    const double2* twf;      // FP64 path: {w, w/q}: [mods][N]
    const double* fpc;       // FP64 path: [mods][4] = {q, 1/q, N^-1, N^-1/q}
    u64 fpmask;              // modulus ids on the FP64 path
    // optional forward epilogue (ModDown / rescale finish fused into the last phase): for polynomial p, limb i,
    // instead of the transform y: out_p[i] = (src_p[i] - y) * f_i (+ add_p[i]) mod q_i   (device tables)
    const u64* const* epi_src;
    u64* const* epi_out;
    const u64* const* epi_add;
    const u64* epi_f;
    const u64* epi_fsh;
    const u64* ninv;
    const u64* ninv_sh;
    int apply_ninv;          // 0: inverse leaves the factor N (the consumer's base-conversion constants absorb N^{-1})
    // optional inverse epilogue (apply_ninv = 0): out = x * post_f[limb] mod q (batch limb index), canonical -- the fast
    // base conversion's per-limb input factor [(Q/q_i)^{-1} N^{-1}]_{q_i} applied where the transform writes its output
    const u64* post_f;
    const u64* post_fsh;
    const double* post_fd;   // FP64 path: {f, fl(f / q)} per limb
    int N, logN, s1, s2;
};

// ---------------------------------------------------------------------------------------------
// Integer path (any q < 2^61): Harvey lazy butterflies, Shoup twiddles with an APPROXIMATE high product.
// h' = a1 w1' + hi32(a1 w0') + hi32(a0 w1') (dropping a0 w0' and the carries out of the low word) lies in
// [h - 2, h] for the exact h = hi64(a w'), so a w - h' q = (a w - h q) + (h - h') q is in [0, 4q) (exact Shoup:
// [0, 2q)).  Written in PTX as 3 IMAD.HI + 1 IMAD + carry ops with no 64-bit addend, so ptxas needs no register-pair
// moves (the C form cost IMAD.MOV shuffles on the fmaheavy pipe, which bounds this path at 77 %: profiles/r01_summary.md).
// The wider product range is absorbed by widening the lazy bounds: forward values in [0, 8q), inverse in [0, 4q).
__device__ __forceinline__ u64 mul_shoup_lazy4(u64 a, u64 w, u64 wp, u64 q) {   // [0, 4q)
    unsigned hl, hh;
    asm("{\n\t.reg .u32 a0, a1, p0, p1, t0, t1, c;\n\t"
        "mov.b64 {a0, a1}, %2;\n\t"
        "mov.b64 {p0, p1}, %3;\n\t"
        "mul.hi.u32 t0, a1, p0;\n\t"
        "mad.hi.cc.u32 t1, a0, p1, t0;\n\t"
        "addc.u32 c, 0, 0;\n\t"
        "mad.lo.cc.u32 %0, a1, p1, t1;\n\t"
        "madc.hi.u32 %1, a1, p1, c;\n\t}"
        : "=r"(hl), "=r"(hh) : "l"(a), "l"(wp));
    const u64 h = ((u64)hh << 32) | hl;
    return a * w - h * q;
}

// Forward (CT): X, Y in [0, 8q) -> x = X mod' 4q in [0, 4q), t in [0, 4q): X' = x + t, Y' = x - t + 4q in [0, 8q).
__device__ __forceinline__ void ct_bfly(u64& X, u64& Y, u64 W, u64 Wp, u64 q, u64 four_q) {
    u64 x = X >= four_q ? X - four_q : X;
    u64 t = mul_shoup_lazy4(Y, W, Wp, q);
    X = x + t;
    Y = x - t + four_q;
}

// Inverse (GS): X, Y in [0, 4q) -> X' = (X + Y) mod' 4q, Y' = (X - Y + 4q) W in [0, 4q).
__device__ __forceinline__ void gs_bfly(u64& X, u64& Y, u64 W, u64 Wp, u64 q, u64 four_q) {
    u64 x = X + Y;
    x = x >= four_q ? x - four_q : x;
    u64 t = X - Y + four_q;
    Y = mul_shoup_lazy4(t, W, Wp, q);
    X = x;
}

// [0, 8q) -> [0, q)
__device__ __forceinline__ u64 canon8(u64 v, u64 q) {
    v = v >= 4 * q ? v - 4 * q : v;
    v = v >= 2 * q ? v - 2 * q : v;
    return v >= q ? v - q : v;
}

struct IntOps {
    using T = u64;
    using TW = ulonglong2;
    u64 q, four_q;
    __device__ __forceinline__ void ct(u64& X, u64& Y, TW w) const { ct_bfly(X, Y, w.x, w.y, q, four_q); }
    __device__ __forceinline__ void gs(u64& X, u64& Y, TW w) const { gs_bfly(X, Y, w.x, w.y, q, four_q); }
};

// q = 2^60 - c with c < 2^32 (every 60-bit prime of the parameter sets: NTT-friendly primes just below 2^60):
// h q = (h << 60) - h c, so the Shoup remainder a w - h q = a w + h c - (h << 60) (mod 2^64, the same integer in
// [0, 4q)) needs h c = one IMAD + one IMAD.WIDE.U32 instead of the three products of h q; h << 60 is one shift of
// the low word.  Same words as mul_shoup_lazy4 by construction; NTT_CQ=0 builds without it (A/B).
#ifndef NTT_CQ
#define NTT_CQ 1
#endif
__device__ __forceinline__ u64 mul_shoup_lazy4_c(u64 a, u64 w, u64 wp, uint32_t c) {   // [0, 4q)
    unsigned hl, hh;
    asm("{\n\t.reg .u32 a0, a1, p0, p1, t0, t1, c;\n\t"
        "mov.b64 {a0, a1}, %2;\n\t"
        "mov.b64 {p0, p1}, %3;\n\t"
        "mul.hi.u32 t0, a1, p0;\n\t"
        "mad.hi.cc.u32 t1, a0, p1, t0;\n\t"
        "addc.u32 c, 0, 0;\n\t"
        "mad.lo.cc.u32 %0, a1, p1, t1;\n\t"
        "madc.hi.u32 %1, a1, p1, c;\n\t}"
        : "=r"(hl), "=r"(hh) : "l"(a), "l"(wp));
    u64 hc;
    asm("{\n\t.reg .u32 t, z;\n\t"
        "mul.lo.u32 t, %1, %3;\n\t"
        "mov.u32 z, 0;\n\t"
        "mov.b64 %0, {z, t};\n\t"
        "mad.wide.u32 %0, %2, %3, %0;\n\t}"
        : "=l"(hc) : "r"(hh), "r"(hl), "r"(c));
    return a * w + hc - ((u64)(hl << 28) << 32);
}
struct IntOpsC : IntOps {
    uint32_t c;
    __device__ __forceinline__ void ct(u64& X, u64& Y, TW w) const {
        u64 x = X >= four_q ? X - four_q : X;
        u64 t = mul_shoup_lazy4_c(Y, w.x, w.y, c);
        X = x + t;
        Y = x - t + four_q;
    }
    __device__ __forceinline__ void gs(u64& X, u64& Y, TW w) const {
        u64 x = X + Y;
        x = x >= four_q ? x - four_q : x;
        u64 t = X - Y + four_q;
        Y = mul_shoup_lazy4_c(t, w.x, w.y, c);
        X = x;
    }
};
__device__ __forceinline__ bool is_q60c(u64 q) { return NTT_CQ && q < (1ull << 60) && q > (1ull << 60) - (1ull << 32); }

// ---------------------------------------------------------------------------------------------
// FP64 path (q < 2^41; sm_100a runs DFMA/DMUL/DADD at 64 lanes/clk/SM on the fp64 pipe, while a 64-bit
// Shoup product costs ~32 fmaheavy cycles per warp on the integer side -- tools/micro/pipes.cu).
// Values are integer-valued doubles, SIGNED, |x| < 2^50.  Product a*w mod q (w in [0,q), wq = fl(w/q)):
//   ph = fl(a w), pl = a w - ph (exact by FMA), qt = round(a wq) (exact via the 1.5*2^52 shifter,
//   |a wq| < 2^51), r = fma(-qt, q, ph) + pl = a w - qt q EXACTLY (|.| < 2^53), |qt - a w/q| < 1 => |r| < q.
// Forward (CT): X' = X + r, Y' = X - r -> the bound grows by q per stage (17q < 2^46 after 16 stages).
// Inverse (GS): X' = X + Y doubles per stage -> a centred reduction after the first phase (2^8 * 2q < 2^50).
// Results are canonical [0, q) at the end of every transform: bit-identical to the integer path.
constexpr double kShift = 6755399441055744.0;   // 1.5 * 2^52
constexpr double kTwo52 = 4503599627370496.0;

__device__ __forceinline__ double fp_mulmod(double a, double w, double wq, double q) {
    const double ph = __dmul_rn(a, w);
    const double pl = __fma_rn(a, w, -ph);
    const double qt = __dsub_rn(__fma_rn(a, wq, kShift), kShift);
    return __dadd_rn(__fma_rn(-qt, q, ph), pl);
}
__device__ __forceinline__ double fp_center(double x, double q, double qinv) {   // |result| <= q/2 + 1
    const double qt = __dsub_rn(__fma_rn(x, qinv, kShift), kShift);
    return __fma_rn(-qt, q, x);
}
__device__ __forceinline__ u64 fp_canon(double r, double q) {   // |r| < q + 1 -> [0, q) as u64
    r = r < 0.0 ? __dadd_rn(r, q) : r;
    r = r >= q ? __dsub_rn(r, q) : r;
    return (u64)__double_as_longlong(__dadd_rn(r, kTwo52)) & ((1ull << 52) - 1);
}
__device__ __forceinline__ double fp_from_u64(u64 v) {   // v < 2^52
    return __dsub_rn(__longlong_as_double((long long)(v | 0x4330000000000000ull)), kTwo52);
}

struct FpOps {
    using T = double;
    using TW = double2;
    double q;
    __device__ __forceinline__ void ct(double& X, double& Y, TW w) const {
        const double t = fp_mulmod(Y, w.x, w.y, q);
        const double x = X;
        X = __dadd_rn(x, t);
        Y = __dsub_rn(x, t);
    }
    __device__ __forceinline__ void gs(double& X, double& Y, TW w) const {
        const double sm = __dadd_rn(X, Y), df = __dsub_rn(X, Y);
        Y = fp_mulmod(df, w.x, w.y, q);
        X = sm;
    }
};

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
#ifndef NTT_SMTW
#define NTT_SMTW 1   // shared-memory twiddle tables (tw_load / tw_store); 0 = per-butterfly __ldg (A/B variant)
#endif
// entry e of a shared twiddle table sits at e + e/8: round B reads entries j << r apart (r <= 3) across the threads j
// of a line, which would otherwise all fall in one 16-byte bank group
__device__ __forceinline__ int tw_pad(int e) { return e + (e >> 3); }

// Round A: local stages 0..EA-1 (forward ascending / inverse descending).  Local block index of the
// pair (k, k+hs) at local stage s is k >> (EA - s); global twiddle index 2^(s0+s) + (boff << s) + blk.
template <int LT, bool INV, class Ops, bool SMTW = false>
__device__ __forceinline__ void round_a(typename Ops::T (&x)[Geo<LT>::E], int s0, int boff,
                                        const typename Ops::TW* __restrict__ tw2, const Ops& ops) {
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
            const typename Ops::TW T = SMTW ? tw2[tw_pad(idx)] : __ldg(tw2 + idx);
            if (!INV) ops.ct(x[k], x[k + hs], T);
            else ops.gs(x[k], x[k + hs], T);
        }
    }
}

// Round B: local stages EA..LT-1.  Element ((j*G+g) << EB) + k'; block index at local stage EA+r is
// ((j*G+g) << r) + (k' >> (EB - r)).
template <int LT, bool INV, class Ops, bool SMTW = false>
__device__ __forceinline__ void round_b(typename Ops::T (&y)[Geo<LT>::E], int j, int s0, int boff,
                                        const typename Ops::TW* __restrict__ tw2, const Ops& ops) {
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
                const typename Ops::TW T = SMTW ? tw2[tw_pad(idx)] : __ldg(tw2 + idx);
                if (!INV) ops.ct(y[g * KB + k], y[g * KB + k + hs], T);
                else ops.gs(y[g * KB + k], y[g * KB + k + hs], T);
            }
        }
    }
}

template <int LT, class T>
__device__ __forceinline__ void sm_put_a(T* line, int j, const T (&x)[Geo<LT>::E]) {
#pragma unroll
    for (int k = 0; k < Geo<LT>::E; k++) line[pad(j + Geo<LT>::TPL * k)] = x[k];
}
template <int LT, class T>
__device__ __forceinline__ void sm_get_a(const T* line, int j, T (&x)[Geo<LT>::E]) {
#pragma unroll
    for (int k = 0; k < Geo<LT>::E; k++) x[k] = line[pad(j + Geo<LT>::TPL * k)];
}
template <int LT, class T>
__device__ __forceinline__ void sm_put_b(T* line, int j, const T (&y)[Geo<LT>::E]) {
    constexpr int EB = Geo<LT>::EB, G = Geo<LT>::G, KB = 1 << EB;
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
        for (int k = 0; k < KB; k++) line[pad(((j * G + g) << EB) + k)] = y[g * KB + k];
}
template <int LT, class T>
__device__ __forceinline__ void sm_get_b(const T* line, int j, T (&y)[Geo<LT>::E]) {
    constexpr int EB = Geo<LT>::EB, G = Geo<LT>::G, KB = 1 << EB;
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
        for (int k = 0; k < KB; k++) y[g * KB + k] = line[pad(((j * G + g) << EB) + k)];
}

// Shared-memory twiddle table of one phase (the L1TEX pipe bounded the rows phase at 84 % with a per-butterfly
// __ldg of its chunk's twiddles, profiles/r02_summary.md): entry i = 2^t + blk (t < LT, blk < 2^t) holds the twiddle of
// local stage t, block blk of chunk c at global stage s0 + t, i.e. tw[2^(s0+t) + (c << t) + blk]; the rounds then index
// it with s0 = 0, boff = 0.  Placed after the phase's data tile (lines x LSP words, rounded to 16 bytes).
// Split in two so the table's load overlaps the phase's data loads: tw_load issues this thread's entry (one per thread,
// 2^LT - 1 <= blockDim entries), tw_store writes it after the data loads are in flight; the caller's next
// __syncthreads publishes the table.
template <int LT, class TW>
__device__ __forceinline__ TW tw_load(const TW* __restrict__ tw2, int s0, int c) {
    const int i = threadIdx.x + 1;
    if (i >= (1 << LT)) return TW{};
    const int t = 31 - __clz(i), blk = i - (1 << t);
    return __ldg(tw2 + (1 << (s0 + t)) + (c << t) + blk);
}
template <int LT, class TW>
__device__ __forceinline__ TW* tw_table(u64* sm_raw, int lines) {
    return reinterpret_cast<TW*>(sm_raw + ((lines * Geo<LT>::LSP + 1) & ~1));
}
template <int LT, class TW>
__device__ __forceinline__ void tw_store(TW* stw, TW v) {
    const int i = threadIdx.x + 1;
    if (i < (1 << LT)) stw[tw_pad(i)] = v;
}

// global word <-> working value.  FIRST: the transform's first phase reads canonical u64 words; later
// phases of the FP64 path read/write raw double bits (signed intermediates), the integer path lazy u64.
__device__ __forceinline__ u64 ld_val(u64 v, const IntOps&, bool) { return v; }
__device__ __forceinline__ double ld_val(u64 v, const FpOps&, bool first) {
    return first ? fp_from_u64(v) : __longlong_as_double((long long)v);
}
__device__ __forceinline__ u64 st_raw(u64 v) { return v; }
__device__ __forceinline__ u64 st_raw(double v) { return (u64)__double_as_longlong(v); }

// Phase A (columns of the R x S limb, R = 2^LT rows).  Forward: stages 0..LT-1 (first phase); inverse:
// LT-1..0 then x N^{-1} and full reduction (last phase).  A CTA owns `lines` consecutive columns.
#ifndef NTT_MINB
#define NTT_MINB 4
#endif
// Thread t of the CTA is (line l = t % lines, j = t / lines): a warp's 32 threads cover consecutive COLUMNS,
// so the round-A register mapping (rows j + TPL k of column l) is read (forward) / written (inverse) straight
// from/to global memory in coalesced row segments; only the round-B mapping goes through shared memory.
template <int LT, bool INV, class Ops>
__device__ __forceinline__ void cols_body(const NttArgs& a, int lines, const Ops& ops, const typename Ops::TW* tw2, int mi,
                                          int bx, int by, int bz) {
    using GG = Geo<LT>;
    using T = typename Ops::T;
    extern __shared__ u64 sm_raw[];
    T* sm = reinterpret_cast<T*>(sm_raw);
    const int limb = by, poly = bz;
    const int S = 1 << a.s2;
    const int c0 = bx * lines;
    u64* g = a.base + (i64)poly * a.poly_stride + (i64)limb * a.N;
    const int lgl = 31 - __clz(lines);
    const int l = threadIdx.x & (lines - 1), j = threadIdx.x >> lgl;
    T* line = sm + l * GG::LSP;
    u64* gc = g + c0 + l + (i64)j * S;            // row j of column c0 + l
    using TWT = typename Ops::TW;
#if NTT_SMTW
    TWT* stw = tw_table<LT, TWT>(sm_raw, lines);
    const TWT twv = tw_load<LT>(tw2, 0, 0);
#else
    const TWT* stw = tw2;   // variant: per-butterfly __ldg twiddles (index formula with s0 = 0, boff = 0 is the same)
#endif
    const i64 rs = (i64)GG::TPL * S;              // TPL rows
    T x[GG::E];
    if (!INV) {
        {
            u64 v[GG::E];
#pragma unroll
            for (int k = 0; k < GG::E; k++) v[k] = __ldcg(gc + k * rs);
#if NTT_SMTW
            tw_store<LT>(stw, twv);
            __syncthreads();
#endif
#pragma unroll
            for (int k = 0; k < GG::E; k++) x[k] = ld_val(v[k], ops, true);
        }
        round_a<LT, false, Ops, NTT_SMTW>(x, 0, 0, stw, ops);
        sm_put_a<LT>(line, j, x);
        __syncthreads();
        sm_get_b<LT>(line, j, x);
        round_b<LT, false, Ops, NTT_SMTW>(x, j, 0, 0, stw, ops);
        sm_put_b<LT>(line, j, x);
        __syncthreads();
        const int tot = GG::T * lines;
        for (int e = threadIdx.x; e < tot; e += blockDim.x) {
            const int r = e >> lgl, c = e & (lines - 1);
            const T v = sm[c * GG::LSP + pad(r)];
            g[(i64)r * S + c0 + c] = st_raw(v);    // forward: lazy u64 [0, 8q) / raw double bits to phase B
        }
    } else {
        {   // all E loads of a thread in flight before the first use (tot = E * blockDim.x)
            u64 v[GG::E];
#pragma unroll
            for (int it = 0; it < GG::E; it++) {
                const int e = threadIdx.x + it * blockDim.x;
                v[it] = __ldcg(g + (i64)(e >> lgl) * S + c0 + (e & (lines - 1)));
            }
#if NTT_SMTW
            tw_store<LT>(stw, twv);
#endif
#pragma unroll
            for (int it = 0; it < GG::E; it++) {
                const int e = threadIdx.x + it * blockDim.x;
                sm[(e & (lines - 1)) * GG::LSP + pad(e >> lgl)] = ld_val(v[it], ops, false);
            }
        }
        __syncthreads();
        sm_get_b<LT>(line, j, x);
        round_b<LT, true, Ops, NTT_SMTW>(x, j, 0, 0, stw, ops);
        sm_put_b<LT>(line, j, x);
        __syncthreads();
        sm_get_a<LT>(line, j, x);
        round_a<LT, true, Ops, NTT_SMTW>(x, 0, 0, stw, ops);
        if constexpr (std::is_same<T, u64>::value) {
            if (a.apply_ninv) {
                const u64 ni = a.ninv[mi], nip = a.ninv_sh[mi];
#pragma unroll
                for (int k = 0; k < GG::E; k++) gc[k * rs] = mul_shoup(x[k], ni, nip, ops.q);
            } else if (a.post_f) {
                const u64 f = a.post_f[limb], fs = a.post_fsh[limb];
#pragma unroll
                for (int k = 0; k < GG::E; k++) gc[k * rs] = mul_shoup(x[k], f, fs, ops.q);
            } else {
#pragma unroll
                for (int k = 0; k < GG::E; k++) gc[k * rs] = canon8(x[k], ops.q);   // GS outputs in [0, 4q)
            }
        } else {
            if (a.apply_ninv) {
                const double ni = a.fpc[4 * mi + 2], niq = a.fpc[4 * mi + 3];
#pragma unroll
                for (int k = 0; k < GG::E; k++) gc[k * rs] = fp_canon(fp_mulmod(x[k], ni, niq, ops.q), ops.q);
            } else if (a.post_f) {
                const double f = a.post_fd[2 * limb], fq = a.post_fd[2 * limb + 1];
#pragma unroll
                for (int k = 0; k < GG::E; k++) gc[k * rs] = fp_canon(fp_mulmod(x[k], f, fq, ops.q), ops.q);
            } else {
                const double qinv = a.fpc[4 * mi + 1];
#pragma unroll
                for (int k = 0; k < GG::E; k++) gc[k * rs] = fp_canon(fp_center(x[k], ops.q, qinv), ops.q);
            }
        }
    }
}

template <int LT, bool INV>
__global__ void __launch_bounds__(kThreads, NTT_MINB) ntt_cols_r(NttArgs a, int lines) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // predecessor's writes visible (PDL)
    const int mi = a.map.mod[blockIdx.y];
    if ((a.fpmask >> mi) & 1ull) {
        cols_body<LT, INV>(a, lines, FpOps{a.fpc[4 * mi]}, a.twf + (size_t)mi * a.N, mi, blockIdx.x, blockIdx.y, blockIdx.z);
    } else {
        const u64 q = a.mod[mi].q;
        if (is_q60c(q))
            cols_body<LT, INV>(a, lines, IntOpsC{{q, 4 * q}, (uint32_t)((1ull << 60) - q)}, a.tw2 + (size_t)mi * a.N, mi, blockIdx.x,
                               blockIdx.y, blockIdx.z);
        else
            cols_body<LT, INV>(a, lines, IntOps{q, 4 * q}, a.tw2 + (size_t)mi * a.N, mi, blockIdx.x, blockIdx.y, blockIdx.z);
    }
}

// Phase B (contiguous chunks of S = 2^LT words).  Forward: stages s1..logN-1 then reduce to [0, q)
// (last phase); the round-A mapping reads the chunk straight from global memory (coalesced).  Inverse:
// stages logN-1..s1 (first phase), lazy output written straight from the round-A registers.
// Line l of a CTA = chunk (blockIdx.x << lgc) + (l & (LC-1)) of polynomial (blockIdx.z << lgp) + (l >> lgc),
// LC = 2^lgc chunks x LP = lines / LC polynomials: with LC = 1 every line of the CTA is the SAME chunk of a
// different polynomial, so all lines share one twiddle set (L1-resident) instead of 16 distinct ones.
template <int LT, bool INV, class Ops>
__device__ __forceinline__ void rows_body(const NttArgs& a, int lines, int lgc, const Ops& ops, const typename Ops::TW* tw2,
                                          int mi, int bx, int by, int bz) {
    using GG = Geo<LT>;
    using T = typename Ops::T;
    extern __shared__ u64 sm_raw[];
    T* sm = reinterpret_cast<T*>(sm_raw);
    const int limb = by;
    const int cmask = (1 << lgc) - 1;
    u64* g0 = a.base + (i64)limb * a.N;
    auto line_off = [&](int ll, i64 pstride) -> i64 {
        return (i64)((bz << (31 - __clz(lines) - lgc)) + (ll >> lgc)) * pstride + (i64)((bx << lgc) + (ll & cmask)) * GG::T;
    };
    auto line_ptr = [&](int ll) -> u64* { return g0 + line_off(ll, a.poly_stride); };
    const int l = threadIdx.x / GG::TPL, j = threadIdx.x % GG::TPL;
    T* line = sm + l * GG::LSP;
    u64* gl = line_ptr(l);
    const int boff = (bx << lgc) + (l & cmask);
    const int tot = GG::T * lines;
    T x[GG::E];
    // every line of the CTA is the same chunk (lgc = 0): its twiddles go through a shared-memory table
    using TWT = typename Ops::TW;
    const bool use_tab = NTT_SMTW && lgc == 0;
    TWT* stw = use_tab ? tw_table<LT, TWT>(sm_raw, lines) : nullptr;
    const TWT twv = use_tab ? tw_load<LT>(tw2, a.s1, bx) : TWT{};
    auto rA = [&](auto inv_tag) {
        constexpr bool I = decltype(inv_tag)::value;
        if (stw) round_a<LT, I, Ops, true>(x, 0, 0, stw, ops); else round_a<LT, I>(x, a.s1, boff, tw2, ops);
    };
    auto rB = [&](auto inv_tag) {
        constexpr bool I = decltype(inv_tag)::value;
        if (stw) round_b<LT, I, Ops, true>(x, j, 0, 0, stw, ops); else round_b<LT, I>(x, j, a.s1, boff, tw2, ops);
    };
    if (!INV) {
#pragma unroll
        for (int k = 0; k < GG::E; k++) x[k] = ld_val(__ldcg(gl + j + GG::TPL * k), ops, false);
        if (use_tab) { tw_store<LT>(stw, twv); __syncthreads(); }
        rA(std::false_type{});
        sm_put_a<LT>(line, j, x);
        __syncthreads();
        sm_get_b<LT>(line, j, x);
        rB(std::false_type{});
        sm_put_b<LT>(line, j, x);
        __syncthreads();
        const u64 qi = a.mod[mi].q;
        const int lgp = 31 - __clz(lines) - lgc;
        if (a.epi_out) {
            // fused ModDown / rescale finish: all E (src, add) loads of a thread in flight before the first use
            const u64 f = a.epi_f[limb], fsh = a.epi_fsh[limb];
            constexpr int HB = GG::E >= 8 ? 8 : GG::E;      // batches of 8 items: 16 loads in flight per thread
#pragma unroll
            for (int b0 = 0; b0 < GG::E; b0 += HB) {
                u64 sv[HB], av[HB];
#pragma unroll
                for (int i2 = 0; i2 < HB; i2++) {
                    const int e = threadIdx.x + (b0 + i2) * blockDim.x;
                    const int ll = e >> LT;
                    const int p = (bz << lgp) + (ll >> lgc);
                    const size_t off = (size_t)limb * a.N + (size_t)(((bx << lgc) + (ll & cmask)) * GG::T + (e & (GG::T - 1)));
                    sv[i2] = a.epi_src[p][off];
                    const u64* ad = a.epi_add[p];
                    av[i2] = ad ? ad[off] : 0;
                }
#pragma unroll
                for (int i2 = 0; i2 < HB; i2++) {
                    const int e = threadIdx.x + (b0 + i2) * blockDim.x;
                    const T v = sm[(e >> LT) * GG::LSP + pad(e & (GG::T - 1))];
                    u64 w;
                    if constexpr (std::is_same<T, u64>::value) {
                        w = canon8(v, ops.q);
                    } else {
                        const double q = ops.q, qinv = a.fpc[4 * mi + 1];
                        w = fp_canon(fp_center(v, q, qinv), q);
                    }
                    const int ll = e >> LT;
                    const int p = (bz << lgp) + (ll >> lgc);
                    const size_t off = (size_t)limb * a.N + (size_t)(((bx << lgc) + (ll & cmask)) * GG::T + (e & (GG::T - 1)));
                    a.epi_out[p][off] = add_mod(mul_shoup(sub_mod(sv[i2], w, qi), f, fsh, qi), av[i2], qi);
                }
            }
            return;
        }
        for (int e = threadIdx.x; e < tot; e += blockDim.x) {
            const T v = sm[(e >> LT) * GG::LSP + pad(e & (GG::T - 1))];
            u64 w;
            if constexpr (std::is_same<T, u64>::value) {
                w = canon8(v, ops.q);
            } else {
                const double q = ops.q, qinv = a.fpc[4 * mi + 1];
                w = fp_canon(fp_center(v, q, qinv), q);
            }
            line_ptr(e >> LT)[e & (GG::T - 1)] = w;
        }
    } else {
        u64 v[GG::E];   // all E loads in flight before the first use (tot = E * blockDim.x)
#pragma unroll
        for (int it = 0; it < GG::E; it++) {
            const int e = threadIdx.x + it * blockDim.x;
            const u64* lp = a.src_base ? a.src_base + (i64)limb * a.N + line_off(e >> LT, a.src_stride) : line_ptr(e >> LT);
            v[it] = __ldcg(lp + (e & (GG::T - 1)));
        }
        if (use_tab) tw_store<LT>(stw, twv);
#pragma unroll
        for (int it = 0; it < GG::E; it++) {
            const int e = threadIdx.x + it * blockDim.x;
            sm[(e >> LT) * GG::LSP + pad(e & (GG::T - 1))] = ld_val(v[it], ops, true);
        }
        __syncthreads();
        sm_get_b<LT>(line, j, x);
        rB(std::true_type{});
        sm_put_b<LT>(line, j, x);
        __syncthreads();
        sm_get_a<LT>(line, j, x);
        rA(std::true_type{});
        if constexpr (std::is_same<T, u64>::value) {
#pragma unroll
            for (int k = 0; k < GG::E; k++) gl[j + GG::TPL * k] = x[k];
        } else {
            const double qinv = a.fpc[4 * mi + 1];
#pragma unroll
            for (int k = 0; k < GG::E; k++) gl[j + GG::TPL * k] = st_raw(fp_center(x[k], ops.q, qinv));
        }
    }
}

template <int LT, bool INV>
__global__ void __launch_bounds__(kThreads, NTT_MINB) ntt_rows_r(NttArgs a, int lines, int lgc) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // predecessor's writes visible (PDL)
    const int mi = a.map.mod[blockIdx.y];
    if ((a.fpmask >> mi) & 1ull) {
        rows_body<LT, INV>(a, lines, lgc, FpOps{a.fpc[4 * mi]}, a.twf + (size_t)mi * a.N, mi, blockIdx.x, blockIdx.y, blockIdx.z);
    } else {
        const u64 q = a.mod[mi].q;
        if (is_q60c(q))
            rows_body<LT, INV>(a, lines, lgc, IntOpsC{{q, 4 * q}, (uint32_t)((1ull << 60) - q)}, a.tw2 + (size_t)mi * a.N, mi,
                               blockIdx.x, blockIdx.y, blockIdx.z);
        else
            rows_body<LT, INV>(a, lines, lgc, IntOps{q, 4 * q}, a.tw2 + (size_t)mi * a.N, mi, blockIdx.x, blockIdx.y, blockIdx.z);
    }
}

// ---------------------------------------------------------------------------------------------
// Fused two-phase transform (ENCF_NTT_FUSED=1; off by default, see ntt_fused): ONE persistent launch runs both
// phases of every limb transform of a batch.  A unit = (limb e, group of LP polynomials) has T1 first-phase tiles and
// T2 second-phase tiles (the same tiles the two-launch path runs).  CTAs draw tickets from a global counter in the
// order [first phase of units 0..D-1] then, per k, [first phase of unit k+D | second phase of unit k]: a unit's
// second phase starts ~D units after its first phase, while the intermediate words (D x LP x 512 KB, ~24 MB) are
// still in the 126 MB L2 -- so the transform reads and writes HBM once instead of twice.  A second-phase tile waits
// (acquire) until the T1 first-phase tiles of its unit have signalled (release); tickets are drawn in order by
// resident CTAs, so every awaited tile is already running (no deadlock).  Data loads bypass L1 (ld.global.cg).
struct FusedSched {
    int* ticket;     // [1] ticket counter, zeroed before the launch
    int* cnt;        // [U] finished first-phase tiles per unit, zeroed before the launch
    int U, D, T1, T2, total;
    int nlimbs, LP, Ab;        // units: u = pg * nlimbs + e; cols tiles per unit = Ab x LP
    int lines_c, lines_r, lgc; // cols-phase lines, rows-phase lines, rows-phase log2(chunks per CTA)
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int LTC, int LTR, bool INV>
#ifndef NTT_FUSED_MINB
#define NTT_FUSED_MINB 3
#endif
__global__ void __launch_bounds__(kThreads, NTT_FUSED_MINB) ntt_fused_r(NttArgs a, FusedSched f) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // predecessor's writes visible (PDL)
    __shared__ int s_t;
    const int nP1 = f.D * f.T1, nMid = (f.U - f.D) * (f.T1 + f.T2);
    while (true) {
        __syncthreads();                                   // previous tile's shared-memory reads are done
        if (threadIdx.x == 0) s_t = atomicAdd(f.ticket, 1);
        __syncthreads();
        const int t = s_t;
        if (t >= f.total) break;
        int phase, u, r;
        if (t < nP1) { phase = 1; u = t / f.T1; r = t % f.T1; }
        else if (t - nP1 < nMid) {
            const int t1 = t - nP1, k = t1 / (f.T1 + f.T2), rr = t1 % (f.T1 + f.T2);
            if (rr < f.T1) { phase = 1; u = k + f.D; r = rr; } else { phase = 2; u = k; r = rr - f.T1; }
        } else {
            const int t2 = t - nP1 - nMid;
            phase = 2; u = f.U - f.D + t2 / f.T2; r = t2 % f.T2;
        }
        if (phase == 2) {
            if (threadIdx.x == 0)
                while (ld_acquire_gpu(f.cnt + u) < f.T1) __nanosleep(64);
            __syncthreads();
        }
        const int e = u % f.nlimbs, pg = u / f.nlimbs;
        const int mi = a.map.mod[e];
        const bool fp = (a.fpmask >> mi) & 1ull;
        if ((phase == 1) != INV) {    // columns phase (forward first / inverse second)
            const int bx = r % f.Ab, bz = pg * f.LP + r / f.Ab;
            if (fp) cols_body<LTC, INV>(a, f.lines_c, FpOps{a.fpc[4 * mi]}, a.twf + (size_t)mi * a.N, mi, bx, e, bz);
            else { const u64 q = a.mod[mi].q; cols_body<LTC, INV>(a, f.lines_c, IntOps{q, 4 * q}, a.tw2 + (size_t)mi * a.N, mi, bx, e, bz); }
        } else {
            if (fp) rows_body<LTR, INV>(a, f.lines_r, f.lgc, FpOps{a.fpc[4 * mi]}, a.twf + (size_t)mi * a.N, mi, r, e, pg);
            else { const u64 q = a.mod[mi].q; rows_body<LTR, INV>(a, f.lines_r, f.lgc, IntOps{q, 4 * q}, a.tw2 + (size_t)mi * a.N, mi, r, e, pg); }
        }
        if (phase == 1) {
            __syncthreads();                               // every thread's words are ordered before thread 0's release
            if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(f.cnt + u) : "memory");
        }
    }
}

// Programmatic dependent launch (ENCF_PDL, default on): every NTT phase kernel is launched with the programmatic
// stream-serialization attribute and waits (griddepcontrol.wait) for its predecessor's memory before its first
// load, so its CTA launch and index set-up overlap the predecessor's tail instead of a full launch gap.
#ifndef NTT_PDL
#define NTT_PDL 1
#endif
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, int threads, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = NTT_PDL;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <bool INV>
void launch_cols(int LT, dim3 grid, int threads, size_t smem, cudaStream_t s, const NttArgs& a, int lines) {
    switch (LT) {
#define C(LTV) case LTV: launch_pdl(ntt_cols_r<LTV, INV>, grid, threads, smem, s, a, lines); break;
        C(2) C(3) C(4) C(5) C(6) C(7) C(8)
#undef C
        default: throw EncfError(ENCF_ERR_ARG, "ntt: unsupported phase size");
    }
}

template <bool INV>
void launch_rows(int LT, dim3 grid, int threads, size_t smem, cudaStream_t s, const NttArgs& a, int lines, int lgc) {
    switch (LT) {
#define C(LTV) case LTV: launch_pdl(ntt_rows_r<LTV, INV>, grid, threads, smem, s, a, lines, lgc); break;
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
    p.smem = ((size_t)lines * (T + T / 16 + 1) + 1) / 2 * 2 * sizeof(u64) + (size_t)(T + T / 8) * 16;   // data | twiddles
    return p;
}

// Rows-phase grid: LP polynomials x LC chunks per CTA (LP = the largest power of two <= lines dividing npolys,
// unless ENCF_NTT_ROWS_CHUNK_MAJOR is set).
struct RowsCfg { dim3 grid; int lgc; };
RowsCfg rows_cfg(const PhaseCfg& B, int nchunks, int npolys, int nlimbs) {
    int lp = 1;
    static const bool chunk_major = std::getenv("ENCF_NTT_ROWS_CHUNK_MAJOR") != nullptr;
    if (!chunk_major)
        while (lp * 2 <= B.lines && npolys % (lp * 2) == 0) lp *= 2;
    const int lc = B.lines / lp;
    int lgc = 0;
    while ((1 << lgc) < lc) lgc++;
    return RowsCfg{dim3(nchunks / lc, nlimbs, npolys / lp), lgc};
}

// Polynomials per launch pair: ENCF_NTT_CHUNK_MB MB of limbs, at least one polynomial; 0 (default) = the whole
// batch in one pair.  Splitting at polynomial granularity keeps every launch's grid identical in shape, so the
// results are the same words either way.
int ntt_chunk_polys(const encf_ctx& c, const PolyBatch& b) {
    // default OFF: measured on the B200 (profiles/r02_summary.md) a 32 MB chunking made the layer's NTT time 29.2 -> 36.1 ms
    // and 64 MB -> 32.6 ms (more, smaller launches; the big batches were not L2-miss-bound enough to win it back)
    static const long mb = [] { const char* e = std::getenv("ENCF_NTT_CHUNK_MB"); return e ? std::atol(e) : 0L; }();
    if (mb <= 0) return b.npolys;
    const long per = (long)b.map.n * c.N * 8;
    return (int)std::max(1L, std::min((long)b.npolys, mb * (1L << 20) / per));
}

// Fused persistent launch (see ntt_fused_r) for 2^12 <= N <= 2^16; returns false when not applicable.
template <int LTC, int LTR>
bool fused_launch(encf_ctx& c, const NttArgs& a, const PolyBatch& b, bool inv, cudaStream_t s) {
    const PhaseCfg A = phase_cfg(LTC, 1 << LTR), B = phase_cfg(LTR, 1 << LTC);
    if (A.threads != kThreads || B.threads != kThreads) return false;
    const RowsCfg R = rows_cfg(B, 1 << LTC, b.npolys, b.map.n);
    const int LP = (int)R.grid.z == 0 ? 1 : b.npolys / (int)R.grid.z;
    FusedSched f;
    f.nlimbs = b.map.n;
    f.LP = LP;
    f.Ab = A.blocks;
    f.lines_c = A.lines;
    f.lines_r = B.lines;
    f.lgc = R.lgc;
    f.U = (b.npolys / LP) * b.map.n;
    const int Tc = A.blocks * LP, Tr = (int)R.grid.x;
    f.T1 = inv ? Tr : Tc;
    f.T2 = inv ? Tc : Tr;
    f.total = f.U * (f.T1 + f.T2);
    const size_t smem = std::max(A.smem, B.smem);
    auto kern = inv ? ntt_fused_r<LTC, LTR, true> : ntt_fused_r<LTC, LTR, false>;
    static int nsm = 0;
    static int occ[2] = {0, 0};
    if (!nsm) CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c.device));
    int& oc = occ[inv ? 1 : 0];
    if (!oc) {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, kern, kThreads, smem));
        if (oc < 1) oc = 1;
    }
    const int grid = std::min(f.total, nsm * oc);
    // delay D: enough units that a unit's first phase has finished when its second phase is drawn, few enough that
    // the intermediate words of the units in flight stay well inside L2 (48 MB)
    const long unit_bytes = (long)LP * c.N * 8;
    int D = (grid + f.T1 - 1) / f.T1 + 1;
    D = (int)std::min<long>(D, std::max(1L, (48L << 20) / unit_bytes));
    f.D = std::max(1, std::min(D, f.U));
    Scratch sc(s);
    int* buf = (int*)sc.get((size_t)(f.U + 2) / 2 + 1);
    CUDA_TRY(cudaMemsetAsync(buf, 0, (size_t)(f.U + 1) * sizeof(int), s));
    f.ticket = buf;
    f.cnt = buf + 1;
    launch_pdl(kern, dim3(grid), kThreads, smem, s, a, f);
    return true;
}

bool ntt_fused(encf_ctx& c, const NttArgs& a, const PolyBatch& b, bool inv, cudaStream_t s) {
    // default OFF: measured on the B200 the fused launch made the layer's NTT time 25.0 -> 29.4 ms (profiles/r02_summary.md)
    static const bool on = [] { const char* e = std::getenv("ENCF_NTT_FUSED"); return e && std::atoi(e) != 0; }();
    // small batches (under one wave: <= ENCF_NTT_FUSED_SMALL limb transforms): one launch instead of two (A/B knob)
    static const int small = [] { const char* e = std::getenv("ENCF_NTT_FUSED_SMALL"); return e ? std::atoi(e) : 0; }();
    if (!on && !(small > 0 && b.npolys * b.map.n <= small)) return false;
    switch (c.logN) {
        case 12: return fused_launch<6, 6>(c, a, b, inv, s);
        case 13: return fused_launch<6, 7>(c, a, b, inv, s);
        case 14: return fused_launch<7, 7>(c, a, b, inv, s);
        case 15: return fused_launch<7, 8>(c, a, b, inv, s);
        case 16: return fused_launch<8, 8>(c, a, b, inv, s);
        default: return false;
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
    a.tw2 = (const ulonglong2*)(inv ? c.d_itw2 : c.d_tw2);
    a.twf = (const double2*)(inv ? c.d_itwf : c.d_twf);
    a.fpc = c.d_fpc;
    a.fpmask = c.fpmask;
    a.ninv = c.d_ninv;
    a.ninv_sh = c.d_ninv_sh;
    a.apply_ninv = 1;
    a.post_f = a.post_fsh = nullptr;
    a.post_fd = nullptr;
    a.src_base = nullptr;
    a.src_stride = b.poly_stride;
    a.epi_src = nullptr;
    a.epi_out = nullptr;
    a.epi_add = nullptr;
    a.epi_f = a.epi_fsh = nullptr;
    a.N = c.N;
    a.logN = c.logN;
    a.s1 = c.s1;
    a.s2 = c.s2;
    return a;
}

}  // namespace

void ntt_forward(encf_ctx& c, const PolyBatch& b, cudaStream_t s) { ntt_forward_epi(c, b, nullptr, s); }

void ntt_forward_epi(encf_ctx& c, const PolyBatch& b, const NttEpilogue* epi, cudaStream_t s) {
    if (b.npolys <= 0 || b.map.n <= 0) return;
    NttArgs a = make_args(c, b, false);
    if (epi) {
        a.epi_src = epi->src; a.epi_out = epi->out; a.epi_add = epi->add; a.epi_f = epi->f; a.epi_fsh = epi->fsh;
    }
    PhaseCfg A = phase_cfg(c.s1, 1 << c.s2), B = phase_cfg(c.s2, 1 << c.s1);
    int slot;
    c.prof_begin("ntt", s, (uint64_t)b.npolys * b.map.n * c.N * 8 * 4, slot);
    // L2-sized chunks of polynomials: the rows phase of a chunk re-reads what the columns phase just wrote while it
    // is still in the 126 MB L2, instead of after a whole multi-hundred-MB batch has streamed through
    const bool fused = ntt_fused(c, a, b, false, s);
    const int cp = fused ? b.npolys : ntt_chunk_polys(c, b);
    for (int p0 = 0; !fused && p0 < b.npolys; p0 += cp) {
        const int np = std::min(cp, b.npolys - p0);
        NttArgs ac = a;
        ac.base = a.base + (i64)p0 * a.poly_stride;
        if (epi) { ac.epi_src = a.epi_src + p0; ac.epi_out = a.epi_out + p0; ac.epi_add = a.epi_add + p0; }
        launch_cols<false>(c.s1, dim3(A.blocks, b.map.n, np), A.threads, A.smem, s, ac, A.lines);
        const RowsCfg R = rows_cfg(B, 1 << c.s1, np, b.map.n);
        launch_rows<false>(c.s2, R.grid, B.threads, B.smem, s, ac, B.lines, R.lgc);
        c.st_launch += 2;
    }
    c.st_launch -= fused ? 1 : 2;
    c.prof_end(slot, s);
    c.st_ntt += (uint64_t)b.npolys * b.map.n;
    {
        int nfp = 0;
        for (int i = 0; i < b.map.n; i++) nfp += (int)((c.fpmask >> b.map.mod[i]) & 1ull);
        c.st_ntt_fp += (uint64_t)b.npolys * nfp;
    }
    c.st_launch += 2;
    c.st_bytes += (uint64_t)b.npolys * b.map.n * c.N * 8 * 4;
    CUDA_TRY(cudaGetLastError());
}

void ntt_inverse(encf_ctx& c, const PolyBatch& b, cudaStream_t s) { ntt_inverse_scaled(c, b, true, s); }

void ntt_inverse_scaled(encf_ctx& c, const PolyBatch& b, bool apply_ninv, cudaStream_t s, const u64* src, const NttPost* post,
                        i64 src_stride) {
    if (b.npolys <= 0 || b.map.n <= 0) return;
    NttArgs a = make_args(c, b, true);
    a.apply_ninv = apply_ninv ? 1 : 0;
    if (post && !apply_ninv) { a.post_f = post->f; a.post_fsh = post->fsh; a.post_fd = post->fd; }
    a.src_base = src;
    if (src_stride >= 0) a.src_stride = src_stride;
    PhaseCfg A = phase_cfg(c.s1, 1 << c.s2), B = phase_cfg(c.s2, 1 << c.s1);
    int slot;
    c.prof_begin("ntt", s, (uint64_t)b.npolys * b.map.n * c.N * 8 * 4, slot);
    const bool fused = ntt_fused(c, a, b, true, s);
    const int cp = fused ? b.npolys : ntt_chunk_polys(c, b);      // L2-sized chunks (see ntt_forward_epi)
    for (int p0 = 0; !fused && p0 < b.npolys; p0 += cp) {
        const int np = std::min(cp, b.npolys - p0);
        NttArgs ac = a;
        ac.base = a.base + (i64)p0 * a.poly_stride;
        if (src) ac.src_base = a.src_base + (i64)p0 * a.src_stride;
        const RowsCfg R = rows_cfg(B, 1 << c.s1, np, b.map.n);
        launch_rows<true>(c.s2, R.grid, B.threads, B.smem, s, ac, B.lines, R.lgc);
        launch_cols<true>(c.s1, dim3(A.blocks, b.map.n, np), A.threads, A.smem, s, ac, A.lines);
        c.st_launch += 2;
    }
    c.st_launch -= fused ? 1 : 2;
    c.prof_end(slot, s);
    c.st_ntt += (uint64_t)b.npolys * b.map.n;
    {
        int nfp = 0;
        for (int i = 0; i < b.map.n; i++) nfp += (int)((c.fpmask >> b.map.mod[i]) & 1ull);
        c.st_ntt_fp += (uint64_t)b.npolys * nfp;
    }
    c.st_launch += 2;
    c.st_bytes += (uint64_t)b.npolys * b.map.n * c.N * 8 * 4;
    CUDA_TRY(cudaGetLastError());
}

// =============================================================================================
// Value-kernel Toeplitz MAC (C8 step 4) as a negacyclic 128-point convolution along the window index.
// For one coefficient k (limb, component) the broadcast MAC computes b_{t0+t} = sum_{u < nu} src[t + dmax - u] n_u
// (t < nt, dmax = nu - 1): with A(X) = sum_{j < nsrc} src[j] X^j and B(X) = sum_{u < nu} n_u X^u this is the
// coefficient of X^{t + dmax} in A B.  Modulo X^128 + 1 a term of degree r + 128 would alias onto r; the largest degree
// is nsrc - 1 + nu - 1 < 128 + dmax whenever nsrc <= 128, so every wanted coefficient (r = t + dmax < 128) is EXACT in
// the negacyclic product, which the ring's own transform computes: the first 128 entries of the N-point merged twiddle
// tables ARE the 128-point ones (psi^{brv_16(i)} = (psi^{N/128})^{brv_7(i)} for i < 128).  Per coefficient: forward
// NTT-128 of the window (CT, bit-reversed spectrum), x B^ (the masks' spectrum times 128^{-1}, precomputed once per mask
// set: bcast_ntt_table), inverse NTT-128 (GS) -> 896 butterflies + 128 products instead of nu nt = 4096 MAC terms.
// The result is the same residue as the direct sum, canonical, so the words are identical to bcast_mac_kernel's.
// A CTA holds 32 coefficients (lines) x 128 window words; 8 threads per line (Geo<7>: E = 16 values per thread).
namespace {

constexpr int TZ_LINES = 32;
#ifndef TZ_MINB
#define TZ_MINB 4   // 4 CTAs/SM (64 registers, ~230 bytes of spills): bcast 2.27 ms vs 2.64 at 3 CTAs/SM (80 registers)
#endif

struct TzArgs {
    const u64* src[128];       // window j (nullptr / j >= nsrc: zero)
    u64* out[64];              // b_{t0 + t}
    const u64* bhat;           // [level][128][N]: spectrum index e (bit-reversed order) of the masks, x 128^{-1}
    u64* bhat_out;             // prep mode: written instead of out
    u64 fac[MAX_LIMBS];        // prep mode: 128^{-1} (FP64-path limbs) or 128^{-1} 2^64 (integer limbs: Montgomery form)
    i64 cs;                    // component stride of src / out (words)
    int nsrc, nt, dmax;
};

template <bool PREP, class Ops>
__device__ __forceinline__ void tz_body(const TzArgs& a, const Ops& ops, const typename Ops::TW* tw, const typename Ops::TW* itw,
                                        const ModConst& mc, double qinv, int limb, int comp, int k0, int N) {
    using GG = Geo<7>;
    using T = typename Ops::T;
    extern __shared__ u64 sm_raw[];
    T* sm = reinterpret_cast<T*>(sm_raw);
    const int l = threadIdx.x & (TZ_LINES - 1), j = threadIdx.x >> 5;
    T* line = sm + l * GG::LSP;
    const size_t off = (size_t)comp * a.cs + (size_t)limb * N + k0 + l;
    T x[GG::E];
    {
        u64 v[GG::E];
#pragma unroll
        for (int k = 0; k < GG::E; k++) {
            const int e = j + GG::TPL * k;
            v[k] = e < a.nsrc ? __ldcs(a.src[e] + off) : 0ull;
        }
#pragma unroll
        for (int k = 0; k < GG::E; k++) x[k] = ld_val(v[k], ops, true);
    }
    round_a<7, false, Ops>(x, 0, 0, tw, ops);
    sm_put_a<7>(line, j, x);
    __syncthreads();
    sm_get_b<7>(line, j, x);
    round_b<7, false, Ops>(x, j, 0, 0, tw, ops);
    constexpr int EB = GG::EB, G = GG::G, KB = 1 << EB;
    if constexpr (PREP) {
        const u64 f = a.fac[limb];
#pragma unroll
        for (int g = 0; g < G; g++)
#pragma unroll
            for (int k = 0; k < KB; k++) {
                const int e = ((j * G + g) << EB) + k;
                u64 w;
                if constexpr (std::is_same<T, u64>::value) w = canon8(x[g * KB + k], mc.q);
                else w = fp_canon(fp_center(x[g * KB + k], ops.q, qinv), ops.q);
                a.bhat_out[((size_t)limb * 128 + e) * N + k0 + l] = mulmod_barrett(w, f, mc.q, mc.rhi, mc.rlo);
            }
        return;
    } else {
        const u64* bh = a.bhat + ((size_t)limb * 128 + ((j * G) << EB)) * N + k0 + l;   // element e of this thread: (e - e0) N
#pragma unroll
        for (int i = 0; i < GG::E; i++) {
            const u64 bvi = __ldg(bh + (size_t)((i / KB) << EB) * N + (size_t)(i % KB) * N);
            if constexpr (std::is_same<T, u64>::value) {
                // bhat in Montgomery form: REDC(x (b 2^64)) = x b mod q in [0, q); x < 8q keeps x b 2^64 < q 2^64
                x[i] = redc128(U128{x[i] * bvi, umulhi(x[i], bvi)}, mc.q, mc.qinv);
            } else {
                const double b = fp_from_u64(bvi);
                x[i] = fp_mulmod(x[i], b, __dmul_rn(b, qinv), ops.q);   // |x| < 8q < 2^44: exact, |result| < q
            }
        }
        round_b<7, true, Ops>(x, j, 0, 0, itw, ops);   // same positions as sm_get_b: no hazard on the line
        sm_put_b<7>(line, j, x);
        __syncthreads();
        sm_get_a<7>(line, j, x);
        round_a<7, true, Ops>(x, 0, 0, itw, ops);
#pragma unroll
        for (int k = 0; k < GG::E; k++) {
            const int t = j + GG::TPL * k - a.dmax;
            if (t >= 0 && t < a.nt) {
                u64 w;
                if constexpr (std::is_same<T, u64>::value) w = canon8(x[k], mc.q);
                else w = fp_canon(fp_center(x[k], ops.q, qinv), ops.q);
                __stcs(a.out[t] + off, w);
            }
        }
    }
}

// grid: x = 2 * (N / 32) (component fastest, so the two components of a tile read the same bhat words back to back
// from L2), y = limb (modulus id = limb: the q-basis).  Prep: x = N / 32, component 0 only.
template <bool PREP>
__global__ void __launch_bounds__(256, TZ_MINB) bcast_ntt_kernel(TzArgs a, int N, const ModConst* __restrict__ mod,
                                                           const ulonglong2* tw2, const ulonglong2* itw2, const double2* twf,
                                                           const double2* itwf, const double* fpc, u64 fpmask) {
    const int limb = blockIdx.y;
    const int comp = PREP ? 0 : (blockIdx.x & 1);
    const int k0 = (PREP ? blockIdx.x : blockIdx.x >> 1) * TZ_LINES;
    const ModConst mc = mod[limb];
    if ((fpmask >> limb) & 1ull) {
        tz_body<PREP>(a, FpOps{fpc[4 * limb]}, twf + (size_t)limb * N, itwf + (size_t)limb * N, mc, fpc[4 * limb + 1], limb, comp,
                      k0, N);
    } else {
        tz_body<PREP>(a, IntOps{mc.q, 4 * mc.q}, tw2 + (size_t)limb * N, itw2 + (size_t)limb * N, mc, 0.0, limb, comp, k0, N);
    }
}

void tz_launch(encf_ctx& c, const TzArgs& a, int level, bool prep, cudaStream_t s) {
    const size_t smem = (size_t)TZ_LINES * Geo<7>::LSP * 8;
    dim3 grid((prep ? 1 : 2) * c.N / TZ_LINES, level);
    if (prep)
        bcast_ntt_kernel<true><<<grid, 256, smem, s>>>(a, c.N, c.d_mod, (const ulonglong2*)c.d_tw2, (const ulonglong2*)c.d_itw2,
                                                       (const double2*)c.d_twf, (const double2*)c.d_itwf, c.d_fpc, c.fpmask);
    else
        bcast_ntt_kernel<false><<<grid, 256, smem, s>>>(a, c.N, c.d_mod, (const ulonglong2*)c.d_tw2, (const ulonglong2*)c.d_itw2,
                                                        (const double2*)c.d_twf, (const double2*)c.d_itwf, c.d_fpc, c.fpmask);
    CUDA_TRY(cudaGetLastError());
}

}  // namespace

// The masks' spectra B^[limb][e][k] = NTT_128(n_0 .. n_{nu-1}, 0 ..)[e] 128^{-1} (Montgomery form on the integer limbs),
// cached per (mask set, level) in the context (first use outside CUDA-graph capture, like the masks themselves).
const u64* bcast_ntt_table(encf_ctx& c, const u64* const* masks, int nu, int level, cudaStream_t s) {
    std::vector<const u64*> key(masks, masks + nu);
    key.push_back(reinterpret_cast<const u64*>((uintptr_t)level));
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.bhat.find(key);
        if (it != c.bhat.end()) return it->second;
    }
    if (c.N % TZ_LINES || nu < 1 || nu > 64) throw EncfError(ENCF_ERR_PLAN_SHAPE, "bcast_ntt: unsupported shape");
    u64* tab = nullptr;
    CUDA_TRY(cudaMalloc(&tab, (size_t)level * 128 * c.N * 8));
    TzArgs a{};
    for (int u = 0; u < nu; u++) a.src[u] = masks[u];
    a.nsrc = nu;
    a.cs = 0;
    a.bhat_out = tab;
    for (int i = 0; i < level; i++) {
        const u64 q = c.mods[i], inv = h_invmod(128, q);
        a.fac[i] = ((c.fpmask >> i) & 1ull) ? inv : h_mulmod(inv, c.mont_R[i], q);
    }
    tz_launch(c, a, level, true, s);
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.bhat.find(key);
    if (it != c.bhat.end()) { cudaFree(tab); return it->second; }
    c.bhat[key] = tab;
    return tab;
}

void k_bcast_ntt(encf_ctx& c, const BcastArgs& A, const u64* bhat, int level, cudaStream_t s) {
    if (A.nsrc > 128 || A.nt > 64 || A.dmax != A.nu - 1) throw EncfError(ENCF_ERR_PLAN_SHAPE, "bcast_ntt: window longer than 128");
    TzArgs a{};
    for (int j = 0; j < A.nsrc; j++) a.src[j] = A.src[j];
    for (int t = 0; t < A.nt; t++) a.out[t] = A.out[t];
    a.bhat = bhat;
    a.cs = (i64)level * c.N;
    a.nsrc = A.nsrc; a.nt = A.nt; a.dmax = A.dmax;
    // algorithmic bytes: the window and the outputs (both components) + the spectrum table once
    const uint64_t bytes = ((uint64_t)A.nsrc * 2 + (uint64_t)A.nt * 2 + 128) * level * c.N * 8;
    int slot;
    c.prof_begin("bcast_mac", s, bytes, slot);
    tz_launch(c, a, level, false, s);
    c.prof_end(slot, s);
    c.st_launch++; c.st_bytes += bytes; c.st_ptmul += (uint64_t)A.nt * A.nu;
}
