// bconv_tc.cu -- the tensor-core base-conversion experiment: fast BConv
//   out[t][k] = sum_{i < NIN} v[i][k] W[i][t]  mod q_t        (v < 2^60, W < q_t, NIN = 8 inputs, NOUT targets)
// on tcgen05.mma .kind::i8 (u8 x u8 -> s32, exact), against the CUDA-core kernel of libencf (30-bit split, 4 IMAD.WIDE
// per product, one Montgomery REDC per output).
//
// Byte decomposition: v_i = sum_a v_i[a] 2^{8a}.  With W'[i][a][t] = 2^{8a} W[i][t] R mod q_t (R = 2^64, Montgomery)
// split into bytes W'[i][a][t][b]:
//   D[k][(t,b)] = sum_{(i,a)} v_i[a](k) W'[i][a][t][b]       (K = NIN*8 = 64 u8 x u8 products, D < 64*255^2 < 2^22)
//   T[t][k] = sum_b D[k][(t,b)] 2^{8b} = sum_i v_i W[i][t] R  (mod q_t),  T < 2^78 < q_t 2^64
//   out[t][k] = REDC(T) = T R^{-1} mod q_t.
// One CTA (128 threads) per 128-coefficient tile: A = the tile's v bytes [128 x 64] (K-major, no swizzle), B = W' bytes
// [NOUT*8 x 64] (constant, K-major), two M128 x N(8 NOUT) x K32 MMAs into TMEM, epilogue tcgen05.ld 32x32b.x8 per
// target (one thread per coefficient row), REDC, coalesced store.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bconv_tc bconv_tc.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>
#include "../../paper_2604_09975_b200/csrc/common.cuh"

constexpr int NIN = 8;
constexpr int TILE = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, SWIZZLE_NONE K-major: core matrix = 8 rows x 16 B contiguous; SBO = byte distance
// between 8-row groups, LBO = byte distance between the two 16-byte K chunks of one K32 step.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;          // version (Blackwell)
    return d;                        // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
// instruction descriptor: D s32, A u8, B u8, both K-major, N, M = 128
__host__ __device__ constexpr uint32_t idesc_i8(int N, int M) {
    return (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int NOUT>
__global__ void __launch_bounds__(128) bconv_tc_kernel(const u64* __restrict__ v, const uint8_t* __restrict__ wbytes,
                                                       const u64* __restrict__ qs, const u64* __restrict__ qinvs,
                                                       u64* __restrict__ out, int N, int npolys) {
    constexpr int NB = NOUT * 8;                              // MMA N
    constexpr int TCOLS = NB <= 32 ? 32 : NB <= 64 ? 64 : NB <= 128 ? 128 : 256;
    __shared__ __align__(1024) uint8_t sA[TILE * NIN * 8];    // [kc 0..3][128 rows][16 B]
    __shared__ __align__(1024) uint8_t sB[NB * NIN * 8];      // [kc 0..3][NB rows][16 B]
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < NB * NIN * 8 / 16; i += 128) ((uint4*)sB)[i] = ((const uint4*)wbytes)[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem_base;
    u64 q[NOUT], qi[NOUT];
#pragma unroll
    for (int t = 0; t < NOUT; t++) { q[t] = qs[t]; qi[t] = qinvs[t]; }
    const int tiles_per_poly = N / TILE;
    const int ntiles = tiles_per_poly * npolys;
    uint32_t phase = 0;
    u64 nx[NIN];       // the next tile's inputs, loaded while the current tile's MMA and epilogue run
    auto load_tile = [&](int tile) {
        if (tile >= ntiles) return;
        const int p = tile / tiles_per_poly, k0 = (tile % tiles_per_poly) * TILE;
        const u64* vp = v + (size_t)p * NIN * N;
#pragma unroll
        for (int i = 0; i < NIN; i++) nx[i] = __ldg(vp + (size_t)i * N + k0 + tid);
    };
    load_tile(blockIdx.x);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int p = tile / tiles_per_poly, k0 = (tile % tiles_per_poly) * TILE;
        // stage A: row m = coefficient k0 + m, bytes (i, a) = v_i little-endian
#pragma unroll
        for (int i = 0; i < NIN; i++) *(u64*)(sA + (i >> 1) * (TILE * 16) + tid * 16 + (i & 1) * 8) = nx[i];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy writes -> tensor core
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (tid == 0) {
            constexpr uint32_t idesc = idesc_i8(NB, TILE);
#pragma unroll
            for (int s = 0; s < 2; s++) {   // K = 64 bytes = 2 steps of K32 (two 16-byte chunks each)
                const uint64_t da = sdesc(smem_u32(sA) + s * 2 * TILE * 16, TILE * 16, 128);
                const uint64_t db = sdesc(smem_u32(sB) + s * 2 * NB * 16, NB * 16, 128);
                const uint32_t acc = s > 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                    ::"r"(tbase), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar))
                         : "memory");
        }
        load_tile(tile + gridDim.x);
        // wait for the MMAs (they also finished reading sA)
        asm volatile(
            "{\n.reg .pred P1;\nWAIT:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
            "@!P1 bra WAIT;\n}" ::"r"(smem_u32(&mbar)), "r"(phase) : "memory");
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        u64* op = out + (size_t)p * NOUT * N + k0 + tid;
#pragma unroll
        for (int t = 0; t < NOUT; t++) {
            uint32_t d[8];
            const uint32_t ta = tbase + ((uint32_t)(warp * 32) << 16) + t * 8;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
                         : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            // T = sum_b d_b 2^{8b}: two 47-bit halves, then 128-bit
            const u64 lo4 = (u64)d[0] + ((u64)d[1] << 8) + ((u64)d[2] << 16) + ((u64)d[3] << 24);
            const u64 hi4 = (u64)d[4] + ((u64)d[5] << 8) + ((u64)d[6] << 16) + ((u64)d[7] << 24);
            U128 T{lo4, 0};
            add128(T, hi4 << 32);
            T.hi += hi4 >> 32;
            op[(size_t)t * N] = redc128(T, q[t], qi[t]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();                 // TMEM and sA may be overwritten by the next tile
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(TCOLS));
}

// CUDA-core reference kernel: the arithmetic of libencf's bconv_batch_kernel (30-bit split, 4 IMAD.WIDE per product).
template <int NOUT>
__global__ void __launch_bounds__(256, 4) bconv_cc_kernel(const u64* __restrict__ v, const u64* __restrict__ wmont,
                                                          const u64* __restrict__ qs, const u64* __restrict__ qinvs,
                                                          u64* __restrict__ out, int N, int npolys) {
    __shared__ u64 sw[NIN * NOUT];
    for (int i = threadIdx.x; i < NIN * NOUT; i += blockDim.x) sw[i] = wmont[i];
    __syncthreads();
    const size_t total = (size_t)N * npolys;
    for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < total; g += (size_t)gridDim.x * blockDim.x) {
        const int p = (int)(g / N), k = (int)(g % N);
        const u64* vp = v + (size_t)p * NIN * N;
        uint32_t vh[NIN], vl[NIN];
#pragma unroll
        for (int i = 0; i < NIN; i++) {
            const u64 x = __ldg(vp + (size_t)i * N + k);
            vh[i] = (uint32_t)(x >> 30); vl[i] = (uint32_t)(x & 0x3FFFFFFFu);
        }
        u64* op = out + (size_t)p * NOUT * N + k;
#pragma unroll 2
        for (int t = 0; t < NOUT; t++) {
            u64 hh = 0, hl = 0, lh = 0, ll = 0;
#pragma unroll
            for (int i = 0; i < NIN; i++) {
                const u64 w = sw[i * NOUT + t];
                const uint32_t wh = (uint32_t)(w >> 30), wlo = (uint32_t)(w & 0x3FFFFFFFu);
                hh += (u64)vh[i] * wh; hl += (u64)vh[i] * wlo; lh += (u64)vl[i] * wh; ll += (u64)vl[i] * wlo;
            }
            U128 acc{ll, 0};
            const u64 mid = hl + lh;
            add128(acc, mid << 30);
            acc.hi += mid >> 34;
            add128(acc, hh << 60);
            acc.hi += hh >> 4;
            op[(size_t)t * N] = redc128(acc, qs[t], qinvs[t]);
        }
    }
}

template <int NOUT>
int run(int npolys, bool narrow_out) {
    const int N = 65536;
    std::mt19937_64 rng(0xB0C0 + NOUT);
    // moduli: inputs 60-bit (largest case), outputs 40-bit or 60-bit primes-like odd numbers (REDC needs odd q only)
    std::vector<u64> qin(NIN), qout(NOUT), qinv(NOUT);
    for (int i = 0; i < NIN; i++) qin[i] = ((1ull << 60) - 1) - 2 * (rng() % 1000000);
    for (int t = 0; t < NOUT; t++) {
        qout[t] = narrow_out ? (((1ull << 40) - 1) - 2 * (rng() % 1000000)) : (((1ull << 60) - 1) - 2 * (rng() % 1000000));
        qinv[t] = h_neg_inv64(qout[t]);
    }
    std::vector<u64> W(NIN * NOUT), Wm(NIN * NOUT);
    for (int i = 0; i < NIN; i++)
        for (int t = 0; t < NOUT; t++) {
            W[i * NOUT + t] = rng() % qout[t];
            Wm[i * NOUT + t] = h_mulmod(W[i * NOUT + t], h_mont_R(qout[t]), qout[t]);
        }
    // W' bytes in the canonical K-major no-swizzle layout: row n = t*8 + b, K byte kk = i*8 + a ->
    // [kk / 16][n][kk % 16]
    constexpr int NB = NOUT * 8;
    std::vector<uint8_t> wb(NB * NIN * 8);
    for (int i = 0; i < NIN; i++)
        for (int a = 0; a < 8; a++)
            for (int t = 0; t < NOUT; t++) {
                const u64 wp = h_mulmod(h_mulmod(W[i * NOUT + t], h_powmod(2, 8 * a, qout[t]), qout[t]), h_mont_R(qout[t]), qout[t]);
                for (int b = 0; b < 8; b++) {
                    const int n = t * 8 + b, kk = i * 8 + a;
                    wb[(kk / 16) * (NB * 16) + n * 16 + (kk % 16)] = (uint8_t)(wp >> (8 * b));
                }
            }
    const size_t nv = (size_t)npolys * NIN * N, no = (size_t)npolys * NOUT * N;
    std::vector<u64> hv(nv);
    for (size_t x = 0; x < nv; x++) hv[x] = rng() % qin[(x / N) % NIN];
    u64 *dv, *dout, *dout2, *dq, *dqi, *dwm;
    uint8_t* dwb;
    cudaMalloc(&dv, nv * 8); cudaMalloc(&dout, no * 8); cudaMalloc(&dout2, no * 8);
    cudaMalloc(&dq, NOUT * 8); cudaMalloc(&dqi, NOUT * 8); cudaMalloc(&dwm, NIN * NOUT * 8); cudaMalloc(&dwb, wb.size());
    cudaMemcpy(dv, hv.data(), nv * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, qout.data(), NOUT * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dqi, qinv.data(), NOUT * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dwm, Wm.data(), NIN * NOUT * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dwb, wb.data(), wb.size(), cudaMemcpyHostToDevice);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bconv_tc_kernel<NOUT>, 128, 0);
    const char* ge = getenv("TC_CTAS_PER_SM");
    if (ge) occ = atoi(ge);
    const int grid_tc = 148 * occ;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms_tc = 0, ms_cc = 0;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        bconv_tc_kernel<NOUT><<<grid_tc, 128>>>(dv, dwb, dq, dqi, dout, N, npolys);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_tc, e0, e1);
        cudaEventRecord(e0);
        bconv_cc_kernel<NOUT><<<148 * 4 * 2, 256>>>(dv, dwm, dq, dqi, dout2, N, npolys);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_cc, e0, e1);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("CUDA error: %s\n", cudaGetErrorString(err)); return 1; }
    std::vector<u64> o1(no), o2(no);
    cudaMemcpy(o1.data(), dout, no * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(o2.data(), dout2, no * 8, cudaMemcpyDeviceToHost);
    size_t bad_tc = 0, bad_cc = 0, checked = 0;
    for (int p = 0; p < npolys; p++)
        for (int k = 0; k < N; k += (p == 0 ? 1 : 97)) {
            for (int t = 0; t < NOUT; t++) {
                unsigned __int128 s = 0;
                for (int i = 0; i < NIN; i++) s += (unsigned __int128)hv[((size_t)p * NIN + i) * N + k] * W[i * NOUT + t];
                const u64 ref = (u64)(s % qout[t]);
                const size_t o = ((size_t)p * NOUT + t) * N + k;
                bad_tc += o1[o] != ref;
                bad_cc += o2[o] != ref;
                checked++;
            }
        }
    const double bytes = (double)(nv + no) * 8;
    printf("NOUT=%d %s-bit targets, %d polys: tcgen05 %.3f ms (%.0f GB/s, occ %d) | CUDA-core %.3f ms (%.0f GB/s) | "
           "mismatches tc %zu cc %zu of %zu checked\n", NOUT, narrow_out ? "40" : "60", npolys, ms_tc, bytes / ms_tc / 1e6, occ,
           ms_cc, bytes / ms_cc / 1e6, bad_tc, bad_cc, checked);
    cudaFree(dv); cudaFree(dout); cudaFree(dout2); cudaFree(dq); cudaFree(dqi); cudaFree(dwm); cudaFree(dwb);
    return bad_tc != 0;
}

int main() {
    int bad = 0;
    bad |= run<6>(64, false);    // ModUp at L = 8: 8 digit limbs -> K = 6 special primes
    bad |= run<8>(64, true);     // ModDown-like: 8 -> 8 body limbs
    bad |= run<16>(32, true);    // 8 -> 16 (a digit of the L = 24 ModUp)
    return bad;
}
