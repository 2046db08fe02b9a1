// Access-pattern microbench on sm_100a: how fast can the diag_mac plaintext stream be READ, with no math?
//   pattern 0 (diag_mac): CTA = 32-coefficient tile of one limb, 16 unit lanes x 16 threads x 16 B, each lane
//             walks units x bank entries (row stride = level x N words) -> 256 B segments of many rows;
//   pattern 1 (tile-major): the same bytes laid out so that each CTA's stream is one contiguous region.
// Prints GB/s of each (CUDA events, best of 5).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int N = 65536, LEVEL = 8, UNITS = 72, NBANK = 64, T = 32;

__global__ void __launch_bounds__(256) pat_diag(const uint64_t* __restrict__ w, uint64_t* out, int limbs) {
    const int kp = threadIdx.x % 16, lane = threadIdx.x / 16;
    const int limb = blockIdx.y, k0 = blockIdx.x * T;
    const size_t pstride = (size_t)LEVEL * N, wus = (size_t)NBANK * pstride;
    const size_t wl = (size_t)limb * N + k0 + 2 * kp;
    uint64_t s = 0;
    for (int u = lane; u < UNITS; u += 16) {
        const uint64_t* wu = w + u * wus + wl;
        for (int q = 0; q < NBANK; q += 8) {
            ulonglong2 x[8];
#pragma unroll
            for (int t = 0; t < 8; t++) x[t] = __ldg((const ulonglong2*)(wu + (size_t)(q + t) * pstride));
#pragma unroll
            for (int t = 0; t < 8; t++) s ^= x[t].x + x[t].y;
        }
    }
    if (s == 0x12345) out[0] = s;
}

__global__ void __launch_bounds__(256) pat_tile(const uint64_t* __restrict__ w, uint64_t* out, int limbs) {
    // CTA (tile, limb) reads UNITS x NBANK x T words contiguously
    const size_t per = (size_t)UNITS * NBANK * T;
    const ulonglong2* base = (const ulonglong2*)(w + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * per);
    uint64_t s = 0;
    const int n2 = (int)(per / 2);
    for (int i0 = threadIdx.x; i0 < n2; i0 += 256 * 8) {
        ulonglong2 x[8];
#pragma unroll
        for (int t = 0; t < 8; t++) x[t] = i0 + t * 256 < n2 ? __ldg(base + i0 + t * 256) : make_ulonglong2(0, 0);
#pragma unroll
        for (int t = 0; t < 8; t++) s ^= x[t].x + x[t].y;
    }
    if (s == 0x12345) out[0] = s;
}

int main() {
    const size_t words = (size_t)UNITS * NBANK * LEVEL * N;   // 2.4 G words = 19.3 GB
    uint64_t *w, *o;
    if (cudaMalloc(&w, words * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&o, 64);
    cudaMemset(w, 1, words * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int limbs = 7;   // the narrow limbs of the QKV launch
    const double bytes = (double)UNITS * NBANK * limbs * N * 8;
    for (int p = 0; p < 2; p++) {
        float best = 1e30f;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(a);
            if (p == 0) pat_diag<<<dim3(N / T, limbs), 256>>>(w, o, limbs);
            else pat_tile<<<dim3(N / T, limbs), 256>>>(w, o, limbs);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%s: %.3f ms, %.1f GB/s\n", p == 0 ? "diag_mac pattern" : "tile-major contiguous", best, bytes / best / 1e6);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
