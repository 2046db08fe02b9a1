// dsmem_bw.cu -- distributed shared memory (DSMEM) bandwidth on the B200, for the single-pass cluster NTT
// decision: a 2^16 limb split over a cluster of C CTAs must move (C-1)/C of its words between
// CTAs once.  Each CTA of a cluster repeatedly stores (or loads) a 64 KB block into (from) the shared memory of
// the next CTA of its cluster with 128-bit accesses; the kernel reports the aggregate bytes/s over the GPU,
// next to a local-smem and an HBM copy of the same volume.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bw dsmem_bw.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int kWords = 8192;   // 64 KB of u64 per CTA

template <bool REMOTE, bool LOAD>
__global__ void dsmem_kernel(int iters, unsigned long long* sink) {
    extern __shared__ ulonglong2 buf[];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank(), n = cl.num_blocks();
    for (int i = threadIdx.x; i < kWords / 2; i += blockDim.x) buf[i] = make_ulonglong2(i, rank);
    cl.sync();
    ulonglong2* peer = REMOTE ? cl.map_shared_rank(buf, (rank + 1) % n) : buf;
    unsigned long long acc = 0;
    for (int it = 0; it < iters; it++) {
        if (LOAD) {
#pragma unroll 4
            for (int i = threadIdx.x; i < kWords / 2; i += blockDim.x) {
                const ulonglong2 v = peer[i];
                acc += v.x ^ v.y;
            }
        } else {
#pragma unroll 4
            for (int i = threadIdx.x; i < kWords / 2; i += blockDim.x) peer[i] = make_ulonglong2(i + it, acc);
        }
        cl.sync();
    }
    if (acc == 0x12345) *sink = acc;
}

__global__ void hbm_copy(const ulonglong2* __restrict__ a, ulonglong2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <bool REMOTE, bool LOAD>
double run(int csize, int iters) {
    cudaLaunchConfig_t cfg = {};
    const int ctas = 148 / csize * csize;
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = kWords * 8;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    auto k = dsmem_kernel<REMOTE, LOAD>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 8);
    if (csize > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    cudaLaunchKernelEx(&cfg, k, iters, sink);   // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 0; }
    cudaFree(sink);
    return (double)ctas * iters * kWords * 8 / (ms * 1e-3) / 1e9;
}

int main() {
    const int iters = 2000;
    for (int cs : {2, 4, 8}) {
        printf("cluster %d: remote store %.0f GB/s, remote load %.0f GB/s, local store %.0f GB/s, local load %.0f GB/s\n", cs,
               run<true, false>(cs, iters), run<true, true>(cs, iters), run<false, false>(cs, iters), run<false, true>(cs, iters));
    }
    size_t n = (size_t)1 << 27;   // 2 GiB per buffer
    ulonglong2 *a, *b;
    cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    hbm_copy<<<148 * 8, 256>>>(a, b, n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    hbm_copy<<<148 * 8, 256>>>(a, b, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("hbm copy (read+write) %.0f GB/s\n", 2.0 * n * 16 / (ms * 1e-3) / 1e9);
    return 0;
}
