// Pipe-throughput microbench on sm_100a: DFMA (fp64 pipe) vs IMAD.WIDE.U32 / IMAD (fmaheavy) per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* outd, uint64_t* outi, int iters, double a, double b, uint32_t ia, uint32_t ib) {
    double d[8]; uint64_t w[8]; uint32_t u[8];
    for (int i = 0; i < 8; i++) { d[i] = threadIdx.x + i; w[i] = threadIdx.x * 7 + i; u[i] = threadIdx.x * 3 + i; }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (OP == 0) d[i] = fma(d[i], a, b);
            if (OP == 1) w[i] = (uint64_t)(uint32_t)w[i] * ia + w[i];           // IMAD.WIDE.U32
            if (OP == 2) u[i] = u[i] * ia + ib;                                  // IMAD
            if (OP == 3) u[i] = __umulhi(u[i], ia) + u[i];                        // IMAD.HI
            if (OP == 4) d[i] = d[i] * a + d[i];                                 // DFMA-ish
            if (OP == 5) d[i] = d[i] + a;                                        // DADD
        }
    }
    double sd = 0; uint64_t sw = 0;
    for (int i = 0; i < 8; i++) { sd += d[i]; sw += w[i] + u[i]; }
    outd[blockIdx.x * blockDim.x + threadIdx.x] = sd; outi[blockIdx.x * blockDim.x + threadIdx.x] = sw;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* od; uint64_t* oi; int blocks = sms * 8, th = 256, iters = 4096;
    cudaMalloc(&od, blocks * th * 8); cudaMalloc(&oi, blocks * th * 8);
    const char* names[] = {"DFMA", "IMAD.WIDE.U32", "IMAD", "IMAD.HI", "DFMA2", "DADD"};
    for (int op = 0; op < 6; op++) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int r = 0; r < 2; r++) {
            cudaEventRecord(a);
            switch (op) {
                case 0: k<0><<<blocks, th>>>(od, oi, iters, 1.0000001, 0.5, 3, 5); break;
                case 1: k<1><<<blocks, th>>>(od, oi, iters, 1.0000001, 0.5, 3, 5); break;
                case 2: k<2><<<blocks, th>>>(od, oi, iters, 1.0000001, 0.5, 3, 5); break;
                case 3: k<3><<<blocks, th>>>(od, oi, iters, 1.0000001, 0.5, 3, 5); break;
                case 4: k<4><<<blocks, th>>>(od, oi, iters, 1.0000001, 0.5, 3, 5); break;
                case 5: k<5><<<blocks, th>>>(od, oi, iters, 1.0000001, 0.5, 3, 5); break;
            }
            cudaEventRecord(b); cudaEventSynchronize(b);
        }
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = (double)blocks * th * iters * 8;
        printf("%-14s %8.3f ms  %.1f Gop/s  %.1f lanes/clk/SM (clk %d MHz)\n", names[op], ms, ops / ms / 1e6,
               ops / (ms * 1e-3) / (sms * (double)clk * 1e3), clk / 1000);
    }
    return 0;
}
