// Dependent-chain latencies on the GPU (cycles per op), one warp.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, float* outf, long long* cyc, const double* src, int iters) {
    __shared__ double sh[64];
    __shared__ float shf[64];
    if (threadIdx.x < 64) { sh[threadIdx.x] = src[threadIdx.x]; shf[threadIdx.x] = (float)src[threadIdx.x]; }
    __syncwarp();
    double a = src[threadIdx.x], b = src[threadIdx.x + 1];
    float fa = (float)a, fb = (float)b;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { a = a + b; a = a + b; a = a + b; a = a + b; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0);
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { a = fma(a, b, b); a = fma(a, b, b); a = fma(a, b, b); a = fma(a, b, b); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0);
    // FFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { fa = fmaf(fa, fb, fb); fa = fmaf(fa, fb, fb); fa = fmaf(fa, fb, fb); fa = fmaf(fa, fb, fb); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0);
    // LDS (dependent address) chain
    int idx = threadIdx.x & 31;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        idx = ((int)sh[idx] & 31); idx = ((int)sh[idx] & 31); idx = ((int)sh[idx] & 31); idx = ((int)sh[idx] & 31);
    }
    t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0);
    // SHFL chain (float)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        fa = __shfl_xor_sync(0xffffffffu, fa, 1); fa = __shfl_xor_sync(0xffffffffu, fa, 2);
        fa = __shfl_xor_sync(0xffffffffu, fa, 4); fa = __shfl_xor_sync(0xffffffffu, fa, 8);
    }
    t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0);
    // DMMA chain (accumulator dependency)
    double d0 = a, d1 = b;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    }
    t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0);
    // REDUX chain
    unsigned u = (unsigned)idx;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { u = __reduce_max_sync(0xffffffffu, u) + 1; u = __reduce_max_sync(0xffffffffu, u) + 1; u = __reduce_max_sync(0xffffffffu, u) + 1; u = __reduce_max_sync(0xffffffffu, u) + 1; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0);
    // DMNMX chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { a = fmax(a, b); a = fmax(a, -b); a = fmax(a, b); a = fmax(a, -b); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0);
    // FMNMX chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { fa = fmaxf(fa, fb); fa = fmaxf(fa, -fb); fa = fmaxf(fa, fb); fa = fmaxf(fa, -fb); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[8] = (t1 - t0);
    // LDS.64 (double, dependent through value)
    double dv = a;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        dv = sh[((int)dv) & 31] + 1.0; dv = sh[((int)dv) & 31] + 1.0; dv = sh[((int)dv) & 31] + 1.0; dv = sh[((int)dv) & 31] + 1.0;
    }
    t1 = clock64(); if (threadIdx.x == 0) cyc[9] = (t1 - t0);
    out[threadIdx.x] = a + d0 + d1 + dv + (double)u;
    outf[threadIdx.x] = fa + (float)idx;
}

int main() {
    double *src, *out; float* outf; long long* cyc;
    cudaMallocManaged(&src, 128 * sizeof(double)); cudaMallocManaged(&out, 128 * sizeof(double));
    cudaMallocManaged(&outf, 128 * sizeof(float)); cudaMallocManaged(&cyc, 16 * sizeof(long long));
    for (int i = 0; i < 128; ++i) src[i] = 1.0 + 1e-9 * i;
    const int iters = 1000;
    k<<<1, 32>>>(out, outf, cyc, src, iters);
    cudaDeviceSynchronize();
    k<<<1, 32>>>(out, outf, cyc, src, iters);
    cudaDeviceSynchronize();
    const char* names[] = {"DADD", "DFMA", "FFMA", "LDS(int addr)", "SHFL", "DMMA 884", "REDUX+IADD", "DMNMX", "FMNMX", "LDS.64+DADD+F2I"};
    for (int i = 0; i < 10; ++i) printf("%-18s %.1f cycles/op\n", names[i], (double)cyc[i] / (4.0 * iters));
    return 0;
}
