// Microbenchmark (dev tool): dependent-chain latency of FP64 ops on this GPU (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, long long* cyc, double x0) {
    double x = x0 + threadIdx.x * 1e-9, y = 1.0000001, z = 1e-9;
    long long t0, t1;
#define CHAIN(name, expr, n) t0 = clock64(); for (int i = 0; i < n; ++i) { expr; } t1 = clock64(); if (threadIdx.x == 0) { cyc[name] = (t1 - t0) / n; }
    CHAIN(0, x = fma(x, y, z), 4096);
    CHAIN(1, x = x * y, 4096);
    CHAIN(2, x = x + z, 4096);
    CHAIN(3, x = rsqrt(x + 1.0), 1024);
    float f = (float)x;
    t0 = clock64(); for (int i = 0; i < 4096; ++i) f = fmaf(f, 1.0000001f, 1e-9f); t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = (t1 - t0) / 4096;
    double a0 = x, a1 = x;
    t0 = clock64();
    for (int i = 0; i < 1024; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(a0), "+d"(a1) : "d"(y), "d"(z));
    t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = (t1 - t0) / 1024;
    __shared__ double sh[64];
    sh[threadIdx.x] = x;
    __syncwarp();
    int idx = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) { double v = sh[idx]; idx = ((int)v & 31) ^ threadIdx.x; sh[idx] = v; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[6] = (t1 - t0) / 1024;
    out[threadIdx.x] = x + a0 + a1 + f + idx;
}
int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64 * 8);
    k_lat<<<1, 32>>>(out, cyc, 1.0);
    cudaDeviceSynchronize();
    k_lat<<<1, 32>>>(out, cyc, 1.0);
    cudaDeviceSynchronize();
    const char* n[] = {"DFMA", "DMUL", "DADD", "rsqrt(double) incl DADD", "FFMA (fp32)", "DMMA m8n8k4", "LDS+STS chain"};
    for (int i = 0; i < 7; ++i) printf("%-26s %lld cycles\n", n[i], cyc[i]);
    return 0;
}
