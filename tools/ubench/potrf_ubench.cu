// Microbenchmark (dev tool): cost of the interface-Cholesky diagonal step potrf_inv_tile alone
// and with a DMMA-saturating CTA co-resident on every SM.
#include "../../paper_2406_15959_b200/csrc/chol.cu"
#include <cstdio>

__global__ void __launch_bounds__(256, 2) k_potrf_bench(double* out, int reps, int* flag) {
    extern __shared__ __align__(128) double sm[];
    double* A = sm;
    double* Y = sm + ELM_TS;
    double* x = Y + ELM_TS;
    for (int r = 0; r < reps; ++r) {
        for (int t = threadIdx.x; t < 64 * 64; t += 256) {
            int i = t & 63, j = t >> 6;
            A[j * ELM_TLD + i] = (i == j ? 64.0 : 0.0) + 1.0 / (1.0 + i + j);
        }
        __syncthreads();
        potrf_inv_tile(A, Y, x);
    }
    if (threadIdx.x == 0) out[blockIdx.x] = Y[5 * ELM_TLD + 7];
    if (threadIdx.x == 0 && flag) atomicExch(flag, 1);
}
__global__ void __launch_bounds__(256, 2) k_hog(double* out, int* flag) {
    double a0 = 0, a1 = 0, b = threadIdx.x * 1e-3, c = 1.0;
    for (long it = 0; it < 2000000; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) dmma_c(a0, a1, b, c);
        if ((it & 1023) == 0 && *(volatile int*)flag) break;
    }
    if (a0 == 12345.0) out[0] = a1;
}
int main() {
    double* out; int* flag;
    cudaMalloc(&out, 4096 * 8); cudaMalloc(&flag, 4);
    int smem = (2 * ELM_TS + 10 * 64) * 8;
    cudaFuncSetAttribute(k_potrf_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int reps = 50;
    k_potrf_bench<<<148, 256, smem>>>(out, 2, nullptr);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k_potrf_bench<<<148, 256, smem>>>(out, reps, nullptr);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("potrf_inv_tile alone: %.2f us per tile\n", 1000.0 * ms / reps);
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaMemset(flag, 0, 4);
    k_hog<<<148, 256, 0, s1>>>(out, flag);
    cudaEventRecord(e0, s2);
    k_potrf_bench<<<148, 256, smem, s2>>>(out, reps, flag);
    cudaEventRecord(e1, s2); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("potrf_inv_tile with a DMMA hog per SM: %.2f us per tile\n", 1000.0 * ms / reps);
    cudaDeviceSynchronize();
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
