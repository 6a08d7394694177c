// DMMA (mma.sync m8n8k4 f64) throughput microbenchmark: independent accumulator chains per warp.
#include <cuda_runtime.h>
#include <stdio.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, int iters, double a, double b) {
    double c[CH][2];
    for (int q = 0; q < CH; ++q) c[q][0] = c[q][1] = threadIdx.x * 1e-3 + q;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int q = 0; q < CH; ++q) dmma(c[q][0], c[q][1], a, b);
    double s = 0;
    for (int q = 0; q < CH; ++q) s += c[q][0] + c[q][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
void run(int warps_per_cta, int ctas_per_sm) {
    double* d; cudaMalloc(&d, 148 * 64 * 1024 * 8);
    const int ctas = 148 * ctas_per_sm, tpb = 32 * warps_per_cta, iters = 4096;
    k<CH><<<ctas, tpb>>>(d, 16, 1.0, 1e-9);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<CH><<<ctas, tpb>>>(d, iters, 1.0, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 8 * 4 * (double)CH * iters * (tpb / 32) * ctas;
    printf("CH=%d warps/SM=%d: %.1f TFLOP/s (%s)\n", CH, warps_per_cta * ctas_per_sm, flops / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}
int main() {
    run<4>(8, 2); run<8>(8, 2); run<16>(8, 2); run<8>(8, 4); run<16>(8, 4); run<4>(4, 1); run<8>(4, 1); run<16>(4, 1); run<8>(8, 1); run<16>(8, 1); run<8>(16, 1);
    return 0;
}
