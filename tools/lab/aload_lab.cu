// Lab (not part of the library): how fast can 148 CTAs (1 per SM, 227 KB smem)
// pull a 144x144 FP64 matrix from L2 into shared memory?  Same matrix for all
// CTAs vs one copy per CTA; TMA bulk rows vs cp.async 16 B vs plain loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o aload_lab aload_lab.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
constexpr int S = 144, AP = 148;
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(256, 1) k(const double* A, int per_cta, int mode, unsigned long long* t, double* sink) {
    extern __shared__ double sm[];
    __shared__ __align__(8) uint64_t bar;
    const double* src0 = A + (per_cta ? (size_t)blockIdx.x * S * S : 0);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (mode == 0) {  // TMA bulk rows
        if (threadIdx.x < 32) {
            if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(S * S * 8));
            __syncwarp();
            for (int i = threadIdx.x; i < S; i += 32)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + i * AP)),
                             "l"(src0 + i * S), "r"(S * 8), "r"(su(&bar)) : "memory");
        }
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"(su(&bar)) : "memory");
    } else if (mode == 1) {  // cp.async 16
        for (int e = threadIdx.x; e < S * S / 2; e += 256) {
            const int i = (2 * e) / S, j = 2 * e - i * S;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(sm + i * AP + j)), "l"(src0 + 2 * e));
        }
        asm volatile("cp.async.commit_group; cp.async.wait_group 0;" ::: "memory");
    } else {  // plain 16 B loads, 8 in flight per thread
        for (int e0 = threadIdx.x; e0 < S * S / 2; e0 += 8 * 256) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * 256;
                if (e < S * S / 2) v[u] = reinterpret_cast<const double2*>(src0)[e];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * 256;
                if (e < S * S / 2) {
                    const int i = (2 * e) / S, j = 2 * e - i * S;
                    sm[i * AP + j] = v[u].x;
                    sm[i * AP + j + 1] = v[u].y;
                }
            }
        }
    }
    __syncthreads();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) {
        t[2 * blockIdx.x] = t0;
        t[2 * blockIdx.x + 1] = t1;
        sink[blockIdx.x] = sm[(blockIdx.x * 97) % (S * AP)];
    }
}
int main() {
    double *A, *sink;
    unsigned long long* t;
    cudaMalloc(&A, 148ull * S * S * 8);
    cudaMemset(A, 0, 148ull * S * S * 8);
    cudaMalloc(&sink, 148 * 8);
    cudaMalloc(&t, 2 * 148 * 8);
    const size_t smem = (size_t)S * AP * 8 + 56832;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned long long h[296];
    char* flush;
    cudaMalloc(&flush, 256 << 20);
    for (int mode = 0; mode < 3; ++mode)
        for (int per = 0; per < 2; ++per)
            for (int rep = 0; rep < 3; ++rep) {
                if (rep == 2) cudaMemset(flush, rep, 256 << 20);  // third rep: L2 flushed
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                k<<<148, 256, smem>>>(A, per, mode, t, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
                double mx = 0, mn = 1e30, mean = 0;
                for (int b = 0; b < 148; ++b) {
                    const double d = (h[2 * b + 1] - h[2 * b]) * 1e-3;
                    mx = d > mx ? d : mx; mn = d < mn ? d : mn; mean += d / 148;
                }
                printf("mode %d per_cta %d: kernel %.2f us, per-CTA load min %.2f mean %.2f max %.2f us (%s)\n", mode, per,
                       ms * 1e3, mn, mean, mx, cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
