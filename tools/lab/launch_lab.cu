// Lab (not part of the library): launch-to-completion cost of a 148-CTA kernel
// as a function of its dynamic shared memory, alone and alternating with a
// small-smem kernel (shared-memory carveout changes between launches).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_lab launch_lab.cu
#include <cuda_runtime.h>
#include <stdio.h>
__global__ void kbig(double* o) {
    extern __shared__ double sm[];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) o[blockIdx.x] = sm[5];
}
__global__ void ksmall(double* o) { o[blockIdx.x * blockDim.x + threadIdx.x] += 1.0; }
int main() {
    double* o;
    cudaMalloc(&o, 1 << 24);
    cudaFuncSetAttribute(kbig, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaStream_t s;
    cudaStreamCreate(&s);
    int sizes[] = {4096, 48 * 1024, 100 * 1024, 150 * 1024, 227 * 1024};
    for (int carve = 0; carve < 2; ++carve) {
        if (carve) {
            cudaFuncSetAttribute(ksmall, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            cudaFuncSetAttribute(kbig, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        }
        for (int alt = 0; alt < 2; ++alt)
            for (int si = 0; si < 5; ++si) {
                const int sm = sizes[si];
                // capture 100 launches in a graph
                cudaGraph_t g;
                cudaGraphExec_t ge;
                cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
                for (int i = 0; i < 100; ++i) {
                    kbig<<<148, 256, sm, s>>>(o);
                    if (alt) ksmall<<<512, 256, 0, s>>>(o);
                }
                cudaStreamEndCapture(s, &g);
                if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
                cudaGraphLaunch(ge, s);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0, s);
                cudaGraphLaunch(ge, s);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("carveout_pref %d alternate %d smem %6d: %.2f us per iteration (%s)\n", carve, alt, sm, ms * 10,
                       cudaGetErrorString(cudaGetLastError()));
            }
    }
    return 0;
}
