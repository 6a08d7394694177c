// Library-wide state of the C-ABI (include/iedd_b200.h): error text and the
// launch counter reported as bench.py's gpu_launches.
#include <stdlib.h>
#include <mutex>
#include <algorithm>
#include <string>

#include "common.cuh"

struct ie_matvec;

namespace ie {
std::atomic<int64_t> g_launches{0};
bool pdl_enabled() {
    static const bool on = !getenv("IEDD_B200_NO_PDL");
    return on;
}
int pdl_early_mask() {
    // default 5: k_iter_a (-0.7 us per config-5 iteration) and the scatter (-0.5 us); k_apply_dmma2's
    // early trigger costs +5 us (the scatter's CTAs park beside the last tiles)
    static const int m = getenv("IEDD_B200_EARLY") ? atoi(getenv("IEDD_B200_EARLY")) : 5;
    return pdl_enabled() ? m : 0;
}
float l2_persist_request(size_t bytes) {
    static std::mutex mu;
    static size_t limit = 0, cap = 0;
    static bool off = getenv("IEDD_B200_NO_L2PERSIST") != nullptr;
    if (off || !bytes) return 0.f;
    std::lock_guard<std::mutex> lk(mu);
    if (!cap) {
        int dev = 0, mx = 0, l2 = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess || mx <= 0) {
            cudaGetLastError();
            off = true;
            return 0.f;
        }
        cap = std::min<size_t>((size_t)mx, (size_t)l2 / 4);
    }
    size_t want = std::min(cap, (bytes + bytes / 7 + ((size_t)1 << 20)) & ~(((size_t)1 << 20) - 1));
    if (const char* e = getenv("IEDD_B200_L2_SETASIDE_MB")) want = (size_t)atoi(e) << 20;  // experiment
    if (want > limit) {
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
            cudaGetLastError();
            off = true;
            return 0.f;
        }
        limit = want;
    }
    return bytes <= limit ? 1.0f : (float)((double)limit / (double)bytes);
}
static thread_local std::string t_err;
void set_error(const std::string& msg) { t_err = msg; }
}  // namespace ie

extern "C" const char* ie_last_error(void) { return ie::t_err.c_str(); }
extern "C" int64_t ie_launch_count(void) { return ie::g_launches.load(); }

// ----------------------------------------------------------------------
// FP64 issue-peak microbenchmark (roofline denominator for K1; not in
// MEASURED_PEAKS.json): 8 independent DFMA chains per thread, all SMs.
namespace ie {
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1234.5678) out[0] = s;  // keep the chains live
}
}  // namespace ie

extern "C" int ie_fp64_peak(double* dfma_per_s, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    double* d;
    IE_CUDA(cudaMalloc(&d, 8));
    cudaEvent_t e0, e1;
    IE_CUDA(cudaEventCreate(&e0));
    IE_CUDA(cudaEventCreate(&e1));
    const int blocks = ie::kNumSMs * 8, threads = 256, iters = 4096;
    for (int rep = 0; rep < 2; ++rep) ie::k_dfma_peak<<<blocks, threads, 0, st>>>(d, iters, 0.999999, 1e-7);
    IE_CUDA(cudaEventRecord(e0, st));
    ie::k_dfma_peak<<<blocks, threads, 0, st>>>(d, iters, 0.999999, 1e-7);
    IE_CUDA(cudaEventRecord(e1, st));
    IE_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    IE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *dfma_per_s = (double)blocks * threads * iters * 8 / (ms * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return IE_OK;
}

// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput microbenchmark: the
// roofline denominator of the class-GEMM apply (k_apply_dmma).  8 independent
// accumulator chains per warp, 8 warps per CTA, 2 CTAs per SM.
namespace ie {
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters, double a, double b) {
    double c[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = threadIdx.x * 1e-3 + q;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[q][0]), "+d"(c[q][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
    if (s == 1234.5678) out[0] = s;
}
}  // namespace ie

extern "C" int ie_dmma_peak(double* flops_per_s, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    double* d;
    IE_CUDA(cudaMalloc(&d, 8));
    cudaEvent_t e0, e1;
    IE_CUDA(cudaEventCreate(&e0));
    IE_CUDA(cudaEventCreate(&e1));
    const int blocks = ie::kNumSMs * 2, threads = 256, iters = 4096;
    for (int rep = 0; rep < 2; ++rep) ie::k_dmma_peak<<<blocks, threads, 0, st>>>(d, iters, 1.0, 1e-9);
    IE_CUDA(cudaEventRecord(e0, st));
    ie::k_dmma_peak<<<blocks, threads, 0, st>>>(d, iters, 1.0, 1e-9);
    IE_CUDA(cudaEventRecord(e1, st));
    IE_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    IE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    // per mma: 8 x 8 x 4 multiply-adds = 512 flops per warp
    *flops_per_s = (double)blocks * (threads / 32) * iters * 8 * 512.0 / (ms * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return IE_OK;
}
