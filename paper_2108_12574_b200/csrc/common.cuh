// Shared device helpers for the Schwarz-PCG hot path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>

#include "../../include/iedd_b200.h"

namespace ie {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);
extern std::atomic<int64_t> g_launches;

#define IE_CUDA(call)                                                        \
    do {                                                                     \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess) {                                             \
            ::ie::set_error(std::string(#call) + ": " + cudaGetErrorString(_e)); \
            return IE_ERR_CUDA;                                              \
        }                                                                    \
    } while (0)

#define IE_LAUNCHED()                                                         \
    do {                                                                      \
        ::ie::g_launches.fetch_add(1, std::memory_order_relaxed);             \
        cudaError_t _e = cudaGetLastError();                                  \
        if (_e != cudaSuccess) {                                              \
            ::ie::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
            return IE_ERR_CUDA;                                               \
        }                                                                     \
    } while (0)

constexpr int kNumSMs = 148;

// ------------------------------------------- programmatic dependent launch --
// The kernels of the PCG iteration are launched with programmatic stream
// serialization (launch_k): a kernel may be scheduled while its predecessor
// drains and runs pdl_wait() (griddepcontrol.wait: the predecessor has
// completed and its writes are visible) before touching anything.  Early
// launch_dependents triggers in every kernel slowed the PCG iteration (196 vs
// 186 us: successor CTAs parked on the SMs beside later waves of the primary),
// while the implicit end-of-kernel trigger hides the launch latency (config-5
// FFT pass 101.5 -> 96 us, apply 48 -> 44 us when launched back to back; ~1 us
// per graph-replayed iteration).  Round 2: early triggers only in kernels whose
// whole grid is resident in one wave -- k_iter_a (-0.7 us per config-5
// iteration) and the apply's scatter (-0.5 us); in k_apply_dmma2 it costs +5 us
// (pdl_early_mask).  A no-op for ordinary launches; IEDD_B200_NO_PDL=1 turns
// the attribute off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// Early trigger, only in kernels whose whole grid is resident in one wave (the
// successor's CTAs can then only take the slots this grid's CTAs free as they
// exit; they run their setup-time prologue and block in pdl_wait()).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
bool pdl_enabled();
int pdl_early_mask();  // IEDD_B200_EARLY: bit 0 k_iter_a, bit 1 k_apply_dmma2, bit 2 k_scatter_fixed

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// L2 set-aside for data every PCG iteration re-reads unchanged (the scatter's
// position table): l2_persist_request(bytes) raises the device's persisting-L2
// limit to cover the largest request (+15%, capped at a quarter of L2) and
// returns the hit ratio to use for a window of that size (0: disabled by
// IEDD_B200_NO_L2PERSIST or unsupported).  Config 5: the 16.8 MB table with a 20
// MB set-aside took 4.0 us off the iteration; a 48 MB set-aside only 0.7 --
// the iteration's ~135 MB working set needs the rest of the 126 MB L2.
float l2_persist_request(size_t bytes);
// launch_k with an L2 access-policy window (persisting hits) over [win, win + bytes)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k_win(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                const void* win, size_t bytes, float hit_ratio, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (win && bytes && hit_ratio > 0.f) {
        at[na].id = cudaLaunchAttributeAccessPolicyWindow;
        at[na].val.accessPolicyWindow.base_ptr = const_cast<void*>(win);
        at[na].val.accessPolicyWindow.num_bytes = bytes;
        at[na].val.accessPolicyWindow.hitRatio = hit_ratio;
        at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------ log table --
// log(d^2) for d^2 = m * s^2 with integer m >= 1 (dims 1 and 2):
//   m = 2^e * f, f in [1,2); k = top 7 mantissa bits of f;
//   c_k = 1/(1 + (k + 1/2)/128);  u = f*c_k - 1, |u| <= 2^-8;
//   log(d^2) = T[e*128+k] + log1p(u),  T = e*ln2 - log(c_k) + 2*log(s)
// T is rounded once from 80-bit arithmetic on the host.  log1p(u) is the
// degree-6 Taylor polynomial (truncation <= 2^-56/7 absolute).
constexpr int kLogK = 128;

struct LogEntry {  // 16 B -> one LDS.128 per pair
    double c;
    double t;
};

// log1p(u) = u * q(u); returns q (degree-5 Horner), the caller folds u*q + t.
__device__ __forceinline__ double log1p_q(double u) {
    double q = -1.0 / 6.0;
    q = fma(q, u, 1.0 / 5.0);
    q = fma(q, u, -1.0 / 4.0);
    q = fma(q, u, 1.0 / 3.0);
    q = fma(q, u, -1.0 / 2.0);
    return fma(q, u, 1.0);
}

// Split the normalised double m (>= 1) into the table index (relative to
// the e=0 entry) and the reduced mantissa f in [1,2).
__device__ __forceinline__ void log_split(double m, int& idx, double& f) {
    const int hi = __double2hiint(m);
    const int lo = __double2loint(m);
    idx = (hi >> 13) - (1023 << 7);
    f = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, lo);
}

// log(m * s^2) with the table in shared or global memory.
__device__ __forceinline__ double log_d2(const LogEntry* __restrict__ tab, double m) {
    int idx;
    double f;
    log_split(m, idx, f);
    const LogEntry e = tab[idx];
    const double u = fma(f, e.c, -1.0);
    return fma(log1p_q(u), u, e.t);
}

// Exact integer -> double for 0 <= m < 2^31 via the 2^52 magic constant
// (one DADD instead of a conversion instruction).
__device__ __forceinline__ double int_to_double_exact(int m) {
    return __hiloint2double(0x43300000, m) - 4503599627370496.0;
}

// ------------------------------------------------------------ geometry --
// Multi-index of global point i in C order (last axis fastest).
template <int DIM>
__device__ __forceinline__ void unravel(int64_t i, int n, int* a) {
#pragma unroll
    for (int d = DIM - 1; d >= 0; --d) {
        a[d] = (int)(i % n);
        i /= n;
    }
}

// Entry A_ij from integer multi-index differences (shared by K1 epilogue
// tests, block extraction K2 and ie_assemble_block_f64).
struct EntryParams {
    int dim;
    double alpha;   // dims 1/2: -weight/(4 pi);  dim 3: weight/(4 pi s)
    double diag;
};

__device__ __forceinline__ double entry_from_m(const EntryParams& P, const LogEntry* tab, int m) {
    if (m == 0) return P.diag;
    const double md = int_to_double_exact(m);
    if (P.dim == 3) return P.alpha * rsqrt(md);
    return P.alpha * log_d2(tab, md);
}

}  // namespace ie
