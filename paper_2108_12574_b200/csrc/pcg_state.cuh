// Device-side PCG state and the fixed-order chunk reductions of the PCG
// kernels (krylov.cu).  Control flow of pcg.py:54-136.
#pragma once

#include "common.cuh"

namespace ie {

constexpr int kPcgChunk = 2048;  // dot-product chunk (fixed: results independent of the launch)
constexpr int kPcgRed = 256;     // threads per chunk CTA

// Device-resident PCG state.  Every iteration kernel returns immediately
// once `stop` is set, so the host can enqueue iterations ahead and read the
// status once per batch (pcg.py's control flow runs in k_iter_a).
struct PcgState {
    double rho[2];  // rho_j = r_j . z_j in slot j & 1 (read and written by different launches)
    double alpha, beta, denom, nf, tol, fail_value;
    // multipliers 2^-e of [p, u] in the next 2-RHS FFT pass (k_iter_b): p from
    // the bound max|z| + |beta| max|p_old| >= max|p_new|, u from max|u| --
    // global maxima known right after the r.z exchange, so a sharded solver
    // needs no extra all-gather of max|p_new| before its row transforms
    double sc[2];
    long long max_iters, n_it, fail_iter;
    long long it_dev;  // iteration index for graph-replayed iterations (it < 0 in the kernel args)
    int status;  // 0 running, 1 converged, 2 stagnated, 3 max_iters, 4 breakdown, 5 non-finite
    int stop;
    unsigned int ticket;  // CTAs of a graph-replayed k_iter_b done (the last one advances it_dev)
};

__device__ __forceinline__ double block_tree(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    return sh[0];
}

__device__ __forceinline__ double reduce_partials(const double* part, int nch, double* sh) {
    double loc = 0.0;
    for (int c = threadIdx.x; c < nch; c += blockDim.x) loc += part[c];
    return block_tree(loc, sh);
}

// PCG chunk record of the apply (4 doubles per dot-product chunk, the r.z
// exchange of the sharded solver): [0] r.z partial, [1] max|z|, [2] max|p|
// of the current search direction, [3] max|u| of the current iterate.
constexpr int kRzRec = 4;

// sum (fixed tree) and max of a CTA's per-thread values -> out[0], out[1];
// sh holds 2 * blockDim.x doubles
__device__ __forceinline__ void chunk_sum_max(double v, double m, double* sh, double* out) {
    sh[threadIdx.x] = v;
    sh[blockDim.x + threadIdx.x] = m;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sh[threadIdx.x] += sh[threadIdx.x + o];
            sh[blockDim.x + threadIdx.x] = fmax(sh[blockDim.x + threadIdx.x], sh[blockDim.x + threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = sh[0];
        out[1] = sh[blockDim.x];
    }
    __syncthreads();
}

// 2^-e with 2^e > max|x| >= 2^(e-1) (frexp; power of two, exact); 1 for 0 / non-finite
__device__ __forceinline__ double pcg_pow2_scale(double mx) {
    if (!(mx > 0.0) || !isfinite(mx)) return 1.0;
    int e;
    frexp(mx, &e);
    return ldexp(1.0, -e);
}

__device__ __forceinline__ double chunk_absmax(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    return sh[0];
}

}  // namespace ie
