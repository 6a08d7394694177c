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
