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

// k_iter_b's update of one chunk: p = z + beta p, max|p| of the chunk into amax[2c]
__device__ __forceinline__ void iter_b_chunk(int c, double beta, double* p, const double* z, int N, double* amax,
                                             double* sh) {
    const int base = c * kPcgChunk;
    double m = 0.0;
#pragma unroll
    for (int e = 0; e < kPcgChunk / kPcgRed; ++e) {
        const int i = base + e * kPcgRed + threadIdx.x;
        if (i < N) {
            const double pn = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
            p[i] = pn;
            m = fmax(m, fabs(pn));
        }
    }
    __syncthreads();
    m = chunk_absmax(m, sh);
    if (threadIdx.x == 0) amax[2 * c] = m;
}

// k_iter_b's control: beta = rho_it / rho_{it-1} from the r.z chunk partials
__device__ __forceinline__ double iter_b_beta(const double* part_rz, int nch, long long it, PcgState* s, double* sh) {
    const double rz = reduce_partials(part_rz, nch, sh);
    const double beta = rz / s->rho[(it - 1) & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s->beta = beta;
        s->rho[it & 1] = rz;
    }
    return beta;
}

}  // namespace ie
