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
    // the latest true residual and its iteration (the host's batch-size policy reads them from the polled state)
    double last_rel;
    long long last_k;
};

// Fixed-order CTA reductions (a shared-memory halving tree over blockDim
// leaves): deterministic, identical on every rank and in every driver.
// (A warp-shuffle butterfly + ordered warp sums was measured: no change in
// the iteration time, 144.5 vs 145.6 us, so the round-1 association stays.)
// Levels with a partner >= 32 threads away go through shared memory; the last
// five run inside warp 0 by shuffles (lane t takes lane t + o: the same pairs in
// the same order, so the same bits), then one broadcast.
__device__ __forceinline__ double block_tree(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = blockDim.x / 2; o >= 32; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x < 32) {
        double a = sh[threadIdx.x];
        for (int o = min(16, (int)blockDim.x / 2); o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
        if (threadIdx.x == 0) sh[0] = a;
    }
    __syncthreads();
    return sh[0];
}
// two trees at once (each value keeps block_tree's pairs): sh holds 2 blockDim doubles
__device__ __forceinline__ void block_tree2(double& va, double& vb, double* sh) {
    double* sb = sh + blockDim.x;
    sh[threadIdx.x] = va;
    sb[threadIdx.x] = vb;
    __syncthreads();
    for (int o = blockDim.x / 2; o >= 32; o >>= 1) {
        if (threadIdx.x < o) {
            sh[threadIdx.x] += sh[threadIdx.x + o];
            sb[threadIdx.x] += sb[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x < 32) {
        double a = sh[threadIdx.x], b = sb[threadIdx.x];
        for (int o = min(16, (int)blockDim.x / 2); o > 0; o >>= 1) {
            a += __shfl_down_sync(0xffffffffu, a, o);
            b += __shfl_down_sync(0xffffffffu, b, o);
        }
        if (threadIdx.x == 0) {
            sh[0] = a;
            sb[0] = b;
        }
    }
    __syncthreads();
    va = sh[0];
    vb = sb[0];
}

__device__ __forceinline__ double reduce_partials(const double* part, int nch, double* sh) {
    double loc = 0.0;
    for (int c = threadIdx.x; c < nch; c += blockDim.x) loc += part[c];
    return block_tree(loc, sh);
}

// Kernels of the PCG iteration folded into the A-pass's line transforms (FFT
// method, 2D / 3D, lines of >= 64 points; csrc/fft.cu LineArgs):
//   first pass (2-RHS): k_iter_b's vector half -- p = z + beta p stored back
//     with beta and the multipliers from the state (pcg_decide), max|p| into
//     the rotating slots pglob[it % 3]; `it` < 0: graph replay;
//   last pass: k_post_pass -- per output line l in [post_lo, post_hi) the
//     partials p.q (q_col >= 0) and |f - w|^2 (w_col >= 0: the output
//     column holding w) at part[2 (line0 + l)], [.. + 1]; p and f are indexed
//     like the output vector.
struct PcgFuse {
    const double* z = nullptr;
    double* pglob = nullptr;
    struct PcgState* s = nullptr;
    long long it = 0;
    const double* p = nullptr;
    const double* f = nullptr;
    double* part = nullptr;
    int line0 = 0, post_lo = 0, post_hi = 0, q_col = -1, w_col = -1;
    // the w = A u column is consumed by the folded post pass alone: its store is skipped
    int skip_w_store = 0;
    // sharded: the partials also written into the peers' arrays + mailbox
    int npeer = 0;
    double* part_peer[16] = {};
    unsigned long long* part_ctr[16] = {};
};

// The sharded driver's transposes folded into the band FFT passes (see
// LineArgs peer_*): mode 1 = row spectra -> column-slab owners, mode 2 =
// column slab -> every rank's need rows.
struct PeerStores {
    int mode = 0, npeer = 0, band_rows = 0;
    double2* peer[16] = {};
    unsigned long long* ctr[16] = {};
    long long line_bytes[16] = {};
    int rlo[16] = {}, rhi[16] = {};
};

// The sharded RZ exchange folded into the apply's scatter: each CTA copies its
// chunk's record (all kRzRec fields) into every rank's array at the same index
// and release-adds the bytes to that rank's mailbox.
struct PeerRec {
    int n = 0;
    double* dst[16] = {};
    unsigned long long* ctr[16] = {};
};

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
    for (int o = blockDim.x / 2; o >= 32; o >>= 1) {
        if (threadIdx.x < o) {
            sh[threadIdx.x] += sh[threadIdx.x + o];
            sh[blockDim.x + threadIdx.x] = fmax(sh[blockDim.x + threadIdx.x], sh[blockDim.x + threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x < 32) {  // the last five levels inside warp 0 (the sum keeps its pairs; a maximum has no order)
        double a = sh[threadIdx.x], b = sh[blockDim.x + threadIdx.x];
        for (int o = min(16, (int)blockDim.x / 2); o > 0; o >>= 1) {
            a += __shfl_down_sync(0xffffffffu, a, o);
            b = fmax(b, __shfl_down_sync(0xffffffffu, b, o));
        }
        if (threadIdx.x == 0) {
            out[0] = a;
            out[1] = b;
        }
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

// k_iter_b's scalar half, run once per iteration by the last CTA of the
// apply's scatter (single-GPU driver with the p update folded into the next
// FFT pass): beta = r.z / rho_prev from the chunk record `rec` (nch chunks),
// rho, and the next 2-RHS multipliers from max|z|, max|u| (record) and
// max|p_old| (pglob[it % 3]; zeroes pglob[(it + 1) % 3] for the next pass's
// atomic max).  it < 0: graph replay -- the iteration comes from the state
// and is advanced here (the iteration's last it_dev reader).  The reduction
// is k_iter_b's (256 threads striding the chunks, block_tree), so the
// values are bitwise those of the sharded driver's k_iter_b.
struct PcgDecide {
    struct PcgState* s = nullptr;
    double* pglob = nullptr;
    long long it = 0;
    int nch = 0;
    int early = 0;  // the scatter triggers its dependents at entry (pdl_trigger)
};

__device__ __forceinline__ double chunk_absmax(double v, double* sh);
__device__ inline void pcg_decide(const double* rec, const PcgDecide& d, double* sh) {
    PcgState* s = d.s;
    const long long itb = d.it < 0 ? s->it_dev : d.it;
    // thread 0's scalars are requested before the reductions (one round trip less in the tail)
    const double rho_prev = threadIdx.x == 0 ? s->rho[(itb - 1) & 1] : 0.0;
    const double mp = threadIdx.x == 0 ? d.pglob[itb % 3] : 0.0;
    double loc = 0.0, mz = 0.0, mu = 0.0;
    for (int c = threadIdx.x; c < d.nch; c += kPcgRed) {
        loc += rec[kRzRec * c];
        mz = fmax(mz, rec[kRzRec * c + 1]);
        mu = fmax(mu, rec[kRzRec * c + 3]);
    }
    const double rz = block_tree(loc, sh);
    __syncthreads();
    mz = chunk_absmax(mz, sh);
    __syncthreads();
    mu = chunk_absmax(mu, sh);
    if (threadIdx.x == 0) {
        const double beta = rz / rho_prev;
        s->beta = beta;
        s->rho[itb & 1] = rz;
        s->sc[0] = pcg_pow2_scale(__dadd_rn(mz, __dmul_rn(fabs(beta), mp)));
        s->sc[1] = pcg_pow2_scale(mu);
        d.pglob[(itb + 1) % 3] = 0.0;
        if (d.it < 0) s->it_dev = itb + 1;
    }
}

__device__ __forceinline__ double chunk_absmax(double v, double* sh) {
    // a maximum has no rounding: warp shuffles, then the warp maxima through shared memory
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();  // (sh may still be read by a previous reduction's last stage)
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double m = sh[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
    return m;
}

}  // namespace ie
