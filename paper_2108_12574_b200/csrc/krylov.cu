// K4 (fused PCG) and K5 (Lanczos) -- replaces pcg.solve
// (/root/reference/pkg/src/iedd/pcg.py:54-136) and
// spectrum.extremal_eigenvalue_lanczos (spectrum.py:133-190).
//
// PCG runs on the device with the reference's control flow.  The true
// residual ||f - A u_k|| (pcg.py:107-108) is not a second matvec: the A-pass
// at the top of iteration k+1 multiplies [p_{k+1}, u_k] (2 RHS, one kernel
// evaluation per pair) and the convergence / stagnation test of iteration k
// runs before the breakdown test of iteration k+1 -- the reference's order.
// z_k = T^{-1} r_k is therefore computed speculatively and discarded when
// iteration k turns out to be the last.  n_it, history and u follow the
// reference's recurrences; only kernel rounding differs.
//
// Dot products: fixed 2048-element chunk partials (in-CTA fixed tree), then a
// fixed-order reduction -- deterministic and independent of the launch.
// Control lives in device state (PcgState / LzState); the steady-state PCG
// iteration and, after 16 steps, the Lanczos step are each one captured CUDA
// graph, the host reading the state every few iterations.  The sharded driver
// (ie_pcg_sharded_f64, end of file) runs the same kernels on row bands with
// NCCL collectives between them.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "pcg_state.cuh"

struct ie_matvec;
struct ie_precond;

namespace ie {

int matvec_launch(const ie_matvec* m, const double* X, int64_t ldx, int nrhs, double* Y, int64_t ldy,
                  int64_t row_begin, int64_t row_end, cudaStream_t st, const int* stop,
                  const double* scales = nullptr, const PcgFuse* fz = nullptr);
int matvec_fused_lines(const ie_matvec* m);
int precond_prepare_stream(const ie_precond* p, cudaStream_t st);
int matvec_prepare_stream(const ie_matvec* m, cudaStream_t st);
int precond_apply(const ie_precond* p, const double* r, double* z, double* partials, cudaStream_t st,
                  const int* stop);
void precond_set_decide(const PcgDecide* d);
void precond_set_staging(double* buf, size_t bytes);
double* matvec_scratch(const ie_matvec* m, cudaStream_t st, size_t* bytes);
void precond_set_peer_record(const PeerRec* r);
int matvec_N(const ie_matvec* m);
uint64_t matvec_uid(const ie_matvec* m);
uint64_t precond_uid(const ie_precond* p);

constexpr int kChunk = kPcgChunk;
constexpr int kRed = kPcgRed;
int dot_chunks(int64_t n) { return (int)((n + kChunk - 1) / kChunk); }

// mode 0: partial of x.y;  mode 1: partial of |x - y|^2
__global__ void __launch_bounds__(kRed) k_dot_partials(const double* x, const double* y, int N, int mode,
                                                       double* part) {
    __shared__ double sh[kRed];
    const int base = blockIdx.x * kChunk;
    double loc = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < N) {
            if (mode == 0) {
                loc = fma(x[i], y[i], loc);
            } else {
                const double d = x[i] - y[i];
                loc = fma(d, d, loc);
            }
        }
    }
    const double t = block_tree(loc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}


// The solve's opening in one pass over f: the graph-stable copy of f, r = f,
// u = 0 and the chunk partials of f.f (k_dot_partials' chain and tree per chunk).
__global__ void __launch_bounds__(kRed) k_pcg_begin(const double* f, double* fcopy, double* r, double* u, int N,
                                                    double* part) {
    __shared__ double sh[kRed];
    const int base = blockIdx.x * kChunk;
    double loc = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < N) {
            const double v = f[i];
            fcopy[i] = v;
            r[i] = v;
            u[i] = 0.0;
            loc = fma(v, v, loc);
        }
    }
    const double t = block_tree(loc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void k_set_it(PcgState* s, long long it) { s->it_dev = it; }

__global__ void k_pcg_init(const double* part, int nch, PcgState* s, double tol, long long max_iters,
                           double* hist) {
    // (rho_0 is set by k_pcg_setup after the first apply)
    __shared__ double sh[kRed];
    if (s->status == 6) return;  // a sharded exchange timed out before the init (k_wait): keep the failure
    const double v = reduce_partials(part, nch, sh);
    if (threadIdx.x == 0) {
        s->nf = sqrt(v);
        s->tol = tol;
        s->max_iters = max_iters;
        s->n_it = 0;
        s->fail_iter = 0;
        s->fail_value = 0.0;
        s->status = 0;
        s->stop = 0;
        s->ticket = 0;
        s->last_rel = 1.0;
        s->last_k = 0;
        hist[0] = 1.0;
        if (s->nf == 0.0) {  // pcg.py:74-78
            hist[0] = 0.0;
            s->status = 1;
            s->stop = 1;
        }
    }
}

// Fused control + update kernels (one CTA per 2048-element chunk).  Every
// CTA reduces the same fixed-chunk partials in the same order, so all CTAs
// take the same decision; CTA 0 records it in the state.
//
// Layouts (global chunk order, shared by the single-GPU and sharded drivers):
//   xpost[2c], xpost[2c + 1]: p.q and |f - A u|^2 partials of chunk c
//                             (k_post_pass; the A-pass exchange);
//   xrz[kRzRec c + 0..3]:      r.z, max|z| (scatter), max|p|, max|u|
//                             (k_iter_a / k_update_u; the apply exchange);
//   pmax[b]:                  max|p_new| of the band's chunk b (k_iter_b),
//                             copied into xrz by the next k_iter_a.
// A kernel's own chunks are [c0, c0 + gridDim) of the global order; its
// vectors are band pointers (index 0 = the first point of chunk c0).

// Halo segments of a sharded band (rows the rank's subdomains read outside
// its band): r -= alpha q is applied there redundantly by extra CTAs of
// k_iter_a (the owner computes the same values), so the apply needs no
// r exchange.  Offsets relative to the band start; zero-length on one GPU.
struct HaloSeg {
    int lo0, len0, lo1, len1;
};

// Graph replay: the last CTA of the iteration's final it_dev reader (every CTA
// has read it) advances the iteration counter.
__device__ __forceinline__ void advance_iteration(PcgState* s) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&s->ticket, 1u) == gridDim.x - 1) {
            s->ticket = 0;
            s->it_dev += 1;
        }
    }
}

// After the A-pass of iteration `it`: residual / stagnation check of
// iteration it-1 (pcg.py:107-119), breakdown test of iteration it
// (pcg.py:99-103), alpha, then u += alpha p, r -= alpha q and max|u| per chunk.
// Every CTA reduces the same partials in the same order and takes the same
// decision; CTA 0 records it in the state.  Every load that does not depend
// on the reduction (state scalars, the history entry of the stagnation test,
// this thread's partials and its p, q, r chunk values) is issued before it, so
// the serial prologue costs about one memory round trip.  CTAs >= nchb update
// the halo segments' r only.  xpost holds npost partial pairs (dot chunks, or
// output lines when the post pass is folded into the FFT); pmax (the
// per-chunk max|p| of k_iter_b, copied into the record) is null when the p
// update is folded into the FFT; ticket: graph replay without k_iter_b, this
// kernel advances the iteration counter.
template <bool WITH_U, bool HALO = false>
__global__ void __launch_bounds__(kRed, 4) k_iter_a(const double* xpost, int npost, int do_p, int pending,
                                                 long long it, PcgState* s, double* hist, double* u, double* r,
                                                 const double* p, const double* q, int nb, int c0, int nchb,
                                                 double* xrz, const double* pmax, HaloSeg hs, int ticket) {
    __shared__ double sh[2 * kRed];
    __shared__ int decided;
    if (ticket & 2) pdl_trigger();  // (ticket bit 1: early trigger; bit 0: advance the iteration counter)
    pdl_wait();
    const int stopv = s->stop;
    if (it < 0) it = s->it_dev;
    const double rho_prev = s->rho[(it - 1) & 1], nf = s->nf, tol = s->tol;
    const long long k = it - 1;
    const double h30 = (pending && k >= 30 && threadIdx.x == 0) ? hist[k - 30] : 0.0;
    const bool halo = HALO && (int)blockIdx.x >= nchb;
    int base, lim;
    if (!halo) {
        base = blockIdx.x * kChunk;
        lim = nb;
    } else {  // halo CTA: segment 0 then segment 1, kChunk points each
        const int h = blockIdx.x - nchb, n0 = (hs.len0 + kChunk - 1) / kChunk;
        base = h < n0 ? hs.lo0 + h * kChunk : hs.lo1 + (h - n0) * kChunk;
        lim = h < n0 ? hs.lo0 + hs.len0 : hs.lo1 + hs.len1;
    }
    // av: p for the in-kernel u update (WITH_U band CTAs), else r (hoisted
    // where registers allow: the 64-register budget holds two chunk arrays)
    const bool ua = WITH_U && !halo;
    double av[kChunk / kRed], qv[kChunk / kRed];
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        const bool in = do_p && i < lim;
        av[e] = in ? (ua ? p[i] : r[i]) : 0.0;
        qv[e] = in ? q[i] : 0.0;
    }
    double lp = 0.0, lr = 0.0;
    for (int c = threadIdx.x; c < npost; c += kRed) {
        if (do_p) lp += xpost[2 * c];
        if (pending) lr += xpost[2 * c + 1];
    }
    if (stopv) return;
    double denom = 0.0, res2 = 0.0;
    if (do_p && pending) {  // both sums in one pass over the tree levels (same pairs)
        denom = lp;
        res2 = lr;
        block_tree2(denom, res2, sh);
    } else {
        if (do_p) denom = block_tree(lp, sh);
        __syncthreads();
        if (pending) res2 = block_tree(lr, sh);
    }
    if (threadIdx.x == 0) {
        int status = 0;
        double rel = 0.0;
        if (pending) {
            rel = sqrt(res2) / nf;
            if (!isfinite(rel)) status = 5;
            else if (rel <= tol) status = 1;
            else if (k >= 30 && rel > (1.0 - 1e-3) * h30) status = 2;
            else if (!do_p) status = 3;
        }
        if (!status && do_p && (!isfinite(denom) || denom <= 0.0)) status = 4;
        decided = status;
        if (blockIdx.x == 0) {
            if (pending && status != 5) {
                hist[k] = rel;
                s->last_rel = rel;
                s->last_k = k;
            }
            if (status) {
                s->status = status;
                s->n_it = k;
                if (status == 5) {
                    s->fail_iter = k;
                    s->fail_value = rel;
                } else if (status == 4) {
                    s->fail_iter = it;
                    s->fail_value = denom;
                }
                s->stop = 1;
            } else if (do_p) {
                s->denom = denom;
                s->alpha = rho_prev / denom;
            }
        }
    }
    __syncthreads();
    if (decided || !do_p) return;
    // max|p| of the direction this pass multiplied (k_iter_b of the previous
    // iteration) into the record, for this iteration's k_iter_b scale bound
    if (pmax && !halo && threadIdx.x == 32) xrz[kRzRec * (c0 + blockIdx.x) + 2] = pmax[blockIdx.x];
    const double al = rho_prev / denom;
    if (!ua) {  // u += alpha p runs concurrently in k_update_u (graph side branch), or a halo CTA
#pragma unroll
        for (int e = 0; e < kChunk / kRed; ++e) {
            const int i = base + e * kRed + threadIdx.x;
            if (i < lim) r[i] = __dsub_rn(av[e], __dmul_rn(al, qv[e]));
        }
        if (ticket & 1) advance_iteration(s);
        return;
    }
    double m = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < nb) {
            const double un = __dadd_rn(u[i], __dmul_rn(al, av[e]));
            u[i] = un;
            r[i] = __dsub_rn(r[i], __dmul_rn(al, qv[e]));
            m = fmax(m, fabs(un));
        }
    }
    m = chunk_absmax(m, sh);
    if (threadIdx.x == 0) xrz[kRzRec * (c0 + blockIdx.x) + 3] = m;
    if (ticket & 1) advance_iteration(s);
}

// k_iter_a's u half: u += alpha p and max|u| per chunk, with the alpha CTA 0 of
// k_iter_a stored (the same quotient every CTA computes).  Off the critical
// path: it runs beside the preconditioner apply and joins before k_iter_b
// rewrites p (the next A-pass is u's only consumer).
__global__ void __launch_bounds__(kRed) k_update_u(const PcgState* s, double* u, const double* p, int N, int c0,
                                                   double* xrz) {
    __shared__ double sh[kRed];
    if (s->stop) return;
    const double al = s->alpha;
    const int base = blockIdx.x * kChunk;
    double uv[kChunk / kRed], pv[kChunk / kRed];  // all loads ahead of the first store
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        uv[e] = i < N ? u[i] : 0.0;
        pv[e] = i < N ? p[i] : 0.0;
    }
    double m = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < N) {
            const double un = __dadd_rn(uv[e], __dmul_rn(al, pv[e]));
            u[i] = un;
            m = fmax(m, fabs(un));
        }
    }
    m = chunk_absmax(m, sh);
    if (threadIdx.x == 0) xrz[kRzRec * (c0 + blockIdx.x) + 3] = m;
}

// After the apply: rho_it = r.z, beta = rho_it / rho_{it-1}, p = z + beta p,
// max|p| per chunk; the independent loads (state, partials, this thread's z
// and p chunk values) are issued ahead of the reduction.  CTA 0 also fixes the
// 2-RHS scales of the next A-pass from the record's global maxima:
// p_new = z + beta p_old, so max|p_new| <= max|z| + |beta| max|p_old| (both
// products rounded as written: the same bound on every rank).  In graph
// replay the last CTA advances the iteration counter.
__global__ void __launch_bounds__(kRed) k_iter_b(const double* xrz, int nch, long long it, PcgState* s, double* p,
                                                 const double* z, int nb, double* pmax) {
    __shared__ double sh[kRed];
    __shared__ double shm[3][kRed];
    pdl_wait();
    const int stopv = s->stop;
    const bool replay = it < 0;
    if (replay) it = s->it_dev;
    const double rho_prev = s->rho[(it - 1) & 1];
    const int base = blockIdx.x * kChunk;
    double zv[kChunk / kRed], pv[kChunk / kRed];
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        zv[e] = i < nb ? z[i] : 0.0;
        pv[e] = i < nb ? p[i] : 0.0;
    }
    double loc = 0.0, mz = 0.0, mp = 0.0, mu = 0.0;
    const bool cta0 = blockIdx.x == 0;
    for (int c = threadIdx.x; c < nch; c += kRed) {
        loc += xrz[kRzRec * c];
        if (cta0) {
            mz = fmax(mz, xrz[kRzRec * c + 1]);
            mp = fmax(mp, xrz[kRzRec * c + 2]);
            mu = fmax(mu, xrz[kRzRec * c + 3]);
        }
    }
    if (stopv) return;
    const double rz = block_tree(loc, sh);
    const double beta = rz / rho_prev;
    if (cta0) {
        shm[0][threadIdx.x] = mz;
        shm[1][threadIdx.x] = mp;
        shm[2][threadIdx.x] = mu;
        __syncthreads();
        for (int o = kRed / 2; o > 0; o >>= 1) {
            if (threadIdx.x < o)
#pragma unroll
                for (int t = 0; t < 3; ++t) shm[t][threadIdx.x] = fmax(shm[t][threadIdx.x], shm[t][threadIdx.x + o]);
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            s->beta = beta;
            s->rho[it & 1] = rz;
            s->sc[0] = pcg_pow2_scale(__dadd_rn(shm[0][0], __dmul_rn(fabs(beta), shm[1][0])));
            s->sc[1] = pcg_pow2_scale(shm[2][0]);
        }
    }
    double m = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < nb) {
            const double pn = __dadd_rn(zv[e], __dmul_rn(beta, pv[e]));
#ifdef IEDD_DEBUG_FUSE
            if (i < 3 && blockIdx.x == 0) printf("iterb i %d z %.17g pold %.17g pnew %.17g beta %.17g\n", i, zv[e], pv[e], pn, beta);
#endif
            p[i] = pn;
            m = fmax(m, fabs(pn));
        }
    }
    __syncthreads();
    m = chunk_absmax(m, sh);
    if (threadIdx.x == 0) pmax[blockIdx.x] = m;
    if (replay) {  // graph replay: the last CTA (every CTA has read it_dev) advances the iteration
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&s->ticket, 1u) == gridDim.x - 1) {
                s->ticket = 0;
                s->it_dev += 1;
            }
        }
    }
}

// After the first apply (pcg.py:85-91): rho_0 = r.z (every CTA reduces, CTA 0
// stores), p = z and max|p| per chunk (= max|z|, the record's field 1).
// pglob (the fused p update's rotating global max|p| slots, zeroed before):
// slot 1 = max|p_1|.
__global__ void __launch_bounds__(kRed) k_pcg_setup(const double* xrz, int nch, PcgState* s, double* p,
                                                    const double* z, int nb, int c0, double* pmax, double* pglob) {
    __shared__ double sh[kRed];
    if (s->stop) return;
    const int base = blockIdx.x * kChunk;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < nb) p[i] = z[i];
    }
    if (threadIdx.x == 0) {
        const double m = xrz[kRzRec * (c0 + blockIdx.x) + 1];
        if (pmax) pmax[blockIdx.x] = m;
        if (pglob) atomicMax(reinterpret_cast<unsigned long long*>(pglob + 1), (unsigned long long)__double_as_longlong(m));
    }
    if (blockIdx.x != 0) return;
    double loc = 0.0;
    for (int c = threadIdx.x; c < nch; c += kRed) loc += xrz[kRzRec * c];
    const double rz = block_tree(loc, sh);
    if (threadIdx.x == 0) s->rho[0] = rz;
}

// The decider (pcg_decide) as a one-CTA kernel: the identity preconditioner
// has no scatter to host it.
__global__ void __launch_bounds__(kRed) k_decide(const double* rec, PcgDecide d, const int* stop) {
    __shared__ double sh[kRed];
    if (*stop) return;
    pcg_decide(rec, d, sh);
}

// The identity preconditioner (pcg.py:68): z = r, with the apply's chunk
// record fields 0 (r.z) and 1 (max|z|).
__global__ void __launch_bounds__(kRed) k_identity_apply(const double* r, double* z, int nb, double* rec,
                                                         const int* stop) {
    __shared__ double sh[2 * kRed];
    if (stop && *stop) return;
    const int base = blockIdx.x * kChunk;
    double loc = 0.0, zm = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < nb) {
            const double v = r[i];
            z[i] = v;
            loc = fma(v, v, loc);
            zm = fmax(zm, fabs(v));
        }
    }
    chunk_sum_max(loc, zm, sh, rec + kRzRec * blockIdx.x);
}

// Chunk partials of p.q (A-pass denominator) and |f - w|^2 (true residual of
// the previous iterate) -> xpost[2c], xpost[2c + 1] (c = c0 + blockIdx.x); the
// loads are issued before the stop flag is tested.
__global__ void k_post_pass(const double* p, const double* q, const double* f, const double* w, int N, int do_p,
                            int pending, double* xpost, const int* stop) {
#ifdef IEDD_DEBUG_FUSE
    if (blockIdx.x == 0 && threadIdx.x < 3 && !*stop) printf("kpost i %d p %.17g q %.17g w %.17g\n", threadIdx.x, p[threadIdx.x], q[threadIdx.x], w[threadIdx.x]);
#endif
    __shared__ double sh[kRed];
    pdl_wait();
    const int stopv = *stop;  // tested after the chunk loads are issued
    const int base = blockIdx.x * kChunk;
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < N) {
            if (do_p) a = fma(p[i], q[i], a);
            if (pending) {
                const double d = f[i] - w[i];
                b = fma(d, d, b);
            }
        }
    }
    if (stopv) return;
    if (do_p) {
        const double t = block_tree(a, sh);
        if (threadIdx.x == 0) xpost[2 * blockIdx.x] = t;
        __syncthreads();
    }
    if (pending) {
        const double t = block_tree(b, sh);
        if (threadIdx.x == 0) xpost[2 * blockIdx.x + 1] = t;
    }
}

__global__ void k_copy_if_running(double* dst, const double* src, int N, const int* stop) {
    pdl_wait();  // (launched with programmatic serialization inside the Lanczos step)
    if (*stop) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) dst[i] = src[i];
}

__global__ void k_reduce_rows(const double* part, int nch, double* out) {
    __shared__ double sh[kRed];
    const double v = reduce_partials(part + (int64_t)blockIdx.x * nch, nch, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = v;
}

constexpr int kLzMaxM = 1024;  // tridiagonal size staged in shared memory by k_lz_control

// Sturm count of eigenvalues < x for the symmetric tridiagonal (a, b2 = b^2)
// from the three-term recurrence of the leading principal minors
// p_i = (a_i - x) p_{i-1} - b_{i-1}^2 p_{i-2}: the count is the number of sign
// changes (a zero minor keeps the previous sign, as the pivot form's tiny
// positive substitute does).  Two dependent FP64 operations per step instead
// of a division; exact power-of-two rescaling keeps the minors in range.
__device__ int sturm_count_minors(const double* a, const double* b2, int m, double x) {
    double pm1 = 1.0, p = a[0] - x;
    bool neg = p < 0.0;
    int cnt = neg ? 1 : 0;
    for (int i = 1; i < m; ++i) {
        const double pn = fma(a[i] - x, p, -b2[i - 1] * pm1);
        pm1 = p;
        p = pn;
        if (p != 0.0) {
            const bool n = p < 0.0;
            cnt += n != neg;
            neg = n;
        }
        const double ap = fabs(p);
        if (ap > 0x1p+500 || (ap < 0x1p-500 && ap != 0.0)) {
            const double sc = ap > 1.0 ? 0x1p-500 : 0x1p+500;
            p *= sc;
            pm1 *= sc;
        }
    }
    return cnt;
}

// Sturm count of eigenvalues < x for the symmetric tridiagonal (a, b).
__device__ int sturm_count(const double* a, const double* b, int m, double x) {
    int cnt = 0;
    double d = a[0] - x;
    if (d < 0) ++cnt;
    for (int i = 1; i < m; ++i) {
        if (d == 0.0) d = 1e-300;
        d = (a[i] - x) - b[i - 1] * b[i - 1] / d;
        if (d < 0) ++cnt;
    }
    return cnt;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    cudaStream_t st;
    explicit DevBuf(cudaStream_t s) : st(s) {}
    cudaError_t alloc(size_t n) { return cudaMallocAsync((void**)&p, n * sizeof(T), st); }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

}  // namespace ie


using namespace ie;

static inline unsigned g1(int64_t n) { return (unsigned)((n + 255) / 256); }

namespace ie {

// Reusable PCG workspace (device vectors, partials, state, pinned status,
// events), cached per (N, history capacity) so repeated solves pay no
// allocation; a busy workspace is never shared between concurrent solves.
struct PcgWork {
    int N = 0;
    int64_t cap = 0;
    double *PU = nullptr, *QW = nullptr, *r = nullptr, *z = nullptr, *part = nullptr, *hist = nullptr;
    // part = [xf: nch | xpost: 2 npmax | xrz: kRzRec nch | pmax: nch | pglob: 3] (layouts above
    // k_iter_a); npmax = max(nch, lines of a 2D / 3D FFT pass) for the folded post pass
    int npmax = 0;
    double* fcopy = nullptr; // the right-hand side (graph-stable address)
    cudaStream_t cap_stream = nullptr;
    cudaStream_t side_stream = nullptr;  // graph side branch (u update)
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    cudaGraphExec_t gexec = nullptr;
    cudaGraphExec_t gexec_b = nullptr;  // kBatch iterations in one graph (no graph boundary between them)
    cudaGraphExec_t gexec_m = nullptr;  // 4 iterations (the remainder of a long batch size)
    uint64_t key_a = 0, key_t = 0;
    int gnodes = 0;  // kernel nodes in the captured iteration
    PcgState* st = nullptr;
    PcgState* host = nullptr;
    PcgState* host2 = nullptr;            // second pinned status slot (pipelined polling)
    cudaEvent_t poll_ev[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev;
    bool busy = false;
    ~PcgWork() {
        cudaFree(PU);
        cudaFree(QW);
        cudaFree(r);
        cudaFree(z);
        cudaFree(part);
        cudaFree(hist);
        cudaFree(fcopy);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (gexec_b) cudaGraphExecDestroy(gexec_b);
        if (gexec_m) cudaGraphExecDestroy(gexec_m);
        if (cap_stream) cudaStreamDestroy(cap_stream);
        if (side_stream) cudaStreamDestroy(side_stream);
        if (fork_ev) cudaEventDestroy(fork_ev);
        if (join_ev) cudaEventDestroy(join_ev);
        cudaFree(st);
        if (host) cudaFreeHost(host);
        if (host2) cudaFreeHost(host2);
        for (auto e : poll_ev)
            if (e) cudaEventDestroy(e);
        for (auto e : ev) cudaEventDestroy(e);
    }
};

static std::mutex g_work_mu;
static std::vector<PcgWork*> g_work;

static PcgWork* work_acquire(int N, int64_t cap, int* rc) {
    {
        std::lock_guard<std::mutex> lk(g_work_mu);
        for (PcgWork* w : g_work)
            if (!w->busy && w->N == N && w->cap >= cap) {
                w->busy = true;
                return w;
            }
    }
    PcgWork* w = new PcgWork();
    w->N = N;
    w->cap = cap;
    const int nch = dot_chunks(N);
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&w->PU, 2 * (size_t)N * 8);
    if (e == cudaSuccess) e = cudaMalloc(&w->QW, 2 * (size_t)N * 8);
    if (e == cudaSuccess) e = cudaMalloc(&w->r, (size_t)N * 8);
    if (e == cudaSuccess) e = cudaMalloc(&w->z, (size_t)N * 8);
    // xpost holds a partial pair per dot chunk, or per FFT output line (<= N^(2/3))
    w->npmax = std::max(nch, (int)ceil(pow((double)N, 2.0 / 3.0)) + 2);
    if (e == cudaSuccess) e = cudaMalloc(&w->part, ((2 + kRzRec) * (size_t)nch + 2 * (size_t)w->npmax + 3) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&w->hist, (size_t)cap * 8);
    if (e == cudaSuccess) e = cudaMalloc(&w->fcopy, (size_t)N * 8);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->cap_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->side_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w->fork_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w->join_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&w->st, sizeof(PcgState));
    if (e == cudaSuccess) e = cudaMallocHost(&w->host, sizeof(PcgState));
    if (e == cudaSuccess) e = cudaMallocHost(&w->host2, sizeof(PcgState));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w->poll_ev[0], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w->poll_ev[1], cudaEventDisableTiming);
    if (e != cudaSuccess) {
        set_error(std::string("pcg workspace: ") + cudaGetErrorString(e));
        delete w;
        *rc = IE_ERR_CUDA;
        return nullptr;
    }
    w->busy = true;
    std::lock_guard<std::mutex> lk(g_work_mu);
    g_work.push_back(w);
    return w;
}

static void work_release(PcgWork* w) {
    std::lock_guard<std::mutex> lk(g_work_mu);
    w->busy = false;
}

static int ensure_events(PcgWork* w, size_t n) {
    while (w->ev.size() < n) {
        cudaEvent_t e;
        IE_CUDA(cudaEventCreate(&e));
        w->ev.push_back(e);
    }
    return IE_OK;
}

}  // namespace ie

// prof != nullptr (ie_pcg_profile_f64): every iteration is launched directly
// (no graph, no side branch) with events between its kernel groups, and
// prof[0..4] accumulate the mean device ms of the steady-state (2-RHS)
// iterations' matvec, k_post_pass, k_iter_a, apply, k_iter_b.
static int pcg_impl(const ie_matvec* A, const ie_precond* T, const double* f, double* u, double tol,
                    int64_t max_iters, double* hist, int64_t* n_it, int32_t* flags, double* times,
                    int64_t* fail_iter, double* fail_value, void* stream, double* prof, double* h_u = nullptr) {
    if (!A || !f || (!u && !h_u) || !hist || !n_it || !flags || !times || max_iters < 0 ||
        !(tol > 0.0 && tol < 1.0)) {
        set_error("ie_pcg_f64: bad arguments");
        return IE_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int N = matvec_N(A);
    const int nch = dot_chunks(N);
    const auto t0 = std::chrono::steady_clock::now();
    int rc = IE_OK;
    int64_t cap = 1024;  // history capacity rounded up: warm-up and timed solves share a workspace
    while (cap < max_iters + 1) cap *= 2;
    PcgWork* W = work_acquire(N, cap, &rc);
    if (!W) return rc;
    struct Release {
        PcgWork* w;
        ~Release() { work_release(w); }
    } rel_guard{W};
    // apply events: pair 0 = initial apply, pair it = speculative apply of iteration it
    // steady iterations per graph replay (= per status poll).  Every replay boundary
    // costs ~10 us of idle GPU (graph launch + the poll's state copy), so large
    // problems take 16 (config 5: 4 -> 8 -1.3 us, -> 16 -2.0 us per iteration); a
    // converged solve runs up to two batches of no-op iterations (every kernel
    // returns on the stop flag, ~12 us per iteration), which small problems, whose
    // real iterations cost little more, cannot afford
    static const long long kb_env = getenv("IEDD_B200_KBATCH") ? atoll(getenv("IEDD_B200_KBATCH")) : 0;
    const int64_t kBatch = kb_env > 0 ? std::min<long long>(kb_env, 64) : (N >= (1 << 18) ? 16 : 4);
    if ((rc = ensure_events(W, 2 * (size_t)(std::min<int64_t>(cap, 4096) + 2)))) return rc;
    double* p = W->PU;
    double* uu = W->PU + N;
    double* q = W->QW;
    double* w = W->QW + N;
    double* xf = W->part;
    double* xpost = W->part + nch;
    double* xrz = xpost + 2 * W->npmax;
    double* pmax = xrz + kRzRec * nch;
    double* pglob = pmax + nch;
    const int* stop = &W->st->stop;
    // Buffers with disjoint lifetimes share storage, so the iteration's working
    // set fits the L2 (config 5: ~128 MB of vectors, work buffer, staging and
    // tables cycled through a 126 MB L2): z (scatter -> next pass's p update)
    // lives in q's storage (row inverse -> k_iter_a), and the apply's staging
    // buffer (class GEMM -> scatter) in the FFT work buffer (row forward -> row
    // inverse).  IEDD_B200_NO_ALIAS=1: separate buffers (comparison).
    static const bool alias = getenv("IEDD_B200_NO_ALIAS") == nullptr;
    double* const zv = alias ? q : W->z;
    // k_iter_b and k_post_pass folded into the FFT passes (2D / 3D FFT plans)
    static const bool no_fuse = getenv("IEDD_B200_NO_FUSE") != nullptr;
    static const bool no_fuse_upd = getenv("IEDD_B200_NO_FUSE_UPD") != nullptr;
    static const bool no_fuse_post = getenv("IEDD_B200_NO_FUSE_POST") != nullptr;
    const int nfl = no_fuse ? 0 : matvec_fused_lines(A);
    const bool fuse_upd = nfl > 0 && !no_fuse_upd, fuse_post = nfl > 0 && !no_fuse_post;
    const bool fused = fuse_upd || fuse_post;
    const int npost = fuse_post ? nfl : nch;
    // z = T^{-1} r and the chunk record's r.z / max|z| fields; with the p
    // update folded into the FFT (fuse_upd), the iteration's decider (beta,
    // rho, the next multipliers) runs on the completed record: in the last
    // CTA of the scatter, or (identity) a one-CTA k_decide
    auto apply_on = [&](const double* rin, double* zout, cudaStream_t s2, int64_t itd) -> int {
        PcgDecide dec;
        if (fuse_upd && itd != 0) {
            dec.s = W->st;
            dec.pglob = pglob;
            dec.it = itd;
            dec.nch = nch;
            dec.early = (pdl_early_mask() & 4) ? 1 : 0;
        }
        if (T) {
            precond_set_decide(&dec);
            if (alias) {  // the stream's idle FFT work buffer is the apply's staging buffer
                size_t sb = 0;
                double* sbuf = matvec_scratch(A, s2, &sb);
                precond_set_staging(sbuf, sb);
            }
            const int r2 = precond_apply(T, rin, zout, xrz, s2, stop);
            precond_set_staging(nullptr, 0);
            precond_set_decide(nullptr);
            return r2;
        }
        k_identity_apply<<<nch, kRed, 0, s2>>>(rin, zout, N, xrz, stop);
        IE_LAUNCHED();
        if (dec.s) {
            k_decide<<<1, kRed, 0, s2>>>(xrz, dec, stop);
            IE_LAUNCHED();
        }
        return IE_OK;
    };
    auto apply = [&](const double* rin, double* zout, int64_t evi) -> int {
        const bool timed = 2 * evi + 1 < (int64_t)W->ev.size();
        if (timed) IE_CUDA(cudaEventRecord(W->ev[2 * evi], st));
        int r2 = apply_on(rin, zout, st, evi);  // (evi: the iteration; 0 = the initial apply)
        if (r2) return r2;
        if (timed) IE_CUDA(cudaEventRecord(W->ev[2 * evi + 1], st));
        return IE_OK;
    };
    // the right-hand side at a stable address (captured graphs reference it)
    // (k_pcg_begin: the copy, r = f, u = 0 and ||f||^2's chunk partials in one pass)
    k_pcg_begin<<<nch, kRed, 0, st>>>(f, W->fcopy, W->r, uu, N, xf);
    IE_LAUNCHED();
    f = W->fcopy;
    // ||f||, state init (pcg.py:72-91)
    k_pcg_init<<<1, kRed, 0, st>>>(xf, nch, W->st, tol, max_iters, W->hist);
    IE_LAUNCHED();
    if ((rc = apply(W->r, zv, 0))) return rc;
    IE_CUDA(cudaMemsetAsync(pglob, 0, 3 * sizeof(double), st));
    k_pcg_setup<<<nch, kRed, 0, st>>>(xrz, nch, W->st, p, zv, N, 0, pmax, fuse_upd ? pglob : nullptr);  // p = z, rho_0
    IE_LAUNCHED();
    // iterations: `it` = the iteration whose A-pass is enqueued; the pass also
    // carries u_{it-1} for the deferred true-residual check of iteration it-1.
    // Steady-state iterations (2 <= it < max_iters) replay one captured CUDA
    // graph that reads `it` from the device state.
    static const bool no_fork = getenv("IEDD_B200_NO_FORK") != nullptr;  // u update in k_iter_a (comparison)
    static const bool keep_w = getenv("IEDD_B200_KEEP_W") != nullptr;    // store the w = A u column (comparison)
    cudaEvent_t pev[6] = {};
    int64_t nprof = 0;
    if (prof) {
        for (auto& e : pev) IE_CUDA(cudaEventCreate(&e));
        for (int i = 0; i < 5; ++i) prof[i] = 0.0;
    }
    struct PevFree {
        cudaEvent_t* e;
        ~PevFree() {
            for (int i = 0; i < 6; ++i)
                if (e[i]) cudaEventDestroy(e[i]);
        }
    } pev_free{pev};
    auto enqueue_iter = [&](int64_t itarg, int do_p, int pending, bool spec, cudaStream_t s2, bool timed_apply,
                            int64_t evi) -> int {
        int r2;
        const bool pf = prof && do_p && pending && spec;
        auto mark = [&](int i) -> int {
            if (pf) IE_CUDA(cudaEventRecord(pev[i], s2));
            return IE_OK;
        };
        if ((r2 = mark(0))) return r2;
        PcgFuse fz;  // (fused: the previous iteration's k_iter_b and this pass's k_post_pass ride in the FFT)
        if (fused) {
            if (fuse_upd && do_p && pending) {
                fz.z = zv;
                fz.pglob = pglob;
                fz.s = W->st;
                fz.it = itarg;
            }
            fz.p = p;
            fz.f = f;
            fz.part = fuse_post ? xpost : nullptr;
            fz.q_col = do_p ? 0 : -1;
            fz.w_col = pending ? (do_p ? 1 : 0) : -1;
            fz.skip_w_store = fuse_post && !keep_w;
        }
        const PcgFuse* fzp = fused ? &fz : nullptr;
        if (do_p && pending) {
            r2 = matvec_launch(A, W->PU, N, 2, W->QW, N, 0, N, s2, stop, W->st->sc, fzp);
        } else if (do_p) {
            r2 = matvec_launch(A, p, N, 1, q, N, 0, N, s2, stop, nullptr, fzp);
        } else {
            r2 = matvec_launch(A, uu, N, 1, w, N, 0, N, s2, stop, nullptr, fzp);
        }
        if (r2 || (r2 = mark(1))) return r2;
        if (!fuse_post) {
            IE_CUDA(launch_k(k_post_pass, dim3(nch), dim3(kRed), 0, s2, (const double*)p, (const double*)q, f,
                             (const double*)w, N, do_p, pending, xpost, stop));
            IE_LAUNCHED();
        }
        if ((r2 = mark(2))) return r2;
        // in the captured iteration u += alpha p forks onto a side branch beside the apply
        const bool fork_u = itarg < 0 && do_p && spec && !no_fork && !prof;
        IE_CUDA(launch_k(fork_u ? k_iter_a<false> : k_iter_a<true>, dim3(nch), dim3(kRed), 0, s2,
                         (const double*)xpost, npost, do_p, pending, (long long)itarg, W->st, W->hist,
                         fork_u ? nullptr : uu, W->r, (const double*)p, (const double*)q, N, 0, nch, xrz,
                         fuse_upd ? nullptr : (const double*)pmax, HaloSeg{0, 0, 0, 0},
                         (pdl_early_mask() & 1) ? 2 : 0));
        IE_LAUNCHED();
        if (fork_u) {
            IE_CUDA(cudaEventRecord(W->fork_ev, s2));
            IE_CUDA(cudaStreamWaitEvent(W->side_stream, W->fork_ev, 0));
            k_update_u<<<nch, kRed, 0, W->side_stream>>>(W->st, uu, p, N, 0, xrz);
            IE_LAUNCHED();
            IE_CUDA(cudaEventRecord(W->join_ev, W->side_stream));
        }
        if (spec) {  // speculative: z_it is discarded if iteration it is the last
            if ((r2 = mark(3))) return r2;
            if (timed_apply && !pf) {
                if ((r2 = apply(W->r, zv, evi))) return r2;
            } else if ((r2 = apply_on(W->r, zv, s2, itarg))) {
                return r2;
            }
            if ((r2 = mark(4))) return r2;
            // k_iter_b (or the next pass's folded p update) rewrites p, which the side branch reads: join first
            if (fork_u) IE_CUDA(cudaStreamWaitEvent(s2, W->join_ev, 0));
            if (!fuse_upd) {
                IE_CUDA(launch_k(k_iter_b, dim3(nch), dim3(kRed), 0, s2, (const double*)xrz, nch,
                                 (long long)itarg, W->st, p, (const double*)zv, N, pmax));
                IE_LAUNCHED();
            }
            if ((r2 = mark(5))) return r2;
        }
        if (pf) {
            IE_CUDA(cudaEventSynchronize(pev[5]));
            float ms[5];
            for (int i = 0; i < 5; ++i) IE_CUDA(cudaEventElapsedTime(&ms[i], pev[i], pev[i + 1]));
            for (int i = 0; i < 5; ++i) prof[i] += ms[i];
            ++nprof;
        }
        return IE_OK;
    };
    const bool use_graph = max_iters >= 3 && !getenv("IEDD_B200_NO_GRAPH") && !prof;
    // kBatch iterations per replay: the iteration boundary inside the graph is an
    // ordinary (programmatic) kernel edge instead of a graph launch
    static const bool no_multi = getenv("IEDD_B200_GRAPH1") != nullptr;  // comparison: one iteration per replay
    if (use_graph) {
        const uint64_t ka = matvec_uid(A), kt = T ? precond_uid(T) : 0;
        if (!W->gexec || W->key_a != ka || W->key_t != kt) {
            for (cudaGraphExec_t* ge : {&W->gexec, &W->gexec_b, &W->gexec_m}) {
                if (*ge) cudaGraphExecDestroy(*ge);
                *ge = nullptr;
            }
            if (T && (rc = precond_prepare_stream(T, W->cap_stream))) return rc;
            if ((rc = matvec_prepare_stream(A, W->cap_stream))) return rc;
            for (int reps : {1, (int)kBatch, kBatch > 4 ? 4 : 0}) {
                if (!reps) continue;
                cudaGraph_t g;
                IE_CUDA(cudaStreamBeginCapture(W->cap_stream, cudaStreamCaptureModeThreadLocal));
                int r2 = IE_OK;
                for (int q = 0; q < reps && !r2; ++q)
                    r2 = enqueue_iter(-1, 1, 1, true, W->cap_stream, false, 0);  // the decider advances it_dev
                cudaError_t ce = cudaStreamEndCapture(W->cap_stream, &g);
                if (r2) return r2;
                IE_CUDA(ce);
                if (reps == 1) {
                    size_t nn = 0;
                    cudaGraphGetNodes(g, nullptr, &nn);
                    std::vector<cudaGraphNode_t> nodes(nn);
                    if (nn) cudaGraphGetNodes(g, nodes.data(), &nn);
                    W->gnodes = 0;
                    for (auto nd : nodes) {
                        cudaGraphNodeType t;
                        if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++W->gnodes;
                    }
                }
                ce = cudaGraphInstantiate(reps == 1 ? &W->gexec : (reps == (int)kBatch ? &W->gexec_b : &W->gexec_m), g, 0);
                cudaGraphDestroy(g);
                IE_CUDA(ce);
            }
            W->key_a = ka;
            W->key_t = kt;
        }
    }
    // pipelined status polling: a batch's state copy is queued behind it, and
    // the host waits on the PREVIOUS batch's copy, so the GPU never drains
    // between batches (at most one batch of no-op iterations -- every kernel
    // returns on the device stop flag -- follows convergence)
    int64_t it = 1, nbatch = 0, since_poll = 0;
    bool stopped = false, u_copied = false;
    // (iteration, true residual) of the last two polled states: the batch-size policy's view
    long long smp_k[2] = {-1, -1};
    double smp_r[2] = {0.0, 0.0};
    int nsmp = 0;
    auto poll = [&]() -> int {
        const int slot = (int)(nbatch & 1);
        PcgState* hs = slot ? W->host2 : W->host;
        IE_CUDA(cudaMemcpyAsync(hs, W->st, sizeof(PcgState), cudaMemcpyDeviceToHost, st));
        IE_CUDA(cudaEventRecord(W->poll_ev[slot], st));
        if (nbatch > 0) {
            IE_CUDA(cudaEventSynchronize(W->poll_ev[slot ^ 1]));
            const PcgState* prev = slot ? W->host : W->host2;
            if (prev->stop) stopped = true;
            if (prev->last_k > smp_k[1]) {
                smp_k[0] = smp_k[1];
                smp_r[0] = smp_r[1];
                smp_k[1] = prev->last_k;
                smp_r[1] = prev->last_rel;
                if (nsmp < 2) ++nsmp;
            }
        }
        ++nbatch;
        since_poll = 0;
        return IE_OK;
    };
    // Long batches (kBatch > 4) only while convergence is not in sight: a run the
    // caller bounded to a few batches, or an extrapolation of the polled residuals
    // that leaves at least three batches to go; otherwise 4-iteration replays (a
    // converged solve runs at most two of its batches as no-op iterations).
    auto long_batch = [&]() -> bool {
        if (kBatch <= 4) return true;  // (the "long" graph is the 4-iteration one)
        if (max_iters <= 4 * kBatch) return true;
        if (nsmp < 2 || !(smp_r[1] > 0.0) || !(smp_r[0] > 0.0)) return false;
        if (!(smp_r[1] < smp_r[0])) return true;  // not converging now
        const double rate = std::log(smp_r[1] / smp_r[0]) / (double)(smp_k[1] - smp_k[0]);
        return std::log(tol / smp_r[1]) / rate >= 3.0 * (double)kBatch;
    };
    while (it <= max_iters + 1 && !stopped) {
        const int do_p = it <= max_iters;
        const int pending = it >= 2;
        const bool spec = do_p && it < max_iters;
        if (use_graph && pending && spec) {
            if (it == 2) {
                k_set_it<<<1, 1, 0, st>>>(W->st, 2);
                IE_LAUNCHED();
            }
            if (!no_multi && it + kBatch - 1 < max_iters && long_batch()) {  // iterations it .. it + kBatch - 1 are all steady-state
                IE_CUDA(cudaGraphLaunch(W->gexec_b, st));
                g_launches.fetch_add(W->gnodes * kBatch, std::memory_order_relaxed);
                it += kBatch;
                since_poll += kBatch;
            } else if (!no_multi && W->gexec_m && it + 3 < max_iters) {
                IE_CUDA(cudaGraphLaunch(W->gexec_m, st));
                g_launches.fetch_add(W->gnodes * 4, std::memory_order_relaxed);
                it += 4;
                since_poll += 4;
            } else {
                IE_CUDA(cudaGraphLaunch(W->gexec, st));
                g_launches.fetch_add(W->gnodes, std::memory_order_relaxed);
                ++it;
                ++since_poll;
            }
        } else {
            if ((rc = enqueue_iter(it, do_p, pending, spec, st, true, it))) return rc;
            if (h_u && it == max_iters && !u_copied) {
                // u is final after this iteration's k_iter_a (every later kernel only reads
                // it, and after a stop every kernel is a no-op): its copy to the host runs
                // on the side stream beside the closing true-residual pass
                IE_CUDA(cudaEventRecord(W->fork_ev, st));
                IE_CUDA(cudaStreamWaitEvent(W->side_stream, W->fork_ev, 0));
                IE_CUDA(cudaMemcpyAsync(h_u, uu, (size_t)N * 8, cudaMemcpyDeviceToHost, W->side_stream));
                IE_CUDA(cudaEventRecord(W->join_ev, W->side_stream));
                u_copied = true;
            }
            ++it;
            ++since_poll;
        }
        // (no poll when at most four iterations remain: they are enqueued either way
        // and the closing copy follows)
        if ((since_poll >= 4 && max_iters - it > 4) || it > max_iters + 1)
            if ((rc = poll())) return rc;
    }
    // one closing round trip: the state, the history (its first entries
    // speculatively: n_it is only known from the state) and u
    const int64_t nh0 = std::min<int64_t>(max_iters + 1, 4096);
    IE_CUDA(cudaMemcpyAsync(W->host, W->st, sizeof(PcgState), cudaMemcpyDeviceToHost, st));
    IE_CUDA(cudaMemcpyAsync(hist, W->hist, (size_t)nh0 * 8, cudaMemcpyDeviceToHost, st));
    if (u) IE_CUDA(cudaMemcpyAsync(u, uu, (size_t)N * 8, cudaMemcpyDeviceToDevice, st));
    if (h_u && !u_copied) IE_CUDA(cudaMemcpyAsync(h_u, uu, (size_t)N * 8, cudaMemcpyDeviceToHost, st));
    IE_CUDA(cudaStreamSynchronize(st));
    if (u_copied) IE_CUDA(cudaEventSynchronize(W->join_ev));
    const PcgState S = *W->host;
    flags[0] = S.status == 1;
    flags[1] = S.status == 2;
    *n_it = S.n_it;
    if (S.status == 4 || S.status == 5) {
        if (fail_iter) *fail_iter = S.fail_iter;
        if (fail_value) *fail_value = S.fail_value;
    }
    const int64_t nh = S.n_it + 1;
    if (nh > nh0) {
        IE_CUDA(cudaMemcpyAsync(hist + nh0, W->hist + nh0, (size_t)(nh - nh0) * 8, cudaMemcpyDeviceToHost, st));
        IE_CUDA(cudaStreamSynchronize(st));
    }
    times[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    // t_s: mean device time of the applies the reference performs (initial + iterations 1..n_it-1)
    double tp = 0.0;
    int64_t np = 0;
    for (int64_t e = 0; e < S.n_it && 2 * e + 1 < (int64_t)W->ev.size(); ++e) {
        if (use_graph && e >= 2 && e < max_iters) continue;  // graph iterations are not event-timed
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, W->ev[2 * e], W->ev[2 * e + 1]) == cudaSuccess) {
            tp += ms * 1e-3;
            ++np;
        }
    }
    if (S.n_it == 0) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, W->ev[0], W->ev[1]) == cudaSuccess) tp = ms * 1e-3, np = 1;
    }
    cudaGetLastError();
    times[1] = np ? tp / (double)np : 0.0;
    if (S.nf == 0.0) times[0] = times[1] = 0.0;  // zero right-hand side (pcg.py:74-78)
    if (prof && nprof)
        for (int i = 0; i < 5; ++i) prof[i] /= (double)nprof;
    if (S.status == 4) return IE_ERR_BREAKDOWN;
    if (S.status == 5) return IE_ERR_NONFINITE;
    return IE_OK;
}

extern "C" int ie_pcg_f64(const ie_matvec* A, const ie_precond* T, const double* f, double* u, double tol,
                          int64_t max_iters, double* hist, int64_t* n_it, int32_t* flags, double* times,
                          int64_t* fail_iter, double* fail_value, void* stream) {
    return pcg_impl(A, T, f, u, tol, max_iters, hist, n_it, flags, times, fail_iter, fail_value, stream, nullptr);
}

extern "C" int ie_pcg_host_f64(const ie_matvec* A, const ie_precond* T, const double* f, double* h_u, double tol,
                               int64_t max_iters, double* hist, int64_t* n_it, int32_t* flags, double* times,
                               int64_t* fail_iter, double* fail_value, void* stream) {
    if (!h_u) {
        set_error("ie_pcg_host_f64: bad arguments");
        return IE_ERR_ARG;
    }
    return pcg_impl(A, T, f, nullptr, tol, max_iters, hist, n_it, flags, times, fail_iter, fail_value, stream, nullptr,
                    h_u);
}

extern "C" int ie_pcg_profile_f64(const ie_matvec* A, const ie_precond* T, const double* f, double* u, double tol,
                                  int64_t max_iters, double* hist, int64_t* n_it, int32_t* flags, double* times,
                                  double* h_phase_ms, void* stream) {
    if (!h_phase_ms) {
        set_error("ie_pcg_profile_f64: bad arguments");
        return IE_ERR_ARG;
    }
    int64_t fi = 0;
    double fv = 0.0;
    return pcg_impl(A, T, f, u, tol, max_iters, hist, n_it, flags, times, &fi, &fv, stream, h_phase_ms);
}

// ---------------------------------------------------------------- K5 --
// Lanczos state on the device (spectrum.py:154-189).  Every step kernel reads
// the step index j from the state and returns at once when `stop` is set, so
// one captured CUDA graph replays every step; the host reads the state every
// 8 steps.  Grids are sized for the largest basis and exit early above j.
struct LzState {
    double beta, est, cur, nrm;
    int have_est, stable, stop, status;  // status 1 converged, 2 beta^2 <= 0, 3 beta < 1e-14
    long long steps;
    long long j;  // current step (basis vectors 0..j)
};

__global__ void k_lz_init(const double* part, int nch, LzState* s) {
    __shared__ double sh[kRed];
    const double v = reduce_partials(part, nch, sh);
    if (threadIdx.x == 0) {
        s->nrm = sqrt(v);
        s->have_est = 0;
        s->stable = 0;
        s->stop = 0;
        s->status = 0;
        s->steps = 0;
        s->est = 0.0;
        s->j = 0;
    }
}

// V[0] = v0 / nrm, AV[0] = av / nrm, avj = AV[0]
__global__ void k_lz_first(double* V, double* AV, double* avj, const double* w, const double* aw, const LzState* s,
                           int N) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double d = s->nrm, wi = w[i], awi = aw[i];  // both loads ahead of the stores
    V[i] = wi / d;
    const double a = awi / d;
    AV[i] = a;
    avj[i] = a;
}

// V[j+1] = w / beta, AV[j+1] = aw / beta, avj = AV[j+1]  (spectrum.py:186-187)
__global__ void k_lz_next(double* V, double* AV, double* avj, const double* w, const double* aw, const LzState* s,
                          int N) {
    pdl_wait();  // (launched with programmatic serialization inside the Lanczos step)
    if (s->stop) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int64_t off = (s->j + 1) * (int64_t)N;
    const double d = s->beta, wi = w[i], awi = aw[i];
    V[off + i] = wi / d;
    const double a = awi / d;
    AV[off + i] = a;
    avj[i] = a;
}

__global__ void k_lz_advance(LzState* s) {
    pdl_wait();  // (launched with programmatic serialization inside the Lanczos step)
    if (!s->stop) s->j += 1;
}

__global__ void k_lz_alpha(const double* part, int nch, double* alphas, const LzState* s) {
    pdl_wait();  // (launched with programmatic serialization inside the Lanczos step)
    __shared__ double sh[kRed];
    if (s->stop) return;
    const double v = reduce_partials(part, nch, sh);
    if (threadIdx.x == 0) alphas[s->j] = v;
}

// beta^2 = w.aw, Ritz value of T_j by 256-way Sturm multisection, the
// reference's stopping rule.  Cauchy interlacing bounds the new extremal
// Ritz value by the previous one (lambda_min(T_m) <= lambda_min(T_{m-1}),
// lambda_max(T_m) >= lambda_max(T_{m-1})), which brackets one side.
__global__ void __launch_bounds__(kRed) k_lz_control(const double* part, int nch, const double* a, double* b,
                                                     int which, double rtol, LzState* s) {
    pdl_wait();  // (launched with programmatic serialization inside the Lanczos step)
    __shared__ double sh[kRed];
    __shared__ double br[2];
    __shared__ unsigned above_mask[kRed / 32];
    if (s->stop) return;
    const int m = (int)(s->j + 1);
    const double beta2 = reduce_partials(part, nch, sh);
    if (!(beta2 > 0.0) || !isfinite(beta2)) {
        if (threadIdx.x == 0) {
            s->status = 2;
            s->stop = 1;
            s->steps = m;
        }
        return;
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp == 0) {
        double lo = a[0], hi = a[0];
        for (int i = lane; i < m; i += 32) {
            const double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i < m - 1 ? fabs(b[i]) : 0.0);
            lo = fmin(lo, a[i] - r);
            hi = fmax(hi, a[i] + r);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        const double span = fmax(hi - lo, 1e-300);
        lo -= 1e-3 * span + 1e-300;
        hi += 1e-3 * span + 1e-300;
        if (lane == 0) {
            if (s->have_est) {  // interlacing bound (with a small rounding margin)
                const double e = s->est, mg = 1e-12 * fabs(e) + 1e-300;
                if (which == 0 && e + mg < hi && e + mg > lo) hi = e + mg;
                if (which == 1 && e - mg > lo && e - mg < hi) lo = e - mg;
            }
            br[0] = lo;
            br[1] = hi;
        }
    }
    __syncthreads();
    const int target = which == 0 ? 1 : m;  // count(x) >= target  <=>  x > lambda
    __shared__ double sa[kLzMaxM], sb2[kLzMaxM];
    const bool smem_tri = m <= kLzMaxM;
    if (smem_tri) {
        for (int i = tid; i < m; i += kRed) {
            sa[i] = a[i];
            sb2[i] = i < m - 1 ? b[i] * b[i] : 0.0;
        }
        __syncthreads();
    }
    // With the previous Ritz value as the interlacing end of the bracket, the
    // first round places its points geometrically towards that end (spacing
    // ratio 2^(64/255): the converging Ritz value sits just beside it); later
    // rounds subdivide uniformly.  About 4 rounds instead of 7.
    const bool geo = s->have_est;
    for (int it = 0; it < 16; ++it) {
        const double lo = br[0], hi = br[1];
        double x;
        if (it == 0 && geo) {  // increasing in tid; dense next to the interlacing end
            const double step = 64.0 / (double)(kRed - 1);
            x = which == 0 ? hi - (hi - lo) * exp2(-(double)tid * step)               // lo .. hi - 2^-64 (hi - lo)
                           : lo + (hi - lo) * exp2(-(double)(kRed - 1 - tid) * step);  // lo + 2^-64 (hi - lo) .. hi
        } else {
            x = lo + (hi - lo) * (double)(tid + 1) / (double)(kRed + 1);
        }
        __shared__ double xs[kRed];
        xs[tid] = x;
        const bool above = (smem_tri ? sturm_count_minors(sa, sb2, m, x) : sturm_count(a, b, m, x)) >= target;
        const unsigned mk = __ballot_sync(0xffffffffu, above);
        if (lane == 0) above_mask[warp] = mk;
        __syncthreads();
        if (tid == 0) {
            int first = kRed;
            for (int w2 = 0; w2 < kRed / 32; ++w2)
                if (above_mask[w2]) {
                    first = w2 * 32 + __ffs(above_mask[w2]) - 1;
                    break;
                }
            // the points increase with tid: lambda lies between point first-1 and point first
            br[0] = first == 0 ? lo : xs[first - 1];
            br[1] = first == kRed ? hi : xs[first];
        }
        __syncthreads();
        const double nlo = br[0], nhi = br[1];
        if ((!(nhi < hi) && !(nlo > lo)) || nhi - nlo <= 2.0 * 2.220446049250313e-16 * fmax(fabs(nlo), fabs(nhi)))
            break;
    }
    if (tid != 0) return;
    const double cur = 0.5 * (br[0] + br[1]);
    const double beta = sqrt(beta2);
    s->cur = cur;
    s->steps = m;
    if (s->have_est && fabs(cur - s->est) <= rtol * fmax(fabs(cur), 1.0)) {
        if (++s->stable >= 5) {
            s->status = 1;
            s->stop = 1;
            return;
        }
    } else {
        s->stable = 0;
    }
    s->est = cur;
    s->have_est = 1;
    if (beta < 1e-14) {
        s->status = 3;
        s->stop = 1;
        return;
    }
    s->beta = beta;
    b[m - 1] = beta;
}

// c_i = AV_i . w for i <= j (grid rows above j exit)
__global__ void k_lz_gemv_t(const double* AV, const double* w, int N, double* part, int nch, const LzState* s) {
    pdl_wait();  // (launched with programmatic serialization inside the Lanczos step)
    __shared__ double sh[kRed];
    if (s->stop || blockIdx.y > s->j) return;
    const double* v = AV + (int64_t)blockIdx.y * N;
    const int base = blockIdx.x * kChunk;
    double loc = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int t = base + e * kRed + threadIdx.x;
        if (t < N) loc = fma(v[t], w[t], loc);
    }
    const double r = block_tree(loc, sh);
    if (threadIdx.x == 0) part[(int64_t)blockIdx.y * nch + blockIdx.x] = r;
}

__global__ void k_lz_reduce_rows(const double* part, int nch, double* out, const LzState* s) {
    pdl_wait();  // (launched with programmatic serialization inside the Lanczos step)
    __shared__ double sh[kRed];
    if (s->stop || blockIdx.x > s->j) return;
    const double v = reduce_partials(part + (int64_t)blockIdx.x * nch, nch, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = v;
}

// w -= sum_{i<=j} c_i V_i: a CTA owns 32 consecutive entries, its 8 warps
// take basis vectors i = warp (mod 8), and the partial sums are combined in
// warp order (fixed association: deterministic).
__global__ void __launch_bounds__(256) k_lz_gemv_sub(double* w, const double* V, const double* c, int N,
                                                     const LzState* s) {
    pdl_wait();  // (launched with programmatic serialization inside the Lanczos step)
    __shared__ double part8[8][32];
    if (s->stop) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    const int nb = (int)(s->j + 1);
    double acc = 0.0;
    if (t < N)
        for (int i = warp; i < nb; i += 8) acc = fma(c[i], V[(int64_t)i * N + t], acc);
    part8[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && t < N) {
        double tot = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) tot += part8[q][lane];
        w[t] -= tot;
    }
}

__global__ void k_lz_dot(const double* x, const double* y, int N, double* part, const LzState* s) {
    pdl_wait();  // (launched with programmatic serialization inside the Lanczos step)
    __shared__ double sh[kRed];
    if (s->stop) return;
    const int base = blockIdx.x * kChunk;
    double loc = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < N) loc = fma(x[i], y[i], loc);
    }
    const double t = block_tree(loc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

extern "C" int ie_lanczos_f64(const ie_matvec* A, const ie_precond* T, const double* v0, int32_t which,
                              int64_t max_iters, double rtol, double* lambda, int64_t* steps, void* stream) {
    if (!A || !v0 || !lambda || (which != 0 && which != 1) || max_iters < 0) {
        set_error("ie_lanczos_f64: bad arguments");
        return IE_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int N = matvec_N(A);
    const int nch = dot_chunks(N);
    const int64_t nb_max = max_iters + 1;
    DevBuf<double> V(st), AV(st), wb(st), awb(st), avj(st), part(st), cbuf(st), tri(st);
    DevBuf<LzState> S(st);
    IE_CUDA(V.alloc((size_t)nb_max * N));
    IE_CUDA(AV.alloc((size_t)nb_max * N));
    IE_CUDA(wb.alloc(N));
    IE_CUDA(awb.alloc(N));
    IE_CUDA(avj.alloc(N));
    IE_CUDA(part.alloc((size_t)std::max<int64_t>(nb_max, 2) * nch));
    IE_CUDA(cbuf.alloc(nb_max + 2));
    IE_CUDA(tri.alloc(2 * (size_t)nb_max + 2));
    IE_CUDA(S.alloc(1));
    // pinned status buffer, one per host thread (allocated once)
    static thread_local LzState* hs = nullptr;
    if (!hs) IE_CUDA(cudaMallocHost(&hs, sizeof(LzState)));
    double* da = tri.p;           // alphas
    double* db = tri.p + nb_max;  // betas
    const int* stop = &S.p->stop;
    int rc;
    // v = v0; av = A v; nrm = sqrt(v.av); v /= nrm; av /= nrm   (spectrum.py:148-153)
    if ((rc = matvec_launch(A, v0, N, 1, awb.p, N, 0, N, st, nullptr))) return rc;
    k_dot_partials<<<nch, kRed, 0, st>>>(v0, awb.p, N, 0, part.p);
    IE_LAUNCHED();
    k_lz_init<<<1, kRed, 0, st>>>(part.p, nch, S.p);
    IE_LAUNCHED();
    k_lz_first<<<g1(N), 256, 0, st>>>(V.p, AV.p, avj.p, v0, awb.p, S.p, N);
    IE_LAUNCHED();
    // one Lanczos step (spectrum.py:160-187) on stream s2
    auto step = [&](cudaStream_t s2) -> int {
        int r2;
        if (T) {
            if ((r2 = precond_apply(T, avj.p, wb.p, nullptr, s2, stop))) return r2;
        } else {  // identity (precond.py:133-134)
            IE_CUDA(launch_k(k_copy_if_running, dim3(g1(N)), dim3(256), 0, s2, wb.p, (const double*)avj.p, N, stop));
            IE_LAUNCHED();
        }
        IE_CUDA(launch_k(k_lz_dot, dim3(nch), dim3(kRed), 0, s2, (const double*)wb.p, (const double*)avj.p, N, part.p, (const LzState*)S.p));
        IE_LAUNCHED();
        IE_CUDA(launch_k(k_lz_alpha, dim3(1), dim3(kRed), 0, s2, (const double*)part.p, nch, da, (const LzState*)S.p));
        IE_LAUNCHED();
        for (int pass = 0; pass < 2; ++pass) {  // two-pass A-orthogonalisation (CGS2)
            IE_CUDA(launch_k(k_lz_gemv_t, dim3(nch, (unsigned)nb_max), dim3(kRed), 0, s2, (const double*)AV.p, (const double*)wb.p, N, part.p, nch, (const LzState*)S.p));
            IE_LAUNCHED();
            IE_CUDA(launch_k(k_lz_reduce_rows, dim3((unsigned)nb_max), dim3(kRed), 0, s2, (const double*)part.p, nch, cbuf.p, (const LzState*)S.p));
            IE_LAUNCHED();
            IE_CUDA(launch_k(k_lz_gemv_sub, dim3((unsigned)((N + 31) / 32)), dim3(256), 0, s2, wb.p, (const double*)V.p, (const double*)cbuf.p, N, (const LzState*)S.p));
            IE_LAUNCHED();
        }
        if ((r2 = matvec_launch(A, wb.p, N, 1, awb.p, N, 0, N, s2, stop))) return r2;
        IE_CUDA(launch_k(k_lz_dot, dim3(nch), dim3(kRed), 0, s2, (const double*)wb.p, (const double*)awb.p, N, part.p, (const LzState*)S.p));
        IE_LAUNCHED();
        IE_CUDA(launch_k(k_lz_control, dim3(1), dim3(kRed), 0, s2, (const double*)part.p, nch, (const double*)da, db, which, rtol, S.p));
        IE_LAUNCHED();
        IE_CUDA(launch_k(k_lz_next, dim3(g1(N)), dim3(256), 0, s2, V.p, AV.p, avj.p, (const double*)wb.p, (const double*)awb.p, (const LzState*)S.p, N));
        IE_LAUNCHED();
        IE_CUDA(launch_k(k_lz_advance, dim3(1), dim3(1), 0, s2, S.p));
        IE_LAUNCHED();
        return IE_OK;
    };
    // the first kGraphAfter steps are launched directly (short runs never pay the
    // capture); longer runs replay one captured step graph
    constexpr int64_t kGraphAfter = 16;
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t cap = nullptr;
    int gnodes = 0;
    struct GraphFree {
        cudaGraphExec_t* e;
        cudaStream_t* c;
        ~GraphFree() {
            if (*e) cudaGraphExecDestroy(*e);
            if (*c) cudaStreamDestroy(*c);
        }
    } gf{&gexec, &cap};
    const bool graph_ok = !getenv("IEDD_B200_NO_GRAPH");
    const int64_t kBatch = 8;
    for (int64_t j = 0; j < max_iters; ++j) {
        if (graph_ok && j >= kGraphAfter && !gexec) {
            IE_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
            if (T && precond_prepare_stream(T, cap)) return IE_ERR_CUDA;
            if (matvec_prepare_stream(A, cap)) return IE_ERR_CUDA;
            cudaGraph_t g;
            IE_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
            rc = step(cap);
            cudaError_t ce = cudaStreamEndCapture(cap, &g);
            if (rc) return rc;
            IE_CUDA(ce);
            size_t nn = 0;
            cudaGraphGetNodes(g, nullptr, &nn);
            gnodes = (int)nn;
            ce = cudaGraphInstantiate(&gexec, g, 0);
            cudaGraphDestroy(g);
            IE_CUDA(ce);
        }
        if (gexec) {
            IE_CUDA(cudaGraphLaunch(gexec, st));
            g_launches.fetch_add(gnodes, std::memory_order_relaxed);
        } else if ((rc = step(st))) {
            return rc;
        }
        if ((j + 1) % kBatch == 0 || j + 1 == max_iters) {
            IE_CUDA(cudaMemcpyAsync(hs, S.p, sizeof(LzState), cudaMemcpyDeviceToHost, st));
            IE_CUDA(cudaStreamSynchronize(st));
            if (hs->stop) break;
        }
    }
    IE_CUDA(cudaMemcpyAsync(hs, S.p, sizeof(LzState), cudaMemcpyDeviceToHost, st));
    IE_CUDA(cudaStreamSynchronize(st));
    if (steps) *steps = hs->steps;
    if (!hs->have_est) {
        set_error("Lanczos produced no Ritz values");
        return IE_ERR_NO_RITZ;
    }
    *lambda = hs->status == 1 ? hs->cur : hs->est;
    return IE_OK;
}

// ------------------------------------------------------------------------
// Vector operations of the PCG iteration exposed for the sharded driver
// (paper_2108_12574_b200/distributed.py).  They are the same kernels and the
// same reduction order as ie_pcg_f64, so a sharded solve reproduces the
// single-GPU one bitwise.
namespace ie {
__global__ void k_update_host(int op, double* a, const double* b, double s, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (op == 0) a[i] = __dadd_rn(a[i], __dmul_rn(s, b[i]));
    else if (op == 1) a[i] = __dsub_rn(a[i], __dmul_rn(s, b[i]));
    else a[i] = __dadd_rn(b[i], __dmul_rn(s, a[i]));
}
}  // namespace ie

extern "C" int64_t ie_dot_chunk(void) { return ie::kChunk; }

extern "C" int ie_dot_partials_f64(const double* x, const double* y, int64_t n, int32_t mode, double* part,
                                   void* stream) {
    if (!x || !y || !part || n < 0 || n > 2147483647LL || (mode != 0 && mode != 1)) {
        set_error("ie_dot_partials_f64: bad arguments");
        return IE_ERR_ARG;
    }
    if (n == 0) return IE_OK;
    k_dot_partials<<<dot_chunks(n), kRed, 0, (cudaStream_t)stream>>>(x, y, (int)n, mode, part);
    IE_LAUNCHED();
    return IE_OK;
}

extern "C" int ie_sum_partials_f64(const double* part, int64_t nch, double* out, void* stream) {
    if (!part || !out || nch < 1) {
        set_error("ie_sum_partials_f64: bad arguments");
        return IE_ERR_ARG;
    }
    k_reduce_rows<<<1, kRed, 0, (cudaStream_t)stream>>>(part, (int)nch, out);
    IE_LAUNCHED();
    return IE_OK;
}

extern "C" int ie_update_f64(int32_t op, double* a, const double* b, double s, int64_t n, void* stream) {
    if (!a || !b || n < 0 || op < 0 || op > 2) {
        set_error("ie_update_f64: bad arguments");
        return IE_ERR_ARG;
    }
    if (n == 0) return IE_OK;
    k_update_host<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(op, a, b, s, n);
    IE_LAUNCHED();
    return IE_OK;
}


// ------------------------------------------------ sharded K4 (NVLink P2P) --
// ie_pcg_f64 on G ranks, one per GPU: rank g owns the grid-row band
// [b0, b1) of every vector (equal, chunk-aligned bands of whole rows; the 2D
// FFT operator with G | 2n).  There is no collective library on this path:
// every exchange is a push of the producer's slab straight into the
// consumers' memory over NVLink (peer pointers from CUDA IPC), followed by a
// system-scope release add of the byte count on the consumer's mailbox
// counter; the consumer's k_wait spins (acquire) until the expected bytes of
// the epoch have arrived.  Per PCG iteration there are four exchange points,
// the dependency chain of the algorithm:
//   FWD   row FFTs of the band -> column slab owners (all-to-all transpose);
//   BACK  column pass -> every rank's NEED rows (band + the rows its
//         subdomains read outside it): the second transpose also carries the
//         r-halo, because the rank recomputes q on its halo rows and applies
//         r -= alpha q there itself, bitwise as the owner does;
//   POST  p.q and |f - A u|^2 chunk partials (all-gather);
//   RZ    the apply's chunk record (r.z, max|z|, max|p|, max|u|): beta and
//         the next pass's 2-RHS scales on every rank (no max|p| exchange).
// Every rank reduces the global chunk order with the single-GPU kernels, so
// n_it, the history and u are bitwise those of ie_pcg_f64 for any G.
// Buffers are single-buffered: each push of epoch e into a peer happens
// after the pusher has consumed that peer's previous exchange, which the peer
// sent only after its last read of the buffer.
// Counters are monotonic over the shard's lifetime (never reset: a peer may
// already be pushing the next solve's first exchange).
//
// The same driver runs G ranks inside one process on one device
// (ie_pcg_sharded_local_f64; peers are plain device pointers): every
// exchange phase runs for all ranks before the next phase starts, so no
// kernel ever waits on work queued behind it.  This is how the G > 1 paths
// are tested on a single B200 (tests/test_gpu_parity.py::TestShardedP2P).
struct ie_fft;
namespace ie {
const ie_fft* matvec_fft(const ie_matvec* m);
int matvec_dim(const ie_matvec* m);
int matvec_n(const ie_matvec* m);
int fft_M(const ie_fft* f);
int fft_band_fwd(const ie_fft* f, const double* X0, const double* X1, int nrows, int parts, double2* out,
                 const double* scales, cudaStream_t st, const int* stop, const PeerStores* ps);
int fft_band_cols(const ie_fft* f, double2* buf, int c0, int ncols, cudaStream_t st, const int* stop,
                  const PeerStores* ps);
int fft_band_inv(const ie_fft* f, const double2* in, int nrows, int parts, double* Y0, double* Y1,
                 const double* scales, cudaStream_t st, const int* stop, const PcgFuse* fz);
int precond_apply_band(const ie_precond* p, const double* r, double* z, double* partials, int64_t i0, int64_t i1,
                       cudaStream_t st, const int* stop);

enum XSlot { kSlotF = 0, kSlotRz, kSlotFwd, kSlotBack, kSlotPost, kNumSlots };
constexpr int kMaxRanks = 16;
constexpr int kPushThreads = 256;

struct PushDesc {
    const char* src;
    char* dst;
    long long bytes;  // multiple of 8
    unsigned long long* ctr;
};
struct PushArgs {
    PushDesc d[kMaxRanks];
    const int* stop;
};

// Copy descriptor blockIdx.y (16-B words, tile t of kPushThreads words to CTA
// t mod gridDim.x; an odd trailing 8-B word by CTA 0), then release-add the
// CTA's bytes to the consumer's counter.  src == dst (a rank's own slab,
// already in place) only counts.
__global__ void __launch_bounds__(kPushThreads) k_push(const __grid_constant__ PushArgs a) {
    pdl_wait();
    if (*a.stop) return;
    const PushDesc d = a.d[blockIdx.y];
    const long long nw = d.bytes >> 4, step = (long long)gridDim.x * kPushThreads;
    if (d.src != d.dst) {
        const int4* s = reinterpret_cast<const int4*>(d.src);
        int4* t = reinterpret_cast<int4*>(d.dst);
        long long w = (long long)blockIdx.x * kPushThreads + threadIdx.x;
        for (; w + 3 * step < nw; w += 4 * step) {  // four loads in flight per thread
            const int4 v0 = s[w], v1 = s[w + step], v2 = s[w + 2 * step], v3 = s[w + 3 * step];
            t[w] = v0;
            t[w + step] = v1;
            t[w + 2 * step] = v2;
            t[w + 3 * step] = v3;
        }
        for (; w < nw; w += step) t[w] = s[w];
        if ((d.bytes & 15) && blockIdx.x == 0 && threadIdx.x == 0)
            reinterpret_cast<double*>(d.dst)[2 * nw] = reinterpret_cast<const double*>(d.src)[2 * nw];
    }
    long long cnt = 0;
    for (long long t0 = (long long)blockIdx.x * kPushThreads; t0 < nw; t0 += step)
        cnt += nw - t0 < kPushThreads ? nw - t0 : kPushThreads;
    cnt <<= 4;
    if (blockIdx.x == 0) cnt += d.bytes & 15;
    __syncthreads();
    if (threadIdx.x == 0 && cnt > 0) {
        __threadfence_system();
        atomicAdd_system(d.ctr, (unsigned long long)cnt);
    }
}

// Spin until the epoch's expected bytes have arrived, then advance the
// target.  A rank whose peers stop sending fails loudly instead of hanging:
// after 30 s the solve stops with status 6 (IE_ERR_CUDA "peer exchange
// timed out").
__global__ void k_wait(const unsigned long long* ctr, unsigned long long* tgt, unsigned long long expect,
                       PcgState* s) {
    if (threadIdx.x != 0 || s->stop) return;
    const unsigned long long target = *tgt + expect;
    unsigned long long t0, t1, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        if (v >= target) break;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 30ull * 1000000000ull) {
            s->status = 6;
            s->stop = 1;
            return;
        }
        __nanosleep(32);
    }
    *tgt = target;
}

__global__ void k_clear_stop(PcgState* s) {
    s->stop = 0;
    s->status = 0;
}
}  // namespace ie

struct ie_shard {
    int G = 1, g = 0;
    const ie_matvec* A = nullptr;
    const ie_precond* T = nullptr;
    const ie_fft* F = nullptr;
    uint64_t key_a = 0, key_t = 0;
    int n = 0, M = 0, Mc = 0, N = 0;
    int64_t b0 = 0, b1 = 0, nb = 0;
    int nrows = 0, row0 = 0, rlo = 0, rhi = 0, R = 0, Rmax = 0;
    int nch = 0, nchb = 0, c0 = 0;
    bool line_post = false;  // k_post_pass folded into the inverse rows (per-row partials), as ie_pcg_f64 does
    bool fused_transposes = true;  // FWD / BACK written by the band passes into the peers (no push kernels)
    std::vector<int> row0_all, nrows_all, rlo_all, rhi_all;
    // symmetric exchange heap (IPC-exported): mailbox counters, F partials,
    // POST partials, RZ records, column slab, need-row block
    char* heap = nullptr;
    size_t heap_bytes = 0, off_xf = 0, off_xpost = 0, off_xrz = 0, off_buf2 = 0, off_buf3 = 0;
    std::vector<char*> peer;
    std::vector<bool> opened;
    bool connected = false, broken = false;
    // rank-local
    double *PU = nullptr, *QW = nullptr, *rfull = nullptr, *z = nullptr, *fb = nullptr, *pmax = nullptr;
    double* dh = nullptr;
    int64_t cap = 0;
    double2* buf1 = nullptr;
    unsigned long long* tgt = nullptr;
    ie::PcgState* S = nullptr;
    ie::PcgState* host = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // the captured steady-state iteration (this rank alone, or -- local
    // mode -- all ranks of the process, owned by rank 0's shard)
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t cap_s = nullptr;
    int gnodes = 0, gmode = 0;

    unsigned long long* mb(int h) const { return reinterpret_cast<unsigned long long*>(peer[h]); }
    double* xf(int h) const { return reinterpret_cast<double*>(peer[h] + off_xf); }
    double* xpost(int h) const { return reinterpret_cast<double*>(peer[h] + off_xpost); }
    double* xrz(int h) const { return reinterpret_cast<double*>(peer[h] + off_xrz); }
    double2* buf2(int h) const { return reinterpret_cast<double2*>(peer[h] + off_buf2); }
    double2* buf3(int h) const { return reinterpret_cast<double2*>(peer[h] + off_buf3); }
    ~ie_shard() {
        for (int h = 0; h < (int)peer.size(); ++h)
            if (h < (int)opened.size() && opened[h]) cudaIpcCloseMemHandle(peer[h]);
        for (void* p : {(void*)heap, (void*)PU, (void*)QW, (void*)rfull, (void*)z, (void*)fb, (void*)pmax, (void*)dh,
                        (void*)buf1, (void*)tgt, (void*)S})
            if (p) cudaFree(p);
        if (host) cudaFreeHost(host);
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (cap_s) cudaStreamDestroy(cap_s);
    }
};

namespace ie {
static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

static int shard_push(const ie_shard* sh, int slot, const PushDesc* d, int nd, cudaStream_t s) {
    if (sh->G == 1 || nd == 0) return IE_OK;
    PushArgs a{};
    long long mx = 0;
    for (int i = 0; i < nd; ++i) {
        a.d[i] = d[i];
        a.d[i].ctr = sh->mb(i) + slot;
        mx = std::max(mx, d[i].bytes);
    }
    a.stop = &sh->S->stop;
    const long long tiles = (mx / 16 + kPushThreads - 1) / kPushThreads;  // (>= 1 CTA even for an 8-B slab)
    const unsigned gx = (unsigned)std::max(1LL, std::min(tiles / 2, 64LL));
    IE_CUDA(launch_k(k_push, dim3(gx, nd), dim3(kPushThreads), 0, s, a));
    IE_LAUNCHED();
    return IE_OK;
}

static int shard_wait(const ie_shard* sh, int slot, unsigned long long expect, cudaStream_t s) {
    if (sh->G == 1) return IE_OK;
    k_wait<<<1, 32, 0, s>>>(sh->mb(sh->g) + slot, sh->tgt + slot, expect, sh->S);
    IE_LAUNCHED();
    return IE_OK;
}

// the rank's slab of a globally indexed exchange array (entries [first,
// first + count) of `per` doubles each), pushed to every rank
static int shard_push_slab(const ie_shard* sh, int slot, double* (ie_shard::*arr)(int) const, int per, int first,
                           int count, cudaStream_t s) {
    PushDesc d[kMaxRanks];
    const size_t off = (size_t)first * per;
    for (int h = 0; h < sh->G; ++h)
        d[h] = PushDesc{(const char*)((sh->*arr)(sh->g) + off), (char*)((sh->*arr)(h) + off),
                        (long long)count * per * 8, nullptr};
    return shard_push(sh, slot, d, sh->G, s);
}

static int shard_push_chunks(const ie_shard* sh, int slot, double* (ie_shard::*arr)(int) const, int per,
                             cudaStream_t s) {
    return shard_push_slab(sh, slot, arr, per, sh->c0, sh->nchb, s);
}

static inline double* q_band(const ie_shard* sh) { return sh->QW + (size_t)(sh->row0 - sh->rlo) * sh->n; }
static inline double* w_band(const ie_shard* sh) {
    return sh->QW + (size_t)sh->R * sh->n + (size_t)(sh->row0 - sh->rlo) * sh->n;
}

// Setup phases (pcg.py:72-91): 0 = ||f|| partials out, 1 = init + first
// apply, record out, 2 = rho_0, p = z_0.
static int shard_setup_phase(ie_shard* sh, int ph, const double* f_need, double tol, int64_t max_iters,
                             cudaStream_t s, bool timed) {
    const int* stop = &sh->S->stop;
    const int nch = sh->nch, nchb = sh->nchb, c0 = sh->c0, n = sh->n;
    double* r = sh->rfull + sh->b0;
    if (ph == 0) {
        k_clear_stop<<<1, 1, 0, s>>>(sh->S);
        IE_LAUNCHED();
        IE_CUDA(cudaMemcpyAsync(sh->rfull + (size_t)sh->rlo * n, f_need, (size_t)sh->R * n * 8,
                                cudaMemcpyDeviceToDevice, s));
        IE_CUDA(cudaMemcpyAsync(sh->fb, f_need + (size_t)(sh->row0 - sh->rlo) * n, sh->nb * 8,
                                cudaMemcpyDeviceToDevice, s));
        k_dot_partials<<<nchb, kRed, 0, s>>>(sh->fb, sh->fb, (int)sh->nb, 0, sh->xf(sh->g) + c0);
        IE_LAUNCHED();
        return shard_push_chunks(sh, kSlotF, &ie_shard::xf, 1, s);
    }
    if (ph == 1) {
        int rc = shard_wait(sh, kSlotF, (unsigned long long)nch * 8, s);
        if (rc) return rc;
        k_pcg_init<<<1, kRed, 0, s>>>(sh->xf(sh->g), nch, sh->S, tol, max_iters, sh->dh);
        IE_LAUNCHED();
        IE_CUDA(cudaMemsetAsync(sh->PU + sh->nb, 0, sh->nb * 8, s));
        if (timed) IE_CUDA(cudaEventRecord(sh->ev[0], s));
        if (sh->T) {
            if ((rc = precond_apply_band(sh->T, sh->rfull, sh->z, sh->xrz(sh->g) + kRzRec * c0, sh->b0, sh->b1, s,
                                         stop)))
                return rc;
        } else {
            k_identity_apply<<<nchb, kRed, 0, s>>>(r, sh->z, (int)sh->nb, sh->xrz(sh->g) + kRzRec * c0, stop);
            IE_LAUNCHED();
        }
        if (timed) IE_CUDA(cudaEventRecord(sh->ev[1], s));
        return shard_push_chunks(sh, kSlotRz, &ie_shard::xrz, kRzRec, s);
    }
    int rc = shard_wait(sh, kSlotRz, (unsigned long long)nch * kRzRec * 8, s);
    if (rc) return rc;
    k_pcg_setup<<<nchb, kRed, 0, s>>>(sh->xrz(sh->g), nch, sh->S, sh->PU, sh->z, (int)sh->nb, c0, sh->pmax, nullptr);
    IE_LAUNCHED();
    return IE_OK;
}

constexpr int kIterPhases = 5;

// Iteration phases of iteration `itarg` (< 0: graph replay, read from the
// state): 0 = row transforms, FWD out; 1 = column pass, BACK out; 2 = inverse
// rows of the need rows, POST out; 3 = control + r, u updates (+ halo r),
// apply, RZ out; 4 = beta, p, next scales.
static int shard_iter_phase(ie_shard* sh, int ph, int64_t itarg, int do_p, int pending, bool spec, cudaStream_t s,
                            bool timed) {
    const int* stop = &sh->S->stop;
    const int G = sh->G, g = sh->g, n = sh->n, Mc = sh->Mc, nch = sh->nch, nchb = sh->nchb, c0 = sh->c0;
    double* p = sh->PU;
    double* uu = sh->PU + sh->nb;
    double* r = sh->rfull + sh->b0;
    double2* b1 = G == 1 ? sh->buf2(g) : sh->buf1;
    double2* b3 = G == 1 ? sh->buf2(g) : sh->buf3(g);
    const bool two = do_p && pending;
    int rc;
    switch (ph) {
        case 0: {
            const double* X0 = do_p ? p : uu;
            if (G > 1 && sh->fused_transposes) {  // the row spectra go straight into the slab owners' buffers
                PeerStores ps;
                ps.mode = 1;
                ps.npeer = G;
                for (int h = 0; h < G; ++h) {
                    ps.peer[h] = sh->buf2(h) + (size_t)sh->row0 * Mc;
                    ps.ctr[h] = sh->mb(h) + kSlotFwd;
                    ps.line_bytes[h] = (long long)Mc * 16;
                }
                return fft_band_fwd(sh->F, X0, two ? uu : nullptr, sh->nrows, G, b1, two ? sh->S->sc : nullptr, s,
                                    stop, &ps);
            }
            if ((rc = fft_band_fwd(sh->F, X0, two ? uu : nullptr, sh->nrows, G, b1, two ? sh->S->sc : nullptr, s,
                                   stop, nullptr)))
                return rc;
            PushDesc d[kMaxRanks];
            for (int h = 0; h < G; ++h)
                d[h] = PushDesc{(const char*)(b1 + (size_t)h * sh->nrows * Mc),
                                (char*)(sh->buf2(h) + (size_t)sh->row0 * Mc), (long long)sh->nrows * Mc * 16, nullptr};
            return shard_push(sh, kSlotFwd, d, G, s);
        }
        case 1: {
            if ((rc = shard_wait(sh, kSlotFwd, (unsigned long long)n * Mc * 16, s))) return rc;
            if (G > 1 && sh->fused_transposes) {  // the column results go straight into every rank's need rows
                PeerStores ps;
                ps.mode = 2;
                ps.npeer = G;
                ps.band_rows = sh->nrows;
                for (int h = 0; h < G; ++h) {
                    const int Rh = sh->rhi_all[h] - sh->rlo_all[h];
                    ps.peer[h] = sh->buf3(h) + (size_t)g * Rh * Mc;
                    ps.ctr[h] = sh->mb(h) + kSlotBack;
                    ps.line_bytes[h] = (long long)Rh * 16;
                    ps.rlo[h] = sh->rlo_all[h];
                    ps.rhi[h] = sh->rhi_all[h];
                }
                return fft_band_cols(sh->F, sh->buf2(g), g * Mc, Mc, s, stop, &ps);
            }
            if ((rc = fft_band_cols(sh->F, sh->buf2(g), g * Mc, Mc, s, stop, nullptr))) return rc;
            PushDesc d[kMaxRanks];
            for (int h = 0; h < G; ++h) {
                const int Rh = sh->rhi_all[h] - sh->rlo_all[h];
                d[h] = PushDesc{(const char*)(sh->buf2(g) + (size_t)sh->rlo_all[h] * Mc),
                                (char*)(sh->buf3(h) + (size_t)g * Rh * Mc), (long long)Rh * Mc * 16, nullptr};
            }
            return shard_push(sh, kSlotBack, d, G, s);
        }
        case 2: {
            if ((rc = shard_wait(sh, kSlotBack, (unsigned long long)G * sh->R * Mc * 16, s))) return rc;
            double* Y0 = do_p ? sh->QW : sh->QW + (size_t)sh->R * n;
            double* Y1 = two ? sh->QW + (size_t)sh->R * n : nullptr;
            if (sh->line_post) {  // k_post_pass folded into the inverse rows: partials per grid row, as on one GPU
                PcgFuse fz;
                const int64_t shift = (int64_t)(sh->row0 - sh->rlo) * n;  // need-row index -> band index
                fz.p = p - shift;
                fz.f = sh->fb - shift;
                fz.part = sh->xpost(g);
                fz.line0 = sh->rlo;
                fz.post_lo = sh->row0 - sh->rlo;
                fz.post_hi = sh->row0 - sh->rlo + sh->nrows;
                fz.q_col = do_p ? 0 : -1;
                fz.w_col = pending ? (do_p ? 1 : 0) : -1;
                if (G > 1 && sh->fused_transposes) {  // the partials go straight to every rank (own one included)
                    fz.npeer = G;
                    for (int h = 0; h < G; ++h) {
                        fz.part_peer[h] = sh->xpost(h);
                        fz.part_ctr[h] = sh->mb(h) + kSlotPost;
                    }
                    return fft_band_inv(sh->F, b3, sh->R, G, Y0, Y1, two ? sh->S->sc : nullptr, s, stop, &fz);
                }
                if ((rc = fft_band_inv(sh->F, b3, sh->R, G, Y0, Y1, two ? sh->S->sc : nullptr, s, stop, &fz)))
                    return rc;
                return shard_push_slab(sh, kSlotPost, &ie_shard::xpost, 2, sh->row0, sh->nrows, s);
            }
            if ((rc = fft_band_inv(sh->F, b3, sh->R, G, Y0, Y1, two ? sh->S->sc : nullptr, s, stop, nullptr)))
                return rc;
            IE_CUDA(launch_k(k_post_pass, dim3(nchb), dim3(kRed), 0, s, (const double*)p, (const double*)q_band(sh),
                             (const double*)sh->fb, (const double*)w_band(sh), (int)sh->nb, do_p, pending,
                             sh->xpost(g) + 2 * c0, stop));
            IE_LAUNCHED();
            return shard_push_chunks(sh, kSlotPost, &ie_shard::xpost, 2, s);
        }
        case 3: {
            const int npost = sh->line_post ? n : nch;
            if ((rc = shard_wait(sh, kSlotPost, (unsigned long long)npost * 16, s))) return rc;
            const HaloSeg hs{(sh->rlo - sh->row0) * n, (sh->row0 - sh->rlo) * n, (int)sh->nb,
                             (sh->rhi - sh->row0 - sh->nrows) * n};
            const int nh = (hs.len0 + kChunk - 1) / kChunk + (hs.len1 + kChunk - 1) / kChunk;
            IE_CUDA(launch_k(k_iter_a<true, true>, dim3(nchb + nh), dim3(kRed), 0, s, (const double*)sh->xpost(g),
                             npost, do_p, pending, (long long)itarg, sh->S, sh->dh, uu, r, (const double*)p,
                             (const double*)q_band(sh), (int)sh->nb, c0, nchb, sh->xrz(g), (const double*)sh->pmax,
                             hs, 0));
            IE_LAUNCHED();
            if (!spec) return IE_OK;
            if (timed) IE_CUDA(cudaEventRecord(sh->ev[2], s));
            const bool fold_rz = G > 1 && sh->fused_transposes && sh->T;  // the scatter pushes its records
            if (sh->T) {
                PeerRec pr;
                if (fold_rz) {
                    pr.n = G;
                    for (int h = 0; h < G; ++h) {
                        pr.dst[h] = sh->xrz(h) + kRzRec * c0;
                        pr.ctr[h] = sh->mb(h) + kSlotRz;
                    }
                }
                precond_set_peer_record(&pr);
                rc = precond_apply_band(sh->T, sh->rfull, sh->z, sh->xrz(g) + kRzRec * c0, sh->b0, sh->b1, s, stop);
                precond_set_peer_record(nullptr);
                if (rc) return rc;
            } else {
                k_identity_apply<<<nchb, kRed, 0, s>>>(r, sh->z, (int)sh->nb, sh->xrz(g) + kRzRec * c0, stop);
                IE_LAUNCHED();
            }
            if (timed) IE_CUDA(cudaEventRecord(sh->ev[3], s));
            if (fold_rz) return IE_OK;
            return shard_push_chunks(sh, kSlotRz, &ie_shard::xrz, kRzRec, s);
        }
        default: {
            if (!spec) return IE_OK;
            if ((rc = shard_wait(sh, kSlotRz, (unsigned long long)nch * kRzRec * 8, s))) return rc;
            IE_CUDA(launch_k(k_iter_b, dim3(nchb), dim3(kRed), 0, s, (const double*)sh->xrz(g), nch,
                             (long long)itarg, sh->S, p, (const double*)sh->z, (int)sh->nb, sh->pmax));
            IE_LAUNCHED();
            return IE_OK;
        }
    }
}

// PCG over the shards of this process (1: one rank per process; G: all ranks
// on one device), phase-major.
static int shard_solve(ie_shard* const* shs, int nloc, const double* const* f_need, double* const* u_band, double tol,
                       int64_t max_iters, double* hist, int64_t* n_it, int32_t* flags, double* times,
                       int64_t* fail_iter, double* fail_value, cudaStream_t st) {
    ie_shard* s0 = shs[0];
    const auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < nloc; ++k)
        if (!shs[k]->connected || shs[k]->broken) {
            set_error("ie_pcg_sharded: shard not connected (ie_shard_connect) or broken by an earlier failure");
            return IE_ERR_ARG;
        }
    int64_t cap = 1024;
    while (cap < max_iters + 1) cap *= 2;
    for (int k = 0; k < nloc; ++k) {
        ie_shard* sh = shs[k];
        if (sh->cap < cap) {
            if (sh->dh) cudaFree(sh->dh);
            IE_CUDA(cudaMalloc(&sh->dh, (size_t)cap * 8));
            sh->cap = cap;
            if (s0->gexec) {  // the captured iteration writes the old history buffer
                cudaGraphExecDestroy(s0->gexec);
                s0->gexec = nullptr;
            }
        }
    }
    int rc;
    auto fail = [&](int code) {
        for (int k = 0; k < nloc; ++k) shs[k]->broken = true;
        return code;
    };
    for (int ph = 0; ph < 3; ++ph)
        for (int k = 0; k < nloc; ++k)
            if ((rc = shard_setup_phase(shs[k], ph, f_need[k], tol, max_iters, st, k == 0))) return fail(rc);
    auto enqueue = [&](int64_t itarg, int do_p, int pending, bool spec, cudaStream_t s, bool timed) -> int {
        for (int ph = 0; ph < kIterPhases; ++ph)
            for (int k = 0; k < nloc; ++k) {
                int r2 = shard_iter_phase(shs[k], ph, itarg, do_p, pending, spec, s, timed && k == 0);
                if (r2) return r2;
            }
        return IE_OK;
    };
    const bool use_graph = max_iters >= 3 && !getenv("IEDD_B200_NO_GRAPH");
    if (use_graph && (!s0->gexec || s0->gmode != nloc)) {
        if (s0->gexec) cudaGraphExecDestroy(s0->gexec);
        s0->gexec = nullptr;
        if (!s0->cap_s) IE_CUDA(cudaStreamCreateWithFlags(&s0->cap_s, cudaStreamNonBlocking));
        for (int k = 0; k < nloc; ++k)
            if (shs[k]->T && (rc = precond_prepare_stream(shs[k]->T, s0->cap_s))) return fail(rc);
        cudaEvent_t ev;
        IE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        IE_CUDA(cudaEventRecord(ev, st));
        IE_CUDA(cudaStreamWaitEvent(s0->cap_s, ev, 0));
        cudaEventDestroy(ev);
        cudaGraph_t gr;
        IE_CUDA(cudaStreamBeginCapture(s0->cap_s, cudaStreamCaptureModeThreadLocal));
        int r2 = enqueue(-1, 1, 1, true, s0->cap_s, false);  // k_iter_b advances it_dev
        cudaError_t ce = cudaStreamEndCapture(s0->cap_s, &gr);
        if (r2) return fail(r2);
        IE_CUDA(ce);
        size_t nn = 0;
        cudaGraphGetNodes(gr, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) cudaGraphGetNodes(gr, nodes.data(), &nn);
        s0->gnodes = 0;
        for (auto nd : nodes) {
            cudaGraphNodeType t;
            if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++s0->gnodes;
        }
        ce = cudaGraphInstantiate(&s0->gexec, gr, 0);
        cudaGraphDestroy(gr);
        IE_CUDA(ce);
        s0->gmode = nloc;
    }
    static const int64_t kBatch = [] {
        const char* e = getenv("IEDD_B200_PCG_BATCH");
        const long long v = e ? atoll(e) : 4;
        return (int64_t)std::max(1LL, std::min(v, 1024LL));
    }();
    for (int64_t it = 1; it <= max_iters + 1; ++it) {
        const int do_p = it <= max_iters;
        const int pending = it >= 2;
        const bool spec = do_p && it < max_iters;
        if (use_graph && pending && spec) {
            if (it == 2)
                for (int k = 0; k < nloc; ++k) {
                    k_set_it<<<1, 1, 0, st>>>(shs[k]->S, 2);
                    IE_LAUNCHED();
                }
            IE_CUDA(cudaGraphLaunch(s0->gexec, st));
            g_launches.fetch_add(s0->gnodes, std::memory_order_relaxed);
        } else if ((rc = enqueue(it, do_p, pending, spec, st, it == 1))) {
            return fail(rc);
        }
        if (it % kBatch == 0 || it == max_iters + 1) {
            IE_CUDA(cudaMemcpyAsync(s0->host, s0->S, sizeof(PcgState), cudaMemcpyDeviceToHost, st));
            IE_CUDA(cudaStreamSynchronize(st));
            if (s0->host->stop) break;
        }
    }
    IE_CUDA(cudaMemcpyAsync(s0->host, s0->S, sizeof(PcgState), cudaMemcpyDeviceToHost, st));
    IE_CUDA(cudaStreamSynchronize(st));
    const PcgState H = *s0->host;
    if (H.status == 6) {
        fail(0);
        set_error("ie_pcg_sharded: peer exchange timed out (a rank stopped sending)");
        return IE_ERR_CUDA;
    }
    flags[0] = H.status == 1;
    flags[1] = H.status == 2;
    *n_it = H.n_it;
    if (H.status == 4 || H.status == 5) {
        if (fail_iter) *fail_iter = H.fail_iter;
        if (fail_value) *fail_value = H.fail_value;
    }
    IE_CUDA(cudaMemcpyAsync(hist, s0->dh, (size_t)(H.n_it + 1) * 8, cudaMemcpyDeviceToHost, st));
    for (int k = 0; k < nloc; ++k)
        IE_CUDA(cudaMemcpyAsync(u_band[k], shs[k]->PU + shs[k]->nb, shs[k]->nb * 8, cudaMemcpyDeviceToDevice, st));
    IE_CUDA(cudaStreamSynchronize(st));
    times[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    // t_s: mean device time of rank 0's event-timed applies (the initial one and iteration 1's)
    double tp = 0.0;
    int np = 0;
    for (int e = 0; e < 2; ++e) {
        if (e == 1 && (H.n_it < 2 || max_iters < 2)) break;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, s0->ev[2 * e], s0->ev[2 * e + 1]) == cudaSuccess) tp += ms * 1e-3, ++np;
    }
    cudaGetLastError();
    times[1] = np ? tp / np : 0.0;
    if (H.nf == 0.0) times[0] = times[1] = 0.0;
    if (H.status == 4) return IE_ERR_BREAKDOWN;
    if (H.status == 5) return IE_ERR_NONFINITE;
    return IE_OK;
}
}  // namespace ie

extern "C" int ie_shard_create(const ie_matvec* A, const ie_precond* T_local, int32_t nranks, int32_t rank,
                               const int64_t* h_bounds, const int64_t* h_need, ie_shard** out) {
    using namespace ie;
    if (!A || !h_bounds || !out || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) {
        set_error("ie_shard_create: bad arguments");
        return IE_ERR_ARG;
    }
    const ie_fft* F = matvec_fft(A);
    const int G = nranks, g = rank;
    const int N = matvec_N(A), n = matvec_n(A), M = F ? fft_M(F) : 0;
    const int64_t nb = h_bounds[1] - h_bounds[0];
    bool ok = F && matvec_dim(A) == 2 && M % G == 0 && (((M / G) & (M / G - 1)) == 0) && h_bounds[0] == 0 &&
              h_bounds[G] == N && nb > 0 && nb % kChunk == 0;
    for (int h = 0; h < G && ok; ++h) ok = h_bounds[h + 1] - h_bounds[h] == nb && h_bounds[h] % n == 0;
    if (!ok) {
        set_error("ie_shard_create: needs the 2D FFT operator, G | M (the circulant size; power-of-two "
                  "slabs) and equal, chunk-aligned bands of whole grid rows");
        return IE_ERR_ARG;
    }
    ie_shard* sh = new ie_shard();
    std::unique_ptr<ie_shard> guard(sh);
    sh->G = G;
    sh->g = g;
    sh->A = A;
    sh->T = T_local;
    sh->F = F;
    sh->n = n;
    sh->M = M;
    sh->Mc = M / G;
    sh->N = N;
    for (int h = 0; h < G; ++h) {
        const int r0 = (int)(h_bounds[h] / n), r1 = (int)(h_bounds[h + 1] / n);
        int lo = r0, hi = r1;
        if (h_need && T_local) {  // need rows: the point range the rank's subdomains read, in whole rows
            lo = std::min(lo, (int)(h_need[2 * h] / n));
            hi = std::max(hi, (int)((h_need[2 * h + 1] + n - 1) / n));
        }
        sh->row0_all.push_back(r0);
        sh->nrows_all.push_back(r1 - r0);
        sh->rlo_all.push_back(std::max(0, lo));
        sh->rhi_all.push_back(std::min(n, hi));
        sh->Rmax = std::max(sh->Rmax, sh->rhi_all[h] - sh->rlo_all[h]);
    }
    sh->b0 = h_bounds[g];
    sh->b1 = h_bounds[g + 1];
    sh->nb = nb;
    sh->row0 = sh->row0_all[g];
    sh->nrows = sh->nrows_all[g];
    sh->rlo = sh->rlo_all[g];
    sh->rhi = sh->rhi_all[g];
    sh->R = sh->rhi - sh->rlo;
    sh->nchb = (int)(nb / kChunk);
    sh->nch = sh->nchb * G;
    sh->c0 = (int)(sh->b0 / kChunk);
    size_t o = align256(kNumSlots * sizeof(unsigned long long));
    sh->off_xf = o;
    o = align256(o + (size_t)sh->nch * 8);
    sh->line_post = !getenv("IEDD_B200_NO_FUSE") && matvec_fused_lines(A) > 0;
    sh->fused_transposes = !getenv("IEDD_B200_PUSH_TRANSPOSES");
    sh->off_xpost = o;
    o = align256(o + (size_t)std::max(sh->nch, n) * 16);
    sh->off_xrz = o;
    o = align256(o + (size_t)sh->nch * kRzRec * 8);
    sh->off_buf2 = o;
    o = align256(o + (size_t)n * sh->Mc * 16);
    sh->off_buf3 = o;
    if (G > 1) o = align256(o + (size_t)G * sh->Rmax * sh->Mc * 16);
    sh->heap_bytes = o;
    IE_CUDA(cudaMalloc(&sh->heap, sh->heap_bytes));
    IE_CUDA(cudaMemset(sh->heap, 0, kNumSlots * sizeof(unsigned long long)));
    IE_CUDA(cudaMalloc(&sh->PU, 2 * nb * 8));
    IE_CUDA(cudaMalloc(&sh->QW, 2 * (size_t)sh->R * n * 8));
    IE_CUDA(cudaMalloc(&sh->rfull, (size_t)N * 8));
    IE_CUDA(cudaMalloc(&sh->z, nb * 8));
    IE_CUDA(cudaMalloc(&sh->fb, nb * 8));
    IE_CUDA(cudaMalloc(&sh->pmax, (size_t)sh->nchb * 8));
    if (G > 1) IE_CUDA(cudaMalloc(&sh->buf1, (size_t)sh->nrows * M * 16));
    IE_CUDA(cudaMalloc(&sh->tgt, kNumSlots * sizeof(unsigned long long)));
    IE_CUDA(cudaMemset(sh->tgt, 0, kNumSlots * sizeof(unsigned long long)));
    IE_CUDA(cudaMalloc(&sh->S, sizeof(PcgState)));
    IE_CUDA(cudaMemset(sh->S, 0, sizeof(PcgState)));
    IE_CUDA(cudaMallocHost(&sh->host, sizeof(PcgState)));
    for (auto& e : sh->ev) IE_CUDA(cudaEventCreate(&e));
    IE_CUDA(cudaDeviceSynchronize());
    sh->peer.assign(G, nullptr);
    sh->opened.assign(G, false);
    sh->peer[g] = sh->heap;
    sh->connected = G == 1;
    *out = guard.release();
    return IE_OK;
}

extern "C" void ie_shard_destroy(ie_shard* s) { delete s; }

extern "C" int64_t ie_shard_handle_bytes(void) { return (int64_t)sizeof(cudaIpcMemHandle_t); }

extern "C" int ie_shard_need_rows(const ie_shard* s, int64_t* out2) {
    if (!s || !out2) return IE_ERR_ARG;
    out2[0] = (int64_t)s->rlo * s->n;
    out2[1] = (int64_t)s->rhi * s->n;
    return IE_OK;
}

extern "C" int ie_shard_export(const ie_shard* s, void* h_out) {
    if (!s || !h_out) return IE_ERR_ARG;
    cudaIpcMemHandle_t h;
    IE_CUDA(cudaIpcGetMemHandle(&h, s->heap));
    memcpy(h_out, &h, sizeof(h));
    return IE_OK;
}

extern "C" int ie_shard_connect(ie_shard* s, const void* h_handles) {
    if (!s || !h_handles) return IE_ERR_ARG;
    const char* base = (const char*)h_handles;
    for (int h = 0; h < s->G; ++h) {
        if (h == s->g) continue;
        cudaIpcMemHandle_t hd;
        memcpy(&hd, base + (size_t)h * sizeof(hd), sizeof(hd));
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            ie::set_error(std::string("ie_shard_connect: cudaIpcOpenMemHandle(rank ") + std::to_string(h) +
                          "): " + cudaGetErrorString(e) + " (no NVLink/P2P path: use the torch.distributed driver)");
            return IE_ERR_CUDA;
        }
        s->peer[h] = (char*)p;
        s->opened[h] = true;
    }
    s->connected = true;
    return IE_OK;
}

extern "C" int ie_shard_connect_local(ie_shard** shards, int32_t nranks) {
    if (!shards || nranks < 1) return IE_ERR_ARG;
    for (int k = 0; k < nranks; ++k)
        if (!shards[k] || shards[k]->G != nranks || shards[k]->g != k) {
            ie::set_error("ie_shard_connect_local: shards must be ranks 0..G-1 of one G-rank plan");
            return IE_ERR_ARG;
        }
    for (int k = 0; k < nranks; ++k) {
        for (int h = 0; h < nranks; ++h) shards[k]->peer[h] = shards[h]->heap;
        shards[k]->connected = true;
    }
    return IE_OK;
}

extern "C" int ie_pcg_sharded_f64(ie_shard* s, const double* d_f_need, double* d_u_band, double tol,
                                  int64_t max_iters, double* hist, int64_t* n_it, int32_t* flags, double* times,
                                  int64_t* fail_iter, double* fail_value, void* stream) {
    if (!s || !d_f_need || !d_u_band || !hist || !n_it || !flags || !times || max_iters < 0 ||
        !(tol > 0.0 && tol < 1.0)) {
        ie::set_error("ie_pcg_sharded_f64: bad arguments");
        return IE_ERR_ARG;
    }
    ie_shard* one[1] = {s};
    const double* f1[1] = {d_f_need};
    double* u1[1] = {d_u_band};
    return ie::shard_solve(one, 1, f1, u1, tol, max_iters, hist, n_it, flags, times, fail_iter, fail_value,
                           (cudaStream_t)stream);
}

extern "C" int ie_pcg_sharded_local_f64(ie_shard** shards, int32_t nranks, const double* const* d_f_need,
                                        double* const* d_u_band, double tol, int64_t max_iters, double* hist,
                                        int64_t* n_it, int32_t* flags, double* times, int64_t* fail_iter,
                                        double* fail_value, void* stream) {
    if (!shards || nranks < 1 || !d_f_need || !d_u_band || !hist || !n_it || !flags || !times || max_iters < 0 ||
        !(tol > 0.0 && tol < 1.0)) {
        ie::set_error("ie_pcg_sharded_local_f64: bad arguments");
        return IE_ERR_ARG;
    }
    for (int k = 0; k < nranks; ++k)
        if (!shards[k] || shards[k]->G != nranks || shards[k]->g != k || shards[k]->peer[0] != shards[0]->heap) {
            ie::set_error("ie_pcg_sharded_local_f64: shards must be ranks 0..G-1 joined by ie_shard_connect_local");
            return IE_ERR_ARG;
        }
    return ie::shard_solve(shards, nranks, d_f_need, d_u_band, tol, max_iters, hist, n_it, flags, times, fail_iter,
                           fail_value, (cudaStream_t)stream);
}

// Per-line partials with the association of the post pass folded into the
// FFT's last line transform (fft.cu kInvCRPost): line l of n points, thread
// j < TPL = M / 8 chains points j + TPL m (m < 4) by FMA, then a halving tree
// over the TPL threads.  mode 0: x.y, mode 1: |x - y|^2.  The torch.distributed
// driver (distributed.py) uses it so its dot products are bitwise those of
// ie_pcg_f64 on one GPU.
namespace ie {
__global__ void k_line_partials(const double* x, const double* y, int n, int tpl, int mode, double* part) {
    extern __shared__ double sl[];
    const int j = threadIdx.x;
    const int64_t base = (int64_t)blockIdx.x * n;
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int l = j + tpl * m;
        if (l < n) {
            if (mode == 0) {
                acc = fma(x[base + l], y[base + l], acc);
            } else {
                const double d = x[base + l] - y[base + l];
                acc = fma(d, d, acc);
            }
        }
    }
    sl[j] = acc;
    __syncthreads();
    for (int off = tpl / 2; off > 0; off >>= 1) {
        if (j < off) sl[j] += sl[j + off];
        __syncthreads();
    }
    if (j == 0) part[blockIdx.x] = sl[0];
}
}  // namespace ie

extern "C" int ie_line_partials_f64(const double* x, const double* y, int64_t nlines, int32_t n, int32_t M,
                                    int32_t mode, double* part, void* stream) {
    const int tpl = M / 8;
    if (!x || !y || !part || nlines < 0 || n < 1 || M < 64 || (M & (M - 1)) || n > M / 2 || tpl > 1024 ||
        (mode != 0 && mode != 1)) {
        ie::set_error("ie_line_partials_f64: bad arguments");
        return IE_ERR_ARG;
    }
    if (nlines == 0) return IE_OK;
    ie::k_line_partials<<<(unsigned)nlines, tpl, tpl * sizeof(double), (cudaStream_t)stream>>>(x, y, n, tpl, mode,
                                                                                               part);
    IE_LAUNCHED();
    return IE_OK;
}
