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
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

#include "common.cuh"
#include "pcg_state.cuh"

struct ie_matvec;
struct ie_precond;

namespace ie {

int matvec_launch(const ie_matvec* m, const double* X, int64_t ldx, int nrhs, double* Y, int64_t ldy,
                  int64_t row_begin, int64_t row_end, cudaStream_t st, const int* stop,
                  const double* amax = nullptr);
int precond_prepare_stream(const ie_precond* p, cudaStream_t st);
int matvec_prepare_stream(const ie_matvec* m, cudaStream_t st);
int precond_apply(const ie_precond* p, const double* r, double* z, double* partials, cudaStream_t st,
                  const int* stop);
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


__global__ void k_set_it(PcgState* s, long long it) { s->it_dev = it; }

__global__ void k_pcg_init(const double* part, int nch, PcgState* s, double tol, long long max_iters,
                           double* hist) {
    // (rho_0 is set by k_pcg_rho0 after the first apply)
    __shared__ double sh[kRed];
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

// After the A-pass of iteration `it`: residual / stagnation check of
// iteration it-1 (pcg.py:107-119), breakdown test of iteration it
// (pcg.py:99-103), alpha, then u += alpha p, r -= alpha q and max|u| per chunk.
// Every CTA reduces the same partials in the same order and takes the same
// decision; CTA 0 records it in the state.  Every load that does not depend
// on the reduction (state scalars, the history entry of the stagnation test,
// this thread's partials and its p, q, r chunk values) is issued before it, so
// the serial prologue costs about one memory round trip.
template <bool WITH_U>
__global__ void __launch_bounds__(kRed, 4) k_iter_a(const double* part_pq, const double* part_res, int nch, int do_p,
                                                 int pending, long long it, PcgState* s, double* hist, double* u,
                                                 double* r, const double* p, const double* q, int N, double* amax) {
    __shared__ double sh[kRed];
    __shared__ int decided;
    pdl_wait();
    const int stopv = s->stop;
    if (it < 0) it = s->it_dev;
    const double rho_prev = s->rho[(it - 1) & 1], nf = s->nf, tol = s->tol;
    const long long k = it - 1;
    const double h30 = (pending && k >= 30 && threadIdx.x == 0) ? hist[k - 30] : 0.0;
    const int base = blockIdx.x * kChunk;
    double pv[kChunk / kRed], qv[kChunk / kRed], rv[kChunk / kRed];
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        pv[e] = (WITH_U && do_p && i < N) ? p[i] : 0.0;  // p only for the in-kernel u update
        qv[e] = (do_p && i < N) ? q[i] : 0.0;
        rv[e] = (!WITH_U && do_p && i < N) ? r[i] : 0.0;  // hoisted where registers allow
    }
    double lp = 0.0, lr = 0.0;
    for (int c = threadIdx.x; c < nch; c += kRed) {
        if (do_p) lp += part_pq[c];
        if (pending) lr += part_res[c];
    }
    if (stopv) return;
    double denom = 0.0, res2 = 0.0;
    if (do_p) denom = block_tree(lp, sh);
    __syncthreads();
    if (pending) res2 = block_tree(lr, sh);
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
            if (pending && status != 5) hist[k] = rel;
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
    const double al = rho_prev / denom;
    if (!WITH_U) {  // u += alpha p runs concurrently in k_update_u (graph side branch)
#pragma unroll
        for (int e = 0; e < kChunk / kRed; ++e) {
            const int i = base + e * kRed + threadIdx.x;
            if (i < N) r[i] = __dsub_rn(rv[e], __dmul_rn(al, qv[e]));
        }
        return;
    }
    double m = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < N) {
            const double un = __dadd_rn(u[i], __dmul_rn(al, pv[e]));
            u[i] = un;
            r[i] = __dsub_rn(r[i], __dmul_rn(al, qv[e]));
            m = fmax(m, fabs(un));
        }
    }
    m = chunk_absmax(m, sh);
    if (threadIdx.x == 0) amax[2 * blockIdx.x + 1] = m;
}

// k_iter_a's u half: u += alpha p and max|u| per chunk, with the alpha CTA 0 of
// k_iter_a stored (the same quotient every CTA computes).  Off the critical
// path: it runs beside the preconditioner apply and joins before k_iter_b
// rewrites p (the next A-pass is u's only consumer).
__global__ void __launch_bounds__(kRed) k_update_u(const PcgState* s, double* u, const double* p, int N,
                                                   double* amax) {
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
    if (threadIdx.x == 0) amax[2 * blockIdx.x + 1] = m;
}

// After the apply: rho_it = r.z, beta = rho_it / rho_{it-1}, p = z + beta p,
// max|p| per chunk.
// After the apply: rho_it = r.z, beta = rho_it / rho_{it-1}, p = z + beta p,
// max|p| per chunk; the independent loads (state, partials, this thread's z
// and p chunk values) are issued ahead of the reduction.  In graph replay the
// last CTA advances the iteration counter.
__global__ void __launch_bounds__(kRed) k_iter_b(const double* part_rz, int nch, long long it, PcgState* s,
                                                 double* p, const double* z, int N, double* amax) {
    __shared__ double sh[kRed];
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
        zv[e] = i < N ? z[i] : 0.0;
        pv[e] = i < N ? p[i] : 0.0;
    }
    double loc = 0.0;
    for (int c = threadIdx.x; c < nch; c += kRed) loc += part_rz[c];
    if (stopv) return;
    const double rz = block_tree(loc, sh);
    const double beta = rz / rho_prev;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s->beta = beta;
        s->rho[it & 1] = rz;
    }
    double m = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int i = base + e * kRed + threadIdx.x;
        if (i < N) {
            const double pn = __dadd_rn(zv[e], __dmul_rn(beta, pv[e]));
            p[i] = pn;
            m = fmax(m, fabs(pn));
        }
    }
    __syncthreads();
    m = chunk_absmax(m, sh);
    if (threadIdx.x == 0) amax[2 * blockIdx.x] = m;
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

__global__ void k_pcg_rho0(const double* part_rz, int nch, PcgState* s) {
    __shared__ double sh[kRed];
    if (s->stop) return;
    const double rz = reduce_partials(part_rz, nch, sh);
    if (threadIdx.x == 0) s->rho[0] = rz;
}

// Chunk partials of p.q (A-pass denominator) and |f - w|^2 (true residual of
// the previous iterate); the loads are issued before the stop flag is tested.
__global__ void k_post_pass(const double* p, const double* q, const double* f, const double* w, int N, int do_p,
                            int pending, double* part_pq, double* part_res, const int* stop) {
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
        if (threadIdx.x == 0) part_pq[blockIdx.x] = t;
        __syncthreads();
    }
    if (pending) {
        const double t = block_tree(b, sh);
        if (threadIdx.x == 0) part_res[blockIdx.x] = t;
    }
}

__global__ void k_copy_if_running(double* dst, const double* src, int N, const int* stop) {
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
    double* amax = nullptr;  // per-chunk max|p|, max|u| (2-RHS FFT column scaling)
    double* fcopy = nullptr; // the right-hand side (graph-stable address)
    cudaStream_t cap_stream = nullptr;
    cudaStream_t side_stream = nullptr;  // graph side branch (u update)
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    cudaGraphExec_t gexec = nullptr;
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
        cudaFree(amax);
        cudaFree(fcopy);
        if (gexec) cudaGraphExecDestroy(gexec);
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
    if (e == cudaSuccess) e = cudaMalloc(&w->part, 3 * (size_t)nch * 8);
    if (e == cudaSuccess) e = cudaMalloc(&w->hist, (size_t)cap * 8);
    if (e == cudaSuccess) e = cudaMalloc(&w->amax, 2 * (size_t)nch * 8);
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

extern "C" int ie_pcg_f64(const ie_matvec* A, const ie_precond* T, const double* f, double* u, double tol,
                          int64_t max_iters, double* hist, int64_t* n_it, int32_t* flags, double* times,
                          int64_t* fail_iter, double* fail_value, void* stream) {
    if (!A || !f || !u || !hist || !n_it || !flags || !times || max_iters < 0 || !(tol > 0.0 && tol < 1.0)) {
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
    const int64_t kBatch = 4;
    if ((rc = ensure_events(W, 2 * (size_t)(std::min<int64_t>(cap, 4096) + 2)))) return rc;
    double* p = W->PU;
    double* uu = W->PU + N;
    double* q = W->QW;
    double* w = W->QW + N;
    double* part_pq = W->part;
    double* part_res = W->part + nch;
    double* part_rz = W->part + 2 * nch;
    const int* stop = &W->st->stop;
    auto apply = [&](const double* rin, double* zout, int64_t evi) -> int {
        const bool timed = 2 * evi + 1 < (int64_t)W->ev.size();
        if (timed) IE_CUDA(cudaEventRecord(W->ev[2 * evi], st));
        if (T) {
            int r2 = precond_apply(T, rin, zout, part_rz, st, stop);
            if (r2) return r2;
        } else {
            k_copy_if_running<<<g1(N), 256, 0, st>>>(zout, rin, N, stop);
            IE_LAUNCHED();
            k_dot_partials<<<nch, kRed, 0, st>>>(rin, zout, N, 0, part_rz);
            IE_LAUNCHED();
        }
        if (timed) IE_CUDA(cudaEventRecord(W->ev[2 * evi + 1], st));
        return IE_OK;
    };
    // the right-hand side at a stable address (captured graphs reference it)
    IE_CUDA(cudaMemcpyAsync(W->fcopy, f, (size_t)N * 8, cudaMemcpyDeviceToDevice, st));
    f = W->fcopy;
    // ||f||, state init (pcg.py:72-91)
    k_dot_partials<<<nch, kRed, 0, st>>>(f, f, N, 0, part_pq);
    IE_LAUNCHED();
    k_pcg_init<<<1, kRed, 0, st>>>(part_pq, nch, W->st, tol, max_iters, W->hist);
    IE_LAUNCHED();
    IE_CUDA(cudaMemsetAsync(uu, 0, (size_t)N * 8, st));
    IE_CUDA(cudaMemcpyAsync(W->r, f, (size_t)N * 8, cudaMemcpyDeviceToDevice, st));
    if ((rc = apply(W->r, W->z, 0))) return rc;
    IE_CUDA(cudaMemcpyAsync(p, W->z, (size_t)N * 8, cudaMemcpyDeviceToDevice, st));
    k_pcg_rho0<<<1, kRed, 0, st>>>(part_rz, nch, W->st);
    IE_LAUNCHED();
    // iterations: `it` = the iteration whose A-pass is enqueued; the pass also
    // carries u_{it-1} for the deferred true-residual check of iteration it-1.
    // Steady-state iterations (2 <= it < max_iters) replay one captured CUDA
    // graph that reads `it` from the device state.
    static const bool no_fork = getenv("IEDD_B200_NO_FORK") != nullptr;  // u update in k_iter_a (comparison)
    auto enqueue_iter = [&](int64_t itarg, int do_p, int pending, bool spec, cudaStream_t s2, bool timed_apply,
                            int64_t evi) -> int {
        int r2;
        if (do_p && pending) {
            r2 = matvec_launch(A, W->PU, N, 2, W->QW, N, 0, N, s2, stop, W->amax);
        } else if (do_p) {
            r2 = matvec_launch(A, p, N, 1, q, N, 0, N, s2, stop);
        } else {
            r2 = matvec_launch(A, uu, N, 1, w, N, 0, N, s2, stop);
        }
        if (r2) return r2;
        IE_CUDA(launch_k(k_post_pass, dim3(nch), dim3(kRed), 0, s2, (const double*)p, (const double*)q, f,
                         (const double*)w, N, do_p, pending, part_pq, part_res, stop));
        IE_LAUNCHED();
        // in the captured iteration u += alpha p forks onto a side branch beside the apply
        const bool fork_u = itarg < 0 && do_p && spec && !no_fork;
        IE_CUDA(launch_k(fork_u ? k_iter_a<false> : k_iter_a<true>, dim3(nch), dim3(kRed), 0, s2, (const double*)part_pq, (const double*)part_res, nch,
                         do_p, pending, (long long)itarg, W->st, W->hist, fork_u ? nullptr : uu, W->r,
                         (const double*)p, (const double*)q, N, W->amax));
        IE_LAUNCHED();
        if (fork_u) {
            IE_CUDA(cudaEventRecord(W->fork_ev, s2));
            IE_CUDA(cudaStreamWaitEvent(W->side_stream, W->fork_ev, 0));
            k_update_u<<<nch, kRed, 0, W->side_stream>>>(W->st, uu, p, N, W->amax);
            IE_LAUNCHED();
            IE_CUDA(cudaEventRecord(W->join_ev, W->side_stream));
        }
        if (spec) {  // speculative: z_it is discarded if iteration it is the last
            if (timed_apply) {
                if ((r2 = apply(W->r, W->z, evi))) return r2;
            } else if (T) {
                if ((r2 = precond_apply(T, W->r, W->z, part_rz, s2, stop))) return r2;
            } else {
                k_copy_if_running<<<g1(N), 256, 0, s2>>>(W->z, W->r, N, stop);
                IE_LAUNCHED();
                k_dot_partials<<<nch, kRed, 0, s2>>>(W->r, W->z, N, 0, part_rz);
                IE_LAUNCHED();
            }
            // k_iter_b rewrites p, which the side branch reads: join first
            if (fork_u) IE_CUDA(cudaStreamWaitEvent(s2, W->join_ev, 0));
            IE_CUDA(launch_k(k_iter_b, dim3(nch), dim3(kRed), 0, s2, (const double*)part_rz, nch, (long long)itarg,
                             W->st, p, (const double*)W->z, N, W->amax));
            IE_LAUNCHED();
        }
        return IE_OK;
    };
    const bool use_graph = max_iters >= 3 && !getenv("IEDD_B200_NO_GRAPH");
    if (use_graph) {
        const uint64_t ka = matvec_uid(A), kt = T ? precond_uid(T) : 0;
        if (!W->gexec || W->key_a != ka || W->key_t != kt) {
            if (W->gexec) {
                cudaGraphExecDestroy(W->gexec);
                W->gexec = nullptr;
            }
            cudaGraph_t g;
            if (T && (rc = precond_prepare_stream(T, W->cap_stream))) return rc;
            if ((rc = matvec_prepare_stream(A, W->cap_stream))) return rc;
            IE_CUDA(cudaStreamBeginCapture(W->cap_stream, cudaStreamCaptureModeThreadLocal));
            int r2 = enqueue_iter(-1, 1, 1, true, W->cap_stream, false, 0);  // k_iter_b advances it_dev
            cudaError_t ce = cudaStreamEndCapture(W->cap_stream, &g);
            if (r2) return r2;
            IE_CUDA(ce);
            size_t nn = 0;
            cudaGraphGetNodes(g, nullptr, &nn);
            std::vector<cudaGraphNode_t> nodes(nn);
            if (nn) cudaGraphGetNodes(g, nodes.data(), &nn);
            W->gnodes = 0;
            for (auto nd : nodes) {
                cudaGraphNodeType t;
                if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++W->gnodes;
            }
            ce = cudaGraphInstantiate(&W->gexec, g, 0);
            cudaGraphDestroy(g);
            IE_CUDA(ce);
            W->key_a = ka;
            W->key_t = kt;
        }
    }
    int64_t it = 1, nbatch = 0;
    for (; it <= max_iters + 1; ++it) {
        const int do_p = it <= max_iters;
        const int pending = it >= 2;
        const bool spec = do_p && it < max_iters;
        if (use_graph && pending && spec) {
            if (it == 2) {
                k_set_it<<<1, 1, 0, st>>>(W->st, 2);
                IE_LAUNCHED();
            }
            IE_CUDA(cudaGraphLaunch(W->gexec, st));
            g_launches.fetch_add(W->gnodes, std::memory_order_relaxed);
        } else {
            if ((rc = enqueue_iter(it, do_p, pending, spec, st, true, it))) return rc;
        }
        if (it % kBatch == 0 || it == max_iters + 1) {
            // pipelined status polling: this batch's state copy is queued behind
            // it, and the host waits on the PREVIOUS batch's copy, so the GPU
            // never drains between batches (at most one batch of no-op
            // iterations -- every kernel returns on the device stop flag --
            // follows convergence)
            const int slot = (int)(nbatch & 1);
            PcgState* hs = slot ? W->host2 : W->host;
            IE_CUDA(cudaMemcpyAsync(hs, W->st, sizeof(PcgState), cudaMemcpyDeviceToHost, st));
            IE_CUDA(cudaEventRecord(W->poll_ev[slot], st));
            if (nbatch > 0) {
                IE_CUDA(cudaEventSynchronize(W->poll_ev[slot ^ 1]));
                if ((slot ? W->host : W->host2)->stop) break;
            }
            ++nbatch;
        }
    }
    IE_CUDA(cudaMemcpyAsync(W->host, W->st, sizeof(PcgState), cudaMemcpyDeviceToHost, st));
    IE_CUDA(cudaStreamSynchronize(st));
    const PcgState S = *W->host;
    flags[0] = S.status == 1;
    flags[1] = S.status == 2;
    *n_it = S.n_it;
    if (S.status == 4 || S.status == 5) {
        if (fail_iter) *fail_iter = S.fail_iter;
        if (fail_value) *fail_value = S.fail_value;
    }
    const int64_t nh = S.n_it + 1;
    IE_CUDA(cudaMemcpyAsync(hist, W->hist, (size_t)nh * 8, cudaMemcpyDeviceToHost, st));
    IE_CUDA(cudaMemcpyAsync(u, uu, (size_t)N * 8, cudaMemcpyDeviceToDevice, st));
    IE_CUDA(cudaStreamSynchronize(st));
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
    if (S.status == 4) return IE_ERR_BREAKDOWN;
    if (S.status == 5) return IE_ERR_NONFINITE;
    return IE_OK;
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
    if (!s->stop) s->j += 1;
}

__global__ void k_lz_alpha(const double* part, int nch, double* alphas, const LzState* s) {
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
    if (!A || !T || !v0 || !lambda || (which != 0 && which != 1) || max_iters < 0) {
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
        if ((r2 = precond_apply(T, avj.p, wb.p, nullptr, s2, stop))) return r2;
        k_lz_dot<<<nch, kRed, 0, s2>>>(wb.p, avj.p, N, part.p, S.p);
        IE_LAUNCHED();
        k_lz_alpha<<<1, kRed, 0, s2>>>(part.p, nch, da, S.p);
        IE_LAUNCHED();
        for (int pass = 0; pass < 2; ++pass) {  // two-pass A-orthogonalisation (CGS2)
            k_lz_gemv_t<<<dim3(nch, (unsigned)nb_max), kRed, 0, s2>>>(AV.p, wb.p, N, part.p, nch, S.p);
            IE_LAUNCHED();
            k_lz_reduce_rows<<<(unsigned)nb_max, kRed, 0, s2>>>(part.p, nch, cbuf.p, S.p);
            IE_LAUNCHED();
            k_lz_gemv_sub<<<(unsigned)((N + 31) / 32), 256, 0, s2>>>(wb.p, V.p, cbuf.p, N, S.p);
            IE_LAUNCHED();
        }
        if ((r2 = matvec_launch(A, wb.p, N, 1, awb.p, N, 0, N, s2, stop))) return r2;
        k_lz_dot<<<nch, kRed, 0, s2>>>(wb.p, awb.p, N, part.p, S.p);
        IE_LAUNCHED();
        k_lz_control<<<1, kRed, 0, s2>>>(part.p, nch, da, db, which, rtol, S.p);
        IE_LAUNCHED();
        k_lz_next<<<g1(N), 256, 0, s2>>>(V.p, AV.p, avj.p, wb.p, awb.p, S.p, N);
        IE_LAUNCHED();
        k_lz_advance<<<1, 1, 0, s2>>>(S.p);
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

// ------------------------------------------------------- sharded K4 (NCCL) --
// ie_pcg_f64 on G ranks (one process per GPU), rank g owning the grid-row band
// [bounds[g], bounds[g+1]) of every vector (distributed.py documents the plan;
// this is its native driver).  Per iteration, on the rank's stream:
//   all-gather of the per-chunk max|p|, max|u| (2-RHS scaling) ->
//   band row FFTs -> all-to-all -> column slab pass -> all-to-all -> inverse
//   rows (q, w on the band) -> post_pass partials -> all-gather -> k_iter_a
//   (every rank reduces all chunks in global order: identical scalars) ->
//   r-halo send/recv -> apply of the rank's subdomains, z on the band ->
//   all-gather of r.z partials -> k_iter_b.
// Device-side control as in ie_pcg_f64; the steady-state iteration, NCCL calls
// included, is one captured CUDA graph.  Every rank takes the same decisions
// from the same reduced scalars, so the collectives stay matched.
struct ie_fft;
namespace ie {
// Device workspace + captured iteration graph of the sharded driver, cached on
// the communicator for repeated solves with the same operator / bands.
struct ShardWork {
    uint64_t key_a = 0, key_t = 0;
    int64_t nb = 0, b0 = 0, cap = 0;
    double *PU = nullptr, *QW = nullptr, *rfull = nullptr, *z = nullptr, *fb = nullptr, *part = nullptr;
    double *amax = nullptr, *dh = nullptr;
    double2 *buf1 = nullptr, *buf2 = nullptr, *buf3 = nullptr;
    PcgState* S = nullptr;
    PcgState* host = nullptr;
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t cap_s = nullptr;
    int gnodes = 0;
    ~ShardWork() {
        for (void* p : {(void*)PU, (void*)QW, (void*)rfull, (void*)z, (void*)fb, (void*)part, (void*)amax,
                        (void*)dh, (void*)buf1, (void*)buf2, (void*)buf3, (void*)S})
            if (p) cudaFree(p);
        if (host) cudaFreeHost(host);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (cap_s) cudaStreamDestroy(cap_s);
    }
};
}  // namespace ie

struct ie_comm {
    ncclComm_t c;
    int nranks, rank;
    ie::ShardWork* work = nullptr;
};

namespace ie {
const ie_fft* matvec_fft(const ie_matvec* m);
int matvec_dim(const ie_matvec* m);
int matvec_n(const ie_matvec* m);
int fft_band_fwd(const ie_fft* f, const double* X0, const double* X1, int nrows, int parts, double2* out,
                 const double* amax, int namax, cudaStream_t st);
int fft_band_cols(const ie_fft* f, double2* buf, int c0, int ncols, cudaStream_t st);
int fft_band_inv(const ie_fft* f, const double2* in, int nrows, int parts, double* Y0, double* Y1,
                 const double* amax, int namax, cudaStream_t st);
int precond_apply_band(const ie_precond* p, const double* r, double* z, double* partials, int64_t i0, int64_t i1,
                       cudaStream_t st, const int* stop);
}  // namespace ie

#define IE_NCCL(call)                                                          \
    do {                                                                       \
        ncclResult_t _r = (call);                                              \
        if (_r != ncclSuccess) {                                               \
            ie::set_error(std::string("nccl: ") + ncclGetErrorString(_r));     \
            return IE_ERR_CUDA;                                                \
        }                                                                      \
    } while (0)

extern "C" int64_t ie_comm_id_bytes(void) { return (int64_t)sizeof(ncclUniqueId); }

extern "C" int ie_comm_unique_id(void* out) {
    if (!out) return IE_ERR_ARG;
    ncclUniqueId id;
    IE_NCCL(ncclGetUniqueId(&id));
    memcpy(out, &id, sizeof(id));
    return IE_OK;
}

extern "C" int ie_comm_create(const void* id, int32_t nranks, int32_t rank, ie_comm** out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) {
        ie::set_error("ie_comm_create: bad arguments");
        return IE_ERR_ARG;
    }
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ie_comm* c = new ie_comm();
    c->nranks = nranks;
    c->rank = rank;
    ncclResult_t r = ncclCommInitRank(&c->c, nranks, uid, rank);
    if (r != ncclSuccess) {
        ie::set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        delete c;
        return IE_ERR_CUDA;
    }
    *out = c;
    return IE_OK;
}

extern "C" void ie_comm_destroy(ie_comm* c) {
    if (!c) return;
    delete c->work;
    ncclCommDestroy(c->c);
    delete c;
}

extern "C" int ie_pcg_sharded_f64(const ie_matvec* A, const ie_precond* T, ie_comm* comm, const int64_t* bounds,
                                  const int64_t* need, const double* f_band, double* u_band, double tol,
                                  int64_t max_iters, double* hist, int64_t* n_it, int32_t* flags, double* times,
                                  int64_t* fail_iter, double* fail_value, void* stream) {
    using namespace ie;
    if (!A || !comm || !bounds || !f_band || !u_band || !hist || !n_it || !flags || !times || max_iters < 0 ||
        !(tol > 0.0 && tol < 1.0)) {
        set_error("ie_pcg_sharded_f64: bad arguments");
        return IE_ERR_ARG;
    }
    const ie_fft* F = matvec_fft(A);
    const int G = comm->nranks, g = comm->rank;
    const int N = matvec_N(A), n = matvec_n(A), M = 2 * n;
    const int64_t nb = bounds[g + 1] - bounds[g];
    bool ok = F && matvec_dim(A) == 2 && M % G == 0 && (((M / G) & (M / G - 1)) == 0) && bounds[0] == 0 &&
              bounds[G] == N;
    for (int h = 0; h < G && ok; ++h)
        ok = (bounds[h + 1] - bounds[h] == nb) && (bounds[h] % kChunk == 0) && (bounds[h] % n == 0);
    if (!ok || nb <= 0 || nb % kChunk) {
        set_error("ie_pcg_sharded_f64: needs the 2D FFT operator, G | 2n (power-of-two slabs) and equal, "
                  "chunk-aligned bands of whole grid rows");
        return IE_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t b0 = bounds[g];
    const int nrows = (int)(nb / n), Mc = M / G;
    const int nchb = (int)(nb / kChunk), nch = nchb * G, c0 = (int)(b0 / kChunk);
    int64_t cap = 1024;
    while (cap < max_iters + 1) cap *= 2;
    const uint64_t ka = matvec_uid(A), kt = T ? precond_uid(T) : 0;
    ShardWork* W = comm->work;
    if (!W || W->key_a != ka || W->key_t != kt || W->nb != nb || W->b0 != b0 || W->cap < cap) {
        delete W;
        comm->work = W = new ShardWork();
        W->key_a = ka;
        W->key_t = kt;
        W->nb = nb;
        W->b0 = b0;
        W->cap = cap;
        const bool one = G == 1;  // one rank: the transposes are the identity (buffers aliased)
        IE_CUDA(cudaMalloc(&W->PU, 2 * nb * 8));
        IE_CUDA(cudaMalloc(&W->QW, 2 * nb * 8));
        IE_CUDA(cudaMalloc(&W->rfull, (size_t)N * 8));
        IE_CUDA(cudaMalloc(&W->z, nb * 8));
        IE_CUDA(cudaMalloc(&W->fb, nb * 8));
        IE_CUDA(cudaMalloc(&W->part, 3 * (size_t)nch * 8));
        IE_CUDA(cudaMalloc(&W->amax, 2 * (size_t)nch * 8));
        IE_CUDA(cudaMalloc(&W->dh, (size_t)cap * 8));
        IE_CUDA(cudaMalloc(&W->buf1, (size_t)nrows * M * 16));
        if (!one) {
            IE_CUDA(cudaMalloc(&W->buf2, (size_t)n * Mc * 16));
            IE_CUDA(cudaMalloc(&W->buf3, (size_t)nrows * M * 16));
        }
        IE_CUDA(cudaMalloc(&W->S, sizeof(PcgState)));
        IE_CUDA(cudaMallocHost(&W->host, sizeof(PcgState)));
    }
    int rc;
    double *PU = W->PU, *QW = W->QW, *rfull = W->rfull, *z = W->z, *fb = W->fb, *part = W->part;
    double *amax = W->amax, *dh = W->dh;
    double2* buf1 = W->buf1;
    double2* buf2 = G == 1 ? W->buf1 : W->buf2;
    double2* buf3 = G == 1 ? W->buf1 : W->buf3;
    PcgState* S = W->S;
    PcgState* host = W->host;
    double* p = PU;
    double* uu = PU + nb;
    double* q = QW;
    double* w = QW + nb;
    double* r = rfull + b0;  // r lives inside the halo buffer
    double* part_pq = part;
    double* part_res = part + nch;
    double* part_rz = part + 2 * nch;
    const int* stop = &S->stop;
    const ncclComm_t cc = comm->c;
    // halo plan: send my band's overlap with each rank's need range, receive theirs with mine
    std::vector<int64_t> s_off(G, 0), s_cnt(G, 0), r_off(G, 0), r_cnt(G, 0);
    if (need && T) {
        const int64_t lo = need[2 * g], hi = need[2 * g + 1];
        for (int h = 0; h < G; ++h) {
            if (h == g) continue;
            const int64_t a = std::max(b0, need[2 * h]), b = std::min(bounds[g + 1], need[2 * h + 1]);
            if (b > a) s_off[h] = a, s_cnt[h] = b - a;
            const int64_t a2 = std::max(bounds[h], lo), b2 = std::min(bounds[h + 1], hi);
            if (b2 > a2) r_off[h] = a2, r_cnt[h] = b2 - a2;
        }
    } else if (T) {  // no need ranges: the whole vector
        for (int h = 0; h < G; ++h)
            if (h != g) s_off[h] = b0, s_cnt[h] = nb, r_off[h] = bounds[h], r_cnt[h] = bounds[h + 1] - bounds[h];
    }
    auto allgather_chunks = [&](double* arr, int per, cudaStream_t s) -> int {  // arr[nch * per], rank slab in place
        IE_NCCL(ncclAllGather(arr + (size_t)c0 * per, arr, (size_t)nchb * per, ncclDouble, cc, s));
        return IE_OK;
    };
    auto alltoall = [&](const double2* src, double2* dst, cudaStream_t s) -> int {  // equal blocks of nrows*Mc
        if (G == 1) return IE_OK;  // identity transpose, aliased buffers
        const size_t cnt = (size_t)nrows * Mc * 2;
        IE_NCCL(ncclGroupStart());
        for (int h = 0; h < G; ++h) {
            IE_NCCL(ncclSend((const double*)src + h * cnt, cnt, ncclDouble, h, cc, s));
            IE_NCCL(ncclRecv((double*)dst + h * cnt, cnt, ncclDouble, h, cc, s));
        }
        IE_NCCL(ncclGroupEnd());
        return IE_OK;
    };
    auto halo = [&](cudaStream_t s) -> int {
        bool any = false;
        for (int h = 0; h < G; ++h) any = any || s_cnt[h] || r_cnt[h];
        if (!any) return IE_OK;
        IE_NCCL(ncclGroupStart());
        for (int h = 0; h < G; ++h) {
            if (s_cnt[h]) IE_NCCL(ncclSend(rfull + s_off[h], (size_t)s_cnt[h], ncclDouble, h, cc, s));
            if (r_cnt[h]) IE_NCCL(ncclRecv(rfull + r_off[h], (size_t)r_cnt[h], ncclDouble, h, cc, s));
        }
        IE_NCCL(ncclGroupEnd());
        return IE_OK;
    };
    auto matvec = [&](const double* X, int nrhs, double* Y, cudaStream_t s) -> int {
        int r2;
        if (nrhs == 2 && (r2 = allgather_chunks(amax, 2, s))) return r2;
        if ((r2 = fft_band_fwd(F, X, nrhs == 2 ? X + nb : nullptr, nrows, G, buf1, amax, nch, s))) return r2;
        if ((r2 = alltoall(buf1, buf2, s))) return r2;
        if ((r2 = fft_band_cols(F, buf2, g * Mc, Mc, s))) return r2;
        if ((r2 = alltoall(buf2, buf3, s))) return r2;
        return fft_band_inv(F, buf3, nrows, G, Y, nrhs == 2 ? Y + nb : nullptr, amax, nch, s);
    };
    auto apply = [&](cudaStream_t s) -> int {  // z (band) and part_rz (rank slab) from r
        int r2;
        if (T) {
            if ((r2 = halo(s))) return r2;
            if ((r2 = precond_apply_band(T, rfull, z, part_rz + c0, b0, b0 + nb, s, stop))) return r2;
        } else {
            k_copy_if_running<<<g1(nb), 256, 0, s>>>(z, r, (int)nb, stop);
            IE_LAUNCHED();
            k_dot_partials<<<nchb, kRed, 0, s>>>(r, z, (int)nb, 0, part_rz + c0);
            IE_LAUNCHED();
        }
        return allgather_chunks(part_rz, 1, s);
    };
    // ||f||, init (pcg.py:72-91)
    IE_CUDA(cudaMemcpyAsync(fb, f_band, nb * 8, cudaMemcpyDeviceToDevice, st));
    k_dot_partials<<<nchb, kRed, 0, st>>>(fb, fb, (int)nb, 0, part_pq + c0);
    IE_LAUNCHED();
    if ((rc = allgather_chunks(part_pq, 1, st))) return rc;
    k_pcg_init<<<1, kRed, 0, st>>>(part_pq, nch, S, tol, max_iters, dh);
    IE_LAUNCHED();
    IE_CUDA(cudaMemsetAsync(uu, 0, nb * 8, st));
    IE_CUDA(cudaMemsetAsync(amax, 0, 2 * (size_t)nch * 8, st));
    IE_CUDA(cudaMemcpyAsync(r, fb, nb * 8, cudaMemcpyDeviceToDevice, st));
    if ((rc = apply(st))) return rc;
    IE_CUDA(cudaMemcpyAsync(p, z, nb * 8, cudaMemcpyDeviceToDevice, st));
    k_pcg_rho0<<<1, kRed, 0, st>>>(part_rz, nch, S);
    IE_LAUNCHED();
    // (the first 2-RHS pass, iteration 2, uses max|u| from k_iter_a and max|p|
    // from k_iter_b of iteration 1, as in ie_pcg_f64)
    auto enqueue_iter = [&](int64_t itarg, int do_p, int pending, bool spec, cudaStream_t s) -> int {
        int r2;
        if (do_p && pending) r2 = matvec(PU, 2, QW, s);
        else if (do_p) r2 = matvec(p, 1, q, s);
        else r2 = matvec(uu, 1, w, s);
        if (r2) return r2;
        k_post_pass<<<nchb, kRed, 0, s>>>(p, q, fb, w, (int)nb, do_p, pending, part_pq + c0, part_res + c0, stop);
        IE_LAUNCHED();
        if (do_p && (r2 = allgather_chunks(part_pq, 1, s))) return r2;
        if (pending && (r2 = allgather_chunks(part_res, 1, s))) return r2;
        (uu ? k_iter_a<true> : k_iter_a<false>)<<<nchb, kRed, 0, s>>>(part_pq, part_res, nch, do_p, pending, itarg, S, dh, uu, r, p, q, (int)nb,
                                       amax + 2 * (size_t)c0);
        IE_LAUNCHED();
        if (spec) {
            if ((r2 = apply(s))) return r2;
            k_iter_b<<<nchb, kRed, 0, s>>>(part_rz, nch, itarg, S, p, z, (int)nb, amax + 2 * (size_t)c0);
            IE_LAUNCHED();
        }
        return IE_OK;
    };
    const bool use_graph = max_iters >= 3 && !getenv("IEDD_B200_NO_GRAPH");
    if (use_graph && !W->gexec) {
        if (!W->cap_s) IE_CUDA(cudaStreamCreateWithFlags(&W->cap_s, cudaStreamNonBlocking));
        cudaStream_t cap_s = W->cap_s;
        // order the capture stream after the setup work on st
        cudaEvent_t ev;
        IE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        IE_CUDA(cudaEventRecord(ev, st));
        IE_CUDA(cudaStreamWaitEvent(cap_s, ev, 0));
        cudaEventDestroy(ev);
        if (T && (rc = precond_prepare_stream(T, cap_s))) return rc;
        cudaGraph_t gr;
        IE_CUDA(cudaStreamBeginCapture(cap_s, cudaStreamCaptureModeThreadLocal));
        int r2 = enqueue_iter(-1, 1, 1, true, cap_s);  // k_iter_b advances it_dev
        cudaError_t ce = cudaStreamEndCapture(cap_s, &gr);
        if (r2) return r2;
        IE_CUDA(ce);
        size_t nn = 0;
        cudaGraphGetNodes(gr, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) cudaGraphGetNodes(gr, nodes.data(), &nn);
        W->gnodes = 0;
        for (auto nd : nodes) {
            cudaGraphNodeType t;
            if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++W->gnodes;
        }
        ce = cudaGraphInstantiate(&W->gexec, gr, 0);
        cudaGraphDestroy(gr);
        IE_CUDA(ce);
    }
    cudaGraphExec_t gexec = W->gexec;
    const int gnodes = W->gnodes;
    static const int64_t kBatch = getenv("IEDD_B200_PCG_BATCH") ? atoll(getenv("IEDD_B200_PCG_BATCH")) : 4;
    for (int64_t it = 1; it <= max_iters + 1; ++it) {
        const int do_p = it <= max_iters;
        const int pending = it >= 2;
        const bool spec = do_p && it < max_iters;
        if (use_graph && pending && spec) {
            if (it == 2) {
                k_set_it<<<1, 1, 0, st>>>(S, 2);
                IE_LAUNCHED();
            }
            IE_CUDA(cudaGraphLaunch(gexec, st));
            g_launches.fetch_add(gnodes, std::memory_order_relaxed);
        } else if ((rc = enqueue_iter(it, do_p, pending, spec, st))) {
            return rc;
        }
        if (it % kBatch == 0 || it == max_iters + 1) {
            IE_CUDA(cudaMemcpyAsync(host, S, sizeof(PcgState), cudaMemcpyDeviceToHost, st));
            IE_CUDA(cudaStreamSynchronize(st));
            if (host->stop) break;
        }
    }
    IE_CUDA(cudaMemcpyAsync(host, S, sizeof(PcgState), cudaMemcpyDeviceToHost, st));
    IE_CUDA(cudaStreamSynchronize(st));
    const PcgState H = *host;
    flags[0] = H.status == 1;
    flags[1] = H.status == 2;
    *n_it = H.n_it;
    if (H.status == 4 || H.status == 5) {
        if (fail_iter) *fail_iter = H.fail_iter;
        if (fail_value) *fail_value = H.fail_value;
    }
    IE_CUDA(cudaMemcpyAsync(hist, dh, (size_t)(H.n_it + 1) * 8, cudaMemcpyDeviceToHost, st));
    IE_CUDA(cudaMemcpyAsync(u_band, uu, nb * 8, cudaMemcpyDeviceToDevice, st));
    IE_CUDA(cudaStreamSynchronize(st));
    times[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    times[1] = 0.0;
    if (H.nf == 0.0) times[0] = 0.0;
    if (H.status == 4) return IE_ERR_BREAKDOWN;
    if (H.status == 5) return IE_ERR_NONFINITE;
    return IE_OK;
}
