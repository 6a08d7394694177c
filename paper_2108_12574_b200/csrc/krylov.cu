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
#include <math.h>

#include <chrono>
#include <vector>

#include "common.cuh"

struct ie_matvec;
struct ie_precond;

namespace ie {

int matvec_launch(const ie_matvec* m, const double* X, int64_t ldx, int nrhs, double* Y, int64_t ldy,
                  int64_t row_begin, int64_t row_end, cudaStream_t st);
int precond_apply(const ie_precond* p, const double* r, double* z, double* partials, cudaStream_t st);
int matvec_N(const ie_matvec* m);

constexpr int kChunk = 2048;
constexpr int kRed = 256;
int dot_chunks(int64_t n) { return (int)((n + kChunk - 1) / kChunk); }

__device__ __forceinline__ double block_tree(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    return sh[0];
}

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

__device__ double reduce_partials(const double* part, int nch, double* sh) {
    double loc = 0.0;
    for (int c = threadIdx.x; c < nch; c += blockDim.x) loc += part[c];
    return block_tree(loc, sh);
}

struct Scal {
    double rho, alpha, beta, denom, rel, nf;
    double pad[2];
};

__global__ void k_set_nf(const double* part, int nch, Scal* sc) {
    __shared__ double sh[kRed];
    const double v = reduce_partials(part, nch, sh);
    if (threadIdx.x == 0) sc->nf = sqrt(v);
}

// After the A-pass: denom = p.q, alpha = rho/denom (when do_p);
// rel = ||f - w|| / ||f|| (when pending).
__global__ void k_control_a(const double* part_pq, const double* part_res, int nch, int do_p, int pending,
                            Scal* sc) {
    __shared__ double sh[kRed];
    double denom = 0.0, res2 = 0.0;
    if (do_p) denom = reduce_partials(part_pq, nch, sh);
    __syncthreads();
    if (pending) res2 = reduce_partials(part_res, nch, sh);
    if (threadIdx.x == 0) {
        if (do_p) {
            sc->denom = denom;
            sc->alpha = sc->rho / denom;
        }
        if (pending) sc->rel = sqrt(res2) / sc->nf;
    }
}

// After the apply: rho' = r.z, beta = rho'/rho, rho = rho'.
__global__ void k_control_b(const double* part_rz, int nch, int first, Scal* sc) {
    __shared__ double sh[kRed];
    const double rz = reduce_partials(part_rz, nch, sh);
    if (threadIdx.x == 0) {
        if (!first) sc->beta = rz / sc->rho;
        sc->rho = rz;
    }
}

__global__ void k_post_pass(const double* p, const double* q, const double* f, const double* w, int N, int do_p,
                            int pending, double* part_pq, double* part_res) {
    __shared__ double sh[kRed];
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

// u += alpha p; r -= alpha q  (products rounded first, as numpy does)
__global__ void k_update_ur(double* u, double* r, const double* p, const double* q, const Scal* sc, int N) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double al = sc->alpha;
    u[i] = __dadd_rn(u[i], __dmul_rn(al, p[i]));
    r[i] = __dsub_rn(r[i], __dmul_rn(al, q[i]));
}

// p = z + beta p
__global__ void k_update_p(double* p, const double* z, const Scal* sc, int N) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    p[i] = __dadd_rn(z[i], __dmul_rn(sc->beta, p[i]));
}

__global__ void k_scale_div(double* x, const double* src, double d, int N) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) x[i] = src[i] / d;
}

// Lanczos: c_i = AV_i . w for i < nb (partials per (i, chunk))
__global__ void __launch_bounds__(kRed) k_gemv_t_partials(const double* AV, int64_t ld, int nb, const double* w,
                                                          int N, double* part, int nch) {
    __shared__ double sh[kRed];
    const int i = blockIdx.y;
    const double* v = AV + (int64_t)i * ld;
    const int base = blockIdx.x * kChunk;
    double loc = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk / kRed; ++e) {
        const int t = base + e * kRed + threadIdx.x;
        if (t < N) loc = fma(v[t], w[t], loc);
    }
    const double s = block_tree(loc, sh);
    if (threadIdx.x == 0) part[(int64_t)i * nch + blockIdx.x] = s;
}

__global__ void k_reduce_rows(const double* part, int nch, double* out) {
    __shared__ double sh[kRed];
    const double v = reduce_partials(part + (int64_t)blockIdx.x * nch, nch, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = v;
}

// w -= sum_i c_i V_i  (ascending i, products rounded first)
__global__ void k_gemv_sub(double* w, const double* V, int64_t ld, int nb, const double* c, int N) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    double x = w[t];
    for (int i = 0; i < nb; ++i) x = __dsub_rn(x, __dmul_rn(c[i], V[(int64_t)i * ld + t]));
    w[t] = x;
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

// Extremal eigenvalue of the m x m tridiagonal by 32-way multisection.
__global__ void k_ritz(const double* a, const double* b, int m, int which, double* out) {
    const int lane = threadIdx.x;
    double lo = a[0], hi = a[0];
    for (int i = 0; i < m; ++i) {
        const double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i < m - 1 ? fabs(b[i]) : 0.0);
        lo = fmin(lo, a[i] - r);
        hi = fmax(hi, a[i] + r);
    }
    const double span = fmax(hi - lo, 1e-300);
    lo -= 1e-3 * span + 1e-300;
    hi += 1e-3 * span + 1e-300;
    const int target = which == 0 ? 1 : m;  // count(x) >= target  <=>  x > lambda
    for (int it = 0; it < 64; ++it) {
        const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
        const bool above = sturm_count(a, b, m, x) >= target;
        const unsigned mask = __ballot_sync(0xffffffffu, above);
        const int first = mask ? __ffs(mask) - 1 : 32;  // first lane above the eigenvalue
        const double nlo = first == 0 ? lo : lo + (hi - lo) * (double)first / 33.0;
        const double nhi = first == 32 ? hi : lo + (hi - lo) * (double)(first + 1) / 33.0;
        if (!(nhi < hi) && !(nlo > lo)) break;  // no progress: interval at rounding level
        lo = nlo;
        hi = nhi;
        if (hi - lo <= 2.0 * 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi))) break;
    }
    if (lane == 0) *out = 0.5 * (lo + hi);
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
    DevBuf<double> PU(st), QW(st), r(st), z(st), part(st);
    DevBuf<Scal> sc(st);
    IE_CUDA(PU.alloc(2 * (size_t)N));
    IE_CUDA(QW.alloc(2 * (size_t)N));
    IE_CUDA(r.alloc(N));
    IE_CUDA(z.alloc(N));
    IE_CUDA(part.alloc(3 * (size_t)nch));
    IE_CUDA(sc.alloc(1));
    Scal* hs = nullptr;
    IE_CUDA(cudaMallocHost(&hs, sizeof(Scal)));
    struct HostFree {
        Scal* h;
        ~HostFree() { cudaFreeHost(h); }
    } hf{hs};
    double* p = PU.p;
    double* uu = PU.p + N;
    double* q = QW.p;
    double* w = QW.p + N;
    double* part_pq = part.p;
    double* part_res = part.p + nch;
    double* part_rz = part.p + 2 * nch;
    cudaEvent_t ev0, ev1;
    IE_CUDA(cudaEventCreate(&ev0));
    IE_CUDA(cudaEventCreate(&ev1));
    struct EvFree {
        cudaEvent_t a, b;
        ~EvFree() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } ef{ev0, ev1};
    double t_prec = 0.0;
    int64_t n_prec = 0;
    auto apply = [&](const double* rin, double* zout) -> int {
        IE_CUDA(cudaEventRecord(ev0, st));
        if (T) {
            int rc = precond_apply(T, rin, zout, part_rz, st);
            if (rc) return rc;
        } else {
            IE_CUDA(cudaMemcpyAsync(zout, rin, (size_t)N * 8, cudaMemcpyDeviceToDevice, st));
            k_dot_partials<<<nch, kRed, 0, st>>>(rin, zout, N, 0, part_rz);
            IE_LAUNCHED();
        }
        IE_CUDA(cudaEventRecord(ev1, st));
        return IE_OK;
    };
    auto apply_time = [&]() -> int {
        float ms = 0.f;
        IE_CUDA(cudaEventSynchronize(ev1));
        IE_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
        t_prec += ms * 1e-3;
        n_prec += 1;
        return IE_OK;
    };
    // ||f||
    k_dot_partials<<<nch, kRed, 0, st>>>(f, f, N, 0, part_pq);
    IE_LAUNCHED();
    k_set_nf<<<1, kRed, 0, st>>>(part_pq, nch, sc.p);
    IE_LAUNCHED();
    IE_CUDA(cudaMemcpyAsync(hs, sc.p, sizeof(Scal), cudaMemcpyDeviceToHost, st));
    IE_CUDA(cudaStreamSynchronize(st));
    flags[0] = flags[1] = 0;
    if (hs->nf == 0.0) {  // pcg.py:74-78
        IE_CUDA(cudaMemsetAsync(u, 0, (size_t)N * 8, st));
        hist[0] = 0.0;
        *n_it = 0;
        flags[0] = 1;
        times[0] = times[1] = 0.0;
        IE_CUDA(cudaStreamSynchronize(st));
        return IE_OK;
    }
    IE_CUDA(cudaMemsetAsync(uu, 0, (size_t)N * 8, st));
    IE_CUDA(cudaMemcpyAsync(r.p, f, (size_t)N * 8, cudaMemcpyDeviceToDevice, st));
    int rc = apply(r.p, z.p);
    if (rc) return rc;
    if ((rc = apply_time())) return rc;
    IE_CUDA(cudaMemcpyAsync(p, z.p, (size_t)N * 8, cudaMemcpyDeviceToDevice, st));
    k_control_b<<<1, kRed, 0, st>>>(part_rz, nch, 1, sc.p);
    IE_LAUNCHED();
    hist[0] = 1.0;
    int64_t k = 0;
    bool pending = false;
    bool spec_apply = false;
    int result = IE_OK;
    while (true) {
        const int64_t next = k + 1;
        const bool do_p = next <= max_iters;
        if (!pending && !do_p) break;
        if (do_p && pending) {
            rc = matvec_launch(A, PU.p, N, 2, QW.p, N, 0, N, st);
        } else if (do_p) {
            rc = matvec_launch(A, p, N, 1, q, N, 0, N, st);
        } else {
            rc = matvec_launch(A, uu, N, 1, w, N, 0, N, st);
        }
        if (rc) return rc;
        k_post_pass<<<nch, kRed, 0, st>>>(p, q, f, w, N, do_p, pending, part_pq, part_res);
        IE_LAUNCHED();
        k_control_a<<<1, kRed, 0, st>>>(part_pq, part_res, nch, do_p, pending, sc.p);
        IE_LAUNCHED();
        IE_CUDA(cudaMemcpyAsync(hs, sc.p, sizeof(Scal), cudaMemcpyDeviceToHost, st));
        IE_CUDA(cudaStreamSynchronize(st));
        if (spec_apply) {
            if ((rc = apply_time())) return rc;
            spec_apply = false;
        }
        if (pending) {
            const double rel = hs->rel;
            if (!std::isfinite(rel)) {  // pcg.py:109-110
                if (fail_iter) *fail_iter = k;
                if (fail_value) *fail_value = rel;
                result = IE_ERR_NONFINITE;
                break;
            }
            hist[k] = rel;
            if (rel <= tol) {
                flags[0] = 1;
                break;
            }
            if (k >= 30 && rel > (1.0 - 1e-3) * hist[k - 30]) {  // pcg.py:115-119
                flags[1] = 1;
                break;
            }
            if (!do_p) break;
        }
        const double denom = hs->denom;
        if (!std::isfinite(denom) || denom <= 0.0) {  // pcg.py:99-103
            if (fail_iter) *fail_iter = next;
            if (fail_value) *fail_value = denom;
            result = IE_ERR_BREAKDOWN;
            break;
        }
        k_update_ur<<<g1(N), 256, 0, st>>>(uu, r.p, p, q, sc.p, N);
        IE_LAUNCHED();
        k = next;
        pending = true;
        if (k < max_iters) {
            if ((rc = apply(r.p, z.p))) return rc;
            spec_apply = true;
            k_control_b<<<1, kRed, 0, st>>>(part_rz, nch, 0, sc.p);
            IE_LAUNCHED();
            k_update_p<<<g1(N), 256, 0, st>>>(p, z.p, sc.p, N);
            IE_LAUNCHED();
        }
    }
    *n_it = k;
    IE_CUDA(cudaMemcpyAsync(u, uu, (size_t)N * 8, cudaMemcpyDeviceToDevice, st));
    IE_CUDA(cudaStreamSynchronize(st));
    times[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    times[1] = t_prec / (double)(n_prec > 0 ? n_prec : 1);
    return result;
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
    DevBuf<double> V(st), AV(st), wb(st), awb(st), part(st), cbuf(st), tri(st), scal(st);
    IE_CUDA(V.alloc((size_t)nb_max * N));
    IE_CUDA(AV.alloc((size_t)nb_max * N));
    IE_CUDA(wb.alloc(N));
    IE_CUDA(awb.alloc(N));
    IE_CUDA(part.alloc((size_t)std::max<int64_t>(nb_max, 2) * nch));
    IE_CUDA(cbuf.alloc(nb_max + 2));
    IE_CUDA(tri.alloc(2 * (size_t)nb_max + 2));
    IE_CUDA(scal.alloc(4));
    double* hsc = nullptr;
    IE_CUDA(cudaMallocHost(&hsc, 4 * sizeof(double)));
    struct HostFree {
        double* h;
        ~HostFree() { cudaFreeHost(h); }
    } hf{hsc};
    double* da = tri.p;            // alphas
    double* db = tri.p + nb_max;   // betas
    auto dot = [&](const double* x, const double* y, double* dst) -> int {
        k_dot_partials<<<nch, kRed, 0, st>>>(x, y, N, 0, part.p);
        IE_LAUNCHED();
        k_reduce_rows<<<1, kRed, 0, st>>>(part.p, nch, dst);
        IE_LAUNCHED();
        return IE_OK;
    };
    int rc;
    // v = v0; av = A v; nrm = sqrt(v.av); v /= nrm; av /= nrm   (spectrum.py:148-153)
    IE_CUDA(cudaMemcpyAsync(wb.p, v0, (size_t)N * 8, cudaMemcpyDeviceToDevice, st));
    if ((rc = matvec_launch(A, wb.p, N, 1, awb.p, N, 0, N, st))) return rc;
    if ((rc = dot(wb.p, awb.p, scal.p))) return rc;
    IE_CUDA(cudaMemcpyAsync(hsc, scal.p, 8, cudaMemcpyDeviceToHost, st));
    IE_CUDA(cudaStreamSynchronize(st));
    const double nrm = sqrt(hsc[0]);
    k_scale_div<<<g1(N), 256, 0, st>>>(V.p, wb.p, nrm, N);
    IE_LAUNCHED();
    k_scale_div<<<g1(N), 256, 0, st>>>(AV.p, awb.p, nrm, N);
    IE_LAUNCHED();
    std::vector<double> alphas, betas;
    bool have_est = false;
    double est = 0.0;
    int stable = 0;
    int64_t j = 0;
    int64_t taken = 0;
    for (j = 0; j < max_iters; ++j) {
        double* Vj = V.p + (size_t)j * N;
        double* AVj = AV.p + (size_t)j * N;
        (void)Vj;
        if ((rc = precond_apply(T, AVj, wb.p, nullptr, st))) return rc;
        if ((rc = dot(wb.p, AVj, da + j))) return rc;
        const int nb = (int)(j + 1);
        for (int pass = 0; pass < 2; ++pass) {  // two-pass A-orthogonalisation (CGS2)
            dim3 grid(nch, nb);
            k_gemv_t_partials<<<grid, kRed, 0, st>>>(AV.p, N, nb, wb.p, N, part.p, nch);
            IE_LAUNCHED();
            k_reduce_rows<<<nb, kRed, 0, st>>>(part.p, nch, cbuf.p);
            IE_LAUNCHED();
            k_gemv_sub<<<g1(N), 256, 0, st>>>(wb.p, V.p, N, nb, cbuf.p, N);
            IE_LAUNCHED();
        }
        if ((rc = matvec_launch(A, wb.p, N, 1, awb.p, N, 0, N, st))) return rc;
        if ((rc = dot(wb.p, awb.p, scal.p + 1))) return rc;
        IE_CUDA(cudaMemcpyAsync(hsc, scal.p + 1, 8, cudaMemcpyDeviceToHost, st));
        double aj = 0.0;
        IE_CUDA(cudaMemcpyAsync(&aj, da + j, 8, cudaMemcpyDeviceToHost, st));
        IE_CUDA(cudaStreamSynchronize(st));
        taken = j + 1;
        alphas.push_back(aj);
        const double beta2 = hsc[0];
        if (!(beta2 > 0.0) || !std::isfinite(beta2)) break;  // spectrum.py:169-170
        const double beta = sqrt(beta2);
        k_ritz<<<1, 32, 0, st>>>(da, db, (int)alphas.size(), which, scal.p + 2);
        IE_LAUNCHED();
        IE_CUDA(cudaMemcpyAsync(hsc + 2, scal.p + 2, 8, cudaMemcpyDeviceToHost, st));
        IE_CUDA(cudaStreamSynchronize(st));
        const double cur = hsc[2];
        if (have_est && fabs(cur - est) <= rtol * fmax(fabs(cur), 1.0)) {  // spectrum.py:174-181
            if (++stable >= 5) {
                *lambda = cur;
                if (steps) *steps = taken;
                return IE_OK;
            }
        } else {
            stable = 0;
        }
        est = cur;
        have_est = true;
        if (beta < 1e-14) break;
        betas.push_back(beta);
        IE_CUDA(cudaMemcpyAsync(db + j, &betas.back(), 8, cudaMemcpyHostToDevice, st));
        k_scale_div<<<g1(N), 256, 0, st>>>(V.p + (size_t)(j + 1) * N, wb.p, beta, N);
        IE_LAUNCHED();
        k_scale_div<<<g1(N), 256, 0, st>>>(AV.p + (size_t)(j + 1) * N, awb.p, beta, N);
        IE_LAUNCHED();
        IE_CUDA(cudaStreamSynchronize(st));  // betas.back() must stay alive for the copy
    }
    if (steps) *steps = taken;
    if (!have_est) {
        set_error("Lanczos produced no Ritz values");
        return IE_ERR_NO_RITZ;
    }
    *lambda = est;
    return IE_OK;
}
