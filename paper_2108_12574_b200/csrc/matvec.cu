// K1: matrix-free FP64 kernel matvec (replaces ToeplitzMatvec.matvec,
// /root/reference/pkg/src/iedd/toeplitz.py:39-50, whose entries are
// kernel.py:170-184).
//
// y_i = diag * x_i + sum_{j != i} A_ij x_j,   A_ij = alpha * L(m_ij)
//   dims 1/2: L(m) = log(m s^2) = log(d^2),      alpha = -w/(4 pi)
//   dim 3:    L(m) = m^{-1/2},                   alpha = w/(4 pi s)
// with m_ij = |a_i - a_j|^2 the squared integer lattice distance.  The pair
// loop clamps m to >= 1, so the self pair contributes L(1) x_i, removed in
// the epilogue: y_i = alpha*acc_i + (diag - alpha*L(1)) x_i.
//
// Layout: one thread owns R target rows; a CTA streams the source vector
// through shared memory in tiles of TS points (NRHS doubles each, read as a
// broadcast), and iterates each tile as runs along the last (contiguous)
// lattice axis so the outer-axis distance is hoisted out of the pair loop.
// The log table (16 B entries {c_k, T}) sits in shared memory.  Per-row sums:
// plain FMA chain inside a tile, Neumaier-compensated across tiles, fixed
// split order across CTAs -- identical for any row range and any NRHS.
#include <math.h>
#include <cmath>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "pcg_state.cuh"

namespace ie {

struct MatvecArgs {
    const double* X;
    int64_t ldx;
    double* Y;
    int64_t ldy;
    double* W;  // split partials [split][row][rhs], or null when nsplit == 1
    const LogEntry* tab;
    int ntab;
    int n;
    int N;
    int row_begin;
    int nrows;
    int TS;
    int split_len;
    double alpha;
    double diag;
    const int* stop;  // device flag: nonzero -> no-op (PCG early exit)
};

template <int DIM>
__device__ __forceinline__ double pair_value(const LogEntry* tab, int m) {
    const double md = int_to_double_exact(m);
    if constexpr (DIM == 3) {
        return rsqrt(md);
    } else {
        return log_d2(tab, md);
    }
}

__device__ __forceinline__ void neumaier(double& s, double& c, double v) {
    const double t = s + v;
    c += (fabs(s) >= fabs(v)) ? ((s - t) + v) : ((v - t) + s);
    s = t;
}

// ADJ: a thread's R rows are R consecutive points of one lattice row (the host
// guarantees n % R == 0 and row_begin % R == 0).  Then row r at source t has
// the same squared distance as row r-1 at source t-1, so each source point
// needs ONE kernel evaluation for all R rows: the values slide through a
// register window (R-1 extra evaluations per run of sources).  Every row's
// pair values and summation order are those of the non-ADJ kernel, so the
// result is bitwise identical; the FP64 work per pair drops from 10 to
// 2 + 8/R instructions (2-RHS, dims 1/2).
template <int DIM, int NRHS, int R, bool ADJ = false>
__global__ void __launch_bounds__(256) k_matvec(MatvecArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (a.stop && *a.stop) return;
    LogEntry* stab = reinterpret_cast<LogEntry*>(smem);
    double* xs = reinterpret_cast<double*>(smem + (DIM == 3 ? 0 : a.ntab * (int)sizeof(LogEntry)));
    const int tid = threadIdx.x;
    if constexpr (DIM != 3) {
        for (int t = tid; t < a.ntab; t += blockDim.x) stab[t] = a.tab[t];
    }

    constexpr int NO = DIM > 1 ? DIM - 1 : 1;  // outer axes
    int to[R][NO];
    int tb[R];
    int gi[R];
    bool valid[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int row = ADJ ? (blockIdx.x * blockDim.x + tid) * R + r : blockIdx.x * blockDim.x * R + r * blockDim.x + tid;
        valid[r] = row < a.nrows;
        gi[r] = a.row_begin + (valid[r] ? row : a.nrows - 1);
        int mi[DIM];
        unravel<DIM>(gi[r], a.n, mi);
#pragma unroll
        for (int k = 0; k < NO; ++k) to[r][k] = (DIM > 1) ? mi[k] : 0;
        tb[r] = mi[DIM - 1];
    }

    // Neumaier accumulators (updated once per source tile): registers, or for
    // R >= 16 shared memory [2][R][NRHS][blockDim] after the x tile
    constexpr bool kSmemAcc = R >= 16;
    double s[kSmemAcc ? 1 : R][NRHS], c[kSmemAcc ? 1 : R][NRHS];
    double* sacc = xs + a.TS * NRHS;
    auto S_ = [&](int r, int q) -> double& {
        if constexpr (kSmemAcc) return sacc[((0 * R + r) * NRHS + q) * blockDim.x + tid];
        else return s[r][q];
    };
    auto C_ = [&](int r, int q) -> double& {
        if constexpr (kSmemAcc) return sacc[((1 * R + r) * NRHS + q) * blockDim.x + tid];
        else return c[r][q];
    };
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int q = 0; q < NRHS; ++q) S_(r, q) = C_(r, q) = 0.0;

    const int src0 = blockIdx.y * a.split_len;
    const int src1 = min(a.N, src0 + a.split_len);
    for (int j0 = src0; j0 < src1; j0 += a.TS) {
        const int len = min(a.TS, src1 - j0);
        __syncthreads();
        for (int t = tid; t < len; t += blockDim.x) {
#pragma unroll
            for (int q = 0; q < NRHS; ++q) xs[t * NRHS + q] = a.X[q * a.ldx + j0 + t];
        }
        __syncthreads();

        double ta[R][NRHS];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int q = 0; q < NRHS; ++q) ta[r][q] = 0.0;

        int j = j0;
        while (j < j0 + len) {
            const int outer = j / a.n;
            const int d0 = j - outer * a.n;
            const int L = min(a.n - d0, j0 + len - j);
            int co[NO];
            {
                int o = outer;
#pragma unroll
                for (int k = NO - 1; k >= 0; --k) {
                    co[k] = (DIM > 1) ? o % a.n : 0;
                    o /= a.n;
                }
            }
            int do2[R], db[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                int acc = 0;
#pragma unroll
                for (int k = 0; k < NO; ++k) {
                    const int dd = to[r][k] - co[k];
                    acc += dd * dd;
                }
                do2[r] = acc;
                db[r] = tb[r] - d0;
            }
            const double* xp = xs + (j - j0) * NRHS;
            if constexpr (ADJ) {
                // win[r] = pair value of row r at the current source t
                double win[R];
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    const int dbt = db[0] + r;
                    win[r] = pair_value<DIM>(stab, max(dbt * dbt + do2[0], 1));
                }
#pragma unroll 8
                for (int t = 0; t < L; ++t) {
                    double xv[NRHS];
                    if constexpr (NRHS == 2) {
                        const double2 x2 = reinterpret_cast<const double2*>(xp)[t];
                        xv[0] = x2.x;
                        xv[1] = x2.y;
                    } else {
                        xv[0] = xp[t];
                    }
                    const int dbt = db[0] - t;
                    win[0] = pair_value<DIM>(stab, max(dbt * dbt + do2[0], 1));
#pragma unroll
                    for (int r = 0; r < R; ++r)
#pragma unroll
                        for (int q = 0; q < NRHS; ++q) ta[r][q] = fma(win[r], xv[q], ta[r][q]);
#pragma unroll
                    for (int r = R - 1; r > 0; --r) win[r] = win[r - 1];
                }
                j += L;
                continue;
            }
#pragma unroll 4
            for (int t = 0; t < L; ++t) {
                double xv[NRHS];
                if constexpr (NRHS == 2) {
                    const double2 x2 = reinterpret_cast<const double2*>(xp)[t];
                    xv[0] = x2.x;
                    xv[1] = x2.y;
                } else {
                    xv[0] = xp[t];
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int dbt = db[r] - t;
                    const int m = max(dbt * dbt + do2[r], 1);
                    const double v = pair_value<DIM>(stab, m);
#pragma unroll
                    for (int q = 0; q < NRHS; ++q) ta[r][q] = fma(v, xv[q], ta[r][q]);
                }
            }
            j += L;
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int q = 0; q < NRHS; ++q) neumaier(S_(r, q), C_(r, q), ta[r][q]);
    }

    if (a.W != nullptr) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (!valid[r]) continue;
            const int row = gi[r] - a.row_begin;
#pragma unroll
            for (int q = 0; q < NRHS; ++q)
                a.W[((int64_t)blockIdx.y * a.nrows + row) * NRHS + q] = S_(r, q) + C_(r, q);
        }
        return;
    }
    const double lself = pair_value<DIM>(stab, 1);
    const double corr = a.diag - a.alpha * lself;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (!valid[r]) continue;
        const int row = gi[r] - a.row_begin;
#pragma unroll
        for (int q = 0; q < NRHS; ++q) {
            const double xi = a.X[q * a.ldx + gi[r]];
            a.Y[q * a.ldy + row] = fma(a.alpha, S_(r, q) + C_(r, q), corr * xi);
        }
    }
}

// Sum split partials in split order and apply the epilogue.
template <int DIM, int NRHS>
__global__ void k_matvec_reduce(MatvecArgs a, int nsplit) {
    if (a.stop && *a.stop) return;
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= a.nrows) return;
    double lself;
    if constexpr (DIM == 3) {
        lself = rsqrt(1.0);
    } else {
        lself = log_d2(a.tab, 1.0);
    }
    const double corr = a.diag - a.alpha * lself;
    const int gi = a.row_begin + row;
#pragma unroll
    for (int q = 0; q < NRHS; ++q) {
        double acc = 0.0;
        for (int sp = 0; sp < nsplit; ++sp) acc += a.W[((int64_t)sp * a.nrows + row) * NRHS + q];
        a.Y[q * a.ldy + row] = fma(a.alpha, acc, corr * a.X[q * a.ldx + gi]);
    }
}

}  // namespace ie

// ------------------------------------------------------------- host side --
struct ie_fft;
namespace ie {
int fft_create(const ie_geom& g, ie_fft** out);
void fft_destroy(ie_fft* f);
int fft_matvec(const ie_fft* f, const double* X0, const double* X1, double* Y0, double* Y1, cudaStream_t st,
               const int* stop, const double* scales, double2* buf_ws, double* amax_ws, const PcgFuse* fz);
bool fft_fusable(const ie_fft* f);
int fft_out_lines(const ie_fft* f);
int64_t fft_buf_elems(const ie_fft* f);
int fft_band_fwd(const ie_fft* f, const double* X0, const double* X1, int nrows, int parts, double2* out,
                 const double* scales, cudaStream_t st, const int* stop = nullptr, const PeerStores* ps = nullptr);
int fft_band_cols(const ie_fft* f, double2* buf, int c0, int ncols, cudaStream_t st, const int* stop = nullptr,
                  const PeerStores* ps = nullptr);
int fft_band_inv(const ie_fft* f, const double2* in, int nrows, int parts, double* Y0, double* Y1,
                 const double* scales, cudaStream_t st, const int* stop = nullptr, const PcgFuse* fz = nullptr);
int fft_absmax2(const double* X0, const double* X1, int64_t N, double* part, cudaStream_t st);
}  // namespace ie

struct ie_matvec {
    ie_geom g;
    uint64_t uid;   // unique per handle (graph cache key)
    int method;     // IE_MATVEC_DIRECT / IE_MATVEC_FFT
    ie_fft* fft;    // FFT plan (method FFT)
    double* d_full; // FFT path: full-range output for partial row requests
    int N;
    ie::LogEntry* d_tab;
    int ntab;
    double alpha;
    // launch plan (depends on N only -> bitwise identical for any row range)
    int R;
    int TS;
    int split_len;
    int nsplit;
    double* d_work;  // split partials, nsplit * N * 2 doubles
    // per-stream scratch (FFT work buffer + chunk maxima, partial-range output,
    // K1 split partials): the plan's own buffers belong to the first stream
    // that uses the handle, other streams get their own
    struct Ws {
        double2* buf = nullptr;
        double* amax = nullptr;
        double* full = nullptr;
        double* work = nullptr;
    };
    std::mutex ws_mu;
    bool ws0_claimed = false;
    cudaStream_t ws0_stream = nullptr;
    std::vector<std::pair<cudaStream_t, Ws>> ws_extra;
};

namespace ie {

// Host-side log table in 80-bit arithmetic (see common.cuh).
std::vector<LogEntry> build_log_table(const ie_geom& g, int* ntab_out) {
    const long double s = (long double)g.spacing;
    const long long mmax = (long long)g.dim * (long long)(g.n - 1) * (long long)(g.n - 1);
    int emax = 0;
    while ((1LL << (emax + 1)) <= mmax) ++emax;
    const int ntab = (emax + 1) * kLogK;
    std::vector<LogEntry> tab(ntab);
    const long double ln2 = 0.693147180559945309417232121458176568L;
    const long double two_log_s = 2.0L * logl(s);
    for (int e = 0; e <= emax; ++e) {
        for (int k = 0; k < kLogK; ++k) {
            const double ck = 128.0 / (128.5 + (double)k);  // rounded once
            const long double t = (long double)e * ln2 - logl((long double)ck) + two_log_s;
            tab[e * kLogK + k] = LogEntry{ck, (double)t};
        }
    }
    *ntab_out = ntab;
    return tab;
}

EntryParams entry_params(const ie_geom& g) {
    EntryParams P;
    P.dim = g.dim;
    P.diag = g.diag;
    const double four_pi = 4.0 * M_PI;
    P.alpha = (g.dim == 3) ? g.weight / (four_pi * g.spacing) : -g.weight / four_pi;
    return P;
}

int make_log_table_device(const ie_geom& g, LogEntry** d_tab, int* ntab) {
    std::vector<LogEntry> tab = build_log_table(g, ntab);
    IE_CUDA(cudaMalloc(d_tab, tab.size() * sizeof(LogEntry)));
    IE_CUDA(cudaMemcpy(*d_tab, tab.data(), tab.size() * sizeof(LogEntry), cudaMemcpyHostToDevice));
    return IE_OK;
}

template <int DIM, int NRHS>
static int launch_dim(const ie_matvec* m, MatvecArgs a, cudaStream_t st) {
    const size_t smem = (DIM == 3 ? 0 : (size_t)m->ntab * sizeof(LogEntry)) + (size_t)m->TS * NRHS * sizeof(double) +
                        (m->R >= 16 ? (size_t)2 * m->R * NRHS * 256 * sizeof(double) : 0);
    const int threads = 256;
    dim3 grid((a.nrows + threads * m->R - 1) / (threads * m->R), m->nsplit);
    a.W = m->nsplit > 1 ? a.W : nullptr;  // the stream's split partials (matvec_launch)
    // adjacent-row variant when each thread's R rows share a lattice row
    const bool adj = m->R > 1 && m->g.n % m->R == 0 && a.row_begin % m->R == 0 && !getenv("IEDD_B200_K1_NOADJ");
    if (m->R == 16) {
        auto kern = adj ? k_matvec<DIM, NRHS, 16, true> : k_matvec<DIM, NRHS, 16, false>;
        IE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, threads, smem, st>>>(a);
    } else if (m->R == 8) {
        auto kern = adj ? k_matvec<DIM, NRHS, 8, true> : k_matvec<DIM, NRHS, 8, false>;
        IE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, threads, smem, st>>>(a);
    } else if (m->R == 4) {
        auto kern = adj ? k_matvec<DIM, NRHS, 4, true> : k_matvec<DIM, NRHS, 4, false>;
        IE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, threads, smem, st>>>(a);
    } else if (m->R == 2) {
        auto kern = adj ? k_matvec<DIM, NRHS, 2, true> : k_matvec<DIM, NRHS, 2, false>;
        IE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, threads, smem, st>>>(a);
    } else {
        auto kern = k_matvec<DIM, NRHS, 1>;
        IE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, threads, smem, st>>>(a);
    }
    IE_LAUNCHED();
    if (m->nsplit > 1) {
        k_matvec_reduce<DIM, NRHS><<<(a.nrows + 255) / 256, 256, 0, st>>>(a, m->nsplit);
        IE_LAUNCHED();
    }
    return IE_OK;
}

static ie_matvec::Ws mv_ws(ie_matvec* m, cudaStream_t st, bool* ok) {
    std::lock_guard<std::mutex> lk(m->ws_mu);
    *ok = true;
    if (!m->ws0_claimed) {
        m->ws0_claimed = true;
        m->ws0_stream = st;
    }
    ie_matvec::Ws own;
    own.buf = nullptr;   // fft_matvec: the plan's own buffer
    own.amax = nullptr;
    own.full = m->d_full;
    own.work = m->d_work;
    if (st == m->ws0_stream) return own;
    for (auto& e : m->ws_extra)
        if (e.first == st) return e.second;
    ie_matvec::Ws w;
    bool good = true;
    if (m->fft) {
        good = good && cudaMalloc(&w.buf, (size_t)fft_buf_elems(m->fft) * sizeof(double2)) == cudaSuccess;
        good = good && cudaMalloc(&w.amax, 2 * (size_t)((m->N + 2047) / 2048) * sizeof(double)) == cudaSuccess;
        good = good && cudaMalloc(&w.full, 2 * (size_t)m->N * sizeof(double)) == cudaSuccess;
    }
    if (good && m->d_work)
        good = cudaMalloc(&w.work, (size_t)m->nsplit * m->N * 2 * sizeof(double)) == cudaSuccess;
    if (!good) {
        cudaFree(w.buf);
        cudaFree(w.amax);
        cudaFree(w.full);
        cudaFree(w.work);
        cudaGetLastError();
        set_error("matvec: out of device memory for a per-stream workspace");
        *ok = false;
        return ie_matvec::Ws{};
    }
    m->ws_extra.emplace_back(st, w);
    return w;
}

// The stream's FFT work buffer (null for the direct sum): between two A-passes
// on that stream nothing in it is live, so the PCG lends it to the apply as
// its staging buffer (one working set less in the L2).
double* matvec_scratch(const ie_matvec* m, cudaStream_t st, size_t* bytes) {
    *bytes = 0;
    if (m->method != IE_MATVEC_FFT) return nullptr;
    bool ok;
    const ie_matvec::Ws W = mv_ws(const_cast<ie_matvec*>(m), st, &ok);
    if (!ok || !W.buf) return nullptr;
    *bytes = (size_t)fft_buf_elems(m->fft) * sizeof(double2);
    return reinterpret_cast<double*>(W.buf);
}

// Allocate the stream's matvec scratch now (before a graph capture on it).
int matvec_prepare_stream(const ie_matvec* m, cudaStream_t st) {
    bool ok;
    mv_ws(const_cast<ie_matvec*>(m), st, &ok);
    return ok ? IE_OK : IE_ERR_CUDA;
}

int matvec_launch(const ie_matvec* m, const double* X, int64_t ldx, int nrhs, double* Y, int64_t ldy,
                  int64_t row_begin, int64_t row_end, cudaStream_t st, const int* stop, const double* scales,
                  const PcgFuse* fz) {
    bool ok;
    const ie_matvec::Ws W = mv_ws(const_cast<ie_matvec*>(m), st, &ok);
    if (!ok) return IE_ERR_CUDA;
    if (m->method == IE_MATVEC_FFT) {
        const double* X1 = nrhs == 2 ? X + ldx : nullptr;
        if (row_begin == 0 && row_end == m->N)
            return fft_matvec(m->fft, X, X1, Y, nrhs == 2 ? Y + ldy : nullptr, st, stop, scales, W.buf, W.amax, fz);
        int rc = fft_matvec(m->fft, X, X1, W.full, nrhs == 2 ? W.full + m->N : nullptr, st, stop, scales, W.buf,
                            W.amax, nullptr);
        if (rc) return rc;
        for (int q = 0; q < nrhs; ++q)
            IE_CUDA(cudaMemcpyAsync(Y + q * ldy, W.full + (int64_t)q * m->N + row_begin,
                                    (row_end - row_begin) * sizeof(double), cudaMemcpyDeviceToDevice, st));
        return IE_OK;
    }
    MatvecArgs a;
    a.X = X;
    a.ldx = ldx;
    a.Y = Y;
    a.ldy = ldy;
    a.W = W.work;
    a.tab = m->d_tab;
    a.ntab = m->ntab;
    a.n = m->g.n;
    a.N = m->N;
    a.row_begin = (int)row_begin;
    a.nrows = (int)(row_end - row_begin);
    a.TS = m->TS;
    a.split_len = m->split_len;
    a.alpha = m->alpha;
    a.diag = m->g.diag;
    a.stop = stop;
    if (a.nrows <= 0) return IE_OK;
    switch (m->g.dim * 4 + nrhs) {
        case 1 * 4 + 1: return launch_dim<1, 1>(m, a, st);
        case 1 * 4 + 2: return launch_dim<1, 2>(m, a, st);
        case 2 * 4 + 1: return launch_dim<2, 1>(m, a, st);
        case 2 * 4 + 2: return launch_dim<2, 2>(m, a, st);
        case 3 * 4 + 1: return launch_dim<3, 1>(m, a, st);
        case 3 * 4 + 2: return launch_dim<3, 2>(m, a, st);
    }
    set_error("matvec: dim must be 1..3 and nrhs 1..2");
    return IE_ERR_ARG;
}

// ---------------------------------------------------- assemble_block ----
__global__ void k_assemble(int dim, int n, EntryParams P, const LogEntry* tab, const int64_t* rows,
                           int64_t nr, const int64_t* cols, int64_t nc, double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nr * nc) return;
    int64_t i = rows[e / nc], j = cols[e % nc];
    int m = 0;
    for (int d = 0; d < dim; ++d) {
        const int dd = (int)(i % n) - (int)(j % n);
        m += dd * dd;
        i /= n;
        j /= n;
    }
    out[e] = entry_from_m(P, tab, m);
}

}  // namespace ie

extern "C" int ie_matvec_create(const ie_geom* g, ie_matvec** out) {
    return ie_matvec_create_method(g, IE_MATVEC_DIRECT, out);
}

extern "C" int ie_matvec_create_method(const ie_geom* g, int32_t method, ie_matvec** out) {
    if (!g || !out || g->dim < 1 || g->dim > 3 || g->n < 2 || (method != IE_MATVEC_DIRECT && method != IE_MATVEC_FFT)) {
        ie::set_error("ie_matvec_create: bad geometry");
        return IE_ERR_ARG;
    }
    const double Nd = pow((double)g->n, g->dim);
    if (Nd >= 2147483647.0) {
        ie::set_error("ie_matvec_create: N must be < 2^31");
        return IE_ERR_ARG;
    }
    ie_matvec* m = new ie_matvec();
    m->g = *g;
    static std::atomic<uint64_t> next_uid{1};
    m->uid = next_uid.fetch_add(1);
    m->N = (int)Nd;
    m->method = method;
    m->fft = nullptr;
    m->d_full = nullptr;
    if (method == IE_MATVEC_FFT) {
        int rc = ie::fft_create(*g, &m->fft);
        if (rc) {
            delete m;
            return rc;
        }
        cudaError_t e = cudaMalloc(&m->d_full, 2 * (size_t)m->N * sizeof(double));
        if (e != cudaSuccess) {
            ie::set_error(cudaGetErrorString(e));
            ie::fft_destroy(m->fft);
            delete m;
            return IE_ERR_CUDA;
        }
    }
    m->alpha = ie::entry_params(*g).alpha;
    int rc = ie::make_log_table_device(*g, &m->d_tab, &m->ntab);
    if (rc) {
        delete m;
        return rc;
    }
    // Launch plan from N only.
    const int N = m->N;
    // rows per thread: more rows share each kernel evaluation (ADJ window); at
    // R = 16 the Neumaier accumulators move to shared memory (R = 32 spills).
    // 2-RHS pass, R = 2 -> 16: config 5 944 -> 242 ms, 2D n=256 4.6 -> 1.0 ms,
    // 3D n=32 0.66 -> 0.35 ms; the launch-bound small sizes prefer 1-2
    m->R = N >= 16384 ? 16 : (N >= 4096 ? 2 : 1);
    m->TS = N >= 65536 ? 1024 : 256;
    const int tiles = (N + m->TS - 1) / m->TS;
    const int ctas = (N + 256 * m->R - 1) / (256 * m->R);
    int nsplit = (4 * ie::kNumSMs + ctas - 1) / ctas;
    if (nsplit > tiles) nsplit = tiles;
    if (nsplit < 1) nsplit = 1;
    if (m->R == 16 && !getenv("IEDD_B200_K1_SPLIT_V1")) {
        // R = 16 keeps one CTA per SM resident (190 KB of shared memory), so the
        // grid runs in rounds of kNumSMs CTAs: pick the split count whose last
        // round is fullest -- on one GPU (weight 0.55) and for the row bands of
        // 2, 4 and 8 ranks (the plan may depend on N only: every rank and every G
        // must sum the same splits in the same order).  Config 5: 256 row CTAs x
        // 3 splits = 5.19 rounds ran as 6 (ncu: 242.6 ms, FP64 pipe 71% busy);
        // x 23 = 39.78 rounds run as 40 (211.4 ms), 19.89 / 9.95 / 4.97 on the
        // bands of 2 / 4 / 8 ranks.
        auto eff = [&](int ns, int G) {
            const double rounds = (double)((ctas + G - 1) / G) * ns / ie::kNumSMs;
            return rounds / std::ceil(rounds);
        };
        double best = -1.0;
        int best_ns = nsplit;
        for (int tps = tiles; tps >= 1; --tps) {
            const int ns = (tiles + tps - 1) / tps;
            if (ns > 32) break;
            const double score = 0.55 * eff(ns, 1) + 0.15 * (eff(ns, 2) + eff(ns, 4) + eff(ns, 8)) - 0.0005 * ns;
            if (score > best) {
                best = score;
                best_ns = ns;
            }
        }
        nsplit = best_ns;
        if (const char* e = getenv("IEDD_B200_K1_NSPLIT")) nsplit = std::max(1, std::min(atoi(e), tiles));
    }
    const int tiles_per_split = (tiles + nsplit - 1) / nsplit;
    m->split_len = tiles_per_split * m->TS;
    m->nsplit = (N + m->split_len - 1) / m->split_len;
    m->d_work = nullptr;
    if (m->nsplit > 1) {
        cudaError_t e = cudaMalloc(&m->d_work, (size_t)m->nsplit * N * 2 * sizeof(double));
        if (e != cudaSuccess) {
            ie::set_error(std::string("ie_matvec_create: ") + cudaGetErrorString(e));
            cudaFree(m->d_tab);
            delete m;
            return IE_ERR_CUDA;
        }
    }
    *out = m;
    return IE_OK;
}

extern "C" void ie_matvec_destroy(ie_matvec* m) {
    if (!m) return;
    if (m->fft) ie::fft_destroy(m->fft);
    if (m->d_full) cudaFree(m->d_full);
    cudaFree(m->d_tab);
    if (m->d_work) cudaFree(m->d_work);
    for (auto& e : m->ws_extra) {
        cudaFree(e.second.buf);
        cudaFree(e.second.amax);
        cudaFree(e.second.full);
        cudaFree(e.second.work);
    }
    delete m;
}

extern "C" int ie_matvec_f64(const ie_matvec* m, const double* X, int64_t ldx, int32_t nrhs, double* Y,
                             int64_t ldy, int64_t row_begin, int64_t row_end, void* stream) {
    if (!m || !X || !Y || nrhs < 1 || nrhs > 2 || row_begin < 0 || row_end > m->N || row_begin > row_end ||
        ldx < m->N || ldy < row_end - row_begin) {
        ie::set_error("ie_matvec_f64: bad arguments");
        return IE_ERR_ARG;
    }
    return ie::matvec_launch(m, X, ldx, nrhs, Y, ldy, row_begin, row_end, (cudaStream_t)stream, nullptr, nullptr,
                             nullptr);
}

// ---- band (slab) passes of the FFT method, for the sharded solver
static bool band_ok(const ie_matvec* m, int64_t row_begin, int64_t row_end, int32_t parts, int32_t nrhs) {
    if (!m || m->method != IE_MATVEC_FFT || m->g.dim != 2 || nrhs < 1 || nrhs > 2 || parts < 1 || row_begin < 0 ||
        row_end > m->N || row_begin > row_end || row_begin % m->g.n || row_end % m->g.n) {
        ie::set_error("band FFT pass: FFT operator in 2D, whole grid rows, nrhs in {1, 2}");
        return false;
    }
    return true;
}

extern "C" int ie_matvec_band_fwd_f64(const ie_matvec* m, const double* X, int64_t ldx, int32_t nrhs,
                                      int64_t row_begin, int64_t row_end, int32_t parts, void* out,
                                      const double* scales, void* stream) {
    if (!band_ok(m, row_begin, row_end, parts, nrhs) || !X || !out || ldx < row_end - row_begin ||
        (nrhs == 2 && !scales)) {
        if (m && X && out) ie::set_error("ie_matvec_band_fwd_f64: bad arguments");
        return IE_ERR_ARG;
    }
    const int nrows = (int)((row_end - row_begin) / m->g.n);
    if (!nrows) return IE_OK;
    return ie::fft_band_fwd(m->fft, X, nrhs == 2 ? X + ldx : nullptr, nrows, parts, (double2*)out, scales,
                            (cudaStream_t)stream);
}

extern "C" int ie_matvec_band_cols_f64(const ie_matvec* m, void* buf, int64_t col_begin, int64_t col_end,
                                       void* stream) {
    if (!band_ok(m, 0, 0, 1, 1) || !buf || col_begin < 0 || col_end <= col_begin) {
        ie::set_error("ie_matvec_band_cols_f64: bad arguments");
        return IE_ERR_ARG;
    }
    return ie::fft_band_cols(m->fft, (double2*)buf, (int)col_begin, (int)(col_end - col_begin), (cudaStream_t)stream);
}

extern "C" int ie_matvec_band_inv_f64(const ie_matvec* m, const void* in, int64_t row_begin, int64_t row_end,
                                      int32_t parts, double* Y, int64_t ldy, int32_t nrhs, const double* scales,
                                      void* stream) {
    if (!band_ok(m, row_begin, row_end, parts, nrhs) || !in || !Y || ldy < row_end - row_begin ||
        (nrhs == 2 && !scales)) {
        if (m && in && Y) ie::set_error("ie_matvec_band_inv_f64: bad arguments");
        return IE_ERR_ARG;
    }
    const int nrows = (int)((row_end - row_begin) / m->g.n);
    if (!nrows) return IE_OK;
    return ie::fft_band_inv(m->fft, (const double2*)in, nrows, parts, Y, nrhs == 2 ? Y + ldy : nullptr, scales,
                            (cudaStream_t)stream);
}

extern "C" int ie_absmax_partials_f64(const double* X, int64_t ldx, int64_t n, double* out, void* stream) {
    if (!X || !out || n < 0 || (ldx < n && ldx != 0)) {  // ldx 0: both columns are x0
        ie::set_error("ie_absmax_partials_f64: bad arguments");
        return IE_ERR_ARG;
    }
    return ie::fft_absmax2(X, X + ldx, n, out, (cudaStream_t)stream);
}

extern "C" int ie_assemble_block_f64(const ie_geom* g, const int64_t* rows, int64_t nr, const int64_t* cols,
                                     int64_t nc, double* out, void* stream) {
    if (!g || g->dim < 1 || g->dim > 3 || nr < 0 || nc < 0) {
        ie::set_error("ie_assemble_block_f64: bad arguments");
        return IE_ERR_ARG;
    }
    if (nr == 0 || nc == 0) return IE_OK;
    ie::LogEntry* tab;
    int ntab;
    int rc = ie::make_log_table_device(*g, &tab, &ntab);
    if (rc) return rc;
    const int64_t tot = nr * nc;
    ie::k_assemble<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        g->dim, g->n, ie::entry_params(*g), tab, rows, nr, cols, nc, out);
    cudaError_t e = cudaGetLastError();
    ie::g_launches.fetch_add(1);
    cudaStreamSynchronize((cudaStream_t)stream);
    cudaFree(tab);
    if (e != cudaSuccess) {
        ie::set_error(cudaGetErrorString(e));
        return IE_ERR_CUDA;
    }
    return IE_OK;
}

namespace ie {
int matvec_N(const ie_matvec* m) { return m->N; }
// lines of the A-pass's last transform when the PCG driver may fold k_iter_b /
// k_post_pass into the FFT passes (full-range 2D / 3D FFT plans), else 0
int matvec_fused_lines(const ie_matvec* m) {
    return (m->method == IE_MATVEC_FFT && fft_fusable(m->fft)) ? fft_out_lines(m->fft) : 0;
}
uint64_t matvec_uid(const ie_matvec* m) { return m->uid; }
const ie_fft* matvec_fft(const ie_matvec* m) { return m->method == IE_MATVEC_FFT ? m->fft : nullptr; }
int matvec_dim(const ie_matvec* m) { return m->g.dim; }
int matvec_n(const ie_matvec* m) { return m->g.n; }
}  // namespace ie
