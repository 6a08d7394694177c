// K1b: O(N log N) matvec by circulant embedding -- the reference's own
// algorithm (ToeplitzMatvec, /root/reference/pkg/src/iedd/toeplitz.py:11-53;
// generator kernel.py:190-199), hand-written for sm_100a in FP64.
//
//  * The (2n)^d embedding of the generator is mirror-even on every axis, so
//    its DFT (the symbol) is real and even: stored folded, (n+1)^d doubles,
//    pre-scaled by 1/(2n)^d (numpy's irfftn normalisation).
//  * The operator is real, so two right-hand sides ride in one complex
//    transform: z = x0 + i x1  ->  IFFT(sym * FFT(z)) = A x0 + i A x1.  The
//    PCG 2-RHS pass [p_k, u_{k-1}] costs one complex round trip.
//  * Zero padding is exploited: axis transforms only touch lines whose
//    not-yet-transformed coordinates are < n, and the last forward axis-0
//    transform, the symbol multiply and the first inverse transform are one
//    fused kernel per line (the spectrum never round-trips HBM).
//  * Each CTA (256 threads; 32 for small transforms) runs a self-sorting
//    Stockham FFT over 4096 complex points in shared memory -- 4096/M lines
//    of length M = 2n <= 4096: radix-16 passes with 16 points per thread in
//    registers, then one radix 8/4/2 pass; split re/im arrays padded one slot
//    per 16 with a per-line skew (conflict-free), radix-major twiddle tables
//    staged by cp.async while the lines load.
//  * The exact power-of-two column scaling keeps the rounding of the small
//    column (PCG's u vs p differ by up to ~1e10) independent of the large one.
//  * Band variants (fft_band_*) split the 2D pass across ranks around two
//    all-to-all transposes (sharded solver).
#include <math.h>
#include <stdlib.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "pcg_state.cuh"

namespace ie {

constexpr int kFftPoints = 4096;     // points per CTA of the radix-16 k_fft_lines (lines M < 64)
constexpr int kFftMaxPoints = 8192;  // longest line (k_fft8: 8 points x 1024 threads)

struct LineArgs {
    int nlines;   // lines in this pass
    int ninner;   // line g -> o = g / ninner, i = g % ninner
    int lg_ninner;  // log2(ninner), or -1 when ninner is not a power of two (3D, non-power-of-two n)
    int L;
    int logL;
    // source
    int in_real;  // 1: real pair x0 (+ i x1); 0: complex buffer
    const double2* in_c;
    const double* x0;
    const double* x1;
    int64_t in_so, in_si, in_sl;
    int in_lsplit;   // >= 0: l = (l >> in_lsplit) blocks of stride in_sh (band layouts); -1: none
    int64_t in_sh;
    int n_in;     // l >= n_in reads as zero
    // destination
    int out_real;
    double2* out_c;
    double* y0;
    double* y1;
    int64_t out_so, out_si, out_sl;
    int out_lsplit;
    int64_t out_sh;
    int n_out;    // only l < n_out is written
    int line0;    // global index of line 0 along the symbol axis (band column pass)
    int sign;     // -1 forward, +1 inverse (ignored when fused)
    int fused;    // forward, * symbol, inverse
    const double* sym;
    int dim;
    int n;
    const double2* tw;  // tw[m] = exp(-2 pi i m / L)
    // exact power-of-two column scaling for 2-RHS packing: input columns are
    // multiplied by 2^-e_c (max|x_c| ~ 1) and outputs by 2^e_c, so the
    // rounding of one column never contaminates the other (PCG's p and u
    // differ by up to ~1e10 in norm).  amax = per-chunk partial max|x_c|.
    const double* amax;
    int namax;
    // or the two multipliers themselves, precomputed by the PCG driver
    // (k_iter_b: one device-side decision instead of a partial-max
    // reduction in every CTA); takes precedence over amax
    const double* scales;
    int scale_in;
    int scale_out;
    const int* stop;  // device flag: nonzero -> no-op (PCG early exit)
    // k_fft8 (radix-8, 8 points per thread): per-pass radix-major twiddles,
    // lines per CTA, strided (column) thread mapping, per-line smem pitch
    const double2* tw8;
    const double2* tw16;  // 16-point plan twiddles (L = 2048)
    int pts;              // points per thread of the k_fft8 launch (8 or 16)
    int g8;
    int strided8;
    int pitch8;
    // strided fused column pass with TMA tile I/O: the buffer as a 2D FP64
    // tensor (4n doubles per row, n rows), boxes of {2 G doubles, 256 rows}
    int tma;
    CUtensorMap tmap;
    // PCG fusions of the single-GPU driver (krylov.cu), contiguous row lines:
    //  kFwdRCUpd (the first pass of a 2-RHS A-pass, x0 = p, x1 = u): k_iter_b's
    //    vector half folded in -- p_new = z + beta p_old stored back to x0
    //    with beta and the 2-RHS multipliers from the state (the decider in
    //    the previous apply's scatter fixed them), max|p_new| into the
    //    rotating slot upd_pglob[it % 3] (upd_it < 0: graph replay, the
    //    iteration from the state).
    //  kInvCRPost (the last pass): k_post_pass folded in -- per output line,
    //    p.q (post_q_col: the output column holding q) and |f - w|^2
    //    (post_w_col) -> post_part[2 (post_line0 + line)], [.. + 1].
    const double* upd_z;
    double* upd_pglob;
    int post_skip_w;  // PcgFuse::skip_w_store
    PcgState* upd_s;
    long long upd_it;
    const double* post_p;
    const double* post_f;
    double* post_part;
    int post_line0;
    int post_lo, post_hi;
    int post_q_col;
    int post_w_col;
    // Sharded transposes folded into the band passes' stores (krylov.cu
    // ie_pcg_sharded_*): the complex outputs go straight into the peers'
    // memory over NVLink, and every CTA release-adds its bytes to each peer's
    // mailbox counter after its stores.
    //  peer_mode 1 (band rows forward, FWD): output column l belongs to slab
    //    h = l >> out_lsplit; element (line o, l) -> peer[h] + o out_so +
    //    (l & (2^out_lsplit - 1)) out_sl (peer[h] already offset to the
    //    sender's rows); every line sends peer_line_bytes[h] to each peer;
    //  peer_mode 2 (column slab, BACK): output row l goes to every rank h whose
    //    need rows [peer_rlo[h], peer_rhi[h]) contain it (the owner l /
    //    peer_band_rows and its two neighbours' halos): peer[h] + (l -
    //    peer_rlo[h]) out_sl + i (peer[h] offset to the sender's slab block).
    int peer_mode;
    int npeer;
    int peer_band_rows;
    double2* peer[16];
    unsigned long long* peer_ctr[16];
    long long peer_line_bytes[16];
    int peer_rlo[16], peer_rhi[16];
    // sharded POST exchange folded into kInvCRPost: the line partials also go
    // to every peer's array (same index), then the CTA's bytes to its mailbox
    int post_npeer;
    double* post_peer[16];
    unsigned long long* post_ctr[16];
};

// 2^-e with 2^e >= max|x| (power of two, exact); 1 for max == 0
__device__ __forceinline__ double pow2_scale(double mx) {
    if (!(mx > 0.0) || !isfinite(mx)) return 1.0;
    int e;
    frexp(mx, &e);
    return ldexp(1.0, -e);
}

// 1 / c when x * (1 / c) rounds exactly as x / c for every x: c a normal power
// of two (its reciprocal is then exact); 0 otherwise (callers divide)
// (c = +2^(ex - 1023), ex in [1, 2045]: 1 / c = 2^(1023 - ex), biased exponent 2046 - ex)
__device__ __forceinline__ double exact_recip(double c) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(c);
    const unsigned ex = (unsigned)(b >> 52);  // sign bit included: negative c -> 0
    return ((b & 0xfffffffffffffull) == 0 && ex >= 1u && ex <= 2045u)
               ? __longlong_as_double((long long)(2046ull - ex) << 52)
               : 0.0;
}

template <int TPB>
__device__ void column_scales(const LineArgs& a, double* sc) {
    if (a.scales) {
        if (threadIdx.x < 2) sc[threadIdx.x] = a.scales[threadIdx.x];
        __syncthreads();
        return;
    }
    __shared__ double red[2][TPB];
    double m0 = 0.0, m1 = 0.0;
    for (int c = threadIdx.x; c < a.namax; c += blockDim.x) {
        m0 = fmax(m0, a.amax[2 * c]);
        m1 = fmax(m1, a.amax[2 * c + 1]);
    }
    red[0][threadIdx.x] = m0;
    red[1][threadIdx.x] = m1;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            red[0][threadIdx.x] = fmax(red[0][threadIdx.x], red[0][threadIdx.x + o]);
            red[1][threadIdx.x] = fmax(red[1][threadIdx.x], red[1][threadIdx.x + o]);
        }
        __syncthreads();
    }
    sc[0] = pow2_scale(red[0][0]);
    sc[1] = pow2_scale(red[1][0]);
}

// per-2048-chunk max|x0|, max|x1|
__global__ void k_absmax2(const double* x0, const double* x1, int N, double* part, const int* stop) {
    if (stop && *stop) return;
    __shared__ double r0[256], r1[256];
    const int base = blockIdx.x * 2048;
    double m0 = 0.0, m1 = 0.0;
    for (int e = 0; e < 8; ++e) {
        const int i = base + e * 256 + threadIdx.x;
        if (i < N) {
            m0 = fmax(m0, fabs(x0[i]));
            m1 = fmax(m1, fabs(x1[i]));
        }
    }
    r0[threadIdx.x] = m0;
    r1[threadIdx.x] = m1;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            r0[threadIdx.x] = fmax(r0[threadIdx.x], r0[threadIdx.x + o]);
            r1[threadIdx.x] = fmax(r1[threadIdx.x], r1[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = r0[0];
        part[2 * blockIdx.x + 1] = r1[0];
    }
}

// ---------------------------------------------------------------------------
// In-register DFTs of size 2, 4, 8, 16 (natural order in and out).
// sign = -1: exp(-2 pi i jk/R) (forward), +1: inverse.
template <int S>
__device__ __forceinline__ void dft2(double& ar, double& ai, double& br, double& bi) {
    const double tr = ar - br, ti = ai - bi;
    ar += br;
    ai += bi;
    br = tr;
    bi = ti;
}

// (x_r + i x_i) * exp(S * 2 pi i m / 16), m a compile-time constant
template <int S, int M>
__device__ __forceinline__ void rot16(double& xr, double& xi) {
    constexpr int m = M & 15;
    if constexpr (m == 0) {
        return;
    } else if constexpr (m == 4) {  // * (S i)
        const double t = xr;
        xr = -S * xi;
        xi = S * t;
    } else if constexpr (m == 8) {
        xr = -xr;
        xi = -xi;
    } else if constexpr (m == 12) {  // * (-S i)
        const double t = xr;
        xr = S * xi;
        xi = -S * t;
    } else {
        constexpr double C[16] = {1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508977, 0.0,
                                  -0.38268343236508977, -0.70710678118654752, -0.92387953251128674, -1.0,
                                  -0.92387953251128674, -0.70710678118654752, -0.38268343236508977, 0.0,
                                  0.38268343236508977, 0.70710678118654752, 0.92387953251128674};
        constexpr double Sn[16] = {0.0, 0.38268343236508977, 0.70710678118654752, 0.92387953251128674, 1.0,
                                   0.92387953251128674, 0.70710678118654752, 0.38268343236508977, 0.0,
                                   -0.38268343236508977, -0.70710678118654752, -0.92387953251128674, -1.0,
                                   -0.92387953251128674, -0.70710678118654752, -0.38268343236508977};
        constexpr double c = C[m], sn = S * Sn[m];
        const double t = xr;
        xr = fma(t, c, -xi * sn);
        xi = fma(t, sn, xi * c);
    }
}

// DFT4 on (x0,x1,x2,x3) in place, natural order
template <int S>
__device__ __forceinline__ void dft4(double* r, double* i, int a0, int a1, int a2, int a3) {
    const double s0r = r[a0] + r[a2], s0i = i[a0] + i[a2];
    const double d0r = r[a0] - r[a2], d0i = i[a0] - i[a2];
    const double s1r = r[a1] + r[a3], s1i = i[a1] + i[a3];
    const double d1r = r[a1] - r[a3], d1i = i[a1] - i[a3];
    // (d1) * (S i)
    const double er = -S * d1i, ei = S * d1r;
    r[a0] = s0r + s1r;
    i[a0] = s0i + s1i;
    r[a2] = s0r - s1r;
    i[a2] = s0i - s1i;
    r[a1] = d0r + er;
    i[a1] = d0i + ei;
    r[a3] = d0r - er;
    i[a3] = d0i - ei;
}

template <int R, int S>
__device__ __forceinline__ void dft_reg(double* r, double* i) {
    if constexpr (R == 2) {
        dft2<S>(r[0], i[0], r[1], i[1]);
    } else if constexpr (R == 4) {
        dft4<S>(r, i, 0, 1, 2, 3);
    } else if constexpr (R == 8) {
        // n = 2 n1 + n2: DFT4 over n1, twiddle w8^(n2 k1) = w16^(2 n2 k1), DFT2 over n2; X[k1 + 4 k2]
        dft4<S>(r, i, 0, 2, 4, 6);
        dft4<S>(r, i, 1, 3, 5, 7);
        rot16<S, 2>(r[3], i[3]);
        rot16<S, 4>(r[5], i[5]);
        rot16<S, 6>(r[7], i[7]);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) dft2<S>(r[2 * k1], i[2 * k1], r[2 * k1 + 1], i[2 * k1 + 1]);
        // X[k1 + 4 k2] sits at register 2*k1 + k2 (see out_slot)
    } else {
        // R == 16: n = 4 n1 + n2; A[n2][k1] = DFT4_n1 x[4 n1 + n2]; * w16^(n2 k1); X[k1 + 4 k2] = DFT4_n2
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) dft4<S>(r, i, n2, n2 + 4, n2 + 8, n2 + 12);
        // element (n2, k1) now sits at 4*k1 + n2
        rot16<S, 1>(r[5], i[5]);
        rot16<S, 2>(r[9], i[9]);
        rot16<S, 3>(r[13], i[13]);
        rot16<S, 2>(r[6], i[6]);
        rot16<S, 4>(r[10], i[10]);
        rot16<S, 6>(r[14], i[14]);
        rot16<S, 3>(r[7], i[7]);
        rot16<S, 6>(r[11], i[11]);
        rot16<S, 9>(r[15], i[15]);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) dft4<S>(r, i, 4 * k1, 4 * k1 + 1, 4 * k1 + 2, 4 * k1 + 3);
        // X[k1 + 4 k2] sits at register 4*k1 + k2 (see out_slot)
    }
}

// dft_reg<8> for inputs 4..7 known to be zero (zero-padded forward lines):
// the same arithmetic minus the additions of zeros, so bitwise the same result.
template <int S>
__device__ __forceinline__ void dft4_half(double* r, double* i, int a0, int a1, int a2, int a3) {
    const double ar = r[a0], ai = i[a0], br = r[a1], bi = i[a1];
    const double er = -S * bi, ei = S * br;
    r[a0] = ar + br;
    i[a0] = ai + bi;
    r[a2] = ar - br;
    i[a2] = ai - bi;
    r[a1] = ar + er;
    i[a1] = ai + ei;
    r[a3] = ar - er;
    i[a3] = ai - ei;
}

template <int S>
__device__ __forceinline__ void dft8_zero_hi(double* r, double* i) {
    dft4_half<S>(r, i, 0, 2, 4, 6);
    dft4_half<S>(r, i, 1, 3, 5, 7);
    rot16<S, 2>(r[3], i[3]);
    rot16<S, 4>(r[5], i[5]);
    rot16<S, 6>(r[7], i[7]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft2<S>(r[2 * k1], i[2 * k1], r[2 * k1 + 1], i[2 * k1 + 1]);
}

// register holding DFT output k after dft_reg<R>
template <int R>
__host__ __device__ constexpr int out_slot(int k) {
    return R == 16 ? 4 * (k & 3) + (k >> 2) : (R == 8 ? 2 * (k & 3) + (k >> 2) : k);
}

// Shared memory: split re / im arrays (8-B accesses) with one pad slot per 16
// elements -> the stride-16 Stockham stores of the first pass and the strided
// loads are bank-conflict free (two wavefronts per warp access).
__device__ __forceinline__ int padi(int i) { return i + (i >> 4); }
// k_fft8 exchange padding: one slot per 2^PADS (PADS = 3 for the strided
// two-line mapping: bank-conflict free for stores and loads, per a half-warp
// model of 8-byte shared accesses; 4 for the contiguous mapping)
// PADS > 0: one pad slot per 2^PADS elements.  PADS == 0: no padding, an XOR
// swizzle of the low four bits by bits 3..6 (a bijection inside each 16-slot
// block) -- the contiguous 8-point mapping's three Stockham exchanges, with
// 64-bit accesses served per half-warp, hit 16 distinct bank pairs for every
// line length 64..8192 (one slot per 16 left pass 2's stores 2-way
// conflicted: 0.28 M excess wavefronts per config-5 row pass).
template <int PADS>
__host__ __device__ __forceinline__ constexpr int padq(int i) {
    if constexpr (PADS == 0) return i ^ ((i >> 3) & 15);
    else return i + (i >> PADS);
}

// One Stockham pass of radix R over the CTA's lines (16 points per thread).
// Twiddles of the Ns = 16 pass, radix-major: t16[r * 16 + k] = exp(-2 pi i r k / (16 R));
// of the Ns = 256 pass: tws[r * 256 + k] (consecutive k on consecutive lanes).
template <int R, int S, int TPB>
__device__ __forceinline__ void stockham(double* sre, double* sim, int logL, int logNs, const double2* tws,
                                         const double2* t16, int skw) {
    constexpr int NB = 16 / R;  // 16 points per thread
    constexpr int LR = R == 16 ? 4 : (R == 8 ? 3 : (R == 4 ? 2 : 1));
    const int lpl = logL - LR;  // log2(L / R)
    const int pl = 1 << lpl;
    // padded strides: padi(x + r*c) = padi(x) + r*(c + c/16) when c % 16 == 0 and
    // x % 16 + r*c stays in the same 16-block for c == 1 (first pass stores)
    const int ld_stride = pl >= 16 ? pl + (pl >> 4) : pl;
    const int Ns = 1 << logNs;
    const int st_stride = Ns >= 16 ? Ns + (Ns >> 4) : Ns;
    double vr[NB][R], vi[NB][R];
    int dst[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int bf = threadIdx.x + b * TPB;
        const int g = bf >> lpl;
        const int j = bf & (pl - 1);
        const int k = j & (Ns - 1);
        const int base = padi((g << logL) + j) + g * skw;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int q = pl >= 16 ? base + r * ld_stride : padi((g << logL) + j + (r << lpl)) + g * skw;
            vr[b][r] = sre[q];
            vi[b][r] = sim[q];
        }
        if (logNs > 0) {
            const int tstep = k << (logL - logNs - LR);
#pragma unroll
            for (int r = 1; r < R; ++r) {
                // logNs == 8 (the last pass when L > 256): tstep == k, table radix-major
                const double2 t = logNs == 4 ? t16[r * 16 + k] : tws[(r << 8) + (tstep & 255)];
                const double ti = S < 0 ? t.y : -t.y;
                const double xr = vr[b][r];
                vr[b][r] = fma(xr, t.x, -vi[b][r] * ti);
                vi[b][r] = fma(xr, ti, vi[b][r] * t.x);
            }
        }
        dft_reg<R, S>(vr[b], vi[b]);
        dst[b] = padi((g << logL) + ((j >> logNs) << (logNs + LR)) + k) + g * skw;
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int q = dst[b] + r * st_stride;
            sre[q] = vr[b][out_slot<R>(r)];
            sim[q] = vi[b][out_slot<R>(r)];
        }
    __syncthreads();
}

template <int S, int TPB>
__device__ void fft_smem(double* sre, double* sim, int logL, const double2* tws, const double2* t16, int skw) {
    int logNs = 0;
    int rem = logL;
    while (rem >= 4) {
        stockham<16, S, TPB>(sre, sim, logL, logNs, tws, t16, skw);
        logNs += 4;
        rem -= 4;
    }
    if (rem == 3) stockham<8, S, TPB>(sre, sim, logL, logNs, tws, t16, skw);
    if (rem == 2) stockham<4, S, TPB>(sre, sim, logL, logNs, tws, t16, skw);
    if (rem == 1) stockham<2, S, TPB>(sre, sim, logL, logNs, tws, t16, skw);
}

// Pass modes: what a line transform reads, does and writes.
enum FftMode { kFwdCC = 0, kInvCC = 1, kFwdRC = 2, kInvCR = 3, kFusedCC = 4, kFusedRR = 5, kFwdRCUpd = 6, kInvCRPost = 7 };

template <int MODE, int TPB>
__global__ void __launch_bounds__(TPB, 2) k_fft_lines(LineArgs a) {
    constexpr int PTS = 16 * TPB;  // points per CTA
    constexpr int LOGPTS = TPB == 256 ? 12 : 9;
    constexpr int SSTR = PTS + PTS / 16 + 16;  // + line skew
    extern __shared__ __align__(16) double smd[];
    constexpr bool in_real = MODE == kFwdRC || MODE == kFusedRR;
    constexpr bool out_real = MODE == kInvCR || MODE == kFusedRR;
    constexpr bool fused = MODE == kFusedCC || MODE == kFusedRR;
    double* sre = smd;
    double* sim = smd + SSTR;
    // Ns = 256 pass twiddles, radix-major: qt[r * 256 + k] = exp(-2 pi i r k / L), r < L / 256
    // (consecutive k on consecutive lanes: conflict-free, unlike tw[r * k])
    double2* qt = reinterpret_cast<double2*>(smd + 2 * SSTR);
    double2* t16 = qt + a.L;                                    // Ns = 16 pass twiddles
    if (a.stop && *a.stop) return;
    __shared__ double csc[2];
    const int L = a.L;
    const int logL = a.logL;
    // twiddle tables by cp.async (no registers, overlaps the line loads below)
    for (int r = threadIdx.x; r < L; r += TPB) {
        const double2* src = a.tw + (logL > 8 ? (r >> 8) * (r & 255) : r);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(qt + r)),
                     "l"(src));
    }
    if (logL > 4) {
        // radix of the Ns = 16 pass: 16 if logL >= 8, else 2^(logL-4)
        const int lr2 = logL >= 8 ? 4 : logL - 4;
        for (int e = threadIdx.x; e < (16 << lr2); e += TPB) {
            const int r = e >> 4, k = e & 15;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(
                             (unsigned)__cvta_generic_to_shared(t16 + e)),
                         "l"(a.tw + ((r * k) << (logL - 4 - lr2))));
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    const int logG = LOGPTS - logL;
    const int G = 1 << logG;
    // per-line skew of 16/G doubles: in the strided (column) modes a warp's
    // lanes cover G lines at the same l, whose padded offsets would otherwise
    // share a bank pair (line pitch L + L/16 == 0 mod 16 words)
    const int skw = logG <= 4 ? (16 >> logG) : 0;
    const int g0 = blockIdx.x * G;
    const int lgi = a.lg_ninner;
    // load: all 16 points per thread issued before the shared-memory stores
    const bool contig_in = in_real || a.in_sl == 1;
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int p = threadIdx.x + q * TPB;
        int g, l;
        if (contig_in) {
            g = p >> logL;
            l = p & (L - 1);
        } else {
            g = p & (G - 1);
            l = p >> logG;
        }
        const int line = g0 + g;
        v[q] = make_double2(0.0, 0.0);
        if (line < a.nlines && l < a.n_in) {
            const int o = lgi >= 0 ? line >> lgi : line / a.ninner;
            const int i = lgi >= 0 ? line & ((1 << lgi) - 1) : line - o * a.ninner;
            const int64_t off = (int64_t)o * a.in_so + (int64_t)i * a.in_si +
                                (a.in_lsplit < 0 ? (int64_t)l * a.in_sl
                                                 : (int64_t)(l >> a.in_lsplit) * a.in_sh +
                                                       (int64_t)(l & ((1 << a.in_lsplit) - 1)) * a.in_sl);
            if constexpr (in_real) {
                v[q].x = __ldg(a.x0 + off);
                if (a.x1) v[q].y = __ldg(a.x1 + off);
            } else {
                v[q] = a.in_c[off];
            }
        }
    }
    if ((in_real && a.scale_in) || (out_real && a.scale_out)) column_scales<TPB>(a, csc);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int p = threadIdx.x + q * TPB;
        int g, l;
        if (contig_in) {
            g = p >> logL;
            l = p & (L - 1);
        } else {
            g = p & (G - 1);
            l = p >> logG;
        }
        if constexpr (in_real) {
            if (a.scale_in) {
                v[q].x *= csc[0];
                v[q].y *= csc[1];
            }
        }
        const int qi = padi(g * L + l) + g * skw;
        sre[qi] = v[q].x;
        sim[qi] = v[q].y;
    }
    __syncthreads();
    if constexpr (fused) {
        fft_smem<-1, TPB>(sre, sim, logL, qt, t16, skw);
        // multiply by the folded real symbol; line (inner index i) enumerates axes 1..dim-1.
        // A thread's 16 points lie on at most 16 lines: per-point line offsets first,
        // then all 16 symbol loads in flight, then the multiplies.
        const int np1 = L / 2 + 1;  // folded symbol extent per axis
        double lam[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int p = threadIdx.x + q * TPB;
            const int g = p >> logL, l = p & (L - 1);
            const int line = g0 + g;
            int tmp = (line & ((1 << lgi) - 1)) + a.line0, off = 0, stride = 1;
            for (int d = a.dim - 1; d >= 1; --d) {
                const int k = tmp & (L - 1);
                tmp >>= logL;
                off += min(k, L - k) * stride;
                stride *= np1;
            }
            lam[q] = line < a.nlines ? __ldg(a.sym + (int64_t)off * np1 + min(l, L - l)) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int pp = threadIdx.x + q * TPB;
            const int qi = padi(pp) + (pp >> logL) * skw;
            sre[qi] *= lam[q];
            sim[qi] *= lam[q];
        }
        __syncthreads();
        fft_smem<+1, TPB>(sre, sim, logL, qt, t16, skw);
    } else if constexpr (MODE == kFwdCC || MODE == kFwdRC) {
        fft_smem<-1, TPB>(sre, sim, logL, qt, t16, skw);
    } else {
        fft_smem<+1, TPB>(sre, sim, logL, qt, t16, skw);
    }
    const bool contig_out = out_real || a.out_sl == 1;
#pragma unroll 4
    for (int q = 0; q < 16; ++q) {
        const int p = threadIdx.x + q * TPB;
        int g, l;
        if (contig_out) {
            g = p >> logL;
            l = p & (L - 1);
        } else {
            g = p & (G - 1);
            l = p >> logG;
        }
        const int line = g0 + g;
        if (line >= a.nlines || l >= a.n_out) continue;
        const int o = lgi >= 0 ? line >> lgi : line / a.ninner;
        const int i = lgi >= 0 ? line & ((1 << lgi) - 1) : line - o * a.ninner;
        const int64_t off = (int64_t)o * a.out_so + (int64_t)i * a.out_si +
                            (a.out_lsplit < 0 ? (int64_t)l * a.out_sl
                                              : (int64_t)(l >> a.out_lsplit) * a.out_sh +
                                                    (int64_t)(l & ((1 << a.out_lsplit) - 1)) * a.out_sl);
        const int qq = padi(g * L + l) + g * skw;
        double2 w = make_double2(sre[qq], sim[qq]);
        if constexpr (out_real) {
            if (a.scale_out) {
                w.x /= csc[0];  // exact: powers of two
                w.y /= csc[1];
            }
            a.y0[off] = w.x;
            if (a.y1) a.y1[off] = w.y;
        } else {
            a.out_c[off] = w;
        }
    }
}

// ---------------------------------------------------------------------------
// k_fft8: the production line FFT for 64 <= L <= 4096.  A line is owned by
// TPL = L/8 threads, 8 points each; passes are radix 8 (the last one radix
// 2^(logL mod 3) when logL is not a multiple of 3).  Every Stockham pass reads
// the thread's positions {j + TPL m : m < 8} (butterfly b of NB = 8/R uses
// m = b + NB r), so the first pass takes the line load straight from
// registers and the last pass leaves position j + TPL m in register m: it is
// stored from registers, or -- in the fused column pass -- multiplied by the
// symbol and fed to the inverse transform without touching shared memory.
// 64 registers, up to 512 threads per CTA, 2-4 CTAs per SM; twiddles are
// per-pass radix-major tables read through the L1 cache.
template <int LOGL>
struct Plan8 {
    static constexpr int L = 1 << LOGL;
    static constexpr int P = (LOGL + 2) / 3;
    static constexpr int TPL = L / 8;
    static constexpr int rlog(int p) { return p < P ? 3 : LOGL - 3 * (P - 1); }  // p = 1..P
    static constexpr int toff(int p) {  // offset of pass p's table (p >= 2)
        int o = 0;
        for (int q = 2; q < p; ++q) o += (1 << rlog(q)) << (3 * (q - 1));
        return o;
    }
};

// in-register DFT_R over the NB-strided inputs v[b + NB r]; outputs in natural order
template <int S, int R>
__device__ __forceinline__ void dft_r8(double* vr, double* vi, int b, int NB) {
    double xr[R], xi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        xr[r] = vr[b + NB * r];
        xi[r] = vi[b + NB * r];
    }
    dft_reg<R, S>(xr, xi);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        vr[b + NB * r] = xr[out_slot<R>(r)];
        vi[b + NB * r] = xi[out_slot<R>(r)];
    }
}

// gather positions j + TPL m (m < 8) of a line from the exchange buffer.  With
// the XOR swizzle (PADS == 0), padq(j + TPL m) = padq(j) ^ padq(TPL m), and for
// TPL >= 128 (a multiple of 16 above j's swizzled bits) that is padq(j) + TPL m:
// one base register and immediate offsets.
template <int PADS, int TPL>
__device__ __forceinline__ void load8(double* vr, double* vi, int j, const double* re, const double* im) {
    const int qj = PADS == 0 ? padq<0>(j) : 0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const int q = PADS != 0 ? padq<PADS>(j + TPL * m) : (TPL >= 128 ? qj + TPL * m : (qj ^ padq<0>(TPL * m)));
        vr[m] = re[q];
        vi[m] = im[q];
    }
}

// twiddles of Stockham pass PASS (> 1) for the thread's NB butterflies:
// t[b (R - 1) + r - 1] = tw8[toff + k_b + r NS]
template <int LOGL, int PASS>
__device__ __forceinline__ void load_tw8(double2* t, int j, const double2* __restrict__ tw8) {
    using PL = Plan8<LOGL>;
    constexpr int R = 1 << PL::rlog(PASS);
    constexpr int NB = 8 / R;
    constexpr int NS = 1 << (3 * (PASS - 1));
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int k = (j + PL::TPL * b) & (NS - 1);
#pragma unroll
        for (int r = 1; r < R; ++r) t[b * (R - 1) + r - 1] = __ldg(tw8 + PL::toff(PASS) + k + r * NS);
    }
}

// Stockham pass p of a line: twiddle (t: this pass's twiddles, loaded by the
// previous pass), butterflies, then (p < P) scatter to the line's shared
// memory, load the next pass's twiddles into t while the barrier drains (the
// line's registers are free between the stores and the gathers), gather.
template <int S, int LOGL, int PASS, int PADS>
__device__ __forceinline__ void pass8(double* vr, double* vi, int j, double* re, double* im,
                                      const double2* __restrict__ tw8, double2* t, bool zero_hi = false) {
    using PL = Plan8<LOGL>;
    constexpr int R = 1 << PL::rlog(PASS);
    constexpr int NB = 8 / R;
    constexpr int NS = 1 << (3 * (PASS - 1));
    constexpr int TPL = PL::TPL;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        if (PASS > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const double2 tt = t[b * (R - 1) + r - 1];
                const double ti = S < 0 ? tt.y : -tt.y;
                const int m = b + NB * r;
                const double xr = vr[m];
                vr[m] = fma(xr, tt.x, -vi[m] * ti);
                vi[m] = fma(xr, ti, vi[m] * tt.x);
            }
        }
        if (PASS == 1 && zero_hi) {  // R == 8, NB == 1: inputs j + TPL m, m >= 4, are zero padding
            dft8_zero_hi<S>(vr, vi);
            double xr[8], xi[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                xr[r] = vr[r];
                xi[r] = vi[r];
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                vr[r] = xr[out_slot<8>(r)];
                vi[r] = xi[out_slot<8>(r)];
            }
        } else {
            dft_r8<S, R>(vr, vi, b, NB);
        }
    }
    if constexpr (PASS == PL::P) {
        return;  // register m now holds position j + TPL m
    } else {
        __syncthreads();  // the previous exchange's reads are done
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int jb = j + TPL * b;
            const int k = jb & (NS - 1);
            const int o0 = (jb / NS) * NS * R + k;
            // PADS == 0: the swizzle is XOR-linear and o0, NS r have disjoint bits,
            // so padq(o0 + NS r) = padq(o0) ^ padq(NS r): one XOR with an immediate
            const int q0 = PADS == 0 ? padq<0>(o0) : 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int q = PADS == 0 ? (q0 ^ padq<0>(NS * r)) : padq<PADS>(o0 + NS * r);
                re[q] = vr[b + NB * r];
                im[q] = vi[b + NB * r];
            }
        }
        load_tw8<LOGL, PASS + 1>(t, j, tw8);
        __syncthreads();
        load8<PADS, TPL>(vr, vi, j, re, im);
    }
}

template <int S, int LOGL, int PADS>
__device__ __forceinline__ void fft8_line(double* vr, double* vi, int j, double* re, double* im,
                                          const double2* __restrict__ tw8, bool zero_hi = false) {
    constexpr int P = Plan8<LOGL>::P;
    double2 t[7];
    pass8<S, LOGL, 1, PADS>(vr, vi, j, re, im, tw8, t, zero_hi);
    if constexpr (P >= 2) pass8<S, LOGL, 2, PADS>(vr, vi, j, re, im, tw8, t);
    if constexpr (P >= 3) pass8<S, LOGL, 3, PADS>(vr, vi, j, re, im, tw8, t);
    if constexpr (P >= 4) pass8<S, LOGL, 4, PADS>(vr, vi, j, re, im, tw8, t);
    if constexpr (P >= 5) pass8<S, LOGL, 5, PADS>(vr, vi, j, re, im, tw8, t);  // L = 8192
}

// 2048-point line with 16 points per thread (128 threads per line): radix 16,
// 16, 8 -- two shared-memory exchanges instead of the three of the 8-point
// plan.  Register m holds position j + 128 m before and after (natural order),
// so the fused column pass keeps the spectrum in registers as with k_fft8.
// Twiddles tw16: pass 2 t[r*16 + k] = w_256^(r k) (r, k < 16), pass 3
// t[256 + r*256 + k] = w_2048^(r k) (r < 8, k < 256).
template <int S, int PADS>
__device__ __forceinline__ void fft16_line_2048(double* vr, double* vi, int j, double* re, double* im,
                                                const double2* __restrict__ tw16, bool zero_hi) {
    constexpr int TPL = 128;
    // pass 1: Ns = 1, radix 16 over positions j + 128 m -> 16 j + k
    if (zero_hi) {  // positions >= 1024 (m >= 8) are zero padding: same arithmetic without the zero adds
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) dft4_half<S>(vr, vi, n2, n2 + 4, n2 + 8, n2 + 12);
        rot16<S, 1>(vr[5], vi[5]);
        rot16<S, 2>(vr[9], vi[9]);
        rot16<S, 3>(vr[13], vi[13]);
        rot16<S, 2>(vr[6], vi[6]);
        rot16<S, 4>(vr[10], vi[10]);
        rot16<S, 6>(vr[14], vi[14]);
        rot16<S, 3>(vr[7], vi[7]);
        rot16<S, 6>(vr[11], vi[11]);
        rot16<S, 9>(vr[15], vi[15]);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) dft4<S>(vr, vi, 4 * k1, 4 * k1 + 1, 4 * k1 + 2, 4 * k1 + 3);
    } else {
        dft_reg<16, S>(vr, vi);
    }
    __syncthreads();  // the previous users of the exchange buffer are done
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int q = padq<PADS>(16 * j + k);
        re[q] = vr[out_slot<16>(k)];
        im[q] = vi[out_slot<16>(k)];
    }
    // the next pass's twiddles are loaded while the exchange barrier drains (the
    // line's registers are free between the stores and the gathers)
    const int k = j & 15;
    double2 t2[15];
#pragma unroll
    for (int r = 1; r < 16; ++r) t2[r - 1] = __ldg(tw16 + r * 16 + k);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int q = padq<PADS>(j + TPL * m);
        vr[m] = re[q];
        vi[m] = im[q];
    }
    // pass 2: Ns = 16, radix 16
    double2 t3[14];
    {
#pragma unroll
        for (int r = 1; r < 16; ++r) {
            const double2 t = t2[r - 1];
            const double ti = S < 0 ? t.y : -t.y;
            const double xr = vr[r];
            vr[r] = fma(xr, t.x, -vi[r] * ti);
            vi[r] = fma(xr, ti, vi[r] * t.x);
        }
        dft_reg<16, S>(vr, vi);
        __syncthreads();
        const int base = (j >> 4) * 256 + k;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            const int q = padq<PADS>(base + 16 * kk);
            re[q] = vr[out_slot<16>(kk)];
            im[q] = vi[out_slot<16>(kk)];
        }
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int r = 1; r < 8; ++r) t3[7 * b + r - 1] = __ldg(tw16 + 256 + r * 256 + j + TPL * b);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int q = padq<PADS>(j + TPL * m);
            vr[m] = re[q];
            vi[m] = im[q];
        }
    }
    // pass 3: Ns = 256, radix 8, butterflies b = 0, 1 at jb = j + 128 b over registers b + 2 r;
    // output k of butterfly b (position jb + 256 k) lands in register b + 2 k
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        double xr[8], xi[8];
        xr[0] = vr[b];
        xi[0] = vi[b];
#pragma unroll
        for (int r = 1; r < 8; ++r) {
            const double2 t = t3[7 * b + r - 1];
            const double ti = S < 0 ? t.y : -t.y;
            const double ar = vr[b + 2 * r], ai = vi[b + 2 * r];
            xr[r] = fma(ar, t.x, -ai * ti);
            xi[r] = fma(ar, ti, ai * t.x);
        }
        dft_reg<8, S>(xr, xi);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            vr[b + 2 * r] = xr[out_slot<8>(r)];
            vi[b + 2 * r] = xi[out_slot<8>(r)];
        }
    }
}

__device__ __forceinline__ int64_t line_off(int64_t so, int64_t si, int64_t sl, int lsplit, int64_t sh, int o, int i,
                                            int l) {
    return (int64_t)o * so + (int64_t)i * si +
           (lsplit < 0 ? (int64_t)l * sl
                       : (int64_t)(l >> lsplit) * sh + (int64_t)(l & ((1 << lsplit) - 1)) * sl);
}

__device__ void column_scales_dyn(const LineArgs& a, double* sc) {
    if (a.scales) {
        if (threadIdx.x < 2) sc[threadIdx.x] = a.scales[threadIdx.x];
        return;
    }
    __shared__ double red[2][32];
    double m0 = 0.0, m1 = 0.0;
    for (int c = threadIdx.x; c < a.namax; c += blockDim.x) {
        m0 = fmax(m0, a.amax[2 * c]);
        m1 = fmax(m1, a.amax[2 * c + 1]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        m0 = fmax(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        m1 = fmax(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = m0;
        red[1][w] = m1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < nw; ++q) {
            m0 = fmax(m0, red[0][q]);
            m1 = fmax(m1, red[1][q]);
        }
        sc[0] = pow2_scale(m0);
        sc[1] = pow2_scale(m1);
    }
}

// TMA (tensor) tile copies for the strided column pass
__device__ __forceinline__ unsigned smem32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
            "r"(smem32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map),
                 "r"(x), "r"(y), "r"(smem32(src))
                 : "memory");
}

// line FFT of the k_fft8 kernel: 8 points per thread (any L in 64..4096) or 16
// (L = 2048)
template <int S, int LOGL, int PADS, int PTS>
__device__ __forceinline__ void fft_line(double* vr, double* vi, int j, double* re, double* im, const LineArgs& a,
                                         bool zero_hi) {
    if constexpr (PTS == 16) fft16_line_2048<S, PADS>(vr, vi, j, re, im, a.tw16, zero_hi);
    else fft8_line<S, LOGL, PADS>(vr, vi, j, re, im, a.tw8, zero_hi);
}

// Tree sums of (a, b) over each line's TPL threads (contiguous mapping: line g
// = threads [g TPL, (g + 1) TPL)); the sums land in thread j == 0 of the line.
// The halving tree a[j] += a[j + off], off = TPL/2 .. 1: levels with off >= 32
// through shared memory, the last five inside the line's first warp by
// shuffles (lane j + off -> j: the same pairs, so the same sums bit for bit).
__device__ __forceinline__ void line_pair_tree(double& a, double& b, int j, int g, int TPL, double* sm) {
    if (TPL > 32) {
        __syncthreads();  // the FFT's exchange buffer is free
        double* sa = sm;
        double* sb = sm + blockDim.x;
        sa[threadIdx.x] = a;
        sb[threadIdx.x] = b;
        __syncthreads();
        for (int off = TPL / 2; off >= 32; off >>= 1) {
            if (j < off) {
                sa[threadIdx.x] += sa[threadIdx.x + off];
                sb[threadIdx.x] += sb[threadIdx.x + off];
            }
            __syncthreads();
        }
        if (j < 32) {
            a = sa[threadIdx.x];
            b = sb[threadIdx.x];
        }
    }
    // lines of <= 32 threads are warp-aligned (TPL a power of two)
    if (j < 32) {
        const unsigned mask = 0xffffffffu;  // whole warps: blockDim is a multiple of 32, lines warp-aligned
        for (int off = min(TPL, 32) / 2; off > 0; off >>= 1) {
            const double ao = __shfl_down_sync(mask, a, off, min(TPL, 32));
            const double bo = __shfl_down_sync(mask, b, off, min(TPL, 32));
            if (j < off) {
                a += ao;
                b += bo;
            }
        }
    }
    // (the sums are consumed by thread j == 0 of each line only)
}

// k_iter_b's vector half folded into the first (row) pass of a 2-RHS A-pass
// (see LineArgs): beta and the multipliers come from the state, fixed by the
// decider in the previous apply's scatter (pcg_decide), so every CTA starts
// its transform after one scalar round trip; p_new = z + beta p_old is stored
// back and max|p_new| goes to the iteration's rotating slot.
template <int PTS, int TPL>
__device__ __forceinline__ void fused_p_update(const LineArgs& a, double* vr, const double* zv, int line, bool live,
                                               int o, int i, double* csc, double* sm) {
    PcgState* s = a.upd_s;
    const int t = threadIdx.x;
    const long long itf = a.upd_it < 0 ? s->it_dev : a.upd_it;
    const double beta = s->beta;
    if (t == 0) {
        csc[0] = s->sc[0];
        csc[1] = s->sc[1];
    }
    double m = 0.0;
    const int j = t % TPL;
#pragma unroll
    for (int q = 0; q < PTS / 2; ++q) {
        const int l = j + TPL * q;
        if (live && l < a.n_in) {
            const int64_t off = line_off(a.in_so, a.in_si, a.in_sl, a.in_lsplit, a.in_sh, o, i, l);
            const double pn = __dadd_rn(zv[q], __dmul_rn(beta, vr[q]));
            const_cast<double*>(a.x0)[off] = pn;
            vr[q] = pn;
            m = fmax(m, fabs(pn));
        }
    }
    // max|p_new| over the CTA -> the iteration's slot (non-negative doubles order as their bits)
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((t & 31) == 0 && m > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(a.upd_pglob + itf % 3),
                  (unsigned long long)__double_as_longlong(m));
    __syncthreads();  // csc
}

// shared-memory pitch of one staged folded-symbol line (fused TMA column pass)
__host__ __device__ constexpr int sym_pitch(int L) { return (L / 2 + 1 + 7) / 16 * 16 + 8; }

// the folded symbol of fused line `line` (axes 1..dim-1 from the line index,
// axis 0 contiguous along the line; see k_fold_symbol)
__device__ __forceinline__ const double* sym_line(const LineArgs& a, int line) {
    const int lgi = a.lg_ninner;
    const int i = lgi >= 0 ? line & ((1 << lgi) - 1) : line % a.ninner;
    const int L = a.L, np1 = L / 2 + 1;
    int tmp = i + a.line0, off = 0, stride = 1;
    for (int d = a.dim - 1; d >= 1; --d) {
        const int k = tmp & (L - 1);
        tmp >>= a.logL;
        off += min(k, L - k) * stride;
        stride *= np1;
    }
    return a.sym + (int64_t)off * np1;
}

// the output side of the exact 2-RHS column scaling: x / c_0, y / c_1 (powers
// of two), as multiplications by the exact reciprocals (a division is a
// ~10-instruction sequence); division kept for a non-power-of-two multiplier
struct OutScale {
    double r0 = 1.0, r1 = 1.0, c0 = 1.0, c1 = 1.0;
    bool div = false;
    __device__ __forceinline__ OutScale(const LineArgs& a, const double* csc) {
        if (a.scale_out) {
            c0 = csc[0];
            c1 = csc[1];
            r0 = exact_recip(c0);
            r1 = exact_recip(c1);
            div = r0 == 0.0 || r1 == 0.0;
        }
    }
    __device__ __forceinline__ void apply(double& x, double& y) const {
        if (div) {
            x /= c0;
            y /= c1;
        } else {
            x *= r0;
            y *= r1;
        }
    }
};

template <int MODE, int LOGL, bool STRIDED, bool TMA = false, int PTS = 8>
__global__ void __launch_bounds__(PTS == 16 ? 256 : 1024, PTS == 16 ? 2 : 1) k_fft8(const __grid_constant__ LineArgs a) {
    static_assert(PTS == 8 || LOGL == 11, "16 points per thread: 2048-point lines only");
    // exchange layout (bank-conflict free per a half-warp model of 8-byte shared
    // accesses): one pad slot per 8 for the strided 8-point mapping, per 16 for
    // 16 points per thread, the XOR swizzle (padq<0>) for contiguous 8-point lines
    constexpr int PADS = STRIDED ? (PTS == 8 ? 3 : 4) : (PTS == 8 ? 0 : 4);
    constexpr int L = 1 << LOGL, TPL = L / PTS;
    // folded symbol line length and its shared-memory pitch (== 8 mod 16
    // doubles: the two column lines of a warp hit disjoint bank halves)
    constexpr int kNp1 = L / 2 + 1, kSymPitch = sym_pitch(L);
    constexpr bool upd = MODE == kFwdRCUpd, post = MODE == kInvCRPost;
    constexpr bool in_real = MODE == kFwdRC || MODE == kFusedRR || upd;
    constexpr bool out_real = MODE == kInvCR || MODE == kFusedRR || post;
    constexpr bool fused = MODE == kFusedCC || MODE == kFusedRR;
    extern __shared__ __align__(128) double sm8[];
    __shared__ double csc[2];
    pdl_wait();
    if (a.stop && *a.stop) return;
    // contiguous 8-point lines: the host's lines per CTA and pitch (L + skew) as
    // compile-time constants, so im[q] is re[q] plus an immediate offset
    constexpr bool cpitch = !STRIDED && PTS == 8;
    constexpr int CG = TPL >= 256 ? 1 : 256 / TPL, CPITCH = L + (TPL < 8 ? TPL : 8);
    // the TMA variant is launched with two lines per CTA
    const int G = TMA ? 2 : (cpitch ? CG : a.g8), t = threadIdx.x;
    int g, j;
    if constexpr (STRIDED) {
        g = t % G;
        j = t / G;
    } else {
        g = t / TPL;
        j = t % TPL;
    }
    const int pitch = cpitch ? CPITCH : a.pitch8;
    double* re = sm8 + (int64_t)g * pitch;
    double* im = sm8 + (int64_t)(G + g) * pitch;
    const int line = blockIdx.x * G + g;
    const bool live = line < a.nlines;
    const int lgi = a.lg_ninner;
    const int o = lgi >= 0 ? line >> lgi : line / a.ninner;
    const int i = lgi >= 0 ? line & ((1 << lgi) - 1) : line - o * a.ninner;
    double vr[PTS], vi[PTS];
    double zv[upd ? PTS / 2 : 1];  // z of the fused p update (real input lines: only m < PTS/2 is data)
    constexpr bool tma_mode = TMA && MODE == kFusedCC && STRIDED;
    if constexpr (tma_mode) {
        {
            // the CTA's G columns x n_in rows land densely in shared memory by TMA
            // (one mbarrier transaction), then each thread reads its 8 points
            __shared__ __align__(8) uint64_t tbar;
            if (t == 0) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem32(&tbar)));
                asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            }
            __syncthreads();
            if (t == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem32(&tbar)),
                             "r"(a.n_in * G * 16)
                             : "memory");
                for (int y = 0; y < a.n_in; y += 256)
                    tma_load_2d(sm8 + y * G * 2, &a.tmap, 2 * G * (int)blockIdx.x, y, &tbar);
            }
            // the folded symbol lines of the CTA's G columns -> shared memory
            // behind the exchange buffers (cp.async, in flight with the tile)
            double* ssym = sm8 + (int64_t)2 * G * pitch;
            for (int gl = 0; gl < G; ++gl) {
                if ((int)blockIdx.x * G + gl >= a.nlines) break;
                const double* sl = sym_line(a, blockIdx.x * G + gl);
                for (int e = t; e < kNp1; e += blockDim.x)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem32(ssym + gl * kSymPitch + e)),
                                 "l"(sl + e)
                                 : "memory");
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
            asm volatile(
                "{\n .reg .pred p;\n TW%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra TW%=;\n}\n" ::"r"(
                    smem32(&tbar))
                : "memory");
#pragma unroll
            for (int m = 0; m < PTS; ++m) {
                const int l = j + TPL * m;
                vr[m] = vi[m] = 0.0;
                if (l < a.n_in) {
                    const double2 v = reinterpret_cast<const double2*>(sm8)[l * G + g];
                    vr[m] = v.x;
                    vi[m] = v.y;
                }
            }
            // own copies landed; the forward transform's first barrier publishes them
            asm volatile("cp.async.wait_all;\n" ::: "memory");
        }
    }
    if constexpr (!tma_mode) {
        auto load_pt = [&](int m, int64_t off) {
            if constexpr (in_real) {
                vr[m] = __ldg(a.x0 + off);
                if (a.x1) vi[m] = __ldg(a.x1 + off);
                if constexpr (upd) {
                    if (m < PTS / 2) zv[m] = __ldg(a.upd_z + off);
                }
            } else {
                const double2 v = a.in_c[off];
                vr[m] = v.x;
                vi[m] = v.y;
            }
        };
#pragma unroll
        for (int m = 0; m < PTS; ++m) vr[m] = vi[m] = 0.0;
        if (a.in_lsplit < 0 && a.in_sl == 1) {  // contiguous line: one base offset, immediate strides
            const int64_t ib = (int64_t)o * a.in_so + (int64_t)i * a.in_si + j;
#pragma unroll
            for (int m = 0; m < PTS; ++m)
                if (live && j + TPL * m < a.n_in) load_pt(m, ib + TPL * m);
        } else {
#pragma unroll
            for (int m = 0; m < PTS; ++m) {
                const int l = j + TPL * m;
                if (live && l < a.n_in) load_pt(m, line_off(a.in_so, a.in_si, a.in_sl, a.in_lsplit, a.in_sh, o, i, l));
            }
        }
    }
    // the column scales (a reduction over the max|x| partials) after the line
    // loads are issued: the two memory round trips overlap
    if constexpr (upd) {
        fused_p_update<PTS, TPL>(a, vr, zv, line, live, o, i, csc, sm8);
    } else if ((in_real && a.scale_in) || (out_real && a.scale_out)) {
        column_scales_dyn(a, csc);
        __syncthreads();
    }
    if constexpr (in_real) {
        if (a.scale_in) {
#pragma unroll
            for (int m = 0; m < PTS; ++m) {
                vr[m] *= csc[0];
                vi[m] *= csc[1];
            }
        }
    }
    const bool zero_hi = a.n_in <= L / 2;  // line positions j + TPL m, m >= PTS / 2, read as zero
    if constexpr (fused) {
        fft_line<-1, LOGL, PADS, PTS>(vr, vi, j, re, im, a, zero_hi);
        // folded real symbol at frequency l = j + TPL m along this line
        if constexpr (tma_mode) {  // staged in shared memory at kernel start
            const double* ss = sm8 + (int64_t)2 * G * pitch + g * kSymPitch;
#pragma unroll
            for (int m = 0; m < PTS; ++m) {
                const int l = j + TPL * m;
                const double lam = live ? ss[min(l, L - l)] : 0.0;
                vr[m] *= lam;
                vi[m] *= lam;
            }
        } else {
            const double* symline = sym_line(a, line);
#pragma unroll
            for (int m = 0; m < PTS; ++m) {
                const int l = j + TPL * m;
                const double lam = live ? __ldg(symline + min(l, L - l)) : 0.0;
                vr[m] *= lam;
                vi[m] *= lam;
            }
        }
        // opaque copy of the line position: the inverse recomputes its exchange
        // addresses instead of keeping the forward's alive (64-register budget)
        int jj = j;
        asm volatile("" : "+r"(jj));
        fft_line<+1, LOGL, PADS, PTS>(vr, vi, jj, re, im, a, false);
    } else if constexpr (MODE == kFwdCC || MODE == kFwdRC || MODE == kFwdRCUpd) {
        fft_line<-1, LOGL, PADS, PTS>(vr, vi, j, re, im, a, zero_hi);
    } else {
        fft_line<+1, LOGL, PADS, PTS>(vr, vi, j, re, im, a, zero_hi);
    }
    if constexpr (tma_mode) {
        {
            // outputs to a dense [n_out][G] tile in shared memory, then TMA stores
            __syncthreads();  // the last exchange's reads are done
#pragma unroll
            for (int m = 0; m < PTS; ++m) {
                const int l = j + TPL * m;
                if (l < a.n_out) reinterpret_cast<double2*>(sm8)[l * G + g] = make_double2(vr[m], vi[m]);
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncthreads();
            if (t == 0) {
                for (int y = 0; y < a.n_out; y += 256)
                    tma_store_2d(&a.tmap, 2 * G * (int)blockIdx.x, y, sm8 + y * G * 2);
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // smem read; the grid completes the writes
            }
            return;
        }
    }
    if constexpr (post) {
        // k_post_pass folded in: every point's p / f load first, then the
        // stores, then the per-line partials (FMA chain over m, tree over the
        // line's threads) -- the order the sharded band pass uses too
        double pa = 0.0, pb = 0.0;
        double pv[PTS / 2], fv[PTS / 2];
        const bool own = live && line >= a.post_lo && line < a.post_hi;  // (halo rows: q only, no partial)
        const bool olin = a.out_lsplit < 0 && a.out_sl == 1;
        const int64_t ob = (int64_t)o * a.out_so + (int64_t)i * a.out_si + j;
        auto ooff = [&](int m) {
            return olin ? ob + TPL * m
                        : line_off(a.out_so, a.out_si, a.out_sl, a.out_lsplit, a.out_sh, o, i, j + TPL * m);
        };
#pragma unroll
        for (int m = 0; m < PTS / 2; ++m) {  // n_out <= L / 2: only m < PTS / 2 is output
            const int l = j + TPL * m;
            pv[m] = fv[m] = 0.0;
            if (own && l < a.n_out) {
                const int64_t off = ooff(m);
                if (a.post_q_col >= 0) pv[m] = __ldg(a.post_p + off);
                if (a.post_w_col >= 0) fv[m] = __ldg(a.post_f + off);
            }
        }
        const OutScale os(a, csc);
#pragma unroll
        for (int m = 0; m < PTS / 2; ++m) {
            const int l = j + TPL * m;
            if (!live || l >= a.n_out) continue;
            const int64_t off = ooff(m);
            double x = vr[m], y = vi[m];
            os.apply(x, y);
            if (!(a.post_skip_w && a.post_w_col == 0)) a.y0[off] = x;
            if (a.y1 && !(a.post_skip_w && a.post_w_col == 1)) a.y1[off] = y;
#ifdef IEDD_DEBUG_FUSE
            if (off < 3) printf("post off %lld p %.17g q %.17g w %.17g csc %g %g\n", (long long)off, pv[m], x, y, csc[0], csc[1]);
#endif
            if (a.post_q_col >= 0) pa = fma(pv[m], x, pa);
            if (a.post_w_col >= 0) {
                const double d = fv[m] - (a.post_w_col == 0 ? x : y);
                pb = fma(d, d, pb);
            }
        }
        line_pair_tree(pa, pb, j, g, TPL, sm8);
        if (live && j == 0 && line >= a.post_lo && line < a.post_hi) {
            const int64_t ix = 2 * ((int64_t)a.post_line0 + line);
            a.post_part[ix] = pa;
            a.post_part[ix + 1] = pb;
            for (int h = 0; h < a.post_npeer; ++h) {
                a.post_peer[h][ix] = pa;
                a.post_peer[h][ix + 1] = pb;
            }
        }
        if (a.post_npeer) {  // every CTA signals the bytes its owned lines sent
            __syncthreads();
            if ((int)threadIdx.x < a.post_npeer) {
                const int G8 = a.g8, l0 = (int)blockIdx.x * G8;
                const int lo = max(l0, a.post_lo), hi = min(min(l0 + G8, a.nlines), a.post_hi);
                if (hi > lo) {
                    __threadfence_system();
                    atomicAdd_system(a.post_ctr[threadIdx.x], (unsigned long long)(hi - lo) * 16ull);
                }
            }
        }
        return;
    }
    if constexpr (!out_real && !tma_mode) {
        if (a.peer_mode) {  // sharded transposes: stores into the peers' buffers, then the mailbox signals
            if (live) {
#pragma unroll
                for (int m = 0; m < PTS; ++m) {
                    const int l = j + TPL * m;
                    if (l >= a.n_out) continue;
                    const double2 v = make_double2(vr[m], vi[m]);
                    if (a.peer_mode == 1) {
                        a.peer[l >> a.out_lsplit][(int64_t)o * a.out_so + (int64_t)i * a.out_si +
                                                  (int64_t)(l & ((1 << a.out_lsplit) - 1)) * a.out_sl] = v;
                    } else {
                        const int own = l / a.peer_band_rows;
                        for (int h = max(0, own - 1); h <= min(a.npeer - 1, own + 1); ++h)
                            if (l >= a.peer_rlo[h] && l < a.peer_rhi[h])
                                a.peer[h][(int64_t)(l - a.peer_rlo[h]) * a.out_sl + i] = v;
                    }
                }
            }
            __syncthreads();
            if ((int)threadIdx.x < a.npeer) {
                const int G8 = TMA ? 2 : a.g8;
                const long long lines = min(G8, a.nlines - (int)blockIdx.x * G8);
                __threadfence_system();
                atomicAdd_system(a.peer_ctr[threadIdx.x],
                                 (unsigned long long)(lines * a.peer_line_bytes[threadIdx.x]));
            }
            return;
        }
    }
    if (!live) return;
    const OutScale os(a, csc);
    auto store_pt = [&](int m, int64_t off) {
        if constexpr (out_real) {
            double x = vr[m], y = vi[m];
            os.apply(x, y);
            a.y0[off] = x;
            if (a.y1) a.y1[off] = y;
        } else {
            a.out_c[off] = make_double2(vr[m], vi[m]);
        }
    };
    if (a.out_lsplit < 0 && a.out_sl == 1) {  // contiguous line
        const int64_t ob = (int64_t)o * a.out_so + (int64_t)i * a.out_si + j;
#pragma unroll
        for (int m = 0; m < PTS; ++m)
            if (j + TPL * m < a.n_out) store_pt(m, ob + TPL * m);
    } else {
#pragma unroll
        for (int m = 0; m < PTS; ++m) {
            const int l = j + TPL * m;
            if (l < a.n_out) store_pt(m, line_off(a.out_so, a.out_si, a.out_sl, a.out_lsplit, a.out_sh, o, i, l));
        }
    }
}

// Embedding of the generator in a circulant of size M >= 2n - 1 per axis,
// mirror-even (toeplitz.py:19-30 uses M = 2n with index n left zero):
// emb[k] = gen[k] (k < n), gen[M - k] (k > M - n), 0 between; entries from the
// same integer-distance formula as K1/K2.  Any M >= 2n - 1 gives the same
// Toeplitz product; a power of two keeps every line transform radix-2^k.
__global__ void k_embed(double2* emb, int dim, int n, int M, EntryParams P, const LogEntry* tab) {
    int64_t tot = 1;
    for (int d = 0; d < dim; ++d) tot *= M;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= tot) return;
    int64_t t = e;
    int m = 0;
    bool zero = false;
    for (int d = 0; d < dim; ++d) {
        const int k = (int)(t % M);
        t /= M;
        if (k >= n && k <= M - n) zero = true;
        const int g = k < n ? k : M - k;
        m += g * g;
    }
    emb[e] = make_double2(zero ? 0.0 : entry_from_m(P, tab, m), 0.0);
}

// sym[k_0 + (M/2+1) * rest(k_1..k_{d-1})] = Re(emb_hat[k]) / M^dim, k folded
// (<= M/2); axis 0 (the fused column pass's line axis) fastest so a line reads
// its symbol contiguously; rest = C order over axes 1..d-1 (last fastest)
__global__ void k_fold_symbol(const double2* emb, double* sym, int dim, int M, double scale) {
    const int np1 = M / 2 + 1;
    int64_t tot = 1;
    for (int d = 0; d < dim; ++d) tot *= np1;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= tot) return;
    int64_t t = e, mul = 1;
    const int k0 = (int)(t % np1);
    t /= np1;
    int64_t src = 0;
    for (int d = dim - 1; d >= 1; --d) {
        const int k = (int)(t % np1);
        t /= np1;
        src += (int64_t)k * mul;
        mul *= M;
    }
    src += (int64_t)k0 * mul;
    sym[e] = emb[src].x * scale;
}

}  // namespace ie

// ------------------------------------------------------------- host side --
struct ie_fft {
    int dim, n, M, logM;
    int N;
    double2* d_tw;
    double2* d_tw8;  // k_fft8 per-pass radix-major twiddles (M >= 64)
    double2* d_tw16 = nullptr;  // 16-point plan twiddles (M = 2048)
    double* d_sym;
    double2* d_buf;
    double* d_amax;  // 2 * ceil(N/2048) partial maxima
    // TMA descriptors of the 2D work buffers (the plan's and per-stream ones), by address
    std::mutex tm_mu;
    std::vector<std::pair<const void*, CUtensorMap>> tmaps;
};

namespace ie {

template <int MODE, int TPB>
static int launch_mode(const LineArgs& a, cudaStream_t st) {
    constexpr int PTS = 16 * TPB;
    const int G = PTS / a.L;
    const int ctas = (a.nlines + G - 1) / G;
    const size_t smem = 2 * (size_t)(PTS + PTS / 16 + 16) * sizeof(double) + (size_t)(a.L + 256) * sizeof(double2);
    static bool attr = false;
    if (!attr) {
        const size_t smax = 2 * (size_t)(PTS + PTS / 16 + 16) * sizeof(double) + (size_t)(PTS + 256) * sizeof(double2);
        IE_CUDA(cudaFuncSetAttribute(k_fft_lines<MODE, TPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
        attr = true;
    }
    k_fft_lines<MODE, TPB><<<ctas, TPB, smem, st>>>(a);
    IE_LAUNCHED();
    return IE_OK;
}

template <int TPB>
static int launch_modes(const LineArgs& a, cudaStream_t st) {
    if (a.fused) return a.in_real ? launch_mode<kFusedRR, TPB>(a, st) : launch_mode<kFusedCC, TPB>(a, st);
    if (a.in_real) return launch_mode<kFwdRC, TPB>(a, st);
    if (a.out_real) return launch_mode<kInvCR, TPB>(a, st);
    return a.sign < 0 ? launch_mode<kFwdCC, TPB>(a, st) : launch_mode<kInvCC, TPB>(a, st);
}

template <int MODE, int LOGL, bool STRIDED, bool TMA = false, int PTS = 8>
static int launch_fft8_ls(const LineArgs& a, int tpb, int ctas, size_t smem, cudaStream_t st) {
    // opt-in dynamic shared memory: raised to the largest request seen (the
    // fused TMA pass at L = 4096 with staged symbol lines needs ~180 KB)
    static std::atomic<size_t> attr{0};
    size_t cur = attr.load();
    if (smem > 48 * 1024 && smem > cur) {
        IE_CUDA(cudaFuncSetAttribute(k_fft8<MODE, LOGL, STRIDED, TMA, PTS>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        while (cur < smem && !attr.compare_exchange_weak(cur, smem)) {
        }
    }
    IE_CUDA(launch_k(k_fft8<MODE, LOGL, STRIDED, TMA, PTS>, dim3(ctas), dim3(tpb), smem, st, a));
    IE_LAUNCHED();
    return IE_OK;
}

// real-in / real-out lines are always contiguous (launch_fft8)
template <int MODE, int LOGL, int PTS>
static int launch_fft8_lp(const LineArgs& a, int tpb, int ctas, size_t smem, cudaStream_t st) {
    if constexpr (MODE == kFusedCC) {
        if (a.strided8 && a.tma) return launch_fft8_ls<MODE, LOGL, true, true, PTS>(a, tpb, ctas, smem, st);
    }
    if constexpr (MODE == kFwdCC || MODE == kInvCC || MODE == kFusedCC) {
        if (a.strided8) return launch_fft8_ls<MODE, LOGL, true, false, PTS>(a, tpb, ctas, smem, st);
    }
    return launch_fft8_ls<MODE, LOGL, false, false, PTS>(a, tpb, ctas, smem, st);
}

template <int MODE, int LOGL>
static int launch_fft8_l(const LineArgs& a, int tpb, int ctas, size_t smem, cudaStream_t st) {
    if constexpr (LOGL == 11) {
        if (a.pts == 16) return launch_fft8_lp<MODE, LOGL, 16>(a, tpb, ctas, smem, st);
    }
    return launch_fft8_lp<MODE, LOGL, 8>(a, tpb, ctas, smem, st);
}

template <int MODE>
static int launch_fft8_m(const LineArgs& a, int tpb, int ctas, size_t smem, cudaStream_t st) {
    switch (a.logL) {
        case 6: return launch_fft8_l<MODE, 6>(a, tpb, ctas, smem, st);
        case 7: return launch_fft8_l<MODE, 7>(a, tpb, ctas, smem, st);
        case 8: return launch_fft8_l<MODE, 8>(a, tpb, ctas, smem, st);
        case 9: return launch_fft8_l<MODE, 9>(a, tpb, ctas, smem, st);
        case 10: return launch_fft8_l<MODE, 10>(a, tpb, ctas, smem, st);
        case 11: return launch_fft8_l<MODE, 11>(a, tpb, ctas, smem, st);
        case 12: return launch_fft8_l<MODE, 12>(a, tpb, ctas, smem, st);
        default: return launch_fft8_l<MODE, 13>(a, tpb, ctas, smem, st);
    }
}

// lines per CTA of a strided (column) k_fft8 launch of line length L
static int fft8_strided_g(int L) {
    static const int gs = getenv("IEDD_B200_FFT_G") ? atoi(getenv("IEDD_B200_FFT_G")) : 2;
    const int tpl = L / 8;
    return std::max(std::min(gs, 1024 / tpl), std::min(32, 256 / tpl));
}

// k_fft8 launch: lines per CTA and thread mapping from the access pattern
static int launch_fft8(LineArgs a, cudaStream_t st) {
    // 16 points per thread for strided (column) 2048-point lines: two exchanges
    // instead of three (config-5 fused column pass 52.6 -> 45.9 us); the
    // contiguous row passes measured faster with 8 (21.5 vs 23.6 us row inverse)
    const bool cin = a.in_real || a.in_sl == 1, cout = a.out_real || a.out_sl == 1;
    static const bool no16 = getenv("IEDD_B200_FFT8_ONLY") != nullptr;
    static const bool rows16 = getenv("IEDD_B200_ROWS16") != nullptr;  // comparison: 16 points on rows too
    a.pts = (a.logL == 11 && a.tw16 && (!cin || rows16) && !no16) ? 16 : 8;
    const int tpl = a.L / a.pts;
    a.strided8 = cin ? 0 : 1;
    int G, skew;
    if (a.strided8) {  // lanes alternate lines: 32-B row segments per warp request (G = 2 measured best)
        G = fft8_strided_g(a.L);
        skew = std::max(1, 16 / G);
    } else {
        G = std::max(1, 256 / tpl);
        skew = std::min(tpl, 8);
    }
    (void)cout;
    a.g8 = G;  // (k_fft8 hard-codes G and pitch8 of the contiguous 8-point case: keep in step)
    const int pads = a.strided8 ? (a.pts == 8 ? 3 : 4) : (a.pts == 8 ? 0 : 4);  // k_fft8's PADS
    a.pitch8 = (pads ? (a.L + (a.L >> pads) + 15) / 16 * 16 : a.L) + skew;
    const int tpb = G * tpl;
    const int ctas = (a.nlines + G - 1) / G;
    size_t smem = (size_t)2 * G * a.pitch8 * sizeof(double);
    if (a.fused && a.tma && a.strided8) smem += (size_t)G * sym_pitch(a.L) * sizeof(double);  // staged symbol
    if (a.fused) return a.in_real ? launch_fft8_m<kFusedRR>(a, tpb, ctas, smem, st)
                                  : launch_fft8_m<kFusedCC>(a, tpb, ctas, smem, st);
    if (a.in_real) return a.upd_s ? launch_fft8_m<kFwdRCUpd>(a, tpb, ctas, smem, st)
                                  : launch_fft8_m<kFwdRC>(a, tpb, ctas, smem, st);
    if (a.out_real) return a.post_part ? launch_fft8_m<kInvCRPost>(a, tpb, ctas, smem, st)
                                       : launch_fft8_m<kInvCR>(a, tpb, ctas, smem, st);
    return a.sign < 0 ? launch_fft8_m<kFwdCC>(a, tpb, ctas, smem, st) : launch_fft8_m<kInvCC>(a, tpb, ctas, smem, st);
}

static int line_launch(const LineArgs& a_in, cudaStream_t st) {
    LineArgs a = a_in;
    a.lg_ninner = 0;
    while ((1 << a.lg_ninner) < a.ninner) ++a.lg_ninner;
    if ((1 << a.lg_ninner) != a.ninner) {
        if (a.fused) {  // the fused pass decomposes its line index into symbol axes by powers of two
            set_error("fft: fused line layout must be a power of two");
            return IE_ERR_ARG;
        }
        a.lg_ninner = -1;
    }
    {
        static const bool v1 = getenv("IEDD_B200_FFT_V1") != nullptr;
        const bool cin = a.in_real || a.in_sl == 1, cout = a.out_real || a.out_sl == 1;
        if (!v1 && a.tw8 && a.logL >= 6 && a.logL <= 13 && cin == cout) return launch_fft8(a, st);
    }
    // 256-thread CTAs (4096 points) unless that leaves the GPU under-filled and
    // the lines fit a 32-thread CTA (512 points)
    const long long big_ctas = ((long long)a.nlines * a.L + 4095) / 4096;
    if (a.L <= 512 && big_ctas < 2 * kNumSMs) return launch_modes<32>(a, st);
    return launch_modes<256>(a, st);
}

static LineArgs base_args(const ie_fft* f) {
    LineArgs a{};
    a.tw8 = f->d_tw8;
    a.tw16 = f->d_tw16;
    a.amax = f->d_amax;
    a.namax = (f->N + 2047) / 2048;
    a.L = f->M;
    a.logL = f->logM;
    a.tw = f->d_tw;
    a.sym = f->d_sym;
    a.dim = f->dim;
    a.n = f->n;
    a.sign = -1;
    a.in_lsplit = a.out_lsplit = -1;
    return a;
}

// Full forward FFT along every axis of a complex M^dim array (symbol setup).
static int fft_full_forward(const ie_fft* f, double2* buf, cudaStream_t st) {
    const int M = f->M;
    int64_t tot = 1;
    for (int d = 0; d < f->dim; ++d) tot *= M;
    for (int ax = f->dim - 1; ax >= 0; --ax) {
        int64_t sl = 1;
        for (int d = ax + 1; d < f->dim; ++d) sl *= M;
        LineArgs a = base_args(f);
        a.nlines = (int)(tot / M);
        a.ninner = (int)sl;
        a.in_c = buf;
        a.out_c = buf;
        a.in_so = a.out_so = sl * M;
        a.in_si = a.out_si = 1;
        a.in_sl = a.out_sl = sl;
        a.n_in = a.n_out = M;
        a.sign = -1;
        int rc = line_launch(a, st);
        if (rc) return rc;
    }
    return IE_OK;
}

int make_log_table_device(const ie_geom& g, LogEntry** d_tab, int* ntab);
EntryParams entry_params(const ie_geom& g);

// Circulant size per axis: the smallest power of two >= 2n - 1 (>= 4); equal
// to the reference's 2n for power-of-two n (bitwise the same plan as before)
int fft_size_for(int n) {
    int M = 4;
    while (M < 2 * n - 1) M *= 2;
    return M;
}

int fft_create(const ie_geom& g, ie_fft** out) {
    int n = g.n, logM = 0;
    const int M = fft_size_for(n);
    while ((1 << logM) < M) ++logM;
    if (n < 1 || M > kFftMaxPoints) {
        set_error("fft matvec needs 1 <= n <= 4096 (circulant size <= 8192 per axis)");
        return IE_ERR_ARG;
    }
    ie_fft* f = new ie_fft();
    f->dim = g.dim;
    f->n = n;
    f->M = M;
    f->logM = logM;
    f->N = 1;
    for (int d = 0; d < g.dim; ++d) f->N *= n;
    IE_CUDA(cudaMalloc(&f->d_amax, 2 * (size_t)((f->N + 2047) / 2048) * sizeof(double)));
    std::vector<double2> tw(M);
    for (int m = 0; m < M; ++m) {
        const long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)m / (long double)M;
        tw[m] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    int64_t totM = 1, totS = 1, totB = 1;
    for (int d = 0; d < g.dim; ++d) {
        totM *= M;
        totS *= (M / 2 + 1);
        totB *= (d == 0 ? n : M);
    }
    IE_CUDA(cudaMalloc(&f->d_tw, M * sizeof(double2)));
    IE_CUDA(cudaMemcpy(f->d_tw, tw.data(), M * sizeof(double2), cudaMemcpyHostToDevice));
    f->d_tw8 = nullptr;
    if (logM >= 6) {
        // pass p >= 2 (Ns = 8^(p-1), radix R_p): t[r * Ns + k] = exp(-2 pi i r k / (R_p Ns)) = tw[r k M / (R_p Ns)]
        const int P = (logM + 2) / 3;
        std::vector<double2> t8;
        for (int p = 2; p <= P; ++p) {
            const int rl = p < P ? 3 : logM - 3 * (P - 1), R = 1 << rl, Ns = 1 << (3 * (p - 1));
            for (int r = 0; r < R; ++r)
                for (int k = 0; k < Ns; ++k) t8.push_back(tw[(int64_t)r * k * (M / (R * Ns)) % M]);
        }
        IE_CUDA(cudaMalloc(&f->d_tw8, t8.size() * sizeof(double2)));
        IE_CUDA(cudaMemcpy(f->d_tw8, t8.data(), t8.size() * sizeof(double2), cudaMemcpyHostToDevice));
    }
    if (M == 2048) {  // 16-point plan: pass 2 w_256^(r k) (r, k < 16), pass 3 w_2048^(r k) (r < 8, k < 256)
        std::vector<double2> t16;
        for (int r = 0; r < 16; ++r)
            for (int k = 0; k < 16; ++k) t16.push_back(tw[(int64_t)r * k * (M / 256) % M]);
        for (int r = 0; r < 8; ++r)
            for (int k = 0; k < 256; ++k) t16.push_back(tw[(int64_t)r * k % M]);
        IE_CUDA(cudaMalloc(&f->d_tw16, t16.size() * sizeof(double2)));
        IE_CUDA(cudaMemcpy(f->d_tw16, t16.data(), t16.size() * sizeof(double2), cudaMemcpyHostToDevice));
    }
    IE_CUDA(cudaMalloc(&f->d_sym, totS * sizeof(double)));
    IE_CUDA(cudaMalloc(&f->d_buf, totB * sizeof(double2)));
    // symbol: embed, full forward FFT, fold
    double2* emb;
    IE_CUDA(cudaMalloc(&emb, totM * sizeof(double2)));
    LogEntry* tab;
    int ntab;
    int rc = make_log_table_device(g, &tab, &ntab);
    if (rc) return rc;
    k_embed<<<(unsigned)((totM + 255) / 256), 256>>>(emb, g.dim, n, M, entry_params(g), tab);
    IE_LAUNCHED();
    if ((rc = fft_full_forward(f, emb, 0))) return rc;
    k_fold_symbol<<<(unsigned)((totS + 255) / 256), 256>>>(emb, f->d_sym, g.dim, M, 1.0 / (double)totM);
    IE_LAUNCHED();
    IE_CUDA(cudaDeviceSynchronize());
    cudaFree(emb);
    cudaFree(tab);
    *out = f;
    return IE_OK;
}

void fft_destroy(ie_fft* f) {
    if (!f) return;
    cudaFree(f->d_tw);
    cudaFree(f->d_tw8);
    cudaFree(f->d_tw16);
    cudaFree(f->d_sym);
    cudaFree(f->d_buf);
    cudaFree(f->d_amax);
    delete f;
}

// the PCG fusions (PcgFuse) on a line pass: the first real-input pass takes the
// p update, the last real-output pass the post pass
static void apply_fuse(LineArgs& a, const PcgFuse* fz) {
    if (!fz) return;
    if (a.in_real && fz->s) {
        a.upd_z = fz->z;
        a.upd_pglob = fz->pglob;
        a.upd_s = fz->s;
        a.upd_it = fz->it;
        a.scale_in = 1;
    }
    if (a.out_real && fz->part) {
        a.post_npeer = fz->npeer;
        for (int h = 0; h < fz->npeer; ++h) {
            a.post_peer[h] = fz->part_peer[h];
            a.post_ctr[h] = fz->part_ctr[h];
        }
        a.post_p = fz->p;
        a.post_f = fz->f;
        a.post_skip_w = fz->skip_w_store;
        a.post_part = fz->part;
        a.post_line0 = fz->line0;
        a.post_lo = fz->post_lo;
        a.post_hi = fz->post_hi;
        a.post_q_col = fz->q_col;
        a.post_w_col = fz->w_col;
    }
}

// ---- 2D band (slab) decomposition of the same three passes, for the sharded
// solver: rank g owns grid rows [row0, row0 + nrows); the M = 2n spectrum
// columns are split into `parts` slabs of Mc = M / parts.
//   band_fwd:  rows of the band, forward along axis 1, written destination-
//              major: out[(h * nrows + r) * Mc + c_local] (column c = h*Mc + c_local)
//              -- slab h is one contiguous all-to-all send block;
//   band_cols: after the all-to-all, buf[r * Mc + c_local] holds every grid row
//              r of columns [c0, c0 + ncols): fused forward * symbol * inverse;
//   band_inv:  after the reverse all-to-all, in[(h * nrows + r) * Mc + c_local]:
//              inverse along axis 1 of the band rows -> real pair.
// Every line goes through the same kernel with the same data as fft_matvec, so
// the result is bitwise that of the single-GPU pass for any `parts`.
static int band_check(const ie_fft* f, int parts) {
    if (f->dim != 2 || parts < 1 || f->M % parts || ((f->M / parts) & (f->M / parts - 1))) {
        set_error("fft band passes: 2D operator, parts a power of two dividing 2n");
        return IE_ERR_ARG;
    }
    return IE_OK;
}

int fft_M(const ie_fft* f) { return f->M; }

static void apply_peers(LineArgs& a, const PeerStores* ps) {
    if (!ps || !ps->mode) return;
    a.peer_mode = ps->mode;
    a.npeer = ps->npeer;
    a.peer_band_rows = ps->band_rows;
    for (int h = 0; h < ps->npeer; ++h) {
        a.peer[h] = ps->peer[h];
        a.peer_ctr[h] = ps->ctr[h];
        a.peer_line_bytes[h] = ps->line_bytes[h];
        a.peer_rlo[h] = ps->rlo[h];
        a.peer_rhi[h] = ps->rhi[h];
    }
}

int fft_band_fwd(const ie_fft* f, const double* X0, const double* X1, int nrows, int parts, double2* out,
                 const double* scales, cudaStream_t st, const int* stop, const PeerStores* ps) {
    int rc = band_check(f, parts);
    if (rc) return rc;
    const int n = f->n, Mc = f->M / parts;
    int lg = 0;
    while ((1 << lg) < Mc) ++lg;
    LineArgs a = base_args(f);
    a.nlines = nrows;
    a.ninner = 1;
    a.in_real = 1;
    a.x0 = X0;
    a.x1 = X1;
    a.in_so = n;
    a.in_sl = 1;
    a.n_in = n;
    a.out_c = out;
    a.out_so = Mc;
    a.out_sl = 1;
    a.out_lsplit = lg;
    a.out_sh = (int64_t)nrows * Mc;
    a.n_out = f->M;
    a.stop = stop;
    if (X1) {
        a.scales = scales;
        a.scale_in = 1;
    }
    apply_peers(a, ps);
    return line_launch(a, st);
}

int fft_band_cols(const ie_fft* f, double2* buf, int c0, int ncols, cudaStream_t st, const int* stop,
                  const PeerStores* ps) {
    int rc = band_check(f, 1);
    if (rc) return rc;
    if (ncols <= 0 || (ncols & (ncols - 1)) || c0 < 0 || c0 + ncols > f->M) {
        set_error("fft band_cols: column slab must be a power of two inside [0, 2n)");
        return IE_ERR_ARG;
    }
    LineArgs c = base_args(f);
    c.nlines = ncols;
    c.ninner = ncols;
    c.line0 = c0;
    c.in_c = buf;
    c.out_c = buf;
    c.in_si = c.out_si = 1;
    c.in_sl = c.out_sl = ncols;
    c.n_in = f->n;
    c.n_out = f->n;
    c.fused = 1;
    c.stop = stop;
    apply_peers(c, ps);
    return line_launch(c, st);
}

int fft_band_inv(const ie_fft* f, const double2* in, int nrows, int parts, double* Y0, double* Y1,
                 const double* scales, cudaStream_t st, const int* stop, const PcgFuse* fz) {
    int rc = band_check(f, parts);
    if (rc) return rc;
    const int n = f->n, Mc = f->M / parts;
    int lg = 0;
    while ((1 << lg) < Mc) ++lg;
    LineArgs e = base_args(f);
    e.nlines = nrows;
    e.ninner = 1;
    e.in_c = in;
    e.in_so = Mc;
    e.in_sl = 1;
    e.in_lsplit = lg;
    e.in_sh = (int64_t)nrows * Mc;
    e.n_in = f->M;
    e.out_real = 1;
    e.y0 = Y0;
    e.y1 = Y1;
    e.out_so = n;
    e.out_sl = 1;
    e.n_out = n;
    e.sign = +1;
    e.stop = stop;
    if (Y1) {
        e.scales = scales;
        e.scale_out = 1;
    }
    apply_fuse(e, fz);
    return line_launch(e, st);
}

int fft_absmax2(const double* X0, const double* X1, int64_t N, double* part, cudaStream_t st) {
    if (N <= 0) return IE_OK;
    k_absmax2<<<(unsigned)((N + 2047) / 2048), 256, 0, st>>>(X0, X1, (int)N, part, nullptr);
    IE_LAUNCHED();
    return IE_OK;
}

// Y0 (+ i Y1) = A (X0 + i X1) over all N rows.
int64_t fft_buf_elems(const ie_fft* f) {
    int64_t t = 1;
    for (int d = 0; d < f->dim; ++d) t *= (d == 0 ? f->n : f->M);
    return t;
}

// TMA descriptor of a 2D work buffer B (n rows of M complex) for the strided
// column pass: FP64 elements, inner dimension 2M doubles, boxes {2G, 256}.
// Built once per buffer address through the driver entry point (no libcuda
// link); false when unavailable (the pass then uses plain loads and stores).
static bool tma_map(ie_fft* f, const double2* B, int G, CUtensorMap* out) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    static bool tried = false;
    static std::mutex mu;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!tried) {
            tried = true;
            cudaDriverEntryPointQueryResult q;
            void* fn = nullptr;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
            cudaGetLastError();
        }
    }
    if (!enc) return false;
    std::lock_guard<std::mutex> lk(f->tm_mu);
    for (auto& e : f->tmaps)
        if (e.first == B) {
            *out = e.second;
            return true;
        }
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)2 * f->M, (cuuint64_t)f->n};
    const cuuint64_t strides[1] = {(cuuint64_t)f->M * 16};
    const cuuint32_t box[2] = {(cuuint32_t)(2 * G), 256u};
    const cuuint32_t estr[2] = {1u, 1u};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)B, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
        return false;
    f->tmaps.emplace_back(B, m);
    *out = m;
    return true;
}

// buf_ws / amax_ws: the calling stream's work buffer and chunk-maxima scratch
// (nullptr: the plan's own).  scales_ext: the 2-RHS column multipliers
// precomputed on the device (PCG); without them the pass reduces max|x_c|.
// can the PCG iteration fold k_iter_b / k_post_pass into this plan's passes
bool fft_fusable(const ie_fft* f) {
    static const bool v1 = getenv("IEDD_B200_FFT_V1") != nullptr;
    return f->dim >= 2 && f->logM >= 6 && !v1 && !getenv("IEDD_B200_NO_FUSE");
}

// output lines of the last (real-output) pass: 2D rows, 3D (a, b) lines
int fft_out_lines(const ie_fft* f) { return f->dim == 3 ? f->n * f->n : f->n; }

int fft_matvec(const ie_fft* f, const double* X0, const double* X1, double* Y0, double* Y1, cudaStream_t st,
               const int* stop, const double* scales_ext, double2* buf_ws, double* amax_ws, const PcgFuse* fz) {
    const int n = f->n, M = f->M, d = f->dim;
    int rc;
    const int two = X1 != nullptr;
    double* amax_own = amax_ws ? amax_ws : f->d_amax;
    if (two && !scales_ext) {
        k_absmax2<<<(f->N + 2047) / 2048, 256, 0, st>>>(X0, X1, f->N, amax_own, stop);
        IE_LAUNCHED();
    }
    auto line_launch = [&](LineArgs a, cudaStream_t s) -> int {
        a.stop = stop;
        a.amax = amax_own;
        a.scales = scales_ext;
        if (two) {
            a.scale_in = a.in_real;
            a.scale_out = a.out_real;
        }
        if (d >= 2) apply_fuse(a, fz);
        if (a.post_part && a.post_hi == 0) a.post_hi = a.nlines;
        return ::ie::line_launch(a, s);
    };
    if (d == 1) {
        LineArgs a = base_args(f);
        a.nlines = 1;
        a.ninner = 1;
        a.in_real = 1;
        a.x0 = X0;
        a.x1 = X1;
        a.in_sl = 1;
        a.n_in = n;
        a.out_real = 1;
        a.y0 = Y0;
        a.y1 = Y1;
        a.out_sl = 1;
        a.n_out = n;
        a.fused = 1;
        return line_launch(a, st);
    }
    double2* B = buf_ws ? buf_ws : f->d_buf;
    if (d == 2) {  // B: (n, M)
        LineArgs a = base_args(f);  // rows a < n, forward along axis 1
        a.nlines = n;
        a.ninner = 1;
        a.in_real = 1;
        a.x0 = X0;
        a.x1 = X1;
        a.in_so = n;
        a.in_sl = 1;
        a.n_in = n;
        a.out_c = B;
        a.out_so = M;
        a.out_sl = 1;
        a.n_out = M;
        if ((rc = line_launch(a, st))) return rc;
        LineArgs c = base_args(f);  // columns: forward * sym * inverse along axis 0
        c.nlines = M;
        c.ninner = M;
        c.in_c = B;
        c.out_c = B;
        c.in_si = c.out_si = 1;
        c.in_sl = c.out_sl = M;
        c.n_in = n;
        c.n_out = n;
        c.fused = 1;
        // TMA tile I/O when the strided launch uses two column lines per CTA
        static const bool no_tma = getenv("IEDD_B200_NO_TMA") != nullptr;
        if (!no_tma && n % 256 == 0 && M >= 64 && M <= 4096 && fft8_strided_g(M) == 2 &&
            tma_map(const_cast<ie_fft*>(f), B, 2, &c.tmap))
            c.tma = 1;
        if ((rc = line_launch(c, st))) return rc;
        LineArgs e = base_args(f);  // rows a < n, inverse along axis 1 -> real pair
        e.nlines = n;
        e.ninner = 1;
        e.in_c = B;
        e.in_so = M;
        e.in_sl = 1;
        e.n_in = M;
        e.out_real = 1;
        e.y0 = Y0;
        e.y1 = Y1;
        e.out_so = n;
        e.out_sl = 1;
        e.n_out = n;
        e.sign = +1;
        return line_launch(e, st);
    }
    // d == 3, B: (n, M, M)
    {
        LineArgs a = base_args(f);  // lines (a<n, b<n) along axis 2
        a.nlines = n * n;
        a.ninner = n;
        a.in_real = 1;
        a.x0 = X0;
        a.x1 = X1;
        a.in_so = (int64_t)n * n;
        a.in_si = n;
        a.in_sl = 1;
        a.n_in = n;
        a.out_c = B;
        a.out_so = (int64_t)M * M;
        a.out_si = M;
        a.out_sl = 1;
        a.n_out = M;
        if ((rc = line_launch(a, st))) return rc;
    }
    {
        LineArgs b = base_args(f);  // lines (a<n, k3) along axis 1, forward
        b.nlines = n * M;
        b.ninner = M;
        b.in_c = b.out_c = B;
        b.in_so = b.out_so = (int64_t)M * M;
        b.in_si = b.out_si = 1;
        b.in_sl = b.out_sl = M;
        b.n_in = n;
        b.n_out = M;
        if ((rc = line_launch(b, st))) return rc;
    }
    {
        LineArgs c = base_args(f);  // lines (k2, k3) along axis 0, fused
        c.nlines = M * M;
        c.ninner = M * M;
        c.in_c = c.out_c = B;
        c.in_si = c.out_si = 1;
        c.in_sl = c.out_sl = (int64_t)M * M;
        c.n_in = n;
        c.n_out = n;
        c.fused = 1;
        if ((rc = line_launch(c, st))) return rc;
    }
    {
        LineArgs b = base_args(f);  // lines (a<n, k3) along axis 1, inverse, keep b<n
        b.nlines = n * M;
        b.ninner = M;
        b.in_c = b.out_c = B;
        b.in_so = b.out_so = (int64_t)M * M;
        b.in_si = b.out_si = 1;
        b.in_sl = b.out_sl = M;
        b.n_in = M;
        b.n_out = n;
        b.sign = +1;
        if ((rc = line_launch(b, st))) return rc;
    }
    LineArgs e = base_args(f);  // lines (a<n, b<n) along axis 2, inverse -> real pair
    e.nlines = n * n;
    e.ninner = n;
    e.in_c = B;
    e.in_so = (int64_t)M * M;
    e.in_si = M;
    e.in_sl = 1;
    e.n_in = M;
    e.out_real = 1;
    e.y0 = Y0;
    e.y1 = Y1;
    e.out_so = (int64_t)n * n;
    e.out_si = n;
    e.out_sl = 1;
    e.n_out = n;
    e.sign = +1;
    return line_launch(e, st);
}

}  // namespace ie
