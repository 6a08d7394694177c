// FFT lab (not part of the library): a 2048-point radix-8 Stockham variant
// with 8 points per thread (one line per 256-thread CTA, first-pass inputs
// straight from the line load, last-pass outputs straight to global), timed
// on 1024 contiguous complex lines and checked against cuFFT.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fft_lab fft_lab.cu -lcufft
#include <cuda_runtime.h>
#include <cufft.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

constexpr int L = 2048, TPB = 256;
__device__ __forceinline__ int padi(int i) { return i + (i >> 4); }

template <int S>
__device__ __forceinline__ void cmul(double& xr, double& xi, double2 t) {
    const double ti = S < 0 ? t.y : -t.y;
    const double r = xr;
    xr = fma(r, t.x, -xi * ti);
    xi = fma(r, ti, xi * t.x);
}

template <int S>
__device__ __forceinline__ void dft4(double* r, double* i, int a0, int a1, int a2, int a3) {
    const double s0r = r[a0] + r[a2], s0i = i[a0] + i[a2], d0r = r[a0] - r[a2], d0i = i[a0] - i[a2];
    const double s1r = r[a1] + r[a3], s1i = i[a1] + i[a3], d1r = r[a1] - r[a3], d1i = i[a1] - i[a3];
    const double er = -S * d1i, ei = S * d1r;
    r[a0] = s0r + s1r; i[a0] = s0i + s1i;
    r[a2] = s0r - s1r; i[a2] = s0i - s1i;
    r[a1] = d0r + er; i[a1] = d0i + ei;
    r[a3] = d0r - er; i[a3] = d0i - ei;
}

// 8-point DFT, natural order in, output k at slot out8(k) = 2*(k&3) + (k>>2)
template <int S>
__device__ __forceinline__ void dft8(double* r, double* i) {
    dft4<S>(r, i, 0, 2, 4, 6);
    dft4<S>(r, i, 1, 3, 5, 7);
    const double c = 0.70710678118654752440;
    {  // * w8^1
        const double xr = r[3], xi = i[3];
        r[3] = c * (xr - S * xi);
        i[3] = c * (xi + S * xr);
    }
    {  // * w8^2 = S i
        const double xr = r[5];
        r[5] = -S * i[5];
        i[5] = S * xr;
    }
    {  // * w8^3
        const double xr = r[7], xi = i[7];
        r[7] = c * (-xr - S * xi);
        i[7] = c * (-xi + S * xr);
    }
    for (int k1 = 0; k1 < 4; ++k1) {
        const double ar = r[2 * k1], ai = i[2 * k1], br = r[2 * k1 + 1], bi = i[2 * k1 + 1];
        r[2 * k1] = ar + br; i[2 * k1] = ai + bi;
        r[2 * k1 + 1] = ar - br; i[2 * k1 + 1] = ai - bi;
    }
}
__device__ __forceinline__ int out8(int k) { return 2 * (k & 3) + (k >> 2); }
__device__ __forceinline__ int out4(int k) { return k; }

// tw tables (global, radix-major): pass Ns: t[r * Ns + k] = exp(-2 pi i r k / (R Ns))
template <int S>
__global__ void __launch_bounds__(TPB, 4) k_fft8(const double2* __restrict__ in, double2* __restrict__ out,
                                                 const double2* __restrict__ t8, const double2* __restrict__ t64,
                                                 const double2* __restrict__ t512) {
    __shared__ double sre[L + L / 16], sim[L + L / 16];
    const int line = blockIdx.x, t = threadIdx.x;
    const double2* x = in + (size_t)line * L;
    double vr[8], vi[8];
    // pass 1 (Ns = 1, radix 8): inputs t + 256 r
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const double2 v = x[t + 256 * r];
        vr[r] = v.x;
        vi[r] = v.y;
    }
    dft8<S>(vr, vi);
    // Stockham: j = t, Ns = 1: output index (j/Ns)*Ns*R + j%Ns + Ns*r = 8 t + r
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int q = padi(8 * t + r);
        sre[q] = vr[out8(r)];
        sim[q] = vi[out8(r)];
    }
    __syncthreads();
    // pass 2 (Ns = 8, radix 8): j = t, inputs j + 256 r, k = j % 8
    {
        const int k = t & 7;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = padi(t + 256 * r);
            vr[r] = sre[q];
            vi[r] = sim[q];
        }
#pragma unroll
        for (int r = 1; r < 8; ++r) cmul<S>(vr[r], vi[r], __ldg(t8 + r * 8 + k));
        dft8<S>(vr, vi);
        __syncthreads();
        const int base = (t >> 3) * 64 + k;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = padi(base + 8 * r);
            sre[q] = vr[out8(r)];
            sim[q] = vi[out8(r)];
        }
    }
    __syncthreads();
    // pass 3 (Ns = 64, radix 8)
    {
        const int k = t & 63;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = padi(t + 256 * r);
            vr[r] = sre[q];
            vi[r] = sim[q];
        }
#pragma unroll
        for (int r = 1; r < 8; ++r) cmul<S>(vr[r], vi[r], __ldg(t64 + r * 64 + k));
        dft8<S>(vr, vi);
        __syncthreads();
        const int base = (t >> 6) * 512 + k;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int q = padi(base + 64 * r);
            sre[q] = vr[out8(r)];
            sim[q] = vi[out8(r)];
        }
    }
    __syncthreads();
    // pass 4 (Ns = 512, radix 4): 512 butterflies, two per thread: j = t, t + 256
    double2* y = out + (size_t)line * L;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        const int j = t + 256 * b;
        double wr[4], wi[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int q = padi(j + 512 * r);
            wr[r] = sre[q];
            wi[r] = sim[q];
        }
#pragma unroll
        for (int r = 1; r < 4; ++r) cmul<S>(wr[r], wi[r], __ldg(t512 + r * 512 + j));
        dft4<S>(wr, wi, 0, 1, 2, 3);
#pragma unroll
        for (int r = 0; r < 4; ++r) y[j + 512 * r] = make_double2(wr[r], wi[r]);
    }
}

static double2 tw(int m, int n) {
    const long double a = -2.0L * 3.141592653589793238462643383279502884L * m / n;
    return make_double2((double)cosl(a), (double)sinl(a));
}

int main() {
    const int nlines = 1024;
    const size_t N = (size_t)nlines * L;
    std::vector<double2> h(N);
    srand(1);
    for (auto& v : h) v = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
    std::vector<double2> h8(8 * 8), h64(8 * 64), h512(4 * 512);
    for (int r = 0; r < 8; ++r)
        for (int k = 0; k < 8; ++k) h8[r * 8 + k] = tw(r * k, 64);
    for (int r = 0; r < 8; ++r)
        for (int k = 0; k < 64; ++k) h64[r * 64 + k] = tw(r * k, 512);
    for (int r = 0; r < 4; ++r)
        for (int k = 0; k < 512; ++k) h512[r * 512 + k] = tw(r * k, 2048);
    double2 *d_in, *d_out, *d_ref, *d8, *d64, *d512;
    cudaMalloc(&d_in, N * 16);
    cudaMalloc(&d_out, N * 16);
    cudaMalloc(&d_ref, N * 16);
    cudaMalloc(&d8, h8.size() * 16);
    cudaMalloc(&d64, h64.size() * 16);
    cudaMalloc(&d512, h512.size() * 16);
    cudaMemcpy(d_in, h.data(), N * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d8, h8.data(), h8.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d64, h64.data(), h64.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d512, h512.data(), h512.size() * 16, cudaMemcpyHostToDevice);
    cufftHandle plan;
    cufftPlan1d(&plan, L, CUFFT_Z2Z, nlines);
    cufftExecZ2Z(plan, (cufftDoubleComplex*)d_in, (cufftDoubleComplex*)d_ref, CUFFT_FORWARD);
    k_fft8<-1><<<nlines, TPB>>>(d_in, d_out, d8, d64, d512);
    cudaDeviceSynchronize();
    std::vector<double2> a(N), b(N);
    cudaMemcpy(a.data(), d_out, N * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), d_ref, N * 16, cudaMemcpyDeviceToHost);
    double num = 0, den = 0;
    for (size_t e = 0; e < N; ++e) {
        num += (a[e].x - b[e].x) * (a[e].x - b[e].x) + (a[e].y - b[e].y) * (a[e].y - b[e].y);
        den += b[e].x * b[e].x + b[e].y * b[e].y;
    }
    printf("rel err vs cuFFT: %.3e  (%s)\n", sqrt(num / den), cudaGetErrorString(cudaGetLastError()));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 50; ++it) k_fft8<-1><<<nlines, TPB>>>(d_in, d_out, d8, d64, d512);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("k_fft8: %.2f us per 1024 lines\n", ms * 1000 / 50);
        cudaEventRecord(e0);
        for (int it = 0; it < 50; ++it)
            cufftExecZ2Z(plan, (cufftDoubleComplex*)d_in, (cufftDoubleComplex*)d_ref, CUFFT_FORWARD);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("cuFFT : %.2f us per 1024 lines\n", ms * 1000 / 50);
    }
    return 0;
}
