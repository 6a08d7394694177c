// Lab (not part of the library): 2048-point line FFT with 16 points per thread
// (128 threads per line: radix 16, 16, 8 -> two shared-memory exchanges instead
// of the three of the 8-points-per-thread kernel), vs cuFFT, on 1024
// contiguous lines and with 2 lines per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fft16_lab fft16_lab.cu -lcufft
#include <cuda_runtime.h>
#include <cufft.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

constexpr int L = 2048, TPL = 128;
__device__ __forceinline__ int padi(int i) { return i + (i >> 4); }

template <int S>
__device__ __forceinline__ void cmulw(double& xr, double& xi, double2 t) {
    const double ti = S < 0 ? t.y : -t.y;
    const double r = xr;
    xr = fma(r, t.x, -xi * ti);
    xi = fma(r, ti, xi * t.x);
}
// in-place DFT4 on (r[a], i[a]) a in {a0..a3}, natural order out
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
// DFT16 of v[0..15] (natural order in); output k = k1 + 4 k2 lands in slot 4 k1 + k2
template <int S>
__device__ __forceinline__ void dft16(double* r, double* i) {
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<S>(r, i, n2, n2 + 4, n2 + 8, n2 + 12);  // y[n2][k1] at n2 + 4 k1
    const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
    // twiddle W16^(n2 k1) at slot n2 + 4 k1
    const double wr[4][4] = {{1, 1, 1, 1}, {1, c1, h, s1}, {1, h, 0, -h}, {1, s1, -h, -c1}};
    const double wi[4][4] = {{0, 0, 0, 0}, {0, s1, h, c1}, {0, h, 1, h}, {0, c1, h, -s1}};
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
        for (int k1 = 1; k1 < 4; ++k1) {
            const int q = n2 + 4 * k1;
            const double a = wr[n2][k1], b = S * wi[n2][k1];  // exp(S 2 pi i n2 k1 / 16)
            const double xr = r[q];
            r[q] = a * xr - b * i[q];
            i[q] = a * i[q] + b * xr;
        }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<S>(r, i, 4 * k1, 4 * k1 + 1, 4 * k1 + 2, 4 * k1 + 3);  // X[k1 + 4 k2] at 4 k1 + k2
}
__device__ __forceinline__ int slot16(int k) { return 4 * (k & 3) + (k >> 2); }
template <int S>
__device__ __forceinline__ void dft8(double* r, double* i, int o) {  // on r[o + 2 q], q < 8? (generic: 8 values at stride 2)
    double xr[8], xi[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { xr[q] = r[o + 2 * q]; xi[q] = i[o + 2 * q]; }
    dft4<S>(xr, xi, 0, 2, 4, 6);
    dft4<S>(xr, xi, 1, 3, 5, 7);
    const double c = 0.70710678118654752440;
    { const double a = xr[3], b = xi[3]; xr[3] = c * (a - S * b); xi[3] = c * (b + S * a); }
    { const double a = xr[5]; xr[5] = -S * xi[5]; xi[5] = S * a; }
    { const double a = xr[7], b = xi[7]; xr[7] = c * (-a - S * b); xi[7] = c * (-b + S * a); }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        const double ar = xr[2 * k1], ai = xi[2 * k1], br = xr[2 * k1 + 1], bi = xi[2 * k1 + 1];
        xr[2 * k1] = ar + br; xi[2 * k1] = ai + bi;
        xr[2 * k1 + 1] = ar - br; xi[2 * k1 + 1] = ai - bi;
    }
    // output k at slot 2 (k & 3) + (k >> 2)
#pragma unroll
    for (int k = 0; k < 8; ++k) { r[o + 2 * k] = xr[2 * (k & 3) + (k >> 2)]; i[o + 2 * k] = xi[2 * (k & 3) + (k >> 2)]; }
}

// G lines per CTA, line g, thread j; register m <-> position j + 128 m
template <int S, int G>
__global__ void __launch_bounds__(TPL * G) k_fft16(const double2* __restrict__ in, double2* __restrict__ out,
                                                   const double2* __restrict__ t16, const double2* __restrict__ t2048) {
    constexpr int PITCH = L + L / 16 + 8;
    extern __shared__ double sm16[];
    double* sre = sm16;
    double* sim = sm16 + G * PITCH;
    const int g = threadIdx.x / TPL, j = threadIdx.x % TPL;
    const int line = blockIdx.x * G + g;
    double* re = sre + g * PITCH;
    double* im = sim + g * PITCH;
    const double2* x = in + (size_t)line * L;
    double vr[16], vi[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const double2 v = x[j + TPL * m];
        vr[m] = v.x;
        vi[m] = v.y;
    }
    // pass 1: Ns = 1, radix 16 -> positions 16 j + k
    dft16<S>(vr, vi);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int q = padi(16 * j + k);
        re[q] = vr[slot16(k)];
        im[q] = vi[slot16(k)];
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int q = padi(j + TPL * m);
        vr[m] = re[q];
        vi[m] = im[q];
    }
    // pass 2: Ns = 16, radix 16, k = j % 16, twiddle w^(k r) over 256
    {
        const int k = j & 15;
#pragma unroll
        for (int r = 1; r < 16; ++r) cmulw<S>(vr[r], vi[r], __ldg(t16 + r * 16 + k));
        dft16<S>(vr, vi);
        __syncthreads();
        const int base = (j >> 4) * 256 + k;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            const int q = padi(base + 16 * kk);
            re[q] = vr[slot16(kk)];
            im[q] = vi[slot16(kk)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int q = padi(j + TPL * m);
        vr[m] = re[q];
        vi[m] = im[q];
    }
    // pass 3: Ns = 256, radix 8, two butterflies b: jb = j + 128 b, inputs at m = b + 2 r
    double2* y = out + (size_t)line * L;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        const int jb = j + TPL * b;
#pragma unroll
        for (int r = 1; r < 8; ++r) cmulw<S>(vr[b + 2 * r], vi[b + 2 * r], __ldg(t2048 + r * 256 + jb));
        dft8<S>(vr, vi, b);
    }
    // outputs jb + 256 k = j + 128 (b + 2 k): register m = b + 2 k
#pragma unroll
    for (int m = 0; m < 16; ++m) y[j + TPL * m] = make_double2(vr[m], vi[m]);
}

static double2 tw(long m, long n) {
    const long double a = -2.0L * 3.141592653589793238462643383279502884L * m / n;
    return make_double2((double)cosl(a), (double)sinl(a));
}

int main() {
    const int nlines = 1024;
    const size_t N = (size_t)nlines * L;
    std::vector<double2> h(N);
    srand(1);
    for (auto& v : h) v = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
    std::vector<double2> h16(16 * 16), h2k(8 * 256);
    for (int r = 0; r < 16; ++r)
        for (int k = 0; k < 16; ++k) h16[r * 16 + k] = tw(r * k, 256);
    for (int r = 0; r < 8; ++r)
        for (int k = 0; k < 256; ++k) h2k[r * 256 + k] = tw(r * k, 2048);
    double2 *d_in, *d_out, *d_ref, *d16, *d2k;
    cudaMalloc(&d_in, N * 16);
    cudaMalloc(&d_out, N * 16);
    cudaMalloc(&d_ref, N * 16);
    cudaMalloc(&d16, h16.size() * 16);
    cudaMalloc(&d2k, h2k.size() * 16);
    cudaMemcpy(d_in, h.data(), N * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d16, h16.data(), h16.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d2k, h2k.data(), h2k.size() * 16, cudaMemcpyHostToDevice);
    cufftHandle plan;
    cufftPlan1d(&plan, L, CUFFT_Z2Z, nlines);
    cufftExecZ2Z(plan, (cufftDoubleComplex*)d_in, (cufftDoubleComplex*)d_ref, CUFFT_FORWARD);
    auto check = [&](const char* name) {
        std::vector<double2> a(N), b(N);
        cudaMemcpy(a.data(), d_out, N * 16, cudaMemcpyDeviceToHost);
        cudaMemcpy(b.data(), d_ref, N * 16, cudaMemcpyDeviceToHost);
        double num = 0, den = 0;
        for (size_t e = 0; e < N; ++e) {
            num += (a[e].x - b[e].x) * (a[e].x - b[e].x) + (a[e].y - b[e].y) * (a[e].y - b[e].y);
            den += b[e].x * b[e].x + b[e].y * b[e].y;
        }
        printf("%s rel err vs cuFFT: %.3e (%s)\n", name, sqrt(num / den), cudaGetErrorString(cudaGetLastError()));
    };
    const size_t sm1 = 2 * (size_t)(L + L / 16 + 8) * 8, sm2 = 2 * sm1;
    cudaFuncSetAttribute(k_fft16<-1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    cudaFuncSetAttribute(k_fft16<-1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    k_fft16<-1, 1><<<nlines, TPL, sm1>>>(d_in, d_out, d16, d2k);
    cudaDeviceSynchronize();
    check("fft16 G1");
    k_fft16<-1, 2><<<nlines / 2, 2 * TPL, sm2>>>(d_in, d_out, d16, d2k);
    cudaDeviceSynchronize();
    check("fft16 G2");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0);
        for (int it = 0; it < 50; ++it) k_fft16<-1, 1><<<nlines, TPL, sm1>>>(d_in, d_out, d16, d2k);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("k_fft16 G1: %.2f us per 1024 lines\n", ms * 1000 / 50);
        cudaEventRecord(e0);
        for (int it = 0; it < 50; ++it) k_fft16<-1, 2><<<nlines / 2, 2 * TPL, sm2>>>(d_in, d_out, d16, d2k);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("k_fft16 G2: %.2f us per 1024 lines\n", ms * 1000 / 50);
        cudaEventRecord(e0);
        for (int it = 0; it < 50; ++it)
            cufftExecZ2Z(plan, (cufftDoubleComplex*)d_in, (cufftDoubleComplex*)d_ref, CUFFT_FORWARD);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("cuFFT     : %.2f us per 1024 lines\n", ms * 1000 / 50);
    }
    return 0;
}
