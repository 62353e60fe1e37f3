// Latency microbenchmarks on sm_100a (clock64, one warp): dependent DFMA, DDIV, DSQRT, FFMA,
// shared-memory load chains, SHFL chains. Informs the latency-bound FFCP/QR kernels.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double* out, long long* cyc, int n, double seed) {
    __shared__ double sm[1024];
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        sm[i] = 1.0 + i * 1e-9;
        idx[i] = (i * 17 + 5) & 1023;
    }
    __syncthreads();
    double a = seed, b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    double d = seed + 2.0;
    for (int i = 0; i < n; ++i) d = 1.0 / (d + 1e-3);
    long long t2 = clock64();
    double e = seed + 3.0;
    for (int i = 0; i < n; ++i) e = sqrt(e + 1.0);
    long long t3 = clock64();
    float f = (float)seed;
    for (int i = 0; i < n; ++i) f = fmaf(f, 1.0000001f, 1e-9f);
    long long t4 = clock64();
    int p = threadIdx.x & 31;
    for (int i = 0; i < n; ++i) p = idx[p];
    long long t5 = clock64();
    double g = seed;
    for (int i = 0; i < n; ++i) g = __shfl_sync(0xffffffffu, g, (threadIdx.x + 1) & 31) + 1e-12;
    long long t6 = clock64();
    double h = seed;
    for (int i = 0; i < n; ++i) h = h / (seed + 1.5 + i * 1e-12);
    long long t7 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6;
    }
    out[threadIdx.x] = a + d + e + f + p + g + h;
}

int main() {
    double* out; long long* cyc; cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 64 * 8);
    const int n = 1000;
    for (int rep = 0; rep < 2; ++rep) lat_kernel<<<1, 32>>>(out, cyc, n, 0.5);
    long long h[8];
    cudaMemcpy(h, cyc, 7 * 8, cudaMemcpyDeviceToHost);
    const char* names[] = {"DFMA", "1/x (DDIV-rcp)", "DSQRT", "FFMA", "LDS chain (int)", "SHFL.f64 chain", "DDIV x/y"};
    for (int i = 0; i < 7; ++i) printf("%-18s %.1f cycles/op\n", names[i], double(h[i]) / n);
    return 0;
}
