// Isolated timing of the warp LDLT factor loop used by the persistent FFCP kernel.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __noinline__ void factor(double* a, double* mm, int R, long long* st) {
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (int k = 0; k < R; ++k) {
        long long t0 = clock64();
        const double* mk = mm + k;
#pragma unroll 1
        for (int i = k + lane; i < R; i += 32) {
            double p0 = 0.0, p1 = 0.0;
            int j = 0;
#pragma unroll 1
            for (; j + 2 <= k; j += 2) {
                p0 = fma(a[i + j * R], mk[j * R], p0);
                p1 = fma(a[i + (j + 1) * R], mk[(j + 1) * R], p1);
            }
            if (j < k) p0 = fma(a[i + j * R], mk[j * R], p0);
            mm[i + k * R] = a[i + k * R] - (p0 + p1);
        }
        __syncwarp();
        long long t1 = clock64();
        const double dk = mm[k + k * R];
        const bool nz = fabs(dk) > 0.0;
#pragma unroll 1
        for (int i = k + lane; i < R; i += 32) {
            const double sv = mm[i + k * R];
            a[i + k * R] = i == k ? dk : (nz ? sv / dk : sv);
        }
        __syncwarp();
        long long t2 = clock64();
        if (lane == 0) { st[2 * k] = t1 - t0; st[2 * k + 1] = t2 - t1; }
    }
}

__global__ void k_ldlt(const double* t, int R, long long* st, double* out) {
    extern __shared__ double sm[];
    double* a = sm;
    double* mm = sm + R * R;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) a[e] = t[e];
    __syncwarp();
    long long t0 = clock64();
    factor(a, mm, R, st);
    long long t1 = clock64();
    if (threadIdx.x == 0) st[200] = t1 - t0;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = a[e];
}

int main() {
    const int R = 20;
    double h[R * R];
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) h[i + j * R] = (i == j ? R + 1.0 : 1.0 / (1 + i + j));
    double *t, *out; long long* st;
    cudaMalloc(&t, sizeof(h)); cudaMalloc(&out, sizeof(h)); cudaMalloc(&st, 256 * 8);
    cudaMemcpy(t, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) k_ldlt<<<1, 32, 2 * R * R * 8>>>(t, R, st, out);
    long long hs[256];
    cudaMemcpy(hs, st, sizeof(hs), cudaMemcpyDeviceToHost);
    printf("total %lld cycles\n", hs[200]);
    for (int k = 0; k < R; k += 4) printf("  k=%2d dot %lld div %lld\n", k, hs[2 * k], hs[2 * k + 1]);
    return 0;
}
