// Isolated timing of the register-row LDLT step loop (as in ffcp.cu warp_ldlt_reg).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __noinline__ void ldlt_reg(const double* t, int R, double* f, double* colk, long long* st) {
    const int lane = threadIdx.x & 31;
    double row[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) row[j] = (lane < R && j < R) ? t[lane + j * R] : 0.0;
    long long t0 = clock64();
#pragma unroll 1
    for (int k = 0; k < R; ++k) {
        double rk = 0.0;
        switch (k) {  // row[k]: k is warp-uniform, so one indexed branch instead of a select chain
#define TK_ROW_CASE(c) \
    case c:            \
        rk = row[c];   \
        break;
            TK_ROW_CASE(0) TK_ROW_CASE(1) TK_ROW_CASE(2) TK_ROW_CASE(3) TK_ROW_CASE(4) TK_ROW_CASE(5) TK_ROW_CASE(6)
            TK_ROW_CASE(7) TK_ROW_CASE(8) TK_ROW_CASE(9) TK_ROW_CASE(10) TK_ROW_CASE(11) TK_ROW_CASE(12)
            TK_ROW_CASE(13) TK_ROW_CASE(14) TK_ROW_CASE(15) TK_ROW_CASE(16) TK_ROW_CASE(17) TK_ROW_CASE(18)
            TK_ROW_CASE(19) TK_ROW_CASE(20) TK_ROW_CASE(21) TK_ROW_CASE(22) TK_ROW_CASE(23) TK_ROW_CASE(24)
            TK_ROW_CASE(25) TK_ROW_CASE(26) TK_ROW_CASE(27) TK_ROW_CASE(28) TK_ROW_CASE(29) TK_ROW_CASE(30)
            TK_ROW_CASE(31)
#undef TK_ROW_CASE
            default:
                break;
        }
        const double d = __shfl_sync(0xffffffffu, rk, k);
        const bool nz = fabs(d) > 0.0;
        const double inv = nz ? 1.0 / d : 0.0;
        const double l = (lane > k && lane < R) ? (nz ? rk * inv : rk) : 0.0;
        if (lane > k && lane < R) f[lane + k * R] = l;
        if (lane == k) f[k + k * R] = d;
        colk[lane] = l * d;  // L(j,k) D(k), zero for j <= k
        __syncwarp();
        // trailing update of the whole row, no masks: entries above the diagonal are never
        // read (row[k] of lane k is the diagonal; lanes i < k have l = 0)
#pragma unroll
        for (int j = 0; j < 32; ++j) row[j] = fma(-l, colk[j], row[j]);
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) st[0] = t1 - t0;
}

__global__ void k_ldlt(const double* t, int R, long long* st, double* out) {
    __shared__ double f[32 * 32];
    __shared__ double colk[32];
    __shared__ double ts[32 * 32];
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) ts[e] = t[e];
    __syncwarp();
    ldlt_reg(ts, R, f, colk, st);
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = f[e];
}

int main() {
    const int R = 20;
    double h[R * R];
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) h[i + j * R] = (i == j ? R + 1.0 : 1.0 / (1 + i + j));
    double *t, *out; long long* st;
    cudaMalloc(&t, sizeof(h)); cudaMalloc(&out, sizeof(h)); cudaMalloc(&st, 64);
    cudaMemcpy(t, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) k_ldlt<<<1, 32>>>(t, R, st, out);
    long long hs[1];
    cudaMemcpy(hs, st, 8, cudaMemcpyDeviceToHost);
    printf("reg ldlt R=%d: %lld cycles (%.0f per step)\n", R, hs[0], double(hs[0]) / R);
    return 0;
}
