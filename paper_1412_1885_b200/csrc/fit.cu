// fit.cu — streaming fit of a Tucker or CP model against a dense tensor, without
// materialising the reconstruction.
//
// Reference: fit (tensor.hpp:282-290) = 1 - ||Y - Yhat||_F / ||Y||_F, with Yhat =
// reconstruct(TuckerModel) (tucker.hpp:63-66) or cp_reconstruct(CpModel) (cp.hpp:118-128),
// as the bench reports fit_obs / fit_gt (bench.hpp:521,530-531). Y is viewed as
// (I_0, I_1, T) with T = prod_{n>=2} I_n; the model is folded into
//     Yhat[:, :, t] = U_0 W_t U_1^T,
// W_t = G x_{n>=2} U_n[i_n(t), :] (Tucker) or diag(prod_{n>=2} A_n[i_n(t), :]) (CP), so one
// pass streams Y once, rebuilds each 64 x 64 tile of a slab in shared memory (fp64) and
// accumulates (y - yhat)^2 and y^2 in fp64. Per-CTA partial sums are reduced in fixed order.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "../../include/tenkit_b200.h"
#include "kernels.cuh"

namespace tkb {
namespace {

constexpr int kFT = 64;        // tile edge (rows of mode 0 and of mode 1)
constexpr int kFThreads = 256;

// out[p + i P + q P I] = sum_r in[p + r P + q P R] u[i + r I]   (X x_n U, U: I x R col-major)
__global__ void expand_mode_kernel(const double* __restrict__ in, const double* __restrict__ u, int64_t P, int R,
                                   int64_t I, int64_t Q, double* __restrict__ out) {
    const int64_t n = P * I * Q;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = t % P, i = (t / P) % I, q = t / (P * I);
        const double* src = in + p + q * P * R;
        double s = 0.0;
        for (int r = 0; r < R; ++r) s = fma(src[r * P], u[i + r * I], s);
        out[t] = s;
    }
}

// c[t + r T] = prod_{n >= 2} A_n[i_n(t), r]  (the Khatri-Rao rows of the trailing modes)
struct KrDesc {
    int nm;                      // trailing modes (order - 2)
    int64_t dims[TK_MAX_ORDER];  // their extents
    const double* a[TK_MAX_ORDER];
};
__global__ void kr_rows_kernel(KrDesc d, int64_t T, int R, double* __restrict__ c) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < T * R; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t t = e % T;
        const int r = static_cast<int>(e / T);
        int64_t rem = t;
        double v = 1.0;
        for (int m = 0; m < d.nm; ++m) {
            const int64_t i = rem % d.dims[m];
            rem /= d.dims[m];
            v *= d.a[m][i + int64_t(r) * d.dims[m]];
        }
        c[e] = v;
    }
}

// One CTA: a 64 x 64 (i0, i1) tile for slabs t = blockIdx.z, blockIdx.z + gridDim.z, ...
// W: diag == 0 -> W_t = w[a + b R0 + t R0 R1]; diag == 1 -> W_t = diag(w[t + b T]) (R0 == R1).
template <typename T>
__global__ void __launch_bounds__(kFThreads) fit_tile_kernel(const T* __restrict__ y, int64_t I0, int64_t I1,
                                                             int64_t NT, const double* __restrict__ u0,
                                                             const double* __restrict__ u1, int R0, int R1,
                                                             const double* __restrict__ w, int diag,
                                                             double* __restrict__ partial) {
    extern __shared__ double fsm[];
    double* s0 = fsm;                 // [R0][kFT]  U0 rows of the tile (transposed)
    double* s1 = s0 + R0 * kFT;       // [R1][kFT]  U1 rows
    double* sw = s1 + R1 * kFT;       // [R0][R1]
    double* sm = sw + R0 * R1;        // [R1][kFT]  M = U0_tile W_t
    __shared__ double red[2][kFThreads];
    const int tid = threadIdx.x;
    const int64_t r0 = int64_t(blockIdx.x) * kFT, c0 = int64_t(blockIdx.y) * kFT;
    const int nr = static_cast<int>(I0 - r0 < kFT ? I0 - r0 : kFT), nc = static_cast<int>(I1 - c0 < kFT ? I1 - c0 : kFT);
    for (int e = tid; e < R0 * kFT; e += kFThreads) {
        const int i = e % kFT, a = e / kFT;
        s0[e] = i < nr ? u0[r0 + i + int64_t(a) * I0] : 0.0;
    }
    for (int e = tid; e < R1 * kFT; e += kFThreads) {
        const int i = e % kFT, b = e / kFT;
        s1[e] = i < nc ? u1[c0 + i + int64_t(b) * I1] : 0.0;
    }
    // thread -> 4 x 4 outputs: rows tx + 16 i (coalesced along mode 0), cols ty * 4 + j
    const int tx = tid % 16, ty = tid / 16;
    double acc_r = 0.0, acc_y = 0.0;
    for (int64_t t = blockIdx.z; t < NT; t += gridDim.z) {
        __syncthreads();  // previous slab done with sw / sm
        if (diag) {
            for (int e = tid; e < R0 * R1; e += kFThreads) sw[e] = 0.0;
            __syncthreads();
            for (int b = tid; b < R1; b += kFThreads) sw[b + b * R0] = w[t + int64_t(b) * NT];
        } else {
            for (int e = tid; e < R0 * R1; e += kFThreads) sw[e] = w[e + t * R0 * R1];
        }
        __syncthreads();
        for (int e = tid; e < R1 * kFT; e += kFThreads) {  // M[i][b] = sum_a U0[i][a] W[a][b]
            const int i = e % kFT, b = e / kFT;
            double s = 0.0;
            for (int a = 0; a < R0; ++a) s = fma(s0[i + a * kFT], sw[a + b * R0], s);
            sm[e] = s;
        }
        __syncthreads();
        double yh[4][4];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) yh[ii][jj] = 0.0;
        for (int b = 0; b < R1; ++b) {
            double mv[4], uv[4];
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) mv[ii] = sm[tx + 16 * ii + b * kFT];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) uv[jj] = s1[ty * 4 + jj + b * kFT];
#pragma unroll
            for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) yh[ii][jj] = fma(mv[ii], uv[jj], yh[ii][jj]);
        }
        const T* ys = y + t * I0 * I1;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int cc = ty * 4 + jj;
            if (cc >= nc) continue;
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) {
                const int rr = tx + 16 * ii;
                if (rr >= nr) continue;
                const double v = static_cast<double>(ys[r0 + rr + (c0 + cc) * I0]);
                const double d = v - yh[ii][jj];
                acc_r = fma(d, d, acc_r);
                acc_y = fma(v, v, acc_y);
            }
        }
    }
    red[0][tid] = acc_r;
    red[1][tid] = acc_y;
    __syncthreads();
    for (int s = kFThreads / 2; s > 0; s >>= 1) {
        if (tid < s) {
            red[0][tid] += red[0][tid + s];
            red[1][tid] += red[1][tid + s];
        }
        __syncthreads();
    }
    if (tid == 0) {
        const int64_t cta = blockIdx.x + int64_t(gridDim.x) * (blockIdx.y + int64_t(gridDim.y) * blockIdx.z);
        partial[2 * cta] = red[0][0];
        partial[2 * cta + 1] = red[1][0];
    }
}

__global__ void fit_final_kernel(const double* __restrict__ partial, int64_t n, double* __restrict__ out) {
    __shared__ double red[2][kFThreads];
    double a = 0.0, b = 0.0;
    for (int64_t e = threadIdx.x; e < n; e += kFThreads) {
        a += partial[2 * e];
        b += partial[2 * e + 1];
    }
    red[0][threadIdx.x] = a;
    red[1][threadIdx.x] = b;
    __syncthreads();
    for (int s = kFThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            red[0][threadIdx.x] += red[0][threadIdx.x + s];
            red[1][threadIdx.x] += red[1][threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = red[0][0];  // ||Y - Yhat||^2
        out[1] = red[1][0];  // ||Y||^2
    }
}

inline unsigned blocks_for(int64_t n) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
}

}  // namespace

// ||Y - Yhat||^2 and ||Y||^2 into sums[0..1] (device). Tucker: core (core_shape) + factors
// (I_n x core_shape[n]); CP (core == nullptr): factors I_n x rank. All device pointers.
template <typename T>
void launch_model_fit(BufPool& pool, const T* y, int order, const int64_t* dims, const double* core,
                      const int64_t* core_shape, const double* const* factors, int64_t rank, double* sums,
                      cudaStream_t s) {
    require(order >= 2 && order <= TK_MAX_ORDER, "fit: tensor order must be in [2, 8]");
    const bool cp = core == nullptr;
    const int R0 = static_cast<int>(cp ? rank : core_shape[0]);
    const int R1 = static_cast<int>(cp ? rank : core_shape[1]);
    require(R0 >= 1 && R1 >= 1 && R0 <= kMaxRank && R1 <= kMaxRank, "fit: model ranks must be in [1, 64]");
    int64_t NT = 1;
    for (int n = 2; n < order; ++n) NT *= dims[n];
    const double* w = nullptr;
    if (cp) {
        double* c = static_cast<double*>(pool.get("fit_kr", sizeof(double) * NT * R0));
        KrDesc d{};
        d.nm = order - 2;
        for (int m = 0; m < d.nm; ++m) {
            d.dims[m] = dims[m + 2];
            d.a[m] = factors[m + 2];
        }
        kr_rows_kernel<<<blocks_for(NT * R0), 256, 0, s>>>(d, NT, R0, c);
        w = c;
    } else {
        // W = G x_2 U_2 ... x_{N-1} U_{N-1}: (R0, R1, I_2, ..., I_{N-1})
        std::vector<int64_t> cur(core_shape, core_shape + order);
        const double* src = core;
        int which = 0;
        for (int n = 2; n < order; ++n) {
            int64_t P = 1, Q = 1;
            for (int k = 0; k < n; ++k) P *= cur[k];
            for (int k = n + 1; k < order; ++k) Q *= cur[k];
            double* dst = static_cast<double*>(pool.get(which ? "fit_wB" : "fit_wA", sizeof(double) * P * dims[n] * Q));
            expand_mode_kernel<<<blocks_for(P * dims[n] * Q), 256, 0, s>>>(src, factors[n], P, static_cast<int>(cur[n]),
                                                                          dims[n], Q, dst);
            cur[n] = dims[n];
            src = dst;
            which ^= 1;
        }
        w = src;
    }
    const unsigned gx = static_cast<unsigned>((dims[0] + kFT - 1) / kFT), gy = static_cast<unsigned>((dims[1] + kFT - 1) / kFT);
    const unsigned gz = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(NT, (148 * 8 + gx * gy - 1) / (gx * gy))));
    const int64_t nblk = int64_t(gx) * gy * gz;
    double* partial = static_cast<double*>(pool.get("fit_partial", sizeof(double) * 2 * nblk));
    const size_t smem = sizeof(double) * (size_t(R0) * kFT + 2 * size_t(R1) * kFT + size_t(R0) * R1);
    static bool attr = false;
    if (!attr) {
        TK_CUDA(cudaFuncSetAttribute(fit_tile_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        TK_CUDA(cudaFuncSetAttribute(fit_tile_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        attr = true;
    }
    fit_tile_kernel<T><<<dim3(gx, gy, gz), kFThreads, smem, s>>>(y, dims[0], dims[1], NT, factors[0], factors[1], R0, R1,
                                                                 w, cp ? 1 : 0, partial);
    fit_final_kernel<<<1, kFThreads, 0, s>>>(partial, nblk, sums);
    TK_LAUNCH_CHECK();
}

template void launch_model_fit<float>(BufPool&, const float*, int, const int64_t*, const double*, const int64_t*,
                                      const double* const*, int64_t, double*, cudaStream_t);
template void launch_model_fit<double>(BufPool&, const double*, int, const int64_t*, const double*, const int64_t*,
                                       const double* const*, int64_t, double*, cudaStream_t);

}  // namespace tkb
