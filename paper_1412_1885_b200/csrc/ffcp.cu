// ffcp.cu — FFCP (flexible fast CP on the Tucker-compressed tensor) on the device, fp64.
//
// Reference: ffcp (ffcp.hpp:94-194), ffcp_h (:33-47), solve_normal / hals_sweep /
// absorb_scales (cp.hpp:63-109). Every operand is core-sized (R~^N) or an I_n x R matrix,
// so each sweep is a handful of small kernels; one sweep (all modes) is captured once as a
// CUDA graph and replayed, with the compressed-space fit read back after every sweep for
// the stopping rule |fit - prev| < fit_tol (identical iteration count to the reference).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tenkit_b200.h"
#include "kernels.cuh"

namespace tkb {
namespace {

constexpr int kMaxOrder = TK_MAX_ORDER;

struct CoreDesc {
    int order;
    int cs[kMaxOrder];        // core extents
    int64_t stride[kMaxOrder];
    const double* V[kMaxOrder];  // V_p = U_p^T A_p (cs[p] x R, column-major)
};

inline unsigned nblocks(int64_t n, int per = 256) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 32)));
}

// Diagonal contraction of one mode q of W against V_q[:, r], where r is W's mode `rpos`:
// out[..., r, ...] = sum_i W[..., i (mode q), ..., r, ...] V_q[i, r]  (mode q removed).
// dims/ndim describe W (column-major); one thread per output element.
struct WDesc {
    int ndim;
    int64_t dims[kMaxOrder];
};
__global__ void diag_contract_kernel(const double* __restrict__ w, WDesc d, int q, int rpos, const double* __restrict__ v,
                                     int ldv, double* __restrict__ out) {
    int64_t before = 1, after = 1;
    for (int k = 0; k < q; ++k) before *= d.dims[k];
    for (int k = q + 1; k < d.ndim; ++k) after *= d.dims[k];
    int64_t rstride = 1;  // stride of the r index in the OUTPUT (mode q removed)
    for (int k = 0; k < rpos; ++k)
        if (k != q) rstride *= d.dims[k];
    const int64_t rdim = d.dims[rpos];
    const int64_t nq = d.dims[q];
    const int64_t total = before * after;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = t % before, a = t / before;
        const int64_t r = (t / rstride) % rdim;
        const double* src = w + b + a * before * nq;
        const double* vr = v + r * ldv;
        double acc = 0.0;
        for (int64_t i = 0; i < nq; ++i) acc = fma(src[i * before], vr[i], acc);
        out[t] = acc;
    }
}

__global__ void finalize_h_kernel(const double* __restrict__ w, int cn, int R, bool transposed, double* __restrict__ h) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cn * R; t += gridDim.x * blockDim.x) {
        const int i = t % cn, r = t / cn;
        h[t] = transposed ? w[r + i * R] : w[t];
    }
}

// C (m x n) = A (m x k, lda) * B (k x n, ldb), one thread per output
__global__ void matmul_nn_kernel(const double* __restrict__ a, int64_t lda, const double* __restrict__ b, int64_t ldb,
                                 double* __restrict__ c, int64_t m, int k, int n) {
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < m * n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = t % m, j = t / m;
        double s = 0.0;
        for (int l = 0; l < k; ++l) s = fma(a[i + l * lda], b[l + j * ldb], s);
        c[t] = s;
    }
}

// C (m x n) = A^T B, A (k x m, lda), B (k x n, ldb): one warp per output, lanes over k
__global__ void matmul_tn_kernel(const double* __restrict__ a, int64_t lda, const double* __restrict__ b, int64_t ldb,
                                 double* __restrict__ c, int m, int64_t k, int n) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = int64_t(gridDim.x) * (blockDim.x / 32);
    for (int64_t o = blockIdx.x * int64_t(blockDim.x / 32) + threadIdx.x / 32; o < int64_t(m) * n; o += nw) {
        const int i = static_cast<int>(o % m), j = static_cast<int>(o / m);
        const double* ac = a + int64_t(i) * lda;
        const double* bc = b + int64_t(j) * ldb;
        double s = 0.0;
        for (int64_t l = lane; l < k; l += 32) s = fma(ac[l], bc[l], s);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) c[o] = s;
    }
}

// T = Hadamard product of the Grams of every mode except n (R x R)
__global__ void hadamard_kernel(const double* const* grams, int order, int n, int R, double* __restrict__ t) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < R * R; e += gridDim.x * blockDim.x) {
        double v = 1.0;
        for (int p = 0; p < order; ++p)
            if (p != n) v *= grams[p][e];
        t[e] = v;
    }
}

// LDLT with diagonal pivoting on the original diagonal (Eigen's left-looking ldlt_inplace),
// one CTA: f = [L (strictly lower) | D (diagonal)] in place, perm = transpositions.
// ridge_flag: when non-null, only runs if *ridge_flag != 0 and adds 1e-12 trace + 1e-300.
__global__ void ldlt_kernel(const double* __restrict__ tin, int R, double* __restrict__ f, int* __restrict__ perm,
                            const int* ridge_flag) {
    if (ridge_flag && *ridge_flag == 0) return;
    __shared__ double a[kMaxRank * kMaxRank];
    __shared__ int best_s;
    const int tid = threadIdx.x;
    for (int e = tid; e < R * R; e += blockDim.x) a[e] = tin[e];
    __syncthreads();
    if (ridge_flag) {
        __shared__ double ridge;
        if (tid == 0) {
            double tr = 0.0;
            for (int i = 0; i < R; ++i) tr += a[i + i * R];
            ridge = 1e-12 * tr + 1e-300;
        }
        __syncthreads();
        for (int i = tid; i < R; i += blockDim.x) a[i + i * R] += ridge;
        __syncthreads();
    }
    for (int k = 0; k < R; ++k) {
        if (tid == 0) {
            int best = k;
            for (int i = k + 1; i < R; ++i)
                if (fabs(a[i + i * R]) > fabs(a[best + best * R])) best = i;
            best_s = best;
            perm[k] = best;
        }
        __syncthreads();
        const int best = best_s;
        if (best != k) {  // symmetric swap of rows/columns k and best
            for (int j = tid; j < R; j += blockDim.x) {
                const double t0 = a[k + j * R];
                a[k + j * R] = a[best + j * R];
                a[best + j * R] = t0;
            }
            __syncthreads();
            for (int i = tid; i < R; i += blockDim.x) {
                const double t0 = a[i + k * R];
                a[i + k * R] = a[i + best * R];
                a[i + best * R] = t0;
            }
            __syncthreads();
        }
        if (tid == 0) {
            double dk = a[k + k * R];
            for (int j = 0; j < k; ++j) dk -= a[k + j * R] * a[k + j * R] * a[j + j * R];
            a[k + k * R] = dk;
        }
        __syncthreads();
        const double dk = a[k + k * R];
        for (int i = k + 1 + tid; i < R; i += blockDim.x) {
            double s = a[i + k * R];
            for (int j = 0; j < k; ++j) s -= a[i + j * R] * a[k + j * R] * a[j + j * R];
            a[i + k * R] = fabs(dk) > 0.0 ? s / dk : s;
        }
        __syncthreads();
    }
    for (int e = tid; e < R * R; e += blockDim.x) f[e] = a[e];
}

// X (m x R) solves X T = Q with T = P^T L D L^T P (one thread per row of Q); sets
// *bad = 1 on a non-finite result (cp.hpp:63-70 falls back to a ridge solve).
// ridge_flag: when non-null, only runs if *ridge_flag != 0.
__global__ void ldlt_solve_kernel(const double* __restrict__ f, const int* __restrict__ perm, int R,
                                  const double* __restrict__ q, int64_t m, double* __restrict__ x, int* bad,
                                  const int* ridge_flag) {
    if (ridge_flag && *ridge_flag == 0) return;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        double b[kMaxRank];
        for (int r = 0; r < R; ++r) b[r] = q[i + r * m];
        for (int k = 0; k < R; ++k) {
            const int p = perm[k];
            const double t0 = b[k];
            b[k] = b[p];
            b[p] = t0;
        }
        for (int r = 0; r < R; ++r)
            for (int j = 0; j < r; ++j) b[r] -= f[r + j * R] * b[j];
        for (int r = 0; r < R; ++r) {
            const double d = f[r + r * R];
            b[r] = fabs(d) > DBL_MIN ? b[r] / d : 0.0;
        }
        for (int r = R - 1; r >= 0; --r)
            for (int j = r + 1; j < R; ++j) b[r] -= f[j + r * R] * b[j];
        for (int k = R - 1; k >= 0; --k) {
            const int p = perm[k];
            const double t0 = b[k];
            b[k] = b[p];
            b[p] = t0;
        }
        bool ok = true;
        for (int r = 0; r < R; ++r) {
            ok = ok && isfinite(b[r]);
            x[i + r * m] = b[r];
        }
        if (!ok && bad) *bad = 1;
    }
}

// constraint updates, one thread per row of A (rows are independent in all three rules)
__global__ void row_update_kernel(double* __restrict__ a, const double* __restrict__ q, const double* __restrict__ t,
                                  int64_t m, int R, int kind, double c) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        if (kind == TK_CP_NONNEG_MU) {  // a *= max(q, 0) / max(a t, eps)   (ffcp.hpp:157-161)
            double at[kMaxRank];
            for (int r = 0; r < R; ++r) {
                double s = 0.0;
                for (int u = 0; u < R; ++u) s += a[i + u * m] * t[u + r * R];
                at[r] = s;
            }
            for (int r = 0; r < R; ++r) a[i + r * m] *= fmax(q[i + r * m], 0.0) / fmax(at[r], 1e-16);
        } else if (kind == TK_CP_NONNEG_HALS) {  // hals_sweep, project = true (cp.hpp:84-92)
            for (int r = 0; r < R; ++r) {
                const double trr = t[r + r * R];
                if (trr < 1e-15) continue;
                double s = 0.0;
                for (int u = 0; u < R; ++u) s += a[i + u * m] * t[u + r * R];
                a[i + r * m] = fmax(a[i + r * m] + (q[i + r * m] - s) / trr, 0.0);
            }
        } else if (kind == TK_CP_SPARSE) {  // soft_threshold (ffcp.hpp:20-27) of the LS solution
            for (int r = 0; r < R; ++r) {
                const double x = a[i + r * m];
                a[i + r * m] = x > c ? x - c : (x < -c ? x + c : 0.0);
            }
        }
    }
}

// res_sq = max(0, yt_sq - 2 <H, V_n> + <T, Gram_n>), fit = 1 - sqrt(res_sq)/yt_norm (ffcp.hpp:174-184)
__global__ void fit_kernel(const double* __restrict__ h, const double* __restrict__ v, int64_t nh,
                           const double* __restrict__ t, const double* __restrict__ gram, int R,
                           const double* __restrict__ yt, double* __restrict__ fit_out) {
    __shared__ double s1[256], s2[256];
    double a = 0.0, b = 0.0;
    for (int64_t e = threadIdx.x; e < nh; e += blockDim.x) a += h[e] * v[e];
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) b += t[e] * gram[e];
    s1[threadIdx.x] = a;
    s2[threadIdx.x] = b;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            s1[threadIdx.x] += s1[threadIdx.x + w];
            s2[threadIdx.x] += s2[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double res = fmax(0.0, yt[0] - 2.0 * s1[0] + s2[0]);
        *fit_out = 1.0 - sqrt(res) / sqrt(yt[0]);
    }
}

__global__ void dot_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n, double* out) {
    __shared__ double s[256];
    double a = 0.0;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) a += x[e] * y[e];
    s[threadIdx.x] = a;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = fmax(0.0, s[0]);
}

__global__ void abs_kernel(double* x, int64_t n) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
        x[e] = fabs(x[e]);
}

// absorb_scales (cp.hpp:96-109): columns of A_0..A_{N-2} to unit norm, scales into A_{N-1}
__global__ void absorb_kernel(double* const* a, const int64_t* rows, int order, int R) {
    const int r = blockIdx.x;
    __shared__ double red[256];
    for (int n = 0; n + 1 < order; ++n) {
        double s = 0.0;
        for (int64_t i = threadIdx.x; i < rows[n]; i += blockDim.x) s += a[n][i + r * rows[n]] * a[n][i + r * rows[n]];
        red[threadIdx.x] = s;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
            __syncthreads();
        }
        const double nrm = sqrt(red[0]);
        __syncthreads();
        if (nrm > 0.0) {
            for (int64_t i = threadIdx.x; i < rows[n]; i += blockDim.x) a[n][i + r * rows[n]] /= nrm;
            const int64_t ml = rows[order - 1];
            for (int64_t i = threadIdx.x; i < ml; i += blockDim.x) a[order - 1][i + r * ml] *= nrm;
        }
        __syncthreads();
    }
}

struct DevBuf {
    std::vector<void*> ptrs;
    ~DevBuf() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <typename T>
    T* get(size_t n) {
        void* p = nullptr;
        TK_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
};

}  // namespace

// Device FFCP. core/factors: device fp64 (factors[n]: rows[n] x core_shape[n]); outputs
// (out_factors[n]: rows[n] x rank, fit_trace: max_iters) are device or host per out_on_device.
void ffcp_device(cudaStream_t s, int64_t order, const int64_t* core_shape, const double* core, const double** factors,
                 const int64_t* rows, int64_t rank, int kind, double c, int max_iters, double fit_tol, Seed seed,
                 double** out_factors, double* fit_trace, int* iterations) {
    require(order >= 2, "ffcp: tensor order must be at least 2");
    require(order <= kMaxOrder, "ffcp: tensor order must be in [2, 8]");
    require(rank >= 1, "ffcp: rank must be positive");
    require(rank <= kMaxRank, "ffcp: rank must be <= 64 on the device path");
    require(c >= 0.0, "ffcp: sparsity level must be nonnegative");
    require(kind >= TK_CP_NONE && kind <= TK_CP_SPARSE, "ffcp: unknown constraint");
    const int R = static_cast<int>(rank);
    const bool nonneg = kind == TK_CP_NONNEG_MU || kind == TK_CP_NONNEG_HALS;
    DevBuf mem;
    CoreDesc cd{};
    cd.order = static_cast<int>(order);
    int64_t gsz = 1, maxrows = 1;
    for (int n = 0; n < order; ++n) {
        require(core_shape[n] >= 1 && core_shape[n] <= kMaxRank, "tucker model: factor columns must match core shape");
        cd.cs[n] = static_cast<int>(core_shape[n]);
        cd.stride[n] = gsz;
        gsz *= core_shape[n];
        maxrows = std::max<int64_t>(maxrows, rows[n]);
    }
    std::vector<double*> A(order), V(order), Gm(order);
    for (int n = 0; n < order; ++n) {
        A[n] = out_factors[n];
        V[n] = mem.get<double>(size_t(core_shape[n]) * R);
        Gm[n] = mem.get<double>(size_t(R) * R);
        cd.V[n] = V[n];
    }
    double* H = mem.get<double>(size_t(kMaxRank) * R);
    int64_t min_cs = kMaxRank;
    for (int n = 0; n < order; ++n) min_cs = std::min<int64_t>(min_cs, core_shape[n]);
    double* hw[2] = {mem.get<double>(size_t(gsz / min_cs) * R), mem.get<double>(size_t(gsz / min_cs) * R)};
    std::vector<double*> vpk(order);
    for (int n = 0; n < order; ++n) vpk[n] = mem.get<double>(size_t(core_shape[n]) * pack_stride(R));
    double* Qm = mem.get<double>(size_t(maxrows) * R);
    double* T = mem.get<double>(size_t(R) * R);
    double* F = mem.get<double>(size_t(R) * R);
    int* perm = mem.get<int>(R);
    int* bad = mem.get<int>(1);
    double* yt = mem.get<double>(1);
    double* fit_dev = mem.get<double>(1);
    double** gram_ptrs = mem.get<double*>(order);
    TK_CUDA(cudaMemcpyAsync(gram_ptrs, Gm.data(), sizeof(double*) * order, cudaMemcpyHostToDevice, s));

    // initial factors (ffcp.hpp:108-116), V = U^T A, Gram = A^T A
    for (int n = 0; n < order; ++n) {
        launch_gaussian_colmajor(A[n], rows[n], R, ffcp_init_seed(seed, n).key(), s);
        if (nonneg) abs_kernel<<<nblocks(rows[n] * R), 256, 0, s>>>(A[n], rows[n] * R);
        matmul_tn_kernel<<<nblocks(int64_t(core_shape[n]) * R * 32), 256, 0, s>>>(factors[n], rows[n], A[n], rows[n],
                                                                               V[n], cd.cs[n], rows[n], R);
        matmul_tn_kernel<<<nblocks(int64_t(R) * R * 32), 256, 0, s>>>(A[n], rows[n], A[n], rows[n], Gm[n], R, rows[n],
                                                                      R);
        launch_pack_factor<double>(V[n], cd.cs[n], cd.cs[n], R, vpk[n], s);
    }
    // ||Y_T||^2 = <G, G x_n (U_n^T U_n)> (ffcp.hpp:118-131)
    {
        std::vector<double*> cur(2);
        cur[0] = mem.get<double>(gsz);
        cur[1] = mem.get<double>(gsz);
        double* uu = mem.get<double>(size_t(kMaxRank) * kMaxRank);
        double* up = mem.get<double>(size_t(kMaxRank) * kMaxRank);
        const double* src = core;
        for (int n = 0; n < order; ++n) {
            const int cn = cd.cs[n];
            matmul_tn_kernel<<<nblocks(int64_t(cn) * cn * 32), 256, 0, s>>>(factors[n], rows[n], factors[n], rows[n], uu,
                                                                            cn, rows[n], cn);
            launch_pack_factor<double>(uu, cn, cn, cn, up, s);  // (U^T U) is symmetric: x_n applies it as is
            launch_ttm<double>(src, up, cur[n & 1], cd.stride[n], cn, gsz / (cd.stride[n] * cn), cn, s);
            src = cur[n & 1];
        }
        dot_kernel<<<1, 256, 0, s>>>(core, src, gsz, yt);
    }
    TK_LAUNCH_CHECK();
    double h_yt = 0.0;
    TK_CUDA(cudaMemcpyAsync(&h_yt, yt, sizeof(double), cudaMemcpyDeviceToHost, s));
    TK_CUDA(cudaStreamSynchronize(s));
    require(std::sqrt(h_yt) > 0.0, "ffcp: compressed tensor has zero norm");

    // one sweep over the modes, captured once as a graph
    auto sweep = [&](cudaStream_t st) {
        for (int n = 0; n < order; ++n) {
            const int cn = cd.cs[n];
            const int64_t m = rows[n];
            // H = unfold(G, n) * KR_{p != n}(V_p) (ffcp_h): one TTM with V_p0 (p0 = last mode
            // != n), then diagonal contractions of the other modes against the same column r
            {
                int p0 = static_cast<int>(order) - 1;
                if (p0 == n) --p0;
                WDesc wd{};
                wd.ndim = static_cast<int>(order);
                for (int p = 0; p < order; ++p) wd.dims[p] = cd.cs[p];
                launch_ttm<double>(core, vpk[p0], hw[0], cd.stride[p0], cd.cs[p0], gsz / (cd.stride[p0] * cd.cs[p0]), R,
                                   st);
                wd.dims[p0] = R;
                int rpos = p0, cur = 0;
                for (int qm = static_cast<int>(order) - 1; qm >= 0; --qm) {
                    if (qm == n || qm == p0) continue;
                    int64_t tot = 1;
                    for (int p = 0; p < wd.ndim; ++p)
                        if (p != qm) tot *= wd.dims[p];
                    diag_contract_kernel<<<nblocks(tot), 256, 0, st>>>(hw[cur], wd, qm, rpos, V[qm], cd.cs[qm],
                                                                        hw[cur ^ 1]);
                    for (int p = qm; p + 1 < wd.ndim; ++p) wd.dims[p] = wd.dims[p + 1];
                    wd.ndim -= 1;
                    if (qm < rpos) rpos -= 1;
                    cur ^= 1;
                }
                // W is now (cs_n, R) [rpos == 1] or (R, cs_n) [rpos == 0]
                finalize_h_kernel<<<nblocks(int64_t(cn) * R), 256, 0, st>>>(hw[cur], cn, R, rpos == 0, H);
            }
            matmul_nn_kernel<<<nblocks(m * R), 256, 0, st>>>(factors[n], m, H, cn, Qm, m, cn, R);
            hadamard_kernel<<<1, 256, 0, st>>>(gram_ptrs, static_cast<int>(order), n, R, T);
            if (kind == TK_CP_NONE || kind == TK_CP_SPARSE) {
                TK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
                ldlt_kernel<<<1, 64, 0, st>>>(T, R, F, perm, nullptr);
                ldlt_solve_kernel<<<nblocks(m, 128), 128, 0, st>>>(F, perm, R, Qm, m, A[n], bad, nullptr);
                ldlt_kernel<<<1, 64, 0, st>>>(T, R, F, perm, bad);  // ridge fallback, device-side
                ldlt_solve_kernel<<<nblocks(m, 128), 128, 0, st>>>(F, perm, R, Qm, m, A[n], nullptr, bad);
                if (kind == TK_CP_SPARSE) row_update_kernel<<<nblocks(m, 128), 128, 0, st>>>(A[n], Qm, T, m, R, kind, c);
            } else {
                row_update_kernel<<<nblocks(m, 128), 128, 0, st>>>(A[n], Qm, T, m, R, kind, c);
            }
            matmul_tn_kernel<<<nblocks(int64_t(R) * R * 32), 256, 0, st>>>(A[n], m, A[n], m, Gm[n], R, m, R);
            matmul_tn_kernel<<<nblocks(int64_t(cn) * R * 32), 256, 0, st>>>(factors[n], m, A[n], m, V[n], cn, m, R);
            launch_pack_factor<double>(V[n], cn, cn, R, vpk[n], st);
            if (n == order - 1)
                fit_kernel<<<1, 256, 0, st>>>(H, V[n], int64_t(cn) * R, T, Gm[n], R, yt, fit_dev);
        }
    };
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cap = nullptr;
    TK_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    TK_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    sweep(cap);
    TK_CUDA(cudaStreamEndCapture(cap, &graph));
    TK_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    double* h_fit = nullptr;
    TK_CUDA(cudaMallocHost(&h_fit, sizeof(double)));
    double prev = -INFINITY;
    int it = 0;
    try {
        for (; it < max_iters;) {
            TK_CUDA(cudaGraphLaunch(exec, s));
            TK_CUDA(cudaMemcpyAsync(h_fit, fit_dev, sizeof(double), cudaMemcpyDeviceToHost, s));
            TK_CUDA(cudaStreamSynchronize(s));
            const double f = *h_fit;
            fit_trace[it] = f;
            ++it;
            if (std::abs(f - prev) < fit_tol) break;
            prev = f;
        }
    } catch (...) {
        cudaFreeHost(h_fit);
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cap);
        throw;
    }
    cudaFreeHost(h_fit);
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cap);
    *iterations = it;
    double** aptrs = mem.get<double*>(order);
    int64_t* rws = mem.get<int64_t>(order);
    TK_CUDA(cudaMemcpyAsync(aptrs, A.data(), sizeof(double*) * order, cudaMemcpyHostToDevice, s));
    TK_CUDA(cudaMemcpyAsync(rws, rows, sizeof(int64_t) * order, cudaMemcpyHostToDevice, s));
    absorb_kernel<<<R, 256, 0, s>>>(aptrs, rws, static_cast<int>(order), R);
    TK_LAUNCH_CHECK();
    TK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace tkb
