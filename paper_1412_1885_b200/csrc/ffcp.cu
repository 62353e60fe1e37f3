// ffcp.cu — FFCP (flexible fast CP on the Tucker-compressed tensor) on the device, fp64.
//
// Reference: ffcp (ffcp.hpp:94-194), ffcp_h (:33-47), solve_normal / hals_sweep /
// absorb_scales (cp.hpp:63-109). Every operand is core-sized (R~^N) or an I_n x R matrix,
// so each sweep is a handful of small kernels; one sweep (all modes) is captured once as a
// CUDA graph and replayed, with the compressed-space fit read back after every sweep for
// the stopping rule |fit - prev| < fit_tol (identical iteration count to the reference).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
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

// ---------------------------------------------------------------------------------------
// Persistent FFCP: every sweep of every iteration in ONE cooperative launch (one CTA per
// SM), with the stopping rule evaluated on the device. Per mode n (ffcp.hpp:139-170):
//   A  H = ffcp_h(G, V, n): one warp per (i, r) over the core slice G[i, ...] staged in
//      shared memory  |  last CTA: T = *_{p!=n} Gram_p and LDLT(T), LDLT(T + ridge) for the
//      least-squares kinds (cp.hpp:63-70), one warp each
//   B  rows of A_n by warps: q = U_n[i,:] H, row update (LS solve / MU / HALS / sparse),
//      per-CTA partial sums of A_n^T A_n and U_n^T A_n in fixed row order
//   C  fixed-order reduction of the partials over CTAs -> Gram_n, V_n
// separated by grid barriers. The compressed-space fit (ffcp.hpp:172-184) is evaluated
// redundantly (bit-identically) by every CTA, so all CTAs take the same stop decision.
// ---------------------------------------------------------------------------------------
namespace cg = cooperative_groups;
constexpr int kPThreads = 256;
constexpr int kPWarps = kPThreads / 32;

struct PersistParams {
    int order, R, kind, max_iters;
    double c, fit_tol;
    int cs[kMaxOrder];
    int64_t gstride[kMaxOrder];
    int64_t rows[kMaxOrder];
    const double* core;
    const double* U[kMaxOrder];
    double* A[kMaxOrder];
    double* V[kMaxOrder];
    double* Gm[kMaxOrder];
    double* H[2];   // c_n x R, by step parity
    double* T[2];   // R x R, by step parity
    double* F;      // LDLT factors of T, and of T + ridge
    double* Fr;
    int* sig;       // pivot order (gather indices), [2][kMaxRank]
    double* part;   // gridDim.x x ps_max partial sums
    int64_t ps_max;
    int* bad;       // [2], by step parity
    const double* yt;
    double* fit_trace;
    int* iters;
    int64_t scratch;  // doubles of the shared scratch region
    int stage_v;      // phase A stages V_q (p != n) in shared memory
    int64_t stage_g;  // doubles available for staged core slices (0: read the core from L2)
    unsigned long long* prof;  // optional: per (step, mark) globaltimer stamps of CTA 0
    unsigned* bar;             // grid barrier: [0] arrivals, [1] generation
    unsigned* fready;          // LDLT factors of step s published: *fready >= s + 1
};

// Split-phase grid barrier for the phase A -> B boundary (all CTAs are co-resident:
// cooperative launch; the other boundaries use the cooperative-groups grid barrier).
// arrive() makes the CTA's prior writes visible and returns the generation to wait on; the
// LDLT CTA arrives early and factorizes while the other CTAs run ahead into phase B.
__device__ __forceinline__ unsigned bar_arrive(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    unsigned g = 0;
    if (threadIdx.x == 0) {
        g = *reinterpret_cast<volatile unsigned*>(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        }
    }
    return g;
}
__device__ __forceinline__ void bar_wait(unsigned* bar, unsigned g) {
    if (threadIdx.x == 0) {
        while (*reinterpret_cast<volatile unsigned*>(bar + 1) == g) {
        }
        __threadfence();
    }
    __syncthreads();
}
__device__ __forceinline__ void bar_sync(unsigned* bar, unsigned nblocks) { bar_wait(bar, bar_arrive(bar, nblocks)); }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PROF_SUB(b, k)                                                                            \
    do {                                                                                          \
        if (p.prof && blockIdx.x == (b) && threadIdx.x == 0 && step < 4096) {                                \
            p.prof[4096 * 4 + step * 8 + (k)] = gtimer();                                                     \
            p.prof[4096 * 12 + step * 8 + (k)] = clock64();                                                   \
        }                                                                                                     \
    } while (0)
#define PROF_MARK(k)                                                                          \
    do {                                                                                      \
        if (p.prof && blockIdx.x == 0 && threadIdx.x == 0 && step < 4096) p.prof[step * 4 + (k)] = gtimer(); \
    } while (0)

// Eigen's LDLT (ldlt_inplace, the restated cp.hpp:64 solve) pivots on the largest remaining
// ORIGINAL diagonal entry (the left-looking update never touches the trailing diagonal), so
// the pivot order is the diagonal sorted by decreasing magnitude (stable); the symmetric
// permutation is applied first (sig[k] = source row of pivot position k) and the
// unpivoted factorization runs right-looking, each entry receiving the same updates in the
// same order as the left-looking loop. One warp, lanes over rows; f = L (strict lower) + D.
__device__ __forceinline__ void pivot_order(const double* t, int R, double ridge, int* sig) {
    for (int ii = threadIdx.x & 31; ii < R; ii += 32) {
        const double di = fabs(t[ii + ii * R] + ridge);
        int rank = 0;
        for (int j = 0; j < R; ++j) {
            const double dj = fabs(t[j + j * R] + ridge);
            rank += (dj > di) || (dj == di && j < ii);
        }
        sig[rank] = ii;
    }
    __syncwarp();
}

// R <= 32: lane i keeps row i of the permuted matrix in registers; right-looking, one step
// per column k with the column of L broadcast through shared memory. Every entry receives
// the same updates in the same order, with the same expression, as the left-looking loop
// below (fma(-(L_ik L_jk), D_k, a_ij)), so both produce the same factors.
__device__ __noinline__ void warp_ldlt_reg(const double* t, int R, double ridge, double* f, int* sig, double* colk) {
    const int lane = threadIdx.x & 31;
    pivot_order(t, R, ridge, sig);
    const int si = lane < R ? sig[lane] : 0;
    double row[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) row[j] = (lane < R && j < R) ? t[si + sig[j] * R] + (lane == j ? ridge : 0.0) : 0.0;
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
        }  // row[k] (dynamic index)
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
}

__device__ __forceinline__ void warp_ldlt(const double* t, int R, double ridge, double* a, int* sig,
                                          unsigned long long* pr = nullptr) {
    const int lane = threadIdx.x & 31;
    if (R <= 32) {  // the factor loop in registers (scratch: the R x R area after the matrix)
        if (pr && lane == 0) pr[0] = pr[1] = pr[2] = clock64();
        warp_ldlt_reg(t, R, ridge, a, sig, a + R * R);
        if (pr && lane == 0) pr[3] = clock64();
        return;
    }
    if (pr && lane == 0) pr[0] = clock64();
    pivot_order(t, R, ridge, sig);
    if (pr && lane == 0) pr[1] = clock64();
    for (int e = lane; e < R * R; e += 32) {
        const int x = e % R, y = e / R;
        a[e] = t[sig[x] + sig[y] * R] + (x == y ? ridge : 0.0);
    }
    __syncwarp();
    // left-looking, lanes over the rows i >= k of column k, read-only inner loop:
    //   s_i = A(i,k) - sum_{j<k} L(i,j) M(k,j),   M(k,j) = L(k,j) D(j) (Eigen's temp = D A10^T)
    // where M(i,k) = s_i, the numerator of L(i,k) = s_i / D(k). D(k) = s_k reaches the other
    // lanes by one shuffle; rolled loops only (this runs once per mode on one CTA and is
    // instruction-fetch bound when unrolled). Per step ~170 cycles + ~15 per dot term.
    double* mm = a + R * R;  // R x R scratch (M)
    if (pr && lane == 0) pr[2] = clock64();
    auto dot = [&](int i, int k) {
        const double* mk = mm + k;  // row k of M: mk[j * R]
        double p0 = 0.0, p1 = 0.0;
        int j = 0;
#pragma unroll 1
        for (; j + 2 <= k; j += 2) {
            p0 = fma(a[i + j * R], mk[j * R], p0);
            p1 = fma(a[i + (j + 1) * R], mk[(j + 1) * R], p1);
        }
        if (j < k) p0 = fma(a[i + j * R], mk[j * R], p0);
        return a[i + k * R] - (p0 + p1);
    };
#pragma unroll 1
    for (int k = 0; k < R; ++k) {
        const int i0 = k + lane, i1 = k + lane + 32;
        const double s0 = i0 < R ? dot(i0, k) : 0.0;
        const double s1 = i1 < R ? dot(i1, k) : 0.0;
        const double dk = __shfl_sync(0xffffffffu, s0, 0);
        const bool nz = fabs(dk) > 0.0;
        const double inv = nz ? 1.0 / dk : 0.0;
        if (lane == 0) {
            a[k + k * R] = dk;
        } else if (i0 < R) {
            a[i0 + k * R] = nz ? s0 * inv : s0;
            mm[i0 + k * R] = nz ? s0 : 0.0;
        }
        if (i1 < R) {
            a[i1 + k * R] = nz ? s1 * inv : s1;
            mm[i1 + k * R] = nz ? s1 : 0.0;
        }
        __syncwarp();
    }
    if (pr && lane == 0) pr[3] = clock64();
}

// b (lane r holds b[r] in b0, b[r + 32] in b1) <- T^{-1} b with T = P^T L D L^T P
// (f, sig in shared memory); returns false when a component is not finite.
__device__ __forceinline__ bool warp_ldlt_solve(const double* f, const int* sig, int R, double* sb, double& b0, double& b1,
                                int lane) {
    sb[lane] = b0;  // gather b[k] = q[sig[k]]
    sb[lane + 32] = b1;
    __syncwarp();
    double x0 = lane < R ? sb[sig[lane]] : 0.0;
    double x1 = lane + 32 < R ? sb[sig[lane + 32]] : 0.0;
    __syncwarp();
    for (int j = 0; j < R; ++j) {  // L y = b (unit lower), column-oriented
        const double bj = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31);
        if (lane > j && lane < R) x0 -= f[lane + j * R] * bj;
        if (lane + 32 > j && lane + 32 < R) x1 -= f[lane + 32 + j * R] * bj;
    }
    if (lane < R) {
        const double d = f[lane + lane * R];
        x0 = fabs(d) > DBL_MIN ? x0 / d : 0.0;
    }
    if (lane + 32 < R) {
        const double d = f[lane + 32 + (lane + 32) * R];
        x1 = fabs(d) > DBL_MIN ? x1 / d : 0.0;
    }
    for (int j = R - 1; j >= 0; --j) {  // L^T x = y
        const double bj = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31);
        if (lane < j) x0 -= f[j + lane * R] * bj;
        if (lane + 32 < j) x1 -= f[j + (lane + 32) * R] * bj;
    }
    if (lane < R) sb[sig[lane]] = x0;  // scatter x[sig[k]] = y[k]
    if (lane + 32 < R) sb[sig[lane + 32]] = x1;
    __syncwarp();
    b0 = lane < R ? sb[lane] : 0.0;
    b1 = lane + 32 < R ? sb[lane + 32] : 0.0;
    __syncwarp();
    const bool ok = isfinite(b0) && isfinite(b1);
    return __all_sync(0xffffffffu, ok);
}

__device__ double block_sum(double v, double* red) {
    red[threadIdx.x] = v;
    __syncthreads();
    for (int w = kPThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// dst[e] = src(e), e < n, by the whole CTA: each thread issues a batch of independent
// (L2) loads before its shared-memory stores, so a staging pass costs ~one round trip.
template <class Src>
__device__ __forceinline__ void stage_copy(double* dst, int n, Src src) {
    constexpr int kB = 8;
    for (int base = threadIdx.x; base < n; base += kB * kPThreads) {
        double v[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            const int e = base + b * kPThreads;
            v[b] = e < n ? src(e) : 0.0;
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            const int e = base + b * kPThreads;
            if (e < n) dst[e] = v[b];
        }
    }
}

__global__ void __launch_bounds__(kPThreads, 1) ffcp_persistent_kernel(PersistParams p) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    const int R = p.R, RR = R * R;
    int maxc = 1;
    for (int q = 0; q < p.order; ++q) maxc = max(maxc, p.cs[q]);
    double* sH = sm;                   // maxc * R, [k * R + r]
    double* sT = sH + maxc * R;        // R * R
    double* sF = sT + RR;              // R * R (+ R * R scratch)
    double* sFr = sF + 2 * RR;         // R * R (+ R * R scratch)
    double* red = sFr + 2 * RR;        // kPThreads
    int* ssig = reinterpret_cast<int*>(red + kPThreads);  // 2 x kMaxRank
    double* scr = reinterpret_cast<double*>(ssig + 2 * kMaxRank);  // p.scratch doubles
    // phase B view of the scratch
    double* acc = scr;                           // R*R + maxc*R
    double* sa = acc + RR + maxc * R;            // kPWarps x kMaxRank (a rows)
    double* su = sa + kPWarps * kMaxRank;        // kPWarps x kMaxRank (U rows)
    double* sb = su + kPWarps * kMaxRank;        // kPWarps x kMaxRank (solve scratch)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const bool ls = p.kind == TK_CP_NONE || p.kind == TK_CP_SPARSE;
    double prev = -INFINITY;
    int it = 0, step = 0;
    bool stop = false;
    while (it < p.max_iters && !stop) {
        for (int n = 0; n < p.order; ++n, ++step) {
            const int cn = p.cs[n];
            const int64_t m = p.rows[n];
            const int par = step & 1;
            double* H = p.H[par];
            double* T = p.T[par];
            PROF_MARK(0);
            // ---------------- phase A
            if (blockIdx.x == 0 && tid == 0) p.bad[par ^ 1] = 0;
            if (blockIdx.x == G - 1) {
                PROF_SUB(G - 1, 0);
                for (int e = tid; e < RR; e += kPThreads) {
                    double g[kMaxOrder];
                    for (int q = 0; q < p.order; ++q) g[q] = q != n ? __ldcg(p.Gm[q] + e) : 1.0;
                    double v = 1.0;
                    for (int q = 0; q < p.order; ++q)
                        if (q != n) v *= g[q];
                    sT[e] = v;
                    T[e] = v;
                }
                const unsigned ga = bar_arrive(p.bar, G);  // phase A arrival; factorize meanwhile
                PROF_SUB(G - 1, 1);
                if (ls && warp < 2) {
                    double ridge = 0.0;
                    if (warp == 1) {
                        double tr = 0.0;
                        for (int i = 0; i < R; ++i) tr += sT[i + i * R];
                        ridge = 1e-12 * tr + 1e-300;
                    }
                    double* f = warp ? sFr : sF;
                    int* sg = ssig + warp * kMaxRank;
                    warp_ldlt(sT, R, ridge, f, sg,
                              (p.prof && warp == 0 && step < 4096) ? p.prof + 4096 * 24 + step * 16 : nullptr);
                    double* gf = warp ? p.Fr : p.F;
                    for (int e = lane; e < RR; e += 32) gf[e] = f[e];
                    for (int e = lane; e < R; e += 32) p.sig[warp * kMaxRank + e] = sg[e];
                }
                __syncthreads();
                if (tid == 0) {
                    __threadfence();
                    atomicMax(p.fready, unsigned(step + 1));
                }
                PROF_SUB(G - 1, 2);
                bar_wait(p.bar, ga);
            } else if (int64_t(blockIdx.x) * kPWarps < int64_t(cn) * R) {
                // H[i, r] = sum over the other modes of G[i, ...] * prod_{q != n} V_q[i_q, r],
                // contracting the last other mode innermost (the reference's ffcp_h contracts
                // trailing modes first, ffcp.hpp:37-41). One warp per (i, r), lanes over the
                // flattened leading other modes.
                int om[kMaxOrder], no = 0;
                for (int q = 0; q < p.order; ++q)
                    if (q != n) om[no++] = q;
                const int last = om[no - 1], cl = p.cs[last];
                int S = 1;
                for (int q = 0; q < no; ++q) S *= p.cs[om[q]];
                const int Sp = S / cl;
                const int Pn = static_cast<int>(p.gstride[n]);  // extent product before mode n
                auto slice_off = [&](int el) { return (el % Pn) + (el / Pn) * Pn * cn; };
                const double* vq[kMaxOrder];
                double* stg = scr;
                if (p.stage_v) {
                    for (int q = 0; q < no; ++q) {
                        const int sz = p.cs[om[q]] * R;
                        const double* src = p.V[om[q]];
                        stage_copy(stg, sz, [&](int e) { return __ldcg(src + e); });
                        vq[q] = stg;
                        stg += sz;
                    }
                } else {
                    for (int q = 0; q < no; ++q) vq[q] = p.V[om[q]];
                }
                const int64_t nw = int64_t(G - 1) * kPWarps;
                PROF_SUB(0, 3);
                for (int64_t base = int64_t(blockIdx.x) * kPWarps; base < int64_t(cn) * R; base += nw) {
                    // this chunk's outputs o = base + warp, (i, r) = (o / R, o % R): stage the
                    // core slices G[i, ...] of its rows (one L2 round trip for the CTA)
                    const int64_t olast = (base + kPWarps < int64_t(cn) * R ? base + kPWarps : int64_t(cn) * R) - 1;
                    const int i0 = static_cast<int>(base / R), i1 = static_cast<int>(olast / R);
                    const bool sg_ok = p.stage_g >= int64_t(i1 - i0 + 1) * S;
                    __syncthreads();  // previous chunk done with the staged slices
                    if (sg_ok)
                        stage_copy(stg, (i1 - i0 + 1) * S, [&](int e) {
                            const int ii = i0 + e / S;
                            return __ldcg(p.core + ii * Pn + slice_off(e % S));
                        });
                    __syncthreads();
                    PROF_SUB(0, 4);
                    const int64_t o = base + warp;
                    if (o <= olast) {
                        const int i = static_cast<int>(o / R), r = static_cast<int>(o % R);
                        const double* vl = vq[no - 1] + int64_t(r) * cl;
                        double accv = 0.0;
                        if (sg_ok) {
                            const double* gs = stg + (i - i0) * S;
                            const int sp = Sp;
                            if (no == 1) {
                                for (int k = lane; k < cl; k += 32) accv = fma(gs[k], vl[k], accv);
                            } else {
                                for (int e = lane; e < sp; e += 32) {
                                    double t = 0.0;
#pragma unroll 8
                                    for (int k = 0; k < cl; ++k) t = fma(gs[e + k * sp], vl[k], t);
                                    int rem = e;
                                    double prod = 1.0;
                                    for (int q = 0; q + 1 < no; ++q) {
                                        const int c = p.cs[om[q]];
                                        prod *= vq[q][rem % c + r * c];
                                        rem /= c;
                                    }
                                    accv = fma(prod, t, accv);
                                }
                            }
                        } else {
                            const double* gi = p.core + i * Pn;
                            if (no == 1) {
                                for (int k = lane; k < cl; k += 32) accv = fma(__ldcg(gi + slice_off(k)), __ldcg(vl + k), accv);
                            } else {
                                for (int e = lane; e < Sp; e += 32) {
                                    double t = 0.0;
#pragma unroll 8
                                    for (int k = 0; k < cl; ++k) t = fma(__ldcg(gi + slice_off(e + k * Sp)), __ldcg(vl + k), t);
                                    int rem = e;
                                    double prod = 1.0;
                                    for (int q = 0; q + 1 < no; ++q) {
                                        const int c = p.cs[om[q]];
                                        prod *= vq[q][rem % c + r * c];
                                        rem /= c;
                                    }
                                    accv = fma(prod, t, accv);
                                }
                            }
                        }
#pragma unroll
                        for (int off = 16; off > 0; off >>= 1) accv += __shfl_xor_sync(0xffffffffu, accv, off);
                        if (lane == 0) H[i + int64_t(r) * cn] = accv;
                    }
                    PROF_SUB(0, 5);
                }
            }
            if (blockIdx.x != G - 1) bar_sync(p.bar, G);
            PROF_MARK(1);
            // ---------------- phase B (and the ridge rerun)
            const int ps = RR + cn * R;
            for (int attempt = 0; attempt < 2; ++attempt) {
                const bool ridge = attempt == 1;
                if (ridge && !(ls && __ldcg(p.bad + par))) break;
                stage_copy(sH, cn * R, [&](int d) { return __ldcg(H + (d / R) + (d % R) * cn); });
                stage_copy(sT, RR, [&](int e) { return __ldcg(T + e); });
                bool fstaged = !ls;
                auto stage_f = [&]() {  // LDLT factors of this step (published by the last CTA)
                    if (tid == 0) {
                        while (*reinterpret_cast<volatile unsigned*>(p.fready) < unsigned(step + 1)) {
                        }
                        __threadfence();
                    }
                    __syncthreads();
                    const double* fsrc = ridge ? p.Fr : p.F;
                    stage_copy(sF, RR, [&](int e) { return __ldcg(fsrc + e); });
                    for (int e = tid; e < R; e += kPThreads) ssig[e] = __ldcg(p.sig + (ridge ? kMaxRank : 0) + e);
                    __syncthreads();
                    fstaged = true;
                };
                if (ridge && ls) stage_f();
                for (int e = tid; e < ps; e += kPThreads) acc[e] = 0.0;
                __syncthreads();
                if (!ridge) PROF_SUB(0, 6);
                const double* U = p.U[n];
                double* A = p.A[n];
                double* wa = sa + warp * kMaxRank;
                double* wu = su + warp * kMaxRank;
                double* wb = sb + warp * kMaxRank;
                // rows over CTAs 0 .. G-2 (the last CTA factorizes T meanwhile)
                const int64_t chunk = int64_t(G - 1) * kPWarps;
                const int64_t first = blockIdx.x == G - 1 ? m : int64_t(blockIdx.x) * kPWarps;
                for (int64_t base = first; base < m; base += chunk) {
                    const int64_t i = base + warp;
                    double q0 = 0.0, q1 = 0.0, a0 = 0.0, a1 = 0.0;
                    if (i < m) {
                        for (int k = lane; k < cn; k += 32) wu[k] = U[i + k * m];
                        if (!ls) {
                            a0 = lane < R ? A[i + int64_t(lane) * m] : 0.0;
                            a1 = lane + 32 < R ? A[i + int64_t(lane + 32) * m] : 0.0;
                        }
                        __syncwarp();
                        if (lane < R) {
#pragma unroll 8
                            for (int k = 0; k < cn; ++k) q0 = fma(wu[k], sH[k * R + lane], q0);
                        }
                        if (lane + 32 < R) {
#pragma unroll 8
                            for (int k = 0; k < cn; ++k) q1 = fma(wu[k], sH[k * R + lane + 32], q1);
                        }
                    }
                    if (!fstaged) stage_f();  // CTA-uniform: first chunk only
                    if (i < m) {
                        if (ls) {
                            a0 = q0;
                            a1 = q1;
                            const bool ok = warp_ldlt_solve(sF, ssig, R, wb, a0, a1, lane);
                            if (!ok && !ridge && lane == 0) p.bad[par] = 1;
                            if (p.kind == TK_CP_SPARSE) {
                                const double cc = p.c;
                                a0 = a0 > cc ? a0 - cc : (a0 < -cc ? a0 + cc : 0.0);
                                a1 = a1 > cc ? a1 - cc : (a1 < -cc ? a1 + cc : 0.0);
                            }
                        } else if (p.kind == TK_CP_NONNEG_MU) {  // ffcp.hpp:157-161
                            wa[lane] = a0;
                            wa[lane + 32] = a1;
                            __syncwarp();
                            double t0 = 0.0, t1 = 0.0;
                            if (lane < R)
                                for (int u = 0; u < R; ++u) t0 += wa[u] * sT[u + lane * R];
                            if (lane + 32 < R)
                                for (int u = 0; u < R; ++u) t1 += wa[u] * sT[u + (lane + 32) * R];
                            a0 *= fmax(q0, 0.0) / fmax(t0, 1e-16);
                            a1 *= fmax(q1, 0.0) / fmax(t1, 1e-16);
                            __syncwarp();
                        } else {  // HALS, projected (cp.hpp:84-92), columns in order
                            wa[lane] = a0;
                            wa[lane + 32] = a1;
                            __syncwarp();
                            for (int r = 0; r < R; ++r) {
                                const double trr = sT[r + r * R];
                                if (trr < 1e-15) continue;
                                double sacc = 0.0;
                                for (int u = 0; u < R; ++u) sacc += wa[u] * sT[u + r * R];
                                const double qr = __shfl_sync(0xffffffffu, r < 32 ? q0 : q1, r & 31);
                                const double nv = fmax(wa[r] + (qr - sacc) / trr, 0.0);
                                __syncwarp();
                                if (lane == 0) wa[r] = nv;
                                __syncwarp();
                            }
                            a0 = wa[lane];
                            a1 = wa[lane + 32];
                            __syncwarp();
                        }
                        if (lane < R) A[i + int64_t(lane) * m] = a0;
                        if (lane + 32 < R) A[i + int64_t(lane + 32) * m] = a1;
                        wa[lane] = a0;
                        wa[lane + 32] = a1;
                    }
                    __syncthreads();
                    const int nrow = static_cast<int>(m - base < kPWarps ? m - base : int64_t(kPWarps));
                    for (int e = tid; e < ps; e += kPThreads) {
                        double v = acc[e];
                        if (e < RR) {
                            const int x = e % R, y = e / R;
#pragma unroll
                            for (int w = 0; w < kPWarps; ++w)
                                if (w < nrow) v = fma(sa[w * kMaxRank + x], sa[w * kMaxRank + y], v);
                        } else {
                            const int e2 = e - RR, k = e2 % cn, r = e2 / cn;
#pragma unroll
                            for (int w = 0; w < kPWarps; ++w)
                                if (w < nrow) v = fma(su[w * kMaxRank + k], sa[w * kMaxRank + r], v);
                        }
                        acc[e] = v;
                    }
                    __syncthreads();
                }
                if (!ridge) PROF_SUB(0, 7);
                for (int e = tid; e < ps; e += kPThreads) p.part[int64_t(blockIdx.x) * p.ps_max + e] = acc[e];
                grid.sync();
                PROF_MARK(2);
            }
            // ---------------- phase C: Gram_n, V_n in fixed order over CTAs
            for (int64_t e = int64_t(blockIdx.x) * kPWarps + warp; e < ps; e += int64_t(G) * kPWarps) {
                double v = 0.0;
                double pv[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const int b = lane + 32 * t;
                    pv[t] = b < G ? __ldcg(p.part + int64_t(b) * p.ps_max + e) : 0.0;
                }
                for (int t = 0; t < 8; ++t) v += pv[t];
                for (int b = lane + 256; b < G; b += 32) v += __ldcg(p.part + int64_t(b) * p.ps_max + e);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0) {
                    if (e < RR) p.Gm[n][e] = v;
                    else p.V[n][e - RR] = v;
                }
            }
            grid.sync();
            PROF_MARK(3);
        }
        // fit (ffcp.hpp:172-184), identical in every CTA
        {
            const int nl = p.order - 1, cn = p.cs[nl];
            const int par = (step - 1) & 1;
            double a = 0.0, b = 0.0;
            for (int e = tid; e < cn * R; e += kPThreads) a += __ldcg(p.H[par] + e) * __ldcg(p.V[nl] + e);
            for (int e = tid; e < RR; e += kPThreads) b += __ldcg(p.T[par] + e) * __ldcg(p.Gm[nl] + e);
            const double inner = block_sum(a, red);
            const double msq = block_sum(b, red);
            const double res = fmax(0.0, p.yt[0] - 2.0 * inner + msq);
            const double f = 1.0 - sqrt(res) / sqrt(p.yt[0]);
            if (blockIdx.x == 0 && tid == 0) p.fit_trace[it] = f;
            ++it;
            stop = fabs(f - prev) < p.fit_tol;
            prev = f;
        }
    }
    if (blockIdx.x == 0 && tid == 0) *p.iters = it;
}

// Shared memory of the persistent kernel: fixed part + `scratch` doubles.
size_t persist_smem(int R, int maxc, int64_t scratch) {
    return sizeof(double) * (size_t(maxc) * R + 5 * size_t(R) * R + kPThreads + size_t(scratch)) +
           sizeof(int) * 2 * kMaxRank;
}

struct DevBuf {  // per-call scratch carved from the context's named pool (no per-call cudaMalloc)
    BufPool& pool;
    int next = 0;
    explicit DevBuf(BufPool& p) : pool(p) {}
    template <typename T>
    T* get(size_t n) {
        return static_cast<T*>(pool.get("ffcp#" + std::to_string(next++), std::max<size_t>(n, 1) * sizeof(T)));
    }
};

}  // namespace

// Device FFCP. core/factors: device fp64 (factors[n]: rows[n] x core_shape[n]); outputs
// (out_factors[n]: rows[n] x rank, fit_trace: max_iters) are device or host per out_on_device.
void ffcp_device(BufPool& pool, cudaStream_t s, int64_t order, const int64_t* core_shape, const double* core, const double** factors,
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
    DevBuf mem(pool);
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

    const char* env = std::getenv("TENKIT_FFCP_GRAPH");
    if (!(env && env[0] == '1')) {  // persistent cooperative kernel (default)
        int dev = 0, nsm = 0, coop = 0, per_sm = 0;
        TK_CUDA(cudaGetDevice(&dev));
        TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        TK_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        require(coop != 0, "ffcp: device lacks cooperative launch");
        int maxc = 1;
        for (int n = 0; n < order; ++n) maxc = std::max(maxc, cd.cs[n]);
        int smem_optin = 0;
        TK_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        // scratch: phase B needs acc + 3 row buffers per warp; phase A stages V_q (q != n)
        // and the core slices G[i, ...] of one chunk of outputs (<= kPWarps / R + 2 rows)
        int64_t gsz_all = 1, vsum = 0, smax = 1;
        for (int n = 0; n < order; ++n) {
            gsz_all *= cd.cs[n];
            vsum += int64_t(cd.cs[n]) * R;
        }
        for (int n = 0; n < order; ++n) smax = std::max<int64_t>(smax, gsz_all / cd.cs[n]);
        const int64_t need_b = int64_t(R) * R + int64_t(maxc) * R + 3 * kPWarps * kMaxRank;
        const int64_t slices = smax * (kPWarps / R + 2);
        const int64_t budget =
            (int64_t(smem_optin) - 2048) / 8 - (int64_t(maxc) * R + 5 * int64_t(R) * R + kPThreads + kMaxRank);
        require(gsz_all < (int64_t(1) << 31), "ffcp: core too large for the device path");
        const char* nostage = std::getenv("TENKIT_FFCP_NOSTAGE");
        const bool allow = !(nostage && nostage[0] == '1');
        bool stage_v = allow && vsum + slices <= budget;
        int64_t scratch = need_b;
        int64_t stage_g = 0;
        if (stage_v) {
            scratch = std::max(need_b, vsum + slices);
            stage_g = scratch - vsum;
        } else if (allow && vsum <= budget) {
            stage_v = true;
            scratch = std::max(need_b, vsum);
        }
        const size_t smem = persist_smem(R, maxc, scratch);
        // The persistent kernel runs where its shared-memory plan holds: V and the core slices
        // staged (stage_g > 0) inside the SM's opt-in limit. Otherwise (large cores with
        // R > 48, e.g. 60^3 / R = 50: the V-only plan faulted, 64^3 / R = 64 exceeded the limit;
        // tools/ffcp_probe.py) the captured sweep graph below runs — same results.
        if (stage_g > 0 && smem + 2048 <= size_t(smem_optin)) {
        TK_CUDA(cudaFuncSetAttribute(ffcp_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
        TK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ffcp_persistent_kernel, kPThreads, smem));
        require(per_sm >= 1, "ffcp: persistent kernel does not fit an SM");
        int G = nsm;  // one CTA per SM (co-resident by construction)
        if (const char* ge = std::getenv("TENKIT_FFCP_GRID")) G = std::max(2, std::min(nsm, std::atoi(ge)));
        PersistParams pp{};
        pp.order = static_cast<int>(order);
        pp.R = R;
        pp.kind = kind;
        pp.max_iters = max_iters;
        pp.c = c;
        pp.fit_tol = fit_tol;
        pp.core = core;
        for (int n = 0; n < order; ++n) {
            pp.cs[n] = cd.cs[n];
            pp.gstride[n] = cd.stride[n];
            pp.rows[n] = rows[n];
            pp.U[n] = factors[n];
            pp.A[n] = A[n];
            pp.V[n] = V[n];
            pp.Gm[n] = Gm[n];
        }
        pp.ps_max = int64_t(R) * R + int64_t(maxc) * R;
        for (int b = 0; b < 2; ++b) {
            pp.H[b] = mem.get<double>(size_t(maxc) * R);
            pp.T[b] = mem.get<double>(size_t(R) * R);
        }
        pp.F = mem.get<double>(size_t(R) * R);
        pp.Fr = mem.get<double>(size_t(R) * R);
        pp.sig = mem.get<int>(2 * kMaxRank);
        pp.part = mem.get<double>(size_t(G) * pp.ps_max);
        pp.bad = mem.get<int>(2);
        pp.yt = yt;
        pp.fit_trace = mem.get<double>(std::max(max_iters, 1));
        pp.iters = mem.get<int>(1);
        pp.bar = mem.get<unsigned>(2);
        pp.fready = mem.get<unsigned>(1);
        TK_CUDA(cudaMemsetAsync(pp.bar, 0, 2 * sizeof(unsigned), s));
        TK_CUDA(cudaMemsetAsync(pp.fready, 0, sizeof(unsigned), s));
        pp.scratch = scratch;
        pp.stage_v = stage_v ? 1 : 0;
        pp.stage_g = stage_g;
        const char* profenv = std::getenv("TENKIT_FFCP_PROF");
        const bool prof = profenv && profenv[0] == '1';
        if (prof) {
            pp.prof = mem.get<unsigned long long>(4096 * 40);
            TK_CUDA(cudaMemsetAsync(pp.prof, 0, 4096 * 40 * sizeof(unsigned long long), s));
        }
        TK_CUDA(cudaMemsetAsync(pp.bad, 0, 2 * sizeof(int), s));
        TK_CUDA(cudaMemsetAsync(pp.iters, 0, sizeof(int), s));
        void* args[] = {&pp};
        TK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(ffcp_persistent_kernel), dim3(G), dim3(kPThreads),
                                            args, smem, s));
        int it = 0;
        TK_CUDA(cudaMemcpyAsync(&it, pp.iters, sizeof(int), cudaMemcpyDeviceToHost, s));
        TK_CUDA(cudaStreamSynchronize(s));
        if (it > 0) TK_CUDA(cudaMemcpyAsync(fit_trace, pp.fit_trace, sizeof(double) * it, cudaMemcpyDeviceToHost, s));
        *iterations = it;
        if (prof) {
            std::vector<unsigned long long> h(4096 * 40);
            TK_CUDA(cudaMemcpy(h.data(), pp.prof, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
            const int steps = std::min(4095, it * static_cast<int>(order));
            double ph[4] = {0, 0, 0, 0};
            for (int st = 1; st + 1 < steps; ++st) {
                ph[0] += double(h[st * 4 + 1] - h[st * 4 + 0]);
                ph[1] += double(h[st * 4 + 2] - h[st * 4 + 1]);
                ph[2] += double(h[st * 4 + 3] - h[st * 4 + 2]);
                ph[3] += double(h[(st + 1) * 4 + 0] - h[st * 4 + 3]);
            }
            double sub[6] = {0, 0, 0, 0, 0, 0};
            for (int st = 1; st + 1 < steps; ++st) {
                const unsigned long long* q = h.data() + 4096 * 4 + st * 8;
                const unsigned long long a0 = h[st * 4 + 0];
                sub[0] += double(q[1] - q[0]);  // T
                sub[1] += double(q[2] - q[1]);  // LDLT
                sub[2] += double(q[0] - a0);    // start skew of the last CTA
                sub[3] += double(q[3] - a0);    // V staging (CTA 0)
                sub[4] += double(q[4] - q[3]);  // slice staging
                sub[5] += double(q[5] - q[4]);  // H compute
            }
            for (double& v : sub) v /= 1e3 * (steps - 2);
            double bsub[3] = {0, 0, 0};
            for (int st = 1; st + 1 < steps; ++st) {
                const unsigned long long* q = h.data() + 4096 * 4 + st * 8;
                bsub[0] += double(q[6] - h[st * 4 + 1]);  // phase B staging
                bsub[1] += double(q[7] - q[6]);           // rows + partial sums
                bsub[2] += double(h[st * 4 + 2] - q[7]);  // partial store + grid sync
            }
            std::fprintf(stderr, "  phase B: stage %.2f rows %.2f store+sync %.2f\n", bsub[0] / 1e3 / (steps - 2),
                         bsub[1] / 1e3 / (steps - 2), bsub[2] / 1e3 / (steps - 2));
            double lc[7] = {0, 0, 0, 0, 0, 0, 0};
            for (int st = 1; st + 1 < steps; ++st) {
                const unsigned long long* q = h.data() + 4096 * 24 + st * 16;
                if (!q[0]) continue;
                lc[0] += double(q[1] - q[0]);
                lc[1] += double(q[2] - q[1]);
                lc[2] += double(q[3] - q[2]);
                lc[3] += double(q[5] - q[4]);
                lc[4] += double(q[6] - q[5]);
                lc[5] += double(q[7] - q[6]);
                lc[6] += double(q[8] - q[7]);
            }
            for (double& v : lc) v /= (steps - 2);
            std::fprintf(stderr, "  ldlt cycles: pivot %.0f copy %.0f factor %.0f | mid step: w %.0f dot %.0f shfl %.0f div+st %.0f\n",
                         lc[0], lc[1], lc[2], lc[3], lc[4], lc[5], lc[6]);
            double cyc[3] = {0, 0, 0};
            for (int st = 1; st + 1 < steps; ++st) {
                const unsigned long long* q = h.data() + 4096 * 12 + st * 8;
                cyc[0] += double(q[2] - q[1]);  // LDLT (cycles)
                cyc[1] += double(q[4] - q[3]);  // slices
                cyc[2] += double(q[5] - q[4]);  // compute
            }
            std::fprintf(stderr, "  cycles: ldlt %.0f slices %.0f compute %.0f\n", cyc[0] / (steps - 2), cyc[1] / (steps - 2),
                         cyc[2] / (steps - 2));
            std::fprintf(stderr, "  ldlt-cta: skew %.2f T %.2f ldlt %.2f | cta0: vstage %.2f slices %.2f compute %.2f\n", sub[2], sub[0],
                         sub[1], sub[3], sub[4], sub[5]);
            std::fprintf(stderr, "ffcp persistent: per mode-step us: A %.2f  B %.2f  C %.2f  fit/loop %.2f  (grid %d, stage %d)\n",
                         ph[0] / 1e3 / (steps - 2), ph[1] / 1e3 / (steps - 2), ph[2] / 1e3 / (steps - 2),
                         ph[3] / 1e3 / (steps - 2), G, int(stage_g > 0));
        }
        double** aptrs = mem.get<double*>(order);
        int64_t* rws = mem.get<int64_t>(order);
        TK_CUDA(cudaMemcpyAsync(aptrs, A.data(), sizeof(double*) * order, cudaMemcpyHostToDevice, s));
        TK_CUDA(cudaMemcpyAsync(rws, rows, sizeof(int64_t) * order, cudaMemcpyHostToDevice, s));
        absorb_kernel<<<R, 256, 0, s>>>(aptrs, rws, static_cast<int>(order), R);
        TK_LAUNCH_CHECK();
        TK_CUDA(cudaStreamSynchronize(s));
        return;
        }
    }

    // one sweep over the modes, captured once as a graph (TENKIT_FFCP_GRAPH=1, or when the
    // persistent kernel's shared-memory plan does not fit)
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
