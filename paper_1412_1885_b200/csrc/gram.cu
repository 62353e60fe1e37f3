// gram.cu — the distributed protocol's Gram-path orthonormalisation on the device:
// gram_orthonormalize / gram_ortho_transform (range_finder.hpp:43-105) as used by
// dist_compress_mode (dist.hpp:688-723): Gram = Z^T Z, symmetric eigendecomposition,
// T = V[:, descending] / sqrt(lambda) with eigenvalues <= 1e-12 * top dropped, U = Z T.
// No sign rule (the reference's dist path applies none).
//
// Three launches, all fp64, no host sync (the kept count goes to *rank_dev like the QR's rank):
//   gram_partial_kernel  row chunks of Z -> per-CTA partial Grams (fixed row order)
//   gram_eig_kernel      one CTA: partials summed in CTA order, cyclic parallel Jacobi with
//                        round-robin pairing (the rounds of oracle sym_eig), sort, cut, T
//   gram_apply_kernel    U = Z T and the packed compute-type copy for the next TTM
// The eigensolver stands in for Eigen's SelfAdjointEigenSolver (tridiagonal QL): the
// eigenpairs agree up to each eigenvector's sign, which the reference leaves unspecified.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace tkb {
namespace {

constexpr int kGramThreads = 256;
constexpr int kGramTileRows = 32;
constexpr int kEigThreads = 512;
constexpr int kJacobiMaxSweeps = 40;  // oracle kJacobiMaxSweeps
constexpr int kMaxPairs = (kMaxRank * kMaxRank + kGramThreads - 1) / kGramThreads;  // 16

int64_t gram_chunk(int64_t rows) {
    const int64_t c = (rows + 147) / 148;
    return std::max<int64_t>(kGramTileRows, (c + kGramTileRows - 1) / kGramTileRows * kGramTileRows);
}

// part[b * n * n + i + j * n] = sum_{rows of chunk b, ascending} z[r, i] z[r, j]
__global__ void __launch_bounds__(kGramThreads) gram_partial_kernel(const double* __restrict__ z, int64_t rows,
                                                                    int64_t ldz, int n, int64_t chunk,
                                                                    double* __restrict__ part) {
    __shared__ double tile[kGramTileRows * kMaxRank];
    const int64_t r0 = blockIdx.x * chunk;
    const int64_t r1 = min(rows, r0 + chunk);
    double acc[kMaxPairs];
#pragma unroll
    for (int e = 0; e < kMaxPairs; ++e) acc[e] = 0.0;
    for (int64_t t0 = r0; t0 < r1; t0 += kGramTileRows) {
        const int len = static_cast<int>(r1 - t0 < kGramTileRows ? r1 - t0 : kGramTileRows);
        for (int e = threadIdx.x; e < kGramTileRows * n; e += kGramThreads) {
            const int kk = e % kGramTileRows, j = e / kGramTileRows;
            tile[kk + j * kGramTileRows] = kk < len ? z[(t0 + kk) + j * ldz] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < kMaxPairs; ++e) {
            const int t = threadIdx.x + e * kGramThreads;
            if (t >= n * n) break;
            const int i = t % n, j = t / n;
            if (i > j) continue;
            const double* a = tile + i * kGramTileRows;
            const double* b = tile + j * kGramTileRows;
            double s = acc[e];
            for (int kk = 0; kk < kGramTileRows; ++kk) s = fma(a[kk], b[kk], s);
            acc[e] = s;
        }
        __syncthreads();
    }
    double* out = part + static_cast<int64_t>(blockIdx.x) * n * n;
#pragma unroll
    for (int e = 0; e < kMaxPairs; ++e) {
        const int t = threadIdx.x + e * kGramThreads;
        if (t >= n * n) break;
        const int i = t % n, j = t / n;
        if (i > j) continue;
        out[i + j * n] = acc[e];
        out[j + i * n] = acc[e];
    }
}

// Jacobi skip rule (oracle sym_eig): the off-diagonal entry is negligible against the diagonal.
__device__ __forceinline__ bool skip_rotation(double apq, double app, double aqq) {
    return apq == 0.0 || fabs(apq) <= 1e-16 * sqrt(fabs(app * aqq));
}

// One CTA. a/v in shared memory with leading dimension n + 1 (row-access bank spread).
// tout: n x n (column pos < kept = V[:, eig] / sqrt(lambda), the rest zero); spectrum[pos]
// for pos < kept, 0 after; *rank_out = kept (0 when the Gram matrix is zero).
__global__ void __launch_bounds__(kEigThreads) gram_eig_kernel(const double* __restrict__ part, int nparts, int n,
                                                               double* __restrict__ tout, double* __restrict__ spectrum,
                                                               int* __restrict__ rank_out) {
    extern __shared__ double sm[];
    const int ld = n + 1;
    double* a = sm;
    double* v = a + n * ld;
    __shared__ double cs[kMaxRank / 2], sn[kMaxRank / 2];
    __shared__ int pp[kMaxRank / 2], qq[kMaxRank / 2];
    __shared__ int rotated[1];
    __shared__ int pos[kMaxRank];
    __shared__ double top_s;
    const int tid = threadIdx.x;
    for (int e = tid; e < n * n; e += kEigThreads) {
        double s = 0.0;
        for (int b = 0; b < nparts; ++b) s += part[static_cast<int64_t>(b) * n * n + e];
        const int i = e % n, j = e / n;
        a[i + j * ld] = s;
        v[i + j * ld] = i == j ? 1.0 : 0.0;
    }
    if (tid == 0) rotated[0] = 0;
    __syncthreads();
    const int m = n + (n & 1);
    const int np = m / 2;
    for (int sweep = 0; sweep < kJacobiMaxSweeps && n > 1; ++sweep) {
        // A sweep without a rotation leaves A unchanged, so "every pair is below the skip
        // threshold now" is the oracle's "the last sweep rotated nothing" without running it.
        for (int e = tid; e < n * n; e += kEigThreads) {
            const int i = e % n, j = e / n;
            if (i < j && !skip_rotation(a[i + j * ld], a[i + i * ld], a[j + j * ld])) rotated[0] = 1;
        }
        __syncthreads();
        const bool any = rotated[0] != 0;
        __syncthreads();
        if (!any) break;
        if (tid == 0) rotated[0] = 0;
        for (int r = 0; r < m - 1; ++r) {
            if (tid < np) {  // pair tid of round r (jacobi_round_pairs): L[k], L[m-1-k]
                const int k = tid;
                const int lk = k == 0 ? 0 : ((k - 1 + r) % (m - 1)) + 1;
                const int km = m - 1 - k;
                const int lm = km == 0 ? 0 : ((km - 1 + r) % (m - 1)) + 1;
                const int p = min(lk, lm), q = max(lk, lm);
                double c = 1.0, s = 0.0;
                if (q < n) {
                    const double apq = a[p + q * ld], app = a[p + p * ld], aqq = a[q + q * ld];
                    if (!skip_rotation(apq, app, aqq)) {
                        const double theta = (aqq - app) / (2.0 * apq);
                        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                        c = 1.0 / sqrt(t * t + 1.0);
                        s = t * c;
                    }
                }
                cs[k] = c, sn[k] = s, pp[k] = p, qq[k] = q;
            }
            __syncthreads();
            // A <- P^T A P one 2x2 block (row pair k1, column pair k2) per item: the blocks are
            // disjoint, so rows and columns rotate in one phase; V <- V P likewise.
            for (int e = tid; e < np * np + np * n; e += kEigThreads) {
                if (e < np * np) {
                    const int k1 = e % np, k2 = e / np;
                    const double c1 = cs[k1], s1 = sn[k1], c2 = cs[k2], s2 = sn[k2];
                    if (s1 == 0.0 && s2 == 0.0) continue;
                    const int p1 = pp[k1], q1 = qq[k1], p2 = pp[k2], q2 = qq[k2];
                    const bool hq1 = q1 < n, hq2 = q2 < n;
                    const double x00 = a[p1 + p2 * ld];
                    const double x01 = hq2 ? a[p1 + q2 * ld] : 0.0;
                    const double x10 = hq1 ? a[q1 + p2 * ld] : 0.0;
                    const double x11 = hq1 && hq2 ? a[q1 + q2 * ld] : 0.0;
                    // rows (P^T A): r0 = c1 x0 - s1 x1, r1 = s1 x0 + c1 x1
                    const double y00 = c1 * x00 - s1 * x10, y10 = s1 * x00 + c1 * x10;
                    const double y01 = c1 * x01 - s1 * x11, y11 = s1 * x01 + c1 * x11;
                    // columns (A P)
                    a[p1 + p2 * ld] = c2 * y00 - s2 * y01;
                    if (hq2) a[p1 + q2 * ld] = s2 * y00 + c2 * y01;
                    if (hq1) a[q1 + p2 * ld] = c2 * y10 - s2 * y11;
                    if (hq1 && hq2) a[q1 + q2 * ld] = s2 * y10 + c2 * y11;
                } else {
                    const int f = e - np * np;
                    const int k = f / n, i = f - (f / n) * n;
                    if (sn[k] == 0.0) continue;
                    const int p = pp[k], q = qq[k];
                    const double vx = v[i + p * ld], vy = v[i + q * ld];
                    v[i + p * ld] = cs[k] * vx - sn[k] * vy;
                    v[i + q * ld] = sn[k] * vx + cs[k] * vy;
                }
            }
            __syncthreads();
        }
    }
    // descending position: the reverse of an ascending stable sort (ties: higher index first)
    if (tid < n) {
        const double lj = a[tid + tid * ld];
        int c = 0;
        for (int k = 0; k < n; ++k) {
            const double lk = a[k + k * ld];
            c += (lk > lj) || (lk == lj && k > tid);
        }
        pos[tid] = c;
        if (c == 0) top_s = lj;
    }
    __syncthreads();
    const double top = top_s;
    int kept = 0;
    if (top > 0.0)
        for (int k = 0; k < n; ++k) kept += a[k + k * ld] > 1e-12 * top;  // kRankDeficiencyTol
    for (int e = tid; e < n * n; e += kEigThreads) {
        const int i = e % n, j = e / n;  // j = eigen index (storage column)
        const int pj = pos[j];
        const double l = a[j + j * ld];
        tout[i + pj * n] = pj < kept ? v[i + j * ld] / sqrt(l) : 0.0;
    }
    if (tid < n) {
        const int pj = pos[tid];
        spectrum[pj] = pj < kept ? a[tid + tid * ld] : 0.0;
    }
    if (tid == 0) *rank_out = kept;
}

// U = Z T: thread per (row, 16-column group); u (rows x ucap, columns >= rank zero), the
// packed copy up[i * pack_stride(rank) + j] (QR output layout, kernels.cuh pack_factor).
constexpr int kApplyCols = 16;
__global__ void __launch_bounds__(256) gram_apply_kernel(const double* __restrict__ z, int64_t rows, int64_t ldz,
                                                         int n, const double* __restrict__ t,
                                                         double* __restrict__ u, int ucap, void* __restrict__ up,
                                                         int up_dtype, const int* __restrict__ rank_dev) {
    __shared__ double ts[kMaxRank * kMaxRank];
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) ts[e] = t[e];
    __syncthreads();
    const int rank = *rank_dev;
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int j0 = blockIdx.y * kApplyCols;
    if (i >= rows) return;
    double acc[kApplyCols];
#pragma unroll
    for (int c = 0; c < kApplyCols; ++c) acc[c] = 0.0;
    for (int k = 0; k < n; ++k) {
        const double zk = z[i + k * ldz];
#pragma unroll
        for (int c = 0; c < kApplyCols; ++c)
            if (j0 + c < n) acc[c] = fma(zk, ts[k + (j0 + c) * n], acc[c]);
    }
    const int stride = (max(rank, 1) + 3) / 4 * 4;  // pack_stride
#pragma unroll
    for (int c = 0; c < kApplyCols; ++c) {
        const int j = j0 + c;
        const double val = j < rank ? acc[c] : 0.0;
        if (j < ucap) u[i + static_cast<int64_t>(j) * rows] = val;
        if (up && j < stride) {
            if (up_dtype == kF32) static_cast<float*>(up)[i * stride + j] = static_cast<float>(val);
            else static_cast<double*>(up)[i * stride + j] = val;
        }
    }
}

size_t eig_smem(int n) { return 2 * size_t(n) * (n + 1) * sizeof(double); }

void launch_eig(const double* part, int nparts, int n, double* tout, double* spectrum, int* rank_dev, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        TK_CUDA(cudaFuncSetAttribute(gram_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(eig_smem(kMaxRank))));
        attr = true;
    }
    gram_eig_kernel<<<1, kEigThreads, eig_smem(n), s>>>(part, nparts, n, tout, spectrum, rank_dev);
    TK_CUDA(cudaGetLastError());
}

}  // namespace

int64_t gram_work_elems(int64_t rows, int ncols) {
    const int64_t parts = (rows + gram_chunk(rows) - 1) / gram_chunk(rows);
    return parts * ncols * ncols + int64_t(ncols) * ncols + ncols;
}

int launch_gram_orthonormal(const double* z, int64_t rows, int64_t ldz, int ncols, double* u, int ucap, void* up,
                            int up_dtype, int* rank_dev, double* spectrum, double* work, cudaStream_t s) {
    require(rows >= 1, "gram_orthonormalize: no blocks");
    require(ncols >= 1 && ncols <= kMaxRank, "gram_orthonormalize: column count must be in [1, 64]");
    const int64_t chunk = gram_chunk(rows);
    const int nparts = static_cast<int>((rows + chunk - 1) / chunk);
    double* part = work;
    double* t = work + int64_t(nparts) * ncols * ncols;
    double* sp = spectrum ? spectrum : t + int64_t(ncols) * ncols;
    gram_partial_kernel<<<nparts, kGramThreads, 0, s>>>(z, rows, ldz, ncols, chunk, part);
    TK_CUDA(cudaGetLastError());
    launch_eig(part, nparts, ncols, t, sp, rank_dev, s);
    const dim3 grid(static_cast<unsigned>((rows + 255) / 256), static_cast<unsigned>((ncols + kApplyCols - 1) / kApplyCols));
    if (ucap > ncols) TK_CUDA(cudaMemsetAsync(u + rows * ncols, 0, sizeof(double) * rows * (ucap - ncols), s));
    gram_apply_kernel<<<grid, 256, 0, s>>>(z, rows, ldz, ncols, t, u, std::min(ucap, ncols), up, up_dtype, rank_dev);
    TK_CUDA(cudaGetLastError());
    return 3;
}

void launch_gram_ortho_transform(const double* gram, int n, double* transform, double* spectrum, int* rank_dev,
                                 cudaStream_t s) {
    require(n >= 1 && n <= kMaxRank, "gram_ortho_transform: size must be in [1, 64]");
    launch_eig(gram, 1, n, transform, spectrum, rank_dev, s);
}

}  // namespace tkb
