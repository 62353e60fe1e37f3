// kernels.cuh — launch interfaces of the sm_100a kernels (implemented in ttm.cu, qr.cu,
// gen.cu). All launches are asynchronous on the given stream; layouts are column-major
// (mode 0 fastest) like the reference DenseTensor (tensor.hpp:31).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "common.cuh"

namespace tkb {

// Dtype tags of the C-ABI (include/tenkit_b200.h)
enum Dtype : int { kF32 = 0, kF64 = 1 };

// TTM column counts supported by the contraction kernels; a factor with `cols`
// columns is packed with stride pack_stride(cols) (zero padded).
constexpr int kMaxRank = 64;
inline int pack_stride(int cols) { return (cols + 3) / 4 * 4; }

// One mode-m tensor-times-matrix on the (P, K, Q) slab view of a column-major tensor
// (P = prod of modes before m, K = I_m, Q = prod after; tensor.hpp:103-116):
//   out[p, r, q] = sum_k in[p, k, q] * U[k, r],  r < cols
// `up` is U packed k-major with stride pack_stride(cols) (pack_factor below), so a
// contiguous row range of U is a contiguous sub-array (used for slab-partitioned Y).
// Counts the launches it makes into *launches when non-null.
// `work` (work_elems elements, may be null) enables split-K when the row tiles alone
// cannot fill the GPU; partials are summed in fixed split order.
template <typename T>
void launch_ttm(const T* in, const T* up, T* out, int64_t P, int64_t K, int64_t Q, int cols,
                cudaStream_t s, int* launches = nullptr, T* work = nullptr, int64_t work_elems = 0);

// tcgen05 path (ttm_tc.cu, fp32 data): 3xTF32 UMMA contraction of the (P, K, Q) view with
// the factor packed by launch_pack_umma ([U_hi | U_lo] core-matrix blocks).
// P == 1 (contraction over the fastest mode) uses the K-major variant (K % 4 == 0, cols <= 32).
// work_elems: capacity of the split-K partial buffer the caller can pass to launch_ttm_tc
// (M-major shapes with too few row tiles run split-K over it).
bool tc_ttm_supported(const float* in, float* out, int64_t P, int64_t K, int64_t Q, int cols, int64_t work_elems = 0);
int64_t umma_pack_bytes(int64_t rows, int cols);
void launch_pack_umma(const double* u, int64_t ld, int64_t rows, int cols, void* out, cudaStream_t s);
// accurate: for P == 1 always use the 128-row K-major tiles with 3 accumulator sets (fp32
// FFMA-level error) instead of the faster single-set 256-row tiles.
// tout (P == 1 only): write the output transposed, out[q + r Q] (the contracted mode moves to
// the slowest position) instead of out[r + q cols].
// Returns the number of kernels launched.
int launch_ttm_tc(const float* in, const void* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
                  cudaStream_t s, bool accurate = false, bool tout = false, float* work = nullptr,
                  int64_t work_elems = 0);
// Second-design Y-streaming pass (ttm_stream.cu, fp32): [y_hi | y_lo] from TMEM, chunked
// accumulation flushed into fp32 registers, factor packed by launch_pack_stream (NH = cols rounded
// up to 8). P == 1: contraction over mode 0 with the transposed output out[q + r Q]; else
// out[p + r P + q P cols]. Persistent, one CTA per SM with two 128-row M tiles.
bool stream_ttm_enabled();
bool stream_ttm_supported(const float* in, float* out, int64_t P, int64_t K, int64_t Q, int cols);
int64_t stream_pack_bytes(int64_t rows, int cols);
void launch_pack_stream(const double* u, int64_t ld, int64_t rows, int cols, void* out, cudaStream_t s);
// k0 (a multiple of 16) / accumulate: one K range of a pass split over K — `in` points at the
// range's first k, K is its length, rows [k0, k0 + K) of the packed factor are used and the
// result is added to `out`.
void launch_ttm_stream(const float* in, const void* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
                       cudaStream_t s, int64_t k0 = 0, bool accumulate = false);
// fp64 arithmetic over fp32 data (ttm_mixed.cu): out (fp64) = in (fp32) x_mode U, U packed
// k-major with stride pack_stride(cols) (launch_pack_factor<double>); M-major shapes, P % 4 == 0.
bool mixed_ttm_supported(const float* in, int64_t P);
void launch_ttm_mixed(const float* in, const double* up, double* out, int64_t P, int64_t K, int64_t Q, int cols,
                      cudaStream_t s);
// out[i] = sum_s part[s * n + i] (fixed split order)
template <typename T>
void launch_splitk_reduce(const T* part, T* out, int64_t n, int splits, cudaStream_t s);

// Pack a column-major double factor (rows x cols, leading dim ld) into T k-major
// [rows][pack_stride(cols)] with zero padding.
template <typename T>
void launch_pack_factor(const double* u, int64_t ld, int64_t rows, int cols, T* up, cudaStream_t s);

// z[i + r ldz] (fp64) = sum_{b,a} x[b + i B + a B I] om[(b + a B) pack_stride(rn) + r]: the
// sketch unfold(X, n) Omega of a (B, I, A) view without materialising the unfolding (split-K
// partials in `work`, sketch_work_elems doubles, reduced in fixed order). Returns launches.
int64_t sketch_work_elems(int64_t I, int rn);
template <typename T>
int launch_sketch(const T* x, int64_t B, int64_t I, int64_t A, const T* om, int rn, double* z, int64_t ldz, double* work,
                  cudaStream_t s);
// The split-K partials only: work[(s * rn + r) * I + i], s < returned split count (summed in
// order s = 0, 1, ... by sketch_reduce_kernel, or by the QR kernel's load: nparts below).
template <typename T>
int launch_sketch_partials(const T* x, int64_t B, int64_t I, int64_t A, const T* om, int rn, double* work,
                           cudaStream_t s, int max_splits = 64);

// Materialise the mode-n unfolding of a (B, I, A) view: out[i + (b + a*B)*I] = x[b + i*B + a*B*I]
template <typename T>
void launch_unfold(const T* x, int64_t B, int64_t I, int64_t A, T* out, cudaStream_t s);

// Omega packed for the TTM kernels (T, k-major, stride pack_stride(cols)):
// out[c * stride + j] = normal_at(key, j * rows_total + row_off + c) for j < cols, 0 for the
// padding: rows [row_off, row_off + rows) of a rows_total x cols gaussian_matrix
// (rows_total <= 0: rows_total = rows).
template <typename T>
void launch_gaussian_packed(T* out, int64_t rows, int cols, uint64_t key, cudaStream_t s, int64_t row_off = 0,
                            int64_t rows_total = 0);

// Omega rows at scattered global positions (a block of a BlockGrid, dist.hpp:496-596): local
// row c has mixed-radix digits d_k over lext[0..nd) (first fastest) and sits at global row
// sum_k (lo[k] + d_k) * gstride[k] of a rows_total x cols gaussian_matrix.
struct RowMap {
    int nd = 0;
    int64_t lext[8] = {0}, lo[8] = {0}, gstride[8] = {0};
    int64_t rows_total = 1;
};
template <typename T>
void launch_gaussian_packed_map(T* out, int64_t rows, int cols, uint64_t key, const RowMap& map, cudaStream_t s);

// out[c] = normal_at(key, global flat index of local element c) for a block (map.lext =
// block extents, lo = block offsets, gstride = global column-major strides), c < n.
void launch_gaussian_fill_map(double* out, int64_t n, uint64_t key, const RowMap& map, cudaStream_t s);

// Counter-RNG fills (random.hpp:85-100): out[i + j*rows] = normal_at(key, j*rows + i).
void launch_gaussian_colmajor(double* out, int64_t rows, int64_t cols, uint64_t key, cudaStream_t s);
// out[t] = normal_at(key, offset + t), t < n (a window of the flat counter stream).
void launch_gaussian_fill(double* out, int64_t n, uint64_t offset, uint64_t key, cudaStream_t s);

template <typename S, typename D>
void launch_cast(const S* in, D* out, int64_t n, cudaStream_t s);
// out (standard column-major, dims[0..order)) = in stored with its modes in the order perm
// (in's storage position k holds mode perm[k]), cast S -> D.
template <typename S, typename D>
void launch_permute_cast(const S* in, D* out, int order, const int64_t* dims, const int* perm, cudaStream_t s);
// out[i + j*ldo] = in[i + j*ldi] (rows x cols)
template <typename S, typename D>
void launch_cast2d(const S* in, int64_t ldi, D* out, int64_t ldo, int64_t rows, int64_t cols, cudaStream_t s);

// Column-pivoted Householder QR + rank cut + explicit Q + sign fix of Z (rows x ncols,
// column-major, ld = rows), the device restatement of orthonormal_basis
// (range_finder.hpp:18-29) + fix_column_signs (tucker.hpp:39-45). Writes U (rows x ucap,
// ld = rows; columns >= rank zeroed), the packed T copy (pack_factor layout for `rank`
// columns, if up != nullptr), rank to *rank_dev and |R_kk| diagnostics to diag (ncols).
// Runs as one thread-block cluster holding Z in distributed shared memory.
// nparts > 0: z holds nparts split-K partials of Z, z[(s * ncols + j) * rows + i], summed in
// order s = 0 .. nparts-1 while loading (launch_sketch_partials' layout).
// margins (3 doubles, may be null): [0] pivot margin = min over pivot steps of (top - second) /
// top of the remaining column norms, [1] sign margin = min over columns of (max |u_i| of the
// chosen sign - max |u_i| of the other) / max |u_i|, [2] 0 = pivoted CholeskyQR2 fast path,
// 1 = Householder path (ill-conditioned Z or a near-tie pivot, kTieGapSq).
// Sketches taller than qr_max_rows(ncols) take the blocked path (TSQR reduction of balanced row
// blocks in front of the cluster QR, same pivots / rank cut / sign rule): it needs `work`,
// qr_work_elems(rows, ncols) doubles (0 when the cluster QR holds Z), and nparts == 0.
// Returns the number of kernel launches.
int launch_orthonormal_basis(const double* z, int64_t rows, int ncols, double* u, int ucap, void* up,
                             int up_dtype, int* rank_dev, double* diag, cudaStream_t s, int nparts = 0,
                             double* margins = nullptr, double* work = nullptr);
int64_t qr_work_elems(int64_t rows, int ncols);
// Gram-path orthonormalisation of the distributed protocol (gram.cu; range_finder.hpp:43-105,
// dist.hpp:688-723): U = Z T with T = V / sqrt(lambda) (descending, eigenvalues <= 1e-12 top
// dropped), no sign rule. Same outputs as launch_orthonormal_basis (u rows x ucap, ld = rows,
// columns >= kept zeroed; packed copy; kept -> *rank_dev); spectrum (ncols, may be null).
// work: gram_work_elems(rows, ncols) doubles. Returns the number of launches.
int64_t gram_work_elems(int64_t rows, int ncols);
int launch_gram_orthonormal(const double* z, int64_t rows, int64_t ldz, int ncols, double* u, int ucap, void* up,
                            int up_dtype, int* rank_dev, double* spectrum, double* work, cudaStream_t s);
// gram_ortho_transform (range_finder.hpp:86-105) of an n x n Gram matrix: transform (n x n,
// columns >= kept zero), spectrum (n), kept -> *rank_dev.
void launch_gram_ortho_transform(const double* gram, int n, double* transform, double* spectrum, int* rank_dev,
                                 cudaStream_t s);
// Largest Z (rows) the single-cluster QR can hold for `ncols` columns (taller: blocked path).
int64_t qr_max_rows(int ncols);

// Named device scratch owned by the caller's context (grows, never shrinks; reused across calls).
struct BufPool {
    virtual void* get(const std::string& name, size_t bytes) = 0;
    virtual ~BufPool() = default;
};

// Streaming fit (fit.cu): ||Y - Yhat||^2 and ||Y||^2 into sums[0..1] (device doubles) for a
// Tucker model (core != nullptr) or a CP model (core == nullptr, factors I_n x rank).
template <typename T>
void launch_model_fit(BufPool& pool, const T* y, int order, const int64_t* dims, const double* core,
                      const int64_t* core_shape, const double* const* factors, int64_t rank, double* sums,
                      cudaStream_t s);

// FFCP on the device (ffcp.cu); all pointers are device pointers, fit_trace is host memory.
void ffcp_device(BufPool& pool, cudaStream_t s, int64_t order, const int64_t* core_shape, const double* core, const double** factors,
                 const int64_t* rows, int64_t rank, int kind, double c, int max_iters, double fit_tol, Seed seed,
                 double** out_factors, double* fit_trace, int* iterations);

}  // namespace tkb
