/* tenkit_b200.h — C-ABI of the B200-native randomized-Tucker hot path.
 *
 * The reference (`tenkit`, arXiv 1412.1885) is a header-only C++20 library with no FFI
 * layer; its boundary is the set of free functions in namespace tenkit. Each
 * entry point below replaces one of them, with plain pointers and sizes (no torch types):
 *
 *   tk_rand_tucker_2i     <- tenkit::rand_tucker_2i      tucker.hpp:136-169 (Alg. 3)
 *   tk_rand_tucker        <- tenkit::rand_tucker         tucker.hpp:108-130 (Alg. 2)
 *   tk_ttm                <- tenkit::ttm                 tensor.hpp:151-176
 *   tk_ttm_all            <- tenkit::ttm_all             tensor.hpp:181-192
 *   tk_unfold_times       <- tenkit::unfold_times        tensor.hpp:195-209
 *   tk_orthonormal_basis  <- tenkit::orthonormal_basis   range_finder.hpp:18-29
 *                            + detail::fix_column_signs  tucker.hpp:39-45
 *   tk_gram_orthonormalize <- tenkit::gram_orthonormalize range_finder.hpp:48-84
 *   tk_gram_ortho_transform <- tenkit::gram_ortho_transform range_finder.hpp:86-105
 *   tk_context_set_orthonormalizer(TK_ORTHO_GRAM) <- the dist protocol's basis,
 *                            detail::dist_compress_mode dist.hpp:688-723
 *   tk_gaussian_matrix    <- tenkit::gaussian_matrix     random.hpp:85-100
 *   tk_gaussian_fill      <- tenkit::gaussian_tensor     random.hpp:124-138 (window at an offset)
 *   tk_gaussian_fill_block   (same, one block of a BlockGrid, dist.hpp:24-123)
 *   tk_dist_multiply      <- tenkit::dist_multiply       dist.hpp:812-846
 *   tk_seed_derived       <- tenkit::SeedSpec::derived   random.hpp:36-41
 *   tk_ffcp(_device)      <- tenkit::ffcp                ffcp.hpp:94-194
 *   tk_model_fit          <- tenkit::fit(y, reconstruct / cp_reconstruct(model))
 *                                                        tensor.hpp:282-290, tucker.hpp:63-66, cp.hpp:118-128
 *
 * Layouts are the reference's: column-major, mode 0 fastest (tensor.hpp:31). Errors: every
 * call returns TK_OK or a code; the reference's std::invalid_argument("tenkit: ...")
 * (tensor.hpp:20-22) maps to TK_ERR_INVALID with the same message in tk_last_error().
 * There is no CPU fallback: without a usable sm_100 device every compute call returns
 * TK_ERR_NO_DEVICE.
 */
#ifndef TENKIT_B200_H
#define TENKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TK_MAX_ORDER 8

enum tk_status { TK_OK = 0, TK_ERR_INVALID = 1, TK_ERR_CUDA = 2, TK_ERR_NO_DEVICE = 3, TK_ERR_INTERNAL = 4 };
enum tk_dtype { TK_F32 = 0, TK_F64 = 1 };
enum tk_constraint { TK_CP_NONE = 0, TK_CP_NONNEG_MU = 1, TK_CP_NONNEG_HALS = 2, TK_CP_SPARSE = 3 };

typedef struct tk_context tk_context;

/* Cross-rank reduction hook for block-partitioned Y (dist.hpp:617-800 semantics: partial
 * sketches and partial cores are summed over ranks). The library writes `count` doubles
 * at the front of `xbuf` (a caller-owned device buffer of `xbuf_capacity` doubles) and
 * calls allreduce_sum(user, count, stream); on return xbuf holds the sum over ranks.
 *
 * Which block of the global tensor this rank holds (BlockGrid, dist.hpp:24-123):
 *   blocked == 0: a slab of the last mode, rows [slab_offset, slab_offset + local I_{N-1})
 *                 of a tensor whose global last-mode size is global_last_dim;
 *   blocked != 0: a general block, indices [block_lo[n], block_lo[n] + local I_n) of mode n
 *                 of a tensor of global_dims[n] (the slab fields are ignored). */
typedef struct tk_comm {
    int rank;
    int world;
    int64_t slab_offset;
    int64_t global_last_dim;
    double* xbuf;
    int64_t xbuf_capacity;
    int (*allreduce_sum)(void* user, int64_t count, void* cuda_stream);
    void* user;
    int blocked;
    int64_t block_lo[TK_MAX_ORDER];
    int64_t global_dims[TK_MAX_ORDER];
} tk_comm;

/* Output of the Tucker drivers (TuckerModel, tucker.hpp:14-33). Pointers are device
 * pointers when on_device != 0, else host pointers; capacities: core prod_n rt_n doubles,
 * factor n I_n*rt_n doubles (rt_n = min(R_n + p, I_n)). Actual shapes are returned. */
typedef struct tk_tucker_out {
    int on_device;
    double* core;
    int64_t core_shape[TK_MAX_ORDER];
    double* factors[TK_MAX_ORDER];
    int64_t factor_cols[TK_MAX_ORDER];
} tk_tucker_out;

typedef struct tk_tucker_opts {
    int explicit_core_pass; /* 1: core = Y x_all U^T as its own pass (reference tucker.hpp:166);
                               0: core = X_{N-1} x_{N-1} U_{N-1}^T (same value, saves a Y pass) */
    int sync_ranks;         /* 1 (default): read each step's rank on the host (exact on rank
                               drop); 0: speculate full rank, verify once at the end, rerun
                               synchronously if any rank dropped */
    int time_kernels;       /* 1: bracket every Y-streaming launch with CUDA events on the
                               call's stream and report their summed device time in stats */
    int overlap;            /* 1: launch the next Y pass on a second stream so it overlaps the
                               current QR (it contracts a mode whose factor is already final) */
    int one_pass_per_step;  /* 1: every range step streams Y itself (the reference's structure,
                               tucker.hpp:149-160); 0: consecutive steps with distinct modes share
                               one Y pass over a mode outside the group (same values up to
                               rounding; N = 3: 3 Y passes instead of 6) */
    int precision;          /* fp32 data only. 0 (default): fp32-accurate tensor-core passes
                               (3xTF32 with chunked round-to-nearest accumulation); 1: fp64
                               arithmetic over the fp32 values (the reference's precision, about
                               3-7x slower) — for data whose discrete QR decisions (pivot / sign,
                               see tk_tucker_stats margins) are closer than fp32 can resolve */
} tk_tucker_opts;

/* Per-call timing/trace (filled when non-null) */
typedef struct tk_tucker_stats {
    int passes;            /* full Y passes */
    int kernel_launches;   /* kernels this call launched */
    double y_bytes;        /* bytes of (local) Y */
    int ranks[2 * TK_MAX_ORDER];
    int stream_launches;   /* Y-streaming (first-stage TTM) launches */
    double stream_ms;      /* their summed CUDA-event time (time_kernels = 1) */
    /* Per range step (pass * N + n; Alg. 2: n) diagnostics of the two discrete choices:
     * pivot margin = min over ColPiv steps of (top - second) / top of the remaining column
     * norms (range_finder.hpp:18-29); sign margin = min over columns of (max |u_i| of the
     * chosen sign - max |u_i| of the other sign) / max |u_i| (tucker.hpp:39-45); qr_path 0 =
     * pivoted CholeskyQR2, 1 = Householder (ill-conditioned Z or a near-tie pivot). */
    double pivot_margin[2 * TK_MAX_ORDER];
    double sign_margin[2 * TK_MAX_ORDER];
    int qr_path[2 * TK_MAX_ORDER];
} tk_tucker_stats;

const char* tk_last_error(void);
int tk_version(void);
/* 1 when a CUDA device of compute capability 10.x is usable */
int tk_device_ok(void);

/* device: CUDA ordinal, or -1 for the calling thread's current device */
int tk_context_create(int device, tk_context** out);
int tk_context_destroy(tk_context* ctx);
/* Run on an external CUDA stream (cudaStream_t), taken literally: NULL is the legacy default
 * stream (torch's default stream). A new context runs on its own non-blocking stream. */
int tk_context_set_stream(tk_context* ctx, void* cuda_stream);
/* Install (or clear, with NULL) the cross-rank reduction hook */
int tk_context_set_comm(tk_context* ctx, const tk_comm* comm);
int tk_context_synchronize(tk_context* ctx);
/* Native NCCL communicator for the cross-rank sums (one process per GPU, NVLink/NVSwitch):
 * rank 0 gets a unique id with tk_nccl_unique_id, the ranks exchange it out of band (e.g. a
 * torch.distributed broadcast), every rank calls tk_context_set_nccl(ctx, id, rank, world).
 * With it installed, tk_context_set_comm's block description (rank/world/blocks) is still
 * required but allreduce_sum / xbuf may be NULL: the partial sketches and cores are summed in
 * place with ncclAllReduce (fp64, sum) on the call's stream, so repeated calls keep their CUDA
 * graph (the collectives are captured). world = 0 tears the communicator down. NCCL is
 * resolved at run time (libnccl.so.2 already loaded by the process, else the system one). */
#define TK_NCCL_UNIQUE_ID_BYTES 128
int tk_nccl_unique_id(unsigned char* out /* TK_NCCL_UNIQUE_ID_BYTES */);
int tk_context_set_nccl(tk_context* ctx, const unsigned char* id, int rank, int world);
/* NCCL version code of the resolved library (e.g. 22809), 0 if unavailable */
int tk_nccl_version(void);
/* Contraction kernels for the Y-streaming TTM passes: 0 auto (tcgen05 3xTF32 UMMA for fp32
 * data when the shape tiles the GPU, FFMA otherwise), 1 FFMA only, 2 tcgen05 whenever the
 * shape is supported (also for the kernel-level tk_ttm), 3 as 2 with the kernel-level tk_ttm
 * on the Y-streaming kernel (ttm_stream.cu) when an M-major shape qualifies */
int tk_context_set_ttm_path(tk_context* ctx, int path);
/* Basis of every range step (tk_rand_tucker_2i / tk_rand_tucker, any comm):
 * TK_ORTHO_COLPIV (default) = orthonormal_basis + fix_column_signs (tucker.hpp:39-45,
 * range_finder.hpp:18-29, single-node semantics); TK_ORTHO_GRAM = the reference's
 * distributed protocol (dist_rand_tucker(_2i), dist.hpp:688-723): Gram-eig transform,
 * U = Z T, columns in descending eigenvalue order, no sign rule. */
#define TK_ORTHO_COLPIV 0
#define TK_ORTHO_GRAM 1
int tk_context_set_orthonormalizer(tk_context* ctx, int kind);

/* Alg. 3. y: dtype TK_F32/TK_F64, dims[order], device pointer if y_on_device else host.
 * Host input is copied in by the call: in last-mode slabs on a copy stream, each slab
 * multiplied by the first Y pass as it lands when that pass runs on the streaming kernel (fp32),
 * else in one copy on the context stream. ranks[order], oversample >= 0,
 * seed = SeedSpec{root, stream}.
 *
 * Device-path limit (the reference accepts any shape; this returns TK_ERR_INVALID):
 *   r~_n = min(R_n + p, I_n) <= 64          "rank + oversample must be <= 64 on this device path"
 * Mode lengths are not limited by the QR: tk_qr_max_rows(r~) is what ONE thread-block cluster
 * holds in shared memory (the sketch Z_n, I_n x r~_n fp64: about 6.6k rows at r~ = 60, 13k at
 * r~ = 30; every BASELINE config is inside); a taller sketch is first reduced by a blocked TSQR
 * (unpivoted Householder QR of balanced row blocks, their R factors stacked) and the cluster
 * QR pivots on the stack - same pivots, rank cut and sign rule (range_finder.hpp:18-29,
 * tucker.hpp:39-45). */
int64_t tk_qr_max_rows(int64_t cols);
int tk_rand_tucker_2i(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* y,
                      int y_on_device, const int64_t* ranks, int64_t oversample, uint64_t seed_root,
                      uint64_t seed_stream, const tk_tucker_opts* opts, tk_tucker_out* out,
                      tk_tucker_stats* stats);

/* Alg. 2 */
int tk_rand_tucker(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* y, int y_on_device,
                   const int64_t* ranks, int64_t oversample, uint64_t seed_root, uint64_t seed_stream,
                   tk_tucker_out* out, tk_tucker_stats* stats);

/* Kernel-level entry points, device pointers, dtype of t/m/out = dtype. */
/* ttm: out = T x_mode M  (M: mrows x dims[mode], column-major) */
int tk_ttm(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* t, int64_t mrows,
           const void* m, int64_t mode, void* out);
/* ttm_all(t, ms, skip, transpose=1): ms[n] is dims[n] x cols[n] double, applied transposed */
int tk_ttm_all(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* t, const double** ms,
               const int64_t* cols, int64_t skip, void* out);
/* unfold_times: z (dims[mode] x bcols double) = unfold(t, mode) * b (b: W x bcols double) */
int tk_unfold_times(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* t, int64_t mode,
                    const double* b, int64_t bcols, double* z);
/* orthonormal_basis + fix_column_signs: q (rows x cols capacity, double) and the rank */
int tk_orthonormal_basis(tk_context* ctx, int64_t rows, int64_t cols, const double* z, double* q, int64_t* rank,
                         double* rdiag);
/* The same with the step's QR diagnostics: margins (host, 3 doubles, may be null) = pivot margin,
 * sign margin, QR path (0 pivoted CholeskyQR2, 1 Householder: ill-conditioned Z or a pivot
 * whose two best candidates are within the near-tie gap), as in tk_tucker_stats. */
int tk_orthonormal_basis_ex(tk_context* ctx, int64_t rows, int64_t cols, const double* z, double* q, int64_t* rank,
                            double* rdiag, double* margins);
/* gram_orthonormalize of the stacked blocks (one device matrix z, rows x cols, cols <= 64):
 * u (rows x cols capacity, columns >= kept zero), spectrum (cols, descending, zero after
 * kept) and kept. TK_ERR_INVALID "all blocks are zero" for a zero Z. */
int tk_gram_orthonormalize(tk_context* ctx, int64_t rows, int64_t cols, const double* z, double* u, double* spectrum,
                           int64_t* kept);
/* gram_ortho_transform of a device n x n Gram matrix: transform (n x n capacity), spectrum, kept */
int tk_gram_ortho_transform(tk_context* ctx, int64_t n, const double* gram, double* transform, double* spectrum,
                            int64_t* kept);
/* gaussian_matrix(rows, cols, SeedSpec{root, stream}) into a device double buffer */
int tk_gaussian_matrix(tk_context* ctx, int64_t rows, int64_t cols, uint64_t seed_root, uint64_t seed_stream,
                       double* out);
/* Streaming fit of a model to y without materialising the reconstruction: sums[0] =
 * ||y - yhat||_F^2, sums[1] = ||y||_F^2 (host doubles), so fit(y, yhat) (tensor.hpp:282-290)
 * = 1 - sqrt(sums[0] / sums[1]). yhat = reconstruct(TuckerModel) (tucker.hpp:63-66) when core
 * is non-null (core_shape[order], factors[n]: dims[n] x core_shape[n]), else
 * cp_reconstruct(CpModel) (cp.hpp:118-128) with factors[n]: dims[n] x rank. y (dtype), core
 * and factors are device pointers; fp64 accumulation, one pass over y. */
int tk_model_fit(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* y,
                 const int64_t* core_shape, const double* core, const double** factors, int64_t rank, double* sums);

/* out[t] = normal_at(SeedSpec{root, stream}, offset + t) for t < n (device doubles): a window of
 * gaussian_tensor's flat counter stream (random.hpp:124-138), e.g. one rank's slab of a
 * globally indexed noise tensor (bench.hpp:100-112 generated blockwise) */
int tk_gaussian_fill(tk_context* ctx, int64_t n, uint64_t offset, uint64_t seed_root, uint64_t seed_stream,
                     double* out);
/* The same for a block of a tensor of global_dims (lo[n] .. lo[n] + len[n] - 1 in mode n): out
 * (prod len doubles, column-major block) holds each entry's draw at its global flat index —
 * one rank's block of a globally indexed noise tensor (dist.hpp:24-123 BlockGrid layout). */
int tk_gaussian_fill_block(tk_context* ctx, int64_t order, const int64_t* global_dims, const int64_t* lo,
                           const int64_t* len, uint64_t seed_root, uint64_t seed_stream, double* out);
uint64_t tk_seed_derived(uint64_t seed_root, uint64_t seed_stream, uint64_t tag);

/* dist_multiply (dist.hpp:812-846): z (global I_mode x r_tilde doubles, device) = unfold(Y, mode) *
 * gaussian_matrix(prod_{k != mode} I_k, r_tilde, SeedSpec{root, stream}) of the global tensor whose
 * block y (device, dims = the block's extents) this rank holds (tk_context_set_comm; without a
 * multi-rank hook the block is the whole tensor). Every rank ends with the whole z; the
 * reference's per-segment row blocks are its row ranges. */
int tk_dist_multiply(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* y, int64_t mode,
                     int64_t r_tilde, uint64_t seed_root, uint64_t seed_stream, double* z);

/* FFCP on a Tucker model (host pointers, fp64; computed on the device). factors[n] is
 * rows[n] x core_shape[n]. out_factors[n]: rows[n] x rank; fit_trace: capacity max_iters. */
int tk_ffcp(tk_context* ctx, int64_t order, const int64_t* core_shape, const double* core, const double** factors,
            const int64_t* rows, int64_t rank, int constraint, double sparsity_c, int max_iters, double fit_tol,
            uint64_t seed_root, uint64_t seed_stream, double** out_factors, double* fit_trace, int* iterations);

/* Same with device pointers for core / factors / out_factors (fit_trace stays host memory):
 * the decomposition's device outputs feed it without a host round trip. */
int tk_ffcp_device(tk_context* ctx, int64_t order, const int64_t* core_shape, const double* core,
                   const double** factors, const int64_t* rows, int64_t rank, int constraint, double sparsity_c,
                   int max_iters, double fit_tol, uint64_t seed_root, uint64_t seed_stream, double** out_factors,
                   double* fit_trace, int* iterations);

#ifdef __cplusplus
}
#endif

#endif /* TENKIT_B200_H */
