// qr.cu — tall-skinny column-pivoted Householder QR on one thread-block cluster (sm_100a).
//
// Device restatement of orthonormal_basis (range_finder.hpp:18-29: Eigen
// ColPivHouseholderQR, rank = #leading |R_kk| > 1e-12 |R_00|, Q = first `rank` Householder
// columns in pivot order) followed by fix_column_signs (tucker.hpp:39-45), all in fp64.
//
// Z (rows x ncols, rows <= a few thousand, ncols <= 64) is split into contiguous row
// blocks held in the shared memory of the cluster's CTAs (distributed shared memory).
// Each Householder step needs exactly one cluster-wide reduction (column-k tail norm, the
// dot products of column k with the trailing columns, and row k itself); partial vectors
// are exchanged through DSMEM and summed in fixed CTA order, so results are deterministic.
// Pivoting is done by a logical->physical column map (no data movement); the pivot
// choice, the Householder scalars and the LAPACK-style norm downdating (direct
// recomputation below sqrt(eps)) are evaluated redundantly and identically in every warp
// of every CTA, which keeps a step at one cluster barrier plus two CTA barriers. Q is then
// formed in place over the stored reflectors (backward accumulation).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tkb {

namespace {

constexpr int kQrThreads = 512;
constexpr int kQrWarps = kQrThreads / 32;
constexpr int kSlot = 3 * kMaxRank + 8;  // exchange vector length (doubles)
constexpr size_t kQrFixedSmem = (3 * kSlot + 6 * kMaxRank + 16) * sizeof(double) + (kMaxRank + 16) * sizeof(int);
constexpr size_t kQrSmemCap = 200 * 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct Xchg {
    cg::cluster_group cl;
    unsigned cs;
    double* slot;  // [2][kSlot]
    double* tot;   // [kSlot]
    int par = 0;

    __device__ double* mine() { return slot + par * kSlot; }
    __device__ void sync_all() {
        if (cs > 1) cl.sync();
        else __syncthreads();
    }
    // Sum of every CTA's slot[par][0:len] in CTA order into tot (block-visible on return)
    __device__ void sum(int len) {
        sync_all();
        double* m = mine();
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            double s = 0.0;
            if (cs > 1)
                for (unsigned c = 0; c < cs; ++c) s += cl.map_shared_rank(m, c)[i];
            else
                s = m[i];
            tot[i] = s;
        }
        par ^= 1;
        __syncthreads();
    }
};

__global__ void __launch_bounds__(kQrThreads, 1)
    qr_colpiv_cluster_kernel(const double* __restrict__ zin, int64_t rows, int ncols, int ld,
                             double* __restrict__ uout, int ucap, void* upout, int up_dtype, int* rank_out,
                             double* diag_out) {
    cg::cluster_group cl = cg::this_cluster();
    const int crank = static_cast<int>(cl.block_rank());
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    extern __shared__ __align__(16) double qsm[];
    double* z = qsm;
    double* slot = z + size_t(ld) * ncols;
    double* tot = slot + 2 * kSlot;
    double* upd = tot + kSlot;
    double* dir = upd + kMaxRank;
    double* beta = dir + kMaxRank;
    double* taus = beta + kMaxRank;
    double* sgn = taus + kMaxRank;
    double* misc = sgn + kMaxRank;
    int* colmap = reinterpret_cast<int*>(misc + 16);
    int* flags = colmap + kMaxRank;  // [0..1] recompute-any flags by step parity

    Xchg X{cl, cl.num_blocks(), slot, tot};
    const int64_t r0 = int64_t(crank) * ld;
    const int nloc = static_cast<int>(lmax(0, lmin(ld, rows - r0)));

    for (int j = 0; j < ncols; ++j)
        for (int i = tid; i < ld; i += kQrThreads) z[i + j * ld] = i < nloc ? zin[(r0 + i) + j * rows] : 0.0;
    for (int j = tid; j < kMaxRank; j += kQrThreads) colmap[j] = j;
    if (tid < 2) flags[tid] = 0;
    __syncthreads();

    // initial column norms (m_qr.col(k).norm())
    for (int j = warp; j < ncols; j += kQrWarps) {
        double s = 0.0;
        for (int i = lane; i < nloc; i += 32) s += z[i + j * ld] * z[i + j * ld];
        s = warp_sum(s);
        if (lane == 0) X.mine()[j] = s;
    }
    X.sum(ncols);
    for (int j = tid; j < ncols; j += kQrThreads) upd[j] = dir[j] = sqrt(tot[j]);
    __syncthreads();

    const double norm_downdate_threshold = sqrt(DBL_EPSILON);
    const int size = static_cast<int>(lmin(rows, ncols));
    int pprev = -1;  // physical column of the previous step (its essential part is written late)
    double dprev = 1.0;
    bool zprev = false;
    int kprev = -1;
    for (int k = 0; k < size; ++k) {
        // ---- pivot: first maximum of the updated norms over logical columns k.. (per warp)
        int best;
        {
            double bv = -1.0;
            int bi = 0x7fffffff;
            for (int j = k + lane; j < ncols; j += 32)
                if (upd[j] > bv) {
                    bv = upd[j];
                    bi = j;
                }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            best = bi;
        }
        // registers: thread 0 swaps colmap[k] / colmap[best] during this step's update phase
        const int ck = colmap[k];
        const int pk = colmap[best];
        auto phys = [&](int j) { return j == best ? ck : colmap[j]; };
        const int lk = static_cast<int>(k - r0);
        const bool owner = lk >= 0 && lk < nloc;
        const int i0 = static_cast<int>(lmax(0, k + 1 - r0));

        // ---- local partials: [j-k] = dot(col k, col j) over rows > k ([0]: tail norm^2),
        //      [kMaxRank + j-k] = row k (owner; others 0)
        {
            double* m = X.mine();
            for (int j = k + warp; j < ncols; j += kQrWarps) {
                const int pj = j == k ? pk : phys(j);
                double s = 0.0;
                for (int i = i0 + lane; i < nloc; i += 32) s += z[i + pk * ld] * z[i + pj * ld];
                s = warp_sum(s);
                if (lane == 0) {
                    m[j - k] = s;
                    m[kMaxRank + (j - k)] = owner ? z[lk + pj * ld] : 0.0;
                }
            }
            if (pprev >= 0) {  // late essential write of the previous step's column
                const int ip = static_cast<int>(lmax(0, kprev + 1 - r0));
                for (int i = ip + tid; i < nloc; i += kQrThreads)
                    z[i + pprev * ld] = zprev ? 0.0 : z[i + pprev * ld] / dprev;
            }
        }
        X.sum(kMaxRank + (ncols - k));

        // ---- Householder scalars (makeHouseholderInPlace), redundantly in every thread
        const double tail_sq = (rows - k == 1) ? 0.0 : tot[0];
        const double c0 = tot[kMaxRank];
        double tau, bta, denom = 1.0;
        bool zero_ess = false;
        if (tail_sq <= DBL_MIN) {
            tau = 0.0;
            bta = c0;
            zero_ess = true;
        } else {
            bta = sqrt(c0 * c0 + tail_sq);
            if (c0 >= 0.0) bta = -bta;
            denom = c0 - bta;
            tau = (bta - c0) / bta;
        }
        if (tid == 0) {
            beta[k] = bta;
            taus[k] = tau;
            flags[(k + 1) & 1] = 0;
        }

        // ---- apply H_k to the trailing columns: w_j = row0_j + dot_j / denom,
        //      col_j -= (tau * v) w_j with v = col_k / denom; norm downdate per column
        for (int j = k + 1 + warp; j < ncols; j += kQrWarps) {
            const int pj = phys(j);
            const double rowk = tot[kMaxRank + (j - k)];
            const double wj = tau != 0.0 ? rowk + tot[j - k] / denom : 0.0;
            const double nrow = tau != 0.0 ? rowk - tau * wj : rowk;
            if (tau != 0.0)
                for (int i = i0 + lane; i < nloc; i += 32) z[i + pj * ld] -= (tau * (z[i + pk * ld] / denom)) * wj;
            if (owner && lane == 0) z[lk + pj * ld] = nrow;
            const double u = (j == best) ? upd[k] : upd[j];
            const double d = (j == best) ? dir[k] : dir[j];
            bool recompute = false;
            double nu = u;
            if (u != 0.0) {
                double temp = fabs(nrow) / u;
                temp = (1.0 + temp) * (1.0 - temp);
                temp = temp < 0.0 ? 0.0 : temp;
                const double ratio = u / d;
                if (temp * ratio * ratio <= norm_downdate_threshold) recompute = true;
                else nu = u * sqrt(temp);
            }
            if (recompute) {  // local partial of the fresh tail norm (rows > k), exchanged below
                __syncwarp();
                double s = 0.0;
                for (int i = i0 + lane; i < nloc; i += 32) s += z[i + pj * ld] * z[i + pj * ld];
                s = warp_sum(s);
                if (lane == 0) {
                    X.mine()[j] = s;
                    atomicOr(&flags[k & 1], 1);
                }
            }
            if (lane == 0) {
                upd[j] = recompute ? -1.0 : nu;  // -1: pending recompute
                dir[j] = d;
            }
        }
        if (owner && tid == 0) z[lk + pk * ld] = bta;
        if (tid == 0 && best != k) {
            const int t = colmap[k];
            colmap[k] = colmap[best];
            colmap[best] = t;
        }
        __syncthreads();
        if (flags[k & 1]) {
            double* m = X.mine();
            for (int j = tid; j < ncols; j += kQrThreads)
                if (j <= k || upd[j] >= 0.0) m[j] = 0.0;
            X.sum(ncols);
            for (int j = k + 1 + tid; j < ncols; j += kQrThreads)
                if (upd[j] < 0.0) upd[j] = dir[j] = sqrt(tot[j]);
            __syncthreads();
        }
        pprev = pk;
        dprev = denom;
        zprev = zero_ess;
        kprev = k;
    }
    if (pprev >= 0) {
        const int ip = static_cast<int>(lmax(0, kprev + 1 - r0));
        for (int i = ip + tid; i < nloc; i += kQrThreads) z[i + pprev * ld] = zprev ? 0.0 : z[i + pprev * ld] / dprev;
    }
    __syncthreads();

    // ---- rank cut (range_finder.hpp:24-26), redundantly
    int rank = 0;
    {
        const double top = fabs(beta[0]);
        while (rank < size && fabs(beta[rank]) > 1e-12 * top) ++rank;
    }

    // ---- explicit Q(:, 0:rank) = H_0 ... H_{rank-1} [I; 0], in place, logical column j at colmap[j]
    for (int k = rank - 1; k >= 0; --k) {
        const double tau = taus[k];
        const int pk = colmap[k];
        const int lk = static_cast<int>(k - r0);
        const bool owner = lk >= 0 && lk < nloc;
        const int i0 = static_cast<int>(lmax(0, k + 1 - r0));
        if (k + 1 < rank) {
            double* m = X.mine();
            for (int j = k + 1 + warp; j < rank; j += kQrWarps) {
                const int pj = colmap[j];
                double s = 0.0;
                for (int i = i0 + lane; i < nloc; i += 32) s += z[i + pk * ld] * z[i + pj * ld];
                s = warp_sum(s);
                if (lane == 0) m[j - k] = s;
            }
            X.sum(rank - k);
            for (int j = k + 1 + warp; j < rank; j += kQrWarps) {
                const int pj = colmap[j];
                const double t = tot[j - k];
                if (tau != 0.0)
                    for (int i = i0 + lane; i < nloc; i += 32) z[i + pj * ld] -= (tau * z[i + pk * ld]) * t;
                if (owner && lane == 0) z[lk + pj * ld] = -tau * t;
            }
            __syncthreads();
        }
        for (int i = tid; i < nloc; i += kQrThreads) {
            const int64_t gi = r0 + i;
            double v;
            if (gi < k) v = 0.0;
            else if (gi == k) v = 1.0 - tau;
            else v = -tau * z[i + pk * ld];
            z[i + pk * ld] = v;
        }
        __syncthreads();
    }

    // ---- sign fix: largest |entry| of each column positive (first maximum on ties)
    if (rank > 0) {
        double* m = X.mine();
        for (int j = warp; j < rank; j += kQrWarps) {
            const int pj = colmap[j];
            double bv = -1.0, val = 0.0;
            int bi = 0x7fffffff;
            for (int i = lane; i < nloc; i += 32) {
                const double a = fabs(z[i + pj * ld]);
                if (a > bv) {
                    bv = a;
                    bi = i;
                    val = z[i + pj * ld];
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                const double ov = __shfl_xor_sync(0xffffffffu, val, o);
                if (ob > bv || (ob == bv && oi < bi)) {
                    bv = ob;
                    bi = oi;
                    val = ov;
                }
            }
            if (lane == 0) {
                m[2 * j] = bv;
                m[2 * j + 1] = val;
            }
        }
        X.sync_all();
        for (int j = tid; j < rank; j += kQrThreads) {
            double bv = -1.0, val = 0.0;
            for (unsigned c = 0; c < X.cs; ++c) {
                const double* ps = X.cs > 1 ? cl.map_shared_rank(m, c) : m;
                if (ps[2 * j] > bv) {  // CTAs hold increasing rows: strict > keeps the first
                    bv = ps[2 * j];
                    val = ps[2 * j + 1];
                }
            }
            sgn[j] = val < 0.0 ? -1.0 : 1.0;
        }
        X.par ^= 1;
        __syncthreads();
    }

    // ---- outputs
    for (int j = 0; j < ucap; ++j) {
        const int pj = j < rank ? colmap[j] : 0;
        for (int i = tid; i < nloc; i += kQrThreads)
            uout[(r0 + i) + int64_t(j) * rows] = j < rank ? sgn[j] * z[i + pj * ld] : 0.0;
    }
    if (upout) {
        const int stride = (rank + 3) / 4 * 4;
        for (int64_t t = tid; t < int64_t(nloc) * stride; t += kQrThreads) {
            const int i = static_cast<int>(t / stride), j = static_cast<int>(t % stride);
            const double v = j < rank ? sgn[j] * z[i + colmap[j] * ld] : 0.0;
            const int64_t o = (r0 + i) * stride + j;
            if (up_dtype == kF32) static_cast<float*>(upout)[o] = static_cast<float>(v);
            else static_cast<double*>(upout)[o] = v;
        }
    }
    if (crank == 0) {
        if (tid == 0) *rank_out = rank;
        if (diag_out)
            for (int k = tid; k < size; k += kQrThreads) diag_out[k] = beta[k];
    }
    if (X.cs > 1) cl.sync();  // keep every CTA's shared memory alive until all DSMEM reads are done
}

int pick_cluster(int64_t rows, int ncols, int* ld_out, size_t* smem_out) {
    for (int cs = 1; cs <= 16; cs *= 2) {
        const int ld = static_cast<int>((rows + cs - 1) / cs);
        const size_t smem = size_t(ld) * ncols * sizeof(double) + kQrFixedSmem;
        if (smem <= kQrSmemCap) {
            *ld_out = ld;
            *smem_out = smem;
            return cs;
        }
    }
    return 0;
}

}  // namespace

int64_t qr_max_rows(int ncols) {
    return static_cast<int64_t>((kQrSmemCap - kQrFixedSmem) / (sizeof(double) * std::max(ncols, 1))) * 16;
}

void launch_orthonormal_basis(const double* z, int64_t rows, int ncols, double* u, int ucap, void* up, int up_dtype,
                              int* rank_dev, double* diag, cudaStream_t s) {
    require(rows >= 1, "orthonormal_basis: empty input");
    require(ncols >= 1 && ncols <= kMaxRank, "orthonormal_basis: column count must be in [1, 64]");
    int ld = 0;
    size_t smem = 0;
    const int cs = pick_cluster(rows, ncols, &ld, &smem);
    require(cs > 0, "orthonormal_basis: sketch too large for the cluster QR");
    static bool attr = false;
    if (!attr) {
        TK_CUDA(cudaFuncSetAttribute(qr_colpiv_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kQrSmemCap)));
        TK_CUDA(cudaFuncSetAttribute(qr_colpiv_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs, 1, 1);
    cfg.blockDim = dim3(kQrThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = cs;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    TK_CUDA(cudaLaunchKernelEx(&cfg, qr_colpiv_cluster_kernel, z, rows, ncols, ld, u, ucap, up, up_dtype, rank_dev,
                               diag));
}

}  // namespace tkb
