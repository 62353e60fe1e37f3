// qr.cu — tall-skinny column-pivoted Householder QR on one thread-block cluster (sm_100a).
//
// Device restatement of orthonormal_basis (range_finder.hpp:18-29: Eigen
// ColPivHouseholderQR, rank = #leading |R_kk| > 1e-12 |R_00|, Q = first `rank` Householder
// columns in pivot order) followed by fix_column_signs (tucker.hpp:39-45), all in fp64.
//
// Z (rows x ncols, rows <= a few thousand, ncols <= 64) is split into contiguous row
// blocks held in the shared memory of the cluster's CTAs (distributed shared memory).
// Each Householder step needs one cluster-wide reduction (column-k tail norm, the dot
// products of column k with the trailing columns and row k itself); partial vectors are
// exchanged through DSMEM and summed in fixed CTA order, so the result is deterministic.
// The pivot choice and the LAPACK-style norm downdating (with direct recomputation below
// sqrt(eps)) are evaluated redundantly and identically by every CTA. Q is then formed in
// place over the stored reflectors (backward accumulation, one reduction per column).
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
constexpr size_t kQrFixedSmem = (2 * kSlot + kSlot + 8 * kMaxRank + 16) * sizeof(double);
constexpr size_t kQrSmemCap = 200 * 1024;

struct QrShared {
    double* z;      // [ld * ncols] own rows, column-major
    double* slot;   // [2][kSlot] exchange buffers (double-buffered)
    double* tot;    // [kSlot] reduced vector
    double* upd;    // [kMaxRank] updated column norms
    double* dir;    // [kMaxRank] directly computed column norms
    double* beta;   // [kMaxRank] R_kk
    double* tau;    // [kMaxRank]
    double* w;      // [kMaxRank]
    double* nrow;   // [kMaxRank] new row k
    double* misc;   // [16]
    int* flags;     // [kMaxRank]
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum of every CTA's slot[par][0:len] in CTA order into tot (block-visible on return).
__device__ void exchange_sum(cg::cluster_group& cl, QrShared& sh, int& par, int len) {
    cl.sync();
    const unsigned cs = cl.num_blocks();
    double* mine = sh.slot + par * kSlot;
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        double s = 0.0;
        for (unsigned c = 0; c < cs; ++c) s += cl.map_shared_rank(mine, c)[i];
        sh.tot[i] = s;
    }
    par ^= 1;
    __syncthreads();
}

__global__ void __launch_bounds__(kQrThreads, 1)
    qr_colpiv_cluster_kernel(const double* __restrict__ zin, int64_t rows, int ncols, int ld,
                             double* __restrict__ uout, int ucap, void* upout, int up_dtype, int* rank_out,
                             double* diag_out) {
    cg::cluster_group cl = cg::this_cluster();
    const int crank = static_cast<int>(cl.block_rank());
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    extern __shared__ __align__(16) double qsm[];
    QrShared sh;
    sh.z = qsm;
    sh.slot = sh.z + size_t(ld) * ncols;
    sh.tot = sh.slot + 2 * kSlot;
    sh.upd = sh.tot + kSlot;
    sh.dir = sh.upd + kMaxRank;
    sh.beta = sh.dir + kMaxRank;
    sh.tau = sh.beta + kMaxRank;
    sh.w = sh.tau + kMaxRank;
    sh.nrow = sh.w + kMaxRank;
    sh.misc = sh.nrow + kMaxRank;
    sh.flags = reinterpret_cast<int*>(sh.misc + 16);

    const int64_t r0 = int64_t(crank) * ld;
    const int nloc = static_cast<int>(lmax(0, lmin(ld, rows - r0)));
    double* z = sh.z;
    int par = 0;

    // load own rows
    for (int j = 0; j < ncols; ++j)
        for (int i = tid; i < ld; i += kQrThreads) z[i + j * ld] = i < nloc ? zin[(r0 + i) + j * rows] : 0.0;
    __syncthreads();

    // initial column norms (m_qr.col(k).norm())
    {
        double* slot = sh.slot + par * kSlot;
        for (int j = warp; j < ncols; j += kQrWarps) {
            double s = 0.0;
            for (int i = lane; i < nloc; i += 32) s += z[i + j * ld] * z[i + j * ld];
            s = warp_sum(s);
            if (lane == 0) slot[j] = s;
        }
        exchange_sum(cl, sh, par, ncols);
        for (int j = tid; j < ncols; j += kQrThreads) sh.upd[j] = sh.dir[j] = sqrt(sh.tot[j]);
        __syncthreads();
    }

    const double norm_downdate_threshold = sqrt(DBL_EPSILON);
    const int size = static_cast<int>(lmin(rows, ncols));
    for (int k = 0; k < size; ++k) {
        // pivot: first maximum of the updated norms over columns k..
        if (tid == 0) {
            int best = k;
            for (int j = k + 1; j < ncols; ++j)
                if (sh.upd[j] > sh.upd[best]) best = j;
            sh.flags[0] = best;
        }
        __syncthreads();
        const int best = sh.flags[0];
        if (best != k) {
            for (int i = tid; i < nloc; i += kQrThreads) {
                const double t = z[i + k * ld];
                z[i + k * ld] = z[i + best * ld];
                z[i + best * ld] = t;
            }
            if (tid == 0) {
                double t = sh.upd[k];
                sh.upd[k] = sh.upd[best];
                sh.upd[best] = t;
                t = sh.dir[k];
                sh.dir[k] = sh.dir[best];
                sh.dir[best] = t;
            }
        }
        __syncthreads();

        // local partials: [0] tail norm^2 of column k (rows > k), [j-k] dot(col k, col j)
        // over rows > k, [kMaxRank + (j-k)] row k (owner only; others contribute 0)
        const int lk = static_cast<int>(k - r0);  // local index of row k (may be outside)
        const bool owner = lk >= 0 && lk < nloc;
        const int i_start = static_cast<int>(lmax(0, k + 1 - r0));
        {
            double* slot = sh.slot + par * kSlot;
            for (int j = k + warp; j < ncols; j += kQrWarps) {
                double s = 0.0;
                for (int i = i_start + lane; i < nloc; i += 32) s += z[i + k * ld] * z[i + j * ld];
                s = warp_sum(s);
                if (lane == 0) {
                    slot[j - k] = s;
                    slot[kMaxRank + (j - k)] = owner ? z[lk + j * ld] : 0.0;
                }
            }
        }
        exchange_sum(cl, sh, par, kMaxRank + (ncols - k));

        // Householder vector of column k (makeHouseholderInPlace) + w = essential^T * bottom + row0
        if (tid == 0) {
            const double tail_sq = (rows - k == 1) ? 0.0 : sh.tot[0];
            const double c0 = sh.tot[kMaxRank];
            double tau, beta, denom = 1.0;
            int zero_ess = 0;
            if (tail_sq <= DBL_MIN) {
                tau = 0.0;
                beta = c0;
                zero_ess = 1;
            } else {
                beta = sqrt(c0 * c0 + tail_sq);
                if (c0 >= 0.0) beta = -beta;
                denom = c0 - beta;
                tau = (beta - c0) / beta;
            }
            sh.beta[k] = beta;
            sh.tau[k] = tau;
            sh.misc[0] = denom;
            sh.flags[1] = zero_ess;
        }
        __syncthreads();
        const double tau = sh.tau[k], denom = sh.misc[0];
        const bool zero_ess = sh.flags[1] != 0;
        for (int j = k + 1 + tid; j < ncols; j += kQrThreads) {
            const double rowk = sh.tot[kMaxRank + (j - k)];
            const double wj = tau != 0.0 ? rowk + sh.tot[j - k] / denom : 0.0;
            sh.w[j] = wj;
            sh.nrow[j] = tau != 0.0 ? rowk - tau * wj : rowk;
        }
        // essential part of column k in place; R_kk on the owner
        for (int i = i_start + tid; i < nloc; i += kQrThreads) z[i + k * ld] = zero_ess ? 0.0 : z[i + k * ld] / denom;
        if (owner && tid == 0) z[lk + k * ld] = sh.beta[k];
        __syncthreads();
        // apply H_k to the trailing columns
        for (int j = k + 1 + warp; j < ncols; j += kQrWarps) {
            const double wj = sh.w[j];
            if (tau != 0.0)
                for (int i = i_start + lane; i < nloc; i += 32) z[i + j * ld] -= (tau * z[i + k * ld]) * wj;
            if (owner && lane == 0) z[lk + j * ld] = sh.nrow[j];
        }
        // norm downdate (LAWN 176 / xGEQP3), redundantly per CTA
        if (tid == 0) sh.flags[2] = 0;
        __syncthreads();
        for (int j = k + 1 + tid; j < ncols; j += kQrThreads) {
            sh.flags[8 + j] = 0;
            const double u = sh.upd[j];
            if (u != 0.0) {
                double temp = fabs(sh.nrow[j]) / u;
                temp = (1.0 + temp) * (1.0 - temp);
                temp = temp < 0.0 ? 0.0 : temp;
                const double ratio = u / sh.dir[j];
                const double temp2 = temp * ratio * ratio;
                if (temp2 <= norm_downdate_threshold) {
                    sh.flags[8 + j] = 1;
                    atomicOr(&sh.flags[2], 1);
                } else {
                    sh.upd[j] = u * sqrt(temp);
                }
            }
        }
        __syncthreads();
        if (sh.flags[2]) {  // direct recomputation of the flagged tail norms (rows > k)
            double* slot = sh.slot + par * kSlot;
            for (int j = k + 1 + warp; j < ncols; j += kQrWarps) {
                double s = 0.0;
                if (sh.flags[8 + j])
                    for (int i = i_start + lane; i < nloc; i += 32) s += z[i + j * ld] * z[i + j * ld];
                s = warp_sum(s);
                if (lane == 0) slot[j] = s;
            }
            exchange_sum(cl, sh, par, ncols);
            for (int j = k + 1 + tid; j < ncols; j += kQrThreads)
                if (sh.flags[8 + j]) sh.upd[j] = sh.dir[j] = sqrt(sh.tot[j]);
            __syncthreads();
        }
    }

    // rank cut (range_finder.hpp:24-26)
    if (tid == 0) {
        const double top = fabs(sh.beta[0]);
        int rank = 0;
        while (rank < size && fabs(sh.beta[rank]) > 1e-12 * top) ++rank;
        sh.flags[3] = rank;
    }
    __syncthreads();
    const int rank = sh.flags[3];

    // explicit Q(:, 0:rank) = H_0 ... H_{rank-1} [I; 0], formed in place
    for (int k = rank - 1; k >= 0; --k) {
        const double tau = sh.tau[k];
        const int lk = static_cast<int>(k - r0);
        const bool owner = lk >= 0 && lk < nloc;
        const int i_start = static_cast<int>(lmax(0, k + 1 - r0));
        if (k + 1 < rank) {
            double* slot = sh.slot + par * kSlot;
            for (int j = k + 1 + warp; j < rank; j += kQrWarps) {
                double s = 0.0;
                for (int i = i_start + lane; i < nloc; i += 32) s += z[i + k * ld] * z[i + j * ld];
                s = warp_sum(s);
                if (lane == 0) slot[j - k] = s;
            }
            exchange_sum(cl, sh, par, rank - k);
            for (int j = k + 1 + warp; j < rank; j += kQrWarps) {
                const double t = sh.tot[j - k];
                if (tau != 0.0)
                    for (int i = i_start + lane; i < nloc; i += 32) z[i + j * ld] -= (tau * z[i + k * ld]) * t;
                if (owner && lane == 0) z[lk + j * ld] = -tau * t;
            }
            __syncthreads();
        }
        // column k <- H_k e_k
        for (int i = tid; i < nloc; i += kQrThreads) {
            const int64_t gi = r0 + i;
            double v;
            if (gi < k) v = 0.0;
            else if (gi == k) v = 1.0 - tau;
            else v = -tau * z[i + k * ld];
            z[i + k * ld] = v;
        }
        __syncthreads();
    }

    // sign fix: largest |entry| of each column positive (first maximum on ties)
    if (rank > 0) {
        double* slot = sh.slot + par * kSlot;
        for (int j = warp; j < rank; j += kQrWarps) {
            double best = -1.0, val = 0.0;
            int bi = 0x7fffffff;
            for (int i = lane; i < nloc; i += 32) {
                const double a = fabs(z[i + j * ld]);
                if (a > best) {
                    best = a;
                    bi = i;
                    val = z[i + j * ld];
                }
            }
            // warp arg-max, first index on ties
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                const double ov = __shfl_xor_sync(0xffffffffu, val, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                    val = ov;
                }
            }
            if (lane == 0) {
                slot[3 * j] = best;
                slot[3 * j + 1] = static_cast<double>(bi);
                slot[3 * j + 2] = val;
            }
        }
        cl.sync();
        const unsigned cs = cl.num_blocks();
        for (int j = tid; j < rank; j += kQrThreads) {
            double best = -1.0, val = 0.0;
            for (unsigned c = 0; c < cs; ++c) {
                const double* ps = cl.map_shared_rank(slot, c);
                if (ps[3 * j] > best) {  // CTAs hold increasing rows: strict > keeps the first
                    best = ps[3 * j];
                    val = ps[3 * j + 2];
                }
            }
            sh.w[j] = val < 0.0 ? -1.0 : 1.0;
        }
        par ^= 1;
        __syncthreads();
    }

    // outputs
    for (int j = 0; j < ucap; ++j)
        for (int i = tid; i < nloc; i += kQrThreads) uout[(r0 + i) + int64_t(j) * rows] = j < rank ? sh.w[j] * z[i + j * ld] : 0.0;
    if (upout) {
        const int stride = (rank + 3) / 4 * 4;
        for (int64_t t = tid; t < int64_t(nloc) * stride; t += kQrThreads) {
            const int i = static_cast<int>(t / stride), j = static_cast<int>(t % stride);
            const double v = j < rank ? sh.w[j] * z[i + j * ld] : 0.0;
            const int64_t o = (r0 + i) * stride + j;
            if (up_dtype == kF32) static_cast<float*>(upout)[o] = static_cast<float>(v);
            else static_cast<double*>(upout)[o] = v;
        }
    }
    if (crank == 0) {
        if (tid == 0) *rank_out = rank;
        if (diag_out)
            for (int k = tid; k < size; k += kQrThreads) diag_out[k] = sh.beta[k];
    }
    cl.sync();  // keep every CTA's shared memory alive until all DSMEM reads are done
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
    require(ucap >= ncols || ucap >= 0, "orthonormal_basis: output capacity");
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
