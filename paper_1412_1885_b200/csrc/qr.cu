// qr.cu — tall-skinny column-pivoted Householder QR on one thread-block cluster (sm_100a).
//
// Device restatement of orthonormal_basis (range_finder.hpp:18-29: Eigen
// ColPivHouseholderQR, rank = #leading |R_kk| > 1e-12 |R_00|, Q = first `rank` Householder
// columns in pivot order) followed by fix_column_signs (tucker.hpp:39-45), all in fp64.
//
// Z (rows x ncols, ncols <= 64) is split into contiguous row blocks held in the shared
// memory of the CTAs of one thread-block cluster. The QR is latency-bound (every step
// depends on the previous one), so a step is kept to: warp-redundant pivot argmax ->
// column swap -> ONE reduction of [col_k . col_j | row_k] (8 threads per column over
// interleaved rows + 3 shuffle rounds, then a DSMEM exchange summed in fixed CTA order)
// -> Householder scalars evaluated redundantly -> 2-D parallel trailing update + one
// thread per column for the LAPACK-style norm downdate (direct recomputation below
// sqrt(eps), as Eigen / xGEQP3). Q is formed in place by backward accumulation with the
// same reduction. All loops stay rolled: the kernel is small enough to live in the
// instruction cache (straight-line unrolled variants were instruction-fetch bound).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace cg = cooperative_groups;

#ifdef TK_QR_TRACE
__device__ long long g_qr_trace[4096];
#define QR_MARK(slot)                                                                            \
    do {                                                                                         \
        if (threadIdx.x == 0 && blockIdx.x == 0 && (slot) < 4096) g_qr_trace[(slot)] = clock64(); \
    } while (0)
#else
#define QR_MARK(slot) \
    do {              \
    } while (0)
#endif

namespace tkb {

namespace {

constexpr int kQrThreads = 256;
constexpr int kTpc = 16;  // threads per column in the reductions (kQrThreads / kTpc columns per pass)
constexpr int kVec = 2 * kMaxRank + 8;
constexpr size_t kQrFixedSmem = (3 * kVec + 6 * kMaxRank) * sizeof(double) + 16 * sizeof(int);
constexpr size_t kQrSmemCap = 200 * 1024;

struct Sh {
    double* z;     // [ncols][ld] own rows, column-major
    double* slot;  // [2][kVec] cluster exchange
    double* tot;   // [kVec]
    double *upd, *dir, *beta, *taus, *sgn, *wv;
    int* flag;
};

// tot[j - j0] (j in [j0, j1)) = sum over own rows i in [i0, nloc) of a[i] * z[j][i], then the
// sum over the cluster's CTAs; extra[e * xstride] (e < nextra; a null `extra` contributes
// zeros) is summed into tot[kMaxRank + e] the same way. Block-visible on return.
__device__ void reduce_dots(Sh& sh, cg::cluster_group& cl, unsigned cs, int& par, const double* a, int ld, int i0,
                            int nloc, int j0, int j1, const double* extra, int xstride, int nextra) {
    const int tid = threadIdx.x, sub = tid % kTpc, grp = tid / kTpc;
    double* m = sh.slot + par * kVec;
    // warp-uniform trip count (the shuffles need all 32 lanes): groups past j1 compute 0
    for (int base = j0; base + (tid / 32) * (32 / kTpc) < j1; base += kQrThreads / kTpc) {
        const int j = base + grp;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (j < j1) {
            const double* b = sh.z + size_t(j) * ld;
            int i = i0 + sub;
            for (; i + 3 * kTpc < nloc; i += 4 * kTpc) {
                s0 = fma(a[i], b[i], s0);
                s1 = fma(a[i + kTpc], b[i + kTpc], s1);
                s2 = fma(a[i + 2 * kTpc], b[i + 2 * kTpc], s2);
                s3 = fma(a[i + 3 * kTpc], b[i + 3 * kTpc], s3);
            }
            for (; i < nloc; i += kTpc) s0 = fma(a[i], b[i], s0);
        }
        double s = (s0 + s1) + (s2 + s3);
        s += __shfl_xor_sync(0xffffffffu, s, 8);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (sub == 0 && j < j1) m[j - j0] = s;
    }
    for (int e = tid; e < nextra; e += kQrThreads) m[kMaxRank + e] = extra ? extra[size_t(e) * xstride] : 0.0;
    const int len = kMaxRank + nextra;
    if (cs > 1) {
        cl.sync();
        for (int t = tid; t < len; t += kQrThreads) {
            if (t >= j1 - j0 && t < kMaxRank) continue;
            double s = 0.0;
            for (unsigned c = 0; c < cs; ++c) s += cl.map_shared_rank(m, c)[t];
            sh.tot[t] = s;
        }
    } else {
        __syncthreads();
        for (int t = tid; t < len; t += kQrThreads) sh.tot[t] = m[t];
    }
    par ^= 1;
    __syncthreads();
}


// ---------------------------------------------------------------------------------------
// Fast path: column-pivoted CholeskyQR2. In exact arithmetic ColPivHouseholderQR's pivot at
// step k is the column of largest remaining norm, i.e. the largest diagonal entry of the
// Schur complement of the Gram matrix G = Z^T Z, and |R_kk| is its square root; so the
// pivoted Cholesky of G gives the same pivots and |R_kk|, and Q = Z_P R^{-1} the same
// columns up to sign (fixed by the sign rule afterwards). One more Cholesky pass on Q
// (CholeskyQR2, applied to first order: Q1^T Q1 = I + O(eps cond^2)) restores orthonormality
// to ~eps. Taken only when Z is well conditioned
// (every R_kk > kFastMinRatio R_00, so the 1e-12 rank cut cannot bite); otherwise the kernel
// falls through to the Householder path with Z untouched. 3 cluster exchanges instead of
// one per Householder step.
// ---------------------------------------------------------------------------------------
constexpr double kFastMinRatio = 1e-4;  // cond(Z) <= 1e4: first-order second pass exact to ~1e-16
// Near-tie guard: the Cholesky Schur diagonals carry a relative error up to ~eps / kFastMinRatio^2
// (cancellation in S_jj = G_jj - sum l^2), the Householder norm downdate (the oracle's and the
// reference's algorithm, range_finder.hpp:18-29) much less; when the two largest remaining
// candidates of a pivot step are closer than kTieGapSq (relative, squared norms) the fast path
// gives up and the Householder path decides the pivot.
constexpr double kTieGapSq = 1e-6;

// gp[a + b n] = sum over own rows of z[:, a] z[:, b] (full symmetric n x n)
__device__ void gram_partial(const double* z, int ld, int nloc, int n, double* gp) {
    const int npair = n * (n + 1) / 2;
    for (int t = threadIdx.x; t < npair; t += kQrThreads) {
        int a = 0, rem = t;
        while (rem >= n - a) {  // t -> (a, b), a <= b
            rem -= n - a;
            ++a;
        }
        const int b = a + rem;
        const double* za = z + size_t(a) * ld;
        const double* zb = z + size_t(b) * ld;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int i = 0;
        for (; i + 4 <= nloc; i += 4) {
            s0 = fma(za[i], zb[i], s0);
            s1 = fma(za[i + 1], zb[i + 1], s1);
            s2 = fma(za[i + 2], zb[i + 2], s2);
            s3 = fma(za[i + 3], zb[i + 3], s3);
        }
        for (; i < nloc; ++i) s0 = fma(za[i], zb[i], s0);
        const double v = (s0 + s1) + (s2 + s3);
        gp[a + b * n] = v;
        gp[b + a * n] = v;
    }
}

// The same on the FP64 tensor cores: each warp takes 8x8 tiles (ti <= tj) of the Gram and
// runs mma.m8n8k4.f64 over the own rows, 4 per step (rows >= nloc count as zero). Lane
// layouts (PTX m8n8k4 .row.col f64): A[m][k] = lane (m = lane / 4, k = lane % 4), B[k][n] =
// lane (k = lane % 4, n = lane / 4), D[m][2 (lane % 4) + e] for m = lane / 4.
__device__ void gram_partial_dmma(const double* z, int nloc, int n, int ld, double* gp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nt = (n + 7) / 8;
    const int ntile = nt * (nt + 1) / 2;
    const int g = lane >> 2, t4 = lane & 3;
    for (int tt = warp; tt < ntile; tt += kQrThreads / 32) {
        int ti = 0, rem = tt;
        while (rem >= nt - ti) {
            rem -= nt - ti;
            ++ti;
        }
        const int tj = ti + rem;
        const int ca = 8 * ti + g, cb = 8 * tj + g;  // A column (row of G) / B column of this lane
        const double* za = z + size_t(ca < n ? ca : 0) * ld;
        const double* zb = z + size_t(cb < n ? cb : 0) * ld;
        double d0 = 0.0, d1 = 0.0;
        for (int r0 = 0; r0 < nloc; r0 += 4) {  // warp-uniform trip count
            const int r = r0 + t4;
            const double a = (ca < n && r < nloc) ? za[r] : 0.0;
            const double b = (cb < n && r < nloc) ? zb[r] : 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                         : "+d"(d0), "+d"(d1)
                         : "d"(a), "d"(b));
        }
        const int row = 8 * ti + g;
        const int c0 = 8 * tj + 2 * t4;
        if (row < n) {
            if (c0 < n) gp[row + c0 * n] = d0, gp[c0 + row * n] = d0;
            if (c0 + 1 < n) gp[row + (c0 + 1) * n] = d1, gp[(c0 + 1) + row * n] = d1;
        }
    }
}

// gs = sum over the cluster's CTAs (fixed order) of gp; every CTA ends with the same gs
__device__ void gram_reduce(cg::cluster_group& cl, unsigned cs, double* gp, double* gs, int n) {
    if (cs > 1) cl.sync();
    else __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += kQrThreads) {
        // all remote loads in flight before the fixed-order sum (DSMEM latency paid once)
        double v = 0.0;
        for (unsigned c0 = 0; c0 < cs; c0 += 8) {
            double t[8];
#pragma unroll
            for (unsigned c = 0; c < 8; ++c)
                t[c] = c0 + c < cs ? (cs > 1 ? cl.map_shared_rank(gp, c0 + c) : gp)[e] : 0.0;
#pragma unroll
            for (unsigned c = 0; c < 8; ++c)
                if (c0 + c < cs) v += t[c];
        }
        gs[e] = v;
    }
    if (cs > 1) cl.sync();  // every CTA done reading the partials before they are rewritten
    else __syncthreads();
}

// Right-looking Cholesky of gs (n x n, full symmetric, destroyed) by the whole CTA, with
// ColPiv pivoting (first largest Schur diagonal) when `pivot`: R (upper, col-major, n x n)
// into rr, 1 / R_kk into rinv, source column of pivot position k into perm[k]. Returns false
// (CTA-uniform) when a pivot is not positive or R_kk <= kFastMinRatio R_00 (the caller then
// takes the Householder path). Per step: warp 0 picks the pivot (exact first-max via three
// warp reductions on the non-negative doubles' bit patterns) and the scalars, all threads
// swap and update the trailing Schur complement; ~3 block barriers per step.
__device__ bool cta_pchol(double* gs, int n, bool pivot, double* rr, double* rinv, int* perm, int* ctl, double* pmargin) {
    const int tid = threadIdx.x, lane = tid & 31;
    for (int j = tid; j < n; j += kQrThreads) perm[j] = j;
    for (int e = tid; e < n * n; e += kQrThreads) rr[e] = 0.0;
    if (tid == 0) {
        ctl[1] = 0;
        *pmargin = 1.0;
    }
    __syncthreads();
    double r00 = 0.0;
    // pivot margin = 1 - sqrt(max over steps of second / top): the largest ratio is tracked as a
    // fraction (cross-multiplied compare), the division and square root happen once at the end
    double mnum = 0.0, mden = 1.0;  // (lane 0 of warp 0)
    for (int k = 0; k < n; ++k) {
        if (tid < 32) {
            int best = k;
            if (pivot) {
                // candidates j = k + lane, k + lane + 32 (n <= 64): first maximum of S_jj >= 0
                unsigned long long b0 = 0, b1 = 0;
                const int j0 = k + lane, j1 = k + lane + 32;
                if (j0 < n) b0 = __double_as_longlong(fmax(gs[j0 + j0 * n], 0.0));
                if (j1 < n) b1 = __double_as_longlong(fmax(gs[j1 + j1 * n], 0.0));
                const unsigned long long bm = b0 > b1 ? b0 : b1;
                const unsigned hi = __reduce_max_sync(0xffffffffu, unsigned(bm >> 32));
                const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned(bm >> 32) == hi) ? unsigned(bm) : 0u);
                const unsigned long long top = (static_cast<unsigned long long>(hi) << 32) | lo;
                const unsigned cand = (j0 < n && b0 == top) ? unsigned(j0) : ((j1 < n && b1 == top) ? unsigned(j1) : 0xffffu);
                best = static_cast<int>(__reduce_min_sync(0xffffffffu, cand));
                if (best >= n) best = k;
                // the largest other candidate: near-tie guard and pivot margin
                const unsigned long long c0 = (j0 == best) ? 0ull : b0, c1 = (j1 == best) ? 0ull : b1;
                const unsigned long long cm = c0 > c1 ? c0 : c1;
                const unsigned h2 = __reduce_max_sync(0xffffffffu, unsigned(cm >> 32));
                const unsigned l2 = __reduce_max_sync(0xffffffffu, (unsigned(cm >> 32) == h2) ? unsigned(cm) : 0u);
                const double dtop = __longlong_as_double(static_cast<long long>(top));
                const double dsec = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(h2) << 32) | l2));
                if (lane == 0 && k + 1 < n) {
                    if (dtop - dsec < kTieGapSq * dtop) ctl[1] = 1;
                    else if (dsec * mden > mnum * dtop) mnum = dsec, mden = dtop;
                }
            }
            if (lane == 0) ctl[0] = best;
        }
        __syncthreads();
        if (pivot && ctl[1]) return false;  // near tie (uniform)
        const int best = ctl[0];
        if (best != k) {  // symmetric swap k <-> best; rows < k of R: swap their columns
            for (int j = tid; j < n; j += kQrThreads) {
                const double t0 = gs[k + j * n];
                gs[k + j * n] = gs[best + j * n];
                gs[best + j * n] = t0;
            }
            __syncthreads();
            for (int i = tid; i < n; i += kQrThreads) {
                const double t0 = gs[i + k * n];
                gs[i + k * n] = gs[i + best * n];
                gs[i + best * n] = t0;
            }
            for (int i = tid; i < k; i += kQrThreads) {
                const double t0 = rr[i + k * n];
                rr[i + k * n] = rr[i + best * n];
                rr[i + best * n] = t0;
            }
            if (tid == 0) {
                const int t0 = perm[k];
                perm[k] = perm[best];
                perm[best] = t0;
            }
            __syncthreads();
        }
        const double d = gs[k + k * n];
        if (k == 0) r00 = d > 0.0 ? sqrt(d) : 0.0;
        const double rkk = d > 0.0 ? sqrt(d) : 0.0;
        if (!(d > 0.0) || !(rkk > kFastMinRatio * r00)) return false;  // uniform: same values everywhere
        const double inv = 1.0 / rkk;
        const int m = n - k - 1;
        // trailing update S_ij -= (S_ki / R_kk)(S_kj / R_kk), i, j > k; the diagonal threads
        // also write row k of R
        // (16 x 16 thread tiles over the trailing block: no integer division in the index math)
        (void)m;
        for (int j = k + 1 + (tid >> 4); j < n; j += kQrThreads / 16) {
            const double rkj = gs[k + j * n] * inv;
            for (int i = k + 1 + (tid & 15); i < n; i += 16) {
                const double rki = gs[k + i * n] * inv;
                gs[i + j * n] = fma(-rki, rkj, gs[i + j * n]);
                if (i == j) rr[k + j * n] = rkj;
            }
        }
        if (tid == 0) {
            rr[k + k * n] = rkk;
            rinv[k] = inv;
        }
        __syncthreads();
    }
    if (tid == 0 && pivot) *pmargin = 1.0 - sqrt(mnum / mden);
    __syncthreads();
    return true;
}

// n <= 32: the pivoted Cholesky by one warp with lane i keeping row i of the Gram matrix in
// registers and its Schur diagonal in `dg`; no physical swaps: the pivot of step k is the
// first largest remaining diagonal (original index order), its column reaches every lane
// through one indexed branch (k-uniform), and the unmasked trailing update leaves finished
// rows/columns untouched (their multipliers are zero). Step k stores l_i = S_ip / d into
// lraw[k n + i] (1 at the pivot) and sqrt(d) into rdk[k]; R is assembled afterwards.
__device__ __noinline__ bool warp_pchol_reg(const double* gs, int n, double* lraw, double* rdk, int* perm, double* colk,
                                            double* pmargin) {
    const int lane = threadIdx.x & 31;
    double row[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) row[j] = (lane < n && j < n) ? gs[lane + j * n] : 0.0;
    double dg = lane < n ? gs[lane + lane * n] : 0.0;
    bool done = lane >= n;
    double r00 = 0.0;
    // first maximum of the remaining Schur diagonal (exact, lowest index on ties), and the
    // largest of the other remaining candidates (the pivot margin, SURVEY §7 hard part 1)
    auto pick = [&](int& pv, double& d, double& d2) {
        const unsigned long long key = done ? 0ull : static_cast<unsigned long long>(__double_as_longlong(fmax(dg, 0.0)));
        const unsigned hi = __reduce_max_sync(0xffffffffu, unsigned(key >> 32));
        const unsigned lo = __reduce_max_sync(0xffffffffu, unsigned(key >> 32) == hi ? unsigned(key) : 0u);
        const bool cand = !done && key == ((static_cast<unsigned long long>(hi) << 32) | lo);
        pv = static_cast<int>(__reduce_min_sync(0xffffffffu, cand ? unsigned(lane) : 0xffffu));
        d = __shfl_sync(0xffffffffu, dg, pv & 31);
        const unsigned long long k2 = (lane == pv) ? 0ull : key;
        const unsigned h2 = __reduce_max_sync(0xffffffffu, unsigned(k2 >> 32));
        const unsigned l2 = __reduce_max_sync(0xffffffffu, unsigned(k2 >> 32) == h2 ? unsigned(k2) : 0u);
        d2 = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(h2) << 32) | l2));
    };
    int pv;
    double d, d2;
    double mnum = 0.0, mden = 1.0;  // largest second / top ratio so far, as a fraction
    pick(pv, d, d2);
#pragma unroll 1
    for (int k = 0; k < n; ++k) {
        QR_MARK(700 + 4 * k);
        if (k == 0) r00 = d;  // (squared) R_00
        // R_kk > kFastMinRatio R_00 tested on the squares: the sqrt stays off the step's chain
        if (pv >= n || !(d > 0.0) || !(d > kFastMinRatio * kFastMinRatio * r00)) return false;
        if (k + 1 < n) {  // near tie: the Householder path decides
            if (d - d2 < kTieGapSq * d) return false;
            if (d2 * mden > mnum * d) mnum = d2, mden = d;  // (no division / square root on the step chain)
        }
        QR_MARK(701 + 4 * k);
        const double rd = 1.0 / d;  // overlaps the row exchange below
        // the pivot lane publishes its Schur row S_p. (= column S_.p, S symmetric): lane i reads
        // its S_ip from it, and the trailing update S_ij -= l_i S_pj reads the whole row
        const bool piv = lane == pv;
        if (piv) {
#pragma unroll
            for (int j = 0; j < 32; ++j) colk[j] = row[j];
        }
        __syncwarp();
        const double cp = colk[lane];
        QR_MARK(702 + 4 * k);
        const double l = (done || piv) ? 0.0 : cp * rd;
        if (lane < n) lraw[k * n + lane] = piv ? 1.0 : l;
        if (piv) {
            done = true;
            perm[k] = pv;
            rdk[k] = d;  // R_kk^2; square roots taken after the loop, off the step chain
        }
        QR_MARK(703 + 4 * k);
        // the diagonal first: the next pivot search overlaps the rest of the row update
        dg = fma(-l, cp, dg);
        int pv1 = n;
        double d1 = 0.0, d12 = 0.0;
        if (k + 1 < n) pick(pv1, d1, d12);
#pragma unroll
        for (int j = 0; j < 32; ++j) row[j] = fma(-l, colk[j], row[j]);
        __syncwarp();
        pv = pv1;
        d = d1;
        d2 = d12;
    }
    for (int k = lane; k < n; k += 32) rdk[k] = sqrt(rdk[k]);
    if (lane == 0) *pmargin = 1.0 - sqrt(mnum / mden);
    __syncwarp();
    return true;
}

// n <= 32: X = R^{-1} (R upper, col-major n x n; rinv = 1 / R_kk) by one warp, lane j holding
// column j in registers: right-looking back substitution (x_i = acc_i / R_ii, then acc_k -=
// R_ki x_i for k < i), so each step's chain is one multiply and one FMA.
__device__ void warp_upper_inv(const double* rr, const double* rinv, int n, double* x) {
    const int j = threadIdx.x & 31;
    double acc[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) acc[k] = k == j ? 1.0 : 0.0;
#pragma unroll
    for (int i = 31; i >= 0; --i) {
        if (i < n) {
            const double xi = acc[i] * rinv[i];
            acc[i] = xi;
            const double* ri = rr + size_t(i) * n;  // column i of R: R[k][i] = ri[k]
#pragma unroll
            for (int k = 0; k < i; ++k) acc[k] = fma(-ri[k], xi, acc[k]);
        }
    }
    if (j < n)
#pragma unroll
        for (int k = 0; k < 32; ++k)
            if (k < n) x[k + size_t(j) * n] = acc[k];
}

// out (own rows, ld) = in_P X on the FP64 tensor cores: each warp takes 8 x 8 output tiles and
// runs mma.m8n8k4.f64 over k (X: n x n col-major; perm: column order of `in`, may be null).
// A[m][k] = in[row0 + m, perm[k0 + k]] (m = lane / 4, k = lane % 4), B[k][c] = X[k0 + k][col0 + c]
// (k = lane % 4, c = lane / 4), D[m][2 (lane % 4) + e].
__device__ void apply_dmma(const double* in, double* out, int ld, int nloc, int n, const double* x, const int* perm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int rt = (nloc + 7) / 8, ct = (n + 7) / 8;
    for (int tt = warp; tt < rt * ct; tt += kQrThreads / 32) {
        const int row0 = (tt % rt) * 8, col0 = (tt / rt) * 8;
        const int ra = row0 + g;      // A row of this lane
        const int cb = col0 + g;      // B column of this lane
        double d0 = 0.0, d1 = 0.0;
        for (int k0 = 0; k0 < n; k0 += 4) {
            const int k = k0 + t4;
            const double a = (ra < nloc && k < n) ? in[ra + size_t(perm ? perm[k] : k) * ld] : 0.0;
            const double b = (k < n && cb < n) ? x[k + size_t(cb) * n] : 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                         : "+d"(d0), "+d"(d1)
                         : "d"(a), "d"(b));
        }
        const int r = row0 + g, c = col0 + 2 * t4;
        if (r < nloc) {
            if (c < n) out[r + size_t(c) * ld] = d0;
            if (c + 1 < n) out[r + size_t(c + 1) * ld] = d1;
        }
    }
}

// n <= 32, one thread per own row i (rows in registers): out_i = in_i,P R^{-1} by forward
// substitution, right-looking (x_k = acc_k / R_kk, then acc_j -= x_k R_kj for j > k: the
// chain per step is one multiply and one FMA). R upper, col-major n x n, rinv = 1 / R_kk.
__device__ void rows_trsm_perm(const double* in, double* out, int ld, int nloc, int n, const double* rr,
                               const double* rinv, const int* perm) {
    for (int i = threadIdx.x; i < nloc; i += kQrThreads) {
        double acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = j < n ? in[i + size_t(perm[j]) * ld] : 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            if (k < n) {
                acc[k] *= rinv[k];
                const double xk = acc[k];
                const double* rk = rr + k;  // R[k][j] = rr[k + j n]
#pragma unroll
                for (int j = k + 1; j < 32; ++j)
                    if (j < n) acc[j] = fma(-xk, rk[size_t(j) * n], acc[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < n) out[i + size_t(j) * ld] = acc[j];
    }
}

// n <= 32, one thread per own row: out_i = in_i M (M upper triangular, col-major n x n)
__device__ void rows_mul_upper(const double* in, double* out, int ld, int nloc, int n, const double* m) {
    for (int i = threadIdx.x; i < nloc; i += kQrThreads) {
        double x[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = j < n ? in[i + size_t(j) * ld] : 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j < n) {
                const double* mj = m + size_t(j) * n;
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int k = 0; k < 32; k += 2) {
                    if (k <= j) a0 = fma(x[k], mj[k], a0);
                    if (k + 1 <= j) a1 = fma(x[k + 1], mj[k + 1], a1);
                }
                out[i + size_t(j) * ld] = a0 + a1;
            }
        }
    }
}

// X = R^{-1} (upper triangular, n x n col-major) by one warp, lanes over the columns j:
// X_jj = 1 / R_jj, X_ij = -(sum_{k=i+1..j} R_ik X_kj) / R_ii for i < j (rolled loops)
__device__ void warp_tri_inv(const double* rr, const double* rinv, int n, double* x) {
    const int lane = threadIdx.x & 31;
    for (int j = lane; j < n; j += 32) {
        double* xj = x + size_t(j) * n;
        for (int i = j + 1; i < n; ++i) xj[i] = 0.0;
        xj[j] = rinv[j];
        for (int i = j - 1; i >= 0; --i) {
            double a0 = 0.0, a1 = 0.0;
            int k = i + 1;
            for (; k + 2 <= j + 1; k += 2) {
                a0 = fma(rr[i + size_t(k) * n], xj[k], a0);
                a1 = fma(rr[i + size_t(k + 1) * n], xj[k + 1], a1);
            }
            if (k <= j) a0 = fma(rr[i + size_t(k) * n], xj[k], a0);
            xj[i] = -(a0 + a1) * rinv[i];
        }
    }
}

// out[:, j] = sum_{k <= j} in[:, perm[k]] X[k, j] for the own rows (X upper triangular)
__device__ void apply_upper(const double* in, double* out, int ld, int nloc, int n, const double* x, const int* perm) {
    for (int e = threadIdx.x; e < nloc * n; e += kQrThreads) {
        const int i = e % nloc, j = e / nloc;
        const double* xj = x + size_t(j) * n;
        double a0 = 0.0, a1 = 0.0;
        int k = 0;
        for (; k + 2 <= j + 1; k += 2) {
            a0 = fma(in[i + size_t(perm[k]) * ld], xj[k], a0);
            a1 = fma(in[i + size_t(perm[k + 1]) * ld], xj[k + 1], a1);
        }
        if (k <= j) a0 = fma(in[i + size_t(perm[k]) * ld], xj[k], a0);
        out[i + size_t(j) * ld] = a0 + a1;
    }
}

// zr[j * ld] = fma(a, w[j], zr[j * ld]) for j in [j0, j1): loads of a group issued before its
// stores (the compiler cannot prove the column stores do not alias the next loads)
__device__ __forceinline__ void axpy_row(double* zr, int ld, int j0, int j1, double a, const double* w) {
    int j = j0;
    for (; j + 4 <= j1; j += 4) {
        const double z0 = zr[j * ld], z1 = zr[(j + 1) * ld], z2 = zr[(j + 2) * ld], z3 = zr[(j + 3) * ld];
        const double w0 = w[j], w1 = w[j + 1], w2 = w[j + 2], w3 = w[j + 3];
        zr[j * ld] = fma(a, w0, z0);
        zr[(j + 1) * ld] = fma(a, w1, z1);
        zr[(j + 2) * ld] = fma(a, w2, z2);
        zr[(j + 3) * ld] = fma(a, w3, z3);
    }
    for (; j < j1; ++j) zr[j * ld] = fma(a, w[j], zr[j * ld]);
}

__global__ void __launch_bounds__(kQrThreads, 1)
    qr_colpiv_cluster_kernel(const double* __restrict__ zin, int64_t rows, int ncols, int ld,
                             double* __restrict__ uout, int ucap, void* upout, int up_dtype, int* rank_out,
                             double* diag_out, int fast, int rowpar, int nparts, double* margin_out, int plain) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned cs = cl.num_blocks();
    const int crank = static_cast<int>(cl.block_rank());
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    extern __shared__ __align__(16) double qsm[];
    Sh sh;
    sh.z = qsm;
    sh.slot = sh.z + size_t(ld) * ncols;
    sh.tot = sh.slot + 2 * kVec;
    sh.upd = sh.tot + kVec;
    sh.dir = sh.upd + kMaxRank;
    sh.beta = sh.dir + kMaxRank;
    sh.taus = sh.beta + kMaxRank;
    sh.sgn = sh.taus + kMaxRank;
    sh.wv = sh.sgn + kMaxRank;
    sh.flag = reinterpret_cast<int*>(sh.wv + kMaxRank);
    double* z = sh.z;
    const int64_t r0 = int64_t(crank) * ld;
    const int nloc = static_cast<int>(lmax(0, lmin(ld, rows - r0)));
    int par = 0;
    QR_MARK(0);

    if (nparts > 0) {  // Z = sum of the sketch's split-K partials, in split order
        // all of an element's partial loads are issued before the (ordered) sum, two elements
        // per iteration: the L2 latency is paid once per pair instead of once per partial
        const int64_t pstride = int64_t(ncols) * rows;
#pragma unroll 2
        for (int t = tid; t < ld * ncols; t += kQrThreads) {
            const int i = t % ld, j = t / ld;
            double pv[16];
            const double* src = zin + int64_t(j) * rows + r0 + i;
#pragma unroll
            for (int sp = 0; sp < 16; ++sp) pv[sp] = (i < nloc && sp < nparts) ? src[sp * pstride] : 0.0;
            double v = 0.0;
#pragma unroll
            for (int sp = 0; sp < 16; ++sp)
                if (sp < nparts) v += pv[sp];
            z[t] = v;
        }
    } else {
#pragma unroll 4
        for (int t = tid; t < ld * ncols; t += kQrThreads) {
            const int i = t % ld, j = t / ld;
            z[t] = i < nloc ? zin[(r0 + i) + int64_t(j) * rows] : 0.0;
        }
    }
    if (tid < 2) sh.flag[tid] = 0;
    __syncthreads();

    int rank = 0;
    const int size = static_cast<int>(lmin(rows, ncols));
    bool fast_ok = false;
    double pmargin = 1.0;  // min over pivot steps of (top - second) / top of the remaining norms
    if (fast && rows >= ncols) {
        const int n = ncols;
        double* q = reinterpret_cast<double*>(sh.flag + 16);  // [n][ld]
        double* gp = q + size_t(ld) * n;                       // n x n partial Gram
        double* gs = gp + n * n;                               // n x n Gram / Schur complement
        double* r1 = gs + n * n;                               // n x n R of pass 1
        double* r2 = r1 + n * n;                               // n x n R of pass 2
        int* perm = reinterpret_cast<int*>(r2 + n * n);        // n: pivot order of pass 1
        int* perm2 = perm + kMaxRank;                          // n: (identity) of pass 2
        int* ctl = perm2 + kMaxRank;                           // scratch
        double* rinv1 = sh.upd;                                // 1 / R_kk (the Householder
                                                               // norms are not in use yet)
        __syncthreads();
        gram_partial_dmma(z, nloc, n, ld, gp);
        gram_reduce(cl, cs, gp, gs, n);
        QR_MARK(600);
        bool ok1;
        if (n <= 32) {  // registers, one warp; lraw (n x n) and the step diagonals in r2 / sh.dir
            if (warp == 0) {
                const bool ok = warp_pchol_reg(gs, n, r2, sh.dir, perm, sh.wv, sh.tot + kVec - 1);
                if (lane == 0) ctl[0] = ok ? 1 : 0;
            }
            __syncthreads();
            ok1 = ctl[0] != 0;
            if (ok1) {  // R[k][m] = sqrt(d_k) l^{(k)}_{perm[m]} (m > k), R_kk = sqrt(d_k)
                for (int e = tid; e < n * n; e += kQrThreads) {
                    const int k = e % n, m = e / n;
                    r1[e] = m < k ? 0.0 : (m == k ? sh.dir[k] : sh.dir[k] * r2[k * n + perm[m]]);
                }
                for (int k = tid; k < n; k += kQrThreads) rinv1[k] = 1.0 / sh.dir[k];
                __syncthreads();
            }
        } else {
            ok1 = cta_pchol(gs, n, true, r1, rinv1, perm, ctl, sh.tot + kVec - 1);
        }
        QR_MARK(601);
        if (ok1) {  // identical in every CTA (same reduced Gram, same arithmetic)
            // Q1 = Z_P R1^{-1}: row-parallel substitution for n <= 32, else with R1^{-1}
            // formed explicitly (parallel application)
            if (n <= 32 && rowpar == 2) {  // R1^{-1} by one warp, applied on the FP64 tensor cores
                if (warp == 0) warp_upper_inv(r1, rinv1, n, r2);
                __syncthreads();
                apply_dmma(z, q, ld, nloc, n, r2, perm);
            } else if (n <= 32 && rowpar) {
                rows_trsm_perm(z, q, ld, nloc, n, r1, rinv1, perm);
            } else {
                if (warp == 0) warp_tri_inv(r1, rinv1, n, r2);
                __syncthreads();
                if (rowpar == 2) apply_dmma(z, q, ld, nloc, n, r2, perm);  // n > 32: FP64 tensor cores as well
                else apply_upper(z, q, ld, nloc, n, r2, perm);
            }
            __syncthreads();
            QR_MARK(602);
            // second pass, to first order: Q1^T Q1 = I + E (E ~ eps cond^2 <= 1e-8), its
            // Cholesky factor is I + V with V = strict_upper(E) + diag(E) / 2, so
            // Q = Q1 (I + V)^{-1} = Q1 (I - V) + O(E^2) and R_kk = R1_kk (1 + V_kk)
            gram_partial_dmma(q, nloc, n, ld, gp);
            gram_reduce(cl, cs, gp, gs, n);
            QR_MARK(603);
            for (int e = tid; e < n * n; e += kQrThreads) {
                const int a = e % n, b = e / n;
                const double g = gs[e] - (a == b ? 1.0 : 0.0);
                r2[e] = a < b ? -g : (a == b ? 1.0 - 0.5 * g : 0.0);  // I - V
            }
            for (int k = tid; k < n; k += kQrThreads) perm2[k] = k;
            __syncthreads();
            QR_MARK(604);
            if (rowpar == 2) apply_dmma(q, z, ld, nloc, n, r2, nullptr);
            else if (n <= 32 && rowpar) rows_mul_upper(q, z, ld, nloc, n, r2);
            else apply_upper(q, z, ld, nloc, n, r2, perm2);
            for (int k = tid; k < n; k += kQrThreads) sh.beta[k] = r1[k + k * n] * (1.0 + 0.5 * (gs[k + k * n] - 1.0));
            __syncthreads();
            fast_ok = true;
            rank = n;
            pmargin = sh.tot[kVec - 1];
            QR_MARK(605);
        }
    }

    if (!fast_ok) {
    // initial column norms (m_qr.col(k).norm()): one reduction of col_j . col_j
    {
        double* m = sh.slot + par * kVec;
        const int sub = tid % kTpc, grp = tid / kTpc;
        for (int base = 0; base + warp * (32 / kTpc) < ncols; base += kQrThreads / kTpc) {
            const int j = base + grp;
            double s = 0.0;
            if (j < ncols) {
                const double* b = z + size_t(j) * ld;
                for (int i = sub; i < nloc; i += kTpc) s = fma(b[i], b[i], s);
            }
            s += __shfl_xor_sync(0xffffffffu, s, 8);
            s += __shfl_xor_sync(0xffffffffu, s, 4);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            if (sub == 0 && j < ncols) m[j] = s;
        }
        if (cs > 1) cl.sync();
        else __syncthreads();
        for (int j = tid; j < ncols; j += kQrThreads) {
            double s = 0.0;
            for (unsigned c = 0; c < cs; ++c) s += (cs > 1 ? cl.map_shared_rank(m, c) : m)[j];
            sh.upd[j] = sh.dir[j] = sqrt(s);
        }
        par ^= 1;
        __syncthreads();
    }

    const double norm_downdate_threshold = sqrt(DBL_EPSILON);
    QR_MARK(1);
    for (int k = 0; k < size; ++k) {
        QR_MARK(7 + 8 * k);
        // ---- pivot: first maximum of the updated norms over columns k.. (every warp)
        double bv = -1.0;
        int best = k;
        for (int j = k + lane; j < ncols; j += 32) {
            const double u = sh.upd[j];
            const bool take = u > bv;
            bv = take ? u : bv;
            best = take ? j : best;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, best, o);
            const bool take = ov > bv || (ov == bv && oi < best);
            bv = take ? ov : bv;
            best = take ? oi : best;
        }
        if (k + 1 < size) {  // the largest other candidate (pivot margin; every thread, same value)
            double sec = 0.0;
            for (int j = k + lane; j < ncols; j += 32)
                if (j != best) sec = fmax(sec, sh.upd[j]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sec = fmax(sec, __shfl_xor_sync(0xffffffffu, sec, o));
            if (bv > 0.0) pmargin = fmin(pmargin, (bv - sec) / bv);
        }
        const double upd_k = sh.upd[k], dir_k = sh.dir[k];
        QR_MARK(6 + 8 * k);
        if (best != k) {  // uniform: swap columns k and best
            for (int i = tid; i < nloc; i += kQrThreads) {
                const double t = z[i + k * ld];
                z[i + k * ld] = z[i + best * ld];
                z[i + best * ld] = t;
            }
            __syncthreads();
        }
        QR_MARK(8 + 8 * k);
        const int lk = static_cast<int>(k - r0);
        const bool owner = lk >= 0 && lk < nloc;
        const int i0 = static_cast<int>(lmax(0, k + 1 - r0));

        // ---- one reduction: tot[j-k] = col_k . col_j over rows > k ([0]: tail norm^2),
        //      tot[kMaxRank + j-k] = row k (contributed by the owner CTA only)
        reduce_dots(sh, cl, cs, par, z + size_t(k) * ld, ld, i0, nloc, k, ncols,
                    owner ? z + lk + size_t(k) * ld : nullptr, ld, ncols - k);
        QR_MARK(10 + 8 * k);

        // ---- Householder scalars (makeHouseholderInPlace), redundantly in every thread
        const double tail_sq = (rows - k == 1) ? 0.0 : sh.tot[0];
        const double c0 = sh.tot[kMaxRank];
        double tau, bta, rden = 0.0;  // essential v = tail * rden, rden = 1 / (c0 - beta)
        if (tail_sq <= DBL_MIN) {
            tau = 0.0;
            bta = c0;
        } else {
            bta = sqrt(c0 * c0 + tail_sq);
            if (c0 >= 0.0) bta = -bta;
            rden = 1.0 / (c0 - bta);
            tau = (bta - c0) / bta;
        }
        if (tid == 0) {
            sh.beta[k] = bta;
            sh.taus[k] = tau;
            sh.flag[(k + 1) & 1] = 0;
        }
        // ---- w_j and the norm downdate, one thread per trailing column (xGEQP3); position
        //      `best` inherits the norms of the column swapped out of position k
        for (int j = k + 1 + tid; j < ncols; j += kQrThreads) {
            const double rowk = sh.tot[kMaxRank + (j - k)];
            const double wj = tau != 0.0 ? rowk + sh.tot[j - k] * rden : 0.0;
            sh.wv[j] = wj;
            const double nrow = tau != 0.0 ? rowk - tau * wj : rowk;
            const double u = (j == best) ? upd_k : sh.upd[j];
            const double d = (j == best) ? dir_k : sh.dir[j];
            double nu = u;
            if (u != 0.0) {
                double temp = fabs(nrow) / u;
                temp = (1.0 + temp) * (1.0 - temp);
                temp = temp < 0.0 ? 0.0 : temp;
                const double ratio = u / d;
                if (temp * ratio * ratio <= norm_downdate_threshold) {
                    nu = -1.0;  // pending direct recomputation
                    atomicOr(&sh.flag[k & 1], 1);
                } else {
                    nu = u * sqrt(temp);
                }
            }
            sh.upd[j] = nu;
            sh.dir[j] = d;
        }
        // essential part of column k in place (rows > k), R_kk on the owner
        for (int i = i0 + tid; i < nloc; i += kQrThreads) z[i + k * ld] *= rden;
        if (owner && tid == 0) z[lk + k * ld] = bta;
        __syncthreads();
        QR_MARK(11 + 8 * k);
        // ---- trailing update col_j -= (tau v) w_j (rows > k); row k = row_k - tau w_j
        if (tau != 0.0) {
            for (int i = i0 + tid; i < nloc; i += kQrThreads) {
                const double tv = tau * z[i + k * ld];
                axpy_row(z + i, ld, k + 1, ncols, -tv, sh.wv);
            }
            if (owner)
                for (int j = k + 1 + tid; j < ncols; j += kQrThreads) z[lk + j * ld] -= tau * sh.wv[j];
        }
        __syncthreads();
        QR_MARK(12 + 8 * k);
        if (sh.flag[k & 1]) {  // identical decision on every CTA
            double* m = sh.slot + par * kVec;
            const int sub = tid % kTpc, grp = tid / kTpc;
            for (int base = k + 1; base + warp * (32 / kTpc) < ncols; base += kQrThreads / kTpc) {
                const int j = base + grp;
                double s = 0.0;
                if (j < ncols && sh.upd[j] < 0.0)
                    for (int i = i0 + sub; i < nloc; i += kTpc) s = fma(z[i + j * ld], z[i + j * ld], s);
                s += __shfl_xor_sync(0xffffffffu, s, 8);
                s += __shfl_xor_sync(0xffffffffu, s, 4);
                s += __shfl_xor_sync(0xffffffffu, s, 2);
                s += __shfl_xor_sync(0xffffffffu, s, 1);
                if (sub == 0 && j < ncols) m[j] = s;
            }
            if (cs > 1) cl.sync();
            else __syncthreads();
            for (int j = k + 1 + tid; j < ncols; j += kQrThreads)
                if (sh.upd[j] < 0.0) {
                    double s = 0.0;
                    for (unsigned c = 0; c < cs; ++c) s += (cs > 1 ? cl.map_shared_rank(m, c) : m)[j];
                    sh.upd[j] = sh.dir[j] = sqrt(s);
                }
            par ^= 1;
            __syncthreads();
        }
    }
    QR_MARK(2);

    // ---- rank cut (range_finder.hpp:24-26), redundantly
    {
        const double top = fabs(sh.beta[0]);
        while (rank < size && fabs(sh.beta[rank]) > 1e-12 * top) ++rank;
    }

    // ---- explicit Q(:, 0:rank) = H_0 ... H_{rank-1} [I; 0], in place
    for (int k = rank - 1; k >= 0; --k) {
        const double tau = sh.taus[k];
        const int lk = static_cast<int>(k - r0);
        const bool owner = lk >= 0 && lk < nloc;
        const int i0 = static_cast<int>(lmax(0, k + 1 - r0));
        if (k + 1 < rank) {
            reduce_dots(sh, cl, cs, par, z + size_t(k) * ld, ld, i0, nloc, k + 1, rank, nullptr, 0, 0);
            if (tau != 0.0)
                for (int i = i0 + tid; i < nloc; i += kQrThreads) {
                    const double tv = tau * z[i + k * ld];
                    axpy_row(z + i, ld, k + 1, rank, -tv, sh.tot - (k + 1));
                }
            if (owner)
                for (int j = k + 1 + tid; j < rank; j += kQrThreads) z[lk + j * ld] = -tau * sh.tot[j - k - 1];
            __syncthreads();
        }
        for (int i = tid; i < nloc; i += kQrThreads) {
            const int64_t gi = r0 + i;
            z[i + k * ld] = gi < k ? 0.0 : (gi == k ? 1.0 - tau : -tau * z[i + k * ld]);
        }
        __syncthreads();
    }
    }  // Householder path
    QR_MARK(3);

    // ---- sign fix: largest |entry| of each column positive (first maximum on ties); `plain`
    //      (the blocked tall path's reduced QR: the sign rule applies to its final product) skips it
    if (plain) {
        for (int j = tid; j < rank; j += kQrThreads) sh.sgn[j] = 1.0;
        if (margin_out && crank == 0 && tid == 0) {
            margin_out[0] = pmargin;
            margin_out[2] = fast_ok ? 0.0 : 1.0;
        }
        __syncthreads();
    } else if (rank > 0) {
        double* m = sh.slot + par * kVec;
        const int sub = tid % kTpc, grp = tid / kTpc;
        for (int base = 0; base + warp * (32 / kTpc) < rank; base += kQrThreads / kTpc) {
            const int j = base + grp;
            double bvv = -1.0, val = 0.0, pmax = 0.0, nmax = 0.0;
            int bi = 0x7fffffff;
            for (int i = sub; j < rank && i < nloc; i += kTpc) {
                const double x = z[i + j * ld];
                const bool take = fabs(x) > bvv;
                bvv = take ? fabs(x) : bvv;
                bi = take ? i : bi;
                val = take ? x : val;
                pmax = x > 0.0 ? fmax(pmax, x) : pmax;
                nmax = x < 0.0 ? fmax(nmax, -x) : nmax;
            }
#pragma unroll
            for (int o = kTpc / 2; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, bvv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                const double ov = __shfl_xor_sync(0xffffffffu, val, o);
                const bool take = ob > bvv || (ob == bvv && oi < bi);
                bvv = take ? ob : bvv;
                bi = take ? oi : bi;
                val = take ? ov : val;
                pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
                nmax = fmax(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
            }
            if (sub == 0 && j < rank) {
                m[2 * j] = bvv;
                m[2 * j + 1] = val;
                sh.upd[j] = pmax;  // (the norms are no longer in use) read remotely below
                sh.dir[j] = nmax;
            }
        }
        if (cs > 1) cl.sync();
        else __syncthreads();
        for (int j = tid; j < rank; j += kQrThreads) {
            double bvv = -1.0, val = 0.0;
            for (unsigned c0 = 0; c0 < cs; c0 += 8) {
                double tb[8], tv[8];
#pragma unroll
                for (unsigned c = 0; c < 8; ++c) {  // remote loads first, then the ordered scan
                    const double* ps = c0 + c < cs ? (cs > 1 ? cl.map_shared_rank(m, c0 + c) : m) : nullptr;
                    tb[c] = ps ? ps[2 * j] : -2.0;
                    tv[c] = ps ? ps[2 * j + 1] : 0.0;
                }
#pragma unroll
                for (unsigned c = 0; c < 8; ++c) {  // CTAs hold increasing rows: strict > keeps the first
                    const bool take = tb[c] > bvv;
                    bvv = take ? tb[c] : bvv;
                    val = take ? tv[c] : val;
                }
            }
            sh.sgn[j] = val < 0.0 ? -1.0 : 1.0;
            if (margin_out && crank == 0) {  // sign margin of column j: (max |u_i| of the winning sign - max of the other) / max
                double pm = 0.0, nm = 0.0;
                for (unsigned c = 0; c < cs; ++c) {
                    pm = fmax(pm, (cs > 1 ? cl.map_shared_rank(sh.upd, c) : sh.upd)[j]);
                    nm = fmax(nm, (cs > 1 ? cl.map_shared_rank(sh.dir, c) : sh.dir)[j]);
                }
                const double top = fmax(pm, nm);
                sh.wv[j] = top > 0.0 ? fabs(pm - nm) / top : 0.0;
            }
        }
        par ^= 1;
        __syncthreads();
        if (margin_out && crank == 0 && tid == 0) {
            double smin = 1.0;
            for (int j = 0; j < rank; ++j) smin = fmin(smin, sh.wv[j]);
            margin_out[0] = pmargin;
            margin_out[1] = smin;
            margin_out[2] = fast_ok ? 0.0 : 1.0;  // 0: pivoted CholeskyQR2, 1: Householder
        }
    }
    QR_MARK(4);

    // ---- outputs
    for (int j = 0; j < ucap; ++j)
        for (int i = tid; i < nloc; i += kQrThreads)
            uout[(r0 + i) + int64_t(j) * rows] = j < rank ? sh.sgn[j] * z[i + j * ld] : 0.0;
    if (upout) {
        const int stride = (rank + 3) / 4 * 4;
        for (int t = tid; t < nloc * stride; t += kQrThreads) {  // < 16 * 128 * 64: 32-bit indices
            const int i = t / stride, j = t - (t / stride) * stride;
            const double v = j < rank ? sh.sgn[j] * z[i + j * ld] : 0.0;
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
    QR_MARK(5);
    if (cs > 1) cl.sync();  // keep every CTA's shared memory alive until all DSMEM reads are done
}

// ---------------------------------------------------------------------------------------
// Blocked path for sketches taller than one cluster's shared memory (rows > qr_max_rows):
// a TSQR reduction in front of the cluster QR. Column pivoting only looks at column norms of
// trailing submatrices, which an orthogonal transform from the left leaves unchanged: with
// Z = Q0 S (unpivoted Householder QR of every row block, S = the stacked n x n R factors),
// ColPivHouseholderQR(Z) = Q0 ColPivHouseholderQR(S) — the same pivots, |R_kk| and rank cut
// (range_finder.hpp:18-29) — and the sign rule (tucker.hpp:39-45) is applied to the product.
//   level l:   tall_block_qr_kernel   one CTA per row block: R_b into the stack, explicit Q_b
//   last:      qr_colpiv_cluster_kernel (plain) on the stack (repeated levels until it fits)
//   back:      tall_apply_kernel      W_l[block b] = Q_b W_{l+1}[b n .. (b + 1) n)
//   finish:    tall_sign_partial_kernel / tall_finish_kernel: sign rule, margins, U + packed copy
// ---------------------------------------------------------------------------------------
constexpr int kTallThreads = 256;
constexpr int kTallMaxBlockRows = 320;  // 320 x 64 doubles = 160 KB of shared memory

// Unpivoted Householder QR (Eigen's makeHouseholderInPlace convention, as the cluster kernel)
// of rows [lo_b, hi_b) of zin, balanced blocks b = blockIdx.x; every block has >= n rows.
__global__ void __launch_bounds__(kTallThreads, 1)
    tall_block_qr_kernel(const double* __restrict__ zin, int64_t rows, int n, int nb, double* __restrict__ qout,
                         double* __restrict__ stack) {
    extern __shared__ __align__(16) double tsm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int kWarps = kTallThreads / 32;
    const int b = blockIdx.x;
    const int64_t lo = rows * b / nb, hi = rows * (b + 1) / nb;
    const int m = static_cast<int>(hi - lo);
    const int ld = m | 1;  // odd leading dimension: column-strided accesses spread over the banks
    double* z = tsm;                       // [n][ld]
    double* taus = z + size_t(ld) * n;     // [n]
    double* betas = taus + kMaxRank;       // [n]
    for (int t = tid; t < m * n; t += kTallThreads) {
        const int i = t % m, j = t / m;
        z[i + size_t(j) * ld] = zin[(lo + i) + int64_t(j) * rows];
    }
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        // scalars of H_k, redundantly per warp (same order everywhere: identical values)
        const double* ck = z + size_t(k) * ld;
        double ts = 0.0;
        for (int i = k + 1 + lane; i < m; i += 32) ts = fma(ck[i], ck[i], ts);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ts += __shfl_xor_sync(0xffffffffu, ts, o);
        const double c0 = ck[k];
        double tau, bta, rden = 0.0;
        if (ts <= DBL_MIN) {
            tau = 0.0;
            bta = c0;
        } else {
            bta = sqrt(c0 * c0 + ts);
            if (c0 >= 0.0) bta = -bta;
            rden = 1.0 / (c0 - bta);
            tau = (bta - c0) / bta;
        }
        if (tau != 0.0) {
            for (int j = k + 1 + warp; j < n; j += kWarps) {  // a warp owns its columns for the step
                double* cj = z + size_t(j) * ld;
                double w = 0.0;
                for (int i = k + 1 + lane; i < m; i += 32) w = fma(ck[i], cj[i], w);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
                w = cj[k] + w * rden;
                const double tw = tau * w;
                for (int i = k + 1 + lane; i < m; i += 32) cj[i] = fma(-tw * rden, ck[i], cj[i]);
                __syncwarp();
                if (lane == 0) cj[k] -= tw;
            }
        }
        __syncthreads();
        // column k is final: essential part scaled in place by one warp (no one reads it again
        // before the Q accumulation), R_kk = beta
        if (warp == k % kWarps) {
            double* wk = z + size_t(k) * ld;
            for (int i = k + 1 + lane; i < m; i += 32) wk[i] *= rden;
            if (lane == 0) {
                taus[k] = tau;
                betas[k] = bta;
            }
        }
    }
    __syncthreads();
    // R_b (upper triangular, diagonal = beta) into rows [b n, (b + 1) n) of the stack
    const int64_t sld = int64_t(nb) * n;
    for (int t = tid; t < n * n; t += kTallThreads) {
        const int i = t % n, j = t / n;
        stack[(int64_t(b) * n + i) + j * sld] = i < j ? z[i + size_t(j) * ld] : (i == j ? betas[i] : 0.0);
    }
    __syncthreads();
    // explicit Q_b = H_0 ... H_{n-1} [I; 0] in place, backward
    for (int k = n - 1; k >= 0; --k) {
        const double tau = taus[k];
        double* vk = z + size_t(k) * ld;
        for (int j = k + 1 + warp; j < n; j += kWarps) {
            double* cj = z + size_t(j) * ld;
            double d = 0.0;
            for (int i = k + 1 + lane; i < m; i += 32) d = fma(vk[i], cj[i], d);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            const double td = tau * d;
            for (int i = k + 1 + lane; i < m; i += 32) cj[i] = fma(-td, vk[i], cj[i]);
            if (lane == 0) cj[k] = -td;
        }
        __syncthreads();
        for (int i = tid; i < m; i += kTallThreads) vk[i] = i < k ? 0.0 : (i == k ? 1.0 - tau : -tau * vk[i]);
        __syncthreads();
    }
    for (int t = tid; t < m * n; t += kTallThreads) {
        const int i = t % m, j = t / m;
        qout[(lo + i) + int64_t(j) * rows] = z[i + size_t(j) * ld];
    }
}

// wout[rows of block b, 0:n) = q[rows of block b, 0:n) win[b n .. (b + 1) n, 0:n)  (balanced
// blocks as above; q, wout: ld = rows; win: ld = nb n). grid (nb, row tiles of 128).
__global__ void __launch_bounds__(128)
    tall_apply_kernel(const double* __restrict__ q, int64_t rows, int n, int nb, const double* __restrict__ win,
                      double* __restrict__ wout) {
    extern __shared__ __align__(16) double apsm[];
    double* ws = apsm;           // [n][n]
    double* qs = ws + n * n;     // [n][128]
    const int b = blockIdx.x;
    const int64_t lo = rows * b / nb, hi = rows * (b + 1) / nb;
    const int64_t r0 = lo + int64_t(blockIdx.y) * 128;
    if (r0 >= hi) return;
    const int nr = static_cast<int>(lmin(128, hi - r0));
    const int64_t wld = int64_t(nb) * n;
    for (int t = threadIdx.x; t < n * n; t += 128) ws[t] = win[(int64_t(b) * n + t % n) + (t / n) * wld];
    for (int t = threadIdx.x; t < n * 128; t += 128) {
        const int i = t & 127, k = t >> 7;
        qs[t] = i < nr ? q[(r0 + i) + int64_t(k) * rows] : 0.0;
    }
    __syncthreads();
    const int i = threadIdx.x;
    if (i >= nr) return;
    for (int j = 0; j < n; ++j) {
        const double* wj = ws + j * n;
        double a0 = 0.0, a1 = 0.0;
        int k = 0;
        for (; k + 2 <= n; k += 2) {
            a0 = fma(qs[i + k * 128], wj[k], a0);
            a1 = fma(qs[i + (k + 1) * 128], wj[k + 1], a1);
        }
        if (k < n) a0 = fma(qs[i + k * 128], wj[k], a0);
        wout[(r0 + i) + int64_t(j) * rows] = a0 + a1;
    }
}

constexpr int kSignChunk = 2048;  // rows per CTA of the sign scans

// part[(c n + j) 4 + {0, 1, 2, 3}] = over rows of chunk c of column j: first largest |w|, its
// value, largest positive entry, largest -negative entry
__global__ void __launch_bounds__(256)
    tall_sign_partial_kernel(const double* __restrict__ w, int64_t rows, int n, double* __restrict__ part) {
    const int c = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t lo = int64_t(c) * kSignChunk, hi = lmin(rows, lo + kSignChunk);
    for (int j = warp; j < n; j += 8) {
        const double* col = w + int64_t(j) * rows;
        double bv = -1.0, val = 0.0, pmax = 0.0, nmax = 0.0;
        int64_t bi = INT64_MAX;
        for (int64_t i = lo + lane; i < hi; i += 32) {
            const double x = col[i];
            const bool take = fabs(x) > bv;
            bv = take ? fabs(x) : bv;
            bi = take ? i : bi;
            val = take ? x : val;
            pmax = x > 0.0 ? fmax(pmax, x) : pmax;
            nmax = x < 0.0 ? fmax(nmax, -x) : nmax;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, bv, o);
            const long long oi = __shfl_xor_sync(0xffffffffu, static_cast<long long>(bi), o);
            const double ov = __shfl_xor_sync(0xffffffffu, val, o);
            const bool take = ob > bv || (ob == bv && oi < bi);
            bv = take ? ob : bv;
            bi = take ? oi : bi;
            val = take ? ov : val;
            pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
            nmax = fmax(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
        }
        if (lane == 0) {
            double* o = part + (size_t(c) * n + j) * 4;
            o[0] = bv;
            o[1] = val;
            o[2] = pmax;
            o[3] = nmax;
        }
    }
}

// sign rule from the chunk partials (scanned in row order: strict > keeps the first maximum),
// then this CTA's rows of U (rows x ucap, columns >= rank zero) and of the packed copy
__global__ void __launch_bounds__(256)
    tall_finish_kernel(const double* __restrict__ w, int64_t rows, int n, int nchunks, const double* __restrict__ part,
                       const int* __restrict__ rank_dev, double* __restrict__ uout, int ucap, void* upout, int up_dtype,
                       double* margin_out) {
    __shared__ double sgn[kMaxRank], smar[kMaxRank];
    const int rank = *rank_dev;
    for (int j = threadIdx.x; j < n; j += 256) {
        double bv = -1.0, val = 0.0, pm = 0.0, nm = 0.0;
        for (int c = 0; c < nchunks; ++c) {
            const double* o = part + (size_t(c) * n + j) * 4;
            const bool take = o[0] > bv;
            bv = take ? o[0] : bv;
            val = take ? o[1] : val;
            pm = fmax(pm, o[2]);
            nm = fmax(nm, o[3]);
        }
        sgn[j] = val < 0.0 ? -1.0 : 1.0;
        const double top = fmax(pm, nm);
        smar[j] = top > 0.0 ? fabs(pm - nm) / top : 0.0;
    }
    __syncthreads();
    if (margin_out && blockIdx.x == 0 && threadIdx.x == 0 && rank > 0) {
        double smin = 1.0;
        for (int j = 0; j < rank; ++j) smin = fmin(smin, smar[j]);
        margin_out[1] = smin;
    }
    const int64_t lo = int64_t(blockIdx.x) * kSignChunk, hi = lmin(rows, lo + kSignChunk);
    const int nr = static_cast<int>(hi - lo);
    for (int j = 0; j < ucap; ++j)
        for (int i = threadIdx.x; i < nr; i += 256)
            uout[(lo + i) + int64_t(j) * rows] = (j < rank && j < n) ? sgn[j] * w[(lo + i) + int64_t(j) * rows] : 0.0;
    if (upout) {
        const int stride = (rank + 3) / 4 * 4;
        for (int t = threadIdx.x; t < nr * stride; t += 256) {
            const int i = t / stride, j = t - i * stride;
            const double v = j < rank ? sgn[j] * w[(lo + i) + int64_t(j) * rows] : 0.0;
            const int64_t o = (lo + i) * stride + j;
            if (up_dtype == kF32) static_cast<float*>(upout)[o] = static_cast<float>(v);
            else static_cast<double*>(upout)[o] = v;
        }
    }
}

int pick_cluster(int64_t rows, int ncols, int* ld_out, size_t* smem_out) {
    static const int min_cs = [] {
        const char* e = std::getenv("TENKIT_QR_MIN_CLUSTER");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    // The QR is latency-bound per Householder step; spreading the rows so that each CTA holds
    // <= 128 of them cuts the per-step reduction and update work (1000 x 30: 8 CTAs, ~30%
    // faster than the 2 the shared memory alone needs; measured with tools/qr_trace.cu).
    static const int kTargetRows = [] {
        const char* e = std::getenv("TENKIT_QR_TARGET_ROWS");
        return e ? std::max(16, std::atoi(e)) : 128;
    }();
    for (int cs = min_cs; cs <= 16; cs *= 2) {
        const int ld = static_cast<int>((rows + cs - 1) / cs);
        const size_t smem = size_t(ld) * ncols * sizeof(double) + kQrFixedSmem;
        if (smem <= kQrSmemCap && (ld <= kTargetRows || cs == 16)) {
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

namespace {

void launch_cluster_qr(const double* z, int64_t rows, int ncols, double* u, int ucap, void* up, int up_dtype,
                       int* rank_dev, double* diag, cudaStream_t s, int nparts, double* margins, int plain) {
    int ld = 0;
    size_t smem = 0;
    const int cs = pick_cluster(rows, ncols, &ld, &smem);
    require(cs > 0, "orthonormal_basis: sketch too large for the cluster QR");
    // fast path scratch: Q of pass 1 (ld x ncols) + 4 n x n + 4 kMaxRank ints
    const size_t fast_extra = (size_t(ld) * ncols + 4 * size_t(ncols) * ncols) * sizeof(double) + 4 * kMaxRank * sizeof(int);
    static const bool no_fast = [] {
        const char* e = std::getenv("TENKIT_QR_NO_FAST");
        return e && e[0] == '1';
    }();
    const int fast = (!no_fast && smem + fast_extra <= kQrSmemCap) ? 1 : 0;
    if (fast) smem += fast_extra;
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
    // A/B knob: 2 (default) = R^-1 by one warp + FP64-tensor-core applications, 1 = row-parallel
    // substitution / multiply, 0 = R^-1 by one warp + gathered FFMA application
    static const int rowpar = [] {
        const char* e = std::getenv("TENKIT_QR_ROWPAR");
        return e ? std::atoi(e) : 2;
    }();
    TK_MAXSMEM((qr_colpiv_cluster_kernel));
    TK_CUDA(cudaLaunchKernelEx(&cfg, qr_colpiv_cluster_kernel, z, rows, ncols, ld, u, ucap, up, up_dtype, rank_dev,
                               diag, fast, rowpar, nparts, margins, plain));
}

// Levels of the blocked path: level l factors a rows[l] x n matrix in nb[l] balanced row blocks
// (each >= n and <= kTallMaxBlockRows rows) into Q_l (rows[l] x n) and a stack of nb[l] n rows;
// the last stack fits the cluster QR.
struct TallPlan {
    std::vector<int64_t> rows;  // rows[0] = the sketch, rows[l + 1] = nb[l] * n; back() = the cluster QR's input
    std::vector<int> nb;
    int64_t work_elems = 0;
};

// Largest sketch the cluster QR takes directly. Above the shared-memory capacity the blocked
// path is the only one; A/B knob TENKIT_QR_TALL_ABOVE=rows sends shorter sketches there too.
int64_t cluster_rows_limit(int n) {
    static const int64_t knob = [] {
        const char* e = std::getenv("TENKIT_QR_TALL_ABOVE");
        return e ? std::max<int64_t>(0, std::atoll(e)) : int64_t(0);  // 0: off
    }();
    const int64_t cap = qr_max_rows(n);
    return knob > 0 ? std::min(cap, std::max<int64_t>(knob, 4 * n)) : cap;
}

TallPlan tall_plan(int64_t rows, int n) {
    TallPlan p;
    p.rows.push_back(rows);
    const int64_t cap = cluster_rows_limit(n);
    const int br = std::max(2 * n, std::min<int>(kTallMaxBlockRows, static_cast<int>((160 * 1024) / (sizeof(double) * n))));
    while (p.rows.back() > cap) {
        const int64_t r = p.rows.back();
        const int64_t nb = (r + br - 1) / br;
        require(nb < (int64_t(1) << 24), "orthonormal_basis: sketch too tall");
        p.nb.push_back(static_cast<int>(nb));
        p.rows.push_back(nb * n);
    }
    // Q_l and W_l per level, the stacks (W of the last level = the cluster QR's output), sign partials
    for (size_t l = 0; l < p.nb.size(); ++l) p.work_elems += 2 * p.rows[l] * n + p.rows[l + 1] * n;
    p.work_elems += p.rows.back() * n;
    p.work_elems += ((rows + kSignChunk - 1) / kSignChunk) * n * 4;
    return p;
}

}  // namespace

int64_t qr_work_elems(int64_t rows, int ncols) {
    if (ncols < 1 || ncols > kMaxRank || rows <= cluster_rows_limit(ncols)) return 0;
    return tall_plan(rows, ncols).work_elems;
}

int launch_orthonormal_basis(const double* z, int64_t rows, int ncols, double* u, int ucap, void* up, int up_dtype,
                             int* rank_dev, double* diag, cudaStream_t s, int nparts, double* margins, double* work) {
    require(rows >= 1, "orthonormal_basis: empty input");
    require(ncols >= 1 && ncols <= kMaxRank, "orthonormal_basis: column count must be in [1, 64]");
    if (rows <= cluster_rows_limit(ncols)) {
        launch_cluster_qr(z, rows, ncols, u, ucap, up, up_dtype, rank_dev, diag, s, nparts, margins, 0);
        return 1;
    }
    require(work != nullptr && nparts == 0, "orthonormal_basis: sketch too large for the cluster QR");
    const int n = ncols;
    const TallPlan p = tall_plan(rows, n);
    const int L = static_cast<int>(p.nb.size());
    std::vector<double*> q(L), w(L + 1), st(L + 1);
    double* cur = work;
    for (int l = 0; l < L; ++l) {
        q[l] = cur, cur += p.rows[l] * n;
        w[l] = cur, cur += p.rows[l] * n;
        st[l + 1] = cur, cur += p.rows[l + 1] * n;
    }
    w[L] = cur, cur += p.rows[L] * n;
    double* part = cur;
    static bool attr = false;
    if (!attr) {
        TK_CUDA(cudaFuncSetAttribute(tall_block_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        TK_CUDA(cudaFuncSetAttribute(tall_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        attr = true;
    }
    int launches = 0;
    const double* src = z;
    for (int l = 0; l < L; ++l) {
        const int64_t mb = (p.rows[l] + p.nb[l] - 1) / p.nb[l] + 1;  // largest balanced block (+1: odd ld)
        const size_t smem = (size_t(mb | 1) * n + 2 * kMaxRank) * sizeof(double);
        tall_block_qr_kernel<<<p.nb[l], kTallThreads, smem, s>>>(src, p.rows[l], n, p.nb[l], q[l], st[l + 1]);
        TK_CUDA(cudaGetLastError());
        src = st[l + 1];
        ++launches;
    }
    // the reduced matrix: pivots, rank cut, |R_kk| diagnostics, pivot margin — no sign rule
    launch_cluster_qr(st[L], p.rows[L], n, w[L], n, nullptr, kF64, rank_dev, diag, s, 0, margins, 1);
    ++launches;
    for (int l = L - 1; l >= 0; --l) {
        const int64_t mb = (p.rows[l] + p.nb[l] - 1) / p.nb[l] + 1;
        const dim3 grid(p.nb[l], static_cast<unsigned>((mb + 127) / 128));
        const size_t smem = (size_t(n) * n + size_t(n) * 128) * sizeof(double);
        tall_apply_kernel<<<grid, 128, smem, s>>>(q[l], p.rows[l], n, p.nb[l], w[l + 1], w[l]);
        TK_CUDA(cudaGetLastError());
        ++launches;
    }
    const int nchunks = static_cast<int>((rows + kSignChunk - 1) / kSignChunk);
    tall_sign_partial_kernel<<<nchunks, 256, 0, s>>>(w[0], rows, n, part);
    TK_CUDA(cudaGetLastError());
    tall_finish_kernel<<<nchunks, 256, 0, s>>>(w[0], rows, n, nchunks, part, rank_dev, u, ucap, up, up_dtype, margins);
    TK_CUDA(cudaGetLastError());
    return launches + 2;
}

}  // namespace tkb
