// tenkit_oracle.cpp — TEST INFRASTRUCTURE ONLY (the parity checker / CPU baseline).
//
// A CPU restatement, in plain C++17 without Eigen, of the reference `tenkit`
// randomized-Tucker hot path (arXiv 1412.1885; /root/reference/proj/include/tenkit).
// The reference cannot be compiled in this image (Eigen3 and Catch2 are absent), so
// this file restates its algorithms function by function; each function cites the
// reference file:line it follows. Eigen's ColPivHouseholderQR / makeHouseholder /
// LDLT are restated from their published algorithms (Eigen >= 3.3, version unpinned
// by the reference: no lockfile, no vendored copy).
//
// Parity pin: the restatement is checked against every known-answer test and
// property test the reference's own suite holds for this path (tests/test_oracle_*.py
// mirror test_tensor.cpp, test_random.cpp, test_range_finder.cpp, test_tucker.cpp,
// test_ffcp.cpp), and its pivoted QR against LAPACK dgeqp3 (scipy) — the algorithm
// Eigen's ColPivHouseholderQR restates. The reference holds no golden vectors for
// the sketch/QR/core.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference leg may
// load this library. The product (paper_1412_1885_b200/) never links or calls it.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <dlfcn.h>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace tko {

using Index = int64_t;

// ---------------------------------------------------------------------------
// Error plumbing: the reference throws std::invalid_argument("tenkit: ...")
// (tensor.hpp:20-22); the C API maps it to a return code + message.
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;

inline void require(bool cond, const std::string& msg) {
    if (!cond) throw std::invalid_argument("tenkit: " + msg);
}

// ---------------------------------------------------------------------------
// Dense column-major matrix and N-way tensor (tensor.hpp:32-97, :15)
// ---------------------------------------------------------------------------
struct Mat {
    Index rows = 0, cols = 0;
    std::vector<double> d;
    Mat() = default;
    Mat(Index r, Index c) : rows(r), cols(c), d(static_cast<size_t>(r * c), 0.0) {}
    double& operator()(Index i, Index j) { return d[static_cast<size_t>(i + j * rows)]; }
    double operator()(Index i, Index j) const { return d[static_cast<size_t>(i + j * rows)]; }
    double* data() { return d.data(); }
    const double* data() const { return d.data(); }
    double* col(Index j) { return d.data() + j * rows; }
    const double* col(Index j) const { return d.data() + j * rows; }
};

inline Mat transpose(const Mat& m) {
    Mat t(m.cols, m.rows);
    for (Index j = 0; j < m.cols; ++j)
        for (Index i = 0; i < m.rows; ++i) t(j, i) = m(i, j);
    return t;
}

struct Tensor {
    std::vector<Index> shape;
    std::vector<double> d;
    Tensor() = default;
    explicit Tensor(std::vector<Index> s) : shape(std::move(s)) {
        require(!shape.empty(), "tensor order must be at least 1");
        Index n = 1;
        for (Index x : shape) {
            require(x >= 1, "tensor dimensions must be positive");
            n *= x;
        }
        d.assign(static_cast<size_t>(n), 0.0);
    }
    Index order() const { return static_cast<Index>(shape.size()); }
    Index size() const { return static_cast<Index>(d.size()); }
    Index dim(Index n) const { return shape.at(static_cast<size_t>(n)); }
    double* data() { return d.data(); }
    const double* data() const { return d.data(); }
};

// SlabDims (tensor.hpp:103-116)
struct Slab {
    Index before, mode, after;
};
inline Slab slab_dims(const std::vector<Index>& shape, Index mode) {
    require(mode >= 0 && mode < static_cast<Index>(shape.size()), "mode index out of range");
    Slab s{1, shape[static_cast<size_t>(mode)], 1};
    for (Index k = 0; k < mode; ++k) s.before *= shape[static_cast<size_t>(k)];
    for (Index k = mode + 1; k < static_cast<Index>(shape.size()); ++k)
        s.after *= shape[static_cast<size_t>(k)];
    return s;
}

// ---------------------------------------------------------------------------
// GEMM: C = alpha * op(A) * op(B) + beta * C, column-major. Uses OpenBLAS (ILP64,
// shipped inside numpy.libs) when tko_blas_init found it, else a portable loop.
// This stands in for Eigen's GEMM at tensor.hpp:161,167,173,201,206.
// ---------------------------------------------------------------------------
using dgemm_fn = void (*)(const char*, const char*, const int64_t*, const int64_t*,
                          const int64_t*, const double*, const double*, const int64_t*,
                          const double*, const int64_t*, const double*, double*,
                          const int64_t*, size_t, size_t);
using setthreads_fn = void (*)(int);
static dgemm_fn g_dgemm = nullptr;
static int g_threads = 1;  // host threads of the oracle (tko_blas_init)
static setthreads_fn g_setthreads = nullptr;

static void gemm(bool ta, bool tb, Index m, Index n, Index k, double alpha, const double* a,
                 Index lda, const double* b, Index ldb, double beta, double* c, Index ldc) {
    if (m == 0 || n == 0) return;
    if (g_dgemm) {
        const char sa = ta ? 'T' : 'N', sb = tb ? 'T' : 'N';
        g_dgemm(&sa, &sb, &m, &n, &k, &alpha, a, &lda, b, &ldb, &beta, c, &ldc, 1, 1);
        return;
    }
    // portable fallback: fixed-order loops (deterministic)
    auto A = [&](Index i, Index p) { return ta ? a[p + i * lda] : a[i + p * lda]; };
    auto B = [&](Index p, Index j) { return tb ? b[j + p * ldb] : b[p + j * ldb]; };
    for (Index j = 0; j < n; ++j) {
        double* cj = c + j * ldc;
        if (beta == 0.0) std::fill(cj, cj + m, 0.0);
        else if (beta != 1.0) for (Index i = 0; i < m; ++i) cj[i] *= beta;
        for (Index p = 0; p < k; ++p) {
            const double bpj = alpha * B(p, j);
            if (bpj == 0.0) continue;
            if (!ta) {
                const double* ap = a + p * lda;
                for (Index i = 0; i < m; ++i) cj[i] += ap[i] * bpj;
            } else {
                for (Index i = 0; i < m; ++i) cj[i] += A(i, p) * bpj;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Counter RNG (random.hpp:12-138) — bit-exact restatement.
// ---------------------------------------------------------------------------
inline uint64_t mix64(uint64_t x) {  // random.hpp:12-18
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
inline uint64_t hash_combine(uint64_t a, uint64_t b) {  // random.hpp:20-22
    return mix64(a ^ (mix64(b) + 0x9E3779B97F4A7C15ull + (a << 6) + (a >> 2)));
}
struct Seed {  // SeedSpec, random.hpp:29-44
    uint64_t root = 0, stream = 0;
    Seed derived(uint64_t t) const { return {root, hash_combine(stream, t)}; }
    Seed derived(uint64_t a, uint64_t b) const { return derived(a).derived(b); }
    uint64_t key() const { return hash_combine(mix64(root), stream); }
};
inline double counter_unit(uint64_t key, uint64_t i) {  // random.hpp:48-56
    return static_cast<double>((mix64(key + i * 0x9E3779B97F4A7C15ull) >> 11) + 1) * 0x1.0p-53;
}
inline double normal_at_key(uint64_t key, uint64_t index) {  // random.hpp:63-71
    const uint64_t pair = index >> 1;
    const double u1 = counter_unit(key, 2 * pair);
    const double u2 = counter_unit(key, 2 * pair + 1);
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double angle = 6.283185307179586476925287 * u2;
    return (index & 1u) ? r * std::sin(angle) : r * std::cos(angle);
}
inline void gaussian_fill_range(double* p, uint64_t lo, uint64_t hi, uint64_t n, uint64_t key) {
    for (uint64_t i = lo; i < hi; i += 2) {  // lo even: Box-Muller pairs (2k, 2k+1)
        const double u1 = counter_unit(key, i);
        const double u2 = counter_unit(key, i + 1);
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double angle = 6.283185307179586476925287 * u2;
        p[i] = r * std::cos(angle);
        if (i + 1 < n) p[i + 1] = r * std::sin(angle);
    }
}
// random.hpp:85-100,124-138: every entry a pure function of (key, index), so the fill is split
// over the oracle's host threads at even boundaries (values independent of the split)
inline void gaussian_fill(double* p, uint64_t n, uint64_t key) {
    const uint64_t nt = std::max<uint64_t>(1, std::min<uint64_t>(static_cast<uint64_t>(g_threads), n >> 20));
    if (nt == 1) return gaussian_fill_range(p, 0, n, n, key);
    std::vector<std::thread> pool;
    for (uint64_t w = 0; w < nt; ++w) {
        const uint64_t lo = (n * w / nt) & ~uint64_t(1), hi = w + 1 == nt ? n : (n * (w + 1) / nt) & ~uint64_t(1);
        pool.emplace_back([=] { gaussian_fill_range(p, lo, hi, n, key); });
    }
    for (auto& th : pool) th.join();
}
inline Mat gaussian_matrix(Index rows, Index cols, const Seed& s) {  // random.hpp:85-100
    require(rows >= 1 && cols >= 1, "gaussian_matrix: dimensions must be positive");
    Mat m(rows, cols);
    gaussian_fill(m.data(), static_cast<uint64_t>(rows * cols), s.key());
    return m;
}

// Seed tags (tucker.hpp:49-58, ffcp.hpp:49-51, bench.hpp:46-48)
inline Seed alg2_omega_seed(const Seed& s, Index n) { return s.derived(0x0A2u, static_cast<uint64_t>(n)); }
inline Seed alg3_init_seed(const Seed& s, Index n) { return s.derived(0x0A3u, static_cast<uint64_t>(n)); }
inline Seed alg3_omega_seed(const Seed& s, Index pass, Index n) {
    return s.derived(0x0B3u + static_cast<uint64_t>(pass), static_cast<uint64_t>(n));
}
inline Seed ffcp_init_seed(const Seed& s, Index n) { return s.derived(0x0FCu, static_cast<uint64_t>(n)); }
inline Seed gen_factor_seed(const Seed& s, Index n) { return s.derived(0x9E4u, static_cast<uint64_t>(n)); }

// ---------------------------------------------------------------------------
// Tensor kernels (tensor.hpp:123-209)
// ---------------------------------------------------------------------------

// unfold (tensor.hpp:123-133)
inline Mat unfold(const Tensor& t, Index mode) {
    const Slab s = slab_dims(t.shape, mode);
    Mat out(s.mode, s.before * s.after);
    for (Index q = 0; q < s.after; ++q)
        for (Index i = 0; i < s.mode; ++i)
            for (Index p = 0; p < s.before; ++p)
                out(i, q * s.before + p) = t.d[static_cast<size_t>(p + i * s.before + q * s.before * s.mode)];
    return out;
}

// ttm (tensor.hpp:151-176): unfold(out, n) = M * unfold(T, n)
inline Tensor ttm(const Tensor& t, const Mat& m, Index mode) {
    const Slab s = slab_dims(t.shape, mode);
    require(m.cols == s.mode, "ttm: matrix columns must match mode dimension");
    std::vector<Index> os = t.shape;
    os[static_cast<size_t>(mode)] = m.rows;
    Tensor out(os);
    if (mode == 0) {  // one GEMM (tensor.hpp:158-163)
        gemm(false, false, m.rows, s.after, s.mode, 1.0, m.data(), m.rows, t.data(), s.mode, 0.0,
             out.data(), m.rows);
        return out;
    }
    // trailing mode (after == 1, tensor.hpp:164-169) is the q-loop with one slab
    for (Index q = 0; q < s.after; ++q)  // slab loop (tensor.hpp:170-175)
        gemm(false, true, s.before, m.rows, s.mode, 1.0, t.data() + q * s.before * s.mode, s.before,
             m.data(), m.rows, 0.0, out.data() + q * s.before * m.rows, s.before);
    return out;
}

// ttm_all (tensor.hpp:181-192): ascending modes, skipping `skip`
inline Tensor ttm_all(const Tensor& t, const std::vector<Mat>& ms, Index skip, bool transpose_m) {
    require(static_cast<Index>(ms.size()) == t.order(), "ttm_all: one matrix per mode required");
    Tensor cur = t;
    for (Index n = 0; n < t.order(); ++n) {
        if (n == skip) continue;
        const Mat& m = ms[static_cast<size_t>(n)];
        cur = transpose_m ? ttm(cur, transpose(m), n) : ttm(cur, m, n);
    }
    return cur;
}

// unfold_times (tensor.hpp:195-209): unfold(T, n) * B without materialising
inline Mat unfold_times(const Tensor& t, Index mode, const Mat& b) {
    const Slab s = slab_dims(t.shape, mode);
    require(b.rows == s.before * s.after, "unfold_times: B rows must match unfolding width");
    Mat z(s.mode, b.cols);
    if (mode == 0) {
        gemm(false, false, s.mode, b.cols, s.after, 1.0, t.data(), s.mode, b.data(), b.rows, 0.0,
             z.data(), s.mode);
        return z;
    }
    for (Index q = 0; q < s.after; ++q)  // fixed-order slab accumulation (:204-207)
        gemm(true, false, s.mode, b.cols, s.before, 1.0, t.data() + q * s.before * s.mode, s.before,
             b.data() + q * s.before, b.rows, 1.0, z.data(), s.mode);
    return z;
}

inline double sq_norm(const double* p, Index n) {
    double s = 0.0;
    for (Index i = 0; i < n; ++i) s += p[i] * p[i];
    return s;
}

// fit (tensor.hpp:282-290)
inline double fit(const Tensor& y, const Tensor& yhat) {
    require(y.shape == yhat.shape, "fit: shape mismatch");
    const double ny = std::sqrt(sq_norm(y.data(), y.size()));
    require(ny > 0.0, "fit: reference tensor has zero norm");
    double r = 0.0;
    for (Index i = 0; i < y.size(); ++i) {
        const double e = y.d[static_cast<size_t>(i)] - yhat.d[static_cast<size_t>(i)];
        r += e * e;
    }
    return 1.0 - std::sqrt(r) / ny;
}

// ---------------------------------------------------------------------------
// Column-pivoted Householder QR — restatement of Eigen::ColPivHouseholderQR::
// computeInPlace (Householder via makeHouseholderInPlace, LAPACK-style norm
// downdating with recompute threshold sqrt(eps)) as used by orthonormal_basis
// (range_finder.hpp:18-29). Q columns come out in pivot order.
// ---------------------------------------------------------------------------
struct ColPivQR {
    Mat qr;                     // R above/on the diagonal, Householder essentials below
    std::vector<double> hcoef;  // tau_k
    std::vector<Index> perm;    // column transpositions
    std::vector<double> pivot_margin;  // diagnostics: relative gap between the top-2 norms at step k
};

inline ColPivQR colpiv_qr(const Mat& z) {
    ColPivQR f;
    f.qr = z;
    Mat& a = f.qr;
    const Index rows = a.rows, cols = a.cols, size = std::min(rows, cols);
    f.hcoef.assign(static_cast<size_t>(size), 0.0);
    f.perm.assign(static_cast<size_t>(cols), 0);
    f.pivot_margin.assign(static_cast<size_t>(size), 0.0);
    std::vector<double> upd(static_cast<size_t>(cols)), dir(static_cast<size_t>(cols));
    for (Index k = 0; k < cols; ++k) {
        dir[static_cast<size_t>(k)] = std::sqrt(sq_norm(a.col(k), rows));
        upd[static_cast<size_t>(k)] = dir[static_cast<size_t>(k)];
    }
    const double eps = std::numeric_limits<double>::epsilon();
    const double norm_downdate_threshold = std::sqrt(eps);
    const double tol = std::numeric_limits<double>::min();
    std::vector<double> tmp(static_cast<size_t>(cols));
    for (Index k = 0; k < size; ++k) {
        // biggest updated norm among columns k.. (first max on ties)
        Index best = k;
        for (Index j = k + 1; j < cols; ++j)
            if (upd[static_cast<size_t>(j)] > upd[static_cast<size_t>(best)]) best = j;
        {
            double second = 0.0;
            for (Index j = k; j < cols; ++j)
                if (j != best) second = std::max(second, upd[static_cast<size_t>(j)]);
            const double top = upd[static_cast<size_t>(best)];
            f.pivot_margin[static_cast<size_t>(k)] = top > 0 ? (top - second) / top : 0.0;
        }
        f.perm[static_cast<size_t>(k)] = best;
        if (best != k) {
            std::swap_ranges(a.col(k), a.col(k) + rows, a.col(best));
            std::swap(upd[static_cast<size_t>(k)], upd[static_cast<size_t>(best)]);
            std::swap(dir[static_cast<size_t>(k)], dir[static_cast<size_t>(best)]);
        }
        // makeHouseholderInPlace on x = a(k:rows, k)
        double* x = a.col(k) + k;
        const Index len = rows - k;
        const double tail_sq = len == 1 ? 0.0 : sq_norm(x + 1, len - 1);
        const double c0 = x[0];
        double tau, beta;
        if (tail_sq <= tol) {
            tau = 0.0;
            beta = c0;
            for (Index i = 1; i < len; ++i) x[i] = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail_sq);
            if (c0 >= 0.0) beta = -beta;
            const double denom = c0 - beta;
            for (Index i = 1; i < len; ++i) x[i] /= denom;
            tau = (beta - c0) / beta;
        }
        f.hcoef[static_cast<size_t>(k)] = tau;
        x[0] = beta;
        // applyHouseholderOnTheLeft to a(k:rows, k+1:cols)
        if (len == 1) {
            for (Index j = k + 1; j < cols; ++j) a(k, j) *= (1.0 - tau);
        } else if (tau != 0.0) {
            for (Index j = k + 1; j < cols; ++j) {
                const double* cj = a.col(j) + k;
                double t = 0.0;
                for (Index i = 1; i < len; ++i) t += x[i] * cj[i];
                tmp[static_cast<size_t>(j)] = t + cj[0];
            }
            for (Index j = k + 1; j < cols; ++j) {
                double* cj = a.col(j) + k;
                const double t = tmp[static_cast<size_t>(j)];
                cj[0] -= tau * t;
                for (Index i = 1; i < len; ++i) cj[i] -= tau * x[i] * t;
            }
        }
        // norm downdate (LAWN 176; LAPACK xGEQP3)
        for (Index j = k + 1; j < cols; ++j) {
            double& u = upd[static_cast<size_t>(j)];
            if (u != 0.0) {
                double temp = std::abs(a(k, j)) / u;
                temp = (1.0 + temp) * (1.0 - temp);
                temp = temp < 0.0 ? 0.0 : temp;
                const double ratio = u / dir[static_cast<size_t>(j)];
                const double temp2 = temp * ratio * ratio;
                if (temp2 <= norm_downdate_threshold) {
                    dir[static_cast<size_t>(j)] = std::sqrt(sq_norm(a.col(j) + k + 1, rows - k - 1));
                    u = dir[static_cast<size_t>(j)];
                } else {
                    u *= std::sqrt(temp);
                }
            }
        }
    }
    return f;
}

// Q(:, 0:ncols) = H_0 H_1 ... H_{size-1} [I; 0]
inline Mat householder_q(const ColPivQR& f, Index ncols) {
    const Index rows = f.qr.rows, size = static_cast<Index>(f.hcoef.size());
    Mat q(rows, ncols);
    for (Index j = 0; j < ncols; ++j) q(j, j) = 1.0;
    for (Index k = size - 1; k >= 0; --k) {
        const double tau = f.hcoef[static_cast<size_t>(k)];
        const Index len = rows - k;
        if (len == 1) {
            for (Index j = 0; j < ncols; ++j) q(k, j) *= (1.0 - tau);
            continue;
        }
        if (tau == 0.0) continue;
        const double* v = f.qr.col(k) + k;  // v[0] = 1 implicit
        for (Index j = 0; j < ncols; ++j) {
            double* cj = q.col(j) + k;
            double t = cj[0];
            for (Index i = 1; i < len; ++i) t += v[i] * cj[i];
            cj[0] -= tau * t;
            for (Index i = 1; i < len; ++i) cj[i] -= tau * v[i] * t;
        }
    }
    return q;
}

constexpr double kRankDeficiencyTol = 1e-12;  // range_finder.hpp:13

// orthonormal_basis (range_finder.hpp:18-29)
inline Mat orthonormal_basis(const Mat& z, ColPivQR* keep = nullptr) {
    require(z.rows >= 1, "orthonormal_basis: empty input");
    if (z.cols == 0) return Mat(z.rows, 0);
    ColPivQR f = colpiv_qr(z);
    const Index kmax = std::min(z.rows, z.cols);
    const double top = std::abs(f.qr(0, 0));
    Index rank = 0;
    while (rank < kmax && std::abs(f.qr(rank, rank)) > kRankDeficiencyTol * top) ++rank;
    Mat q = householder_q(f, rank);
    if (keep) *keep = std::move(f);
    return q;
}

// fix_column_signs (tucker.hpp:39-45)
inline void fix_column_signs(Mat& u) {
    for (Index j = 0; j < u.cols; ++j) {
        Index imax = 0;
        double best = -1.0;
        for (Index i = 0; i < u.rows; ++i)
            if (std::abs(u(i, j)) > best) {
                best = std::abs(u(i, j));
                imax = i;
            }
        if (u(imax, j) < 0)
            for (Index i = 0; i < u.rows; ++i) u(i, j) = -u(i, j);
    }
}

// ---------------------------------------------------------------------------
// Gram-path orthonormalisation of the distributed protocol (range_finder.hpp:43-105,
// used by dist_compress_mode, dist.hpp:688-699). Eigen's SelfAdjointEigenSolver
// (tridiagonalisation + implicit QL) is stood in for by a cyclic Jacobi eigensolver
// with round-robin (tournament) pairing: the eigenpairs are unique up to the sign of
// each eigenvector (distinct eigenvalues), which is all the reference's result
// depends on (its dist path applies no sign rule, and its tests compare subspaces,
// test_dist.cpp:141-152). The device kernel (csrc/gram.cu) runs the same rounds.
// ---------------------------------------------------------------------------

// Pairs of round r of the circle method over m (even) players: position 0 fixed,
// positions 1..m-1 rotate; pair k = (L[k], L[m-1-k]).
inline void jacobi_round_pairs(int m, int r, std::vector<std::pair<int, int>>& pairs) {
    std::vector<int> l(static_cast<size_t>(m));
    l[0] = 0;
    for (int k = 1; k < m; ++k) l[static_cast<size_t>(k)] = ((k - 1 + r) % (m - 1)) + 1;
    pairs.clear();
    for (int k = 0; k < m / 2; ++k) pairs.emplace_back(l[static_cast<size_t>(k)], l[static_cast<size_t>(m - 1 - k)]);
}

constexpr int kJacobiMaxSweeps = 40;

// a (n x n symmetric) -> eigenvalues ascending (Eigen's order) + eigenvectors (columns)
inline void sym_eig(const Mat& a_in, std::vector<double>& evals, Mat& evecs) {
    const int n = static_cast<int>(a_in.rows);
    Mat a = a_in;
    Mat v(n, n);
    for (int i = 0; i < n; ++i) v(i, i) = 1.0;
    const int m = n + (n & 1);
    std::vector<std::pair<int, int>> pairs;
    std::vector<double> cs(static_cast<size_t>(m / 2)), sn(static_cast<size_t>(m / 2));
    for (int sweep = 0; sweep < kJacobiMaxSweeps && n > 1; ++sweep) {
        bool rotated = false;
        for (int r = 0; r < m - 1; ++r) {
            jacobi_round_pairs(m, r, pairs);
            // rotation parameters of every pair from the same A (they act on disjoint rows)
            for (size_t k = 0; k < pairs.size(); ++k) {
                int p = pairs[k].first, q = pairs[k].second;
                if (p > q) std::swap(p, q);
                cs[k] = 1.0, sn[k] = 0.0;
                if (q >= n) continue;
                const double apq = a(p, q), app = a(p, p), aqq = a(q, q);
                if (std::abs(apq) <= 1e-16 * std::sqrt(std::abs(app * aqq)) || apq == 0.0) continue;  // gram.cu skip_rotation
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                cs[k] = 1.0 / std::sqrt(t * t + 1.0);
                sn[k] = t * cs[k];
                rotated = true;
            }
            // A <- P^T A (rows), then A <- A P and V <- V P (columns)
            for (size_t k = 0; k < pairs.size(); ++k) {
                int p = pairs[k].first, q = pairs[k].second;
                if (p > q) std::swap(p, q);
                if (q >= n || sn[k] == 0.0) continue;
                for (int c = 0; c < n; ++c) {
                    const double x = a(p, c), y = a(q, c);
                    a(p, c) = cs[k] * x - sn[k] * y;
                    a(q, c) = sn[k] * x + cs[k] * y;
                }
            }
            for (size_t k = 0; k < pairs.size(); ++k) {
                int p = pairs[k].first, q = pairs[k].second;
                if (p > q) std::swap(p, q);
                if (q >= n || sn[k] == 0.0) continue;
                for (int i = 0; i < n; ++i) {
                    const double x = a(i, p), y = a(i, q);
                    a(i, p) = cs[k] * x - sn[k] * y;
                    a(i, q) = sn[k] * x + cs[k] * y;
                    const double vx = v(i, p), vy = v(i, q);
                    v(i, p) = cs[k] * vx - sn[k] * vy;
                    v(i, q) = sn[k] * vx + cs[k] * vy;
                }
            }
        }
        if (!rotated) break;
    }
    // ascending order; ties keep the lower index first
    std::vector<int> idx(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) idx[static_cast<size_t>(i)] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return a(x, x) < a(y, y); });
    evals.assign(static_cast<size_t>(n), 0.0);
    evecs = Mat(n, n);
    for (int j = 0; j < n; ++j) {
        const int s = idx[static_cast<size_t>(j)];
        evals[static_cast<size_t>(j)] = a(s, s);
        for (int i = 0; i < n; ++i) evecs(i, j) = v(i, s);
    }
}

// gram_ortho_transform (range_finder.hpp:86-105): T with stacked-Z * T orthonormal,
// columns in descending eigenvalue order, eigenvalues <= 1e-12 * top dropped.
inline Mat gram_ortho_transform(const Mat& gram, std::vector<double>* spectrum) {
    require(gram.rows == gram.cols, "gram_ortho_transform: square Gram matrix required");
    std::vector<double> ev;
    Mat vec;
    sym_eig(gram, ev, vec);
    const Index r = gram.rows;
    const double top = r > 0 ? ev[static_cast<size_t>(r - 1)] : 0.0;
    require(top > 0.0, "gram_ortho_transform: zero Gram matrix");
    Index kept = 0;
    for (Index i = r - 1; i >= 0; --i) {
        if (ev[static_cast<size_t>(i)] > 1e-12 * top) ++kept;  // kRankDeficiencyTol
        else break;
    }
    Mat t(r, kept);
    if (spectrum) spectrum->assign(static_cast<size_t>(kept), 0.0);
    for (Index j = 0; j < kept; ++j) {
        const Index src = r - 1 - j;
        const double l = ev[static_cast<size_t>(src)];
        if (spectrum) (*spectrum)[static_cast<size_t>(j)] = l;
        for (Index i = 0; i < r; ++i) t(i, j) = vec(i, src) / std::sqrt(l);
    }
    return t;
}

// gram_orthonormalize (range_finder.hpp:48-84) on the stacked row blocks of z
// (block_rows[s] rows each): Gram = sum_s Z_s^T Z_s in block order, U = Z T.
inline Mat gram_orthonormalize(const Mat& z, const std::vector<Index>& block_rows, std::vector<double>* spectrum) {
    require(!block_rows.empty(), "gram_orthonormalize: no blocks");
    const Index r = z.cols;
    Mat gram(r, r);
    Index at = 0;
    for (Index len : block_rows) {
        for (Index j = 0; j < r; ++j)
            for (Index i = 0; i < r; ++i) {
                double acc = 0.0;
                for (Index k = 0; k < len; ++k) acc += z(at + k, i) * z(at + k, j);
                gram(i, j) += acc;
            }
        at += len;
    }
    require(at == z.rows, "gram_orthonormalize: block rows do not cover Z");
    const Mat t = gram_ortho_transform(gram, spectrum);
    Mat u(z.rows, t.cols);
    gemm(false, false, z.rows, t.cols, r, 1.0, z.data(), z.rows, t.data(), t.rows, 0.0, u.data(), u.rows);
    return u;
}

// U_n of one distributed compression step (dist.hpp:688-723): Z summed over blocks,
// Gram-eig transform, U = Z T; no sign rule.
inline Mat gram_basis(const Mat& z) { return gram_orthonormalize(z, {z.rows}, nullptr); }

struct Tucker {
    Tensor core;
    std::vector<Mat> factors;
};

// rand_tucker (Alg. 2, tucker.hpp:108-130)
// gram = true: the distributed protocol's orthonormalisation (dist_rand_tucker,
// dist.hpp:852-879: Gram-eig basis, no sign rule) on the assembled tensor.
inline Tucker rand_tucker(const Tensor& y, const std::vector<Index>& ranks, Index p, const Seed& seed,
                          bool gram = false) {
    require(static_cast<Index>(ranks.size()) == y.order(), "rand_tucker: one rank per mode required");
    require(p >= 0, "rand_tucker: oversampling must be nonnegative");
    Tucker m;
    m.factors.resize(static_cast<size_t>(y.order()));
    Tensor cur = y;
    for (Index n = 0; n < y.order(); ++n) {
        const Index rt = std::min(ranks[static_cast<size_t>(n)] + p, cur.dim(n));
        const Index width = cur.size() / cur.dim(n);
        const Mat omega = gaussian_matrix(width, rt, alg2_omega_seed(seed, n));
        Mat u;
        if (gram) {
            u = gram_basis(unfold_times(cur, n, omega));
        } else {
            u = orthonormal_basis(unfold_times(cur, n, omega));
            fix_column_signs(u);
        }
        cur = ttm(cur, transpose(u), n);
        m.factors[static_cast<size_t>(n)] = std::move(u);
    }
    m.core = std::move(cur);
    return m;
}

// rand_tucker_2i (Alg. 3, tucker.hpp:136-169). `z_out`, if given, receives the
// 2N sketches Z (diagnostics for the parity tests).
inline Tucker rand_tucker_2i(const Tensor& y, const std::vector<Index>& ranks, Index p,
                             const Seed& seed, std::vector<Mat>* z_out = nullptr, bool gram = false) {
    require(static_cast<Index>(ranks.size()) == y.order(), "rand_tucker_2i: one rank per mode required");
    require(p >= 0, "rand_tucker_2i: oversampling must be nonnegative");
    const Index order = y.order();
    std::vector<Mat> factors(static_cast<size_t>(order));
    for (Index n = 0; n < order; ++n) {
        const Index rt = std::min(ranks[static_cast<size_t>(n)] + p, y.dim(n));
        factors[static_cast<size_t>(n)] = gaussian_matrix(y.dim(n), rt, alg3_init_seed(seed, n));
    }
    for (Index pass = 0; pass < 2; ++pass) {
        for (Index n = 0; n < order; ++n) {
            const Tensor x = ttm_all(y, factors, n, true);
            const Index rt = std::min(ranks[static_cast<size_t>(n)] + p, y.dim(n));
            const Index width = x.size() / x.dim(n);
            const Mat omega = gaussian_matrix(width, rt, alg3_omega_seed(seed, pass, n));
            Mat z = unfold_times(x, n, omega);
            if (z_out) z_out->push_back(z);
            Mat u;
            if (gram) {  // dist_rand_tucker_2i (dist.hpp:884-936): Gram-eig basis, no sign rule
                u = gram_basis(z);
            } else {
                u = orthonormal_basis(z);
                fix_column_signs(u);
            }
            factors[static_cast<size_t>(n)] = std::move(u);
        }
    }
    Tucker m;
    m.core = ttm_all(y, factors, -1, true);  // tucker.hpp:166
    m.factors = std::move(factors);
    return m;
}

// ---------------------------------------------------------------------------
// Streamed-slab restatement of rand_tucker_2i for tensors whose fp64 copy does not fit in
// host memory (BASELINE cfgs 3-5: 55-256 GB of fp32). Y is read as contiguous slabs of its
// last mode (fp32 -> fp64 per slab) and every ttm_all is accumulated slab by slab in slab
// order, the pattern of the reference's streamed_block_product (dist.hpp:496-596) and
// dist_project (dist.hpp:617-651): with slab s = Y[..., a:b],
//   ttm_all(Y, U, skip) = sum_s ttm_all(Y_s, U, skip) restricted to rows a:b of U_last
// (skip != last) or the slabs of ttm_all(Y_s, U, skip) placed at a:b (skip == last).
// Same modes, same order of application (ascending, tensor.hpp:186-190) and the same
// rand_tucker_2i control flow (tucker.hpp:136-169) as rand_tucker_2i() above; only the
// summation order over the last mode differs (per slab, then over slabs, fp64).
// ---------------------------------------------------------------------------
struct SlabSource {
    const float* y32 = nullptr;
    std::vector<Index> shape;
    Index front = 1;      // prod of all but the last extent
    Index slab_len = 1;   // last-mode rows per slab
};

// fp32 -> fp64 copy of rows [a, b) of the last mode into `t` (reused across slabs: one
// allocation, no per-slab zero fill or page faults), split over g_threads host threads
inline void load_slab(const SlabSource& src, Index a, Index b, Tensor& t) {
    std::vector<Index> s = src.shape;
    s.back() = b - a;
    const Index n = src.front * (b - a);
    if (static_cast<Index>(t.d.size()) < n) t.d.resize(static_cast<size_t>(n));
    t.d.resize(static_cast<size_t>(n));
    t.shape = s;
    const float* from = src.y32 + a * src.front;
    double* to = t.data();
    const int nt = std::max(1, std::min<int>(g_threads, static_cast<int>(n / (1 << 20)) + 1));
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w) {
        const Index lo = n * w / nt, hi = n * (w + 1) / nt;
        pool.emplace_back([=] {
            for (Index i = lo; i < hi; ++i) to[i] = static_cast<double>(from[i]);
        });
    }
    for (auto& th : pool) th.join();
}

// ttm_all(Y, ms, skip, transpose=true) over the slabs of Y (skip = -1: every mode)
inline Tensor ttm_all_streamed(const SlabSource& src, const std::vector<Mat>& ms, Index skip) {
    const Index order = static_cast<Index>(src.shape.size());
    const Index last = order - 1;
    const Index L = src.shape.back();
    std::vector<Index> os(src.shape);
    for (Index n = 0; n < order; ++n)
        if (n != skip) os[static_cast<size_t>(n)] = ms[static_cast<size_t>(n)].cols;
    Tensor x(os);
    std::vector<Mat> mt(static_cast<size_t>(order));
    for (Index n = 0; n < last; ++n)
        if (n != skip) mt[static_cast<size_t>(n)] = transpose(ms[static_cast<size_t>(n)]);
    Tensor slab;
    slab.d.reserve(static_cast<size_t>(src.front * std::min(L, src.slab_len)));
    for (Index a = 0; a < L; a += src.slab_len) {
        const Index b = std::min(L, a + src.slab_len);
        load_slab(src, a, b, slab);
        Tensor cur;
        bool first = true;
        for (Index n = 0; n < last; ++n) {  // ascending modes, as tensor.hpp:186-190
            if (n == skip) continue;
            cur = ttm(first ? slab : cur, mt[static_cast<size_t>(n)], n);
            first = false;
        }
        if (first) cur = slab;  // order 1 + skip: nothing to contract before the last mode
        if (skip == last) {  // the slab's rows of X (contiguous: last mode slowest)
            std::copy(cur.d.begin(), cur.d.end(), x.d.begin() + a * (x.size() / L));
            continue;
        }
        // X += cur x_last U_last[a:b, :]^T (the slab's share of the last-mode contraction)
        const Mat& u = ms[static_cast<size_t>(last)];
        const Index front = cur.size() / (b - a);
        gemm(false, false, front, u.cols, b - a, 1.0, cur.data(), front, u.data() + a, u.rows, 1.0, x.data(), front);
    }
    return x;
}

// Diagnostics of the two discrete choices of a range step (hard part 1):
// pivot margin = min_k (top - second) / top of the updated column norms at ColPiv step k
// (range_finder.hpp:18-29); sign margin = min over columns of (|u|_max - max |u_i| over the
// entries of the opposite sign) / |u|_max (fix_column_signs, tucker.hpp:39-45): how close the
// sign rule is to picking an entry of the other sign.
inline double sign_margin(const Mat& u) {
    double m = 1.0;
    for (Index j = 0; j < u.cols; ++j) {
        Index imax = 0;
        double best = -1.0;
        for (Index i = 0; i < u.rows; ++i)
            if (std::abs(u(i, j)) > best) best = std::abs(u(i, j)), imax = i;
        const bool pos = u(imax, j) >= 0;
        double opp = 0.0;
        for (Index i = 0; i < u.rows; ++i)
            if ((u(i, j) >= 0) != pos) opp = std::max(opp, std::abs(u(i, j)));
        if (best > 0) m = std::min(m, (best - opp) / best);
    }
    return m;
}

inline Tucker rand_tucker_2i_streamed(const SlabSource& src, const std::vector<Index>& ranks, Index p,
                                      const Seed& seed, std::vector<Mat>* z_out, std::vector<double>* margins) {
    const Index order = static_cast<Index>(src.shape.size());
    require(order >= 2, "rand_tucker_2i: streamed oracle needs order >= 2");
    require(static_cast<Index>(ranks.size()) == order, "rand_tucker_2i: one rank per mode required");
    require(p >= 0, "rand_tucker_2i: oversampling must be nonnegative");
    std::vector<Mat> factors(static_cast<size_t>(order));
    for (Index n = 0; n < order; ++n) {  // tucker.hpp:141-147
        const Index rt = std::min(ranks[static_cast<size_t>(n)] + p, src.shape[static_cast<size_t>(n)]);
        factors[static_cast<size_t>(n)] = gaussian_matrix(src.shape[static_cast<size_t>(n)], rt, alg3_init_seed(seed, n));
    }
    for (Index pass = 0; pass < 2; ++pass) {  // tucker.hpp:149-162
        for (Index n = 0; n < order; ++n) {
            const Tensor x = ttm_all_streamed(src, factors, n);
            const Index rt = std::min(ranks[static_cast<size_t>(n)] + p, src.shape[static_cast<size_t>(n)]);
            const Index width = x.size() / x.dim(n);
            const Mat omega = gaussian_matrix(width, rt, alg3_omega_seed(seed, pass, n));
            Mat z = unfold_times(x, n, omega);
            ColPivQR f;
            Mat u = orthonormal_basis(z, &f);
            fix_column_signs(u);
            if (margins) {
                double pm = 1.0;
                for (Index k = 0; k + 1 < u.cols; ++k) pm = std::min(pm, f.pivot_margin[static_cast<size_t>(k)]);
                margins->push_back(pm);
                margins->push_back(sign_margin(u));
            }
            if (z_out) z_out->push_back(std::move(z));
            factors[static_cast<size_t>(n)] = std::move(u);
        }
    }
    Tucker m;
    m.core = ttm_all_streamed(src, factors, -1);  // tucker.hpp:166
    m.factors = std::move(factors);
    return m;
}

// reconstruct (tucker.hpp:63-66)
inline Tensor reconstruct(const Tucker& m) { return ttm_all(m.core, m.factors, -1, false); }

// ---------------------------------------------------------------------------
// Generators (bench.hpp:56-112) + the configs' U(0,1) / |N| variants
// (uniform_at(gen_factor_seed(seed,n), j*I_n+i)).
// ---------------------------------------------------------------------------
inline Tensor gaussian_tensor(const std::vector<Index>& shape, const Seed& s) {  // random.hpp:124-138
    Tensor t(shape);
    gaussian_fill(t.data(), static_cast<uint64_t>(t.size()), s.key());
    return t;
}

inline Tensor gen_tucker_tensor(const std::vector<Index>& dims, const std::vector<Index>& mlr,
                                const Seed& seed, Tucker* model_out) {  // bench.hpp:83-95
    require(dims.size() == mlr.size(), "gen_tucker_tensor: rank list mismatch");
    Tucker m;
    m.core = gaussian_tensor(mlr, seed.derived(0xC0DEu));
    m.factors.resize(dims.size());
    for (size_t n = 0; n < dims.size(); ++n)
        m.factors[n] = gaussian_matrix(dims[n], mlr[n], gen_factor_seed(seed, static_cast<Index>(n)));
    Tensor t = reconstruct(m);
    if (model_out) *model_out = std::move(m);
    return t;
}

// kind: 0 gaussian, 1 exponential-sparse, 2 uniform(0,1]
inline Tensor gen_cp_tensor(const std::vector<Index>& dims, Index rank, int kind, double zero_frac,
                            const Seed& seed, std::vector<Mat>* factors_out) {  // bench.hpp:56-80
    require(rank >= 1, "gen_cp_tensor: rank must be positive");
    require(zero_frac >= 0.0 && zero_frac < 1.0, "gen_cp_tensor: bad zero fraction");
    std::vector<Mat> fs(dims.size());
    for (size_t n = 0; n < dims.size(); ++n) {
        const Seed s = gen_factor_seed(seed, static_cast<Index>(n));
        Mat a(dims[n], rank);
        if (kind == 1) {
            const Seed zs = s.derived(0x5Au);
            for (Index j = 0; j < rank; ++j)
                for (Index i = 0; i < dims[n]; ++i) {
                    const uint64_t idx = static_cast<uint64_t>(j * dims[n] + i);
                    const bool zero = counter_unit(zs.key(), idx) <= zero_frac;
                    a(i, j) = zero ? 0.0 : -10.0 * std::log(counter_unit(s.key(), idx));
                }
        } else if (kind == 2) {
            const uint64_t key = s.key();
            for (Index j = 0; j < rank; ++j)
                for (Index i = 0; i < dims[n]; ++i)
                    a(i, j) = counter_unit(key, static_cast<uint64_t>(j * dims[n] + i));
        } else {
            a = gaussian_matrix(dims[n], rank, s);
        }
        fs[n] = std::move(a);
    }
    // cp_reconstruct (cp.hpp:118-128): unfold(Y,0) = A0 * KR(A_{N-1},...,A_1)^T
    Tensor t(dims);
    const Index order = static_cast<Index>(dims.size());
    if (order == 1) {
        for (Index i = 0; i < dims[0]; ++i) {
            double s = 0.0;
            for (Index r = 0; r < rank; ++r) s += fs[0](i, r);
            t.d[static_cast<size_t>(i)] = s;
        }
    } else {
        Index width = 1;
        for (Index n = 1; n < order; ++n) width *= dims[static_cast<size_t>(n)];
        Mat kr(width, rank);
        std::vector<Index> sub(static_cast<size_t>(order), 0);
        for (Index c = 0; c < width; ++c) {
            for (Index r = 0; r < rank; ++r) {
                double v = 1.0;
                for (Index n = order - 1; n >= 1; --n) v *= fs[static_cast<size_t>(n)](sub[static_cast<size_t>(n)], r);
                kr(c, r) = v;
            }
            for (Index n = 1; n < order; ++n) {
                if (++sub[static_cast<size_t>(n)] < dims[static_cast<size_t>(n)]) break;
                sub[static_cast<size_t>(n)] = 0;
            }
        }
        gemm(false, true, dims[0], width, rank, 1.0, fs[0].data(), dims[0], kr.data(), width, 0.0,
             t.data(), dims[0]);
    }
    if (factors_out) *factors_out = std::move(fs);
    return t;
}

// add_noise (bench.hpp:100-112); abs_noise=true is the |N(0,sigma)| variant of cfg 4.
inline void add_noise(Tensor& y, double snr_db, const Seed& seed, bool abs_noise) {
    if (std::isinf(snr_db) && snr_db > 0) return;
    require(std::isfinite(snr_db), "add_noise: SNR must be finite or +inf");
    const double ny = std::sqrt(sq_norm(y.data(), y.size()));
    require(ny > 0.0, "add_noise: zero tensor input");
    Tensor e = gaussian_tensor(y.shape, seed.derived(0x7015Eu));
    if (abs_noise)
        for (auto& v : e.d) v = std::abs(v);
    const double ne = std::sqrt(sq_norm(e.data(), e.size()));
    require(ne > 0.0, "add_noise: degenerate noise draw");
    const double sigma = ny / (ne * std::pow(10.0, snr_db / 20.0));
    for (Index i = 0; i < y.size(); ++i) y.d[static_cast<size_t>(i)] += sigma * e.d[static_cast<size_t>(i)];
}

// ---------------------------------------------------------------------------
// FFCP (ffcp.hpp:33-194) with the cp.hpp helpers it uses (cp.hpp:63-113)
// ---------------------------------------------------------------------------

// LDLT with symmetric (max-diagonal) pivoting, restating Eigen::LDLT, then solve
// X * BtB = YB  (cp.hpp:63-70, solve_normal)
inline bool ldlt_solve(const Mat& a_in, Mat& rhs_t /* n x m, solved in place */) {
    const Index n = a_in.rows;
    Mat a = a_in;
    std::vector<Index> tr(static_cast<size_t>(n));
    for (Index k = 0; k < n; ++k) {
        Index best = k;
        double bv = std::abs(a(k, k));
        for (Index i = k + 1; i < n; ++i)
            if (std::abs(a(i, i)) > bv) {
                bv = std::abs(a(i, i));
                best = i;
            }
        tr[static_cast<size_t>(k)] = best;
        if (best != k) {  // symmetric swap of row/col k and best (lower part used)
            for (Index j = 0; j < n; ++j) std::swap(a(k, j), a(best, j));
            for (Index i = 0; i < n; ++i) std::swap(a(i, k), a(i, best));
        }
        // a(k,k) -= sum_{j<k} L(k,j)^2 D(j)
        double dk = a(k, k);
        for (Index j = 0; j < k; ++j) dk -= a(k, j) * a(k, j) * a(j, j);
        a(k, k) = dk;
        for (Index i = k + 1; i < n; ++i) {
            double s = a(i, k);
            for (Index j = 0; j < k; ++j) s -= a(i, j) * a(k, j) * a(j, j);
            a(i, k) = std::abs(dk) > 0.0 ? s / dk : s;  // Eigen leaves A21 undivided on a zero pivot
        }
    }
    // solve for every column of rhs_t
    for (Index c = 0; c < rhs_t.cols; ++c) {
        double* b = rhs_t.col(c);
        for (Index k = 0; k < n; ++k) std::swap(b[k], b[tr[static_cast<size_t>(k)]]);
        for (Index i = 0; i < n; ++i)
            for (Index j = 0; j < i; ++j) b[i] -= a(i, j) * b[j];
        // D^{-1} with Eigen's pseudo-inverse rule for vanishing pivots
        for (Index i = 0; i < n; ++i) {
            if (std::abs(a(i, i)) > std::numeric_limits<double>::min()) b[i] /= a(i, i);
            else b[i] = 0.0;
        }
        for (Index i = n - 1; i >= 0; --i)
            for (Index j = i + 1; j < n; ++j) b[i] -= a(j, i) * b[j];
        for (Index k = n - 1; k >= 0; --k) std::swap(b[k], b[tr[static_cast<size_t>(k)]]);
    }
    for (double v : rhs_t.d)
        if (!std::isfinite(v)) return false;
    return true;
}

inline Mat solve_normal(const Mat& yb, const Mat& btb) {  // cp.hpp:63-70
    Mat xt = transpose(yb);
    if (ldlt_solve(btb, xt)) return transpose(xt);
    double tr = 0.0;
    for (Index i = 0; i < btb.rows; ++i) tr += btb(i, i);
    const double ridge = 1e-12 * tr + 1e-300;
    Mat reg = btb;
    for (Index i = 0; i < reg.rows; ++i) reg(i, i) += ridge;
    xt = transpose(yb);
    ldlt_solve(reg, xt);
    return transpose(xt);
}

inline void hals_sweep(Mat& a, const Mat& q, const Mat& t, bool project) {  // cp.hpp:84-92
    std::vector<double> col(static_cast<size_t>(a.rows));
    for (Index r = 0; r < a.cols; ++r) {
        const double trr = t(r, r);
        if (trr < 1e-15) continue;
        for (Index i = 0; i < a.rows; ++i) {
            double at = 0.0;
            for (Index s = 0; s < a.cols; ++s) at += a(i, s) * t(s, r);
            double v = a(i, r) + (q(i, r) - at) / trr;
            if (project) v = std::max(v, 0.0);
            col[static_cast<size_t>(i)] = v;
        }
        for (Index i = 0; i < a.rows; ++i) a(i, r) = col[static_cast<size_t>(i)];
    }
}

inline void absorb_scales(std::vector<Mat>& f) {  // cp.hpp:96-109
    if (f.size() < 2) return;
    Mat& last = f.back();
    for (size_t n = 0; n + 1 < f.size(); ++n) {
        Mat& a = f[n];
        for (Index r = 0; r < a.cols; ++r) {
            const double norm = std::sqrt(sq_norm(a.col(r), a.rows));
            if (norm > 0.0) {
                for (Index i = 0; i < a.rows; ++i) a(i, r) /= norm;
                for (Index i = 0; i < last.rows; ++i) last(i, r) *= norm;
            }
        }
    }
}

inline Mat matmul_tn(const Mat& a, const Mat& b) {  // a^T b
    Mat c(a.cols, b.cols);
    gemm(true, false, a.cols, b.cols, a.rows, 1.0, a.data(), a.rows, b.data(), b.rows, 0.0, c.data(), c.rows);
    return c;
}
inline Mat matmul(const Mat& a, const Mat& b) {
    Mat c(a.rows, b.cols);
    gemm(false, false, a.rows, b.cols, a.cols, 1.0, a.data(), a.rows, b.data(), b.rows, 0.0, c.data(), c.rows);
    return c;
}

// ffcp_h (ffcp.hpp:33-47)
inline Mat ffcp_h(const Tensor& core, const std::vector<Mat>& v, Index mode) {
    const Index rank = v[static_cast<size_t>(mode == 0 ? 1 : 0)].cols;
    Mat h(core.dim(mode), rank);
    for (Index r = 0; r < rank; ++r) {
        Tensor cur = core;
        for (Index p = core.order() - 1; p >= 0; --p) {
            if (p == mode) continue;
            const Mat& vp = v[static_cast<size_t>(p)];
            Mat vr(1, vp.rows);
            for (Index i = 0; i < vp.rows; ++i) vr(0, i) = vp(i, r);
            cur = ttm(cur, vr, p);
        }
        std::copy(cur.d.begin(), cur.d.end(), h.col(r));
    }
    return h;
}

enum Constraint { kNone = 0, kNonnegMu = 1, kNonnegHals = 2, kSparse = 3 };

struct FfcpOut {
    std::vector<Mat> factors;
    std::vector<double> fit_trace;
    int iterations = 0;
};

inline FfcpOut ffcp(const Tucker& model, Index rank, int kind, double c, int max_iters,
                    double fit_tol, const Seed& seed) {  // ffcp.hpp:94-194
    const Index order = model.core.order();
    require(static_cast<Index>(model.factors.size()) == order, "tucker model: one factor per mode required");
    for (Index n = 0; n < order; ++n)
        require(model.factors[static_cast<size_t>(n)].cols == model.core.dim(n),
                "tucker model: factor columns must match core shape");
    require(order >= 2, "ffcp: tensor order must be at least 2");
    require(rank >= 1, "ffcp: rank must be positive");
    require(c >= 0.0, "ffcp: sparsity level must be nonnegative");
    const bool nonneg = kind == kNonnegMu || kind == kNonnegHals;
    FfcpOut out;
    out.factors.resize(static_cast<size_t>(order));
    std::vector<Mat> v(static_cast<size_t>(order)), grams(static_cast<size_t>(order));
    for (Index n = 0; n < order; ++n) {
        const Mat& u = model.factors[static_cast<size_t>(n)];
        Mat a = gaussian_matrix(u.rows, rank, ffcp_init_seed(seed, n));
        if (nonneg)
            for (auto& x : a.d) x = std::abs(x);
        v[static_cast<size_t>(n)] = matmul_tn(u, a);
        grams[static_cast<size_t>(n)] = matmul_tn(a, a);
        out.factors[static_cast<size_t>(n)] = std::move(a);
    }
    double yt_sq;
    {
        std::vector<Mat> uu(static_cast<size_t>(order));
        for (Index n = 0; n < order; ++n)
            uu[static_cast<size_t>(n)] = matmul_tn(model.factors[static_cast<size_t>(n)], model.factors[static_cast<size_t>(n)]);
        const Tensor guu = ttm_all(model.core, uu, -1, false);
        double s = 0.0;
        for (Index i = 0; i < guu.size(); ++i) s += model.core.d[static_cast<size_t>(i)] * guu.d[static_cast<size_t>(i)];
        yt_sq = std::max(0.0, s);
    }
    const double yt_norm = std::sqrt(yt_sq);
    require(yt_norm > 0.0, "ffcp: compressed tensor has zero norm");
    const double eps = 1e-16;
    double prev_fit = -std::numeric_limits<double>::infinity();
    for (int it = 0; it < max_iters; ++it) {
        double res_sq = 0.0;
        for (Index n = 0; n < order; ++n) {
            const Mat h = ffcp_h(model.core, v, n);
            const Mat& u = model.factors[static_cast<size_t>(n)];
            const Mat q = matmul(u, h);
            Mat t(rank, rank);
            std::fill(t.d.begin(), t.d.end(), 1.0);
            for (Index p = 0; p < order; ++p)
                if (p != n)
                    for (size_t i = 0; i < t.d.size(); ++i) t.d[i] *= grams[static_cast<size_t>(p)].d[i];
            Mat& a = out.factors[static_cast<size_t>(n)];
            switch (kind) {
                case kNone: a = solve_normal(q, t); break;
                case kNonnegMu: {
                    const Mat at = matmul(a, t);
                    for (size_t i = 0; i < a.d.size(); ++i)
                        a.d[i] *= std::max(q.d[i], 0.0) / std::max(at.d[i], eps);
                    break;
                }
                case kNonnegHals: hals_sweep(a, q, t, true); break;
                case kSparse: {
                    a = solve_normal(q, t);
                    for (auto& x : a.d) x = x > c ? x - c : (x < -c ? x + c : 0.0);  // ffcp.hpp:20-27
                    break;
                }
                default: require(false, "ffcp: unknown constraint");
            }
            grams[static_cast<size_t>(n)] = matmul_tn(a, a);
            v[static_cast<size_t>(n)] = matmul_tn(u, a);
            if (n == order - 1) {
                double inner = 0.0, model_sq = 0.0;
                for (size_t i = 0; i < h.d.size(); ++i) inner += h.d[i] * v[static_cast<size_t>(n)].d[i];
                for (size_t i = 0; i < t.d.size(); ++i) model_sq += t.d[i] * grams[static_cast<size_t>(n)].d[i];
                res_sq = std::max(0.0, yt_sq - 2.0 * inner + model_sq);
            }
        }
        const double f = 1.0 - std::sqrt(res_sq) / yt_norm;
        out.fit_trace.push_back(f);
        out.iterations = it + 1;
        if (std::abs(f - prev_fit) < fit_tol) break;
        prev_fit = f;
    }
    absorb_scales(out.factors);
    return out;
}

// cp_reconstruct (cp.hpp:118-128) as a direct sum of outer products
inline Tensor cp_reconstruct(const std::vector<Mat>& f) {
    std::vector<Index> shape;
    for (const Mat& a : f) shape.push_back(a.rows);
    Tensor t(shape);
    const Index order = static_cast<Index>(f.size()), rank = f[0].cols;
    std::vector<Index> sub(static_cast<size_t>(order), 0);
    for (Index idx = 0; idx < t.size(); ++idx) {
        double s = 0.0;
        for (Index r = 0; r < rank; ++r) {
            double v = 1.0;
            for (Index n = 0; n < order; ++n) v *= f[static_cast<size_t>(n)](sub[static_cast<size_t>(n)], r);
            s += v;
        }
        t.d[static_cast<size_t>(idx)] = s;
        for (Index n = 0; n < order; ++n) {
            if (++sub[static_cast<size_t>(n)] < shape[static_cast<size_t>(n)]) break;
            sub[static_cast<size_t>(n)] = 0;
        }
    }
    return t;
}

}  // namespace tko

// ===========================================================================
// C API (ctypes). Every entry returns 0 on success, 1 on invalid_argument, 2 on
// other errors; tko_last_error() holds the message.
// ===========================================================================
using namespace tko;

#define TKO_TRY(...)                                        \
    try {                                                   \
        __VA_ARGS__;                                        \
        return 0;                                           \
    } catch (const std::invalid_argument& e) {              \
        g_last_error = e.what();                            \
        return 1;                                           \
    } catch (const std::exception& e) {                     \
        g_last_error = e.what();                            \
        return 2;                                           \
    }

static std::vector<Index> to_shape(const int64_t* s, int64_t order) {
    return std::vector<Index>(s, s + order);
}
static Tensor to_tensor(const int64_t* s, int64_t order, const double* data) {
    Tensor t(to_shape(s, order));
    std::memcpy(t.data(), data, sizeof(double) * static_cast<size_t>(t.size()));
    return t;
}
static Mat to_mat(int64_t r, int64_t c, const double* d) {
    Mat m(r, c);
    std::memcpy(m.data(), d, sizeof(double) * static_cast<size_t>(r * c));
    return m;
}

// factor output convention: caller passes, per mode, a buffer of I_n * rt_n doubles
// (column-major) and receives the actual column count in cols[n].
static void write_model(const Tucker& m, double* core, int64_t* core_shape, double** factors,
                        int64_t* cols) {
    std::memcpy(core, m.core.data(), sizeof(double) * static_cast<size_t>(m.core.size()));
    for (size_t n = 0; n < m.factors.size(); ++n) {
        core_shape[n] = m.core.shape[n];
        cols[n] = m.factors[n].cols;
        std::memcpy(factors[n], m.factors[n].data(), sizeof(double) * m.factors[n].d.size());
    }
}

extern "C" {

const char* tko_last_error() { return g_last_error.c_str(); }

// Load OpenBLAS (ILP64) for the large GEMMs; returns 1 if found.
int tko_blas_init(const char* path, int threads) {
    if (path && *path) {
        void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
        if (h) {
            g_dgemm = reinterpret_cast<dgemm_fn>(dlsym(h, "scipy_dgemm_64_"));
            g_setthreads = reinterpret_cast<setthreads_fn>(dlsym(h, "scipy_openblas_set_num_threads64_"));
        }
    }
    g_threads = threads > 0 ? threads : 1;
    if (g_setthreads) g_setthreads(g_threads);
    return g_dgemm ? 1 : 0;
}
void tko_blas_disable() { g_dgemm = nullptr; }

uint64_t tko_mix64(uint64_t x) { return mix64(x); }
uint64_t tko_seed_key(uint64_t root, uint64_t stream) { return Seed{root, stream}.key(); }
uint64_t tko_seed_derived(uint64_t root, uint64_t stream, uint64_t tag) {
    return Seed{root, stream}.derived(tag).stream;
}
double tko_normal_at(uint64_t root, uint64_t stream, uint64_t idx) {
    return normal_at_key(Seed{root, stream}.key(), idx);
}
double tko_uniform_at(uint64_t root, uint64_t stream, uint64_t idx) {
    return counter_unit(Seed{root, stream}.key(), idx);
}
int tko_gaussian_matrix(int64_t rows, int64_t cols, uint64_t root, uint64_t stream, double* out) {
    TKO_TRY({
        Mat m = gaussian_matrix(rows, cols, Seed{root, stream});
        std::memcpy(out, m.data(), sizeof(double) * m.d.size());
    })
}
int tko_gaussian_rows(int64_t total_rows, int64_t cols, uint64_t root, uint64_t stream,
                      const int64_t* row_ids, int64_t nrows, double* out) {  // random.hpp:105-116
    TKO_TRY({
        const uint64_t key = Seed{root, stream}.key();
        for (int64_t j = 0; j < cols; ++j)
            for (int64_t i = 0; i < nrows; ++i)
                out[i + j * nrows] = normal_at_key(key, static_cast<uint64_t>(j) * static_cast<uint64_t>(total_rows) +
                                                            static_cast<uint64_t>(row_ids[i]));
    })
}

int tko_unfold(const int64_t* shape, int64_t order, const double* t, int64_t mode, double* out) {
    TKO_TRY({
        Mat m = unfold(to_tensor(shape, order, t), mode);
        std::memcpy(out, m.data(), sizeof(double) * m.d.size());
    })
}
int tko_ttm(const int64_t* shape, int64_t order, const double* t, int64_t mrows, int64_t mcols,
            const double* m, int64_t mode, double* out) {
    TKO_TRY({
        Tensor r = ttm(to_tensor(shape, order, t), to_mat(mrows, mcols, m), mode);
        std::memcpy(out, r.data(), sizeof(double) * r.d.size());
    })
}
// matrices[n] is rows[n] x cols[n]; with transpose=1 each is applied transposed
int tko_ttm_all(const int64_t* shape, int64_t order, const double* t, const double** ms,
                const int64_t* rows, const int64_t* cols, int64_t skip, int transpose_m,
                double* out, int64_t* out_shape) {
    TKO_TRY({
        std::vector<Mat> v;
        for (int64_t n = 0; n < order; ++n) v.push_back(to_mat(rows[n], cols[n], ms[n]));
        Tensor r = ttm_all(to_tensor(shape, order, t), v, skip, transpose_m != 0);
        std::memcpy(out, r.data(), sizeof(double) * r.d.size());
        for (int64_t n = 0; n < order; ++n) out_shape[n] = r.shape[static_cast<size_t>(n)];
    })
}
int tko_unfold_times(const int64_t* shape, int64_t order, const double* t, int64_t mode,
                     int64_t brows, int64_t bcols, const double* b, double* out) {
    TKO_TRY({
        Mat z = unfold_times(to_tensor(shape, order, t), mode, to_mat(brows, bcols, b));
        std::memcpy(out, z.data(), sizeof(double) * z.d.size());
    })
}
// q: rows x cols buffer; returns rank; perm (cols) and diag (min(rows,cols)) optional
int tko_orthonormal_basis(int64_t rows, int64_t cols, const double* z, double* q, int64_t* rank,
                          int64_t* perm, double* rdiag, double* pivot_margin) {
    TKO_TRY({
        ColPivQR f;
        Mat u = orthonormal_basis(to_mat(rows, cols, z), &f);
        *rank = u.cols;
        std::memcpy(q, u.data(), sizeof(double) * u.d.size());
        if (cols > 0) {
            const int64_t size = std::min(rows, cols);
            if (perm) for (int64_t k = 0; k < cols; ++k) perm[k] = f.perm[static_cast<size_t>(k)];
            if (rdiag) for (int64_t k = 0; k < size; ++k) rdiag[k] = f.qr(k, k);
            if (pivot_margin) for (int64_t k = 0; k < size; ++k) pivot_margin[k] = f.pivot_margin[static_cast<size_t>(k)];
        }
    })
}
int tko_sym_eig(int64_t n, const double* a, double* evals, double* evecs) {
    TKO_TRY({
        std::vector<double> ev;
        Mat v;
        sym_eig(to_mat(n, n, a), ev, v);
        std::memcpy(evals, ev.data(), sizeof(double) * ev.size());
        std::memcpy(evecs, v.data(), sizeof(double) * v.d.size());
    })
}
int tko_gram_ortho_transform(int64_t n, const double* gram, double* transform, double* spectrum, int64_t* kept) {
    TKO_TRY({
        std::vector<double> sp;
        Mat t = gram_ortho_transform(to_mat(n, n, gram), &sp);
        *kept = t.cols;
        std::memcpy(transform, t.data(), sizeof(double) * t.d.size());
        std::memcpy(spectrum, sp.data(), sizeof(double) * sp.size());
    })
}
int tko_gram_orthonormalize(int64_t nblocks, const int64_t* block_rows, int64_t cols, const double* z, double* u,
                            double* spectrum, int64_t* kept) {
    TKO_TRY({
        std::vector<Index> br(block_rows, block_rows + nblocks);
        Index rows = 0;
        for (Index b : br) rows += b;
        std::vector<double> sp;
        Mat q = gram_orthonormalize(to_mat(rows, cols, z), br, &sp);
        *kept = q.cols;
        std::memcpy(u, q.data(), sizeof(double) * q.d.size());
        std::memcpy(spectrum, sp.data(), sizeof(double) * sp.size());
    })
}
int tko_fix_column_signs(int64_t rows, int64_t cols, double* u) {
    TKO_TRY({
        Mat m = to_mat(rows, cols, u);
        fix_column_signs(m);
        std::memcpy(u, m.data(), sizeof(double) * m.d.size());
    })
}

int tko_rand_tucker_2i(const int64_t* shape, int64_t order, const double* y, const int64_t* ranks,
                       int64_t p, uint64_t root, uint64_t stream, double* core, int64_t* core_shape,
                       double** factors, int64_t* cols, double** z_out) {
    TKO_TRY({
        std::vector<Mat> zs;
        Tucker m = rand_tucker_2i(to_tensor(shape, order, y), to_shape(ranks, order), p, Seed{root, stream},
                                  z_out ? &zs : nullptr);
        write_model(m, core, core_shape, factors, cols);
        if (z_out)
            for (size_t i = 0; i < zs.size(); ++i)
                std::memcpy(z_out[i], zs[i].data(), sizeof(double) * zs[i].d.size());
    })
}
// Streamed-slab rand_tucker_2i on an fp32 host tensor (slab_elems: target fp64 elements per
// slab of the last mode); margins (optional, 4N doubles): per step (pivot margin, sign margin).
int tko_rand_tucker_2i_f32_streamed(const int64_t* shape, int64_t order, const float* y, const int64_t* ranks,
                                    int64_t p, uint64_t root, uint64_t stream, int64_t slab_elems, double* core,
                                    int64_t* core_shape, double** factors, int64_t* cols, double** z_out,
                                    double* margins) {
    TKO_TRY({
        SlabSource src;
        src.y32 = y;
        src.shape = to_shape(shape, order);
        for (int64_t n = 0; n + 1 < order; ++n) src.front *= shape[n];
        src.slab_len = std::max<Index>(1, std::min<Index>(shape[order - 1], slab_elems / src.front));
        std::vector<Mat> zs;
        std::vector<double> mg;
        Tucker m = rand_tucker_2i_streamed(src, to_shape(ranks, order), p, Seed{root, stream}, z_out ? &zs : nullptr,
                                           margins ? &mg : nullptr);
        write_model(m, core, core_shape, factors, cols);
        if (z_out)
            for (size_t i = 0; i < zs.size(); ++i)
                std::memcpy(z_out[i], zs[i].data(), sizeof(double) * zs[i].d.size());
        if (margins) std::memcpy(margins, mg.data(), sizeof(double) * mg.size());
    })
}
// The reference's distributed algorithms (dist.hpp:852-936) on the assembled tensor:
// alg 2 = dist_rand_tucker, alg 3 = dist_rand_tucker_2i (Gram-eig orthonormalisation).
int tko_dist_rand_tucker_gram(int alg, const int64_t* shape, int64_t order, const double* y, const int64_t* ranks,
                              int64_t p, uint64_t root, uint64_t stream, double* core, int64_t* core_shape,
                              double** factors, int64_t* cols) {
    TKO_TRY({
        const Tensor t = to_tensor(shape, order, y);
        const Seed sd{root, stream};
        Tucker m = alg == 2 ? rand_tucker(t, to_shape(ranks, order), p, sd, true)
                            : rand_tucker_2i(t, to_shape(ranks, order), p, sd, nullptr, true);
        write_model(m, core, core_shape, factors, cols);
    })
}
int tko_rand_tucker(const int64_t* shape, int64_t order, const double* y, const int64_t* ranks,
                    int64_t p, uint64_t root, uint64_t stream, double* core, int64_t* core_shape,
                    double** factors, int64_t* cols) {
    TKO_TRY({
        Tucker m = rand_tucker(to_tensor(shape, order, y), to_shape(ranks, order), p, Seed{root, stream});
        write_model(m, core, core_shape, factors, cols);
    })
}
int tko_reconstruct(const int64_t* core_shape, int64_t order, const double* core, const double** factors,
                    const int64_t* rows, double* out) {
    TKO_TRY({
        Tucker m;
        m.core = to_tensor(core_shape, order, core);
        for (int64_t n = 0; n < order; ++n) m.factors.push_back(to_mat(rows[n], core_shape[n], factors[n]));
        Tensor r = reconstruct(m);
        std::memcpy(out, r.data(), sizeof(double) * r.d.size());
    })
}
int tko_fit(const int64_t* shape, int64_t order, const double* y, const double* yhat, double* out) {
    TKO_TRY({ *out = fit(to_tensor(shape, order, y), to_tensor(shape, order, yhat)); })
}
int tko_gen_tucker(const int64_t* dims, const int64_t* mlr, int64_t order, uint64_t root, uint64_t stream,
                   double* out) {
    TKO_TRY({
        Tensor t = gen_tucker_tensor(to_shape(dims, order), to_shape(mlr, order), Seed{root, stream}, nullptr);
        std::memcpy(out, t.data(), sizeof(double) * t.d.size());
    })
}
int tko_gen_cp(const int64_t* dims, int64_t order, int64_t rank, int kind, double zero_frac, uint64_t root,
               uint64_t stream, double* out, double** factors_out) {
    TKO_TRY({
        std::vector<Mat> fs;
        Tensor t = gen_cp_tensor(to_shape(dims, order), rank, kind, zero_frac, Seed{root, stream}, &fs);
        std::memcpy(out, t.data(), sizeof(double) * t.d.size());
        if (factors_out)
            for (int64_t n = 0; n < order; ++n)
                std::memcpy(factors_out[n], fs[static_cast<size_t>(n)].data(), sizeof(double) * fs[static_cast<size_t>(n)].d.size());
    })
}
int tko_add_noise(const int64_t* shape, int64_t order, double* y, double snr_db, uint64_t root,
                  uint64_t stream, int abs_noise) {
    TKO_TRY({
        Tensor t = to_tensor(shape, order, y);
        add_noise(t, snr_db, Seed{root, stream}, abs_noise != 0);
        std::memcpy(y, t.data(), sizeof(double) * t.d.size());
    })
}
int tko_ffcp(const int64_t* core_shape, int64_t order, const double* core, const double** ufactors,
             const int64_t* rows, int64_t rank, int kind, double c, int max_iters, double fit_tol,
             uint64_t root, uint64_t stream, double** out_factors, double* fit_trace, int* iterations) {
    TKO_TRY({
        Tucker m;
        m.core = to_tensor(core_shape, order, core);
        for (int64_t n = 0; n < order; ++n) m.factors.push_back(to_mat(rows[n], core_shape[n], ufactors[n]));
        FfcpOut o = ffcp(m, rank, kind, c, max_iters, fit_tol, Seed{root, stream});
        for (int64_t n = 0; n < order; ++n)
            std::memcpy(out_factors[n], o.factors[static_cast<size_t>(n)].data(), sizeof(double) * o.factors[static_cast<size_t>(n)].d.size());
        std::memcpy(fit_trace, o.fit_trace.data(), sizeof(double) * o.fit_trace.size());
        *iterations = o.iterations;
    })
}
int tko_cp_reconstruct(const int64_t* dims, int64_t order, int64_t rank, const double** factors, double* out) {
    TKO_TRY({
        std::vector<Mat> f;
        for (int64_t n = 0; n < order; ++n) f.push_back(to_mat(dims[n], rank, factors[n]));
        Tensor t = cp_reconstruct(f);
        std::memcpy(out, t.data(), sizeof(double) * t.d.size());
    })
}

}  // extern "C"
