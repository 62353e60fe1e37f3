// ffcp.cpp — FFCP (flexible fast CP on the Tucker-compressed tensor), host fp64.
//
// Reference: ffcp (ffcp.hpp:94-194), ffcp_h (:33-47), solve_normal / hals_sweep /
// absorb_scales (cp.hpp:63-109). The north star keeps FFCP off the hot path: every
// operand is a core-sized tensor (R~^N) or an I_n x R matrix, so it runs on the host
// next to the device decomposition. The compressed-space contractions are organised as
// column-batched products (one pass over the core per mode instead of R passes).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/tenkit_b200.h"
#include "common.cuh"

namespace tkb {
namespace {

struct M {  // column-major dense matrix
    int64_t r = 0, c = 0;
    std::vector<double> d;
    M() = default;
    M(int64_t rr, int64_t cc, double v = 0.0) : r(rr), c(cc), d(size_t(rr * cc), v) {}
    double& operator()(int64_t i, int64_t j) { return d[size_t(i + j * r)]; }
    double operator()(int64_t i, int64_t j) const { return d[size_t(i + j * r)]; }
};

M tn(const M& a, const M& b) {  // a^T b
    M o(a.c, b.c);
    for (int64_t j = 0; j < b.c; ++j)
        for (int64_t i = 0; i < a.c; ++i) {
            double s = 0.0;
            for (int64_t k = 0; k < a.r; ++k) s += a(k, i) * b(k, j);
            o(i, j) = s;
        }
    return o;
}
M nn(const M& a, const M& b) {
    M o(a.r, b.c);
    for (int64_t j = 0; j < b.c; ++j)
        for (int64_t k = 0; k < a.c; ++k) {
            const double bk = b(k, j);
            for (int64_t i = 0; i < a.r; ++i) o(i, j) += a(i, k) * bk;
        }
    return o;
}

// H = unfold(G, n) * KR_{p != n}(V_p): column r is G contracted with v_r^(p) over every
// mode p != n (trailing modes first, as ffcp_h does).
M ffcp_h(const std::vector<int64_t>& shape, const std::vector<double>& g, const std::vector<M>& v, int n, int64_t R) {
    const int order = static_cast<int>(shape.size());
    M h(shape[n], R);
    std::vector<double> cur, nxt;
    for (int64_t r = 0; r < R; ++r) {
        cur = g;
        std::vector<int64_t> cs = shape;
        for (int p = order - 1; p >= 0; --p) {
            if (p == n) continue;
            int64_t before = 1, after = 1;
            for (int q = 0; q < p; ++q) before *= cs[q];
            for (int q = p + 1; q < order; ++q) after *= cs[q];
            nxt.assign(size_t(before * after), 0.0);
            for (int64_t a = 0; a < after; ++a)
                for (int64_t k = 0; k < cs[p]; ++k) {
                    const double w = v[p](k, r);
                    const double* src = cur.data() + (a * cs[p] + k) * before;
                    double* dst = nxt.data() + a * before;
                    for (int64_t b = 0; b < before; ++b) dst[b] += src[b] * w;
                }
            cs[p] = 1;
            cur.swap(nxt);
        }
        std::memcpy(&h(0, r), cur.data(), sizeof(double) * shape[n]);
    }
    return h;
}

bool ldlt_solve(const M& ain, M& bt) {  // Eigen-style LDLT (diagonal pivoting), solves A X = B
    const int64_t n = ain.r;
    M a = ain;
    std::vector<int64_t> tr(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
        int64_t best = k;
        for (int64_t i = k + 1; i < n; ++i)
            if (std::abs(a(i, i)) > std::abs(a(best, best))) best = i;
        tr[size_t(k)] = best;
        if (best != k) {
            for (int64_t j = 0; j < n; ++j) std::swap(a(k, j), a(best, j));
            for (int64_t i = 0; i < n; ++i) std::swap(a(i, k), a(i, best));
        }
        double dk = a(k, k);
        for (int64_t j = 0; j < k; ++j) dk -= a(k, j) * a(k, j) * a(j, j);
        a(k, k) = dk;
        for (int64_t i = k + 1; i < n; ++i) {
            double s = a(i, k);
            for (int64_t j = 0; j < k; ++j) s -= a(i, j) * a(k, j) * a(j, j);
            a(i, k) = std::abs(dk) > 0.0 ? s / dk : s;
        }
    }
    for (int64_t c = 0; c < bt.c; ++c) {
        double* b = &bt(0, c);
        for (int64_t k = 0; k < n; ++k) std::swap(b[k], b[tr[size_t(k)]]);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < i; ++j) b[i] -= a(i, j) * b[j];
        for (int64_t i = 0; i < n; ++i) b[i] = std::abs(a(i, i)) > std::numeric_limits<double>::min() ? b[i] / a(i, i) : 0.0;
        for (int64_t i = n - 1; i >= 0; --i)
            for (int64_t j = i + 1; j < n; ++j) b[i] -= a(j, i) * b[j];
        for (int64_t k = n - 1; k >= 0; --k) std::swap(b[k], b[tr[size_t(k)]]);
    }
    for (double x : bt.d)
        if (!std::isfinite(x)) return false;
    return true;
}

M transpose(const M& a) {
    M t(a.c, a.r);
    for (int64_t j = 0; j < a.c; ++j)
        for (int64_t i = 0; i < a.r; ++i) t(j, i) = a(i, j);
    return t;
}

M solve_normal(const M& q, const M& t) {  // X * T = Q (cp.hpp:63-70)
    M xt = transpose(q);
    if (ldlt_solve(t, xt)) return transpose(xt);
    double tr = 0.0;
    for (int64_t i = 0; i < t.r; ++i) tr += t(i, i);
    M reg = t;
    for (int64_t i = 0; i < t.r; ++i) reg(i, i) += 1e-12 * tr + 1e-300;
    xt = transpose(q);
    ldlt_solve(reg, xt);
    return transpose(xt);
}

}  // namespace
}  // namespace tkb

using namespace tkb;

extern "C" int tk_ffcp(tk_context* /*ctx*/, int64_t order, const int64_t* core_shape, const double* core,
                       const double** factors, const int64_t* rows, int64_t rank, int constraint, double c,
                       int max_iters, double fit_tol, uint64_t seed_root, uint64_t seed_stream,
                       double** out_factors, double* fit_trace, int* iterations) {
    extern int tk_ffcp_fail(int, const char*);
    try {
        require(order >= 2, "ffcp: tensor order must be at least 2");
        require(rank >= 1, "ffcp: rank must be positive");
        require(c >= 0.0, "ffcp: sparsity level must be nonnegative");
        require(constraint >= TK_CP_NONE && constraint <= TK_CP_SPARSE, "ffcp: unknown constraint");
        const bool nonneg = constraint == TK_CP_NONNEG_MU || constraint == TK_CP_NONNEG_HALS;
        std::vector<int64_t> shape(core_shape, core_shape + order);
        int64_t gsz = 1;
        for (int64_t s : shape) {
            require(s >= 1, "tucker model: factor columns must match core shape");
            gsz *= s;
        }
        std::vector<double> g(core, core + gsz);
        const size_t no = static_cast<size_t>(order);
        std::vector<M> U(no), A(no), V(no), G(no);
        const Seed seed{seed_root, seed_stream};
        for (int64_t n = 0; n < order; ++n) {
            U[n] = M(rows[n], shape[n]);
            std::memcpy(U[n].d.data(), factors[n], sizeof(double) * U[n].d.size());
            // initial A_n = gaussian_matrix(rows, R, ffcp_init_seed) (|.| when nonnegative)
            A[n] = M(rows[n], rank);
            const uint64_t key = ffcp_init_seed(seed, n).key();
            const uint64_t cnt = uint64_t(rows[n] * rank);
            for (uint64_t i = 0; i < cnt; i += 2) {
                const double u1 = counter_unit(key, i), u2 = counter_unit(key, i + 1);
                const double rr = std::sqrt(-2.0 * std::log(u1)), ang = 6.283185307179586476925287 * u2;
                A[n].d[i] = rr * std::cos(ang);
                if (i + 1 < cnt) A[n].d[i + 1] = rr * std::sin(ang);
            }
            if (nonneg)
                for (double& x : A[n].d) x = std::abs(x);
            V[n] = tn(U[n], A[n]);
            G[n] = tn(A[n], A[n]);
        }
        // ||Y_T||^2 = <G, G x_n (U^T U)>
        double yt_sq;
        {
            std::vector<double> cur = g, nxt;
            std::vector<int64_t> cs = shape;
            for (int64_t p = 0; p < order; ++p) {
                const M uu = tn(U[p], U[p]);
                int64_t before = 1, after = 1;
                for (int64_t q = 0; q < p; ++q) before *= cs[q];
                for (int64_t q = p + 1; q < order; ++q) after *= cs[q];
                nxt.assign(cur.size(), 0.0);
                for (int64_t a = 0; a < after; ++a)
                    for (int64_t i = 0; i < cs[p]; ++i)
                        for (int64_t k = 0; k < cs[p]; ++k) {
                            const double w = uu(i, k);
                            const double* src = cur.data() + (a * cs[p] + k) * before;
                            double* dst = nxt.data() + (a * cs[p] + i) * before;
                            for (int64_t b = 0; b < before; ++b) dst[b] += w * src[b];
                        }
                cur.swap(nxt);
            }
            double s = 0.0;
            for (int64_t i = 0; i < gsz; ++i) s += g[i] * cur[i];
            yt_sq = std::max(0.0, s);
        }
        const double yt_norm = std::sqrt(yt_sq);
        require(yt_norm > 0.0, "ffcp: compressed tensor has zero norm");
        double prev = -std::numeric_limits<double>::infinity();
        int it = 0;
        for (; it < max_iters;) {
            double res_sq = 0.0;
            for (int64_t n = 0; n < order; ++n) {
                const M h = ffcp_h(shape, g, V, static_cast<int>(n), rank);
                const M q = nn(U[n], h);
                M t(rank, rank, 1.0);
                for (int64_t p = 0; p < order; ++p)
                    if (p != n)
                        for (size_t i = 0; i < t.d.size(); ++i) t.d[i] *= G[p].d[i];
                M& a = A[n];
                if (constraint == TK_CP_NONE) {
                    a = solve_normal(q, t);
                } else if (constraint == TK_CP_NONNEG_MU) {
                    const M at = nn(a, t);
                    for (size_t i = 0; i < a.d.size(); ++i) a.d[i] *= std::max(q.d[i], 0.0) / std::max(at.d[i], 1e-16);
                } else if (constraint == TK_CP_NONNEG_HALS) {
                    std::vector<double> col(static_cast<size_t>(a.r));
                    for (int64_t r = 0; r < a.c; ++r) {
                        const double trr = t(r, r);
                        if (trr < 1e-15) continue;
                        for (int64_t i = 0; i < a.r; ++i) {
                            double at = 0.0;
                            for (int64_t s2 = 0; s2 < a.c; ++s2) at += a(i, s2) * t(s2, r);
                            col[size_t(i)] = std::max(a(i, r) + (q(i, r) - at) / trr, 0.0);
                        }
                        for (int64_t i = 0; i < a.r; ++i) a(i, r) = col[size_t(i)];
                    }
                } else {
                    a = solve_normal(q, t);
                    for (double& x : a.d) x = x > c ? x - c : (x < -c ? x + c : 0.0);
                }
                G[n] = tn(a, a);
                V[n] = tn(U[n], a);
                if (n == order - 1) {
                    double inner = 0.0, msq = 0.0;
                    for (size_t i = 0; i < h.d.size(); ++i) inner += h.d[i] * V[n].d[i];
                    for (size_t i = 0; i < t.d.size(); ++i) msq += t.d[i] * G[n].d[i];
                    res_sq = std::max(0.0, yt_sq - 2.0 * inner + msq);
                }
            }
            const double f = 1.0 - std::sqrt(res_sq) / yt_norm;
            fit_trace[it] = f;
            ++it;
            if (std::abs(f - prev) < fit_tol) break;
            prev = f;
        }
        *iterations = it;
        // absorb_scales (cp.hpp:96-109)
        M& last = A[size_t(order - 1)];
        for (int64_t n = 0; n + 1 < order; ++n)
            for (int64_t r = 0; r < rank; ++r) {
                double nr = 0.0;
                for (int64_t i = 0; i < A[n].r; ++i) nr += A[n](i, r) * A[n](i, r);
                nr = std::sqrt(nr);
                if (nr > 0.0) {
                    for (int64_t i = 0; i < A[n].r; ++i) A[n](i, r) /= nr;
                    for (int64_t i = 0; i < last.r; ++i) last(i, r) *= nr;
                }
            }
        for (int64_t n = 0; n < order; ++n) std::memcpy(out_factors[n], A[n].d.data(), sizeof(double) * A[n].d.size());
        return TK_OK;
    } catch (const InvalidArgument& e) {
        return tk_ffcp_fail(TK_ERR_INVALID, e.what());
    } catch (const std::exception& e) {
        return tk_ffcp_fail(TK_ERR_INTERNAL, e.what());
    }
}
