// eigen_shim.hpp — TEST INFRASTRUCTURE ONLY. A minimal, eager (no expression templates)
// stand-in for the parts of the Eigen 3 API that the reference's hot-path headers use
// (tensor.hpp, random.hpp, range_finder.hpp, tucker.hpp under /root/reference/proj/include/
// tenkit), so those headers compile and RUN here unmodified from where they lie
// (oracle/Makefile target `ref` -> oracle/_ref/libtenkit_ref.so). Eigen itself is absent
// from the image and the reference pins no version.
//
// What is Eigen's arithmetic is replaced by plain fixed-order loops (products, norms) and
// by LAPACK (resolved at run time from the OpenBLAS build numpy ships, see
// eigen_shim_lapack_init): ColPivHouseholderQR -> dgeqp3 (the LAPACK routine Eigen's
// ColPivHouseholderQR restates: column pivoting on the largest updated norm, Householder
// reflectors with beta = -sign(alpha) ||x||), householderQ() -> the reflectors applied
// explicitly; SelfAdjointEigenSolver -> dsyev (ascending eigenvalues, like Eigen);
// BDCSVD -> dgesvd. Nothing here restates the reference's own code.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <dlfcn.h>
#include <stdexcept>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;

enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum UpLoType { Lower = 1, Upper = 2, StrictlyLower = 3, StrictlyUpper = 4 };
enum DecompositionOptions { ComputeThinU = 0x08, ComputeThinV = 0x20 };

// ----------------------------------------------------------------------------- LAPACK
namespace shim {
using i64 = int64_t;
using dgeqp3_fn = void (*)(const i64*, const i64*, double*, const i64*, i64*, double*, double*, const i64*, i64*);
using dsyev_fn = void (*)(const char*, const char*, const i64*, double*, const i64*, double*, double*, const i64*, i64*,
                          size_t, size_t);
using dgesvd_fn = void (*)(const char*, const char*, const i64*, const i64*, double*, const i64*, double*, double*,
                           const i64*, double*, const i64*, double*, const i64*, i64*, size_t, size_t);
struct Lapack {
    dgeqp3_fn dgeqp3 = nullptr;
    dsyev_fn dsyev = nullptr;
    dgesvd_fn dgesvd = nullptr;
};
inline Lapack& lapack() {
    static Lapack l;
    return l;
}
}  // namespace shim

// path: an ILP64 OpenBLAS with the scipy_ symbol prefix (numpy.libs/libscipy_openblas64_*.so)
inline bool eigen_shim_lapack_init(const char* path) {
    void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) return false;
    auto& l = shim::lapack();
    l.dgeqp3 = reinterpret_cast<shim::dgeqp3_fn>(dlsym(h, "scipy_dgeqp3_64_"));
    l.dsyev = reinterpret_cast<shim::dsyev_fn>(dlsym(h, "scipy_dsyev_64_"));
    l.dgesvd = reinterpret_cast<shim::dgesvd_fn>(dlsym(h, "scipy_dgesvd_64_"));
    return l.dgeqp3 && l.dsyev && l.dgesvd;
}

// ----------------------------------------------------------------------------- views
class MatrixXd;

// A (possibly strided) column-major view. Const-ness is the caller's business (the shim
// only writes through views that came from non-const storage).
struct View {
    double* p = nullptr;
    Index r = 0, c = 0, ld = 0;
    double& operator()(Index i, Index j) const { return p[i + j * ld]; }
    double& operator()(Index i) const { return c == 1 ? p[i] : p[i * ld]; }
    Index rows() const { return r; }
    Index cols() const { return c; }
    Index size() const { return r * c; }
};

// eager evaluation: every expression below returns a MatrixXd
class MatrixXd {
public:
    MatrixXd() = default;
    MatrixXd(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), 0.0) {}
    MatrixXd(const View& v) : MatrixXd(v.r, v.c) {  // NOLINT: implicit, as Eigen's expression -> Matrix
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) (*this)(i, j) = v(i, j);
    }
    static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
    static MatrixXd Ones(Index r, Index c) {
        MatrixXd m(r, c);
        std::fill(m.d_.begin(), m.d_.end(), 1.0);
        return m;
    }
    static MatrixXd Identity(Index r, Index c) {
        MatrixXd m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
        return m;
    }
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double* data() { return d_.data(); }
    const double* data() const { return d_.data(); }
    double& operator()(Index i, Index j) { return d_[static_cast<size_t>(i + j * r_)]; }
    double operator()(Index i, Index j) const { return d_[static_cast<size_t>(i + j * r_)]; }
    double& operator()(Index i) { return d_[static_cast<size_t>(i)]; }
    double operator()(Index i) const { return d_[static_cast<size_t>(i)]; }
    void resize(Index r, Index c) {
        r_ = r, c_ = c;
        d_.assign(static_cast<size_t>(r * c), 0.0);
    }
    View view() const { return View{const_cast<double*>(d_.data()), r_, c_, r_}; }

    // blocks (views into this matrix)
    struct Block;
    Block col(Index j) const;
    Block middleCols(Index j, Index n) const;
    Block leftCols(Index n) const;
    Block middleRows(Index i, Index n) const;
    Block block(Index i, Index j, Index r, Index c) const;

    MatrixXd transpose() const;
    MatrixXd cwiseAbs() const {
        MatrixXd m = *this;
        for (double& x : m.d_) x = std::abs(x);
        return m;
    }
    double maxCoeff(Index* at) const {  // first maximum in storage order (vectors)
        Index best = 0;
        for (Index i = 1; i < size(); ++i)
            if (d_[static_cast<size_t>(i)] > d_[static_cast<size_t>(best)]) best = i;
        if (at) *at = best;
        return d_[static_cast<size_t>(best)];
    }
    double squaredNorm() const {
        double s = 0.0;
        for (double x : d_) s += x * x;
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    MatrixXd& noalias() { return *this; }
    MatrixXd& operator+=(const MatrixXd& o) {
        for (size_t i = 0; i < d_.size(); ++i) d_[i] += o.d_[i];
        return *this;
    }
    MatrixXd operator-() const {
        MatrixXd m = *this;
        for (double& x : m.d_) x = -x;
        return m;
    }
    struct ArrayRef;
    ArrayRef array();
    ArrayRef array() const;
    template <int Mode>
    struct SelfAdjoint;
    template <int Mode>
    SelfAdjoint<Mode> selfadjointView() { return SelfAdjoint<Mode>{this}; }
    template <int Mode>
    struct Triangular;
    template <int Mode>
    Triangular<Mode> triangularView() { return Triangular<Mode>{this}; }

protected:
    Index r_ = 0, c_ = 0;
    std::vector<double> d_;
};

class VectorXd : public MatrixXd {
public:
    VectorXd() = default;
    explicit VectorXd(Index n) : MatrixXd(n, 1) {}
    VectorXd(const MatrixXd& m) : MatrixXd(m) {}  // NOLINT
};
using ArrayXd = VectorXd;

// a view with assignment semantics (Eigen Block / Map)
struct MatrixXd::Block : View {
    Block() = default;
    Block(const View& v) : View(v) {}  // NOLINT
    Block& noalias() { return *this; }
    Block& operator=(const MatrixXd& m) {
        if (m.rows() != r || m.cols() != c) throw std::invalid_argument("eigen shim: block assignment shape");
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) (*this)(i, j) = m(i, j);
        return *this;
    }
    Block& operator=(const Block& b) { return *this = MatrixXd(static_cast<const View&>(b)); }
    Block& operator+=(const MatrixXd& m) {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) (*this)(i, j) += m(i, j);
        return *this;
    }
    Block& operator*=(double s) {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) (*this)(i, j) *= s;
        return *this;
    }
    Block& operator/=(double s) {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) (*this)(i, j) /= s;
        return *this;
    }
    MatrixXd transpose() const { return MatrixXd(static_cast<const View&>(*this)).transpose(); }
    MatrixXd cwiseAbs() const { return MatrixXd(static_cast<const View&>(*this)).cwiseAbs(); }
    double norm() const { return MatrixXd(static_cast<const View&>(*this)).norm(); }
    double squaredNorm() const { return MatrixXd(static_cast<const View&>(*this)).squaredNorm(); }
    MatrixXd operator-() const { return -MatrixXd(static_cast<const View&>(*this)); }
    Block reshaped(Index nr, Index nc) const {  // contiguous block only (a column)
        if (nr * nc != r * c || (c > 1 && ld != r)) throw std::invalid_argument("eigen shim: reshaped");
        return Block(View{p, nr, nc, nr});
    }
    Block col(Index j) const { return Block(View{p + j * ld, r, 1, ld}); }
};

inline MatrixXd::Block MatrixXd::col(Index j) const { return block(0, j, r_, 1); }
inline MatrixXd::Block MatrixXd::middleCols(Index j, Index n) const { return block(0, j, r_, n); }
inline MatrixXd::Block MatrixXd::leftCols(Index n) const { return block(0, 0, r_, n); }
inline MatrixXd::Block MatrixXd::middleRows(Index i, Index n) const { return block(i, 0, n, c_); }
inline MatrixXd::Block MatrixXd::block(Index i, Index j, Index r, Index c) const {
    if (i < 0 || j < 0 || i + r > r_ || j + c > c_) throw std::invalid_argument("eigen shim: block out of range");
    return Block(View{const_cast<double*>(d_.data()) + i + j * r_, r, c, r_});
}

inline MatrixXd MatrixXd::transpose() const {
    MatrixXd t(c_, r_);
    for (Index j = 0; j < c_; ++j)
        for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
}

// Map<Matrix> / Map<const Matrix> / Map<const Vector> / Map<ArrayXd> / Map<const ArrayXd>
template <class T>
struct Map : MatrixXd::Block {
    Map(const double* p, Index r, Index c) : MatrixXd::Block(View{const_cast<double*>(p), r, c, r}) {}
    Map(const double* p, Index n) : MatrixXd::Block(View{const_cast<double*>(p), n, 1, n}) {}
    using MatrixXd::Block::operator=;
    Map& operator=(const MatrixXd& m) {
        MatrixXd::Block::operator=(m);
        return *this;
    }
    double minCoeff() const {
        double m = (*this)(0, 0);
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) m = std::min(m, (*this)(i, j));
        return m;
    }
};

// ----------------------------------------------------------------------------- arithmetic
inline MatrixXd as_mat(const MatrixXd& m) { return m; }
inline MatrixXd as_mat(const View& v) { return MatrixXd(v); }

// C = A B, fixed-order loops (j, k, i)
inline MatrixXd matmul(const MatrixXd& a, const MatrixXd& b) {
    if (a.cols() != b.rows()) throw std::invalid_argument("eigen shim: product shape");
    MatrixXd c(a.rows(), b.cols());
    for (Index j = 0; j < b.cols(); ++j)
        for (Index k = 0; k < a.cols(); ++k) {
            const double bkj = b(k, j);
            if (bkj == 0.0) continue;
            for (Index i = 0; i < a.rows(); ++i) c(i, j) += a(i, k) * bkj;
        }
    return c;
}
inline MatrixXd operator*(const MatrixXd& a, const MatrixXd& b) { return matmul(a, b); }
inline MatrixXd operator*(const View& a, const MatrixXd& b) { return matmul(MatrixXd(a), b); }
inline MatrixXd operator*(const MatrixXd& a, const View& b) { return matmul(a, MatrixXd(b)); }
inline MatrixXd operator*(const View& a, const View& b) { return matmul(MatrixXd(a), MatrixXd(b)); }
inline MatrixXd operator*(double s, const MatrixXd& b) {
    MatrixXd m = b;
    for (Index i = 0; i < m.size(); ++i) m(i) *= s;
    return m;
}
inline MatrixXd operator*(double s, const View& b) { return s * MatrixXd(b); }
inline MatrixXd operator/(const MatrixXd& b, double s) {
    MatrixXd m = b;
    for (Index i = 0; i < m.size(); ++i) m(i) /= s;
    return m;
}
inline MatrixXd operator/(const View& b, double s) { return MatrixXd(b) / s; }
inline MatrixXd operator+(const MatrixXd& a, const MatrixXd& b) {
    MatrixXd m = a;
    for (Index i = 0; i < m.size(); ++i) m(i) += b(i);
    return m;
}
inline MatrixXd operator-(const MatrixXd& a, const MatrixXd& b) {
    MatrixXd m = a;
    for (Index i = 0; i < m.size(); ++i) m(i) -= b(i);
    return m;
}
inline MatrixXd operator-(const View& a, const View& b) { return MatrixXd(a) - MatrixXd(b); }

// elementwise (array) views
struct MatrixXd::ArrayRef {
    MatrixXd* m;
    ArrayRef& operator*=(const ArrayRef& o) {
        for (Index i = 0; i < m->size(); ++i) (*m)(i) *= (*o.m)(i);
        return *this;
    }
};
inline MatrixXd::ArrayRef MatrixXd::array() { return ArrayRef{this}; }
inline MatrixXd::ArrayRef MatrixXd::array() const { return ArrayRef{const_cast<MatrixXd*>(this)}; }

// g.selfadjointView<Lower>().rankUpdate(A): lower triangle of g += A A^T
template <int Mode>
struct MatrixXd::SelfAdjoint {
    MatrixXd* g;
    void rankUpdate(const MatrixXd& a) {
        for (Index k = 0; k < a.cols(); ++k)
            for (Index j = 0; j < g->cols(); ++j) {
                const double ajk = a(j, k);
                for (Index i = (Mode == Lower ? j : 0); i < (Mode == Lower ? g->rows() : j + 1); ++i)
                    (*g)(i, j) += a(i, k) * ajk;
            }
    }
};
// g.triangularView<StrictlyUpper>() = m
template <int Mode>
struct MatrixXd::Triangular {
    MatrixXd* g;
    Triangular& operator=(const MatrixXd& m) {
        for (Index j = 0; j < g->cols(); ++j)
            for (Index i = 0; i < g->rows(); ++i) {
                const bool in = Mode == StrictlyUpper ? i < j : Mode == Upper ? i <= j : Mode == StrictlyLower ? i > j : i >= j;
                if (in) (*g)(i, j) = m(i, j);
            }
        return *this;
    }
};

// ----------------------------------------------------------------------------- decompositions
template <class M>
class ColPivHouseholderQR {
public:
    explicit ColPivHouseholderQR(const MatrixXd& z) : qr_(z), tau_(static_cast<size_t>(std::min(z.rows(), z.cols()))) {
        auto& l = shim::lapack();
        if (!l.dgeqp3) throw std::runtime_error("eigen shim: LAPACK not initialised");
        const shim::i64 m = z.rows(), n = z.cols(), lda = std::max<shim::i64>(1, m);
        std::vector<shim::i64> jpvt(static_cast<size_t>(n), 0);
        shim::i64 info = 0, lwork = -1;
        double wq = 0.0;
        l.dgeqp3(&m, &n, qr_.data(), &lda, jpvt.data(), tau_.data(), &wq, &lwork, &info);
        lwork = static_cast<shim::i64>(wq);
        std::vector<double> work(static_cast<size_t>(std::max<shim::i64>(1, lwork)));
        l.dgeqp3(&m, &n, qr_.data(), &lda, jpvt.data(), tau_.data(), work.data(), &lwork, &info);
        if (info != 0) throw std::runtime_error("eigen shim: dgeqp3 failed");
    }
    const MatrixXd& matrixR() const { return qr_; }  // R in the upper triangle (Eigen: matrixQR)
    struct HouseholderSequence {
        const ColPivHouseholderQR* q;
        // H_0 H_1 ... H_{k-1} B (the reflectors applied right to left)
        MatrixXd operator*(const MatrixXd& b) const {
            MatrixXd x = b;
            const MatrixXd& a = q->qr_;
            for (Index k = static_cast<Index>(q->tau_.size()) - 1; k >= 0; --k) {
                const double t = q->tau_[static_cast<size_t>(k)];
                if (t == 0.0) continue;
                for (Index j = 0; j < x.cols(); ++j) {
                    double s = x(k, j);
                    for (Index i = k + 1; i < a.rows(); ++i) s += a(i, k) * x(i, j);
                    s *= t;
                    x(k, j) -= s;
                    for (Index i = k + 1; i < a.rows(); ++i) x(i, j) -= s * a(i, k);
                }
            }
            return x;
        }
    };
    HouseholderSequence householderQ() const { return HouseholderSequence{this}; }

private:
    MatrixXd qr_;
    std::vector<double> tau_;
};

template <class M>
class SelfAdjointEigenSolver {
public:
    explicit SelfAdjointEigenSolver(const MatrixXd& a) : vec_(a), val_(a.rows()) {
        auto& l = shim::lapack();
        if (!l.dsyev) throw std::runtime_error("eigen shim: LAPACK not initialised");
        const shim::i64 n = a.rows(), lda = std::max<shim::i64>(1, n);
        shim::i64 info = 0, lwork = -1;
        double wq = 0.0;
        l.dsyev("V", "L", &n, vec_.data(), &lda, val_.data(), &wq, &lwork, &info, 1, 1);
        lwork = static_cast<shim::i64>(wq);
        std::vector<double> work(static_cast<size_t>(std::max<shim::i64>(1, lwork)));
        l.dsyev("V", "L", &n, vec_.data(), &lda, val_.data(), work.data(), &lwork, &info, 1, 1);
        info_ = info == 0 ? Success : NoConvergence;
    }
    ComputationInfo info() const { return info_; }
    const VectorXd& eigenvalues() const { return val_; }  // ascending
    const MatrixXd& eigenvectors() const { return vec_; }

private:
    MatrixXd vec_;
    VectorXd val_;
    ComputationInfo info_ = Success;
};

template <class M>
class BDCSVD {
public:
    BDCSVD(const MatrixXd& a, int /*options*/) {
        auto& l = shim::lapack();
        if (!l.dgesvd) throw std::runtime_error("eigen shim: LAPACK not initialised");
        MatrixXd w = a;
        const shim::i64 m = a.rows(), n = a.cols(), lda = std::max<shim::i64>(1, m), k = std::min(m, n);
        u_.resize(m, k);
        std::vector<double> s(static_cast<size_t>(k));
        shim::i64 info = 0, lwork = -1, ldu = std::max<shim::i64>(1, m), ldvt = 1;
        double wq = 0.0, vt = 0.0;
        l.dgesvd("S", "N", &m, &n, w.data(), &lda, s.data(), u_.data(), &ldu, &vt, &ldvt, &wq, &lwork, &info, 1, 1);
        lwork = static_cast<shim::i64>(wq);
        std::vector<double> work(static_cast<size_t>(std::max<shim::i64>(1, lwork)));
        l.dgesvd("S", "N", &m, &n, w.data(), &lda, s.data(), u_.data(), &ldu, &vt, &ldvt, work.data(), &lwork, &info,
                 1, 1);
        if (info != 0) throw std::runtime_error("eigen shim: dgesvd failed");
    }
    const MatrixXd& matrixU() const { return u_; }

private:
    MatrixXd u_;
};

}  // namespace Eigen
