// tenkit_b200.hpp — C++ host mirror of the reference's hot-path API over the C-ABI.
//
// The reference (`tenkit`, header-only C++20) is called as free functions with value
// semantics on owning, column-major containers. This header restates that
// surface — same type names, member names, argument meaning and exception types — on top
// of include/tenkit_b200.h, so a reference caller switches by changing the include and
// the namespace (`namespace tenkit = tenkit_b200;`). Compute runs on the B200; there is
// no CPU path (every call throws std::runtime_error without a device).
//
//   DenseTensor            tensor.hpp:32-97        (plus DenseTensorF: fp32 data, cfgs 2-5)
//   TuckerModel            tucker.hpp:14-33
//   CpModel                cp.hpp:17-30
//   SeedSpec               random.hpp:29-44
//   StopRule               cp.hpp:38-41
//   ConstraintKind/Spec    ffcp.hpp:12-17
//   FfcpResult             ffcp.hpp:81-86 (without the per-sweep wall-clock records)
//   rand_tucker_2i         tucker.hpp:136-169
//   rand_tucker            tucker.hpp:108-130
//   ffcp                   ffcp.hpp:94-194
//   ttm / ttm_all / unfold_times   tensor.hpp:151-209
//   orthonormal_basis      range_finder.hpp:18-29 (+ fix_column_signs, tucker.hpp:39-45)
//   gram_orthonormalize    range_finder.hpp:48-84 (GramOrthoResult, range_finder.hpp:38-41)
//   gram_ortho_transform   range_finder.hpp:86-105
//   gaussian_matrix        random.hpp:85-100
//
// Errors: TK_ERR_INVALID -> std::invalid_argument, anything else -> std::runtime_error,
// with tk_last_error()'s "tenkit: ..." message (tensor.hpp:20-22).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tenkit_b200.h"

namespace tenkit_b200 {

using Index = std::int64_t;

namespace detail {

inline void check(int rc) {
    if (rc == TK_OK) return;
    const char* m = tk_last_error();
    const std::string msg = (m && *m) ? m : "tenkit: error " + std::to_string(rc);
    if (rc == TK_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline void require(bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(std::string("tenkit: ") + what);
}

inline void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("tenkit: ") + cudaGetErrorString(e));
}

inline Index shape_product(const std::vector<Index>& s) {
    Index p = 1;
    for (Index d : s) p *= d;
    return p;
}

inline std::uint64_t mix64(std::uint64_t x) {  // random.hpp:12-18
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

inline std::uint64_t hash_combine(std::uint64_t a, std::uint64_t b) {  // random.hpp:20-22
    return mix64(a ^ (mix64(b) + 0x9E3779B97F4A7C15ull + (a << 6) + (a >> 2)));
}

// Owning device buffer (RAII), used to stage kernel-level calls.
template <class T>
struct DeviceBuffer {
    T* p = nullptr;
    explicit DeviceBuffer(std::size_t n) {
        if (n) cuda(cudaMalloc(reinterpret_cast<void**>(&p), n * sizeof(T)));
    }
    DeviceBuffer(const T* host, std::size_t n) : DeviceBuffer(n) {
        if (n) cuda(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice));
    }
    ~DeviceBuffer() {
        if (p) cudaFree(p);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    void to_host(T* host, std::size_t n) const {
        if (n) cuda(cudaMemcpy(host, p, n * sizeof(T), cudaMemcpyDeviceToHost));
    }
};

}  // namespace detail

/// Column-major dense matrix (the reference's Eigen::MatrixXd, tensor.hpp:15).
class Matrix {
public:
    Matrix() = default;
    Matrix(Index rows, Index cols) : rows_(rows), cols_(cols), data_(static_cast<std::size_t>(rows * cols), 0.0) {
        detail::require(rows >= 0 && cols >= 0, "matrix dimensions must be nonnegative");
    }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index size() const { return rows_ * cols_; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    double operator()(Index i, Index j) const { return data_[static_cast<std::size_t>(j * rows_ + i)]; }
    double& operator()(Index i, Index j) { return data_[static_cast<std::size_t>(j * rows_ + i)]; }
    Matrix transpose() const {
        Matrix t(cols_, rows_);
        for (Index j = 0; j < cols_; ++j)
            for (Index i = 0; i < rows_; ++i) t(j, i) = (*this)(i, j);
        return t;
    }

private:
    Index rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

/// Dense N-way array, column-major (tensor.hpp:32-97). T = double is the reference's
/// DenseTensor; T = float holds the fp32 data of cfgs 2-5.
template <class T>
class BasicDenseTensor {
public:
    using value_type = T;
    BasicDenseTensor() = default;
    explicit BasicDenseTensor(std::vector<Index> shape) : shape_(std::move(shape)), data_(check_shape(shape_), T(0)) {}
    BasicDenseTensor(std::vector<Index> shape, std::vector<T> data) : shape_(std::move(shape)), data_(std::move(data)) {
        detail::require(static_cast<Index>(data_.size()) == check_shape(shape_), "tensor data length does not match shape");
    }
    Index order() const { return static_cast<Index>(shape_.size()); }
    const std::vector<Index>& shape() const { return shape_; }
    Index dim(Index mode) const { return shape_.at(static_cast<std::size_t>(mode)); }
    Index size() const { return static_cast<Index>(data_.size()); }
    T* data() { return data_.data(); }
    const T* data() const { return data_.data(); }
    std::vector<T>& storage() { return data_; }
    const std::vector<T>& storage() const { return data_; }
    T operator[](Index i) const { return data_[static_cast<std::size_t>(i)]; }
    T& operator[](Index i) { return data_[static_cast<std::size_t>(i)]; }
    T at(const std::vector<Index>& subs) const { return data_[flat_index(subs)]; }
    T& at(const std::vector<Index>& subs) { return data_[flat_index(subs)]; }
    bool same_shape(const BasicDenseTensor& o) const { return shape_ == o.shape_; }

private:
    static Index check_shape(const std::vector<Index>& shape) {
        detail::require(!shape.empty(), "tensor order must be at least 1");
        for (Index d : shape) detail::require(d >= 1, "tensor dimensions must be positive");
        return detail::shape_product(shape);
    }
    std::size_t flat_index(const std::vector<Index>& subs) const {
        detail::require(subs.size() == shape_.size(), "subscript order mismatch");
        Index flat = 0, stride = 1;
        for (std::size_t k = 0; k < shape_.size(); ++k) {
            detail::require(subs[k] >= 0 && subs[k] < shape_[k], "subscript out of range");
            flat += subs[k] * stride;
            stride *= shape_[k];
        }
        return static_cast<std::size_t>(flat);
    }
    std::vector<Index> shape_;
    std::vector<T> data_;
};

using DenseTensor = BasicDenseTensor<double>;
using DenseTensorF = BasicDenseTensor<float>;

struct TuckerModel {  // tucker.hpp:14-33
    DenseTensor core;
    std::vector<Matrix> factors;
    Index order() const { return core.order(); }
    void validate() const {
        detail::require(static_cast<Index>(factors.size()) == core.order(), "tucker model: one factor per mode required");
        for (Index n = 0; n < core.order(); ++n)
            detail::require(factors[static_cast<std::size_t>(n)].cols() == core.dim(n),
                            "tucker model: factor columns must match core shape");
    }
    std::vector<Index> full_shape() const {
        std::vector<Index> s(factors.size());
        for (std::size_t n = 0; n < factors.size(); ++n) s[n] = factors[n].rows();
        return s;
    }
};

struct CpModel {  // cp.hpp:17-30
    std::vector<Matrix> factors;
    Index order() const { return static_cast<Index>(factors.size()); }
    Index rank() const { return factors.empty() ? 0 : factors.front().cols(); }
};

struct SeedSpec {  // random.hpp:29-44
    std::uint64_t root = 0;
    std::uint64_t stream = 0;
    SeedSpec with_stream(std::uint64_t s) const { return {root, s}; }
    SeedSpec derived(std::uint64_t tag) const { return {root, tk_seed_derived(root, stream, tag)}; }
    SeedSpec derived(std::uint64_t a, std::uint64_t b) const { return derived(a).derived(b); }
    std::uint64_t key() const { return detail::hash_combine(detail::mix64(root), stream); }
};

struct StopRule {  // cp.hpp:38-41
    int max_iters = 1000;
    double fit_tol = 1e-6;
};

enum class ConstraintKind { none, nonneg_mu, nonneg_hals, sparse };  // ffcp.hpp:12

struct ConstraintSpec {  // ffcp.hpp:14-17
    ConstraintKind kind = ConstraintKind::none;
    double sparsity_c = 0.0;
};

struct FfcpResult {  // ffcp.hpp:81-86
    CpModel model;
    std::vector<double> fit_trace;
    int iterations = 0;
};

/// One library context (CUDA stream + buffer pool) per host thread, created on first use.
class Device {
public:
    static tk_context* context() {
        thread_local Device d;
        return d.ctx_.get();
    }

private:
    struct Del {
        void operator()(tk_context* c) const { tk_context_destroy(c); }
    };
    Device() {
        tk_context* c = nullptr;
        detail::check(tk_context_create(-1, &c));
        ctx_.reset(c);
    }
    std::unique_ptr<tk_context, Del> ctx_;
};

namespace detail {

template <class T>
constexpr int dtype_of() {
    return sizeof(T) == 4 ? TK_F32 : TK_F64;
}

template <class T>
TuckerModel tucker_call(bool two_pass, const BasicDenseTensor<T>& y, const std::vector<Index>& ranks, Index oversample,
                        const SeedSpec& seed) {
    const Index N = y.order();
    require(static_cast<Index>(ranks.size()) == N, two_pass ? "rand_tucker_2i: one rank per mode required"
                                                            : "rand_tucker: one rank per mode required");
    require(N >= 1 && N <= TK_MAX_ORDER, "tensor order out of range");
    std::vector<Index> rt(N);
    Index core_cap = 1;
    for (Index n = 0; n < N; ++n) {
        rt[n] = std::min<Index>(ranks[n] + oversample, y.dim(n));
        core_cap *= std::max<Index>(rt[n], 1);
    }
    std::vector<double> core(static_cast<std::size_t>(core_cap));
    std::vector<std::vector<double>> fac(N);
    tk_tucker_out out{};
    out.on_device = 0;
    out.core = core.data();
    for (Index n = 0; n < N; ++n) {
        fac[n].resize(static_cast<std::size_t>(y.dim(n) * std::max<Index>(rt[n], 1)));
        out.factors[n] = fac[n].data();
    }
    tk_context* ctx = Device::context();
    if (two_pass) {
        tk_tucker_opts opts{0, 1, 0, 1, 0, 0};
        check(tk_rand_tucker_2i(ctx, dtype_of<T>(), N, y.shape().data(), y.data(), 0, ranks.data(), oversample,
                                seed.root, seed.stream, &opts, &out, nullptr));
    } else {
        check(tk_rand_tucker(ctx, dtype_of<T>(), N, y.shape().data(), y.data(), 0, ranks.data(), oversample, seed.root,
                             seed.stream, &out, nullptr));
    }
    TuckerModel m;
    std::vector<Index> cs(out.core_shape, out.core_shape + N);
    core.resize(static_cast<std::size_t>(shape_product(cs)));
    m.core = DenseTensor(cs, std::move(core));
    for (Index n = 0; n < N; ++n) {
        Matrix u(y.dim(n), out.factor_cols[n]);
        std::copy(fac[n].begin(), fac[n].begin() + u.size(), u.data());
        m.factors.push_back(std::move(u));
    }
    return m;
}

}  // namespace detail

/// Alg. 3, two passes per mode (tucker.hpp:136-169).
template <class T>
TuckerModel rand_tucker_2i(const BasicDenseTensor<T>& y, const std::vector<Index>& ranks, Index oversample,
                           const SeedSpec& seed) {
    return detail::tucker_call(true, y, ranks, oversample, seed);
}

/// Alg. 2, one pass per mode (tucker.hpp:108-130).
template <class T>
TuckerModel rand_tucker(const BasicDenseTensor<T>& y, const std::vector<Index>& ranks, Index oversample,
                        const SeedSpec& seed) {
    return detail::tucker_call(false, y, ranks, oversample, seed);
}

/// FFCP on a Tucker model (ffcp.hpp:94-194); fit in compressed space.
inline FfcpResult ffcp(const TuckerModel& model, Index rank, const ConstraintSpec& constraint, const StopRule& stop,
                       const SeedSpec& seed) {
    model.validate();
    const Index N = model.order();
    std::vector<const double*> fs(N);
    std::vector<Index> rows(N);
    FfcpResult r;
    r.model.factors.resize(N);
    std::vector<double*> outs(N);
    for (Index n = 0; n < N; ++n) {
        fs[n] = model.factors[n].data();
        rows[n] = model.factors[n].rows();
        r.model.factors[n] = Matrix(rows[n], rank);
        outs[n] = r.model.factors[n].data();
    }
    r.fit_trace.resize(static_cast<std::size_t>(std::max(stop.max_iters, 0)));
    detail::check(tk_ffcp(Device::context(), N, model.core.shape().data(), model.core.data(), fs.data(), rows.data(),
                          rank, static_cast<int>(constraint.kind), constraint.sparsity_c, stop.max_iters, stop.fit_tol,
                          seed.root, seed.stream, outs.data(), r.fit_trace.data(), &r.iterations));
    r.fit_trace.resize(static_cast<std::size_t>(r.iterations));
    return r;
}

/// N(0,1) matrix from the counter RNG, column-major counter order (random.hpp:85-100).
inline Matrix gaussian_matrix(Index rows, Index cols, const SeedSpec& seed) {
    detail::require(rows >= 1 && cols >= 1, "gaussian_matrix: dimensions must be positive");
    Matrix m(rows, cols);
    detail::DeviceBuffer<double> d(static_cast<std::size_t>(m.size()));
    detail::check(tk_gaussian_matrix(Device::context(), rows, cols, seed.root, seed.stream, d.p));
    detail::check(tk_context_synchronize(Device::context()));
    d.to_host(m.data(), static_cast<std::size_t>(m.size()));
    return m;
}

/// Column-pivoted QR basis, rank cut 1e-12|R_00|, pivot-ordered Q (range_finder.hpp:18-29),
/// with the Tucker sign rule applied (tucker.hpp:39-45).
inline Matrix orthonormal_basis(const Matrix& z) {
    detail::require(z.rows() >= 1 && z.cols() >= 1, "orthonormal_basis: empty matrix");
    detail::DeviceBuffer<double> dz(z.data(), static_cast<std::size_t>(z.size()));
    detail::DeviceBuffer<double> dq(static_cast<std::size_t>(z.size()));
    Index rank = 0;
    detail::check(tk_orthonormal_basis(Device::context(), z.rows(), z.cols(), dz.p, dq.p, &rank, nullptr));
    Matrix q(z.rows(), rank);
    dq.to_host(q.data(), static_cast<std::size_t>(q.size()));
    return q;
}

/// Gram-path result (range_finder.hpp:38-41): the orthonormalised row blocks and the kept
/// eigenvalues, descending.
struct GramOrthoResult {
    std::vector<Matrix> blocks;
    std::vector<double> spectrum;
};

/// gram_orthonormalize (range_finder.hpp:48-84): sum_s Z_s^T Z_s = U S U^T, blocks Z_s U S^-1/2
/// (eigenvalues <= 1e-12 top dropped); eigenvector signs are the device eigensolver's.
inline GramOrthoResult gram_orthonormalize(const std::vector<Matrix>& z_blocks) {
    detail::require(!z_blocks.empty(), "gram_orthonormalize: no blocks");
    const Index r = z_blocks.front().cols();
    Index rows = 0;
    for (const Matrix& z : z_blocks) {
        detail::require(z.cols() == r, "gram_orthonormalize: column-count mismatch");
        rows += z.rows();
    }
    Matrix stacked(rows, r);
    Index at = 0;
    for (const Matrix& z : z_blocks) {
        for (Index j = 0; j < r; ++j)
            for (Index i = 0; i < z.rows(); ++i) stacked(at + i, j) = z(i, j);
        at += z.rows();
    }
    detail::DeviceBuffer<double> dz(stacked.data(), static_cast<std::size_t>(stacked.size()));
    detail::DeviceBuffer<double> du(static_cast<std::size_t>(stacked.size()));
    detail::DeviceBuffer<double> ds(static_cast<std::size_t>(r));
    Index kept = 0;
    detail::check(tk_gram_orthonormalize(Device::context(), rows, r, dz.p, du.p, ds.p, &kept));
    Matrix u(rows, kept);
    du.to_host(u.data(), static_cast<std::size_t>(u.size()));
    GramOrthoResult out;
    out.spectrum.resize(static_cast<std::size_t>(r));
    ds.to_host(out.spectrum.data(), out.spectrum.size());
    out.spectrum.resize(static_cast<std::size_t>(kept));
    at = 0;
    for (const Matrix& z : z_blocks) {
        Matrix b(z.rows(), kept);
        for (Index j = 0; j < kept; ++j)
            for (Index i = 0; i < z.rows(); ++i) b(i, j) = u(at + i, j);
        out.blocks.push_back(std::move(b));
        at += z.rows();
    }
    return out;
}

/// gram_ortho_transform (range_finder.hpp:86-105): T (n x kept) with stacked-Z * T orthonormal.
inline std::pair<Matrix, std::vector<double>> gram_ortho_transform(const Matrix& gram_sum) {
    detail::require(gram_sum.rows() == gram_sum.cols() && gram_sum.rows() >= 1,
                    "gram_ortho_transform: square Gram matrix required");
    const Index n = gram_sum.rows();
    detail::DeviceBuffer<double> dg(gram_sum.data(), static_cast<std::size_t>(gram_sum.size()));
    detail::DeviceBuffer<double> dt(static_cast<std::size_t>(n * n));
    detail::DeviceBuffer<double> ds(static_cast<std::size_t>(n));
    Index kept = 0;
    detail::check(tk_gram_ortho_transform(Device::context(), n, dg.p, dt.p, ds.p, &kept));
    Matrix t(n, kept);
    dt.to_host(t.data(), static_cast<std::size_t>(t.size()));
    std::vector<double> sp(static_cast<std::size_t>(n));
    ds.to_host(sp.data(), sp.size());
    sp.resize(static_cast<std::size_t>(kept));
    return {std::move(t), std::move(sp)};
}

/// out = t x_mode m (tensor.hpp:151-176).
inline DenseTensor ttm(const DenseTensor& t, const Matrix& m, Index mode) {
    detail::require(mode >= 0 && mode < t.order(), "mode index out of range");
    detail::require(m.cols() == t.dim(mode), "ttm: matrix columns must match tensor dimension");
    std::vector<Index> os = t.shape();
    os[static_cast<std::size_t>(mode)] = m.rows();
    DenseTensor out(os);
    detail::DeviceBuffer<double> dt(t.data(), static_cast<std::size_t>(t.size()));
    detail::DeviceBuffer<double> dm(m.data(), static_cast<std::size_t>(m.size()));
    detail::DeviceBuffer<double> dout(static_cast<std::size_t>(out.size()));
    detail::check(tk_ttm(Device::context(), TK_F64, t.order(), t.shape().data(), dt.p, m.rows(), dm.p, mode, dout.p));
    detail::check(tk_context_synchronize(Device::context()));
    dout.to_host(out.data(), static_cast<std::size_t>(out.size()));
    return out;
}

/// t x_{n != skip} ms[n]^T (transpose) or ms[n] (tensor.hpp:181-192).
inline DenseTensor ttm_all(const DenseTensor& t, const std::vector<Matrix>& ms, Index skip = -1, bool transpose = true) {
    const Index N = t.order();
    detail::require(static_cast<Index>(ms.size()) == N, "ttm_all: one matrix per mode required");
    std::vector<Matrix> tr;  // the C-ABI applies dims[n] x cols[n] matrices transposed
    std::vector<std::unique_ptr<detail::DeviceBuffer<double>>> dms;
    std::vector<const double*> ptrs(N, nullptr);
    std::vector<Index> cols(N, 0);
    std::vector<Index> os = t.shape();
    for (Index n = 0; n < N; ++n) {
        if (n == skip) continue;
        const Matrix& m = transpose ? ms[n] : (tr.push_back(ms[n].transpose()), tr.back());
        detail::require(m.rows() == t.dim(n), "ttm_all: matrix rows must match tensor dimension");
        dms.emplace_back(new detail::DeviceBuffer<double>(m.data(), static_cast<std::size_t>(m.size())));
        ptrs[n] = dms.back()->p;
        cols[n] = m.cols();
        os[n] = m.cols();
    }
    DenseTensor out(os);
    detail::DeviceBuffer<double> dt(t.data(), static_cast<std::size_t>(t.size()));
    detail::DeviceBuffer<double> dout(static_cast<std::size_t>(out.size()));
    detail::check(tk_ttm_all(Device::context(), TK_F64, N, t.shape().data(), dt.p, ptrs.data(), cols.data(), skip, dout.p));
    detail::check(tk_context_synchronize(Device::context()));
    dout.to_host(out.data(), static_cast<std::size_t>(out.size()));
    return out;
}

/// unfold(t, mode) * b without materialising the unfolding (tensor.hpp:195-209).
inline Matrix unfold_times(const DenseTensor& t, Index mode, const Matrix& b) {
    detail::require(mode >= 0 && mode < t.order(), "mode index out of range");
    detail::require(b.rows() * t.dim(mode) == t.size(), "unfold_times: inner dimensions must agree");
    Matrix z(t.dim(mode), b.cols());
    detail::DeviceBuffer<double> dt(t.data(), static_cast<std::size_t>(t.size()));
    detail::DeviceBuffer<double> db(b.data(), static_cast<std::size_t>(b.size()));
    detail::DeviceBuffer<double> dz(static_cast<std::size_t>(z.size()));
    detail::check(tk_unfold_times(Device::context(), TK_F64, t.order(), t.shape().data(), dt.p, mode, db.p, b.cols(), dz.p));
    detail::check(tk_context_synchronize(Device::context()));
    dz.to_host(z.data(), static_cast<std::size_t>(z.size()));
    return z;
}

}  // namespace tenkit_b200
