// ref_entry.cpp — TEST INFRASTRUCTURE ONLY: the reference's own hot-path code, compiled from
// where it lies (/root/reference/proj/include/tenkit/{tensor,random,range_finder,tucker}.hpp,
// unmodified) against oracle/ref_shim (a minimal eager Eigen-API stand-in over LAPACK), and
// exposed through a C API for generating reference-run fixtures (tests/golden/make_ref_fixtures.py).
// Built only where /root/reference exists (oracle/Makefile target `ref` -> oracle/_ref/); the
// fixtures it produces are committed, the library itself is not.
#include <tenkit/tucker.hpp>

#include <cstring>
#include <string>

namespace {
thread_local std::string g_err;

tenkit::DenseTensor to_tensor(const int64_t* shape, int64_t order, const double* y) {
    std::vector<tenkit::Index> s(shape, shape + order);
    tenkit::DenseTensor t(s);
    std::memcpy(t.data(), y, sizeof(double) * static_cast<size_t>(t.size()));
    return t;
}

tenkit::Matrix to_mat(int64_t r, int64_t c, const double* d) {
    tenkit::Matrix m(r, c);
    std::memcpy(m.data(), d, sizeof(double) * static_cast<size_t>(r * c));
    return m;
}

void write_model(const tenkit::TuckerModel& m, double* core, int64_t* core_shape, double** factors, int64_t* cols) {
    std::memcpy(core, m.core.data(), sizeof(double) * static_cast<size_t>(m.core.size()));
    for (size_t n = 0; n < m.factors.size(); ++n) {
        core_shape[n] = m.core.dim(static_cast<tenkit::Index>(n));
        cols[n] = m.factors[n].cols();
        std::memcpy(factors[n], m.factors[n].data(), sizeof(double) * static_cast<size_t>(m.factors[n].size()));
    }
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}
}  // namespace

extern "C" {

const char* tkr_last_error() { return g_err.c_str(); }

int tkr_init(const char* openblas_path) { return Eigen::eigen_shim_lapack_init(openblas_path) ? 0 : 2; }

double tkr_normal_at(uint64_t root, uint64_t stream, uint64_t idx) {
    return tenkit::normal_at(tenkit::SeedSpec{root, stream}, idx);
}

uint64_t tkr_seed_derived(uint64_t root, uint64_t stream, uint64_t tag) {
    return tenkit::SeedSpec{root, stream}.derived(tag).stream;
}

int tkr_gaussian_matrix(int64_t rows, int64_t cols, uint64_t root, uint64_t stream, double* out) {
    return guarded([&] {
        const tenkit::Matrix m = tenkit::gaussian_matrix(rows, cols, tenkit::SeedSpec{root, stream});
        std::memcpy(out, m.data(), sizeof(double) * static_cast<size_t>(m.size()));
    });
}

int tkr_ttm(const int64_t* shape, int64_t order, const double* t, int64_t mrows, int64_t mcols, const double* m,
            int64_t mode, double* out) {
    return guarded([&] {
        const tenkit::DenseTensor r = tenkit::ttm(to_tensor(shape, order, t), to_mat(mrows, mcols, m), mode);
        std::memcpy(out, r.data(), sizeof(double) * static_cast<size_t>(r.size()));
    });
}

int tkr_unfold_times(const int64_t* shape, int64_t order, const double* t, int64_t mode, int64_t brows,
                     int64_t bcols, const double* b, double* out) {
    return guarded([&] {
        const tenkit::Matrix z = tenkit::unfold_times(to_tensor(shape, order, t), mode, to_mat(brows, bcols, b));
        std::memcpy(out, z.data(), sizeof(double) * static_cast<size_t>(z.size()));
    });
}

// orthonormal_basis + fix_column_signs (what every Tucker factor goes through)
int tkr_orthonormal_basis(int64_t rows, int64_t cols, const double* z, double* q, int64_t* rank) {
    return guarded([&] {
        tenkit::Matrix u = tenkit::orthonormal_basis(to_mat(rows, cols, z));
        tenkit::detail::fix_column_signs(u);
        *rank = u.cols();
        std::memcpy(q, u.data(), sizeof(double) * static_cast<size_t>(u.size()));
    });
}

int tkr_rand_tucker_2i(const int64_t* shape, int64_t order, const double* y, const int64_t* ranks, int64_t p,
                       uint64_t root, uint64_t stream, double* core, int64_t* core_shape, double** factors,
                       int64_t* cols) {
    return guarded([&] {
        const tenkit::TuckerModel m = tenkit::rand_tucker_2i(
            to_tensor(shape, order, y), std::vector<tenkit::Index>(ranks, ranks + order), p, tenkit::SeedSpec{root, stream});
        write_model(m, core, core_shape, factors, cols);
    });
}

int tkr_rand_tucker(const int64_t* shape, int64_t order, const double* y, const int64_t* ranks, int64_t p,
                    uint64_t root, uint64_t stream, double* core, int64_t* core_shape, double** factors,
                    int64_t* cols) {
    return guarded([&] {
        const tenkit::TuckerModel m = tenkit::rand_tucker(
            to_tensor(shape, order, y), std::vector<tenkit::Index>(ranks, ranks + order), p, tenkit::SeedSpec{root, stream});
        write_model(m, core, core_shape, factors, cols);
    });
}

}  // extern "C"
