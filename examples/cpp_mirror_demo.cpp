// Reference-style caller of the C++ mirror (include/tenkit_b200.hpp): the same code a
// tenkit user writes (bench.hpp:505-506 calls rand_tucker_2i then ffcp), with only the
// include and namespace changed. Prints the Tucker core norm, factor shapes and the FFCP
// fit trace so tests/test_cpp_mirror.py can compare them with the oracle.
//   usage: cpp_mirror_demo I J K R p ffcp_rank   (data: seeded N(0,1) Tucker + noise-free)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "tenkit_b200.hpp"

namespace tenkit = tenkit_b200;

int main(int argc, char** argv) {
    if (argc < 7) {
        std::fprintf(stderr, "usage: %s I J K R p ffcp_rank\n", argv[0]);
        return 2;
    }
    const tenkit::Index I = std::atoll(argv[1]), J = std::atoll(argv[2]), K = std::atoll(argv[3]);
    const tenkit::Index R = std::atoll(argv[4]), p = std::atoll(argv[5]), cr = std::atoll(argv[6]);
    try {
        // Y = G x1 A x2 B x3 C from the counter RNG (core 3x3x3, factors N(0,1)).
        const tenkit::SeedSpec data{0, 0};
        tenkit::Matrix a = tenkit::gaussian_matrix(I, 3, data.derived(1));
        tenkit::Matrix b = tenkit::gaussian_matrix(J, 3, data.derived(2));
        tenkit::Matrix c = tenkit::gaussian_matrix(K, 3, data.derived(3));
        tenkit::Matrix g = tenkit::gaussian_matrix(27, 1, data.derived(4));
        tenkit::DenseTensor core({3, 3, 3}, std::vector<double>(g.data(), g.data() + 27));
        tenkit::DenseTensor y = tenkit::ttm_all(core, {a, b, c}, -1, /*transpose=*/false);
        tenkit::TuckerModel m = tenkit::rand_tucker_2i(y, {R, R, R}, p, tenkit::SeedSpec{7, 0});
        double gsq = 0.0;
        for (tenkit::Index i = 0; i < m.core.size(); ++i) gsq += m.core[i] * m.core[i];
        double ysq = 0.0;
        for (tenkit::Index i = 0; i < y.size(); ++i) ysq += y[i] * y[i];
        std::printf("core_sq %.17g\ny_sq %.17g\n", gsq, ysq);
        for (const auto& u : m.factors) std::printf("factor %lld %lld\n", (long long)u.rows(), (long long)u.cols());
        tenkit::FfcpResult f = tenkit::ffcp(m, cr, tenkit::ConstraintSpec{}, tenkit::StopRule{30, 0.0}, {8, 0});
        std::printf("iterations %d\n", f.iterations);
        for (double v : f.fit_trace) std::printf("fit %.17g\n", v);
        // the distributed protocol's basis on two row blocks of a sketch (range_finder.hpp:48-84)
        tenkit::Matrix z = tenkit::gaussian_matrix(40, 5, tenkit::SeedSpec{6, 0});
        tenkit::Matrix z0(15, 5), z1(25, 5);
        for (tenkit::Index j = 0; j < 5; ++j)
            for (tenkit::Index i = 0; i < 40; ++i) (i < 15 ? z0(i, j) : z1(i - 15, j)) = z(i, j);
        tenkit::GramOrthoResult gr = tenkit::gram_orthonormalize({z0, z1});
        double defect = 0.0;
        for (tenkit::Index a = 0; a < 5; ++a)
            for (tenkit::Index c = 0; c < 5; ++c) {
                double d = 0.0;
                for (const auto& blk : gr.blocks)
                    for (tenkit::Index i = 0; i < blk.rows(); ++i) d += blk(i, a) * blk(i, c);
                defect = std::max(defect, std::abs(d - (a == c ? 1.0 : 0.0)));
            }
        std::printf("gram_kept %zu\ngram_defect %.3e\n", gr.spectrum.size(), defect);
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument: %s\n", e.what());
        return 3;
    } catch (const std::runtime_error& e) {
        std::printf("runtime_error: %s\n", e.what());
        return 4;
    }
    return 0;
}
