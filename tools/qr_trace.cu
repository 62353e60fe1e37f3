// Phase timing of the cluster QR kernel (clock64 marks of CTA 0 / thread 0): build with
// nvcc -DTK_QR_TRACE; not part of the library.
#define TK_QR_TRACE 1
#include "../paper_1412_1885_b200/csrc/qr.cu"
#include <cstdio>
#include <random>
#include <vector>
int main() {
    int shapes[][2] = {{300, 20}, {1000, 30}, {2400, 40}, {4000, 60}};
    for (auto& sh : shapes) {
        const int rows = sh[0], cols = sh[1];
        std::vector<double> h(rows * cols);
        std::mt19937 g(1);
        std::normal_distribution<double> nd;
        for (auto& x : h) x = nd(g);
        double *z, *u;
        int* rk;
        cudaMalloc(&z, h.size() * 8);
        cudaMalloc(&u, h.size() * 8);
        cudaMalloc(&rk, 4);
        cudaMemcpy(z, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        double* work = nullptr;
        if (tkb::qr_work_elems(rows, cols) > 0) cudaMalloc(&work, tkb::qr_work_elems(rows, cols) * 8);
        float* upk;
        cudaMalloc(&upk, size_t(rows) * 64 * 4);
        for (int it = 0; it < 3; ++it) tkb::launch_orthonormal_basis(z, rows, cols, u, cols, upk, 0, rk, nullptr, 0, 0, nullptr, work);
        cudaDeviceSynchronize();
        {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            for (int it = 0; it < 20; ++it)
                tkb::launch_orthonormal_basis(z, rows, cols, u, cols, upk, 0, rk, nullptr, 0, 0, nullptr, work);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            int clk = 0;
            cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            printf("%dx%d: %.1f us per launch (back to back, events), SM clock attr %d MHz\n", rows, cols, 1e3 * ms / 20, clk / 1000);
            // in-situ-like: each QR right after a 2 GB memset (HBM-bound work before it)
            void* big = nullptr;
            cudaMalloc(&big, size_t(2) << 30);
            float tot = 0.f;
            for (int it = 0; it < 10; ++it) {
                cudaMemsetAsync(big, it, size_t(2) << 30);
                cudaEventRecord(e0);
                tkb::launch_orthonormal_basis(z, rows, cols, u, cols, upk, 0, rk, nullptr, 0, 0, nullptr, work);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float m1 = 0.f;
                cudaEventElapsedTime(&m1, e0, e1);
                tot += m1;
            }
            cudaFree(big);
            printf("%dx%d: %.1f us per launch after a 2 GB memset each\n", rows, cols, 1e3 * tot / 10);
        }
        long long t[4096];
        cudaMemcpyFromSymbol(t, g_qr_trace, sizeof(t));
        if (t[605] > t[600])
            printf("%dx%d fast path: gram1 %lld pchol1 %lld trsm1 %lld gram2 %lld chol2 %lld trsm2 %lld | sign %lld out %lld total %lld\n",
                   rows, cols, t[600] - t[0], t[601] - t[600], t[602] - t[601], t[603] - t[602], t[604] - t[603],
                   t[605] - t[604], t[4] - t[3], t[5] - t[4], t[5] - t[0]);
        if (t[705] > t[700])
            printf("  pchol step 1: reduce+pivot %lld publish+read %lld div+stores %lld update %lld (cycles)\n",
                   t[705] - t[704], t[706] - t[705],
                   t[707] - t[706], t[708] - t[707]);
        printf("%dx%d: load+norms %lld\n", rows, cols, t[1] - t[0]);
        for (int k = 1; k < 4; ++k)
            printf("  step %d: pivot %lld swap %lld reduce %lld scal+downdate+essential %lld update %lld\n", k,
                   t[6 + 8 * k] - t[7 + 8 * k], t[8 + 8 * k] - t[6 + 8 * k], t[10 + 8 * k] - t[8 + 8 * k],
                   t[11 + 8 * k] - t[10 + 8 * k], t[12 + 8 * k] - t[11 + 8 * k]);
        printf("  factor %lld Q %lld sign %lld out %lld total %lld cycles\n", t[2] - t[1], t[3] - t[2], t[4] - t[3],
               t[5] - t[4], t[5] - t[0]);
    }
    return 0;
}
