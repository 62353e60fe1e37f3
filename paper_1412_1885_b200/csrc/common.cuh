// common.cuh — shared device helpers for the B200 (sm_100a) randomized-Tucker path:
// error plumbing, the reference's counter RNG as device functions, mbarrier / bulk-copy
// PTX wrappers.
#pragma once
#include <cstdlib>

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace tkb {

// The reference raises std::invalid_argument("tenkit: ...") (tensor.hpp:20-22); the
// C-ABI maps it to TK_ERR_INVALID, CUDA failures to TK_ERR_CUDA.
struct InvalidArgument : std::invalid_argument {
    explicit InvalidArgument(const std::string& m) : std::invalid_argument("tenkit: " + m) {}
};
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& m) : std::runtime_error("tenkit: CUDA: " + m) {}
};

inline void require(bool cond, const std::string& msg) {
    if (!cond) throw InvalidArgument(msg);
}

#define TK_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            throw ::tkb::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));   \
    } while (0)

#define TK_LAUNCH_CHECK() TK_CUDA(cudaGetLastError())
// A/B knob TENKIT_CARVEOUT=1: every kernel of the path prefers the maximum shared-memory
// carveout, so consecutive kernels never make the SMs switch their L1/shared split.
inline bool tk_carveout_on() {
    static const bool on = [] {
        const char* e = std::getenv("TENKIT_CARVEOUT");
        return e && e[0] == '1';
    }();
    return on;
}
#define TK_MAXSMEM(k)                                                                                         \
    do {                                                                                                      \
        static const bool tk_co_ = tk_carveout_on() &&                                                        \
            cudaFuncSetAttribute(reinterpret_cast<const void*>(k), cudaFuncAttributePreferredSharedMemoryCarveout, \
                                 100) == cudaSuccess;                                                         \
        (void)tk_co_;                                                                                         \
    } while (0)

// ---------------------------------------------------------------------------
// Counter RNG (reference random.hpp:12-71), host + device. Bit-exact in the integer
// part; the Box-Muller transcendental kernels are CUDA's double-precision ones
// (<=1-2 ulp from glibc).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t hash_combine(uint64_t a, uint64_t b) {
    return mix64(a ^ (mix64(b) + 0x9E3779B97F4A7C15ull + (a << 6) + (a >> 2)));
}
struct Seed {  // SeedSpec (random.hpp:29-44)
    uint64_t root = 0, stream = 0;
    __host__ __device__ Seed derived(uint64_t t) const { return {root, hash_combine(stream, t)}; }
    __host__ __device__ Seed derived(uint64_t a, uint64_t b) const { return derived(a).derived(b); }
    __host__ __device__ uint64_t key() const { return hash_combine(mix64(root), stream); }
};
__host__ __device__ __forceinline__ double counter_unit(uint64_t key, uint64_t i) {
    return static_cast<double>((mix64(key + i * 0x9E3779B97F4A7C15ull) >> 11) + 1) * 0x1.0p-53;
}
#ifdef __CUDACC__
__device__ __forceinline__ double normal_at_key(uint64_t key, uint64_t index) {
    const uint64_t pair = index >> 1;
    const double u1 = counter_unit(key, 2 * pair);
    const double u2 = counter_unit(key, 2 * pair + 1);
    const double r = sqrt(-2.0 * log(u1));
    const double angle = 6.283185307179586476925287 * u2;
    return (index & 1u) ? r * sin(angle) : r * cos(angle);
}
#endif

// Seed tags (tucker.hpp:49-58, bench.hpp:46-48, ffcp.hpp:49-51)
inline Seed alg2_omega_seed(const Seed& s, int64_t n) { return s.derived(0x0A2u, static_cast<uint64_t>(n)); }
inline Seed alg3_init_seed(const Seed& s, int64_t n) { return s.derived(0x0A3u, static_cast<uint64_t>(n)); }
inline Seed alg3_omega_seed(const Seed& s, int64_t pass, int64_t n) {
    return s.derived(0x0B3u + static_cast<uint64_t>(pass), static_cast<uint64_t>(n));
}
inline Seed ffcp_init_seed(const Seed& s, int64_t n) { return s.derived(0x0FCu, static_cast<uint64_t>(n)); }
inline Seed gen_factor_seed(const Seed& s, int64_t n) { return s.derived(0x9E4u, static_cast<uint64_t>(n)); }

#ifdef __CUDACC__
// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA engine, non-tensor form) PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy completing on an mbarrier (size % 16 == 0, 16 B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

#endif  // __CUDACC__

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

template <typename T>
__host__ __device__ constexpr T ceil_div(T a, T b) {
    return (a + b - 1) / b;
}

}  // namespace tkb
