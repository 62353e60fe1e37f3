// ttm_tc.cu — the Y-streaming TTM on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Same contraction as ttm_mmajor_kernel (out[p, r, q] = sum_k Y[p, k, q] U[k, r], the
// first stage of every X_n = Y x_{p != n} U_p^T, tensor.hpp:151-192), but the FFMA loop is
// replaced by tf32 UMMAs in an fp32-accurate 3-pass split (plain TF32 flips
// the sign rule; 3xTF32 keeps ~2^-21 relative error per product):
//     y u ~= y_hi u_hi + y_hi u_lo + y_lo u_hi,   x_hi = rna_tf32(x), x_lo = x - x_hi (exact)
// Warp roles (one 512-row tile of Y per CTA, K streamed in 16-column stages):
//   warp 8      producer: TMA tensor loads (256-row x 16-k boxes of the (P, K, Q) view,
//               zero-filled out of bounds) + a bulk copy of the packed [U_hi | U_lo] stage
//               into a 4-deep shared-memory ring (mbarrier complete_tx)
//   warps 0-7   converters: LDS.128 of 4 rows per thread, split y into (hi, lo) and
//               tcgen05.st them as the A operands in TMEM (row 4L+j of the tile goes to
//               TMEM lane L of M-tile j; warps w and w+4 share lane quarter w and split the
//               16 k of a stage), then the epilogue (warps 0-3: tcgen05.ld, D_hi + D_lo)
//   warp 9      TMEM allocator + single-thread MMA issuer:
//               D_j[0:2NH] += A_hi_j [U_hi | U_lo]   (N = 2NH)
//               D_j[0:NH]  += A_lo_j  U_hi           (N = NH)
// Accumulators stay in TMEM for the whole K loop; Y is read from HBM exactly once.
#include <cuda.h>

#include <stdexcept>

namespace {
// The driver entry point is resolved through the runtime (no link-time libcuda dependency,
// so the library loads on hosts without a driver and fails only when a kernel is launched).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        return (e == cudaSuccess && q == cudaDriverEntryPointSuccess) ? reinterpret_cast<EncodeTiledFn>(p) : nullptr;
    }();
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled entry point unavailable");
    return fn;
}
}  // namespace

#include <algorithm>

#include "kernels.cuh"

namespace tkb {

namespace {

constexpr int kTcConv = 8;                      // converter warps: 2 per TMEM lane quarter (k halves)
constexpr int kTcThreads = (kTcConv + 2) * 32;  // + producer warp + MMA warp
constexpr int kTcBK = 16;                       // K per pipeline stage (2 MMA k-steps of 8)
constexpr int kTcStages = 4;

template <int NH>
struct TcCfg {
    static constexpr int MT = NH <= 32 ? 4 : 2;  // 128-row M tiles per CTA
    static constexpr int BM = 128 * MT;
    static constexpr int BBYTES = 64 * NH;       // one k-step of [U_hi | U_lo]: 2NH rows x 8 tf32
    static constexpr int STAGE_Y = kTcBK * BM * 4;
    static constexpr int STAGE_B = 2 * BBYTES;
    static constexpr int D_COLS = MT * 2 * NH;
    static constexpr int A_COLS = MT * 32;       // per A stage and tile: 16 hi + 16 lo columns
    static_assert(D_COLS + 2 * A_COLS <= 512, "TMEM budget");
    static constexpr size_t smem = size_t(kTcStages) * (STAGE_Y + STAGE_B) + 256 + 128;
};

__device__ __forceinline__ uint32_t f2tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return r;
}

// round-to-nearest (ties away) to tf32 on the magnitude bits; the residual x - hi is exact
// in fp32 and is handed to the MMA as is (the tensor core reads its top 19 bits)
__device__ __forceinline__ uint32_t tf32_hi_bits(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}

// UMMA shared-memory descriptor: K-major, no swizzle (core matrices of 8 rows x 16 B),
// LBO = 128 B between the two 16-B K chunks of a k-step, SBO = 256 B between 8-row groups.
__device__ __forceinline__ uint64_t bdesc(const void* smem) {
    const uint64_t a = smem_u32(smem);
    return ((a >> 4) & 0x3FFFull) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (1ull << 46);
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

template <int NH>
__global__ void __launch_bounds__(kTcThreads, 1)
    ttm_tc_kernel(const __grid_constant__ CUtensorMap ymap, const uint8_t* __restrict__ bpk, float* __restrict__ out,
                  int64_t P, int64_t K, int cols, int64_t tiles_p) {
    using C = TcCfg<NH>;
    constexpr int MT = C::MT, BM = C::BM;
    extern __shared__ __align__(1024) uint8_t tsm[];
    uint8_t* sY = tsm;  // [stages][BM/256 boxes][kTcBK][256] fp32
    uint8_t* sB = tsm + size_t(kTcStages) * C::STAGE_Y;           // [stages][2][2NH x 8] tf32 core matrices
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + size_t(kTcStages) * C::STAGE_B);
    uint64_t* full = bars;                   // [stages]  producer -> (converters, MMA)
    uint64_t* empty = bars + kTcStages;      // [stages]  converters (4) + MMA commit (1) -> producer
    uint64_t* afull = bars + 2 * kTcStages;  // [2]       converters -> MMA
    uint64_t* aempty = afull + 2;            // [2]       MMA commit -> converters
    uint64_t* dfull = aempty + 2;            // [1]       MMA commit -> epilogue
    uint32_t* tbase_sm = reinterpret_cast<uint32_t*>(dfull + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t q = blockIdx.x / tiles_p;
    const int64_t p0 = (blockIdx.x % tiles_p) * BM;
    const int rows = static_cast<int>(lmin(BM, P - p0));
    const int nk = static_cast<int>((K + kTcBK - 1) / kTcBK);

    if (tid == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTcConv + 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&afull[a], kTcConv);
            mbar_init(&aempty[a], 1);
        }
        mbar_init(dfull, 1);
        mbar_fence_init();
    }
    if (warp == kTcConv + 1) {  // TMEM allocation (whole warp)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tbase_sm)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tbase_sm;

    if (warp == kTcConv) {
        // ===== producer =====
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&ymap) : "memory");
            for (int kc = 0; kc < nk; ++kc) {
                const int s = kc % kTcStages;
                mbar_wait(&empty[s], ((kc / kTcStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], C::STAGE_Y + C::STAGE_B);
                uint8_t* dy = sY + size_t(s) * C::STAGE_Y;
#pragma unroll
                for (int b = 0; b < BM / 256; ++b)
                    tma_load_3d(dy + b * (kTcBK * 256 * 4), &ymap, static_cast<int>(p0 + 256 * b), kc * kTcBK,
                                static_cast<int>(q), &full[s]);
                bulk_g2s(sB + size_t(s) * C::STAGE_B, bpk + size_t(kc) * C::STAGE_B, C::STAGE_B, &full[s]);
            }
        }
    } else if (warp == kTcConv + 1) {
        // ===== MMA issuer =====
        if (lane == 0) {
            const uint32_t id_full = idesc_tf32(2 * NH), id_hi = idesc_tf32(NH);
            for (int kc = 0; kc < nk; ++kc) {
                const int s = kc % kTcStages, a = kc & 1;
                mbar_wait(&full[s], (kc / kTcStages) & 1);
                mbar_wait(&afull[a], (kc >> 1) & 1);
                fence_after();
                const uint8_t* bs = sB + size_t(s) * C::STAGE_B;
#pragma unroll
                for (int j = 0; j < MT; ++j) {
                    const uint32_t d = tmem + uint32_t(j * 2 * NH);
                    const uint32_t ahi = tmem + uint32_t(C::D_COLS + a * C::A_COLS + j * 32);
#pragma unroll
                    for (int ks = 0; ks < 2; ++ks) {
                        const uint64_t b = bdesc(bs + ks * C::BBYTES);
                        mma_tf32_ts(d, ahi + ks * 8, b, id_full, (kc > 0 || ks > 0) ? 1u : 0u);
                        mma_tf32_ts(d, ahi + 16 + ks * 8, b, id_hi, 1u);
                    }
                }
                mma_commit(&aempty[a]);
                mma_commit(&empty[s]);
            }
            mma_commit(dfull);
        }
    } else {
        // ===== converters (warps 0-7): Y tile -> (hi, lo) tf32 A operands in TMEM =====
        const int quarter = warp & 3, khalf = warp >> 2;
        const int L = quarter * 32 + lane;                    // TMEM lane of this thread
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        for (int kc = 0; kc < nk; ++kc) {
            const int s = kc % kTcStages, a = kc & 1;
            mbar_wait(&full[s], (kc / kTcStages) & 1);
            uint32_t hi[MT][8], lo[MT][8];
            // rows MT*L .. MT*L+MT-1 of the tile sit in box (MT*L)/256 at row (MT*L)%256
            const float* ys = reinterpret_cast<const float*>(sY + size_t(s) * C::STAGE_Y) +
                              ((MT * L) / 256) * (kTcBK * 256) + (MT * L) % 256 + khalf * 8 * 256;
            auto split = [&](int kk, bool live) {
                float y[MT];
                if constexpr (MT == 4) {
                    const float4 v = *reinterpret_cast<const float4*>(ys + kk * 256);
                    y[0] = v.x, y[1] = v.y, y[2] = v.z, y[3] = v.w;
                } else {
                    const float2 v = *reinterpret_cast<const float2*>(ys + kk * 256);
                    y[0] = v.x, y[1] = v.y;
                }
#pragma unroll
                for (int j = 0; j < MT; ++j) {
                    const float x = live ? y[j] : 0.f;
                    const uint32_t h = tf32_hi_bits(x);
                    hi[j][kk] = h;
                    lo[j][kk] = __float_as_uint(x - __uint_as_float(h));
                }
            };
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) split(kk, true);  // the K tail is zero-filled by the TMA
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // Y stage consumed (B: the MMA commit)
            mbar_wait(&aempty[a], ((kc >> 1) & 1) ^ 1);
            fence_after();
#pragma unroll
            for (int j = 0; j < MT; ++j) {
                const uint32_t ta = tmem + lane_off + uint32_t(C::D_COLS + a * C::A_COLS + j * 32 + khalf * 8);
                tmem_st8(ta, hi[j]);
                tmem_st8(ta + 16, lo[j]);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&afull[a]);
        }
        if (khalf == 1) goto done;  // the epilogue runs on warps 0-3 (one per lane quarter)
        // ===== epilogue: D = D[:, 0:NH] + D[:, NH:2NH], rows MT*L + j =====
        mbar_wait(dfull, 0);
        fence_after();
        float* o = out + q * P * cols + p0 + MT * L;
        const bool live = MT * L < rows;
#pragma unroll
        for (int rc = 0; rc < NH; rc += 16) {
            float acc[MT][16];
#pragma unroll
            for (int j = 0; j < MT; ++j) {
                uint32_t vh[16], vl[16];
                const uint32_t td = tmem + lane_off + uint32_t(j * 2 * NH + rc);
                tmem_ld16(td, vh);
                tmem_ld16(td + NH, vl);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[j][e] = __uint_as_float(vh[e]) + __uint_as_float(vl[e]);
            }
            if (live) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int r = rc + e;
                    if (r < cols) {
                        if constexpr (MT == 4) {
                            *reinterpret_cast<float4*>(o + int64_t(r) * P) =
                                make_float4(acc[0][e], acc[1][e], acc[2][e], acc[3][e]);
                        } else {
                            *reinterpret_cast<float2*>(o + int64_t(r) * P) = make_float2(acc[0][e], acc[1][e]);
                        }
                    }
                }
            }
        }
    }
done:
    fence_before();
    __syncthreads();
    if (warp == kTcConv + 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

// [U_hi | U_lo] of a column-major fp64 factor (rows x cols, ld), tf32 in the UMMA K-major
// no-swizzle core-matrix layout, one 64*NH-byte block per k-step of 8 rows of U.
template <int NH>
__global__ void pack_umma_kernel(const double* __restrict__ u, int64_t ld, int64_t rows, int cols, int64_t ksteps,
                                 uint32_t* __restrict__ out) {
    const int64_t n_el = ksteps * 2 * NH * 8;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n_el; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t g = t / (2 * NH * 8);
        const int rem = static_cast<int>(t % (2 * NH * 8));
        const int n = rem / 8, kk = rem % 8;
        const int64_t k = g * 8 + kk;
        const int r = n < NH ? n : n - NH;
        const float uf = (k < rows && r < cols) ? static_cast<float>(u[k + int64_t(r) * ld]) : 0.f;
        const uint32_t h = f2tf32(uf);
        const uint32_t v = n < NH ? h : f2tf32(uf - __uint_as_float(h));
        const int64_t byte = g * (64 * NH) + (n / 8) * 256 + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4;
        out[byte / 4] = v;
    }
}

template <int NH>
void launch_tc(const float* in, const uint8_t* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
               cudaStream_t s) {
    using C = TcCfg<NH>;
    static bool attr = false;
    if (!attr) {
        TK_CUDA(cudaFuncSetAttribute(ttm_tc_kernel<NH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(C::smem)));
        attr = true;
    }
    const int64_t tiles_p = (P + C::BM - 1) / C::BM;
    const int64_t grid = tiles_p * Q;
    require(grid < (int64_t(1) << 31), "ttm: grid too large");
    require(K < (int64_t(1) << 31) && Q < (int64_t(1) << 31) && P < (int64_t(1) << 31), "ttm: extent too large for TMA");
    CUtensorMap map;
    const cuuint64_t dims[3] = {cuuint64_t(P), cuuint64_t(K), cuuint64_t(Q)};
    const cuuint64_t strides[2] = {cuuint64_t(P) * 4, cuuint64_t(P) * cuuint64_t(K) * 4};
    const cuuint32_t box[3] = {256, kTcBK, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(in), dims,
                                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    ttm_tc_kernel<NH><<<static_cast<unsigned>(grid), kTcThreads, C::smem, s>>>(map, bpk, out, P, K, cols, tiles_p);
    TK_LAUNCH_CHECK();
}

inline int tc_nh(int cols) { return cols <= 16 ? 16 : cols <= 32 ? 32 : cols <= 48 ? 48 : 64; }

}  // namespace

int64_t umma_pack_bytes(int64_t rows, int cols) {
    const int64_t ksteps = (rows + kTcBK - 1) / kTcBK * 2;
    return ksteps * 64 * tc_nh(cols);
}

void launch_pack_umma(const double* u, int64_t ld, int64_t rows, int cols, void* out, cudaStream_t s) {
    require(cols >= 1 && cols <= kMaxRank, "ttm: factor column count must be in [1, 64]");
    const int64_t ksteps = (rows + kTcBK - 1) / kTcBK * 2;
    const int nh = tc_nh(cols);
    const int64_t n = ksteps * 2 * nh * 8;
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
    uint32_t* o = static_cast<uint32_t*>(out);
    switch (nh) {
        case 16: pack_umma_kernel<16><<<grid, 256, 0, s>>>(u, ld, rows, cols, ksteps, o); break;
        case 32: pack_umma_kernel<32><<<grid, 256, 0, s>>>(u, ld, rows, cols, ksteps, o); break;
        case 48: pack_umma_kernel<48><<<grid, 256, 0, s>>>(u, ld, rows, cols, ksteps, o); break;
        default: pack_umma_kernel<64><<<grid, 256, 0, s>>>(u, ld, rows, cols, ksteps, o); break;
    }
    TK_LAUNCH_CHECK();
}

bool tc_ttm_supported(const float* in, float* out, int64_t P, int64_t Q, int cols) {
    const int bm = tc_nh(cols) <= 32 ? 512 : 256;
    const int64_t tiles = (P + bm - 1) / bm * Q;
    return P % 4 == 0 && P >= 256 && tiles >= 2 * 148 && reinterpret_cast<uintptr_t>(in) % 16 == 0 &&
           reinterpret_cast<uintptr_t>(out) % 16 == 0;
}

void launch_ttm_tc(const float* in, const void* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
                   cudaStream_t s) {
    const uint8_t* b = static_cast<const uint8_t*>(bpk);
    switch (tc_nh(cols)) {
        case 16: return launch_tc<16>(in, b, out, P, K, Q, cols, s);
        case 32: return launch_tc<32>(in, b, out, P, K, Q, cols, s);
        case 48: return launch_tc<48>(in, b, out, P, K, Q, cols, s);
        default: return launch_tc<64>(in, b, out, P, K, Q, cols, s);
    }
}

}  // namespace tkb
