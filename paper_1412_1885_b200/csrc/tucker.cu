// tucker.cu — host driver of the randomized Tucker decompositions on one B200 (and one
// rank of a slab-partitioned multi-GPU run) + the C-ABI (include/tenkit_b200.h).
//
// rand_tucker_2i (reference tucker.hpp:136-169, paper Alg. 3) per (pass, n):
//   X_n = Y x_{p != n} U_p^T   first stage streams Y once (ttm.cu), later stages are small
//   Z_n = unfold(X_n, n) * Omega_n          (Omega regenerated from the seed, never stored)
//   U_n = orthonormal_basis(Z_n), sign-fixed (qr.cu, one cluster)
// core = X_{N-1} x_{N-1} U_{N-1}^T (the reference's extra pass at tucker.hpp:166 computes
// the same tensor with the same operation order; opts.explicit_core_pass restores it).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/tenkit_b200.h"
#include "kernels.cuh"

using namespace tkb;

namespace {
// NCCL resolved at run time (no link-time dependency: the library loads on hosts without NCCL
// and fails only when a native communicator is requested). The process's already-loaded
// libnccl.so.2 (torch's) is preferred; TENKIT_NCCL_LIB overrides the path.
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
    bool ok = false;
};

const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = nullptr;
        if (const char* e = std::getenv("TENKIT_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.get_version = reinterpret_cast<decltype(a.get_version)>(dlsym(h, "ncclGetVersion"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.comm_destroy && a.error_string;
        return a;
    }();
    if (!api.ok) throw std::runtime_error("NCCL (libnccl.so.2) unavailable");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string("nccl: ") + what + ": " + nccl_api().error_string(r));
}
}  // namespace

struct tk_context {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    bool has_comm = false;
    int ttm_path = 0;  // 0 auto (tcgen05 for fp32 Y streams), 1 FFMA only, 2 tcgen05 whenever supported
    int ortho = TK_ORTHO_COLPIV;  // range-step basis: ColPiv QR + sign rule, or the dist protocol's Gram-eig
    tk_comm comm{};
    // native NCCL communicator (tk_context_set_nccl): the partial sketches / cores are
    // all-reduced in place on the call's stream, no host callback, CUDA graphs stay enabled
    ncclComm_t nccl = nullptr;
    int nccl_rank = 0, nccl_world = 0;
    uint64_t nccl_gen = 0;  // bumped per communicator (part of the graph key)
    std::map<std::string, std::pair<void*, size_t>> bufs;
    int* rank_host = nullptr;  // pinned
    cudaStream_t side = nullptr;  // second stream: next Y pass overlapped with the current QR
    cudaEvent_t ev_free = nullptr, ev_fs = nullptr;
    cudaStream_t cap = nullptr;   // private stream the CUDA graph is captured on
    cudaEvent_t ev_cap = nullptr;
    // A repeated rand_tucker_2i call (same shapes, seed, input pointer and options) is captured
    // once as a CUDA graph and replayed: one launch per decomposition instead of ~60.
    struct Graph {
        std::string key;
        int seen = 0;
        cudaGraphExec_t exec = nullptr;
        std::vector<cudaEvent_t> marks;  // Y-pass timing events (time_kernels)
        double* core = nullptr;
        std::vector<double*> U;
        std::vector<int64_t> cshape, cols;
        int64_t gsize = 0;
        int passes = 0, launches = 0;
        std::vector<int> rt;
        uint64_t buf_gen = 0;
        void reset() {
            if (exec) cudaGraphExecDestroy(exec);
            exec = nullptr;
            for (auto e : marks) cudaEventDestroy(e);
            marks.clear();
            seen = 0;
        }
    } g2i;

    // copy stream + events of the host-input landing (TuckerRun::land_stream)
    static constexpr int kLandEvents = 5;
    cudaStream_t copy = nullptr;
    cudaEvent_t land_ev[kLandEvents] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    void ensure_copy() {
        if (!copy) {
            TK_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
            for (auto& e : land_ev) TK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
    }

    void ensure_side() {
        if (!side) {
            // lowest priority: when the QR cluster (main stream) and the next Y pass become
            // runnable together, the QR is dispatched first and the pass takes the other SMs
            int lo = 0, hi = 0;
            TK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            TK_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo));
            TK_CUDA(cudaEventCreateWithFlags(&ev_free, cudaEventDisableTiming));
            TK_CUDA(cudaEventCreateWithFlags(&ev_fs, cudaEventDisableTiming));
        }
    }

    uint64_t buf_gen = 0;  // bumped whenever a buffer is (re)allocated: captured graphs go stale
    void* buf(const std::string& name, size_t bytes) {
        auto& e = bufs[name];
        if (e.second < bytes) {
            ++buf_gen;
            if (e.first) TK_CUDA(cudaFree(e.first));
            e.first = nullptr;
            TK_CUDA(cudaMalloc(&e.first, std::max<size_t>(bytes, 256)));
            e.second = std::max<size_t>(bytes, 256);
        }
        return e.first;
    }
    void drop_nccl() {
        if (nccl) nccl_api().comm_destroy(nccl);
        nccl = nullptr;
        nccl_world = 0;
    }
    ~tk_context() {
        g2i.reset();
        try {
            drop_nccl();
        } catch (...) {
        }
        if (ev_cap) cudaEventDestroy(ev_cap);
        if (cap) cudaStreamDestroy(cap);
        for (auto& kv : bufs)
            if (kv.second.first) cudaFree(kv.second.first);
        if (rank_host) cudaFreeHost(rank_host);
        if (ev_free) cudaEventDestroy(ev_free);
        if (ev_fs) cudaEventDestroy(ev_fs);
        if (side) cudaStreamDestroy(side);
        for (auto e : land_ev)
            if (e) cudaEventDestroy(e);
        if (copy) cudaStreamDestroy(copy);
        if (own) cudaStreamDestroy(own);
    }
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return TK_OK;
    } catch (const InvalidArgument& e) {
        return fail(TK_ERR_INVALID, e.what());
    } catch (const CudaError& e) {
        return fail(TK_ERR_CUDA, e.what());
    } catch (const std::exception& e) {
        return fail(TK_ERR_INTERNAL, std::string("tenkit: ") + e.what());
    }
}

bool qr_fuse();

int64_t prod(const std::vector<int64_t>& v, int64_t skip = -1) {
    int64_t p = 1;
    for (size_t i = 0; i < v.size(); ++i)
        if (static_cast<int64_t>(i) != skip) p *= v[i];
    return p;
}

size_t dsize(int dtype) { return dtype == TK_F32 ? 4 : 8; }

void check_ctx(tk_context* ctx) {
    require(ctx != nullptr, "null context");
    TK_CUDA(cudaSetDevice(ctx->device));
}

// This rank's block of the global tensor (BlockGrid, dist.hpp:24-123): global extents gd and
// the global index of the block's first row in each mode. Without a multi-rank comm hook the
// block is the whole tensor.
void block_of(const tk_context* ctx, const std::vector<int64_t>& ld, std::vector<int64_t>& gd,
              std::vector<int64_t>& lo) {
    const size_t order = ld.size();
    gd = ld;
    lo.assign(order, 0);
    if (!ctx->has_comm || ctx->comm.world <= 1) return;
    const tk_comm& c = ctx->comm;
    if (c.blocked) {
        for (size_t n = 0; n < order; ++n) {
            gd[n] = c.global_dims[n];
            lo[n] = c.block_lo[n];
            require(lo[n] >= 0 && lo[n] + ld[n] <= gd[n], "comm: block outside the global tensor");
        }
    } else {
        gd[order - 1] = c.global_last_dim;
        lo[order - 1] = c.slab_offset;
        require(lo[order - 1] >= 0 && lo[order - 1] + ld[order - 1] <= gd[order - 1],
                "comm: slab outside the global tensor");
    }
}

// Per range step QR diagnostics into the stats (the "margins" context buffer, 3 doubles per
// step: pivot margin, sign margin, QR path); steps = 2N (Alg. 3) or N (Alg. 2).
void read_margins(tk_context* ctx, int64_t order, cudaStream_t s, tk_tucker_stats* stats, int64_t steps = -1) {
    if (steps < 0) steps = 2 * order;
    double hm[3 * 2 * TK_MAX_ORDER];
    const double* md = static_cast<const double*>(ctx->buf("margins", sizeof(double) * 3 * 2 * TK_MAX_ORDER));
    TK_CUDA(cudaMemcpyAsync(hm, md, sizeof(double) * 3 * steps, cudaMemcpyDeviceToHost, s));
    TK_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < 2 * TK_MAX_ORDER; ++i) {
        const bool v = i < steps;
        stats->pivot_margin[i] = v ? hm[3 * i] : 0.0;
        stats->sign_margin[i] = v ? hm[3 * i + 1] : 0.0;
        stats->qr_path[i] = v ? static_cast<int>(hm[3 * i + 2]) : -1;
    }
}

// ---------------------------------------------------------------------------
// One decomposition run for value type T.
// ---------------------------------------------------------------------------
template <typename T>
struct TuckerRun {
    tk_context* ctx;
    cudaStream_t s;
    int64_t order;
    std::vector<int64_t> ldims;  // local dims of Y on this rank
    std::vector<int64_t> gdims;  // global dims
    std::vector<int64_t> off;    // global index of this rank's first row in each mode (BlockGrid lo)
    const T* y;
    std::vector<int> rt, cols;
    std::vector<double*> U;  // global factors, gdims[n] x rt[n] (ld gdims[n])
    std::vector<T*> Up;      // packed k-major copies
    int launches = 0;
    int passes = 0;
    int group_count = 0;
    int* rank_dev = nullptr;
    double* margins_dev = nullptr;  // per range step: pivot margin, sign margin, QR path
    bool time_kernels = false;
    std::vector<cudaEvent_t> ev;  // (start, stop) pairs around Y-streaming launches

    ~TuckerRun() {
        for (auto e : ev) cudaEventDestroy(e);
    }
    bool capture = false;        // compute only: no host syncs, outputs stay in context buffers
    double* core_out = nullptr;  // capture: the fp64 core (context buffer)
    std::vector<int64_t> core_shape;
    // TENKIT_PHASE_TIMING=1 (eager runs only): CUDA events around every phase of the step,
    // summed per category and printed to stderr (a diagnostic of where a decomposition goes).
    bool phase_on = [] {
        const char* e = std::getenv("TENKIT_PHASE_TIMING");
        return e && e[0] == '1';
    }();
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> phases;
    // precision = fp64 on fp32 data (T = double): the Y passes read this fp32 tensor and
    // compute in fp64 (ttm_mixed.cu); y is unused then
    const float* y32 = nullptr;
    // Host input (tk_rand_tucker_2i with y_on_device = 0): `y` is the device landing buffer and
    // `land_src` the caller's host tensor, not yet copied. The first Y pass copies it in
    // last-mode slabs on the context's copy stream and, when that pass contracts the last mode
    // on the streaming kernel, multiplies each slab as it lands (a pass split over K, partial
    // sums added in slab order), so only the last slab's share of the pass is not hidden behind
    // the host link (bench.hpp:456-520 times the copy-in with the decomposition).
    const T* land_src = nullptr;
    void land_all() {  // plain path: the whole tensor on the compute stream
        if (!land_src) return;
        TK_CUDA(cudaMemcpyAsync(const_cast<T*>(y), land_src, sizeof(T) * prod(ldims), cudaMemcpyHostToDevice, s));
        land_src = nullptr;
    }
    void ph_begin(int cat) {
        if (!phase_on || capture) return;
        cudaEvent_t a, b;
        TK_CUDA(cudaEventCreate(&a));
        TK_CUDA(cudaEventCreate(&b));
        TK_CUDA(cudaEventRecord(a, s));
        phases.push_back({cat, {a, b}});
    }
    void ph_end() {
        if (!phase_on || capture || phases.empty()) return;
        TK_CUDA(cudaEventRecord(phases.back().second.second, s));
    }
    void ph_report() {
        if (!phase_on || capture || phases.empty()) return;
        static const char* names[] = {"y_pass", "stage2", "sketch", "qr", "core"};
        double tot[5] = {0, 0, 0, 0, 0};
        int cnt[5] = {0, 0, 0, 0, 0};
        std::string each;  // the Y passes one by one
        for (auto& p : phases) {
            TK_CUDA(cudaEventSynchronize(p.second.second));
            float ms = 0.f;
            TK_CUDA(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
            tot[p.first] += ms;
            ++cnt[p.first];
            if (p.first == 0) each += " " + std::to_string(static_cast<int>(1e3 * ms));
        }
        float span = 0.f;
        TK_CUDA(cudaEventElapsedTime(&span, phases.front().second.first, phases.back().second.second));
        std::fprintf(stderr, "tenkit phases:");
        for (int c = 0; c < 5; ++c) std::fprintf(stderr, " %s %.1f us (%d)", names[c], 1e3 * tot[c], cnt[c]);
        std::fprintf(stderr, " | span %.1f us | y_pass each (us):%s\n", 1e3 * span, each.c_str());
        for (auto& p : phases) {
            cudaEventDestroy(p.second.first);
            cudaEventDestroy(p.second.second);
        }
        phases.clear();
    }
    void mark() {
        cudaEvent_t e;
        TK_CUDA(cudaEventCreate(&e));
        // in a captured graph the record must be an external event node to be re-recorded
        TK_CUDA(capture ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s));
        ev.push_back(e);
    }
    double streamed_ms() {
        double ms = 0.0;
        for (size_t i = 0; i + 1 < ev.size(); i += 2) {
            TK_CUDA(cudaEventSynchronize(ev[i + 1]));
            float t = 0.f;
            TK_CUDA(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
            ms += t;
        }
        return ms;
    }

    const T* factor_rows(int m) const {  // rows of U_m matching this rank's block
        const T* p = Up[m];
        p += off[m] * pack_stride(cols[m]);
        return p;
    }

    const char* work_name = "splitk";  // split-K scratch of the stream currently launching
    cudaEvent_t qr_event = nullptr;     // recorded just before the next QR launch (overlap gate)

    // Mode contracted first (the one pass that streams Y): the last mode (a plain M-major GEMM)
    // unless it is kept, and never `avoid` (the factor the still-running QR is producing) when
    // another mode with a wide enough row block exists, so that pass can overlap the QR.
    int first_mode(int skip, int avoid) const {
        auto ok = [&](int m) { return m >= 0 && m < order && m != skip; };
        for (int m = static_cast<int>(order) - 1; m >= 0; --m) {
            if (!ok(m) || m == avoid) continue;
            if (prod(std::vector<int64_t>(ldims.begin(), ldims.begin() + m)) >= 256) return m;
            if (m == 0 && km_stream_ok()) return m;  // K-major tcgen05 pass over mode 0
        }
        for (int m = static_cast<int>(order) - 1; m >= 0; --m)
            if (ok(m)) return m;
        return -1;
    }

    // A/B knob: TENKIT_NO_REUSE=1 recomputes every step's first small contraction
    static bool reuse_first() {
        static const bool on = [] {
            const char* e = std::getenv("TENKIT_NO_REUSE");
            return !(e && e[0] == '1');
        }();
        return on;
    }

    // Leader of a shared Y pass for a group of steps whose modes are `mask`: a mode outside the
    // group that can lead a pass (first_mode's rule), preferring one other than `avoid`.
    int leader_mode(uint32_t mask, int avoid) const {
        int fallback = -1;
        for (int m = static_cast<int>(order) - 1; m >= 0; --m) {
            if (mask & (1u << m)) continue;
            // small tensors (latency-bound passes): any mode can lead (FFMA kernels)
            static const bool no_km_leader = [] {  // A/B knob: mode 0 never leads a shared pass
                const char* e = std::getenv("TENKIT_NO_KM_LEADER");
                return e && e[0] == '1';
            }();
            const bool capable = prod(std::vector<int64_t>(ldims.begin(), ldims.begin() + m)) >= 256 ||
                                 (m == 0 && !no_km_leader && km_stream_ok()) ||
                                 prod(ldims) * int64_t(sizeof(T)) <= (int64_t(256) << 20);
            if (!capable) continue;
            if (m != avoid) return m;
            fallback = m;
        }
        return fallback;
    }

    // Mode 0 can lead a Y pass when the K-major tcgen05 kernel takes it (fp32, I_0 % 4 == 0,
    // r~_0 <= TENKIT_KM_LEAD_MAX = 64, >= 148 row tiles), on the auto and tc paths (not the
    // FFMA-only path 1). stream_ttm always asks for the accurate variant: 128-row tiles with
    // 2-4 accumulator sets (the truncating tensor-core accumulation over K = I_0 is split
    // across the sets; a 512-row single-set tile doubled the fp32 basis error at cfg 2).
    bool km_stream_ok() const {
        if constexpr (sizeof(T) != 4) {
            return false;
        } else {
            if (ctx->ttm_path == 1 || cols.empty()) return false;
            const int64_t K = ldims[0];
            const int64_t Q = prod(ldims) / K;
            static const int km_max = [] {  // A/B knob: widest factor a mode-0 Y pass may use
                const char* e = std::getenv("TENKIT_KM_LEAD_MAX");
                return e ? std::atoi(e) : 64;
            }();
            return K % 4 == 0 && K >= 16 && cols[0] <= km_max && (Q + 127) / 128 >= 148 &&
                   reinterpret_cast<uintptr_t>(y) % 16 == 0;
        }
    }

    // Intermediate tensors may hold their modes in a permuted storage order: xd are the extents
    // in storage order and xp[k] the mode stored at position k (identity unless a mode-0 Y
    // pass wrote its output transposed, moving mode 0 to the slowest position).
    std::vector<int> ident() const {
        std::vector<int> v(static_cast<size_t>(order));
        std::iota(v.begin(), v.end(), 0);
        return v;
    }
    static int pos_of(const std::vector<int>& xp, int m) {
        for (size_t k = 0; k < xp.size(); ++k)
            if (xp[k] == m) return static_cast<int>(k);
        return -1;
    }

    // First stage: Y x_f U_f^T into "proj1" (dims updated). Runs on the current stream `s`.
    // A mode-0 pass (K-major tcgen05 kernel) writes its output transposed (mode 0 last), so the
    // later contractions of the group see the big modes first (M-major / K-major shapes).
    const T* first_stage(int f, std::vector<int64_t>& xd, std::vector<int>& xp) {
        xd = ldims;
        xp = ident();
        if (f < 0) {
            land_all();
            return y;
        }
        const int64_t P = prod(std::vector<int64_t>(xd.begin(), xd.begin() + f));
        const int64_t K = xd[f];
        const int64_t Q = prod(std::vector<int64_t>(xd.begin() + f + 1, xd.end()));
        T* out = static_cast<T*>(ctx->buf("proj1", sizeof(T) * P * cols[f] * Q));
        bool tout = false;
        if (land_src && land_stream(f, out, P, K)) {
            ++passes;
            xd[f] = cols[f];
            return out;
        }
        land_all();
        ph_begin(0);
        if constexpr (sizeof(T) == 8) {
            if (y32) {  // fp64 arithmetic over the fp32 tensor
                if (time_kernels) mark();
                launch_ttm_mixed(y32, reinterpret_cast<const double*>(factor_rows(f)), reinterpret_cast<double*>(out),
                                 P, K, Q, cols[f], s);
                ++launches;
                if (time_kernels) mark();
                ph_end();
                ++passes;
                xd[f] = cols[f];
                return out;
            }
        }
        if (!stream_ttm(y, f, out, P, K, Q, true, &tout)) {
            if (time_kernels) mark();
            ttm(y, factor_rows(f), out, P, K, Q, cols[f]);
            if (time_kernels) mark();
        }
        ph_end();
        ++passes;
        xd[f] = cols[f];
        if (tout) {  // storage (1, 2, ..., N-1, 0)
            std::rotate(xd.begin(), xd.begin() + 1, xd.end());
            std::rotate(xp.begin(), xp.begin() + 1, xp.end());
        }
        return out;
    }

    // The first Y pass of a host-input call, contracting the last mode (Q = 1): the tensor is
    // copied slab by slab on the copy stream and every slab is multiplied as it lands.
    bool land_stream(int f, T* out, int64_t P, int64_t K) {
        if constexpr (sizeof(T) != 4) {
            return false;
        } else {
            static const int nslabs = [] {  // A/B knob: TENKIT_LAND_SLABS=1 copies first, then one pass
                const char* e = std::getenv("TENKIT_LAND_SLABS");
                return e ? std::max(1, std::atoi(e)) : 8;
            }();
            if (f != order - 1 || order < 2 || nslabs < 2 || ctx->ttm_path == 1 || !stream_ttm_enabled() ||
                U.size() <= size_t(f) || !U[f])
                return false;
            const int64_t kstep = ((K + nslabs - 1) / nslabs + 15) / 16 * 16;
            float* fy = reinterpret_cast<float*>(const_cast<T*>(y));
            float* fout = reinterpret_cast<float*>(out);
            if (kstep >= K || !stream_ttm_supported(fy, fout, P, std::min(kstep, K - (K - 1) / kstep * kstep), 1, cols[f]))
                return false;
            void* bpk = ctx->buf("stream_pack", static_cast<size_t>(stream_pack_bytes(K, cols[f])));
            launch_pack_stream(U[f] + off[f], gdims[f], K, cols[f], bpk, s);
            ++launches;
            ctx->ensure_copy();
            // the landing buffer may still be read by earlier work on the compute stream
            TK_CUDA(cudaEventRecord(ctx->land_ev[0], s));
            TK_CUDA(cudaStreamWaitEvent(ctx->copy, ctx->land_ev[0], 0));
            const float* src = reinterpret_cast<const float*>(land_src);
            int slab = 0;
            for (int64_t k0 = 0; k0 < K; k0 += kstep, ++slab) {
                const int64_t kn = std::min(kstep, K - k0);
                TK_CUDA(cudaMemcpyAsync(fy + k0 * P, src + k0 * P, sizeof(float) * kn * P, cudaMemcpyHostToDevice, ctx->copy));
                cudaEvent_t e = ctx->land_ev[1 + slab % (tk_context::kLandEvents - 1)];
                TK_CUDA(cudaEventRecord(e, ctx->copy));
                TK_CUDA(cudaStreamWaitEvent(s, e, 0));
                launch_ttm_stream(fy + k0 * P, bpk, fout, P, kn, 1, cols[f], s, k0, k0 > 0);
                ++launches;
            }
            land_src = nullptr;
            return true;
        }
    }

    // The first contraction of the previous finish() (T x_m U_m^T in "projA"): consecutive steps
    // of a group that contract the same mode first, with the same factor, out of the same Y pass
    // reuse it (N = 4: steps (0, 1) both start with x_2 U_2, steps (3, 0') with x_3 U_3').
    struct FirstCache {
        int pass = -1, mode = -1, ver = -1;
        const void* src = nullptr;
        void* out = nullptr;
        int64_t P = 0, K = 0, Q = 0;
    } fc;
    std::vector<int> fver;  // per mode: bumped whenever U_m is rewritten

    // Remaining (small) contractions of every mode except skip and f, descending. A contraction
    // over the storage-fastest mode on the streaming kernel writes its output transposed (that
    // mode moves to the slowest storage position): xd / xp follow the storage order.
    const T* finish(const T* cur, std::vector<int64_t>& xd, std::vector<int>& xp, int skip, int f) {
        int which = 0;
        bool first = true;
        for (int m = static_cast<int>(order) - 1; m >= 0; --m) {
            if (m == skip || m == f) continue;
            const int k = pos_of(xp, m);
            const int64_t P = prod(std::vector<int64_t>(xd.begin(), xd.begin() + k));
            const int64_t K = xd[k];
            const int64_t Q = prod(std::vector<int64_t>(xd.begin() + k + 1, xd.end()));
            T* out = static_cast<T*>(ctx->buf(which ? "projB" : "projA", sizeof(T) * P * cols[m] * Q));
            const int ver = fver.empty() ? 0 : fver[m];
            const bool hit = first && reuse_first() && fc.pass == passes && fc.mode == m && fc.ver == ver &&
                             fc.src == cur && fc.out == out && fc.P == P && fc.K == K && fc.Q == Q;
            if (first) fc = FirstCache{passes, m, ver, cur, out, P, K, Q};
            else if (!which) fc.pass = -1;  // a later contraction overwrites projA
            first = false;
            ph_begin(1);
            // the streaming kernel's K-major form (transposed output) is deterministic in the
            // shapes, so a cache hit rotates the storage order exactly as the computing step did
            bool tout = P == 1 && stream_second_ok(cur, out, P, K, Q, cols[m]);
            if (!hit) {
                bool tr = false;
                if (!stream_ttm(cur, m, out, P, K, Q, false, tout ? &tr : nullptr))
                    ttm(cur, factor_rows(m), out, P, K, Q, cols[m]);
                tout = tr;
            }
            ph_end();
            xd[k] = cols[m];
            if (tout) {  // storage (1, ..., N-1, 0): the contracted mode last
                std::rotate(xd.begin(), xd.begin() + 1, xd.end());
                std::rotate(xp.begin(), xp.begin() + 1, xp.end());
            }
            cur = out;
            which ^= 1;
        }
        return cur;
    }

    // A second-stage contraction on the streaming kernel (TENKIT_STREAM_SECOND=0: first design)
    bool stream_second_ok(const T* in, T* out, int64_t P, int64_t K, int64_t Q, int c) const {
        if constexpr (sizeof(T) != 4) {
            return false;
        } else {
            static const bool on = [] {
                const char* e = std::getenv("TENKIT_STREAM_SECOND");
                return !(e && e[0] == '0');
            }();
            return on && ctx->ttm_path != 1 && stream_ttm_enabled() &&
                   stream_ttm_supported(reinterpret_cast<const float*>(in), reinterpret_cast<float*>(out), P, K, Q, c);
        }
    }

    // Y x_{p != skip} U_p^T (skip = -1: all modes), on the current stream.
    const T* project(int skip, std::vector<int64_t>& xd, std::vector<int>& xp) {
        if (order == 1 && skip == 0) {
            xd = ldims;
            xp = ident();
            land_all();
            return y;
        }
        const int f = first_mode(skip, -1);
        const T* t1 = first_stage(f, xd, xp);
        return finish(t1, xd, xp, skip, f);
    }

    // The Y-streaming contraction on the tcgen05 tensor cores (3xTF32, ttm_tc.cu) when the data
    // is fp32 and the shape tiles the GPU; returns false to fall back to the FFMA kernels.
    bool stream_ttm(const T* in, int m, T* out, int64_t P, int64_t K, int64_t Q, bool streams_y,
                    bool* tout = nullptr) {
        if constexpr (sizeof(T) != 4) {
            return false;
        } else {
            const int path = ctx->ttm_path;
            // auto: every contraction the tensor-core kernels take (Y passes; later M-major
            // stages, split over K when their row tiles cannot fill the GPU; K-major stages)
            if (path == 1 || U.size() <= size_t(m) || !U[m]) return false;
            const float* fin = reinterpret_cast<const float*>(in);
            float* fout = reinterpret_cast<float*>(out);
            // the Y passes (and the second stages that tile the GPU): second-design streaming
            // kernel (ttm_stream.cu); K-major only with the transposed output
            if ((streams_y || stream_second_ok(in, out, P, K, Q, cols[m])) && stream_ttm_enabled() &&
                (P != 1 || tout) && stream_ttm_supported(fin, fout, P, K, Q, cols[m])) {
                void* bpk = ctx->buf(streams_y ? "stream_pack" : "stream_pack2",
                                     static_cast<size_t>(stream_pack_bytes(K, cols[m])));
                launch_pack_stream(U[m] + off[m], gdims[m], K, cols[m], bpk, s);
                if (streams_y && time_kernels) mark();
                launch_ttm_stream(fin, bpk, fout, P, K, Q, cols[m], s);
                launches += 2;
                if (P == 1) *tout = true;
                if (streams_y && time_kernels) mark();
                return true;
            }
            const int64_t welems = std::min<int64_t>(P * cols[m] * Q * 16, int64_t(64) << 20);
            if (!tc_ttm_supported(fin, fout, P, K, Q, cols[m], welems)) return false;
            void* bpk = ctx->buf(streams_y ? "umma_pack" : "umma_pack2", static_cast<size_t>(umma_pack_bytes(K, cols[m])));
            const double* u = U[m] + off[m];
            launch_pack_umma(u, gdims[m], K, cols[m], bpk, s);
            if (streams_y && time_kernels) mark();
            const bool tr = tout && P == 1;  // a mode-0 Y pass: transposed output
            float* work = static_cast<float*>(
                ctx->buf(work_name == std::string("splitk") ? "splitk_tc" : "splitk_tc_side", sizeof(float) * welems));
            launches += 1 + launch_ttm_tc(fin, bpk, fout, P, K, Q, cols[m], s, /*accurate=*/true, tr, work, welems);
            if (tr) *tout = true;
            if (streams_y && time_kernels) mark();
            return true;
        }
    }

    void ttm(const T* in, const T* up, T* out, int64_t P, int64_t K, int64_t Q, int c) {
        const int64_t welems = std::min<int64_t>(P * c * Q * 2 * 148, int64_t(32) << 20);
        T* work = static_cast<T*>(ctx->buf(work_name, sizeof(T) * welems));
        launch_ttm<T>(in, up, out, P, K, Q, c, s, &launches, work, welems);
    }

    void allreduce(double* buf, int64_t count) {
        if (!ctx->has_comm) return;
        if (ctx->nccl) {  // in place, on this call's stream (captured into the graph when capturing)
            nccl_check(nccl_api().all_reduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum, ctx->nccl, s),
                       "ncclAllReduce");
            return;
        }
        if (ctx->comm.world <= 1) return;
        const tk_comm& c = ctx->comm;
        require(count <= c.xbuf_capacity, "comm: exchange buffer too small");
        if (buf != c.xbuf) TK_CUDA(cudaMemcpyAsync(c.xbuf, buf, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
        require(c.allreduce_sum(c.user, count, s) == 0, "comm: allreduce failed");
        if (buf != c.xbuf) TK_CUDA(cudaMemcpyAsync(buf, c.xbuf, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }

    // Z = unfold(X, n) * Omega (tensor.hpp:195-209) straight into fp64 z (leading dimension
    // ldz) for the QR: one split-K kernel over the (B, I, A) view, no materialised unfolding.
    // x stored with mode order xp; omp must hold Omega's rows in the matching column order.
    void sketch(const T* x, const std::vector<int64_t>& xd, const std::vector<int>& xp, int n, const T* omp, int rn,
                double* z, int64_t ldz) {
        const int k = pos_of(xp, n);
        const int64_t B = prod(std::vector<int64_t>(xd.begin(), xd.begin() + k));
        const int64_t I = xd[k];
        const int64_t A = prod(std::vector<int64_t>(xd.begin() + k + 1, xd.end()));
        double* work = static_cast<double*>(ctx->buf(work_name == std::string("splitk") ? "sketch_part" : "sketch_part_side",
                                                     sizeof(double) * sketch_work_elems(I, rn)));
        launches += launch_sketch<T>(x, B, I, A, omp, rn, z, ldz, work, s);
    }

    // One range-finding step for mode n: Z = unfold(X, n) Omega, U_n = basis(Z)
    void range_step(const T* x, const std::vector<int64_t>& xd, const std::vector<int>& xp, int n,
                    const Seed& omega_seed, int step, bool sync) {
        const int64_t W = prod(std::vector<int64_t>(cols.begin(), cols.end()), n);
        const int rn = rt[n];
        T* omp = static_cast<T*>(ctx->buf("omega_p", sizeof(T) * W * pack_stride(rn)));
        ph_begin(2);
        // Omega rows follow the unfolding's columns (modes != n ascending, tensor.hpp:103-116);
        // for a permuted x its storage columns map to them through a mixed-radix RowMap
        bool ordered = true;
        RowMap map;
        {
            std::vector<int64_t> stride(static_cast<size_t>(order), 0);
            int64_t st = 1;
            for (int m = 0; m < order; ++m)
                if (m != n) stride[m] = st, st *= cols[m];
            int prev = -1;
            for (int k = 0; k < order; ++k) {
                if (xp[k] == n) continue;
                ordered = ordered && xp[k] > prev;
                prev = xp[k];
                map.lext[map.nd] = xd[k];
                map.gstride[map.nd] = stride[xp[k]];
                ++map.nd;
            }
            map.rows_total = W;
        }
        if (ordered) launch_gaussian_packed<T>(omp, W, rn, omega_seed.key(), s);
        else launch_gaussian_packed_map<T>(omp, W, rn, omega_seed.key(), map, s);
        ++launches;
        const int64_t In = gdims[n];
        double* z = static_cast<double*>(ctx->buf("z", sizeof(double) * In * rn));
        const bool ranks_sum = ctx->has_comm && ctx->comm.world > 1;
        int nparts = 0;
        if (ldims[n] != In) {  // this rank's rows of Z, the others zero (summed over ranks)
            TK_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * In * rn, s));
            sketch(x, xd, xp, n, omp, rn, z + off[n], In);
        } else if (!ranks_sum && qr_fuse() && ctx->ortho != TK_ORTHO_GRAM && qr_work_elems(In, rn) == 0) {  // the QR sums the split-K partials while loading Z
            const int k = pos_of(xp, n);
            const int64_t B = prod(std::vector<int64_t>(xd.begin(), xd.begin() + k));
            const int64_t A = prod(std::vector<int64_t>(xd.begin() + k + 1, xd.end()));
            z = static_cast<double*>(ctx->buf(work_name == std::string("splitk") ? "sketch_part" : "sketch_part_side",
                                              sizeof(double) * sketch_work_elems(In, rn)));
            nparts = launch_sketch_partials<T>(x, B, In, A, omp, rn, z, s, 16);  // the QR load sums <= 16
            ++launches;
        } else {
            sketch(x, xd, xp, n, omp, rn, z, In);
        }
        ph_end();
        if (!fver.empty()) ++fver[n];  // U_n is rewritten below
        if (!nparts) allreduce(z, In * rn);
        if (qr_event) TK_CUDA(cudaEventRecord(qr_event, s));
        ph_begin(3);
        if (ctx->ortho == TK_ORTHO_GRAM) {
            double* gw = static_cast<double*>(ctx->buf("gram_work", sizeof(double) * gram_work_elems(In, rn)));
            launches += launch_gram_orthonormal(z, In, In, rn, U[n], rt[n], Up[n], sizeof(T) == 4 ? kF32 : kF64,
                                                rank_dev + step, nullptr, gw, s);
        } else {
            const int64_t qw = qr_work_elems(In, rn);  // > 0: taller than one cluster holds (blocked path)
            double* qwork = qw ? static_cast<double*>(ctx->buf("qr_work", sizeof(double) * qw)) : nullptr;
            launches += launch_orthonormal_basis(z, In, rn, U[n], rt[n], Up[n], sizeof(T) == 4 ? kF32 : kF64,
                                                 rank_dev + step, nullptr, s, nparts, margins_dev + 3 * step, qwork);
        }
        ph_end();
        if (sync) sync_rank(n, step);
    }

    void sync_rank(int n, int step) {
        TK_CUDA(cudaMemcpyAsync(ctx->rank_host, rank_dev + step, sizeof(int), cudaMemcpyDeviceToHost, s));
        TK_CUDA(cudaStreamSynchronize(s));
        const int r = *ctx->rank_host;
        require(r >= 1, "tensor dimensions must be positive");  // a rank-0 factor (zero data)
        cols[n] = r;
    }

    void run(const std::vector<int64_t>& ranks, int64_t p, const Seed& seed, const tk_tucker_opts& opt,
             tk_tucker_out* out, tk_tucker_stats* stats) {
        rt.resize(order);
        cols.resize(order);
        U.resize(order);
        Up.resize(order);
        fver.assign(order, 0);
        fc = FirstCache{};
        for (int n = 0; n < order; ++n) {
            rt[n] = static_cast<int>(std::min<int64_t>(ranks[n] + p, gdims[n]));
            require(rt[n] >= 1, "gaussian_matrix: dimensions must be positive");
            require(rt[n] <= kMaxRank, "rank + oversample must be <= 64 on this device path");
            cols[n] = rt[n];
            U[n] = static_cast<double*>(ctx->buf("U" + std::to_string(n), sizeof(double) * gdims[n] * rt[n]));
            Up[n] = static_cast<T*>(ctx->buf("Up" + std::to_string(n), sizeof(T) * gdims[n] * pack_stride(rt[n])));
            launch_gaussian_colmajor(U[n], gdims[n], rt[n], alg3_init_seed(seed, n).key(), s);
            launch_pack_factor<T>(U[n], gdims[n], gdims[n], rt[n], Up[n], s);
            launches += 2;
        }
        rank_dev = static_cast<int*>(ctx->buf("ranks", sizeof(int) * 2 * TK_MAX_ORDER));
        margins_dev = static_cast<double*>(ctx->buf("margins", sizeof(double) * 3 * 2 * TK_MAX_ORDER));
        TK_CUDA(cudaMemsetAsync(margins_dev, 0, sizeof(double) * 3 * 2 * TK_MAX_ORDER, s));
        const bool sync = opt.sync_ranks != 0;
        const T* xlast = nullptr;
        std::vector<int64_t> xd;
        // Steps (pass, n). Consecutive steps with distinct modes form a group that shares ONE Y
        // pass: the group's first-stage contraction is over a mode m outside the group (its
        // factor is final for every step of the group), so T = Y x_m U_m^T serves them all and
        // each step only contracts T with the group's other factors (N = 3: 6 steps -> 3 Y
        // passes; N = 4: 8 -> 3). opt.one_pass_per_step = 1 keeps one pass per step. A group's
        // Y pass that does not contract the factor the previous step's QR is producing is
        // launched on the side stream right after that QR, so the latency-bound QR runs under
        // the bandwidth-bound pass (2 of the 148 SMs for the QR cluster).
        const int nsteps = 2 * static_cast<int>(order);
        const bool overlap = opt.overlap && order > 1;
        if (overlap) ctx->ensure_side();
        struct Group {
            int s, e, leader;
        };
        std::vector<Group> groups;
        for (int st = 0; st < nsteps;) {
            const int avoid = st > 0 ? (st - 1) % static_cast<int>(order) : -1;
            Group g{st, st + 1, order == 1 ? -1 : first_mode(st % static_cast<int>(order), avoid)};
            while (opt.one_pass_per_step == 0 && order > 2 && g.e < nsteps) {
                uint32_t mask = 0;
                bool distinct = true;
                for (int k = g.s; k <= g.e; ++k) {
                    const uint32_t bit = 1u << (k % static_cast<int>(order));
                    distinct = distinct && !(mask & bit);
                    mask |= bit;
                }
                const int l = distinct ? leader_mode(mask, avoid) : -1;
                if (l < 0) break;
                g.e += 1;
                g.leader = l;
            }
            groups.push_back(g);
            st = g.e;
        }
        std::vector<int64_t> d1;
        std::vector<int> p1, xp;
        const T* t1 = nullptr;
        int f = -1;
        bool on_side = false;
        auto launch_first = [&](int leader, bool side) {
            f = leader;
            on_side = side && f >= 0;
            if (on_side) {
                TK_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_free, 0));  // finish() done with proj1
                cudaStream_t keep = s;
                s = ctx->side;
                work_name = "splitk_side";
                t1 = first_stage(f, d1, p1);
                TK_CUDA(cudaEventRecord(ctx->ev_fs, s));
                s = keep;
                work_name = "splitk";
            } else {
                t1 = first_stage(f, d1, p1);
            }
        };
        launch_first(groups[0].leader, false);
        for (size_t gi = 0; gi < groups.size(); ++gi) {
            const Group& g = groups[gi];
            for (int step = g.s; step < g.e; ++step) {
                const int pass = step / static_cast<int>(order), n = step % static_cast<int>(order);
                if (on_side && step == g.s) TK_CUDA(cudaStreamWaitEvent(s, ctx->ev_fs, 0));
                xd = d1;
                xp = p1;
                const T* x = (order == 1) ? y : finish(t1, xd, xp, n, f);
                const bool last = step + 1 == g.e;
                const bool next = gi + 1 < groups.size();
                // the sketch must not read proj1; the next pass must not need this step's U_n
                const bool can_overlap = overlap && x != t1 && last && next && groups[gi + 1].leader != n;
                qr_event = can_overlap ? ctx->ev_free : nullptr;  // recorded right before this step's QR
                range_step(x, xd, xp, n, alg3_omega_seed(seed, pass, n), step, false);
                qr_event = nullptr;
                xlast = x;
                if (can_overlap) {
                    launch_first(groups[gi + 1].leader, true);  // independent of this QR
                    if (sync) sync_rank(n, step);
                } else {
                    if (sync) sync_rank(n, step);
                    if (last && next) launch_first(groups[gi + 1].leader, false);
                }
            }
        }
        group_count = static_cast<int>(groups.size());
        if (!sync && !capture) {  // verify the full-rank speculation
            int hr[2 * TK_MAX_ORDER];
            TK_CUDA(cudaMemcpyAsync(hr, rank_dev, sizeof(int) * 2 * order, cudaMemcpyDeviceToHost, s));
            TK_CUDA(cudaStreamSynchronize(s));
            for (int i = 0; i < 2 * order; ++i)
                if (hr[i] != rt[i % order]) throw std::runtime_error("rank-drop");  // caller reruns synchronously
        }
        // core
        std::vector<int64_t> gd;  // core extents in storage order, then standard order
        const T* g;
        if (opt.explicit_core_pass || order == 1) {
            g = project(-1, gd, xp);
        } else {
            gd = xd;  // X_{N-1}: cols everywhere except mode N-1 (local extent)
            const int m = static_cast<int>(order - 1);
            const int k = pos_of(xp, m);
            const int64_t P = prod(std::vector<int64_t>(gd.begin(), gd.begin() + k));
            const int64_t Q = prod(std::vector<int64_t>(gd.begin() + k + 1, gd.end()));
            T* o = static_cast<T*>(ctx->buf("core", sizeof(T) * P * cols[m] * Q));
            ph_begin(4);
            ttm(xlast, factor_rows(m), o, P, gd[k], Q, cols[m]);
            ph_end();
            gd[k] = cols[m];
            g = o;
        }
        const int64_t gsize = prod(gd);
        double* gdv = static_cast<double*>(ctx->buf("core64", sizeof(double) * gsize));
        if (xp == ident()) {
            if constexpr (sizeof(T) == 4) launch_cast<float, double>(reinterpret_cast<const float*>(g), gdv, gsize, s);
            else launch_cast<double, double>(reinterpret_cast<const double*>(g), gdv, gsize, s);
        } else {  // back to the standard mode order
            std::vector<int64_t> sd(static_cast<size_t>(order));
            for (int k = 0; k < order; ++k) sd[xp[k]] = gd[k];
            gd = sd;
            launch_permute_cast<T, double>(g, gdv, static_cast<int>(order), gd.data(), xp.data(), s);
        }
        ++launches;
        allreduce(gdv, gsize);
        ph_report();
        if (capture) {
            core_out = gdv;
            core_shape = gd;
            return;
        }
        // outputs
        const cudaMemcpyKind kind = out->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        TK_CUDA(cudaMemcpyAsync(out->core, gdv, sizeof(double) * gsize, kind, s));
        for (int n = 0; n < order; ++n) {
            out->core_shape[n] = gd[n];
            out->factor_cols[n] = cols[n];
            TK_CUDA(cudaMemcpyAsync(out->factors[n], U[n], sizeof(double) * gdims[n] * cols[n], kind, s));
        }
        if (stats) {
            stats->passes = passes;
            stats->kernel_launches = launches;
            stats->stream_launches = passes;
            stats->stream_ms = time_kernels ? streamed_ms() : 0.0;
            stats->y_bytes = static_cast<double>(prod(ldims)) * sizeof(T);
            int hr[2 * TK_MAX_ORDER] = {0};
            TK_CUDA(cudaMemcpyAsync(hr, rank_dev, sizeof(int) * 2 * order, cudaMemcpyDeviceToHost, s));
            TK_CUDA(cudaStreamSynchronize(s));
            for (int i = 0; i < 2 * order; ++i) stats->ranks[i] = hr[i];
            read_margins(ctx, order, s, stats);
        }
        if (!out->on_device) TK_CUDA(cudaStreamSynchronize(s));
    }
};

// rand_tucker (Alg. 2, tucker.hpp:108-130): Z = unfold(cur, n) * Omega (dense Omega of
// width prod_{k != n} cur.dim(k), regenerated from the seed), U_n = basis(Z),
// cur <- cur x_n U_n^T; the core is the final cur. Single device.
template <typename T>
void rand_tucker_impl(tk_context* ctx, int64_t order, const int64_t* dims, const void* y, int y_on_device,
                      const int64_t* ranks, int64_t p, Seed seed, tk_tucker_out* out, tk_tucker_stats* stats) {
    cudaStream_t s = ctx->stream;
    std::vector<int64_t> cd(dims, dims + order);  // current (local) extents
    std::vector<int64_t> gd, lo;                  // global extents, block offsets (dist.hpp:24-123)
    block_of(ctx, cd, gd, lo);
    const T* cur = static_cast<const T*>(y);
    if (!y_on_device) {
        T* buf = static_cast<T*>(ctx->buf("y_in", sizeof(T) * prod(cd)));
        TK_CUDA(cudaMemcpyAsync(buf, y, sizeof(T) * prod(cd), cudaMemcpyHostToDevice, s));
        cur = buf;
    }
    TuckerRun<T> r{ctx, s, order, cd, gd, lo, cur};
    r.rank_dev = static_cast<int*>(ctx->buf("ranks", sizeof(int) * 2 * TK_MAX_ORDER));
    double* margins = static_cast<double*>(ctx->buf("margins", sizeof(double) * 3 * 2 * TK_MAX_ORDER));
    TK_CUDA(cudaMemsetAsync(margins, 0, sizeof(double) * 3 * 2 * TK_MAX_ORDER, s));
    std::vector<double*> U(order);
    std::vector<int64_t> fcols(order);
    int which = 0;
    for (int n = 0; n < order; ++n) {
        const int rt = static_cast<int>(std::min<int64_t>(ranks[n] + p, gd[n]));
        require(rt >= 1, "gaussian_matrix: dimensions must be positive");
        require(rt <= kMaxRank, "rank + oversample must be <= 64 on this device path");
        // Omega_n: (global width) x rt. Column c of this rank's mode-n unfolding sits at global
        // column sum_k (lo_k + digit_k) * stride_k of the global unfolding (modes k != n ascending,
        // already contracted modes at their full rank with lo = 0): streamed_block_product,
        // dist.hpp:496-596.
        const int64_t width = prod(cd) / cd[n];
        RowMap map;
        map.rows_total = 1;
        for (int k = 0; k < order; ++k) {
            if (k == n) continue;
            const int64_t ge = k < n ? cd[k] : gd[k];
            map.lext[map.nd] = cd[k];
            map.lo[map.nd] = k < n ? 0 : lo[k];
            map.gstride[map.nd] = map.rows_total;
            map.rows_total *= ge;
            ++map.nd;
        }
        const Seed os = alg2_omega_seed(seed, n);
        double* z = static_cast<double*>(ctx->buf("z", sizeof(double) * gd[n] * rt));
        T* op = static_cast<T*>(ctx->buf("omega_packed", sizeof(T) * width * pack_stride(rt)));
        launch_gaussian_packed_map<T>(op, width, rt, os.key(), map, s);
        const bool part = cd[n] != gd[n];  // a partitioned mode: own rows of Z, the others zero
        if (part) TK_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * gd[n] * rt, s));
        double* zown = z + lo[n];
        if (n == 0) {  // contiguous unfolding: Z = Y_(0) Omega, split-K TTM
            T* zt = static_cast<T*>(ctx->buf("zt", sizeof(T) * cd[0] * rt));
            r.ttm(cur, op, zt, cd[0], width, 1, rt);
            if constexpr (sizeof(T) == 4)
                launch_cast2d<float, double>(reinterpret_cast<const float*>(zt), cd[0], zown, gd[0], cd[0], rt, s);
            else
                launch_cast2d<double, double>(reinterpret_cast<const double*>(zt), cd[0], zown, gd[0], cd[0], rt, s);
            r.launches += 2;
        } else {
            r.sketch(cur, cd, r.ident(), n, op, rt, zown, gd[n]);
            ++r.launches;
        }
        r.allreduce(z, gd[n] * rt);  // partial sketches summed over ranks (no-op on one rank)
        U[n] = static_cast<double*>(ctx->buf("U" + std::to_string(n), sizeof(double) * gd[n] * rt));
        T* up = static_cast<T*>(ctx->buf("Up" + std::to_string(n), sizeof(T) * gd[n] * pack_stride(rt)));
        if (ctx->ortho == TK_ORTHO_GRAM) {
            double* gw = static_cast<double*>(ctx->buf("gram_work", sizeof(double) * gram_work_elems(gd[n], rt)));
            r.launches += launch_gram_orthonormal(z, gd[n], gd[n], rt, U[n], rt, up, sizeof(T) == 4 ? kF32 : kF64,
                                                  r.rank_dev + n, nullptr, gw, s);
        } else {
            const int64_t qw = qr_work_elems(gd[n], rt);
            double* qwork = qw ? static_cast<double*>(ctx->buf("qr_work", sizeof(double) * qw)) : nullptr;
            r.launches += launch_orthonormal_basis(z, gd[n], rt, U[n], rt, up, sizeof(T) == 4 ? kF32 : kF64,
                                                   r.rank_dev + n, nullptr, s, 0, margins + 3 * n, qwork);
        }
        TK_CUDA(cudaMemcpyAsync(ctx->rank_host, r.rank_dev + n, sizeof(int), cudaMemcpyDeviceToHost, s));
        TK_CUDA(cudaStreamSynchronize(s));
        const int rank = *ctx->rank_host;
        require(rank >= 1, "tensor dimensions must be positive");
        fcols[n] = rank;
        const int64_t P = prod(std::vector<int64_t>(cd.begin(), cd.begin() + n));
        const int64_t Q = prod(std::vector<int64_t>(cd.begin() + n + 1, cd.end()));
        T* nxt = static_cast<T*>(ctx->buf(which ? "a2B" : "a2A", sizeof(T) * P * rank * Q));
        const T* upl = up + lo[n] * pack_stride(rank);  // this rank's rows of U
        bool done = false;
        if constexpr (sizeof(T) == 4) {  // the Y-sized mode-0 shrink on the tensor cores (K-major)
            if (n == 0 && P == 1 && ctx->ttm_path != 1 &&
                tc_ttm_supported(reinterpret_cast<const float*>(cur), reinterpret_cast<float*>(nxt), 1, cd[0], Q, rank)) {
                void* bpk = ctx->buf("umma_pack", static_cast<size_t>(umma_pack_bytes(cd[0], rank)));
                launch_pack_umma(U[0] + lo[0], gd[0], cd[0], rank, bpk, s);
                launch_ttm_tc(reinterpret_cast<const float*>(cur), bpk, reinterpret_cast<float*>(nxt), 1, cd[0], Q, rank, s,
                              true);
                r.launches += 2;
                done = true;
            }
        }
        if (!done) r.ttm(cur, upl, nxt, P, cd[n], Q, rank);
        if (n == 0) ++r.passes;
        cd[n] = rank;
        cur = nxt;
        which ^= 1;
    }
    const int64_t gsize = prod(cd);
    double* gdv = static_cast<double*>(ctx->buf("core64", sizeof(double) * gsize));
    if constexpr (sizeof(T) == 4) launch_cast<float, double>(reinterpret_cast<const float*>(cur), gdv, gsize, s);
    else launch_cast<double, double>(reinterpret_cast<const double*>(cur), gdv, gsize, s);
    r.allreduce(gdv, gsize);  // partial cores summed over ranks
    const cudaMemcpyKind kind = out->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    TK_CUDA(cudaMemcpyAsync(out->core, gdv, sizeof(double) * gsize, kind, s));
    for (int n = 0; n < order; ++n) {
        out->core_shape[n] = cd[n];
        out->factor_cols[n] = fcols[n];
        TK_CUDA(cudaMemcpyAsync(out->factors[n], U[n], sizeof(double) * gd[n] * fcols[n], kind, s));
    }
    if (stats) {
        stats->passes = r.passes + 1;  // the Z sketch of mode 0 streams Y as well
        stats->kernel_launches = r.launches + 1;
        stats->y_bytes = static_cast<double>(prod(std::vector<int64_t>(dims, dims + order))) * sizeof(T);
        for (int n = 0; n < order; ++n) stats->ranks[n] = static_cast<int>(fcols[n]);
        read_margins(ctx, order, s, stats, order);
    }
    TK_CUDA(cudaStreamSynchronize(s));
}

// A/B knob: TENKIT_QR_FUSE=1 lets the QR kernel sum the sketch partials while loading Z (one
// launch less per step, but 8 SMs read the partials: measured ~20 us slower per decomposition
// at cfg 2 than the whole-GPU reduce kernel, so off by default)
bool qr_fuse() {
    static const bool on = [] {
        const char* e = std::getenv("TENKIT_QR_FUSE");
        return e && e[0] == '1';
    }();
    return on;
}

bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TENKIT_NO_GRAPH");
        return !(e && e[0] == '1');
    }();
    return on;
}

// Replays (or, on the second identical call, captures) the decomposition as a CUDA graph on
// the context's private stream, then copies the model out and verifies the speculated ranks.
// Returns false when the eager path must run (first sighting of this call, or a rank drop).
template <typename T>
bool graph_2i(tk_context* ctx, int64_t order, const std::vector<int64_t>& ld, const std::vector<int64_t>& gd,
              const std::vector<int64_t>& off, const T* ydev, const std::vector<int64_t>& rk, int64_t p,
              const Seed& seed, const tk_tucker_opts& opt, tk_tucker_out* out, tk_tucker_stats* stats,
              const float* y32 = nullptr) {
    std::string key = std::to_string(sizeof(T)) + "|" + std::to_string(reinterpret_cast<uintptr_t>(ydev)) + "|" +
                      std::to_string(reinterpret_cast<uintptr_t>(y32)) + "|" +
                      std::to_string(p) + "|" + std::to_string(seed.root) + "|" + std::to_string(seed.stream) + "|" +
                      std::to_string(opt.explicit_core_pass) + std::to_string(opt.overlap) + std::to_string(opt.one_pass_per_step) +
                      std::to_string(opt.time_kernels) + "|" + std::to_string(ctx->ttm_path) + "|" + std::to_string(ctx->ortho) +
                      "|nccl" + std::to_string(ctx->has_comm && ctx->nccl ? ctx->nccl_gen : 0);
    for (int64_t n = 0; n < order; ++n)
        key += "|" + std::to_string(ld[n]) + "x" + std::to_string(rk[n]) + "@" + std::to_string(off[n]) + "/" +
               std::to_string(gd[n]);
    auto& g = ctx->g2i;
    if (g.key != key || (g.exec && g.buf_gen != ctx->buf_gen)) {
        g.reset();
        g.key = key;
    }
    if (!g.exec) {
        if (g.seen++ == 0) return false;  // first sighting: eager (allocates every buffer)
        if (!ctx->cap) {
            TK_CUDA(cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking));
            TK_CUDA(cudaEventCreateWithFlags(&ctx->ev_cap, cudaEventDisableTiming));
        }
        ctx->ensure_side();
        TuckerRun<T> r{ctx, ctx->cap, order, ld, gd, off, ydev};
        r.y32 = y32;
        r.time_kernels = opt.time_kernels != 0;
        r.capture = true;
        cudaGraph_t graph = nullptr;
        TK_CUDA(cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeThreadLocal));
        try {
            r.run(rk, p, seed, opt, out, nullptr);
        } catch (...) {
            cudaStreamEndCapture(ctx->cap, &graph);
            if (graph) cudaGraphDestroy(graph);
            g.reset();
            throw;
        }
        TK_CUDA(cudaStreamEndCapture(ctx->cap, &graph));
        const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        TK_CUDA(ie);
        g.marks.swap(r.ev);  // the graph records these events on every replay
        g.core = r.core_out;
        g.cshape = r.core_shape;
        g.gsize = prod(r.core_shape);
        g.U = r.U;
        g.cols = std::vector<int64_t>(r.cols.begin(), r.cols.end());
        g.rt = r.rt;
        g.passes = r.passes;
        g.launches = r.launches;
        g.buf_gen = ctx->buf_gen;
    }
    cudaStream_t s = ctx->stream;
    TK_CUDA(cudaGraphLaunch(g.exec, s));
    int hr[2 * TK_MAX_ORDER] = {0};
    const int* rank_dev = static_cast<const int*>(ctx->buf("ranks", sizeof(int) * 2 * TK_MAX_ORDER));
    TK_CUDA(cudaMemcpyAsync(hr, rank_dev, sizeof(int) * 2 * order, cudaMemcpyDeviceToHost, s));
    const cudaMemcpyKind kind = out->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    TK_CUDA(cudaMemcpyAsync(out->core, g.core, sizeof(double) * g.gsize, kind, s));
    for (int64_t n = 0; n < order; ++n) {
        out->core_shape[n] = g.cshape[n];
        out->factor_cols[n] = g.cols[n];
        TK_CUDA(cudaMemcpyAsync(out->factors[n], g.U[n], sizeof(double) * gd[n] * g.cols[n], kind, s));
    }
    TK_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < 2 * order; ++i)
        if (hr[i] != g.rt[i % order]) return false;  // a rank dropped: rerun eagerly (synchronous ranks)
    if (stats) {
        stats->passes = g.passes;
        stats->kernel_launches = g.launches;
        stats->stream_launches = g.passes;
        double ms = 0.0;
        for (size_t i = 0; i + 1 < g.marks.size(); i += 2) {
            float t = 0.f;
            TK_CUDA(cudaEventElapsedTime(&t, g.marks[i], g.marks[i + 1]));
            ms += t;
        }
        stats->stream_ms = ms;
        stats->y_bytes = static_cast<double>(prod(ld)) * (y32 ? sizeof(float) : sizeof(T));
        for (int i = 0; i < 2 * order; ++i) stats->ranks[i] = hr[i];
        read_margins(ctx, order, s, stats);
    }
    return true;
}

template <typename T>
void rand_tucker_2i_impl(tk_context* ctx, int64_t order, const int64_t* dims, const void* y, int y_on_device,
                         const int64_t* ranks, int64_t p, Seed seed, const tk_tucker_opts& opt, tk_tucker_out* out,
                         tk_tucker_stats* stats, const float* y32 = nullptr) {
    std::vector<int64_t> ld(dims, dims + order), rk(ranks, ranks + order);
    std::vector<int64_t> gd, offset;
    block_of(ctx, ld, gd, offset);
    const T* ydev = static_cast<const T*>(y);
    const T* land = nullptr;  // host input: copied in by the run's first Y pass (land_stream / land_all)
    if (!y_on_device && !y32) {
        ydev = static_cast<T*>(ctx->buf("y_in", sizeof(T) * prod(ld)));
        land = static_cast<const T*>(y);
    }
    auto attempt = [&](const tk_tucker_opts& o) {
        TuckerRun<T> r{ctx, ctx->stream, order, ld, gd, offset, ydev};
        r.land_src = land;
        land = nullptr;  // a rerun (rank drop) finds the tensor in the landing buffer
        r.y32 = y32;
        r.time_kernels = o.time_kernels != 0;
        r.run(rk, p, seed, o, out, stats);
        if (stats && y32) stats->y_bytes = static_cast<double>(prod(ld)) * sizeof(float);
    };
    // graphs: single process, or a native NCCL communicator (its all-reduces are captured);
    // the host-callback hook runs eagerly
    if (!opt.sync_ranks && (y_on_device || y32) && !(ctx->has_comm && ctx->comm.world > 1 && !ctx->nccl) &&
        graphs_enabled() && graph_2i<T>(ctx, order, ld, gd, offset, ydev, rk, p, seed, opt, out, stats, y32))
        return;
    if (opt.sync_ranks) {
        attempt(opt);
    } else {
        try {
            attempt(opt);
        } catch (const std::runtime_error& e) {
            if (std::string(e.what()) != "rank-drop") throw;
            tk_tucker_opts o2 = opt;
            o2.sync_ranks = 1;
            attempt(o2);
        }
    }
}

// precision = fp64 on fp32 data (tk_tucker_opts.precision = 1): the reference's own precision
// on the fp32 tensor. Small tensors (fp64 copy <= 2 GB) are cast to fp64 once and run the fp64
// path; large ones keep the fp32 tensor and run their Y passes in fp64 arithmetic over it
// (ttm_mixed.cu), everything after the first stage in fp64.
void rand_tucker_2i_fp64_on_f32(tk_context* ctx, int64_t order, const int64_t* dims, const void* y, int y_on_device,
                                const int64_t* ranks, int64_t p, Seed seed, const tk_tucker_opts& opt,
                                tk_tucker_out* out, tk_tucker_stats* stats) {
    const int64_t n = prod(std::vector<int64_t>(dims, dims + order));
    const float* y32 = static_cast<const float*>(y);
    if (!y_on_device) {
        float* buf = static_cast<float*>(ctx->buf("y_in", sizeof(float) * n));
        TK_CUDA(cudaMemcpyAsync(buf, y, sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        y32 = buf;
    }
    if (n * int64_t(sizeof(double)) <= (int64_t(2) << 30)) {
        double* y64 = static_cast<double*>(ctx->buf("y_fp64", sizeof(double) * n));
        launch_cast<float, double>(y32, y64, n, ctx->stream);
        rand_tucker_2i_impl<double>(ctx, order, dims, y64, 1, ranks, p, seed, opt, out, stats);
        if (stats) stats->y_bytes = static_cast<double>(n) * sizeof(float);  // the caller's fp32 tensor
        return;
    }
    rand_tucker_2i_impl<double>(ctx, order, dims, nullptr, 1, ranks, p, seed, opt, out, stats, y32);
}

void validate_common(int dtype, int64_t order, const int64_t* dims, const int64_t* ranks, int64_t p,
                     const char* who) {
    require(dtype == TK_F32 || dtype == TK_F64, "unsupported dtype");
    require(order >= 1 && order <= TK_MAX_ORDER, "tensor order must be in [1, 8]");
    for (int64_t n = 0; n < order; ++n) require(dims[n] >= 1, "tensor dimensions must be positive");
    require(ranks != nullptr, std::string(who) + ": one rank per mode required");
    require(p >= 0, std::string(who) + ": oversampling must be nonnegative");
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* tk_last_error(void) { return g_err.c_str(); }
int tk_version(void) { return 1; }

int tk_device_ok(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
        cudaGetLastError();
        return 0;
    }
    cudaDeviceProp pr{};
    if (cudaGetDeviceProperties(&pr, 0) != cudaSuccess) return 0;
    return pr.major == 10 ? 1 : 0;
}

namespace {
struct CtxPool : tkb::BufPool {
    tk_context* c;
    explicit CtxPool(tk_context* ctx) : c(ctx) {}
    void* get(const std::string& name, size_t bytes) override { return c->buf(name, bytes); }
};
}  // namespace

int tk_context_create(int device, tk_context** out) {
    if (!tk_device_ok()) return fail(TK_ERR_NO_DEVICE, "tenkit: no sm_100 CUDA device available (no CPU fallback)");
    return guarded([&] {
        require(out != nullptr, "null output");
        auto ctx = std::make_unique<tk_context>();
        if (device < 0) TK_CUDA(cudaGetDevice(&device));  // -1: the calling thread's current device
        ctx->device = device;
        TK_CUDA(cudaSetDevice(device));
        TK_CUDA(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
        ctx->stream = ctx->own;
        TK_CUDA(cudaMallocHost(&ctx->rank_host, sizeof(int) * 4));
        if (const char* e = std::getenv("TENKIT_TTM_PATH")) ctx->ttm_path = std::max(0, std::min(3, std::atoi(e)));  // A/B knob
        *out = ctx.release();
    });
}

int tk_context_destroy(tk_context* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        delete ctx;
    });
}

int tk_context_set_stream(tk_context* ctx, void* st) {
    return guarded([&] {
        check_ctx(ctx);
        ctx->stream = static_cast<cudaStream_t>(st);  // NULL: the legacy default stream (torch's default)
    });
}

int tk_context_set_comm(tk_context* ctx, const tk_comm* comm) {
    return guarded([&] {
        check_ctx(ctx);
        if (!comm) {
            ctx->has_comm = false;
            return;
        }
        require(comm->world >= 1 && comm->rank >= 0 && comm->rank < comm->world, "comm: bad rank/world");
        if (ctx->nccl)
            require(comm->world == ctx->nccl_world && comm->rank == ctx->nccl_rank,
                    "comm: rank/world differ from the native NCCL communicator");
        else
            require(comm->world == 1 || (comm->allreduce_sum && comm->xbuf), "comm: missing reduction hook");
        ctx->comm = *comm;
        ctx->has_comm = true;
    });
}

int64_t tk_qr_max_rows(int64_t cols) { return cols >= 1 && cols <= kMaxRank ? qr_max_rows(static_cast<int>(cols)) : 0; }

int tk_nccl_unique_id(unsigned char* out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        ncclUniqueId id;
        nccl_check(nccl_api().get_unique_id(&id), "ncclGetUniqueId");
        static_assert(sizeof(id) == TK_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
        std::memcpy(out, &id, sizeof(id));
    });
}

int tk_nccl_version(void) {
    try {
        int v = 0;
        const NcclApi& a = nccl_api();
        if (a.get_version && a.get_version(&v) == ncclSuccess) return v;
    } catch (...) {
    }
    return 0;
}

int tk_context_set_nccl(tk_context* ctx, const unsigned char* id, int rank, int world) {
    return guarded([&] {
        check_ctx(ctx);
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->g2i.reset();  // captured graphs hold the old communicator's collectives
        ctx->drop_nccl();
        if (world == 0) return;  // tear down only
        require(id != nullptr && world >= 1 && rank >= 0 && rank < world, "nccl: bad rank/world");
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        ncclComm_t c = nullptr;
        nccl_check(nccl_api().comm_init_rank(&c, world, uid, rank), "ncclCommInitRank");
        ctx->nccl = c;
        ctx->nccl_rank = rank;
        ctx->nccl_world = world;
        ++ctx->nccl_gen;
        if (std::getenv("TENKIT_NCCL_VERBOSE"))
            std::fprintf(stderr, "tenkit: native NCCL communicator %d.%d rank %d of %d on device %d\n",
                         tk_nccl_version() / 10000, (tk_nccl_version() / 100) % 100, rank, world, ctx->device);
    });
}

int tk_context_set_ttm_path(tk_context* ctx, int path) {
    return guarded([&] {
        check_ctx(ctx);
        require(path >= 0 && path <= 3, "ttm path must be 0 (auto), 1 (FFMA), 2 (tcgen05) or 3 (streaming kernel)");
        ctx->ttm_path = path;
    });
}

int tk_context_set_orthonormalizer(tk_context* ctx, int kind) {
    return guarded([&] {
        check_ctx(ctx);
        require(kind == TK_ORTHO_COLPIV || kind == TK_ORTHO_GRAM,
                "orthonormalizer must be TK_ORTHO_COLPIV (0) or TK_ORTHO_GRAM (1)");
        ctx->ortho = kind;
    });
}

int tk_context_synchronize(tk_context* ctx) {
    return guarded([&] {
        check_ctx(ctx);
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int tk_rand_tucker_2i(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* y, int y_on_device,
                      const int64_t* ranks, int64_t oversample, uint64_t seed_root, uint64_t seed_stream,
                      const tk_tucker_opts* opts, tk_tucker_out* out, tk_tucker_stats* stats) {
    return guarded([&] {
        check_ctx(ctx);
        validate_common(dtype, order, dims, ranks, oversample, "rand_tucker_2i");
        require(out != nullptr && y != nullptr, "rand_tucker_2i: null argument");
        tk_tucker_opts o{0, 1, 0, 1, 0, 0};
        if (opts) o = *opts;
        const Seed seed{seed_root, seed_stream};
        require(o.precision == 0 || o.precision == 1, "rand_tucker_2i: precision must be 0 (native) or 1 (fp64)");
        if (dtype == TK_F32 && o.precision == 1)
            rand_tucker_2i_fp64_on_f32(ctx, order, dims, y, y_on_device, ranks, oversample, seed, o, out, stats);
        else if (dtype == TK_F32) rand_tucker_2i_impl<float>(ctx, order, dims, y, y_on_device, ranks, oversample, seed, o, out, stats);
        else rand_tucker_2i_impl<double>(ctx, order, dims, y, y_on_device, ranks, oversample, seed, o, out, stats);
    });
}

int tk_rand_tucker(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* y, int y_on_device,
                   const int64_t* ranks, int64_t oversample, uint64_t seed_root, uint64_t seed_stream,
                   tk_tucker_out* out, tk_tucker_stats* stats) {
    return guarded([&] {
        check_ctx(ctx);
        validate_common(dtype, order, dims, ranks, oversample, "rand_tucker");
        require(out != nullptr && y != nullptr, "rand_tucker: null argument");
        const Seed seed{seed_root, seed_stream};
        if (dtype == TK_F32) rand_tucker_impl<float>(ctx, order, dims, y, y_on_device, ranks, oversample, seed, out, stats);
        else rand_tucker_impl<double>(ctx, order, dims, y, y_on_device, ranks, oversample, seed, out, stats);
    });
}

int tk_ffcp_device(tk_context* ctx, int64_t order, const int64_t* core_shape, const double* core,
                   const double** factors, const int64_t* rows, int64_t rank, int constraint, double sparsity_c,
                   int max_iters, double fit_tol, uint64_t seed_root, uint64_t seed_stream, double** out_factors,
                   double* fit_trace, int* iterations) {
    return guarded([&] {
        check_ctx(ctx);
        require(order >= 2 && order <= TK_MAX_ORDER, "ffcp: tensor order must be at least 2");
        CtxPool pool(ctx);
        ffcp_device(pool, ctx->stream, order, core_shape, core, factors, rows, rank, constraint, sparsity_c, max_iters,
                    fit_tol, Seed{seed_root, seed_stream}, out_factors, fit_trace, iterations);
    });
}

int tk_ffcp(tk_context* ctx, int64_t order, const int64_t* core_shape, const double* core, const double** factors,
            const int64_t* rows, int64_t rank, int constraint, double sparsity_c, int max_iters, double fit_tol,
            uint64_t seed_root, uint64_t seed_stream, double** out_factors, double* fit_trace, int* iterations) {
    return guarded([&] {
        check_ctx(ctx);
        require(order >= 2 && order <= TK_MAX_ORDER, "ffcp: tensor order must be at least 2");
        require(rank >= 1, "ffcp: rank must be positive");
        cudaStream_t s = ctx->stream;
        int64_t gsz = 1;
        for (int64_t n = 0; n < order; ++n) gsz *= core_shape[n];
        double* dcore = static_cast<double*>(ctx->buf("ffcp_core", sizeof(double) * gsz));
        TK_CUDA(cudaMemcpyAsync(dcore, core, sizeof(double) * gsz, cudaMemcpyHostToDevice, s));
        std::vector<const double*> df(order);
        std::vector<double*> dout(order);
        for (int64_t n = 0; n < order; ++n) {
            double* u = static_cast<double*>(ctx->buf("ffcp_u" + std::to_string(n), sizeof(double) * rows[n] * core_shape[n]));
            TK_CUDA(cudaMemcpyAsync(u, factors[n], sizeof(double) * rows[n] * core_shape[n], cudaMemcpyHostToDevice, s));
            df[n] = u;
            dout[n] = static_cast<double*>(ctx->buf("ffcp_a" + std::to_string(n), sizeof(double) * rows[n] * rank));
        }
        CtxPool pool(ctx);
        ffcp_device(pool, s, order, core_shape, dcore, df.data(), rows, rank, constraint, sparsity_c, max_iters, fit_tol,
                    Seed{seed_root, seed_stream}, dout.data(), fit_trace, iterations);
        for (int64_t n = 0; n < order; ++n)
            TK_CUDA(cudaMemcpyAsync(out_factors[n], dout[n], sizeof(double) * rows[n] * rank, cudaMemcpyDeviceToHost, s));
        TK_CUDA(cudaStreamSynchronize(s));
    });
}

uint64_t tk_seed_derived(uint64_t root, uint64_t stream, uint64_t tag) { return Seed{root, stream}.derived(tag).stream; }

int tk_gaussian_matrix(tk_context* ctx, int64_t rows, int64_t cols, uint64_t root, uint64_t stream, double* out) {
    return guarded([&] {
        check_ctx(ctx);
        require(rows >= 1 && cols >= 1, "gaussian_matrix: dimensions must be positive");
        launch_gaussian_colmajor(out, rows, cols, Seed{root, stream}.key(), ctx->stream);
    });
}

int tk_model_fit(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* y,
                 const int64_t* core_shape, const double* core, const double** factors, int64_t rank, double* sums) {
    return guarded([&] {
        check_ctx(ctx);
        require(y != nullptr && factors != nullptr && sums != nullptr, "fit: null argument");
        require(order >= 2 && order <= TK_MAX_ORDER, "fit: tensor order must be in [2, 8]");
        for (int64_t n = 0; n < order; ++n) require(dims[n] >= 1, "tensor dimensions must be positive");
        require(core != nullptr || rank >= 1, "fit: CP rank must be positive");
        CtxPool pool(ctx);
        double* d = static_cast<double*>(ctx->buf("fit_sums", 2 * sizeof(double)));
        if (dtype == TK_F32)
            launch_model_fit<float>(pool, static_cast<const float*>(y), static_cast<int>(order), dims, core, core_shape,
                                    factors, rank, d, ctx->stream);
        else
            launch_model_fit<double>(pool, static_cast<const double*>(y), static_cast<int>(order), dims, core,
                                     core_shape, factors, rank, d, ctx->stream);
        TK_CUDA(cudaMemcpyAsync(sums, d, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
        require(sums[1] > 0.0, "fit: reference tensor has zero norm");
    });
}

int tk_gaussian_fill(tk_context* ctx, int64_t n, uint64_t offset, uint64_t root, uint64_t stream, double* out) {
    return guarded([&] {
        check_ctx(ctx);
        require(n >= 0, "gaussian_fill: negative length");
        launch_gaussian_fill(out, n, offset, Seed{root, stream}.key(), ctx->stream);
    });
}

int tk_gaussian_fill_block(tk_context* ctx, int64_t order, const int64_t* global_dims, const int64_t* lo,
                           const int64_t* len, uint64_t root, uint64_t stream, double* out) {
    return guarded([&] {
        check_ctx(ctx);
        require(order >= 1 && order <= TK_MAX_ORDER, "tensor order must be in [1, 8]");
        RowMap map;
        int64_t n = 1;
        for (int k = 0; k < order; ++k) {
            require(len[k] >= 0 && lo[k] >= 0 && lo[k] + len[k] <= global_dims[k], "gaussian_fill: block outside the tensor");
            map.lext[k] = std::max<int64_t>(len[k], 1);
            map.lo[k] = lo[k];
            map.gstride[k] = map.rows_total;
            map.rows_total *= global_dims[k];
            n *= len[k];
        }
        map.nd = static_cast<int>(order);
        if (n > 0) launch_gaussian_fill_map(out, n, Seed{root, stream}.key(), map, ctx->stream);
    });
}

int tk_orthonormal_basis(tk_context* ctx, int64_t rows, int64_t cols, const double* z, double* q, int64_t* rank,
                         double* rdiag) {
    return guarded([&] {
        check_ctx(ctx);
        require(rows >= 1, "orthonormal_basis: empty input");
        if (cols == 0) {
            *rank = 0;
            return;
        }
        require(cols <= rows, "orthonormal_basis: wide inputs are not supported on the device path");
        int* rd = static_cast<int*>(ctx->buf("qr_rank", sizeof(int)));
        const int64_t qw = qr_work_elems(rows, static_cast<int>(cols));
        double* qwork = qw ? static_cast<double*>(ctx->buf("qr_work", sizeof(double) * qw)) : nullptr;
        launch_orthonormal_basis(z, rows, static_cast<int>(cols), q, static_cast<int>(cols), nullptr, kF64, rd, rdiag,
                                 ctx->stream, 0, nullptr, qwork);
        TK_CUDA(cudaMemcpyAsync(ctx->rank_host, rd, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
        *rank = *ctx->rank_host;
    });
}

int tk_orthonormal_basis_ex(tk_context* ctx, int64_t rows, int64_t cols, const double* z, double* q, int64_t* rank,
                            double* rdiag, double* margins) {
    return guarded([&] {
        check_ctx(ctx);
        require(rows >= 1, "orthonormal_basis: empty input");
        if (cols == 0) {
            *rank = 0;
            return;
        }
        require(cols <= rows, "orthonormal_basis: wide inputs are not supported on the device path");
        int* rd = static_cast<int*>(ctx->buf("qr_rank", sizeof(int)));
        double* md = static_cast<double*>(ctx->buf("qr_margins", 3 * sizeof(double)));
        const int64_t qw = qr_work_elems(rows, static_cast<int>(cols));
        double* qwork = qw ? static_cast<double*>(ctx->buf("qr_work", sizeof(double) * qw)) : nullptr;
        launch_orthonormal_basis(z, rows, static_cast<int>(cols), q, static_cast<int>(cols), nullptr, kF64, rd, rdiag,
                                 ctx->stream, 0, md, qwork);
        TK_CUDA(cudaMemcpyAsync(ctx->rank_host, rd, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        if (margins) TK_CUDA(cudaMemcpyAsync(margins, md, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
        *rank = *ctx->rank_host;
    });
}

int tk_gram_orthonormalize(tk_context* ctx, int64_t rows, int64_t cols, const double* z, double* u, double* spectrum,
                           int64_t* kept) {
    return guarded([&] {
        check_ctx(ctx);
        require(rows >= 1 && cols >= 1, "gram_orthonormalize: no blocks");
        require(cols <= kMaxRank, "gram_orthonormalize: column count must be <= 64 on the device path");
        int* rd = static_cast<int*>(ctx->buf("qr_rank", sizeof(int)));
        double* gw = static_cast<double*>(ctx->buf("gram_work", sizeof(double) * gram_work_elems(rows, int(cols))));
        launch_gram_orthonormal(z, rows, rows, static_cast<int>(cols), u, static_cast<int>(cols), nullptr, kF64, rd,
                                spectrum, gw, ctx->stream);
        TK_CUDA(cudaMemcpyAsync(ctx->rank_host, rd, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
        *kept = *ctx->rank_host;
        require(*kept >= 1, "gram_orthonormalize: all blocks are zero");
    });
}

int tk_gram_ortho_transform(tk_context* ctx, int64_t n, const double* gram, double* transform, double* spectrum,
                            int64_t* kept) {
    return guarded([&] {
        check_ctx(ctx);
        require(n >= 1 && n <= kMaxRank, "gram_ortho_transform: size must be in [1, 64] on the device path");
        int* rd = static_cast<int*>(ctx->buf("qr_rank", sizeof(int)));
        launch_gram_ortho_transform(gram, static_cast<int>(n), transform, spectrum, rd, ctx->stream);
        TK_CUDA(cudaMemcpyAsync(ctx->rank_host, rd, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
        *kept = *ctx->rank_host;
        require(*kept >= 1, "gram_ortho_transform: zero Gram matrix");
    });
}

int tk_ttm(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* t, int64_t mrows,
           const void* m, int64_t mode, void* out) {
    return guarded([&] {
        check_ctx(ctx);
        require(order >= 1 && order <= TK_MAX_ORDER, "tensor order must be in [1, 8]");
        require(mode >= 0 && mode < order, "mode index out of range");
        require(mrows >= 1 && mrows <= kMaxRank, "ttm: matrix rows must be in [1, 64] on the device path");
        std::vector<int64_t> d(dims, dims + order);
        const int64_t P = prod(std::vector<int64_t>(d.begin(), d.begin() + mode));
        const int64_t Q = prod(std::vector<int64_t>(d.begin() + mode + 1, d.end()));
        // m is mrows x I_mode column-major (dtype); pack M^T k-major
        const int stride = pack_stride(static_cast<int>(mrows));
        double* md = static_cast<double*>(ctx->buf("ttm_m64", sizeof(double) * mrows * d[mode]));
        // M^T (I_mode x mrows, ld I_mode) as double
        std::vector<double> host(mrows * d[mode]);
        const size_t es = dsize(dtype);
        std::vector<unsigned char> raw(es * mrows * d[mode]);
        TK_CUDA(cudaMemcpyAsync(raw.data(), m, raw.size(), cudaMemcpyDeviceToHost, ctx->stream));
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int64_t k = 0; k < d[mode]; ++k)
            for (int64_t r = 0; r < mrows; ++r) {
                const int64_t src = r + k * mrows;
                host[k + r * d[mode]] = dtype == TK_F32 ? reinterpret_cast<float*>(raw.data())[src]
                                                        : reinterpret_cast<double*>(raw.data())[src];
            }
        TK_CUDA(cudaMemcpyAsync(md, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, ctx->stream));
        if (dtype == TK_F32) {
            const float* ft = static_cast<const float*>(t);
            float* fo = static_cast<float*>(out);
            if (ctx->ttm_path == 3 && P > 1 && stream_ttm_supported(ft, fo, P, d[mode], Q, static_cast<int>(mrows))) {
                // the Y-streaming kernel on an M-major contraction (K-major passes write transposed
                // output, exercised through tk_rand_tucker_2i / tk_ttm_all)
                void* bpk = ctx->buf("stream_pack", static_cast<size_t>(stream_pack_bytes(d[mode], static_cast<int>(mrows))));
                launch_pack_stream(md, d[mode], d[mode], static_cast<int>(mrows), bpk, ctx->stream);
                launch_ttm_stream(ft, bpk, fo, P, d[mode], Q, static_cast<int>(mrows), ctx->stream);
                TK_CUDA(cudaStreamSynchronize(ctx->stream));
                return;
            }
            if (ctx->ttm_path >= 2 && tc_ttm_supported(ft, fo, P, d[mode], Q, static_cast<int>(mrows))) {
                void* bpk = ctx->buf("umma_pack", static_cast<size_t>(umma_pack_bytes(d[mode], static_cast<int>(mrows))));
                launch_pack_umma(md, d[mode], d[mode], static_cast<int>(mrows), bpk, ctx->stream);
                launch_ttm_tc(ft, bpk, fo, P, d[mode], Q, static_cast<int>(mrows), ctx->stream);
                TK_CUDA(cudaStreamSynchronize(ctx->stream));
                return;
            }
            float* up = static_cast<float*>(ctx->buf("ttm_up", sizeof(float) * d[mode] * stride));
            launch_pack_factor<float>(md, d[mode], d[mode], static_cast<int>(mrows), up, ctx->stream);
            launch_ttm<float>(ft, up, fo, P, d[mode], Q, static_cast<int>(mrows), ctx->stream);
        } else {
            double* up = static_cast<double*>(ctx->buf("ttm_up", sizeof(double) * d[mode] * stride));
            launch_pack_factor<double>(md, d[mode], d[mode], static_cast<int>(mrows), up, ctx->stream);
            launch_ttm<double>(static_cast<const double*>(t), up, static_cast<double*>(out), P, d[mode], Q,
                               static_cast<int>(mrows), ctx->stream);
        }
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int tk_ttm_all(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* t, const double** ms,
               const int64_t* cols, int64_t skip, void* out) {
    return guarded([&] {
        check_ctx(ctx);
        require(order >= 1 && order <= TK_MAX_ORDER, "tensor order must be in [1, 8]");
        std::vector<int64_t> d(dims, dims + order);
        auto body = [&](auto tag) {
            using T = decltype(tag);
            TuckerRun<T> r{ctx, ctx->stream, order, d, d, std::vector<int64_t>(order, 0), static_cast<const T*>(t)};
            r.cols.resize(order);
            r.Up.resize(order);
            r.U.assign(order, nullptr);
            for (int n = 0; n < order; ++n) {
                r.cols[n] = static_cast<int>(cols[n]);
                if (n == skip) continue;
                require(cols[n] >= 1 && cols[n] <= kMaxRank, "ttm_all: factor columns must be in [1, 64]");
                r.Up[n] = static_cast<T*>(ctx->buf("tall_up" + std::to_string(n), sizeof(T) * d[n] * pack_stride(r.cols[n])));
                launch_pack_factor<T>(ms[n], d[n], d[n], r.cols[n], r.Up[n], ctx->stream);
                r.U[n] = const_cast<double*>(ms[n]);
            }
            std::vector<int64_t> xd;
            std::vector<int> xp;
            const T* x = r.project(static_cast<int>(skip), xd, xp);
            if (xp == r.ident()) {
                TK_CUDA(cudaMemcpyAsync(out, x, sizeof(T) * prod(xd), cudaMemcpyDeviceToDevice, ctx->stream));
            } else {
                std::vector<int64_t> sd(static_cast<size_t>(order));
                for (int k = 0; k < order; ++k) sd[xp[k]] = xd[k];
                launch_permute_cast<T, T>(x, static_cast<T*>(out), static_cast<int>(order), sd.data(), xp.data(),
                                          ctx->stream);
            }
        };
        if (dtype == TK_F32) body(float{});
        else body(double{});
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int tk_unfold_times(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* t, int64_t mode,
                    const double* b, int64_t bcols, double* z) {
    return guarded([&] {
        check_ctx(ctx);
        require(mode >= 0 && mode < order, "mode index out of range");
        std::vector<int64_t> d(dims, dims + order);
        const int64_t B = prod(std::vector<int64_t>(d.begin(), d.begin() + mode));
        const int64_t A = prod(std::vector<int64_t>(d.begin() + mode + 1, d.end()));
        const int64_t W = B * A;
        require(bcols >= 1 && bcols <= kMaxRank, "unfold_times: B columns must be in [1, 64] on the device path");
        auto body = [&](auto tag) {
            using T = decltype(tag);
            TuckerRun<T> r{ctx, ctx->stream, order, d, d, std::vector<int64_t>(order, 0), static_cast<const T*>(t)};
            T* bp = static_cast<T*>(ctx->buf("ut_bp", sizeof(T) * W * pack_stride(static_cast<int>(bcols))));
            launch_pack_factor<T>(b, W, W, static_cast<int>(bcols), bp, ctx->stream);
            r.sketch(static_cast<const T*>(t), d, r.ident(), static_cast<int>(mode), bp, static_cast<int>(bcols), z, d[mode]);
        };
        if (dtype == TK_F32) body(float{});
        else body(double{});
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int tk_dist_multiply(tk_context* ctx, int dtype, int64_t order, const int64_t* dims, const void* y, int64_t mode,
                     int64_t r_tilde, uint64_t seed_root, uint64_t seed_stream, double* z) {
    return guarded([&] {
        check_ctx(ctx);
        require(order >= 1 && order <= TK_MAX_ORDER, "tensor order must be in [1, 8]");
        require(mode >= 0 && mode < order, "dist_multiply: mode out of range");
        require(r_tilde >= 1, "dist_multiply: r_tilde must be positive");
        require(r_tilde <= kMaxRank, "dist_multiply: r_tilde must be <= 64 on this device path");
        std::vector<int64_t> ld(dims, dims + order), gd, lo;
        for (auto v : ld) require(v >= 1, "tensor dimensions must be positive");
        block_of(ctx, ld, gd, lo);
        const int n = static_cast<int>(mode), rt = static_cast<int>(r_tilde);
        // Omega = gaussian_matrix(prod_{k != n} I_k, r~, seed) (random.hpp:85-100) restricted to this
        // block's unfolding columns at their global ids (streamed_block_product, dist.hpp:496-596)
        RowMap map;
        map.rows_total = 1;
        for (int k = 0; k < order; ++k) {
            if (k == n) continue;
            map.lext[map.nd] = ld[k];
            map.lo[map.nd] = lo[k];
            map.gstride[map.nd] = map.rows_total;
            map.rows_total *= gd[k];
            ++map.nd;
        }
        const int64_t width = prod(ld) / ld[n];
        const int64_t In = gd[n];
        auto body = [&](auto tag) {
            using T = decltype(tag);
            cudaStream_t s = ctx->stream;
            TuckerRun<T> r{ctx, s, order, ld, gd, lo, static_cast<const T*>(y)};
            T* op = static_cast<T*>(ctx->buf("dm_omega", sizeof(T) * width * pack_stride(rt)));
            launch_gaussian_packed_map<T>(op, width, rt, Seed{seed_root, seed_stream}.key(), map, s);
            TK_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * In * rt, s));
            r.sketch(static_cast<const T*>(y), ld, r.ident(), n, op, rt, z + lo[n], In);
            // partial products summed over the ranks (the row leaders' reduction, dist.hpp:818-845)
            r.allreduce(z, In * rt);
        };
        if (dtype == TK_F32) body(float{});
        else body(double{});
        TK_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
