// C-ABI implementation of include/qsv.h: contexts, state shards, program
// upload/compilation, reductions and checks.  The pass kernel lives in
// pass_kernel.cu and the qubit swap in swap.cu.
//
// Nothing in this file has a CPU compute fallback: every amplitude operation
// is a CUDA kernel; a missing device fails with QSV_E_NODEV.
#include "qsv_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <complex>
#include <cstring>
#include <string>
#include <thread>
#include <chrono>
#include <vector>

namespace qsv {

namespace {
thread_local std::string t_err;
}

void set_error(const std::string& msg) { t_err = msg; }

} // namespace qsv

using qsv::set_error;

#define QSV_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));              \
            return e_ == cudaErrorMemoryAllocation ? QSV_E_NOMEM : QSV_E_CUDA;          \
        }                                                                               \
    } while (0)

#define QSV_REQUIRE(cond, msg)          \
    do {                                \
        if (!(cond)) {                  \
            set_error(msg);             \
            return QSV_E_ARG;           \
        }                               \
    } while (0)

// ======================================================================= kernels
namespace {

constexpr int kRedThreads = 256;

__device__ __forceinline__ void kahan_add(double& s, double& c, double x) {
    const double y = x - c;
    const double t = s + y;
    c = (t - s) - y;
    s = t;
}

// Per-thread Kahan sums of |a|^2, then a block tree: the 2^n-term norm stays
// well inside the 1e-12 budget (SURVEY §7 hard part 6).
__global__ void norm_partial_kernel(const double2* __restrict__ a, uint64_t n, double* partials) {
    double s = 0.0, c = 0.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double2 v = __ldcs(a + i);
        kahan_add(s, c, fma(v.x, v.x, v.y * v.y));
    }
    __shared__ double sh[32];
    double v = s - c;
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x % 32 == 0)
        sh[threadIdx.x / 32] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0, tc = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w)
            kahan_add(t, tc, sh[w]);
        partials[blockIdx.x] = t;
    }
}

__global__ void sum_partials_kernel(const double* partials, int n, double* out) {
    double s = 0.0, c = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        kahan_add(s, c, partials[i]);
    __shared__ double sh[kRedThreads];
    sh[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0, tc = 0.0;
        for (int i = 0; i < static_cast<int>(blockDim.x); ++i)
            kahan_add(t, tc, sh[i]);
        *out = t;
    }
}

__global__ void max_partials_kernel(const double* partials, int n, double* out) {
    double m = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        m = fmax(m, partials[i]);
    __shared__ double sh[kRedThreads];
    sh[threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < static_cast<int>(blockDim.x); ++i)
            t = fmax(t, sh[i]);
        *out = t;
    }
}

__device__ void block_max_store(double m, double* partials) {
    __shared__ double sh[32];
    for (int o = 16; o > 0; o >>= 1)
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x % 32 == 0)
        sh[threadIdx.x / 32] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w)
            t = fmax(t, sh[w]);
        partials[blockIdx.x] = t;
    }
}

__global__ void diff_partial_kernel(const double2* __restrict__ a, const double2* __restrict__ b,
                                    uint64_t n, double* partials) {
    double m = 0.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double2 x = a[i], y = b[i];
        const double d = hypot(x.x - y.x, x.y - y.y);
        m = (d != d) ? INFINITY : fmax(m, d);  // NaN poisons the check
    }
    block_max_store(m, partials);
}

// Analytic QFT of |x>: psi[y] = exp(2 pi i x y / 2^n) / 2^{n/2}.  The phase is
// reduced exactly in integers (x*y mod 2^n via uint64 wrap-around).
__global__ void qft_check_kernel(const double2* __restrict__ a, uint64_t n_amps, uint64_t rank_base,
                                 int n_total, uint64_t x, double* partials) {
    const uint64_t mask = (n_total >= 64) ? ~0ull : ((1ull << n_total) - 1ull);
    const double scale = exp2(-0.5 * n_total);
    const double inv = exp2(1.0 - n_total);  // sincospi(2 * p / 2^n) = sincospi(p * 2^{1-n})
    double m = 0.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_amps;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t y = rank_base | i;
        const uint64_t p = (x * y) & mask;
        double s, c;
        sincospi(static_cast<double>(p) * inv, &s, &c);
        const double2 v = a[i];
        const double d = hypot(v.x - c * scale, v.y - s * scale);
        m = (d != d) ? INFINITY : fmax(m, d);
    }
    block_max_store(m, partials);
}

__global__ void digest_kernel(const unsigned long long* __restrict__ w, uint64_t nwords,
                              unsigned long long* out) {
    unsigned long long x = 0, s = 0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nwords;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long v = w[i];
        x ^= v * 0x9E3779B97F4A7C15ull + i;
        s += v;
    }
    for (int o = 16; o > 0; o >>= 1) {
        x ^= __shfl_xor_sync(0xffffffffu, x, o);
        s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if (threadIdx.x % 32 == 0) {
        atomicXor(out, x);
        atomicAdd(out + 1, s);
    }
}

__global__ void set_one_kernel(double2* p) { *p = make_double2(1.0, 0.0); }
__global__ void set_amp_kernel(double2* p, double re) { *p = make_double2(re, 0.0); }

int reduce_grid(const qsv_ctx* ctx) { return ctx->sm_count * 8; }

int ensure_partials(qsv_ctx* ctx) {
    const size_t need = static_cast<size_t>(reduce_grid(ctx)) + 8;
    if (ctx->partials_cap >= need)
        return QSV_OK;
    if (ctx->d_partials)
        qsv::dev_free(ctx, ctx->d_partials, 3);
    QSV_CUDA(qsv::dev_alloc(ctx, reinterpret_cast<void**>(&ctx->d_partials), need * sizeof(double), 3));
    ctx->partials_cap = need;
    return QSV_OK;
}

// Finish a max-style reduction of `grid` partials into *out (synchronous).
int finish_max(qsv_ctx* ctx, int grid, double* out) {
    max_partials_kernel<<<1, kRedThreads, 0, ctx->stream>>>(ctx->d_partials, grid,
                                                           ctx->d_partials + ctx->partials_cap - 1);
    QSV_CUDA(cudaGetLastError());
    QSV_CUDA(cudaMemcpyAsync(ctx->h_result, ctx->d_partials + ctx->partials_cap - 1, sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
    QSV_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = ctx->h_result[0];
    return QSV_OK;
}

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

int log2i(int x) {
    int l = 0;
    while ((1 << l) < x)
        ++l;
    return l;
}

} // namespace

// ======================================================================= devices
extern "C" int qsv_device_count(int* n) {
    QSV_REQUIRE(n != nullptr, "qsv_device_count: null output");
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        *n = 0;
        set_error(std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
        return QSV_E_NODEV;
    }
    *n = c;
    return QSV_OK;
}

extern "C" int qsv_comm_unique_id(void* out) {
    QSV_REQUIRE(out != nullptr, "qsv_comm_unique_id: null output");
    static_assert(sizeof(ncclUniqueId) == QSV_NCCL_ID_BYTES, "NCCL id size");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        set_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
        return QSV_E_NCCL;
    }
    std::memcpy(out, &id, sizeof(id));
    return QSV_OK;
}

extern "C" int qsv_ctx_create(int device, int rank, int nranks, const void* comm_id, qsv_ctx** out) {
    QSV_REQUIRE(out != nullptr, "qsv_ctx_create: null output");
    QSV_REQUIRE(is_pow2(nranks), "qsv_ctx_create: nranks must be a power of two (SPEC:341)");
    QSV_REQUIRE(rank >= 0 && rank < nranks, "qsv_ctx_create: rank out of range");
    QSV_REQUIRE(nranks == 1 || comm_id != nullptr, "qsv_ctx_create: nranks > 1 needs a comm id");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        set_error("qsv_ctx_create: no CUDA device (the simulator has no CPU fallback)");
        return QSV_E_NODEV;
    }
    QSV_REQUIRE(device >= 0 && device < ndev, "qsv_ctx_create: device index out of range");
    QSV_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    QSV_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
        set_error("qsv_ctx_create: device is not sm_100-class (built for sm_100a only)");
        return QSV_E_NODEV;
    }
    auto* ctx = new qsv_ctx();
    ctx->device = device;
    ctx->rank = rank;
    ctx->nranks = nranks;
    ctx->sm_count = prop.multiProcessorCount;
    QSV_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    QSV_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    QSV_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    QSV_CUDA(cudaEventCreateWithFlags(&ctx->ev_a, cudaEventDisableTiming));
    QSV_CUDA(cudaEventCreateWithFlags(&ctx->ev_b, cudaEventDisableTiming));
    QSV_CUDA(cudaMallocHost(&ctx->h_result, 4 * sizeof(double)));
    if (nranks > 1) {
        // local allocations first; the init is joined whatever their outcome (the peers
        // are already inside it) and a rank whose allocations failed aborts right after,
        // so the others see an async error instead of waiting forever
        const cudaError_t ea = qsv::dev_alloc(ctx, reinterpret_cast<void**>(&ctx->d_coll),
                                              128 * static_cast<size_t>(nranks) + 64, 3);
        const cudaError_t eb =
            ea == cudaSuccess ? qsv::dev_alloc(ctx, reinterpret_cast<void**>(&ctx->d_sync), 2 * sizeof(double), 3) : ea;
        if (eb == cudaSuccess)
            cudaMemset(ctx->d_sync, 0, 2 * sizeof(double));
        cudaGetLastError();
        ncclUniqueId id;
        std::memcpy(&id, comm_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, id, rank);
        if (r != ncclSuccess || ea != cudaSuccess || eb != cudaSuccess) {
            const std::string why = r != ncclSuccess ? std::string("ncclCommInitRank: ") + ncclGetErrorString(r)
                                                     : std::string("collective scratch cudaMalloc: ") +
                                                           cudaGetErrorString(ea != cudaSuccess ? ea : eb);
            if (r == ncclSuccess)
                ncclCommAbort(ctx->comm);
            if (ctx->d_coll) cudaFree(ctx->d_coll);
            if (ctx->d_sync) cudaFree(ctx->d_sync);
            cudaFreeHost(ctx->h_result);
            set_error("qsv_ctx_create (rank " + std::to_string(rank) + "): " + why);
            delete ctx;
            return r != ncclSuccess ? QSV_E_NCCL : QSV_E_NOMEM;
        }
    }
    *out = ctx;
    return QSV_OK;
}

namespace qsv {

void abort_comm(qsv_ctx* ctx, const std::string& why) {
    {
        std::lock_guard<std::mutex> g(ctx->abort_lock);
        if (ctx->abort_reason.empty())
            ctx->abort_reason = why;  // the first reason wins
    }
    ctx->aborted.store(1);
    if (ctx->comm && ctx->comm_aborted.exchange(1) == 0)
        ncclCommAbort(ctx->comm);  // unblocks every NCCL kernel of this rank
}

int check_aborted(qsv_ctx* ctx, const char* what) {
    if (!ctx->aborted.load())
        return QSV_OK;
    std::string reason;
    {
        std::lock_guard<std::mutex> g(ctx->abort_lock);
        reason = ctx->abort_reason;
    }
    set_error(std::string(what) + " (rank " + std::to_string(ctx->rank) + "): collective aborted: " + reason);
    return QSV_E_NCCL;
}

int wait_stream(qsv_ctx* ctx, cudaStream_t stream, const char* what) {
    if (ctx->nranks < 2 || ctx->comm == nullptr) {
        const cudaError_t e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) {
            set_error(std::string(what) + ": " + cudaGetErrorString(e));
            return QSV_E_CUDA;
        }
        return QSV_OK;
    }
    static const double timeout_s = [] {
        const char* v = std::getenv("QSV_COLL_TIMEOUT_S");
        const double t = v ? std::atof(v) : 900.0;
        return t > 0 ? t : 900.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    int sleep_us = 20;
    for (;;) {
        const cudaError_t q = cudaStreamQuery(stream);
        if (q == cudaSuccess)
            return check_aborted(ctx, what);
        if (q != cudaErrorNotReady) {
            abort_comm(ctx, std::string("CUDA error on rank ") + std::to_string(ctx->rank) + ": " +
                                cudaGetErrorString(q));
            set_error(std::string(what) + " (rank " + std::to_string(ctx->rank) + "): " + cudaGetErrorString(q));
            return QSV_E_CUDA;
        }
        if (ctx->aborted.load()) {
            abort_comm(ctx, "aborted");  // make sure the comm is torn down too (the first reason is kept)
            // the NCCL kernels exit after the abort; let the stream drain
            cudaStreamSynchronize(stream);
            cudaGetLastError();
            return check_aborted(ctx, what);
        }
        if (!ctx->comm_aborted.load()) {
            ncclResult_t ae = ncclSuccess;
            if (ncclCommGetAsyncError(ctx->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
                abort_comm(ctx, std::string("NCCL async error on rank ") + std::to_string(ctx->rank) + ": " +
                                    ncclGetErrorString(ae));
        }
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > timeout_s && !ctx->aborted.load())
            abort_comm(ctx, "rank " + std::to_string(ctx->rank) + " waited " + std::to_string(static_cast<int>(el)) +
                                " s in " + what + " (QSV_COLL_TIMEOUT_S): a peer rank is gone or hung");
        std::this_thread::sleep_for(std::chrono::microseconds(sleep_us));
        sleep_us = std::min(sleep_us * 2, 1000);
    }
}

cudaError_t dev_alloc(qsv_ctx* ctx, void** p, size_t bytes, int kind) {
    const cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess)
        return e;
    ctx->mem_sizes[*p] = bytes;
    const size_t cur = ctx->mem_cur += bytes;
    size_t pk = ctx->mem_peak.load();
    while (cur > pk && !ctx->mem_peak.compare_exchange_weak(pk, cur)) {
    }
    if (ctx->alloc_hook)
        ctx->alloc_hook(ctx->alloc_user, static_cast<int64_t>(bytes), kind);
    return e;
}

void dev_free(qsv_ctx* ctx, void* p, int kind) {
    if (!p)
        return;
    cudaFree(p);
    auto it = ctx->mem_sizes.find(p);
    if (it == ctx->mem_sizes.end())
        return;
    const size_t bytes = it->second;
    ctx->mem_sizes.erase(it);
    ctx->mem_cur -= bytes;
    if (ctx->alloc_hook)
        ctx->alloc_hook(ctx->alloc_user, -static_cast<int64_t>(bytes), kind);
}

int trace_open(qsv_ctx* ctx, int kind, int chunk, int stream_id, cudaStream_t s) {
    if (!ctx->trace_on)
        return -1;
    qsv_ctx::TraceEv ev{kind, ctx->trace_step, chunk, stream_id, nullptr, nullptr};
    if (cudaEventCreate(&ev.a) != cudaSuccess || cudaEventCreate(&ev.b) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    cudaEventRecord(ev.a, s);
    ctx->trace.push_back(ev);
    return static_cast<int>(ctx->trace.size()) - 1;
}

void trace_close(qsv_ctx* ctx, int idx, cudaStream_t s) {
    if (idx >= 0 && idx < static_cast<int>(ctx->trace.size()))
        cudaEventRecord(ctx->trace[idx].b, s);
}

void trace_clear(qsv_ctx* ctx) {
    for (auto& e : ctx->trace) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    ctx->trace.clear();
}

} // namespace qsv

extern "C" int qsv_ctx_set_alloc_hook(qsv_ctx* ctx, qsv_alloc_hook hook, void* user) {
    QSV_REQUIRE(ctx != nullptr, "qsv_ctx_set_alloc_hook: null context");
    ctx->alloc_hook = hook;
    ctx->alloc_user = user;
    return QSV_OK;
}

extern "C" int qsv_ctx_mem(qsv_ctx* ctx, size_t* live_bytes, size_t* peak_bytes) {
    QSV_REQUIRE(ctx != nullptr, "qsv_ctx_mem: null context");
    if (live_bytes)
        *live_bytes = ctx->mem_cur.load();
    if (peak_bytes)
        *peak_bytes = ctx->mem_peak.load();
    return QSV_OK;
}

extern "C" int qsv_ctx_mem_reset_peak(qsv_ctx* ctx) {
    QSV_REQUIRE(ctx != nullptr, "qsv_ctx_mem_reset_peak: null context");
    ctx->mem_peak = ctx->mem_cur.load();
    return QSV_OK;
}

extern "C" int qsv_trace_enable(qsv_ctx* ctx, int on) {
    QSV_REQUIRE(ctx != nullptr, "qsv_trace_enable: null context");
    QSV_CUDA(cudaSetDevice(ctx->device));
    qsv::trace_clear(ctx);
    ctx->trace_on = on != 0;
    if (ctx->trace_on) {
        if (!ctx->trace_base)
            QSV_CUDA(cudaEventCreate(&ctx->trace_base));
        QSV_CUDA(cudaEventRecord(ctx->trace_base, ctx->stream));
    }
    return QSV_OK;
}

extern "C" int qsv_trace_read(qsv_ctx* ctx, qsv_trace_rec* out, int cap, int* n) {
    QSV_REQUIRE(ctx != nullptr && n != nullptr && (out != nullptr || cap == 0), "qsv_trace_read: null argument");
    QSV_CUDA(cudaSetDevice(ctx->device));
    for (cudaStream_t s : {ctx->stream, ctx->comm_stream, ctx->copy_stream})
        if (int rc = qsv::wait_stream(ctx, s, "qsv_trace_read"); rc != QSV_OK)
            return rc;
    *n = static_cast<int>(ctx->trace.size());
    for (int i = 0; i < *n && i < cap; ++i) {
        const auto& e = ctx->trace[i];
        float a = 0, b = 0;
        QSV_CUDA(cudaEventElapsedTime(&a, ctx->trace_base, e.a));
        QSV_CUDA(cudaEventElapsedTime(&b, ctx->trace_base, e.b));
        out[i] = qsv_trace_rec{e.kind, e.step, e.chunk, e.stream, a, b};
    }
    return QSV_OK;
}

extern "C" int qsv_ctx_abort(qsv_ctx* ctx, const char* reason) {
    QSV_REQUIRE(ctx != nullptr, "qsv_ctx_abort: null context");
    qsv::abort_comm(ctx, reason ? reason : "aborted by the caller");
    return QSV_OK;
}

extern "C" int qsv_ctx_aborted(qsv_ctx* ctx, int* out) {
    QSV_REQUIRE(ctx != nullptr && out != nullptr, "qsv_ctx_aborted: null argument");
    *out = ctx->aborted.load();
    return QSV_OK;
}

extern "C" int qsv_ctx_destroy(qsv_ctx* ctx) {
    if (!ctx)
        return QSV_OK;
    cudaSetDevice(ctx->device);
    if (ctx->aborted.load())
        cudaStreamSynchronize(ctx->stream);  // NCCL kernels have exited after the abort
    else
        qsv::wait_stream(ctx, ctx->stream, "qsv_ctx_destroy");
    if (ctx->comm && !ctx->comm_aborted.load())
        ncclCommDestroy(ctx->comm);
    qsv::dev_free(ctx, ctx->d_partials, 3);
    qsv::dev_free(ctx, ctx->d_stage, 1);
    qsv::dev_free(ctx, ctx->d_scratch, 3);
    qsv::dev_free(ctx, ctx->d_sync, 3);
    qsv::dev_free(ctx, ctx->d_coll, 3);
    qsv::trace_clear(ctx);
    if (ctx->trace_base) cudaEventDestroy(ctx->trace_base);
    if (ctx->h_result) cudaFreeHost(ctx->h_result);
    cudaEventDestroy(ctx->ev_a);
    cudaEventDestroy(ctx->ev_b);
    cudaStreamDestroy(ctx->stream);
    cudaStreamDestroy(ctx->comm_stream);
    cudaStreamDestroy(ctx->copy_stream);
    delete ctx;
    return QSV_OK;
}

extern "C" int qsv_ctx_staging_bytes(qsv_ctx* ctx, size_t* out) {
    QSV_REQUIRE(ctx != nullptr && out != nullptr, "qsv_ctx_staging_bytes: null argument");
    *out = ctx->stage_bytes;
    return QSV_OK;
}

extern "C" void* qsv_ctx_stream(qsv_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

extern "C" int qsv_sync(qsv_ctx* ctx) {
    QSV_REQUIRE(ctx != nullptr, "qsv_sync: null context");
    QSV_CUDA(cudaSetDevice(ctx->device));
    return qsv::wait_stream(ctx, ctx->stream, "qsv_sync");
}

extern "C" const char* qsv_last_error(void) { return qsv::t_err.c_str(); }

// ======================================================================= states
extern "C" int qsv_state_alloc(qsv_ctx* ctx, int n_local, qsv_state** out, size_t* bytes) {
    QSV_REQUIRE(ctx != nullptr && out != nullptr, "qsv_state_alloc: null argument");
    QSV_REQUIRE(n_local >= 1 && n_local <= 40, "qsv_state_alloc: n_local must be in [1, 40]");
    QSV_CUDA(cudaSetDevice(ctx->device));
    auto* st = new qsv_state();
    st->ctx = ctx;
    st->n_local = n_local;
    st->size = 1ull << n_local;
    const size_t b = sizeof(double2) * st->size;
    // multi-rank shards carry the fused-swap flags after the amplitudes (peers reach them
    // through the same mapping as the amplitudes)
    const size_t extra = ctx->nranks > 1 ? qsv::kFlagBytes : 0;
    cudaError_t e = qsv::dev_alloc(ctx, reinterpret_cast<void**>(&st->amps), b + extra, 0);
    if (e != cudaSuccess) {
        delete st;
        set_error("qsv_state_alloc: cudaMalloc of " + std::to_string(b) + " bytes failed: " +
                  cudaGetErrorString(e));
        return QSV_E_NOMEM;
    }
    if (extra && (e = cudaMemset(st->amps + st->size, 0, extra)) != cudaSuccess) {
        qsv::dev_free(ctx, st->amps, 0);
        delete st;
        set_error(std::string("qsv_state_alloc: flag init: ") + cudaGetErrorString(e));
        return QSV_E_CUDA;
    }
    if (bytes)
        *bytes = b;
    *out = st;
    return QSV_OK;
}

extern "C" int qsv_state_free(qsv_state* st) {
    if (!st)
        return QSV_OK;
    cudaSetDevice(st->ctx->device);
    cudaStreamSynchronize(st->ctx->stream);
    cudaStreamSynchronize(st->ctx->comm_stream);
    for (size_t q = 0; q < st->peer_amps.size(); ++q)
        if (st->peer_ipc[q] && st->peer_amps[q])
            cudaIpcCloseMemHandle(st->peer_amps[q]);
    qsv::dev_free(st->ctx, st->amps, 0);
    delete st;
    return QSV_OK;
}

extern "C" int qsv_state_set_basis(qsv_state* st, uint64_t global_index) {
    QSV_REQUIRE(st != nullptr, "qsv_state_set_basis: null state");
    qsv_ctx* ctx = st->ctx;
    QSV_CUDA(cudaSetDevice(ctx->device));
    QSV_CUDA(cudaMemsetAsync(st->amps, 0, sizeof(double2) * st->size, ctx->stream));
    const uint64_t owner = global_index >> st->n_local;
    QSV_REQUIRE(owner < static_cast<uint64_t>(ctx->nranks), "qsv_state_set_basis: index >= 2^n");
    if (owner == static_cast<uint64_t>(ctx->rank)) {
        set_one_kernel<<<1, 1, 0, ctx->stream>>>(st->amps + (global_index & (st->size - 1)));
        QSV_CUDA(cudaGetLastError());
    }
    st->is_basis = true;
    st->basis = global_index;
    return QSV_OK;
}

extern "C" int qsv_state_upload(qsv_state* st, const double* host, uint64_t offset, uint64_t count) {
    QSV_REQUIRE(st != nullptr && (host != nullptr || count == 0), "qsv_state_upload: null argument");
    st->is_basis = false;
    QSV_REQUIRE(offset <= st->size && count <= st->size - offset, "qsv_state_upload: range outside shard");
    QSV_CUDA(cudaSetDevice(st->ctx->device));
    QSV_CUDA(cudaMemcpyAsync(st->amps + offset, host, count * sizeof(double2), cudaMemcpyHostToDevice,
                             st->ctx->stream));
    return QSV_OK;
}

extern "C" int qsv_state_download(qsv_state* st, double* host, uint64_t offset, uint64_t count) {
    QSV_REQUIRE(st != nullptr && (host != nullptr || count == 0), "qsv_state_download: null argument");
    QSV_REQUIRE(offset <= st->size && count <= st->size - offset, "qsv_state_download: range outside shard");
    QSV_CUDA(cudaSetDevice(st->ctx->device));
    QSV_CUDA(cudaMemcpyAsync(host, st->amps + offset, count * sizeof(double2), cudaMemcpyDeviceToHost,
                             st->ctx->stream));
    QSV_CUDA(cudaStreamSynchronize(st->ctx->stream));
    return QSV_OK;
}

extern "C" int qsv_state_download_async(qsv_state* st, double* host, uint64_t offset, uint64_t count) {
    QSV_REQUIRE(st != nullptr && (host != nullptr || count == 0), "qsv_state_download_async: null argument");
    QSV_REQUIRE(offset <= st->size && count <= st->size - offset, "qsv_state_download_async: range outside shard");
    QSV_CUDA(cudaSetDevice(st->ctx->device));
    QSV_CUDA(cudaMemcpyAsync(host, st->amps + offset, count * sizeof(double2), cudaMemcpyDeviceToHost,
                             st->ctx->stream));
    return QSV_OK;
}

extern "C" int qsv_event_create(void** ev) {
    QSV_REQUIRE(ev != nullptr, "qsv_event_create: null output");
    cudaEvent_t e;
    QSV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    *ev = e;
    return QSV_OK;
}

extern "C" int qsv_event_destroy(void* ev) {
    if (ev)
        QSV_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(ev)));
    return QSV_OK;
}

extern "C" int qsv_event_record(void* ev, void* stream) {
    QSV_REQUIRE(ev != nullptr, "qsv_event_record: null event");
    QSV_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), static_cast<cudaStream_t>(stream)));
    return QSV_OK;
}

extern "C" int qsv_stream_wait_event(void* stream, void* ev) {
    QSV_REQUIRE(ev != nullptr, "qsv_stream_wait_event: null event");
    QSV_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(ev), 0));
    return QSV_OK;
}

extern "C" int qsv_state_device_ptr(qsv_state* st, void** ptr) {
    QSV_REQUIRE(st != nullptr && ptr != nullptr, "qsv_state_device_ptr: null argument");
    *ptr = st->amps;
    st->is_basis = false;  // the caller may write through the pointer
    return QSV_OK;
}

extern "C" int qsv_host_alloc(size_t bytes, void** ptr) {
    QSV_REQUIRE(ptr != nullptr, "qsv_host_alloc: null output");
    QSV_CUDA(cudaMallocHost(ptr, bytes));
    return QSV_OK;
}

extern "C" int qsv_host_free(void* ptr) {
    if (ptr)
        QSV_CUDA(cudaFreeHost(ptr));
    return QSV_OK;
}

// ======================================================================= programs
namespace {

struct BlobBuilder {
    std::vector<unsigned char> bytes;
    uint32_t append(const void* p, size_t n) {
        const size_t at = (bytes.size() + 15) & ~size_t{15};
        bytes.resize(at + n);
        std::memcpy(bytes.data() + at, p, n);
        return static_cast<uint32_t>(at);
    }
};

// XOR-linear enumeration of a 2^K tile for the pass relabel (relabel_op): column c
// is the source index contributed by bit c of x = thread | iteration << log2(NT); the
// destination column is its image under the bit permutation rel.  Columns 0..2 (the
// lane bits of a quarter-warp) are picked so that both the source and the destination
// low-3 bits (the 16-B bank slot) are linearly independent, i.e. conflict-free.
void relabel_columns(int K, const int32_t* rel, uint16_t* scol, uint16_t* dcol) {
    auto image = [&](uint32_t v) {
        uint32_t d = 0;
        for (int b = 0; b < K; ++b)
            if (v >> b & 1u)
                d |= 1u << rel[b];
        return d;
    };
    auto rank3 = [](uint32_t a, uint32_t b, uint32_t c) {  // GF(2) rank of the low-3-bit projections
        a &= 7u;
        b &= 7u;
        c &= 7u;
        return a && b && c && a != b && c != a && c != b && (a ^ b) != c;
    };
    std::vector<uint32_t> cols;
    if (K >= 3) {
        std::vector<uint32_t> cand;
        for (int a = 0; a < K; ++a)
            cand.push_back(1u << a);
        for (int a = 0; a < K; ++a)
            for (int b = a + 1; b < K; ++b)
                cand.push_back((1u << a) | (1u << b));
        bool found = false;
        for (size_t i = 0; i < cand.size() && !found; ++i)
            for (size_t j = i + 1; j < cand.size() && !found; ++j)
                for (size_t k = j + 1; k < cand.size() && !found; ++k)
                    if (rank3(cand[i], cand[j], cand[k]) &&
                        rank3(image(cand[i]), image(cand[j]), image(cand[k]))) {
                        cols = {cand[i], cand[j], cand[k]};
                        found = true;
                    }
    }
    // complete to a basis of GF(2)^K with unit vectors (pivot on the highest set bit)
    uint32_t piv[16] = {};
    auto insert = [&](uint32_t v) {
        for (int b = 15; b >= 0; --b) {
            if (!(v >> b & 1u))
                continue;
            if (!piv[b]) {
                piv[b] = v;
                return true;
            }
            v ^= piv[b];
        }
        return false;
    };
    for (uint32_t c : cols)
        insert(c);
    for (int b = 0; b < K && static_cast<int>(cols.size()) < K; ++b)
        if (insert(1u << b))
            cols.push_back(1u << b);
    for (int c = 0; c < 16; ++c) {
        scol[c] = c < K ? static_cast<uint16_t>(cols[c]) : 0;
        dcol[c] = c < K ? static_cast<uint16_t>(image(cols[c])) : 0;
    }
}

// Minimum DFMA/DMUL count per amplitude of a 4-qubit register block's primitive list
// for it to run as a dense DMMA16 op (QSV_DMMA_MIN_PIPE; 0, the default, keeps every block
// on the DFMA primitives).  Measured on random-30: thresholds 32 / 40 / 56 give 420 / 303 /
// 281 ms against 280 ms without, HEA-30 120 vs 115 ms: the dense form costs 128 flop per
// amplitude where the primitive lists of these circuits cost 50-100, and the DMMA ops reach
// ~21 TF (0.57 of the measured 37.1 TF) at 12 warps per SM (profiles/r02_kernel_ab.md).
int dmma_min_pipe_ops() {
    static const int v = [] {
        const char* e = std::getenv("QSV_DMMA_MIN_PIPE");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

int compile_pass(const qsv_step_desc& d, int n_total, int n_local, int rank,
                 const qsv_op_desc* ops, int nops, const qsv_prim_desc* prims, int nprims,
                 const double* pool, size_t pool_len, qsv::Step& step,
                 std::vector<unsigned char>& blob_out) {
    using qsv::TileOp;
    const int K = d.tile_k;
    QSV_REQUIRE(K >= 1 && K <= QSV_MAX_TILE_K && K <= n_local,
                "pass: tile_k must be in [1, min(12, n_local)] (12: specialised kernels only)");
    const int nhi = K > 5 ? 1 << (K - 5) : 1;  // entries of the high-tile-bit tables
    QSV_REQUIRE(d.nhigh >= 0 && d.nhigh <= QSV_MAX_HIGH && d.nhigh <= K, "pass: bad nhigh");
    const int L = K - d.nhigh;
    int tpos_of[64];
    for (int q = 0; q < 64; ++q)
        tpos_of[q] = (q < L) ? q : -1;
    for (int i = 0; i < d.nhigh; ++i) {
        const int h = d.high[i];
        QSV_REQUIRE(h >= L && h < n_local, "pass: high tile qubit must be local and above the low run");
        QSV_REQUIRE(i == 0 || h > d.high[i - 1], "pass: high tile qubits must be ascending");
        tpos_of[h] = L + i;
    }
    QSV_REQUIRE(d.op_begin >= 0 && d.op_count >= 0 && d.op_begin + d.op_count <= nops,
                "pass: op range outside the op array");
    step.geom.K = K;
    step.geom.L = L;
    step.geom.nhigh = d.nhigh;
    for (int i = 0; i < d.nhigh; ++i)
        step.geom.high[i] = d.high[i];
    step.geom.kmax = 0;
    step.nops = d.op_count;

    const uint64_t full_mask = (n_total >= 64) ? ~0ull : ((1ull << n_total) - 1ull);
    const uint64_t rank_bits = static_cast<uint64_t>(rank) << n_local;
    std::vector<TileOp> tops(d.op_count);
    QSV_REQUIRE(d.has_relabel == 0 || d.has_relabel == 1, "pass: has_relabel must be 0 or 1");
    if (d.has_relabel) {
        uint32_t seen = 0;
        for (int i = 0; i < K; ++i) {
            const int r = d.relabel[i];
            QSV_REQUIRE(r >= 0 && r < K && !(seen >> r & 1u), "pass: relabel must be a permutation of the tile bits");
            seen |= 1u << r;
        }
    }
    struct Payload { int op; std::vector<uint32_t> off; std::vector<double> data; std::vector<uint8_t> ptab;
                     std::vector<qsv::DevPrim> dprims; std::vector<std::vector<double>> pdata; std::vector<qsv::ExtFactor> ext; };
    std::vector<Payload> payloads;
    double flops = 0.0;
    const double amps = std::ldexp(1.0, n_local);

    for (int oi = 0; oi < d.op_count; ++oi) {
        const qsv_op_desc& od = ops[d.op_begin + oi];
        TileOp t{};
        t.kind = od.kind;
        t.k = od.k;
        QSV_REQUIRE((od.ctrl_mask & ~full_mask) == 0, "op: control bit >= n_total");
        uint64_t qmask = 0;
        for (int i = 0; i < od.k; ++i) {
            const int q = od.qubits[i];
            QSV_REQUIRE(q >= 0 && q < n_total, "op: qubit out of range");
            QSV_REQUIRE(!(qmask >> q & 1), "op: duplicate qubit");
            qmask |= 1ull << q;
        }
        QSV_REQUIRE((qmask & od.ctrl_mask) == 0, "op: control overlaps a target (SPEC:51)");
        // controls: tile-local ones restrict enumeration, the rest are CTA-uniform tests
        std::vector<int> fix;
        for (int c = 0; c < n_total; ++c) {
            if (!(od.ctrl_mask >> c & 1))
                continue;
            if (c < n_local && tpos_of[c] >= 0) {
                t.tctrl |= 1u << tpos_of[c];
                fix.push_back(tpos_of[c]);
            } else {
                t.xctrl |= 1ull << c;
            }
        }
        const int nctrl = __builtin_popcountll(od.ctrl_mask);
        // fraction of this rank's amplitudes the op touches
        const bool rank_ok = ((rank_bits & t.xctrl) >> n_local) == ((t.xctrl & ~((1ull << n_local) - 1)) >> n_local);
        const int local_ctrls = __builtin_popcountll(od.ctrl_mask & ((1ull << n_local) - 1));
        const double frac = rank_ok ? std::ldexp(1.0, -local_ctrls) : 0.0;
        (void)nctrl;
        Payload pl;
        pl.op = oi;
        if (od.kind == QSV_OP_DENSE || od.kind == QSV_OP_XPERM) {
            QSV_REQUIRE(od.k >= 1 && od.k <= (od.kind == QSV_OP_XPERM ? 1 : QSV_MAX_DENSE_K),
                        "op: dense arity must be in [1, 5] (XPERM: 1)");
            for (int i = 0; i < od.k; ++i) {
                const int q = od.qubits[i];
                QSV_REQUIRE(q < n_local && tpos_of[q] >= 0,
                            "op: dense/XPERM target " + std::to_string(q) + " is not in the pass tile");
                t.tpos[i] = static_cast<int8_t>(tpos_of[q]);
                fix.push_back(tpos_of[q]);
            }
            if (od.kind == QSV_OP_DENSE) {
                const int D = 1 << od.k;
                QSV_REQUIRE(od.mat_off >= 0 && static_cast<size_t>(od.mat_off) + D * D <= pool_len,
                            "op: matrix outside the pool");
                pl.off.resize(D);
                for (int j = 0; j < D; ++j) {
                    uint32_t o = 0;
                    for (int i = 0; i < od.k; ++i)
                        if (j >> i & 1)
                            o |= 1u << t.tpos[i];
                    pl.off[j] = o;
                }
                pl.data.assign(pool + 2 * od.mat_off, pool + 2 * (od.mat_off + D * D));
                step.geom.kmax = std::max(step.geom.kmax, od.k);
                flops += 8.0 * D * amps * frac;
            }
        } else if (od.kind == QSV_OP_RBLOCK) {
            double prim_flops = 0.0;
            int pipe_ops = 0;  // DFMA/DMUL per amplitude of the primitive list
            QSV_REQUIRE(od.k == 3 || od.k == 4, "op: RBLOCK needs 3 or 4 block qubits");
            QSV_REQUIRE(od.prim_begin >= 0 && od.nprim >= 1 && od.prim_begin + od.nprim <= nprims,
                        "op: RBLOCK primitive range outside the primitive array");
            QSV_REQUIRE(K >= od.k, "op: RBLOCK wider than the tile");
            const int KB = od.k;
            for (int i = 0; i < KB; ++i) {
                const int q = od.qubits[i];
                QSV_REQUIRE(q < n_local && tpos_of[q] >= 0,
                            "op: RBLOCK qubit " + std::to_string(q) + " is not in the pass tile");
                t.tpos[i] = static_cast<int8_t>(tpos_of[q]);
                fix.push_back(tpos_of[q]);
            }
            for (int pi = 0; pi < od.nprim; ++pi) {
                const qsv_prim_desc& pd = prims[od.prim_begin + pi];
                qsv::DevPrim dp{};
                dp.kind = static_cast<uint8_t>(pd.kind);
                dp.a = static_cast<uint8_t>(pd.a);
                dp.b = static_cast<uint8_t>(pd.b);
                int ne = 0;
                double fl = 0;
                switch (pd.kind) {
                case QSV_PRIM_U1:
                case QSV_PRIM_U1R:
                case QSV_PRIM_U1I:
                    QSV_REQUIRE(pd.a >= 0 && pd.a < KB, "prim: U1 qubit index outside the block");
                    dp.b = 0;
                    ne = 4;
                    fl = pd.kind == QSV_PRIM_U1 ? 16 : 8;
                    if (pd.kind != QSV_PRIM_U1) {
                        QSV_REQUIRE(pd.mat_off >= 0 && static_cast<size_t>(pd.mat_off) + 4 <= pool_len,
                                    "prim: matrix outside the pool");
                        const double* m = pool + 2 * pd.mat_off;
                        const bool ok = pd.kind == QSV_PRIM_U1R
                                            ? (m[1] == 0 && m[3] == 0 && m[5] == 0 && m[7] == 0)
                                            : (m[1] == 0 && m[2] == 0 && m[4] == 0 && m[7] == 0);
                        QSV_REQUIRE(ok, "prim: U1R needs a real matrix, U1I real diagonal / imaginary off-diagonal");
                    }
                    break;
                case QSV_PRIM_U2:
                    QSV_REQUIRE(pd.a >= 0 && pd.b > pd.a && pd.b < KB, "prim: U2 needs 0 <= a < b < k");
                    ne = 16;
                    fl = 32;
                    break;
                case QSV_PRIM_CX:
                    QSV_REQUIRE(pd.a >= 0 && pd.a < KB && pd.b >= 0 && pd.b < KB && pd.a != pd.b,
                                "prim: CX needs distinct block qubits");
                    break;
                case QSV_PRIM_DIAG16:
                    dp.a = 3;  // routes to the default (diagonal) case of the switch
                    dp.b = 3;
                    ne = 1 << KB;
                    fl = 6;
                    break;
                default:
                    QSV_REQUIRE(false, "prim: unknown RBLOCK primitive kind");
                }
                std::vector<double> d;
                if (ne) {
                    QSV_REQUIRE(pd.mat_off >= 0 && static_cast<size_t>(pd.mat_off) + ne <= pool_len,
                                "prim: matrix outside the pool");
                    const double* m = pool + 2 * pd.mat_off;
                    if (pd.kind != QSV_PRIM_DIAG16) {
                        // rotation variants: M_s[i][j] = M[i ^ s][j ^ s]
                        const int dim = pd.kind == QSV_PRIM_U2 ? 4 : 2;
                        for (int sv = 0; sv < dim; ++sv)
                            for (int i = 0; i < dim; ++i)
                                for (int j = 0; j < dim; ++j) {
                                    d.push_back(m[2 * ((i ^ sv) * dim + (j ^ sv))]);
                                    d.push_back(m[2 * ((i ^ sv) * dim + (j ^ sv)) + 1]);
                                }
                    } else {
                        d.assign(m, m + 2 * ne);
                    }
                }
                pl.pdata.push_back(std::move(d));
                pl.dprims.push_back(dp);
                flops += fl * amps * frac;
                prim_flops += fl * amps * frac;
                pipe_ops += pd.kind == QSV_PRIM_U1 ? 8 : pd.kind == QSV_PRIM_U2 ? 16 : pd.kind == QSV_PRIM_CX ? 0 : 4;
            }
            t.nprim = od.nprim;
            step.geom.kmax = std::max(step.geom.kmax, KB == 4 ? 4 : 1);
            // Heavy 4-qubit blocks go to the FP64 tensor cores: the block's dense 16x16 unitary
            // (the primitive product, formed here in double) costs 64 DMMA MACs per amplitude
            // in ~1/4 instruction, against `pipe_ops` DFMA/DMUL per amplitude issued one by one.
            if (KB == 4 && dmma_min_pipe_ops() > 0 && pipe_ops >= dmma_min_pipe_ops()) {
                std::vector<double> mat(2 * 256, 0.0);  // M[r][c], row-major complex
                for (int c = 0; c < 16; ++c) {
                    std::complex<double> v[16];
                    v[c] = 1.0;
                    for (int pi = 0; pi < od.nprim; ++pi) {
                        const qsv_prim_desc& pd = prims[od.prim_begin + pi];
                        const std::complex<double>* m = reinterpret_cast<const std::complex<double>*>(pool) + pd.mat_off;
                        if (pd.kind == QSV_PRIM_CX) {
                            for (int j = 0; j < 16; ++j)
                                if ((j >> pd.a & 1) && !(j >> pd.b & 1))
                                    std::swap(v[j], v[j | (1 << pd.b)]);
                        } else if (pd.kind == QSV_PRIM_DIAG16) {
                            for (int j = 0; j < 16; ++j)
                                v[j] *= m[j];
                        } else if (pd.kind == QSV_PRIM_U2) {
                            const int A = 1 << pd.a, B = 1 << pd.b;
                            for (int j = 0; j < 16; ++j) {
                                if (j & (A | B))
                                    continue;
                                const std::complex<double> x[4] = {v[j], v[j | A], v[j | B], v[j | A | B]};
                                std::complex<double> y[4];
                                for (int r = 0; r < 4; ++r)
                                    y[r] = m[4 * r] * x[0] + m[4 * r + 1] * x[1] + m[4 * r + 2] * x[2] + m[4 * r + 3] * x[3];
                                v[j] = y[0];
                                v[j | A] = y[1];
                                v[j | B] = y[2];
                                v[j | A | B] = y[3];
                            }
                        } else {  // U1 / U1R / U1I: the full 2x2 as given
                            const int A = 1 << pd.a;
                            for (int j = 0; j < 16; ++j) {
                                if (j & A)
                                    continue;
                                const std::complex<double> x0 = v[j], x1 = v[j | A];
                                v[j] = m[0] * x0 + m[1] * x1;
                                v[j | A] = m[2] * x0 + m[3] * x1;
                            }
                        }
                    }
                    for (int r = 0; r < 16; ++r) {
                        mat[2 * (16 * r + c)] = v[r].real();
                        mat[2 * (16 * r + c) + 1] = v[r].imag();
                    }
                }
                t.kind = QSV_OP_DMMA16;
                t.nprim = 0;
                pl.dprims.clear();
                pl.pdata.clear();
                pl.data = std::move(mat);
                flops += 128.0 * amps * frac - prim_flops;
            }
        } else if (od.kind == QSV_OP_PHASEPROD) {
            QSV_REQUIRE(od.k == 0, "op: PHASEPROD takes its qubits as FACTOR primitives (k = 0)");
            QSV_REQUIRE(od.prim_begin >= 0 && od.nprim >= 0 && od.prim_begin + od.nprim <= nprims,
                        "op: PHASEPROD primitive range outside the primitive array");
            QSV_REQUIRE(od.mat_off >= 0 && static_cast<size_t>(od.mat_off) + 1 <= pool_len,
                        "op: PHASEPROD constant outside the pool");
            // table: [c][A: 32 low tile bits][B: 2^(K-5) high tile bits]
            std::vector<double> tab(2 * (33 + nhi), 0.0);
            for (int e = 0; e < 33 + nhi; ++e)
                tab[2 * e] = 1.0;
            tab[0] = pool[2 * od.mat_off];
            tab[1] = pool[2 * od.mat_off + 1];
            auto mul_into = [&](int e, double fr, double fi) {
                const double r = tab[2 * e], im = tab[2 * e + 1];
                tab[2 * e] = r * fr - im * fi;
                tab[2 * e + 1] = r * fi + im * fr;
            };
            for (int pi = 0; pi < od.nprim; ++pi) {
                const qsv_prim_desc& pd = prims[od.prim_begin + pi];
                QSV_REQUIRE(pd.kind == QSV_PRIM_FACTOR, "prim: PHASEPROD accepts FACTOR primitives only");
                QSV_REQUIRE(pd.a >= 0 && pd.a < n_total, "prim: FACTOR qubit out of range");
                QSV_REQUIRE(pd.mat_off >= 0 && static_cast<size_t>(pd.mat_off) + 1 <= pool_len,
                            "prim: FACTOR value outside the pool");
                const double fr = pool[2 * pd.mat_off], fi = pool[2 * pd.mat_off + 1];
                const int q = pd.a;
                const int tp = (q < n_local) ? tpos_of[q] : -1;
                if (tp >= 0 && tp < 5) {
                    for (int e = 0; e < 32; ++e)
                        if (e >> tp & 1)
                            mul_into(1 + e, fr, fi);
                } else if (tp >= 5) {
                    for (int e = 0; e < nhi; ++e)
                        if (e >> (tp - 5) & 1)
                            mul_into(33 + e, fr, fi);
                } else {
                    qsv::ExtFactor xf{};
                    xf.re = fr;
                    xf.im = fi;
                    xf.bit = q;
                    pl.ext.push_back(xf);
                }
            }
            pl.data = std::move(tab);
            t.nprim = static_cast<int32_t>(pl.ext.size());
            flops += 18.0 * amps * frac;
        } else if (od.kind == QSV_OP_PARPHASE) {
            QSV_REQUIRE(od.k == 0, "op: PARPHASE takes its qubits in qmask (k = 0)");
            QSV_REQUIRE((od.qmask & ~full_mask) == 0, "op: PARPHASE mask bit >= n_total");
            QSV_REQUIRE((od.qmask & od.ctrl_mask) == 0, "op: PARPHASE mask overlaps a control");
            QSV_REQUIRE(od.mat_off >= 0 && static_cast<size_t>(od.mat_off) + 2 <= pool_len,
                        "op: PARPHASE phases outside the pool");
            for (int q = 0; q < n_total; ++q) {
                if (!(od.qmask >> q & 1))
                    continue;
                if (q < n_local && tpos_of[q] >= 0)
                    t.tmask |= 1u << tpos_of[q];
                else
                    t.xmask |= 1ull << q;
            }
            pl.data.assign(pool + 2 * od.mat_off, pool + 2 * (od.mat_off + 2));
            flops += 6.0 * amps * frac;
        } else if (od.kind == QSV_OP_DIAG) {
            QSV_REQUIRE(od.k >= 0 && od.k <= QSV_MAX_DIAG_K, "op: diagonal arity must be in [0, 8]");
            const int D = 1 << od.k;
            QSV_REQUIRE(od.mat_off >= 0 && static_cast<size_t>(od.mat_off) + D <= pool_len,
                        "op: diagonal outside the pool");
            // in-tile qubits first (ascending tile position), then out-of-tile ones
            std::vector<int> order;  // new bit -> original bit
            std::vector<std::pair<int, int>> in;
            std::vector<int> outb;
            for (int i = 0; i < od.k; ++i) {
                const int q = od.qubits[i];
                if (q < n_local && tpos_of[q] >= 0)
                    in.push_back({tpos_of[q], i});
                else
                    outb.push_back(i);
            }
            std::sort(in.begin(), in.end());
            t.nin = static_cast<int32_t>(in.size());
            for (auto& pr : in) {
                t.tmask |= 1u << pr.first;
                order.push_back(pr.second);
            }
            for (size_t j = 0; j < outb.size(); ++j) {
                t.xbit[j] = static_cast<int8_t>(od.qubits[outb[j]]);
                order.push_back(outb[j]);
            }
            pl.data.resize(2 * D);
            for (int e = 0; e < D; ++e) {
                int src = 0;
                for (int nb = 0; nb < od.k; ++nb)
                    if (e >> nb & 1)
                        src |= 1 << order[nb];
                pl.data[2 * e] = pool[2 * (od.mat_off + src)];
                pl.data[2 * e + 1] = pool[2 * (od.mat_off + src) + 1];
            }
            flops += 6.0 * amps * frac;
        } else {
            QSV_REQUIRE(false, "op: unknown kind " + std::to_string(od.kind));
        }
        std::sort(fix.begin(), fix.end());
        QSV_REQUIRE(fix.size() <= sizeof(t.fixpos), "op: too many fixed tile bits");
        if (t.kind == QSV_OP_RBLOCK) {
            // Lanes i = 0..7 of a quarter-warp own groups whose low free bits are
            // the lowest free tile positions.  The first `a` of them lie in tile
            // bits 0..2 (the SMEM bank bits of 16-B amplitudes); lanes that differ
            // only in the next bits would hit the same banks, so their member
            // order is rotated by XOR over the block slots sitting in bits 0..2.
            std::vector<int> lowslots;
            for (int sl = 0; sl < od.k; ++sl)
                if (t.tpos[sl] < 3)
                    lowslots.push_back(sl);
            int a = 0;
            for (int pbit = 0; pbit < 3 && pbit < K; ++pbit)
                if (std::find(fix.begin(), fix.end(), pbit) == fix.end())
                    ++a;
            for (int i = 0; i < 8; ++i) {
                const int hi = i >> a;
                uint32_t r = 0;
                for (size_t j = 0; j < lowslots.size(); ++j)
                    if (hi >> j & 1)
                        r |= 1u << lowslots[j];
                t.rot_tab |= r << (4 * i);
            }
        }
        t.nfix = static_cast<int32_t>(fix.size());
        for (size_t i = 0; i < fix.size(); ++i) {
            t.fixpos[i] = static_cast<int8_t>(fix[i]);
            t.fmask |= 1u << fix[i];
        }
        if (od.kind == QSV_OP_DIAG && t.nin > 0) {
            // pext(idx, tmask) = ptab_lo[idx & 31] | ptab_hi[idx >> 5]
            pl.ptab.resize(32 + nhi);
            for (int j = 0; j < 32 + nhi; ++j) {
                const uint32_t idx = j < 32 ? static_cast<uint32_t>(j) : static_cast<uint32_t>(j - 32) << 5;
                uint32_t e = 0, m = t.tmask;
                for (int bit = 0; m; ++bit) {
                    const int pbit = __builtin_ctz(m);
                    e |= ((idx >> pbit) & 1u) << bit;
                    m &= m - 1;
                }
                pl.ptab[j] = static_cast<uint8_t>(e);
            }
        }
        tops[oi] = t;
        if (!pl.data.empty() || !pl.off.empty() || !pl.ptab.empty() || !pl.dprims.empty() || !pl.ext.empty())
            payloads.push_back(std::move(pl));
    }
    std::vector<uint16_t> relabel_tab;
    if (d.has_relabel) {
        TileOp t{};
        t.kind = QSV_OP_RELABEL;
        t.k = K;
        // the permutation itself, for the JIT (a register block may store through it)
        for (int i = 0; i < K; ++i) {
            if (i < 8)
                t.tpos[i] = static_cast<int8_t>(d.relabel[i]);
            else
                t.xbit[i - 8] = static_cast<int8_t>(d.relabel[i]);
        }
        relabel_tab.assign(32, 0);
        relabel_columns(K, d.relabel, relabel_tab.data(), relabel_tab.data() + 16);
        tops.push_back(t);
        step.nops = d.op_count + 1;
    }
    BlobBuilder bb;
    bb.append(tops.data(), tops.size() * sizeof(TileOp));
    if (d.has_relabel)
        tops.back().mat_byte = bb.append(relabel_tab.data(), relabel_tab.size() * sizeof(uint16_t));
    for (auto& pl : payloads) {
        TileOp& t = tops[pl.op];
        if (!pl.off.empty())
            t.off_byte = bb.append(pl.off.data(), pl.off.size() * sizeof(uint32_t));
        if (!pl.data.empty())
            t.mat_byte = bb.append(pl.data.data(), pl.data.size() * sizeof(double));
        if (!pl.ptab.empty())
            t.ptab_byte = bb.append(pl.ptab.data(), pl.ptab.size());
        if (!pl.dprims.empty()) {
            for (size_t i = 0; i < pl.dprims.size(); ++i)
                if (!pl.pdata[i].empty())
                    pl.dprims[i].data_byte = bb.append(pl.pdata[i].data(), pl.pdata[i].size() * sizeof(double));
            t.prim_byte = bb.append(pl.dprims.data(), pl.dprims.size() * sizeof(qsv::DevPrim));
        }
        if (!pl.ext.empty())
            t.prim_byte = bb.append(pl.ext.data(), pl.ext.size() * sizeof(qsv::ExtFactor));
    }
    std::memcpy(bb.bytes.data(), tops.data(), tops.size() * sizeof(TileOp));
    bb.bytes.resize((bb.bytes.size() + 15) & ~size_t{15});
    QSV_REQUIRE(bb.bytes.size() <= qsv::kMaxBlobBytes,
                "pass: ops + matrices exceed the per-pass shared-memory budget (" +
                    std::to_string(bb.bytes.size()) + " > " + std::to_string(qsv::kMaxBlobBytes) + " B)");
    step.blob_bytes = static_cast<uint32_t>(bb.bytes.size());
    step.hbm_bytes = 32.0 * amps;
    step.flops = flops;
    blob_out = std::move(bb.bytes);
    return QSV_OK;
}

} // namespace

extern "C" int qsv_program_create(qsv_ctx* ctx, int n_total, int n_local, const qsv_step_desc* steps,
                                  int nsteps, const qsv_op_desc* ops, int nops, const qsv_prim_desc* prims,
                                  int nprims, const double* pool, size_t pool_len, qsv_program** out) {
    QSV_REQUIRE(ctx != nullptr && out != nullptr, "qsv_program_create: null argument");
    QSV_REQUIRE(nsteps >= 0 && (steps != nullptr || nsteps == 0), "qsv_program_create: bad steps");
    QSV_REQUIRE(nops >= 0 && (ops != nullptr || nops == 0), "qsv_program_create: bad ops");
    QSV_REQUIRE(pool != nullptr || pool_len == 0, "qsv_program_create: null pool");
    QSV_REQUIRE(n_total >= 1 && n_total <= QSV_MAX_QUBITS, "qsv_program_create: bad n_total");
    QSV_REQUIRE(n_total - n_local == log2i(ctx->nranks) && (1 << (n_total - n_local)) == ctx->nranks,
                "qsv_program_create: n_total - n_local must equal log2(nranks)");
    QSV_CUDA(cudaSetDevice(ctx->device));
    auto* prog = new qsv_program();
    prog->ctx = ctx;
    prog->n_total = n_total;
    prog->n_local = n_local;
    std::vector<unsigned char> all;
    for (int i = 0; i < nsteps; ++i) {
        qsv::Step s;
        s.desc = steps[i];
        if (steps[i].kind == QSV_STEP_PASS) {
            std::vector<unsigned char> blob;
            int rc = compile_pass(steps[i], n_total, n_local, ctx->rank, ops, nops, prims, nprims, pool,
                                  pool_len, s, blob);
            if (rc != QSV_OK) {
                set_error("step " + std::to_string(i) + ": " + qsv_last_error());
                delete prog;
                return rc;
            }
            s.blob_off = all.size();
            all.insert(all.end(), blob.begin(), blob.end());
        } else if (steps[i].kind == QSV_STEP_SWAP) {
            const qsv_step_desc& d = steps[i];
            if (!(d.swap_global >= n_local && d.swap_global < n_total && d.swap_local >= 0 &&
                  d.swap_local < n_local && d.chunk_log2 >= 0 && d.chunk_log2 <= n_local - 1 &&
                  d.nbuf >= 1 && d.nbuf <= 8)) {
                delete prog;
                set_error("step " + std::to_string(i) + ": bad swap (global/local/chunk/nbuf)");
                return QSV_E_ARG;
            }
            s.nvl_bytes = 16.0 * std::ldexp(1.0, n_local - 1);
            s.hbm_bytes = 4.0 * s.nvl_bytes;  // read+write of the sent and the received half
            prog->has_collective = true;
        } else {
            delete prog;
            set_error("step " + std::to_string(i) + ": unknown step kind");
            return QSV_E_ARG;
        }
        prog->steps.push_back(s);
    }
    if (!all.empty()) {
        cudaError_t e = qsv::dev_alloc(ctx, reinterpret_cast<void**>(&prog->d_blobs), all.size(), 2);
        if (e != cudaSuccess) {
            delete prog;
            set_error(std::string("qsv_program_create: cudaMalloc: ") + cudaGetErrorString(e));
            return QSV_E_NOMEM;
        }
        e = cudaMemcpy(prog->d_blobs, all.data(), all.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            qsv::dev_free(ctx, prog->d_blobs, 2);
            delete prog;
            set_error(std::string("qsv_program_create: upload: ") + cudaGetErrorString(e));
            return QSV_E_CUDA;
        }
        prog->blob_total = all.size();
        prog->host_blobs = std::move(all);
    }
    *out = prog;
    return QSV_OK;
}

namespace {

// Shared by qsv_program_validate / qsv_program_jit_check: host compile of every step.
int compile_steps_host(int n_total, int n_local, int rank, const qsv_step_desc* steps, int nsteps,
                       const qsv_op_desc* ops, int nops, const qsv_prim_desc* prims, int nprims,
                       const double* pool, size_t pool_len, std::vector<qsv::Step>* out_steps,
                       std::vector<unsigned char>* out_blobs) {
    QSV_REQUIRE(nsteps >= 0 && (steps != nullptr || nsteps == 0), "qsv_program_validate: bad steps");
    QSV_REQUIRE(nops >= 0 && (ops != nullptr || nops == 0), "qsv_program_validate: bad ops");
    QSV_REQUIRE(n_total >= 1 && n_total <= QSV_MAX_QUBITS && n_local >= 1 && n_local <= n_total,
                "qsv_program_validate: bad sizes");
    QSV_REQUIRE(rank >= 0 && (static_cast<uint64_t>(rank) >> (n_total - n_local)) == 0,
                "qsv_program_validate: rank out of range");
    for (int i = 0; i < nsteps; ++i) {
        qsv::Step s;
        s.desc = steps[i];
        if (steps[i].kind == QSV_STEP_PASS) {
            std::vector<unsigned char> blob;
            const int rc = compile_pass(steps[i], n_total, n_local, rank, ops, nops, prims, nprims, pool,
                                        pool_len, s, blob);
            if (rc != QSV_OK) {
                set_error("step " + std::to_string(i) + ": " + qsv_last_error());
                return rc;
            }
            if (out_blobs) {
                s.blob_off = out_blobs->size();
                out_blobs->insert(out_blobs->end(), blob.begin(), blob.end());
            }
        } else if (steps[i].kind == QSV_STEP_SWAP) {
            const qsv_step_desc& d = steps[i];
            QSV_REQUIRE(d.swap_global >= n_local && d.swap_global < n_total && d.swap_local >= 0 &&
                            d.swap_local < n_local && d.chunk_log2 >= 0 && d.chunk_log2 <= n_local - 1 &&
                            d.nbuf >= 1 && d.nbuf <= 8,
                        "step " + std::to_string(i) + ": bad swap (global/local/chunk/nbuf)");
        } else {
            QSV_REQUIRE(false, "step " + std::to_string(i) + ": unknown step kind");
        }
        if (out_steps)
            out_steps->push_back(s);
    }
    return QSV_OK;
}

} // namespace

extern "C" int qsv_program_validate(int n_total, int n_local, int rank, const qsv_step_desc* steps,
                                    int nsteps, const qsv_op_desc* ops, int nops, const qsv_prim_desc* prims,
                                    int nprims, const double* pool, size_t pool_len) {
    return compile_steps_host(n_total, n_local, rank, steps, nsteps, ops, nops, prims, nprims, pool, pool_len,
                              nullptr, nullptr);
}

extern "C" int qsv_program_jit_check(int n_total, int n_local, int rank, const qsv_step_desc* steps,
                                     int nsteps, const qsv_op_desc* ops, int nops, const qsv_prim_desc* prims,
                                     int nprims, const double* pool, size_t pool_len, int max_kernels,
                                     int* kernels) {
    std::vector<qsv::Step> st;
    std::vector<unsigned char> blobs;
    const int rc = compile_steps_host(n_total, n_local, rank, steps, nsteps, ops, nops, prims, nprims, pool,
                                      pool_len, &st, &blobs);
    if (rc != QSV_OK)
        return rc;
    return qsv::jit_check(st, blobs.data(), max_kernels, kernels);
}

extern "C" int qsv_program_time(qsv_state* st, qsv_program* prog, int iters, int64_t basis, float* ms) {
    QSV_REQUIRE(st != nullptr && prog != nullptr && ms != nullptr && iters >= 1, "qsv_program_time: bad argument");
    qsv_ctx* ctx = st->ctx;
    QSV_CUDA(cudaSetDevice(ctx->device));
    cudaEvent_t a, b;
    QSV_CUDA(cudaEventCreate(&a));
    QSV_CUDA(cudaEventCreate(&b));
    QSV_CUDA(cudaEventRecord(a, ctx->stream));
    int rc = QSV_OK;
    for (int i = 0; i < iters && rc == QSV_OK; ++i) {
        if (basis >= 0)
            rc = qsv_state_set_basis(st, static_cast<uint64_t>(basis));
        if (rc == QSV_OK)
            rc = qsv_program_run(st, prog);
    }
    QSV_CUDA(cudaEventRecord(b, ctx->stream));
    QSV_CUDA(cudaEventSynchronize(b));
    QSV_CUDA(cudaEventElapsedTime(ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return rc;
}

extern "C" int qsv_program_free(qsv_program* prog) {
    if (!prog)
        return QSV_OK;
    cudaSetDevice(prog->ctx->device);
    cudaStreamSynchronize(prog->ctx->stream);
    for (auto& kv : prog->graphs)
        cudaGraphExecDestroy(kv.second);
    qsv::jit_release(prog);
    if (prog->d_blobs)
        qsv::dev_free(prog->ctx, prog->d_blobs, 2);
    delete prog;
    return QSV_OK;
}

extern "C" int qsv_program_jit(qsv_program* prog, int max_kernels, double* seconds) {
    QSV_REQUIRE(prog != nullptr, "qsv_program_jit: null program");
    QSV_REQUIRE(max_kernels >= 0, "qsv_program_jit: max_kernels must be >= 0");
    QSV_CUDA(cudaSetDevice(prog->ctx->device));
    QSV_CUDA(cudaStreamSynchronize(prog->ctx->stream));
    return qsv::jit_program(prog, max_kernels, seconds);
}

extern "C" int qsv_program_jit_async(qsv_program* prog, int max_kernels) {
    QSV_REQUIRE(prog != nullptr, "qsv_program_jit_async: null program");
    QSV_REQUIRE(max_kernels >= 0, "qsv_program_jit_async: max_kernels must be >= 0");
    if (prog->ctx->nranks > 1) {  // every rank must switch kernels at the same run: compile now
        double s = 0;
        return qsv_program_jit(prog, max_kernels, &s);
    }
    return qsv::jit_start_async(prog, max_kernels);
}

extern "C" int qsv_program_jit_wait(qsv_program* prog, int block, int* done, double* seconds) {
    QSV_REQUIRE(prog != nullptr, "qsv_program_jit_wait: null program");
    const int rc = qsv::jit_poll(prog, block != 0);
    if (done)
        *done = qsv::jit_pending(prog) ? 0 : 1;
    if (seconds)
        *seconds = prog->jit_seconds;
    return rc;
}

extern "C" int qsv_program_jit_info(qsv_program* prog, int* kernels, int* steps_jitted) {
    QSV_REQUIRE(prog != nullptr, "qsv_program_jit_info: null program");
    if (kernels)
        *kernels = static_cast<int>(prog->jit_kernels.size());
    if (steps_jitted) {
        int c = 0;
        for (int j : prog->jit_of_step)
            c += j >= 0;
        *steps_jitted = c;
    }
    return QSV_OK;
}

namespace {

// BBOP overlap: can pass `p` run region by region behind swap (v, b)?  Region c of
// a swap = the shard slice whose half-index (index with bit v removed) has top
// bits c; a pass qualifies when none of its tile qubits is a region bit, so its
// tiles split into contiguous per-region ranges (region bits = top non-tile bits).
bool region_pass_ok(const qsv::Step& p, int v, int b, int l) {
    if (p.desc.kind != QSV_STEP_PASS)
        return false;
    const int minR = b < v ? b : b + 1;
    bool v_in_tile = false;
    for (int q = 0; q < p.geom.L; ++q) {
        if (q == v)
            v_in_tile = true;
        else if (q >= minR)
            return false;
    }
    for (int i = 0; i < p.geom.nhigh; ++i) {
        const int q = p.geom.high[i];
        if (q == v)
            v_in_tile = true;
        else if (q >= minR)
            return false;
    }
    if (v > minR && !v_in_tile)
        return false;
    return p.geom.K <= b + 1 && b + 1 < l;
}

int env_int(const char* name, int dflt) {
    const char* s = std::getenv(name);
    return s ? std::atoi(s) : dflt;
}

cudaError_t launch_step(qsv_state* st, qsv_program* prog, size_t i, uint64_t rank_base,
                        const qsv::LaunchRange& rg = qsv::LaunchRange{}, int region = -1) {
    const qsv::Step& s = prog->steps[i];
    qsv_ctx* ctx = st->ctx;
    ctx->trace_step = static_cast<int>(i);
    const int tr = qsv::trace_open(ctx, QSV_TRACE_PASS, region, 0, ctx->stream);
    cudaError_t e;
    if (!prog->jit_of_step.empty() && prog->jit_of_step[i] >= 0)
        e = qsv::launch_jit(prog, st, i, prog->d_blobs + s.blob_off, rank_base, ctx->stream, rg);
    else
        e = qsv::launch_pass(st, s, prog->d_blobs + s.blob_off, rank_base, ctx->stream, rg);
    qsv::trace_close(ctx, tr, ctx->stream);
    return e;
}

uint64_t tile_mask(const qsv::Step& p) {
    uint64_t m = (1ull << p.geom.L) - 1ull;
    for (int h = 0; h < p.geom.nhigh; ++h)
        m |= 1ull << p.geom.high[h];
    return m;
}

// BBOP over NVLink P2P: a swap split into 4 regions (two local bits outside the tiles
// of the passes around it) overlaps the passes before it (region c of the swap starts
// once region c of those passes is written) and after it (region c of those passes
// starts once region c of the swap has landed).
struct SwapOverlap {
    uint64_t rmask = 0;
    size_t pre_begin = 0;  // passes [pre_begin, swap) run region by region before it
    size_t post_end = 0;   // passes (swap, post_end] run region by region after it
};

std::map<size_t, SwapOverlap> plan_overlap(const qsv_program* prog, int l) {
    std::map<size_t, SwapOverlap> plans;
    size_t free_from = 0;  // first step not claimed by an earlier swap's post range
    const size_t n = prog->steps.size();
    for (size_t i = 0; i < n; ++i) {
        const qsv::Step& s = prog->steps[i];
        if (s.desc.kind != QSV_STEP_SWAP)
            continue;
        const int v = s.desc.swap_local;
        int best = 0;
        SwapOverlap bp;
        for (int b1 = l - 1; b1 >= 5; --b1)
            for (int b2 = b1 - 1; b2 >= 5; --b2) {
                if (b1 == v || b2 == v)
                    continue;
                const uint64_t rm = (1ull << b1) | (1ull << b2);
                auto ok = [&](const qsv::Step& p) {
                    return p.desc.kind == QSV_STEP_PASS && !(tile_mask(p) & rm) && p.geom.K + 2 <= l - 1;
                };
                size_t pre = i;
                while (pre > free_from && ok(prog->steps[pre - 1]))
                    --pre;
                size_t post = i;
                while (post + 1 < n && ok(prog->steps[post + 1]))
                    ++post;
                const int k = static_cast<int>((i - pre) + (post - i));
                if (k > best) {
                    best = k;
                    bp.rmask = rm;
                    bp.pre_begin = pre;
                    bp.post_end = post;
                }
            }
        if (best > 0) {
            plans[i] = bp;
            free_from = bp.post_end + 1;
        } else {
            free_from = i + 1;
        }
    }
    return plans;
}

// Do all ranks hold the same basis state |x> (set_basis on every rank, nothing run since)?
// Collective: one 16-byte max all-reduce of (v, -v), v = x or -1, so the ranks cannot diverge.
int agree_basis(qsv_state* st, bool* same) {
    qsv_ctx* ctx = st->ctx;
    *same = false;
    int64_t* d = reinterpret_cast<int64_t*>(ctx->d_coll + 128 * static_cast<size_t>(ctx->nranks) + 16);
    const int64_t v = st->is_basis ? static_cast<int64_t>(st->basis) : -1;
    int64_t h[2] = {v, -v};
    // on the comm stream only: the agreement does not wait for the compute stream's queue
    if (cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, ctx->comm_stream) != cudaSuccess) {
        cudaGetLastError();
        cudaMemsetAsync(d, 0xff, sizeof(h), ctx->comm_stream);  // (-1, -1): max = -1, never agreed
    }
    const ncclResult_t r = ncclAllReduce(d, d, 2, ncclInt64, ncclMax, ctx->comm, ctx->comm_stream);
    if (r != ncclSuccess) {
        qsv::abort_comm(ctx, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
        return qsv::check_aborted(ctx, "qsv_program_run: basis agreement");
    }
    if (int rc = qsv::wait_stream(ctx, ctx->comm_stream, "qsv_program_run: basis agreement"); rc != QSV_OK)
        return rc;
    QSV_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, ctx->comm_stream));
    QSV_CUDA(cudaStreamSynchronize(ctx->comm_stream));
    *same = h[0] >= 0 && h[0] == -h[1];
    return QSV_OK;
}

int enqueue_steps(qsv_state* st, qsv_program* prog, cudaEvent_t* evs) {
    qsv_ctx* ctx = st->ctx;
    // Leading qubit swaps on a basis state |x>: every rank knows x, so the swaps become x with
    // the swapped bits exchanged, set locally — no NVLink transfer.  The condition is rank-uniform
    // (same program, same env); the state test is agreed collectively.
    size_t first = 0;
    bool basis_start = false;
    if (evs == nullptr && ctx->nranks > 1 && ctx->comm != nullptr && !prog->steps.empty() &&
        prog->steps[0].desc.kind == QSV_STEP_SWAP && env_int("QSV_BASIS_SWAPS", 1) != 0 &&
        env_int("QSV_OVERLAP", 0) == 0) {  // the region-overlap schedule pairs passes with every swap
        QSV_CUDA(cudaSetDevice(ctx->device));
        if (int rc = agree_basis(st, &basis_start); rc != QSV_OK)
            return rc;
    }
    st->is_basis = false;  // the program below modifies the shard
    if (basis_start) {
        uint64_t x = st->basis;
        while (first < prog->steps.size() && prog->steps[first].desc.kind == QSV_STEP_SWAP) {
            const int g = prog->steps[first].desc.swap_global, v = prog->steps[first].desc.swap_local;
            const uint64_t bg = (x >> g) & 1ull, bv = (x >> v) & 1ull;
            if (bg != bv)
                x ^= (1ull << g) | (1ull << v);
            ++first;
        }
        if (first > 0 && x != st->basis) {
            // move the single 1 from |basis> to |x> (the rest of every shard is already zero)
            const uint64_t lmask = st->size - 1, me = static_cast<uint64_t>(ctx->rank);
            QSV_CUDA(cudaSetDevice(ctx->device));
            if ((st->basis >> st->n_local) == me)
                set_amp_kernel<<<1, 1, 0, ctx->stream>>>(st->amps + (st->basis & lmask), 0.0);
            if ((x >> st->n_local) == me)
                set_amp_kernel<<<1, 1, 0, ctx->stream>>>(st->amps + (x & lmask), 1.0);
            QSV_CUDA(cudaGetLastError());
        }
    }
    const uint64_t rank_base = static_cast<uint64_t>(ctx->rank) << st->n_local;
    const bool overlap = evs == nullptr && env_int("QSV_OVERLAP", 0) != 0;
    const int reserve = std::max(0, env_int("QSV_OVERLAP_RESERVE_SMS", 8));
    const int l = st->n_local;
    // P2P region schedule (collective check on the first swap: all ranks agree)
    std::map<size_t, SwapOverlap> p2p_plan;
    bool p2p = false;
    if (overlap && prog->has_collective) {
        for (const qsv::Step& s : prog->steps)
            if (s.desc.kind == QSV_STEP_SWAP) {
                p2p = qsv::p2p_swap_ready(st, s.desc.swap_global);
                break;
            }
        if (p2p)
            p2p_plan = plan_overlap(prog, l);
    }
    const int swap_sms = std::max(1, std::min(ctx->sm_count - 1, env_int("QSV_SWAP_SMS", 16)));
    auto region_of = [&](uint64_t rm, uint64_t c) {
        qsv::LaunchRange rg;
        rg.rmask = rm;
        int k = 0;
        for (int q = 0; q < 64; ++q)
            if ((rm >> q) & 1ull)
                rg.rval |= ((c >> k++) & 1ull) << q;
        return rg;
    };
    // pre-pass start index -> swap index
    std::map<size_t, size_t> pre_start;
    for (const auto& kv : p2p_plan)
        if (kv.second.pre_begin < kv.first)
            pre_start[kv.second.pre_begin] = kv.first;
    for (size_t i = first; i < prog->steps.size(); ++i) {
        const qsv::Step& s = prog->steps[i];
        ctx->trace_step = static_cast<int>(i);
        if (evs)
            QSV_CUDA(cudaEventRecord(evs[i], ctx->stream));
        auto ps = pre_start.find(i);
        if (ps != pre_start.end()) {
            // passes [i, swap) region by region, then the swap fed region by region,
            // then the post passes region by region
            const size_t w = ps->second;
            const SwapOverlap& ov = p2p_plan[w];
            const qsv::Step& sw = prog->steps[w];
            std::vector<cudaEvent_t> pre_ev, done;
            cudaError_t err = cudaSuccess;
            for (uint64_t c = 0; c < 4 && err == cudaSuccess; ++c) {
                qsv::LaunchRange rg = region_of(ov.rmask, c);
                rg.sms = c > 0 ? ctx->sm_count - swap_sms : 0;
                for (size_t p = i; p < w && err == cudaSuccess; ++p)
                    err = launch_step(st, prog, p, rank_base, rg, static_cast<int>(c));
                cudaEvent_t e;
                cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
                cudaEventRecord(e, ctx->stream);
                pre_ev.push_back(e);
            }
            ctx->trace_step = static_cast<int>(w);
            int rc = err == cudaSuccess ? qsv::run_swap(st, sw.desc.swap_global, sw.desc.swap_local, sw.desc.chunk_log2,
                                                        sw.desc.nbuf, &done, ov.rmask, &pre_ev)
                                        : QSV_E_CUDA;
            for (uint64_t c = 0; c < done.size() && err == cudaSuccess && rc == QSV_OK; ++c) {
                err = cudaStreamWaitEvent(ctx->stream, done[c], 0);
                qsv::LaunchRange rg = region_of(ov.rmask, c);
                rg.sms = c + 1 < done.size() ? ctx->sm_count - swap_sms : 0;
                for (size_t p = w + 1; p <= ov.post_end && err == cudaSuccess; ++p)
                    err = launch_step(st, prog, p, rank_base, rg, static_cast<int>(c));
            }
            qsv::join_swap(ctx);
            for (cudaEvent_t e : pre_ev)
                cudaEventDestroy(e);
            for (cudaEvent_t e : done)
                cudaEventDestroy(e);
            QSV_CUDA(err);
            if (rc != QSV_OK)
                return rc;
            i = ov.post_end;
            continue;
        }
        if (s.desc.kind == QSV_STEP_PASS) {
            // BBOP push (QSV_FUSE_SWAP=2, default): a swap right after this pass rides in its
            // stores — the runs that move are posted into the peer's shard over NVLink, so the
            // pass's compute and HBM traffic hide under the transfer (QFT-32 on 2 GPUs: 25.8 ms
            // for the fused step vs 11.9 + 24.9 ms; profiles/r02_bbop.md)
            if (evs == nullptr && !overlap && env_int("QSV_FUSE_SWAP", 2) == 2 && i + 1 < prog->steps.size() &&
                prog->steps[i + 1].desc.kind == QSV_STEP_SWAP &&
                // a run of swaps goes to the merged all-to-all instead
                !(i + 2 < prog->steps.size() && prog->steps[i + 2].desc.kind == QSV_STEP_SWAP) &&
                (prog->jit_of_step.empty() || prog->jit_of_step[i] < 0 ||
                 prog->jit_kernels[prog->jit_of_step[i]].mt == 1)) {
                const qsv_step_desc& sw = prog->steps[i + 1].desc;
                qsv::FusedSwap fs;
                const int rc = qsv::fused_swap_prepare(st, sw.swap_global, sw.swap_local, s, &fs);
                if (rc == QSV_OK) {
                    fs.push = 1;
                    qsv::LaunchRange rg;
                    rg.fuse = &fs;
                    QSV_CUDA(launch_step(st, prog, i, rank_base, rg, -2));
                    ctx->trace_step = static_cast<int>(i + 1);
                    if (int rc2 = qsv::fused_swap_finish(st, sw.swap_global); rc2 != QSV_OK)
                        return rc2;
                    ++i;
                    continue;
                }
                if (rc != QSV_E_STATE)
                    return rc;
            }
            QSV_CUDA(launch_step(st, prog, i, rank_base));
            continue;
        }
        const int v = s.desc.swap_local, b = s.desc.chunk_log2;
        // BBOP pull: the swap fused into the next pass (the pass streams the peer's half over
        // NVLink in its own loads), when P2P is up and the pass geometry allows it.  Opt-in
        // (QSV_FUSE_SWAP=1): bitwise equal to swap + pass, but its remote TMA loads reach
        // ~420 GB/s against the swap kernel's 695 (QFT-32 on 2 GPUs: 40.9 ms fused vs
        // 24.7 + 15.0 ms), and random-34 on 2 GPUs ran 4.5 s vs 2.8 s (profiles/r02_bbop.md).
        // The default is the push form above (QSV_FUSE_SWAP=2; 0 = separate swaps).
        if (evs == nullptr && !overlap && env_int("QSV_FUSE_SWAP", 0) == 1 && i + 1 < prog->steps.size() &&
            prog->steps[i + 1].desc.kind == QSV_STEP_PASS &&
            (prog->jit_of_step.empty() || prog->jit_of_step[i + 1] < 0 ||
             prog->jit_kernels[prog->jit_of_step[i + 1]].mt == 1)) {
            qsv::FusedSwap fs;
            const int rc = qsv::fused_swap_prepare(st, s.desc.swap_global, v, prog->steps[i + 1], &fs);
            if (rc == QSV_OK) {
                qsv::LaunchRange rg;
                rg.fuse = &fs;
                QSV_CUDA(launch_step(st, prog, i + 1, rank_base, rg, -2));
                ++i;
                continue;
            }
            if (rc != QSV_E_STATE)
                return rc;
        }
        if (evs == nullptr && !overlap && env_int("QSV_MERGE_SWAPS", 1) != 0 && i + 1 < prog->steps.size() &&
            prog->steps[i + 1].desc.kind == QSV_STEP_SWAP && qsv::p2p_swap_ready(st, s.desc.swap_global)) {
            // consecutive swaps of distinct global and distinct local qubits: one all-to-all
            int gs[3] = {s.desc.swap_global, 0, 0}, vs[3] = {v, 0, 0}, k = 1;
            size_t j = i + 1;
            while (k < 3 && j < prog->steps.size() && prog->steps[j].desc.kind == QSV_STEP_SWAP) {
                const qsv_step_desc& d2 = prog->steps[j].desc;
                bool disjoint = true;
                for (int q = 0; q < k; ++q)
                    disjoint = disjoint && d2.swap_global != gs[q] && d2.swap_local != vs[q];
                if (!disjoint)
                    break;
                gs[k] = d2.swap_global;
                vs[k] = d2.swap_local;
                ++k;
                ++j;
            }
            if (k >= 2) {
                const int rc = qsv::run_multi_swap(st, gs, vs, k);
                if (rc == QSV_OK) {
                    i = j - 1;
                    continue;
                }
                if (rc != QSV_E_STATE)
                    return rc;
            }
        }
        if (p2p) {
            auto it = p2p_plan.find(i);
            if (it != p2p_plan.end() && it->second.post_end > i) {
                // no pre passes: the swap, then its post passes region by region
                std::vector<cudaEvent_t> done;
                const int rc = qsv::run_swap(st, s.desc.swap_global, v, b, s.desc.nbuf, &done, it->second.rmask);
                cudaError_t err = cudaSuccess;
                for (uint64_t c = 0; c < done.size() && err == cudaSuccess && rc == QSV_OK; ++c) {
                    err = cudaStreamWaitEvent(ctx->stream, done[c], 0);
                    qsv::LaunchRange rg = region_of(it->second.rmask, c);
                    rg.sms = c + 1 < done.size() ? ctx->sm_count - swap_sms : 0;
                    for (size_t p = i + 1; p <= it->second.post_end && err == cudaSuccess; ++p)
                        err = launch_step(st, prog, p, rank_base, rg, static_cast<int>(c));
                }
                qsv::join_swap(ctx);
                for (cudaEvent_t e : done)
                    cudaEventDestroy(e);
                QSV_CUDA(err);
                if (rc != QSV_OK)
                    return rc;
                i = it->second.post_end;
                continue;
            }
            const int rc = qsv::run_swap(st, s.desc.swap_global, v, b, s.desc.nbuf);
            if (rc != QSV_OK)
                return rc;
            continue;
        }
        size_t j = i + 1;
        while (overlap && j < prog->steps.size() && region_pass_ok(prog->steps[j], v, b, l))
            ++j;
        if (j > i + 1) {
            std::vector<cudaEvent_t> done;
            const int rc = qsv::run_swap(st, s.desc.swap_global, v, b, s.desc.nbuf, &done);
            if (rc != QSV_OK) {
                for (cudaEvent_t e : done)
                    cudaEventDestroy(e);
                return rc;
            }
            const uint64_t C = done.size();
            const int sms = std::max(1, ctx->sm_count - reserve);
            cudaError_t err = cudaSuccess;
            for (uint64_t c = 0; c < C && err == cudaSuccess; ++c) {
                err = cudaStreamWaitEvent(ctx->stream, done[c], 0);
                for (size_t p = i + 1; p < j && err == cudaSuccess; ++p) {
                    const uint64_t T = st->size >> prog->steps[p].geom.K;
                    qsv::LaunchRange rg;
                    rg.tile0 = c * (T / C);
                    rg.count = T / C;
                    rg.sms = c + 1 < C ? sms : 0;  // the last region runs after the transfers
                    err = launch_step(st, prog, p, rank_base, rg, static_cast<int>(c));
                }
            }
            qsv::join_swap(ctx);
            for (cudaEvent_t e : done)
                cudaEventDestroy(e);
            QSV_CUDA(err);
            i = j - 1;
            continue;
        }
        {
            const int rc = qsv::run_swap(st, s.desc.swap_global, s.desc.swap_local, s.desc.chunk_log2,
                                         s.desc.nbuf);
            if (rc != QSV_OK)
                return rc;
        }
    }
    if (evs)
        QSV_CUDA(cudaEventRecord(evs[prog->steps.size()], ctx->stream));
    return QSV_OK;
}

} // namespace

extern "C" int qsv_program_run(qsv_state* st, qsv_program* prog) {
    QSV_REQUIRE(st != nullptr && prog != nullptr, "qsv_program_run: null argument");
    QSV_REQUIRE(st->ctx == prog->ctx, "qsv_program_run: state and program belong to different contexts");
    QSV_REQUIRE(st->n_local == prog->n_local, "qsv_program_run: state size differs from the program's");
    qsv_ctx* ctx = st->ctx;
    if (int rc = qsv::check_aborted(ctx, "qsv_program_run"); rc != QSV_OK)
        return rc;
    QSV_CUDA(cudaSetDevice(ctx->device));
    if (qsv::jit_poll(prog, false) != QSV_OK) {  // a failed background compile: keep the interpreter
        std::fprintf(stderr, "qsv: background JIT failed, using the interpreter pass kernel (%s)\n",
                     qsv_last_error());
    }
    if (prog->has_collective || prog->steps.size() < 4 || ctx->trace_on || qsv::jit_pending(prog))
        return enqueue_steps(st, prog, nullptr);
    auto it = prog->graphs.find(st->amps);
    if (it == prog->graphs.end()) {
        // First run on this buffer: run eagerly (configures kernel attributes),
        // then capture the launch sequence as a CUDA graph for later runs.
        int rc = enqueue_steps(st, prog, nullptr);
        if (rc != QSV_OK)
            return rc;
        cudaGraph_t g = nullptr;
        QSV_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        rc = enqueue_steps(st, prog, nullptr);
        cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
        if (rc != QSV_OK)
            return rc;
        QSV_CUDA(e);
        cudaGraphExec_t ge = nullptr;
        QSV_CUDA(cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
        prog->graphs[st->amps] = ge;
        return QSV_OK;
    }
    st->is_basis = false;
    QSV_CUDA(cudaGraphLaunch(it->second, ctx->stream));
    return QSV_OK;
}

extern "C" int qsv_program_profile(qsv_state* st, qsv_program* prog, float* ms_out) {
    QSV_REQUIRE(st != nullptr && prog != nullptr && ms_out != nullptr, "qsv_program_profile: null argument");
    qsv_ctx* ctx = st->ctx;
    QSV_CUDA(cudaSetDevice(ctx->device));
    if (qsv::jit_poll(prog, false) != QSV_OK)
        std::fprintf(stderr, "qsv: background JIT failed, using the interpreter pass kernel (%s)\n", qsv_last_error());
    const size_t n = prog->steps.size();
    std::vector<cudaEvent_t> evs(n + 1);
    for (auto& e : evs)
        QSV_CUDA(cudaEventCreate(&e));
    int rc = enqueue_steps(st, prog, evs.data());
    if (rc == QSV_OK) {
        QSV_CUDA(cudaEventSynchronize(evs[n]));
        for (size_t i = 0; i < n; ++i)
            QSV_CUDA(cudaEventElapsedTime(&ms_out[i], evs[i], evs[i + 1]));
    }
    for (auto& e : evs)
        cudaEventDestroy(e);
    return rc;
}

extern "C" int qsv_program_step_cost(qsv_program* prog, int i, double* hbm_bytes, double* flops,
                                     double* nvlink_bytes) {
    QSV_REQUIRE(prog != nullptr && i >= 0 && i < static_cast<int>(prog->steps.size()),
                "qsv_program_step_cost: bad step index");
    const qsv::Step& s = prog->steps[i];
    if (hbm_bytes) *hbm_bytes = s.hbm_bytes;
    if (flops) *flops = s.flops;
    if (nvlink_bytes) *nvlink_bytes = s.nvl_bytes;
    return QSV_OK;
}

extern "C" int qsv_apply_fused(qsv_state* st, int k, const int* targets, uint64_t ctrl_mask,
                               const double* mat) {
    QSV_REQUIRE(st != nullptr && targets != nullptr && mat != nullptr, "qsv_apply_fused: null argument");
    st->is_basis = false;
    QSV_REQUIRE(k >= 1 && k <= QSV_MAX_DENSE_K, "qsv_apply_fused: k must be in [1, 5] (SPEC:89)");
    qsv_ctx* ctx = st->ctx;
    const int n_local = st->n_local;
    const int n_total = n_local + log2i(ctx->nranks);
    qsv_op_desc op{};
    op.kind = QSV_OP_DENSE;
    op.k = k;
    for (int i = 0; i < k; ++i)
        op.qubits[i] = targets[i];
    op.ctrl_mask = ctrl_mask;
    op.mat_off = 0;
    // tile: low run plus the targets above it
    qsv_step_desc sd{};
    sd.kind = QSV_STEP_PASS;
    const int K = std::min(10, n_local);
    std::vector<int> high;
    for (int i = 0; i < k; ++i)
        if (targets[i] >= K - k)
            high.push_back(targets[i]);
    std::sort(high.begin(), high.end());
    // shrink until the high set is consistent with the low run
    int nh = static_cast<int>(high.size());
    while (true) {
        const int L = K - nh;
        std::vector<int> hh;
        for (int i = 0; i < k; ++i)
            if (targets[i] >= L)
                hh.push_back(targets[i]);
        std::sort(hh.begin(), hh.end());
        if (static_cast<int>(hh.size()) == nh) {
            high = hh;
            break;
        }
        nh = static_cast<int>(hh.size());
    }
    sd.tile_k = K;
    sd.nhigh = static_cast<int>(high.size());
    for (size_t i = 0; i < high.size(); ++i)
        sd.high[i] = high[i];
    sd.op_begin = 0;
    sd.op_count = 1;
    qsv_program* prog = nullptr;
    int rc = qsv_program_create(ctx, n_total, n_local, &sd, 1, &op, 1, nullptr, 0, mat,
                                static_cast<size_t>(1) << (2 * k), &prog);
    if (rc != QSV_OK)
        return rc;
    rc = qsv_program_run(st, prog);
    qsv_program_free(prog);
    return rc;
}

// ======================================================================= reductions
extern "C" int qsv_norm_sq(qsv_state* st, double* out) {
    QSV_REQUIRE(st != nullptr && out != nullptr, "qsv_norm_sq: null argument");
    qsv_ctx* ctx = st->ctx;
    QSV_CUDA(cudaSetDevice(ctx->device));
    int rc = ensure_partials(ctx);
    if (rc != QSV_OK)
        return rc;
    const int grid = reduce_grid(ctx);
    norm_partial_kernel<<<grid, kRedThreads, 0, ctx->stream>>>(st->amps, st->size, ctx->d_partials);
    QSV_CUDA(cudaGetLastError());
    sum_partials_kernel<<<1, kRedThreads, 0, ctx->stream>>>(ctx->d_partials, grid,
                                                           ctx->d_partials + ctx->partials_cap - 1);
    QSV_CUDA(cudaGetLastError());
    QSV_CUDA(cudaMemcpyAsync(ctx->h_result, ctx->d_partials + ctx->partials_cap - 1, sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
    QSV_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = ctx->h_result[0];
    return QSV_OK;
}

extern "C" int qsv_max_abs_diff(qsv_state* st, const double* host_ref, uint64_t offset, uint64_t count,
                                double* out) {
    QSV_REQUIRE(st != nullptr && out != nullptr && (host_ref != nullptr || count == 0),
                "qsv_max_abs_diff: null argument");
    QSV_REQUIRE(offset <= st->size && count <= st->size - offset, "qsv_max_abs_diff: range outside shard");
    qsv_ctx* ctx = st->ctx;
    QSV_CUDA(cudaSetDevice(ctx->device));
    int rc = ensure_partials(ctx);
    if (rc != QSV_OK)
        return rc;
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 26);  // 1 GiB staging at most
    if (ctx->scratch_bytes < chunk * sizeof(double2)) {
        if (ctx->d_scratch)
            qsv::dev_free(ctx, ctx->d_scratch, 3);
        ctx->d_scratch = nullptr;
        ctx->scratch_bytes = 0;
        QSV_CUDA(qsv::dev_alloc(ctx, reinterpret_cast<void**>(&ctx->d_scratch),
                                std::max<uint64_t>(chunk, 1) * sizeof(double2), 3));
        ctx->scratch_bytes = std::max<uint64_t>(chunk, 1) * sizeof(double2);
    }
    double worst = 0.0;
    const int grid = reduce_grid(ctx);
    for (uint64_t done = 0; done < count; done += chunk) {
        const uint64_t c = std::min(chunk, count - done);
        QSV_CUDA(cudaMemcpyAsync(ctx->d_scratch, host_ref + 2 * done, c * sizeof(double2),
                                 cudaMemcpyHostToDevice, ctx->stream));
        diff_partial_kernel<<<grid, kRedThreads, 0, ctx->stream>>>(
            st->amps + offset + done, reinterpret_cast<const double2*>(ctx->d_scratch), c, ctx->d_partials);
        QSV_CUDA(cudaGetLastError());
        double m = 0.0;
        rc = finish_max(ctx, grid, &m);
        if (rc != QSV_OK)
            return rc;
        worst = std::max(worst, m);
    }
    *out = worst;
    return QSV_OK;
}

extern "C" int qsv_check_qft_basis(qsv_state* st, int n_total, uint64_t x, double* out) {
    QSV_REQUIRE(st != nullptr && out != nullptr, "qsv_check_qft_basis: null argument");
    QSV_REQUIRE(n_total >= st->n_local && n_total <= QSV_MAX_QUBITS, "qsv_check_qft_basis: bad n_total");
    qsv_ctx* ctx = st->ctx;
    QSV_CUDA(cudaSetDevice(ctx->device));
    int rc = ensure_partials(ctx);
    if (rc != QSV_OK)
        return rc;
    const int grid = reduce_grid(ctx);
    qft_check_kernel<<<grid, kRedThreads, 0, ctx->stream>>>(
        st->amps, st->size, static_cast<uint64_t>(ctx->rank) << st->n_local, n_total, x, ctx->d_partials);
    QSV_CUDA(cudaGetLastError());
    return finish_max(ctx, grid, out);
}

extern "C" int qsv_state_digest(qsv_state* st, uint64_t* out) {
    QSV_REQUIRE(st != nullptr && out != nullptr, "qsv_state_digest: null argument");
    qsv_ctx* ctx = st->ctx;
    QSV_CUDA(cudaSetDevice(ctx->device));
    int rc = ensure_partials(ctx);
    if (rc != QSV_OK)
        return rc;
    unsigned long long* d = reinterpret_cast<unsigned long long*>(ctx->d_partials);
    QSV_CUDA(cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), ctx->stream));
    digest_kernel<<<reduce_grid(ctx), kRedThreads, 0, ctx->stream>>>(
        reinterpret_cast<const unsigned long long*>(st->amps), 2 * st->size, d);
    QSV_CUDA(cudaGetLastError());
    QSV_CUDA(cudaMemcpyAsync(ctx->h_result, d, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             ctx->stream));
    QSV_CUDA(cudaStreamSynchronize(ctx->stream));
    uint64_t w[2];
    std::memcpy(w, ctx->h_result, sizeof(w));
    *out = w[0] ^ (w[1] * 0xD6E8FEB86659FD93ull);
    return QSV_OK;
}

extern "C" int qsv_swap(qsv_state* st, int g, int v, int chunk_log2, int nbuf) {
    QSV_REQUIRE(st != nullptr, "qsv_swap: null state");
    st->is_basis = false;
    return qsv::run_swap(st, g, v, chunk_log2, nbuf);
}
