// Internal (non-ABI) structures shared by the libqsv translation units.
#pragma once

#include "qsv.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "device_types.h"

static_assert(QSV_OP_RBLOCK == 3 && QSV_OP_PHASEPROD == 4 && QSV_OP_PARPHASE == 5 && QSV_PRIM_U1I == 6 &&
                  QSV_MAX_HIGH == 8,
              "device_types.h constants must mirror include/qsv.h");

namespace qsv {

// Tile geometry of one pass: tile = [0, L) U {high[0..nhigh)} in local index bits.
struct PassGeom {
    int32_t K;        // tile qubits
    int32_t L;        // contiguous low run
    int32_t nhigh;
    int32_t high[QSV_MAX_HIGH];
    int32_t kmax;     // largest dense arity in the pass (selects the kernel variant)
};

struct Step {
    qsv_step_desc desc;
    PassGeom geom{};
    int nops = 0;
    uint64_t blob_off = 0;   // byte offset of this pass's blob in Program::d_blobs
    uint32_t blob_bytes = 0;
    double hbm_bytes = 0, flops = 0, nvl_bytes = 0;
};

} // namespace qsv

struct qsv_ctx {
    int device = 0;
    int rank = 0;
    int nranks = 1;
    int sm_count = 0;
    cudaStream_t stream = nullptr;      // compute stream (all public work is ordered here)
    cudaStream_t comm_stream = nullptr; // NCCL transfers of a swap
    cudaStream_t copy_stream = nullptr; // staging copy-back of a swap
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    ncclComm_t comm = nullptr;
    // reduction scratch
    double* d_partials = nullptr;
    double* h_result = nullptr;   // pinned, 4 doubles
    size_t partials_cap = 0;
    // swap staging (nbuf chunks)
    void* d_stage = nullptr;
    size_t stage_bytes = 0;
    // host->device scratch for diff checks
    double* d_scratch = nullptr;
    size_t scratch_bytes = 0;
    // pairwise barrier tokens of the P2P swap (2 doubles)
    double* d_sync = nullptr;
    // collective scratch (peer-handle exchange: 128 B per rank + a flag), allocated
    // before the communicator so that no rank leaves a collective early
    unsigned char* d_coll = nullptr;
    // failure semantics: set by qsv_ctx_abort (any thread) or by a failed
    // wait; once set, every later call on this context fails with QSV_E_NCCL
    std::atomic<int> aborted{0};
    std::atomic<int> comm_aborted{0};
    std::mutex abort_lock;      // guards abort_reason (written by the aborting thread)
    std::string abort_reason;
    // PipelineTrace: timing events around every pass launch, swap kernel,
    // send/recv chunk and copy-back while tracing is on (qsv_trace_enable)
    bool trace_on = false;
    cudaEvent_t trace_base = nullptr;
    struct TraceEv {
        int32_t kind, step, chunk, stream;
        cudaEvent_t a, b;
    };
    std::vector<TraceEv> trace;
    int trace_step = -1;  // step being enqueued (read by the swap code)
    // instrumented device memory: every cudaMalloc/cudaFree of the
    // library goes through qsv::dev_alloc / dev_free, which keep these counters and call
    // the caller's hook (qsim feeds memtrack from it)
    std::atomic<size_t> mem_cur{0}, mem_peak{0};
    std::map<void*, size_t> mem_sizes;
    qsv_alloc_hook alloc_hook = nullptr;
    void* alloc_user = nullptr;
};

struct qsv_state {
    qsv_ctx* ctx = nullptr;
    int n_local = 0;
    uint64_t size = 0;     // 2^n_local amplitudes
    double2* amps = nullptr;
    // peer shards mapped into this process (NVLink P2P swaps); filled by the first
    // collective swap: same-process ranks by peer access, other processes by CUDA IPC
    bool peers_ready = false;
    std::vector<double2*> peer_amps;   // per rank, nullptr = not mapped
    std::vector<char> peer_ipc;        // 1 = opened with cudaIpcOpenMemHandle (close on free)
    uint64_t fused_epoch = 0;          // fused swaps run on this buffer (flag epochs)
    // the shard holds the basis state |basis> set by qsv_state_set_basis and nothing has
    // touched it since: leading qubit swaps of a program then relabel the index instead of
    // moving data (a swap maps a basis state to a basis state)
    bool is_basis = false;
    uint64_t basis = 0;
};

namespace qsv {
struct JitKernel {
    void* func = nullptr;    // CUfunction
    int nt = 0;              // threads per CTA (mt tile groups)
    int mt = 1;
    size_t tile_smem = 0;
};
struct JitBuild;             // compiled + loaded kernels not yet adopted by the program (jit.cu)
} // namespace qsv

struct qsv_program {
    qsv_ctx* ctx = nullptr;
    int n_total = 0, n_local = 0;
    std::vector<qsv::Step> steps;
    unsigned char* d_blobs = nullptr;
    size_t blob_total = 0;
    std::vector<unsigned char> host_blobs;     // host copy (JIT code generation)
    std::vector<int> jit_of_step;              // JIT kernel per step, -1 = interpreter
    std::vector<qsv::JitKernel> jit_kernels;
    std::vector<void*> jit_modules;            // CUmodule
    // background compile (qsv_program_jit_async): the thread fills `jit_build` and sets
    // jit_done; the host thread adopts the kernels at the next run (interpreter until then)
    std::thread jit_thread;
    std::atomic<bool> jit_done{false};
    qsv::JitBuild* jit_build = nullptr;
    double jit_seconds = 0;                    // compile + load time of the adopted kernels
    bool has_collective = false;
    // one captured graph per state buffer it was run on
    std::map<const void*, cudaGraphExec_t> graphs;
    // tile tensor maps per (step, state buffer) (jit.cu tile_tensor_map)
    mutable std::map<std::pair<const void*, const void*>, qsv::TmaDesc> tmaps;
};

namespace qsv {
void set_error(const std::string& msg);
// A qubit swap fused into the pass that follows it (GeomArg::peer and friends).
struct FusedSwap {
    const double2* peer = nullptr;
    unsigned long long* flag_mine = nullptr;
    unsigned long long* flag_peer = nullptr;
    uint64_t epoch = 0;
    int sv = 0, sv_tile = 0, sv_tidx = 0;
    uint32_t sgbit = 0;
    int push = 0;  // 1: fused into the pass before the swap (remote stores), else after (remote loads)
};
// Tile range and SM budget of one pass launch (default: every tile, every SM).
struct LaunchRange {
    const FusedSwap* fuse = nullptr;  // the pass runs with a swap fused into its loads
    uint64_t tile0 = 0;
    uint64_t count = ~0ull;  // clipped to the pass's tile count
    int sms = 0;             // 0: all SMs; else persistent grid over this many SMs
    uint64_t rmask = 0;      // region bits (<= 3, outside the pass's tile)
    uint64_t rval = 0;       // their values (a subset of rmask)
};
// Fills the region fields of `ga` from rg; returns the number of tiles of the region.
uint64_t apply_region(GeomArg& ga, const LaunchRange& rg, uint64_t all_tiles);
// Launches the pass kernel variant for `geom` on `st` (compute stream).
cudaError_t launch_pass(const qsv_state* st, const Step& step, const unsigned char* d_blob,
                        uint64_t rank_base, cudaStream_t stream, const LaunchRange& rg = LaunchRange{});
// NVRTC specialisation (jit.cu).
bool jit_available(std::string& why);
int jit_program(qsv_program* prog, int max_kernels, double* seconds);
int jit_start_async(qsv_program* prog, int max_kernels);
// adopts a finished background compile (waits for it when `wait`); returns QSV_OK while it runs
int jit_poll(qsv_program* prog, bool wait);
bool jit_pending(const qsv_program* prog);
// Host-only: NVRTC-compiles the distinct pass kernels of compiled steps (no device).
int jit_check(const std::vector<Step>& steps, const unsigned char* host_blobs, int max_kernels, int* kernels);
cudaError_t launch_jit(const qsv_program* prog, const qsv_state* st, size_t step, const unsigned char* d_blob,
                       uint64_t rank_base, cudaStream_t stream, const LaunchRange& rg = LaunchRange{});
void jit_release(qsv_program* prog);
// Runs one chunked qubit swap (BBOP) of `st` with its peer; see qsv_swap.
// With `chunk_done`, one event per chunk (recorded when the chunk's region is
// final) is appended and the join with the compute stream is left to the caller
// (join_swap), so that region passes can start chunk by chunk (BBOP overlap).
// P2P mode: `region_mask` (<= 2 local bits, not v) splits the swap into regions, one
// event each; otherwise chunks follow the NCCL top-bit order.
// `pre_ready` (4 events, P2P regions only): region c starts once pre_ready[c] fired on
// this rank and the matching event on the peer (pair barrier) instead of after all
// earlier work on the compute stream.
int run_swap(qsv_state* st, int g, int v, int chunk_log2, int nbuf,
             std::vector<cudaEvent_t>* chunk_done = nullptr, uint64_t region_mask = 0,
             const std::vector<cudaEvent_t>* pre_ready = nullptr);
// Collective on first use: maps the peers' shards; true when swap g will use NVLink P2P.
bool p2p_swap_ready(qsv_state* st, int g);
void join_swap(qsv_ctx* ctx);
// Fused swap (g <-> v) into the pass `step` that follows it: maps the peers (collective on
// first use), orders the compute stream after a pair barrier with the peer (both shards
// final) and fills `out`.  QSV_E_STATE when P2P is unavailable or the pass geometry does
// not allow it (v in the pass's contiguous low run): run a plain swap instead.
int fused_swap_prepare(qsv_state* st, int g, int v, const Step& step, FusedSwap* out);
// Push mode: after the pass that pushed its half to the peer, order the compute stream after
// a pair barrier (the peer's pushes into this shard have landed).
int fused_swap_finish(qsv_state* st, int g);
// k = 2 or 3 consecutive disjoint swaps (gs[i] <-> vs[i]) as one NVLink P2P all-to-all
// among the 2^k ranks that differ in the g bits.  QSV_E_STATE when P2P is unavailable.
int run_multi_swap(qsv_state* st, const int* gs, const int* vs, int k);
// Fused-swap flags (one per CTA) live after the 2^l amplitudes of a state buffer.
constexpr size_t kFlagBytes = 4096 * sizeof(unsigned long long);
// Waits for `stream` on a multi-rank context without hanging on a dead peer: polls
// the stream, the context's abort flag and ncclCommGetAsyncError, and aborts the
// communicator (ncclCommAbort) after QSV_COLL_TIMEOUT_S seconds (default 900).
// Single-rank contexts synchronize directly.  Returns QSV_OK or QSV_E_NCCL/QSV_E_CUDA.
int wait_stream(qsv_ctx* ctx, cudaStream_t stream, const char* what);
// Aborts the communicator once (safe from any thread) and records `why`.
void abort_comm(qsv_ctx* ctx, const std::string& why);
// QSV_E_NCCL with the abort reason when the context was aborted, else QSV_OK.
int check_aborted(qsv_ctx* ctx, const char* what);
// Device allocations of a context (counted, reported to the context's hook).
cudaError_t dev_alloc(qsv_ctx* ctx, void** p, size_t bytes, int kind);
void dev_free(qsv_ctx* ctx, void* p, int kind);
// Trace records (no-ops unless tracing is on): open records an event on `s` before the
// traced work and returns its index, close records the end event after it.
int trace_open(qsv_ctx* ctx, int kind, int chunk, int stream_id, cudaStream_t s);
void trace_close(qsv_ctx* ctx, int idx, cudaStream_t s);
} // namespace qsv
