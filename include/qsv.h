/*
 * qsv.h — the C-ABI between the C++ host library (qsim, the reference API of
 * proj/include/qsim) and the sm_100a CUDA kernels in libqsv.so.
 *
 * This is the ONLY host->device crossing of the simulator.  Signatures are
 * plain C: pointers, sizes, integer handles, no torch or C++ types, no
 * exceptions.  Every entry point returns QSV_OK (0) or a negative QSV_E_* code;
 * qsv_last_error() returns a thread-local message for the last failure.
 *
 * The reference (arXiv 2509.04955, /root/reference/proj) ships no kernels, so
 * each entry point below names the SPEC/PAPER operation or reference header it
 * replaces (SPEC = /root/reference/SPEC.md, PAPER = /root/reference/PAPER.md,
 * ref = /root/reference/proj).  Caller-side bindings (C++ qsim, Python ctypes)
 * are shown in INTEGRATION.md.
 *
 * Data layout (ref types.hpp:9-19): an amplitude is two fp64
 * values (re, im) interleaved, 16 B; qubit k is bit k of the index.  A rank
 * owns 2^l consecutive amplitudes whose top m = n - l index bits equal the
 * rank id.  Device buffers are 256-B aligned.
 *
 * Threading: calls on one context are stream-ordered and asynchronous until
 * qsv_sync(); a context must not be used from two host threads at once
 * (SPEC:132, :424).
 */
#ifndef QSV_H
#define QSV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ------------------------------------------------------- */
#define QSV_OK 0
#define QSV_E_ARG (-1)     /* parameter error            */
#define QSV_E_CUDA (-2)    /* CUDA runtime failure                           */
#define QSV_E_NCCL (-3)    /* collective failure            */
#define QSV_E_NOMEM (-4)   /* device allocation failed                       */
#define QSV_E_STATE (-5)   /* call not valid in the current state            */
#define QSV_E_NODEV (-6)   /* no CUDA device / wrong architecture            */

/* ---- limits ------------------------------------------------------------ */
#define QSV_MAX_QUBITS 62   /* total qubits n (uint64 index arithmetic)      */
#define QSV_MAX_DENSE_K 5   /* largest dense fused block (32x32 complex)     */
#define QSV_MAX_DIAG_K 8    /* largest tabulated diagonal block              */
#define QSV_MAX_HIGH 8      /* high (non-contiguous) tile qubits per pass    */
#define QSV_MAX_TILE_K 12   /* tile qubits per pass (12 only with specialised kernels) */
#define QSV_NCCL_ID_BYTES 128

typedef struct qsv_ctx qsv_ctx;         /* one GPU + its stream(s) + comm   */
typedef struct qsv_state qsv_state;     /* one rank's 2^l-amplitude shard   */
typedef struct qsv_program qsv_program; /* a planned circuit, device-resident */

/* ---- devices and contexts ---------------------------------------------- */

/* Number of visible CUDA devices. */
int qsv_device_count(int* n);

/* Fills `out` (QSV_NCCL_ID_BYTES) with a fresh NCCL unique id; rank 0 calls
 * this and broadcasts the bytes to the other ranks out of band. */
int qsv_comm_unique_id(void* out);

/* Creates a context on `device` for rank `rank` of `nranks` (a power of two).
 * For nranks > 1 `comm_id` is the QSV_NCCL_ID_BYTES id from rank 0 and the
 * call is collective over all ranks (ncclCommInitRank).  Replaces the
 * Transport construction of SPEC:399-407 (in_process / local_sockets). */
int qsv_ctx_create(int device, int rank, int nranks, const void* comm_id, qsv_ctx** out);
int qsv_ctx_destroy(qsv_ctx* ctx);
/* The cudaStream_t (as void*) all work of this context is ordered on. */
void* qsv_ctx_stream(qsv_ctx* ctx);
/* Bytes of swap staging buffers currently held by the context (BBOP memory
 * accounting: per rank <= (2^l + B*2^b)*16 B + overhead). */
int qsv_ctx_staging_bytes(qsv_ctx* ctx, size_t* out);
/* Blocks until all work queued on the context has finished. */
int qsv_sync(qsv_ctx* ctx);
/* Collective failure semantics ("any collective error aborts all ranks
 * with diagnostics").  qsv_ctx_abort tears down the context's communicator
 * (ncclCommAbort) from any thread, so every rank blocked in a swap or barrier
 * returns QSV_E_NCCL instead of waiting for a peer that will never arrive; the
 * reason is reported by every later call on the context.  Waits on multi-rank
 * contexts also poll ncclCommGetAsyncError and abort after QSV_COLL_TIMEOUT_S
 * seconds (default 900).  qsv_ctx_aborted reports whether the context was aborted. */
int qsv_ctx_abort(qsv_ctx* ctx, const char* reason);
int qsv_ctx_aborted(qsv_ctx* ctx, int* out);

/* PipelineTrace: with tracing on, every pass launch (per
 * region when a swap is overlapped), P2P swap kernel, NCCL send/recv chunk and
 * staging copy-back is bracketed by CUDA events on the stream it runs on.
 * qsv_trace_enable(ctx, 1) clears the trace and sets the time origin (an event on the
 * compute stream; CUDA-graph replay is bypassed while tracing); qsv_trace_read waits
 * for the context's streams and writes up to cap records (*n = records available). */
#define QSV_TRACE_PASS 0       /* pass kernel (chunk = region, -1 = whole shard)   */
#define QSV_TRACE_SWAP 1       /* P2P swap kernel (chunk = region, -1 = whole)    */
#define QSV_TRACE_SENDRECV 2   /* NCCL send/recv of one chunk (+ its send gather)   */
#define QSV_TRACE_COPYBACK 3   /* copy-back / scatter of one received chunk       */
#define QSV_TRACE_BARRIER 4    /* pairwise barrier of a P2P swap                  */
typedef struct qsv_trace_rec {
    int32_t kind, step, chunk, stream; /* stream: 0 compute, 1 comm, 2 copy */
    double start_ms, end_ms;           /* relative to qsv_trace_enable     */
} qsv_trace_rec;
int qsv_trace_enable(qsv_ctx* ctx, int on);
/* Instrumented device memory of a context (the SPEC:397 / :573 memory audit): every
 * device allocation the library makes for the context (state shard, swap staging,
 * program blobs, collective and reduction scratch) is counted; qsv_ctx_mem reports the
 * live bytes and the high-water mark since creation or the last reset.  An optional hook
 * sees every allocation (+bytes) and release (-bytes) on the calling thread; kind:
 * 0 state, 1 swap staging, 2 program, 3 scratch. */
typedef void (*qsv_alloc_hook)(void* user, int64_t delta_bytes, int kind);
int qsv_ctx_set_alloc_hook(qsv_ctx* ctx, qsv_alloc_hook hook, void* user);
int qsv_ctx_mem(qsv_ctx* ctx, size_t* live_bytes, size_t* peak_bytes);
int qsv_ctx_mem_reset_peak(qsv_ctx* ctx);
int qsv_trace_read(qsv_ctx* ctx, qsv_trace_rec* out, int cap, int* n);
/* Thread-local description of the last failure on this thread. */
const char* qsv_last_error(void);

/* ---- state shards (replaces StateVector) -------------------- */

/* Allocates this rank's shard of 2^n_local amplitudes (uninitialised).
 * *bytes receives the size so the C++ caller can report it to
 * qsim::memtrack::on_alloc (ref memtrack.hpp:20). */
int qsv_state_alloc(qsv_ctx* ctx, int n_local, qsv_state** out, size_t* bytes);
int qsv_state_free(qsv_state* st);
/* Sets the distributed state to the basis state |global_index> (SPEC:392:
 * "|0...0> constructed"); ranks not owning the index get all zeros.  Every rank passes the same
 * index.  The state remembers it until the next run, upload, apply, swap or device_ptr call: a
 * multi-rank program that then starts with qubit swaps relabels the index instead of moving the
 * shard (the ranks agree on it with one 16-byte all-reduce; QSV_BASIS_SWAPS=0 disables it). */
int qsv_state_set_basis(qsv_state* st, uint64_t global_index);
/* Host <-> device copies of `count` amplitudes starting at local `offset`,
 * interleaved (re, im) doubles.  Stream-ordered; host memory should be pinned
 * (qsv_host_alloc) for asynchronous overlap. */
int qsv_state_upload(qsv_state* st, const double* host, uint64_t offset, uint64_t count);
int qsv_state_download(qsv_state* st, double* host, uint64_t offset, uint64_t count);
/* Stream-ordered download (no host sync): the copy completes in order with the
 * context stream; call qsv_sync before reading `host`.  With pinned host memory it
 * overlaps other contexts' work (used for pipelined end-to-end streaming). */
int qsv_state_download_async(qsv_state* st, double* host, uint64_t offset, uint64_t count);
/* Stream events between contexts (e.g. staggering several engines' copies and runs):
 * `stream` is a handle from qsv_ctx_stream / qsim_engine_stream. */
int qsv_event_create(void** ev);
int qsv_event_destroy(void* ev);
int qsv_event_record(void* ev, void* stream);
int qsv_stream_wait_event(void* stream, void* ev);
/* Raw device pointer of the shard (double2*), for interop/tests.  Fetch it after
 * qsv_state_set_basis if you write through it (the call forgets the basis-state mark). */
int qsv_state_device_ptr(qsv_state* st, void** ptr);
/* Pinned host buffers for the upload/download paths. */
int qsv_host_alloc(size_t bytes, void** ptr);
int qsv_host_free(void* ptr);

/* ---- single fused gate (replaces apply_single_naive/grouped, apply_controlled,
 *      apply_multi — SPEC:55-93, PAPER Alg. 1-4 :176-257) --------------------
 * Applies the dense 2^k x 2^k row-major complex matrix `mat` (2*4^k doubles,
 * re/im interleaved) on `targets` (LOCAL physical qubits; targets[p] is bit p
 * of the matrix index) to every amplitude group whose index has all
 * bits of `ctrl_mask` set (GLOBAL index bits: controls may be rank qubits;
 * SPEC:362 CONTROL_REMOTE).  1 <= k <= QSV_MAX_DENSE_K.  One HBM pass. */
int qsv_apply_fused(qsv_state* st, int k, const int* targets, uint64_t ctrl_mask,
                    const double* mat);

/* ---- planned programs (SMGP multi-block passes + BBOP swaps) ------------- */

/* Op kinds inside a pass. */
#define QSV_OP_DENSE 0  /* dense 2^k matrix on k LOCAL targets (+ controls)          */
#define QSV_OP_DIAG 1   /* diagonal of 2^k entries on k qubits (any, incl. global) */
#define QSV_OP_XPERM 2  /* Pauli-X permutation on one LOCAL target (+ controls)    */
#define QSV_OP_RBLOCK 3 /* register block: a list of primitives (U1/U2/CX/DIAG16) on
                         * k = 3 or 4 LOCAL tile qubits qubits[0..k), applied to each
                         * 2^k-amplitude group in registers (one SMEM round trip for
                         * the whole list) */
#define QSV_OP_PHASEPROD 4 /* separable phase product: for amplitudes with all ctrl_mask
                         * bits set, multiply by pool[mat_off] * prod over FACTOR
                         * primitives (qubit q set) of pool[prim.mat_off]; qubits
                         * anywhere (tile, out-of-tile, rank).  CP/CZ chains (QFT).   */

#define QSV_OP_PARPHASE 5 /* parity phase: amplitudes with all ctrl_mask bits set are
                         * multiplied by pool[mat_off + parity(index & qmask)]; qmask
                         * may hold any qubits (a CX ladder . RZ . ladder^-1 string). */

/* Primitive kinds (RBLOCK: a, b index qubits[0..3] of the op; PHASEPROD: a is a
 * physical qubit).  Matrices are complex, row-major, in the pool. */
#define QSV_PRIM_U1 0      /* 2x2 on block qubit a                                   */
#define QSV_PRIM_U2 1      /* 4x4 on block qubits (a, b), a < b, a = low matrix bit   */
#define QSV_PRIM_CX 2      /* X on block qubit b controlled by block qubit a          */
#define QSV_PRIM_DIAG16 3  /* 2^k-entry diagonal over the k block qubits (bit i = qubits[i]) */
#define QSV_PRIM_FACTOR 4  /* PHASEPROD factor: multiply when physical qubit a is 1    */
#define QSV_PRIM_U1R 5     /* 2x2 with real entries (H, RY): 4 DFMA per amplitude     */
#define QSV_PRIM_U1I 6     /* 2x2 real diagonal, imaginary off-diagonal (RX)          */

typedef struct qsv_prim_desc {
    int32_t kind;
    int32_t a, b;
    int32_t pad;
    int64_t mat_off;       /* complex offset into the pool                          */
} qsv_prim_desc;

typedef struct qsv_op_desc {
    int32_t kind;          /* QSV_OP_*                                              */
    int32_t k;             /* number of entries in qubits[]                         */
    int32_t qubits[QSV_MAX_DIAG_K]; /* physical qubits; qubits[p] = bit p of the matrix index */
    uint64_t ctrl_mask;    /* physical GLOBAL index bits that must all be 1         */
    int64_t mat_off;       /* offset (complex entries) into the program's pool       */
    int32_t prim_begin;    /* RBLOCK / PHASEPROD: primitives [prim_begin, +nprim)    */
    int32_t nprim;
    uint64_t qmask;        /* PARPHASE: physical qubits whose parity selects the phase */
} qsv_op_desc;

/* Step kinds of a program. */
#define QSV_STEP_PASS 0  /* one HBM round trip applying ops[op_begin, +op_count)   */
#define QSV_STEP_SWAP 1  /* qubit swap global<->local (collective over ranks)      */

typedef struct qsv_step_desc {
    int32_t kind;
    /* PASS: tile of 2^tile_k amplitudes = the low run [0, tile_k - nhigh) plus the
     * high tile qubits the ops need (local, ascending, above the low run).     */
    int32_t tile_k;
    int32_t nhigh;
    int32_t high[QSV_MAX_HIGH];
    int32_t op_begin, op_count;
    /* PASS, optional relabel applied after the ops: tile bit i (0..L-1 = the low run,
     * L.. = high[] in order) moves to tile bit relabel[i], i.e. the physical qubit
     * slots of the tile are permuted in place (a bijection on the tile's bits). */
    int32_t has_relabel;
    int32_t relabel[16];
    /* SWAP: exchange physical global qubit g with local qubit v, moving 2^chunk_log2
     * amplitudes per message with nbuf staging buffers (BBOP b and B). */
    int32_t swap_global, swap_local, chunk_log2, nbuf;
} qsv_step_desc;

/* Uploads a program for states of `n_total` qubits split as 2^n_local per rank.
 * `pool` holds 2*pool_len doubles (complex entries) referenced by ops.  The
 * library validates every op (targets local and inside the pass tile, k
 * limits, pool bounds) and compiles it to the tile layout of its pass. */
int qsv_program_create(qsv_ctx* ctx, int n_total, int n_local,
                       const qsv_step_desc* steps, int nsteps,
                       const qsv_op_desc* ops, int nops,
                       const qsv_prim_desc* prims, int nprims,
                       const double* pool, size_t pool_len, qsv_program** out);
int qsv_program_free(qsv_program* prog);
/* Specialises the program's passes: each distinct pass structure is emitted
 * as straight-line CUDA (constants for the tile enumeration, slot positions and
 * primitive sequence) and compiled by NVRTC for sm_100a; at most max_kernels
 * distinct kernels (other passes keep the interpreter kernel).  Synchronous;
 * *seconds receives the compile time (0 for disk-cache hits).  Returns
 * QSV_E_STATE when NVRTC is unavailable (the program stays valid). */
int qsv_program_jit(qsv_program* prog, int max_kernels, double* seconds);
/* The same specialisation on a background host thread: runs of the program use the interpreter
 * kernel until the compile has finished, and the first run after that switches to the
 * specialised kernels (results agree to rounding, not bitwise, across the switch).  Single-rank
 * contexts only; on a multi-rank context this compiles synchronously, so that every rank
 * switches at the same run. */
int qsv_program_jit_async(qsv_program* prog, int max_kernels);
/* Adopts a finished background compile (block != 0: waits for it).  *done = 1 once no compile
 * is pending; *seconds = compile + load time of the adopted kernels.  Returns the compile's error
 * if it failed (the program keeps the interpreter). */
int qsv_program_jit_wait(qsv_program* prog, int block, int* done, double* seconds);
int qsv_program_jit_info(qsv_program* prog, int* kernels, int* steps_jitted);
/* Host-only dry run of qsv_program_create's validation and tile compilation
 * (no device needed): returns QSV_OK iff the program would be accepted for
 * rank `rank`.  Used by CPU tests of the planner. */
int qsv_program_validate(int n_total, int n_local, int rank, const qsv_step_desc* steps, int nsteps,
                         const qsv_op_desc* ops, int nops, const qsv_prim_desc* prims, int nprims,
                         const double* pool, size_t pool_len);
/* Host-only: qsv_program_validate plus an NVRTC compile (sm_100a cubin) of the
 * program's distinct specialised pass kernels, as qsv_program_jit would build them;
 * *kernels receives their number.  No device needed (CPU tests of the JIT path). */
int qsv_program_jit_check(int n_total, int n_local, int rank, const qsv_step_desc* steps, int nsteps,
                          const qsv_op_desc* ops, int nops, const qsv_prim_desc* prims, int nprims,
                          const double* pool, size_t pool_len, int max_kernels, int* kernels);
/* Enqueues every step of the program on the context stream (a CUDA graph when
 * the program has no collective steps).  Replaces run_local and
 * run_distributed's dispatch loop. */
int qsv_program_run(qsv_state* st, qsv_program* prog);
/* Runs the program once with CUDA events around every step; ms_out[nsteps]
 * receives per-step device times (profiling aid, not used on the timed path). */
int qsv_program_profile(qsv_state* st, qsv_program* prog, float* ms_out);
/* Times `iters` back-to-back runs of the program with CUDA events recorded on
 * the context stream (synchronous); *ms receives the total device time.  When
 * basis >= 0 every run starts with qsv_state_set_basis(basis) inside the
 * timed region (a full simulation step from a basis state). */
int qsv_program_time(qsv_state* st, qsv_program* prog, int iters, int64_t basis, float* ms);
/* Static description of step `i`: algorithmic bytes moved through HBM and
 * DP flops it performs per launch (the roofline numerators). */
int qsv_program_step_cost(qsv_program* prog, int i, double* hbm_bytes, double* flops,
                          double* nvlink_bytes);

/* ---- qubit swap (BBOP, Eq. 5) ------
 * Collective over all ranks: exchanges physical global qubit g (>= n_local)
 * with local qubit v.  Each rank sends the half of its shard whose bit v differs
 * from its own bit (g - n_local) to peer r ^ (1 << (g - n_local)), in chunks of
 * 2^chunk_log2 amplitudes through nbuf staging buffers, and receives the peer's
 * half into the vacated slots. */
int qsv_swap(qsv_state* st, int g, int v, int chunk_log2, int nbuf);

/* ---- reductions and checks --------------------------------------------- */
/* Sum |a|^2 over this rank's shard (pairwise tree in fp64). */
int qsv_norm_sq(qsv_state* st, double* out);
/* max |psi[offset+i] - host_ref[i]| over i < count (host_ref interleaved). */
int qsv_max_abs_diff(qsv_state* st, const double* host_ref, uint64_t offset, uint64_t count,
                     double* out);
/* max |psi[y] - e^{2 pi i x y / 2^n} / 2^{n/2}| over this shard: the analytic
 * QFT of the basis state |x> (used where the CPU cannot hold the
 * state).  `n_total` = n. */
int qsv_check_qft_basis(qsv_state* st, int n_total, uint64_t x, double* out);
/* Bitwise digest (xor/sum of the 64-bit words) of the shard, for cross-P
 * bitwise-equality checks. */
int qsv_state_digest(qsv_state* st, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* QSV_H */
