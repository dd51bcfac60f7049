/*
 * qsim_c.h — plain-C facade of the qsim host library (libqsim.so) for callers
 * that cannot use the C++ API (Python ctypes in tests/ and bench.py, other
 * FFIs).  It exposes the reference-level objects — circuits, generators, the
 * DAGC/SMGP planner and the device engine — with the same error convention as
 * include/qsv.h: 0 on success, negative QSV_E_* codes on failure, message in
 * qsim_last_error() (thread-local).  C++ exceptions never cross this boundary.
 *
 * Reference interfaces mirrored (SPEC = /root/reference/SPEC.md):
 *   qsim_circuit_*   Circuit / Gate / from_mnemonic (ref gate.hpp:33-92)
 *   qsim_circuit_generate  gen_qft/gen_qaoa/gen_hea + random / uccsd
 *   qsim_run_local_host    run_local on host amplitudes
 *   qsim_engine_*          run_local / run_distributed with a device-resident state
 */
#ifndef QSIM_C_H
#define QSIM_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qsim_circuit qsim_circuit;
typedef struct qsim_engine qsim_engine;

/* Flat gate record (layout shared with the test oracle's orc_gate). */
typedef struct qsim_gate_rec {
    int32_t arity;          /* 0 = barrier                                     */
    int32_t nctrl;
    int32_t targets[8];
    int32_t controls[8];
    int64_t mat_off;        /* complex offset of the 4^arity matrix in the pool */
} qsim_gate_rec;

typedef struct qsim_plan_opts {
    int32_t tile_k;           /* tile qubits per pass (<= 11)                   */
    int32_t min_low;          /* contiguous low qubits in every tile             */
    int32_t fuse_k;           /* largest fused dense block (<= 5)               */
    int32_t fusion;           /* DAGC on (1) / off (0)                          */
    int32_t multi_op_passes;  /* SMGP multi-block passes on (1) / off (0)       */
    int32_t chunk_log2;       /* BBOP batch 2^b amplitudes                      */
    int32_t nbuf;             /* BBOP buffers B                                 */
    int32_t register_blocks;  /* group native gates on <= 4 qubits (RBLOCK)     */
    double pass_budget;       /* DP cost units per amplitude per pass           */
    int32_t rblock_k;         /* register-block width: 3 or 4 qubits            */
    int32_t jit;              /* NVRTC-specialised pass kernels (1), compiled in the background with
                                 interpreted runs until they load (2), or the interpreter (0) */
    int32_t relabel;          /* tile-qubit relabel at pass ends: 0 off, 1 auto, 2 always */
    double max_sweeps;        /* SMEM sweeps of the tile per pass                */
    int32_t list_schedule;    /* single rank: also try a DAG list schedule       */
    int32_t jit_max_kernels;  /* distinct specialised pass kernels compiled at most */
    int32_t logical_swaps;    /* also plan SWAP gates (CX triples) as relabellings  */
} qsim_plan_opts;

typedef struct qsim_plan_stats {
    int64_t gates_in, ops_lowered, ops_fused, ops_final, passes, swaps;
    double cost_units;
    int32_t max_dense_k, n, n_local, nsteps;
} qsim_plan_stats;

const char* qsim_last_error(void);
void qsim_default_opts(qsim_plan_opts* out);

/* ---- circuits ---- */
int qsim_circuit_generate(const char* spec, qsim_circuit** out);
int qsim_circuit_new(int n, qsim_circuit** out);
int qsim_circuit_add(qsim_circuit* c, const char* mnemonic, const double* params, int nparams,
                     const int* qubits, int nqubits);
int qsim_circuit_add_unitary(qsim_circuit* c, int k, const int* targets, int nctrl, const int* controls,
                             const double* mat, const char* label);
int qsim_circuit_add_barrier(qsim_circuit* c, int nqubits, const int* qubits);
/* n, number of records (gates incl. barriers), pool length in complex entries */
int qsim_circuit_info(const qsim_circuit* c, int* n, int64_t* nrecs, int64_t* pool_len);
int qsim_circuit_export(const qsim_circuit* c, qsim_gate_rec* recs, double* pool);
/* Gates [begin, end) as a new circuit (used for bounded CPU-baseline samples). */
int qsim_circuit_slice(const qsim_circuit* c, int64_t begin, int64_t end, qsim_circuit** out);
/* The fused op list the planner would execute, as a circuit of FUSED gates. */
int qsim_circuit_fused(const qsim_circuit* c, const qsim_plan_opts* opts, qsim_circuit** out);
/* Plans for n_local local qubits (-1 = all) and validates the program with the
 * device library's host-side compiler; fills stats.  No GPU needed. */
int qsim_circuit_plan(const qsim_circuit* c, const qsim_plan_opts* opts, int n_local, int rank,
                      qsim_plan_stats* stats);
void qsim_circuit_free(qsim_circuit* c);
/* OpenQASM 2.0 subset (qsim/qasm.hpp).  parse: text of len bytes (need not be
 * NUL-terminated); on a syntax/semantic error returns QSV_E_ARG with the 1-based location in
 * *line / *col (either may be NULL) and the message in qsim_last_error().
 * emit: writes at most cap bytes (NUL-terminated when it fits) and the full length without
 * the NUL to *needed; call with cap = 0 to size the buffer.  matrix_export != 0 writes gates
 * outside the mnemonic set as `// qsv-unitary` directives (otherwise QSV_E_ARG). */
int qsim_circuit_parse_qasm(const char* text, int64_t len, qsim_circuit** out, int* line, int* col);
int qsim_circuit_emit_qasm(const qsim_circuit* c, int matrix_export, char* buf, int64_t cap, int64_t* needed);
/* Exports the device program of the plan (include/qsv.h structures).  Call
 * with NULL arrays to get the counts, then again with buffers of that size:
 * on input the counts are the capacities of the non-NULL arrays; the plan is
 * rebuilt, and if it no longer fits (its options read the environment) the call
 * writes the needed sizes back and returns QSV_E_ARG without copying. */
int qsim_plan_export(const qsim_circuit* c, const qsim_plan_opts* opts, int n_local, int* nsteps, int* nops,
                     int* nprims, int64_t* pool_len, void* steps, void* ops, void* prims, double* pool);

/* ---- engine: one rank's GPU, a planned circuit and its device state ---- */
int qsim_engine_create(const qsim_circuit* c, const qsim_plan_opts* opts, int device, int rank,
                       int nranks, const void* comm_id, qsim_engine** out);
void qsim_engine_free(qsim_engine* e);
int qsim_engine_stats(qsim_engine* e, qsim_plan_stats* out);
void* qsim_engine_stream(qsim_engine* e);      /* cudaStream_t */
void* qsim_engine_qsv_state(qsim_engine* e);   /* qsv_state*   */
void* qsim_engine_qsv_program(qsim_engine* e); /* qsv_program* */
void* qsim_engine_qsv_ctx(qsim_engine* e);     /* qsv_ctx* (trace, abort)  */
int qsim_engine_set_basis(qsim_engine* e, uint64_t global_index);
int qsim_engine_upload(qsim_engine* e, const double* amps, uint64_t offset, uint64_t count);
int qsim_engine_download(qsim_engine* e, double* amps, uint64_t offset, uint64_t count);
/* Stream-ordered (returns before the copy completes; qsim_engine_sync waits). */
int qsim_engine_download_async(qsim_engine* e, double* amps, uint64_t offset, uint64_t count);
int qsim_engine_run(qsim_engine* e);           /* enqueue (asynchronous) */
int qsim_engine_sync(qsim_engine* e);
int qsim_engine_time(qsim_engine* e, int iters, int64_t basis, float* ms);
int qsim_engine_norm_sq(qsim_engine* e, double* out);
int qsim_engine_max_abs_diff(qsim_engine* e, const double* ref, uint64_t offset, uint64_t count,
                             double* out);
int qsim_engine_check_qft(qsim_engine* e, uint64_t x, double* out);
int qsim_engine_digest(qsim_engine* e, uint64_t* out);
int qsim_engine_nsteps(qsim_engine* e);
int qsim_engine_step_info(qsim_engine* e, int i, int* kind, int* nops, double* hbm_bytes, double* flops,
                          double* nvl_bytes);
int qsim_engine_profile(qsim_engine* e, float* ms_per_step);
/* JIT statistics: distinct specialised kernels and compile seconds (0 = cache hits). */
int qsim_engine_jit_info(qsim_engine* e, int* kernels, double* seconds);
/* Waits for the engine's background compile (jit = 2) and adopts its kernels. */
int qsim_engine_jit_wait(qsim_engine* e);

/* ---- SPEC-level passes (reference semantics) ---- */
typedef struct qsim_fusion_stats {
    int64_t gates_before, gates_after, merges_same_qubit, merges_cu, merges_kronecker, passes;
    double compression_ratio, cost_before, cost_after;
} qsim_fusion_stats;

typedef struct qsim_dist_report {
    int32_t ranks, reserved;
    int64_t swaps;
    double seconds;
    int64_t peak_bytes[64];
} qsim_dist_report;

/* build_dag: writes up to cap (i, j) edge pairs; returns the edge count (< 0: error). */
int64_t qsim_dag_edges(const qsim_circuit* c, int32_t* pairs, int64_t cap);
/* gate_cost of gate i for an n-qubit state. */
int qsim_gate_cost(const qsim_circuit* c, int64_t i, int n, double* out);
/* contract(c, cap) -> FUSED circuit + stats. */
int qsim_contract(const qsim_circuit* c, int cap, qsim_circuit** out, qsim_fusion_stats* stats);
/* plan_groups: group_of[i] = group id of gate i or -1 (residual); returns #groups. */
int qsim_plan_groups(const qsim_circuit* c, int S, int local_qubits, int32_t* group_of);
/* stagger_schedule(G, S): table[g*S + tau]. */
int qsim_stagger_schedule(int G, int S, int32_t* table);
/* execute_staggered on host amplitudes for the gates whose group id == group. */
int qsim_execute_staggered(const qsim_circuit* c, int S, int local_qubits, int group, double* amps);
/* classify_gate (0 LOCAL, 1 TARGET_REMOTE, 2 CONTROL_REMOTE, 3 BOTH_REMOTE). */
int qsim_classify_gate(const qsim_circuit* c, int64_t i, int m, int* out);
int qsim_peer_rank(int r, int t, int l, int* out);
/* run_distributed over 2^m GPUs (devices[r], NULL = 0..2^m-1) from |0...0>;
 * gathers all 2^n amplitudes into amps (host). */
int qsim_run_distributed(const qsim_circuit* c, int m, int b, int buffers, const int* devices,
                         const qsim_plan_opts* opts, double* amps, qsim_dist_report* report);
/* The same run without a gather: rank r writes its shard to
 * <dir>/shard_r<r>_of_<R>.bin (complex128 LE, global indices [r 2^l, (r+1) 2^l)) and
 * <dir>/manifest.json is written.  qsim_run_distributed refuses states above the
 * single-host cap QSV_GATHER_CAP_GIB (default 64) with QSV_E_ARG. */
int qsim_run_distributed_files(const qsim_circuit* c, int m, int b, int buffers, const int* devices,
                               const qsim_plan_opts* opts, const char* dir, qsim_dist_report* report);

/* ---- memtrack (ref memtrack.hpp:12-26) scripted session, for parity tests ----
 * ops[2*i] = kind (0 enable, 1 register_thread, 2 set_phase, 3 on_alloc,
 * 4 on_free, 5 reset, 6 disable), ops[2*i+1] = argument; writes
 * peak_bytes(rank, phase) for rank < nranks, phase < 2. */
void qsim_memtrack_script(const long long* ops, int nops, int nranks, unsigned long long* peaks);

/* ---- reference-facing single call: run_local on host amplitudes ---------
 * Uploads `amps` (2^n interleaved complex, ideally pinned), runs the planned
 * circuit on device 0, downloads the result into `amps`. */
int qsim_run_local_host(const qsim_circuit* c, const qsim_plan_opts* opts, double* amps);

#ifdef __cplusplus
}
#endif

#endif
