/*
 * oracle.h — CPU restatement of the reference simulator's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker the CUDA path is
 * compared against (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline
 * leg and `bench.py --impl reference`).  The product library (libqsv.so,
 * libqsim.so) never links, loads or calls it.
 *
 * The reference ships no kernel sources (kernels.cpp, statevector.cpp,
 * dense_oracle.cpp and worker_pool.cpp are listed in proj/CMakeLists.txt:16-21
 * but absent), so these functions restate the published algorithms:
 *   PAPER = /root/reference/PAPER.md (Alg. 1 :176-190, Alg. 2 :192-210,
 *           Alg. 3 :221-236, Alg. 4 :238-257, Eq. 3 :124-148, Eq. 4 :160-169)
 *   SPEC  = /root/reference/SPEC.md  (sv-core :24-140)
 * Parity pinning: there are no reference tests or golden
 * vectors; the oracle is pinned by (1) the SPEC known answers, (2) the analytic
 * QFT of basis states, (3) an independent explicit-matrix dense oracle and (4)
 * gate matrices bit-compared with the reference's own compiled gate.cpp
 * (oracle/_ref, built by oracle/build_ref.sh).
 */
#ifndef QSV_ORACLE_H
#define QSV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One gate in flat form (same layout as qsim_gate_rec in include/qsim_c.h).
 * arity == 0 is a barrier (no-op).  The matrix is 4^arity complex entries,
 * row-major, at pool[2*mat_off ...] (re, im interleaved); targets[p] is bit p
 * of the matrix index; every control must be 1. */
typedef struct orc_gate {
    int32_t arity;
    int32_t nctrl;
    int32_t targets[8];
    int32_t controls[8];
    int64_t mat_off;
} orc_gate;

/* Alg. 1: visit every index, update pairs with bit t clear. */
int orc_apply_single_naive(int n, double* amps, int t, const double* u);
/* Alg. 3: groups of 2^{t+1}, first half traversed; threads
 * split the group range. Bitwise equal to Alg. 1. */
int orc_apply_single_grouped(int n, double* amps, int t, const double* u, int threads);
/* Alg. 4 with the c > t role swap: only pairs with
 * bit c set, exactly 2^{n-2} pairs. */
int orc_apply_controlled(int n, double* amps, int c, int t, const double* u, int threads);
/* apply_multi: 2^k-group gather, M x group, scatter, for groups
 * with all controls 1. */
int orc_apply_multi(int n, double* amps, int k, const int* targets, int nctrl, const int* controls,
                    const double* m, int threads);
/* run_local: gates in program order, dispatching as the
 * reference does (1q -> Alg. 3, 1q+1 control -> Alg. 4, else apply_multi). */
int orc_run_local(int n, const orc_gate* gates, int64_t ngates, const double* pool, double* amps,
                  int threads);
/* The same run_local as a cache-blocked schedule: maximal runs of consecutive
 * gates whose qubits fit in block_bits bits are applied block by block
 * (gather 2^block_bits amplitudes, the run's gates in program order, scatter).
 * Bitwise equal to orc_run_local; used to check full-size states in tests. */
int orc_run_local_blocked(int n, const orc_gate* gates, int64_t ngates, const double* pool, double* amps,
                          int threads, int block_bits);
/* dense_oracle: every gate embedded as an explicit 2^n x 2^n
 * matrix (row by row) and multiplied into the state; n <= 12. */
int orc_dense_oracle(int n, const orc_gate* gates, int64_t ngates, const double* pool,
                     const double* in, double* out);
/* Workload generators restated for the reference arm (oracle/gen.cpp): the
 * spec's gates as mnemonic instructions (code = ORC_*, q0 = first qubit /
 * control, q1 = target of a two-qubit gate or -1, params = angle).  Returns the
 * gate count (fills the arrays when cap >= count), -1 on a bad spec. */
enum { ORC_H = 0, ORC_RX = 1, ORC_RY = 2, ORC_RZ = 3, ORC_CX = 4, ORC_CP = 5 };
int64_t orc_generate(const char* spec, int* n, int32_t* codes, int32_t* q0, int32_t* q1, double* params,
                     int64_t cap);
/* |index> into a 2^n buffer, zero-filled by the worker pool (parallel first touch). */
int orc_fill_basis(int n, double* amps, uint64_t index, int threads);
/* Hardware threads the oracle uses by default. */
int orc_default_threads(void);

#ifdef __cplusplus
}
#endif

#endif
