// The B200 circuit planner: the host pass that turns a Circuit into the
// device program uploaded through include/qsv.h.
//
//   lower()     gate -> op: DENSE (general), DIAG (diagonal, incl. CP/CZ/RZ/S/T;
//               controlled diagonals with a single non-unit entry become a
//               "phase on all-ones pattern"), XPERM (X / CX).
//   fuse_ops()  DAGC re-targeted to the fp64/HBM roofline (PAPER:391-483,
//               SPEC:232-331): greedy merge of each op into the latest op on
//               its qubits when the merged block stays <= fuse_k qubits and the
//               per-amplitude DP cost does not grow (same-support runs,
//               CU consolidation, Kronecker products are all special cases).
//               Barriers are fences.
//   pack()      SMGP re-designed as multi-block passes: ops are
//               packed, in program order, into passes whose dense targets fit
//               one 2^K-amplitude tile (>= 2^5 contiguous low amplitudes) and
//               whose DP cost per amplitude stays under the roofline budget, so
//               each pass is one HBM round trip.
//   partition   (multi-GPU) the top log2(P) physical qubits are global
//               (PAPER:280); a dense target on a global qubit
//               inserts a BBOP qubit swap with a local victim (swap.cu).
#pragma once

#include "qsim/circuit.hpp"
#include "qsv.h"

#include <string>
#include <vector>

namespace qsim {

// Swap: a SWAP gate (a CX triple) executed as a relabelling of its two qubits' physical
// slots (no data movement; the final layout is restored at the end of the plan).
enum class OpKind { Dense, Diag, XPerm, PhaseProd, ParPhase, RBlock, Fence, Swap };

// RBLOCK primitive (block-local qubit indices into Op::qubits).
struct Prim {
    int kind = QSV_PRIM_U1;     // QSV_PRIM_U1 / U2 / CX / DIAG16
    int a = 0, b = 0;
    std::vector<Amp> data;      // U1: 4, U2: 16, DIAG16: 16 entries
};

// One lowered op on LOGICAL qubits.
struct Op {
    OpKind kind = OpKind::Dense;
    std::vector<int> qubits;    // Dense/XPerm: targets; Diag: diagonal qubits (qubits[p] = bit p);
                                // RBlock: block qubits (<= 4)
    std::vector<int> controls;  // all must be 1
    std::vector<Amp> data;      // Dense: 4^k entries row-major; Diag: 2^k entries;
                                // PhaseProd: data[0] = constant factor;
                                // ParPhase: {phase if parity(qubits) even, phase if odd}
    std::vector<std::pair<int, Amp>> factors;  // PhaseProd: multiply by f when qubit is 1
    std::vector<Prim> prims;    // RBlock
    int width = 0;              // RBlock: register-block width (3 or 4 slots)
    int first_gate = -1;        // provenance (gate index range)
    int last_gate = -1;
    int ngates = 0;             // source gates merged into this op
};

struct PlanOptions {
    int tile_k = 11;          // tile qubits per pass (<= 11)
    int min_low = 5;          // contiguous low run: 2^5 amplitudes = 512-B DRAM runs
    int fuse_k = 2;           // largest dense block fusion may create (<= QSV_MAX_DENSE_K)
    bool register_blocks = true;  // group native gates on <= rblock_k qubits into RBLOCK ops
    int rblock_k = 4;         // register-block width: 3 (8 amplitudes/thread) or 4 (16)
    bool fusion = true;       // DAGC on/off (BASELINE configs[1]: "contraction on vs off")
    bool multi_op_passes = true;  // SMGP on/off: off = one op per pass
    double pass_budget = 120; // DP cost units (DFMA) per amplitude allowed in one pass
    double max_sweeps = 8;    // SMEM sweeps of the tile per pass (diagonal epilogues count 1/2)
    bool list_schedule = true;  // single rank: also try a DAG list schedule (ready op that fits first)
    int n_local = -1;         // local qubits per rank (-1: all, single GPU)
    int chunk_log2 = 26;      // BBOP batch: 2^b amplitudes per swap message; 1 GiB NCCL messages reach ~530 GB/s on NVLink 5 vs ~275 GB/s at 2^22
    int nbuf = 2;             // BBOP buffers B (default 2)
    bool jit = true;          // NVRTC-specialised pass kernels (falls back to the interpreter kernel)
    bool jit_async = false;   // compile them on a background thread; runs interpret until they load
    int jit_max_kernels = 8192; // distinct pass structures compiled at most (the rest interpreted)
    int logical_swaps = 0;    // SWAP gates (CX triples) as free relabellings: 0 off, 1 when the
                              // time model prefers it, 2 always (tests)
    int relabel = 1;          // tile-qubit relabelling at pass ends: 0 off, 1 auto (kept when it
                              // saves passes), 2 always (tests)
};

struct PlanStats {
    std::size_t gates_in = 0;      // gates excluding barriers (gates/s numerator)
    std::size_t ops_lowered = 0;
    std::size_t ops_fused = 0;     // ops after fusion
    std::size_t ops_final = 0;     // ops after register blocking (what the kernels run)
    std::size_t passes = 0;
    std::size_t swaps = 0;
    double cost_units = 0;         // sum of op costs (DP units / amplitude)
    int max_dense_k = 0;
};

struct Plan {
    int n = 0;
    int n_local = 0;
    std::vector<qsv_step_desc> steps;
    std::vector<qsv_op_desc> ops;
    std::vector<qsv_prim_desc> prims;
    std::vector<double> pool;          // complex entries, re/im interleaved
    std::vector<Op> fused;             // fused ops (logical qubits), for inspection/tests
    PlanStats stats;
};

// Classification helpers.
std::vector<Op> lower(const Circuit& c);
// CX(c,t) . P . CX(c,t) with P a parity phase whose mask holds t equals the
// parity phase on mask ^ {c}: collapses CX-ladder / RZ / reverse-ladder Pauli
// strings (UCCSD) into single diagonal ops that need no tile residency.
std::vector<Op> reduce_parity(const std::vector<Op>& ops);
std::vector<Op> fuse_ops(const std::vector<Op>& ops, const PlanOptions& opt);
// Groups ops acting on <= 4 qubits into register blocks (RBLOCK); a block holds
// at most max_high qubits at or above min_low (it must fit one pass tile).
std::vector<Op> form_blocks(const std::vector<Op>& ops, int min_low = 5, int max_high = 5, int width = 3);
// Relative DP cost per amplitude of one op (the packing / fusion currency).
double op_cost(const Op& op);
// Builds the full plan (lower -> fuse -> partition/swaps -> pack).
Plan make_plan(const Circuit& c, const PlanOptions& opt);
// Re-expresses fused ops as a Circuit of FUSED gates (for oracle checks of the
// fusion, SPEC:312 semantic preservation).
Circuit ops_to_circuit(int n, const std::vector<Op>& ops);

} // namespace qsim
