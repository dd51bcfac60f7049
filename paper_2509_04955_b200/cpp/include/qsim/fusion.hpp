// DAGC as the SPEC defines it: cost model,
// the three fusion rules and greedy contraction to a fixed point, with stats.
// This is the reference-semantics DAGC (FUSED gates, compression ratio).  The
// B200 execution path uses the roofline-retargeted planner in planner.hpp,
// which applies the same rules plus register blocking.
#pragma once

#include "qsim/circuit.hpp"
#include "qsim/dag.hpp"

#include <tuple>
#include <vector>

namespace qsim {

// (2*4^k + 2^k) * 2^{n-k}, halved per control: 10*2^{n-1} (k=1), 36*2^{n-2}
// (k=2) — the paper's counting of mults + adds + copies.
double gate_cost(const Gate& g, int n);

// M_b * M_a on the same target set.
Gate fuse_same_qubit(const Gate& a, const Gate& b);
// M_2 (x) M_1 on the union of two disjoint uncontrolled target sets; the lower
// first target is the least-significant fused bit (Eq. 7).
Gate fuse_kronecker(const Gate& a, const Gate& b);
// CU with U = U_b * U_a for identical controls and targets.
Gate fuse_cu(const Gate& a, const Gate& b);

enum class FusionRule { SameQubit = 0, CU = 1, Kronecker = 2 };

struct FusionStep {
    std::vector<int> gates;  // constituent indices (into the input of that pass)
    FusionRule rule;
    int pass = 0;
};

struct FusionPlan {
    std::vector<FusionStep> steps;
};

struct FusionStats {
    std::size_t gates_before = 0;
    std::size_t gates_after = 0;
    double compression_ratio = 0.0;  // (before - after) / before (Fig. 14)
    std::size_t merges_same_qubit = 0, merges_cu = 0, merges_kronecker = 0;
    std::size_t passes = 0;
    double cost_before = 0.0, cost_after = 0.0;
};

// Greedy contraction in program order, rules tried same-qubit -> CU ->
// Kronecker, a merge accepted iff the total gate_cost decreases; repeated until
// a full pass makes no merge.  Barriers are never
// crossed; Kronecker fusion across a control qubit is forbidden.
std::tuple<Circuit, FusionPlan, FusionStats> contract(const Circuit& c, int cap = 2);

} // namespace qsim
