// SMGP — staggered multi-gate parallelism.
// The Latin-rectangle schedule and group planning are kept as the SPEC
// defines them; execution on the B200 applies a whole group in ONE HBM pass
// (every member applied in program order to each SMEM tile), which is bitwise
// equal to sequential application.
#pragma once

#include "qsim/circuit.hpp"
#include "qsim/dag.hpp"
#include "qsim/statevector.hpp"

#include <utility>
#include <vector>

namespace qsim {

struct StaggerGroup {
    std::vector<int> gates;                   // circuit gate indices, pairwise qubit-disjoint
    int s = 0;                                // segment bits, S = 2^s
    std::vector<std::vector<int>> schedule;   // schedule[g][tau] = segment of gate g at step tau
};

// Segment of gate g at step tau: (g + tau) mod S (Table 3).
std::vector<std::vector<int>> stagger_schedule(int G, int S);

// Maximal groups of <= S pairwise qubit-disjoint, mutually independent gates
// whose qubits are all < local_qubits - log2(S); everything
// else is returned as residual gate indices.
std::pair<std::vector<StaggerGroup>, std::vector<int>> plan_groups(const Circuit& c, const DepGraph& dag,
                                                                   int S, int local_qubits = -1);

// Applies the group's gates to `state` in one GPU pass.
// `workers` is accepted for API compatibility.
void execute_staggered(StateVector& state, const Circuit& c, const StaggerGroup& group, int workers = 1);

} // namespace qsim
