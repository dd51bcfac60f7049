// Dependency DAG over a circuit's gates.
// Reconstructed: the reference's src/dag.cpp is absent (proj/CMakeLists.txt:24).
#pragma once

#include "qsim/circuit.hpp"

#include <utility>
#include <vector>

namespace qsim {

struct DepGraph {
    int n_gates = 0;
    std::vector<std::vector<int>> succ;    // i -> j edges (i < j)
    std::vector<std::vector<int>> pred;
    std::vector<std::vector<int>> qubits;  // Q_i = targets U controls (barrier: its qubits)

    bool has_edge(int i, int j) const;
    std::vector<std::pair<int, int>> edges() const;
    // True when j is reachable from i (i < j).
    bool has_path(int i, int j) const;
};

// Edge i -> j iff Q_i and Q_j intersect and i is the latest gate before j on a
// shared qubit wire ("transitive-reduction form" per wire).  Barrier
// pseudo-gates are nodes on their qubits, so they fence every gate on them.
DepGraph build_dag(const Circuit& c);

} // namespace qsim
