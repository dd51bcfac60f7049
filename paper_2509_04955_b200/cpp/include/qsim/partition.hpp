// Global/local qubit partitioning (Eq. 5).
#pragma once

#include "qsim/gate.hpp"

namespace qsim {

// n = m + l: the top m qubits select the rank (2^m ranks), the low l are local;
// batches of 2^b amplitudes move through `buffers` staging buffers (BBOP).
struct PartitionPlan {
    int n = 1, m = 0, l = 1, b = 0, buffers = 2;
    PartitionPlan() = default;
    // Throws std::invalid_argument unless 0 <= m < n and 0 <= b < l, buffers >= 1.
    PartitionPlan(int n_qubits, int m_global, int b_batch, int nbuffers = 2);
    int ranks() const { return 1 << m; }
};

enum class Locality { LOCAL, TARGET_REMOTE, CONTROL_REMOTE, BOTH_REMOTE };

// LOCAL: every qubit < l; TARGET_REMOTE: a target >= l with all controls local;
// CONTROL_REMOTE: targets local, some control >= l (acts only on ranks whose
// control bits are set, no communication); BOTH_REMOTE: both.
Locality classify_gate(const Gate& g, const PartitionPlan& plan);

// r XOR (1 << (t - l)) (Eq. 5); throws for t < l.
int peer_rank(int r, int t, int l);

} // namespace qsim
