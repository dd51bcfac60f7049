// Seeded workload generators plus the two families the
// north-star configs need that the reference does not define: random
// H/RX/RZ + CNOT-brick circuits and UCCSD-style Pauli-exponential ladders
// (BASELINE.json configs[1], [2]).
#pragma once

#include "qsim/circuit.hpp"

#include <cstdint>
#include <string>

namespace qsim {

// H(j) then cp(pi/2^{j-k}) for k = j-1..0, for j = n-1..0, then the
// floor(n/2) swap layer q <-> n-1-q lowered to three CX (SPEC:168, :184 with
// the angle typo corrected — SURVEY App. D).  n(n+1)/2 + 3*floor(n/2) gates.
Circuit gen_qft(int n);

// H on all qubits; per layer ZZ blocks CX(i,j) RZ(gamma)(j) CX(i,j) over the
// ring edges (i, i+1 mod n), deduplicated, then RX(beta) on all.
Circuit gen_qaoa(int n, int layers, std::uint64_t seed);

// Per layer (1-based): RX, RY, RZ on every qubit, then CX on even pairs
// (0,1),(2,3).. in odd layers and odd pairs (1,2),(3,4).. in even layers
// (SPEC:201-209).  gen_hea(4,1,s) = 12 rotations + 2 CX.
Circuit gen_hea(int n, int layers, std::uint64_t seed);

// Per layer (0-based) each qubit gets one of H, RX(theta), RZ(theta) chosen
// uniformly, then CX on even pairs in even layers / odd pairs in odd layers
// (SURVEY §8d config 2).
Circuit gen_random(int n, int depth, std::uint64_t seed);

// exp(-i theta/2 P) for random Pauli strings P on contiguous ranges [i, j]
// (length >= 2): basis change (H for X, RX(pi/2) for Y), CX ladder i..j,
// RZ(theta) on j, reverse ladder, undo the basis change.  Strings are added
// until the CX count reaches target_cx.
Circuit gen_uccsd_ladder(int n, std::uint64_t target_cx, std::uint64_t seed);

// "qft:n" | "qaoa:n:p:seed" | "hea:n:layers:seed" | "random:n:depth:seed" |
// "uccsd:n:target_cx:seed" (SPEC:504 generator specs) | "qasm:<path>" (parse_qasm_file,
// qsim/qasm.hpp).
Circuit generate(const std::string& spec);

} // namespace qsim
