// Circuit — qubit count plus a program-ordered gate list.
// Reconstructed from the reference CMake source list (proj/CMakeLists.txt:19,
// src/circuit.cpp) and SPEC Appendix-B-style signatures; not present in the
// reference tree.
#pragma once

#include "qsim/gate.hpp"

#include <string>
#include <vector>

namespace qsim {

struct Circuit {
    int n = 1;                 // qubit count, >= 1
    std::vector<Gate> gates;   // execution order
    std::string source;        // provenance: generator spec or file path

    Circuit() = default;
    // Throws std::invalid_argument for n < 1 ("n = 0 rejected").
    explicit Circuit(int n_qubits, std::string src = {});
    Circuit(int n_qubits, std::vector<Gate> gs, std::string src);

    // Appends after checking every qubit index is < n.
    void add(Gate g);
    // Re-checks the whole gate list (throws std::invalid_argument).
    void validate() const;
    // Gates excluding barriers (the gates/s numerator).
    std::size_t gate_count() const;
};

} // namespace qsim
