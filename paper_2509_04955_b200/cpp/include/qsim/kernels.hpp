// The reference's sv-core operations (absent reference file
// src/kernels.cpp, proj/CMakeLists.txt:18) on a host StateVector, executed on
// the B200 through the C-ABI.  Same names, argument meaning and errors:
// std::invalid_argument for parameter errors.  Each call
// uploads the state, runs one fused-pass program and downloads the result, so
// these are drop-in but not the fast path — Engine/DeviceState keep the state
// resident in HBM across a whole circuit.
#pragma once

#include "qsim/circuit.hpp"
#include "qsim/statevector.hpp"

namespace qsim {

// Alg. 1 — single-qubit gate, no controls.
void apply_single_naive(StateVector& state, const Gate& gate);
// Alg. 3 — same contract, grouped traversal.
void apply_single_grouped(StateVector& state, const Gate& gate);
// Alg. 4 — single-qubit gate with one control.
void apply_controlled(StateVector& state, const Gate& gate);
// apply_multi: k-qubit gate with optional controls; throws if k > cap.
void apply_multi(StateVector& state, const Gate& gate, int cap = 5);
// run_local: the whole circuit, DAGC + multi-block passes on the
// GPU.  `threads` is accepted for API compatibility; the GPU ignores it (the
// result is independent of it, as the SPEC requires).
void run_local(const Circuit& circuit, StateVector& state, int threads = 1);

} // namespace qsim
