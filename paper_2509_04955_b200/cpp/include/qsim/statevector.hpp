// StateVector — host owner of 2^n complex128 amplitudes.
// Reconstructed (reference src/statevector.cpp is absent, proj/CMakeLists.txt:17).
// The B200 path keeps the authoritative state in HBM (qsim::DeviceState in
// device.hpp); this host type is the reference-facing input/output buffer of
// run_local and the kernels API.  Allocation is reported to memtrack.
#pragma once

#include "qsim/types.hpp"

#include <vector>

namespace qsim {

class StateVector {
  public:
    // |0...0> of n qubits.  Throws std::invalid_argument for n < 1
    // or n > 40.
    explicit StateVector(int n);
    StateVector(const StateVector& other);
    StateVector& operator=(const StateVector& other);
    StateVector(StateVector&& other) noexcept;
    StateVector& operator=(StateVector&& other) noexcept;
    ~StateVector();

    int n() const { return n_; }
    Index size() const { return index_bit(n_); }
    Amp* data() { return amps_.data(); }
    const Amp* data() const { return amps_.data(); }
    Amp& operator[](Index i) { return amps_[i]; }
    const Amp& operator[](Index i) const { return amps_[i]; }

    // Sum of |a_i|^2 (compensated summation).
    double norm_sq() const;
    // Sets |index>.
    void set_basis(Index index);

  private:
    int n_;
    std::vector<Amp> amps_;
};

} // namespace qsim
