// Definitions for qsim/circuit.hpp and qsim/statevector.hpp.
#include "qsim/circuit.hpp"
#include "qsim/memtrack.hpp"
#include "qsim/statevector.hpp"

#include <stdexcept>

namespace qsim {

namespace {
void check_gate(const Gate& g, int n) {
    for (int q : g.qubits())
        if (q < 0 || q >= n)
            throw std::invalid_argument("circuit: gate '" + g.label() + "' touches qubit " +
                                        std::to_string(q) + " outside [0, " + std::to_string(n) + ")");
}
} // namespace

Circuit::Circuit(int n_qubits, std::string src) : n(n_qubits), source(std::move(src)) {
    if (n < 1)
        throw std::invalid_argument("circuit: qubit count must be >= 1");
}

Circuit::Circuit(int n_qubits, std::vector<Gate> gs, std::string src)
    : n(n_qubits), gates(std::move(gs)), source(std::move(src)) {
    validate();
}

void Circuit::add(Gate g) {
    check_gate(g, n);
    gates.push_back(std::move(g));
}

void Circuit::validate() const {
    if (n < 1)
        throw std::invalid_argument("circuit: qubit count must be >= 1");
    for (const Gate& g : gates)
        check_gate(g, n);
}

std::size_t Circuit::gate_count() const {
    std::size_t c = 0;
    for (const Gate& g : gates)
        c += g.is_fence() ? 0 : 1;
    return c;
}

// ------------------------------------------------------------------ StateVector
StateVector::StateVector(int n) : n_(n) {
    if (n < 1 || n > 40)
        throw std::invalid_argument("StateVector: n must be in [1, 40]");
    amps_.assign(index_bit(n), Amp{0.0, 0.0});
    amps_[0] = Amp{1.0, 0.0};
    memtrack::on_alloc(amps_.size() * sizeof(Amp));
}

StateVector::StateVector(const StateVector& o) : n_(o.n_), amps_(o.amps_) {
    memtrack::on_alloc(amps_.size() * sizeof(Amp));
}

StateVector& StateVector::operator=(const StateVector& o) {
    if (this != &o) {
        memtrack::on_free(amps_.size() * sizeof(Amp));
        n_ = o.n_;
        amps_ = o.amps_;
        memtrack::on_alloc(amps_.size() * sizeof(Amp));
    }
    return *this;
}

StateVector::StateVector(StateVector&& o) noexcept : n_(o.n_), amps_(std::move(o.amps_)) {}

StateVector& StateVector::operator=(StateVector&& o) noexcept {
    if (this != &o) {
        memtrack::on_free(amps_.size() * sizeof(Amp));
        n_ = o.n_;
        amps_ = std::move(o.amps_);
    }
    return *this;
}

StateVector::~StateVector() { memtrack::on_free(amps_.size() * sizeof(Amp)); }

double StateVector::norm_sq() const {
    double s = 0.0, c = 0.0;
    for (const Amp& a : amps_) {
        const double y = std::norm(a) - c;
        const double t = s + y;
        c = (t - s) - y;
        s = t;
    }
    return s;
}

void StateVector::set_basis(Index index) {
    if (index >= size())
        throw std::invalid_argument("StateVector::set_basis: index out of range");
    std::fill(amps_.begin(), amps_.end(), Amp{0.0, 0.0});
    amps_[index] = Amp{1.0, 0.0};
}

} // namespace qsim
