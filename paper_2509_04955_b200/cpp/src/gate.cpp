// Definitions for qsim/gate.hpp.  Behaviour follows the reference
// (proj/src/gate.cpp) — same matrices, same validation and exception types —
// but the code is an independent implementation.
#include "qsim/gate.hpp"

#include <cmath>
#include <numbers>
#include <stdexcept>
#include <unordered_map>

namespace qsim {

namespace {

// Entry-wise unitarity test of M^dagger M against the identity, tolerance 1e-10
// per entry (ref gate.cpp:11-27).  G = M^H M is accumulated row by row of M so
// the inner loop streams contiguous memory; only the upper triangle is formed
// because G is Hermitian (|G_cr| = |G_rc|).
bool is_unitary(int arity, const std::vector<Amp>& m) {
    constexpr double kTol = 1e-10;
    const std::size_t d = std::size_t{1} << arity;
    std::vector<Amp> g(d * d, Amp{0.0, 0.0});
    for (std::size_t k = 0; k < d; ++k) {
        const Amp* row = &m[k * d];
        for (std::size_t r = 0; r < d; ++r) {
            const Amp a = std::conj(row[r]);
            Amp* gr = &g[r * d];
            for (std::size_t c = r; c < d; ++c)
                gr[c] += a * row[c];
        }
    }
    for (std::size_t r = 0; r < d; ++r)
        for (std::size_t c = r; c < d; ++c) {
            const Amp want = (r == c) ? Amp{1.0, 0.0} : Amp{0.0, 0.0};
            if (std::abs(g[r * d + c] - want) > kTol)
                return false;
        }
    return true;
}

void require_distinct_nonnegative(const std::vector<int>& qs, std::vector<int>& seen,
                                  const char* what) {
    for (int q : qs) {
        if (q < 0)
            throw std::invalid_argument(std::string(what) + ": negative qubit index");
        for (int s : seen)
            if (s == q)
                throw std::invalid_argument(std::string(what) + ": duplicate qubit " +
                                            std::to_string(q));
        seen.push_back(q);
    }
}

} // namespace

GateMatrix::GateMatrix(int arity, std::vector<Amp> entries)
    : arity_(arity), entries_(std::move(entries)) {
    if (arity_ < 1)
        throw std::invalid_argument("GateMatrix: arity must be at least 1");
    const Index d = dim();
    if (entries_.size() != d * d)
        throw std::invalid_argument("GateMatrix: expected " + std::to_string(d * d) +
                                    " entries, got " + std::to_string(entries_.size()));
    if (!is_unitary(arity_, entries_))
        throw std::invalid_argument("GateMatrix: matrix is not unitary within 1e-10");
}

GateMatrix GateMatrix::identity(int arity) {
    if (arity < 1)
        throw std::invalid_argument("GateMatrix: arity must be at least 1");
    const Index d = index_bit(arity);
    std::vector<Amp> e(d * d);
    for (Index i = 0; i < d; ++i)
        e[i * (d + 1)] = Amp{1.0, 0.0};
    return GateMatrix(arity, std::move(e));
}

Gate Gate::unitary(GateMatrix matrix, std::vector<int> targets, std::vector<int> controls,
                   std::string label, std::vector<double> params) {
    if (targets.size() != static_cast<std::size_t>(matrix.arity()))
        throw std::invalid_argument("Gate: number of targets differs from matrix arity");
    std::vector<int> seen;
    seen.reserve(targets.size() + controls.size());
    require_distinct_nonnegative(targets, seen, "Gate targets");
    require_distinct_nonnegative(controls, seen, "Gate controls");
    Gate g;
    g.matrix_.emplace(std::move(matrix));
    g.targets_ = std::move(targets);
    g.controls_ = std::move(controls);
    g.label_ = std::move(label);
    g.params_ = std::move(params);
    return g;
}

Gate Gate::barrier(std::vector<int> qubits) {
    std::vector<int> seen;
    require_distinct_nonnegative(qubits, seen, "barrier");
    Gate g;
    g.targets_ = std::move(qubits);
    g.label_ = "barrier";
    return g;
}

std::vector<int> Gate::qubits() const {
    std::vector<int> all;
    all.reserve(targets_.size() + controls_.size());
    all.insert(all.end(), targets_.begin(), targets_.end());
    all.insert(all.end(), controls_.begin(), controls_.end());
    return all;
}

int Gate::max_qubit() const {
    int hi = -1;
    for (int q : targets_) hi = q > hi ? q : hi;
    for (int q : controls_) hi = q > hi ? q : hi;
    return hi;
}

namespace gates {

namespace {

// Matrix entries use the same formulas as the reference so the matrices are
// bit-identical (checked against the compiled reference in tests/test_oracle.py):
// 1/sqrt(2) is computed as 1.0/std::sqrt(2.0) and phases via std::polar.
const double kRsqrt2 = 1.0 / std::sqrt(2.0);
constexpr Amp kJ{0.0, 1.0};

Gate one_qubit(int q, std::vector<Amp> m, const char* label, std::vector<double> ps = {}) {
    return Gate::unitary(GateMatrix(1, std::move(m)), {q}, {}, label, std::move(ps));
}

Gate ctrl_one_qubit(int c, int t, std::vector<Amp> m, const char* label,
                    std::vector<double> ps = {}) {
    return Gate::unitary(GateMatrix(1, std::move(m)), {t}, {c}, label, std::move(ps));
}

std::vector<Amp> phase_diag(double lambda) { return {1.0, 0.0, 0.0, std::polar(1.0, lambda)}; }

} // namespace

Gate h(int q) { return one_qubit(q, {kRsqrt2, kRsqrt2, kRsqrt2, -kRsqrt2}, "h"); }
Gate x(int q) { return one_qubit(q, {0.0, 1.0, 1.0, 0.0}, "x"); }
Gate y(int q) { return one_qubit(q, {0.0, -kJ, kJ, 0.0}, "y"); }
Gate z(int q) { return one_qubit(q, {1.0, 0.0, 0.0, -1.0}, "z"); }
Gate s(int q) { return one_qubit(q, {1.0, 0.0, 0.0, kJ}, "s"); }
Gate sdg(int q) { return one_qubit(q, {1.0, 0.0, 0.0, -kJ}, "sdg"); }
Gate t(int q) { return one_qubit(q, phase_diag(std::numbers::pi / 4), "t"); }
Gate tdg(int q) { return one_qubit(q, phase_diag(-std::numbers::pi / 4), "tdg"); }

Gate rx(int q, double theta) {
    const double c = std::cos(theta / 2), sn = std::sin(theta / 2);
    const Amp off = -kJ * sn;
    return one_qubit(q, {c, off, off, c}, "rx", {theta});
}

Gate ry(int q, double theta) {
    const double c = std::cos(theta / 2), sn = std::sin(theta / 2);
    return one_qubit(q, {c, -sn, sn, c}, "ry", {theta});
}

Gate rz(int q, double theta) {
    return one_qubit(q, {std::polar(1.0, -theta / 2), 0.0, 0.0, std::polar(1.0, theta / 2)},
                     "rz", {theta});
}

Gate u1(int q, double lambda) { return one_qubit(q, phase_diag(lambda), "u1", {lambda}); }
Gate p(int q, double lambda) { return one_qubit(q, phase_diag(lambda), "p", {lambda}); }

Gate cx(int control, int target) { return ctrl_one_qubit(control, target, {0.0, 1.0, 1.0, 0.0}, "cx"); }
Gate cz(int control, int target) { return ctrl_one_qubit(control, target, {1.0, 0.0, 0.0, -1.0}, "cz"); }

Gate cp(int control, int target, double lambda) {
    return ctrl_one_qubit(control, target, phase_diag(lambda), "cp", {lambda});
}

Gate cu1(int control, int target, double lambda) {
    return ctrl_one_qubit(control, target, phase_diag(lambda), "cu1", {lambda});
}

Gate cu(int control, int target, GateMatrix u, std::string label) {
    if (u.arity() != 1)
        throw std::invalid_argument("cu: the controlled matrix must be single-qubit");
    return Gate::unitary(std::move(u), {target}, {control}, std::move(label));
}

Gate from_mnemonic(const std::string& mnemonic, const std::vector<double>& params,
                   const std::vector<int>& qubits) {
    enum Kind { H, X, Y, Z, S, SDG, T, TDG, RX, RY, RZ, U1, P, CX, CZ, CP, CU1 };
    struct Sig { Kind kind; std::size_t nparams, nqubits; };
    static const std::unordered_map<std::string, Sig> table = {
        {"h", {H, 0, 1}},   {"x", {X, 0, 1}},     {"y", {Y, 0, 1}},   {"z", {Z, 0, 1}},
        {"s", {S, 0, 1}},   {"sdg", {SDG, 0, 1}}, {"t", {T, 0, 1}},   {"tdg", {TDG, 0, 1}},
        {"rx", {RX, 1, 1}}, {"ry", {RY, 1, 1}},   {"rz", {RZ, 1, 1}}, {"u1", {U1, 1, 1}},
        {"p", {P, 1, 1}},   {"cx", {CX, 0, 2}},   {"cz", {CZ, 0, 2}}, {"cp", {CP, 1, 2}},
        {"cu1", {CU1, 1, 2}},
    };
    const auto it = table.find(mnemonic);
    if (it == table.end())
        throw std::invalid_argument("unknown gate mnemonic '" + mnemonic + "'");
    const Sig sig = it->second;
    if (params.size() != sig.nparams)
        throw std::invalid_argument("gate '" + mnemonic + "' takes " +
                                    std::to_string(sig.nparams) + " parameter(s), got " +
                                    std::to_string(params.size()));
    if (qubits.size() != sig.nqubits)
        throw std::invalid_argument("gate '" + mnemonic + "' takes " +
                                    std::to_string(sig.nqubits) + " qubit(s), got " +
                                    std::to_string(qubits.size()));
    const int a = qubits[0];
    const int b = sig.nqubits > 1 ? qubits[1] : -1;
    const double th = sig.nparams ? params[0] : 0.0;
    switch (sig.kind) {
    case H: return h(a);
    case X: return x(a);
    case Y: return y(a);
    case Z: return z(a);
    case S: return s(a);
    case SDG: return sdg(a);
    case T: return t(a);
    case TDG: return tdg(a);
    case RX: return rx(a, th);
    case RY: return ry(a, th);
    case RZ: return rz(a, th);
    case U1: return u1(a, th);
    case P: return p(a, th);
    case CX: return cx(a, b);
    case CZ: return cz(a, b);
    case CP: return cp(a, b, th);
    case CU1: return cu1(a, b, th);
    }
    throw std::invalid_argument("unreachable mnemonic");
}

} // namespace gates

} // namespace qsim
