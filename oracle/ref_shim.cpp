// Thin C shim over the REFERENCE's own gate.cpp / memtrack.cpp (compiled from
// /root/reference/proj/src by oracle/build_ref.sh into oracle/_ref/).  Used only
// by tests/golden/make_golden.py to pin gate matrices and memtrack semantics
// against the reference itself.  TEST INFRASTRUCTURE ONLY.
#include "qsim/gate.hpp"
#include "qsim/memtrack.hpp"

#include <cstring>
#include <exception>
#include <string>
#include <vector>

extern "C" {

// Builds gates::from_mnemonic(name, params, qubits) with the reference code and
// writes arity, targets, controls and the 4^arity matrix entries (re, im).
// Returns 0, or -1 if the reference threw (error text in err, 256 bytes).
int ref_gate(const char* name, const double* params, int np, const int* qubits, int nq, int* arity,
             int* targets, int* ntargets, int* controls, int* nctrl, double* mat, char* err) {
    try {
        std::vector<double> ps(params, params + np);
        std::vector<int> qs(qubits, qubits + nq);
        qsim::Gate g = qsim::gates::from_mnemonic(name, ps, qs);
        *arity = g.arity();
        *ntargets = static_cast<int>(g.targets().size());
        for (int i = 0; i < *ntargets; ++i) targets[i] = g.targets()[i];
        *nctrl = static_cast<int>(g.controls().size());
        for (int i = 0; i < *nctrl; ++i) controls[i] = g.controls()[i];
        const auto& e = g.matrix().entries();
        for (std::size_t i = 0; i < e.size(); ++i) {
            mat[2 * i] = e[i].real();
            mat[2 * i + 1] = e[i].imag();
        }
        return 0;
    } catch (const std::exception& ex) {
        std::strncpy(err, ex.what(), 255);
        err[255] = 0;
        return -1;
    }
}

// GateMatrix unitarity check of the reference: 1 = accepted, 0 = rejected.
int ref_matrix_accepts(int arity, const double* mat) {
    try {
        const std::size_t d = std::size_t{1} << arity;
        std::vector<qsim::Amp> e(d * d);
        for (std::size_t i = 0; i < d * d; ++i) e[i] = qsim::Amp(mat[2 * i], mat[2 * i + 1]);
        qsim::GateMatrix m(arity, std::move(e));
        return 1;
    } catch (...) {
        return 0;
    }
}

// Scripted memtrack session: ops[i] = {kind, arg} with kind 0 enable(arg),
// 1 register_thread(arg), 2 set_phase(arg), 3 on_alloc(arg), 4 on_free(arg),
// 5 reset, 6 disable.  Writes peak_bytes(rank, phase) for rank < nranks, phase < 2.
void ref_memtrack_script(const long long* ops, int nops, int nranks, unsigned long long* peaks) {
    using namespace qsim::memtrack;
    for (int i = 0; i < nops; ++i) {
        const long long k = ops[2 * i], a = ops[2 * i + 1];
        switch (k) {
        case 0: enable(static_cast<int>(a)); break;
        case 1: register_thread(static_cast<int>(a)); break;
        case 2: set_phase(static_cast<Phase>(a)); break;
        case 3: on_alloc(static_cast<std::size_t>(a)); break;
        case 4: on_free(static_cast<std::size_t>(a)); break;
        case 5: reset(); break;
        case 6: disable(); break;
        default: break;
        }
    }
    for (int r = 0; r < nranks; ++r)
        for (int p = 0; p < 2; ++p)
            peaks[2 * r + p] = peak_bytes(r, static_cast<Phase>(p));
    unregister_thread();
}

} // extern "C"
