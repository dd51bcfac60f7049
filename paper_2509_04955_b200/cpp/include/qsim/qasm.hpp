// OpenQASM 2.0 subset ingestion and export.
// Reconstructed from the reference CMake source list (proj/CMakeLists.txt:21,
// src/qasm.cpp — absent from the reference tree) and the SPEC [OP] signatures.
//
// Grammar (one statement per `;`, `//` comments, UTF-8/ASCII text):
//
//   program   := [ "OPENQASM" real ";" ] { include | qreg | gate | barrier }
//   include   := "include" "\"qelib1.inc\"" ";"          (any other file is rejected)
//   qreg      := "qreg" id "[" int "]" ";"                (exactly one, before any gate)
//   gate      := mnemonic [ "(" expr { "," expr } ")" ] arg { "," arg } ";"
//   barrier   := "barrier" arg { "," arg } ";"
//   arg       := id [ "[" int "]" ]                       (a bare register broadcasts
//                                                          single-qubit gates / barriers)
//   expr      := real | int | "pi" | fn "(" expr ")" | "(" expr ")" | -expr | expr op expr
//                with op in + - * / ^ and fn in sin cos tan exp ln sqrt
//
//   mnemonic ∈ {h x y z s sdg t tdg rx ry rz u1 p cx cz cp cu1 swap}
//   swap a,b  → cx(a→b), cx(b→a), cx(a→b)
//   barrier   → a fusion-fence pseudo-gate
//
// `measure`, `creg`, `if`, `reset`, `gate`/`opaque` definitions and includes other than
// qelib1.inc are rejected.  Every error is a QasmError carrying the 1-based
// line and column of the offending token; the parser never crashes on arbitrary bytes
// (fuzzed in tests/test_qasm.py).
//
// Matrix export: gates outside the mnemonic set (fused "FUSED" blocks, CU,
// user unitaries) are written as a comment directive other QASM tools ignore,
//
//   // qsv-unitary "LABEL" (re00, im00, re01, ...) q[t0], q[t1] | q[c0];
//
// which parse_qasm reads back to a Gate with a bit-identical matrix (%.17g round trip).
#pragma once

#include "qsim/circuit.hpp"

#include <stdexcept>
#include <string>
#include <string_view>

namespace qsim {

// Parameter error with a location (std::invalid_argument like every reference parameter
// error, ref gate.cpp:24).  what() = "qasm:<line>:<col>: <message>".
class QasmError : public std::invalid_argument {
  public:
    QasmError(int line, int column, const std::string& message);
    int line() const { return line_; }
    int column() const { return column_; }

  private:
    int line_;
    int column_;
};

// SPEC:161-170.  `source` becomes Circuit::source (provenance).
Circuit parse_qasm(std::string_view text, std::string source = "qasm");
// Reads a file and parses it; source = the path.
Circuit parse_qasm_file(const std::string& path);

struct QasmEmitOptions {
    // Export gates outside the mnemonic set as `// qsv-unitary` directives; without it
    // such a gate is an error.
    bool matrix_export = false;
};

// header + `qreg q[n];` + one statement per gate, angles as %.17g so that
// parse_qasm(emit_qasm(c)) reproduces every matrix bit for bit.
std::string emit_qasm(const Circuit& c, const QasmEmitOptions& opts = {});

} // namespace qsim
