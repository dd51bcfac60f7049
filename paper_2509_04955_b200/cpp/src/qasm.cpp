// OpenQASM 2.0 subset parser / emitter.  See qsim/qasm.hpp for the
// grammar.  Host-only ingestion code: it produces the same qsim::Circuit the generators
// produce, so everything downstream (planner, device engine, oracle) is shared.
#include "qsim/qasm.hpp"

#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <numbers>
#include <optional>
#include <sstream>
#include <unordered_map>

namespace qsim {

QasmError::QasmError(int line, int column, const std::string& message)
    : std::invalid_argument("qasm:" + std::to_string(line) + ":" + std::to_string(column) + ": " +
                            message),
      line_(line), column_(column) {}

namespace {

enum class Tok { Ident, Int, Real, String, Sym, Directive, End };

struct Token {
    Tok kind;
    std::string text;
    int line, col;
};

std::string printable(unsigned char ch) {
    if (ch >= 0x20 && ch < 0x7f)
        return std::string("'") + static_cast<char>(ch) + "'";
    char buf[8];
    std::snprintf(buf, sizeof buf, "0x%02x", ch);
    return buf;
}

bool is_ident_start(unsigned char ch) { return std::isalpha(ch) || ch == '_'; }
bool is_ident_char(unsigned char ch) { return std::isalnum(ch) || ch == '_'; }

// Splits the text into tokens; `// qsv-unitary` opens a directive statement, every
// other `//` comment runs to the end of the line.
std::vector<Token> lex(std::string_view s) {
    std::vector<Token> out;
    int line = 1, col = 1;
    std::size_t i = 0;
    auto adv = [&](std::size_t k) {
        for (std::size_t j = 0; j < k && i < s.size(); ++j, ++i) {
            if (s[i] == '\n') {
                ++line;
                col = 1;
            } else {
                ++col;
            }
        }
    };
    while (i < s.size()) {
        const unsigned char ch = static_cast<unsigned char>(s[i]);
        if (ch == ' ' || ch == '\t' || ch == '\r' || ch == '\n' || ch == '\f' || ch == '\v') {
            adv(1);
            continue;
        }
        const int l0 = line, c0 = col;
        if (ch == '/' && i + 1 < s.size() && s[i + 1] == '/') {
            std::size_t j = i + 2;
            while (j < s.size() && (s[j] == ' ' || s[j] == '\t'))
                ++j;
            constexpr std::string_view kDir = "qsv-unitary";
            if (s.substr(j, kDir.size()) == kDir) {
                out.push_back({Tok::Directive, std::string(kDir), l0, c0});
                adv(j + kDir.size() - i);
                continue;
            }
            while (i < s.size() && s[i] != '\n')
                adv(1);
            continue;
        }
        if (is_ident_start(ch)) {
            std::size_t j = i;
            while (j < s.size() && is_ident_char(static_cast<unsigned char>(s[j])))
                ++j;
            out.push_back({Tok::Ident, std::string(s.substr(i, j - i)), l0, c0});
            adv(j - i);
            continue;
        }
        if (std::isdigit(ch) || (ch == '.' && i + 1 < s.size() && std::isdigit(static_cast<unsigned char>(s[i + 1])))) {
            std::size_t j = i;
            bool real = false;
            while (j < s.size() && std::isdigit(static_cast<unsigned char>(s[j])))
                ++j;
            if (j < s.size() && s[j] == '.') {
                real = true;
                ++j;
                while (j < s.size() && std::isdigit(static_cast<unsigned char>(s[j])))
                    ++j;
            }
            if (j < s.size() && (s[j] == 'e' || s[j] == 'E')) {
                std::size_t k = j + 1;
                if (k < s.size() && (s[k] == '+' || s[k] == '-'))
                    ++k;
                if (k < s.size() && std::isdigit(static_cast<unsigned char>(s[k]))) {
                    real = true;
                    j = k;
                    while (j < s.size() && std::isdigit(static_cast<unsigned char>(s[j])))
                        ++j;
                } else {
                    throw QasmError(line, col + static_cast<int>(j - i), "malformed exponent");
                }
            }
            out.push_back({real ? Tok::Real : Tok::Int, std::string(s.substr(i, j - i)), l0, c0});
            adv(j - i);
            continue;
        }
        if (ch == '"') {
            std::size_t j = i + 1;
            while (j < s.size() && s[j] != '"' && s[j] != '\n')
                ++j;
            if (j >= s.size() || s[j] != '"')
                throw QasmError(l0, c0, "unterminated string");
            out.push_back({Tok::String, std::string(s.substr(i + 1, j - i - 1)), l0, c0});
            adv(j + 1 - i);
            continue;
        }
        // {}<>=! are not part of the subset; lexing them lets the parser name the
        // unsupported statement (`measure q -> c`, `if (c==1)`, gate bodies) instead.
        if (std::string_view(";,()[]+-*/^|{}<>=!").find(static_cast<char>(ch)) != std::string_view::npos) {
            out.push_back({Tok::Sym, std::string(1, static_cast<char>(ch)), l0, c0});
            adv(1);
            continue;
        }
        throw QasmError(l0, c0, "unexpected character " + printable(ch));
    }
    out.push_back({Tok::End, "", line, col});
    return out;
}

struct Arg {
    int qubit;  // -1 = whole register
    int line, col;
};

class Parser {
  public:
    Parser(std::vector<Token> toks, std::string source) : t_(std::move(toks)), source_(std::move(source)) {}

    Circuit run() {
        bool first = true;
        while (peek().kind != Tok::End) {
            statement(first);
            first = false;
        }
        if (!circ_)
            throw QasmError(peek().line, peek().col, "missing qreg declaration");
        return std::move(*circ_);
    }

  private:
    std::vector<Token> t_;
    std::size_t p_ = 0;
    std::string source_;
    std::string reg_;
    std::optional<Circuit> circ_;
    int depth_ = 0;

    const Token& peek() const { return t_[p_]; }
    const Token& next() { return t_[p_ < t_.size() - 1 ? p_++ : p_]; }
    [[noreturn]] void fail(const Token& at, const std::string& msg) const { throw QasmError(at.line, at.col, msg); }
    bool is_sym(const Token& t, char c) const { return t.kind == Tok::Sym && t.text[0] == c; }

    const Token& expect_sym(char c) {
        const Token& t = next();
        if (!is_sym(t, c))
            fail(t, std::string("expected '") + c + "', found " + describe(t));
        return t;
    }

    static std::string describe(const Token& t) {
        switch (t.kind) {
        case Tok::End: return "end of input";
        case Tok::String: return "string \"" + t.text + "\"";
        case Tok::Directive: return "qsv-unitary directive";
        default: return "'" + t.text + "'";
        }
    }

    int parse_int(const Token& t, long long max_value) const {
        if (t.kind != Tok::Int)
            fail(t, "expected an integer, found " + describe(t));
        long long v = 0;
        for (char ch : t.text) {
            v = v * 10 + (ch - '0');
            if (v > max_value)
                fail(t, "integer " + t.text + " out of range");
        }
        return static_cast<int>(v);
    }

    // ---- expressions (angles are concrete numbers) -------------------------
    double expr() {
        if (++depth_ > 200)
            fail(peek(), "expression nested too deeply");
        double v = term();
        while (is_sym(peek(), '+') || is_sym(peek(), '-')) {
            const char op = next().text[0];
            const double r = term();
            v = op == '+' ? v + r : v - r;
        }
        --depth_;
        return v;
    }
    double term() {
        double v = power();
        while (is_sym(peek(), '*') || is_sym(peek(), '/')) {
            const Token& opt = next();
            const double r = power();
            if (opt.text[0] == '/' && r == 0.0)
                fail(opt, "division by zero");
            v = opt.text[0] == '*' ? v * r : v / r;
        }
        return v;
    }
    double power() {
        const double b = unary();
        if (is_sym(peek(), '^')) {
            next();
            if (++depth_ > 200)
                fail(peek(), "expression nested too deeply");
            const double e = power();
            --depth_;
            return std::pow(b, e);
        }
        return b;
    }
    double unary() {
        if (is_sym(peek(), '-') || is_sym(peek(), '+')) {
            const char op = next().text[0];
            if (++depth_ > 200)
                fail(peek(), "expression nested too deeply");
            const double v = unary();
            --depth_;
            return op == '-' ? -v : v;
        }
        return primary();
    }
    double primary() {
        const Token& t = next();
        if (t.kind == Tok::Int || t.kind == Tok::Real) {
            double v = 0.0;
            const auto r = std::from_chars(t.text.data(), t.text.data() + t.text.size(), v);
            if (r.ec != std::errc() || !std::isfinite(v))
                fail(t, "number " + t.text + " out of range");
            return v;
        }
        if (t.kind == Tok::Ident) {
            if (t.text == "pi")
                return std::numbers::pi;
            static const std::unordered_map<std::string, double (*)(double)> fns = {
                {"sin", [](double x) { return std::sin(x); }},   {"cos", [](double x) { return std::cos(x); }},
                {"tan", [](double x) { return std::tan(x); }},   {"exp", [](double x) { return std::exp(x); }},
                {"ln", [](double x) { return std::log(x); }},    {"sqrt", [](double x) { return std::sqrt(x); }},
            };
            const auto it = fns.find(t.text);
            if (it == fns.end())
                fail(t, "unknown identifier '" + t.text + "' in expression");
            expect_sym('(');
            const double a = expr();
            expect_sym(')');
            return it->second(a);
        }
        if (is_sym(t, '(')) {
            const double v = expr();
            expect_sym(')');
            return v;
        }
        fail(t, "expected an expression, found " + describe(t));
    }

    std::vector<double> param_list() {
        std::vector<double> ps;
        if (!is_sym(peek(), '('))
            return ps;
        next();
        if (is_sym(peek(), ')')) {
            next();
            return ps;
        }
        for (;;) {
            const Token& at = peek();
            const double v = expr();
            if (!std::isfinite(v))
                fail(at, "angle is not a finite number");
            ps.push_back(v);
            if (is_sym(peek(), ','))
                next();
            else
                break;
        }
        expect_sym(')');
        return ps;
    }

    Arg arg() {
        const Token& id = next();
        if (id.kind != Tok::Ident)
            fail(id, "expected a qubit operand, found " + describe(id));
        if (!circ_)
            fail(id, "qubit operand before the qreg declaration (missing qreg)");
        if (id.text != reg_)
            fail(id, "unknown register '" + id.text + "' (declared: '" + reg_ + "')");
        if (!is_sym(peek(), '['))
            return {-1, id.line, id.col};
        next();
        const Token& it = next();
        const int q = parse_int(it, 1LL << 30);
        if (q >= circ_->n)
            fail(it, "qubit " + reg_ + "[" + std::to_string(q) + "] out of range (qreg size " +
                         std::to_string(circ_->n) + ")");
        expect_sym(']');
        return {q, id.line, id.col};
    }

    std::vector<Arg> arg_list(char stop) {
        std::vector<Arg> as;
        for (;;) {
            as.push_back(arg());
            if (is_sym(peek(), ','))
                next();
            else
                break;
        }
        if (stop != 0 && !is_sym(peek(), stop))
            fail(peek(), std::string("expected ',' or '") + stop + "', found " + describe(peek()));
        return as;
    }

    void add(Gate g, const Token& at) {
        try {
            circ_->add(std::move(g));
        } catch (const QasmError&) {
            throw;
        } catch (const std::invalid_argument& e) {
            fail(at, e.what());
        }
    }

    void require_distinct(const std::vector<Arg>& as) const {
        for (std::size_t i = 0; i < as.size(); ++i)
            for (std::size_t j = 0; j < i; ++j)
                if (as[i].qubit == as[j].qubit)
                    throw QasmError(as[i].line, as[i].col,
                                    "qubit " + reg_ + "[" + std::to_string(as[i].qubit) + "] repeated");
    }

    void statement(bool first) {
        const Token& kw = next();
        if (kw.kind == Tok::Directive)
            return directive(kw);
        if (kw.kind != Tok::Ident)
            fail(kw, "expected a statement, found " + describe(kw));
        const std::string& w = kw.text;
        if (w == "OPENQASM") {
            if (!first)
                fail(kw, "OPENQASM header must be the first statement");
            const Token& v = next();
            if ((v.kind != Tok::Real && v.kind != Tok::Int) || (v.text != "2.0" && v.text != "2"))
                fail(v, "only OPENQASM 2.0 is supported, found " + describe(v));
            expect_sym(';');
            return;
        }
        if (w == "include") {
            const Token& f = next();
            if (f.kind != Tok::String)
                fail(f, "expected a quoted file name, found " + describe(f));
            if (f.text != "qelib1.inc")
                fail(f, "include of '" + f.text + "' is not supported (only qelib1.inc)");
            expect_sym(';');
            return;
        }
        if (w == "qreg") {
            if (circ_)
                fail(kw, "only one qreg declaration is supported");
            const Token& id = next();
            if (id.kind != Tok::Ident)
                fail(id, "expected a register name, found " + describe(id));
            expect_sym('[');
            const Token& nt = next();
            const int n = parse_int(nt, 63);
            if (n < 1)
                fail(nt, "qreg size must be >= 1");
            expect_sym(']');
            expect_sym(';');
            reg_ = id.text;
            circ_.emplace(n, source_);
            return;
        }
        static const char* const kRejected[] = {"measure", "creg", "if", "reset", "gate", "opaque", "U", "CX"};
        for (const char* r : kRejected)
            if (w == r)
                fail(kw, "'" + w + "' is not supported by the simulator's QASM subset");
        if (!circ_)
            fail(kw, "gate '" + w + "' before the qreg declaration (missing qreg)");
        if (w == "barrier") {
            const std::vector<Arg> as = arg_list(';');
            next();
            std::vector<int> qs;
            for (const Arg& a : as) {
                if (a.qubit < 0) {
                    for (int q = 0; q < circ_->n; ++q)
                        qs.push_back(q);
                } else {
                    qs.push_back(a.qubit);
                }
            }
            std::vector<int> uniq;
            for (int q : qs) {
                bool dup = false;
                for (int u : uniq)
                    dup |= u == q;
                if (!dup)
                    uniq.push_back(q);
            }
            add(Gate::barrier(std::move(uniq)), kw);
            return;
        }
        std::vector<double> ps = param_list();
        const std::vector<Arg> as = arg_list(';');
        next();
        const bool broadcast = as.size() == 1 && as[0].qubit < 0;
        for (const Arg& a : as)
            if (a.qubit < 0 && !broadcast)
                throw QasmError(a.line, a.col, "register broadcast is only supported for single-qubit gates");
        if (w == "swap") {
            if (!ps.empty())
                fail(kw, "gate 'swap' takes 0 parameter(s), got " + std::to_string(ps.size()));
            if (as.size() != 2 || broadcast)
                fail(kw, "gate 'swap' takes 2 qubit(s), got " + std::to_string(as.size()));
            require_distinct(as);
            const int a = as[0].qubit, b = as[1].qubit;
            add(gates::cx(a, b), kw);
            add(gates::cx(b, a), kw);
            add(gates::cx(a, b), kw);
            return;
        }
        std::vector<std::vector<int>> apps;
        if (broadcast) {
            for (int q = 0; q < circ_->n; ++q)
                apps.push_back({q});
        } else {
            require_distinct(as);
            std::vector<int> qs;
            for (const Arg& a : as)
                qs.push_back(a.qubit);
            apps.push_back(std::move(qs));
        }
        for (const auto& qs : apps) {
            Gate g = [&]() -> Gate {
                try {
                    return gates::from_mnemonic(w, ps, qs);
                } catch (const std::invalid_argument& e) {
                    fail(kw, e.what());
                }
            }();
            add(std::move(g), kw);
        }
    }

    // // qsv-unitary "LABEL" (v...) targets [| controls] ;
    void directive(const Token& kw) {
        if (!circ_)
            fail(kw, "qsv-unitary directive before the qreg declaration (missing qreg)");
        const Token& lab = next();
        if (lab.kind != Tok::String)
            fail(lab, "expected a quoted label, found " + describe(lab));
        const Token& popen = peek();
        std::vector<double> vals = param_list();
        std::vector<Arg> ts = arg_list(0);
        std::vector<Arg> cs;
        if (is_sym(peek(), '|')) {
            next();
            cs = arg_list(0);
        }
        expect_sym(';');
        std::vector<Arg> all = ts;
        all.insert(all.end(), cs.begin(), cs.end());
        for (const Arg& a : all)
            if (a.qubit < 0)
                throw QasmError(a.line, a.col, "qsv-unitary operands must be indexed qubits");
        require_distinct(all);
        const std::size_t k = ts.size();
        if (k < 1 || k > 10)
            fail(kw, "qsv-unitary needs 1..10 targets");
        const std::size_t dim = std::size_t{1} << k;
        if (vals.size() != 2 * dim * dim)
            fail(popen, "qsv-unitary on " + std::to_string(k) + " target(s) needs " +
                            std::to_string(2 * dim * dim) + " numbers, got " + std::to_string(vals.size()));
        std::vector<Amp> m(dim * dim);
        for (std::size_t i = 0; i < m.size(); ++i)
            m[i] = Amp{vals[2 * i], vals[2 * i + 1]};
        std::vector<int> tq, cq;
        for (const Arg& a : ts)
            tq.push_back(a.qubit);
        for (const Arg& a : cs)
            cq.push_back(a.qubit);
        Gate g = [&]() -> Gate {
            try {
                return Gate::unitary(GateMatrix(static_cast<int>(k), std::move(m)), tq, cq, lab.text);
            } catch (const std::invalid_argument& e) {
                fail(kw, e.what());
            }
        }();
        add(std::move(g), kw);
    }
};

std::string num(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

// A gate is emitted by mnemonic only if rebuilding it from (label, params, qubits)
// gives back the identical matrix; anything else needs the matrix directive.
bool emit_mnemonic(const Gate& g, std::string& line) {
    static const char* const kNames[] = {"h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx",
                                         "ry", "rz", "u1", "p", "cx", "cz", "cp", "cu1"};
    bool known = false;
    for (const char* nm : kNames)
        known |= g.label() == nm;
    if (!known || g.targets().size() != 1 || g.controls().size() > 1)
        return false;
    std::vector<int> qs;
    if (!g.controls().empty())
        qs.push_back(g.controls()[0]);
    qs.push_back(g.targets()[0]);
    try {
        const Gate r = gates::from_mnemonic(g.label(), g.params(), qs);
        if (r.targets() != g.targets() || r.controls() != g.controls() ||
            r.matrix().entries() != g.matrix().entries())
            return false;
    } catch (const std::invalid_argument&) {
        return false;
    }
    std::ostringstream o;
    o << g.label();
    if (!g.params().empty()) {
        o << '(';
        for (std::size_t i = 0; i < g.params().size(); ++i)
            o << (i ? "," : "") << num(g.params()[i]);
        o << ')';
    }
    for (std::size_t i = 0; i < qs.size(); ++i)
        o << (i ? ", " : " ") << "q[" << qs[i] << ']';
    o << ';';
    line = o.str();
    return true;
}

} // namespace

Circuit parse_qasm(std::string_view text, std::string source) {
    Parser p(lex(text), std::move(source));
    return p.run();
}

Circuit parse_qasm_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f)
        throw std::invalid_argument("qasm: cannot open '" + path + "'");
    std::ostringstream ss;
    ss << f.rdbuf();
    return parse_qasm(ss.str(), path);
}

std::string emit_qasm(const Circuit& c, const QasmEmitOptions& opts) {
    std::ostringstream o;
    o << "OPENQASM 2.0;\ninclude \"qelib1.inc\";\n";
    if (!c.source.empty() && c.source.find('\n') == std::string::npos)
        o << "// source: " << c.source << '\n';
    o << "qreg q[" << c.n << "];\n";
    for (std::size_t gi = 0; gi < c.gates.size(); ++gi) {
        const Gate& g = c.gates[gi];
        if (g.is_fence()) {
            if (g.targets().empty()) {
                o << "barrier q;\n";
            } else {
                o << "barrier";
                for (std::size_t i = 0; i < g.targets().size(); ++i)
                    o << (i ? ", " : " ") << "q[" << g.targets()[i] << ']';
                o << ";\n";
            }
            continue;
        }
        std::string line;
        if (emit_mnemonic(g, line)) {
            o << line << '\n';
            continue;
        }
        if (!opts.matrix_export)
            throw std::invalid_argument("emit_qasm: gate " + std::to_string(gi) + " ('" + g.label() +
                                        "') is not in the QASM subset; enable matrix export");
        std::string label = g.label();
        for (char& ch : label)
            if (ch == '"' || ch == '\n')
                ch = '_';
        o << "// qsv-unitary \"" << label << "\" (";
        const auto& es = g.matrix().entries();
        for (std::size_t i = 0; i < es.size(); ++i)
            o << (i ? ", " : "") << num(es[i].real()) << ", " << num(es[i].imag());
        o << ')';
        for (std::size_t i = 0; i < g.targets().size(); ++i)
            o << (i ? ", " : " ") << "q[" << g.targets()[i] << ']';
        if (!g.controls().empty()) {
            o << " |";
            for (std::size_t i = 0; i < g.controls().size(); ++i)
                o << (i ? ", " : " ") << "q[" << g.controls()[i] << ']';
        }
        o << ";\n";
    }
    return o.str();
}

} // namespace qsim
