// Definitions for qsim/fusion.hpp (SPEC DAGC, reference semantics).
#include "qsim/fusion.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace qsim {

namespace {

bool same_set(std::vector<int> a, std::vector<int> b) {
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    return a == b;
}

bool intersects(const std::vector<int>& a, const std::vector<int>& b) {
    for (int x : a)
        if (std::find(b.begin(), b.end(), x) != b.end())
            return true;
    return false;
}

// Matrix of an uncontrolled gate embedded on the ordered target list T.
std::vector<Amp> embed(const Gate& g, const std::vector<int>& T) {
    const std::size_t D = std::size_t{1} << T.size();
    const std::size_t k = g.targets().size();
    std::vector<int> p(k);
    std::size_t gm = 0;
    for (std::size_t i = 0; i < k; ++i) {
        p[i] = static_cast<int>(std::find(T.begin(), T.end(), g.targets()[i]) - T.begin());
        gm |= std::size_t{1} << p[i];
    }
    std::vector<Amp> out(D * D, Amp{0.0, 0.0});
    const GateMatrix& m = g.matrix();
    for (std::size_t col = 0; col < D; ++col) {
        std::size_t lc = 0;
        for (std::size_t i = 0; i < k; ++i)
            lc |= ((col >> p[i]) & 1) << i;
        const std::size_t rest = col & ~gm;
        for (std::size_t lr = 0; lr < (std::size_t{1} << k); ++lr) {
            std::size_t row = rest;
            for (std::size_t i = 0; i < k; ++i)
                row |= ((lr >> i) & 1) << p[i];
            out[row * D + col] = m.at(lr, lc);
        }
    }
    return out;
}

std::vector<Amp> mul(const std::vector<Amp>& a, const std::vector<Amp>& b, std::size_t D) {
    std::vector<Amp> c(D * D, Amp{0.0, 0.0});
    for (std::size_t i = 0; i < D; ++i)
        for (std::size_t k = 0; k < D; ++k)
            for (std::size_t j = 0; j < D; ++j)
                c[i * D + j] += a[i * D + k] * b[k * D + j];
    return c;
}

} // namespace

double gate_cost(const Gate& g, int n) {
    if (g.is_fence())
        return 0.0;
    const int k = g.arity();
    const double per_group = 2.0 * std::ldexp(1.0, 2 * k) + std::ldexp(1.0, k);
    return per_group * std::ldexp(1.0, n - k) * std::ldexp(1.0, -static_cast<int>(g.controls().size()));
}

Gate fuse_same_qubit(const Gate& a, const Gate& b) {
    if (a.is_fence() || b.is_fence() || a.is_controlled() || b.is_controlled() ||
        !same_set(a.targets(), b.targets()))
        throw std::invalid_argument("fuse_same_qubit: needs two uncontrolled gates on the same targets");
    const std::vector<int>& T = a.targets();
    const std::size_t D = std::size_t{1} << T.size();
    return Gate::unitary(GateMatrix(static_cast<int>(T.size()), mul(embed(b, T), embed(a, T), D)), T, {},
                         "FUSED");
}

Gate fuse_kronecker(const Gate& a, const Gate& b) {
    if (a.is_fence() || b.is_fence() || a.is_controlled() || b.is_controlled() ||
        intersects(a.targets(), b.targets()))
        throw std::invalid_argument("fuse_kronecker: needs uncontrolled gates on disjoint targets");
    std::vector<int> T = a.targets();
    T.insert(T.end(), b.targets().begin(), b.targets().end());
    std::sort(T.begin(), T.end());
    const std::size_t D = std::size_t{1} << T.size();
    return Gate::unitary(GateMatrix(static_cast<int>(T.size()), mul(embed(b, T), embed(a, T), D)), T, {},
                         "FUSED");
}

Gate fuse_cu(const Gate& a, const Gate& b) {
    if (a.is_fence() || b.is_fence() || !a.is_controlled() || !same_set(a.controls(), b.controls()) ||
        !same_set(a.targets(), b.targets()))
        throw std::invalid_argument("fuse_cu: needs identical controls and targets");
    const std::vector<int>& T = a.targets();
    const std::size_t D = std::size_t{1} << T.size();
    return Gate::unitary(GateMatrix(static_cast<int>(T.size()), mul(embed(b, T), embed(a, T), D)), T,
                         a.controls(), "FUSED");
}

std::tuple<Circuit, FusionPlan, FusionStats> contract(const Circuit& c, int cap) {
    if (cap < 1)
        throw std::invalid_argument("contract: cap must be >= 1");
    c.validate();
    FusionPlan plan;
    FusionStats st;
    st.gates_before = c.gate_count();
    for (const Gate& g : c.gates)
        st.cost_before += gate_cost(g, c.n);
    std::vector<Gate> gates = c.gates;
    constexpr int kWindow = 64;  // Kronecker partner search distance
    bool changed = true;
    while (changed) {
        changed = false;
        const int N = static_cast<int>(gates.size());
        std::vector<char> used(static_cast<std::size_t>(N), 0);
        std::vector<Gate> out;
        out.reserve(gates.size());
        for (int i = 0; i < N; ++i) {
            if (used[i])
                continue;
            const Gate& g = gates[i];
            if (g.is_fence()) {
                out.push_back(g);
                continue;
            }
            const std::vector<int> qi = g.qubits();
            // first later gate on any of g's qubits (its DAG successor on those wires)
            int j = -1;
            for (int x = i + 1; x < N; ++x)
                if (!used[x] && intersects(gates[x].qubits(), qi)) {
                    j = x;
                    break;
                }
            bool merged = false;
            if (j >= 0 && !gates[j].is_fence()) {
                const Gate& h = gates[j];
                const double before = gate_cost(g, c.n) + gate_cost(h, c.n);
                // (1) same-qubit merge
                if (!g.is_controlled() && !h.is_controlled() && same_set(g.targets(), h.targets())) {
                    Gate f = fuse_same_qubit(g, h);
                    if (gate_cost(f, c.n) < before) {
                        out.push_back(std::move(f));
                        used[j] = 1;
                        plan.steps.push_back({{i, j}, FusionRule::SameQubit, static_cast<int>(st.passes)});
                        ++st.merges_same_qubit;
                        merged = true;
                    }
                }
                // (2) CU consolidation
                if (!merged && g.is_controlled() && same_set(g.controls(), h.controls()) &&
                    same_set(g.targets(), h.targets())) {
                    Gate f = fuse_cu(g, h);
                    if (gate_cost(f, c.n) < before) {
                        out.push_back(std::move(f));
                        used[j] = 1;
                        plan.steps.push_back({{i, j}, FusionRule::CU, static_cast<int>(st.passes)});
                        ++st.merges_cu;
                        merged = true;
                    }
                }
            }
            // (3) Kronecker with the nearest independent gate that can move up to i
            if (!merged && !g.is_controlled() && g.arity() < cap) {
                for (int x = i + 1; x < N && x <= i + kWindow; ++x) {
                    if (used[x])
                        continue;
                    const Gate& h = gates[x];
                    if (h.is_fence()) {
                        if (intersects(h.targets(), qi))
                            break;
                        continue;
                    }
                    if (h.is_controlled() || intersects(h.targets(), qi) || g.arity() + h.arity() > cap)
                        continue;
                    // h must not depend on anything between i and x, and no controlled
                    // gate in between may use a qubit of either
                    bool ok = true;
                    for (int y = i + 1; y < x && ok; ++y) {
                        if (used[y])
                            continue;
                        const Gate& z = gates[y];
                        if (intersects(z.qubits(), h.targets()))
                            ok = false;
                        for (int cq : z.controls())
                            if (std::find(qi.begin(), qi.end(), cq) != qi.end())
                                ok = false;
                    }
                    if (!ok)
                        continue;
                    Gate f = fuse_kronecker(g, h);
                    if (gate_cost(f, c.n) < gate_cost(g, c.n) + gate_cost(h, c.n)) {
                        out.push_back(std::move(f));
                        used[x] = 1;
                        plan.steps.push_back({{i, x}, FusionRule::Kronecker, static_cast<int>(st.passes)});
                        ++st.merges_kronecker;
                        merged = true;
                    }
                    break;  // only the nearest candidate is tried
                }
            }
            if (merged)
                changed = true;
            else
                out.push_back(g);
        }
        gates = std::move(out);
        ++st.passes;
    }
    Circuit res(c.n, std::move(gates), c.source + "+contract");
    st.gates_after = res.gate_count();
    st.compression_ratio = st.gates_before
                               ? static_cast<double>(st.gates_before - st.gates_after) / st.gates_before
                               : 0.0;
    for (const Gate& g : res.gates)
        st.cost_after += gate_cost(g, c.n);
    return {std::move(res), std::move(plan), st};
}

} // namespace qsim
