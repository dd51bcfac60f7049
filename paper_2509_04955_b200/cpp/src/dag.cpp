// Definitions for qsim/dag.hpp.
#include "qsim/dag.hpp"

#include <algorithm>

namespace qsim {

bool DepGraph::has_edge(int i, int j) const {
    if (i < 0 || i >= n_gates)
        return false;
    return std::find(succ[i].begin(), succ[i].end(), j) != succ[i].end();
}

std::vector<std::pair<int, int>> DepGraph::edges() const {
    std::vector<std::pair<int, int>> e;
    for (int i = 0; i < n_gates; ++i)
        for (int j : succ[i])
            e.push_back({i, j});
    return e;
}

bool DepGraph::has_path(int i, int j) const {
    if (i >= j)
        return false;
    std::vector<char> seen(static_cast<std::size_t>(n_gates), 0);
    std::vector<int> stack = {i};
    while (!stack.empty()) {
        const int u = stack.back();
        stack.pop_back();
        for (int v : succ[u]) {
            if (v == j)
                return true;
            if (v < j && !seen[v]) {
                seen[v] = 1;
                stack.push_back(v);
            }
        }
    }
    return false;
}

DepGraph build_dag(const Circuit& c) {
    DepGraph g;
    g.n_gates = static_cast<int>(c.gates.size());
    g.succ.resize(g.n_gates);
    g.pred.resize(g.n_gates);
    g.qubits.resize(g.n_gates);
    std::vector<int> last(static_cast<std::size_t>(c.n), -1);
    for (int j = 0; j < g.n_gates; ++j) {
        g.qubits[j] = c.gates[j].qubits();
        for (int q : g.qubits[j]) {
            const int i = last[q];
            if (i >= 0 && !g.has_edge(i, j)) {
                g.succ[i].push_back(j);
                g.pred[j].push_back(i);
            }
            last[q] = j;
        }
    }
    return g;
}

} // namespace qsim
