// Definitions for qsim/partition.hpp and qsim/stagger.hpp.
#include "qsim/device.hpp"
#include "qsim/partition.hpp"
#include "qsim/stagger.hpp"

#include <algorithm>
#include <stdexcept>

namespace qsim {

PartitionPlan::PartitionPlan(int n_qubits, int m_global, int b_batch, int nbuffers)
    : n(n_qubits), m(m_global), l(n_qubits - m_global), b(b_batch), buffers(nbuffers) {
    if (n < 1 || m < 0 || m >= n)
        throw std::invalid_argument("PartitionPlan: need 0 <= m < n");
    if (b < 0 || b >= l)
        throw std::invalid_argument("PartitionPlan: need 0 <= b < l");
    if (buffers < 1)
        throw std::invalid_argument("PartitionPlan: need at least one buffer");
}

Locality classify_gate(const Gate& g, const PartitionPlan& p) {
    if (g.is_fence())
        return Locality::LOCAL;
    bool tr = false, cr = false;
    for (int t : g.targets())
        tr = tr || t >= p.l;
    for (int c : g.controls())
        cr = cr || c >= p.l;
    if (tr && cr)
        return Locality::BOTH_REMOTE;
    if (tr)
        return Locality::TARGET_REMOTE;
    if (cr)
        return Locality::CONTROL_REMOTE;
    return Locality::LOCAL;
}

int peer_rank(int r, int t, int l) {
    if (t < l)
        throw std::invalid_argument("peer_rank: target " + std::to_string(t) + " is local (t < l)");
    return r ^ (1 << (t - l));
}

std::vector<std::vector<int>> stagger_schedule(int G, int S) {
    if (S < 1 || G < 0 || G > S)
        throw std::invalid_argument("stagger_schedule: need 0 <= G <= S, S >= 1");
    std::vector<std::vector<int>> t(static_cast<std::size_t>(G), std::vector<int>(static_cast<std::size_t>(S)));
    for (int g = 0; g < G; ++g)
        for (int tau = 0; tau < S; ++tau)
            t[g][tau] = (g + tau) % S;
    return t;
}

std::pair<std::vector<StaggerGroup>, std::vector<int>> plan_groups(const Circuit& c, const DepGraph& dag, int S,
                                                                   int local_qubits) {
    if (S < 1 || (S & (S - 1)))
        throw std::invalid_argument("plan_groups: S must be a power of two");
    (void)dag;
    int s = 0;
    while ((1 << s) < S)
        ++s;
    const int l = local_qubits < 0 ? c.n : local_qubits;
    const int limit = l - s;  // every qubit of a member must lie below the segment bits
    std::vector<StaggerGroup> groups;
    std::vector<int> residual;
    std::vector<int> cur;
    std::vector<int> used_q;
    auto close = [&] {
        if (cur.size() >= 2) {
            StaggerGroup g;
            g.gates = cur;
            g.s = s;
            g.schedule = stagger_schedule(static_cast<int>(cur.size()), S);
            groups.push_back(std::move(g));
        } else {
            residual.insert(residual.end(), cur.begin(), cur.end());
        }
        cur.clear();
        used_q.clear();
    };
    for (int i = 0; i < static_cast<int>(c.gates.size()); ++i) {
        const Gate& g = c.gates[i];
        const std::vector<int> q = g.qubits();
        bool eligible = !g.is_fence();
        for (int x : q)
            eligible = eligible && x < limit;
        bool disjoint = true;
        for (int x : q)
            disjoint = disjoint && std::find(used_q.begin(), used_q.end(), x) == used_q.end();
        if (!eligible) {
            close();
            residual.push_back(i);
            continue;
        }
        if (!disjoint || static_cast<int>(cur.size()) >= S)
            close();
        cur.push_back(i);
        used_q.insert(used_q.end(), q.begin(), q.end());
    }
    close();
    std::sort(residual.begin(), residual.end());
    return {std::move(groups), std::move(residual)};
}

void execute_staggered(StateVector& state, const Circuit& c, const StaggerGroup& group, int workers) {
    if (workers < 1)
        throw std::invalid_argument("execute_staggered: workers must be >= 1");
    Circuit sub(c.n, c.source + "[group]");
    for (int gi : group.gates)
        sub.add(c.gates.at(static_cast<std::size_t>(gi)));
    PlanOptions opt;
    opt.fusion = false;  // members applied as given, in order, inside one pass
    opt.pass_budget = 1e30;
    DeviceContext& ctx = DeviceContext::default_context();
    Engine eng(ctx, sub, opt);
    DeviceState d(ctx, state.n());
    d.upload(state.data(), 0, state.size());
    eng.run(d);
    d.download(state.data(), 0, state.size());
}

} // namespace qsim
