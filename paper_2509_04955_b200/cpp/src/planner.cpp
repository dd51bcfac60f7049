// Definitions for qsim/planner.hpp.
#include "qsim/planner.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>

namespace qsim {

namespace {

bool matrix_is_diagonal(const GateMatrix& m) {
    const Index d = m.dim();
    for (Index r = 0; r < d; ++r)
        for (Index c = 0; c < d; ++c)
            if (r != c && m.at(r, c) != Amp{0.0, 0.0})
                return false;
    return true;
}

bool matrix_is_x(const GateMatrix& m) {
    return m.arity() == 1 && m.at(0, 0) == Amp{0.0, 0.0} && m.at(1, 1) == Amp{0.0, 0.0} &&
           m.at(0, 1) == Amp{1.0, 0.0} && m.at(1, 0) == Amp{1.0, 0.0};
}

std::vector<int> all_qubits(const Op& o) {
    std::vector<int> q = o.qubits;
    q.insert(q.end(), o.controls.begin(), o.controls.end());
    return q;
}

bool contains(const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); }

int index_of(const std::vector<int>& v, int x) {
    for (std::size_t i = 0; i < v.size(); ++i)
        if (v[i] == x)
            return static_cast<int>(i);
    return -1;
}

// Dense matrix (2^|T| x 2^|T|, row-major) of `op` acting on the ordered qubit
// list T (bit p <-> T[p]) inside the subspace where the controls NOT in T are 1.
// Requires op.qubits within T; op.controls within T or within the kept controls.
std::vector<Amp> expand_dense(const Op& op, const std::vector<int>& T) {
    const std::size_t D = std::size_t{1} << T.size();
    std::vector<Amp> out(D * D, Amp{0.0, 0.0});
    std::vector<int> p(op.qubits.size());
    std::size_t opmask = 0;
    for (std::size_t i = 0; i < op.qubits.size(); ++i) {
        p[i] = index_of(T, op.qubits[i]);
        opmask |= std::size_t{1} << p[i];
    }
    std::size_t cmask = 0;
    for (int c : op.controls) {
        const int pc = index_of(T, c);
        if (pc >= 0)
            cmask |= std::size_t{1} << pc;
    }
    const std::size_t k = op.qubits.size();
    const std::size_t dk = std::size_t{1} << k;
    for (std::size_t j = 0; j < D; ++j) {
        if ((j & cmask) != cmask) {
            out[j * D + j] = Amp{1.0, 0.0};
            continue;
        }
        std::size_t lin = 0;
        for (std::size_t i = 0; i < k; ++i)
            lin |= ((j >> p[i]) & 1) << i;
        const std::size_t rest = j & ~opmask;
        switch (op.kind) {
        case OpKind::Dense:
            for (std::size_t rl = 0; rl < dk; ++rl) {
                std::size_t row = rest;
                for (std::size_t i = 0; i < k; ++i)
                    row |= ((rl >> i) & 1) << p[i];
                out[row * D + j] = op.data[rl * dk + lin];
            }
            break;
        case OpKind::Diag:
            out[j * D + j] = op.data[lin];
            break;
        case OpKind::XPerm:
            out[(j ^ (std::size_t{1} << p[0])) * D + j] = Amp{1.0, 0.0};
            break;
        case OpKind::Fence:
            throw std::logic_error("expand_dense: fence");
        }
    }
    return out;
}

std::vector<Amp> matmul(const std::vector<Amp>& a, const std::vector<Amp>& b, std::size_t D) {
    std::vector<Amp> c(D * D, Amp{0.0, 0.0});
    for (std::size_t i = 0; i < D; ++i)
        for (std::size_t k = 0; k < D; ++k) {
            const Amp aik = a[i * D + k];
            if (aik == Amp{0.0, 0.0})
                continue;
            for (std::size_t j = 0; j < D; ++j)
                c[i * D + j] += aik * b[k * D + j];
        }
    return c;
}

// A diagonal op with a single non-unit entry at the all-ones pattern becomes a
// "phase on all-ones" op: k = 0 diag whose qubits all moved into the controls.
void canonical_phase(Op& o) {
    if (o.kind != OpKind::Diag || o.qubits.empty())
        return;
    const std::size_t D = o.data.size();
    for (std::size_t e = 0; e + 1 < D; ++e)
        if (o.data[e] != Amp{1.0, 0.0})
            return;
    const Amp last = o.data[D - 1];
    o.controls.insert(o.controls.end(), o.qubits.begin(), o.qubits.end());
    o.qubits.clear();
    o.data.assign(1, last);
}

// Merge B (later) into A (earlier); returns false when the result would exceed
// the arity limits.
bool merge_ops(const Op& A, const Op& B, int fuse_k, Op& out) {
    std::vector<int> C;  // controls common to both stay controls
    for (int c : A.controls)
        if (contains(B.controls, c))
            C.push_back(c);
    std::vector<int> T;
    for (const Op* o : {&A, &B})
        for (int q : all_qubits(*o))
            if (!contains(C, q) && !contains(T, q))
                T.push_back(q);
    std::sort(T.begin(), T.end());
    std::sort(C.begin(), C.end());
    const bool both_diag = A.kind == OpKind::Diag && B.kind == OpKind::Diag;
    const int limit = both_diag ? QSV_MAX_DIAG_K : fuse_k;
    if (static_cast<int>(T.size()) > limit)
        return false;
    if (!both_diag && T.empty())
        return false;
    const std::size_t D = std::size_t{1} << T.size();
    out = Op{};
    out.qubits = T;
    out.controls = C;
    out.first_gate = std::min(A.first_gate, B.first_gate);
    out.last_gate = std::max(A.last_gate, B.last_gate);
    out.ngates = A.ngates + B.ngates;
    if (both_diag) {
        out.kind = OpKind::Diag;
        out.data.assign(D, Amp{1.0, 0.0});
        for (const Op* o : {&A, &B}) {
            // diagonal entry of o at T-pattern e
            std::vector<int> p(o->qubits.size());
            for (std::size_t i = 0; i < p.size(); ++i)
                p[i] = index_of(T, o->qubits[i]);
            std::size_t cm = 0;
            for (int c : o->controls) {
                const int pc = index_of(T, c);
                if (pc >= 0)
                    cm |= std::size_t{1} << pc;
            }
            for (std::size_t e = 0; e < D; ++e) {
                if ((e & cm) != cm)
                    continue;
                std::size_t lin = 0;
                for (std::size_t i = 0; i < p.size(); ++i)
                    lin |= ((e >> p[i]) & 1) << i;
                out.data[e] = o->data[lin] * out.data[e];
            }
        }
        canonical_phase(out);
        return true;
    }
    out.kind = OpKind::Dense;
    out.data = matmul(expand_dense(B, T), expand_dense(A, T), D);
    return true;
}

bool is_identity(const Op& o) {
    if (o.kind == OpKind::XPerm || o.kind == OpKind::Fence)
        return false;
    const std::size_t D = o.kind == OpKind::Dense ? std::size_t{1} << o.qubits.size() : o.data.size();
    for (std::size_t r = 0; r < D; ++r) {
        if (o.kind == OpKind::Diag) {
            if (o.data[r] != Amp{1.0, 0.0}) return false;
            continue;
        }
        for (std::size_t c = 0; c < D; ++c)
            if (o.data[r * D + c] != (r == c ? Amp{1.0, 0.0} : Amp{0.0, 0.0}))
                return false;
    }
    return true;
}

} // namespace

double op_cost(const Op& o) {
    const double ctl = std::ldexp(1.0, -static_cast<int>(o.controls.size()));
    switch (o.kind) {
    case OpKind::Dense: return 4.0 * std::ldexp(1.0, static_cast<int>(o.qubits.size())) * ctl + 2.0;
    case OpKind::Diag: return 4.0 * ctl + 2.0;
    case OpKind::XPerm: return 1.0 * ctl + 1.0;
    case OpKind::Fence: return 0.0;
    }
    return 0.0;
}

std::vector<Op> lower(const Circuit& c) {
    std::vector<Op> ops;
    ops.reserve(c.gates.size());
    for (std::size_t gi = 0; gi < c.gates.size(); ++gi) {
        const Gate& g = c.gates[gi];
        Op o;
        o.first_gate = o.last_gate = static_cast<int>(gi);
        o.ngates = 1;
        if (g.is_fence()) {
            o.kind = OpKind::Fence;
            o.qubits = g.targets();
            o.ngates = 0;
            ops.push_back(std::move(o));
            continue;
        }
        const GateMatrix& m = g.matrix();
        o.qubits = g.targets();
        o.controls = g.controls();
        if (matrix_is_x(m)) {
            o.kind = OpKind::XPerm;
        } else if (matrix_is_diagonal(m)) {
            o.kind = OpKind::Diag;
            for (Index i = 0; i < m.dim(); ++i)
                o.data.push_back(m.at(i, i));
            canonical_phase(o);
        } else {
            o.kind = OpKind::Dense;
            o.data = m.entries();
        }
        ops.push_back(std::move(o));
    }
    return ops;
}

std::vector<Op> fuse_ops(const std::vector<Op>& in, const PlanOptions& opt) {
    std::vector<Op> out;
    out.reserve(in.size());
    int nq = 0;
    for (const Op& o : in)
        for (int q : all_qubits(o))
            nq = std::max(nq, q + 1);
    std::vector<int> frontier(static_cast<std::size_t>(nq), -1);
    for (const Op& b : in) {
        const std::vector<int> qb = all_qubits(b);
        int a = -1;
        for (int q : qb)
            a = std::max(a, frontier[q]);
        if (b.kind != OpKind::Fence && a >= 0 && out[a].kind != OpKind::Fence) {
            Op merged;
            if (merge_ops(out[a], b, opt.fuse_k, merged) &&
                op_cost(merged) <= op_cost(out[a]) + op_cost(b) + 1e-9) {
                out[a] = std::move(merged);
                for (int q : all_qubits(out[a]))
                    frontier[q] = std::max(frontier[q], a);
                continue;
            }
        }
        out.push_back(b);
        for (int q : qb)
            frontier[q] = static_cast<int>(out.size()) - 1;
    }
    // Exact identities (e.g. H.H, CX.CX) are dropped — an optimiser choice, the
    // kernel itself never special-cases identity.
    std::vector<Op> kept;
    kept.reserve(out.size());
    for (Op& o : out)
        if (o.kind != OpKind::Fence && !is_identity(o))
            kept.push_back(std::move(o));
    return kept;
}

namespace {

struct Packer {
    const PlanOptions& opt;
    int n, n_local, K, Lmin;
    Plan& plan;
    std::vector<int> pos;          // logical -> physical
    // current pass
    std::vector<int> targets;      // physical dense/xperm targets in the pass
    std::vector<qsv_op_desc> cur_ops;
    double cur_cost = 0;
    std::size_t cur_bytes = 0;

    Packer(const PlanOptions& o, int n_, int nl, Plan& p) : opt(o), n(n_), n_local(nl), plan(p) {
        K = std::min(opt.tile_k, n_local);
        Lmin = std::min(opt.min_low, K);
        pos.resize(n);
        for (int q = 0; q < n; ++q)
            pos[q] = q;
    }

    // Largest L >= Lmin with L + |{t >= L}| <= K, or -1 when infeasible.
    int low_run(const std::vector<int>& t) const {
        int best = -1;
        for (int L = Lmin; L <= K; ++L) {
            int hi = 0;
            for (int q : t)
                hi += q >= L;
            if (L + hi <= K && hi <= QSV_MAX_HIGH)
                best = L;
        }
        return best;
    }

    void close_pass() {
        if (cur_ops.empty())
            return;
        const int L = low_run(targets);
        if (L < 0)
            throw std::logic_error("planner: infeasible pass tile");
        qsv_step_desc s{};
        s.kind = QSV_STEP_PASS;
        s.tile_k = K;
        std::vector<int> high;
        for (int q : targets)
            if (q >= L)
                high.push_back(q);
        std::sort(high.begin(), high.end());
        // pad the tile with high qubits when targets don't fill it (K - L slots)
        const int want_high = K - L;
        for (int q = n_local - 1; static_cast<int>(high.size()) < want_high && q >= L; --q)
            if (!contains(high, q))
                high.push_back(q);
        std::sort(high.begin(), high.end());
        s.nhigh = static_cast<int>(high.size());
        for (std::size_t i = 0; i < high.size(); ++i)
            s.high[i] = high[i];
        s.op_begin = static_cast<int>(plan.ops.size());
        s.op_count = static_cast<int>(cur_ops.size());
        plan.ops.insert(plan.ops.end(), cur_ops.begin(), cur_ops.end());
        plan.steps.push_back(s);
        plan.stats.passes++;
        cur_ops.clear();
        targets.clear();
        cur_cost = 0;
        cur_bytes = 0;
    }

    qsv_op_desc to_desc(const Op& o) {
        qsv_op_desc d{};
        d.k = static_cast<int>(o.qubits.size());
        for (std::size_t i = 0; i < o.qubits.size(); ++i)
            d.qubits[i] = pos[o.qubits[i]];
        for (int c : o.controls)
            d.ctrl_mask |= 1ull << pos[c];
        d.kind = o.kind == OpKind::Dense ? QSV_OP_DENSE : (o.kind == OpKind::Diag ? QSV_OP_DIAG : QSV_OP_XPERM);
        d.mat_off = static_cast<int64_t>(plan.pool.size() / 2);
        for (const Amp& a : o.data) {
            plan.pool.push_back(a.real());
            plan.pool.push_back(a.imag());
        }
        return d;
    }

    static std::size_t blob_bytes(const Op& o) {
        // TileOp record + member offsets + matrix/table, 16-B aligned pieces
        std::size_t b = 96;
        if (o.kind == OpKind::Dense) {
            const std::size_t D = std::size_t{1} << o.qubits.size();
            b += ((D * 4 + 15) & ~std::size_t{15}) + D * D * 16;
        } else if (o.kind == OpKind::Diag) {
            b += o.data.size() * 16;
        }
        return b;
    }

    void add(const Op& o) {
        std::vector<int> need = targets;
        if (o.kind == OpKind::Dense || o.kind == OpKind::XPerm)
            for (int q : o.qubits)
                if (!contains(need, pos[q]))
                    need.push_back(pos[q]);
        const double c = op_cost(o);
        const std::size_t b = blob_bytes(o);
        const bool fits = low_run(need) >= 0 && (cur_ops.empty() || cur_cost + c <= opt.pass_budget) &&
                          cur_bytes + b <= 36 * 1024 && (opt.multi_op_passes || cur_ops.empty());
        if (!fits && !cur_ops.empty()) {
            close_pass();
            add(o);
            return;
        }
        if (low_run(need) < 0)
            throw std::logic_error("planner: op does not fit a tile (k too large for tile_k)");
        targets = need;
        cur_ops.push_back(to_desc(o));
        cur_cost += c;
        cur_bytes += b;
    }

    void swap(int g_phys, int v_phys) {
        close_pass();
        qsv_step_desc s{};
        s.kind = QSV_STEP_SWAP;
        s.swap_global = g_phys;
        s.swap_local = v_phys;
        s.chunk_log2 = std::min(opt.chunk_log2, n_local - 1);
        s.nbuf = opt.nbuf;
        plan.steps.push_back(s);
        plan.stats.swaps++;
        int lg = -1, lv = -1;
        for (int q = 0; q < n; ++q) {
            if (pos[q] == g_phys) lg = q;
            if (pos[q] == v_phys) lv = q;
        }
        std::swap(pos[lg], pos[lv]);
    }
};

} // namespace

Plan make_plan(const Circuit& c, const PlanOptions& opt) {
    c.validate();
    if (opt.fuse_k < 1 || opt.fuse_k > QSV_MAX_DENSE_K)
        throw std::invalid_argument("make_plan: fuse_k must be in [1, 5]");
    if (opt.tile_k < 1 || opt.tile_k > 11)
        throw std::invalid_argument("make_plan: tile_k must be in [1, 11]");
    Plan plan;
    plan.n = c.n;
    plan.n_local = opt.n_local < 0 ? c.n : opt.n_local;
    if (plan.n_local < 1 || plan.n_local > c.n)
        throw std::invalid_argument("make_plan: n_local must be in [1, n]");
    plan.stats.gates_in = c.gate_count();
    std::vector<Op> ops = lower(c);
    plan.stats.ops_lowered = ops.size();
    if (opt.fusion) {
        ops = fuse_ops(ops, opt);
    } else {
        std::vector<Op> kept;
        for (Op& o : ops)
            if (o.kind != OpKind::Fence)
                kept.push_back(std::move(o));
        ops = std::move(kept);
    }
    plan.stats.ops_fused = ops.size();
    for (const Op& o : ops) {
        plan.stats.cost_units += op_cost(o);
        if (o.kind == OpKind::Dense)
            plan.stats.max_dense_k = std::max(plan.stats.max_dense_k, static_cast<int>(o.qubits.size()));
    }

    Packer pk(opt, c.n, plan.n_local, plan);
    // next-use table for victim selection: for each op index, when is logical q
    // next needed as a dense/xperm target?
    const int nops = static_cast<int>(ops.size());
    auto needs_tile = [](const Op& o, int q) {
        return (o.kind == OpKind::Dense || o.kind == OpKind::XPerm) && contains(o.qubits, q);
    };
    std::vector<std::vector<int>> uses(c.n);
    for (int i = 0; i < nops; ++i)
        for (int q : ops[i].qubits)
            if (needs_tile(ops[i], q))
                uses[q].push_back(i);
    std::vector<std::size_t> cursor(c.n, 0);
    auto next_use = [&](int q, int from) {
        auto& u = uses[q];
        std::size_t& k = cursor[q];
        while (k < u.size() && u[k] < from)
            ++k;
        return k < u.size() ? u[k] : std::numeric_limits<int>::max();
    };
    for (int i = 0; i < nops; ++i) {
        const Op& o = ops[i];
        if (o.kind == OpKind::Dense || o.kind == OpKind::XPerm) {
            for (int q : o.qubits) {
                if (pk.pos[q] < plan.n_local)
                    continue;
                // choose the local victim whose next tile use is farthest away,
                // preferring high physical positions (contiguous swap chunks)
                int best = -1;
                long long best_score = -1;
                for (int l = 0; l < c.n; ++l) {
                    const int p = pk.pos[l];
                    if (p >= plan.n_local || contains(o.qubits, l))
                        continue;
                    if (contains(pk.targets, p))
                        continue;
                    const long long nu = next_use(l, i);
                    const long long score = nu * 64 + p;
                    if (score > best_score) {
                        best_score = score;
                        best = l;
                    }
                }
                if (best < 0)
                    throw std::logic_error("planner: no swap victim available");
                pk.swap(pk.pos[q], pk.pos[best]);
            }
        }
        pk.add(o);
    }
    pk.close_pass();
    // restore the logical qubit order so the final state is in standard layout
    for (int q = 0; q < c.n; ++q) {
        if (pk.pos[q] == q)
            continue;
        // q sits at pos[q]; whoever sits at q must move. One swap per global slot.
        int other = -1;
        for (int r = 0; r < c.n; ++r)
            if (pk.pos[r] == q)
                other = r;
        const int a = pk.pos[q], b = q;  // physical slots to exchange
        if (a >= plan.n_local && b < plan.n_local)
            pk.swap(a, b);
        else if (b >= plan.n_local && a < plan.n_local)
            pk.swap(b, a);
        else if (a < plan.n_local && b < plan.n_local) {
            // local-local relabel: a SWAP of two local qubits as one dense pass
            Op sw;
            sw.kind = OpKind::Dense;
            sw.qubits = {q, other};
            sw.data.assign(16, Amp{0.0, 0.0});
            sw.data[0] = sw.data[15] = Amp{1.0, 0.0};
            sw.data[1 * 4 + 2] = sw.data[2 * 4 + 1] = Amp{1.0, 0.0};
            // pos[] maps logical->physical: the op must act on the physical
            // slots a and b, and afterwards q sits at b and other at a.
            pk.add(sw);
            pk.close_pass();
            std::swap(pk.pos[q], pk.pos[other]);
        } else {
            // both slots global: (a b) = (a t)(b t)(a t) through a local slot t
            const int t = plan.n_local - 1;
            pk.swap(a, t);
            pk.swap(b, t);
            pk.swap(a, t);
        }
    }
    plan.fused = std::move(ops);
    return plan;
}

Circuit ops_to_circuit(int n, const std::vector<Op>& ops) {
    Circuit c(n, "fused");
    for (const Op& o : ops) {
        if (o.kind == OpKind::Fence)
            continue;
        std::vector<int> t = o.qubits, ctl = o.controls;
        std::vector<Amp> m;
        int k = static_cast<int>(t.size());
        if (o.kind == OpKind::Dense) {
            m = o.data;
        } else if (o.kind == OpKind::XPerm) {
            m = {0.0, 1.0, 1.0, 0.0};
        } else if (k == 0) {
            // phase on all-ones of the controls: diag(1, e) on the last control
            t = {ctl.back()};
            ctl.pop_back();
            m = {1.0, 0.0, 0.0, o.data[0]};
            k = 1;
        } else {
            const std::size_t D = o.data.size();
            m.assign(D * D, Amp{0.0, 0.0});
            for (std::size_t i = 0; i < D; ++i)
                m[i * D + i] = o.data[i];
        }
        c.add(Gate::unitary(GateMatrix(k, std::move(m)), t, ctl, "FUSED"));
    }
    return c;
}

} // namespace qsim
