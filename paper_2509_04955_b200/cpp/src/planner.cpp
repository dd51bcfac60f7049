// Definitions for qsim/planner.hpp.
#include "qsim/planner.hpp"

#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <optional>
#include <stdexcept>

namespace qsim {

namespace {

using Factors = std::vector<std::pair<int, Amp>>;

bool contains(const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); }

int index_of(const std::vector<int>& v, int x) {
    for (std::size_t i = 0; i < v.size(); ++i)
        if (v[i] == x)
            return static_cast<int>(i);
    return -1;
}

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

bool diag_like(const Op& o) {
    return o.kind == OpKind::Diag || o.kind == OpKind::PhaseProd || o.kind == OpKind::ParPhase;
}

// Every qubit an op reads or writes (its DAG footprint).
std::vector<int> footprint(const Op& o) {
    std::vector<int> q = o.qubits;
    for (int c : o.controls)
        if (!contains(q, c))
            q.push_back(c);
    for (const auto& f : o.factors)
        if (!contains(q, f.first))
            q.push_back(f.first);
    return q;
}

// Diagonal value of a diag-like op on a basis state given by bit(q).
template <typename Bit>
Amp diag_value(const Op& o, Bit&& bit) {
    for (int c : o.controls)
        if (!bit(c))
            return Amp{1.0, 0.0};
    if (o.kind == OpKind::Diag) {
        std::size_t lin = 0;
        for (std::size_t i = 0; i < o.qubits.size(); ++i)
            lin |= static_cast<std::size_t>(bit(o.qubits[i])) << i;
        return o.data[lin];
    }
    if (o.kind == OpKind::ParPhase) {
        int par = 0;
        for (int q : o.qubits)
            par ^= bit(q) & 1;
        return o.data[par];
    }
    Amp v = o.data[0];
    for (const auto& f : o.factors)
        if (bit(f.first))
            v *= f.second;
    return v;
}

// Dense matrix (2^|T| x 2^|T|, row-major) of `op` acting on the ordered qubit
// list T (bit p <-> T[p]) inside the subspace where the controls NOT in T are 1.
std::vector<Amp> expand_dense(const Op& op, const std::vector<int>& T) {
    const std::size_t D = std::size_t{1} << T.size();
    std::vector<Amp> out(D * D, Amp{0.0, 0.0});
    if (diag_like(op)) {
        for (std::size_t j = 0; j < D; ++j)
            out[j * D + j] = diag_value(op, [&](int q) {
                const int p = index_of(T, q);
                return p < 0 ? 1 : static_cast<int>((j >> p) & 1);
            });
        return out;
    }
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
        if (op.kind == OpKind::Dense) {
            for (std::size_t rl = 0; rl < dk; ++rl) {
                std::size_t row = rest;
                for (std::size_t i = 0; i < k; ++i)
                    row |= ((rl >> i) & 1) << p[i];
                out[row * D + j] = op.data[rl * dk + lin];
            }
        } else if (op.kind == OpKind::XPerm) {
            out[(j ^ (std::size_t{1} << p[0])) * D + j] = Amp{1.0, 0.0};
        } else {
            throw std::logic_error("expand_dense: unsupported op kind");
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

// Re-express a diag-like op as a phase product controlled by exactly C.
std::optional<std::pair<Factors, Amp>> as_phaseprod(const Op& o, const std::vector<int>& C) {
    std::vector<int> own = o.controls;
    for (int c : C)
        if (!contains(own, c))
            return std::nullopt;  // C must be a subset of the op's controls
    std::vector<int> extra;
    for (int c : own)
        if (!contains(C, c))
            extra.push_back(c);
    Factors f;
    Amp c0{1.0, 0.0};
    if (o.kind == OpKind::ParPhase && o.qubits.size() != 1) {
        return std::nullopt;
    } else if (o.kind == OpKind::PhaseProd) {
        f = o.factors;
        c0 = o.data[0];
    } else if (o.qubits.empty()) {
        c0 = o.data[0];
    } else if (o.qubits.size() == 1 && o.data[0] != Amp{0.0, 0.0}) {
        c0 = o.data[0];
        f.push_back({o.qubits[0], o.data[1] / o.data[0]});
    } else {
        return std::nullopt;
    }
    if (extra.size() > 1)
        return std::nullopt;
    if (extra.size() == 1) {
        if (!f.empty())
            return std::nullopt;  // c0 * prod f under an extra control is not separable
        f.push_back({extra[0], c0});
        c0 = Amp{1.0, 0.0};
    }
    return std::make_pair(f, c0);
}

Op make_phaseprod(const Op& A, const Op& B, const std::vector<int>& C, const Factors& fa, Amp ca,
                  const Factors& fb, Amp cb) {
    Op out;
    out.kind = OpKind::PhaseProd;
    out.controls = C;
    std::map<int, Amp> acc;
    for (const auto* fs : {&fa, &fb})
        for (const auto& f : *fs) {
            auto it = acc.find(f.first);
            if (it == acc.end())
                acc[f.first] = f.second;
            else
                it->second *= f.second;
        }
    for (const auto& kv : acc)
        if (!contains(C, kv.first))
            out.factors.push_back(kv);
    Amp c = ca * cb;
    for (const auto& kv : acc)
        if (contains(C, kv.first))
            c *= kv.second;  // a factor on a control qubit is always applied
    out.data = {c};
    out.first_gate = std::min(A.first_gate, B.first_gate);
    out.last_gate = std::max(A.last_gate, B.last_gate);
    out.ngates = A.ngates + B.ngates;
    return out;
}

// Merge B (later) into A (earlier); false when no legal/within-limit merge exists.
bool merge_ops(const Op& A, const Op& B, int fuse_k, int min_low, int max_high, Op& out) {
    if (A.kind == OpKind::Fence || B.kind == OpKind::Fence || A.kind == OpKind::RBlock ||
        B.kind == OpKind::RBlock || A.kind == OpKind::Swap || B.kind == OpKind::Swap)
        return false;
    if (diag_like(A) && diag_like(B)) {
        // (1) separable phase product under the common controls
        std::vector<int> C;
        for (int c : A.controls)
            if (contains(B.controls, c))
                C.push_back(c);
        std::sort(C.begin(), C.end());
        const auto pa = as_phaseprod(A, C);
        const auto pb = as_phaseprod(B, C);
        if (pa && pb) {
            out = make_phaseprod(A, B, C, pa->first, pa->second, pb->first, pb->second);
            return true;
        }
    }
    std::vector<int> C;  // controls common to both stay controls
    if (A.kind != OpKind::PhaseProd && B.kind != OpKind::PhaseProd)
        for (int c : A.controls)
            if (contains(B.controls, c))
                C.push_back(c);
    std::vector<int> T;
    for (const Op* o : {&A, &B})
        for (int q : footprint(*o))
            if (!contains(C, q) && !contains(T, q))
                T.push_back(q);
    std::sort(T.begin(), T.end());
    std::sort(C.begin(), C.end());
    const bool both_diag = diag_like(A) && diag_like(B);
    const int limit = both_diag ? QSV_MAX_DIAG_K : fuse_k;
    if (static_cast<int>(T.size()) > limit)
        return false;
    if (!both_diag) {
        // a dense block must fit one tile: at most max_high targets above the low run
        int high = 0;
        for (int q : T)
            high += q >= min_low;
        if (high > max_high)
            return false;
    }
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
        out.data.resize(D);
        for (std::size_t e = 0; e < D; ++e) {
            auto bit = [&](int q) {
                const int p = index_of(T, q);
                return p < 0 ? 1 : static_cast<int>((e >> p) & 1);
            };
            out.data[e] = diag_value(B, bit) * diag_value(A, bit);
        }
        canonical_phase(out);
        return true;
    }
    out.kind = OpKind::Dense;
    out.data = matmul(expand_dense(B, T), expand_dense(A, T), D);
    return true;
}

bool is_identity(const Op& o) {
    if (o.kind == OpKind::XPerm || o.kind == OpKind::Fence || o.kind == OpKind::RBlock || o.kind == OpKind::Swap)
        return false;
    if (o.kind == OpKind::PhaseProd) {
        if (o.data[0] != Amp{1.0, 0.0})
            return false;
        for (const auto& f : o.factors)
            if (f.second != Amp{1.0, 0.0})
                return false;
        return true;
    }
    if (o.kind == OpKind::Diag || o.kind == OpKind::ParPhase) {
        for (const Amp& a : o.data)
            if (a != Amp{1.0, 0.0})
                return false;
        return true;
    }
    const std::size_t D = std::size_t{1} << o.qubits.size();
    for (std::size_t r = 0; r < D; ++r)
        for (std::size_t c = 0; c < D; ++c)
            if (o.data[r * D + c] != (r == c ? Amp{1.0, 0.0} : Amp{0.0, 0.0}))
                return false;
    return true;
}

// ------------------------------------------------------------ register blocks
bool block_eligible(const Op& o, int width) {
    switch (o.kind) {
    case OpKind::Dense: return o.qubits.size() + o.controls.size() <= 2;
    case OpKind::XPerm: return o.controls.size() <= 1;
    case OpKind::Diag:
    case OpKind::ParPhase:
    case OpKind::PhaseProd: return static_cast<int>(footprint(o).size()) <= width;
    default: return false;
    }
}

double prim_cost(const Prim& p) {
    switch (p.kind) {
    case QSV_PRIM_U1R:
    case QSV_PRIM_U1I: return 4.0;
    case QSV_PRIM_U1: return 8.0;
    case QSV_PRIM_U2: return 16.0;
    case QSV_PRIM_CX: return 0.5;
    default: return 4.0;
    }
}

// Converts the member ops of a block (qubits sorted = slots) into primitives.
// Diagonal tables are laid out over 2^width entries (padded slots repeat).
std::vector<Prim> block_prims(const std::vector<int>& slots, const std::vector<Op>& members, int width) {
    const int ND = 1 << width;
    std::vector<Prim> out;
    auto slot = [&](int q) { return index_of(slots, q); };
    for (const Op& o : members) {
        Prim p;
        if (diag_like(o)) {
            p.kind = QSV_PRIM_DIAG16;
            p.data.resize(ND);
            for (int e = 0; e < ND; ++e)
                p.data[e] = diag_value(o, [&](int q) { return (e >> slot(q)) & 1; });
            if (!out.empty() && out.back().kind == QSV_PRIM_DIAG16) {
                for (int e = 0; e < ND; ++e)
                    out.back().data[e] = p.data[e] * out.back().data[e];
                continue;
            }
        } else if (o.kind == OpKind::XPerm && o.controls.size() == 1) {
            p.kind = QSV_PRIM_CX;
            p.a = slot(o.controls[0]);
            p.b = slot(o.qubits[0]);
        } else if (footprint(o).size() == 1) {
            p.kind = QSV_PRIM_U1;
            p.a = slot(o.qubits[0]);
            p.data = expand_dense(o, {o.qubits[0]});
            if (!out.empty() && out.back().kind == QSV_PRIM_U1 && out.back().a == p.a) {
                out.back().data = matmul(p.data, out.back().data, 2);
                continue;
            }
        } else {
            std::vector<int> fp = footprint(o);
            std::sort(fp.begin(), fp.end());
            p.kind = QSV_PRIM_U2;
            p.a = slot(fp[0]);
            p.b = slot(fp[1]);
            p.data = expand_dense(o, fp);
        }
        out.push_back(std::move(p));
    }
    // structured 2x2 primitives: half the DFMA work of a general complex 2x2
    for (Prim& p : out) {
        if (p.kind != QSV_PRIM_U1)
            continue;
        const auto& m = p.data;
        if (m[0].imag() == 0 && m[1].imag() == 0 && m[2].imag() == 0 && m[3].imag() == 0)
            p.kind = QSV_PRIM_U1R;
        else if (m[0].imag() == 0 && m[3].imag() == 0 && m[1].real() == 0 && m[2].real() == 0)
            p.kind = QSV_PRIM_U1I;
    }
    return out;
}

} // namespace

double op_cost(const Op& o) {
    const double ctl = std::ldexp(1.0, -static_cast<int>(o.controls.size()));
    switch (o.kind) {
    case OpKind::Dense: return 4.0 * std::ldexp(1.0, static_cast<int>(o.qubits.size())) * ctl + 3.0;
    case OpKind::Diag: return 4.0 * ctl + 3.0;
    case OpKind::PhaseProd: return 8.0 * ctl + 3.0;
    case OpKind::ParPhase: return 4.0 * ctl + 3.0;
    case OpKind::XPerm: return 1.0 * ctl + 2.0;
    case OpKind::RBlock: {
        double c = 3.0;
        for (const Prim& p : o.prims)
            c += prim_cost(p);
        return c;
    }
    case OpKind::Fence:
    case OpKind::Swap: return 0.0;
    }
    return 0.0;
}

std::vector<Op> reduce_parity(const std::vector<Op>& in) {
    int nq = 0;
    for (const Op& o : in)
        for (int q : footprint(o))
            nq = std::max(nq, q + 1);
    std::vector<Op> out;
    out.reserve(in.size());
    std::vector<char> alive;
    std::vector<std::vector<int>> wire(static_cast<std::size_t>(nq));  // alive op indices per qubit
    auto is_cx = [](const Op& o, int& c, int& t) {
        if (o.kind != OpKind::XPerm || o.controls.size() != 1)
            return false;
        c = o.controls[0];
        t = o.qubits[0];
        return true;
    };
    // parity view of a diagonal op: (mask, p0, p1)
    auto as_parity = [](const Op& o, std::vector<int>& mask, Amp& p0, Amp& p1) {
        if (!o.controls.empty())
            return false;
        if (o.kind == OpKind::ParPhase) {
            mask = o.qubits;
            p0 = o.data[0];
            p1 = o.data[1];
            return true;
        }
        if (o.kind == OpKind::Diag && o.qubits.size() == 1) {
            mask = o.qubits;
            p0 = o.data[0];
            p1 = o.data[1];
            return true;
        }
        return false;
    };
    auto erase_from = [](std::vector<int>& w, int idx) {
        for (std::size_t i = w.size(); i-- > 0;)
            if (w[i] == idx) {
                w.erase(w.begin() + static_cast<std::ptrdiff_t>(i));
                return;
            }
    };
    for (const Op& b : in) {
        int c = -1, t = -1;
        if (is_cx(b, c, t) && wire[t].size() >= 2) {
            const int y = wire[t].back();
            const int z = wire[t][wire[t].size() - 2];
            int zc = -1, zt = -1;
            std::vector<int> mask;
            Amp p0, p1;
            if (alive[y] && alive[z] && is_cx(out[z], zc, zt) && zc == c && zt == t &&
                as_parity(out[y], mask, p0, p1) && contains(mask, t)) {
                const bool c_in = contains(mask, c);
                const auto& wc = wire[c];
                const bool c_ok = c_in ? (wc.size() >= 2 && wc.back() == y && wc[wc.size() - 2] == z)
                                       : (!wc.empty() && wc.back() == z);
                if (c_ok) {
                    Op p;
                    p.kind = OpKind::ParPhase;
                    p.qubits = mask;
                    if (c_in)
                        p.qubits.erase(std::find(p.qubits.begin(), p.qubits.end(), c));
                    else
                        p.qubits.push_back(c);
                    std::sort(p.qubits.begin(), p.qubits.end());
                    p.data = {p0, p1};
                    p.first_gate = std::min(out[z].first_gate, out[y].first_gate);
                    p.last_gate = b.last_gate;
                    p.ngates = out[z].ngates + out[y].ngates + b.ngates;
                    alive[z] = 0;
                    erase_from(wire[c], z);
                    erase_from(wire[t], z);
                    if (c_in)
                        erase_from(wire[c], y);
                    else
                        wire[c].push_back(y);
                    out[y] = std::move(p);
                    continue;
                }
            }
        }
        const int idx = static_cast<int>(out.size());
        out.push_back(b);
        alive.push_back(1);
        for (int q : footprint(b))
            wire[q].push_back(idx);
    }
    std::vector<Op> res;
    res.reserve(out.size());
    for (std::size_t i = 0; i < out.size(); ++i)
        if (alive[i])
            res.push_back(std::move(out[i]));
    return res;
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
    const int min_low = opt.min_low;
    const int max_high = std::min(QSV_MAX_HIGH, std::max(opt.tile_k - opt.min_low, 0));
    std::vector<Op> out;
    out.reserve(in.size());
    int nq = 0;
    for (const Op& o : in)
        for (int q : footprint(o))
            nq = std::max(nq, q + 1);
    std::vector<int> frontier(static_cast<std::size_t>(nq), -1);
    for (const Op& b : in) {
        const std::vector<int> qb = footprint(b);
        int a = -1;
        for (int q : qb)
            a = std::max(a, frontier[q]);
        if (b.kind != OpKind::Fence && a >= 0 && out[a].kind != OpKind::Fence) {
            Op merged;
            if (merge_ops(out[a], b, opt.fuse_k, min_low, max_high, merged) &&
                op_cost(merged) <= op_cost(out[a]) + op_cost(b) + 1e-9) {
                out[a] = std::move(merged);
                for (int q : footprint(out[a]))
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

std::vector<Op> form_blocks(const std::vector<Op>& in, int min_low, int max_high, int width) {
    // Greedy register blocking over the dependency DAG: a block starts at the
    // earliest unprocessed op and repeatedly absorbs any *available* op (every
    // earlier op on its qubits already placed) whose qubits keep the block within
    // `width` qubits (and within `max_high` qubits above the tile's low run).
    // Ops are emitted in block order, which respects every dependency.
    const int nops = static_cast<int>(in.size());
    int nq = 0;
    std::vector<std::vector<int>> fp(nops);
    for (int i = 0; i < nops; ++i) {
        fp[i] = footprint(in[i]);
        for (int q : fp[i])
            nq = std::max(nq, q + 1);
    }
    std::vector<std::vector<int>> on_qubit(nq);
    for (int i = 0; i < nops; ++i)
        for (int q : fp[i])
            on_qubit[q].push_back(i);
    std::vector<std::size_t> next(nq, 0);
    std::vector<char> done(nops, 0);
    auto available = [&](int i) {
        for (int q : fp[i])
            if (next[q] >= on_qubit[q].size() || on_qubit[q][next[q]] != i)
                return false;
        return true;
    };
    auto take = [&](int i) {
        done[i] = 1;
        for (int q : fp[i])
            ++next[q];
    };
    auto high_count = [&](const std::vector<int>& u) {
        int h = 0;
        for (int q : u)
            h += q >= min_low;
        return h;
    };
    std::vector<Op> res;
    res.reserve(in.size());
    int cursor = 0;
    while (true) {
        while (cursor < nops && done[cursor])
            ++cursor;
        if (cursor >= nops)
            break;
        const int g0 = cursor;  // earliest unprocessed op: always available
        if (!block_eligible(in[g0], width) || high_count(fp[g0]) > max_high) {
            take(g0);
            res.push_back(in[g0]);
            continue;
        }
        std::vector<int> S = fp[g0];
        std::vector<int> members = {g0};
        take(g0);
        while (true) {
            int best = -1, best_growth = 1 << 20;
            std::vector<int> best_u;
            for (int q = 0; q < nq; ++q) {
                if (next[q] >= on_qubit[q].size())
                    continue;
                const int i = on_qubit[q][next[q]];
                if (done[i] || !available(i) || !block_eligible(in[i], width))
                    continue;
                std::vector<int> u = S;
                for (int x : fp[i])
                    if (!contains(u, x))
                        u.push_back(x);
                if (static_cast<int>(u.size()) > width || high_count(u) > max_high)
                    continue;
                const int growth = static_cast<int>(u.size() - S.size());
                if (growth < best_growth || (growth == best_growth && i < best)) {
                    best = i;
                    best_growth = growth;
                    best_u = u;
                }
            }
            if (best < 0)
                break;
            S = best_u;
            members.push_back(best);
            take(best);
        }
        const Op& first = in[members[0]];
        const bool single_diag = members.size() == 1 && (diag_like(first) || first.kind == OpKind::XPerm);
        if (single_diag) {
            res.push_back(first);
            continue;
        }
        Op blk;
        blk.kind = OpKind::RBlock;
        blk.qubits = S;
        std::sort(blk.qubits.begin(), blk.qubits.end());
        std::vector<Op> mops;
        for (int m : members)
            mops.push_back(in[m]);
        blk.prims = block_prims(blk.qubits, mops, width);
        blk.width = width;
        blk.first_gate = in[members.front()].first_gate;
        blk.last_gate = in[members.back()].last_gate;
        for (const Op& m : mops)
            blk.ngates += m.ngates;
        res.push_back(std::move(blk));
    }
    return res;
}

namespace {

struct Packer {
    const PlanOptions& opt;
    int n, n_local, K, Lmin;
    Plan& plan;
    std::vector<int> pos;          // logical -> physical
    // current pass
    std::vector<int> targets;      // physical tile-resident targets of the pass
    std::vector<qsv_op_desc> cur_ops;
    double cur_cost = 0;
    double cur_sweeps = 0;
    std::size_t cur_bytes = 0;
    // in-pass relabelling lookahead (single rank): the op sequence and the next op index
    const std::vector<Op>* seq = nullptr;
    std::size_t cursor = 0;
    int relabels = 0;

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

    // logical qubit -> index of its next tile use at or after `cursor` (large = none)
    std::vector<long> next_use() const {
        std::vector<long> nu(static_cast<std::size_t>(n), 1L << 40);
        int found = 0;
        for (std::size_t i = cursor; seq && i < seq->size() && i < cursor + 4096 && found < n; ++i) {
            const Op& o = (*seq)[i];
            if (o.kind != OpKind::Dense && o.kind != OpKind::XPerm && o.kind != OpKind::RBlock)
                continue;
            for (int q : o.qubits)
                if (nu[q] > static_cast<long>(i)) {
                    nu[q] = static_cast<long>(i);
                    ++found;
                }
        }
        return nu;
    }

    static constexpr long kNever = 1L << 40;

    // Chooses where every tile qubit lives after the pass (tile-bit relabel, applied
    // by the kernel after the pass's ops).  Policy: the L tile qubits needed soonest
    // take the low run (it is in every later tile for free); qubits with no further
    // use go back to their home slot when it is in the tile (so the final state needs
    // little or no restoring); the rest keep their slot when possible.
    bool relabel_tile(int L, const std::vector<int>& high, const std::vector<long>& nu, qsv_step_desc& s) {
        std::vector<int> slots;
        for (int p = 0; p < L; ++p)
            slots.push_back(p);
        for (int p : high)
            slots.push_back(p);
        const int ns = static_cast<int>(slots.size());
        std::vector<int> inv(static_cast<std::size_t>(n_local), -1);
        for (int q = 0; q < n; ++q)
            if (pos[q] < n_local)
                inv[pos[q]] = q;
        std::vector<int> qs;
        for (int p : slots)
            qs.push_back(inv[p]);
        auto slot_of = [&](int p) {
            for (int i = 0; i < ns; ++i)
                if (slots[i] == p)
                    return i;
            return -1;
        };
        std::vector<int> dest(static_cast<std::size_t>(ns), -1);   // by source slot index
        std::vector<char> taken(static_cast<std::size_t>(ns), 0);  // by destination slot index
        auto assign = [&](int src, int dst) {
            dest[src] = dst;
            taken[dst] = 1;
        };
        std::vector<int> order;
        for (int i = 0; i < ns; ++i)
            if (nu[qs[i]] < kNever)
                order.push_back(i);
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return nu[qs[x]] < nu[qs[y]]; });
        if (static_cast<int>(order.size()) > L)
            order.resize(static_cast<std::size_t>(L));
        auto is_home_of_finished = [&](int d) {
            for (int i = 0; i < ns; ++i)
                if (nu[qs[i]] >= kNever && qs[i] == slots[d])
                    return true;
            return false;
        };
        for (int i : order)
            if (i < L)
                assign(i, i);  // already low: stays
        for (int i : order) {
            if (dest[i] >= 0)
                continue;
            int pick = -1;
            for (int d = 0; d < L && pick < 0; ++d)
                if (!taken[d] && !is_home_of_finished(d))
                    pick = d;
            for (int d = 0; d < L && pick < 0; ++d)
                if (!taken[d])
                    pick = d;
            assign(i, pick);
        }
        for (int i = 0; i < ns; ++i) {
            if (dest[i] >= 0 || nu[qs[i]] < kNever)
                continue;
            const int h = qs[i] < n_local ? slot_of(qs[i]) : -1;
            if (h >= 0 && !taken[h])
                assign(i, h);
        }
        for (int i = 0; i < ns; ++i)
            if (dest[i] < 0 && !taken[i])
                assign(i, i);
        for (int i = 0; i < ns; ++i) {
            if (dest[i] >= 0)
                continue;
            // prefer a high slot for qubits with a later use, any free slot otherwise
            int pick = -1;
            for (int d = L; d < ns && pick < 0; ++d)
                if (!taken[d])
                    pick = d;
            for (int d = 0; d < ns && pick < 0; ++d)
                if (!taken[d])
                    pick = d;
            assign(i, pick);
        }
        bool moved = false;
        for (int i = 0; i < ns; ++i) {
            s.relabel[i] = dest[i];
            moved |= dest[i] != i;
        }
        if (!moved)
            return false;
        s.has_relabel = 1;
        for (int i = 0; i < ns; ++i)
            pos[qs[i]] = slots[dest[i]];
        return true;
    }

    int misplaced_local() const {
        int m = 0;
        for (int q = 0; q < n_local; ++q)
            m += pos[q] != q;
        return m;
    }

    // force: emit the pass even without ops (a pure relabel pass)
    void close_pass(bool force = false) {
        if (cur_ops.empty() && !force)
            return;
        const bool rl = opt.relabel && seq != nullptr;
        if (low_run(targets) < 0)
            throw std::logic_error("planner: infeasible pass tile");
        // with relabelling the low run stays at Lmin so the high slots can carry lookahead qubits
        const int L = (rl || std::getenv("QSV_PLAN_FIXED_L")) ? Lmin : low_run(targets);
        qsv_step_desc s{};
        s.kind = QSV_STEP_PASS;
        s.tile_k = K;
        std::vector<int> high;
        for (int q : targets)
            if (q >= L)
                high.push_back(q);
        const int want_high = std::min(K - L, QSV_MAX_HIGH);
        std::vector<long> nu;
        if (rl) {
            nu = next_use();
            // lookahead padding: the qubits needed soonest, so the relabel can bring them low
            std::vector<int> cand;
            for (int q = 0; q < n; ++q)
                if (pos[q] >= L && pos[q] < n_local && !contains(high, pos[q]) && nu[q] < kNever)
                    cand.push_back(q);
            std::stable_sort(cand.begin(), cand.end(), [&](int x, int y) { return nu[x] < nu[y]; });
            for (int q : cand)
                if (static_cast<int>(high.size()) < want_high)
                    high.push_back(pos[q]);
            // restore padding: finished qubits away from home, cheapest first (a qubit
            // whose current and home slots are both in the tile goes home this pass)
            for (;;) {
                int best = -1, best_cost = 3;
                for (int q = 0; q < n_local; ++q) {
                    if (pos[q] == q || nu[q] < kNever || pos[q] >= n_local)
                        continue;
                    int cost = 0;
                    for (int p : {pos[q], q})
                        cost += p >= L && !contains(high, p);
                    if (cost > 0 && cost < best_cost && static_cast<int>(high.size()) + cost <= want_high) {
                        best_cost = cost;
                        best = q;
                    }
                }
                if (best < 0)
                    break;
                for (int p : {pos[best], best})
                    if (p >= L && !contains(high, p))
                        high.push_back(p);
            }
        }
        // pad the tile with high qubits when targets don't fill it (K - L slots)
        for (int q = n_local - 1; static_cast<int>(high.size()) < want_high && q >= L; --q)
            if (!contains(high, q))
                high.push_back(q);
        std::sort(high.begin(), high.end());
        if (rl)
            relabels += relabel_tile(L, high, nu, s);
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
        cur_sweeps = 0;
        cur_bytes = 0;
    }

    int64_t put(const std::vector<Amp>& d) {
        const int64_t off = static_cast<int64_t>(plan.pool.size() / 2);
        for (const Amp& a : d) {
            plan.pool.push_back(a.real());
            plan.pool.push_back(a.imag());
        }
        return off;
    }

    // Physical slots of a register block: its qubits plus low-run padding.
    std::vector<int> block_slots(const Op& o) const {
        std::vector<int> phys;
        for (int q : o.qubits)
            phys.push_back(pos[q]);
        const std::size_t width = static_cast<std::size_t>(o.width);
        for (int p = 0; phys.size() < width && p < Lmin; ++p)
            if (!contains(phys, p))
                phys.push_back(p);
        return phys;
    }

    // physical positions the op needs inside the tile
    std::vector<int> tile_needs(const Op& o) const {
        if (o.kind == OpKind::Dense || o.kind == OpKind::XPerm) {
            std::vector<int> t;
            for (int q : o.qubits)
                t.push_back(pos[q]);
            return t;
        }
        if (o.kind == OpKind::RBlock)
            return block_slots(o);
        return {};
    }

    qsv_op_desc to_desc(const Op& o) {
        qsv_op_desc d{};
        for (int c : o.controls)
            d.ctrl_mask |= 1ull << pos[c];
        switch (o.kind) {
        case OpKind::Dense:
        case OpKind::XPerm:
        case OpKind::Diag:
            d.kind = o.kind == OpKind::Dense ? QSV_OP_DENSE : (o.kind == OpKind::Diag ? QSV_OP_DIAG : QSV_OP_XPERM);
            d.k = static_cast<int>(o.qubits.size());
            for (std::size_t i = 0; i < o.qubits.size(); ++i)
                d.qubits[i] = pos[o.qubits[i]];
            d.mat_off = put(o.data);
            break;
        case OpKind::ParPhase:
            d.kind = QSV_OP_PARPHASE;
            d.k = 0;
            for (int q : o.qubits)
                d.qmask |= 1ull << pos[q];
            d.mat_off = put(o.data);
            break;
        case OpKind::PhaseProd:
            d.kind = QSV_OP_PHASEPROD;
            d.k = 0;
            d.mat_off = put(o.data);
            d.prim_begin = static_cast<int>(plan.prims.size());
            for (const auto& f : o.factors) {
                qsv_prim_desc p{};
                p.kind = QSV_PRIM_FACTOR;
                p.a = pos[f.first];
                p.mat_off = put({f.second});
                plan.prims.push_back(p);
            }
            d.nprim = static_cast<int>(o.factors.size());
            break;
        case OpKind::RBlock: {
            d.kind = QSV_OP_RBLOCK;
            const std::vector<int> phys = block_slots(o);
            d.k = static_cast<int>(phys.size());
            for (int i = 0; i < d.k; ++i)
                d.qubits[i] = phys[i];
            d.prim_begin = static_cast<int>(plan.prims.size());
            // slot data is laid out over the block's own qubits (slots 0..|q|-1);
            // padded slots are untouched qubits, so DIAG16 entries just repeat.
            for (const Prim& pr : o.prims) {
                qsv_prim_desc p{};
                p.kind = pr.kind;
                p.a = pr.a;
                p.b = pr.b;
                if (pr.kind == QSV_PRIM_DIAG16) {
                    p.mat_off = put(pr.data);
                } else if (!pr.data.empty()) {
                    p.mat_off = put(pr.data);
                }
                plan.prims.push_back(p);
            }
            d.nprim = static_cast<int>(o.prims.size());
            break;
        }
        case OpKind::Fence:
        case OpKind::Swap:
            throw std::logic_error("to_desc: fence/swap have no device op");
        }
        return d;
    }

    static std::size_t blob_bytes(const Op& o) {
        std::size_t b = 96;
        switch (o.kind) {
        case OpKind::Dense: {
            const std::size_t D = std::size_t{1} << o.qubits.size();
            b += ((D * 4 + 15) & ~std::size_t{15}) + D * D * 16;
            break;
        }
        case OpKind::Diag: b += o.data.size() * 16 + 96; break;
        case OpKind::PhaseProd: b += 97 * 16 + o.factors.size() * 32; break;
        case OpKind::ParPhase: b += 32; break;
        case OpKind::RBlock:
            for (const Prim& p : o.prims)
                b += 8 + (p.kind == QSV_PRIM_U1 ? 64 : (p.kind == QSV_PRIM_CX ? 0 : 256)) + 16;
            break;
        default: break;
        }
        return b;
    }

    // Would `o` join the open pass without closing it?
    bool fits(const Op& o) const {
        if (cur_ops.empty() || o.kind == OpKind::Swap)
            return true;
        std::vector<int> need = targets;
        for (int p : tile_needs(o))
            if (!contains(need, p))
                need.push_back(p);
        const bool diag = o.kind == OpKind::Diag || o.kind == OpKind::PhaseProd || o.kind == OpKind::ParPhase;
        const double sw = diag && cur_ops.back().kind == QSV_OP_RBLOCK ? 0.5 : 1.0;
        return low_run(need) >= 0 && cur_cost + op_cost(o) <= opt.pass_budget && cur_sweeps + sw <= opt.max_sweeps &&
               cur_bytes + blob_bytes(o) <= 36 * 1024 && opt.multi_op_passes;
    }

    void add(const Op& o) {
        if (o.kind == OpKind::Swap) {
            // SWAP as a relabelling: the two logical qubits trade physical slots
            std::swap(pos[o.qubits[0]], pos[o.qubits[1]]);
            return;
        }
        std::vector<int> need = targets;
        for (int p : tile_needs(o))
            if (!contains(need, p))
                need.push_back(p);
        const double c = op_cost(o);
        const std::size_t b = blob_bytes(o);
        // SMEM sweeps: every op reads and writes the tile once; a diagonal op right after a
        // register block rides in its registers (JIT epilogue) and costs about half
        const bool diag = o.kind == OpKind::Diag || o.kind == OpKind::PhaseProd || o.kind == OpKind::ParPhase;
        const double sw = diag && !cur_ops.empty() && cur_ops.back().kind == QSV_OP_RBLOCK ? 0.5 : 1.0;
        const bool fits = low_run(need) >= 0 && (cur_ops.empty() || cur_cost + c <= opt.pass_budget) &&
                          (cur_ops.empty() || cur_sweeps + sw <= opt.max_sweeps) &&
                          cur_bytes + b <= 36 * 1024 && (opt.multi_op_passes || cur_ops.empty());
        if (!fits && !cur_ops.empty()) {
            close_pass();
            add(o);
            return;
        }
        if (low_run(need) < 0)
            throw std::logic_error("planner: op does not fit a tile (k too large for tile_k)");
        if (b > 36 * 1024)
            throw std::logic_error("planner: op too large for one pass");
        targets = need;
        cur_ops.push_back(to_desc(o));
        cur_cost += c;
        cur_sweeps += sw;
        cur_bytes += b;
    }

    // Swap two logical qubits (one global, one local).  Positions are read after the
    // open pass is closed, since closing it may relabel the tile.
    void swap_logical(int qg, int qv) {
        close_pass();
        swap(pos[qg], pos[qv]);
    }

    void swap(int g_phys, int v_phys) {
        close_pass();
        qsv_step_desc s{};
        s.kind = QSV_STEP_SWAP;
        s.swap_global = g_phys;
        s.swap_local = v_phys;
        // >= 4 chunks per swap so region passes can overlap the transfer (BBOP)
        s.chunk_log2 = std::max(0, std::min(opt.chunk_log2, n_local - 3));
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

// logical qubits an op needs local (inside the tile)
std::vector<int> local_needs(const Op& o) {
    if (o.kind == OpKind::Dense || o.kind == OpKind::XPerm || o.kind == OpKind::RBlock)
        return o.qubits;
    return {};
}

} // namespace

// CX(a,b) CX(b,a) CX(a,b) with nothing else on a or b in between is a SWAP of a and b:
// replaced by one Swap op (planned as a free relabelling).  Returns the number found.
int find_logical_swaps(std::vector<Op>& ops) {
    auto cx = [](const Op& o, int& c, int& t) {
        if (o.kind != OpKind::XPerm || o.controls.size() != 1 || o.qubits.size() != 1)
            return false;
        c = o.controls[0];
        t = o.qubits[0];
        return true;
    };
    int nq = 0;
    for (const Op& o : ops)
        for (int q : footprint(o))
            nq = std::max(nq, q + 1);
    std::vector<std::vector<int>> wire(static_cast<std::size_t>(nq));  // live op indices per qubit
    std::vector<char> dead(ops.size(), 0);
    int found = 0;
    for (int i = 0; i < static_cast<int>(ops.size()); ++i) {
        int c, t, c1, t1, c2, t2;
        if (cx(ops[i], c, t) && wire[c].size() >= 2 && wire[t].size() >= 2) {
            const int j = wire[c].back(), k = wire[c][wire[c].size() - 2];
            if (wire[t].back() == j && wire[t][wire[t].size() - 2] == k && cx(ops[j], c1, t1) && c1 == t &&
                t1 == c && cx(ops[k], c2, t2) && c2 == c && t2 == t) {
                Op sw;
                sw.kind = OpKind::Swap;
                sw.qubits = {std::min(c, t), std::max(c, t)};
                sw.first_gate = ops[k].first_gate;
                sw.last_gate = ops[i].last_gate;
                sw.ngates = 3;
                ops[k] = sw;
                dead[j] = 1;
                dead[i] = 1;
                wire[c].pop_back();
                wire[t].pop_back();
                ++found;
                continue;
            }
        }
        for (int q : footprint(ops[i]))
            wire[q].push_back(i);
    }
    std::vector<Op> out;
    out.reserve(ops.size());
    for (std::size_t i = 0; i < ops.size(); ++i)
        if (!dead[i])
            out.push_back(std::move(ops[i]));
    ops = std::move(out);
    return found;
}

// Relative time of a plan in units of one HBM round trip, from the B200
// measurements in profiles/ (r01): a relabel costs an extra SMEM sweep (~17 % of
// a pass) and runs shorter than 1 KB lose DRAM efficiency (~16 % at 512 B).
static double plan_time_model(const Plan& p) {
    double t = 0;
    for (const qsv_step_desc& s : p.steps) {
        if (s.kind != QSV_STEP_PASS) {
            // a swap moves 16 B per amplitude pair over NVLink (~685 GB/s P2P) against a
            // pass's 32 B per amplitude over HBM: ~2.4 pass-equivalents
            t += 2.4;
            continue;
        }
        const int L = s.tile_k - s.nhigh;
        int m = 0;
        while (m < s.nhigh && s.high[m] == L + m)
            ++m;
        const int run = L + m;
        t += 1.0 + (s.has_relabel ? 0.17 : 0.0) + (run <= 5 ? 0.16 : (run == 6 ? 0.05 : 0.0));
    }
    return t;
}

// Packs the final op list into passes (SMGP) and, across ranks, BBOP swaps.
// A multi-rank schedule: op indices (>= 0) and swaps of logical qubits (-1 - i into swaps).
struct Schedule {
    std::vector<int> order;
    std::vector<std::pair<int, int>> swaps;  // (logical global qubit, logical victim)
};

static void finish_plan(const Circuit& c, const PlanOptions& opt, Packer& pk, Plan& plan);

// Replays a multi-rank schedule with tile relabelling (lookahead over the scheduled order).
static Plan replay_schedule(const Circuit& c, const std::vector<Op>& ops, const Schedule& sch,
                            const PlanOptions& opt, Plan plan) {
    Packer pk(opt, c.n, plan.n_local, plan);
    std::vector<Op> seq;
    for (int e : sch.order)
        if (e >= 0)
            seq.push_back(ops[e]);
    pk.seq = &seq;
    std::size_t cur = 0;
    for (int e : sch.order) {
        if (e >= 0) {
            pk.cursor = cur++;
            pk.add(ops[e]);
        } else {
            pk.cursor = cur;
            const auto& sw = sch.swaps[static_cast<std::size_t>(-1 - e)];
            pk.swap_logical(sw.first, sw.second);
        }
    }
    pk.cursor = seq.size();
    finish_plan(c, opt, pk, plan);
    return plan;
}

static Plan pack_ops(const Circuit& c, const std::vector<Op>& ops, const PlanOptions& opt, Plan plan,
                     Schedule* sched = nullptr) {
    Packer pk(opt, c.n, plan.n_local, plan);
    const int nops = static_cast<int>(ops.size());
    if (plan.n_local == c.n && !sched) {
        pk.seq = &ops;
        for (std::size_t i = 0; i < ops.size(); ++i) {
            pk.cursor = i;
            pk.add(ops[i]);
        }
        pk.cursor = ops.size();
    } else if (plan.n_local == c.n) {
        // single rank, list-scheduled: the earliest ready op that fits the open pass
        // (commuting ops move up into it); the order is recorded for a relabel replay
        std::vector<int> npred(nops, 0);
        std::vector<std::vector<int>> succ(nops);
        std::vector<int> last(static_cast<std::size_t>(c.n), -1);
        for (int i = 0; i < nops; ++i) {
            std::vector<int> preds;
            for (int q : footprint(ops[i])) {
                if (last[q] >= 0 && !contains(preds, last[q]))
                    preds.push_back(last[q]);
                last[q] = i;
            }
            npred[i] = static_cast<int>(preds.size());
            for (int p : preds)
                succ[p].push_back(i);
        }
        std::vector<int> ready;
        for (int i = 0; i < nops; ++i)
            if (npred[i] == 0)
                ready.push_back(i);
        for (int done = 0; done < nops; ++done) {
            int pick = -1;
            for (int i : ready)
                if ((pick < 0 || i < pick) && pk.fits(ops[i]))
                    pick = i;
            if (pick < 0)
                pick = *std::min_element(ready.begin(), ready.end());
            ready.erase(std::find(ready.begin(), ready.end(), pick));
            sched->order.push_back(pick);
            pk.add(ops[pick]);
            for (int sI : succ[pick])
                if (--npred[sI] == 0)
                    ready.push_back(sI);
        }
    } else {
        // Local-first list scheduling over the dependency DAG (multi-GPU): run
        // every ready op whose tile qubits are all local; only when none is ready
        // bring the needed global qubits in with BBOP swaps, evicting the local
        // qubits with the fewest remaining uses (finished qubits first).
        std::vector<std::vector<int>> fp(nops);
        std::vector<int> npred(nops, 0);
        std::vector<std::vector<int>> succ(nops);
        std::vector<int> last(static_cast<std::size_t>(c.n), -1);
        for (int i = 0; i < nops; ++i) {
            fp[i] = footprint(ops[i]);
            std::vector<int> preds;
            for (int q : fp[i]) {
                if (last[q] >= 0 && !contains(preds, last[q]))
                    preds.push_back(last[q]);
                last[q] = i;
            }
            npred[i] = static_cast<int>(preds.size());
            for (int p : preds)
                succ[p].push_back(i);
        }
        std::vector<int> remaining(static_cast<std::size_t>(c.n), 0);
        for (int i = 0; i < nops; ++i)
            for (int q : local_needs(ops[i]))
                ++remaining[q];
        std::vector<int> ready;
        for (int i = 0; i < nops; ++i)
            if (npred[i] == 0)
                ready.push_back(i);
        auto is_local = [&](int i) {
            for (int q : local_needs(ops[i]))
                if (pk.pos[q] >= plan.n_local)
                    return false;
            return true;
        };
        int done = 0;
        std::vector<char> placed(static_cast<std::size_t>(nops), 0);
        const bool remaining_only = std::getenv("QSV_VICTIM_REMAINING") != nullptr;
        while (done < nops) {
            int pick = -1;
            // local ops that join the open pass first, then any local op; with
            // list_schedule off the ops keep program order (the SURVEY §8e cross-P
            // invariant: every P applies the same op sequence, bitwise equal results)
            if (opt.list_schedule) {
                for (int i : ready)
                    if (is_local(i) && (pick < 0 || i < pick) && pk.fits(ops[i]))
                        pick = i;
                if (pick < 0)
                    for (int i : ready)
                        if (is_local(i) && (pick < 0 || i < pick))
                            pick = i;
            }
            if (pick < 0) {
                pick = *std::min_element(ready.begin(), ready.end());
                const std::vector<int> need = local_needs(ops[pick]);
                for (int q : need) {
                    if (pk.pos[q] < plan.n_local)
                        continue;
                    // victims: local, not needed by this op, preferably outside the low
                    // run (contiguous swap chunks) and outside the open pass's tile;
                    // Belady: the qubit whose next local use is farthest, then the one
                    // with the fewest remaining uses, then the highest slot
                    std::vector<long long> next_need(static_cast<std::size_t>(c.n), 1LL << 40);
                    if (!remaining_only) {
                        int found = 0;
                        for (int i = 0; i < nops && found < c.n; ++i) {
                            if (placed[i])
                                continue;
                            for (int x : local_needs(ops[i]))
                                if (next_need[x] == (1LL << 40)) {
                                    next_need[x] = i;
                                    ++found;
                                }
                        }
                    }
                    // victim order: farthest next local use (Belady), then fewest remaining
                    // uses, then the highest slot — compared as a tuple, not a packed score
                    int best = -1;
                    for (int relax = 0; relax < 2 && best < 0; ++relax) {
                        auto key = [&](int l) {
                            return std::make_tuple(-static_cast<long long>(next_need[l]),
                                                   static_cast<long long>(remaining[l]), -pk.pos[l]);
                        };
                        for (int l = 0; l < c.n; ++l) {
                            const int p = pk.pos[l];
                            if (p >= plan.n_local || contains(need, l))
                                continue;
                            if (relax == 0 && (p < pk.Lmin || contains(pk.targets, p)))
                                continue;
                            if (best < 0 || key(l) < key(best))
                                best = l;
                        }
                    }
                    if (best < 0)
                        throw std::logic_error("planner: no swap victim available");
                    if (sched) {
                        sched->swaps.emplace_back(q, best);
                        sched->order.push_back(-static_cast<int>(sched->swaps.size()));
                    }
                    pk.swap_logical(q, best);
                }
            }
            ready.erase(std::find(ready.begin(), ready.end(), pick));
            placed[pick] = 1;
            if (sched)
                sched->order.push_back(pick);
            pk.add(ops[pick]);
            for (int q : local_needs(ops[pick]))
                --remaining[q];
            ++done;
            for (int sI : succ[pick])
                if (--npred[sI] == 0)
                    ready.push_back(sI);
        }
    }
    finish_plan(c, opt, pk, plan);
    return plan;
}

// Closes the last pass, restores the logical qubit order (relabel passes, then swaps
// and local slot swaps) so the final state is in the standard layout.
static void finish_plan(const Circuit& c, const PlanOptions& opt, Packer& pk, Plan& plan) {
    pk.close_pass();
    // 1. global slots first: one swap brings each global slot's own qubit home
    for (int G = plan.n_local; G < c.n; ++G) {
        if (pk.pos[G] == G)
            continue;
        int at = pk.pos[G];
        if (at >= plan.n_local) {  // it sits in another global slot: route through a local slot
            const int t = plan.n_local - 1;
            pk.swap(at, t);
            at = t;
        }
        pk.swap(G, at);
    }
    // 2. local slots: pure relabel passes (each fixes the cycles its tile holds)
    if (pk.seq != nullptr && opt.relabel) {
        if (std::getenv("QSV_PLAN_DEBUG"))
            std::fprintf(stderr, "plan: before restore passes=%zu misplaced=%d\n", plan.stats.passes, pk.misplaced_local());
        for (int guard = 0; guard < 64 && pk.misplaced_local() > 0; ++guard) {
            const int before = pk.misplaced_local();
            pk.close_pass(true);
            if (pk.misplaced_local() >= before)
                break;
        }
    }
    if (std::getenv("QSV_PLAN_DEBUG")) {
        int mis = 0;
        for (int q = 0; q < c.n; ++q) mis += pk.pos[q] != q;
        std::fprintf(stderr, "plan: passes=%zu relabels=%d misplaced=%d\n", plan.stats.passes, pk.relabels, mis);
    }
    // restore the logical qubit order so the final state is in standard layout
    for (int q = 0; q < c.n; ++q) {
        if (pk.pos[q] == q)
            continue;
        int other = -1;
        for (int r = 0; r < c.n; ++r)
            if (pk.pos[r] == q)
                other = r;
        const int a = pk.pos[q], b = q;  // physical slots to exchange
        if (a >= plan.n_local && b < plan.n_local) {
            pk.swap(a, b);
        } else if (b >= plan.n_local && a < plan.n_local) {
            pk.swap(b, a);
        } else if (a < plan.n_local && b < plan.n_local) {
            // local-local relabel: a SWAP of the two physical slots as one dense op
            Op sw;
            sw.kind = OpKind::Dense;
            sw.qubits = {q, other};
            sw.data.assign(16, Amp{0.0, 0.0});
            sw.data[0] = sw.data[15] = Amp{1.0, 0.0};
            sw.data[1 * 4 + 2] = sw.data[2 * 4 + 1] = Amp{1.0, 0.0};
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
}

// The DAGC stages: lower -> (logical swaps) -> parity peephole -> fuse -> register blocks.
// Returns false when `swaps` is requested but the circuit has no SWAP triple.
static bool build_ops(const Circuit& c, const PlanOptions& opt, bool swaps, Plan& plan, std::vector<Op>& ops) {
    ops = lower(c);
    plan.stats.ops_lowered = ops.size();
    if (swaps && find_logical_swaps(ops) == 0)
        return false;
    if (opt.fusion) {
        ops = reduce_parity(ops);
        PlanOptions fo = opt;
        fo.tile_k = std::min(opt.tile_k, plan.n_local);
        fo.min_low = std::min(opt.min_low, fo.tile_k);
        ops = fuse_ops(ops, fo);
    } else {
        std::vector<Op> kept;
        for (Op& o : ops)
            if (o.kind != OpKind::Fence)
                kept.push_back(std::move(o));
        ops = std::move(kept);
    }
    plan.stats.ops_fused = ops.size();
    const int K = std::min(opt.tile_k, plan.n_local);
    if (opt.fusion && opt.register_blocks && K >= std::max(opt.min_low, 5) && opt.multi_op_passes) {
        const int lo = std::min(opt.min_low, K);
        const int max_high = std::min(QSV_MAX_HIGH, K - lo);
        // with SWAPs relabelled any logical qubit may sit above the low run: blocks must
        // then fit the high slots on their own
        ops = swaps ? form_blocks(ops, 0, max_high, std::min(opt.rblock_k, std::max(max_high, 3)))
                    : form_blocks(ops, lo, max_high, opt.rblock_k);
    }
    plan.stats.ops_final = ops.size();
    plan.stats.cost_units = 0;
    plan.stats.max_dense_k = 0;
    for (const Op& o : ops) {
        plan.stats.cost_units += op_cost(o);
        if (o.kind == OpKind::Dense)
            plan.stats.max_dense_k = std::max(plan.stats.max_dense_k, static_cast<int>(o.qubits.size()));
    }
    return true;
}

// Packing candidates for one op list: {program order, list schedule} x {plain,
// relabelled}; the one the time model rates fastest wins.
static Plan choose_pack(const Circuit& c, std::vector<Op> ops, const PlanOptions& opt, const Plan& plan) {
    PlanOptions o_plain = opt;
    o_plain.relabel = 0;
    const bool single = plan.n_local == c.n;
    Schedule sch;
    Plan best = (opt.relabel == 2 && single) ? pack_ops(c, ops, opt, plan)
                                             : pack_ops(c, ops, o_plain, plan, single ? nullptr : &sch);
    if (!single && opt.relabel == 2)
        best = replay_schedule(c, ops, sch, opt, plan);
    auto consider = [&](auto&& make) {
        try {
            Plan alt = make();
            if (plan_time_model(alt) < plan_time_model(best))
                best = std::move(alt);
        } catch (const std::logic_error&) {
            // the blocks were formed for the caller's low run; a longer one may not fit
        }
    };
    Schedule lsch;
    if (single && opt.multi_op_passes && opt.list_schedule && opt.relabel != 2)  // list-scheduled order
        consider([&] { return pack_ops(c, ops, o_plain, plan, &lsch); });
    if (opt.relabel == 1) {
        // relabelled plans keep >= 1 KB HBM runs (min_low 6): 512-B runs cost ~16 %
        PlanOptions o_rl = opt;
        o_rl.min_low = std::max(opt.min_low, 6);
        // multi-rank: the list schedule (swaps included) is kept, only packing changes
        consider([&] { return single ? pack_ops(c, ops, o_rl, plan) : replay_schedule(c, ops, sch, o_rl, plan); });
        if (!lsch.order.empty())
            consider([&] { return replay_schedule(c, ops, lsch, o_rl, plan); });
    }
    best.fused = std::move(ops);
    return best;
}

Plan make_plan(const Circuit& c, const PlanOptions& opt) {
    c.validate();
    if (opt.fuse_k < 1 || opt.fuse_k > QSV_MAX_DENSE_K)
        throw std::invalid_argument("make_plan: fuse_k must be in [1, 5]");
    if (opt.tile_k < 1 || opt.tile_k > QSV_MAX_TILE_K)
        throw std::invalid_argument("make_plan: tile_k must be in [1, 12] (12 needs the specialised kernels)");
    if (opt.rblock_k != 3 && opt.rblock_k != 4)
        throw std::invalid_argument("make_plan: rblock_k must be 3 or 4");
    if (opt.relabel < 0 || opt.relabel > 2)
        throw std::invalid_argument("make_plan: relabel must be 0, 1 or 2");
    Plan plan;
    plan.n = c.n;
    plan.n_local = opt.n_local < 0 ? c.n : opt.n_local;
    if (plan.n_local < 1 || plan.n_local > c.n)
        throw std::invalid_argument("make_plan: n_local must be in [1, n]");
    plan.stats.gates_in = c.gate_count();
    std::vector<Op> ops;
    Plan base = plan;
    build_ops(c, opt, false, base, ops);
    Plan best = choose_pack(c, std::move(ops), opt, base);
    // 8-member register blocks as a candidate: circuits whose gates form 3-qubit clusters
    // (QAOA rings) pack into fewer passes that way (QAOA-30: 12 vs 14 passes, 81 vs 87 ms),
    // others into more (random-30: 55 vs 35).  An 8-member pass does less per HBM round trip
    // than the model's one unit, so the candidate must save >= 7 %: UCCSD-24 804 vs 831
    // passes measured 110 vs 105 ms, UCCSD-28 4273 vs 4439 passes 9.0 vs 8.7 s
    if (opt.rblock_k == 4 && opt.register_blocks && opt.fusion && !std::getenv("QSV_PLAN_NO_RB3")) {
        PlanOptions o3 = opt;
        o3.rblock_k = 3;
        Plan p3 = plan;
        std::vector<Op> ops3;
        build_ops(c, o3, false, p3, ops3);
        Plan alt = choose_pack(c, std::move(ops3), o3, p3);
        if (plan_time_model(alt) < 0.93 * plan_time_model(best))
            best = std::move(alt);
    }
    if (opt.logical_swaps < 0 || opt.logical_swaps > 2)
        throw std::invalid_argument("make_plan: logical_swaps must be 0, 1 or 2");
    if (opt.logical_swaps && opt.fusion) {
        // SWAP gates as relabellings: free when the final layout restore is cheap
        Plan sb = plan;
        try {
            if (build_ops(c, opt, true, sb, ops)) {
                Plan alt = choose_pack(c, std::move(ops), opt, sb);
                if (opt.logical_swaps == 2 || plan_time_model(alt) < plan_time_model(best))
                    best = std::move(alt);
            }
        } catch (const std::logic_error&) {
            if (opt.logical_swaps == 2)
                throw;  // forced: report why the relabelled plan is infeasible
        }
    }
    return best;
}

Circuit ops_to_circuit(int n, const std::vector<Op>& ops) {
    Circuit c(n, "fused");
    auto add_matrix = [&](std::vector<int> t, std::vector<int> ctl, std::vector<Amp> m) {
        const int k = static_cast<int>(t.size());
        c.add(Gate::unitary(GateMatrix(k, std::move(m)), std::move(t), std::move(ctl), "FUSED"));
    };
    auto add_phase = [&](std::vector<int> ctl, Amp e, int anchor) {
        // phase e on the all-ones pattern of ctl (global phase when ctl is empty)
        if (ctl.empty()) {
            add_matrix({anchor}, {}, {e, 0.0, 0.0, e});
            return;
        }
        const int t = ctl.back();
        ctl.pop_back();
        add_matrix({t}, ctl, {1.0, 0.0, 0.0, e});
    };
    for (const Op& o : ops) {
        switch (o.kind) {
        case OpKind::Fence: break;
        case OpKind::Swap:
            add_matrix({o.qubits[1]}, {o.qubits[0]}, {0.0, 1.0, 1.0, 0.0});
            add_matrix({o.qubits[0]}, {o.qubits[1]}, {0.0, 1.0, 1.0, 0.0});
            add_matrix({o.qubits[1]}, {o.qubits[0]}, {0.0, 1.0, 1.0, 0.0});
            break;
        case OpKind::Dense: add_matrix(o.qubits, o.controls, o.data); break;
        case OpKind::XPerm: add_matrix(o.qubits, o.controls, {0.0, 1.0, 1.0, 0.0}); break;
        case OpKind::Diag:
            if (o.qubits.empty()) {
                add_phase(o.controls, o.data[0], 0);
            } else {
                const std::size_t D = o.data.size();
                std::vector<Amp> m(D * D, Amp{0.0, 0.0});
                for (std::size_t i = 0; i < D; ++i)
                    m[i * D + i] = o.data[i];
                add_matrix(o.qubits, o.controls, m);
            }
            break;
        case OpKind::ParPhase: {
            // parity into the last mask qubit with a CX ladder, the phase, ladder back
            const std::vector<int>& m = o.qubits;
            if (m.empty()) {
                add_phase({}, o.data[0], 0);
                break;
            }
            for (std::size_t i = 0; i + 1 < m.size(); ++i)
                add_matrix({m[i + 1]}, {m[i]}, {0.0, 1.0, 1.0, 0.0});
            add_matrix({m.back()}, {}, {o.data[0], 0.0, 0.0, o.data[1]});
            for (std::size_t i = m.size() - 1; i-- > 0;)
                add_matrix({m[i + 1]}, {m[i]}, {0.0, 1.0, 1.0, 0.0});
            break;
        }
        case OpKind::PhaseProd:
            add_phase(o.controls, o.data[0], 0);
            for (const auto& f : o.factors) {
                std::vector<int> ctl = o.controls;
                ctl.push_back(f.first);
                add_phase(ctl, f.second, 0);
            }
            break;
        case OpKind::RBlock:
            for (const Prim& p : o.prims) {
                const std::vector<int>& s = o.qubits;
                if (p.kind == QSV_PRIM_U1 || p.kind == QSV_PRIM_U1R || p.kind == QSV_PRIM_U1I) {
                    add_matrix({s[p.a]}, {}, p.data);
                } else if (p.kind == QSV_PRIM_U2) {
                    add_matrix({s[p.a], s[p.b]}, {}, p.data);
                } else if (p.kind == QSV_PRIM_CX) {
                    add_matrix({s[p.b]}, {s[p.a]}, {0.0, 1.0, 1.0, 0.0});
                } else {
                    const int nb = static_cast<int>(s.size());
                    const std::size_t D = std::size_t{1} << nb;
                    std::vector<Amp> m(D * D, Amp{0.0, 0.0});
                    for (std::size_t i = 0; i < D; ++i)
                        m[i * D + i] = p.data[i];
                    add_matrix(s, {}, m);
                }
            }
            break;
        }
    }
    return c;
}

} // namespace qsim
