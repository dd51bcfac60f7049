// Definitions for include/qsim_c.h: exception-free C facade over qsim.
#include "qsim_c.h"

#include "qsim/dag.hpp"
#include "qsim/device.hpp"
#include "qsim/exchange.hpp"
#include "qsim/fusion.hpp"
#include "qsim/partition.hpp"
#include "qsim/stagger.hpp"
#include "qsim/generators.hpp"
#include "qsim/memtrack.hpp"
#include "qsim/planner.hpp"
#include "qsim/qasm.hpp"

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

struct qsim_circuit {
    qsim::Circuit c;
};

struct qsim_engine {
    std::unique_ptr<qsim::DeviceContext> ctx;
    std::unique_ptr<qsim::DeviceState> st;
    std::unique_ptr<qsim::Engine> eng;
};

namespace {

thread_local std::string t_err;

template <typename F>
int guard(F&& f) {
    try {
        return f();
    } catch (const std::invalid_argument& e) {
        t_err = e.what();
        return QSV_E_ARG;
    } catch (const std::bad_alloc&) {
        t_err = "host allocation failed";
        return QSV_E_NOMEM;
    } catch (const std::exception& e) {
        t_err = e.what();
        return QSV_E_CUDA;
    } catch (...) {
        t_err = "unknown C++ exception";
        return QSV_E_CUDA;
    }
}

qsim::PlanOptions to_opts(const qsim_plan_opts* o) {
    qsim::PlanOptions p;
    if (!o)
        return p;
    p.tile_k = o->tile_k;
    p.min_low = o->min_low;
    p.fuse_k = o->fuse_k;
    p.fusion = o->fusion != 0;
    p.multi_op_passes = o->multi_op_passes != 0;
    p.register_blocks = o->register_blocks != 0;
    p.chunk_log2 = o->chunk_log2;
    p.nbuf = o->nbuf;
    p.pass_budget = o->pass_budget;
    p.rblock_k = o->rblock_k;
    p.jit = o->jit != 0;
    p.jit_async = o->jit == 2;
    p.relabel = o->relabel;
    p.max_sweeps = o->max_sweeps;
    p.list_schedule = o->list_schedule != 0;
    p.jit_max_kernels = o->jit_max_kernels;
    p.logical_swaps = o->logical_swaps;
    return p;
}

void fill_stats(const qsim::Plan& p, qsim_plan_stats* s) {
    s->gates_in = static_cast<int64_t>(p.stats.gates_in);
    s->ops_lowered = static_cast<int64_t>(p.stats.ops_lowered);
    s->ops_fused = static_cast<int64_t>(p.stats.ops_fused);
    s->ops_final = static_cast<int64_t>(p.stats.ops_final);
    s->passes = static_cast<int64_t>(p.stats.passes);
    s->swaps = static_cast<int64_t>(p.stats.swaps);
    s->cost_units = p.stats.cost_units;
    s->max_dense_k = p.stats.max_dense_k;
    s->n = p.n;
    s->n_local = p.n_local;
    s->nsteps = static_cast<int32_t>(p.steps.size());
}

std::vector<qsim::Amp> read_matrix(int k, const double* mat) {
    const std::size_t d = std::size_t{1} << k;
    std::vector<qsim::Amp> m(d * d);
    for (std::size_t i = 0; i < d * d; ++i)
        m[i] = qsim::Amp(mat[2 * i], mat[2 * i + 1]);
    return m;
}

#define REQUIRE(cond, msg)                  \
    do {                                    \
        if (!(cond)) {                      \
            t_err = (msg);                  \
            return QSV_E_ARG;               \
        }                                   \
    } while (0)

} // namespace

extern "C" {

const char* qsim_last_error(void) { return t_err.c_str(); }

void qsim_default_opts(qsim_plan_opts* out) {
    const qsim::PlanOptions p;
    std::memset(out, 0, sizeof(*out));
    out->tile_k = p.tile_k;
    out->min_low = p.min_low;
    out->fuse_k = p.fuse_k;
    out->fusion = p.fusion;
    out->multi_op_passes = p.multi_op_passes;
    out->register_blocks = p.register_blocks;
    out->chunk_log2 = p.chunk_log2;
    out->nbuf = p.nbuf;
    out->pass_budget = p.pass_budget;
    out->rblock_k = p.rblock_k;
    out->jit = p.jit ? (p.jit_async ? 2 : 1) : 0;
    out->relabel = p.relabel;
    out->max_sweeps = p.max_sweeps;
    out->list_schedule = p.list_schedule;
    out->jit_max_kernels = p.jit_max_kernels;
    out->logical_swaps = p.logical_swaps;
}

int qsim_circuit_generate(const char* spec, qsim_circuit** out) {
    return guard([&] {
        REQUIRE(spec && out, "qsim_circuit_generate: null argument");
        *out = new qsim_circuit{qsim::generate(spec)};
        return QSV_OK;
    });
}

int qsim_circuit_new(int n, qsim_circuit** out) {
    return guard([&] {
        REQUIRE(out, "qsim_circuit_new: null output");
        *out = new qsim_circuit{qsim::Circuit(n, "api")};
        return QSV_OK;
    });
}

int qsim_circuit_add(qsim_circuit* c, const char* mnemonic, const double* params, int nparams,
                     const int* qubits, int nqubits) {
    return guard([&] {
        REQUIRE(c && mnemonic && nparams >= 0 && nqubits >= 0, "qsim_circuit_add: bad argument");
        std::vector<double> ps(params, params + nparams);
        std::vector<int> qs(qubits, qubits + nqubits);
        c->c.add(qsim::gates::from_mnemonic(mnemonic, ps, qs));
        return QSV_OK;
    });
}

int qsim_circuit_add_unitary(qsim_circuit* c, int k, const int* targets, int nctrl, const int* controls,
                             const double* mat, const char* label) {
    return guard([&] {
        REQUIRE(c && targets && mat && k >= 1 && k <= 8 && nctrl >= 0 && (nctrl == 0 || controls),
                "qsim_circuit_add_unitary: bad argument");
        c->c.add(qsim::Gate::unitary(qsim::GateMatrix(k, read_matrix(k, mat)),
                                     std::vector<int>(targets, targets + k),
                                     std::vector<int>(controls, controls + nctrl), label ? label : "U"));
        return QSV_OK;
    });
}

int qsim_circuit_add_barrier(qsim_circuit* c, int nqubits, const int* qubits) {
    return guard([&] {
        REQUIRE(c && nqubits >= 0 && (nqubits == 0 || qubits), "qsim_circuit_add_barrier: bad argument");
        c->c.add(qsim::Gate::barrier(std::vector<int>(qubits, qubits + nqubits)));
        return QSV_OK;
    });
}

int qsim_circuit_info(const qsim_circuit* c, int* n, int64_t* nrecs, int64_t* pool_len) {
    return guard([&] {
        REQUIRE(c, "qsim_circuit_info: null circuit");
        int64_t pl = 0;
        for (const auto& g : c->c.gates)
            if (!g.is_fence())
                pl += static_cast<int64_t>(g.matrix().entries().size());
        if (n) *n = c->c.n;
        if (nrecs) *nrecs = static_cast<int64_t>(c->c.gates.size());
        if (pool_len) *pool_len = pl;
        return QSV_OK;
    });
}

int qsim_circuit_export(const qsim_circuit* c, qsim_gate_rec* recs, double* pool) {
    return guard([&] {
        REQUIRE(c && recs && pool, "qsim_circuit_export: null argument");
        int64_t off = 0;
        for (std::size_t i = 0; i < c->c.gates.size(); ++i) {
            const qsim::Gate& g = c->c.gates[i];
            qsim_gate_rec r{};
            REQUIRE(g.targets().size() <= 8 && g.controls().size() <= 8, "qsim_circuit_export: gate too wide");
            if (!g.is_fence()) {
                r.arity = g.arity();
                r.nctrl = static_cast<int32_t>(g.controls().size());
                for (std::size_t t = 0; t < g.targets().size(); ++t) r.targets[t] = g.targets()[t];
                for (std::size_t t = 0; t < g.controls().size(); ++t) r.controls[t] = g.controls()[t];
                r.mat_off = off;
                for (const auto& a : g.matrix().entries()) {
                    pool[2 * off] = a.real();
                    pool[2 * off + 1] = a.imag();
                    ++off;
                }
            }
            recs[i] = r;
        }
        return QSV_OK;
    });
}

int qsim_circuit_parse_qasm(const char* text, int64_t len, qsim_circuit** out, int* line, int* col) {
    if (line)
        *line = 0;
    if (col)
        *col = 0;
    return guard([&] {
        REQUIRE(out && len >= 0 && (text || len == 0), "qsim_circuit_parse_qasm: bad argument");
        try {
            *out = new qsim_circuit{qsim::parse_qasm(std::string_view(text ? text : "", static_cast<std::size_t>(len)))};
        } catch (const qsim::QasmError& e) {
            if (line)
                *line = e.line();
            if (col)
                *col = e.column();
            throw;
        }
        return QSV_OK;
    });
}

int qsim_circuit_emit_qasm(const qsim_circuit* c, int matrix_export, char* buf, int64_t cap, int64_t* needed) {
    return guard([&] {
        REQUIRE(c && needed && cap >= 0 && (buf || cap == 0), "qsim_circuit_emit_qasm: bad argument");
        qsim::QasmEmitOptions o;
        o.matrix_export = matrix_export != 0;
        const std::string s = qsim::emit_qasm(c->c, o);
        *needed = static_cast<int64_t>(s.size());
        if (cap > 0) {
            const std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
            std::memcpy(buf, s.data(), n);
            buf[n] = '\0';
        }
        return QSV_OK;
    });
}

int qsim_circuit_slice(const qsim_circuit* c, int64_t begin, int64_t end, qsim_circuit** out) {
    return guard([&] {
        REQUIRE(c && out && begin >= 0 && begin <= end &&
                    end <= static_cast<int64_t>(c->c.gates.size()),
                "qsim_circuit_slice: bad range");
        qsim::Circuit s(c->c.n, c->c.source + "[slice]");
        for (int64_t i = begin; i < end; ++i)
            s.gates.push_back(c->c.gates[i]);
        *out = new qsim_circuit{std::move(s)};
        return QSV_OK;
    });
}

int qsim_circuit_fused(const qsim_circuit* c, const qsim_plan_opts* opts, qsim_circuit** out) {
    return guard([&] {
        REQUIRE(c && out, "qsim_circuit_fused: null argument");
        const qsim::PlanOptions o = to_opts(opts);
        std::vector<qsim::Op> ops = qsim::lower(c->c);
        if (o.fusion) {
            ops = qsim::reduce_parity(ops);
            ops = qsim::fuse_ops(ops, o);
            if (o.register_blocks)
                ops = qsim::form_blocks(ops, o.min_low, std::max(o.tile_k - o.min_low, 0), o.rblock_k);
        }
        std::vector<qsim::Op> kept;
        for (auto& op : ops)
            if (op.kind != qsim::OpKind::Fence)
                kept.push_back(op);
        *out = new qsim_circuit{qsim::ops_to_circuit(c->c.n, kept)};
        return QSV_OK;
    });
}

int qsim_circuit_plan(const qsim_circuit* c, const qsim_plan_opts* opts, int n_local, int rank,
                      qsim_plan_stats* stats) {
    return guard([&] {
        REQUIRE(c, "qsim_circuit_plan: null circuit");
        qsim::PlanOptions o = to_opts(opts);
        o.n_local = n_local;
        const qsim::Plan p = qsim::make_plan(c->c, o);
        const int rc = qsv_program_validate(p.n, p.n_local, rank, p.steps.data(),
                                            static_cast<int>(p.steps.size()), p.ops.data(),
                                            static_cast<int>(p.ops.size()), p.prims.data(),
                                            static_cast<int>(p.prims.size()), p.pool.data(), p.pool.size() / 2);
        if (rc != QSV_OK) {
            t_err = std::string("plan rejected by the device compiler: ") + qsv_last_error();
            return rc;
        }
        if (stats)
            fill_stats(p, stats);
        return QSV_OK;
    });
}

void qsim_circuit_free(qsim_circuit* c) { delete c; }

int qsim_plan_export(const qsim_circuit* c, const qsim_plan_opts* opts, int n_local, int* nsteps, int* nops,
                     int* nprims, int64_t* pool_len, void* steps, void* ops, void* prims, double* pool) {
    return guard([&] {
        REQUIRE(c && nsteps && nops && nprims && pool_len, "qsim_plan_export: null argument");
        qsim::PlanOptions o = to_opts(opts);
        o.n_local = n_local;
        const qsim::Plan p = qsim::make_plan(c->c, o);
        // in: capacities of the non-null arrays; out: the sizes the plan needs
        const bool fits = (!steps || static_cast<size_t>(std::max(*nsteps, 0)) >= p.steps.size()) &&
                          (!ops || static_cast<size_t>(std::max(*nops, 0)) >= p.ops.size()) &&
                          (!prims || static_cast<size_t>(std::max(*nprims, 0)) >= p.prims.size()) &&
                          (!pool || static_cast<size_t>(std::max<int64_t>(*pool_len, 0)) >= p.pool.size() / 2);
        *nsteps = static_cast<int>(p.steps.size());
        *nops = static_cast<int>(p.ops.size());
        *nprims = static_cast<int>(p.prims.size());
        *pool_len = static_cast<int64_t>(p.pool.size() / 2);
        REQUIRE(fits, "qsim_plan_export: a buffer is smaller than the plan (the needed sizes were written back)");
        if (steps)
            std::memcpy(steps, p.steps.data(), p.steps.size() * sizeof(qsv_step_desc));
        if (ops)
            std::memcpy(ops, p.ops.data(), p.ops.size() * sizeof(qsv_op_desc));
        if (prims)
            std::memcpy(prims, p.prims.data(), p.prims.size() * sizeof(qsv_prim_desc));
        if (pool)
            std::memcpy(pool, p.pool.data(), p.pool.size() * sizeof(double));
        return QSV_OK;
    });
}

int qsim_engine_create(const qsim_circuit* c, const qsim_plan_opts* opts, int device, int rank, int nranks,
                       const void* comm_id, qsim_engine** out) {
    return guard([&] {
        REQUIRE(c && out, "qsim_engine_create: null argument");
        auto e = std::make_unique<qsim_engine>();
        e->ctx = std::make_unique<qsim::DeviceContext>(device, rank, nranks, comm_id);
        e->eng = std::make_unique<qsim::Engine>(*e->ctx, c->c, to_opts(opts));
        e->st = std::make_unique<qsim::DeviceState>(*e->ctx, e->eng->plan().n_local);
        *out = e.release();
        return QSV_OK;
    });
}

void qsim_engine_free(qsim_engine* e) {
    if (!e)
        return;
    e->eng.reset();
    e->st.reset();
    e->ctx.reset();
    delete e;
}

int qsim_engine_stats(qsim_engine* e, qsim_plan_stats* out) {
    return guard([&] {
        REQUIRE(e && out, "qsim_engine_stats: null argument");
        fill_stats(e->eng->plan(), out);
        return QSV_OK;
    });
}

void* qsim_engine_stream(qsim_engine* e) { return e ? qsv_ctx_stream(e->ctx->get()) : nullptr; }
void* qsim_engine_qsv_state(qsim_engine* e) { return e ? e->st->get() : nullptr; }
void* qsim_engine_qsv_program(qsim_engine* e) { return e ? e->eng->program() : nullptr; }
void* qsim_engine_qsv_ctx(qsim_engine* e) { return e ? e->ctx->get() : nullptr; }

int qsim_engine_set_basis(qsim_engine* e, uint64_t idx) {
    return guard([&] {
        REQUIRE(e, "qsim_engine_set_basis: null engine");
        e->st->set_basis(idx);
        return QSV_OK;
    });
}

int qsim_engine_upload(qsim_engine* e, const double* amps, uint64_t offset, uint64_t count) {
    return guard([&] {
        REQUIRE(e, "qsim_engine_upload: null engine");
        qsim::qsv_check(qsv_state_upload(e->st->get(), amps, offset, count), "qsv_state_upload");
        return QSV_OK;
    });
}

int qsim_engine_download(qsim_engine* e, double* amps, uint64_t offset, uint64_t count) {
    return guard([&] {
        REQUIRE(e, "qsim_engine_download: null engine");
        qsim::qsv_check(qsv_state_download(e->st->get(), amps, offset, count), "qsv_state_download");
        return QSV_OK;
    });
}

int qsim_engine_download_async(qsim_engine* e, double* amps, uint64_t offset, uint64_t count) {
    return guard([&] {
        REQUIRE(e, "qsim_engine_download_async: null engine");
        qsim::qsv_check(qsv_state_download_async(e->st->get(), amps, offset, count), "qsv_state_download_async");
        return QSV_OK;
    });
}

int qsim_engine_run(qsim_engine* e) {
    return guard([&] {
        REQUIRE(e, "qsim_engine_run: null engine");
        e->eng->run(*e->st);
        return QSV_OK;
    });
}

int qsim_engine_sync(qsim_engine* e) {
    return guard([&] {
        REQUIRE(e, "qsim_engine_sync: null engine");
        e->ctx->sync();
        return QSV_OK;
    });
}

int qsim_engine_time(qsim_engine* e, int iters, int64_t basis, float* ms) {
    return guard([&] {
        REQUIRE(e && ms, "qsim_engine_time: null argument");
        qsim::qsv_check(qsv_program_time(e->st->get(), e->eng->program(), iters, basis, ms), "qsv_program_time");
        return QSV_OK;
    });
}

int qsim_engine_norm_sq(qsim_engine* e, double* out) {
    return guard([&] {
        REQUIRE(e && out, "qsim_engine_norm_sq: null argument");
        *out = e->st->norm_sq();
        return QSV_OK;
    });
}

int qsim_engine_max_abs_diff(qsim_engine* e, const double* ref, uint64_t offset, uint64_t count, double* out) {
    return guard([&] {
        REQUIRE(e && out, "qsim_engine_max_abs_diff: null argument");
        qsim::qsv_check(qsv_max_abs_diff(e->st->get(), ref, offset, count, out), "qsv_max_abs_diff");
        return QSV_OK;
    });
}

int qsim_engine_check_qft(qsim_engine* e, uint64_t x, double* out) {
    return guard([&] {
        REQUIRE(e && out, "qsim_engine_check_qft: null argument");
        qsim::qsv_check(qsv_check_qft_basis(e->st->get(), e->eng->plan().n, x, out), "qsv_check_qft_basis");
        return QSV_OK;
    });
}

int qsim_engine_digest(qsim_engine* e, uint64_t* out) {
    return guard([&] {
        REQUIRE(e && out, "qsim_engine_digest: null argument");
        qsim::qsv_check(qsv_state_digest(e->st->get(), out), "qsv_state_digest");
        return QSV_OK;
    });
}

int qsim_engine_nsteps(qsim_engine* e) { return e ? static_cast<int>(e->eng->plan().steps.size()) : 0; }

int qsim_engine_step_info(qsim_engine* e, int i, int* kind, int* nops, double* hbm_bytes, double* flops,
                          double* nvl_bytes) {
    return guard([&] {
        REQUIRE(e && i >= 0 && i < static_cast<int>(e->eng->plan().steps.size()), "qsim_engine_step_info: bad index");
        const qsv_step_desc& s = e->eng->plan().steps[i];
        if (kind) *kind = s.kind;
        if (nops) *nops = s.kind == QSV_STEP_PASS ? s.op_count : 0;
        qsim::qsv_check(qsv_program_step_cost(e->eng->program(), i, hbm_bytes, flops, nvl_bytes),
                        "qsv_program_step_cost");
        return QSV_OK;
    });
}

int qsim_engine_profile(qsim_engine* e, float* ms) {
    return guard([&] {
        REQUIRE(e && ms, "qsim_engine_profile: null argument");
        qsim::qsv_check(qsv_program_profile(e->st->get(), e->eng->program(), ms), "qsv_program_profile");
        return QSV_OK;
    });
}

int64_t qsim_dag_edges(const qsim_circuit* c, int32_t* pairs, int64_t cap) {
    if (!c) {
        t_err = "qsim_dag_edges: null circuit";
        return QSV_E_ARG;
    }
    int64_t n = 0;
    const int rc = guard([&] {
        const qsim::DepGraph g = qsim::build_dag(c->c);
        for (const auto& e : g.edges()) {
            if (pairs && n < cap) {
                pairs[2 * n] = e.first;
                pairs[2 * n + 1] = e.second;
            }
            ++n;
        }
        return QSV_OK;
    });
    return rc == QSV_OK ? n : rc;
}

int qsim_gate_cost(const qsim_circuit* c, int64_t i, int n, double* out) {
    return guard([&] {
        REQUIRE(c && out && i >= 0 && i < static_cast<int64_t>(c->c.gates.size()), "qsim_gate_cost: bad argument");
        *out = qsim::gate_cost(c->c.gates[i], n);
        return QSV_OK;
    });
}

int qsim_contract(const qsim_circuit* c, int cap, qsim_circuit** out, qsim_fusion_stats* stats) {
    return guard([&] {
        REQUIRE(c && out, "qsim_contract: null argument");
        auto [res, plan, st] = qsim::contract(c->c, cap);
        (void)plan;
        if (stats) {
            stats->gates_before = static_cast<int64_t>(st.gates_before);
            stats->gates_after = static_cast<int64_t>(st.gates_after);
            stats->merges_same_qubit = static_cast<int64_t>(st.merges_same_qubit);
            stats->merges_cu = static_cast<int64_t>(st.merges_cu);
            stats->merges_kronecker = static_cast<int64_t>(st.merges_kronecker);
            stats->passes = static_cast<int64_t>(st.passes);
            stats->compression_ratio = st.compression_ratio;
            stats->cost_before = st.cost_before;
            stats->cost_after = st.cost_after;
        }
        *out = new qsim_circuit{std::move(res)};
        return QSV_OK;
    });
}

int qsim_plan_groups(const qsim_circuit* c, int S, int local_qubits, int32_t* group_of) {
    int ng = 0;
    const int rc = guard([&] {
        REQUIRE(c && group_of, "qsim_plan_groups: null argument");
        auto [groups, residual] = qsim::plan_groups(c->c, qsim::build_dag(c->c), S, local_qubits);
        for (std::size_t i = 0; i < c->c.gates.size(); ++i)
            group_of[i] = -1;
        for (std::size_t g = 0; g < groups.size(); ++g)
            for (int gi : groups[g].gates)
                group_of[gi] = static_cast<int32_t>(g);
        ng = static_cast<int>(groups.size());
        return QSV_OK;
    });
    return rc == QSV_OK ? ng : rc;
}

int qsim_stagger_schedule(int G, int S, int32_t* table) {
    return guard([&] {
        REQUIRE(table, "qsim_stagger_schedule: null table");
        const auto t = qsim::stagger_schedule(G, S);
        for (int g = 0; g < G; ++g)
            for (int tau = 0; tau < S; ++tau)
                table[g * S + tau] = t[g][tau];
        return QSV_OK;
    });
}

int qsim_execute_staggered(const qsim_circuit* c, int S, int local_qubits, int group, double* amps) {
    return guard([&] {
        REQUIRE(c && amps, "qsim_execute_staggered: null argument");
        auto [groups, residual] = qsim::plan_groups(c->c, qsim::build_dag(c->c), S, local_qubits);
        REQUIRE(group >= 0 && group < static_cast<int>(groups.size()), "qsim_execute_staggered: no such group");
        qsim::StateVector sv(c->c.n);
        std::memcpy(static_cast<void*>(sv.data()), amps, sizeof(qsim::Amp) * sv.size());
        qsim::execute_staggered(sv, c->c, groups[group], 1);
        std::memcpy(amps, sv.data(), sizeof(qsim::Amp) * sv.size());
        return QSV_OK;
    });
}

int qsim_classify_gate(const qsim_circuit* c, int64_t i, int m, int* out) {
    return guard([&] {
        REQUIRE(c && out && i >= 0 && i < static_cast<int64_t>(c->c.gates.size()), "qsim_classify_gate: bad argument");
        const qsim::PartitionPlan p(c->c.n, m, 0, 2);
        *out = static_cast<int>(qsim::classify_gate(c->c.gates[i], p));
        return QSV_OK;
    });
}

int qsim_peer_rank(int r, int t, int l, int* out) {
    return guard([&] {
        REQUIRE(out, "qsim_peer_rank: null output");
        *out = qsim::peer_rank(r, t, l);
        return QSV_OK;
    });
}

int qsim_run_distributed(const qsim_circuit* c, int m, int b, int buffers, const int* devices,
                         const qsim_plan_opts* opts, double* amps, qsim_dist_report* report) {
    return guard([&] {
        REQUIRE(c && amps, "qsim_run_distributed: null argument");
        const qsim::PartitionPlan p(c->c.n, m, b, buffers);
        std::vector<int> dev;
        if (devices)
            dev.assign(devices, devices + p.ranks());
        qsim::DistributedReport rep;
        qsim::StateVector sv = qsim::run_distributed(c->c, p, dev, &rep, to_opts(opts));
        std::memcpy(amps, sv.data(), sizeof(qsim::Amp) * sv.size());
        if (report) {
            report->ranks = rep.ranks;
            report->swaps = static_cast<int64_t>(rep.swaps);
            report->seconds = rep.seconds;
            for (std::size_t r = 0; r < rep.peak_bytes.size() && r < 64; ++r)
                report->peak_bytes[r] = static_cast<int64_t>(rep.peak_bytes[r]);
        }
        return QSV_OK;
    });
}

int qsim_run_distributed_files(const qsim_circuit* c, int m, int b, int buffers, const int* devices,
                               const qsim_plan_opts* opts, const char* dir, qsim_dist_report* report) {
    return guard([&] {
        REQUIRE(c && dir, "qsim_run_distributed_files: null argument");
        const qsim::PartitionPlan p(c->c.n, m, b, buffers);
        std::vector<int> dev;
        if (devices)
            dev.assign(devices, devices + p.ranks());
        qsim::DistributedReport rep;
        qsim::run_distributed_to_files(c->c, p, dir, dev, &rep, to_opts(opts));
        if (report) {
            report->ranks = rep.ranks;
            report->swaps = static_cast<int64_t>(rep.swaps);
            report->seconds = rep.seconds;
            for (std::size_t r = 0; r < rep.peak_bytes.size() && r < 64; ++r)
                report->peak_bytes[r] = static_cast<int64_t>(rep.peak_bytes[r]);
        }
        return QSV_OK;
    });
}

void qsim_memtrack_script(const long long* ops, int nops, int nranks, unsigned long long* peaks) {
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

int qsim_engine_jit_wait(qsim_engine* e) {
    return guard([&] {
        REQUIRE(e, "qsim_engine_jit_wait: null engine");
        e->eng->jit_wait();
        return QSV_OK;
    });
}

int qsim_engine_jit_info(qsim_engine* e, int* kernels, double* seconds) {
    return guard([&] {
        REQUIRE(e, "qsim_engine_jit_info: null engine");
        if (kernels) *kernels = e->eng->jit_kernels();
        if (seconds) *seconds = e->eng->jit_seconds();
        return QSV_OK;
    });
}

int qsim_run_local_host(const qsim_circuit* c, const qsim_plan_opts* opts, double* amps) {
    return guard([&] {
        REQUIRE(c && amps, "qsim_run_local_host: null argument");
        qsim::DeviceContext& ctx = qsim::DeviceContext::default_context();
        qsim::Engine eng(ctx, c->c, to_opts(opts));
        qsim::DeviceState st(ctx, c->c.n);
        const qsim::Index N = qsim::index_bit(c->c.n);
        st.upload(reinterpret_cast<const qsim::Amp*>(amps), 0, N);
        eng.run(st);
        st.download(reinterpret_cast<qsim::Amp*>(amps), 0, N);
        return QSV_OK;
    });
}

} // extern "C"
