// Definitions for qsim/device.hpp and qsim/kernels.hpp.
#include "qsim/device.hpp"
#include "qsim/kernels.hpp"
#include "qsim/memtrack.hpp"

#include <cstdio>
#include <mutex>

namespace qsim {

void qsv_check(int rc, const std::string& what) {
    if (rc == QSV_OK)
        return;
    const std::string msg = what + ": " + qsv_last_error();
    if (rc == QSV_E_ARG)
        throw std::invalid_argument(msg);
    throw std::runtime_error(msg + " (qsv code " + std::to_string(rc) + ")");
}

namespace {
// Every device allocation of the library for this context, as it happens, on the
// calling thread's memtrack rank/phase (ref memtrack.hpp:20-21): the instrumented
// BBOP memory audit.
void memtrack_hook(void*, int64_t delta, int) {
    if (delta >= 0)
        memtrack::on_alloc(static_cast<std::size_t>(delta));
    else
        memtrack::on_free(static_cast<std::size_t>(-delta));
}
} // namespace

DeviceContext::DeviceContext(int device, int rank, int nranks, const void* comm_id)
    : rank_(rank), nranks_(nranks) {
    qsv_check(qsv_ctx_create(device, rank, nranks, comm_id, &ctx_), "rank " + std::to_string(rank) + ": qsv_ctx_create");
    qsv_ctx_set_alloc_hook(ctx_, memtrack_hook, nullptr);
}

DeviceContext::~DeviceContext() { qsv_ctx_destroy(ctx_); }

void DeviceContext::sync() const { qsv_check(qsv_sync(ctx_), "qsv_sync"); }

DeviceContext& DeviceContext::default_context() {
    static std::once_flag once;
    static std::unique_ptr<DeviceContext> ctx;
    std::call_once(once, [] { ctx = std::make_unique<DeviceContext>(0, 0, 1, nullptr); });
    return *ctx;
}

DeviceState::DeviceState(DeviceContext& ctx, int n_local) : ctx_(ctx), n_local_(n_local) {
    qsv_check(qsv_state_alloc(ctx.get(), n_local, &st_, &bytes_), "qsv_state_alloc");  // memtrack via the hook
}

DeviceState::~DeviceState() { qsv_state_free(st_); }

void DeviceState::set_basis(Index global_index) {
    qsv_check(qsv_state_set_basis(st_, global_index), "qsv_state_set_basis");
}

void DeviceState::upload(const Amp* host, Index offset, Index count) {
    qsv_check(qsv_state_upload(st_, reinterpret_cast<const double*>(host), offset, count), "qsv_state_upload");
}

void DeviceState::download(Amp* host, Index offset, Index count) const {
    qsv_check(qsv_state_download(st_, reinterpret_cast<double*>(host), offset, count), "qsv_state_download");
}

double DeviceState::norm_sq() const {
    double v = 0;
    qsv_check(qsv_norm_sq(st_, &v), "qsv_norm_sq");
    return v;
}

double DeviceState::max_abs_diff(const Amp* host_ref, Index offset, Index count) const {
    double v = 0;
    qsv_check(qsv_max_abs_diff(st_, reinterpret_cast<const double*>(host_ref), offset, count, &v),
              "qsv_max_abs_diff");
    return v;
}

Engine::Engine(DeviceContext& ctx, const Circuit& c, const PlanOptions& opt) : ctx_(ctx) {
    PlanOptions o = opt;
    int m = 0;
    while ((1 << m) < ctx.nranks())
        ++m;
    o.n_local = c.n - m;
    plan_ = make_plan(c, o);
    qsv_check(qsv_program_create(ctx.get(), plan_.n, plan_.n_local, plan_.steps.data(),
                                 static_cast<int>(plan_.steps.size()), plan_.ops.data(),
                                 static_cast<int>(plan_.ops.size()), plan_.prims.data(),
                                 static_cast<int>(plan_.prims.size()), plan_.pool.data(),
                                 plan_.pool.size() / 2, &prog_),
              "qsv_program_create");
    if (o.jit && o.jit_max_kernels > 0) {
        double secs = 0;
        const int rc = o.jit_async ? qsv_program_jit_async(prog_, o.jit_max_kernels)
                                   : qsv_program_jit(prog_, o.jit_max_kernels, &secs);
        if (rc != QSV_OK) {
            static bool warned = false;
            if (!warned) {
                std::fprintf(stderr, "qsim: JIT unavailable, using the interpreter pass kernel (%s)\n",
                             qsv_last_error());
                warned = true;
            }
        }
    }
}

Engine::~Engine() { qsv_program_free(prog_); }

double Engine::jit_seconds() const {
    int done = 0;
    double s = 0;
    qsv_program_jit_wait(prog_, 0, &done, &s);
    return s;
}

int Engine::jit_kernels() const {
    int done = 0, k = 0, steps = 0;
    qsv_program_jit_wait(prog_, 0, &done, nullptr);
    qsv_program_jit_info(prog_, &k, &steps);
    return k;
}

void Engine::jit_wait() const {
    int done = 0;
    qsv_check(qsv_program_jit_wait(prog_, 1, &done, nullptr), "qsv_program_jit_wait");
}

void Engine::run(DeviceState& st) const { qsv_check(qsv_program_run(st.get(), prog_), "qsv_program_run"); }

// ------------------------------------------------------------------ kernels.hpp
namespace {

void check_targets(const StateVector& s, const Gate& g) {
    if (g.is_fence())
        throw std::invalid_argument("kernel: barrier has no matrix");
    for (int q : g.qubits())
        if (q < 0 || q >= s.n())
            throw std::invalid_argument("kernel: qubit " + std::to_string(q) + " out of range");
}

void run_single_gate(StateVector& s, const Gate& g) {
    DeviceContext& ctx = DeviceContext::default_context();
    DeviceState d(ctx, s.n());
    d.upload(s.data(), 0, s.size());
    std::vector<double> m;
    for (const Amp& a : g.matrix().entries()) {
        m.push_back(a.real());
        m.push_back(a.imag());
    }
    uint64_t cm = 0;
    for (int c : g.controls())
        cm |= 1ull << c;
    qsv_check(qsv_apply_fused(d.get(), g.arity(), g.targets().data(), cm, m.data()), "qsv_apply_fused");
    d.download(s.data(), 0, s.size());
}

} // namespace

void apply_single_naive(StateVector& s, const Gate& g) {
    check_targets(s, g);
    if (g.arity() != 1 || g.is_controlled())
        throw std::invalid_argument("apply_single_naive: needs a single-qubit gate without controls");
    run_single_gate(s, g);
}

void apply_single_grouped(StateVector& s, const Gate& g) {
    check_targets(s, g);
    if (g.arity() != 1 || g.is_controlled())
        throw std::invalid_argument("apply_single_grouped: needs a single-qubit gate without controls");
    run_single_gate(s, g);
}

void apply_controlled(StateVector& s, const Gate& g) {
    check_targets(s, g);
    if (g.arity() != 1 || g.controls().size() != 1)
        throw std::invalid_argument("apply_controlled: needs a single-qubit gate with one control");
    run_single_gate(s, g);
}

void apply_multi(StateVector& s, const Gate& g, int cap) {
    check_targets(s, g);
    if (g.arity() > cap)
        throw std::invalid_argument("apply_multi: arity " + std::to_string(g.arity()) +
                                    " exceeds the fusion cap " + std::to_string(cap));
    if (g.arity() > QSV_MAX_DENSE_K)
        throw std::invalid_argument("apply_multi: arity above the device limit (5)");
    run_single_gate(s, g);
}

void run_local(const Circuit& c, StateVector& s, int threads) {
    if (threads < 1)
        throw std::invalid_argument("run_local: threads must be >= 1");
    if (c.n != s.n())
        throw std::invalid_argument("run_local: circuit and state sizes differ");
    DeviceContext& ctx = DeviceContext::default_context();
    Engine eng(ctx, c, PlanOptions{});
    DeviceState d(ctx, s.n());
    d.upload(s.data(), 0, s.size());
    eng.run(d);
    d.download(s.data(), 0, s.size());
}

} // namespace qsim
