// RAII C++ wrappers over the C-ABI (include/qsv.h): the only way the qsim host
// library touches the GPU.  QSV_E_ARG maps to std::invalid_argument (the
// reference's parameter-error type, ref gate.cpp:24); every other failure to
// std::runtime_error carrying rank context.
#pragma once

#include "qsim/planner.hpp"
#include "qsim/statevector.hpp"
#include "qsv.h"

#include <memory>
#include <stdexcept>
#include <string>

namespace qsim {

// Throws for rc != QSV_OK.
void qsv_check(int rc, const std::string& what);

class DeviceContext {
  public:
    DeviceContext(int device = 0, int rank = 0, int nranks = 1, const void* comm_id = nullptr);
    ~DeviceContext();
    DeviceContext(const DeviceContext&) = delete;
    DeviceContext& operator=(const DeviceContext&) = delete;

    qsv_ctx* get() const { return ctx_; }
    int rank() const { return rank_; }
    int nranks() const { return nranks_; }
    void sync() const;
    // Process-wide context on device 0 used by the reference-API free functions.
    static DeviceContext& default_context();

  private:
    qsv_ctx* ctx_ = nullptr;
    int rank_ = 0, nranks_ = 1;
};

// One rank's shard of 2^n_local amplitudes in HBM.  The allocation is reported
// to memtrack by the constructing thread (ref memtrack.hpp:20-21).
class DeviceState {
  public:
    DeviceState(DeviceContext& ctx, int n_local);
    ~DeviceState();
    DeviceState(const DeviceState&) = delete;
    DeviceState& operator=(const DeviceState&) = delete;

    qsv_state* get() const { return st_; }
    int n_local() const { return n_local_; }
    Index size() const { return index_bit(n_local_); }
    void set_basis(Index global_index);
    void upload(const Amp* host, Index offset, Index count);
    void download(Amp* host, Index offset, Index count) const;
    double norm_sq() const;  // this shard only
    double max_abs_diff(const Amp* host_ref, Index offset, Index count) const;

  private:
    DeviceContext& ctx_;
    qsv_state* st_ = nullptr;
    int n_local_;
    std::size_t bytes_ = 0;
};

// A planned circuit uploaded to one GPU.
class Engine {
  public:
    Engine(DeviceContext& ctx, const Circuit& c, const PlanOptions& opt);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    const Plan& plan() const { return plan_; }
    // live figures: a background compile (PlanOptions::jit_async) counts once it is adopted
    double jit_seconds() const;
    int jit_kernels() const;
    // waits for a background compile and adopts it (no-op otherwise)
    void jit_wait() const;
    qsv_program* program() const { return prog_; }
    // Enqueues the whole circuit on the context stream (asynchronous).
    void run(DeviceState& st) const;

  private:
    DeviceContext& ctx_;
    Plan plan_;
    qsv_program* prog_ = nullptr;
};

} // namespace qsim
