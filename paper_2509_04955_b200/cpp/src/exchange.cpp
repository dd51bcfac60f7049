// Definitions for qsim/exchange.hpp: one host thread per GPU rank.
#include "qsim/device.hpp"
#include "qsim/exchange.hpp"
#include "qsim/memtrack.hpp"

#include <chrono>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <exception>
#include <mutex>
#include <thread>

namespace qsim {

StateVector run_distributed(const Circuit& c, const PartitionPlan& plan, const std::vector<int>& devices,
                            DistributedReport* report, const PlanOptions& opt) {
    if (plan.n != c.n)
        throw std::invalid_argument("run_distributed: plan and circuit qubit counts differ");
    const int R = plan.ranks();
    std::vector<int> dev = devices;
    if (dev.empty())
        for (int r = 0; r < R; ++r)
            dev.push_back(r);
    if (static_cast<int>(dev.size()) != R)
        throw std::invalid_argument("run_distributed: need one device per rank");
    StateVector out(c.n);
    unsigned char id[QSV_NCCL_ID_BYTES] = {};
    if (R > 1)
        qsv_check(qsv_comm_unique_id(id), "qsv_comm_unique_id");
    PlanOptions o = opt;
    o.chunk_log2 = plan.b;
    o.nbuf = plan.buffers;
    std::mutex err_lock;
    std::exception_ptr err;
    std::string diagnostics;
    // live contexts, so that a failing rank can abort the others
    std::mutex ctx_lock;
    std::vector<qsv_ctx*> live(static_cast<std::size_t>(R), nullptr);
    auto abort_others = [&](int failed, const std::string& why) {
        std::lock_guard<std::mutex> g(ctx_lock);
        const std::string reason = "rank " + std::to_string(failed) + " failed: " + why;
        for (int q = 0; q < R; ++q)
            if (q != failed && live[static_cast<std::size_t>(q)])
                qsv_ctx_abort(live[static_cast<std::size_t>(q)], reason.c_str());
    };
    const char* inj = std::getenv("QSV_INJECT_FAIL_RANK");  // failure-injection test hook
    const int inject_rank = inj ? std::atoi(inj) : -1;
    std::vector<std::size_t> peaks(static_cast<std::size_t>(R), 0);
    std::size_t swaps = 0;
    const auto t0 = std::chrono::steady_clock::now();
    auto rank_main = [&](int r) {
        qsv_ctx* mine = nullptr;
        try {
            memtrack::register_thread(r);
            DeviceContext ctx(dev[r], r, R, R > 1 ? id : nullptr);
            mine = ctx.get();
            {
                std::lock_guard<std::mutex> g(ctx_lock);
                live[static_cast<std::size_t>(r)] = mine;
            }
            struct Unregister {  // before the context is destroyed
                std::mutex& m;
                std::vector<qsv_ctx*>& v;
                int r;
                ~Unregister() {
                    std::lock_guard<std::mutex> g(m);
                    v[static_cast<std::size_t>(r)] = nullptr;
                }
            } unregister{ctx_lock, live, r};
            Engine eng(ctx, c, o);
            DeviceState st(ctx, plan.l);
            st.set_basis(0);
            if (r == inject_rank)
                throw std::runtime_error("injected failure (QSV_INJECT_FAIL_RANK)");
            eng.run(st);
            ctx.sync();
            std::size_t stage = 0;
            qsv_check(qsv_ctx_staging_bytes(ctx.get(), &stage), "qsv_ctx_staging_bytes");
            memtrack::on_alloc(stage);
            peaks[r] = (std::size_t{16} << plan.l) + stage;
            if (r == 0)
                swaps = eng.plan().stats.swaps;
            memtrack::set_phase(memtrack::Phase::gather);
            st.download(out.data() + (static_cast<Index>(r) << plan.l), 0, index_bit(plan.l));
            memtrack::on_free(stage);
            memtrack::unregister_thread();
        } catch (const std::exception& ex) {
            abort_others(r, ex.what());
            std::lock_guard<std::mutex> g(err_lock);
            diagnostics += (diagnostics.empty() ? "" : "; ") + std::string("rank ") + std::to_string(r) + ": " +
                           ex.what();
            if (!err)
                err = std::current_exception();
        } catch (...) {
            abort_others(r, "unknown exception");
            std::lock_guard<std::mutex> g(err_lock);
            if (!err)
                err = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (int r = 0; r < R; ++r)
        th.emplace_back(rank_main, r);
    for (auto& t : th)
        t.join();
    if (err) {
        if (!diagnostics.empty())
            throw std::runtime_error("run_distributed: " + diagnostics);
        std::rethrow_exception(err);
    }
    if (report) {
        report->ranks = R;
        report->swaps = swaps;
        report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        report->peak_bytes = peaks;
    }
    return out;
}

} // namespace qsim
