// Definitions for qsim/exchange.hpp: one host thread per GPU rank.
#include "qsim/device.hpp"
#include "qsim/exchange.hpp"
#include "qsim/memtrack.hpp"

#include <chrono>
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
    std::vector<std::size_t> peaks(static_cast<std::size_t>(R), 0);
    std::size_t swaps = 0;
    const auto t0 = std::chrono::steady_clock::now();
    auto rank_main = [&](int r) {
        try {
            memtrack::register_thread(r);
            DeviceContext ctx(dev[r], r, R, R > 1 ? id : nullptr);
            Engine eng(ctx, c, o);
            DeviceState st(ctx, plan.l);
            st.set_basis(0);
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
        } catch (...) {
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
    if (err)
        std::rethrow_exception(err);
    if (report) {
        report->ranks = R;
        report->swaps = swaps;
        report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        report->peak_bytes = peaks;
    }
    return out;
}

} // namespace qsim
