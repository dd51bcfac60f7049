// Definitions for qsim/exchange.hpp: one host thread per GPU rank.
#include "qsim/device.hpp"
#include "qsim/exchange.hpp"
#include "qsim/memtrack.hpp"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <functional>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <exception>
#include <mutex>
#include <thread>

namespace qsim {

std::size_t gather_cap_bytes() {
    const char* e = std::getenv("QSV_GATHER_CAP_GIB");
    const double gib = e ? std::atof(e) : 64.0;
    return static_cast<std::size_t>(gib * 1073741824.0);
}

namespace {

// One rank's result sink: gather into the host state (rank r's slice) or a shard file.
using Sink = std::function<void(int r, DeviceState& st)>;

void run_ranks(const Circuit& c, const PartitionPlan& plan, const std::vector<int>& devices,
               DistributedReport* report, const PlanOptions& opt, const Sink& sink);

} // namespace

StateVector run_distributed(const Circuit& c, const PartitionPlan& plan, const std::vector<int>& devices,
                            DistributedReport* report, const PlanOptions& opt) {
    if (plan.n != c.n)
        throw std::invalid_argument("run_distributed: plan and circuit qubit counts differ");
    const double bytes = 16.0 * std::ldexp(1.0, c.n);
    if (bytes > static_cast<double>(gather_cap_bytes()))
        throw std::invalid_argument("run_distributed: gathering 2^" + std::to_string(c.n) + " amplitudes (" +
                                    std::to_string(static_cast<long long>(bytes / 1073741824.0)) +
                                    " GiB) exceeds the single-host cap QSV_GATHER_CAP_GIB; use "
                                    "run_distributed_to_files (per-rank shard files, SPEC:421)");
    StateVector out(c.n);
    run_ranks(c, plan, devices, report, opt, [&](int r, DeviceState& st) {
        memtrack::set_phase(memtrack::Phase::gather);
        st.download(out.data() + (static_cast<Index>(r) << plan.l), 0, index_bit(plan.l));
    });
    return out;
}

void run_distributed_to_files(const Circuit& c, const PartitionPlan& plan, const std::string& dir,
                              const std::vector<int>& devices, DistributedReport* report, const PlanOptions& opt) {
    if (plan.n != c.n)
        throw std::invalid_argument("run_distributed_to_files: plan and circuit qubit counts differ");
    if (dir.empty())
        throw std::invalid_argument("run_distributed_to_files: empty output directory");
    const int R = plan.ranks();
    std::vector<std::string> names(static_cast<std::size_t>(R));
    for (int r = 0; r < R; ++r)
        names[static_cast<std::size_t>(r)] =
            dir + "/shard_r" + std::to_string(r) + "_of_" + std::to_string(R) + ".bin";
    run_ranks(c, plan, devices, report, opt, [&](int r, DeviceState& st) {
        memtrack::set_phase(memtrack::Phase::gather);
        std::FILE* f = std::fopen(names[static_cast<std::size_t>(r)].c_str(), "wb");
        if (!f)
            throw std::runtime_error("run_distributed_to_files: cannot create " + names[static_cast<std::size_t>(r)]);
        const Index shard = index_bit(plan.l);
        const Index chunk = std::min<Index>(shard, Index{1} << 24);  // 256 MiB through the host
        std::vector<Amp> buf(static_cast<std::size_t>(chunk));
        bool ok = true;
        for (Index off = 0; off < shard && ok; off += chunk) {
            const Index cnt = std::min(chunk, shard - off);
            st.download(buf.data(), off, cnt);
            ok = std::fwrite(buf.data(), sizeof(Amp), static_cast<std::size_t>(cnt), f) == cnt;
        }
        ok = (std::fclose(f) == 0) && ok;
        if (!ok)
            throw std::runtime_error("run_distributed_to_files: short write to " + names[static_cast<std::size_t>(r)]);
    });
    {
        std::FILE* m = std::fopen((dir + "/manifest.json").c_str(), "w");
        if (!m)
            throw std::runtime_error("run_distributed_to_files: cannot write the manifest");
        std::fprintf(m, "{\"n\": %d, \"ranks\": %d, \"local_qubits\": %d, \"format\": "
                        "\"complex128 little-endian interleaved (re, im)\", \"files\": [",
                     c.n, R, plan.l);
        for (int r = 0; r < R; ++r)
            std::fprintf(m, "%s{\"rank\": %d, \"first_index\": %llu, \"amplitudes\": %llu, \"path\": \"%s\"}",
                         r ? ", " : "", r, static_cast<unsigned long long>(static_cast<Index>(r) << plan.l),
                         static_cast<unsigned long long>(index_bit(plan.l)),
                         names[static_cast<std::size_t>(r)].c_str());
        std::fprintf(m, "]}\n");
        std::fclose(m);
    }
    if (report)
        report->files = names;
}

namespace {

void run_ranks(const Circuit& c, const PartitionPlan& plan, const std::vector<int>& devices,
               DistributedReport* report, const PlanOptions& opt, const Sink& sink) {
    const int R = plan.ranks();
    std::vector<int> dev = devices;
    if (dev.empty())
        for (int r = 0; r < R; ++r)
            dev.push_back(r);
    if (static_cast<int>(dev.size()) != R)
        throw std::invalid_argument("run_distributed: need one device per rank");
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
            // instrumented: the high-water mark of every device allocation this rank's
            // context made (state, swap staging, program blobs, scratch), not a formula
            std::size_t live = 0, peak = 0;
            qsv_check(qsv_ctx_mem(ctx.get(), &live, &peak), "qsv_ctx_mem");
            peaks[r] = peak;
            if (r == 0)
                swaps = eng.plan().stats.swaps;
            sink(r, st);
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
}

} // namespace

} // namespace qsim
