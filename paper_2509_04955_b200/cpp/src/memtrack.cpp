// Definitions for qsim/memtrack.hpp.  Semantics follow the reference
// (proj/src/memtrack.cpp:11-80): disabled by default, a thread-local rank and
// phase, per-(rank, phase) current and peak byte counters, releases clamp at
// zero, unknown ranks are ignored.  Independent implementation.
#include "qsim/memtrack.hpp"

#include <algorithm>
#include <array>
#include <atomic>
#include <mutex>
#include <vector>

namespace qsim::memtrack {

namespace {

struct Counters {
    std::array<std::size_t, 2> live{};
    std::array<std::size_t, 2> high{};
};

struct Registry {
    std::mutex lock;
    std::vector<Counters> ranks;
    std::atomic<bool> on{false};
};

Registry& registry() {
    static Registry r;
    return r;
}

struct ThreadSlot {
    int rank = -1;
    Phase phase = Phase::execute;
};
thread_local ThreadSlot tls;

template <typename F>
void with_my_counters(F&& f) {
    Registry& r = registry();
    if (!r.on.load(std::memory_order_acquire) || tls.rank < 0)
        return;
    std::lock_guard<std::mutex> g(r.lock);
    if (static_cast<std::size_t>(tls.rank) >= r.ranks.size())
        return;
    f(r.ranks[static_cast<std::size_t>(tls.rank)], static_cast<std::size_t>(tls.phase));
}

} // namespace

void enable(int ranks) {
    Registry& r = registry();
    {
        std::lock_guard<std::mutex> g(r.lock);
        r.ranks.clear();
        r.ranks.resize(static_cast<std::size_t>(std::max(ranks, 0)));
    }
    r.on.store(true, std::memory_order_release);
}

void disable() { registry().on.store(false, std::memory_order_release); }

bool enabled() { return registry().on.load(std::memory_order_acquire); }

void register_thread(int rank) {
    tls.rank = rank;
    tls.phase = Phase::execute;
}

void unregister_thread() { tls.rank = -1; }

void set_phase(Phase phase) { tls.phase = phase; }

void on_alloc(std::size_t bytes) {
    with_my_counters([bytes](Counters& c, std::size_t p) {
        c.live[p] += bytes;
        c.high[p] = std::max(c.high[p], c.live[p]);
    });
}

void on_free(std::size_t bytes) {
    with_my_counters([bytes](Counters& c, std::size_t p) {
        c.live[p] = bytes >= c.live[p] ? 0 : c.live[p] - bytes;
    });
}

std::size_t peak_bytes(int rank, Phase phase) {
    Registry& r = registry();
    std::lock_guard<std::mutex> g(r.lock);
    if (rank < 0 || static_cast<std::size_t>(rank) >= r.ranks.size())
        return 0;
    return r.ranks[static_cast<std::size_t>(rank)].high[static_cast<std::size_t>(phase)];
}

void reset() {
    Registry& r = registry();
    std::lock_guard<std::mutex> g(r.lock);
    for (Counters& c : r.ranks)
        c = Counters{};
}

} // namespace qsim::memtrack
