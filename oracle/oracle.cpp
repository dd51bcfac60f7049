// CPU restatement of the reference hot path — TEST INFRASTRUCTURE ONLY (see
// oracle.h).  std::complex<double> arithmetic exactly as written in the
// paper's pseudo-code; one temporary per pair.
//
// Scheduling (not semantics): every kernel is a "range" function over its pair
// (or group) index space, and a persistent worker pool hands out fixed-size
// chunks of that space from an atomic counter.  All workers therefore stream
// through neighbouring chunks at any moment.  The earlier split into one
// contiguous slab per thread put all 2·T streams on the same address bits
// modulo a large power of two, which ran targets 14-22 at one eighth of the
// bandwidth (cache-set / DRAM-bank conflicts).  Per-pair arithmetic does not
// depend on the split, so results stay bitwise independent of the worker count
// (SPEC:108, :121).
#include "oracle.h"

#include <algorithm>
#include <atomic>
#include <complex>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace {

using cd = std::complex<double>;
using u64 = uint64_t;

cd* as_c(double* p) { return reinterpret_cast<cd*>(p); }
const cd* as_c(const double* p) { return reinterpret_cast<const cd*>(p); }

// ---------------------------------------------------------------- worker pool
class Pool {
public:
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_)
            t.join();
    }
    // Runs f(lo, hi) over [0, count) in chunks of `chunk`, on `threads` threads
    // (the caller included).
    void run(u64 count, u64 chunk, int threads, const std::function<void(u64, u64)>& f) {
        if (threads <= 1 || count <= chunk) {
            f(0, count);
            return;
        }
        std::lock_guard<std::mutex> serial(call_m_);  // one parallel region at a time
        const int want = static_cast<int>(std::min<u64>(threads - 1, (count + chunk - 1) / chunk - 1));
        grow(want);
        {
            std::lock_guard<std::mutex> lk(m_);
            job_ = &f;
            count_ = count;
            chunk_ = chunk;
            next_.store(0);
            want_ = want;
            active_ = want;
            ++gen_;
        }
        cv_.notify_all();
        drain();
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [&] { return active_ == 0; });
        job_ = nullptr;
    }

private:
    void grow(int n) {
        while (static_cast<int>(th_.size()) < n) {
            const int id = static_cast<int>(th_.size());
            th_.emplace_back([this, id] { worker(id); });
        }
    }
    void drain() {
        for (;;) {
            const u64 c = next_.fetch_add(1);
            const u64 lo = c * chunk_;
            if (lo >= count_)
                return;
            (*job_)(lo, std::min(count_, lo + chunk_));
        }
    }
    void worker(int id) {
        u64 seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_)
                return;
            seen = gen_;
            if (id >= want_)
                continue;
            lk.unlock();
            drain();
            lk.lock();
            if (--active_ == 0)
                done_cv_.notify_one();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_, call_m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(u64, u64)>* job_ = nullptr;
    u64 count_ = 0, chunk_ = 1, gen_ = 0;
    std::atomic<u64> next_{0};
    int want_ = 0, active_ = 0;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p;
    return p;
}

constexpr u64 kChunk = u64{1} << 13;  // pairs per chunk: 2 x 128 KiB streams

template <typename F>
void parallel_for(u64 count, int threads, F&& f) {
    if (threads <= 1 || count < 2 * kChunk) {
        f(u64{0}, count);
        return;
    }
    const std::function<void(u64, u64)> fn = [&f](u64 lo, u64 hi) { f(lo, hi); };
    pool().run(count, kChunk, threads, fn);
}

// Alg. 1/3 inner body: temp; a_i = u00 a_i + u01 a_j; a_j = u10 temp + u11 a_j.
inline void pair_update(cd* a, u64 i, u64 j, const cd* u) {
    const cd temp = a[i];
    a[i] = u[0] * a[i] + u[1] * a[j];
    a[j] = u[2] * temp + u[3] * a[j];
}

// ---------------------------------------------------------------- range kernels
// Each is out of line so the global (pooled) and the cache-blocked run_local
// execute the same machine code: the blocked schedule is bitwise equal.

// Alg. 3 over pair indices [lo, hi): pair p -> i = p with a 0 inserted at bit t.
__attribute__((noinline)) void single_range(cd* a, int t, const cd* U, u64 lo, u64 hi) {
    const u64 mask = u64{1} << t, low = mask - 1;
    for (u64 p = lo; p < hi;) {
        const u64 i = ((p >> t) << (t + 1)) | (p & low);
        const u64 run = std::min(hi - p, mask - (p & low));
        for (u64 q = 0; q < run; ++q)
            pair_update(a, i + q, i + q + mask, U);
        p += run;
    }
}

// Alg. 4 over pair indices [lo, hi) of the 2^{n-2} pairs with bit c = 1
// (SPEC:78, :119); c > t is the role swap of SPEC:138 — the same pair set.
__attribute__((noinline)) void controlled_range(cd* a, int c, int t, const cd* U, u64 lo, u64 hi) {
    const int b0 = std::min(c, t), b1 = std::max(c, t);
    const u64 m0 = (u64{1} << b0) - 1, m1 = (u64{1} << b1) - 1;
    const u64 mask_t = u64{1} << t, mask_c = u64{1} << c;
    for (u64 p = lo; p < hi;) {
        u64 i = ((p >> b0) << (b0 + 1)) | (p & m0);
        i = ((i >> b1) << (b1 + 1)) | (i & m1);
        i |= mask_c;
        const u64 run = std::min(hi - p, (m0 + 1) - (p & m0));
        for (u64 q = 0; q < run; ++q)
            pair_update(a, i + q, i + q + mask_t, U);
        p += run;
    }
}

struct MultiPlan {
    int k = 0;
    u64 D = 0, cmask = 0;
    std::vector<u64> off;
    std::vector<int> fixed;  // ascending used bits (targets + controls)
};

// apply_multi over groups [lo, hi): gather 2^k, M x group, scatter.
__attribute__((noinline)) void multi_range(cd* a, const MultiPlan& P, const cd* M, u64 lo, u64 hi) {
    const u64 D = P.D;
    cd in[256];
    for (u64 g = lo; g < hi; ++g) {
        u64 base = g;
        for (int p : P.fixed) {  // ascending: insert a zero at each used bit
            const u64 low = base & ((u64{1} << p) - 1);
            base = ((base >> p) << (p + 1)) | low;
        }
        base |= P.cmask;
        for (u64 j = 0; j < D; ++j)
            in[j] = a[base | P.off[j]];
        for (u64 r = 0; r < D; ++r) {
            cd acc = 0.0;
            for (u64 j = 0; j < D; ++j)
                acc += M[r * D + j] * in[j];
            a[base | P.off[r]] = acc;
        }
    }
}

bool make_multi(int n, int k, const int* targets, int nctrl, const int* controls, MultiPlan& P) {
    if (k < 1 || k > 8 || nctrl < 0 || k + nctrl > n) return false;
    u64 used = 0;
    P = MultiPlan{};
    P.k = k;
    for (int i = 0; i < k; ++i) {
        if (targets[i] < 0 || targets[i] >= n || (used >> targets[i] & 1)) return false;
        used |= u64{1} << targets[i];
    }
    for (int i = 0; i < nctrl; ++i) {
        if (controls[i] < 0 || controls[i] >= n || (used >> controls[i] & 1)) return false;
        used |= u64{1} << controls[i];
        P.cmask |= u64{1} << controls[i];
    }
    P.D = u64{1} << k;
    P.off.assign(P.D, 0);
    for (u64 j = 0; j < P.D; ++j)
        for (int i = 0; i < k; ++i)
            if (j >> i & 1)
                P.off[j] |= u64{1} << targets[i];
    for (int q = 0; q < n; ++q)
        if (used >> q & 1)
            P.fixed.push_back(q);
    return true;
}

// One gate of run_local, dispatched as the reference does (1q -> Alg. 3,
// 1q + 1 control -> Alg. 4, else apply_multi), prepared for a 2^n buffer.
struct Prepared {
    int kind = 0;  // 1 single, 2 controlled, 3 multi
    int t = 0, c = 0;
    const cd* m = nullptr;
    MultiPlan P;
    u64 count = 0;  // pairs or groups
    void range(cd* a, u64 lo, u64 hi) const {
        if (kind == 1) single_range(a, t, m, lo, hi);
        else if (kind == 2) controlled_range(a, c, t, m, lo, hi);
        else multi_range(a, P, m, lo, hi);
    }
};

bool prepare(int n, const orc_gate& g, const double* pool_, Prepared& out) {
    out.m = as_c(pool_ + 2 * g.mat_off);
    if (g.arity == 1 && g.nctrl == 0) {
        if (n < 1 || g.targets[0] < 0 || g.targets[0] >= n) return false;
        out.kind = 1;
        out.t = g.targets[0];
        out.count = u64{1} << (n - 1);
        return true;
    }
    if (g.arity == 1 && g.nctrl == 1) {
        const int c = g.controls[0], t = g.targets[0];
        if (n < 2 || c < 0 || t < 0 || c >= n || t >= n || c == t) return false;
        out.kind = 2;
        out.c = c;
        out.t = t;
        out.count = u64{1} << (n - 2);
        return true;
    }
    if (!make_multi(n, g.arity, g.targets, g.nctrl, g.controls, out.P)) return false;
    out.kind = 3;
    out.count = u64{1} << (n - g.arity - g.nctrl);
    return true;
}

int apply_gate(int n, cd* a, const orc_gate& g, const double* pool_, int threads) {
    Prepared pg;
    if (!prepare(n, g, pool_, pg)) return -1;
    parallel_for(pg.count, threads, [&](u64 lo, u64 hi) { pg.range(a, lo, hi); });
    return 0;
}

u64 gate_qubits(const orc_gate& g) {
    u64 s = 0;
    for (int i = 0; i < g.arity; ++i) s |= u64{1} << g.targets[i];
    for (int i = 0; i < g.nctrl; ++i) s |= u64{1} << g.controls[i];
    return s;
}

} // namespace

extern "C" {

int orc_default_threads(void) {
    const unsigned h = std::thread::hardware_concurrency();
    return h ? static_cast<int>(h) : 1;
}

int orc_apply_single_naive(int n, double* amps, int t, const double* u) {
    if (n < 1 || t < 0 || t >= n) return -1;
    cd* a = as_c(amps);
    const cd* U = as_c(u);
    const u64 mask = u64{1} << t;
    const u64 N = u64{1} << n;
    for (u64 i = 0; i < N; ++i)
        if ((i & mask) == 0)
            pair_update(a, i, i + mask, U);
    return 0;
}

int orc_apply_single_grouped(int n, double* amps, int t, const double* u, int threads) {
    if (n < 1 || t < 0 || t >= n) return -1;
    cd* a = as_c(amps);
    const cd* U = as_c(u);
    parallel_for(u64{1} << (n - 1), threads, [&](u64 lo, u64 hi) { single_range(a, t, U, lo, hi); });
    return 0;
}

int orc_apply_controlled(int n, double* amps, int c, int t, const double* u, int threads) {
    if (n < 2 || c < 0 || t < 0 || c >= n || t >= n || c == t) return -1;
    cd* a = as_c(amps);
    const cd* U = as_c(u);
    parallel_for(u64{1} << (n - 2), threads, [&](u64 lo, u64 hi) { controlled_range(a, c, t, U, lo, hi); });
    return 0;
}

int orc_apply_multi(int n, double* amps, int k, const int* targets, int nctrl, const int* controls,
                    const double* m, int threads) {
    MultiPlan P;
    if (!make_multi(n, k, targets, nctrl, controls, P)) return -1;
    cd* a = as_c(amps);
    const cd* M = as_c(m);
    parallel_for(u64{1} << (n - k - nctrl), threads, [&](u64 lo, u64 hi) { multi_range(a, P, M, lo, hi); });
    return 0;
}

int orc_run_local(int n, const orc_gate* gates, int64_t ngates, const double* pool_, double* amps,
                  int threads) {
    if (n < 1 || threads < 1) return -1;
    for (int64_t gi = 0; gi < ngates; ++gi) {
        if (gates[gi].arity == 0)
            continue;  // barrier: fusion fence only
        const int rc = apply_gate(n, as_c(amps), gates[gi], pool_, threads);
        if (rc != 0)
            return rc;
    }
    return 0;
}

// Cache-blocked schedule of run_local (test infrastructure for full-size
// parity): a maximal run of consecutive gates whose qubits fit in B bits is
// applied block by block — gather the 2^B amplitudes that share the other n-B
// index bits, apply the run's gates in program order with the same range
// kernels, scatter back.  Every amplitude sees the same pair updates in the
// same order with the same code, so the result is bitwise equal to
// orc_run_local (tests/test_oracle.py checks it).
int orc_run_local_blocked(int n, const orc_gate* gates, int64_t ngates, const double* pool_, double* amps,
                          int threads, int block_bits) {
    if (n < 1 || threads < 1) return -1;
    const int B = std::min(n, std::max(block_bits, 4));
    cd* a = as_c(amps);
    int64_t gi = 0;
    while (gi < ngates) {
        if (gates[gi].arity == 0) {
            ++gi;
            continue;
        }
        u64 S = gate_qubits(gates[gi]);
        if (__builtin_popcountll(S) > B) {  // wider than a block: apply globally
            const int rc = apply_gate(n, a, gates[gi], pool_, threads);
            if (rc != 0) return rc;
            ++gi;
            continue;
        }
        int64_t end = gi + 1;
        while (end < ngates) {
            if (gates[end].arity == 0) { ++end; continue; }
            const u64 s2 = S | gate_qubits(gates[end]);
            if (__builtin_popcountll(s2) > B) break;
            S = s2;
            ++end;
        }
        for (int q = 0; q < n && __builtin_popcountll(S) < B; ++q)  // pad with low qubits: contiguous runs
            S |= u64{1} << q;
        int pos[64], local[64];
        int np = 0;
        for (int q = 0; q < n; ++q) {
            local[q] = -1;
            if (S >> q & 1) { local[q] = np; pos[np++] = q; }
        }
        // the run's gates with remapped qubits, prepared for a 2^B block
        std::vector<Prepared> run;
        for (int64_t j = gi; j < end; ++j) {
            if (gates[j].arity == 0) continue;
            orc_gate g = gates[j];
            for (int i = 0; i < g.arity; ++i) g.targets[i] = local[g.targets[i]];
            for (int i = 0; i < g.nctrl; ++i) g.controls[i] = local[g.controls[i]];
            run.emplace_back();
            if (!prepare(B, g, pool_, run.back())) return -1;
        }
        const u64 DB = u64{1} << B;
        std::vector<u64> off(DB);
        for (u64 j = 0; j < DB; ++j) {
            u64 o = 0;
            for (int i = 0; i < B; ++i)
                if (j >> i & 1) o |= u64{1} << pos[i];
            off[j] = o;
        }
        std::vector<int> outer;
        for (int q = 0; q < n; ++q)
            if (!(S >> q & 1)) outer.push_back(q);
        const u64 nblocks = u64{1} << (n - B);
        const std::function<void(u64, u64)> body = [&](u64 lo, u64 hi) {
            thread_local std::vector<cd> buf;
            if (buf.size() < DB) buf.resize(DB);
            for (u64 b = lo; b < hi; ++b) {
                u64 base = 0;
                for (size_t i = 0; i < outer.size(); ++i)
                    if (b >> i & 1) base |= u64{1} << outer[i];
                for (u64 j = 0; j < DB; ++j) buf[j] = a[base | off[j]];
                for (const Prepared& g : run)
                    g.range(buf.data(), 0, g.count);
                for (u64 j = 0; j < DB; ++j) a[base | off[j]] = buf[j];
            }
        };
        if (threads <= 1 || nblocks == 1)
            body(0, nblocks);
        else
            pool().run(nblocks, 1, threads, body);
        gi = end;
    }
    return 0;
}

int orc_fill_basis(int n, double* amps, uint64_t index, int threads) {
    if (n < 1 || n > 62 || index >= (u64{1} << n)) return -1;
    cd* a = as_c(amps);
    // parallel first touch: pages land where the pooled kernels will stream them
    parallel_for(u64{1} << n, threads, [&](u64 lo, u64 hi) { std::fill(a + lo, a + hi, cd(0.0)); });
    a[index] = 1.0;
    return 0;
}

int orc_dense_oracle(int n, const orc_gate* gates, int64_t ngates, const double* pool_,
                     const double* in, double* out) {
    if (n < 1 || n > 12) return -2;  // scale guard
    const u64 N = u64{1} << n;
    std::vector<cd> cur(as_c(in), as_c(in) + N), nxt(N);
    std::vector<cd> row(N);
    for (int64_t gi = 0; gi < ngates; ++gi) {
        const orc_gate& g = gates[gi];
        if (g.arity == 0)
            continue;
        const cd* M = as_c(pool_ + 2 * g.mat_off);
        const u64 D = u64{1} << g.arity;
        u64 tmask = 0, cmask = 0;
        for (int i = 0; i < g.arity; ++i) tmask |= u64{1} << g.targets[i];
        for (int i = 0; i < g.nctrl; ++i) cmask |= u64{1} << g.controls[i];
        auto local = [&](u64 idx) {  // bits of idx at the targets -> matrix index
            u64 r = 0;
            for (int i = 0; i < g.arity; ++i)
                r |= ((idx >> g.targets[i]) & 1) << i;
            return r;
        };
        // Row i of the embedded operator G = |controls off><..| (x) I + |on><on| (x) M:
        // G[i][j] = delta_ij if controls of i not all set, else
        //           M[local(i)][local(j)] when i, j agree outside the targets.
        for (u64 i = 0; i < N; ++i) {
            for (u64 j = 0; j < N; ++j) {
                cd e = 0.0;
                if ((i & cmask) != cmask) {
                    e = (i == j) ? cd(1.0) : cd(0.0);
                } else if ((i & ~tmask) == (j & ~tmask)) {
                    e = M[local(i) * D + local(j)];
                }
                row[j] = e;
            }
            cd acc = 0.0;
            for (u64 j = 0; j < N; ++j)
                acc += row[j] * cur[j];
            nxt[i] = acc;
        }
        cur.swap(nxt);
    }
    std::memcpy(out, cur.data(), N * sizeof(cd));
    return 0;
}

} // extern "C"
