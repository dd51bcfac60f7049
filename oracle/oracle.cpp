// CPU restatement of the reference hot path — TEST INFRASTRUCTURE ONLY (see
// oracle.h).  std::complex<double> arithmetic exactly as written in the
// paper's pseudo-code; one temporary per pair.
#include "oracle.h"

#include <algorithm>
#include <complex>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

namespace {

using cd = std::complex<double>;
using u64 = uint64_t;

cd* as_c(double* p) { return reinterpret_cast<cd*>(p); }
const cd* as_c(const double* p) { return reinterpret_cast<const cd*>(p); }

// Split [0, count) into `threads` contiguous ranges and run f(lo, hi) on each.
// Ranges are disjoint and per-element arithmetic does not depend on the split,
// so results are bitwise independent of the worker count.
template <typename F>
void parallel_for(u64 count, int threads, F&& f) {
    if (threads <= 1 || count < 4096) {
        f(u64{0}, count);
        return;
    }
    const int nt = static_cast<int>(std::min<u64>(threads, count));
    std::vector<std::thread> pool;
    pool.reserve(nt);
    for (int w = 0; w < nt; ++w) {
        const u64 lo = count * w / nt, hi = count * (w + 1) / nt;
        pool.emplace_back([&f, lo, hi] { f(lo, hi); });
    }
    for (auto& th : pool)
        th.join();
}

// Alg. 1/3 inner body: temp; a_i = u00 a_i + u01 a_j; a_j = u10 temp + u11 a_j.
inline void pair_update(cd* a, u64 i, u64 j, const cd* u) {
    const cd temp = a[i];
    a[i] = u[0] * a[i] + u[1] * a[j];
    a[j] = u[2] * temp + u[3] * a[j];
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
    const u64 mask = u64{1} << t;
    const u64 group = mask << 1;
    const u64 ngroups = (u64{1} << n) / group;
    // Parallelise over groups when there are many, over the inner range otherwise.
    if (ngroups >= static_cast<u64>(std::max(threads, 1))) {
        parallel_for(ngroups, threads, [&](u64 lo, u64 hi) {
            for (u64 g = lo * group; g < hi * group; g += group)
                for (u64 i = g; i < g + mask; ++i)
                    pair_update(a, i, i + mask, U);
        });
    } else {
        for (u64 g = 0; g < (u64{1} << n); g += group)
            parallel_for(mask, threads, [&](u64 lo, u64 hi) {
                for (u64 i = g + lo; i < g + hi; ++i)
                    pair_update(a, i, i + mask, U);
            });
    }
    return 0;
}

int orc_apply_controlled(int n, double* amps, int c, int t, const double* u, int threads) {
    if (n < 2 || c < 0 || t < 0 || c >= n || t >= n || c == t) return -1;
    cd* a = as_c(amps);
    const cd* U = as_c(u);
    const u64 mask_c = u64{1} << c, mask_t = u64{1} << t;
    const u64 N = u64{1} << n;
    if (c < t) {
        // Alg. 4 as printed: groups of 2^{t+1}; sub-groups s stepping 2^{c+1}
        // starting at g + mask_c; inner run of mask_c indices.
        const u64 gt = mask_t << 1, gc = mask_c << 1;
        parallel_for(N / gt, threads, [&](u64 lo, u64 hi) {
            for (u64 g = lo * gt; g < hi * gt; g += gt)
                for (u64 s = g + mask_c; s < g + mask_t; s += gc)
                    for (u64 i = s; i < s + mask_c; ++i)
                        pair_update(a, i, i + mask_t, U);
        });
    } else {
        // Role swap for c > t: outer groups of 2^{c+1}, take the
        // upper half (bit c = 1), then Alg. 3 over t inside it.
        const u64 gc = mask_c << 1, gt = mask_t << 1;
        parallel_for(N / gc, threads, [&](u64 lo, u64 hi) {
            for (u64 g = lo * gc + mask_c; g < hi * gc; g += gc)
                for (u64 s = g; s < g + mask_c; s += gt)
                    for (u64 i = s; i < s + mask_t; ++i)
                        pair_update(a, i, i + mask_t, U);
        });
    }
    return 0;
}

int orc_apply_multi(int n, double* amps, int k, const int* targets, int nctrl, const int* controls,
                    const double* m, int threads) {
    if (k < 1 || k > 8 || nctrl < 0 || k + nctrl > n) return -1;
    u64 used = 0, cmask = 0;
    for (int i = 0; i < k; ++i) {
        if (targets[i] < 0 || targets[i] >= n || (used >> targets[i] & 1)) return -1;
        used |= u64{1} << targets[i];
    }
    for (int i = 0; i < nctrl; ++i) {
        if (controls[i] < 0 || controls[i] >= n || (used >> controls[i] & 1)) return -1;
        used |= u64{1} << controls[i];
        cmask |= u64{1} << controls[i];
    }
    cd* a = as_c(amps);
    const cd* M = as_c(m);
    const u64 D = u64{1} << k;
    std::vector<u64> off(D, 0);
    for (u64 j = 0; j < D; ++j)
        for (int i = 0; i < k; ++i)
            if (j >> i & 1)
                off[j] |= u64{1} << targets[i];
    std::vector<int> fixed;
    for (int q = 0; q < n; ++q)
        if (used >> q & 1)
            fixed.push_back(q);
    const u64 ngroups = u64{1} << (n - k - nctrl);
    parallel_for(ngroups, threads, [&](u64 lo, u64 hi) {
        std::vector<cd> in(D);
        for (u64 g = lo; g < hi; ++g) {
            u64 base = g;
            for (int p : fixed) {  // ascending: insert a zero at each used bit
                const u64 low = base & ((u64{1} << p) - 1);
                base = ((base >> p) << (p + 1)) | low;
            }
            base |= cmask;
            for (u64 j = 0; j < D; ++j)
                in[j] = a[base | off[j]];
            for (u64 r = 0; r < D; ++r) {
                cd acc = 0.0;
                for (u64 j = 0; j < D; ++j)
                    acc += M[r * D + j] * in[j];
                a[base | off[r]] = acc;
            }
        }
    });
    return 0;
}

int orc_run_local(int n, const orc_gate* gates, int64_t ngates, const double* pool, double* amps,
                  int threads) {
    if (n < 1 || threads < 1) return -1;
    for (int64_t gi = 0; gi < ngates; ++gi) {
        const orc_gate& g = gates[gi];
        if (g.arity == 0)
            continue;  // barrier: fusion fence only
        const double* m = pool + 2 * g.mat_off;
        int rc;
        if (g.arity == 1 && g.nctrl == 0)
            rc = orc_apply_single_grouped(n, amps, g.targets[0], m, threads);
        else if (g.arity == 1 && g.nctrl == 1)
            rc = orc_apply_controlled(n, amps, g.controls[0], g.targets[0], m, threads);
        else
            rc = orc_apply_multi(n, amps, g.arity, g.targets, g.nctrl, g.controls, m, threads);
        if (rc != 0)
            return rc;
    }
    return 0;
}

int orc_dense_oracle(int n, const orc_gate* gates, int64_t ngates, const double* pool,
                     const double* in, double* out) {
    if (n < 1 || n > 12) return -2;  // scale guard
    const u64 N = u64{1} << n;
    std::vector<cd> cur(as_c(in), as_c(in) + N), nxt(N);
    std::vector<cd> row(N);
    for (int64_t gi = 0; gi < ngates; ++gi) {
        const orc_gate& g = gates[gi];
        if (g.arity == 0)
            continue;
        const cd* M = as_c(pool + 2 * g.mat_off);
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
