// Workload generators restated for the CPU reference arm — TEST / BASELINE
// INFRASTRUCTURE ONLY.  The reference arm of bench.py must not load the
// product libraries (libqsv.so / libqsim.so), so it regenerates the synthetic
// circuits here and builds their gate matrices with the reference's own
// gates::from_mnemonic (oracle/_ref, see pyoracle.generate).
//
// Gate sequences follow SPEC:181-209 (QFT with the corrected cp(pi/2^{j-k})
// angle; QAOA ring; HEA brick) and SURVEY §8(d) (random
// H/RX/RZ + brick CNOT; UCCSD Pauli-exponential ladders), drawing from
// std::mt19937_64 with the same distributions in the same order as the
// product's generators, so the circuits are gate-for-gate and bit-for-bit the
// same (tests/test_oracle.py::test_generator_restatement_matches_product).
#include "oracle.h"

#include <cmath>
#include <cstring>
#include <numbers>
#include <random>
#include <sstream>
#include <string>
#include <vector>

namespace {

struct Instr {
    int code;  // orc_mnemonic index
    int q0, q1;
    double param;
};

constexpr double kTwoPi = 2.0 * std::numbers::pi;

struct Gen {
    std::vector<Instr> out;
    void add(int code, int q0, int q1 = -1, double p = 0.0) { out.push_back({code, q0, q1, p}); }
    void h(int q) { add(ORC_H, q); }
    void rx(int q, double t) { add(ORC_RX, q, -1, t); }
    void ry(int q, double t) { add(ORC_RY, q, -1, t); }
    void rz(int q, double t) { add(ORC_RZ, q, -1, t); }
    void cx(int c, int t) { add(ORC_CX, c, t); }
    void cp(int c, int t, double l) { add(ORC_CP, c, t, l); }
    void swap(int a, int b) {
        cx(a, b);
        cx(b, a);
        cx(a, b);
    }
};

struct Angles {
    std::mt19937_64 rng;
    std::uniform_real_distribution<double> u{0.0, kTwoPi};
    explicit Angles(uint64_t seed) : rng(seed) {}
    double next() { return u(rng); }
};

void qft(Gen& g, int n) {
    for (int j = n - 1; j >= 0; --j) {
        g.h(j);
        for (int k = j - 1; k >= 0; --k)
            g.cp(k, j, std::numbers::pi / std::ldexp(1.0, j - k));
    }
    for (int q = 0; q < n / 2; ++q)
        g.swap(q, n - 1 - q);
}

void qaoa(Gen& g, int n, int layers, uint64_t seed) {
    Angles ang(seed);
    for (int q = 0; q < n; ++q) g.h(q);
    std::vector<std::pair<int, int>> edges;
    for (int i = 0; i < n; ++i) {
        int a = i, b = (i + 1) % n;
        if (a > b) std::swap(a, b);
        bool dup = false;
        for (auto& e : edges) dup = dup || (e.first == a && e.second == b);
        if (!dup) edges.push_back({a, b});
    }
    for (int l = 0; l < layers; ++l) {
        const double gamma = ang.next(), beta = ang.next();
        for (auto& e : edges) {
            g.cx(e.first, e.second);
            g.rz(e.second, gamma);
            g.cx(e.first, e.second);
        }
        for (int q = 0; q < n; ++q) g.rx(q, beta);
    }
}

void hea(Gen& g, int n, int layers, uint64_t seed) {
    Angles ang(seed);
    for (int l = 1; l <= layers; ++l) {
        for (int q = 0; q < n; ++q) {
            const double a = ang.next();
            const double b = ang.next();
            const double c = ang.next();
            g.rx(q, a);
            g.ry(q, b);
            g.rz(q, c);
        }
        for (int q = (l % 2 == 1) ? 0 : 1; q + 1 < n; q += 2) g.cx(q, q + 1);
    }
}

void random_circuit(Gen& g, int n, int depth, uint64_t seed) {
    Angles ang(seed);
    std::uniform_int_distribution<int> pick(0, 2);
    for (int l = 0; l < depth; ++l) {
        for (int q = 0; q < n; ++q) {
            switch (pick(ang.rng)) {
            case 0: g.h(q); break;
            case 1: g.rx(q, ang.next()); break;
            default: g.rz(q, ang.next()); break;
            }
        }
        for (int q = (l % 2 == 0) ? 0 : 1; q + 1 < n; q += 2) g.cx(q, q + 1);
    }
}

void uccsd(Gen& g, int n, uint64_t target_cx, uint64_t seed) {
    Angles ang(seed);
    std::uniform_int_distribution<int> pauli(0, 2);
    const double half_pi = std::numbers::pi / 2;
    uint64_t cx = 0;
    std::vector<int> p;
    while (cx < target_cx) {
        const int i = std::uniform_int_distribution<int>(0, n - 2)(ang.rng);
        const int j = std::uniform_int_distribution<int>(i + 1, n - 1)(ang.rng);
        p.assign(j - i + 1, 2);
        for (int q = i; q <= j; ++q) p[q - i] = pauli(ang.rng);
        const double theta = ang.next();
        for (int q = i; q <= j; ++q) {
            if (p[q - i] == 0) g.h(q);
            else if (p[q - i] == 1) g.rx(q, half_pi);
        }
        for (int q = i; q < j; ++q) g.cx(q, q + 1);
        g.rz(j, theta);
        for (int q = j - 1; q >= i; --q) g.cx(q, q + 1);
        for (int q = i; q <= j; ++q) {
            if (p[q - i] == 0) g.h(q);
            else if (p[q - i] == 1) g.rx(q, -half_pi);
        }
        cx += 2ull * static_cast<uint64_t>(j - i);
    }
}

} // namespace

extern "C" {

int64_t orc_generate(const char* spec, int* n_out, int32_t* codes, int32_t* q0, int32_t* q1, double* params,
                     int64_t cap) {
    std::vector<std::string> f;
    std::stringstream ss(spec ? spec : "");
    std::string item;
    while (std::getline(ss, item, ':')) f.push_back(item);
    if (f.empty()) return -1;
    auto num = [&](size_t i, long long dflt) -> long long {
        if (i >= f.size()) return dflt;
        return std::stoll(f[i]);
    };
    Gen g;
    int n = 0;
    try {
        n = static_cast<int>(num(1, 8));
        if (n < 2) return -1;
        if (f[0] == "qft") qft(g, n);
        else if (f[0] == "qaoa") qaoa(g, n, static_cast<int>(num(2, 1)), num(3, 1));
        else if (f[0] == "hea") hea(g, n, static_cast<int>(num(2, 5)), num(3, 4));
        else if (f[0] == "random") random_circuit(g, n, static_cast<int>(num(2, 20)), num(3, 2));
        else if (f[0] == "uccsd") uccsd(g, n, num(2, 100000), num(3, 3));
        else return -1;
    } catch (...) {
        return -1;
    }
    *n_out = n;
    const int64_t cnt = static_cast<int64_t>(g.out.size());
    if (cap >= cnt) {
        for (int64_t i = 0; i < cnt; ++i) {
            codes[i] = g.out[i].code;
            q0[i] = g.out[i].q0;
            q1[i] = g.out[i].q1;
            params[i] = g.out[i].param;
        }
    }
    return cnt;
}

} // extern "C"
