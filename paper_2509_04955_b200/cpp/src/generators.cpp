// Definitions for qsim/generators.hpp.
#include "qsim/generators.hpp"
#include "qsim/qasm.hpp"

#include <cmath>
#include <numbers>
#include <random>
#include <sstream>
#include <stdexcept>
#include <vector>

namespace qsim {

namespace {

constexpr double kTwoPi = 2.0 * std::numbers::pi;

struct Angles {
    std::mt19937_64 rng;
    std::uniform_real_distribution<double> u{0.0, kTwoPi};
    explicit Angles(std::uint64_t seed) : rng(seed) {}
    double next() { return u(rng); }
};

void add_swap(Circuit& c, int a, int b) {
    // swap a,b -> cx(a,b) cx(b,a) cx(a,b)
    c.add(gates::cx(a, b));
    c.add(gates::cx(b, a));
    c.add(gates::cx(a, b));
}

} // namespace

Circuit gen_qft(int n) {
    Circuit c(n, "qft:" + std::to_string(n));
    for (int j = n - 1; j >= 0; --j) {
        c.add(gates::h(j));
        for (int k = j - 1; k >= 0; --k)
            c.add(gates::cp(k, j, std::numbers::pi / std::ldexp(1.0, j - k)));
    }
    for (int q = 0; q < n / 2; ++q)
        add_swap(c, q, n - 1 - q);
    return c;
}

Circuit gen_qaoa(int n, int layers, std::uint64_t seed) {
    if (n < 2 || layers < 1)
        throw std::invalid_argument("gen_qaoa: need n >= 2 and layers >= 1");
    Circuit c(n, "qaoa:" + std::to_string(n) + ":" + std::to_string(layers) + ":" + std::to_string(seed));
    Angles ang(seed);
    for (int q = 0; q < n; ++q)
        c.add(gates::h(q));
    // ring edges, deduplicated (for n = 2 both edges are the pair {0,1})
    std::vector<std::pair<int, int>> edges;
    for (int i = 0; i < n; ++i) {
        int a = i, b = (i + 1) % n;
        if (a > b) std::swap(a, b);
        bool dup = false;
        for (auto& e : edges) dup = dup || (e.first == a && e.second == b);
        if (!dup) edges.push_back({a, b});
    }
    for (int l = 0; l < layers; ++l) {
        const double gamma = ang.next();
        const double beta = ang.next();
        for (auto& e : edges) {
            c.add(gates::cx(e.first, e.second));
            c.add(gates::rz(e.second, gamma));
            c.add(gates::cx(e.first, e.second));
        }
        for (int q = 0; q < n; ++q)
            c.add(gates::rx(q, beta));
    }
    return c;
}

Circuit gen_hea(int n, int layers, std::uint64_t seed) {
    if (n < 2 || layers < 1)
        throw std::invalid_argument("gen_hea: need n >= 2 and layers >= 1");
    Circuit c(n, "hea:" + std::to_string(n) + ":" + std::to_string(layers) + ":" + std::to_string(seed));
    Angles ang(seed);
    for (int l = 1; l <= layers; ++l) {
        for (int q = 0; q < n; ++q) {
            c.add(gates::rx(q, ang.next()));
            c.add(gates::ry(q, ang.next()));
            c.add(gates::rz(q, ang.next()));
        }
        const int first = (l % 2 == 1) ? 0 : 1;
        for (int q = first; q + 1 < n; q += 2)
            c.add(gates::cx(q, q + 1));
    }
    return c;
}

Circuit gen_random(int n, int depth, std::uint64_t seed) {
    if (n < 2 || depth < 1)
        throw std::invalid_argument("gen_random: need n >= 2 and depth >= 1");
    Circuit c(n, "random:" + std::to_string(n) + ":" + std::to_string(depth) + ":" + std::to_string(seed));
    Angles ang(seed);
    std::uniform_int_distribution<int> pick(0, 2);
    for (int l = 0; l < depth; ++l) {
        for (int q = 0; q < n; ++q) {
            switch (pick(ang.rng)) {
            case 0: c.add(gates::h(q)); break;
            case 1: c.add(gates::rx(q, ang.next())); break;
            default: c.add(gates::rz(q, ang.next())); break;
            }
        }
        for (int q = (l % 2 == 0) ? 0 : 1; q + 1 < n; q += 2)
            c.add(gates::cx(q, q + 1));
    }
    return c;
}

Circuit gen_uccsd_ladder(int n, std::uint64_t target_cx, std::uint64_t seed) {
    if (n < 2)
        throw std::invalid_argument("gen_uccsd_ladder: need n >= 2");
    Circuit c(n, "uccsd:" + std::to_string(n) + ":" + std::to_string(target_cx) + ":" + std::to_string(seed));
    Angles ang(seed);
    std::uniform_int_distribution<int> pauli(0, 2);  // 0 = X, 1 = Y, 2 = Z
    const double half_pi = std::numbers::pi / 2;
    std::uint64_t cx = 0;
    std::vector<int> p;
    while (cx < target_cx) {
        const int i = std::uniform_int_distribution<int>(0, n - 2)(ang.rng);
        const int j = std::uniform_int_distribution<int>(i + 1, n - 1)(ang.rng);
        p.assign(j - i + 1, 2);
        for (int q = i; q <= j; ++q)
            p[q - i] = pauli(ang.rng);
        const double theta = ang.next();
        for (int q = i; q <= j; ++q) {
            if (p[q - i] == 0) c.add(gates::h(q));
            else if (p[q - i] == 1) c.add(gates::rx(q, half_pi));
        }
        for (int q = i; q < j; ++q)
            c.add(gates::cx(q, q + 1));
        c.add(gates::rz(j, theta));
        for (int q = j - 1; q >= i; --q)
            c.add(gates::cx(q, q + 1));
        for (int q = i; q <= j; ++q) {
            if (p[q - i] == 0) c.add(gates::h(q));
            else if (p[q - i] == 1) c.add(gates::rx(q, -half_pi));
        }
        cx += 2ull * static_cast<std::uint64_t>(j - i);
    }
    return c;
}

Circuit generate(const std::string& spec) {
    if (spec.rfind("qasm:", 0) == 0)
        return parse_qasm_file(spec.substr(5));  // OpenQASM 2.0 file
    std::vector<std::string> f;
    std::stringstream ss(spec);
    std::string item;
    while (std::getline(ss, item, ':'))
        f.push_back(item);
    auto num = [&](std::size_t i, long long dflt) -> long long {
        if (i >= f.size()) return dflt;
        try {
            std::size_t used = 0;
            const long long v = std::stoll(f[i], &used);
            if (used != f[i].size()) throw std::invalid_argument("");
            return v;
        } catch (...) {
            throw std::invalid_argument("generator spec '" + spec + "': field " + std::to_string(i) +
                                        " is not an integer");
        }
    };
    if (f.empty())
        throw std::invalid_argument("empty generator spec");
    const std::string& k = f[0];
    if (k == "qft") return gen_qft(static_cast<int>(num(1, 8)));
    if (k == "qaoa") return gen_qaoa(static_cast<int>(num(1, 8)), static_cast<int>(num(2, 1)), num(3, 1));
    if (k == "hea") return gen_hea(static_cast<int>(num(1, 8)), static_cast<int>(num(2, 5)), num(3, 4));
    if (k == "random") return gen_random(static_cast<int>(num(1, 8)), static_cast<int>(num(2, 20)), num(3, 2));
    if (k == "uccsd") return gen_uccsd_ladder(static_cast<int>(num(1, 8)), num(2, 100000), num(3, 3));
    throw std::invalid_argument("unknown generator '" + k + "' (qft|qaoa|hea|random|uccsd|qasm:<file>)");
}

} // namespace qsim
