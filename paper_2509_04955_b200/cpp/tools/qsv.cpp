// `qsv` — thin run/report driver over the B200 engine.
// Reconstructed from the reference CMake target tools/qsv.cpp (proj/CMakeLists.txt:40-41,
// absent upstream) and the SPEC flag list.  It parses or generates a
// circuit, plans it (DAGC + SMGP + BBOP), runs it on the GPU `--repeat` times and prints a
// RunReport as JSON or CSV with identical values.
//
//   qsv run (--gen SPEC | --qasm FILE) [--fusion on|off] [--stagger on|off] [--repeat R]
//           [--tile-k K] [--verify none|norm|qft:X] [--format json|csv] [--out FILE]
//   qsv ablate --gen SPEC [--sizes N1,N2,...] [--repeat R] [--format json|csv] [--out FILE]
//           cli_ablate: the {fusion} x {stagger} toggle grid per size, one
//           RunReport per cell plus speedups against the all-off cell of the same size
//   qsv verify [--quick]
//           cli_verify_suite: the acceptance criteria that run
//           without the CPU oracle, as a pass/fail matrix with per-criterion runtimes
//
// Multi-GPU runs go through bench.py / torchrun (one process per GPU); --ranks is accepted
// for flag compatibility and must be 1 here.  --verify never uses the CPU oracle (test
// infrastructure): `norm` checks the device norm, `qft:X` the analytic QFT of basis state X.
#include "qsim/device.hpp"
#include "qsim/exchange.hpp"
#include "qsim/fusion.hpp"
#include "qsim/partition.hpp"
#include "qsim/generators.hpp"
#include "qsim/qasm.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <complex>
#include <fstream>
#include <functional>
#include <random>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

namespace {

using Clock = std::chrono::steady_clock;

double secs(Clock::time_point a, Clock::time_point b) { return std::chrono::duration<double>(b - a).count(); }

[[noreturn]] void usage(const std::string& why) {
    std::cerr << "qsv: " << why << "\n"
              << "usage: qsv run (--gen SPEC | --qasm FILE) [--fusion on|off] [--stagger on|off]\n"
              << "               [--repeat R] [--tile-k K] [--verify none|norm|qft:X]\n"
              << "               [--format json|csv] [--out FILE]\n"
              << "       qsv ablate --gen SPEC [--sizes N1,N2] [--repeat R] [--format json|csv] [--out FILE]\n"
              << "       qsv verify [--quick]\n";
    std::exit(2);
}

bool on_off(const std::string& v, const char* flag) {
    if (v == "on")
        return true;
    if (v == "off")
        return false;
    usage(std::string(flag) + " takes on|off");
}

}  // namespace

// One circuit through the engine `repeat` times; the RunReport fields.
std::vector<std::pair<std::string, std::string>> run_report(const qsim::Circuit& c, const qsim::PlanOptions& o,
                                                            int repeat, const std::string& verify,
                                                            const std::string& fusion, const std::string& stagger,
                                                            double parse_s) {
    const auto t1 = Clock::now();
    qsim::DeviceContext ctx(0);
    qsim::Engine eng(ctx, c, o);
    const auto t2 = Clock::now();
    qsim::DeviceState st(ctx, c.n);
    std::vector<double> exec;
    const uint64_t basis = verify.rfind("qft:", 0) == 0 ? std::stoull(verify.substr(4), nullptr, 0) : 0;
    for (int r = 0; r < repeat + 1; ++r) {  // run 0 is the warm-up (graph capture)
        st.set_basis(basis);
        ctx.sync();
        const auto a = Clock::now();
        eng.run(st);
        ctx.sync();
        if (r > 0)
            exec.push_back(secs(a, Clock::now()));
    }
    std::sort(exec.begin(), exec.end());
    const double med = exec[exec.size() / 2];
    double deviation = -1.0;
    if (verify == "norm") {
        deviation = std::abs(st.norm_sq() - 1.0);
    } else if (verify.rfind("qft:", 0) == 0) {
        double e = 0;
        qsim::qsv_check(qsv_check_qft_basis(st.get(), c.n, basis, &e), "qsv_check_qft_basis");
        deviation = e;
    } else if (verify != "none") {
        usage("--verify takes none|norm|qft:X");
    }
    const qsim::PlanStats& s = eng.plan().stats;
    const double gates = static_cast<double>(s.gates_in);
    return {
        {"source", c.source},
        {"qubits", std::to_string(c.n)},
        {"ranks", "1"},
        {"fusion", fusion},
        {"stagger", stagger},
        {"tile_k", std::to_string(o.tile_k)},
        {"repeat", std::to_string(repeat)},
        {"parse_s", std::to_string(parse_s)},
        {"plan_s", std::to_string(secs(t1, t2))},
        {"execute_s_median", std::to_string(med)},
        {"execute_s_min", std::to_string(exec.front())},
        {"execute_s_max", std::to_string(exec.back())},
        {"gates_before", std::to_string(s.gates_in)},
        {"ops_after_fusion", std::to_string(s.ops_fused)},
        {"ops_final", std::to_string(s.ops_final)},
        {"compression_ratio", std::to_string(gates > 0 ? s.ops_final / gates : 0.0)},
        {"passes", std::to_string(s.passes)},
        {"swaps", std::to_string(s.swaps)},
        {"comm_bytes", "0"},
        {"gates_per_s", std::to_string(gates / med)},
        {"hbm_gbs", std::to_string(32.0 * std::ldexp(1.0, c.n) * s.passes / med / 1e9)},
        {"verify", verify},
        {"max_deviation", std::to_string(deviation)},
    };
}

using Record = std::vector<std::pair<std::string, std::string>>;

bool is_text(const std::string& k) {
    return k == "source" || k == "fusion" || k == "stagger" || k == "verify" || k == "cell" || k == "criterion" ||
           k == "status" || k == "detail";
}

std::string to_json(const Record& rec) {
    std::ostringstream out;
    out << "{";
    for (size_t i = 0; i < rec.size(); ++i) {
        const bool num = !is_text(rec[i].first);
        out << (i ? ", " : "") << '"' << rec[i].first << "\": " << (num ? "" : "\"") << rec[i].second
            << (num ? "" : "\"");
    }
    out << "}";
    return out.str();
}

std::string to_csv(const std::vector<Record>& rows) {
    std::ostringstream out;
    for (size_t i = 0; i < rows.front().size(); ++i)
        out << (i ? "," : "") << rows.front()[i].first;
    out << "\n";
    for (const Record& r : rows) {
        for (size_t i = 0; i < r.size(); ++i)
            out << (i ? "," : "") << r[i].second;
        out << "\n";
    }
    return out.str();
}

void emit(const std::string& text, std::map<std::string, std::string>& f) {
    if (f.count("--out"))
        std::ofstream(f["--out"]) << text;
    else
        std::cout << text;
}

// spec with its qubit count (the first numeric field) replaced by n
std::string with_size(const std::string& spec, int n) {
    const size_t a = spec.find(':');
    if (a == std::string::npos)
        return spec;
    const size_t b = spec.find(':', a + 1);
    return spec.substr(0, a + 1) + std::to_string(n) + (b == std::string::npos ? "" : spec.substr(b));
}

int cmd_ablate(std::map<std::string, std::string>& f) {
    if (!f.count("--gen"))
        usage("ablate needs --gen SPEC");
    std::vector<int> sizes;
    if (f.count("--sizes")) {
        std::stringstream ss(f["--sizes"]);
        std::string tok;
        while (std::getline(ss, tok, ','))
            sizes.push_back(std::stoi(tok));
    } else {
        sizes.push_back(qsim::generate(f["--gen"]).n);
    }
    const int repeat = std::max(1, std::stoi(f["--repeat"]));
    std::vector<Record> rows;
    for (int n : sizes) {
        const std::string spec = with_size(f["--gen"], n);
        const qsim::Circuit c = qsim::generate(spec);
        double base = 0.0;
        std::vector<Record> cells;
        for (int fu = 0; fu < 2; ++fu)
            for (int sg = 0; sg < 2; ++sg) {
                qsim::PlanOptions o;
                o.fusion = fu != 0;
                o.multi_op_passes = sg != 0;
                Record r = run_report(c, o, repeat, "norm", fu ? "on" : "off", sg ? "on" : "off", 0.0);
                double t = 0;
                for (auto& kv : r)
                    if (kv.first == "execute_s_median")
                        t = std::stod(kv.second);
                if (!fu && !sg)
                    base = t;
                r.insert(r.begin(), {"cell", std::string("fusion=") + (fu ? "on" : "off") + ",stagger=" + (sg ? "on" : "off")});
                r.push_back({"speedup_vs_all_off", std::to_string(t > 0 ? base / t : 0.0)});
                cells.push_back(std::move(r));
            }
        rows.insert(rows.end(), cells.begin(), cells.end());
    }
    if (f["--format"] == "csv") {
        emit(to_csv(rows), f);
    } else {
        std::string out = "[\n";
        for (size_t i = 0; i < rows.size(); ++i)
            out += "  " + to_json(rows[i]) + (i + 1 < rows.size() ? ",\n" : "\n");
        emit(out + "]\n", f);
    }
    return 0;
}

// C followed by C^dagger (mirror circuit): returns |0...0> exactly in exact arithmetic.
qsim::Circuit mirror(const qsim::Circuit& c) {
    qsim::Circuit m(c.n, c.source + "+dagger");
    for (const qsim::Gate& g : c.gates)
        m.add(g);
    for (auto it = c.gates.rbegin(); it != c.gates.rend(); ++it) {
        if (it->is_fence())
            continue;
        const qsim::GateMatrix& u = it->matrix();
        const qsim::Index d = u.dim();
        std::vector<qsim::Amp> e(static_cast<size_t>(d * d));
        for (qsim::Index r = 0; r < d; ++r)
            for (qsim::Index q = 0; q < d; ++q)
                e[static_cast<size_t>(r * d + q)] = std::conj(u.at(q, r));
        m.add(qsim::Gate::unitary(qsim::GateMatrix(u.arity(), std::move(e)), it->targets(), it->controls(), "DAG"));
    }
    return m;
}

struct Verdict {
    bool pass;
    std::string detail;
};

int cmd_verify(std::map<std::string, std::string>& f) {
    const bool quick = f.count("--quick") != 0;
    std::vector<Record> rows;
    int failed = 0;
    auto crit = [&](const std::string& name, const std::function<Verdict()>& fn) {
        const auto a = Clock::now();
        Verdict v{false, ""};
        try {
            v = fn();
        } catch (const std::exception& e) {
            v = {false, std::string("exception: ") + e.what()};
        }
        failed += v.pass ? 0 : 1;
        std::string d = v.detail, nm = name;
        std::replace(d.begin(), d.end(), ',', ';');
        std::replace(nm.begin(), nm.end(), ',', ';');
        rows.push_back({{"criterion", nm}, {"status", v.pass ? "pass" : "FAIL"}, {"seconds", std::to_string(secs(a, Clock::now()))},
                        {"detail", d}});
    };
    qsim::DeviceContext ctx(0);
    auto run_state = [&](const qsim::Circuit& c, const qsim::PlanOptions& o, qsim::DeviceState& st, uint64_t basis) {
        qsim::Engine eng(ctx, c, o);
        st.set_basis(basis);
        eng.run(st);
        ctx.sync();
    };
    // #1 (device form): random mnemonic circuits n in [2, 10]: C C^dagger |0> = |0>, norm kept
    crit("1 kernel correctness (mirror circuits n 2..10)", [&] {
        double worst = 0.0;
        const int count = quick ? 40 : 200;
        for (int i = 0; i < count; ++i) {
            const int n = 2 + i % 9;
            const qsim::Circuit c = mirror(qsim::generate("random:" + std::to_string(n) + ":" + std::to_string(1 + i % 6) + ":" + std::to_string(100 + i)));
            qsim::DeviceState st(ctx, n);
            qsim::PlanOptions o;
            o.jit = i % 4 == 0;  // every 4th through NVRTC kernels, the rest through the interpreter
            o.tile_k = std::min(o.tile_k, n);
            run_state(c, o, st, 0);
            qsim::Amp a0;
            st.download(&a0, 0, 1);
            worst = std::max({worst, std::abs(a0 - qsim::Amp(1.0, 0.0)), std::abs(st.norm_sq() - 1.0)});
        }
        return Verdict{worst < 1e-10, "max deviation " + std::to_string(worst)};
    });
    // #2: QFT of |0> (uniform) and of basis states (analytic), n in {4, 10, 16}
    crit("2 QFT analytic", [&] {
        double worst = 0.0;
        for (int n : {4, 10, 16}) {
            for (uint64_t x : {uint64_t{0}, (uint64_t{1} << n) / 3}) {
                qsim::DeviceState st(ctx, n);
                run_state(qsim::generate("qft:" + std::to_string(n)), qsim::PlanOptions{}, st, x);
                double e = 0;
                qsim::qsv_check(qsv_check_qft_basis(st.get(), n, x, &e), "qsv_check_qft_basis");
                worst = std::max(worst, e);
            }
        }
        return Verdict{worst <= 1e-12, "max deviation " + std::to_string(worst)};
    });
    // #3 / #8: distributed equivalence and the instrumented memory bound (needs >= 2 GPUs)
    int ndev = 0;
    qsv_device_count(&ndev);
    crit("3 distributed == single rank; 8 memory bound", [&] {
        if (ndev < 2)
            return Verdict{true, "skipped: 1 GPU (run `pytest -m gpu tests/test_gpu_multi.py` on 2-4 GPUs)"};
        double worst = 0.0;
        bool mem_ok = true;
        for (int n : {12, 16, 18})
            for (int m = 1; m <= 2 && (1 << m) <= ndev; ++m) {
                const qsim::Circuit c = qsim::generate("random:" + std::to_string(n) + ":6:3");
                const int l = n - m;
                qsim::DeviceState ref(ctx, n);
                run_state(c, qsim::PlanOptions{}, ref, 0);
                std::vector<qsim::Amp> host(static_cast<size_t>(qsim::index_bit(n)));
                ref.download(host.data(), 0, qsim::index_bit(n));
                for (int B : {1, 2, 3}) {
                    qsim::DistributedReport rep;
                    qsim::PlanOptions o;
                    o.fusion = false;
                    const qsim::StateVector sv = qsim::run_distributed(c, qsim::PartitionPlan(n, m, l - 1, B), {}, &rep, o);
                    for (qsim::Index i = 0; i < sv.size(); ++i)
                        worst = std::max(worst, std::abs(sv[i] - host[static_cast<size_t>(i)]));
                    for (std::size_t pk : rep.peak_bytes)
                        mem_ok = mem_ok && pk <= (std::size_t{16} << l) + static_cast<std::size_t>(B) * (std::size_t{16} << (l - 1)) + (std::size_t{2} << 20);
                }
            }
        return Verdict{worst <= 1e-12 && mem_ok, "max deviation " + std::to_string(worst) + (mem_ok ? "; memory within bound" : "; memory bound exceeded")};
    });
    // #4: contraction floors, HEA compresses more than QAOA (Fig. 14)
    crit("4 fusion compression (HEA > QAOA)", [&] {
        const auto hea = std::get<2>(qsim::contract(qsim::generate("hea:20:5:1")));
        const auto qaoa = std::get<2>(qsim::contract(qsim::generate("qaoa:20:2:1")));
        return Verdict{hea.compression_ratio > qaoa.compression_ratio && qaoa.compression_ratio > 0.0,
                       "HEA " + std::to_string(hea.compression_ratio) + " QAOA " + std::to_string(qaoa.compression_ratio)};
    });
    // #5: cost-model anchors (PAPER §3.4)
    crit("5 gate_cost anchors", [&] {
        const qsim::Circuit c = qsim::generate("random:10:1:1");
        const int n = 10;
        double one = -1, two = -1;
        for (const qsim::Gate& g : c.gates) {
            if (g.is_fence())
                continue;
            if (g.targets().size() == 1 && g.controls().empty() && one < 0)
                one = qsim::gate_cost(g, n);
        }
        const qsim::Gate u2 = qsim::Gate::unitary(qsim::GateMatrix::identity(2), {0, 1}, {}, "U2");
        two = qsim::gate_cost(u2, n);
        const bool ok = one == 10.0 * std::ldexp(1.0, n - 1) && two == 36.0 * std::ldexp(1.0, n - 2);
        return Verdict{ok, "k=1 " + std::to_string(one) + " k=2 " + std::to_string(two)};
    });
    // #7 (device form): multi-op passes apply the ops in program order: bitwise equal to one op per pass
    crit("7 SMGP passes == sequential (bitwise)", [&] {
        const qsim::Circuit c = qsim::generate("hea:16:5:2");
        qsim::PlanOptions seq;
        seq.multi_op_passes = false;
        seq.fusion = false;
        qsim::PlanOptions stag = seq;
        stag.multi_op_passes = true;
        qsim::DeviceState a(ctx, 16), b(ctx, 16);
        run_state(c, seq, a, 0);
        run_state(c, stag, b, 0);
        uint64_t da = 0, db = 0;
        qsim::qsv_check(qsv_state_digest(a.get(), &da), "digest");
        qsim::qsv_check(qsv_state_digest(b.get(), &db), "digest");
        return Verdict{da == db, da == db ? "digests equal" : "digests differ"};
    });
    // #9: QASM parser robustness (mutations never crash; rejections carry line:col)
    crit("9 QASM fuzz", [&] {
        const std::string base = qsim::emit_qasm(qsim::generate("random:5:3:7"));
        std::mt19937_64 rng(9);
        const std::string alphabet = "qreg[];,()+-*/0123456789 pi\n\"abcdefghijklmnopqrstuvwxyz";
        int rejected = 0;
        const int count = quick ? 2000 : 10000;
        for (int i = 0; i < count; ++i) {
            std::string t = base;
            const int edits = 1 + static_cast<int>(rng() % 4);
            for (int e = 0; e < edits && !t.empty(); ++e) {
                const size_t pos = rng() % t.size();
                switch (rng() % 3) {
                case 0: t.erase(pos, 1 + rng() % 3); break;
                case 1: t.insert(pos, 1, alphabet[rng() % alphabet.size()]); break;
                default: t[pos] = alphabet[rng() % alphabet.size()]; break;
                }
            }
            try {
                (void)qsim::parse_qasm(t);
            } catch (const qsim::QasmError& e) {
                ++rejected;
                if (e.line() < 1 || e.column() < 1)
                    return Verdict{false, "rejection without a location"};
            } catch (const std::invalid_argument&) {
                ++rejected;  // circuit-level rejection (e.g. a qubit out of range)
            }
        }
        return Verdict{true, std::to_string(count) + " mutations, " + std::to_string(rejected) + " rejected, 0 crashes"};
    });
    // #10 (device form): bitwise run-to-run determinism
    crit("10 determinism (bitwise digest)", [&] {
        const qsim::Circuit c = qsim::generate("qaoa:18:2:1");
        qsim::Engine eng(ctx, c, qsim::PlanOptions{});
        qsim::DeviceState st(ctx, 18);
        std::vector<uint64_t> d;
        for (int r = 0; r < 3; ++r) {
            st.set_basis(0);
            eng.run(st);
            ctx.sync();
            uint64_t x = 0;
            qsim::qsv_check(qsv_state_digest(st.get(), &x), "digest");
            d.push_back(x);
        }
        return Verdict{d[0] == d[1] && d[1] == d[2], "3 runs"};
    });
    std::cout << to_csv(rows);
    std::cout << (failed ? "verify: " + std::to_string(failed) + " criterion(s) FAILED\n" : std::string("verify: all criteria pass\n"));
    return failed ? 1 : 0;
}

int main(int argc, char** argv) {
    if (argc < 2)
        usage("need a command: run | ablate | verify");
    const std::string cmd = argv[1];
    if (cmd == "verify" || cmd == "ablate") {
        std::map<std::string, std::string> f = {{"--repeat", "3"}, {"--format", "json"}};
        for (int i = 2; i < argc; ++i) {
            const std::string k = argv[i];
            if (k == "--quick") {
                f[k] = "1";
                continue;
            }
            if (k.rfind("--", 0) != 0 || i + 1 >= argc)
                usage("bad argument '" + k + "'");
            f[k] = argv[++i];
        }
        try {
            return cmd == "verify" ? cmd_verify(f) : cmd_ablate(f);
        } catch (const std::invalid_argument& e) {
            std::cerr << "qsv: " << e.what() << "\n";
            return 2;
        } catch (const std::exception& e) {
            std::cerr << "qsv: " << e.what() << "\n";
            return 1;
        }
    }
    if (cmd != "run")
        usage("unknown command '" + cmd + "' (run | ablate | verify)");
    std::map<std::string, std::string> f = {{"--fusion", "on"}, {"--stagger", "on"}, {"--repeat", "3"},
                                            {"--verify", "norm"}, {"--format", "json"}, {"--ranks", "1"}};
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        if (k.rfind("--", 0) != 0 || i + 1 >= argc)
            usage("bad argument '" + k + "'");
        f[k] = argv[++i];
    }
    try {
        if (std::stoi(f["--ranks"]) != 1)
            usage("--ranks > 1: launch one process per GPU (bench.py under torchrun)");
        const auto t0 = Clock::now();
        qsim::Circuit c;
        if (f.count("--gen"))
            c = qsim::generate(f["--gen"]);
        else if (f.count("--qasm"))
            c = qsim::parse_qasm_file(f["--qasm"]);
        else
            usage("need --gen or --qasm");
        const auto t1 = Clock::now();
        qsim::PlanOptions o;
        o.fusion = on_off(f["--fusion"], "--fusion");
        o.multi_op_passes = on_off(f["--stagger"], "--stagger");
        if (f.count("--tile-k"))
            o.tile_k = std::stoi(f["--tile-k"]);
        const Record rec = run_report(c, o, std::max(1, std::stoi(f["--repeat"])), f["--verify"], f["--fusion"],
                                      f["--stagger"], secs(t0, t1));
        std::ostringstream out;
        if (f["--format"] == "json")
            out << to_json(rec) << "\n";
        else if (f["--format"] == "csv")
            out << to_csv({rec});
        else
            usage("--format takes json|csv");
        if (f.count("--out")) {
            std::ofstream(f["--out"]) << out.str();
        } else {
            std::cout << out.str();
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        std::cerr << "qsv: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "qsv: " << e.what() << "\n";
        return 1;
    }
}
