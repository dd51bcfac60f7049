// `qsv` — thin run/report driver over the B200 engine.
// Reconstructed from the reference CMake target tools/qsv.cpp (proj/CMakeLists.txt:40-41,
// absent upstream) and the SPEC flag list.  It parses or generates a
// circuit, plans it (DAGC + SMGP + BBOP), runs it on the GPU `--repeat` times and prints a
// RunReport as JSON or CSV with identical values.
//
//   qsv run (--gen SPEC | --qasm FILE) [--fusion on|off] [--stagger on|off] [--repeat R]
//           [--tile-k K] [--verify none|norm|qft:X] [--format json|csv] [--out FILE]
//
// Multi-GPU runs go through bench.py / torchrun (one process per GPU); --ranks is accepted
// for flag compatibility and must be 1 here.  --verify never uses the CPU oracle (test
// infrastructure): `norm` checks the device norm, `qft:X` the analytic QFT of basis state X.
#include "qsim/device.hpp"
#include "qsim/generators.hpp"
#include "qsim/qasm.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
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
              << "               [--format json|csv] [--out FILE]\n";
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

int main(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) != "run")
        usage("the only command is `run`");
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
        qsim::DeviceContext ctx(0);
        qsim::Engine eng(ctx, c, o);
        const auto t2 = Clock::now();
        qsim::DeviceState st(ctx, c.n);
        const int repeat = std::max(1, std::stoi(f["--repeat"]));
        std::vector<double> exec;
        const std::string verify = f["--verify"];
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
        std::vector<std::pair<std::string, std::string>> rec = {
            {"source", c.source},
            {"qubits", std::to_string(c.n)},
            {"ranks", "1"},
            {"fusion", f["--fusion"]},
            {"stagger", f["--stagger"]},
            {"tile_k", std::to_string(o.tile_k)},
            {"repeat", std::to_string(repeat)},
            {"parse_s", std::to_string(secs(t0, t1))},
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
        std::ostringstream out;
        if (f["--format"] == "json") {
            out << "{";
            for (size_t i = 0; i < rec.size(); ++i) {
                const bool num = rec[i].first != "source" && rec[i].first != "fusion" && rec[i].first != "stagger" &&
                                 rec[i].first != "verify";
                out << (i ? ", " : "") << '"' << rec[i].first << "\": " << (num ? "" : "\"") << rec[i].second
                    << (num ? "" : "\"");
            }
            out << "}\n";
        } else if (f["--format"] == "csv") {
            for (size_t i = 0; i < rec.size(); ++i)
                out << (i ? "," : "") << rec[i].first;
            out << "\n";
            for (size_t i = 0; i < rec.size(); ++i)
                out << (i ? "," : "") << rec[i].second;
            out << "\n";
        } else {
            usage("--format takes json|csv");
        }
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
