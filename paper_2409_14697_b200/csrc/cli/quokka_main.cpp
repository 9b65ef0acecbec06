// `quokka_b200`: command-line drop-in for the reference CLI's hot-path
// subcommands (proj/tools/main.cpp:290-377), on the B200 engine.
//
//   quokka_b200 optimize -i circuit [-o program] --config cfg.ini
//   quokka_b200 optimize circuit chunk inrank total ims xrs fusion_qbit fusion
//   quokka_b200 simulate -i cfg.ini -c program [--raw] [--dump-state] [--initial K]
//   quokka_b200 validate circuit program [-i cfg.ini]
//   quokka_b200 tune -i circuit -n N [-r R] [-o cfg.ini]        (GPU-aware config, this framework's addition)
//   quokka_b200 gen qft|qaoa|bv|gate|random|grover -n N [-o file] [-l L] [-g G]
//                   [--seed S] [--secret X] [--kind K]
//   quokka_b200 bench [-n N] [-g G] [--seed S] [--engine blockwise|gate_by_gate]
//                     [--compare] [--repeats R] [--circuit random|qft|qaoa] [--threads T]
//
// Same outputs and exit codes as the reference: program / circuit text,
// "qubits: / gates: / wall_time_s: / norm:" on stdout, "index re im" lines for
// --dump-state (<= 20 qubits, logical order), 1 ParseError, 2 ConfigError
// (also bad command lines), 3 SimulationError.  The simulation runs on cuda:0
// with the state resident in HBM; simulate's wall time spans initState to the
// last item (main.cpp:126-145).  No CLI11: a small parser of its own.
#include <algorithm>
#include <cctype>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "qk.h"
#include "quokka/distributed.hpp"
#include "quokka/engine.hpp"
#include "quokka/optimizer.hpp"
#include "quokka/tools.hpp"

namespace {

using namespace quokka;

struct Args {
    std::vector<std::string> positional;
    std::map<std::string, std::string> opts;  // canonical long name -> value ("" for flags)
};

// name aliases: short -> long, and which options are flags
Args parseArgs(int argc, char** argv, int first, const std::map<std::string, std::string>& alias,
               const std::vector<std::string>& flags) {
    Args a;
    for (int i = first; i < argc; i++) {
        std::string t = argv[i];
        if (t.size() > 1 && t[0] == '-' && !(t.size() > 1 && (std::isdigit(static_cast<unsigned char>(t[1])) != 0))) {
            std::string name = t, value;
            const size_t eq = t.find('=');
            if (eq != std::string::npos) {
                name = t.substr(0, eq);
                value = t.substr(eq + 1);
            }
            auto it = alias.find(name);
            if (it == alias.end()) throw ConfigError("unknown option " + name);
            name = it->second;
            const bool isFlag = std::find(flags.begin(), flags.end(), name) != flags.end();
            if (!isFlag && eq == std::string::npos) {
                if (i + 1 >= argc) throw ConfigError("option " + name + " needs a value");
                value = argv[++i];
            }
            a.opts[name] = value;
        } else {
            a.positional.push_back(t);
        }
    }
    return a;
}

void writeText(const std::string& path, const std::string& text) {
    if (path.empty()) {
        std::cout << text;
        return;
    }
    std::ofstream out(path);
    if (!out) throw ParseError("cannot open output file: " + path);
    out << text;
}

// Base-10 parsing like the reference (std::stoi / CLI11's integral options).
long long toInt(const std::string& s, const std::string& what) {
    try {
        size_t pos = 0;
        const long long v = std::stoll(s, &pos, 10);
        if (pos != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (...) {
        throw ConfigError("bad numeric parameter '" + s + "' for " + what);
    }
}

// uint64 options (--initial, --seed, --secret): the full unsigned range.
std::uint64_t toU64(const std::string& s, const std::string& what) {
    try {
        size_t pos = 0;
        if (!s.empty() && s[0] == '-') throw std::invalid_argument(s);
        const unsigned long long v = std::stoull(s, &pos, 10);
        if (pos != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (...) {
        throw ConfigError("bad numeric parameter '" + s + "' for " + what);
    }
}

double seconds(std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

int runOptimize(const Args& a) {
    Config cfg;
    std::string input = a.opts.count("--input") ? a.opts.at("--input") : "";
    std::vector<std::string> nums = a.positional;
    if (a.opts.count("--config")) {
        if (!nums.empty() && !(input.empty() && nums.size() == 1))
            throw ConfigError("--config and the positional parameter form are exclusive");
        if (input.empty() && !nums.empty()) input = nums.front();
        cfg = parseConfigFile(a.opts.at("--config"));
    } else {
        // compatibility form: circuit chunk inrank total ims xrs fusion_qbit fusion
        if (input.empty() && !nums.empty()) {
            input = nums.front();
            nums.erase(nums.begin());
        }
        if (nums.size() != 7)
            throw ConfigError("expected: optimize <circuit> <chunk_qbit> <inrank_qbit> <total_qbit> <ims> <xrs> "
                              "<fusion_qbit> <fusion>");
        long long v[7];
        for (int i = 0; i < 7; i++) v[i] = toInt(nums[size_t(i)], "optimize");
        cfg.chunkQubits = int(v[0]);
        cfg.totalQubits = int(v[2]);
        cfg.rankQubits = int(v[2] - v[1]);
        cfg.imsEnabled = v[3] != 0;
        cfg.xrsEnabled = v[4] != 0;
        cfg.fusionQubits = int(v[5]);
        cfg.fusionEnabled = v[6] != 0;
        cfg.diagonalFusionEnabled = v[6] != 0;
        cfg.finalize();
    }
    if (input.empty()) throw ConfigError("no circuit file given");
    const Circuit c = parseCircuitFile(input, cfg.totalQubits);
    const auto t0 = std::chrono::steady_clock::now();
    const Program p = aioOptimize(c, cfg);
    const auto t1 = std::chrono::steady_clock::now();
    writeText(a.opts.count("--output") ? a.opts.at("--output") : "", serializeProgram(p));
    std::cerr << "gates: " << c.gates.size() << " blocks: " << p.blockCount()
              << " in-memory swaps: " << p.swapCount(SwapOp::InMemory)
              << " cross-rank swaps: " << p.swapCount(SwapOp::CrossRank) << " wall_time_s: " << seconds(t0, t1)
              << "\n";
    return 0;
}

int runSimulate(const Args& a) {
    if (!a.opts.count("--config") || !a.opts.count("--circuit"))
        throw ConfigError("simulate needs -i <config> and -c <program>");
    const Config cfg = parseConfigFile(a.opts.at("--config"));
    const Index initial = a.opts.count("--initial") ? Index(toU64(a.opts.at("--initial"), "--initial")) : 0;
    const bool dump = a.opts.count("--dump-state") != 0;
    const bool dumpable = dump && cfg.totalQubits <= 20;  // the limit is reported after the summary (main.cpp:151-152)
    size_t gates = 0;
    double wall = 0, norm = 0;
    StateVector state;
    QubitLayout layout = QubitLayout::identity(cfg.totalQubits);
    if (a.opts.count("--raw")) {  // gate by gate (engine.cpp:299-322 semantics), on the device
        const Circuit c = parseCircuitFile(a.opts.at("--circuit"), cfg.totalQubits);
        gates = c.gates.size();
        const auto t0 = std::chrono::steady_clock::now();
        state = simulateGateByGate(c, initial);
        wall = seconds(t0, std::chrono::steady_clock::now());
        norm = state.norm();
    } else {
        const Program p = parseProgramFile(a.opts.at("--circuit"), cfg);
        gates = p.gateCount();
        if (cfg.rankQubits > 0) {
            const auto t0 = std::chrono::steady_clock::now();
            MultiRankResult r = spawnRanks(p, cfg, initial);
            wall = seconds(t0, std::chrono::steady_clock::now());
            state = std::move(r.state);
            layout = r.layout;
            size_t sent = 0, peak = 0;
            for (const RankStats& st : r.stats) {
                sent += st.bytesSent;
                peak = std::max(peak, st.peakBufferBytes);
            }
            std::cerr << "ranks: " << (1 << cfg.rankQubits) << " bytes_sent: " << sent
                      << " peak_buffer_bytes: " << peak << "\n";
            norm = state.norm();
        } else {
            DeviceState dev(cfg.totalQubits, 0, 0, 0, cfg.bufferQubits);  // resident: no host copy
            const auto t0 = std::chrono::steady_clock::now();
            simulateProgramDevice(dev, p, cfg, initial);
            wall = seconds(t0, std::chrono::steady_clock::now());
            norm = dev.norm();
            layout = p.finalLayout;
            if (dumpable) {
                state.nQubits = cfg.totalQubits;
                state.amps.resize(size_t(1) << cfg.totalQubits);
                dev.download(0, state.amps.size(), state.amps.data());
            }
        }
    }
    std::cout << "qubits: " << cfg.totalQubits << "\n";
    std::cout << "gates: " << gates << "\n";
    std::cout << "wall_time_s: " << fmt17(wall) << "\n";
    std::cout << "norm: " << fmt17(norm) << "\n";
    if (dump) {
        if (!dumpable) throw ConfigError("state dumps are limited to 20 qubits");
        const StateVector logical = layoutApply(state, layout);
        for (Index i = 0; i < Index(logical.amps.size()); i++)
            std::cout << i << " " << fmt17(logical.amps[i].real()) << " " << fmt17(logical.amps[i].imag()) << "\n";
    }
    return 0;
}

GateKind kindFromName(const std::string& name) {
    static const std::pair<const char*, GateKind> table[] = {
        {"H", GateKind::H},   {"U", GateKind::U},     {"X", GateKind::X},   {"CX", GateKind::CX},
        {"CP", GateKind::CP}, {"SWAP", GateKind::SWAP}, {"RX", GateKind::RX}, {"RY", GateKind::RY},
        {"RZ", GateKind::RZ}, {"RZZ", GateKind::RZZ},
    };
    for (const auto& e : table)
        if (name == e.first) return e.second;
    throw ConfigError("unknown gate kind '" + name + "'");
}

int runGen(const Args& a) {
    if (a.positional.size() != 1) throw ConfigError("gen needs exactly one generator name");
    if (!a.opts.count("--qubits")) throw ConfigError("gen needs -n <qubits>");
    const std::string which = a.positional[0];
    const int n = int(toInt(a.opts.at("--qubits"), "-n"));
    auto opt = [&](const char* k, long long d) { return a.opts.count(k) ? toInt(a.opts.at(k), k) : d; };
    auto optU = [&](const char* k, std::uint64_t d) { return a.opts.count(k) ? toU64(a.opts.at(k), k) : d; };
    const std::uint64_t seed = optU("--seed", 12345);
    Circuit c;
    if (which == "qft") c = genQft(n);
    else if (which == "qaoa") c = genQaoa(n, int(opt("--layers", 1)), seed);
    else if (which == "bv") c = a.opts.count("--secret") ? genBv(n, optU("--secret", 0)) : genBvAllOnes(n);
    else if (which == "gate") c = genGateBench(kindFromName(a.opts.count("--kind") ? a.opts.at("--kind") : "H"), n);
    else if (which == "random") c = genRandom(n, int(opt("--gates", 100)), seed);
    else if (which == "grover") c = genGrover(n, optU("--secret", 5), int(opt("--layers", 0)));
    else throw ConfigError("unknown generator '" + which + "'");
    writeText(a.opts.count("--output") ? a.opts.at("--output") : "", serializeCircuit(c));
    std::cerr << "qubits: " << c.nQubits << " gates: " << c.gates.size() << "\n";
    return 0;
}

// validate <circuit> <program> [-i cfg.ini] (main.cpp:167-192): exit 4 and
// "validation failed: ..." on stderr when the program is not a faithful
// reordering of the raw circuit.
int runValidate(const Args& a) {
    if (a.positional.size() != 2) throw ConfigError("validate needs <circuit> <program>");
    Config cfg;
    Circuit raw;
    Program p;
    if (a.opts.count("--config")) {
        cfg = parseConfigFile(a.opts.at("--config"));
        raw = parseCircuitFile(a.positional[0], cfg.totalQubits);
        p = parseProgramFile(a.positional[1], cfg);
    } else {
        raw = parseCircuitFile(a.positional[0]);
        cfg.totalQubits = raw.nQubits;
        cfg.rankQubits = 0;
        cfg.chunkQubits = raw.nQubits;
        cfg.cacheLineQubits = 0;
        cfg.fusionQubits = raw.nQubits;
        cfg.bufferQubits = raw.nQubits;
        p = parseProgramFile(a.positional[1], cfg, /*lenient=*/true);
    }
    const OrderReport rep = validateOrder(raw, p);
    if (!rep.ok) {
        std::cerr << "validation failed: " << rep.message << "\n";
        return 4;
    }
    std::cout << "Passed all circuit order validations\n";
    return 0;
}

// bench (main.cpp:236-286): the same CSV schema, median of --repeats timed
// runs per engine; "blockwise" = simulateProgram of the unfused Program,
// "gate_by_gate" = simulateGateByGate, both on the device here.
int runBench(const Args& a) {
    auto opt = [&](const char* k, long long d) { return a.opts.count(k) ? toInt(a.opts.at(k), k) : d; };
    const int n = int(opt("--qubits", 24)), ngates = int(opt("--gates", 200)), repeats = int(opt("--repeats", 10));
    const std::uint64_t seed = a.opts.count("--seed") ? toU64(a.opts.at("--seed"), "--seed") : 12345;
    const std::string circuit = a.opts.count("--circuit") ? a.opts.at("--circuit") : "random";
    Circuit c;
    if (circuit == "random") c = genRandom(n, ngates, seed);
    else if (circuit == "qft") c = genQft(n);
    else if (circuit == "qaoa") c = genQaoa(n, 1, seed);
    else throw ConfigError("unknown bench circuit '" + circuit + "'");
    Config cfg;
    cfg.totalQubits = n;
    cfg.rankQubits = 0;
    cfg.fusionEnabled = false;
    cfg.diagonalFusionEnabled = false;
    cfg.finalize();
    std::vector<std::string> engines;
    if (a.opts.count("--compare")) engines = {"blockwise", "gate_by_gate"};
    else engines = {a.opts.count("--engine") ? a.opts.at("--engine") : "blockwise"};
    std::cout << "name,n_qubits,ranks,gates,engine,wall_time_s,time_per_gate_s\n";
    double blockTime = 0.0, rawTime = 0.0;
    for (const std::string& eng : engines) {
        std::vector<double> times;
        if (eng == "blockwise") {
            const Program p = aioOptimize(c, cfg);
            for (int r = 0; r < repeats; r++) {
                const auto t0 = std::chrono::steady_clock::now();
                SimResult res = simulateProgram(p, cfg, 0, 0);
                times.push_back(seconds(t0, std::chrono::steady_clock::now()));
            }
        } else if (eng == "gate_by_gate") {
            for (int r = 0; r < repeats; r++) {
                const auto t0 = std::chrono::steady_clock::now();
                StateVector res = simulateGateByGate(c, 0, 0);
                times.push_back(seconds(t0, std::chrono::steady_clock::now()));
            }
        } else {
            throw ConfigError("unknown engine '" + eng + "' (blockwise, gate_by_gate)");
        }
        std::sort(times.begin(), times.end());
        const size_t m = times.size() / 2;
        const double med = times.empty() ? 0.0 : times.size() % 2 ? times[m] : 0.5 * (times[m - 1] + times[m]);
        (eng == "blockwise" ? blockTime : rawTime) = med;
        std::cout << circuit << "," << n << ",1," << c.gates.size() << "," << eng << "," << fmt17(med) << ","
                  << fmt17(med / double(c.gates.size())) << "\n";
    }
    if (engines.size() == 2 && blockTime > 0.0) std::cerr << "speedup: " << fmt17(rawTime / blockTime) << "\n";
    return 0;
}

// tune -i circuit -n N [-r R] [-o cfg.ini]: the GPU-aware configuration
// (qk_config_tune) as an INI file; the candidates and costs on stderr.  Then
// `optimize --config cfg.ini` produces the Program with the reference's
// optimizer, unchanged.
int runTune(const Args& a) {
    if (!a.opts.count("--input") && a.positional.empty()) throw ConfigError("tune needs -i <circuit>");
    if (!a.opts.count("--qubits")) throw ConfigError("tune needs -n <qubits>");
    const std::string path = a.opts.count("--input") ? a.opts.at("--input") : a.positional.front();
    const int n = int(toInt(a.opts.at("--qubits"), "-n"));
    const int r = a.opts.count("--rank-qubits") ? int(toInt(a.opts.at("--rank-qubits"), "-r")) : 0;
    std::ifstream in(path);
    if (!in) throw ParseError("cannot open circuit file: " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    qk_config c;
    char* report = nullptr;
    if (qk_config_tune(ss.str().c_str(), n, r, 0.0, &c, &report) != QK_OK) throw ConfigError(qk_last_error());
    std::cerr << report;
    qk_free(report);
    char* ini = nullptr;
    if (qk_config_serialize(&c, &ini) != QK_OK) throw ConfigError(qk_last_error());
    writeText(a.opts.count("--output") ? a.opts.at("--output") : "", ini);
    qk_free(ini);
    return 0;
}

int usage() {
    std::cerr << "usage: quokka_b200 optimize|simulate|validate|gen|bench|tune ... (see the header of "
                 "csrc/cli/quokka_main.cpp)\n";
    return 2;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        if (cmd == "optimize")
            return runOptimize(parseArgs(argc, argv, 2,
                                         {{"-i", "--input"}, {"--input", "--input"}, {"-o", "--output"},
                                          {"--output", "--output"}, {"--config", "--config"}},
                                         {}));
        if (cmd == "simulate")
            return runSimulate(parseArgs(argc, argv, 2,
                                         {{"-i", "--config"}, {"--config", "--config"}, {"-c", "--circuit"},
                                          {"--circuit", "--circuit"}, {"--raw", "--raw"},
                                          {"--dump-state", "--dump-state"}, {"--initial", "--initial"},
                                          {"--threads", "--threads"}},
                                         {"--raw", "--dump-state"}));
        if (cmd == "tune")
            return runTune(parseArgs(argc, argv, 2,
                                     {{"-i", "--input"}, {"--input", "--input"}, {"-n", "--qubits"},
                                      {"--qubits", "--qubits"}, {"-r", "--rank-qubits"},
                                      {"--rank-qubits", "--rank-qubits"}, {"-o", "--output"},
                                      {"--output", "--output"}},
                                     {}));
        if (cmd == "validate")
            return runValidate(parseArgs(argc, argv, 2, {{"-i", "--config"}, {"--config", "--config"}}, {}));
        if (cmd == "bench")
            return runBench(parseArgs(argc, argv, 2,
                                      {{"-n", "--qubits"}, {"--qubits", "--qubits"}, {"-g", "--gates"},
                                       {"--gates", "--gates"}, {"--seed", "--seed"}, {"--engine", "--engine"},
                                       {"--compare", "--compare"}, {"--repeats", "--repeats"},
                                       {"--circuit", "--circuit"}, {"--threads", "--threads"}},
                                      {"--compare"}));
        if (cmd == "gen")
            return runGen(parseArgs(argc, argv, 2,
                                    {{"-n", "--qubits"}, {"--qubits", "--qubits"}, {"-o", "--output"},
                                     {"--output", "--output"}, {"-l", "--layers"}, {"--layers", "--layers"},
                                     {"-g", "--gates"}, {"--gates", "--gates"}, {"--seed", "--seed"},
                                     {"--secret", "--secret"}, {"--kind", "--kind"}},
                                    {}));
        return usage();
    } catch (const ParseError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const ConfigError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const SimulationError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    }
}
