// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference implementation (Quokka, the C++
// re-creation of Queen, /root/reference/proj), compiled with the namespace
// renamed to quokka_ref (-Dquokka=quokka_ref) so it can sit beside the
// product's own `quokka::` symbols in one process.  Only tests/, smoke()
// and bench.py's cpu_baseline / --impl reference leg load this library.
//
// Every entry point is a thin adapter from plain pointers / text to the
// reference's public API:
//   gen*             -> proj/src/tools.cpp:169-272
//   aioOptimize      -> proj/src/optimizer.cpp:478-485
//   simulateProgram  -> proj/src/engine.cpp:283-297
//   spawnRanks       -> proj/src/distributed.cpp:140-206
//   applyBlock       -> proj/src/engine.cpp:262-281
//   applyGate        -> proj/src/engine.cpp:258-260
//   imsSwap          -> proj/src/engine.cpp:86-101
//   xrsSwap          -> proj/src/distributed.cpp:124-138
//   oracleSimulate   -> proj/src/tools.cpp:10-40
//   layoutApply      -> proj/src/tools.cpp:42-55
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "quokka/circuit.hpp"
#include "quokka/distributed.hpp"
#include "quokka/engine.hpp"
#include "quokka/optimizer.hpp"
#include "quokka/tools.hpp"

using namespace quokka;  // expands to quokka_ref

namespace {

thread_local std::string g_err;

char* dupString(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

template <class F>
int guard(F f) {
    try {
        f();
        return 0;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 1;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const SimulationError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

Config cfgFromText(const char* text) {
    std::istringstream in(text);
    return parseConfig(in);
}

void copyOut(const std::vector<Amp>& amps, double* out) {
    std::memcpy(out, amps.data(), amps.size() * sizeof(Amp));
}

void copyIn(StateVector& sv, int n, const double* in) {
    sv.nQubits = n;
    sv.amps.resize(Index(1) << n);
    std::memcpy(sv.amps.data(), in, sv.amps.size() * sizeof(Amp));
}

std::vector<std::pair<int, int>> pairsOf(const int* outs, const int* ins, int s) {
    std::vector<std::pair<int, int>> p;
    for (int i = 0; i < s; i++) p.emplace_back(outs[i], ins[i]);
    return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

// kind: "qft" | "qaoa" | "bv" | "bvones" | "random" | "bench:<KIND>"
int ref_gen(const char* kind, int n, long a, unsigned long long seed, char** out) {
    return guard([&] {
        std::string k = kind;
        Circuit c;
        if (k == "qft") c = genQft(n);
        else if (k == "qaoa") c = genQaoa(n, int(a), seed);
        else if (k == "bv") c = genBv(n, seed);
        else if (k == "bvones") c = genBvAllOnes(n);
        else if (k == "random") c = genRandom(n, int(a), seed);
        else if (k.rfind("bench:", 0) == 0) {
            std::string tok = k.substr(6);
            GateKind gk = GateKind::H;
            const char* names[] = {"H", "U", "X", "CX", "CP", "SWAP", "RX", "RY", "RZ", "RZZ"};
            GateKind kinds[] = {GateKind::H,  GateKind::U,    GateKind::X,  GateKind::CX,
                                GateKind::CP, GateKind::SWAP, GateKind::RX, GateKind::RY,
                                GateKind::RZ, GateKind::RZZ};
            bool found = false;
            for (int i = 0; i < 10; i++)
                if (tok == names[i]) { gk = kinds[i]; found = true; }
            if (!found) throw ConfigError("unknown bench kind");
            c = genGateBench(gk, n);
        } else {
            throw ConfigError("unknown generator " + k);
        }
        *out = dupString(serializeCircuit(c));
    });
}

int ref_optimize(const char* circuitText, const char* cfgText, char** out) {
    return guard([&] {
        Config cfg = cfgFromText(cfgText);
        std::istringstream in(circuitText);
        Circuit c = parseCircuit(in, cfg.totalQubits);
        Program p = aioOptimize(c, cfg);
        *out = dupString(serializeProgram(p));
    });
}

// Parse + re-serialize (program text normal form / parser parity).
int ref_program_roundtrip(const char* progText, const char* cfgText, int lenient, char** out) {
    return guard([&] {
        Config cfg = cfgFromText(cfgText);
        std::istringstream in(progText);
        Program p = parseProgram(in, cfg, lenient != 0);
        *out = dupString(serializeProgram(p));
    });
}

int ref_circuit_roundtrip(const char* text, int n, char** out) {
    return guard([&] {
        std::istringstream in(text);
        *out = dupString(serializeCircuit(parseCircuit(in, n)));
    });
}

int ref_config_roundtrip(const char* text, char** out) {
    return guard([&] { *out = dupString(serializeConfig(cfgFromText(text))); });
}

// Full program run. state: 2^N complex (interleaved) out, physical order.
// physToLog: N ints out. stats (R>0): per rank {bytesSent, bytesReceived,
// peakBufferBytes, rounds} as 4 u64 each. seconds: wall time of the run.
int ref_simulate(const char* progText, const char* cfgText, unsigned long long initial,
                 int threads, double* state, int* physToLog, unsigned long long* stats,
                 double* seconds) {
    return guard([&] {
        Config cfg = cfgFromText(cfgText);
        std::istringstream in(progText);
        Program p = parseProgram(in, cfg);
        auto t0 = std::chrono::steady_clock::now();
        if (cfg.rankQubits == 0) {
            SimResult r = simulateProgram(p, cfg, initial, threads);
            auto t1 = std::chrono::steady_clock::now();
            if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
            if (state) copyOut(r.state.amps, state);
            if (physToLog)
                for (int i = 0; i < p.nQubits; i++) physToLog[i] = r.layout.physToLog[i];
        } else {
            MultiRankResult r = spawnRanks(p, cfg, initial);
            auto t1 = std::chrono::steady_clock::now();
            if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
            if (state) copyOut(r.state.amps, state);
            if (physToLog)
                for (int i = 0; i < p.nQubits; i++) physToLog[i] = r.layout.physToLog[i];
            if (stats)
                for (size_t k = 0; k < r.stats.size(); k++) {
                    stats[4 * k + 0] = r.stats[k].bytesSent;
                    stats[4 * k + 1] = r.stats[k].bytesReceived;
                    stats[4 * k + 2] = r.stats[k].peakBufferBytes;
                    stats[4 * k + 3] = r.stats[k].rounds;
                }
        }
    });
}

// Timed applyBlock/imsSwap loop on a caller-owned state (bounded CPU sample
// for bench.py): runs items [first, last) of the program over `state`.
int ref_run_items(const char* progText, const char* cfgText, double* state, int first, int last,
                  int threads, double* seconds) {
    return guard([&] {
        Config cfg = cfgFromText(cfgText);
        std::istringstream in(progText);
        Program p = parseProgram(in, cfg);
        StateVector sv;
        copyIn(sv, p.nQubits - p.rankQubits, state);
        auto t0 = std::chrono::steady_clock::now();
        for (int i = first; i < last && i < int(p.items.size()); i++) {
            const ProgramItem& it = p.items[i];
            if (it.type == ProgramItem::Block)
                applyBlock(sv, it.block, p.chunkQubits, threads);
            else if (it.swap.kind == SwapOp::InMemory)
                imsSwap(sv, it.swap, cfg.cacheLineQubits, threads);
        }
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        copyOut(sv.amps, state);
    });
}

// applyBlock on a caller state; block = the gate lines (physical positions).
int ref_apply_block(double* state, int n, const char* gateLines, int chunkQubits, int threads) {
    return guard([&] {
        StateVector sv;
        copyIn(sv, n, state);
        GateBlock blk;
        std::istringstream in(gateLines);
        std::string line;
        int no = 0;
        while (std::getline(in, line)) {
            no++;
            bool blank = true;
            for (char ch : line)
                if (!isspace(static_cast<unsigned char>(ch))) blank = false;
            if (blank) continue;
            blk.gates.push_back(parseGateLine(line, no));
        }
        applyBlock(sv, blk, chunkQubits, threads);
        copyOut(sv.amps, state);
    });
}

int ref_apply_gate(double* state, int n, const char* gateLine) {
    return guard([&] {
        StateVector sv;
        copyIn(sv, n, state);
        applyGate(sv, parseGateLine(gateLine, 1));
        copyOut(sv.amps, state);
    });
}

int ref_ims_swap(double* state, int n, const int* outs, const int* ins, int s, int cl,
                 int threads) {
    return guard([&] {
        StateVector sv;
        copyIn(sv, n, state);
        SwapOp op;
        op.kind = SwapOp::InMemory;
        op.pairs = pairsOf(outs, ins, s);
        imsSwap(sv, op, cl, threads);
        copyOut(sv.amps, state);
    });
}

unsigned long long ref_bitswap(unsigned long long x, const int* outs, const int* ins, int s) {
    return bitswap(x, pairsOf(outs, ins, s));
}

unsigned long long ref_bitshift(unsigned long long x, const int* outs, const int* ins, int s,
                                int cl) {
    return bitshift(x, pairsOf(outs, ins, s), cl);
}

// xrsSwap over the full 2^n state split into 2^r slices (rank-major).
int ref_xrs_swap(double* state, int n, int r, int bufferQubits, const int* outs, const int* ins,
                 int s, unsigned long long* stats) {
    return guard([&] {
        Config cfg;
        cfg.totalQubits = n;
        cfg.rankQubits = r;
        cfg.chunkQubits = 1;
        cfg.fusionQubits = 1;
        cfg.bufferQubits = bufferQubits;
        cfg.finalize();
        int ranks = 1 << r;
        Index per = Index(1) << (n - r);
        std::vector<std::vector<Amp>> slices(ranks);
        const Amp* src = reinterpret_cast<const Amp*>(state);
        for (int k = 0; k < ranks; k++) slices[k].assign(src + k * per, src + (k + 1) * per);
        SwapOp op;
        op.kind = SwapOp::CrossRank;
        op.pairs = pairsOf(outs, ins, s);
        std::vector<RankStats> st(ranks);
        xrsSwap(slices, op, cfg, &st);
        Amp* dst = reinterpret_cast<Amp*>(state);
        for (int k = 0; k < ranks; k++)
            std::memcpy(dst + k * per, slices[k].data(), per * sizeof(Amp));
        if (stats)
            for (int k = 0; k < ranks; k++) {
                stats[4 * k + 0] = st[k].bytesSent;
                stats[4 * k + 1] = st[k].bytesReceived;
                stats[4 * k + 2] = st[k].peakBufferBytes;
                stats[4 * k + 3] = st[k].rounds;
            }
    });
}

int ref_oracle_simulate(const char* circuitText, int n, unsigned long long initial,
                        double* state) {
    return guard([&] {
        std::istringstream in(circuitText);
        Circuit c = parseCircuit(in, n);
        copyOut(oracleSimulate(c, initial).amps, state);
    });
}

int ref_layout_apply(double* state, int n, const int* physToLog) {
    return guard([&] {
        StateVector sv;
        copyIn(sv, n, state);
        QubitLayout l = QubitLayout::identity(n);
        for (int p = 0; p < n; p++) {
            l.physToLog[p] = physToLog[p];
            l.logToPhys[physToLog[p]] = p;
        }
        copyOut(layoutApply(sv, l).amps, state);
    });
}

// validateOrder: 1 = ok, 0 = not ok (message via ref_last_error).
int ref_validate_order(const char* circuitText, const char* progText, const char* cfgText) {
    int ok = 0;
    int rc = guard([&] {
        Config cfg = cfgFromText(cfgText);
        std::istringstream ci(circuitText);
        Circuit c = parseCircuit(ci, cfg.totalQubits);
        std::istringstream pi(progText);
        Program p = parseProgram(pi, cfg);
        OrderReport r = validateOrder(c, p);
        ok = r.ok ? 1 : 0;
        if (!r.ok) g_err = r.message;
    });
    return rc ? -rc : ok;
}

}  // extern "C"
