// Layout helpers and synthetic circuit generators (host side).
//
// Generators reproduce the reference's circuits gate for gate (same order,
// same ids, same RNG draws; proj/src/tools.cpp:169-272) so benchmark inputs
// and optimized Programs are identical; tests/test_host_formats.py compares
// the serialized text.  genGrover is this framework's addition.
#include <cmath>
#include <map>
#include <string>
#include <vector>

#include "quokka/tools.hpp"

namespace quokka {

namespace {
constexpr double kPi = 3.14159265358979323846;
}

StateVector layoutApply(const StateVector& sv, const QubitLayout& layout) {
    if (layout.size() != sv.nQubits) throw SimulationError("layout size does not match the state");
    if (layout.isIdentity()) return sv;
    StateVector out;
    out.nQubits = sv.nQubits;
    out.amps.resize(sv.amps.size());
    for (Index i = 0; i < Index(sv.amps.size()); i++) {
        Index logical = 0;
        for (int p = 0; p < sv.nQubits; p++) logical |= ((i >> p) & 1) << layout.physToLog[size_t(p)];
        out.amps[logical] = sv.amps[i];
    }
    return out;
}

double fidelity(const StateVector& u, const StateVector& v) {
    if (u.amps.size() != v.amps.size()) throw SimulationError("fidelity needs state vectors of equal size");
    Amp ip(0.0, 0.0);
    for (size_t i = 0; i < u.amps.size(); i++) ip += std::conj(u.amps[i]) * v.amps[i];
    return std::norm(ip);
}

Circuit genQft(int n) {
    Circuit c;
    c.nQubits = n;
    long id = 0;
    for (int t = 0; t < n; t++) {
        c.gates.push_back(makeH(t, id++));
        for (int ctl = t + 1; ctl < n; ctl++)
            c.gates.push_back(makeCP(ctl, t, kPi / double(Index(1) << (ctl - t)), id++));
    }
    return c;
}

Circuit genQaoa(int n, int layers, std::uint64_t seed) {
    Circuit c;
    c.nQubits = n;
    Rng rng(seed);
    long id = 0;
    for (int q = 0; q < n; q++) c.gates.push_back(makeH(q, id++));
    for (int layer = 0; layer < layers; layer++) {
        for (int a = 0; a < n; a++)
            for (int b = a + 1; b < n; b++) c.gates.push_back(makeRZZ(a, b, rng.nextDouble() * (2.0 * kPi), id++));
        for (int q = 0; q < n; q++) c.gates.push_back(makeRX(q, rng.nextDouble() * (2.0 * kPi), id++));
    }
    return c;
}

Circuit genBv(int n, std::uint64_t secret) {
    if (n < 2) throw ConfigError("the hidden-string circuit needs at least 2 qubits");
    secret &= (std::uint64_t(1) << (n - 1)) - 1;
    const int anc = n - 1;
    Circuit c;
    c.nQubits = n;
    long id = 0;
    c.gates.push_back(makeX(anc, id++));
    for (int q = 0; q < n; q++) c.gates.push_back(makeH(q, id++));
    for (int q = 0; q < anc; q++)
        if ((secret >> q) & 1) c.gates.push_back(makeCX(q, anc, id++));
    for (int q = 0; q < anc; q++) c.gates.push_back(makeH(q, id++));
    return c;
}

Circuit genBvAllOnes(int n) { return genBv(n, ~std::uint64_t(0)); }

Circuit genGateBench(GateKind kind, int n) {
    Circuit c;
    c.nQubits = n;
    long id = 0;
    auto angle = [n](int q) { return 2.0 * kPi * double(q + 1) / double(n + 1); };
    if (kindArity(kind) == 1) {
        for (int q = 0; q < n; q++) {
            std::vector<double> ps;
            if (kind == GateKind::U) ps = {angle(q), angle(q) / 2.0, angle(q) / 3.0};
            else if (kindParamCount(kind) == 1) ps = {angle(q)};
            c.gates.push_back(makeGate(kind, {q}, {}, ps, id++));
        }
        return c;
    }
    for (int q = 0; q + 1 < n; q++) {
        std::vector<double> ps;
        if (kindParamCount(kind) == 1) ps = {angle(q)};
        if (kind == GateKind::CX || kind == GateKind::CP) c.gates.push_back(makeGate(kind, {q + 1}, {q}, ps, id++));
        else c.gates.push_back(makeGate(kind, {q, q + 1}, {}, ps, id++));
    }
    return c;
}

Circuit genRandom(int n, int gates, std::uint64_t seed) {
    static const GateKind kPool[] = {GateKind::H,  GateKind::U,    GateKind::X,  GateKind::CX, GateKind::CP,
                                     GateKind::SWAP, GateKind::RX, GateKind::RY, GateKind::RZ, GateKind::RZZ};
    constexpr std::uint64_t kPoolSize = sizeof(kPool) / sizeof(kPool[0]);
    Circuit c;
    c.nQubits = n;
    Rng rng(seed);
    for (long id = 0; id < gates; id++) {
        GateKind kind = kPool[rng.nextBelow(kPoolSize)];
        while (n < 2 && kindArity(kind) == 2) kind = kPool[rng.nextBelow(kPoolSize)];
        std::vector<double> ps;
        for (int i = 0; i < kindParamCount(kind); i++) ps.push_back(rng.nextDouble() * (2.0 * kPi));
        if (kindArity(kind) == 1) {
            c.gates.push_back(makeGate(kind, {int(rng.nextBelow(std::uint64_t(n)))}, {}, ps, id));
            continue;
        }
        const int a = int(rng.nextBelow(std::uint64_t(n)));
        int b = int(rng.nextBelow(std::uint64_t(n - 1)));
        if (b >= a) b++;
        if (kind == GateKind::CX || kind == GateKind::CP) c.gates.push_back(makeGate(kind, {b}, {a}, ps, id));
        else c.gates.push_back(makeGate(kind, {a, b}, {}, ps, id));
    }
    return c;
}

namespace {

// Exact Toffoli from H, CX and T = U(0,0,pi/4) / T^dagger = U(0,0,-pi/4).
void toffoli(Circuit& c, long& id, int a, int b, int t) {
    auto T = [&](int q, double s) { c.gates.push_back(makeU(q, 0.0, 0.0, s * kPi / 4.0, id++)); };
    auto CX = [&](int x, int y) { c.gates.push_back(makeCX(x, y, id++)); };
    c.gates.push_back(makeH(t, id++));
    CX(b, t);
    T(t, -1);
    CX(a, t);
    T(t, +1);
    CX(b, t);
    T(t, -1);
    CX(a, t);
    T(b, +1);
    T(t, +1);
    c.gates.push_back(makeH(t, id++));
    CX(a, b);
    T(a, +1);
    T(b, -1);
    CX(a, b);
}

// Z on |1...1> of data qubits [0, m): AND-chain into ancillas [m, 2m-2),
// CZ (= CP(pi)) between the last ancilla and qubit m-1, uncompute.
void multiZ(Circuit& c, long& id, int m) {
    if (m == 1) {
        c.gates.push_back(makeU(0, 0.0, 0.0, kPi, id++));
        return;
    }
    if (m == 2) {
        c.gates.push_back(makeCP(0, 1, kPi, id++));
        return;
    }
    const int anc0 = m;
    toffoli(c, id, 0, 1, anc0);
    for (int j = 2; j < m - 1; j++) toffoli(c, id, anc0 + j - 2, j, anc0 + j - 1);
    const int last = anc0 + m - 3;
    c.gates.push_back(makeCP(last, m - 1, kPi, id++));
    for (int j = m - 2; j >= 2; j--) toffoli(c, id, anc0 + j - 2, j, anc0 + j - 1);
    toffoli(c, id, 0, 1, anc0);
}

}  // namespace

// validateOrder: each logical qubit keeps a cursor into the ids of its raw
// gates; replaying the program (SQS / CSQS move the layout, fused gates expand
// into their constituents) must advance every cursor by exactly the gate it
// meets, and finish with every cursor at its end.
OrderReport validateOrder(const Circuit& raw, const Program& p) {
    OrderReport rep;
    auto fail = [&rep](const std::string& msg, int qubit, long expected, long got) {
        if (!rep.ok) return;  // keep the first divergence
        rep = OrderReport{false, msg, qubit, expected, got};
    };
    if (raw.nQubits != p.nQubits) {
        fail("qubit count mismatch", -1, -1, -1);
        return rep;
    }
    std::vector<std::vector<long>> order(static_cast<size_t>(raw.nQubits));
    std::map<long, const Gate*> byId;
    for (const Gate& g : raw.gates) {
        byId[g.id] = &g;
        for (int q : g.qubits()) order[size_t(q)].push_back(g.id);
    }
    std::vector<size_t> cursor(static_cast<size_t>(raw.nQubits), 0);
    QubitLayout layout = QubitLayout::identity(raw.nQubits);
    auto visit = [&](const Gate& g) {
        std::vector<int> logical;
        for (int q : g.qubits()) logical.push_back(layout.physToLog[size_t(q)]);
        const int first = logical.empty() ? -1 : logical[0];
        const auto it = byId.find(g.id);
        if (it == byId.end()) {
            fail("gate id " + std::to_string(g.id) + " does not appear in the raw circuit", first, -1, g.id);
            return;
        }
        const Gate& want = *it->second;
        if (g.kind != want.kind || g.params != want.params || logical != want.qubits()) {
            fail("gate " + std::to_string(g.id) + " differs from its raw form", first, g.id, g.id);
            return;
        }
        for (int q : logical) {
            const std::vector<long>& ids = order[size_t(q)];
            size_t& c = cursor[size_t(q)];
            if (c >= ids.size()) {
                fail("qubit " + std::to_string(q) + " sees extra gate " + std::to_string(g.id), q, -1, g.id);
                return;
            }
            if (ids[c] != g.id) {
                fail("qubit " + std::to_string(q) + " expected gate " + std::to_string(ids[c]) + " but found " +
                         std::to_string(g.id),
                     q, ids[c], g.id);
                return;
            }
            c++;
        }
    };
    for (const ProgramItem& it : p.items) {
        if (!rep.ok) break;
        if (it.type == ProgramItem::Swap) {
            layout.applyPairs(it.swap.pairs);
            continue;
        }
        for (const Gate& g : it.block.gates) {
            if (!rep.ok) break;
            const bool fused = g.kind == GateKind::FusedDiag || g.kind == GateKind::FusedDense;
            if (!fused) {
                visit(g);
                continue;
            }
            if (g.constituents.empty()) {
                fail("fused gate " + std::to_string(g.id) + " carries no constituent records", -1, -1, g.id);
                break;
            }
            for (const Gate& c : g.constituents) {
                visit(c);
                if (!rep.ok) break;
            }
        }
    }
    for (int q = 0; rep.ok && q < raw.nQubits; q++)
        if (cursor[size_t(q)] != order[size_t(q)].size())
            fail("qubit " + std::to_string(q) + " is missing gate " + std::to_string(order[size_t(q)][cursor[size_t(q)]]),
                 q, order[size_t(q)][cursor[size_t(q)]], -1);
    return rep;
}

Circuit genGrover(int n, std::uint64_t marked, int iterations) {
    if (n < 2) throw ConfigError("grover needs at least 2 qubits");
    const int m = (n + 2) / 2;  // data qubits; m-2 ancillas; (n - (2m-2)) idle qubits
    marked &= (m >= 64) ? ~std::uint64_t(0) : ((std::uint64_t(1) << m) - 1);
    if (iterations <= 0) iterations = int(std::floor(kPi / 4.0 * std::sqrt(double(Index(1) << m))));
    Circuit c;
    c.nQubits = n;
    long id = 0;
    for (int q = 0; q < m; q++) c.gates.push_back(makeH(q, id++));
    for (int it = 0; it < iterations; it++) {
        // Oracle: -1 phase on |marked>.
        for (int q = 0; q < m; q++)
            if (!((marked >> q) & 1)) c.gates.push_back(makeX(q, id++));
        multiZ(c, id, m);
        for (int q = 0; q < m; q++)
            if (!((marked >> q) & 1)) c.gates.push_back(makeX(q, id++));
        // Diffusion (up to a global -1): H X (Z on |1..1>) X H.
        for (int q = 0; q < m; q++) c.gates.push_back(makeH(q, id++));
        for (int q = 0; q < m; q++) c.gates.push_back(makeX(q, id++));
        multiZ(c, id, m);
        for (int q = 0; q < m; q++) c.gates.push_back(makeX(q, id++));
        for (int q = 0; q < m; q++) c.gates.push_back(makeH(q, id++));
    }
    return c;
}

}  // namespace quokka
