// The reference-signature C++ engine API (include/quokka/engine.hpp,
// distributed.hpp) implemented on the device C-ABI (include/qk.h).
//
// Host StateVectors are staging copies: each call uploads, runs the sm_100a
// kernels, and downloads.  There is deliberately no host arithmetic path.
#include <algorithm>
#include <cstring>
#include <iterator>
#include <memory>

#include "qk.h"
#include "quokka/distributed.hpp"
#include "quokka/engine.hpp"

namespace quokka {

namespace {

void check(int rc) {
    if (rc == QK_OK) return;
    const std::string msg = qk_last_error();
    if (rc == QK_ERR_PARSE) throw ParseError(msg);
    if (rc == QK_ERR_CONFIG) throw ConfigError(msg);
    throw SimulationError(msg);
}

int log2Exact(size_t n) {
    int b = 0;
    while ((size_t(1) << b) < n) b++;
    if ((size_t(1) << b) != n) throw SimulationError("state size is not a power of two");
    return b;
}

struct Slice {
    qk_state* st = nullptr;
    Slice(int n, int R = 0, int rank = 0, int B = -1, int dev = 0) { check(qk_create(n, R, rank, B, dev, &st)); }
    ~Slice() { qk_destroy(st); }
    void up(const std::vector<Amp>& v) {
        check(qk_upload(st, 0, v.size(), reinterpret_cast<const double*>(v.data())));
    }
    void down(std::vector<Amp>& v) { check(qk_download(st, 0, v.size(), reinterpret_cast<double*>(v.data()))); }
};

qk_gate toC(const Gate& g) {
    qk_gate c{};
    c.kind = static_cast<int32_t>(g.kind);
    const std::vector<int> qs = g.qubits();
    c.nqubits = int32_t(qs.size());
    for (size_t i = 0; i < qs.size() && i < 16; i++) c.qubits[i] = qs[i];
    for (size_t i = 0; i < g.params.size() && i < 3; i++) c.params[i] = g.params[i];
    c.payload = g.payload.empty() ? nullptr : reinterpret_cast<const double*>(g.payload.data());
    c.id = g.id;
    return c;
}

qk_config toC(const Config& q) {
    qk_config c;
    c.total_qubits = q.totalQubits;
    c.rank_qubits = q.rankQubits;
    c.buffer_qubits = q.bufferQubits;
    c.chunk_qubits = q.chunkQubits;
    c.fusion_qubits = q.fusionQubits;
    c.cache_line_qubits = q.cacheLineQubits;
    c.ims = q.imsEnabled;
    c.xrs = q.xrsEnabled;
    c.fusion = q.fusionEnabled;
    c.diagonal_fusion = q.diagonalFusionEnabled;
    return c;
}

struct ProgramHandle {
    qk_program* p = nullptr;
    ProgramHandle(const Program& prog, const Config& cfg) {
        const qk_config c = toC(cfg);
        check(qk_program_parse(serializeProgram(prog).c_str(), &c, 1, &p));
    }
    ~ProgramHandle() { qk_program_destroy(p); }
};

}  // namespace

double StateVector::norm() const {
    if (amps.empty()) return 0.0;
    Slice s(log2Exact(amps.size()));
    s.up(amps);
    double v = 0;
    check(qk_norm(s.st, &v));
    return v;
}

StateVector initState(int nQubits, Index initial) {
    if (nQubits < 1 || nQubits > 40) throw SimulationError("qubit count " + std::to_string(nQubits) + " out of range");
    if (initial >= (Index(1) << nQubits)) throw SimulationError("initial basis state out of range");
    StateVector sv;
    sv.nQubits = nQubits;
    sv.amps.assign(size_t(1) << nQubits, Amp(0.0, 0.0));
    sv.amps[initial] = Amp(1.0, 0.0);
    return sv;
}

Index bitswap(Index x, const std::vector<std::pair<int, int>>& pairs) {
    for (const auto& [a, b] : pairs)
        if (((x >> a) ^ (x >> b)) & 1) x ^= (Index(1) << a) | (Index(1) << b);
    return x;
}

// The reference's cache-line traversal order (engine.cpp:40-60): in-positions
// of pairs straddling CL are routed to the lowest slots >= CL.  The device IMS
// kernel does not need it (it is a visiting order, not a result); kept for
// API parity.
Index bitshift(Index t, const std::vector<std::pair<int, int>>& pairs, int cl) {
    std::vector<int> crossing;
    for (const auto& [a, b] : pairs)
        if (std::min(a, b) < cl && std::max(a, b) >= cl) crossing.push_back(std::max(a, b));
    std::sort(crossing.begin(), crossing.end());
    std::vector<int> slots, onlySlots, onlyCrossing;
    for (size_t j = 0; j < crossing.size(); j++) slots.push_back(cl + int(j));
    std::set_difference(slots.begin(), slots.end(), crossing.begin(), crossing.end(), std::back_inserter(onlySlots));
    std::set_difference(crossing.begin(), crossing.end(), slots.begin(), slots.end(), std::back_inserter(onlyCrossing));
    std::vector<std::pair<int, int>> route;
    for (size_t j = 0; j < onlySlots.size(); j++) route.emplace_back(onlySlots[j], onlyCrossing[j]);
    return bitswap(t, route);
}

void imsSwap(StateVector& sv, const SwapOp& op, int cacheLineQubits, int /*threads*/) {
    if (op.pairs.empty()) return;
    Slice s(log2Exact(sv.amps.size()));
    s.up(sv.amps);
    std::vector<int> outs, ins;
    for (const auto& [a, b] : op.pairs) {
        outs.push_back(a);
        ins.push_back(b);
    }
    check(qk_ims_swap(s.st, outs.data(), ins.data(), int(outs.size()), cacheLineQubits));
    s.down(sv.amps);
}

void applyGate(StateVector& sv, const Gate& g) {
    Slice s(log2Exact(sv.amps.size()));
    s.up(sv.amps);
    const qk_gate c = toC(g);
    check(qk_apply_gate(s.st, &c));
    s.down(sv.amps);
}

void applyBlock(StateVector& sv, const GateBlock& block, int chunkQubits, int /*threads*/) {
    for (const Gate& g : block.gates)
        for (int q : g.qubits())
            if (q >= chunkQubits)
                throw SimulationError("block gate " + std::to_string(g.id) + " reaches outside the chunk");
    Slice s(log2Exact(sv.amps.size()));
    s.up(sv.amps);
    std::vector<qk_gate> cs;
    for (const Gate& g : block.gates) cs.push_back(toC(g));
    check(qk_apply_block(s.st, cs.data(), int(cs.size()), chunkQubits));
    s.down(sv.amps);
}

SimResult simulateProgram(const Program& p, const Config& cfg, Index initial, int /*threads*/) {
    if (initial >= (Index(1) << p.nQubits)) throw SimulationError("initial basis state out of range");
    if (p.swapCount(SwapOp::CrossRank) > 0)  // engine.cpp:291-293, whatever the config's rank split
        throw SimulationError("cross-rank swap in a single-rank run; use the multi-rank engine");
    ProgramHandle h(p, cfg);
    Slice s(p.nQubits);
    const qk_config c = toC(cfg);
    check(qk_simulate(s.st, h.p, &c, initial, nullptr));
    SimResult r;
    r.state.nQubits = p.nQubits;
    r.state.amps.resize(size_t(1) << p.nQubits);
    s.down(r.state.amps);
    r.layout = p.finalLayout;
    return r;
}

StateVector simulateGateByGate(const Circuit& c, Index initial, int /*threads*/) {
    Slice s(c.nQubits);
    check(qk_set_basis(s.st, initial));
    for (const Gate& g : c.gates) {
        const qk_gate cg = toC(g);
        check(qk_apply_gate(s.st, &cg));
    }
    StateVector sv;
    sv.nQubits = c.nQubits;
    sv.amps.resize(size_t(1) << c.nQubits);
    s.down(sv.amps);
    return sv;
}

int resolveThreads(int requested) { return requested > 0 ? requested : 1; }

// ---- DeviceState ----------------------------------------------------------------

DeviceState::DeviceState(int nQubits, int rankQubits, int rank, int device, int bufferQubits) {
    check(qk_create(nQubits, rankQubits, rank, bufferQubits, device, &st_));
}
DeviceState::~DeviceState() { qk_destroy(st_); }
void DeviceState::setBasis(Index initial) { check(qk_set_basis(st_, initial)); }
double DeviceState::norm() const {
    double v = 0;
    check(qk_norm(st_, &v));
    return v;
}
void DeviceState::download(Index off, Index cnt, Amp* host) const {
    check(qk_download(st_, off, cnt, reinterpret_cast<double*>(host)));
}
void DeviceState::upload(Index off, Index cnt, const Amp* host) {
    check(qk_upload(st_, off, cnt, reinterpret_cast<const double*>(host)));
}
void DeviceState::synchronize() const { check(qk_synchronize(st_)); }

void simulateProgramDevice(DeviceState& st, const Program& p, const Config& cfg, Index initial) {
    ProgramHandle h(p, cfg);
    const qk_config c = toC(cfg);
    check(qk_simulate(st.handle(), h.p, &c, initial, nullptr));
}

// ---- multi-rank (distributed.hpp) -------------------------------------------------

Index rankSliceBase(int rank, const Config& cfg) { return Index(rank) << cfg.rankRegion(); }

StateVector gatherState(const std::vector<std::vector<Amp>>& slices, int nQubits) {
    StateVector sv;
    sv.nQubits = nQubits;
    for (const auto& s : slices) sv.amps.insert(sv.amps.end(), s.begin(), s.end());
    if (sv.amps.size() != (size_t(1) << nQubits)) throw SimulationError("gathered slices do not form a full state vector");
    return sv;
}

namespace {

// Rank r's slice lives on device r mod (visible devices): one GPU per rank
// when there are enough (the runtime enables peer access between them for
// the in-place slab swap), else several slices share a device.
struct SliceSet {
    std::vector<std::unique_ptr<Slice>> owned;
    std::vector<qk_state*> raw;
    SliceSet(const Config& cfg) {
        int ndev = 1;
        check(qk_device_count(&ndev));
        const int ranks = 1 << cfg.rankQubits;
        for (int r = 0; r < ranks; r++) {
            owned.push_back(std::make_unique<Slice>(cfg.totalQubits, cfg.rankQubits, r, cfg.bufferQubits,
                                                    ndev > 0 ? r % ndev : 0));
            raw.push_back(owned.back()->st);
        }
    }
};

// The reference's RankStats for one cross-rank swap, added to `out` the way
// xrsFill / xrsDeliver accumulate them (distributed.cpp:87-93, 116-119): per
// window round, bytes sent (= received) and one perRound entry.  The round
// structure is the runtime's own message plan (qk_xrs_plan).
void accountSwap(const SwapOp& op, const Config& cfg, std::vector<RankStats>& out) {
    const int ranks = 1 << cfg.rankQubits;
    if (int(out.size()) != ranks) out.resize(size_t(ranks));
    std::vector<int> outs, ins;
    for (const auto& [a, b] : op.pairs) {
        outs.push_back(a);
        ins.push_back(b);
    }
    const int s = int(outs.size());
    const Index slabOffsets = Index(1) << (cfg.rankRegion() - s);
    const Index window = std::min(slabOffsets, Index(1) << (cfg.bufferQubits - s));
    const Index rounds = (slabOffsets + window - 1) / window;
    const int slabsOut = (1 << s) - 1;
    std::vector<qk_xrs_msg> msgs(size_t(slabsOut) * size_t(rounds) + 1);
    for (int r = 0; r < ranks; r++) {
        int nm = 0;
        check(qk_xrs_plan(cfg.totalQubits, cfg.rankQubits, cfg.bufferQubits, r, outs.data(), ins.data(), s,
                          msgs.data(), int(msgs.size()), &nm));
        RankStats& st = out[size_t(r)];
        std::vector<std::size_t> perRound(size_t(rounds), 0);
        for (int m = 0; m < nm; m++) perRound[size_t(msgs[size_t(m)].round)] += msgs[size_t(m)].count * sizeof(Amp);
        for (std::size_t bytes : perRound) {
            st.bytesSent += bytes;
            st.bytesReceived += bytes;
            st.peakBufferBytes = std::max<std::size_t>(st.peakBufferBytes, std::size_t(slabsOut) * window * sizeof(Amp));
            st.rounds++;
            st.perRound.emplace_back(bytes, bytes);
        }
    }
}

}  // namespace

MultiRankResult spawnRanks(const Program& p, const Config& cfg, Index initial) {
    if (p.nQubits != cfg.totalQubits || p.rankQubits != cfg.rankQubits)
        throw ConfigError("program and config disagree on the qubit split");
    ProgramHandle h(p, cfg);
    SliceSet set(cfg);
    const qk_config c = toC(cfg);
    std::vector<qk_xrs_stats> cs(set.raw.size());
    check(qk_simulate_local(set.raw.data(), int(set.raw.size()), h.p, &c, initial, cs.data()));
    MultiRankResult r;
    std::vector<std::vector<Amp>> slices(set.raw.size());
    for (size_t k = 0; k < slices.size(); k++) {
        slices[k].resize(size_t(1) << cfg.rankRegion());
        set.owned[k]->down(slices[k]);
    }
    r.state = gatherState(slices, p.nQubits);
    r.layout = p.finalLayout;
    r.stats.assign(set.raw.size(), RankStats{});
    for (const ProgramItem& it : p.items)
        if (it.type == ProgramItem::Swap && it.swap.kind == SwapOp::CrossRank) accountSwap(it.swap, cfg, r.stats);
    return r;
}

void xrsSwap(std::vector<std::vector<Amp>>& slices, const SwapOp& op, const Config& cfg,
             std::vector<RankStats>* stats) {
    if (op.kind != SwapOp::CrossRank) throw SimulationError("xrsSwap needs a cross-rank swap op");
    if (int(slices.size()) != (1 << cfg.rankQubits)) throw SimulationError("slice count does not match the rank count");
    SliceSet set(cfg);
    for (size_t k = 0; k < slices.size(); k++) set.owned[k]->up(slices[k]);
    std::vector<int> outs, ins;
    for (const auto& [a, b] : op.pairs) {
        outs.push_back(a);
        ins.push_back(b);
    }
    std::vector<qk_xrs_stats> cs(slices.size());
    check(qk_xrs_swap_local(set.raw.data(), int(set.raw.size()), outs.data(), ins.data(), int(outs.size()), cs.data()));
    for (size_t k = 0; k < slices.size(); k++) set.owned[k]->down(slices[k]);
    if (stats) accountSwap(op, cfg, *stats);
}

}  // namespace quokka
