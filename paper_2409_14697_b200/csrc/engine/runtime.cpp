// Runtime + C-ABI (include/qk.h): device-resident rank slices, program
// compilation cache, the item dispatcher, XRS over NCCL or peer memory.
//
// Replaces the reference's L5/L6 drivers: simulateProgram
// (proj/src/engine.cpp:283-297), spawnRanks / xrsSwap / planXrs
// (proj/src/distributed.cpp:25-206).  There is no CPU fallback: every
// amplitude update is a kernel from block_pass.cu / perm.cu; without a CUDA
// device the calls fail with QK_ERR_SIM.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "qk.h"
#include "quokka/circuit.hpp"
#include "quokka/optimizer.hpp"
#include "quokka/tools.hpp"
#include "ipc.h"
#include "jit.h"
#include "schedule.h"

namespace qkdev {
cudaError_t launchBlockPass(double2*, const double2*, const PassParams&, int, uint64_t, cudaStream_t);
cudaError_t launchDenseGroup(double2*, const double2*, int, const int*, uint64_t, int, cudaStream_t);
cudaError_t launchDenseTile(double2*, const double2*, const int*, int, int, int, int, cudaStream_t, uint64_t,
                            uint64_t);
cudaError_t launchIms(double2*, int, const int*, const int*, int, cudaStream_t);
void setImsMode(int);
cudaError_t launchSlabSwap(int, double2* const*, double2* const*, const uint64_t*, const uint64_t*, const int*, int,
                           cudaStream_t);
cudaError_t launchWindowPack(double2*, const double2*, uint64_t, uint64_t, const int*, int, cudaStream_t);
cudaError_t launchWindowUnpack(double2*, const double2*, uint64_t, uint64_t, const int*, int, cudaStream_t);
cudaError_t launchDiagTable(double2*, const double2*, uint64_t, const int*, int, cudaStream_t);
cudaError_t launchNorm(const double2*, uint64_t, double*, double*, cudaStream_t);
cudaError_t launchSumTiles(const double*, uint64_t, double*, double*, cudaStream_t);
size_t normScratchDoubles();
cudaError_t launchSetBasis(double2*, uint64_t, cudaStream_t, double);
cudaError_t launchZeroOutside(double2*, uint64_t, uint64_t, uint64_t, int, cudaStream_t);
cudaError_t launchMarginal(const double2*, uint64_t, const int*, int, double*, double*, cudaStream_t);
size_t marginalScratchDoubles(int k);
}  // namespace qkdev

using quokka::ConfigError;
using quokka::Index;
using quokka::ParseError;
using quokka::SimulationError;

namespace {

thread_local std::string g_lastError;

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw SimulationError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
void nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw SimulationError(std::string("NCCL error in ") + what + ": " + ncclGetErrorString(r));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return QK_OK;
    } catch (const ParseError& e) {
        g_lastError = e.what();
        return QK_ERR_PARSE;
    } catch (const ConfigError& e) {
        g_lastError = e.what();
        return QK_ERR_CONFIG;
    } catch (const SimulationError& e) {
        g_lastError = e.what();
        return QK_ERR_SIM;
    } catch (const std::exception& e) {
        g_lastError = e.what();
        return QK_ERR_SIM;
    }
}

char* dupText(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size() + 1);
    return p;
}

quokka::Config toConfig(const qk_config& c) {
    quokka::Config q;
    q.totalQubits = c.total_qubits;
    q.rankQubits = c.rank_qubits;
    q.bufferQubits = c.buffer_qubits;
    q.chunkQubits = c.chunk_qubits;
    q.fusionQubits = c.fusion_qubits;
    q.cacheLineQubits = c.cache_line_qubits;
    q.imsEnabled = c.ims != 0;
    q.xrsEnabled = c.xrs != 0;
    q.fusionEnabled = c.fusion != 0;
    q.diagonalFusionEnabled = c.diagonal_fusion != 0;
    return q;
}

qk_config fromConfig(const quokka::Config& q) {
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

// ---- XRS plan (distributed.cpp:25-71 semantics) ------------------------------

struct XrsPlan {
    std::vector<int> outs, insRel;  // ascending outs, rank-bit indices
    int s = 0;
    Index slabOffsets = 0, window = 0, rounds = 0;
};

XrsPlan planXrs(const quokka::SwapOp& op, int n, int R, int B) {
    if (op.kind != quokka::SwapOp::CrossRank) throw SimulationError("xrsSwap needs a cross-rank swap op");
    const int region = n - R;
    XrsPlan p;
    for (const auto& [o, i] : op.pairs) {
        if (o < 0 || o >= region || i < region || i >= n)
            throw SimulationError("cross-rank swap positions out of range");
        p.outs.push_back(o);
        p.insRel.push_back(i - region);
    }
    p.s = int(op.pairs.size());
    if (B < p.s) throw SimulationError("exchange buffer smaller than one amplitude per slab");
    p.slabOffsets = Index(1) << (region - p.s);
    p.window = std::min(p.slabOffsets, Index(1) << (B - p.s));
    p.rounds = (p.slabOffsets + p.window - 1) / p.window;
    return p;
}

int ownSlab(int rank, const XrsPlan& p) {
    int v = 0;
    for (int j = 0; j < p.s; j++) v |= ((rank >> p.insRel[size_t(j)]) & 1) << j;
    return v;
}

int partnerOf(int rank, int slab, const XrsPlan& p) {
    for (int j = 0; j < p.s; j++) {
        rank &= ~(1 << p.insRel[size_t(j)]);
        rank |= ((slab >> j) & 1) << p.insRel[size_t(j)];
    }
    return rank;
}

Index slabBits(int slab, const XrsPlan& p) {
    Index b = 0;
    for (int j = 0; j < p.s; j++) b |= Index((slab >> j) & 1) << p.outs[size_t(j)];
    return b;
}

// This rank's message schedule for one CSQS: per window round, for every slab
// pa != own, send slab pa's window to the rank whose swapped bits equal pa and
// receive that rank's slab `own` window into receive-buffer section `sec`,
// which is copied back into slab pa (distributed.cpp:76-120).  The NCCL path
// executes exactly this list; tests/test_xrs_plan.py executes it over gloo.
std::vector<qk_xrs_msg> xrsMessages(const XrsPlan& p, int rank) {
    std::vector<qk_xrs_msg> out;
    if (p.s == 0) return out;
    const int own = ownSlab(rank, p), slabs = 1 << p.s;
    int round = 0;
    for (Index w0 = 0; w0 < p.slabOffsets; w0 += p.window, round++) {
        const Index cnt = std::min(p.window, p.slabOffsets - w0);
        for (int pa = 0, sec = 0; pa < slabs; pa++) {
            if (pa == own) continue;
            out.push_back(qk_xrs_msg{round, partnerOf(rank, pa, p), pa, sec++, w0, cnt});
        }
    }
    return out;
}

// The reference's RankStats accounting for one CSQS (distributed.cpp:87-93, 116-119).
void accountXrs(const XrsPlan& p, qk_xrs_stats* st) {
    if (!st) return;
    const Index other = (Index(1) << p.s) - 1;
    st->bytes_sent += other * p.slabOffsets * 16;
    st->bytes_received += other * p.slabOffsets * 16;
    st->peak_buffer_bytes = std::max<uint64_t>(st->peak_buffer_bytes, other * p.window * 16);
    st->rounds += p.rounds;
}

// ---- compiled programs ----------------------------------------------------------

struct CompiledItem {
    enum Kind { Block, Ims, Xrs } kind = Block;
    std::vector<qkeng::Step> steps;  // Block
    std::vector<int> outs, ins;      // Ims / Xrs
    double flopsPerAmp = 0;
    uint64_t denseTargetsOff = 0;    // int offset into the device target table
};

// Tile-size autotune (qkdev::tileTune): items [first, last) of `items` (a
// gate stream scheduled with 2^13 tiles plus its materialization) have an
// alternative `b` (the same stream with 2^12 tiles).  Run 1 times A, run 2
// times B; once A's per-pass register-width tuning has settled, the faster
// schedule is kept.
struct ChoiceTune {
    int runs = 0;
    float msA = -1, msB = -1;  // group device time: A's first run, B's fastest run
    float msA2 = -1;           // A's fastest run once its passes' register widths are tuned
    int runsB = 0, runsA2 = 0; // B and tuned A are timed twice each (a first run can be slow)
    int choice = -1;
};

struct Alternative {
    size_t first = 0, last = 0;
    std::vector<CompiledItem> b;
    std::shared_ptr<ChoiceTune> tune = std::make_shared<ChoiceTune>();
};

struct Compiled {
    int nLocal = 0;
    // Initial memory layout (program position p of the slice at memory bit
    // mem0[p]); identity unless compiled for a run from a basis state.
    std::vector<int> mem0;
    std::vector<CompiledItem> items;
    std::vector<Alternative> alts;  // sorted by first
    std::vector<double> gtab;     // host copy of device tables
    std::vector<int> targets;     // dense-group target lists
    double basisAmp = 1.0;        // |initial> amplitude the run starts from (deferred H normalization)
};

struct DeviceTables {
    double2* gtab = nullptr;
    int* targets = nullptr;
};

}  // namespace

struct qk_program {
    quokka::Program prog;
    std::mutex mu;
    std::map<int, std::shared_ptr<Compiled>> compiled;            // by nLocal
    // (schedule, device): each compiled schedule (slice size x layout x kernel
    // family) has its own gtab / target tables
    std::map<std::pair<const Compiled*, int>, DeviceTables> tables;
    ~qk_program() {
        for (auto& kv : tables) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(kv.first.second);
            cudaFree(kv.second.gtab);
            cudaFree(kv.second.targets);
            cudaSetDevice(prev);
        }
    }
};

struct qk_state {
    int n = 0, R = 0, rank = 0, B = 0, device = 0, nLocal = 0;
    uint64_t count = 0;
    double2* amps = nullptr;
    cudaStream_t stream = nullptr;
    double* normScratch = nullptr;
    double* normOut = nullptr;
    double2* recvBuf = nullptr;   // two halves of bufAmps / 2: round k receives into half k % 2
    double2* packBuf = nullptr;
    uint64_t bufAmps = 0;
    cudaStream_t aux = nullptr;   // NCCL XRS: copy-back of round k overlaps the transfer of round k + 1
    cudaEvent_t xrsDone[2] = {nullptr, nullptr}, unpackDone[2] = {nullptr, nullptr};
    ncclComm_t comm = nullptr;
    qkipc::Group* ipc = nullptr;  // peer-memory rank group (qk_ipc_init)
    bool profiling = false;
    qk_run_stats last{};
    // Fused norm: the program's last pass wrote per-warp partial sums of
    // |a|^2 and normOut holds their fold; valid until the state changes again.
    double* normTiles = nullptr;
    uint64_t normTilesCap = 0;
    bool normValid = false;
};

namespace {

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

bool lazyIms() {
    static const bool on = [] {
        const char* v = std::getenv("QK_LAZY_IMS");
        return !(v && v[0] == '0');
    }();
    return on;
}

// IMS pair sets that move the data at memory bit mem[p] to bit p for every p:
// each cycle of the bit permutation is a product of two reflections
// (c_i -> c_{-i}, then c_i -> c_{1-i}), so at most two IMS passes.
std::vector<std::vector<std::pair<int, int>>> materializePairs(const std::vector<int>& mem) {
    const int n = int(mem.size());
    std::vector<int> dest(static_cast<size_t>(n));  // data at bit b must go to bit dest[b]
    for (int p = 0; p < n; p++) dest[size_t(mem[size_t(p)])] = p;
    std::vector<std::pair<int, int>> t1, t2;
    std::vector<char> seen(static_cast<size_t>(n), 0);
    for (int s = 0; s < n; s++) {
        if (seen[size_t(s)] || dest[size_t(s)] == s) continue;
        std::vector<int> cyc;  // cyc[i+1] = dest[cyc[i]]
        for (int b = s; !seen[size_t(b)]; b = dest[size_t(b)]) {
            seen[size_t(b)] = 1;
            cyc.push_back(b);
        }
        const int k = int(cyc.size());
        for (int i = 1; i < k - i; i++) t1.emplace_back(cyc[size_t(i)], cyc[size_t(k - i)]);
        for (int i = 0; i < k; i++) {
            const int j = ((1 - i) % k + k) % k;
            if (i < j) t2.emplace_back(cyc[size_t(i)], cyc[size_t(j)]);
        }
    }
    std::vector<std::vector<std::pair<int, int>>> out;
    for (auto* t : {&t1, &t2}) {
        if (t->empty()) continue;
        for (auto& pr : *t)
            if (pr.first > pr.second) std::swap(pr.first, pr.second);
        std::sort(t->begin(), t->end());
        out.push_back(*t);
    }
    return out;
}

bool useJit(int nLocal);

// QK_PARTIAL_MATERIALIZE (default 1): before a CSQS only its staged positions
// are put in place (the rest of the lazy relabeling carries on).
bool partialMaterialize() {
    static const bool v = [] {
        const char* e = std::getenv("QK_PARTIAL_MATERIALIZE");
        return !e || std::atoi(e) != 0;
    }();
    return v;
}

// QK_DEFER_H (default 1): see compileLayout.
bool deferHScales() {
    static const bool v = [] {
        const char* e = std::getenv("QK_DEFER_H");
        return !e || std::atoi(e) != 0;
    }();
    return v;
}

// QK_BASIS_LAYOUT (default 1): see compileFor(fromBasis).
bool basisLayout() {
    static const bool v = [] {
        const char* e = std::getenv("QK_BASIS_LAYOUT");
        return !e || std::atoi(e) != 0;
    }();
    return v;
}

// Process-wide schedule cache (a plan cache): programs with identical items
// on the same slice size share one compiled schedule, its device-independent
// tables and its autotune state, so re-parsing a program text does not
// re-schedule or re-tune it.  Keyed by the items' binary content.
std::string scheduleKey(const quokka::Program& prog, int nLocal) {
    std::string k;
    auto put = [&](const void* d, size_t n) { k.append(static_cast<const char*>(d), n); };
    auto putInts = [&](const std::vector<int>& v) {
        const uint32_t n = uint32_t(v.size());
        put(&n, sizeof n);
        put(v.data(), v.size() * sizeof(int));
    };
    put(&nLocal, sizeof nLocal);
    for (const quokka::ProgramItem& it : prog.items) {
        const int t = int(it.type);
        put(&t, sizeof t);
        if (it.type == quokka::ProgramItem::Block) {
            const uint32_t n = uint32_t(it.block.gates.size());
            put(&n, sizeof n);
            for (const quokka::Gate& g : it.block.gates) {
                const int kind = int(g.kind);
                put(&kind, sizeof kind);
                putInts(g.targets);
                putInts(g.controls);
                const uint32_t np = uint32_t(g.params.size()), na = uint32_t(g.payload.size());
                put(&np, sizeof np);
                put(g.params.data(), g.params.size() * sizeof(double));
                put(&na, sizeof na);
                put(g.payload.data(), g.payload.size() * sizeof(quokka::Amp));
            }
        } else {
            const int kind = int(it.swap.kind);
            put(&kind, sizeof kind);
            for (const auto& [a, b] : it.swap.pairs) {
                put(&a, sizeof a);
                put(&b, sizeof b);
            }
            const int end = -1;
            put(&end, sizeof end);
        }
    }
    return k;
}

struct ScheduleCache {
    std::mutex mu;
    std::map<std::string, std::shared_ptr<Compiled>> byKey;
    std::vector<std::string> order;  // insertion order (evict the oldest)
    static constexpr size_t kMax = 32;
};
ScheduleCache& scheduleCache() {
    static ScheduleCache c;
    return c;
}

// Estimated cost of a compiled program in slice sweeps: every step of a
// block and every IMS / XRS item reads and writes the slice once; a block
// step runs at ~1.5x the time of an IMS (B200: ~73 vs ~44 ms at 2^33), so
// steps weigh 3 and permutations 2.
uint64_t swapBitsOf(uint64_t x, const std::vector<int>& outs, const std::vector<int>& ins) {
    for (size_t j = 0; j < outs.size(); j++) {
        const uint64_t d = ((x >> outs[j]) ^ (x >> ins[j])) & 1u;
        x ^= (d << outs[j]) | (d << ins[j]);
    }
    return x;
}

// In a run from a basis state a pass whose input still has known zeros reads
// almost nothing and its output stays partial or is the one filling write:
// it weighs 1 (support tracked as the runtime does, schedule.h supportAfter).
size_t sweeps(const Compiled& c, bool fromBasis = false) {
    size_t n = 0;
    uint64_t mask = fromBasis ? (c.nLocal >= 64 ? ~uint64_t(0) : (uint64_t(1) << c.nLocal) - 1) : 0, val = 0;
    for (const CompiledItem& it : c.items) {
        if (it.kind != CompiledItem::Block) {
            n += 2;
            if (it.kind == CompiledItem::Xrs) mask = 0;
            else mask = swapBitsOf(mask, it.outs, it.ins);
            continue;
        }
        for (const qkeng::Step& s : it.steps) {
            if (s.kind != qkeng::Step::Pass) {
                n += 3;
                for (size_t j = 1; j < s.targets.size(); j++) mask &= ~(uint64_t(1) << s.targets[j]);
                continue;
            }
            n += mask ? 1 : 3;
            qkeng::supportAfter(s, s.pass->tile_mask, mask, val);
        }
    }
    return n;
}

// One compilation of p's items for a slice of 2^nLocal amplitudes, starting
// from memory layout mem0 (program position p at memory bit mem0[p]).
std::shared_ptr<Compiled> compileLayout(qk_program* p, int nLocal, const std::vector<int>& mem0, bool synthFirst,
                                        bool interp) {
    auto c = std::make_shared<Compiled>();
    c->nLocal = nLocal;
    // Runs from a basis state on the specialized kernels: Hadamard butterflies
    // skip their 1/sqrt2 and the initial amplitude carries the product (one
    // fewer multiply per amplitude in passes that would scale on their own,
    // e.g. QFT's last pass).  Not beyond 1000 H (the start value would leave
    // the double range).
    int deferH = 0;
    std::unique_ptr<qkeng::DeferHScales> deferScope;
    if (synthFirst && !interp && nLocal >= 4 && deferHScales()) {
        long nh = 0;
        for (const quokka::ProgramItem& item : p->prog.items)
            if (item.type == quokka::ProgramItem::Block)
                for (const quokka::Gate& g : item.block.gates) nh += g.kind == quokka::GateKind::H;
        if (nh <= 1000) deferScope = std::make_unique<qkeng::DeferHScales>(&deferH);
    }
    // Lazy in-memory swaps: an SQS (and a SWAP gate) only relabels which
    // memory bit holds which program position (mem[p]); later gates address
    // their qubits through `mem`, so it costs no HBM pass.  Gates between
    // materializations form one stream, which the scheduler cuts into passes
    // (qkeng::compileBlock: diagonal gates ride along with any pass).  The
    // relabeling is materialized (<= 2 IMS passes) only before a cross-rank
    // swap and at the end, so the final state is in the program's physical
    // order.
    std::vector<int> mem = mem0;
    const bool lazy = lazyIms();
    c->mem0 = mem;
    std::vector<quokka::Gate> stream;
    // keep == nullptr: materialize the whole layout (mem = identity: the end of
    // the program).  Before a CSQS only its staged positions (`keep`, the
    // outs) must sit at their own memory bits; the rest of the relabeling
    // stays lazy (the XRS moves memory bits outs <-> rank bits and leaves mem
    // valid), which takes at most as many IMS sweeps and often none.
    auto flushStream = [&](bool beforeMaterialize, int tileBits = 0, const std::vector<int>* keep = nullptr) {
        if (stream.empty()) return;
        CompiledItem ci;
        ci.kind = CompiledItem::Block;
        if (lazy && beforeMaterialize) {
            // route the data toward the program's physical order (mem = identity),
            // or only the kept positions (the rest stays where it is)
            std::vector<int> dest(static_cast<size_t>(nLocal)), moved;
            if (keep) {
                for (int b = 0; b < nLocal; b++) dest[size_t(b)] = b;
                std::vector<char> claimed(static_cast<size_t>(nLocal), 0);
                for (int o : *keep) claimed[size_t(o)] = 1;
                for (int o : *keep) dest[size_t(mem[size_t(o)])] = o;
                // a bit displaced from a kept target goes to the source the target's data leaves
                for (int o : *keep)
                    if (!claimed[size_t(mem[size_t(o)])] && mem[size_t(o)] != o) dest[size_t(o)] = mem[size_t(o)];
            } else {
                for (int q = 0; q < nLocal; q++) dest[size_t(mem[size_t(q)])] = q;
            }
            ci.steps = qkeng::compileBlock(stream, nLocal, c->gtab, &dest, &moved, tileBits, synthFirst && c->items.empty(),
                                           interp);
            for (int q = 0; q < nLocal; q++) mem[size_t(q)] = moved[size_t(mem[size_t(q)])];
        } else {
            ci.steps = qkeng::compileBlock(stream, nLocal, c->gtab, nullptr, nullptr, tileBits,
                                           synthFirst && c->items.empty(), interp);
        }
        for (qkeng::Step& s : ci.steps) {
            ci.flopsPerAmp += s.flopsPerAmp;
            if (s.kind != qkeng::Step::Pass) {
                const uint64_t off = c->targets.size();
                c->targets.insert(c->targets.end(), s.targets.begin(), s.targets.end());
                s.targets.insert(s.targets.begin(), int(off));  // [0] = device offset
            }
        }
        c->items.push_back(std::move(ci));
    };
    auto materialize = [&](const std::vector<int>* keep = nullptr) {
        // tau: memory bit b's data goes to tau[b]; full: mem -> identity;
        // partial: transpositions (mem[o], o) for the kept positions only
        std::vector<int> tau(static_cast<size_t>(nLocal));
        if (!keep) {
            for (int q = 0; q < nLocal; q++) tau[size_t(mem[size_t(q)])] = q;
        } else {
            for (int b = 0; b < nLocal; b++) tau[size_t(b)] = b;
            std::vector<int> cur = mem;  // cur[p] = memory bit of position p after the moves so far
            std::vector<int> at(static_cast<size_t>(nLocal));  // at[b] = position held by memory bit b
            for (int q = 0; q < nLocal; q++) at[size_t(cur[size_t(q)])] = q;
            for (int o : *keep) {
                const int x = cur[size_t(o)];
                if (x == o) continue;
                const int p2 = at[size_t(o)];  // the position now at memory bit o moves to x
                for (int b = 0; b < nLocal; b++) {  // compose: data headed for x goes to o and vice versa
                    if (tau[size_t(b)] == x) tau[size_t(b)] = o;
                    else if (tau[size_t(b)] == o) tau[size_t(b)] = x;
                }
                std::swap(cur[size_t(o)], cur[size_t(p2)]);
                at[size_t(o)] = o;
                at[size_t(x)] = p2;
            }
        }
        std::vector<int> inv(static_cast<size_t>(nLocal));  // materializePairs moves memory bit inv[q] -> q
        for (int b = 0; b < nLocal; b++) inv[size_t(tau[size_t(b)])] = b;
        for (const auto& pairs : materializePairs(inv)) {
            CompiledItem ci;
            ci.kind = CompiledItem::Ims;
            for (const auto& [o, i] : pairs) {
                ci.outs.push_back(o);
                ci.ins.push_back(i);
            }
            c->items.push_back(std::move(ci));
        }
        for (int q = 0; q < nLocal; q++) mem[size_t(q)] = tau[size_t(mem[size_t(q)])];
    };
    // A stream, routed and materialized (mem ends as the identity, or with the
    // kept positions in place); with tile autotune also the 2^12-tile
    // alternative of the same range.
    auto flushAndMaterialize = [&](const std::vector<int>* keep = nullptr) {
        const size_t first = c->items.size();
        const std::vector<int> mem0 = mem;
        flushStream(true, 0, keep);
        materialize(keep);
        const std::vector<int> memA = mem;
        const int deferA = deferH;  // the alternative applies the same H gates
        if (lazy && !stream.empty() && qkdev::tileTune() && !interp && nLocal > 13) {
            const size_t last = c->items.size();
            std::vector<CompiledItem> a(std::make_move_iterator(c->items.begin() + long(first)),
                                        std::make_move_iterator(c->items.end()));
            c->items.resize(first);
            mem = mem0;
            try {
                flushStream(true, 12, keep);
                materialize(keep);
                if (mem != memA) throw SimulationError("alternative ends in another layout");
                Alternative alt;
                alt.first = first;
                alt.last = last;
                alt.b.assign(std::make_move_iterator(c->items.begin() + long(first)),
                             std::make_move_iterator(c->items.end()));
                const auto firstIsPass = [](const std::vector<CompiledItem>& v) {
                    return !v.empty() && v[0].kind == CompiledItem::Block && !v[0].steps.empty() &&
                           v[0].steps[0].kind == qkeng::Step::Pass;
                };
                if (firstIsPass(alt.b) == firstIsPass(a)) c->alts.push_back(std::move(alt));
            } catch (const SimulationError&) {
            }
            c->items.resize(first);
            for (auto& x : a) c->items.push_back(std::move(x));
            mem = memA;
            deferH = deferA;
        }
        stream.clear();
    };
    const auto& items = p->prog.items;
    for (size_t idx = 0; idx < items.size(); idx++) {
        const quokka::ProgramItem& item = items[idx];
        if (item.type == quokka::ProgramItem::Block) {
            for (const quokka::Gate& g : item.block.gates) {
                if (lazy && g.kind == quokka::GateKind::SWAP) {  // relabel: no data moves
                    std::swap(mem[size_t(g.targets[0])], mem[size_t(g.targets[1])]);
                    continue;
                }
                quokka::Gate m = g;
                m.constituents.clear();
                for (int& q : m.targets) q = mem[size_t(q)];
                for (int& q : m.controls) q = mem[size_t(q)];
                stream.push_back(std::move(m));
            }
            continue;
        }
        if (item.swap.kind == quokka::SwapOp::InMemory && lazy) {
            for (const auto& [o, i] : item.swap.pairs) std::swap(mem[size_t(o)], mem[size_t(i)]);
            continue;
        }
        const bool cross = item.swap.kind == quokka::SwapOp::CrossRank;
        if (cross) {
            std::vector<int> outs;
            for (const auto& [o, i] : item.swap.pairs) outs.push_back(o);
            if (partialMaterialize()) flushAndMaterialize(&outs);
            else flushAndMaterialize();
        } else {
            flushStream(false);
            stream.clear();
        }
        CompiledItem ci;
        ci.kind = cross ? CompiledItem::Xrs : CompiledItem::Ims;
        for (const auto& [o, i] : item.swap.pairs) {
            ci.outs.push_back(o);
            ci.ins.push_back(i);
        }
        c->items.push_back(std::move(ci));
    }
    flushAndMaterialize();
    // The program's last pass also writes per-tile sums of |a|^2, so the norm
    // after a run needs no extra sweep of the slice (qk_norm).  Not for the
    // synthesized single-tile first pass, nor the TMA-pipelined kernels.
    auto markNorm = [&](std::vector<CompiledItem>& items, bool firstIsSynth) {
        if (items.empty() || items.back().kind != CompiledItem::Block || items.back().steps.empty()) return;
        qkeng::Step& s = items.back().steps.back();
        if (s.kind != qkeng::Step::Pass) return;
        if (firstIsSynth && items.size() == 1 && items[0].steps.size() == 1) return;
        s.pass->norm_out = 1;
        for (auto& a : s.alts) a->norm_out = 1;
    };
    for (Alternative& alt : c->alts)
        if (alt.last == c->items.size()) markNorm(alt.b, synthFirst && alt.first == 0);
    markNorm(c->items, synthFirst);
    if (deferScope) {
        deferScope.reset();
        c->basisAmp = qkeng::deferredHScale(deferH);
        auto stamp = [&](std::vector<CompiledItem>& items) {  // the synthesized basis pass
            if (items.empty() || items[0].kind != CompiledItem::Block || items[0].steps.empty()) return;
            qkeng::Step& s0 = items[0].steps[0];
            if (s0.kind != qkeng::Step::Pass) return;
            s0.pass->synth_amp = c->basisAmp;
            for (auto& a : s0.alts) a->synth_amp = c->basisAmp;
        };
        stamp(c->items);
        for (Alternative& alt : c->alts)
            if (alt.first == 0) stamp(alt.b);
    }
    return c;
}

// fromBasis: the run starts from a basis state (qk_simulate), whose memory
// layout is free: |x> with its bits permuted is just another basis state.
// The slice then starts in the layout that the first gate stream's lazy
// SQS / SWAP relabels carry to the program's physical order, so that stream
// ends with nothing to materialize (no IMS pass).  Runs on an existing state
// (qk_apply_block) start from the identity layout.
// jit: schedule for the specialized kernels (1), the interpreter (0), or
// whichever runs a 2^nLocal slice (-1).  The two get different schedules
// (interpreter: rb = 3, tiles <= 2^12).
// share = false: neither read nor fill the process-wide cache (throwaway
// compilations, e.g. qk_config_tune's candidates, must not evict live ones).
std::shared_ptr<Compiled> compileFor(qk_program* p, int nLocal, bool fromBasis = true, int jit = -1,
                                     bool share = true) {
    std::lock_guard<std::mutex> lk(p->mu);
    const bool interp = jit < 0 ? !useJit(nLocal) : jit == 0;
    const int slot = (fromBasis ? nLocal : -1 - nLocal) * 2 + (interp ? 1 : 0);
    auto it = p->compiled.find(slot);
    if (it != p->compiled.end()) return it->second;
    const std::string key = share ? scheduleKey(p->prog, slot) : std::string();
    if (share) {
        ScheduleCache& sc = scheduleCache();
        std::lock_guard<std::mutex> g(sc.mu);
        auto hit = sc.byKey.find(key);
        if (hit != sc.byKey.end()) return p->compiled[slot] = hit->second;
    }
    std::vector<int> ident(static_cast<size_t>(nLocal));
    for (int b = 0; b < nLocal; b++) ident[size_t(b)] = b;
    std::shared_ptr<Compiled> c = compileLayout(p, nLocal, ident, fromBasis, interp);
    if (lazyIms() && fromBasis && basisLayout()) {
        // sim = the first stream's relabels applied to the identity; starting
        // from its inverse, mem is the identity when that stream ends.  The
        // layout changes the scheduler's tiles too, so keep whichever
        // compilation costs fewer weighted sweeps (ties: the free layout).
        std::vector<int> sim = ident, mem0(static_cast<size_t>(nLocal));
        for (const quokka::ProgramItem& item : p->prog.items) {
            if (item.type == quokka::ProgramItem::Block) {
                for (const quokka::Gate& g : item.block.gates)
                    if (g.kind == quokka::GateKind::SWAP) std::swap(sim[size_t(g.targets[0])], sim[size_t(g.targets[1])]);
                continue;
            }
            if (item.swap.kind != quokka::SwapOp::InMemory) break;
            for (const auto& [o, i] : item.swap.pairs) std::swap(sim[size_t(o)], sim[size_t(i)]);
        }
        for (int q = 0; q < nLocal; q++) mem0[size_t(sim[size_t(q)])] = q;
        if (mem0 != ident) {
            std::shared_ptr<Compiled> b = compileLayout(p, nLocal, mem0, fromBasis, interp);
            if (sweeps(*b, fromBasis) <= sweeps(*c, fromBasis)) c = b;
        }
    }
    p->compiled[slot] = c;
    if (share) {
        ScheduleCache& sc = scheduleCache();
        std::lock_guard<std::mutex> g(sc.mu);
        if (sc.byKey.emplace(key, c).second) {
            sc.order.push_back(key);
            if (sc.order.size() > ScheduleCache::kMax) {
                sc.byKey.erase(sc.order.front());
                sc.order.erase(sc.order.begin());
            }
        }
    }
    return c;
}

DeviceTables tablesFor(qk_program* p, const Compiled& c, int device) {
    std::lock_guard<std::mutex> lk(p->mu);
    auto key = std::make_pair(&c, device);
    auto it = p->tables.find(key);
    if (it != p->tables.end()) return it->second;
    DeviceTables t;
    DeviceGuard g(device);
    const size_t gbytes = std::max<size_t>(16, c.gtab.size() * sizeof(double));
    cuda(cudaMalloc(&t.gtab, gbytes), "cudaMalloc(gtab)");
    if (!c.gtab.empty()) cuda(cudaMemcpy(t.gtab, c.gtab.data(), c.gtab.size() * sizeof(double), cudaMemcpyHostToDevice), "upload gtab");
    const size_t tbytes = std::max<size_t>(4, c.targets.size() * sizeof(int));
    cuda(cudaMalloc(&t.targets, tbytes), "cudaMalloc(targets)");
    if (!c.targets.empty()) cuda(cudaMemcpy(t.targets, c.targets.data(), c.targets.size() * sizeof(int), cudaMemcpyHostToDevice), "upload targets");
    p->tables[key] = t;
    return t;
}

// Profiling: CUDA events on the state's stream around each launch class.
struct Timer {
    qk_state* st;
    // classes: 0 block items, 1 IMS, 2 XRS, 3 full-slice fused passes, 4 init (first pass / memset)
    static constexpr int kClasses = 6;  // + 5: passes with known zeros in their input
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[kClasses];
    explicit Timer(qk_state* s) : st(s) {}
    template <class F>
    void time(int cls, F&& f) {
        if (!st->profiling) {
            f();
            return;
        }
        cudaEvent_t a, b;
        cuda(cudaEventCreate(&a), "event");
        cuda(cudaEventCreate(&b), "event");
        cuda(cudaEventRecord(a, st->stream), "event record");
        f();
        cuda(cudaEventRecord(b, st->stream), "event record");
        ev[cls].emplace_back(a, b);
    }
    void collect(double out[kClasses]) {
        for (int c = 0; c < kClasses; c++) {
            out[c] = 0;
            for (auto& [a, b] : ev[c]) {
                float ms = 0;
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                out[c] += ms;
                static const bool perItem = std::getenv("QK_PROFILE_ITEMS") != nullptr;
                static const char* names[kClasses] = {"block", "ims", "xrs", "pass", "init", "sparse pass"};
                if (perItem) std::fprintf(stderr, "qk item %s %.3f ms\n", names[c], ms);
                cudaEventDestroy(a);
                cudaEventDestroy(b);
            }
            ev[c].clear();
        }
    }
};

// Large slices run each pass as a straight-line specialized kernel (jit.h);
// the interpreter kernel serves small slices (no compile latency).
bool useJit(int nLocal) { return qkjit::minQubits() >= 0 && nLocal >= qkjit::minQubits(); }

// Compile (once, cached by content hash) every pass of a compiled program.
void prepareJit(const Compiled& c, int device) {
    if (!useJit(c.nLocal)) return;
    std::vector<const qkdev::PassParams*> passes;
    auto add = [&](const std::vector<CompiledItem>& items) {
        for (const CompiledItem& it : items)
            for (const qkeng::Step& s : it.steps)
                if (s.kind == qkeng::Step::Pass) {
                    passes.push_back(s.pass.get());
                    for (const auto& a : s.alts) passes.push_back(a.get());
                }
    };
    add(c.items);
    for (const Alternative& a : c.alts) add(a.b);
    qkjit::prepare(passes, device);
}

constexpr uint64_t kNoBasis = ~uint64_t(0);

// Autotune state (Step::Tune, ChoiceTune) lives in schedules shared through
// the process-wide cache; one host thread per GPU may run the same schedule
// concurrently, so every read-modify-write of it holds this lock.
std::mutex& tuneMu() {
    static std::mutex m;
    return m;
}

// QK_SPARSE_START (default 1): passes of a run from a basis state skip the
// reads (and whole tiles) known to be zero, and the basis pass skips the
// memset when the next pass writes every tile.
bool sparseStart() {
    static const bool v = [] {
        const char* e = std::getenv("QK_SPARSE_START");
        return !e || std::atoi(e) != 0;
    }();
    return v;
}

// QK_DEFER_ZEROS (default 1): a sparse pass followed by another sparse pass
// leaves its zero tiles unwritten (the chain's last pass writes them).
bool deferZeros() {
    static const bool v = [] {
        const char* e = std::getenv("QK_DEFER_ZEROS");
        return !e || std::atoi(e) != 0;
    }();
    return v;
}

// QK_DENSE_MODE: 0 = DFMA, 1 = DMMA (FP64 tensor cores) for the U5 tile
// kernel; unset = time both on a step's first executions, keep the faster.
std::atomic<int>& denseModeVar() {
    static std::atomic<int> v{[] {
        const char* e = std::getenv("QK_DENSE_MODE");
        return e ? std::atoi(e) : -1;
    }()};
    return v;
}
int denseMode() { return denseModeVar().load(); }

int smCountOf(int device) {
    static std::mutex mu;
    static std::map<int, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(device);
    if (it != cache.end()) return it->second;
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return cache[device] = n;
}

// basis != kNoBasis: the first step is a pass that synthesizes |basis> (slice
// index) instead of reading the slice (replaces initState's memset + store).
// Support of a run from a basis state (qk_simulate): the slice is zero
// outside {i : (i ^ val) & mask == 0}.  Every pass, dense group and IMS
// frees or permutes bits; mask == 0 means "no known zeros".  Specialized
// passes use it to skip the reads (and, for whole tiles outside it, the
// arithmetic) of amplitudes known to be zero.
struct Support {
    uint64_t mask = 0, val = 0;
    // the whole slice is zero (a rank that does not hold |initial>, before its
    // first cross-rank swap): every block and IMS step is skipped -- zeros in,
    // zeros out -- instead of sweeping HBM for nothing (on 2^R GPUs these
    // ranks would otherwise be the critical path to the first XRS barrier)
    bool empty = false;
};

void runBlock(qk_state* st, const CompiledItem& ci, const DeviceTables& t, qk_run_stats& rs,
              uint64_t basis = kNoBasis, Timer* timer = nullptr, Support* sup = nullptr) {
    const double amps = double(st->count);
    for (size_t si = 0; si < ci.steps.size(); si++) {
        const qkeng::Step& s = ci.steps[si];
        st->normValid = false;
        if (sup && sup->empty && !(s.kind == qkeng::Step::Pass && basis != kNoBasis)) continue;  // zeros stay zeros
        if (s.kind == qkeng::Step::Pass) {
            const bool jit = useJit(st->nLocal);
            // known zeros in this pass's input (not for the basis-synthesizing pass)
            const uint64_t smask = (jit && sup && basis == kNoBasis) ? sup->mask : 0;
            // Register-width autotune: the first two executions of a pass time
            // each variant (events, synchronous); later ones take the faster.
            // (With known zeros the TMA-pipelined variant reads only the
            // support and writes its tiles through TMA bulk stores.)
            const int nv = 1 + int(s.alts.size());
            int v = 0;
            bool timing = false;
            if (s.tune) {
                std::lock_guard<std::mutex> lk(tuneMu());
                v = s.tune->choice(nv);
                timing = s.tune->needsTiming(v);
            }
            const qkdev::PassParams& P = v ? *s.alts[size_t(v - 1)] : *s.pass;
            // The basis pass computes one tile; the memset of the rest is
            // skipped when the next step is a specialized pass that writes
            // every tile itself (launched with the known zeros).
            const bool zeroFill = !(sup && sup->mask && jit && basis != kNoBasis && (basis >> st->nLocal) == 0 &&
                                    si + 1 < ci.steps.size() && ci.steps[si + 1].kind == qkeng::Step::Pass);
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (timing) {
                cuda(cudaEventCreate(&e0), "event");
                cuda(cudaEventCreate(&e1), "event");
                cuda(cudaEventRecord(e0, st->stream), "event");
            }
            const bool fusedNorm = P.norm_out && useJit(st->nLocal) && basis == kNoBasis;
            // one partial sum per warp of every tile (2^(ct-rb-5) warps per tile)
            const uint64_t normParts = st->count >> std::min(P.ct, P.rb + 5);
            if (P.norm_out && useJit(st->nLocal)) {
                const uint64_t tiles = normParts;
                if (st->normTilesCap < tiles) {
                    cudaFree(st->normTiles);
                    st->normTiles = nullptr;
                    cuda(cudaMalloc(&st->normTiles, tiles * sizeof(double)), "cudaMalloc(norm tiles)");
                    st->normTilesCap = tiles;
                }
            }
            // Tiles with rows under 128 B write zeros inefficiently: a sparse
            // pass over such tiles leaves the ones outside the support to one
            // coalesced zero-fill (disjoint from the support, so any order).
            //
            // Deferred zeros: when the support is still partial after this pass
            // and the next step is a pass that runs with it, this pass need
            // not write its zero tiles at all -- the next pass reads only
            // inside the support (= this pass's written tiles), and the last
            // pass of the chain writes every tile.  QFT-33's middle pass then
            // computes only the tiles meeting the support.
            // known zeros after this pass (bits no non-diagonal gate touched stay known)
            uint64_t afterMask = smask, afterVal = smask ? sup->val : 0;
            if (smask) qkeng::supportAfter(s, P.tile_mask, afterMask, afterVal);
            const bool nextSparse = afterMask && si + 1 < ci.steps.size() &&
                                    ci.steps[si + 1].kind == qkeng::Step::Pass && deferZeros();
            const bool fillShort = smask && !nextSparse && qkjit::lowRunOf(P) < 3;
            const bool zeroSkip = nextSparse || fillShort;
            auto launchPass = [&] {
                if (fillShort)
                    cuda(qkdev::launchZeroOutside(st->amps, st->count, smask & ~P.tile_mask, sup->val,
                                                  smCountOf(st->device), st->stream),
                         "zero-fill outside the support");
                if (jit)
                    cuda(qkjit::launch(P, st->amps, t.gtab, st->nLocal, basis, st->stream,
                                       P.norm_out ? st->normTiles : nullptr, smask, smask ? sup->val : 0, zeroFill,
                                       nextSparse && !P.norm_out ? 2 : zeroSkip ? 1 : 0),
                         "specialized block pass");
                else
                    cuda(qkdev::launchBlockPass(st->amps, t.gtab, P, st->nLocal, basis, st->stream), "block pass");
            };
            if (timer) timer->time(basis != kNoBasis ? 4 : smask ? 5 : 3, launchPass);
            else launchPass();
            if (fillShort) rs.kernel_launches++;
            // algorithmic bytes: write every amplitude; read those not known to be zero
            if (basis != kNoBasis) {
                rs.block_bytes += zeroFill ? 16.0 * amps : 16.0 * double(uint64_t(1) << P.ct);
            } else if (smask) {
                const double written = nextSparse ? std::ldexp(amps, -__builtin_popcountll(afterMask)) : amps;
                const double b = 16.0 * written + 16.0 * std::ldexp(amps, -__builtin_popcountll(smask));
                rs.sparse_pass_launches++;
                rs.sparse_pass_bytes += b;
                rs.block_bytes += b;
            } else {
                rs.full_pass_launches++;
                rs.full_pass_bytes += 32.0 * amps;
                rs.block_bytes += 32.0 * amps;
            }
            if (sup && jit) qkeng::supportAfter(s, P.tile_mask, sup->mask, sup->val);  // frees the bits it mixes
            if (timing) {
                float ms = 0;
                cuda(cudaEventRecord(e1, st->stream), "event");
                cuda(cudaEventSynchronize(e1), "event");
                cudaEventElapsedTime(&ms, e0, e1);
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
                std::lock_guard<std::mutex> lk(tuneMu());
                s.tune->record(v, ms);
                s.tune->runs[v]++;
                rs.tuning_runs++;
                if (std::getenv("QK_DEBUG_TUNE")) {
                    const qkdev::PassParams& Q = v ? *s.alts[size_t(v - 1)] : *s.pass;
                    std::fprintf(stderr, "pass variant %d (ct %d rb %d segs %d%s): %.3f ms\n", v, Q.ct, Q.rb, Q.nsegs,
                                 qkjit::pipelinedPass(Q) ? ", TMA-pipelined" : "", double(ms));
                }
            } else if (s.tune) {
                std::lock_guard<std::mutex> lk(tuneMu());
                s.tune->runs[v]++;
            }
            if (fusedNorm) {
                cuda(qkdev::launchSumTiles(st->normTiles, normParts, st->normScratch, st->normOut, st->stream),
                     "norm fold");
                rs.kernel_launches += 2;  // k_sum_partial + k_norm_final
                st->normValid = true;
            }
            basis = kNoBasis;
        } else if (s.kind == qkeng::Step::DiagTable) {
            rs.block_bytes += 32.0 * amps;
            cuda(qkdev::launchDiagTable(st->amps, t.gtab + s.matOff, st->count, s.targets.data() + 1, s.k, st->stream),
                 "diag table");
        } else if (s.k == 5 && st->nLocal >= 12 && denseMode() != 2) {
            rs.block_bytes += 32.0 * amps;
            const uint64_t dmask = (sup && useJit(st->nLocal)) ? sup->mask : 0;  // known zeros of this step's input
            if (sup)
                for (size_t j = 1; j < s.targets.size(); j++) sup->mask &= ~(uint64_t(1) << s.targets[j]);
            // U5 tile kernel, DFMA or DMMA: the first two executions time
            // both (events, synchronous), later ones take the faster
            int v = denseMode();
            bool timing = false;
            if (v < 0) {
                std::lock_guard<std::mutex> lk(tuneMu());
                v = s.tune ? s.tune->choice(2) : 0;
                timing = s.tune && s.tune->needsTiming(v);
            }
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (timing) {
                cuda(cudaEventCreate(&e0), "event");
                cuda(cudaEventCreate(&e1), "event");
                cuda(cudaEventRecord(e0, st->stream), "event");
            }
            cuda(qkdev::launchDenseTile(st->amps, t.gtab + s.matOff, s.targets.data() + 1, s.k, st->nLocal, v,
                                        smCountOf(st->device), st->stream, dmask, dmask ? sup->val : 0),
                 "dense U5 tile");
            if (timing) {
                float ms = 0;
                cuda(cudaEventRecord(e1, st->stream), "event");
                cuda(cudaEventSynchronize(e1), "event");
                cudaEventElapsedTime(&ms, e0, e1);
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
                std::lock_guard<std::mutex> lk(tuneMu());
                s.tune->record(v, ms);
                rs.tuning_runs++;
                if (std::getenv("QK_DEBUG_TUNE"))
                    std::fprintf(stderr, "dense U5 %s: %.3f ms\n", v ? "DMMA" : "DFMA", double(ms));
            }
            if (s.tune) {
                std::lock_guard<std::mutex> lk(tuneMu());
                s.tune->runs[v]++;
            }
        } else {
            uint64_t mask = 0;
            for (size_t j = 1; j < s.targets.size(); j++) mask |= uint64_t(1) << s.targets[j];
            rs.block_bytes += 32.0 * amps;
            if (sup) sup->mask &= ~mask;
            cuda(qkdev::launchDenseGroup(st->amps, t.gtab + s.matOff, s.k, t.targets + s.targets[0], mask, st->nLocal,
                                         st->stream),
                 "dense group");
        }
        rs.kernel_launches++;
        rs.block_launches++;
    }
    rs.block_flops += ci.flopsPerAmp * double(st->count);
}

uint64_t swapBits(uint64_t x, const std::vector<int>& outs, const std::vector<int>& ins) {
    for (size_t j = 0; j < outs.size(); j++) {
        const uint64_t d = ((x >> outs[j]) ^ (x >> ins[j])) & 1u;
        x ^= (d << outs[j]) | (d << ins[j]);
    }
    return x;
}

void runIms(qk_state* st, const std::vector<int>& outs, const std::vector<int>& ins, qk_run_stats& rs,
            Support* sup = nullptr) {
    st->normValid = false;
    if (sup && sup->empty) return;  // a permutation of zeros
    if (sup) {  // a[bitswap(i)] <- a[i]: the known-zero coset moves with its bits
        sup->mask = swapBits(sup->mask, outs, ins);
        sup->val = swapBits(sup->val, outs, ins);
    }
    if (outs.empty()) return;
    cuda(qkdev::launchIms(st->amps, st->nLocal, outs.data(), ins.data(), int(outs.size()), st->stream), "ims");
    rs.kernel_launches++;
    rs.ims_launches++;
    rs.ims_bytes += 32.0 * double(st->count) * (1.0 - std::ldexp(1.0, -int(outs.size())));
}

void ensureXrsBuffers(qk_state* st, uint64_t amps, bool pack) {
    if (st->bufAmps < amps) {
        DeviceGuard g(st->device);
        cudaFree(st->recvBuf);
        cudaFree(st->packBuf);
        st->recvBuf = st->packBuf = nullptr;
        cuda(cudaMalloc(&st->recvBuf, amps * sizeof(double2)), "cudaMalloc(recv buffer)");
        st->bufAmps = amps;
    }
    if (pack && !st->packBuf) cuda(cudaMalloc(&st->packBuf, st->bufAmps * sizeof(double2)), "cudaMalloc(pack buffer)");
}

// NCCL XRS for this rank (one process per GPU): per window round, one grouped
// ncclSend/ncclRecv per partner into a single receive buffer, then copy-back.
// One rank's side of an XRS (distributed.cpp:76-120) as the NCCL path runs
// it: per window round, pack (only if the outs are not the AIO-staged top S
// in-rank positions), exchange, copy back from the single receive buffer.
struct XrsRank {
    qk_state* st;
    const XrsPlan& p;
    bool contiguous = true;
    std::vector<qk_xrs_msg> msgs;
    XrsRank(qk_state* s, const XrsPlan& plan) : st(s), p(plan) {
        for (int j = 0; j < p.s; j++) contiguous &= p.outs[size_t(j)] == st->nLocal - p.s + j;
        ensureXrsBuffers(st, 2 * uint64_t((1 << p.s) - 1) * p.window, !contiguous);  // two receive halves
        msgs = xrsMessages(p, st->rank);
    }
    const double2* sendSrc(const qk_xrs_msg& x) const {
        return contiguous ? st->amps + slabBits(x.slab, p) + x.w0 : st->packBuf + uint64_t(x.section) * x.count;
    }
    double2* recvDst(const qk_xrs_msg& x) const { return st->recvBuf + uint64_t(x.section) * x.count; }
    void pack(size_t a, size_t b, qk_run_stats& rs) {
        if (contiguous) return;
        for (size_t m = a; m < b; m++) {
            cuda(qkdev::launchWindowPack(st->packBuf + uint64_t(msgs[m].section) * msgs[m].count,
                                         st->amps + slabBits(msgs[m].slab, p), msgs[m].w0, msgs[m].count,
                                         p.outs.data(), p.s, st->stream),
                 "xrs pack");
            rs.kernel_launches++;
        }
    }
    void unpack(size_t a, size_t b, qk_run_stats& rs, cudaStream_t on = nullptr, uint64_t bufOffset = 0) {
        for (size_t m = a; m < b; m++) {
            const qk_xrs_msg& x = msgs[m];
            cuda(qkdev::launchWindowUnpack(st->amps + slabBits(x.slab, p), recvDst(x) + bufOffset, x.w0, x.count,
                                           p.outs.data(), p.s, on ? on : st->stream),
                 "xrs copy-back");
            rs.kernel_launches++;
        }
    }
    size_t roundEnd(size_t a) const {
        size_t b = a;
        while (b < msgs.size() && msgs[b].round == msgs[a].round) b++;
        return b;
    }
};

// NCCL XRS for this rank (one process per GPU): per window round, one grouped
// ncclSend/ncclRecv per partner into the receive buffer, then copy-back
// (distributed.cpp:183-191).  The buffer is double-buffered: round k lands
// in half k % 2 and its copy-back runs on a second stream, overlapping the
// transfer of round k + 1; round k + 2 waits for that copy-back before it
// reuses the half.  Sends read the slab windows in place when the outs are
// the AIO-staged top S positions (else a pack kernel fills packBuf).
void runXrsNccl(qk_state* st, const XrsPlan& p, qk_run_stats& rs) {
    st->normValid = false;
    if (!st->comm)
        throw SimulationError("cross-rank swap needs a communicator (qk_comm_init / qk_ipc_init) or qk_simulate_local");
    if (p.s == 0) return;
    XrsRank x(st, p);
    if (!st->aux) {
        cuda(cudaStreamCreateWithFlags(&st->aux, cudaStreamNonBlocking), "xrs copy-back stream");
        for (int h = 0; h < 2; h++) {
            cuda(cudaEventCreateWithFlags(&st->xrsDone[h], cudaEventDisableTiming), "event");
            cuda(cudaEventCreateWithFlags(&st->unpackDone[h], cudaEventDisableTiming), "event");
        }
    }
    const uint64_t half = uint64_t((1 << p.s) - 1) * p.window;  // one round's receive sections
    bool used[2] = {false, false};
    int round = 0;
    for (size_t a = 0; a < x.msgs.size(); round++) {
        const size_t b = x.roundEnd(a);
        const int h = round & 1;
        if (used[h]) cuda(cudaStreamWaitEvent(st->stream, st->unpackDone[h], 0), "xrs wait copy-back");
        x.pack(a, b, rs);
        nccl(ncclGroupStart(), "ncclGroupStart");
        for (size_t m = a; m < b; m++) {
            const qk_xrs_msg& msg = x.msgs[m];
            nccl(ncclSend(x.sendSrc(msg), 2 * msg.count, ncclDouble, msg.peer, st->comm, st->stream), "ncclSend");
            nccl(ncclRecv(x.recvDst(msg) + uint64_t(h) * half, 2 * msg.count, ncclDouble, msg.peer, st->comm,
                          st->stream),
                 "ncclRecv");
        }
        nccl(ncclGroupEnd(), "ncclGroupEnd");
        cuda(cudaEventRecord(st->xrsDone[h], st->stream), "event");
        cuda(cudaStreamWaitEvent(st->aux, st->xrsDone[h], 0), "xrs copy-back wait");
        x.unpack(a, b, rs, st->aux, uint64_t(h) * half);
        cuda(cudaEventRecord(st->unpackDone[h], st->aux), "event");
        used[h] = true;
        rs.xrs_rounds++;
        a = b;
    }
    for (int h = 0; h < 2; h++)
        if (used[h]) cuda(cudaStreamWaitEvent(st->stream, st->unpackDone[h], 0), "xrs join copy-back");
    rs.xrs_bytes += 16.0 * double(st->count) * (1.0 - std::ldexp(1.0, -p.s));
}

// The same per-rank schedule with every rank in this process and the NCCL
// transfer replaced by device copies (send matched to receive by peer and
// round, as NCCL's grouped point-to-point does).  Test hook for the NCCL
// path's plan, pack and copy-back kernels on a single GPU.
void runXrsLoopback(qk_state** sl, int ns, const XrsPlan& p) {
    for (int k = 0; k < ns; k++) sl[k]->normValid = false;
    if (p.s == 0) return;
    std::vector<std::unique_ptr<XrsRank>> rk;
    for (int r = 0; r < ns; r++) rk.push_back(std::make_unique<XrsRank>(sl[r], p));
    qk_run_stats rs{};
    std::vector<size_t> pos(static_cast<size_t>(ns), 0);
    for (;;) {
        bool any = false;
        std::vector<size_t> end(static_cast<size_t>(ns));
        for (int r = 0; r < ns; r++) {
            end[size_t(r)] = pos[size_t(r)] < rk[size_t(r)]->msgs.size() ? rk[size_t(r)]->roundEnd(pos[size_t(r)])
                                                                        : pos[size_t(r)];
            any |= end[size_t(r)] > pos[size_t(r)];
        }
        if (!any) break;
        for (int r = 0; r < ns; r++) {
            DeviceGuard g(sl[r]->device);
            rk[size_t(r)]->pack(pos[size_t(r)], end[size_t(r)], rs);
        }
        for (int r = 0; r < ns; r++) cuda(cudaStreamSynchronize(sl[r]->stream), "loopback pack");
        for (int r = 0; r < ns; r++)
            for (size_t m = pos[size_t(r)]; m < end[size_t(r)]; m++) {
                const qk_xrs_msg& in = rk[size_t(r)]->msgs[m];  // r receives from in.peer
                const XrsRank& q = *rk[size_t(in.peer)];
                const qk_xrs_msg* out = nullptr;
                for (size_t k = pos[size_t(in.peer)]; k < end[size_t(in.peer)]; k++)
                    if (q.msgs[k].peer == r) out = &q.msgs[k];
                if (!out || out->count != in.count) throw SimulationError("xrs loopback: unmatched message");
                cuda(cudaMemcpyAsync(rk[size_t(r)]->recvDst(in), q.sendSrc(*out), in.count * sizeof(double2),
                                     cudaMemcpyDeviceToDevice, sl[r]->stream),
                     "loopback copy");
            }
        for (int r = 0; r < ns; r++) cuda(cudaStreamSynchronize(sl[r]->stream), "loopback copy");
        for (int r = 0; r < ns; r++) {
            DeviceGuard g(sl[r]->device);
            rk[size_t(r)]->unpack(pos[size_t(r)], end[size_t(r)], rs);
        }
        for (int r = 0; r < ns; r++) cuda(cudaStreamSynchronize(sl[r]->stream), "loopback unpack");
        pos = end;
    }
}

// Slices of one process on different GPUs: map every pair of their devices
// for peer loads/stores (NVLink) so the slab-swap kernel can reach both.
void enablePeers(qk_state** sl, int ns) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    for (int a = 0; a < ns; a++)
        for (int b = 0; b < ns; b++) {
            const int da = sl[a]->device, db = sl[b]->device;
            if (da == db) continue;
            int can = 0;
            cuda(cudaDeviceCanAccessPeer(&can, da, db), "cudaDeviceCanAccessPeer");
            if (!can) throw SimulationError("devices " + std::to_string(da) + " and " + std::to_string(db) +
                                            " have no peer access: use one process per GPU (qk_comm_init)");
            DeviceGuard g(da);
            const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else cuda(e, "cudaDeviceEnablePeerAccess");
        }
}

// In-process XRS: every slab pair swapped in place by one kernel reading and
// writing both slices (same device or peer-mapped).  No buffer, no copy-back.
void runXrsLocal(qk_state** sl, int ns, const XrsPlan& p) {
    for (int k = 0; k < ns; k++) sl[k]->normValid = false;
    for (int k = 0; k < ns; k++) cuda(cudaStreamSynchronize(sl[k]->stream), "xrs pre-sync");
    const int slabs = 1 << p.s;
    for (int r = 0; r < ns; r++) {
        const int own = ownSlab(r, p);
        std::vector<double2*> A, B;
        for (int pa = 0; pa < slabs; pa++) {
            if (pa == own) continue;
            const int q = partnerOf(r, pa, p);
            if (q < r) continue;  // each unordered slab pair once
            A.push_back(sl[r]->amps + slabBits(pa, p));
            B.push_back(sl[q]->amps + slabBits(own, p));
        }
        if (A.empty()) continue;
        const std::vector<uint64_t> o0(A.size(), 0), cnt(A.size(), p.slabOffsets);
        DeviceGuard g(sl[r]->device);
        cuda(qkdev::launchSlabSwap(int(A.size()), A.data(), B.data(), o0.data(), cnt.data(), p.outs.data(), p.s,
                                   sl[r]->stream),
             "xrs slab swap");
    }
    for (int k = 0; k < ns; k++) cuda(cudaStreamSynchronize(sl[k]->stream), "xrs post-sync");
}

// Multi-process XRS over peer memory (qk_ipc_init): every rank maps every
// other rank's slice, so a CSQS is one in-place swap kernel per rank over all
// its partner slab pairs -- no exchange buffer, no copy-back pass.  Each
// unordered slab pair is split in halves: the lower rank swaps the first
// half of its elements, the higher rank the second, so both directions of
// every link carry half the slab.  Host barriers bracket the kernel: every
// rank's earlier items are done before any peer touches its slice, and every
// swap is done before any rank goes on.
void runXrsIpc(qk_state* st, const XrsPlan& p, qk_run_stats& rs) {
    st->normValid = false;
    if (p.s == 0) return;
    cuda(cudaStreamSynchronize(st->stream), "xrs pre-sync");
    qkipc::barrier(st->ipc);
    const int own = ownSlab(st->rank, p), slabs = 1 << p.s;
    const uint64_t half = p.slabOffsets / 2;
    std::vector<double2*> A, B;
    std::vector<uint64_t> o0, cnt;
    for (int pa = 0; pa < slabs; pa++) {
        if (pa == own) continue;
        const int q = partnerOf(st->rank, pa, p);
        A.push_back(st->amps + slabBits(pa, p));
        B.push_back(static_cast<double2*>(qkipc::peer(st->ipc, q)) + slabBits(own, p));
        o0.push_back(st->rank < q ? 0 : half);
        cnt.push_back(st->rank < q ? half : p.slabOffsets - half);
    }
    cuda(qkdev::launchSlabSwap(int(A.size()), A.data(), B.data(), o0.data(), cnt.data(), p.outs.data(), p.s,
                               st->stream),
         "xrs peer swap");
    rs.kernel_launches += (A.size() + 7) / 8;
    cuda(cudaStreamSynchronize(st->stream), "xrs peer swap");
    qkipc::barrier(st->ipc);
    rs.xrs_rounds++;
    rs.xrs_bytes += 16.0 * double(st->count) * (1.0 - std::ldexp(1.0, -p.s));
}

// qk_gate[] -> quokka::Gate list (matrix order: controls first), validating
// arity and the chunk bound (engine.cpp:264-268).
std::vector<quokka::Gate> gatesFromC(const qk_gate* gates, int ngates, int bound) {
    std::vector<quokka::Gate> out;
    for (int i = 0; i < ngates; i++) {
        const qk_gate& g = gates[i];
        if (g.kind < QK_H || g.kind > QK_FUSED_DENSE) throw SimulationError("unknown gate kind");
        quokka::Gate q;
        q.kind = static_cast<quokka::GateKind>(g.kind);
        q.id = long(g.id);
        const int nq = g.nqubits;
        if (nq < 1 || nq > 16) throw SimulationError("bad gate arity");
        const bool fused = g.kind == QK_FUSED_DIAG || g.kind == QK_FUSED_DENSE;
        if (!fused && quokka::kindArity(q.kind) != nq) throw SimulationError("gate arity does not match its kind");
        if (g.kind == QK_CX || g.kind == QK_CP) {
            q.controls = {g.qubits[0]};
            q.targets = {g.qubits[1]};
        } else {
            q.targets.assign(g.qubits, g.qubits + nq);
        }
        for (int j = 0; j < quokka::kindParamCount(q.kind); j++) q.params.push_back(g.params[j]);
        if (fused) {
            if (!g.payload) throw SimulationError("fused gate without payload");
            const size_t e = size_t(1) << (g.kind == QK_FUSED_DIAG ? nq : 2 * nq);
            for (size_t j = 0; j < e; j++) q.payload.emplace_back(g.payload[2 * j], g.payload[2 * j + 1]);
        }
        for (int qq : q.qubits())
            if (qq < 0 || qq >= bound)
                throw SimulationError("block gate " + std::to_string(q.id) + " reaches outside the chunk");
        out.push_back(std::move(q));
    }
    return out;
}

// JSON dump of the compiled steps (scheduler test hook: tests/emulator.py
// replays the pass programs on the CPU to check the scheduler without a GPU).
std::string stepsJson(const std::vector<qkeng::Step>& steps, const std::vector<double>& gtab) {
    std::ostringstream o;
    o.precision(17);
    o << "{\"gtab\":[";
    for (size_t i = 0; i < gtab.size(); i++) o << (i ? "," : "") << gtab[i];
    o << "],\"steps\":[";
    for (size_t si = 0; si < steps.size(); si++) {
        const qkeng::Step& s = steps[si];
        o << (si ? "," : "") << "{\"kind\":" << int(s.kind) << ",\"k\":" << s.k << ",\"mat\":" << s.matOff
          << ",\"targets\":[";
        for (size_t j = 0; j < s.targets.size(); j++) o << (j ? "," : "") << s.targets[j];
        o << "]";
        if (s.kind == qkeng::Step::Pass) {
            const qkdev::PassParams& P = *s.pass;
            o << ",\"keep\":[";
            for (size_t j = 0; j < s.keep.size(); j++)
                o << (j ? "," : "") << "[" << s.keep[j].first << "," << s.keep[j].second << "]";
            o << "]";
            o << ",\"ct\":" << P.ct << ",\"rb\":" << P.rb << ",\"nsegs\":" << P.nsegs << ",\"tile_phys\":[";
            for (int j = 0; j < P.ct; j++) o << (j ? "," : "") << int(P.tile_phys[j]);
            o << "],\"map_in\":[";
            for (int g = 0; g < P.nsegs; g++) {
                o << (g ? "," : "") << "[";
                for (int j = 0; j < P.ct; j++) o << (j ? "," : "") << int(P.map_in[g][j]);
                o << "]";
            }
            o << "],\"map_out\":[";
            for (int g = 0; g < P.nsegs; g++) {
                o << (g ? "," : "") << "[";
                for (int j = 0; j < P.ct; j++) o << (j ? "," : "") << int(P.map_out[g][j]);
                o << "]";
            }
            o << "],\"xmask_out\":[";
            for (int g = 0; g < P.nsegs; g++) o << (g ? "," : "") << P.xmask_out[g];
            o << "],\"ops\":[";
            for (int i = 0; i < P.nops; i++) {
                const qkdev::DevOp& d = P.ops[i];
                o << (i ? "," : "") << "[" << int(d.type) << "," << int(d.a) << "," << int(d.b) << "," << int(d.k)
                  << "," << d.c << "," << d.c16 << "," << d.x16 << "]";
            }
            o << "],\"coef\":[";
            for (int i = 0; i < 2 * qkdev::kMaxCoef; i++) o << (i ? "," : "") << P.coef[i];
            o << "],\"contrib\":[";
            for (int i = 0; i < qkdev::kMaxContrib; i++) o << (i ? "," : "") << P.contrib[i];
            o << "],\"ncta\":" << P.ncta << ",\"cta_end\":[";
            for (int f = 0; f < P.ncta; f++) o << (f ? "," : "") << P.cta_end[f];
            o << "],\"cta_terms\":[";
            const int nterms = P.ncta ? P.cta_end[P.ncta - 1] : 0;
            for (int t = 0; t < nterms; t++)
                o << (t ? "," : "") << "[" << int(P.cta_terms[t].b1) << "," << int(P.cta_terms[t].b2) << ","
                  << P.cta_terms[t].c << "]";
            o << "]";
        }
        o << "}";
    }
    o << "]}";
    return o.str();
}

void checkProgramAgainst(const quokka::Program& prog, const quokka::Config& cfg, int n, int R) {
    if (prog.nQubits != cfg.totalQubits || prog.rankQubits != cfg.rankQubits)
        throw ConfigError("program and config disagree on the qubit split");
    if (n != cfg.totalQubits || R != cfg.rankQubits) throw ConfigError("state and config disagree on the qubit split");
    const int region = cfg.rankRegion();
    // Validate every item up front (distributed.cpp:149-164): nothing throws mid-run.
    for (const quokka::ProgramItem& it : prog.items) {
        if (it.type == quokka::ProgramItem::Block) {
            for (const quokka::Gate& g : it.block.gates)
                for (int q : g.qubits())
                    if (q < 0 || q >= prog.chunkQubits)
                        throw SimulationError("block gate " + std::to_string(g.id) + " reaches outside the chunk");
        } else if (it.swap.kind == quokka::SwapOp::InMemory) {
            for (const auto& [a, b] : it.swap.pairs)
                if (a < 0 || b < 0 || a >= region || b >= region)
                    throw SimulationError("in-memory swap reaches into the rank bits");
        } else {
            if (R == 0) throw SimulationError("cross-rank swap in a single-rank run; use the multi-rank engine");
            planXrs(it.swap, cfg.totalQubits, cfg.rankQubits, cfg.bufferQubits);
        }
    }
}

// Slice-local index of a basis state in the memory layout `mem0` (program
// position p at memory bit mem0[p]).
uint64_t layoutIndex(uint64_t local, const std::vector<int>& mem0) {
    uint64_t x = 0;
    for (size_t p = 0; p < mem0.size(); p++) x |= ((local >> p) & 1) << mem0[p];
    return x;
}

void setBasis(qk_state* st, Index global, const std::vector<int>* mem0 = nullptr, double amp = 1.0) {
    st->normValid = false;
    if (global >= (Index(1) << st->n)) throw SimulationError("initial basis state out of range");
    cuda(cudaMemsetAsync(st->amps, 0, st->count * sizeof(double2), st->stream), "memset");
    uint64_t local = global & (st->count - 1);
    if (mem0) local = layoutIndex(local, *mem0);
    if ((global >> st->nLocal) == Index(st->rank)) cuda(qkdev::launchSetBasis(st->amps, local, st->stream, amp), "set basis");
}

}  // namespace

// ================================================================ C-ABI ======

extern "C" {

const char* qk_last_error(void) { return g_lastError.c_str(); }
void qk_free(void* p) { std::free(p); }

int qk_device_count(int* count) {
    return guard([&] { cuda(cudaGetDeviceCount(count), "cudaGetDeviceCount"); });
}

int qk_create(int n, int R, int rank, int B, int device, qk_state** out) {
    return guard([&] {
        if (n < 1 || n > 40) throw SimulationError("qubit count " + std::to_string(n) + " out of range");
        if (R < 0 || R >= n) throw ConfigError("rank_qbit must leave at least one in-rank qubit");
        if (rank < 0 || rank >= (1 << R)) throw ConfigError("rank out of range");
        int ndev = 0;
        cuda(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) throw SimulationError("no such CUDA device");
        auto st = std::make_unique<qk_state>();
        st->n = n;
        st->R = R;
        st->rank = rank;
        st->nLocal = n - R;
        st->B = B < 0 ? std::min(n - R, 28) : B;
        st->device = device;
        st->count = uint64_t(1) << st->nLocal;
        DeviceGuard g(device);
        cuda(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking), "stream");
        cuda(cudaMalloc(&st->amps, st->count * sizeof(double2)), "cudaMalloc(state)");
        cuda(cudaMalloc(&st->normScratch, qkdev::normScratchDoubles() * sizeof(double)), "cudaMalloc(norm)");
        cuda(cudaMalloc(&st->normOut, sizeof(double)), "cudaMalloc(norm)");
        setBasis(st.get(), Index(rank) << st->nLocal);
        *out = st.release();
    });
}

int qk_destroy(qk_state* st) {
    return guard([&] {
        if (!st) return;
        DeviceGuard g(st->device);
        cudaStreamSynchronize(st->stream);
        if (st->comm) ncclCommDestroy(st->comm);
        qkipc::leave(st->ipc);
        cudaFree(st->amps);
        cudaFree(st->normScratch);
        cudaFree(st->normOut);
        cudaFree(st->normTiles);
        cudaFree(st->recvBuf);
        cudaFree(st->packBuf);
        for (int h = 0; h < 2; h++) {
            if (st->xrsDone[h]) cudaEventDestroy(st->xrsDone[h]);
            if (st->unpackDone[h]) cudaEventDestroy(st->unpackDone[h]);
        }
        if (st->aux) cudaStreamDestroy(st->aux);
        cudaStreamDestroy(st->stream);
        delete st;
    });
}

int qk_set_basis(qk_state* st, uint64_t global) {
    return guard([&] {
        DeviceGuard g(st->device);
        setBasis(st, global);
    });
}

int qk_upload(qk_state* st, uint64_t off, uint64_t cnt, const double* host) {
    return guard([&] {
        st->normValid = false;
        if (off + cnt > st->count) throw SimulationError("upload range outside the slice");
        DeviceGuard g(st->device);
        cuda(cudaMemcpyAsync(st->amps + off, host, cnt * sizeof(double2), cudaMemcpyHostToDevice, st->stream), "upload");
        cuda(cudaStreamSynchronize(st->stream), "upload sync");
    });
}

int qk_download(qk_state* st, uint64_t off, uint64_t cnt, double* host) {
    return guard([&] {
        if (off + cnt > st->count) throw SimulationError("download range outside the slice");
        DeviceGuard g(st->device);
        cuda(cudaMemcpyAsync(host, st->amps + off, cnt * sizeof(double2), cudaMemcpyDeviceToHost, st->stream), "download");
        cuda(cudaStreamSynchronize(st->stream), "download sync");
    });
}

int qk_download_stream(qk_state* st, uint64_t off, uint64_t cnt, uint64_t chunk, qk_chunk_sink sink, void* user) {
    return guard([&] {
        if (off + cnt > st->count) throw SimulationError("download range outside the slice");
        if (!sink) throw SimulationError("no chunk sink");
        if (chunk == 0) chunk = uint64_t(1) << 22;  // 64 MiB per buffer
        chunk = std::min(chunk, std::max<uint64_t>(cnt, 1));
        DeviceGuard g(st->device);
        double2* buf[2] = {nullptr, nullptr};
        cudaEvent_t done[2] = {nullptr, nullptr};
        auto cleanup = [&] {
            for (int h = 0; h < 2; h++) {
                if (buf[h]) cudaFreeHost(buf[h]);
                if (done[h]) cudaEventDestroy(done[h]);
            }
        };
        try {
            for (int h = 0; h < 2; h++) {
                cuda(cudaMallocHost(&buf[h], chunk * sizeof(double2)), "cudaMallocHost(stream buffer)");
                cuda(cudaEventCreateWithFlags(&done[h], cudaEventDisableTiming), "event");
            }
            const uint64_t n = (cnt + chunk - 1) / chunk;
            auto issue = [&](uint64_t k) {
                const uint64_t o = off + k * chunk, m = std::min(chunk, cnt - k * chunk);
                const int h = int(k & 1);
                cuda(cudaMemcpyAsync(buf[h], st->amps + o, m * sizeof(double2), cudaMemcpyDeviceToHost, st->stream),
                     "stream chunk");
                cuda(cudaEventRecord(done[h], st->stream), "event");
            };
            if (n) issue(0);
            for (uint64_t k = 0; k < n; k++) {
                const int h = int(k & 1);
                cuda(cudaEventSynchronize(done[h]), "stream chunk");
                if (k + 1 < n) issue(k + 1);  // the other buffer: its sink call has returned
                const uint64_t m = std::min(chunk, cnt - k * chunk);
                if (sink(reinterpret_cast<const double*>(buf[h]), m, user) != 0)
                    throw SimulationError("download stream stopped by its sink");
            }
        } catch (...) {
            cudaStreamSynchronize(st->stream);
            cleanup();
            throw;
        }
        cleanup();
    });
}

int qk_norm(qk_state* st, double* out) {
    return guard([&] {
        DeviceGuard g(st->device);
        if (!st->normValid)  // else the last pass already folded sum |a|^2 into normOut
            cuda(qkdev::launchNorm(st->amps, st->count, st->normScratch, st->normOut, st->stream), "norm");
        cuda(cudaMemcpyAsync(out, st->normOut, sizeof(double), cudaMemcpyDeviceToHost, st->stream), "norm copy");
        cuda(cudaStreamSynchronize(st->stream), "norm sync");
    });
}

int qk_marginal(qk_state* st, const int* bits, int k, double* out) {
    return guard([&] {
        if (k < 0 || k > 10) throw SimulationError("marginal: 0 <= k <= 10 bits");
        for (int j = 0; j < k; j++)
            if (bits[j] < 0 || bits[j] >= st->nLocal) throw SimulationError("marginal: bit outside the slice");
        DeviceGuard g(st->device);
        double *scratch = nullptr, *dout = nullptr;
        cuda(cudaMallocAsync(&scratch, qkdev::marginalScratchDoubles(k) * sizeof(double), st->stream), "marginal");
        cuda(cudaMallocAsync(&dout, sizeof(double) << k, st->stream), "marginal");
        cuda(qkdev::launchMarginal(st->amps, st->count, bits, k, scratch, dout, st->stream), "marginal");
        cuda(cudaMemcpyAsync(out, dout, sizeof(double) << k, cudaMemcpyDeviceToHost, st->stream), "marginal copy");
        cuda(cudaFreeAsync(scratch, st->stream), "marginal");
        cuda(cudaFreeAsync(dout, st->stream), "marginal");
        cuda(cudaStreamSynchronize(st->stream), "marginal sync");
    });
}

int qk_synchronize(qk_state* st) {
    return guard([&] { cuda(cudaStreamSynchronize(st->stream), "synchronize"); });
}

int qk_stream(qk_state* st, void** s) {
    return guard([&] { *s = st->stream; });
}

int qk_set_profiling(qk_state* st, int on) {
    return guard([&] { st->profiling = on != 0; });
}

int qk_apply_block(qk_state* st, const qk_gate* gates, int ngates, int chunk) {
    return guard([&] {
        quokka::Program p;
        p.nQubits = st->n;
        p.rankQubits = st->R;
        p.chunkQubits = chunk;
        quokka::GateBlock blk;
        blk.gates = gatesFromC(gates, ngates, chunk);
        if (chunk < 1 || chunk > st->nLocal) throw SimulationError("chunk size out of range");
        p.items.push_back(quokka::ProgramItem::makeBlock(std::move(blk)));
        qk_program prog;
        prog.prog = std::move(p);
        DeviceGuard g(st->device);
        auto c = compileFor(&prog, st->nLocal, false);
        DeviceTables t = tablesFor(&prog, *c, st->device);
        prepareJit(*c, st->device);
        qk_run_stats rs{};
        for (const CompiledItem& it : c->items) {  // passes, then the materialization of SWAP relabels
            if (it.kind == CompiledItem::Block) runBlock(st, it, t, rs);
            else runIms(st, it.outs, it.ins, rs);
        }
        cuda(cudaStreamSynchronize(st->stream), "apply block");
    });
}

int qk_debug_compile_block(const qk_gate* gates, int ngates, int nLocal, char** json) {
    return guard([&] {
        std::vector<double> gtab;
        const std::vector<qkeng::Step> steps = qkeng::compileBlock(gatesFromC(gates, ngates, nLocal), nLocal, gtab);
        *json = dupText(stepsJson(steps, gtab));
    });
}

int qk_set_jit_min_qubits(int v) {
    return guard([&] { qkjit::setMinQubits(v); });
}

int qk_debug_jit_compile(const qk_gate* gates, int ngates, int nLocal, char** source) {
    return guard([&] {
        std::vector<double> gtab;
        const std::vector<qkeng::Step> steps = qkeng::compileBlock(gatesFromC(gates, ngates, nLocal), nLocal, gtab);
        std::string all;
        for (const qkeng::Step& s : steps)
            if (s.kind == qkeng::Step::Pass) {
                const std::string src = qkjit::generatePassSource(*s.pass, "qk_test_pass");
                qkjit::compileToCubin(src, "qk_test_pass");  // throws with the NVRTC log on failure
                all += src;
            }
        *source = dupText(all);
    });
}

// Specialized-kernel sources of every pass of a compiled program, in item /
// step order, separated by "//@@PASS <name>" lines, each also compiled by
// NVRTC for sm_100a (host only; tests replay them on the CPU through
// tests/host/jit_host_shim.h).
int qk_debug_jit_program(const qk_program* cp, int nLocal, char** sources) {
    return guard([&] {
        qk_program* p = const_cast<qk_program*>(cp);
        auto c = compileFor(p, nLocal, std::getenv("QK_DEBUG_FROM_BASIS") != nullptr, 1);  // specialized-kernel schedule
        std::string all;
        int k = 0;
        for (const CompiledItem& it : c->items)
            for (const qkeng::Step& s : it.steps)
                if (s.kind == qkeng::Step::Pass) {
                    const std::string name = "qk_host_pass_" + std::to_string(k++);
                    const std::string src = qkjit::generatePassSource(*s.pass, name);
                    if (!std::getenv("QK_JIT_DEBUG_NOCOMPILE"))
                        qkjit::compileToCubin(src, name);  // NVRTC (no GPU needed): throws with the log
                    all += "//@@PASS " + name + "\n" + src;
                }
        *sources = dupText(all);
    });
}

int qk_debug_compile_program(const qk_program* cp, int nLocal, char** json) {
    return guard([&] {
        qk_program* p = const_cast<qk_program*>(cp);
        auto c = compileFor(p, nLocal, std::getenv("QK_DEBUG_FROM_BASIS") != nullptr);
        std::ostringstream o;
        o << "{\"items\":[";
        for (size_t i = 0; i < c->items.size(); i++) {
            const CompiledItem& it = c->items[i];
            o << (i ? "," : "") << "{\"kind\":" << int(it.kind) << ",\"pairs\":[";
            for (size_t j = 0; j < it.outs.size(); j++) o << (j ? "," : "") << "[" << it.outs[j] << "," << it.ins[j] << "]";
            o << "]";
            if (it.kind == CompiledItem::Block) {
                std::vector<qkeng::Step> steps = it.steps;
                for (qkeng::Step& s : steps)
                    if (s.kind != qkeng::Step::Pass) s.targets.erase(s.targets.begin());
                o << ",\"block\":" << stepsJson(steps, c->gtab);
            }
            o << "}";
        }
        o << "],\"mem0\":[";
        for (size_t q = 0; q < c->mem0.size(); q++) o << (q ? "," : "") << c->mem0[q];
        o << "]}";
        *json = dupText(o.str());
    });
}

int qk_apply_gate(qk_state* st, const qk_gate* gate) {
    return qk_apply_block(st, gate, 1, st->nLocal);
}

int qk_ims_swap(qk_state* st, const int* outs, const int* ins, int s, int /*cacheLineQubits*/) {
    return guard([&] {
        for (int j = 0; j < s; j++)
            if (outs[j] < 0 || ins[j] < 0 || outs[j] >= st->nLocal || ins[j] >= st->nLocal)
                throw SimulationError("in-memory swap position outside the slice");
        DeviceGuard g(st->device);
        qk_run_stats rs{};
        runIms(st, std::vector<int>(outs, outs + s), std::vector<int>(ins, ins + s), rs);
        cuda(cudaStreamSynchronize(st->stream), "ims");
    });
}

int qk_set_dense_mode(int mode) {
    return guard([&] {
        if (mode < -1 || mode > 2) throw ConfigError("dense mode must be -1, 0, 1 or 2");
        denseModeVar().store(mode);
    });
}

int qk_set_ims_mode(int mode) {
    return guard([&] {
        if (mode < 0 || mode > 2) throw ConfigError("ims mode must be 0, 1 or 2");
        qkdev::setImsMode(mode);
    });
}

int qk_xrs_swap_local(qk_state** sl, int ns, const int* outs, const int* ins, int s, qk_xrs_stats* stats) {
    return guard([&] {
        if (ns < 1) throw SimulationError("no slices");
        const int n = sl[0]->n, R = sl[0]->R, B = sl[0]->B;
        if (ns != (1 << R)) throw SimulationError("slice count does not match the rank count");
        for (int k = 0; k < ns; k++)
            if (sl[k]->rank != k || sl[k]->n != n || sl[k]->R != R) throw SimulationError("slices are not ranks 0..2^R-1");
        quokka::SwapOp op;
        op.kind = quokka::SwapOp::CrossRank;
        for (int j = 0; j < s; j++) op.pairs.emplace_back(outs[j], ins[j]);
        const XrsPlan p = planXrs(op, n, R, B);
        if (stats)
            for (int k = 0; k < ns; k++) accountXrs(p, &stats[k]);
        enablePeers(sl, ns);
        if (p.s) runXrsLocal(sl, ns, p);
    });
}

int qk_comm_unique_id(unsigned char id[128]) {
    return guard([&] {
        ncclUniqueId u;
        nccl(ncclGetUniqueId(&u), "ncclGetUniqueId");
        static_assert(sizeof(u) == 128, "nccl id size");
        std::memcpy(id, &u, 128);
    });
}

int qk_comm_init(qk_state* st, const unsigned char id[128], int nranks, int rank) {
    return guard([&] {
        if (nranks != (1 << st->R) || rank != st->rank) throw ConfigError("communicator does not match the rank split");
        ncclUniqueId u;
        std::memcpy(&u, id, 128);
        DeviceGuard g(st->device);
        nccl(ncclCommInitRank(&st->comm, nranks, u, rank), "ncclCommInitRank");
    });
}

int qk_ipc_init(qk_state* st, const char* job, int nranks, int rank) {
    return guard([&] {
        if (nranks != (1 << st->R) || rank != st->rank) throw ConfigError("rank group does not match the rank split");
        if (st->ipc) throw SimulationError("ipc group already joined");
        const char* t = std::getenv("QK_IPC_TIMEOUT");
        DeviceGuard g(st->device);
        cuda(cudaStreamSynchronize(st->stream), "ipc init");
        st->ipc = qkipc::join(job ? job : "", nranks, rank, st->amps, st->device, t ? std::atof(t) : 600.0);
    });
}

int qk_debug_host_barrier(const char* job, int nranks, int rank, int rounds, double timeout_s) {
    return guard([&] {
        qkipc::Barrier* b = qkipc::barrierOpen(job ? job : "", nranks, rank, timeout_s);
        try {
            for (int i = 0; i < rounds; i++) qkipc::barrierWait(b);
        } catch (...) {
            qkipc::barrierClose(b);
            throw;
        }
        qkipc::barrierClose(b);
    });
}

int qk_xrs_swap(qk_state* st, const int* outs, const int* ins, int s, qk_xrs_stats* stats) {
    return guard([&] {
        quokka::SwapOp op;
        op.kind = quokka::SwapOp::CrossRank;
        for (int j = 0; j < s; j++) op.pairs.emplace_back(outs[j], ins[j]);
        const XrsPlan p = planXrs(op, st->n, st->R, st->B);
        accountXrs(p, stats);
        DeviceGuard g(st->device);
        qk_run_stats rs{};
        if (st->ipc) runXrsIpc(st, p, rs);
        else runXrsNccl(st, p, rs);
        cuda(cudaStreamSynchronize(st->stream), "xrs");
    });
}

int qk_xrs_swap_loopback(qk_state** sl, int ns, const int* outs, const int* ins, int s, qk_xrs_stats* stats) {
    return guard([&] {
        if (ns < 1 || (ns & (ns - 1))) throw SimulationError("slice count must be a power of two");
        for (int r = 0; r < ns; r++)
            if (sl[r]->rank != r || (1 << sl[r]->R) != ns) throw SimulationError("slices must be ranks 0..2^R-1");
        quokka::SwapOp op;
        op.kind = quokka::SwapOp::CrossRank;
        for (int j = 0; j < s; j++) op.pairs.emplace_back(outs[j], ins[j]);
        const XrsPlan p = planXrs(op, sl[0]->n, sl[0]->R, sl[0]->B);
        for (int r = 0; r < ns; r++) accountXrs(p, stats ? stats + r : nullptr);
        runXrsLoopback(sl, ns, p);
    });
}

int qk_xrs_plan(int n, int R, int B, int rank, const int* outs, const int* ins, int s, qk_xrs_msg* msgs, int cap,
                int* nmsgs) {
    return guard([&] {
        quokka::SwapOp op;
        op.kind = quokka::SwapOp::CrossRank;
        for (int j = 0; j < s; j++) op.pairs.emplace_back(outs[j], ins[j]);
        const XrsPlan p = planXrs(op, n, R, B);
        const std::vector<qk_xrs_msg> m = xrsMessages(p, rank);
        *nmsgs = int(m.size());
        if (int(m.size()) > cap) throw SimulationError("message buffer too small");
        std::copy(m.begin(), m.end(), msgs);
    });
}

int qk_xrs_slab_index(int n, int R, const int* outs, int s, int slab, uint64_t offset, uint64_t* index) {
    return guard([&] {
        quokka::SwapOp op;
        op.kind = quokka::SwapOp::CrossRank;
        for (int j = 0; j < s; j++) op.pairs.emplace_back(outs[j], n - R + j);
        XrsPlan p = planXrs(op, n, R, n - R);
        Index o = offset;
        for (int j = 0; j < s; j++) {  // deposit around the ascending out positions
            const int q = p.outs[size_t(j)];
            o = ((o >> q) << (q + 1)) | (o & ((Index(1) << q) - 1));
        }
        *index = o | slabBits(slab, p);
    });
}

int qk_config_parse(const char* text, qk_config* out) {
    return guard([&] {
        std::istringstream in(text);
        *out = fromConfig(quokka::parseConfig(in));
    });
}

int qk_config_finalize(qk_config* cfg) {
    return guard([&] {
        quokka::Config c = toConfig(*cfg);
        c.finalize();
        *cfg = fromConfig(c);
    });
}

int qk_config_serialize(const qk_config* cfg, char** text) {
    return guard([&] { *text = dupText(quokka::serializeConfig(toConfig(*cfg))); });
}

int qk_program_parse(const char* text, const qk_config* cfg, int lenient, qk_program** out) {
    return guard([&] {
        std::istringstream in(text);
        auto p = std::make_unique<qk_program>();
        p->prog = quokka::parseProgram(in, toConfig(*cfg), lenient != 0);
        *out = p.release();
    });
}

int qk_program_optimize(const char* circuit, const qk_config* cfg, qk_program** out) {
    return guard([&] {
        const quokka::Config c = toConfig(*cfg);
        std::istringstream in(circuit);
        const quokka::Circuit circ = quokka::parseCircuit(in, c.totalQubits);
        auto p = std::make_unique<qk_program>();
        p->prog = quokka::aioOptimize(circ, c);
        *out = p.release();
    });
}

// GPU-aware AIO configuration: the Config under which the
// reference's own optimizer (aioOptimize, unchanged) produces the Program this
// engine runs fastest.  Candidates: chunk_qbit 12 / 13 (2^12-2^13-amplitude
// tiles), fusion off / fusion_qbit 4 (dense gates the register window holds)
// / 5 (U5 tile kernel), diagonal fusion on / off.  Each candidate Program is
// compiled by this engine's scheduler and priced in slice sweeps: a pass or
// an IMS 1, a fused U5 2.7 (FP64-bound, measured 115 ms vs a 42 ms sweep at 33
// qubits), another dense / diagonal-table step 1 + its flops over the FP64
// rate, an XRS 16 B/amp (1 - 2^-S) over NVLink against 32 B/amp over HBM.
// buffer_qbit: the largest 2^B receive buffer (double-buffered: 2 x 2^B x 16
// B) that fits the HBM left beside the slice.
int qk_config_tune(const char* circuitText, int n, int R, double hbmBytes, qk_config* out, char** report) {
    return guard([&] {
        if (n < 1 || R < 0 || R >= n) throw ConfigError("bad qubit split");
        std::istringstream in(circuitText);
        const quokka::Circuit circ = quokka::parseCircuit(in, n);
        const int region = n - R;
        const double slice = 16.0 * std::ldexp(1.0, region);
        const double headroom = (hbmBytes > 0 ? hbmBytes : 180e9) - slice - 2e9;  // tables, norm, NCCL
        int B = region;
        while (B > 0 && 32.0 * std::ldexp(1.0, B) > headroom) B--;
        if (B < R) B = R;
        std::ostringstream rep;
        double best = 1e300;
        quokka::Config bestCfg;
        for (int C : {13, 12})
            for (int F : {0, 4, 5})
                for (int diag : {0, 1}) {
                    quokka::Config cfg;
                    cfg.totalQubits = n;
                    cfg.rankQubits = R;
                    cfg.chunkQubits = std::min(C, region);
                    cfg.bufferQubits = B;
                    cfg.fusionEnabled = F > 0;
                    cfg.fusionQubits = F > 0 ? std::min(F, cfg.chunkQubits) : -1;
                    cfg.diagonalFusionEnabled = diag != 0;
                    cfg.finalize();
                    qk_program prog;
                    prog.prog = quokka::aioOptimize(circ, cfg);
                    auto comp = compileFor(&prog, region, true, 1, false);
                    double cost = 0;
                    for (const CompiledItem& it : comp->items) {
                        if (it.kind == CompiledItem::Ims) cost += 1;
                        else if (it.kind == CompiledItem::Xrs)
                            cost += (16.0 / 900.0) / (32.0 / 6500.0) * (1.0 - std::ldexp(1.0, -int(it.outs.size())));
                        else
                            for (const qkeng::Step& st : it.steps) {
                                if (st.kind == qkeng::Step::Pass) cost += 1;
                                else if (st.kind == qkeng::Step::DenseGroup && st.k == 5) cost += 2.7;
                                else cost += 1 + st.flopsPerAmp * 6500e9 / 32.0 / 36.5e12;
                            }
                    }
                    rep << "chunk " << cfg.chunkQubits << " fusion " << F << " diagonal_fusion " << diag << ": "
                        << prog.prog.blockCount() << " blocks, " << comp->items.size() << " device items, cost "
                        << cost << " sweeps\n";
                    if (cost < best - 1e-9) {
                        best = cost;
                        bestCfg = cfg;
                    }
                }
        rep << "chosen: chunk " << bestCfg.chunkQubits << " fusion " << (bestCfg.fusionEnabled ? bestCfg.fusionQubits : 0)
            << " diagonal_fusion " << bestCfg.diagonalFusionEnabled << " buffer_qbit " << bestCfg.bufferQubits << "\n";
        *out = fromConfig(bestCfg);
        if (report) *report = dupText(rep.str());
    });
}

int qk_program_serialize(const qk_program* p, char** text) {
    return guard([&] { *text = dupText(quokka::serializeProgram(p->prog)); });
}

int qk_program_counts(const qk_program* p, int64_t* blocks, int64_t* sqs, int64_t* csqs, int64_t* gates) {
    return guard([&] {
        if (blocks) *blocks = int64_t(p->prog.blockCount());
        if (sqs) *sqs = int64_t(p->prog.swapCount(quokka::SwapOp::InMemory));
        if (csqs) *csqs = int64_t(p->prog.swapCount(quokka::SwapOp::CrossRank));
        if (gates) *gates = int64_t(p->prog.gateCount());
    });
}

int qk_program_final_layout(const qk_program* p, int* physToLog) {
    return guard([&] {
        for (int i = 0; i < p->prog.finalLayout.size(); i++) physToLog[i] = p->prog.finalLayout.physToLog[size_t(i)];
    });
}

int qk_program_destroy(qk_program* p) {
    return guard([&] { delete p; });
}

int qk_circuit_roundtrip(const char* text, int n, char** out) {
    return guard([&] {
        std::istringstream in(text);
        *out = dupText(quokka::serializeCircuit(quokka::parseCircuit(in, n)));
    });
}

int qk_circuit_generate(const char* kind, int n, int64_t a, uint64_t seed, char** text) {
    return guard([&] {
        const std::string k = kind;
        quokka::Circuit c;
        if (k == "qft") c = quokka::genQft(n);
        else if (k == "qaoa") c = quokka::genQaoa(n, int(a), seed);
        else if (k == "bv") c = quokka::genBv(n, seed);
        else if (k == "bvones") c = quokka::genBvAllOnes(n);
        else if (k == "random") c = quokka::genRandom(n, int(a), seed);
        else if (k == "grover") c = quokka::genGrover(n, seed, int(a));
        else if (k.rfind("bench:", 0) == 0) {
            int found = -1;
            for (int kk = 0; kk <= static_cast<int>(quokka::GateKind::RZZ); kk++)
                if (k.substr(6) == quokka::kindName(static_cast<quokka::GateKind>(kk))) found = kk;
            if (found < 0) throw ConfigError("unknown gate kind '" + k.substr(6) + "'");
            c = quokka::genGateBench(static_cast<quokka::GateKind>(found), n);
        } else {
            throw ConfigError("unknown generator '" + k + "'");
        }
        *text = dupText(quokka::serializeCircuit(c));
    });
}

// Tile-size choice for one alternative range (ChoiceTune): A first, then B,
// then A until its passes' register-width variants are all timed, then B
// once more; then the faster of B (its better run) and A's best estimate
// (A's first run with every pass replaced by its fastest variant).
// Tile-size choice for one alternative range: A (2^13 tiles) once, B (2^12)
// once, A until its passes' register-width variants are all timed, B again,
// then A twice with its tuned variants; the faster of tuned A and B (each its
// best run) is kept.  phase: which timing this run records (0 none, 1 A's
// first run, 2 B, 3 tuned A).
int chooseTileVariant(const Compiled& c, const Alternative& alt, int& phase) {
    ChoiceTune& t = *alt.tune;
    phase = 0;
    if (t.choice >= 0) return t.choice;
    if (t.msA < 0) return phase = 1, 0;
    if (t.runsB == 0) return phase = 2, 1;
    for (size_t k = alt.first; k < alt.last; k++)
        for (const qkeng::Step& s : c.items[k].steps) {
            if (!s.tune) continue;
            const int nv = 1 + int(s.alts.size());
            for (int v = 0; v < nv; v++)
                if (s.tune->needsTiming(v)) return 0;  // A still tuning its register widths
        }
    if (t.runsB < 2) return phase = 2, 1;
    if (t.runsA2 < 2) return phase = 3, 0;
    t.choice = t.msB < t.msA2 ? 1 : 0;
    if (std::getenv("QK_DEBUG_TUNE"))
        std::fprintf(stderr, "tile tune [%zu,%zu): A first run %.2f ms, A tuned %.2f ms, B (2^12) %.2f ms -> %s\n",
                     alt.first, alt.last, double(t.msA), double(t.msA2), double(t.msB), t.choice ? "B" : "A");
    return t.choice;
}

int qk_simulate(qk_state* st, const qk_program* cp, const qk_config* cfg, uint64_t initial, qk_run_stats* stats) {
    return guard([&] {
        qk_program* p = const_cast<qk_program*>(cp);
        const quokka::Config c = toConfig(*cfg);
        checkProgramAgainst(p->prog, c, st->n, st->R);
        if (c.bufferQubits != st->B) st->B = c.bufferQubits;
        DeviceGuard g(st->device);
        auto comp = compileFor(p, st->nLocal);
        const DeviceTables t = tablesFor(p, *comp, st->device);
        prepareJit(*comp, st->device);
        if (initial >= (Index(1) << st->n)) throw SimulationError("initial basis state out of range");
        qk_run_stats rs{};
        Timer timer(st);
        cudaEvent_t e0, e1;
        cuda(cudaEventCreate(&e0), "event");
        cuda(cudaEventCreate(&e1), "event");
        cuda(cudaEventRecord(e0, st->stream), "event");
        // initState (engine.cpp:18-28): folded into the first pass when the
        // program starts with one, else memset + one store.
        const bool synth = !comp->items.empty() && comp->items[0].kind == CompiledItem::Block &&
                           !comp->items[0].steps.empty() && comp->items[0].steps[0].kind == qkeng::Step::Pass;
        uint64_t basis = kNoBasis;
        Support sup;  // the run starts from |initial>: one nonzero amplitude (this rank) or none
        if (synth) {
            const bool here = (initial >> st->nLocal) == Index(st->rank);
            basis = here ? layoutIndex(initial & (st->count - 1), comp->mem0) : st->count;
            if (here) sup = Support{st->count - 1, basis, false};
            else sup.empty = true;  // the basis pass only zero-fills this slice
        } else {
            timer.time(4, [&] { setBasis(st, initial, &comp->mem0, comp->basisAmp); });
            sup.empty = (initial >> st->nLocal) != Index(st->rank);
        }
        if (!sparseStart()) sup = Support{};
        auto runItem = [&](const CompiledItem& it) {
            if (it.kind == CompiledItem::Block) {
                timer.time(0, [&] { runBlock(st, it, t, rs, basis, &timer, &sup); });
                basis = kNoBasis;
            }
            else if (it.kind == CompiledItem::Ims) timer.time(1, [&] { runIms(st, it.outs, it.ins, rs, &sup); });
            else {
                sup = Support{};  // data arrives from the other ranks
                quokka::SwapOp op;
                op.kind = quokka::SwapOp::CrossRank;
                for (size_t j = 0; j < it.outs.size(); j++) op.pairs.emplace_back(it.outs[j], it.ins[j]);
                const XrsPlan plan = planXrs(op, st->n, st->R, st->B);
                timer.time(2, [&] {
                    if (st->ipc) runXrsIpc(st, plan, rs);
                    else runXrsNccl(st, plan, rs);
                });
            }
        };
        size_t nextAlt = 0;
        for (size_t i = 0; i < comp->items.size();) {
            if (nextAlt < comp->alts.size() && comp->alts[nextAlt].first == i) {
                const Alternative& alt = comp->alts[nextAlt++];
                int v, phase;
                bool timing;
                {
                    std::lock_guard<std::mutex> lk(tuneMu());
                    v = chooseTileVariant(*comp, alt, phase);
                    timing = phase != 0;
                }
                cudaEvent_t a0 = nullptr, a1 = nullptr;
                if (timing) {
                    cuda(cudaEventCreate(&a0), "event");
                    cuda(cudaEventCreate(&a1), "event");
                    cuda(cudaEventRecord(a0, st->stream), "event");
                    rs.tuning_runs++;
                }
                if (v == 1)
                    for (const CompiledItem& it : alt.b) runItem(it);
                else
                    for (size_t k = alt.first; k < alt.last; k++) runItem(comp->items[k]);
                if (timing) {
                    float ms = 0;
                    cuda(cudaEventRecord(a1, st->stream), "event");
                    cuda(cudaEventSynchronize(a1), "event");
                    cudaEventElapsedTime(&ms, a0, a1);
                    cudaEventDestroy(a0);
                    cudaEventDestroy(a1);
                    std::lock_guard<std::mutex> lk(tuneMu());
                    if (phase == 2) {
                        alt.tune->msB = alt.tune->runsB ? std::min(alt.tune->msB, ms) : ms;
                        alt.tune->runsB++;
                    } else if (phase == 3) {
                        alt.tune->msA2 = alt.tune->runsA2 ? std::min(alt.tune->msA2, ms) : ms;
                        alt.tune->runsA2++;
                    } else {
                        alt.tune->msA = ms;
                    }
                }
                {
                    std::lock_guard<std::mutex> lk(tuneMu());
                    alt.tune->runs++;
                }
                i = alt.last;
                continue;
            }
            runItem(comp->items[i++]);
        }
        cuda(cudaEventRecord(e1, st->stream), "event");
        cuda(cudaEventSynchronize(e1), "simulate");
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        double cls[Timer::kClasses];
        timer.collect(cls);
        rs.block_ms = cls[0];
        rs.ims_ms = cls[1];
        rs.xrs_ms = cls[2];
        rs.full_pass_ms = cls[3];
        rs.init_ms = cls[4];
        rs.sparse_pass_ms = cls[5];
        rs.total_ms = ms;
        st->last = rs;
        if (stats) *stats = rs;
    });
}

int qk_simulate_local(qk_state** sl, int ns, const qk_program* cp, const qk_config* cfg, uint64_t initial,
                      qk_xrs_stats* stats) {
    return guard([&] {
        qk_program* p = const_cast<qk_program*>(cp);
        const quokka::Config c = toConfig(*cfg);
        if (ns < 1 || ns != (1 << c.rankQubits)) throw SimulationError("slice count does not match the rank count");
        for (int k = 0; k < ns; k++) {
            if (sl[k]->rank != k) throw SimulationError("slices must be ranks 0..2^R-1 in order");
            checkProgramAgainst(p->prog, c, sl[k]->n, sl[k]->R);
        }
        if (initial >= (Index(1) << c.totalQubits)) throw SimulationError("initial basis state out of range");
        auto comp = compileFor(p, sl[0]->nLocal);
        enablePeers(sl, ns);
        std::vector<DeviceTables> tabs;
        for (int k = 0; k < ns; k++) {
            sl[k]->B = c.bufferQubits;
            tabs.push_back(tablesFor(p, *comp, sl[k]->device));
            DeviceGuard g(sl[k]->device);
            prepareJit(*comp, sl[k]->device);
            setBasis(sl[k], initial, &comp->mem0, comp->basisAmp);
        }
        if (stats)
            for (int k = 0; k < ns; k++) stats[k] = qk_xrs_stats{};
        for (const CompiledItem& it : comp->items) {
            if (it.kind == CompiledItem::Xrs) {
                quokka::SwapOp op;
                op.kind = quokka::SwapOp::CrossRank;
                for (size_t j = 0; j < it.outs.size(); j++) op.pairs.emplace_back(it.outs[j], it.ins[j]);
                const XrsPlan plan = planXrs(op, c.totalQubits, c.rankQubits, c.bufferQubits);
                if (stats)
                    for (int k = 0; k < ns; k++) accountXrs(plan, &stats[k]);
                if (plan.s) runXrsLocal(sl, ns, plan);
                continue;
            }
            for (int k = 0; k < ns; k++) {
                DeviceGuard g(sl[k]->device);
                qk_run_stats rs{};
                if (it.kind == CompiledItem::Block) runBlock(sl[k], it, tabs[size_t(k)], rs);
                else runIms(sl[k], it.outs, it.ins, rs);
            }
        }
        for (int k = 0; k < ns; k++) cuda(cudaStreamSynchronize(sl[k]->stream), "simulate local");
    });
}

}  // extern "C"
