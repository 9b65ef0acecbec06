// Host-side compiler from a GateBlock to fused-pass programs (pass_program.h).
//
// Semantics: applying the returned steps in order equals applying the
// block's gates in order to every chunk (proj/src/engine.cpp:262-281): gates
// only ever address index bits, and a tile that contains all bits a gate
// touches is closed under it, so tiling the slice by any superset of the
// chunk bits gives the same result as the reference's 2^C chunk loop.
//
// Per pass the scheduler:
//   1. picks ct tile bits = the union of the pass's gate qubits padded with the
//      lowest physical bits (coalesced 128-B+ rows);
//   2. walks the gates keeping a slot->tile-bit map; a gate that needs a qubit
//      in a register slot (1-qubit dense, CX target, dense U_k) but finds it in
//      the thread index starts a new segment = one shared-memory exchange, with
//      the next register set chosen by look-ahead over the following gates;
//   3. lowers each gate to a register op, a deferred per-thread factor
//      (diagonals touching thread-index bits: one scalar multiply per thread
//      instead of a sweep over the registers), or a relabel (SWAP never moves
//      data).
// H's 1/sqrt2 is not multiplied per gate: every H scales all amplitudes by
// the same factor, so the product is folded into one exact power-of-two (x
// 1/sqrt2) scale applied with the next full flush.
#include "schedule.h"
#include "jit.h"

#include <algorithm>
#include <array>
#include <sstream>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace qkdev {

namespace {
int envInt(const char* name, int dflt, int lo, int hi) {
    const char* v = std::getenv(name);
    if (!v) return dflt;
    const int x = std::atoi(v);
    return (x >= lo && x <= hi) ? x : dflt;
}
}  // namespace

int maxTileBits() {
    static const int v = envInt("QK_MAX_TILE_BITS", kMaxTileBits, 4, kMaxTileBits);
    return v;
}

// QK_TUNE_TILE (default 1): a gate stream is also scheduled with 2^12
// tiles (two CTAs per SM overlap one tile's loads with the other's math) and
// the runtime keeps whichever schedule ran faster.
bool tileTune() {
    static const bool v = maxTileBits() == kMaxTileBits && envInt("QK_TUNE_TILE", 1, 0, 1) != 0 &&
                          envInt("QK_TUNE", 1, 0, 1) != 0;
    return v;
}

// QK_JIT_TMA=1: specialized kernels stream the next tile through shared
// memory, so exchanges must be splittable into halves (see chooseMap).
// QK_WIDE_ACCESS (default 1): first segments hold memory bit 0 in a register
// slot so tile loads / stores are 256-bit (LDG.256 / STG.256, sm_100).
bool wideAccess() {
    static const bool v = envInt("QK_WIDE_ACCESS", 1, 0, 1) != 0;
    return v;
}

// QK_GTERMS (default 1): register-pair phases are deferred and applied with
// the slot flush of whichever of their bits is touched first.
// QK_STORE_WIDE (default 1): later segments prefer memory bit 0 in a free
// register slot (256-bit stores at the end of the pass).
bool storeWide() {
    static const bool v = envInt("QK_STORE_WIDE", 1, 0, 1) != 0;
    return v;
}

bool deferPairPhases() {
    static const bool v = envInt("QK_GTERMS", 1, 0, 1) != 0;
    return v;
}

// QK_WIDE_FORCE=1: reserve a register slot for memory bit 0 even when the
// first segment's gates could use all slots (costs an exchange, saves half
// the load instructions).  Default: only use a free slot.
bool wideLoadsForceSlot() {
    static const bool v = envInt("QK_WIDE_FORCE", 0, 0, 1) != 0;
    return v;
}

// QK_CARRY (default 1): at an exchange, pending diagonal factors are not
// applied; the per-thread accumulators are reset and the pending diagonal
// gates re-issued in the next segment's map (no per-amplitude flush).
bool carryPending() {
    static const bool v = envInt("QK_CARRY", 1, 0, 1) != 0;
    return v;
}

// QK_STAGE_DENSE=1: passes whose input is dense stage their output tiles
// through shared memory and TMA stores too (stage_out = 2; see jit.cpp).
// Off: measured on B200 at 33 qubits, QAOA 283 -> 302 ms, random 632 -> 628
// ms (the tile's register loads, not its stores, hold a dense pass back).
bool stageDense() {
    static const bool v = envInt("QK_STAGE_DENSE", 0, 0, 1) != 0;
    return v;
}

bool halfExchanges() {
    static const bool v = envInt("QK_JIT_TMA", 0, 0, 1) != 0;
    return v;
}

int regBitsFor(int ct) {
    static const int rb13 = envInt("QK_RB13", 5, 3, 5);
    static const int rb12 = envInt("QK_RB12", 4, 3, 5);
    return ct >= 13 ? rb13 : ct == 12 ? rb12 : (ct < 4 ? ct : 4);
}

// QK_RB13 unset: 2^13-amplitude passes are scheduled both ways (5 and 4
// register bits) and the runtime keeps the faster per pass.
bool tuneRegBits() {
    static const bool v = std::getenv("QK_RB13") == nullptr && envInt("QK_TUNE", 1, 0, 1) != 0;
    return v;
}

}  // namespace qkdev

namespace qkeng {

using namespace qkdev;
using quokka::Amp;
using quokka::Gate;
using quokka::GateKind;
using quokka::SimulationError;

double referenceFlopsPerAmp(const Gate& g) {
    switch (g.kind) {
        case GateKind::H:
        case GateKind::U:
        case GateKind::X:
        case GateKind::RX:
        case GateKind::RY:
            return 14;
        case GateKind::RZ:
        case GateKind::RZZ:
        case GateKind::CP:
        case GateKind::FusedDiag:
            return 6;
        case GateKind::CX:
        case GateKind::SWAP:
            return 0;
        case GateKind::FusedDense:
            return 8.0 * double(1 << g.targets.size()) - 2;
    }
    return 0;
}

namespace {

// Remapped gate qubits: tile index (< 64) or kCta + memory bit for a bit
// outside the tile (a constant of the CTA; only diagonal gates may have them).
constexpr int kCta = 64;
bool isCtaBit(int q) { return q >= kCta; }

bool denseInRegs(const Gate& g, int rb) {
    return g.kind == GateKind::FusedDense && g.targets.size() >= 2 && int(g.targets.size()) <= std::min(4, rb);
}

// 1-qubit matrices that are diagonal (e.g. U(0,0,lambda) = T) run as diagonals.
bool diagonalMatrix(const std::vector<Amp>& m) { return m.size() == 4 && m[1] == Amp(0) && m[2] == Amp(0); }

bool oneQubitDense(const Gate& g, const Gate& orig) {
    switch (g.kind) {
        case GateKind::H:
        case GateKind::X:
            return true;
        case GateKind::U:
        case GateKind::RX:
        case GateKind::RY:
            return !diagonalMatrix(quokka::gateMatrix(orig));
        case GateKind::FusedDense:
            return g.targets.size() == 1 && !diagonalMatrix(orig.payload);
        default:
            return false;
    }
}

}  // namespace

bool isDiagonalGate(const Gate& g) {
    switch (g.kind) {
        case GateKind::RZ:
        case GateKind::CP:
        case GateKind::RZZ:
        case GateKind::FusedDiag:
            return true;
        case GateKind::U:
        case GateKind::RX:
        case GateKind::RY:
            return diagonalMatrix(quokka::gateMatrix(g));
        case GateKind::FusedDense:
            return g.targets.size() == 1 && diagonalMatrix(g.payload);
        default:
            return false;
    }
}

double passCodeBudget();

thread_local int* tlDeferH = nullptr;
DeferHScales::DeferHScales(int* count) : prev(tlDeferH) { tlDeferH = count; }
DeferHScales::~DeferHScales() { tlDeferH = prev; }

namespace {

// Tile bits that must sit in register slots when `g` runs.
std::vector<int> regNeeds(const Gate& g, const Gate& orig) {
    if (oneQubitDense(g, orig) || g.kind == GateKind::CX) return {g.targets[0]};
    if (g.kind == GateKind::FusedDense && g.targets.size() > 1) return g.targets;
    return {};
}

void appendComplex(std::vector<double>& v, const std::vector<Amp>& xs) {
    for (const Amp& a : xs) {
        v.push_back(a.real());
        v.push_back(a.imag());
    }
}

Amp ratio(Amp num, Amp den) {
    if (den == Amp(0.0, 0.0)) throw SimulationError("diagonal gate with a zero entry cannot be deferred");
    return num / den;
}

class PassBuilder {
public:
    PassBuilder(const std::vector<Gate>& tg, const std::vector<Gate>& orig, const std::vector<int>& tilePhys,
                std::vector<double>& gtab, int rb = -1, bool halfX = false, bool sparseIn = false)
        : tg_(tg), orig_(orig), gtab_(gtab), ct_(int(tilePhys.size())),
          rb_(rb > 0 ? rb : regBitsFor(int(tilePhys.size()))), halfX_(halfX || halfExchanges()), sparseIn_(sparseIn) {
        tilePhys_ = tilePhys;
    }

    // Compile gates [i, ...) into one PassParams; returns the next gate index.
    size_t build(size_t i, Step& step) {
        auto P = std::make_shared<PassParams>();
        std::memset(P.get(), 0, sizeof(PassParams));
        P_ = P.get();
        P_->half_x = halfX_ ? 1 : 0;
        P_->stage_out = sparseIn_ ? 1 : stageDense() ? 2 : 0;
        P_->ct = ct_;
        P_->rb = rb_;
        for (int j = 0; j < ct_; j++) {
            P_->tile_phys[j] = int8_t(tilePhys_[size_t(j)]);
            P_->tile_mask |= uint64_t(1) << tilePhys_[size_t(j)];
        }
        nops_ = ncoef_ = ncontrib_ = ncta_ = ncterms_ = 0;
        seg_ = 0;
        hcount_ = 0;
        pendScalar_ = false;
        std::fill(pendSlot_, pendSlot_ + kMaxRegBits, false);
        flips_ = 0;
        batchReset();
        gterms_.clear();
        carry_.clear();
        pend_.clear();
        pendConst_ = Amp(1.0, 0.0);
        carryOk_ = true;
        carried_ = false;
        chooseMap(i, nullptr, wideAccess() && tilePhys_[0] == 0);
        std::memcpy(P_->map_in[0], map_, sizeof map_);

        const size_t first = i;
        double flops = 0, code = 0;
        while (i < tg_.size()) {
            if (code > passCodeBudget() && i > first) {  // NVRTC time grows super-linearly with a pass's length
                if (std::getenv("QK_DEBUG_SPLIT")) std::fprintf(stderr, "pass split at gate %zu: code %.0f\n", i, code);
                break;
            }
            // room for what is still queued: batched register ops, pair-phase
            // flushes, and one re-issue of the pending gates (tables fold into
            // <= rb + 2 ops; CTA-bit gates add up to 2 terms / coefficients each)
            const int pendCta = carryAffordable() ? pendCtaCost() : 0;
            const int queuedOps = int(regOps_.size() + gterms_.size() + 2 * carry_.size()) + (pend_.empty() ? 0 : rb_ + ct_ + 4);
            const int queuedCoef = int(4 * regOps_.size() + 17 * gterms_.size() + 8 * carry_.size()) + pendCta;
            if (kMaxOps - nops_ - queuedOps < 16 + ct_ || kMaxCoef - ncoef_ - queuedCoef - pendingCtaTerms() < 40 ||
                kMaxContrib - ncontrib_ < 48 + ct_ || kMaxSegs - seg_ < 3 || kMaxCtaFactors - ncta_ < 2 * ct_ + 4 ||
                kMaxCtaTerms - ncterms_ - pendingCtaTerms() - pendCta < 12) {
                if (std::getenv("QK_DEBUG_SPLIT"))
                    std::fprintf(stderr, "pass split at gate %zu: ops %d+%d coef %d+%d+%d cta %d terms %d+%d+%d\n", i, nops_,
                                 queuedOps, ncoef_, queuedCoef, pendingCtaTerms(), ncta_, ncterms_, pendingCtaTerms(),
                                 pendCta);
                break;
            }
            if (!satisfied(tg_[i], orig_[i])) {
                flushAll(true);
                closeSegment();
                seg_++;
                chooseMap(i, halfX_ ? &P_->xsplit[seg_] : nullptr, false, storeBit0());
                if (!halfX_) P_->xsplit[seg_] = 255;
                std::memcpy(P_->map_in[seg_], map_, sizeof map_);
                emit(OP_EXCHANGE, 0, 0, 0, uint32_t(seg_));
                relowerCarried();
            }
            lower(tg_[i], orig_[i]);
            flops += referenceFlopsPerAmp(orig_[i]);
            code += codeWork(orig_[i]);
            i++;
        }
        flushAll();
        closeSegment();
        P_->nsegs = seg_ + 1;
        P_->nops = nops_;
        P_->ncta = ncta_;
        step.kind = Step::Pass;
        step.pass = P;
        step.flopsPerAmp = flops;
        step.gates = int(i - first);
        return i;
    }

private:
    // Straight-line code a gate adds per thread, in complex multiply-adds:
    // a dense k-qubit gate is a 2^k x 2^k matvec on each of the 2^(rb-k)
    // register groups; diagonals mostly fold into phase tables.
    double codeWork(const Gate& g) const {
        const double slots = double(1 << rb_);
        if (isDiagonalGate(g)) return 0.25 * slots;
        if (g.kind == GateKind::CX || g.kind == GateKind::SWAP || g.kind == GateKind::X) return 0.0;
        const int k = g.kind == GateKind::FusedDense ? int(g.targets.size()) : 1;
        return slots * double(1 << k);
    }

    bool isReg(int slot) const { return slot < rb_; }
    // Slot holds its tile bit inverted (an X was applied as a relabel).
    int flip(int slot) const { return int((flips_ >> slot) & 1u); }

    void closeSegment() {
        P_->seg_end[seg_] = uint16_t(nops_);
        std::memcpy(P_->map_out[seg_], map_, sizeof map_);
        uint32_t xm = 0;
        for (int s = 0; s < ct_; s++)
            if (flip(s)) xm |= 1u << map_[s];
        P_->xmask_out[seg_] = uint16_t(xm);
        flips_ = 0;  // the exchange / store writes the data at its true index
    }

    bool satisfied(const Gate& g, const Gate& orig) const {
        if (denseInRegs(g, rb_)) {
            const int k = int(g.targets.size());
            for (int j = 0; j < k; j++)
                if (inv_[g.targets[size_t(j)]] != k - 1 - j) return false;
            return true;
        }
        for (int b : regNeeds(g, orig))
            if (!isReg(inv_[b])) return false;
        return true;
    }

    // Choose which tile bits occupy the register slots from gate i onward.
    // For an exchange (`split` != nullptr) one register slot keeps its tile
    // bit (tile index >= 3) across it: the exchange can then run in two
    // halves split on that bit, through a half-tile shared-memory buffer.
    // wantBit0: hold tile bit 0 (= memory bit 0) in a register slot, so each
    // thread's amplitudes pair up into 32-B neighbours (one 256-bit load each).
    // preferBit0: a later segment holds memory bit 0 in a register slot when
    // one is free, so that if it is the pass's last segment the tile is
    // stored with 256-bit stores (half the store instructions).  Only for
    // passes of a basis run that still have known zeros in their input: they
    // read almost nothing, so their stores are the memory stream (QFT-33 pass 3
    // 48.6 -> 47.6 ms); on full passes it moved QAOA-33 297 -> 312 ms.
    bool storeBit0() const { return sparseIn_ && wideAccess() && tilePhys_[0] == 0 && qkdev::storeWide(); }
    void chooseMap(size_t i, uint8_t* split = nullptr, bool wantBit0 = false, bool preferBit0 = false) {
        int prev[kMaxRegBits];
        for (int s = 0; s < rb_; s++) prev[s] = map_[s];
        int slotBit[kMaxRegBits];
        bool fixedSlot[kMaxRegBits] = {};
        std::fill(slotBit, slotBit + kMaxRegBits, -1);
        std::vector<int> regs;  // tile bits at time i
        if (i < tg_.size() && denseInRegs(tg_[i], rb_)) {
            const Gate& g = tg_[i];
            const int k = int(g.targets.size());
            for (int j = 0; j < k; j++) slotBit[k - 1 - j] = g.targets[size_t(j)];
            for (int j = 0; j < k; j++) fixedSlot[k - 1 - j] = true;
            for (int j = 0; j < k; j++) regs.push_back(g.targets[size_t(j)]);
        }
        // Look ahead: add needed bits in order of first use while they fit.
        std::vector<int> origin(static_cast<size_t>(ct_));  // current bit -> bit at time i (SWAP relabels)
        for (int b = 0; b < ct_; b++) origin[size_t(b)] = b;
        std::vector<char> inSet(static_cast<size_t>(ct_), 0);
        for (int b : regs) inSet[size_t(b)] = 1;
        for (size_t j = i; j < tg_.size() && int(regs.size()) <= rb_; j++) {
            const Gate& g = tg_[j];
            if (g.kind == GateKind::SWAP) {
                const int a = g.targets[0], b = g.targets[1];
                std::swap(origin[size_t(a)], origin[size_t(b)]);
                std::swap(inSet[size_t(a)], inSet[size_t(b)]);
                continue;
            }
            if (j > i && denseInRegs(g, rb_)) break;
            std::vector<int> need;
            for (int b : regNeeds(g, orig_[j]))
                if (!inSet[size_t(b)]) need.push_back(b);
            if (need.empty()) continue;
            if (regs.size() + need.size() > size_t(rb_)) break;
            for (int b : need) {
                inSet[size_t(b)] = 1;
                regs.push_back(origin[size_t(b)]);
            }
        }
        if (preferBit0 && !wantBit0 && int(regs.size()) < rb_ &&
            std::find(regs.begin(), regs.end(), 0) == regs.end())
            regs.push_back(0);
        if (wantBit0 && std::find(regs.begin(), regs.end(), 0) == regs.end()) {
            if (int(regs.size()) < rb_) {
                regs.push_back(0);
            } else if (wideLoadsForceSlot()) {
                std::vector<char> must(static_cast<size_t>(ct_), 0);
                if (i < tg_.size())
                    for (int b : regNeeds(tg_[i], orig_[i])) must[size_t(b)] = 1;
                for (size_t j = regs.size(); j-- > 0;)
                    if (!must[size_t(regs[j])] && std::find(slotBit, slotBit + rb_, regs[j]) == slotBit + rb_) {
                        regs[j] = 0;
                        break;
                    }
            }
        }
        // Fill with the highest remaining tile bits (keeps low bits in lanes),
        // avoiding upcoming CX controls: a thread-resident control lets a
        // pending phase on the target ride through the swap (OP_CX_PEND).
        std::vector<char> used(static_cast<size_t>(ct_), 0);
        for (int b : regs) used[size_t(b)] = 1;
        std::vector<char> ctrl(static_cast<size_t>(ct_), 0);
        for (size_t j = i; j < tg_.size() && j < i + 96; j++)
            if (tg_[j].kind == GateKind::CX && tg_[j].controls[0] < ct_) ctrl[size_t(tg_[j].controls[0])] = 1;
        for (int pass = 0; pass < 2; pass++)
            for (int b = ct_ - 1; b >= 0 && int(regs.size()) < rb_; b--)
                if (!used[size_t(b)] && (pass == 1 || !ctrl[size_t(b)])) {
                    used[size_t(b)] = 1;
                    regs.push_back(b);
                }
        // Assign register slots (canonical dense slots already fixed).
        size_t r = 0;
        auto taken = [&](int b) { return std::find(slotBit, slotBit + rb_, b) != slotBit + rb_; };
        for (int s = 0; s < rb_; s++) {
            if (slotBit[s] >= 0) continue;
            while (r < regs.size() && taken(regs[r])) r++;
            slotBit[s] = regs[r++];
        }
        if (split) {
            std::vector<char> must(static_cast<size_t>(ct_), 0);  // needed by gate i itself
            if (i < tg_.size())
                for (int b : regNeeds(tg_[i], orig_[i])) must[size_t(b)] = 1;
            int common = -1;
            for (int s = 0; s < rb_ && common < 0; s++)
                if (slotBit[s] == prev[s] && prev[s] >= 3) common = s;
            for (int s = 0; s < rb_ && common < 0; s++) {  // an old register bit moved slots: move it back
                if (prev[s] < 3 || fixedSlot[s]) continue;
                for (int s2 = 0; s2 < rb_; s2++)
                    if (slotBit[s2] == prev[s] && !fixedSlot[s2]) {
                        std::swap(slotBit[s], slotBit[s2]);
                        common = s;
                        break;
                    }
            }
            for (int s = 0; s < rb_ && common < 0; s++)  // keep an old register bit instead of a spare new one
                if (!fixedSlot[s] && prev[s] >= 3 && !taken(prev[s]) && !must[size_t(slotBit[s])]) {
                    slotBit[s] = prev[s];
                    common = s;
                }
            *split = uint8_t(common < 0 ? 255 : common);
        }
        // Thread bits ascending; lane bits 0..2 with distinct residues mod 3
        // (conflict-free swizzled exchange).
        std::vector<int> rest;
        for (int b = 0; b < ct_; b++)
            if (!taken(b)) rest.push_back(b);
        std::vector<int> lanes;
        for (int want = 0; want < 3 && !rest.empty(); want++) {
            size_t pick = rest.size();
            for (size_t q = 0; q < rest.size(); q++) {
                bool clash = false;
                for (int l : lanes) clash |= (l % 3) == (rest[q] % 3);
                if (!clash) {
                    pick = q;
                    break;
                }
            }
            if (pick == rest.size()) break;
            lanes.push_back(rest[pick]);
            rest.erase(rest.begin() + long(pick));
        }
        lanes.insert(lanes.end(), rest.begin(), rest.end());
        std::memset(map_, 0, sizeof map_);
        for (int s = 0; s < rb_; s++) map_[s] = uint8_t(slotBit[s]);
        for (size_t t = 0; t < lanes.size(); t++) map_[size_t(rb_) + t] = uint8_t(lanes[t]);
        for (int s = 0; s < ct_; s++) inv_[map_[s]] = s;
    }

    uint32_t addCoef(const std::vector<Amp>& xs) {
        const uint32_t at = uint32_t(ncoef_);
        for (const Amp& a : xs) {
            P_->coef[2 * ncoef_] = a.real();
            P_->coef[2 * ncoef_ + 1] = a.imag();
            ncoef_++;
        }
        return at;
    }

    uint32_t addTable(const std::vector<Amp>& xs) {
        const uint32_t at = uint32_t(gtab_.size() / 2);
        appendComplex(gtab_, xs);
        return at;
    }

    void emit(OpType t, int a = 0, int b = 0, int k = 0, uint32_t c = 0, uint16_t c16 = 0) {
        DevOp& o = P_->ops[nops_++];
        o.type = t;
        o.a = uint8_t(a);
        o.b = uint8_t(b);
        o.k = uint8_t(k);
        o.c = c;
        o.c16 = c16;
    }

    bool slotHasPairPhase(int slot) const {
        for (const GTerm& g : gterms_)
            if (g.a == slot || g.b == slot) return true;
        return false;
    }

    // Apply everything pending on slot `slot` (its phase R and the pair phases
    // involving it) to the amplitudes whose slot bit is 1.
    void flushSlot(int slot) {
        if (!isReg(slot)) return;
        consumeSlot(slot);
        std::vector<GTerm> mine, rest;
        for (const GTerm& g : gterms_) (g.a == slot || g.b == slot ? mine : rest).push_back(g);
        if (mine.empty()) {
            if (pendSlot_[slot]) emit(OP_FLUSH_SLOT, slot);
            pendSlot_[slot] = false;
            return;
        }
        uint32_t mask = 0;  // other slots the pair phases depend on
        for (const GTerm& g : mine) mask |= 1u << (g.a == slot ? g.b : g.a);
        // per-thread complex multiplies: one table flush over the slot's half,
        // or each pair phase on its quarter plus a plain slot flush
        const int half = 1 << (rb_ - 1), quarter = 1 << (rb_ - 2);
        const int costTable = half + (pendSlot_[slot] ? (1 << __builtin_popcount(mask)) : 0);
        const int costSplit = quarter * int(mine.size()) + (pendSlot_[slot] ? half : 0);
        if (costSplit < costTable) {
            for (const GTerm& g : mine) {
                const int lo = std::min(g.a, g.b), hi = std::max(g.a, g.b);
                emit(OP_CPHASE_RR, lo, hi, 3, addCoef({g.v}));
            }
            if (pendSlot_[slot]) emit(OP_FLUSH_SLOT, slot);
            pendSlot_[slot] = false;
            gterms_ = rest;
            return;
        }
        std::vector<int> bits;
        for (int k = 0; k < rb_; k++)
            if ((mask >> k) & 1u) bits.push_back(k);
        std::vector<Amp> tab(size_t(1) << bits.size(), Amp(1.0, 0.0));
        for (size_t idx = 0; idx < tab.size(); idx++)
            for (const GTerm& g : mine) {
                const int o = g.a == slot ? g.b : g.a;
                const size_t j = size_t(std::find(bits.begin(), bits.end(), o) - bits.begin());
                if ((idx >> j) & 1) tab[idx] *= g.v;
            }
        emit(OP_FLUSH_SLOT_G, slot, int(mask), 0, addCoef(tab));
        pendSlot_[slot] = false;
        gterms_ = rest;
    }

    // carry: an exchange follows -- pair phases (constants, known here) are
    // not applied but re-issued as diagonal gates in the next segment's map.
    void flushAll(bool carry = false) {
        if (carry && carryOk_ && carryPending() && deferPairPhases() && carryAffordable()) {
            // nothing is applied: drop the accumulators and the unemitted batch;
            // reissuePending() re-lowers every pending gate in the next map
            batchReset();
            gterms_.clear();
            bool any = pendScalar_;
            for (int s = 0; s < rb_; s++) any |= pendSlot_[s];
            if (any) emit(OP_RESET);
            pendScalar_ = false;
            std::fill(pendSlot_, pendSlot_ + kMaxRegBits, false);
            carried_ = true;
            return;
        }
        carried_ = false;
        pend_.clear();  // everything below is applied
        pendConst_ = Amp(1.0, 0.0);
        carryOk_ = true;
        emitBatch();
        if (tlDeferH) {  // the run's initial amplitude carries the normalization
            *tlDeferH += hcount_;
            hcount_ = 0;
        }
        bool any = hcount_ > 0 || pendScalar_;
        for (int s = 0; s < rb_; s++) any |= pendSlot_[s];
        uint16_t dtab = 0;  // 1 + coef index of a 2^rb pair-phase table, 0: none
        if (carry) {
            for (const GTerm& g : gterms_) {  // physical slot bits -> true tile bits
                std::vector<Amp> dl(4, Amp(1.0, 0.0));
                dl[size_t(2 * (1 ^ flip(g.a)) + (1 ^ flip(g.b)))] = g.v;
                carry_.push_back({map_[g.a], map_[g.b], dl});
            }
            gterms_.clear();
        } else if (!gterms_.empty()) {
            std::vector<Amp> D(size_t(1) << rb_, Amp(1.0, 0.0));
            for (size_t sidx = 0; sidx < D.size(); sidx++)
                for (const GTerm& g : gterms_)
                    if (((sidx >> g.a) & 1) && ((sidx >> g.b) & 1)) D[sidx] *= g.v;
            dtab = uint16_t(1 + addCoef(D));
            gterms_.clear();
            any = true;
        }
        if (!any) return;
        // (1/sqrt2)^h exactly: a power of two, times 1/sqrt2 when h is odd.
        const double root = 1.0 / std::sqrt(2.0);
        const double scale = std::ldexp(hcount_ % 2 ? root : 1.0, -(hcount_ / 2));
        emit(OP_FLUSH, 0, 0, 0, addCoef({Amp(scale, 0.0)}), dtab);
        hcount_ = 0;
        pendScalar_ = false;
        std::fill(pendSlot_, pendSlot_ + kMaxRegBits, false);
    }

    // Re-issue carried pair phases (or every pending gate) after an exchange
    // (new map, no flips).
    void relowerCarried() {
        if (carried_) {
            carried_ = false;
            carryOk_ = true;
            carry_.clear();
            reissuePending();
            return;
        }
        std::vector<Carried> c;
        c.swap(carry_);
        for (const Carried& x : c) gate2(x.a, x.b, x.d);
    }

    void scalar(const std::vector<Amp>& d, OpType t, int a = 0, int b = 0) {
        emit(t, a, b, 0, addCoef(d));
        pendScalar_ = true;
    }
    void pending(int slot, const std::vector<Amp>& r, OpType t, int b = 0) {
        emit(t, slot, b, 0, addCoef(r));
        pendSlot_[slot] = true;
    }

    // ---- diagonal batches -------------------------------------------------
    // Consecutive diagonal gates commute, so a run of them (CP / RZ / RZZ /
    // diagonal U / D_1 / D_2) is folded on the host into at most: one
    // per-thread scalar table (factors of thread-index bits), one per-slot
    // pending-phase table per register slot (factors of slot bit x thread
    // bits), and register-only factors.  Tables are indexed by the compacted
    // thread bits they depend on (<= 256 entries, L1-resident).  A 42-gate
    // controlled-phase block becomes ~7 device ops instead of 42.
    int nthr() const { return 1 << (ct_ - rb_); }

    void batchReset() {
        batchAny_ = false;
        tabP_.assign(size_t(nthr()), Amp(1.0, 0.0));
        maskP_ = 0;
        usedP_ = false;
        for (int s = 0; s < kMaxRegBits; s++) {
            tabR_[s].assign(size_t(nthr()), Amp(1.0, 0.0));
            maskR_[s] = 0;
            usedR_[s] = false;
        }
        regOps_.clear();
        ctaP_.clear();
        for (auto& v : ctaBit_) v.clear();
    }

    // ---- CTA-dependent factors (bits outside the tile) ---------------------
    struct Term {
        int b1, b2;  // memory bits (b1 < 0: unconditional)
        Amp v;
    };
    int pendingCtaTerms() const {
        size_t n = ctaP_.size();
        for (const auto& v : ctaBit_) n += v.size();
        return int(n);
    }
    static void addTerm(std::vector<Term>& to, int b1, int b2, Amp v) {
        if (v != Amp(1.0, 0.0)) to.push_back({b1, b2, v});
    }
    // Registers one factor (product of `terms`) for this tile; returns its index.
    uint32_t ctaFactor(const std::vector<Term>& terms) {
        const int f = ncta_++;
        for (const Term& t : terms) {
            CtaTerm& ct = P_->cta_terms[ncterms_++];
            ct.b1 = uint8_t(t.b1 < 0 ? 255 : t.b1);
            ct.b2 = uint8_t(t.b1 < 0 ? 255 : t.b2);
            ct.c = uint16_t(addCoef({t.v}));
        }
        P_->cta_end[f] = uint16_t(ncterms_);
        return uint32_t(f);
    }
    void emitCtaBatch() {
        if (!ctaP_.empty()) {
            emit(OP_SCAL_CTA, 0, 0, 0, ctaFactor(ctaP_));
            pendScalar_ = true;
        }
        for (int b = 0; b < ct_; b++) {
            if (ctaBit_[size_t(b)].empty()) continue;
            const int s = inv_[b];
            const uint32_t f = ctaFactor(ctaBit_[size_t(b)]);
            if (isReg(s)) {
                emit(OP_PEND_CTA, s, 0, 0, f);
                pendSlot_[s] = true;
            } else {
                emit(OP_SCAL_TCTA, 0, s - rb_, 0, f);
                pendScalar_ = true;
            }
        }
    }

    // table over thread index t: t -> f(t)
    template <class F>
    void mulP(uint32_t mask, F f) {
        for (int t = 0; t < nthr(); t++) tabP_[size_t(t)] *= f(t);
        maskP_ |= mask;
        usedP_ = batchAny_ = true;
    }
    template <class F>
    void mulR(int s, uint32_t mask, F f) {
        for (int t = 0; t < nthr(); t++) tabR_[s][size_t(t)] *= f(t);
        maskR_[s] |= mask;
        usedR_[s] = batchAny_ = true;
    }

    // compacted table over the bits of `mask` (the factor does not depend on others)
    uint32_t compactTable(const std::vector<Amp>& full, uint32_t mask) {
        std::vector<Amp> out;
        const int bits = __builtin_popcount(mask);
        for (int i = 0; i < (1 << bits); i++) {
            int t = 0, r = 0;
            for (int j = 0; j < 16; j++)
                if ((mask >> j) & 1) t |= ((i >> r++) & 1) << j;
            out.push_back(full[size_t(t)]);
        }
        return addTable(out);
    }

    static bool allOne(const std::vector<Amp>& v) {
        for (const Amp& a : v)
            if (a != Amp(1.0, 0.0)) return false;
        return true;
    }

    void emitBatch() {
        if (!batchAny_) return;
        emitCtaBatch();
        usedP_ = usedP_ && !allOne(tabP_);
        for (int s = 0; s < rb_; s++) usedR_[s] = usedR_[s] && !allOne(tabR_[s]);
        if (usedP_) {
            emit(OP_SCAL_TAB, 0, 0, 0, compactTable(tabP_, maskP_));
            P_->ops[nops_ - 1].x16 = uint16_t(maskP_);  // thread-bit mask (up to 9 bits at 512 threads)
            pendScalar_ = true;
        }
        for (int s = 0; s < rb_; s++)
            if (usedR_[s]) {
                emit(OP_PEND_TAB, s, 0, 0, compactTable(tabR_[s], maskR_[s]));
                P_->ops[nops_ - 1].x16 = uint16_t(maskR_[s]);
                pendSlot_[s] = true;
            }
        for (const auto& op : regOps_) emit(op.t, op.a, op.b, op.k, addCoef(op.coef));
        batchReset();
    }

    // ---- pending diagonal gates (carried across exchanges) -----------------
    struct PendGate {
        int q0, q1;             // logical tile bits or kCta + memory bit; q1 < 0: one-qubit
        std::vector<Amp> d;     // logical diagonal (q0 = MSB)
    };
    std::vector<PendGate> pend_;
    Amp pendConst_ = Amp(1.0, 0.0);
    bool carryOk_ = true;

    void gate1(int q, const std::vector<Amp>& d) {
        pend_.push_back({q, -1, d});
        diag1(q, d);
    }
    void gate2(int q0, int q1, const std::vector<Amp>& d) {
        pend_.push_back({q0, q1, d});
        diag2(q0, q1, d);
    }
    // Re-issuing CTA-bit gates rebuilds their per-CTA terms: carry only while
    // that stays small (else flush at the exchange as usual).
    int pendCtaCost() const {
        int c = 0;
        for (const PendGate& pg : pend_) c += (isCtaBit(pg.q0) || (pg.q1 >= 0 && isCtaBit(pg.q1))) ? 2 : 0;
        return c;
    }
    bool carryAffordable() const { return pendCtaCost() <= 64 && int(pend_.size()) <= 96; }
    bool touchesPending(int q) const {
        for (const PendGate& pg : pend_)
            if (pg.q0 == q || pg.q1 == q) return true;
        return false;
    }
    // The slot-`slot` part of every pending gate has just been applied to the
    // amplitudes (physical slot bit 1 half): what stays pending is the gate
    // restricted to physical bit 0, i.e. logical value flip(slot).
    void consumeSlot(int slot) {
        const int q = map_[slot], v = flip(slot);
        std::vector<PendGate> keep;
        for (PendGate& pg : pend_) {
            if (pg.q0 != q && pg.q1 != q) {
                keep.push_back(pg);
                continue;
            }
            if (pg.q1 < 0) {
                pendConst_ *= pg.d[size_t(v)];
                continue;
            }
            // restrict the 2-qubit diagonal: remaining one-qubit gate on the other bit
            const bool msb = pg.q0 == q;
            const int other = msb ? pg.q1 : pg.q0;
            std::vector<Amp> r(2);
            for (int x = 0; x < 2; x++) r[size_t(x)] = msb ? pg.d[size_t(2 * v + x)] : pg.d[size_t(2 * x + v)];
            if (r[0] == r[1]) pendConst_ *= r[0];
            else keep.push_back({other, -1, r});
        }
        pend_.swap(keep);
    }
    // After an exchange: the accumulators were reset; re-issue what is pending.
    void reissuePending() {
        std::vector<PendGate> p;
        p.swap(pend_);
        const Amp c = pendConst_;
        pendConst_ = Amp(1.0, 0.0);
        if (c != Amp(1.0, 0.0)) {
            batchAny_ = true;
            mulP(0, [&](int) { return c; });
            pendConst_ = c;
        }
        for (const PendGate& pg : p) {
            if (pg.q1 < 0) gate1(pg.q0, pg.d);
            else gate2(pg.q0, pg.q1, pg.d);
        }
    }

    // amplitude *= d[logical bit q].  Slot semantics are physical: a flipped
    // slot holds the logical bit inverted, so the entry pair swaps.
    void diag1(int q, std::vector<Amp> d) {
        if (isCtaBit(q)) {  // amplitude *= d[c]: d0 now, d1/d0 when the CTA bit is set
            batchAny_ = true;
            if (d[0] != Amp(1.0, 0.0)) mulP(0, [&](int) { return d[0]; });
            addTerm(ctaP_, q - kCta, q - kCta, ratio(d[1], d[0]));
            return;
        }
        const int s = inv_[q];
        if (flip(s)) std::swap(d[0], d[1]);
        if (!isReg(s)) {
            const int tb = s - rb_;
            return mulP(1u << tb, [&](int t) { return d[size_t((t >> tb) & 1)]; });
        }
        if (d[0] != Amp(1.0, 0.0)) mulP(0, [&](int) { return d[0]; });
        const Amp r = ratio(d[1], d[0]);
        mulR(s, 0, [&](int) { return r; });
    }

    // amplitude *= d[2 bit(q0) + bit(q1)] (logical bits).
    void diag2(int q0, int q1, const std::vector<Amp>& dl) {
        if (isCtaBit(q0) && isCtaBit(q1)) {  // d[2 c0 + c1] = d00 (c0? r0) (c1? r1) (c0 c1? r01)
            const int c0 = q0 - kCta, c1 = q1 - kCta;
            batchAny_ = true;
            if (dl[0] != Amp(1.0, 0.0)) mulP(0, [&](int) { return dl[0]; });
            const Amp r0 = ratio(dl[2], dl[0]), r1 = ratio(dl[1], dl[0]);
            addTerm(ctaP_, c0, c0, r0);
            addTerm(ctaP_, c1, c1, r1);
            addTerm(ctaP_, c0, c1, ratio(dl[3], dl[0] * r0 * r1));
            return;
        }
        if (isCtaBit(q0) || isCtaBit(q1)) {
            // e(x, c) with x the tile bit (logical), c the CTA bit:
            //   e(x, c) = e(0, c) * (x ? e(1, c) / e(0, c) : 1)
            const bool ctaIsMsb = isCtaBit(q0);
            const int c = (ctaIsMsb ? q0 : q1) - kCta, q = ctaIsMsb ? q1 : q0;
            auto e = [&](int x, int cv) { return ctaIsMsb ? dl[size_t(2 * cv + x)] : dl[size_t(2 * x + cv)]; };
            diag1(q, {e(0, 0), e(1, 0)});                       // the c = 0 values
            addTerm(ctaP_, c, c, ratio(e(0, 1), e(0, 0)));      // x = 0 part when c = 1
            const Amp b0 = ratio(e(1, 0), e(0, 0)), b1 = ratio(e(1, 1), e(0, 1));
            // x = 1 part when c = 1, relative to the c = 0 value already applied
            const Amp rel = ratio(b1, b0);
            if (rel != Amp(1.0, 0.0)) {
                batchAny_ = true;
                const int s = inv_[q];
                if (flip(s)) {  // physical bit = logical ^ 1: factor on physical 0 = rel * (phys ? 1/rel : 1)
                    addTerm(ctaP_, c, c, rel);
                    addTerm(ctaBit_[size_t(q)], c, c, ratio(Amp(1.0, 0.0), rel));
                } else {
                    addTerm(ctaBit_[size_t(q)], c, c, rel);
                }
            }
            return;
        }
        const int s0 = inv_[q0], s1 = inv_[q1], f0 = flip(s0), f1 = flip(s1);
        std::vector<Amp> d(4);  // physical entries
        for (int b0 = 0; b0 < 2; b0++)
            for (int b1 = 0; b1 < 2; b1++) d[size_t(2 * b0 + b1)] = dl[size_t(2 * (b0 ^ f0) + (b1 ^ f1))];
        if (isReg(s0) && isReg(s1) && deferPairPhases()) {
            // d(b0, b1) = d00 (b0 ? r0) (b1 ? r1) (b0 b1 ? g): the constant and
            // single-slot parts join the pending scalar / slot phases, the pair
            // part waits (gterms_) for the first non-diagonal op on either slot
            if (d[0] == Amp(1.0, 0.0) && d[1] == d[0] && d[2] == d[0] && d[3] == d[0]) return;
            batchAny_ = true;
            if (d[0] != Amp(1.0, 0.0)) mulP(0, [&](int) { return d[0]; });
            const Amp r0 = ratio(d[2], d[0]), r1 = ratio(d[1], d[0]);
            if (r0 != Amp(1.0, 0.0)) mulR(s0, 0, [&](int) { return r0; });
            if (r1 != Amp(1.0, 0.0)) mulR(s1, 0, [&](int) { return r1; });
            const Amp g = ratio(d[3], d[0] * r0 * r1);
            if (g != Amp(1.0, 0.0)) gterms_.push_back({s0, s1, g});
            return;
        }
        if (isReg(s0) && isReg(s1)) {
            // one non-unit entry: multiply only that quarter (CP-like)
            int nonUnit = -1, count = 0;
            for (int e = 0; e < 4; e++)
                if (d[size_t(e)] != Amp(1.0, 0.0)) {
                    nonUnit = e;
                    count++;
                }
            if (count == 0) return;
            batchAny_ = true;
            const int lo = std::min(s0, s1), hi = std::max(s0, s1);
            if (count == 1) {  // pattern over (slot lo, slot hi)
                const int b0 = nonUnit >> 1, b1 = nonUnit & 1;
                const int pat = s0 == lo ? (b0 << 1 | b1) : (b1 << 1 | b0);
                regOps_.push_back({OP_CPHASE_RR, lo, hi, pat, {d[size_t(nonUnit)]}});
            } else {
                regOps_.push_back({OP_DIAG2_RR, s0, s1, 0, d});
            }
        } else if (isReg(s0) || isReg(s1)) {
            // factor(r, t): r = register slot bit, t = thread bit
            const bool regIsMsb = isReg(s0);
            const int rs = regIsMsb ? s0 : s1, tb = (regIsMsb ? s1 : s0) - rb_;
            auto at = [&](int r, int t) { return regIsMsb ? d[size_t(2 * r + t)] : d[size_t(2 * t + r)]; };
            mulP(1u << tb, [&](int t) { return at(0, (t >> tb) & 1); });
            mulR(rs, 1u << tb, [&](int t) { return ratio(at(1, (t >> tb) & 1), at(0, (t >> tb) & 1)); });
        } else {
            const int ta = s0 - rb_, tb = s1 - rb_;
            mulP((1u << ta) | (1u << tb), [&](int t) { return d[size_t(2 * ((t >> ta) & 1) + ((t >> tb) & 1))]; });
        }
    }

    void mat1(int q, std::vector<Amp> m) {
        const int s = inv_[q];
        if (flip(s)) m = {m[3], m[2], m[1], m[0]};  // X M X
        emitBatch();
        flushSlot(s);
        emit(OP_MAT1, s, 0, 0, addCoef(m));
    }

    void lower(const Gate& g, const Gate& orig) {
        switch (g.kind) {
            case GateKind::H: {
                const int s = inv_[g.targets[0]];
                emitBatch();
                flushSlot(s);
                emit(OP_H, s);
                hcount_++;
                if (flip(s)) {  // H on a flipped slot leaves it unflipped with the |1> half negated
                    flips_ ^= 1u << s;
                    gate1(g.targets[0], {Amp(1.0, 0.0), Amp(-1.0, 0.0)});
                }
                return;
            }
            case GateKind::X:  // relabel: no data moves
                if (touchesPending(g.targets[0])) carryOk_ = false;  // pending factors would need X conjugation
                flips_ ^= 1u << inv_[g.targets[0]];
                return;
            case GateKind::U:
            case GateKind::RX:
            case GateKind::RY: {
                const std::vector<Amp> m = quokka::gateMatrix(orig);
                if (diagonalMatrix(m)) return gate1(g.targets[0], {m[0], m[3]});
                return mat1(g.targets[0], m);
            }
            case GateKind::CX: {
                // controls outside the tile are constants of the CTA (selects on its base index)
                auto ctl = [&](int q, int& idx, int& pol, int& thr, int& cta) {
                    if (isCtaBit(q)) {
                        idx = q - kCta, pol = 0, thr = 0, cta = 1;
                        return;
                    }
                    const int sl = inv_[q];
                    pol = flip(sl);  // physical control value meaning logical 1: 1 ^ pol
                    thr = isReg(sl) ? 0 : 1;
                    idx = isReg(sl) ? sl : sl - rb_;
                    cta = 0;
                };
                if (g.controls.size() == 2) {  // fused Toffoli (fuseToffolis): rename / selects, no arithmetic
                    const int t = inv_[g.targets[0]];
                    int i1, p1, t1, x1, i2, p2, t2, x2;
                    ctl(g.controls[0], i1, p1, t1, x1);
                    ctl(g.controls[1], i2, p2, t2, x2);
                    emitBatch();
                    flushSlot(t);
                    emit(OP_CCX, t, i1, t1 | p1 << 1 | t2 << 2 | p2 << 3 | x1 << 4 | x2 << 5, uint32_t(i2));
                    return;
                }
                if (isCtaBit(g.controls[0])) {
                    const int t = inv_[g.targets[0]];
                    emitBatch();
                    flushSlot(t);
                    emit(OP_CX, t, g.controls[0] - kCta, 4);
                    return;
                }
                const int t = inv_[g.targets[0]], c = inv_[g.controls[0]];
                emitBatch();
                const int pol = flip(c);  // physical control value that means logical 1 is (1 ^ pol)
                if (!isReg(c) && isReg(t) && pendSlot_[t] && !slotHasPairPhase(t)) {
                    // X_t diag(1, r) X_t = r diag(1, 1/r): carry the pending phase
                    // through the swap per thread instead of flushing 16 amplitudes
                    emit(OP_CX_PEND, t, c - rb_, pol << 1);
                    pendScalar_ = true;
                    carryOk_ = false;  // thread-conditional rewrite of the pending factors
                } else {
                    flushSlot(t);
                }
                if (isReg(c)) emit(OP_CX, t, c, pol << 1);
                else emit(OP_CX, t, c - rb_, 1 | (pol << 1));
                return;
            }
            case GateKind::SWAP: {  // relabel only (pending factors and flips stay with their slots' data)
                const int a = g.targets[0], b = g.targets[1], sa = inv_[a], sb = inv_[b];
                map_[sa] = uint8_t(b);
                map_[sb] = uint8_t(a);
                inv_[a] = sb;
                inv_[b] = sa;
                for (PendGate& pg : pend_)  // the data that was logical a is now logical b
                    for (int* q : {&pg.q0, &pg.q1}) {
                        if (*q == a) *q = b;
                        else if (*q == b) *q = a;
                    }
                return;
            }
            case GateKind::RZ:
                gate1(g.targets[0], quokka::gateDiagonal(orig));
                return;
            case GateKind::CP:
                gate2(g.controls[0], g.targets[0], quokka::gateDiagonal(orig));
                return;
            case GateKind::RZZ: {
                const std::vector<int> qs = g.qubits();
                gate2(qs[0], qs[1], quokka::gateDiagonal(orig));
                return;
            }
            case GateKind::FusedDiag: {
                const int k = int(g.targets.size());
                if (k == 1) return gate1(g.targets[0], orig.payload);
                if (k == 2) return gate2(g.targets[0], g.targets[1], orig.payload);
                const uint16_t c16 = uint16_t(ncontrib_);
                uint32_t x = 0;
                for (int s = 0; s < ct_; s++) P_->contrib[ncontrib_ + s] = 0;
                std::vector<std::pair<int, int>> cta;  // (memory bit, table-index value)
                for (int j = 0; j < k; j++) {
                    const int q = g.targets[size_t(j)];
                    if (isCtaBit(q)) {
                        cta.emplace_back(q - kCta, 1 << (k - 1 - j));
                        continue;
                    }
                    const int s = inv_[q];
                    P_->contrib[ncontrib_ + s] = uint16_t(1u << (k - 1 - j));
                    if (flip(s)) x |= 1u << (k - 1 - j);
                }
                ncontrib_ += ct_;
                P_->contrib[ncontrib_++] = uint16_t(cta.size());
                for (const auto& [b, v] : cta) {
                    P_->contrib[ncontrib_++] = uint16_t(b);
                    P_->contrib[ncontrib_++] = uint16_t(v);
                }
                emit(OP_DTABLE, 0, 0, k, addTable(orig.payload), c16);
                P_->ops[nops_ - 1].x16 = uint16_t(x);
                return;
            }
            case GateKind::FusedDense: {
                const int k = int(g.targets.size());
                if (k == 1) {
                    if (diagonalMatrix(orig.payload)) return gate1(g.targets[0], {orig.payload[0], orig.payload[3]});
                    return mat1(g.targets[0], orig.payload);
                }
                // canonical slots: sub-index bit b <-> slot b; flipped slots permute the matrix
                const uint32_t f = flips_ & ((1u << k) - 1);
                const size_t dim = size_t(1) << k;
                std::vector<Amp> m(dim * dim);
                for (size_t r = 0; r < dim; r++)
                    for (size_t c = 0; c < dim; c++) m[r * dim + c] = orig.payload[(r ^ f) * dim + (c ^ f)];
                emitBatch();
                for (int s = 0; s < k; s++) flushSlot(s);
                emit(OP_DENSE, 0, 0, k, addTable(m));
                return;
            }
        }
    }

    const std::vector<Gate>& tg_;
    const std::vector<Gate>& orig_;
    std::vector<double>& gtab_;
    std::vector<int> tilePhys_;
    int ct_, rb_;
    bool halfX_;
    bool sparseIn_;  // the pass's input has known zeros (a basis run before every bit was touched)
    PassParams* P_ = nullptr;
    int nops_ = 0, ncoef_ = 0, ncontrib_ = 0, seg_ = 0, hcount_ = 0;
    bool pendScalar_ = false;
    bool pendSlot_[kMaxRegBits] = {};
    // current diagonal batch
    struct RegOp {
        OpType t;
        int a, b, k;
        std::vector<Amp> coef;
    };
    bool batchAny_ = false, usedP_ = false;
    std::vector<Amp> tabP_;
    uint32_t maskP_ = 0;
    std::vector<Amp> tabR_[kMaxRegBits];
    uint32_t maskR_[kMaxRegBits] = {};
    bool usedR_[kMaxRegBits] = {};
    std::vector<RegOp> regOps_;
    struct GTerm {
        int a, b;  // physical register slots: amplitudes with both slot bits 1 get v
        Amp v;
    };
    std::vector<GTerm> gterms_;
    struct Carried {
        int a, b;              // true tile bits
        std::vector<Amp> d;    // 4-entry diagonal, first bit = MSB
    };
    std::vector<Carried> carry_;
    bool carried_ = false;
    std::vector<Term> ctaP_;            // CTA-dependent factor of every amplitude (this batch)
    std::vector<Term> ctaBit_[16];      // ... of the amplitudes whose tile bit b is 1
    int ncta_ = 0, ncterms_ = 0;
    uint32_t flips_ = 0;  // slots (register and thread) holding an inverted bit
    uint8_t map_[16] = {};
    int inv_[16] = {};
};

Gate remapQubits(const Gate& g, const int* tileOf) {
    Gate t;
    t.kind = g.kind;
    t.id = g.id;
    for (int q : g.targets) t.targets.push_back(tileOf[q] >= 0 ? tileOf[q] : kCta + q);
    for (int q : g.controls) t.controls.push_back(tileOf[q] >= 0 ? tileOf[q] : kCta + q);
    return t;
}

void compileGroup(const std::vector<Gate>& gates, uint64_t used, int ct, int nLocal, std::vector<double>& gtab,
                  std::vector<Step>& out, int rb = -1, bool halfX = false, bool sparseIn = false) {
    // Tile bits: every bit the group touches, padded with the lowest others.
    uint64_t tile = used;
    for (int b = 0; b < nLocal && __builtin_popcountll(tile) < ct; b++) tile |= uint64_t(1) << b;
    std::vector<int> phys;
    int tileOf[64];
    std::fill(tileOf, tileOf + 64, -1);
    for (int b = 0; b < nLocal; b++)
        if ((tile >> b) & 1) {
            tileOf[b] = int(phys.size());
            phys.push_back(b);
        }
    std::vector<Gate> tg;
    for (const Gate& g : gates) tg.push_back(remapQubits(g, tileOf));
    PassBuilder pb(tg, gates, phys, gtab, rb, halfX, sparseIn);
    size_t i = 0;
    while (i < gates.size()) {
        Step st;
        i = pb.build(i, st);
        out.push_back(std::move(st));
    }
}

}  // namespace

// QK_PASS_WORK (default 3000): most reference-formula flops per amplitude
// one pass may carry.  NVRTC's time on a straight-line
// pass grows super-linearly with its length (QFT-33's ~1300-flop passes
// compile in ~1 s, a 150-gate U3 stream at n = 13 took minutes); a pass
// this heavy is FP64-bound, so the extra HBM sweep of a cut costs < 10 %.
double passWorkBudget() {
    static const double v = envInt("QK_PASS_WORK", 3000, 50, 1 << 30);
    return v;
}
// QK_PASS_CODE (default 4096): most complex multiply-adds of straight-line
// code per thread in one pass (PassBuilder::codeWork); the pass is cut there.
double passCodeBudget() {
    static const double v = envInt("QK_PASS_CODE", 4096, 64, 1 << 30);
    return v;
}

// Pass cost model of the DP (units: one HBM sweep of the slice).  Row
// penalty by the number L of contiguous lowest memory bits in the tile
// (QK_ROW_PEN="p0,p1,p2,p3", default 1.0,0.6,0.3,0) and the cost of each
// extra segment (QK_XCHG_COST, default 0).  A steeper row penalty
// (1.7,1.0,0.4,0.1) with 0.2 per exchange was measured on B200 at 33 qubits
// (profiles/r2_dp_model_ab.txt): QFT 0.153 -> 0.161 s, QAOA / random / Grover
// within 1 %, BV unchanged (its L = 0 pass has no cheaper cut) -- kept as
// knobs, not defaults.
const double* rowPenalty() {
    static const std::vector<double> v = [] {
        std::vector<double> p = {1.0, 0.6, 0.3, 0.0};
        if (const char* e = std::getenv("QK_ROW_PEN")) {
            std::istringstream in(e);
            std::string tok;
            for (size_t i = 0; i < p.size() && std::getline(in, tok, ','); i++) p[i] = std::atof(tok.c_str());
        }
        return p;
    }();
    return v.data();
}
double exchangeCost() {
    static const double v = [] {
        const char* e = std::getenv("QK_XCHG_COST");
        return e ? std::atof(e) : 0.0;
    }();
    return v;
}

int lowTileBits() {
    static const int v = envInt("QK_TILE_LOW", 3, 0, 8);
    return v;
}

// Support-aware pricing of runs from a basis state (QK_SPARSE_DP, default 1):
// a pass whose output support is still partial reads and writes only that
// support (sparse loads, deferred zeros), so it costs its support fraction of
// a sweep; the pass that first fills the slice writes it all and reads only
// its input support.  Work (reference flops/amp) is priced at QK_DP_FLOP
// sweeps per 10^5 flops (default 250: a 14-flop butterfly level ~ 0.035 of a
// sweep, as the filling passes measure) on the amplitudes it touches, so the
// DP moves gates into the cheap sparse passes and leaves the full-output pass
// as little arithmetic as the tile allows (QFT-33: 13 + 11 + 9 -> 2 + 13 + 13
// + 5 H levels, the last pass without an exchange; sweep 25 / 60 / 120 / 250
// in profiles/r2_families_ab.txt).  QK_SPARSE_DP=0 restores the
// support-blind model.
// QK_TIGHT_SUPPORT (default 1): a pass frees only the tile bits its
// non-diagonal gates touch; padding bits of a run from a basis state stay
// known (Step::keep), so later passes read and write less.
bool tightSupport() {
    static const bool v = envInt("QK_TIGHT_SUPPORT", 1, 0, 1) != 0;
    return v;
}

bool sparseDp() {
    static const bool v = envInt("QK_SPARSE_DP", 1, 0, 1) != 0;
    return v;
}
double sparsePen0() {
    static const double v = envInt("QK_SPARSE_PEN0", 8, 0, 1000);
    return v;
}
double dpFlopWeight() {
    static const double v = envInt("QK_DP_FLOP", 250, 0, 100000) * 1e-5;
    return v;
}

// QK_CTA_CONTROLS (default 1): CX / CCX controls may lie outside the tile
// (constants of the CTA, applied as selects on its base index), so a gate of
// the X family needs only its target in the tile: Grover's AND chain and
// BV's oracle fit many more gates per pass.
bool ctaControls() {
    static const bool v = envInt("QK_CTA_CONTROLS", 1, 0, 1) != 0;
    return v;
}
// Memory bits a gate needs inside a pass's tile.
uint64_t tileMaskOf(const Gate& g) {
    if (isDiagonalGate(g)) return 0;
    if (g.kind == GateKind::CX && ctaControls()) return uint64_t(1) << g.targets[0];
    return g.depMask();
}

// QK_FUSE_CCX (default 1): a run of 1-qubit gates and CX on three qubits
// whose product is exactly a Toffoli (entries within 1e-12 of the
// permutation: the 15-gate H / T / CX decomposition Grover's AND chain uses)
// is applied as one CCX -- a register rename or a select, no arithmetic --
// instead of two butterflies, seven phases and six CX.  Gates on other qubits
// that sit between them commute with the run (disjoint qubits) and keep
// their order.
bool fuseCcx() {
    static const bool v = envInt("QK_FUSE_CCX", 1, 0, 1) != 0;
    return v;
}

namespace {
using Mat8 = std::array<Amp, 64>;  // row-major over 3 local bits

bool windowGate(const Gate& g) {
    switch (g.kind) {
        case GateKind::H:
        case GateKind::U:
        case GateKind::X:
        case GateKind::RX:
        case GateKind::RY:
        case GateKind::RZ:
            return g.targets.size() == 1 && g.controls.empty();
        case GateKind::CX:
            return g.targets.size() == 1 && g.controls.size() == 1;
        default:
            return false;
    }
}

void applyToMat(Mat8& M, const Gate& g, const int* local) {
    if (g.kind == GateKind::CX) {
        const int c = local[0], t = local[1];
        for (int r = 0; r < 8; r++)
            if (((r >> c) & 1) && !((r >> t) & 1))
                for (int col = 0; col < 8; col++) std::swap(M[size_t(r * 8 + col)], M[size_t((r | (1 << t)) * 8 + col)]);
        return;
    }
    const std::vector<Amp> m = quokka::gateMatrix(g);
    const int j = local[0];
    for (int r = 0; r < 8; r++) {
        if ((r >> j) & 1) continue;
        const int r1 = r | (1 << j);
        for (int col = 0; col < 8; col++) {
            const Amp x = M[size_t(r * 8 + col)], y = M[size_t(r1 * 8 + col)];
            M[size_t(r * 8 + col)] = m[0] * x + m[1] * y;
            M[size_t(r1 * 8 + col)] = m[2] * x + m[3] * y;
        }
    }
}

// Local target bit of the Toffoli M equals, else -1.
int toffoliTarget(const Mat8& M) {
    for (int t = 0; t < 3; t++) {
        const int c1 = (t + 1) % 3, c2 = (t + 2) % 3;
        bool ok = true;
        for (int r = 0; r < 8 && ok; r++) {
            const int want = (((r >> c1) & 1) && ((r >> c2) & 1)) ? (r ^ (1 << t)) : r;
            for (int col = 0; col < 8 && ok; col++)
                ok = std::abs(M[size_t(want * 8 + col)] - Amp(col == r ? 1.0 : 0.0, 0.0)) < 1e-12;
        }
        if (ok) return t;
    }
    return -1;
}
}  // namespace

std::vector<Gate> fuseToffolis(const std::vector<Gate>& gates) {
    const size_t n = gates.size();
    std::vector<char> drop(n, 0);
    std::vector<Gate> at(n);  // replacement placed at a window's last gate
    std::vector<char> has(n, 0);
    for (size_t i = 0; i < n; i++) {
        if (drop[i] || has[i] || gates[i].kind != GateKind::H) continue;
        std::vector<int> Q;
        uint64_t skipped = 0;  // qubits of gates skipped over (they must stay outside Q)
        Mat8 M{};
        for (int r = 0; r < 8; r++) M[size_t(r * 9)] = Amp(1.0, 0.0);
        std::vector<size_t> taken;
        for (size_t j = i; j < n && j < i + 64 && taken.size() < 32; j++) {
            if (drop[j] || has[j]) break;
            const Gate& g = gates[j];
            const std::vector<int> qs = g.qubits();
            bool anyIn = false;
            for (int q : qs) anyIn |= std::find(Q.begin(), Q.end(), q) != Q.end();
            if (!anyIn && j != i) {  // disjoint: commutes with the window, stays where it is
                for (int q : qs) skipped |= uint64_t(1) << q;
                continue;
            }
            if (!windowGate(g)) break;
            bool fits = true;
            std::vector<int> add;
            for (int q : qs)
                if (std::find(Q.begin(), Q.end(), q) == Q.end()) {
                    if ((skipped >> q) & 1) fits = false;
                    add.push_back(q);
                }
            if (!fits || Q.size() + add.size() > 3) break;
            Q.insert(Q.end(), add.begin(), add.end());
            int local[2];
            for (size_t k = 0; k < qs.size(); k++)
                local[k] = int(std::find(Q.begin(), Q.end(), qs[k]) - Q.begin());
            applyToMat(M, g, local);
            taken.push_back(j);
            if (Q.size() == 3 && taken.size() >= 3) {
                const int t = toffoliTarget(M);
                if (t >= 0) {
                    Gate f = gates[i];
                    f.kind = GateKind::CX;
                    f.targets = {Q[size_t(t)]};
                    f.controls = {Q[size_t((t + 1) % 3)], Q[size_t((t + 2) % 3)]};
                    f.params.clear();
                    f.payload.clear();
                    f.constituents.clear();
                    for (size_t k : taken) drop[k] = 1;
                    drop[j] = 0;
                    at[j] = f;
                    has[j] = 1;
                    break;
                }
            }
        }
    }
    std::vector<Gate> out;
    out.reserve(n);
    for (size_t k = 0; k < n; k++) {
        if (has[k]) out.push_back(at[k]);
        else if (!drop[k]) out.push_back(gates[k]);
    }
    return out;
}

// Gates (memory-bit positions, program order) -> steps.  Consecutive gates
// share a pass while the bits their NON-diagonal gates touch fit in one tile
// (padded with the lowest memory bits for coalesced rows): diagonal gates
// never constrain the tile (bits outside it are constants of the CTA), so
// runs of controlled-phase / RZ / RZZ / D_k gates ride along with whichever
// pass is open.  Gate order is never changed; the cut points minimize the
// estimated HBM cost.
// Store permutation of a pass: the data of tile bit j is written to tile bit
// sigma[j] (map_out of the last segment relabelled; no extra traffic).
void applyStorePermutation(PassParams& P, const std::vector<int>& sigma) {
    const int last = P.nsegs - 1;
    for (int s = 0; s < P.ct; s++) P.map_out[last][s] = uint8_t(sigma[P.map_out[last][s]]);
    uint32_t xm = 0;
    for (int j = 0; j < P.ct; j++)
        if ((P.xmask_out[last] >> j) & 1) xm |= 1u << sigma[size_t(j)];
    P.xmask_out[last] = uint16_t(xm);
}

std::vector<Step> compileBlock(const std::vector<Gate>& gates, int nLocal, std::vector<double>& gtab,
                               const std::vector<int>* dest, std::vector<int>* relabel, int tileBits,
                               bool synthFirst, bool interp) {
    std::vector<Step> steps;
    // Routing (dest given): memory bit b's data should end at memory bit
    // dest[b].  Each pass stores its tile with the permutation that puts every
    // tile bit whose destination lies in the tile where it belongs, so the
    // materialization after the stream shrinks or vanishes.  R[b] = memory bit
    // that now holds the data that started at b; later gates are relabelled.
    std::vector<int> R(static_cast<size_t>(nLocal)), Rinv(static_cast<size_t>(nLocal));
    for (int b = 0; b < nLocal; b++) R[size_t(b)] = Rinv[size_t(b)] = b;
    auto relabelGate = [&](const Gate& g) {
        Gate m = g;
        for (int& q : m.targets) q = R[size_t(q)];
        for (int& q : m.controls) q = R[size_t(q)];
        return m;
    };
    auto route = [&](size_t firstStep) {
        if (!dest) return;
        for (size_t k = steps.size(); k-- > firstStep;) {
            if (steps[k].kind != Step::Pass) continue;
            PassParams& P = *steps[k].pass;
            const int ct = P.ct;
            std::vector<int> where(static_cast<size_t>(nLocal), -1);  // memory bit -> tile index
            for (int j = 0; j < ct; j++) where[size_t(P.tile_phys[j])] = j;
            std::vector<int> sigma(static_cast<size_t>(ct), -1);
            std::vector<char> taken(static_cast<size_t>(ct), 0);
            // Memory bits 0..2 keep their data: the store's lane bits write
            // them (128-B coalesced rows), whatever the routing would like.
            auto pinned = [&](int j) { return P.tile_phys[j] < 3; };
            for (int j = 0; j < ct; j++)
                if (pinned(j)) sigma[size_t(j)] = j, taken[size_t(j)] = 1;
            for (int j = 0; j < ct; j++) {
                if (pinned(j)) continue;
                const int d = where[size_t((*dest)[size_t(Rinv[size_t(P.tile_phys[j])])])];
                if (d >= 0 && !taken[size_t(d)]) sigma[size_t(j)] = d, taken[size_t(d)] = 1;
            }
            for (int j = 0; j < ct; j++)  // the rest: stay put where free, else any free slot
                if (sigma[size_t(j)] < 0 && !taken[size_t(j)]) sigma[size_t(j)] = j, taken[size_t(j)] = 1;
            int free = 0;
            for (int j = 0; j < ct; j++)
                if (sigma[size_t(j)] < 0) {
                    while (taken[size_t(free)]) free++;
                    sigma[size_t(j)] = free;
                    taken[size_t(free)] = 1;
                }
            applyStorePermutation(P, sigma);
            for (auto& a : steps[k].alts) applyStorePermutation(*a, sigma);  // same tile, same sigma
            for (auto& kp : steps[k].keep) kp.second = P.tile_phys[sigma[size_t(where[size_t(kp.second)])]];
            std::vector<int> moved(static_cast<size_t>(nLocal));
            for (int b = 0; b < nLocal; b++) moved[size_t(b)] = b;
            for (int j = 0; j < ct; j++) moved[size_t(P.tile_phys[j])] = P.tile_phys[sigma[size_t(j)]];
            for (int b = 0; b < nLocal; b++) R[size_t(b)] = moved[size_t(R[size_t(b)])];
            for (int b = 0; b < nLocal; b++) Rinv[size_t(R[size_t(b)])] = b;
            return;  // the group's last pass only
        }
    };
    for (const Gate& g : gates)
        for (int q : g.qubits())
            if (q < 0 || q >= nLocal)
                throw SimulationError("gate " + std::to_string(g.id) + " reaches outside the local slice");

    auto denseStep = [&](const std::vector<Amp>& m, const std::vector<int>& targets, double flops) {
        Step s;
        s.kind = Step::DenseGroup;
        s.k = int(targets.size());
        s.matOff = gtab.size() / 2;
        appendComplex(gtab, m);
        s.targets = targets;
        s.flopsPerAmp = flops;
        s.gates = 1;
        if (s.k == 5) s.tune = std::make_shared<Step::Tune>();  // DFMA / DMMA tile kernels
        steps.push_back(std::move(s));
    };

    std::vector<Gate> fusedGates;
    if (fuseCcx() && nLocal >= 4) {
        fusedGates = fuseToffolis(gates);
        if (fusedGates.size() != gates.size())
            return compileBlock(fusedGates, nLocal, gtab, dest, relabel, tileBits, synthFirst, interp);
    }
    if (relabel) *relabel = R;  // identity unless passes route data (below)
    if (nLocal < 4) {  // too small for a register tile: every gate as a dense group
        for (const Gate& g : gates) denseStep(quokka::gateMatrix(g), g.qubits(), referenceFlopsPerAmp(g));
        return steps;
    }
    const int ct = std::min(tileBits > 0 ? tileBits : maxTileBits(), nLocal);
    const int rb = interp ? std::min(ct, 3) : regBitsFor(ct);
    if (interp && ct > 12) return compileBlock(gates, nLocal, gtab, dest, relabel, 12, synthFirst, true);
    // Cut each run of gates (between wide dense steps) into passes by dynamic
    // programming over cut points.  A pass costs one HBM round trip, more when
    // its tile cannot start with >= 3 contiguous low memory bits (rows under
    // 128 B; measured ~1.7x slower at 16-32 B rows).
    auto passCost = [&](uint64_t used) {
        uint64_t tile = used;
        for (int b = 0; b < nLocal && __builtin_popcountll(tile) < ct; b++) tile |= uint64_t(1) << b;
        int L = 0;
        while (L < ct && ((tile >> L) & 1)) L++;
        const double* pen = rowPenalty();
        double c = 1.0 + pen[std::min(L, lowTileBits())];
        // exchanges: the register window holds rb of the tile's bits, so a
        // pass whose non-diagonal gates touch u bits needs >= ceil(u / rb)
        // segments; each extra one is a shared-memory round trip of the tile
        const int u = __builtin_popcountll(used);
        c += exchangeCost() * double(std::max(0, (u + rb - 1) / rb - 1));
        return c;
    };
    // support of a run from a basis state, as the runtime will track it: every
    // pass frees its tile bits, every dense step its targets
    uint64_t sparseMask = synthFirst ? (nLocal >= 64 ? ~uint64_t(0) : (uint64_t(1) << nLocal) - 1) : 0;
    std::vector<Gate> run;
    auto cutRun = [&] {
        const size_t m = run.size();
        if (!m) return;
        const bool synthRun = synthFirst && steps.empty();
        std::vector<uint64_t> mask(m);
        for (size_t k = 0; k < m; k++) mask[k] = tileMaskOf(run[k]);
        std::vector<double> work(m);  // reference-formula flops/amp: bounds a pass's straight-line code
        for (size_t k = 0; k < m; k++) work[k] = referenceFlopsPerAmp(run[k]);
        // support-aware model: free[k] = bits the support spans before gate k
        // (the run's fixed bits minus every bit a non-diagonal gate touched;
        // earlier passes' padding bits are not counted)
        const bool sparseModel = sparseDp() && sparseMask != 0;
        const uint64_t all = nLocal >= 64 ? ~uint64_t(0) : (uint64_t(1) << nLocal) - 1;
        std::vector<uint64_t> freeAt(m + 1, all & ~sparseMask);
        for (size_t k = 0; k < m; k++) freeAt[k + 1] = freeAt[k] | mask[k];
        auto sparseCost = [&](size_t j, uint64_t used, double w) {
            uint64_t tile = used;
            for (int b = 0; b < nLocal && __builtin_popcountll(tile) < ct; b++) tile |= uint64_t(1) << b;
            int L = 0;
            while (L < ct && ((tile >> L) & 1)) L++;
            const double pen = rowPenalty()[std::min(L, lowTileBits())];
            const double fin = std::ldexp(1.0, __builtin_popcountll(freeAt[j]) - nLocal);
            const double fout = std::ldexp(1.0, __builtin_popcountll(freeAt[j] | tile) - nLocal);
            const double comp = dpFlopWeight() * w;
            // deferred zeros: support in, support out.  A partial pass whose tile
            // has no memory bit 0 writes 16-B fragments (a TMA box one amplitude
            // wide): QFT-30's middle pass took ~3x its 32-B-row time, so L = 0
            // costs QK_SPARSE_PEN0 (default 8) there
            if (fout < 1.0) return fout * (1.0 + (L == 0 ? std::max(pen, sparsePen0()) : pen) + comp);
            return 0.5 * (1.0 + pen) * (1.0 + fin) + comp;      // every tile written, support read
        };
        std::vector<double> best(m + 1, 1e300);
        std::vector<size_t> from(m + 1, 0);
        best[0] = 0;
        for (size_t i = 1; i <= m; i++) {
            uint64_t used = 0;
            double w = 0;
            for (size_t j = i; j-- > 0;) {
                used |= mask[j];
                w += work[j];
                if (__builtin_popcountll(used) > ct) break;
                if (w > passWorkBudget() && j + 1 < i) break;
                const double c = best[j] + (sparseModel           ? sparseCost(j, used, w)
                                            : (synthRun && j == 0) ? 1.0
                                                                   : passCost(used));
                if (c < best[i] - 1e-9) {
                    best[i] = c;
                    from[i] = j;
                }
            }
        }
        std::vector<size_t> cuts;
        for (size_t i = m; i > 0; i = from[i]) cuts.push_back(from[i]);
        std::reverse(cuts.begin(), cuts.end());
        cuts.push_back(m);
        for (size_t c = 0; c + 1 < cuts.size(); c++) {
            std::vector<Gate> group;
            uint64_t used = 0;
            for (size_t k = cuts[c]; k < cuts[c + 1]; k++) {
                group.push_back(relabelGate(run[k]));
                used |= tileMaskOf(group.back());
            }
            const size_t first = steps.size();
            // a run from a basis state: the support grows by each pass's tile
            const bool sparseIn = sparseMask != 0;
            compileGroup(group, used, ct, nLocal, gtab, steps, interp ? rb : -1, false, sparseIn);
            for (size_t k = first; k < steps.size(); k++)
                if (steps[k].kind == Step::Pass && tightSupport())
                    for (int j = 0; j < steps[k].pass->ct; j++) {
                        const int b = steps[k].pass->tile_phys[j];
                        if (!((used >> b) & 1)) steps[k].keep.emplace_back(b, b);
                    }
            if (!interp && ct == 13 && tuneRegBits() && steps.size() == first + 1 && steps[first].kind == Step::Pass) {
                // the variants apply the same gates: their deferred H are not counted again
                int variantH = 0;
                int* const countH = tlDeferH;
                if (countH) tlDeferH = &variantH;
                for (int rbAlt : {4, 3}) {  // 16 and 8 amplitudes per thread (512 / 1024 threads)
                    std::vector<Step> alt;
                    compileGroup(group, used, ct, nLocal, gtab, alt, rbAlt, false, sparseIn);
                    if (alt.size() == 1 && alt[0].kind == Step::Pass) steps[first].alts.push_back(alt[0].pass);
                }
                if (qkjit::stagedPass(*steps[first].pass)) {  // register stores instead of staged TMA stores
                    auto p = std::make_shared<qkdev::PassParams>(*steps[first].pass);
                    p->stage_out = 0;
                    steps[first].alts.push_back(p);
                }
                if (!halfExchanges()) {  // 32 per thread, half-splittable exchanges: the TMA-pipelined kernel
                    std::vector<Step> alt;
                    compileGroup(group, used, ct, nLocal, gtab, alt, 5, true, sparseIn);
                    if (alt.size() == 1 && alt[0].kind == Step::Pass) steps[first].alts.push_back(alt[0].pass);
                }
                tlDeferH = countH;
                if (steps[first].alts.size() >= size_t(Step::Tune::kMax)) steps[first].alts.resize(Step::Tune::kMax - 1);
                if (!steps[first].alts.empty()) steps[first].tune = std::make_shared<Step::Tune>();
            }
            route(first);
            for (size_t k = first; k < steps.size(); k++)
                if (steps[k].kind == Step::Pass) {
                    uint64_t v = 0;
                    supportAfter(steps[k], steps[k].pass->tile_mask, sparseMask, v);
                }
        }
        run.clear();
    };
    for (const Gate& g : gates) {
        if (g.kind == GateKind::FusedDense && g.targets.size() > size_t(std::min(4, rb)) && !isDiagonalGate(g)) {
            if (g.targets.size() > size_t(kMaxTileBits))
                throw SimulationError("fused dense gate " + std::to_string(g.id) + " wider than 13 qubits");
            cutRun();
            const Gate m = relabelGate(g);
            denseStep(m.payload, m.targets, referenceFlopsPerAmp(m));
            for (int q : m.targets) sparseMask &= ~(uint64_t(1) << q);
            continue;
        }
        run.push_back(g);
    }
    cutRun();
    if (relabel) *relabel = R;
    return steps;
}

}  // namespace qkeng
