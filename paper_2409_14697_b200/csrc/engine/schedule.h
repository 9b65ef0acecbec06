// Host-side compiler: GateBlock (physical positions) -> device steps.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "pass_program.h"
#include "quokka/gates.hpp"

namespace qkeng {

struct Step {
    enum Kind { Pass, DenseGroup, DiagTable } kind = Pass;
    std::shared_ptr<qkdev::PassParams> pass;  // Kind::Pass
    // Kind::Pass: the same pass scheduled with other register widths (2^13
    // tiles: 32, 16 or 8 amplitudes per thread); the runtime times each on its
    // first execution and keeps the fastest (`tune`, shared by copies).
    std::vector<std::shared_ptr<qkdev::PassParams>> alts;
    struct Tune {
        // rb 5 / 4 / 3, rb 5 with register stores in runs with known zeros
        // (stage_out = 0), rb 5 with half-splittable exchanges (TMA-pipelined)
        static constexpr int kMax = 5;
        static constexpr int kTimings = 2;  // each variant timed twice, round robin; its best time counts
        float ms[kMax] = {};
        int runs[kMax] = {};
        int timed[kMax] = {};
        // the variant to run next: an untimed one while any is left, else the fastest
        int choice(int n) const {  // n = 1 + alts
            for (int r = 0; r < kTimings; r++)
                for (int v = 0; v < n; v++)
                    if (timed[v] == r) return v;
            int best = 0;
            for (int v = 1; v < n; v++)
                if (ms[v] < ms[best]) best = v;
            return best;
        }
        bool needsTiming(int v) const { return timed[v] < kTimings; }
        void record(int v, float t) {
            ms[v] = timed[v] ? std::min(ms[v], t) : t;
            timed[v]++;
        }
    };
    std::shared_ptr<Tune> tune;
    // Kind::Pass: tile bits no non-diagonal gate of the pass touches, as
    // (memory bit before, memory bit after the store permutation): a bit known
    // to be fixed in the input support stays fixed (same value) in the output.
    std::vector<std::pair<int, int>> keep;
    // Kind::DenseGroup / DiagTable: matrix (or diagonal) at gtab offset `matOff`,
    // targets (j -> sub-index bit k-1-j)
    int k = 0;
    uint64_t matOff = 0;
    std::vector<int> targets;
    // algorithmic accounting: reference-formula flops per amplitude
    double flopsPerAmp = 0;
    int gates = 0;
};

// Appends device tables (fused-diagonal payloads, dense matrices) to `gtab`
// (interleaved complex) and returns the steps that apply `gates` in order to a
// slice of 2^nLocal amplitudes.  Throws SimulationError if a gate reaches a
// position >= nLocal.
// With `dest` (memory bit -> memory bit where its data should end up), the
// passes also route data toward dest with free in-tile store permutations;
// `relabel` receives the resulting move (data that started at memory bit b is
// now at relabel[b]).  tileBits > 0 overrides the tile size (QK_MAX_TILE_BITS).
// synthFirst: the first pass will synthesize its input from a basis state
// (one tile computed, the rest zero-filled), so its tile needs no coalescing
// padding with the lowest memory bits.
// interp: the passes will run on the pass interpreter (k_block_pass, slices
// below the specialization threshold): 8 amplitudes per thread (rb = 3), no
// register-width variants, so its registers never spill.
std::vector<Step> compileBlock(const std::vector<quokka::Gate>& gates, int nLocal, std::vector<double>& gtab,
                               const std::vector<int>* dest = nullptr, std::vector<int>* relabel = nullptr,
                               int tileBits = 0, bool synthFirst = false, bool interp = false);

// Support mask after pass `s` (bits of `mask` stay fixed only where the pass
// keeps them; `val` moves with them).
inline void supportAfter(const Step& s, uint64_t tileMask, uint64_t& mask, uint64_t& val) {
    uint64_t m = mask & ~tileMask, v = val & ~tileMask;
    for (const auto& [from, to] : s.keep)
        if ((mask >> from) & 1) {
            m |= uint64_t(1) << to;
            v |= ((val >> from) & 1) << to;
        }
    mask = m;
    val = v;
}

// While alive (one per compilation, this thread): passes leave the 1/sqrt2
// of their Hadamard butterflies out (no scaling multiplies) and add their
// count to *count; the run then starts from |basis> scaled by
// (1/sqrt2)^count instead (linear, so the final state is the same up to
// rounding).  Only for runs that start from a basis state.
struct DeferHScales {
    explicit DeferHScales(int* count);
    ~DeferHScales();
    DeferHScales(const DeferHScales&) = delete;
    DeferHScales& operator=(const DeferHScales&) = delete;
    int* prev;
};
inline double deferredHScale(int h) { return std::ldexp(h % 2 ? 0.70710678118654752440 : 1.0, -(h / 2)); }

// Reference-formula flops per amplitude for one gate.
double referenceFlopsPerAmp(const quokka::Gate& g);

}  // namespace qkeng
