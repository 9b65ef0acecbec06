// Pass program: the compiled form of (part of) one GateBlock, shared by the
// host scheduler (schedule.cpp) and the fused gate-block kernel (block_pass.cu).
//
// One "pass" = one read + one write of the whole slice in HBM.  The kernel
// runs one CTA per tile of 2^ct amplitudes; a tile is the set of indices that
// vary over `ct` chosen physical bits (`tile_phys`, ascending) with all other
// bits fixed by the CTA index.  Inside the CTA each thread keeps 16 amplitudes
// in registers: 4 tile bits are "register slots" (0..3) and the remaining
// ct-4 tile bits are thread-index bits (slots 4..ct-1: lane bits first, then
// warp bits).  `maps[seg][slot]` = tile bit held by that slot.  Gates run
// in registers; a segment boundary is a shared-memory exchange that re-deals
// which tile bits sit in registers.
//
// The struct is passed BY VALUE as a __grid_constant__ kernel parameter
// (CUDA >= 12.1 allows 32 764 B), so every op/coefficient read is a uniform
// constant-bank load: no per-launch memcpy, graph-capturable, no races
// between slices on different streams.
#pragma once

#include <stdint.h>

namespace qkdev {

constexpr int kRegBits = 4;                 // register slots per thread
constexpr int kRegAmps = 1 << kRegBits;     // amplitudes per thread
constexpr int kMaxTileBits = 13;            // 2^13 x 16 B = 128 KiB of smem
constexpr int kMaxOps = 640;
constexpr int kMaxCoef = 900;               // complex coefficients (double2)
constexpr int kMaxSegs = 96;
constexpr int kMaxContrib = 512;            // uint16 words for fused-diagonal index maps

enum OpType : uint8_t {
    OP_MAT1 = 0,      // a = slot; coef[c..c+3] = 2x2 row-major
    OP_H,             // a = slot; butterfly without the 1/sqrt2 (folded into the flush scale)
    OP_X,             // a = slot; register swap
    OP_CX_RR,         // a = target slot, b = control slot
    OP_CX_RT,         // a = target slot, b = control thread bit
    OP_DIAG1_R,       // a = slot; coef[c], coef[c+1]
    OP_DIAG1_T,       // a = thread bit; coef[c], coef[c+1] -> per-thread scalar
    OP_DIAG2_RR,      // a = MSB slot, b = LSB slot; coef[c..c+3]
    OP_DIAG2_RT,      // a = slot, b = thread bit, k = 1 if the thread bit is the MSB; coef[c..c+3]
    OP_DIAG2_TT,      // a = MSB thread bit, b = LSB thread bit; coef[c..c+3]
    OP_CPHASE_RR,     // a, b = slots; coef[c] applied where both bits are 1
    OP_CPHASE_RT,     // a = slot, b = thread bit; coef[c]
    OP_CPHASE_TT,     // a, b = thread bits; coef[c]
    OP_DTABLE,        // fused diagonal: k targets; contrib[c16 .. c16+ct) index map; table at gtab + c
    OP_DENSE,         // fused dense 2^k (k <= 4): targets in canonical slots; matrix at gtab + c
    OP_FLUSH,         // multiply every amplitude by (per-thread scalar) * coef[c].x; reset scalar
    OP_SWAP_RR,       // a, b = slots: register permutation (SWAP when mapping relabel is not allowed)
};

struct DevOp {
    uint8_t type, a, b, k;
    uint32_t c;       // coefficient index (coef[]) or gtab offset (in double2 units)
    uint16_t c16;     // contrib[] offset for OP_DTABLE
    uint16_t pad;
};

struct PassParams {
    int32_t ct;                       // tile bits
    int32_t nsegs;
    int32_t nops;
    int32_t pad0;
    uint64_t tile_mask;               // physical tile bits (for the CTA base deposit)
    int8_t tile_phys[16];             // physical bit of tile bit j (ascending)
    uint16_t seg_end[kMaxSegs];       // ops [seg_end[s-1], seg_end[s]) run in segment s
    uint8_t map_in[kMaxSegs][16];     // mapping at segment start (load / exchange-read)
    uint8_t map_out[kMaxSegs][16];    // mapping at segment end (exchange-write / store)
    DevOp ops[kMaxOps];
    double coef[2 * kMaxCoef];        // interleaved complex coefficients
    uint16_t contrib[kMaxContrib];
};

static_assert(sizeof(PassParams) <= 32000, "kernel parameter limit");

}  // namespace qkdev
