// Pass program: the compiled form of (part of) one GateBlock, shared by the
// host scheduler (schedule.cpp) and the fused gate-block kernel (block_pass.cu).
//
// One "pass" = one read + one write of the whole slice in HBM.  The kernel
// runs one CTA per tile of 2^ct amplitudes; a tile is the set of indices that
// vary over `ct` chosen physical bits (`tile_phys`, ascending) with all other
// bits fixed by the CTA index.  Inside the CTA each thread keeps 2^rb
// amplitudes in registers: rb tile bits are "register slots" (0..rb-1) and the
// remaining ct-rb tile bits are thread-index bits (slots rb..ct-1: lane bits
// first, then warp bits).  `map_*[seg][slot]` = tile bit held by that slot.
// Gates run in registers; a segment boundary is a shared-memory exchange that
// re-deals which tile bits sit in registers.  X gates never move data: the
// scheduler tracks which slots hold a flipped bit and `xmask_out` corrects the
// exchange / store addresses (register renaming inside the op loop would make
// ptxas copy the whole register array every iteration).
//
// Diagonal factors that depend on thread-index bits are not applied to the
// registers when they occur: each thread accumulates them into one scalar P
// and one "pending phase" R[a] per register slot (applied to the amplitudes
// whose slot-a bit is 1).  They are flushed into the registers only when a
// non-diagonal op touches slot a, or at an exchange / the final store.
//
// The struct is passed BY VALUE as a __grid_constant__ kernel parameter
// (CUDA >= 12.1 allows 32 764 B), so every op/coefficient read is a uniform
// constant-bank load: no per-launch memcpy, graph-capturable, no races
// between slices on different streams.
#pragma once

#include <stdint.h>

namespace qkdev {

constexpr int kMaxRegBits = 5;              // register slots per thread (rb <= 5)
constexpr int kMaxTileBits = 13;            // 2^13 x 16 B = 128 KiB of smem
constexpr int kMaxOps = 700;
constexpr int kMaxCoef = 860;               // complex coefficients (double2)
constexpr int kMaxSegs = 96;
constexpr int kMaxContrib = 512;            // uint16 words for fused-diagonal index maps
constexpr int kMaxCtaFactors = 128;         // per-CTA diagonal factors (functions of non-tile bits)
constexpr int kMaxCtaTerms = 640;

// Register bits used for a tile of ct bits: 16 amplitudes per thread up to
// ct = 12 (<= 256 threads, no register cap), 32 per thread at ct = 13 (256
// threads x <= 255 registers: the 2^13-amplitude tile never spills).
// Tuning knobs (host; schedule.cpp): QK_MAX_TILE_BITS = 12|13 (default 13),
// QK_RB13 = 4|5 register bits at ct = 13 (default 5).
int maxTileBits();
int regBitsFor(int ct);
bool storeWide();
bool tileTune();
bool halfExchanges();
bool stageDense();
bool wideAccess();

enum OpType : uint8_t {
    OP_MAT1 = 0,      // a = slot; coef[c..c+3] = 2x2 row-major
    OP_H,             // a = slot; butterfly without 1/sqrt2 (folded into the final scale)
    OP_CX,            // a = target slot; k bit0: control is thread bit b (else slot b); k bit1: control polarity;
                      // k bit2: control is memory bit b outside the tile (a constant of the CTA)
    OP_DIAG1_R,       // a = slot; coef[c], coef[c+1] applied directly
    OP_DIAG2_RR,      // a = MSB slot, b = LSB slot; coef[c..c+3] applied directly
    OP_CPHASE_RR,     // a = MSB slot, b = LSB slot; coef[c] where (bit a, bit b) == pattern k
    OP_PEND_R,        // R[a] *= coef[c]
    OP_PEND_RT,       // R[a] *= coef[c + bit_b(thread)]
    OP_SCAL,          // P *= coef[c]
    OP_SCAL_T,        // P *= coef[c + bit_a(thread)]
    OP_SCAL_TT,       // P *= coef[c + 2 bit_a(thread) + bit_b(thread)]
    OP_FLUSH_SLOT,    // amplitudes with slot-a bit 1 *= R[a]; R[a] = 1
    OP_FLUSH,         // all amplitudes *= P * coef[c].x * prod_{a: bit a} R[a] (* coef[c16 - 1 + s] if c16); reset
    OP_DTABLE,        // fused diagonal: k targets; contrib[c16 .. c16+ct) index map; table at gtab + c
    OP_DENSE,         // fused dense 2^k (k <= 4): targets in canonical slots; matrix at gtab + c
    OP_EXCHANGE,      // shared-memory exchange: map_out[c-1] -> map_in[c] (segment c starts)
    OP_SCAL_TAB,      // P *= gtab[c + pext(thread, x16)]    (x16 = thread-bit mask)
    OP_PEND_TAB,      // R[a] *= gtab[c + pext(thread, x16)]
    OP_SCAL_CTA,      // P *= F[c]                          (F = this CTA's factors, see cta_terms)
    OP_PEND_CTA,      // R[a] *= F[c]
    OP_SCAL_TCTA,     // P *= bit_b(thread) ? F[c] : 1
    OP_FLUSH_SLOT_G,  // amplitudes with slot-a bit 1 *= R[a] * coef[c + pext(slot bits, b)]; R[a] = 1
    OP_RESET,         // P = 1, R[*] = 1 (the pending factors are re-issued for the next segment)
    OP_CX_PEND,       // before a thread-controlled CX on slot a (control thread bit b, k bit1 = polarity):
                      // where it fires, P *= R[a]; R[a] = 1 / R[a]  (the pending phase follows the swap)
    OP_CCX,           // Toffoli on target slot a: control 1 = b (k bit0: thread bit, else slot; k bit1: polarity),
                      // control 2 = c (k bit2: thread bit, else slot; k bit3: polarity); k bit4 / bit5: control
                      // 1 / 2 is memory bit b / c outside the tile (CTA constant)
};

// Diagonal gates never need their qubits inside the tile: a bit outside the
// tile is a constant of the CTA (a bit of its base index).  Factors that
// depend on such bits are computed once per tile: F[f] = product over terms
// [cta_end[f-1], cta_end[f]) of coef[c] if (base bit b1) & (base bit b2)
// (b1 = 255: unconditional).  OP_DTABLE indices take CTA bits from the
// contrib list after the ct tile words: count m, then m (memory bit, value).
struct CtaTerm {
    uint8_t b1, b2;
    uint16_t c;
};

struct DevOp {
    uint8_t type, a, b, k;
    uint32_t c;       // coefficient index (coef[]) or gtab offset (in double2 units)
    uint16_t c16;     // contrib[] offset for OP_DTABLE
    uint16_t x16;     // OP_DTABLE: XOR applied to the table index (flipped slots)
};

struct PassParams {
    int32_t ct;                       // tile bits
    int32_t rb;                       // register bits (must equal regBitsFor(ct))
    int32_t nsegs;
    int32_t nops;
    uint64_t tile_mask;               // physical tile bits
    int8_t tile_phys[16];             // physical bit of tile bit j (ascending)
    uint16_t seg_end[kMaxSegs];       // ops [seg_end[s-1], seg_end[s]) run in segment s
    uint16_t xmask_out[kMaxSegs];     // tile-index XOR of the data at segment end (X gates are relabels)
    uint8_t xsplit[kMaxSegs];         // exchange into segment c: register slot holding the same tile bit (>= 3)
                                      // before and after (255: none) -> two half-tile exchange phases
    uint8_t map_in[kMaxSegs][16];     // mapping at segment start (load / exchange-read)
    uint8_t map_out[kMaxSegs][16];    // mapping at segment end (exchange-write / store)
    DevOp ops[kMaxOps];
    double coef[2 * kMaxCoef];        // interleaved complex coefficients
    uint16_t contrib[kMaxContrib];
    int32_t ncta;                     // CTA factors (0: none)
    uint16_t cta_end[kMaxCtaFactors];
    CtaTerm cta_terms[kMaxCtaTerms];
    int32_t norm_out;  // specialized kernels: also write sum |a|^2 of each output tile to np[tile]
    int32_t half_x;    // exchanges scheduled splittable in halves (xsplit): TMA-pipelined kernel eligible
    int32_t stage_out;  // specialized kernels: in runs with known zeros, the output tile leaves through shared
                        // memory and the TMA engine (set for passes whose input is sparse in a basis run)
    double synth_amp;   // specialized basis pass: value of the synthesized |basis> amplitude (0: 1.0); the
                        // run's deferred H normalization (qkeng::DeferHScales)
};

static_assert(sizeof(PassParams) <= 32000, "kernel parameter limit");

}  // namespace qkdev
