// Fused gate-block kernel (sm_100a).
//
// Replaces the reference's chunk loop applyBlock -> applyPrepared -> kern::apply1/
// diag1/diag2 + inline CX/SWAP/D_k/U_k loops (proj/src/engine.cpp:189-281,
// proj/src/kernels.cpp:16-48): instead of one sweep of a 2^C chunk per gate,
// one CTA streams a 2^ct-amplitude tile from HBM ONCE, applies a whole run of
// gates with the amplitudes held in registers (2^rb per thread), re-deals
// register bits through a swizzled shared-memory exchange only when a gate
// needs a qubit that currently sits in the thread index, and writes the tile
// back ONCE.  HBM traffic per pass: 32 B per amplitude, independent of the
// number of gates in it.
//
// The op list is a __grid_constant__ kernel parameter (pass_program.h), so ops
// and coefficients are uniform constant-bank reads.
#include <cuda_runtime.h>

#include "pass_program.h"

namespace qkdev {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cinv(double2 a) {
    const double d = 1.0 / fma(a.x, a.x, a.y * a.y);
    return make_double2(a.x * d, -a.y * d);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// acc + m * x
__device__ __forceinline__ double2 cmac(double2 acc, double2 m, double2 x) {
    acc.x = fma(m.x, x.x, acc.x);
    acc.x = fma(-m.y, x.y, acc.x);
    acc.y = fma(m.x, x.y, acc.y);
    acc.y = fma(m.y, x.x, acc.y);
    return acc;
}

// XOR swizzle of a tile index for conflict-free 16-byte shared-memory access.
// Linear over GF(2): swz(x ^ y) = swz(x) ^ swz(y).  Tile bit p lands in bank
// group (p mod 3), so three lane bits with distinct residues never conflict.
__device__ __forceinline__ uint32_t swz(uint32_t u) {
    return u ^ (((u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12)) & 7u);
}

// Bits of t selected by mask m, compacted (PEXT over the <= 9 thread-index bits).
__device__ __forceinline__ uint32_t pextT(uint32_t t, uint32_t m) {
    uint32_t r = 0, i = 0;
#pragma unroll
    for (int j = 0; j < 10; j++)
        if ((m >> j) & 1u) r |= ((t >> j) & 1u) << i++;
    return r;
}

__device__ __forceinline__ double2 coefAt(const PassParams& P, uint32_t i) {
    return make_double2(P.coef[2 * i], P.coef[2 * i + 1]);
}

// ---- register-slot gate bodies (K, J compile-time slots, NA amplitudes) -----

template <int NA, int K>
__device__ __forceinline__ void opH(double2 (&a)[NA]) {
    if constexpr ((1 << K) < NA) {
#pragma unroll
        for (int s = 0; s < NA; s++)
            if (!(s & (1 << K))) {
                const double2 x = a[s], y = a[s | (1 << K)];
                a[s] = cadd(x, y);
                a[s | (1 << K)] = csub(x, y);
            }
    }
}

__device__ __forceinline__ double selD(bool p, double x, double y) {
    double r;
    asm("{ .reg .pred q; setp.ne.u32 q, %3, 0; selp.f64 %0, %1, %2, q; }" : "=d"(r) : "d"(x), "d"(y), "r"(int(p)));
    return r;
}

// Controlled swap of the slot-K pairs: a data-dependent select per pair, never
// a register renaming (renaming inside the op switch makes ptxas copy the
// whole register array every iteration).  cond(s) = control bit of s (slot
// control: (s & cm) == cv) and thread-level condition `thr`.
template <int NA, int K>
__device__ __forceinline__ void opCx(double2 (&a)[NA], uint32_t cm, uint32_t cv, bool thr) {
    if constexpr ((1 << K) < NA) {
#pragma unroll
        for (int s = 0; s < NA; s++)
            if (!(s & (1 << K))) {
                const bool c = thr && ((uint32_t(s) & cm) == cv);
                const double2 x = a[s], y = a[s | (1 << K)];
                a[s] = make_double2(selD(c, y.x, x.x), selD(c, y.y, x.y));
                a[s | (1 << K)] = make_double2(selD(c, x.x, y.x), selD(c, x.y, y.y));
            }
    }
}

template <int NA, int K>
__device__ __forceinline__ void opMat1(double2 (&a)[NA], double2 m0, double2 m1, double2 m2, double2 m3) {
    if constexpr ((1 << K) < NA) {
#pragma unroll
        for (int s = 0; s < NA; s++)
            if (!(s & (1 << K))) {
                const double2 x = a[s], y = a[s | (1 << K)];
                a[s] = cmac(cmul(m0, x), m1, y);
                a[s | (1 << K)] = cmac(cmul(m2, x), m3, y);
            }
    }
}

template <int NA, int K>
__device__ __forceinline__ void opDiag1(double2 (&a)[NA], double2 d0, double2 d1) {
    if constexpr ((1 << K) < NA) {
#pragma unroll
        for (int s = 0; s < NA; s++) a[s] = cmul(a[s], (s & (1 << K)) ? d1 : d0);
    }
}

// amplitudes whose slot-K bit is 1 *= e
template <int NA, int K>
__device__ __forceinline__ void opPhaseSlot(double2 (&a)[NA], double2 e) {
    if constexpr ((1 << K) < NA) {
#pragma unroll
        for (int s = 0; s < NA; s++)
            if (s & (1 << K)) a[s] = cmul(a[s], e);
    }
}

// MSB slot K, LSB slot J
template <int NA, int K, int J>
__device__ __forceinline__ void opDiag2RR(double2 (&a)[NA], const double2 (&d)[4]) {
    if constexpr (K != J && (1 << K) < NA && (1 << J) < NA) {
#pragma unroll
        for (int s = 0; s < NA; s++) a[s] = cmul(a[s], d[(((s >> K) & 1) << 1) | ((s >> J) & 1)]);
    }
}

// amplitudes whose (slot K, slot J) bits equal (pat >> 1, pat & 1) *= e;
// K < J, pattern already adjusted by the scheduler for any operand order.
template <int NA, int K, int J>
__device__ __forceinline__ void opCphaseRR(double2 (&a)[NA], double2 e, uint32_t pat) {
    if constexpr (K < J && (1 << J) < NA) {
        // Four candidate patterns; multiply only the matching quarter of the registers.
#pragma unroll
        for (uint32_t p = 0; p < 4; p++)
            if (p == pat) {
#pragma unroll
                for (int s = 0; s < NA; s++)
                    if ((((s >> K) & 1) << 1 | ((s >> J) & 1)) == int(p)) a[s] = cmul(a[s], e);
            }
    }
}

// Fused dense 2^KK x 2^KK in canonical slots (target j at slot KK-1-j):
// inputs parked in this thread's column of shared memory (layout
// [slot][thread], conflict-free), outputs accumulated back into registers.
template <int NA, int KK>
__device__ __forceinline__ void opDense(double2 (&a)[NA], const double2* __restrict__ M, double2* sm, int nt) {
    constexpr int D = 1 << KK, G = NA >> KK;
    const int tid = threadIdx.x;
    __syncthreads();  // others may still read the exchange buffer
#pragma unroll
    for (int s = 0; s < NA; s++) sm[s * nt + tid] = a[s];
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
        for (int r = 0; r < D; r++) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll 4
            for (int s = 0; s < D; s++) acc = cmac(acc, __ldg(M + r * D + s), sm[(g * D + s) * nt + tid]);
            a[g * D + r] = acc;
        }
}

// R[K] *= e (pending phase of slot K)
template <int RB, int K>
__device__ __forceinline__ void mulSlot(double2 (&R)[RB], double2 e) {
    if constexpr (K < RB) R[K] = cmul(R[K], e);
}

// amplitudes with slot-K bit 1 *= R[K]; R[K] = 1
template <int RB, int K>
__device__ __forceinline__ void flushSlot(double2 (&a)[1 << RB], double2 (&R)[RB]) {
    if constexpr (K < RB) {
        opPhaseSlot<(1 << RB), K>(a, R[K]);
        R[K] = make_double2(1.0, 0.0);
    }
}

#define QK_SLOT1(v, F, NA_, ...)                \
    switch (v) {                                \
        case 0: F<NA_, 0>(__VA_ARGS__); break;  \
        case 1: F<NA_, 1>(__VA_ARGS__); break;  \
        case 2: F<NA_, 2>(__VA_ARGS__); break;  \
        case 3: F<NA_, 3>(__VA_ARGS__); break;  \
        default: F<NA_, 4>(__VA_ARGS__); break; \
    }
#define QK_SLOT2_INNER(K, w, F, NA_, ...)          \
    switch (w) {                                   \
        case 0: F<NA_, K, 0>(__VA_ARGS__); break;  \
        case 1: F<NA_, K, 1>(__VA_ARGS__); break;  \
        case 2: F<NA_, K, 2>(__VA_ARGS__); break;  \
        case 3: F<NA_, K, 3>(__VA_ARGS__); break;  \
        default: F<NA_, K, 4>(__VA_ARGS__); break; \
    }
#define QK_SLOT2(v, w, F, NA_, ...)                                \
    switch (v) {                                                   \
        case 0: QK_SLOT2_INNER(0, w, F, NA_, __VA_ARGS__) break;   \
        case 1: QK_SLOT2_INNER(1, w, F, NA_, __VA_ARGS__) break;   \
        case 2: QK_SLOT2_INNER(2, w, F, NA_, __VA_ARGS__) break;   \
        case 3: QK_SLOT2_INNER(3, w, F, NA_, __VA_ARGS__) break;   \
        default: QK_SLOT2_INNER(4, w, F, NA_, __VA_ARGS__) break;  \
    }

template <int RB>
__device__ __forceinline__ uint64_t slotOffset(int s, const uint64_t (&st)[RB]) {
    uint64_t o = 0;
#pragma unroll
    for (int k = 0; k < RB; k++) o |= ((s >> k) & 1) ? st[k] : 0;
    return o;
}
template <int RB>
__device__ __forceinline__ uint32_t slotOffset(int s, const uint32_t (&st)[RB]) {
    uint32_t o = 0;
#pragma unroll
    for (int k = 0; k < RB; k++) o ^= ((s >> k) & 1) ? st[k] : 0;
    return o;
}

// Global offset of this thread's slot-0 amplitude and per-slot strides under map m.
template <int CT, int RB>
__device__ __forceinline__ void globalLayout(const PassParams& P, const uint8_t* m, uint32_t tid, uint64_t& off,
                                             uint64_t (&stride)[RB]) {
    off = 0;
#pragma unroll
    for (int j = 0; j < CT - RB; j++) off |= uint64_t((tid >> j) & 1u) << P.tile_phys[m[RB + j]];
#pragma unroll
    for (int k = 0; k < RB; k++) stride[k] = uint64_t(1) << P.tile_phys[m[k]];
}

template <int CT, int RB>
__device__ __forceinline__ void smemLayout(const uint8_t* m, uint32_t tid, uint32_t& u, uint32_t (&su)[RB]) {
    uint32_t t = 0;
#pragma unroll
    for (int j = 0; j < CT - RB; j++) t |= ((tid >> j) & 1u) << m[RB + j];
    u = swz(t);
#pragma unroll
    for (int k = 0; k < RB; k++) su[k] = swz(1u << m[k]);
}

__host__ __device__ constexpr int lowBit(int x) { return (x & 1) ? 0 : 1 + lowBit(x >> 1); }

// a[s] *= scale * P * prod_{k: bit k of s} R[k]; done as (low 2 slots) x (high slots)
// factor tables so each amplitude costs ~2 complex multiplies.
template <int RB>
__device__ __forceinline__ void flushAll(double2 (&a)[1 << RB], double2 P, double scale, double2 (&R)[RB],
                                         const double* D) {
    constexpr int NA = 1 << RB;
    const double2 base = make_double2(P.x * scale, P.y * scale);
    if constexpr (RB < 2) {
#pragma unroll
        for (int s = 0; s < NA; s++) {
            double2 f = base;
            if (s & 1) f = cmul(f, R[0]);
            a[s] = cmul(a[s], f);
        }
    } else {
        double2 lo[4];
        lo[0] = base;
        lo[1] = cmul(base, R[0]);
        lo[2] = cmul(base, R[1]);
        lo[3] = cmul(lo[1], R[1]);
        constexpr int NH = NA >> 2;
        double2 hi[NH];
        hi[0] = make_double2(1.0, 0.0);
#pragma unroll
        for (int h = 1; h < NH; h++) {
            const int low = lowBit(h);
            hi[h] = (h & (h - 1)) ? cmul(hi[h & (h - 1)], R[2 + low]) : R[2 + low];
        }
#pragma unroll
        for (int h = 0; h < NH; h++)
#pragma unroll
            for (int l = 0; l < 4; l++) a[h * 4 + l] = cmul(a[h * 4 + l], h ? cmul(lo[l], hi[h]) : lo[l]);
    }
    if (D) {  // constant register-pair phases
#pragma unroll
        for (int s = 0; s < NA; s++) a[s] = cmul(a[s], make_double2(D[2 * s], D[2 * s + 1]));
    }
#pragma unroll
    for (int k = 0; k < RB; k++) R[k] = make_double2(1.0, 0.0);
}

}  // namespace

template <int CT, int RB, int MINB>
__global__ void __launch_bounds__(1 << (CT - RB), MINB)
    k_block_pass(double2* __restrict__ state, const double2* __restrict__ gtab, const __grid_constant__ PassParams P,
                 const uint64_t basis) {
    constexpr int NT = 1 << (CT - RB);
    constexpr int NA = 1 << RB;
    extern __shared__ double2 sm[];
    const uint32_t tid = threadIdx.x;

    // CTA base index: blockIdx deposited into the non-tile bits.
    uint64_t base = blockIdx.x;
#pragma unroll
    for (int j = 0; j < CT; j++) {
        const int p = P.tile_phys[j];
        base = ((base >> p) << (p + 1)) | (base & ((uint64_t(1) << p) - 1));
    }

    double2 a[NA];
    if (basis != ~uint64_t(0) && ((basis ^ base) & ~P.tile_mask) != 0) {
        // first pass of a run, tile without the basis index: zeros in, zeros out
        uint64_t off, st[RB];
        globalLayout<CT, RB>(P, P.map_in[0], tid, off, st);
        off |= base;
#pragma unroll
        for (int s = 0; s < NA; s++) __stcs(state + (off | slotOffset<RB>(s, st)), make_double2(0.0, 0.0));
        return;
    }
    {
        uint64_t off, st[RB];
        globalLayout<CT, RB>(P, P.map_in[0], tid, off, st);
        off |= base;
        if (basis == ~uint64_t(0)) {
#pragma unroll
            for (int s = 0; s < NA; s++) a[s] = __ldcs(state + (off | slotOffset<RB>(s, st)));
        } else {  // first pass of a run: synthesize the basis state |basis> instead of reading it
#pragma unroll
            for (int s = 0; s < NA; s++)
                a[s] = make_double2((off | slotOffset<RB>(s, st)) == basis ? 1.0 : 0.0, 0.0);
        }
    }

    // Per-CTA diagonal factors (functions of the non-tile bits of `base`).
    double2* F = sm + (1 << CT);
    if (P.ncta) {  // warp per factor, lanes over its terms, shuffle-tree product
        const int w = int(tid >> 5), l = int(tid & 31u);
        for (int f = w; f < P.ncta; f += (NT + 31) / 32) {
            double2 acc = make_double2(1.0, 0.0);
            for (int t = (f ? P.cta_end[f - 1] : 0) + l; t < P.cta_end[f]; t += 32) {
                const CtaTerm& ct = P.cta_terms[t];
                if (ct.b1 == 255 || ((base >> ct.b1) & (base >> ct.b2) & 1u)) acc = cmul(acc, coefAt(P, ct.c));
            }
            const unsigned mask = NT >= 32 ? 0xffffffffu : ((1u << NT) - 1u);
            for (int o = (NT >= 32 ? 16 : NT / 2); o > 0; o >>= 1)
                acc = cmul(acc, make_double2(__shfl_xor_sync(mask, acc.x, o), __shfl_xor_sync(mask, acc.y, o)));
            if (l == 0) F[f] = acc;
        }
        __syncthreads();
    }

    double2 Pt = make_double2(1.0, 0.0);  // pending per-thread scalar
    double2 R[RB];                         // pending per-slot phases (amplitudes with slot bit 1)
#pragma unroll
    for (int k = 0; k < RB; k++) R[k] = make_double2(1.0, 0.0);

    // One flat loop over the ops (a nested segment loop makes ptxas re-copy
    // the whole register array at every iteration).
    const int nops = P.nops;
    for (int op = 0; op < nops; op++) {
        {
            const DevOp o = P.ops[op];
            switch (o.type) {
                case OP_EXCHANGE: {  // re-deal register bits through shared memory
                    uint32_t u, su[RB];
                    __syncthreads();
                    smemLayout<CT, RB>(P.map_out[o.c - 1], tid, u, su);
                    u ^= swz(P.xmask_out[o.c - 1]);  // flipped slots (X relabels)
#pragma unroll
                    for (int s = 0; s < NA; s++) sm[u ^ slotOffset<RB>(s, su)] = a[s];
                    __syncthreads();
                    smemLayout<CT, RB>(P.map_in[o.c], tid, u, su);
#pragma unroll
                    for (int s = 0; s < NA; s++) a[s] = sm[u ^ slotOffset<RB>(s, su)];
                    break;
                }
                case OP_H: QK_SLOT1(o.a, opH, NA, a) break;
                case OP_MAT1: {
                    const double2 m0 = coefAt(P, o.c), m1 = coefAt(P, o.c + 1), m2 = coefAt(P, o.c + 2),
                                  m3 = coefAt(P, o.c + 3);
                    QK_SLOT1(o.a, opMat1, NA, a, m0, m1, m2, m3)
                    break;
                }
                case OP_CX: {
                    const uint32_t pol = (o.k >> 1) & 1u;
                    uint32_t cm = 0, cv = 0;
                    bool thr = true;
                    if (o.k & 4u) thr = ((base >> o.b) & 1u) != 0;  // CTA-bit control
                    else if (o.k & 1u) thr = (((tid >> o.b) & 1u) ^ pol) != 0;
                    else {
                        cm = 1u << o.b;
                        cv = (1u ^ pol) << o.b;
                    }
                    QK_SLOT1(o.a, opCx, NA, a, cm, cv, thr)
                    break;
                }
                case OP_CCX: {
                    uint32_t cm = 0, cv = 0;
                    bool thr = true;
                    const uint32_t p1 = (o.k >> 1) & 1u, p2 = (o.k >> 3) & 1u;
                    if (o.k & 16u) thr = ((base >> o.b) & 1u) != 0;  // CTA-bit control
                    else if (o.k & 1u) thr = (((tid >> o.b) & 1u) ^ p1) != 0;
                    else {
                        cm |= 1u << o.b;
                        cv |= (1u ^ p1) << o.b;
                    }
                    if (o.k & 32u) thr = thr && (((base >> o.c) & 1u) != 0);
                    else if (o.k & 4u) thr = thr && ((((tid >> o.c) & 1u) ^ p2) != 0);
                    else {
                        cm |= 1u << o.c;
                        cv |= (1u ^ p2) << o.c;
                    }
                    QK_SLOT1(o.a, opCx, NA, a, cm, cv, thr)
                    break;
                }
                case OP_DIAG1_R: {
                    const double2 d0 = coefAt(P, o.c), d1 = coefAt(P, o.c + 1);
                    QK_SLOT1(o.a, opDiag1, NA, a, d0, d1)
                    break;
                }
                case OP_DIAG2_RR: {
                    const double2 d[4] = {coefAt(P, o.c), coefAt(P, o.c + 1), coefAt(P, o.c + 2), coefAt(P, o.c + 3)};
                    QK_SLOT2(o.a, o.b, opDiag2RR, NA, a, d)
                    break;
                }
                case OP_CPHASE_RR: {
                    const double2 e = coefAt(P, o.c);
                    const uint32_t pat = o.k;
                    QK_SLOT2(o.a, o.b, opCphaseRR, NA, a, e, pat)
                    break;
                }
                case OP_PEND_R: {
                    const double2 e = coefAt(P, o.c);
#pragma unroll
                    for (int k = 0; k < RB; k++)
                        if (k == o.a) R[k] = cmul(R[k], e);
                    break;
                }
                case OP_PEND_RT: {
                    const uint32_t tb = (tid >> o.b) & 1u;
                    const double2 e0 = coefAt(P, o.c), e1 = coefAt(P, o.c + 1);  // uniform loads, then select
                    const double2 e = make_double2(tb ? e1.x : e0.x, tb ? e1.y : e0.y);
#pragma unroll
                    for (int k = 0; k < RB; k++)
                        if (k == o.a) R[k] = cmul(R[k], e);
                    break;
                }
                case OP_SCAL_TAB: Pt = cmul(Pt, __ldg(gtab + o.c + pextT(tid, o.x16))); break;
                case OP_SCAL_CTA: Pt = cmul(Pt, F[o.c]); break;
                case OP_RESET:
                    Pt = make_double2(1.0, 0.0);
#pragma unroll
                    for (int k = 0; k < RB; k++) R[k] = make_double2(1.0, 0.0);
                    break;
                case OP_FLUSH_SLOT_G: {
                    double2 rk = R[0];
#pragma unroll
                    for (int k = 1; k < RB; k++)
                        if (k == o.a) rk = R[k];
#pragma unroll
                    for (int s = 0; s < NA; s++)
                        if ((s >> o.a) & 1) {
                            uint32_t idx = 0, q = 0;
#pragma unroll
                            for (int k = 0; k < RB; k++)
                                if ((o.b >> k) & 1u) idx |= uint32_t((s >> k) & 1) << q++;
                            a[s] = cmul(a[s], cmul(rk, coefAt(P, o.c + idx)));
                        }
#pragma unroll
                    for (int k = 0; k < RB; k++)
                        if (k == o.a) R[k] = make_double2(1.0, 0.0);
                    break;
                }
                case OP_CX_PEND:
                    if ((((tid >> o.b) & 1u) ^ ((o.k >> 1) & 1u)) != 0u) {
#pragma unroll
                        for (int k = 0; k < RB; k++)
                            if (k == o.a) {
                                Pt = cmul(Pt, R[k]);
                                R[k] = cinv(R[k]);
                            }
                    }
                    break;
                case OP_SCAL_TCTA:
                    if ((tid >> o.b) & 1u) Pt = cmul(Pt, F[o.c]);
                    break;
                case OP_PEND_CTA: {
                    const double2 e = F[o.c];
#pragma unroll
                    for (int k = 0; k < RB; k++)
                        if (k == o.a) R[k] = cmul(R[k], e);
                    break;
                }
                case OP_PEND_TAB: {
                    const double2 e = __ldg(gtab + o.c + pextT(tid, o.x16));
#pragma unroll
                    for (int k = 0; k < RB; k++)
                        if (k == o.a) R[k] = cmul(R[k], e);
                    break;
                }
                case OP_SCAL: Pt = cmul(Pt, coefAt(P, o.c)); break;
                case OP_SCAL_T: {
                    const uint32_t tb = (tid >> o.a) & 1u;
                    const double2 e0 = coefAt(P, o.c), e1 = coefAt(P, o.c + 1);
                    Pt = cmul(Pt, make_double2(tb ? e1.x : e0.x, tb ? e1.y : e0.y));
                    break;
                }
                case OP_SCAL_TT: {
                    const uint32_t i = (((tid >> o.a) & 1u) << 1) | ((tid >> o.b) & 1u);
                    const double2 e0 = coefAt(P, o.c), e1 = coefAt(P, o.c + 1), e2 = coefAt(P, o.c + 2),
                                  e3 = coefAt(P, o.c + 3);
                    const double2 lo = (i & 1u) ? e1 : e0, hi = (i & 1u) ? e3 : e2;
                    Pt = cmul(Pt, (i & 2u) ? hi : lo);
                    break;
                }
                case OP_FLUSH_SLOT: {
                    double2 e = R[0];
#pragma unroll
                    for (int k = 1; k < RB; k++)
                        if (k == o.a) e = R[k];
                    QK_SLOT1(o.a, opPhaseSlot, NA, a, e)
#pragma unroll
                    for (int k = 0; k < RB; k++)
                        if (k == o.a) R[k] = make_double2(1.0, 0.0);
                    break;
                }
                case OP_FLUSH:
                    flushAll<RB>(a, Pt, P.coef[2 * o.c], R, o.c16 ? &P.coef[2 * (o.c16 - 1)] : nullptr);
                    Pt = make_double2(1.0, 0.0);
                    break;
                case OP_DTABLE: {
                    const uint16_t* cb = &P.contrib[o.c16];
                    const uint32_t flipx = o.x16;
                    uint32_t sub = 0;
#pragma unroll
                    for (int j = RB; j < CT; j++)
                        if ((tid >> (j - RB)) & 1u) sub |= cb[j];
                    for (int j = 0; j < cb[CT]; j++)  // bits outside the tile: constants of the CTA
                        if ((base >> cb[CT + 1 + 2 * j]) & 1u) sub |= cb[CT + 2 + 2 * j];
                    uint32_t cr[RB];
#pragma unroll
                    for (int k = 0; k < RB; k++) cr[k] = cb[k];
                    const double2* tab = gtab + o.c;
#pragma unroll
                    for (int s = 0; s < NA; s++) {
                        uint32_t i = sub;
#pragma unroll
                        for (int k = 0; k < RB; k++) i |= ((s >> k) & 1) ? cr[k] : 0u;
                        a[s] = cmul(a[s], __ldg(tab + (i ^ flipx)));
                    }
                    break;
                }
                case OP_DENSE:
                    if constexpr (RB >= 2) {
                        if (o.k == 2) opDense<NA, 2>(a, gtab + o.c, sm, NT);
                        else if constexpr (RB >= 3) {
                            if (o.k == 3) opDense<NA, 3>(a, gtab + o.c, sm, NT);
                            else if constexpr (RB >= 4) opDense<NA, 4>(a, gtab + o.c, sm, NT);
                        }
                    }
                    break;
                default: break;
            }
        }
    }

    // A single-segment pass may store through a different map than it loaded
    // with (free in-tile output permutation): wait until every thread of the
    // CTA has loaded before anyone overwrites the tile.
    if (P.nsegs == 1) __syncthreads();
    {
        uint64_t off, st[RB];
        globalLayout<CT, RB>(P, P.map_out[P.nsegs - 1], tid, off, st);
        off |= base;
        const uint32_t xm = P.xmask_out[P.nsegs - 1];  // flipped slots (X relabels)
#pragma unroll
        for (int j = 0; j < CT; j++) off ^= uint64_t((xm >> j) & 1u) << P.tile_phys[j];
#pragma unroll
        for (int s = 0; s < NA; s++) __stcs(state + (off ^ slotOffset<RB>(s, st)), a[s]);
    }
}

// One CTA per 2^k group: the generic dense path for fused gates wider than the
// register window (U5 from the reference's default fusion_qbit = 5) and for
// slices too small for a tile.  Targets: target j = sub-index bit (k-1-j).
__global__ void k_dense_group(double2* __restrict__ state, const double2* __restrict__ M, int k,
                              uint64_t targetMask, const int* __restrict__ tgt, uint64_t groups) {
    extern __shared__ double2 buf[];
    const int dim = 1 << k;
    for (uint64_t g = blockIdx.x; g < groups; g += gridDim.x) {
        // deposit g into the non-target bits
        uint64_t base = 0, rest = g;
        for (int p = 0; rest; p++) {
            if ((targetMask >> p) & 1) continue;
            base |= (rest & 1) << p;
            rest >>= 1;
        }
        for (int s = threadIdx.x; s < dim; s += blockDim.x) {
            uint64_t o = base;
            for (int j = 0; j < k; j++) o |= uint64_t((s >> (k - 1 - j)) & 1) << tgt[j];
            buf[s] = state[o];
        }
        __syncthreads();
        for (int r = threadIdx.x; r < dim; r += blockDim.x) {
            double2 acc = make_double2(0.0, 0.0);
            for (int s = 0; s < dim; s++) acc = cmac(acc, __ldg(M + uint64_t(r) * dim + s), buf[s]);
            uint64_t o = base;
            for (int j = 0; j < k; j++) o |= uint64_t((r >> (k - 1 - j)) & 1) << tgt[j];
            state[o] = acc;
        }
        __syncthreads();
    }
}

// ---- launchers --------------------------------------------------------------

// The interpreter runs tiles of <= 2^12 amplitudes, 8 per thread (RB = 3):
// 512 threads and 128 registers at CT = 12, two CTAs per SM below.  Its
// register budget then holds the amplitudes, pending phases and op operands
// without spilling (the specialized kernels, not this one, serve slices
// >= 2^22).
template <int CT, int RB = (CT < 3 ? CT : 3)>
static cudaError_t launchCT(double2* state, const double2* gtab, const PassParams& P, uint64_t ctas,
                            uint64_t basis, cudaStream_t stream) {
    constexpr int NT = 1 << (CT - RB);
    constexpr int MINB = CT <= 11 ? 2 : 1;
    const size_t smem = (sizeof(double2) << CT) + sizeof(double2) * kMaxCtaFactors;
    if (smem > 48 * 1024) {  // per-device attribute; cheap to re-apply
        cudaError_t e = cudaFuncSetAttribute(k_block_pass<CT, RB, MINB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    k_block_pass<CT, RB, MINB><<<dim3(unsigned(ctas)), NT, smem, stream>>>(state, gtab, P, basis);
    return cudaGetLastError();
}

cudaError_t launchBlockPass(double2* state, const double2* gtab, const PassParams& P, int nLocal, uint64_t basis,
                            cudaStream_t stream) {
    if (P.rb != (P.ct < 3 ? P.ct : 3))
        return cudaErrorInvalidValue;  // compiled for the specialized kernels (compileBlock interp = false)
    const uint64_t ctas = uint64_t(1) << (nLocal - P.ct);
    switch (P.ct) {
        case 4: return launchCT<4>(state, gtab, P, ctas, basis, stream);
        case 5: return launchCT<5>(state, gtab, P, ctas, basis, stream);
        case 6: return launchCT<6>(state, gtab, P, ctas, basis, stream);
        case 7: return launchCT<7>(state, gtab, P, ctas, basis, stream);
        case 8: return launchCT<8>(state, gtab, P, ctas, basis, stream);
        case 9: return launchCT<9>(state, gtab, P, ctas, basis, stream);
        case 10: return launchCT<10>(state, gtab, P, ctas, basis, stream);
        case 11: return launchCT<11>(state, gtab, P, ctas, basis, stream);
        case 12: return launchCT<12>(state, gtab, P, ctas, basis, stream);
        default: return cudaErrorInvalidValue;  // interpreter tiles are <= 2^12 (compileBlock interp)
    }
}

cudaError_t launchDenseGroup(double2* state, const double2* M, int k, const int* dTargets, uint64_t targetMask,
                             int nLocal, cudaStream_t stream) {
    const uint64_t groups = uint64_t(1) << (nLocal - k);
    const int threads = k >= 8 ? 256 : (1 << k) < 32 ? 32 : (1 << k);
    const size_t smem = sizeof(double2) << k;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_dense_group, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    const uint64_t grid = groups < (uint64_t(1) << 20) ? groups : (uint64_t(1) << 20);
    k_dense_group<<<unsigned(grid), threads, smem, stream>>>(state, M, k, targetMask, dTargets, groups);
    return cudaGetLastError();
}

}  // namespace qkdev
