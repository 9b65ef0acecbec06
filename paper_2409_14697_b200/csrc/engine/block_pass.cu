// Fused gate-block kernel (sm_100a).
//
// Replaces the reference's chunk loop applyBlock -> applyPrepared -> kern::apply1/
// diag1/diag2 + inline CX/SWAP/D_k/U_k loops (proj/src/engine.cpp:189-281,
// proj/src/kernels.cpp:16-48): instead of one sweep of a 2^C chunk per gate,
// one CTA streams a 2^ct-amplitude tile from HBM ONCE, applies a whole run of
// gates with the amplitudes held in registers (16 per thread), re-deals
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

__device__ __forceinline__ double2 coefAt(const PassParams& P, uint32_t i) {
    return make_double2(P.coef[2 * i], P.coef[2 * i + 1]);
}

using Regs = double2[kRegAmps];

// ---- register-slot gate bodies (K, J compile-time slots) -------------------

template <int K>
__device__ __forceinline__ void opH(Regs& a) {
#pragma unroll
    for (int s = 0; s < kRegAmps; s++)
        if (!(s & (1 << K))) {
            const double2 x = a[s], y = a[s | (1 << K)];
            a[s] = cadd(x, y);
            a[s | (1 << K)] = csub(x, y);
        }
}

template <int K>
__device__ __forceinline__ void opX(Regs& a) {
#pragma unroll
    for (int s = 0; s < kRegAmps; s++)
        if (!(s & (1 << K))) {
            const double2 t = a[s];
            a[s] = a[s | (1 << K)];
            a[s | (1 << K)] = t;
        }
}

template <int K>
__device__ __forceinline__ void opMat1(Regs& a, double2 m0, double2 m1, double2 m2, double2 m3) {
#pragma unroll
    for (int s = 0; s < kRegAmps; s++)
        if (!(s & (1 << K))) {
            const double2 x = a[s], y = a[s | (1 << K)];
            a[s] = cmac(cmul(m0, x), m1, y);
            a[s | (1 << K)] = cmac(cmul(m2, x), m3, y);
        }
}

template <int K>
__device__ __forceinline__ void opDiag1(Regs& a, double2 d0, double2 d1) {
#pragma unroll
    for (int s = 0; s < kRegAmps; s++) a[s] = cmul(a[s], (s & (1 << K)) ? d1 : d0);
}

// target slot K, control slot J
template <int K, int J>
__device__ __forceinline__ void opCxRR(Regs& a) {
    if constexpr (K != J) {
#pragma unroll
        for (int s = 0; s < kRegAmps; s++)
            if ((s & (1 << J)) && !(s & (1 << K))) {
                const double2 t = a[s];
                a[s] = a[s | (1 << K)];
                a[s | (1 << K)] = t;
            }
    }
}

// MSB slot K, LSB slot J
template <int K, int J>
__device__ __forceinline__ void opDiag2RR(Regs& a, const double2 (&d)[4]) {
    if constexpr (K != J) {
#pragma unroll
        for (int s = 0; s < kRegAmps; s++) a[s] = cmul(a[s], d[(((s >> K) & 1) << 1) | ((s >> J) & 1)]);
    }
}

template <int K, int J>
__device__ __forceinline__ void opCphaseRR(Regs& a, double2 e) {
    if constexpr (K != J) {
#pragma unroll
        for (int s = 0; s < kRegAmps; s++)
            if ((s & (1 << K)) && (s & (1 << J))) a[s] = cmul(a[s], e);
    }
}

template <int K>
__device__ __forceinline__ void opCphaseR(Regs& a, double2 e) {
#pragma unroll
    for (int s = 0; s < kRegAmps; s++)
        if (s & (1 << K)) a[s] = cmul(a[s], e);
}

template <int K, int J>
__device__ __forceinline__ void opSwapRR(Regs& a) {
    if constexpr (K < J) {
#pragma unroll
        for (int s = 0; s < kRegAmps; s++)
            if ((s & (1 << K)) && !(s & (1 << J))) {
                const int t = s ^ (1 << K) ^ (1 << J);
                const double2 x = a[s];
                a[s] = a[t];
                a[t] = x;
            }
    }
}

// Fused dense 2^KK x 2^KK in canonical slots (target j at slot KK-1-j).
// KK = 2 runs from registers; the matrix streams from the L1-cached table.
template <int KK>
__device__ __forceinline__ void opDenseReg(Regs& a, const double2* __restrict__ M) {
    constexpr int D = 1 << KK, G = kRegAmps >> KK;
#pragma unroll
    for (int g = 0; g < G; g++) {
        double2 out[D];
#pragma unroll
        for (int r = 0; r < D; r++) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int s = 0; s < D; s++) acc = cmac(acc, __ldg(M + r * D + s), a[g * D + s]);
            out[r] = acc;
        }
#pragma unroll
        for (int r = 0; r < D; r++) a[g * D + r] = out[r];
    }
}

// KK = 3, 4: inputs parked in this thread's column of shared memory
// (layout [slot][thread], conflict-free), outputs accumulated into registers.
template <int KK>
__device__ __forceinline__ void opDenseSmem(Regs& a, const double2* __restrict__ M, double2* sm, int nt) {
    constexpr int D = 1 << KK, G = kRegAmps >> KK;
    const int tid = threadIdx.x;
    __syncthreads();  // others may still read the exchange buffer
#pragma unroll
    for (int s = 0; s < kRegAmps; s++) sm[s * nt + tid] = a[s];
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

#define QK_SLOT1(v, F, ...)               \
    switch (v) {                          \
        case 0: F<0>(__VA_ARGS__); break; \
        case 1: F<1>(__VA_ARGS__); break; \
        case 2: F<2>(__VA_ARGS__); break; \
        default: F<3>(__VA_ARGS__); break; \
    }
#define QK_SLOT2_INNER(K, w, F, ...)         \
    switch (w) {                             \
        case 0: F<K, 0>(__VA_ARGS__); break; \
        case 1: F<K, 1>(__VA_ARGS__); break; \
        case 2: F<K, 2>(__VA_ARGS__); break; \
        default: F<K, 3>(__VA_ARGS__); break; \
    }
#define QK_SLOT2(v, w, F, ...)                                 \
    switch (v) {                                               \
        case 0: QK_SLOT2_INNER(0, w, F, __VA_ARGS__) break;    \
        case 1: QK_SLOT2_INNER(1, w, F, __VA_ARGS__) break;    \
        case 2: QK_SLOT2_INNER(2, w, F, __VA_ARGS__) break;    \
        default: QK_SLOT2_INNER(3, w, F, __VA_ARGS__) break;   \
    }

// Global offset of this thread's slot-0 amplitude and per-slot strides under map m.
template <int CT>
__device__ __forceinline__ void globalLayout(const PassParams& P, const uint8_t* m, uint32_t tid, uint64_t& off,
                                             uint64_t (&stride)[kRegBits]) {
    off = 0;
#pragma unroll
    for (int j = 0; j < CT - kRegBits; j++) off |= uint64_t((tid >> j) & 1u) << P.tile_phys[m[kRegBits + j]];
#pragma unroll
    for (int k = 0; k < kRegBits; k++) stride[k] = uint64_t(1) << P.tile_phys[m[k]];
}

template <int CT>
__device__ __forceinline__ void smemLayout(const uint8_t* m, uint32_t tid, uint32_t& u, uint32_t (&su)[kRegBits]) {
    uint32_t t = 0;
#pragma unroll
    for (int j = 0; j < CT - kRegBits; j++) t |= ((tid >> j) & 1u) << m[kRegBits + j];
    u = swz(t);
#pragma unroll
    for (int k = 0; k < kRegBits; k++) su[k] = swz(1u << m[k]);
}

__device__ __forceinline__ uint64_t slotOffset(int s, const uint64_t (&st)[kRegBits]) {
    return ((s & 1) ? st[0] : 0) | ((s & 2) ? st[1] : 0) | ((s & 4) ? st[2] : 0) | ((s & 8) ? st[3] : 0);
}
__device__ __forceinline__ uint32_t slotOffset(int s, const uint32_t (&st)[kRegBits]) {
    return ((s & 1) ? st[0] : 0) ^ ((s & 2) ? st[1] : 0) ^ ((s & 4) ? st[2] : 0) ^ ((s & 8) ? st[3] : 0);
}

}  // namespace

template <int CT>
__global__ void __launch_bounds__(1 << (CT - kRegBits), 1)
    k_block_pass(double2* __restrict__ state, const double2* __restrict__ gtab, const __grid_constant__ PassParams P) {
    constexpr int NT = 1 << (CT - kRegBits);
    extern __shared__ double2 sm[];
    const uint32_t tid = threadIdx.x;

    // CTA base index: blockIdx deposited into the non-tile bits.
    uint64_t base = blockIdx.x;
#pragma unroll
    for (int j = 0; j < CT; j++) {
        const int p = P.tile_phys[j];
        base = ((base >> p) << (p + 1)) | (base & ((uint64_t(1) << p) - 1));
    }

    Regs a;
    {
        uint64_t off, st[kRegBits];
        globalLayout<CT>(P, P.map_in[0], tid, off, st);
        off += base;
#pragma unroll
        for (int s = 0; s < kRegAmps; s++) a[s] = state[off | slotOffset(s, st)];
    }

    double2 scal = make_double2(1.0, 0.0);  // pending per-thread factor (thread-bit-only diagonals)
    int op = 0;
    for (int sg = 0; sg < P.nsegs; sg++) {
        if (sg > 0) {  // re-deal register bits through shared memory
            uint32_t u, su[kRegBits];
            __syncthreads();
            smemLayout<CT>(P.map_out[sg - 1], tid, u, su);
#pragma unroll
            for (int s = 0; s < kRegAmps; s++) sm[u ^ slotOffset(s, su)] = a[s];
            __syncthreads();
            smemLayout<CT>(P.map_in[sg], tid, u, su);
#pragma unroll
            for (int s = 0; s < kRegAmps; s++) a[s] = sm[u ^ slotOffset(s, su)];
        }
        const int end = P.seg_end[sg];
        for (; op < end; op++) {
            const DevOp o = P.ops[op];
            switch (o.type) {
                case OP_H: QK_SLOT1(o.a, opH, a) break;
                case OP_X: QK_SLOT1(o.a, opX, a) break;
                case OP_MAT1: {
                    const double2 m0 = coefAt(P, o.c), m1 = coefAt(P, o.c + 1), m2 = coefAt(P, o.c + 2),
                                  m3 = coefAt(P, o.c + 3);
                    QK_SLOT1(o.a, opMat1, a, m0, m1, m2, m3)
                    break;
                }
                case OP_CX_RR: QK_SLOT2(o.a, o.b, opCxRR, a) break;
                case OP_CX_RT:
                    if ((tid >> o.b) & 1u) QK_SLOT1(o.a, opX, a)
                    break;
                case OP_DIAG1_R: {
                    const double2 d0 = coefAt(P, o.c), d1 = coefAt(P, o.c + 1);
                    QK_SLOT1(o.a, opDiag1, a, d0, d1)
                    break;
                }
                case OP_DIAG1_T:
                    scal = cmul(scal, coefAt(P, o.c + ((tid >> o.a) & 1u)));
                    break;
                case OP_DIAG2_RR: {
                    const double2 d[4] = {coefAt(P, o.c), coefAt(P, o.c + 1), coefAt(P, o.c + 2), coefAt(P, o.c + 3)};
                    QK_SLOT2(o.a, o.b, opDiag2RR, a, d)
                    break;
                }
                case OP_DIAG2_RT: {
                    const uint32_t tb = (tid >> o.b) & 1u;
                    // thread bit MSB: entries (2tb, 2tb+1); thread bit LSB: (tb, 2+tb)
                    const double2 d0 = coefAt(P, o.c + (o.k ? 2 * tb : tb));
                    const double2 d1 = coefAt(P, o.c + (o.k ? 2 * tb + 1 : 2 + tb));
                    QK_SLOT1(o.a, opDiag1, a, d0, d1)
                    break;
                }
                case OP_DIAG2_TT:
                    scal = cmul(scal, coefAt(P, o.c + ((((tid >> o.a) & 1u) << 1) | ((tid >> o.b) & 1u))));
                    break;
                case OP_CPHASE_RR: {
                    const double2 e = coefAt(P, o.c);
                    QK_SLOT2(o.a, o.b, opCphaseRR, a, e)
                    break;
                }
                case OP_CPHASE_RT:
                    if ((tid >> o.b) & 1u) {
                        const double2 e = coefAt(P, o.c);
                        QK_SLOT1(o.a, opCphaseR, a, e)
                    }
                    break;
                case OP_CPHASE_TT:
                    if (((tid >> o.a) & (tid >> o.b)) & 1u) scal = cmul(scal, coefAt(P, o.c));
                    break;
                case OP_DTABLE: {
                    const uint16_t* cb = &P.contrib[o.c16];
                    uint32_t sub = 0;
#pragma unroll
                    for (int j = kRegBits; j < CT; j++)
                        if ((tid >> (j - kRegBits)) & 1u) sub |= cb[j];
                    const uint32_t c0 = cb[0], c1 = cb[1], c2 = cb[2], c3 = cb[3];
                    const double2* tab = gtab + o.c;
#pragma unroll
                    for (int s = 0; s < kRegAmps; s++) {
                        const uint32_t i = sub | ((s & 1) ? c0 : 0) | ((s & 2) ? c1 : 0) | ((s & 4) ? c2 : 0) |
                                           ((s & 8) ? c3 : 0);
                        a[s] = cmul(a[s], __ldg(tab + i));
                    }
                    break;
                }
                case OP_DENSE:
                    if (o.k == 2) opDenseReg<2>(a, gtab + o.c);
                    else if (o.k == 3) opDenseSmem<3>(a, gtab + o.c, sm, NT);
                    else opDenseSmem<4>(a, gtab + o.c, sm, NT);
                    break;
                case OP_FLUSH: {
                    const double2 f = make_double2(scal.x * P.coef[2 * o.c], scal.y * P.coef[2 * o.c]);
#pragma unroll
                    for (int s = 0; s < kRegAmps; s++) a[s] = cmul(a[s], f);
                    scal = make_double2(1.0, 0.0);
                    break;
                }
                case OP_SWAP_RR: QK_SLOT2(o.a, o.b, opSwapRR, a) break;
                default: break;
            }
        }
    }

    {
        uint64_t off, st[kRegBits];
        globalLayout<CT>(P, P.map_out[P.nsegs - 1], tid, off, st);
        off += base;
#pragma unroll
        for (int s = 0; s < kRegAmps; s++) state[off | slotOffset(s, st)] = a[s];
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

template <int CT>
static cudaError_t launchCT(double2* state, const double2* gtab, const PassParams& P, uint64_t ctas,
                            cudaStream_t stream) {
    constexpr int NT = 1 << (CT - kRegBits);
    const size_t smem = sizeof(double2) << CT;
    if (smem > 48 * 1024) {  // per-device attribute; cheap to re-apply
        cudaError_t e = cudaFuncSetAttribute(k_block_pass<CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    k_block_pass<CT><<<dim3(unsigned(ctas)), NT, smem, stream>>>(state, gtab, P);
    return cudaGetLastError();
}

cudaError_t launchBlockPass(double2* state, const double2* gtab, const PassParams& P, int nLocal,
                            cudaStream_t stream) {
    const uint64_t ctas = uint64_t(1) << (nLocal - P.ct);
    switch (P.ct) {
        case 4: return launchCT<4>(state, gtab, P, ctas, stream);
        case 5: return launchCT<5>(state, gtab, P, ctas, stream);
        case 6: return launchCT<6>(state, gtab, P, ctas, stream);
        case 7: return launchCT<7>(state, gtab, P, ctas, stream);
        case 8: return launchCT<8>(state, gtab, P, ctas, stream);
        case 9: return launchCT<9>(state, gtab, P, ctas, stream);
        case 10: return launchCT<10>(state, gtab, P, ctas, stream);
        case 11: return launchCT<11>(state, gtab, P, ctas, stream);
        case 12: return launchCT<12>(state, gtab, P, ctas, stream);
        case 13: return launchCT<13>(state, gtab, P, ctas, stream);
        default: return cudaErrorInvalidValue;
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
