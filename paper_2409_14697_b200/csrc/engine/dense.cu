// Fused dense U5 (the reference's default fusion_qbit = 5) over the whole
// slice: y_g = M x_g for every group g of 32 amplitudes that differ only in
// the 5 target bits (proj/src/engine.cpp:228-251: gather 2^k, row-major
// matvec, scatter; sub-index bit k-1-j = target j, engine.cpp:176-182).
//
// A CTA stages a 2^12-amplitude tile (the 5 target bits + the 7 lowest other
// bits, so rows are coalesced) in shared memory as two planes, re and im,
// [s][g] (s = target sub-index, g = one of the tile's 128 groups), applies M
// to its 128 groups and writes the tile back: one HBM round trip per U5
// (32 B/amp) and 128 complex multiply-adds per amplitude (FP64-bound on
// B200: 36.5 TF vs 6.5 TB/s).  Two ways to do the math, chosen by timing:
//   FMA  -- each thread holds one group's 32 inputs in registers and forms
//           its 32 outputs with DFMA, M broadcast from shared memory;
//   MMA  -- the tile as a real GEMM on the FP64 tensor cores (DMMA,
//           mma.sync.m8n8k4.f64): Y(64x128) = A(64x64) X(64x128) with
//           A = [[Mr, -Mi], [Mi, Mr]] in register fragments.
#include <cuda_runtime.h>
#include <stdint.h>

namespace qkdev {

namespace {

constexpr int kDk = 5;      // target bits
constexpr int kDctMax = 12;  // tile bits: 12 (DFMA, 128 groups), 11 (DMMA, 64 groups)
// Plane row stride (doubles).  DFMA (128 groups): +8, rows 16 banks apart.
// DMMA (64 groups): +4, rows 8 banks apart, so each half-warp of a B-fragment
// load (4 k-rows x 4 columns of doubles) hits 16 distinct bank pairs.
template <int CT>
struct TileShape {
    static constexpr int groups = 1 << (CT - kDk);
    static constexpr int stride = groups + (CT == 11 ? 4 : 8);
    static constexpr int plane = 32 * stride;
};

struct DenseSpec {
    int tbit[kDctMax];   // tile index bit j -> memory bit
    int vslot[kDctMax];  // tile index bit j -> plane offset contribution (s row or g column)
    int nfree;           // memory bits outside the tile (ascending)
    int fbit[40];
    uint64_t tileMask;   // memory bits of the tile
    uint64_t smask, sval;  // known zeros: the slice is zero outside {i : (i ^ sval) & smask == 0}
};

__device__ __forceinline__ double2 cmacD(double2 acc, double2 m, double2 x) {
    acc.x = fma(m.x, x.x, acc.x);
    acc.x = fma(-m.y, x.y, acc.x);
    acc.y = fma(m.x, x.y, acc.y);
    acc.y = fma(m.y, x.x, acc.y);
    return acc;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Real block matrix A[i][k] of the complex M (row-major 32x32 double2).
__device__ __forceinline__ double blockA(const double2* __restrict__ M, int i, int k) {
    const double2 m = __ldg(M + (i & 31) * 32 + (k & 31));
    if (i < 32) return k < 32 ? m.x : -m.y;
    return k < 32 ? m.y : m.x;
}

// FMA: 128 threads, one group each (its 32 inputs in registers, outputs
// written back into its own plane column: no other thread reads it), two
// CTAs per SM.  MMA: 2^11-amplitude tiles (64 groups), 256 threads, 8 warps
// each owning an 8 x 64 block of Y, three CTAs per SM (80 registers, 34 KiB
// of planes + 32 KiB of A fragments each) so some CTAs' loads and stores
// overlap the others' tensor-core work.
template <bool MMA>
__global__ void __launch_bounds__(MMA ? 256 : 128, MMA ? 3 : 2) k_dense_tile(double2* __restrict__ st, const double2* __restrict__ M,
                                                                  const __grid_constant__ DenseSpec sp, uint64_t ntiles) {
    constexpr int CT = MMA ? 11 : 12;
    constexpr int kDstride = TileShape<CT>::stride;
    constexpr int kDplane = TileShape<CT>::plane;
    constexpr int kDgroups = TileShape<CT>::groups;
    static_assert(kDgroups == 64 || kDgroups == 128, "tile shapes: 2^11 (DMMA) or 2^12 (DFMA) amplitudes");
    constexpr int LOGNT = MMA ? 8 : 7;
    constexpr int NT = 1 << LOGNT;
    constexpr int PER = (1 << CT) / NT;  // amplitudes per thread in the load / store phases
    constexpr int HI = CT - LOGNT;
    extern __shared__ double smd[];
    double* const Xr = smd;
    double* const Xi = smd + kDplane;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

    // this thread's part of every tile: t = tid | i << LOGNT
    uint64_t depLo = 0;
    int slotLo = 0;
#pragma unroll
    for (int j = 0; j < LOGNT; j++)
        if ((tid >> j) & 1) {
            depLo |= uint64_t(1) << sp.tbit[j];
            slotLo += sp.vslot[j];
        }

    // MMA: A = [[Mr, -Mi], [Mi, Mr]] (64 x 64) in shared memory in fragment
    // order, As[(rowTile * 16 + kk) * 32 + lane] = lane's A element for the
    // 8-row tile rowTile at k-step kk (one conflict-free LDS per k-step).
    // FMA: M itself in shared memory, read as warp-wide broadcasts.
    double2* const Ms = reinterpret_cast<double2*>(smd + 2 * kDplane);
    double* const As = smd + 2 * kDplane;
    if (MMA) {
        for (int e = tid; e < 8 * 16 * 32; e += NT) {
            const int l = e & 31, kk = (e >> 5) & 15, rt = e >> 9;
            As[e] = blockA(M, 8 * rt + (l >> 2), 4 * kk + (l & 3));
        }
    } else {
        for (int e = tid; e < 32 * 32; e += NT) Ms[e] = __ldg(M + e);
    }
    uint64_t depHi[HI];
    int slotHi[HI];
#pragma unroll
    for (int j = 0; j < HI; j++) {
        depHi[j] = uint64_t(1) << sp.tbit[LOGNT + j];
        slotHi[j] = sp.vslot[LOGNT + j];
    }

    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        uint64_t base = 0;
        for (int j = 0; j < sp.nfree; j++) base |= ((tile >> j) & 1) << sp.fbit[j];
        if (((base ^ sp.sval) & sp.smask & ~sp.tileMask) != 0) {  // outside the support: zeros in, zeros out
            const uint64_t b = base | depLo;
#pragma unroll 1
            for (int i = 0; i < PER; i++) {
                uint64_t a = b;
#pragma unroll
                for (int j = 0; j < HI; j++)
                    if ((i >> j) & 1) a |= depHi[j];
                __stcs(st + a, make_double2(0.0, 0.0));
            }
            continue;
        }
        __syncthreads();  // the previous tile's stores read the planes
        base |= depLo;
#pragma unroll 1
        for (int b8 = 0; b8 < PER; b8 += 8) {  // 8 loads in flight per thread per batch
            double2 v[8];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const int ii = b8 + i;
                uint64_t a = base;
#pragma unroll
                for (int j = 0; j < HI; j++)
                    if ((ii >> j) & 1) a |= depHi[j];
                v[i] = ((a ^ sp.sval) & sp.smask) == 0 ? __ldcs(st + a) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const int ii = b8 + i;
                int slot = slotLo;
#pragma unroll
                for (int j = 0; j < HI; j++)
                    if ((ii >> j) & 1) slot += slotHi[j];
                Xr[slot] = v[i].x;
                Xi[slot] = v[i].y;
            }
        }
        __syncthreads();
        if (!MMA) {
            const int g = tid;
            double2 x[32];
#pragma unroll
            for (int s = 0; s < 32; s++) x[s] = make_double2(Xr[s * kDstride + g], Xi[s * kDstride + g]);
#pragma unroll 1
            for (int r0 = 0; r0 < 32; r0 += 8) {  // 8 rows: 16 independent FMA chains per thread
                double2 acc[8];
#pragma unroll
                for (int q = 0; q < 8; q++) acc[q] = make_double2(0.0, 0.0);
#pragma unroll
                for (int s = 0; s < 32; s++)
#pragma unroll
                    for (int q = 0; q < 8; q++) acc[q] = cmacD(acc[q], Ms[(r0 + q) * 32 + s], x[s]);
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    Xr[(r0 + q) * kDstride + g] = acc[q].x;
                    Xi[(r0 + q) * kDstride + g] = acc[q].y;
                }
            }
        } else {
            // warp w: row tiles 2 (w & 3) .. +1, column tiles 4 (w >> 2) .. +3
            // (Y = 8 row tiles x 8 column tiles of 8 x 8): per k-step 2 A and
            // 4 B fragment loads feed 8 DMMAs
            const int rp = w & 3, ch = w >> 2;
            double acc[2][4][2];
#pragma unroll
            for (int r = 0; r < 2; r++)
#pragma unroll
                for (int c = 0; c < 4; c++) acc[r][c][0] = acc[r][c][1] = 0.0;
#pragma unroll 2
            for (int kk = 0; kk < 16; kk++) {
                const int k = 4 * kk + (lane & 3);
                const double a0 = As[((2 * rp) * 16 + kk) * 32 + lane];
                const double a1 = As[((2 * rp + 1) * 16 + kk) * 32 + lane];
                const double* const row = (k < 32 ? Xr : Xi) + (k & 31) * kDstride + 32 * ch + (lane >> 2);
                double b[4];
#pragma unroll
                for (int c = 0; c < 4; c++) b[c] = row[8 * c];
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    dmma(acc[0][c][0], acc[0][c][1], a0, b[c]);
                    dmma(acc[1][c][0], acc[1][c][1], a1, b[c]);
                }
            }
            __syncthreads();  // every warp has read X before Y overwrites it
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const int i = 8 * (2 * rp + r) + (lane >> 2);
                double* const plane = (i < 32 ? Xr : Xi) + (i & 31) * kDstride + 32 * ch + 2 * (lane & 3);
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    plane[8 * c] = acc[r][c][0];
                    plane[8 * c + 1] = acc[r][c][1];
                }
            }
        }
        __syncthreads();
#pragma unroll 1
        for (int b8 = 0; b8 < PER; b8 += 8) {  // batches of 8 stores (bounded register use)
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const int ii = b8 + i;
                uint64_t a = base;
                int slot = slotLo;
#pragma unroll
                for (int j = 0; j < HI; j++)
                    if ((ii >> j) & 1) {
                        a |= depHi[j];
                        slot += slotHi[j];
                    }
                __stcs(st + a, make_double2(Xr[slot], Xi[slot]));
            }
        }
    }
}

}  // namespace

// U5 over a slice of 2^nLocal >= 2^12 amplitudes; targets[j] = memory bit of
// sub-index bit (4 - j).  mode 0 = DFMA, 1 = DMMA.  smask != 0: the slice is
// zero outside {i : (i ^ sval) & smask == 0} (a run from a basis state): tiles
// outside it are written as zeros, inside only the support is read.
cudaError_t launchDenseTile(double2* state, const double2* M, const int* targets, int k, int nLocal, int mode,
                            int smCount, cudaStream_t stream, uint64_t smask, uint64_t sval) {
    const int kDct = mode ? 11 : 12;
    if (k != kDk || nLocal < kDct) return cudaErrorInvalidValue;
    const int kDstride = mode ? TileShape<11>::stride : TileShape<12>::stride;
    const int kDplane = 32 * kDstride;
    DenseSpec sp{};
    uint64_t tmask = 0;
    for (int j = 0; j < k; j++) tmask |= uint64_t(1) << targets[j];
    uint64_t tile = tmask;
    for (int b = 0; b < nLocal && __builtin_popcountll(tile) < kDct; b++) tile |= uint64_t(1) << b;
    int j = 0, gbit = 0;
    for (int b = 0; b < nLocal; b++) {
        if (!((tile >> b) & 1)) {
            sp.fbit[sp.nfree++] = b;
            continue;
        }
        sp.tbit[j] = b;
        int q = -1;
        for (int t = 0; t < k; t++)
            if (targets[t] == b) q = t;
        sp.vslot[j] = q >= 0 ? (1 << (k - 1 - q)) * kDstride : (1 << gbit++);
        j++;
    }
    sp.tileMask = tile;
    sp.smask = smask;
    sp.sval = sval;
    const uint64_t ntiles = uint64_t(1) << (nLocal - kDct);
    const size_t smem = sizeof(double) * 2 * kDplane + (mode ? sizeof(double) * 64 * 64 : sizeof(double2) * 32 * 32);
    const uint64_t resident = uint64_t(smCount) * (mode ? 3 : 2);
    const unsigned grid = unsigned(ntiles < resident ? ntiles : resident);
    cudaError_t e;
    if (mode) {
        e = cudaFuncSetAttribute(k_dense_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        k_dense_tile<true><<<grid, 256, smem, stream>>>(state, M, sp, ntiles);  // 8 warps x (8 rows x 64 groups)
    } else {
        e = cudaFuncSetAttribute(k_dense_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        k_dense_tile<false><<<grid, 128, smem, stream>>>(state, M, sp, ntiles);  // one group per thread
    }
    return cudaGetLastError();
}

}  // namespace qkdev
