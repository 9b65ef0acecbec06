// Data-movement and reduction kernels (sm_100a): IMS, XRS slab swap / window
// copies, norm, basis init, whole-slice diagonal tables.
//
//   k_ims          replaces imsSwap (proj/src/engine.cpp:86-101)
//   k_slab_swap    replaces xrsFill + xrsDeliver for slices in one process
//                  (proj/src/distributed.cpp:76-120): in-place pairwise swap, no buffer
//   k_window_pack / k_window_unpack
//                  the NCCL path's send pack / copy-back (distributed.cpp:76-120)
//   k_norm_*       StateVector::norm (engine.cpp:12-16), deterministic tree order
//   k_set_basis    initState (engine.cpp:18-28) after a memset
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

namespace qkdev {

struct PairSpec {
    int s;
    int out[40];
    int in[40];
};

// x with bits out[j] <-> in[j] exchanged (a GF(2)-linear bit permutation).
__device__ __forceinline__ uint64_t bitswapDev(uint64_t x, const PairSpec& p) {
    for (int j = 0; j < p.s; j++) {
        const uint64_t d = ((x >> p.out[j]) ^ (x >> p.in[j])) & 1u;
        x ^= (d << p.out[j]) | (d << p.in[j]);
    }
    return x;
}

// In-place a[bitswap(i)] <- a[i].  Thread t owns x = t | (k << logT) for
// k = 0..; bitswap is linear, so P(x) = P(t) ^ P(k << logT), and P(k << logT)
// is advanced incrementally from a table of P(trailing-ones masks): a handful
// of integer ops per element instead of 5 per pair.  Each orbit {x, P(x)} is
// swapped once, by its smaller member (the reference swaps from the larger
// one; the permutation is the same).
__global__ void __launch_bounds__(256) k_ims(double2* __restrict__ a, int logN, int logT, const __grid_constant__ PairSpec p) {
    __shared__ uint64_t steps[64];
    const int hiBits = logN - logT;
    if (threadIdx.x < hiBits + 1) {
        const int j = threadIdx.x;  // mask of (j+1) trailing ones, shifted to the high part
        const uint64_t m = (j + 1 >= 64) ? ~uint64_t(0) : ((uint64_t(1) << (j + 1)) - 1);
        steps[j] = bitswapDev(m << logT, p);
    }
    __syncthreads();
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint64_t px = bitswapDev(t, p);  // P(t | 0)
    const uint64_t K = uint64_t(1) << hiBits;
    uint64_t k = 0;
    while (k < K) {
        // 8 independent elements per trip for memory-level parallelism.
        uint64_t xs[8], ys[8];
        int n = 0;
#pragma unroll
        for (int u = 0; u < 8; u++) {
            if (k < K) {
                xs[u] = t | (k << logT);
                ys[u] = px;
                n = u + 1;
                const int tz = __ffsll((long long)(~k)) - 1;  // trailing ones of k
                if (k + 1 < K) px ^= steps[tz];
                k++;
            }
        }
        double2 vx[8], vy[8];
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (u < n && xs[u] < ys[u]) {
                vx[u] = __ldcs(a + xs[u]);
                vy[u] = __ldcs(a + ys[u]);
            }
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (u < n && xs[u] < ys[u]) {
                __stcs(a + xs[u], vy[u]);
                __stcs(a + ys[u], vx[u]);
            }
    }
}

// Tiled IMS.  T = a P-closed set of k <= 6 bits containing memory bits 0..2
// (128-B rows) and their pair partners; a "tile" is the 2^k indices varying
// over T.  P maps tile(h) onto tile(P(h)) (h = the non-T bits), permuting the
// tile coordinates by pi.  One warp per orbit {h, P(h)}: both tiles are read
// with coalesced 128-B rows, staged in warp-private shared memory, and written
// back permuted, so pairs with a low "out" bit cost no sector waste (k_ims
// reads 1.4x the bytes for those).
struct ImsTileSpec {
    int k;                 // tile bits
    int n;                 // slice bits
    int tbit[8];           // tile coordinate r -> memory bit (ascending)
    int pi[8];             // tile coordinate r -> coordinate of P(bit)
    int nfree;             // non-tile bits, ascending
    int fbit[58];
    int nhp;               // pairs among non-tile bits (memory bits)
    int ho[29], hi[29];
    int swz[5];            // staging swizzle: coordinate bit 3+i XORs swz[i] into bits 0..2
    int a;                 // 2^a warps; warp w walks g = w | (k << a)
    int piIdentity;        // pi fixes every tile coordinate: self-mapped tiles need no work
    uint64_t hstep[58];    // dep(trailing-ones mask j+1, shifted by a): h(k+1) = h(k) ^ hstep[tz(~k)]
    uint64_t pstep[58];    // P(hstep[j])
};

// Staging index: coordinate u with bits 0..2 XORed by a linear function of
// bits 3..5, chosen on the host so both the write pattern (lanes 0..7 vary
// coordinate bits 0..2) and the permuted read pattern are bank-conflict free.
__device__ __forceinline__ int stageIdx(int u, const ImsTileSpec& sp) {
    int x = u;
#pragma unroll
    for (int i = 0; i < 5; i++)
        if ((u >> (3 + i)) & 1) x ^= sp.swz[i];
    return x;
}

// PER amplitudes per lane per tile (tiles of 32 * PER = 2^k amplitudes), U
// orbits per trip; each warp stages one tile pair at a time.
template <int PER, int U>
__global__ void __launch_bounds__(256) k_ims_tiled(double2* __restrict__ a, const __grid_constant__ ImsTileSpec sp) {
    extern __shared__ double2 tbuf[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double2* const bufA = tbuf + size_t(w) * 2 * 32 * PER;
    double2* const bufB = bufA + 32 * PER;
    // tile coordinates handled by this lane: their memory offsets, staging
    // slots, and the staging slot of the permuted source coordinate
    uint64_t off[PER];
    int tpi[PER], sidx[PER];
#pragma unroll
    for (int e = 0; e < PER; e++) {
        const int t = lane + 32 * e;
        uint64_t o = 0;
        int u = 0;
        for (int r = 0; r < sp.k; r++)
            if ((t >> r) & 1) {
                o |= uint64_t(1) << sp.tbit[r];
                u |= 1 << sp.pi[r];
            }
        off[e] = o;
        tpi[e] = stageIdx(u, sp);  // pi(t): source coordinate for output coordinate t (pi is an involution)
        sidx[e] = stageIdx(t, sp);
    }
    // Warp w walks h = dep(w | k << a) for k = 0.. with incremental XOR steps
    // (deposit and P are GF(2)-linear), a handful of integer ops per orbit.
    const uint64_t wid = uint64_t(blockIdx.x) * (blockDim.x >> 5) + w;
    uint64_t h = 0;
    for (int j = 0; j < sp.a; j++) h |= ((wid >> j) & 1) << sp.fbit[j];
    uint64_t ph = h;
    for (int j = 0; j < sp.nhp; j++) {
        const uint64_t d = ((ph >> sp.ho[j]) ^ (ph >> sp.hi[j])) & 1u;
        ph ^= (d << sp.ho[j]) | (d << sp.hi[j]);
    }
    const uint64_t K = uint64_t(1) << (sp.nfree - sp.a);
    for (uint64_t k = 0; k < K; k += U) {
        uint64_t hs[U], ps[U];
        bool lead[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            const uint64_t kk = k + q;
            if (kk) {
                const int tz = __ffsll((long long)(~(kk - 1))) - 1;
                h ^= sp.hstep[tz];
                ph ^= sp.pstep[tz];
            }
            hs[q] = h;
            ps[q] = ph;
            // the orbit's smaller member does the work; a tile mapped onto
            // itself with pi = identity does not move at all
            lead[q] = kk < K && ph >= h && !(ph == h && sp.piIdentity);
        }
        double2 va[U][PER], vb[U][PER];  // every load of the trip in flight at once
#pragma unroll
        for (int q = 0; q < U; q++)
            if (lead[q]) {
#pragma unroll
                for (int e = 0; e < PER; e++) va[q][e] = __ldcs(a + (hs[q] | off[e]));
                if (ps[q] != hs[q])
#pragma unroll
                    for (int e = 0; e < PER; e++) vb[q][e] = __ldcs(a + (ps[q] | off[e]));
            }
#pragma unroll
        for (int q = 0; q < U; q++) {
            if (!lead[q]) continue;  // warp-uniform
#pragma unroll
            for (int e = 0; e < PER; e++) {
                bufA[sidx[e]] = va[q][e];
                if (ps[q] != hs[q]) bufB[sidx[e]] = vb[q][e];
            }
            __syncwarp();
            // tile(ph)[t] <- tile(h)[pi(t)];  tile(h)[t] <- tile(ph)[pi(t)]
#pragma unroll
            for (int e = 0; e < PER; e++) __stcs(a + (ps[q] | off[e]), bufA[tpi[e]]);
            if (ps[q] != hs[q])
#pragma unroll
                for (int e = 0; e < PER; e++) __stcs(a + (hs[q] | off[e]), bufB[tpi[e]]);
            __syncwarp();
        }
    }
}

// Offsets of a slab element: o deposited around the (ascending) out positions.
struct SlabSpec {
    int s;
    int outs[8];   // ascending
};

__device__ __forceinline__ uint64_t depositAround(uint64_t o, const SlabSpec& sp) {
    for (int j = 0; j < sp.s; j++) {
        const int p = sp.outs[j];
        o = ((o >> p) << (p + 1)) | (o & ((uint64_t(1) << p) - 1));
    }
    return o;
}

// Swap slab elements pairwise: A[dep(o)] <-> B[dep(o)] for o in [o0, o0 + cnt),
// where A and B already point at their slab's bit pattern (B may be peer
// memory: NVLink loads/stores, or another process's slice on this GPU).  Up
// to kSwapJobs slab pairs per launch (blockIdx.y); 4 elements per thread per
// trip, every load in flight before the stores.
constexpr int kSwapJobs = 8;
struct SwapJobs {
    int n;
    double2* A[kSwapJobs];
    double2* B[kSwapJobs];
    uint64_t o0[kSwapJobs], cnt[kSwapJobs];
    SlabSpec sp;
};

__global__ void __launch_bounds__(256) k_slab_swap(const __grid_constant__ SwapJobs j) {
    constexpr int U = 4;
    const int job = blockIdx.y;
    double2* const A = j.A[job];
    double2* const B = j.B[job];
    const uint64_t o0 = j.o0[job], cnt = j.cnt[job];
    const uint64_t tile = uint64_t(blockDim.x) * U;
    for (uint64_t base = uint64_t(blockIdx.x) * tile; base < cnt; base += uint64_t(gridDim.x) * tile) {
        uint64_t idx[U];
        double2 x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t o = base + threadIdx.x + uint64_t(u) * blockDim.x;
            idx[u] = o < cnt ? depositAround(o0 + o, j.sp) : ~uint64_t(0);
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            if (idx[u] != ~uint64_t(0)) {
                x[u] = A[idx[u]];
                y[u] = B[idx[u]];
            }
#pragma unroll
        for (int u = 0; u < U; u++)
            if (idx[u] != ~uint64_t(0)) {
                A[idx[u]] = y[u];
                B[idx[u]] = x[u];
            }
    }
}

// buf[o - w0] = S[dep(o)] for o in [w0, w0 + cnt)  (S points at the slab pattern)
__global__ void __launch_bounds__(256) k_window_pack(double2* __restrict__ buf, const double2* __restrict__ S, uint64_t w0,
                                                     uint64_t cnt, const __grid_constant__ SlabSpec sp) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t o = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; o < cnt; o += stride)
        buf[o] = S[depositAround(w0 + o, sp)];
}

__global__ void __launch_bounds__(256) k_window_unpack(double2* __restrict__ S, const double2* __restrict__ buf,
                                                       uint64_t w0, uint64_t cnt, const __grid_constant__ SlabSpec sp) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t o = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; o < cnt; o += stride)
        S[depositAround(w0 + o, sp)] = buf[o];
}

// a[i] *= tab[sub(i)], sub bit (k-1-j) = bit tgt[j] of i: fused diagonals wider
// than a tile (k > 13 when chunk_qbit > 13).
struct DiagSpec {
    int k;
    int tgt[40];
};
__global__ void __launch_bounds__(256) k_diag_table(double2* __restrict__ a, const double2* __restrict__ tab, uint64_t n,
                                                    const __grid_constant__ DiagSpec d) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint64_t sub = 0;
        for (int j = 0; j < d.k; j++) sub |= ((i >> d.tgt[j]) & 1u) << (d.k - 1 - j);
        const double2 c = __ldg(tab + sub), x = a[i];
        a[i] = make_double2(fma(x.x, c.x, -x.y * c.y), fma(x.x, c.y, x.y * c.x));
    }
}

// ---- norm: per-thread compensated sums, fixed-order tree per block, then one
// block folds the partials in index order (bitwise deterministic).
__device__ __forceinline__ void twoSum(double& s, double& c, double x) {
    const double t = s + x;
    const double bp = t - s;
    c += (s - (t - bp)) + (x - bp);
    s = t;
}

__global__ void __launch_bounds__(256) k_norm_partial(const double2* __restrict__ a, uint64_t n, double* __restrict__ part) {
    __shared__ double ss[256], sc[256];
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = per * blockIdx.x, hi = lo + per < n ? lo + per : n;
    double s = 0, c = 0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double2 x = a[i];
        twoSum(s, c, fma(x.x, x.x, x.y * x.y));
    }
    ss[threadIdx.x] = s;
    sc[threadIdx.x] = c;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            double s2 = ss[threadIdx.x], c2 = sc[threadIdx.x] + sc[threadIdx.x + w];
            twoSum(s2, c2, ss[threadIdx.x + w]);
            ss[threadIdx.x] = s2;
            sc[threadIdx.x] = c2;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = ss[0];
        part[2 * blockIdx.x + 1] = sc[0];
    }
}

__global__ void k_norm_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0, c = 0;
        for (int b = 0; b < nb; b++) {
            twoSum(s, c, part[2 * b]);
            c += part[2 * b + 1];
        }
        out[0] = s + c;
    }
}

// Fold of per-tile sums of |a|^2 (written by a specialized pass with
// norm_out): same compensated fixed-order tree as k_norm_partial.
__global__ void __launch_bounds__(256) k_sum_partial(const double* __restrict__ x, uint64_t n, double* __restrict__ part) {
    __shared__ double ss[256], sc[256];
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = per * blockIdx.x, hi = lo + per < n ? lo + per : n;
    double s = 0, c = 0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) twoSum(s, c, x[i]);
    ss[threadIdx.x] = s;
    sc[threadIdx.x] = c;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            double s2 = ss[threadIdx.x], c2 = sc[threadIdx.x] + sc[threadIdx.x + w];
            twoSum(s2, c2, ss[threadIdx.x + w]);
            ss[threadIdx.x] = s2;
            sc[threadIdx.x] = c2;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = ss[0];
        part[2 * blockIdx.x + 1] = sc[0];
    }
}

__global__ void k_set_basis(double2* a, uint64_t idx, double v) { a[idx] = make_double2(v, 0.0); }

// Zeros at every i with ((i ^ val) & m) != 0: the tiles a sparse pass skips
// (outside its input's support), written as one coalesced stream of 32-B
// stores instead of tile by tile (tiles with short rows).
__global__ void __launch_bounds__(256) k_zero_outside(double2* __restrict__ a, uint64_t n, uint64_t m, uint64_t val) {
    const uint64_t stride = 2 * uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = 2 * (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x); i < n; i += stride) {
        const bool z0 = ((i ^ val) & m) != 0, z1 = (((i | 1) ^ val) & m) != 0;
        const double2 z = make_double2(0.0, 0.0);
        if (z0 && z1) {
            asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(a + i), "d"(0.0), "d"(0.0), "d"(0.0), "d"(0.0)
                         : "memory");
        } else {
            if (z0) __stcs(a + i, z);
            if (z1) __stcs(a + i + 1, z);
        }
    }
}

// Marginal probabilities over k <= 10 slice bits: part[block][v] = sum of
// |a_i|^2 over this block's range with bits(i) = v (bit j of v = slice bit
// bits[j]).  Shared-memory atomics within a block; blocks fold in order.
struct MargSpec {
    int k;
    int bits[10];
};
__global__ void __launch_bounds__(256) k_marginal_partial(const double2* __restrict__ a, uint64_t n,
                                                          const __grid_constant__ MargSpec m, double* __restrict__ part) {
    __shared__ double bins[1024];
    const int nb = 1 << m.k;
    for (int v = threadIdx.x; v < nb; v += blockDim.x) bins[v] = 0.0;
    __syncthreads();
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = per * blockIdx.x, hi = lo + per < n ? lo + per : n;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double2 x = __ldcs(a + i);
        int v = 0;
        for (int j = 0; j < m.k; j++) v |= int((i >> m.bits[j]) & 1u) << j;
        atomicAdd(&bins[v], fma(x.x, x.x, x.y * x.y));
    }
    __syncthreads();
    for (int v = threadIdx.x; v < nb; v += blockDim.x) part[uint64_t(blockIdx.x) * nb + v] = bins[v];
}
__global__ void k_marginal_final(const double* __restrict__ part, int nblocks, int nb, double* __restrict__ out) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nb; v += gridDim.x * blockDim.x) {
        double s = 0.0, c = 0.0;  // compensated, fixed block order
        for (int b = 0; b < nblocks; b++) {
            const double y = part[uint64_t(b) * nb + v] - c, t = s + y;
            c = (t - s) - y;
            s = t;
        }
        out[v] = s;
    }
}

// ---- launchers ----------------------------------------------------------------

static unsigned gridFor(uint64_t work, unsigned threads, unsigned cap) {
    uint64_t g = (work + threads - 1) / threads;
    if (g > cap) g = cap;
    return unsigned(g ? g : 1);
}

cudaError_t launchImsGeneric(double2* a, int logN, const int* outs, const int* ins, int s, cudaStream_t st) {
    PairSpec p{};
    p.s = s;
    for (int j = 0; j < s; j++) {
        p.out[j] = outs[j];
        p.in[j] = ins[j];
    }
    // 2^logT threads, each walking 2^(logN-logT) elements.
    int logT = logN < 20 ? logN : 20;
    if (logT < 0) logT = 0;
    const uint64_t T = uint64_t(1) << logT;
    const unsigned threads = T < 256 ? unsigned(T) : 256u;
    k_ims<<<unsigned(T / threads), threads, 0, st>>>(a, logN, logT, p);
    return cudaGetLastError();
}

// Tiled IMS when the slice has >= 6 bits and a P-closed 5..6-bit tile exists.
static bool imsTileSpec(int logN, const int* outs, const int* ins, int s, ImsTileSpec& sp) {
    if (logN < 6) return false;
    int partner[64];
    for (int b = 0; b < 64; b++) partner[b] = b;
    for (int j = 0; j < s; j++) {
        partner[outs[j]] = ins[j];
        partner[ins[j]] = outs[j];
    }
    // T: memory bits 0..2 and their partners, then the lowest bits (with
    // partners) up to 8 bits: longer contiguous rows (bits 0..L-1) first.
    uint64_t T = 0;
    for (int b = 0; b < 3; b++) T |= (uint64_t(1) << b) | (uint64_t(1) << partner[b]);
    if (__builtin_popcountll(T) > 8) return false;
    for (int b = 0; b < logN && __builtin_popcountll(T) < 8; b++) {
        if ((T >> b) & 1) continue;
        const uint64_t add = (uint64_t(1) << b) | (uint64_t(1) << partner[b]);
        if (__builtin_popcountll(T | add) <= 8) T |= add;
    }
    const int k = __builtin_popcountll(T);
    if (k < 5 || k > logN - 1) return false;
    sp = ImsTileSpec{};
    sp.k = k;
    sp.n = logN;
    int coord[64];
    int r = 0;
    for (int b = 0; b < logN; b++)
        if ((T >> b) & 1) {
            coord[b] = r;
            sp.tbit[r++] = b;
        }
    for (int q = 0; q < k; q++) sp.pi[q] = coord[partner[sp.tbit[q]]];
    sp.piIdentity = 1;
    for (int q = 0; q < k; q++) sp.piIdentity &= sp.pi[q] == q;
    for (int b = 0; b < logN; b++)
        if (!((T >> b) & 1)) sp.fbit[sp.nfree++] = b;
    for (int j = 0; j < s; j++)
        if (!((T >> outs[j]) & 1)) {
            sp.ho[sp.nhp] = outs[j];
            sp.hi[sp.nhp] = ins[j];
            sp.nhp++;
        }
    sp.a = sp.nfree < 16 ? sp.nfree : 16;  // 65536 warps: ~9 waves of resident CTAs (small tail)
    auto depFree = [&](uint64_t g) {
        uint64_t h = 0;
        for (int j = 0; j < sp.nfree; j++) h |= ((g >> j) & 1) << sp.fbit[j];
        return h;
    };
    auto Ph = [&](uint64_t h) {
        for (int j = 0; j < sp.nhp; j++) {
            const uint64_t d = ((h >> sp.ho[j]) ^ (h >> sp.hi[j])) & 1u;
            h ^= (d << sp.ho[j]) | (d << sp.hi[j]);
        }
        return h;
    };
    for (int j = 0; j + sp.a < sp.nfree && j < 58; j++) {
        const uint64_t m = ((uint64_t(2) << j) - 1) << sp.a;
        sp.hstep[j] = depFree(m);
        sp.pstep[j] = Ph(sp.hstep[j]);
    }
    // Swizzle: bank(u) = (u & 7) ^ sum_i bit_{3+i}(u) * swz[i] must be
    // injective on the lane patterns of the writes (span of coordinate bits
    // 0..2, always) and of the permuted reads (span of pi(0..2)).
    int img[3];
    for (int i = 0; i < 3; i++) img[i] = 1 << sp.pi[i];
    for (int m = 0; m < (1 << 15); m++) {
        const int z[5] = {m & 7, (m >> 3) & 7, (m >> 6) & 7, (m >> 9) & 7, (m >> 12) & 7};
        auto bank = [&](int u) {
            int x = u & 7;
            for (int i = 0; i < 5; i++)
                if ((u >> (3 + i)) & 1) x ^= z[i];
            return x;
        };
        bool ok = true;
        for (int c = 1; c < 8 && ok; c++) {
            int u = 0;
            for (int i = 0; i < 3; i++)
                if ((c >> i) & 1) u ^= img[i];
            ok = bank(u) != 0;
        }
        if (ok) {
            for (int i = 0; i < 5; i++) sp.swz[i] = z[i];
            break;
        }
    }
    return true;
}

// QK_IMS_TILED: 0 = always the per-element kernel, 1 (default) = tiled
// whenever possible (2^8-amplitude tiles: 6.2-6.5 TB/s on every pair pattern
// measured), 2 = tiled only when a pair moves memory bit 0 or 1.
static int g_imsMode = -1;  // -1: not set yet (QK_IMS_TILED, default 1)
static int imsMode() {
    if (g_imsMode < 0) {
        const char* e = std::getenv("QK_IMS_TILED");
        g_imsMode = e ? std::atoi(e) : 1;
    }
    return g_imsMode;
}
void setImsMode(int v) { g_imsMode = v; }

cudaError_t launchIms(double2* a, int logN, const int* outs, const int* ins, int s, cudaStream_t st) {
    ImsTileSpec sp;
    bool lowPair = false;
    for (int j = 0; j < s; j++) lowPair |= outs[j] < 2 || ins[j] < 2;  // sub-64-B neighbours move apart
    const int mode = imsMode();
    if (mode == 0 || (mode == 2 && !lowPair) || !imsTileSpec(logN, outs, ins, s, sp))
        return launchImsGeneric(a, logN, outs, ins, s, st);
    const uint64_t ctas = ((uint64_t(1) << sp.a) + 7) / 8;  // 8 warps per CTA
    const unsigned threads = sp.a >= 3 ? 256 : (32 << sp.a);
    const int per = 1 << (sp.k - 5);
    const size_t smem = size_t(threads / 32) * 2 * 32 * per * sizeof(double2);
    switch (per) {
        case 1: k_ims_tiled<1, 4><<<unsigned(ctas), threads, smem, st>>>(a, sp); break;
        case 2: k_ims_tiled<2, 2><<<unsigned(ctas), threads, smem, st>>>(a, sp); break;
        case 4: k_ims_tiled<4, 1><<<unsigned(ctas), threads, smem, st>>>(a, sp); break;
        default: {
            cudaError_t e = cudaFuncSetAttribute(k_ims_tiled<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            if (e != cudaSuccess) return e;
            k_ims_tiled<8, 1><<<unsigned(ctas), threads, smem, st>>>(a, sp);
        }
    }
    return cudaGetLastError();
}

// n slab pairs (A[k], B[k]) swapped over element ranges [o0[k], o0[k] + cnt[k]).
cudaError_t launchSlabSwap(int n, double2* const* A, double2* const* B, const uint64_t* o0, const uint64_t* cnt,
                           const int* outsSorted, int s, cudaStream_t st) {
    for (int first = 0; first < n; first += kSwapJobs) {
        SwapJobs j{};
        j.n = n - first < kSwapJobs ? n - first : kSwapJobs;
        j.sp.s = s;
        for (int q = 0; q < s; q++) j.sp.outs[q] = outsSorted[q];
        uint64_t most = 0;
        for (int k = 0; k < j.n; k++) {
            j.A[k] = A[first + k];
            j.B[k] = B[first + k];
            j.o0[k] = o0[first + k];
            j.cnt[k] = cnt[first + k];
            if (j.cnt[k] > most) most = j.cnt[k];
        }
        if (!most) continue;
        const unsigned gx = gridFor((most + 3) / 4, 256, (148u * 8u + unsigned(j.n) - 1) / unsigned(j.n));
        k_slab_swap<<<dim3(gx, unsigned(j.n)), 256, 0, st>>>(j);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launchWindowPack(double2* buf, const double2* S, uint64_t w0, uint64_t cnt, const int* outsSorted, int s,
                             cudaStream_t st) {
    SlabSpec sp{};
    sp.s = s;
    for (int j = 0; j < s; j++) sp.outs[j] = outsSorted[j];
    k_window_pack<<<gridFor(cnt, 256, 148 * 16), 256, 0, st>>>(buf, S, w0, cnt, sp);
    return cudaGetLastError();
}

cudaError_t launchWindowUnpack(double2* S, const double2* buf, uint64_t w0, uint64_t cnt, const int* outsSorted, int s,
                               cudaStream_t st) {
    SlabSpec sp{};
    sp.s = s;
    for (int j = 0; j < s; j++) sp.outs[j] = outsSorted[j];
    k_window_unpack<<<gridFor(cnt, 256, 148 * 16), 256, 0, st>>>(S, buf, w0, cnt, sp);
    return cudaGetLastError();
}

cudaError_t launchDiagTable(double2* a, const double2* tab, uint64_t n, const int* tgt, int k, cudaStream_t st) {
    DiagSpec d{};
    d.k = k;
    for (int j = 0; j < k; j++) d.tgt[j] = tgt[j];
    k_diag_table<<<gridFor(n, 256, 148 * 16), 256, 0, st>>>(a, tab, n, d);
    return cudaGetLastError();
}

constexpr int kNormBlocks = 1184;  // 148 SMs x 8

cudaError_t launchNorm(const double2* a, uint64_t n, double* scratch, double* out, cudaStream_t st) {
    k_norm_partial<<<kNormBlocks, 256, 0, st>>>(a, n, scratch);
    k_norm_final<<<1, 32, 0, st>>>(scratch, kNormBlocks, out);
    return cudaGetLastError();
}
size_t normScratchDoubles() { return 2 * kNormBlocks; }

cudaError_t launchSumTiles(const double* x, uint64_t n, double* scratch, double* out, cudaStream_t st) {
    k_sum_partial<<<kNormBlocks, 256, 0, st>>>(x, n, scratch);
    k_norm_final<<<1, 32, 0, st>>>(scratch, kNormBlocks, out);
    return cudaGetLastError();
}

constexpr int kMargBlocks = 1184;
size_t marginalScratchDoubles(int k) { return size_t(kMargBlocks) << k; }
cudaError_t launchMarginal(const double2* a, uint64_t n, const int* bits, int k, double* scratch, double* out,
                           cudaStream_t st) {
    MargSpec m{};
    m.k = k;
    for (int j = 0; j < k; j++) m.bits[j] = bits[j];
    k_marginal_partial<<<kMargBlocks, 256, 0, st>>>(a, n, m, scratch);
    k_marginal_final<<<((1 << k) + 255) / 256, 256, 0, st>>>(scratch, kMargBlocks, 1 << k, out);
    return cudaGetLastError();
}

cudaError_t launchZeroOutside(double2* a, uint64_t n, uint64_t m, uint64_t val, int smCount, cudaStream_t st) {
    k_zero_outside<<<unsigned(smCount) * 8u, 256, 0, st>>>(a, n, m, val);
    return cudaGetLastError();
}

cudaError_t launchSetBasis(double2* a, uint64_t idx, cudaStream_t st, double v) {
    k_set_basis<<<1, 1, 0, st>>>(a, idx, v);
    return cudaGetLastError();
}

}  // namespace qkdev
