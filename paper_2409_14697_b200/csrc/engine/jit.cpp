// Straight-line pass specialization: PassParams -> CUDA C++ -> NVRTC cubin.
//
// Emits exactly the semantics of k_block_pass (block_pass.cu) for one
// PassParams, with everything the interpreter decides at run time resolved
// at generation time: the op switch disappears, coefficients become
// literals, register swaps (CX with a register control) become variable
// renames, and deferred factors that are statically untouched are skipped.
// The whole pass is one basic block per segment, so ptxas schedules the
// independent amplitude updates of consecutive gates together (ILP the
// interpreter's per-op dispatch cannot give).
#include "jit.h"

#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>
#include <nvrtc.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <thread>

#include "quokka/common.hpp"

namespace qkjit {

using qkdev::DevOp;
using qkdev::PassParams;
using quokka::SimulationError;

bool nvrtcSupportsWideAccess();  // NVRTC >= 12.9 (sm_100 256-bit accesses)

namespace {

std::string lit(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%a", v);
    return buf;
}

std::string c2(double re, double im) { return "C2(" + lit(re) + "," + lit(im) + ")"; }

uint32_t swzHost(uint32_t u) { return u ^ (((u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12)) & 7u); }

const char* kPrologue = R"(
#include <cuda_runtime.h>
typedef unsigned long long u64;
typedef unsigned int u32;
#define C2(r, i) make_double2((r), (i))
static __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
static __device__ __forceinline__ double2 cmac(double2 acc, double2 m, double2 x) {
    acc.x = fma(m.x, x.x, acc.x); acc.x = fma(-m.y, x.y, acc.x);
    acc.y = fma(m.x, x.y, acc.y); acc.y = fma(m.y, x.x, acc.y);
    return acc;
}
// Literal coefficients with a zero part (the generator picks these): real r,
// imaginary i.  Same results as cmul / cmac up to the sign of zero.
static __device__ __forceinline__ double2 cmulr(double2 a, double r) { return make_double2(a.x * r, a.y * r); }
static __device__ __forceinline__ double2 cmuli(double2 a, double i) { return make_double2(-(a.y * i), a.x * i); }
static __device__ __forceinline__ double2 cmacr(double2 acc, double r, double2 x) {
    return make_double2(fma(r, x.x, acc.x), fma(r, x.y, acc.y));
}
static __device__ __forceinline__ double2 cmaci(double2 acc, double i, double2 x) {
    return make_double2(fma(-i, x.y, acc.x), fma(i, x.x, acc.y));
}
static __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
static __device__ __forceinline__ double2 cinv(double2 a) {
    const double d = 1.0 / fma(a.x, a.x, a.y * a.y);
    return make_double2(a.x * d, -a.y * d);
}
static __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
static __device__ __forceinline__ double2 csel(bool c, double2 x, double2 y) {
    return make_double2(c ? x.x : y.x, c ? x.y : y.y);
}
static __device__ __forceinline__ u32 swz(u32 u) { return u ^ (((u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12)) & 7u); }
// 256-bit global accesses (two neighbouring amplitudes), sm_100.
static __device__ __forceinline__ void ld256(const double2* p, double2& lo, double2& hi) {
#ifdef __CUDA_ARCH__
    asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(lo.x), "=d"(lo.y), "=d"(hi.x), "=d"(hi.y) : "l"(p));
#else
    lo = p[0]; hi = p[1];
#endif
}
static __device__ __forceinline__ void st256(double2* p, const double2& lo, const double2& hi) {
#ifdef __CUDA_ARCH__
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(lo.x), "d"(lo.y), "d"(hi.x), "d"(hi.y) : "memory");
#else
    p[0] = lo; p[1] = hi;
#endif
}
// TMA bulk copies into shared memory, tracked by an mbarrier (host builds of
// the generated source, tests/host/jit_host_shim.h, copy synchronously).
static __device__ __forceinline__ u32 smem_u32(const void* p) {
#ifdef __CUDA_ARCH__
    return (u32)__cvta_generic_to_shared(p);
#else
    return 0u;
#endif
}
static __device__ __forceinline__ void mbar_init(u64* m) {
#ifdef __CUDA_ARCH__
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#endif
}
static __device__ __forceinline__ void mbar_expect_tx(u64* m, u32 bytes) {
#ifdef __CUDA_ARCH__
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
#endif
}
static __device__ __forceinline__ void mbar_wait(u64* m, u32 phase) {
#ifdef __CUDA_ARCH__
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
                 ::"r"(smem_u32(m)), "r"(phase) : "memory");
#else
    __syncthreads();  // host replay: the synchronous copies are done once every thread is here
#endif
}
static __device__ __forceinline__ void fence_async() {
#ifdef __CUDA_ARCH__
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
}
static __device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* m) {
#ifdef __CUDA_ARCH__
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)) : "memory");
#else
    memcpy(dst, src, bytes);
#endif
}
// TMA bulk store of a contiguous shared-memory row to global memory (async
// proxy, bulk group of the issuing thread), and the group waits.
static __device__ __forceinline__ void bulk_s2g(void* dst, const void* src, u32 bytes) {
#ifdef __CUDA_ARCH__
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
#else
    memcpy(dst, src, bytes);
#endif
}
static __device__ __forceinline__ void bulk_commit() {
#ifdef __CUDA_ARCH__
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
#endif
}
static __device__ __forceinline__ void bulk_wait_read() {  // sources of committed stores may be reused
#ifdef __CUDA_ARCH__
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
}
// The tile as one box of a tensor view of the slice (cuTensorMapEncodeTiled,
// built by launch()); passed to the TMA-pipelined kernels by value.
struct __align__(64) QkTmap {
    unsigned long long v[16];
};
static __device__ __forceinline__ void bulk_wait_read1() {  // all but the newest group have left shared memory
#ifdef __CUDA_ARCH__
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
#endif
}
static __device__ __forceinline__ void bulk_wait_all() {
#ifdef __CUDA_ARCH__
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
}
// One line of the next tile's support into L2 (sparse runs, persistent grid).
static __device__ __forceinline__ void pf_line(const void* p) {
#ifdef __CUDA_ARCH__
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#endif
}
// TMA-engine prefetch of a contiguous row into L2 (no registers, no smem).
static __device__ __forceinline__ void pf_l2(const void* p, u32 bytes) {
#ifdef __CUDA_ARCH__
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
#endif
}
)";

// Tuning knobs (read once): QK_JIT_PERSIST=1 launches a persistent grid (one
// CTA per SM walking tiles) instead of one CTA per tile; QK_JIT_PF=0 then
// disables its L2 prefetch of the next tile.  Measured on QFT-33 (B200): one
// CTA per tile 305 ms of passes, persistent 325 ms, persistent + prefetch 342 ms.
int knob(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}
bool usePersistent() {
    static const bool v = knob("QK_JIT_PERSIST", 0) != 0;
    return v;
}
bool usePrefetch() {
    static const bool v = usePersistent() && knob("QK_JIT_PF", 1) != 0;
    return v;
}
// QK_JIT_PF_SPARSE (default 1; persistent grids: the TMA-pipelined form, and
// the plain form under QK_JIT_PERSIST=1): in a run with known zeros, each
// thread prefetches into L2 the support amplitudes its slots will read in the
// CTA's next tile, so the next tile's loads do not wait on HBM.
bool useSparsePrefetch() {
    static const bool v = knob("QK_JIT_PF_SPARSE", 1) != 0;
    return v;
}

// Per-CTA factors as straight-line code with literal terms, or as a loop over
// device term tables.  QK_CTA_LITERAL=1 / 0 forces one form; by default a
// pass with more than QK_CTA_LITERAL_MAX (128) terms takes the tables: the
// literal code of QAOA's passes (92-473 terms) misses the instruction cache
// (ncu: no_instructions 24 %).  Measured at 33 qubits: all-table QAOA 284 ->
// 273 ms but random (<= 28 terms per pass) 639 -> 660 ms.
bool literalFactors(const PassParams& P) {
    static const int force = knob("QK_CTA_LITERAL", -1), cap = knob("QK_CTA_LITERAL_MAX", 128);
    if (force >= 0) return force != 0;
    return !P.ncta || P.cta_end[P.ncta - 1] <= cap;
}

// QK_JIT_TMAP (default 1): the TMA-pipelined kernels move a tile with one
// tensor-map op (cuTensorMapEncodeTiled) instead of one bulk copy per row.
bool useTensorMaps() {
    static const bool v = knob("QK_JIT_TMAP", 1) != 0;
    return v;
}

// Resident CTAs per SM of a pass kernel (register / shared-memory bound).
int blocksPerSm(int ct, int rb) { return (ct == 12 && rb >= 4) ? 2 : ct <= 11 ? 2 : 1; }

int smCount(int dev) {
    static std::mutex mu;
    static std::map<int, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
    return n;
}

// Contiguous low tile bits (tile bit j == memory bit j): the tile's row length.
int lowRun(const PassParams& P) {
    int L = 0;
    while (L < P.ct && P.tile_phys[L] == L) L++;
    return L;
}

// The tile as a box of a <= 5-D tensor view of the slice in doubles:
// dimension d spans memory bits [lo[d], lo[d+1]) (the last one up to the
// slice's top bit) and the box its low tb[d] bits, which are tile bits (<= 8
// per dimension, <= cap0 <= 7 in dimension 0 whose elements are the two
// halves of an amplitude).  Returns the rank, 0 when the tile needs more than 5
// dimensions or does not hold memory bits 0-2 (rows under 128 B).
int tensorDims(const PassParams& P, int lo[5], int tb[5], int cap0 = 7) {
    if (lowRun(P) < 3) return 0;
    int nd = 0;
    for (int j = 0; j < P.ct;) {
        const int start = P.tile_phys[j], cap = nd == 0 ? cap0 : 8;
        int len = 1;
        while (j + len < P.ct && P.tile_phys[j + len] == start + len && len < cap) len++;
        if (nd == 5) return 0;
        lo[nd] = start;
        tb[nd] = len;
        nd++;
        j += len;
    }
    for (int d = 0; d + 1 < nd; d++)
        if (lo[d + 1] - lo[d] + (d == 0 ? 1 : 0) > 32) return 0;  // extents <= 2^32
    return nd;
}

// TMA-pipelined form (an autotune variant of every 2^13-tile pass; the default
// for all passes under QK_JIT_TMA=1): a persistent CTA per SM keeps the NEXT
// tile streaming into a 128 KB shared-memory buffer PB (one tensor-map TMA
// load per tile, swizzled, mbarrier) while the current tile computes in
// registers, and in runs with known zeros stages its output tile in PB for
// one TMA store that drains while the next tile computes; exchanges run in
// two halves through a 64 KB buffer, split on a tile bit that stays in the
// same register slot (schedule.cpp guarantees one).  Needs 2^13 tiles, 32
// amplitudes per thread and >= 128-B rows.  Measured on B200 (QFT / QAOA /
// Grover at 33 qubits) it loses to the plain kernel by 5-30 %: the
// half-splittable exchanges cost extra segments (QFT pass 3: 3 instead of 2).
bool pipelined(const PassParams& P) {
    if (!P.half_x || P.ct != 13 || P.rb != 5 || lowRun(P) < 3) return false;
    for (int c = 1; c < P.nsegs; c++) {
        const int k = P.xsplit[c];
        if (k >= P.rb || P.map_out[c - 1][k] != P.map_in[c][k] || P.map_out[c - 1][k] < 3) return false;
    }
    return true;
}
}  // namespace
bool pipelinedPass(const PassParams& P) { return pipelined(P); }

// Shared-memory wavefronts of one tile's warp-wide 16-byte accesses to PB
// (every register slot, warp 0; other warps differ by a constant XOR) when
// the amplitude at tile coordinate u sits at chunk u ^ ((u >> 3) & (2^mode -
// 1)): a phase is 8 consecutive lanes and costs the largest number of
// distinct chunks sharing a bank group.
int pbWavefronts(const PassParams& P, const uint8_t* m, int mode) {
    const uint32_t msk = (1u << mode) - 1;
    int total = 0;
    for (int s = 0; s < (1 << P.rb); s++) {
        uint32_t us = 0;
        for (int k = 0; k < P.rb; k++)
            if ((s >> k) & 1) us |= 1u << m[k];
        for (int ph = 0; ph < 4; ph++) {
            uint32_t chunk[8];
            for (int l = 0; l < 8; l++) {
                const uint32_t lane = uint32_t(ph * 8 + l);
                uint32_t u = us;
                for (int j = 0; j < 5 && j < P.ct - P.rb; j++) u |= ((lane >> j) & 1u) << m[P.rb + j];
                chunk[l] = u ^ ((u >> 3) & msk);
            }
            int worst = 0;
            for (int g = 0; g < 8; g++) {
                int distinct = 0;
                for (int l = 0; l < 8; l++) {
                    if ((chunk[l] & 7u) != uint32_t(g)) continue;
                    bool seen = false;
                    for (int e = 0; e < l; e++) seen = seen || chunk[e] == chunk[l];
                    distinct += seen ? 0 : 1;
                }
                worst = std::max(worst, distinct);
            }
            total += worst;
        }
    }
    return total;
}

// QK_STAGED_STORES (default 1): in runs with known zeros the plain kernel
// writes its output tile through shared memory and the TMA engine instead of
// register stores (stagedLayout).
bool stagedStores() {
    static const bool v = knob("QK_STAGED_STORES", 1) != 0;
    return v;
}

// The plain kernel's staged output: the tile leaves as two half boxes of a
// tensor view of the slice, split on its top tile bit -- half 0 staged in a
// half-tile buffer S and drained across the whole next tile, half 1 in the
// exchange buffer and drained before the next tile's first exchange -- so the
// SM computes the next tile while the TMA engine writes this one (register
// stores serialize with the compute: profiles/r2_store_path_probe.txt).
// Rank 0: register stores only.  The swizzle minimizes the staging writes'
// bank conflicts.
int stagedLayout(const PassParams& P, int lo[5], int tb[5], int* swizzle) {
    *swizzle = 0;
    if (!stagedStores() || !P.stage_out || pipelined(P) || P.ct != 13) return 0;  // 2^12 tiles: two CTAs per SM overlap already
    int best = -1, bestNd = 0;
    for (int mode = 0; mode <= 3; mode++) {
        int l[5], t[5];
        const int nd = tensorDims(P, l, t, mode ? mode : 7);
        if (!nd) continue;
        const int cost = pbWavefronts(P, P.map_out[P.nsegs - 1], mode);
        if (best >= 0 && cost >= best) continue;
        best = cost;
        bestNd = nd;
        *swizzle = mode;
        std::memcpy(lo, l, sizeof l);
        std::memcpy(tb, t, sizeof t);
    }
    return bestNd;
}
// QK_JIT_PERSIST=1 with QK_JIT_PF (default 1): a dense-input 2^13-tile pass
// runs on a persistent grid and prefetches its CTA's next tile into L2 with
// two tensor-map TMA prefetches.  Off by default: measured at 33 qubits,
// random 638 -> 615 ms but QAOA 285 -> 326 ms; as a per-pass autotune
// variant (rb 5 only) it gained nothing (random 640, QAOA 287 ms).
bool prefetchTiles(const PassParams& P) { return usePrefetch() && P.ct == 13 && !pipelined(P); }
bool stagedPass(const PassParams& P) {
    int lo[5], tb[5], swizzle;
    return stagedLayout(P, lo, tb, &swizzle) > 0;
}

// The TMA-pipelined kernel's tensor view: rank (0: rows only) and the PB
// swizzle (0 none, 1 / 2 / 3: the 32 / 64 / 128-byte hardware patterns) with
// the fewest shared-memory wavefronts for the tile's reads (dense runs) and
// staged writes (sparse runs).  A swizzle limits dimension 0 to its span.
int tensorLayout(const PassParams& P, int lo[5], int tb[5], int* swizzle) {
    *swizzle = 0;
    if (!pipelined(P)) return 0;
    int best = -1, bestNd = 0;
    for (int mode = 0; mode <= 3; mode++) {
        int l[5], t[5];
        const int nd = tensorDims(P, l, t, mode ? mode : 7);
        if (!nd) continue;
        const int cost = pbWavefronts(P, P.map_in[0], mode) + pbWavefronts(P, P.map_out[P.nsegs - 1], mode);
        if (best >= 0 && cost >= best) continue;
        best = cost;
        bestNd = nd;
        *swizzle = mode;
        std::memcpy(lo, l, sizeof l);
        std::memcpy(tb, t, sizeof t);
    }
    return bestNd;
}
int lowRunOf(const PassParams& P) { return lowRun(P); }
namespace {
constexpr int kPipeSmemAmps = (1 << 13) + (1 << 12) + qkdev::kMaxCtaFactors + 1;  // PB | XS | F | mbarrier

// Dynamic shared memory of a pass kernel: PB | XS | F | mbarrier (pipelined),
// exchange buffer [| S] | F (plain).
unsigned kernelSmem(const PassParams& P) {
    if (pipelined(P)) return unsigned(sizeof(double2) * kPipeSmemAmps);
    int lo[5], tb[5], swizzle;
    const bool staged = stagedLayout(P, lo, tb, &swizzle) > 0;
    return unsigned((sizeof(double2) << P.ct) + (staged ? sizeof(double2) << (P.ct - 1) : 0) +
                    sizeof(double2) * qkdev::kMaxCtaFactors + 256);
}

class Gen {
public:
    explicit Gen(const PassParams& P)
        : P_(P), ct_(P.ct), rb_(P.rb), na_(1 << P.rb), nt_(1 << (P.ct - P.rb)), pipe_(pipelined(P)) {
        for (int s = 0; s < na_; s++) nm_.push_back(s);
    }

    // Persistent kernel: each CTA walks tiles blockIdx.x, +gridDim.x, ...  While
    // tile k computes, the rows of the CTA's next tile are prefetched into L2
    // by the TMA engine, so that tile's register loads hit L2 and the SM's
    // load phase overlaps its compute phase (one CTA per SM at ct = 13).
    std::string run(const std::string& name) {
        if (pipe_) return runPipelined(name);
        const int minb = blocksPerSm(ct_, rb_);
        o_ << kPrologue;
        ctaTables();
        o_ << "extern \"C\" __global__ void __launch_bounds__(" << nt_ << "," << minb << ") " << name
           << "(double2* __restrict__ st, const double2* __restrict__ gt, const u32 ntiles, const u64 basis, const u32 tile0, double* __restrict__ np, const u64 smask, const u64 sval, const u32 zskip, const __grid_constant__ QkTmap tm, const u32 tmv) {\n";
        tmNd_ = stagedLayout(P_, tmLo_, tmTb_, &tmSwz_);
        staged_ = tmNd_ > 0;
        if (!staged_ && prefetchTiles(P_)) tmNd_ = tensorDims(P_, tmLo_, tmTb_);  // the next tile's L2 prefetch only
        if (staged_)  // exchange buffer | S (half tile) | F
            o_ << "  extern __shared__ double2 sm[];\n  double2* const S = sm + " << (1 << ct_) << ";\n  double2* const F = sm + "
               << (3 << (ct_ - 1)) << ";\n  const u32 tid = threadIdx.x;\n"
               << "#ifdef __CUDA_ARCH__\n  const bool stg_ = " << (P_.stage_out == 2 ? "" : "smask != 0ull && ")
               << "tmv != 0u;\n#else\n  const bool stg_ = " << (P_.stage_out == 2 ? "true" : "smask != 0ull") << ";\n#endif\n";
        else
            o_ << "  extern __shared__ double2 sm[];\n  double2* const F = sm + " << (1 << ct_)
               << ";\n  const u32 tid = threadIdx.x;\n";
        hoistTables();
        o_ << "  for (u32 tile = blockIdx.x + tile0; tile < ntiles; tile += gridDim.x) {\n";
        o_ << "  " << tileBase() << "\n";
        zeroTile();
        std::string decl = "  double2 ";
        for (int s = 0; s < na_; s++) decl += (s ? ", a" : "a") + std::to_string(s);
        o_ << decl << ";\n  double2 P = C2(1.0, 0.0);\n" << pendDecl();
        // load (map_in[0], no flips).  smask != 0: the input is zero outside
        // the coset {i : (i ^ sval) & smask == 0} (a run from a basis state,
        // before its passes have touched every bit): only those amplitudes
        // are read, the rest are zeros that need no memory.
        o_ << "  { const u64 off = base | " << threadGlobal(P_.map_in[0]) << ";\n  if (smask != 0ull) {\n";
        sparseLoads("  ");
        o_ << "  } else if (basis == ~0ull) {\n";
        const int kl = slotOfMem0(P_.map_in[0]);
        for (int s = 0; s < na_; s++) {
            if (kl >= 0) {  // neighbours (slot kl = 0 / 1) in one 256-bit load
                if (!((s >> kl) & 1))
                    o_ << "  ld256(st + (off | " << regGlobal(P_.map_in[0], s) << "ull), a" << s << ", a" << (s | (1 << kl))
                       << ");\n";
                continue;
            }
            o_ << "  a" << s << " = __ldcs(st + (off | " << regGlobal(P_.map_in[0], s) << "ull));\n";
        }
        o_ << "  } else {  // first pass of a run: synthesize |basis> instead of reading it\n";
        for (int s = 0; s < na_; s++)
            o_ << "  a" << s << " = C2((off | " << regGlobal(P_.map_in[0], s) << "ull) == basis ? " << lit(P_.synth_amp ? P_.synth_amp : 1.0) << " : 0.0, 0.0);\n";
        o_ << "  }\n  }\n";
        prefetchNext();
        ctaFactors();

        for (int i = 0; i < P_.nops; i++) op(P_.ops[i]);

        // store (map_out[last] with flips)
        const int last = P_.nsegs - 1;
        uint64_t gx = 0;
        for (int j = 0; j < ct_; j++)
            if ((P_.xmask_out[last] >> j) & 1) gx |= uint64_t(1) << P_.tile_phys[j];
        // Single-segment pass whose store map differs from its load map: other
        // threads may still be loading the addresses this thread stores to.
        if (P_.nsegs == 1 && (std::memcmp(P_.map_in[0], P_.map_out[0], sizeof P_.map_in[0]) != 0 || P_.xmask_out[0]))
            o_ << "  __syncthreads();\n";
        if (P_.norm_out) emitNorm();
        if (staged_) {
            stageHalves(last);
            o_ << "  } else\n";
        }
        o_ << "  { const u64 off = (base | " << threadGlobal(P_.map_out[last]) << ") ^ " << gx << "ull;\n";
        const int ks = slotOfMem0(P_.map_out[last]);
        for (int s = 0; s < na_; s++) {
            if (ks >= 0) {  // slot ks stores memory bit 0: neighbours in one 256-bit store
                if ((s >> ks) & 1) continue;
                const int s1 = s | (1 << ks);
                const bool swap = gx & 1;  // memory bit 0 flipped: slot value 0 lands on the odd address
                o_ << "  st256(st + ((off ^ " << regGlobal(P_.map_out[last], s) << "ull) & ~1ull), a"
                   << nm_[size_t(swap ? s1 : s)] << ", a" << nm_[size_t(swap ? s : s1)] << ");\n";
                continue;
            }
            o_ << "  __stcs(st + (off ^ " << regGlobal(P_.map_out[last], s) << "ull), a" << nm_[size_t(s)] << ");\n";
        }
        o_ << "  }\n";
        // The next iteration's first shared-memory write must not overtake a
        // slow thread still reading this tile's last exchange.
        o_ << "  if (tile + gridDim.x < ntiles) __syncthreads();\n  }\n";
        if (staged_) o_ << "  if (tid == 0u) bulk_wait_all();\n";
        o_ << "}\n";
        return o_.str();
    }

    std::string runPipelined(const std::string& name) {
        const int L = lowRun(P_);
        tensorView();
        o_ << kPrologue;
        ctaTables();
        o_ << "extern \"C\" __global__ void __launch_bounds__(" << nt_ << ",1) " << name
           << "(double2* __restrict__ st, const double2* __restrict__ gt, const u32 ntiles, const u64 basis, const u32 tile0, double* __restrict__ np, const u64 smask, const u64 sval, const u32 zskip, const __grid_constant__ QkTmap tm, const u32 tmv) {\n"
           << "  extern __shared__ double2 sm[];  // PB: next tile (linear tile coordinates) | XS | F | mbarrier\n"
           << "  double2* const XS = sm + 8192;\n  double2* const F = sm + 12288;\n"
           << "  u64* const mbar = (u64*)(sm + " << (12288 + qkdev::kMaxCtaFactors) << ");\n  const u32 tid = threadIdx.x;\n"
           << "  const bool tma = basis == ~0ull && smask == 0ull;  // sparse runs: no whole-tile streaming\n  u32 phase = 0u;\n"
           << "  if (tid == 0) mbar_init(mbar);\n  __syncthreads();\n";
        hoistTables();
        o_ << ""
           << "  if (tma && blockIdx.x < ntiles) {\n";
        issueTile("blockIdx.x", L);
        o_ << "  }\n  for (u32 tile = blockIdx.x + tile0; tile < ntiles; tile += gridDim.x) {\n"
           << "  " << tileBase() << "\n";
        zeroTile();
        std::string decl = "  double2 ";
        for (int s = 0; s < na_; s++) decl += (s ? ", a" : "a") + std::to_string(s);
        o_ << decl << ";\n  double2 P = C2(1.0, 0.0);\n" << pendDecl();
        o_ << "  if (tma) {\n    mbar_wait(mbar, phase);\n    phase ^= 1u;\n    { const u32 u = "
           << pbSwExpr(threadSmem(P_.map_in[0])) << ";\n";
        for (int s = 0; s < na_; s++) o_ << "    a" << s << " = sm[u ^ " << pbSw(regCoord(P_.map_in[0], s)) << "u];\n";
        o_ << "    }\n    __syncthreads();  // PB drained: stream the next tile into it\n"
           << "    if (tile + gridDim.x < ntiles) {\n";
        issueTile("tile + gridDim.x", L);
        o_ << "    }\n  } else if (smask != 0ull) {  // known zeros: read only the support\n"
           << "    const u64 off = base | " << threadGlobal(P_.map_in[0]) << ";\n";
        sparseLoads("    ");
        prefetchSupportNext();
        o_ << "  } else {  // first pass of a run: synthesize |basis>\n"
           << "    const u64 off = base | " << threadGlobal(P_.map_in[0]) << ";\n";
        for (int s = 0; s < na_; s++)
            o_ << "    a" << s << " = C2((off | " << regGlobal(P_.map_in[0], s) << "ull) == basis ? " << lit(P_.synth_amp ? P_.synth_amp : 1.0) << " : 0.0, 0.0);\n";
        o_ << "  }\n";
        ctaFactors();
        for (int i = 0; i < P_.nops; i++) op(P_.ops[i]);
        const int last = P_.nsegs - 1;
        uint64_t gx = 0;
        for (int j = 0; j < ct_; j++)
            if ((P_.xmask_out[last] >> j) & 1) gx |= uint64_t(1) << P_.tile_phys[j];
        if (P_.norm_out) emitNorm();
        // Sparse runs (PB is free: no tile streams in): stage the output tile
        // in PB and let the TMA engine write its rows, so the HBM write of this
        // tile drains while the CTA computes the next one.
        o_ << "  if (smask != 0ull) {\n    bulk_wait_read();  // this thread's previous rows have left PB\n"
           << "    __syncthreads();\n    { const u32 u = "
           << pbSwExpr(threadSmem(P_.map_out[last]) + " ^ " + std::to_string(uint32_t(P_.xmask_out[last])) + "u") << ";\n";
        for (int s = 0; s < na_; s++)
            o_ << "    sm[u ^ " << pbSw(regCoord(P_.map_out[last], s)) << "u] = a" << nm_[size_t(s)] << ";\n";
        o_ << "    }\n    fence_async();\n    __syncthreads();\n";
        storeTile(L);
        o_ << "  } else {\n";
        o_ << "  { const u64 off = (base | " << threadGlobal(P_.map_out[last]) << ") ^ " << gx << "ull;\n";
        for (int s = 0; s < na_; s++)
            o_ << "  __stcs(st + (off ^ " << regGlobal(P_.map_out[last], s) << "ull), a" << nm_[size_t(s)] << ");\n";
        // (TMA tiles re-synchronize after draining PB; synthesized tiles must
        // not start writing F / XS while a slow thread still reads them.)
        o_ << "  }\n  }\n  if (!tma && tile + gridDim.x < ntiles) __syncthreads();\n  }\n"
           << "  if (smask != 0ull) bulk_wait_all();\n}\n";
        return o_.str();
    }

private:
    // Sum |a|^2 of each warp's part of the output tile into
    // np[tile * warps + warp] (fixed order: slots, xor butterfly); no CTA
    // barrier.  The runtime folds the array (launchSumTiles).
    void emitNorm() {
        const int warps = nt_ / 32 > 0 ? nt_ / 32 : 1;
        o_ << "  { double s_ = 0.0;\n";
        for (int s = 0; s < na_; s++)
            o_ << "    s_ = fma(" << A(s) << ".x, " << A(s) << ".x, fma(" << A(s) << ".y, " << A(s) << ".y, s_));\n";
        o_ << "    for (int o_ = 16; o_ > 0; o_ >>= 1) s_ += __shfl_xor_sync(0xffffffffu, s_, o_);\n"
           << "    if ((tid & 31u) == 0u) np[(u64)tile * " << warps << "u + (tid >> 5)] = s_;\n  }\n";
    }

    // A tile whose input is all zeros -- the first pass of a run (|basis>
    // synthesized) for every tile but the basis's, or any tile outside the
    // support coset (smask / sval) -- stays all zeros under the pass's linear
    // map: write the zeros, skip the loads and the arithmetic.
    void zeroTile() {
        o_ << "  if ((basis != ~0ull && ((basis ^ base) & " << (~P_.tile_mask) << "ull) != 0ull) ||\n"
           << "      ((base ^ sval) & smask & " << (~P_.tile_mask) << "ull) != 0ull) {\n"
           << "    const u64 zoff = base | " << threadGlobal(P_.map_in[0]) << ";\n"
           << "    if (!zskip) {  // else a coalesced zero-fill kernel writes the tiles outside the support\n";
        const int kl = slotOfMem0(P_.map_in[0]);
        for (int s = 0; s < na_; s++) {
            if (kl >= 0) {
                if (!((s >> kl) & 1))
                    o_ << "    st256(st + (zoff | " << regGlobal(P_.map_in[0], s) << "ull), C2(0.0, 0.0), C2(0.0, 0.0));\n";
                continue;
            }
            o_ << "    __stcs(st + (zoff | " << regGlobal(P_.map_in[0], s) << "ull), C2(0.0, 0.0));\n";
        }
        o_ << "    }\n";
        if (P_.norm_out) {  // this tile's share of sum |a|^2 is 0
            const int warps = nt_ / 32 > 0 ? nt_ / 32 : 1;
            o_ << "    if ((tid & 31u) == 0u) np[(u64)tile * " << warps << "u + (tid >> 5)] = 0.0;\n";
        }
        o_ << "    continue;\n  }\n";
    }
    bool staged_ = false;
    // Staged store of the output tile (stagedLayout), opening the `if (stg_)`
    // branch: half 0 (top tile bit 0) into S, half 1 into the exchange buffer,
    // then one TMA store per half (half 1 first: it must drain sooner).
    void stageHalves(int last) {
        const uint32_t half = 1u << (ct_ - 1);
        const int d = tmNd_ - 1;
        o_ << "  if (stg_) {\n    if (tid == 0u) bulk_wait_read();  // both halves of the previous tile have left\n"
           << "    __syncthreads();\n    { const u32 u = "
           << pbSwExpr(threadSmem(P_.map_out[last]) + " ^ " + std::to_string(uint32_t(P_.xmask_out[last])) + "u") << ";\n"
           << "    double2* const H0 = (u & " << half << "u) ? sm : S;\n    double2* const H1 = (u & " << half
           << "u) ? S : sm;\n";
        for (int s = 0; s < na_; s++) {
            const uint32_t w = pbSw(regCoord(P_.map_out[last], s));
            o_ << "    " << ((w & half) ? "H1" : "H0") << "[(u ^ " << w << "u) & " << (half - 1) << "u] = a" << nm_[size_t(s)]
               << ";\n";
        }
        o_ << "    }\n    fence_async();\n    __syncthreads();\n";
        const std::string hiCoords = [&] {
            std::string c = tmCoords("base");
            // the top dimension's coordinate of half 1: + half its box
            const std::string key = "\"r\"((int)(base >> " + std::to_string(tmLo_[d]) + ")";
            const size_t at = c.rfind(key);
            c.insert(at + key.size(), " + " + std::to_string(1 << (tmTb_[d] - 1)));
            return c;
        }();
        o_ << "#ifdef __CUDA_ARCH__\n    if (tid == 0u) {\n"
           << "      asm volatile(\"cp.async.bulk.tensor." << tmNd_ << "d.global.shared::cta.bulk_group [%0, " << tmOperands(2)
           << "], [%1];\" :: \"l\"(&tm), \"r\"(smem_u32(sm)), " << hiCoords << " : \"memory\");\n      bulk_commit();\n"
           << "      asm volatile(\"cp.async.bulk.tensor." << tmNd_ << "d.global.shared::cta.bulk_group [%0, " << tmOperands(2)
           << "], [%1];\" :: \"l\"(&tm), \"r\"(smem_u32(S)), " << tmCoords("base") << " : \"memory\");\n      bulk_commit();\n"
           << "    }\n#else\n    if (tid == 0u) {\n      static const unsigned char tp_[] = {";
        for (int j = 0; j < ct_; j++) o_ << (j ? "," : "") << int(P_.tile_phys[j]);
        o_ << "};\n      for (u32 h = 0; h < 2u; h++)\n        for (u32 v = 0; v < " << half << "u; v++) {\n"
           << "          u64 o = base | ((u64)h << tp_[" << (ct_ - 1) << "]);\n"
           << "          for (int j = 0; j < " << (ct_ - 1) << "; j++) o |= (u64)((v >> j) & 1u) << tp_[j];\n"
           << "          st[o] = (h ? sm : S)[" << pbSwExpr("v") << "];\n        }\n    }\n#endif\n";
    }
    // Tensor view of the tile (tensorLayout): rank, dimensions, PB swizzle.
    int tmNd_ = 0, tmLo_[5] = {}, tmTb_[5] = {}, tmSwz_ = 0;
    void tensorView() { tmNd_ = tensorLayout(P_, tmLo_, tmTb_, &tmSwz_); }
    // PB chunk of tile coordinate u under the swizzle (GF(2)-linear: the
    // thread part and each slot's part are swizzled separately).
    uint32_t pbSw(uint32_t u) const { return u ^ ((u >> 3) & ((1u << tmSwz_) - 1)); }
    std::string pbSwExpr(const std::string& u) const {
        if (!tmSwz_) return u;
        return "((" + u + ") ^ (((" + u + ") >> 3) & " + std::to_string((1u << tmSwz_) - 1) + "u))";
    }
    // Box coordinates of the tile at `b` ("r" operands).
    std::string tmCoords(const std::string& b) const {
        std::string c;
        for (int d = 0; d < tmNd_; d++) {
            std::string e = d ? "(" + b + " >> " + std::to_string(tmLo_[d]) + ")" : "(" + b + " << 1)";
            if (d + 1 < tmNd_)
                e = "(" + e + " & " + std::to_string((uint64_t(1) << (tmLo_[d + 1] - tmLo_[d] + (d ? 0 : 1))) - 1) + "ull)";
            c += std::string(d ? ", " : "") + "\"r\"((int)" + e + ")";
        }
        return c;
    }
    std::string tmOperands(int first) const {
        std::string s = "{";
        for (int d = 0; d < tmNd_; d++) s += (d ? ", %" : "%") + std::to_string(first + d);
        return s + "}";
    }
    // Host builds (tests/host/jit_host_shim.h) replay a tensor-map copy of the
    // tile at `b` element by element, swizzle included.
    void hostTileCopy(const std::string& b, bool toGlobal) {
        o_ << "#else\n    if (tid == 0u) {\n      static const unsigned char tp_[] = {";
        for (int j = 0; j < ct_; j++) o_ << (j ? "," : "") << int(P_.tile_phys[j]);
        o_ << "};\n      for (u32 v = 0; v < " << (1u << ct_) << "u; v++) {\n        u64 o = " << b
           << ";\n        for (int j = 0; j < " << ct_ << "; j++) o |= (u64)((v >> j) & 1u) << tp_[j];\n        const u32 c = "
           << pbSwExpr("v") << ";\n        " << (toGlobal ? "st[o] = sm[c];" : "sm[c] = st[o];") << "\n      }\n    }\n#endif\n";
    }
    // The staged tile (PB) to global memory: one tensor-map TMA store (tmv:
    // launch() encoded the map), else one bulk store per row (unswizzled PB
    // only).
    void storeTile(int Lrun) {
        if (!tmNd_) {
            storeRows(Lrun);
            return;
        }
        o_ << "#ifdef __CUDA_ARCH__\n    if (tmv) {\n      if (tid == 0u) {\n        asm volatile(\"cp.async.bulk.tensor." << tmNd_
           << "d.global.shared::cta.bulk_group [%0, " << tmOperands(2) << "], [%1];\" :: \"l\"(&tm), \"r\"(smem_u32(sm)), "
           << tmCoords("base") << " : \"memory\");\n        bulk_commit();\n      }\n    } else {\n";
        if (tmSwz_)
            o_ << "      __trap();  // a swizzled PB has no row form\n";
        else
            storeRows(Lrun);
        o_ << "    }\n";
        hostTileCopy("base", true);
    }
    // One bulk store per contiguous row, rows spread over all threads, each
    // thread committing its own bulk group.
    void storeRows(int Lrun) {
        const int L = std::min(Lrun, 8);  // rows of <= 4 KB
        const int rows = 1 << (ct_ - L);
        o_ << "    for (u32 r = tid; r < " << rows << "u; r += " << nt_ << "u) {\n      u64 o = base;\n";
        for (int j = L; j < ct_; j++)
            o_ << "      o |= (u64)((r >> " << (j - L) << ") & 1u) << " << int(P_.tile_phys[j]) << ";\n";
        o_ << "      bulk_s2g(st + o, sm + (r << " << L << "), " << (16u << L) << "u);\n    }\n    bulk_commit();\n";
    }
    // Stream tile `t` into PB: one tensor-map TMA load, else one bulk copy per
    // contiguous row.
    void issueTile(const std::string& t, int Lrun) {
        const int L = std::min(Lrun, 8);  // rows of <= 4 KB, spread over all threads
        const int rows = 1 << (ct_ - L);
        o_ << "    {\n      " << deposit("nb", "(u64)(" + t + ")") << "\n"
           << "      fence_async();\n      if (tid == 0u) mbar_expect_tx(mbar, " << (16u << ct_) << "u);\n"
           << "      __syncthreads();\n";
        auto rowsLoop = [&]() {
            o_ << "      for (u32 r = tid; r < " << rows << "u; r += " << nt_ << "u) {\n        u64 o = nb;\n";
            for (int j = L; j < ct_; j++)
                o_ << "        o |= (u64)((r >> " << (j - L) << ") & 1u) << " << int(P_.tile_phys[j]) << ";\n";
            o_ << "        bulk_g2s(sm + (r << " << L << "), st + o, " << (16u << L) << "u, mbar);\n      }\n";
        };
        if (!tmNd_) {
            rowsLoop();
            o_ << "    }\n";
            return;
        }
        o_ << "#ifdef __CUDA_ARCH__\n      if (tmv) {\n        if (tid == 0u)\n          asm volatile(\"cp.async.bulk.tensor." << tmNd_
           << "d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, " << tmOperands(3)
           << "], [%2];\" :: \"r\"(smem_u32(sm)), \"l\"(&tm), \"r\"(smem_u32(mbar)), " << tmCoords("nb")
           << " : \"memory\");\n      } else {\n";
        if (tmSwz_)
            o_ << "      __trap();  // a swizzled PB has no row form\n";
        else
            rowsLoop();
        o_ << "      }\n";
        hostTileCopy("nb", false);
        o_ << "    }\n";
    }
    // Register slot whose tile bit is memory bit 0 (-1: none / wide access off).
    int slotOfMem0(const uint8_t* m) const {
        if (!qkdev::wideAccess() || !nvrtcSupportsWideAccess() || P_.tile_phys[0] != 0) return -1;
        for (int k = 0; k < rb_; k++)
            if (m[k] == 0) return k;
        return -1;
    }
    uint32_t regCoord(const uint8_t* m, int s) const {
        uint32_t u = 0;
        for (int k = 0; k < rb_; k++)
            if ((s >> k) & 1) u |= 1u << m[k];
        return u;
    }
    // Loads of a pass with known zeros (smask / sval): a thread whose own
    // index bits already leave the support has only zeros (one test, no
    // loads); otherwise each register slot is read only if its slot bits
    // match the support.
    void sparseLoads(const std::string& ind) {
        // QK_SPARSE_EARLY_OUT=1: a per-thread test first.  Measured slower
        // and bimodal on QFT-33 (50-64 ms vs 47.8 ms for per-slot tests).
        if (!knob("QK_SPARSE_EARLY_OUT", 0)) {
            for (int s = 0; s < na_; s++)
                o_ << ind << "{ const u64 i_ = off | " << regGlobal(P_.map_in[0], s) << "ull; a" << s
                   << " = ((i_ ^ sval) & smask) == 0ull ? __ldcs(st + i_) : C2(0.0, 0.0); }\n";
            return;
        }
        uint64_t slots = 0;
        for (int s = 0; s < na_; s++) slots |= regGlobal(P_.map_in[0], s);
        o_ << ind << "if (((off ^ sval) & smask & " << (~slots) << "ull) != 0ull) {\n";
        for (int s = 0; s < na_; s++) o_ << ind << "  a" << s << " = C2(0.0, 0.0);\n";
        o_ << ind << "} else {\n";
        for (int s = 0; s < na_; s++) {
            const uint64_t r = regGlobal(P_.map_in[0], s);
            o_ << ind << "  a" << s << " = ((" << r << "ull ^ sval) & smask & " << slots << "ull) == 0ull ? __ldcs(st + (off | "
               << r << "ull)) : C2(0.0, 0.0);\n";
        }
        o_ << ind << "}\n";
    }
    // Per-thread table factors (OP_SCAL_TAB / OP_PEND_TAB) depend only on the
    // thread index: with QK_HOIST_TAB=1 they are all loaded at the kernel's
    // start, before the tile loop.  Off by default: measured on B200 at 33
    // qubits it gains 1 % on QFT but costs 5 % on QAOA and 29 % on Grover
    // (register pressure in passes with many table ops).
    void hoistTables() {
        tabName_.clear();
        if (!knob("QK_HOIST_TAB", 0)) return;
        int k = 0;
        for (int i = 0; i < P_.nops; i++) {
            const DevOp& d = P_.ops[i];
            if (d.type != qkdev::OP_SCAL_TAB && d.type != qkdev::OP_PEND_TAB) continue;
            const std::string nm = "T" + std::to_string(k++);
            o_ << "  const double2 " << nm << " = __ldg(gt + " << d.c << "u + " << pext(d.x16) << ");\n";
            tabName_[i] = nm;
        }
    }
    std::string tabLoad(const DevOp& d) {
        const auto it = tabName_.find(int(&d - P_.ops));
        if (it != tabName_.end()) return it->second;
        return "__ldg(gt + " + std::to_string(d.c) + "u + " + pext(d.x16) + ")";
    }
    std::map<int, std::string> tabName_;
    // Base index of tile `tile`.  zskip == 2: only the tiles meeting the
    // support {i : (i ^ sval) & smask == 0} are enumerated -- the tile index
    // is deposited into the non-tile bits the support leaves free, and the
    // fixed ones come from sval (the pass runs on 2^free tiles instead of
    // launching every tile to skip most of them).
    std::string tileBase(const std::string& var = "base", const std::string& t = "tile") const {
        const std::string all = deposit(var, "(u64)(" + t + ")");
        const std::string nt = std::to_string(~P_.tile_mask) + "ull";
        return all + "\n  if (zskip == 2u) {\n    const u64 fixed_ = smask & " + nt + ";\n" +
               "    u64 m_ = " + nt + " & ~fixed_, t_ = (u64)(" + t + ");\n    " + var + " = sval & fixed_;\n" +
               "    while (t_) { const u64 low_ = m_ & (0ull - m_); if (t_ & 1ull) " + var +
               " |= low_; t_ >>= 1; m_ ^= low_; }\n  }";
    }
    // CTA index deposited into the non-tile bits of the slice index.
    // Statement block declaring `u64 var` = v deposited into the non-tile bits.
    std::string deposit(const std::string& var, const std::string& v) const {
        std::string e = "u64 " + var + " = " + v + ";";
        for (int j = 0; j < ct_; j++) {
            const int p = P_.tile_phys[j];
            e += " " + var + " = ((" + var + " >> " + std::to_string(p) + ") << " + std::to_string(p + 1) + ") | (" +
                 var + " & " + std::to_string((uint64_t(1) << p) - 1) + "ull);";
        }
        return e;
    }
    // Rows of the tile: the run of tile bits that are the lowest memory bits is
    // contiguous; the remaining tile bits enumerate rows.
    void prefetchNext() {
        if (usePersistent()) prefetchSupportNext();
        if (tmNd_ && prefetchTiles(P_)) {  // one tensor prefetch per half tile
            const int d = tmNd_ - 1;
            std::string hi = tmCoords("nb_");
            const std::string key = "\"r\"((int)(nb_ >> " + std::to_string(tmLo_[d]) + ")";
            hi.insert(hi.rfind(key) + key.size(), " + " + std::to_string(1 << (tmTb_[d] - 1)));
            o_ << "#ifdef __CUDA_ARCH__\n  if (basis == ~0ull && smask == 0ull && tmv && tid == 0u && tile + gridDim.x < ntiles) {\n  "
               << tileBase("nb_", "tile + gridDim.x") << "\n"
               << "    asm volatile(\"cp.async.bulk.prefetch.tensor." << tmNd_ << "d.L2.global.tile [%0, " << tmOperands(1)
               << "];\" :: \"l\"(&tm), " << tmCoords("nb_") << " : \"memory\");\n"
               << "    asm volatile(\"cp.async.bulk.prefetch.tensor." << tmNd_ << "d.L2.global.tile [%0, " << tmOperands(1)
               << "];\" :: \"l\"(&tm), " << hi << " : \"memory\");\n  }\n#endif\n";
            return;
        }
        int L = 0;
        while (L < ct_ && P_.tile_phys[L] == L) L++;
        if (L < 3 || !usePrefetch()) return;  // rows under 128 B: not worth a TMA op each
        const int rows = 1 << (ct_ - L);
        const unsigned bytes = 16u << L;
        o_ << "  if (smask == 0ull && basis == ~0ull && tile + gridDim.x < ntiles) {\n    u64 nb = (u64)(tile + gridDim.x);\n";
        for (int j = 0; j < ct_; j++) {
            const int p = P_.tile_phys[j];
            o_ << "    nb = ((nb >> " << p << ") << " << (p + 1) << ") | (nb & " << ((uint64_t(1) << p) - 1) << "ull);\n";
        }
        o_ << "    for (u32 r = tid; r < " << rows << "u; r += " << nt_ << "u) {\n      u64 o = nb;\n";
        for (int j = L; j < ct_; j++)
            o_ << "      o |= (u64)((r >> " << (j - L) << ") & 1u) << " << int(P_.tile_phys[j]) << ";\n";
        o_ << "      pf_l2(st + o, " << bytes << "u);\n    }\n  }\n";
    }
    // Each thread prefetches into L2 the support amplitudes its slots read in
    // the CTA's next tile (a run with known zeros, persistent grid).
    void prefetchSupportNext() {
        if (useSparsePrefetch()) {
            uint64_t slots = 0;
            for (int s = 0; s < na_; s++) slots |= regGlobal(P_.map_in[0], s);
            o_ << "  if (smask != 0ull && tile + gridDim.x < ntiles) {\n  " << tileBase("nb_", "tile + gridDim.x") << "\n"
               << "    const u64 noff_ = nb_ | " << threadGlobal(P_.map_in[0]) << ";\n"
               << "    if (((noff_ ^ sval) & smask & " << (~slots) << "ull) == 0ull) {\n";
            for (int s = 0; s < na_; s++) {
                const uint64_t r = regGlobal(P_.map_in[0], s);
                o_ << "      if (((" << r << "ull ^ sval) & smask & " << slots << "ull) == 0ull) pf_line(st + (noff_ | " << r
                   << "ull));\n";
            }
            o_ << "    }\n  }\n";
        }
    }
    // Factor f is computed by warp f mod #warps: lane j takes term j (mod 32)
    // with its condition and value as literals (no table loads), then the
    // partial products meet in a shuffle tree.
    // Per-CTA factor terms as device tables (literalFactors false).
    void ctaTables() {
        if (!P_.ncta || literalFactors(P_)) return;
        const int nt = P_.cta_end[P_.ncta - 1];
        o_ << "static __device__ const unsigned char qk_tb[] = {";
        for (int t = 0; t < nt; t++) o_ << (t ? "," : "") << int(P_.cta_terms[t].b1) << "," << int(P_.cta_terms[t].b2);
        o_ << "};\nstatic __device__ const double2 qk_tv[] = {";
        for (int t = 0; t < nt; t++) {
            const uint32_t c = P_.cta_terms[t].c;
            o_ << (t ? ",{" : "{") << lit(P_.coef[2 * c]) << "," << lit(P_.coef[2 * c + 1]) << "}";
        }
        o_ << "};\nstatic __device__ const unsigned short qk_te[] = {";
        for (int f = 0; f < P_.ncta; f++) o_ << (f ? "," : "") << P_.cta_end[f];
        o_ << "};\n";
    }
    void ctaFactorsTable() {
        o_ << "  { const u32 w = tid >> 5, l = tid & 31u;\n"
           << "    for (u32 f = w; f < " << P_.ncta << "u; f += " << std::max(1, nt_ / 32) << "u) {\n"
           << "      double2 acc = C2(1.0, 0.0);\n"
           << "      for (u32 t = (f ? qk_te[f - 1] : 0u) + l; t < qk_te[f]; t += 32u) {\n"
           << "        const u32 b1 = qk_tb[2 * t], b2 = qk_tb[2 * t + 1];\n"
           << "        if (b1 == 255u || ((base >> b1) & (base >> b2) & 1ull)) acc = cmul(acc, qk_tv[t]);\n"
           << "      }\n"
           << "      for (int o = 16; o > 0; o >>= 1)\n"
           << "        acc = cmul(acc, make_double2(__shfl_xor_sync(0xffffffffu, acc.x, o), "
              "__shfl_xor_sync(0xffffffffu, acc.y, o)));\n"
           << "      if (l == 0u) F[f] = acc;\n    }\n  }\n  __syncthreads();\n";
    }
    void ctaFactors() {
        if (!P_.ncta) return;
        if (!literalFactors(P_)) return ctaFactorsTable();
        const int nw = std::max(1, nt_ / 32);
        o_ << "  { const u32 w = tid >> 5, l = tid & 31u;\n";
        for (int f = 0; f < P_.ncta; f++) {
            const int t0 = f ? P_.cta_end[f - 1] : 0, t1 = P_.cta_end[f], nterm = t1 - t0;
            o_ << "    if (w == " << (f % nw) << "u) {\n      double2 acc = C2(1.0, 0.0);\n";
            for (int t = t0; t < t1; t++) {
                const qkdev::CtaTerm& ct = P_.cta_terms[t];
                const std::string cond =
                    ct.b1 == 255 ? std::string("true")
                                 : "((base >> " + std::to_string(int(ct.b1)) + ") & (base >> " + std::to_string(int(ct.b2)) +
                                       ") & 1ull)";
                const std::string v = c2(P_.coef[2 * ct.c], P_.coef[2 * ct.c + 1]);
                if (t - t0 < 32)
                    o_ << "      if (l == " << (t - t0) << "u && " << cond << ") acc = " << v << ";\n";
                else
                    o_ << "      if (l == " << ((t - t0) % 32) << "u && " << cond << ") acc = cmul(acc, " << v << ");\n";
            }
            const int width = std::min(nterm, 32);
            int span = 1;
            while (span < width) span <<= 1;
            for (int off = span / 2; off > 0; off >>= 1)
                o_ << "      acc = cmul(acc, make_double2(__shfl_xor_sync(0xffffffffu, acc.x, " << off
                   << "), __shfl_xor_sync(0xffffffffu, acc.y, " << off << ")));\n";
            o_ << "      if (l == 0u) F[" << f << "] = acc;\n    }\n";
        }
        o_ << "  }\n  __syncthreads();\n";
    }
    std::string pendDecl() {
        std::string d;
        for (int k = 0; k < rb_; k++) d += "  double2 R" + std::to_string(k) + " = C2(1.0, 0.0);\n";
        return d;
    }
    std::string tb(int j) const { return "((tid >> " + std::to_string(j) + ") & 1u)"; }

    // thread part of the global offset under map m
    std::string threadGlobal(const uint8_t* m) const {
        std::string e = "(u64)0";
        for (int j = 0; j < ct_ - rb_; j++)
            e += " | ((u64)" + tb(j) + " << " + std::to_string(int(P_.tile_phys[m[rb_ + j]])) + ")";
        return "(" + e + ")";
    }
    uint64_t regGlobal(const uint8_t* m, int s) const {
        uint64_t o = 0;
        for (int k = 0; k < rb_; k++)
            if ((s >> k) & 1) o |= uint64_t(1) << P_.tile_phys[m[k]];
        return o;
    }
    std::string threadSmem(const uint8_t* m) const {
        std::string e = "0u";
        for (int j = 0; j < ct_ - rb_; j++) e += " | (" + tb(j) + " << " + std::to_string(int(m[rb_ + j])) + ")";
        return "(" + e + ")";
    }
    uint32_t regSmem(const uint8_t* m, int s) const {
        uint32_t u = 0;
        for (int k = 0; k < rb_; k++)
            if ((s >> k) & 1) u |= 1u << m[k];
        return swzHost(u);
    }

    std::string lc(uint32_t i) const { return c2(P_.coef[2 * i], P_.coef[2 * i + 1]); }
    // Phase literals: a part below 2^-50 of a unit-modulus coefficient is the
    // rounding residue of cos / sin at a multiple of pi/2 (cos(pi/2) =
    // 6.1e-17); it is taken as 0 so the multiply specializes.  This moves
    // results by < 1e-16 relative per multiply (the north star's bar is 1e-10).
    static void snap(double& re, double& im) {
        const double tiny = 0x1p-50;
        if (std::fabs(re) < tiny && std::fabs(std::fabs(im) - 1.0) < tiny) re = 0.0, im = im > 0 ? 1.0 : -1.0;
        if (std::fabs(im) < tiny && std::fabs(std::fabs(re) - 1.0) < tiny) im = 0.0, re = re > 0 ? 1.0 : -1.0;
    }
    // x * (re + i im) for a literal coefficient, specialized when a part is 0.
    static std::string mulK(const std::string& x, double re, double im) {
        snap(re, im);
        if (re == 0.0 && im == 0.0) return "C2(0.0, 0.0)";
        if (im == 0.0) return re == 1.0 ? x : "cmulr(" + x + ", " + lit(re) + ")";
        if (re == 0.0) return "cmuli(" + x + ", " + lit(im) + ")";
        return "cmul(" + x + ", " + c2(re, im) + ")";
    }
    // acc + (re + i im) * x
    static std::string macK(const std::string& acc, double re, double im, const std::string& x) {
        snap(re, im);
        if (re == 0.0 && im == 0.0) return acc;
        if (im == 0.0) return "cmacr(" + acc + ", " + lit(re) + ", " + x + ")";
        if (re == 0.0) return "cmaci(" + acc + ", " + lit(im) + ", " + x + ")";
        return "cmac(" + acc + ", " + c2(re, im) + ", " + x + ")";
    }
    std::string mulC(const std::string& x, uint32_t i) const { return mulK(x, P_.coef[2 * i], P_.coef[2 * i + 1]); }
    std::string macC(const std::string& acc, uint32_t i, const std::string& x) const {
        return macK(acc, P_.coef[2 * i], P_.coef[2 * i + 1], x);
    }
    std::string A(int s) const { return "a" + std::to_string(nm_[size_t(s)]); }

    void mulAmp(int s, const std::string& e) { o_ << "  " << A(s) << " = cmul(" << A(s) << ", " << e << ");\n"; }

    std::string pext(uint32_t mask) const {
        std::string e = "0u";
        int r = 0;
        for (int j = 0; j < 16; j++)
            if ((mask >> j) & 1) e += " | (" + tb(j) + " << " + std::to_string(r++) + ")";
        return "(" + e + ")";
    }

    void op(const DevOp& d) {
        const int a = d.a, b = d.b, K = 1 << d.a;
        switch (d.type) {
            case qkdev::OP_H:
                for (int s = 0; s < na_; s++)
                    if (!(s & K))
                        o_ << "  { const double2 x = " << A(s) << ", y = " << A(s | K) << "; " << A(s)
                           << " = cadd(x, y); " << A(s | K) << " = csub(x, y); }\n";
                return;
            case qkdev::OP_MAT1:
                for (int s = 0; s < na_; s++)
                    if (!(s & K))
                        o_ << "  { const double2 x = " << A(s) << ", y = " << A(s | K) << "; " << A(s) << " = "
                           << macC(mulC("x", d.c), d.c + 1, "y") << "; " << A(s | K) << " = "
                           << macC(mulC("x", d.c + 2), d.c + 3, "y") << "; }\n";
                return;
            case qkdev::OP_CX: {
                const int pol = (d.k >> 1) & 1;
                if (d.k & 5) {  // thread-bit or CTA-bit control: selects
                    if (d.k & 4) o_ << "  { const bool c = ((base >> " << b << ") & 1ull) != 0ull;\n";
                    else o_ << "  { const bool c = (" << tb(b) << " ^ " << pol << "u) != 0u;\n";
                    for (int s = 0; s < na_; s++)
                        if (!(s & K))
                            o_ << "    { const double2 x = " << A(s) << ", y = " << A(s | K) << "; " << A(s)
                               << " = csel(c, y, x); " << A(s | K) << " = csel(c, x, y); }\n";
                    o_ << "  }\n";
                } else {  // register control: pure rename
                    for (int s = 0; s < na_; s++)
                        if (!(s & K) && ((s >> b) & 1) == (1 ^ pol)) std::swap(nm_[size_t(s)], nm_[size_t(s | K)]);
                }
                return;
            }
            case qkdev::OP_CCX: {  // register controls: rename; thread controls: selects
                const int b2 = int(d.c);
                const bool x1 = (d.k >> 4) & 1, x2 = (d.k >> 5) & 1;  // CTA-bit controls
                const bool t1 = (d.k & 1) || x1, t2 = ((d.k >> 2) & 1) || x2;  // runtime conditions
                const int p1 = (d.k >> 1) & 1, p2 = (d.k >> 3) & 1;
                auto term = [&](bool x, int bit, int pol) {
                    return x ? "((base >> " + std::to_string(bit) + ") & 1ull) != 0ull"
                             : "(" + tb(bit) + " ^ " + std::to_string(pol) + "u) != 0u";
                };
                std::string cond;
                if (t1) cond = term(x1, b, p1);
                if (t2) cond += (cond.empty() ? "" : " && ") + term(x2, b2, p2);
                if (!cond.empty()) o_ << "  { const bool c = " << cond << ";\n";
                for (int s = 0; s < na_; s++) {
                    if (s & K) continue;
                    if (!t1 && ((s >> b) & 1) != (1 ^ p1)) continue;
                    if (!t2 && ((s >> b2) & 1) != (1 ^ p2)) continue;
                    if (cond.empty()) {
                        std::swap(nm_[size_t(s)], nm_[size_t(s | K)]);
                        continue;
                    }
                    o_ << "    { const double2 x = " << A(s) << ", y = " << A(s | K) << "; " << A(s)
                       << " = csel(c, y, x); " << A(s | K) << " = csel(c, x, y); }\n";
                }
                if (!cond.empty()) o_ << "  }\n";
                return;
            }
            case qkdev::OP_DIAG1_R:
                for (int s = 0; s < na_; s++) {
                    const std::string e = mulC(A(s), d.c + ((s >> a) & 1));
                    if (e != A(s)) o_ << "  " << A(s) << " = " << e << ";\n";
                }
                return;
            case qkdev::OP_DIAG2_RR:
                for (int s = 0; s < na_; s++) mulAmp(s, lc(d.c + ((((s >> a) & 1) << 1) | ((s >> b) & 1))));
                return;
            case qkdev::OP_CPHASE_RR:
                for (int s = 0; s < na_; s++)
                    if (((((s >> a) & 1) << 1) | ((s >> b) & 1)) == d.k) mulAmp(s, lc(d.c));
                return;
            case qkdev::OP_PEND_R:
                o_ << "  R" << a << " = cmul(R" << a << ", " << lc(d.c) << ");\n";
                dirtyR_[a] = true;
                return;
            case qkdev::OP_PEND_RT:
                o_ << "  R" << a << " = cmul(R" << a << ", " << tb(b) << " ? " << lc(d.c + 1) << " : " << lc(d.c)
                   << ");\n";
                dirtyR_[a] = true;
                return;
            case qkdev::OP_SCAL:
                o_ << "  P = cmul(P, " << lc(d.c) << ");\n";
                dirtyP_ = true;
                return;
            case qkdev::OP_SCAL_T:
                o_ << "  P = cmul(P, " << tb(a) << " ? " << lc(d.c + 1) << " : " << lc(d.c) << ");\n";
                dirtyP_ = true;
                return;
            case qkdev::OP_SCAL_TT:
                o_ << "  { const u32 i = (" << tb(a) << " << 1) | " << tb(b) << "; P = cmul(P, i == 0u ? " << lc(d.c)
                   << " : i == 1u ? " << lc(d.c + 1) << " : i == 2u ? " << lc(d.c + 2) << " : " << lc(d.c + 3)
                   << "); }\n";
                dirtyP_ = true;
                return;
            case qkdev::OP_SCAL_TAB:
                o_ << "  P = cmul(P, " << tabLoad(d) << ");\n";
                dirtyP_ = true;
                return;
            case qkdev::OP_PEND_TAB:
                o_ << "  R" << a << " = cmul(R" << a << ", " << tabLoad(d) << ");\n";
                dirtyR_[a] = true;
                return;
            case qkdev::OP_CX_PEND:
                o_ << "  if ((" << tb(b) << " ^ " << ((d.k >> 1) & 1) << "u) != 0u) { P = cmul(P, R" << a << "); R" << a
                   << " = cinv(R" << a << "); }\n";
                dirtyP_ = true;
                dirtyR_[a] = true;
                return;
            case qkdev::OP_SCAL_CTA:
                o_ << "  P = cmul(P, F[" << d.c << "]);\n";
                dirtyP_ = true;
                return;
            case qkdev::OP_SCAL_TCTA:
                o_ << "  { const double2 e = F[" << d.c << "]; if (" << tb(b) << ") P = cmul(P, e); }\n";
                dirtyP_ = true;
                return;
            case qkdev::OP_PEND_CTA:
                o_ << "  R" << a << " = cmul(R" << a << ", F[" << d.c << "]);\n";
                dirtyR_[a] = true;
                return;
            case qkdev::OP_FLUSH_SLOT:
                if (!dirtyR_[a]) return;
                for (int s = 0; s < na_; s++)
                    if (s & K) mulAmp(s, "R" + std::to_string(a));
                o_ << "  R" << a << " = C2(1.0, 0.0);\n";
                dirtyR_[a] = false;
                return;
            case qkdev::OP_FLUSH:
                flush(P_.coef[2 * d.c], d.c16 ? &P_.coef[2 * (d.c16 - 1)] : nullptr);
                return;
            case qkdev::OP_RESET:
                if (dirtyP_) o_ << "  P = C2(1.0, 0.0);\n";
                for (int k = 0; k < rb_; k++)
                    if (dirtyR_[k]) o_ << "  R" << k << " = C2(1.0, 0.0);\n";
                dirtyP_ = false;
                for (int k = 0; k < rb_; k++) dirtyR_[k] = false;
                return;
            case qkdev::OP_FLUSH_SLOT_G: {
                // amplitudes with slot-a bit 1 *= R_a * G[pext(s, b)] (G literal)
                std::vector<int> bits;
                for (int k = 0; k < rb_; k++)
                    if ((d.b >> k) & 1) bits.push_back(k);
                const int ng = 1 << bits.size();
                o_ << "  {\n";
                if (dirtyR_[a])
                    for (int j = 0; j < ng; j++)
                        o_ << "    const double2 h" << j << " = " << mulC("R" + std::to_string(a), d.c + uint32_t(j)) << ";\n";
                for (int s = 0; s < na_; s++) {
                    if (!((s >> a) & 1)) continue;
                    int j = 0;
                    for (size_t q = 0; q < bits.size(); q++) j |= ((s >> bits[q]) & 1) << q;
                    if (dirtyR_[a]) {
                        o_ << "  ";
                        mulAmp(s, "h" + std::to_string(j));
                        continue;
                    }
                    // literal factor: specialized multiply (none at all for 1)
                    const std::string m = mulC(A(s), d.c + uint32_t(j));
                    if (m != A(s)) o_ << "  " << A(s) << " = " << m << ";\n";
                }
                o_ << "  }\n";
                if (dirtyR_[a]) o_ << "  R" << a << " = C2(1.0, 0.0);\n";
                dirtyR_[a] = false;
                return;
            }
            case qkdev::OP_DTABLE: {
                const uint16_t* cb = &P_.contrib[d.c16];
                std::string sub = "0u";
                for (int j = rb_; j < ct_; j++)
                    if (cb[j]) sub += " | (" + tb(j - rb_) + " ? " + std::to_string(cb[j]) + "u : 0u)";
                for (int j = 0; j < cb[ct_]; j++)  // bits outside the tile: constants of the CTA
                    sub += " | (((base >> " + std::to_string(cb[ct_ + 1 + 2 * j]) + ") & 1ull) ? " +
                           std::to_string(cb[ct_ + 2 + 2 * j]) + "u : 0u)";
                o_ << "  { const u32 sub = " << sub << ";\n";
                for (int s = 0; s < na_; s++) {
                    uint32_t cs = 0;
                    for (int k = 0; k < rb_; k++)
                        if ((s >> k) & 1) cs |= cb[k];
                    o_ << "  " << A(s) << " = cmul(" << A(s) << ", __ldg(gt + " << d.c << "u + ((sub | " << cs << "u) ^ "
                       << d.x16 << "u)));\n";
                }
                o_ << "  }\n";
                return;
            }
            case qkdev::OP_DENSE: {
                const int D = 1 << d.k;
                for (int g = 0; g < na_ / D; g++) {
                    o_ << "  {\n";
                    for (int s = 0; s < D; s++) o_ << "    const double2 x" << s << " = " << A(g * D + s) << ";\n";
                    for (int r = 0; r < D; r++) {
                        o_ << "    { double2 acc = C2(0.0, 0.0);";
                        for (int s = 0; s < D; s++)
                            o_ << " acc = cmac(acc, __ldg(gt + " << (d.c + uint32_t(r * D + s)) << "u), x" << s << ");";
                        o_ << " " << A(g * D + r) << " = acc; }\n";
                    }
                    o_ << "  }\n";
                }
                return;
            }
            case qkdev::OP_EXCHANGE: {
                const uint8_t* mo = P_.map_out[d.c - 1];
                const uint8_t* mi = P_.map_in[d.c];
                if (pipe_) return halfExchange(d.c, mo, mi);
                if (staged_)  // the previous tile's half 1 must have left the exchange buffer
                    o_ << "  if (stg_ && tid == 0u) bulk_wait_read1();\n";
                o_ << "  __syncthreads();\n  { const u32 u = swz(" << threadSmem(mo) << ") ^ "
                   << swzHost(P_.xmask_out[d.c - 1]) << "u;\n";
                for (int s = 0; s < na_; s++) o_ << "  sm[u ^ " << regSmem(mo, s) << "u] = " << A(s) << ";\n";
                o_ << "  }\n  __syncthreads();\n  { const u32 u = swz(" << threadSmem(mi) << ");\n";
                for (int s = 0; s < na_; s++) nm_[size_t(s)] = s;
                for (int s = 0; s < na_; s++) o_ << "  " << A(s) << " = sm[u ^ " << regSmem(mi, s) << "u];\n";
                o_ << "  }\n";
                return;
            }
            default:
                throw SimulationError("jit: unknown op");
        }
    }

    // Exchange in two phases through the 2^12-amplitude XS buffer, split on
    // tile bit x held by register slot k before and after.  Phase h moves the
    // amplitudes whose (true) bit x is h; they are read back into exactly the
    // registers that phase freed, so no value is overwritten before it is
    // written out.  XS index = swizzled tile coordinate with bit x removed
    // (x >= 3: the swizzle only touches bits 0..2, so banks are unchanged).
    void halfExchange(int c, const uint8_t* mo, const uint8_t* mi) {
        const int k = P_.xsplit[c], x = mo[k];
        const int fx = (P_.xmask_out[c - 1] >> x) & 1;
        const uint32_t lo = (1u << x) - 1;
        auto cmp = [&](uint32_t v) { return (v & lo) | ((v >> (x + 1)) << x); };
        const std::string cmpE = [&](const std::string& v) {
            return "((" + v + ") & " + std::to_string(lo) + "u) | (((" + v + ") >> " + std::to_string(x + 1) + ") << " +
                   std::to_string(x) + ")";
        }("v");
        std::vector<int> nm(nm_);
        for (int h = 0; h < 2; h++) {
            std::vector<int> freed;
            o_ << "  __syncthreads();\n  { const u32 v = swz(" << threadSmem(mo) << ") ^ " << swzHost(P_.xmask_out[c - 1])
               << "u; const u32 u = " << cmpE << ";\n";
            for (int s = 0; s < na_; s++)
                if ((((s >> k) & 1) ^ fx) == h) {
                    o_ << "  XS[u ^ " << cmp(regSmem(mo, s)) << "u] = a" << nm_[size_t(s)] << ";\n";
                    freed.push_back(nm_[size_t(s)]);
                }
            std::sort(freed.begin(), freed.end());
            o_ << "  }\n  __syncthreads();\n  { const u32 v = swz(" << threadSmem(mi) << "); const u32 u = " << cmpE
               << ";\n";
            size_t f = 0;
            for (int s = 0; s < na_; s++)
                if (((s >> k) & 1) == h) {
                    nm[size_t(s)] = freed[f++];
                    o_ << "  a" << nm[size_t(s)] << " = XS[u ^ " << cmp(regSmem(mi, s)) << "u];\n";
                }
            o_ << "  }\n";
        }
        nm_ = nm;
    }

    // a[s] *= scale * P * prod_{k: bit k of s} R[k], touching only dirty factors.
    void flush(double scale, const double* D = nullptr) {
        bool anyR = false;
        for (int k = 0; k < rb_; k++) anyR |= dirtyR_[k];
        auto dOne = [&](int s) { return !D || (D[2 * s] == 1.0 && D[2 * s + 1] == 0.0); };
        bool anyD = false;
        for (int s = 0; s < na_; s++) anyD |= !dOne(s);
        if (anyD && !anyR && !dirtyP_) {  // constant pair phases (and the scale) only: literal factors
            for (int s = 0; s < na_; s++) {
                if (dOne(s) && scale == 1.0) continue;
                mulAmp(s, c2(D[2 * s] * scale, D[2 * s + 1] * scale));
            }
            return;
        }
        if (!anyR && !dirtyP_) {
            if (scale != 1.0)
                for (int s = 0; s < na_; s++)
                    o_ << "  " << A(s) << " = make_double2(" << A(s) << ".x * " << lit(scale) << ", " << A(s) << ".y * "
                       << lit(scale) << ");\n";
            return;
        }
        o_ << "  {\n    const double2 f0 = " << (dirtyP_ ? "make_double2(P.x * " + lit(scale) + ", P.y * " + lit(scale) + ")"
                                                         : c2(scale, 0.0))
           << ";\n";
        // f_s = f_{s without its highest set bit} * R_high ; computed on the fly per s
        for (int s = 1; s < na_; s++) {
            int hi = 31 - __builtin_clz(unsigned(s));
            const int rest = s & ~(1 << hi);
            if (dirtyR_[hi]) o_ << "    const double2 f" << s << " = cmul(f" << rest << ", R" << hi << ");\n";
            else o_ << "    const double2 f" << s << " = f" << rest << ";\n";
        }
        for (int s = 0; s < na_; s++)
            mulAmp(s, dOne(s) ? "f" + std::to_string(s) : mulK("f" + std::to_string(s), D[2 * s], D[2 * s + 1]));
        o_ << "  }\n  P = C2(1.0, 0.0);\n";
        for (int k = 0; k < rb_; k++)
            if (dirtyR_[k]) o_ << "  R" << k << " = C2(1.0, 0.0);\n";
        dirtyP_ = false;
        for (int k = 0; k < rb_; k++) dirtyR_[k] = false;
    }

    const PassParams& P_;
    int ct_, rb_, na_, nt_;
    bool pipe_;
    std::vector<int> nm_;
    bool dirtyP_ = false;
    bool dirtyR_[qkdev::kMaxRegBits] = {};
    std::ostringstream o_;
};

// ---- compile / load / launch -------------------------------------------------

// Bump when the generated code changes for the same PassParams (on-disk cache key).
constexpr uint64_t kGeneratorVersion = 35;

uint64_t hashPass(const PassParams& P) {
    uint64_t h = 1469598103934665603ull ^ (kGeneratorVersion * 0x9E3779B97F4A7C15ull) ^ (usePrefetch() ? 1u : 0u) ^ (usePersistent() ? 2u : 0u) ^ (useSparsePrefetch() ? 8u : 0u) ^
                 (qkdev::halfExchanges() ? 4u : 0u);
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&P);
    for (size_t i = 0; i < sizeof(PassParams); i++) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

// Driver API through dlopen: the library must load on hosts without libcuda.
struct Driver {
    using Res = int;
    Res (*moduleLoadData)(void**, const void*) = nullptr;
    Res (*moduleGetFunction)(void**, void*, const char*) = nullptr;
    Res (*funcSetAttribute)(void*, int, int) = nullptr;
    Res (*launchKernel)(void*, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, void*, void**,
                        void**) = nullptr;
    Res (*tensorMapEncodeTiled)(void*, int, unsigned, void*, const uint64_t*, const uint64_t*, const unsigned*,
                                const unsigned*, int, int, int, int) = nullptr;  // optional
    bool ok = false;
    Driver() {
        void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        moduleLoadData = reinterpret_cast<decltype(moduleLoadData)>(dlsym(h, "cuModuleLoadData"));
        moduleGetFunction = reinterpret_cast<decltype(moduleGetFunction)>(dlsym(h, "cuModuleGetFunction"));
        funcSetAttribute = reinterpret_cast<decltype(funcSetAttribute)>(dlsym(h, "cuFuncSetAttribute"));
        launchKernel = reinterpret_cast<decltype(launchKernel)>(dlsym(h, "cuLaunchKernel"));
        tensorMapEncodeTiled = reinterpret_cast<decltype(tensorMapEncodeTiled)>(dlsym(h, "cuTensorMapEncodeTiled"));
        ok = moduleLoadData && moduleGetFunction && funcSetAttribute && launchKernel;
    }
};

Driver& driver() {
    static Driver d;
    return d;
}

struct Entry {
    std::vector<char> cubin;
    std::map<int, void*> func;  // device -> CUfunction
};

std::mutex g_mu;
std::map<uint64_t, Entry> g_cache;

std::string kernelName(uint64_t h) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "qk_pass_%016llx", static_cast<unsigned long long>(h));
    return buf;
}

// On-disk cubin cache.  Directory: QK_JIT_CACHE, else $XDG_CACHE_HOME/qk_jit,
// else $HOME/.cache/qk_jit, else /tmp/qk_jit_cache_<uid>; created 0700 and
// used only if this user owns it and nobody else can write it.  Each file
// carries a header (magic, NVRTC version, target arch, hash of the generated
// source, length and FNV-1a checksum of the cubin) that must match before the
// cubin is loaded; anything else is recompiled.  Files are written to a temp
// name and renamed into place only after a complete, checked write.
uint64_t fnv1a(const char* p, size_t n) {
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < n; i++) h = (h ^ uint64_t(uint8_t(p[i]))) * 1099511628211ull;
    return h;
}

struct CacheHeader {
    char magic[8];        // "QKJIT02\0"
    int32_t nvrtcMajor, nvrtcMinor;
    char arch[16];        // "sm_100a"
    uint64_t sourceHash;  // FNV-1a of the generated CUDA source
    uint64_t size;        // cubin bytes
    uint64_t checksum;    // FNV-1a of the cubin
};

bool makePrivateDir(const std::string& dir) {
    std::string cur;
    for (size_t i = 0; i <= dir.size(); i++) {
        if (i < dir.size() && dir[i] != '/') continue;
        cur = dir.substr(0, i);
        if (cur.empty()) continue;
        if (mkdir(cur.c_str(), 0700) != 0 && errno != EEXIST) return false;
    }
    struct stat sb;
    if (stat(dir.c_str(), &sb) != 0 || !S_ISDIR(sb.st_mode)) return false;
    return sb.st_uid == getuid() && (sb.st_mode & (S_IWGRP | S_IWOTH)) == 0;
}

const std::string& cacheDir() {  // "" = no disk cache
    static const std::string dir = [] {
        std::string d;
        if (const char* e = std::getenv("QK_JIT_CACHE")) d = e;
        else if (const char* x = std::getenv("XDG_CACHE_HOME")) d = std::string(x) + "/qk_jit";
        else if (const char* h = std::getenv("HOME")) d = std::string(h) + "/.cache/qk_jit";
        else d = "/tmp/qk_jit_cache_" + std::to_string(getuid());
        return makePrivateDir(d) ? d : std::string();
    }();
    return dir;
}

CacheHeader headerFor(const std::string& src, const std::vector<char>& bin);

std::vector<char> cubinFor(const PassParams& P, uint64_t h) {
    const std::string src = generatePassSource(P, kernelName(h));
    const std::string& dir = cacheDir();
    const std::string path = dir.empty() ? std::string() : dir + "/" + kernelName(h) + ".cubin";
    if (!path.empty()) {
        std::ifstream in(path, std::ios::binary);
        CacheHeader hd{};
        if (in && in.read(reinterpret_cast<char*>(&hd), sizeof hd)) {
            std::vector<char> bin(hd.size < (uint64_t(1) << 30) ? size_t(hd.size) : 0);
            const CacheHeader want = headerFor(src, bin);
            if (!bin.empty() && in.read(bin.data(), std::streamsize(bin.size())) &&
                std::memcmp(hd.magic, want.magic, sizeof hd.magic) == 0 && hd.nvrtcMajor == want.nvrtcMajor &&
                hd.nvrtcMinor == want.nvrtcMinor && std::memcmp(hd.arch, want.arch, sizeof hd.arch) == 0 &&
                hd.sourceHash == want.sourceHash && hd.checksum == fnv1a(bin.data(), bin.size()))
                return bin;
        }
    }
    std::vector<char> bin = compileToCubin(src, kernelName(h));
    if (!path.empty()) {
        const CacheHeader hd = headerFor(src, bin);
        const std::string tmp = path + ".tmp" + std::to_string(getpid()) + "_" +
                                std::to_string(reinterpret_cast<uintptr_t>(&bin));
        bool ok;
        {
            std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
            out.write(reinterpret_cast<const char*>(&hd), sizeof hd);
            out.write(bin.data(), std::streamsize(bin.size()));
            out.close();
            ok = bool(out);
        }
        if (!ok || std::rename(tmp.c_str(), path.c_str()) != 0) std::remove(tmp.c_str());
    }
    return bin;
}

void* functionFor(const PassParams& P, uint64_t h, int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    Entry& e = g_cache[h];
    auto it = e.func.find(device);
    if (it != e.func.end()) return it->second;
    if (e.cubin.empty()) throw SimulationError("jit: pass not prepared");
    Driver& d = driver();
    if (!d.ok) throw SimulationError("jit: libcuda.so.1 not available");
    void* mod = nullptr;
    void* fn = nullptr;
    if (d.moduleLoadData(&mod, e.cubin.data()) != 0) throw SimulationError("jit: cuModuleLoadData failed");
    if (d.moduleGetFunction(&fn, mod, kernelName(h).c_str()) != 0) throw SimulationError("jit: cuModuleGetFunction failed");
    const int smem = int(kernelSmem(P));
    if (smem > 48 * 1024 && d.funcSetAttribute(fn, 8 /*CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES*/, smem) != 0)
        throw SimulationError("jit: cuFuncSetAttribute failed");
    e.func[device] = fn;
    return fn;
}

}  // namespace

std::string generatePassSource(const PassParams& P, const std::string& name) { return Gen(P).run(name); }

namespace {
// NVRTC, loaded by absolute path with RTLD_LOCAL: a process that imported
// torch first already has torch's own libnvrtc.so.12 (an older 12.x) under the
// same soname, whose ptxas rejects sm_100 256-bit accesses.  QK_NVRTC_PATH
// overrides the path.
struct Nvrtc {
    nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
    nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
    nvrtcResult (*logSize)(nvrtcProgram, size_t*) = nullptr;
    nvrtcResult (*getLog)(nvrtcProgram, char*) = nullptr;
    nvrtcResult (*cubinSize)(nvrtcProgram, size_t*) = nullptr;
    nvrtcResult (*getCubin)(nvrtcProgram, char*) = nullptr;
    nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
    nvrtcResult (*version)(int*, int*) = nullptr;
    int major = 0, minor = 0;
    Nvrtc() {
        const char* env = std::getenv("QK_NVRTC_PATH");
        const char* paths[] = {env, "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12"};
        for (const char* path : paths) {
            if (!path) continue;
            void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
            if (!h) continue;
            create = reinterpret_cast<decltype(create)>(dlsym(h, "nvrtcCreateProgram"));
            compile = reinterpret_cast<decltype(compile)>(dlsym(h, "nvrtcCompileProgram"));
            logSize = reinterpret_cast<decltype(logSize)>(dlsym(h, "nvrtcGetProgramLogSize"));
            getLog = reinterpret_cast<decltype(getLog)>(dlsym(h, "nvrtcGetProgramLog"));
            cubinSize = reinterpret_cast<decltype(cubinSize)>(dlsym(h, "nvrtcGetCUBINSize"));
            getCubin = reinterpret_cast<decltype(getCubin)>(dlsym(h, "nvrtcGetCUBIN"));
            destroy = reinterpret_cast<decltype(destroy)>(dlsym(h, "nvrtcDestroyProgram"));
            version = reinterpret_cast<decltype(version)>(dlsym(h, "nvrtcVersion"));
            if (create && compile && logSize && getLog && cubinSize && getCubin && destroy && version) {
                version(&major, &minor);
                return;
            }
        }
        create = nullptr;
    }
};
Nvrtc& nvrtc() {
    static Nvrtc n;
    return n;
}

CacheHeader headerFor(const std::string& src, const std::vector<char>& bin) {
    CacheHeader h{};
    std::memcpy(h.magic, "QKJIT02", 8);
    h.nvrtcMajor = nvrtc().major;
    h.nvrtcMinor = nvrtc().minor;
    std::snprintf(h.arch, sizeof h.arch, "%s", "sm_100a");
    h.sourceHash = fnv1a(src.data(), src.size());
    h.size = bin.size();
    h.checksum = fnv1a(bin.data(), bin.size());
    return h;
}
}  // namespace

bool nvrtcSupportsWideAccess() {
    const Nvrtc& n = nvrtc();
    return n.create && (n.major > 12 || (n.major == 12 && n.minor >= 9));
}

std::vector<char> compileToCubin(const std::string& src, const std::string& name) {
    Nvrtc& N = nvrtc();
    if (!N.create) throw SimulationError("jit: libnvrtc.so.12 not found (set QK_NVRTC_PATH)");
    nvrtcProgram prog;
    if (N.create(&prog, src.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS)
        throw SimulationError("jit: nvrtcCreateProgram failed");
    const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device", "-lineinfo",
                          "-I/usr/local/cuda/include", "-diag-suppress=177"};
    const nvrtcResult r = N.compile(prog, 6, opts);
    if (r != NVRTC_SUCCESS) {
        size_t n = 0;
        N.logSize(prog, &n);
        std::string log(n, '\0');
        N.getLog(prog, &log[0]);
        N.destroy(&prog);
        std::string errs;  // error lines first (warnings can be long)
        std::istringstream ls(log);
        for (std::string line; std::getline(ls, line);)
            if (line.find("error") != std::string::npos) errs += line + "\n";
        throw SimulationError("jit: NVRTC failed: " + (errs + log).substr(0, 3000));
    }
    size_t n = 0;
    N.cubinSize(prog, &n);
    std::vector<char> bin(n);
    N.getCubin(prog, bin.data());
    N.destroy(&prog);
    return bin;
}

namespace {
std::atomic<int>& minQubitsVar() {
    static std::atomic<int> v{[] {
        const char* e = std::getenv("QK_JIT_MIN_QUBITS");
        return e ? std::atoi(e) : 22;
    }()};
    return v;
}
}  // namespace

int minQubits() { return minQubitsVar().load(); }
void setMinQubits(int v) { minQubitsVar().store(v); }

void prepare(const std::vector<const PassParams*>& passes, int device) {
    std::vector<std::pair<uint64_t, const PassParams*>> todo;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        std::map<uint64_t, bool> seen;
        for (const PassParams* P : passes) {
            const uint64_t h = hashPass(*P);
            if (seen[h] || !g_cache[h].cubin.empty()) continue;
            seen[h] = true;
            todo.emplace_back(h, P);
        }
    }
    std::atomic<size_t> next{0};
    std::string err;
    std::mutex errMu;
    auto worker = [&] {
        for (size_t i; (i = next++) < todo.size();) {
            try {
                std::vector<char> bin = cubinFor(*todo[i].second, todo[i].first);
                std::lock_guard<std::mutex> lk(g_mu);
                g_cache[todo[i].first].cubin = std::move(bin);
            } catch (const std::exception& e) {
                std::lock_guard<std::mutex> lk(errMu);
                err = e.what();
            }
        }
    };
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < std::min<unsigned>(hw, unsigned(todo.size())); t++) ts.emplace_back(worker);
    for (auto& t : ts) t.join();
    if (!err.empty()) throw SimulationError(err);
    for (const PassParams* P : passes) functionFor(*P, hashPass(*P), device);
}

cudaError_t launch(const PassParams& P, double2* state, const double2* gtab, int nLocal, uint64_t basis,
                   cudaStream_t stream, double* np, uint64_t smask, uint64_t sval, bool zeroFill, int zeroSkip) {
    int dev = 0;
    cudaGetDevice(&dev);
    void* fn = functionFor(P, hashPass(P), dev);
    unsigned ntiles = unsigned(uint64_t(1) << (nLocal - P.ct));
    unsigned tile0 = 0;
    unsigned ctas;
    const bool pipe = pipelined(P);
    if (basis != ~uint64_t(0)) {
        // First pass of a run: every tile but the one holding |basis> is zeros
        // in and zeros out -- memset the slice, compute that one tile.
        if (zeroFill) {  // else the next pass writes every tile (launched with smask / sval)
            const cudaError_t e = cudaMemsetAsync(state, 0, sizeof(double2) << nLocal, stream);
            if (e != cudaSuccess) return e;
        }
        if (basis >> nLocal) return cudaSuccess;  // the basis state lives on another rank
        uint32_t t = 0, q = 0;  // tile index = the basis's non-tile bits, compacted
        for (int b = 0; b < nLocal; b++)
            if (!((P.tile_mask >> b) & 1)) t |= uint32_t((basis >> b) & 1) << q++;
        tile0 = t;
        ntiles = t + 1;
        ctas = 1;
    } else {
        if (zeroSkip == 2)  // only the tiles meeting the support
            ntiles = unsigned(uint64_t(1) << (nLocal - P.ct - __builtin_popcountll(smask & ~P.tile_mask)));
        const unsigned resident = unsigned(smCount(dev) * blocksPerSm(P.ct, P.rb));
        ctas = (ntiles < resident || !(usePersistent() || pipe)) ? ntiles : resident;
    }
    int lo[5], tb[5], swizzle = 0;
    int nd = pipe ? tensorLayout(P, lo, tb, &swizzle) : stagedLayout(P, lo, tb, &swizzle);
    const bool staged = !pipe && nd > 0;
    if (!pipe && !staged && prefetchTiles(P)) nd = tensorDims(P, lo, tb);
    const unsigned nt = 1u << (P.ct - P.rb);
    const unsigned smem = kernelSmem(P);
    unsigned zskip = unsigned(zeroSkip);
    // TMA-pipelined kernels: the tile as one box of a tensor view of the
    // slice (tensorDims), so a tile moves in one TMA op instead of one per row.
    alignas(64) uint64_t tmap[16] = {};
    unsigned tmv = 0;
    if (nd && (useTensorMaps() || swizzle || !pipe) && driver().tensorMapEncodeTiled && nLocal - lo[nd - 1] <= 32) {
        uint64_t dim[5], stride[4];
        unsigned box[5], es[5];
        for (int d = 0; d < nd; d++) {
            const int hi = d + 1 < nd ? lo[d + 1] : nLocal;
            dim[d] = uint64_t(1) << (hi - lo[d] + (d ? 0 : 1));
            box[d] = 1u << (tb[d] + (d ? 0 : 1) - (!pipe && d == nd - 1 ? 1 : 0));  // plain kernels: half boxes
            es[d] = 1u;
            if (d) stride[d - 1] = uint64_t(16) << lo[d];
        }
        constexpr int kFloat64 = 8, kL2Promote256 = 3;  // CU_TENSOR_MAP_DATA_TYPE_FLOAT64, ..._L2_PROMOTION_L2_256B
        if (driver().tensorMapEncodeTiled(tmap, kFloat64, unsigned(nd), state, dim, stride, box, es, 0, swizzle,
                                          kL2Promote256, 0) == 0)
            tmv = 1;
    }
    if (pipe && nd && swizzle && !tmv) return cudaErrorInvalidValue;  // a swizzled PB needs the tensor map
    // staged stores drain while the CTA's next tile computes: a persistent grid
    if (staged && tmv && (smask != 0 || P.stage_out == 2) && basis == ~uint64_t(0)) {
        const unsigned resident = unsigned(smCount(dev) * blocksPerSm(P.ct, P.rb));
        ctas = std::min(ntiles - tile0, resident);
    }
    void* args[] = {&state, &gtab, &ntiles, &basis, &tile0, &np, &smask, &sval, &zskip, tmap, &tmv};
    if (driver().launchKernel(fn, ctas, 1, 1, nt, 1, 1, smem, stream, args, nullptr) != 0)
        return cudaErrorLaunchFailure;
    return cudaSuccess;
}

}  // namespace qkjit
