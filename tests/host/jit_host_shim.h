// TEST INFRASTRUCTURE: lets a generated specialized pass kernel (jit.cpp's
// CUDA source) compile and run on the CPU with g++.  One std::thread per CUDA
// thread of a CTA, std::barrier for __syncthreads, one CTA at a time with a
// static shared-memory array.  Semantics only (no performance meaning).
#pragma once
#include <barrier>
#include <cmath>
#include <cstring>
#include <memory>
#include <cstdint>
#include <thread>
#include <type_traits>
#include <vector>

struct double2 {
    double x, y;
};
static inline double2 make_double2(double x, double y) { return {x, y}; }
struct QkDim3 {
    unsigned x;
};
inline thread_local unsigned qk_tl_tid = 0, qk_tl_bid = 0;
#define threadIdx (QkDim3{qk_tl_tid})
#define blockIdx (QkDim3{qk_tl_bid})
inline unsigned qk_grid = 1;
#define gridDim (QkDim3{qk_grid})
inline std::barrier<>* qk_bar = nullptr;
static inline void __syncthreads() { qk_bar->arrive_and_wait(); }
static inline void __syncwarp() {}
// Warp shuffles: per-warp exchange slots + a 32-thread barrier.
struct QkWarp {
    std::barrier<>* bar;
    double buf[32];
};
inline QkWarp* qk_warps = nullptr;
static inline double __shfl_xor_sync(unsigned, double v, int o) {
    QkWarp& w = qk_warps[qk_tl_tid >> 5];
    const unsigned l = qk_tl_tid & 31u;
    w.buf[l] = v;
    w.bar->arrive_and_wait();
    const double r = w.buf[l ^ unsigned(o)];
    w.bar->arrive_and_wait();
    return r;
}
template <class T>
static inline T __ldcs(const T* p) { return *p; }
template <class T>
static inline T __ldg(const T* p) { return *p; }
template <class T>
static inline void __stcs(T* p, T v) { *p = v; }
#define __global__
#define __device__
#define __forceinline__ inline
#define __launch_bounds__(a, b)
#define __restrict__
#define __shared__
#define __grid_constant__
#define __align__(n) alignas(n)
// `extern __shared__ double2 sm[];` in the kernel binds to this array.
extern "C" double2 sm[1 << 14];

// Launch: a persistent grid of min(ntiles, 3) CTAs run one after another
// (each walks its tiles), nt threads each.
// qk_host_launch2: tiles [tile0, ntiles) (0 = all) with the known-zero
// coset (smask, sval), as the runtime launches the passes of a basis run.
#define QK_HOST_LAUNCHER(KERNEL)                                                              \
    double2 sm[1 << 14];                                                                      \
    extern "C" void qk_host_launch2(double2* st, const double2* gt, int nLocal, int ct, int rb,   \
                                    unsigned long long basis, unsigned tile0, unsigned tiles,   \
                                    unsigned long long smask, unsigned long long sval,          \
                                    unsigned zskip) {                                           \
        const unsigned ntiles = tiles ? tiles : 1u << (nLocal - ct), nt = 1u << (ct - rb);   \
        std::vector<double> npv(size_t(ntiles) * (nt >= 32u ? nt / 32u : 1u)); /* norm partials */ \
        double* const np = npv.data();                                                        \
        qk_grid = ntiles - tile0 < 3u ? ntiles - tile0 : 3u;                                  \
        for (unsigned b = 0; b < qk_grid; b++) {                                              \
            std::barrier<> bar(nt);                                                           \
            qk_bar = &bar;                                                                    \
            std::vector<std::unique_ptr<std::barrier<>>> wbars;                               \
            std::vector<QkWarp> warps(nt / 32 + 1);                                           \
            for (unsigned w = 0; w < nt / 32 + 1; w++) {                                      \
                wbars.push_back(std::make_unique<std::barrier<>>(nt >= 32 ? 32 : nt));        \
                warps[w].bar = wbars.back().get();                                            \
            }                                                                                 \
            qk_warps = warps.data();                                                          \
            std::vector<std::thread> ts;                                                      \
            for (unsigned t = 0; t < nt; t++)                                                 \
                ts.emplace_back([=] {                                                         \
                    qk_tl_tid = t;                                                            \
                    qk_tl_bid = b;                                                            \
                    auto call = [&](auto k) { /* TMA-pipelined kernels: no tensor map (rows) */ \
                        if constexpr (std::is_invocable_v<decltype(k), double2*, const double2*,    \
                                          unsigned, unsigned long long, unsigned, double*,          \
                                          unsigned long long, unsigned long long, unsigned,         \
                                          QkTmap, unsigned>)                                        \
                            k(st, gt, ntiles, basis, tile0, np, smask, sval, zskip, QkTmap{}, 0u);  \
                        else                                                                        \
                            k(st, gt, ntiles, basis, tile0, np, smask, sval, zskip);                \
                    };                                                                              \
                    call(KERNEL);                                                                   \
                });                                                                           \
            for (auto& th : ts) th.join();                                                    \
        }                                                                                     \
    }                                                                                         \
    extern "C" void qk_host_launch(double2* st, const double2* gt, int nLocal, int ct, int rb,    \
                                   unsigned long long basis) {                              \
        qk_host_launch2(st, gt, nLocal, ct, rb, basis, 0u, 0u, 0ull, 0ull, 0u);                \
    }
