// Probe: does the memory layout of a pass's output tile (row length) bound a
// write-heavy pass?  One CTA (256 threads x 32 amplitudes, 2^13-amplitude
// tile) per SM, K dependent FP64 FMAs per amplitude, then the tile's stores
// under three layouts of the 13 tile bits in a 2^33-amplitude state:
//   scattered: thread bits -> memory bits {0,1,2,23,24,25,26,31}, slots ->
//              {32,29,30,27,28} (QFT-33 pass 3 as scheduled: 128-B rows)
//   rows4k:    thread bits -> {0..7}, slots -> {8, 29,30,27,28} (4-KB rows)
//   contig:    thread bits -> {0..7}, slots -> {8..12} (one 128-KB row)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a store_layout.cu -o /tmp/store_layout
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t dep(uint64_t v, const int* pos, int n) {
    uint64_t r = 0;
    for (int i = 0; i < n; i++) r |= ((v >> i) & 1ull) << pos[i];
    return r;
}

template <int LAYOUT>
__global__ void __launch_bounds__(256, 1) k_store(double2* st, int nq, int K, double seed, unsigned ntiles, int stagger) {
    extern __shared__ double2 pad[];
    int tb[8], sb[5];
    if (LAYOUT == 0) { int t[8] = {0, 1, 2, 23, 24, 25, 26, 31}; int s[5] = {32, 29, 30, 27, 28}; for (int i = 0; i < 8; i++) tb[i] = t[i]; for (int i = 0; i < 5; i++) sb[i] = s[i]; }
    if (LAYOUT == 1) { int s[5] = {8, 29, 30, 27, 28}; for (int i = 0; i < 8; i++) tb[i] = i; for (int i = 0; i < 5; i++) sb[i] = s[i]; }
    if (LAYOUT == 2) { for (int i = 0; i < 8; i++) tb[i] = i; for (int i = 0; i < 5; i++) sb[i] = 8 + i; }
    uint64_t tmask = 0;
    for (int i = 0; i < 8; i++) tmask |= 1ull << tb[i];
    for (int i = 0; i < 5; i++) tmask |= 1ull << sb[i];
    if (stagger && ((threadIdx.x >> 5) & 1)) __nanosleep(stagger);
    for (unsigned tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // tile index -> the non-tile bits
    uint64_t base = 0, t = tile;
    int q = 0;
    for (int b = 0; b < nq; b++)
        if (!((tmask >> b) & 1)) base |= ((t >> q++) & 1ull) << b;
    const uint64_t off = base | dep(threadIdx.x, tb, 8);
    double2 a[32];
#pragma unroll
    for (int s = 0; s < 32; s++) a[s] = make_double2(seed + s, seed - s);
    for (int k = 0; k < K; k++) {
#pragma unroll
        for (int s = 0; s < 32; s++) {
            a[s].x = fma(a[s].x, 0.999, a[s].y * 1e-3);
            a[s].y = fma(a[s].y, 0.999, -a[s].x * 1e-3);
        }
    }
#pragma unroll
    for (int s = 0; s < 32; s++) {
        uint64_t o = off;
        for (int i = 0; i < 5; i++) o |= uint64_t((s >> i) & 1) << sb[i];
        __stcs(st + o, a[s]);
    }
    }
}

// TMA variant: the tile (contiguous layout) is staged in shared memory and
// written by cp.async.bulk (ROWS rows per tile), draining while the next
// tile computes.
template <int ROWBYTES>
__global__ void __launch_bounds__(256, 1) k_store_tma(double2* st, int K, double seed, unsigned ntiles) {
    extern __shared__ __align__(128) double2 pb[];
    double2 a[32];
    for (unsigned tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
#pragma unroll
        for (int s = 0; s < 32; s++) a[s] = make_double2(seed + s + tile, seed - s);
        for (int k = 0; k < K; k++) {
#pragma unroll
            for (int s = 0; s < 32; s++) {
                a[s].x = fma(a[s].x, 0.999, a[s].y * 1e-3);
                a[s].y = fma(a[s].y, 0.999, -a[s].x * 1e-3);
            }
        }
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
#pragma unroll
        for (int s = 0; s < 32; s++) pb[(s << 8) | threadIdx.x] = a[s];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        constexpr int rows = (16 << 13) / ROWBYTES;
        for (int r = threadIdx.x; r < rows; r += 256) {
            const char* src = reinterpret_cast<const char*>(pb) + size_t(r) * ROWBYTES;
            char* dst = reinterpret_cast<char*>(st + (size_t(tile) << 13)) + size_t(r) * ROWBYTES;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                         "r"(unsigned(__cvta_generic_to_shared(src))), "r"(ROWBYTES) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const int nq = 33;
    double2* st;
    if (cudaMalloc(&st, sizeof(double2) << nq) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    const unsigned tiles = 1u << (nq - 13);
    const int smem = 120 * 1024;  // 1 CTA per SM
    cudaFuncSetAttribute(k_store<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Case { int K; unsigned grid; int stagger; const char* what; };
    const Case cases[] = {{0, tiles, 0, "one CTA per tile"}, {0, 148, 0, "persistent 148"}, {0, 74, 0, "persistent 74 SMs"},
                          {0, 37, 0, "persistent 37 SMs"}, {8, tiles, 0, "one CTA per tile"}, {8, 148, 0, "persistent 148"},
                          {8, 148, 1000, "persistent, odd warps +1us"}, {8, 148, 2000, "persistent, odd warps +2us"},
                          {8, 74, 0, "persistent 74 SMs"}};
    for (const Case& c : cases) {
        float best = 1e9;
        for (int r = 0; r < 3; r++) {
            cudaEventRecord(e0);
            k_store<2><<<c.grid, 256, smem>>>(st, nq, c.K, 1.0, tiles, c.stagger);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("K=%2d grid %7u %-28s %8.2f ms  %6.0f GB/s write\n", c.K, c.grid, c.what, best,
               double(sizeof(double2) << nq) / (best * 1e-3) / 1e9);
    }
    const int tsmem = 128 * 1024 + 1024;
    cudaFuncSetAttribute(k_store_tma<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);
    cudaFuncSetAttribute(k_store_tma<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);
    cudaFuncSetAttribute(k_store_tma<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);
    struct TCase { int K; unsigned grid; int row; };
    const TCase tc[] = {{0, 148, 4096}, {0, 74, 4096}, {0, 37, 4096}, {0, 148, 16384}, {0, 37, 16384}, {0, 148, 512}, {0, 37, 512},
                        {8, 148, 4096}, {8, 148, 16384}, {8, 148, 512}};
    for (const TCase& c : tc) {
        float best = 1e9;
        for (int r = 0; r < 3; r++) {
            cudaEventRecord(e0);
            if (c.row == 4096) k_store_tma<4096><<<c.grid, 256, tsmem>>>(st, c.K, 1.0, tiles);
            if (c.row == 16384) k_store_tma<16384><<<c.grid, 256, tsmem>>>(st, c.K, 1.0, tiles);
            if (c.row == 512) k_store_tma<512><<<c.grid, 256, tsmem>>>(st, c.K, 1.0, tiles);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("TMA K=%2d grid %4u rows %5d B %8.2f ms  %6.0f GB/s write\n", c.K, c.grid, c.row, best,
               double(sizeof(double2) << nq) / (best * 1e-3) / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
