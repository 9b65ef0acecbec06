// FP64 peak on this B200: DFMA on CUDA cores vs DMMA (mma.sync m8n8k4 f64 tensor
// path).  Evidence for DESIGN.md: the fused-gate kernels stay on DFMA unless
// DMMA is measurably faster (north star).  Build & run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_dfma(double* out, double a, double b) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < kIters; it++)
#pragma unroll
        for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) s += x[i];
    if (s == 123.456) out[0] = s;
}

__global__ void k_dmma(double* out, double a) {
    // 4 independent 8x8x4 accumulators per warp
    double c[4][2];
    double av = a + threadIdx.x * 1e-12, bv = 1.0 - threadIdx.x * 1e-12;
#pragma unroll
    for (int j = 0; j < 4; j++) c[j][0] = c[j][1] = 0.0;
    for (int it = 0; it < kIters; it++)
#pragma unroll
        for (int j = 0; j < 4; j++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[j][0]), "+d"(c[j][1])
                         : "d"(av), "d"(bv));
    double s = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1];
    if (s == 123.456) out[0] = s;
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256;
    float ms;
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, 1.0000001, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    const double dfma_flops = 2.0 * 16 * kIters * double(blocks) * threads;
    std::printf("DFMA  %.2f TFLOP/s (FP64 CUDA cores)\n", dfma_flops / (ms * 1e-3) / 1e12);
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(out, 1.0000001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    const double dmma_flops = 2.0 * 8 * 8 * 4 * 4 * kIters * double(blocks) * (threads / 32);
    std::printf("DMMA  %.2f TFLOP/s (mma.sync m8n8k4 f64)\n", dmma_flops / (ms * 1e-3) / 1e12);
    std::printf("sms %d err %s\n", sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
