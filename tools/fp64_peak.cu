// FP64 peak microbenchmark for the pass roofline's compute side (B200, sm_100a).
//   dfma: every thread runs 8 independent DFMA chains (FMA = 2 flop)
//   dmma: every warp runs 4 independent mma.sync.m8n8k4.f64 chains (512 flop each)
// Timed with CUDA events after a warm-up, grid = 148 SMs x resident CTAs, prints
// one JSON line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

constexpr int kIters = 1 << 14;

__global__ void dfma_kernel(double* out, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;  // never true; keeps the chains live
}

__global__ void dmma_kernel(double* out, double a0, double b0) {
    double a = a0 + threadIdx.x * 1e-6, b = b0 - threadIdx.x * 1e-6;
    double c[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess) {                                                        \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                    \
        }                                                                               \
    } while (0)

template <typename K>
double run(K kern, int blocks, int threads, double flop_per_thread_iter, double* out) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int w = 0; w < 3; ++w) kern<<<blocks, threads>>>(out, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        kern<<<blocks, threads>>>(out, 1.0000001, 1e-9);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    const double flops = double(blocks) * threads * kIters * flop_per_thread_iter;
    return flops / (best * 1e-3) / 1e12;
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    double* out;
    CK(cudaMalloc(&out, 1024 * sizeof(double)));
    const int sms = p.multiProcessorCount;
    double best_dfma = 0, best_dmma = 0;
    int bd = 0, bm = 0;
    for (int per_sm : {2, 4, 8}) {
        const double t = run(dfma_kernel, sms * per_sm, 256, 8 * 2.0, out);
        if (t > best_dfma) best_dfma = t, bd = per_sm;
        // per warp: 4 mma of 8x8x4 (2 flop per MAC) = 4 * 512 flop / 32 threads
        const double m = run(dmma_kernel, sms * per_sm, 256, 4 * 512.0 / 32.0, out);
        if (m > best_dmma) best_dmma = m, bm = per_sm;
    }
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("{\"device\": \"%s\", \"sms\": %d, \"dfma_tflops\": %.3f, \"dfma_ctas_per_sm\": %d, "
           "\"dmma_tflops\": %.3f, \"dmma_ctas_per_sm\": %d, \"max_clock_mhz\": %d}\n",
           p.name, sms, best_dfma, bd, best_dmma, bm, clk_khz / 1000);
    return 0;
}
