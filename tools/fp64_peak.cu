// fp64_peak.cu -- microbenchmark: FP64 pipe throughput of one B200
// (DFMA and DADD, independent chains, all SMs).  The roofline denominator of
// the FP64-bound kernels (Monte Carlo K3, chain K1): SURVEY.md 8(d) asks for a
// measured figure instead of the datasheet's ~37 TFLOP/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/fp64_peak tools/fp64_peak.cu
// Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;  // independent dependency chains per thread (covers DFMA latency)

template <int OP>  // 0: DFMA a = a*b + c, 1: DADD a = a + b, 2: DMUL a = a*b
__global__ void __launch_bounds__(256) fp64_kernel(int iters, double seed, double* sink) {
    double a[kChains];
    const double b = 1.0 + 1e-9 * threadIdx.x, c = 1e-12 * seed;
#pragma unroll
    for (int q = 0; q < kChains; ++q) a[q] = seed + q;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int q = 0; q < kChains; ++q) {
                if (OP == 0) a[q] = fma(a[q], b, c);
                else if (OP == 1) a[q] = a[q] + c;
                else a[q] = a[q] * b;
            }
        }
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kChains; ++q) s += a[q];
    if (s == 12345.678) sink[threadIdx.x] = s;  // keep the chains live
}

template <int OP>
double run(int sms, int blocks_per_sm, int iters, double* sink) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * blocks_per_sm;
    fp64_kernel<OP><<<grid, 256>>>(iters / 10, 1.0, sink);  // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        fp64_kernel<OP><<<grid, 256>>>(iters, 1.0, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double ops = double(grid) * 256 * iters * 16 * kChains;  // instructions (per thread)
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ops / (best * 1e-3);  // FP64 instructions per second
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double* sink;
    cudaMalloc(&sink, 4096 * sizeof(double));
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int sms = p.multiProcessorCount;
    const int iters = 4000;
    const double fma_ips = run<0>(sms, 8, iters, sink);
    const double add_ips = run<1>(sms, 8, iters, sink);
    const double mul_ips = run<2>(sms, 8, iters, sink);
    const double per_clk_sm = fma_ips / (double(sms) * clk_khz * 1e3);
    std::printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_mhz_nominal\": %.0f, "
                "\"dfma_per_s\": %.4e, \"dadd_per_s\": %.4e, \"dmul_per_s\": %.4e, "
                "\"fp64_tflops_fma\": %.3f, \"fp64_inst_per_clk_per_sm\": %.2f, "
                "\"how\": \"%d CTAs x 256 threads, %d independent chains/thread, best of 5, CUDA events\"}\n",
                p.name, sms, clk_khz / 1e3, fma_ips, add_ips, mul_ips, 2.0 * fma_ips / 1e12,
                per_clk_sm, sms * 8, kChains);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        std::fprintf(stderr, "cuda error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
