// tmem_bw.cu -- microbenchmark: tcgen05.ld / tcgen05.st throughput per SM
// (informs where the heat kernel's per-thread pipeline state can live).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tools/tmem_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int NW, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) tmem_kernel(int iters, unsigned long long* out, double* sink) {
    __shared__ unsigned base;
    __shared__ double sm[NW * 32 * 8];
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const unsigned ta = base + (static_cast<unsigned>(32 * (warp & 3)) << 16) + 64u * (warp >> 2);
    unsigned acc = 0;
    double dacc = 0.0;
    for (int i = 0; i < NW * 32 * 8; i += NW * 32) sm[i + threadIdx.x] = threadIdx.x;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // tcgen05.ld 32x32b.x8 (32 B per thread), 4 in flight, one wait
            unsigned r[32];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                             : "=r"(r[8 * q]), "=r"(r[8 * q + 1]), "=r"(r[8 * q + 2]), "=r"(r[8 * q + 3]),
                               "=r"(r[8 * q + 4]), "=r"(r[8 * q + 5]), "=r"(r[8 * q + 6]), "=r"(r[8 * q + 7])
                             : "r"(ta + 8 * q));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int q = 0; q < 32; ++q) acc += r[q];
        } else if (MODE == 1) {  // tcgen05.st 32x32b.x8
#pragma unroll
            for (int q = 0; q < 4; ++q)
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(
                                 ta + 8 * q),
                             "r"(acc + q));
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            acc += 1;
        } else if (MODE == 2) {  // LDS.64: 16 conflict-free loads per thread
            const double* p = sm + threadIdx.x;
#pragma unroll
            for (int q = 0; q < 16; ++q) dacc += p[((q + it) & 7) * NW * 32];
        } else {  // SHFL: 16 independent 32-bit shuffles per thread
            unsigned v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = __shfl_down_sync(0xffffffffu, acc + q, 1 + (q & 1));
#pragma unroll
            for (int q = 0; q < 16; ++q) acc ^= v[q];
        }
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345 || dacc == 1.2345) sink[0] = acc + dacc;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(base));
}

template <int NW, int MODE>
void run(const char* name) {
    const int iters = 4096;
    unsigned long long* d;
    double* s;
    cudaMalloc(&d, 148 * sizeof(unsigned long long));
    cudaMalloc(&s, 8);
    tmem_kernel<NW, MODE><<<148, NW * 32>>>(iters, d, s);
    tmem_kernel<NW, MODE><<<148, NW * 32>>>(iters, d, s);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const double bytes = MODE == 2 ? 16.0 * 8 : MODE == 3 ? 16.0 * 4 : 4.0 * 32;  // per thread per iteration
    const double cyc = static_cast<double>(h[0]);
    printf("%-28s warps=%2d  %8.1f B/clk/SM  (%s)\n", name, NW, bytes * NW * 32 * iters / cyc,
           cudaGetErrorString(e));
    cudaFree(d);
    cudaFree(s);
}

int main() {
    run<4, 0>("tcgen05.ld 32x32b.x8 x4");
    run<8, 0>("tcgen05.ld 32x32b.x8 x4");
    run<16, 0>("tcgen05.ld 32x32b.x8 x4");
    run<4, 1>("tcgen05.st 32x32b.x8 x4");
    run<8, 1>("tcgen05.st 32x32b.x8 x4");
    run<8, 2>("LDS.64 reference");
    run<16, 2>("LDS.64 reference");
    run<8, 3>("SHFL.32 (bytes = 4/lane)");
    run<16, 3>("SHFL.32 (bytes = 4/lane)");
    run<32, 3>("SHFL.32 (bytes = 4/lane)");
    return 0;
}
