// Exact-mode instantiations: compiled with -fmad=false -DPIRK_TU_EXACT=1, so
// every kernel here rounds exactly like the reference's non-FMA build.
#include "chain.cuh"
#include "heat2x2.cuh"
#include "small.cuh"

namespace pirk {

template cudaError_t launch_chain_step<true>(const ChainModel&, const WindowArgs&,
                                             const StepConsts&, unsigned long long,
                                             unsigned long long*, cudaStream_t);
template cudaError_t launch_chain_steps<true>(const ChainModel&, const WindowArgs&, const StepConstsN&, int,
                                                unsigned long long, unsigned long long*, cudaStream_t);
template cudaError_t launch_heat_step<true>(const HeatModel&, const WindowArgs&,
                                            const StepConsts&, unsigned long long,
                                            unsigned long long*, cudaStream_t, int);
template cudaError_t launch_small_integrate<true>(const SmallModel&, int, const double*,
                                                  const double*, double, double, double,
                                                  unsigned long long, unsigned long long,
                                                  double*, unsigned long long*, cudaStream_t);
template cudaError_t launch_monte_carlo<true>(const SmallModel&, const McArgs&, cudaStream_t);

// ---------------------------------------------------------------- epilogues

__global__ void order_check_kernel(const double* __restrict__ lo, const double* __restrict__ hi,
                                   uint64_t n, unsigned long long* fail) {
    // reach.cpp:181-186: first i with lo[i] > hi[i]
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (lo[i] > hi[i]) atomicMin(fail, (unsigned long long)i);
}

__global__ void gb_box_kernel(const double* __restrict__ c, const double* __restrict__ r,
                              double* __restrict__ lo, double* __restrict__ hi, uint64_t n,
                              unsigned long long* neg) {
    // reach.cpp:121-134 clamp, then from_center_radius (interval.cpp:49-50)
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double ri = r[i];
        if (ri < 0.0) {
            if (ri < -1e-12) atomicMin(neg, (unsigned long long)i);
            ri = 0.0;
        }
        lo[i] = c[i] - ri;
        hi[i] = c[i] + ri;
    }
}

__global__ void gb_negval_kernel(const double* r, const unsigned long long* neg, double* out) {
    if (*neg != ~0ull) *out = r[*neg];
}

__global__ void box_check_kernel(const double* __restrict__ lo, const double* __restrict__ hi,
                                 uint64_t n, unsigned long long* bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (!finite_d(lo[i]) || !finite_d(hi[i]) || lo[i] > hi[i])
            atomicMin(bad, (unsigned long long)i);
}

__global__ void center_radius_kernel(double* __restrict__ a, double* __restrict__ b, uint64_t n) {
    // interval.cpp:25-37: c = 0.5*(u+l), r = 0.5*(u-l)
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double l = a[i], u = b[i];
        a[i] = 0.5 * (u + l);
        b[i] = 0.5 * (u - l);
    }
}

__global__ void fill_kernel(unsigned long long* p, unsigned long long v, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// Cross-process step flag (pirk_signal_flag): stream order puts this after the
// launches that stored halo units into the peer's window; the system-scope
// fence plus release store make those stores visible to the peer GPU before
// the flag is.
__global__ void signal_flag_kernel(unsigned* flag, unsigned v) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}

static unsigned grid_for(uint64_t n) {
    uint64_t b = (n + 255) / 256;
    if (b > 148ull * 16) b = 148ull * 16;
    return static_cast<unsigned>(b ? b : 1);
}

cudaError_t launch_order_check(const double* lo, const double* hi, uint64_t n,
                               unsigned long long* fail, cudaStream_t stream) {
    order_check_kernel<<<grid_for(n), 256, 0, stream>>>(lo, hi, n, fail);
    return cudaGetLastError();
}
cudaError_t launch_gb_box(const double* c, const double* r, double* lo, double* hi, uint64_t n,
                          unsigned long long* neg, cudaStream_t stream) {
    gb_box_kernel<<<grid_for(n), 256, 0, stream>>>(c, r, lo, hi, n, neg);
    return cudaGetLastError();
}
cudaError_t launch_gb_negval(const double* r, const unsigned long long* neg, double* neg_val,
                             cudaStream_t stream) {
    gb_negval_kernel<<<1, 1, 0, stream>>>(r, neg, neg_val);
    return cudaGetLastError();
}
cudaError_t launch_box_check(const double* lo, const double* hi, uint64_t n,
                             unsigned long long* bad, cudaStream_t stream) {
    box_check_kernel<<<grid_for(n), 256, 0, stream>>>(lo, hi, n, bad);
    return cudaGetLastError();
}
cudaError_t launch_center_radius(double* a, double* b, uint64_t n, cudaStream_t stream) {
    center_radius_kernel<<<grid_for(n), 256, 0, stream>>>(a, b, n);
    return cudaGetLastError();
}
cudaError_t launch_fill(unsigned long long* p, unsigned long long v, uint64_t n,
                        cudaStream_t stream) {
    fill_kernel<<<grid_for(n), 256, 0, stream>>>(p, v, n);
    return cudaGetLastError();
}
cudaError_t launch_signal_flag(unsigned* flag, unsigned v, cudaStream_t stream) {
    signal_flag_kernel<<<1, 1, 0, stream>>>(flag, v);
    return cudaGetLastError();
}

}  // namespace pirk
