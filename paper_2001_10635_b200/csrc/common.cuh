// common.cuh -- shared device helpers for the PIRK B200 kernels.
//
// Arithmetic modes.  Each kernel template takes `bool Exact`.  Exact
// instantiations live in *_exact.cu translation units compiled with
// -fmad=false (PIRK_TU_EXACT=1), so plain C++ expressions round exactly like
// the reference's non-FMA x86-64 build (SURVEY.md 8c "Arithmetic regime") and
// follow its left-to-right expression order.  Fast instantiations live in
// *_fast.cu compiled with FMA contraction and may restructure expressions
// (reciprocal constants, sum-then-subtract stencils) within the tolerance
// contract of SURVEY.md 8(d).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifndef PIRK_TU_EXACT
#error "define PIRK_TU_EXACT (1 in -fmad=false translation units, 0 otherwise)"
#endif

namespace pirk {

// A kernel instantiated with Exact must come from an exact TU and vice versa.
template <bool Exact>
struct ModeCheck {
    static_assert(Exact == (PIRK_TU_EXACT != 0),
                  "exact kernels must be compiled with -fmad=false (PIRK_TU_EXACT=1)");
};

// std::min / std::max semantics: min(a,b) = (b < a) ? b : a (libstdc++).
__device__ __forceinline__ double ref_min(double a, double b) { return (b < a) ? b : a; }

// Non-finite check without relying on fast-math-sensitive isfinite.
// Cheap screen over 8 doubles on the FP32 pipe: the high word of a double
// read as a float is inf / NaN whenever the double is (its exponent bits 30..23
// are all ones).  A float sum of the 8 words is therefore non-finite whenever
// some value is; it can also be non-finite for finite values >= 2^1009 (huge
// words overflowing the float sum), so a true result only means "check each
// value with finite_d" (the callers' cold paths do).
__device__ __forceinline__ bool maybe_nonfinite8(const double (&y)[8]) {
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = __int_as_float(__double2hiint(y[i]));
    const float s = ((f[0] + f[1]) + (f[2] + f[3])) + ((f[4] + f[5]) + (f[6] + f[7]));
    return (__float_as_int(s) & 0x7f800000) == 0x7f800000;
}

__device__ __forceinline__ bool finite_d(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return ((b >> 52) & 0x7ffull) != 0x7ffull;
}

// Failure key: (step << 40) | component, min-reduced with atomicMin so the
// first failing step and, within it, the lowest component win -- the order in
// which the reference scans (rk4.cpp:72-75, rk4_serial.cpp:48-50).
constexpr int kFailCompBits = 40;
constexpr unsigned long long kNoFail = ~0ull;

__device__ __forceinline__ void record_fail(unsigned long long* fail, unsigned long long step,
                                            unsigned long long comp) {
    if (fail) atomicMin(fail, (step << kFailCompBits) | comp);
}

// Monotone map double -> uint64 for atomic min/max of doubles (exact; -0 < +0).
__device__ __forceinline__ unsigned long long ord_key(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double ord_val(unsigned long long k) {
    const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(b));
#else
    double d;
    __builtin_memcpy(&d, &b, sizeof d);
    return d;
#endif
}

// Per-step RK4 constants, computed on the host exactly as rk4.cpp:99-100 and
// :38-39 do (t = t0 + k*h, hk = last ? t1 - t : h, h2 = 0.5*hk, h6 = hk/6).
struct StepConsts {
    double t, hk, h2, h6;
};

// rng.hpp:11-23 -- integer-only, so bit-exact on the GPU.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double u01(uint64_t seed, uint64_t stream, uint64_t index) {
    const uint64_t z = mix64(mix64(mix64(seed) ^ (stream * 0xd1342543de82ef95ull)) ^
                             (index * 0xaf251af3b0f025b5ull));
    return static_cast<double>(z >> 11) * 0x1.0p-53;  // exact: 53-bit int * 2^-53
}
// rng.hpp:26-29.  Explicit round-to-nearest intrinsics: the draw is bit-exact
// in both arithmetic modes (no contraction into an FMA).
__device__ __forceinline__ double uniform_in(double lo, double hi, double u) {
    if (lo == hi) return lo;
    return __dadd_rn(lo, __dmul_rn(u, __dsub_rn(hi, lo)));
}

// rk4.cpp:99-100 and :38-39 evaluated on the device with explicit rounding, so
// a step loop running inside a kernel sees exactly the host's t, hk, h2, h6.
__device__ __forceinline__ StepConsts step_consts(double t0, double t1, double h,
                                                  unsigned long long k,
                                                  unsigned long long total) {
    StepConsts c;
    c.t = __dadd_rn(t0, __dmul_rn(static_cast<double>(k), h));
    c.hk = (k + 1 == total) ? __dsub_rn(t1, c.t) : h;
    c.h2 = __dmul_rn(0.5, c.hk);
    c.h6 = __ddiv_rn(c.hk, 6.0);
    return c;
}

}  // namespace pirk
