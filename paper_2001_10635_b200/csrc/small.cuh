// small.cuh -- K3/K4: small dense systems (n <= 64).
//
//  * monte_carlo_kernel: one sample per thread, state in registers, in-kernel
//    counter-based sampling (draw_sample, reach.cpp:202-212 + rng.hpp), RK4
//    (rk4_serial.cpp:33-50), hull fold at record slots (HullAccumulator,
//    reach.cpp:214-242) as warp-shuffle -> shared-memory -> one atomic min/max
//    per CTA on order-preserving integer keys (min/max is exact, so the
//    result does not depend on reduction order).
//  * small_integrate_kernel: one thread integrates one small system (the
//    embedding for mixed monotonicity, or f / growth for growth bound),
//    recording the states of the record schedule.
//
// Vector fields restate models.cpp with the reference's expression order;
// in exact TUs (-fmad=false) they round identically except for libm
// sin/cos (arch-quadrotor), which CUDA does not reproduce bit-for-bit.
#pragma once

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace pirk {

enum {
    kZero = 0, kScalarDecay = 1, kScalarLinear = 2, kTraffic = 3, kHeat3d = 4, kChain = 5,
    kLaubLoomis = 6, kArchQuad = 7, kVdp = 8
};
enum { kDecompNone = 0, kDecompNative = 1, kDecompJacobian = 2 };

// ---------------------------------------------------------------- vector fields

__device__ __forceinline__ double sm_traffic_flux(const SmallModel& m, double from, double into) {
    const double v = m.P[0], w = m.P[1], c = m.P[2], xbar = m.P[3], beta = m.P[5];
    return ref_min(c, ref_min(v * from, w * (xbar - into) / beta));  // models.cpp:59-61
}

// f_i(x, p) for the generic (runtime-n) path.
static __device__ double sm_f(const SmallModel& m, int i, const double* x, const double* p) {
    const int n = m.n;
    switch (m.kind) {
        case kZero: return 0.0;
        case kScalarDecay: return -x[0] + p[0];
        case kScalarLinear: return m.P[0] * x[0];
        case kTraffic: {  // models.cpp:64-75
            const double v = m.P[0], c = m.P[2], beta = m.P[5];
            const double inv_t = 1.0 / m.P[4];
            const double in = (i == 0) ? beta * p[0] : beta * sm_traffic_flux(m, x[i - 1], x[i]);
            const double out = (i + 1 == n) ? ref_min(c, v * x[i]) : sm_traffic_flux(m, x[i], x[i + 1]);
            return inv_t * (in - out);
        }
        case kHeat3d: {  // models.cpp:99-127
            const int g = static_cast<int>(m.grid), g2 = g * g;
            const double delta = 1.0 / static_cast<double>(g - 1);
            const double k = m.P[0] / (delta * delta);
            const double robin = 2.0 * delta * m.P[1];
            const int ix = i % g, iy = (i / g) % g, iz = i / g2;
            const double self = x[i];
            double acc = 0.0;
            if (ix > 0) acc += x[i - 1] - self;
            else acc += (x[i + 1] - self) - robin * self;
            if (ix + 1 < g) acc += x[i + 1] - self;
            if (iy > 0) acc += x[i - g] - self;
            if (iy + 1 < g) acc += x[i + g] - self;
            if (iz > 0) acc += x[i - g2] - self;
            if (iz + 1 < g) acc += x[i + g2] - self;
            return k * acc;
        }
        case kChain: {
            const double sl = (i == 0) ? 0.0 : x[i - 1] / (1.0 + fabs(x[i - 1]));
            const double sr = (i + 1 == n) ? 0.0 : x[i + 1] / (1.0 + fabs(x[i + 1]));
            return ((-m.P[0]) * x[i] + m.P[1] * sl - m.P[2] * sr) + p[0];
        }
        case kLaubLoomis:  // models.cpp:470-485
            switch (i) {
                case 0: return 1.4 * x[2] - 0.9 * x[0];
                case 1: return 2.5 * x[4] - 1.5 * x[1];
                case 2: return 0.6 * x[6] - 0.8 * x[1] * x[2];
                case 3: return 2.0 - 1.3 * x[2] * x[3];
                case 4: return 0.7 * x[0] - x[3] * x[4];
                case 5: return 0.3 * x[0] - 3.1 * x[5];
                default: return 1.8 * x[5] - 1.5 * x[1] * x[6];
            }
        case kVdp:  // models.cpp:452-456
            if (i == 0) return x[1];
            return m.P[0] * (1.0 - x[0] * x[0]) * x[1] - x[0];
        default: return __longlong_as_double(0x7ff8000000000000ll);
    }
}

// arch-quadrotor, all 12 components with the trig evaluated once (the
// reference recomputes identical values per component, models.cpp:522-524).
__device__ __forceinline__ void aq_f_all(const SmallModel& m, const double* x, double* f) {
    const double mass = m.P[0], gravity = m.P[1], jx = m.P[2], jy = m.P[3];
    const double kx = m.Q[0], ky = m.Q[1], kz = m.Q[2];  // (jy - jz) / jx, ... (host, same IEEE division)
    double s7, c7, s8, c8, s9, c9;
    sincos(x[6], &s7, &c7);
    sincos(x[7], &s8, &c8);
    sincos(x[8], &s9, &c9);
    f[0] = c8 * c9 * x[3] + (s7 * s8 * c9 - c7 * s9) * x[4] + (c7 * s8 * c9 + s7 * s9) * x[5];
    f[1] = c8 * s9 * x[3] + (s7 * s8 * s9 + c7 * c9) * x[4] + (c7 * s8 * s9 - s7 * c9) * x[5];
    f[2] = s8 * x[3] - s7 * c8 * x[4] - c7 * c8 * x[5];
    f[3] = x[11] * x[4] - x[10] * x[5] - gravity * s8;
    f[4] = x[9] * x[5] - x[11] * x[3] + gravity * c8 * s7;
    {
        const double thrust = mass * gravity - 10.0 * (x[2] - 1.0) + 3.0 * x[5];
        f[5] = x[10] * x[3] - x[9] * x[4] + gravity * c8 * c7 - thrust / mass;
    }
    f[6] = x[9] + s7 * (s8 / c8) * x[10] + c7 * (s8 / c8) * x[11];
    f[7] = c7 * x[10] - s7 * x[11];
    f[8] = s7 / c8 * x[10] + c7 / c8 * x[11];
    f[9] = kx * x[10] * x[11] - (x[6] + x[9]) / jx;
    f[10] = ky * x[9] * x[11] - (x[7] + x[10]) / jy;
    f[11] = kz * x[9] * x[10];
}

// Fast-mode sin and cos of a small angle (|x| <= 1e5; larger arguments take
// CUDA's sincos): Cody-Waite reduction by pi/2 in two parts, then the fdlibm /
// musl kernels __sin and __cos on [-pi/4, pi/4] (error < 1 ulp of the result
// there).  CUDA's sincos spends most of its instructions on the general
// Payne-Hanek path (integer ops and branches: profiles/r01_mc_archquad.txt).
// The coefficients live in constant memory so the DFMAs read them as
// constant-bank operands: as immediates every use was rebuilt with two UMOVs
// (20% of the MC kernel's instructions, profiles/r01_mc_archquad_fast_v3.txt).
static __constant__ double kSinCos[15] = {
    0.63661977236758134308,     // 2/pi
    1.57079632673412561417e+00,  // pio2_1 (33 bits: exact product)
    6.07710050650619224932e-11,  // pio2_1t
    8.33333333332248946124e-03, -1.98412698298579493134e-04, 2.75573137070700676789e-06,
    -2.50507602534068634195e-08, 1.58969099521155010221e-10, -1.66666666666666324348e-01,  // __sin
    4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
    -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11};  // __cos
__device__ __forceinline__ void small_sincos(double x, double* s, double* c) {
    if (!(fabs(x) <= 1e5)) {
        sincos(x, s, c);
        return;
    }
    const double* K = kSinCos;
    const double q = rint(x * K[0]);
    double r = fma(-q, K[1], x);
    r = fma(-q, K[2], r);
    const double z = r * r, w = z * z;
    const double ps = K[3] + z * (K[4] + z * K[5]) + z * w * (K[6] + z * K[7]);
    const double sr = r + (z * r) * (K[8] + z * ps);
    const double pc = z * (K[9] + z * (K[10] + z * K[11])) + w * w * (K[12] + z * (K[13] + z * K[14]));
    const double hz = 0.5 * z, v = 1.0 - hz;
    const double cr = v + (((1.0 - v) - hz) + z * pc);
    switch (static_cast<int>(q) & 3) {
        case 0: *s = sr; *c = cr; break;
        case 1: *s = cr; *c = -sr; break;
        case 2: *s = -sr; *c = -cr; break;
        default: *s = -cr; *c = sr; break;
    }
}

// arch-quadrotor in fast mode: the same field with small_sincos, one 1/cos
// and the constant quotients folded (tolerance-only in both modes: glibc and
// CUDA trig differ in the last ulp, DESIGN.md (c))
__device__ __forceinline__ void aq_f_all_fast(const SmallModel& m, const double* x, double* f) {
    const double mass = m.P[0], gravity = m.P[1];
    const double kx = m.Q[0], ky = m.Q[1], kz = m.Q[2];  // uniform divisions, computed on the host
    const double ijx = m.Q[3], ijy = m.Q[4], imass = m.Q[5];
    double s7, c7, s8, c8, s9, c9;
    small_sincos(x[6], &s7, &c7);
    small_sincos(x[7], &s8, &c8);
    small_sincos(x[8], &s9, &c9);
    // 1/c8: hardware reciprocal estimate + two Newton steps (~1 ulp; fast mode),
    // without the division's special-case branch (c8 = cos(theta) is nonzero on
    // the model's operating box)
    double ic8;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(ic8) : "d"(c8));
    {
        double e = fma(-c8, ic8, 1.0);
        ic8 = fma(ic8, e, ic8);
        e = fma(-c8, ic8, 1.0);
        ic8 = fma(ic8, e, ic8);
    }
    const double t8 = s8 * ic8;
    f[0] = c8 * c9 * x[3] + (s7 * s8 * c9 - c7 * s9) * x[4] + (c7 * s8 * c9 + s7 * s9) * x[5];
    f[1] = c8 * s9 * x[3] + (s7 * s8 * s9 + c7 * c9) * x[4] + (c7 * s8 * s9 - s7 * c9) * x[5];
    f[2] = s8 * x[3] - s7 * c8 * x[4] - c7 * c8 * x[5];
    f[3] = x[11] * x[4] - x[10] * x[5] - gravity * s8;
    f[4] = x[9] * x[5] - x[11] * x[3] + gravity * c8 * s7;
    {
        const double thrust = mass * gravity - 10.0 * (x[2] - 1.0) + 3.0 * x[5];
        f[5] = x[10] * x[3] - x[9] * x[4] + gravity * c8 * c7 - thrust * imass;
    }
    f[6] = x[9] + s7 * t8 * x[10] + c7 * t8 * x[11];
    f[7] = c7 * x[10] - s7 * x[11];
    f[8] = s7 * ic8 * x[10] + c7 * ic8 * x[11];
    f[9] = kx * x[10] * x[11] - (x[6] + x[9]) * ijx;
    f[10] = ky * x[9] * x[11] - (x[7] + x[10]) * ijy;
    f[11] = kz * x[9] * x[10];
}

__device__ __forceinline__ void ll_f_all(const double* x, double* f) {
    f[0] = 1.4 * x[2] - 0.9 * x[0];
    f[1] = 2.5 * x[4] - 1.5 * x[1];
    f[2] = 0.6 * x[6] - 0.8 * x[1] * x[2];
    f[3] = 2.0 - 1.3 * x[2] * x[3];
    f[4] = 0.7 * x[0] - x[3] * x[4];
    f[5] = 0.3 * x[0] - 3.1 * x[5];
    f[6] = 1.8 * x[5] - 1.5 * x[1] * x[6];
}

static __device__ void sm_f_all(const SmallModel& m, const double* x, const double* p, double* f) {
    if (m.kind == kArchQuad) { aq_f_all(m, x, f); return; }
    if (m.kind == kLaubLoomis) { ll_f_all(x, f); return; }
    for (int i = 0; i < m.n; ++i) f[i] = sm_f(m, i, x, p);
}

// growth_rhs g_i(r, w): models.cpp:78-87 (traffic), :130 (heat), :624/:637/:651
// (trivial models), growth_from_matrix (system_model.cpp:107-121) otherwise.
static __device__ double sm_g(const SmallModel& m, int i, const double* r, const double* w) {
    const int n = m.n;
    switch (m.kind) {
        case kZero: return 0.0;
        case kScalarDecay: return -r[0] + w[0];
        case kScalarLinear: return m.P[0] * r[0];
        case kTraffic: {
            const double v = m.P[0], wc = m.P[1], beta = m.P[5];
            const double inv_t = 1.0 / m.P[4];
            const double a_prev = beta * v * inv_t;
            const double a_next = (wc / beta) * inv_t;
            const double a_in = beta * inv_t;
            double gv = (i == 0) ? a_in * w[0] : a_prev * r[i - 1];
            if (i + 1 < n) gv += a_next * r[i + 1];
            return gv;
        }
        case kHeat3d: return sm_f(m, i, r, w);
        default: {
            double acc = 0.0;
            for (int j = 0; j < n; ++j) acc += m.C[i * n + j] * r[j];
            return acc;
        }
    }
}

// Embedding derivative of dimension 2n (system_model.cpp:67-75) for the
// native (cooperative / chain) and Jacobian-bound decompositions.
static __device__ void sm_embed_all(const SmallModel& m, const double* y, const double* p, double* k) {
    const int n = m.n, ni = m.ni;
    const double* xl = y;
    const double* xu = y + n;
    const double* pl = p;
    const double* pu = p + ni;
    if (m.kind == kChain) {
        for (int i = 0; i < n; ++i) {
            const double sl = (i == 0) ? 0.0 : xl[i - 1] / (1.0 + fabs(xl[i - 1]));
            const double sr = (i + 1 == n) ? 0.0 : xu[i + 1] / (1.0 + fabs(xu[i + 1]));
            k[i] = ((-m.P[0]) * xl[i] + m.P[1] * sl - m.P[2] * sr) + pl[0];
        }
        for (int i = 0; i < n; ++i) {
            const double sl = (i == 0) ? 0.0 : xu[i - 1] / (1.0 + fabs(xu[i - 1]));
            const double sr = (i + 1 == n) ? 0.0 : xl[i + 1] / (1.0 + fabs(xl[i + 1]));
            k[n + i] = ((-m.P[0]) * xu[i] + m.P[1] * sl - m.P[2] * sr) + pu[0];
        }
        return;
    }
    sm_f_all(m, xl, pl, k);
    sm_f_all(m, xu, pu, k + n);
    if (m.decomp == kDecompJacobian) {
        for (int i = 0; i < n; ++i) {
            double al = k[i], au = k[n + i];
            for (int j = 0; j < n; ++j) {
                const double cij = m.C[i * n + j];
                if (j == i || cij == 0.0) continue;
                al = al + cij * (xl[j] - xu[j]);
                au = au + cij * (xu[j] - xl[j]);
            }
            k[i] = al;
            k[n + i] = au;
        }
    }
}

static __device__ void sm_eval(const SmallModel& m, int which, const double* y, const double* p,
                        double* k) {
    if (which == 0) sm_f_all(m, y, p, k);
    else if (which == 1) { for (int i = 0; i < m.n; ++i) k[i] = sm_g(m, i, y, p); }
    else sm_embed_all(m, y, p, k);
}

// --------------------------------------------------- single-trajectory integrator

template <bool Exact>
__global__ void small_integrate_kernel(const SmallModel m, const int which, const double* x0,
                                       const double* p, const double t0, const double t1,
                                       const double h, const unsigned long long total,
                                       const unsigned long long stride, double* rec,
                                       unsigned long long* fail) {
    (void)sizeof(ModeCheck<Exact>);
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int D = (which == 2) ? 2 * m.n : m.n;
    double x[2 * kSmallMax], u[2 * kSmallMax], k[2 * kSmallMax], acc[2 * kSmallMax];
    for (int i = 0; i < D; ++i) x[i] = x0[i];
    unsigned long long slot = 0;
    if (stride > 0) {
        for (int i = 0; i < D; ++i) rec[i] = x[i];
        slot = 1;
    }
    for (unsigned long long s = 0; s < total; ++s) {
        const StepConsts c = step_consts(t0, t1, h, s, total);
        sm_eval(m, which, x, p, k);
        for (int i = 0; i < D; ++i) { acc[i] = k[i]; u[i] = x[i] + c.h2 * k[i]; }
        sm_eval(m, which, u, p, k);
        for (int i = 0; i < D; ++i) { acc[i] = acc[i] + 2.0 * k[i]; u[i] = x[i] + c.h2 * k[i]; }
        sm_eval(m, which, u, p, k);
        for (int i = 0; i < D; ++i) { acc[i] = acc[i] + 2.0 * k[i]; u[i] = x[i] + c.hk * k[i]; }
        sm_eval(m, which, u, p, k);
        for (int i = 0; i < D; ++i) x[i] = x[i] + c.h6 * (acc[i] + k[i]);
        for (int i = 0; i < D; ++i) {
            if (!finite_d(x[i])) {
                record_fail(fail, s, static_cast<unsigned long long>(i));
                return;  // the reference throws at the first failing step
            }
        }
        if (s + 1 == total || (stride > 0 && (s + 1) % stride == 0)) {
            for (int i = 0; i < D; ++i) rec[slot * D + i] = x[i];
            ++slot;
        }
    }
}

// ------------------------------------------- warp-parallel single-trajectory integrator
//
// The same integration as small_integrate_kernel with the components of each
// stage spread over the 32 lanes of one warp (the reference parallelises
// integrate_step over components the same way, rk4.cpp:47-76): lane l owns
// components l, l+32, ...; the stage inputs live in shared memory (ping-pong,
// so a stage reads one buffer while it writes the other), one __syncwarp per
// stage.  Every component is evaluated with exactly the serial kernel's
// expression, so results are bit-identical to it; the latency of a step drops
// from D component evaluations in sequence to about one.

// f_i alone (arch-quadrotor / Laub-Loomis evaluate all components together;
// fast mode: the small-angle arch-quadrotor field of the MC kernel)
template <bool Exact>
static __device__ double sm_f_comp(const SmallModel& m, int i, const double* x, const double* p) {
    if (m.kind == kArchQuad) {
        double f[12];
        if constexpr (Exact) aq_f_all(m, x, f);
        else aq_f_all_fast(m, x, f);
        return f[i];
    }
    if (m.kind == kLaubLoomis) {
        double f[7];
        ll_f_all(x, f);
        return f[i];
    }
    return sm_f(m, i, x, p);
}

// embedding component c of [x | xh] (sm_embed_all, one component)
template <bool Exact>
static __device__ double sm_embed_comp(const SmallModel& m, int c, const double* y, const double* p) {
    const int n = m.n, ni = m.ni;
    const bool up = c >= n;
    const int i = up ? c - n : c;
    const double* xa = up ? y + n : y;
    const double* xb = up ? y : y + n;
    const double* pa = up ? p + ni : p;
    if (m.kind == kChain) {
        const double sl = (i == 0) ? 0.0 : xa[i - 1] / (1.0 + fabs(xa[i - 1]));
        const double sr = (i + 1 == n) ? 0.0 : xb[i + 1] / (1.0 + fabs(xb[i + 1]));
        return ((-m.P[0]) * xa[i] + m.P[1] * sl - m.P[2] * sr) + pa[0];
    }
    double a = sm_f_comp<Exact>(m, i, xa, pa);
    if (m.decomp == kDecompJacobian) {
        for (int j = 0; j < n; ++j) {
            const double cij = m.C[i * n + j];
            if (j == i || cij == 0.0) continue;
            a = a + cij * (xa[j] - xb[j]);
        }
    }
    return a;
}

template <bool Exact>
static __device__ double sm_comp(const SmallModel& m, int which, int c, const double* y, const double* p) {
    if (which == 0) return sm_f_comp<Exact>(m, c, y, p);
    if (which == 1) return sm_g(m, c, y, p);
    return sm_embed_comp<Exact>(m, c, y, p);
}

template <bool Exact>
__global__ void __launch_bounds__(32) small_warp_kernel(const SmallModel m, const int which, const double* x0,
                                                         const double* p, const double t0, const double t1,
                                                         const double h, const unsigned long long total,
                                                         const unsigned long long stride, double* rec,
                                                         unsigned long long* fail) {
    (void)sizeof(ModeCheck<Exact>);
    constexpr int kMax = 2 * kSmallMax;
    constexpr int kPer = kMax / 32;
    __shared__ double X[kMax], UA[kMax], UB[kMax];
    const int lane = threadIdx.x;
    const int D = (which == 2) ? 2 * m.n : m.n;
    double acc[kPer];
    for (int q = 0; q < kPer; ++q) {
        const int c = lane + 32 * q;
        if (c < D) X[c] = x0[c];
    }
    __syncwarp();
    unsigned long long slot = 0;
    if (stride > 0) {
        for (int q = 0; q < kPer; ++q) {
            const int c = lane + 32 * q;
            if (c < D) rec[c] = X[c];
        }
        slot = 1;
    }
    for (unsigned long long s = 0; s < total; ++s) {
        const StepConsts sc = step_consts(t0, t1, h, s, total);
        // stage 1: k0 = F(x); acc = k0; u1 = x + h2 k0
        for (int q = 0; q < kPer; ++q) {
            const int c = lane + 32 * q;
            if (c >= D) continue;
            const double k = sm_comp<Exact>(m, which, c, X, p);
            acc[q] = k;
            UA[c] = X[c] + sc.h2 * k;
        }
        __syncwarp();
        // stage 2: k1 = F(u1); acc += 2 k1; u2 = x + h2 k1
        for (int q = 0; q < kPer; ++q) {
            const int c = lane + 32 * q;
            if (c >= D) continue;
            const double k = sm_comp<Exact>(m, which, c, UA, p);
            acc[q] = acc[q] + 2.0 * k;
            UB[c] = X[c] + sc.h2 * k;
        }
        __syncwarp();
        // stage 3: k2 = F(u2); acc += 2 k2; u3 = x + hk k2
        for (int q = 0; q < kPer; ++q) {
            const int c = lane + 32 * q;
            if (c >= D) continue;
            const double k = sm_comp<Exact>(m, which, c, UB, p);
            acc[q] = acc[q] + 2.0 * k;
            UA[c] = X[c] + sc.hk * k;
        }
        __syncwarp();
        // stage 4: k3 = F(u3); x = x + h6 (acc + k3) (no lane reads X in this stage)
        unsigned bad = 0xffffffffu;
        for (int q = 0; q < kPer; ++q) {
            const int c = lane + 32 * q;
            if (c >= D) continue;
            const double k = sm_comp<Exact>(m, which, c, UA, p);
            const double xn = X[c] + sc.h6 * (acc[q] + k);
            X[c] = xn;
            if (!finite_d(xn) && static_cast<unsigned>(c) < bad) bad = static_cast<unsigned>(c);
        }
        __syncwarp();
        bad = __reduce_min_sync(0xffffffffu, bad);
        if (bad != 0xffffffffu) {  // the reference throws at the first failing step, lowest component
            if (lane == 0) record_fail(fail, s, static_cast<unsigned long long>(bad));
            return;
        }
        if (s + 1 == total || (stride > 0 && (s + 1) % stride == 0)) {
            for (int q = 0; q < kPer; ++q) {
                const int c = lane + 32 * q;
                if (c < D) rec[slot * D + c] = X[c];
            }
            ++slot;
        }
    }
}

template <bool Exact>
cudaError_t launch_small_integrate(const SmallModel& m, int which, const double* x0,
                                   const double* p, double t0, double t1, double h,
                                   unsigned long long total, unsigned long long stride,
                                   double* rec, unsigned long long* fail, cudaStream_t stream) {
    // PIRK_SMALL_SERIAL=1: the one-thread kernel (A/B; both are bit-identical)
    static const bool serial = [] {
        const char* v = std::getenv("PIRK_SMALL_SERIAL");
        return v && v[0] == '1';
    }();
    if (serial)
        small_integrate_kernel<Exact><<<1, 32, 0, stream>>>(m, which, x0, p, t0, t1, h, total, stride, rec, fail);
    else
        small_warp_kernel<Exact><<<1, 32, 0, stream>>>(m, which, x0, p, t0, t1, h, total, stride, rec, fail);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ Monte Carlo

constexpr int kMcThreads = 128;

// Functors giving f for a compile-time dimension (N > 0) or the generic path.
template <int N, bool Exact>
struct McField {
    __device__ static void eval(const SmallModel& m, const double* x, const double* p, double* f) {
        if constexpr (N == 12 && !Exact) aq_f_all_fast(m, x, f);
        else if constexpr (N == 12) aq_f_all(m, x, f);
        else if constexpr (N == 7) ll_f_all(x, f);
        else sm_f_all(m, x, p, f);
    }
};

__device__ __forceinline__ double shfl_xor_d(double v, int lane_mask) {
    return __shfl_xor_sync(0xffffffffu, v, lane_mask);
}

// Fold the CTA's current states into hull[slot]: warp shuffle, then shared
// memory across warps, then one atomic per (component, bound) per CTA.
template <int NA>
__device__ void hull_fold(const double* x, bool active, int n, unsigned long long* hull_slot,
                          double* red /* [warps][NA][2] */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int W = kMcThreads / 32;
    for (int i = 0; i < n; ++i) {
        double lo = active ? x[i] : __longlong_as_double(0x7ff0000000000000ll);
        double hi = active ? x[i] : __longlong_as_double(0xfff0000000000000ll);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = ref_min(lo, shfl_xor_d(lo, o));
            const double oh = shfl_xor_d(hi, o);
            hi = (oh > hi) ? oh : hi;
        }
        if (lane == 0) {
            red[(warp * NA + i) * 2 + 0] = lo;
            red[(warp * NA + i) * 2 + 1] = hi;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * n; t += blockDim.x) {
        const int i = t >> 1, b = t & 1;
        double v = red[(0 * NA + i) * 2 + b];
        for (int wi = 1; wi < W; ++wi) {
            const double o = red[(wi * NA + i) * 2 + b];
            v = b ? ((o > v) ? o : v) : ref_min(v, o);
        }
        if (b == 0) atomicMin(hull_slot + i, ord_key(v));
        else atomicMax(hull_slot + n + i, ord_key(v));
    }
    __syncthreads();
}

#ifndef PIRK_MC_MINB
#define PIRK_MC_MINB 4  // 16 warps/SM: arch-quad fast m=1e6 5.62 vs 5.91 ms at 1 (5: 5.60)
#endif
template <bool Exact, int N>
__global__ void __launch_bounds__(kMcThreads, PIRK_MC_MINB)
monte_carlo_kernel(const SmallModel m, const McArgs a) {
    (void)sizeof(ModeCheck<Exact>);
    constexpr int NA = (N > 0) ? N : kSmallMax;
    __shared__ double red[(kMcThreads / 32) * NA * 2];
    const int n = (N > 0) ? N : m.n;
    const int ni = m.ni;
    const unsigned long long s =
        a.s_begin + static_cast<unsigned long long>(blockIdx.x) * kMcThreads + threadIdx.x;
    bool active = s < a.s_end;
    const bool coverage = a.outside != nullptr;

    double x[NA], u[NA], k[NA], acc[NA], p[8];
    // draw_sample (reach.cpp:202-212): x0[i] = uniform_in(lo_i, hi_i, u01(seed, s, i)),
    // p[j] = uniform_in(plo_j, phi_j, u01(seed, s, n + j))
#pragma unroll
    for (int i = 0; i < NA; ++i)
        if (i < n) x[i] = uniform_in(a.lo[i], a.hi[i], u01(a.seed, s, static_cast<uint64_t>(i)));
    for (int j = 0; j < ni && j < 8; ++j)
        p[j] = uniform_in(a.plo[j], a.phi[j], u01(a.seed, s, static_cast<uint64_t>(n + j)));

    unsigned long long slot = 0;
    if (a.stride > 0 && !coverage) {
        hull_fold<NA>(x, active, n, a.hull, red);
        slot = 1;
    }
    bool dead = false;
    for (unsigned long long st = 0; st < a.total; ++st) {
        const StepConsts c = step_consts(a.t0, a.t1, a.h, st, a.total);
        if (active && !dead) {
            McField<N, Exact>::eval(m, x, p, k);
#pragma unroll
            for (int i = 0; i < NA; ++i)
                if (i < n) { acc[i] = k[i]; u[i] = x[i] + c.h2 * k[i]; }
            McField<N, Exact>::eval(m, u, p, k);
#pragma unroll
            for (int i = 0; i < NA; ++i)
                if (i < n) { acc[i] = acc[i] + 2.0 * k[i]; u[i] = x[i] + c.h2 * k[i]; }
            McField<N, Exact>::eval(m, u, p, k);
#pragma unroll
            for (int i = 0; i < NA; ++i)
                if (i < n) { acc[i] = acc[i] + 2.0 * k[i]; u[i] = x[i] + c.hk * k[i]; }
            McField<N, Exact>::eval(m, u, p, k);
#pragma unroll
            for (int i = 0; i < NA; ++i)
                if (i < n) x[i] = x[i] + c.h6 * (acc[i] + k[i]);
            int bad = -1;
#pragma unroll
            for (int i = NA - 1; i >= 0; --i)
                if (i < n && !finite_d(x[i])) bad = i;
            if (bad >= 0) {
                // lowest failing sample wins; its step and component ride along
                // (host validates s < 2^34, steps < 2^20, n <= 64 for this packing)
                if (a.fail)
                    atomicMin(a.fail, ((s - a.s_begin) << 30) | (st << 10) |
                                          static_cast<unsigned long long>(bad));
                dead = true;
            }
        }
        if (!coverage && (st + 1 == a.total || (a.stride > 0 && (st + 1) % a.stride == 0))) {
            hull_fold<NA>(x, active && !dead, n, a.hull + slot * 2 * n, red);
            ++slot;
        }
    }
    if (coverage && active && !dead) {
        bool out = false;
        for (int i = 0; i < n; ++i)
            if (x[i] < a.box_lo[i] || x[i] > a.box_hi[i]) out = true;  // interval.cpp:55-62
        if (out) atomicAdd(a.outside, 1ull);
    }
}

template <bool Exact>
cudaError_t launch_monte_carlo(const SmallModel& m, const McArgs& a, cudaStream_t stream) {
    if (a.s_end <= a.s_begin) return cudaSuccess;
    const unsigned long long count = a.s_end - a.s_begin;
    const unsigned int blocks = static_cast<unsigned int>((count + kMcThreads - 1) / kMcThreads);
    if (m.kind == kArchQuad)
        monte_carlo_kernel<Exact, 12><<<blocks, kMcThreads, 0, stream>>>(m, a);
    else if (m.kind == kLaubLoomis)
        monte_carlo_kernel<Exact, 7><<<blocks, kMcThreads, 0, stream>>>(m, a);
    else
        monte_carlo_kernel<Exact, 0><<<blocks, kMcThreads, 0, stream>>>(m, a);
    return cudaGetLastError();
}

}  // namespace pirk
