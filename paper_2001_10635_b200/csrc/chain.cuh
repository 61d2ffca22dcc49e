// chain.cuh -- K1: fused 4-stage RK4 step for 1-D radius-1 models on two fields.
//
// Replaces one call of integrate_step (rk4.cpp:30-76) on the embedding
// (system_model.cpp:56-77) of traffic (models.cpp:47-90) or the coupled chain
// (SURVEY.md 8d C4), or on the growth-bound pair [center | radius]
// (reach.cpp:103-114).  One CTA owns a tile of T components of BOTH fields
// (so coupled decompositions read the other field in shared memory), loads it
// with a halo of 4 (one per RK stage), runs the four stages in shared memory
// and writes the tile once: 16 B of HBM traffic per state-update instead of
// the reference's 144 B.
//
// Per-component arithmetic is exactly integrate_step's in exact mode:
//   k0 = f(x); u1 = x + h2*k0; k1 = f(u1); u2 = x + h2*k1; k2 = f(u2);
//   u3 = x + hk*k2; k3 = f(u3); x' = x + h6*(((k0 + 2k1) + 2k2) + k3).
#pragma once

#ifndef PIRK_DEV_VARIANTS
#define PIRK_DEV_VARIANTS 0  // 1: also build the rejected smem-tile chain kernel
#endif

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace pirk {

constexpr int kChainThreads = 256;
constexpr int kChainPerThread = 4;
constexpr int kChainSpan = kChainThreads * kChainPerThread;  // loaded elements per tile
constexpr int kChainHalo = 4;
constexpr int kChainTile = kChainSpan - 2 * kChainHalo;      // outputs per tile

enum { kKindTraffic = 3, kKindChain = 5 };
enum { kMethodMM = 0, kMethodGB = 1 };

// traffic flux (models.cpp:59-61): min(c, min(v*from, w*(xbar-into)/beta)).
template <bool Exact>
__device__ __forceinline__ double traffic_flux(const ChainModel& m, double from, double into) {
    const double v = m.P[0], w = m.P[1], c = m.P[2], xbar = m.P[3], beta = m.P[5];
    if constexpr (Exact) {
        return ref_min(c, ref_min(v * from, w * (xbar - into) / beta));
    } else {
        return ref_min(c, ref_min(v * from, m.wb * (xbar - into)));
    }
}

// s(z) = z / (1 + |z|) for the coupled chain.  Exact mode: IEEE division.
// Fast mode: the denominator lies in [1, inf), so a hardware reciprocal
// estimate refined by two Newton steps (~1 ulp) replaces the full division
// and its special-case branches.
template <bool Exact>
__device__ __forceinline__ double chain_sat(double z) {
    const double d = 1.0 + fabs(z);
    if constexpr (Exact) {
        return z / d;
    } else {
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
        double e = fma(-d, r, 1.0);
        r = fma(r, e, r);
        e = fma(-d, r, 1.0);
        r = fma(r, e, r);
        return z * r;
    }
}

#if PIRK_DEV_VARIANTS  // the rejected shared-memory tile kernel (A/B and reference only)
template <bool Exact, int Kind, int Method>
__global__ void __launch_bounds__(kChainThreads)
chain_step_kernel(const ChainModel m, const WindowArgs w, const StepConsts sc,
                  const unsigned long long step, unsigned long long* __restrict__ fail) {
    (void)sizeof(ModeCheck<Exact>);
    __shared__ double sU[2][2][kChainSpan];   // [buffer][field][j] stage input ping-pong
    __shared__ double sA[2][kChainSpan];      // [field][j] per-stage auxiliary (edge flux / s(u))

    const int tid = threadIdx.x;
    const uint64_t n = m.n;
    const long long o0 = static_cast<long long>(w.out_begin) +
                         static_cast<long long>(blockIdx.x) * kChainTile;
    const long long base = o0 - kChainHalo;  // global index of local j = 0

    double x0[kChainPerThread], x1[kChainPerThread];
    double acc0[kChainPerThread], acc1[kChainPerThread];

    // ---- load the tile (+halo) of both fields; positions outside the window are NaN
#pragma unroll
    for (int r = 0; r < kChainPerThread; ++r) {
        const int j = tid + r * kChainThreads;
        const long long g = base + j;
        double a = __longlong_as_double(0x7ff8000000000000ll), b = a;
        if (g >= static_cast<long long>(w.win_begin) && g < static_cast<long long>(w.win_end)) {
            a = w.in0[g - static_cast<long long>(w.win_begin)];
            b = w.in1[g - static_cast<long long>(w.win_begin)];
        }
        x0[r] = a;
        x1[r] = b;
        sU[0][0][j] = a;
        sU[0][1][j] = b;
        acc0[r] = 0.0;
        acc1[r] = 0.0;
    }
    __syncthreads();

    int cur = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const double* u0 = sU[cur][0];
        const double* u1 = sU[cur][1];

        // ---- phase A: per-element / per-edge precompute over [s, span - s)
        if constexpr (Kind == kKindTraffic) {
#pragma unroll
            for (int r = 0; r < kChainPerThread; ++r) {
                const int j = tid + r * kChainThreads;
                if (j >= s && j < kChainSpan - 1 - s) {
                    sA[0][j] = traffic_flux<Exact>(m, u0[j], u0[j + 1]);  // edge j -> j+1
                    if constexpr (Method == kMethodMM)
                        sA[1][j] = traffic_flux<Exact>(m, u1[j], u1[j + 1]);
                }
            }
            __syncthreads();
        } else if constexpr (Kind == kKindChain) {
#pragma unroll
            for (int r = 0; r < kChainPerThread; ++r) {
                const int j = tid + r * kChainThreads;
                if (j >= s && j < kChainSpan - s) {
                    sA[0][j] = chain_sat<Exact>(u0[j]);
                    sA[1][j] = chain_sat<Exact>(u1[j]);
                }
            }
            __syncthreads();
        }

        // ---- phase B: stage derivative and update over [s+1, span-1-s)
        double* n0 = sU[cur ^ 1][0];
        double* n1 = sU[cur ^ 1][1];
#pragma unroll
        for (int r = 0; r < kChainPerThread; ++r) {
            const int j = tid + r * kChainThreads;
            const long long g = base + j;
            if (j < s + 1 || j >= kChainSpan - 1 - s) continue;
            if (g < 0 || g >= static_cast<long long>(n)) continue;
            const bool first = (g == 0);
            const bool last = (g + 1 == static_cast<long long>(n));
            double k0v, k1v;
            if constexpr (Kind == kKindTraffic) {
                const double v = m.P[0], c = m.P[2], beta = m.P[5];
                // models.cpp:68-74 with the flux of each edge shared by its two
                // end components (same inputs, hence bit-identical).
                {
                    const double in = first ? beta * m.p0 : beta * sA[0][j - 1];
                    const double out = last ? ref_min(c, v * u0[j]) : sA[0][j];
                    k0v = m.inv_t * (in - out);
                }
                if constexpr (Method == kMethodMM) {
                    const double in = first ? beta * m.p1 : beta * sA[1][j - 1];
                    const double out = last ? ref_min(c, v * u1[j]) : sA[1][j];
                    k1v = m.inv_t * (in - out);
                } else {
                    // growth_rhs, models.cpp:78-87
                    double gv = first ? m.a_in * m.p1 : m.a_prev * u1[j - 1];
                    if (!last) gv += m.a_next * u1[j + 1];
                    k1v = gv;
                }
            } else {  // coupled chain: d_i(x,p,xh,ph) = ((-a) x_i + b s(x_{i-1}) - c s(xh_{i+1})) + p
                const double na = -m.P[0], b = m.P[1], c = m.P[2];
                {
                    const double sl = first ? 0.0 : sA[0][j - 1];
                    const double sr = last ? 0.0 : sA[1][j + 1];
                    k0v = (na * u0[j] + b * sl - c * sr) + m.p0;
                }
                {
                    const double sl = first ? 0.0 : sA[1][j - 1];
                    const double sr = last ? 0.0 : sA[0][j + 1];
                    k1v = (na * u1[j] + b * sl - c * sr) + m.p1;
                }
            }
            if (s == 0) {
                acc0[r] = k0v;
                acc1[r] = k1v;
                n0[j] = x0[r] + sc.h2 * k0v;
                n1[j] = x1[r] + sc.h2 * k1v;
            } else if (s == 1) {
                acc0[r] = acc0[r] + 2.0 * k0v;
                acc1[r] = acc1[r] + 2.0 * k1v;
                n0[j] = x0[r] + sc.h2 * k0v;
                n1[j] = x1[r] + sc.h2 * k1v;
            } else if (s == 2) {
                acc0[r] = acc0[r] + 2.0 * k0v;
                acc1[r] = acc1[r] + 2.0 * k1v;
                n0[j] = x0[r] + sc.hk * k0v;
                n1[j] = x1[r] + sc.hk * k1v;
            } else {
                // final update; j in [4, span-4) here, i.e. the tile's own outputs
                x0[r] = x0[r] + sc.h6 * (acc0[r] + k0v);
                x1[r] = x1[r] + sc.h6 * (acc1[r] + k1v);
            }
        }
        if (s < 3) __syncthreads();
        cur ^= 1;
    }

    // ---- store the tile's outputs and flag non-finite values
#pragma unroll
    for (int r = 0; r < kChainPerThread; ++r) {
        const int j = tid + r * kChainThreads;
        const long long g = base + j;
        if (j < kChainHalo || j >= kChainSpan - kChainHalo) continue;
        if (g < static_cast<long long>(w.out_begin) || g >= static_cast<long long>(w.out_end))
            continue;
        const long long o = g - static_cast<long long>(w.out_begin);
        w.out0[o] = x0[r];
        w.out1[o] = x1[r];
        if (!finite_d(x0[r]) || !finite_d(x1[r])) {
            if constexpr (Method == kMethodMM) {
                // embedding components are numbered [x | xh] (system_model.cpp:67-75)
                const unsigned long long comp =
                    finite_d(x0[r]) ? static_cast<unsigned long long>(g) + n
                                    : static_cast<unsigned long long>(g);
                record_fail(fail, step, comp);
            } else {
                if (!finite_d(x0[r])) record_fail(fail, step, static_cast<unsigned long long>(g));
                if (!finite_d(x1[r]) && fail)
                    record_fail(fail + 1, step, static_cast<unsigned long long>(g));
            }
        }
    }
}
#endif  // PIRK_DEV_VARIANTS

// ---------------------------------------------------------------------------
// Warp-tiled variant (the default): each warp owns a segment of 32 * kCwP
// consecutive components of both fields, kCwP per lane, and runs the four
// stages in registers.  Neighbours across lanes come by shuffle; the segment's
// 4 outermost components per side are the halo (recomputed by the neighbouring
// warps, whose shuffles at lanes 0 / 31 produce garbage that never reaches
// the outputs).  No shared memory and no barriers: 16 B of HBM traffic per
// state-update plus 8 halo loads per 120 outputs.  Per-component arithmetic
// is the expression-for-expression restatement of chain_step_kernel above.
#ifndef PIRK_CW_P
#define PIRK_CW_P 4  // 8 per lane measured slower (n=1e7 chain 0.092 ms at 2 CTAs/SM vs 0.087)
#endif
constexpr int kCwP = PIRK_CW_P;              // components per lane
constexpr int kCwSeg = 32 * kCwP;            // loaded per warp
constexpr int kCwOut = kCwSeg - 2 * kChainHalo;  // 120 outputs per warp
constexpr int kCwWarps = 8;
#ifndef PIRK_CW_MINB
#define PIRK_CW_MINB 3  // CTAs per SM: 3 for the chain (4 spills), 4 for traffic (n=1e7: 0.0914 vs 0.0968 ms)
#endif
#ifndef PIRK_CW_VEC
#define PIRK_CW_VEC 1
#endif

// S RK4 steps per launch (S = 2: temporal blocking for full-domain runs; the
// segment keeps 128 - 8S outputs, the halo grows to 4S per side, each step's
// non-finite values are recorded under their own step index).
template <int S>
constexpr int cw_out() { return kCwSeg - 2 * kChainHalo * S; }

template <bool Exact, int Kind, int Method, int S = 1>
__global__ void __launch_bounds__(32 * kCwWarps, (Kind == kKindTraffic && PIRK_CW_MINB == 3) ? 4 : PIRK_CW_MINB)
chain_warp_kernel(const ChainModel m, const WindowArgs w, const StepConstsN scs,
                  const unsigned long long step, unsigned long long* __restrict__ fail) {
    (void)sizeof(ModeCheck<Exact>);
    const int lane = threadIdx.x & 31;
    const long long n = static_cast<long long>(m.n);
    const long long seg = static_cast<long long>(w.out_begin) +
                          (static_cast<long long>(blockIdx.x) * kCwWarps + (threadIdx.x >> 5)) * cw_out<S>() -
                          kChainHalo * S;
    if (seg + kChainHalo * S >= static_cast<long long>(w.out_end)) return;  // whole warp: uniform
    const long long g0 = seg + kCwP * lane;  // global index of this lane's first component
    const long long wb = static_cast<long long>(w.win_begin), we = static_cast<long long>(w.win_end);

    double x0[kCwP], x1[kCwP], u0[kCwP], u1[kCwP], acc0[kCwP], acc1[kCwP];
    const long long off = g0 - wb;
    if (PIRK_CW_VEC && g0 >= wb && g0 + kCwP <= we && ((reinterpret_cast<uintptr_t>(w.in0 + off) |
                                                          reinterpret_cast<uintptr_t>(w.in1 + off)) & 15) == 0) {
#pragma unroll
        for (int k = 0; k < kCwP; k += 2) {  // 16-byte loads: a lane's components are contiguous
            const double2 a = *reinterpret_cast<const double2*>(w.in0 + off + k);
            const double2 b = *reinterpret_cast<const double2*>(w.in1 + off + k);
            x0[k] = a.x, x0[k + 1] = a.y, x1[k] = b.x, x1[k + 1] = b.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kCwP; ++k) {
            const long long g = g0 + k;
            double a = __longlong_as_double(0x7ff8000000000000ll), b = a;  // NaN outside the window
            if (g >= wb && g < we) {
                a = w.in0[g - wb];
                b = w.in1[g - wb];
            }
            x0[k] = a;
            x1[k] = b;
        }
    }
#pragma unroll
    for (int k = 0; k < kCwP; ++k) {
        u0[k] = x0[k];
        u1[k] = x1[k];
        acc0[k] = acc1[k] = 0.0;
    }
    unsigned first = 0, last = 0;  // bit k: component g0 + k is 0 / n-1
#pragma unroll
    for (int k = 0; k < kCwP; ++k) {
        first |= static_cast<unsigned>(g0 + k == 0) << k;
        last |= static_cast<unsigned>(g0 + k + 1 == n) << k;
    }
    const unsigned full = 0xffffffffu;
    // The boundary flags matter only in the (at most two) warps holding
    // component 0 or n-1: every other warp runs the stages without them.
    auto stages = [&](auto edge_tag, const StepConsts& sc) {
    constexpr bool Edge = decltype(edge_tag)::value;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        double k0[kCwP], k1[kCwP];
        if constexpr (Kind == kKindTraffic) {
            const double v = m.P[0], c = m.P[2], beta = m.P[5];
            double F0[kCwP], F1[kCwP];  // flux of edge k -> k+1 (field 0; field 1 under MM)
            const double r0 = __shfl_down_sync(full, u0[0], 1);
#pragma unroll
            for (int k = 0; k < kCwP; ++k) F0[k] = traffic_flux<Exact>(m, u0[k], k + 1 < kCwP ? u0[k + 1] : r0);
            const double l0 = __shfl_up_sync(full, F0[kCwP - 1], 1);
            if constexpr (Method == kMethodMM) {
                const double r1 = __shfl_down_sync(full, u1[0], 1);
#pragma unroll
                for (int k = 0; k < kCwP; ++k)
                    F1[k] = traffic_flux<Exact>(m, u1[k], k + 1 < kCwP ? u1[k + 1] : r1);
            }
            const double l1 = Method == kMethodMM ? __shfl_up_sync(full, F1[kCwP - 1], 1) : 0.0;
            double gl = 0.0, gr = 0.0;  // growth: radius neighbours across lanes
            if constexpr (Method == kMethodGB) {
                gl = __shfl_up_sync(full, u1[kCwP - 1], 1);
                gr = __shfl_down_sync(full, u1[0], 1);
            }
#pragma unroll
            for (int k = 0; k < kCwP; ++k) {
                const bool fs = Edge && ((first >> k) & 1), ls = Edge && ((last >> k) & 1);
                {  // models.cpp:68-74, one flux per edge shared by its two ends
                    const double in = fs ? beta * m.p0 : beta * (k ? F0[k - 1] : l0);
                    const double out = ls ? ref_min(c, v * u0[k]) : F0[k];
                    k0[k] = m.inv_t * (in - out);
                }
                if constexpr (Method == kMethodMM) {
                    const double in = fs ? beta * m.p1 : beta * (k ? F1[k - 1] : l1);
                    const double out = ls ? ref_min(c, v * u1[k]) : F1[k];
                    k1[k] = m.inv_t * (in - out);
                } else {  // growth_rhs, models.cpp:78-87
                    double gv = fs ? m.a_in * m.p1 : m.a_prev * (k ? u1[k - 1] : gl);
                    if (!ls) gv += m.a_next * (k + 1 < kCwP ? u1[k + 1] : gr);
                    k1[k] = gv;
                }
            }
        } else {  // coupled chain: d_i(x,p,xh,ph) = ((-a) x_i + b s(x_{i-1}) - c s(xh_{i+1})) + p
            const double na = -m.P[0], b = m.P[1], c = m.P[2];
            double S0[kCwP], S1[kCwP];
#pragma unroll
            for (int k = 0; k < kCwP; ++k) {
                S0[k] = chain_sat<Exact>(u0[k]);
                S1[k] = chain_sat<Exact>(u1[k]);
            }
            const double S0l = __shfl_up_sync(full, S0[kCwP - 1], 1), S1l = __shfl_up_sync(full, S1[kCwP - 1], 1);
            const double S0r = __shfl_down_sync(full, S0[0], 1), S1r = __shfl_down_sync(full, S1[0], 1);
#pragma unroll
            for (int k = 0; k < kCwP; ++k) {
                const bool fs = Edge && ((first >> k) & 1), ls = Edge && ((last >> k) & 1);
                {
                    const double sl = fs ? 0.0 : (k ? S0[k - 1] : S0l);
                    const double sr = ls ? 0.0 : (k + 1 < kCwP ? S1[k + 1] : S1r);
                    k0[k] = (na * u0[k] + b * sl - c * sr) + m.p0;
                }
                {
                    const double sl = fs ? 0.0 : (k ? S1[k - 1] : S1l);
                    const double sr = ls ? 0.0 : (k + 1 < kCwP ? S0[k + 1] : S0r);
                    k1[k] = (na * u1[k] + b * sl - c * sr) + m.p1;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kCwP; ++k) {  // rk4.cpp:50-68, as chain_step_kernel
            if (s == 0) {
                acc0[k] = k0[k];
                acc1[k] = k1[k];
                u0[k] = x0[k] + sc.h2 * k0[k];
                u1[k] = x1[k] + sc.h2 * k1[k];
            } else if (s == 1) {
                acc0[k] = acc0[k] + 2.0 * k0[k];
                acc1[k] = acc1[k] + 2.0 * k1[k];
                u0[k] = x0[k] + sc.h2 * k0[k];
                u1[k] = x1[k] + sc.h2 * k1[k];
            } else if (s == 2) {
                acc0[k] = acc0[k] + 2.0 * k0[k];
                acc1[k] = acc1[k] + 2.0 * k1[k];
                u0[k] = x0[k] + sc.hk * k0[k];
                u1[k] = x1[k] + sc.hk * k1[k];
            } else {
                x0[k] = x0[k] + sc.h6 * (acc0[k] + k0[k]);
                x1[k] = x1[k] + sc.h6 * (acc1[k] + k1[k]);
            }
        }
    }
    };
    const bool edge = __any_sync(full, (first | last) != 0);
    // a component this warp outputs (the others are halo, owned by a neighbour)
    auto owned = [&](int k) {
        const int e = kCwP * lane + k;
        const long long g = g0 + k;
        return e >= kChainHalo * S && e < kCwSeg - kChainHalo * S && g >= static_cast<long long>(w.out_begin) &&
               g < static_cast<long long>(w.out_end);
    };
    auto flag = [&](int k, unsigned long long at) {  // rk4.cpp:72-75 key: (step, component)
        const long long g = g0 + k;
        if constexpr (Method == kMethodMM) {
            const unsigned long long comp =
                finite_d(x0[k]) ? static_cast<unsigned long long>(g) + static_cast<unsigned long long>(n)
                                : static_cast<unsigned long long>(g);
            record_fail(fail, at, comp);
        } else {
            if (!finite_d(x0[k])) record_fail(fail, at, static_cast<unsigned long long>(g));
            if (!finite_d(x1[k]) && fail) record_fail(fail + 1, at, static_cast<unsigned long long>(g));
        }
    };
#pragma unroll
    for (int st = 0; st < S; ++st) {
        const StepConsts& sc = scs.s[st];
        if (edge)
            stages(std::true_type{}, sc);
        else
            stages(std::false_type{}, sc);
        if (st + 1 < S) {  // intermediate state: flag it under its own step, restart the stages
#pragma unroll
            for (int k = 0; k < kCwP; ++k) {
                if (owned(k) && (!finite_d(x0[k]) || !finite_d(x1[k]))) flag(k, step + st);
                u0[k] = x0[k];
                u1[k] = x1[k];
                acc0[k] = acc1[k] = 0.0;
            }
        }
    }

    // ---- store the segment's outputs and flag non-finite values
#pragma unroll
    for (int k = 0; k < kCwP; ++k) {
        if (!owned(k)) continue;
        const long long g = g0 + k;
        const long long o = g - static_cast<long long>(w.out_begin);
        w.out0[o] = x0[k];
        w.out1[o] = x1[k];
        // units the neighbours need as halo: also into their windows, over peer memory
        if (w.mir0 && static_cast<uint64_t>(g) < w.mir_lo_end) {
            w.mir0[o] = x0[k];
            w.mir1[o] = x1[k];
        }
        if (w.mirh0 && static_cast<uint64_t>(g) >= w.mir_hi_begin) {
            w.mirh0[o] = x0[k];
            w.mirh1[o] = x1[k];
        }
        if (!finite_d(x0[k]) || !finite_d(x1[k])) flag(k, step + S - 1);
    }
}

template <bool Exact, int S>
cudaError_t launch_chain_warp(const ChainModel& m, const WindowArgs& w, const StepConstsN& scs,
                              unsigned long long step, unsigned long long* fail, cudaStream_t stream) {
    const uint64_t count = w.out_end - w.out_begin;
    const uint64_t per_block = static_cast<uint64_t>(kCwWarps) * cw_out<S>();
    dim3 wgrid(static_cast<unsigned>((count + per_block - 1) / per_block)), wblock(32 * kCwWarps);
    if (m.kind == kKindTraffic && m.method == kMethodMM)
        chain_warp_kernel<Exact, kKindTraffic, kMethodMM, S><<<wgrid, wblock, 0, stream>>>(m, w, scs, step, fail);
    else if (m.kind == kKindTraffic && m.method == kMethodGB)
        chain_warp_kernel<Exact, kKindTraffic, kMethodGB, S><<<wgrid, wblock, 0, stream>>>(m, w, scs, step, fail);
    else if (m.kind == kKindChain && m.method == kMethodMM)
        chain_warp_kernel<Exact, kKindChain, kMethodMM, S><<<wgrid, wblock, 0, stream>>>(m, w, scs, step, fail);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

// S = 2..4 RK4 steps in one launch (full-domain engine runs; temporal blocking).
template <bool Exact>
cudaError_t launch_chain_steps(const ChainModel& m, const WindowArgs& w, const StepConstsN& scs, int S,
                               unsigned long long step, unsigned long long* fail, cudaStream_t stream) {
    if (w.out_end <= w.out_begin) return cudaSuccess;
    switch (S) {
        case 2: return launch_chain_warp<Exact, 2>(m, w, scs, step, fail, stream);
        case 3: return launch_chain_warp<Exact, 3>(m, w, scs, step, fail, stream);
        case 4: return launch_chain_warp<Exact, 4>(m, w, scs, step, fail, stream);
        default: return cudaErrorInvalidValue;
    }
}

template <bool Exact>
cudaError_t launch_chain_step(const ChainModel& m, const WindowArgs& w, const StepConsts& sc,
                              unsigned long long step, unsigned long long* fail,
                              cudaStream_t stream) {
    if (w.out_end <= w.out_begin) return cudaSuccess;
    const uint64_t count = w.out_end - w.out_begin;
    // The warp-tiled kernel in both modes (n = 1e7, ms per step, warp vs smem
    // tiles: fast traffic 0.097 vs 0.139, chain 0.0995 vs 0.135; exact traffic
    // 0.165 vs 0.202, chain 0.153 vs 0.163).  PIRK_CHAIN_KERNEL=smem|warp
    // overrides (A/B comparisons, parity tests of both kernels).
#if PIRK_DEV_VARIANTS
    static const bool use_smem = [] {
        const char* v = std::getenv("PIRK_CHAIN_KERNEL");
        return v && std::strcmp(v, "smem") == 0;
    }();
#else
    const bool use_smem = false;
#endif
    if (!use_smem) {
        StepConstsN one;
        one.s[0] = sc;
        return launch_chain_warp<Exact, 1>(m, w, one, step, fail, stream);
    }
#if PIRK_DEV_VARIANTS
    const unsigned int blocks = static_cast<unsigned int>((count + kChainTile - 1) / kChainTile);
    dim3 grid(blocks), block(kChainThreads);
    if (m.kind == kKindTraffic && m.method == kMethodMM)
        chain_step_kernel<Exact, kKindTraffic, kMethodMM><<<grid, block, 0, stream>>>(m, w, sc, step, fail);
    else if (m.kind == kKindTraffic && m.method == kMethodGB)
        chain_step_kernel<Exact, kKindTraffic, kMethodGB><<<grid, block, 0, stream>>>(m, w, sc, step, fail);
    else if (m.kind == kKindChain && m.method == kMethodMM)
        chain_step_kernel<Exact, kKindChain, kMethodMM><<<grid, block, 0, stream>>>(m, w, sc, step, fail);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
#else
    (void)count;
    return cudaErrorInvalidValue;
#endif
}

}  // namespace pirk
