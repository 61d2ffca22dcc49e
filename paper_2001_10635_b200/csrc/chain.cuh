// chain.cuh -- K1: fused 4-stage RK4 step for 1-D radius-1 models on two fields.
//
// Replaces one call of integrate_step (rk4.cpp:30-76) on the embedding
// (system_model.cpp:56-77) of traffic (models.cpp:47-90) or the coupled chain
// (SURVEY.md 8d C4), or on the growth-bound pair [center | radius]
// (reach.cpp:103-114).
//
// A CTA of 256 threads owns a tile of 2048 components of BOTH fields (so a
// coupled decomposition reads the other field locally): 2040 outputs plus a
// halo of 4 (one per RK stage) on each side.  Each thread keeps 8 consecutive
// components of both fields in registers through all four stages; the
// radius-1 neighbours across thread boundaries come from warp shuffles, and
// across warp boundaries from a 16-double shared exchange -- one barrier per
// stage.  The tile is read once and written once: 16 B of HBM traffic per
// state-update instead of the reference's 144 B.
//
// Per-component arithmetic is exactly integrate_step's in exact mode:
//   k0 = f(x); u1 = x + h2*k0; k1 = f(u1); u2 = x + h2*k1; k2 = f(u2);
//   u3 = x + hk*k2; k3 = f(u3); x' = x + h6*(((k0 + 2k1) + 2k2) + k3).
// Traffic computes each edge flux once and uses it for both end components
// (identical inputs, so bit-identical to the reference's two evaluations).
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace pirk {

constexpr int kChainThreads = 256;
constexpr int kChainPerThread = 4;
constexpr int kChainSpan = kChainThreads * kChainPerThread;  // 1024 loaded components
constexpr int kChainHalo = 4;
constexpr int kChainTile = kChainSpan - 2 * kChainHalo;      // 1016 outputs per tile
constexpr int kChainWarps = kChainThreads / 32;

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

// s(z) = z / (1 + |z|) for the coupled chain.
__device__ __forceinline__ double chain_sat(double z) { return z / (1.0 + fabs(z)); }

__device__ __forceinline__ double shfl_up_d(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shfl_down_d(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

template <bool Exact, int Kind, int Method>
__global__ void __launch_bounds__(kChainThreads)
chain_step_kernel(const ChainModel m, const WindowArgs w, const StepConsts sc,
                  const unsigned long long step, unsigned long long* __restrict__ fail) {
    (void)sizeof(ModeCheck<Exact>);
    constexpr int E = kChainPerThread;
    // warp-edge exchange: [field][warp] first / last element of the warp
    __shared__ double sFirst[2][kChainWarps], sLast[2][kChainWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long n = static_cast<long long>(m.n);
    const long long base = static_cast<long long>(w.out_begin) +
                           static_cast<long long>(blockIdx.x) * kChainTile - kChainHalo;
    const long long g0 = base + static_cast<long long>(tid) * E;  // global index of element 0
    const long long wb = static_cast<long long>(w.win_begin), we = static_cast<long long>(w.win_end);

    double x0[E], x1[E], u0[E], u1[E], a0[E], a1[E];
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const long long g = g0 + e;
        const bool ok = g >= wb && g < we;
        x0[e] = ok ? __ldg(w.in0 + (g - wb)) : qnan;
        x1[e] = ok ? __ldg(w.in1 + (g - wb)) : qnan;
        u0[e] = x0[e];
        u1[e] = x1[e];
    }

#pragma unroll
    for (int s = 0; s < 4; ++s) {
        // ---- radius-1 neighbours of the thread's run: left of element 0, right of element 7
        double l0 = shfl_up_d(u0[E - 1]), l1 = shfl_up_d(u1[E - 1]);
        double r0 = shfl_down_d(u0[0]), r1 = shfl_down_d(u1[0]);
        if (lane == 0) {
            sFirst[0][warp] = u0[0];
            sFirst[1][warp] = u1[0];
        }
        if (lane == 31) {
            sLast[0][warp] = u0[E - 1];
            sLast[1][warp] = u1[E - 1];
        }
        __syncthreads();
        if (lane == 0 && warp > 0) {
            l0 = sLast[0][warp - 1];
            l1 = sLast[1][warp - 1];
        }
        if (lane == 31 && warp + 1 < kChainWarps) {
            r0 = sFirst[0][warp + 1];
            r1 = sFirst[1][warp + 1];
        }
        // (thread 0's left and thread 255's right neighbours are outside the
        // tile; they only feed halo components that never reach an output)

        double k0[E], k1[E];
        if constexpr (Kind == kKindTraffic) {
            const double v = m.P[0], c = m.P[2], beta = m.P[5];
            // edge fluxes F[e] = flux(u[e-1], u[e]) for e = 0..E (e=0: from the left neighbour)
            double F0[E + 1], F1[E + 1];
            F0[0] = traffic_flux<Exact>(m, l0, u0[0]);
#pragma unroll
            for (int e = 1; e < E; ++e) F0[e] = traffic_flux<Exact>(m, u0[e - 1], u0[e]);
            F0[E] = traffic_flux<Exact>(m, u0[E - 1], r0);
            if constexpr (Method == kMethodMM) {
                F1[0] = traffic_flux<Exact>(m, l1, u1[0]);
#pragma unroll
                for (int e = 1; e < E; ++e) F1[e] = traffic_flux<Exact>(m, u1[e - 1], u1[e]);
                F1[E] = traffic_flux<Exact>(m, u1[E - 1], r1);
            }
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const long long g = g0 + e;
                const bool first = (g == 0), last = (g + 1 == n);
                // models.cpp:68-74
                const double in0 = first ? beta * m.p0 : beta * F0[e];
                const double out0 = last ? ref_min(c, v * u0[e]) : F0[e + 1];
                k0[e] = m.inv_t * (in0 - out0);
                if constexpr (Method == kMethodMM) {
                    const double in1 = first ? beta * m.p1 : beta * F1[e];
                    const double out1 = last ? ref_min(c, v * u1[e]) : F1[e + 1];
                    k1[e] = m.inv_t * (in1 - out1);
                } else {
                    // growth_rhs, models.cpp:78-87
                    const double rl = (e == 0) ? l1 : u1[e - 1];
                    const double rr = (e == E - 1) ? r1 : u1[e + 1];
                    double gv = first ? m.a_in * m.p1 : m.a_prev * rl;
                    if (!last) gv += m.a_next * rr;
                    k1[e] = gv;
                }
            }
        } else {
            // coupled chain: d_i(x,p,xh,ph) = ((-a) x_i + b s(x_{i-1}) - c s(xh_{i+1})) + p
            const double na = -m.P[0], b = m.P[1], c = m.P[2];
            double S0[E + 2], S1[E + 2];  // s(u) at elements -1 .. E
            S0[0] = chain_sat(l0);
            S1[0] = chain_sat(l1);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                S0[e + 1] = chain_sat(u0[e]);
                S1[e + 1] = chain_sat(u1[e]);
            }
            S0[E + 1] = chain_sat(r0);
            S1[E + 1] = chain_sat(r1);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const long long g = g0 + e;
                const bool first = (g == 0), last = (g + 1 == n);
                const double sl0 = first ? 0.0 : S0[e], sr0 = last ? 0.0 : S1[e + 2];
                const double sl1 = first ? 0.0 : S1[e], sr1 = last ? 0.0 : S0[e + 2];
                k0[e] = (na * u0[e] + b * sl0 - c * sr0) + m.p0;
                k1[e] = (na * u1[e] + b * sl1 - c * sr1) + m.p1;
            }
        }

        // ---- stage update (integrate_step, rk4.cpp:50-68)
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (s == 0) {
                a0[e] = k0[e];
                a1[e] = k1[e];
                u0[e] = x0[e] + sc.h2 * k0[e];
                u1[e] = x1[e] + sc.h2 * k1[e];
            } else if (s == 1) {
                a0[e] = fma(2.0, k0[e], a0[e]);  // acc + 2.0*k (exact: 2k is exact)
                a1[e] = fma(2.0, k1[e], a1[e]);
                u0[e] = x0[e] + sc.h2 * k0[e];
                u1[e] = x1[e] + sc.h2 * k1[e];
            } else if (s == 2) {
                a0[e] = fma(2.0, k0[e], a0[e]);
                a1[e] = fma(2.0, k1[e], a1[e]);
                u0[e] = x0[e] + sc.hk * k0[e];
                u1[e] = x1[e] + sc.hk * k1[e];
            } else {
                x0[e] = x0[e] + sc.h6 * (a0[e] + k0[e]);
                x1[e] = x1[e] + sc.h6 * (a1[e] + k1[e]);
            }
        }
        if (s < 3) __syncthreads();  // the edge exchange buffers are rewritten next stage
    }

    // ---- store the tile's outputs and flag non-finite values
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int j = tid * E + e;
        const long long g = g0 + e;
        if (j < kChainHalo || j >= kChainSpan - kChainHalo) continue;
        if (g < static_cast<long long>(w.out_begin) || g >= static_cast<long long>(w.out_end))
            continue;
        const long long o = g - static_cast<long long>(w.out_begin);
        w.out0[o] = x0[e];
        w.out1[o] = x1[e];
        if (!finite_d(x0[e]) || !finite_d(x1[e])) {
            if constexpr (Method == kMethodMM) {
                // embedding components are numbered [x | xh] (system_model.cpp:67-75)
                const unsigned long long comp =
                    finite_d(x0[e]) ? static_cast<unsigned long long>(g + n)
                                    : static_cast<unsigned long long>(g);
                record_fail(fail, step, comp);
            } else {
                if (!finite_d(x0[e])) record_fail(fail, step, static_cast<unsigned long long>(g));
                if (!finite_d(x1[e]) && fail)
                    record_fail(fail + 1, step, static_cast<unsigned long long>(g));
            }
        }
    }
}

template <bool Exact>
cudaError_t launch_chain_step(const ChainModel& m, const WindowArgs& w, const StepConsts& sc,
                              unsigned long long step, unsigned long long* fail,
                              cudaStream_t stream) {
    if (w.out_end <= w.out_begin) return cudaSuccess;
    const uint64_t count = w.out_end - w.out_begin;
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
}

}  // namespace pirk
