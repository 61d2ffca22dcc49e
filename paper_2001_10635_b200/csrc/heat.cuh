// heat.cuh -- K2: fused 4-stage RK4 step of the heat3d 7-point stencil.
//
// Replaces integrate_step (rk4.cpp:30-76) on the embedding of heat3d
// (models.cpp:92-133; cooperative, so the lower and upper fields evolve
// independently and each is the plain stencil) and on the growth-bound pair
// (growth_rhs == rhs for heat3d, models.cpp:130).
//
// Design (2.5-D z-streaming).  A CTA of 512 threads owns a 32x32 x-y tile of
// one field and streams z.  Iteration j
//     - issues the global loads of x-plane j+1 (tile + halo 4) into registers,
//     - stage 1 (k0, u1) at plane j-1 on the tile + halo 3,
//     - stage 2 (k1, u2) at plane j-2 on the tile + halo 2,
//     - stage 3 (k2, u3) at plane j-3 on the tile + halo 1,
//     - stage 4 (k3, x') at plane j-4 on the tile, stored to HBM,
//     - writes plane j+1 into the shared-memory x ring.
// Shared memory holds rings of planes (x: 5, u1/u2/u3: 3 each), all with the
// same 40x40 pitch so every buffer uses the same neighbour offsets.  Each
// thread owns two tile points (rows t/32 and t/32+16) whose RK accumulator
// and x values live in registers across the four lagged stages, plus at most
// one point of each level's halo ring; all shared-memory offsets are computed
// once per CTA.  HBM sees each x once and each x' once: 16 B/state-update.
//
// Boundaries.  Interior tiles (the halo-4 footprint inside the grid in x and
// y) run without per-point checks.  The insulated z faces use the centre
// plane as the missing neighbour: the term (s - s) = +0.0 leaves the sum
// unchanged exactly as skipping it does (the running sum is never -0.0: it
// starts at +0.0 and round-to-nearest sums of nonzero terms are never -0).
// Edge tiles evaluate models.cpp:113-126 with per-point face flags.
//
// Exact mode evaluates models.cpp:113-126 literally (acc = 0.0; acc += ...
// in the order x-, x+, y-, y+, z-, z+, the Robin term at ix = 0, k*acc) and
// integrate_step's stage arithmetic (acc + 2.0*k as an exact FMA).  Fast mode
// uses ghost values, one sum-then-subtract and constants folded with k.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace pirk {

constexpr int kHeatT = 32;                 // output tile edge (x and y)
constexpr int kHeatH = 4;                  // halo = number of RK stages
constexpr int kHeatP = kHeatT + 2 * kHeatH;  // 40: pitch of every plane buffer
constexpr int kHeatPlane = kHeatP * kHeatP;  // 1600
constexpr int kHeatThreads = 512;
constexpr int kHeatRing = 4;               // planes per ring (x, u1, u2, u3)
constexpr int kHeatLoads = (kHeatPlane + kHeatThreads - 1) / kHeatThreads;  // 4
constexpr size_t kHeatSmemBytes = size_t(4 * kHeatRing) * kHeatPlane * sizeof(double);  // 204,800 B

struct HeatStepParams {
    double kk, robin;
    double h2kk, hkk, h6kk;  // fast-mode folded constants
};

// face flags for edge tiles
enum : int { kXm = 1, kXp = 2, kYm = 4, kYp = 8, kIn = 16 };

// One stencil evaluation at level-0 offset `o` of plane c (neighbour planes
// zm/zp, equal to c on an insulated z face).  Exact: returns k = kk*acc.
// Fast: returns t = (sum of neighbours) - 6*self (k = kk*t is folded later).
template <bool Exact, bool Interior>
__device__ __forceinline__ double heat_eval(const double* __restrict__ c,
                                            const double* __restrict__ zm,
                                            const double* __restrict__ zp, int o, int flags,
                                            const HeatStepParams& hp) {
    const double s = c[o];
    const double xm = c[o - 1], xp = c[o + 1];
    const double ym = c[o - kHeatP], yp = c[o + kHeatP];
    const double vzm = zm[o], vzp = zp[o];
    if constexpr (Exact) {
        double acc = 0.0;
        if constexpr (Interior) {
            acc += xm - s;
            acc += xp - s;
            acc += ym - s;
            acc += yp - s;
        } else {
            acc += (flags & kXm) ? (xm - s) : ((xp - s) - hp.robin * s);
            acc += (flags & kXp) ? (xp - s) : 0.0;
            acc += (flags & kYm) ? (ym - s) : 0.0;
            acc += (flags & kYp) ? (yp - s) : 0.0;
        }
        acc += vzm - s;
        acc += vzp - s;
        return hp.kk * acc;
    } else {
        double gxm = xm, gxp = xp, gym = ym, gyp = yp;
        if constexpr (!Interior) {
            gxm = (flags & kXm) ? xm : fma(-hp.robin, s, xp);
            gxp = (flags & kXp) ? xp : s;
            gym = (flags & kYm) ? ym : s;
            gyp = (flags & kYp) ? yp : s;
        }
        const double sum = ((gxm + gxp) + (gym + gyp)) + (vzm + vzp);
        return fma(-6.0, s, sum);
    }
}

struct HeatThread {
    int own_off[2];     // level-0 offsets of the two own points
    int own_flags[2];
    int own_g[2];       // in-plane global offset iy*g + ix (valid iff flags & kIn)
    int ring_off[3];    // level L = 1..3 halo-ring point (-1: none)
    int ring_flags[3];
    int ld_q[kHeatLoads];   // smem offset of each prefetched element (-1: none)
    int ld_g[kHeatLoads];   // in-plane global offset
};

__device__ __forceinline__ int face_flags(long long ix, long long iy, long long g) {
    int f = 0;
    if (ix >= 0 && ix < g && iy >= 0 && iy < g) f |= kIn;
    if (ix > 0) f |= kXm;
    if (ix + 1 < g) f |= kXp;
    if (iy > 0) f |= kYm;
    if (iy + 1 < g) f |= kYp;
    return f;
}

// Shared-memory rings: 4 slots per level (x, u1, u2, u3), slot of plane p =
// (p - zs) mod 4.  With the plane loop unrolled by 4, every slot offset below
// is a compile-time immediate.
template <int PH, int Back>
__device__ __forceinline__ constexpr int heat_slot(int level) {
    return (level * kHeatRing + ((PH - Back + 8) & 3)) * kHeatPlane;
}

template <bool Exact, bool Interior, int PH>
__device__ __forceinline__ void heat_iteration(const HeatModel& m, const HeatStepParams& hp,
                                               const StepConsts& sc, unsigned long long step,
                                               unsigned long long* fail, const HeatThread& th,
                                               double* __restrict__ smem, int field, int j,
                                               int zs, int ze, int ob, int oe, int lo_shift,
                                               int hi_shift, int g, long long g2,
                                               const double* __restrict__ src,
                                               double* __restrict__ dst, double (&xr)[2][4],
                                               double (&ar)[2][4], double (&pre)[kHeatLoads]) {
    __syncthreads();
    const bool more = j + 1 < ze;
    if (more) {
        const double* plane = src + static_cast<long long>(j + 1) * g2;
#pragma unroll
        for (int i = 0; i < kHeatLoads; ++i)
            if (th.ld_q[i] >= 0) pre[i] = __ldg(plane + th.ld_g[i]);
    }

    // ---- stage 1 at plane p = j - 1 (own points + level-1 ring point)
    {
        const int p = j - 1;
        if (p >= zs + lo_shift && p < ze - hi_shift) {
            const double* c = smem + heat_slot<PH, 1>(0);
            const double* zm = (p > 0) ? smem + heat_slot<PH, 2>(0) : c;
            const double* zp = (p + 1 < g) ? smem + heat_slot<PH, 0>(0) : c;
            double* u = smem + heat_slot<PH, 1>(1);
            constexpr int R = (PH + 3) & 3;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (!Interior && !(th.own_flags[k] & kIn)) continue;
                const int o = th.own_off[k];
                const double kv = heat_eval<Exact, Interior>(c, zm, zp, o, th.own_flags[k], hp);
                const double x = c[o];
                xr[k][R] = x;
                ar[k][R] = kv;
                u[o] = Exact ? x + sc.h2 * kv : fma(hp.h2kk, kv, x);
            }
            const int o = th.ring_off[0];
            if (o >= 0 && (Interior || (th.ring_flags[0] & kIn))) {
                const double kv = heat_eval<Exact, Interior>(c, zm, zp, o, th.ring_flags[0], hp);
                u[o] = Exact ? c[o] + sc.h2 * kv : fma(hp.h2kk, kv, c[o]);
            }
        }
    }
    __syncthreads();
    // ---- stage 2 at plane j - 2
    {
        const int p = j - 2;
        if (p >= zs + 2 * lo_shift && p < ze - 2 * hi_shift) {
            const double* c = smem + heat_slot<PH, 2>(1);
            const double* zm = (p > 0) ? smem + heat_slot<PH, 3>(1) : c;
            const double* zp = (p + 1 < g) ? smem + heat_slot<PH, 1>(1) : c;
            double* u = smem + heat_slot<PH, 2>(2);
            constexpr int R = (PH + 2) & 3;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (!Interior && !(th.own_flags[k] & kIn)) continue;
                const int o = th.own_off[k];
                const double kv = heat_eval<Exact, Interior>(c, zm, zp, o, th.own_flags[k], hp);
                const double x = xr[k][R];
                ar[k][R] = fma(2.0, kv, ar[k][R]);  // acc + 2.0*k (exact: 2k is exact)
                u[o] = Exact ? x + sc.h2 * kv : fma(hp.h2kk, kv, x);
            }
            const int o = th.ring_off[1];
            if (o >= 0 && (Interior || (th.ring_flags[1] & kIn))) {
                const double kv = heat_eval<Exact, Interior>(c, zm, zp, o, th.ring_flags[1], hp);
                const double x = smem[heat_slot<PH, 2>(0) + o];
                u[o] = Exact ? x + sc.h2 * kv : fma(hp.h2kk, kv, x);
            }
        }
    }
    __syncthreads();
    // ---- stage 3 at plane j - 3
    {
        const int p = j - 3;
        if (p >= zs + 3 * lo_shift && p < ze - 3 * hi_shift) {
            const double* c = smem + heat_slot<PH, 3>(2);
            const double* zm = (p > 0) ? smem + heat_slot<PH, 4>(2) : c;
            const double* zp = (p + 1 < g) ? smem + heat_slot<PH, 2>(2) : c;
            double* u = smem + heat_slot<PH, 3>(3);
            constexpr int R = (PH + 1) & 3;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (!Interior && !(th.own_flags[k] & kIn)) continue;
                const int o = th.own_off[k];
                const double kv = heat_eval<Exact, Interior>(c, zm, zp, o, th.own_flags[k], hp);
                const double x = xr[k][R];
                ar[k][R] = fma(2.0, kv, ar[k][R]);
                u[o] = Exact ? x + sc.hk * kv : fma(hp.hkk, kv, x);
            }
            const int o = th.ring_off[2];
            if (o >= 0 && (Interior || (th.ring_flags[2] & kIn))) {
                const double kv = heat_eval<Exact, Interior>(c, zm, zp, o, th.ring_flags[2], hp);
                const double x = smem[heat_slot<PH, 3>(0) + o];
                u[o] = Exact ? x + sc.hk * kv : fma(hp.hkk, kv, x);
            }
        }
    }
    __syncthreads();
    // x plane j+1 takes the slot of plane j-3, dead after stage 3
    if (more) {
        double* slot = smem + heat_slot<PH, 3>(0);
#pragma unroll
        for (int i = 0; i < kHeatLoads; ++i)
            if (th.ld_q[i] >= 0) slot[th.ld_q[i]] = pre[i];
    }
    // ---- stage 4 at plane j - 4 (own points only), stored to HBM
    {
        const int p = j - 4;
        if (p >= ob && p < oe) {
            const double* c = smem + heat_slot<PH, 4>(3);
            const double* zm = (p > 0) ? smem + heat_slot<PH, 5>(3) : c;
            const double* zp = (p + 1 < g) ? smem + heat_slot<PH, 3>(3) : c;
            constexpr int R = PH & 3;
            double* out = dst + static_cast<long long>(p) * g2;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (!Interior && !(th.own_flags[k] & kIn)) continue;
                const int o = th.own_off[k];
                const double kv = heat_eval<Exact, Interior>(c, zm, zp, o, th.own_flags[k], hp);
                const double x = xr[k][R];
                const double xn =
                    Exact ? x + sc.h6 * (ar[k][R] + kv) : fma(hp.h6kk, ar[k][R] + kv, x);
                out[th.own_g[k]] = xn;
                if (!finite_d(xn)) {
                    const unsigned long long gi = static_cast<unsigned long long>(
                        static_cast<long long>(p) * g2 + th.own_g[k]);
                    if (m.method == 0)
                        record_fail(fail, step,
                                    gi + (field ? static_cast<unsigned long long>(g2 * g) : 0ull));
                    else if (fail)
                        record_fail(fail + field, step, gi);
                }
            }
        }
    }
}

template <bool Exact, bool Interior>
__device__ __forceinline__ void heat_stream(const HeatModel& m, const HeatStepParams& hp,
                                            const WindowArgs& w, const StepConsts& sc,
                                            unsigned long long step, unsigned long long* fail,
                                            const HeatThread& th, double* smem, int field,
                                            int ob, int oe) {
    const int g = static_cast<int>(m.g);
    const long long g2 = static_cast<long long>(g) * g;
    const int zs = (ob - kHeatH > 0) ? ob - kHeatH : 0;
    const int ze = (oe + kHeatH < g) ? oe + kHeatH : g;
    const int lo_shift = (zs > 0) ? 1 : 0;
    const int hi_shift = (ze < g) ? 1 : 0;
    const double* __restrict__ src =
        (field ? w.in1 : w.in0) - static_cast<long long>(w.win_begin) * g2;
    double* __restrict__ dst = (field ? w.out1 : w.out0) - static_cast<long long>(w.out_begin) * g2;

    double xr[2][4], ar[2][4], pre[kHeatLoads];
    {  // plane zs -> x slot 0
        const double* plane = src + static_cast<long long>(zs) * g2;
#pragma unroll
        for (int i = 0; i < kHeatLoads; ++i)
            if (th.ld_q[i] >= 0) smem[th.ld_q[i]] = __ldg(plane + th.ld_g[i]);
    }
    const int jend = ze + kHeatH;
#define PIRK_HEAT_IT(PH)                                                                        \
    heat_iteration<Exact, Interior, PH>(m, hp, sc, step, fail, th, smem, field, j + PH, zs, ze, \
                                        ob, oe, lo_shift, hi_shift, g, g2, src, dst, xr, ar, pre)
    for (int j = zs; j < jend; j += 4) {
        PIRK_HEAT_IT(0);
        if (j + 1 < jend) PIRK_HEAT_IT(1);
        if (j + 2 < jend) PIRK_HEAT_IT(2);
        if (j + 3 < jend) PIRK_HEAT_IT(3);
    }
#undef PIRK_HEAT_IT
}

template <bool Exact>
__global__ void __launch_bounds__(kHeatThreads, 1)
heat_step_kernel(const HeatModel m, const HeatStepParams hp, const WindowArgs w,
                 const StepConsts sc, const unsigned long long step, const uint64_t zchunk,
                 unsigned long long* __restrict__ fail) {
    (void)sizeof(ModeCheck<Exact>);
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x;
    const long long g = static_cast<long long>(m.g);
    const int field = blockIdx.z & 1;
    const long long chunk = blockIdx.z >> 1;
    const long long ix0 = static_cast<long long>(blockIdx.x) * kHeatT;
    const long long iy0 = static_cast<long long>(blockIdx.y) * kHeatT;
    const long long ob = static_cast<long long>(w.out_begin) + chunk * static_cast<long long>(zchunk);
    long long oe = ob + static_cast<long long>(zchunk);
    if (oe > static_cast<long long>(w.out_end)) oe = static_cast<long long>(w.out_end);
    if (ob >= oe) return;

    // ---- per-thread static assignment
    HeatThread th;
    {
        const int ox = tid & 31, oy = tid >> 5;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int y = oy + 16 * k;
            th.own_off[k] = (y + kHeatH) * kHeatP + (ox + kHeatH);
            const long long ix = ix0 + ox, iy = iy0 + y;
            th.own_flags[k] = face_flags(ix, iy, g);
            th.own_g[k] = static_cast<int>(iy * g + ix);
        }
#pragma unroll
        for (int L = 1; L <= 3; ++L) {
            const int hw = kHeatH - L, W = kHeatT + 2 * hw;
            const int count = W * W - kHeatT * kHeatT;
            th.ring_off[L - 1] = -1;
            th.ring_flags[L - 1] = 0;
            if (tid < count) {
                int r = tid, x, y;
                if (r < hw * W) { y = r / W; x = r % W; }
                else if ((r -= hw * W) < hw * W) { y = W - hw + r / W; x = r % W; }
                else { r -= hw * W; y = hw + r / (2 * hw); const int c = r % (2 * hw); x = (c < hw) ? c : kHeatT + c; }
                th.ring_off[L - 1] = (y + L) * kHeatP + (x + L);
                th.ring_flags[L - 1] = face_flags(ix0 - hw + x, iy0 - hw + y, g);
            }
        }
#pragma unroll
        for (int i = 0; i < kHeatLoads; ++i) {
            const int q = tid + i * kHeatThreads;
            th.ld_q[i] = -1;
            th.ld_g[i] = 0;
            if (q < kHeatPlane) {
                const long long ix = ix0 - kHeatH + q % kHeatP, iy = iy0 - kHeatH + q / kHeatP;
                if (ix >= 0 && ix < g && iy >= 0 && iy < g) {
                    th.ld_q[i] = q;
                    th.ld_g[i] = static_cast<int>(iy * g + ix);
                }
            }
        }
    }
    const bool interior = ix0 - kHeatH >= 0 && ix0 + kHeatT + kHeatH <= g && iy0 - kHeatH >= 0 &&
                          iy0 + kHeatT + kHeatH <= g;
    if (interior)
        heat_stream<Exact, true>(m, hp, w, sc, step, fail, th, smem, field,
                                  static_cast<int>(ob), static_cast<int>(oe));
    else
        heat_stream<Exact, false>(m, hp, w, sc, step, fail, th, smem, field,
                                  static_cast<int>(ob), static_cast<int>(oe));
}

template <bool Exact>
cudaError_t launch_heat_step(const HeatModel& m, const WindowArgs& w, const StepConsts& sc,
                             unsigned long long step, unsigned long long* fail,
                             cudaStream_t stream) {
    if (w.out_end <= w.out_begin) return cudaSuccess;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(heat_step_kernel<Exact>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kHeatSmemBytes));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    HeatStepParams hp;
    hp.kk = m.kk;
    hp.robin = m.robin;
    hp.h2kk = sc.h2 * m.kk;
    hp.hkk = sc.hk * m.kk;
    hp.h6kk = sc.h6 * m.kk;
    const uint64_t planes = w.out_end - w.out_begin;
    // z chunks: enough CTAs to fill the machine, few enough to keep the
    // 8-plane halo overhead per chunk small.
    const uint64_t tx = (m.g + kHeatT - 1) / kHeatT;
    uint64_t nchunks = 1;
    while (tx * tx * 2 * nchunks < 4 * 148 && planes / (nchunks * 2) >= 64) nchunks *= 2;
    const uint64_t zchunk = (planes + nchunks - 1) / nchunks;
    nchunks = (planes + zchunk - 1) / zchunk;
    dim3 grid(static_cast<unsigned>(tx), static_cast<unsigned>(tx), static_cast<unsigned>(2 * nchunks));
    heat_step_kernel<Exact><<<grid, kHeatThreads, kHeatSmemBytes, stream>>>(m, hp, w, sc, step, zchunk, fail);
    return cudaGetLastError();
}

}  // namespace pirk
