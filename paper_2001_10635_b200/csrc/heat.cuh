// heat.cuh -- K2: fused 4-stage RK4 step of the heat3d 7-point stencil.
//
// Replaces integrate_step (rk4.cpp:30-76) on the embedding of heat3d
// (models.cpp:92-133; cooperative, so the lower and upper fields evolve
// independently and each is the plain stencil) and on the growth-bound pair
// (growth_rhs == rhs for heat3d, models.cpp:130).
//
// Design (2.5-D z-streaming): a CTA owns a 32x32 x-y tile of one field and
// streams z.  Iteration j loads plane j (x-y halo 4, cp.async, one plane of
// prefetch), then computes
//     stage 1 (k0, u1) at plane j-1 on the tile + halo 3,
//     stage 2 (k1, u2) at plane j-2 on the tile + halo 2,
//     stage 3 (k2, u3) at plane j-3 on the tile + halo 1,
//     stage 4 (k3, x') at plane j-4 on the tile,
// keeping rings of planes for x (6), u1/u2/u3 (3 each) and the RK
// accumulator (4) in shared memory.  HBM sees each x once and each x' once:
// 16 B per state-update.
//
// Exact mode evaluates models.cpp:113-126 literally (acc = 0.0; acc += ...
// in the order x-, x+, y-, y+, z-, z+; the Robin ghost at ix = 0; k*acc).  A
// skipped (insulated) face adds +0.0, which leaves acc unchanged because acc
// is never -0.0 (it starts at +0.0 and round-to-nearest sums of nonzero terms
// are never -0).  Fast mode uses ghost values (insulated: ghost = self; Robin:
// ghost = x[i+1] - robin*self), one sum-then-subtract and folded constants.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace pirk {

constexpr int kHeatT = 32;                  // output tile edge (x and y)
constexpr int kHeatH = 4;                   // halo = number of RK stages
constexpr int kHeatThreads = 512;
constexpr int kHeatW0 = kHeatT + 2 * kHeatH;  // 40: loaded x plane edge
constexpr int kHeatW1 = kHeatW0 - 2;          // 38: u1 plane edge
constexpr int kHeatW2 = kHeatW0 - 4;          // 36
constexpr int kHeatW3 = kHeatW0 - 6;          // 34
constexpr int kHeatXRing = 6;                 // planes j-4 .. j+1
constexpr int kHeatURing = 3;
constexpr int kHeatARing = 4;

constexpr size_t kHeatSmemDoubles =
    size_t(kHeatXRing) * kHeatW0 * kHeatW0 + size_t(kHeatURing) * kHeatW1 * kHeatW1 +
    size_t(kHeatURing) * kHeatW2 * kHeatW2 + size_t(kHeatURing) * kHeatW3 * kHeatW3 +
    size_t(kHeatARing) * kHeatT * kHeatT;
constexpr size_t kHeatSmemBytes = kHeatSmemDoubles * sizeof(double);

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

struct HeatStepParams {
    double kk, robin;
    // fast-mode folded constants
    double h2kk, hkk, h6kk;
};

// One stencil evaluation.  Returns k (exact) or t = sum - 6 self with k = kk*t (fast).
template <bool Exact>
__device__ __forceinline__ double heat_point(double s, double xm, double xp, double ym, double yp,
                                             double zm, double zp, bool hx_m, bool hx_p,
                                             bool hy_m, bool hy_p, bool hz_m, bool hz_p,
                                             double robin, double kk) {
    if constexpr (Exact) {
        double acc = 0.0;
        acc += hx_m ? (xm - s) : ((xp - s) - robin * s);
        acc += hx_p ? (xp - s) : 0.0;
        acc += hy_m ? (ym - s) : 0.0;
        acc += hy_p ? (yp - s) : 0.0;
        acc += hz_m ? (zm - s) : 0.0;
        acc += hz_p ? (zp - s) : 0.0;
        return kk * acc;
    } else {
        const double gxm = hx_m ? xm : fma(-robin, s, xp);
        const double gxp = hx_p ? xp : s;
        const double gym = hy_m ? ym : s;
        const double gyp = hy_p ? yp : s;
        const double gzm = hz_m ? zm : s;
        const double gzp = hz_p ? zp : s;
        const double sum = ((gxm + gxp) + (gym + gyp)) + (gzm + gzp);
        return fma(-6.0, s, sum);
    }
}

template <bool Exact>
__global__ void __launch_bounds__(kHeatThreads, 1)
heat_step_kernel(const HeatModel m, const HeatStepParams hp, const WindowArgs w,
                 const StepConsts sc, const unsigned long long step, const uint64_t zchunk,
                 unsigned long long* __restrict__ fail) {
    (void)sizeof(ModeCheck<Exact>);
    extern __shared__ __align__(16) double smem[];
    double* sX = smem;                                            // [6][40*40]
    double* sU1 = sX + kHeatXRing * kHeatW0 * kHeatW0;            // [3][38*38]
    double* sU2 = sU1 + kHeatURing * kHeatW1 * kHeatW1;           // [3][36*36]
    double* sU3 = sU2 + kHeatURing * kHeatW2 * kHeatW2;           // [3][34*34]
    double* sAcc = sU3 + kHeatURing * kHeatW3 * kHeatW3;          // [4][32*32]

    const int tid = threadIdx.x;
    const long long g = static_cast<long long>(m.g);
    const long long g2 = g * g;
    const int field = blockIdx.z & 1;
    const long long chunk = blockIdx.z >> 1;
    const long long ix0 = static_cast<long long>(blockIdx.x) * kHeatT;
    const long long iy0 = static_cast<long long>(blockIdx.y) * kHeatT;

    const long long ob = static_cast<long long>(w.out_begin) + chunk * static_cast<long long>(zchunk);
    long long oe = ob + static_cast<long long>(zchunk);
    if (oe > static_cast<long long>(w.out_end)) oe = static_cast<long long>(w.out_end);
    if (ob >= oe) return;
    // planes streamed through the CTA and the validity of each stage level
    const long long zs = (ob - kHeatH > 0) ? ob - kHeatH : 0;
    const long long ze = (oe + kHeatH < g) ? oe + kHeatH : g;
    const long long lo_shift = (zs > 0) ? 1 : 0;
    const long long hi_shift = (ze < g) ? 1 : 0;

    const double* __restrict__ src = field ? w.in1 : w.in0;
    double* __restrict__ dst = field ? w.out1 : w.out0;
    const long long wb = static_cast<long long>(w.win_begin);

    auto load_plane = [&](long long p) {
        double* slot = sX + (p % kHeatXRing) * (kHeatW0 * kHeatW0);
        const double* plane = src + (p - wb) * g2;
        for (int q = tid; q < kHeatW0 * kHeatW0; q += kHeatThreads) {
            const int y = q / kHeatW0, x = q - (q / kHeatW0) * kHeatW0;
            const long long ix = ix0 - kHeatH + x, iy = iy0 - kHeatH + y;
            if (ix >= 0 && ix < g && iy >= 0 && iy < g) cp_async8(slot + q, plane + iy * g + ix);
        }
        cp_async_commit();
    };

    load_plane(zs);

    for (long long j = zs; j < ze + kHeatH; ++j) {
        cp_async_wait_all();
        __syncthreads();
        if (j + 1 < ze) load_plane(j + 1);

        // stages 1..4 at planes j-1 .. j-4
#pragma unroll
        for (int L = 1; L <= 4; ++L) {
            const long long p = j - L;
            const bool valid = (p >= zs + L * lo_shift) && (p < ze - L * hi_shift) &&
                               (L < 4 || (p >= ob && p < oe));
            if (valid) {
                const int Wd = kHeatW0 - 2 * L;      // this level's edge
                const int Ws = Wd + 2;               // source level's edge
                const int off = kHeatH - L;          // level origin relative to tile origin
                const double* sp;                    // source ring
                int sring;
                if (L == 1) { sp = sX; sring = kHeatXRing; }
                else if (L == 2) { sp = sU1; sring = kHeatURing; }
                else if (L == 3) { sp = sU2; sring = kHeatURing; }
                else { sp = sU3; sring = kHeatURing; }
                const int splane = Ws * Ws;
                const double* s_c = sp + (p % sring) * splane;
                const double* s_m = (p > 0) ? sp + ((p - 1) % sring) * splane : s_c;
                const double* s_p = (p + 1 < g) ? sp + ((p + 1) % sring) * splane : s_c;
                const double* xc = sX + (p % kHeatXRing) * (kHeatW0 * kHeatW0);
                double* ud = (L == 1) ? sU1 + (p % kHeatURing) * (kHeatW1 * kHeatW1)
                           : (L == 2) ? sU2 + (p % kHeatURing) * (kHeatW2 * kHeatW2)
                           : (L == 3) ? sU3 + (p % kHeatURing) * (kHeatW3 * kHeatW3)
                                      : nullptr;
                double* acc = sAcc + (p % kHeatARing) * (kHeatT * kHeatT);
                const bool hz_m = p > 0, hz_p = p + 1 < g;
                for (int q = tid; q < Wd * Wd; q += kHeatThreads) {
                    const int y = q / Wd, x = q - (q / Wd) * Wd;
                    const long long ix = ix0 - off + x, iy = iy0 - off + y;
                    if (ix < 0 || ix >= g || iy < 0 || iy >= g) continue;
                    const int si = (y + 1) * Ws + (x + 1);
                    const double s = s_c[si];
                    const double kv = heat_point<Exact>(
                        s, s_c[si - 1], s_c[si + 1], s_c[si - Ws], s_c[si + Ws], s_m[si], s_p[si],
                        ix > 0, ix + 1 < g, iy > 0, iy + 1 < g, hz_m, hz_p, hp.robin, hp.kk);
                    const double xv = xc[(y + L) * kHeatW0 + (x + L)];  // level-L (x,y) is level-0 (x+L, y+L)
                    const int ax = x - off, ay = y - off;  // accumulator coordinates
                    const bool own = ax >= 0 && ax < kHeatT && ay >= 0 && ay < kHeatT;
                    const int ai = ay * kHeatT + ax;
                    if constexpr (Exact) {
                        if (L == 1) {
                            ud[q] = xv + sc.h2 * kv;
                            if (own) acc[ai] = kv;
                        } else if (L == 2) {
                            ud[q] = xv + sc.h2 * kv;
                            if (own) acc[ai] = acc[ai] + 2.0 * kv;
                        } else if (L == 3) {
                            ud[q] = xv + sc.hk * kv;
                            if (own) acc[ai] = acc[ai] + 2.0 * kv;
                        } else {
                            const double xn = xv + sc.h6 * (acc[ai] + kv);
                            const long long gi = ((p * g) + iy) * g + ix;
                            dst[(p - static_cast<long long>(w.out_begin)) * g2 + iy * g + ix] = xn;
                            if (!finite_d(xn)) {
                                if (m.method == 0)
                                    record_fail(fail, step, static_cast<unsigned long long>(gi) +
                                                                (field ? static_cast<unsigned long long>(g2 * g) : 0ull));
                                else if (fail)
                                    record_fail(fail + field, step, static_cast<unsigned long long>(gi));
                            }
                        }
                    } else {
                        // kv is t = sum - 6 self; k = kk * t folded into the constants
                        if (L == 1) {
                            ud[q] = fma(hp.h2kk, kv, xv);
                            if (own) acc[ai] = kv;
                        } else if (L == 2) {
                            ud[q] = fma(hp.h2kk, kv, xv);
                            if (own) acc[ai] = fma(2.0, kv, acc[ai]);
                        } else if (L == 3) {
                            ud[q] = fma(hp.hkk, kv, xv);
                            if (own) acc[ai] = fma(2.0, kv, acc[ai]);
                        } else {
                            const double xn = fma(hp.h6kk, acc[ai] + kv, xv);
                            const long long gi = ((p * g) + iy) * g + ix;
                            dst[(p - static_cast<long long>(w.out_begin)) * g2 + iy * g + ix] = xn;
                            if (!finite_d(xn)) {
                                if (m.method == 0)
                                    record_fail(fail, step, static_cast<unsigned long long>(gi) +
                                                                (field ? static_cast<unsigned long long>(g2 * g) : 0ull));
                                else if (fail)
                                    record_fail(fail + field, step, static_cast<unsigned long long>(gi));
                            }
                        }
                    }
                }
            }
            if (L < 4) __syncthreads();
        }
    }
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
    const uint64_t tiles = ((m.g + kHeatT - 1) / kHeatT) * ((m.g + kHeatT - 1) / kHeatT);
    uint64_t nchunks = 1;
    while (tiles * 2 * nchunks < 4 * 148 && planes / (nchunks * 2) >= 64) nchunks *= 2;
    const uint64_t zchunk = (planes + nchunks - 1) / nchunks;
    nchunks = (planes + zchunk - 1) / zchunk;
    const unsigned tx = static_cast<unsigned>((m.g + kHeatT - 1) / kHeatT);
    dim3 grid(tx, tx, static_cast<unsigned>(2 * nchunks)), block(kHeatThreads);
    heat_step_kernel<Exact><<<grid, block, kHeatSmemBytes, stream>>>(m, hp, w, sc, step, zchunk, fail);
    return cudaGetLastError();
}

}  // namespace pirk
