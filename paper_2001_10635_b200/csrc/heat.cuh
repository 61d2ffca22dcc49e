// heat.cuh -- K2: fused 4-stage RK4 step of the heat3d 7-point stencil.
//
// Replaces integrate_step (rk4.cpp:30-76) on the embedding of heat3d
// (models.cpp:92-133; cooperative, so the lower and upper fields evolve
// independently and each is the plain stencil) and on the growth-bound pair
// (growth_rhs == rhs for heat3d, models.cpp:130).
//
// Design: 2.5-D z-streaming with register-resident z histories.
//   A CTA of 256 threads owns a 32x32 x-y tile of one field and streams the
//   planes of a z-chunk.  Iteration j loads x-plane j+1 (tile + halo 4) and
//   evaluates stage 1 at plane j-1, stage 2 at j-2, stage 3 at j-3 and stage 4
//   (the RK4 combination, stored to HBM) at j-4.  Every (x, y) column of the
//   40x40 footprint is owned by one thread for the whole run, so the values of
//   a column at neighbouring planes (the z+-1 terms, the RK accumulator, x for
//   the stage updates) live in that thread's registers.  Shared memory only
//   carries the in-plane (x+-1, y+-1) exchange: two planes per level (x, u1,
//   u2, u3), each stage reading the plane its predecessor wrote in the
//   previous iteration -- so one __syncthreads per plane, no intra-plane
//   barriers.  Own points are 2x2 register blocks (inner neighbours from
//   registers; 6 shared loads per block per stage), halo-ring columns are
//   single points with up to three per thread.  HBM sees each x once and each
//   x' once: 16 B per state-update.
//
// Boundaries.  Interior tiles (halo-4 footprint inside the grid in x and y)
// run without per-point checks.  Insulated z faces use the centre value as
// the missing neighbour: the term (s - s) = +0.0 leaves the running sum
// exactly as skipping it does (the sum is never -0.0: it starts at +0.0 and
// round-to-nearest sums of nonzero terms are never -0).  Edge tiles use
// per-column face flags; exact mode then evaluates models.cpp:113-126
// literally (Robin term at ix = 0).
//
// Exact mode follows the reference's expression order (acc = 0.0; acc += ...
// x-, x+, y-, y+, z-, z+; k*acc; x + h2*k; acc + 2k as an exact FMA; x +
// h6*(acc + k3)).  Fast mode uses ghost values, one sum-then-subtract and
// constants folded with k.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace pirk {

constexpr int kHeatT = 32;                   // output tile edge (x and y)
constexpr int kHeatH = 4;                    // halo = number of RK stages
constexpr int kHeatP = kHeatT + 2 * kHeatH;  // 40: pitch of every plane buffer
constexpr int kHeatPlane = kHeatP * kHeatP;  // 1600
constexpr int kHeatThreads = 256;            // one 2x2 own block per thread
constexpr int kHeatRingSlots = 3;            // halo columns per thread (576 <= 3*256)
constexpr size_t kHeatSmemBytes = size_t(8) * kHeatPlane * sizeof(double);  // 102,400 B

struct HeatStepParams {
    double kk, robin;
    double h2kk, hkk, h6kk;  // fast-mode folded constants
};

// face flags (edge tiles)
enum : int { kXm = 1, kXp = 2, kYm = 4, kYp = 8, kIn = 16 };

__device__ __forceinline__ int face_flags(long long ix, long long iy, long long g) {
    int f = 0;
    if (ix >= 0 && ix < g && iy >= 0 && iy < g) f |= kIn;
    if (ix > 0) f |= kXm;
    if (ix + 1 < g) f |= kXp;
    if (iy > 0) f |= kYm;
    if (iy + 1 < g) f |= kYp;
    return f;
}

// Stencil value from the six neighbours.  Exact: k = kk*acc.  Fast: t = sum - 6 s.
template <bool Exact, bool Interior>
__device__ __forceinline__ double heat_pt(double s, double xm, double xp, double ym, double yp,
                                          double zm, double zp, int flags,
                                          const HeatStepParams& hp) {
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
        acc += zm - s;
        acc += zp - s;
        return hp.kk * acc;
    } else {
        if constexpr (!Interior) {
            xm = (flags & kXm) ? xm : fma(-hp.robin, s, xp);
            xp = (flags & kXp) ? xp : s;
            ym = (flags & kYm) ? ym : s;
            yp = (flags & kYp) ? yp : s;
        }
        const double sum = ((xm + xp) + (ym + yp)) + (zm + zp);
        return fma(-6.0, s, sum);
    }
}

// smem offset (in doubles) of level L's slot for plane parity `par`
__device__ __forceinline__ constexpr int lvl(int L, int par) { return (2 * L + par) * kHeatPlane; }

struct HeatCols {
    int ob;                   // own 2x2 block: smem offset of its top-left column
    int og[4];                // in-plane global offsets (iy*g + ix): (x,y), (x+1,y), (x,y+1), (x+1,y+1)
    int of[4];                // face flags
    int ro[kHeatRingSlots];   // halo-ring columns: smem offset (-1: none)
    int rg[kHeatRingSlots];
    int rf[kHeatRingSlots];
    int rd[kHeatRingSlots];   // number of stages computed at the column (0..3; -1: none)
};

template <bool Exact, bool Interior>
struct HeatRun {
    const HeatStepParams& hp;
    const StepConsts& sc;
    const HeatCols& c;
    double* __restrict__ S;   // shared memory
    int zs, ze, ob, oe, g, lo_shift, hi_shift;
    long long g2;
    const double* __restrict__ src;
    double* __restrict__ dst;
    int field, method;
    unsigned long long step;
    unsigned long long* fail;
    unsigned long long n_total;

    // register state: slot (p - zs) & 3 of plane p; prefetch by parity
    double ox[4][4], opre[4][2], ou1[4][4], ou2[4][4], ou3[4][4], oacc[4][4];
    double r0x[4], r0pre[2], r0u1[4], r0u2[4];   // ring slot 0 (depth <= 3)
    double r1x[4], r1pre[2], r1u1[4];            // ring slot 1 (depth <= 2)
    double r2pre[2];                              // ring slot 2 (depth 0: load only)

    __device__ __forceinline__ bool in(int k) const { return Interior || (c.of[k] & kIn); }

    __device__ __forceinline__ void load(int p, int par) {
        const double* plane = src + static_cast<long long>(p) * g2;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (in(k)) opre[k][par] = __ldg(plane + c.og[k]);
        if (c.rd[0] >= 0) r0pre[par] = __ldg(plane + c.rg[0]);
        if (c.rd[1] >= 0) r1pre[par] = __ldg(plane + c.rg[1]);
        if (c.rd[2] >= 0) r2pre[par] = __ldg(plane + c.rg[2]);
    }

    __device__ __forceinline__ void store_x(int par_slot, int par_pre) {
        double* X = S + lvl(0, par_slot);
        *reinterpret_cast<double2*>(X + c.ob) = make_double2(opre[0][par_pre], opre[1][par_pre]);
        *reinterpret_cast<double2*>(X + c.ob + kHeatP) = make_double2(opre[2][par_pre], opre[3][par_pre]);
        if (c.rd[0] >= 0) X[c.ro[0]] = r0pre[par_pre];
        if (c.rd[1] >= 0) X[c.ro[1]] = r1pre[par_pre];
        if (c.rd[2] >= 0) X[c.ro[2]] = r2pre[par_pre];
    }

    // Own 2x2 block at level L-1: centres ctr[4], z neighbours zm/zp[4],
    // in-plane neighbours from shared slot `in_off`.
    __device__ __forceinline__ void block_eval(const double* ctr, const double* zm, const double* zp,
                                               int in_off, double* kv) const {
        const double* B = S + in_off + c.ob;
        const double l0 = B[-1], l1 = B[kHeatP - 1];
        const double r0 = B[2], r1 = B[kHeatP + 2];
        const double2 up = *reinterpret_cast<const double2*>(B - kHeatP);
        const double2 dn = *reinterpret_cast<const double2*>(B + 2 * kHeatP);
        kv[0] = heat_pt<Exact, Interior>(ctr[0], l0, ctr[1], up.x, ctr[2], zm[0], zp[0], c.of[0], hp);
        kv[1] = heat_pt<Exact, Interior>(ctr[1], ctr[0], r0, up.y, ctr[3], zm[1], zp[1], c.of[1], hp);
        kv[2] = heat_pt<Exact, Interior>(ctr[2], l1, ctr[3], ctr[0], dn.x, zm[2], zp[2], c.of[2], hp);
        kv[3] = heat_pt<Exact, Interior>(ctr[3], ctr[2], r1, ctr[1], dn.y, zm[3], zp[3], c.of[3], hp);
    }

    __device__ __forceinline__ void block_store(int out_off, const double* v) const {
        double* B = S + out_off + c.ob;
        *reinterpret_cast<double2*>(B) = make_double2(v[0], v[1]);
        *reinterpret_cast<double2*>(B + kHeatP) = make_double2(v[2], v[3]);
    }

    __device__ __forceinline__ double ring_eval(int o, int f, double s, double zm, double zp,
                                                int in_off) const {
        const double* B = S + in_off + o;
        return heat_pt<Exact, Interior>(s, B[-1], B[1], B[-kHeatP], B[kHeatP], zm, zp, f, hp);
    }

    template <int PH>
    __device__ __forceinline__ void iteration(int j) {
        // register slots of planes j, j-1, j-2, j-3 (j-4 shares j's slot)
        constexpr int I0 = PH & 3, I1 = (PH + 3) & 3, I2 = (PH + 2) & 3, I3 = (PH + 1) & 3;
        constexpr int P0 = PH & 1, P1 = (PH + 1) & 1;  // parities of j and j-1
        const bool more = j + 1 < ze;
        if (more) load(j + 1, P1);      // x(j+1) -> prefetch[parity of j+1]
        if (j < ze) store_x(P0, P0);    // x(j) -> shared, read by stage 1 of iteration j+1

        // ---------------- stage 1 at plane p = j-1
        {
            const int p = j - 1;
            if (p >= zs + lo_shift && p < ze - hi_shift) {
                const bool hm = p > 0, hpz = p + 1 < g;
                double ctr[4], zm[4], zp[4], kv[4], u[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    ctr[k] = ox[k][I1];
                    zm[k] = hm ? ox[k][I2] : ctr[k];
                    zp[k] = hpz ? opre[k][P0] : ctr[k];
                }
                block_eval(ctr, zm, zp, lvl(0, P1), kv);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    u[k] = Exact ? ctr[k] + sc.h2 * kv[k] : fma(hp.h2kk, kv[k], ctr[k]);
                    ou1[k][I1] = u[k];
                    oacc[k][I1] = kv[k];
                }
                block_store(lvl(1, P1), u);
                if (c.rd[0] >= 1) {
                    const double s = r0x[I1];
                    const double kr = ring_eval(c.ro[0], c.rf[0], s, hm ? r0x[I2] : s, hpz ? r0pre[P0] : s, lvl(0, P1));
                    const double uu = Exact ? s + sc.h2 * kr : fma(hp.h2kk, kr, s);
                    r0u1[I1] = uu;
                    S[lvl(1, P1) + c.ro[0]] = uu;
                }
                if (c.rd[1] >= 1) {
                    const double s = r1x[I1];
                    const double kr = ring_eval(c.ro[1], c.rf[1], s, hm ? r1x[I2] : s, hpz ? r1pre[P0] : s, lvl(0, P1));
                    const double uu = Exact ? s + sc.h2 * kr : fma(hp.h2kk, kr, s);
                    r1u1[I1] = uu;
                    S[lvl(1, P1) + c.ro[1]] = uu;
                }
            }
        }
        // ---------------- stage 2 at plane p = j-2
        {
            const int p = j - 2;
            if (p >= zs + 2 * lo_shift && p < ze - 2 * hi_shift) {
                const bool hm = p > 0, hpz = p + 1 < g;
                double ctr[4], zm[4], zp[4], kv[4], u[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    ctr[k] = ou1[k][I2];
                    zm[k] = hm ? ou1[k][I3] : ctr[k];
                    zp[k] = hpz ? ou1[k][I1] : ctr[k];
                }
                block_eval(ctr, zm, zp, lvl(1, P0), kv);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double x = ox[k][I2];
                    u[k] = Exact ? x + sc.h2 * kv[k] : fma(hp.h2kk, kv[k], x);
                    ou2[k][I2] = u[k];
                    oacc[k][I2] = fma(2.0, kv[k], oacc[k][I2]);  // acc + 2k (exact: 2k is exact)
                }
                block_store(lvl(2, P0), u);
                if (c.rd[0] >= 2) {
                    const double s = r0u1[I2];
                    const double kr = ring_eval(c.ro[0], c.rf[0], s, hm ? r0u1[I3] : s, hpz ? r0u1[I1] : s, lvl(1, P0));
                    const double x = r0x[I2];
                    const double uu = Exact ? x + sc.h2 * kr : fma(hp.h2kk, kr, x);
                    r0u2[I2] = uu;
                    S[lvl(2, P0) + c.ro[0]] = uu;
                }
                if (c.rd[1] >= 2) {
                    const double s = r1u1[I2];
                    const double kr = ring_eval(c.ro[1], c.rf[1], s, hm ? r1u1[I3] : s, hpz ? r1u1[I1] : s, lvl(1, P0));
                    const double x = r1x[I2];
                    const double uu = Exact ? x + sc.h2 * kr : fma(hp.h2kk, kr, x);
                    S[lvl(2, P0) + c.ro[1]] = uu;
                }
            }
        }
        // ---------------- stage 3 at plane p = j-3
        {
            const int p = j - 3;
            if (p >= zs + 3 * lo_shift && p < ze - 3 * hi_shift) {
                const bool hm = p > 0, hpz = p + 1 < g;
                double ctr[4], zm[4], zp[4], kv[4], u[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    ctr[k] = ou2[k][I3];
                    zm[k] = hm ? ou2[k][I0] : ctr[k];   // plane j-4 shares slot I0
                    zp[k] = hpz ? ou2[k][I2] : ctr[k];
                }
                block_eval(ctr, zm, zp, lvl(2, P1), kv);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double x = ox[k][I3];
                    u[k] = Exact ? x + sc.hk * kv[k] : fma(hp.hkk, kv[k], x);
                    ou3[k][I3] = u[k];
                    oacc[k][I3] = fma(2.0, kv[k], oacc[k][I3]);
                }
                block_store(lvl(3, P1), u);
                if (c.rd[0] >= 3) {
                    const double s = r0u2[I3];
                    const double kr = ring_eval(c.ro[0], c.rf[0], s, hm ? r0u2[I0] : s, hpz ? r0u2[I2] : s, lvl(2, P1));
                    const double x = r0x[I3];
                    const double uu = Exact ? x + sc.hk * kr : fma(hp.hkk, kr, x);
                    S[lvl(3, P1) + c.ro[0]] = uu;
                }
            }
        }
        // ---------------- stage 4 at plane p = j-4 (own block), stored to HBM
        {
            const int p = j - 4;
            if (p >= ob && p < oe) {
                const bool hm = p > 0, hpz = p + 1 < g;
                double ctr[4], zm[4], zp[4], kv[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    ctr[k] = ou3[k][I0];
                    zm[k] = hm ? ou3[k][I1] : ctr[k];   // plane j-5 shares slot I1
                    zp[k] = hpz ? ou3[k][I3] : ctr[k];
                }
                block_eval(ctr, zm, zp, lvl(3, P0), kv);
                double* out = dst + static_cast<long long>(p) * g2;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (!in(k)) continue;
                    const double x = ox[k][I0];
                    const double xn = Exact ? x + sc.h6 * (oacc[k][I0] + kv[k])
                                            : fma(hp.h6kk, oacc[k][I0] + kv[k], x);
                    out[c.og[k]] = xn;
                    if (!finite_d(xn)) {
                        const unsigned long long gi = static_cast<unsigned long long>(
                            static_cast<long long>(p) * g2 + c.og[k]);
                        if (method == 0)
                            record_fail(fail, step, gi + (field ? n_total : 0ull));
                        else if (fail)
                            record_fail(fail + field, step, gi);
                    }
                }
            }
        }
        // x(j) moves from the prefetch register into the history slot of x(j-4)
#pragma unroll
        for (int k = 0; k < 4; ++k) ox[k][I0] = opre[k][P0];
        r0x[I0] = r0pre[P0];
        r1x[I0] = r1pre[P0];
        __syncthreads();
    }

    __device__ __forceinline__ void run() {
        if (zs < ze) load(zs, 0);
        const int jend = ze + kHeatH;
        for (int j = zs; j < jend; j += 4) {
            iteration<0>(j);
            if (j + 1 < jend) iteration<1>(j + 1);
            if (j + 2 < jend) iteration<2>(j + 2);
            if (j + 3 < jend) iteration<3>(j + 3);
        }
    }
};

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
    const long long obz = static_cast<long long>(w.out_begin) + chunk * static_cast<long long>(zchunk);
    long long oez = obz + static_cast<long long>(zchunk);
    if (oez > static_cast<long long>(w.out_end)) oez = static_cast<long long>(w.out_end);
    if (obz >= oez) return;

    // ---- static column assignment
    HeatCols c;
    {
        const int bx = tid & 15, by = tid >> 4;
        c.ob = (2 * by + kHeatH) * kHeatP + (2 * bx + kHeatH);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const long long ix = ix0 + 2 * bx + (k & 1), iy = iy0 + 2 * by + (k >> 1);
            c.of[k] = face_flags(ix, iy, g);
            c.og[k] = (c.of[k] & kIn) ? static_cast<int>(iy * g + ix) : 0;
        }
        // halo-ring columns ordered by distance d = 1..4 from the tile
        // (a column at distance d is computed at stages 1 .. 4-d)
#pragma unroll
        for (int s = 0; s < kHeatRingSlots; ++s) {
            int r = tid + s * kHeatThreads;
            c.ro[s] = 0;
            c.rg[s] = 0;
            c.rf[s] = 0;
            c.rd[s] = -1;
            for (int d = 1; d <= kHeatH; ++d) {
                const int side = kHeatT + 2 * d, cnt = 4 * side - 4;
                if (r < cnt) {
                    const int lo = kHeatH - d;  // region coordinate of the band's first row/col
                    int x, y;
                    if (r < side) { y = lo; x = lo + r; }
                    else if (r < 2 * side) { y = lo + side - 1; x = lo + (r - side); }
                    else if (r < 3 * side - 2) { x = lo; y = lo + 1 + (r - 2 * side); }
                    else { x = lo + side - 1; y = lo + 1 + (r - (3 * side - 2)); }
                    const long long ix = ix0 - kHeatH + x, iy = iy0 - kHeatH + y;
                    c.ro[s] = y * kHeatP + x;
                    c.rf[s] = face_flags(ix, iy, g);
                    if (c.rf[s] & kIn) {
                        c.rg[s] = static_cast<int>(iy * g + ix);
                        c.rd[s] = kHeatH - d;
                    }
                    break;
                }
                r -= cnt;
            }
        }
    }
    const bool interior = ix0 - kHeatH >= 0 && ix0 + kHeatT + kHeatH <= g && iy0 - kHeatH >= 0 &&
                          iy0 + kHeatT + kHeatH <= g;
    const long long g2 = g * g;
    const int zs = static_cast<int>((obz - kHeatH > 0) ? obz - kHeatH : 0);
    const int ze = static_cast<int>((oez + kHeatH < g) ? oez + kHeatH : g);
    const double* src = (field ? w.in1 : w.in0) - static_cast<long long>(w.win_begin) * g2;
    double* dst = (field ? w.out1 : w.out0) - static_cast<long long>(w.out_begin) * g2;
    const unsigned long long n_total = static_cast<unsigned long long>(g2 * g);
    if (interior) {
        HeatRun<Exact, true> r{hp, sc, c, smem, zs, ze, static_cast<int>(obz), static_cast<int>(oez),
                               static_cast<int>(g), zs > 0, ze < g, g2, src, dst, field, m.method,
                               step, fail, n_total};
        r.run();
    } else {
        HeatRun<Exact, false> r{hp, sc, c, smem, zs, ze, static_cast<int>(obz), static_cast<int>(oez),
                                static_cast<int>(g), zs > 0, ze < g, g2, src, dst, field, m.method,
                                step, fail, n_total};
        r.run();
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
