// heat.cuh -- K2: fused 4-stage RK4 step of the heat3d 7-point stencil.
//
// Replaces integrate_step (rk4.cpp:30-76) on the embedding of heat3d
// (models.cpp:92-133; cooperative, so the lower and upper fields evolve
// independently and each is the plain stencil) and on the growth-bound pair
// (growth_rhs == rhs for heat3d, models.cpp:130).
//
// Design: 2.5-D z-streaming with register-resident z histories.
//   A CTA (one per SM: 185 KB of shared memory) owns a 32x32 x-y tile of one
//   field and streams the planes of a z-chunk.  Iteration j waits for x-plane
//   j (tile + halo 4, a 42x40 TMA box with out-of-grid cells zero-filled,
//   completing on an mbarrier), issues the TMA load of plane j+3 into an
//   8-slot ring, and evaluates stage 1 at plane j-1, stage 2 at j-2, stage 3
//   at j-3 and stage 4 (the RK4 combination, stored to HBM) at j-4.  Every
//   (x, y) column of the 40x40 footprint belongs to one thread for the whole
//   run, so a column's values at neighbouring planes (the z+-1 terms) stay in
//   that thread's registers; its RK accumulators live in TMEM (tcgen05.st/ld,
//   one 32-lane quadrant per warp), which keeps the kernel spill-free.
//   Shared memory carries only the in-plane (x+-1, y+-1) exchange: u1/u2/u3
//   planes double-buffered, each stage reading the plane its predecessor
//   wrote in the previous iteration -- one __syncthreads per plane.  u rows
//   have an odd pitch (41 doubles) with even and odd columns de-interleaved,
//   so row-wise and column-wise neighbour loads of a warp are bank-conflict
//   free; x planes are row-major (pitch 42, the TMA box).  Own points are 1x2
//   register pairs (the pair's inner neighbours come from registers); the 576
//   halo-ring columns are single points (one or two per thread), grouped by
//   depth so that ring stages branch per warp, not per lane.  HBM sees each x
//   once and each x' once: 16 B per state-update (plus halo re-reads that
//   miss L2; profiles/heat_traffic.json).  heat2x2.cuh is the 2x2-block
//   variant of this kernel (the fast-mode default).
//
// Boundaries.  Interior tiles (halo-4 footprint inside the grid in x and y)
// run without per-point checks.  Insulated z faces: the history slot of the
// missing plane (-1 or g) holds the boundary plane's value, so the term
// (s - s) = +0.0 leaves the running sum exactly as skipping it does (the sum
// is never -0.0: it starts at +0.0 and round-to-nearest sums of nonzero terms
// are never -0); these iterations are peeled off the main loop.  Edge tiles
// use per-column face flags; exact mode then evaluates models.cpp:113-126
// literally (Robin term at ix = 0).
//
// Exact mode follows the reference's expression order (acc = 0.0; acc += ...
// x-, x+, y-, y+, z-, z+; k*acc; x + h2*k; acc + 2k as an exact FMA; x +
// h6*(acc + k3)).  Fast mode uses ghost values, one sum-then-subtract and
// constants folded with k.
#pragma once

#include <cuda.h>  // CUtensorMap (encoded through cudaGetDriverEntryPoint)

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace pirk {

constexpr int kHeatT = 32;                   // output tile edge (x and y)
constexpr int kHeatH = 4;                    // halo = number of RK stages
constexpr int kHeatW = kHeatT + 2 * kHeatH;  // 40: footprint edge
constexpr int kHeatHalf = kHeatW / 2;        // 20: even / odd column sub-rows
constexpr int kHeatP = kHeatW + 1;           // 41: odd row pitch (bank-conflict free)
constexpr int kHeatPlane = kHeatW * kHeatP;  // 1640
constexpr int kHeatThreads = 512;            // one 1x2 own pair per thread
constexpr int kHeatXRing = 8;                // x planes j-7 .. j (slot (p - zs) & 7)
// x planes are row-major with pitch 42 (the TMA box is 42 x 40: rows stay 16-byte
// aligned as TMA requires, and 42 doubles = 20 banks mod 32 keeps column-wise
// halo reads at most 2-way conflicted); slot = 1680 doubles = 105 x 128 B
constexpr int kHeatXP = 42;
constexpr int kHeatXSlot = kHeatXP * kHeatW;
constexpr size_t kHeatSmemBytes =
    size_t(kHeatXRing) * kHeatXSlot * sizeof(double) + size_t(6) * kHeatPlane * sizeof(double);  // 185,216 B

struct HeatStepParams {
    double kk, robin;
    double h2kk, hkk, h6kk;  // fast-mode folded constants
    // fast-mode Horner coefficients hk*kk/4, /3, /2, /1 (heat2x2.cuh): for a
    // linear autonomous field RK4 is x + hL(x + hL/2(x + hL/3(x + hL/4 x)))
    double hn[4];
    // fast-mode strip kernel (heat_strip.cuh PIRK_STRIP_SFORM): RK4 of the
    // linear field as a polynomial in the neighbour-sum operator S (L = S - 6),
    // P(z(S - 6)) = q0 + q1 S + .. + q4 S^4, z = hk*kk, evaluated as
    // w1 = S x + sf[0] x, w2 = S w1 + sf[1] x, w3 = S w2 + sf[2] x,
    // y = sf[3] S w3 + sf[4] x  (sf = q3/q4, q2/q4, q1/q4, q4, q0)
    double sf[5];
};

// S-form coefficients for z = hk*kk (host).  Returns false when z is outside
// the range the strip kernel's S form is used for: its stage values grow like
// |w3| ~ 24/z^3 |x|, so tiny z (the remainder step of a plan, very small h)
// runs the Horner-in-L kernels instead.
inline bool heat_sform_coeffs(double z, double* sf) {
    if (!(z >= 1e-6) || !(z < 1e6)) return false;
    const long double Z = z, Z2 = Z * Z, Z3 = Z2 * Z, Z4 = Z3 * Z;
    const long double q4 = Z4 / 24.0L;
    const long double q3 = Z3 * (1.0L - 6.0L * Z) / 6.0L;
    const long double q2 = Z2 * (1.0L - 6.0L * Z + 18.0L * Z2) / 2.0L;
    const long double q1 = Z * (1.0L - 6.0L * Z + 18.0L * Z2 - 36.0L * Z3);
    const long double q0 = 1.0L - 6.0L * Z + 18.0L * Z2 - 36.0L * Z3 + 54.0L * Z4;
    if (sf) {
        sf[0] = static_cast<double>(q3 / q4);
        sf[1] = static_cast<double>(q2 / q4);
        sf[2] = static_cast<double>(q1 / q4);
        sf[3] = static_cast<double>(q4);
        sf[4] = static_cast<double>(q0);
    }
    return true;
}

// face flags (edge tiles); kOdd marks an odd footprint column (neighbour offsets)
enum : int { kXm = 1, kXp = 2, kYm = 4, kYp = 8, kIn = 16, kOdd = 32 };

__device__ __forceinline__ int face_flags(long long ix, long long iy, long long g) {
    int f = 0;
    if (ix >= 0 && ix < g && iy >= 0 && iy < g) f |= kIn;
    if (ix > 0) f |= kXm;
    if (ix + 1 < g) f |= kXp;
    if (iy > 0) f |= kYm;
    if (iy + 1 < g) f |= kYp;
    return f;
}

// shared index of footprint column (x, y)
__device__ __forceinline__ int heat_sidx(int x, int y) {
    return y * kHeatP + (x & 1) * kHeatHalf + (x >> 1);
}

// buffer bases: x ring slot s (0..7, row-major); level L (1..3) parity par (de-interleaved)
__device__ __forceinline__ constexpr int xbuf(int s) { return s * kHeatXSlot; }
__device__ __forceinline__ constexpr int ubuf(int L, int par) {
    return kHeatXRing * kHeatXSlot + (2 * (L - 1) + par) * kHeatPlane;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// TMA: one 40x40 x-plane box per iteration, completing on an mbarrier.
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
#ifndef PIRK_MBAR_HINT
#define PIRK_MBAR_HINT 0  // try_wait suspend-time hint in ns (0: none)
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
#if PIRK_MBAR_HINT > 0
    // a waiting warp sleeps in try_wait instead of spinning on issue slots
    asm volatile(
        "{\n .reg .pred p;\nPIRK_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra PIRK_WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity), "n"(PIRK_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n .reg .pred p;\nPIRK_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra PIRK_WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
#endif
}
__device__ __forceinline__ void tma_load_plane(double* dst, const void* tmap, int x, int y, int z,
                                               unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// L2 prefetch of the same box (no shared-memory destination, no completion)
__device__ __forceinline__ void tma_prefetch_l2(const void* tmap, int x, int y, int z) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];\n" ::"l"(tmap), "r"(x), "r"(y),
                 "r"(z)
                 : "memory");
}

// TMEM as per-thread pipeline storage: each warp owns a 32-lane quadrant
// (warp % 4) and a 128-column slice (warp / 4) of the CTA's 512 columns; a
// thread keeps its two RK accumulators per plane in flight there (4 planes x
// 2 doubles = 16 columns), freeing registers for the stencil pipeline.
__device__ __forceinline__ void tmem_alloc512(unsigned* dst) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(dst))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc512(unsigned taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// No "memory" clobbers: TMEM is not compiler-visible memory, and volatile asm
// statements keep their relative order (st before a later ld of the slot), so
// shared-memory loads remain free to be scheduled across these.
__device__ __forceinline__ void tmem_st2(unsigned taddr, double a, double b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr),
                 "r"(__double2loint(a)), "r"(__double2hiint(a)), "r"(__double2loint(b)),
                 "r"(__double2hiint(b)));
}
__device__ __forceinline__ void tmem_ld2(unsigned taddr, double& a, double& b) {
    unsigned r0, r1, r2, r3;
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3));
    a = __hiloint2double(static_cast<int>(r1), static_cast<int>(r0));
    b = __hiloint2double(static_cast<int>(r3), static_cast<int>(r2));
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

struct HeatCols {
    int xe;        // row-major x-ring index of the pair's even column (odd: xe + 1)
    int xr[2];     // row-major x-ring index of the halo-ring columns
    int oe;        // shared index of the pair's even column (the odd one is oe + 20)
    int og;        // in-plane global offset of the even column (odd: og + 1)
    int of[2];     // face flags of the two own columns
    int ro[2];     // halo-ring columns: shared index
    int rg[2];     // in-plane global offset
    int rf[2];     // face flags (| kOdd)
    int rd[2];     // number of stages computed at the column (0..3; -1: none)
    // Warp-uniform max of rd[0]: ring stage L runs in every lane of a warp that
    // has any lane needing it.  A lane computing a level beyond its column's
    // depth only writes shared cells (and its own registers) that no stage
    // reads: a level-L value at distance d > 4-L is never a neighbour of a
    // level-(L+1) evaluation (those sit at distance <= 3-L).
    int wd;
};

template <bool Exact, bool Interior, bool Tma, bool Mirror = false>
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
    // TMA: tensor map of this field's window, box origin (x, y), window start plane, barriers
    const void* tmap;
    int bx0, by0, wbz;
    unsigned long long* bars;
    double* mdst;  // Mirror: the low neighbour's halo planes (WindowArgs::mir0/1), indexed like dst
    double* mhdst;  // Mirror: the high neighbour's (WindowArgs::mirh0/1)
    int m_lo_end, m_hi_begin;  // planes < m_lo_end go to mdst, planes >= m_hi_begin to mhdst

    // register state: slot (p - zs) & 3 of plane p
    double ox[2][4], ou1[2][4], ou2[2][4], ou3[2][4];
    unsigned tacc;   // TMEM address of this thread's accumulator slots (4 columns per plane slot)

    __device__ __forceinline__ void acc_st(int slot, double a, double b) const {
        tmem_st2(tacc + 4 * slot, a, b);
    }
    __device__ __forceinline__ void acc_ld(int slot, double& a, double& b) const {
        tmem_ld2(tacc + 4 * slot, a, b);
    }
    double rx[4], ru1[4], ru2[4];   // ring slot 0 (depth <= 3)

    __device__ __forceinline__ bool in(int k) const { return Interior || (c.of[k] & kIn); }

    // running plane pointers: x-plane j+1 (loads) and output plane j-4 (stores)
    const double* ldp;
    double* stp;
    double* mtp;  // Mirror: stp in the low neighbour's window
    double* mhp;  // Mirror: stp in the high neighbour's window

    // x-plane p -> x-ring slot s.  TMA: one thread issues the whole 40x40 box
    // (out-of-grid cells zero-filled), completion on bars[s].  Fallback: each
    // thread cp.asyncs its own columns (completed by cp_async_wait_all).
    __device__ __forceinline__ void load(const double* plane, int p, int s) {
        double* X = S + xbuf(s);
        if constexpr (Tma) {
            if (threadIdx.x == 0) {
                mbar_expect_tx(bars + s, kHeatXSlot * sizeof(double));
                tma_load_plane(X, tmap, bx0, by0, p - wbz, bars + s);
            }
        } else {
            if (in(0)) cp_async8(X + c.xe, plane + c.og);
            if (in(1)) cp_async8(X + c.xe + 1, plane + c.og + 1);
            if (c.rd[0] >= 0) cp_async8(X + c.xr[0], plane + c.rg[0]);
            if (c.rd[1] >= 0) cp_async8(X + c.xr[1], plane + c.rg[1]);
            cp_async_commit();
        }
    }

    // stage 1 reads the row-major x plane
    __device__ __forceinline__ void pair_eval_x(double c0, double c1, double zm0, double zm1,
                                                double zp0, double zp1, int x_off, double& k0,
                                                double& k1) const {
        const double* B = S + x_off + c.xe;
        const double l = B[-1], r = B[2];
        const double2 u = *reinterpret_cast<const double2*>(B - kHeatXP);  // xe is even: aligned
        const double2 d = *reinterpret_cast<const double2*>(B + kHeatXP);
        k0 = heat_pt<Exact, Interior>(c0, l, c1, u.x, d.x, zm0, zp0, c.of[0], hp);
        k1 = heat_pt<Exact, Interior>(c1, c0, r, u.y, d.y, zm1, zp1, c.of[1], hp);
    }

    __device__ __forceinline__ double ring_eval_x(double s, double zm, double zp, int x_off) const {
        const double* B = S + x_off + c.xr[0];
        return heat_pt<Exact, Interior>(s, B[-1], B[1], B[-kHeatXP], B[kHeatXP], zm, zp, c.rf[0], hp);
    }

    __device__ __forceinline__ double2 own_x(int x_off) const {
        return *reinterpret_cast<const double2*>(S + x_off + c.xe);
    }

    // own pair: centres c0 (even col) and c1 (odd col) at level L-1 of plane p,
    // z neighbours, in-plane neighbours from the shared buffer at `in_off`
    __device__ __forceinline__ void pair_eval(double c0, double c1, double zm0, double zm1,
                                              double zp0, double zp1, int in_off, double& k0,
                                              double& k1) const {
        const double* B = S + in_off;
        const int e = c.oe, o = c.oe + kHeatHalf;
        const double l = B[o - 1];            // (X0-1, Y): odd column of the previous pair
        const double r = B[e + 1];            // (X0+2, Y): even column of the next pair
        const double u0 = B[e - kHeatP], u1 = B[o - kHeatP];
        const double d0 = B[e + kHeatP], d1 = B[o + kHeatP];
        k0 = heat_pt<Exact, Interior>(c0, l, c1, u0, d0, zm0, zp0, c.of[0], hp);
        k1 = heat_pt<Exact, Interior>(c1, c0, r, u1, d1, zm1, zp1, c.of[1], hp);
    }

    __device__ __forceinline__ double ring_eval(double s, double zm, double zp, int in_off) const {
        const double* B = S + in_off + c.ro[0];
        const int dm = (c.rf[0] & kOdd) ? -kHeatHalf : kHeatHalf - 1;  // offset of x-1
        const double xm = B[dm], xp = B[dm + 1];                      // x+1 is the next slot
        return heat_pt<Exact, Interior>(s, xm, xp, B[-kHeatP], B[kHeatP], zm, zp, c.rf[0], hp);
    }

    __device__ __forceinline__ double upd(double x, double k, double ce, double cf) const {
        return Exact ? x + ce * k : fma(cf, k, x);
    }

    // ZEdge: the iteration touches an insulated z face (planes -1 or g)
    template <int PH, bool ZEdge>
    __device__ __forceinline__ void iteration(int j) {
        // register/x-ring slots of planes j, j-1, j-2, j-3 (j-4 shares j's, j-5 shares j-1's)
        constexpr int I0 = PH & 3, I1 = (PH + 3) & 3, I2 = (PH + 2) & 3, I3 = (PH + 1) & 3;
        constexpr int P0 = PH & 1, P1 = (PH + 1) & 1;  // parities of j and j-1
        const int x8 = (j - zs) & 7;                   // x-ring slot of plane j
        const int X0 = xbuf(x8), X1 = xbuf((x8 + 7) & 7), X3 = xbuf((x8 + 5) & 7),
                  X4 = xbuf((x8 + 4) & 7);
        if constexpr (Tma) {
            // three planes of prefetch: x(j+3) into the slot of x(j-5), last read
            // (stage 4) in iteration j-1; issued before waiting for x(j)
            if (j + 3 < ze) load(nullptr, j + 3, (x8 + 3) & 7);
            if (j < ze) mbar_wait(bars + x8, ((j - zs) >> 3) & 1);  // x(j) landed
        } else {
            if (j + 1 < ze) load(ldp, j + 1, (x8 + 1) & 7);  // x(j+1) into the slot of x(j-7)
        }
        // own x(j): the z+ neighbour of stage 1
        const double2 xj = own_x(X0);
        double xj0 = xj.x, xj1 = xj.y;
        double rxj = S[X0 + c.xr[0]];
        if (ZEdge && j == g) {  // insulated top face: x(g) := x(g-1)
            xj0 = ox[0][I1];
            xj1 = ox[1][I1];
            rxj = rx[I1];
        }

        // ---------------- stage 1 at plane p = j-1
        {
            const int p = j - 1;
            if (!ZEdge || (p >= zs + lo_shift && p < ze - hi_shift)) {
                double k0, k1;
                pair_eval_x(ox[0][I1], ox[1][I1], ox[0][I2], ox[1][I2], xj0, xj1, X1, k0, k1);
                const double u0 = upd(ox[0][I1], k0, sc.h2, hp.h2kk);
                const double u1 = upd(ox[1][I1], k1, sc.h2, hp.h2kk);
                ou1[0][I1] = u0;
                ou1[1][I1] = u1;
                acc_st(I1, k0, k1);
                S[ubuf(1, P1) + c.oe] = u0;
                S[ubuf(1, P1) + c.oe + kHeatHalf] = u1;
                if (ZEdge && p == 0) {  // insulated bottom face: u1(-1) := u1(0)
                    ou1[0][I2] = u0;
                    ou1[1][I2] = u1;
                }
                if (c.wd >= 1) {
                    const double s = rx[I1];
                    const double kr = ring_eval_x(s, rx[I2], rxj, X1);
                    const double uu = upd(s, kr, sc.h2, hp.h2kk);
                    ru1[I1] = uu;
                    S[ubuf(1, P1) + c.ro[0]] = uu;
                    if (ZEdge && p == 0) ru1[I2] = uu;
                }
            } else if (ZEdge && p == g) {  // top face: u1(g) := u1(g-1)
                ou1[0][I1] = ou1[0][I2];
                ou1[1][I1] = ou1[1][I2];
                ru1[I1] = ru1[I2];
            }
        }
        // ---------------- stage 2 at plane p = j-2
        {
            const int p = j - 2;
            if (!ZEdge || (p >= zs + 2 * lo_shift && p < ze - 2 * hi_shift)) {
                double k0, k1;
                pair_eval(ou1[0][I2], ou1[1][I2], ou1[0][I3], ou1[1][I3], ou1[0][I1], ou1[1][I1],
                          ubuf(1, P0), k0, k1);
                const double u0 = upd(ox[0][I2], k0, sc.h2, hp.h2kk);
                const double u1 = upd(ox[1][I2], k1, sc.h2, hp.h2kk);
                ou2[0][I2] = u0;
                ou2[1][I2] = u1;
                double a0, a1;
                acc_ld(I2, a0, a1);
                acc_st(I2, fma(2.0, k0, a0), fma(2.0, k1, a1));  // acc + 2k (exact: 2k is exact)
                S[ubuf(2, P0) + c.oe] = u0;
                S[ubuf(2, P0) + c.oe + kHeatHalf] = u1;
                if (ZEdge && p == 0) {
                    ou2[0][I3] = u0;
                    ou2[1][I3] = u1;
                }
                if (c.wd >= 2) {
                    const double s = ru1[I2];
                    const double kr = ring_eval(s, ru1[I3], ru1[I1], ubuf(1, P0));
                    const double uu = upd(rx[I2], kr, sc.h2, hp.h2kk);
                    ru2[I2] = uu;
                    S[ubuf(2, P0) + c.ro[0]] = uu;
                    if (ZEdge && p == 0) ru2[I3] = uu;
                }
            } else if (ZEdge && p == g) {
                ou2[0][I2] = ou2[0][I3];
                ou2[1][I2] = ou2[1][I3];
                ru2[I2] = ru2[I3];
            }
        }
        // ---------------- stage 3 at plane p = j-3
        {
            const int p = j - 3;
            if (!ZEdge || (p >= zs + 3 * lo_shift && p < ze - 3 * hi_shift)) {
                double k0, k1;
                pair_eval(ou2[0][I3], ou2[1][I3], ou2[0][I0], ou2[1][I0], ou2[0][I2], ou2[1][I2],
                          ubuf(2, P1), k0, k1);
                // x(j-3) from the shared x ring (keeps the register budget at 128)
                const double2 x3 = own_x(X3);
                const double u0 = upd(x3.x, k0, sc.hk, hp.hkk);
                const double u1 = upd(x3.y, k1, sc.hk, hp.hkk);
                ou3[0][I3] = u0;
                ou3[1][I3] = u1;
                double a0, a1;
                acc_ld(I3, a0, a1);
                acc_st(I3, fma(2.0, k0, a0), fma(2.0, k1, a1));
                S[ubuf(3, P1) + c.oe] = u0;
                S[ubuf(3, P1) + c.oe + kHeatHalf] = u1;
                if (ZEdge && p == 0) {
                    ou3[0][I0] = u0;
                    ou3[1][I0] = u1;
                }
                if (c.wd >= 3) {
                    const double s = ru2[I3];
                    const double kr = ring_eval(s, ru2[I0], ru2[I2], ubuf(2, P1));
                    S[ubuf(3, P1) + c.ro[0]] = upd(S[X3 + c.xr[0]], kr, sc.hk, hp.hkk);
                }
            } else if (ZEdge && p == g) {
                ou3[0][I3] = ou3[0][I0];
                ou3[1][I3] = ou3[1][I0];
            }
        }
        // ---------------- stage 4 at plane p = j-4 (own pair), stored to HBM
        {
            const int p = j - 4;
            if (!ZEdge || (p >= ob && p < oe)) {
                double k0, k1;
                pair_eval(ou3[0][I0], ou3[1][I0], ou3[0][I1], ou3[1][I1], ou3[0][I3], ou3[1][I3],
                          ubuf(3, P0), k0, k1);
                double* out = stp;
                const double kk[2] = {k0, k1};
                const double2 x4 = own_x(X4);  // x(j-4)
                const double xs[2] = {x4.x, x4.y};
                double xn[2], acc[2];
                acc_ld(I0, acc[0], acc[1]);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    xn[k] = Exact ? xs[k] + sc.h6 * (acc[k] + kk[k])
                                  : fma(hp.h6kk, acc[k] + kk[k], xs[k]);
                    if (in(k)) {
                        out[c.og + k] = xn[k];
                        if constexpr (Mirror) {
                            if (p < m_lo_end) mtp[c.og + k] = xn[k];
                            if (p >= m_hi_begin) mhp[c.og + k] = xn[k];
                        }
                    }
                }
                // one test per pair: the sum is non-finite whenever either value
                // is (a finite overflow only sends the pair to the exact check)
                if (!finite_d(xn[0] + xn[1])) {
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        if (!in(k) || finite_d(xn[k])) continue;
                        const unsigned long long gi = static_cast<unsigned long long>(
                            static_cast<long long>(p) * g2 + c.og + k);
                        if (method == 0)
                            record_fail(fail, step, gi + (field ? n_total : 0ull));
                        else if (fail)
                            record_fail(fail + field, step, gi);
                    }
                }
            }
        }
        // x(j) joins the history in the slot of x(j-4)
        ox[0][I0] = xj0;
        ox[1][I0] = xj1;
        rx[I0] = rxj;
        if (ZEdge && j == 0) {  // insulated bottom face: x(-1) := x(0)
            ox[0][I1] = xj0;
            ox[1][I1] = xj1;
            rx[I1] = rxj;
        }
        ldp += g2;
        stp += g2;
        if constexpr (Mirror) {
            mtp += g2;
            mhp += g2;
        }
        if constexpr (!Tma) cp_async_wait_all();  // x(j+1) landed (own copies); barrier publishes it
        __syncthreads();
    }

    template <bool ZEdge>
    __device__ __forceinline__ void one(int j) {
        switch ((j - zs) & 3) {
            case 0: iteration<0, ZEdge>(j); break;
            case 1: iteration<1, ZEdge>(j); break;
            case 2: iteration<2, ZEdge>(j); break;
            default: iteration<3, ZEdge>(j); break;
        }
    }

    __device__ __forceinline__ void run() {
        if (zs < ze) {
            load(src + static_cast<long long>(zs) * g2, zs, 0);  // x(zs) -> slot 0
            if constexpr (Tma) {
                if (zs + 1 < ze) load(nullptr, zs + 1, 1);       // x(zs+1) -> slot 1
                if (zs + 2 < ze) load(nullptr, zs + 2, 2);       // x(zs+2) -> slot 2
            }
            if constexpr (!Tma) cp_async_wait_all();
        }
        __syncthreads();
        ldp = src + static_cast<long long>(zs + 1) * g2;
        stp = dst + static_cast<long long>(zs - 4) * g2;
        if constexpr (Mirror) {
            mtp = mdst + static_cast<long long>(zs - 4) * g2;
            mhp = mhdst + static_cast<long long>(zs - 4) * g2;
        }
        const int jend = ze + kHeatH;
        // Steady-state iterations: all four stages valid and planes j-5 .. j
        // clear of the insulated z faces, so the unrolled main loop carries no
        // validity or boundary branches.
        int a = zs + 3 + 3 * lo_shift;
        if (a < ob + 4) a = ob + 4;
        if (a < 5) a = 5;
        a = zs + ((a - zs + 3) & ~3);          // keep (j - zs) % 4 == 0 at the main loop start
        int b = ze + 1 - hi_shift;
        if (b > oe + 4) b = oe + 4;
        if (b > g) b = g;
        if (b < a) b = a;
        const int main_end = a + ((b - a) & ~3);
        int j = zs;
        for (; j < a && j < jend; ++j) one<true>(j);
        for (; j < main_end; j += 4) {
            iteration<0, false>(j);
            iteration<1, false>(j + 1);
            iteration<2, false>(j + 2);
            iteration<3, false>(j + 3);
        }
        for (; j < jend; ++j) one<true>(j);
    }
};

// Tensor maps of the two fields' windows (used when `tma` is set): a
// 3-D (x, y, plane) fp64 view with a 40x40x1 box.
struct HeatTmaps {
    CUtensorMap f[2];
};

template <bool Exact, bool Mirror = false>
__global__ void __launch_bounds__(kHeatThreads, 1)
heat_step_kernel(const HeatModel m, const HeatStepParams hp, const WindowArgs w,
                 const StepConsts sc, const unsigned long long step, const uint64_t zchunk,
                 unsigned long long* __restrict__ fail, const __grid_constant__ HeatTmaps tm,
                 const int tma) {
    (void)sizeof(ModeCheck<Exact>);
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) unsigned long long bars[kHeatXRing];
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
        const int bx = tid & 15, by = tid >> 4;           // own pair (2bx, by) in tile coords
        c.oe = heat_sidx(2 * bx + kHeatH, by + kHeatH);
        c.xe = (by + kHeatH) * kHeatXP + (2 * bx + kHeatH);
        const long long ix = ix0 + 2 * bx, iy = iy0 + by;
        c.of[0] = face_flags(ix, iy, g);
        c.of[1] = face_flags(ix + 1, iy, g);
        c.og = (c.of[0] & kIn) ? static_cast<int>(iy * g + ix) : 0;
        // halo-ring columns ordered by distance d = 1..4 from the tile (a column
        // at distance d is computed at stages 1 .. 4-d); slot 0: ring index tid,
        // slot 1: ring index 512 + tid (distance 4, load only)
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            int r = tid + s * kHeatThreads;
            // the computed bands (d = 1..3) fill ring indices [0, 420); the
            // load-only band d = 4 starts at the warp boundary 448 so that no
            // warp mixes the two (see HeatCols::wd)
            constexpr int kComputed = 132 + 140 + 148, kLoadStart = 448;
            if (r >= kComputed) r = (r < kLoadStart) ? -1 : r - kLoadStart + kComputed;
            // a lane without a column may still run a ring stage (wd): point it
            // at never-read pad cells (U: row 1, index 40; x ring: row 1, col 41)
            // so its neighbour reads stay inside the buffers and its writes are dead
            c.ro[s] = kHeatP + kHeatW;
            c.xr[s] = kHeatXP + kHeatXP - 1;
            c.rg[s] = 0;
            c.rf[s] = 0;
            c.rd[s] = -1;
            for (int d = 1; d <= kHeatH && r >= 0; ++d) {
                const int side = kHeatT + 2 * d, cnt = 4 * side - 4;
                if (r < cnt) {
                    const int lo = kHeatH - d;  // footprint coordinate of the band's first row/col
                    int x, y;
                    if (r < side) { y = lo; x = lo + r; }
                    else if (r < 2 * side) { y = lo + side - 1; x = lo + (r - side); }
                    else if (r < 3 * side - 2) { x = lo; y = lo + 1 + (r - 2 * side); }
                    else { x = lo + side - 1; y = lo + 1 + (r - (3 * side - 2)); }
                    const long long gx = ix0 - kHeatH + x, gy = iy0 - kHeatH + y;
                    c.ro[s] = heat_sidx(x, y);
                    c.xr[s] = y * kHeatXP + x;
                    c.rf[s] = face_flags(gx, gy, g) | ((x & 1) ? kOdd : 0);
                    if (c.rf[s] & kIn) {
                        c.rg[s] = static_cast<int>(gy * g + gx);
                        c.rd[s] = kHeatH - d;
                    }
                    break;
                }
                r -= cnt;
            }
        }
    }
    c.wd = __reduce_max_sync(0xffffffffu, c.rd[0]);
    const bool interior = ix0 - kHeatH >= 0 && ix0 + kHeatT + kHeatH <= g && iy0 - kHeatH >= 0 &&
                          iy0 + kHeatT + kHeatH <= g;
    const long long g2 = g * g;
    const int zs = static_cast<int>((obz - kHeatH > 0) ? obz - kHeatH : 0);
    const int ze = static_cast<int>((oez + kHeatH < g) ? oez + kHeatH : g);
    const double* src = (field ? w.in1 : w.in0) - static_cast<long long>(w.win_begin) * g2;
    double* dst = (field ? w.out1 : w.out0) - static_cast<long long>(w.out_begin) * g2;
    const unsigned long long n_total = static_cast<unsigned long long>(g2 * g);
    __shared__ unsigned tmem_base;
    const int warp = tid >> 5;
    if (warp == 0) tmem_alloc512(&tmem_base);  // one CTA per SM: the 512 columns are free
    if (tma && tid == 0) {
        for (int s = 0; s < kHeatXRing; ++s) mbar_init(bars + s, 1);
        mbar_fence_init();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    // (through a warp reduction: the base then sits in a uniform register)
    const unsigned tacc = __reduce_or_sync(0xffffffffu, tmem_base + (static_cast<unsigned>(32 * (warp & 3)) << 16) +
                                                            static_cast<unsigned>(128 * (warp >> 2)));
    const void* tmap = &tm.f[field];
    const int bx0 = static_cast<int>(ix0) - kHeatH, by0 = static_cast<int>(iy0) - kHeatH;
    const int wbz = static_cast<int>(w.win_begin);
    double* mdst = Mirror ? (field ? w.mir1 : w.mir0) - static_cast<long long>(w.out_begin) * g2 : nullptr;
    double* mhdst = Mirror ? (field ? w.mirh1 : w.mirh0) - static_cast<long long>(w.out_begin) * g2 : nullptr;
    const MirrorLimits mlim = MirrorLimits::of(w);
#define PIRK_HEAT_RUN(INTERIOR, TMA)                                                               \
    {                                                                                              \
        HeatRun<Exact, INTERIOR, TMA, Mirror> r{hp, sc, c, smem, zs, ze, static_cast<int>(obz),   \
                                        static_cast<int>(oez), static_cast<int>(g), zs > 0, ze < g, \
                                        g2, src, dst, field, m.method, step, fail, n_total, tmap,  \
                                        bx0, by0, wbz, bars, mdst, mhdst, mlim.lo_end, mlim.hi_begin};                                \
        r.tacc = tacc;                                                                             \
        r.run();                                                                                   \
    }
    if (tma) {
#ifdef PIRK_HEAT_TIMING_ONLY_INTERIOR  // A/B timing only (wrong at edge tiles)
        PIRK_HEAT_RUN(true, true)
#else
        if (interior) PIRK_HEAT_RUN(true, true) else PIRK_HEAT_RUN(false, true)
#endif
    } else {
        if (interior) PIRK_HEAT_RUN(true, false) else PIRK_HEAT_RUN(false, false)
    }
#undef PIRK_HEAT_RUN
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc512(tmem_base);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
inline bool heat_encode_tmap(CUtensorMap* out, const double* base, uint64_t g, uint64_t planes,
                             cuuint32_t box_x = kHeatXP, cuuint32_t box_y = kHeatW) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);
    static Encode encode = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<Encode>(fn);
    }
    if (!encode) return false;
    // strides must be 16-byte multiples and the base 16-byte aligned
    if ((g * sizeof(double)) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) % 16) != 0) return false;
    const cuuint64_t dims[3] = {g, g, planes};
    const cuuint64_t strides[2] = {g * sizeof(double), g * g * sizeof(double)};
    const cuuint32_t box[3] = {box_x, box_y, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    // L2 fill granularity of the box loads: a box row is 336 B at a 32 B
    // misalignment, so 64 B fills fetch the least from DRAM (measured, g=800:
    // 9.95 GB read per launch vs 12.08 GB at 256 B).  PIRK_TMA_PROMO overrides.
    static const CUtensorMapL2promotion promo = [] {
        const char* v = std::getenv("PIRK_TMA_PROMO");
        if (!v) return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
        const int b = std::atoi(v);
        return b == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
               : b == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
               : b == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                          : CU_TENSOR_MAP_L2_PROMOTION_NONE;
    }();
    return encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace pirk
