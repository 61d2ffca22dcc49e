// heat2x2.cuh -- K2 variant: the heat3d RK4 step with 2x2 register blocks.
//
// Same algorithm, buffers and boundary handling as heat.cuh (z-streaming,
// four lagged stages, x ring filled by TMA, double-buffered de-interleaved
// u planes, accumulators in TMEM); see that file for the design.  What
// changes is the ownership of the 32x32 tile: 256 threads each own a 2x2
// block instead of 512 threads each owning a 1x2 pair.  Inside a block, each
// point has two of its four in-plane neighbours in the same thread's
// registers, so a stage reads 8 neighbour values from shared memory per 4
// points instead of 12: about a quarter less shared-memory traffic, which is
// what bounds the 1x2 kernel (profiles/r01_heat_v12*).  The 576 halo-ring
// columns of the footprint are spread over three ring slots per thread:
// slot 0 (ring indices 0..255, computed up to stage 3), slot 1 (256..511,
// up to stage 2) and slot 2 (load only; nothing to do under TMA).
#pragma once

#include <cstdlib>

#include "heat.cuh"
#ifndef PIRK_DEV_VARIANTS
#define PIRK_DEV_VARIANTS 0  // 1: also build the rejected A/B variants (4x4 heat blocks, smem chain tiles)
#endif
#if PIRK_DEV_VARIANTS
#include "heat4x4.cuh"
#endif
#include <atomic>
#include "heat_strip.cuh"

namespace pirk {

constexpr int kHeat2Threads = 256;
// per-thread TMEM columns: RK accumulators of 4 plane slots at [0, 32), own x
// history (x(j-3), x(j-4) for stages 3 and 4) at [32, 64)
constexpr unsigned kXHist = 32;

// TMEM: 4 doubles = 8 columns per plane slot, 4 plane slots = 32 columns.
__device__ __forceinline__ void tmem_st4(unsigned taddr, const double (&v)[4]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
        "r"(__double2loint(v[0])), "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])),
        "r"(__double2hiint(v[1])), "r"(__double2loint(v[2])), "r"(__double2hiint(v[2])),
        "r"(__double2loint(v[3])), "r"(__double2hiint(v[3])));
}
__device__ __forceinline__ void tmem_ld4(unsigned taddr, double (&v)[4]) {
    unsigned r[8];
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                   "+r"(r[7]));
#pragma unroll
    for (int k = 0; k < 4; ++k)
        v[k] = __hiloint2double(static_cast<int>(r[2 * k + 1]), static_cast<int>(r[2 * k]));
}

// two slots with one wait (the accumulator and x history of one plane)
__device__ __forceinline__ void tmem_ld4x2(unsigned ta, unsigned tb, double (&a)[4], double (&b)[4]) {
    unsigned r[16];
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(ta));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15])
                 : "r"(tb));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                   "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                   "+r"(r[14]), "+r"(r[15]));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        a[k] = __hiloint2double(static_cast<int>(r[2 * k + 1]), static_cast<int>(r[2 * k]));
        b[k] = __hiloint2double(static_cast<int>(r[2 * k + 9]), static_cast<int>(r[2 * k + 8]));
    }
}

struct Heat2Cols {
    int ue;        // de-interleaved index of the block's (X0, Y0); (X0+1): +20, row Y0+1: +41
    int xe;        // row-major x-ring index of (X0, Y0); (X0+1): +1, row Y0+1: +42
    int og;        // in-plane global offset of (X0, Y0) (0 when outside the grid)
    int of[4];     // face flags of the block's points, k = dx + 2 dy
    int ro[3], xr[3], rg[3], rf[3], rd[3];  // halo-ring slots, as HeatCols
    int wd[2];     // warp-uniform max depth of ring slots 0 and 1
};

template <bool Exact, bool Interior, bool Tma, bool Mirror = false>
struct Heat2Run {
    const HeatStepParams& hp;
    const StepConsts& sc;
    const Heat2Cols& c;
    double* __restrict__ S;
    int zs, ze, ob, oe, g, lo_shift, hi_shift;
    long long g2;
    const double* __restrict__ src;
    double* __restrict__ dst;
    int field, method;
    unsigned long long step;
    unsigned long long* fail;
    unsigned long long n_total;
    const void* tmap;
    int bx0, by0, wbz;
    unsigned long long* bars;
    double* mdst;  // Mirror: the low neighbour's halo planes, indexed like dst
    double* mhdst;  // Mirror: the high neighbour's
    int m_lo_end, m_hi_begin;  // planes < m_lo_end go to mdst, planes >= m_hi_begin to mhdst

    // own block: [point k][plane slot (p - zs) & 3]
    double ox[4][4], ou1[4][4], ou2[4][4], ou3[4][4];
    // ring slot 0 (depth <= 3) and slot 1 (depth <= 2)
    double rx[4], ru1[4], ru2[4];
    double sx[4], su1[4];
    unsigned tacc;
    bool vec;  // outputs 16-byte aligned at even offsets (g even, aligned windows)
    const double* ldp;
    double* stp;
    double* mtp;  // Mirror: stp in the low neighbour's window
    double* mhp;  // Mirror: stp in the high neighbour's window

    __device__ __forceinline__ bool in(int k) const { return Interior || (c.of[k] & kIn); }
    __device__ __forceinline__ int goff(int k) const { return c.og + (k & 1) + (k >> 1) * g; }

    __device__ __forceinline__ void load(const double* plane, int p, int s) {
        double* X = S + xbuf(s);
        if constexpr (Tma) {
            if (threadIdx.x == 0) {
                mbar_expect_tx(bars + s, kHeatXSlot * sizeof(double));
                tma_load_plane(X, tmap, bx0, by0, p - wbz, bars + s);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (in(k)) cp_async8(X + c.xe + (k & 1) + (k >> 1) * kHeatXP, plane + goff(k));
#pragma unroll
            for (int s2 = 0; s2 < 3; ++s2)
                if (c.rd[s2] >= 0) cp_async8(X + c.xr[s2], plane + c.rg[s2]);
            cp_async_commit();
        }
    }

    __device__ __forceinline__ void own_x(int x_off, double (&v)[4]) const {
        const double2 a = *reinterpret_cast<const double2*>(S + x_off + c.xe);
        const double2 b = *reinterpret_cast<const double2*>(S + x_off + c.xe + kHeatXP);
        v[0] = a.x;
        v[1] = a.y;
        v[2] = b.x;
        v[3] = b.y;
    }

    // the four stencil values of the block from centres ce, z neighbours zm/zp
    // and in-plane neighbours l/r (per row) and u/d (per column)
    __device__ __forceinline__ void block_pts(const double (&ce)[4], const double (&zm)[4],
                                              const double (&zp)[4], double l0, double r0, double l1,
                                              double r1, double u0, double u1, double d0, double d1,
                                              double (&k)[4]) const {
        if constexpr (!Exact && Interior) {
            // fast interior: (ce1 + ce2) is in the sums of points 0 and 3,
            // (ce0 + ce3) in those of points 1 and 2
            const double a = ce[1] + ce[2], b = ce[0] + ce[3];
            k[0] = fma(-6.0, ce[0], (a + (l0 + u0)) + (zm[0] + zp[0]));
            k[1] = fma(-6.0, ce[1], (b + (r0 + u1)) + (zm[1] + zp[1]));
            k[2] = fma(-6.0, ce[2], (b + (l1 + d0)) + (zm[2] + zp[2]));
            k[3] = fma(-6.0, ce[3], (a + (r1 + d1)) + (zm[3] + zp[3]));
            return;
        }
        k[0] = heat_pt<Exact, Interior>(ce[0], l0, ce[1], u0, ce[2], zm[0], zp[0], c.of[0], hp);
        k[1] = heat_pt<Exact, Interior>(ce[1], ce[0], r0, u1, ce[3], zm[1], zp[1], c.of[1], hp);
        k[2] = heat_pt<Exact, Interior>(ce[2], l1, ce[3], ce[0], d0, zm[2], zp[2], c.of[2], hp);
        k[3] = heat_pt<Exact, Interior>(ce[3], ce[2], r1, ce[1], d1, zm[3], zp[3], c.of[3], hp);
    }

    // stage 1: neighbours from the row-major x plane
    __device__ __forceinline__ void block_eval_x(const double (&ce)[4], const double (&zm)[4],
                                                 const double (&zp)[4], int x_off,
                                                 double (&k)[4]) const {
        const double* B = S + x_off + c.xe;
        const double2 u = *reinterpret_cast<const double2*>(B - kHeatXP);
        const double2 d = *reinterpret_cast<const double2*>(B + 2 * kHeatXP);
        block_pts(ce, zm, zp, B[-1], B[2], B[kHeatXP - 1], B[kHeatXP + 2], u.x, u.y, d.x, d.y, k);
    }

    // stages 2-4: neighbours from a de-interleaved u plane
    __device__ __forceinline__ void block_eval(const double (&ce)[4], const double (&zm)[4],
                                               const double (&zp)[4], int in_off,
                                               double (&k)[4]) const {
        const double* B = S + in_off + c.ue;
        block_pts(ce, zm, zp, B[kHeatHalf - 1], B[1], B[kHeatP + kHeatHalf - 1], B[kHeatP + 1],
                  B[-kHeatP], B[kHeatHalf - kHeatP], B[2 * kHeatP], B[2 * kHeatP + kHeatHalf], k);
    }

    __device__ __forceinline__ void block_store(int off, const double (&v)[4]) const {
        double* B = S + off + c.ue;
        B[0] = v[0];
        B[kHeatHalf] = v[1];
        B[kHeatP] = v[2];
        B[kHeatP + kHeatHalf] = v[3];
    }

    template <int R>
    __device__ __forceinline__ double ring_eval_x(double s, double zm, double zp, int x_off) const {
        const double* B = S + x_off + c.xr[R];
        return heat_pt<Exact, Interior>(s, B[-1], B[1], B[-kHeatXP], B[kHeatXP], zm, zp, c.rf[R], hp);
    }
    template <int R>
    __device__ __forceinline__ double ring_eval(double s, double zm, double zp, int in_off) const {
        const double* B = S + in_off + c.ro[R];
        const int dm = (c.rf[R] & kOdd) ? -kHeatHalf : kHeatHalf - 1;
        return heat_pt<Exact, Interior>(s, B[dm], B[dm + 1], B[-kHeatP], B[kHeatP], zm, zp, c.rf[R], hp);
    }

    __device__ __forceinline__ double upd(double x, double k, double ce, double cf) const {
        return Exact ? x + ce * k : fma(cf, k, x);
    }

    template <int PH, bool ZEdge>
    __device__ __forceinline__ void iteration(int j) {
        constexpr int I0 = PH & 3, I1 = (PH + 3) & 3, I2 = (PH + 2) & 3, I3 = (PH + 1) & 3;
        constexpr int P0 = PH & 1, P1 = (PH + 1) & 1;
        const int x8 = (j - zs) & 7;
        const int X0 = xbuf(x8), X1 = xbuf((x8 + 7) & 7);
        if constexpr (Tma) {
            if (j + 3 < ze) load(nullptr, j + 3, (x8 + 3) & 7);  // into the slot of x(j-5)
            if (j < ze) mbar_wait(bars + x8, ((j - zs) >> 3) & 1);
        } else {
            if (j + 1 < ze) load(ldp, j + 1, (x8 + 1) & 7);
        }
        double xj[4];
        own_x(X0, xj);
        double rxj = S[X0 + c.xr[0]];
        double sxj = S[X0 + c.xr[1]];
        if (ZEdge && j == g) {  // insulated top face: x(g) := x(g-1)
#pragma unroll
            for (int k = 0; k < 4; ++k) xj[k] = ox[k][I1];
            rxj = rx[I1];
            sxj = sx[I1];
        }

        // ---------------- stage 1 at plane p = j-1
        {
            const int p = j - 1;
            if (!ZEdge || (p >= zs + lo_shift && p < ze - hi_shift)) {
                double ce[4], zm[4], kv[4], u[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    ce[k] = ox[k][I1];
                    zm[k] = ox[k][I2];
                }
                block_eval_x(ce, zm, xj, X1, kv);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    u[k] = upd(ce[k], kv[k], sc.h2, hp.hn[0]);
                    ou1[k][I1] = u[k];
                    if (ZEdge && p == 0) ou1[k][I2] = u[k];  // u1(-1) := u1(0)
                }
                if constexpr (Exact) tmem_st4(tacc + 8 * I1, kv);
                block_store(ubuf(1, P1), u);
                {  // slot 0 spans ring indices 0..255 (bands d = 1, 2): every warp runs stages 1-2
                    const double s = rx[I1];
                    const double uu = upd(s, ring_eval_x<0>(s, rx[I2], rxj, X1), sc.h2, hp.hn[0]);
                    ru1[I1] = uu;
                    S[ubuf(1, P1) + c.ro[0]] = uu;
                    if (ZEdge && p == 0) ru1[I2] = uu;
                }
                if (c.wd[1] >= 1) {
                    const double s = sx[I1];
                    const double uu = upd(s, ring_eval_x<1>(s, sx[I2], sxj, X1), sc.h2, hp.hn[0]);
                    su1[I1] = uu;
                    S[ubuf(1, P1) + c.ro[1]] = uu;
                    if (ZEdge && p == 0) su1[I2] = uu;
                }
            } else if (ZEdge && p == g) {  // u1(g) := u1(g-1)
#pragma unroll
                for (int k = 0; k < 4; ++k) ou1[k][I1] = ou1[k][I2];
                ru1[I1] = ru1[I2];
                su1[I1] = su1[I2];
            }
        }
        // ---------------- stage 2 at plane p = j-2
        {
            const int p = j - 2;
            if (!ZEdge || (p >= zs + 2 * lo_shift && p < ze - 2 * hi_shift)) {
                double ce[4], zm[4], zp[4], kv[4], u[4], a[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    ce[k] = ou1[k][I2];
                    zm[k] = ou1[k][I3];
                    zp[k] = ou1[k][I1];
                }
                block_eval(ce, zm, zp, ubuf(1, P0), kv);
                if constexpr (Exact) tmem_ld4(tacc + 8 * I2, a);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    u[k] = upd(ox[k][I2], kv[k], sc.h2, hp.hn[1]);
                    ou2[k][I2] = u[k];
                    if (ZEdge && p == 0) ou2[k][I3] = u[k];
                    if constexpr (Exact) a[k] = fma(2.0, kv[k], a[k]);  // acc + 2k (2k is exact)
                }
                if constexpr (Exact) tmem_st4(tacc + 8 * I2, a);
                block_store(ubuf(2, P0), u);
                {
                    const double uu = upd(rx[I2], ring_eval<0>(ru1[I2], ru1[I3], ru1[I1], ubuf(1, P0)),
                                          sc.h2, hp.hn[1]);
                    ru2[I2] = uu;
                    S[ubuf(2, P0) + c.ro[0]] = uu;
                    if (ZEdge && p == 0) ru2[I3] = uu;
                }
                if (c.wd[1] >= 2) {
                    S[ubuf(2, P0) + c.ro[1]] =
                        upd(sx[I2], ring_eval<1>(su1[I2], su1[I3], su1[I1], ubuf(1, P0)), sc.h2, hp.hn[1]);
                }
            } else if (ZEdge && p == g) {
#pragma unroll
                for (int k = 0; k < 4; ++k) ou2[k][I2] = ou2[k][I3];
                ru2[I2] = ru2[I3];
            }
        }
        // ---------------- stage 3 at plane p = j-3
        {
            const int p = j - 3;
            if (!ZEdge || (p >= zs + 3 * lo_shift && p < ze - 3 * hi_shift)) {
                double ce[4], zm[4], zp[4], kv[4], u[4], a[4], x3[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    ce[k] = ou2[k][I3];
                    zm[k] = ou2[k][I0];
                    zp[k] = ou2[k][I2];
                }
                block_eval(ce, zm, zp, ubuf(2, P1), kv);
                if constexpr (Exact) {
                    tmem_ld4x2(tacc + 8 * I3, tacc + kXHist + 8 * I3, a, x3);  // acc, x(j-3)
                } else {
                    tmem_ld4(tacc + kXHist + 8 * I3, x3);  // x(j-3)
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    u[k] = upd(x3[k], kv[k], sc.hk, hp.hn[2]);
                    ou3[k][I3] = u[k];
                    if (ZEdge && p == 0) ou3[k][I0] = u[k];
                    if constexpr (Exact) a[k] = fma(2.0, kv[k], a[k]);
                }
                if constexpr (Exact) tmem_st4(tacc + 8 * I3, a);
                block_store(ubuf(3, P1), u);
                if (c.wd[0] >= 3) {
                    S[ubuf(3, P1) + c.ro[0]] = upd(
                        rx[I3], ring_eval<0>(ru2[I3], ru2[I0], ru2[I2], ubuf(2, P1)), sc.hk, hp.hn[2]);
                }
            } else if (ZEdge && p == g) {
#pragma unroll
                for (int k = 0; k < 4; ++k) ou3[k][I3] = ou3[k][I0];
            }
        }
        // ---------------- stage 4 at plane p = j-4, stored to HBM
        {
            const int p = j - 4;
            if (!ZEdge || (p >= ob && p < oe)) {
                double ce[4], zm[4], zp[4], kv[4], a[4], x4[4], xn[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    ce[k] = ou3[k][I0];
                    zm[k] = ou3[k][I1];
                    zp[k] = ou3[k][I3];
                }
                block_eval(ce, zm, zp, ubuf(3, P0), kv);
                if constexpr (Exact) {
                    tmem_ld4x2(tacc + 8 * I0, tacc + kXHist + 8 * I0, a, x4);  // acc, x(j-4)
#pragma unroll
                    for (int k = 0; k < 4; ++k) xn[k] = x4[k] + sc.h6 * (a[k] + kv[k]);
                } else {
                    tmem_ld4(tacc + kXHist + 8 * I0, x4);  // x(j-4)
#pragma unroll
                    for (int k = 0; k < 4; ++k) xn[k] = fma(hp.hn[3], kv[k], x4[k]);
                }
                double* out = stp + c.og;
                if (Interior && vec) {  // og even: 16-byte aligned pairs
                    *reinterpret_cast<double2*>(out) = make_double2(xn[0], xn[1]);
                    *reinterpret_cast<double2*>(out + g) = make_double2(xn[2], xn[3]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (in(k)) out[(k & 1) + (k >> 1) * g] = xn[k];
                }
                if constexpr (Mirror) {
                    if (p < m_lo_end) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (in(k)) mtp[c.og + (k & 1) + (k >> 1) * g] = xn[k];
                    }
                    if (p >= m_hi_begin) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (in(k)) mhp[c.og + (k & 1) + (k >> 1) * g] = xn[k];
                    }
                }
                if (!finite_d((xn[0] + xn[1]) + (xn[2] + xn[3]))) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (!in(k) || finite_d(xn[k])) continue;
                        const unsigned long long gi =
                            static_cast<unsigned long long>(static_cast<long long>(p) * g2 + goff(k));
                        if (method == 0)
                            record_fail(fail, step, gi + (field ? n_total : 0ull));
                        else if (fail)
                            record_fail(fail + field, step, gi);
                    }
                }
            }
        }
        tmem_st4(tacc + kXHist + 8 * I0, xj);  // x(j) for stages 3 and 4 (slot of x(j-4), read above)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            ox[k][I0] = xj[k];
            if (ZEdge && j == 0) ox[k][I1] = xj[k];  // x(-1) := x(0)
        }
        rx[I0] = rxj;
        sx[I0] = sxj;
        if (ZEdge && j == 0) {
            rx[I1] = rxj;
            sx[I1] = sxj;
        }
        ldp += g2;
        stp += g2;
        if constexpr (Mirror) {
            mtp += g2;
            mhp += g2;
        }
        if constexpr (!Tma) cp_async_wait_all();
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
            load(src + static_cast<long long>(zs) * g2, zs, 0);
            if constexpr (Tma) {
                if (zs + 1 < ze) load(nullptr, zs + 1, 1);
                if (zs + 2 < ze) load(nullptr, zs + 2, 2);
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
        // steady-state bounds: as HeatRun::run
        int a = zs + 3 + 3 * lo_shift;
        if (a < ob + 4) a = ob + 4;
        if (a < 5) a = 5;
        a = zs + ((a - zs + 3) & ~3);
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

template <bool Exact, bool Mirror = false>
__global__ void __launch_bounds__(kHeat2Threads, 1)
heat2_step_kernel(const HeatModel m, const HeatStepParams hp, const WindowArgs w,
                  const StepConsts sc, const unsigned long long step, const uint64_t zchunk,
                  unsigned long long* __restrict__ fail, const __grid_constant__ HeatTmaps tm,
                  const int flags) {
    (void)sizeof(ModeCheck<Exact>);
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) unsigned long long bars[kHeatXRing];
    const bool tma = flags & 1;
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

    Heat2Cols c;
    {
        const int bx = tid & 15, by = tid >> 4;  // own block (2bx, 2by) in tile coords
        const int fx = 2 * bx + kHeatH, fy = 2 * by + kHeatH;
        c.ue = heat_sidx(fx, fy);
        c.xe = fy * kHeatXP + fx;
        const long long ix = ix0 + 2 * bx, iy = iy0 + 2 * by;
#pragma unroll
        for (int k = 0; k < 4; ++k) c.of[k] = face_flags(ix + (k & 1), iy + (k >> 1), g);
        c.og = (c.of[0] & kIn) ? static_cast<int>(iy * g + ix) : 0;
        // ring index r = tid + 256 s, mapped as in heat_step_kernel: computed
        // bands at [0, 420), padding to the warp boundary 448, load-only band
        // from 448.  Slot 0 holds depths <= 3, slot 1 depths <= 2 (its first
        // computed index is 256, inside band d = 2), slot 2 is load-only.
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            int r = tid + s * kHeat2Threads;
            constexpr int kComputed = 132 + 140 + 148, kLoadStart = 448;
            if (r >= kComputed) r = (r < kLoadStart) ? -1 : r - kLoadStart + kComputed;
            c.ro[s] = kHeatP + kHeatW;  // never-read pad cells for lanes without a column
            c.xr[s] = kHeatXP + kHeatXP - 1;
            c.rg[s] = 0;
            c.rf[s] = 0;
            c.rd[s] = -1;
            for (int d = 1; d <= kHeatH && r >= 0; ++d) {
                const int side = kHeatT + 2 * d, cnt = 4 * side - 4;
                if (r < cnt) {
                    const int lo = kHeatH - d;
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
    c.wd[0] = __reduce_max_sync(0xffffffffu, c.rd[0]);
    c.wd[1] = __reduce_max_sync(0xffffffffu, c.rd[1]);
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
    if (warp == 0) tmem_alloc512(&tmem_base);
    if (tma && tid == 0) {
        for (int s = 0; s < kHeatXRing; ++s) mbar_init(bars + s, 1);
        mbar_fence_init();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    // warp w: TMEM lane quadrant w % 4, columns 64 (w / 4) .. +63
    const unsigned tacc = __reduce_or_sync(0xffffffffu, tmem_base + (static_cast<unsigned>(32 * (warp & 3)) << 16) +
                                                            static_cast<unsigned>(64 * (warp >> 2)));
    const void* tmap = &tm.f[field];
    const int bx0 = static_cast<int>(ix0) - kHeatH, by0 = static_cast<int>(iy0) - kHeatH;
    const int wbz = static_cast<int>(w.win_begin);
    double* mdst = Mirror ? (field ? w.mir1 : w.mir0) - static_cast<long long>(w.out_begin) * g2 : nullptr;
    double* mhdst = Mirror ? (field ? w.mirh1 : w.mirh0) - static_cast<long long>(w.out_begin) * g2 : nullptr;
    const MirrorLimits mlim = MirrorLimits::of(w);
#define PIRK_HEAT2_RUN(INTERIOR, TMA)                                                              \
    {                                                                                              \
        Heat2Run<Exact, INTERIOR, TMA, Mirror> r{hp, sc, c, smem, zs, ze, static_cast<int>(obz),  \
                                         static_cast<int>(oez), static_cast<int>(g), zs > 0,      \
                                         ze < g, g2, src, dst, field, m.method, step, fail,        \
                                         n_total, tmap, bx0, by0, wbz, bars, mdst, mhdst, mlim.lo_end, mlim.hi_begin};                \
        r.tacc = tacc;                                                                             \
        r.vec = (flags & 2) != 0;                                                                  \
        r.run();                                                                                   \
    }
    if (tma) {
        if (interior) PIRK_HEAT2_RUN(true, true) else PIRK_HEAT2_RUN(false, true)
    } else {
        if (interior) PIRK_HEAT2_RUN(true, false) else PIRK_HEAT2_RUN(false, false)
    }
#undef PIRK_HEAT2_RUN
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc512(tmem_base);
}

// z-chunk length for one-CTA-per-SM heat kernels over tx x tx tiles and two
// fields: the count minimising waves x (planes per chunk + 8 halo planes
// recomputed per chunk), i.e. the wave quantisation of nf tx^2 CTAs per chunk
inline uint64_t heat_zchunk(uint64_t tx, uint64_t planes, int n_sm, unsigned nf = 2) {
    static const int forced = [] {  // PIRK_HEAT_ZCHUNKS=c forces c chunks (A/B only)
        const char* v = std::getenv("PIRK_HEAT_ZCHUNKS");
        return v ? std::atoi(v) : 0;
    }();
    if (forced > 0) return (planes + forced - 1) / forced;
    uint64_t best = 1;
    double best_cost = 0.0;
    for (uint64_t c = 1; c <= 8 && c <= planes; ++c) {
        const uint64_t zc = (planes + c - 1) / c;
        const uint64_t ctas = tx * tx * nf * ((planes + zc - 1) / zc);
        const double cost = static_cast<double>((ctas + n_sm - 1) / n_sm) *
                            static_cast<double>(zc + (c > 1 ? 2 * kHeatH : 0));
        if (c == 1 || cost < best_cost) best = c, best_cost = cost;
    }
    return (planes + best - 1) / best;
}

template <bool Exact>
cudaError_t launch_heat_step(const HeatModel& m, const WindowArgs& w, const StepConsts& sc,
                             unsigned long long step, unsigned long long* fail,
                             cudaStream_t stream, int field_only) {
    if (w.out_end <= w.out_begin) return cudaSuccess;
    // field_only >= 0: advance that field alone (grid z = chunks, flags bit 2 + index)
    const unsigned nf = field_only < 0 ? 2u : 1u;
    const int fsel = field_only < 0 ? 0 : (4 | ((field_only & 1) << 3));
    // Kernel variant.  Fast mode: warp-wide strips with TMEM histories
    // (heat_strip.cuh) whenever its TMA path is available (even g, aligned
    // windows), else 2x2 blocks.  Exact mode: 1x2 pairs (its longer per-point
    // expression does not fit 2x2 blocks in registers; measured faster as pairs).
    // PIRK_HEAT_BLOCK=1x2|2x2|4x4|strip overrides (A/B comparisons; 4x4 and
    // strip are fast-only).
    static const int variant = [] {
        const char* v = std::getenv("PIRK_HEAT_BLOCK");
        if (v && std::strcmp(v, "1x2") == 0) return 0;
        if (v && std::strcmp(v, "2x2") == 0) return 1;
        if (v && std::strcmp(v, "4x4") == 0) return 2;
        if (v && std::strcmp(v, "strip") == 0) return 3;
        return Exact ? 0 : 3;
    }();
    // one-field launches exist for the strip kernel only (fast mode, even g);
    // the engine's field-pipelined driver checks that before using them
    if (field_only >= 0 && (Exact || variant != 3 || m.g % 2 != 0 ||
                            (PIRK_STRIP_SFORM && !heat_sform_coeffs(sc.hk * m.kk, nullptr))))
        return cudaErrorInvalidValue;

    // dynamic shared memory opt-in is per device: once per kernel and device
    static std::atomic<unsigned long long> attr_done{0};
    int cur_dev = 0;
    if (cudaGetDevice(&cur_dev) != cudaSuccess) return cudaErrorInvalidDevice;
    const unsigned long long dev_bit = 1ull << (cur_dev & 63);
    if (!(attr_done.load(std::memory_order_acquire) & dev_bit)) {
        cudaError_t e = cudaFuncSetAttribute(heat_step_kernel<Exact>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kHeatSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(heat_step_kernel<Exact, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kHeatSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(heat2_step_kernel<Exact>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kHeatSmemBytes));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(heat2_step_kernel<Exact, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kHeatSmemBytes));
        if constexpr (!Exact) {
#if PIRK_DEV_VARIANTS
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(heat4_step_kernel<Exact>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(k4SmemBytes));
#endif
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(heat_strip_kernel<Exact, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSSmemBytes));
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(heat_strip_kernel<Exact, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSSmemBytes));
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(heat_strip_kernel<Exact, false, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSSmemBytes));
        }
        if (e != cudaSuccess) return e;
        attr_done.fetch_or(dev_bit, std::memory_order_acq_rel);
    }
    static const int n_sm = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    HeatStepParams hp{};
    hp.kk = m.kk;
    hp.robin = m.robin;
    hp.h2kk = sc.h2 * m.kk;
    hp.hkk = sc.hk * m.kk;
    hp.h6kk = sc.h6 * m.kk;
    hp.hn[3] = sc.hk * m.kk;
    hp.hn[0] = hp.hn[3] / 4.0;
    hp.hn[1] = hp.hn[3] / 3.0;
    hp.hn[2] = hp.hn[3] / 2.0;
    // the strip kernel's S form needs z = hk*kk in heat_sform_coeffs' range
    const bool sform_ok = !PIRK_STRIP_SFORM || heat_sform_coeffs(sc.hk * m.kk, hp.sf);
    const uint64_t planes = w.out_end - w.out_begin;
    const uint64_t wplanes = w.win_end - w.win_begin;
    const bool vec = (m.g % 2 == 0) && reinterpret_cast<uintptr_t>(w.out0) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(w.out1) % 16 == 0;
    HeatTmaps tm;
    std::memset(&tm, 0, sizeof tm);
    if constexpr (!Exact) {
        if (variant == 3 && sform_ok && heat_encode_tmap(&tm.f[0], w.in0, m.g, wplanes, kSF, kSF) &&
            heat_encode_tmap(&tm.f[1], w.in1, m.g, wplanes, kSF, kSF)) {
            const uint64_t tx = (m.g + kST - 1) / kST;
            const uint64_t zchunk = heat_zchunk(tx, planes, n_sm, nf);
            const uint64_t nchunks = (planes + zchunk - 1) / zchunk;
            dim3 grid(static_cast<unsigned>(tx), static_cast<unsigned>(tx), static_cast<unsigned>(nf * nchunks));
            if (field_only >= 0)
                heat_strip_kernel<Exact, true><<<grid, kSThreads, kSSmemBytes, stream>>>(
                    m, hp, w, sc, step, zchunk, fail, tm, 1 | (vec ? 2 : 0) | fsel);
            else if (w.mirrored())
                heat_strip_kernel<Exact, false, true><<<grid, kSThreads, kSSmemBytes, stream>>>(
                    m, hp, w, sc, step, zchunk, fail, tm, 1 | (vec ? 2 : 0));
            else
                heat_strip_kernel<Exact, false><<<grid, kSThreads, kSSmemBytes, stream>>>(
                    m, hp, w, sc, step, zchunk, fail, tm, 1 | (vec ? 2 : 0));
            return cudaGetLastError();
        }
        std::memset(&tm, 0, sizeof tm);
#if PIRK_DEV_VARIANTS
        // 16-byte copies need even g and 16-byte aligned windows
        if (variant == 2 && m.g % 2 == 0 && reinterpret_cast<uintptr_t>(w.in0) % 16 == 0 &&
            reinterpret_cast<uintptr_t>(w.in1) % 16 == 0) {
            const uint64_t tx = (m.g + k4T - 1) / k4T;
            const uint64_t zchunk = heat_zchunk(tx, planes, n_sm, nf);
            const uint64_t nchunks = (planes + zchunk - 1) / zchunk;
            dim3 grid(static_cast<unsigned>(tx), static_cast<unsigned>(tx), static_cast<unsigned>(nf * nchunks));
            heat4_step_kernel<Exact><<<grid, k4Threads, k4SmemBytes, stream>>>(m, hp, w, sc, step, zchunk, fail,
                                                                                tm, 1 | (vec ? 2 : 0));
            return cudaGetLastError();
        }
#endif
    }
    // z chunks: enough CTAs to fill the machine, few enough to keep the
    // 8-plane halo overhead per chunk small.
    const uint64_t tx = (m.g + kHeatT - 1) / kHeatT;
    uint64_t nchunks = 1;
    while (tx * tx * nf * nchunks < 4 * static_cast<uint64_t>(n_sm) && planes / (nchunks * 2) >= 64) nchunks *= 2;
    const uint64_t zchunk = (planes + nchunks - 1) / nchunks;
    nchunks = (planes + zchunk - 1) / zchunk;
    dim3 grid(static_cast<unsigned>(tx), static_cast<unsigned>(tx), static_cast<unsigned>(nf * nchunks));
    const int tma = heat_encode_tmap(&tm.f[0], w.in0, m.g, wplanes) &&
                    heat_encode_tmap(&tm.f[1], w.in1, m.g, wplanes);
    if (variant >= 1) {
        if (w.mirrored())
            heat2_step_kernel<Exact, true><<<grid, kHeat2Threads, kHeatSmemBytes, stream>>>(
                m, hp, w, sc, step, zchunk, fail, tm, tma | (vec ? 2 : 0));
        else
            heat2_step_kernel<Exact><<<grid, kHeat2Threads, kHeatSmemBytes, stream>>>(
                m, hp, w, sc, step, zchunk, fail, tm, tma | (vec ? 2 : 0));
    } else if (w.mirrored()) {
        heat_step_kernel<Exact, true><<<grid, kHeatThreads, kHeatSmemBytes, stream>>>(m, hp, w, sc, step, zchunk,
                                                                                      fail, tm, tma);
    } else {
        heat_step_kernel<Exact><<<grid, kHeatThreads, kHeatSmemBytes, stream>>>(m, hp, w, sc, step, zchunk,
                                                                                fail, tm, tma);
    }
    return cudaGetLastError();
}


}  // namespace pirk
