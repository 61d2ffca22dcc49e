// heat_strip.cuh -- K2 v16 (fast mode): the heat3d RK4 step with warp-wide
// row strips: x-neighbours by shuffle, y-neighbours by one row exchange in
// shared memory, z-histories in TMEM.
//
// Replaces integrate_step (rk4.cpp:30-76) on the heat3d embedding / growth
// pair exactly as heat.cuh does (models.cpp:92-133; both fields evolve
// independently under the same linear 7-point operator), held to the fast-mode
// contract (relative <= 1e-12, never tighter; tests/helpers.assert_within).
//
// Why.  heat.cuh / heat2x2.cuh spend ~1.4 shared-memory wavefronts per
// state-update (67% of the crossbar at g=800, profiles/r01_heat_v14_g800.txt):
// every stage value is stored and 2-3 neighbours are read back per point.
// Measured on this B200 (tools/tmem_bw.cu): a 32-bit warp shuffle issues at
// ~2 per clock per SM, so exchanging a double by shuffle costs a quarter of a
// shared-memory store + load (4 wavefronts per 32 doubles); tcgen05.ld/st
// move ~430/360 B/clk/SM, 3x the shared-memory crossbar.
//
// Geometry.  A CTA (one per SM) owns a 56x56 x-y tile of one field and streams
// the planes of a z-chunk; the footprint with the 4-cell halo is 64x64.  Lane l
// of warp w (16 warps) owns the 2x4 block at footprint columns 2l, 2l+1 and rows
// 4w .. 4w+3, so a warp spans the whole footprint width: every x-neighbour is
// in the same thread or the adjacent lane (shfl_up / shfl_down; lanes 0 and 31
// are halo columns whose garbage never reaches the tile), and every
// y-neighbour is in the same thread or the same lane of the warp above/below
// (one double2 row exchanged through shared memory, conflict-free).  Blocks in
// the 4-cell halo recompute stages 1-3 (the dependency cone); the inner 14x14
// blocks run stage 4 and store to HBM.  Every thread runs the same code; only
// the HBM store is predicated.
//
// Pipeline.  Iteration j waits for x-plane j (a 64x64 TMA box, zero-filled
// outside the grid, 4-slot ring, prefetched 2 planes ahead) and evaluates stage
// 1 at plane j-1, stage 2 at j-2, stage 3 at j-3 and stage 4 at j-4 (the lagged
// schedule of heat.cuh).  Fast mode evaluates RK4 for this linear autonomous
// field in Horner form, x + hL(x + hL/2(x + hL/3(x + hL/4 x))): a stage is
// v_s = x + c_s (sum6(v_{s-1}) - 6 v_{s-1}), c = hk*kk/{4,3,2,1}.  Stage 4's z-
// and centre terms are folded one iteration early into
// A4(p) = x(p) + c4 (u3(p-1) - 6 u3(p)).  TMEM holds, per thread, 8 plane slots
// of its block (16 columns each): x(j-2), x(j-3), u1(j-2), u1(j-3), u2(j-3),
// u2(j-4), u3(j-4), A4(j-4); x(j-1) and x(j) are read from the x ring.  Each
// slot a stage overwrites is read (it is the next stage's z- plane) before
// the stage runs, so every result is stored as soon as it exists.
//
// Exchange.  Three levels (u1, u2, u3), each TOP[512] and BOT[512] double2
// (the first and last row of every block), double-buffered by iteration
// parity: a stage reads the rows its predecessor published in the previous
// iteration and publishes its own rows as soon as they exist, so one barrier
// per plane suffices.  Stage 1 reads the rows above / below straight from the
// x ring.
//
// Boundaries.  Edge tiles substitute ghost values per point (Robin at x = 0,
// insulated elsewhere) as heat_pt does; insulated z faces replicate the boundary
// plane, as heat.cuh.
#pragma once

#include "heat.cuh"
#include "tmem_io.cuh"

#ifndef PIRK_STRIP_CSE
#define PIRK_STRIP_CSE 1   // interior tiles share anti-diagonal pair sums
#endif
#ifndef PIRK_STRIP_L2PF
#define PIRK_STRIP_L2PF 0  // L2 prefetch of x planes beyond the smem ring (measured: 1, 2, 4 planes all slightly slower)
#endif
#ifndef PIRK_STRIP_SPLITBAR
#define PIRK_STRIP_SPLITBAR 1  // split per-plane barrier (mbarrier arrive at the end, wait before the first publish): 38.2 -> 35.1 ms at g=1600
#endif
#ifndef PIRK_STRIP_XSWAP
#define PIRK_STRIP_XSWAP 1  // x(j-1) to TMEM from stage 1, A4 formed in stage 3: 35.0 -> 34.9 ms
#endif
#ifndef PIRK_STRIP_XCARRY
#define PIRK_STRIP_XCARRY 0  // x(j) kept in registers as the next centre: 36.9 vs 34.9 ms (pressure)
#endif
#ifndef PIRK_STRIP_LADDER
#define PIRK_STRIP_LADDER 0  // 1/2: per-level publish barriers (2: TMA after stage 3): 37.1 / 37.3 vs 35.0 ms at g=1600
#endif
#if PIRK_STRIP_LADDER && !PIRK_STRIP_SPLITBAR
#error "PIRK_STRIP_LADDER needs PIRK_STRIP_SPLITBAR"
#endif
#ifndef PIRK_STRIP_EDGECSE
#define PIRK_STRIP_EDGECSE 1  // edge tiles of g % 4 == 0 grids: ghost values substituted per exchanged neighbour, shared pair sums
#endif
#ifndef PIRK_STRIP_SANITIZE
// 1 (racecheck builds only): the halo warps' reads of the rows outside the
// footprint (warp 0's row -1, warp 15's row 64) go to a private dummy row
// instead of wrapping into the exchange region / the next x slot.  Those
// values only ever feed halo cells (garbage by design, never stored), so the
// wrap is benign -- but racecheck reports it; with this on, any remaining
// hazard would be a real one.
#define PIRK_STRIP_SANITIZE 0
#endif
#ifndef PIRK_STRIP_SFORM
// 1: RK4 as a polynomial in the neighbour-sum operator S (HeatStepParams::sf):
// a stage is w = S(v) + a x, one DFMA instead of Horner-in-L's two
// (x + c (S(v) - 6 v)); stage 4 is y = q4 S(w3) + q0 x
#define PIRK_STRIP_SFORM 1
#endif
#ifndef PIRK_STRIP_F32CHK
// 1: the per-block non-finite screen sums the values' high words on the FP32
// pipe (common.cuh maybe_nonfinite8) instead of 7 DADDs on the FP64 pipe
#define PIRK_STRIP_F32CHK 1
#endif
#ifndef PIRK_STRIP_EARLYLD
// 1: steady-state iterations issue stage 1's three TMEM loads (x(j-3), x(j-2),
// u1(j-3)) before the x-plane wait and complete them just before use
#define PIRK_STRIP_EARLYLD 0
#endif
#ifndef PIRK_STRIP_S4SKIP
#define PIRK_STRIP_S4SKIP 0  // halo warps 0 and 15 skip stage 4 (measured slower: 7.40 vs 6.55 ms, g=800)
#endif

namespace pirk {

constexpr int kST = 56;                 // output tile edge
constexpr int kSF = 64;                 // footprint edge
constexpr int kSThreads = 512;          // 16 warps x 32 lanes, one 2x4 block each
constexpr int kSXSlots = 4;             // x planes j-1 .. j+2
constexpr int kSXSlot = kSF * kSF;      // doubles per x slot (row-major, pitch 64)
constexpr int kSLevel = 2 * kSThreads;  // double2 entries per exchange level: TOP, BOT
constexpr size_t kSEdgeBytes = size_t(2 * 3) * kSLevel * sizeof(double2);      // 96 KB: 2 buffers x 3 levels
constexpr size_t kSRingBytes = size_t(kSXSlots) * kSXSlot * sizeof(double);    // 128 KB
// [exchange][x ring][one row of padding]: the rows above / below the
// footprint that halo blocks read land in the exchange region or the padding
constexpr size_t kSSmemBytes = kSEdgeBytes + kSRingBytes + kSF * sizeof(double);

// TMEM plane slots of a thread (16 columns = 8 doubles each)
enum : int { kSX = 0, kSU1 = 2, kSU2 = 4, kSU3 = 6, kSA4 = 7 };

// Non-finite output at plane p (cold path): read the block's stored cells back
// and record each bad one (atomicMin keeps the lowest component).
__device__ __forceinline__ void heat_strip_report(const double* stp, int g, long long g2, int p, int gout,
                                                  unsigned mask, int field, int method,
                                                  unsigned long long step, unsigned long long* fail,
                                                  unsigned long long n_total) {
#pragma unroll 1
    for (int i = 0; i < 8; ++i) {
        const int r = i >> 1, c = i & 1;
        if (!((mask >> i) & 1)) continue;
        if (finite_d(stp[r * g + c])) continue;
        const unsigned long long gi =
            static_cast<unsigned long long>(static_cast<long long>(p) * g2 + gout + r * g + c);
        if (method == 0)
            record_fail(fail, step, gi + (field ? n_total : 0ull));
        else if (fail)
            record_fail(fail + field, step, gi);
    }
}

// Kind: 0 interior tile, 1 edge tile of a g % 4 == 0 grid (PIRK_STRIP_EDGECSE),
// 2 any other edge tile
template <int Kind, bool Mirror = false>
struct HeatStrip {
    static constexpr bool Interior = Kind == 0;
    static constexpr bool EdgeCse = Kind == 1;
    const HeatStepParams& hp;
    double2* __restrict__ EX;  // exchange levels
    double* __restrict__ XR;   // x ring
    int t;                     // thread = block index (warp * 32 + lane)
    bool inner;                // warps 1..14: rows of the tile (stage 4 runs)
    int xo;                    // own block offset in an x slot: row 4w, column 2l
    int zs, ze, ob, oe, g, lo_shift, hi_shift;
    long long g2;
    double* __restrict__ stp;  // output plane j-4 at the own block's (0,0)
    double* mtp;               // Mirror: stp in the low neighbour's window (planes < m_lo_end)
    double* mhp;               // Mirror: stp in the high neighbour's window (planes >= m_hi_begin)
    int m_lo_end, m_hi_begin;
    bool st_own;               // own block with all 8 cells in the grid (vector stores)
    unsigned st_mask;          // edge tiles: per-cell store mask (bit 2r+c)
    int gout;                  // in-plane global offset of the block's (0,0) cell
    int fx0, fxg, fy0, fyg;    // edge tiles: columns at x=0 / x=g-1 (2 bits), rows at y=0 / y=g-1 (4 bits)
    int field, method;
    unsigned long long step;
    unsigned long long* fail;
    unsigned long long n_total;
    const void* tmap;
    int bx0, by0, wbz;
    unsigned long long* bars;
    unsigned long long* done;  // split barrier: warps arrive when a plane's exchange work is complete
    unsigned tt;  // TMEM address of slot 0
    int xs;       // x ring slot of plane j
    int xph;      // mbarrier phase bit per slot
    double xc[8];  // XCARRY: own block of x(j) for the next iteration (valid after any iteration)

    __device__ __forceinline__ unsigned ts(int slot) const { return tt + 16u * slot; }
    // stage coefficient s (0..2) and stage 4's S coefficient
    __device__ __forceinline__ double cst(int s) const { return PIRK_STRIP_SFORM ? hp.sf[s] : hp.hn[s]; }
    __device__ __forceinline__ double c4() const { return PIRK_STRIP_SFORM ? hp.sf[3] : hp.hn[3]; }
    // A4(p) from u3(p-1), u3(p), x(p)
    __device__ __forceinline__ double a4_of(double um, double u, double x) const {
        if constexpr (PIRK_STRIP_SFORM)
            return fma(hp.sf[3], um, hp.sf[4] * x);
        else
            return fma(hp.hn[3], fma(-6.0, u, um), x);
    }
    __device__ __forceinline__ double* xslot(int s) const { return XR + s * kSXSlot; }

#ifndef PIRK_STRIP_ST2
#define PIRK_STRIP_ST2 1
#endif
    // Store a plane slot.  One 2-column store per double: an x16 store needs its
    // 16 source registers contiguous, which costs ~16 register moves per store.
    __device__ __forceinline__ void st8(unsigned ta, const double (&v)[8]) const {
        if constexpr (PIRK_STRIP_ST2) {
#pragma unroll
            for (int i = 0; i < 8; ++i) tm_st1(ta + 2 * i, v[i]);
        } else {
            tm_st8(ta, v);
        }
    }

    __device__ __forceinline__ void tma(int p, int s) {
        mbar_expect_tx(bars + s, kSXSlot * sizeof(double));
        tma_load_plane(xslot(s), tmap, bx0, by0, p - wbz, bars + s);
    }

    // own 2x4 block of an x slot (v[2r + c])
    __device__ __forceinline__ void own_x(const double* X, double (&v)[8]) const {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const double2 a = *reinterpret_cast<const double2*>(X + xo + r * kSF);
            v[2 * r] = a.x;
            v[2 * r + 1] = a.y;
        }
    }

    // rows above / below the block: from the x slot (stage 1) or a level
    __device__ __forceinline__ const double* dummy_row() const {
        return XR + kSXSlots * kSXSlot + 2 * (t & 31);  // the padding row after the ring
    }
    __device__ __forceinline__ void x_tb(const double* X, double (&T)[2], double (&B)[2]) const {
        const double* pa = X + xo - kSF;
        const double* pc = X + xo + 4 * kSF;
        if constexpr (PIRK_STRIP_SANITIZE) {
            if (t < 32) pa = dummy_row();
            if (t >= kSThreads - 32) pc = dummy_row();
        }
        const double2 a = *reinterpret_cast<const double2*>(pa);
        const double2 c = *reinterpret_cast<const double2*>(pc);
        T[0] = a.x, T[1] = a.y, B[0] = c.x, B[1] = c.y;
    }
    // exchange buffer `buf` (iteration parity) of level 0..2 (u1..u3)
    __device__ __forceinline__ void u_tb(int buf, int level, double (&T)[2], double (&B)[2]) const {
        const double2* L = EX + (3 * buf + level) * kSLevel;
        const double2* pa = L + kSThreads + t - 32;  // BOT of the block above
        const double2* pc = L + t + 32;              // TOP of the block below
        if constexpr (PIRK_STRIP_SANITIZE) {
            if (t < 32) pa = reinterpret_cast<const double2*>(dummy_row());
            if (t >= kSThreads - 32) pc = reinterpret_cast<const double2*>(dummy_row());
        }
        const double2 a = *pa;
        const double2 c = *pc;
        T[0] = a.x, T[1] = a.y, B[0] = c.x, B[1] = c.y;
    }
    __device__ __forceinline__ void publish(int buf, int level, const double (&v)[8]) const {
        double2* L = EX + (3 * buf + level) * kSLevel;
        L[t] = make_double2(v[0], v[1]);
        L[kSThreads + t] = make_double2(v[6], v[7]);
    }

    // anti-diagonal pair sums P(r, c) = v(r, c+1) + v(r+1, c) are shared:
    // point (r, 0) sums P(r, 0) + P(r-1, -1), point (r, 1) P(r, 1) + P(r-1, 0)
    __device__ __forceinline__ static void cse_sums(const double (&C)[8], const double (&T)[2],
                                                    const double (&B)[2], const double (&L)[4],
                                                    const double (&R)[4], double (&s)[8]) {
        auto V = [&](int r, int c) -> double {
            if (r < 0) return T[c];
            if (r > 3) return B[c];
            if (c < 0) return L[r];
            if (c > 1) return R[r];
            return C[2 * r + c];
        };
        double pm = V(-1, 0) + V(0, -1);  // P(r-1, -1)
        double p0 = V(-1, 1) + V(0, 0);   // P(r-1, 0)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const double q0 = V(r, 1) + V(r + 1, 0);  // P(r, 0)
            const double q1 = V(r, 2) + V(r + 1, 1);  // P(r, 1)
            s[2 * r] = q0 + pm;
            s[2 * r + 1] = q1 + p0;
            if (r < 3) pm = V(r, 0) + V(r + 1, -1);  // P(r, -1)
            p0 = q0;
        }
    }

    // in-plane sums xm + xp + ym + yp of the 8 points of centre plane C
    __device__ __forceinline__ void inplane(const double (&C)[8], const double (&T)[2], const double (&B)[2],
                                            double (&s)[8]) const {
        double L[4], R[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            L[r] = __shfl_up_sync(0xffffffffu, C[2 * r + 1], 1);
            R[r] = __shfl_down_sync(0xffffffffu, C[2 * r], 1);
        }
        if constexpr (Interior && PIRK_STRIP_CSE) {
            cse_sums(C, T, B, L, R, s);
            return;
        }
        if constexpr (EdgeCse) {
            // g % 4 == 0: every grid face lies on a block edge -- x = 0 at a
            // lane's column 0, x = g-1 at column 1, y = 0 at row 0, y = g-1 at
            // row 3 -- so the ghost value of a face cell replaces exactly one
            // exchanged neighbour (L, R, T or B), used by that cell alone:
            // substitute it, then share pair sums as interior tiles do.
            {
                double L2[4], R2[4], T2[2], B2[2];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    L2[r] = (fx0 & 1) ? fma(-hp.robin, C[2 * r], C[2 * r + 1]) : L[r];  // Robin ghost
                    R2[r] = (fxg & 2) ? C[2 * r + 1] : R[r];                             // insulated
                }
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    T2[c] = (fy0 & 1) ? C[c] : T[c];
                    B2[c] = (fyg & 8) ? C[6 + c] : B[c];
                }
                cse_sums(C, T2, B2, L2, R2, s);
                return;
            }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const double ctr = C[2 * r + c];
                double xm = c ? C[2 * r] : L[r];
                double xp = c ? R[r] : C[2 * r + 1];
                double ym = r > 0 ? C[2 * (r - 1) + c] : T[c];
                double yp = r < 3 ? C[2 * (r + 1) + c] : B[c];
                if constexpr (!Interior) {
                    xm = ((fx0 >> c) & 1) ? fma(-hp.robin, ctr, xp) : xm;
                    xp = ((fxg >> c) & 1) ? ctr : xp;
                    ym = ((fy0 >> r) & 1) ? ctr : ym;
                    yp = ((fyg >> r) & 1) ? ctr : yp;
                }
                s[2 * r + c] = (xm + xp) + (ym + yp);
            }
        }
    }

    // Horner in L: o = base + cs (inplane + zm + zp - 6 C)
    // S form:      o = (inplane + zm + zp) + cs base
    __device__ __forceinline__ void stage(const double (&C)[8], const double (&T)[2], const double (&B)[2],
                                          const double (&zm)[8], const double (&zp)[8], const double (&bs)[8],
                                          double cs, double (&o)[8]) const {
        double s[8];
        inplane(C, T, B, s);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (PIRK_STRIP_SFORM)
                o[i] = fma(cs, bs[i], s[i] + (zm[i] + zp[i]));
            else
                o[i] = fma(cs, fma(-6.0, C[i], s[i] + (zm[i] + zp[i])), bs[i]);
        }
    }

    // One plane of the pipeline.  edge: the iteration touches a chunk edge or
    // an insulated z face (validity and face tests, uniform branches).
    template <int PH>
    __device__ __forceinline__ void iteration(int j, bool edge) {
        // x(q) in TMEM slot kSX + (q & 1); u1(q) in kSU1 + (q & 1); u2(q) in kSU2 + (q & 1)
        constexpr int XA = kSX + PH, XB = kSX + (PH ^ 1);      // x(j-2), x(j-3)
        constexpr int U1A = kSU1 + PH, U1B = kSU1 + (PH ^ 1);  // u1(j-2), u1(j-3)
        constexpr int U2A = kSU2 + (PH ^ 1), U2B = kSU2 + PH;  // u2(j-3), u2(j-4)
        const bool v1 = !edge || (j - 1 >= zs + lo_shift && j - 1 < ze - hi_shift);
        const bool v2 = !edge || (j - 2 >= zs + 2 * lo_shift && j - 2 < ze - 2 * hi_shift);
        const bool v3 = !edge || (j - 3 >= zs + 3 * lo_shift && j - 3 < ze - 3 * hi_shift);
        const bool v4 = !edge || (j - 4 >= ob && j - 4 < oe);
        const bool a4 = !edge || (v3 && j - 3 >= ob && j - 3 < oe);  // A4(j-3) needed next iteration
        const bool has_x = !edge || j < ze;

        if constexpr (!PIRK_TM_LD_WAITST) tm_wait_st();  // the previous plane's TMEM stores land before its slots are read
        const bool early = PIRK_STRIP_EARLYLD && PIRK_STRIP_XSWAP && !edge;
        unsigned er[48];
        if (early) tm_ld8x3_issue(ts(XB), ts(XA), ts(U1B), er);
        // ---- x(j): wait for its box; prefetch x(j+2) into the slot of x(j-2)
        const double* Xj = xslot(xs);
        const double* Xm = xslot((xs + 3) & 3);  // x(j-1)
        // split barrier: the previous plane's arrivals (completion j-1-zs)
        // (ladder: done[1] / done[2] complete when every warp has published
        // level 1 / level 2 of a plane, so a fast warp waits only for the
        // exchange rows it is about to overwrite)
        auto wait_bar = [&](int b) {
            if (PIRK_STRIP_SPLITBAR && j > zs) mbar_wait(done + b, static_cast<unsigned>(j - 1 - zs) & 1u);
        };
        auto wait_prev = [&]() { wait_bar(PIRK_STRIP_LADDER ? 1 : 0); };
        auto arrive = [&](int b) {
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(done + b);
        };
        if (has_x) {  // issue first: a late x(j) must not delay the prefetch behind it
            if (PIRK_STRIP_LADDER < 2 && threadIdx.x == 0 && (!edge || j + 2 < ze)) {
                wait_bar(0);  // the target slot (x(j-2)) was read in the previous iteration
                tma(j + 2, (xs + 2) & 3);
            }
            if (PIRK_STRIP_L2PF > 0 && threadIdx.x == 0 && j + 2 + PIRK_STRIP_L2PF < ze)
                tma_prefetch_l2(tmap, bx0, by0, j + 2 + PIRK_STRIP_L2PF - wbz);  // warm L2 further ahead
            mbar_wait(bars + xs, (xph >> xs) & 1);
        }

        // ---- stage 1 at p = j-1: centre and base x(j-1), z- x(j-2), z+ x(j)
        double o1[8], zm2[8];
        double xb[8];  // XSWAP: x(j-3), the base of stage 3, read before x(j-1) replaces it
        if (v1) {
            double C[8], zm[8], zp[8], T[2], B[2];
            if (PIRK_STRIP_XCARRY && !edge) {
#pragma unroll
                for (int i = 0; i < 8; ++i) C[i] = xc[i];
            } else {
                own_x(Xm, C);
            }
            if (early) {
                tm_ld_wait48(er);
                tm_unpack8(er, xb);
                tm_unpack8(er + 16, zm);
                tm_unpack8(er + 32, zm2);
                st8(ts(XB), C);  // x(j-1) replaces x(j-3)
            } else {
                if constexpr (PIRK_STRIP_XSWAP) {
                    tm_ld8(ts(XB), xb);
                    st8(ts(XB), C);  // x(j-1) replaces x(j-3)
                }
                tm_ld8x2(ts(XA), ts(U1B), zm, zm2);  // x(j-2); u1(j-3) before it is overwritten
            }
            if (!edge || j < g) {
                own_x(Xj, zp);
            } else {  // x(g) := x(g-1)
#pragma unroll
                for (int i = 0; i < 8; ++i) zp[i] = C[i];
            }
            if constexpr (PIRK_STRIP_XCARRY) {
#pragma unroll
                for (int i = 0; i < 8; ++i) xc[i] = zp[i];  // (beyond g only edge iterations follow)
            }
            if (edge && j - 1 == 0) {  // x(-1) := x(0)
#pragma unroll
                for (int i = 0; i < 8; ++i) zm[i] = C[i];
            }
            x_tb(Xm, T, B);
            stage(C, T, B, zm, zp, C, cst(0), o1);
            st8(ts(U1B), o1);  // u1(j-1) replaces u1(j-3)
            wait_prev();  // every warp is past the previous plane's exchange reads
            publish(PH, 0, o1);
        } else {
            if constexpr (PIRK_STRIP_XSWAP) {
                double w[8];
                tm_ld8(ts(XB), xb);
                own_x(Xm, w);
                st8(ts(XB), w);
            }
            if (PIRK_STRIP_XCARRY && has_x) own_x(Xj, xc);  // (only edge iterations get here)
            wait_prev();
            if (v2) tm_ld8(ts(U1B), zm2);
        }
        // ---- stage 2 at p = j-2: centre u1(j-2), z- u1(j-3), z+ u1(j-1), base x(j-2)
        double o2[8], zm3[8];
        if (v2) {
            double C[8], bs[8], T[2], B[2];
            tm_ld8x2(ts(U1A), ts(XA), C, bs);
            tm_ld8(ts(U2B), zm3);  // u2(j-4) before it is overwritten
            if (edge && j - 2 == 0) {  // u1(-1) := u1(0)
#pragma unroll
                for (int i = 0; i < 8; ++i) zm2[i] = C[i];
            }
            if (edge && j - 2 == g - 1) {  // u1(g) := u1(g-1)
#pragma unroll
                for (int i = 0; i < 8; ++i) o1[i] = C[i];
            }
            u_tb(PH ^ 1, 0, T, B);
            stage(C, T, B, zm2, o1, bs, cst(1), o2);
            st8(ts(U2B), o2);  // u2(j-2) replaces u2(j-4)
            if (PIRK_STRIP_LADDER) wait_bar(2);
            publish(PH, 1, o2);
        } else {
            if (PIRK_STRIP_LADDER) wait_bar(2);
            if (v3) tm_ld8(ts(U2B), zm3);
        }
        if (PIRK_STRIP_LADDER) arrive(1);
        // ---- stage 3 at p = j-3: centre u2(j-3), z- u2(j-4), z+ u2(j-2), base x(j-3)
        double o3[8], C4[8], av[8];
        const bool s4 = (v4 || a4) && inner;     // halo warps 0 and 15 never run stage 4
        if (s4) tm_ld8(ts(kSU3), C4);  // u3(j-4) before it is overwritten
        if (v3) {
            double C[8], bs[8], T[2], B[2];
            if constexpr (PIRK_STRIP_XSWAP) {
                tm_ld8(ts(U2A), C);
#pragma unroll
                for (int i = 0; i < 8; ++i) bs[i] = xb[i];
            } else {
                tm_ld8x2(ts(U2A), ts(XB), C, bs);
            }
            if (edge && j - 3 == 0) {
#pragma unroll
                for (int i = 0; i < 8; ++i) zm3[i] = C[i];
            }
            if (edge && j - 3 == g - 1) {
#pragma unroll
                for (int i = 0; i < 8; ++i) o2[i] = C[i];
            }
            u_tb(PH ^ 1, 1, T, B);
            stage(C, T, B, zm3, o2, bs, cst(2), o3);
            if (inner) st8(ts(kSU3), o3);  // u3(j-3) replaces u3(j-4)
            if (PIRK_STRIP_LADDER) wait_bar(0);
            publish(PH, 2, o3);
            if (PIRK_STRIP_XSWAP && s4) {  // A4(j-3) = x(j-3) + c4 (u3(j-4) - 6 u3(j-3)); A4(j-4) first
                if (edge && j - 3 == 0) {  // u3(-1) := u3(0) (stage 4 does not run)
#pragma unroll
                    for (int i = 0; i < 8; ++i) C4[i] = o3[i];
                }
                tm_ld8(ts(kSA4), av);
                if (a4) {
                    double an[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) an[i] = a4_of(C4[i], o3[i], bs[i]);
                    st8(ts(kSA4), an);
                }
            }
        } else if (PIRK_STRIP_LADDER) {
            wait_bar(0);
        }
        if (PIRK_STRIP_LADDER == 2 && has_x && threadIdx.x == 0 && (!edge || j + 2 < ze))
            tma(j + 2, (xs + 2) & 3);  // every warp is past the previous plane: its x slot is free
        if (PIRK_STRIP_LADDER) arrive(2);
        // ---- stage 4 at p = j-4: y = A4(j-4) + c4 (inplane(u3(j-4)) + u3(j-3)) to
        // HBM; A4(j-3) = x(j-3) + c4 (u3(j-4) - 6 u3(j-3)); x(j-1) replaces x(j-3)
        if (s4) {
            double x3[8];
            if constexpr (PIRK_STRIP_XSWAP) {
                if (!v3) tm_ld8(ts(kSA4), av);  // (a4 implies v3)
            } else {
                tm_ld8x2(ts(kSA4), ts(XB), av, x3);
            }
            if (edge && j - 4 == g - 1) {  // u3(g) := u3(g-1) (stage 3 did not run)
#pragma unroll
                for (int i = 0; i < 8; ++i) o3[i] = C4[i];
            }
            if (!PIRK_STRIP_XSWAP && edge && j - 3 == 0) {  // u3(-1) := u3(0) (stage 4 does not run)
#pragma unroll
                for (int i = 0; i < 8; ++i) C4[i] = o3[i];
            }
            if (v4) {
                double T[2], B[2], s[8], y[8];  // (halo lanes compute garbage, store nothing)
                u_tb(PH ^ 1, 2, T, B);
                inplane(C4, T, B, s);
#pragma unroll
                for (int i = 0; i < 8; ++i) y[i] = fma(c4(), s[i] + o3[i], av[i]);
                if (st_own) {
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        *reinterpret_cast<double2*>(stp + r * g) = make_double2(y[2 * r], y[2 * r + 1]);
                } else if (st_mask) {
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if ((st_mask >> i) & 1) stp[(i >> 1) * g + (i & 1)] = y[i];
                }
                if constexpr (Mirror) {  // the same cells into the neighbours' halos, over peer memory
                    const unsigned mk = st_own ? 0xffu : st_mask;
                    if (j - 4 < m_lo_end) {
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            if ((mk >> i) & 1) mtp[(i >> 1) * g + (i & 1)] = y[i];
                    }
                    if (j - 4 >= m_hi_begin) {
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            if ((mk >> i) & 1) mhp[(i >> 1) * g + (i & 1)] = y[i];
                    }
                }
                if ((st_own || st_mask) &&
                    (PIRK_STRIP_F32CHK ? maybe_nonfinite8(y)
                                       : !finite_d(((y[0] + y[1]) + (y[2] + y[3])) + ((y[4] + y[5]) + (y[6] + y[7])))))
                    heat_strip_report(stp, g, g2, j - 4, gout, st_own ? 0xffu : st_mask, field, method, step,
                                      fail, n_total);
            }
            if (!PIRK_STRIP_XSWAP && a4) {
                double an[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) an[i] = a4_of(C4[i], o3[i], x3[i]);
                st8(ts(kSA4), an);
            }
        }
        if constexpr (!PIRK_STRIP_XSWAP) {
            double w[8];
            own_x(Xm, w);
            st8(ts(XB), w);  // x(j-1) replaces x(j-3)
        }
        if (has_x) {
            xph ^= 1 << xs;
            xs = (xs + 1) & 3;
        }
        stp += g2;
        if constexpr (Mirror) {
            mtp += g2;
            mhp += g2;
        }
        // one barrier per plane: this iteration's rows (buffer j & 1) become
        // readable, and the next iteration may overwrite buffer (j - 1) & 1
        if constexpr (PIRK_STRIP_SPLITBAR) {
            arrive(0);
        } else {
            __syncthreads();
        }
    }

    __device__ __forceinline__ void one(int j, bool edge) {
        if (j & 1)
            iteration<1>(j, edge);
        else
            iteration<0>(j, edge);
    }

    __device__ __forceinline__ void run() {
        xs = 0;
        xph = 0;
        if (threadIdx.x == 0) {
            if (zs < ze) tma(zs, 0);
            if (zs + 1 < ze) tma(zs + 1, 1);
        }
        const int jend = ze + 4;
        // steady state: all stages valid, planes j-5 .. j clear of the z faces
        // (heat.cuh's bounds) and x(j+2) inside the window
        int a = zs + 3 + 3 * lo_shift;
        if (a < ob + 4) a = ob + 4;
        if (a < 5) a = 5;
        int bnd = ze - 2;
        if (bnd > oe + 4) bnd = oe + 4;
        if (bnd > g) bnd = g;
        if (bnd < a) bnd = a;
        int j = zs;
        for (; j < a && j < jend; ++j) one(j, true);
        if ((j & 1) && j < bnd) iteration<1>(j++, false);
        for (; j + 1 < bnd; j += 2) {
            iteration<0>(j, false);
            iteration<1>(j + 1, false);
        }
        for (; j < jend; ++j) one(j, j >= bnd);
    }
};

template <bool Exact, bool One = false, bool Mirror = false>
__global__ void __launch_bounds__(kSThreads, 1)
heat_strip_kernel(const HeatModel m, const HeatStepParams hp, const WindowArgs w, const StepConsts sc,
                  const unsigned long long step, const uint64_t zchunk,
                  unsigned long long* __restrict__ fail, const __grid_constant__ HeatTmaps tm, const int flags) {
    static_assert(!Exact, "heat_strip_kernel is the fast-mode kernel");
    (void)sizeof(ModeCheck<Exact>);
    (void)sc;
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) unsigned long long bars[kSXSlots];
    __shared__ __align__(8) unsigned long long done_bar[3];
    __shared__ unsigned tmem_base;
    const int tid = threadIdx.x;
    const long long g = static_cast<long long>(m.g);
    // One: a single field (index in flags bit 3) per launch, grid z = chunks
    // (field-pipelined runs); a separate instantiation, so the two-field
    // kernel is untouched
    const int field = One ? ((flags >> 3) & 1) : static_cast<int>(blockIdx.z & 1);
    const long long chunk = One ? static_cast<long long>(blockIdx.z) : static_cast<long long>(blockIdx.z >> 1);
    const long long ix0 = static_cast<long long>(blockIdx.x) * kST;
    const long long iy0 = static_cast<long long>(blockIdx.y) * kST;
    const long long obz = static_cast<long long>(w.out_begin) + chunk * static_cast<long long>(zchunk);
    long long oez = obz + static_cast<long long>(zchunk);
    if (oez > static_cast<long long>(w.out_end)) oez = static_cast<long long>(w.out_end);
    if (obz >= oez) return;

    const int warp = tid >> 5, lane = tid & 31;
    const long long gx0 = ix0 - kHeatH + 2 * lane, gy0 = iy0 - kHeatH + 4 * warp;
    const bool own = lane >= 2 && lane <= 29 && warp >= 1 && warp <= 14;
    const bool interior = ix0 - kHeatH >= 0 && ix0 + kST + kHeatH <= g && iy0 - kHeatH >= 0 &&
                          iy0 + kST + kHeatH <= g;
    unsigned st_mask = 0;
    int fx0 = 0, fxg = 0, fy0 = 0, fyg = 0;
    for (int c = 0; c < 2; ++c) {
        fx0 |= (gx0 + c == 0) << c;
        fxg |= (gx0 + c == g - 1) << c;
    }
    for (int r = 0; r < 4; ++r) {
        fy0 |= (gy0 + r == 0) << r;
        fyg |= (gy0 + r == g - 1) << r;
    }
    if (own) {
        for (int i = 0; i < 8; ++i) {
            const long long x = gx0 + (i & 1), y = gy0 + (i >> 1);
            if (x >= 0 && x < g && y >= 0 && y < g) st_mask |= 1u << i;
        }
    }
    const bool st_own = own && st_mask == 0xffu && (flags & 2);
    if (st_own) st_mask = 0;  // vector path
    const int gout = (gx0 >= 0 && gy0 >= 0) ? static_cast<int>(gy0 * g + gx0) : 0;

    const long long g2 = g * g;
    const int zs = static_cast<int>((obz - kHeatH > 0) ? obz - kHeatH : 0);
    const int ze = static_cast<int>((oez + kHeatH < g) ? oez + kHeatH : g);
    double* dst = (field ? w.out1 : w.out0) - static_cast<long long>(w.out_begin) * g2;
    double* mdst = Mirror ? (field ? w.mir1 : w.mir0) - static_cast<long long>(w.out_begin) * g2 : nullptr;
    double* mhdst = Mirror ? (field ? w.mirh1 : w.mirh0) - static_cast<long long>(w.out_begin) * g2 : nullptr;
    const MirrorLimits mlim = MirrorLimits::of(w);

    if (warp == 0) tmem_alloc512(&tmem_base);
    if (tid == 0) {
        for (int s = 0; s < kSXSlots; ++s) mbar_init(bars + s, 1);
        for (int b = 0; b < 3; ++b) mbar_init(done_bar + b, kSThreads / 32);
        mbar_fence_init();
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    // warp w: TMEM lane quadrant w % 4, columns 128 (w / 4) .. +127 (8 slots of 16)
    // (through a warp reduction: its result lives in a uniform register, so the
    // TMEM addresses of the loop's tcgen05 ops need no per-use R2UR)
    const unsigned tt = __reduce_or_sync(0xffffffffu, tmem_base + (static_cast<unsigned>(32 * (warp & 3)) << 16) +
                                                          static_cast<unsigned>(128 * (warp >> 2)));
#define PIRK_STRIP_RUN(INTERIOR)                                                                     \
    {                                                                                                \
        HeatStrip<INTERIOR, Mirror> r{hp};                                                           \
        r.EX = reinterpret_cast<double2*>(smem);                                                     \
        r.XR = smem + kSEdgeBytes / sizeof(double);                                                  \
        r.t = tid;                                                                                   \
        r.inner = !PIRK_STRIP_S4SKIP || (warp >= 1 && warp <= 14);                                   \
        r.xo = 4 * warp * kSF + 2 * lane;                                                            \
        r.zs = zs, r.ze = ze, r.ob = static_cast<int>(obz), r.oe = static_cast<int>(oez);           \
        r.g = static_cast<int>(g), r.lo_shift = zs > 0, r.hi_shift = ze < g;                         \
        r.g2 = g2;                                                                                   \
        r.gout = gout;                                                                               \
        r.stp = dst + static_cast<long long>(zs - 4) * g2 + gout;                                    \
        if constexpr (Mirror) {                                                                      \
            r.mtp = mdst + static_cast<long long>(zs - 4) * g2 + gout;                               \
            r.mhp = mhdst + static_cast<long long>(zs - 4) * g2 + gout;                              \
            r.m_lo_end = mlim.lo_end, r.m_hi_begin = mlim.hi_begin;                                  \
        }                                                                                            \
        r.st_own = st_own, r.st_mask = st_mask;                                                      \
        r.fx0 = fx0, r.fxg = fxg, r.fy0 = fy0, r.fyg = fyg;                                          \
        r.field = field, r.method = m.method, r.step = step, r.fail = fail;                          \
        r.n_total = static_cast<unsigned long long>(g2 * g);                                         \
        r.tmap = &tm.f[field];                                                                       \
        r.bx0 = static_cast<int>(ix0) - kHeatH, r.by0 = static_cast<int>(iy0) - kHeatH;              \
        r.wbz = static_cast<int>(w.win_begin);                                                       \
        r.bars = bars;                                                                               \
        r.done = done_bar;                                                                           \
        r.tt = tt;                                                                                   \
        r.run();                                                                                     \
    }
#if defined(PIRK_STRIP_TIMING_ONLY_INTERIOR)  // A/B timing only: every tile runs the interior code (wrong at edges)
    PIRK_STRIP_RUN(0)
#elif defined(PIRK_STRIP_TIMING_SKIP_EDGES)  // A/B timing only: edge tiles do nothing
    if (interior) PIRK_STRIP_RUN(0)
#elif defined(PIRK_STRIP_TIMING_NO_KIND2)  // A/B timing only: no generic edge path (g % 4 == 0 only)
    if (interior) PIRK_STRIP_RUN(0)
    else PIRK_STRIP_RUN(1)
#else
    if (interior) PIRK_STRIP_RUN(0)
    else if (PIRK_STRIP_EDGECSE && g % 4 == 0) PIRK_STRIP_RUN(1)
    else PIRK_STRIP_RUN(2)
#endif
#undef PIRK_STRIP_RUN
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc512(tmem_base);
}

}  // namespace pirk
