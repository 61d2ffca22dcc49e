// heat4x4.cuh -- K2 v15 (fast mode): the heat3d RK4 step with 4x4 register
// blocks, z-histories in TMEM and the in-plane exchange through SoA edge arrays.
//
// Replaces integrate_step (rk4.cpp:30-76) on the heat3d embedding / growth
// pair exactly as heat.cuh does (models.cpp:92-133; both fields evolve
// independently under the same linear 7-point operator), held to the fast-mode
// contract (relative <= 1e-12, never tighter; tests/helpers.assert_within).
//
// Why a third variant.  The 1x2 / 2x2 kernels are bound by shared-memory
// wavefronts (~1.4 per state-update, 67% of the crossbar at g=800 in
// profiles/r01_heat_v14_g800.txt), because every stage value of every point is
// stored to shared memory and 2-3 neighbours are read back per point.  With a
// 4x4 block per thread only the block perimeter is exchanged: per stage a
// thread publishes its four edges (16 values) and reads the four facing edges
// of its neighbours (16 values) for 16 points.  The cost is state: a block's
// z-history is 8 planes x 16 doubles, which does not fit in registers, so it
// lives in tensor memory (TMEM).  Measured on this B200 (tools/tmem_bw.cu):
// tcgen05.ld moves ~430 B/clk/SM and tcgen05.st ~360 B/clk/SM, against 128 B/clk
// for the shared-memory crossbar -- TMEM is the cheap place for per-thread
// pipeline state.
//
// Geometry.  A CTA (one per SM: 226 KB of shared memory, all 512 TMEM columns)
// owns a 56x56 x-y tile of one field and streams the planes of a z-chunk; its
// footprint with the 4-cell halo is 64x64 = 16x16 blocks, one per thread.
// Ring blocks (the outermost block ring) recompute stages 1-3 of the halo; own
// blocks (the inner 14x14) also run stage 4 and store to HBM.  Every thread runs
// the same code; only the HBM store is predicated.
//
// Pipeline.  Iteration j reads x-plane j (64x64 footprint, zero-filled
// outside the grid, 4-slot ring, fetched 2 planes ahead) and evaluates stage
// 1 at plane j-1, stage 2 at j-2, stage 3 at j-3 and stage 4 at j-4 -- the
// lagged schedule of heat.cuh.  Fast mode evaluates RK4 for this linear
// autonomous field in Horner form, x + hL(x + hL/2(x + hL/3(x + hL/4 x))), so a
// stage is v_s = x + c_s (sum6(v_{s-1}) - 6 v_{s-1}), c = hk*kk/{4,3,2,1}.
// Stage 4's z- and centre terms are folded one iteration early into
// A4(p) = x(p) + c4 (u3(p-1) - 6 u3(p)), so x(p) and u3(p-1) need no slot.
// TMEM slots (32 columns = one 4x4 plane of doubles each): x(j-2), x(j-3),
// u1(j-2), u1(j-3), u2(j-3), u2(j-4), u3(j-4), A4(j-4); x(j-1) and x(j) are
// read from the x ring.  Planes stream through the stages in row pairs, each
// consumed row pair of a dying slot being overwritten by the new plane's.
//
// x planes.  Block-major: block b's 16 values occupy 128 contiguous bytes, its
// eight 16-byte chunks (row r, half h: q = 2r + h) swizzled to positions
// q ^ (b & 7), which makes a warp's reads of its own blocks (and, in stage 1,
// of the neighbours' facing edges) conflict-free or 2-way at worst.  TMA
// cannot produce this layout (a 5-D block view has 32-byte inner rows, which
// the 128-byte swizzle pads to 128 bytes each), so the planes arrive by
// cp.async: each warp copies whole 512-byte footprint rows (coalesced, 16
// bytes per lane; zero-filled outside the grid) into their swizzled places.
//
// Exchange.  Three levels (u1, u2, u3) of edge arrays in shared memory, each
// eight SoA arrays of double2 indexed by block: N (row 0), W (column 0), E
// (column 3), S (row 3), low and high halves.  Lane i of a warp handles block
// 32w + i, so every edge load and store is a conflict-free 16-byte access.
// Phase A (all four stages) reads the levels published in the previous
// iteration; after a barrier, phase B publishes this iteration's u1(j-1),
// u2(j-2), u3(j-3) into the same arrays; a second barrier closes the plane.
//
// Arithmetic (fast mode).  Interior tiles share the in-plane pair sums along
// anti-diagonals: with P(r,c) = v(r,c+1) + v(r+1,c), point (r,c) sums
// P(r,c) + P(r-1,c-1), about 4.4 DADD + 2 DFMA per point-stage.  Edge tiles
// substitute ghost values per point (Robin at x = 0, insulated elsewhere) as
// heat_pt does.  Insulated z faces replicate the boundary plane, as heat.cuh.
#pragma once

#include "heat.cuh"
#include "tmem_io.cuh"
#if !PIRK_TM_LD_WAITST
#error "heat4x4.cuh relies on per-load store waits: build dev variants with -DPIRK_TM_LD_WAITST=1"
#endif

namespace pirk {

constexpr int k4T = 56;             // output tile edge
constexpr int k4F = 64;             // footprint edge
constexpr int k4Threads = 256;      // one 4x4 block per thread (16 x 16 blocks)
constexpr int k4XSlots = 4;         // x planes j-1 .. j+2
constexpr int k4XSlot = k4F * k4F;  // doubles per x slot (block-major, swizzled)
constexpr int k4Arr = 256;          // double2 entries per edge array
constexpr int k4Level = 8 * k4Arr;  // double2 entries per exchange level
constexpr int k4Levels = 3;         // u1, u2, u3
constexpr size_t k4LevelBytes = size_t(k4Level) * sizeof(double2);            // 32 KB
constexpr size_t k4RingBytes = size_t(k4XSlots) * k4XSlot * sizeof(double);    // 128 KB
// [u1 edges][<= 1 KB alignment gap][x ring, 1024-byte aligned][u2, u3 edges]
constexpr size_t k4SmemBytes = k4Levels * k4LevelBytes + k4RingBytes + 1024;  // 230,400 B

// Edge arrays of a level, lo half at +0 and hi half at +1.  Ring blocks read
// past the footprint (b-1, b+1, b-16, b+16); in this order those reads land in
// a neighbouring array of the same level: N is read at b+16 (next array), W at
// b+1, E at b-1, S at b-16 (previous array).  The x ring sits between edge
// levels, so its reads at blocks -17 .. 271 stay inside the allocation too.
enum : int { kEN = 0, kEW = 2, kEE = 4, kES = 6 };

// TMEM plane slots of a thread (32 columns each)
enum : int { kTX = 0, kTU1 = 2, kTU2 = 4, kTU3 = 6, kTA4 = 7 };

// 16-byte chunk q (row q >> 1, columns 2(q & 1) .. +1) of block b in a
// swizzled x slot
__device__ __forceinline__ const double* xchunk(const double* X, int b, int q) {
    return X + b * 16 + ((q ^ (b & 7)) << 1);
}

// 16-byte global -> shared copy, zero-filled when !valid (L2 only: each x
// value is read by exactly one CTA's copy, halo re-reads aside)
__device__ __forceinline__ void cp_async16(double* dst, const double* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Non-finite output at plane p (cold path): read the block's stored cells back
// and record each bad one (atomicMin keeps the lowest component).
__device__ __forceinline__ void heat4_report(const double* stp, int g, long long g2, int p, int gout,
                                             unsigned mask, int field, int method, unsigned long long step,
                                             unsigned long long* fail, unsigned long long n_total) {
#pragma unroll 1
    for (int i = 0; i < 16; ++i) {
        const int r = i >> 2, c = i & 3;
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

template <bool Interior>
struct Heat4Run {
    const HeatStepParams& hp;
    double2* __restrict__ E1;  // u1 edge level
    double2* __restrict__ E23; // u2, u3 edge levels
    double* __restrict__ XR;   // x ring
    int b;                     // block = thread index
    int zs, ze, ob, oe, g, lo_shift, hi_shift;
    long long g2;
    double* __restrict__ stp;  // output plane j-4 at the own block's (0,0)
    bool st_own;               // own block with all 16 cells in the grid (vector stores)
    unsigned st_mask;          // edge tiles: per-cell store mask (bit 4r+c)
    int gout;                  // in-plane global offset of the block's (0,0) cell
    int fx0, fxg, fy0, fyg;    // edge tiles: masks of columns at x=0 / x=g-1, rows at y=0 / y=g-1
    int field, method;
    unsigned long long step;
    unsigned long long* fail;
    unsigned long long n_total;
    // x copies: this thread moves chunk `lane` of footprint rows warp + 8k
    const double* ldp;         // plane j+2 (the next plane to fetch)
    long long coff;            // in-plane offset of this thread's first row / chunk
    int cdst;                  // shared offset (doubles) of the first chunk in a slot
    unsigned cvalid;           // bit k: row warp + 8k inside the grid (and chunk column too)
    unsigned tt;  // TMEM address of slot 0
    int xs;       // x ring slot of plane j

    __device__ __forceinline__ unsigned ts(int slot) const { return tt + 32u * slot; }
    __device__ __forceinline__ double* xslot(int s) const { return XR + s * k4XSlot; }

    // copy the footprint of the plane at ldp into ring slot s (one commit group)
    __device__ __forceinline__ void fetch(int s) {
        double* X = xslot(s) + cdst;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            cp_async16(X + 512 * k, (cvalid >> k) & 1 ? ldp + coff + 8 * k * static_cast<long long>(g) : ldp,
                       (cvalid >> k) & 1);
        cp_async_commit();
        ldp += g2;
    }

    // rows 2rp, 2rp+1 of the own block in x slot X
    __device__ __forceinline__ void own_rows(const double* X, int rp, double (&v)[8]) const {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 a = *reinterpret_cast<const double2*>(xchunk(X, b, 4 * rp + q));
            v[2 * q] = a.x;
            v[2 * q + 1] = a.y;
        }
    }
    __device__ __forceinline__ void own_plane(const double* X, double (&v)[16]) const {
        double a[8], c[8];
        own_rows(X, 0, a);
        own_rows(X, 1, c);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = a[k], v[8 + k] = c[k];
    }

    // Neighbour edges of rows 2rp, 2rp+1: the left / right neighbours' facing
    // columns and the row above (rp == 0) or below (rp == 1).  Levels 0-2 are
    // u1-u3 in the edge arrays; stage 1 reads the x slot directly (xring).
    __device__ __forceinline__ void edges(int level, int rp, double (&l)[2], double (&r)[2],
                                          double (&ud)[4]) const {
        const double2* A = level == 0 ? E1 : E23 + (level - 1) * k4Level;
        const double2 e = A[(kEE + rp) * k4Arr + b - 1];
        const double2 w = A[(kEW + rp) * k4Arr + b + 1];
        l[0] = e.x, l[1] = e.y, r[0] = w.x, r[1] = w.y;
        if (rp == 0) {  // row above: S row of block b-16
            const double2 s0 = A[kES * k4Arr + b - 16], s1 = A[(kES + 1) * k4Arr + b - 16];
            ud[0] = s0.x, ud[1] = s0.y, ud[2] = s1.x, ud[3] = s1.y;
        } else {  // row below: N row of block b+16
            const double2 n0 = A[kEN * k4Arr + b + 16], n1 = A[(kEN + 1) * k4Arr + b + 16];
            ud[0] = n0.x, ud[1] = n0.y, ud[2] = n1.x, ud[3] = n1.y;
        }
    }
    __device__ __forceinline__ void xedges(const double* X, int rp, double (&l)[2], double (&r)[2],
                                           double (&ud)[4]) const {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int y = 2 * rp + q;
            l[q] = xchunk(X, b - 1, 2 * y + 1)[1];  // (y, 3) of the left block
            r[q] = xchunk(X, b + 1, 2 * y)[0];      // (y, 0) of the right block
        }
        const int nb = rp == 0 ? b - 16 : b + 16;
        const int q0 = rp == 0 ? 6 : 0;  // row 3 of the block above, row 0 of the one below
        const double2 a = *reinterpret_cast<const double2*>(xchunk(X, nb, q0));
        const double2 c = *reinterpret_cast<const double2*>(xchunk(X, nb, q0 + 1));
        ud[0] = a.x, ud[1] = a.y, ud[2] = c.x, ud[3] = c.y;
    }

    __device__ __forceinline__ void publish(int level, const double (&v)[16]) const {
        double2* A = level == 0 ? E1 : E23 + (level - 1) * k4Level;
        A[kEN * k4Arr + b] = make_double2(v[0], v[1]);
        A[(kEN + 1) * k4Arr + b] = make_double2(v[2], v[3]);
        A[kEW * k4Arr + b] = make_double2(v[0], v[4]);
        A[(kEW + 1) * k4Arr + b] = make_double2(v[8], v[12]);
        A[kEE * k4Arr + b] = make_double2(v[3], v[7]);
        A[(kEE + 1) * k4Arr + b] = make_double2(v[11], v[15]);
        A[kES * k4Arr + b] = make_double2(v[12], v[13]);
        A[(kES + 1) * k4Arr + b] = make_double2(v[14], v[15]);
    }

    // In-plane neighbour sums of rows 2rp, 2rp+1 of centre plane C.  pp
    // carries the anti-diagonal pair sums P(y-1, c-1), c = 0..3, to the next
    // row (interior tiles); P(y, c) = v(y, c+1) + v(y+1, c).
    __device__ __forceinline__ void inplane(int rp, const double (&C)[16], const double (&l)[2],
                                            const double (&r)[2], const double (&ud)[4], double (&pp)[4],
                                            double (&out)[8]) const {
        auto V = [&](int y, int x) -> double {  // y in [2rp-1, 2rp+2], x in [-1, 4]
            if (y < 0 || y > 3) return ud[x];
            if (x < 0) return l[y - 2 * rp];
            if (x > 3) return r[y - 2 * rp];
            return C[4 * y + x];
        };
        if constexpr (Interior) {
            if (rp == 0) {  // P(-1, c-1) = v(-1, c) + v(0, c-1)
#pragma unroll
                for (int c = 0; c < 4; ++c) pp[c] = V(-1, c) + V(0, c - 1);
            } else {  // P(1, -1) = v(1, 0) + v(2, -1): needs this pair's left column
                pp[0] = C[4] + l[0];
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int y = 2 * rp + q;
                double np[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const double pr = V(y, c + 1) + V(y + 1, c);  // P(y, c)
                    out[4 * q + c] = pr + pp[c];
                    if (c < 3) np[c + 1] = pr;
                }
                np[0] = (q == 0) ? V(y, 0) + V(y + 1, -1) : pp[0];  // P(y, -1); q == 1: next pair sets it
#pragma unroll
                for (int c = 0; c < 4; ++c) pp[c] = np[c];
            }
        } else {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int y = 2 * rp + q;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const double s = C[4 * y + c];
                    double xm = V(y, c - 1), xp = V(y, c + 1), ym = V(y - 1, c), yp = V(y + 1, c);
                    xm = ((fx0 >> c) & 1) ? fma(-hp.robin, s, xp) : xm;
                    xp = ((fxg >> c) & 1) ? s : xp;
                    ym = ((fy0 >> y) & 1) ? s : ym;
                    yp = ((fyg >> y) & 1) ? s : yp;
                    out[4 * q + c] = (xm + xp) + (ym + yp);
                }
            }
        }
    }

    // o = base + cs (inplane + zm + zp - 6 C) on row pair rp
    __device__ __forceinline__ void combine(int rp, const double (&C)[16], const double (&s)[8],
                                           const double (&zm)[8], const double (&zp)[8], const double (&bs)[8],
                                           double cs, double (&o)[16]) const {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = 8 * rp + k;
            o[i] = fma(cs, fma(-6.0, C[i], s[k] + (zm[k] + zp[k])), bs[k]);
        }
    }

    // one plane of the pipeline.  edge: the iteration touches a chunk edge or
    // an insulated z face (validity and face tests; uniform branches)
    __device__ __forceinline__ void iteration(int j, bool edge) {
        // x(q) in TMEM slot kTX + (q & 1); u1(q) in kTU1 + (q & 1); u2(q) in kTU2 + (q & 1)
        const int ph = j & 1;
        const unsigned XA = ts(kTX + ph), XB = ts(kTX + (ph ^ 1));      // x(j-2), x(j-3)
        const unsigned U1A = ts(kTU1 + ph), U1B = ts(kTU1 + (ph ^ 1));  // u1(j-2), u1(j-3)
        const unsigned U2A = ts(kTU2 + (ph ^ 1)), U2B = ts(kTU2 + ph);  // u2(j-3), u2(j-4)
        const unsigned U3 = ts(kTU3), A4 = ts(kTA4);
        const bool v1 = !edge || (j - 1 >= zs + lo_shift && j - 1 < ze - hi_shift);
        const bool v2 = !edge || (j - 2 >= zs + 2 * lo_shift && j - 2 < ze - 2 * hi_shift);
        const bool v3 = !edge || (j - 3 >= zs + 3 * lo_shift && j - 3 < ze - 3 * hi_shift);
        const bool v4 = !edge || (j - 4 >= ob && j - 4 < oe);
        const bool a4 = !edge || (v3 && j - 3 >= ob && j - 3 < oe);  // A4(j-3) needed next iteration
        const bool has_x = !edge || j < ze;

        // ---- x(j) landed in the previous iteration; fetch x(j+2) into the slot
        // of x(j-2) (one commit group per iteration, possibly empty)
        const double* Xj = xslot(xs);
        const double* Xm = xslot((xs + 3) & 3);  // x(j-1)
        if (!edge || j + 2 < ze)
            fetch((xs + 2) & 3);
        else
            cp_async_commit();

        // ---- stage 1 at p = j-1: centre and base x(j-1), z- x(j-2), z+ x(j)
        double o1[16];
        if (v1) {
            double C[16], pp[4];
            own_plane(Xm, C);
#pragma unroll
            for (int rp = 0; rp < 2; ++rp) {
                double zm[8], zp[8], bs[8], l[2], r[2], ud[4], s[8];
                tm_ld8(XA + 16 * rp, zm);
#pragma unroll
                for (int k = 0; k < 8; ++k) bs[k] = C[8 * rp + k];
                if (!edge || j < g) {
                    own_rows(Xj, rp, zp);
                } else {  // x(g) := x(g-1)
#pragma unroll
                    for (int k = 0; k < 8; ++k) zp[k] = bs[k];
                }
                if (edge && j - 1 == 0) {  // x(-1) := x(0)
#pragma unroll
                    for (int k = 0; k < 8; ++k) zm[k] = bs[k];
                }
                xedges(Xm, rp, l, r, ud);
                inplane(rp, C, l, r, ud, pp, s);
                combine(rp, C, s, zm, zp, bs, hp.hn[0], o1);
            }
        }
        // ---- stage 2 at p = j-2: centre u1(j-2), z- u1(j-3), z+ u1(j-1), base x(j-2)
        double o2[16];
        {
            double C[16], pp[4];
            if (v2) tm_ld16(U1A, C);
            if (edge && j - 2 == g - 1) {  // u1(g) := u1(g-1)
#pragma unroll
                for (int i = 0; i < 16; ++i) o1[i] = C[i];
            }
#pragma unroll
            for (int rp = 0; rp < 2; ++rp) {
                if (v2) {
                    double zm[8], zp[8], bs[8], l[2], r[2], ud[4], s[8];
                    tm_ld8x2(U1B + 16 * rp, XA + 16 * rp, zm, bs);
#pragma unroll
                    for (int k = 0; k < 8; ++k) zp[k] = o1[8 * rp + k];
                    if (edge && j - 2 == 0) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) zm[k] = C[8 * rp + k];
                    }
                    edges(0, rp, l, r, ud);
                    inplane(rp, C, l, r, ud, pp, s);
                    combine(rp, C, s, zm, zp, bs, hp.hn[1], o2);
                }
                if (v1) {  // u1(j-1) replaces the consumed rows of u1(j-3)
#pragma unroll
                    for (int k = 0; k < 8; ++k) tm_st1(U1B + 16 * rp + 2 * k, o1[8 * rp + k]);
                }
            }
        }
        // ---- stage 3 at p = j-3: centre u2(j-3), z- u2(j-4), z+ u2(j-2), base x(j-3)
        double o3[16];
        {
            double C[16], pp[4];
            if (v3) tm_ld16(U2A, C);
            if (edge && j - 3 == g - 1) {
#pragma unroll
                for (int i = 0; i < 16; ++i) o2[i] = C[i];
            }
#pragma unroll
            for (int rp = 0; rp < 2; ++rp) {
                if (v3) {
                    double zm[8], zp[8], bs[8], l[2], r[2], ud[4], s[8];
                    tm_ld8x2(U2B + 16 * rp, XB + 16 * rp, zm, bs);
#pragma unroll
                    for (int k = 0; k < 8; ++k) zp[k] = o2[8 * rp + k];
                    if (edge && j - 3 == 0) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) zm[k] = C[8 * rp + k];
                    }
                    edges(1, rp, l, r, ud);
                    inplane(rp, C, l, r, ud, pp, s);
                    combine(rp, C, s, zm, zp, bs, hp.hn[2], o3);
                }
                if (v2) {  // u2(j-2) replaces the consumed rows of u2(j-4)
#pragma unroll
                    for (int k = 0; k < 8; ++k) tm_st1(U2B + 16 * rp + 2 * k, o2[8 * rp + k]);
                }
            }
        }
        // ---- stage 4 at p = j-4: y = A4(j-4) + c4 (inplane(u3(j-4)) + u3(j-3)),
        // stored to HBM; A4(j-3) = x(j-3) + c4 (u3(j-4) - 6 u3(j-3)) for the next
        // iteration; x(j-1) replaces x(j-3), u3(j-3) replaces u3(j-4)
        {
            double C[16], pp[4];
            if (v4 || a4) tm_ld16(U3, C);
            // z faces (stage 3 did not run at plane g, stage 4 does not run at -1):
            // o3 is stage 4's z+ and C the z- of A4(j-3)
            if (edge && j - 4 == g - 1) {  // u3(g) := u3(g-1)
#pragma unroll
                for (int i = 0; i < 16; ++i) o3[i] = C[i];
            }
            if (edge && j - 3 == 0) {  // u3(-1) := u3(0)
#pragma unroll
                for (int i = 0; i < 16; ++i) C[i] = o3[i];
            }
            bool bad = false;
#pragma unroll
            for (int rp = 0; rp < 2; ++rp) {
                double av[8], x3[8];
                tm_ld8x2(A4 + 16 * rp, XB + 16 * rp, av, x3);
                if (v4) {
                    double l[2], r[2], ud[4], s[8], y[8];
                    edges(2, rp, l, r, ud);
                    inplane(rp, C, l, r, ud, pp, s);
#pragma unroll
                    for (int k = 0; k < 8; ++k) y[k] = fma(hp.hn[3], s[k] + o3[8 * rp + k], av[k]);
                    double* out = stp + 2 * rp * g;
                    if (st_own) {
                        *reinterpret_cast<double2*>(out) = make_double2(y[0], y[1]);
                        *reinterpret_cast<double2*>(out + 2) = make_double2(y[2], y[3]);
                        *reinterpret_cast<double2*>(out + g) = make_double2(y[4], y[5]);
                        *reinterpret_cast<double2*>(out + g + 2) = make_double2(y[6], y[7]);
                    } else if (st_mask) {
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            if ((st_mask >> (8 * rp + k)) & 1) out[(k >> 2) * g + (k & 3)] = y[k];
                    }
                    if (st_own || st_mask)
                        bad |= !finite_d(((y[0] + y[1]) + (y[2] + y[3])) + ((y[4] + y[5]) + (y[6] + y[7])));
                }
                if (a4) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int i = 8 * rp + k;
                        tm_st1(A4 + 16 * rp + 2 * k, fma(hp.hn[3], fma(-6.0, o3[i], C[i]), x3[k]));
                    }
                }
                {
                    double w[8];
                    own_rows(Xm, rp, w);
#pragma unroll
                    for (int k = 0; k < 8; ++k) tm_st1(XB + 16 * rp + 2 * k, w[k]);  // x(j-1) replaces x(j-3)
                }
                if (v3) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) tm_st1(U3 + 16 * rp + 2 * k, o3[8 * rp + k]);
                }
            }
            if (bad)  // cold path: locate the bad cells
                heat4_report(stp, g, g2, j - 4, gout, st_own ? 0xffffu : st_mask, field, method, step, fail,
                             n_total);
        }
        if (has_x) xs = (xs + 1) & 3;
        __syncthreads();  // phase A's edge reads are complete
        // ---- phase B: publish u1(j-1), u2(j-2), u3(j-3) (back from TMEM: keeping
        // them in registers through phase A would spill)
        if (v1) {
            double t[16];
            tm_ld16(U1B, t);
            publish(0, t);
        }
        if (v2) {
            double t[16];
            tm_ld16(U2B, t);
            publish(1, t);
        }
        if (v3) {
            double t[16];
            tm_ld16(U3, t);
            publish(2, t);
        }
        stp += g2;
        cp_async_wait1();  // x(j+1) landed (only x(j+2)'s group may still be in flight)
        __syncthreads();
    }

    __device__ __forceinline__ void run() {
        xs = 0;
        if (zs < ze) fetch(0); else cp_async_commit();
        if (zs + 1 < ze) fetch(1); else cp_async_commit();
        cp_async_wait1();
        __syncthreads();
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
        const int main_end = bnd;
        int j = zs;
        for (; j < jend; ++j) iteration(j, j < a || j >= main_end);
    }
};

template <bool Exact>
__global__ void __launch_bounds__(k4Threads, 1)
heat4_step_kernel(const HeatModel m, const HeatStepParams hp, const WindowArgs w, const StepConsts sc,
                  const unsigned long long step, const uint64_t zchunk,
                  unsigned long long* __restrict__ fail, const __grid_constant__ HeatTmaps tm, const int flags) {
    static_assert(!Exact, "heat4_step_kernel is the fast-mode kernel");
    (void)sizeof(ModeCheck<Exact>);
    (void)sc;
    extern __shared__ __align__(128) double smem[];
    __shared__ unsigned tmem_base;
    const int tid = threadIdx.x;
    const long long g = static_cast<long long>(m.g);
    const int field = blockIdx.z & 1;
    const long long chunk = blockIdx.z >> 1;
    const long long ix0 = static_cast<long long>(blockIdx.x) * k4T;
    const long long iy0 = static_cast<long long>(blockIdx.y) * k4T;
    const long long obz = static_cast<long long>(w.out_begin) + chunk * static_cast<long long>(zchunk);
    long long oez = obz + static_cast<long long>(zchunk);
    if (oez > static_cast<long long>(w.out_end)) oez = static_cast<long long>(w.out_end);
    if (obz >= oez) return;

    const int bxi = tid & 15, byi = tid >> 4;
    const long long gx0 = ix0 - kHeatH + 4 * bxi, gy0 = iy0 - kHeatH + 4 * byi;
    const bool own = bxi >= 1 && bxi <= 14 && byi >= 1 && byi <= 14;
    const bool interior = ix0 - kHeatH >= 0 && ix0 + k4T + kHeatH <= g && iy0 - kHeatH >= 0 &&
                          iy0 + k4T + kHeatH <= g;
    unsigned st_mask = 0;
    int fx0 = 0, fxg = 0, fy0 = 0, fyg = 0;
    for (int c = 0; c < 4; ++c) {
        fx0 |= (gx0 + c == 0) << c;
        fxg |= (gx0 + c == g - 1) << c;
        fy0 |= (gy0 + c == 0) << c;
        fyg |= (gy0 + c == g - 1) << c;
    }
    if (own) {
        for (int i = 0; i < 16; ++i) {
            const long long x = gx0 + (i & 3), y = gy0 + (i >> 2);
            if (x >= 0 && x < g && y >= 0 && y < g) st_mask |= 1u << i;
        }
    }
    const bool st_own = own && st_mask == 0xffffu && (flags & 2);
    if (st_own) st_mask = 0;  // vector path
    const int gout = (gx0 >= 0 && gy0 >= 0) ? static_cast<int>(gy0 * g + gx0) : 0;

    const long long g2 = g * g;
    const int zs = static_cast<int>((obz - kHeatH > 0) ? obz - kHeatH : 0);
    const int ze = static_cast<int>((oez + kHeatH < g) ? oez + kHeatH : g);
    double* dst = (field ? w.out1 : w.out0) - static_cast<long long>(w.out_begin) * g2;

    // x copies: warp w moves footprint rows w + 8k (k = 0..7), 512 contiguous
    // bytes per row.  Lane l takes half h = (l >> 3) & 1 of row w % 4 of block
    // (l & 7) + 8 (l >> 4): each 8-lane phase writes one half of 8 consecutive
    // blocks, whose swizzled positions differ (conflict-free).  The position is
    // the same for every k; the slot offset advances by 32 blocks per k.
    const int warp = tid >> 5, lane = tid & 31;
    const int cbl = (lane & 7) + 8 * (lane >> 4), chalf = (lane >> 3) & 1;  // block in row, half
    const int cb = (warp >> 2) * 16 + cbl;
    const int cdst = cb * 16 + (((2 * (warp & 3) + chalf) ^ (cb & 7)) << 1);
    const long long cgx = ix0 - kHeatH + 4 * cbl + 2 * chalf, cgy = iy0 - kHeatH + warp;
    unsigned cvalid = 0;
    for (int k = 0; k < 8; ++k)
        if (cgx >= 0 && cgx < g && cgy + 8 * k >= 0 && cgy + 8 * k < g) cvalid |= 1u << k;
    const double* ldp0 = (field ? w.in1 : w.in0) +
                         (static_cast<long long>(zs) - static_cast<long long>(w.win_begin)) * g2;  // plane zs
    if (warp == 0) tmem_alloc512(&tmem_base);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    // warp w: TMEM lane quadrant w % 4, columns 256 (w / 4) .. +255 (8 plane slots)
    // the x ring must start on a 1024-byte boundary: TMA's 128-byte swizzle
    // pattern is a function of the shared address modulo 1024
    double* ring = smem + k4LevelBytes / sizeof(double);
    ring += ((1024u - (smem_u32(ring) & 1023u)) & 1023u) / sizeof(double);
    const unsigned tt = tmem_base + (static_cast<unsigned>(32 * (warp & 3)) << 16) +
                        static_cast<unsigned>(256 * (warp >> 2));
#define PIRK_HEAT4_RUN(INTERIOR)                                                                     \
    {                                                                                                \
        Heat4Run<INTERIOR> r{hp};                                                                    \
        r.E1 = reinterpret_cast<double2*>(smem);                                                     \
        r.XR = ring;                                                                                 \
        r.E23 = reinterpret_cast<double2*>(ring + k4XSlots * k4XSlot);                               \
        r.b = tid;                                                                                   \
        r.zs = zs, r.ze = ze, r.ob = static_cast<int>(obz), r.oe = static_cast<int>(oez);           \
        r.g = static_cast<int>(g), r.lo_shift = zs > 0, r.hi_shift = ze < g;                         \
        r.g2 = g2;                                                                                   \
        r.gout = gout;                                                                               \
        r.stp = dst + static_cast<long long>(zs - 4) * g2 + gout;                                    \
        r.st_own = st_own, r.st_mask = st_mask;                                                      \
        r.fx0 = fx0, r.fxg = fxg, r.fy0 = fy0, r.fyg = fyg;                                          \
        r.field = field, r.method = m.method, r.step = step, r.fail = fail;                          \
        r.n_total = static_cast<unsigned long long>(g2 * g);                                         \
        r.ldp = ldp0, r.coff = cgy * g + cgx, r.cdst = cdst, r.cvalid = cvalid;                      \
        r.tt = tt;                                                                                   \
        r.run();                                                                                     \
    }
    if (interior) PIRK_HEAT4_RUN(true) else PIRK_HEAT4_RUN(false)
#undef PIRK_HEAT4_RUN
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc512(tmem_base);
}

}  // namespace pirk
