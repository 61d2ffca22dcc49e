// user_rt.cuh -- device source (compiled at run time with NVRTC, sm_100a) for
// USER-DEFINED models: the reference's SystemModel with arbitrary std::function
// evaluators (system_model.hpp:14-43) becomes CUDA device functions the caller
// writes, with the same arguments:
//
//   RhsFn     __device__ double pirk_rhs(u64 i, double t, const double* x, const double* p);
//   GrowthFn  __device__ double pirk_growth(u64 i, double t, const double* r, const double* w);
//   DecompFn  __device__ double pirk_decomposition(u64 i, double t, const double* x, const double* p,
//                                                 const double* xh, const double* ph);
//
// (`u64` = unsigned long long; PIRK_N / PIRK_NI are the model's dim and
// input_dim; pirk_min / pirk_max have std::min / std::max semantics.)  The
// library pastes the caller's source between kPrelude and kKernels and
// compiles it with --fmad=false in exact mode (so +,-,*,/ round exactly like
// the reference's non-FMA x86-64 build) or with FMA contraction in fast mode.
//
// Kernels (extern "C", looked up by name):
//   pirk_user_small  -- one thread integrates a whole plan (f, g, or the 2n
//                       embedding), recording slots: the serial loop of
//                       rk4.cpp:30-76 / rk4_serial.cpp, for n <= kUserSmallMax
//   pirk_user_stage  -- one RK4 stage over all components, one thread per
//                       component (any n): 4 launches per step
//   pirk_user_mc     -- Monte Carlo, one sample per thread (reach.cpp:246-323),
//                       hull folded with warp shuffles + ordered-key atomics
//   pirk_user_tile   -- a whole RK4 step per launch for models declared as
//                       radius-r 1-D stencils (pirk_program_set_stencil): a CTA
//                       stages its tile of both fields plus a 4r halo in shared
//                       memory and runs the four stages there (16 B of HBM per
//                       state-update instead of the stage kernels' ~100)
#pragma once

namespace pirk {

// n up to which MM/GB of a user model run as one device thread per integration
constexpr unsigned long long kUserSmallMax = 64;
// Monte Carlo keeps a sample's state in registers/local memory; the failure
// key packs the component into 10 bits
constexpr unsigned long long kUserMcMax = 1024;
// radius-r tile kernel: outputs per CTA and threads; shared memory holds
// 2 fields x 4 arrays (x, u ping-pong, acc) x (kUserTile + 8 r) doubles
constexpr unsigned long long kUserTile = 1024;
constexpr unsigned kUserTileThreads = 256;
constexpr unsigned long long kUserStencilMax = 64;

static const char* kUserPrelude = R"PIRK(
typedef unsigned long long u64;
#define PIRK_DEV __device__ __forceinline__
PIRK_DEV double pirk_min(double a, double b) { return (b < a) ? b : a; }
PIRK_DEV double pirk_max(double a, double b) { return (a < b) ? b : a; }
)PIRK";

static const char* kUserKernels = R"PIRK(
#if !PIRK_HAS_RHS
__device__ double pirk_rhs(u64, double, const double*, const double*) { return 0.0; }
#endif
#if !PIRK_HAS_GROWTH
__device__ double pirk_growth(u64, double, const double*, const double*) { return 0.0; }
#endif
#if !PIRK_HAS_DECOMP
__device__ double pirk_decomposition(u64, double, const double*, const double*, const double*,
                                     const double*) { return 0.0; }
#endif

namespace pirk_rt {

constexpr int kFailCompBits = 40;

PIRK_DEV bool finite_d(double v) {
    const u64 b = (u64)__double_as_longlong(v);
    return ((b >> 52) & 0x7ffull) != 0x7ffull;
}
PIRK_DEV u64 ord_key(double v) {
    const u64 b = (u64)__double_as_longlong(v);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
// rng.hpp:11-29 (integer-only; the draw rounds explicitly, so it is bit-exact
// in both modes)
PIRK_DEV u64 mix64(u64 z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
PIRK_DEV double u01(u64 seed, u64 stream, u64 index) {
    const u64 z = mix64(mix64(mix64(seed) ^ (stream * 0xd1342543de82ef95ull)) ^ (index * 0xaf251af3b0f025b5ull));
    return (double)(z >> 11) * 0x1.0p-53;
}
PIRK_DEV double uniform_in(double lo, double hi, double u) {
    if (lo == hi) return lo;
    return __dadd_rn(lo, __dmul_rn(u, __dsub_rn(hi, lo)));
}
struct StepConsts { double t, hk, h2, h6, th2, thk; };
// rk4.cpp:99-100 and :38-39 with explicit rounding (= the host's values)
PIRK_DEV StepConsts step_consts(double t0, double t1, double h, u64 k, u64 total) {
    StepConsts c;
    c.t = __dadd_rn(t0, __dmul_rn((double)k, h));
    c.hk = (k + 1 == total) ? __dsub_rn(t1, c.t) : h;
    c.h2 = __dmul_rn(0.5, c.hk);
    c.h6 = __ddiv_rn(c.hk, 6.0);
    c.th2 = __dadd_rn(c.t, c.h2);  // stage times t + h2, t + h (rk4.cpp:54-62)
    c.thk = __dadd_rn(c.t, c.hk);
    return c;
}

// which: 0 = rhs under p, 1 = growth under w, 2 = the embedding of
// system_model.cpp:56-77 over S = [x | xh], P = [p | ph]
template <int W>
PIRK_DEV double F(u64 i, double t, const double* S, const double* P) {
    if (W == 0) return pirk_rhs(i, t, S, P);
    if (W == 1) return pirk_growth(i, t, S, P);
    if (i < PIRK_N) return pirk_decomposition(i, t, S, P, S + PIRK_N, P + PIRK_NI);
    return pirk_decomposition(i - PIRK_N, t, S + PIRK_N, P + PIRK_NI, S, P);
}

// one RK4 step over D components held by this thread (rk4.cpp:30-76: every
// stage evaluates all components before the stage state is overwritten);
// returns the lowest non-finite component or -1
template <int W, int D>
PIRK_DEV int serial_step(double* x, double* u, double* k, double* acc, const double* p, const StepConsts& c) {
    for (int i = 0; i < D; ++i) k[i] = F<W>((u64)i, c.t, x, p);
    for (int i = 0; i < D; ++i) { acc[i] = k[i]; u[i] = x[i] + c.h2 * k[i]; }
    for (int i = 0; i < D; ++i) k[i] = F<W>((u64)i, c.th2, u, p);
    for (int i = 0; i < D; ++i) { acc[i] = acc[i] + 2.0 * k[i]; u[i] = x[i] + c.h2 * k[i]; }
    for (int i = 0; i < D; ++i) k[i] = F<W>((u64)i, c.th2, u, p);
    for (int i = 0; i < D; ++i) { acc[i] = acc[i] + 2.0 * k[i]; u[i] = x[i] + c.hk * k[i]; }
    for (int i = 0; i < D; ++i) k[i] = F<W>((u64)i, c.thk, u, p);
    int bad = -1;
    for (int i = 0; i < D; ++i) {
        x[i] = x[i] + c.h6 * (acc[i] + k[i]);
        if (bad < 0 && !finite_d(x[i])) bad = i;
    }
    return bad;
}

template <int W>
__device__ void small_run(const double* x0, const double* p, double t0, double t1, double h, u64 total,
                          u64 stride, double* rec, u64* fail) {
    constexpr int D = (W == 2) ? 2 * PIRK_N : PIRK_N;
    double x[D], u[D], k[D], acc[D];
    for (int i = 0; i < D; ++i) x[i] = x0[i];
    u64 slot = 0;
    if (stride > 0) {
        for (int i = 0; i < D; ++i) rec[i] = x[i];
        slot = 1;
    }
    for (u64 st = 0; st < total; ++st) {
        const StepConsts c = step_consts(t0, t1, h, st, total);
        const int bad = serial_step<W, D>(x, u, k, acc, p, c);
        if (bad >= 0) {  // IntegrationError (rk4.cpp:72-75): stop at the failing step
            atomicMin(fail, (st << kFailCompBits) | (u64)bad);
            return;
        }
        if (st + 1 == total || (stride > 0 && (st + 1) % stride == 0)) {
            for (int i = 0; i < D; ++i) rec[slot * D + i] = x[i];
            ++slot;
        }
    }
}

}  // namespace pirk_rt

extern "C" __global__ void pirk_user_small(int which, const double* x0, const double* p, double t0, double t1,
                                           double h, u64 total, u64 stride, double* rec, u64* fail) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (which == 0) pirk_rt::small_run<0>(x0, p, t0, t1, h, total, stride, rec, fail);
    else if (which == 1) pirk_rt::small_run<1>(x0, p, t0, t1, h, total, stride, rec, fail);
    else pirk_rt::small_run<2>(x0, p, t0, t1, h, total, stride, rec, fail);
}

// One RK4 stage for all D components (one thread each), rk4.cpp:50-75:
//   stage 0: k = F(t, x);      acc = k;          uo = x + h2*k
//   stage 1: k = F(t+h2, ui);  acc = acc + 2k;   uo = x + h2*k
//   stage 2: k = F(t+h2, ui);  acc = acc + 2k;   uo = x + hk*k
//   stage 3: k = F(t+hk, ui);  x = x + h6*(acc + k)   (in place: no thread reads x)
extern "C" __global__ void pirk_user_stage(int which, int stage, double t0, double t1, double h, u64 step,
                                           u64 total, double* x, const double* ui, double* uo, double* acc,
                                           const double* p, u64 D, u64* fail) {
    const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D) return;
    const pirk_rt::StepConsts c = pirk_rt::step_consts(t0, t1, h, step, total);
    const double* S = stage == 0 ? x : ui;
    const double t = stage == 0 ? c.t : (stage == 3 ? c.thk : c.th2);
    double k;
    if (which == 0) k = pirk_rt::F<0>(i, t, S, p);
    else if (which == 1) k = pirk_rt::F<1>(i, t, S, p);
    else k = pirk_rt::F<2>(i, t, S, p);
    if (stage == 0) {
        acc[i] = k;
        uo[i] = x[i] + c.h2 * k;
    } else if (stage < 3) {
        acc[i] = acc[i] + 2.0 * k;
        uo[i] = x[i] + (stage == 1 ? c.h2 : c.hk) * k;
    } else {
        const double xn = x[i] + c.h6 * (acc[i] + k);
        x[i] = xn;
        if (!pirk_rt::finite_d(xn)) atomicMin(fail, (step << pirk_rt::kFailCompBits) | i);
    }
}

// One RK4 step of a radius-R 1-D stencil model (pirk_program_set_stencil): the
// CTA owns outputs [c0, c1) and stages x on [lo, hi) = [c0 - 4R, c1 + 4R) of
// both fields (clamped to the domain).  Stage s is evaluated on the range that
// shrinks by R per stage away from the domain ends (the 4-stage dependency
// cone), in shared memory, with the expressions and stage times of
// pirk_user_stage (rk4.cpp:50-75): bit-identical to it.  The user functions
// see pointers rebased so that x[i] is component i.
//   which 0: f on field 0 (p); 1: g on field 0 (w); 2: the embedding, field 0
//   = x under d(x, p, xh, ph), field 1 = xh under d(xh, ph, x, p)
#if PIRK_STENCIL > 0
extern "C" __global__ void __launch_bounds__(256) pirk_user_tile(int which, double t0, double t1, double h,
        u64 step, u64 total, const double* __restrict__ in0, const double* __restrict__ in1,
        double* __restrict__ out0, double* __restrict__ out1, const double* __restrict__ p, u64 n,
        u64* fail) {
    constexpr long long R = PIRK_STENCIL;
    constexpr long long TO = 1024;
    constexpr long long L = TO + 8 * R;
    extern __shared__ double sm[];
    const int nf = which == 2 ? 2 : 1;
    const long long c0 = (long long)blockIdx.x * TO;
    long long c1 = c0 + TO;
    if (c1 > (long long)n) c1 = (long long)n;
    const long long lo = c0 - 4 * R > 0 ? c0 - 4 * R : 0;
    const long long hi = c1 + 4 * R < (long long)n ? c1 + 4 * R : (long long)n;
    double* X[2];
    double* UA[2];
    double* UB[2];
    double* AC[2];
    for (int f = 0; f < 2; ++f) {
        X[f] = sm + (4 * f + 0) * L;
        UA[f] = sm + (4 * f + 1) * L;
        UB[f] = sm + (4 * f + 2) * L;
        AC[f] = sm + (4 * f + 3) * L;
    }
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        X[0][i - lo] = in0[i];
        if (nf == 2) X[1][i - lo] = in1[i];
    }
    __syncthreads();
    const pirk_rt::StepConsts c = pirk_rt::step_consts(t0, t1, h, step, total);
    const double* P0 = p;
    const double* P1 = p + PIRK_NI;
    for (int stage = 0; stage < 4; ++stage) {
        // valid range of this stage's output: shrinks by R per stage, not at the domain ends
        const long long a = lo == 0 ? 0 : lo + (stage + 1) * R;
        const long long b = hi == (long long)n ? (long long)n : hi - (stage + 1) * R;
        const double tt = stage == 0 ? c.t : (stage == 3 ? c.thk : c.th2);
        for (long long i = a + threadIdx.x; i < b; i += blockDim.x) {
            const long long o = i - lo;
            for (int f = 0; f < nf; ++f) {
                const double* S0 = (stage == 0 ? X[0] : UA[0]) - lo;   // rebased: S0[j] is component j
                const double* S1 = (stage == 0 ? X[1] : UA[1]) - lo;
                double k;
                if (which == 0) k = pirk_rhs((u64)i, tt, S0, P0);
                else if (which == 1) k = pirk_growth((u64)i, tt, S0, P0);
                else if (f == 0) k = pirk_decomposition((u64)i, tt, S0, P0, S1, P1);
                else k = pirk_decomposition((u64)i, tt, S1, P1, S0, P0);
                const double x = X[f][o];
                if (stage == 0) {
                    AC[f][o] = k;
                    UB[f][o] = x + c.h2 * k;
                } else if (stage < 3) {
                    AC[f][o] = AC[f][o] + 2.0 * k;
                    UB[f][o] = x + (stage == 1 ? c.h2 : c.hk) * k;
                } else if (i >= c0 && i < c1) {
                    const double xn = x + c.h6 * (AC[f][o] + k);
                    (f == 0 ? out0 : out1)[i] = xn;
                    if (!pirk_rt::finite_d(xn))
                        atomicMin(fail, (step << pirk_rt::kFailCompBits) | ((u64)i + (which == 2 && f == 1 ? n : 0ull)));
                }
            }
        }
        __syncthreads();
        for (int f = 0; f < 2; ++f) {
            double* tmp = UA[f];
            UA[f] = UB[f];
            UB[f] = tmp;
        }
    }
}
#endif

struct UserMcArgs {
    const double* lo;
    const double* hi;
    const double* plo;
    const double* phi;
    u64 seed, s_begin, s_end;
    double t0, t1, h;
    u64 total, stride, slots;
    u64* hull;  // slots x [min n | max n] ordered keys
    u64* fail;
    const double* box_lo;
    const double* box_hi;
    u64* outside;
};

namespace pirk_rt {
// min / max of the warp's keys, then one atomic per component and bound
PIRK_DEV void fold_keys(const double* x, bool live, u64* hull_slot) {
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < PIRK_N; ++i) {
        const u64 key = ord_key(x[i]);
        u64 lo = live ? key : ~0ull, hi = live ? key : 0ull;
        for (int o = 16; o > 0; o >>= 1) {
            const u64 ol = __shfl_xor_sync(0xffffffffu, lo, o);
            const u64 oh = __shfl_xor_sync(0xffffffffu, hi, o);
            lo = ol < lo ? ol : lo;
            hi = oh > hi ? oh : hi;
        }
        if (lane == 0) {
            if (lo != ~0ull) atomicMin(hull_slot + i, lo);
            if (hi != 0ull) atomicMax(hull_slot + PIRK_N + i, hi);
        }
    }
}
}  // namespace pirk_rt

extern "C" __global__ void __launch_bounds__(128) pirk_user_mc(const UserMcArgs a) {
    const u64 s = a.s_begin + (u64)blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = s < a.s_end;
    const bool coverage = a.outside != nullptr;
    constexpr int NP = PIRK_NI > 0 ? PIRK_NI : 1;
    double x[PIRK_N], u[PIRK_N], k[PIRK_N], acc[PIRK_N], p[NP];
    // draw_sample (reach.cpp:202-212)
    for (int i = 0; i < PIRK_N; ++i) x[i] = active ? pirk_rt::uniform_in(a.lo[i], a.hi[i], pirk_rt::u01(a.seed, s, (u64)i)) : 0.0;
    for (int j = 0; j < NP; ++j)
        p[j] = (active && j < PIRK_NI) ? pirk_rt::uniform_in(a.plo[j], a.phi[j], pirk_rt::u01(a.seed, s, (u64)(PIRK_N + j))) : 0.0;
    u64 slot = 0;
    if (a.stride > 0 && !coverage) {
        pirk_rt::fold_keys(x, active, a.hull);
        slot = 1;
    }
    bool dead = !active;
    for (u64 st = 0; st < a.total; ++st) {
        const pirk_rt::StepConsts c = pirk_rt::step_consts(a.t0, a.t1, a.h, st, a.total);
        if (!dead) {
            const int bad = pirk_rt::serial_step<0, PIRK_N>(x, u, k, acc, p, c);
            if (bad >= 0) {  // lowest failing sample wins (host: s < 2^34, steps < 2^20, n <= 1024)
                atomicMin(a.fail, ((s - a.s_begin) << 30) | (st << 10) | (u64)bad);
                dead = true;
            }
        }
        if (!coverage && (st + 1 == a.total || (a.stride > 0 && (st + 1) % a.stride == 0))) {
            pirk_rt::fold_keys(x, !dead, a.hull + slot * 2 * PIRK_N);
            ++slot;
        }
    }
    if (coverage && !dead) {
        bool out = false;
        for (int i = 0; i < PIRK_N; ++i)
            if (x[i] < a.box_lo[i] || x[i] > a.box_hi[i]) out = true;  // interval.cpp:55-62
        if (out) atomicAdd(a.outside, 1ull);
    }
}
)PIRK";

}  // namespace pirk
