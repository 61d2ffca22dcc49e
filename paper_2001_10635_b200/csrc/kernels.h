// kernels.h -- host-visible launch interface of the PIRK device kernels.
// Each launcher exists in an exact (-fmad=false) and a fast instantiation.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pirk {

struct StepConsts;

// Two-field window of a 1-D or 3-D state on the device (see pirk_c.h
// pirk_window).  Units: components (chain) or z-planes (heat3d).
struct WindowArgs {
    const double* in0;
    const double* in1;
    double* out0;
    double* out1;
    uint64_t win_begin, win_end;
    uint64_t out_begin, out_end;
    // mirror outputs (or null): a value of unit u stored to out0[k] / out1[k]
    // (k = u - out_begin) is also stored to mir0[k] / mir1[k] when
    // u < mir_lo_end, and to mirh0[k] / mirh1[k] when u >= mir_hi_begin -- the
    // neighbours' halos over NVLink peer memory, written by the kernel that
    // computes them (engine.cu run_large_multi, sharded.PeerStores).  The
    // defaults mirror every unit to mir0/1 and none to mirh0/1.
    double* mir0 = nullptr;
    double* mir1 = nullptr;
    uint64_t mir_lo_end = ~0ull;
    double* mirh0 = nullptr;
    double* mirh1 = nullptr;
    uint64_t mir_hi_begin = ~0ull;

    __host__ __device__ bool mirrored() const { return mir0 != nullptr || mirh0 != nullptr; }
};

// Per-launch plane limits of the two mirror targets as ints (planes < 2^31):
// units u < lo_end go to the low target, u >= hi_begin to the high one.
struct MirrorLimits {
    int lo_end, hi_begin;
    __host__ __device__ static MirrorLimits of(const WindowArgs& w) {
        MirrorLimits m;
        m.lo_end = !w.mir0 ? -0x7fffffff : (w.mir_lo_end >= 0x7fffffffull ? 0x7fffffff : static_cast<int>(w.mir_lo_end));
        m.hi_begin = !w.mirh0 ? 0x7fffffff : (w.mir_hi_begin >= 0x7fffffffull ? 0x7fffffff
                                                                                : static_cast<int>(w.mir_hi_begin));
        return m;
    }
};

// 1-D radius-1 models on two fields (traffic MM/GB, coupled chain MM).
struct ChainModel {
    int kind;      // PIRK_TRAFFIC or PIRK_CHAIN
    int method;    // PIRK_METHOD_MM or PIRK_METHOD_GB
    uint64_t n;
    double P[8];   // make_* parameters
    double p0, p1; // field inputs: MM (p_lo, p_hi); GB (center, half-width)
    // host-derived constants (rounded exactly as the reference computes them)
    double inv_t, a_prev, a_next, a_in, wb;
};

// heat3d (models.cpp:92-133) on two independent fields.
struct HeatModel {
    int method;
    uint64_t g;
    double kk;      // alpha / (delta*delta)
    double robin;   // 2*delta*exchange
};

// Small dense systems (n <= 64): one thread per trajectory.
constexpr int kSmallMax = 64;
struct SmallModel {
    int kind, decomp;
    int n, ni;
    uint64_t grid;
    double P[8];
    int has_C;
    double C[12 * 12];  // dense growth matrix (row-major n x n) for n <= 12
    // host-derived constants, each the same IEEE operation the device would do
    // per evaluation (arch-quadrotor: (jy-jz)/jx, (jz-jx)/jy, (jx-jy)/jz, 1/jx,
    // 1/jy, 1/mass; models.cpp:520-552)
    double Q[8];
};

template <bool Exact>
cudaError_t launch_chain_step(const ChainModel& m, const WindowArgs& w, const StepConsts& sc,
                              unsigned long long step, unsigned long long* fail,
                              cudaStream_t stream);

// S (2..4) chain steps per launch (step .. step+S-1) with the warp-tiled kernel.
struct StepConstsN {
    StepConsts s[4];
};
template <bool Exact>
cudaError_t launch_chain_steps(const ChainModel& m, const WindowArgs& w, const StepConstsN& scs, int S,
                               unsigned long long step, unsigned long long* fail, cudaStream_t stream);

// Fast mode: whether a step of length hk can run the strip kernel (and so a
// one-field launch, field_only >= 0); defined in inst_fast.cu.
bool heat_strip_step_ok(const HeatModel& m, double hk);

template <bool Exact>
cudaError_t launch_heat_step(const HeatModel& m, const WindowArgs& w, const StepConsts& sc,
                             unsigned long long step, unsigned long long* fail,
                             cudaStream_t stream, int field_only = -1);

// which: 0 = f under p, 1 = growth under w, 2 = embedding (dim 2n, p = [p_lo | p_hi]).
// One thread integrates the whole plan, recording `slots` states into rec.
template <bool Exact>
cudaError_t launch_small_integrate(const SmallModel& m, int which, const double* x0,
                                   const double* p, double t0, double t1, double h,
                                   unsigned long long total, unsigned long long stride,
                                   double* rec, unsigned long long* fail, cudaStream_t stream);

struct McArgs {
    const double* lo;   // device, n
    const double* hi;
    const double* plo;  // device, ni (may be null when ni == 0)
    const double* phi;
    uint64_t seed, s_begin, s_end;
    double t0, t1, h;
    unsigned long long total, stride, slots;
    unsigned long long* hull;        // slots x [min n | max n] ordered keys
    unsigned long long* fail;        // packed (sample, step, comp) of the lowest failing sample
    // coverage mode: count final states outside [box_lo, box_hi]
    const double* box_lo;
    const double* box_hi;
    unsigned long long* outside;
};

template <bool Exact>
cudaError_t launch_monte_carlo(const SmallModel& m, const McArgs& a, cudaStream_t stream);

// Embedding-order check (reach.cpp:181-186): fail = min i with lo[i] > hi[i].
cudaError_t launch_order_check(const double* lo, const double* hi, uint64_t n,
                               unsigned long long* fail, cudaStream_t stream);
// Validation of an uploaded box (IntervalVector ctor, interval.cpp:14-22):
// bad = min i with a non-finite bound or lo[i] > hi[i].
cudaError_t launch_box_check(const double* lo, const double* hi, uint64_t n,
                             unsigned long long* bad, cudaStream_t stream);
// Growth-bound box epilogue (reach.cpp:121-134, interval.cpp:39-53):
// r in [-1e-12, 0) -> 0, r < -1e-12 -> neg = min i; lo = c - r, hi = c + r.
cudaError_t launch_gb_box(const double* c, const double* r, double* lo, double* hi, uint64_t n,
                          unsigned long long* neg, cudaStream_t stream);
// center = 0.5*(u+l), radius = 0.5*(u-l) (interval.cpp:25-37), in place.
// neg_val[0] = r[*neg] if *neg was set (the value quoted in the error message).
cudaError_t launch_gb_negval(const double* r, const unsigned long long* neg, double* neg_val,
                             cudaStream_t stream);
cudaError_t launch_center_radius(double* lo_to_c, double* hi_to_r, uint64_t n,
                                 cudaStream_t stream);
cudaError_t launch_fill(unsigned long long* p, unsigned long long v, uint64_t n,
                        cudaStream_t stream);
// *flag = v (release, system scope) after all prior work on the stream.
cudaError_t launch_signal_flag(unsigned* flag, unsigned v, cudaStream_t stream);

}  // namespace pirk
