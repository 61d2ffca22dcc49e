/*
 * pirk_c.h -- C ABI of the B200-native PIRK reachability hot path.
 *
 * Drop-in boundary for the reference's entry points (relative to
 * /root/reference/proj):
 *
 *   pirk_mixed_monotonicity  replaces  ivreach::mixed_monotonicity  include/ivreach/reach.hpp:50-53
 *                                                                   (src/reach.cpp:139-196)
 *   pirk_growth_bound        replaces  ivreach::growth_bound        include/ivreach/reach.hpp:43-48
 *                                                                   (src/reach.cpp:65-137)
 *   pirk_monte_carlo         replaces  ivreach::monte_carlo         include/ivreach/reach.hpp:62-71
 *                                                                   (src/reach.cpp:246-323)
 *   pirk_coverage_estimate   replaces  ivreach::coverage_estimate   include/ivreach/reach.hpp:73-78
 *                                                                   (src/reach.cpp:325-358)
 *   pirk_sample_count        replaces  ivreach::sample_count        include/ivreach/reach.hpp:59-60
 *   pirk_plan_steps          replaces  ivreach::plan_steps          include/ivreach/rk4.hpp:37-39
 *   pirk_record_schedule     restates  record_schedule (file-local) src/reach.cpp:28-39
 *   pirk_engine_*            replace   ivreach::Rk4Engine           include/ivreach/rk4.hpp:66-82
 *                                      run on the embedding (src/system_model.cpp:56-77)
 *   pirk_step_window         replaces  ivreach::integrate_step      include/ivreach/rk4.hpp:54-60
 *                                      restricted to a window (for state-sharded multi-GPU runs)
 *
 * The reference's SystemModel carries std::function evaluators
 * (system_model.hpp:14-43), which cannot execute on a GPU.  Here a model is a
 * plain descriptor (pirk_model): a kind from the reference catalog
 * (models.hpp:17-93) or the synthetic coupled chain of SURVEY.md 8(d), its
 * resolved parameters, and which decomposition to use.  A model the device
 * library does not implement is rejected with PIRK_EUNSUPPORTED; there is no
 * CPU fallback anywhere behind this ABI.
 *
 * All host arrays are borrowed for the duration of a call.  Device pointers
 * (pirk_step_window) are caller-owned.  Calls on one pirk_ctx serialise on
 * the context's mutex (like a non-reentrant Rk4Engine); distinct contexts run
 * concurrently from distinct threads.
 */
#ifndef PIRK_C_H
#define PIRK_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PIRK_ABI_VERSION 1

typedef enum pirk_status {
    PIRK_OK = 0,
    PIRK_EINVAL = 1,          /* std::invalid_argument in the reference          */
    PIRK_EINTEGRATION = 2,    /* IntegrationError (rk4.hpp:41-47) wrapped in runtime_error */
    PIRK_EORDER = 3,          /* embedding order violated (reach.cpp:181-186)    */
    PIRK_ENEGRADIUS = 4,      /* growth-bound radius < -1e-12 (reach.cpp:124-131) */
    PIRK_ENOMEM = 5,          /* std::bad_alloc / cudaErrorMemoryAllocation       */
    PIRK_ECUDA = 6,           /* any other CUDA error                             */
    PIRK_EUNSUPPORTED = 7     /* model/method combination has no device kernel    */
} pirk_status;

/* Model kinds (numbering shared with oracle/pirk_oracle.h). */
typedef enum pirk_model_kind {
    PIRK_ZERO = 0,          /* make_zero(dim)                       models.cpp:615-627 */
    PIRK_SCALAR_DECAY = 1,  /* make_scalar_decay()                  models.cpp:629-641 */
    PIRK_SCALAR_LINEAR = 2, /* make_scalar_linear(a)                models.cpp:643-655 */
    PIRK_TRAFFIC = 3,       /* make_traffic(n, v,w,c,xbar,period,beta)  models.cpp:47-90 */
    PIRK_HEAT3D = 4,        /* make_heat3d(grid, alpha, exchange)   models.cpp:92-133  */
    PIRK_CHAIN = 5,         /* synthetic coupled chain (a, b, c)  */
    PIRK_LAUB_LOOMIS = 6,   /* make_laub_loomis()                   models.cpp:463-502 */
    PIRK_ARCH_QUAD = 7,     /* make_arch_quadrotor(mass,g,jx,jy,jz) models.cpp:504-613 */
    PIRK_VDP = 8,           /* make_vdp(mu, op_x, op_y)             models.cpp:444-461 */
    PIRK_USER = 9           /* user-defined evaluators: pirk_model.program            */
} pirk_model_kind;

typedef enum pirk_decomp {
    PIRK_DECOMP_NONE = 0,     /* SystemModel::decomposition empty                        */
    PIRK_DECOMP_NATIVE = 1,   /* cooperative(f) (models.cpp:20-27) or the chain's own d  */
    PIRK_DECOMP_JACOBIAN = 2  /* d_i = f_i(x) + sum_{j!=i,C_ij!=0} C_ij (x_j - xh_j), C = growth matrix */
} pirk_decomp;

typedef struct pirk_program pirk_program;

typedef struct pirk_model {
    int32_t kind;        /* pirk_model_kind */
    int32_t decomp;      /* pirk_decomp */
    uint64_t dim;        /* n (heat3d: grid^3) */
    uint64_t input_dim;
    uint64_t grid;       /* heat3d nodes per axis, else 0 */
    double params[8];    /* kind-specific, in make_* argument order */
    const pirk_program* program;  /* PIRK_USER: the compiled evaluators, else NULL */
} pirk_model;

/* ---- user-defined models (the reference's SystemModel with arbitrary
 * std::function evaluators, system_model.hpp:14-43) ----
 * `source` is CUDA C++ defining, as the flags say,
 *   __device__ double pirk_rhs(u64 i, double t, const double* x, const double* p);
 *   __device__ double pirk_decomposition(u64 i, double t, const double* x, const double* p,
 *                                        const double* xh, const double* ph);
 *   __device__ double pirk_growth(u64 i, double t, const double* r, const double* w);
 * (u64 = unsigned long long; PIRK_N / PIRK_NI = dim / input_dim; pirk_min /
 * pirk_max = std::min / std::max).  It is compiled with NVRTC for sm_100a on
 * first use in each arithmetic mode (exact: --fmad=false, so +,-,*,/ round
 * like the reference's build).  Use it through a pirk_model with kind
 * PIRK_USER, dim / input_dim equal to the program's, and .program set; every
 * entry point accepts it (MM / GB: one device thread per integration for
 * n <= 64, else one thread per component and stage; MC: n <= 1024). */
enum {
    PIRK_HAS_RHS = 1,
    PIRK_HAS_DECOMPOSITION = 2,
    PIRK_HAS_GROWTH = 4,
    PIRK_INPUT_AFFINE = 8      /* SystemModel::input_affine (growth bound needs it) */
};
pirk_status pirk_program_create(const char* source, uint64_t dim, uint64_t input_dim, uint32_t flags,
                                pirk_program** out);
/* Compile now (no device needed) in `mode`; on failure log receives the NVRTC
 * log.  *cubin_bytes (may be NULL) receives the size of the sm_100a image. */
pirk_status pirk_program_compile(pirk_program* prog, int32_t mode, char* log, size_t log_len,
                                 uint64_t* cubin_bytes);
/* Declare the model a radius-r 1-D stencil: f_i, d_i and g_i read only
 * components in [i - r, i + r] of each state argument (plus the inputs).  MM
 * and GB then advance one whole RK4 step per launch with a shared-memory tile
 * of both fields and a 4r halo (16 B of HBM per state-update) instead of four
 * stage launches.  1 <= r <= 64; call before the first compile. */
pirk_status pirk_program_set_stencil(pirk_program* prog, uint64_t radius);
/* Copy the compiled sm_100a cubin of `mode` (after pirk_program_compile). */
pirk_status pirk_program_cubin(const pirk_program* prog, int32_t mode, void* buf, uint64_t len);
void pirk_program_destroy(pirk_program* prog);

/* ReachProblem (system_model.hpp:47-55). inputs may be NULL iff input_dim == 0. */
typedef struct pirk_problem {
    const double* init_lower;   /* n  */
    const double* init_upper;   /* n  */
    const double* input_lower;  /* input_dim */
    const double* input_upper;  /* input_dim */
    double t0, t1, h;
    uint64_t tube_stride;       /* 0 = final set only */
} pirk_problem;

/* MonteCarloSpec (reach.hpp:55-60). */
typedef struct pirk_mc_spec {
    double epsilon;
    double delta;
    uint64_t seed;
    uint64_t samples_override;  /* 0 = sample_count(n, epsilon, delta) */
} pirk_mc_spec;

/* Output tube (ReachTube entries, reach.hpp:32-41), caller-allocated:
 * times[max_slots], lower/upper[max_slots * n] row-major by slot.  lower/upper
 * may be NULL to skip the device->host transfer (times and n_slots are still
 * filled).  max_slots must be >= pirk_record_schedule(...). */
typedef struct pirk_tube {
    double* times;
    double* lower;
    double* upper;
    uint64_t max_slots;
    uint64_t n_slots;           /* out */
} pirk_tube;

/* RunReport + PhaseTimes (reach.hpp:13-30), plus device-side accounting. */
typedef struct pirk_report {
    uint64_t n;
    uint64_t m;
    uint64_t steps;
    uint64_t peak_state_bytes;   /* the reference's analytic value, for interface parity */
    uint64_t device_state_bytes; /* device bytes actually allocated for the state */
    int32_t workers;             /* shard lanes used (pirk_create_multi; 1 otherwise) */
    int32_t exact;               /* 1 = bit-exact arithmetic mode */
    double setup_s;
    double integration_s;
    double reduction_s;
    uint64_t kernel_launches;
} pirk_report;

typedef enum pirk_mode {
    PIRK_MODE_EXACT = 0,  /* no FMA contraction, reference expression order: bit-identical */
    PIRK_MODE_FAST = 1    /* FMA + restructured stencils: relative <= 1e-12 of the reference */
} pirk_mode;

typedef enum pirk_method {
    PIRK_METHOD_MM = 0,   /* mixed monotonicity (embedding) */
    PIRK_METHOD_GB = 1    /* growth bound ([center | radius]) */
} pirk_method;

typedef struct pirk_ctx pirk_ctx;
typedef struct pirk_engine pirk_engine;

/* ---- context ---- */
int32_t pirk_abi_version(void);
pirk_status pirk_create(int device, pirk_ctx** out);
/* A context of n_lanes shard lanes, lane r on CUDA device devices[r] (ids may
 * repeat: several lanes then share one GPU).  Chain and heat3d MM/GB runs
 * shard the state across the lanes (contiguous component ranges / z-slabs,
 * 4-unit halos exchanged every RK4 step: the boundary launches store their
 * units into the neighbours' halos over NVLink peer memory, then the interior
 * runs; peer copies where peer access is missing); Monte Carlo shards the
 * sample range and min/max-folds the hulls.  Results are bit-identical for
 * any lane count.  This is what the reference's `workers` argument maps to
 * (reach.hpp:48,53,70).  Lane 0 is the primary device (pirk_set_stream). */
pirk_status pirk_create_multi(int n_lanes, const int* devices, pirk_ctx** out);
int32_t pirk_lane_count(const pirk_ctx* ctx);
/* Visible CUDA devices (0 when there is none). */
int32_t pirk_device_count(void);
int32_t pirk_lane_device(const pirk_ctx* ctx, int32_t lane);
/* Streaming observer (StepObserver, rk4.hpp:63-64, called as rk4.cpp:106-111
 * does): when set, every run on the context calls fn once per recorded slot,
 * in slot order, with that slot's box (MM: x / x-hat; GB: the clamped box; MC:
 * the hull) in host memory valid for the duration of the call.  For chain /
 * heat3d / user models the callback for slot s runs while the device
 * integrates towards slot s+1, so a tube larger than host memory can be
 * consumed slot by slot (pirk_tube.lower / .upper may then be NULL).  A run
 * that fails delivers the slots recorded before the failure was detected and
 * then returns the error.  fn = NULL disables it. */
typedef void (*pirk_record_fn)(void* user, uint64_t slot, uint64_t step, double t, const double* lower,
                               const double* upper, uint64_t n);
pirk_status pirk_set_record_callback(pirk_ctx* ctx, pirk_record_fn fn, void* user);
/* Free the state buffers a context keeps between runs of the same size. */
pirk_status pirk_release_cache(pirk_ctx* ctx);
void pirk_destroy(pirk_ctx* ctx);
const char* pirk_last_error(const pirk_ctx* ctx);
pirk_status pirk_set_mode(pirk_ctx* ctx, int32_t mode);
/* Launch on this cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * NULL is the CUDA default stream.  pirk_get_stream right after pirk_create
 * returns the context's own (non-blocking) stream. */
pirk_status pirk_set_stream(pirk_ctx* ctx, void* stream);
void* pirk_get_stream(pirk_ctx* ctx);
uint64_t pirk_launch_count(const pirk_ctx* ctx);

/* ---- host-side helpers (no device work) ---- */
pirk_status pirk_plan_steps(double t0, double t1, double h, uint64_t* full_steps,
                            int32_t* has_remainder);
uint64_t pirk_record_schedule(double t0, double t1, double h, uint64_t stride,
                              uint64_t* steps_out, double* times_out);
pirk_status pirk_sample_count(uint64_t n, double epsilon, double delta, uint64_t* out);
/* 1 if the device library implements (kind, method) with this decomposition. */
int32_t pirk_supports(const pirk_model* model, int32_t method_or_mc);

/* ---- reference entry points (host buffers in, host tube out) ---- */
pirk_status pirk_mixed_monotonicity(pirk_ctx* ctx, const pirk_model* model,
                                    const pirk_problem* problem, pirk_tube* tube,
                                    pirk_report* report);
pirk_status pirk_growth_bound(pirk_ctx* ctx, const pirk_model* model,
                              const pirk_problem* problem, pirk_tube* tube,
                              pirk_report* report);
pirk_status pirk_monte_carlo(pirk_ctx* ctx, const pirk_model* model,
                             const pirk_problem* problem, const pirk_mc_spec* spec,
                             pirk_tube* tube, pirk_report* report);
/* Monte Carlo over samples [s_begin, s_end) only, folding into tube->lower/upper
 * (which the caller initialises to +inf/-inf): the per-rank piece of a
 * sample-sharded run. */
pirk_status pirk_monte_carlo_range(pirk_ctx* ctx, const pirk_model* model,
                                   const pirk_problem* problem, uint64_t seed,
                                   uint64_t s_begin, uint64_t s_end, pirk_tube* tube,
                                   pirk_report* report);
pirk_status pirk_coverage_estimate(pirk_ctx* ctx, const pirk_model* model,
                                   const pirk_problem* problem, const double* box_lower,
                                   const double* box_upper, uint64_t fresh_samples,
                                   uint64_t seed, double* fraction);

/* ---- engine: device-resident state, for benchmarks and streaming callers ---- */
pirk_status pirk_engine_create(pirk_ctx* ctx, const pirk_model* model, int32_t method,
                               const pirk_problem* problem, pirk_engine** out);
/* Advance up to nsteps steps of the plan, asynchronously on the ctx stream. */
pirk_status pirk_engine_advance(pirk_engine* e, uint64_t nsteps);
/* Synchronise; report completed steps and the first failure (PIRK_EINTEGRATION). */
pirk_status pirk_engine_status(pirk_engine* e, uint64_t* steps_done);
/* Current box (MM: [x | xh]; GB: center -/+ clamped radius) into host arrays (n each). */
pirk_status pirk_engine_read(pirk_engine* e, double* lower, double* upper);
void pirk_engine_destroy(pirk_engine* e);

/* ---- one windowed RK4 step on caller-owned device buffers (multi-GPU shards) ----
 * Fields: MM -> (x, xh); GB -> (center, radius).  Units are components for
 * 1-D models and z-planes (grid^2 components) for heat3d.  in0/in1 hold global
 * units [win_begin, win_begin + win_len); out0/out1 receive global units
 * [out_begin, out_end) (out0[0] is unit out_begin).  Requires
 * out_begin - 4 >= win_begin unless out_begin < 4, and
 * out_end + 4 <= win_begin + win_len unless out_end + 4 > total units (the
 * 4-stage dependency cone).  p0/p1: host input vectors (MM: p_lo, p_hi;
 * GB: center, half-width).  fail: device uint64[2] (or NULL) receiving
 * atomicMin((step << 40) | component) of non-finite outputs. */
typedef struct pirk_window {
    const double* in0;
    const double* in1;
    double* out0;
    double* out1;
    uint64_t win_begin, win_len;
    uint64_t out_begin, out_end;
} pirk_window;

pirk_status pirk_step_window(pirk_ctx* ctx, const pirk_model* model, int32_t method,
                             const pirk_window* win, const double* p0, const double* p1,
                             double t, double hk, uint64_t step_index, uint64_t* fail);

/* ---- one process per GPU: halos by peer stores (replaces the shared address
 * space the reference's OpenMP workers integrate in, rk4.cpp:47-75) ----
 * A rank's boundary launch also stores its output units into the neighbour's
 * window over NVLink and then raises the neighbour's step flag; the
 * neighbour's stream waits for the flag before its next boundary launch.
 *
 * pirk_step_window_mirror: pirk_step_window that also stores output units
 *   into the neighbours' windows (typically a peer process's buffers opened
 *   with pirk_ipc_open): unit u (u < lo_end) also to lo0/lo1[u - out_begin],
 *   unit u (u >= hi_begin) also to hi0/hi1[u - out_begin].  NULL lo0 / hi0
 *   disables that side.  One launch over a rank's whole slab with lo_end =
 *   out_begin + 4 and hi_begin = out_end - 4 computes and sends its halos.
 * pirk_ipc_export: IPC handle (64 bytes) of the allocation holding dptr and the
 *   byte offset of dptr inside it (dptr may be a sub-allocation, e.g. torch's).
 * pirk_ipc_open: map a peer process's allocation on `device`; returns its base
 *   (add the exported offset).  Mapping the same handle again returns the same
 *   base (reference-counted); pirk_ipc_close unmaps when the count drops to 0.
 * pirk_wait_flag: the ctx stream waits until (int32_t)(*flag - value) >= 0;
 *   flag is a uint32 in this process's device memory.
 * pirk_signal_flag: after all prior work on the ctx stream, *flag = value
 *   (system-scope release; flag may be a peer process's memory). */
typedef struct pirk_mirror {
    double* lo0;
    double* lo1;
    uint64_t lo_end;
    double* hi0;
    double* hi1;
    uint64_t hi_begin;
} pirk_mirror;
pirk_status pirk_step_window_mirror(pirk_ctx* ctx, const pirk_model* model, int32_t method,
                                    const pirk_window* win, const pirk_mirror* mirror,
                                    const double* p0, const double* p1, double t, double hk,
                                    uint64_t step_index, uint64_t* fail);
pirk_status pirk_ipc_export(const void* dptr, unsigned char handle[64], uint64_t* offset);
pirk_status pirk_ipc_open(int device, const unsigned char handle[64], void** base);
pirk_status pirk_ipc_close(void* base);
pirk_status pirk_wait_flag(pirk_ctx* ctx, const uint32_t* flag, uint32_t value);
pirk_status pirk_signal_flag(pirk_ctx* ctx, uint32_t* flag, uint32_t value);

#ifdef __cplusplus
}
#endif

#endif /* PIRK_C_H */
