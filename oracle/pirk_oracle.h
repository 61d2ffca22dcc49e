/*
 * pirk_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's reachability hot path
 * (/root/reference/proj, "ivreach"), used solely as the parity checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  Nothing in
 * paper_2001_10635_b200/ links, imports or calls this code.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against the
 * reference's own known-answer tests (test_rk4.cpp, test_models.cpp,
 * test_reach.cpp, test_rng.cpp) and against golden vectors produced by the
 * reference itself (oracle/_ref, built from /root/reference/proj/src by
 * oracle/Makefile; fixtures in tests/golden/ made by tests/golden/make_golden.py).
 *
 * Arithmetic regime: IEEE binary64, no FMA contraction (built with
 * -ffp-contract=off, no -march), matching the reference build
 * (proj/CMakeLists.txt:12-13, SURVEY.md 8c "Arithmetic regime").
 */
#ifndef PIRK_ORACLE_H
#define PIRK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Model kinds; numbering shared with include/pirk_c.h (same meaning). */
enum {
    PO_ZERO = 0,          /* models.cpp:615-627   params: -                          */
    PO_SCALAR_DECAY = 1,  /* models.cpp:629-641   params: -                          */
    PO_SCALAR_LINEAR = 2, /* models.cpp:643-655   params: a                          */
    PO_TRAFFIC = 3,       /* models.cpp:47-90     params: v, w, c, xbar, period, beta */
    PO_HEAT3D = 4,        /* models.cpp:92-133    params: alpha, exchange (dim=g^3)  */
    PO_CHAIN = 5,         /* SURVEY.md 8d C4      params: a, b, c                    */
    PO_LAUB_LOOMIS = 6,   /* models.cpp:463-502   params: -                          */
    PO_ARCH_QUAD = 7,     /* models.cpp:504-613   params: mass, gravity, jx, jy, jz  */
    PO_VDP = 8,           /* models.cpp:444-461   params: mu, op_x, op_y             */
    /* User-defined systems of the reference's own tests, built from the same
     * lambdas by oracle/ref_shim.cpp only (the device runs them as NVRTC user
     * models, tests/test_gpu_user.py). */
    PO_T_ORDER = 100,     /* test_reach.cpp:190-206: f = (x1, -1), d = (xh1, -1)     */
    PO_T_EMBED = 101,     /* test_system_model.cpp:74-96: f = -x0, d = -xh0          */
    PO_T_DRIFT = 102,     /* test_reach.cpp:208-230: make_zero(1), growth = params[0] */
    PO_T_BARE = 103       /* test_reach.cpp:176-188: rhs = -x0 only                  */
};

/* Decomposition variants. */
enum {
    PO_DECOMP_NONE = 0,      /* model has no decomposition                                   */
    PO_DECOMP_NATIVE = 1,    /* the model's own d (cooperative(f) for catalog models,
                                models.cpp:20-27; the coupled d for PO_CHAIN)               */
    PO_DECOMP_JACOBIAN = 2   /* d_i = f_i(x) + sum_{j!=i, C_ij!=0} C_ij (x_j - xh_j), with C
                                the model's growth matrix                */
};

typedef struct {
    int32_t kind;
    int32_t decomp;
    uint64_t dim;        /* n */
    uint64_t input_dim;
    uint64_t grid;       /* heat3d nodes per axis (dim == grid^3); 0 otherwise */
    double params[8];
} po_model;

/* Error codes (mirror of include/pirk_c.h status values). */
enum { PO_OK = 0, PO_EINVAL = 1, PO_EINTEGRATION = 2, PO_EORDER = 3, PO_ENEGRADIUS = 4, PO_ENOMEM = 5 };

/* rng.hpp:11-29 */
uint64_t po_mix64(uint64_t z);
double po_u01(uint64_t seed, uint64_t stream, uint64_t index);
double po_uniform_in(double lo, double hi, double u);

/* rk4.cpp:8-17 */
int po_plan_steps(double t0, double t1, double h, uint64_t* full_steps, int* has_remainder);
/* reach.cpp:28-39: number of record slots and (optionally) their steps/times */
uint64_t po_record_schedule(double t0, double t1, double h, uint64_t stride,
                            uint64_t* steps_out, double* times_out);
/* reach.cpp:55-63 */
int po_sample_count(uint64_t n, double epsilon, double delta, uint64_t* out);

/* Component evaluators. */
double po_rhs(const po_model* m, uint64_t i, double t, const double* x, const double* p);
double po_growth(const po_model* m, uint64_t i, double t, const double* r, const double* w);
double po_decomp(const po_model* m, uint64_t i, double t, const double* x, const double* p,
                 const double* xh, const double* ph);
/* Dense growth matrix (row-major n x n) for the small models; returns 0 if none. */
int po_growth_matrix(const po_model* m, double* C);

/* Plain RK4 of x' = f(t,x,p) (rk4_serial.cpp:10-61); records like
 * Rk4Engine::run (rk4.cpp:96-111).  states_out: slots x dim. */
int po_integrate(const po_model* m, const double* x0, const double* p, double t0, double t1,
                 double h, uint64_t stride, double* times_out, double* states_out,
                 uint64_t* err_step, uint64_t* err_comp, double* err_t);

/* Methods.  Output arrays are slots x n (lower, upper); slots from
 * po_record_schedule.  On failure returns the error code and fills
 * err (a message formatted like the reference's exceptions). */
int po_mixed_monotonicity(const po_model* m, const double* lo, const double* hi,
                          const double* plo, const double* phi, double t0, double t1,
                          double h, uint64_t stride, double* times, double* out_lo,
                          double* out_hi, char* err, int errlen);
int po_growth_bound(const po_model* m, const double* lo, const double* hi,
                    const double* plo, const double* phi, double t0, double t1, double h,
                    uint64_t stride, double* times, double* out_lo, double* out_hi,
                    char* err, int errlen);
/* Samples [s_begin, s_end) only (so a sharded run can be checked piecewise);
 * out_lo/out_hi must be initialised by the caller (+inf / -inf) and are folded into. */
int po_monte_carlo(const po_model* m, const double* lo, const double* hi, const double* plo,
                   const double* phi, double t0, double t1, double h, uint64_t stride,
                   uint64_t seed, uint64_t s_begin, uint64_t s_end, double* times,
                   double* out_lo, double* out_hi, char* err, int errlen);
/* reach.cpp:325-358 (single-threaded). */
int po_coverage_estimate(const po_model* m, const double* lo, const double* hi,
                         const double* plo, const double* phi, double t0, double t1,
                         double h, const double* box_lo, const double* box_hi,
                         uint64_t fresh, uint64_t seed, double* fraction);

/* One RK4 step of the 2n embedding (method 0) or of the growth-bound pair
 * [c | r] (method 1) restricted to a window of the global state, used by the
 * sharded-driver tests: win_lo/win_hi hold global components
 * [win_begin, win_begin + win_len) (chain models) or global z-planes (heat3d,
 * grid^2 components per plane); outputs are produced for global
 * [out_begin, out_end) in the same window coordinates.  Components outside the
 * window are never read; the caller guarantees out range +-4 lies inside the
 * window or on the global boundary.  Arithmetic is exactly integrate_step's
 * (rk4.cpp:30-76) evaluated per component. */
int po_step_window(const po_model* m, int method, const double* in0, const double* in1,
                   double* out0, double* out1, uint64_t win_begin, uint64_t win_len,
                   uint64_t out_begin, uint64_t out_end, const double* p0, const double* p1,
                   double t, double hk);

#ifdef __cplusplus
}
#endif

#endif
