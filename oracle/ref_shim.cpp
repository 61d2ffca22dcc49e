// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" adapter over the UNMODIFIED reference library (ivreach, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It
// builds ivreach::ReachProblem objects through the reference's own public API
// (models.hpp make_* constructors, reach.hpp entry points) so that tests and
// the bench's reference arm can run the reference CPU path on exactly the
// inputs given to the CUDA path.  Only tests/, smoke() and bench.py's
// cpu_baseline / --impl reference leg load the resulting library.
#include <omp.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "ivreach/models.hpp"
#include "ivreach/reach.hpp"
#include "ivreach/rk4.hpp"
#include "ivreach/rng.hpp"
#include "ivreach/system_model.hpp"

#include "pirk_oracle.h"  // po_model layout and kind numbering only

using namespace ivreach;

namespace {

void set_err(char* err, int errlen, const std::string& msg) {
    if (err && errlen > 0) std::snprintf(err, static_cast<std::size_t>(errlen), "%s", msg.c_str());
}

// Synthetic coupled chain, SURVEY.md 8d (C4).  The same expression order as
// the CUDA functor and oracle/pirk_oracle.c chain_d.
SystemModel make_chain(std::size_t n, double a, double b, double c) {
    auto s = [](double z) { return z / (1.0 + std::fabs(z)); };
    SystemModel m;
    m.dim = n;
    m.input_dim = 1;
    m.input_affine = true;
    m.sparsity_note = "tridiagonal, non-cooperative";
    m.decomposition = [n, a, b, c, s](std::size_t i, double, std::span<const double> x,
                                      std::span<const double> p, std::span<const double> xh,
                                      std::span<const double>) {
        const double sl = (i == 0) ? 0.0 : s(x[i - 1]);
        const double sr = (i + 1 == n) ? 0.0 : s(xh[i + 1]);
        return ((-a) * x[i] + b * sl - c * sr) + p[0];
    };
    const DecompFn d = m.decomposition;
    m.rhs = [d](std::size_t i, double t, std::span<const double> x, std::span<const double> p) {
        return d(i, t, x, p, x, p);
    };
    return m;
}

// d_i = f_i(x) + sum_{j != i, C_ij != 0} C_ij (x_j - xh_j); C probed from the
// model's own growth_rhs (growth_from_matrix, system_model.cpp:107-121).
void add_jacobian_decomposition(SystemModel& m) {
    const std::size_t n = m.dim;
    std::vector<double> C(n * n, 0.0);
    std::vector<double> e(n, 0.0), w(m.input_dim, 0.0);
    for (std::size_t j = 0; j < n; ++j) {
        e[j] = 1.0;
        for (std::size_t i = 0; i < n; ++i) C[i * n + j] = m.growth_rhs(i, 0.0, e, w);
        e[j] = 0.0;
    }
    const RhsFn f = m.rhs;
    m.decomposition = [f, C, n](std::size_t i, double t, std::span<const double> x,
                                std::span<const double> p, std::span<const double> xh,
                                std::span<const double>) {
        double acc = f(i, t, x, p);
        for (std::size_t j = 0; j < n; ++j) {
            const double cij = C[i * n + j];
            if (j == i || cij == 0.0) continue;
            acc = acc + cij * (x[j] - xh[j]);
        }
        return acc;
    };
}

SystemModel build_model(const po_model* pm) {
    const double* P = pm->params;
    SystemModel m;
    switch (pm->kind) {
        case PO_ZERO: m = make_zero(pm->dim); break;
        case PO_SCALAR_DECAY: m = make_scalar_decay(); break;
        case PO_SCALAR_LINEAR: m = make_scalar_linear(P[0]); break;
        case PO_TRAFFIC: m = make_traffic(pm->dim, P[0], P[1], P[2], P[3], P[4], P[5]); break;
        case PO_HEAT3D: m = make_heat3d(pm->grid, P[0], P[1]); break;
        case PO_CHAIN: m = make_chain(pm->dim, P[0], P[1], P[2]); break;
        case PO_LAUB_LOOMIS: m = make_laub_loomis(); break;
        case PO_ARCH_QUAD: m = make_arch_quadrotor(P[0], P[1], P[2], P[3], P[4]); break;
        case PO_VDP: m = make_vdp(P[0], P[1], P[2]); break;
        case PO_T_ORDER:  // test_reach.cpp:190-206, verbatim lambdas
            m.dim = 2;
            m.input_dim = 0;
            m.rhs = [](std::size_t i, double, std::span<const double> x,
                       std::span<const double>) { return i == 0 ? x[1] : -1.0; };
            m.decomposition = [](std::size_t i, double, std::span<const double>,
                                 std::span<const double>, std::span<const double> xh,
                                 std::span<const double>) { return i == 0 ? xh[1] : -1.0; };
            return m;
        case PO_T_EMBED:  // test_system_model.cpp:74-96
            m.dim = 1;
            m.input_dim = 0;
            m.rhs = [](std::size_t, double, std::span<const double> x,
                       std::span<const double>) { return -x[0]; };
            m.decomposition = [](std::size_t, double, std::span<const double>,
                                 std::span<const double>, std::span<const double> xh,
                                 std::span<const double>) { return -xh[0]; };
            return m;
        case PO_T_DRIFT: {  // test_reach.cpp:208-230
            m = make_zero(1);
            const double g = P[0];
            m.growth_rhs = [g](std::size_t, double, std::span<const double>,
                               std::span<const double>) { return g; };
            return m;
        }
        case PO_T_BARE:  // test_reach.cpp:176-188
            m.dim = 1;
            m.input_dim = 0;
            m.rhs = [](std::size_t, double, std::span<const double> x,
                       std::span<const double>) { return -x[0]; };
            return m;
        default: throw std::invalid_argument("ref_shim: unknown model kind");
    }
    if (pm->decomp == PO_DECOMP_JACOBIAN) add_jacobian_decomposition(m);
    if (pm->decomp == PO_DECOMP_NONE) m.decomposition = nullptr;
    return m;
}

ReachProblem build_problem(const po_model* pm, const double* lo, const double* hi,
                           const double* plo, const double* phi, double t0, double t1,
                           double h, uint64_t stride) {
    SystemModel m = build_model(pm);
    const std::size_t n = m.dim;
    std::optional<IntervalVector> inputs;
    if (m.input_dim > 0)
        inputs = IntervalVector(std::vector<double>(plo, plo + m.input_dim),
                                std::vector<double>(phi, phi + m.input_dim));
    return ReachProblem{std::move(m),
                        IntervalVector(std::vector<double>(lo, lo + n),
                                       std::vector<double>(hi, hi + n)),
                        std::move(inputs), t0, t1, h, static_cast<std::size_t>(stride)};
}

}  // namespace

extern "C" {

int ref_max_threads(void) { return omp_get_max_threads(); }

double ref_u01(uint64_t seed, uint64_t stream, uint64_t index) { return u01(seed, stream, index); }

int ref_sample_count(uint64_t n, double eps, double delta, uint64_t* out) {
    try {
        *out = sample_count(n, eps, delta);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

int ref_plan_steps(double t0, double t1, double h, uint64_t* full, int* rem) {
    try {
        const StepPlan p = plan_steps(t0, t1, h);
        *full = p.full_steps;
        *rem = p.has_remainder ? 1 : 0;
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

// Vector-field evaluation through the reference's SystemModel (which = 0: rhs,
// 1: growth_rhs, 2: decomposition with xh/ph).
int ref_eval(const po_model* pm, int which, double t, const double* x, const double* p,
             const double* xh, const double* ph, double* out, char* err, int errlen) {
    try {
        const SystemModel m = build_model(pm);
        const std::size_t n = m.dim, ni = m.input_dim;
        std::span<const double> sx(x, n), sp(p ? p : x, p ? ni : 0);
        for (std::size_t i = 0; i < n; ++i) {
            if (which == 0) out[i] = m.rhs(i, t, sx, sp);
            else if (which == 1) out[i] = m.growth_rhs(i, t, sx, sp);
            else
                out[i] = m.decomposition(i, t, sx, sp, std::span<const double>(xh, n),
                                         std::span<const double>(ph ? ph : x, ph ? ni : 0));
        }
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// Serial reference integrator (rk4_serial.cpp) of x' = f.
int ref_integrate(const po_model* pm, const double* x0, const double* p, double t0, double t1,
                  double h, uint64_t stride, double* times, double* states, uint64_t max_slots,
                  uint64_t* n_slots, char* err, int errlen) {
    try {
        const SystemModel m = build_model(pm);
        IntegrationJob job;
        job.model = &m;
        job.x0.assign(x0, x0 + m.dim);
        job.p.assign(p, p + m.input_dim);
        job.t0 = t0;
        job.t1 = t1;
        job.h = h;
        job.record_stride = stride;
        const Trajectory tr = reference::integrate(job);
        if (tr.times.size() > max_slots) throw std::length_error("ref_integrate: too many slots");
        for (std::size_t s = 0; s < tr.times.size(); ++s) {
            times[s] = tr.times[s];
            std::memcpy(states + s * m.dim, tr.states[s].data(), m.dim * sizeof(double));
        }
        *n_slots = tr.times.size();
        return 0;
    } catch (const IntegrationError& e) {
        set_err(err, errlen, e.what());
        return 2;
    } catch (const std::invalid_argument& e) {
        set_err(err, errlen, e.what());
        return 1;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 2;
    }
}

// method: 0 mixed_monotonicity, 1 growth_bound, 2 monte_carlo.
// report[0..3] = n, m, steps, peak_state_bytes; phases[0..2] = setup, integration, reduction.
int ref_reach(const po_model* pm, int method, const double* lo, const double* hi,
              const double* plo, const double* phi, double t0, double t1, double h,
              uint64_t stride, int workers, uint64_t samples, uint64_t seed, double eps,
              double delta, double* times, double* out_lo, double* out_hi, uint64_t max_slots,
              uint64_t* n_slots, uint64_t* report, double* phases, double* wall_s, char* err,
              int errlen) {
    try {
        const ReachProblem problem = build_problem(pm, lo, hi, plo, phi, t0, t1, h, stride);
        const auto start = std::chrono::steady_clock::now();
        ReachTube tube;
        if (method == 0) {
            tube = mixed_monotonicity(problem, workers);
        } else if (method == 1) {
            tube = growth_bound(problem, workers);
        } else {
            MonteCarloSpec spec;
            spec.epsilon = eps;
            spec.delta = delta;
            spec.seed = seed;
            spec.samples_override = samples;
            tube = monte_carlo(problem, spec, workers);
        }
        if (wall_s)
            *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
        const std::size_t n = problem.model.dim;
        if (tube.entries.size() > max_slots) throw std::length_error("ref_reach: too many slots");
        for (std::size_t s = 0; s < tube.entries.size(); ++s) {
            if (times) times[s] = tube.entries[s].t;
            if (out_lo)
                std::memcpy(out_lo + s * n, tube.entries[s].box.lower().data(), n * sizeof(double));
            if (out_hi)
                std::memcpy(out_hi + s * n, tube.entries[s].box.upper().data(), n * sizeof(double));
        }
        *n_slots = tube.entries.size();
        if (report) {
            report[0] = tube.report.n;
            report[1] = tube.report.m;
            report[2] = tube.report.steps;
            report[3] = tube.report.peak_state_bytes;
        }
        if (phases) {
            phases[0] = tube.report.phases.setup_s;
            phases[1] = tube.report.phases.integration_s;
            phases[2] = tube.report.phases.reduction_s;
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        set_err(err, errlen, e.what());
        return 1;
    } catch (const std::bad_alloc&) {
        set_err(err, errlen, "out of memory");
        return 5;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 2;
    }
}

int ref_coverage(const po_model* pm, const double* lo, const double* hi, const double* plo,
                 const double* phi, double t0, double t1, double h, const double* box_lo,
                 const double* box_hi, uint64_t fresh, uint64_t seed, double* fraction,
                 char* err, int errlen) {
    try {
        const ReachProblem problem = build_problem(pm, lo, hi, plo, phi, t0, t1, h, 0);
        const std::size_t n = problem.model.dim;
        ReachTube tube;
        tube.entries.push_back({t1, IntervalVector(std::vector<double>(box_lo, box_lo + n),
                                                   std::vector<double>(box_hi, box_hi + n))});
        *fraction = coverage_estimate(problem, MonteCarloSpec{}, tube, fresh, seed);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

}  // extern "C"
