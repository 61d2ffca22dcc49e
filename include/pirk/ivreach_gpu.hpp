// ivreach_gpu.hpp -- header-only C++ shim over pirk_c.h that keeps the
// reference's C++ interface (namespace ivreach, /root/reference/proj/include/
// ivreach/{interval,system_model,reach,models}.hpp) so a C++ caller can switch
// its #include and link line and keep its call sites:
//
//     ivreach::ReachTube t = ivreach::mixed_monotonicity(problem, workers);
//
// Differences, all forced by running on a GPU:
//  * SystemModel is a descriptor (kind + parameters + decomposition choice),
//    made by the same make_* constructors, not a bag of std::function: the
//    vector fields are compiled device functors.  A model the device library
//    does not implement throws std::invalid_argument("... no device kernel ...")
//    -- there is no CPU fallback.
//  * `workers` must be >= 1 (as in the reference); it selects the number of
//    shard lanes (ivreach_gpu::Device::current(workers)): chain / heat3d runs
//    shard the state across them and Monte Carlo the samples, bit-identical
//    to workers = 1.
// Exceptions and messages are the reference's: std::invalid_argument for
// validation and missing capability, std::runtime_error for integration
// failure, order violation and negative radius (reach.cpp:66-72, 107-117,
// 140-144, 181-192, 306-312), std::bad_alloc for memory exhaustion.
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <new>
#include <optional>
#include <stdexcept>
#include <cstdio>
#include <string>
#include <vector>

#include "../pirk_c.h"

namespace ivreach_gpu {

class Device {
public:
    explicit Device(int device = 0, pirk_mode mode = PIRK_MODE_EXACT) : Device(std::vector<int>{device}, mode) {}
    // One shard lane per entry of `devices` (ids may repeat), see pirk_create_multi.
    explicit Device(const std::vector<int>& devices, pirk_mode mode = PIRK_MODE_EXACT) {
        if (pirk_create_multi(static_cast<int>(devices.size()), devices.data(), &ctx_) != PIRK_OK)
            throw std::runtime_error("pirk_create: no usable CUDA device " + std::to_string(devices.at(0)));
        pirk_set_mode(ctx_, mode);
    }
    ~Device() { pirk_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    pirk_ctx* get() const { return ctx_; }
    void set_mode(pirk_mode m) { pirk_set_mode(ctx_, m); }
    int lanes() const { return pirk_lane_count(ctx_); }

    // The context a reference call with `workers` runs on: `workers` shard
    // lanes spread round-robin over the visible GPUs (workers == GPU count puts
    // one shard on each GPU; on a one-GPU box the lanes share it).  One set of
    // contexts per calling thread, so concurrent reference calls from distinct
    // threads run on distinct contexts and streams.  Never
    // destroyed: releasing CUDA resources from a static/thread-exit destructor
    // can race the CUDA runtime's own teardown at exit.
    static Device& current(int workers = 1) {
        thread_local std::map<int, Device*> per_thread;
        Device*& d = per_thread[workers];
        if (!d) {
            int count = pirk_device_count();
            if (count < 1) count = 1;  // pirk_create_multi then reports the missing device
            std::vector<int> devs(static_cast<std::size_t>(workers < 1 ? 1 : workers));
            for (std::size_t r = 0; r < devs.size(); ++r) devs[r] = static_cast<int>(r % static_cast<std::size_t>(count));
            d = new Device(devs);
        }
        return *d;
    }

private:
    pirk_ctx* ctx_ = nullptr;
};

inline void throw_status(pirk_status st, pirk_ctx* ctx) {
    const std::string msg = pirk_last_error(ctx);
    switch (st) {
        case PIRK_OK: return;
        case PIRK_EINVAL: throw std::invalid_argument(msg);
        case PIRK_EUNSUPPORTED: throw std::invalid_argument(msg);
        case PIRK_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

}  // namespace ivreach_gpu

namespace ivreach {

// ------------------------------------------------------------ interval.hpp
class IntervalVector {
public:
    IntervalVector(std::vector<double> lower, std::vector<double> upper)
        : lower_(std::move(lower)), upper_(std::move(upper)) {
        if (lower_.size() != upper_.size())
            throw std::invalid_argument("interval: lower has " + std::to_string(lower_.size()) +
                                        " components, upper has " + std::to_string(upper_.size()));
        if (lower_.empty()) throw std::invalid_argument("interval: dimension must be at least 1");
        for (std::size_t i = 0; i < lower_.size(); ++i) {
            if (!std::isfinite(lower_[i]) || !std::isfinite(upper_[i]))
                throw std::invalid_argument("interval: non-finite bound at component " + std::to_string(i));
            if (lower_[i] > upper_[i])
                throw std::invalid_argument("interval: lower > upper at component " + std::to_string(i));
        }
    }
    std::size_t dim() const { return lower_.size(); }
    const std::vector<double>& lower() const { return lower_; }
    const std::vector<double>& upper() const { return upper_; }
    double lower(std::size_t i) const { return lower_[i]; }
    double upper(std::size_t i) const { return upper_[i]; }
    bool operator==(const IntervalVector& o) const = default;

private:
    std::vector<double> lower_, upper_;
};

// -------------------------------------------------------- system_model.hpp
struct SystemModel {
    pirk_model desc{};
    std::size_t dim = 0;
    std::size_t input_dim = 0;
    bool input_affine = true;
    std::string sparsity_note;
    // user-defined evaluators (make_user_model); shared by copies of the model
    std::shared_ptr<pirk_program> program;
    bool has_growth() const {
        if (desc.kind == PIRK_USER) return user_flags & PIRK_HAS_GROWTH;
        return desc.kind != PIRK_CHAIN;
    }
    bool has_decomposition() const {
        if (desc.kind == PIRK_USER) return user_flags & PIRK_HAS_DECOMPOSITION;
        return desc.decomp != PIRK_DECOMP_NONE;
    }
    std::uint32_t user_flags = 0;
};

struct ReachProblem {
    SystemModel model;
    IntervalVector initial;
    std::optional<IntervalVector> inputs;
    double t0 = 0.0;
    double t1 = 0.0;
    double h = 0.0;
    std::size_t tube_stride = 0;
};

// --------------------------------------------------------------- models.hpp
namespace detail {
inline SystemModel make(int kind, std::size_t dim, std::size_t ni, std::vector<double> p,
                        int decomp, std::size_t grid = 0) {
    SystemModel m;
    m.desc.kind = kind;
    m.desc.decomp = decomp;
    m.desc.dim = dim;
    m.desc.input_dim = ni;
    m.desc.grid = grid;
    for (std::size_t i = 0; i < p.size() && i < 8; ++i) m.desc.params[i] = p[i];
    m.dim = dim;
    m.input_dim = ni;
    return m;
}
inline void require(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}
}  // namespace detail

inline SystemModel make_traffic(std::size_t segments, double v = 0.5, double w = 1.0 / 6.0,
                                double c = 40.0, double xbar = 320.0, double period = 30.0,
                                double beta = 0.75) {
    detail::require(segments >= 3, "traffic model needs at least 3 segments");
    detail::require(v > 0 && w > 0 && c > 0 && xbar > 0 && period > 0,
                    "traffic parameters must be positive");
    detail::require(beta > 0 && beta <= 1, "traffic beta must lie in (0, 1]");
    return detail::make(PIRK_TRAFFIC, segments, 1, {v, w, c, xbar, period, beta}, PIRK_DECOMP_NATIVE);
}
inline SystemModel make_heat3d(std::size_t grid, double alpha = 1.0, double exchange = 1.0) {
    detail::require(grid >= 2, "heat3d model needs at least 2 grid points per axis");
    detail::require(alpha > 0, "heat3d alpha must be positive");
    detail::require(exchange >= 0, "heat3d exchange coefficient must be nonnegative");
    return detail::make(PIRK_HEAT3D, grid * grid * grid, 0, {alpha, exchange}, PIRK_DECOMP_NATIVE, grid);
}
inline SystemModel make_chain(std::size_t n, double a = 1.0, double b = 0.5, double c = 0.25) {
    return detail::make(PIRK_CHAIN, n, 1, {a, b, c}, PIRK_DECOMP_NATIVE);
}
inline SystemModel make_laub_loomis() { return detail::make(PIRK_LAUB_LOOMIS, 7, 0, {}, PIRK_DECOMP_NONE); }
inline SystemModel make_arch_quadrotor(double mass = 1.4, double gravity = 9.81, double jx = 0.054,
                                       double jy = 0.054, double jz = 0.104) {
    return detail::make(PIRK_ARCH_QUAD, 12, 0, {mass, gravity, jx, jy, jz}, PIRK_DECOMP_NONE);
}
inline SystemModel make_vdp(double mu = 1.0, double op_x = 2.5, double op_y = 3.0) {
    return detail::make(PIRK_VDP, 2, 0, {mu, op_x, op_y}, PIRK_DECOMP_NONE);
}
inline SystemModel make_zero(std::size_t dim = 2) { return detail::make(PIRK_ZERO, dim, 0, {}, PIRK_DECOMP_NATIVE); }
inline SystemModel make_scalar_decay() { return detail::make(PIRK_SCALAR_DECAY, 1, 1, {}, PIRK_DECOMP_NATIVE); }
inline SystemModel make_scalar_linear(double a = 1.0) {
    return detail::make(PIRK_SCALAR_LINEAR, 1, 0, {a}, PIRK_DECOMP_NATIVE);
}
// A model with caller-written evaluators -- the reference's SystemModel built
// from arbitrary std::function rhs / decomposition / growth_rhs
// (system_model.hpp:14-43) -- as CUDA device functions with the same arguments:
//
//   __device__ double pirk_rhs(u64 i, double t, const double* x, const double* p);
//   __device__ double pirk_decomposition(u64 i, double t, const double* x, const double* p,
//                                        const double* xh, const double* ph);
//   __device__ double pirk_growth(u64 i, double t, const double* r, const double* w);
//
// compiled by NVRTC for sm_100a on first use (pirk_c.h).  A source that does
// not compile is reported by the entry points as std::invalid_argument with
// the compiler's log.
inline SystemModel make_user_model(const std::string& source, std::size_t dim, std::size_t input_dim,
                                   bool has_decomposition, bool has_growth, bool input_affine) {
    detail::require(dim >= 1, "user model needs at least 1 state");
    const std::uint32_t flags = PIRK_HAS_RHS | (has_decomposition ? PIRK_HAS_DECOMPOSITION : 0u) |
                                (has_growth ? PIRK_HAS_GROWTH : 0u) | (input_affine ? PIRK_INPUT_AFFINE : 0u);
    pirk_program* raw = nullptr;
    if (pirk_program_create(source.c_str(), dim, input_dim, flags, &raw) != PIRK_OK)
        throw std::invalid_argument("user model: invalid source or dimension");
    SystemModel m = detail::make(PIRK_USER, dim, input_dim, {}, has_decomposition ? PIRK_DECOMP_NATIVE : PIRK_DECOMP_NONE);
    m.program.reset(raw, pirk_program_destroy);
    m.desc.program = raw;
    m.user_flags = flags;
    m.input_affine = input_affine;
    return m;
}

// User-supplied decomposition d_i = f_i(x) + sum_{j!=i} C_ij (x_j - xh_j) (see pirk_c.h).
inline SystemModel with_jacobian_decomposition(SystemModel m) {
    m.desc.decomp = PIRK_DECOMP_JACOBIAN;
    return m;
}

// ---------------------------------------------------------------- reach.hpp
struct PhaseTimes {
    double setup_s = 0.0, integration_s = 0.0, reduction_s = 0.0;
};
struct RunReport {
    std::string method;
    std::size_t n = 0, m = 0;
    int workers = 1;
    std::size_t steps = 0, peak_state_bytes = 0;
    PhaseTimes phases;
};
struct TubeEntry {
    double t;
    IntervalVector box;
};
struct ReachTube {
    std::string method;
    std::vector<TubeEntry> entries;
    RunReport report;
};
struct MonteCarloSpec {
    double epsilon = 0.05;
    double delta = 0.01;
    std::uint64_t seed = 1;
    std::size_t samples_override = 0;
};

namespace detail {
struct Marshal {
    pirk_problem p{};
    explicit Marshal(const ReachProblem& pr) {
        p.init_lower = pr.initial.lower().data();
        p.init_upper = pr.initial.upper().data();
        p.input_lower = pr.inputs ? pr.inputs->lower().data() : nullptr;
        p.input_upper = pr.inputs ? pr.inputs->upper().data() : nullptr;
        p.t0 = pr.t0;
        p.t1 = pr.t1;
        p.h = pr.h;
        p.tube_stride = pr.tube_stride;
    }
};

template <typename Call>
ReachTube run(const ReachProblem& pr, int workers, const char* method, Call&& call) {
    if (workers < 1)
        throw std::invalid_argument(std::string(method) + ": workers must be >= 1");
    if (pr.initial.dim() != pr.model.dim)
        throw std::invalid_argument("problem: initial box dim " + std::to_string(pr.initial.dim()) +
                                    " does not match model dim " + std::to_string(pr.model.dim));
    auto& dev = ivreach_gpu::Device::current(workers);
    Marshal mar(pr);
    const std::size_t n = pr.model.dim;
    const std::uint64_t slots = pirk_record_schedule(pr.t0, pr.t1, pr.h, pr.tube_stride, nullptr, nullptr);
    std::vector<double> times(slots ? slots : 1), lo(slots * n), hi(slots * n);
    pirk_tube tube{times.data(), lo.data(), hi.data(), slots, 0};
    pirk_report rep{};
    ivreach_gpu::throw_status(call(dev.get(), &pr.model.desc, &mar.p, &tube, &rep), dev.get());
    ReachTube out;
    out.method = method;
    for (std::uint64_t s = 0; s < tube.n_slots; ++s)
        out.entries.push_back({times[s], IntervalVector(std::vector<double>(lo.begin() + s * n, lo.begin() + (s + 1) * n),
                                                        std::vector<double>(hi.begin() + s * n, hi.begin() + (s + 1) * n))});
    out.report.method = method;
    out.report.n = rep.n;
    out.report.m = rep.m;
    out.report.workers = workers;
    out.report.steps = rep.steps;
    out.report.peak_state_bytes = rep.peak_state_bytes;
    out.report.phases = {rep.setup_s, rep.integration_s, rep.reduction_s};
    return out;
}
}  // namespace detail

inline std::size_t sample_count(std::size_t n, double epsilon, double delta) {
    std::uint64_t out = 0;
    if (n == 0) throw std::invalid_argument("sample_count: n must be positive");
    if (!(epsilon > 0.0) || !(epsilon < 1.0))
        throw std::invalid_argument("sample_count: epsilon must be in (0, 1)");
    if (!(delta > 0.0) || !(delta < 1.0))
        throw std::invalid_argument("sample_count: delta must be in (0, 1)");
    pirk_sample_count(n, epsilon, delta, &out);
    return out;
}

inline ReachTube growth_bound(const ReachProblem& problem, int workers) {
    return detail::run(problem, workers, "growth-bound", [](auto c, auto m, auto p, auto t, auto r) {
        return pirk_growth_bound(c, m, p, t, r);
    });
}
inline ReachTube mixed_monotonicity(const ReachProblem& problem, int workers) {
    return detail::run(problem, workers, "mixed-monotonicity", [](auto c, auto m, auto p, auto t, auto r) {
        return pirk_mixed_monotonicity(c, m, p, t, r);
    });
}
inline ReachTube monte_carlo(const ReachProblem& problem, const MonteCarloSpec& spec, int workers) {
    pirk_mc_spec s{spec.epsilon, spec.delta, spec.seed, spec.samples_override};
    ReachTube t = detail::run(problem, workers, "monte-carlo", [&](auto c, auto m, auto p, auto tb, auto r) {
        return pirk_monte_carlo(c, m, p, &s, tb, r);
    });
    return t;
}

// driver.cpp:28-34: route a method name to its entry point.
inline ReachTube dispatch(const std::string& method, const ReachProblem& problem, const MonteCarloSpec& mc,
                          int workers) {
    if (method == "growth-bound") return growth_bound(problem, workers);
    if (method == "mixed-monotonicity") return mixed_monotonicity(problem, workers);
    if (method == "monte-carlo") return monte_carlo(problem, mc, workers);
    throw std::invalid_argument("unknown method: " + method);
}

// io.cpp:84-103: `t,lower0,upper0,...` with %.17g values, byte-identical to
// the reference's tube_to_csv.
inline std::string tube_to_csv(const ReachTube& tube) {
    auto put = [](std::string& out, double v) {
        char buf[32];
        std::snprintf(buf, sizeof(buf), "%.17g", v);
        out += buf;
    };
    std::string out = "t";
    const std::size_t n = tube.entries.empty() ? 0 : tube.entries.front().box.dim();
    for (std::size_t i = 0; i < n; ++i) {
        out += ",lower" + std::to_string(i);
        out += ",upper" + std::to_string(i);
    }
    out += "\n";
    for (const auto& e : tube.entries) {
        put(out, e.t);
        for (std::size_t i = 0; i < e.box.dim(); ++i) {
            out += ',';
            put(out, e.box.lower(i));
            out += ',';
            put(out, e.box.upper(i));
        }
        out += '\n';
    }
    return out;
}

}  // namespace ivreach
