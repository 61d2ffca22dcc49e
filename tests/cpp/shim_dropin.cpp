// Drop-in check of include/pirk/ivreach_gpu.hpp: reference-style C++ call
// sites (test_reach.cpp / acceptance.cpp idioms) compiled against the shim and
// run on the GPU.  Prints one line per check; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "pirk/ivreach_gpu.hpp"

using namespace ivreach;

static int failures = 0;
static void check(bool ok, const char* what) {
    std::printf("%s: %s\n", ok ? "ok" : "FAIL", what);
    std::fflush(stdout);
    if (!ok) ++failures;
}

int main(int argc, char** argv) {
    const double kE = 2.718281828459045;
    const std::string golden = argc > 1 ? argv[1] : "";  // tests/golden/io/traffic_mm.csv
    {   // test_reach.cpp:70-75
        ReachProblem p{make_scalar_linear(), IntervalVector({1.0}, {2.0}), std::nullopt, 0.0, 1.0, 0.001, 0};
        const ReachTube tube = mixed_monotonicity(p, 1);
        const IntervalVector& fin = tube.entries.back().box;
        check(std::fabs(fin.lower(0) - kE) <= 1e-4 && std::fabs(fin.upper(0) - 2 * kE) <= 1e-4,
              "mixed monotonicity exact on xdot = x");
    }
    {   // SURVEY.md 8c survey golden values of the reference (config 3 shape)
        const std::size_t n = 1000000;
        ReachProblem p{make_traffic(n), IntervalVector(std::vector<double>(n, 10.0), std::vector<double>(n, 20.0)),
                       IntervalVector({4.0}, {6.0}), 0.0, 30.0, 0.5, 0};
        const ReachTube t = mixed_monotonicity(p, 1);
        const IntervalVector& fin = t.entries.back().box;
        check(fin.lower(0) == 8.4261226388996242 && fin.upper(0) == 15.671837256973982 &&
                  fin.lower(n - 1) == 8.8249690258461371,
              "traffic n=1e6 CTMM bit-identical to the reference golden values");
        check(t.report.steps == 60 && t.report.peak_state_bytes == 112 * n, "report fields");
    }
    {   // test_reach.cpp:77-86
        check(sample_count(2, 0.05, 0.01) == 480 && sample_count(1, 0.5, 0.5) == 6, "sample_count");
    }
    {   // missing capability -> std::invalid_argument (test_reach.cpp:176-188)
        ReachProblem p{make_laub_loomis(), IntervalVector(std::vector<double>(7, 1.0), std::vector<double>(7, 1.1)),
                       std::nullopt, 0.0, 1.0, 0.1, 0};
        bool threw = false;
        try { mixed_monotonicity(p, 1); } catch (const std::invalid_argument&) { threw = true; }
        check(threw, "no decomposition -> invalid_argument");
    }
    {   // non-finite -> std::runtime_error naming the step (test_rk4.cpp:138-154)
        ReachProblem p{make_scalar_linear(5.0), IntervalVector({1.0}, {1.0}), std::nullopt, 0.0, 600.0, 10.0, 0};
        bool threw = false;
        try { mixed_monotonicity(p, 1); } catch (const std::runtime_error& e) {
            threw = std::string(e.what()).find("non-finite value at step") != std::string::npos;
        }
        check(threw, "integration failure -> runtime_error");
    }
    {   // Monte Carlo determinism in the seed (test_reach.cpp:88-111)
        ReachProblem p{make_traffic(6), IntervalVector(std::vector<double>(6, 10.0), std::vector<double>(6, 20.0)),
                       IntervalVector({4.0}, {6.0}), 0.0, 3.0, 0.5, 2};
        MonteCarloSpec s; s.seed = 42; s.samples_override = 64;
        const ReachTube a = monte_carlo(p, s, 1), b = monte_carlo(p, s, 8);
        check(a.entries.back().box == b.entries.back().box, "monte carlo deterministic across workers");
    }
    {   // driver.cpp dispatch + io.cpp tube_to_csv: byte-identical to the reference's file
        ReachProblem p{make_traffic(5), IntervalVector(std::vector<double>(5, 10.0), std::vector<double>(5, 20.0)),
                       IntervalVector({4.0}, {6.0}), 0.0, 3.0, 0.5, 2};
        const ReachTube t = dispatch("mixed-monotonicity", p, MonteCarloSpec{}, 1);
        std::ifstream f(golden, std::ios::binary);
        std::stringstream ss;
        ss << f.rdbuf();
        check(!golden.empty() && tube_to_csv(t) == ss.str(), "dispatch + tube_to_csv == reference io.cpp bytes");
        bool threw = false;
        try { dispatch("bogus", p, MonteCarloSpec{}, 1); } catch (const std::invalid_argument&) { threw = true; }
        check(threw, "dispatch: unknown method -> invalid_argument");
    }
    {   // workers -> shard lanes (ivreach_gpu::Device::current(workers)): the
        // sharded run is bit-identical to one lane
        const std::size_t n = 1000000;
        ReachProblem p{make_traffic(n), IntervalVector(std::vector<double>(n, 10.0), std::vector<double>(n, 20.0)),
                       IntervalVector({4.0}, {6.0}), 0.0, 30.0, 0.5, 10};
        const ReachTube one = mixed_monotonicity(p, 1), three = mixed_monotonicity(p, 3);
        bool same = one.entries.size() == three.entries.size();
        for (std::size_t s = 0; same && s < one.entries.size(); ++s)
            same = one.entries[s].t == three.entries[s].t && one.entries[s].box == three.entries[s].box;
        check(same, "traffic n=1e6 CTMM: mixed_monotonicity(p, 3) == mixed_monotonicity(p, 1)");
        const IntervalVector& fin = three.entries.back().box;
        check(fin.lower(0) == 8.4261226388996242 && fin.lower(n - 1) == 8.8249690258461371,
              "3-lane traffic CTMM bit-identical to the reference golden values");
        check(three.report.workers == 3, "report.workers == 3");
        const ReachTube g1 = growth_bound(p, 1), g3 = growth_bound(p, 3);
        check(g1.entries.back().box == g3.entries.back().box, "traffic GB: workers 3 == workers 1");
    }
    {   // heat3d z-slabs over 3 lanes
        const std::size_t g = 40, n = g * g * g;
        std::vector<double> lo(n), hi(n);
        for (std::size_t i = 0; i < n; ++i) { lo[i] = 0.9 + 0.001 * static_cast<double>(i % 13); hi[i] = lo[i] + 0.2; }
        const double h = 0.2 / 39.0 / 39.0;
        ReachProblem p{make_heat3d(g), IntervalVector(lo, hi), std::nullopt, 0.0, 6 * h, h, 2};
        const ReachTube a = mixed_monotonicity(p, 1), b = mixed_monotonicity(p, 3);
        bool same = a.entries.size() == b.entries.size();
        for (std::size_t s = 0; same && s < a.entries.size(); ++s) same = a.entries[s].box == b.entries[s].box;
        check(same, "heat3d g=40 CTMM: workers 3 == workers 1");
    }
    {   // Monte Carlo sample ranges over 3 lanes, hull folded exactly
        ReachProblem p{make_laub_loomis(), IntervalVector({1.15, 1.0, 1.45, 2.35, 0.95, 0.05, 0.4},
                                                          {1.25, 1.1, 1.55, 2.45, 1.05, 0.15, 0.5}),
                       std::nullopt, 0.0, 1.0, 0.01, 10};
        MonteCarloSpec s; s.seed = 3; s.samples_override = 10007;
        const ReachTube a = monte_carlo(p, s, 1), b = monte_carlo(p, s, 3);
        bool same = a.entries.size() == b.entries.size();
        for (std::size_t k = 0; same && k < a.entries.size(); ++k) same = a.entries[k].box == b.entries[k].box;
        check(same, "laub-loomis MC: workers 3 == workers 1");
    }
    {   // test_reach.cpp:190-206 through the shim: a user decomposition that
        // violates the embedding order is a runtime_error, as in the reference
        const std::string src = R"(
__device__ double pirk_rhs(u64 i, double, const double* x, const double*) { return i == 0 ? x[1] : -1.0; }
__device__ double pirk_decomposition(u64 i, double, const double*, const double*, const double* xh,
                                     const double*) { return i == 0 ? xh[1] : -1.0; })";
        SystemModel m = make_user_model(src, 2, 0, true, false, false);
        ReachProblem p{m, IntervalVector({0.0, 0.0}, {1.0, 0.5}), std::nullopt, 0.0, 3.0, 0.1, 1};
        bool threw = false;
        try { mixed_monotonicity(p, 1); } catch (const std::runtime_error& e) {
            threw = std::string(e.what()) == "mixed-monotonicity: embedding order violated at step 20, t = 2.000000, component 0";
        }
        check(threw, "user model: order-violating decomposition -> runtime_error (reference message)");
        bool invalid = false;
        try { growth_bound(p, 1); } catch (const std::invalid_argument&) { invalid = true; }
        check(invalid, "user model without growth_rhs: growth_bound -> invalid_argument");
        SystemModel bad = make_user_model("__device__ double pirk_rhs(u64, double, const double*, const double*) { return nope; }",
                                          1, 0, false, false, false);
        ReachProblem pb{bad, IntervalVector({0.0}, {1.0}), std::nullopt, 0.0, 1.0, 0.1, 0};
        bool bad_src = false;
        try { monte_carlo(pb, MonteCarloSpec{}, 1); } catch (const std::invalid_argument& e) {
            bad_src = std::string(e.what()).find("nope") != std::string::npos;
        }
        check(bad_src, "user model that does not compile -> invalid_argument with the NVRTC log");
    }
    return failures;
}
