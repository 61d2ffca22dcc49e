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
    return failures;
}
