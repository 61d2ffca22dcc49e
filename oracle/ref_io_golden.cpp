// ref_io_golden.cpp -- TEST INFRASTRUCTURE ONLY.  Writes golden serialisations
// produced by the UNMODIFIED reference (io.cpp, driver.cpp's bench_csv) for the
// format tests (tests/test_formats.py).  Built by `make -C oracle golden-io`
// against the reference sources in place; run once here, outputs committed
// under tests/golden/io/ together with this program.
//
//   traffic_mm.csv / .json : ivreach::mixed_monotonicity on make_traffic(5),
//                            box [10,20], p in [4,6], t in [0,3], h=0.5, stride 2,
//                            report phases fixed to (0.25, 0.5, 0.125)
//   synthetic.json         : a hand-built tube exercising nlohmann's double
//                            formatting (tiny, huge, negative, integral values)
//   bench.csv              : bench_csv over three synthetic rows
//   configs/<name>.parsed  : serialize_config(parse_config_file(proj/configs/<name>.cfg))
//   configs/errors.tsv     : parse_config's invalid_argument message per bad config text
//   configs/<name>.json    : run_config's tube file (and .report.json) for the
//                            configs the device library supports (`<dir> configs <cfgdir>`)
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include <filesystem>
#include <stdexcept>

#include "ivreach/config.hpp"
#include "ivreach/driver.hpp"
#include "ivreach/io.hpp"
#include "ivreach/models.hpp"
#include "ivreach/reach.hpp"

using namespace ivreach;

static void put(const std::string& dir, const std::string& name, const std::string& text) {
    std::ofstream f(dir + "/" + name, std::ios::binary);
    f << text;
}

static int configs(const std::string& dir, const std::string& cfgdir) {
    namespace fs = std::filesystem;
    fs::create_directories(dir);
    for (const auto& e : fs::directory_iterator(cfgdir)) {
        if (e.path().extension() != ".cfg") continue;
        const std::string name = e.path().stem().string();
        RunConfig cfg = parse_config_file(e.path().string());
        put(dir, name + ".parsed", serialize_config(cfg));
        static const char* runnable[] = {"traffic", "heat3d", "laub-loomis", "arch-quadrotor", "vdp",
                                         "vdp-mc", "scalar-decay", "scalar-linear"};
        bool run = false;
        for (const char* r : runnable) run = run || name == r;
        if (!run) continue;
        cfg.output = dir + "/" + name;
        cfg.workers = 1;
        run_config(cfg);
    }
    // parse errors (config.cpp messages, with line numbers)
    const std::vector<std::pair<std::string, std::string>> bad = {
        {"no_model", "method = growth-bound\n"},
        {"unknown_key", "model = vdp\ncolour = red\n"},
        {"no_equals", "model = vdp\njust words\n"},
        {"unknown_model", "model = banana\n"},
        {"unknown_param", "model = vdp\nparam.nope = 1\n"},
        {"bad_number", "model = vdp\nt1 = 1.0x\n"},
        {"bad_method", "model = vdp\nmethod = magic\n"},
        {"unsupported_method", "model = vdp\nmethod = mixed-monotonicity\n"},
        {"box_length", "model = vdp\ninitial.lower = 1, 2, 3\n"},
        {"inputs_on_autonomous", "model = vdp\ninput.lower = 1\n"},
        {"negative_stride", "model = vdp\ntube_stride = -1\n"},
        {"epsilon_range", "model = vdp\nepsilon = 1.5\n"},
        {"bad_format", "model = vdp\nformat = xml\n"},
        {"bad_grid", "model = heat3d\nparam.grid = 2.5\n"},
        {"empty_param", "model = vdp\nparam. = 1\n"},
        {"empty_vector", "model = traffic\ninitial.lower = \n"},
        {"too_many_workers", "model = vdp\nworkers = 5000\n"},
    };
    std::string tsv;
    for (const auto& [k, text] : bad) {
        std::string msg = "(no error)";
        try { parse_config(text); } catch (const std::invalid_argument& e) { msg = e.what(); }
        tsv += k + "\t" + msg + "\n";
    }
    put(dir, "errors.tsv", tsv);
    return 0;
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    if (argc > 3 && std::string(argv[2]) == "configs") return configs(dir, argv[3]);
    SystemModel m = make_traffic(5);
    ReachProblem p{m, IntervalVector(std::vector<double>(5, 10.0), std::vector<double>(5, 20.0)),
                   IntervalVector(std::vector<double>{4.0}, std::vector<double>{6.0}), 0.0, 3.0, 0.5, 2};
    ReachTube tube = mixed_monotonicity(p, 1);
    tube.report.phases = PhaseTimes{0.25, 0.5, 0.125};
    put(dir, "traffic_mm.csv", tube_to_csv(tube));
    put(dir, "traffic_mm.json", tube_to_json(tube));

    ReachTube syn;
    syn.method = "monte-carlo";
    syn.entries.push_back(TubeEntry{0.0, IntervalVector({-1e-05, 1.0, 123456789.0, -0.1},
                                                        {1e-300, 1e+20, 1.2345678901234567e+16, 2.5})});
    syn.entries.push_back(TubeEntry{0.1, IntervalVector({-3.0, 1.0 / 3.0, 5e-324, 1e15},
                                                        {-2.0, 2.0 / 3.0, 1e-4, 1e16})});
    syn.report.method = "monte-carlo";
    syn.report.n = 4;
    syn.report.m = 1000;
    syn.report.workers = 3;
    syn.report.steps = 7;
    syn.report.peak_state_bytes = 123456;
    syn.report.phases = PhaseTimes{1.5e-06, 2.0, 0.0};
    put(dir, "synthetic.json", tube_to_json(syn));
    put(dir, "synthetic.report.json", report_to_json(syn.report));

    std::vector<BenchRow> rows(3);
    rows[0] = BenchRow{1000, 1, 0.0123456789, 60, "ok"};
    rows[1] = BenchRow{1000, 8, 0.5, 60, "ok"};
    rows[2] = BenchRow{64, 2, 0.0, 0, "error: bad, input"};
    put(dir, "bench.csv", bench_csv(rows));
    return 0;
}
