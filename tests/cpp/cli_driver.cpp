// cli_driver.cpp -- drives the command layer and JSON views (tmatch/cli.hpp,
// tmatch/serialize.hpp) for tests/test_cli.py.  Built twice from this one source: against
// this repo's headers + libtmatch.so (paper_1407_3535_b200/lib/cli_driver) and, with
// -DTM_REF, against the reference's headers + the reference library compiled by
// oracle/Makefile (oracle/_ref/cli_driver_ref, which also offers the reference's synth).
//   cli_driver json                              -> three JSON dumps of fixed records
//   cli_driver bench <corpus> <csv> <modes,..> [parallel]
//   cli_driver match <template.pgm> <image.pgm> <out.json> <mode> [parallel]  (exit code)
//   cli_driver_ref synth <dir> <rows> <cols> <images> <size> <per_size> <seed>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "tmatch/cli.hpp"
#include "tmatch/serialize.hpp"

using namespace tmatch;

static std::vector<std::string> split(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string x;
    while (std::getline(ss, x, ',')) out.push_back(x);
    return out;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string cmd = argv[1];
    if (cmd == "json") {
        MatchResult r;
        r.mode = MatchMode::opta;
        r.best_row = 17;
        r.best_col = 23;
        r.best_rho = 0.9562393943290236;
        r.refined_row = 18;
        r.refined_col = 22;
        r.refined_rho = 0.97150000000000003;
        r.below_threshold = true;
        r.stats.centers = 438244;
        r.stats.eliminated = 3501937;
        r.stats.retained = 44;
        r.stats.elim_pct = 88.8765743073048;
        r.stats.ops = 438288;
        r.stats.wall_ms = 0.28125;
        std::cout << to_json(r).dump() << "\n";
        EGSResult e;
        e.h = e.w = 5;
        for (int h = 3; h <= 5; h += 2) {
            EgsIteration it;
            it.h = it.w = h;
            it.cost.total = 1234.5 / h;
            e.trace.push_back(it);
        }
        e.cost.total = e.trace.back().cost.total;
        std::cout << to_json(e).dump() << "\n";
        OptAResult o;
        o.egs = e;
        o.kappa = 2;
        o.lambda = 0.9473499399519517;
        o.trace.push_back(OptAIteration{5, 5, 100.25, 205});
        o.trace.push_back(OptAIteration{5, 5, 99.5, 957});
        std::cout << opta_sidecar(o).dump() << "\n";
        return 0;
    }
    if (cmd == "bench" && argc >= 5) {
        cli::BenchOptions b;
        b.corpus_dir = argv[2];
        b.out_csv = argv[3];
        b.out_json = std::string(argv[3]) + ".json";
        b.modes = split(argv[4]);
        if (argc >= 6 && std::string(argv[5]) == "parallel") {
            b.params.parallel = true;
            b.params.threads = 4;
        }
        b.quiet = true;
        return cli::cmd_bench(b);
    }
    if (cmd == "match" && argc >= 6) {
        cli::MatchOptions o;
        o.template_path = argv[2];
        o.image_path = argv[3];
        o.out_path = argv[4];
        const std::string mode = argv[5];
        o.params.mode = mode == "brute" ? MatchMode::brute
                        : mode == "opta" ? MatchMode::opta : MatchMode::egs;
        if (argc >= 7 && std::string(argv[6]) == "parallel") {
            o.params.parallel = true;
            o.params.threads = 4;
        }
        return cli::cmd_match(o);
    }
#ifdef TM_REF
    if (cmd == "synth" && argc == 9) {
        cli::SynthOptions s;
        s.out_dir = argv[2];
        s.spec.image.rows = std::atoi(argv[3]);
        s.spec.image.cols = std::atoi(argv[4]);
        s.spec.image_count = std::atoi(argv[5]);
        s.spec.template_sizes = {std::atoi(argv[6])};
        s.spec.per_size = std::atoi(argv[7]);
        s.spec.seed = std::strtoull(argv[8], nullptr, 10);
        return cli::cmd_synth(s);
    }
#endif
    return 2;
}
