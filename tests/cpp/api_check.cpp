// api_check.cpp -- drives the reference C++ API (include/tmatch/*.hpp) of the B200 build
// the way the reference's own tests and acceptance program do, and prints one line per
// check.  Built by __graft_entry__.build(); run by tests/test_cpp_api.py on a GPU.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "tmatch/bounds.hpp"
#include "tmatch/detail.hpp"
#include "tmatch/matcher.hpp"

using namespace tmatch;

static int g_fail = 0;
static void check(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++g_fail;
}

static Image smooth_image(int rows, int cols, unsigned seed) {
    std::mt19937 rng(seed);
    std::normal_distribution<double> nd(0.0, 1.0);
    Image raw(rows, cols);
    for (double& v : raw.data()) v = nd(rng);
    Image out = blur(blur(raw, BlurKernel::default_profile()), BlurKernel::default_profile());
    double lo = 1e300, hi = -1e300;
    for (double v : out.data()) lo = std::min(lo, v), hi = std::max(hi, v);
    for (double& v : out.data()) v = std::round((v - lo) / (hi - lo) * 255.0);
    return out;
}

int main() {
    const Image I = smooth_image(160, 200, 7);
    Image t(21, 17);
    for (int r = 0; r < 21; ++r)
        for (int c = 0; c < 17; ++c) t(r, c) = std::min(255.0, std::round(I(60 + r, 90 + c) * 0.9 + 8));

    const MatchResult brute = brute_force_match(t, I);
    check(brute.best_row == 60 && brute.best_col == 90, "brute finds the planted template");

    MatchParams p;
    const MatchResult egs = match(t, I, p);
    check(egs.best_row == brute.best_row && egs.best_col == brute.best_col &&
              egs.best_rho == brute.best_rho, "match(egs) == brute (location and rho bits)");
    p.mode = MatchMode::opta;
    const MatchResult opta = match(t, I, p);
    check(opta.refined_row == brute.best_row && opta.refined_col == brute.best_col,
          "match(opta) refined == brute");

    MatchParams q;
    const PreparedEgs pe = prepare_egs(I, 21, 17, q);
    const MatchResult r1 = run_egs(t, I, pe, q);
    check(r1.best_rho == egs.best_rho && r1.stats.eliminated == egs.stats.eliminated,
          "prepare_egs + run_egs == match(egs), skip count included");
    const MatchResult r2 = transitive_search(t, I, pe.egs.map, pe.egs.grid);
    check(r2.best_row == r1.best_row && r2.stats.eliminated == r1.stats.eliminated,
          "transitive_search on the host map == run_egs");
    check(pe.egs.cost.retained == retained_count(pe.egs.map, q.rho_th),
          "EGS cost n_r == retained_count(map) (acceptance c6)");
    check(pe.egs.cost.central == double(pe.egs.grid.group_count()), "c_c == group count");

    const WindowStats ws = window_stats(I, 21, 17);
    const detail::TemplateStats ts = detail::template_stats(t);
    const double direct = detail::zncc_at(t, ts, I, ws, brute.best_row, brute.best_col);
    check(direct == brute.best_rho, "host zncc_at == device rho (bit exact)");

    const CenterScan cs = center_scan(t, I, pe.egs.grid);
    bool cs_ok = cs.rho.size() == pe.egs.grid.groups().size();
    for (std::size_t g = 0; cs_ok && g < cs.rho.size(); g += 97) {
        const Group& gr = pe.egs.grid.groups()[g];
        cs_ok = cs.rho[g] == detail::zncc_at(t, ts, I, ws, gr.center_row, gr.center_col);
    }
    check(cs_ok, "center_scan rho == zncc_at at sampled centres");

    const BestCell rf = refine_localization(t, I, 58, 93, 4);
    check(rf.row == 60 && rf.col == 90, "refine_localization recovers the offset");

    const BoundPair b = transitive_bounds(0.61, 0.81);
    check(std::abs(b.lower - 0.0294) < 1e-4 && std::abs(b.upper - 0.9588) < 1e-4,
          "bound algebra (0.61, 0.81)");
    check(std::abs(quality_threshold(0.8, 0.95) - 0.947349939) < 1e-6, "lambda(0.8, 0.95)");

    const PreparedOptA po = prepare_opta(I, 21, 17, q);
    const FidelityMap fid = blur_fidelity_map(I, po.opta.image, 21, 17);
    long long bad = 0;
    for (double v : fid.values) bad += (v < po.opta.lambda - 1e-6 && v != 0.0);
    check(po.opta.kappa >= 0 && po.opta.trace.size() == std::size_t(po.opta.kappa) + 1,
          "OptA trace carries kappa+1 accepted iterations");

    {
        // a caller edits the Image in place between prepare_egs and run_egs: the device copy
        // of the preparation must not serve the stale pixels (the reference always
        // correlates against the current contents of I)
        Image J = I;
        const PreparedEgs pj = prepare_egs(J, 21, 17, q);
        const MatchResult stale = run_egs(t, J, pj, q);  // served by the device preparation
        for (int r = 0; r < 21; ++r)
            for (int c = 0; c < 17; ++c) J(100 + r, 150 + c) = t(r, c);  // plant an exact copy
        const MatchResult after = run_egs(t, J, pj, q);
        std::printf("  (stale %d,%d %.6f; after edit %d,%d %.6f)\n", stale.best_row,
                    stale.best_col, stale.best_rho, after.best_row, after.best_col,
                    after.best_rho);
        // (the prepared statistics are the old pixels', so windows over the planted copy
        // score up to the clamp at 1: the reference semantics, checked bit for bit against
        // the oracle in tests/test_gpu_parity.py::test_transitive_search_with_prepared_statistics)
        check(stale.best_row == 60 && stale.best_col == 90 && after.best_rho == 1.0 &&
                  after.best_row >= 100 - 20 && after.best_row <= 100 + 20 &&
                  after.best_col >= 150 - 16 && after.best_col <= 150 + 16,
              "run_egs after an in-place edit sees the current pixels");
    }

    {
        // amortised EGS cost (egs.cpp:65-67): include_autocorr_cost is honoured
        EgsParams ep;
        ep.include_autocorr_cost = true;
        ep.n_templates = 4;
        const EGSResult ea = efficient_group_size(I, 21, 17, ep);
        const double extent = double(I.rows() - 20) * double(I.cols() - 16);
        bool am_ok = !ea.trace.empty();
        for (const auto& it : ea.trace)
            am_ok = am_ok && it.cost.amortized ==
                                 (double(it.h) * it.w - 1.0) * extent / (21.0 * 17.0 * 4);
        check(am_ok && ea.map.values.size() == std::size_t(extent),
              "efficient_group_size with include_autocorr_cost (amortised term)");
    }

    try {
        Image flat(5, 5, 3.0);
        match(flat, I, MatchParams{});
        check(false, "constant template rejected");
    } catch (const std::invalid_argument& e) {
        check(std::string(e.what()).find("constant template") != std::string::npos,
              "constant template rejected with the reference message");
    }
    std::printf("api_check: %s\n", g_fail ? "FAILURES" : "ALL PASS");
    return g_fail ? 1 : 0;
}
