// ref_capi.cpp -- TEST INFRASTRUCTURE.  Exposes the UNMODIFIED reference library
// (compiled by oracle/Makefile straight from /root/reference/proj/src, never copied)
// behind the same C interface as the C restatement (tmatch_oracle.h), so tests and
// bench.py can drive "the reference itself" and "the port" through one ctypes binding.
// Output: oracle/_ref/libtmatch_ref.so (git-ignored; travels to the GPU box).
#include <chrono>
#include <cstdint>
#include <optional>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "tmatch/autocorr.hpp"
#include "tmatch/blur.hpp"
#include "tmatch/bounds.hpp"
#include "tmatch/detail.hpp"
#include "tmatch/egs.hpp"
#include "tmatch/image.hpp"
#include "tmatch/matcher.hpp"
#include "tmatch/stats.hpp"
#include "tmatch/synth.hpp"

extern "C" {
#include "tmatch_oracle.h"
}

using namespace tmatch;

namespace {
thread_local std::string g_err;

Image wrap(const double* p, int rows, int cols) {
    return Image(rows, cols, std::vector<double>(p, p + std::size_t(rows) * cols));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

void fill(const MatchResult& r, tmo_result* o) {
    std::memset(o, 0, sizeof *o);
    o->mode = int(r.mode);
    o->best_row = r.best_row;
    o->best_col = r.best_col;
    o->best_degenerate = r.best_degenerate;
    o->best_rho = r.best_rho;
    o->refined_row = r.refined_row;
    o->refined_col = r.refined_col;
    o->refined_rho = r.refined_rho;
    o->below_threshold = r.below_threshold;
    o->extent_rows = r.extent_rows;
    o->extent_cols = r.extent_cols;
    o->final_threshold = r.final_threshold;
    o->centers = r.stats.centers;
    o->eliminated = r.stats.eliminated;
    o->retained = r.stats.retained;
    o->ops = r.stats.ops;
    o->elim_pct = r.stats.elim_pct;
    o->wall_ms = r.stats.wall_ms;
}

MatchParams to_params(const tmo_params* p) {
    MatchParams mp;
    mp.mode = MatchMode(p->mode);
    mp.h0 = p->h0;
    mp.w0 = p->w0;
    if (p->has_init_threshold) mp.init_threshold = p->init_threshold;
    mp.rho_th = p->rho_th;
    mp.rho_max = p->rho_max;
    mp.xi_fraction = p->xi_fraction;
    mp.opta_margin = p->opta_margin;
    mp.kernel = BlurKernel{p->kernel_len / 2,
                           std::vector<double>(p->kernel_profile, p->kernel_profile + p->kernel_len)};
    mp.parallel = p->parallel != 0;
    mp.threads = p->threads;
    mp.record_visits = p->record_visits != 0;
    return mp;
}

WindowStats to_ws(const double* mu, const double* om, const uint8_t* fl, int er, int ec, int m,
                  int n) {
    WindowStats ws;
    ws.win_rows = m;
    ws.win_cols = n;
    ws.rows = er;
    ws.cols = ec;
    const std::size_t E = std::size_t(er) * ec;
    ws.mean.assign(mu, mu + E);
    ws.norm.assign(om, om + E);
    ws.flat_map.assign(fl, fl + E);
    return ws;
}
}  // namespace

extern "C" {

const char* tmo_last_error(void) { return g_err.c_str(); }

void tmo_default_params(tmo_params* p) {
    static const double kProfile[5] = {0.05, 0.20, 0.50, 0.20, 0.05};
    std::memset(p, 0, sizeof *p);
    p->mode = 1;
    p->h0 = 3;
    p->w0 = 3;
    p->rho_th = 0.8;
    p->rho_max = 0.95;
    p->xi_fraction = 0.005;
    p->opta_margin = 0.005;
    p->kernel_profile = kProfile;
    p->kernel_len = 5;
    p->threads = 2;
}

int tmo_running_sum(const double* src, int p, int q, int m, int n, double* out) {
    return guard([&] {
        const SumTable t = running_sum(wrap(src, p, q), m, n);
        std::memcpy(out, t.sums.data(), t.sums.size() * 8);
    });
}

int tmo_window_stats(const double* img, int p, int q, int m, int n, double* mu, double* omega,
                     uint8_t* flat) {
    return guard([&] {
        const WindowStats ws = window_stats(wrap(img, p, q), m, n);
        std::memcpy(mu, ws.mean.data(), ws.mean.size() * 8);
        std::memcpy(omega, ws.norm.data(), ws.norm.size() * 8);
        std::memcpy(flat, ws.flat_map.data(), ws.flat_map.size());
    });
}

void tmo_template_stats(const double* t, int m, int n, double* mu, double* omega, int* flat) {
    const detail::TemplateStats ts = detail::template_stats(wrap(t, m, n));
    *mu = ts.mu;
    *omega = ts.omega;
    *flat = ts.flat;
}

double tmo_zncc_at(const double* t, int m, int n, double t_mu, double t_omega, int t_flat,
                   const double* img, int q, const double* mu, const double* omega,
                   const uint8_t* flat, int ec, int r, int c) {
    // Scalar evaluation straight through detail::zncc_at on wrapped views.
    const int p = r + m;  // only rows up to r+m-1 are read
    Image I(p, q);
    std::memcpy(I.data().data(), img, std::size_t(p) * q * 8);
    WindowStats ws;
    ws.win_rows = m;
    ws.win_cols = n;
    ws.rows = r + 1;
    ws.cols = ec;
    const std::size_t E = std::size_t(r + 1) * ec;
    ws.mean.assign(mu, mu + E);
    ws.norm.assign(omega, omega + E);
    ws.flat_map.assign(flat, flat + E);
    detail::TemplateStats ts{t_mu, t_omega, t_flat != 0};
    return detail::zncc_at(wrap(t, m, n), ts, I, ws, r, c);
}

int tmo_brute(const double* t, int m, int n, const double* img, int p, int q, tmo_result* res,
              double* surface) {
    return guard([&] {
        BruteOptions bo;
        bo.record_surface = surface != nullptr;
        bo.threads = 1;
        const MatchResult r = brute_force_match(wrap(t, m, n), wrap(img, p, q), bo);
        fill(r, res);
        if (surface) std::memcpy(surface, r.surface.data(), r.surface.size() * 8);
    });
}

int tmo_transitive_bounds(double rho_tc, double rho_co, double* lower, double* upper) {
    return guard([&] {
        const BoundPair b = transitive_bounds(rho_tc, rho_co);
        *lower = b.lower;
        *upper = b.upper;
    });
}
int tmo_transitive_gap(double rho_tc, double rho_co, double* gap) {
    return guard([&] { *gap = transitive_gap(rho_tc, rho_co); });
}
int tmo_sec_holds(double rho_tb, double rho_tc, double rho_co, int* holds) {
    return guard([&] { *holds = sec_holds(rho_tb, rho_tc, rho_co); });
}
int tmo_elimination_autocorr_threshold(double rho_tb, double rho_tc, double* out) {
    return guard([&] { *out = elimination_autocorr_threshold(rho_tb, rho_tc); });
}
int tmo_expected_elimination_threshold(double rho_tb, double* out) {
    return guard([&] { *out = expected_elimination_threshold(rho_tb); });
}

int64_t tmo_group_count(int er, int ec, int h, int w) {
    int64_t out = -1;
    guard([&] { out = GroupGrid(er, ec, h, w).group_count(); });
    return out;
}

int tmo_local_autocorrelation(const double* img, int p, int q, int m, int n, int h, int w,
                              const double* mu, const double* omega, const uint8_t* flat,
                              double* map) {
    return guard([&] {
        const GroupGrid grid = build_group_grid(p, q, m, n, h, w);
        const WindowStats ws = to_ws(mu, omega, flat, p - m + 1, q - n + 1, m, n);
        const AutoCorrMap a = local_autocorrelation(wrap(img, p, q), m, n, grid, ws);
        std::memcpy(map, a.values.data(), a.values.size() * 8);
    });
}

int64_t tmo_retained_count(const double* map, int er, int ec, int h, int w, double rho_tb) {
    int64_t out = -1;
    guard([&] {
        AutoCorrMap a;
        a.rows = er;
        a.cols = ec;
        a.group_h = h;
        a.group_w = w;
        a.values.assign(map, map + std::size_t(er) * ec);
        out = retained_count(a, rho_tb);
    });
    return out;
}

int tmo_efficient_group_size(const double* img, int p, int q, int m, int n, int h0, int w0,
                             double rho_tb, double xi, int max_group, const double* mu,
                             const double* omega, const uint8_t* flat, int* h_out, int* w_out,
                             tmo_egs_iter* trace, int max_trace, int* trace_len,
                             double* map_out) {
    return guard([&] {
        EgsParams ep;
        ep.h0 = h0;
        ep.w0 = w0;
        ep.rho_tb = rho_tb;
        ep.xi_fraction = xi;
        ep.max_group = max_group;
        const WindowStats ws = to_ws(mu, omega, flat, p - m + 1, q - n + 1, m, n);
        const EGSResult r = efficient_group_size(wrap(img, p, q), m, n, ep, ws);
        *h_out = r.h;
        *w_out = r.w;
        *trace_len = int(r.trace.size());
        for (std::size_t k = 0; k < r.trace.size() && int(k) < max_trace; ++k) {
            trace[k].h = r.trace[k].h;
            trace[k].w = r.trace[k].w;
            trace[k].central = r.trace[k].cost.central;
            trace[k].retained_cost = r.trace[k].cost.retained_cost;
            trace[k].amortized = r.trace[k].cost.amortized;
            trace[k].total = r.trace[k].cost.total;
            trace[k].retained = r.trace[k].cost.retained;
        }
        if (map_out) std::memcpy(map_out, r.map.values.data(), r.map.values.size() * 8);
    });
}

int tmo_blur(const double* img, int p, int q, const double* profile, int len, double* out) {
    return guard([&] {
        const BlurKernel k{len / 2, std::vector<double>(profile, profile + len)};
        const Image b = blur(wrap(img, p, q), k);
        std::memcpy(out, b.data().data(), b.size() * 8);
    });
}

int tmo_quality_threshold(double rho_th, double rho_max, double* out) {
    return guard([&] { *out = quality_threshold(rho_th, rho_max); });
}

int tmo_blur_fidelity_map(const double* I, const double* I_blur, int p, int q, int m, int n,
                          double* fid) {
    return guard([&] {
        const FidelityMap f = blur_fidelity_map(wrap(I, p, q), wrap(I_blur, p, q), m, n);
        std::memcpy(fid, f.values.data(), f.values.size() * 8);
    });
}

int tmo_optimize_autocorrelation(const double* img, int p, int q, int m, int n,
                                 const tmo_params* prm, double* image_out, int* kappa,
                                 double* lambda, int* h_out, int* w_out, double* cost_out,
                                 double* trace, int max_trace, int* trace_len, double* map_out) {
    return guard([&] {
        const MatchParams mp = to_params(prm);
        OptAParams op;
        op.rho_th = mp.rho_th;
        op.rho_max = mp.rho_max;
        op.kernel = mp.kernel;
        op.margin = mp.opta_margin;
        op.egs.h0 = mp.h0;
        op.egs.w0 = mp.w0;
        op.egs.rho_tb = mp.rho_th;
        op.egs.xi_fraction = mp.xi_fraction;
        const OptAResult r = optimize_autocorrelation(wrap(img, p, q), m, n, op);
        std::memcpy(image_out, r.image.data().data(), r.image.size() * 8);
        *kappa = r.kappa;
        *lambda = r.lambda;
        *h_out = r.egs.h;
        *w_out = r.egs.w;
        *cost_out = r.egs.cost.total;
        *trace_len = int(r.trace.size());
        for (std::size_t k = 0; k < r.trace.size() && int(k) < max_trace; ++k) {
            trace[4 * k + 0] = r.trace[k].h;
            trace[4 * k + 1] = r.trace[k].w;
            trace[4 * k + 2] = r.trace[k].cost;
            trace[4 * k + 3] = double(r.trace[k].restored);
        }
        if (map_out) std::memcpy(map_out, r.egs.map.values.data(), r.egs.map.values.size() * 8);
    });
}

int tmo_transitive_search(const double* t, int m, int n, const double* img, int p, int q,
                          const double* map, int h, int w, const double* mu,
                          const double* omega, const uint8_t* flat, int has_init,
                          double init_threshold, int parallel, int threads, tmo_result* res,
                          uint8_t* visits) {
    return guard([&] {
        // Route through run_egs so the caller-supplied window stats are used
        // (transitive_search() recomputes them from I, which is identical).
        const int er = p - m + 1, ec = q - n + 1;
        PreparedEgs prep;
        prep.ws = to_ws(mu, omega, flat, er, ec, m, n);
        prep.egs.h = h;
        prep.egs.w = w;
        prep.egs.grid = GroupGrid(er, ec, h, w);
        prep.egs.map.rows = er;
        prep.egs.map.cols = ec;
        prep.egs.map.group_h = h;
        prep.egs.map.group_w = w;
        prep.egs.map.values.assign(map, map + std::size_t(er) * ec);
        MatchParams mp;
        if (has_init) mp.init_threshold = init_threshold;
        mp.parallel = parallel != 0;
        mp.threads = threads;
        mp.record_visits = visits != nullptr;
        const MatchResult r = run_egs(wrap(t, m, n), wrap(img, p, q), prep, mp);
        fill(r, res);
        if (visits) std::memcpy(visits, r.visits.data(), r.visits.size());
    });
}

int tmo_refine(const double* t, int m, int n, const double* img, int p, int q, int loc_row,
               int loc_col, int d, int* row, int* col, double* rho, int* degenerate) {
    return guard([&] {
        const BestCell b = refine_localization(wrap(t, m, n), wrap(img, p, q), loc_row, loc_col, d);
        *row = b.row;
        *col = b.col;
        *rho = b.rho;
        *degenerate = b.degenerate;
    });
}

int tmo_match(const double* t, int m, int n, const double* img, int p, int q,
              const tmo_params* prm, tmo_result* res, uint8_t* visits) {
    return guard([&] {
        MatchParams mp = to_params(prm);
        mp.record_visits = visits != nullptr;
        const MatchResult r = match(wrap(t, m, n), wrap(img, p, q), mp);
        fill(r, res);
        if (visits && !r.visits.empty()) std::memcpy(visits, r.visits.data(), r.visits.size());
    });
}

// ---- extras only the reference build offers: the reference's own corpus generator,
// so the acceptance corpora (synth.cpp, mt19937_64) can be regenerated bit-exactly. ----
int ref_synth_search_image(int rows, int cols, double sigma, int passes, double lo, double hi,
                           uint64_t seed, double* out) {
    return guard([&] {
        std::mt19937_64 rng(seed);
        SynthImageConfig cfg;
        cfg.rows = rows;
        cfg.cols = cols;
        cfg.smooth_sigma = sigma;
        cfg.smooth_passes = passes;
        cfg.lo = lo;
        cfg.hi = hi;
        const Image img = synth_search_image(cfg, rng);
        std::memcpy(out, img.data().data(), img.size() * 8);
    });
}

// synth_corpus (synth.cpp:53-83) for square templates of one size; images out is
// count*rows*cols doubles, entries out is count*per_size*2 ints (row, col).
int ref_synth_corpus(int rows, int cols, double sigma, int count, int m, int per_size,
                     uint64_t seed, double* images, int* entries) {
    return guard([&] {
        CorpusSpec spec;
        spec.seed = seed;
        spec.image.rows = rows;
        spec.image.cols = cols;
        spec.image.smooth_sigma = sigma;
        spec.image_count = count;
        spec.template_sizes = {m};
        spec.per_size = per_size;
        const Corpus c = synth_corpus(spec);
        for (int i = 0; i < count; ++i)
            std::memcpy(images + std::size_t(i) * rows * cols, c.images[i].data().data(),
                        std::size_t(rows) * cols * 8);
        for (std::size_t k = 0; k < c.entries.size(); ++k) {
            entries[2 * k] = c.entries[k].row;
            entries[2 * k + 1] = c.entries[k].col;
        }
    });
}

// Wall-clock helper for the CPU baseline: prepare_egs once + run_egs, reference policy
// selected by parallel/threads (frozen needs threads >= 2, matcher.cpp:129).
int ref_prepare_run_egs(const double* t, int m, int n, const double* img, int p, int q,
                        int parallel, int threads, tmo_result* res, double* prep_ms,
                        double* run_ms) {
    return guard([&] {
        MatchParams mp;
        mp.parallel = parallel != 0;
        mp.threads = threads;
        const Image I = wrap(img, p, q);
        const Image T = wrap(t, m, n);
        const auto t0 = std::chrono::steady_clock::now();
        const PreparedEgs prep = prepare_egs(I, m, n, mp);
        const auto t1 = std::chrono::steady_clock::now();
        const MatchResult r = run_egs(T, I, prep, mp);
        const auto t2 = std::chrono::steady_clock::now();
        fill(r, res);
        *prep_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        *run_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
    });
}

// ---- reference-only extras for the per-config goldens and the map-cache interop -------

// brute_force_match (stats.cpp:156-213) with the reference's own row-partitioned threads.
int ref_brute_threads(const double* t, int m, int n, const double* img, int p, int q,
                      int threads, tmo_result* res) {
    return guard([&] {
        BruteOptions bo;
        bo.threads = threads;
        fill(brute_force_match(wrap(t, m, n), wrap(img, p, q), bo), res);
    });
}

// One preparation (prepare_egs matcher.cpp:205 or prepare_opta :217) shared by a batch of
// templates of one size, then run_egs/run_opta per template -- cmd_bench's cache
// (cli.cpp:213-237).  info = {h_e, w_e, kappa, lambda}; run_ms per template.
int ref_prepare_run_batch(const double* tmpls, int ntmpl, int m, int n, const double* img,
                          int p, int q, int mode, int parallel, int threads, tmo_result* res,
                          double* info, double* prep_ms, double* run_ms) {
    return guard([&] {
        MatchParams mp;
        mp.parallel = parallel != 0;
        mp.threads = threads;
        const Image I = wrap(img, p, q);
        const std::size_t mn = std::size_t(m) * n;
        const auto t0 = std::chrono::steady_clock::now();
        std::optional<PreparedEgs> pe;
        std::optional<PreparedOptA> po;
        if (mode == 2) {
            po.emplace(prepare_opta(I, m, n, mp));
            info[0] = po->opta.egs.h;
            info[1] = po->opta.egs.w;
            info[2] = po->opta.kappa;
            info[3] = po->opta.lambda;
        } else {
            pe.emplace(prepare_egs(I, m, n, mp));
            info[0] = pe->egs.h;
            info[1] = pe->egs.w;
            info[2] = 0;
            info[3] = 0;
        }
        *prep_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count();
        for (int k = 0; k < ntmpl; ++k) {
            const Image T = wrap(tmpls + k * mn, m, n);
            const auto t1 = std::chrono::steady_clock::now();
            const MatchResult r = mode == 2 ? run_opta(T, I, *po, mp) : run_egs(T, I, *pe, mp);
            run_ms[k] = std::chrono::duration<double, std::milli>(
                            std::chrono::steady_clock::now() - t1).count();
            fill(r, res + k);
        }
    });
}

// image.cpp:215-228 and autocorr.cpp:102-153, compiled from the reference sources.
uint64_t ref_content_hash(const double* img, int p, int q) { return content_hash(wrap(img, p, q)); }

uint64_t ref_autocorr_cache_key(const double* img, int p, int q, int m, int n, int h, int w) {
    return autocorr_cache_key(wrap(img, p, q), m, n, h, w);
}

int ref_save_autocorr(const double* map, int rows, int cols, int h, int w, uint64_t key,
                      const char* path) {
    return guard([&] {
        AutoCorrMap a;
        a.rows = rows;
        a.cols = cols;
        a.group_h = h;
        a.group_w = w;
        a.values.assign(map, map + std::size_t(rows) * cols);
        save_autocorr(a, key, path);
    });
}

// 1 = loaded into map (rows*cols doubles; header checked against rows/cols/h/w), 0 = miss.
int ref_load_autocorr(const char* path, uint64_t key, int rows, int cols, int h, int w,
                      double* map) {
    const auto a = load_autocorr(path, key);
    if (!a || a->rows != rows || a->cols != cols || a->group_h != h || a->group_w != w) return 0;
    std::memcpy(map, a->values.data(), a->values.size() * 8);
    return 1;
}

// PGM I/O (image.cpp:25-84, 187-213): load into out (rows*cols) or report the size.
int ref_load_image(const char* path, int* rows, int* cols, double* out, int cap) {
    return guard([&] {
        const Image I = load_image(path);
        *rows = I.rows();
        *cols = I.cols();
        if (out && cap >= int(I.size())) std::memcpy(out, I.data().data(), I.size() * 8);
    });
}

int ref_save_image(const double* img, int p, int q, const char* path) {
    return guard([&] { save_image(wrap(img, p, q), path); });
}

}  // extern "C"
