/*
 * tmatch_oracle.c -- CPU restatement of the reference hot path.  TEST INFRASTRUCTURE:
 * the parity checker for the CUDA product, never part of it (see tmatch_oracle.h).
 *
 * Compile with -ffp-contract=off: every FP64 expression below is written in the
 * reference's evaluation order (left-to-right, no fused multiply-add), which is what
 * g++ -O3 produces for the reference on x86-64 without -march.
 */
#define _POSIX_C_SOURCE 200809L
#include "tmatch_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[256];

static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}

const char* tmo_last_error(void) { return g_err; }

static const double kEps = 2.220446049250313e-16;

/* std::max / std::min / std::clamp semantics (algorithm: (a < b) ? b : a). */
static inline double dmax(double a, double b) { return (a < b) ? b : a; }
static inline double dmin(double a, double b) { return (b < a) ? b : a; }
static inline double dclamp(double v, double lo, double hi) {
    return (v < lo) ? lo : ((hi < v) ? hi : v);
}
static inline int imin(int a, int b) { return a < b ? a : b; }
static inline int imax(int a, int b) { return a > b ? a : b; }

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

void tmo_default_params(tmo_params* p) {
    static const double kDefaultProfile[5] = {0.05, 0.20, 0.50, 0.20, 0.05};
    memset(p, 0, sizeof *p);
    p->mode = 1;
    p->h0 = 3;
    p->w0 = 3;
    p->rho_th = 0.8;
    p->rho_max = 0.95;
    p->xi_fraction = 0.005;
    p->opta_margin = 0.005;
    p->kernel_profile = kDefaultProfile;
    p->kernel_len = 5;
    p->parallel = 0;
    p->threads = 2;
}

/* ---- stats.cpp:19-53 -------------------------------------------------------------- */
int tmo_running_sum(const double* src, int p, int q, int m, int n, double* out) {
    if (m < 1 || n < 1 || m > p || n > q) return fail("running_sum: window does not fit the source");
    const size_t pw = (size_t)q + 1;
    double* prefix = (double*)calloc((size_t)(p + 1) * pw, sizeof(double));
    if (!prefix) return fail("running_sum: out of memory");
    for (int r = 0; r < p; ++r) {
        const double* srow = src + (size_t)r * q;
        const double* prev = prefix + (size_t)r * pw;
        double* cur = prefix + (size_t)(r + 1) * pw;
        double row_acc = 0.0;
        for (int c = 0; c < q; ++c) {
            row_acc += srow[c];
            cur[c + 1] = prev[c + 1] + row_acc;
        }
    }
    const int er = p - m + 1, ec = q - n + 1;
    for (int r = 0; r < er; ++r) {
        const double* top = prefix + (size_t)r * pw;
        const double* bot = prefix + (size_t)(r + m) * pw;
        double* o = out + (size_t)r * ec;
        for (int c = 0; c < ec; ++c) o[c] = bot[c + n] - top[c + n] - bot[c] + top[c];
    }
    free(prefix);
    return 0;
}

/* ---- detail.hpp:18-22 ------------------------------------------------------------ */
static int variance_is_flat(double var_sum, double q_sum, long long mn) {
    const double abs_tol = 1e-9 * (double)mn;
    const double rel = dmax(1e-13, 4.0 * kEps * (double)mn);
    return var_sum <= dmax(abs_tol * abs_tol, rel * q_sum);
}

/* ---- stats.cpp:55-94 ------------------------------------------------------------- */
int tmo_window_stats(const double* img, int p, int q, int m, int n, double* mu, double* omega,
                     uint8_t* flat) {
    return tmo_window_stats_floor(img, p, q, m, n, NAN, mu, omega, flat);
}

/* window_stats with the flat-noise floor given (NaN: the image's own, stats.cpp:78-81) --
 * a row strip of a larger image takes the floor of the whole image (row-strip tests). */
int tmo_window_stats_floor(const double* img, int p, int q, int m, int n, double floor_in,
                           double* mu, double* omega, uint8_t* flat) {
    const int er = p - m + 1, ec = q - n + 1;
    if (m < 1 || n < 1 || er < 1 || ec < 1) return fail("running_sum: window does not fit the source");
    const size_t E = (size_t)er * ec, P = (size_t)p * q;
    double* s = (double*)malloc(E * sizeof(double));
    double* sq = (double*)malloc(E * sizeof(double));
    double* squared = (double*)malloc(P * sizeof(double));
    if (!s || !sq || !squared) return fail("window_stats: out of memory");
    tmo_running_sum(img, p, q, m, n, s);
    for (size_t i = 0; i < P; ++i) squared[i] = img[i] * img[i];
    tmo_running_sum(squared, p, q, m, n, sq);
    const double inv_mn = 1.0 / ((double)m * (double)n);
    const long long mn = (long long)m * n;
    double q_total = 0.0;
    for (size_t i = 0; i < P; ++i) q_total += squared[i];
    const double prefix_noise = isnan(floor_in) ? (double)(p + q) * kEps * q_total : floor_in;
    for (size_t i = 0; i < E; ++i) {
        const double sum = s[i];
        const double sqs = sq[i];
        const double var_sum = sqs - sum * sum * inv_mn;
        const int f = variance_is_flat(var_sum, sqs, mn) || var_sum <= prefix_noise;
        mu[i] = sum * inv_mn;
        omega[i] = f ? 0.0 : sqrt(dmax(0.0, var_sum));
        flat[i] = (uint8_t)(f ? 1 : 0);
    }
    free(s);
    free(sq);
    free(squared);
    return 0;
}

/* ---- stats.cpp:98-111 ------------------------------------------------------------ */
void tmo_template_stats(const double* t, int m, int n, double* mu, double* omega, int* flat) {
    double sum = 0.0, sq = 0.0;
    const size_t N = (size_t)m * n;
    for (size_t i = 0; i < N; ++i) {
        sum += t[i];
        sq += t[i] * t[i];
    }
    const long long mn = (long long)m * n;
    const double var_sum = sq - sum * sum / (double)mn;
    *mu = sum / (double)mn;
    *omega = sqrt(dmax(0.0, var_sum));
    *flat = variance_is_flat(var_sum, sq, mn);
}

/* ---- detail.hpp:32-51 ------------------------------------------------------------ */
static double window_dot(const double* t, int m, int n, const double* img, int q, int r, int c) {
    double acc = 0.0;
    for (int i = 0; i < m; ++i) {
        const double* pt = t + (size_t)i * n;
        const double* pi = img + (size_t)(r + i) * q + c;
        for (int j = 0; j < n; ++j) acc += pt[j] * pi[j];
    }
    return acc;
}

double tmo_zncc_at(const double* t, int m, int n, double t_mu, double t_omega, int t_flat,
                   const double* img, int q, const double* mu, const double* omega,
                   const uint8_t* flat, int ec, int r, int c) {
    const size_t k = (size_t)r * ec + c;
    if (t_flat || flat[k]) return 0.0;
    const double mn = (double)m * (double)n;
    const double num = window_dot(t, m, n, img, q, r, c) - mn * t_mu * mu[k];
    return dclamp(num / (t_omega * omega[k]), -1.0, 1.0);
}

/* ---- stats.cpp:147-154: non-degenerate > degenerate, larger rho, smaller (row,col) -- */
typedef struct {
    int row, col;
    double rho;
    int degenerate, valid;
} cell;

static const cell kNoCell = {-1, -1, 0.0, 1, 0};

static int better(const cell* a, const cell* b) {
    if (!a->valid) return 0;
    if (!b->valid) return 1;
    if (a->degenerate != b->degenerate) return !a->degenerate;
    if (a->rho != b->rho) return a->rho > b->rho;
    if (a->row != b->row) return a->row < b->row;
    return a->col < b->col;
}

/* ---- stats.cpp:156-213 ----------------------------------------------------------- */
int tmo_brute(const double* t, int m, int n, const double* img, int p, int q, tmo_result* res,
              double* surface) {
    if (m > p || n > q) return fail("brute_force_match: template larger than search image");
    const int er = p - m + 1, ec = q - n + 1;
    const size_t E = (size_t)er * ec;
    double* mu = (double*)malloc(E * 8);
    double* om = (double*)malloc(E * 8);
    uint8_t* fl = (uint8_t*)malloc(E);
    if (tmo_window_stats(img, p, q, m, n, mu, om, fl)) return -1;
    double tmu, tom;
    int tfl;
    tmo_template_stats(t, m, n, &tmu, &tom, &tfl);
    cell best = kNoCell;
    for (int r = 0; r < er; ++r)
        for (int c = 0; c < ec; ++c) {
            const double rho = tmo_zncc_at(t, m, n, tmu, tom, tfl, img, q, mu, om, fl, ec, r, c);
            if (surface) surface[(size_t)r * ec + c] = rho;
            cell cand = {r, c, rho, tfl || fl[(size_t)r * ec + c], 1};
            if (better(&cand, &best)) best = cand;
        }
    memset(res, 0, sizeof *res);
    res->mode = 0;
    res->extent_rows = er;
    res->extent_cols = ec;
    res->best_row = res->refined_row = best.row;
    res->best_col = res->refined_col = best.col;
    res->best_rho = res->refined_rho = best.rho;
    res->best_degenerate = best.degenerate;
    res->final_threshold = best.degenerate ? 0.0 : best.rho;
    res->retained = (int64_t)er * ec;
    res->ops = (int64_t)er * ec;
    res->elim_pct = 0.0;
    free(mu);
    free(om);
    free(fl);
    return 0;
}

/* ---- bounds.cpp:13-59 ------------------------------------------------------------ */
static int checked(double rho, const char* name, double* out) {
    if (fabs(rho) > 1.0 + 1e-9) {
        snprintf(g_err, sizeof g_err, "correlation out of [-1,1]: %s", name);
        return -1;
    }
    *out = dclamp(rho, -1.0, 1.0);
    return 0;
}

static double half_gap(double a, double b) {
    return sqrt(dmax(0.0, 1.0 - a * a)) * sqrt(dmax(0.0, 1.0 - b * b));
}

int tmo_transitive_bounds(double rho_tc, double rho_co, double* lower, double* upper) {
    double a, b;
    if (checked(rho_tc, "rho_tc", &a) || checked(rho_co, "rho_co", &b)) return -1;
    const double center = a * b;
    const double s = half_gap(a, b);
    *lower = dclamp(center - s, -1.0, 1.0);
    *upper = dclamp(center + s, -1.0, 1.0);
    return 0;
}

int tmo_transitive_gap(double rho_tc, double rho_co, double* gap) {
    double a, b;
    if (checked(rho_tc, "rho_tc", &a) || checked(rho_co, "rho_co", &b)) return -1;
    *gap = 2.0 * half_gap(a, b);
    return 0;
}

int tmo_sec_holds(double rho_tb, double rho_tc, double rho_co, int* holds) {
    double tb, a, b;
    if (checked(rho_tb, "rho_tb", &tb) || checked(rho_tc, "rho_tc", &a) ||
        checked(rho_co, "rho_co", &b))
        return -1;
    *holds = tb >= a * b + half_gap(a, b);
    return 0;
}

int tmo_elimination_autocorr_threshold(double rho_tb, double rho_tc, double* out) {
    double tb, tc;
    if (checked(rho_tb, "rho_tb", &tb) || checked(rho_tc, "rho_tc", &tc)) return -1;
    const double radicand = 1.0 + tc * tc * tb * tb - (tc * tc + tb * tb);
    *out = tb * tc + sqrt(dmax(0.0, radicand));
    return 0;
}

int tmo_expected_elimination_threshold(double rho_tb, double* out) {
    double tb;
    if (checked(rho_tb, "rho_tb", &tb)) return -1;
    *out = sqrt(dmax(0.0, 1.0 - tb * tb));
    return 0;
}

/* ---- autocorr.cpp:12-32 group geometry ------------------------------------------- */
typedef struct {
    int er, ec, h, w, tr, tc;
} grid_t;

static int make_grid(int er, int ec, int h, int w, grid_t* g) {
    if (er < 1 || ec < 1) return fail("group grid: empty search extent");
    if (h < 1 || w < 1 || h % 2 == 0 || w % 2 == 0)
        return fail("group grid: group size must be odd and >= 1");
    g->er = er;
    g->ec = ec;
    g->h = h;
    g->w = w;
    g->tr = (er + h - 1) / h;
    g->tc = (ec + w - 1) / w;
    return 0;
}

/* Group tile ti,tj: rows [ti*h, min(ti*h+h, er)-1], centre = (r0+r1)/2. */
static void group_bounds(const grid_t* g, int ti, int tj, int* r0, int* r1, int* c0, int* c1,
                         int* cr, int* cc) {
    *r0 = ti * g->h;
    *r1 = imin(*r0 + g->h, g->er) - 1;
    *c0 = tj * g->w;
    *c1 = imin(*c0 + g->w, g->ec) - 1;
    *cr = (*r0 + *r1) / 2;
    *cc = (*c0 + *c1) / 2;
}

static int is_center(const grid_t* g, int r, int c) {
    const int ti = imin(r / g->h, g->tr - 1), tj = imin(c / g->w, g->tc - 1);
    int r0, r1, c0, c1, cr, cc;
    group_bounds(g, ti, tj, &r0, &r1, &c0, &c1, &cr, &cc);
    return cr == r && cc == c;
}

int64_t tmo_group_count(int er, int ec, int h, int w) {
    grid_t g;
    if (make_grid(er, ec, h, w, &g)) return -1;
    return (int64_t)g.tr * g.tc;
}

/* ---- autocorr.cpp:40-96 ---------------------------------------------------------- */
int tmo_local_autocorrelation(const double* img, int p, int q, int m, int n, int h, int w,
                              const double* mu, const double* omega, const uint8_t* flat,
                              double* map) {
    const int er = p - m + 1, ec = q - n + 1;
    grid_t g;
    if (make_grid(er, ec, h, w, &g)) return -1;
    memset(map, 0, sizeof(double) * (size_t)er * ec);
    const int hr = h / 2, wr = w / 2;
    const double mn = (double)m * (double)n;
    double* product = (double*)malloc(sizeof(double) * (size_t)p * q);
    double* cross = (double*)malloc(sizeof(double) * (size_t)p * q);
    for (int di = -hr; di <= hr; ++di)
        for (int dj = -wr; dj <= wr; ++dj) {
            if (di == 0 && dj == 0) continue;
            const int orr = imax(0, -di), occ = imax(0, -dj);
            const int ph = p - abs(di), pw = q - abs(dj);
            if (ph < m || pw < n) continue;
            for (int a = 0; a < ph; ++a) {
                const double* base = img + (size_t)(a + orr) * q + occ;
                const double* shifted = img + (size_t)(a + orr + di) * q + occ + dj;
                double* o = product + (size_t)a * pw;
                for (int b = 0; b < pw; ++b) o[b] = base[b] * shifted[b];
            }
            tmo_running_sum(product, ph, pw, m, n, cross);
            const int cec = pw - n + 1;
            for (int ti = 0; ti < g.tr; ++ti)
                for (int tj = 0; tj < g.tc; ++tj) {
                    int r0, r1, c0, c1, cr, cc;
                    group_bounds(&g, ti, tj, &r0, &r1, &c0, &c1, &cr, &cc);
                    const int mr = cr + di, mc = cc + dj;
                    if (mr < r0 || mr > r1 || mc < c0 || mc > c1) continue;
                    const size_t kc = (size_t)cr * ec + cc, km = (size_t)mr * ec + mc;
                    if (flat[kc] || flat[km]) continue;
                    const double cross_sum = cross[(size_t)(cr - orr) * cec + (cc - occ)];
                    const double num = cross_sum - mn * mu[kc] * mu[km];
                    const double rho = num / (omega[kc] * omega[km]);
                    map[km] = dclamp(rho, -1.0, 1.0);
                }
        }
    for (int ti = 0; ti < g.tr; ++ti)
        for (int tj = 0; tj < g.tc; ++tj) {
            int r0, r1, c0, c1, cr, cc;
            group_bounds(&g, ti, tj, &r0, &r1, &c0, &c1, &cr, &cc);
            map[(size_t)cr * ec + cc] = 1.0;
        }
    free(product);
    free(cross);
    return 0;
}

/* ---- egs.cpp:12-25 --------------------------------------------------------------- */
int64_t tmo_retained_count(const double* map, int er, int ec, int h, int w, double rho_tb) {
    if (rho_tb < 0.0 || rho_tb > 1.0) {
        fail("retained_count: rho_tb must be in [0,1]");
        return -1;
    }
    double threshold;
    tmo_expected_elimination_threshold(rho_tb, &threshold);
    grid_t g;
    if (make_grid(er, ec, h, w, &g)) return -1;
    int64_t count = 0;
    for (int r = 0; r < er; ++r)
        for (int c = 0; c < ec; ++c) {
            if (is_center(&g, r, c)) continue;
            if (map[(size_t)r * ec + c] < threshold) ++count;
        }
    return count;
}

/* ---- egs.cpp:27-37 --------------------------------------------------------------- */
static void total_cost(int er, int ec, int h, int w, int64_t n_r, double amortized,
                       tmo_egs_iter* it) {
    it->h = h;
    it->w = w;
    it->central = (double)((er + h - 1) / h) * (double)((ec + w - 1) / w);
    it->retained = n_r;
    it->retained_cost = (double)n_r;
    it->amortized = amortized;
    it->total = it->central + it->retained_cost + it->amortized;
}

/* ---- egs.cpp:39-91 --------------------------------------------------------------- */
int tmo_efficient_group_size(const double* img, int p, int q, int m, int n, int h0, int w0,
                             double rho_tb, double xi, int max_group, const double* mu,
                             const double* omega, const uint8_t* flat, int* h_out, int* w_out,
                             tmo_egs_iter* trace, int max_trace, int* trace_len,
                             double* map_out) {
    if (h0 < 1 || w0 < 1 || h0 % 2 == 0 || w0 % 2 == 0)
        return fail("efficient_group_size: initial group size must be odd");
    if (rho_tb <= 0.0 || rho_tb >= 1.0)
        return fail("efficient_group_size: rho_tb must be in (0,1)");
    const int er = p - m + 1, ec = q - n + 1;
    if (er < 1 || ec < 1) return fail("efficient_group_size: template does not fit");
    int cap = max_group > 0 ? max_group : 0x7fffffff;
    if (cap % 2 == 0) ++cap;
    const size_t E = (size_t)er * ec;
    double* map = (double*)malloc(E * 8);
    double prev_cost = INFINITY;
    int h = h0, w = w0, len = 0;
    *h_out = 0;
    *w_out = 0;
    for (;;) {
        if (tmo_local_autocorrelation(img, p, q, m, n, h, w, mu, omega, flat, map)) {
            free(map);
            return -1;
        }
        const int64_t n_r = tmo_retained_count(map, er, ec, h, w, rho_tb);
        tmo_egs_iter it;
        total_cost(er, ec, h, w, n_r, 0.0, &it);
        const int accepted = !isfinite(prev_cost) || prev_cost - it.total > xi * prev_cost;
        if (!accepted) break;
        *h_out = h;
        *w_out = w;
        if (map_out) memcpy(map_out, map, E * 8);
        if (len < max_trace) trace[len] = it;
        ++len;
        prev_cost = it.total;
        if ((h >= er && w >= ec) || (h >= cap && w >= cap)) break;
        h = imin(h + 2, cap);
        w = imin(w + 2, cap);
    }
    *trace_len = len;
    free(map);
    return 0;
}

/* ---- blur.cpp:57-86 -------------------------------------------------------------- */
int tmo_blur(const double* img, int p, int q, const double* prof, int len, double* out) {
    const int d = len / 2;
    if (d == 0 && len == 1) {
        memcpy(out, img, sizeof(double) * (size_t)p * q);
        return 0;
    }
    double* tmp = (double*)malloc(sizeof(double) * (size_t)p * q);
    for (int r = 0; r < p; ++r) {
        const double* in = img + (size_t)r * q;
        double* o = tmp + (size_t)r * q;
        for (int c = 0; c < q; ++c) {
            double acc = 0.0;
            for (int k = -d; k <= d; ++k) {
                int cc = c + k;
                cc = cc < 0 ? 0 : (cc > q - 1 ? q - 1 : cc);
                acc += prof[k + d] * in[cc];
            }
            o[c] = acc;
        }
    }
    for (int r = 0; r < p; ++r) {
        double* o = out + (size_t)r * q;
        for (int c = 0; c < q; ++c) o[c] = 0.0;
        for (int k = -d; k <= d; ++k) {
            const double wk = prof[k + d];
            int rr = r + k;
            rr = rr < 0 ? 0 : (rr > p - 1 ? p - 1 : rr);
            const double* in = tmp + (size_t)rr * q;
            for (int c = 0; c < q; ++c) o[c] += wk * in[c];
        }
    }
    free(tmp);
    return 0;
}

/* ---- blur.cpp:88-94 -------------------------------------------------------------- */
int tmo_quality_threshold(double rho_th, double rho_max, double* out) {
    if (rho_th < 0.0 || rho_th > 1.0 || rho_max < 0.0 || rho_max > 1.0)
        return fail("quality_threshold: inputs must be in [0,1]");
    if (rho_max < rho_th) return fail("quality_threshold: rho_max must be >= rho_th");
    return tmo_elimination_autocorr_threshold(rho_th, rho_max, out);
}

/* ---- blur.cpp:96-125 (variant reusing ws of the original) ------------------------ */
static int fidelity_with_ws(const double* I, const double* mu_o, const double* om_o,
                            const uint8_t* fl_o, const double* I_blur, int p, int q, int m,
                            int n, double* fid) {
    const int er = p - m + 1, ec = q - n + 1;
    const size_t E = (size_t)er * ec, P = (size_t)p * q;
    double* product = (double*)malloc(P * 8);
    double* cross = (double*)malloc(E * 8);
    double* mu_b = (double*)malloc(E * 8);
    double* om_b = (double*)malloc(E * 8);
    uint8_t* fl_b = (uint8_t*)malloc(E);
    for (size_t i = 0; i < P; ++i) product[i] = I_blur[i] * I[i];
    tmo_running_sum(product, p, q, m, n, cross);
    tmo_window_stats(I_blur, p, q, m, n, mu_b, om_b, fl_b);
    const double mn = (double)m * (double)n;
    for (size_t k = 0; k < E; ++k) {
        double rho = 0.0;
        if (!fl_o[k] && !fl_b[k]) {
            const double num = cross[k] - mn * mu_b[k] * mu_o[k];
            rho = dclamp(num / (om_b[k] * om_o[k]), -1.0, 1.0);
        }
        fid[k] = rho;
    }
    free(product);
    free(cross);
    free(mu_b);
    free(om_b);
    free(fl_b);
    return 0;
}

int tmo_blur_fidelity_map(const double* I, const double* I_blur, int p, int q, int m, int n,
                          double* fid) {
    const int er = p - m + 1, ec = q - n + 1;
    if (er < 1 || ec < 1) return fail("running_sum: window does not fit the source");
    const size_t E = (size_t)er * ec;
    double* mu = (double*)malloc(E * 8);
    double* om = (double*)malloc(E * 8);
    uint8_t* fl = (uint8_t*)malloc(E);
    tmo_window_stats(I, p, q, m, n, mu, om, fl);
    fidelity_with_ws(I, mu, om, fl, I_blur, p, q, m, n, fid);
    free(mu);
    free(om);
    free(fl);
    return 0;
}

/* ---- blur.cpp:137-179: pixel restored iff a marked window covers it -------------- */
static void restore_marked(double* blurred, const double* original, const uint8_t* marks,
                           int er, int ec, int m, int n, int p, int q) {
    const size_t pw = (size_t)ec + 1;
    long long* prefix = (long long*)calloc((size_t)(er + 1) * pw, sizeof(long long));
    for (int r = 0; r < er; ++r) {
        long long acc = 0;
        for (int c = 0; c < ec; ++c) {
            acc += marks[(size_t)r * ec + c];
            prefix[(size_t)(r + 1) * pw + c + 1] = prefix[(size_t)r * pw + c + 1] + acc;
        }
    }
    for (int x = 0; x < p; ++x)
        for (int y = 0; y < q; ++y) {
            const int r0 = imax(0, x - m + 1), r1 = imin(er - 1, x);
            const int c0 = imax(0, y - n + 1), c1 = imin(ec - 1, y);
            if (r0 > r1 || c0 > c1) continue;
            const long long s = prefix[(size_t)(r1 + 1) * pw + c1 + 1] -
                                prefix[(size_t)r0 * pw + c1 + 1] -
                                prefix[(size_t)(r1 + 1) * pw + c0] + prefix[(size_t)r0 * pw + c0];
            if (s > 0) blurred[(size_t)x * q + y] = original[(size_t)x * q + y];
        }
    free(prefix);
}

/* ---- blur.cpp:208-239 ------------------------------------------------------------ */
static long long repair_to_fixed_point(double* blurred, const double* original, const double* mu,
                                       const double* om, const uint8_t* fl, int p, int q, int m,
                                       int n, double lambda) {
    const int er = p - m + 1, ec = q - n + 1;
    const size_t E = (size_t)er * ec, P = (size_t)p * q;
    double* fid = (double*)malloc(E * 8);
    double* changed = (double*)malloc(P * 8);
    double* in_win = (double*)malloc(E * 8);
    uint8_t* marks = (uint8_t*)malloc(E);
    long long total = 0;
    for (;;) {
        fidelity_with_ws(original, mu, om, fl, blurred, p, q, m, n, fid);
        for (size_t i = 0; i < P; ++i) changed[i] = blurred[i] != original[i] ? 1.0 : 0.0;
        tmo_running_sum(changed, p, q, m, n, in_win);
        long long count = 0;
        for (size_t k = 0; k < E; ++k) {
            marks[k] = 0;
            if (fid[k] >= lambda) continue;
            if (in_win[k] == 0.0) continue;
            marks[k] = 1;
            ++count;
        }
        if (count == 0) break;
        restore_marked(blurred, original, marks, er, ec, m, n, p, q);
        total += count;
    }
    free(fid);
    free(changed);
    free(in_win);
    free(marks);
    return total;
}

/* ---- blur.cpp:243-278 ------------------------------------------------------------ */
int tmo_optimize_autocorrelation(const double* img, int p, int q, int m, int n,
                                 const tmo_params* prm, double* image_out, int* kappa,
                                 double* lambda_out, int* h_out, int* w_out, double* cost_out,
                                 double* trace, int max_trace, int* trace_len, double* map_out) {
    double lambda;
    if (tmo_quality_threshold(prm->rho_th, prm->rho_max, &lambda)) return -1;
    const int er = p - m + 1, ec = q - n + 1;
    if (er < 1 || ec < 1) return fail("running_sum: window does not fit the source");
    const size_t E = (size_t)er * ec, P = (size_t)p * q;
    double* mu = (double*)malloc(E * 8);
    double* om = (double*)malloc(E * 8);
    uint8_t* fl = (uint8_t*)malloc(E);
    double* mu_b = (double*)malloc(E * 8);
    double* om_b = (double*)malloc(E * 8);
    uint8_t* fl_b = (uint8_t*)malloc(E);
    double* current = (double*)malloc(P * 8);
    double* blurred = (double*)malloc(P * 8);
    double* map_k = map_out ? (double*)malloc(E * 8) : NULL;
    tmo_window_stats(img, p, q, m, n, mu, om, fl);
    tmo_egs_iter egs_trace[64];
    int tl, h, w;
    if (tmo_efficient_group_size(img, p, q, m, n, prm->h0, prm->w0, prm->rho_th, prm->xi_fraction,
                                 127, mu, om, fl, &h, &w, egs_trace, 64, &tl, map_out))
        return -1;
    double prev_cost = egs_trace[tl - 1].total;
    int len = 0;
    if (len < max_trace) {
        trace[4 * len + 0] = h;
        trace[4 * len + 1] = w;
        trace[4 * len + 2] = prev_cost;
        trace[4 * len + 3] = 0;
    }
    ++len;
    memcpy(current, img, P * 8);
    memcpy(image_out, img, P * 8);
    *kappa = 0;
    *h_out = h;
    *w_out = w;
    *cost_out = prev_cost;
    for (int iter = 1; iter <= 64; ++iter) {
        tmo_blur(current, p, q, prm->kernel_profile, prm->kernel_len, blurred);
        const long long restored = repair_to_fixed_point(blurred, img, mu, om, fl, p, q, m, n, lambda);
        tmo_window_stats(blurred, p, q, m, n, mu_b, om_b, fl_b);
        int hk, wk, tlk;
        if (tmo_efficient_group_size(blurred, p, q, m, n, h, w, prm->rho_th, prm->xi_fraction, 127,
                                     mu_b, om_b, fl_b, &hk, &wk, egs_trace, 64, &tlk, map_k))
            return -1;
        const double cost = egs_trace[tlk - 1].total;
        const double improvement = prev_cost - cost;
        if (!(improvement >= prm->opta_margin * cost)) break;
        if (len < max_trace) {
            trace[4 * len + 0] = hk;
            trace[4 * len + 1] = wk;
            trace[4 * len + 2] = cost;
            trace[4 * len + 3] = (double)restored;
        }
        ++len;
        *kappa = iter;
        prev_cost = cost;
        h = hk;
        w = wk;
        *h_out = h;
        *w_out = w;
        *cost_out = cost;
        memcpy(current, blurred, P * 8);
        memcpy(image_out, blurred, P * 8);
        if (map_out) memcpy(map_out, map_k, E * 8);
    }
    *trace_len = len;
    *lambda_out = lambda;
    free(mu);
    free(om);
    free(fl);
    free(mu_b);
    free(om_b);
    free(fl_b);
    free(current);
    free(blurred);
    free(map_k);
    return 0;
}

/* ---- matcher.cpp:95-177 ---------------------------------------------------------- */
static int search_impl(const double* t, int m, int n, const double* img, int p, int q,
                       const double* map, int h, int w, const double* mu, const double* om,
                       const uint8_t* fl, int has_init, double init, int parallel, int threads,
                       tmo_result* res, uint8_t* visits) {
    double tmu, tom;
    int tfl;
    tmo_template_stats(t, m, n, &tmu, &tom, &tfl);
    if (tfl) return fail("transitive_search: constant template has no defined correlation");
    const int er = p - m + 1, ec = q - n + 1;
    grid_t g;
    if (make_grid(er, ec, h, w, &g)) return -1;
    if (has_init && fabs(init) > 1.0 + 1e-9)
        return fail("transitive_search: init threshold out of [-1,1]");
    const double t0 = now_ms();
    memset(res, 0, sizeof *res);
    res->mode = 1;
    res->extent_rows = er;
    res->extent_cols = ec;
    if (visits) memset(visits, 0, (size_t)er * ec);
    const int64_t G = (int64_t)g.tr * g.tc;
    double* rho_c = (double*)malloc(G * 8);
    uint8_t* deg_c = (uint8_t*)malloc(G);
    cell cbest = kNoCell;
    for (int ti = 0; ti < g.tr; ++ti)
        for (int tj = 0; tj < g.tc; ++tj) {
            int r0, r1, c0, c1, cr, cc;
            group_bounds(&g, ti, tj, &r0, &r1, &c0, &c1, &cr, &cc);
            const int64_t gi = (int64_t)ti * g.tc + tj;
            rho_c[gi] = tmo_zncc_at(t, m, n, tmu, tom, tfl, img, q, mu, om, fl, ec, cr, cc);
            deg_c[gi] = tfl || fl[(size_t)cr * ec + cc];
            cell cand = {cr, cc, rho_c[gi], deg_c[gi], 1};
            if (better(&cand, &cbest)) cbest = cand;
        }
    int64_t ops = G;
    double rho_tb = -INFINITY;
    for (int64_t i = 0; i < G; ++i)
        if (!deg_c[i]) rho_tb = dmax(rho_tb, rho_c[i]);
    if (has_init) rho_tb = dmax(rho_tb, dclamp(init, -1.0, 1.0));
    /* Frozen (matcher.cpp:129-143) iff parallel && threads>1 && groups>1.  Frozen
     * results are independent of the worker partition (strict total order merge,
     * additive counts), so one pass with running_update=false reproduces them. */
    const int running = !(parallel && threads > 1 && G > 1);
    double thr = rho_tb;
    cell best = kNoCell;
    int64_t elim = 0, kept = 0;
    for (int ti = 0; ti < g.tr; ++ti)
        for (int tj = 0; tj < g.tc; ++tj) {
            int r0, r1, c0, c1, cr, cc;
            group_bounds(&g, ti, tj, &r0, &r1, &c0, &c1, &cr, &cc);
            const int64_t gi = (int64_t)ti * g.tc + tj;
            const double rho_tc = rho_c[gi];
            const int cdeg = deg_c[gi];
            for (int r = r0; r <= r1; ++r)
                for (int c = c0; c <= c1; ++c) {
                    if (r == cr && c == cc) continue;
                    const size_t k = (size_t)r * ec + c;
                    const int mflat = tfl || fl[k];
                    if (!cdeg && !mflat && thr >= -1.0) {
                        int holds = 0;
                        if (tmo_sec_holds(dmin(thr, 1.0), rho_tc, map[k], &holds)) return -1;
                        if (holds) {
                            ++elim;
                            if (visits) visits[k] = 1;
                            continue;
                        }
                    }
                    const double rho =
                        tmo_zncc_at(t, m, n, tmu, tom, tfl, img, q, mu, om, fl, ec, r, c);
                    ++kept;
                    if (visits) visits[k] = 2;
                    cell cand = {r, c, rho, mflat, 1};
                    if (better(&cand, &best)) best = cand;
                    if (running && !mflat && rho > thr) thr = rho;
                }
        }
    cell fin = cbest;
    if (better(&best, &fin)) fin = best;
    double final_thr = dmax(rho_tb, thr);
    ops += kept;
    res->best_row = res->refined_row = fin.row;
    res->best_col = res->refined_col = fin.col;
    res->best_rho = res->refined_rho = fin.rho;
    res->best_degenerate = fin.degenerate;
    res->final_threshold = isfinite(final_thr) ? final_thr : 0.0;
    res->below_threshold = has_init && (fin.degenerate || fin.rho < init);
    res->centers = G;
    res->eliminated = elim;
    res->retained = kept;
    res->elim_pct = 100.0 * (double)elim / ((double)er * (double)ec);
    res->ops = ops;
    res->wall_ms = now_ms() - t0;
    free(rho_c);
    free(deg_c);
    return 0;
}

int tmo_transitive_search(const double* t, int m, int n, const double* img, int p, int q,
                          const double* map, int h, int w, const double* mu,
                          const double* omega, const uint8_t* flat, int has_init,
                          double init_threshold, int parallel, int threads, tmo_result* res,
                          uint8_t* visits) {
    return search_impl(t, m, n, img, p, q, map, h, w, mu, omega, flat, has_init, init_threshold,
                       parallel, threads, res, visits);
}

/* ---- matcher.cpp:80-93 ----------------------------------------------------------- */
static cell refine_cells(const double* t, int m, int n, double tmu, double tom, int tfl,
                         const double* img, int q, const double* mu, const double* om,
                         const uint8_t* fl, int er, int ec, int lr, int lc, int d,
                         int64_t* ops) {
    const int r0 = imax(0, lr - d), r1 = imin(er - 1, lr + d);
    const int c0 = imax(0, lc - d), c1 = imin(ec - 1, lc + d);
    cell best = kNoCell;
    for (int r = r0; r <= r1; ++r)
        for (int c = c0; c <= c1; ++c) {
            const double rho = tmo_zncc_at(t, m, n, tmu, tom, tfl, img, q, mu, om, fl, ec, r, c);
            ++*ops;
            cell cand = {r, c, rho, tfl || fl[(size_t)r * ec + c], 1};
            if (better(&cand, &best)) best = cand;
        }
    return best;
}

int tmo_refine(const double* t, int m, int n, const double* img, int p, int q, int loc_row,
               int loc_col, int d, int* row, int* col, double* rho, int* degenerate) {
    if (d < 0) return fail("refine_localization: d must be >= 0");
    const int er = p - m + 1, ec = q - n + 1;
    if (er < 1 || ec < 1) return fail("running_sum: window does not fit the source");
    const size_t E = (size_t)er * ec;
    double tmu, tom;
    int tfl;
    tmo_template_stats(t, m, n, &tmu, &tom, &tfl);
    double* mu = (double*)malloc(E * 8);
    double* om = (double*)malloc(E * 8);
    uint8_t* fl = (uint8_t*)malloc(E);
    tmo_window_stats(img, p, q, m, n, mu, om, fl);
    if (loc_row < 0 || loc_row >= er || loc_col < 0 || loc_col >= ec) {
        free(mu);
        free(om);
        free(fl);
        return fail("refine_localization: location outside the extent");
    }
    int64_t ops = 0;
    cell b = refine_cells(t, m, n, tmu, tom, tfl, img, q, mu, om, fl, er, ec, loc_row, loc_col, d,
                          &ops);
    *row = b.row;
    *col = b.col;
    *rho = b.rho;
    *degenerate = b.degenerate;
    free(mu);
    free(om);
    free(fl);
    return 0;
}

/* ---- matcher.cpp:205-307 --------------------------------------------------------- */
int tmo_match(const double* t, int m, int n, const double* img, int p, int q,
              const tmo_params* prm, tmo_result* res, uint8_t* visits) {
    if (m > p || n > q) return fail("match: template larger than search image");
    double tmu, tom;
    int tfl;
    tmo_template_stats(t, m, n, &tmu, &tom, &tfl);
    if (prm->mode != 0 && tfl) return fail("match: constant template has no defined correlation");
    const double t0 = now_ms();
    const int er = p - m + 1, ec = q - n + 1;
    const size_t E = (size_t)er * ec;
    int rc = 0;
    if (prm->mode == 0) {
        rc = tmo_brute(t, m, n, img, p, q, res, NULL);
        if (!rc && visits) memset(visits, 2, E);
    } else if (prm->mode == 1) {
        double* mu = (double*)malloc(E * 8);
        double* om = (double*)malloc(E * 8);
        uint8_t* fl = (uint8_t*)malloc(E);
        double* map = (double*)malloc(E * 8);
        tmo_window_stats(img, p, q, m, n, mu, om, fl);
        tmo_egs_iter tr[64];
        int h, w, tl;
        rc = tmo_efficient_group_size(img, p, q, m, n, prm->h0, prm->w0, prm->rho_th,
                                      prm->xi_fraction, 127, mu, om, fl, &h, &w, tr, 64, &tl, map);
        if (!rc)
            rc = search_impl(t, m, n, img, p, q, map, h, w, mu, om, fl, prm->has_init_threshold,
                             prm->init_threshold, prm->parallel, prm->threads, res, visits);
        if (!rc) res->mode = 1;
        free(mu);
        free(om);
        free(fl);
        free(map);
    } else {
        const size_t P = (size_t)p * q;
        double* blurred = (double*)malloc(P * 8);
        double trace[4 * 65];
        int kappa, h, w, tl;
        double lambda, cost;
        double* map = (double*)malloc(E * 8);
        rc = tmo_optimize_autocorrelation(img, p, q, m, n, prm, blurred, &kappa, &lambda, &h, &w,
                                          &cost, trace, 65, &tl, map);
        if (!rc) {
            double* mu = (double*)malloc(E * 8);
            double* om = (double*)malloc(E * 8);
            uint8_t* fl = (uint8_t*)malloc(E);
            double* mu_o = (double*)malloc(E * 8);
            double* om_o = (double*)malloc(E * 8);
            uint8_t* fl_o = (uint8_t*)malloc(E);
            tmo_window_stats(blurred, p, q, m, n, mu, om, fl);
            tmo_window_stats(img, p, q, m, n, mu_o, om_o, fl_o);
            if (!rc)
                rc = search_impl(t, m, n, blurred, p, q, map, h, w, mu, om, fl,
                                 prm->has_init_threshold, prm->init_threshold, prm->parallel,
                                 prm->threads, res, visits);
            if (!rc) {
                res->mode = 2;
                const int d = kappa * (prm->kernel_len / 2);
                int64_t rops = 0;
                cell rb = refine_cells(t, m, n, tmu, tom, tfl, img, q, mu_o, om_o, fl_o, er, ec,
                                       res->best_row, res->best_col, d, &rops);
                res->refined_row = rb.row;
                res->refined_col = rb.col;
                res->refined_rho = rb.rho;
                res->ops += rops;
                if (prm->has_init_threshold)
                    res->below_threshold = rb.degenerate || rb.rho < prm->init_threshold;
            }
            free(mu);
            free(om);
            free(fl);
            free(mu_o);
            free(om_o);
            free(fl_o);
        }
        free(map);
        free(blurred);
    }
    if (!rc) res->wall_ms = now_ms() - t0;
    return rc;
}
