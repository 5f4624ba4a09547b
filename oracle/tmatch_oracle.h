/*
 * tmatch_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This is the parity CHECKER, not the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_1407_3535_b200/csrc, libtmatch_cuda.so) never links or calls it.
 *
 * Plain C99 restatement of /root/reference/proj/src/{stats,bounds,autocorr,egs,blur,
 * matcher}.cpp.  Every function cites the reference lines it follows.  Arithmetic is
 * kept in the reference's FP64 operation order (compile with -ffp-contract=off) so the
 * results are bit-identical to the reference on the same inputs; this is pinned by
 * tests/test_oracle_pin.py against the reference itself (oracle/_ref, built from the
 * read-only sources by oracle/Makefile) and against tests/golden/ fixtures.
 *
 * Conventions: images are row-major double arrays (reference Image, image.hpp:14-55).
 * Functions return 0 on success and a negative code on a precondition failure (the
 * reference throws std::invalid_argument; tmo_last_error() holds the message).
 */
#ifndef TMATCH_ORACLE_H
#define TMATCH_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as tm_match_result in include/tmatch_cuda.h (reference MatchResult,
 * result.hpp:32-60, MatchStats result.hpp:23-30). */
typedef struct {
    int32_t mode; /* 0 brute, 1 egs, 2 opta */
    int32_t best_row, best_col;
    int32_t best_degenerate;
    double best_rho;
    int32_t refined_row, refined_col;
    double refined_rho;
    int32_t below_threshold;
    int32_t extent_rows, extent_cols;
    int32_t _pad0;
    double final_threshold;
    int64_t centers, eliminated, retained, ops;
    double elim_pct;
    double wall_ms;
} tmo_result;

/* Reference MatchParams (matcher.hpp:45-58) flattened; kernel profile passed by pointer. */
typedef struct {
    int32_t mode;
    int32_t h0, w0;
    int32_t has_init_threshold;
    double init_threshold;
    double rho_th, rho_max;
    double xi_fraction;
    double opta_margin;
    const double* kernel_profile; /* normalised 1-D profile, odd length */
    int32_t kernel_len;
    int32_t parallel, threads;
    int32_t record_visits;
} tmo_params;

typedef struct {
    int32_t h, w;
    double central, retained_cost, amortized, total;
    int64_t retained;
} tmo_egs_iter;

const char* tmo_last_error(void);
void tmo_default_params(tmo_params* p);

/* stats.cpp:19-53 -- zero-padded FP64 prefix, 4-read window difference. */
int tmo_running_sum(const double* src, int p, int q, int m, int n, double* out);
/* stats.cpp:55-94 */
int tmo_window_stats(const double* img, int p, int q, int m, int n, double* mu, double* omega,
                     uint8_t* flat);
/* Port only: window_stats with an externally given flat-noise floor (NaN = the image's own
 * stats.cpp:78-81 value), for row strips of a larger image. */
int tmo_window_stats_floor(const double* img, int p, int q, int m, int n, double floor_in,
                           double* mu, double* omega, uint8_t* flat);
/* stats.cpp:98-111 */
void tmo_template_stats(const double* t, int m, int n, double* mu, double* omega, int* flat);
/* detail.hpp:45-51 (window_dot detail.hpp:32-41) */
double tmo_zncc_at(const double* t, int m, int n, double t_mu, double t_omega, int t_flat,
                   const double* img, int q, const double* mu, const double* omega,
                   const uint8_t* flat, int ec, int r, int c);
/* stats.cpp:156-213 */
int tmo_brute(const double* t, int m, int n, const double* img, int p, int q, tmo_result* res,
              double* surface);

/* bounds.cpp:27-59 */
int tmo_transitive_bounds(double rho_tc, double rho_co, double* lower, double* upper);
int tmo_transitive_gap(double rho_tc, double rho_co, double* gap);
int tmo_sec_holds(double rho_tb, double rho_tc, double rho_co, int* holds);
int tmo_elimination_autocorr_threshold(double rho_tb, double rho_tc, double* out);
int tmo_expected_elimination_threshold(double rho_tb, double* out);

/* autocorr.cpp:12-32 geometry; returns group count, fills centres (may be NULL). */
int64_t tmo_group_count(int er, int ec, int h, int w);
/* autocorr.cpp:40-96 */
int tmo_local_autocorrelation(const double* img, int p, int q, int m, int n, int h, int w,
                              const double* mu, const double* omega, const uint8_t* flat,
                              double* map);
/* egs.cpp:12-25 */
int64_t tmo_retained_count(const double* map, int er, int ec, int h, int w, double rho_tb);
/* egs.cpp:39-91; trace has room for max_trace entries; map_out E-sized (may be NULL). */
int tmo_efficient_group_size(const double* img, int p, int q, int m, int n, int h0, int w0,
                             double rho_tb, double xi, int max_group, const double* mu,
                             const double* omega, const uint8_t* flat, int* h_out, int* w_out,
                             tmo_egs_iter* trace, int max_trace, int* trace_len,
                             double* map_out);

/* blur.cpp:57-86 */
int tmo_blur(const double* img, int p, int q, const double* profile, int len, double* out);
/* blur.cpp:88-94 */
int tmo_quality_threshold(double rho_th, double rho_max, double* out);
/* blur.cpp:96-125 */
int tmo_blur_fidelity_map(const double* I, const double* I_blur, int p, int q, int m, int n,
                          double* fid);
/* blur.cpp:243-278; image_out p*q; trace rows {h, w, cost, restored}. */
int tmo_optimize_autocorrelation(const double* img, int p, int q, int m, int n,
                                 const tmo_params* prm, double* image_out, int* kappa,
                                 double* lambda, int* h_out, int* w_out, double* cost_out,
                                 double* trace, int max_trace, int* trace_len,
                                 double* map_out);

/* matcher.cpp:95-177 with an explicit precomputed map/grid/ws; policy follows the
 * reference: frozen iff parallel && threads > 1 && groups > 1, else sequential. */
int tmo_transitive_search(const double* t, int m, int n, const double* img, int p, int q,
                          const double* map, int h, int w, const double* mu,
                          const double* omega, const uint8_t* flat, int has_init,
                          double init_threshold, int parallel, int threads, tmo_result* res,
                          uint8_t* visits);
/* matcher.cpp:80-93 (refine_impl) */
int tmo_refine(const double* t, int m, int n, const double* img, int p, int q, int loc_row,
               int loc_col, int d, int* row, int* col, double* rho, int* degenerate);
/* matcher.cpp:278-307 (match = prepare_* + run_*) */
int tmo_match(const double* t, int m, int n, const double* img, int p, int q,
              const tmo_params* prm, tmo_result* res, uint8_t* visits);

#ifdef __cplusplus
}
#endif
#endif
