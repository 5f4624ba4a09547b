/*
 * tmatch_cuda.h -- C ABI of the B200-native tmatch hot path (libtmatch_cuda.so).
 *
 * This is the drop-in boundary for the reference matcher path (arXiv 1407.3535,
 * /root/reference/proj).  Plain pointers and sizes only; no C++ or torch types.  Every
 * entry point names the reference interface it replaces (file:line in
 * /root/reference/proj/include/tmatch).  The C++ API in include/tmatch/ (a source-level
 * drop-in for the reference headers) is implemented on top of these calls, and the
 * Python package binds them with ctypes.
 *
 * Errors: every int-returning call returns TM_OK (0) or a negative TM_E* code; the
 * thread-local message is in tm_last_error().  TM_EINVAL corresponds to the reference's
 * std::invalid_argument (same message text), TM_ECUDA to a device failure.  There is no
 * CPU fallback: without a usable sm_100a device every call fails with TM_ENODEV.
 *
 * Threading: a tm_ctx owns one CUDA stream and its scratch memory; calls on the same
 * context are serialised internally (mutex), calls on different contexts may run
 * concurrently (the reference is pure and re-entrant).
 */
#ifndef TMATCH_CUDA_H
#define TMATCH_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TM_OK 0
#define TM_EINVAL (-1)
#define TM_ECUDA (-2)
#define TM_ENODEV (-3)
#define TM_ENOMEM (-4)

/* MatchMode (result.hpp:11) */
#define TM_MODE_BRUTE 0
#define TM_MODE_EGS 1
#define TM_MODE_OPTA 2

/* Threshold policy of scan 2 (matcher.cpp:129-148).
 *  TM_POLICY_REFERENCE  follow MatchParams: frozen iff parallel && threads > 1 && groups > 1,
 *                       else the sequential running threshold -- skip counts identical to
 *                       the reference in both cases;
 *  TM_POLICY_FROZEN     threshold frozen at the scan-1 maximum (reference --parallel);
 *  TM_POLICY_SEQUENTIAL running threshold in scan order (reference default);
 *  TM_POLICY_SEEDED     B200 best-first: groups whose centre rho is within seed_margin of
 *                       the scan-1 maximum are searched first and raise the threshold, then
 *                       scan 2 runs frozen at that value.  Sound (every threshold is an
 *                       achieved rho), same argmax, far fewer evaluations. */
#define TM_POLICY_REFERENCE 0
#define TM_POLICY_FROZEN 1
#define TM_POLICY_SEQUENTIAL 2
#define TM_POLICY_SEEDED 3

/* Visit codes (result.hpp:17-21) */
#define TM_VISIT_CENTER 0
#define TM_VISIT_ELIMINATED 1
#define TM_VISIT_RETAINED 2

/* MatchResult + MatchStats (result.hpp:23-60). */
typedef struct {
    int32_t mode;
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
} tm_match_result;

/* MatchParams (matcher.hpp:45-58) plus the B200 policy extension. */
typedef struct {
    int32_t mode;
    int32_t h0, w0;
    int32_t has_init_threshold;
    double init_threshold;
    double rho_th, rho_max;
    double xi_fraction;
    double opta_margin;
    const double* kernel_profile; /* BlurKernel profile (normalised), odd length */
    int32_t kernel_len;
    int32_t parallel, threads;
    int32_t record_visits;
    int32_t policy;     /* TM_POLICY_* */
    int32_t max_group;  /* EgsParams::max_group (egs.hpp:36), default 127 */
    double seed_margin; /* TM_POLICY_SEEDED: centre-rho window for the first pass */
} tm_match_params;

/* EgsIteration / CostEstimate (egs.hpp:15-45) */
typedef struct {
    int32_t h, w;
    double central;
    int64_t retained;
    double retained_cost, amortized, total;
} tm_egs_iter;

/* OptAIteration (blur.hpp:78-83) */
typedef struct {
    int32_t h, w;
    double cost;
    int64_t restored;
} tm_opta_iter;

#define TM_MAX_TRACE 64

/* Summary of a prepared state (PreparedEgs / PreparedOptA, matcher.hpp:61-69). */
typedef struct {
    int32_t mode;                 /* TM_MODE_EGS or TM_MODE_OPTA */
    int32_t m, n;                 /* template size it was prepared for */
    int32_t h, w;                 /* h_e, w_e */
    int32_t extent_rows, extent_cols;
    int32_t kappa;                /* OptA accepted blur iterations */
    double lambda;                /* OptA quality threshold */
    tm_egs_iter cost;             /* final cost estimate */
    int32_t egs_trace_len;
    tm_egs_iter egs_trace[TM_MAX_TRACE];
    int32_t opta_trace_len;
    tm_opta_iter opta_trace[TM_MAX_TRACE + 1];
    double prep_ms;               /* device time of the preparation */
} tm_prep_info;

typedef struct tm_ctx tm_ctx;
typedef struct tm_image tm_image;
typedef struct tm_prep tm_prep;

const char* tm_last_error(void);
void tm_default_params(tm_match_params* p); /* MatchParams defaults, TM_POLICY_REFERENCE */

/* ---- context and images ------------------------------------------------------------ */
int tm_ctx_create(int device, tm_ctx** out);
void tm_ctx_destroy(tm_ctx* ctx);
int tm_ctx_synchronize(tm_ctx* ctx);

/* Image (image.hpp:14-55): host FP64 raster (the reference's storage) or 8-bit pixels.
 * Integer-valued [0,255] images take the exact integer path; anything else takes the FP64
 * replica path. */
int tm_image_create(tm_ctx* ctx, const double* pixels, int rows, int cols, tm_image** out);
int tm_image_create_u8(tm_ctx* ctx, const uint8_t* pixels, int rows, int cols, tm_image** out);
/* Re-upload pixels into an existing image of the same size (no reallocation). */
int tm_image_upload_u8(tm_ctx* ctx, tm_image* img, const uint8_t* pixels);
int tm_image_download(tm_ctx* ctx, const tm_image* img, double* out);
int tm_image_is_integer(const tm_image* img);
void tm_image_destroy(tm_image* img);

/* ---- stats.hpp ---------------------------------------------------------------------- */
/* running_sum (stats.hpp:25): out (rows-m+1)*(cols-n+1) doubles. */
int tm_running_sum(tm_ctx* ctx, tm_image* img, int m, int n, double* out);
/* window_stats (stats.hpp:49): any output pointer may be NULL. */
int tm_window_stats(tm_ctx* ctx, tm_image* img, int m, int n, double* mu, double* omega,
                    uint8_t* flat);
/* brute_force_match (stats.hpp:67); surface optional (extent doubles). */
int tm_brute_force_match(tm_ctx* ctx, const double* tmpl, int m, int n, tm_image* img,
                         tm_match_result* out, double* surface);

/* ---- autocorr.hpp / egs.hpp ----------------------------------------------------------- */
/* local_autocorrelation (autocorr.hpp:73-75) on build_group_grid(p,q,m,n,h,w). */
int tm_local_autocorrelation(tm_ctx* ctx, tm_image* img, int m, int n, int h, int w,
                             double* map);
/* retained_count (egs.hpp:21) of the map just built for (m,n,h,w). */
int tm_autocorr_retained(tm_ctx* ctx, tm_image* img, int m, int n, int h, int w, double rho_tb,
                         int64_t* n_r);
/* efficient_group_size (egs.hpp:57-59); map optional (extent doubles). */
int tm_efficient_group_size(tm_ctx* ctx, tm_image* img, int m, int n, int h0, int w0,
                            double rho_tb, double xi_fraction, int max_group, int* h, int* w,
                            tm_egs_iter* trace, int* trace_len, double* map);

/* ---- blur.hpp ---------------------------------------------------------------------- */
/* blur (blur.hpp:59-61): out rows*cols doubles. */
int tm_blur(tm_ctx* ctx, tm_image* img, const double* profile, int len, double* out);
/* blur_fidelity_map (blur.hpp:65-66): fid extent doubles. */
int tm_blur_fidelity_map(tm_ctx* ctx, tm_image* img, tm_image* blurred, int m, int n,
                         double* fid);

/* unblur_violations (blur.hpp:70-71): restore the window of every location whose fidelity
 * (fid, extent doubles) is below lambda; out = restored image, count = marked windows. */
int tm_unblur_violations(tm_ctx* ctx, tm_image* blurred, tm_image* original, const double* fid,
                         int m, int n, double lambda, double* out, int64_t* count);

/* ---- matcher.hpp ------------------------------------------------------------------- */
/* prepare_egs / prepare_opta (matcher.hpp:71-72): device-resident PreparedEgs/PreparedOptA
 * (window statistics, R_co map, OptA image) reusable across templates of size m x n. */
int tm_prepare(tm_ctx* ctx, tm_image* img, int m, int n, const tm_match_params* params,
               tm_prep** out);
int tm_prep_get_info(const tm_prep* prep, tm_prep_info* info);
/* Host views of the prepared state (lazy download): map = extent doubles; image = the
 * search image of the preparation (OptA: the optimised blurred image). */
int tm_prep_download(tm_ctx* ctx, const tm_prep* prep, double* map, double* image);
void tm_prep_destroy(tm_prep* prep);

/* run_egs / run_opta (matcher.hpp:74-77) for a batch of ntmpl templates (m x n each,
 * contiguous FP64), one result per template.  visits optional: ntmpl * extent bytes. */
int tm_run(tm_ctx* ctx, tm_prep* prep, tm_image* img, const double* tmpls, int ntmpl,
           const tm_match_params* params, tm_match_result* out, uint8_t* visits);
/* Same with 8-bit templates (no host-side conversion). */
int tm_run_u8(tm_ctx* ctx, tm_prep* prep, tm_image* img, const uint8_t* tmpls, int ntmpl,
              const tm_match_params* params, tm_match_result* out, uint8_t* visits);

/* One full search on a device-resident image: prepare_egs / prepare_opta + run_egs /
 * run_opta (matcher.hpp:80 match, without the image upload).  The template is uploaded
 * while the preparation's kernels run, and no preparation handle is returned. */
int tm_search(tm_ctx* ctx, tm_image* img, const double* tmpl, int m, int n,
              const tm_match_params* params, tm_match_result* out);
int tm_search_u8(tm_ctx* ctx, tm_image* img, const uint8_t* tmpl, int m, int n,
                 const tm_match_params* params, tm_match_result* out);
/* match (matcher.hpp:80) from host memory in one call: upload the 8-bit pixels (rows x
 * cols of `img`) into `img`, then tm_search_u8 (same results as tm_image_upload_u8 +
 * tm_search_u8). */
int tm_search_upload_u8(tm_ctx* ctx, tm_image* img, const uint8_t* pixels, const uint8_t* tmpl,
                        int m, int n, const tm_match_params* params, tm_match_result* out);
/* A stream of matches (match, matcher.hpp:80, once per image; the reference CLI's bench
 * loop over a corpus, cli.cpp:239-293): nimg 8-bit host images of rows x cols, one 8-bit
 * template.  out[i] equals tm_search_upload_u8 on images[i].  Two device image slots owned
 * by the context: image i+1 is copied on a copy stream while image i is searched, so with
 * pinned host buffers the PCIe transfer hides behind the previous search. */
int tm_search_stream_u8(tm_ctx* ctx, const uint8_t* const* images, int nimg, int rows, int cols,
                        const uint8_t* tmpl, int m, int n, const tm_match_params* params,
                        tm_match_result* out);

/* transitive_search (matcher.hpp:37-38) with a caller-supplied map/grid. */
int tm_transitive_search(tm_ctx* ctx, const double* tmpl, int m, int n, tm_image* img,
                         const double* map, int h, int w, const tm_match_params* params,
                         tm_match_result* out, uint8_t* visits);
/* The same with caller-supplied window statistics (E = extent doubles / bytes): run_egs /
 * run_opta on a preparation whose statistics (PreparedEgs::ws, PreparedOptA::ws_blur) were
 * computed from earlier pixels -- the reference correlates the current pixels of I with
 * the prepared statistics and map (matcher.cpp:235-276). */
int tm_transitive_search_ws(tm_ctx* ctx, const double* tmpl, int m, int n, tm_image* img,
                            const double* map, int h, int w, const double* mu,
                            const double* omega, const uint8_t* flat,
                            const tm_match_params* params, tm_match_result* out,
                            uint8_t* visits);
/* center_scan (matcher.hpp:24): rho/degenerate per group in grid order; best cell. */
int tm_center_scan(tm_ctx* ctx, const double* tmpl, int m, int n, tm_image* img, int h, int w,
                   double* rho, uint8_t* degenerate, int* best_row, int* best_col,
                   double* best_rho, int* best_degenerate);
/* refine_localization (matcher.hpp:42-43). */
int tm_refine_localization(tm_ctx* ctx, const double* tmpl, int m, int n, tm_image* original,
                           int loc_row, int loc_col, int d, int* row, int* col, double* rho,
                           int* degenerate);
/* match (matcher.hpp:80): one-shot, host FP64 buffers in and out (the end-to-end path). */
int tm_match(tm_ctx* ctx, const double* tmpl, int m, int n, const double* image, int rows,
             int cols, const tm_match_params* params, tm_match_result* out, uint8_t* visits);

/* ---- row-strip sharding (multi-GPU) ------------------------------------
 * Rank r of W processes the group rows [floor(r*tr/W), floor((r+1)*tr/W)) of the grid; the
 * host exchanges the few scalars between the phases (paper_1407_3535_b200/distributed.py):
 *   EGS:    tm_strip_autocorr per candidate -> allreduce SUM n_r -> egs.cpp:61-88 decision
 *           -> tm_strip_commit of the accepted candidate;
 *   search: tm_strip_search_begin (scan 1, local threshold) -> allreduce MAX ->
 *           [seeded: tm_strip_search_seed -> allreduce MAX] -> tm_strip_search_finish ->
 *           allgather of tm_strip_part -> better_candidate merge, sums of the counts.
 * Frozen and seeded policies only (the sequential threshold is a single global scan). */
typedef struct {
    double best_rho;
    int32_t best_row, best_col, best_flags; /* flags: bit0 valid, bit1 degenerate */
    int32_t _pad0;
    int64_t centers, eliminated, retained;
    double final_threshold; /* max(threshold used, best non-degenerate survivor rho) */
} tm_strip_part;

int tm_strip_autocorr(tm_ctx* ctx, tm_image* img, int m, int n, int h, int w, int rank, int world,
                      double rho_tb, int slot, int64_t* n_r);
int tm_strip_commit(tm_ctx* ctx, tm_image* img, int m, int n, int slot, int h, int w,
                    const tm_match_params* params, const tm_egs_iter* trace, int trace_len,
                    tm_prep** out);
/* Row-strip images (one rank of a strip-sharded search): a rows x cols 8-bit image of
 * which only rows [row0, row0 + nrows) -- the rank's strip plus its template_height-1 halo
 * -- are uploaded (pixels: nrows x cols); window statistics are computed for the extent
 * rows whose windows lie in them.  The image-global flat-noise floor (stats.cpp:78-81) is
 * set from the allreduced sum of squares: each rank sums a disjoint row range
 * (tm_image_sum_sq_rows), the caller allreduces, tm_image_set_noise_floor applies it. */
int tm_image_create_strip_u8(tm_ctx* ctx, int rows, int cols, int row0, int nrows,
                             const uint8_t* pixels, tm_image** out);
int tm_image_upload_strip_u8(tm_ctx* ctx, tm_image* img, const uint8_t* pixels);
int tm_image_sum_sq_rows(tm_ctx* ctx, tm_image* img, int row0, int nrows, uint64_t* q_sum);
int tm_image_set_noise_floor(tm_ctx* ctx, tm_image* img, uint64_t q_total);
int tm_strip_search_begin(tm_ctx* ctx, tm_prep* prep, tm_image* img, const double* tmpl,
                          const tm_match_params* params, int rank, int world, double* T0);
int tm_strip_search_seed(tm_ctx* ctx, double T, double* T1);
int tm_strip_search_finish(tm_ctx* ctx, double T, tm_strip_part* out);
/* Fused row-strip protocol (8-bit data, EGS, frozen / seeded policies): the single-GPU
 * fused search split at its global decisions -- begin (strip statistics + scan 1 on the
 * predicted grid -> T0), [seed -> T1], egs (the candidate batch on the strip, scan 2 fused
 * into the predicted size's R_co at the global T -> local retained counts per candidate),
 * finish (after the allreduced counts confirm the predicted size: survivors -> part).
 * *supported == 0 from begin: use the tm_strip_search_* protocol instead. */
int tm_strip_fused_begin(tm_ctx* ctx, tm_image* img, const double* tmpl, int m, int n,
                         const tm_match_params* params, int rank, int world, int pred,
                         int* supported, double* T0);
int tm_strip_fused_seed(tm_ctx* ctx, double T, double* T1);
int tm_strip_fused_egs(tm_ctx* ctx, double T, int* nc, int* hs, int64_t* n_r);
int tm_strip_fused_finish(tm_ctx* ctx, tm_strip_part* out);

/* Instrumentation: number of kernels this context launched (bench gpu_launches). */
int64_t tm_ctx_launch_count(const tm_ctx* ctx);
/* tm_search h_e predictions (the fused scan-2 path ran on the accepted size / did not). */
int tm_ctx_search_stats(const tm_ctx* ctx, int64_t* fused_hits, int64_t* fused_misses);
/* Split tensor-core screening of non-integer images (detail.hpp:32-51 bracketed on three
 * byte planes, see k_tc.cu): locations bracketed / locations re-evaluated by the FP64
 * replica since the context was created. */
int tm_ctx_split_stats(const tm_ctx* ctx, int64_t* screened, int64_t* exact);
/* The context's CUDA stream (cudaStream_t) for callers that time or order work on it. */
void* tm_ctx_stream(tm_ctx* ctx);
/* Per-phase device timing with CUDA events on the context stream (off by default). */
int tm_ctx_set_profiling(tm_ctx* ctx, int enable);
/* JSON {"phase": [launch_groups, total_ms], ...} accumulated since profiling was enabled. */
int tm_ctx_phase_times(tm_ctx* ctx, char* buf, size_t len);
/* Drop the cached window statistics so the next call recomputes them (benchmarks). */
int tm_image_reset_cache(tm_image* img);

#ifdef __cplusplus
}
#endif
#endif
