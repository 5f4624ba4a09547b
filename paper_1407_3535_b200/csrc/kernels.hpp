// kernels.hpp -- host-callable launchers for the tmatch sm_100a kernels.
//
// Every launcher is asynchronous on the given stream and returns the launch error.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace tmk {

constexpr int kU8PadRows = 16;  // zero rows stored below every 8-bit image

// Survivor evaluation: the masked dense tensor-core pass over the strip costs about as much
// as listing E / 1500 survivors on CUDA cores (C5, 96x96: dense 3.8 ms for the whole extent
// vs 22.5 ns per listed survivor), so lists longer than E / kDenseDiv go dense.
constexpr unsigned long long kDenseDiv = 1024;

struct DevStats {  // WindowStats (stats.hpp:35-47) resident in HBM
    double* mu = nullptr;
    double* omega = nullptr;
    uint8_t* flat = nullptr;
    int er = 0, ec = 0, m = 0, n = 0;
};

struct GridDesc {  // GroupGrid (autocorr.hpp:24-52)
    int er, ec, h, w, tr, tc;
    // group rows this device processes (row strip); [0, tr) = everything
    int ti_lo, ti_hi;
};

struct TStatsH {  // TemplateStats (detail.hpp:24-28) + mn
    double mu, omega, mn;
    int flat;
};

struct CellH {  // BestCell, device layout of tmk::Cell
    double rho;
    int row, col;
    int flags;  // bit0 valid, bit1 degenerate
};

struct Tally {  // accumulated on device by the search kernels
    unsigned long long eliminated;
    unsigned long long retained;
    unsigned long long survivors;  // entries appended to the survivor list
    unsigned long long pad;        // sequential replay: candidates alive at their key
    // Retained FLAT members (matcher.cpp:57-76: never eliminated; zncc_at is 0 without a
    // dot, detail.hpp:47) are not listed for evaluation: their cell is (rho 0, degenerate),
    // so only the first one in (row, col) order can matter.  flat_key = max of
    // flat_member_key over them (0: none), flat_n = how many.
    unsigned long long flat_key;
    unsigned long long flat_n;
};

// Survivor tile flags: one byte per (16 extent rows) x (2048 columns) block, set by the
// scan-2 passes for every listed survivor; the masked dense pass (k_tc_corr<2>) skips the
// (band, column tile) tasks whose blocks hold none.  p == nullptr: every task runs.
struct TileFlags {
    uint8_t* p = nullptr;
    int cols = 0;  // ceil(ec / 2048)
};
inline __host__ __device__ size_t tile_flag_bytes(int er, int ec) {
    return size_t((er + 15) >> 4) * size_t((ec + 2047) >> 11);
}
#ifdef __CUDACC__
__device__ __forceinline__ void mark_tile(const TileFlags& f, int r, int c) {
    if (f.p) f.p[size_t(r >> 4) * f.cols + (c >> 11)] = 1;
}
#endif

// Order-reversing key of a position: max over keys = min (row, col) (better_candidate's
// tie order among equal-rho degenerate cells, stats.cpp:147-154).
inline __host__ __device__ unsigned long long flat_member_key(int r, int c) {
    return ((unsigned long long)(0x7FFFFFFFu - unsigned(r)) << 32) |
           (unsigned long long)(0xFFFFFFFFu - unsigned(c));
}
inline __host__ __device__ int flat_key_row(unsigned long long k) {
    return int(0x7FFFFFFFu - unsigned(k >> 32));
}
inline __host__ __device__ int flat_key_col(unsigned long long k) {
    return int(0xFFFFFFFFu - unsigned(k & 0xFFFFFFFFull));
}

// Host-readable result block (one device->host copy per search / EGS batch).
struct ResultBlock {
    unsigned long long nr[4];  // EGS retained counts of a candidate batch
    unsigned long long spec;   // EGS speculation gate of the batch (k_egs_decide)
    unsigned long long seq;    // written last by the batch's final decide (host polls it)
    CellH cells[3];            // best centre, best seeded member, best survivor
    Tally tally;
    double thr;                // threshold after the search
};

// efficient_group_size's accept/stop step (egs.cpp:61-88) after one candidate: the body of
// k_egs_decide, optionally fused into the tail of the candidate's R_co launch (the CTA that
// finishes last runs it; ticket zero between launches, null = not fused).
struct EgsDecide {
    unsigned* ticket = nullptr;
    const unsigned long long* n_r = nullptr;
    double* prev = nullptr;
    int* stop = nullptr;
    int er = 0, ec = 0, h = 0, w = 0;
    double xi = 0.0;
    int cap = 0;
    int* h_acc = nullptr;
    int want = 0;
    unsigned long long* gate = nullptr;
    const unsigned long long* nr_all = nullptr;
    int nc = 0;
    ResultBlock* out = nullptr;  // last candidate of a batch: counts + gate for the host
    unsigned long long seq = 0;
    // with out: k_survivor_dispatch's choice for the survivors enqueued behind the batch
    // (gated: nothing to evaluate unless the gate is set); null = not fused
    const Tally* disp_tally = nullptr;
    unsigned long long disp_E = 0;
    int* disp_dense = nullptr;
    unsigned long long* disp_list = nullptr;
    // Segment order of a count-only candidate: the batch's first candidate (two-pass h = 3
    // R_co) counts its retained members per extent row into rows_out; a later count-only
    // candidate with in-kernel rejection reads them as rows_in and walks its row segments in
    // decreasing order of that density (zorder, set by the launcher), so its partial count
    // reaches the rejection bound after fewer segments.  Null: launch order.
    unsigned* rows_out = nullptr;
    const unsigned* rows_in = nullptr;
    const int* zorder = nullptr;
    // phase B of a two-phase count-only candidate (k_autocorr.cu, k_rco5_s): the members at
    // dj = +-hr of the regular group columns are already counted
    int outer_done = 0;
};

// Scan 2 fused into the R_co launch of the predicted group size (tm_search): scan 1 and the
// seeding ran before it, so each member's bound test (matcher.cpp:48-78 with sec_holds,
// bounds.cpp:41-46) runs where its R_co is computed -- no E-sized map round trip and no
// separate bound pass.  Same decisions, counts, visit codes and survivor list as k_sec_rows.
struct SecFuse {
    const double* thr = nullptr;  // threshold after scan 1 / seeding (null: not fused)
    const double* rho_c = nullptr;
    const double* sa_c = nullptr;  // per-group half_gap factor sqrt(1 - rho_c^2)
    const uint8_t* deg_c = nullptr;
    const uint8_t* seeded = nullptr;  // seeded policy: groups already searched (may be null)
    int tflat = 0;
    int2* locs = nullptr;
    unsigned long long max_locs = 0;
    Tally* tally = nullptr;
    uint8_t* visits = nullptr;
    TileFlags tf{};
};

// Scan 2 of a template batch (k_sec_rows_multi): per-template arrays are [K][G] (group
// level), [K] (thresholds, tallies), [K][cap] (survivor lists), [K][E] (visit codes).
constexpr int kMaxBatch = 32;
struct SecMulti {
    int K = 0;
    size_t G = 0, E = 0;
    const float2* rec = nullptr;      // [K][G] batch_records (the fast test's inputs)
    const double* rho_c = nullptr;    // [K][G] FP64 (the exact test inside the margin)
    const double* sa_c = nullptr;
    const double* thr = nullptr;
    int2* locs = nullptr;
    unsigned long long cap = 0;
    Tally* tally = nullptr;
    uint8_t* visits = nullptr;
    TileFlags tf{};       // template k's flags at tf.p + k * tf_stride
    size_t tf_stride = 0;
};

// Work fused into an argmax reduction (saves launches on the search's critical path).
struct ReduceOp {
    int kind = 0;  // 0 none, 1 threshold init (matcher.cpp:121-125), 2 raise, 3 pack
    int has_init = 0;
    double init = 0.0;
    double* thr = nullptr;
    unsigned long long* zero64 = nullptr;  // kind 1: zeroed counters
    int nzero64 = 0;
    Tally* zero_tally = nullptr;  // kind 1: zeroed tally
    const CellH* cells = nullptr;  // kind 3: cells[0..2] to pack
    const Tally* tally = nullptr;
    ResultBlock* packed = nullptr;
    // kind 1 (fused tm_search path): the EGS batch state k_egs_init would set
    int* egs_stop = nullptr;
    double* egs_prev = nullptr;
    unsigned long long* egs_nr4 = nullptr;
    int* egs_hacc = nullptr;
    unsigned long long* egs_gate = nullptr;
};

// A reduction fused into the tail of the kernel producing the last partials of a phase: the
// block that finishes last reduces partials[0, n) (earlier kernels' included) into *out and
// applies op -- k_reduce_cells without its own launch.  ticket: zero between launches.
struct TailReduce {
    const CellH* partials = nullptr;
    int n = 0;
    CellH* out = nullptr;
    unsigned* ticket = nullptr;  // null: no fused reduction
    ReduceOp op{};
};

// ---- image preparation ---------------------------------------------------------------
cudaError_t check_u8_domain(const double* img, size_t n, int* bad, cudaStream_t s);
cudaError_t f64_to_u8(const double* img, size_t n, uint8_t* out, cudaStream_t s);
cudaError_t u8_to_f32_pitched(const uint8_t* img, int p, int q, float* out, int pitch,
                              cudaStream_t s);
cudaError_t u8_to_f64(const uint8_t* img, size_t n, double* out, cudaStream_t s);
// q_total (stats.cpp:78-79) and prefix_noise (stats.cpp:80-81) on the device.  The 8-bit
// sum is exact; the FP64 sum is a parallel tree sum (parity notes).
cudaError_t prefix_noise_u8(const uint8_t* img, int p, int q, unsigned long long* q_total,
                            double* out, cudaStream_t s);
// Non-integer images: deterministic parallel q_total (`part`: prefix_noise_f64_parts()
// doubles) and the bracketed noise block `nbk` (8 doubles, layout in k_stats.cu).
cudaError_t prefix_noise_f64(const double* img, int p, int q, double* part, double* nbk,
                             cudaStream_t s);
size_t prefix_noise_f64_parts();

// ---- window statistics, exact integer path (stats.cpp:55-94) ---------------------------
// hs/hq scratch: p * ec int32 each.
bool window_stats4_supported(int p, int q, int m, int n, int pitch);
// extent rows [rlo, rhi) only (a row strip; default everything)
cudaError_t window_stats4_u8(const uint8_t* imgp, int pitch, int p, int q, int m, int n,
                             const double* prefix_noise, DevStats st, cudaStream_t s,
                             int rlo = 0, int rhi = 1 << 30);
cudaError_t sum_sq_rows_u8(const uint8_t* img, int q, int r0, int nrows, unsigned long long* out,
                           cudaStream_t s);
cudaError_t window_stats_u8(const uint8_t* img, int p, int q, int m, int n,
                            const double* prefix_noise,
                            int* hs, int* hq, DevStats st, cudaStream_t s);
// Window sums of an 8-bit image as exact doubles (running_sum on integer data).
cudaError_t window_sums_u8(const uint8_t* img, int p, int q, int m, int n, int* hs,
                           double* out, cudaStream_t s);

// ---- FP64 replica running sums (stats.cpp:19-53 operation order) -----------------------
// Source of the prefix table: value(a,b) = X[(a+xo_r)*xq + b+xo_c] (* Y[...] when Y != 0,
// or squared when square != 0), over a rows x cols region.
struct ProdSrc {
    const double* X;
    int xq, xr, xc;
    const double* Y;
    int yq, yr, yc;
    int square;
    const int* stop = nullptr;  // device flag: skip the work when set (EGS early exit)
};
// Up to kProdBatch independent prefix problems per launch (R_co replica offsets).
constexpr int kProdBatch = 16;
struct ProdBatch {
    ProdSrc src[kProdBatch];
    int rows[kProdBatch], cols[kProdBatch];
    int n;
    size_t slot, pslot;  // per-problem stride of rowacc / prefix (elements)
};
cudaError_t replica_prefix_batch(const ProdBatch& b, double* rowacc, double* prefix,
                                 cudaStream_t s);
// rowacc: rows*cols; prefix: (rows+1)*(cols+1) with zero first row/col.
cudaError_t replica_prefix(ProdSrc src, int rows, int cols, double* rowacc, double* prefix,
                           cudaStream_t s);
// out[r][c] = bot[c+n] - top[c+n] - bot[c] + top[c] for the full (rows-m+1)x(cols-n+1).
cudaError_t replica_window_diff(const double* prefix, int rows, int cols, int m, int n,
                                double* out, cudaStream_t s);
// stats epilogue from FP64 window sums S, Q (E entries).
cudaError_t stats_from_sums(const double* S, const double* Q, size_t E, int m, int n,
                            const double* img, int p, int q, double* nbk, DevStats st,
                            cudaStream_t s);

// ---- local auto-correlation + retained count (autocorr.cpp:40-96, egs.cpp:12-25) -------
cudaError_t autocorr_u8(const uint8_t* img, int p, int q, int m, int n, GridDesc g, DevStats st,
                        double retain_threshold, double* map, unsigned long long* n_r,
                        cudaStream_t s);
// Two-pass variant (row walk + column slide) for w in {1,3,...,11}; H scratch of
// autocorr_rowsum_bytes(p, g) bytes.
size_t autocorr_rowsum_bytes(int p, GridDesc g);
bool autocorr_two_pass_supported(int m, int n, GridDesc g);
cudaError_t autocorr_u8_two_pass(const uint8_t* img, int p, int q, int m, int n, GridDesc g,
                                 DevStats st, double retain_threshold, double* map,
                                 unsigned long long* n_r, int* H, cudaStream_t s);
// Fused sliding-window variant (preferred): no scratch, one launch.
bool autocorr_fused_supported(int m, int n, GridDesc g);
cudaError_t autocorr_u8_fused(const uint8_t* img, int p, int q, int m, int n, GridDesc g,
                              DevStats st, double retain_threshold, double* map,
                              unsigned long long* n_r, int* stop, cudaStream_t s,
                              const double* egs_prev = nullptr, double egs_central = 0.0,
                              double egs_xi = 0.0, const uint8_t* imgp = nullptr, int pitch = 0,
                              const EgsDecide* dec = nullptr, bool* decided = nullptr,
                              const SecFuse* fuse = nullptr, int* launches = nullptr);
// The group-column R_co kernel can run scan 2 in its epilogue (SecFuse) for this geometry.
bool autocorr_sec_fuse_supported(int m, int n, GridDesc g);
// k_egs_decide with a full decision record (the dispatch fields included)
cudaError_t egs_decide_d(const EgsDecide& d, cudaStream_t s);
cudaError_t egs_decide(const unsigned long long* n_r, double* prev_cost, int* stop, int er, int ec,
                       int h, int w, double xi, int cap, int* h_acc, int want,
                       unsigned long long* gate, cudaStream_t s,
                       const unsigned long long* nr_all = nullptr, int nc = 0,
                       ResultBlock* out = nullptr, unsigned long long seq = 0);
// Column-walk variant: V scratch of autocorr_colwalk_bytes(q, g) bytes.
size_t autocorr_colwalk_bytes(int q, GridDesc g);
bool autocorr_colwalk_supported(int m, int n, int q, GridDesc g);
cudaError_t autocorr_u8_colwalk(const uint8_t* img, int p, int q, int m, int n, GridDesc g,
                                DevStats st, double retain_threshold, double* map,
                                unsigned long long* n_r, unsigned* V, cudaStream_t s);
// replica path, one offset: cross-sum prefix table of the product image for (di,dj).
// the R_co epilogue of a batch of offsets (one launch; prefix tables pslot apart)
struct OffBatch {
    int n = 0;
    int di[kProdBatch], dj[kProdBatch], pw[kProdBatch];
};
cudaError_t autocorr_offset_epilogue_b(const double* prefix, size_t pslot, const OffBatch& ob,
                                       int m, int n, GridDesc g, DevStats st, double* map,
                                       cudaStream_t s, const int* stop);
cudaError_t autocorr_offset_epilogue(const double* prefix, int ph, int pw, int m, int n,
                                     GridDesc g, DevStats st, int di, int dj, double* map,
                                     cudaStream_t s, const int* stop = nullptr);
cudaError_t autocorr_init(double* map, GridDesc g, cudaStream_t s,
                          const int* stop = nullptr);  // zeros + centres=1
cudaError_t retained_count(const double* map, GridDesc g, double threshold,
                           unsigned long long* n_r, cudaStream_t s, const int* stop = nullptr);

// ---- correlation -----------------------------------------------------------------------
struct CorrJob {
    // image (integer path: imgb for the list kernel, imgf for the dense CUDA-core band
    // kernel; FP64 path: imgd)
    const float* imgf;
    int pitch;  // floats per row of imgf
    const uint8_t* imgb;  // the 16-byte-pitched 8-bit copy
    int bpitch;
    const double* imgd;
    int q;  // columns of imgd
    // template
    const float* tf;  // m x npad, zero padded
    int npad;
    const double* td;  // m x n
    int m, n;
    int flush_rows;  // FP32-exact flush period in template rows
    TStatsH ts;
    DevStats st;
};

// Dense band evaluation over rows[] x {cbase + k*sw : k < nc}.  mode 0: argmax (+surface
// if out_rho != 0, indexed r*ec + c); mode 1: centre scan (out_rho/out_deg indexed
// yi*tc + k + col0); mode 2: masked by visits == 2 (survivor tiles).
struct BandTask {
    const int* rows;
    int nrows;
    int cbase, sw, nc;
    int mode;
    int yi_base;   // mode 1: group row of rows[0] (row strips)
    int row_span;  // max over 8-row bands of rows[yb+7]-rows[yb] (staging height - kIC)
    int col0;  // column-index offset for mode 1 group indexing
    int tc;    // groups per grid row (mode 1)
    double* out_rho;
    uint8_t* out_deg;
    const uint8_t* mask;  // mode 2
    // K split: ksplit CTAs per output tile, each over `ms` template rows; partial dots are
    // atomically accumulated into `dot` (exact integers in FP64) and no epilogue runs.
    int ksplit;
    int ms;
    double* dot;
};
cudaError_t corr_band(const CorrJob& job, const BandTask& task, CellH* partials,
                      int* n_partials, cudaStream_t s);
// Warp-per-location evaluation of a location list (int2 row,col), argmax into partials.
// out_rho/out_deg (optional) are indexed by list position.
// out_rho indexed by list position, or by location (r*ec+c) when rho_by_loc.
cudaError_t corr_list(const CorrJob& job, const int2* locs, const unsigned long long* count,
                      int max_count, double* out_rho, uint8_t* out_deg, CellH* partials,
                      int n_partials, cudaStream_t s, int rho_by_loc = 0,
                      const TailReduce* tail = nullptr);
// FP64 replica (window_dot order, detail.hpp:32-41) over a location list or a dense range.
cudaError_t corr_list_f64(const CorrJob& job, const int2* locs, const unsigned long long* count,
                          int max_count, double* out_rho, uint8_t* out_deg, CellH* partials,
                          int n_partials, cudaStream_t s, int rho_by_loc = 0);
cudaError_t corr_dense_f64(const CorrJob& job, double* surface, CellH* partials, int n_partials,
                           cudaStream_t s);

// Epilogue of a K-split centre scan (rho/deg from the accumulated dots + argmax partials).
struct CentreStats {  // window statistics of the group centres, one entry per group
    double* mu = nullptr;
    double* om = nullptr;
    uint8_t* fl = nullptr;
};
cudaError_t centre_epilogue(const CorrJob& job, GridDesc g, const int* rows, int cbase, int sw,
                            int nc, int col0, const double* dot, double* rho_c, uint8_t* deg_c,
                            CellH* partials, int n_partials, cudaStream_t s, int c_last = -1,
                            const TailReduce* tail = nullptr, const int* gate = nullptr,
                            double* sa_out = nullptr,
                            float2* rec_out = nullptr, const CentreStats* cs = nullptr);
// cs[gi] = statistics at group gi's centre (a template batch gathers them once)
cudaError_t gather_centre_stats(GridDesc g, DevStats st, CentreStats out, cudaStream_t s);
// rho_c[i*tc + col] = rho[i] (clipped last centre column after a list evaluation).
cudaError_t scatter_column(const double* rho, const uint8_t* deg, int n, int tc, int col,
                           double* rho_c, uint8_t* deg_c, cudaStream_t s);
// Reduce partial cells -> out[0] (better_candidate order).
cudaError_t reduce_cells(const CellH* partials, int n, CellH* out, cudaStream_t s,
                         const ReduceOp* op = nullptr);
// dst[i] = src[i] for i < n (one thread; dst may be mapped pinned host memory).
// EGS batch start: stop = 0, prev cost = +inf, nr[0..3] = 0 (one launch).
cudaError_t egs_init(int* stop, double* prev, unsigned long long* nr4, cudaStream_t s,
                     int* h_acc = nullptr, unsigned long long* gate = nullptr);

// ---- scan 2 (matcher.cpp:48-78) ---------------------------------------------------------
// threshold read from *thr (device).  Survivors appended to locs (int2) with counters in
// tally.  visits (optional, E bytes) receives kVisit codes.
cudaError_t sec_compact(GridDesc g, const double* map, const double* rho_c,
                        const uint8_t* deg_c, const uint8_t* flat, int tflat, const double* thr,
                        const uint8_t* seeded, int2* locs, unsigned long long max_locs,
                        Tally* tally, uint8_t* visits, cudaStream_t s);
// Threshold bootstrap: thr = max(best non-degenerate centre rho, init) (matcher.cpp:121-125)
// Row-structured scan 2 (same results as sec_compact); sa_c: G doubles of scratch.
cudaError_t sec_rows_multi(GridDesc g, const double* map, const uint8_t* flat,
                           const SecMulti& sm, cudaStream_t s);
// K rounded up to a power of two (>= 2): the kernel variant of a batch
int batch_kp(int K);
// rec[g] = {float(clamp(rho_c)), float(sa_c) | -1 degenerate | -2 seeded} for one template
cudaError_t batch_records(const double* rho_c, const double* sa_c, const uint8_t* deg_c,
                          const uint8_t* seeded, size_t G, float2* rec, cudaStream_t s);
// y = sqrt(max(0, 1 - clamp(x)^2)) (one half_gap factor, bounds.cpp:21-23)
cudaError_t sqrt_gap(const double* x, double* y, size_t n, cudaStream_t s);
cudaError_t sec_rows(GridDesc g, const double* map, const double* rho_c, double* sa_c,
                     const uint8_t* deg_c, const uint8_t* flat, int tflat, const double* thr,
                     const uint8_t* seeded, int2* locs, unsigned long long max_locs, Tally* tally,
                     uint8_t* visits, cudaStream_t s, bool sa_ready = false, TileFlags tf = TileFlags{});
cudaError_t threshold_init(const CellH* centre_best, int has_init, double init, double* thr,
                           cudaStream_t s);
// Seeded policy: members of every group whose centre rho >= thr - margin -> list.
cudaError_t seed_members(GridDesc g, const double* rho_c, const uint8_t* deg_c, const double* thr,
                         double margin, uint8_t* seeded, int2* locs, unsigned long long* count,
                         unsigned long long max_locs, unsigned long long* n_groups,
                         unsigned long long max_groups, cudaStream_t s,
                         float2* rec = nullptr);
cudaError_t threshold_raise(const CellH* best, double* thr, cudaStream_t s);
// Sequential policy replay: candidates = scan-2 survivors at T0 with their rho.
// rho: extent-sized, indexed by location.
cudaError_t first_record(GridDesc g, const int2* locs, const unsigned long long* count,
                         const double* rho, const double* map,
                         const double* rho_c, const uint8_t* deg_c, const uint8_t* flat, int tflat,
                         double T, unsigned long long after, unsigned long long* best_key,
                         cudaStream_t s);
cudaError_t fetch_record_rho(GridDesc g, const int2* locs, const unsigned long long* count,
                             const double* rho, unsigned long long key, double* out,
                             cudaStream_t s);
cudaError_t seq_final(GridDesc g, const int2* locs, const unsigned long long* count,
                      const double* rho, const double* map,
                      const double* rho_c, const uint8_t* deg_c, const uint8_t* flat, int tflat,
                      double T0, const unsigned long long* rec_key, const double* rec_T, int n_rec,
                      Tally* tally, uint8_t* visits, CellH* partials, int n_partials,
                      cudaStream_t s);

// ---- blur / OptA (blur.cpp) -----------------------------------------------------------
cudaError_t blur_replica(const double* img, int p, int q, const double* prof_dev, int len,
                         double* tmp, double* out, cudaStream_t s);
cudaError_t fidelity_epilogue(const double* cross, DevStats orig, DevStats blur, double* fid,
                              cudaStream_t s);
cudaError_t changed_mask(const double* a, const double* b, size_t n, uint8_t* out,
                         cudaStream_t s);
cudaError_t mark_violations(const double* fid, const double* changed_in_window, size_t E,
                            double lambda, uint8_t* marks, unsigned long long* count,
                            cudaStream_t s);
cudaError_t restore_covered(double* blurred, const double* original, const uint8_t* marks,
                            int er, int ec, int m, int n, int p, int q, int* scratch,
                            cudaStream_t s);


// ---- integer tensor-core correlation (k_tc.cu) --------------------------------------
constexpr int kTcMaxChunks = 8;
constexpr int kTcMaxClasses = 12;
struct TcPlan {  // B arrangement + shared-memory plan for one (template size, row stride)
    int kx = 0, sr = 1, nch = 0;
    int a_bytes = 0, a_slot = 0, stages = 0, header = 0;
    int i0[kTcMaxChunks] = {}, i1[kTcMaxChunks] = {};
    int cls_off[kTcMaxChunks][kTcMaxClasses] = {};
    int cls_max[kTcMaxChunks][kTcMaxClasses] = {};
    size_t b_off[kTcMaxChunks] = {}, b_bytes[kTcMaxChunks] = {};
    size_t total_bytes = 0, b_smem = 0, smem = 0;
};
struct TcJob {
    const uint8_t* imgp;  // pitched 8-bit image (tc_pitch), zero padded
    int pitch;
    // split modes (3, 4): three byte planes of a non-integer image (tc_split_image), plane
    // pl at imgp + pl*plane_stride; scr_delta / scr_gamma: the error model of tc_split.
    size_t plane_stride = 0;
    double scr_delta = 0.0, scr_gamma = 0.0;
    const uint8_t* bglob;  // tc_build_b output
    TcPlan plan;
    TStatsH ts;
    DevStats st;
};
struct TcBand {  // output rows r0 + sr*k, k < cnt (cnt <= 16); yi0 = group row of k = 0
    int r0, sr, cnt, yi0;
};
struct TcTask {
    const TcBand* bands;
    int nbands, ntc;  // tiles = bands x 2048-column tiles
    int mode;         // 0 dense (out_rho = surface), 1 centres, 2 dense masked (mask == 2),
                      // 3 dense screening of a split (non-integer) image: out_ub = upper
                      // bounds of rho, partials = the largest lower bound (mask != null:
                      // only locations with mask == 2 compete), 4 centres of a split image
    int kp;           // split modes: TMEM slot stride between planes (rows per band <= kp)
    float* out_ub;    // mode 3: upper bound of rho per location (-2 at flat windows)
    int c_lim;        // modes 0/2: output columns < c_lim
    int cbase, cstep, nc, tc;  // mode 1: centre columns cbase + cstep*tj, tj < nc; tc = row stride
    int c_last;                // mode 1: clipped last group's centre column (tj = tc-1) or -1
    double* out_rho;
    uint8_t* out_deg;
    const uint8_t* mask;
    TileFlags tf;       // mode 2: skip (band, column tile) tasks without survivors
    long long* dbg;     // optional per-CTA pipeline wait counters (8 per CTA)
    int dbg_flags;      // timing experiments only: 1 = no image copies, 2 = no epilogue
    const int* gate;    // optional device flag: 0 -> the launch only writes empty partials
    const int4* sched;  // tc_schedule() rows, per chunk at sched_off[ch], sched_len[ch]
    int sched_total;    // rows over all chunks
    int sched_off[kTcMaxChunks], sched_len[kTcMaxChunks];
};
// Device-side choice between the dense (tensor-core) and list survivor evaluation:
// dense_flag = survivors*16 > E, list_count = dense ? 0 : survivors.
cudaError_t survivor_dispatch(const Tally* tally, unsigned long long E, int* dense_flag,
                              unsigned long long* list_count, cudaStream_t s,
                              const unsigned long long* gate = nullptr);
bool tc_supported(int m, int n);
TcPlan tc_plan(int m, int n, int sr, size_t smem_budget);
// rows of a band of rmax rows, see k_tc.cu (4 ints per row)
std::vector<int> tc_schedule(const TcPlan& plan, int rmax, int* off, int* len);
int tc_pitch(int q, int ec);
int tc_tile_cols();
cudaError_t tc_pitch_image(const uint8_t* img, int p, int q, uint8_t* out, int pitch, int rows,
                           cudaStream_t s);
cudaError_t tc_build_b(const float* tf, int npad, int m, int n, const TcPlan& plan, uint8_t* out,
                       cudaStream_t s,
                       const int* gate = nullptr);
cudaError_t tc_corr(const TcJob& job, const TcTask& task, CellH* partials, int* nparts,
                    cudaStream_t s);
// Split (non-integer image) variant, see k_tc.cu "split planes".  tc_split_image writes the
// three zero-padded byte planes of floor(v * 2^16) and raises *bad when a pixel lies outside
// [0, 256); tc_screen_compact lists the locations whose upper bound reaches the largest
// lower bound (best->rho); count may exceed max_count (the caller then falls back).
struct SplitModel {  // dot_ref in [dot_a (1 - gamma), (dot_a + delta)(1 + gamma)]
    double delta, gamma;
};
// Split centre scan (scan 1 on a non-integer image): brackets per centre, the centres whose
// exact rho is still needed (best-centre candidates, undecided seeding / bound tests), and
// the exact values scattered back.  Lists have capacity G; gflag = (G + 3) & ~3 zeroed bytes.
cudaError_t split_centre_epilogue(GridDesc g, const double* dot, DevStats st, TStatsH ts,
                                  SplitModel sm, double* rho_c, double* rad_c, uint8_t* deg_c,
                                  CellH* partials, int n_partials, cudaStream_t s);
cudaError_t split_pick(GridDesc g, const double* rho_c, const double* rad_c, const uint8_t* deg_c,
                       int mode, const CellH* lim, const double* thr, double margin, int2* locs,
                       int* gidx, unsigned long long* count, cudaStream_t s);
cudaError_t split_scatter(const double* rho, const int* gidx, const unsigned long long* count,
                          double* rho_c, double* rad_c, cudaStream_t s);
cudaError_t split_sec_uncertain(GridDesc g, const double* map, const double* rho_c,
                                const double* rad_c, const uint8_t* deg_c, const uint8_t* flat,
                                const double* thr, const uint8_t* seeded, uint8_t* gflag,
                                int2* locs, int* gidx, unsigned long long* count, cudaStream_t s,
                                int moving = 0);
constexpr int kTcSplitPlanes = 3;
constexpr int kTcSplitRows = 5;  // rows per band: 3 planes x 5 rows <= 16 TMEM slots
cudaError_t tc_split_image(const double* img, int p, int q, uint8_t* out, int pitch, int rows,
                           size_t plane_stride, int* bad, cudaStream_t s);
cudaError_t tc_screen_compact(const float* ub, int er, int ec, const CellH* best, int2* locs,
                              unsigned long long* count, unsigned long long max_count,
                              cudaStream_t s);

}  // namespace tmk
