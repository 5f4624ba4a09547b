// engine.cpp -- host orchestration of the B200 tmatch hot path behind the C ABI
// (include/tmatch_cuda.h).  C++ host code; all arithmetic on images runs in the sm_100a
// kernels of k_*.cu, the host only sequences them and runs the scalar decisions the
// reference makes between passes (EGS accept/stop, OptA accept, repair fixed point).
//
// Reference control flow mirrored here (file:line in /root/reference/proj/src):
//   window_stats            stats.cpp:55-94        -> WS cache per (image, m, n)
//   efficient_group_size    egs.cpp:39-91          -> run_egs_search()
//   optimize_autocorrelation blur.cpp:243-278      -> run_opta_prep()
//   repair_to_fixed_point   blur.cpp:208-239       -> repair()
//   transitive_search_impl  matcher.cpp:95-177     -> search()
//   refine_impl             matcher.cpp:80-93      -> refine()
//   match / prepare / run   matcher.cpp:205-307    -> tm_prepare / tm_run / tm_match
//
// Compile with -ffp-contract=off: the few host-side FP64 expressions (template stats,
// thresholds, costs) follow the reference's evaluation order.
#include <algorithm>
#include <chrono>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "kernels.hpp"
#include "tmatch_cuda.h"

namespace {

thread_local std::string g_err;

struct TmError {
    int code;
    std::string msg;
};

[[noreturn]] void invalid(const std::string& msg) { throw TmError{TM_EINVAL, msg}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw TmError{TM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
#define CK(x) ck((x), #x)

constexpr double kEps = 2.220446049250313e-16;

// Optional host timeline (TMATCH_HOST_TRACE=1): labelled timestamps printed per API call.
struct HostTrace {
    bool on = std::getenv("TMATCH_HOST_TRACE") != nullptr;
    std::vector<std::pair<const char*, std::chrono::steady_clock::time_point>> pts;
    void mark(const char* l) {
        if (on) pts.emplace_back(l, std::chrono::steady_clock::now());
    }
    void flush(const char* call) {
        if (!on || pts.empty()) return;
        std::fprintf(stderr, "[host] %s:", call);
        for (size_t i = 1; i < pts.size(); ++i)
            std::fprintf(stderr, " %s=%.1f", pts[i].first,
                         std::chrono::duration<double, std::micro>(pts[i].second - pts[i - 1].second)
                             .count());
        std::fprintf(stderr, "\n");
        pts.clear();
    }
};
HostTrace& htrace() {
    static thread_local HostTrace t;
    return t;
}
#define HT(label) htrace().mark(label)

// Stream the current API call runs on (set by guard()); device buffers are allocated and
// freed stream-ordered from the device's memory pool, so buffer churn never synchronises.
thread_local cudaStream_t g_stream = nullptr;

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void ensure(size_t n) {
        if (n <= cap && p) return;
        release();
        s = g_stream;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T), s));
        cap = std::max<size_t>(n, 1);
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        cap = 0;
    }
    void swap(DBuf& o) {
        std::swap(p, o.p);
        std::swap(cap, o.cap);
        std::swap(s, o.s);
    }
};

// Pinned host staging for small uploads (templates, row lists): a copy from it is truly
// asynchronous; the event guards reuse of the buffer.
struct Pinned {
    void* p = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;
    ~Pinned() {
        if (p) cudaFreeHost(p);
        if (done) cudaEventDestroy(done);
    }
    void* get(size_t n) {
        if (!done) CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        CK(cudaEventSynchronize(done));  // previous copy out of this buffer finished
        if (n > cap) {
            if (p) cudaFreeHost(p);
            CK(cudaMallocHost(&p, n));
            cap = n;
        }
        return p;
    }
    void upload(void* dst, const void* src, size_t n, cudaStream_t st) {
        void* h = get(n);
        std::memcpy(h, src, n);
        CK(cudaMemcpyAsync(dst, h, n, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(done, st));
    }
};

// detail.hpp:18-22
bool variance_is_flat_h(double var_sum, double q_sum, long long mn) {
    const double abs_tol = 1e-9 * double(mn);
    const double rel = std::max(1e-13, 4.0 * kEps * double(mn));
    return var_sum <= std::max(abs_tol * abs_tol, rel * q_sum);
}

double clampd(double v, double lo, double hi) { return std::clamp(v, lo, hi); }

// bounds.cpp:13-17
double checked(double rho, const char* name) {
    if (std::abs(rho) > 1.0 + 1e-9) invalid(std::string("correlation out of [-1,1]: ") + name);
    return clampd(rho, -1.0, 1.0);
}

// bounds.cpp:48-59
double elimination_autocorr_threshold_h(double rho_tb, double rho_tc) {
    const double tb = checked(rho_tb, "rho_tb");
    const double tc = checked(rho_tc, "rho_tc");
    const double radicand = 1.0 + tc * tc * tb * tb - (tc * tc + tb * tb);
    return tb * tc + std::sqrt(std::max(0.0, radicand));
}
double expected_elimination_threshold_h(double rho_tb) {
    const double tb = checked(rho_tb, "rho_tb");
    return std::sqrt(std::max(0.0, 1.0 - tb * tb));
}

bool better_h(const tmk::CellH& a, const tmk::CellH& b) {
    if (!(a.flags & 1)) return false;
    if (!(b.flags & 1)) return true;
    const bool da = a.flags & 2, db = b.flags & 2;
    if (da != db) return !da;
    if (a.rho != b.rho) return a.rho > b.rho;
    if (a.row != b.row) return a.row < b.row;
    return a.col < b.col;
}

// The cell of the first retained flat member (Tally::flat_key), invalid if none: rho 0,
// degenerate (zncc_at detail.hpp:47; matcher.cpp:69 marks member_flat as degenerate).
tmk::CellH flat_cell(const tmk::Tally& t) {
    tmk::CellH c{};
    if (t.flat_n) {
        c.rho = 0.0;
        c.row = tmk::flat_key_row(t.flat_key);
        c.col = tmk::flat_key_col(t.flat_key);
        c.flags = 3;
    }
    return c;
}

// Wait for an event by polling (no blocking-sync wake-up latency at the end of a search;
// TMATCH_SPIN=0 uses cudaEventSynchronize).
void spin_wait(cudaEvent_t ev) {
    static const bool spin = [] {
        const char* e = std::getenv("TMATCH_SPIN");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    if (!spin) {
        CK(cudaEventSynchronize(ev));
        return;
    }
    for (;;) {
        const cudaError_t q = cudaEventQuery(ev);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) CK(q);
    }
}

double ms_between(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

}  // namespace

struct Tmpl {
    int m = 0, n = 0, npad = 0;
    bool integer = false;
    tmk::TStatsH ts{};
    int flush_rows = 0;
    const float* tf = nullptr;   // device copies (m x npad FP32, m x n FP64)
    const double* td = nullptr;
};

// Geometry-dependent tensor-core launch data (band table, row schedule, plan), built and
// uploaded once per (template size, row set) and reused by every later search.
struct TcGeo {
    tmk::TcPlan plan{};
    DBuf<tmk::TcBand> bands;
    DBuf<int4> sched;
    DBuf<int> rows;  // the row list itself (centre epilogue)
    int nbands = 0, ntc = 0, sched_total = 0;
    int sched_off[tmk::kTcMaxChunks] = {}, sched_len[tmk::kTcMaxChunks] = {};
};

// ==== context ========================================================================
struct WS {
    DBuf<double> mu, om;
    DBuf<uint8_t> fl;
    int er = 0, ec = 0, m = 0, n = 0;
    bool valid = false;  // false: the image changed; recomputed into the same buffers
    tmk::DevStats dev() const { return tmk::DevStats{mu.p, om.p, fl.p, er, ec, m, n}; }
};

struct tm_ctx {
    ~tm_ctx();
    int device = 0;
    cudaStream_t s = nullptr;
    std::mutex mu;
    // images and preparations keep their context alive: tm_ctx_destroy only marks it
    // closing, and the last dependent object releases it
    std::atomic<int> refs{0};
    std::atomic<bool> closing{false};
    int64_t launches = 0;
    int64_t fused_hits = 0, fused_misses = 0;  // tm_search h_e prediction outcomes
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // scratch (grow-only)
    DBuf<int> hs, hq, markP, acH;
    DBuf<double> rowacc, prefix, S, Q, fid, cross, inwin, dtmp;
    DBuf<uint8_t> u8tmp, marks;
    DBuf<tmk::CellH> partials, cells;
    DBuf<double> thr, seq_rho, rec_T, prof;
    DBuf<tmk::Tally> tally;
    DBuf<unsigned long long> counters, rec_key;
    DBuf<int2> locs, seed_locs;
    DBuf<uint8_t> seq_deg, seeded, deg_c, visits;
    DBuf<double> rho_c, surface, dotbuf;
    DBuf<float> ub_surface;  // split screening: upper bounds of rho
    // split centre scan: bracket radius per group (0 = rho_c exact), the centres picked for
    // the exact replay (location, group index, exact rho) and the per-group listed flags
    DBuf<double> rad_c, split_rho;
    DBuf<int2> split_locs;
    DBuf<int> split_gidx;
    DBuf<uint8_t> split_flag;
    int64_t split_centres = 0;  // centres bracketed by the split centre scan
    // TMATCH_TC_SPLIT: 0 = non-integer images stay on the FP64 replica, 1 (default) = split
    // planes when the pass is large enough to pay for their fixed cost, 2 = always
    int tc_split = 1;
    int64_t split_screened = 0, split_exact = 0;  // locations bracketed / re-evaluated exactly
    DBuf<float> tf;
    DBuf<double> td;
    // the template ctx->tf / ctx->td hold (upload_template skips identical re-uploads);
    // anything else writing tf / td resets tmpl_m
    std::vector<double> tmpl_last;
    int tmpl_m = 0, tmpl_n = 0;
    DBuf<int> rows_list;
    DBuf<double> map_tmp, map_user, map_fused;
    DBuf<double> egs_maps[4];
    DBuf<double> sa_c;  // per-group half_gap factor sqrt(1 - rho_c^2) (scan 2)
    DBuf<unsigned> egs_rows;  // per-extent-row retained counts of a batch's first candidate
    bool sa_ready = false;  // sa_c filled by this search's centre epilogue
    float2* batch_rec = nullptr;  // run_batch: the centre epilogue also writes the records
    // run_batch: the centres' window statistics gathered once per batch (compact, per group)
    DBuf<double> cs_mu, cs_om;
    DBuf<uint8_t> cs_fl;
    bool batch_cs = false;
    Pinned pin_tf, pin_td, pin_rows, pin_locs, pin_cnt, pin_egs;
    // row-strip search protocol state (tm_strip_search_*)
    struct StripState {
        bool active = false;
        tm_prep* prep = nullptr;
        tm_image* img = nullptr;
        tmk::GridDesc g{};
        tm_match_params P{};
        int policy = TM_POLICY_FROZEN;
        int m = 0, n = 0;
        Tmpl T{};
        // fused protocol (tm_strip_fused_*): predicted group size, its strip grid, the
        // extent, the survivor tile flags and the EGS candidates of the batch
        bool fused = false;
        int pred = 0, er = 0, ec = 0, rank = 0, world = 1;
        tmk::TileFlags tf{};
        int nc = 0, cand_h[4] = {0, 0, 0, 0};
    } strip;
    void add(int k) { launches += k; }
    // optional per-phase device timing (CUDA events on the context stream)
    bool profiling = false;
    // R_co kernel choice: fused sliding-window (default) or the column-walk + line-scan pair
    // (TMATCH_AUTOCORR=colwalk; kept for A/B measurements and as a cross-check in tests)
    bool ac_fused = true;
    // EGS count-only candidates ordered by the first candidate's row density (TMATCH_EGS_ORDER=0
    // keeps the launch order)
    bool egs_order = [] {
        const char* e = std::getenv("TMATCH_EGS_ORDER");
        return !(e && std::atoi(e) == 0);
    }();
    // window statistics: four columns per thread (TMATCH_WSTATS=column: one per column)
    bool ws4 = true;
    // integer tensor-core correlation (tcgen05 kind::i8) for centre scans / dense work;
    // TMATCH_TC=0 selects the CUDA-core FP32-exact kernels (A/B measurements, cross-checks)
    bool tc = true;
    DBuf<uint8_t> tc_b;
    std::map<std::vector<long long>, std::unique_ptr<TcGeo>> tc_geo;
    // pinned readback block: device->host copies into it are asynchronous, so the host can
    // keep working (e.g. upload the next template) until it synchronises
    // template batches (run_batch): per-template scan-1 state, scan-2 outputs, results
    DBuf<uint8_t> tflags;  // survivor tile flags of the current search (tmk::TileFlags)
    struct Batch {
        DBuf<uint8_t> tflags;
        DBuf<float> tf;
        DBuf<double> td, rho, sa, thr;
        DBuf<uint8_t> vis;
        DBuf<float2> rec;
        DBuf<int2> locs;
        DBuf<tmk::Tally> tally;
        DBuf<tmk::CellH> cells;
        DBuf<tmk::ResultBlock> packed;
        Pinned pin_tf, pin_td;
        std::vector<tmk::ResultBlock> host;
    } batch;
    using HostRes = tmk::ResultBlock;
    HostRes* hres = nullptr;      // pinned, mapped: kernels write results straight into it
    HostRes* hres_dev = nullptr;  // its device address
    // side stream for template uploads overlapped with the preparation's kernels
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev_t = nullptr;
    cudaEvent_t ev_egs = nullptr;  // end of an EGS batch's count copy
    // speculative B build on the side stream: tc_b sized before the EGS batch (ev_b0), the
    // build done (ev_b1); spec_b: this search's hook may build B on the side stream
    cudaEvent_t ev_b0 = nullptr, ev_b1 = nullptr;
    bool spec_b = false;
    // speculative centre scan (tm_search): predicted group size passed to the EGS decide
    // kernels, and what was enqueued for it
    int spec_want = 0;
    unsigned long long egs_seq = 0;  // EGS batches launched (ResultBlock::seq)
    struct Spec {
        bool armed = false;
        tmk::GridDesc g{};
        const int* rows_dev = nullptr;
    } spec;
    std::map<std::vector<long long>, int> last_he;  // (p, q, m, n, h0, w0) -> last accepted h
    // streamed searches (tm_search_stream_u8): two device image slots and a copy stream, so
    // image i+1 crosses PCIe while image i is searched
    cudaStream_t s_up = nullptr;
    cudaEvent_t ev_up[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
    std::unique_ptr<tm_image> sslot[2];
    // enqueued by search() right before its final synchronisation (tm_search_stream_u8: the
    // next image's layout copy and window statistics run while the host reads this result)
    std::function<void()> before_final_sync;
    bool ev1_set = false;  // search() recorded ev1 before running before_final_sync
    struct Mark {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Mark> pending;
    std::vector<cudaEvent_t> pool;
    std::map<std::string, std::pair<long long, double>> phase_ms;  // name -> (count, ms)
    cudaEvent_t get_event() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    void resolve() {  // call after a stream synchronisation
        for (auto& mk : pending) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, mk.a, mk.b);
            auto& slot = phase_ms[mk.name];
            slot.first += 1;
            slot.second += ms;
            pool.push_back(mk.a);
            pool.push_back(mk.b);
        }
        pending.clear();
    }
};

// RAII phase timer: brackets the launches issued in its scope with two events.
struct Phase {
    tm_ctx* ctx;
    const char* name;
    cudaEvent_t a = nullptr;
    Phase(tm_ctx* c, const char* n) : ctx(c), name(n) {
        if (ctx->profiling) {
            a = ctx->get_event();
            cudaEventRecord(a, ctx->s);
        }
    }
    ~Phase() {
        if (ctx->profiling) {
            cudaEvent_t b = ctx->get_event();
            cudaEventRecord(b, ctx->s);
            ctx->pending.push_back(tm_ctx::Mark{name, a, b});
        }
    }
};

struct tm_image {
    tm_ctx* ctx = nullptr;
    int p = 0, q = 0;
    bool integer = false;
    DBuf<uint8_t> u8;
    DBuf<float> f32;
    bool have_f32 = false;  // f32 is current (made on demand, ensure_f32)
    int pitch = 0;
    DBuf<double> f64;
    bool have_f64 = false;
    bool have_qtotal = false;  // prefix_noise computed on the device
    DBuf<double> pn;           // [1] prefix_noise; FP64 path: the noise block (k_stats.cu)
    DBuf<double> pnpart;       // FP64 path: per-block partial sums of squares
    DBuf<unsigned long long> qt;
    std::map<std::pair<int, int>, std::unique_ptr<WS>> ws_cache;
    // 16-byte pitched zero-padded 8-bit copy for the tensor-core path (k_tc.cu)
    DBuf<uint8_t> u8p;
    int u8p_pitch = 0;
    int u8p_rows = 0;
    // non-integer images: the three byte planes of floor(v * 2^16) for the split
    // tensor-core screening (k_tc.cu, "split planes"); split_ok = every pixel in [0, 256)
    DBuf<uint8_t> split;
    int split_pitch = 0;
    size_t split_stride = 0;
    bool have_split = false, split_ok = false;
    // Row-strip image (tm_image_create_strip_u8): only image rows [row_lo, row_hi) hold
    // pixels (the rank's strip + halo); window statistics cover the extent rows whose
    // windows lie inside them; prefix_noise comes from the allreduced global q_total.
    int row_lo = 0, row_hi = 1 << 30;
    bool noise_external = false;
};

tm_ctx::~tm_ctx() {
    sslot[0].reset();  // stream-ordered frees on s, before the scratch buffers
    sslot[1].reset();
}

struct tm_prep {
    tm_match_params params{};
    std::vector<double> profile;
    int mode = TM_MODE_EGS;
    int m = 0, n = 0, h = 0, w = 0;
    tmk::GridDesc g{};
    DBuf<double> map;
    std::unique_ptr<tm_image> search_img;  // OptA: optimised image (owned)
    std::unique_ptr<WS> search_ws;          // OptA: window stats of the optimised image
    int kappa = 0, radius = 0;
    double lambda = 1.0;
    tm_egs_iter cost{};
    std::vector<tm_egs_iter> egs_trace;
    std::vector<tm_opta_iter> opta_trace;
    double prep_ms = -1.0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    tm_image* source = nullptr;  // not owned
    tm_ctx* ctx = nullptr;       // keeps the context alive (ref)
    ~tm_prep() {
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
    }
};

namespace {

tmk::GridDesc make_grid(int er, int ec, int h, int w) {
    if (er < 1 || ec < 1) invalid("group grid: empty search extent");
    if (h < 1 || w < 1 || h % 2 == 0 || w % 2 == 0)
        invalid("group grid: group size must be odd and >= 1");
    const int tr = (er + h - 1) / h, tc = (ec + w - 1) / w;
    return tmk::GridDesc{er, ec, h, w, tr, tc, 0, tr};
}

// Row strip `rank` of `world`: an even split of the group rows.
tmk::GridDesc strip_of(tmk::GridDesc g, int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) invalid("strip: bad rank/world");
    g.ti_lo = int((long long)g.tr * rank / world);
    g.ti_hi = int((long long)g.tr * (rank + 1) / world);
    return g;
}

int centre_row_h(const tmk::GridDesc& g, int ti) {
    const int r0 = ti * g.h, r1 = std::min(r0 + g.h, g.er) - 1;
    return (r0 + r1) / 2;
}
int centre_col_h(const tmk::GridDesc& g, int tj) {
    const int c0 = tj * g.w, c1 = std::min(c0 + g.w, g.ec) - 1;
    return (c0 + c1) / 2;
}

// ---- images ----------------------------------------------------------------------------
// 8-bit pixels are stored with tmk::kU8PadRows zero rows below the image, so row walks
// may read a few rows past the bottom without bounds checks (k_acf).
void alloc_u8(tm_ctx* ctx, tm_image* img) {
    const size_t N = size_t(img->p) * img->q;
    const size_t pad = size_t(tmk::kU8PadRows) * img->q;
    img->u8.ensure(N + pad);
    CK(cudaMemsetAsync(img->u8.p + N, 0, pad, ctx->s));
}

// Layout conversions of a new 8-bit raster: the FP32 copy (list kernels) and the
// 16-byte-pitched copy for the tensor-core kernels (sized for any template width).
void tc_pitch_copy(tm_ctx* ctx, tm_image* img) {
    const int pitch = tmk::tc_pitch(img->q, img->q);
    const int rows = img->p + tmk::kU8PadRows;  // zero rows below: look-ahead reads
    img->u8p.ensure(size_t(rows) * pitch);
    CK(tmk::tc_pitch_image(img->u8.p, img->p, img->q, img->u8p.p, pitch, rows, ctx->s));
    ctx->add(1);
    img->u8p_pitch = pitch;
    img->u8p_rows = rows;
}

// The 16-byte-pitched copy is made at upload (tensor-core kernels, R_co, window statistics
// and the list kernel read it); the FP32 copy only when a CUDA-core band kernel needs it.
void finish_integer_image(tm_ctx* ctx, tm_image* img) {
    img->pitch = ((img->q + 3) & ~3) + 128;  // zero pad: vector loads past the last column
    img->have_f32 = false;
    tc_pitch_copy(ctx, img);
}

void ensure_f32(tm_ctx* ctx, tm_image* img) {
    if (!img->integer || img->have_f32) return;
    img->f32.ensure(size_t(img->p) * img->pitch);
    CK(tmk::u8_to_f32_pitched(img->u8.p, img->p, img->q, img->f32.p, img->pitch, ctx->s));
    ctx->add(1);
    img->have_f32 = true;
}

void ensure_f64(tm_ctx* ctx, tm_image* img) {
    if (img->have_f64) return;
    img->f64.ensure(size_t(img->p) * img->q);
    CK(tmk::u8_to_f64(img->u8.p, size_t(img->p) * img->q, img->f64.p, ctx->s));
    ctx->add(1);
    img->have_f64 = true;
}

// Adopt a device FP64 raster (already in img->f64); classify and derive the u8/f32 views.
void classify_device_image(tm_ctx* ctx, tm_image* img) {
    const size_t N = size_t(img->p) * img->q;
    int* bad = reinterpret_cast<int*>(ctx->counters.p);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), ctx->s));
    CK(tmk::check_u8_domain(img->f64.p, N, bad, ctx->s));
    int hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    ctx->add(1);
    img->have_f64 = true;
    img->integer = hbad == 0;
    if (img->integer) {
        alloc_u8(ctx, img);
        CK(tmk::f64_to_u8(img->f64.p, N, img->u8.p, ctx->s));
        ctx->add(1);
        finish_integer_image(ctx, img);
    }
}

// prefix_noise (stats.cpp:78-81) on the device; returns a device pointer.
const double* image_prefix_noise(tm_ctx* ctx, tm_image* img) {
    if (img->noise_external) return img->pn.p + 1;
    if (!img->have_qtotal) {
        img->pn.ensure(8);
        if (img->integer) {
            if (!img->qt.p) {  // running sum + block counter, kept zero between uses
                img->qt.ensure(2);
                CK(cudaMemsetAsync(img->qt.p, 0, 16, ctx->s));
            }
            CK(tmk::prefix_noise_u8(img->u8.p, img->p, img->q, img->qt.p, img->pn.p + 1, ctx->s));
        } else {
            img->pnpart.ensure(tmk::prefix_noise_f64_parts());
            CK(tmk::prefix_noise_f64(img->f64.p, img->p, img->q, img->pnpart.p, img->pn.p, ctx->s));
        }
        ctx->add(2);
        img->have_qtotal = true;
    }
    return img->pn.p + 1;
}

// Replica prefix over a product source; the full window-sum table lands in `out`.
void replica_sums(tm_ctx* ctx, tmk::ProdSrc src, int rows, int cols, int m, int n, double* out) {
    ctx->rowacc.ensure(size_t(rows) * cols);
    ctx->prefix.ensure(size_t(rows + 1) * (cols + 1));
    CK(tmk::replica_prefix(src, rows, cols, ctx->rowacc.p, ctx->prefix.p, ctx->s));
    CK(tmk::replica_window_diff(ctx->prefix.p, rows, cols, m, n, out, ctx->s));
    ctx->add(3);
}

// window_stats (stats.cpp:55-94) into `ws`.
void compute_ws(tm_ctx* ctx, tm_image* img, int m, int n, WS& ws) {
    const int p = img->p, q = img->q;
    if (m < 1 || n < 1 || m > p || n > q) invalid("running_sum: window does not fit the source");
    const int er = p - m + 1, ec = q - n + 1;
    const size_t E = size_t(er) * ec;
    ws.mu.ensure(E);
    ws.om.ensure(E);
    ws.fl.ensure(E);
    ws.er = er;
    ws.ec = ec;
    ws.m = m;
    ws.n = n;
    const double* prefix_noise = image_prefix_noise(ctx, img);
    Phase ph(ctx, "window_stats");
    if (img->integer && ctx->ws4 && img->u8p.p && img->u8p_rows >= p + tmk::kU8PadRows &&
        tmk::window_stats4_supported(p, q, m, n, img->u8p_pitch)) {
        // four columns per thread from the 16-byte-pitched copy
        CK(tmk::window_stats4_u8(img->u8p.p, img->u8p_pitch, p, q, m, n, prefix_noise, ws.dev(),
                                 ctx->s, img->row_lo, img->row_hi - m + 1));
        ctx->add(1);
    } else if (img->integer) {
        ctx->hs.ensure(size_t(p) * ec);
        ctx->hq.ensure(size_t(p) * ec);
        CK(tmk::window_stats_u8(img->u8.p, p, q, m, n, prefix_noise, ctx->hs.p, ctx->hq.p, ws.dev(),
                                ctx->s));
        ctx->add(2);
    } else {
        ctx->S.ensure(E);
        ctx->Q.ensure(E);
        // S (pixels) and Q (squares): two independent prefix problems in one batch
        tmk::ProdBatch bt{};
        bt.n = 2;
        bt.slot = size_t(p) * q;
        bt.pslot = size_t(p + 1) * (q + 1);
        bt.src[0] = tmk::ProdSrc{img->f64.p, q, 0, 0, nullptr, 0, 0, 0, 0};
        bt.src[1] = tmk::ProdSrc{img->f64.p, q, 0, 0, nullptr, 0, 0, 0, 1};
        bt.rows[0] = bt.rows[1] = p;
        bt.cols[0] = bt.cols[1] = q;
        ctx->rowacc.ensure(2 * bt.slot);
        ctx->prefix.ensure(2 * bt.pslot);
        CK(tmk::replica_prefix_batch(bt, ctx->rowacc.p, ctx->prefix.p, ctx->s));
        CK(tmk::replica_window_diff(ctx->prefix.p, p, q, m, n, ctx->S.p, ctx->s));
        CK(tmk::replica_window_diff(ctx->prefix.p + bt.pslot, p, q, m, n, ctx->Q.p, ctx->s));
        ctx->add(4);
        // the flat floor against the bracket of the reference's sequential q_total;
        // undecided windows trigger the sequential replay and a redo (k_stats.cu)
        CK(tmk::stats_from_sums(ctx->S.p, ctx->Q.p, E, m, n, img->f64.p, p, q, img->pn.p,
                                ws.dev(), ctx->s));
        ctx->add(4);
    }
}

// The image's pixels changed: its cached window statistics are stale (kept allocated and
// recomputed in place by the next get_ws).
void invalidate_ws(tm_image* img) {
    for (auto& kv : img->ws_cache) kv.second->valid = false;
    img->have_split = false;
}

WS& get_ws(tm_ctx* ctx, tm_image* img, int m, int n) {
    auto key = std::make_pair(m, n);
    auto it = img->ws_cache.find(key);
    if (it != img->ws_cache.end()) {
        if (!it->second->valid) {  // stale (new pixels): recompute, no buffer churn
            compute_ws(ctx, img, m, n, *it->second);
            it->second->valid = true;
        }
        return *it->second;
    }
    auto ws = std::make_unique<WS>();
    compute_ws(ctx, img, m, n, *ws);
    ws->valid = true;
    WS& ref = *ws;
    img->ws_cache[key] = std::move(ws);
    return ref;
}

// Survivor tile flags for an extent (zeroed on the stream): scan 2 marks the blocks holding
// survivors, the masked dense pass skips the rest.
tmk::TileFlags zero_tile_flags(tm_ctx* ctx, DBuf<uint8_t>& buf, int er, int ec, int count = 1) {
    const size_t bytes = tmk::tile_flag_bytes(er, ec);
    buf.ensure(bytes * count);
    CK(cudaMemsetAsync(buf.p, 0, bytes * count, ctx->s));
    return tmk::TileFlags{buf.p, (ec + 2047) >> 11};
}

// ---- templates ---------------------------------------------------------------------------

// template_stats (stats.cpp:98-111) in reference order (host), no upload.
Tmpl template_host_stats(const double* t, int m, int n) {
    Tmpl T;
    T.m = m;
    T.n = n;
    T.npad = (n + 15) & ~15;
    double sum = 0.0, sq = 0.0;
    bool integer = true;
    for (size_t i = 0; i < size_t(m) * n; ++i) {
        sum += t[i];
        sq += t[i] * t[i];
        if (!(t[i] >= 0.0 && t[i] <= 255.0) || t[i] != std::rint(t[i])) integer = false;
    }
    const long long mn = (long long)m * n;
    const double var_sum = sq - sum * sum / double(mn);
    T.ts.mu = sum / double(mn);
    T.ts.omega = std::sqrt(std::max(0.0, var_sum));
    T.ts.flat = variance_is_flat_h(var_sum, sq, mn);
    T.ts.mn = double(m) * double(n);
    T.integer = integer;
    T.flush_rows = int(16777216LL / (65025LL * n));
    return T;
}

// template_stats, then upload to the context's template buffers.
Tmpl upload_template(tm_ctx* ctx, const double* t, int m, int n, bool side = false) {
    Tmpl T = template_host_stats(t, m, n);
    // the device copy already holds this template (same bytes as the last upload): no copy
    // (a stream of searches with one template uploads it once)
    const size_t mnz = size_t(m) * n;
    if (ctx->tmpl_m == m && ctx->tmpl_n == n && ctx->tmpl_last.size() == mnz && ctx->tf.p &&
        ctx->td.p && std::memcmp(ctx->tmpl_last.data(), t, mnz * sizeof(double)) == 0) {
        T.tf = ctx->tf.p;
        T.td = ctx->td.p;
        return T;
    }
    ctx->tmpl_m = ctx->tmpl_n = 0;  // (re-set below once the copies are enqueued)
    std::vector<float> tf(size_t(m) * T.npad, 0.f);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) tf[size_t(i) * T.npad + j] = float(t[size_t(i) * n + j]);
    // side stream only when the device buffers already exist (a fresh stream-ordered
    // allocation on ctx->s must not be touched from another stream)
    side = side && ctx->tf.p && ctx->tf.cap >= tf.size() && ctx->td.p &&
           ctx->td.cap >= size_t(m) * n;
    ctx->tf.ensure(tf.size());
    ctx->td.ensure(size_t(m) * n);
    cudaStream_t us = side ? ctx->s2 : ctx->s;
    ctx->pin_tf.upload(ctx->tf.p, tf.data(), tf.size() * 4, us);
    ctx->pin_td.upload(ctx->td.p, t, size_t(m) * n * 8, us);
    if (side) {  // the main stream waits for the copies before any later work
        CK(cudaEventRecord(ctx->ev_t, ctx->s2));
        CK(cudaStreamWaitEvent(ctx->s, ctx->ev_t, 0));
    }
    ctx->tmpl_last.assign(t, t + mnz);
    ctx->tmpl_m = m;
    ctx->tmpl_n = n;
    T.tf = ctx->tf.p;
    T.td = ctx->td.p;
    return T;
}

bool fp32_path(const tm_image* img, const Tmpl& T) {
    return img->integer && T.integer && T.flush_rows >= 1;
}

tmk::CorrJob make_job(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T) {
    tmk::CorrJob j{};
    const bool fp32 = fp32_path(img, T);
    if (!fp32) ensure_f64(ctx, img);
    j.imgf = img->f32.p;
    j.pitch = img->pitch;
    j.imgb = img->u8p.p;
    j.bpitch = img->u8p_pitch;
    j.imgd = img->f64.p;
    j.q = img->q;
    j.tf = T.tf;
    j.npad = T.npad;
    j.td = T.td;
    j.m = T.m;
    j.n = T.n;
    j.flush_rows = std::max(1, T.flush_rows);
    j.ts = T.ts;
    j.st = ws.dev();
    return j;
}

// A job for the CUDA-core band kernel (corr_band), which reads the FP32 copy (made on demand).
tmk::CorrJob band_job(tm_ctx* ctx, tm_image* img, tmk::CorrJob j) {
    ensure_f32(ctx, img);
    j.imgf = img->f32.p;
    j.pitch = img->pitch;
    return j;
}

int nw_for(int sw) { return sw == 1 ? 4 : (sw == 3 ? 2 : 1); }

int band_partials(int nrows, int nc, int sw) {
    const int nw = nw_for(sw);
    return ((nc + nw * 32 - 1) / (nw * 32)) * ((nrows + 7) / 8);
}

int row_span(const std::vector<int>& rows) {
    int span = 0;
    for (size_t yb = 0; yb < rows.size(); yb += 8) {
        const size_t yl = std::min(rows.size() - 1, yb + 7);
        span = std::max(span, rows[yl] - rows[yb]);
    }
    return span;
}


// ---- integer tensor-core path (k_tc.cu) -------------------------------------------------
constexpr size_t kTcSmemBudget = 224 * 1024;  // 227 KB opt-in minus static shared memory

bool tc_path(tm_ctx* ctx, const tm_image* img, const Tmpl& T) {
    return ctx->tc && fp32_path(img, T) && tmk::tc_supported(T.m, T.n) &&
           tmk::tc_plan(T.m, T.n, 1, kTcSmemBudget).nch > 0;
}

const uint8_t* tc_image(tm_ctx* ctx, tm_image* img, int ec) {
    if (img->u8p_pitch < tmk::tc_pitch(img->q, ec)) tc_pitch_copy(ctx, img);
    return img->u8p.p;
}

// Error model of the split planes (k_tc.cu): the truncation is < 2^-16 per pixel, i.e.
// < 2^-16 * sum(T) per dot; the reference's sequential FP64 sum of m*n non-negative products
// (detail.hpp:32-41) is within gamma_{mn} of the true dot (twice the textbook bound here).
tmk::SplitModel split_model(const Tmpl& T) {
    return tmk::SplitModel{T.ts.mn * T.ts.mu * (1.0 + 1e-9) / 65536.0,
                           (T.ts.mn + 4.0) * 2.220446049250313e-16};
}

// Non-integer image + integer template: the byte planes for the split tensor-core
// screening, made on first use.  False when a pixel lies outside [0, 256) (FP64 replica).
// work = multiply-adds of the pass, min_work = the size below which the FP64 replica is as
// fast (measured: brute force crosses over near 256^2 x 32^2, scan 1 near 5,000 centres of
// 32^2; tools/tiny_split_probe.py).
bool split_path(tm_ctx* ctx, tm_image* img, const Tmpl& T, double work, double min_work) {
    if (!ctx->tc || ctx->tc_split <= 0 || img->integer || !T.integer || T.ts.flat) return false;
    if (ctx->tc_split == 1 && work < min_work) return false;
    if (img->row_lo != 0 || img->row_hi < img->p) return false;  // strip images: 8-bit only
    if (!tmk::tc_supported(T.m, T.n) || tmk::tc_plan(T.m, T.n, 1, kTcSmemBudget).nch == 0)
        return false;
    if (!img->have_split) {
        const int pitch = tmk::tc_pitch(img->q, img->q);
        const int rows = img->p + tmk::kU8PadRows;
        img->split_stride = size_t(rows) * pitch;
        img->split.ensure(img->split_stride * tmk::kTcSplitPlanes);
        int* bad = reinterpret_cast<int*>(ctx->counters.p + 34);
        CK(cudaMemsetAsync(bad, 0, sizeof(int), ctx->s));
        CK(tmk::tc_split_image(img->f64.p, img->p, img->q, img->split.p, pitch, rows,
                               img->split_stride, bad, ctx->s));
        ctx->add(1);
        int hbad = 0;
        CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        img->split_pitch = pitch;
        img->have_split = true;
        img->split_ok = hbad == 0;
    }
    return img->split_ok;
}

// Bands of up to `rmax` output rows r0 + sr*k; a list of rows with irregular spacing
// becomes single-row bands.
std::vector<tmk::TcBand> tc_bands(const std::vector<int>& rows, const std::vector<int>& yi, int sr,
                                  int rmax) {
    std::vector<tmk::TcBand> out;
    size_t i = 0;
    while (i < rows.size()) {
        size_t j = i + 1;
        while (j < rows.size() && int(j - i) < rmax && rows[j] - rows[j - 1] == sr &&
               yi[j] - yi[j - 1] == 1)
            ++j;
        const int cnt = int(j - i);
        out.push_back(tmk::TcBand{rows[i], cnt > 1 ? sr : 1, cnt, yi[i]});
        i = j;
    }
    return out;
}

// Runs the tensor-core kernel over `rows` (group-row indices `yi`) -> partials, returns #.
// Output rows of a tensor-core launch, described without materialising them (the host
// only builds the vectors when the geometry is not cached yet).
struct RowSet {
    int kind = 0;  // 0: extent rows [lo, hi); 1: centre rows of group rows [lo, hi) of g
    int lo = 0, hi = 0;
    tmk::GridDesc g{};
    void materialise(std::vector<int>& rows, std::vector<int>& yi) const {
        rows.clear();
        yi.clear();
        for (int i = lo; i < hi; ++i) {
            rows.push_back(kind == 0 ? i : centre_row_h(g, i));
            yi.push_back(i);
        }
    }
};

TcGeo& tc_geometry(tm_ctx* ctx, const WS& ws, const Tmpl& T, const RowSet& rs, int sr,
                   int band_rows = 16) {
    const std::vector<long long> key = {T.m, T.n, sr, ws.ec, rs.kind, rs.lo, rs.hi,
                                        rs.kind ? rs.g.er : 0, rs.kind ? rs.g.h : 0, band_rows};
    auto it = ctx->tc_geo.find(key);
    if (it != ctx->tc_geo.end()) return *it->second;
    if (ctx->tc_geo.size() > 64) ctx->tc_geo.clear();
    std::vector<int> rows, yi;
    rs.materialise(rows, yi);
    auto geo = std::make_unique<TcGeo>();
    geo->plan = tmk::tc_plan(T.m, T.n, sr, kTcSmemBudget);
    if (geo->plan.nch == 0) invalid("tensor-core plan unavailable");
    geo->ntc = (ws.ec + tmk::tc_tile_cols() - 1) / tmk::tc_tile_cols();
    // rows per band: the fewest waves of 148 persistent CTAs with <= 16 rows per band, then
    // bands as equal as possible so every CTA gets the same number of tiles
    const size_t work = rows.size() * size_t(geo->ntc);
    const size_t br = size_t(band_rows);
    const size_t waves = std::max<size_t>(1, (work + 148 * br - 1) / (148 * br));
    int rmax = int(std::min<size_t>(br, std::max<size_t>(1, (work + 148 * waves - 1) / (148 * waves))));
    const std::vector<tmk::TcBand> bands = tc_bands(rows, yi, sr, rmax);
    geo->nbands = int(bands.size());
    geo->bands.ensure(bands.size());
    CK(cudaMemcpyAsync(geo->bands.p, bands.data(), bands.size() * sizeof(tmk::TcBand),
                       cudaMemcpyHostToDevice, ctx->s));
    const std::vector<int> sched = tmk::tc_schedule(geo->plan, rmax, geo->sched_off, geo->sched_len);
    geo->sched_total = int(sched.size() / 4);
    geo->sched.ensure(sched.size() / 4 + 1);
    CK(cudaMemcpyAsync(geo->sched.p, sched.data(), sched.size() * sizeof(int),
                       cudaMemcpyHostToDevice, ctx->s));
    geo->rows.ensure(rows.size() + 1);
    CK(cudaMemcpyAsync(geo->rows.p, rows.data(), rows.size() * sizeof(int), cudaMemcpyHostToDevice,
                       ctx->s));
    CK(cudaStreamSynchronize(ctx->s));  // host vectors go out of scope (pageable copies)
    TcGeo& ref = *geo;
    ctx->tc_geo.emplace(key, std::move(geo));
    return ref;
}

// Runs the tensor-core kernel over `rows` (group-row indices `yi`) -> partials, returns #.
int tc_run(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T, const RowSet& rs, int sr,
           tmk::TcTask task, const int** rows_dev = nullptr, bool side_build = false) {
    const bool split = task.mode >= 3;
    TcGeo& geo = tc_geometry(ctx, ws, T, rs, sr, split ? tmk::kTcSplitRows : 16);
    HT("tc_geo");
    const tmk::TcPlan& plan = geo.plan;
    if (side_build && ctx->tc_b.cap >= plan.total_bytes) {
        // speculative centre scan: B built on the side stream while the EGS batch runs
        // (ungated: the gate is decided later; a miss rebuilds B on the main stream)
        CK(cudaStreamWaitEvent(ctx->s2, ctx->ev_b0, 0));
        CK(tmk::tc_build_b(T.tf, T.npad, T.m, T.n, plan, ctx->tc_b.p, ctx->s2));
        CK(cudaEventRecord(ctx->ev_b1, ctx->s2));
        CK(cudaStreamWaitEvent(ctx->s, ctx->ev_b1, 0));
    } else {
        ctx->tc_b.ensure(plan.total_bytes);
        CK(tmk::tc_build_b(T.tf, T.npad, T.m, T.n, plan, ctx->tc_b.p, ctx->s, task.gate));
    }
    HT("build_b");
    tmk::TcJob job{};
    if (split) {
        // error model of the split (k_tc.cu): truncation < 2^-16 per pixel, times sum(T);
        // the reference's sequential FP64 sum is within gamma_mn of the true dot
        job.imgp = img->split.p;
        job.pitch = img->split_pitch;
        job.plane_stride = img->split_stride;
        const tmk::SplitModel sm = split_model(T);
        job.scr_delta = sm.delta;
        job.scr_gamma = sm.gamma;
        task.kp = tmk::kTcSplitRows;
    } else {
        job.imgp = tc_image(ctx, img, ws.ec);
        job.pitch = img->u8p_pitch;
    }
    job.bglob = ctx->tc_b.p;
    job.plan = plan;
    job.ts = T.ts;
    job.st = ws.dev();
    task.bands = geo.bands.p;
    task.nbands = geo.nbands;
    task.ntc = geo.ntc;
    task.sched = geo.sched.p;
    task.sched_total = geo.sched_total;
    for (int c = 0; c < tmk::kTcMaxChunks; ++c) {
        task.sched_off[c] = geo.sched_off[c];
        task.sched_len[c] = geo.sched_len[c];
    }
    if (rows_dev) *rows_dev = geo.rows.p;
    int np = 0;  // caller sizes ctx->partials for >= 148 entries
    static const bool dbg = std::getenv("TMATCH_TC_DEBUG") != nullptr;
    DBuf<long long> dbuf;
    if (dbg) {
        dbuf.ensure(148 * 8);
        CK(cudaMemsetAsync(dbuf.p, 0, 148 * 8 * 8, ctx->s));
        task.dbg = dbuf.p;
        task.dbg_flags = std::atoi(std::getenv("TMATCH_TC_DEBUG"));
    }
    CK(tmk::tc_corr(job, task, ctx->partials.p, &np, ctx->s));
    HT("tc_corr");
    ctx->add(2);
    if (dbg) {
        std::vector<long long> h(148 * 8);
        CK(cudaMemcpyAsync(h.data(), dbuf.p, h.size() * 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        double a[8] = {};
        for (int b = 0; b < np; ++b)
            for (int j = 0; j < 8; ++j) a[j] += double(h[b * 8 + j]) / np;
        std::fprintf(stderr,
                     "[tc] ctas=%d bands=%d ntc=%d rows/cta=%.0f | producer total=%.0f wait_empty=%.0f "
                     "wait_bempty=%.0f | mma total=%.0f wait_full=%.0f wait_dempty=%.0f wait_bfull=%.0f\n",
                     np, task.nbands, task.ntc, a[3], a[0], a[1], a[2], a[4], a[5], a[6], a[7]);
    }
    return np;
}

void upload_rows(tm_ctx* ctx, const std::vector<int>& rows) {
    ctx->rows_list.ensure(rows.size());
    ctx->pin_rows.upload(ctx->rows_list.p, rows.data(), rows.size() * 4, ctx->s);
}

constexpr int kListBlocks = 148 * 4;

// Reduce `n` partial cells to ctx->cells[slot].
void reduce_to(tm_ctx* ctx, int n, int slot, const tmk::ReduceOp* op = nullptr) {
    // n = 0 writes the empty cell (the kernel's loop does not run)
    CK(tmk::reduce_cells(ctx->partials.p, std::max(n, 0), ctx->cells.p + slot, ctx->s, op));
    ctx->add(1);
}

// Scan 1's reduction op: the threshold bootstrap (matcher.cpp:121-125) plus the zeroing of
// the seeding counters and the scan-2 tally.
tmk::ReduceOp centre_op(tm_ctx* ctx, const tm_match_params& P) {
    tmk::ReduceOp op{};
    op.kind = 1;
    op.has_init = P.has_init_threshold;
    op.init = P.init_threshold;
    op.thr = ctx->thr.p;
    op.zero64 = ctx->counters.p + 4;
    op.nzero64 = 2;
    op.zero_tally = ctx->tally.p;
    return op;
}

// The same reduction fused into the tail of the kernel that writes the phase's last
// partials (partials[0, n) -> cells[slot], then op).
tmk::TailReduce tail_to(tm_ctx* ctx, int n, int slot, const tmk::ReduceOp* op = nullptr) {
    tmk::TailReduce t;
    t.partials = ctx->partials.p;
    t.n = n;
    t.out = ctx->cells.p + slot;
    t.ticket = reinterpret_cast<unsigned*>(ctx->counters.p + 26);
    if (op) t.op = *op;
    return t;
}

// Evaluate a device location list (count on device) -> cells[slot].
void eval_list(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T, const int2* locs,
               const unsigned long long* count, int max_count, double* out_rho,
               uint8_t* out_deg, int slot, const tmk::ReduceOp* op = nullptr) {
    const tmk::CorrJob job = make_job(ctx, img, ws, T);
    ctx->partials.ensure(kListBlocks);
    Phase ph(ctx, slot == 1 ? "seed_eval" : (slot == 2 ? "survivor_eval" : "list_eval"));
    if (fp32_path(img, T)) {  // reduction fused into the list kernel's tail
        const tmk::TailReduce tail = tail_to(ctx, kListBlocks, slot, op);
        CK(tmk::corr_list(job, locs, count, max_count, out_rho, out_deg, ctx->partials.p,
                          kListBlocks, ctx->s, 0, &tail));
        ctx->add(1);
        return;
    }
    CK(tmk::corr_list_f64(job, locs, count, max_count, out_rho, out_deg, ctx->partials.p,
                          kListBlocks, ctx->s));
    ctx->add(1);
    reduce_to(ctx, kListBlocks, slot, op);
}

// ---- scan 1: every group centre (matcher.cpp:23-37) -> rho_c, deg_c, cells[0] --------
// side_b: B is built on the side stream (tc_b pre-sized and ev_b0 recorded by the caller)
void centre_scan(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T,
                 const tmk::GridDesc& g, const tmk::ReduceOp* op = nullptr,
                 bool side_b = false) {
    const size_t G = size_t(g.tr) * g.tc;
    ctx->sa_ready = false;  // set below only by the epilogues that write sa_c
    ctx->rho_c.ensure(G);
    ctx->deg_c.ensure(G);
    const tmk::CorrJob job = make_job(ctx, img, ws, T);
    const int wr = g.w / 2;
    Phase ph(ctx, "centre_scan");
    if (tc_path(ctx, img, T) && g.h <= tmk::kTcMaxClasses) {
        const int nstrip = g.ti_hi - g.ti_lo;
        if (nstrip <= 0) {
            reduce_to(ctx, 0, 0, op);
            return;
        }
        RowSet rs;
        rs.kind = 1;
        rs.lo = g.ti_lo;
        rs.hi = g.ti_hi;
        rs.g = g;
        const bool clipped = size_t(g.tc) * g.w > size_t(g.ec);
        const int nc_reg = clipped ? g.tc - 1 : g.tc;
        int n1 = 0, n2 = 0;
        // partials: <= 148 from the tensor-core kernel + the clipped column's list blocks
        // (sized once: a later ensure() could reallocate under pending writes)
        ctx->partials.ensure(size_t(148 + kListBlocks) + 1);
        {
            // exact centre dots on the tensor cores -> dotbuf (the clipped last group
            // column included, at tj = tc-1), then the FP64 epilogue
            ctx->dotbuf.ensure(G);
            tmk::TcTask task{};
            task.mode = 1;
            task.cbase = wr;
            task.cstep = g.w;
            task.nc = nc_reg;
            task.tc = g.tc;
            task.c_last = clipped ? centre_col_h(g, g.tc - 1) : -1;
            task.out_rho = ctx->dotbuf.p;
            const int* rows_dev = nullptr;
            // already enqueued behind the EGS batch (tm_search) and confirmed by the device
            // decision for this grid: the dots are in flight, skip the launches
            const auto& sp = ctx->spec;
            const bool hit = sp.armed && sp.g.er == g.er && sp.g.ec == g.ec && sp.g.h == g.h &&
                             sp.g.w == g.w && sp.g.ti_lo == g.ti_lo && sp.g.ti_hi == g.ti_hi &&
                             ctx->hres->spec == 1;
            ctx->spec.armed = false;
            ctx->sa_c.ensure(G);
            ctx->sa_ready = true;  // both epilogues below write scan 2's half-gap factors
            if (hit) return;  // dots, epilogue and its reduction are already in flight
            tc_run(ctx, img, ws, T, rs, g.h, task, &rows_dev, side_b);
            n1 = std::min(kListBlocks, int((size_t(nstrip) * g.tc + 255) / 256));
            const tmk::TailReduce tail = tail_to(ctx, n1 + n2, 0, op);  // n2 = 0 here
            const tmk::CentreStats cs{ctx->cs_mu.p, ctx->cs_om.p, ctx->cs_fl.p};
            CK(tmk::centre_epilogue(job, g, rows_dev, wr, g.w, g.tc, 0, ctx->dotbuf.p,
                                    ctx->rho_c.p, ctx->deg_c.p, ctx->partials.p, n1, ctx->s,
                                    task.c_last, &tail, nullptr, ctx->sa_c.p, ctx->batch_rec,
                                    ctx->batch_cs ? &cs : nullptr));
            HT("centre_epi");
            ctx->add(1);
        }
        return;
    }
    if (fp32_path(img, T) && (g.w == 1 || g.w == 3 || g.w == 5 || g.w == 7)) {
        const int nstrip = g.ti_hi - g.ti_lo;
        if (nstrip <= 0) {
            reduce_to(ctx, 0, 0, op);
            return;
        }
        std::vector<int> rows(nstrip);
        for (int ti = g.ti_lo; ti < g.ti_hi; ++ti) rows[ti - g.ti_lo] = centre_row_h(g, ti);
        upload_rows(ctx, rows);
        const bool clipped = size_t(g.tc) * g.w > size_t(g.ec);
        const int nc_reg = clipped ? g.tc - 1 : g.tc;
        const int np_main = nc_reg > 0 ? band_partials(nstrip, nc_reg, g.w) : 0;
        const int np_last = clipped ? band_partials(nstrip, 1, 1) : 0;
        // sized once for every writer below (a later ensure() could reallocate under
        // pending writes): the band or K-split epilogue partials + the clipped column
        ctx->partials.ensure(size_t(std::max(np_main, kListBlocks) + np_last) + 1);
        int n1 = 0, n2 = 0;
        tmk::BandTask t{};
        t.rows = ctx->rows_list.p;
        t.nrows = nstrip;
        t.yi_base = g.ti_lo;
        t.mode = 1;
        t.row_span = row_span(rows);
        t.ksplit = 1;
        t.ms = T.m;
        t.tc = g.tc;
        t.out_rho = ctx->rho_c.p;
        t.out_deg = ctx->deg_c.p;
        if (nc_reg > 0) {
            t.cbase = wr;
            t.sw = g.w;
            t.nc = nc_reg;
            t.col0 = 0;
            // split the template rows across CTAs until the grid covers ~3 waves
            const int tiles = band_partials(nstrip, nc_reg, g.w);
            int ks = std::max(1, std::min(8, (148 * 6 * 3) / std::max(1, tiles)));
            ks = std::min(ks, std::max(1, T.m / 8));
            if (ks > 1) {
                t.ksplit = ks;
                t.ms = ((T.m + ks - 1) / ks + 7) & ~7;
                t.ksplit = (T.m + t.ms - 1) / t.ms;
                ctx->dotbuf.ensure(G);
                CK(cudaMemsetAsync(ctx->dotbuf.p, 0, G * sizeof(double), ctx->s));
                t.dot = ctx->dotbuf.p;
                int dummy = 0;
                CK(tmk::corr_band(band_job(ctx, img, job), t, ctx->partials.p, &dummy, ctx->s));
                n1 = std::min(kListBlocks, int((size_t(nstrip) * nc_reg + 255) / 256));
                CK(tmk::centre_epilogue(job, g, ctx->rows_list.p, wr, g.w, nc_reg, 0, ctx->dotbuf.p,
                                        ctx->rho_c.p, ctx->deg_c.p, ctx->partials.p, n1, ctx->s));
                ctx->add(2);
                t.ksplit = 1;
                t.ms = T.m;
                t.dot = nullptr;
            } else {
                t.ksplit = 1;
                t.ms = T.m;
                CK(tmk::corr_band(band_job(ctx, img, job), t, ctx->partials.p, &n1, ctx->s));
                ctx->add(1);
            }
        }
        if (clipped) {
            // the clipped last group column: one centre per group row, list kernel
            std::vector<int2> last(nstrip);
            const int cc = centre_col_h(g, g.tc - 1);
            for (int i = 0; i < nstrip; ++i) last[i] = make_int2(rows[i], cc);
            ctx->seed_locs.ensure(size_t(nstrip));
            ctx->pin_locs.upload(ctx->seed_locs.p, last.data(), last.size() * sizeof(int2), ctx->s);
            const unsigned long long cnt = nstrip;
            ctx->pin_cnt.upload(ctx->counters.p + 12, &cnt, 8, ctx->s);
            ctx->seq_rho.ensure(size_t(nstrip));
            ctx->seq_deg.ensure(size_t(nstrip));
            n2 = std::min(kListBlocks, (nstrip + 7) / 8);
            CK(tmk::corr_list(job, ctx->seed_locs.p, ctx->counters.p + 12, nstrip, ctx->seq_rho.p,
                              ctx->seq_deg.p, ctx->partials.p + n1, n2, ctx->s));
            const size_t off = size_t(g.ti_lo) * g.tc;
            CK(tmk::scatter_column(ctx->seq_rho.p, ctx->seq_deg.p, nstrip, g.tc, g.tc - 1,
                                   ctx->rho_c.p + off, ctx->deg_c.p + off, ctx->s));
            ctx->add(2);
        }
        reduce_to(ctx, n1 + n2, 0, op);
        return;
    }
    // general path: explicit centre list in grid order
    const size_t off = size_t(g.ti_lo) * g.tc;
    const size_t GS = size_t(g.ti_hi - g.ti_lo) * g.tc;
    std::vector<int2> locs(GS);
    for (int ti = g.ti_lo; ti < g.ti_hi; ++ti)
        for (int tj = 0; tj < g.tc; ++tj)
            locs[size_t(ti - g.ti_lo) * g.tc + tj] =
                make_int2(centre_row_h(g, ti), centre_col_h(g, tj));
    if (GS == 0) {
        reduce_to(ctx, 0, 0, op);
        return;
    }
    ctx->seed_locs.ensure(GS);
    ctx->pin_locs.upload(ctx->seed_locs.p, locs.data(), GS * sizeof(int2), ctx->s);
    unsigned long long cnt = GS;
    CK(cudaMemcpyAsync(ctx->counters.p + 4, &cnt, 8, cudaMemcpyHostToDevice, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    eval_list(ctx, img, ws, T, ctx->seed_locs.p, ctx->counters.p + 4, int(GS), ctx->rho_c.p + off,
              ctx->deg_c.p + off, 0, op);
}

// ---- scan 1 on a non-integer image through the split planes ---------------------------
// Every decision that reads rho_c (best centre, seeding, members' bound tests) is either
// settled by the centre's bracket or the centre is re-evaluated by the FP64 replica first,
// so counts, visit codes and results equal the all-exact path's.  Sequential policy: the
// running threshold only rises from scan 1's, so members certainly eliminated at it stay
// eliminated; every other member's group gets its exact rho_c (the replay re-tests them).
bool split_centres_ok(tm_ctx* ctx, tm_image* img, const Tmpl& T, const tmk::GridDesc& g) {
    const double work = double(g.tr) * g.tc * T.m * T.n;
    return g.h <= tmk::kTcMaxClasses && g.ti_lo == 0 && g.ti_hi == g.tr &&
           split_path(ctx, img, T, work, 2097152.0) &&
           tmk::tc_plan(T.m, T.n, g.h, kTcSmemBudget).nch > 0;
}

// The centres listed in split_locs / split_gidx (count on the device) -> exact rho by the
// FP64 replica, scattered into rho_c (radius 0); their best -> cells[slot] (+ op).
void split_exact(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T, size_t G,
                 unsigned long long* cnt, int slot, const tmk::ReduceOp* op = nullptr) {
    eval_list(ctx, img, ws, T, ctx->split_locs.p, cnt, int(std::min<size_t>(G, INT_MAX)),
              ctx->split_rho.p, nullptr, slot, op);
    CK(tmk::split_scatter(ctx->split_rho.p, ctx->split_gidx.p, cnt, ctx->rho_c.p, ctx->rad_c.p,
                          ctx->s));
    ctx->add(1);
}

void centre_scan_split(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T,
                       const tmk::GridDesc& g, const tmk::ReduceOp* op) {
    const size_t G = size_t(g.tr) * g.tc;
    ctx->sa_ready = false;
    ctx->rho_c.ensure(G);
    ctx->deg_c.ensure(G);
    ctx->rad_c.ensure(G);
    ctx->dotbuf.ensure(G);
    ctx->split_rho.ensure(G);
    ctx->split_locs.ensure(G);
    ctx->split_gidx.ensure(G);
    ctx->partials.ensure(size_t(148 + kListBlocks) + 1);
    unsigned long long* cnt = ctx->counters.p + 35;
    {
        Phase ph(ctx, "centre_scan");
        RowSet rs;
        rs.kind = 1;
        rs.lo = 0;
        rs.hi = g.tr;
        rs.g = g;
        const bool clipped = size_t(g.tc) * g.w > size_t(g.ec);
        tmk::TcTask task{};
        task.mode = 4;
        task.cbase = g.w / 2;
        task.cstep = g.w;
        task.nc = clipped ? g.tc - 1 : g.tc;
        task.tc = g.tc;
        task.c_last = clipped ? centre_col_h(g, g.tc - 1) : -1;
        task.out_rho = ctx->dotbuf.p;
        tc_run(ctx, img, ws, T, rs, g.h, task);
        const int n1 = int(std::min<size_t>(kListBlocks, (G + 255) / 256));
        CK(tmk::split_centre_epilogue(g, ctx->dotbuf.p, ws.dev(), T.ts, split_model(T),
                                      ctx->rho_c.p, ctx->rad_c.p, ctx->deg_c.p, ctx->partials.p,
                                      n1, ctx->s));
        ctx->add(1);
        reduce_to(ctx, n1, 3);  // cells[3]: the largest lower bound
        CK(cudaMemsetAsync(cnt, 0, 8, ctx->s));
        CK(tmk::split_pick(g, ctx->rho_c.p, ctx->rad_c.p, ctx->deg_c.p, 0, ctx->cells.p + 3,
                           ctx->thr.p, 0.0, ctx->split_locs.p, ctx->split_gidx.p, cnt, ctx->s));
        ctx->add(1);
    }
    ctx->split_centres += (long long)G;
    split_exact(ctx, img, ws, T, G, cnt, 0, op);  // exact best centre -> cells[0], threshold
}

// Seeded policy: centres whose seeding decision (rho_c >= thr - margin, k_seed_members) the
// bracket leaves open get their exact rho first.
void split_refine_seeding(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T,
                          const tmk::GridDesc& g, double margin) {
    const size_t G = size_t(g.tr) * g.tc;
    unsigned long long* cnt = ctx->counters.p + 35;
    CK(cudaMemsetAsync(cnt, 0, 8, ctx->s));
    CK(tmk::split_pick(g, ctx->rho_c.p, ctx->rad_c.p, ctx->deg_c.p, 1, ctx->cells.p + 3,
                       ctx->thr.p, margin, ctx->split_locs.p, ctx->split_gidx.p, cnt, ctx->s));
    ctx->add(1);
    split_exact(ctx, img, ws, T, G, cnt, 3);
}

// Scan 2: groups with a member whose bound test the centre's bracket leaves open.
void split_refine_bounds(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T,
                         const tmk::GridDesc& g, const double* map, const uint8_t* seeded,
                         bool moving) {
    const size_t G = size_t(g.tr) * g.tc;
    unsigned long long* cnt = ctx->counters.p + 35;
    const size_t fl = (G + 3) & ~size_t(3);
    ctx->split_flag.ensure(fl);
    CK(cudaMemsetAsync(ctx->split_flag.p, 0, fl, ctx->s));
    CK(cudaMemsetAsync(cnt, 0, 8, ctx->s));
    {
        Phase ph(ctx, "split_bounds");
        CK(tmk::split_sec_uncertain(g, map, ctx->rho_c.p, ctx->rad_c.p, ctx->deg_c.p, ws.fl.p,
                                    ctx->thr.p, seeded, ctx->split_flag.p, ctx->split_locs.p,
                                    ctx->split_gidx.p, cnt, ctx->s, moving ? 1 : 0));
        ctx->add(1);
    }
    split_exact(ctx, img, ws, T, G, cnt, 3);
}

// Speculative centre scan for tm_search: the B build and the tensor-core centre dots for a
// predicted group size, enqueued behind an EGS batch and gated on the device decision
// (k_egs_decide: EGS finished with h_e == predicted).  On a wrong prediction both kernels
// exit at entry and centre_scan launches the real ones.
void spec_centre(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T, const tmk::GridDesc& g,
                 const tm_match_params& P) {
    ctx->spec.armed = false;
    if (!(tc_path(ctx, img, T) && g.h <= tmk::kTcMaxClasses) || g.ti_hi <= g.ti_lo) return;
    const size_t G = size_t(g.tr) * g.tc;
    ctx->rho_c.ensure(G);
    ctx->deg_c.ensure(G);
    ctx->partials.ensure(size_t(148 + kListBlocks) + 1);
    ctx->dotbuf.ensure(G);
    RowSet rs;
    rs.kind = 1;
    rs.lo = g.ti_lo;
    rs.hi = g.ti_hi;
    rs.g = g;
    const bool clipped = size_t(g.tc) * g.w > size_t(g.ec);
    tmk::TcTask task{};
    task.mode = 1;
    task.cbase = g.w / 2;
    task.cstep = g.w;
    task.nc = clipped ? g.tc - 1 : g.tc;
    task.tc = g.tc;
    task.c_last = clipped ? centre_col_h(g, g.tc - 1) : -1;
    task.out_rho = ctx->dotbuf.p;
    task.gate = reinterpret_cast<const int*>(ctx->counters.p + 24);
    const int* rows_dev = nullptr;
    Phase ph(ctx, "centre_scan");
    tc_run(ctx, img, ws, T, rs, g.h, task, &rows_dev, /*side_build=*/ctx->spec_b);
    // the epilogue + scan 1's reduction (the same op search() would use), same gate
    const int n1 = std::min(kListBlocks, int((size_t(g.ti_hi - g.ti_lo) * g.tc + 255) / 256));
    const tmk::ReduceOp op = centre_op(ctx, P);
    const tmk::TailReduce tail = tail_to(ctx, n1, 0, &op);
    ctx->sa_c.ensure(G);
    CK(tmk::centre_epilogue(make_job(ctx, img, ws, T), g, rows_dev, g.w / 2, g.w, g.tc, 0,
                            ctx->dotbuf.p, ctx->rho_c.p, ctx->deg_c.p, ctx->partials.p, n1, ctx->s,
                            task.c_last, &tail, task.gate, ctx->sa_c.p));
    ctx->add(1);
    ctx->spec.armed = true;
    ctx->spec.g = g;
    ctx->spec.rows_dev = rows_dev;
}

// ---- EGS: local auto-correlation + retained count ----------------------------------------
// Launch the R_co map + retained count for one group size; n_r lands in *nr (device).
// count_only: an EGS candidate whose map may never be used -- the fused 8-bit kernels then
// produce the retained count alone (no map stores, no divisions away from the threshold);
// returns whether `map` was written.
bool autocorr_launch(tm_ctx* ctx, tm_image* img, const WS& ws, const tmk::GridDesc& g,
                     double thr, double* map, unsigned long long* nr, int* stop = nullptr,
                     const double* egs_prev = nullptr, double egs_xi = 0.0,
                     bool count_only = false, const tmk::EgsDecide* dec = nullptr,
                     bool* decided = nullptr, const tmk::SecFuse* fuse = nullptr) {
    if (decided) *decided = false;
    const int m = ws.m, n = ws.n, p = img->p, q = img->q;
    if (!egs_prev) CK(cudaMemsetAsync(nr, 0, 8, ctx->s));  // EGS batches: egs_init zeroes it
    // (count-only candidates are timed apart: their work stops at the EGS rejection point)
    const bool fused_count = count_only && img->integer && ctx->ac_fused &&
                             tmk::autocorr_fused_supported(ws.m, ws.n, g);
    Phase ph(ctx, !img->integer ? "autocorr_replica"
                  : fused_count ? "autocorr_count"
                  : fuse        ? "autocorr_sec"
                                : "autocorr_u8");
    if (img->integer) {
        const size_t vbytes = tmk::autocorr_colwalk_bytes(q, g);
        const size_t hbytes = tmk::autocorr_rowsum_bytes(p, g);
        if (ctx->ac_fused && tmk::autocorr_fused_supported(m, n, g)) {
            // total_cost's central term (egs.cpp:28-37) for the in-kernel early rejection
            const double central = double((g.er + g.h - 1) / g.h) * double((g.ec + g.w - 1) / g.w);
            // (the group-column kernel stages rows from the 16-byte-pitched copy)
            const bool pitched = img->u8p.p && img->u8p_rows >= p + tmk::kU8PadRows;
            int nl = 1;
            CK(tmk::autocorr_u8_fused(img->u8.p, p, q, m, n, g, ws.dev(), thr,
                                      count_only ? nullptr : map, nr, stop, ctx->s, egs_prev,
                                      central, egs_xi, pitched ? img->u8p.p : nullptr,
                                      img->u8p_pitch, dec, decided, fuse, &nl));
            ctx->add(nl);
            return !count_only && !fuse;
        } else if (tmk::autocorr_colwalk_supported(m, n, q, g) && vbytes <= (size_t(16) << 30)) {
            ctx->acH.ensure(vbytes / sizeof(int));
            CK(tmk::autocorr_u8_colwalk(img->u8.p, p, q, m, n, g, ws.dev(), thr, map, nr,
                                        reinterpret_cast<unsigned*>(ctx->acH.p), ctx->s));
            ctx->add(3);
        } else if (tmk::autocorr_two_pass_supported(m, n, g) && hbytes <= (size_t(16) << 30)) {
            ctx->acH.ensure(hbytes / sizeof(int));
            CK(tmk::autocorr_u8_two_pass(img->u8.p, p, q, m, n, g, ws.dev(), thr, map, nr,
                                         ctx->acH.p, ctx->s));
            ctx->add(3);
        } else {
            CK(tmk::autocorr_u8(img->u8.p, p, q, m, n, g, ws.dev(), thr, map, nr, ctx->s));
            ctx->add(1);
        }
        return true;
    }
    CK(tmk::autocorr_init(map, g, ctx->s, stop));
    ctx->add(1);
    // the (di, dj) offsets in batches: their prefix problems are independent, one launch
    // each for the row scans and the column accumulations of a batch
    const int hr = g.h / 2, wr = g.w / 2;
    struct Off {
        int di, dj;
    };
    std::vector<Off> offs;
    for (int di = -hr; di <= hr; ++di)
        for (int dj = -wr; dj <= wr; ++dj) {
            if (di == 0 && dj == 0) continue;
            if (p - std::abs(di) < m || q - std::abs(dj) < n) continue;
            offs.push_back(Off{di, dj});
        }
    const size_t slot = size_t(p) * q, pslot = size_t(p + 1) * (q + 1);
    // batch size bounded so the scratch stays modest (<= ~4.5 GB for 4096^2 images)
    const int kb = int(std::max<size_t>(1, std::min<size_t>(tmk::kProdBatch,
                                                             (size_t(4) << 30) / (16 * pslot))));
    for (size_t o0 = 0; o0 < offs.size(); o0 += kb) {
        const int nb = int(std::min<size_t>(kb, offs.size() - o0));
        tmk::ProdBatch bt{};
        bt.n = nb;
        bt.slot = slot;
        bt.pslot = pslot;
        for (int k = 0; k < nb; ++k) {
            const int di = offs[o0 + k].di, dj = offs[o0 + k].dj;
            const int orr = std::max(0, -di), occ = std::max(0, -dj);
            bt.src[k] = tmk::ProdSrc{img->f64.p, q, orr, occ, img->f64.p, q, orr + di, occ + dj, 0,
                                     stop};
            bt.rows[k] = p - std::abs(di);
            bt.cols[k] = q - std::abs(dj);
        }
        ctx->rowacc.ensure(slot * nb);
        ctx->prefix.ensure(pslot * nb);
        CK(tmk::replica_prefix_batch(bt, ctx->rowacc.p, ctx->prefix.p, ctx->s));
        ctx->add(2);
        tmk::OffBatch ob;  // the batch's R_co epilogues in one launch
        ob.n = nb;
        for (int k = 0; k < nb; ++k) {
            ob.di[k] = offs[o0 + k].di;
            ob.dj[k] = offs[o0 + k].dj;
            ob.pw[k] = bt.cols[k];
        }
        CK(tmk::autocorr_offset_epilogue_b(ctx->prefix.p, pslot, ob, m, n, g, ws.dev(), map,
                                           ctx->s, stop));
        ctx->add(1);
    }
    CK(tmk::retained_count(map, g, thr, nr, ctx->s, stop));
    ctx->add(1);
    return true;
}

long long autocorr_map(tm_ctx* ctx, tm_image* img, const WS& ws, const tmk::GridDesc& g,
                       double thr, double* map, bool count_only = false) {
    unsigned long long* nr = ctx->counters.p + 2;
    autocorr_launch(ctx, img, ws, g, thr, map, nr, nullptr, nullptr, 0.0, count_only);
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, nr, 8, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return (long long)v;
}

// total_cost (egs.cpp:27-37)
tm_egs_iter total_cost_h(int er, int ec, int h, int w, long long n_r, double amortized) {
    if (h < 1 || w < 1) invalid("total_cost: group size must be >= 1");
    tm_egs_iter it{};
    it.h = h;
    it.w = w;
    it.central = double((er + h - 1) / h) * double((ec + w - 1) / w);
    it.retained = n_r;
    it.retained_cost = double(n_r);
    it.amortized = amortized;
    it.total = it.central + it.retained_cost + it.amortized;
    return it;
}

struct EgsOut {
    int h = 0, w = 0;
    tm_egs_iter cost{};
    std::vector<tm_egs_iter> trace;
};

// efficient_group_size (egs.cpp:39-91); best map ends in `best`.
// fuse (tm_search): the candidate of the predicted size runs scan 2 in its R_co launch
// instead of writing its map (SecFuse); *fuse_hit tells whether EGS accepted that size, in
// which case no map exists (and none is needed).  On a miss the accepted size's map is
// computed as usual.
EgsOut run_egs_search(tm_ctx* ctx, tm_image* img, const WS& ws, int m, int n, int h0, int w0,
                      double rho_tb, double xi, int max_group, DBuf<double>& best,
                      const std::function<void()>* before_sync = nullptr,
                      const tmk::SecFuse* fuse = nullptr, bool* fuse_hit = nullptr,
                      bool egs_preinit = false) {
    if (fuse_hit) *fuse_hit = false;
    bool fused_ran = false;  // the fused candidate was launched in the first batch
    unsigned long long first_seq = 0;
    if (h0 < 1 || w0 < 1 || h0 % 2 == 0 || w0 % 2 == 0)
        invalid("efficient_group_size: initial group size must be odd");
    if (rho_tb <= 0.0 || rho_tb >= 1.0)
        invalid("efficient_group_size: rho_tb must be in (0,1)");
    const int er = img->p - m + 1, ec = img->q - n + 1;
    if (er < 1 || ec < 1) invalid("efficient_group_size: template does not fit");
    if (rho_tb < 0.0 || rho_tb > 1.0) invalid("retained_count: rho_tb must be in [0,1]");
    const double thr = expected_elimination_threshold_h(rho_tb);
    int cap = max_group > 0 ? max_group : INT_MAX;
    if (cap % 2 == 0) ++cap;
    const size_t E = size_t(er) * ec;
    best.ensure(E);
    EgsOut out;
    double prev_cost = std::numeric_limits<double>::infinity();
    int h = h0, w = w0;
    bool done = false;
    // Candidates are launched in batches of up to four group sizes and decided after one
    // readback; the accept/stop sequence is exactly egs.cpp:61-88.  A one-thread kernel
    // replays the same decision on the device after each candidate, so candidates the host
    // is going to ignore (after the first rejection) exit at entry instead of running.
    double* dprev = reinterpret_cast<double*>(ctx->counters.p + 20);
    int* dstop = reinterpret_cast<int*>(ctx->counters.p + 21);
    unsigned long long* dgate = ctx->counters.p + 24;  // speculation gate (tm_search)
    int* dhacc = reinterpret_cast<int*>(ctx->counters.p + 25);
    bool first_batch = true;
    // Only the accepted size's map is used: the predicted h_e (the last one seen for this
    // image / template shape, else h0) writes its map, the other candidates count only, and
    // a size accepted without a map is recomputed once after the loop (count re-checked).
    int map_h = -1, map_w = -1;
    const std::vector<long long> he_key = {img->p, img->q, m, n, h0, w0};
    int pred = h0;
    if (h0 == w0) {
        const auto it = ctx->last_he.find(he_key);
        if (it != ctx->last_he.end()) pred = it->second;
    }
    while (!done) {
        struct Cand {
            int h, w;
        } cand[4];
        int nc = 0;
        int hh = h, ww = w;
        // first batch: up to one size past the predicted h_e (a misprediction costs another
        // batch); later batches: four
        const int nmax = first_batch ? std::max(2, std::min(4, (pred - h) / 2 + 2)) : 4;
        for (; nc < nmax;) {
            cand[nc++] = Cand{hh, ww};
            if ((hh >= er && ww >= ec) || (hh >= cap && ww >= cap)) break;
            hh = std::min(hh + 2, cap);
            ww = std::min(ww + 2, cap);
        }
        bool map_written[4] = {false, false, false, false};
        const unsigned long long batch_seq = ++ctx->egs_seq;
        if (first_batch) first_seq = batch_seq;
        if (first_batch) {  // stop = 0, prev = +inf, nr[0..3] = 0, h_acc = 0, gate = 0
            if (!egs_preinit) {  // (else done by the centre scan's reduction)
                CK(tmk::egs_init(dstop, dprev, ctx->counters.p + 8, ctx->s, dhacc, dgate));
                ctx->add(1);
            }
            first_batch = false;
        } else {
            CK(cudaMemsetAsync(ctx->counters.p + 8, 0, 32, ctx->s));
        }
        for (int k = 0; k < nc; ++k) {
            const tmk::GridDesc g = make_grid(er, ec, cand[k].h, cand[k].w);
            ctx->egs_maps[k].ensure(E);
            // the decision after the candidate (after the last one too: the speculation gate
            // needs the final decision, and that decide also writes the counts + gate into
            // the mapped pinned block); fused into the R_co launch's tail where supported
            const bool last = k + 1 == nc;
            tmk::EgsDecide dec{};
            dec.ticket = reinterpret_cast<unsigned*>(ctx->counters.p + 27);
            dec.n_r = ctx->counters.p + 8 + k;
            dec.prev = dprev;
            dec.stop = dstop;
            dec.er = er;
            dec.ec = ec;
            dec.h = cand[k].h;
            dec.w = cand[k].w;
            dec.xi = xi;
            dec.cap = cap;
            dec.h_acc = dhacc;
            dec.want = ctx->spec_want;
            dec.gate = dgate;
            dec.nr_all = ctx->counters.p + 8;
            dec.nc = nc;
            dec.out = last ? ctx->hres_dev : nullptr;
            dec.seq = batch_seq;
            if (fuse && last && batch_seq == first_seq) {  // the gated survivors' dispatch
                dec.disp_tally = ctx->tally.p;
                dec.disp_E = E;
                dec.disp_dense = reinterpret_cast<int*>(ctx->counters.p + 22);
                dec.disp_list = ctx->counters.p + 23;
            }
            // the first candidate counts retained members per extent row; later count-only
            // candidates (in-kernel rejection) walk their segments densest first
            if (ctx->egs_order && nc > 1) {
                if (k == 0) {
                    ctx->egs_rows.ensure(size_t(er));
                    CK(cudaMemsetAsync(ctx->egs_rows.p, 0, size_t(er) * sizeof(unsigned), ctx->s));
                    dec.rows_out = ctx->egs_rows.p;
                } else {
                    dec.rows_in = ctx->egs_rows.p;
                }
            }
            bool decided = false;
            const bool is_pred = cand[k].h == pred && cand[k].w == pred;
            const bool fuse_here = fuse && is_pred && !fused_ran;
            map_written[k] = autocorr_launch(ctx, img, ws, g, thr,
                                             fuse_here ? nullptr : ctx->egs_maps[k].p,
                                             ctx->counters.p + 8 + k, dstop, dprev, xi,
                                             /*count_only=*/!is_pred, &dec, &decided,
                                             fuse_here ? fuse : nullptr);
            if (fuse_here) fused_ran = true;
            if (!decided) {
                CK(tmk::egs_decide_d(dec, ctx->s));
                ctx->add(1);
            }
        }
        // the host waits for this point only, so work enqueued by the hook keeps the device
        // busy meanwhile
        CK(cudaEventRecord(ctx->ev_egs, ctx->s));
        if (before_sync && *before_sync) {  // host work overlapped with the candidates
            (*before_sync)();
            before_sync = nullptr;
        }
        ctx->spec_want = 0;  // later batches: the speculation (if any) was for this one
        HT("egs_enqueued");
        // poll the sequence number the last decide writes into mapped pinned memory after
        // the counts (lower wake-up latency than an event wait); the event still guards
        // against a device error
        {
            const volatile unsigned long long* sq = &ctx->hres->seq;
            for (unsigned spins = 0; *sq != batch_seq; ++spins) {
                if ((spins & 255) == 255) {
                    const cudaError_t q = cudaEventQuery(ctx->ev_egs);
                    if (q == cudaSuccess) break;
                    if (q != cudaErrorNotReady) CK(q);
                }
            }
            CK(cudaEventSynchronize(ctx->ev_egs));  // normally complete already
        }
        HT("egs_sync");
        unsigned long long nr[4] = {0, 0, 0, 0};
        for (int k = 0; k < nc; ++k) nr[k] = ctx->hres->nr[k];
        for (int k = nc; k < 4; ++k) map_written[k] = false;
        for (int k = 0; k < nc; ++k) {
            const tm_egs_iter cost = total_cost_h(er, ec, cand[k].h, cand[k].w, (long long)nr[k], 0.0);
            const bool accepted =
                !std::isfinite(prev_cost) || prev_cost - cost.total > xi * prev_cost;
            if (!accepted) {
                done = true;
                break;
            }
            out.h = cand[k].h;
            out.w = cand[k].w;
            out.cost = cost;
            out.trace.push_back(cost);
            if (fuse_hit) *fuse_hit = fused_ran && cand[k].h == pred && cand[k].w == pred;
            if (map_written[k]) {
                best.swap(ctx->egs_maps[k]);
                map_h = cand[k].h;
                map_w = cand[k].w;
            }
            prev_cost = cost.total;
            if ((cand[k].h >= er && cand[k].w >= ec) || (cand[k].h >= cap && cand[k].w >= cap)) {
                done = true;
                break;
            }
            h = std::min(cand[k].h + 2, cap);
            w = std::min(cand[k].w + 2, cap);
        }
    }
    if (fuse_hit && *fuse_hit && !(out.h == pred && out.w == pred)) *fuse_hit = false;
    if ((out.h != map_h || out.w != map_w) && !(fuse_hit && *fuse_hit)) {
        best.ensure(E);
        const long long n_r = autocorr_map(ctx, img, ws, make_grid(er, ec, out.h, out.w), thr,
                                           best.p);
        if (n_r != out.cost.retained)
            throw TmError{TM_ECUDA, "efficient_group_size: map recount mismatch"};
    }
    if (h0 == w0 && out.h == out.w) {
        if (ctx->last_he.size() > 256) ctx->last_he.clear();
        ctx->last_he[he_key] = out.h;
    }
    return out;
}

// ---- OptA -----------------------------------------------------------------------------
double quality_threshold_h(double rho_th, double rho_max) {
    if (rho_th < 0.0 || rho_th > 1.0 || rho_max < 0.0 || rho_max > 1.0)
        invalid("quality_threshold: inputs must be in [0,1]");
    if (rho_max < rho_th) invalid("quality_threshold: rho_max must be >= rho_th");
    return elimination_autocorr_threshold_h(rho_th, rho_max);
}

std::unique_ptr<tm_image> device_image_like(tm_ctx* ctx, int p, int q) {
    auto img = std::make_unique<tm_image>();
    img->ctx = ctx;
    img->p = p;
    img->q = q;
    img->f64.ensure(size_t(p) * q);
    img->have_f64 = true;
    return img;
}

void fidelity(tm_ctx* ctx, tm_image* orig, const WS& ws_orig, tm_image* blurred, WS& ws_b,
              double* fid) {
    const int p = orig->p, q = orig->q, m = ws_orig.m, n = ws_orig.n;
    const size_t E = size_t(ws_orig.er) * ws_orig.ec;
    ctx->cross.ensure(E);
    // product = I_blur * I (blur.cpp:101-103)
    replica_sums(ctx, tmk::ProdSrc{blurred->f64.p, q, 0, 0, orig->f64.p, q, 0, 0, 0}, p, q, m, n,
                 ctx->cross.p);
    blurred->have_qtotal = false;
    compute_ws(ctx, blurred, m, n, ws_b);
    CK(tmk::fidelity_epilogue(ctx->cross.p, ws_orig.dev(), ws_b.dev(), fid, ctx->s));
    ctx->add(1);
}

// repair_to_fixed_point (blur.cpp:208-239); leaves ws_b = window_stats(final blurred).
long long repair(tm_ctx* ctx, tm_image* blurred, tm_image* orig, const WS& ws_orig, double lambda,
                 WS& ws_b) {
    const int p = orig->p, q = orig->q, m = ws_orig.m, n = ws_orig.n;
    const int er = ws_orig.er, ec = ws_orig.ec;
    const size_t E = size_t(er) * ec, N = size_t(p) * q;
    ctx->fid.ensure(E);
    ctx->inwin.ensure(E);
    ctx->u8tmp.ensure(N);
    ctx->marks.ensure(E);
    ctx->markP.ensure(size_t(er + 1) * (ec + 1));
    ctx->hs.ensure(size_t(p) * ec);
    long long total = 0;
    for (;;) {
        fidelity(ctx, orig, ws_orig, blurred, ws_b, ctx->fid.p);
        CK(tmk::changed_mask(blurred->f64.p, orig->f64.p, N, ctx->u8tmp.p, ctx->s));
        CK(tmk::window_sums_u8(ctx->u8tmp.p, p, q, m, n, ctx->hs.p, ctx->inwin.p, ctx->s));
        CK(tmk::mark_violations(ctx->fid.p, ctx->inwin.p, E, lambda, ctx->marks.p,
                                ctx->counters.p + 3, ctx->s));
        ctx->add(4);
        unsigned long long count = 0;
        CK(cudaMemcpyAsync(&count, ctx->counters.p + 3, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        if (count == 0) break;
        CK(tmk::restore_covered(blurred->f64.p, orig->f64.p, ctx->marks.p, er, ec, m, n, p, q,
                                ctx->markP.p, ctx->s));
        ctx->add(3);
        total += (long long)count;
    }
    return total;
}

// optimize_autocorrelation (blur.cpp:243-278) + prepare_opta (matcher.cpp:217-233).
void run_opta_prep(tm_ctx* ctx, tm_image* img, tm_prep* prep) {
    const tm_match_params& P = prep->params;
    const int m = prep->m, n = prep->n, p = img->p, q = img->q;
    const double lambda = quality_threshold_h(P.rho_th, P.rho_max);
    WS& ws_orig = get_ws(ctx, img, m, n);
    ensure_f64(ctx, img);
    EgsOut e0 = run_egs_search(ctx, img, ws_orig, m, n, P.h0, P.w0, P.rho_th, P.xi_fraction,
                               P.max_group, prep->map);
    prep->lambda = lambda;
    prep->kappa = 0;
    prep->opta_trace.clear();
    prep->opta_trace.push_back(tm_opta_iter{e0.h, e0.w, e0.cost.total, 0});
    double prev_cost = e0.cost.total;
    int h = e0.h, w = e0.w;
    prep->h = h;
    prep->w = w;
    prep->cost = e0.cost;
    prep->egs_trace = e0.trace;

    const size_t N = size_t(p) * q;
    ctx->prof.ensure(prep->profile.size());
    CK(cudaMemcpyAsync(ctx->prof.p, prep->profile.data(), prep->profile.size() * 8,
                       cudaMemcpyHostToDevice, ctx->s));
    const int len = int(prep->profile.size());
    const bool identity = (len == 1);  // blur.cpp:59: radius 0 and one tap returns img
    auto current = device_image_like(ctx, p, q);
    CK(cudaMemcpyAsync(current->f64.p, img->f64.p, N * 8, cudaMemcpyDeviceToDevice, ctx->s));
    std::unique_ptr<tm_image> accepted;  // optimised image (nullptr: the original)
    std::unique_ptr<WS> accepted_ws;
    DBuf<double> map_k;
    ctx->dtmp.ensure(N);
    for (int iter = 1; iter <= 64; ++iter) {
        auto blurred = device_image_like(ctx, p, q);
        if (identity) {
            CK(cudaMemcpyAsync(blurred->f64.p, current->f64.p, N * 8, cudaMemcpyDeviceToDevice,
                               ctx->s));
        } else {
            CK(tmk::blur_replica(current->f64.p, p, q, ctx->prof.p, len, ctx->dtmp.p,
                                 blurred->f64.p, ctx->s));
            ctx->add(2);
        }
        auto ws_b = std::make_unique<WS>();
        const long long restored = repair(ctx, blurred.get(), img, ws_orig, lambda, *ws_b);
        // efficient_group_size(blurred) recomputes window_stats(blurred) == ws_b
        blurred->integer = false;
        EgsOut ek = run_egs_search(ctx, blurred.get(), *ws_b, m, n, h, w, P.rho_th, P.xi_fraction,
                                   P.max_group, map_k);
        const double improvement = prev_cost - ek.cost.total;
        if (!(improvement >= P.opta_margin * ek.cost.total)) break;
        prep->opta_trace.push_back(tm_opta_iter{ek.h, ek.w, ek.cost.total, restored});
        prep->kappa = iter;
        prev_cost = ek.cost.total;
        h = ek.h;
        w = ek.w;
        prep->h = h;
        prep->w = w;
        prep->cost = ek.cost;
        prep->egs_trace = ek.trace;
        prep->map.swap(map_k);
        // the accepted image becomes the next iteration's input
        auto cur_copy = device_image_like(ctx, p, q);
        CK(cudaMemcpyAsync(cur_copy->f64.p, blurred->f64.p, N * 8, cudaMemcpyDeviceToDevice,
                           ctx->s));
        current = std::move(cur_copy);
        accepted = std::move(blurred);
        accepted_ws = std::move(ws_b);
    }
    if (accepted) {
        // classify (an exact-integer optimised image would take the integer kernels)
        accepted->have_qtotal = false;
        classify_device_image(ctx, accepted.get());
        if (accepted->integer) accepted_ws.reset();  // recompute through the integer path
        prep->search_img = std::move(accepted);
        if (accepted_ws) {
            prep->search_ws = std::move(accepted_ws);
        } else {
            prep->search_ws = std::make_unique<WS>();
            compute_ws(ctx, prep->search_img.get(), m, n, *prep->search_ws);
        }
    }
    prep->radius = len / 2;
    CK(cudaStreamSynchronize(ctx->s));
}

// ---- scan 2 / transitive search (matcher.cpp:95-177) -----------------------------------
struct SearchIn {
    tm_image* img;
    const WS* ws;
    tmk::GridDesc g;
    const double* map;  // device
    // scan 1, the seeding and scan 2 already ran (fused into the R_co launch, tm_search):
    // only the survivors and the result remain
    bool prescanned = false;
    // ... and the survivor evaluation is already enqueued (gated on the EGS decision)
    bool survivors_enqueued = false;
};

// Scan-2 survivors (listed in ctx->locs, marked 2 in ctx->visits) -> cells[2].  Dense
// survivor sets run the band kernel masked by the visit map; sparse ones one warp per
// location.  rho_loc (optional, extent-sized) receives rho by location.
bool brute_split(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T,
                 const uint8_t* mask = nullptr);

void eval_survivors(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T,
                    const tmk::GridDesc& g, unsigned long long survivors, double* rho_loc,
                    const tmk::TileFlags* tflags = nullptr) {
    cudaStream_t s = ctx->s;
    const size_t E = size_t(g.er) * g.ec;
    const unsigned long long* count = &ctx->tally.p->survivors;
    uint8_t* visits = ctx->visits.p;
    const bool dense = survivors * tmk::kDenseDiv > E && fp32_path(img, T);
    if (dense && tc_path(ctx, img, T)) {
        const int rlo = g.ti_lo * g.h, rhi = std::min(g.ti_hi * g.h, g.er);
        RowSet rs;
        rs.lo = rlo;
        rs.hi = std::max(rlo, rhi);
        tmk::TcTask task{};
        task.mode = 2;
        task.c_lim = g.ec;
        task.c_last = -1;
        task.mask = visits;
        task.tf = tflags ? *tflags : tmk::TileFlags{};
        task.out_rho = rho_loc;
        ctx->partials.ensure(148 + 1);
        int np = 0;
        if (rs.hi > rs.lo) {
            Phase ph(ctx, "survivor_dense");
            np = tc_run(ctx, img, ws, T, rs, 1, task);
        }
        reduce_to(ctx, np, 2);
    } else if (dense) {
        const tmk::CorrJob job = make_job(ctx, img, ws, T);
        const int rlo = g.ti_lo * g.h, rhi = std::min(g.ti_hi * g.h, g.er);
        std::vector<int> rows(std::max(0, rhi - rlo));
        for (int r = rlo; r < rhi; ++r) rows[r - rlo] = r;
        upload_rows(ctx, rows);
        tmk::BandTask t{};
        t.rows = ctx->rows_list.p;
        t.nrows = int(rows.size());
        t.cbase = 0;
        t.sw = 1;
        t.nc = g.ec;
        t.mode = 2;
        t.row_span = 7;
        t.ksplit = 1;
        t.ms = T.m;
        t.out_rho = rho_loc;
        t.mask = visits;
        ctx->partials.ensure(size_t(band_partials(std::max(1, int(rows.size())), g.ec, 1)));
        int np = 0;
        {
            Phase ph(ctx, "survivor_dense");
            CK(tmk::corr_band(band_job(ctx, img, job), t, ctx->partials.p, &np, s));
            ctx->add(1);
        }
        reduce_to(ctx, np, 2);
    } else if (survivors > 0) {
        // non-integer image, many survivors whose rho only matters for the argmax (frozen /
        // seeded): bracket them all on the split planes (masked by the visit codes) and
        // replay the few that can still win
        if (!rho_loc && survivors > std::max<unsigned long long>(16 * kListBlocks, E / 64) &&
            g.ti_lo == 0 && g.ti_hi == g.tr &&
            split_path(ctx, img, T, double(E) * T.m * T.n, 67108864.0) &&
            brute_split(ctx, img, ws, T, visits))
            return;
        const tmk::CorrJob job = make_job(ctx, img, ws, T);
        ctx->partials.ensure(kListBlocks);
        {
            Phase ph(ctx, "survivor_eval");
            if (fp32_path(img, T))
                CK(tmk::corr_list(job, ctx->locs.p, count, int(std::min<size_t>(E, INT_MAX)),
                                  rho_loc, nullptr, ctx->partials.p, kListBlocks, s, 1));
            else
                CK(tmk::corr_list_f64(job, ctx->locs.p, count, int(std::min<size_t>(E, INT_MAX)),
                                      rho_loc, nullptr, ctx->partials.p, kListBlocks, s, 1));
            ctx->add(1);
        }
        reduce_to(ctx, kListBlocks, 2);
    } else {
        reduce_to(ctx, 0, 2);
    }

}

// eval_survivors without the host round trip (tensor-core path): the survivor count stays
// on the device; survivor_dispatch selects dense (masked tensor-core kernel) or list, the
// other launch only writes empty partials.
// dispatched: the dense/list choice is already made on the device (by the last EGS decision)
// locs / mask / packed: a batch template's survivor list, visit codes and result slot
// (default: the context's own).
void eval_survivors_dev(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T,
                        const tmk::GridDesc& g, double* rho_loc,
                        const unsigned long long* gate = nullptr, bool dispatched = false,
                        const int2* locs = nullptr, const uint8_t* mask = nullptr,
                        tmk::ResultBlock* packed = nullptr,
                        const tmk::TileFlags* tflags = nullptr) {
    cudaStream_t s = ctx->s;
    const size_t E = size_t(g.er) * g.ec;
    if (!locs) locs = ctx->locs.p;
    if (!mask) mask = ctx->visits.p;
    if (!packed) packed = ctx->hres_dev;
    int* dense_flag = reinterpret_cast<int*>(ctx->counters.p + 22);
    unsigned long long* list_count = ctx->counters.p + 23;
    if (!dispatched) CK(tmk::survivor_dispatch(ctx->tally.p, E, dense_flag, list_count, s, gate));
    ctx->partials.ensure(size_t(148 + kListBlocks) + 1);
    const int rlo = g.ti_lo * g.h, rhi = std::min(g.ti_hi * g.h, g.er);
    int np = 0;
    if (rhi > rlo) {
        RowSet rs;
        rs.lo = rlo;
        rs.hi = rhi;
        tmk::TcTask task{};
        task.mode = 2;
        task.c_lim = g.ec;
        task.c_last = -1;
        task.mask = mask;
        task.tf = tflags ? *tflags : tmk::TileFlags{};
        task.out_rho = rho_loc;
        task.gate = dense_flag;
        Phase ph(ctx, "survivor_eval");
        np = tc_run(ctx, img, ws, T, rs, 1, task);
    }
    const tmk::CorrJob job = make_job(ctx, img, ws, T);
    tmk::ReduceOp op_pack{};  // the final reduction packs the result into pinned host memory
    op_pack.kind = 3;
    op_pack.cells = ctx->cells.p;
    op_pack.tally = ctx->tally.p;
    op_pack.thr = ctx->thr.p;
    op_pack.packed = packed;
    // fused into the list kernel's tail: the tensor-core partials [0, np) are already in
    const tmk::TailReduce tail = tail_to(ctx, np + kListBlocks, 2, &op_pack);
    Phase ph(ctx, "survivor_list");
    CK(tmk::corr_list(job, locs, list_count, int(std::min<size_t>(E, INT_MAX)), rho_loc,
                      nullptr, ctx->partials.p + np, kListBlocks, s, 1, &tail));
    ctx->add(2);
}

tm_match_result search(tm_ctx* ctx, const SearchIn& in, const Tmpl& T,
                       const tm_match_params& P, uint8_t* visits_host) {
    const tmk::GridDesc& g = in.g;
    if (T.ts.flat) invalid("transitive_search: constant template has no defined correlation");
    if (P.has_init_threshold && std::abs(P.init_threshold) > 1.0 + 1e-9)
        invalid("transitive_search: init threshold out of [-1,1]");
    const size_t E = size_t(g.er) * g.ec, G = size_t(g.tr) * g.tc;
    tm_image* img = in.img;
    const WS& ws = *in.ws;
    cudaStream_t s = ctx->s;

    int policy = P.policy;
    if (policy == TM_POLICY_REFERENCE)
        policy = (P.parallel && P.threads > 1 && G > 1) ? TM_POLICY_FROZEN : TM_POLICY_SEQUENTIAL;
    const bool seq = policy == TM_POLICY_SEQUENTIAL;

    // ---- scan 1 + threshold bootstrap (matcher.cpp:116-125) ---------------------------
    HT("search_begin");
    // the centre reduction also bootstraps the threshold (matcher.cpp:121-125) and zeroes
    // the seeding counters and the scan-2 tally
    const uint8_t* seeded = nullptr;
    bool split_c = false;  // scan 1 bracketed on the split planes (non-integer image)
    if (!in.prescanned) {
    const tmk::ReduceOp op_init = centre_op(ctx, P);
    split_c = split_centres_ok(ctx, img, T, g);
    if (split_c)
        centre_scan_split(ctx, img, ws, T, g, &op_init);
    else
        centre_scan(ctx, img, ws, T, g, &op_init);
    HT("centre_scan");

    if (policy == TM_POLICY_SEEDED) {
        if (split_c) split_refine_seeding(ctx, img, ws, T, g, P.seed_margin);
        const unsigned long long max_groups = 256;
        const unsigned long long max_locs = max_groups * (unsigned long long)(g.h * g.w);
        ctx->seed_locs.ensure(max_locs);
        ctx->seeded.ensure(G);
        CK(tmk::seed_members(g, ctx->rho_c.p, ctx->deg_c.p, ctx->thr.p, P.seed_margin,
                             ctx->seeded.p, ctx->seed_locs.p, ctx->counters.p + 4, max_locs,
                             ctx->counters.p + 5, max_groups, s));
        ctx->add(1);
        tmk::ReduceOp op_raise{};  // the seed reduction raises the threshold
        op_raise.kind = 2;
        op_raise.thr = ctx->thr.p;
        eval_list(ctx, img, ws, T, ctx->seed_locs.p, ctx->counters.p + 4, int(max_locs), nullptr,
                  nullptr, 1, &op_raise);
        seeded = ctx->seeded.p;
        HT("seeds");
    }
    }

    // ---- scan 2: bound test + survivor compaction -------------------------------------
    ctx->visits.ensure(E);
    uint8_t* visits = ctx->visits.p;
    ctx->locs.ensure(E);
    if (split_c) split_refine_bounds(ctx, img, ws, T, g, in.map, seeded, seq);
    if (!in.prescanned) {
        Phase ph(ctx, "sec_compact");
        ctx->sa_c.ensure(G);
        // frozen / seeded on the exact 8-bit path: a survivor list longer than E/16 is never
        // read (the dense path takes over, driven by the visit mask), so only that many
        // locations are written; the sequential replay and the FP64 path read every one
        const unsigned long long max_locs = (!seq && fp32_path(img, T)) ? E / 16 + 1 : E;
        const tmk::TileFlags tf = zero_tile_flags(ctx, ctx->tflags, g.er, g.ec);
        CK(tmk::sec_rows(g, in.map, ctx->rho_c.p, ctx->sa_c.p, ctx->deg_c.p, ws.fl.p, T.ts.flat,
                         ctx->thr.p, seeded, ctx->locs.p, max_locs, ctx->tally.p, visits, s,
                         ctx->sa_ready, tf));
        ctx->add(ctx->sa_ready ? 1 : 2);
    }
    double T0 = 0.0;
    tmk::Tally tally{};
    const unsigned long long* count = &ctx->tally.p->survivors;
    double* rho_loc = nullptr;
    HT("sec_compact");
    const bool device_dispatch = !seq && tc_path(ctx, img, T);
    if (device_dispatch) {
        // frozen / seeded: nothing changes the threshold after scan 2's bound test, so the
        // final readback gives T0; the survivor count never leaves the device
        const tmk::TileFlags tf{ctx->tflags.p, (g.ec + 2047) >> 11};
        if (!in.survivors_enqueued)
            eval_survivors_dev(ctx, img, ws, T, g, nullptr, nullptr, false, nullptr, nullptr,
                               nullptr, &tf);
    } else {
        CK(cudaMemcpyAsync(&T0, ctx->thr.p, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&tally, ctx->tally.p, sizeof tally, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (seq) {
            ctx->seq_rho.ensure(E);
            rho_loc = ctx->seq_rho.p;
        }
        eval_survivors(ctx, img, ws, T, g, tally.survivors, rho_loc);
    }

    double final_T = T0;
    if (seq) {
        // Replay the running threshold (matcher.cpp:73-74): records in scan order.
        Phase ph(ctx, "sequential_replay");
        std::vector<unsigned long long> rk;
        std::vector<double> rt;
        double Tcur = T0;
        unsigned long long after = ~0ull;
        for (;;) {
            CK(tmk::first_record(g, ctx->locs.p, count, rho_loc, in.map, ctx->rho_c.p,
                                 ctx->deg_c.p, ws.fl.p, T.ts.flat, Tcur, after,
                                 ctx->counters.p + 6, s));
            ctx->add(1);
            unsigned long long key = 0;
            CK(cudaMemcpyAsync(&key, ctx->counters.p + 6, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (key == ~0ull) break;
            double rho = 0.0;
            CK(tmk::fetch_record_rho(g, ctx->locs.p, count, rho_loc, key, ctx->thr.p + 1, s));
            ctx->add(1);
            CK(cudaMemcpyAsync(&rho, ctx->thr.p + 1, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            rk.push_back(key);
            rt.push_back(rho);
            Tcur = rho;
            after = key;
        }
        ctx->rec_key.ensure(rk.size() + 1);
        ctx->rec_T.ensure(rk.size() + 1);
        if (!rk.empty()) {
            CK(cudaMemcpyAsync(ctx->rec_key.p, rk.data(), rk.size() * 8, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(ctx->rec_T.p, rt.data(), rt.size() * 8, cudaMemcpyHostToDevice, s));
        }
        ctx->partials.ensure(kListBlocks);
        CK(tmk::seq_final(g, ctx->locs.p, count, rho_loc, in.map, ctx->rho_c.p, ctx->deg_c.p,
                          ws.fl.p, T.ts.flat, T0, ctx->rec_key.p, ctx->rec_T.p, int(rk.size()),
                          ctx->tally.p, visits, ctx->partials.p, kListBlocks, s));
        ctx->add(1);
        reduce_to(ctx, kListBlocks, 2);
        final_T = Tcur;
    }
    HT("survivors");
    tm_ctx::HostRes* hr = ctx->hres;
    if (device_dispatch) {
        // already packed into the mapped pinned block by the final reduction
    } else {
        CK(cudaMemcpyAsync(hr->cells, ctx->cells.p, sizeof hr->cells, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&hr->tally, ctx->tally.p, sizeof hr->tally, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&hr->thr, ctx->thr.p, 8, cudaMemcpyDeviceToHost, s));
    }
    if (visits_host) CK(cudaMemcpyAsync(visits_host, visits, E, cudaMemcpyDeviceToHost, s));
    HT("readback_enq");
    if (ctx->before_final_sync) {  // wait for this search only, not for the hook's work
        // (ev1 doubles as the end mark of tm_search's wall time)
        CK(cudaEventRecord(ctx->ev1, s));
        ctx->ev1_set = true;
        const std::function<void()> f = std::move(ctx->before_final_sync);
        ctx->before_final_sync = nullptr;
        f();
        spin_wait(ctx->ev1);
    } else {
        CK(cudaEventRecord(ctx->ev1, s));
        ctx->ev1_set = true;
        spin_wait(ctx->ev1);
    }
    HT("sync");
    tmk::CellH cells[3] = {hr->cells[0], hr->cells[1], hr->cells[2]};
    tally = hr->tally;
    const double thr_after = hr->thr;

    tmk::CellH best = cells[0];
    if (policy == TM_POLICY_SEEDED && better_h(cells[1], best)) best = cells[1];
    if (better_h(cells[2], best)) best = cells[2];
    if (better_h(flat_cell(tally), best)) best = flat_cell(tally);

    const long long eliminated = (long long)tally.eliminated;
    // sequential: alive candidates (dead ones were moved to `eliminated` by seq_final) and
    // the retained flat members, which are never listed
    const long long retained =
        seq ? (long long)(tally.pad + tally.flat_n) : (long long)tally.retained;
    if (device_dispatch) final_T = thr_after;  // = T0 (see above)
    if (policy == TM_POLICY_SEEDED) {
        final_T = thr_after;
        if ((cells[2].flags & 1) && !(cells[2].flags & 2)) final_T = std::max(final_T, cells[2].rho);
    }
    tm_match_result r{};
    r.mode = TM_MODE_EGS;
    r.extent_rows = g.er;
    r.extent_cols = g.ec;
    r.best_row = r.refined_row = best.row;
    r.best_col = r.refined_col = best.col;
    r.best_rho = r.refined_rho = best.rho;
    r.best_degenerate = (best.flags & 2) != 0;
    r.final_threshold = std::isfinite(final_T) ? final_T : 0.0;
    r.below_threshold =
        P.has_init_threshold && (r.best_degenerate || best.rho < P.init_threshold);
    r.centers = (long long)G;
    r.eliminated = eliminated;
    r.retained = retained;
    r.elim_pct = 100.0 * double(eliminated) / (double(g.er) * double(g.ec));
    r.ops = (long long)G + retained;
    return r;
}

// refine_impl (matcher.cpp:80-93) on the original image.
tmk::CellH refine(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T, int lr, int lc, int d,
                  long long* ops) {
    const int r0 = std::max(0, lr - d), r1 = std::min(ws.er - 1, lr + d);
    const int c0 = std::max(0, lc - d), c1 = std::min(ws.ec - 1, lc + d);
    std::vector<int2> locs;
    for (int r = r0; r <= r1; ++r)
        for (int c = c0; c <= c1; ++c) locs.push_back(make_int2(r, c));
    *ops += (long long)locs.size();
    ctx->seed_locs.ensure(locs.size());
    ctx->pin_locs.upload(ctx->seed_locs.p, locs.data(), locs.size() * sizeof(int2), ctx->s);
    unsigned long long cnt = locs.size();
    CK(cudaMemcpyAsync(ctx->counters.p + 7, &cnt, 8, cudaMemcpyHostToDevice, ctx->s));
    eval_list(ctx, img, ws, T, ctx->seed_locs.p, ctx->counters.p + 7, int(locs.size()), nullptr,
              nullptr, 3);
    tmk::CellH c;
    CK(cudaMemcpyAsync(&c, ctx->cells.p + 3, sizeof c, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    return c;
}

// brute_force_match on a non-integer image: bracket rho everywhere with the split
// tensor-core pass, list the locations whose upper bound reaches the largest lower bound,
// evaluate those with the FP64 replica (window_dot order) -> cells[2].  False: the list
// overflowed or nothing was non-flat (the caller runs the dense FP64 replica instead).
// mask: only the locations with mask == 2 compete (scan-2 survivors of a frozen / seeded
// search).
bool brute_split(tm_ctx* ctx, tm_image* img, const WS& ws, const Tmpl& T,
                 const uint8_t* mask) {
    const int er = ws.er, ec = ws.ec;
    const size_t E = size_t(er) * ec;
    RowSet rs;
    rs.lo = 0;
    rs.hi = er;
    tmk::TcTask task{};
    task.mode = 3;
    task.c_lim = ec;
    task.c_last = -1;
    task.mask = mask;
    ctx->ub_surface.ensure(E);
    task.out_ub = ctx->ub_surface.p;
    ctx->partials.ensure(size_t(148 + kListBlocks) + 1);
    const int np = tc_run(ctx, img, ws, T, rs, 1, task);
    reduce_to(ctx, np, 3);  // cells[3].rho = the largest lower bound
    const size_t cap = std::min<size_t>(E, size_t(1) << 20);
    ctx->split_locs.ensure(cap);
    unsigned long long* cnt = ctx->counters.p + 35;
    CK(cudaMemsetAsync(cnt, 0, 8, ctx->s));
    CK(tmk::tc_screen_compact(ctx->ub_surface.p, er, ec, ctx->cells.p + 3, ctx->split_locs.p, cnt, cap,
                              ctx->s));
    ctx->add(1);
    unsigned long long n = 0;
    CK(cudaMemcpyAsync(&n, cnt, 8, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    if (n == 0 || n > cap) return false;
    ctx->split_screened += (long long)E;
    ctx->split_exact += (long long)n;
    eval_list(ctx, img, ws, T, ctx->split_locs.p, cnt, int(cap), nullptr, nullptr, 2);
    return true;
}

// brute_force_match (stats.cpp:156-213)
tm_match_result brute(tm_ctx* ctx, tm_image* img, const Tmpl& T, double* surface_host) {
    const int m = T.m, n = T.n;
    if (m > img->p || n > img->q)
        invalid("brute_force_match: template larger than search image");
    WS& ws = get_ws(ctx, img, m, n);
    const int er = ws.er, ec = ws.ec;
    const size_t E = size_t(er) * ec;
    double* surface = nullptr;
    if (surface_host) {
        ctx->surface.ensure(E);
        surface = ctx->surface.p;
    }
    const tmk::CorrJob job = make_job(ctx, img, ws, T);
    Phase ph(ctx, "brute_dense");
    if (tc_path(ctx, img, T)) {
        RowSet rs;
        rs.lo = 0;
        rs.hi = er;
        tmk::TcTask task{};
        task.mode = 0;
        task.c_lim = ec;
        task.c_last = -1;
        task.out_rho = surface;
        ctx->partials.ensure(148 + 1);
        const int np = tc_run(ctx, img, ws, T, rs, 1, task);
        reduce_to(ctx, np, 2);
    } else if (fp32_path(img, T)) {
        std::vector<int> rows(er);
        for (int r = 0; r < er; ++r) rows[r] = r;
        upload_rows(ctx, rows);
        tmk::BandTask t{};
        t.rows = ctx->rows_list.p;
        t.nrows = er;
        t.cbase = 0;
        t.sw = 1;
        t.nc = ec;
        t.mode = 0;
        t.row_span = 7;
        t.ksplit = 1;
        t.ms = T.m;
        t.ksplit = 1;
        t.ms = T.m;
        t.out_rho = surface;
        ctx->partials.ensure(size_t(band_partials(er, ec, 1)));
        int np = 0;
        CK(tmk::corr_band(band_job(ctx, img, job), t, ctx->partials.p, &np, ctx->s));
        ctx->add(1);
        reduce_to(ctx, np, 2);
    } else if (!surface && split_path(ctx, img, T, double(E) * T.m * T.n, 67108864.0) &&
               brute_split(ctx, img, ws, T)) {
        // screened on the tensor cores, the near-maximal locations re-evaluated exactly
    } else {
        ctx->partials.ensure(kListBlocks);
        CK(tmk::corr_dense_f64(job, surface, ctx->partials.p, kListBlocks, ctx->s));
        ctx->add(1);
        reduce_to(ctx, kListBlocks, 2);
    }
    tmk::CellH best;
    CK(cudaMemcpyAsync(&best, ctx->cells.p + 2, sizeof best, cudaMemcpyDeviceToHost, ctx->s));
    if (surface_host)
        CK(cudaMemcpyAsync(surface_host, surface, E * 8, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    tm_match_result r{};
    r.mode = TM_MODE_BRUTE;
    r.extent_rows = er;
    r.extent_cols = ec;
    r.best_row = r.refined_row = best.row;
    r.best_col = r.refined_col = best.col;
    r.best_rho = r.refined_rho = best.rho;
    r.best_degenerate = (best.flags & 2) != 0;
    r.final_threshold = r.best_degenerate ? 0.0 : best.rho;
    r.retained = (long long)er * ec;
    r.ops = (long long)er * ec;
    return r;
}

std::vector<double> params_profile(const tm_match_params& P) {
    if (!P.kernel_profile || P.kernel_len < 1) return {0.05, 0.20, 0.50, 0.20, 0.05};
    if (P.kernel_len % 2 == 0) invalid("blur kernel profile must have odd length");
    return std::vector<double>(P.kernel_profile, P.kernel_profile + P.kernel_len);
}

tm_prep* prepare(tm_ctx* ctx, tm_image* img, int m, int n, const tm_match_params& P,
                 const std::function<void()>* before_sync = nullptr, bool timed = true) {
    auto prep = std::make_unique<tm_prep>();
    prep->params = P;
    prep->profile = params_profile(P);
    prep->params.kernel_profile = nullptr;
    prep->m = m;
    prep->n = n;
    prep->source = img;
    prep->mode = P.mode == TM_MODE_OPTA ? TM_MODE_OPTA : TM_MODE_EGS;
    if (m > img->p || n > img->q) invalid("match: template larger than search image");
    // (tm_search skips the timing events: an event record between two kernels breaks the
    // programmatic-launch chain of the search that follows)
    if (timed) {
        CK(cudaEventCreate(&prep->ev0));
        CK(cudaEventCreate(&prep->ev1));
        CK(cudaEventRecord(prep->ev0, ctx->s));
    }
    if (prep->mode == TM_MODE_EGS) {
        WS& ws = get_ws(ctx, img, m, n);
        EgsOut e = run_egs_search(ctx, img, ws, m, n, P.h0, P.w0, P.rho_th, P.xi_fraction,
                                  P.max_group, prep->map, before_sync);
        prep->h = e.h;
        prep->w = e.w;
        prep->cost = e.cost;
        prep->egs_trace = e.trace;
    } else {
        run_opta_prep(ctx, img, prep.get());
    }
    if (timed) CK(cudaEventRecord(prep->ev1, ctx->s));
    prep->g = make_grid(img->p - m + 1, img->q - n + 1, prep->h, prep->w);
    HT("prep_end");
    return prep.release();
}

tm_match_result run_uploaded(tm_ctx* ctx, tm_prep* prep, tm_image* img, const Tmpl& T,
                             const tm_match_params& P, uint8_t* visits);

tm_match_result run_one(tm_ctx* ctx, tm_prep* prep, tm_image* img, const double* t,
                        const tm_match_params& P, uint8_t* visits) {
    HT("start");
    const Tmpl T = upload_template(ctx, t, prep->m, prep->n);
    HT("template");
    return run_uploaded(ctx, prep, img, T, P, visits);
}

// run_egs / run_opta with the template already uploaded (ctx->tf / ctx->td).
tm_match_result run_uploaded(tm_ctx* ctx, tm_prep* prep, tm_image* img, const Tmpl& T,
                             const tm_match_params& P, uint8_t* visits) {
    const int m = prep->m, n = prep->n;
    tm_image* search_img = prep->search_img ? prep->search_img.get() : img;
    const WS* ws = prep->search_img ? prep->search_ws.get() : &get_ws(ctx, img, m, n);
    SearchIn in{search_img, ws, prep->g, prep->map.p};
    tm_match_result r = search(ctx, in, T, P, visits);
    HT("search_end");
    htrace().flush("run");
    if (prep->mode == TM_MODE_OPTA) {
        r.mode = TM_MODE_OPTA;
        const int d = prep->kappa * prep->radius;
        long long rops = 0;
        WS& ws_orig = get_ws(ctx, img, m, n);
        const tmk::CellH c = refine(ctx, img, ws_orig, T, r.best_row, r.best_col, d, &rops);
        r.refined_row = c.row;
        r.refined_col = c.col;
        r.refined_rho = c.rho;
        r.ops += rops;
        if (P.has_init_threshold)
            r.below_threshold = (c.flags & 2) || c.rho < P.init_threshold;
    }
    return r;
}

template <class F>
int guard(tm_ctx* ctx, F&& f) {
    try {
        if (ctx) {
            std::lock_guard<std::mutex> lk(ctx->mu);
            CK(cudaSetDevice(ctx->device));
            g_stream = ctx->s;
            f();
            if (ctx->profiling) {
                CK(cudaStreamSynchronize(ctx->s));
                ctx->resolve();
            }
        } else {
            f();
        }
        return TM_OK;
    } catch (const TmError& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return TM_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TM_EINVAL;
    }
}

}  // namespace

// Actually free a context (no dependents left).
void ctx_release(tm_ctx* ctx) {
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->s;
    cudaStreamSynchronize(st);
    cudaEventDestroy(ctx->ev0);
    cudaEventDestroy(ctx->ev1);
    for (cudaEvent_t ev : ctx->pool) cudaEventDestroy(ev);
    if (ctx->s2) {
        cudaStreamSynchronize(ctx->s2);
        cudaStreamDestroy(ctx->s2);
    }
    if (ctx->ev_t) cudaEventDestroy(ctx->ev_t);
    if (ctx->ev_egs) cudaEventDestroy(ctx->ev_egs);
    if (ctx->ev_b0) cudaEventDestroy(ctx->ev_b0);
    if (ctx->ev_b1) cudaEventDestroy(ctx->ev_b1);
    if (ctx->hres) cudaFreeHost(ctx->hres);
    if (ctx->s_up) {
        cudaStreamSynchronize(ctx->s_up);
        cudaStreamDestroy(ctx->s_up);
    }
    for (int k = 0; k < 2; ++k) {
        if (ctx->ev_up[k]) cudaEventDestroy(ctx->ev_up[k]);
        if (ctx->ev_free[k]) cudaEventDestroy(ctx->ev_free[k]);
    }
    delete ctx;  // stream-ordered frees of the scratch buffers
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
}

void ctx_unref(tm_ctx* ctx) {
    if (ctx && --ctx->refs == 0 && ctx->closing) ctx_release(ctx);
}

// ==== C ABI ===========================================================================
extern "C" {

const char* tm_last_error(void) { return g_err.c_str(); }

void tm_default_params(tm_match_params* p) {
    std::memset(p, 0, sizeof *p);
    p->mode = TM_MODE_EGS;
    p->h0 = 3;
    p->w0 = 3;
    p->rho_th = 0.8;
    p->rho_max = 0.95;
    p->xi_fraction = 0.005;
    p->opta_margin = 0.005;
    p->kernel_profile = nullptr;  // default {.05,.2,.5,.2,.05}
    p->kernel_len = 0;
    p->parallel = 0;
    p->threads = 2;
    p->policy = TM_POLICY_REFERENCE;
    p->max_group = 127;
    p->seed_margin = 0.02;
}

int tm_ctx_create(int device, tm_ctx** out) {
    return guard(nullptr, [&] {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw TmError{TM_ENODEV, "no CUDA device available (the tmatch path is GPU-only)"};
        if (device < 0 || device >= ndev) invalid("tm_ctx_create: bad device index");
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            throw TmError{TM_ENODEV, "tmatch kernels are built for sm_100a (Blackwell)"};
        auto ctx = std::make_unique<tm_ctx>();
        ctx->device = device;
        if (const char* e = std::getenv("TMATCH_AUTOCORR")) ctx->ac_fused = std::strcmp(e, "colwalk") != 0;
        if (const char* e = std::getenv("TMATCH_WSTATS")) ctx->ws4 = std::strcmp(e, "column") != 0;
        if (const char* e = std::getenv("TMATCH_TC")) ctx->tc = std::strcmp(e, "0") != 0;
        if (const char* e = std::getenv("TMATCH_TC_SPLIT")) ctx->tc_split = std::atoi(e);
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&ctx->s, cudaStreamNonBlocking));
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = UINT64_MAX;  // keep freed blocks cached in the pool
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        g_stream = ctx->s;
        CK(cudaEventCreate(&ctx->ev0));
        CK(cudaEventCreate(&ctx->ev1));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->hres), sizeof(tm_ctx::HostRes),
                         cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->hres_dev), ctx->hres, 0));
        CK(cudaStreamCreateWithFlags(&ctx->s2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->ev_t, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_egs, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_b0, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_b1, cudaEventDisableTiming));
        ctx->counters.ensure(40);
        CK(cudaMemsetAsync(ctx->counters.p, 0, 40 * sizeof(unsigned long long), ctx->s));
        ctx->cells.ensure(8);
        ctx->thr.ensure(2);
        ctx->tally.ensure(1);
        *out = ctx.release();
    });
}

void tm_ctx_destroy(tm_ctx* ctx) {
    if (!ctx) return;
    ctx->closing = true;
    if (ctx->refs.load() == 0) ctx_release(ctx);
}

int tm_ctx_synchronize(tm_ctx* ctx) {
    return guard(ctx, [&] { CK(cudaStreamSynchronize(ctx->s)); });
}

int64_t tm_ctx_launch_count(const tm_ctx* ctx) { return ctx ? ctx->launches : 0; }

int tm_ctx_search_stats(const tm_ctx* ctx, int64_t* fused_hits, int64_t* fused_misses) {
    if (!ctx || !fused_hits || !fused_misses) return TM_EINVAL;
    *fused_hits = ctx->fused_hits;
    *fused_misses = ctx->fused_misses;
    return TM_OK;
}

int tm_ctx_split_stats(const tm_ctx* ctx, int64_t* screened, int64_t* exact) {
    if (!ctx || !screened || !exact) return TM_EINVAL;
    *screened = ctx->split_screened + ctx->split_centres;
    *exact = ctx->split_exact;
    return TM_OK;
}

void* tm_ctx_stream(tm_ctx* ctx) { return ctx ? reinterpret_cast<void*>(ctx->s) : nullptr; }

int tm_ctx_set_profiling(tm_ctx* ctx, int enable) {
    return guard(ctx, [&] {
        ctx->profiling = enable != 0;
        ctx->phase_ms.clear();
    });
}

int tm_ctx_phase_times(tm_ctx* ctx, char* buf, size_t len) {
    return guard(ctx, [&] {
        std::string js = "{";
        bool first = true;
        for (auto& kv : ctx->phase_ms) {
            char item[160];
            std::snprintf(item, sizeof item, "%s\"%s\": [%lld, %.6f]", first ? "" : ", ",
                          kv.first.c_str(), kv.second.first, kv.second.second);
            js += item;
            first = false;
        }
        js += "}";
        if (js.size() + 1 > len) invalid("tm_ctx_phase_times: buffer too small");
        std::memcpy(buf, js.c_str(), js.size() + 1);
    });
}

int tm_image_reset_cache(tm_image* img) {
    if (!img) return TM_EINVAL;
    tm_ctx* ctx = img->ctx;
    return guard(ctx, [&] {
        invalidate_ws(img);
        img->have_qtotal = false;
    });
}

int tm_image_create(tm_ctx* ctx, const double* pixels, int rows, int cols, tm_image** out) {
    return guard(ctx, [&] {
        if (rows < 1 || cols < 1) invalid("image dimensions must be at least 1x1");
        auto img = std::make_unique<tm_image>();
        img->ctx = ctx;
        img->p = rows;
        img->q = cols;
        const size_t N = size_t(rows) * cols;
        img->f64.ensure(N);
        ++ctx->refs;
        CK(cudaMemcpyAsync(img->f64.p, pixels, N * 8, cudaMemcpyHostToDevice, ctx->s));
        classify_device_image(ctx, img.get());
        *out = img.release();
    });
}

int tm_image_create_u8(tm_ctx* ctx, const uint8_t* pixels, int rows, int cols, tm_image** out) {
    return guard(ctx, [&] {
        if (rows < 1 || cols < 1) invalid("image dimensions must be at least 1x1");
        auto img = std::make_unique<tm_image>();
        img->ctx = ctx;
        img->p = rows;
        img->q = cols;
        img->integer = true;
        ++ctx->refs;
        const size_t N = size_t(rows) * cols;
        alloc_u8(ctx, img.get());
        CK(cudaMemcpyAsync(img->u8.p, pixels, N, cudaMemcpyHostToDevice, ctx->s));
        finish_integer_image(ctx, img.get());
        CK(cudaStreamSynchronize(ctx->s));
        *out = img.release();
    });
}

int tm_image_upload_u8(tm_ctx* ctx, tm_image* img, const uint8_t* pixels) {
    return guard(ctx, [&] {
        if (!img->integer) invalid("tm_image_upload_u8: image is not an 8-bit image");
        const size_t N = size_t(img->p) * img->q;
        CK(cudaMemcpyAsync(img->u8.p, pixels, N, cudaMemcpyHostToDevice, ctx->s));
        img->have_f32 = false;
        img->have_f64 = false;
        img->have_qtotal = false;
        tc_pitch_copy(ctx, img);
        invalidate_ws(img);
    });
}

int tm_image_create_strip_u8(tm_ctx* ctx, int rows, int cols, int row0, int nrows,
                             const uint8_t* pixels, tm_image** out) {
    return guard(ctx, [&] {
        if (rows < 1 || cols < 1) invalid("image dimensions must be at least 1x1");
        if (row0 < 0 || nrows < 1 || row0 + nrows > rows)
            invalid("tm_image_create_strip_u8: rows outside the image");
        auto img = std::make_unique<tm_image>();
        img->ctx = ctx;
        img->p = rows;
        img->q = cols;
        img->integer = true;
        img->row_lo = row0;
        img->row_hi = row0 + nrows;
        ++ctx->refs;
        alloc_u8(ctx, img.get());
        CK(cudaMemsetAsync(img->u8.p, 0, size_t(rows) * cols, ctx->s));
        CK(cudaMemcpyAsync(img->u8.p + size_t(row0) * cols, pixels, size_t(nrows) * cols,
                           cudaMemcpyHostToDevice, ctx->s));
        finish_integer_image(ctx, img.get());
        CK(cudaStreamSynchronize(ctx->s));
        *out = img.release();
    });
}

int tm_image_upload_strip_u8(tm_ctx* ctx, tm_image* img, const uint8_t* pixels) {
    return guard(ctx, [&] {
        if (!img || !img->integer) invalid("tm_image_upload_strip_u8: not an 8-bit image");
        const int nrows = std::min(img->row_hi, img->p) - img->row_lo;
        CK(cudaMemcpyAsync(img->u8.p + size_t(img->row_lo) * img->q, pixels,
                           size_t(nrows) * img->q, cudaMemcpyHostToDevice, ctx->s));
        img->have_f32 = false;
        img->have_f64 = false;
        if (!img->noise_external) img->have_qtotal = false;
        tc_pitch_copy(ctx, img);
        invalidate_ws(img);
    });
}

int tm_image_sum_sq_rows(tm_ctx* ctx, tm_image* img, int row0, int nrows, uint64_t* q_sum) {
    return guard(ctx, [&] {
        if (!img || !img->integer || !q_sum) invalid("tm_image_sum_sq_rows: needs an 8-bit image");
        if (row0 < img->row_lo || row0 + nrows > std::min(img->row_hi, img->p) || nrows < 0)
            invalid("tm_image_sum_sq_rows: rows outside the pixels held");
        unsigned long long* d = ctx->counters.p + 30;
        CK(tmk::sum_sq_rows_u8(img->u8.p, img->q, row0, nrows, d, ctx->s));
        ctx->add(1);
        unsigned long long v = 0;
        CK(cudaMemcpyAsync(&v, d, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        *q_sum = v;
    });
}

int tm_image_set_noise_floor(tm_ctx* ctx, tm_image* img, uint64_t q_total) {
    return guard(ctx, [&] {
        if (!img || !img->integer) invalid("tm_image_set_noise_floor: needs an 8-bit image");
        // stats.cpp:80-81 with the GLOBAL rows + cols and sum of squares (exact for 8-bit
        // data: q_total < 2^53)
        const double pn = double(img->p + img->q) * 2.220446049250313e-16 * double(q_total);
        img->pn.ensure(8);
        CK(cudaMemcpyAsync(img->pn.p + 1, &pn, 8, cudaMemcpyHostToDevice, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        img->noise_external = true;
        img->have_qtotal = true;
        invalidate_ws(img);
    });
}

int tm_image_download(tm_ctx* ctx, const tm_image* cimg, double* out) {
    tm_image* img = const_cast<tm_image*>(cimg);
    return guard(ctx, [&] {
        const size_t N = size_t(img->p) * img->q;
        if (!img->have_f64) ensure_f64(ctx, img);
        CK(cudaMemcpyAsync(out, img->f64.p, N * 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    });
}

int tm_image_is_integer(const tm_image* img) { return img && img->integer ? 1 : 0; }

void tm_image_destroy(tm_image* img) {
    if (!img) return;
    tm_ctx* ctx = img->ctx;
    if (ctx) {
        {
            // stream-ordered frees (cudaFreeAsync on the context stream): no sync needed
            std::lock_guard<std::mutex> lk(ctx->mu);
            cudaSetDevice(ctx->device);
            g_stream = ctx->s;
            delete img;
        }
        ctx_unref(ctx);
    } else {
        delete img;
    }
}

int tm_running_sum(tm_ctx* ctx, tm_image* img, int m, int n, double* out) {
    return guard(ctx, [&] {
        const int p = img->p, q = img->q;
        if (m < 1 || n < 1 || m > p || n > q) invalid("running_sum: window does not fit the source");
        const size_t E = size_t(p - m + 1) * (q - n + 1);
        ctx->S.ensure(E);
        if (img->integer) {
            ctx->hs.ensure(size_t(p) * (q - n + 1));
            CK(tmk::window_sums_u8(img->u8.p, p, q, m, n, ctx->hs.p, ctx->S.p, ctx->s));
            ctx->add(2);
        } else {
            replica_sums(ctx, tmk::ProdSrc{img->f64.p, q, 0, 0, nullptr, 0, 0, 0, 0}, p, q, m, n,
                         ctx->S.p);
        }
        CK(cudaMemcpyAsync(out, ctx->S.p, E * 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    });
}

int tm_window_stats(tm_ctx* ctx, tm_image* img, int m, int n, double* mu, double* omega,
                    uint8_t* flat) {
    return guard(ctx, [&] {
        WS& ws = get_ws(ctx, img, m, n);
        const size_t E = size_t(ws.er) * ws.ec;
        if (mu) CK(cudaMemcpyAsync(mu, ws.mu.p, E * 8, cudaMemcpyDeviceToHost, ctx->s));
        if (omega) CK(cudaMemcpyAsync(omega, ws.om.p, E * 8, cudaMemcpyDeviceToHost, ctx->s));
        if (flat) CK(cudaMemcpyAsync(flat, ws.fl.p, E, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    });
}

int tm_brute_force_match(tm_ctx* ctx, const double* tmpl, int m, int n, tm_image* img,
                         tm_match_result* out, double* surface) {
    return guard(ctx, [&] {
        if (m > img->p || n > img->q)
            invalid("brute_force_match: template larger than search image");
        CK(cudaEventRecord(ctx->ev0, ctx->s));
        const Tmpl T = upload_template(ctx, tmpl, m, n);
        *out = brute(ctx, img, T, surface);
        CK(cudaEventRecord(ctx->ev1, ctx->s));
        CK(cudaEventSynchronize(ctx->ev1));
        out->wall_ms = ms_between(ctx->ev0, ctx->ev1);
    });
}

int tm_local_autocorrelation(tm_ctx* ctx, tm_image* img, int m, int n, int h, int w,
                             double* map) {
    return guard(ctx, [&] {
        if (m > img->p || n > img->q) invalid("group grid: template does not fit the image");
        const tmk::GridDesc g = make_grid(img->p - m + 1, img->q - n + 1, h, w);
        WS& ws = get_ws(ctx, img, m, n);
        const size_t E = size_t(g.er) * g.ec;
        ctx->map_user.ensure(E);
        autocorr_map(ctx, img, ws, g, 0.6, ctx->map_user.p);
        CK(cudaMemcpyAsync(map, ctx->map_user.p, E * 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    });
}

int tm_autocorr_retained(tm_ctx* ctx, tm_image* img, int m, int n, int h, int w, double rho_tb,
                         int64_t* n_r) {
    return guard(ctx, [&] {
        if (rho_tb < 0.0 || rho_tb > 1.0) invalid("retained_count: rho_tb must be in [0,1]");
        if (m > img->p || n > img->q) invalid("group grid: template does not fit the image");
        const tmk::GridDesc g = make_grid(img->p - m + 1, img->q - n + 1, h, w);
        WS& ws = get_ws(ctx, img, m, n);
        ctx->map_user.ensure(size_t(g.er) * g.ec);
        *n_r = autocorr_map(ctx, img, ws, g, expected_elimination_threshold_h(rho_tb),
                            ctx->map_user.p, /*count_only=*/true);
    });
}

int tm_efficient_group_size(tm_ctx* ctx, tm_image* img, int m, int n, int h0, int w0,
                            double rho_tb, double xi_fraction, int max_group, int* h, int* w,
                            tm_egs_iter* trace, int* trace_len, double* map) {
    return guard(ctx, [&] {
        if (m > img->p || n > img->q) invalid("efficient_group_size: template does not fit");
        WS& ws = get_ws(ctx, img, m, n);
        DBuf<double> best;
        EgsOut e = run_egs_search(ctx, img, ws, m, n, h0, w0, rho_tb, xi_fraction, max_group, best);
        *h = e.h;
        *w = e.w;
        *trace_len = int(e.trace.size());
        for (size_t k = 0; k < e.trace.size() && k < TM_MAX_TRACE; ++k) trace[k] = e.trace[k];
        if (map)
            CK(cudaMemcpyAsync(map, best.p, size_t(ws.er) * ws.ec * 8, cudaMemcpyDeviceToHost,
                               ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    });
}

int tm_blur(tm_ctx* ctx, tm_image* img, const double* profile, int len, double* out) {
    return guard(ctx, [&] {
        if (len < 1 || len % 2 == 0) invalid("blur kernel profile must have odd length");
        ensure_f64(ctx, img);
        const size_t N = size_t(img->p) * img->q;
        if (len == 1) {
            CK(cudaMemcpyAsync(out, img->f64.p, N * 8, cudaMemcpyDeviceToHost, ctx->s));
        } else {
            ctx->prof.ensure(len);
            ctx->dtmp.ensure(N);
            ctx->rowacc.ensure(N);
            CK(cudaMemcpyAsync(ctx->prof.p, profile, len * 8, cudaMemcpyHostToDevice, ctx->s));
            CK(tmk::blur_replica(img->f64.p, img->p, img->q, ctx->prof.p, len, ctx->dtmp.p,
                                 ctx->rowacc.p, ctx->s));
            ctx->add(2);
            CK(cudaMemcpyAsync(out, ctx->rowacc.p, N * 8, cudaMemcpyDeviceToHost, ctx->s));
        }
        CK(cudaStreamSynchronize(ctx->s));
    });
}

int tm_blur_fidelity_map(tm_ctx* ctx, tm_image* img, tm_image* blurred, int m, int n,
                         double* fid) {
    return guard(ctx, [&] {
        if (img->p != blurred->p || img->q != blurred->q)
            invalid("blur_fidelity_map: dimension mismatch");
        WS& ws_o = get_ws(ctx, img, m, n);
        ensure_f64(ctx, img);
        ensure_f64(ctx, blurred);
        WS ws_b;
        ctx->fid.ensure(size_t(ws_o.er) * ws_o.ec);
        // the blurred image's stats must come from the FP64 replica (window_stats on I_blur)
        const bool was_int = blurred->integer;
        blurred->integer = false;
        fidelity(ctx, img, ws_o, blurred, ws_b, ctx->fid.p);
        blurred->integer = was_int;
        blurred->have_qtotal = false;
        CK(cudaMemcpyAsync(fid, ctx->fid.p, size_t(ws_o.er) * ws_o.ec * 8, cudaMemcpyDeviceToHost,
                           ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    });
}

int tm_unblur_violations(tm_ctx* ctx, tm_image* blurred, tm_image* original, const double* fid,
                         int m, int n, double lambda, double* out, int64_t* count) {
    return guard(ctx, [&] {
        if (blurred->p != original->p || blurred->q != original->q)
            invalid("unblur_violations: shape mismatch");
        const int p = original->p, q = original->q;
        const int er = p - m + 1, ec = q - n + 1;
        if (er < 1 || ec < 1) invalid("unblur_violations: window does not fit");
        const size_t E = size_t(er) * ec, N = size_t(p) * q;
        ensure_f64(ctx, blurred);
        ensure_f64(ctx, original);
        ctx->fid.ensure(E);
        ctx->marks.ensure(E);
        ctx->markP.ensure(size_t(er + 1) * (ec + 1));
        ctx->dtmp.ensure(N);
        CK(cudaMemcpyAsync(ctx->fid.p, fid, E * 8, cudaMemcpyHostToDevice, ctx->s));
        CK(cudaMemcpyAsync(ctx->dtmp.p, blurred->f64.p, N * 8, cudaMemcpyDeviceToDevice, ctx->s));
        // blur.cpp:188-199: mark every location below lambda, then restore their windows
        CK(tmk::mark_violations(ctx->fid.p, nullptr, E, lambda, ctx->marks.p,
                                ctx->counters.p + 3, ctx->s));
        CK(tmk::restore_covered(ctx->dtmp.p, original->f64.p, ctx->marks.p, er, ec, m, n, p, q,
                                ctx->markP.p, ctx->s));
        ctx->add(4);
        unsigned long long c = 0;
        CK(cudaMemcpyAsync(&c, ctx->counters.p + 3, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaMemcpyAsync(out, ctx->dtmp.p, N * 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        *count = (int64_t)c;
    });
}

int tm_prepare(tm_ctx* ctx, tm_image* img, int m, int n, const tm_match_params* params,
               tm_prep** out) {
    return guard(ctx, [&] {
        *out = prepare(ctx, img, m, n, *params);
        (*out)->ctx = ctx;
        ++ctx->refs;
    });
}

int tm_prep_get_info(const tm_prep* prep, tm_prep_info* info) {
    return guard(nullptr, [&] {
        std::memset(info, 0, sizeof *info);
        info->mode = prep->mode;
        info->m = prep->m;
        info->n = prep->n;
        info->h = prep->h;
        info->w = prep->w;
        info->extent_rows = prep->g.er;
        info->extent_cols = prep->g.ec;
        info->kappa = prep->kappa;
        info->lambda = prep->lambda;
        info->cost = prep->cost;
        info->egs_trace_len = int(prep->egs_trace.size());
        for (size_t k = 0; k < prep->egs_trace.size() && k < TM_MAX_TRACE; ++k)
            info->egs_trace[k] = prep->egs_trace[k];
        info->opta_trace_len = int(prep->opta_trace.size());
        for (size_t k = 0; k < prep->opta_trace.size() && k < TM_MAX_TRACE + 1; ++k)
            info->opta_trace[k] = prep->opta_trace[k];
        if (prep->prep_ms < 0 && prep->ev1) {
            cudaEventSynchronize(prep->ev1);
            const_cast<tm_prep*>(prep)->prep_ms = ms_between(prep->ev0, prep->ev1);
        }
        info->prep_ms = prep->prep_ms;
    });
}

int tm_prep_download(tm_ctx* ctx, const tm_prep* prep, double* map, double* image) {
    return guard(ctx, [&] {
        const size_t E = size_t(prep->g.er) * prep->g.ec;
        if (map) CK(cudaMemcpyAsync(map, prep->map.p, E * 8, cudaMemcpyDeviceToHost, ctx->s));
        if (image) {
            tm_image* src = prep->search_img ? prep->search_img.get() : prep->source;
            ensure_f64(ctx, src);
            CK(cudaMemcpyAsync(image, src->f64.p, size_t(src->p) * src->q * 8,
                               cudaMemcpyDeviceToHost, ctx->s));
        }
        CK(cudaStreamSynchronize(ctx->s));
    });
}

void tm_prep_destroy(tm_prep* prep) {
    if (!prep) return;
    tm_ctx* ctx = prep->ctx;
    if (ctx) {
        {
            std::lock_guard<std::mutex> lk(ctx->mu);
            cudaSetDevice(ctx->device);
            g_stream = ctx->s;
            delete prep;
        }
        ctx_unref(ctx);
    } else {
        delete prep;
    }
}

// ---- template batches ---------------------------------------------------------------------
// run_egs / run_opta for K templates of one preparation (cmd_bench's loop over a cached
// preparation, cli.cpp:213-237) as one device pipeline with ONE host synchronisation:
//   1. per template: scan 1 (tensor-core centre scan) + threshold bootstrap [+ seeding],
//      its group-level results copied to the template's slot;
//   2. one bound pass for all K templates (k_sec_rows_multi): every member's R_co and flat
//      flag are read once;
//   3. per template: survivor evaluation (dense tensor-core pass or list) and the packed
//      result, then one readback of all K results.
// Same results and counts as K separate runs (frozen / seeded policies on the 8-bit
// tensor-core path; other cases take the per-template loop).
bool batch_applies(tm_ctx* ctx, tm_prep* prep, tm_image* img, const double* tmpls, int K,
                   const tm_match_params& P, const uint8_t* visits) {
    if (K < 2 || K > tmk::kMaxBatch || visits || P.record_visits) return false;
    int policy = P.policy;
    const size_t G = size_t(prep->g.tr) * prep->g.tc;
    if (policy == TM_POLICY_REFERENCE)
        policy = (P.parallel && P.threads > 1 && G > 1) ? TM_POLICY_FROZEN : TM_POLICY_SEQUENTIAL;
    if (policy != TM_POLICY_FROZEN && policy != TM_POLICY_SEEDED) return false;
    tm_image* simg = prep->search_img ? prep->search_img.get() : img;
    if (prep->g.h > tmk::kTcMaxClasses || !prep->map.p) return false;
    const size_t mn = size_t(prep->m) * prep->n;
    for (int k = 0; k < K; ++k) {
        const Tmpl T = template_host_stats(tmpls + k * mn, prep->m, prep->n);
        if (T.ts.flat || !tc_path(ctx, simg, T)) return false;
    }
    return true;
}

void run_batch(tm_ctx* ctx, tm_prep* prep, tm_image* img, const double* tmpls, int K,
               const tm_match_params& P, tm_match_result* out) {
    const int m = prep->m, n = prep->n;
    const size_t mn = size_t(m) * n;
    tm_image* simg = prep->search_img ? prep->search_img.get() : img;
    const WS& ws = prep->search_img ? *prep->search_ws : get_ws(ctx, img, m, n);
    const tmk::GridDesc g = prep->g;
    const size_t E = size_t(g.er) * g.ec, G = size_t(g.tr) * g.tc;
    cudaStream_t s = ctx->s;
    int policy = P.policy;
    if (policy == TM_POLICY_REFERENCE) policy = TM_POLICY_FROZEN;  // (batch_applies checked)
    const bool seeded_pol = policy == TM_POLICY_SEEDED;
    auto& B = ctx->batch;
    // templates: host statistics, one upload of all K (FP32 rows padded, FP64)
    std::vector<Tmpl> Ts(K);
    const int npad = (n + 15) & ~15;
    std::vector<float> tf(size_t(K) * m * npad, 0.f);
    for (int k = 0; k < K; ++k) {
        Ts[k] = template_host_stats(tmpls + k * mn, m, n);
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < n; ++j)
                tf[(size_t(k) * m + i) * npad + j] = float(tmpls[k * mn + size_t(i) * n + j]);
    }
    B.tf.ensure(tf.size());
    B.td.ensure(size_t(K) * mn);
    B.pin_tf.upload(B.tf.p, tf.data(), tf.size() * 4, s);
    B.pin_td.upload(B.td.p, tmpls, size_t(K) * mn * 8, s);
    for (int k = 0; k < K; ++k) {
        Ts[k].tf = B.tf.p + size_t(k) * m * npad;
        Ts[k].td = B.td.p + size_t(k) * mn;
    }
    B.rho.ensure(size_t(K) * G);
    B.sa.ensure(size_t(K) * G);
    B.rec.ensure(size_t(K) * G);
    B.thr.ensure(size_t(K));
    B.cells.ensure(size_t(K) * 3);
    B.tally.ensure(size_t(K));
    B.vis.ensure(size_t(K) * E);
    const unsigned long long cap = E / tmk::kDenseDiv + 1;  // longer lists go dense
    B.locs.ensure(size_t(K) * cap);
    B.packed.ensure(size_t(K));

    // 1. scan 1 (+ seeding) per template; the tensor-core centre epilogue writes the
    //    template's batch records directly, the seeding marks its seeded groups in them
    //    (the centres' window statistics are gathered once for the whole batch)
    ctx->cs_mu.ensure(G);
    ctx->cs_om.ensure(G);
    ctx->cs_fl.ensure(G);
    CK(tmk::gather_centre_stats(g, ws.dev(),
                                tmk::CentreStats{ctx->cs_mu.p, ctx->cs_om.p, ctx->cs_fl.p}, s));
    ctx->add(1);
    for (int k = 0; k < K; ++k) {
        const Tmpl& T = Ts[k];
        const tmk::ReduceOp op_init = centre_op(ctx, P);
        float2* recs = B.rec.p + size_t(k) * G;
        ctx->batch_rec = recs;
        ctx->batch_cs = true;
        centre_scan(ctx, simg, ws, T, g, &op_init);
        ctx->batch_rec = nullptr;
        ctx->batch_cs = false;
        const bool recs_written = ctx->sa_ready;  // (the tensor-core epilogue ran)
        if (!ctx->sa_ready) {  // (the tensor-core epilogue writes it; keep the invariant)
            CK(tmk::sqrt_gap(ctx->rho_c.p, ctx->sa_c.p, G, s));
            ctx->add(1);
        }
        if (seeded_pol) {
            const unsigned long long max_groups = 256;
            const unsigned long long max_locs = max_groups * (unsigned long long)(g.h * g.w);
            ctx->seed_locs.ensure(max_locs);
            ctx->seeded.ensure(G);
            CK(tmk::seed_members(g, ctx->rho_c.p, ctx->deg_c.p, ctx->thr.p, P.seed_margin,
                                 ctx->seeded.p, ctx->seed_locs.p, ctx->counters.p + 4, max_locs,
                                 ctx->counters.p + 5, max_groups, s,
                                 recs_written ? recs : nullptr));
            ctx->add(1);
            tmk::ReduceOp op_raise{};
            op_raise.kind = 2;
            op_raise.thr = ctx->thr.p;
            eval_list(ctx, simg, ws, T, ctx->seed_locs.p, ctx->counters.p + 4, int(max_locs),
                      nullptr, nullptr, 1, &op_raise);
        }
        CK(cudaMemcpyAsync(B.rho.p + size_t(k) * G, ctx->rho_c.p, G * 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(B.sa.p + size_t(k) * G, ctx->sa_c.p, G * 8, cudaMemcpyDeviceToDevice, s));
        if (!recs_written) {
            CK(tmk::batch_records(ctx->rho_c.p, ctx->sa_c.p, ctx->deg_c.p,
                                  seeded_pol ? ctx->seeded.p : nullptr, G, recs, s));
            ctx->add(1);
        }
        CK(cudaMemcpyAsync(B.thr.p + k, ctx->thr.p, 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(B.cells.p + 3 * k, ctx->cells.p, 2 * sizeof(tmk::CellH),
                           cudaMemcpyDeviceToDevice, s));
    }
    // 2. one bound pass for every template
    CK(cudaMemsetAsync(B.tally.p, 0, size_t(K) * sizeof(tmk::Tally), s));
    tmk::SecMulti sm;
    sm.K = K;
    sm.G = G;
    sm.E = E;
    sm.rec = B.rec.p;
    sm.rho_c = B.rho.p;
    sm.sa_c = B.sa.p;
    sm.thr = B.thr.p;
    sm.locs = B.locs.p;
    sm.cap = cap;
    sm.tally = B.tally.p;
    sm.visits = B.vis.p;
    sm.tf = zero_tile_flags(ctx, B.tflags, g.er, g.ec, K);
    sm.tf_stride = tmk::tile_flag_bytes(g.er, g.ec);
    {
        Phase ph(ctx, "sec_multi");
        CK(tmk::sec_rows_multi(g, prep->map.p, ws.fl.p, sm, s));
        ctx->add(1);
    }
    // 3. survivors + packed result per template
    for (int k = 0; k < K; ++k) {
        CK(cudaMemcpyAsync(ctx->tally.p, B.tally.p + k, sizeof(tmk::Tally),
                           cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(ctx->thr.p, B.thr.p + k, 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(ctx->cells.p, B.cells.p + 3 * k, 2 * sizeof(tmk::CellH),
                           cudaMemcpyDeviceToDevice, s));
        const tmk::TileFlags tfk{sm.tf.p + size_t(k) * sm.tf_stride, sm.tf.cols};
        eval_survivors_dev(ctx, simg, ws, Ts[k], g, nullptr, nullptr, false,
                           B.locs.p + size_t(k) * cap, B.vis.p + size_t(k) * E, B.packed.p + k,
                           &tfk);
    }
    B.host.resize(K);
    CK(cudaMemcpyAsync(B.host.data(), B.packed.p, size_t(K) * sizeof(tmk::ResultBlock),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int k = 0; k < K; ++k) {
        const tmk::ResultBlock& hr = B.host[k];
        tmk::CellH best = hr.cells[0];
        if (seeded_pol && better_h(hr.cells[1], best)) best = hr.cells[1];
        if (better_h(hr.cells[2], best)) best = hr.cells[2];
        if (better_h(flat_cell(hr.tally), best)) best = flat_cell(hr.tally);
        double final_T = hr.thr;
        if (seeded_pol && (hr.cells[2].flags & 1) && !(hr.cells[2].flags & 2))
            final_T = std::max(final_T, hr.cells[2].rho);
        tm_match_result r{};
        r.mode = prep->mode == TM_MODE_OPTA ? TM_MODE_OPTA : TM_MODE_EGS;
        r.extent_rows = g.er;
        r.extent_cols = g.ec;
        r.best_row = r.refined_row = best.row;
        r.best_col = r.refined_col = best.col;
        r.best_rho = r.refined_rho = best.rho;
        r.best_degenerate = (best.flags & 2) != 0;
        r.final_threshold = std::isfinite(final_T) ? final_T : 0.0;
        r.below_threshold =
            P.has_init_threshold && (r.best_degenerate || best.rho < P.init_threshold);
        r.centers = (long long)G;
        r.eliminated = (long long)hr.tally.eliminated;
        r.retained = (long long)hr.tally.retained;
        r.elim_pct = 100.0 * double(r.eliminated) / (double(g.er) * double(g.ec));
        r.ops = (long long)G + r.retained;
        if (prep->mode == TM_MODE_OPTA) {  // refine_impl on the original image
            const int d = prep->kappa * prep->radius;
            long long rops = 0;
            WS& ws_orig = get_ws(ctx, img, m, n);
            const tmk::CellH c = refine(ctx, img, ws_orig, Ts[k], r.best_row, r.best_col, d, &rops);
            r.refined_row = c.row;
            r.refined_col = c.col;
            r.refined_rho = c.rho;
            r.ops += rops;
            if (P.has_init_threshold)
                r.below_threshold = (c.flags & 2) || c.rho < P.init_threshold;
        }
        out[k] = r;
    }
}

int tm_run(tm_ctx* ctx, tm_prep* prep, tm_image* img, const double* tmpls, int ntmpl,
           const tm_match_params* params, tm_match_result* out, uint8_t* visits) {
    return guard(ctx, [&] {
        if (batch_applies(ctx, prep, img, tmpls, ntmpl, *params, visits)) {
            CK(cudaEventRecord(ctx->ev0, ctx->s));
            run_batch(ctx, prep, img, tmpls, ntmpl, *params, out);
            CK(cudaEventRecord(ctx->ev1, ctx->s));
            CK(cudaEventSynchronize(ctx->ev1));
            const double ms = ms_between(ctx->ev0, ctx->ev1) / ntmpl;
            for (int k = 0; k < ntmpl; ++k) out[k].wall_ms = ms;
            return;
        }
        const size_t mn = size_t(prep->m) * prep->n;
        const size_t E = size_t(prep->g.er) * prep->g.ec;
        for (int k = 0; k < ntmpl; ++k) {
            CK(cudaEventRecord(ctx->ev0, ctx->s));
            out[k] = run_one(ctx, prep, img, tmpls + k * mn, *params, visits ? visits + k * E : nullptr);
            CK(cudaEventRecord(ctx->ev1, ctx->s));
            CK(cudaEventSynchronize(ctx->ev1));
            out[k].wall_ms = ms_between(ctx->ev0, ctx->ev1);
        }
    });
}

int tm_run_u8(tm_ctx* ctx, tm_prep* prep, tm_image* img, const uint8_t* tmpls, int ntmpl,
              const tm_match_params* params, tm_match_result* out, uint8_t* visits) {
    const size_t mn = size_t(prep->m) * prep->n;
    std::vector<double> t(mn * size_t(ntmpl));
    for (size_t i = 0; i < t.size(); ++i) t[i] = tmpls[i];
    return tm_run(ctx, prep, img, t.data(), ntmpl, params, out, visits);
}

// tm_search with scan 2 fused into the R_co launch of the predicted group size: scan 1
// and the seeding run first on the predicted grid (they need only the window statistics and
// the template), then the EGS batch, whose predicted candidate also runs the bound test on
// every member as its R_co is computed (SecFuse) -- the E-sized map is neither written nor
// read back, and the separate bound pass is gone.  If EGS accepts another size, the
// standard path reruns on the accepted grid.  Applies to EGS on 8-bit images with the
// frozen / seeded policies on the tensor-core path; returns false (nothing enqueued) when
// it does not apply.  Results, counts and visit codes are those of prepare + run.
// The first half of search_fused (scan 1 and the seeding on the predicted grid); the state
// the second half needs.  A stream of searches runs the next image's first half behind the
// current search, before the host waits for its result (tm_search_stream_u8).
struct FusedPre {
    bool ok = false;
    const tm_image* img = nullptr;
    int m = 0, n = 0, pred = 0, policy = 0;
    std::vector<double> tmpl;  // the template it was started with
    Tmpl T{};
    tmk::GridDesc g{};
    const uint8_t* seeded = nullptr;
    void swap_from(FusedPre& o) {
        std::swap(*this, o);
        o.ok = false;
    }
};

bool search_fused_begin(tm_ctx* ctx, tm_image* img, const double* tmpl, int m, int n,
                        const tm_match_params& P, int pred, FusedPre& fp) {
    fp.ok = false;
    static const bool off = [] {
        const char* e = std::getenv("TMATCH_FUSE_SCAN2");
        return e && std::strcmp(e, "0") == 0;
    }();
    if (off || P.mode == TM_MODE_OPTA || !img->integer || !ctx->ac_fused || !ctx->tc) return false;
    if (P.h0 != P.w0 || m > img->p || n > img->q) return false;
    int policy = P.policy;
    const int er = img->p - m + 1, ec = img->q - n + 1;
    const tmk::GridDesc g = make_grid(er, ec, pred, pred);
    const size_t G = size_t(g.tr) * g.tc;
    if (policy == TM_POLICY_REFERENCE)
        policy = (P.parallel && P.threads > 1 && G > 1) ? TM_POLICY_FROZEN : TM_POLICY_SEQUENTIAL;
    if (policy != TM_POLICY_SEEDED && policy != TM_POLICY_FROZEN) return false;
    if (!(img->u8p.p && img->u8p_rows >= img->p + tmk::kU8PadRows)) return false;
    if (!tmk::autocorr_sec_fuse_supported(m, n, g) || g.h > tmk::kTcMaxClasses) return false;
    // the template: exact 8-bit path (tensor cores) only
    bool t_u8 = true;
    for (size_t i = 0; i < size_t(m) * n && t_u8; ++i)
        t_u8 = tmpl[i] >= 0.0 && tmpl[i] <= 255.0 && tmpl[i] == std::rint(tmpl[i]);
    if (!t_u8) return false;
    // the 8-bit tensor-core path for this template size (tc_path / fp32_path of the Tmpl)
    if (!tmk::tc_supported(m, n) || tmk::tc_plan(m, n, 1, kTcSmemBudget).nch == 0 ||
        16777216LL / (65025LL * n) < 1)
        return false;
    if (P.has_init_threshold && std::abs(P.init_threshold) > 1.0 + 1e-9)
        invalid("transitive_search: init threshold out of [-1,1]");

    HT("fused_begin");
    // the window statistics first: the device starts while the host prepares the template;
    // the template copies and the centre scan's B build go to the side stream, overlapping
    // the statistics (tc_b sized on the main stream first: ev_b0)
    WS& ws = get_ws(ctx, img, m, n);
    HT("fused_ws");
    const tmk::TcPlan bplan = tmk::tc_plan(m, n, pred, kTcSmemBudget);
    const bool side_b = bplan.nch > 0;
    if (side_b && !(ctx->spec_b && ctx->tc_b.cap >= bplan.total_bytes)) {
        ctx->tc_b.ensure(bplan.total_bytes);  // (not sized before the statistics by b_early)
        CK(cudaEventRecord(ctx->ev_b0, ctx->s));
    }
    ctx->spec_b = false;
    const Tmpl T = upload_template(ctx, tmpl, m, n, /*side=*/true);
    if (T.ts.flat) invalid("transitive_search: constant template has no defined correlation");
    HT("fused_template");
    if (!tc_path(ctx, img, T) || !fp32_path(img, T))  // (implied by the checks above)
        throw TmError{TM_ECUDA, "search_fused: template not on the 8-bit tensor-core path"};
    // scan 1 on the predicted grid (+ threshold bootstrap, tally zeroing) and the seeding
    tmk::ReduceOp op_init = centre_op(ctx, P);
    op_init.egs_stop = reinterpret_cast<int*>(ctx->counters.p + 21);  // (k_egs_init's work)
    op_init.egs_prev = reinterpret_cast<double*>(ctx->counters.p + 20);
    op_init.egs_nr4 = ctx->counters.p + 8;
    op_init.egs_hacc = reinterpret_cast<int*>(ctx->counters.p + 25);
    op_init.egs_gate = ctx->counters.p + 24;
    centre_scan(ctx, img, ws, T, g, &op_init, side_b);
    HT("fused_centre");
    if (!ctx->sa_ready) throw TmError{TM_ECUDA, "search_fused: centre factors missing"};
    const uint8_t* seeded = nullptr;
    if (policy == TM_POLICY_SEEDED) {
        const unsigned long long max_groups = 256;
        const unsigned long long max_locs = max_groups * (unsigned long long)(g.h * g.w);
        ctx->seed_locs.ensure(max_locs);
        ctx->seeded.ensure(G);
        CK(tmk::seed_members(g, ctx->rho_c.p, ctx->deg_c.p, ctx->thr.p, P.seed_margin,
                             ctx->seeded.p, ctx->seed_locs.p, ctx->counters.p + 4, max_locs,
                             ctx->counters.p + 5, max_groups, ctx->s));
        ctx->add(1);
        tmk::ReduceOp op_raise{};
        op_raise.kind = 2;
        op_raise.thr = ctx->thr.p;
        eval_list(ctx, img, ws, T, ctx->seed_locs.p, ctx->counters.p + 4, int(max_locs), nullptr,
                  nullptr, 1, &op_raise);
        seeded = ctx->seeded.p;
    }
    HT("fused_scan1");
    fp.ok = true;
    fp.img = img;
    fp.m = m;
    fp.n = n;
    fp.pred = pred;
    fp.policy = policy;
    fp.tmpl.assign(tmpl, tmpl + size_t(m) * n);
    fp.T = T;
    fp.g = g;
    fp.seeded = seeded;
    return true;
}

// The second half: the EGS batch whose predicted candidate runs scan 2 (SecFuse), the
// survivors behind it (gated on the device decision), the result.
void search_fused_end(tm_ctx* ctx, tm_image* img, const tm_match_params& P, const FusedPre& fp,
                      tm_match_result* out) {
    const int m = fp.m, n = fp.n, pred = fp.pred;
    const int er = img->p - m + 1, ec = img->q - n + 1;
    const size_t E = size_t(er) * ec;
    const tmk::GridDesc& g = fp.g;
    const Tmpl& T = fp.T;
    WS& ws = get_ws(ctx, img, m, n);
    ctx->visits.ensure(E);
    ctx->locs.ensure(E);
    tmk::SecFuse sf{};
    sf.thr = ctx->thr.p;
    sf.rho_c = ctx->rho_c.p;
    sf.sa_c = ctx->sa_c.p;
    sf.deg_c = ctx->deg_c.p;
    sf.seeded = fp.seeded;
    sf.tflat = T.ts.flat;
    sf.locs = ctx->locs.p;
    sf.max_locs = E / 16 + 1;  // longer survivor lists go to the dense pass (visit mask)
    sf.tally = ctx->tally.p;
    sf.visits = ctx->visits.p;
    sf.tf = zero_tile_flags(ctx, ctx->tflags, g.er, g.ec);
    bool hit = false;
    // the survivor evaluation is enqueued behind the EGS batch, gated on the device decision
    // (EGS finished with h_e == pred), so the device keeps working while the host reads the
    // counts; on a miss its kernels do nothing and the standard path follows
    const unsigned long long* gate = ctx->counters.p + 24;
    const std::function<void()> hook = [&] {
        // (the dense/list choice is made by the batch's last EGS decision)
        eval_survivors_dev(ctx, img, ws, T, g, nullptr, gate, /*dispatched=*/true, nullptr,
                           nullptr, nullptr, &sf.tf);
    };
    ctx->spec_want = pred;  // the decide kernels set the gate for this size
    const EgsOut e = run_egs_search(ctx, img, ws, m, n, P.h0, P.w0, P.rho_th, P.xi_fraction,
                                    P.max_group, ctx->map_fused, &hook, &sf, &hit,
                                    /*egs_preinit=*/true);  // (search_fused_begin's centre reduction)
    ctx->spec_want = 0;
    HT("fused_egs");
    ++(hit ? ctx->fused_hits : ctx->fused_misses);
    if (hit && ctx->hres->spec != 1)
        throw TmError{TM_ECUDA, "search_fused: device gate disagrees with the EGS decision"};
    if (hit) {
        SearchIn in{img, &ws, g, nullptr};
        in.prescanned = true;
        in.survivors_enqueued = true;
        *out = search(ctx, in, T, P, nullptr);
    } else {  // EGS accepted another size: the standard scans on its grid
        const tmk::GridDesc ga = make_grid(er, ec, e.h, e.w);
        *out = search(ctx, SearchIn{img, &ws, ga, ctx->map_fused.p}, T, P, nullptr);
    }
    HT("fused_end");
    htrace().flush("search_fused");
}

// tm_search with scan 2 fused into the R_co launch of the predicted group size: scan 1
// and the seeding run first on the predicted grid (they need only the window statistics and
// the template), then the EGS batch, whose predicted candidate also runs the bound test on
// every member as its R_co is computed (SecFuse) -- the E-sized map is neither written nor
// read back, and the separate bound pass is gone.  If EGS accepts another size, the
// standard path reruns on the accepted grid.  Applies to EGS on 8-bit images with the
// frozen / seeded policies on the tensor-core path; returns false (nothing enqueued but
// cacheable window statistics) when it does not apply.  Results, counts and visit codes are
// those of prepare + run.  `pre`: a first half already enqueued for this call (stream).
bool search_fused(tm_ctx* ctx, tm_image* img, const double* tmpl, int m, int n,
                  const tm_match_params& P, int pred, tm_match_result* out,
                  const FusedPre* pre = nullptr) {
    FusedPre local;
    const FusedPre* fp = pre;
    if (!fp || !fp->ok || fp->img != img || fp->m != m || fp->n != n || fp->pred != pred ||
        std::memcmp(fp->tmpl.data(), tmpl, size_t(m) * n * sizeof(double)) != 0) {
        // (a first half enqueued for other inputs is simply redone: its state is rewritten)
        if (!search_fused_begin(ctx, img, tmpl, m, n, P, pred, local)) return false;
        fp = &local;
    }
    search_fused_end(ctx, img, P, *fp, out);
    return true;
}

// prepare + run of one template on a resident image (tm_search's body; ev0 recorded).
// Size tc_b for the predicted centre scan and record ev_b0 (the side-stream B build waits
// only for it), before the call's first kernel; sets spec_b.
void b_early(tm_ctx* ctx, const tm_image* img, int m, int n, int want) {
    ctx->spec_b = false;
    if (want > 0 && ctx->tc && m >= 1 && n >= 1 && m <= img->p && n <= img->q) {
        const tmk::TcPlan plan = tmk::tc_plan(m, n, want, kTcSmemBudget);
        if (plan.nch > 0) {
            ctx->tc_b.ensure(plan.total_bytes);
            CK(cudaEventRecord(ctx->ev_b0, ctx->s));
            ctx->spec_b = true;
        }
    }
}

// Predicted h_e of a search: the last one seen for this image/template shape (else h0);
// 0 when no prediction applies.
int predicted_he(tm_ctx* ctx, const tm_image* img, int m, int n, const tm_match_params& P) {
    const bool egs = P.mode != TM_MODE_OPTA && P.h0 == P.w0;
    if (!(egs && img->integer && m <= img->p && n <= img->q)) return 0;
    const std::vector<long long> key = {img->p, img->q, m, n, P.h0, P.w0};
    const auto it = ctx->last_he.find(key);
    return it != ctx->last_he.end() ? it->second : P.h0;
}

void search_resident(tm_ctx* ctx, tm_image* img, const double* tmpl, int m, int n,
                     const tm_match_params* params, tm_match_result* out,
                     const FusedPre* pre = nullptr) {
    ctx->ev1_set = false;
    Tmpl T;
    bool uploaded = false;
    // Predicted h_e: the last one seen for this image/template shape (else h0).  Fused
    // path: scan 1 on its grid first, scan 2 inside its R_co launch.  Otherwise its centre
    // scan is enqueued behind the first EGS batch, gated on the device decision, so the
    // device does not idle while the host reads the counts.
    const int want = predicted_he(ctx, img, m, n, *params);
    ctx->spec_want = want;
    ctx->spec.armed = false;
    // B of the predicted centre scan is built on the side stream (during the statistics on
    // the fused path, during the EGS batch otherwise): its buffer is sized now, before any
    // kernel of this call is enqueued, so the side stream waits for nothing of this call
    ctx->spec_b = false;
    if (!pre || !pre->ok) b_early(ctx, img, m, n, want);
    // the window statistics next (every path needs them): the device starts while the host
    // does the rest of the call's set-up
    if (m >= 1 && n >= 1 && m <= img->p && n <= img->q) get_ws(ctx, img, m, n);
    HT("ws_enqueued");
    const std::function<void()> hook = [&] {
        T = upload_template(ctx, tmpl, m, n, /*side=*/true);
        uploaded = true;
        if (want > 0)
            spec_centre(ctx, img, get_ws(ctx, img, m, n),
                        T, make_grid(img->p - m + 1, img->q - n + 1, want, want), *params);
    };
    if (want > 0 && search_fused(ctx, img, tmpl, m, n, *params, want, out, pre)) {
        ctx->spec_want = 0;
        ctx->spec_b = false;
        ctx->spec.armed = false;
        if (!ctx->ev1_set) CK(cudaEventRecord(ctx->ev1, ctx->s));
        ctx->ev1_set = false;
        spin_wait(ctx->ev1);
        out->wall_ms = ms_between(ctx->ev0, ctx->ev1);
        return;
    }
    std::unique_ptr<tm_prep> prep;
    try {
        prep.reset(prepare(ctx, img, m, n, *params, &hook, /*timed=*/false));
    } catch (...) {
        ctx->spec_want = 0;
        ctx->spec_b = false;
        ctx->spec.armed = false;
        throw;
    }
    ctx->spec_want = 0;  // (run_egs_search recorded h_e for the next prediction)
    ctx->spec_b = false;
    prep->ctx = nullptr;  // internal: not counted as a context reference
    if (!uploaded) T = upload_template(ctx, tmpl, m, n);
    *out = run_uploaded(ctx, prep.get(), img, T, *params, nullptr);
    if (!ctx->ev1_set) CK(cudaEventRecord(ctx->ev1, ctx->s));
    ctx->ev1_set = false;
    spin_wait(ctx->ev1);
    out->wall_ms = ms_between(ctx->ev0, ctx->ev1);
}

int tm_search(tm_ctx* ctx, tm_image* img, const double* tmpl, int m, int n,
              const tm_match_params* params, tm_match_result* out) {
    return guard(ctx, [&] {
        if (!img || !tmpl || !params || !out) invalid("tm_search: null argument");
        HT("start");
        CK(cudaEventRecord(ctx->ev0, ctx->s));
        search_resident(ctx, img, tmpl, m, n, params, out);
    });
}

int tm_search_upload_u8(tm_ctx* ctx, tm_image* img, const uint8_t* pixels, const uint8_t* tmpl,
                        int m, int n, const tm_match_params* params, tm_match_result* out) {
    return guard(ctx, [&] {
        if (!img || !pixels || !tmpl || !params || !out)
            invalid("tm_search_upload_u8: null argument");
        if (!img->integer) invalid("tm_image_upload_u8: image is not an 8-bit image");
        if (m < 1 || n < 1) invalid("tm_search_upload_u8: invalid template");
        HT("start");
        CK(cudaEventRecord(ctx->ev0, ctx->s));
        // (a row-chunked upload overlapping the window statistics with the copy was measured
        // slower on C2: per-chunk statistics launches cost more than the copy they hide)
        const size_t N = size_t(img->p) * img->q;
        CK(cudaMemcpyAsync(img->u8.p, pixels, N, cudaMemcpyHostToDevice, ctx->s));
        img->have_f32 = img->have_f64 = false;
        img->have_qtotal = false;
        tc_pitch_copy(ctx, img);
        invalidate_ws(img);
        std::vector<double> t(size_t(m) * n);
        for (size_t i = 0; i < t.size(); ++i) t[i] = tmpl[i];
        search_resident(ctx, img, t.data(), m, n, params, out);
    });
}

int tm_search_stream_u8(tm_ctx* ctx, const uint8_t* const* images, int nimg, int rows, int cols,
                        const uint8_t* tmpl, int m, int n, const tm_match_params* params,
                        tm_match_result* out) {
    return guard(ctx, [&] {
        if (!images || !tmpl || !params || !out) invalid("tm_search_stream_u8: null argument");
        if (nimg < 0) invalid("tm_search_stream_u8: negative image count");
        if (rows < 1 || cols < 1) invalid("image dimensions must be at least 1x1");
        if (m < 1 || n < 1) invalid("tm_search_stream_u8: invalid template");
        for (int i = 0; i < nimg; ++i)
            if (!images[i]) invalid("tm_search_stream_u8: null image pointer");
        if (nimg == 0) return;
        if (!ctx->s_up) {
            CK(cudaStreamCreateWithFlags(&ctx->s_up, cudaStreamNonBlocking));
            for (int k = 0; k < 2; ++k) {
                CK(cudaEventCreateWithFlags(&ctx->ev_up[k], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ctx->ev_free[k], cudaEventDisableTiming));
            }
        }
        for (int k = 0; k < 2; ++k) {
            auto& sl = ctx->sslot[k];
            if (!sl || sl->p != rows || sl->q != cols) {
                sl.reset();  // stream-ordered free
                sl = std::make_unique<tm_image>();
                sl->ctx = ctx;  // internal: owned by the context, no reference
                sl->p = rows;
                sl->q = cols;
                sl->integer = true;
                sl->pitch = ((cols + 3) & ~3) + 128;
                alloc_u8(ctx, sl.get());
            }
            // the slot's buffer is free (allocated / last read) at this point of stream s
            CK(cudaEventRecord(ctx->ev_free[k], ctx->s));
        }
        std::vector<double> t(size_t(m) * n);
        for (size_t i = 0; i < t.size(); ++i) t[i] = tmpl[i];
        const size_t N = size_t(rows) * cols;
        auto enqueue_upload = [&](int i) {
            const int k = i & 1;
            CK(cudaStreamWaitEvent(ctx->s_up, ctx->ev_free[k], 0));
            CK(cudaMemcpyAsync(ctx->sslot[k]->u8.p, images[i], N, cudaMemcpyHostToDevice,
                               ctx->s_up));
            CK(cudaEventRecord(ctx->ev_up[k], ctx->s_up));
        };
        // an image's prologue: its layout copy and window statistics (they need only the
        // pixels); image i+1's is enqueued behind search i, before the host waits for that
        // result, so the device does not idle while the host finishes search i
        auto prologue = [&](int i) {
            tm_image* img = ctx->sslot[i & 1].get();
            CK(cudaStreamWaitEvent(ctx->s, ctx->ev_up[i & 1], 0));
            img->have_f32 = img->have_f64 = false;
            img->have_qtotal = false;
            tc_pitch_copy(ctx, img);
            invalidate_ws(img);
            get_ws(ctx, img, m, n);
        };
        const bool ws_ok = m <= rows && n <= cols;  // (else the search reports the error)
        enqueue_upload(0);
        bool pro_done = false;
        FusedPre next_pre;  // the next image's first half, enqueued behind the current search
        for (int i = 0; i < nimg; ++i) {
            tm_image* img = ctx->sslot[i & 1].get();
            HT("start");
            CK(cudaEventRecord(ctx->ev0, ctx->s));
            // the next image crosses PCIe while this one is searched (the other slot's last
            // reader, search i-1, has completed: search_resident returns after its readback)
            if (i + 1 < nimg) enqueue_upload(i + 1);
            if (!pro_done) {
                if (ws_ok) {
                    prologue(i);
                } else {
                    CK(cudaStreamWaitEvent(ctx->s, ctx->ev_up[i & 1], 0));
                    img->have_f32 = img->have_f64 = img->have_qtotal = false;
                    tc_pitch_copy(ctx, img);
                    invalidate_ws(img);
                }
            }
            pro_done = false;
            FusedPre cur_pre;
            cur_pre.swap_from(next_pre);
            if (ws_ok && i + 1 < nimg)
                ctx->before_final_sync = [&, i] {
                    tm_image* nimg_ = ctx->sslot[(i + 1) & 1].get();
                    const int pred = predicted_he(ctx, nimg_, m, n, *params);
                    b_early(ctx, nimg_, m, n, pred);  // (B build overlaps the statistics)
                    prologue(i + 1);
                    pro_done = true;
                    // ... and the next search's scan 1 + seeding when it takes the fused path
                    if (pred > 0)
                        search_fused_begin(ctx, nimg_, t.data(), m, n, *params, pred, next_pre);
                    ctx->spec_b = false;
                };
            try {
                search_resident(ctx, img, t.data(), m, n, params, &out[i],
                                cur_pre.ok ? &cur_pre : nullptr);
            } catch (...) {
                ctx->before_final_sync = nullptr;
                throw;
            }
            if (ctx->before_final_sync) {  // (a search path without the hook: run it now)
                ctx->before_final_sync = nullptr;
                prologue(i + 1);
                pro_done = true;
            }
            CK(cudaEventRecord(ctx->ev_free[i & 1], ctx->s));
        }
    });
}

int tm_search_u8(tm_ctx* ctx, tm_image* img, const uint8_t* tmpl, int m, int n,
                 const tm_match_params* params, tm_match_result* out) {
    if (!tmpl || m < 1 || n < 1) {
        g_err = "tm_search_u8: invalid template";
        return TM_EINVAL;
    }
    std::vector<double> t(size_t(m) * n);
    for (size_t i = 0; i < t.size(); ++i) t[i] = tmpl[i];
    return tm_search(ctx, img, t.data(), m, n, params, out);
}

int tm_transitive_search(tm_ctx* ctx, const double* tmpl, int m, int n, tm_image* img,
                         const double* map, int h, int w, const tm_match_params* params,
                         tm_match_result* out, uint8_t* visits) {
    return guard(ctx, [&] {
        if (m > img->p || n > img->q) invalid("group grid: template does not fit the image");
        const tmk::GridDesc g = make_grid(img->p - m + 1, img->q - n + 1, h, w);
        WS& ws = get_ws(ctx, img, m, n);
        const size_t E = size_t(g.er) * g.ec;
        ctx->map_user.ensure(E);
        CK(cudaMemcpyAsync(ctx->map_user.p, map, E * 8, cudaMemcpyHostToDevice, ctx->s));
        CK(cudaEventRecord(ctx->ev0, ctx->s));
        const Tmpl T = upload_template(ctx, tmpl, m, n);
        *out = search(ctx, SearchIn{img, &ws, g, ctx->map_user.p}, T, *params, visits);
        CK(cudaEventRecord(ctx->ev1, ctx->s));
        CK(cudaEventSynchronize(ctx->ev1));
        out->wall_ms = ms_between(ctx->ev0, ctx->ev1);
    });
}

int tm_transitive_search_ws(tm_ctx* ctx, const double* tmpl, int m, int n, tm_image* img,
                            const double* map, int h, int w, const double* mu,
                            const double* omega, const uint8_t* flat,
                            const tm_match_params* params, tm_match_result* out,
                            uint8_t* visits) {
    return guard(ctx, [&] {
        if (!mu || !omega || !flat) invalid("tm_transitive_search_ws: null window statistics");
        if (m > img->p || n > img->q) invalid("group grid: template does not fit the image");
        const tmk::GridDesc g = make_grid(img->p - m + 1, img->q - n + 1, h, w);
        // the caller's statistics in place of the image's own for this search (a preparation
        // of earlier pixels: run_egs with prep.ws, matcher.cpp:235-246), then dropped
        WS& ws = get_ws(ctx, img, m, n);
        const size_t E = size_t(g.er) * g.ec;
        CK(cudaMemcpyAsync(ws.mu.p, mu, E * 8, cudaMemcpyHostToDevice, ctx->s));
        CK(cudaMemcpyAsync(ws.om.p, omega, E * 8, cudaMemcpyHostToDevice, ctx->s));
        CK(cudaMemcpyAsync(ws.fl.p, flat, E, cudaMemcpyHostToDevice, ctx->s));
        ctx->map_user.ensure(E);
        CK(cudaMemcpyAsync(ctx->map_user.p, map, E * 8, cudaMemcpyHostToDevice, ctx->s));
        CK(cudaEventRecord(ctx->ev0, ctx->s));
        const Tmpl T = upload_template(ctx, tmpl, m, n);
        try {
            *out = search(ctx, SearchIn{img, &ws, g, ctx->map_user.p}, T, *params, visits);
        } catch (...) {
            invalidate_ws(img);
            throw;
        }
        invalidate_ws(img);  // the next user of the image recomputes its own statistics
        CK(cudaEventRecord(ctx->ev1, ctx->s));
        CK(cudaEventSynchronize(ctx->ev1));
        out->wall_ms = ms_between(ctx->ev0, ctx->ev1);
    });
}

int tm_center_scan(tm_ctx* ctx, const double* tmpl, int m, int n, tm_image* img, int h, int w,
                   double* rho, uint8_t* degenerate, int* best_row, int* best_col,
                   double* best_rho, int* best_degenerate) {
    return guard(ctx, [&] {
        if (m > img->p || n > img->q) invalid("center_scan: grid extent mismatch");
        const tmk::GridDesc g = make_grid(img->p - m + 1, img->q - n + 1, h, w);
        WS& ws = get_ws(ctx, img, m, n);
        const Tmpl T = upload_template(ctx, tmpl, m, n);
        centre_scan(ctx, img, ws, T, g);
        const size_t G = size_t(g.tr) * g.tc;
        tmk::CellH c;
        CK(cudaMemcpyAsync(&c, ctx->cells.p, sizeof c, cudaMemcpyDeviceToHost, ctx->s));
        if (rho) CK(cudaMemcpyAsync(rho, ctx->rho_c.p, G * 8, cudaMemcpyDeviceToHost, ctx->s));
        if (degenerate)
            CK(cudaMemcpyAsync(degenerate, ctx->deg_c.p, G, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        *best_row = c.row;
        *best_col = c.col;
        *best_rho = c.rho;
        *best_degenerate = (c.flags & 2) != 0;
    });
}

int tm_refine_localization(tm_ctx* ctx, const double* tmpl, int m, int n, tm_image* original,
                           int loc_row, int loc_col, int d, int* row, int* col, double* rho,
                           int* degenerate) {
    return guard(ctx, [&] {
        if (d < 0) invalid("refine_localization: d must be >= 0");
        WS& ws = get_ws(ctx, original, m, n);
        if (loc_row < 0 || loc_row >= ws.er || loc_col < 0 || loc_col >= ws.ec)
            invalid("refine_localization: location outside the extent");
        const Tmpl T = upload_template(ctx, tmpl, m, n);
        long long ops = 0;
        const tmk::CellH c = refine(ctx, original, ws, T, loc_row, loc_col, d, &ops);
        *row = c.row;
        *col = c.col;
        *rho = c.rho;
        *degenerate = (c.flags & 2) != 0;
    });
}

// ---- row-strip protocol (multi-GPU; orchestrated by paper_1407_3535_b200/distributed.py) ----
int tm_strip_autocorr(tm_ctx* ctx, tm_image* img, int m, int n, int h, int w, int rank, int world,
                      double rho_tb, int slot, int64_t* n_r) {
    return guard(ctx, [&] {
        if (slot < 0 || slot > 2) invalid("tm_strip_autocorr: slot must be 0..2");
        if (m > img->p || n > img->q) invalid("efficient_group_size: template does not fit");
        if (rho_tb < 0.0 || rho_tb > 1.0) invalid("retained_count: rho_tb must be in [0,1]");
        const tmk::GridDesc g =
            strip_of(make_grid(img->p - m + 1, img->q - n + 1, h, w), rank, world);
        WS& ws = get_ws(ctx, img, m, n);
        ctx->egs_maps[slot].ensure(size_t(g.er) * g.ec);
        *n_r = autocorr_map(ctx, img, ws, g, expected_elimination_threshold_h(rho_tb),
                            ctx->egs_maps[slot].p);
    });
}

int tm_strip_commit(tm_ctx* ctx, tm_image* img, int m, int n, int slot, int h, int w,
                    const tm_match_params* params, const tm_egs_iter* trace, int trace_len,
                    tm_prep** out) {
    return guard(ctx, [&] {
        if (slot < 0 || slot > 2) invalid("tm_strip_commit: slot must be 0..2");
        auto prep = std::make_unique<tm_prep>();
        prep->params = *params;
        prep->profile = params_profile(*params);
        prep->params.kernel_profile = nullptr;
        prep->mode = TM_MODE_EGS;
        prep->m = m;
        prep->n = n;
        prep->h = h;
        prep->w = w;
        prep->source = img;
        prep->g = make_grid(img->p - m + 1, img->q - n + 1, h, w);
        prep->map.swap(ctx->egs_maps[slot]);
        prep->egs_trace.assign(trace, trace + std::max(0, trace_len));
        if (trace_len > 0) prep->cost = trace[trace_len - 1];
        prep->prep_ms = 0.0;
        prep->ctx = ctx;
        ++ctx->refs;
        *out = prep.release();
    });
}

int tm_strip_search_begin(tm_ctx* ctx, tm_prep* prep, tm_image* img, const double* tmpl,
                          const tm_match_params* params, int rank, int world, double* T0) {
    return guard(ctx, [&] {
        auto& S = ctx->strip;
        S = tm_ctx::StripState{};
        S.prep = prep;
        S.img = img;
        S.P = *params;
        S.m = prep->m;
        S.n = prep->n;
        S.g = strip_of(prep->g, rank, world);
        S.policy = params->policy == TM_POLICY_SEEDED ? TM_POLICY_SEEDED : TM_POLICY_FROZEN;
        if (params->policy == TM_POLICY_SEQUENTIAL ||
            (params->policy == TM_POLICY_REFERENCE && !(params->parallel && params->threads > 1)))
            invalid("row strips support the frozen and seeded policies (the sequential running "
                    "threshold is defined by a single global scan order)");
        S.T = upload_template(ctx, tmpl, S.m, S.n);
        const Tmpl& T = S.T;
        if (T.ts.flat) invalid("transitive_search: constant template has no defined correlation");
        if (params->has_init_threshold && std::abs(params->init_threshold) > 1.0 + 1e-9)
            invalid("transitive_search: init threshold out of [-1,1]");
        tm_image* simg = prep->search_img ? prep->search_img.get() : img;
        const WS* ws = prep->search_img ? prep->search_ws.get() : &get_ws(ctx, img, S.m, S.n);
        const size_t G = size_t(S.g.tr) * S.g.tc;
        ctx->rho_c.ensure(G);
        ctx->deg_c.ensure(G);
        centre_scan(ctx, simg, *ws, T, S.g);
        CK(tmk::threshold_init(ctx->cells.p + 0, params->has_init_threshold,
                               params->init_threshold, ctx->thr.p, ctx->s));
        ctx->add(1);
        CK(cudaMemcpyAsync(T0, ctx->thr.p, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        S.active = true;
    });
}

int tm_strip_search_seed(tm_ctx* ctx, double T, double* T1) {
    return guard(ctx, [&] {
        auto& S = ctx->strip;
        if (!S.active) invalid("tm_strip_search_seed: no strip search in progress");
        tm_image* simg = S.prep->search_img ? S.prep->search_img.get() : S.img;
        const WS* ws = S.prep->search_img ? S.prep->search_ws.get() : &get_ws(ctx, S.img, S.m, S.n);
        const Tmpl& Tm = S.T;
        const tmk::GridDesc& g = S.g;
        const size_t G = size_t(g.tr) * g.tc;
        CK(cudaMemcpyAsync(ctx->thr.p, &T, 8, cudaMemcpyHostToDevice, ctx->s));
        const unsigned long long max_groups = 256;
        const unsigned long long max_locs = max_groups * (unsigned long long)(g.h * g.w);
        ctx->seed_locs.ensure(max_locs);
        ctx->seeded.ensure(G);
        CK(cudaMemsetAsync(ctx->counters.p + 4, 0, 16, ctx->s));
        CK(tmk::seed_members(g, ctx->rho_c.p, ctx->deg_c.p, ctx->thr.p, S.P.seed_margin,
                             ctx->seeded.p, ctx->seed_locs.p, ctx->counters.p + 4, max_locs,
                             ctx->counters.p + 5, max_groups, ctx->s));
        ctx->add(1);
        eval_list(ctx, simg, *ws, Tm, ctx->seed_locs.p, ctx->counters.p + 4, int(max_locs), nullptr,
                  nullptr, 1);
        CK(tmk::threshold_raise(ctx->cells.p + 1, ctx->thr.p, ctx->s));
        ctx->add(1);
        CK(cudaMemcpyAsync(T1, ctx->thr.p, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    });
}

int tm_strip_search_finish(tm_ctx* ctx, double T, tm_strip_part* out) {
    return guard(ctx, [&] {
        auto& S = ctx->strip;
        if (!S.active) invalid("tm_strip_search_finish: no strip search in progress");
        tm_image* simg = S.prep->search_img ? S.prep->search_img.get() : S.img;
        const WS* ws = S.prep->search_img ? S.prep->search_ws.get() : &get_ws(ctx, S.img, S.m, S.n);
        const Tmpl& Tm = S.T;
        const tmk::GridDesc& g = S.g;
        const size_t E = size_t(g.er) * g.ec;
        CK(cudaMemcpyAsync(ctx->thr.p, &T, 8, cudaMemcpyHostToDevice, ctx->s));
        ctx->visits.ensure(E);
        ctx->locs.ensure(E);
        CK(cudaMemsetAsync(ctx->tally.p, 0, sizeof(tmk::Tally), ctx->s));
        const uint8_t* seeded = S.policy == TM_POLICY_SEEDED ? ctx->seeded.p : nullptr;
        // scan 2 over the strip's rows (k_sec_rows: flat members kept but not listed,
        // survivor tile flags for the masked dense pass)
        const size_t G = size_t(g.tr) * g.tc;
        ctx->sa_c.ensure(G);
        const tmk::TileFlags tf = zero_tile_flags(ctx, ctx->tflags, g.er, g.ec);
        const unsigned long long max_locs = fp32_path(simg, Tm) ? E / tmk::kDenseDiv + 1 : E;
        CK(tmk::sec_rows(g, S.prep->map.p, ctx->rho_c.p, ctx->sa_c.p, ctx->deg_c.p, ws->fl.p,
                         Tm.ts.flat, ctx->thr.p, seeded, ctx->locs.p, max_locs, ctx->tally.p,
                         ctx->visits.p, ctx->s, ctx->sa_ready, tf));
        ctx->add(ctx->sa_ready ? 1 : 2);
        tmk::Tally tally{};
        CK(cudaMemcpyAsync(&tally, ctx->tally.p, sizeof tally, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        eval_survivors(ctx, simg, *ws, Tm, g, tally.survivors, nullptr, &tf);
        tmk::CellH cells[3];
        CK(cudaMemcpyAsync(cells, ctx->cells.p, sizeof cells, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        tmk::CellH best = cells[0];
        if (S.policy == TM_POLICY_SEEDED && better_h(cells[1], best)) best = cells[1];
        if (better_h(cells[2], best)) best = cells[2];
        if (better_h(flat_cell(tally), best)) best = flat_cell(tally);
        double fin = T;
        if ((cells[2].flags & 1) && !(cells[2].flags & 2) && cells[2].rho > fin) fin = cells[2].rho;
        std::memset(out, 0, sizeof *out);
        out->best_rho = best.rho;
        out->best_row = best.row;
        out->best_col = best.col;
        out->best_flags = best.flags;
        out->centers = (int64_t)(g.ti_hi - g.ti_lo) * g.tc;
        out->eliminated = (int64_t)tally.eliminated;
        out->retained = (int64_t)tally.retained;
        out->final_threshold = fin;
        S.active = false;
    });
}

// ---- fused row-strip protocol (scan 2 inside the strip's R_co launch) ---------------------
// The single-GPU fused search (search_fused_begin / _end) split at its global decisions:
//   begin   window statistics of the strip, scan 1 on the PREDICTED grid's strip -> T0
//   [seed   the seeded policy's groups -> T1]                     (allreduce MAX between)
//   egs     the EGS candidate batch on the strip: the predicted size with scan 2 fused
//           (thresholded at the global T), the others count-only -> local retained counts
//   finish  (after the allreduced counts confirm the predicted size) survivors -> part
// 4 host round trips instead of ~7, no R_co map round trip.  *supported = 0: not applicable
// (non-8-bit data, OptA, other policies): the caller uses the tm_strip_search_* protocol.
int tm_strip_fused_begin(tm_ctx* ctx, tm_image* img, const double* tmpl, int m, int n,
                         const tm_match_params* params, int rank, int world, int pred,
                         int* supported, double* T0) {
    return guard(ctx, [&] {
        auto& S = ctx->strip;
        S = tm_ctx::StripState{};
        *supported = 0;
        const tm_match_params& P = *params;
        if (P.mode == TM_MODE_OPTA || !img->integer || !ctx->ac_fused || !ctx->tc) return;
        if (P.h0 != P.w0 || m > img->p || n > img->q || pred < 1 || pred % 2 == 0) return;
        int policy = P.policy;
        if (policy == TM_POLICY_REFERENCE)
            policy = (P.parallel && P.threads > 1) ? TM_POLICY_FROZEN : TM_POLICY_SEQUENTIAL;
        if (policy != TM_POLICY_SEEDED && policy != TM_POLICY_FROZEN) return;
        if (!(img->u8p.p && img->u8p_rows >= img->p + tmk::kU8PadRows)) return;
        const int er = img->p - m + 1, ec = img->q - n + 1;
        const tmk::GridDesc g = strip_of(make_grid(er, ec, pred, pred), rank, world);
        if (!tmk::autocorr_sec_fuse_supported(m, n, g) || g.h > tmk::kTcMaxClasses) return;
        const Tmpl probe = template_host_stats(tmpl, m, n);
        if (probe.ts.flat) invalid("transitive_search: constant template has no defined correlation");
        if (!tc_path(ctx, img, probe)) return;
        if (P.has_init_threshold && std::abs(P.init_threshold) > 1.0 + 1e-9)
            invalid("transitive_search: init threshold out of [-1,1]");
        WS& ws = get_ws(ctx, img, m, n);  // the strip's rows (strip image) or all
        S.T = upload_template(ctx, tmpl, m, n);
        S.img = img;
        S.P = P;
        S.P.kernel_profile = nullptr;
        S.policy = policy;
        S.m = m;
        S.n = n;
        S.g = g;
        S.pred = pred;
        S.er = er;
        S.ec = ec;
        S.rank = rank;
        S.world = world;
        S.fused = true;
        const size_t G = size_t(g.tr) * g.tc;
        ctx->rho_c.ensure(G);
        ctx->deg_c.ensure(G);
        const tmk::ReduceOp op_init = centre_op(ctx, P);  // threshold init, tally zeroing
        centre_scan(ctx, img, ws, S.T, g, &op_init);
        if (!ctx->sa_ready) {
            ctx->sa_c.ensure(G);
            CK(tmk::sqrt_gap(ctx->rho_c.p, ctx->sa_c.p, G, ctx->s));
            ctx->add(1);
            ctx->sa_ready = true;
        }
        CK(cudaMemcpyAsync(T0, ctx->thr.p, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        S.active = true;
        *supported = 1;
    });
}

int tm_strip_fused_seed(tm_ctx* ctx, double T, double* T1) {
    return guard(ctx, [&] {
        auto& S = ctx->strip;
        if (!S.active || !S.fused) invalid("tm_strip_fused_seed: no fused strip search in progress");
        const tmk::GridDesc& g = S.g;
        const size_t G = size_t(g.tr) * g.tc;
        WS& ws = get_ws(ctx, S.img, S.m, S.n);
        CK(cudaMemcpyAsync(ctx->thr.p, &T, 8, cudaMemcpyHostToDevice, ctx->s));
        const unsigned long long max_groups = 256;
        const unsigned long long max_locs = max_groups * (unsigned long long)(g.h * g.w);
        ctx->seed_locs.ensure(max_locs);
        ctx->seeded.ensure(G);
        CK(cudaMemsetAsync(ctx->counters.p + 4, 0, 16, ctx->s));
        CK(tmk::seed_members(g, ctx->rho_c.p, ctx->deg_c.p, ctx->thr.p, S.P.seed_margin,
                             ctx->seeded.p, ctx->seed_locs.p, ctx->counters.p + 4, max_locs,
                             ctx->counters.p + 5, max_groups, ctx->s));
        ctx->add(1);
        tmk::ReduceOp op_raise{};
        op_raise.kind = 2;
        op_raise.thr = ctx->thr.p;
        eval_list(ctx, S.img, ws, S.T, ctx->seed_locs.p, ctx->counters.p + 4, int(max_locs),
                  nullptr, nullptr, 1, &op_raise);
        CK(cudaMemcpyAsync(T1, ctx->thr.p, 8, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
    });
}

int tm_strip_fused_egs(tm_ctx* ctx, double T, int* nc, int* hs, int64_t* n_r) {
    return guard(ctx, [&] {
        auto& S = ctx->strip;
        if (!S.active || !S.fused) invalid("tm_strip_fused_egs: no fused strip search in progress");
        tm_image* img = S.img;
        WS& ws = get_ws(ctx, img, S.m, S.n);
        const tm_match_params& P = S.P;
        const size_t E = size_t(S.er) * S.ec;
        CK(cudaMemcpyAsync(ctx->thr.p, &T, 8, cudaMemcpyHostToDevice, ctx->s));
        // the first EGS batch of the single-GPU path: h0 .. one size past the prediction
        int cap = P.max_group > 0 ? P.max_group : INT_MAX;
        if (cap % 2 == 0) ++cap;
        const int nmax = std::max(2, std::min(4, (S.pred - P.h0) / 2 + 2));
        S.nc = 0;
        for (int h = P.h0; S.nc < nmax;) {
            S.cand_h[S.nc++] = h;
            if ((h >= S.er && h >= S.ec) || h >= cap) break;
            h = std::min(h + 2, cap);
        }
        const double thr = expected_elimination_threshold_h(P.rho_th);
        tmk::SecFuse sf{};
        sf.thr = ctx->thr.p;
        sf.rho_c = ctx->rho_c.p;
        sf.sa_c = ctx->sa_c.p;
        sf.deg_c = ctx->deg_c.p;
        sf.seeded = S.policy == TM_POLICY_SEEDED ? ctx->seeded.p : nullptr;
        sf.tflat = S.T.ts.flat;
        ctx->locs.ensure(E / tmk::kDenseDiv + 1);
        ctx->visits.ensure(E);
        sf.locs = ctx->locs.p;
        sf.max_locs = E / tmk::kDenseDiv + 1;
        sf.tally = ctx->tally.p;  // (zeroed by the centre reduction)
        sf.visits = ctx->visits.p;
        sf.tf = zero_tile_flags(ctx, ctx->tflags, S.er, S.ec);
        S.tf = sf.tf;
        bool fused_ran = false;
        for (int k = 0; k < S.nc; ++k) {
            const int h = S.cand_h[k];
            const tmk::GridDesc g = strip_of(make_grid(S.er, S.ec, h, h), S.rank, S.world);
            const bool is_pred = h == S.pred && !fused_ran;
            ctx->egs_maps[k].ensure(1);
            // no in-kernel EGS rejection: a strip's partial count says nothing about the
            // global one (the decision is the host's, on the allreduced counts)
            autocorr_launch(ctx, img, ws, g, thr, nullptr, ctx->counters.p + 8 + k, nullptr,
                            nullptr, 0.0, /*count_only=*/!is_pred, nullptr, nullptr,
                            is_pred ? &sf : nullptr);
            if (is_pred) fused_ran = true;
        }
        if (!fused_ran) invalid("tm_strip_fused_egs: the predicted size is not in the batch");
        unsigned long long v[4] = {0, 0, 0, 0};
        CK(cudaMemcpyAsync(v, ctx->counters.p + 8, 8 * S.nc, cudaMemcpyDeviceToHost, ctx->s));
        CK(cudaStreamSynchronize(ctx->s));
        *nc = S.nc;
        for (int k = 0; k < S.nc; ++k) {
            hs[k] = S.cand_h[k];
            n_r[k] = (int64_t)v[k];
        }
    });
}

int tm_strip_fused_finish(tm_ctx* ctx, tm_strip_part* out) {
    return guard(ctx, [&] {
        auto& S = ctx->strip;
        if (!S.active || !S.fused) invalid("tm_strip_fused_finish: no fused strip search in progress");
        tm_image* img = S.img;
        WS& ws = get_ws(ctx, img, S.m, S.n);
        const tmk::GridDesc& g = S.g;
        // survivors (dense or list on the device; the reduction packs the mapped block)
        eval_survivors_dev(ctx, img, ws, S.T, g, nullptr, nullptr, false, nullptr, nullptr,
                           nullptr, &S.tf);
        CK(cudaEventRecord(ctx->ev1, ctx->s));
        spin_wait(ctx->ev1);
        const tm_ctx::HostRes* hr = ctx->hres;
        tmk::CellH best = hr->cells[0];
        if (S.policy == TM_POLICY_SEEDED && better_h(hr->cells[1], best)) best = hr->cells[1];
        if (better_h(hr->cells[2], best)) best = hr->cells[2];
        if (better_h(flat_cell(hr->tally), best)) best = flat_cell(hr->tally);
        double fin = hr->thr;
        if ((hr->cells[2].flags & 1) && !(hr->cells[2].flags & 2) && hr->cells[2].rho > fin)
            fin = hr->cells[2].rho;
        std::memset(out, 0, sizeof *out);
        out->best_rho = best.rho;
        out->best_row = best.row;
        out->best_col = best.col;
        out->best_flags = best.flags;
        out->centers = (int64_t)(g.ti_hi - g.ti_lo) * g.tc;
        out->eliminated = (int64_t)hr->tally.eliminated;
        out->retained = (int64_t)hr->tally.retained;
        out->final_threshold = fin;
        S.active = false;
    });
}

int tm_match(tm_ctx* ctx, const double* tmpl, int m, int n, const double* image, int rows,
             int cols, const tm_match_params* params, tm_match_result* out, uint8_t* visits) {
    tm_image* img = nullptr;
    int rc = tm_image_create(ctx, image, rows, cols, &img);
    if (rc != TM_OK) return rc;
    rc = guard(ctx, [&] {
        if (m > rows || n > cols) invalid("match: template larger than search image");
        CK(cudaEventRecord(ctx->ev0, ctx->s));
        const auto t0 = std::chrono::steady_clock::now();
        if (params->mode == TM_MODE_BRUTE) {
            const Tmpl T = upload_template(ctx, tmpl, m, n);
            *out = brute(ctx, img, T, nullptr);
            if (visits) std::memset(visits, TM_VISIT_RETAINED, size_t(out->extent_rows) * out->extent_cols);
        } else {
            const Tmpl T = upload_template(ctx, tmpl, m, n);
            if (T.ts.flat) invalid("match: constant template has no defined correlation");
            if (params->mode != TM_MODE_OPTA && !visits) {
                // no preparation handle or visit map leaves the call: tm_search's path (scan 2
                // fused into R_co for the frozen / seeded policies), same results
                search_resident(ctx, img, tmpl, m, n, params, out);
            } else {
                std::unique_ptr<tm_prep> prep(prepare(ctx, img, m, n, *params));
                *out = run_one(ctx, prep.get(), img, tmpl, *params, visits);
                prep.reset();
            }
        }
        out->wall_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
    tm_image_destroy(img);
    return rc;
}

}  // extern "C"
static_assert(sizeof(tm_match_result) == 112, "tm_match_result layout is part of the ABI");
static_assert(sizeof(tm_egs_iter) == 48, "tm_egs_iter layout is part of the ABI");
