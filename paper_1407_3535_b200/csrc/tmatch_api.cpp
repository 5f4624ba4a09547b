// tmatch_api.cpp -- the reference C++ API (include/tmatch/*.hpp, mirroring
// /root/reference/proj/include/tmatch) implemented over the C ABI of libtmatch_cuda.so.
//
// Every image-sized computation (window statistics, running sums, auto-correlation, EGS,
// blur/fidelity/OptA, the searches) runs on the GPU; this file only marshals the
// reference's value types to and from the device and keeps the reference's error
// conventions (std::invalid_argument with the same messages, std::runtime_error for I/O).
// Scalar helpers (bounds algebra, grid geometry, kernel profiles, template statistics) are
// host code, as in the reference.  Compiled with -ffp-contract=off.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <sstream>
#include <stdexcept>

#include "tmatch/autocorr.hpp"
#include "tmatch/blur.hpp"
#include "tmatch/bounds.hpp"
#include "tmatch/detail.hpp"
#include "tmatch/egs.hpp"
#include "tmatch/image.hpp"
#include "tmatch/matcher.hpp"
#include "tmatch/result.hpp"
#include "tmatch/stats.hpp"
#include "tmatch_cuda.h"

namespace tmatch {

// ---- device plumbing ---------------------------------------------------------------
namespace {

std::atomic<std::uint64_t> g_tables{0};

void check(int rc) {
    if (rc == TM_OK) return;
    const std::string msg = tm_last_error();
    if (rc == TM_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("tmatch device error: " + msg);
}

// One context per host thread (the reference is re-entrant; contexts do not share state).
tm_ctx* ctx() {
    struct Holder {
        tm_ctx* c = nullptr;
        ~Holder() {
            if (c) tm_ctx_destroy(c);
        }
    };
    thread_local Holder h;
    if (!h.c) {
        const char* dev = std::getenv("TMATCH_DEVICE");
        check(tm_ctx_create(dev ? std::atoi(dev) : 0, &h.c));
    }
    return h.c;
}

struct DevImage {
    tm_image* h = nullptr;
    explicit DevImage(const Image& img) {
        if (img.empty()) throw std::invalid_argument("image dimensions must be at least 1x1");
        check(tm_image_create(ctx(), img.data().data(), img.rows(), img.cols(), &h));
    }
    ~DevImage() { tm_image_destroy(h); }
    DevImage(const DevImage&) = delete;
    DevImage& operator=(const DevImage&) = delete;
};

tm_match_params to_c(const MatchParams& p) {
    tm_match_params c;
    tm_default_params(&c);
    c.mode = int(p.mode);
    c.h0 = p.h0;
    c.w0 = p.w0;
    c.has_init_threshold = p.init_threshold.has_value();
    c.init_threshold = p.init_threshold.value_or(0.0);
    c.rho_th = p.rho_th;
    c.rho_max = p.rho_max;
    c.xi_fraction = p.xi_fraction;
    c.opta_margin = p.opta_margin;
    c.kernel_profile = p.kernel.profile.data();
    c.kernel_len = int(p.kernel.profile.size());
    c.parallel = p.parallel;
    c.threads = p.threads;
    c.record_visits = p.record_visits;
    c.policy = int(p.policy);
    return c;
}

MatchResult from_c(const tm_match_result& r) {
    MatchResult o;
    o.mode = MatchMode(r.mode);
    o.best_row = r.best_row;
    o.best_col = r.best_col;
    o.best_rho = r.best_rho;
    o.best_degenerate = r.best_degenerate != 0;
    o.refined_row = r.refined_row;
    o.refined_col = r.refined_col;
    o.refined_rho = r.refined_rho;
    o.below_threshold = r.below_threshold != 0;
    o.final_threshold = r.final_threshold;
    o.stats.centers = r.centers;
    o.stats.eliminated = r.eliminated;
    o.stats.retained = r.retained;
    o.stats.elim_pct = r.elim_pct;
    o.stats.ops = r.ops;
    o.stats.wall_ms = r.wall_ms;
    o.extent_rows = r.extent_rows;
    o.extent_cols = r.extent_cols;
    return o;
}

WindowStats download_ws(tm_image* img, int m, int n, int er, int ec) {
    WindowStats ws;
    ws.win_rows = m;
    ws.win_cols = n;
    ws.rows = er;
    ws.cols = ec;
    const std::size_t E = std::size_t(er) * ec;
    ws.mean.resize(E);
    ws.norm.resize(E);
    ws.flat_map.resize(E);
    check(tm_window_stats(ctx(), img, m, n, ws.mean.data(), ws.norm.data(), ws.flat_map.data()));
    return ws;
}

EGSResult egs_from_info(const tm_prep_info& info, std::vector<double> map) {
    EGSResult e;
    e.h = info.h;
    e.w = info.w;
    e.grid = GroupGrid(info.extent_rows, info.extent_cols, info.h, info.w);
    e.map.rows = info.extent_rows;
    e.map.cols = info.extent_cols;
    e.map.group_h = info.h;
    e.map.group_w = info.w;
    e.map.values = std::move(map);
    auto cost = [](const tm_egs_iter& c) {
        return CostEstimate{c.central, c.retained, c.retained_cost, c.amortized, c.total};
    };
    e.cost = cost(info.cost);
    for (int k = 0; k < info.egs_trace_len; ++k)
        e.trace.push_back(EgsIteration{info.egs_trace[k].h, info.egs_trace[k].w,
                                       cost(info.egs_trace[k])});
    return e;
}

}  // namespace

// 64-bit fingerprint of an image's pixel words (8 independent multiply-xor lanes, several
// GB/s per core).  Not the reference's content_hash (that one keys the TMACMAP1 cache and
// is byte-serial FNV-1a); this only detects that a caller changed an Image in place
// between prepare_* and run_*.
std::uint64_t pixel_fingerprint(const Image& I) {
    constexpr std::uint64_t kMul = 0x9E3779B97F4A7C15ull;
    std::uint64_t lane[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    const double* d = I.data().data();
    const std::size_t n = I.data().size();
    std::size_t i = 0;
    for (; i + 8 <= n; i += 8)
        for (int k = 0; k < 8; ++k) {
            std::uint64_t w;
            std::memcpy(&w, d + i + k, 8);
            lane[k] = (lane[k] ^ w) * kMul;
        }
    for (; i < n; ++i) {
        std::uint64_t w;
        std::memcpy(&w, d + i, 8);
        lane[0] = (lane[0] ^ w) * kMul;
    }
    std::uint64_t h = std::uint64_t(I.rows()) * kMul ^ std::uint64_t(I.cols());
    for (int k = 0; k < 8; ++k) h = (h ^ (lane[k] >> 29) ^ lane[k]) * kMul;
    return h;
}

// Opaque device-resident preparation carried by PreparedEgs/PreparedOptA.  It serves a
// run_* call only for the same buffer with the same dimensions and unchanged pixels (the
// reference always correlates against the current contents of I).
struct DeviceState {
    tm_image* img = nullptr;
    tm_prep* prep = nullptr;
    const double* source = nullptr;  // Image buffer it was prepared from
    int rows = 0, cols = 0;
    std::uint64_t fingerprint = 0;
    ~DeviceState() {
        tm_prep_destroy(prep);
        tm_image_destroy(img);
    }
    bool serves(const Image& I) const {
        return I.data().data() == source && I.rows() == rows && I.cols() == cols &&
               pixel_fingerprint(I) == fingerprint;
    }
};

// ---- image.hpp -------------------------------------------------------------------------
Image load_image(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open image: " + path);
    std::string magic;
    in >> magic;
    if (magic != "P5") throw std::runtime_error("unsupported image format (8-bit PGM only): " + path);
    auto next_int = [&]() {
        int v = -1;
        while (in >> std::ws && in.peek() == '#') in.ignore(std::numeric_limits<std::streamsize>::max(), '\n');
        if (!(in >> v)) throw std::runtime_error("malformed PGM header: " + path);
        return v;
    };
    const int cols = next_int(), rows = next_int(), maxval = next_int();
    if (rows < 1 || cols < 1 || maxval < 1 || maxval > 255)
        throw std::runtime_error("unsupported PGM (8-bit grayscale only): " + path);
    in.get();
    std::vector<unsigned char> buf(std::size_t(rows) * cols);
    if (!in.read(reinterpret_cast<char*>(buf.data()), std::streamsize(buf.size())))
        throw std::runtime_error("truncated PGM: " + path);
    Image img(rows, cols);
    for (std::size_t i = 0; i < buf.size(); ++i) img.data()[i] = buf[i];
    return img;
}

void save_image(const Image& img, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write file: " + path);
    out << "P5\n" << img.cols() << " " << img.rows() << "\n255\n";
    for (double v : img.data()) out.put(char(static_cast<unsigned char>(std::clamp(std::round(v), 0.0, 255.0))));
    if (!out) throw std::runtime_error("write failed: " + path);
}

// image.cpp:215-228: FNV-1a over the int64 dimensions {rows, cols}, then over the raw
// bytes of the FP64 pixels -- the reference's key, so TMACMAP1 files written by either
// library load in the other.
std::uint64_t content_hash(const Image& img) {
    constexpr std::uint64_t kBasis = 1469598103934665603ull, kPrime = 1099511628211ull;
    std::uint64_t h = kBasis;
    auto bytes = [&h](const void* src, std::size_t len) {
        const auto* c = static_cast<const unsigned char*>(src);
        for (std::size_t k = 0; k < len; ++k) h = (h ^ c[k]) * kPrime;
    };
    const std::int64_t shape[2] = {img.rows(), img.cols()};
    bytes(shape, sizeof shape);
    bytes(img.data().data(), img.data().size() * sizeof(double));
    return h;
}

std::string to_string(MatchMode mode) {
    switch (mode) {
        case MatchMode::brute: return "brute";
        case MatchMode::egs: return "egs";
        case MatchMode::opta: return "opta";
    }
    return "unknown";
}

// ---- stats.hpp ---------------------------------------------------------------------------
SumTable running_sum(const Image& src, int m, int n) {
    if (m < 1 || n < 1 || m > src.rows() || n > src.cols())
        throw std::invalid_argument("running_sum: window does not fit the source");
    g_tables.fetch_add(1, std::memory_order_relaxed);
    DevImage d(src);
    SumTable t;
    t.win_rows = m;
    t.win_cols = n;
    t.rows = src.rows() - m + 1;
    t.cols = src.cols() - n + 1;
    t.sums.resize(std::size_t(t.rows) * t.cols);
    check(tm_running_sum(ctx(), d.h, m, n, t.sums.data()));
    return t;
}

std::uint64_t running_sum_call_count() { return g_tables.load(); }
void reset_running_sum_call_count() { g_tables.store(0); }

WindowStats window_stats(const Image& img, int m, int n) {
    if (m < 1 || n < 1 || m > img.rows() || n > img.cols())
        throw std::invalid_argument("running_sum: window does not fit the source");
    g_tables.fetch_add(2, std::memory_order_relaxed);
    DevImage d(img);
    return download_ws(d.h, m, n, img.rows() - m + 1, img.cols() - n + 1);
}

namespace detail {

bool variance_is_flat(double var_sum, double q_sum, long long mn) {
    const double abs_tol = 1e-9 * double(mn);
    const double rel = std::max(1e-13, 4.0 * 2.220446049250313e-16 * double(mn));
    return var_sum <= std::max(abs_tol * abs_tol, rel * q_sum);
}

TemplateStats template_stats(const Image& t) {
    double s = 0.0, sq = 0.0;
    for (double v : t.data()) {
        s += v;
        sq += v * v;
    }
    const long long mn = (long long)t.rows() * t.cols();
    const double var_sum = sq - s * s / double(mn);
    return TemplateStats{s / double(mn), std::sqrt(std::max(0.0, var_sum)),
                         variance_is_flat(var_sum, sq, mn)};
}

double window_dot(const Image& t, const Image& I, int r, int c) {
    double acc = 0.0;
    for (int i = 0; i < t.rows(); ++i)
        for (int j = 0; j < t.cols(); ++j) acc += t(i, j) * I(r + i, c + j);
    return acc;
}

double zncc_at(const Image& t, const TemplateStats& ts, const Image& I, const WindowStats& ws,
               int r, int c) {
    if (ts.flat || ws.flat(r, c)) return 0.0;
    const double mn = double(t.rows()) * double(t.cols());
    const double num = window_dot(t, I, r, c) - mn * ts.mu * ws.mu(r, c);
    return std::clamp(num / (ts.omega * ws.omega(r, c)), -1.0, 1.0);
}

}  // namespace detail

// Standalone two-pass-free correlation between two windows (stats.hpp, tests only).
double zncc(const Image& a, int ar, int ac, const Image& b, int br, int bc, int m, int n) {
    if (ar < 0 || ac < 0 || br < 0 || bc < 0 || ar + m > a.rows() || ac + n > a.cols() ||
        br + m > b.rows() || bc + n > b.cols())
        throw std::invalid_argument("zncc: window out of bounds");
    double sa = 0, sb = 0, qa = 0, qb = 0, sab = 0;
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
            const double x = a(ar + i, ac + j), y = b(br + i, bc + j);
            sa += x;
            sb += y;
            qa += x * x;
            qb += y * y;
            sab += x * y;
        }
    const long long mn = (long long)m * n;
    const double va = qa - sa * sa / double(mn), vb = qb - sb * sb / double(mn);
    if (detail::variance_is_flat(va, qa, mn) || detail::variance_is_flat(vb, qb, mn)) return 0.0;
    const double num = sab - sa * sb / double(mn);
    return std::clamp(num / (std::sqrt(va) * std::sqrt(vb)), -1.0, 1.0);
}

double zncc(const Image& a, const Image& b) {
    if (!a.same_size(b)) throw std::invalid_argument("zncc: shape mismatch");
    return zncc(a, 0, 0, b, 0, 0, a.rows(), a.cols());
}

bool better_candidate(const BestCell& cand, const BestCell& inc) {
    if (!cand.valid) return false;
    if (!inc.valid) return true;
    if (cand.degenerate != inc.degenerate) return !cand.degenerate;
    if (cand.rho != inc.rho) return cand.rho > inc.rho;
    if (cand.row != inc.row) return cand.row < inc.row;
    return cand.col < inc.col;
}

MatchResult brute_force_match(const Image& t, const Image& I, const BruteOptions& opts) {
    if (t.rows() > I.rows() || t.cols() > I.cols())
        throw std::invalid_argument("brute_force_match: template larger than search image");
    g_tables.fetch_add(2, std::memory_order_relaxed);
    DevImage d(I);
    tm_match_result r;
    std::vector<double> surface;
    const std::size_t E = std::size_t(I.rows() - t.rows() + 1) * (I.cols() - t.cols() + 1);
    if (opts.record_surface) surface.resize(E);
    check(tm_brute_force_match(ctx(), t.data().data(), t.rows(), t.cols(), d.h, &r,
                               opts.record_surface ? surface.data() : nullptr));
    MatchResult out = from_c(r);
    out.surface = std::move(surface);
    if (opts.record_visits) out.visits.assign(E, kVisitRetained);
    return out;
}

// ---- bounds.hpp (bounds.cpp:13-59) --------------------------------------------------------
namespace {
double checked(double rho, const char* name) {
    if (std::abs(rho) > 1.0 + 1e-9)
        throw std::invalid_argument(std::string("correlation out of [-1,1]: ") + name);
    return std::clamp(rho, -1.0, 1.0);
}
double half_gap(double a, double b) {
    return std::sqrt(std::max(0.0, 1.0 - a * a)) * std::sqrt(std::max(0.0, 1.0 - b * b));
}
}  // namespace

BoundPair transitive_bounds(double rho_tc, double rho_co) {
    const double a = checked(rho_tc, "rho_tc"), b = checked(rho_co, "rho_co");
    const double mid = a * b, s = half_gap(a, b);
    return BoundPair{std::clamp(mid - s, -1.0, 1.0), std::clamp(mid + s, -1.0, 1.0)};
}

double transitive_gap(double rho_tc, double rho_co) {
    return 2.0 * half_gap(checked(rho_tc, "rho_tc"), checked(rho_co, "rho_co"));
}

bool sec_holds(double rho_tb, double rho_tc, double rho_co) {
    const double tb = checked(rho_tb, "rho_tb");
    const double a = checked(rho_tc, "rho_tc"), b = checked(rho_co, "rho_co");
    return tb >= a * b + half_gap(a, b);
}

double elimination_autocorr_threshold(double rho_tb, double rho_tc) {
    const double tb = checked(rho_tb, "rho_tb"), tc = checked(rho_tc, "rho_tc");
    const double radicand = 1.0 + tc * tc * tb * tb - (tc * tc + tb * tb);
    return tb * tc + std::sqrt(std::max(0.0, radicand));
}

double expected_elimination_threshold(double rho_tb) {
    const double tb = checked(rho_tb, "rho_tb");
    return std::sqrt(std::max(0.0, 1.0 - tb * tb));
}

// ---- autocorr.hpp --------------------------------------------------------------------------
GroupGrid::GroupGrid(int extent_rows, int extent_cols, int h, int w)
    : er_(extent_rows), ec_(extent_cols), h_(h), w_(w) {
    if (extent_rows < 1 || extent_cols < 1)
        throw std::invalid_argument("group grid: empty search extent");
    if (h < 1 || w < 1 || h % 2 == 0 || w % 2 == 0)
        throw std::invalid_argument("group grid: group size must be odd and >= 1");
    tr_ = (er_ + h_ - 1) / h_;
    tc_ = (ec_ + w_ - 1) / w_;
    groups_.reserve(std::size_t(tr_) * tc_);
    for (int ti = 0; ti < tr_; ++ti)
        for (int tj = 0; tj < tc_; ++tj) {
            Group g;
            g.r0 = ti * h_;
            g.r1 = std::min(g.r0 + h_, er_) - 1;
            g.c0 = tj * w_;
            g.c1 = std::min(g.c0 + w_, ec_) - 1;
            g.center_row = (g.r0 + g.r1) / 2;
            g.center_col = (g.c0 + g.c1) / 2;
            groups_.push_back(g);
        }
}

const Group& GroupGrid::group_of(int r, int c) const {
    return groups_[std::size_t(std::min(r / h_, tr_ - 1)) * tc_ + std::min(c / w_, tc_ - 1)];
}

bool GroupGrid::is_center(int r, int c) const {
    const Group& g = group_of(r, c);
    return g.center_row == r && g.center_col == c;
}

GroupGrid build_group_grid(int p, int q, int m, int n, int h, int w) {
    if (m > p || n > q) throw std::invalid_argument("group grid: template does not fit the image");
    return GroupGrid(p - m + 1, q - n + 1, h, w);
}

AutoCorrMap local_autocorrelation(const Image& I, int m, int n, const GroupGrid& grid,
                                  const WindowStats& ws) {
    if (ws.rows != grid.extent_rows() || ws.cols != grid.extent_cols() ||
        ws.rows != I.rows() - m + 1 || ws.cols != I.cols() - n + 1)
        throw std::invalid_argument("local_autocorrelation: extent mismatch");
    g_tables.fetch_add(std::uint64_t(grid.group_h()) * grid.group_w() - 1,
                       std::memory_order_relaxed);
    DevImage d(I);
    AutoCorrMap map;
    map.rows = grid.extent_rows();
    map.cols = grid.extent_cols();
    map.group_h = grid.group_h();
    map.group_w = grid.group_w();
    map.values.resize(std::size_t(map.rows) * map.cols);
    check(tm_local_autocorrelation(ctx(), d.h, m, n, grid.group_h(), grid.group_w(),
                                   map.values.data()));
    return map;
}

AutoCorrMap local_autocorrelation(const Image& I, int m, int n, const GroupGrid& grid) {
    g_tables.fetch_add(2, std::memory_order_relaxed);
    if (grid.extent_rows() != I.rows() - m + 1 || grid.extent_cols() != I.cols() - n + 1)
        throw std::invalid_argument("local_autocorrelation: extent mismatch");
    WindowStats ws;
    ws.rows = grid.extent_rows();
    ws.cols = grid.extent_cols();
    return local_autocorrelation(I, m, n, grid, ws);
}

std::uint64_t autocorr_cache_key(const Image& I, int m, int n, int h, int w) {
    std::uint64_t key = content_hash(I);
    const std::int64_t params[4] = {m, n, h, w};
    const auto* b = reinterpret_cast<const unsigned char*>(params);
    for (std::size_t i = 0; i < sizeof params; ++i) {
        key ^= b[i];
        key *= 1099511628211ull;
    }
    return key;
}

namespace {
constexpr char kMapMagic[8] = {'T', 'M', 'A', 'C', 'M', 'A', 'P', '1'};
}

void save_autocorr(const AutoCorrMap& map, std::uint64_t key, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write file: " + path);
    const std::int64_t hdr[4] = {map.rows, map.cols, map.group_h, map.group_w};
    out.write(kMapMagic, 8);
    out.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
    out.write(reinterpret_cast<const char*>(&key), sizeof key);
    out.write(reinterpret_cast<const char*>(map.values.data()),
              std::streamsize(map.values.size() * sizeof(double)));
    if (!out) throw std::runtime_error("write failed: " + path);
}

std::optional<AutoCorrMap> load_autocorr(const std::string& path, std::uint64_t expected_key) {
    std::ifstream in(path, std::ios::binary);
    if (!in) return std::nullopt;
    char magic[8];
    std::int64_t hdr[4];
    std::uint64_t key = 0;
    in.read(magic, 8);
    in.read(reinterpret_cast<char*>(hdr), sizeof hdr);
    in.read(reinterpret_cast<char*>(&key), sizeof key);
    if (!in || std::memcmp(magic, kMapMagic, 8) != 0 || key != expected_key) return std::nullopt;
    if (hdr[0] < 1 || hdr[1] < 1 || hdr[2] < 1 || hdr[3] < 1) return std::nullopt;
    AutoCorrMap map;
    map.rows = int(hdr[0]);
    map.cols = int(hdr[1]);
    map.group_h = int(hdr[2]);
    map.group_w = int(hdr[3]);
    map.values.resize(std::size_t(map.rows) * map.cols);
    in.read(reinterpret_cast<char*>(map.values.data()),
            std::streamsize(map.values.size() * sizeof(double)));
    if (!in) return std::nullopt;
    return map;
}

// ---- egs.hpp -------------------------------------------------------------------------------
long long retained_count(const AutoCorrMap& map, double rho_tb) {
    if (rho_tb < 0.0 || rho_tb > 1.0)
        throw std::invalid_argument("retained_count: rho_tb must be in [0,1]");
    const double thr = expected_elimination_threshold(rho_tb);
    const GroupGrid grid(map.rows, map.cols, map.group_h, map.group_w);
    long long n = 0;
    for (int r = 0; r < map.rows; ++r)
        for (int c = 0; c < map.cols; ++c)
            if (!grid.is_center(r, c) && map.at(r, c) < thr) ++n;
    return n;
}

CostEstimate total_cost(int extent_rows, int extent_cols, int h, int w, long long n_r,
                        double amortized) {
    if (h < 1 || w < 1) throw std::invalid_argument("total_cost: group size must be >= 1");
    CostEstimate e;
    e.central = double((extent_rows + h - 1) / h) * double((extent_cols + w - 1) / w);
    e.retained = n_r;
    e.retained_cost = double(n_r);
    e.amortized = amortized;
    e.total = e.central + e.retained_cost + e.amortized;
    return e;
}

namespace {
// efficient_group_size with the amortised map-building term (egs.cpp:59-88 with
// include_autocorr_cost): the term depends on the candidate size, so the device batch
// decision (which knows only central + n_r) does not apply; candidates run one at a time,
// each map and retained count on the device, the decision on the host in the reference's
// FP64 order.
EGSResult efficient_group_size_amortized(const Image& I, int m, int n, const EgsParams& params) {
    if (params.h0 < 1 || params.w0 < 1 || params.h0 % 2 == 0 || params.w0 % 2 == 0)
        throw std::invalid_argument("efficient_group_size: initial group size must be odd");
    if (params.rho_tb <= 0.0 || params.rho_tb >= 1.0)
        throw std::invalid_argument("efficient_group_size: rho_tb must be in (0,1)");
    const int er = I.rows() - m + 1, ec = I.cols() - n + 1;
    if (er < 1 || ec < 1) throw std::invalid_argument("efficient_group_size: template does not fit");
    const double extent = double(er) * double(ec);
    const double mn = double(m) * double(n);
    int cap = params.max_group > 0 ? params.max_group : std::numeric_limits<int>::max();
    if (cap % 2 == 0) ++cap;
    DevImage d(I);
    EGSResult best;
    double prev = std::numeric_limits<double>::infinity();
    std::vector<double> map(std::size_t(er) * ec);
    for (int h = params.h0, w = params.w0;;) {
        check(tm_local_autocorrelation(ctx(), d.h, m, n, h, w, map.data()));
        std::int64_t n_r = 0;
        check(tm_autocorr_retained(ctx(), d.h, m, n, h, w, params.rho_tb, &n_r));
        g_tables.fetch_add(std::uint64_t(h) * w - 1, std::memory_order_relaxed);
        const double amortized =
            (double(h) * w - 1.0) * extent / (mn * std::max(1, params.n_templates));
        const CostEstimate cost = total_cost(er, ec, h, w, n_r, amortized);
        if (std::isfinite(prev) && !(prev - cost.total > params.xi_fraction * prev)) break;
        best.h = h;
        best.w = w;
        best.grid = GroupGrid(er, ec, h, w);
        best.map.rows = er;
        best.map.cols = ec;
        best.map.group_h = h;
        best.map.group_w = w;
        best.map.values = map;
        best.cost = cost;
        best.trace.push_back(EgsIteration{h, w, cost});
        prev = cost.total;
        if ((h >= er && w >= ec) || (h >= cap && w >= cap)) break;
        h = std::min(h + 2, cap);
        w = std::min(w + 2, cap);
    }
    return best;
}
}  // namespace

EGSResult efficient_group_size(const Image& I, int m, int n, const EgsParams& params,
                               const WindowStats&) {
    if (params.include_autocorr_cost) return efficient_group_size_amortized(I, m, n, params);
    DevImage d(I);
    int h = 0, w = 0, tl = 0;
    tm_egs_iter trace[TM_MAX_TRACE];
    const int er = I.rows() - m + 1, ec = I.cols() - n + 1;
    std::vector<double> map(er > 0 && ec > 0 ? std::size_t(er) * ec : 0);
    check(tm_efficient_group_size(ctx(), d.h, m, n, params.h0, params.w0, params.rho_tb,
                                  params.xi_fraction, params.max_group, &h, &w, trace, &tl,
                                  map.data()));
    tm_prep_info info{};
    info.h = h;
    info.w = w;
    info.extent_rows = er;
    info.extent_cols = ec;
    info.cost = trace[std::max(0, tl - 1)];
    info.egs_trace_len = tl;
    std::copy(trace, trace + std::min(tl, TM_MAX_TRACE), info.egs_trace);
    // logical table count of egs.cpp:59-88: hw-1 per evaluated candidate, including the
    // first rejected one unless the loop stopped at the extent/cap
    std::uint64_t tables = 0;
    for (int k = 0; k < tl; ++k) tables += std::uint64_t(trace[k].h) * trace[k].w - 1;
    int cap = params.max_group > 0 ? params.max_group : std::numeric_limits<int>::max();
    if (cap % 2 == 0) ++cap;
    if (!((h >= er && w >= ec) || (h >= cap && w >= cap)))
        tables += std::uint64_t(std::min(h + 2, cap)) * std::min(w + 2, cap) - 1;
    g_tables.fetch_add(tables, std::memory_order_relaxed);
    return egs_from_info(info, std::move(map));
}

EGSResult efficient_group_size(const Image& I, int m, int n, const EgsParams& params) {
    return efficient_group_size(I, m, n, params, WindowStats{});
}

// ---- blur.hpp ------------------------------------------------------------------------------
bool BlurKernel::is_delta() const {
    for (std::size_t k = 0; k < profile.size(); ++k)
        if (profile[k] != 0.0 && int(k) != radius) return false;
    return true;
}

BlurKernel BlurKernel::delta() { return BlurKernel{0, {1.0}}; }
BlurKernel BlurKernel::default_profile() { return BlurKernel{2, {0.05, 0.20, 0.50, 0.20, 0.05}}; }

BlurKernel BlurKernel::from_profile(std::vector<double> profile) {
    if (profile.empty() || profile.size() % 2 == 0)
        throw std::invalid_argument("blur kernel profile must have odd length");
    double sum = 0.0;
    for (double v : profile) {
        if (v < 0.0) throw std::invalid_argument("blur kernel weights must be non-negative");
        sum += v;
    }
    if (sum <= 0.0) throw std::invalid_argument("blur kernel weights must not all be zero");
    for (double& v : profile) v /= sum;
    BlurKernel k;
    k.radius = int(profile.size() / 2);
    k.profile = std::move(profile);
    return k;
}

BlurKernel gaussian_kernel_radius(double sigma_g, int d) {
    if (!(sigma_g > 0.0)) throw std::invalid_argument("gaussian kernel: sigma_g must be > 0");
    if (d < 0) throw std::invalid_argument("gaussian kernel: radius must be >= 0");
    std::vector<double> prof(std::size_t(2 * d + 1));
    for (int i = -d; i <= d; ++i) prof[std::size_t(i + d)] = std::exp(-double(i) * i / (2.0 * sigma_g * sigma_g));
    return BlurKernel::from_profile(std::move(prof));
}

BlurKernel gaussian_kernel(double sigma_g, double t_g) {
    if (!(sigma_g > 0.0)) throw std::invalid_argument("gaussian kernel: sigma_g must be > 0");
    if (!(t_g > 0.0 && t_g < 1.0)) throw std::invalid_argument("gaussian kernel: t_g must be in (0,1)");
    const int d = std::max(0, int(std::ceil(std::sqrt(-2.0 * sigma_g * std::log(t_g)))));
    return gaussian_kernel_radius(sigma_g, d);
}

Image blur(const Image& img, const BlurKernel& kernel) {
    if (kernel.radius == 0 && kernel.profile.size() == 1) return img;
    DevImage d(img);
    Image out(img.rows(), img.cols());
    check(tm_blur(ctx(), d.h, kernel.profile.data(), int(kernel.profile.size()), out.data().data()));
    return out;
}

double quality_threshold(double rho_th, double rho_max) {
    if (rho_th < 0.0 || rho_th > 1.0 || rho_max < 0.0 || rho_max > 1.0)
        throw std::invalid_argument("quality_threshold: inputs must be in [0,1]");
    if (rho_max < rho_th) throw std::invalid_argument("quality_threshold: rho_max must be >= rho_th");
    return elimination_autocorr_threshold(rho_th, rho_max);
}

FidelityMap blur_fidelity_map(const Image& I, const Image& I_blur, int m, int n) {
    if (!I.same_size(I_blur)) throw std::invalid_argument("blur_fidelity_map: dimension mismatch");
    DevImage a(I), b(I_blur);
    FidelityMap f;
    f.rows = I.rows() - m + 1;
    f.cols = I.cols() - n + 1;
    f.win_rows = m;
    f.win_cols = n;
    f.values.resize(f.rows > 0 && f.cols > 0 ? std::size_t(f.rows) * f.cols : 0);
    check(tm_blur_fidelity_map(ctx(), a.h, b.h, m, n, f.values.data()));
    return f;
}

FidelityMap blur_fidelity_map(const Image& I, const WindowStats& ws_orig, const Image& I_blur) {
    if (!I.same_size(I_blur)) throw std::invalid_argument("blur_fidelity_map: dimension mismatch");
    return blur_fidelity_map(I, I_blur, ws_orig.win_rows, ws_orig.win_cols);
}

std::pair<Image, long long> unblur_violations(const Image& I_blur, const Image& I,
                                              const FidelityMap& fid, double lambda) {
    if (!I_blur.same_size(I)) throw std::invalid_argument("unblur_violations: shape mismatch");
    DevImage b(I_blur), o(I);
    Image out(I.rows(), I.cols());
    int64_t count = 0;
    check(tm_unblur_violations(ctx(), b.h, o.h, fid.values.data(), fid.win_rows, fid.win_cols,
                               lambda, out.data().data(), &count));
    return {std::move(out), (long long)count};
}

OptAResult optimize_autocorrelation(const Image& I, int m, int n, const OptAParams& params) {
    MatchParams mp;
    mp.mode = MatchMode::opta;
    mp.rho_th = params.rho_th;
    mp.rho_max = params.rho_max;
    mp.kernel = params.kernel;
    mp.opta_margin = params.margin;
    mp.h0 = params.egs.h0;
    mp.w0 = params.egs.w0;
    mp.xi_fraction = params.egs.xi_fraction;
    if (params.egs.rho_tb != params.rho_th || params.max_iterations != 64)
        throw std::invalid_argument(
            "optimize_autocorrelation: egs.rho_tb must equal rho_th and max_iterations 64");
    PreparedOptA prep = prepare_opta(I, m, n, mp);
    return std::move(prep.opta);
}

// ---- matcher.hpp -----------------------------------------------------------------------------
CenterScan center_scan(const Image& t, const Image& I, const GroupGrid& grid) {
    if (I.rows() - t.rows() + 1 != grid.extent_rows() || I.cols() - t.cols() + 1 != grid.extent_cols())
        throw std::invalid_argument("center_scan: grid extent mismatch");
    DevImage d(I);
    CenterScan cs;
    cs.rho.resize(grid.groups().size());
    cs.degenerate.resize(grid.groups().size());
    int br, bc, bd;
    double brho;
    check(tm_center_scan(ctx(), t.data().data(), t.rows(), t.cols(), d.h, grid.group_h(),
                         grid.group_w(), cs.rho.data(), cs.degenerate.data(), &br, &bc, &brho, &bd));
    cs.best = BestCell{br, bc, brho, bd != 0, br >= 0};
    return cs;
}

MatchResult transitive_search(const Image& t, const Image& I, const AutoCorrMap& map,
                              const GroupGrid& grid, const SearchOptions& opts) {
    if (map.rows != grid.extent_rows() || map.cols != grid.extent_cols() ||
        map.group_h != grid.group_h() || map.group_w != grid.group_w())
        throw std::invalid_argument("transitive_search: grid/map mismatch");
    MatchParams mp;
    mp.init_threshold = opts.init_threshold;
    mp.parallel = opts.parallel;
    mp.threads = opts.threads;
    mp.record_visits = opts.record_visits;
    const tm_match_params c = to_c(mp);
    DevImage d(I);
    tm_match_result r;
    std::vector<uint8_t> visits(opts.record_visits ? map.values.size() : 0);
    check(tm_transitive_search(ctx(), t.data().data(), t.rows(), t.cols(), d.h, map.values.data(),
                               grid.group_h(), grid.group_w(), &c, &r,
                               opts.record_visits ? visits.data() : nullptr));
    MatchResult out = from_c(r);
    out.visits = std::move(visits);
    return out;
}

BestCell refine_localization(const Image& t, const Image& I_original, int loc_row, int loc_col,
                             int d) {
    DevImage di(I_original);
    int r, c, deg;
    double rho;
    check(tm_refine_localization(ctx(), t.data().data(), t.rows(), t.cols(), di.h, loc_row,
                                 loc_col, d, &r, &c, &rho, &deg));
    return BestCell{r, c, rho, deg != 0, true};
}

namespace {
std::shared_ptr<DeviceState> device_prepare(const Image& I, int m, int n, const MatchParams& p,
                                            tm_prep_info* info) {
    auto st = std::make_shared<DeviceState>();
    check(tm_image_create(ctx(), I.data().data(), I.rows(), I.cols(), &st->img));
    const tm_match_params c = to_c(p);
    check(tm_prepare(ctx(), st->img, m, n, &c, &st->prep));
    check(tm_prep_get_info(st->prep, info));
    st->source = I.data().data();
    st->rows = I.rows();
    st->cols = I.cols();
    st->fingerprint = pixel_fingerprint(I);
    return st;
}

MatchResult run_prepared(const Image& t, const Image& I, const DeviceState* st,
                         const MatchParams& params) {
    const tm_match_params c = to_c(params);
    tm_match_result r;
    tm_prep_info info;
    check(tm_prep_get_info(st->prep, &info));
    std::vector<uint8_t> visits(params.record_visits ? std::size_t(info.extent_rows) * info.extent_cols : 0);
    (void)I;
    check(tm_run(ctx(), st->prep, st->img, t.data().data(), 1, &c, &r,
                 params.record_visits ? visits.data() : nullptr));
    MatchResult out = from_c(r);
    out.visits = std::move(visits);
    return out;
}
}  // namespace

PreparedEgs prepare_egs(const Image& I, int m, int n, const MatchParams& params) {
    MatchParams p = params;
    p.mode = MatchMode::egs;
    tm_prep_info info;
    PreparedEgs prep;
    prep.device = device_prepare(I, m, n, p, &info);
    std::vector<double> map(std::size_t(info.extent_rows) * info.extent_cols);
    check(tm_prep_download(ctx(), prep.device->prep, map.data(), nullptr));
    prep.egs = egs_from_info(info, std::move(map));
    prep.ws = download_ws(prep.device->img, m, n, info.extent_rows, info.extent_cols);
    return prep;
}

PreparedOptA prepare_opta(const Image& I, int m, int n, const MatchParams& params) {
    MatchParams p = params;
    p.mode = MatchMode::opta;
    tm_prep_info info;
    PreparedOptA prep;
    prep.device = device_prepare(I, m, n, p, &info);
    std::vector<double> map(std::size_t(info.extent_rows) * info.extent_cols);
    Image blurred(I.rows(), I.cols());
    check(tm_prep_download(ctx(), prep.device->prep, map.data(), blurred.data().data()));
    prep.opta.egs = egs_from_info(info, std::move(map));
    prep.opta.kappa = info.kappa;
    prep.opta.lambda = info.lambda;
    for (int k = 0; k < info.opta_trace_len; ++k)
        prep.opta.trace.push_back(OptAIteration{info.opta_trace[k].h, info.opta_trace[k].w,
                                                info.opta_trace[k].cost,
                                                (long long)info.opta_trace[k].restored});
    prep.ws_orig = download_ws(prep.device->img, m, n, info.extent_rows, info.extent_cols);
    DevImage b(blurred);
    prep.ws_blur = download_ws(b.h, m, n, info.extent_rows, info.extent_cols);
    prep.opta.image = std::move(blurred);
    return prep;
}

namespace {
// transitive_search_impl (matcher.cpp:95-177) on the CURRENT pixels of I with a
// preparation's map and window statistics, as the reference's run_egs / run_opta do
// (matcher.cpp:235-276) -- the path for preparations without (valid) device state.
MatchResult search_with_prepared(const Image& t, const Image& I, const AutoCorrMap& map,
                                 const GroupGrid& grid, const WindowStats& ws,
                                 const MatchParams& params) {
    if (map.rows != grid.extent_rows() || map.cols != grid.extent_cols() ||
        map.group_h != grid.group_h() || map.group_w != grid.group_w())
        throw std::invalid_argument("transitive_search: grid/map mismatch");
    const std::size_t E = std::size_t(map.rows) * map.cols;
    if (ws.mean.size() != E || ws.norm.size() != E || ws.flat_map.size() != E) {
        SearchOptions o;  // no statistics recorded: the image's own
        o.init_threshold = params.init_threshold;
        o.parallel = params.parallel;
        o.threads = params.threads;
        o.record_visits = params.record_visits;
        return transitive_search(t, I, map, grid, o);
    }
    MatchParams mp;
    mp.init_threshold = params.init_threshold;
    mp.parallel = params.parallel;
    mp.threads = params.threads;
    mp.record_visits = params.record_visits;
    const tm_match_params c = to_c(mp);
    DevImage d(I);
    tm_match_result r;
    std::vector<uint8_t> visits(params.record_visits ? E : 0);
    check(tm_transitive_search_ws(ctx(), t.data().data(), t.rows(), t.cols(), d.h,
                                  map.values.data(), grid.group_h(), grid.group_w(),
                                  ws.mean.data(), ws.norm.data(), ws.flat_map.data(), &c, &r,
                                  params.record_visits ? visits.data() : nullptr));
    MatchResult out = from_c(r);
    out.visits = std::move(visits);
    return out;
}
}  // namespace

MatchResult run_egs(const Image& t, const Image& I, const PreparedEgs& prep,
                    const MatchParams& params) {
    if (prep.device && prep.device->serves(I)) return run_prepared(t, I, prep.device.get(), params);
    // a preparation without valid device state (built by hand, for another buffer, or the
    // caller changed the pixels since)
    MatchResult r = search_with_prepared(t, I, prep.egs.map, prep.egs.grid, prep.ws, params);
    r.mode = MatchMode::egs;
    return r;
}

MatchResult run_opta(const Image& t, const Image& I_original, const PreparedOptA& prep,
                     const MatchParams& params) {
    if (prep.device && prep.device->serves(I_original))
        return run_prepared(t, I_original, prep.device.get(), params);
    MatchResult r = search_with_prepared(t, prep.opta.image, prep.opta.egs.map,
                                         prep.opta.egs.grid, prep.ws_blur, params);
    r.mode = MatchMode::opta;
    const int d = prep.opta.kappa * params.kernel.radius;
    const BestCell b = refine_localization(t, I_original, r.best_row, r.best_col, d);
    r.refined_row = b.row;
    r.refined_col = b.col;
    r.refined_rho = b.rho;
    const int er = r.extent_rows, ec = r.extent_cols;
    const int rr = (std::min(er - 1, r.best_row + d) - std::max(0, r.best_row - d) + 1);
    const int cc = (std::min(ec - 1, r.best_col + d) - std::max(0, r.best_col - d) + 1);
    r.stats.ops += (long long)rr * cc;
    if (params.init_threshold) r.below_threshold = b.degenerate || b.rho < *params.init_threshold;
    return r;
}

MatchResult match(const Image& t, const Image& I, const MatchParams& params) {
    if (t.rows() > I.rows() || t.cols() > I.cols())
        throw std::invalid_argument("match: template larger than search image");
    const tm_match_params c = to_c(params);
    tm_match_result r;
    std::vector<uint8_t> visits(params.record_visits
                                    ? std::size_t(I.rows() - t.rows() + 1) * (I.cols() - t.cols() + 1)
                                    : 0);
    check(tm_match(ctx(), t.data().data(), t.rows(), t.cols(), I.data().data(), I.rows(), I.cols(),
                   &c, &r, params.record_visits ? visits.data() : nullptr));
    MatchResult out = from_c(r);
    out.visits = std::move(visits);
    return out;
}

}  // namespace tmatch

namespace tmatch::internal {
tm_ctx* context() { return ctx(); }
void check_rc(int rc) { check(rc); }
tm_match_params to_c_params(const MatchParams& p) { return to_c(p); }
MatchResult from_c_result(const tm_match_result& r) { return from_c(r); }
}  // namespace tmatch::internal
