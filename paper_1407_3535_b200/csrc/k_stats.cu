// k_stats.cu -- image preparation, window statistics and running sums (sm_100a).
//
// Integer path (8-bit images, the reference's input domain): window sums S and Q are
// exact integers, accumulated with a row-sliding pass then a column-sliding pass; the
// FP64 epilogue replays stats.cpp:83-92 with _rn intrinsics, so mu/omega/flat are bit
// identical to the reference.
//
// Replica path (non-integer images, e.g. OptA's blurred image): the reference's FP64
// prefix table (stats.cpp:26-37: sequential row accumulation, then prefix[r+1] =
// prefix[r] + row_acc) is rebuilt in the same operation order -- one thread scans one
// row (through a shared-memory transpose for coalescing), one thread accumulates one
// column -- and window sums use the reference's difference order (stats.cpp:50).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kernels.hpp"
#include "tm_common.cuh"

namespace tmk {

namespace {

__global__ void k_check_u8(const double* __restrict__ img, size_t n, int* bad) {
    int local = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const double v = img[i];
        if (!(v >= 0.0 && v <= 255.0) || v != rint(v)) local = 1;
    }
    if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(bad, 1);
}

__global__ void k_f64_to_u8(const double* __restrict__ img, size_t n, uint8_t* __restrict__ out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        out[i] = uint8_t(img[i]);
}

__global__ void k_u8_to_f64(const uint8_t* __restrict__ img, size_t n, double* __restrict__ out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        out[i] = double(img[i]);
}

// Float copy with a padded pitch; the pad columns are zero so vector loads past the last
// column read zeros.
__global__ void k_u8_to_f32(const uint8_t* __restrict__ img, int p, int q, float* __restrict__ out,
                            int pitch) {
    const int r = blockIdx.y;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < pitch; c += gridDim.x * blockDim.x)
        out[size_t(r) * pitch + c] = c < q ? float(img[size_t(r) * q + c]) : 0.0f;
}

// Sum of squares of all pixels (q_total for 8-bit images, exact in u64): 16-byte loads,
// block reduction, one atomic per block.
__global__ void __launch_bounds__(256) k_sum_sq_u8(const uint8_t* __restrict__ img, size_t n,
                                                   unsigned long long* acc_ctr, int rows,
                                                   int cols, double* noise_out) {
    pdl_wait();
    // acc_ctr[0]: running sum, acc_ctr[1]: finished-block counter; both zero on entry and
    // reset by the last block, which also writes prefix_noise (stats.cpp:79-81).
    unsigned long long* out = acc_ctr;
    __shared__ unsigned long long part[8];
    unsigned long long acc = 0;
    const size_t nv = n / 16;
    const uint4* v4 = reinterpret_cast<const uint4*>(img);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nv;
         i += size_t(gridDim.x) * blockDim.x) {
        const uint4 v = __ldg(v4 + i);
        const unsigned w[4] = {v.x, v.y, v.z, v.w};
        unsigned s = 0;  // 16 squares <= 16 * 65025 fit in 32 bits
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const unsigned x = (w[k] >> (8 * b)) & 0xffu;
                s += x * x;
            }
        acc += s;
    }
    if (blockIdx.x == 0)  // tail bytes
        for (size_t i = nv * 16 + threadIdx.x; i < n; i += blockDim.x) {
            const unsigned x = img[i];
            acc += x * x;
        }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
        atomicAdd(out, t);
        __threadfence();
        const unsigned long long ticket = atomicAdd(acc_ctr + 1, 1ull);
        if (ticket == gridDim.x - 1) {  // last block: every partial is in
            const unsigned long long q_total = atomicAdd(out, 0ull);
            *noise_out = __dmul_rn(__dmul_rn(double(rows + cols), kEps), double(q_total));
            acc_ctr[0] = 0ull;
            acc_ctr[1] = 0ull;
        }
    }
}

// q_total for non-integer images (stats.cpp:78-81).  The reference adds the squares
// sequentially, and a parallel sum differs from that in the last bits, which matters only
// for windows whose variance sits on the prefix-noise floor.  So the flat decision is
// made against a guaranteed bracket [pn_lo, pn_hi] of the reference's prefix_noise, and
// only if some window falls inside the bracket is the sequential sum replayed on the
// device (one warp, reference order) and that window-statistics pass redone with the
// exact value.  Layout of the image's noise block `nb` (doubles):
//   [0] q_par  [1] prefix_noise (exact once resolved)  [2] pn_lo  [3] pn_hi
//   [4] ambiguous-window count (u64)  [5] resolved flag (u64)
constexpr int kSqBlocks = 592, kSqThreads = 256;

__global__ void __launch_bounds__(kSqThreads)
    k_sum_sq_f64(const double* __restrict__ img, size_t n, double* __restrict__ part) {
    double acc = 0.0;  // fixed per-thread order: deterministic, unlike atomics
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        acc = __dadd_rn(acc, __dmul_rn(img[i], img[i]));
    acc = warp_sum(acc);
    __shared__ double ws[kSqThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < kSqThreads / 32; ++w) b = __dadd_rn(b, ws[w]);
        part[blockIdx.x] = b;
    }
}

// All addends are >= 0, so any summation order of k terms is within gamma_k = k*u/(1-k*u)
// of the exact sum S* of the (identically rounded) squares: the sequential sum within
// gamma_n, this tree within gamma_depth.  The bracket of q_seq is then monotonically
// mapped through prefix_noise = RN(RN((rows + cols) * eps) * q_total).
__global__ void k_prefix_noise_f64(const double* __restrict__ part, int nb, size_t n, int rows,
                                   int cols, double* __restrict__ nbk, int widen) {
    double q = 0.0;
    for (int b = 0; b < nb; ++b) q = __dadd_rn(q, part[b]);
    const double per_thread = double((n + size_t(nb) * kSqThreads - 1) / (size_t(nb) * kSqThreads));
    const double u = 1.0000001 * 1.1102230246251565e-16;  // 2^-53 with slack
    const double depth = per_thread + 5.0 + 3.0 + double(nb);
    const double d_par = depth * u / (1.0 - depth * u);
    const double d_seq = double(n) * u / (1.0 - double(n) * u);
    const double delta = __ddiv_ru(__dadd_ru(d_par, d_seq), __dsub_rd(1.0, d_par));
    const double q_lo = __dmul_rd(q, __dsub_rd(1.0, delta));
    const double q_hi = __dmul_ru(q, __dadd_ru(1.0, delta));
    const double c = __dmul_rn(double(rows + cols), kEps);
    nbk[0] = q;
    nbk[1] = __dmul_rn(c, q);
    nbk[2] = widen ? -INFINITY : __dmul_rn(c, q_lo);  // widen: test hook, every window
    nbk[3] = widen ? INFINITY : __dmul_rn(c, q_hi);   // undecided -> the sequential replay
    reinterpret_cast<unsigned long long*>(nbk)[4] = 0ull;
    reinterpret_cast<unsigned long long*>(nbk)[5] = 0ull;
}

// The reference's sequential q_total (stats.cpp:79: q_total += v*v over the row-major
// image), replayed only when a window was undecided: one warp streams coalesced chunks
// of squares into shared memory and lane 0 adds them in order.
__global__ void __launch_bounds__(32)
    k_resolve_prefix_noise(const double* __restrict__ img, size_t n, int rows, int cols,
                           double* __restrict__ nbk) {
    auto* cnt = reinterpret_cast<unsigned long long*>(nbk);
    if (cnt[4] == 0ull || cnt[5] != 0ull) return;
    constexpr int kC = 32 * 16;
    __shared__ double sq[kC];
    double q = 0.0;
    for (size_t base = 0; base < n; base += kC) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const size_t i = base + size_t(j) * 32 + threadIdx.x;
            const double v = i < n ? img[i] : 0.0;
            sq[j * 32 + threadIdx.x] = __dmul_rn(v, v);
        }
        __syncwarp();
        if (threadIdx.x == 0) {
            const int lim = int(n - base < size_t(kC) ? n - base : size_t(kC));
            for (int k = 0; k < lim; ++k) q = __dadd_rn(q, sq[k]);
        }
        __syncwarp();
    }
    if (threadIdx.x == 0) {
        const double pn = __dmul_rn(__dmul_rn(double(rows + cols), kEps), q);
        nbk[0] = q;
        nbk[1] = pn;
        nbk[2] = pn;
        nbk[3] = pn;
        cnt[5] = 1ull;
    }
}

constexpr int kChunk = 32;

// Row pass: hs[r][c] = sum_{j<n} I(r, c+j), hq likewise for I^2; one thread owns kChunk
// consecutive output columns of one row and slides the window.
__global__ void k_hsum_u8(const uint8_t* __restrict__ img, int p, int q, int n,
                          int* __restrict__ hs, int* __restrict__ hq) {
    const int ec = q - n + 1;
    const int r = blockIdx.y;
    const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * kChunk;
    if (c0 >= ec) return;
    const uint8_t* row = img + size_t(r) * q;
    int s = 0, sq = 0;
    for (int j = 0; j < n; ++j) {
        const int v = row[c0 + j];
        s += v;
        sq += v * v;
    }
    const int c1 = min(c0 + kChunk, ec);
    int* os = hs + size_t(r) * ec;
    int* oq = hq ? hq + size_t(r) * ec : nullptr;
    for (int c = c0; c < c1; ++c) {
        os[c] = s;
        if (oq) oq[c] = sq;
        if (c + 1 < c1) {
            const int vin = row[c + n], vout = row[c];
            s += vin - vout;
            sq += vin * vin - vout * vout;
        }
    }
}

// Column pass + FP64 epilogue: S, Q over m rows of the row sums; one thread owns kChunk
// consecutive output rows of one column (coalesced across the warp).
__global__ void k_vsum_stats(const int* __restrict__ hs, const int* __restrict__ hq, int p,
                             int ec, int m, int n, const double* __restrict__ pn, DevStats st) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int er = p - m + 1;
    const int r0 = blockIdx.y * kChunk;
    if (c >= ec || r0 >= er) return;
    long long s = 0, sq = 0;
    for (int i = 0; i < m; ++i) {
        s += hs[size_t(r0 + i) * ec + c];
        sq += hq[size_t(r0 + i) * ec + c];
    }
    const double inv_mn = 1.0 / (double(m) * double(n));
    const long long mn = (long long)m * n;
    const double prefix_noise = *pn;
    const int r1 = min(r0 + kChunk, er);
    for (int r = r0; r < r1; ++r) {
        const size_t k = size_t(r) * ec + c;
        double mu, om;
        uint8_t fl;
        window_epilogue(double(s), double(sq), inv_mn, mn, prefix_noise, mu, om, fl);
        st.mu[k] = mu;
        st.omega[k] = om;
        st.flat[k] = fl;
        if (r + 1 < r1) {
            s += hs[size_t(r + m) * ec + c] - hs[size_t(r) * ec + c];
            sq += hq[size_t(r + m) * ec + c] - hq[size_t(r) * ec + c];
        }
    }
}

__global__ void k_vsum_only(const int* __restrict__ hs, int p, int ec, int m,
                            double* __restrict__ out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int er = p - m + 1;
    const int r0 = blockIdx.y * kChunk;
    if (c >= ec || r0 >= er) return;
    long long s = 0;
    for (int i = 0; i < m; ++i) s += hs[size_t(r0 + i) * ec + c];
    const int r1 = min(r0 + kChunk, er);
    for (int r = r0; r < r1; ++r) {
        out[size_t(r) * ec + c] = double(s);
        if (r + 1 < r1) s += hs[size_t(r + m) * ec + c] - hs[size_t(r) * ec + c];
    }
}

// ---- replica prefix ------------------------------------------------------------------
__device__ __forceinline__ double src_value(const ProdSrc& s, int a, int b) {
    const double x = s.X[size_t(a + s.xr) * s.xq + (b + s.xc)];
    if (s.square) return __dmul_rn(x, x);
    if (s.Y) return __dmul_rn(x, s.Y[size_t(a + s.yr) * s.yq + (b + s.yc)]);
    return x;
}

// The 32 source values of a warp's 32-row x 32-column tile column `c` (rows r0..r0+31):
// every load issued before any use (branch-free: the source kind is uniform), so the tile
// costs one memory latency instead of 32 serialised ones.
__device__ __forceinline__ void src_column32(const ProdSrc& s, int r0, int c, int rows, int cols,
                                             double (&v)[32]) {
    const bool cin = c < cols;
    const double* xp = s.X + size_t(r0 + s.xr) * s.xq + (c + s.xc);
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = (cin && r0 + k < rows) ? __ldg(xp + size_t(k) * s.xq) : 0.0;
    if (s.square) {
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = __dmul_rn(v[k], v[k]);
    } else if (s.Y) {
        const double* yp = s.Y + size_t(r0 + s.yr) * s.yq + (c + s.yc);
#pragma unroll
        for (int h = 0; h < 32; h += 16) {  // (two halves: register budget)
            double y[16];
#pragma unroll
            for (int k = 0; k < 16; ++k)
                y[k] = (cin && r0 + h + k < rows) ? __ldg(yp + size_t(h + k) * s.yq) : 0.0;
#pragma unroll
            for (int k = 0; k < 16; ++k) v[h + k] = __dmul_rn(v[h + k], y[k]);
        }
    }
}

// One warp = 32 rows.  Tiles of 32 columns are staged through shared memory so global
// reads/writes stay coalesced while each lane scans its own row sequentially
// (row_acc += v, stats.cpp:34).
__global__ void k_rowscan(ProdSrc src, int rows, int cols, double* __restrict__ rowacc) {
    if (src.stop && *src.stop) return;
    __shared__ double tile[4][32][33];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int r0 = (blockIdx.x * 4 + wid) * 32;
    if (r0 >= rows) return;
    double acc = 0.0;
    for (int c0 = 0; c0 < cols; c0 += 32) {
        const int c = c0 + lane;
        double v[32];
        src_column32(src, r0, c, rows, cols, v);
#pragma unroll
        for (int k = 0; k < 32; ++k) tile[wid][k][lane] = v[k];
        __syncwarp();
        const int cn = min(32, cols - c0);
        for (int j = 0; j < cn; ++j) {
            acc = __dadd_rn(acc, tile[wid][lane][j]);
            tile[wid][lane][j] = acc;
        }
        __syncwarp();
        for (int k = 0; k < 32; ++k) {
            const int r = r0 + k;
            if (r < rows && c < cols) rowacc[size_t(r) * cols + c] = tile[wid][k][lane];
        }
        __syncwarp();
    }
}

// prefix[(r+1)][c+1] = prefix[r][c+1] + rowacc[r][c]  (stats.cpp:35), one thread per column.
__global__ void k_colacc(const double* __restrict__ rowacc, int rows, int cols,
                         double* __restrict__ prefix, const int* stop) {
    if (stop && *stop) return;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t pw = size_t(cols) + 1;
    if (c > cols) return;
    prefix[c] = 0.0;  // zero top row
    if (c == cols) {
        for (int r = 0; r < rows; ++r) prefix[size_t(r + 1) * pw] = 0.0;  // zero first col
        return;
    }
    // rows in chunks of 16: the next chunk's loads are in flight while this chunk is
    // accumulated (the additions stay sequential, stats.cpp:35)
    constexpr int kC = 16;
    double cur[kC], nxt[kC];
#pragma unroll
    for (int j = 0; j < kC; ++j) cur[j] = j < rows ? rowacc[size_t(j) * cols + c] : 0.0;
    double acc = 0.0;
    for (int r0 = 0; r0 < rows; r0 += kC) {
#pragma unroll
        for (int j = 0; j < kC; ++j)
            nxt[j] = r0 + kC + j < rows ? rowacc[size_t(r0 + kC + j) * cols + c] : 0.0;
#pragma unroll
        for (int j = 0; j < kC; ++j) {
            if (r0 + j >= rows) break;
            acc = __dadd_rn(acc, cur[j]);
            prefix[size_t(r0 + j + 1) * pw + c + 1] = acc;
        }
#pragma unroll
        for (int j = 0; j < kC; ++j) cur[j] = nxt[j];
    }
}

// Batched replica prefixes: grid.y = offset k of a ProdBatch, each with its own source
// (X, Y row/column offsets), extent and scratch slot; per offset the operations are
// exactly k_rowscan / k_colacc's (same sequential order per row / column), so only the
// amount of independent work per launch grows (one offset alone leaves ~128 warps).
__global__ void k_rowscan_b(ProdBatch b, double* __restrict__ rowacc) {
    const int k = blockIdx.y;
    const ProdSrc src = b.src[k];
    if (src.stop && *src.stop) return;
    const int rows = b.rows[k], cols = b.cols[k];
    double* out = rowacc + size_t(k) * b.slot;
    __shared__ double tile[4][32][33];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int r0 = (blockIdx.x * 4 + wid) * 32;
    if (r0 >= rows) return;
    double acc = 0.0;
    for (int c0 = 0; c0 < cols; c0 += 32) {
        const int c = c0 + lane;
        double v[32];
        src_column32(src, r0, c, rows, cols, v);
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) tile[wid][kk][lane] = v[kk];
        __syncwarp();
        const int cn = min(32, cols - c0);
        for (int jj = 0; jj < cn; ++jj) {
            acc = __dadd_rn(acc, tile[wid][lane][jj]);
            tile[wid][lane][jj] = acc;
        }
        __syncwarp();
        for (int kk = 0; kk < 32; ++kk) {
            const int r = r0 + kk;
            if (r < rows && c < cols) out[size_t(r) * cols + c] = tile[wid][kk][lane];
        }
        __syncwarp();
    }
}

__global__ void k_colacc_b(ProdBatch b, const double* __restrict__ rowacc,
                           double* __restrict__ prefix) {
    const int k = blockIdx.y;
    if (b.src[k].stop && *b.src[k].stop) return;
    const int rows = b.rows[k], cols = b.cols[k];
    const double* in = rowacc + size_t(k) * b.slot;
    double* pre = prefix + size_t(k) * b.pslot;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t pw = size_t(cols) + 1;
    if (c > cols) return;
    pre[c] = 0.0;  // zero top row
    if (c == cols) {
        for (int r = 0; r < rows; ++r) pre[size_t(r + 1) * pw] = 0.0;  // zero first col
        return;
    }
    constexpr int kC = 16;  // as k_colacc: next chunk's loads in flight
    double cur[kC], nxt[kC];
#pragma unroll
    for (int j = 0; j < kC; ++j) cur[j] = j < rows ? in[size_t(j) * cols + c] : 0.0;
    double acc = 0.0;
    for (int r0 = 0; r0 < rows; r0 += kC) {
#pragma unroll
        for (int j = 0; j < kC; ++j)
            nxt[j] = r0 + kC + j < rows ? in[size_t(r0 + kC + j) * cols + c] : 0.0;
#pragma unroll
        for (int j = 0; j < kC; ++j) {
            if (r0 + j >= rows) break;
            acc = __dadd_rn(acc, cur[j]);
            pre[size_t(r0 + j + 1) * pw + c + 1] = acc;
        }
#pragma unroll
        for (int j = 0; j < kC; ++j) cur[j] = nxt[j];
    }
}

__global__ void k_window_diff(const double* __restrict__ prefix, int rows, int cols, int m, int n,
                              double* __restrict__ out) {
    const int er = rows - m + 1, ec = cols - n + 1;
    const size_t pw = size_t(cols) + 1;
    const size_t total = size_t(er) * ec;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < total;
         k += size_t(gridDim.x) * blockDim.x) {
        const int r = int(k / ec), c = int(k % ec);
        const double* top = prefix + size_t(r) * pw;
        const double* bot = prefix + size_t(r + m) * pw;
        out[k] = __dadd_rn(__dsub_rn(__dsub_rn(bot[c + n], top[c + n]), bot[c]), top[c]);
    }
}

// stats.cpp:84-92 on replica window sums (non-integer images).  The prefix-noise floor is
// tested against the bracket [pn_lo, pn_hi] (k_prefix_noise_f64): outside it the decision
// equals the reference's; inside it the window is counted as undecided.  `fix` = the
// redo pass after k_resolve_prefix_noise: runs only if windows were undecided, with the
// exact floor, and clears the count.
__global__ void k_stats_from_sums(const double* __restrict__ S, const double* __restrict__ Q,
                                  size_t E, int m, int n, double* __restrict__ nbk,
                                  DevStats st, int fix) {
    auto* cnt = reinterpret_cast<unsigned long long*>(nbk);
    if (fix && cnt[4] == 0ull) return;
    const double pn = nbk[1], pn_lo = nbk[2], pn_hi = nbk[3];
    const double inv_mn = 1.0 / (double(m) * double(n));
    const long long mn = (long long)m * n;
    unsigned undecided = 0;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < E;
         k += size_t(gridDim.x) * blockDim.x) {
        double mu, om;
        uint8_t fl;
        window_epilogue(S[k], Q[k], inv_mn, mn, pn, mu, om, fl);
        if (!fix) {
            const double var_sum = __dsub_rn(Q[k], __dmul_rn(__dmul_rn(S[k], S[k]), inv_mn));
            undecided += !variance_is_flat(var_sum, Q[k], mn) && var_sum > pn_lo &&
                         var_sum <= pn_hi;
        }
        st.mu[k] = mu;
        st.omega[k] = om;
        st.flat[k] = fl;
    }
    if (!fix) {
        undecided = warp_sum(undecided);
        if ((threadIdx.x & 31) == 0 && undecided) atomicAdd(cnt + 4, (unsigned long long)undecided);
    }
}

__global__ void k_clear_undecided(double* nbk) {
    reinterpret_cast<unsigned long long*>(nbk)[4] = 0ull;
}

int grid_for(size_t n, int threads) {
    const size_t b = (n + threads - 1) / threads;
    return int(b < 148 * 16 ? (b ? b : 1) : 148 * 16);
}

}  // namespace

cudaError_t check_u8_domain(const double* img, size_t n, int* bad, cudaStream_t s) {
    k_check_u8<<<grid_for(n, 256), 256, 0, s>>>(img, n, bad);
    return cudaGetLastError();
}
cudaError_t f64_to_u8(const double* img, size_t n, uint8_t* out, cudaStream_t s) {
    k_f64_to_u8<<<grid_for(n, 256), 256, 0, s>>>(img, n, out);
    return cudaGetLastError();
}
cudaError_t u8_to_f64(const uint8_t* img, size_t n, double* out, cudaStream_t s) {
    k_u8_to_f64<<<grid_for(n, 256), 256, 0, s>>>(img, n, out);
    return cudaGetLastError();
}
cudaError_t u8_to_f32_pitched(const uint8_t* img, int p, int q, float* out, int pitch,
                              cudaStream_t s) {
    dim3 grid((pitch + 255) / 256, p);
    k_u8_to_f32<<<grid, 256, 0, s>>>(img, p, q, out, pitch);
    return cudaGetLastError();
}
cudaError_t prefix_noise_u8(const uint8_t* img, int p, int q, unsigned long long* q_total,
                            double* out, cudaStream_t s) {
    const size_t n = size_t(p) * q;
    const int blocks = int(std::min<size_t>(148 * 4, (n / 16 + 255) / 256 + 1));
    launch_pdl(k_sum_sq_u8, dim3(blocks), dim3(256), 0, s, img, n, q_total, p, q, out);  // q_total: 2 u64, zeroed
    return cudaGetLastError();
}
cudaError_t prefix_noise_f64(const double* img, int p, int q, double* part, double* nbk,
                             cudaStream_t s) {
    const size_t n = size_t(p) * q;
    k_sum_sq_f64<<<kSqBlocks, kSqThreads, 0, s>>>(img, n, part);
    // TMATCH_PN_REPLAY=1 (tests): force the sequential q_total replay for every image
    const char* e = std::getenv("TMATCH_PN_REPLAY");
    const int widen = e && std::atoi(e) ? 1 : 0;
    k_prefix_noise_f64<<<1, 1, 0, s>>>(part, kSqBlocks, n, p, q, nbk, widen);
    return cudaGetLastError();
}

size_t prefix_noise_f64_parts() { return kSqBlocks; }

namespace {

// Fused window statistics (preferred integer path).  CTA = (column tile [c0, c0+tw),
// segment of extent rows); thread = one image column of the tile plus its n-1 halo.  Each
// thread slides the vertical sums s(y) = sum_{a<m} I(r+a, y) and q(y) (squares) down the
// rows (leading row in, row m above out; exact u32), and at every extent row the CTA
// scans s and q along y (warp prefixes + double-buffered warp totals, one barrier per
// row) so the window sums are S = P[c+n-1] - P[c-1].  The FP64 epilogue
// (stats.cpp:84-91) runs on consecutive columns, so mu/omega/flat are written coalesced.
__global__ void __launch_bounds__(512)
    k_wstats_u8(const uint8_t* __restrict__ img, int p, int q, int m, int n, int tw, int seg,
                const double* __restrict__ pn, DevStats st) {
    pdl_wait();
    __shared__ unsigned ls[2][2][512], wtot[2][2][16];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int er = p - m + 1, ec = q - n + 1;
    const int c0 = blockIdx.x * tw;
    const int r0 = blockIdx.y * seg, r1 = min(r0 + seg, er);
    if (r0 >= er || c0 >= ec) return;
    const int y = min(c0 + int(threadIdx.x), q - 1);  // clamped halo columns are never read
    const uint8_t* lead = img + size_t(r0) * q + y;
    const uint8_t* trail = lead;
    unsigned vs = 0, vq = 0;
#pragma unroll 4
    for (int a = 0; a < m; ++a) {
        const unsigned v = __ldg(lead);
        lead += q;
        vs += v;
        vq += v * v;
    }
    const double inv_mn = 1.0 / (double(m) * double(n));
    const long long mn = (long long)m * n;
    const double prefix_noise = *pn;
    const int c = c0 + int(threadIdx.x);
    const bool out_ok = int(threadIdx.x) < tw && c < ec;
    const int i1 = threadIdx.x + n - 1, w1 = i1 >> 5;
    const int w0 = threadIdx.x > 0 ? (int(threadIdx.x) - 1) >> 5 : 0;
    int par = 0;
    // next row's leading/trailing pixels, loaded before this row's scan + epilogue so the
    // load latency hides behind them
    unsigned vi = 0, vo = 0;
#pragma unroll 1
    for (int r = r0;;) {
        if (r + 1 < r1) {
            vi = __ldg(lead);
            vo = __ldg(trail);
        }
        unsigned a = vs, b = vq;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned ta = __shfl_up_sync(0xffffffffu, a, o);
            const unsigned tb = __shfl_up_sync(0xffffffffu, b, o);
            if (lane >= o) {
                a += ta;
                b += tb;
            }
        }
        ls[par][0][threadIdx.x] = a;
        ls[par][1][threadIdx.x] = b;
        if (lane == 31) {
            wtot[par][0][wid] = a;
            wtot[par][1][wid] = b;
        }
        __syncthreads();
        if (out_ok) {
            unsigned S = ls[par][0][i1], Q = ls[par][1][i1];
            if (threadIdx.x > 0) {
                S -= ls[par][0][threadIdx.x - 1];
                Q -= ls[par][1][threadIdx.x - 1];
            }
            for (int ww = w0; ww < w1; ++ww) {
                S += wtot[par][0][ww];
                Q += wtot[par][1][ww];
            }
            double mu, om;
            uint8_t fl;
            window_epilogue(double(S), double(Q), inv_mn, mn, prefix_noise, mu, om, fl);
            const size_t k = size_t(r) * ec + c;
            st.mu[k] = mu;
            st.omega[k] = om;
            st.flat[k] = fl;
        }
        par ^= 1;
        if (++r >= r1) break;
        lead += q;
        trail += q;
        vs += vi - vo;
        vq += vi * vi - vo * vo;
    }
}

// Fused window statistics, W (2 or 4) columns per thread (preferred when the 16-byte-pitched
// copy exists).  Thread t of a CTA owns image columns [c0 + Wt, c0 + Wt + W): one aligned
// load per row and edge, the vertical sums of its columns (pixel sums packed two per
// register as 16-bit lanes -- exact while m*255 + 255 < 2^16 -- and squares in u32), and at
// every extent row one block scan over W-column blocks.  Each thread publishes the
// warp-local exclusive column prefixes PC(Wt + r), r < W (one vector store per quantity);
// its W window sums are S(c) = PC(c + n) - PC(c) (+ the warp totals in between), and the
// FP64 epilogue (stats.cpp:84-91) runs for W consecutive outputs.
template <int NT, int W>
__global__ void __launch_bounds__(NT)
    k_wstats4(const uint8_t* __restrict__ img, int P, int p, int q, int m, int n, int G, int seg,
              int rlo, int rhi, const double* __restrict__ pn, DevStats st) {
    static_assert(W == 2 || W == 4, "two or four columns per thread");
    pdl_wait();
    constexpr int NW = NT / 32;
    constexpr int TSH = W == 4 ? 7 : 6;  // log2(32 * W): tile column -> warp
    __shared__ __align__(16) unsigned pcs[2][NT * W], pcq[2][NT * W];
    __shared__ unsigned wts[2][NW + 1], wtq[2][NW + 1];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int er = p - m + 1, ec = q - n + 1;
    const int c0 = blockIdx.x * (W * G);
    const int r0 = rlo + blockIdx.y * seg, r1 = min(r0 + seg, min(rhi, er));
    if (r0 >= r1 || c0 >= ec) return;
    // columns past the image read the zero padding / the next row: only sums no output reads
    const uint8_t* col = img + (c0 + W * t);
    const uint8_t* lead = col + size_t(r0) * P;
    const uint8_t* trail = lead;
    auto ld = [&](const uint8_t* ptr) -> unsigned {
        if constexpr (W == 4) return __ldg(reinterpret_cast<const unsigned*>(ptr));
        else return unsigned(__ldg(reinterpret_cast<const unsigned short*>(ptr)));
    };
    // packed pixel sums: W = 4 -> lanes (0,2) and (1,3); W = 2 -> lanes (0,1) in s02
    unsigned s02 = 0, s13 = 0, qq[W];
#pragma unroll
    for (int j = 0; j < W; ++j) qq[j] = 0;
    auto lanes = [&](unsigned x, unsigned& e, unsigned& o) {
        if constexpr (W == 4) {
            e = x & 0x00ff00ffu;
            o = (x >> 8) & 0x00ff00ffu;
        } else {
            e = (x & 0xffu) | ((x & 0xff00u) << 8);
            o = 0;
        }
    };
#pragma unroll 4
    for (int a = 0; a < m; ++a) {
        const unsigned x = ld(lead);
        lead += P;
        unsigned e, o;
        lanes(x, e, o);
        s02 += e;
        s13 += o;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const unsigned bj = (x >> (8 * j)) & 0xffu;
            qq[j] += bj * bj;
        }
    }
    const double inv_mn = 1.0 / (double(m) * double(n));
    const long long mn = (long long)m * n;
    const double prefix_noise = *pn;
    const int cbase = c0 + W * t;
    const bool any_out = t < G && cbase < ec;
    const int idx = W * t + n;  // tile-local column of PC(c + n) for j = 0
    const bool vec = (n % W) == 0;
    int par = 0;
    unsigned vi = 0, vo = 0;
#pragma unroll 1
    for (int r = r0;;) {
        if (r + 1 < r1) {  // next row's edges, loaded before this row's scan + epilogue
            vi = ld(lead);
            vo = ld(trail);
        }
        unsigned sc[W];
        if constexpr (W == 4) {
            sc[0] = s02 & 0xffffu; sc[1] = s13 & 0xffffu; sc[2] = s02 >> 16; sc[3] = s13 >> 16;
        } else {
            sc[0] = s02 & 0xffffu; sc[1] = s02 >> 16;
        }
        unsigned bs = 0, bq = 0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            bs += sc[j];
            bq += qq[j];
        }
        unsigned a = bs, b = bq;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned ta = __shfl_up_sync(0xffffffffu, a, o);
            const unsigned tb = __shfl_up_sync(0xffffffffu, b, o);
            if (lane >= o) {
                a += ta;
                b += tb;
            }
        }
        // warp-local exclusive prefixes at the block's W columns
        unsigned own_s[W], own_q[W];
        own_s[0] = a - bs;
        own_q[0] = b - bq;
#pragma unroll
        for (int j = 1; j < W; ++j) {
            own_s[j] = own_s[j - 1] + sc[j - 1];
            own_q[j] = own_q[j - 1] + qq[j - 1];
        }
        if constexpr (W == 4) {
            *reinterpret_cast<uint4*>(&pcs[par][4 * t]) = make_uint4(own_s[0], own_s[1], own_s[2], own_s[3]);
            *reinterpret_cast<uint4*>(&pcq[par][4 * t]) = make_uint4(own_q[0], own_q[1], own_q[2], own_q[3]);
        } else {
            *reinterpret_cast<uint2*>(&pcs[par][2 * t]) = make_uint2(own_s[0], own_s[1]);
            *reinterpret_cast<uint2*>(&pcq[par][2 * t]) = make_uint2(own_q[0], own_q[1]);
        }
        if (lane == 31) {
            wts[par][wid] = a;
            wtq[par][wid] = b;
        }
        __syncthreads();
        if (any_out) {
            unsigned hs[W], hq[W];
            if (vec) {
                if constexpr (W == 4) {
                    const uint4 xs = *reinterpret_cast<const uint4*>(&pcs[par][idx]);
                    const uint4 xq = *reinterpret_cast<const uint4*>(&pcq[par][idx]);
                    hs[0] = xs.x; hs[1] = xs.y; hs[2] = xs.z; hs[3] = xs.w;
                    hq[0] = xq.x; hq[1] = xq.y; hq[2] = xq.z; hq[3] = xq.w;
                } else {
                    const uint2 xs = *reinterpret_cast<const uint2*>(&pcs[par][idx]);
                    const uint2 xq = *reinterpret_cast<const uint2*>(&pcq[par][idx]);
                    hs[0] = xs.x; hs[1] = xs.y;
                    hq[0] = xq.x; hq[1] = xq.y;
                }
            } else {
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    hs[j] = pcs[par][idx + j];
                    hq[j] = pcq[par][idx + j];
                }
            }
            const size_t k = size_t(r) * ec + cbase;
            const int nout = min(W, ec - cbase);
#pragma unroll
            for (int j = 0; j < W; ++j) {
                // + warp totals between this warp and the warp holding PC(c + n + j)
                // (n + W <= 128 + W: at most two warps in between -- predicated, no loop;
                // wts has NW + 1 slots so both reads stay inside)
                const int wj = (idx + j) >> TSH;
                unsigned S = hs[j] - own_s[j], Qs = hq[j] - own_q[j];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int w = min(wid + u, NW);
                    const unsigned xs = wts[par][w], xq = wtq[par][w];
                    S += wid + u < wj ? xs : 0u;
                    Qs += wid + u < wj ? xq : 0u;
                }
                double mu, om;
                uint8_t fl;
                window_epilogue(double(S), double(Qs), inv_mn, mn, prefix_noise, mu, om, fl);
                if (j < nout) {
                    st.mu[k + j] = mu;
                    st.omega[k + j] = om;
                    st.flat[k + j] = fl;
                }
            }
        }
        par ^= 1;
        if (++r >= r1) break;
        lead += P;
        trail += P;
        // slide: + leading row, - trailing row (packed lanes stay in [0, 2^16))
        {
            unsigned ei, oi, eo, oo;
            lanes(vi, ei, oi);
            lanes(vo, eo, oo);
            s02 += ei;
            s13 += oi;
            s02 -= eo;
            s13 -= oo;
        }
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const unsigned ij = (vi >> (8 * j)) & 0xffu, oj = (vo >> (8 * j)) & 0xffu;
            qq[j] += ij * ij - oj * oj;
        }
    }
}

}  // namespace

bool window_stats4_supported(int p, int q, int m, int n, int pitch) {
    const int ec = q - n + 1, er = p - m + 1;
    return er >= 1 && ec >= 1 && pitch % 16 == 0 && m <= 255 &&
           double(m) * double(n) * 65025.0 < 4294967296.0 && (n + 1) / 2 <= 64;
}

template <int NT, int W>
cudaError_t launch_wstats4(const uint8_t* imgp, int pitch, int p, int q, int m, int n,
                           const double* prefix_noise, DevStats st, cudaStream_t s, int rlo,
                           int rhi) {
    const int ec = q - n + 1;
    rlo = std::max(0, rlo);
    rhi = std::min(rhi, p - m + 1);
    const int er = std::max(0, rhi - rlo);  // extent rows of this launch (a strip or all)
    if (er == 0) return cudaSuccess;
    const int G = NT - (n + W - 1) / W;  // output blocks per tile (PC(c + n) stays in the tile)
    const int ntiles = (ec + W * G - 1) / (W * G);
    // one wave of resident CTAs: a segment's m-row warm-up (~15 instructions a row) is small
    // next to its output rows, so short segments beyond one wave only add tail
    static int resident = 0;
    if (!resident &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_wstats4<NT, W>, NT, 0) != cudaSuccess)
        resident = 2;
    resident = std::max(resident, 1);
    int nseg = std::max(1, (148 * resident) / ntiles);
    int seg = std::max(4, (er + nseg - 1) / nseg);
    nseg = (er + seg - 1) / seg;
    dim3 grid(ntiles, nseg);
    launch_pdl(k_wstats4<NT, W>, grid, dim3(NT), 0, s, imgp, pitch, p, q, m, n, G, seg, rlo,
               rhi, prefix_noise, st);
    return cudaGetLastError();
}

// CTA shape: 256 threads x 2 columns (default; C2 36.5 us vs 46 us for one column per
// thread and 61 us for four, whose four serial FP64 epilogues per row leave too few warps
// to hide their latency).  TMATCH_WSTATS4=256x4|128x4|128x2 for A/B measurements.
int wstats4_variant() {
    static int v = [] {
        const char* e = std::getenv("TMATCH_WSTATS4");
        if (!e) return 2;
        if (!std::strcmp(e, "256x4")) return 0;
        if (!std::strcmp(e, "128x4")) return 1;
        if (!std::strcmp(e, "128x2")) return 3;
        return 2;
    }();
    return v;
}

cudaError_t window_stats4_u8(const uint8_t* imgp, int pitch, int p, int q, int m, int n,
                             const double* prefix_noise, DevStats st, cudaStream_t s, int rlo,
                             int rhi) {
    switch (wstats4_variant()) {
        case 1: return launch_wstats4<128, 4>(imgp, pitch, p, q, m, n, prefix_noise, st, s, rlo, rhi);
        case 2: return launch_wstats4<256, 2>(imgp, pitch, p, q, m, n, prefix_noise, st, s, rlo, rhi);
        case 3: return launch_wstats4<128, 2>(imgp, pitch, p, q, m, n, prefix_noise, st, s, rlo, rhi);
        default: return launch_wstats4<256, 4>(imgp, pitch, p, q, m, n, prefix_noise, st, s, rlo, rhi);
    }
}

// Sum of squares of rows [r0, r0 + nrows) of an 8-bit image (the rank's share of the
// image-global q_total, stats.cpp:78-79, before the allreduce of a row-strip search).
__global__ void k_sum_sq_rows(const uint8_t* __restrict__ img, size_t n,
                              unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const unsigned x = img[i];
        acc += x * x;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

cudaError_t sum_sq_rows_u8(const uint8_t* img, int q, int r0, int nrows, unsigned long long* out,
                           cudaStream_t s) {
    cudaMemsetAsync(out, 0, sizeof *out, s);
    const size_t n = size_t(nrows) * q;
    if (n) k_sum_sq_rows<<<grid_for(n, 256), 256, 0, s>>>(img + size_t(r0) * q, n, out);
    return cudaGetLastError();
}

cudaError_t window_stats_u8(const uint8_t* img, int p, int q, int m, int n, const double* prefix_noise,
                            int* hs, int* hq, DevStats st, cudaStream_t s) {
    const int ec = q - n + 1, er = p - m + 1;
    // fused path: u32 sums exact while m*n*255^2 < 2^32; column tile + halo <= 512 threads
    if (double(m) * double(n) * 65025.0 < 4294967296.0 && n <= 384) {
        int ny = std::max(256, ((4 * n + 31) / 32) * 32);  // halo n-1 of ny columns
        ny = std::min(ny, 512);
        const int tw = ny - n + 1;
        const int ntiles = (ec + tw - 1) / tw;
        // segments: ~4 resident waves of CTAs, each walking at least 2m rows of output
        int nseg = std::max(1, (148 * 16) / ntiles);
        int seg = std::max(std::min(m, 32), (er + nseg - 1) / nseg);
        nseg = (er + seg - 1) / seg;
        dim3 grid(ntiles, nseg);
        launch_pdl(k_wstats_u8, dim3(grid), dim3(ny), 0, s, img, p, q, m, n, tw, seg, prefix_noise, st);
        return cudaGetLastError();
    }
    const int tpr = (ec + kChunk - 1) / kChunk;
    dim3 g1((tpr + 127) / 128, p);
    k_hsum_u8<<<g1, 128, 0, s>>>(img, p, q, n, hs, hq);
    dim3 g2((ec + 127) / 128, (er + kChunk - 1) / kChunk);
    k_vsum_stats<<<g2, 128, 0, s>>>(hs, hq, p, ec, m, n, prefix_noise, st);
    return cudaGetLastError();
}

cudaError_t window_sums_u8(const uint8_t* img, int p, int q, int m, int n, int* hs, double* out,
                           cudaStream_t s) {
    const int ec = q - n + 1, er = p - m + 1;
    const int tpr = (ec + kChunk - 1) / kChunk;
    dim3 g1((tpr + 127) / 128, p);
    k_hsum_u8<<<g1, 128, 0, s>>>(img, p, q, n, hs, nullptr);
    dim3 g2((ec + 127) / 128, (er + kChunk - 1) / kChunk);
    k_vsum_only<<<g2, 128, 0, s>>>(hs, p, ec, m, out);
    return cudaGetLastError();
}

cudaError_t replica_prefix_batch(const ProdBatch& b, double* rowacc, double* prefix,
                                 cudaStream_t s) {
    int maxr = 0, maxc = 0;
    for (int k = 0; k < b.n; ++k) {
        maxr = std::max(maxr, b.rows[k]);
        maxc = std::max(maxc, b.cols[k]);
    }
    const int warps = (maxr + 31) / 32;
    k_rowscan_b<<<dim3((warps + 3) / 4, b.n), 128, 0, s>>>(b, rowacc);
    k_colacc_b<<<dim3((maxc + 1 + 127) / 128, b.n), 128, 0, s>>>(b, rowacc, prefix);
    return cudaGetLastError();
}

cudaError_t replica_prefix(ProdSrc src, int rows, int cols, double* rowacc, double* prefix,
                           cudaStream_t s) {
    const int warps = (rows + 31) / 32;
    k_rowscan<<<(warps + 3) / 4, 128, 0, s>>>(src, rows, cols, rowacc);
    k_colacc<<<(cols + 1 + 127) / 128, 128, 0, s>>>(rowacc, rows, cols, prefix, src.stop);
    return cudaGetLastError();
}

cudaError_t replica_window_diff(const double* prefix, int rows, int cols, int m, int n,
                                double* out, cudaStream_t s) {
    const size_t E = size_t(rows - m + 1) * (cols - n + 1);
    k_window_diff<<<grid_for(E, 256), 256, 0, s>>>(prefix, rows, cols, m, n, out);
    return cudaGetLastError();
}

cudaError_t stats_from_sums(const double* S, const double* Q, size_t E, int m, int n,
                            const double* img, int p, int q, double* nbk, DevStats st,
                            cudaStream_t s) {
    k_stats_from_sums<<<grid_for(E, 256), 256, 0, s>>>(S, Q, E, m, n, nbk, st, 0);
    k_resolve_prefix_noise<<<1, 32, 0, s>>>(img, size_t(p) * q, p, q, nbk);
    k_stats_from_sums<<<grid_for(E, 256), 256, 0, s>>>(S, Q, E, m, n, nbk, st, 1);
    k_clear_undecided<<<1, 1, 0, s>>>(nbk);
    return cudaGetLastError();
}

}  // namespace tmk
