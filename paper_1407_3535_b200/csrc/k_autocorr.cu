// k_autocorr.cu -- local auto-correlation map R_co and the EGS retained count (sm_100a).
//
// Reference: local_autocorrelation (autocorr.cpp:40-96) builds, for each of the hw-1
// offsets, a full-image product table and its FP64 prefix sums, then reads one window
// sum per group centre.  On 8-bit data those cross sums are exact integers, so here one
// fused pass computes them directly, and only at the centres:
//
//   S_d(c) = sum_{a<m, b<n} I(cr+a, cc+b) * I(cr+di+a, cc+dj+b)
//
// A CTA owns a tile of GTR x GTC groups, stages the image region it needs in shared
// memory once, and loops over all offsets: a row pass slides an n-wide window along the
// centre columns (H), a column pass slides an m-tall window along the centre rows, and the
// FP64 epilogue replays autocorr.cpp:84-88 op for op.  The retained count (egs.cpp:12-25,
// members with R_co < sqrt(1 - rho_tb^2)) is reduced in the same kernel.  Algorithmic
// work is O((hw-1) * p * q) integer MACs per candidate size instead of the reference's
// (hw-1) full-image FP64 prefix passes.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kernels.hpp"
#include "tm_common.cuh"

namespace tmk {

namespace {

struct ACParams {
    const uint8_t* img;
    int p, q, m, n;
    Grid g;
    DevStats st;
    double thr;
    double* map;
    unsigned long long* n_r;
    int gtr, gtc;   // groups per CTA tile
    int nx_max;     // H rows per tile
    int spitch;     // staged image pitch (bytes)
    int srows;
    int noff_per;   // offsets handled per CTA (blockIdx.z selects the slice)
};

__device__ __forceinline__ int ccol(const Grid& g, int tj) { return g.center_col(tj); }
__device__ __forceinline__ int crow(const Grid& g, int ti) { return g.center_row(ti); }

__global__ void k_autocorr_u8(ACParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Grid& g = P.g;
    const int ti0 = g.ti_lo + blockIdx.y * P.gtr, tj0 = blockIdx.x * P.gtc;
    const int nti = min(P.gtr, g.ti_hi - ti0), ntj = min(P.gtc, g.tc - tj0);
    if (nti <= 0) return;
    const int hr = g.h >> 1, wr = g.w >> 1;
    const int crA = crow(g, ti0), crB = crow(g, ti0 + nti - 1);
    const int ccA = ccol(g, tj0), ccB = ccol(g, tj0 + ntj - 1);
    const int R0 = crA - hr, C0 = ccA - wr;  // staged region origin (may be < 0: zeros)
    const int nrows = (crB + hr + P.m) - R0;
    const int ncols = (ccB + wr + P.n) - C0;

    uint8_t* simg = smem;
    int* H = reinterpret_cast<int*>(smem + ((size_t(P.srows) * P.spitch + 15) & ~size_t(15)));
    int* scc = H + size_t(P.nx_max) * P.gtc;
    int* scr = scc + P.gtc;
    __shared__ unsigned long long blk_nr;

    if (threadIdx.x == 0) blk_nr = 0;
    for (int k = threadIdx.x; k < ntj; k += blockDim.x) scc[k] = ccol(g, tj0 + k);
    for (int k = threadIdx.x; k < nti; k += blockDim.x) scr[k] = crow(g, ti0 + k);
    for (int idx = threadIdx.x; idx < nrows * ncols; idx += blockDim.x) {
        const int a = idx / ncols, b = idx % ncols;
        const int r = R0 + a, c = C0 + b;
        simg[size_t(a) * P.spitch + b] =
            (r >= 0 && r < P.p && c >= 0 && c < P.q) ? P.img[size_t(r) * P.q + c] : 0;
    }
    __syncthreads();

    const int nx = crB - crA + P.m;  // H rows: x = crA + xi
    constexpr int kTJ = 8;           // centre columns per row-pass item
    constexpr int kTI = 4;           // centre rows per column-pass item
    const int nch = (ntj + kTJ - 1) / kTJ;
    const double mn = double(P.m) * double(P.n);
    unsigned long long local_nr = 0;

    // offsets in raster order, centre (0,0) skipped; this CTA takes a contiguous slice
    const int noff = g.h * g.w - 1;
    const int o0 = blockIdx.z * P.noff_per, o1 = min(noff, o0 + P.noff_per);
    for (int oi = o0; oi < o1; ++oi) {
        {
            const int ro = oi < (noff / 2) ? oi : oi + 1;  // skip the centre slot
            const int di = ro / g.w - hr, dj = ro % g.w - wr;
            // ---- row pass: H[xi][tj] = sum_b I(x, cc+b) * I(x+di, cc+dj+b) ----------
            for (int item = threadIdx.x; item < nx * nch; item += blockDim.x) {
                const int xi = item / nch, ch = item % nch;
                const int x = crA + xi;
                const uint8_t* ra = simg + size_t(x - R0) * P.spitch - C0;
                const uint8_t* rb = simg + size_t(x + di - R0) * P.spitch - C0 + dj;
                const int k0 = ch * kTJ, k1 = min(k0 + kTJ, ntj);
                int cc = scc[k0];
                int s = 0;
                for (int b = 0; b < P.n; ++b) s += int(ra[cc + b]) * int(rb[cc + b]);
                H[size_t(xi) * P.gtc + k0] = s;
                for (int k = k0 + 1; k < k1; ++k) {
                    const int nc = scc[k];
                    for (int c = cc; c < nc; ++c)
                        s += int(ra[c + P.n]) * int(rb[c + P.n]) - int(ra[c]) * int(rb[c]);
                    cc = nc;
                    H[size_t(xi) * P.gtc + k] = s;
                }
            }
            __syncthreads();
            // ---- column pass + epilogue --------------------------------------------
            const int nic = (nti + kTI - 1) / kTI;
            for (int item = threadIdx.x; item < ntj * nic; item += blockDim.x) {
                const int k = item % ntj, ic = item / ntj;
                const int i0 = ic * kTI, i1 = min(i0 + kTI, nti);
                int cr = scr[i0];
                long long S = 0;
                for (int a = 0; a < P.m; ++a) S += H[size_t(cr - crA + a) * P.gtc + k];
                const int cc = scc[k];
                const int tj = tj0 + k;
                const int c0 = tj * g.w, c1 = min(c0 + g.w, g.ec) - 1;
                const int mc = cc + dj;
                for (int i = i0; i < i1; ++i) {
                    if (i > i0) {
                        const int ncr = scr[i];
                        for (int x = cr; x < ncr; ++x)
                            S += (long long)H[size_t(x + P.m - crA) * P.gtc + k] -
                                 H[size_t(x - crA) * P.gtc + k];
                        cr = ncr;
                    }
                    const int ti = ti0 + i;
                    const int r0 = ti * g.h, r1 = min(r0 + g.h, g.er) - 1;
                    const int mr = cr + di;
                    if (mr < r0 || mr > r1 || mc < c0 || mc > c1) continue;
                    const size_t kc = size_t(cr) * g.ec + cc, km = size_t(mr) * g.ec + mc;
                    double v = 0.0;
                    if (!P.st.flat[kc] && !P.st.flat[km]) {
                        const double num =
                            __dsub_rn(double(S), __dmul_rn(__dmul_rn(mn, P.st.mu[kc]), P.st.mu[km]));
                        v = dclamp(__ddiv_rn(num, __dmul_rn(P.st.omega[kc], P.st.omega[km])), -1.0,
                                   1.0);
                    }
                    P.map[km] = v;
                    if (v < P.thr) ++local_nr;
                }
            }
            __syncthreads();
        }
    }
    // centres carry exactly 1 (autocorr.cpp:92-93)
    for (int idx = threadIdx.x; blockIdx.z == 0 && idx < nti * ntj; idx += blockDim.x) {
        const int i = idx / ntj, k = idx % ntj;
        P.map[size_t(scr[i]) * g.ec + scc[k]] = 1.0;
    }
    local_nr = warp_sum(local_nr);
    if ((threadIdx.x & 31) == 0 && local_nr) atomicAdd(&blk_nr, local_nr);
    __syncthreads();
    if (threadIdx.x == 0 && blk_nr) atomicAdd(P.n_r, blk_nr);
}

// ---- three-pass R_co (row walk, column prefix, epilogue), for w in {1,3,...,11} -----
//
// Pass 1 (k_ac_rows): a CTA owns 128 consecutive image rows x for one row offset di and one
// segment of centre columns; it stages rows x and x+di of that segment in shared memory
// (coalesced), then each thread walks its row once.  A W-entry register ring holds
// I(x+di, y-wr .. y+wr), so a pixel costs two shared-memory byte loads and W integer MACs
// -- one per column offset dj -- accumulated as running prefixes R_dj(y).  At a centre
// column cc (y = cc) the prefixes are recorded (shared-memory ring), at y = cc + n the
// row-window sum  H[di,dj](k, x) = sum_b I(x, cc+b) I(x+di, cc+dj+b)  is emitted.  Centre
// columns are cc_k = wr + k*w, so with the walk aligned to multiples of W every ring
// index and event position is static inside a W-step unrolled block.
// Pass 2 (k_ac_scan): one warp per (offset, centre column) line turns H into its inclusive
// prefix over rows, in place, in wrapping 32-bit arithmetic (window sums < 2^31 are then
// exact differences).
// Pass 3 (k_ac_epi): S = P[cr+m-1] - P[cr-1] per (offset, centre), FP64 epilogue of
// autocorr.cpp:84-88, map write and the retained count of egs.cpp:12-25.
// H layout [di][dj][k][x] (x fastest).
constexpr int kAcRows = 128;

template <int W>
__global__ void __launch_bounds__(kAcRows)
    k_ac_rows(const uint8_t* __restrict__ img, int p, int q, int n, int tcr, int tc, int seg,
              int ring, int spitch, unsigned* __restrict__ H) {
    extern __shared__ __align__(16) unsigned char sm[];
    constexpr int wr = W / 2;
    const int x0 = blockIdx.x * kAcRows;
    const int dii = blockIdx.y;
    const int hr = gridDim.y / 2;
    const int di = dii - hr;
    const int k0 = blockIdx.z * seg, k1 = min(k0 + seg, tcr);
    if (k0 >= k1) return;
    const int y_s = k0 * W;                   // walk start (multiple of W)
    const int y_e = wr + (k1 - 1) * W + n;    // last window-end event
    const int c_lo = y_s - wr;                // staged columns [c_lo, c_lo + swid)
    const int swid = (y_e + W) - c_lo + wr + 1;
    const int r_lo = x0 + min(0, di);         // staged rows [r_lo, r_lo + srow); row srow = 0s
    const int srow = kAcRows + abs(di);
    uint8_t* simg = sm;
    int* rec = reinterpret_cast<int*>(sm + ((size_t(srow + 1) * spitch + 15) & ~size_t(15)));
    // staging: one warp per staged row, 8 independent loads in flight per lane
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int a = wid; a <= srow; a += kAcRows / 32) {
        const int r = r_lo + a;
        uint8_t* dst = simg + a * spitch;
        const bool rok = a < srow && r >= 0 && r < p;
        const uint8_t* src = img + size_t(rok ? r : 0) * q;
        for (int b0 = 0; b0 < swid; b0 += 32 * 8) {
            uint8_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int c = c_lo + b0 + u * 32 + lane;
                v[u] = (rok && c >= 0 && c < q) ? __ldg(src + c) : uint8_t(0);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int b = b0 + u * 32 + lane;
                if (b < swid) dst[b] = v[u];
            }
        }
    }
    __syncthreads();
    const int x = x0 + threadIdx.x;
    const bool row_ok = x < p && x + di >= 0 && x + di < p;
    // invalid rows read the zero row, so the walk needs no per-pixel guards
    const uint8_t* ra = simg + (row_ok ? (x - r_lo) : srow) * spitch - c_lo;
    const uint8_t* rb = simg + (row_ok ? (x + di - r_lo) : srow) * spitch - c_lo;
    int acc[W];
    int rg[W];
#pragma unroll
    for (int t = 0; t < W; ++t) {
        acc[t] = 0;
        rg[t] = (t < W - 1) ? int(rb[y_s - wr + t]) : 0;
    }
    const size_t plane = size_t(tc) * p;
    unsigned* hout = H + size_t(dii) * W * plane + size_t(x);
    int* recp = rec + threadIdx.x;
    constexpr int kEndS = (wr + (W > 0 ? 0 : 0)) + 0;  // placeholder to keep W-dependent names
    (void)kEndS;
    const int end_s = (wr + n) % W;
    // centre k opens at y = wr + k*W (slot k % ring) and closes at y = wr + k*W + n
    int open_k = k0, open_slot = k0 % ring;
    int close_k = k0, close_slot = k0 % ring;
    const int first_close = wr + k0 * W + n;
    for (int y0 = y_s; y0 <= y_e; y0 += W) {
#pragma unroll
        for (int s = 0; s < W; ++s) {
            const int y = y0 + s;
            if (s == wr && open_k < k1) {  // window start: record the prefix before P(y)
#pragma unroll
                for (int t = 0; t < W; ++t) recp[(open_slot * W + t) * kAcRows] = acc[t];
                ++open_k;
                if (++open_slot == ring) open_slot = 0;
            }
            if (s == end_s && y >= first_close && close_k < k1) {  // window end
                if (x < p) {
#pragma unroll
                    for (int t = 0; t < W; ++t)
                        hout[size_t(t) * plane + size_t(close_k) * p] =
                            unsigned(acc[t] - recp[(close_slot * W + t) * kAcRows]);
                }
                ++close_k;
                if (++close_slot == ring) close_slot = 0;
            }
            rg[(s + W - 1) % W] = int(rb[y + wr]);  // I(x+di, y+wr)
            const int a = int(ra[y]);
#pragma unroll
            for (int t = 0; t < W; ++t) acc[t] += a * rg[(s + t) % W];  // dj = t - wr
        }
    }
}

// Clipped last centre column (irregular position): one warp per (offset, row), lanes
// over the n template columns, exact integer warp reduction.
__global__ void k_ac_rows_last(const uint8_t* __restrict__ img, int p, int q, int n, int h, int w,
                               int cc, int kcol, int tc, unsigned* __restrict__ H) {
    const int lane = threadIdx.x & 31;
    const long long wg = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long items = (long long)h * w * p;
    const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long it = wg; it < items; it += nw) {
        const int oi = int(it / p), x = int(it % p);
        const int di = oi / w - h / 2, dj = oi % w - w / 2;
        int s = 0;
        if (x + di >= 0 && x + di < p) {
            const uint8_t* ra = img + size_t(x) * q + cc;
            const uint8_t* rb = img + size_t(x + di) * q;
            for (int b = lane; b < n; b += 32) {
                const int cb = cc + dj + b;
                s += int(ra[b]) * ((cb >= 0 && cb < q) ? int(rb[cb]) : 0);
            }
        }
        s = warp_sum(s);
        if (lane == 0) H[(size_t(oi) * tc + kcol) * p + x] = unsigned(s);
    }
}

// Inclusive prefix over rows of 32 consecutive (offset, centre column) lines per CTA,
// transposed on the way out: H[oi][k][x] -> P[oi][x][k] (k fastest), wrapping u32.
__global__ void __launch_bounds__(1024)
    k_ac_scan(const unsigned* __restrict__ H, unsigned* __restrict__ P, int p, int tc, int hw) {
    __shared__ unsigned tile[32][33];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int kblocks = (tc + 31) / 32;
    const int oi = blockIdx.x / kblocks, k0 = (blockIdx.x % kblocks) * 32;
    if (oi >= hw) return;
    const int k = k0 + wid;  // this warp's line
    const unsigned* L = H + (size_t(oi) * tc + min(k, tc - 1)) * p;
    unsigned* out = P + size_t(oi) * p * tc;
    unsigned carry = 0;
    for (int x0 = 0; x0 < p; x0 += 32) {
        const int x = x0 + lane;
        unsigned v = (x < p && k < tc) ? L[x] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        v += carry;
        carry = __shfl_sync(0xffffffffu, v, 31);
        tile[wid][lane] = v;
        __syncthreads();
        // warp wid writes row x0+wid: 32 consecutive k
        const int xr = x0 + wid, kk = k0 + lane;
        if (xr < p && kk < tc) out[size_t(xr) * tc + kk] = tile[lane][wid];
        __syncthreads();
    }
}

// Epilogue: thread = (offset, centre row ti, centre column k), lanes over k; reads the
// transposed prefix P[oi][x][k] coalesced.
__global__ void __launch_bounds__(256)
    k_ac_epi(const unsigned* __restrict__ P, int p, int m, int n, Grid g, DevStats st, double thr,
             double* __restrict__ map, unsigned long long* n_r) {
    const int hw = g.h * g.w;
    const long long items = (long long)hw * g.tr * g.tc;
    const double mn = double(m) * double(n);
    const int hr = g.h / 2, wr = g.w / 2;
    unsigned long long local = 0;
    for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < items;
         it += (long long)gridDim.x * blockDim.x) {
        const int k = int(it % g.tc);
        const long long rest = it / g.tc;
        const int ti = int(rest % g.tr);
        const int oi = int(rest / g.tr);
        const int di = oi / g.w - hr, dj = oi % g.w - wr;
        const int cc = g.center_col(k), cr = g.center_row(ti);
        if (di == 0 && dj == 0) {  // centres carry exactly 1 (autocorr.cpp:92-93)
            map[size_t(cr) * g.ec + cc] = 1.0;
            continue;
        }
        const int c0 = k * g.w, c1 = min(c0 + g.w, g.ec) - 1;
        const int r0 = ti * g.h, r1 = min(r0 + g.h, g.er) - 1;
        const int mr = cr + di, mc = cc + dj;
        if (mr < r0 || mr > r1 || mc < c0 || mc > c1) continue;  // not this group's member
        const unsigned* L = P + size_t(oi) * p * g.tc + k;
        const unsigned S = L[size_t(cr + m - 1) * g.tc] - (cr > 0 ? L[size_t(cr - 1) * g.tc] : 0u);
        const size_t kc = size_t(cr) * g.ec + cc, km = size_t(mr) * g.ec + mc;
        double v = 0.0;
        if (!st.flat[kc] && !st.flat[km]) {
            const double num = __dsub_rn(double(S), __dmul_rn(__dmul_rn(mn, st.mu[kc]), st.mu[km]));
            v = dclamp(__ddiv_rn(num, __dmul_rn(st.omega[kc], st.omega[km])), -1.0, 1.0);
        }
        map[km] = v;
        if (v < thr) ++local;
    }
    local = warp_sum(local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(n_r, local);
}

// ---- column-walk R_co (preferred path) -----------------------------------------------
//
// Pass 1 (k_acv<H>): thread = (image column y, column offset dj, segment of centre rows).
// It walks down the rows once; lanes are consecutive columns, so every load is coalesced
// and no staging is needed.  A register ring holds I(x+di, y+dj) for the h row offsets
// di, so a row step costs two byte loads and h integer MACs accumulated as running
// prefixes R_di(x).  At a centre row cr the prefixes are recorded (shared-memory ring);
// at x = cr + m the vertical window sums V[di,dj](ti, y) = R_di(cr+m) - R_di(cr) are
// written (coalesced).  Centre rows are cr_ti = hr + ti*h, so with the walk aligned to
// multiples of H every ring index and event position is static in an H-step block.
// Pass 2 (k_ac_hline): one warp per (offset, centre row): the V line is scanned along y in
// shared memory (per-lane chunks + warp scan), then S = P[cc+n-1] - P[cc-1] for every
// centre column and the FP64 epilogue / retained count.  V layout [di][dj][ti][y].
constexpr int kAcvThreads = 128;

template <int H, int D>
__global__ void __launch_bounds__(kAcvThreads)
    k_acv(const uint8_t* __restrict__ img, int p, int q, int m, int W, int trr, int tr,
          int seg, unsigned* __restrict__ V, int ti_base) {
    constexpr int hr = H / 2;
    constexpr int P = D * H;  // prefetch distance in rows (a multiple of H)
    const int y = blockIdx.x * kAcvThreads + threadIdx.x;
    const int t = blockIdx.y;  // dj index
    const int dj = t - W / 2;
    const int ti0 = ti_base + blockIdx.z * seg, ti1 = min(ti0 + seg, trr);
    if (ti0 >= ti1) return;
    const int yb = y + dj;
    const bool col_ok = y < q && yb >= 0 && yb < q;
    const bool a_ok = y < q;
    const uint8_t* ca = img + (a_ok ? y : 0);
    const uint8_t* cb = img + (col_ok ? yb : 0);
    auto A = [&](int x) -> int { return (a_ok && x < p) ? int(__ldg(ca + size_t(x) * q)) : 0; };
    auto B = [&](int x) -> int {
        return (col_ok && x >= 0 && x < p) ? int(__ldg(cb + size_t(x) * q)) : 0;
    };
    const int x_s = ti0 * H;
    const int x_e = hr + (ti1 - 1) * H + m;
    int acc[H];
    int rg[H];
#pragma unroll
    for (int d = 0; d < H; ++d) {
        acc[d] = 0;
        rg[d] = (d < H - 1) ? B(x_s - hr + d) : 0;  // rows x_s-hr .. x_s+hr-1 in slots 0..H-2
    }
    int pa[P], pb[P];  // loads for the next P rows, issued one superblock ahead
#pragma unroll
    for (int j = 0; j < P; ++j) {
        pa[j] = A(x_s + j);
        pb[j] = B(x_s + j + hr);
    }
    const size_t plane = size_t(tr) * q;
    // window-start prefixes are parked in the output slot and turned into the window sum
    // at the window end (same thread, same address)
    unsigned* vout = V + size_t(t) * plane + (a_ok ? y : 0);
    const size_t dplane = size_t(W) * plane;
    const int end_s = (hr + m) % H;
    const int first_close = hr + ti0 * H + m;
    int open_t = ti0, close_t = ti0;
    for (int x0 = x_s; x0 <= x_e; x0 += P) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
            constexpr int dummy = 0;
            (void)dummy;
            const int s = j % H;
            const int x = x0 + j;
            if (s == hr && open_t < ti1) {  // window start (prefix before row x)
                if (a_ok) {
#pragma unroll
                    for (int d = 0; d < H; ++d)
                        vout[size_t(d) * dplane + size_t(open_t) * q] = unsigned(acc[d]);
                }
                ++open_t;
            }
            if (s == end_s && x >= first_close && close_t < ti1) {  // window end
                if (a_ok) {
#pragma unroll
                    for (int d = 0; d < H; ++d) {
                        unsigned* slot = vout + size_t(d) * dplane + size_t(close_t) * q;
                        *slot = unsigned(acc[d]) - *slot;
                    }
                }
                ++close_t;
            }
            rg[(s + H - 1) % H] = pb[j];  // I(x+hr, y+dj)
            const int a = pa[j];
            pa[j] = A(x + P);
            pb[j] = B(x + P + hr);
#pragma unroll
            for (int d = 0; d < H; ++d) acc[d] += a * rg[(s + d) % H];  // di = d - hr
        }
    }
}

// Clipped last centre row (irregular position): thread = (column y, dj, di).
__global__ void k_acv_last(const uint8_t* __restrict__ img, int p, int q, int m, int h, int w,
                           int cr, int tlast, int tr, unsigned* __restrict__ V) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y, d = blockIdx.z;
    const int dj = t - w / 2, di = d - h / 2;
    if (y >= q) return;
    const int yb = y + dj;
    unsigned acc = 0;
    if (yb >= 0 && yb < q) {
        const int a0 = max(0, -(cr + di)), a1 = min(m, p - (cr + di));
        const uint8_t* ca = img + size_t(cr) * q + y;
        const uint8_t* cb = img + size_t(cr + di) * q + yb;
#pragma unroll 8
        for (int a = a0; a < a1; ++a)
            acc += unsigned(__ldg(ca + size_t(a) * q)) * unsigned(__ldg(cb + size_t(a) * q));
    }
    V[((size_t(d) * w + t) * tr + tlast) * q + y] = acc;
}

// Pass 2: CTA per (centre row ti, row offset di, column tile [c0, c0+tw)).  For fixed
// (ti, di) the members of all groups in the tile row form one contiguous extent row
// mr = cr + di, so statistics loads and map writes are coalesced.  The W lines
// V[di,dj](ti, .) over [c0-1, c0+tw+n-1) are first prefix-summed (one warp per line,
// warp scans) into shared memory; then S = L_dj[cc+n-1] - L_dj[cc-1] and the FP64
// epilogue (autocorr.cpp:84-88) + retained count (egs.cpp:12-25) per member.
__global__ void __launch_bounds__(128)
    k_ac_hrow(const unsigned* __restrict__ V, int q, int m, int n, Grid g, DevStats st,
              double thr, double* __restrict__ map, unsigned long long* n_r, int tw, int lpitch) {
    extern __shared__ __align__(16) unsigned lines[];  // W lines x lpitch
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int ti = g.ti_lo + blockIdx.x, dii = blockIdx.y;
    const int c0 = blockIdx.z * tw;  // multiple of w: every tile here starts at or after c0
    const int hr = g.h / 2, wr = g.w / 2;
    const int di = dii - hr;
    const int cr = g.center_row(ti);
    const int r0 = ti * g.h, r1 = min(r0 + g.h, g.er) - 1;
    const int mr = cr + di;
    if (mr < r0 || mr > r1 || c0 >= g.ec) return;  // uniform across the CTA
    const int c1 = min(c0 + tw, g.ec);
    const int len = (c1 - c0) + n;  // local index u <-> column c0 - 1 + u
    // 1. prefix of each dj line over the tile (+ one column before, n-1 after)
    for (int t = wid; t < g.w; t += blockDim.x / 32) {
        const unsigned* src = V + ((size_t(dii) * g.w + t) * g.tr + ti) * q;
        unsigned* L = lines + size_t(t) * lpitch;
        unsigned carry = 0;
        for (int u0 = 0; u0 < len; u0 += 32) {
            const int u = u0 + lane;
            const int c = c0 - 1 + u;
            unsigned v = (u < len && c >= 0 && c < q) ? __ldg(src + c) : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned x = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += x;
            }
            v += carry;
            if (u < len) L[u] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    }
    __syncthreads();
    // 2. members of row mr in [c0, c1)
    const double mn = double(m) * double(n);
    unsigned long long local = 0;
    for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
        const int k = g.tile_c(c);
        const int cc = g.center_col(k);
        const int dj = c - cc;
        const size_t km = size_t(mr) * g.ec + c;
        if (di == 0 && dj == 0) {  // centres carry exactly 1 (autocorr.cpp:92-93)
            map[km] = 1.0;
            continue;
        }
        const unsigned* L = lines + size_t(dj + wr) * lpitch;
        const unsigned S = L[cc + n - c0] - L[cc - c0];  // P[cc+n-1] - P[cc-1]
        const size_t kc = size_t(cr) * g.ec + cc;
        double v = 0.0;
        if (!st.flat[kc] && !st.flat[km]) {
            const double num = __dsub_rn(double(S), __dmul_rn(__dmul_rn(mn, st.mu[kc]), st.mu[km]));
            v = dclamp(__ddiv_rn(num, __dmul_rn(st.omega[kc], st.omega[km])), -1.0, 1.0);
        }
        map[km] = v;
        if (v < thr) ++local;
    }
    local = warp_sum(local);
    if (lane == 0 && local) atomicAdd(n_r, local);
}

Grid to_grid(GridDesc d);

// ---- fused sliding-window R_co (preferred path) -----------------------------------------
//
// CTA = (column offset dj, column tile [c0, c0+tw), segment of centre rows).  Thread = one
// image column y of the tile plus its n-1 halo (NY = blockDim.x columns).  Each thread keeps
// the vertical window sums V_di(y) = sum_{a<m} I(cr+a, y) * I(cr+di+a, y+dj) for all h row
// offsets di as SLIDING sums: every row step adds the leading row and subtracts the row m
// above it (two register rings of B values, u32 arithmetic exact mod 2^32 and the true sums
// are < 2^32), so any centre row - the clipped last one included - is just an event on the
// walk.  At the event the CTA scans the h lines along y (block-wide inclusive scan into
// shared memory) and evaluates its members directly: S = L[cc+n-1] - L[cc-1], then the FP64
// epilogue of autocorr.cpp:84-88 and the retained count of egs.cpp:12-25.  Nothing but the
// map goes to HBM.
template <int H>
__global__ void __launch_bounds__(512)
    k_acf(const uint8_t* __restrict__ img, int p, int q, int m, int n, Grid g, DevStats st,
          double thr, double* __restrict__ map, unsigned long long* __restrict__ n_r, int tw,
          int seg, int* __restrict__ stop, const double* __restrict__ egs_prev, double egs_central,
          double egs_xi) {
    pdl_wait();
    if (stop && *stop) return;  // EGS already decided (egs_decide): candidate not needed
    constexpr int hr = H / 2;
    extern __shared__ __align__(16) unsigned acf_smem[];
    const int NY = blockDim.x;
    unsigned* L = acf_smem;  // 2 x [H][NY] warp-inclusive prefixes along y
    unsigned* wt = acf_smem + 2 * H * NY;  // 2 x [H][32] warp totals
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int dj = int(blockIdx.x) - g.w / 2;
    const int c0 = blockIdx.y * tw;
    const int ti0 = g.ti_lo + blockIdx.z * seg;
    const int ti1 = min(ti0 + seg, g.ti_hi);
    if (ti0 >= ti1 || c0 >= g.ec) return;  // uniform
    // Columns outside the image and rows below it only feed window sums that no valid
    // member reads (member windows lie inside the image), so the walk clamps columns and
    // relies on the kU8PadRows zero rows under the image instead of bounds checks.
    const int y = c0 + threadIdx.x;
    const uint8_t* ca = img + min(y, q - 1);
    const uint8_t* cb = img + min(max(y + dj, 0), q - 1);
    unsigned V[H], rl[H], rt[H];
    int cr = g.center_row(ti0);
#pragma unroll
    for (int d = 0; d < H; ++d) {
        V[d] = 0u;
        const int xr = max(cr - 1 - hr + d, 0);  // rows cr-hr .. cr+hr-1 in slots 1..H-1
        rl[d] = d >= 1 ? unsigned(__ldg(cb + unsigned(xr) * unsigned(q))) : 0u;
        rt[d] = rl[d];
    }
    // leading edge: A row x, B row x+hr; trailing edge: the same m rows above
    const uint8_t* la = ca + unsigned(cr) * unsigned(q);
    const uint8_t* lb = cb + unsigned(cr + hr) * unsigned(q);
    const uint8_t* ta = la;
    const uint8_t* tb = lb;
    auto lead_v = [&](unsigned a, unsigned b) {
#pragma unroll
        for (int d = 0; d < H - 1; ++d) rl[d] = rl[d + 1];
        rl[H - 1] = b;
#pragma unroll
        for (int d = 0; d < H; ++d) V[d] += a * rl[d];  // di = d - hr
    };
    auto trail_v = [&](unsigned a, unsigned b) {  // remove the row m above the leading edge
#pragma unroll
        for (int d = 0; d < H - 1; ++d) rt[d] = rt[d + 1];
        rt[H - 1] = b;
#pragma unroll
        for (int d = 0; d < H; ++d) V[d] -= a * rt[d];
    };
    auto lead = [&]() {
        const unsigned b = unsigned(__ldg(lb)), a = unsigned(__ldg(la));
        la += q;
        lb += q;
        lead_v(a, b);
    };
    auto trail = [&]() {
        const unsigned b = unsigned(__ldg(tb)), a = unsigned(__ldg(ta));
        ta += q;
        tb += q;
        trail_v(a, b);
    };

    // warm-up: the first window rows [cr, cr+m)
    {
        int x = cr;
        const int xe = cr + m;
#pragma unroll 1
        for (; x + H <= xe; x += H) {
#pragma unroll
            for (int j = 0; j < H; ++j) lead();
        }
#pragma unroll 1
        for (; x < xe; ++x) lead();
    }
    const double mn = double(m) * double(n);
    const int tj0 = c0 / g.w;
    const int tj1 = min(g.tc, (c0 + tw) / g.w);
    const int ng = tj1 - tj0;
    // Fixed member slots: slot j of this thread is member i = tid + j*NY of every event,
    // (row offset d = i / ng, group k = i % ng); the column side is constant per CTA.
    constexpr int kSlots = 1;  // acf_geom keeps h * groups-per-tile <= NY
    int s_d[kSlots], s_c[kSlots], s_cc[kSlots], s_u[kSlots];
    bool s_ok[kSlots];
#pragma unroll
    for (int j = 0; j < kSlots; ++j) {
        const int i = threadIdx.x + j * NY;
        s_ok[j] = i < H * ng;
        const int d = s_ok[j] ? i / ng : 0, k = s_ok[j] ? i - d * ng : 0;
        const int tj = tj0 + k;
        const int gc0 = tj * g.w, gc1 = min(gc0 + g.w, g.ec) - 1;
        const int cc = (gc0 + gc1) >> 1;
        const int c = cc + dj;
        s_ok[j] = s_ok[j] && c >= gc0 && c <= gc1;
        s_d[j] = d;
        s_c[j] = c;
        s_cc[j] = cc;
        s_u[j] = cc - c0;
    }
    // statistics of the next event's members, loaded one walk ahead
    uint8_t pf_fc[kSlots], pf_fm[kSlots];
    double pf_mc[kSlots], pf_mm[kSlots], pf_oc[kSlots], pf_om[kSlots];
    bool pf_row[kSlots];
    auto prefetch = [&](int tin, int crn) {
        const int r0 = tin * g.h, r1 = min(r0 + g.h, g.er) - 1;
#pragma unroll
        for (int j = 0; j < kSlots; ++j) {
            const int mr = crn + s_d[j] - hr;
            pf_row[j] = s_ok[j] && mr >= r0 && mr <= r1;
            const unsigned kc = pf_row[j] ? unsigned(crn) * unsigned(g.ec) + unsigned(s_cc[j]) : 0u;
            const unsigned km = pf_row[j] ? unsigned(mr) * unsigned(g.ec) + unsigned(s_c[j]) : 0u;
            pf_fc[j] = st.flat[kc];
            pf_fm[j] = st.flat[km];
            pf_mc[j] = st.mu[kc];
            pf_mm[j] = st.mu[km];
            pf_oc[j] = st.omega[kc];
            pf_om[j] = st.omega[km];
        }
    };
    prefetch(ti0, cr);
    // Retained count: per-event warp sums into a CTA counter.  Inside an EGS batch
    // (egs_prev != 0) thread 0 flushes it to the global count every 2 events and replays
    // the acceptance test of egs.cpp:61-88 (same FP64 operations as k_egs_decide): the test
    // is monotone in n_r, so once the partial count already rejects the candidate the rest
    // of its work cannot change the decision -- the CTA stops, and the stop flag makes the
    // remaining CTAs and candidates exit.  Accepted candidates are always counted in full.
    __shared__ unsigned cta_cnt;
    if (threadIdx.x == 0) cta_cnt = 0u;
    const double prev = (egs_prev && stop) ? *egs_prev : 0.0;
    const bool can_reject = egs_prev && stop && fabs(prev) <= 1.7976931348623157e308;
    int my_abort = 0, ev = 0;
    int parity = 0;
#pragma unroll 1
    for (int ti = ti0;;) {
        // ---- event: window [cr, cr+m) complete in V ----
        // warp-local inclusive prefixes + warp totals, double-buffered by event parity so a
        // single barrier per event suffices (the next writer of this buffer is two events
        // away, behind the next event's barrier).
        unsigned* Lb = L + (parity ? H * NY : 0);
        unsigned* wb = wt + (parity ? H * 32 : 0);
        parity ^= 1;
        {
            unsigned v[H];
#pragma unroll
            for (int d = 0; d < H; ++d) v[d] = V[d];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                for (int d = 0; d < H; ++d) {
                    const unsigned t = __shfl_up_sync(0xffffffffu, v[d], o);
                    if (lane >= o) v[d] += t;
                }
            }
#pragma unroll
            for (int d = 0; d < H; ++d) {
                Lb[d * NY + threadIdx.x] = v[d];
                if (lane == 31) wb[d * 32 + wid] = v[d];
            }
        }
        if (__syncthreads_or(my_abort)) break;  // uniform: thread 0's flag from a past event
        if (can_reject && threadIdx.x == 0 && (++ev & 1) == 0) {
            const unsigned c = atomicExch(&cta_cnt, 0u);
            const unsigned long long tot = atomicAdd(n_r, (unsigned long long)c) + c;
            const double total = __dadd_rn(__dadd_rn(egs_central, double(tot)), 0.0);
            if (!(__dsub_rn(prev, total) > __dmul_rn(egs_xi, prev))) {
                my_abort = 1;
                *reinterpret_cast<volatile int*>(stop) = 1;
            }
        }
        unsigned evc = 0;
#pragma unroll
        for (int j = 0; j < kSlots; ++j) {
            if (!pf_row[j]) continue;
            const int d = s_d[j];
            const unsigned km = unsigned(cr + d - hr) * unsigned(g.ec) + unsigned(s_c[j]);
            if (d == hr && dj == 0) {  // centres carry exactly 1 (autocorr.cpp:92-93)
                if (map) map[km] = 1.0;
                continue;
            }
            // S = P[u+n-1] - P[u-1], P the block prefix = warp prefix + earlier warp totals
            // (at most kSpan warp totals between the two ends; wt is padded for the reads)
            const int u = s_u[j];
            const int i1 = u + n - 1, w1 = i1 >> 5;
            const unsigned* Ld = Lb + d * NY;
            unsigned S = Ld[i1];
            int w0 = 0;
            if (u > 0) {
                S -= Ld[u - 1];
                w0 = (u - 1) >> 5;
            }
            const unsigned* wd = wb + d * 32 + w0;
            constexpr int kSpan = 8;
#pragma unroll
            for (int k = 0; k < kSpan; ++k) S += (w0 + k < w1) ? wd[k] : 0u;
            const bool flat = pf_fc[j] || pf_fm[j];
            const double num = __dsub_rn(double(S), __dmul_rn(__dmul_rn(mn, pf_mc[j]), pf_mm[j]));
            const double den = __dmul_rn(pf_oc[j], pf_om[j]);
            if (!map) {  // EGS candidate: retained count only
                if (flat ? 0.0 < thr : retained_below(num, den, thr)) ++evc;
                continue;
            }
            const double val = flat ? 0.0 : dclamp(__ddiv_rn(num, den), -1.0, 1.0);
            map[km] = val;
            if (val < thr) ++evc;
        }
        evc = __reduce_add_sync(0xffffffffu, evc);
        if (lane == 0 && evc) atomicAdd(&cta_cnt, evc);
        if (++ti >= ti1) break;
        // ---- advance the window to the next centre row ----
        const int crn = g.center_row(ti);
        prefetch(ti, crn);
        if (crn - cr == H) {
#pragma unroll
            for (int j = 0; j < H; ++j) {
                lead();
                trail();
            }
        } else {
#pragma unroll 1
            for (int x = cr; x < crn; ++x) {
                lead();
                trail();
            }
        }
        cr = crn;
    }
    __syncthreads();
    if (threadIdx.x == 0 && cta_cnt) atomicAdd(n_r, (unsigned long long)cta_cnt);
}

struct AcfGeom {
    int ny, tw, seg, nseg, ntiles;
    size_t smem;
};

AcfGeom acf_geom(int m, int n, GridDesc gd, int resident = 0) {
    AcfGeom a{};
    int ny = std::max(128, 4 * n);
    ny = std::max(ny, n - 1 + 2 * gd.w);
    ny = (ny + 31) & ~31;
    if (ny > 512) return AcfGeom{};
    a.ny = ny;
    a.tw = ((a.ny - n + 1) / gd.w) * gd.w;
    if (a.tw < gd.w) return AcfGeom{};
    a.tw = std::min(a.tw, (a.ny / gd.h) * gd.w);  // one member slot per thread
    if (a.tw < gd.w) return AcfGeom{};
    a.ntiles = (gd.ec + a.tw - 1) / a.tw;
    const int rows = gd.ti_hi - gd.ti_lo;
    const int seg_min = std::max(1, (m + gd.h - 1) / gd.h);
    if (resident <= 0) resident = std::max(1, 2048 / a.ny);
    // As few waves of resident CTAs as keep segments short: each segment pays its m-row
    // warm-up once, and with one wave the EGS early rejection reaches every CTA at the same
    // fraction of its work; long segments (large images) get up to 4 waves for balance.
    const int slots = 148 * resident;
    const int per_wave = std::max(1, slots / std::max(1, gd.w * a.ntiles));
    const int seg_1 = (rows + per_wave - 1) / per_wave;
    const int waves = std::min(4, std::max(1, (seg_1 + 4 * seg_min - 1) / (4 * seg_min)));
    int nseg = std::max(1, waves * per_wave);
    nseg = std::min(nseg, std::max(1, (rows + seg_min - 1) / seg_min));
    a.seg = std::max(1, (rows + nseg - 1) / nseg);
    a.nseg = std::max(1, (rows + a.seg - 1) / a.seg);
    a.smem = (2 * size_t(gd.h) * (a.ny + 32) + 16) * sizeof(unsigned);  // + padding (kSpan)
    return a;
}

template <int H>
cudaError_t launch_acf(const uint8_t* img, int p, int q, int m, int n, GridDesc gd, DevStats st,
                       double thr, double* map, unsigned long long* n_r, int* stop,
                       const double* egs_prev, double egs_central, double egs_xi, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_acf<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        attr = true;
    }
    const AcfGeom a0 = acf_geom(m, n, gd);
    if (a0.ny == 0) return cudaErrorInvalidValue;
    int occ = 0;  // resident CTAs per SM for this block size / shared memory
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_acf<H>, a0.ny, a0.smem) != cudaSuccess)
        occ = 0;
    const AcfGeom a = acf_geom(m, n, gd, occ);
    dim3 grid(gd.w, a.ntiles, a.nseg);
    if (gd.ti_hi > gd.ti_lo)
        launch_pdl(k_acf<H>, dim3(grid), dim3(a.ny), a.smem, s, img, p, q, m, n, to_grid(gd), st, thr, map, n_r, a.tw,
                                            a.seg, stop, egs_prev, egs_central, egs_xi);
    return cudaGetLastError();
}

__device__ void egs_decide_run(const EgsDecide& d) {
    if (!*d.stop) {
        const double central =
            __dmul_rn(double((d.er + d.h - 1) / d.h), double((d.ec + d.w - 1) / d.w));
        const double total = __dadd_rn(__dadd_rn(central, double(*d.n_r)), 0.0);
        const double prev = *d.prev;
        const bool first = !(fabs(prev) <= 1.7976931348623157e308);  // !isfinite
        const bool accepted = first || __dsub_rn(prev, total) > __dmul_rn(d.xi, prev);
        if (!accepted) {
            *d.stop = 1;
        } else {
            *d.prev = total;
            *d.h_acc = d.h;
            if ((d.h >= d.er && d.w >= d.ec) || (d.h >= d.cap && d.w >= d.cap)) *d.stop = 1;
        }
    }
    // (a stop set at entry came from an earlier decision or from the candidate's own
    // in-kernel rejection; either way h_acc is final)
    const unsigned long long gv = (*d.stop && d.want > 0 && *d.h_acc == d.want) ? 1ull : 0ull;
    *d.gate = gv;
    if (d.out && d.disp_dense) {  // k_survivor_dispatch for the gated survivors behind
        const unsigned long long ns = gv ? d.disp_tally->survivors : 0ull;
        const bool dense = ns * kDenseDiv > d.disp_E;
        *d.disp_dense = dense ? 1 : 0;
        *d.disp_list = dense ? 0ull : ns;
    }
    if (d.out) {  // last candidate of the batch: counts + gate into the mapped result block
        for (int i = 0; i < d.nc; ++i) d.out->nr[i] = d.nr_all[i];
        d.out->spec = gv;
        __threadfence_system();  // counts visible to the host before the sequence number
        *reinterpret_cast<volatile unsigned long long*>(&d.out->seq) = d.seq;
    }
}

// Tail of a fused R_co launch: every thread of every block calls it once, after the block's
// count is published; the last block to take a ticket runs the decision.
__device__ __forceinline__ void egs_tail(const EgsDecide& d) {
    if (!d.ticket) return;  // uniform
    __shared__ int is_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(d.ticket, 1u) == gridDim.x * gridDim.y * gridDim.z - 1;
    }
    __syncthreads();
    if (is_last && threadIdx.x == 0) {
        __threadfence();
        *d.ticket = 0u;
        egs_decide_run(d);
    }
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// ---- fused R_co, one thread per group column (square groups, h <= 5) ----------------------
//
// The walk of k_acf, but thread t owns the W = h image columns [cc_k, cc_k + W) of group
// column k = k0 + t (cc_k = k*W + W/2, the centre column of a full group).  The W x h
// vertical sliding sums stay in registers, the block scan runs over group blocks
// B(t) = sum_j V[di][j] (W times fewer scan steps than per column), and at each event the
// thread evaluates the h members of its own group (one centre statistic for h members).
// A window [cc_k, cc_k + n) is the Q = n / W whole blocks t .. t+Q-1 plus the first
// R = n % W columns of block t+Q ("head").  The clipped last group column (ec % W != 0) has
// its centre delta columns left of cc_k: its window is the last delta columns of block t-1
// ("tail"), Qc whole blocks from t and the first Rc columns of block t+Qc; the tile
// geometry keeps that group off thread 0.  Same sums, same FP64 epilogue, same map and
// count as k_acf (u32 sums are exact mod 2^32 and the true sums are < 2^32).
//
// Image rows reach the walk through a shared-memory ring (RR = m + 2h + h/2 rows of the
// tile's SW-byte column span, A and B sides share it): the rows of the next transition
// are copied with 16-byte cp.async one event ahead, so the walk reads bytes at shared-
// memory latency instead of waiting on L2 for the trailing rows m rows back.  `img` is the
// 16-byte-pitched zero-padded copy (pitch P, >= p + kU8PadRows rows).
constexpr int kAcgWb = 8;  // warp-total stride (NT <= 256, read as uint4: NT % 128 == 0)
// staged bytes per ring row: NT*W tile columns + 2*(h/2) for the B offsets + 16-byte alignment
// (+8: the packed walk reads two aligned words from up to 3 bytes before a thread's columns)
__host__ __device__ constexpr int acg_span(int nt, int h) { return (15 + nt * h + 2 * (h / 2) + 8 + 15) & ~15; }

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    const unsigned sa = unsigned(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void opaque(unsigned& x) { asm("" : "+r"(x)); }
__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
    const unsigned sa = unsigned(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// NP > 0: packed walk.  A thread's W columns are cut into NP parts (each <= 4 columns) at
// the column counts its block sums are read at -- R = n % W for every thread, plus the
// clipped group's tail (W - delta) and head (Rc) on the two threads that provide them --
// and each part's vertical sum is one dp4a per row step (u8 x u8 -> u32, exact): the A row
// part words are byte permutes of two aligned shared-memory words, the B row part words
// (kept in the register ring for H steps) are masked to the part's bytes.  Leading and
// trailing rows accumulate separately (dp4a only adds) and are subtracted at the events.
// NP = 2 when the grid has no clipped group column, 3 otherwise; NP = 0 is the per-column
// walk (one IMAD per column, offset and row step).
// FUSE: scan 2 in the epilogue (SecFuse; the map is not written).
template <int H, int NT, int NP, bool FUSE>
__global__ void __launch_bounds__(NT)
    k_acg(const uint8_t* __restrict__ img, int P, int q, int m, int n, Grid g, DevStats st,
          double thr, double* __restrict__ map, unsigned long long* __restrict__ n_r, int G,
          int seg, int RR, int* __restrict__ stop, const double* __restrict__ egs_prev,
          double egs_central, double egs_xi, EgsDecide dec, SecFuse sf, int tile_base) {
    static_assert(NT % 128 == 0 && NT <= 32 * kAcgWb, "warp totals are read as uint4");
    pdl_wait();
    constexpr int W = H, hr = H / 2;
    constexpr int SW = acg_span(NT, H);  // staged bytes per ring row
    constexpr int NCH = SW / 16;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    // Launch order: (dj, tile, segment) with dj fastest.  A count-only candidate with a
    // segment order (EgsDecide::zorder) runs dj slowest instead, the outer column offsets
    // first (|dj| = hr members are retained about twice as often as the inner ones: C5,
    // h = 5: 65 % vs 26-34 %), segments densest first, so its in-kernel rejection comes
    // after fewer CTAs (any subset count reaching the bound rejects: the test is monotone).
    int bdj = int(blockIdx.x), btile = int(blockIdx.y), bseg = int(blockIdx.z);
    if (dec.zorder) {
        const int ny = int(gridDim.y), nz = int(gridDim.z);
        const int L = int(blockIdx.x) + int(gridDim.x) * (int(blockIdx.y) + ny * int(blockIdx.z));
        const int djr = L / (ny * nz), rem = L - djr * (ny * nz);
        bseg = dec.zorder[rem / ny];
        btile = rem - (rem / ny) * ny;
        // rank -> offset: -hr, +hr, -(hr-1), +(hr-1), ..., 0
        const int mag = hr - (djr >> 1);
        bdj = hr + ((djr & 1) ? mag : -mag);
    }
    const int dj = bdj - hr;
    const int k0 = (btile + tile_base) * G;
    const int zseg = bseg;
    const int ti0 = g.ti_lo + zseg * seg;
    const int ti1 = min(ti0 + seg, g.ti_hi);
    {
        // skipped candidate (an earlier decision stopped EGS) or empty block: one read of
        // the flag per block so the exit is uniform
        __shared__ int skip;
        // phase B after k_rco5_s / k_rco5_cnt: an outer-offset CTA runs only for the tile
        // holding the clipped last group column (if any), for that group alone
        const int wlc = g.ec - (g.tc - 1) * W;
        const bool outer_skip = dec.outer_done && (dj == -hr || dj == hr) &&
                                !(wlc < W && g.tc - 1 >= k0 && g.tc - 1 < k0 + G);
        if (t == 0) skip = (stop && *reinterpret_cast<volatile int*>(stop)) || ti0 >= ti1 ||
                           k0 >= g.tc || outer_skip;
        __syncthreads();
        if (skip) {
            egs_tail(dec);
            return;
        }
    }
    const int k = k0 + t;
    const int Q = n / W, R = n - Q * W;
    const int wl = g.ec - (g.tc - 1) * W;  // width of the last group column
    const bool clip_tile = wl < W && g.tc - 1 < k0 + G;  // uniform
    const int delta = hr - ((wl - 1) >> 1);
    const int Qc = (n - delta) / W, Rc = (n - delta) - Qc * W;
    extern __shared__ __align__(16) unsigned acg_smem[];
    constexpr int PS = H * (4 * NT + kAcgWb);  // per parity: Lb | Hh | Tt | Hc [H][NT], wb [H][8]
    uint8_t* ring = reinterpret_cast<uint8_t*>(acg_smem + 2 * PS);
    const int s0 = (k0 * W) & ~15;  // first staged column (16-byte aligned)
    auto stage = [&](int r_lo, int nrows) {  // rows [r_lo, r_lo + nrows) -> ring slots
        const int slot0 = r_lo % RR;
        for (int i = t; i < nrows * NCH; i += NT) {
            const int rr = i / NCH, c = i - rr * NCH;
            int slot = slot0 + rr;
            if (slot >= RR) slot -= RR;
            cp_async16(ring + slot * SW + c * 16, img + size_t(r_lo + rr) * P + s0 + c * 16);
        }
        cp_async_commit();
    };

    const int y0 = k * W + hr;  // every thread's columns lie inside the staged span
    const int oa = y0 - s0, ob = y0 + dj - s0;
    // this thread's group column geometry (also used by the packed walk's cuts)
    const int tcl = g.tc - 1 - k0;  // tile-local index of the clipped group column (if here)
    constexpr int NPV = NP > 0 ? NP : 1;
    constexpr int NA = NP > 0 ? NP : W;  // accumulators per row offset
    unsigned V[H][NA], Vt[H][NP > 0 ? NP : 1], rl[H][NA], rt[H][NA];
    // packed walk: parts [plo[i], plo[i+1]) of the W columns, selectors and masks
    unsigned selA[NPV], selB[NPV], mskB[NPV];
    unsigned pm_h = 0, pm_t = 0, pm_c = 0;  // parts inside the head R / tail / clipped head
    if constexpr (NP > 0) {
        int cut[4], nc = 0;
        auto add_cut = [&](int c) {
            if (c <= 0 || c >= W) return;
            for (int i = 0; i < nc; ++i)
                if (cut[i] == c) return;
            cut[nc++] = c;
        };
        add_cut(R);
        if (clip_tile && tcl >= 1 && t == tcl - 1) add_cut(W - delta);
        if (clip_tile && tcl >= 0 && t == tcl + Qc) add_cut(Rc);
        if (nc == 0 && W > 4) add_cut(4);  // every part fits one 32-bit word
        for (int i = 1; i < nc; ++i)       // sort (nc <= 3)
            for (int j = i; j > 0 && cut[j - 1] > cut[j]; --j) {
                const int x = cut[j];
                cut[j] = cut[j - 1];
                cut[j - 1] = x;
            }
        const int sha = oa & 3, shb = ob & 3;
#pragma unroll
        for (int i = 0; i < NPV; ++i) {
            const int lo = i == 0 ? 0 : (i - 1 < nc ? cut[i - 1] : W);
            const int hi = i < nc ? cut[i] : W;
            unsigned sa = 0, sb = 0, mb = 0;
            for (int b = 0; b < 4; ++b) {
                if (lo + b < hi) {
                    sa |= unsigned(sha + lo + b) << (4 * b);
                    sb |= unsigned(shb + lo + b) << (4 * b);
                    mb |= 0xffu << (8 * b);
                }
            }
            selA[i] = sa;
            selB[i] = sb;
            mskB[i] = mb;
            if (hi > lo && hi <= R) pm_h |= 1u << i;
            if (hi > lo && lo >= W - delta) pm_t |= 1u << i;
            if (hi > lo && hi <= Rc) pm_c |= 1u << i;
        }
    }
    const int oa4 = NP > 0 ? (oa & ~3) : oa, ob4 = NP > 0 ? (ob & ~3) : ob;
    int cr = g.center_row(ti0);
    stage(cr, m + H + hr);
#pragma unroll
    for (int d = 0; d < H; ++d) {
        const int xr = max(cr - 1 - hr + d, 0);
        if constexpr (NP > 0) {
            // ring prefill from global memory (the staged ring starts at row cr)
            unsigned w0 = 0, w1 = 0;
            if (d >= 1) {
                const uint8_t* src = img + size_t(xr) * P + s0 + ob4;
                w0 = __ldg(reinterpret_cast<const unsigned*>(src));
                w1 = __ldg(reinterpret_cast<const unsigned*>(src + 4));
            }
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                V[d][i] = 0u;
                Vt[d][i] = 0u;
                rl[d][i] = __byte_perm(w0, w1, selB[i]) & mskB[i];
                rt[d][i] = rl[d][i];
            }
        } else {
#pragma unroll
            for (int j = 0; j < W; ++j) {
                V[d][j] = 0u;
                rl[d][j] = d >= 1 ? unsigned(__ldg(img + size_t(xr) * P + y0 + dj + j)) : 0u;
                rt[d][j] = rl[d][j];
            }
        }
    }
    // ring byte offsets of the leading / trailing A and B rows (wrap at RR * SW)
    const int ring_bytes = RR * SW;
    int la = (cr % RR) * SW, lb = ((cr + hr) % RR) * SW;
    int ta = la, tb = lb;
    auto bump = [&](int& o, int by) {
        o += by;
        if (o >= ring_bytes) o -= ring_bytes;
    };
    auto lead_at = [&](const uint8_t* pa, const uint8_t* pb) {
        if constexpr (NP > 0) {
            const unsigned a0 = *reinterpret_cast<const unsigned*>(pa);
            const unsigned a1 = *reinterpret_cast<const unsigned*>(pa + 4);
            const unsigned b0 = *reinterpret_cast<const unsigned*>(pb);
            const unsigned b1 = *reinterpret_cast<const unsigned*>(pb + 4);
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const unsigned aw = __byte_perm(a0, a1, selA[i]);  // bytes past the part: x 0
#pragma unroll
                for (int d = 0; d < H - 1; ++d) rl[d][i] = rl[d + 1][i];
                rl[H - 1][i] = __byte_perm(b0, b1, selB[i]) & mskB[i];
#pragma unroll
                for (int d = 0; d < H; ++d) V[d][i] = __dp4a(aw, rl[d][i], V[d][i]);
            }
        } else {
            unsigned a[W], b[W];
#pragma unroll
            for (int j = 0; j < W; ++j) {
                b[j] = pb[j];
                a[j] = pa[j];
                opaque(a[j]);  // plain IMADs: keeps nvcc from packing bytes into IDP (PRMT-heavy)
                opaque(b[j]);
            }
#pragma unroll
            for (int j = 0; j < W; ++j) {
#pragma unroll
                for (int d = 0; d < H - 1; ++d) rl[d][j] = rl[d + 1][j];
                rl[H - 1][j] = b[j];
#pragma unroll
                for (int d = 0; d < H; ++d) V[d][j] += a[j] * rl[d][j];
            }
        }
    };
    auto trail_at = [&](const uint8_t* pa, const uint8_t* pb) {
        if constexpr (NP > 0) {
            const unsigned a0 = *reinterpret_cast<const unsigned*>(pa);
            const unsigned a1 = *reinterpret_cast<const unsigned*>(pa + 4);
            const unsigned b0 = *reinterpret_cast<const unsigned*>(pb);
            const unsigned b1 = *reinterpret_cast<const unsigned*>(pb + 4);
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const unsigned aw = __byte_perm(a0, a1, selA[i]);
#pragma unroll
                for (int d = 0; d < H - 1; ++d) rt[d][i] = rt[d + 1][i];
                rt[H - 1][i] = __byte_perm(b0, b1, selB[i]) & mskB[i];
#pragma unroll
                for (int d = 0; d < H; ++d) Vt[d][i] = __dp4a(aw, rt[d][i], Vt[d][i]);
            }
        } else {
            unsigned a[W], b[W];
#pragma unroll
            for (int j = 0; j < W; ++j) {
                b[j] = pb[j];
                // h = 5: negated once so the H updates are single IMADs (measured: h = 3 is
                // faster with the plain subtraction, which nvcc schedules better there)
                a[j] = H >= 5 ? 0u - unsigned(pa[j]) : unsigned(pa[j]);
                opaque(a[j]);
                opaque(b[j]);
            }
#pragma unroll
            for (int j = 0; j < W; ++j) {
#pragma unroll
                for (int d = 0; d < H - 1; ++d) rt[d][j] = rt[d + 1][j];
                rt[H - 1][j] = b[j];
#pragma unroll
                for (int d = 0; d < H; ++d) {
                    if (H >= 5) V[d][j] += a[j] * rt[d][j];  // exact mod 2^32
                    else V[d][j] -= a[j] * rt[d][j];
                }
            }
        }
    };
    auto lead = [&]() {
        lead_at(ring + la + oa4, ring + lb + ob4);
        bump(la, SW);
        bump(lb, SW);
    };
    auto trail = [&]() {
        trail_at(ring + ta + oa4, ring + tb + ob4);
        bump(ta, SW);
        bump(tb, SW);
    };
    // H row steps; straight-line (immediate ring offsets) unless a stream wraps inside them
    const int lim = ring_bytes - (H - 1) * SW;
    auto advance_lead = [&]() {
        if (la < lim && lb < lim) {
            const uint8_t* pa = ring + la + oa4;
            const uint8_t* pb = ring + lb + ob4;
#pragma unroll
            for (int s = 0; s < H; ++s) lead_at(pa + s * SW, pb + s * SW);
            bump(la, H * SW);
            bump(lb, H * SW);
        } else {
#pragma unroll
            for (int s = 0; s < H; ++s) lead();
        }
    };
    auto advance_both = [&]() {
        if (la < lim && lb < lim && ta < lim && tb < lim) {
            const uint8_t* pa = ring + la + oa4;
            const uint8_t* pb = ring + lb + ob4;
            const uint8_t* qa = ring + ta + oa4;
            const uint8_t* qb = ring + tb + ob4;
#pragma unroll
            for (int s = 0; s < H; ++s) {
                lead_at(pa + s * SW, pb + s * SW);
                trail_at(qa + s * SW, qb + s * SW);
            }
            bump(la, H * SW);
            bump(lb, H * SW);
            bump(ta, H * SW);
            bump(tb, H * SW);
        } else {
#pragma unroll
            for (int s = 0; s < H; ++s) {
                lead();
                trail();
            }
        }
    };
    cp_async_wait_all();
    __syncthreads();
    {
        int x = cr;
        const int xe = cr + m;
#pragma unroll 1
        for (; x + H <= xe; x += H) advance_lead();
#pragma unroll 1
        for (; x < xe; ++x) lead();
    }
    const double mn = double(m) * double(n);
    // this thread's group: members (di, dj) of group column k, all h row offsets
    const bool owner = t < G && k < g.tc &&
                       !(dec.outer_done && (dj == -hr || dj == hr) && k != g.tc - 1);
    const int gc0 = k * W, gc1 = min(gc0 + W, g.ec) - 1;
    const int cc = (gc0 + gc1) >> 1;
    const int c = cc + dj;
    const bool col_ok = owner && c >= gc0 && c <= gc1;
    const bool clipped = owner && gc1 - gc0 + 1 < W;
    const int hi = clipped ? t + Qc : t + Q;  // whole blocks [t, hi)
    const bool has_head = clipped ? Rc > 0 : R > 0;
    const int i1 = hi - 1;
    const int w0 = t > 0 ? (t - 1) >> 5 : 0, w1 = i1 >= 0 ? i1 >> 5 : 0;
    uint8_t pf_fc, pf_fm[H];
    double pf_mc, pf_oc, pf_mm[H], pf_om[H];
    bool pf_row[H];
    // FUSE: the group's scan-1 values (one group per thread and event)
    double pf_ra = 0.0, pf_sa = 0.0;
    uint8_t pf_dg = 0, pf_sd = 0;
    auto prefetch = [&](int tin, int crn) {
        const int r0 = tin * g.h, r1 = min(r0 + g.h, g.er) - 1;
        if constexpr (FUSE) {
            const size_t gi = col_ok ? size_t(tin) * g.tc + k : 0;
            pf_ra = sf.rho_c[gi];
            pf_sa = sf.sa_c[gi];
            pf_dg = sf.deg_c[gi];
            pf_sd = sf.seeded ? sf.seeded[gi] : uint8_t(0);
        }
        const unsigned kc = col_ok ? unsigned(crn) * unsigned(g.ec) + unsigned(cc) : 0u;
        pf_fc = st.flat[kc];
        pf_mc = st.mu[kc];
        pf_oc = st.omega[kc];
#pragma unroll
        for (int d = 0; d < H; ++d) {
            const int mr = crn + d - hr;
            pf_row[d] = col_ok && mr >= r0 && mr <= r1;
            const unsigned km = pf_row[d] ? unsigned(mr) * unsigned(g.ec) + unsigned(c) : 0u;
            pf_fm[d] = st.flat[km];
            pf_mm[d] = st.mu[km];
            pf_om[d] = st.omega[km];
        }
    };
    prefetch(ti0, cr);
    __shared__ unsigned cta_cnt;
    if (t == 0) cta_cnt = 0u;
    const double prev = (egs_prev && stop) ? *egs_prev : 0.0;
    const bool can_reject = egs_prev && stop && fabs(prev) <= 1.7976931348623157e308;
    int my_abort = 0, ev = 0, parity = 0;
    // FUSE: scan-2 state (k_sec_rows): threshold, tallies, survivor-list state of this warp
    double sec_tb = 0.0;
    float sec_tbf = 0.f;
    bool thr_ok = false;
    if constexpr (FUSE) {
        const double T = *sf.thr;
        sec_tb = dclamp(dmin(T, 1.0), -1.0, 1.0);
        sec_tbf = float(sec_tb);
        thr_ok = T >= -1.0;
    }
    unsigned n_elim = 0, n_keep = 0, n_flat = 0;
    unsigned long long fkey = 0;  // retained flat members: first position (Tally::flat_key)
    bool list_full = false;
    unsigned long long surv_local = 0;
#pragma unroll 1
    for (int ti = ti0;;) {
        unsigned* Lb = acg_smem + (parity ? PS : 0);
        unsigned* Hh = Lb + H * NT;
        unsigned* Tt = Hh + H * NT;
        unsigned* Hc = Tt + H * NT;
        unsigned* wb = Hc + H * NT;
        parity ^= 1;
        {
            unsigned v[H];
#pragma unroll
            for (int d = 0; d < H; ++d) {
                unsigned bs = 0u, hh = 0u, tt = 0u, hc = 0u;
                if constexpr (NP > 0) {
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        const unsigned x = V[d][i] - Vt[d][i];  // exact mod 2^32
                        bs += x;
                        if ((pm_h >> i) & 1u) hh += x;
                        if ((pm_t >> i) & 1u) tt += x;
                        if ((pm_c >> i) & 1u) hc += x;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < W; ++j) {
                        bs += V[d][j];
                        if (j < R) hh += V[d][j];
                        if (j >= W - delta) tt += V[d][j];
                        if (j < Rc) hc += V[d][j];
                    }
                }
                v[d] = bs;
                Hh[d * NT + t] = hh;
                if (clip_tile) {
                    Tt[d * NT + t] = tt;
                    Hc[d * NT + t] = hc;
                }
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                for (int d = 0; d < H; ++d) {
                    const unsigned u = __shfl_up_sync(0xffffffffu, v[d], o);
                    if (lane >= o) v[d] += u;
                }
            }
#pragma unroll
            for (int d = 0; d < H; ++d) {
                Lb[d * NT + t] = v[d];
                if (lane == 31) wb[d * kAcgWb + wid] = v[d];
            }
        }
        cp_async_wait_all();                    // this thread's rows of the next transition
        if (__syncthreads_or(my_abort)) break;  // uniform
        if (ti + 2 < ti1) stage(g.center_row(ti + 1) + m + hr, H);  // the one after it
        if (can_reject && t == 0 && (++ev & 1) == 0) {
            const unsigned cn = atomicExch(&cta_cnt, 0u);
            const unsigned long long tot = atomicAdd(n_r, (unsigned long long)cn) + cn;
            const double total = __dadd_rn(__dadd_rn(egs_central, double(tot)), 0.0);
            if (!(__dsub_rn(prev, total) > __dmul_rn(egs_xi, prev))) {
                my_abort = 1;
                *reinterpret_cast<volatile int*>(stop) = 1;
            }
        }
        unsigned evc = 0;
        unsigned surv = 0;  // FUSE: members of this event that survive the bound test (bit d)
        // FUSE: this event's group constants (centre rho clamped, its FP32 copies)
        bool grp_test = false;
        double g_a = 0.0;
        float g_af = 0.f, g_saf = 0.f;
        if constexpr (FUSE) {
            grp_test = thr_ok && !pf_dg && !sf.tflat;
            g_a = dclamp(pf_ra, -1.0, 1.0);
            g_af = float(g_a);
            g_saf = float(pf_sa);
        }
        if (col_ok) {
#pragma unroll
            for (int d = 0; d < H; ++d) {
                if (!pf_row[d]) continue;
                const unsigned km = unsigned(cr + d - hr) * unsigned(g.ec) + unsigned(c);
                if (d == hr && dj == 0) {  // centres carry exactly 1 (autocorr.cpp:92-93)
                    if (map) map[km] = 1.0;
                    if constexpr (FUSE) sf.visits[km] = 0;  // a centre is not a member
                    continue;
                }
                const unsigned* Ld = Lb + d * NT;
                unsigned S = 0u;
                if (hi > t) {
                    S = Ld[i1];
                    if (t > 0) S -= Ld[t - 1];
                    // + the warp totals of warps [w0, w1): vector reads, predicated adds
                    const uint4* wq = reinterpret_cast<const uint4*>(wb + d * kAcgWb);
#pragma unroll
                    for (int v = 0; v < NT / 128; ++v) {
                        const uint4 x = wq[v];
                        const unsigned span = unsigned(w1 - w0);
                        S += unsigned(4 * v + 0 - w0) < span ? x.x : 0u;
                        S += unsigned(4 * v + 1 - w0) < span ? x.y : 0u;
                        S += unsigned(4 * v + 2 - w0) < span ? x.z : 0u;
                        S += unsigned(4 * v + 3 - w0) < span ? x.w : 0u;
                    }
                }
                if (has_head) S += (clipped ? Hc : Hh)[d * NT + hi];
                if (clipped) S += Tt[d * NT + t - 1];
                const bool flat = pf_fc || pf_fm[d];
                const double num =
                    __dsub_rn(double(S), __dmul_rn(__dmul_rn(mn, pf_mc), pf_mm[d]));
                const double den = __dmul_rn(pf_oc, pf_om[d]);
                if (!FUSE && !map) {  // EGS candidate: retained count only (no map, no division)
                    if (flat ? 0.0 < thr : retained_below(num, den, thr)) ++evc;
                    continue;
                }
                if constexpr (!FUSE) {
                    const double val = flat ? 0.0 : dclamp(__ddiv_rn(num, den), -1.0, 1.0);
                    if (map) map[km] = val;
                    if (val < thr) ++evc;
                }
                if constexpr (FUSE) {  // retained count + scan 2 (matcher.cpp:48-78)
                    // R_co = clamp(RN(num / den)) is needed exactly only near a decision:
                    // the FP32 quotient qf (num, den rounded to FP32, times the approximate
                    // reciprocal: relative error < 5 * 2^-24 < 3e-7) decides the retained test (R_co < thr) and the
                    // bound test outside margins that cover that error; the FP64 quotient
                    // is formed only inside them (or near |R_co| = 1, where the bound's
                    // slope in R_co is unbounded).
                    float qf = 0.f;
                    bool fast = !flat;
                    if (fast) {
                        qf = __fmul_rn(float(num), rcp_approx(float(den)));  // rel. error < 3e-7
                        fast = fabsf(qf) < 0.99f;
                    }
                    double val = 0.0;
                    bool have_val = flat;  // flat: R_co = 0 exactly
                    auto exact = [&]() {
                        if (!have_val) {
                            val = dclamp(__ddiv_rn(num, den), -1.0, 1.0);
                            have_val = true;
                        }
                        return val;
                    };
                    bool ret;
                    if (flat) {
                        ret = 0.0 < thr;
                    } else if (fast && qf < float(thr) - 1e-6f) {
                        ret = true;
                    } else if (fast && qf > float(thr) + 1e-6f) {
                        ret = false;
                    } else {
                        ret = exact() < thr;
                    }
                    if (ret) ++evc;
                    uint8_t vis = 2;
                    if (pf_sd) {
                        ++n_keep;  // a seeded group: its members were evaluated already
                    } else {
                        bool elim = grp_test && !pf_fm[d];
                        if (elim) {
                            // FP32 decision with a margin covering the FP32 bound's error
                            // (inputs exactly rounded values in [-1, 1], x = 1 - b^2 formed
                            // before its square root: < 1e-6 with the exact b; with the FP32
                            // quotient for b, |dbound/db| <= 1 + 0.99 / sqrt(1 - 0.99^2) < 8
                            // adds < 8 * 3e-7 < 2.5e-6), the exact FP64 test of k_sec_rows inside it
                            const float b = have_val ? float(val) : qf;
                            const float x = have_val ? float(fma(-val, val, 1.0))
                                                     : fmaf(-qf, qf, 1.0f);
                            const float s = sqrt_approx(fmaxf(x, 0.f));
                            const float f = fmaf(g_af, b, g_saf * s);
                            const float margin = have_val ? 4e-6f : 1e-5f;
                            if (sec_tbf >= f + margin) {
                                elim = true;
                            } else if (sec_tbf < f - margin) {
                                elim = false;
                            } else {
                                const double v = exact();
                                const double xx = dmax(0.0, __dsub_rn(1.0, __dmul_rn(v, v)));
                                elim = sec_tb >= __dadd_rn(__dmul_rn(g_a, v),
                                                           __dmul_rn(pf_sa, __dsqrt_rn(xx)));
                            }
                        }
                        if (elim) {
                            ++n_elim;
                            vis = 1;
                        } else if (pf_fm[d] || sf.tflat) {  // rho 0 without a dot
                            ++n_keep;
                            ++n_flat;
                            fkey = max(fkey, flat_member_key(cr + d - hr, c));
                        } else {
                            ++n_keep;
                            surv |= 1u << d;
                            mark_tile(sf.tf, cr + d - hr, c);
                        }
                    }
                    sf.visits[km] = vis;
                }
            }
        }
        // survivor compaction, one ballot per member row offset (skipped by the whole warp
        // when none of its members survived: the common case)
        if (FUSE && __any_sync(0xffffffffu, surv != 0u)) {
#pragma unroll
            for (int d = 0; d < H; ++d) {
                const bool sv = (surv >> d) & 1u;
                const unsigned ballot = __ballot_sync(0xffffffffu, sv);
                if (!ballot) continue;
                if (list_full) {  // nothing more can be listed: count only
                    surv_local += __popc(ballot);
                    continue;
                }
                unsigned long long basepos = 0;
                if (lane == 0)
                    basepos = atomicAdd(&sf.tally->survivors, (unsigned long long)__popc(ballot));
                basepos = __shfl_sync(0xffffffffu, basepos, 0);
                list_full = basepos + __popc(ballot) >= sf.max_locs;
                if (sv) {
                    const unsigned long long pos = basepos + __popc(ballot & ((1u << lane) - 1));
                    if (pos < sf.max_locs) sf.locs[pos] = make_int2(cr + d - hr, c);
                }
            }
        }
        evc = __reduce_add_sync(0xffffffffu, evc);
        if (lane == 0 && evc) atomicAdd(&cta_cnt, evc);
        if (++ti >= ti1) break;
        const int crn = g.center_row(ti);
        prefetch(ti, crn);
        if (crn - cr == H) {
            advance_both();
        } else {
#pragma unroll 1
            for (int x = cr; x < crn; ++x) {
                lead();
                trail();
            }
        }
        cr = crn;
    }
    __syncthreads();
    if (t == 0 && cta_cnt) atomicAdd(n_r, (unsigned long long)cta_cnt);
    if constexpr (FUSE) {
        const unsigned long long ne = warp_sum((unsigned long long)n_elim);
        const unsigned long long nk = warp_sum((unsigned long long)n_keep);
        const unsigned long long nf = warp_sum((unsigned long long)n_flat);
        fkey = warp_max_u64(fkey);
        if (lane == 0) {  // (surv_local is warp-uniform)
            if (ne) atomicAdd(&sf.tally->eliminated, ne);
            if (nk) atomicAdd(&sf.tally->retained, nk);
            if (surv_local) atomicAdd(&sf.tally->survivors, surv_local);
            if (nf) {
                atomicAdd(&sf.tally->flat_n, nf);
                atomicMax(&sf.tally->flat_key, fkey);
            }
        }
    }
    egs_tail(dec);
}

// Segment order for a count-only candidate (EgsDecide::zorder): segment z covers group rows
// [ti_lo + z*seg, ...) = extent rows [that * h, ...); its density is the earlier candidate's
// retained count over those rows.  One CTA ranks the segments (descending, ties by index).
__global__ void __launch_bounds__(1024)
    k_seg_order(const unsigned* __restrict__ rows, int er, int h, int ti_lo, int seg, int nseg,
                int* __restrict__ order) {
    pdl_wait();
    extern __shared__ unsigned long long segc[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int z = wid; z < nseg; z += blockDim.x >> 5) {  // one warp per segment
        const int r0 = (ti_lo + z * seg) * h, r1 = min((ti_lo + (z + 1) * seg) * h, er);
        unsigned long long c = 0;
        for (int r = r0 + lane; r < r1; r += 32) c += rows[r];
        c = warp_sum(c);
        if (lane == 0) segc[z] = c;
    }
    __syncthreads();
    for (int z = threadIdx.x; z < nseg; z += blockDim.x) {
        const unsigned long long c = segc[z];
        int rank = 0;
        for (int y = 0; y < nseg; ++y) {
            const unsigned long long d = segc[y];
            rank += (d > c || (d == c && y < z)) ? 1 : 0;
        }
        order[rank] = z;
    }
}

// ---- Count-only 5x5 candidate, phase A: the outer column offsets in two passes -----------
//
// A rejected EGS candidate needs only SOME members whose retained count reaches the
// rejection bound (the test is monotone in n_r), and the members at dj = +-2 are retained
// about twice as often as the others (C5: 65 % vs 26-34 %).  Phase A counts exactly those
// members of the regular group columns: k_rco5_s walks them (thread = group column, the ten
// offsets di in [-2, 2] x dj = +-2; per row step and offset one dp4a over the first four
// columns of the block + one IMAD for the fifth, + one masked dp4a for the head when
// n % 5 != 0) and stores their cross sums; k_rco5_cnt evaluates the retained test
// (autocorr.cpp:84-88, egs.cpp:12-25) with the in-kernel rejection of k_acg.  If the
// candidate survives, phase B (k_acg with EgsDecide::outer_done) counts the remaining
// members -- dj in {-1, 0, 1} and the clipped last column -- and decides on its tail.
template <int NT, bool HEAD>
__global__ void __launch_bounds__(NT, NT == 128 ? 3 : 1)
    k_rco5_s(const uint8_t* __restrict__ img, int P, int m, int n, Grid g,
             unsigned* __restrict__ Sout, int G, int seg, int tc_reg, const int* __restrict__ stop) {
    constexpr int NW = NT / 32, NC = 10;
    __shared__ unsigned Lb[2][NC][NT];
    __shared__ unsigned Hb[2][HEAD ? NC : 1][NT];
    __shared__ unsigned Wb[2][NC][NW + 2];
    pdl_wait();
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int k0 = int(blockIdx.x) * G;
    const int ti0 = g.ti_lo + int(blockIdx.y) * seg;
    const int ti1 = min(ti0 + seg, g.ti_hi);
    if ((stop && *reinterpret_cast<const volatile int*>(stop)) || ti0 >= ti1 || k0 >= tc_reg)
        return;
    const int k = k0 + t;
    const int Q = n / 5, R = n - 5 * Q;
    const unsigned hmask = R >= 4 ? 0xffffffffu : ((1u << (8 * R)) - 1u);
    const int sh = (5 * k) & 3;
    const uint8_t* colp = img + ((5 * k) & ~3);
    // one row: A = I(x, 5k+2 .. 5k+6), B(-2) = I(x, 5k .. 5k+4), B(+2) = I(x, 5k+4 .. 5k+8)
    struct Row {
        unsigned aw, ab, mw, mb, pw, pb;
    };
    auto ldrow = [&](int x, unsigned (&w)[3]) {
        const uint8_t* p = colp + size_t(max(x, 0)) * P;
        w[0] = __ldg(reinterpret_cast<const unsigned*>(p));
        w[1] = __ldg(reinterpret_cast<const unsigned*>(p + 4));
        w[2] = __ldg(reinterpret_cast<const unsigned*>(p + 8));
    };
    auto unpack = [&](const unsigned (&w)[3]) {
        Row r;
        const unsigned lo = __funnelshift_r(w[0], w[1], 8 * sh);   // bytes 5k   .. 5k+3
        const unsigned mid = __funnelshift_r(w[1], w[2], 8 * sh);  // bytes 5k+4 .. 5k+7
        const unsigned top = (w[2] >> (8 * sh)) & 0xffu;           // byte  5k+8
        r.mw = lo;
        r.mb = mid & 0xffu;
        r.pw = mid;
        r.pb = top;
        r.aw = __funnelshift_r(lo, mid, 16);  // bytes 5k+2 .. 5k+5
        r.ab = (mid >> 16) & 0xffu;           // byte  5k+6
        return r;
    };
    unsigned VL[NC], VT[NC], HL[HEAD ? NC : 1], HT[HEAD ? NC : 1];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        VL[c] = VT[c] = 0u;
        if constexpr (HEAD) HL[c] = HT[c] = 0u;
    }
    Row LR[4], TR[4];  // rows x-2 .. x+1 at the lead / trail position
    // one row step: A row x (ring[2]), B rows x-2 .. x+2 (ring[0..3], nr)
    auto step = [&](Row (&ring)[4], const Row& nr, unsigned* Vb, unsigned* Hh) {
        const unsigned a = ring[2].aw, ab = ring[2].ab, ah = a & hmask;
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            const Row& b = d < 4 ? ring[d] : nr;
            Vb[2 * d] = __dp4a(a, b.mw, Vb[2 * d]) + ab * b.mb;
            Vb[2 * d + 1] = __dp4a(a, b.pw, Vb[2 * d + 1]) + ab * b.pb;
            if constexpr (HEAD) {
                Hh[2 * d] = __dp4a(ah, b.mw, Hh[2 * d]);
                Hh[2 * d + 1] = __dp4a(ah, b.pw, Hh[2 * d + 1]);
            }
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) ring[i] = ring[i + 1];
        ring[3] = nr;
    };
    int cr = g.center_row(ti0);
    {
        unsigned w[3];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            ldrow(cr - 2 + i, w);
            LR[i] = unpack(w);
            TR[i] = LR[i];
        }
        // warm-up: lead rows [cr, cr + m), loads one step ahead
        unsigned pw[3];
        ldrow(cr + 2, pw);
#pragma unroll 1
        for (int x = cr; x < cr + m; ++x) {
            const Row nr = unpack(pw);
            if (x + 1 < cr + m) ldrow(x + 3, pw);
            step(LR, nr, VL, HL);
        }
    }
    const bool owner = t < G && k < tc_reg;
    const int hi = t + Q;
    const int whi = (hi - 1) >> 5;
    const int cc = 5 * k + 2;
    int par = 0;
#pragma unroll 1
    for (int ti = ti0;;) {
        const bool more = ti + 1 < ti1;
        const int crn = more ? g.center_row(ti + 1) : cr;
        const bool regular = crn - cr == 5;
        unsigned pl[5][3], pt[5][3];
        if (more && regular) {
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                ldrow(cr + m + 2 + i, pl[i]);
                ldrow(cr + 2 + i, pt[i]);
            }
        }
        unsigned x[NC], B[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) x[c] = B[c] = VL[c] - VT[c];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const unsigned u = __shfl_up_sync(0xffffffffu, x[c], o);
                if (lane >= o) x[c] += u;
            }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            Lb[par][c][t] = x[c];
            if constexpr (HEAD) Hb[par][c][t] = HL[c] - HT[c];
            if (lane == 31) Wb[par][c][wid] = x[c];
        }
        __syncthreads();
        if (owner) {
            const int r0 = ti * 5, r1 = min(r0 + 5, g.er) - 1;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const int di = c / 2 - 2, dj = (c & 1) ? 2 : -2;
                const int r = cr + di;
                if (r < r0 || r > r1) continue;
                unsigned S = Lb[par][c][hi - 1] - (x[c] - B[c]);
                const unsigned wa = Wb[par][c][wid], wb2 = Wb[par][c][wid + 1];
                S += wid < whi ? wa : 0u;
                S += wid + 1 < whi ? wb2 : 0u;
                if constexpr (HEAD) S += Hb[par][c][hi];
                // compact layout [extent row][group column][dj = -2, +2]
                Sout[(size_t(r - g.row_lo()) * tc_reg + k) * 2 + (c & 1)] = S;
            }
        }
        par ^= 1;
        if (!more) break;
        if (regular) {
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                step(LR, unpack(pl[i]), VL, HL);
                step(TR, unpack(pt[i]), VT, HT);
            }
        } else {
#pragma unroll 1
            for (int xx = cr; xx < crn; ++xx) {
                unsigned w[3];
                ldrow(xx + m + 2, w);
                step(LR, unpack(w), VL, HL);
                ldrow(xx + 2, w);
                step(TR, unpack(w), VT, HT);
            }
        }
        cr = crn;
        ++ti;
    }
}

// Phase A's retained count of the dj = +-2 members of the regular group columns: CTA =
// extent rows (grid-strided), thread = one group's two outer columns of a row; the CTA's
// count is flushed every row and the rejection test of k_acg replayed on the running
// total (sets *stop: later rows, phase B and the decision see it).
__global__ void __launch_bounds__(256)
    k_rco5_cnt(Grid g, const unsigned* __restrict__ Sin, DevStats st, double mn, double thr,
               int tc_reg, unsigned long long* __restrict__ n_r, int* stop,
               const double* __restrict__ egs_prev, double egs_central, double egs_xi) {
    pdl_wait();
    __shared__ unsigned cta_cnt;
    __shared__ int quit;
    if (threadIdx.x == 0) {
        cta_cnt = 0u;
        quit = *reinterpret_cast<volatile int*>(stop);
    }
    __syncthreads();
    if (quit) return;
    const int lane = threadIdx.x & 31;
    const double prev = *egs_prev;
    const bool can_reject = fabs(prev) <= 1.7976931348623157e308;
    const int r_lo = g.row_lo(), r_hi = g.row_hi();
    for (int r = r_lo + blockIdx.x; r < r_hi; r += gridDim.x) {
        const int ti = g.tile_r(r);
        const int cr = g.center_row(ti);
        const unsigned krow = unsigned(r) * unsigned(g.ec), kcrow = unsigned(cr) * unsigned(g.ec);
        unsigned cnt = 0;
        const uint2* srow = reinterpret_cast<const uint2*>(Sin) + size_t(r - r_lo) * tc_reg;
        for (int tj = threadIdx.x; tj < tc_reg; tj += blockDim.x) {
            const int cc = 5 * tj + 2;
            const unsigned kc = kcrow + unsigned(cc), km = krow + unsigned(cc - 2),
                           kp = krow + unsigned(cc + 2);
            // every load first (independent), then the two retained tests
            const uint2 sv = __ldg(srow + tj);
            const double mc = __ldg(st.mu + kc), oc = __ldg(st.omega + kc);
            const double mm0 = __ldg(st.mu + km), om0 = __ldg(st.omega + km);
            const double mm1 = __ldg(st.mu + kp), om1 = __ldg(st.omega + kp);
            const bool fc = __ldg(st.flat + kc) != 0;
            const bool f0 = fc || __ldg(st.flat + km) != 0, f1 = fc || __ldg(st.flat + kp) != 0;
            const double mnmc = __dmul_rn(mn, mc);
            const double n0 = __dsub_rn(double(sv.x), __dmul_rn(mnmc, mm0));
            const double n1 = __dsub_rn(double(sv.y), __dmul_rn(mnmc, mm1));
            if (f0 ? 0.0 < thr : retained_below(n0, __dmul_rn(oc, om0), thr)) ++cnt;
            if (f1 ? 0.0 < thr : retained_below(n1, __dmul_rn(oc, om1), thr)) ++cnt;
        }
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0 && cnt) atomicAdd(&cta_cnt, cnt);
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned c = cta_cnt;
            cta_cnt = 0u;
            int q = *reinterpret_cast<volatile int*>(stop);
            if (c) {
                const unsigned long long tot = atomicAdd(n_r, (unsigned long long)c) + c;
                const double total = __dadd_rn(__dadd_rn(egs_central, double(tot)), 0.0);
                if (can_reject && !(__dsub_rn(prev, total) > __dmul_rn(egs_xi, prev))) {
                    *reinterpret_cast<volatile int*>(stop) = 1;
                    q = 1;
                }
            }
            quit = q;
        }
        __syncthreads();
        if (quit) return;
    }
}

// launches made by launch_acg_f beside k_acg itself (phase A, k_seg_order): reported by
// autocorr_u8_fused for the context's launch count
thread_local int g_acg_extra = 0;

// Phase A launcher (count-only h = 5 with in-kernel rejection): S raster of the outer
// members, k_rco5_s, k_rco5_cnt.  False: not applicable (phase B then counts everything).
// TMATCH_RCO5=0 disables it.
bool rco5_phase_a(const uint8_t* imgp, int pitch, int m, int n, GridDesc gd, DevStats st,
                  double thr, unsigned long long* n_r, int* stop, const double* egs_prev,
                  double egs_central, double egs_xi, cudaStream_t s) {
    static const bool on = [] {
        const char* e = std::getenv("TMATCH_RCO5");
        return !(e && std::atoi(e) == 0);
    }();
    if (!on || gd.h != 5 || gd.w != 5 || gd.ec < 5) return false;
    const int Q = n / 5, R = n % 5;
    constexpr int NT = 128;
    const int G = NT - Q - (R > 0) + 1;
    if (Q < 1 || Q > 65 || G < 32) return false;
    const int tc_reg = gd.ec % 5 == 0 ? gd.tc : gd.tc - 1;
    if (tc_reg < 1) return false;
    const int ntiles = (tc_reg + G - 1) / G;
    const int rows = gd.ti_hi - gd.ti_lo;
    const int per_wave = std::max(1, (148 * 3) / ntiles);
    int seg = std::max(1, (rows + per_wave - 1) / per_wave);
    seg = std::min(seg, std::max(m / 5 + 1, 40));
    const int nseg = (rows + seg - 1) / seg;
    const Grid g = to_grid(gd);
    // (only worth it with several waves of the count kernel: one wave has no order to use;
    // TMATCH_RCO5_MIN overrides the minimum extent, e.g. 0 for the variant tests)
    static const double min_extent = [] {
        const char* e = std::getenv("TMATCH_RCO5_MIN");
        return e ? std::atof(e) : 3.2e7;
    }();
    if (double(gd.er) * double(gd.ec) < min_extent) return false;
    const size_t cells = size_t(g.row_hi() - g.row_lo()) * tc_reg * 2;
    unsigned* Sbuf = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&Sbuf), cells * sizeof(unsigned), s) != cudaSuccess)
        return false;
    unsigned* S = Sbuf;  // compact [extent row - row_lo][tc_reg][2]
    if (R > 0)
        launch_pdl(k_rco5_s<NT, true>, dim3(ntiles, nseg), dim3(NT), 0, s, imgp, pitch, m, n, g, S,
                   G, seg, tc_reg, static_cast<const int*>(stop));
    else
        launch_pdl(k_rco5_s<NT, false>, dim3(ntiles, nseg), dim3(NT), 0, s, imgp, pitch, m, n, g,
                   S, G, seg, tc_reg, static_cast<const int*>(stop));
    const int blocks = std::min(g.row_hi() - g.row_lo(), 148 * 8);
    launch_pdl(k_rco5_cnt, dim3(blocks), dim3(256), 0, s, g, static_cast<const unsigned*>(S), st,
               double(m) * double(n), thr, tc_reg, n_r, stop, egs_prev, egs_central, egs_xi);
    cudaFreeAsync(Sbuf, s);
    return cudaGetLastError() == cudaSuccess;
}

struct AcgGeom {
    int nt = 0, G = 0, ntiles = 0, seg = 0, nseg = 0, SW = 0, RR = 0;
    size_t smem = 0;
};

constexpr size_t kAcgSmemMax = 200 * 1024;

AcgGeom acg_geom(int m, int n, GridDesc gd, int nt, int resident = 0) {
    AcgGeom a{};
    const int W = gd.w, hr = gd.h / 2;
    if (gd.h != gd.w || (W != 3 && W != 5) || nt > 256 || nt % 32) return a;
    const int Q = n / W, R = n % W;
    int G = nt - (Q + (R > 0)) + 1;
    if (G < 2) return a;
    const bool clipped = gd.ec % W != 0;
    if (clipped) {
        if (gd.tc < 2) return a;
        while (G > 1 && (gd.tc - 1) % G == 0) --G;  // keep the clipped group off thread 0
        if ((gd.tc - 1) % G == 0) return a;
    }
    a.SW = acg_span(nt, gd.h);
    a.RR = m + 2 * gd.h + hr;
    a.smem = 2 * size_t(gd.h) * (4 * size_t(nt) + kAcgWb) * sizeof(unsigned) +
             size_t(a.RR) * a.SW;
    if (a.smem > kAcgSmemMax) return AcgGeom{};
    a.nt = nt;
    a.G = G;
    a.ntiles = (gd.tc + G - 1) / G;
    // Exactly one wave of resident CTAs, segments as short as that needs: every CTA has the
    // same work (equal segments), so the critical path is one segment's m-row warm-up plus
    // its events, and the EGS early rejection reaches all CTAs at the same fraction of work.
    const int rows = gd.ti_hi - gd.ti_lo;
    if (resident <= 0) resident = std::max(1, 1024 / nt);
    const int slots = 148 * resident;
    const int per_wave = std::max(1, slots / std::max(1, gd.w * a.ntiles));
    static const int force_nseg = [] {
        const char* e = std::getenv("TMATCH_ACG_NSEG");
        return e ? std::atoi(e) : 0;
    }();
    // Large images: segments of at most ~96 group rows even when that means several waves
    // -- one wave of whole-image segments leaves too few warps in flight to hide the walk's
    // latency (C5, 265 M locations: fused h = 3 launch 7.66 -> 4.7 ms at 57 segments per
    // tile column, count-only h = 5 4.07 -> 2.4 ms; C2-sized images keep one wave).
    const int by_len = (rows + 95) / 96;
    const int nseg = std::max(1, std::min(force_nseg > 0 ? force_nseg
                                                        : std::max(per_wave, by_len), rows));
    a.seg = std::max(1, (rows + nseg - 1) / nseg);
    a.nseg = std::max(1, (rows + a.seg - 1) / a.seg);
    return a;
}

// CTA size per group size: 256 threads for h = 3 (2 CTAs/SM, 9% halo threads at n = 64);
// 128 for h = 5 (its 25 sliding sums + rings cap 256-thread CTAs at one per SM).
// TMATCH_ACG_THREADS=128|256 forces one size for both (A/B measurements).
int acg_threads(const GridDesc& gd) {
    static int forced = [] {
        const char* e = std::getenv("TMATCH_ACG_THREADS");
        const int v = e ? std::atoi(e) : 0;
        return (v == 128 || v == 256) ? v : 0;
    }();
    if (forced) return forced;
    // h = 3: 256-thread CTAs on C2-sized extents, 128 on large ones (C5: 4.60 -> 4.47 ms;
    // C2: 73 -> 79 us with 128)
    const bool large = double(gd.er) * double(gd.ec) > 3.2e7;
    return gd.h >= 5 || large ? 128 : 256;
}

bool acg_enabled() {
    static bool on = [] {
        const char* e = std::getenv("TMATCH_ACF");
        return !(e && std::strcmp(e, "column") == 0);
    }();
    return on;
}

// tiles [tile_lo, tile_hi) of the launch geometry (tile_hi < 0: to the end)
template <int H, int NT, int NP, bool FUSE>
cudaError_t launch_acg_f(const uint8_t* imgp, int pitch, int q, int m, int n, GridDesc gd,
                         DevStats st, double thr, double* map, unsigned long long* n_r, int* stop,
                         const double* egs_prev, double egs_central, double egs_xi,
                         cudaStream_t s, const EgsDecide& dec, const SecFuse& sf,
                         int tile_lo = 0, int tile_hi = -1) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_acg<H, NT, NP, FUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kAcgSmemMax));
        attr = true;
    }
    const AcgGeom a0 = acg_geom(m, n, gd, NT);
    if (a0.nt == 0) return cudaErrorInvalidValue;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_acg<H, NT, NP, FUSE>, NT,
                                                      a0.smem) != cudaSuccess)
        occ = 0;
    const AcgGeom a = acg_geom(m, n, gd, NT, occ);
    const int t1 = tile_hi < 0 ? a.ntiles : std::min(tile_hi, a.ntiles);
    dim3 grid(gd.w, std::max(0, t1 - tile_lo), a.nseg);
    EgsDecide d = dec;
    if constexpr (H == 5 && !FUSE) {
        if (!map && stop && egs_prev && gd.ti_hi > gd.ti_lo && rco5_phase_a(imgp, pitch, m, n, gd,
                                                                            st, thr, n_r, stop,
                                                                            egs_prev, egs_central,
                                                                            egs_xi, s)) {
            d.outer_done = 1;
            g_acg_extra += 2;
        }
    }
    int* order = nullptr;
    // (only when the launch runs in several waves: one wave has no order to exploit)
    const long long waves = (long long)grid.x * grid.y * grid.z / std::max(1, 148 * occ);
    if (!FUSE && !map && stop && egs_prev && dec.rows_in && a.nseg > 1 && a.nseg <= 4096 &&
        waves >= 3 && gd.ti_hi > gd.ti_lo && grid.y > 0 &&
        cudaMallocAsync(reinterpret_cast<void**>(&order), size_t(a.nseg) * sizeof(int), s) ==
            cudaSuccess) {
        launch_pdl(k_seg_order, dim3(1), dim3(1024), size_t(a.nseg) * 8, s, dec.rows_in, gd.er,
                   gd.h, gd.ti_lo, a.seg, a.nseg, order);
        d.zorder = order;
        ++g_acg_extra;
    }
    if (gd.ti_hi > gd.ti_lo && grid.y > 0)
        launch_pdl(k_acg<H, NT, NP, FUSE>, grid, dim3(NT), a.smem, s, imgp, pitch, q, m, n,
                   to_grid(gd), st, thr, map, n_r, a.G, a.seg, a.RR, stop, egs_prev, egs_central,
                   egs_xi, d, sf, tile_lo);
    if (order) cudaFreeAsync(order, s);
    return cudaGetLastError();
}

int acg_ntiles(int m, int n, GridDesc gd, int nt) { return acg_geom(m, n, gd, nt).ntiles; }

template <int H, int NT, int NP>
cudaError_t launch_acg_nt(const uint8_t* imgp, int pitch, int q, int m, int n, GridDesc gd,
                          DevStats st, double thr, double* map, unsigned long long* n_r, int* stop,
                          const double* egs_prev, double egs_central, double egs_xi,
                          cudaStream_t s, const EgsDecide& dec, const SecFuse& sf,
                          int tile_lo = 0, int tile_hi = -1) {
    if (sf.thr)
        return launch_acg_f<H, NT, NP, true>(imgp, pitch, q, m, n, gd, st, thr, map, n_r, stop,
                                             egs_prev, egs_central, egs_xi, s, dec, sf, tile_lo,
                                             tile_hi);
    return launch_acg_f<H, NT, NP, false>(imgp, pitch, q, m, n, gd, st, thr, map, n_r, stop,
                                          egs_prev, egs_central, egs_xi, s, dec, sf, tile_lo,
                                          tile_hi);
}

// Packed (dp4a) walk for h = 5 (NP = 2 without a clipped group column, else 3); the
// per-column walk for h = 3, where a packed row step saves nothing (W = 3 columns: two
// parts cost as many loads and permutes as three IMADs).  TMATCH_ACG_PACK=0|1 forces the
// per-column / packed walk for both sizes (A/B measurements, parity tests).
int acg_pack(int h) {
    static int forced = [] {
        const char* e = std::getenv("TMATCH_ACG_PACK");
        return e ? (std::atoi(e) ? 1 : 0) : -1;
    }();
    // h = 0: the single-part h = 3 walk (n a multiple of 3), off unless forced on
    // (measured on C5: 4.82 ms vs 4.58 ms for the per-column IMAD walk -- the walk is not
    // what bounds this kernel)
    if (h == 0) return forced >= 0 ? forced : 0;
    return forced >= 0 ? forced : (h >= 5 ? 1 : 0);
}

template <int H, int NT>
cudaError_t launch_acg_np(const uint8_t* imgp, int pitch, int q, int m, int n, GridDesc gd,
                          DevStats st, double thr, double* map, unsigned long long* n_r, int* stop,
                          const double* egs_prev, double egs_central, double egs_xi,
                          cudaStream_t s, const EgsDecide& dec, const SecFuse& sf) {
    if (H == 3 && n % 3 == 0 && acg_pack(0)) {
        // n a multiple of the 3-column groups: every unclipped group column is ONE packed part
        // (one dp4a per row offset and row step instead of three IMADs); the tile holding
        // the clipped last group column (if any) runs its own launch with the cut parts
        // (NP = 3), and carries the EGS decision (stream order: it runs after the first)
        if (gd.ec % gd.w == 0)
            return launch_acg_nt<H, NT, 1>(imgp, pitch, q, m, n, gd, st, thr, map, n_r, stop,
                                           egs_prev, egs_central, egs_xi, s, dec, sf);
        const int nt = acg_ntiles(m, n, gd, NT);
        cudaError_t e = launch_acg_nt<H, NT, 1>(imgp, pitch, q, m, n, gd, st, thr, map, n_r, stop,
                                               egs_prev, egs_central, egs_xi, s, EgsDecide{}, sf,
                                               0, nt - 1);
        if (e != cudaSuccess) return e;
        return launch_acg_nt<H, NT, 3>(imgp, pitch, q, m, n, gd, st, thr, map, n_r, stop,
                                       egs_prev, egs_central, egs_xi, s, dec, sf, nt - 1, nt);
    }
    if (!acg_pack(H))
        return launch_acg_nt<H, NT, 0>(imgp, pitch, q, m, n, gd, st, thr, map, n_r, stop,
                                       egs_prev, egs_central, egs_xi, s, dec, sf);
    if (gd.ec % gd.w == 0)
        return launch_acg_nt<H, NT, 2>(imgp, pitch, q, m, n, gd, st, thr, map, n_r, stop,
                                       egs_prev, egs_central, egs_xi, s, dec, sf);
    return launch_acg_nt<H, NT, 3>(imgp, pitch, q, m, n, gd, st, thr, map, n_r, stop, egs_prev,
                                   egs_central, egs_xi, s, dec, sf);
}

template <int H>
cudaError_t launch_acg(const uint8_t* imgp, int pitch, int q, int m, int n, GridDesc gd,
                       DevStats st, double thr, double* map, unsigned long long* n_r, int* stop,
                       const double* egs_prev, double egs_central, double egs_xi, cudaStream_t s,
                       const EgsDecide& dec, const SecFuse& sf) {
    if (acg_threads(gd) == 128)
        return launch_acg_np<H, 128>(imgp, pitch, q, m, n, gd, st, thr, map, n_r, stop, egs_prev,
                                     egs_central, egs_xi, s, dec, sf);
    return launch_acg_np<H, 256>(imgp, pitch, q, m, n, gd, st, thr, map, n_r, stop, egs_prev,
                                 egs_central, egs_xi, s, dec, sf);
}

// ---- R_co of 3x3 groups in two passes: exact cross sums (k_rco3_s), then the per-member
// epilogue as a streaming pass (k_rco_epi) ---------------------------------------------------
//
// Pass 1, k_rco3_s: thread = one regular group column k (centre column cc = 3k+1) and ALL
// nine offsets (di, dj) of its group, so an image row is loaded once for the nine cross sums
// (the k_acg design runs one CTA per dj).  A row step of the vertical walk needs the bytes
// I(x, 3k .. 3k+4) of one new row: they are packed as three words (the three dj shifts of
// the group's three columns, fourth byte zero) and every offset's column-block sum is ONE
// dp4a per row step (u8 x u8 -> u32, exact; leading and trailing rows in separate
// accumulators since dp4a only adds); with n % 3 = R != 0 a second dp4a per offset sums the
// first R columns ("head").  A's word of row x is B's dj = 0 word of row x, so the two-row
// register ring of B words serves both sides.  Rows come straight from L2/HBM into
// registers one event ahead (no shared-memory ring, no m-row staging).  At each event
// (centre row) one warp scan per offset, warp totals in shared memory, and each thread forms
// its window sums S = whole blocks [t, t+Q) + head of block t+Q -- exactly the autocorr.cpp
// :77-83 cross sums -- and stores the eight members' S (u32, exact: m*n*255^2 < 2^32) in the
// E-sized raster `Sout`.  The clipped last group column (ec % 3 != 0) is not walked here
// (k_rco3_clip sums its few members directly).
//
// Pass 2, k_rco_epi<MODE>: thread = one extent location, rows grid-strided: the FP64
// epilogue of autocorr.cpp:84-88 from S and the window statistics (the same operations as
// k_acg), then the retained count (egs.cpp:12-25), and by MODE: 0 count only, 1 the R_co map,
// 2 scan 2 fused (SecFuse: bound test, visit codes, tallies, survivor list -- the k_acg FUSE
// epilogue).  Every load is coalesced along the row; the EGS decision rides on its tail.


// One member's R_co epilogue (autocorr.cpp:84-88: num = S - (mn*mu_c)*mu_m, den = om_c*om_m,
// R_co = clamp(RN(num/den)), 0 for flat windows) and, by MODE, 0: the retained count
// (egs.cpp:12-25), 1: + the map store, 2: + scan 2 (the k_acg FUSE epilogue: FP32 quotient
// outside the margins, FP64 inside; visit code, tallies).  Returns whether the member survives
// (MODE 2: it goes to the survivor list).
struct RcoTally {
    unsigned evc = 0, n_elim = 0, n_keep = 0, n_flat = 0;
    unsigned long long fkey = 0;
};
struct SecCtx {
    double tb = 0.0;
    float tbf = 0.f;
    bool thr_ok = false;
};
template <int MODE>
__device__ __forceinline__ bool rco_member(RcoTally& T, int r, int c, unsigned k, unsigned S,
                                           double mm, double om, bool fm, double mnmc, double oc,
                                           bool fc, double ra, double sa, bool dg, bool sd,
                                           double thr, const SecCtx& sc, double* map,
                                           const SecFuse& sf) {
    const bool flat = fc || fm;
    const double num = __dsub_rn(double(S), __dmul_rn(mnmc, mm));
    const double den = __dmul_rn(oc, om);
    if constexpr (MODE == 0) {
        if (flat ? 0.0 < thr : retained_below(num, den, thr)) ++T.evc;
        return false;
    } else if constexpr (MODE == 1) {
        const double val = flat ? 0.0 : dclamp(__ddiv_rn(num, den), -1.0, 1.0);
        map[k] = val;
        if (val < thr) ++T.evc;
        return false;
    } else {
        float qf = 0.f;
        bool fast = !flat;
        if (fast) {
            qf = __fmul_rn(float(num), rcp_approx(float(den)));
            fast = fabsf(qf) < 0.99f;
        }
        double val = 0.0;
        bool have_val = flat;
        auto exact = [&]() {
            if (!have_val) {
                val = dclamp(__ddiv_rn(num, den), -1.0, 1.0);
                have_val = true;
            }
            return val;
        };
        bool ret;
        if (flat) {
            ret = 0.0 < thr;
        } else if (fast && qf < float(thr) - 1e-6f) {
            ret = true;
        } else if (fast && qf > float(thr) + 1e-6f) {
            ret = false;
        } else {
            ret = exact() < thr;
        }
        if (ret) ++T.evc;
        uint8_t vis = 2;
        bool survivor = false;
        if (sd) {
            ++T.n_keep;
        } else {
            bool elim = sc.thr_ok && !dg && !sf.tflat && !fm;
            if (elim) {
                const double g_a = dclamp(ra, -1.0, 1.0);
                const float b = have_val ? float(val) : qf;
                const float xf = have_val ? float(fma(-val, val, 1.0)) : fmaf(-qf, qf, 1.0f);
                const float sq = sqrt_approx(fmaxf(xf, 0.f));
                const float f = fmaf(float(g_a), b, float(sa) * sq);
                const float margin = have_val ? 4e-6f : 1e-5f;
                if (sc.tbf >= f + margin) {
                    elim = true;
                } else if (sc.tbf < f - margin) {
                    elim = false;
                } else {
                    const double v = exact();
                    const double xx = dmax(0.0, __dsub_rn(1.0, __dmul_rn(v, v)));
                    elim = sc.tb >= __dadd_rn(__dmul_rn(g_a, v), __dmul_rn(sa, __dsqrt_rn(xx)));
                }
            }
            if (elim) {
                ++T.n_elim;
                vis = 1;
            } else if (fm || sf.tflat) {
                ++T.n_keep;
                ++T.n_flat;
                T.fkey = max(T.fkey, flat_member_key(r, c));
            } else {
                ++T.n_keep;
                survivor = true;
                mark_tile(sf.tf, r, c);
            }
        }
        sf.visits[k] = vis;
        return survivor;
    }
}

// Warp-aggregated append of this thread's survivors (bit i of `bits`: member (rows[i], cols[i]))
template <int NB>
__device__ __forceinline__ void rco_list(unsigned bits, const int* rr, const int* cc, const SecFuse& sf,
                                         bool& list_full, unsigned long long& surv_local) {
    const int lane = threadIdx.x & 31;
    if (!__any_sync(0xffffffffu, bits != 0u)) return;
    const unsigned cnt = __popc(bits);
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
    if (list_full) {
        surv_local += tot;
        return;
    }
    unsigned long long basepos = 0;
    if (lane == 0) basepos = atomicAdd(&sf.tally->survivors, (unsigned long long)tot);
    basepos = __shfl_sync(0xffffffffu, basepos, 0);
    list_full = basepos + tot >= sf.max_locs;
    unsigned long long pos = basepos + (incl - cnt);
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        if ((bits >> i) & 1u) {
            if (pos < sf.max_locs) sf.locs[pos] = make_int2(rr[i], cc[i]);
            ++pos;
        }
    }
}

// Final tallies of an R_co epilogue: warp sums, one atomic per warp (MODE 2 tallies) and per
// CTA (retained count), then the EGS decision on the launch's tail.
template <int MODE>
__device__ __forceinline__ void rco_finish(const RcoTally& T, unsigned long long surv_local,
                                           unsigned long long* n_r, const SecFuse& sf,
                                           const EgsDecide& dec) {
    const int lane = threadIdx.x & 31;
    __shared__ unsigned cta_cnt;
    if (threadIdx.x == 0) cta_cnt = 0u;
    __syncthreads();
    const unsigned evc = __reduce_add_sync(0xffffffffu, T.evc);
    if (lane == 0 && evc) atomicAdd(&cta_cnt, evc);
    if constexpr (MODE == 2) {
        const unsigned long long ne = warp_sum((unsigned long long)T.n_elim);
        const unsigned long long nk = warp_sum((unsigned long long)T.n_keep);
        const unsigned long long nf = warp_sum((unsigned long long)T.n_flat);
        const unsigned long long fk = warp_max_u64(T.fkey);
        if (lane == 0) {
            if (ne) atomicAdd(&sf.tally->eliminated, ne);
            if (nk) atomicAdd(&sf.tally->retained, nk);
            if (surv_local) atomicAdd(&sf.tally->survivors, surv_local);
            if (nf) {
                atomicAdd(&sf.tally->flat_n, nf);
                atomicMax(&sf.tally->flat_key, fk);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && cta_cnt) atomicAdd(n_r, (unsigned long long)cta_cnt);
    egs_tail(dec);
}

template <int NT, bool HEAD>
__global__ void __launch_bounds__(NT, 512 / NT)
    k_rco3_s(const uint8_t* __restrict__ img, int P, int m, int n, Grid g,
             unsigned* __restrict__ Sout, int G, int seg, int tc_reg, const int* __restrict__ stop) {
    constexpr int NW = NT / 32;
    __shared__ unsigned Lb[2][9][NT];               // inclusive warp prefixes of the block sums
    __shared__ unsigned Hb[2][HEAD ? 9 : 1][NT];    // head sums (first R columns of a block)
    __shared__ unsigned Wb[2][9][NW + 2];           // warp totals (+ 2 pad slots)
    pdl_wait();
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int k0 = int(blockIdx.x) * G;
    const int ti0 = g.ti_lo + int(blockIdx.y) * seg;
    const int ti1 = min(ti0 + seg, g.ti_hi);
    if ((stop && *reinterpret_cast<const volatile int*>(stop)) || ti0 >= ti1 || k0 >= tc_reg)
        return;  // uniform, before any barrier
    const int k = k0 + t;
    const int Q = n / 3, R = n - 3 * Q;
    const unsigned hmask = R == 1 ? 0xffu : 0xffffu;  // A bytes of the head columns
    const int sh = (3 * k) & 3;
    const uint8_t* colp = img + ((3 * k) & ~3);
    // B words of one row: bytes I(x, 3k+j+1+dj), j < 3, for dj = -1, 0, +1 (byte 3 zero)
    auto ldrow = [&](int x, unsigned& w0, unsigned& w1) {
        const uint8_t* p = colp + size_t(max(x, 0)) * P;
        w0 = __ldg(reinterpret_cast<const unsigned*>(p));
        w1 = __ldg(reinterpret_cast<const unsigned*>(p + 4));
    };
    auto words = [&](unsigned w0, unsigned w1, unsigned (&o)[3]) {
        const unsigned lo = __funnelshift_r(w0, w1, 8 * sh);
        const unsigned b4 = (w1 >> (8 * sh)) & 0xffu;
        o[0] = lo & 0x00ffffffu;
        o[1] = lo >> 8;
        o[2] = __byte_perm(lo, b4, 0x5432);
    };
    unsigned VL[9], VT[9], HL[HEAD ? 9 : 1], HT[HEAD ? 9 : 1];
#pragma unroll
    for (int c = 0; c < 9; ++c) {
        VL[c] = VT[c] = 0u;
        if constexpr (HEAD) HL[c] = HT[c] = 0u;
    }
    unsigned LW[2][3], TW[2][3];  // B words of rows x-1, x at the lead / trail position
    // one row step: A row x (= ring[1]'s dj = 0 word), B rows x-1, x, x+1 (ring[0], ring[1], nw)
    auto step = [&](unsigned (&ring)[2][3], unsigned w0, unsigned w1, unsigned* Vb,
                    unsigned* Hh) {
        unsigned nw[3];
        words(w0, w1, nw);
        const unsigned a = ring[1][1];
        const unsigned ah = a & hmask;
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            Vb[0 + dj] = __dp4a(a, ring[0][dj], Vb[0 + dj]);
            Vb[3 + dj] = __dp4a(a, ring[1][dj], Vb[3 + dj]);
            Vb[6 + dj] = __dp4a(a, nw[dj], Vb[6 + dj]);
            if constexpr (HEAD) {
                Hh[0 + dj] = __dp4a(ah, ring[0][dj], Hh[0 + dj]);
                Hh[3 + dj] = __dp4a(ah, ring[1][dj], Hh[3 + dj]);
                Hh[6 + dj] = __dp4a(ah, nw[dj], Hh[6 + dj]);
            }
        }
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            ring[0][dj] = ring[1][dj];
            ring[1][dj] = nw[dj];
        }
    };
    int cr = g.center_row(ti0);
    {
        unsigned w0, w1;
        ldrow(cr - 1, w0, w1);
        words(w0, w1, LW[0]);
        ldrow(cr, w0, w1);
        words(w0, w1, LW[1]);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            TW[0][j] = LW[0][j];
            TW[1][j] = LW[1][j];
        }
        // warm-up: the m lead rows [cr, cr + m), loads three rows ahead
        unsigned pw[3][2];
#pragma unroll
        for (int i = 0; i < 3; ++i) ldrow(cr + 1 + i, pw[i][0], pw[i][1]);
        int x = cr;
#pragma unroll 1
        for (; x + 3 <= cr + m; x += 3) {
            unsigned cw[3][2];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                cw[i][0] = pw[i][0];
                cw[i][1] = pw[i][1];
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) ldrow(x + 4 + i, pw[i][0], pw[i][1]);
#pragma unroll
            for (int i = 0; i < 3; ++i) step(LW, cw[i][0], cw[i][1], VL, HL);
        }
#pragma unroll 1
        for (; x < cr + m; ++x) {
            unsigned w0b, w1b;
            ldrow(x + 1, w0b, w1b);
            step(LW, w0b, w1b, VL, HL);
        }
    }
    const bool owner = t < G && k < tc_reg;
    const int hi = t + Q;  // whole blocks [t, hi), head from block hi
    const int whi = (hi - 1) >> 5;
    const int cc = 3 * k + 1;
    int par = 0;
#pragma unroll 1
    for (int ti = ti0;;) {
        // loads of the next transition's rows (lead rows x+1 for x in [cr+m, crn+m), trail
        // rows x+1 for x in [cr, crn)), one event ahead of their use
        const bool more = ti + 1 < ti1;
        const int crn = more ? g.center_row(ti + 1) : cr;
        const bool regular = crn - cr == 3;
        unsigned pl[3][2], pt[3][2];
        if (more && regular) {
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                ldrow(cr + m + 1 + i, pl[i][0], pl[i][1]);
                ldrow(cr + 1 + i, pt[i][0], pt[i][1]);
            }
        }
        unsigned x[9], B[9];
#pragma unroll
        for (int c = 0; c < 9; ++c) x[c] = B[c] = VL[c] - VT[c];  // exact mod 2^32
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
            for (int c = 0; c < 9; ++c) {
                const unsigned u = __shfl_up_sync(0xffffffffu, x[c], o);
                if (lane >= o) x[c] += u;
            }
        }
#pragma unroll
        for (int c = 0; c < 9; ++c) {
            Lb[par][c][t] = x[c];
            if constexpr (HEAD) Hb[par][c][t] = HL[c] - HT[c];
            if (lane == 31) Wb[par][c][wid] = x[c];
        }
        __syncthreads();
        if (owner) {
            const int r0 = ti * 3, r1 = min(r0 + 3, g.er) - 1;
#pragma unroll
            for (int c = 0; c < 9; ++c) {
                if (c == 4) continue;  // the centre
                const int di = c / 3 - 1, dj = c % 3 - 1;
                const int r = cr + di;
                if (r < r0 || r > r1) continue;
                unsigned S = Lb[par][c][hi - 1] - (x[c] - B[c]);
                const unsigned wa = Wb[par][c][wid], wb2 = Wb[par][c][wid + 1];
                S += wid < whi ? wa : 0u;
                S += wid + 1 < whi ? wb2 : 0u;
                if constexpr (HEAD) S += Hb[par][c][hi];
                Sout[unsigned(r) * unsigned(g.ec) + unsigned(cc + dj)] = S;
            }
        }
        par ^= 1;
        if (!more) break;
        if (regular) {
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                step(LW, pl[i][0], pl[i][1], VL, HL);
                step(TW, pt[i][0], pt[i][1], VT, HT);
            }
        } else {  // the clipped last group row: row by row
#pragma unroll 1
            for (int xx = cr; xx < crn; ++xx) {
                unsigned w0, w1;
                ldrow(xx + m + 1, w0, w1);
                step(LW, w0, w1, VL, HL);
                ldrow(xx + 1, w0, w1);
                step(TW, w0, w1, VT, HT);
            }
        }
        cr = crn;
        ++ti;
    }
}

// The clipped last group column (ec % 3 != 0: width wl = 1 or 2, centre column cc = 3*(tc-1),
// members dj in [0, wl), di in {-1, 0, 1}): two small passes instead of a walk.
// k_rco3_clip_rows: one warp per image row x, the row products
//   Rp[c][x] = sum_{b<n} I(x, cc+b) * I(x+di, cc+dj+b)   (c = (di+1)*2 + dj, lanes over b);
// k_rco3_clip_sum: one thread per (group row, member), S = sum_{a<m} Rp[c][cr+a] (exact u32).
__global__ void __launch_bounds__(256)
    k_rco3_clip_rows(const uint8_t* __restrict__ img, int P, int n, int cc, int x0, int nx,
                     unsigned* __restrict__ Rp) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    for (int xi = blockIdx.x * 8 + (threadIdx.x >> 5); xi < nx; xi += gridDim.x * 8) {
        const int x = x0 + xi;
        unsigned acc[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) acc[c] = 0u;
        const uint8_t* ra = img + size_t(x) * P + cc;
        for (int b = lane; b < n; b += 32) {
            const unsigned a = ra[b];
#pragma unroll
            for (int di = -1; di <= 1; ++di) {
                const uint8_t* rb = img + size_t(max(x + di, 0)) * P + cc + b;
                acc[(di + 1) * 2 + 0] += a * unsigned(rb[0]);
                acc[(di + 1) * 2 + 1] += a * unsigned(rb[1]);
            }
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            const unsigned v = warp_sum(acc[c]);
            if (lane == 0) Rp[size_t(c) * nx + xi] = v;
        }
    }
}

__global__ void __launch_bounds__(256)
    k_rco3_clip_sum(const unsigned* __restrict__ Rp, int m, Grid g, int cc, int wl, int x0, int nx,
                    unsigned* __restrict__ Sout, unsigned* __restrict__ Scomp) {
    pdl_wait();
    const int items = (g.ti_hi - g.ti_lo) * 6;
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < items; it += gridDim.x * blockDim.x) {
        const int ti = g.ti_lo + it / 6, c = it % 6;
        const int di = c / 2 - 1, dj = c % 2;
        const int r0 = ti * 3, r1 = min(r0 + 3, g.er) - 1, cr = (r0 + r1) >> 1;
        const int r = cr + di;
        if ((di == 0 && dj == 0) || dj >= wl || r < r0 || r > r1) continue;
        const unsigned* rp = Rp + size_t(c) * nx + (cr - x0);
        unsigned s = 0u;
        for (int a = 0; a < m; ++a) s += rp[a];
        if (Scomp) Scomp[size_t(ti - g.ti_lo) * 6 + c] = s;  // [group row][slot] (fused path)
        else Sout[unsigned(r) * unsigned(g.ec) + unsigned(cc + dj)] = s;
    }
}

template <int MODE, int MINB, int V>
__global__ void __launch_bounds__(256, MINB)
    k_rco_epi(Grid g, const unsigned* __restrict__ Sin, DevStats st, double mn, double thr,
              double* __restrict__ map, unsigned long long* __restrict__ n_r, int* stop,
              EgsDecide dec, SecFuse sf) {
    pdl_wait();
    {
        __shared__ int skip;
        if (threadIdx.x == 0) skip = stop && *reinterpret_cast<volatile int*>(stop);
        __syncthreads();
        if (skip) {
            egs_tail(dec);
            return;
        }
    }
    const int lane = threadIdx.x & 31;
    double sec_tb = 0.0;
    float sec_tbf = 0.f;
    bool thr_ok = false;
    if constexpr (MODE == 2) {
        const double T = *sf.thr;
        sec_tb = dclamp(dmin(T, 1.0), -1.0, 1.0);
        sec_tbf = float(sec_tb);
        thr_ok = T >= -1.0;
    }
    unsigned evc = 0, n_elim = 0, n_keep = 0, n_flat = 0;
    unsigned long long fkey = 0, surv_local = 0;
    bool list_full = false;
    // CTA = one extent row at a time (grid-strided); thread = 4-location chunks of the linear
    // extent index aligned to the strip's base (vector loads of S and the statistics), the
    // row's partial edge chunks masked; the <= 2 groups a chunk touches are gathered once
    const unsigned kb = unsigned(g.row_lo()) * unsigned(g.ec);
    const unsigned ke = unsigned(g.row_hi()) * unsigned(g.ec);
    const int r_lo = g.row_lo(), r_hi = g.row_hi();
    for (int r = r_lo + blockIdx.x; r < r_hi; r += gridDim.x) {
        const unsigned evc_row = evc;  // (EgsDecide::rows_out: this row's retained count)
        const int ti = g.tile_r(r);
        const int cr = g.center_row(ti);
        const unsigned krow = unsigned(r) * unsigned(g.ec);          // first location of the row
        const unsigned kcrow = unsigned(cr) * unsigned(g.ec);
        const unsigned gbase = unsigned(ti) * unsigned(g.tc);
        constexpr int LV = V == 4 ? 2 : 1;
        const unsigned ch0 = (krow - kb) >> LV, ch1 = (krow + g.ec - kb + V - 1) >> LV;
        // whole warps per row (ballots)
        const unsigned nthr = ((ch1 - ch0 + 31) / 32) * 32;
        for (unsigned i = threadIdx.x; i < nthr; i += blockDim.x) {
            const unsigned ch = ch0 + i;
            const bool active = ch < ch1;
            const unsigned k0 = kb + V * (active ? ch : ch0);
            const int c0 = int(k0) - int(krow);  // column of element 0 (may be < 0 at the row start)
            unsigned sv[V];
            double mm[V], om[V];
            uint8_t fm[V];
            if (k0 + V <= ke) {
                if constexpr (V == 4) {
                    const uint4 s4 = *reinterpret_cast<const uint4*>(Sin + k0);
                    const double2 m01 = *reinterpret_cast<const double2*>(st.mu + k0);
                    const double2 m23 = *reinterpret_cast<const double2*>(st.mu + k0 + 2);
                    const double2 o01 = *reinterpret_cast<const double2*>(st.omega + k0);
                    const double2 o23 = *reinterpret_cast<const double2*>(st.omega + k0 + 2);
                    const unsigned f4 = *reinterpret_cast<const unsigned*>(st.flat + k0);
                    sv[0] = s4.x; sv[1] = s4.y; sv[2] = s4.z; sv[3] = s4.w;
                    mm[0] = m01.x; mm[1] = m01.y; mm[2] = m23.x; mm[3] = m23.y;
                    om[0] = o01.x; om[1] = o01.y; om[2] = o23.x; om[3] = o23.y;
#pragma unroll
                    for (int j = 0; j < V; ++j) fm[j] = uint8_t(f4 >> (8 * j));
                } else {
                    const uint2 s2 = *reinterpret_cast<const uint2*>(Sin + k0);
                    const double2 m01 = *reinterpret_cast<const double2*>(st.mu + k0);
                    const double2 o01 = *reinterpret_cast<const double2*>(st.omega + k0);
                    const unsigned f2 = *reinterpret_cast<const unsigned short*>(st.flat + k0);
                    sv[0] = s2.x; sv[1] = s2.y;
                    mm[0] = m01.x; mm[1] = m01.y;
                    om[0] = o01.x; om[1] = o01.y;
                    fm[0] = uint8_t(f2);
                    fm[1] = uint8_t(f2 >> 8);
                }
            } else {
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const unsigned kj = k0 + j < ke ? k0 + j : krow;
                    sv[j] = Sin[kj];
                    mm[j] = st.mu[kj];
                    om[j] = st.omega[kj];
                    fm[j] = st.flat[kj];
                }
            }
            // the (at most two) groups of the chunk: tj0 = first in-row column / 3
            const int cfirst = max(c0, 0);
            const int tj0 = int(__umulhi(unsigned(cfirst), 0xAAAAAAABu) >> 1);
            const int tj1 = min(tj0 + 1, g.tc - 1);
            double mcg[2], ocg[2], rag[2] = {0.0, 0.0}, sag[2] = {0.0, 0.0};
            uint8_t fcg[2], dgg[2] = {0, 0}, sdg[2] = {0, 0};
            int ccg[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int tj = u ? tj1 : tj0;
                ccg[u] = g.center_col(tj);
                const unsigned kc = kcrow + unsigned(ccg[u]);
                mcg[u] = __ldg(st.mu + kc);
                ocg[u] = __ldg(st.omega + kc);
                fcg[u] = __ldg(st.flat + kc);
                if constexpr (MODE == 2) {
                    const unsigned gi = gbase + unsigned(tj);
                    rag[u] = __ldg(sf.rho_c + gi);
                    sag[u] = __ldg(sf.sa_c + gi);
                    dgg[u] = __ldg(sf.deg_c + gi);
                    sdg[u] = sf.seeded ? __ldg(sf.seeded + gi) : uint8_t(0);
                }
            }
            const int cnext = 3 * tj1;  // first column of the second group
            uint8_t vis4[V] = {};
            unsigned surv = 0, mine = 0;  // bit j: element j survives / belongs to this row
            // phase 1 (branch-free over the four elements): membership, R_co's FP64 numerator
            // and denominator, the FP32 quotient
            unsigned memb = 0, flatm = 0, ucol = 0;
            double num[V], den[V];
            float qf[V];
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int c = c0 + j;
                const bool in = active && c >= 0 && c < g.ec;
                const bool u = tj1 != tj0 && c >= cnext;  // (selects: no local-memory arrays)
                const double mcu = u ? mcg[1] : mcg[0], ocu = u ? ocg[1] : ocg[0];
                const bool fl = (u ? fcg[1] : fcg[0]) || fm[j];
                const bool centre = r == cr && c == (u ? ccg[1] : ccg[0]);
                mine |= unsigned(in) << j;
                memb |= unsigned(in && !centre) << j;
                flatm |= unsigned(fl) << j;
                ucol |= unsigned(u) << j;
                num[j] = __dsub_rn(double(sv[j]), __dmul_rn(__dmul_rn(mn, mcu), mm[j]));
                den[j] = __dmul_rn(ocu, om[j]);
                qf[j] = __fmul_rn(float(num[j]), rcp_approx(float(den[j])));
            }
            if constexpr (MODE != 2) {
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    if (!((mine >> j) & 1u)) continue;
                    const unsigned k = k0 + j;
                    const bool flat = (flatm >> j) & 1u;
                    if (!((memb >> j) & 1u)) {
                        if constexpr (MODE == 1) map[k] = 1.0;  // autocorr.cpp:92-93
                        continue;
                    }
                    if constexpr (MODE == 0) {
                        if (flat ? 0.0 < thr : retained_below(num[j], den[j], thr)) ++evc;
                    } else {
                        const double val =
                            flat ? 0.0 : dclamp(__ddiv_rn(num[j], den[j]), -1.0, 1.0);
                        map[k] = val;
                        if (val < thr) ++evc;
                    }
                }
            } else {
                // phase 2: the retained test and the scan-2 bound test of every member from
                // the FP32 quotient with margins covering its error (see the k_acg FUSE
                // epilogue); members whose tests fall inside a margin (or |qf| >= 0.99) take
                // the exact FP64 path of phase 3
                const float thr_lo = float(thr) - 1e-6f, thr_hi = float(thr) + 1e-6f;
                unsigned slow = 0;
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    if (!((memb >> j) & 1u)) continue;
                    const bool flat = (flatm >> j) & 1u, u = (ucol >> j) & 1u;
                    const bool fast = !flat && fabsf(qf[j]) < 0.99f;
                    if (flat) {
                        if (0.0 < thr) ++evc;
                    } else if (fast && qf[j] < thr_lo) {
                        ++evc;
                    } else if (!(fast && qf[j] > thr_hi)) {
                        slow |= 1u << j;
                        continue;
                    }
                    uint8_t vis = 2;
                    if (u ? sdg[1] : sdg[0]) {
                        ++n_keep;
                    } else {
                        bool elim = thr_ok && !sf.tflat && !fm[j] && !(u ? dgg[1] : dgg[0]);
                        if (elim) {
                            // flat: R_co = 0 exactly (margin 4e-6), else qf (margin 1e-5)
                            const float b = flat ? 0.f : qf[j];
                            const float sq = sqrt_approx(fmaxf(fmaf(-b, b, 1.0f), 0.f));
                            const float f = fmaf(float(dclamp(u ? rag[1] : rag[0], -1.0, 1.0)), b,
                                                 float(u ? sag[1] : sag[0]) * sq);
                            const float margin = flat ? 4e-6f : 1e-5f;
                            if (sec_tbf >= f + margin) {
                                elim = true;
                            } else if (sec_tbf < f - margin) {
                                elim = false;
                            } else {
                                slow |= 1u << j;
                                continue;
                            }
                        }
                        if (elim) {
                            ++n_elim;
                            vis = 1;
                        } else if (fm[j] || sf.tflat) {
                            ++n_keep;
                            ++n_flat;
                            fkey = max(fkey, flat_member_key(r, c0 + j));
                        } else {
                            ++n_keep;
                            surv |= 1u << j;
                            mark_tile(sf.tf, r, c0 + j);
                        }
                    }
                    vis4[j] = vis;
                }
                // phase 3 (rare): the exact R_co = clamp(RN(num / den)) decides both tests
                // (k_sec_rows' FP64 bound test inside the FP32 margin)
                if (slow) {
#pragma unroll 1
                    for (int j = 0; j < V; ++j) {
                        if (!((slow >> j) & 1u)) continue;
                        const bool flat = (flatm >> j) & 1u, u = (ucol >> j) & 1u;
                        double nj = num[0], dj2 = den[0];
                        bool fmj = fm[0];
#pragma unroll
                        for (int i = 1; i < V; ++i)
                            if (j == i) {
                                nj = num[i];
                                dj2 = den[i];
                                fmj = fm[i];
                            }
                        const double val = flat ? 0.0 : dclamp(__ddiv_rn(nj, dj2), -1.0, 1.0);
                        if (val < thr) ++evc;
                        uint8_t vis = 2;
                        if (u ? sdg[1] : sdg[0]) {
                            ++n_keep;
                        } else {
                            bool elim = thr_ok && !sf.tflat && !fmj && !(u ? dgg[1] : dgg[0]);
                            if (elim) {
                                const double g_a = dclamp(u ? rag[1] : rag[0], -1.0, 1.0);
                                const double g_sa = u ? sag[1] : sag[0];
                                const float b = float(val);
                                const float xf = float(fma(-val, val, 1.0));
                                const float sq = sqrt_approx(fmaxf(xf, 0.f));
                                const float f = fmaf(float(g_a), b, float(g_sa) * sq);
                                if (sec_tbf >= f + 4e-6f) {
                                    elim = true;
                                } else if (sec_tbf < f - 4e-6f) {
                                    elim = false;
                                } else {
                                    const double xx = dmax(0.0, __dsub_rn(1.0, __dmul_rn(val, val)));
                                    elim = sec_tb >= __dadd_rn(__dmul_rn(g_a, val),
                                                               __dmul_rn(g_sa, __dsqrt_rn(xx)));
                                }
                            }
                            if (elim) {
                                ++n_elim;
                                vis = 1;
                            } else if (fmj || sf.tflat) {
                                ++n_keep;
                                ++n_flat;
                                fkey = max(fkey, flat_member_key(r, c0 + j));
                            } else {
                                ++n_keep;
                                surv |= 1u << j;
                                mark_tile(sf.tf, r, c0 + j);
                            }
                        }
#pragma unroll
                        for (int i = 0; i < V; ++i)
                            if (j == i) vis4[i] = vis;
                    }
                }
            }
            if constexpr (MODE == 2) {
                if (mine == (1u << V) - 1u) {
                    if constexpr (V == 4)
                        *reinterpret_cast<unsigned*>(sf.visits + k0) =
                            unsigned(vis4[0]) | (unsigned(vis4[1]) << 8) |
                            (unsigned(vis4[2]) << 16) | (unsigned(vis4[3]) << 24);
                    else
                        *reinterpret_cast<unsigned short*>(sf.visits + k0) =
                            (unsigned short)(unsigned(vis4[0]) | (unsigned(vis4[1]) << 8));
                } else {
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        if ((mine >> j) & 1u) sf.visits[k0 + j] = vis4[j];
                }
                if (__any_sync(0xffffffffu, surv != 0u)) {
                    const unsigned cnt = __popc(surv);
                    unsigned incl = cnt;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += v;
                    }
                    const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
                    if (list_full) {
                        surv_local += tot;
                    } else {
                        unsigned long long basepos = 0;
                        if (lane == 0)
                            basepos = atomicAdd(&sf.tally->survivors, (unsigned long long)tot);
                        basepos = __shfl_sync(0xffffffffu, basepos, 0);
                        list_full = basepos + tot >= sf.max_locs;
                        unsigned long long pos = basepos + (incl - cnt);
#pragma unroll
                        for (int j = 0; j < V; ++j) {
                            if ((surv >> j) & 1u) {
                                if (pos < sf.max_locs) sf.locs[pos] = make_int2(r, c0 + j);
                                ++pos;
                            }
                        }
                    }
                }
            }
        }
        if (dec.rows_out) {  // CTA-uniform
            const unsigned d = __reduce_add_sync(0xffffffffu, evc - evc_row);
            if (lane == 0 && d) atomicAdd(dec.rows_out + r, d);
        }
    }
    __shared__ unsigned cta_cnt;
    if (threadIdx.x == 0) cta_cnt = 0u;
    __syncthreads();
    evc = __reduce_add_sync(0xffffffffu, evc);
    if (lane == 0 && evc) atomicAdd(&cta_cnt, evc);
    if constexpr (MODE == 2) {
        const unsigned long long ne = warp_sum((unsigned long long)n_elim);
        const unsigned long long nk = warp_sum((unsigned long long)n_keep);
        const unsigned long long nf = warp_sum((unsigned long long)n_flat);
        fkey = warp_max_u64(fkey);
        if (lane == 0) {
            if (ne) atomicAdd(&sf.tally->eliminated, ne);
            if (nk) atomicAdd(&sf.tally->retained, nk);
            if (surv_local) atomicAdd(&sf.tally->survivors, surv_local);
            if (nf) {
                atomicAdd(&sf.tally->flat_n, nf);
                atomicMax(&sf.tally->flat_key, fkey);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && cta_cnt) atomicAdd(n_r, (unsigned long long)cta_cnt);
    egs_tail(dec);
}

// ---- Fused variant: the walk of k_rco3_s with the member epilogue in the same CTA --------
//
// k_rco3_f<NT, HEAD, MODE>: the walk and event scan of k_rco3_s, but instead of storing the
// eight members' cross sums each thread evaluates them at once (rco_member: R_co, retained
// count, map / scan 2).  The window statistics of the event's three extent rows over the
// tile's columns are staged into shared memory by cp.async two events ahead (three buffers,
// issued after the event barrier so no buffer is overwritten while read), so no E-sized S
// round trip and no gathers: the group centre's statistics are in the staged middle row.
// The clipped last group column goes through k_rco3_clip_* + k_rco3_clip_epi.
constexpr int kRcoStages = 3;
// (even / multiple of 4 so every staged row stays 16- / 4-byte aligned for cp.async)
__host__ __device__ constexpr int rco_sc(int G) { return (3 * G + 3) & ~1; }    // doubles per row
__host__ __device__ constexpr int rco_scf(int G) { return (3 * G + 11) & ~3; }  // flag bytes per row
__host__ __device__ constexpr size_t rco_stage_bytes(int G) {
    return size_t(3) * rco_sc(G) * 16 + ((size_t(3) * rco_scf(G) + 15) & ~size_t(15));
}

template <int NT, bool HEAD, int MODE>
__global__ void __launch_bounds__(NT, NT == 128 ? 3 : 1)
    k_rco3_f(const uint8_t* __restrict__ img, int P, int m, int n, Grid g, DevStats st, double mn,
             double thr, double* __restrict__ map, unsigned long long* __restrict__ n_r, int G,
             int seg, int tc_reg, int* stop, EgsDecide dec, SecFuse sf) {
    constexpr int NW = NT / 32;
    __shared__ unsigned Lb[2][9][NT];
    __shared__ unsigned Hb[2][HEAD ? 9 : 1][NT];
    __shared__ unsigned Wb[2][9][NW + 2];
    extern __shared__ __align__(16) unsigned char rco_stage[];
    pdl_wait();
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int k0 = int(blockIdx.x) * G;
    const int ti0 = g.ti_lo + int(blockIdx.y) * seg;
    const int ti1 = min(ti0 + seg, g.ti_hi);
    {
        __shared__ int skip;
        if (t == 0)
            skip = (stop && *reinterpret_cast<volatile int*>(stop)) || ti0 >= ti1 || k0 >= tc_reg;
        __syncthreads();
        if (skip) {
            egs_tail(dec);
            return;
        }
    }
    SecCtx sc;
    if constexpr (MODE == 2) {
        const double T = *sf.thr;
        sc.tb = dclamp(dmin(T, 1.0), -1.0, 1.0);
        sc.tbf = float(sc.tb);
        sc.thr_ok = T >= -1.0;
    }
    RcoTally tal;
    bool list_full = false;
    unsigned long long surv_local = 0;
    const int k = k0 + t;
    const int Q = n / 3, R = n - 3 * Q;
    const unsigned hmask = R == 1 ? 0xffu : 0xffffu;
    const int sh = (3 * k) & 3;
    const uint8_t* colp = img + ((3 * k) & ~3);
    const int cbase = 3 * k0;                                 // first staged column
    const int ncols = min(3 * G, 3 * tc_reg - cbase);         // staged columns
    const unsigned strip_end = unsigned(g.row_hi()) * unsigned(g.ec);
    // ---- window statistics of the event's rows -> stage buffer (cp.async, private copies)
    auto stage_of = [&](int b) { return rco_stage + size_t(b) * rco_stage_bytes(G); };
    auto stage_stats = [&](int ti, int b) {
        unsigned char* sb = stage_of(b);
        double* smu = reinterpret_cast<double*>(sb);
        double* som = smu + 3 * rco_sc(G);
        uint8_t* sfl = reinterpret_cast<uint8_t*>(som + 3 * rco_sc(G));
        const int r0 = ti * 3, r1 = min(r0 + 3, g.er) - 1, crr = (r0 + r1) >> 1;
#pragma unroll 1
        for (int rr = 0; rr < 3; ++rr) {
            const int r = crr - 1 + rr;
            if (r < r0 || r > r1) continue;
            const unsigned base = unsigned(r) * unsigned(g.ec) + unsigned(cbase);
            const unsigned lo2 = base & ~1u, lo4 = base & ~3u;
            const unsigned end = base + unsigned(ncols);
            const int n2 = int((end - lo2 + 1) >> 1), n4 = int((end - lo4 + 3) >> 2);
            for (int i = t; i < n2; i += NT) {
                const unsigned e0 = lo2 + 2 * i;
                double* dm = smu + rr * rco_sc(G) + 2 * i;
                double* dq = som + rr * rco_sc(G) + 2 * i;
                if (e0 + 2 <= strip_end) {
                    cp_async16(dm, st.mu + e0);
                    cp_async16(dq, st.omega + e0);
                } else {
                    dm[0] = st.mu[e0];
                    dq[0] = st.omega[e0];
                }
            }
            for (int i = t; i < n4; i += NT) {
                const unsigned e0 = lo4 + 4 * i;
                uint8_t* df = sfl + rr * rco_scf(G) + 4 * i;
                if (e0 + 4 <= strip_end) {
                    cp_async4(df, st.flat + e0);
                } else {
                    for (unsigned e = e0; e < strip_end; ++e) df[e - e0] = st.flat[e];
                }
            }
        }
        cp_async_commit();
    };
    auto ldrow = [&](int x, unsigned& w0, unsigned& w1) {
        const uint8_t* p = colp + size_t(max(x, 0)) * P;
        w0 = __ldg(reinterpret_cast<const unsigned*>(p));
        w1 = __ldg(reinterpret_cast<const unsigned*>(p + 4));
    };
    auto words = [&](unsigned w0, unsigned w1, unsigned (&o)[3]) {
        const unsigned lo = __funnelshift_r(w0, w1, 8 * sh);
        const unsigned b4 = (w1 >> (8 * sh)) & 0xffu;
        o[0] = lo & 0x00ffffffu;
        o[1] = lo >> 8;
        o[2] = __byte_perm(lo, b4, 0x5432);
    };
    unsigned VL[9], VT[9], HL[HEAD ? 9 : 1], HT[HEAD ? 9 : 1];
#pragma unroll
    for (int c = 0; c < 9; ++c) {
        VL[c] = VT[c] = 0u;
        if constexpr (HEAD) HL[c] = HT[c] = 0u;
    }
    unsigned LW[2][3], TW[2][3];
    auto step = [&](unsigned (&ring)[2][3], unsigned w0, unsigned w1, unsigned* Vb,
                    unsigned* Hh) {
        unsigned nw[3];
        words(w0, w1, nw);
        const unsigned a = ring[1][1];
        const unsigned ah = a & hmask;
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            Vb[0 + dj] = __dp4a(a, ring[0][dj], Vb[0 + dj]);
            Vb[3 + dj] = __dp4a(a, ring[1][dj], Vb[3 + dj]);
            Vb[6 + dj] = __dp4a(a, nw[dj], Vb[6 + dj]);
            if constexpr (HEAD) {
                Hh[0 + dj] = __dp4a(ah, ring[0][dj], Hh[0 + dj]);
                Hh[3 + dj] = __dp4a(ah, ring[1][dj], Hh[3 + dj]);
                Hh[6 + dj] = __dp4a(ah, nw[dj], Hh[6 + dj]);
            }
        }
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            ring[0][dj] = ring[1][dj];
            ring[1][dj] = nw[dj];
        }
    };
    // the first two events' statistics in flight during the warm-up
    stage_stats(ti0, 0);
    if (ti0 + 1 < ti1) stage_stats(ti0 + 1, 1);
    else cp_async_commit();
    int cr = g.center_row(ti0);
    {
        unsigned w0, w1;
        ldrow(cr - 1, w0, w1);
        words(w0, w1, LW[0]);
        ldrow(cr, w0, w1);
        words(w0, w1, LW[1]);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            TW[0][j] = LW[0][j];
            TW[1][j] = LW[1][j];
        }
        unsigned pw[3][2];
#pragma unroll
        for (int i = 0; i < 3; ++i) ldrow(cr + 1 + i, pw[i][0], pw[i][1]);
        int x = cr;
#pragma unroll 1
        for (; x + 3 <= cr + m; x += 3) {
            unsigned cw[3][2];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                cw[i][0] = pw[i][0];
                cw[i][1] = pw[i][1];
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) ldrow(x + 4 + i, pw[i][0], pw[i][1]);
#pragma unroll
            for (int i = 0; i < 3; ++i) step(LW, cw[i][0], cw[i][1], VL, HL);
        }
#pragma unroll 1
        for (; x < cr + m; ++x) {
            unsigned w0b, w1b;
            ldrow(x + 1, w0b, w1b);
            step(LW, w0b, w1b, VL, HL);
        }
    }
    const bool owner = t < G && k < tc_reg;
    const int hi = t + Q;
    const int whi = (hi - 1) >> 5;
    const int cc = 3 * k + 1;
    int par = 0, sbuf = 0;
#pragma unroll 1
    for (int ti = ti0;;) {
        const bool more = ti + 1 < ti1;
        const int crn = more ? g.center_row(ti + 1) : cr;
        const bool regular = crn - cr == 3;
        unsigned pl[3][2], pt[3][2];
        if (more && regular) {
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                ldrow(cr + m + 1 + i, pl[i][0], pl[i][1]);
                ldrow(cr + 1 + i, pt[i][0], pt[i][1]);
            }
        }
        // this event's group record (MODE 2)
        double ra = 0.0, sa = 0.0;
        bool dg = false, sd = false;
        if constexpr (MODE == 2) {
            if (owner) {
                const size_t gi = size_t(ti) * g.tc + k;
                ra = __ldg(sf.rho_c + gi);
                sa = __ldg(sf.sa_c + gi);
                dg = __ldg(sf.deg_c + gi);
                sd = sf.seeded ? __ldg(sf.seeded + gi) != 0 : false;
            }
        }
        unsigned x[9], B[9];
#pragma unroll
        for (int c = 0; c < 9; ++c) x[c] = B[c] = VL[c] - VT[c];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
            for (int c = 0; c < 9; ++c) {
                const unsigned u = __shfl_up_sync(0xffffffffu, x[c], o);
                if (lane >= o) x[c] += u;
            }
        }
#pragma unroll
        for (int c = 0; c < 9; ++c) {
            Lb[par][c][t] = x[c];
            if constexpr (HEAD) Hb[par][c][t] = HL[c] - HT[c];
            if (lane == 31) Wb[par][c][wid] = x[c];
        }
        cp_async_wait_1();  // this event's statistics (this thread's copies)
        __syncthreads();    // ... everyone's, and the published sums
        // two events ahead into the buffer read by the event before this one
        if (ti + 2 < ti1) stage_stats(ti + 2, sbuf == 0 ? 2 : sbuf - 1);
        else cp_async_commit();
        unsigned sbits = 0;
        int srr[8], scc[8];
        unsigned evr[3] = {0u, 0u, 0u};  // retained per member row (EgsDecide::rows_out)
        if (owner) {
            const unsigned char* sb = stage_of(sbuf);
            const double* smu = reinterpret_cast<const double*>(sb);
            const double* som = smu + 3 * rco_sc(G);
            const uint8_t* sfl = reinterpret_cast<const uint8_t*>(som + 3 * rco_sc(G));
            const int r0 = ti * 3, r1 = min(r0 + 3, g.er) - 1;
            // centre statistics: middle staged row
            const unsigned cbk = unsigned(cr) * unsigned(g.ec) + unsigned(cbase);
            const int cci = cc - cbase;
            const double mc = smu[rco_sc(G) + int(cbk & 1u) + cci];
            const double oc = som[rco_sc(G) + int(cbk & 1u) + cci];
            const bool fc = sfl[rco_scf(G) + int(cbk & 3u) + cci];
            const double mnmc = __dmul_rn(mn, mc);
            const unsigned kcen = unsigned(cr) * unsigned(g.ec) + unsigned(cc);
            if constexpr (MODE == 1) map[kcen] = 1.0;  // autocorr.cpp:92-93
            if constexpr (MODE == 2) sf.visits[kcen] = 0;
#pragma unroll
            for (int c = 0; c < 9; ++c) {
                if (c == 4) continue;
                const int di = c / 3 - 1, dj = c % 3 - 1;
                const int r = cr + di;
                if (r < r0 || r > r1) continue;
                unsigned S = Lb[par][c][hi - 1] - (x[c] - B[c]);
                const unsigned wa = Wb[par][c][wid], wb2 = Wb[par][c][wid + 1];
                S += wid < whi ? wa : 0u;
                S += wid + 1 < whi ? wb2 : 0u;
                if constexpr (HEAD) S += Hb[par][c][hi];
                const int col = cc + dj;
                const unsigned kk = unsigned(r) * unsigned(g.ec) + unsigned(col);
                const unsigned rb = unsigned(r) * unsigned(g.ec) + unsigned(cbase);
                const int rr = di + 1, ci = col - cbase;
                const double mm = smu[rr * rco_sc(G) + int(rb & 1u) + ci];
                const double om = som[rr * rco_sc(G) + int(rb & 1u) + ci];
                const bool fm = sfl[rr * rco_scf(G) + int(rb & 3u) + ci];
                const unsigned e0 = tal.evc;
                const bool sv = rco_member<MODE>(tal, r, col, kk, S, mm, om, fm, mnmc, oc, fc, ra,
                                                 sa, dg, sd, thr, sc, map, sf);
                evr[rr] += tal.evc - e0;
                if constexpr (MODE == 2) {
                    const int slot = c < 4 ? c : c - 1;
                    sbits |= unsigned(sv) << slot;
                    srr[slot] = r;
                    scc[slot] = col;
                }
            }
        }
        if constexpr (MODE == 2) rco_list<8>(sbits, srr, scc, sf, list_full, surv_local);
        if (dec.rows_out) {  // CTA-uniform
#pragma unroll
            for (int rr = 0; rr < 3; ++rr) {
                const unsigned d = __reduce_add_sync(0xffffffffu, evr[rr]);
                if (lane == 0 && d) atomicAdd(dec.rows_out + (cr - 1 + rr), d);
            }
        }
        par ^= 1;
        sbuf = sbuf == 2 ? 0 : sbuf + 1;
        if (!more) break;
        if (regular) {
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                step(LW, pl[i][0], pl[i][1], VL, HL);
                step(TW, pt[i][0], pt[i][1], VT, HT);
            }
        } else {
#pragma unroll 1
            for (int xx = cr; xx < crn; ++xx) {
                unsigned w0, w1;
                ldrow(xx + m + 1, w0, w1);
                step(LW, w0, w1, VL, HL);
                ldrow(xx + 1, w0, w1);
                step(TW, w0, w1, VT, HT);
            }
        }
        cr = crn;
        ++ti;
    }
    cp_async_wait_all();
    rco_finish<MODE>(tal, surv_local, n_r, sf, dec);
}

// The clipped last group column's epilogue (its members' S from k_rco3_clip_sum, compact
// [group row][6] layout): one thread per (group row, member slot), rco_member as above.
template <int MODE>
__global__ void __launch_bounds__(256)
    k_rco3_clip_epi(Grid g, const unsigned* __restrict__ Sc, DevStats st, double mn, double thr,
                    double* __restrict__ map, unsigned long long* __restrict__ n_r, EgsDecide dec,
                    SecFuse sf) {
    pdl_wait();
    SecCtx sc;
    if constexpr (MODE == 2) {
        const double T = *sf.thr;
        sc.tb = dclamp(dmin(T, 1.0), -1.0, 1.0);
        sc.tbf = float(sc.tb);
        sc.thr_ok = T >= -1.0;
    }
    RcoTally tal;
    bool list_full = false;
    unsigned long long surv_local = 0;
    const int kc = g.tc - 1, gc0 = 3 * kc, gc1 = g.ec - 1, ccol = (gc0 + gc1) >> 1;
    const int wl = gc1 - gc0 + 1;
    const int items = (g.ti_hi - g.ti_lo) * 6;
    const int nit = ((items + 31) / 32) * 32;
    for (int it = blockIdx.x * blockDim.x + threadIdx.x; it - int(threadIdx.x & 31) < nit;
         it += gridDim.x * blockDim.x) {
        if (it - int(threadIdx.x & 31) >= items) break;  // warp-uniform
        bool sv = false;
        int r = 0, c = 0;
        if (it < items) {
            const int ti = g.ti_lo + it / 6, slot = it % 6;
            const int di = slot / 2 - 1, dj = slot % 2;
            const int r0 = ti * 3, r1 = min(r0 + 3, g.er) - 1, cr = (r0 + r1) >> 1;
            r = cr + di;
            c = ccol + dj;
            if (dj < wl && r >= r0 && r <= r1) {
                const unsigned k = unsigned(r) * unsigned(g.ec) + unsigned(c);
                if (di == 0 && dj == 0) {
                    if constexpr (MODE == 1) map[k] = 1.0;
                    if constexpr (MODE == 2) sf.visits[k] = 0;
                } else {
                    const unsigned kcn = unsigned(cr) * unsigned(g.ec) + unsigned(ccol);
                    const size_t gi = size_t(ti) * g.tc + kc;
                    const double mnmc = __dmul_rn(mn, st.mu[kcn]);
                    double ra = 0.0, sa = 0.0;
                    bool dg = false, sd = false;
                    if constexpr (MODE == 2) {
                        ra = sf.rho_c[gi];
                        sa = sf.sa_c[gi];
                        dg = sf.deg_c[gi];
                        sd = sf.seeded ? sf.seeded[gi] != 0 : false;
                    }
                    sv = rco_member<MODE>(tal, r, c, k, Sc[size_t(ti - g.ti_lo) * 6 + slot],
                                          st.mu[k], st.omega[k], st.flat[k] != 0, mnmc,
                                          st.omega[kcn], st.flat[kcn] != 0, ra, sa, dg, sd, thr,
                                          sc, map, sf);
                }
            }
        }
        if constexpr (MODE == 2) rco_list<1>(unsigned(sv), &r, &c, sf, list_full, surv_local);
    }
    rco_finish<MODE>(tal, surv_local, n_r, sf, dec);
}

// TMATCH_RCO3_FUSED=1 selects the single-kernel form (k_rco3_f) for A/B runs.
// (measured on C5: 4.13 ms fused vs 2.79 ms for the two kernels -- the fused CTA runs 12
// warps per SM at 168 registers and its eight serial member epilogues per event leave the
// SM latency-bound; the streaming epilogue runs at twice the occupancy)
bool rco3_fused() {
    static bool on = [] {
        const char* e = std::getenv("TMATCH_RCO3_FUSED");
        return e ? std::atoi(e) != 0 : false;
    }();
    return on;
}

// k_rco_epg<MODE, MINB>: pass 2 of the h = 3 R_co with thread = one group's 3-column segment
// of an extent row (CTA = extent rows, grid-strided): the three locations share the group's
// centre statistics and record, so nothing is selected per location; S, mu, omega and the
// flags of the segment are three coalesced scalar loads each (the warp reads 96 consecutive
// locations).  Same decisions as k_rco_epi (rco_member).
template <int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_rco_epg(Grid g, const unsigned* __restrict__ Sin, DevStats st, double mn, double thr,
              double* __restrict__ map, unsigned long long* __restrict__ n_r, int* stop,
              EgsDecide dec, SecFuse sf) {
    pdl_wait();
    {
        __shared__ int skip;
        if (threadIdx.x == 0) skip = stop && *reinterpret_cast<volatile int*>(stop);
        __syncthreads();
        if (skip) {
            egs_tail(dec);
            return;
        }
    }
    const int lane = threadIdx.x & 31;
    SecCtx sc;
    if constexpr (MODE == 2) {
        const double T = *sf.thr;
        sc.tb = dclamp(dmin(T, 1.0), -1.0, 1.0);
        sc.tbf = float(sc.tb);
        sc.thr_ok = T >= -1.0;
    }
    RcoTally tal;
    bool list_full = false;
    unsigned long long surv_local = 0;
    const int r_lo = g.row_lo(), r_hi = g.row_hi();
    const int ntj = ((g.tc + 31) / 32) * 32;  // whole warps per row (ballots)
    for (int r = r_lo + blockIdx.x; r < r_hi; r += gridDim.x) {
        const unsigned evc_row = tal.evc;
        const int ti = g.tile_r(r);
        const int cr = g.center_row(ti);
        const unsigned krow = unsigned(r) * unsigned(g.ec), kcrow = unsigned(cr) * unsigned(g.ec);
        const unsigned gbase = unsigned(ti) * unsigned(g.tc);
        for (int tj = threadIdx.x; tj < ntj; tj += blockDim.x) {
            const bool active = tj < g.tc;
            const int tq = active ? tj : 0;
            const int c0 = 3 * tq, c1 = min(c0 + 3, g.ec) - 1, ccol = (c0 + c1) >> 1;
            const int nc = c1 - c0 + 1;
            unsigned sv[3];
            double mm[3], om[3];
            bool fm[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const unsigned k = krow + unsigned(c0 + min(j, nc - 1));
                sv[j] = __ldg(Sin + k);
                mm[j] = __ldg(st.mu + k);
                om[j] = __ldg(st.omega + k);
                fm[j] = __ldg(st.flat + k) != 0;
            }
            const unsigned kc = kcrow + unsigned(ccol);
            const double mc = __ldg(st.mu + kc), oc = __ldg(st.omega + kc);
            const bool fc = __ldg(st.flat + kc) != 0;
            double ra = 0.0, sa = 0.0;
            bool dg = false, sd = false;
            if constexpr (MODE == 2) {
                const unsigned gi = gbase + unsigned(tq);
                ra = __ldg(sf.rho_c + gi);
                sa = __ldg(sf.sa_c + gi);
                dg = __ldg(sf.deg_c + gi) != 0;
                sd = sf.seeded ? __ldg(sf.seeded + gi) != 0 : false;
            }
            const double mnmc = __dmul_rn(mn, mc);
            unsigned sbits = 0;
            int srr[3], scc[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int c = c0 + j;
                srr[j] = r;
                scc[j] = c;
                if (!active || j >= nc) continue;
                const unsigned k = krow + unsigned(c);
                if (r == cr && c == ccol) {  // the group's centre (autocorr.cpp:92-93)
                    if constexpr (MODE == 1) map[k] = 1.0;
                    if constexpr (MODE == 2) sf.visits[k] = 0;
                    continue;
                }
                const bool s = rco_member<MODE>(tal, r, c, k, sv[j], mm[j], om[j], fm[j], mnmc, oc,
                                                fc, ra, sa, dg, sd, thr, sc, map, sf);
                sbits |= unsigned(s) << j;
            }
            if constexpr (MODE == 2) rco_list<3>(sbits, srr, scc, sf, list_full, surv_local);
        }
        if (dec.rows_out) {  // CTA-uniform
            const unsigned d = __reduce_add_sync(0xffffffffu, tal.evc - evc_row);
            if (lane == 0 && d) atomicAdd(dec.rows_out + r, d);
        }
    }
    rco_finish<MODE>(tal, surv_local, n_r, sf, dec);
}

// k_rco_epg9<MODE, MINB>: pass 2 with thread = one whole 3x3 group (CTA = group rows,
// grid-strided; threads over the group columns): its three rows' S / mu / omega / flags are
// coalesced loads along each row, the centre's statistics come from the middle row's own
// loads (no gather of the centre row by the rows above and below it) and the group record is
// read once for nine locations.  Same decisions as k_rco_epg (rco_member).
template <int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_rco_epg9(Grid g, const unsigned* __restrict__ Sin, DevStats st, double mn, double thr,
               double* __restrict__ map, unsigned long long* __restrict__ n_r, int* stop,
               EgsDecide dec, SecFuse sf) {
    pdl_wait();
    {
        __shared__ int skip;
        if (threadIdx.x == 0) skip = stop && *reinterpret_cast<volatile int*>(stop);
        __syncthreads();
        if (skip) {
            egs_tail(dec);
            return;
        }
    }
    const int lane = threadIdx.x & 31;
    SecCtx sc;
    if constexpr (MODE == 2) {
        const double T = *sf.thr;
        sc.tb = dclamp(dmin(T, 1.0), -1.0, 1.0);
        sc.tbf = float(sc.tb);
        sc.thr_ok = T >= -1.0;
    }
    RcoTally tal;
    bool list_full = false;
    unsigned long long surv_local = 0;
    const int ntj = ((g.tc + 31) / 32) * 32;  // whole warps (ballots)
    for (int ti = g.ti_lo + blockIdx.x; ti < g.ti_hi; ti += gridDim.x) {
        const int r0 = ti * 3, r1 = min(r0 + 3, g.er) - 1, cr = (r0 + r1) >> 1;
        const int nr = r1 - r0 + 1, rc = cr - r0;  // rows of the group row, centre's row slot
        const unsigned gbase = unsigned(ti) * unsigned(g.tc);
        unsigned evr[3] = {0u, 0u, 0u};
        for (int tj = threadIdx.x; tj < ntj; tj += blockDim.x) {
            const bool active = tj < g.tc;
            const int tq = active ? tj : 0;
            const int c0 = 3 * tq, c1 = min(c0 + 3, g.ec) - 1, ccol = (c0 + c1) >> 1;
            const int nc = c1 - c0 + 1, jc = ccol - c0;
            unsigned sv[3][3];
            double mm[3][3], om[3][3];
            bool fm[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const unsigned krow = unsigned(r0 + min(i, nr - 1)) * unsigned(g.ec);
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const unsigned k = krow + unsigned(c0 + min(j, nc - 1));
                    sv[i][j] = __ldg(Sin + k);
                    mm[i][j] = __ldg(st.mu + k);
                    om[i][j] = __ldg(st.omega + k);
                    fm[i][j] = __ldg(st.flat + k) != 0;
                }
            }
            double ra = 0.0, sa = 0.0;
            bool dg = false, sd = false;
            if constexpr (MODE == 2) {
                const unsigned gi = gbase + unsigned(tq);
                ra = __ldg(sf.rho_c + gi);
                sa = __ldg(sf.sa_c + gi);
                dg = __ldg(sf.deg_c + gi) != 0;
                sd = sf.seeded ? __ldg(sf.seeded + gi) != 0 : false;
            }
            // the centre's statistics from the loaded rows (selects: no local-memory arrays)
            auto pick = [&](const double (&a)[3][3]) {
                const double r0v = jc == 1 ? a[0][1] : a[0][0];
                const double r1v = jc == 1 ? a[1][1] : a[1][0];
                return rc == 1 ? r1v : r0v;
            };
            const double mc = pick(mm), oc = pick(om);
            const bool fc = rc == 1 ? (jc == 1 ? fm[1][1] : fm[1][0]) : (jc == 1 ? fm[0][1] : fm[0][0]);
            const double mnmc = __dmul_rn(mn, mc);
            unsigned sbits = 0;
            int srr[9], scc[9];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const int r = r0 + i, c = c0 + j;
                    srr[3 * i + j] = r;
                    scc[3 * i + j] = c;
                    if (!active || i >= nr || j >= nc) continue;
                    const unsigned k = unsigned(r) * unsigned(g.ec) + unsigned(c);
                    if (i == rc && j == jc) {  // the group's centre (autocorr.cpp:92-93)
                        if constexpr (MODE == 1) map[k] = 1.0;
                        if constexpr (MODE == 2) sf.visits[k] = 0;
                        continue;
                    }
                    const unsigned e0 = tal.evc;
                    const bool s = rco_member<MODE>(tal, r, c, k, sv[i][j], mm[i][j], om[i][j],
                                                    fm[i][j], mnmc, oc, fc, ra, sa, dg, sd, thr,
                                                    sc, map, sf);
                    evr[i] += tal.evc - e0;
                    sbits |= unsigned(s) << (3 * i + j);
                }
            }
            if constexpr (MODE == 2) rco_list<9>(sbits, srr, scc, sf, list_full, surv_local);
        }
        if (dec.rows_out) {  // CTA-uniform
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const unsigned d = __reduce_add_sync(0xffffffffu, evr[i]);
                if (lane == 0 && d && i < nr) atomicAdd(dec.rows_out + r0 + i, d);
            }
        }
    }
    rco_finish<MODE>(tal, surv_local, n_r, sf, dec);
}

struct Rco3Geom {
    int nt = 0, G = 0, ntiles = 0, seg = 0, nseg = 0, tc_reg = 0;
};

// TMATCH_RCO3=0 keeps the single-pass k_acg for h = 3; TMATCH_RCO3_NT=128|256 and
// TMATCH_RCO3_SEG (group rows per segment) for A/B runs.
bool rco3_enabled() {
    static bool on = [] {
        const char* e = std::getenv("TMATCH_RCO3");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

Rco3Geom rco3_geom(int m, int n, GridDesc gd, bool fused) {
    Rco3Geom a{};
    if (gd.h != 3 || gd.w != 3) return a;
    static const int force_nt = [] {
        const char* e = std::getenv("TMATCH_RCO3_NT");
        const int v = e ? std::atoi(e) : 0;
        return (v == 128 || v == 256) ? v : 0;
    }();
    static const int force_seg = [] {
        const char* e = std::getenv("TMATCH_RCO3_SEG");
        return e ? std::max(0, std::atoi(e)) : 0;
    }();
    const int Q = n / 3, R = n % 3;
    if (Q < 1 || Q > 65) return a;  // the window's warp totals span at most two warps
    if (gd.ec < 4) return a;        // k_rco_epi: a 4-location chunk wraps at most one row
    const int nt = force_nt ? force_nt : (fused ? 128 : 256);
    const int resident = fused ? (nt == 128 ? 3 : 1) : 2;  // CTAs per SM
    const int G = nt - Q - (R > 0) + 1;
    if (G < 32) return a;
    a.nt = nt;
    a.G = G;
    a.tc_reg = gd.ec % 3 == 0 ? gd.tc : gd.tc - 1;
    a.ntiles = (a.tc_reg + G - 1) / G;
    const int rows = gd.ti_hi - gd.ti_lo;
    // segments long enough that the m-row warm-up is a small share of the walk, short enough
    // for a few waves of resident CTAs (2 per SM)
    const int per_wave = std::max(1, (148 * resident) / std::max(1, a.ntiles));
    int seg = force_seg > 0 ? force_seg : std::max((rows + per_wave - 1) / per_wave, 1);
    if (!force_seg) seg = std::min(seg, std::max(m, 96));
    a.seg = std::max(1, std::min(seg, std::max(rows, 1)));
    a.nseg = std::max(1, (rows + a.seg - 1) / a.seg);
    return a;
}

template <int NT, bool HEAD>
void launch_rco3_s(const uint8_t* imgp, int pitch, int m, int n, const Grid& g, unsigned* S,
                   const Rco3Geom& a, const int* stop, cudaStream_t s) {
    launch_pdl(k_rco3_s<NT, HEAD>, dim3(a.ntiles, a.nseg), dim3(NT), 0, s, imgp, pitch, m, n, g,
               S, a.G, a.seg, a.tc_reg, stop);
}

// k_rco_epi's vector loads/stores: the strip's first location must start 16-byte aligned
// statistics (4-byte aligned flags / visit codes); the allocations are, strips offset them
bool rco3_aligned(GridDesc gd, const DevStats& st, const SecFuse& sf) {
    const size_t kb = size_t(gd.ti_lo) * gd.h * gd.ec;
    auto al = [](const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; };
    if (rco3_fused())  // k_rco3_f stages pairs / words at even / 4-aligned global indices
        return al(st.mu, 16) && al(st.omega, 16) && al(st.flat, 4);
    return al(st.mu + kb, 16) && al(st.omega + kb, 16) && al(st.flat + kb, 4) &&
           (!sf.thr || al(sf.visits + kb, 4));
}

template <int NT, bool HEAD, int MODE>
void launch_rco3_f1(const uint8_t* imgp, int pitch, int m, int n, const Grid& g, DevStats st,
                    double mn, double thr, double* map, unsigned long long* n_r, const Rco3Geom& a,
                    int* stop, cudaStream_t s, const EgsDecide& dec, const SecFuse& sf) {
    const size_t smem = kRcoStages * rco_stage_bytes(a.G);
    static size_t attr = 0;
    if (attr < smem) {
        cudaFuncSetAttribute(k_rco3_f<NT, HEAD, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem));
        attr = smem;
    }
    launch_pdl(k_rco3_f<NT, HEAD, MODE>, dim3(a.ntiles, a.nseg), dim3(NT), smem, s, imgp, pitch, m,
               n, g, st, mn, thr, map, n_r, a.G, a.seg, a.tc_reg, stop, dec, sf);
}

template <int NT, bool HEAD>
void launch_rco3_f2(const uint8_t* imgp, int pitch, int m, int n, const Grid& g, DevStats st,
                    double mn, double thr, double* map, unsigned long long* n_r, const Rco3Geom& a,
                    int* stop, cudaStream_t s, const EgsDecide& dec, const SecFuse& sf) {
    if (sf.thr)
        launch_rco3_f1<NT, HEAD, 2>(imgp, pitch, m, n, g, st, mn, thr, map, n_r, a, stop, s, dec, sf);
    else if (map)
        launch_rco3_f1<NT, HEAD, 1>(imgp, pitch, m, n, g, st, mn, thr, map, n_r, a, stop, s, dec, sf);
    else
        launch_rco3_f1<NT, HEAD, 0>(imgp, pitch, m, n, g, st, mn, thr, map, n_r, a, stop, s, dec, sf);
}

cudaError_t launch_rco3_fused(const uint8_t* imgp, int pitch, int m, int n, GridDesc gd,
                              DevStats st, double thr, double* map, unsigned long long* n_r,
                              int* stop, cudaStream_t s, const EgsDecide& dec, const SecFuse& sf,
                              Rco3Geom a) {
    const Grid g = to_grid(gd);
    const double mn = double(m) * double(n);
    cudaError_t e = cudaSuccess;
    unsigned *Rp = nullptr, *Sc = nullptr;
    if (a.tc_reg < gd.tc) {  // the clipped last group column first (no EGS tail on these)
        const int cc = 3 * (gd.tc - 1), wl = gd.ec - cc;
        const int x0 = g.center_row(gd.ti_lo), x1 = g.center_row(gd.ti_hi - 1) + m;
        const int nx = x1 - x0;
        const int items = (gd.ti_hi - gd.ti_lo) * 6;
        e = cudaMallocAsync(reinterpret_cast<void**>(&Rp), size_t(6) * nx * sizeof(unsigned), s);
        if (e == cudaSuccess)
            e = cudaMallocAsync(reinterpret_cast<void**>(&Sc), size_t(items) * sizeof(unsigned), s);
        if (e != cudaSuccess) return e;
        launch_pdl(k_rco3_clip_rows, dim3(std::min((nx + 7) / 8, 148 * 8)), dim3(256), 0, s, imgp,
                   pitch, n, cc, x0, nx, Rp);
        launch_pdl(k_rco3_clip_sum, dim3(std::min((items + 255) / 256, 148 * 4)), dim3(256), 0, s,
                   Rp, m, g, cc, wl, x0, nx, static_cast<unsigned*>(nullptr), Sc);
        EgsDecide d0{};  // counts only; the decision rides on the main launch
        const dim3 cg(std::min((items + 255) / 256, 148 * 4));
        if (sf.thr)
            launch_pdl(k_rco3_clip_epi<2>, cg, dim3(256), 0, s, g, Sc, st, mn, thr, map, n_r, d0, sf);
        else if (map)
            launch_pdl(k_rco3_clip_epi<1>, cg, dim3(256), 0, s, g, Sc, st, mn, thr, map, n_r, d0, sf);
        else
            launch_pdl(k_rco3_clip_epi<0>, cg, dim3(256), 0, s, g, Sc, st, mn, thr, map, n_r, d0, sf);
    }
    if (a.ntiles > 0) {
        const bool head = n % 3 != 0;
        if (a.nt == 128) {
            if (head) launch_rco3_f2<128, true>(imgp, pitch, m, n, g, st, mn, thr, map, n_r, a, stop, s, dec, sf);
            else launch_rco3_f2<128, false>(imgp, pitch, m, n, g, st, mn, thr, map, n_r, a, stop, s, dec, sf);
        } else {
            if (head) launch_rco3_f2<256, true>(imgp, pitch, m, n, g, st, mn, thr, map, n_r, a, stop, s, dec, sf);
            else launch_rco3_f2<256, false>(imgp, pitch, m, n, g, st, mn, thr, map, n_r, a, stop, s, dec, sf);
        }
    }
    e = cudaGetLastError();
    if (Rp) cudaFreeAsync(Rp, s);
    if (Sc) cudaFreeAsync(Sc, s);
    return e;
}

cudaError_t launch_rco3(const uint8_t* imgp, int pitch, int m, int n, GridDesc gd, DevStats st,
                        double thr, double* map, unsigned long long* n_r, int* stop,
                        cudaStream_t s, const EgsDecide& dec, const SecFuse& sf) {
    const Rco3Geom a = rco3_geom(m, n, gd, rco3_fused());
    if (a.nt == 0) return cudaErrorInvalidValue;
    const Grid g = to_grid(gd);
    const int row_lo = g.row_lo(), row_hi = g.row_hi();
    if (row_hi <= row_lo) return cudaSuccess;
    if (rco3_fused())
        return launch_rco3_fused(imgp, pitch, m, n, gd, st, thr, map, n_r, stop, s, dec, sf, a);
    const size_t cells = size_t(row_hi - row_lo) * gd.ec;
    unsigned* Sbuf = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&Sbuf),
                                    ((cells + 3) & ~size_t(3)) * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    unsigned* S = Sbuf - size_t(row_lo) * gd.ec;  // indexed by global extent position
    const bool head = n % 3 != 0;
    if (a.ntiles > 0) {
        if (a.nt == 128) {
            if (head) launch_rco3_s<128, true>(imgp, pitch, m, n, g, S, a, stop, s);
            else launch_rco3_s<128, false>(imgp, pitch, m, n, g, S, a, stop, s);
        } else {
            if (head) launch_rco3_s<256, true>(imgp, pitch, m, n, g, S, a, stop, s);
            else launch_rco3_s<256, false>(imgp, pitch, m, n, g, S, a, stop, s);
        }
    }
    unsigned* Rp = nullptr;
    if (a.tc_reg < gd.tc) {  // the clipped last group column
        const int cc = 3 * (gd.tc - 1), wl = gd.ec - cc;
        const int x0 = g.center_row(gd.ti_lo), x1 = g.center_row(gd.ti_hi - 1) + m;
        const int nx = x1 - x0;
        e = cudaMallocAsync(reinterpret_cast<void**>(&Rp), size_t(6) * nx * sizeof(unsigned), s);
        if (e != cudaSuccess) return e;
        launch_pdl(k_rco3_clip_rows, dim3(std::min((nx + 7) / 8, 148 * 8)), dim3(256), 0, s, imgp,
                   pitch, n, cc, x0, nx, Rp);
        const int items = (gd.ti_hi - gd.ti_lo) * 6;
        launch_pdl(k_rco3_clip_sum, dim3(std::min((items + 255) / 256, 148 * 4)), dim3(256), 0, s,
                   Rp, m, g, cc, wl, x0, nx, S, static_cast<unsigned*>(nullptr));
    }
    const double mn = double(m) * double(n);
    const int blocks = std::min(row_hi - row_lo, 148 * 8);
    static const int minb = [] {  // TMATCH_EPI_MINB: resident CTAs the epilogue is built for
        const char* e = std::getenv("TMATCH_EPI_MINB");
        const int v = e ? std::atoi(e) : 0;
        return (v >= 2 && v <= 4) ? v : 3;
    }();
    auto epi = [&](auto kern) {
        launch_pdl(kern, dim3(blocks), dim3(256), 0, s, g, S, st, mn, thr, map, n_r, stop, dec, sf);
    };
    // TMATCH_EPI_V: 2 or 4 aligned locations per thread, 3: one group segment (default on
    // small extents: C2 37 vs 43 us), 9: one whole group (default on large ones: C5 1.51 vs
    // 1.61 ms -- 2 CTAs/SM at 128 registers want many group rows)
    static const int vw_env = [] {
        const char* e = std::getenv("TMATCH_EPI_V");
        const int v = e ? std::atoi(e) : 0;
        return (v == 2 || v == 4 || v == 3 || v == 9) ? v : 0;
    }();
    const int vw = vw_env ? vw_env : (double(gd.er) * double(gd.ec) > 3.2e7 ? 9 : 3);
    const int mode = sf.thr ? 2 : (map ? 1 : 0);
    if (vw == 9) {
        auto epi9 = [&](auto kern) {
            const int gblocks = std::min(gd.ti_hi - gd.ti_lo, 148 * 8);
            launch_pdl(kern, dim3(gblocks), dim3(256), 0, s, g, S, st, mn, thr, map, n_r, stop, dec,
                       sf);
        };
        if (mode == 2) {
            if (minb == 3 && std::getenv("TMATCH_EPI_MINB")) epi9(k_rco_epg9<2, 3>);
            else if (minb == 4) epi9(k_rco_epg9<2, 4>);
            else epi9(k_rco_epg9<2, 2>);
        } else if (mode == 1) {
            epi9(k_rco_epg9<1, 2>);
        } else {
            epi9(k_rco_epg9<0, 2>);
        }
    } else if (vw == 3) {
        if (mode == 2) {  // (4 resident CTAs unless TMATCH_EPI_MINB says otherwise)
            if (minb == 3 && std::getenv("TMATCH_EPI_MINB")) epi(k_rco_epg<2, 3>);
            else if (minb == 2) epi(k_rco_epg<2, 2>);
            else epi(k_rco_epg<2, 4>);
        } else if (mode == 1) {
            epi(k_rco_epg<1, 3>);
        } else {
            epi(k_rco_epg<0, 3>);
        }
    } else if (mode == 2) {
        if (vw == 2) {
            if (minb == 4) epi(k_rco_epi<2, 4, 2>);
            else epi(k_rco_epi<2, 3, 2>);
        } else {
            if (minb == 4) epi(k_rco_epi<2, 4, 4>);
            else if (minb == 2) epi(k_rco_epi<2, 2, 4>);
            else epi(k_rco_epi<2, 3, 4>);
        }
    } else if (mode == 1) {
        epi(k_rco_epi<1, 3, 4>);
    } else {
        epi(k_rco_epi<0, 3, 4>);
    }
    e = cudaGetLastError();
    cudaFreeAsync(Sbuf, s);
    if (Rp) cudaFreeAsync(Rp, s);
    return e;
}

template <int H>
cudaError_t launch_acv(const uint8_t* img, int p, int q, int m, int w, int ti_base, int trr,
                       int tr, unsigned* V, cudaStream_t s) {
    constexpr int D = H == 1 ? 16 : (H == 3 ? 8 : (H == 5 ? 4 : (H == 7 ? 3 : 2)));
    // segments of centre rows: enough CTAs for ~4 waves, at least 2*m rows of walk each
    const int colblocks = (q + kAcvThreads - 1) / kAcvThreads;
    int nseg = std::max(1, (148 * 16) / std::max(1, colblocks * w));
    const int rows = trr - ti_base;
    int seg = std::max((2 * m) / H + 1, (rows + nseg - 1) / nseg);
    nseg = (rows + seg - 1) / seg;
    dim3 grid(colblocks, w, std::max(1, nseg));
    if (rows > 0)
        k_acv<H, D><<<grid, kAcvThreads, 0, s>>>(img, p, q, m, w, trr, tr, seg, V, ti_base);
    return cudaGetLastError();
}

bool acv_supported(int m, int h) {
    (void)m;
    return h <= 11 && h % 2 == 1;
}

struct AcRowsGeom {
    int seg, ring, spitch;
    size_t smem;
};

template <int W>
AcRowsGeom ac_rows_geom(int n, int h) {
    AcRowsGeom g;
    g.seg = std::max(4, 256 / W);
    g.ring = (n + W - 1) / W + 2;
    const int swid = g.seg * W + n + 2 * W + 2;
    int pitch = (swid + 3) & ~3;
    if (((pitch / 4) & 1) == 0) pitch += 4;  // rows 4 mod 8 bytes apart: no bank conflicts
    g.spitch = pitch;
    const int srow = kAcRows + h / 2 + 1;  // + the zero row
    g.smem = ((size_t(srow) * pitch + 15) & ~size_t(15)) + size_t(g.ring) * W * kAcRows * 4;
    return g;
}

template <int W>
cudaError_t launch_ac_rows(const uint8_t* img, int p, int q, int n, int h, int tcr, int tc,
                           unsigned* H, cudaStream_t s) {
    const AcRowsGeom geo = ac_rows_geom<W>(n, h);
    if (geo.smem > 200 * 1024) return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_ac_rows<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    dim3 grid((p + kAcRows - 1) / kAcRows, h, (tcr + geo.seg - 1) / geo.seg);
    if (tcr > 0)
        k_ac_rows<W><<<grid, kAcRows, geo.smem, s>>>(img, p, q, n, tcr, tc, geo.seg, geo.ring,
                                                      geo.spitch, H);
    return cudaGetLastError();
}

bool ac_supported(int n, int h, int w) {
    size_t smem = 0;
    switch (w) {
        case 1: smem = ac_rows_geom<1>(n, h).smem; break;
        case 3: smem = ac_rows_geom<3>(n, h).smem; break;
        case 5: smem = ac_rows_geom<5>(n, h).smem; break;
        case 7: smem = ac_rows_geom<7>(n, h).smem; break;
        case 9: smem = ac_rows_geom<9>(n, h).smem; break;
        case 11: smem = ac_rows_geom<11>(n, h).smem; break;
        default: return false;
    }
    return smem <= 200 * 1024;
}

// ---- replica path helpers ---------------------------------------------------------------

__global__ void k_autocorr_init(double* map, Grid g, const int* stop) {
    if (stop && *stop) return;
    const size_t E = size_t(g.er) * g.ec;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < E;
         k += size_t(gridDim.x) * blockDim.x) {
        int r, c;
        g.rc(k, r, c);
        const int ti = g.tile_r(r), tj = g.tile_c(c);
        map[k] = (g.center_row(ti) == r && g.center_col(tj) == c) ? 1.0 : 0.0;
    }
}

// One offset: prefix is the (ph+1) x (pw+1) replica prefix table of the product image
// whose origin is (orr, occ) (autocorr.cpp:64-76); cross sum at the centre is the window
// difference at (cr - orr, cc - occ) in stats.cpp:50 order.
__global__ void k_autocorr_offset(const double* __restrict__ prefix, int ph, int pw, int m, int n,
                                  Grid g, DevStats st, int di, int dj, double* __restrict__ map,
                                  const int* stop) {
    if (stop && *stop) return;
    const long long G = (long long)g.tr * g.tc;
    const int orr = max(0, -di), occ = max(0, -dj);
    const size_t ppw = size_t(pw) + 1;
    const double mn = double(m) * double(n);
    for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < G;
         gi += (long long)gridDim.x * blockDim.x) {
        const int ti = int(gi / g.tc), tj = int(gi % g.tc);
        if (ti < g.ti_lo || ti >= g.ti_hi) continue;
        const int cr = g.center_row(ti), cc = g.center_col(tj);
        const int r0 = ti * g.h, r1 = min(r0 + g.h, g.er) - 1;
        const int c0 = tj * g.w, c1 = min(c0 + g.w, g.ec) - 1;
        const int mr = cr + di, mc = cc + dj;
        if (mr < r0 || mr > r1 || mc < c0 || mc > c1) continue;
        const size_t kc = size_t(cr) * g.ec + cc, km = size_t(mr) * g.ec + mc;
        if (st.flat[kc] || st.flat[km]) continue;
        const int r = cr - orr, c = cc - occ;
        const double* top = prefix + size_t(r) * ppw;
        const double* bot = prefix + size_t(r + m) * ppw;
        const double cross = __dadd_rn(__dsub_rn(__dsub_rn(bot[c + n], top[c + n]), bot[c]), top[c]);
        const double num = __dsub_rn(cross, __dmul_rn(__dmul_rn(mn, st.mu[kc]), st.mu[km]));
        map[km] = dclamp(__ddiv_rn(num, __dmul_rn(st.omega[kc], st.omega[km])), -1.0, 1.0);
    }
}

// k_autocorr_offset for a batch of offsets (grid.y = offset k of the batch; its prefix
// table at prefix + k * pslot): one launch instead of one per offset.
__global__ void k_autocorr_offset_b(const double* __restrict__ prefix, size_t pslot, OffBatch ob,
                                    int m, int n, Grid g, DevStats st, double* __restrict__ map,
                                    const int* stop) {
    if (stop && *stop) return;
    const int kb = blockIdx.y;
    const int di = ob.di[kb], dj = ob.dj[kb], pw = ob.pw[kb];
    const double* pre = prefix + size_t(kb) * pslot;
    const long long G = (long long)g.tr * g.tc;
    const int orr = max(0, -di), occ = max(0, -dj);
    const size_t ppw = size_t(pw) + 1;
    const double mn = double(m) * double(n);
    for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < G;
         gi += (long long)gridDim.x * blockDim.x) {
        const int ti = int(gi / g.tc), tj = int(gi % g.tc);
        if (ti < g.ti_lo || ti >= g.ti_hi) continue;
        const int cr = g.center_row(ti), cc = g.center_col(tj);
        const int r0 = ti * g.h, r1 = min(r0 + g.h, g.er) - 1;
        const int c0 = tj * g.w, c1 = min(c0 + g.w, g.ec) - 1;
        const int mr = cr + di, mc = cc + dj;
        if (mr < r0 || mr > r1 || mc < c0 || mc > c1) continue;
        const size_t kc = size_t(cr) * g.ec + cc, km = size_t(mr) * g.ec + mc;
        if (st.flat[kc] || st.flat[km]) continue;
        const int r = cr - orr, c = cc - occ;
        const double* top = pre + size_t(r) * ppw;
        const double* bot = pre + size_t(r + m) * ppw;
        const double cross = __dadd_rn(__dsub_rn(__dsub_rn(bot[c + n], top[c + n]), bot[c]), top[c]);
        const double num = __dsub_rn(cross, __dmul_rn(__dmul_rn(mn, st.mu[kc]), st.mu[km]));
        map[km] = dclamp(__ddiv_rn(num, __dmul_rn(st.omega[kc], st.omega[km])), -1.0, 1.0);
    }
}

__global__ void k_retained(const double* __restrict__ map, Grid g, double thr,
                           unsigned long long* n_r, const int* stop) {
    if (stop && *stop) return;
    const size_t k0 = size_t(g.row_lo()) * g.ec, k1 = size_t(g.row_hi()) * g.ec;
    unsigned long long local = 0;
    for (size_t k = k0 + blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < k1;
         k += size_t(gridDim.x) * blockDim.x) {
        int r, c;
        g.rc(k, r, c);
        const int ti = g.tile_r(r), tj = g.tile_c(c);
        if (g.center_row(ti) == r && g.center_col(tj) == c) continue;
        if (map[k] < thr) ++local;
    }
    local = warp_sum(local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(n_r, local);
}

Grid to_grid(GridDesc d) {
    return Grid::make(d.er, d.ec, d.h, d.w, d.tr, d.tc, d.ti_lo, d.ti_hi);
}

}  // namespace

cudaError_t autocorr_u8(const uint8_t* img, int p, int q, int m, int n, GridDesc gd, DevStats st,
                        double retain_threshold, double* map, unsigned long long* n_r,
                        cudaStream_t s) {
    ACParams P;
    P.img = img;
    P.p = p;
    P.q = q;
    P.m = m;
    P.n = n;
    P.g = to_grid(gd);
    P.st = st;
    P.thr = retain_threshold;
    P.map = map;
    P.n_r = n_r;
    const int hr = gd.h / 2, wr = gd.w / 2;
    // Choose the group tile so the staged image + H fit in ~96 KB of shared memory.
    int gtr = 16, gtc = 32;
    size_t bytes = 0;
    for (;;) {
        const int srows = (gtr - 1) * gd.h + 2 * hr + m + 1;
        const int scols = (gtc - 1) * gd.w + 2 * wr + n + 1;
        // bytes per staged row = 4 mod 8: lanes on consecutive rows hit distinct banks
        int spitch = (scols + 3) & ~3;
        if (((spitch / 4) & 1) == 0) spitch += 4;
        const int nx = (gtr - 1) * gd.h + m + 1;
        bytes = ((size_t(srows) * spitch + 15) & ~size_t(15)) + size_t(nx) * gtc * 4 +
                size_t(gtc + gtr) * 4;
        P.srows = srows;
        P.spitch = spitch;
        P.nx_max = nx;
        if (bytes <= 96 * 1024 || (gtr == 1 && gtc == 1)) break;
        if (gtc >= gtr && gtc > 1) gtc /= 2;
        else if (gtr > 1) gtr /= 2;
    }
    P.gtr = gtr;
    P.gtc = gtc;
    if (bytes > 200 * 1024) return cudaErrorInvalidValue;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_autocorr_u8, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    const int strip_rows = std::max(1, gd.ti_hi - gd.ti_lo);
    const int base = ((gd.tc + gtc - 1) / gtc) * ((strip_rows + gtr - 1) / gtr);
    const int noff = gd.h * gd.w - 1;
    int splits = std::max(1, std::min(noff, (148 * 6 + base - 1) / base));
    P.noff_per = std::max(1, (noff + splits - 1) / splits);
    splits = std::max(1, (noff + P.noff_per - 1) / P.noff_per);
    dim3 grid((gd.tc + gtc - 1) / gtc, (strip_rows + gtr - 1) / gtr, std::max(splits, 1));
    k_autocorr_u8<<<grid, 256, bytes, s>>>(P);
    return cudaGetLastError();
}

size_t autocorr_rowsum_bytes(int p, GridDesc g) {  // H and its transposed prefix P
    return 2 * size_t(g.h) * g.w * g.tc * p * sizeof(unsigned);
}

// The 8-bit R_co kernels (k_acg, k_acf, the column walk and the two-pass kernel) keep the
// centre-member cross sum S = sum of m*n products of two bytes in u32: exact only while
// m*n*255^2 < 2^32 (m*n < 66051).  Larger templates take the generic k_autocorr_u8 (s64).
static bool u32_cross_exact(int m, int n) {
    return double(m) * double(n) * 65025.0 < 4294967296.0;
}

bool autocorr_two_pass_supported(int m, int n, GridDesc g) {
    return u32_cross_exact(m, n) && ac_supported(n, g.h, g.w);
}


// One EGS acceptance step on the device (egs.cpp:61-88 with total_cost of egs.cpp:28-37,
// the same FP64 operations as the host replay in engine.cpp): after candidate (h, w) with
// retained count *n_r, set *stop when it is rejected or is the last one, so the kernels of
// the remaining candidates of the batch exit at entry.  The host still decides from the
// counts; this only skips work the host would ignore.  *h_acc tracks the last accepted
// size and *gate = (EGS finished with h_e == want): the speculative centre scan enqueued
// behind the batch for the predicted size `want` runs only then (0 = no speculation).  A
// stop already set at entry came from an earlier decision or from the candidate's own
// in-kernel rejection; either way the gate is final.
__global__ void k_egs_decide(EgsDecide d) {
    pdl_wait();
    egs_decide_run(d);
}

cudaError_t egs_decide_d(const EgsDecide& d, cudaStream_t s) {
    launch_pdl(k_egs_decide, dim3(1), dim3(1), 0, s, d);
    return cudaGetLastError();
}

cudaError_t egs_decide(const unsigned long long* n_r, double* prev_cost, int* stop, int er, int ec,
                       int h, int w, double xi, int cap, int* h_acc, int want,
                       unsigned long long* gate, cudaStream_t s, const unsigned long long* nr_all,
                       int nc, ResultBlock* out, unsigned long long seq) {
    EgsDecide d{};
    d.n_r = n_r;
    d.prev = prev_cost;
    d.stop = stop;
    d.er = er;
    d.ec = ec;
    d.h = h;
    d.w = w;
    d.xi = xi;
    d.cap = cap;
    d.h_acc = h_acc;
    d.want = want;
    d.gate = gate;
    d.nr_all = nr_all;
    d.nc = nc;
    d.out = out;
    d.seq = seq;
    launch_pdl(k_egs_decide, dim3(1), dim3(1), 0, s, d);
    return cudaGetLastError();
}

bool autocorr_sec_fuse_supported(int m, int n, GridDesc g) {
    return autocorr_fused_supported(m, n, g) && acg_enabled() && (g.h == 3 || g.h == 5) &&
           g.h == g.w && acg_geom(m, n, g, acg_threads(g)).nt > 0;
}

bool autocorr_fused_supported(int m, int n, GridDesc g) {
    // 32-bit row offsets; the walk may read h/2 <= kU8PadRows rows below the image
    const size_t p = size_t(g.er) + m - 1, q = size_t(g.ec) + n - 1;
    return u32_cross_exact(m, n) && g.h % 2 == 1 && g.h / 2 <= kU8PadRows && g.h <= 11 &&
           (p + kU8PadRows) * q < (size_t(1) << 31) &&
           size_t(g.er) * g.ec < (size_t(1) << 32) &&
           (acf_geom(m, n, g).ny > 0 || acg_geom(m, n, g, acg_threads(g)).nt > 0);
}

cudaError_t autocorr_u8_fused(const uint8_t* img, int p, int q, int m, int n, GridDesc gd,
                              DevStats st, double retain_threshold, double* map,
                              unsigned long long* n_r, int* stop, cudaStream_t s,
                              const double* egs_prev, double egs_central, double egs_xi,
                              const uint8_t* imgp, int pitch, const EgsDecide* dec,
                              bool* decided, const SecFuse* fuse, int* launches) {
    if (decided) *decided = false;
    if (launches) *launches = 1;
    if (imgp && pitch % 16 == 0 && acg_enabled() && acg_geom(m, n, gd, acg_threads(gd)).nt > 0 &&
        (gd.h == 3 || gd.h == 5)) {
        // the EGS decision rides on the launch's tail (no k_egs_decide launch)
        const EgsDecide d = dec ? *dec : EgsDecide{};
        const SecFuse f = fuse ? *fuse : SecFuse{};
        if (decided) *decided = d.ticket != nullptr;
        if (gd.h == 3 && rco3_enabled() && rco3_geom(m, n, gd, rco3_fused()).nt > 0 && rco3_aligned(gd, st, f)) {
            if (launches)
                *launches = rco3_geom(m, n, gd, rco3_fused()).tc_reg < gd.tc ? 4
                            : rco3_fused()                                  ? 1 : 2;
            return launch_rco3(imgp, pitch, m, n, gd, st, retain_threshold, map, n_r, stop, s, d,
                               f);
        }
        g_acg_extra = 0;
        struct Extra {  // k_acg's extra launches into *launches on every return below
            int* out;
            ~Extra() {
                if (out) *out += g_acg_extra;
            }
        } extra{launches};
        if (gd.h == 3)
            return launch_acg<3>(imgp, pitch, q, m, n, gd, st, retain_threshold, map, n_r, stop,
                                 egs_prev, egs_central, egs_xi, s, d, f);
        return launch_acg<5>(imgp, pitch, q, m, n, gd, st, retain_threshold, map, n_r, stop,
                             egs_prev, egs_central, egs_xi, s, d, f);
    }
    if (fuse && fuse->thr) return cudaErrorInvalidValue;  // scan 2 fuses into k_acg only
    switch (gd.h) {
        case 1: return launch_acf<1>(img, p, q, m, n, gd, st, retain_threshold, map, n_r, stop,
                                     egs_prev, egs_central, egs_xi, s);
        case 3: return launch_acf<3>(img, p, q, m, n, gd, st, retain_threshold, map, n_r, stop,
                                     egs_prev, egs_central, egs_xi, s);
        case 5: return launch_acf<5>(img, p, q, m, n, gd, st, retain_threshold, map, n_r, stop,
                                     egs_prev, egs_central, egs_xi, s);
        case 7: return launch_acf<7>(img, p, q, m, n, gd, st, retain_threshold, map, n_r, stop,
                                     egs_prev, egs_central, egs_xi, s);
        case 9: return launch_acf<9>(img, p, q, m, n, gd, st, retain_threshold, map, n_r, stop,
                                     egs_prev, egs_central, egs_xi, s);
        case 11: return launch_acf<11>(img, p, q, m, n, gd, st, retain_threshold, map, n_r, stop,
                                     egs_prev, egs_central, egs_xi, s);
        default: return cudaErrorInvalidValue;
    }
}

size_t autocorr_colwalk_bytes(int q, GridDesc g) {
    return size_t(g.h) * g.w * g.tr * q * sizeof(unsigned);
}

bool autocorr_colwalk_supported(int m, int n, int q, GridDesc g) {
    (void)q;
    return u32_cross_exact(m, n) && acv_supported(m, g.h) && g.w <= 11;
}

cudaError_t autocorr_u8_colwalk(const uint8_t* img, int p, int q, int m, int n, GridDesc gd,
                                DevStats st, double retain_threshold, double* map,
                                unsigned long long* n_r, unsigned* V, cudaStream_t s) {
    const bool clipped = size_t(gd.tr) * gd.h > size_t(gd.er);
    // regular centre rows of this strip: [ti_lo, trr)
    const int trr = std::min(gd.ti_hi, clipped ? gd.tr - 1 : gd.tr);
    const int tb = gd.ti_lo;
    cudaError_t e = cudaSuccess;
    switch (gd.h) {
        case 1: e = launch_acv<1>(img, p, q, m, gd.w, tb, trr, gd.tr, V, s); break;
        case 3: e = launch_acv<3>(img, p, q, m, gd.w, tb, trr, gd.tr, V, s); break;
        case 5: e = launch_acv<5>(img, p, q, m, gd.w, tb, trr, gd.tr, V, s); break;
        case 7: e = launch_acv<7>(img, p, q, m, gd.w, tb, trr, gd.tr, V, s); break;
        case 9: e = launch_acv<9>(img, p, q, m, gd.w, tb, trr, gd.tr, V, s); break;
        case 11: e = launch_acv<11>(img, p, q, m, gd.w, tb, trr, gd.tr, V, s); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    const Grid g = to_grid(gd);
    if (clipped && gd.tr - 1 >= gd.ti_lo && gd.tr - 1 < gd.ti_hi) {
        dim3 grid((q + 127) / 128, gd.w, gd.h);
        k_acv_last<<<grid, 128, 0, s>>>(img, p, q, m, gd.h, gd.w, g.center_row(gd.tr - 1),
                                        gd.tr - 1, gd.tr, V);
    }
    // column tiles: a multiple of w, sized so the W prefix lines fit in ~64 KB
    int tw = std::max(gd.w, (384 / gd.w) * gd.w);
    tw = std::min(tw, (gd.ec + gd.w - 1) / gd.w * gd.w);
    const int lpitch = ((tw + n + 1) + 3) & ~3;
    const size_t smem = size_t(gd.w) * lpitch * sizeof(unsigned);
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_ac_hrow, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    dim3 grid(std::max(1, gd.ti_hi - gd.ti_lo), gd.h, (gd.ec + tw - 1) / tw);
    if (gd.ti_hi > gd.ti_lo)
        k_ac_hrow<<<grid, 128, smem, s>>>(V, q, m, n, g, st, retain_threshold, map, n_r, tw, lpitch);
    return cudaGetLastError();
}

cudaError_t autocorr_u8_two_pass(const uint8_t* img, int p, int q, int m, int n, GridDesc gd,
                                 DevStats st, double retain_threshold, double* map,
                                 unsigned long long* n_r, int* Hraw, cudaStream_t s) {
    unsigned* H = reinterpret_cast<unsigned*>(Hraw);
    const bool clipped = size_t(gd.tc) * gd.w > size_t(gd.ec);
    const int tcr = clipped ? gd.tc - 1 : gd.tc;
    cudaError_t e = cudaSuccess;
    switch (gd.w) {
        case 1: e = launch_ac_rows<1>(img, p, q, n, gd.h, tcr, gd.tc, H, s); break;
        case 3: e = launch_ac_rows<3>(img, p, q, n, gd.h, tcr, gd.tc, H, s); break;
        case 5: e = launch_ac_rows<5>(img, p, q, n, gd.h, tcr, gd.tc, H, s); break;
        case 7: e = launch_ac_rows<7>(img, p, q, n, gd.h, tcr, gd.tc, H, s); break;
        case 9: e = launch_ac_rows<9>(img, p, q, n, gd.h, tcr, gd.tc, H, s); break;
        case 11: e = launch_ac_rows<11>(img, p, q, n, gd.h, tcr, gd.tc, H, s); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    const Grid g = to_grid(gd);
    if (clipped) {
        const long long items = (long long)gd.h * gd.w * p;
        const int blocks = int(std::min<long long>((items * 32 + 255) / 256, 148 * 32));
        k_ac_rows_last<<<blocks, 256, 0, s>>>(img, p, q, n, gd.h, gd.w, g.center_col(gd.tc - 1),
                                              gd.tc - 1, gd.tc, H);
    }
    const int hw = gd.h * gd.w;
    unsigned* P = H + size_t(hw) * gd.tc * p;  // second half of the scratch
    k_ac_scan<<<hw * ((gd.tc + 31) / 32), 1024, 0, s>>>(H, P, p, gd.tc, hw);
    const long long items = (long long)hw * gd.tr * gd.tc;
    const int blocks = int(std::min<long long>((items + 255) / 256, 148 * 32));
    k_ac_epi<<<blocks, 256, 0, s>>>(P, p, m, n, g, st, retain_threshold, map, n_r);
    return cudaGetLastError();
}

cudaError_t autocorr_init(double* map, GridDesc g, cudaStream_t s, const int* stop) {
    const size_t E = size_t(g.er) * g.ec;
    const int blocks = int(std::min<size_t>((E + 255) / 256, 148 * 16));
    k_autocorr_init<<<blocks, 256, 0, s>>>(map, to_grid(g), stop);
    return cudaGetLastError();
}

cudaError_t autocorr_offset_epilogue(const double* prefix, int ph, int pw, int m, int n,
                                     GridDesc g, DevStats st, int di, int dj, double* map,
                                     cudaStream_t s, const int* stop) {
    const long long G = (long long)g.tr * g.tc;
    const int blocks = int(std::min<long long>((G + 255) / 256, 148 * 16));
    k_autocorr_offset<<<blocks, 256, 0, s>>>(prefix, ph, pw, m, n, to_grid(g), st, di, dj, map,
                                             stop);
    return cudaGetLastError();
}

cudaError_t autocorr_offset_epilogue_b(const double* prefix, size_t pslot, const OffBatch& ob,
                                       int m, int n, GridDesc g, DevStats st, double* map,
                                       cudaStream_t s, const int* stop) {
    const long long G = (long long)g.tr * g.tc;
    const int blocks = int(std::min<long long>((G + 255) / 256, 148 * 4));
    if (ob.n > 0)
        k_autocorr_offset_b<<<dim3(blocks, ob.n), 256, 0, s>>>(prefix, pslot, ob, m, n, to_grid(g),
                                                              st, map, stop);
    return cudaGetLastError();
}

cudaError_t retained_count(const double* map, GridDesc g, double threshold,
                           unsigned long long* n_r, cudaStream_t s, const int* stop) {
    const size_t E = size_t(g.er) * g.ec;
    const int blocks = int(std::min<size_t>((E + 255) / 256, 148 * 16));
    k_retained<<<blocks, 256, 0, s>>>(map, to_grid(g), threshold, n_r, stop);
    return cudaGetLastError();
}

}  // namespace tmk
