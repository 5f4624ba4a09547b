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
    const int ti0 = blockIdx.y * P.gtr, tj0 = blockIdx.x * P.gtc;
    const int nti = min(P.gtr, g.tr - ti0), ntj = min(P.gtc, g.tc - tj0);
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
    const int r_lo = x0 + min(0, di);         // staged rows [r_lo, r_lo + srow)
    const int srow = kAcRows + abs(di);
    uint8_t* simg = sm;
    int* rec = reinterpret_cast<int*>(sm + ((size_t(srow) * spitch + 15) & ~size_t(15)));
    for (int idx = threadIdx.x; idx < srow * swid; idx += kAcRows) {
        const int a = idx / swid, b = idx - a * swid;
        const int r = r_lo + a, c = c_lo + b;
        simg[a * spitch + b] = (r >= 0 && r < p && c >= 0 && c < q) ? img[size_t(r) * q + c] : 0;
    }
    __syncthreads();
    const int x = x0 + threadIdx.x;
    const bool row_ok = x < p && x + di >= 0 && x + di < p;
    // local column index of image column c is c - c_lo
    const uint8_t* ra = simg + (x - r_lo) * spitch - c_lo;
    const uint8_t* rb = simg + (x + di - r_lo) * spitch - c_lo;
    // ring slot of column c is (c - y_s + wr) mod W: static (s + t) % W inside a block
    int acc[W];
    int rg[W];
#pragma unroll
    for (int t = 0; t < W; ++t) {
        acc[t] = 0;
        rg[t] = (t < W - 1 && row_ok) ? int(rb[y_s - wr + t]) : 0;
    }
    const size_t plane = size_t(tc) * p;  // one (di,dj) plane of H
    for (int y0 = y_s; y0 <= y_e; y0 += W) {
#pragma unroll
        for (int s = 0; s < W; ++s) {
            const int y = y0 + s;
            // events use the prefix before P(y) is added
            if (s == wr) {  // window start of centre k = (y - wr) / W
                const int k = (y - wr) / W;
                if (k < k1) {
                    const int slot = k % ring;
#pragma unroll
                    for (int t = 0; t < W; ++t) rec[(slot * W + t) * kAcRows + threadIdx.x] = acc[t];
                }
            }
            if (s == (wr + n) % W) {  // window end of centre k = (y - n - wr) / W
                const int kk = y - n - wr;
                if (kk >= k0 * W && kk < k1 * W) {
                    const int k = kk / W;
                    const int slot = k % ring;
                    if (x < p) {
#pragma unroll
                        for (int t = 0; t < W; ++t)
                            H[(size_t(dii) * W + t) * plane + size_t(k) * p + x] =
                                unsigned(acc[t] - rec[(slot * W + t) * kAcRows + threadIdx.x]);
                    }
                }
            }
            rg[(s + W - 1) % W] = row_ok ? int(rb[y + wr]) : 0;  // I(x+di, y+wr)
            const int a = row_ok ? int(ra[y]) : 0;
#pragma unroll
            for (int t = 0; t < W; ++t) acc[t] += a * rg[(s + t) % W];  // dj = t - wr
        }
    }
}

// Clipped last centre column (irregular position): direct n-wide sums.
__global__ void k_ac_rows_last(const uint8_t* __restrict__ img, int p, int q, int n, int h, int w,
                               int cc, int kcol, int tc, unsigned* __restrict__ H) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int oi = blockIdx.y;  // (di, dj) raster index in [0, h*w)
    const int di = oi / w - h / 2, dj = oi % w - w / 2;
    if (x >= p) return;
    int s = 0;
    if (x + di >= 0 && x + di < p) {
        const uint8_t* ra = img + size_t(x) * q + cc;
        const uint8_t* rb = img + size_t(x + di) * q + cc + dj;
        for (int b = 0; b < n; ++b) {
            const int cb = cc + dj + b;
            s += int(ra[b]) * ((cb >= 0 && cb < q) ? int(rb[b]) : 0);
        }
    }
    H[size_t(oi) * tc * p + size_t(kcol) * p + x] = unsigned(s);
}

// In-place inclusive prefix along x of every (offset, centre column) line (wrapping u32).
__global__ void k_ac_scan(unsigned* __restrict__ H, int p, long long lines) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long li = warp; li < lines; li += nwarps) {
        unsigned* L = H + li * p;
        unsigned carry = 0;
        for (int x0 = 0; x0 < p; x0 += 32) {
            const int x = x0 + lane;
            unsigned v = x < p ? L[x] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += u;
            }
            v += carry;
            if (x < p) L[x] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    }
}

// Epilogue: thread = (offset, centre row ti, centre column k), lanes over k.
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
        const unsigned* L = P + (size_t(oi) * g.tc + k) * p;
        const unsigned S = L[cr + m - 1] - (cr > 0 ? L[cr - 1] : 0u);
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
    const int srow = kAcRows + h / 2;
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

__global__ void k_autocorr_init(double* map, Grid g) {
    const size_t E = size_t(g.er) * g.ec;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < E;
         k += size_t(gridDim.x) * blockDim.x) {
        const int r = int(k / g.ec), c = int(k % g.ec);
        const int ti = g.tile_r(r), tj = g.tile_c(c);
        map[k] = (g.center_row(ti) == r && g.center_col(tj) == c) ? 1.0 : 0.0;
    }
}

// One offset: prefix is the (ph+1) x (pw+1) replica prefix table of the product image
// whose origin is (orr, occ) (autocorr.cpp:64-76); cross sum at the centre is the window
// difference at (cr - orr, cc - occ) in stats.cpp:50 order.
__global__ void k_autocorr_offset(const double* __restrict__ prefix, int ph, int pw, int m, int n,
                                  Grid g, DevStats st, int di, int dj, double* __restrict__ map) {
    const long long G = (long long)g.tr * g.tc;
    const int orr = max(0, -di), occ = max(0, -dj);
    const size_t ppw = size_t(pw) + 1;
    const double mn = double(m) * double(n);
    for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < G;
         gi += (long long)gridDim.x * blockDim.x) {
        const int ti = int(gi / g.tc), tj = int(gi % g.tc);
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

__global__ void k_retained(const double* __restrict__ map, Grid g, double thr,
                           unsigned long long* n_r) {
    const size_t E = size_t(g.er) * g.ec;
    unsigned long long local = 0;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < E;
         k += size_t(gridDim.x) * blockDim.x) {
        const int r = int(k / g.ec), c = int(k % g.ec);
        const int ti = g.tile_r(r), tj = g.tile_c(c);
        if (g.center_row(ti) == r && g.center_col(tj) == c) continue;
        if (map[k] < thr) ++local;
    }
    local = warp_sum(local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(n_r, local);
}

Grid to_grid(GridDesc d) { return Grid{d.er, d.ec, d.h, d.w, d.tr, d.tc}; }

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
    const int base = ((gd.tc + gtc - 1) / gtc) * ((gd.tr + gtr - 1) / gtr);
    const int noff = gd.h * gd.w - 1;
    int splits = std::max(1, std::min(noff, (148 * 6 + base - 1) / base));
    P.noff_per = std::max(1, (noff + splits - 1) / splits);
    splits = std::max(1, (noff + P.noff_per - 1) / P.noff_per);
    dim3 grid((gd.tc + gtc - 1) / gtc, (gd.tr + gtr - 1) / gtr, std::max(splits, 1));
    k_autocorr_u8<<<grid, 256, bytes, s>>>(P);
    return cudaGetLastError();
}

size_t autocorr_rowsum_bytes(int p, GridDesc g) {
    return size_t(g.h) * g.w * g.tc * p * sizeof(unsigned);
}

bool autocorr_two_pass_supported(int n, GridDesc g) { return ac_supported(n, g.h, g.w); }

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
        dim3 grid((p + 127) / 128, gd.h * gd.w);
        k_ac_rows_last<<<grid, 128, 0, s>>>(img, p, q, n, gd.h, gd.w, g.center_col(gd.tc - 1),
                                            gd.tc - 1, gd.tc, H);
    }
    const long long lines = (long long)gd.h * gd.w * gd.tc;
    k_ac_scan<<<int(std::min<long long>((lines + 7) / 8, 148 * 32)), 256, 0, s>>>(H, p, lines);
    const long long items = (long long)gd.h * gd.w * gd.tr * gd.tc;
    const int blocks = int(std::min<long long>((items + 255) / 256, 148 * 32));
    k_ac_epi<<<blocks, 256, 0, s>>>(H, p, m, n, g, st, retain_threshold, map, n_r);
    return cudaGetLastError();
}

cudaError_t autocorr_init(double* map, GridDesc g, cudaStream_t s) {
    const size_t E = size_t(g.er) * g.ec;
    const int blocks = int(std::min<size_t>((E + 255) / 256, 148 * 16));
    k_autocorr_init<<<blocks, 256, 0, s>>>(map, to_grid(g));
    return cudaGetLastError();
}

cudaError_t autocorr_offset_epilogue(const double* prefix, int ph, int pw, int m, int n,
                                     GridDesc g, DevStats st, int di, int dj, double* map,
                                     cudaStream_t s) {
    const long long G = (long long)g.tr * g.tc;
    const int blocks = int(std::min<long long>((G + 255) / 256, 148 * 16));
    k_autocorr_offset<<<blocks, 256, 0, s>>>(prefix, ph, pw, m, n, to_grid(g), st, di, dj, map);
    return cudaGetLastError();
}

cudaError_t retained_count(const double* map, GridDesc g, double threshold,
                           unsigned long long* n_r, cudaStream_t s) {
    const size_t E = size_t(g.er) * g.ec;
    const int blocks = int(std::min<size_t>((E + 255) / 256, 148 * 16));
    k_retained<<<blocks, 256, 0, s>>>(map, to_grid(g), threshold, n_r);
    return cudaGetLastError();
}

}  // namespace tmk
