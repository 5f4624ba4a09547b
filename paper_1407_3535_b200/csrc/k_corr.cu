// k_corr.cu -- template correlation, scan-2 elimination and argmax (sm_100a).
//
// window_dot (detail.hpp:32-41) on 8-bit data is an exact integer <= 255^2*m*n, so the
// CUDA-core kernels accumulate u8*u8 products in FP32 FMA -- exact while a partial stays
// below 2^24, i.e. for flush_rows*n*255^2 < 2^24 -- and flush into FP64 every flush_rows
// template rows.  The dot therefore equals the reference's FP64 sum bit for bit, and the
// zncc_at epilogue (detail.hpp:45-51) is replayed with _rn intrinsics.
//
// corr_band: the dense engine.  A CTA owns a band of 8 output rows (taken from a row
// list, so centre rows at stride h work the same as consecutive rows) times NW*32 column
// indices at column stride SW.  Lane (ry, sx) = (lane/4, lane%4) owns 8 outputs of one row;
// it keeps a register window of (8-1)*SW+16 image values per 16-column template block so
// every staged float feeds 8 FMAs.  Template rows are staged IC at a time with the image
// rows they touch; the staged pitch is 4 mod 8 words so the 8 lanes of each LDS.128 phase
// hit 8 distinct bank groups (row strides are odd).
#include <algorithm>

#include "kernels.hpp"
#include "tm_common.cuh"

namespace tmk {

namespace {

constexpr int kRX = 8;   // outputs per lane
constexpr int kJB = 16;  // template columns per register block
constexpr int kIC = 8;   // template rows per shared-memory stage

__host__ __device__ constexpr int win_floats(int sw) { return (((kRX - 1) * sw + kJB) + 3) & ~3; }

__device__ __forceinline__ TStats to_ts(const TStatsH& h) {
    return TStats{h.mu, h.omega, h.mn, h.flat};
}

__device__ __forceinline__ void store_partial(const Cell& c, CellH* partials, int idx) {
    partials[idx] = CellH{c.rho, c.row, c.col, c.flags};
}

struct BandGeom {
    int spitch;  // staged floats per row (4 mod 8)
    int srows;   // staged rows
    size_t smem;
};

template <int SW, int NW>
__host__ BandGeom band_geom(int span_rows, int npad) {
    BandGeom g;
    const int width = (NW * 32 - 1) * SW + npad + 4;
    int pitch = (width + 3) & ~3;
    if (((pitch / 4) & 1) == 0) pitch += 4;
    g.spitch = pitch;
    g.srows = span_rows;
    g.smem = size_t(span_rows) * pitch * 4 + size_t(kIC) * npad * 4;
    return g;
}

template <int SW, int NW>
__global__ void __launch_bounds__(NW * 32)
    k_corr_band(CorrJob job, BandTask task, int spitch, int srows, CellH* partials) {
    extern __shared__ __align__(16) float sm[];
    float* simg = sm;
    float* stp = sm + size_t(srows) * spitch;
    __shared__ Cell scratch[NW];

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int ry = lane >> 2, sx = lane & 3;
    const int yb = blockIdx.y * 8;
    const int ylast = min(yb + 7, task.nrows - 1);
    const int yi = yb + ry;
    const bool row_ok = yi < task.nrows;
    const int r = task.rows[row_ok ? yi : ylast];
    const int r_first = task.rows[yb];
    const int span = task.rows[ylast] - r_first + kIC;
    const int kb = blockIdx.x * (NW * 32);
    const int cstart = task.cbase + kb * SW;
    const int width = (NW * 32 - 1) * SW + job.npad;
    const int lane_col = (wid * 32 + sx * kRX) * SW;  // staged column of output x=0
    const int yo = r - r_first;

    float acc[kRX];
    double dacc[kRX];
#pragma unroll
    for (int x = 0; x < kRX; ++x) {
        acc[x] = 0.f;
        dacc[x] = 0.0;
    }
    constexpr int W = win_floats(SW);
    const int p_rows = job.st.er + job.m - 1;  // image rows
    const int q_cols = job.st.ec + job.n - 1;

    // template-row slice of this CTA (K split across blockIdx.z)
    const int i_lo = blockIdx.z * task.ms, i_hi = min(job.m, i_lo + task.ms);
    for (int i0 = i_lo; i0 < i_hi; i0 += kIC) {
        __syncthreads();
        // stage image rows [r_first + i0, r_first + i0 + span), columns [cstart, +width):
        // one warp per row, 8 independent coalesced loads in flight per lane
        for (int a = wid; a < span; a += NW) {
            const int gr = r_first + i0 + a;
            const bool rok = gr < p_rows;
            const float* src = job.imgf + size_t(rok ? gr : 0) * job.pitch;
            float* dst = simg + a * spitch;
            for (int b0 = 0; b0 < width; b0 += 32 * 8) {
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int gc = cstart + b0 + u * 32 + lane;
                    v[u] = (rok && gc < q_cols) ? __ldg(src + gc) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int b = b0 + u * 32 + lane;
                    if (b < width) dst[b] = v[u];
                }
            }
        }
        for (int idx = threadIdx.x; idx < kIC * job.npad; idx += NW * 32) {
            const int a = idx / job.npad, b = idx - a * job.npad;
            stp[idx] = (i0 + a < i_hi) ? job.tf[size_t(i0 + a) * job.npad + b] : 0.f;
        }
        __syncthreads();
        const int nii = min(kIC, i_hi - i0);
        for (int ii = 0; ii < nii; ++ii) {
            const float* irow = simg + (yo + ii) * spitch + lane_col;
            const float* trow = stp + ii * job.npad;
            for (int jb = 0; jb < job.npad; jb += kJB) {
                float win[W];
#pragma unroll
                for (int v = 0; v < W / 4; ++v) {
                    const float4 t4 = *reinterpret_cast<const float4*>(irow + jb + 4 * v);
                    win[4 * v + 0] = t4.x;
                    win[4 * v + 1] = t4.y;
                    win[4 * v + 2] = t4.z;
                    win[4 * v + 3] = t4.w;
                }
                float tv[kJB];
#pragma unroll
                for (int v = 0; v < kJB / 4; ++v) {
                    const float4 t4 = *reinterpret_cast<const float4*>(trow + jb + 4 * v);
                    tv[4 * v + 0] = t4.x;
                    tv[4 * v + 1] = t4.y;
                    tv[4 * v + 2] = t4.z;
                    tv[4 * v + 3] = t4.w;
                }
#pragma unroll
                for (int j = 0; j < kJB; ++j)
#pragma unroll
                    for (int x = 0; x < kRX; ++x) acc[x] = fmaf(tv[j], win[x * SW + j], acc[x]);
            }
            if ((i0 + ii + 1 - i_lo) % job.flush_rows == 0) {
#pragma unroll
                for (int x = 0; x < kRX; ++x) {
                    dacc[x] += double(acc[x]);
                    acc[x] = 0.f;
                }
            }
        }
    }
#pragma unroll
    for (int x = 0; x < kRX; ++x) dacc[x] += double(acc[x]);

    const int k0 = kb + wid * 32 + sx * kRX;
    if (task.dot) {  // K split: exact integer partial dots accumulate in FP64
#pragma unroll
        for (int x = 0; x < kRX; ++x) {
            const int k = k0 + x;
            if (!row_ok || k >= task.nc) continue;
            const int c = task.cbase + k * SW;
            const size_t idx = task.mode == 1 ? size_t(task.yi_base + yi) * task.tc + task.col0 + k
                                              : size_t(r) * job.st.ec + c;
            atomicAdd(task.dot + idx, dacc[x]);
        }
        return;
    }
    // ---- epilogue ---------------------------------------------------------------------
    const TStats ts = to_ts(job.ts);
    Cell best = no_cell();
#pragma unroll
    for (int x = 0; x < kRX; ++x) {
        const int k = k0 + x;
        if (!row_ok || k >= task.nc) continue;
        const int c = task.cbase + k * SW;
        const size_t kk = size_t(r) * job.st.ec + c;
        if (task.mode == 2 && task.mask[kk] != 2) continue;
        const bool wflat = job.st.flat[kk];
        const double rho = zncc_epilogue(dacc[x], ts, job.st.mu[kk], job.st.omega[kk], wflat);
        const bool deg = ts.flat || wflat;
        if (task.mode == 1) {
            const size_t gi = size_t(task.yi_base + yi) * task.tc + task.col0 + k;
            task.out_rho[gi] = rho;
            task.out_deg[gi] = deg;
        } else if (task.out_rho) {
            task.out_rho[kk] = rho;
        }
        const Cell cand = make_cell(r, c, rho, deg);
        if (better(cand, best)) best = cand;
    }
    best = block_best(best, scratch);
    if (threadIdx.x == 0) store_partial(best, partials, blockIdx.y * gridDim.x + blockIdx.x);
}

// nblocks: blocks taking a ticket (default: the grid); n: partials to reduce (default tr.n)
__device__ void tail_reduce(const TailReduce& tr, Cell* scratch, unsigned nblocks = 0,
                            int n = -1);

// Epilogue of a K-split centre scan: rho/deg per group from the accumulated dots.
__global__ void __launch_bounds__(256)
    k_centre_epi(CorrJob job, Grid g, const int* __restrict__ rows, int cbase, int sw, int nc,
                 int col0, const double* __restrict__ dot, double* rho_c, uint8_t* deg_c,
                 CellH* partials, int c_last, TailReduce tail, const int* __restrict__ gate,
                 double* __restrict__ sa_out, float2* __restrict__ rec_out, CentreStats cs) {
    pdl_wait();
    if (gate && !*gate) return;  // speculative launch not confirmed (every block: no ticket)
    __shared__ Cell scratch[8];
    const TStats ts = to_ts(job.ts);
    Cell best = no_cell();
    const int nrows = g.ti_hi - g.ti_lo;
    const unsigned total = unsigned(nrows) * unsigned(nc);  // group count: < 2^32
    for (unsigned it = blockIdx.x * blockDim.x + threadIdx.x; it < total;
         it += gridDim.x * blockDim.x) {
        const unsigned yq = it / unsigned(nc);  // 32-bit division (a 64-bit one per centre
        const int yi = int(yq), k = int(it - yq * unsigned(nc));  // cost more than the epilogue)
        const int r = rows[yi];
        const int c = (c_last >= 0 && col0 + k == g.tc - 1) ? c_last : cbase + k * sw;
        const size_t gi = size_t(g.ti_lo + yi) * g.tc + col0 + k;
        const size_t kk = size_t(r) * job.st.ec + c;
        // a template batch reads the centres' statistics from compact per-group arrays
        // (gathered once for all templates: coalesced 17 B instead of ~51 B of sectors)
        const bool wflat = cs.mu ? cs.fl[gi] != 0 : job.st.flat[kk] != 0;
        const double mu_w = cs.mu ? cs.mu[gi] : job.st.mu[kk];
        const double om_w = cs.mu ? cs.om[gi] : job.st.omega[kk];
        const double rho = zncc_epilogue(dot[gi], ts, mu_w, om_w, wflat);
        const bool deg = ts.flat || wflat;
        rho_c[gi] = rho;
        deg_c[gi] = deg;
        if (sa_out || rec_out) {  // scan 2's centre half-gap factor (k_sqrt_gap, bounds.cpp:21-23)
            const double a = dclamp(rho, -1.0, 1.0);
            const double sa = __dsqrt_rn(dmax(0.0, __dsub_rn(1.0, __dmul_rn(a, a))));
            if (sa_out) sa_out[gi] = sa;
            // a template batch's record (k_sec_rows_multi): -1 marks a degenerate centre
            if (rec_out) rec_out[gi] = make_float2(float(a), deg ? -1.f : float(sa));
        }
        const Cell cand = make_cell(r, c, rho, deg);
        if (better(cand, best)) best = cand;
    }
    best = block_best(best, scratch);
    if (threadIdx.x == 0) store_partial(best, partials, blockIdx.x);
    tail_reduce(tail, scratch);
}

// The window statistics of every group centre, compacted per group (template batches).
__global__ void __launch_bounds__(256)
    k_gather_centre_stats(Grid g, DevStats st, double* __restrict__ mu_c,
                          double* __restrict__ om_c, uint8_t* __restrict__ fl_c) {
    pdl_wait();
    const size_t G0 = size_t(g.ti_lo) * g.tc, G1 = size_t(g.ti_hi) * g.tc;
    for (size_t gi = G0 + blockIdx.x * size_t(blockDim.x) + threadIdx.x; gi < G1;
         gi += size_t(gridDim.x) * blockDim.x) {
        const int ti = int(gi / size_t(g.tc)), tj = int(gi - size_t(ti) * g.tc);
        const size_t kk = size_t(g.center_row(ti)) * st.ec + g.center_col(tj);
        mu_c[gi] = st.mu[kk];
        om_c[gi] = st.omega[kk];
        fl_c[gi] = st.flat[kk];
    }
}

// ---- sparse: one warp per location ----------------------------------------------------
// The template is staged once per CTA in shared memory; lanes own template columns
// j = lane, lane+32, ...; the row loop is unrolled for memory-level parallelism.
__global__ void __launch_bounds__(256)
    k_corr_list(CorrJob job, const int2* __restrict__ locs, const unsigned long long* count,
                int max_count, double* out_rho, uint8_t* out_deg, CellH* partials,
                int lane_flush, int rho_by_loc, TailReduce tail) {
    pdl_wait();
    // One CTA per location (grid-stride): warp w owns template rows [w*m/8, (w+1)*m/8), so
    // a location costs one or two batches of independent loads per warp instead of m/8
    // dependent batches for a single warp.  Each lane's FP32 partials cover < lane_flush
    // rows of one column (exact); warp and block sums of these exact integers in FP64 are
    // order-independent.
    __shared__ Cell scratch[8];
    __shared__ double wsum[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long nloc = min((long long)*count, (long long)max_count);
    // only the blocks with a location take part (short lists: no empty blocks queueing on the
    // reduction ticket); without a fused reduction every block still writes its partial
    const int active = int(max(1LL, min((long long)gridDim.x, nloc)));
    if (int(blockIdx.x) >= active) {
        if (!tail.ticket && threadIdx.x == 0) store_partial(no_cell(), partials, blockIdx.x);
        return;
    }
    const TStats ts = to_ts(job.ts);
    const int rows_per = (job.m + 7) / 8;
    const int i_lo = min(job.m, wid * rows_per), i_hi = min(job.m, i_lo + rows_per);
    Cell best = no_cell();
    for (long long li = blockIdx.x; li < nloc; li += gridDim.x) {
        const int2 rc = locs[li];
        double dacc = 0.0;
        const uint8_t* ib = job.imgb + size_t(rc.x) * job.bpitch + rc.y;  // pixels as bytes
        for (int j = lane; j < job.n; j += 32) {
            const float* tp = job.tf + j;
            for (int i0 = i_lo; i0 < i_hi; i0 += 2 * lane_flush) {
                const int i1 = min(i_hi, i0 + 2 * lane_flush);
                float a0 = 0.f, a1 = 0.f;
                for (int i = i0; i < i1; i += 8) {
                    float v[8], t[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const bool ok = i + u < i1;
                        v[u] = ok ? float(__ldg(ib + size_t(i + u) * job.bpitch + j)) : 0.f;
                        t[u] = ok ? __ldg(tp + size_t(i + u) * job.npad) : 0.f;
                    }
#pragma unroll
                    for (int u = 0; u < 8; u += 2) {
                        a0 = fmaf(t[u], v[u], a0);
                        a1 = fmaf(t[u + 1], v[u + 1], a1);
                    }
                }
                dacc += double(a0) + double(a1);
            }
        }
        dacc = warp_sum(dacc);
        if (lane == 0) wsum[wid] = dacc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double d = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) d += wsum[w];
            const size_t kk = size_t(rc.x) * job.st.ec + rc.y;
            const bool wflat = job.st.flat[kk];
            const double rho = zncc_epilogue(d, ts, job.st.mu[kk], job.st.omega[kk], wflat);
            if (out_rho) out_rho[rho_by_loc ? kk : li] = rho;
            if (out_deg) out_deg[li] = ts.flat || wflat;
            const Cell cand = make_cell(rc.x, rc.y, rho, ts.flat || wflat);
            if (better(cand, best)) best = cand;
        }
        __syncthreads();
    }
    best = block_best(best, scratch);
    if (threadIdx.x == 0) store_partial(best, partials, blockIdx.x);
    tail_reduce(tail, scratch, unsigned(active), tail.n - int(gridDim.x) + active);
}

// ---- FP64 replica (non-integer images / templates) --------------------------------------
__device__ __forceinline__ double dot_f64(const CorrJob& job, int r, int c) {
    double acc = 0.0;
    for (int i = 0; i < job.m; ++i) {
        const double* pt = job.td + size_t(i) * job.n;
        const double* pi = job.imgd + size_t(r + i) * job.q + c;
        for (int j = 0; j < job.n; ++j) acc = __dadd_rn(acc, __dmul_rn(pt[j], pi[j]));
    }
    return acc;
}

// The same sum by a whole CTA, for SHORT lists (a single thread's replay of m*n dependent
// loads takes ~1 ms at 128x128): the products t*I are independent, only the additions must
// run in window_dot's order.  Warps 1.. fill a shared-memory chunk of products (rounded once,
// like the reference's pt[j] * pi[j]) while thread 0 adds the previous chunk in sequence.
// Returns the dot in thread 0.
constexpr int kF64Chunk = 2048;
__device__ double dot_f64_cta(const CorrJob& job, int r, int c, double (*buf)[kF64Chunk]) {
    const int total = job.m * job.n;
    const int nch = (total + kF64Chunk - 1) / kF64Chunk;
    const int tid = threadIdx.x;
    auto fill = [&](int k, int first, int step) {
        const int e0 = k * kF64Chunk, e1 = min(total, e0 + kF64Chunk);
        for (int e = e0 + first; e < e1; e += step) {
            const int i = e / job.n, j = e - i * job.n;
            buf[k & 1][e - e0] =
                __dmul_rn(job.td[e], job.imgd[size_t(r + i) * job.q + c + j]);
        }
    };
    fill(0, tid, blockDim.x);
    __syncthreads();
    double acc = 0.0;
    for (int k = 0; k < nch; ++k) {
        if (tid >= 32) {
            if (k + 1 < nch) fill(k + 1, tid - 32, blockDim.x - 32);
        } else if (tid == 0) {
            const double* b = buf[k & 1];
            const int cnt = min(kF64Chunk, total - k * kF64Chunk);
            int e = 0;
            for (; e + 8 <= cnt; e += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = b[e + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
            }
            for (; e < cnt; ++e) acc = __dadd_rn(acc, b[e]);
        }
        __syncthreads();
    }
    return acc;
}

__global__ void __launch_bounds__(256)
    k_list_f64(CorrJob job, const int2* __restrict__ locs, const unsigned long long* count,
               int max_count, double* out_rho, uint8_t* out_deg, CellH* partials,
               int rho_by_loc) {
    __shared__ Cell scratch[8];
    __shared__ double prod[2][kF64Chunk];
    const long long nloc = min((long long)*count, (long long)max_count);
    const TStats ts = to_ts(job.ts);
    Cell best = no_cell();
    if (nloc <= 16ll * gridDim.x) {  // short list: one CTA per location
        for (long long li = blockIdx.x; li < nloc; li += gridDim.x) {
            const int2 rc = locs[li];
            const size_t kk = size_t(rc.x) * job.st.ec + rc.y;
            const bool wflat = job.st.flat[kk];
            const bool deg = ts.flat || wflat;
            const double dot = deg ? 0.0 : dot_f64_cta(job, rc.x, rc.y, prod);  // block-uniform
            if (threadIdx.x == 0) {
                const double rho =
                    deg ? 0.0 : zncc_epilogue(dot, ts, job.st.mu[kk], job.st.omega[kk], wflat);
                if (out_rho) out_rho[rho_by_loc ? kk : li] = rho;
                if (out_deg) out_deg[li] = deg;
                const Cell cand = make_cell(rc.x, rc.y, rho, deg);
                if (better(cand, best)) best = cand;
            }
        }
        best = block_best(best, scratch);
        if (threadIdx.x == 0) store_partial(best, partials, blockIdx.x);
        return;
    }
    for (long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x; li < nloc;
         li += (long long)gridDim.x * blockDim.x) {
        const int2 rc = locs[li];
        const size_t kk = size_t(rc.x) * job.st.ec + rc.y;
        const bool wflat = job.st.flat[kk];
        const double rho = (ts.flat || wflat)
                               ? 0.0
                               : zncc_epilogue(dot_f64(job, rc.x, rc.y), ts, job.st.mu[kk],
                                               job.st.omega[kk], wflat);
        if (out_rho) out_rho[rho_by_loc ? kk : li] = rho;
        if (out_deg) out_deg[li] = ts.flat || wflat;
        const Cell cand = make_cell(rc.x, rc.y, rho, ts.flat || wflat);
        if (better(cand, best)) best = cand;
    }
    best = block_best(best, scratch);
    if (threadIdx.x == 0) store_partial(best, partials, blockIdx.x);
}

__global__ void __launch_bounds__(256)
    k_dense_f64(CorrJob job, double* surface, CellH* partials) {
    __shared__ Cell scratch[8];
    const long long E = (long long)job.st.er * job.st.ec;
    const TStats ts = to_ts(job.ts);
    Cell best = no_cell();
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < E;
         k += (long long)gridDim.x * blockDim.x) {
        const int r = int(k / job.st.ec), c = int(k % job.st.ec);
        const bool wflat = job.st.flat[k];
        const double rho = (ts.flat || wflat) ? 0.0
                                              : zncc_epilogue(dot_f64(job, r, c), ts, job.st.mu[k],
                                                              job.st.omega[k], wflat);
        if (surface) surface[k] = rho;
        const Cell cand = make_cell(r, c, rho, ts.flat || wflat);
        if (better(cand, best)) best = cand;
    }
    best = block_best(best, scratch);
    if (threadIdx.x == 0) store_partial(best, partials, blockIdx.x);
}

// ---- reductions -----------------------------------------------------------------------
// The best cell of a phase -> *out, then the phase's follow-up (thread 0).
__device__ void apply_reduce_op(const Cell& best, CellH* out, const ReduceOp& op) {
    const CellH b{best.rho, best.row, best.col, best.flags};
    out[0] = b;
    if (op.kind == 1) {  // k_threshold_init + the zeroing the search needs next
        double t = -INFINITY;
        if ((b.flags & 1) && !(b.flags & 2)) t = b.rho;
        if (op.has_init) t = dmax(t, dclamp(op.init, -1.0, 1.0));
        *op.thr = t;
        for (int i = 0; i < op.nzero64; ++i) op.zero64[i] = 0ull;
        if (op.zero_tally) *op.zero_tally = Tally{0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
        if (op.egs_stop) {  // k_egs_init
            *op.egs_stop = 0;
            *op.egs_prev = INFINITY;
            for (int i = 0; i < 4; ++i) op.egs_nr4[i] = 0ull;
            *op.egs_hacc = 0;
            *op.egs_gate = 0ull;
        }
    } else if (op.kind == 2) {  // k_threshold_raise
        if ((b.flags & 1) && !(b.flags & 2) && b.rho > *op.thr) *op.thr = b.rho;
    } else if (op.kind == 3) {  // result block for one device->host copy
        for (int i = 0; i < 3; ++i) op.packed->cells[i] = op.cells[i];
        op.packed->cells[2] = b;  // this reduction's own slot (cells[2])
        op.packed->tally = *op.tally;
        op.packed->thr = *op.thr;
    }
}

__global__ void k_reduce_cells(const CellH* __restrict__ partials, int n, CellH* out, ReduceOp op) {
    pdl_wait();
    __shared__ Cell scratch[32];
    Cell best = no_cell();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const CellH h = partials[i];
        const Cell c{h.rho, h.row, h.col, h.flags};
        if (better(c, best)) best = c;
    }
    best = block_best(best, scratch);
    if (threadIdx.x == 0) apply_reduce_op(best, out, op);
}

// Fused tail reduction (TailReduce): called by every thread of every block after the
// block's partial is stored.  The last block to take a ticket reads all partials through
// L2 (other SMs wrote them) and finishes the phase like k_reduce_cells.
__device__ void tail_reduce(const TailReduce& tr, Cell* scratch, unsigned nblocks, int n) {
    if (!tr.ticket) return;  // uniform
    if (nblocks == 0) nblocks = gridDim.x * gridDim.y * gridDim.z;
    const int nred = n >= 0 ? n : tr.n;
    __shared__ int is_last;
    if (threadIdx.x == 0) {  // thread 0 stored this block's partial: publish it, take a ticket
        __threadfence();
        is_last = atomicAdd(tr.ticket, 1u) == nblocks - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    Cell best = no_cell();
    // all of a thread's partials loaded before any comparison (one L2 latency, not n/blockDim)
    constexpr int kU = 4;
    for (int i0 = threadIdx.x; i0 < nred; i0 += kU * blockDim.x) {
        Cell c[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = i0 + u * blockDim.x;
            c[u] = no_cell();
            if (i < nred) {
                const CellH* h = tr.partials + i;
                c[u] = Cell{__ldcg(&h->rho), __ldcg(&h->row), __ldcg(&h->col), __ldcg(&h->flags)};
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (better(c[u], best)) best = c[u];
    }
    best = block_best(best, scratch);
    const ReduceOp& op = tr.op;
    if (op.kind == 3) {  // pack the result block with several threads (independent copies)
        const int t = threadIdx.x;
        if (t == 0) {
            const CellH b{best.rho, best.row, best.col, best.flags};
            tr.out[0] = b;
            op.packed->cells[2] = b;
            *tr.ticket = 0u;
        } else if (t <= 2) {
            op.packed->cells[t - 1] = op.cells[t - 1];
        } else if (t == 3) {
            op.packed->tally = *op.tally;
        } else if (t == 4) {
            op.packed->thr = *op.thr;
        }
        return;
    }
    if (threadIdx.x == 0) {
        apply_reduce_op(best, tr.out, tr.op);
        *tr.ticket = 0u;
    }
}

__global__ void k_egs_init(int* stop, double* prev, unsigned long long* nr4, int* h_acc,
                           unsigned long long* gate) {
    pdl_wait();
    *stop = 0;
    *prev = INFINITY;
    for (int i = 0; i < 4; ++i) nr4[i] = 0ull;
    if (h_acc) *h_acc = 0;
    if (gate) *gate = 0ull;
}

// ---- scan 2: SEC test + survivor compaction (matcher.cpp:48-78, bounds.cpp:41-46) -------
__global__ void __launch_bounds__(256)
    k_sec_compact(Grid g, const double* __restrict__ map, const double* __restrict__ rho_c,
                  const uint8_t* __restrict__ deg_c, const uint8_t* __restrict__ flat, int tflat,
                  const double* __restrict__ thr_ptr, const uint8_t* __restrict__ seeded,
                  int2* locs, unsigned long long max_locs, Tally* tally, uint8_t* visits) {
    const double T = *thr_ptr;
    const double tb = dmin(T, 1.0);
    const size_t K0 = size_t(g.row_lo()) * g.ec, E = size_t(g.row_hi()) * g.ec;
    const int lane = threadIdx.x & 31;
    unsigned long long n_elim = 0, n_keep = 0;
    for (size_t base = K0 + blockIdx.x * size_t(blockDim.x); base < E;
         base += size_t(gridDim.x) * blockDim.x) {
        const size_t k = base + threadIdx.x;
        bool survivor = false;
        int r = 0, c = 0;
        if (k < E) {
            g.rc(k, r, c);
            const int ti = g.tile_r(r), tj = g.tile_c(c);
            const bool centre = g.center_row(ti) == r && g.center_col(tj) == c;
            if (centre) {
                if (visits) visits[k] = 0;
            } else {
                const size_t gi = size_t(ti) * g.tc + tj;
                if (seeded && seeded[gi]) {
                    ++n_keep;  // evaluated by the seeding pass
                    if (visits) visits[k] = 2;
                } else {
                    const bool mflat = tflat || flat[k];
                    const bool elim =
                        !deg_c[gi] && !mflat && T >= -1.0 && sec_holds(tb, rho_c[gi], map[k]);
                    if (elim) {
                        ++n_elim;
                        if (visits) visits[k] = 1;
                    } else {
                        ++n_keep;
                        survivor = true;
                        if (visits) visits[k] = 2;
                    }
                }
            }
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, survivor);
        if (ballot) {
            unsigned long long basepos = 0;
            if (lane == 0) basepos = atomicAdd(&tally->survivors, (unsigned long long)__popc(ballot));
            basepos = __shfl_sync(0xffffffffu, basepos, 0);
            if (survivor) {
                const unsigned long long pos = basepos + __popc(ballot & ((1u << lane) - 1));
                if (pos < max_locs) locs[pos] = make_int2(r, c);
            }
        }
    }
    n_elim = warp_sum(n_elim);
    n_keep = warp_sum(n_keep);
    if (lane == 0) {
        if (n_elim) atomicAdd(&tally->eliminated, n_elim);
        if (n_keep) atomicAdd(&tally->retained, n_keep);
    }
}

// The member bound test of scan 2, tb >= RN(RN(a*b) + RN(sa * RN(sqrt(x)))) with
// x = RN(1 - RN(b*b)) in [0, 1] and sa in [0, 1] (bounds.cpp:21-23, 41-46), decided from an
// FP32 square root (sqrt.approx.f32: relative error < 2^-21 after the conversions) unless
// tb lies within 4e-6 of the approximate bound: the exact bound differs from it by at most
// sa * |sqrt(x) - approx| + a few FP64 ulps < 1e-6, so outside that band the decision is
// the exact one; inside it the exact FP64 expression decides.
__device__ __forceinline__ bool sec_test_fast(double tb, double a, double b, double sa, double x) {
    float sf;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(sf) : "f"(__double2float_rn(x)));
    const double ab = __dmul_rn(a, b);
    const double approx = __dadd_rn(ab, __dmul_rn(sa, double(sf)));
    if (tb >= __dadd_rn(approx, 4e-6)) return true;
    if (tb < __dsub_rn(approx, 4e-6)) return false;
    return tb >= __dadd_rn(ab, __dmul_rn(sa, __dsqrt_rn(x)));
}

// Scan 2 over explicit extent rows: row-level quantities (group row, centre row) once per
// row, the centre's half_gap factor sa precomputed per group (k_sqrt_gap, same
// operations as half_gap), so a member costs one FastDiv, its own square root and the
// bound test.  Same decisions, counts, visit codes and survivor list as k_sec_compact.
__global__ void __launch_bounds__(256)
    k_sec_rows(Grid g, const double* __restrict__ map, const double* __restrict__ rho_c,
               const double* __restrict__ sa_c, const uint8_t* __restrict__ deg_c,
               const uint8_t* __restrict__ flat, int tflat, const double* __restrict__ thr_ptr,
               const uint8_t* __restrict__ seeded, int2* locs, unsigned long long max_locs,
               Tally* tally, uint8_t* visits, TileFlags tf) {
    pdl_wait();
    const double T = *thr_ptr;
    const double tb = dclamp(dmin(T, 1.0), -1.0, 1.0);
    const bool thr_ok = T >= -1.0;
    const int lane = threadIdx.x & 31;
    unsigned long long n_elim = 0, n_keep = 0, n_flat = 0, fkey = 0;
    bool list_full = false;            // this warp saw the survivor list reach max_locs
    unsigned long long surv_local = 0;  // survivors counted after that (one atomic at the end)
    const int r_lo = g.row_lo(), r_hi = g.row_hi();
    const int cols = ((g.ec + 31) / 32) * 32;  // whole warps per row (ballots)
    for (int r = r_lo + blockIdx.x; r < r_hi; r += gridDim.x) {
        const int ti = g.tile_r(r);
        const bool centre_row = g.center_row(ti) == r;
        const size_t rowk = size_t(r) * g.ec;
        const size_t gbase = size_t(ti) * g.tc;
        // software pipeline: every load of the next column is in flight while this one is
        // tested (one memory latency per two columns, not a chain through the tests)
        struct Elem {
            double mv, ra, sa;
            uint8_t fv, sd, dg;
            int tj;
        };
        auto load = [&](int c, Elem& e) {
            const bool in = c < g.ec;
            const size_t k = rowk + (in ? c : 0);
            e.tj = g.tile_c(in ? c : 0);
            const size_t gi = gbase + e.tj;
            e.mv = __ldg(map + k);
            e.fv = __ldg(flat + k);
            e.sd = seeded ? __ldg(seeded + gi) : uint8_t(0);
            e.dg = __ldg(deg_c + gi);
            e.ra = __ldg(rho_c + gi);
            e.sa = __ldg(sa_c + gi);
        };
        Elem cur;
        load(threadIdx.x, cur);
        for (int c = threadIdx.x; c < cols; c += blockDim.x) {
            Elem nxt = cur;
            if (c + int(blockDim.x) < cols) load(c + blockDim.x, nxt);
            bool survivor = false;
            if (c < g.ec) {
                const size_t k = rowk + c;
                const int tj = cur.tj;
                const double mv = cur.mv, ra = cur.ra, sa = cur.sa;
                const uint8_t fv = cur.fv, sd = cur.sd, dg = cur.dg;
                if (centre_row && g.center_col(tj) == c) {
                    if (visits) visits[k] = 0;
                } else {
                    if (sd) {
                        ++n_keep;
                        if (visits) visits[k] = 2;
                    } else {
                        bool elim = thr_ok && !dg && !(tflat || fv);
                        if (elim) {
                            const double a = dclamp(ra, -1.0, 1.0);
                            const double b = dclamp(mv, -1.0, 1.0);
                            const double x = dmax(0.0, __dsub_rn(1.0, __dmul_rn(b, b)));
                            elim = sec_test_fast(tb, a, b, sa, x);
                        }
                        if (elim) {
                            ++n_elim;
                            if (visits) visits[k] = 1;
                        } else if (tflat || fv) {  // retained, rho 0 without a dot
                            ++n_keep;
                            ++n_flat;
                            fkey = max(fkey, flat_member_key(r, c));
                            if (visits) visits[k] = 2;
                        } else {
                            ++n_keep;
                            survivor = true;
                            if (visits) visits[k] = 2;
                            mark_tile(tf, r, c);
                        }
                    }
                }
            }
            const unsigned ballot = __ballot_sync(0xffffffffu, survivor);
            if (ballot) {
                if (list_full) {  // nothing more can be listed: count only (no atomics)
                    surv_local += __popc(ballot);
                } else {
                    unsigned long long basepos = 0;
                    if (lane == 0)
                        basepos = atomicAdd(&tally->survivors, (unsigned long long)__popc(ballot));
                    basepos = __shfl_sync(0xffffffffu, basepos, 0);
                    list_full = basepos + __popc(ballot) >= max_locs;  // warp-uniform
                    if (survivor) {
                        const unsigned long long pos = basepos + __popc(ballot & ((1u << lane) - 1));
                        if (pos < max_locs) locs[pos] = make_int2(r, c);
                    }
                }
            }
            cur = nxt;
        }
    }
    n_elim = warp_sum(n_elim);
    n_keep = warp_sum(n_keep);
    n_flat = warp_sum(n_flat);
    fkey = warp_max_u64(fkey);
    if (lane == 0) {
        if (n_elim) atomicAdd(&tally->eliminated, n_elim);
        if (n_keep) atomicAdd(&tally->retained, n_keep);
        if (surv_local) atomicAdd(&tally->survivors, surv_local);
        if (n_flat) {
            atomicAdd(&tally->flat_n, n_flat);
            atomicMax(&tally->flat_key, fkey);
        }
    }
}

// Scan 2 for a batch of K templates on one preparation (cmd_bench's loop, cli.cpp:213-237,
// as one pass): every member's R_co, flat flag and half-gap factor are read and formed ONCE
// for all templates, with the same decisions as k_sec_rows per template.  Thread = member;
// the K templates are an unrolled loop (KP = K rounded up to a power of two) with the
// counters in registers; group-level scan-1 values are per-template planes [K][G] (the
// lanes of a warp read a few consecutive groups of one plane); visit codes go to plane k
// (the dense pass's mask); survivor lists are warp-aggregated (one atomic per warp and
// template that has survivors).
// The exact FP64 bound test of k_sec_rows (inside the fast test's margin; rare): out of
// line so the unrolled template loop stays small.
__device__ __noinline__ bool sec_exact_multi(const SecMulti& sm, int k, size_t gk, double b,
                                             double x) {
    const double T = sm.thr[k];
    const double tb = dclamp(dmin(T, 1.0), -1.0, 1.0);
    const double a = dclamp(sm.rho_c[gk], -1.0, 1.0);
    return tb >= __dadd_rn(__dmul_rn(a, b), __dmul_rn(sm.sa_c[gk], __dsqrt_rn(x)));
}

template <int KP>
__global__ void __launch_bounds__(256)
    k_sec_rows_multi(Grid g, const double* __restrict__ map, const uint8_t* __restrict__ flat,
                     SecMulti sm) {
    pdl_wait();
    // rarely-updated per-template counters (flat members, survivors past a full list) are
    // block-level in shared memory; every member is either eliminated or kept, so a thread
    // counts its members once and its eliminations per template in registers
    __shared__ unsigned long long s_flat[KP], s_fkey[KP], s_surv[KP];
    for (int k = threadIdx.x; k < KP; k += blockDim.x) s_flat[k] = s_fkey[k] = s_surv[k] = 0ull;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned n_elim[KP];
    float tbf[KP];  // clamped thresholds (FP32 decision; the FP64 one inside the margin)
    unsigned thr_ok = 0u;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
        n_elim[k] = 0u;
        const double T = k < sm.K ? sm.thr[k] : -2.0;
        tbf[k] = float(dclamp(dmin(T, 1.0), -1.0, 1.0));
        if (T >= -1.0) thr_ok |= 1u << k;
    }
    unsigned members = 0;
    unsigned full = 0u;  // templates whose list this warp saw fill up
    const int r_lo = g.row_lo(), r_hi = g.row_hi();
    const int cols = ((g.ec + 31) / 32) * 32;
    for (int r = r_lo + blockIdx.x; r < r_hi; r += gridDim.x) {
        const int ti = g.tile_r(r);
        const bool centre_row = g.center_row(ti) == r;
        const size_t rowk = size_t(r) * g.ec;
        const size_t gbase = size_t(ti) * g.tc;
        for (int c = threadIdx.x; c < cols; c += blockDim.x) {
            const bool in = c < g.ec;
            const size_t kk = rowk + (in ? c : 0);
            const int tj = g.tile_c(in ? c : 0);
            const size_t gi = gbase + tj;
            const bool member = in && !(centre_row && g.center_col(tj) == c);
            members += member;
            const double b = member ? dclamp(__ldg(map + kk), -1.0, 1.0) : 0.0;
            const bool fv = member && __ldg(flat + kk) != 0;
            const double x = dmax(0.0, __dsub_rn(1.0, __dmul_rn(b, b)));
            float sq;
            asm("sqrt.approx.f32 %0, %1;" : "=f"(sq) : "f"(__double2float_rn(x)));
            const float bf = float(b);
            // every template's group record first (independent loads, one latency)
            float2 rec[KP];
#pragma unroll
            for (int k = 0; k < KP; ++k)
                rec[k] = k < sm.K ? __ldg(sm.rec + size_t(k) * sm.G + gi) : make_float2(0.f, -2.f);
            // member: seeded group -> kept (evaluated already); else eliminated iff the bound
            // holds (FP32 with a 4e-6 margin, FP64 inside it); kept flat members are not
            // listed (rho 0 without a dot).  Branch-free per template: bit masks of the
            // certain eliminations, of the templates inside the margin (decided exactly after
            // the loop; rare) and of the seeded groups.
            unsigned el = 0u, amb = 0u, sd = 0u;
            const bool testable = member && !fv;
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const float ry = rec[k].y;  // -1 degenerate centre, -2 seeded group (or k >= K)
                const float f = fmaf(rec[k].x, bf, ry * sq);
                const bool t = testable && ry >= 0.f && ((thr_ok >> k) & 1u);
                const bool sure = tbf[k] >= f + 4e-6f;
                const bool maybe = !sure && tbf[k] >= f - 4e-6f;
                if (t && sure) el |= 1u << k;  // (predicated ORs with an immediate)
                if (t && maybe) amb |= 1u << k;
                if (ry == -2.f) sd |= 1u << k;
            }
            while (amb) {  // inside the FP32 margin: the exact FP64 bound test
                const int k = __ffs(amb) - 1;
                amb &= amb - 1u;
                if (sec_exact_multi(sm, k, size_t(k) * sm.G + gi, b, x)) el |= 1u << k;
            }
            const unsigned kmask = sm.K >= 32 ? 0xffffffffu : (1u << sm.K) - 1u;
            const unsigned listed = member ? (~el & ~sd & kmask) : 0u;  // kept, not seeded
            const unsigned smask = fv ? 0u : listed, fmask = fv ? listed : 0u;
            if (in && sm.visits) {
                uint8_t* vp = sm.visits + kk;
                const unsigned base = member ? 2u : 0u;  // el is 0 for a non-member
#pragma unroll
                for (int k = 0; k < KP; ++k) {
                    if (k >= sm.K) break;
                    *vp = uint8_t(base - ((el >> k) & 1u));  // 2 kept, 1 eliminated, 0 centre
                    vp += sm.E;
                }
            }
#pragma unroll
            for (int k = 0; k < KP; ++k) n_elim[k] += (el >> k) & 1u;
            // templates with a survivor / kept flat member in this warp (warp-uniform mask):
            // only those are visited (weak templates of a batch keep most warps busy here,
            // the others never)
            unsigned todo = __reduce_or_sync(0xffffffffu, smask | fmask);
            {
#pragma unroll 1
                while (todo) {
                    const int k = __ffs(todo) - 1;
                    todo &= todo - 1u;
                    const bool fk = (fmask >> k) & 1u, sk = (smask >> k) & 1u;
                    const unsigned bfl = __ballot_sync(0xffffffffu, fk);
                    if (bfl) {
                        const unsigned long long key =
                            warp_max_u64(fk ? flat_member_key(r, c) : 0ull);
                        if (lane == 0) {
                            atomicAdd(&s_flat[k], (unsigned long long)__popc(bfl));
                            atomicMax(&s_fkey[k], key);
                        }
                    }
                    const unsigned ball = __ballot_sync(0xffffffffu, sk);
                    if (!ball) continue;
                    if (sk && sm.tf.p)
                        mark_tile(TileFlags{sm.tf.p + size_t(k) * sm.tf_stride, sm.tf.cols}, r, c);
                    if ((full >> k) & 1u) {
                        if (lane == 0) atomicAdd(&s_surv[k], (unsigned long long)__popc(ball));
                        continue;
                    }
                    unsigned long long base = 0;
                    if (lane == 0)
                        base = atomicAdd(&sm.tally[k].survivors, (unsigned long long)__popc(ball));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (sk) {
                        const unsigned long long pos = base + __popc(ball & ((1u << lane) - 1));
                        if (pos < sm.cap) sm.locs[size_t(k) * sm.cap + pos] = make_int2(r, c);
                    }
                    if (base + __popc(ball) >= sm.cap) full |= 1u << k;
                }
            }
        }
    }
    const unsigned long long nm = warp_sum((unsigned long long)members);
#pragma unroll
    for (int k = 0; k < KP; ++k) {
        if (k >= sm.K) break;
        const unsigned long long ne = warp_sum((unsigned long long)n_elim[k]);
        if (lane == 0) {
            if (ne) atomicAdd(&sm.tally[k].eliminated, ne);
            if (nm - ne) atomicAdd(&sm.tally[k].retained, nm - ne);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < sm.K; k += blockDim.x) {
        Tally* t = sm.tally + k;
        if (s_surv[k]) atomicAdd(&t->survivors, s_surv[k]);
        if (s_flat[k]) {
            atomicAdd(&t->flat_n, s_flat[k]);
            atomicMax(&t->flat_key, s_fkey[k]);
        }
    }
}

// One template's batch record per group: {float(clamp(rho_c)), float(sa_c)}, the flags in
// the (otherwise non-negative) second field: -1 degenerate centre, -2 seeded group.
__global__ void k_batch_records(const double* __restrict__ rho_c, const double* __restrict__ sa_c,
                                const uint8_t* __restrict__ deg_c,
                                const uint8_t* __restrict__ seeded, size_t G,
                                float2* __restrict__ rec) {
    pdl_wait();
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < G;
         i += size_t(gridDim.x) * blockDim.x) {
        const float sa = seeded && seeded[i] ? -2.f : (deg_c[i] ? -1.f : float(sa_c[i]));
        rec[i] = make_float2(float(dclamp(rho_c[i], -1.0, 1.0)), sa);
    }
}

// y = sqrt(max(0, 1 - clamp(x)^2)): one factor of half_gap (bounds.cpp:21-23).
__global__ void k_sqrt_gap(const double* __restrict__ x, double* __restrict__ y, size_t n) {
    pdl_wait();
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const double a = dclamp(x[i], -1.0, 1.0);
        y[i] = __dsqrt_rn(dmax(0.0, __dsub_rn(1.0, __dmul_rn(a, a))));
    }
}

__global__ void k_threshold_init(const CellH* best, int has_init, double init, double* thr) {
    double t = -INFINITY;
    const CellH b = *best;
    if ((b.flags & 1) && !(b.flags & 2)) t = b.rho;
    if (has_init) t = dmax(t, dclamp(init, -1.0, 1.0));
    *thr = t;
}

__global__ void k_threshold_raise(const CellH* best, double* thr) {
    const CellH b = *best;
    if ((b.flags & 1) && !(b.flags & 2) && b.rho > *thr) *thr = b.rho;
}

// Seeded policy: every group whose centre rho is within `margin` of the best centre is
// searched exhaustively first; its best member raises the threshold before scan 2.
__global__ void k_seed_members(Grid g, const double* __restrict__ rho_c,
                               const uint8_t* __restrict__ deg_c, const double* thr,
                               double margin, uint8_t* seeded, int2* locs,
                               unsigned long long* count, unsigned long long max_locs,
                               unsigned long long* n_groups, unsigned long long max_groups,
                               float2* rec) {
    pdl_wait();
    const long long G = (long long)g.ti_hi * g.tc;
    const double T = *thr;
    for (long long gi = (long long)g.ti_lo * g.tc + blockIdx.x * (long long)blockDim.x + threadIdx.x;
         gi < G; gi += (long long)gridDim.x * blockDim.x) {
        seeded[gi] = 0;
        if (deg_c[gi] || !(rho_c[gi] >= T - margin)) continue;
        const unsigned long long slot = atomicAdd(n_groups, 1ull);
        if (slot >= max_groups) continue;
        const int ti = int(gi / g.tc), tj = int(gi % g.tc);
        const int r0 = ti * g.h, r1 = min(r0 + g.h, g.er) - 1;
        const int c0 = tj * g.w, c1 = min(c0 + g.w, g.ec) - 1;
        const int cr = (r0 + r1) >> 1, cc = (c0 + c1) >> 1;
        const unsigned long long nm = (unsigned long long)(r1 - r0 + 1) * (c1 - c0 + 1) - 1;
        const unsigned long long pos = atomicAdd(count, nm);
        if (pos + nm > max_locs) continue;
        seeded[gi] = 1;
        if (rec) rec[gi].y = -2.f;  // a template batch's record: a seeded group
        unsigned long long o = pos;
        for (int r = r0; r <= r1; ++r)
            for (int c = c0; c <= c1; ++c)
                if (r != cr || c != cc) locs[o++] = make_int2(r, c);
    }
}

// ---- sequential policy (matcher.cpp:48-78 with running_update): exact replay ----------
// Scan order key of a member: group index * (h*w) + row-major offset inside its tile.
__device__ __forceinline__ unsigned long long scan_key(const Grid& g, int r, int c) {
    const int ti = g.tile_r(r), tj = g.tile_c(c);
    return ((unsigned long long)ti * g.tc + tj) * (unsigned long long)(g.h * g.w) +
           (unsigned long long)((r - ti * g.h) * g.w + (c - tj * g.w));
}

__device__ __forceinline__ bool alive_at(const Grid& g, int r, int c, double T,
                                         const double* map, const double* rho_c,
                                         const uint8_t* deg_c, const uint8_t* flat, int tflat) {
    const size_t k = size_t(r) * g.ec + c;
    const size_t gi = size_t(g.tile_r(r)) * g.tc + g.tile_c(c);
    const bool mflat = tflat || flat[k];
    if (deg_c[gi] || mflat || !(T >= -1.0)) return true;
    return !sec_holds(dmin(T, 1.0), rho_c[gi], map[k]);
}

// First (in scan order, key > after) candidate that is alive at T and sets a new record.
__global__ void k_first_record(Grid g, const int2* __restrict__ locs,
                               const unsigned long long* count, const double* __restrict__ rho,
                               const double* map,
                               const double* rho_c, const uint8_t* deg_c, const uint8_t* flat,
                               int tflat, double T, unsigned long long after,
                               unsigned long long* best_key) {
    const unsigned long long n = *count;
    unsigned long long mine = ~0ull;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const int2 rc = locs[i];
        const size_t kk = size_t(rc.x) * g.ec + rc.y;
        if (tflat || flat[kk] || !(rho[kk] > T)) continue;
        const unsigned long long key = scan_key(g, rc.x, rc.y);
        if ((after != ~0ull && key <= after) || key >= mine) continue;
        if (alive_at(g, rc.x, rc.y, T, map, rho_c, deg_c, flat, tflat)) mine = key;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) mine = min(mine, __shfl_xor_sync(0xffffffffu, mine, s));
    if ((threadIdx.x & 31) == 0 && mine != ~0ull) atomicMin(best_key, mine);
}

__global__ void k_fetch_rho(Grid g, const int2* __restrict__ locs, const unsigned long long* count,
                            const double* __restrict__ rho, unsigned long long key, double* out) {
    const unsigned long long n = *count;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const int2 rc = locs[i];
        if (scan_key(g, rc.x, rc.y) == key) *out = rho[size_t(rc.x) * g.ec + rc.y];
    }
}

// Final pass: each candidate sees the threshold of the last record before it.
__global__ void k_seq_final(Grid g, const int2* __restrict__ locs, const unsigned long long* count,
                            const double* __restrict__ rho, const double* map, const double* rho_c, const uint8_t* deg_c,
                            const uint8_t* flat, int tflat, double T0,
                            const unsigned long long* __restrict__ rec_key,
                            const double* __restrict__ rec_T, int n_rec, Tally* tally,
                            uint8_t* visits, CellH* partials) {
    __shared__ Cell scratch[8];
    const unsigned long long n = *count;
    unsigned long long dead = 0, alive = 0;
    Cell best = no_cell();
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const int2 rc = locs[i];
        const unsigned long long key = scan_key(g, rc.x, rc.y);
        // threshold in effect: last record with rec_key < key (records sorted ascending)
        int lo = 0, hi = n_rec;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (rec_key[mid] < key) lo = mid + 1; else hi = mid;
        }
        const double T = lo == 0 ? T0 : rec_T[lo - 1];
        if (alive_at(g, rc.x, rc.y, T, map, rho_c, deg_c, flat, tflat)) {
            ++alive;
            const size_t kk = size_t(rc.x) * g.ec + rc.y;
            const Cell cand = make_cell(rc.x, rc.y, rho[kk], tflat || flat[kk]);
            if (better(cand, best)) best = cand;
        } else {
            ++dead;
            if (visits) visits[size_t(rc.x) * g.ec + rc.y] = 1;
        }
    }
    dead = warp_sum(dead);
    alive = warp_sum(alive);
    if ((threadIdx.x & 31) == 0) {
        if (dead) atomicAdd(&tally->eliminated, dead);
        if (alive) atomicAdd(&tally->pad, alive);
    }
    best = block_best(best, scratch);
    if (threadIdx.x == 0) store_partial(best, partials, blockIdx.x);
}

Grid to_grid(GridDesc d) {
    return Grid::make(d.er, d.ec, d.h, d.w, d.tr, d.tc, d.ti_lo, d.ti_hi);
}

template <int SW, int NW>
cudaError_t launch_band(const CorrJob& job, const BandTask& task, CellH* partials, int* n_partials,
                        cudaStream_t s) {
    const int bands = (task.nrows + 7) / 8;
    // span of staged rows: max over bands of (rows[yb+7] - rows[yb]) + kIC; rows are
    // increasing with the largest step at most the row stride, bounded by the caller.
    const int span = task.row_span + kIC;
    const BandGeom geo = band_geom<SW, NW>(span, job.npad);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_corr_band<SW, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr = true;
    }
    if (geo.smem > 200 * 1024) return cudaErrorInvalidValue;
    dim3 grid((task.nc + NW * 32 - 1) / (NW * 32), bands, std::max(1, task.ksplit));
    k_corr_band<SW, NW><<<grid, NW * 32, geo.smem, s>>>(job, task, geo.spitch, geo.srows, partials);
    *n_partials = task.dot ? 0 : int(grid.x * grid.y);
    return cudaGetLastError();
}

}  // namespace

cudaError_t corr_band(const CorrJob& job, const BandTask& task, CellH* partials, int* n_partials,
                      cudaStream_t s) {
    if (task.nrows <= 0 || task.nc <= 0) {
        *n_partials = 0;
        return cudaSuccess;
    }
    switch (task.sw) {
        case 1: return launch_band<1, 4>(job, task, partials, n_partials, s);
        case 3: return launch_band<3, 2>(job, task, partials, n_partials, s);
        case 5: return launch_band<5, 1>(job, task, partials, n_partials, s);
        case 7: return launch_band<7, 1>(job, task, partials, n_partials, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t corr_list(const CorrJob& job, const int2* locs, const unsigned long long* count,
                      int max_count, double* out_rho, uint8_t* out_deg, CellH* partials,
                      int n_partials, cudaStream_t s, int rho_by_loc, const TailReduce* tail) {
    // one FP32 partial covers lane_flush rows of one template column: < 2^24 exactly
    const int lane_flush = int(16777216LL / 65025LL);
    launch_pdl(k_corr_list, dim3(n_partials), dim3(256), 0, s, job, locs, count, max_count,
               out_rho, out_deg, partials, lane_flush, rho_by_loc, tail ? *tail : TailReduce{});
    return cudaGetLastError();
}

cudaError_t corr_list_f64(const CorrJob& job, const int2* locs, const unsigned long long* count,
                          int max_count, double* out_rho, uint8_t* out_deg, CellH* partials,
                          int n_partials, cudaStream_t s, int rho_by_loc) {
    k_list_f64<<<n_partials, 256, 0, s>>>(job, locs, count, max_count, out_rho, out_deg,
                                          partials, rho_by_loc);
    return cudaGetLastError();
}


cudaError_t corr_dense_f64(const CorrJob& job, double* surface, CellH* partials, int n_partials,
                           cudaStream_t s) {
    k_dense_f64<<<n_partials, 256, 0, s>>>(job, surface, partials);
    return cudaGetLastError();
}

__global__ void k_scatter_column(const double* rho, const uint8_t* deg, int n, int tc, int col,
                                 double* rho_c, uint8_t* deg_c) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        rho_c[size_t(i) * tc + col] = rho[i];
        deg_c[size_t(i) * tc + col] = deg[i];
    }
}

cudaError_t centre_epilogue(const CorrJob& job, GridDesc g, const int* rows, int cbase, int sw,
                            int nc, int col0, const double* dot, double* rho_c, uint8_t* deg_c,
                            CellH* partials, int n_partials, cudaStream_t s, int c_last,
                            const TailReduce* tail, const int* gate, double* sa_out,
                            float2* rec_out, const CentreStats* cs) {
    launch_pdl(k_centre_epi, dim3(n_partials), dim3(256), 0, s, job, to_grid(g), rows, cbase, sw,
               nc, col0, dot, rho_c, deg_c, partials, c_last, tail ? *tail : TailReduce{}, gate,
               sa_out, rec_out, cs ? *cs : CentreStats{});
    return cudaGetLastError();
}

cudaError_t gather_centre_stats(GridDesc g, DevStats st, CentreStats out, cudaStream_t s) {
    const size_t G = size_t(g.ti_hi - g.ti_lo) * g.tc;
    launch_pdl(k_gather_centre_stats, dim3(int(std::min<size_t>((G + 255) / 256, 148 * 8))),
               dim3(256), 0, s, to_grid(g), st, out.mu, out.om, out.fl);
    return cudaGetLastError();
}

cudaError_t scatter_column(const double* rho, const uint8_t* deg, int n, int tc, int col,
                           double* rho_c, uint8_t* deg_c, cudaStream_t s) {
    k_scatter_column<<<(n + 255) / 256, 256, 0, s>>>(rho, deg, n, tc, col, rho_c, deg_c);
    return cudaGetLastError();
}

cudaError_t reduce_cells(const CellH* partials, int n, CellH* out, cudaStream_t s,
                         const ReduceOp* op) {
    launch_pdl(k_reduce_cells, dim3(1), dim3(1024), 0, s, partials, n, out, op ? *op : ReduceOp{});
    return cudaGetLastError();
}

cudaError_t egs_init(int* stop, double* prev, unsigned long long* nr4, cudaStream_t s, int* h_acc,
                     unsigned long long* gate) {
    launch_pdl(k_egs_init, dim3(1), dim3(1), 0, s, stop, prev, nr4, h_acc, gate);
    return cudaGetLastError();
}

cudaError_t sec_compact(GridDesc g, const double* map, const double* rho_c, const uint8_t* deg_c,
                        const uint8_t* flat, int tflat, const double* thr, const uint8_t* seeded,
                        int2* locs, unsigned long long max_locs, Tally* tally, uint8_t* visits,
                        cudaStream_t s) {
    const size_t E = size_t(g.er) * g.ec;
    const int blocks = int(std::min<size_t>((E + 255) / 256, 148 * 8));
    k_sec_compact<<<blocks, 256, 0, s>>>(to_grid(g), map, rho_c, deg_c, flat, tflat, thr, seeded,
                                         locs, max_locs, tally, visits);
    return cudaGetLastError();
}

cudaError_t sqrt_gap(const double* x, double* y, size_t n, cudaStream_t s) {
    launch_pdl(k_sqrt_gap, dim3(int(std::min<size_t>((n + 255) / 256, 148 * 8))), dim3(256), 0,
               s, x, y, n);
    return cudaGetLastError();
}

int batch_kp(int K) {
    int kp = 1;
    while (kp < K) kp <<= 1;
    return kp;
}

cudaError_t sec_rows_multi(GridDesc g, const double* map, const uint8_t* flat,
                           const SecMulti& sm, cudaStream_t s) {
    if (sm.K < 1 || sm.K > kMaxBatch) return cudaErrorInvalidValue;
    const int rows = std::max(1, std::min(g.ti_hi * g.h, g.er) - g.ti_lo * g.h);
    const int blocks = std::max(1, std::min(rows, 148 * 8));
    switch (batch_kp(sm.K)) {
        case 1: case 2: launch_pdl(k_sec_rows_multi<2>, dim3(blocks), dim3(256), 0, s, to_grid(g), map, flat, sm); break;
        case 4: launch_pdl(k_sec_rows_multi<4>, dim3(blocks), dim3(256), 0, s, to_grid(g), map, flat, sm); break;
        case 8: launch_pdl(k_sec_rows_multi<8>, dim3(blocks), dim3(256), 0, s, to_grid(g), map, flat, sm); break;
        case 16: launch_pdl(k_sec_rows_multi<16>, dim3(blocks), dim3(256), 0, s, to_grid(g), map, flat, sm); break;
        default: launch_pdl(k_sec_rows_multi<32>, dim3(blocks), dim3(256), 0, s, to_grid(g), map, flat, sm); break;
    }
    return cudaGetLastError();
}

cudaError_t batch_records(const double* rho_c, const double* sa_c, const uint8_t* deg_c,
                          const uint8_t* seeded, size_t G, float2* rec, cudaStream_t s) {
    launch_pdl(k_batch_records, dim3(int(std::min<size_t>((G + 255) / 256, 148 * 8))), dim3(256),
               0, s, rho_c, sa_c, deg_c, seeded, G, rec);
    return cudaGetLastError();
}

cudaError_t sec_rows(GridDesc g, const double* map, const double* rho_c, double* sa_c,
                     const uint8_t* deg_c, const uint8_t* flat, int tflat, const double* thr,
                     const uint8_t* seeded, int2* locs, unsigned long long max_locs, Tally* tally,
                     uint8_t* visits, cudaStream_t s, bool sa_ready, TileFlags tf) {
    const size_t G = size_t(g.tr) * g.tc;
    if (!sa_ready)
        launch_pdl(k_sqrt_gap, dim3(int(std::min<size_t>((G + 255) / 256, 148 * 8))), dim3(256), 0, s, rho_c, sa_c, G);
    const int rows = std::max(1, std::min(g.ti_hi * g.h, g.er) - g.ti_lo * g.h);
    const int blocks = std::max(1, std::min(rows, 148 * 8));
    launch_pdl(k_sec_rows, dim3(blocks), dim3(256), 0, s, to_grid(g), map, rho_c, sa_c, deg_c, flat, tflat, thr, seeded,
                                      locs, max_locs, tally, visits, tf);
    return cudaGetLastError();
}

cudaError_t threshold_init(const CellH* centre_best, int has_init, double init, double* thr,
                           cudaStream_t s) {
    k_threshold_init<<<1, 1, 0, s>>>(centre_best, has_init, init, thr);
    return cudaGetLastError();
}

cudaError_t threshold_raise(const CellH* best, double* thr, cudaStream_t s) {
    k_threshold_raise<<<1, 1, 0, s>>>(best, thr);
    return cudaGetLastError();
}

cudaError_t seed_members(GridDesc g, const double* rho_c, const uint8_t* deg_c, const double* thr,
                         double margin, uint8_t* seeded, int2* locs, unsigned long long* count,
                         unsigned long long max_locs, unsigned long long* n_groups,
                         unsigned long long max_groups, cudaStream_t s, float2* rec) {
    const long long G = (long long)g.tr * g.tc;
    const int blocks = int(std::min<long long>((G + 255) / 256, 148 * 8));
    launch_pdl(k_seed_members, dim3(blocks), dim3(256), 0, s, to_grid(g), rho_c, deg_c, thr, margin, seeded, locs, count,
                                          max_locs, n_groups, max_groups, rec);
    return cudaGetLastError();
}

cudaError_t first_record(GridDesc g, const int2* locs, const unsigned long long* count,
                         const double* rho, const double* map,
                         const double* rho_c, const uint8_t* deg_c, const uint8_t* flat, int tflat,
                         double T, unsigned long long after, unsigned long long* best_key,
                         cudaStream_t s) {
    cudaMemsetAsync(best_key, 0xff, sizeof(*best_key), s);
    k_first_record<<<148 * 4, 256, 0, s>>>(to_grid(g), locs, count, rho, map, rho_c, deg_c,
                                           flat, tflat, T, after, best_key);
    return cudaGetLastError();
}

cudaError_t fetch_record_rho(GridDesc g, const int2* locs, const unsigned long long* count,
                             const double* rho, unsigned long long key, double* out,
                             cudaStream_t s) {
    k_fetch_rho<<<148 * 4, 256, 0, s>>>(to_grid(g), locs, count, rho, key, out);
    return cudaGetLastError();
}

cudaError_t seq_final(GridDesc g, const int2* locs, const unsigned long long* count,
                      const double* rho, const double* map,
                      const double* rho_c, const uint8_t* deg_c, const uint8_t* flat, int tflat,
                      double T0, const unsigned long long* rec_key, const double* rec_T, int n_rec,
                      Tally* tally, uint8_t* visits, CellH* partials, int n_partials,
                      cudaStream_t s) {
    k_seq_final<<<n_partials, 256, 0, s>>>(to_grid(g), locs, count, rho, map, rho_c, deg_c,
                                           flat, tflat, T0, rec_key, rec_T, n_rec, tally, visits,
                                           partials);
    return cudaGetLastError();
}

}  // namespace tmk
