// tm_common.cuh -- device helpers shared by the tmatch sm_100a kernels.
//
// Bit-exactness discipline: every FP64 expression that the reference evaluates in a
// fixed order is written with explicit _rn intrinsics (no FMA contraction), mirroring
// the cited reference line.  Integer work (window sums, dot products on u8 data) is
// exact in any order and is free to be re-associated.
#pragma once
#include <utility>

#include <cstdint>
#include <cuda_runtime.h>

namespace tmk {

// Programmatic dependent launch: kernels on the search path start with pdl_wait() (a
// no-op unless launched with launch_pdl), so the next kernel's launch overlaps the tail
// of the previous one; nothing produced by earlier work is touched before the wait.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}


constexpr double kEps = 2.220446049250313e-16;

__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }
// std::clamp(v, lo, hi)
__device__ __forceinline__ double dclamp(double v, double lo, double hi) {
    return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// The retained test of egs.cpp:12-25 on a non-flat member, clamp(num / den, -1, 1) < thr with
// the division rounded to nearest (autocorr.cpp:84-88), decided without the division unless
// num / den lies within 1e-9 (relative) of thr: for 0 < thr <= 1 and den > 0 the clamp
// cannot change the outcome, and num < thr*den*(1 - 1e-9) implies RN(num/den) < thr (the
// margin is 10^7 ulps; the FP64 products below are off by at most 2 ulps).
__device__ __forceinline__ bool retained_below(double num, double den, double thr) {
    if (thr > 0.0 && thr <= 1.0 && den > 1e-290 && den < 1e290) {
        const double lim = __dmul_rn(thr, den);
        const double eps = __dmul_rn(lim, 2e-9);
        if (num < __dsub_rn(lim, eps)) return true;
        if (num > __dadd_rn(lim, eps)) return false;
    }
    return dclamp(__ddiv_rn(num, den), -1.0, 1.0) < thr;
}

// detail.hpp:18-22 variance_is_flat
__device__ __forceinline__ bool variance_is_flat(double var_sum, double q_sum, long long mn) {
    const double abs_tol = __dmul_rn(1e-9, double(mn));
    const double rel = dmax(1e-13, __dmul_rn(__dmul_rn(4.0, kEps), double(mn)));
    return var_sum <= dmax(__dmul_rn(abs_tol, abs_tol), __dmul_rn(rel, q_sum));
}

// stats.cpp:84-91: per-window epilogue from exact sums S, Q.
__device__ __forceinline__ void window_epilogue(double sum, double sq, double inv_mn,
                                                long long mn, double prefix_noise, double& mu,
                                                double& omega, uint8_t& flat) {
    const double var_sum = __dsub_rn(sq, __dmul_rn(__dmul_rn(sum, sum), inv_mn));
    const bool f = variance_is_flat(var_sum, sq, mn) || var_sum <= prefix_noise;
    mu = __dmul_rn(sum, inv_mn);
    omega = f ? 0.0 : __dsqrt_rn(dmax(0.0, var_sum));
    flat = f ? 1 : 0;
}

// Template statistics shared by every correlation launch (stats.cpp:98-111, computed on
// the host in reference order).
struct TStats {
    double mu, omega;
    double mn;  // double(m) * double(n)
    int flat;
};

// detail.hpp:45-51 zncc_at epilogue given the window dot product.
__device__ __forceinline__ double zncc_epilogue(double dot, const TStats& ts, double mu_w,
                                                double omega_w, bool flat_w) {
    if (ts.flat || flat_w) return 0.0;
    const double num = __dsub_rn(dot, __dmul_rn(__dmul_rn(ts.mn, ts.mu), mu_w));
    return dclamp(__ddiv_rn(num, __dmul_rn(ts.omega, omega_w)), -1.0, 1.0);
}

// bounds.cpp:21-23, 41-46 (inputs already clamped, so `checked` never throws here).
__device__ __forceinline__ double half_gap(double a, double b) {
    return __dmul_rn(__dsqrt_rn(dmax(0.0, __dsub_rn(1.0, __dmul_rn(a, a)))),
                     __dsqrt_rn(dmax(0.0, __dsub_rn(1.0, __dmul_rn(b, b)))));
}
__device__ __forceinline__ bool sec_holds(double tb, double a, double b) {
    tb = dclamp(tb, -1.0, 1.0);
    a = dclamp(a, -1.0, 1.0);
    b = dclamp(b, -1.0, 1.0);
    return tb >= __dadd_rn(__dmul_rn(a, b), half_gap(a, b));
}

// ---- BestCell (stats.hpp:71-79) and better_candidate (stats.cpp:147-154) ----------
struct Cell {
    double rho;
    int row, col;
    int flags;  // bit0 valid, bit1 degenerate
};

__device__ __forceinline__ Cell no_cell() { return Cell{0.0, -1, -1, 2}; }
__device__ __forceinline__ Cell make_cell(int r, int c, double rho, bool degenerate) {
    return Cell{rho, r, c, 1 | (degenerate ? 2 : 0)};
}

__device__ __forceinline__ bool better(const Cell& a, const Cell& b) {
    if (!(a.flags & 1)) return false;
    if (!(b.flags & 1)) return true;
    const bool da = a.flags & 2, db = b.flags & 2;
    if (da != db) return !da;
    if (a.rho != b.rho) return a.rho > b.rho;
    if (a.row != b.row) return a.row < b.row;
    return a.col < b.col;
}

__device__ __forceinline__ Cell shfl_cell(const Cell& c, int src_lane_xor) {
    Cell o;
    o.rho = __shfl_xor_sync(0xffffffffu, c.rho, src_lane_xor);
    o.row = __shfl_xor_sync(0xffffffffu, c.row, src_lane_xor);
    o.col = __shfl_xor_sync(0xffffffffu, c.col, src_lane_xor);
    o.flags = __shfl_xor_sync(0xffffffffu, c.flags, src_lane_xor);
    return o;
}

__device__ __forceinline__ Cell warp_best(Cell c) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const Cell o = shfl_cell(c, s);
        if (better(o, c)) c = o;
    }
    return c;
}

// Block-wide best; result valid in thread 0.  `scratch` needs blockDim/32 Cells.
__device__ __forceinline__ Cell block_best(Cell c, Cell* scratch) {
    c = warp_best(c);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) scratch[wid] = c;
    __syncthreads();
    if (wid == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        c = lane < nw ? scratch[lane] : no_cell();
        c = warp_best(c);
    }
    __syncthreads();
    return c;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    return v;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, s);
        v = o > v ? o : v;
    }
    return v;
}

// Exact unsigned division by a runtime constant without the XU pipe: floor(x / d) =
// umulhi64(x, ceil(2^64 / d)) for every 32-bit x (the error term x*eps/2^64 < 1/d).
struct FastDiv {
    unsigned long long magic;  // 0 encodes d == 1
    __host__ __device__ static FastDiv make(unsigned d) {
        FastDiv f;
        f.magic = d <= 1 ? 0ull : (~0ull) / d + 1ull;
        return f;
    }
    __host__ __device__ __forceinline__ unsigned div(unsigned x) const {
#ifdef __CUDA_ARCH__
        return magic ? unsigned(__umul64hi((unsigned long long)x, magic)) : x;
#else
        return magic ? unsigned(((unsigned __int128)x * magic) >> 64) : x;
#endif
    }
};

// Group geometry (autocorr.cpp:12-32): tiles anchored at (0,0), clipped edge tiles,
// centre = (r0 + r1) / 2.  fh/fw/fec divide by h, w and ec on the fast path.
struct Grid {
    int er, ec, h, w, tr, tc;
    int ti_lo, ti_hi;  // group-row range of this device (row strip)
    FastDiv fh, fw, fec;
    __host__ static Grid make(int er, int ec, int h, int w, int tr, int tc, int ti_lo, int ti_hi) {
        return Grid{er, ec, h, w, tr, tc, ti_lo, ti_hi, FastDiv::make(unsigned(h)),
                    FastDiv::make(unsigned(w)), FastDiv::make(unsigned(ec))};
    }
    // extent rows [row_lo, row_hi) owned by the strip
    __host__ __device__ __forceinline__ int row_lo() const { return ti_lo * h; }
    __host__ __device__ __forceinline__ int row_hi() const { return ti_hi * h < er ? ti_hi * h : er; }
    __host__ __device__ __forceinline__ int tile_r(int r) const {
#ifdef __CUDA_ARCH__
        return min(int(fh.div(r)), tr - 1);
#else
        return r / h < tr - 1 ? r / h : tr - 1;
#endif
    }
    __host__ __device__ __forceinline__ int tile_c(int c) const {
#ifdef __CUDA_ARCH__
        return min(int(fw.div(c)), tc - 1);
#else
        return c / w < tc - 1 ? c / w : tc - 1;
#endif
    }
    // linear extent index -> (row, col)
    __host__ __device__ __forceinline__ void rc(size_t k, int& r, int& c) const {
#ifdef __CUDA_ARCH__
        r = int(fec.div(unsigned(k)));
#else
        r = int(k / size_t(ec));
#endif
        c = int(k) - r * ec;
    }
    __host__ __device__ __forceinline__ int center_row(int ti) const {
        const int r0 = ti * h, r1 = min(r0 + h, er) - 1;
        return (r0 + r1) >> 1;
    }
    __host__ __device__ __forceinline__ int center_col(int tj) const {
        const int c0 = tj * w, c1 = min(c0 + w, ec) - 1;
        return (c0 + c1) >> 1;
    }
};

}  // namespace tmk
