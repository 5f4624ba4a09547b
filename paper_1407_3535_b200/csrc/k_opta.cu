// k_opta.cu -- OptA kernels: separable blur, blur fidelity, violation marks and the
// coverage restore of repair_to_fixed_point (blur.cpp:57-239), sm_100a.
//
// The blurred image is non-integer, so these kernels replay the reference's FP64
// operation order exactly: taps accumulate left to right from 0.0 with separate multiply
// and add (blur.cpp:69-83), so the optimised image is bit-identical to the reference's.
// Marks and coverage are integer and exact in any order.
#include <algorithm>

#include "kernels.hpp"
#include "tm_common.cuh"

namespace tmk {

namespace {

__global__ void k_blur_rows(const double* __restrict__ img, int p, int q,
                            const double* __restrict__ prof, int d, double* __restrict__ tmp) {
    const size_t N = size_t(p) * q;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < N;
         k += size_t(gridDim.x) * blockDim.x) {
        const int r = int(k / q), c = int(k % q);
        const double* in = img + size_t(r) * q;
        double acc = 0.0;
        for (int t = -d; t <= d; ++t) {
            const int cc = min(max(c + t, 0), q - 1);
            acc = __dadd_rn(acc, __dmul_rn(prof[t + d], in[cc]));
        }
        tmp[k] = acc;
    }
}

__global__ void k_blur_cols(const double* __restrict__ tmp, int p, int q,
                            const double* __restrict__ prof, int d, double* __restrict__ out) {
    const size_t N = size_t(p) * q;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < N;
         k += size_t(gridDim.x) * blockDim.x) {
        const int r = int(k / q), c = int(k % q);
        double acc = 0.0;
        for (int t = -d; t <= d; ++t) {
            const int rr = min(max(r + t, 0), p - 1);
            acc = __dadd_rn(acc, __dmul_rn(prof[t + d], tmp[size_t(rr) * q + c]));
        }
        out[k] = acc;
    }
}

// blur.cpp:115-123 (fidelity against the original's window statistics)
__global__ void k_fidelity(const double* __restrict__ cross, DevStats o, DevStats b,
                           double* __restrict__ fid) {
    const size_t E = size_t(o.er) * o.ec;
    const double mn = double(o.m) * double(o.n);
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < E;
         k += size_t(gridDim.x) * blockDim.x) {
        double rho = 0.0;
        if (!o.flat[k] && !b.flat[k]) {
            const double num = __dsub_rn(cross[k], __dmul_rn(__dmul_rn(mn, b.mu[k]), o.mu[k]));
            rho = dclamp(__ddiv_rn(num, __dmul_rn(b.omega[k], o.omega[k])), -1.0, 1.0);
        }
        fid[k] = rho;
    }
}

__global__ void k_changed(const double* __restrict__ a, const double* __restrict__ b, size_t n,
                          uint8_t* __restrict__ out) {
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n;
         k += size_t(gridDim.x) * blockDim.x)
        out[k] = a[k] != b[k] ? 1 : 0;
}

// blur.cpp:225-233
__global__ void k_marks(const double* __restrict__ fid, const double* __restrict__ in_win,
                        size_t E, double lambda, uint8_t* __restrict__ marks,
                        unsigned long long* count) {
    unsigned long long local = 0;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < E;
         k += size_t(gridDim.x) * blockDim.x) {
        const bool mk = !(fid[k] >= lambda) && (in_win == nullptr || in_win[k] != 0.0);
        marks[k] = mk;
        local += mk;
    }
    local = warp_sum(local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

// Integer prefix of the marks (CoverageQuery, blur.cpp:137-150): rows then columns.
// Integer prefix of the marks: exact in any order, so a warp scans a row 32 columns at a
// time (coalesced, shuffle scan) and the column pass prefetches 16 rows ahead.
__global__ void k_mark_rows(const uint8_t* __restrict__ marks, int er, int ec, int* __restrict__ P) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const size_t pw = size_t(ec) + 1;
    if (r > er) return;
    if (r == 0) {
        for (int c = lane; c <= ec; c += 32) P[c] = 0;
        return;
    }
    if (lane == 0) P[size_t(r) * pw] = 0;
    int carry = 0;
    for (int c0 = 0; c0 < ec; c0 += 32) {
        const int c = c0 + lane;
        int v = c < ec ? marks[size_t(r - 1) * ec + c] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (c < ec) P[size_t(r) * pw + c + 1] = carry + v;
        carry += __shfl_sync(0xffffffffu, v, 31);
    }
}

__global__ void k_mark_cols(int er, int ec, int* __restrict__ P) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t pw = size_t(ec) + 1;
    if (c > ec) return;
    constexpr int kC = 16;
    int acc = 0;
    for (int r0 = 1; r0 <= er; r0 += kC) {
        int v[kC];
#pragma unroll
        for (int j = 0; j < kC; ++j) v[j] = r0 + j <= er ? P[size_t(r0 + j) * pw + c] : 0;
#pragma unroll
        for (int j = 0; j < kC; ++j) {
            if (r0 + j > er) break;
            acc += v[j];
            P[size_t(r0 + j) * pw + c] = acc;
        }
    }
}

// restore_marked (blur.cpp:170-179): pixel (x,y) restored iff a marked window covers it.
__global__ void k_restore(double* __restrict__ blurred, const double* __restrict__ original,
                          const int* __restrict__ P, int er, int ec, int m, int n, int p, int q) {
    const size_t N = size_t(p) * q;
    const size_t pw = size_t(ec) + 1;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < N;
         k += size_t(gridDim.x) * blockDim.x) {
        const int x = int(k / q), y = int(k % q);
        const int r0 = max(0, x - m + 1), r1 = min(er - 1, x);
        const int c0 = max(0, y - n + 1), c1 = min(ec - 1, y);
        if (r0 > r1 || c0 > c1) continue;
        const int s = P[size_t(r1 + 1) * pw + c1 + 1] - P[size_t(r0) * pw + c1 + 1] -
                      P[size_t(r1 + 1) * pw + c0] + P[size_t(r0) * pw + c0];
        if (s > 0) blurred[k] = original[k];
    }
}

int blocks_for(size_t n) { return int(std::min<size_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

cudaError_t blur_replica(const double* img, int p, int q, const double* prof_dev, int len,
                         double* tmp, double* out, cudaStream_t s) {
    const size_t N = size_t(p) * q;
    const int d = len / 2;
    k_blur_rows<<<blocks_for(N), 256, 0, s>>>(img, p, q, prof_dev, d, tmp);
    k_blur_cols<<<blocks_for(N), 256, 0, s>>>(tmp, p, q, prof_dev, d, out);
    return cudaGetLastError();
}

cudaError_t fidelity_epilogue(const double* cross, DevStats orig, DevStats blur, double* fid,
                              cudaStream_t s) {
    const size_t E = size_t(orig.er) * orig.ec;
    k_fidelity<<<blocks_for(E), 256, 0, s>>>(cross, orig, blur, fid);
    return cudaGetLastError();
}

cudaError_t changed_mask(const double* a, const double* b, size_t n, uint8_t* out,
                         cudaStream_t s) {
    k_changed<<<blocks_for(n), 256, 0, s>>>(a, b, n, out);
    return cudaGetLastError();
}

cudaError_t mark_violations(const double* fid, const double* changed_in_window, size_t E,
                            double lambda, uint8_t* marks, unsigned long long* count,
                            cudaStream_t s) {
    cudaMemsetAsync(count, 0, sizeof(*count), s);
    k_marks<<<blocks_for(E), 256, 0, s>>>(fid, changed_in_window, E, lambda, marks, count);
    return cudaGetLastError();
}

cudaError_t restore_covered(double* blurred, const double* original, const uint8_t* marks,
                            int er, int ec, int m, int n, int p, int q, int* scratch,
                            cudaStream_t s) {
    k_mark_rows<<<(er + 1 + 7) / 8, 256, 0, s>>>(marks, er, ec, scratch);  // warp per row
    k_mark_cols<<<(ec + 1 + 127) / 128, 128, 0, s>>>(er, ec, scratch);
    k_restore<<<blocks_for(size_t(p) * q), 256, 0, s>>>(blurred, original, scratch, er, ec, m, n,
                                                        p, q);
    return cudaGetLastError();
}

}  // namespace tmk
