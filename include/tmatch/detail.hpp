// tmatch/detail.hpp -- scalar evaluation helpers of the reference API
// (proj/include/tmatch/detail.hpp:18-51).  Declared here for source compatibility and
// defined out of line in csrc/tmatch_api.cpp; they are host scalars used by callers and
// tests -- the search itself evaluates correlations in the sm_100a kernels, which replay
// the same zncc_at epilogue bit for bit.
#pragma once

#include "tmatch/image.hpp"
#include "tmatch/stats.hpp"

namespace tmatch::detail {

// var_sum <= max((1e-9*mn)^2, max(1e-13, 4*eps*mn) * q_sum)
bool variance_is_flat(double var_sum, double q_sum, long long mn);

struct TemplateStats {
    double mu = 0.0;
    double omega = 0.0;
    bool flat = true;
};

TemplateStats template_stats(const Image& t);

// Row-major FP64 dot product of t with the window of I at (r, c).
double window_dot(const Image& t, const Image& I, int r, int c);

// Correlation at (r, c) from precomputed window statistics; flat windows give 0.
double zncc_at(const Image& t, const TemplateStats& ts, const Image& I, const WindowStats& ws,
               int r, int c);

}  // namespace tmatch::detail
