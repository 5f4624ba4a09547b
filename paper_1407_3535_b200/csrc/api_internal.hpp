// api_internal.hpp -- shared plumbing of the C++ reference API (tmatch_api.cpp) for the
// other translation units of libtmatch.so (tmatch_cli.cpp).  Not installed.
#pragma once

#include "tmatch/matcher.hpp"
#include "tmatch_cuda.h"

namespace tmatch::internal {
tm_ctx* context();                 // the calling thread's device context
void check_rc(int rc);             // C ABI status -> the reference's exception types
tm_match_params to_c_params(const MatchParams& p);
MatchResult from_c_result(const tm_match_result& r);
}  // namespace tmatch::internal
