// tmatch/bounds.hpp -- transitive correlation bound algebra (reference
// proj/include/tmatch/bounds.hpp:9-34).  Scalar host functions; the per-member bound test
// of scan 2 runs in k_sec_compact with the identical expression order.
#pragma once

namespace tmatch {

struct BoundPair {
    double lower;
    double upper;
};

BoundPair transitive_bounds(double rho_tc, double rho_co);
double transitive_gap(double rho_tc, double rho_co);
bool sec_holds(double rho_tb, double rho_tc, double rho_co);
double elimination_autocorr_threshold(double rho_tb, double rho_tc);
double expected_elimination_threshold(double rho_tb);

}  // namespace tmatch
