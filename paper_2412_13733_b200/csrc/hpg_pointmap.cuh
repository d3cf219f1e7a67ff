// Pointwise LVPP maps (stage (b)) shared by the warp and CTA kernels.
#pragma once
#include "hpg_common.cuh"

namespace hpg {

// v: synthesized fields at one quadrature point (mode-dependent meaning),
// phi: obstacle-free gradient bound sample, wcin/wcout: cached weights,
// vw: the fields handed to the analysis stage.
template <int MODE>
__device__ __forceinline__ void point_map(const double* v, double phi, const double* wcin,
                                          double* wcout, double* vw, bool& flag) {
  if constexpr (MODE == M_OBST_RES) {
    // assembly.py:545-547
    double e = clamped_exp_neg(v[0], flag);
    wcout[0] = e;
    vw[0] = e;
  } else if constexpr (MODE == M_OBST_APPLY) {
    // assembly.py:562-566 / 265-269 (flag not reported by apply_D)
    bool dummy = false;
    double e = clamped_exp_neg(v[0], dummy);
    vw[0] = v[1] * e;
  } else if constexpr (MODE == M_OBST_CACHED) {
    vw[0] = v[0] * wcin[0];
  } else if constexpr (MODE == M_GRAD_RES) {
    // nl_moments, assembly.py:786-790; kernel fields :796-801.  One
    // reciprocal square root (rsqrt, <= 1 ulp) replaces the reference's
    // sqrt + divisions: phi v / sqrt(r2) and r2^{-1/2}, r2^{-3/2} agree to a
    // few ulp, far inside the 1e-12 parity bar, at a fraction of the cost of
    // IEEE division (the dominant FP64 work of the gradient map)
    double vx = v[0], vy = v[1];
    double r2 = 1.0 + vx * vx + vy * vy;
    double inv = rsqrt(r2);
    double pinv = phi * inv;
    vw[0] = pinv * vx;
    vw[1] = pinv * vy;
    double inv3 = inv * inv * inv;
    wcout[0] = phi * (inv - vx * vx * inv3);
    wcout[1] = phi * (-vx * vy * inv3);
    wcout[2] = phi * (inv - vy * vy * inv3);
  } else if constexpr (MODE == M_GRAD_APPLY) {
    // apply_D, assembly.py:820-829
    double vx = v[0], vy = v[1];
    double r2 = 1.0 + vx * vx + vy * vy;
    double inv = rsqrt(r2);
    double inv3 = inv * inv * inv;
    double kxx = phi * (inv - vx * vx * inv3);
    double kxy = phi * (-vx * vy * inv3);
    double kyy = phi * (inv - vy * vy * inv3);
    vw[0] = kxx * v[2] + kxy * v[3];
    vw[1] = kxy * v[2] + kyy * v[3];
  } else if constexpr (MODE == M_GRAD_CACHED) {
    vw[0] = wcin[0] * v[0] + wcin[1] * v[1];
    vw[1] = wcin[1] * v[0] + wcin[2] * v[1];
  }
}

}  // namespace hpg
