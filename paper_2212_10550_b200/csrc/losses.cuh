// losses.cuh -- the training losses of SPEC.md:454-489 (Eq. 9-11 of the paper) as per-ray
// device functions, evaluated in double on the f32 rendered values (the values the
// reference's render reports, R/render.hpp:167-171). The reference code base has no loss
// (SURVEY.md §8f row 1); oracle/arf_oracle.c arfo_losses restates the same formulas.
//
//   L_rgb   = mean_r huber(|C_r - C*_r|)        huber(r) = r^2/2 (r <= d), d (r - d/2) else
//   L_alpha = mean_r |A_r - A*_r|               subgradient 0 at equality
//   L_hard  = mean_r -ln(e^-|A| + e^-|A-1|) + ln(1 + e^-1)
//             d/dA at A = 0 / 1: the one-sided limit from inside [0, 1]
//   total   = w_rgb L_rgb + w_alpha L_alpha + w_hard L_hard   (L_density: separate pass)
// Upstream gradients dL/dC, dL/dA of the total are rounded to f32, as the reference-shaped
// composite_backward consumes them (arfx_train_fwd_bwd).
#pragma once

#include "arfx_internal.h"

namespace arfx {

struct LossCfg {
  double w_rgb, w_alpha, w_hard, w_density, huber_delta;
};

struct RayLoss {
  double rgb, alpha, hard;  // per-ray terms (unweighted, before the mean)
  float dC[3], dA;          // upstream gradient of the weighted batch mean
};

__device__ __forceinline__ RayLoss ray_loss(float r, float g, float b, float a, const float* gt_rgb, float gt_a,
                                            const LossCfg& L, double inv_n) {
  RayLoss o;
  const double ex = __dsub_rn(static_cast<double>(r), static_cast<double>(gt_rgb[0]));
  const double ey = __dsub_rn(static_cast<double>(g), static_cast<double>(gt_rgb[1]));
  const double ez = __dsub_rn(static_cast<double>(b), static_cast<double>(gt_rgb[2]));
  const double rn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez)));
  const double d = L.huber_delta;
  double gs;  // d huber / d e  = e * gs
  if (rn <= d) {
    o.rgb = __dmul_rn(0.5, __dmul_rn(rn, rn));
    gs = 1.0;
  } else {
    o.rgb = __dmul_rn(d, __dsub_rn(rn, __dmul_rn(0.5, d)));
    gs = __ddiv_rn(d, rn);
  }
  const double crgb = __dmul_rn(L.w_rgb, inv_n);
  o.dC[0] = static_cast<float>(__dmul_rn(crgb, __dmul_rn(ex, gs)));
  o.dC[1] = static_cast<float>(__dmul_rn(crgb, __dmul_rn(ey, gs)));
  o.dC[2] = static_cast<float>(__dmul_rn(crgb, __dmul_rn(ez, gs)));
  const double A = static_cast<double>(a);
  const double ea = __dsub_rn(A, static_cast<double>(gt_a));
  o.alpha = fabs(ea);
  const double sa1 = ea > 0.0 ? 1.0 : (ea < 0.0 ? -1.0 : 0.0);
  const double p = exp(-fabs(A)), q = exp(-fabs(__dsub_rn(A, 1.0)));
  const double sum = __dadd_rn(p, q);
  o.hard = __dadd_rn(-log(sum), log1p(exp(-1.0)));
  const double sp = A < 0.0 ? -1.0 : 1.0;   // d|A|/dA, +1 at A = 0 (inside)
  const double sq = A > 1.0 ? 1.0 : -1.0;   // d|A-1|/dA, -1 at A = 1 (inside)
  const double dh = __ddiv_rn(__dadd_rn(__dmul_rn(sp, p), __dmul_rn(sq, q)), sum);
  o.dA = static_cast<float>(
      __dmul_rn(__dadd_rn(__dmul_rn(L.w_alpha, sa1), __dmul_rn(L.w_hard, dh)), inv_n));
  return o;
}

}  // namespace arfx
