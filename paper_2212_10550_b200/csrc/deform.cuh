// deform.cuh -- Fast-SNARF correspondence search on sm_100a, bit-exact FP64.
//
// Restates, per posed point x':
//   SkinningGrid::interpolate   R/skinning.hpp:25-55
//   lbs_apply                   R/articulation.hpp:45-50
//   inverse_lbs_ctx             R/articulation.hpp:94-145 (damped Newton, frozen
//                               Jacobian J = sum w_i R_i, 4-step halving line search,
//                               stall break, <= max_iterations)
//   InverseRoots::push          R/articulation.hpp:66-81
//
// B200 layout: the skinning grid is read through a per-cell packed table (see
// SkinView): one 32-bit mask of the bones that are nonzero at any of the cell's 8
// corners, then 8 contiguous doubles per such bone -> one eval touches ~6 bones x
// 64 B contiguous instead of 8 corners x n_bones x 8 B scattered. Skipping bones
// that are zero at every corner is exact (adding +0.0 to a non-negative sum is the
// identity). The lbs sum and the Jacobian are accumulated in
// the same pass over the union bones, so the Jacobian of the accepted line-search
// candidate is ready for the next iteration (the reference recomputes it from the
// same weights, R/articulation.hpp:110-112 -- identical operand order).
#pragma once

#include "arfx_internal.h"
#include "exact.cuh"

namespace arfx {

struct Roots {
  int count;
  double x[kMaxRoots][3];
  double r[kMaxRoots];
};

// R/articulation.hpp:66-81
__device__ __forceinline__ void roots_push(Roots& R, d3 p, double res, double dedup) {
  for (int i = 0; i < R.count; ++i) {
    const d3 q = make3(R.x[i][0], R.x[i][1], R.x[i][2]);
    if (norm3(sub3(q, p)) < dedup) {
      if (res < R.r[i]) {
        R.x[i][0] = p.x;
        R.x[i][1] = p.y;
        R.x[i][2] = p.z;
        R.r[i] = res;
      }
      return;
    }
  }
  if (R.count < kMaxRoots) {
    R.x[R.count][0] = p.x;
    R.x[R.count][1] = p.y;
    R.x[R.count][2] = p.z;
    R.r[R.count] = res;
    ++R.count;
  }
}

#ifndef ARFX_DS_LD256
#define ARFX_DS_LD256 1
#endif
// 32 bytes (4 doubles, 32-B aligned) through the read-only path in one 256-bit request
__device__ __forceinline__ void ldg256(const double* p, double* o) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
}

// Skinning weights at x (trilinear over the packed cell table + renormalisation),
// then g = lbs(x) - x_target, |g| and J = sum_{w_i != 0} w_i R_i.
// `ws` is per-thread scratch for the union bones' raw weights (smem, stride apart).
// Returns the number of union bones visited (work accounting for the roofline).
#ifndef ARFX_DS_NOSKIP_W0
#define ARFX_DS_NOSKIP_W0 1
#endif
__device__ __forceinline__ int skin_eval(const SkinView& S, const PoseCtx* __restrict__ P, d3 x,
                                         d3 xt, double* ws, int stride, d3& g, double& gn,
                                         double J[9]) {
  // clamp_inside: cwise_max(lo, cwise_min(hi, x))  R/math.hpp:245-247
  double p[3] = {x.x, x.y, x.z};
  const int res[3] = {S.rx, S.ry, S.rz};
  int c[3];
  double f[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double v = (p[a] < S.hi[a]) ? p[a] : S.hi[a];
    v = (S.lo[a] < v) ? v : S.lo[a];
    const double u = dmul(ddiv(dsub(v, S.lo[a]), S.e[a]), static_cast<double>(res[a] - 1));
    double fl = floor(u);
    if (fl > static_cast<double>(res[a] - 2)) fl = static_cast<double>(res[a] - 2);
    if (fl < 0) fl = 0;
    c[a] = static_cast<int>(fl);
    f[a] = dsub(u, fl);
  }
  double wt[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double wx = (k & 1) ? f[0] : dsub(1.0, f[0]);
    const double wy = (k & 2) ? f[1] : dsub(1.0, f[1]);
    const double wz = (k & 4) ? f[2] : dsub(1.0, f[2]);
    wt[k] = dmul(dmul(wx, wy), wz);
  }
  const int cell = (c[2] * (S.ry - 1) + c[1]) * (S.rx - 1) + c[0];
  const uint2 mo = __ldg(S.cell_mo + cell);
  const uint32_t mask = mo.x;
  const double* vals = S.cell_vals + static_cast<size_t>(mo.y) * 8;
  // pass 1: raw interpolated weights per union bone, and their sum (bone order); two
  // bones per trip so 8 independent 16-byte loads are in flight before the math
  double sum = 0.0;
  const int nu = __popc(mask);
  for (int j = 0; j < nu; j += 2) {
    const bool two = j + 1 < nu;
#if ARFX_DS_LD256
    // 256-bit loads (LDG.E.ENL2.256): a lane's 64-B bone row in two requests instead of four;
    // scattered lanes cost one L1 data wavefront per line per request
    double va[8], vb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    ldg256(vals + 8 * j, va);
    ldg256(vals + 8 * j + 4, va + 4);
    if (two) {
      ldg256(vals + 8 * j + 8, vb);
      ldg256(vals + 8 * j + 12, vb + 4);
    }
#else
    const double2* v2 = reinterpret_cast<const double2*>(vals + 8 * j);
    const double2 a0 = __ldg(v2 + 0), a1 = __ldg(v2 + 1), a2 = __ldg(v2 + 2), a3 = __ldg(v2 + 3);
    double2 b0 = make_double2(0, 0), b1 = b0, b2 = b0, b3 = b0;
    if (two) {
      b0 = __ldg(v2 + 4);
      b1 = __ldg(v2 + 5);
      b2 = __ldg(v2 + 6);
      b3 = __ldg(v2 + 7);
    }
    const double va[8] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y, a3.x, a3.y};
    const double vb[8] = {b0.x, b0.y, b1.x, b1.y, b2.x, b2.y, b3.x, b3.y};
#endif
    // The reference skips corners with wt == 0 (R/skinning.hpp:45); adding the
    // product instead is bit-identical: wt * v = +-0 for finite v, acc starts at +0 and
    // x + (+-0) == x, (+0) + (-0) == +0 -- so the data-dependent branch (and its DSETP/FSEL
    // per corner per bone) is dropped.
    double acc = 0.0, acc2 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      acc = dadd(acc, dmul(wt[k], va[k]));
      acc2 = dadd(acc2, dmul(wt[k], vb[k]));
    }
    ws[j * stride] = acc;
    sum = dadd(sum, acc);
    if (two) {
      ws[(j + 1) * stride] = acc2;
      sum = dadd(sum, acc2);
    }
  }
  int j = 0;
  const bool renorm = sum > 0;
  const double inv = renorm ? ddiv(1.0, sum) : 1.0;
  // pass 2: normalised weights -> lbs and Jacobian
  d3 out = make3(0.0, 0.0, 0.0);
#pragma unroll
  for (int e = 0; e < 9; ++e) J[e] = 0.0;
  j = 0;
  for (uint32_t m = mask; m; m &= m - 1, ++j) {
    const int b = __ffs(m) - 1;
    double w = ws[j * stride];
    if (renorm) w = dmul(w, inv);
#if ARFX_DS_NOSKIP_W0
    // no w != 0 branch: for w == +-0 every added product is +-0 (T, x finite), and
    // out / J + (+-0) leaves them bit-identical (they start at +0; x + (+-0) == x for x != 0
    // and (+0) + (-0) == +0), exactly like skipping the bone
    {
#else
    if (w != 0.0) {
#endif
      const double* T = P->bone[b];
      const d3 a = rigid_apply(T, x);
      out = add3(out, mul3(a, w));
#pragma unroll
      for (int e = 0; e < 9; ++e) J[e] = dadd(J[e], dmul(T[e], w));
    }
  }
  g = sub3(out, xt);
  gn = norm3(g);
  return nu;
}

// Skinning weights only (SkinningGrid::interpolate), dense output over n_bones.
__device__ __forceinline__ void skin_weights_dense(const SkinView& S, d3 x, double* w_out) {
  double p[3] = {x.x, x.y, x.z};
  const int res[3] = {S.rx, S.ry, S.rz};
  int c[3];
  double f[3];
  for (int a = 0; a < 3; ++a) {
    double v = (p[a] < S.hi[a]) ? p[a] : S.hi[a];
    v = (S.lo[a] < v) ? v : S.lo[a];
    const double u = dmul(ddiv(dsub(v, S.lo[a]), S.e[a]), static_cast<double>(res[a] - 1));
    double fl = floor(u);
    if (fl > static_cast<double>(res[a] - 2)) fl = static_cast<double>(res[a] - 2);
    if (fl < 0) fl = 0;
    c[a] = static_cast<int>(fl);
    f[a] = dsub(u, fl);
  }
  for (int i = 0; i < S.nb; ++i) w_out[i] = 0.0;
  for (int k = 0; k < 8; ++k) {
    const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
    const double wt = dmul(dmul(dx ? f[0] : dsub(1.0, f[0]), dy ? f[1] : dsub(1.0, f[1])),
                           dz ? f[2] : dsub(1.0, f[2]));
    if (wt == 0.0) continue;
    const double* nw =
        S.weights + ((static_cast<size_t>(c[2] + dz) * S.ry + (c[1] + dy)) * S.rx + (c[0] + dx)) * S.nb;
    for (int i = 0; i < S.nb; ++i) w_out[i] = dadd(w_out[i], dmul(wt, nw[i]));
  }
  double sum = 0.0;
  for (int i = 0; i < S.nb; ++i) sum = dadd(sum, w_out[i]);
  if (sum > 0) {
    const double inv = ddiv(1.0, sum);
    for (int i = 0; i < S.nb; ++i) w_out[i] = dmul(w_out[i], inv);
  }
}

// The per-start Newton iteration itself (inverse_lbs_ctx's loop body) lives in the start
// pipeline's state machine, deform_starts.cuh start_newton_kernel.

}  // namespace arfx
