// ray.cuh -- camera ray generation + normalized-space slab test + sample positions,
// shared by the march (render.cu) and the analytic-figure renderer (scene.cu).
#pragma once

#include "arfx_internal.h"
#include "exact.cuh"

namespace arfx {

struct RayGeom {
  d3 o, d;
  double tn, tf;
  bool valid;  // hit && tn < tf
};

// generate_ray + normalized-space slab test  (R/camera.hpp:61-70, R/render.hpp:190-196, :15-37)
__device__ __forceinline__ RayGeom make_ray(const CameraView& cam, const double* w2n, const double* nlo,
                                            const double* nhi, int px, int py) {
  RayGeom R;
  const double dcx = ddiv(dsub(dadd(static_cast<double>(px), 0.5), cam.cx), cam.fx);
  const double dcy = ddiv(dsub(dadd(static_cast<double>(py), 0.5), cam.cy), cam.fy);
  const double* e = cam.ext;
  const double rt[9] = {e[0], e[3], e[6], e[1], e[4], e[7], e[2], e[5], e[8]};
  const d3 ot = matvec(rt, make3(e[9], e[10], e[11]));
  R.o = make3(-ot.x, -ot.y, -ot.z);
  const d3 dr = matvec(rt, make3(dcx, dcy, 1.0));
  const double n = norm3(dr);
  R.d = make3(ddiv(dr.x, n), ddiv(dr.y, n), ddiv(dr.z, n));
  const d3 on = rigid_apply(w2n, R.o);
  const d3 dn = sub3(rigid_apply(w2n, add3(R.o, mul3(R.d, 1.0))), on);
  double t0 = 0.0, t1 = 1.7976931348623157e308;
  const double oo[3] = {on.x, on.y, on.z}, dd[3] = {dn.x, dn.y, dn.z};
  bool hit = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (!hit) break;
    const double o = oo[a], d = dd[a];
    if (fabs(d) < 1e-300) {
      if (o < nlo[a] || o > nhi[a]) hit = false;
      continue;
    }
    double ta = ddiv(dsub(nlo[a], o), d);
    double tb = ddiv(dsub(nhi[a], o), d);
    if (ta > tb) {
      const double t = ta;
      ta = tb;
      tb = t;
    }
    t0 = (t0 < ta) ? ta : t0;
    t1 = (tb < t1) ? tb : t1;
    if (t0 > t1) hit = false;
  }
  R.tn = t0;
  R.tf = t1;
  R.valid = hit && (t0 < t1);
  return R;
}

// t_i = t_near + (i + jitter) * step  (R/render.hpp:79-83)
__device__ __forceinline__ double sample_t(double tn, double step, int i, double jitter) {
  return dadd(tn, dmul(dadd(static_cast<double>(i), jitter), step));
}

}  // namespace arfx
