// scene.cu -- the analytic ground truth on sm_100a (SPEC.md scenegen).
//
// arf::CapsuleFigure / PosedFigure (R/scene.hpp:10-126) rendered through the renderer's
// dense path: render_image (R/render.hpp:178-218) with field(x) = PosedFigure::query(x)
// (matter iff density > 0), to_norm = G^-1, no occupancy grid, and the exact silhouette
// PosedFigure::ray_hits (R/scene.hpp:123-130) as the alpha mask. Thread per ray; every
// double op is the reference's, in its order (explicit _rn intrinsics, no FMA), so the
// sample positions, per-sample densities/colors and mask are bit-exact; composite uses
// CUDA expm1 (<= 1 ulp vs glibc).
//
//   figure_query_kernel   analytic_query / PosedFigure::query over a point batch
//   figure_render_kernel  image mode (thread = pixel) or list mode (thread = training ray)
#include <cuda_runtime.h>

#include <algorithm>

#include "model.h"
#include "ray.cuh"

namespace arfx {
namespace {

// smoothstep01(t) = clamp01(t)^2 (3 - 2 clamp01(t))  R/math.hpp:25-35
__device__ __forceinline__ double smoothstep01(double t) {
  t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);
  return dmul(dmul(t, t), dsub(3.0, dmul(2.0, t)));
}

struct FigSample {
  double density;
  d3 color;
};

// PosedFigure::query (R/scene.hpp:79-97); analytic_query (:31-50) when a/b are the rest segments
__device__ __forceinline__ FigSample figure_query(const FigureView& F, d3 x) {
  double total = 0.0;
  d3 acc = make3(0.0, 0.0, 0.0);
  for (int i = 0; i < F.nb; ++i) {
    const double d = point_segment_distance(x, make3(F.a[i][0], F.a[i][1], F.a[i][2]),
                                            make3(F.b[i][0], F.b[i][1], F.b[i][2]));
    if (d >= F.radius[i]) continue;
    const double s = smoothstep01(ddiv(dsub(F.radius[i], d), F.soft));
    if (s <= 0.0) continue;
    const double dens = dmul(F.amp[i], s);
    total = dadd(total, dens);
    acc = add3(acc, mul3(make3(F.col[i][0], F.col[i][1], F.col[i][2]), dens));
  }
  FigSample r{0.0, make3(0.0, 0.0, 0.0)};
  if (total > 0.0) {
    r.density = total;
    r.color = make3(ddiv(acc.x, total), ddiv(acc.y, total), ddiv(acc.z, total));
  }
  return r;
}

// ray_segment_distance (R/scene.hpp:103-117): 65 samples along the segment, ray t >= 0
__device__ __forceinline__ double ray_segment_distance(d3 o, d3 d, d3 a, d3 b) {
  const d3 ab = sub3(b, a);
  double best = 1.7976931348623157e308;
  for (int i = 0; i <= 64; ++i) {
    const double u = ddiv(static_cast<double>(i), 64.0);
    const d3 p = add3(a, mul3(ab, u));
    const double tt = dot3(sub3(p, o), d);
    const double t = (0.0 < tt) ? tt : 0.0;
    const double v = norm3(sub3(p, add3(o, mul3(d, t))));
    best = (v < best) ? v : best;
  }
  return best;
}

__device__ __forceinline__ bool ray_hits(const FigureView& F, d3 o, d3 d) {
  for (int i = 0; i < F.nb; ++i)
    if (ray_segment_distance(o, d, make3(F.a[i][0], F.a[i][1], F.a[i][2]), make3(F.b[i][0], F.b[i][1], F.b[i][2])) <
        F.radius[i])
      return true;
  return false;
}

__global__ void figure_query_kernel(FigureView F, const double* __restrict__ pts, long long n,
                                    double* __restrict__ dens, double* __restrict__ col) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const FigSample r = figure_query(F, make3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
    dens[i] = r.density;
    col[3 * i + 0] = r.color.x;
    col[3 * i + 1] = r.color.y;
    col[3 * i + 2] = r.color.z;
  }
}

struct FigRenderArgs {
  FigureView F;
  CameraView cam;
  double w2n[12];
  double nlo[3], nhi[3];
  int N, stratified;
  double eps;
  uint64_t seed, frame;
  long long n;                // rays
  const int32_t *lpx, *lpy;   // list mode; null -> ray r = pixel r of the image
  float *rgb, *alpha;
  uint8_t* mask;
};

__global__ void __launch_bounds__(128) figure_render_kernel(const __grid_constant__ FigRenderArgs A) {
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < A.n;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int px = A.lpx ? A.lpx[r] : static_cast<int>(r % A.cam.width);
    const int py = A.lpy ? A.lpy[r] : static_cast<int>(r / A.cam.width);
    const RayGeom R = make_ray(A.cam, A.w2n, A.nlo, A.nhi, px, py);
    if (A.mask) A.mask[r] = ray_hits(A.F, R.o, R.d) ? 1 : 0;
    double cr = 0.0, cg = 0.0, cb = 0.0, acc = 0.0;
    if (R.valid && A.N > 0) {
      const double step = ddiv(dsub(R.tf, R.tn), static_cast<double>(A.N));
      Pcg32 rng = keyed_rng(A.seed, A.frame, static_cast<uint64_t>(py) * A.cam.width + px);
      double jit = A.stratified ? pcg_double(rng) : 0.5;
      double t = sample_t(R.tn, step, 0, jit);
      double T = 1.0;
      for (int i = 0; i < A.N; ++i) {  // composite R/render.hpp:98-119
        double tn1 = 0.0;
        if (i + 1 < A.N) {
          jit = A.stratified ? pcg_double(rng) : 0.5;
          tn1 = sample_t(R.tn, step, i + 1, jit);
        }
        const double delta = (i + 1 < A.N) ? dsub(tn1, t) : dsub(R.tf, t);
        if (A.eps > 0 && T <= A.eps) break;
        const FigSample q = figure_query(A.F, add3(R.o, mul3(R.d, t)));
        t = tn1;
        if (q.density <= 0.0) continue;  // field() == false: skipped
        const double alpha = -expm1(-dmul(q.density, delta));
        const double w = dmul(alpha, T);
        cr = dadd(cr, dmul(q.color.x, w));
        cg = dadd(cg, dmul(q.color.y, w));
        cb = dadd(cb, dmul(q.color.z, w));
        acc = dadd(acc, w);
        T = dmul(T, dsub(1.0, alpha));
      }
    }
    A.rgb[3 * r + 0] = static_cast<float>(cr);
    A.rgb[3 * r + 1] = static_cast<float>(cg);
    A.rgb[3 * r + 2] = static_cast<float>(cb);
    A.alpha[r] = static_cast<float>(acc);
  }
}

unsigned blocks_for_rays(long long n, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + threads - 1) / threads, 16LL * sms)));
}

}  // namespace

void figure_query_batch(const FigureView& F, const double* d_pts, long long n, double* d_dens, double* d_col,
                        cudaStream_t s) {
  if (n <= 0) return;
  figure_query_kernel<<<blocks_for_rays(n, 128), 128, 0, s>>>(F, d_pts, n, d_dens, d_col);
  ARFX_CUDA(cudaGetLastError());
}

void figure_render(const FigureView& F, const HostCamera& cam, const double* w2n12, const double* nlo,
                   const double* nhi, int N, bool stratified, double eps, uint64_t seed, uint64_t frame, long long n,
                   const int32_t* d_px, const int32_t* d_py, float* d_rgb, float* d_alpha, uint8_t* d_mask,
                   cudaStream_t s) {
  if (n <= 0) return;
  FigRenderArgs A{};
  A.F = F;
  A.cam = CameraView{cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, {}};
  std::copy(cam.ext, cam.ext + 12, A.cam.ext);
  std::copy(w2n12, w2n12 + 12, A.w2n);
  std::copy(nlo, nlo + 3, A.nlo);
  std::copy(nhi, nhi + 3, A.nhi);
  A.N = N;
  A.stratified = stratified ? 1 : 0;
  A.eps = eps;
  A.seed = seed;
  A.frame = frame;
  A.n = n;
  A.lpx = d_px;
  A.lpy = d_py;
  A.rgb = d_rgb;
  A.alpha = d_alpha;
  A.mask = d_mask;
  figure_render_kernel<<<blocks_for_rays(n, 128), 128, 0, s>>>(A);
  ARFX_CUDA(cudaGetLastError());
}

}  // namespace arfx
