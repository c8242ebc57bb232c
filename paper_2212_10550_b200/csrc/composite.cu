// composite.cu -- volume compositing on explicit per-ray sample sets (one thread per ray).
//   composite           R/render.hpp:98-119  (front-to-back, early termination T <= eps)
//   composite_backward  R/render.hpp:125-157 (suffix accumulators, tail gets no gradient)
// Used by the batched C-ABI entry points; the render path fuses its own copy of the
// forward pass with root selection (render.cu K4).
#include <cuda_runtime.h>

#include "exact.cuh"
#include "model.h"

namespace arfx {

namespace {

__device__ __forceinline__ double alpha_of(double sigma, double delta) {
  return -expm1(-dmul(sigma, delta));
}

__global__ void composite_explicit_kernel(int n_rays, const int64_t* __restrict__ off,
                                          const double* __restrict__ delta,
                                          const uint8_t* __restrict__ skipped,
                                          const float* __restrict__ dens, const float* __restrict__ col,
                                          double eps, double* out_c3, double* out_a, int32_t* term) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const int64_t b = off[r], n = off[r + 1] - off[r];
  double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0, acc = 0.0;
  int64_t i = 0;
  for (; i < n; ++i) {
    if (eps > 0 && T <= eps) break;
    const int64_t s = b + i;
    const double sigma = skipped[s] ? 0.0 : static_cast<double>(dens[s]);
    if (sigma <= 0.0) continue;
    const double alpha = alpha_of(sigma, delta[s]);
    const double w = dmul(alpha, T);
    cr = dadd(cr, dmul(static_cast<double>(col[3 * s + 0]), w));
    cg = dadd(cg, dmul(static_cast<double>(col[3 * s + 1]), w));
    cb = dadd(cb, dmul(static_cast<double>(col[3 * s + 2]), w));
    acc = dadd(acc, w);
    T = dmul(T, dsub(1.0, alpha));
  }
  out_c3[3 * r + 0] = cr;
  out_c3[3 * r + 1] = cg;
  out_c3[3 * r + 2] = cb;
  out_a[r] = acc;
  term[r] = static_cast<int32_t>(i);
}

__global__ void composite_backward_kernel(int n_rays, const int64_t* __restrict__ off,
                                          const double* __restrict__ delta,
                                          const uint8_t* __restrict__ skipped,
                                          const float* __restrict__ dens, const float* __restrict__ col,
                                          double eps, const double* __restrict__ dC3,
                                          const double* __restrict__ dA, double* trans,
                                          double* d_sigma, double* d_c3) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const int64_t b = off[r], n = off[r + 1] - off[r];
  // forward to find terminated_at  (composite, R/render.hpp:110-123)
  double T = 1.0;
  int64_t m = 0;
  for (; m < n; ++m) {
    if (eps > 0 && T <= eps) break;
    const int64_t s = b + m;
    const double sigma = skipped[s] ? 0.0 : static_cast<double>(dens[s]);
    if (sigma <= 0.0) continue;
    T = dmul(T, dsub(1.0, alpha_of(sigma, delta[s])));
  }
  for (int64_t i = 0; i < n; ++i) {
    d_sigma[b + i] = 0.0;
    d_c3[3 * (b + i) + 0] = d_c3[3 * (b + i) + 1] = d_c3[3 * (b + i) + 2] = 0.0;
  }
  // transmittance into each accumulated sample  R/render.hpp:141-147
  double t = 1.0;
  for (int64_t i = 0; i < m; ++i) {
    const int64_t s = b + i;
    trans[s] = t;
    const double sigma = skipped[s] ? 0.0 : static_cast<double>(dens[s]);
    const double alpha = sigma <= 0.0 ? 0.0 : alpha_of(sigma, delta[s]);
    t = dmul(t, dsub(1.0, alpha));
  }
  const double dcx = dC3[3 * r + 0], dcy = dC3[3 * r + 1], dcz = dC3[3 * r + 2], da = dA[r];
  double chx = 0.0, chy = 0.0, chz = 0.0, ahat = 0.0;
  for (int64_t i = m - 1; i >= 0; --i) {  // R/render.hpp:148-162
    const int64_t s = b + i;
    if (skipped[s]) continue;
    const double sigma = static_cast<double>(dens[s]);
    const double alpha = sigma <= 0.0 ? 0.0 : alpha_of(sigma, delta[s]);
    const double cx = static_cast<double>(col[3 * s + 0]), cy = static_cast<double>(col[3 * s + 1]),
                 cz = static_cast<double>(col[3 * s + 2]);
    const double dC_dalpha =
        dadd(dadd(dmul(dcx, dsub(cx, chx)), dmul(dcy, dsub(cy, chy))), dmul(dcz, dsub(cz, chz)));
    const double dA_dalpha = dsub(1.0, ahat);
    const double d_alpha_total = dmul(trans[s], dadd(dC_dalpha, dmul(da, dA_dalpha)));
    const double om = dsub(1.0, alpha);
    d_sigma[s] = dmul(dmul(d_alpha_total, delta[s]), om);
    const double at = dmul(alpha, trans[s]);
    d_c3[3 * s + 0] = dmul(dcx, at);
    d_c3[3 * s + 1] = dmul(dcy, at);
    d_c3[3 * s + 2] = dmul(dcz, at);
    chx = dadd(dmul(cx, alpha), dmul(chx, om));
    chy = dadd(dmul(cy, alpha), dmul(chy, om));
    chz = dadd(dmul(cz, alpha), dmul(chz, om));
    ahat = dadd(alpha, dmul(ahat, om));
  }
}

}  // namespace

void composite_explicit(int n_rays, const int64_t* d_off, const double* d_delta, const uint8_t* d_skip,
                        const float* d_dens, const float* d_col, double eps, double* d_c3, double* d_a,
                        int32_t* d_term, cudaStream_t s) {
  if (n_rays <= 0) return;
  composite_explicit_kernel<<<(n_rays + 127) / 128, 128, 0, s>>>(n_rays, d_off, d_delta, d_skip, d_dens,
                                                                 d_col, eps, d_c3, d_a, d_term);
  ARFX_CUDA(cudaGetLastError());
}

void composite_backward_explicit(int n_rays, const int64_t* d_off, const double* d_delta,
                                 const uint8_t* d_skip, const float* d_dens, const float* d_col,
                                 double eps, const double* d_dC3, const double* d_dA, double* d_trans,
                                 double* d_sigma, double* d_c3, cudaStream_t s) {
  if (n_rays <= 0) return;
  composite_backward_kernel<<<(n_rays + 127) / 128, 128, 0, s>>>(n_rays, d_off, d_delta, d_skip, d_dens,
                                                                 d_col, eps, d_dC3, d_dA, d_trans,
                                                                 d_sigma, d_c3);
  ARFX_CUDA(cudaGetLastError());
}

}  // namespace arfx
