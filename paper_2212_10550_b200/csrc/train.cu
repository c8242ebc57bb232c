// train.cu -- training forward + backward on sm_100a.
//
// The reference has no training function; the step is composed from its pieces exactly
// as oracle/ref_driver.cpp arfr_train_fwd_bwd does: per ray the render forward
// (stratified), composite_backward (R/render.hpp:125-157) with upstream dL/dC, dL/dA,
// then CanonicalField::query_backward (R/field.hpp:91-103) at every accumulated
// non-skipped sample's selected canonical root, accumulated into FieldGrads.
//
//   K1..K3 as in render (march in ray-list mode, deformer, field forward over the pool)
//   K7 train_composite_kernel  thread per ray: selection + composite forward (rgb, alpha,
//                              terminated_at) + exact reverse pass; dsigma / dc land on the
//                              selected root's pool entry (R/render.hpp:148-162)
//   K8 field_backward_kernel   thread per flagged pool entry: exact forward recompute
//                              (encode + MLP, activations in smem), reference-order MLP
//                              backward per query (R/mlp.hpp:116-154); weight gradients
//                              warp-reduced then one atomic per weight per warp; the
//                              encode backward scatters w*up into the grid gradient with
//                              f32 atomics (R/hash_grid.hpp:155-169).
// Gradient sums are therefore order-different from the reference's serial per-thread
// buffers (SPEC.md:426 allows reassociation); everything upstream is bit-exact.
#include <cuda_runtime.h>

#include <algorithm>

#include "field.cuh"
#include "losses.cuh"
#include "model.h"

namespace arfx {
namespace {

__device__ __forceinline__ int select_root_t(const uint8_t* snroot, const int32_t* sbase, const float4* pres,
                                             long long s, float4& best) {
  const int nin = snroot[s];
  if (nin == 0) return -1;
  const int base = sbase[s];
  int sel = 0;
  best = pres[base];
  for (int k = 1; k < nin; ++k) {
    const float4 v = pres[base + k];
    if (v.x > best.x) {
      best = v;
      sel = k;
    }
  }
  return sel;
}

struct TrainCompositeArgs {
  long long n_rays;
  int N;
  double eps;
  const int32_t *ray_first, *ray_count;
  const int16_t* sidx;
  const double* sdelta;
  const uint8_t* snroot;
  const int32_t* sbase;
  const float4* pres;
  double* strans;  // scratch: transmittance before each posed sample
  const float* dC;
  const float* dA;
  // fused losses: when gt_rgb != null, dC / dA come from ray_loss instead
  const float* gt_rgb;
  const float* gt_alpha;
  LossCfg loss;
  double inv_n;
  double* ray_terms;  // [n_rays][3] unweighted per-ray loss terms
  float *rgb, *alpha;
  float* pgs;      // per pool entry: dsigma (f32, as passed to query_backward)
  float* pgc;      // per pool entry: dcolor[3]
  uint8_t* pflag;  // per pool entry: needs query_backward
};

__global__ void train_composite_kernel(TrainCompositeArgs A) {
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < A.n_rays;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int first = A.ray_first[r], cnt = A.ray_count[r];
    // ---- forward (composite R/render.hpp:98-119) ----
    double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0, acc = 0.0;
    int m = A.N;  // terminated_at (index into the full N-sample list)
    if (A.eps > 0 && T <= A.eps) m = 0;
    for (int j = 0; j < cnt && m == A.N; ++j) {
      const long long s = first + j;
      A.strans[s] = T;
      float4 v;
      const int sel = select_root_t(A.snroot, A.sbase, A.pres, s, v);
      if (sel < 0) continue;
      const double sigma = static_cast<double>(v.x);
      if (sigma <= 0.0) continue;
      const double alpha = -expm1(-__dmul_rn(sigma, A.sdelta[s]));
      const double w = __dmul_rn(alpha, T);
      cr = __dadd_rn(cr, __dmul_rn(static_cast<double>(v.y), w));
      cg = __dadd_rn(cg, __dmul_rn(static_cast<double>(v.z), w));
      cb = __dadd_rn(cb, __dmul_rn(static_cast<double>(v.w), w));
      acc = __dadd_rn(acc, w);
      T = __dmul_rn(T, __dsub_rn(1.0, alpha));
      if (A.eps > 0 && T <= A.eps) m = A.sidx[s] + 1;
    }
    if (cnt == 0) m = 0;
    const float fr = static_cast<float>(cr), fg = static_cast<float>(cg), fb = static_cast<float>(cb);
    const float fa = static_cast<float>(acc);
    A.rgb[3 * r + 0] = fr;
    A.rgb[3 * r + 1] = fg;
    A.rgb[3 * r + 2] = fb;
    A.alpha[r] = fa;
    // ---- upstream: given, or the fused loss gradient of this ray ----
    double dcx, dcy, dcz, da;
    if (A.gt_rgb) {
      const RayLoss L = ray_loss(fr, fg, fb, fa, A.gt_rgb + 3 * r, A.gt_alpha[r], A.loss, A.inv_n);
      A.ray_terms[3 * r + 0] = L.rgb;
      A.ray_terms[3 * r + 1] = L.alpha;
      A.ray_terms[3 * r + 2] = L.hard;
      dcx = L.dC[0], dcy = L.dC[1], dcz = L.dC[2], da = L.dA;
    } else {
      dcx = A.dC[3 * r + 0], dcy = A.dC[3 * r + 1], dcz = A.dC[3 * r + 2], da = A.dA[r];
    }
    // ---- backward (composite_backward R/render.hpp:125-157), reverse over i < m ----
    double chx = 0.0, chy = 0.0, chz = 0.0, ahat = 0.0;
    for (int j = cnt - 1; j >= 0; --j) {
      const long long s = first + j;
      if (A.sidx[s] >= m) continue;
      float4 v;
      const int sel = select_root_t(A.snroot, A.sbase, A.pres, s, v);
      if (sel < 0) continue;  // skipped (no root)
      const double sigma = static_cast<double>(v.x);
      const double alpha = sigma <= 0.0 ? 0.0 : -expm1(-__dmul_rn(sigma, A.sdelta[s]));
      const double cx = static_cast<double>(v.y), cy = static_cast<double>(v.z), cz = static_cast<double>(v.w);
      const double dCda = __dadd_rn(__dadd_rn(__dmul_rn(dcx, __dsub_rn(cx, chx)), __dmul_rn(dcy, __dsub_rn(cy, chy))),
                                    __dmul_rn(dcz, __dsub_rn(cz, chz)));
      const double dAda = __dsub_rn(1.0, ahat);
      const double trans = A.strans[s];
      const double dat = __dmul_rn(trans, __dadd_rn(dCda, __dmul_rn(da, dAda)));
      const double om = __dsub_rn(1.0, alpha);
      const double ds = __dmul_rn(__dmul_rn(dat, A.sdelta[s]), om);
      const double at = __dmul_rn(alpha, trans);
      const long long p = A.sbase[s] + sel;
      A.pgs[p] = static_cast<float>(ds);
      A.pgc[3 * p + 0] = static_cast<float>(__dmul_rn(dcx, at));
      A.pgc[3 * p + 1] = static_cast<float>(__dmul_rn(dcy, at));
      A.pgc[3 * p + 2] = static_cast<float>(__dmul_rn(dcz, at));
      A.pflag[p] = 1;
      chx = __dadd_rn(__dmul_rn(cx, alpha), __dmul_rn(chx, om));
      chy = __dadd_rn(__dmul_rn(cy, alpha), __dmul_rn(chy, om));
      chz = __dadd_rn(__dmul_rn(cz, alpha), __dmul_rn(chz, om));
      ahat = __dadd_rn(alpha, __dmul_rn(ahat, om));
    }
  }
}

constexpr int kFbThreads = 64;
constexpr int kIn = 32, kHid = 64, kOut = 4;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// K8. Activations per thread live in smem as [k][thread] (conflict-free):
//   X[32] input features, H1[64], H2[64], D[64] (gradient scratch).
__global__ void __launch_bounds__(kFbThreads) field_backward_kernel(FieldView F, const double* __restrict__ px,
                                                                    const double* __restrict__ py,
                                                                    const double* __restrict__ pz,
                                                                    const uint8_t* __restrict__ pflag,
                                                                    const float* __restrict__ pgs,
                                                                    const float* __restrict__ pgc,
                                                                    const unsigned long long* n_dev, long long cap,
                                                                    float* __restrict__ grid_grad,
                                                                    float* __restrict__ mlp_grad) {
  extern __shared__ float fb_smem[];
  const int t = threadIdx.x;
  float* X = fb_smem;                    // [kIn][kFbThreads]
  float* H1 = X + kIn * kFbThreads;      // [kHid][kFbThreads]
  float* H2 = H1 + kHid * kFbThreads;    // [kHid][kFbThreads]
  float* D = H2 + kHid * kFbThreads;     // [kHid][kFbThreads]
  const float* W = F.mlp;
  const float* W0 = W;
  const float* B0 = W0 + kIn * kHid;
  const float* W1 = B0 + kHid;
  const float* B1 = W1 + kHid * kHid;
  const float* W2 = B1 + kHid;
  const float* B2 = W2 + kOut * kHid;
  float* gW0 = mlp_grad;
  float* gB0 = gW0 + kIn * kHid;
  float* gW1 = gB0 + kHid;
  float* gB1 = gW1 + kHid * kHid;
  float* gW2 = gB1 + kHid;
  float* gB2 = gW2 + kOut * kHid;
  long long n = static_cast<long long>(*n_dev);
  n = n < cap ? n : cap;
  for (long long base = static_cast<long long>(blockIdx.x) * kFbThreads; base < n;
       base += static_cast<long long>(gridDim.x) * kFbThreads) {
    const long long q = base + t;
    const bool act = q < n && pflag[q] != 0;
    const d3 x = act ? make3(px[q], py[q], pz[q]) : make3(0, 0, 0);
    // ---- forward recompute (CanonicalField::query_backward re-runs the forward) ----
    float feats[kIn];
    if (act) hash_encode_f2(F, x, feats);
    else
      for (int i = 0; i < kIn; ++i) feats[i] = 0.0f;
    for (int i = 0; i < kIn; ++i) X[i * kFbThreads + t] = feats[i];
    for (int o = 0; o < kHid; ++o) {
      float a = B0[o];
      for (int i = 0; i < kIn; ++i) a = fadd(a, fmul(__ldg(W0 + o * kIn + i), feats[i]));
      H1[o * kFbThreads + t] = (a < 0.0f) ? 0.0f : a;
    }
    for (int o = 0; o < kHid; ++o) {
      float a = B1[o];
      for (int i = 0; i < kHid; ++i) a = fadd(a, fmul(__ldg(W1 + o * kHid + i), H1[i * kFbThreads + t]));
      H2[o * kFbThreads + t] = (a < 0.0f) ? 0.0f : a;
    }
    float lg[kOut];
    for (int o = 0; o < kOut; ++o) {
      float a = B2[o];
      for (int i = 0; i < kHid; ++i) a = fadd(a, fmul(__ldg(W2 + o * kHid + i), H2[i * kFbThreads + t]));
      lg[o] = a;
    }
    // ---- d logits (R/field.hpp:95-99) ----
    float u2[kOut] = {0.f, 0.f, 0.f, 0.f};
    if (act) {
      u2[0] = fmul(pgs[q], logistic_f(lg[0]));
      for (int c = 0; c < 3; ++c) {
        const float v = logistic_f(lg[1 + c]);
        u2[1 + c] = fmul(fmul(pgc[3 * q + c], v), __fsub_rn(1.0f, v));
      }
    }
    // ---- output layer backward: gb2 += u; gW2 += u*h2; dprev = sum_o u*W2 (u != 0) ----
    for (int i = 0; i < kHid; ++i) D[i * kFbThreads + t] = 0.0f;
    for (int o = 0; o < kOut; ++o) {
      const float u = u2[o];
      const float sb = warp_sum(u);
      if ((t & 31) == 0 && sb != 0.0f) atomicAdd(gB2 + o, sb);
      for (int i = 0; i < kHid; ++i) {
        const float g = warp_sum(fmul(u, H2[i * kFbThreads + t]));
        if ((t & 31) == 0 && g != 0.0f) atomicAdd(gW2 + o * kHid + i, g);
      }
      if (u != 0.0f)
        for (int i = 0; i < kHid; ++i) D[i * kFbThreads + t] = fadd(D[i * kFbThreads + t], fmul(u, __ldg(W2 + o * kHid + i)));
    }
    // ReLU mask on hidden layer 2 (post == 0), then the gradient w.r.t. h2 lives in H2
    for (int i = 0; i < kHid; ++i) {
      const float d = D[i * kFbThreads + t];
      H2[i * kFbThreads + t] = (H2[i * kFbThreads + t] == 0.0f) ? 0.0f : d;
    }
    // ---- hidden layer 1 backward (input = h1) ----
    for (int i = 0; i < kHid; ++i) D[i * kFbThreads + t] = 0.0f;
    for (int o = 0; o < kHid; ++o) {
      const float u = H2[o * kFbThreads + t];
      const float sb = warp_sum(u);
      if ((t & 31) == 0 && sb != 0.0f) atomicAdd(gB1 + o, sb);
      if (__any_sync(0xffffffffu, u != 0.0f)) {
        for (int i = 0; i < kHid; ++i) {
          const float g = warp_sum(fmul(u, H1[i * kFbThreads + t]));
          if ((t & 31) == 0 && g != 0.0f) atomicAdd(gW1 + o * kHid + i, g);
        }
      }
      if (u != 0.0f)
        for (int i = 0; i < kHid; ++i) D[i * kFbThreads + t] = fadd(D[i * kFbThreads + t], fmul(u, __ldg(W1 + o * kHid + i)));
    }
    for (int i = 0; i < kHid; ++i) {
      const float d = D[i * kFbThreads + t];
      H1[i * kFbThreads + t] = (H1[i * kFbThreads + t] == 0.0f) ? 0.0f : d;
    }
    // ---- first layer backward (input = features) -> d features ----
    float din[kIn];
    for (int i = 0; i < kIn; ++i) din[i] = 0.0f;
    for (int o = 0; o < kHid; ++o) {
      const float u = H1[o * kFbThreads + t];
      const float sb = warp_sum(u);
      if ((t & 31) == 0 && sb != 0.0f) atomicAdd(gB0 + o, sb);
      if (__any_sync(0xffffffffu, u != 0.0f)) {
        for (int i = 0; i < kIn; ++i) {
          const float g = warp_sum(fmul(u, X[i * kFbThreads + t]));
          if ((t & 31) == 0 && g != 0.0f) atomicAdd(gW0 + o * kIn + i, g);
        }
      }
      if (u != 0.0f)
        for (int i = 0; i < kIn; ++i) din[i] = fadd(din[i], fmul(u, __ldg(W0 + o * kIn + i)));
    }
    // ---- encode backward (R/hash_grid.hpp:155-169) ----
    if (act) {
      double u[3];
      normalize_point(F, x, u);
      for (int l = 0; l < F.L; ++l) {
        LevelCorners lc;
        level_corners(F, l, u, lc);
        float* gt = grid_grad + static_cast<size_t>(l) * F.T * 2;
        for (int k = 0; k < 8; ++k) {
          const float w = lc.w[k];
          if (w == 0.0f) continue;
          atomicAdd(gt + 2 * static_cast<size_t>(lc.idx[k]) + 0, fmul(w, din[2 * l + 0]));
          atomicAdd(gt + 2 * static_cast<size_t>(lc.idx[k]) + 1, fmul(w, din[2 * l + 1]));
        }
      }
    }
  }
}

int sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace

void field_backward_pool(ModelImpl& m, const unsigned long long* d_n, long long cap, const uint8_t* flag,
                         const float* gs, const float* gc, cudaStream_t s) {
  if (!(m.fv.F == 2 && m.fv.in_dim == kIn && m.fv.hidden == kHid && m.fv.n_layers == 3 && m.fv.out_dim == kOut))
    throw std::invalid_argument("train path: libarfx implements the 32-64-64-4 decoder (levels*F == 32)");
  const size_t smem = static_cast<size_t>(kIn + 3 * kHid) * kFbThreads * sizeof(float);
  static bool attr = false;
  if (!attr) {
    ARFX_CUDA(cudaFuncSetAttribute(field_backward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    attr = true;
  }
  const long long blocks = std::min<long long>((cap + kFbThreads - 1) / kFbThreads, static_cast<long long>(sms()) * 8);
  m.prof.begin("field_backward", s);
  field_backward_kernel<<<static_cast<unsigned>(std::max<long long>(blocks, 1)), kFbThreads, smem, s>>>(
      m.fv, m.ws.px.ptr, m.ws.py.ptr, m.ws.pz.ptr, flag, gs, gc, d_n, cap, m.grid_grad.ptr, m.mlp_grad.ptr);
  ARFX_CUDA(cudaGetLastError());
  m.prof.end(s);
}

void train_composite(ModelImpl& m, long long n_rays, int N, double eps, const float* d_dC, const float* d_dA,
                     float* d_rgb, float* d_alpha, cudaStream_t s, const LossTargets* lt) {
  Workspace& w = m.ws;
  TrainCompositeArgs A{n_rays, N, eps, w.ray_first.ptr, w.ray_count.ptr, w.sidx.ptr, w.sdelta.ptr, w.snroot.ptr,
                       w.sbase.ptr, w.pres.ptr, w.strans.ptr, d_dC, d_dA, nullptr, nullptr, LossCfg{}, 0.0, nullptr,
                       d_rgb, d_alpha, w.pgs.ptr, w.pgc.ptr, w.pflag.ptr};
  if (lt) {
    A.gt_rgb = lt->gt_rgb;
    A.gt_alpha = lt->gt_alpha;
    A.loss = LossCfg{lt->w_rgb, lt->w_alpha, lt->w_hard, lt->w_density, lt->huber_delta};
    A.inv_n = 1.0 / static_cast<double>(n_rays);
    A.ray_terms = lt->ray_terms;
  }
  m.prof.begin("train_composite", s);
  train_composite_kernel<<<static_cast<unsigned>(std::max<long long>(1, (n_rays + 127) / 128)), 128, 0, s>>>(A);
  ARFX_CUDA(cudaGetLastError());
  m.prof.end(s);
}

namespace {
// loss4 = (L_rgb, L_alpha, L_hard, w_rgb L_rgb + w_alpha L_alpha + w_hard L_hard): batch means of
// the per-ray terms; one block, fixed strided order + fixed tree -> deterministic
__global__ void __launch_bounds__(256) loss_reduce_kernel(const double* __restrict__ t, long long n, LossCfg L,
                                                          double* __restrict__ out4) {
  __shared__ double sh[3][256];
  double a = 0.0, b = 0.0, c = 0.0;
  for (long long i = threadIdx.x; i < n; i += 256) {
    a += t[3 * i + 0];
    b += t[3 * i + 1];
    c += t[3 * i + 2];
  }
  sh[0][threadIdx.x] = a;
  sh[1][threadIdx.x] = b;
  sh[2][threadIdx.x] = c;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int k = 0; k < 3; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double inv = n > 0 ? 1.0 / static_cast<double>(n) : 0.0;
    const double lr = sh[0][0] * inv, la = sh[1][0] * inv, lh = sh[2][0] * inv;
    out4[0] = lr;
    out4[1] = la;
    out4[2] = lh;
    out4[3] = L.w_rgb * lr + L.w_alpha * la + L.w_hard * lh;
  }
}

__global__ void ray_loss_kernel(long long n, const float* __restrict__ rgb, const float* __restrict__ alpha,
                                const float* __restrict__ gt_rgb, const float* __restrict__ gt_alpha, LossCfg L,
                                double* __restrict__ terms, float* __restrict__ d_rgb, float* __restrict__ d_alpha) {
  const double inv_n = 1.0 / static_cast<double>(n);
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const RayLoss o = ray_loss(rgb[3 * r], rgb[3 * r + 1], rgb[3 * r + 2], alpha[r], gt_rgb + 3 * r, gt_alpha[r], L,
                               inv_n);
    terms[3 * r + 0] = o.rgb;
    terms[3 * r + 1] = o.alpha;
    terms[3 * r + 2] = o.hard;
    if (d_rgb) {
      d_rgb[3 * r + 0] = o.dC[0];
      d_rgb[3 * r + 1] = o.dC[1];
      d_rgb[3 * r + 2] = o.dC[2];
    }
    if (d_alpha) d_alpha[r] = o.dA;
  }
}
}  // namespace

void loss_reduce(const double* d_terms, long long n, const LossTargets& lt, double* d_out4, cudaStream_t s) {
  loss_reduce_kernel<<<1, 256, 0, s>>>(d_terms, n, LossCfg{lt.w_rgb, lt.w_alpha, lt.w_hard, lt.w_density,
                                                           lt.huber_delta}, d_out4);
  ARFX_CUDA(cudaGetLastError());
}

void ray_losses(long long n, const float* d_rgb, const float* d_alpha, const LossTargets& lt, float* d_grad_rgb,
                float* d_grad_alpha, cudaStream_t s) {
  if (n <= 0) return;
  ray_loss_kernel<<<static_cast<unsigned>(std::min<long long>((n + 127) / 128, 4096)), 128, 0, s>>>(
      n, d_rgb, d_alpha, lt.gt_rgb, lt.gt_alpha,
      LossCfg{lt.w_rgb, lt.w_alpha, lt.w_hard, lt.w_density, lt.huber_delta}, lt.ray_terms, d_grad_rgb, d_grad_alpha);
  ARFX_CUDA(cudaGetLastError());
}

}  // namespace arfx
