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


// K8a: one thread per flagged pool entry (query): exact forward recompute (encode + MLP
// in the reference's summation order, activations in smem as [k][thread], conflict-free),
// then the per-query half of DecoderMlp::backward (R/mlp.hpp:116-154): logit deltas, the
// dprev chains through ReLU masks, the hash-grid scatter (R/hash_grid.hpp:155-169, f32
// atomics). The operands of the weight gradients (inputs and deltas of each layer) go to a
// compacted per-query record; K8b reduces them over queries.
constexpr int kBwdRec = kIn + kHid + kHid + kOut + kHid + kHid;  // X, H1, H2, u2, dh2, dh1 = 292 floats
constexpr int kRecX = 0, kRecH1 = kIn, kRecH2 = kIn + kHid, kRecU2 = kIn + 2 * kHid, kRecD2 = kRecU2 + kOut,
              kRecD1 = kRecD2 + kHid;

__global__ void __launch_bounds__(kFbThreads) field_bwd_query_kernel(FieldView F, const double* __restrict__ px,
                                                                     const double* __restrict__ py,
                                                                     const double* __restrict__ pz,
                                                                     const uint8_t* __restrict__ pflag,
                                                                     const float* __restrict__ pgs,
                                                                     const float* __restrict__ pgc,
                                                                     const unsigned long long* n_dev, long long cap,
                                                                     float* __restrict__ grid_grad,
                                                                     float* __restrict__ rec, long long rec_cap,
                                                                     unsigned long long* n_rec) {
  extern __shared__ float fb_smem[];
  const int t = threadIdx.x, lane = t & 31;
  float* X = fb_smem;                    // [kIn][kFbThreads]
  float* H1 = X + kIn * kFbThreads;      // [kHid][kFbThreads]
  float* H2 = H1 + kHid * kFbThreads;    // [kHid][kFbThreads]
  float* D = H2 + kHid * kFbThreads;     // [kHid][kFbThreads]
  const float* W0 = F.mlp;
  const float* B0 = W0 + kIn * kHid;
  const float* W1 = B0 + kHid;
  const float* B1 = W1 + kHid * kHid;
  const float* W2 = B1 + kHid;
  const float* B2 = W2 + kOut * kHid;
  long long n = static_cast<long long>(*n_dev);
  n = n < cap ? n : cap;
  for (long long base = static_cast<long long>(blockIdx.x) * kFbThreads; base < n;
       base += static_cast<long long>(gridDim.x) * kFbThreads) {
    const long long q = base + t;
    const bool act = q < n && pflag[q] != 0;
    const unsigned am = __ballot_sync(0xffffffffu, act);
    if (!am) continue;  // warp-uniform: the whole warp skips unflagged stretches of the pool
    long long slot = 0;
    if (lane == 0) slot = static_cast<long long>(atomicAdd(n_rec, static_cast<unsigned long long>(__popc(am))));
    slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(am & ((1u << lane) - 1u));
    if (!act) continue;
    float* R = rec + (slot < rec_cap ? slot : rec_cap) * kBwdRec;  // rec holds rec_cap + 1 records
    const d3 x = make3(px[q], py[q], pz[q]);
    // ---- forward recompute (CanonicalField::query_backward re-runs the forward) ----
    float feats[kIn];
    hash_encode_f2(F, x, feats);
    for (int i = 0; i < kIn; ++i) {
      X[i * kFbThreads + t] = feats[i];
      R[kRecX + i] = feats[i];
    }
    for (int o = 0; o < kHid; ++o) {
      float a = B0[o];
      for (int i = 0; i < kIn; ++i) a = fadd(a, fmul(__ldg(W0 + o * kIn + i), feats[i]));
      const float h = (a < 0.0f) ? 0.0f : a;
      H1[o * kFbThreads + t] = h;
      R[kRecH1 + o] = h;
    }
    for (int o = 0; o < kHid; ++o) {
      float a = B1[o];
      for (int i = 0; i < kHid; ++i) a = fadd(a, fmul(__ldg(W1 + o * kHid + i), H1[i * kFbThreads + t]));
      const float h = (a < 0.0f) ? 0.0f : a;
      H2[o * kFbThreads + t] = h;
      R[kRecH2 + o] = h;
    }
    float lg[kOut];
    for (int o = 0; o < kOut; ++o) {
      float a = B2[o];
      for (int i = 0; i < kHid; ++i) a = fadd(a, fmul(__ldg(W2 + o * kHid + i), H2[i * kFbThreads + t]));
      lg[o] = a;
    }
    // ---- d logits (R/field.hpp:95-99) ----
    float u2[kOut];
    u2[0] = fmul(pgs[q], logistic_f(lg[0]));
    for (int c = 0; c < 3; ++c) {
      const float v = logistic_f(lg[1 + c]);
      u2[1 + c] = fmul(fmul(pgc[3 * q + c], v), __fsub_rn(1.0f, v));
    }
    for (int o = 0; o < kOut; ++o) R[kRecU2 + o] = u2[o];
    // ---- dprev through the output layer (u != 0 only), ReLU mask of hidden layer 2 ----
    for (int i = 0; i < kHid; ++i) D[i * kFbThreads + t] = 0.0f;
    for (int o = 0; o < kOut; ++o) {
      const float u = u2[o];
      if (u != 0.0f)
        for (int i = 0; i < kHid; ++i) D[i * kFbThreads + t] = fadd(D[i * kFbThreads + t], fmul(u, __ldg(W2 + o * kHid + i)));
    }
    for (int i = 0; i < kHid; ++i) {
      const float d = (H2[i * kFbThreads + t] == 0.0f) ? 0.0f : D[i * kFbThreads + t];
      H2[i * kFbThreads + t] = d;  // H2 now holds d h2
      R[kRecD2 + i] = d;
    }
    // ---- hidden layer 1 ----
    for (int i = 0; i < kHid; ++i) D[i * kFbThreads + t] = 0.0f;
    for (int o = 0; o < kHid; ++o) {
      const float u = H2[o * kFbThreads + t];
      if (u != 0.0f)
        for (int i = 0; i < kHid; ++i) D[i * kFbThreads + t] = fadd(D[i * kFbThreads + t], fmul(u, __ldg(W1 + o * kHid + i)));
    }
    for (int i = 0; i < kHid; ++i) {
      const float d = (H1[i * kFbThreads + t] == 0.0f) ? 0.0f : D[i * kFbThreads + t];
      H1[i * kFbThreads + t] = d;  // H1 now holds d h1
      R[kRecD1 + i] = d;
    }
    // ---- first layer -> d features ----
    float din[kIn];
    for (int i = 0; i < kIn; ++i) din[i] = 0.0f;
    for (int o = 0; o < kHid; ++o) {
      const float u = H1[o * kFbThreads + t];
      if (u != 0.0f)
        for (int i = 0; i < kIn; ++i) din[i] = fadd(din[i], fmul(u, __ldg(W0 + o * kIn + i)));
    }
    // ---- encode backward (R/hash_grid.hpp:155-169) ----
    double uu[3];
    normalize_point(F, x, uu);
    for (int l = 0; l < F.L; ++l) {
      LevelCorners lc;
      level_corners(F, l, uu, lc);
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

// K8b: MLP weight / bias gradients, gW[o][i] = sum_q delta[q][o] * in[q][i] and gb[o] =
// sum_q delta[q][o], over the K8a records: a block stages kWq records in smem (row-major,
// so threads walking i read consecutive words) and each thread owns a strided set of the
// 6,532 parameters; one f32 atomic per parameter per block.
constexpr int kWq = 32;
constexpr int kWThreads = 256;
__global__ void __launch_bounds__(kWThreads) field_bwd_weights_kernel(const float* __restrict__ rec,
                                                                      const unsigned long long* n_rec,
                                                                      long long rec_cap,
                                                                      float* __restrict__ mlp_grad) {
  __shared__ float S[kWq][kBwdRec + 1];
  long long n = static_cast<long long>(*n_rec);
  n = n < rec_cap ? n : rec_cap;
  constexpr int kW0 = kHid * kIn, kB0 = kW0 + kHid, kW1 = kB0 + kHid * kHid, kB1 = kW1 + kHid,
                kW2 = kB1 + kOut * kHid, kB2 = kW2 + kOut;
  for (long long c0 = static_cast<long long>(blockIdx.x) * kWq; c0 < n; c0 += static_cast<long long>(gridDim.x) * kWq) {
    const int nq = static_cast<int>(n - c0 < kWq ? n - c0 : kWq);
    __syncthreads();
    for (int e = threadIdx.x; e < nq * kBwdRec; e += kWThreads) S[e / kBwdRec][e % kBwdRec] = rec[c0 * kBwdRec + e];
    __syncthreads();
    for (int p = threadIdx.x; p < kB2; p += kWThreads) {
      int dOff, iOff, o, i;  // delta offset / input offset (-1: bias)
      if (p < kW0) {
        o = p / kIn, i = p % kIn, dOff = kRecD1, iOff = kRecX;
      } else if (p < kB0) {
        o = p - kW0, i = 0, dOff = kRecD1, iOff = -1;
      } else if (p < kW1) {
        o = (p - kB0) / kHid, i = (p - kB0) % kHid, dOff = kRecD2, iOff = kRecH1;
      } else if (p < kB1) {
        o = p - kW1, i = 0, dOff = kRecD2, iOff = -1;
      } else if (p < kW2) {
        o = (p - kB1) / kHid, i = (p - kB1) % kHid, dOff = kRecU2, iOff = kRecH2;
      } else {
        o = p - kW2, i = 0, dOff = kRecU2, iOff = -1;
      }
      float acc = 0.0f;
      if (iOff >= 0)
        for (int qq = 0; qq < nq; ++qq) acc = fadd(acc, fmul(S[qq][dOff + o], S[qq][iOff + i]));
      else
        for (int qq = 0; qq < nq; ++qq) acc = fadd(acc, S[qq][dOff + o]);
      if (acc != 0.0f) atomicAdd(mlp_grad + p, acc);
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
    ARFX_CUDA(cudaFuncSetAttribute(field_bwd_query_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    attr = true;
  }
  Workspace& w = m.ws;
  const long long rec_cap = cap;
  w.bwd_rec.ensure(static_cast<size_t>(rec_cap + 1) * kBwdRec);
  w.bwd_n.ensure(1);
  ARFX_CUDA(cudaMemsetAsync(w.bwd_n.ptr, 0, sizeof(unsigned long long), s));
  const long long blocks = std::min<long long>((cap + kFbThreads - 1) / kFbThreads, static_cast<long long>(sms()) * 8);
  m.prof.begin("field_backward", s);
  field_bwd_query_kernel<<<static_cast<unsigned>(std::max<long long>(blocks, 1)), kFbThreads, smem, s>>>(
      m.fv, w.px.ptr, w.py.ptr, w.pz.ptr, flag, gs, gc, d_n, cap, m.grid_grad.ptr, w.bwd_rec.ptr, rec_cap,
      w.bwd_n.ptr);
  ARFX_CUDA(cudaGetLastError());
  field_bwd_weights_kernel<<<static_cast<unsigned>(sms() * 4), kWThreads, 0, s>>>(w.bwd_rec.ptr, w.bwd_n.ptr, rec_cap,
                                                                                m.mlp_grad.ptr);
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
