// train.cu -- training forward + backward on sm_100a.
//
// The reference has no training function; the step is composed from its pieces exactly
// as oracle/ref_driver.cpp arfr_train_fwd_bwd does: per ray the render forward
// (stratified), composite_backward (R/render.hpp:125-157) with upstream dL/dC, dL/dA,
// then CanonicalField::query_backward (R/field.hpp:91-103) at every accumulated
// non-skipped sample's selected canonical root, accumulated into FieldGrads.
//
//   K1..K3 as in render (march in ray-list mode, deformer, exact field over the pool)
//   K7  train_composite_warp_kernel  warp per ray: selection + composite forward (rgb, alpha,
//                               terminated_at), the SPEC losses and their gradient when
//                               targets are given (losses.cuh), then the exact reverse
//                               pass; dsigma / dc land on the selected root's pool entry
//   K8a flag_list + field_bwd_team_kernel  64-thread team per 4 flagged queries: forward
//                               recompute (bit-identical to K3), dprev chains in the
//                               reference's order, per-query records of layer inputs/deltas
//   K8c grid_scatter_kernel     warp-aggregated hash-grid scatter-add (R/hash_grid.hpp:155-169)
//   K8b/K8d field_bwd_weights + weights_reduce  MLP weight gradients over the records,
//                               register-accumulated per CTA, fixed-order row reduction
// Gradient sums are order-different from the reference's serial per-thread buffers
// (SPEC.md:426 allows reassociation); everything upstream is bit-exact.
#include <cuda_runtime.h>

#include <algorithm>

#include "field.cuh"
#include "fixed.cuh"
#include "losses.cuh"
#include "model.h"
#include "umma.cuh"

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
  const int32_t *gpx, *gpy;  // gt_w > 0: targets are frames read at the ray's pixel
  long long gt_w, gt_h;
  LossCfg loss;
  double inv_n;
  double* ray_terms;  // [n_rays][3] unweighted per-ray loss terms
  float *rgb, *alpha;
  float* pgs;      // per pool entry: dsigma (f32, as passed to query_backward)
  float* pgc;      // per pool entry: dcolor[3]
  uint8_t* pflag;  // per pool entry: needs query_backward
};

// K7, warp per ray: lanes take 32 consecutive samples at a time and do the independent
// per-sample work in parallel (root selection, alpha = -expm1(-sigma delta), the gradient
// outputs); only the reference's sequential recurrences -- T, C, A forward and the suffix
// C^, A^ backward -- walk the samples one by one, every lane running the same chain on
// values broadcast by shuffle. Same operations in the same order as the per-sample loop
// of R/render.hpp:98-157, so bit-identical; a 4,096-ray batch fills 4,096 warps instead
// of 32 blocks of threads.
__device__ __forceinline__ double shfl_dd(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

__global__ void __launch_bounds__(128) train_composite_warp_kernel(TrainCompositeArgs A) {
  const int lane = threadIdx.x & 31;
  for (long long r = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < A.n_rays;
       r += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const int first = A.ray_first[r], cnt = A.ray_count[r];
    // ---- forward (composite R/render.hpp:98-119) ----
    double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0, acc = 0.0;
    int m = A.N;  // terminated_at
    if (A.eps > 0 && T <= A.eps) m = 0;
    for (int c0 = 0; c0 < cnt && m == A.N; c0 += 32) {
      const int j = c0 + lane;
      const long long s = first + j;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      double alpha = 0.0;
      bool contrib = false;
      int sid = 0;
      if (j < cnt) {
        const int sel = select_root_t(A.snroot, A.sbase, A.pres, s, v);
        contrib = sel >= 0 && static_cast<double>(v.x) > 0.0;
        if (contrib) alpha = -expm1(-__dmul_rn(static_cast<double>(v.x), A.sdelta[s]));
        sid = A.sidx[s];
      }
      const unsigned cmask = __ballot_sync(0xffffffffu, contrib);
      const int kn = min(32, cnt - c0);
      double myT = 0.0;
      int k = 0;
      for (; k < kn; ++k) {  // uniform across the warp
        if (lane == k) myT = T;
        if (!((cmask >> k) & 1u)) continue;
        const double a = shfl_dd(alpha, k);
        const double w = __dmul_rn(a, T);
        cr = __dadd_rn(cr, __dmul_rn(static_cast<double>(__shfl_sync(0xffffffffu, v.y, k)), w));
        cg = __dadd_rn(cg, __dmul_rn(static_cast<double>(__shfl_sync(0xffffffffu, v.z, k)), w));
        cb = __dadd_rn(cb, __dmul_rn(static_cast<double>(__shfl_sync(0xffffffffu, v.w, k)), w));
        acc = __dadd_rn(acc, w);
        T = __dmul_rn(T, __dsub_rn(1.0, a));
        if (A.eps > 0 && T <= A.eps) {
          m = __shfl_sync(0xffffffffu, sid, k) + 1;
          ++k;
          break;
        }
      }
      if (lane < k) A.strans[s] = myT;  // samples the forward visited
    }
    if (cnt == 0) m = 0;
    const float fr = static_cast<float>(cr), fg = static_cast<float>(cg), fb = static_cast<float>(cb);
    const float fa = static_cast<float>(acc);
    // ---- upstream: given, or the fused loss gradient of this ray (uniform in the warp) ----
    double dcx, dcy, dcz, da;
    if (A.gt_rgb) {
      const float zero3[3] = {0.0f, 0.0f, 0.0f};
      const float* grgb = A.gt_rgb + 3 * r;
      float galpha = 0.0f;
      if (A.gt_w > 0) {
        const long long x = A.gpx[r], y = A.gpy[r];
        const bool in = x >= 0 && y >= 0 && x < A.gt_w && y < A.gt_h;
        grgb = in ? A.gt_rgb + 3 * (y * A.gt_w + x) : zero3;
        galpha = in ? A.gt_alpha[y * A.gt_w + x] : 0.0f;
      } else {
        galpha = A.gt_alpha[r];
      }
      const RayLoss L = ray_loss(fr, fg, fb, fa, grgb, galpha, A.loss, A.inv_n);
      if (lane == 0) {
        A.ray_terms[3 * r + 0] = L.rgb;
        A.ray_terms[3 * r + 1] = L.alpha;
        A.ray_terms[3 * r + 2] = L.hard;
      }
      dcx = L.dC[0], dcy = L.dC[1], dcz = L.dC[2], da = L.dA;
    } else {
      dcx = A.dC[3 * r + 0], dcy = A.dC[3 * r + 1], dcz = A.dC[3 * r + 2], da = A.dA[r];
    }
    if (lane == 0) {
      A.rgb[3 * r + 0] = fr;
      A.rgb[3 * r + 1] = fg;
      A.rgb[3 * r + 2] = fb;
      A.alpha[r] = fa;
    }
    // ---- backward (composite_backward R/render.hpp:125-157), reverse over i < m ----
    double chx = 0.0, chy = 0.0, chz = 0.0, ahat = 0.0;
    for (int c0 = ((cnt - 1) / 32) * 32; cnt > 0 && c0 >= 0; c0 -= 32) {
      const int j = c0 + lane;
      const long long s = first + j;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      int sel = -1;
      double alpha = 0.0;
      if (j < cnt && A.sidx[s] < m) {
        sel = select_root_t(A.snroot, A.sbase, A.pres, s, v);
        if (sel >= 0 && static_cast<double>(v.x) > 0.0)
          alpha = -expm1(-__dmul_rn(static_cast<double>(v.x), A.sdelta[s]));
      }
      const unsigned vmask = __ballot_sync(0xffffffffu, sel >= 0);
      if (!vmask) continue;
      double mx = 0.0, my = 0.0, mz = 0.0, ma = 0.0;  // C^, A^ seen by this lane's sample
      for (int k = 31 - __clz(vmask); k >= 0; --k) {  // uniform, reverse sample order
        if (!((vmask >> k) & 1u)) continue;
        if (lane == k) mx = chx, my = chy, mz = chz, ma = ahat;
        const double a = shfl_dd(alpha, k);
        const double om = __dsub_rn(1.0, a);
        chx = __dadd_rn(__dmul_rn(static_cast<double>(__shfl_sync(0xffffffffu, v.y, k)), a), __dmul_rn(chx, om));
        chy = __dadd_rn(__dmul_rn(static_cast<double>(__shfl_sync(0xffffffffu, v.z, k)), a), __dmul_rn(chy, om));
        chz = __dadd_rn(__dmul_rn(static_cast<double>(__shfl_sync(0xffffffffu, v.w, k)), a), __dmul_rn(chz, om));
        ahat = __dadd_rn(a, __dmul_rn(ahat, om));
      }
      if (sel >= 0) {
        const double cx = static_cast<double>(v.y), cy = static_cast<double>(v.z), cz = static_cast<double>(v.w);
        const double dCda = __dadd_rn(__dadd_rn(__dmul_rn(dcx, __dsub_rn(cx, mx)), __dmul_rn(dcy, __dsub_rn(cy, my))),
                                      __dmul_rn(dcz, __dsub_rn(cz, mz)));
        const double dAda = __dsub_rn(1.0, ma);
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
      }
    }
  }
}

constexpr int kIn = 32, kHid = 64, kOut = 4;


// K8a: one 64-thread team per flagged pool entry (query), 4 teams per block, the decoder
// weights staged once per block in smem (rows padded: conflict-free both for row-wise
// forward dots and column-wise backward dots). Thread l < 16 encodes level l; thread o
// computes hidden unit o of each layer with its inputs in the reference's order, so the
// forward recompute is bit-identical to K3's; the backward dprev chains (R/mlp.hpp:116-154,
// u != 0 only, ReLU mask where post == 0) run one output per thread in the reference's
// o-order; thread l < 16 scatters level l of the encode backward (R/hash_grid.hpp:155-169,
// f32 atomics). The layer inputs and deltas go to a per-query record for K8b.
constexpr int kBwdRec = kIn + kHid + kHid + kOut + kHid + kHid;  // X, H1, H2, u2, dh2, dh1 = 292 floats
constexpr int kRecX = 0, kRecH1 = kIn, kRecH2 = kIn + kHid, kRecU2 = kIn + 2 * kHid, kRecD2 = kRecU2 + kOut,
              kRecD1 = kRecD2 + kHid;
constexpr int kTeam = 64, kTeams = 4, kTeamThreads = kTeam * kTeams;
constexpr int kRecDin = kBwdRec;                  // + d features (32) for the scatter kernel
constexpr int kRecStride = kBwdRec + kIn;         // floats per query record in global memory
constexpr int kTeamSmem = kRecStride + kOut;      // record + d features + logits
constexpr int kW0s = kIn + 1, kW1s = kHid + 1;  // padded row strides


__global__ void flag_list_kernel(const uint8_t* __restrict__ pflag, const unsigned long long* n_dev, long long cap,
                                 int32_t* __restrict__ list, unsigned long long* n_list) {
  long long n = static_cast<long long>(*n_dev);
  n = n < cap ? n : cap;
  const int lane = threadIdx.x & 31;
  for (long long base = static_cast<long long>(blockIdx.x) * blockDim.x; base < n;
       base += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long q = base + threadIdx.x;
    const bool f = q < n && pflag[q] != 0;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (!m) continue;
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(n_list, static_cast<unsigned long long>(__popc(m)));
    b = __shfl_sync(0xffffffffu, b, 0);
    if (f) list[b + __popc(m & ((1u << lane) - 1u))] = static_cast<int32_t>(q);
  }
}

__device__ __forceinline__ void team_sync(int team) {
  asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "n"(kTeam) : "memory");
}

// A team carries kTQ queries at once: the 64 threads cover 16 levels x 4 queries in the
// encode phases, and each hidden-unit thread runs kTQ independent dot-product chains (one
// weight load serves all of them), so no phase leaves most of the team idle at a barrier.
constexpr int kTQ = 4;

__global__ void __launch_bounds__(kTeamThreads) field_bwd_team_kernel(FieldView F, const double* __restrict__ px,
                                                                      const double* __restrict__ py,
                                                                      const double* __restrict__ pz,
                                                                      const int32_t* __restrict__ list,
                                                                      const unsigned long long* n_list,
                                                                      const float* __restrict__ pgs,
                                                                      const float* __restrict__ pgc,
                                                                      float* __restrict__ grid_grad,
                                                                      float* __restrict__ rec,
                                                                      const float* __restrict__ act,
                                                                      const unsigned long long* pool_n,
                                                                      bool tc_active) {
  // the tensor-core backward (field_bwd_tc_kernel) takes every launch with saved activations
  if (tc_active && act != nullptr && static_cast<long long>(*pool_n) <= kTeamMaxQueries) return;
  extern __shared__ float bw_smem[];
  float* W0p = bw_smem;                    // [64][33]
  float* W1p = W0p + kHid * kW0s;          // [64][65]
  float* W2p = W1p + kHid * kW1s;          // [4][65]
  float* Bs = W2p + kOut * kW1s;           // b0[64] b1[64] b2[4]
  float* TS = Bs + 2 * kHid + kOut;        // [kTeams][kTQ][kTeamSmem]
  const float* W = F.mlp;
  for (int e = threadIdx.x; e < kHid * kIn; e += kTeamThreads) W0p[(e / kIn) * kW0s + e % kIn] = __ldg(W + e);
  const float* W1g = W + kIn * kHid + kHid;
  for (int e = threadIdx.x; e < kHid * kHid; e += kTeamThreads) W1p[(e / kHid) * kW1s + e % kHid] = __ldg(W1g + e);
  const float* W2g = W1g + kHid * kHid + kHid;
  for (int e = threadIdx.x; e < kOut * kHid; e += kTeamThreads) W2p[(e / kHid) * kW1s + e % kHid] = __ldg(W2g + e);
  for (int e = threadIdx.x; e < kHid; e += kTeamThreads) {
    Bs[e] = __ldg(W + kIn * kHid + e);
    Bs[kHid + e] = __ldg(W1g + kHid * kHid + e);
  }
  if (threadIdx.x < kOut) Bs[2 * kHid + threadIdx.x] = __ldg(W2g + kOut * kHid + threadIdx.x);
  __syncthreads();
  const int team = threadIdx.x / kTeam, t = threadIdx.x % kTeam;
  float* S0 = TS + team * kTQ * kTeamSmem;
  auto S = [&](int j) { return S0 + j * kTeamSmem; };
  const long long n = static_cast<long long>(*n_list);
  // the forward's saved activations are valid when it ran the team decoder (pool <= 64 Ki)
  const bool use_act = act != nullptr && static_cast<long long>(*pool_n) <= kTeamMaxQueries;
  const int ej = t >> 4, el = t & 15;  // encode phases: query ej, level el
  for (long long k0 = (static_cast<long long>(blockIdx.x) * kTeams + team) * kTQ; k0 < n;
       k0 += static_cast<long long>(gridDim.x) * kTeams * kTQ) {
    const int nq = static_cast<int>(n - k0 < kTQ ? n - k0 : kTQ);
    if (use_act) {  // X | H1 | H2 | logits as the forward computed them (bit-identical)
      for (int j = 0; j < nq; ++j) {
        const float* A = act + static_cast<long long>(list[k0 + j]) * kActStride;
        if (t < kIn) S(j)[kRecX + t] = A[t];
        S(j)[kRecH1 + t] = A[kIn + t];
        S(j)[kRecH2 + t] = A[kIn + kHid + t];
        if (t < kOut) S(j)[kRecStride + t] = A[kIn + 2 * kHid + t];
      }
      team_sync(team);
    } else {
    // ---- encode (thread = (query ej, level el)) ----
    double u[3] = {0.0, 0.0, 0.0};
    long long qe = -1;
    if (ej < nq) {
      qe = list[k0 + ej];
      normalize_point(F, make3(px[qe], py[qe], pz[qe]), u);
      const float2 o = encode_level_f2(F, el, u);
      S(ej)[kRecX + 2 * el] = o.x;
      S(ej)[kRecX + 2 * el + 1] = o.y;
    }
    team_sync(team);
    {  // hidden layer 1 (R/mlp.hpp:100-104 order), kTQ chains
      float a[kTQ];
#pragma unroll
      for (int j = 0; j < kTQ; ++j) a[j] = Bs[t];
      for (int i = 0; i < kIn; ++i) {
        const float w = W0p[t * kW0s + i];
#pragma unroll
        for (int j = 0; j < kTQ; ++j) a[j] = fadd(a[j], fmul(w, S(j)[kRecX + i]));
      }
#pragma unroll
      for (int j = 0; j < kTQ; ++j) S(j)[kRecH1 + t] = (a[j] < 0.0f) ? 0.0f : a[j];
    }
    team_sync(team);
    {
      float a[kTQ];
#pragma unroll
      for (int j = 0; j < kTQ; ++j) a[j] = Bs[kHid + t];
      for (int i = 0; i < kHid; ++i) {
        const float w = W1p[t * kW1s + i];
#pragma unroll
        for (int j = 0; j < kTQ; ++j) a[j] = fadd(a[j], fmul(w, S(j)[kRecH1 + i]));
      }
#pragma unroll
      for (int j = 0; j < kTQ; ++j) S(j)[kRecH2 + t] = (a[j] < 0.0f) ? 0.0f : a[j];
    }
    team_sync(team);
    }  // recompute
    if (t < kTQ * kOut) {  // logits + d logits (R/field.hpp:95-99), thread = (query, output)
      const int j = t / kOut, o = t % kOut;
      if (j < nq) {
        const long long q = list[k0 + j];
        float a;
        if (use_act) {
          a = S(j)[kRecStride + o];
        } else {
          a = Bs[2 * kHid + o];
          for (int i = 0; i < kHid; ++i) a = fadd(a, fmul(W2p[o * kW1s + i], S(j)[kRecH2 + i]));
        }
        float uo;
        if (o == 0) {
          uo = fmul(pgs[q], logistic_f(a));
        } else {
          const float v = logistic_f(a);
          uo = fmul(fmul(pgc[3 * q + o - 1], v), __fsub_rn(1.0f, v));
        }
        S(j)[kRecU2 + o] = uo;
        S(j)[kRecStride + o] = a;
      } else {
        S(j)[kRecU2 + o] = 0.0f;
      }
    }
    team_sync(team);
    {  // dprev through the output layer (u != 0 only), ReLU mask of hidden layer 2
      float d[kTQ];
#pragma unroll
      for (int j = 0; j < kTQ; ++j) d[j] = 0.0f;
      for (int o = 0; o < kOut; ++o) {
        const float w = W2p[o * kW1s + t];
#pragma unroll
        for (int j = 0; j < kTQ; ++j) {
          const float uo = S(j)[kRecU2 + o];
          if (uo != 0.0f) d[j] = fadd(d[j], fmul(uo, w));
        }
      }
#pragma unroll
      for (int j = 0; j < kTQ; ++j) S(j)[kRecD2 + t] = (S(j)[kRecH2 + t] == 0.0f) ? 0.0f : d[j];
    }
    team_sync(team);
    {
      float d[kTQ];
#pragma unroll
      for (int j = 0; j < kTQ; ++j) d[j] = 0.0f;
      for (int o = 0; o < kHid; ++o) {
        const float w = W1p[o * kW1s + t];
#pragma unroll
        for (int j = 0; j < kTQ; ++j) {
          const float uo = S(j)[kRecD2 + o];
          if (uo != 0.0f) d[j] = fadd(d[j], fmul(uo, w));
        }
      }
#pragma unroll
      for (int j = 0; j < kTQ; ++j) S(j)[kRecD1 + t] = (S(j)[kRecH1 + t] == 0.0f) ? 0.0f : d[j];
    }
    team_sync(team);
    {  // d features: thread = (query pair, input i), kTQ / 2 chains each
      const int i = t & (kIn - 1), jb = (t >> 5) * (kTQ / 2);
      float d[kTQ / 2];
#pragma unroll
      for (int j = 0; j < kTQ / 2; ++j) d[j] = 0.0f;
      for (int o = 0; o < kHid; ++o) {
        const float w = W0p[o * kW0s + i];
#pragma unroll
        for (int j = 0; j < kTQ / 2; ++j) {
          const float uo = S(jb + j)[kRecD1 + o];
          if (uo != 0.0f) d[j] = fadd(d[j], fmul(uo, w));
        }
      }
#pragma unroll
      for (int j = 0; j < kTQ / 2; ++j) S(jb + j)[kRecDin + i] = d[j];
    }
    team_sync(team);
    for (int j = 0; j < nq; ++j) {
      float* R = rec + (k0 + j) * kRecStride;
      for (int e = t; e < kRecStride; e += kTeam) R[e] = S(j)[e];
    }
    team_sync(team);
  }
}

// K8c: hash-grid scatter-add of the encode backward (R/hash_grid.hpp:155-169), warp-
// aggregated: a warp takes one level for 32 consecutive queries of the compacted list
// (spatially coherent: the pool follows ray order); lanes whose corner hits the same table
// row are grouped with __match_any_sync and summed by shuffles, and one lane per distinct
// row issues the atomics -- coarse (dense) levels collapse many contributions per row.
template <bool Det>
__global__ void __launch_bounds__(256) grid_scatter_kernel(FieldView F, const double* __restrict__ px,
                                                           const double* __restrict__ py,
                                                           const double* __restrict__ pz,
                                                           const int32_t* __restrict__ list,
                                                           const unsigned long long* n_list,
                                                           const float* __restrict__ rec,
                                                           float* __restrict__ grid_grad,
                                                           long long* __restrict__ grid_acc) {
  const long long n = static_cast<long long>(*n_list);
  const int lane = threadIdx.x & 31;
  const long long chunks = (n + 31) / 32;
  // a warp task = 32 consecutive queries x kScatterLevels levels (1: the most tasks -- more
  // levels per task normalise the point fewer times but were measured slower, 30 -> 35 / 41 /
  // 102 us for 2 / 4 / 16); each level's corners are aggregated over the warp
#ifndef ARFX_SCATTER_LEVELS
#define ARFX_SCATTER_LEVELS 1
#endif
  constexpr int kScatterLevels = ARFX_SCATTER_LEVELS;
  const int groups = (F.L + kScatterLevels - 1) / kScatterLevels;
  const long long total = chunks * groups;
  for (long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; gw < total;
       gw += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const int l0 = static_cast<int>(gw % groups) * kScatterLevels;
    const long long k = (gw / groups) * 32 + lane;
    const bool act = k < n;
    double u[3] = {0.0, 0.0, 0.0};
    if (act) {
      const long long q = list[k];
      normalize_point(F, make3(px[q], py[q], pz[q]), u);
    }
    for (int l = l0; l < l0 + kScatterLevels && l < F.L; ++l) {
      LevelCorners lc;
      float d0 = 0.0f, d1 = 0.0f;
      if (act) {
        level_corners(F, l, u, lc);
        d0 = rec[k * kRecStride + kRecDin + 2 * l];
        d1 = rec[k * kRecStride + kRecDin + 2 * l + 1];
      }
      float* gt = grid_grad + static_cast<size_t>(l) * F.T * 2;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        const bool has = act && lc.w[c] != 0.0f;
        const uint32_t key = has ? lc.idx[c] : 0xffffffffu;
        const float v0 = has ? fmul(lc.w[c], d0) : 0.0f, v1 = has ? fmul(lc.w[c], d1) : 0.0f;
        const unsigned g = __match_any_sync(0xffffffffu, key);
        if (Det) {
          // fixed point: exact integer sums, independent of which lanes / warps meet a row
          long long a0 = f32_to_fix(v0), a1 = f32_to_fix(v1);
          if (g == 0xffffffffu) {  // the whole warp on one row (coarse levels): butterfly
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              a0 += __shfl_xor_sync(0xffffffffu, a0, o);
              a1 += __shfl_xor_sync(0xffffffffu, a1, o);
            }
          } else {
            const long long i0 = a0, i1 = a1;
            a0 = a1 = 0;
            for (unsigned mm = g; mm; mm &= mm - 1) {
              const int src = __ffs(mm) - 1;
              a0 += __shfl_sync(g, i0, src);
              a1 += __shfl_sync(g, i1, src);
            }
          }
          if (has && lane == __ffs(g) - 1) {
            unsigned long long* ga =
                reinterpret_cast<unsigned long long*>(grid_acc + 2 * (static_cast<size_t>(l) * F.T + key));
            atomicAdd(ga + 0, static_cast<unsigned long long>(a0));
            atomicAdd(ga + 1, static_cast<unsigned long long>(a1));
          }
          continue;
        }
        float s0, s1;
        if (g == 0xffffffffu) {  // f32 atomics are unordered anyway: any summation order
          s0 = v0;
          s1 = v1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            s0 = fadd(s0, __shfl_xor_sync(0xffffffffu, s0, o));
            s1 = fadd(s1, __shfl_xor_sync(0xffffffffu, s1, o));
          }
        } else {
          s0 = 0.0f;
          s1 = 0.0f;
          for (unsigned mm = g; mm; mm &= mm - 1) {
            const int src = __ffs(mm) - 1;
            s0 = fadd(s0, __shfl_sync(g, v0, src));
            s1 = fadd(s1, __shfl_sync(g, v1, src));
          }
        }
        // one 8-byte vector atomic per row (sm_90+), both features
        if (has && lane == __ffs(g) - 1) atomicAdd(reinterpret_cast<float2*>(gt) + key, make_float2(s0, s1));
      }
    }
  }
}


// Deterministic mode: the hash-grid gradient stays in grid_acc (exact int64 sums, one per
// grid_grad element) until a consumer needs it -- Adam folds it in during its own sweep
// (optim.cu); anything else calls flush_grad_acc, this sweep: grad += acc * 2^-46 and
// acc = 0 wherever acc != 0 (same f32 expression as Adam's, so both give equal bits).
__global__ void __launch_bounds__(256) grid_flush_kernel(long long n2, longlong2* __restrict__ acc,
                                                         float2* __restrict__ grad) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n2;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const longlong2 a = acc[i];
    if ((a.x | a.y) == 0) continue;
    acc[i] = make_longlong2(0, 0);
    float2 g = grad[i];
    if (a.x) g.x = fadd(g.x, fix_to_f32(a.x));
    if (a.y) g.y = fadd(g.y, fix_to_f32(a.y));
    grad[i] = g;
  }
}

// Deterministic K8 list: flagged pool entries in owner order (training: rays in batch
// order, each ray's samples front to back; L_density: points; query_backward: the pool
// itself), so the K8a records and K8b's per-CTA chunks -- hence the f32 weight-gradient
// sums -- are the same on every run. Count (warp per owner) -> one-block scan -> write.
struct OwnerRanges {
  long long n_owner;
  const int32_t *first, *count;  // target range per owner; nullptr: owner o = target o
  bool pool_is_target;           // the pool entries are the targets (no root lists)
};

__device__ __forceinline__ long long owner_candidate(const OwnerRanges& O, const uint8_t* snroot,
                                                     const int32_t* sbase, const uint8_t* pflag, long long t) {
  if (O.pool_is_target) return pflag[t] ? t : -1;
  const int nr = snroot[t];
  if (nr == 0) return -1;
  const long long b = sbase[t];
  for (int k = 0; k < nr; ++k)
    if (pflag[b + k]) return b + k;  // at most one root per target is flagged (the selected one)
  return -1;
}

template <bool Write>
__global__ void __launch_bounds__(256) owner_list_kernel(OwnerRanges O, const uint8_t* __restrict__ snroot,
                                                         const int32_t* __restrict__ sbase,
                                                         const uint8_t* __restrict__ pflag,
                                                         uint32_t* __restrict__ cnt_or_off,
                                                         int32_t* __restrict__ list) {
  const int lane = threadIdx.x & 31;
  for (long long o = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; o < O.n_owner;
       o += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const long long t0 = O.first ? O.first[o] : o;
    const int nt = O.count ? O.count[o] : 1;
    uint32_t run = Write ? cnt_or_off[o] : 0u;
    for (int j0 = 0; j0 < nt; j0 += 32) {
      const long long q = j0 + lane < nt ? owner_candidate(O, snroot, sbase, pflag, t0 + j0 + lane) : -1;
      const unsigned b = __ballot_sync(0xffffffffu, q >= 0);
      if (Write && q >= 0) list[run + __popc(b & ((1u << lane) - 1u))] = static_cast<int32_t>(q);
      run += __popc(b);
    }
    if (!Write && lane == 0) cnt_or_off[o] = run;
  }
}

__global__ void __launch_bounds__(1024) owner_scan_kernel(uint32_t* __restrict__ a, long long n,
                                                          unsigned long long* __restrict__ total) {
  __shared__ uint32_t ws[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t carry = 0;
  for (long long b0 = 0; b0 < n; b0 += 1024) {
    const long long i = b0 + threadIdx.x;
    const uint32_t v = i < n ? a[i] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = ws[lane];
      uint32_t xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += t;
      }
      ws[lane] = xi - x;
      if (lane == 31) ws[32] = xi;
    }
    __syncthreads();
    if (i < n) a[i] = carry + ws[warp] + incl - v;
    carry += ws[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// K8b: MLP weight / bias gradients, gW[o][i] = sum_q delta[q][o] * in[q][i] and gb[o] =
// sum_q delta[q][o], over the K8a records: a block stages kWq records at a time in smem
// (row-major: threads walking i read consecutive words); each thread owns ~26 of the 6,532
// parameters and accumulates them in registers over all of the block's chunks, then
// writes one partial row; K8d sums the partial rows in block order (deterministic, no
// atomics).
constexpr int kWq = 32;
constexpr int kWThreads = 256;
constexpr int kNParams = kHid * kIn + kHid + kHid * kHid + kHid + kOut * kHid + kOut;  // 6,532
constexpr long long kWMin = 128;
__host__ __device__ __forceinline__ long long wblocks_used(long long n, long long grid) {
  const long long want = (n + kWMin - 1) / kWMin;
  return want < 1 ? 1 : (want < grid ? want : grid);
}

__global__ void __launch_bounds__(kWThreads) field_bwd_weights_kernel(const float* __restrict__ rec,
                                                                      const unsigned long long* n_rec,
                                                                      long long rec_cap,
                                                                      float* __restrict__ partial,
                                                                      const unsigned long long* tc_pool_n) {
  if (tc_pool_n && static_cast<long long>(*tc_pool_n) <= kTeamMaxQueries) return;  // K8-TC wrote the rows
  __shared__ float S[kWq][kRecStride + 1];
  long long n = static_cast<long long>(*n_rec);
  n = n < rec_cap ? n : rec_cap;
  constexpr int kW0 = kHid * kIn, kB0 = kW0 + kHid, kW1 = kB0 + kHid * kHid, kB1 = kW1 + kHid,
                kW2 = kB1 + kOut * kHid, kB2 = kW2 + kOut;
  static_assert(kB2 == kNParams, "parameter count");
  constexpr int kPer = (kB2 + kWThreads - 1) / kWThreads;  // parameters per thread (26)
  int dOff[kPer], iOff[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int p = threadIdx.x + j * kWThreads;
    int d = -1, in = -1;
    if (p < kW0) d = kRecD1 + p / kIn, in = kRecX + p % kIn;
    else if (p < kB0) d = kRecD1 + (p - kW0);
    else if (p < kW1) d = kRecD2 + (p - kB0) / kHid, in = kRecH1 + (p - kB0) % kHid;
    else if (p < kB1) d = kRecD2 + (p - kW1);
    else if (p < kW2) d = kRecU2 + (p - kB1) / kHid, in = kRecH2 + (p - kB1) % kHid;
    else if (p < kB2) d = kRecU2 + (p - kW2);
    dOff[j] = d;
    iOff[j] = in;
  }
  // blocks in use: one per kWMin queries (at most the grid) -- small batches write and reduce
  // only that many partial rows; the split depends on n alone (deterministic)
  const long long used = wblocks_used(n, gridDim.x);
  if (blockIdx.x >= used) return;
  float acc[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) acc[j] = 0.0f;
  for (long long c0 = static_cast<long long>(blockIdx.x) * kWq; c0 < n; c0 += used * kWq) {
    const int nq = static_cast<int>(n - c0 < kWq ? n - c0 : kWq);
    __syncthreads();
    const float* src = rec + c0 * kRecStride;
    for (int e = threadIdx.x; e < nq * kRecStride; e += kWThreads) S[e / kRecStride][e % kRecStride] = src[e];
    __syncthreads();
    for (int qq = 0; qq < nq; ++qq) {
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        if (dOff[j] < 0) continue;
        const float dv = S[qq][dOff[j]];
        acc[j] = fadd(acc[j], iOff[j] >= 0 ? fmul(dv, S[qq][iOff[j]]) : dv);
      }
    }
  }
  float* row = partial + static_cast<size_t>(blockIdx.x) * kNParams;
#pragma unroll
  for (int j = 0; j < kPer; ++j)
    if (dOff[j] >= 0) row[threadIdx.x + j * kWThreads] = acc[j];
}

// K8d: mlp_grad[p] += sum over blocks of partial[b][p]: a block takes 32 parameters, its 8
// warps sum interleaved row subsets (coalesced 128-B rows), then a fixed-order combine --
// deterministic, no atomics
__global__ void __launch_bounds__(256) weights_reduce_kernel(const float* __restrict__ partial, int grid,
                                                             const unsigned long long* n_rec, long long rec_cap,
                                                             float* __restrict__ mlp_grad,
                                                             const unsigned long long* tc_pool_n, int tc_grid) {
  __shared__ float part[8][32];
  long long nr = static_cast<long long>(*n_rec);
  nr = nr < rec_cap ? nr : rec_cap;
  const bool tc = tc_pool_n && static_cast<long long>(*tc_pool_n) <= kTeamMaxQueries;
  const int n_blocks = tc ? tc_grid : static_cast<int>(wblocks_used(nr, grid));
  const int pi = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int p = blockIdx.x * 32 + pi;
  float a = 0.0f;
  if (p < kNParams)
    for (int b = wp; b < n_blocks; b += 8) a = fadd(a, partial[static_cast<size_t>(b) * kNParams + p]);
  part[wp][pi] = a;
  __syncthreads();
  if (wp == 0 && p < kNParams) {
    float t = part[0][pi];
    for (int k = 1; k < 8; ++k) t = fadd(t, part[k][pi]);
    mlp_grad[p] = fadd(mlp_grad[p], t);
  }
}

// ---- K8-TC: the MLP backward on the 5th-gen tensor cores (split-bf16, f32 accumulate) ----
//
// One persistent 128-thread CTA per SM; a tile = 128 consecutive entries of the backward
// list, thread r = row r. Per tile, from the forward's saved activations (X | H1 | H2 |
// logits, bit-identical to a recompute) and the upstream dsigma / dcolor:
//   u2  = d logits (R/field.hpp:95-99)                                SIMT, as K8a
//   d2  = ReLU'(H2) * (u2 . W2)  (R/mlp.hpp:130-150, u != 0 only)     SIMT (K = 4), as K8a
//   dH1 = d2 . W1          D[128 x 64]  = A[q][o] B[i][o]             tcgen05, TMEM cols [0, 64)
//   d1  = ReLU'(H1) * dH1
//   dX  = d1 . W0          D[128 x 32]                                tcgen05, TMEM cols [64, 96)
//   [dW1 | db1 ; dW0 | db0] += [d2^T ; d1^T] . [H1 | X | 1]           tcgen05, K = the tile's
//                          128 queries, accumulated over all of the CTA's tiles in TMEM
//                          cols [128, 240) (rows 0-63: d2^T, rows 64-127: d1^T)
//   dW2, db2 += u2^T . H2 (4 x 64 + 4)                                SIMT over smem, fixed order
// dX goes to the record's d-feature slot for the hash-grid scatter (K8c); each CTA writes
// its MLP-gradient partial row, summed in fixed order by weights_reduce (deterministic).
// Products are hi*hi + hi*lo + lo*hi of bf16 halves (~16 significant bits); the tolerance
// vs the reference's serial f32 sums is the gradient parity bar.
namespace bwdtc {
using namespace umma;
constexpr int kT = 128;   // queries per tile (rows of the MMAs)
constexpr int kThreads = 4 * kT;  // 4 threads per row: column parts
constexpr int kNW = 112;  // weight-grad B rows: H1^T (64) | X^T (32) | ones (1) | zero pad
constexpr int kWB1T = 0;                                   // B for dH1: (n=i 64, k=o 64), 2 planes
constexpr int kW1P = kHid * kHid * 2;
constexpr int kWB0T = kWB1T + 2 * kW1P;                    // B for dX: (n=i 32, k=o 64)
constexpr int kW0P = kIn * kHid * 2;
constexpr int kAD = kWB0T + 2 * kW0P;                      // A for dH1 / dX: (m=q 128, k=o 64)
constexpr int kADP = kT * kHid * 2;
constexpr int kAW = kAD + 2 * kADP;                        // A for the weight grads: (m=128, k=q 128)
constexpr int kAWP = kT * kT * 2;
constexpr int kBW = kAW + 2 * kAWP;                        // B for the weight grads: (n=112, k=q 128)
constexpr int kBWP = kNW * kT * 2;
constexpr int kW2F = kBW + 2 * kBWP;                       // W2 f32 [4][64]
constexpr int kH2F = kW2F + kOut * kHid * 4;               // H2 f32 [128][65]
constexpr int kU2F = kH2F + kT * (kHid + 1) * 4;           // u2 f32 [128][4]
constexpr int kBAR = kU2F + kT * kOut * 4;                 // mbarrier
constexpr int kTADDR = kBAR + 8;
constexpr int kSmem = kTADDR + 8;
constexpr uint32_t kTmemCols = 256;
constexpr int kColDH1 = 0, kColDX = 64, kColW = 128;
constexpr int kColOnes = 96;  // B_w row of ones -> bias gradients

__device__ __forceinline__ void put_split(unsigned char* base, int plane, int off, float x) {
  __nv_bfloat16 hi, lo;
  split_bf16(x, hi, lo);
  *reinterpret_cast<__nv_bfloat16*>(base + off) = hi;
  *reinterpret_cast<__nv_bfloat16*>(base + off + plane) = lo;
}

// row r, k = [c, c + 8) of a K-major split operand with R rows
__device__ __forceinline__ void put_row8(unsigned char* base, int plane, int R, int r, int c, const float* x) {
  __nv_bfloat16 hi[8], lo[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) split_bf16(x[j], hi[j], lo[j]);
  *reinterpret_cast<uint4*>(base + kmaj_off(r, c, R)) = *reinterpret_cast<const uint4*>(hi);
  *reinterpret_cast<uint4*>(base + plane + kmaj_off(r, c, R)) = *reinterpret_cast<const uint4*>(lo);
}
}  // namespace bwdtc

__global__ void __launch_bounds__(bwdtc::kThreads, 1) field_bwd_tc_kernel(FieldView F, const int32_t* __restrict__ list,
                                                                        const unsigned long long* n_list,
                                                                        const float* __restrict__ pgs,
                                                                        const float* __restrict__ pgc,
                                                                        const float* __restrict__ act,
                                                                        const unsigned long long* pool_n,
                                                                        float* __restrict__ rec,
                                                                        float* __restrict__ partial) {
  using namespace bwdtc;
  if (static_cast<long long>(*pool_n) > kTeamMaxQueries) return;  // no saved activations: K8a/K8b run
  extern __shared__ __align__(1024) unsigned char bt_smem[];
  // 4 threads per tile row: r = row (the TMEM lane of warp quadrant warp % 4), p = column part
  const int tid = threadIdx.x, warp = tid >> 5;
  const int r = (warp & 3) * 32 + (tid & 31), p = warp >> 2;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(bt_smem));
  const uint32_t mbar = sbase + kBAR;
  float* W2f = reinterpret_cast<float*>(bt_smem + kW2F);
  float* H2f = reinterpret_cast<float*>(bt_smem + kH2F);
  float* U2f = reinterpret_cast<float*>(bt_smem + kU2F);
  const long long n = static_cast<long long>(*n_list);
  // ---- weights: B operands (W1^T, W0^T: element (n = i, k = o) = W[o][i]), W2 in f32 ----
  const float* W0 = F.mlp;
  const float* W1 = W0 + kIn * kHid + kHid;
  const float* W2 = W1 + kHid * kHid + kHid;
  {  // all weight loads in flight before the first conversion (one L2 round trip)
    constexpr int n1 = kHid * kHid / kThreads, n0 = kHid * kIn / kThreads;
    float w1[n1], w0[n0], w2 = 0.0f;
#pragma unroll
    for (int j = 0; j < n1; ++j) w1[j] = __ldg(W1 + tid + j * kThreads);
#pragma unroll
    for (int j = 0; j < n0; ++j) w0[j] = __ldg(W0 + tid + j * kThreads);
    if (tid < kOut * kHid) w2 = __ldg(W2 + tid);
#pragma unroll
    for (int j = 0; j < n1; ++j) {
      const int e = tid + j * kThreads, o = e / kHid, i = e % kHid;
      put_split(bt_smem + kWB1T, kW1P, kmaj_off(i, o, kHid), w1[j]);
    }
#pragma unroll
    for (int j = 0; j < n0; ++j) {
      const int e = tid + j * kThreads, o = e / kIn, i = e % kIn;
      put_split(bt_smem + kWB0T, kW0P, kmaj_off(i, o, kIn), w0[j]);
    }
    if (tid < kOut * kHid) W2f[tid] = w2;
  }
  // B_w rows 96..111 (ones row for the bias gradients, zero padding) are constant
  for (int e = tid; e < (kNW - kColOnes) * kT; e += kThreads) {
    const int nrow = kColOnes + e / kT, k = e % kT;
    put_split(bt_smem + kBW, kBWP, kmaj_off(nrow, k, kNW), nrow == kColOnes ? 1.0f : 0.0f);
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sbase + kTADDR),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<uint32_t*>(bt_smem + kTADDR);
  const uint32_t trow = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  uint32_t phase = 0;
  float acc2 = 0.0f;  // dW2 (tid < 256: o = tid / 64, i = tid % 64) or db2 (256 <= tid < 260)
  bool any = false;
  for (long long k0 = static_cast<long long>(blockIdx.x) * kT; k0 < n; k0 += static_cast<long long>(gridDim.x) * kT) {
    const long long k = k0 + r;
    const bool live = k < n;
    // ---- row r, column part p: saved activations, u2, d2 (SIMT, K8a's expressions) ----
    const float4* A4 = nullptr;
    float u2[kOut] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (live) {
      const long long q = list[k];
      const float* A = act + q * kActStride;
      A4 = reinterpret_cast<const float4*>(A);
      const float4 lg = A4[(kIn + 2 * kHid) / 4];
      const float a[kOut] = {lg.x, lg.y, lg.z, lg.w};
      u2[0] = fmul(pgs[q], logistic_f(a[0]));
#pragma unroll
      for (int o = 1; o < kOut; ++o) {
        const float v = logistic_f(a[o]);
        u2[o] = fmul(fmul(pgc[3 * q + o - 1], v), __fsub_rn(1.0f, v));
      }
    }
    if (p == 0) {
#pragma unroll
      for (int o = 0; o < kOut; ++o) U2f[r * kOut + o] = u2[o];
    }
    {  // X columns [8p, 8p + 8) -> B_w rows 64 + i
      float x[8];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const float4 t = live ? A4[2 * p + v] : make_float4(0.f, 0.f, 0.f, 0.f);
        x[4 * v] = t.x, x[4 * v + 1] = t.y, x[4 * v + 2] = t.z, x[4 * v + 3] = t.w;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) put_split(bt_smem + kBW, kBWP, kmaj_off(kHid + 8 * p + j, r, kNW), x[j]);
    }
    {  // H1 columns [16p, 16p + 16) -> B_w rows i
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const float4 t = live ? A4[(kIn + 16 * p) / 4 + v] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float h[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) put_split(bt_smem + kBW, kBWP, kmaj_off(16 * p + 4 * v + j, r, kNW), h[j]);
      }
    }
    {  // H2 / d2 columns [16p, 16p + 16)
      float d2[16];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const float4 t = live ? A4[(kIn + kHid + 16 * p) / 4 + v] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float h[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = 16 * p + 4 * v + j;
          float d = 0.0f;
#pragma unroll
          for (int o = 0; o < kOut; ++o)
            if (u2[o] != 0.0f) d = fadd(d, fmul(u2[o], W2f[o * kHid + i]));
          d2[4 * v + j] = (h[j] == 0.0f) ? 0.0f : d;
          H2f[r * (kHid + 1) + i] = h[j];
          put_split(bt_smem + kAW, kAWP, kmaj_off(i, r, kT), d2[4 * v + j]);  // A_w rows 0-63: d2^T
        }
      }
      put_row8(bt_smem + kAD, kADP, kT, r, 16 * p, d2);  // A for dH1: row r
      put_row8(bt_smem + kAD, kADP, kT, r, 16 * p + 8, d2 + 8);
    }
    tc_fence_before();
    fence_async_smem();
    __syncthreads();
    // ---- dH1 = d2 . W1 ----
    if (tid == 0) {
      tc_fence_after();
      mma_split(tmem + kColDH1, sbase + kAD, kADP, kT, sbase + kWB1T, kW1P, kHid, kHid, idesc_bf16(kT, kHid));
      mma_commit(mbar);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    tc_fence_after();
    {  // d1 = ReLU'(H1) * dH1 on columns [16p, 16p + 16) (the mask from the exact H1)
      float v[16];
      tmem_ld16(trow + kColDH1 + 16 * p, v);
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const float4 t = live ? A4[(kIn + 16 * p) / 4 + q4] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float h[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = 4 * q4 + j;
          v[c] = (h[j] == 0.0f) ? 0.0f : v[c];
          put_split(bt_smem + kAW, kAWP, kmaj_off(kHid + 16 * p + c, r, kT), v[c]);  // A_w rows 64-127: d1^T
        }
      }
      tc_fence_before();
      __syncthreads();  // every part has read its dH1 columns before A_d is overwritten
      put_row8(bt_smem + kAD, kADP, kT, r, 16 * p, v);
      put_row8(bt_smem + kAD, kADP, kT, r, 16 * p + 8, v + 8);
    }
    tc_fence_before();
    fence_async_smem();
    __syncthreads();
    // ---- dX = d1 . W0 ; [dW1 | db1 ; dW0 | db0] += A_w . B_w ----
    if (tid == 0) {
      tc_fence_after();
      mma_split(tmem + kColDX, sbase + kAD, kADP, kT, sbase + kWB0T, kW0P, kIn, kHid, idesc_bf16(kT, kIn));
      mma_split(tmem + kColW, sbase + kAW, kAWP, kT, sbase + kBW, kBWP, kNW, kT, idesc_bf16(kT, kNW), any);
      mma_commit(mbar);
    }
    any = true;
    {  // dW2 / db2 (SIMT, fixed order over the tile's rows) while the MMAs run
      const int nq = static_cast<int>(n - k0 < kT ? n - k0 : kT);
      float sum = 0.0f;
      if (tid < kOut * kHid) {
        const int o = tid / kHid, i = tid % kHid;
        for (int j = 0; j < nq; ++j) sum = fadd(sum, fmul(U2f[j * kOut + o], H2f[j * (kHid + 1) + i]));
      } else if (tid < kOut * kHid + kOut) {
        for (int j = 0; j < nq; ++j) sum = fadd(sum, U2f[j * kOut + tid - kOut * kHid]);
      }
      acc2 = fadd(acc2, sum);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    tc_fence_after();
    if (p < 2) {  // dX columns [16p, 16p + 16) -> the record's d-feature slot (K8c)
      float v[16];
      tmem_ld16(trow + kColDX + 16 * p, v);
      if (live) {
        float4* R = reinterpret_cast<float4*>(rec + k * kRecStride + kRecDin + 16 * p);
#pragma unroll
        for (int j = 0; j < 4; ++j) R[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    }
    tc_fence_before();
    __syncthreads();  // smem operands and the dH1 / dX columns are reused by the next tile
  }
  // ---- this CTA's partial MLP-gradient row (parameter layout R/mlp.hpp:40-48) ----
  constexpr int pW0 = 0, pB0 = kHid * kIn, pW1 = pB0 + kHid, pB1 = pW1 + kHid * kHid, pW2 = pB1 + kHid,
                pB2 = pW2 + kOut * kHid;
  float* row = partial + static_cast<size_t>(blockIdx.x) * kNParams;
  tc_fence_after();
  if (any) {
    // TMEM rows 0-63: d2^T . [H1 | X | 1] -> dW1[o][i], db1[o]; rows 64-127: d1^T -> dW0, db0
    const int o = r & (kHid - 1);
    const bool top = r < kHid;
    for (int c = 16 * p; c < kNW; c += 64) {  // parts take 16-column chunks 0,4 | 1,5 | 2,6 | 3
      float v[16];
      tmem_ld16(trow + kColW + c, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int col = c + j;
        if (top && col < kHid) row[pW1 + o * kHid + col] = v[j];
        if (!top && col >= kHid && col < kHid + kIn) row[pW0 + o * kIn + (col - kHid)] = v[j];
        if (col == kColOnes) row[(top ? pB1 : pB0) + o] = v[j];
      }
    }
  } else {
    for (int e = tid; e < pW2; e += kThreads) row[e] = 0.0f;
  }
  if (tid < kOut * kHid + kOut) row[pW2 + tid] = acc2;  // pB2 == pW2 + 256
  static_assert(pB2 == pW2 + kOut * kHid, "dW2 then db2");
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
}

int sms() { return device_sm_count(); }

// roofline accounting (arfx_stats_*): stats[i] += *src (device count) + add
__global__ void stat_add_kernel(unsigned long long* stats, int i, const unsigned long long* src, unsigned long long add) {
  if (threadIdx.x == 0 && blockIdx.x == 0) stats[i] += (src ? *src : 0ull) + add;
}

}  // namespace

void stat_add(ModelImpl& m, int i, const unsigned long long* d_src, unsigned long long add, cudaStream_t s) {
  if (!m.stats_on) return;
  stat_add_kernel<<<1, 32, 0, s>>>(m.stats.ptr, i, d_src, add);
  ARFX_CUDA(cudaGetLastError());
}

void field_backward_pool(ModelImpl& m, const unsigned long long* d_n, long long cap, const uint8_t* flag,
                         const float* gs, const float* gc, cudaStream_t s, const BwdOwners* own, const float* act) {
  if (!(m.fv.F == 2 && m.fv.in_dim == kIn && m.fv.hidden == kHid && m.fv.n_layers == 3 && m.fv.out_dim == kOut))
    throw std::invalid_argument("train path: libarfx implements the 32-64-64-4 decoder (levels*F == 32)");
  Workspace& w = m.ws();
  const long long rec_cap = cap;
  w.bwd_rec.ensure(static_cast<size_t>(rec_cap + 1) * kRecStride);
  w.bwd_list.ensure(static_cast<size_t>(rec_cap + 1));
  w.bwd_n.ensure(1);
  ARFX_CUDA(cudaMemsetAsync(w.bwd_n.ptr, 0, sizeof(unsigned long long), s));
  m.wait_params(s);
  m.prof.begin("bwd_list", s);
  if (m.det && own) {
    w.bwd_own.ensure(static_cast<size_t>(std::max<long long>(own->n_owner, 1)));
    OwnerRanges O{own->n_owner, own->first, own->count, own->pool_is_target};
    const unsigned ob = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((own->n_owner + 7) / 8,
                                                                                         sms() * 16LL)));
    owner_list_kernel<false><<<ob, 256, 0, s>>>(O, w.snroot.ptr, w.sbase.ptr, flag, w.bwd_own.ptr, nullptr);
    owner_scan_kernel<<<1, 1024, 0, s>>>(w.bwd_own.ptr, own->n_owner, w.bwd_n.ptr);
    owner_list_kernel<true><<<ob, 256, 0, s>>>(O, w.snroot.ptr, w.sbase.ptr, flag, w.bwd_own.ptr, w.bwd_list.ptr);
  } else {
    flag_list_kernel<<<static_cast<unsigned>(std::max<long long>(1, std::min<long long>((cap + 255) / 256,
                                                                                         static_cast<long long>(sms()) * 8))),
                       256, 0, s>>>(flag, d_n, cap, w.bwd_list.ptr, w.bwd_n.ptr);
  }
  m.prof.end(s);
  stat_add(m, 7, w.bwd_n.ptr, 0, s);  // backward queries
  const size_t team_smem = (static_cast<size_t>(kHid) * kW0s + kHid * kW1s + kOut * kW1s + 2 * kHid + kOut +
                            static_cast<size_t>(kTeams) * kTQ * kTeamSmem) * sizeof(float);
  ensure_dyn_smem(reinterpret_cast<const void*>(field_bwd_team_kernel), team_smem);
  const int bwd_per_sm =  // persistent: exactly the resident blocks (one wave)
      blocks_per_sm(reinterpret_cast<const void*>(field_bwd_team_kernel), kTeamThreads, team_smem);
  // tcgen05 backward (K8-TC) when the forward saved its activations (decided on the device:
  // pool <= 64 Ki); otherwise the SIMT K8a / K8b below run
  const bool tc = m.bwd_tc && act != nullptr;
  const int tc_grid = sms();
  const int wblocks = sms() * 4;
  w.bwd_partial.ensure(static_cast<size_t>(std::max(wblocks, tc_grid)) * kNParams);
  m.prof.begin("bwd_field", s);
  field_bwd_team_kernel<<<static_cast<unsigned>(sms() * std::max(bwd_per_sm, 1)), kTeamThreads, team_smem, s>>>(
      m.fv, w.px.ptr, w.py.ptr, w.pz.ptr, w.bwd_list.ptr, w.bwd_n.ptr, gs, gc, m.grid_grad.ptr, w.bwd_rec.ptr, act,
      d_n, tc);
  ARFX_CUDA(cudaGetLastError());
  if (tc) {
    ensure_dyn_smem(reinterpret_cast<const void*>(field_bwd_tc_kernel), bwdtc::kSmem + 1024);
    field_bwd_tc_kernel<<<static_cast<unsigned>(tc_grid), bwdtc::kThreads, bwdtc::kSmem + 1024, s>>>(
        m.fv, w.bwd_list.ptr, w.bwd_n.ptr, gs, gc, act, d_n, w.bwd_rec.ptr, w.bwd_partial.ptr);
    ARFX_CUDA(cudaGetLastError());
  }
  m.prof.end(s);
  // K8b + K8d (MLP weights, smem/FP32) run on the aux stream beside K8c (hash-grid
  // scatter, L2 atomics); both only read the K8a records. The join keeps the next
  // gradient writer on `s` ordered after K8d's non-atomic mlp_grad update.
  if (!m.aux) {
    ARFX_CUDA(cudaStreamCreateWithFlags(&m.aux, cudaStreamNonBlocking));
    ARFX_CUDA(cudaEventCreateWithFlags(&m.ev_aux_fork, cudaEventDisableTiming));
    ARFX_CUDA(cudaEventCreateWithFlags(&m.ev_aux_join, cudaEventDisableTiming));
  }
  ARFX_CUDA(cudaEventRecord(m.ev_aux_fork, s));
  ARFX_CUDA(cudaStreamWaitEvent(m.aux, m.ev_aux_fork, 0));
  m.prof.begin("bwd_weights", m.aux);
  field_bwd_weights_kernel<<<static_cast<unsigned>(wblocks), kWThreads, 0, m.aux>>>(
      w.bwd_rec.ptr, w.bwd_n.ptr, rec_cap, w.bwd_partial.ptr, tc ? d_n : nullptr);
  weights_reduce_kernel<<<(kNParams + 31) / 32, 256, 0, m.aux>>>(w.bwd_partial.ptr, wblocks, w.bwd_n.ptr, rec_cap,
                                                                 m.mlp_grad.ptr, tc ? d_n : nullptr, tc_grid);
  ARFX_CUDA(cudaGetLastError());
  m.prof.end(m.aux);
  ARFX_CUDA(cudaEventRecord(m.ev_aux_join, m.aux));
  m.prof.begin("bwd_scatter", s);
  if (m.det) {
    const size_t n_acc = static_cast<size_t>(m.fv.L) * m.fv.T * 2;  // == n_grid
    if (m.grid_acc.n < n_acc) {  // zeroed once; consumers leave it all-zero
      m.grid_acc.alloc(n_acc);
      ARFX_CUDA(cudaMemsetAsync(m.grid_acc.ptr, 0, n_acc * sizeof(long long), s));
    }
    grid_scatter_kernel<true><<<resident_grid(grid_scatter_kernel<true>, 256, 0, 1LL << 40), 256, 0, s>>>(
        m.fv, w.px.ptr, w.py.ptr, w.pz.ptr, w.bwd_list.ptr, w.bwd_n.ptr, w.bwd_rec.ptr, m.grid_grad.ptr,
        m.grid_acc.ptr);
    m.acc_pending = true;
  } else {
    grid_scatter_kernel<false><<<resident_grid(grid_scatter_kernel<false>, 256, 0, 1LL << 40), 256, 0, s>>>(
        m.fv, w.px.ptr, w.py.ptr, w.pz.ptr, w.bwd_list.ptr, w.bwd_n.ptr, w.bwd_rec.ptr, m.grid_grad.ptr, nullptr);
  }
  m.prof.end(s);
  ARFX_CUDA(cudaStreamWaitEvent(s, m.ev_aux_join, 0));
  ARFX_CUDA(cudaGetLastError());
}

void flush_grad_acc(ModelImpl& m, cudaStream_t s) {
  if (!m.acc_pending) return;
  m.wait_params(s);
  const long long n2 = static_cast<long long>(m.grid_acc.n / 2);
  grid_flush_kernel<<<static_cast<unsigned>(std::min<long long>((n2 + 255) / 256, sms() * 16LL)), 256, 0, s>>>(
      n2, reinterpret_cast<longlong2*>(m.grid_acc.ptr), reinterpret_cast<float2*>(m.grid_grad.ptr));
  ARFX_CUDA(cudaGetLastError());
  m.acc_pending = false;
}

void train_composite(ModelImpl& m, long long n_rays, int N, double eps, const float* d_dC, const float* d_dA,
                     float* d_rgb, float* d_alpha, cudaStream_t s, const LossTargets* lt) {
  Workspace& w = m.ws();
  TrainCompositeArgs A{n_rays, N, eps, w.ray_first.ptr, w.ray_count.ptr, w.sidx.ptr, w.sdelta.ptr, w.snroot.ptr,
                       w.sbase.ptr, w.pres.ptr, w.strans.ptr, d_dC, d_dA, nullptr, nullptr, nullptr, nullptr, 0, 0,
                       LossCfg{}, 0.0, nullptr,
                       d_rgb, d_alpha, w.pgs.ptr, w.pgc.ptr, w.pflag.ptr};
  if (lt) {
    A.gt_rgb = lt->gt_rgb;
    A.gt_alpha = lt->gt_alpha;
    A.gpx = lt->px;
    A.gpy = lt->py;
    A.gt_w = lt->gt_w;
    A.gt_h = lt->gt_h;
    A.loss = LossCfg{lt->w_rgb, lt->w_alpha, lt->w_hard, lt->w_density, lt->huber_delta};
    A.inv_n = 1.0 / static_cast<double>(n_rays);
    A.ray_terms = lt->ray_terms;
  }
  m.prof.begin("train_composite", s);
  train_composite_warp_kernel<<<static_cast<unsigned>(std::max<long long>(1, (n_rays + 3) / 4)), 128, 0, s>>>(A);
  ARFX_CUDA(cudaGetLastError());
  m.prof.end(s);
  stat_add(m, 8, w.counters.ptr, 0, s);                                   // composited posed samples
  stat_add(m, 9, nullptr, static_cast<unsigned long long>(n_rays), s);   // rays
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
