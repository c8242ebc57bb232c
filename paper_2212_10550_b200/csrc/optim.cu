// optim.cu -- Adam over the flat [grid | mlp] parameter vector, with the zero-grad fused
// (adaptive moments, lr 1e-2 grid / 1e-3 MLP, cosine decay; beta1 0.9,
// beta2 0.99, eps 1e-15 follow the cited encoding system's practice -- the paper names no
// optimizer). One pass, HBM-bound: reads p, g, m, v and writes p, m, v, g = 0 (32 B per
// parameter), float4-vectorised. f32 arithmetic, no FMA (--fmad=false), fixed op order:
//   m = b1 m + (1 - b1) g;  v = b2 v + (1 - b2) g g
//   p = p - lr_t * (m c1) / (sqrt(v c2) + eps),   c1 = 1/(1 - b1^t), c2 = 1/(1 - b2^t)
// so oracle/arf_oracle.c arfo_adam reproduces it bit for bit. [begin, end) selects a shard
// of the flat vector (data-parallel training: reduce-scatter -> sharded Adam -> all-gather).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "fixed.cuh"
#include "model.h"

namespace arfx {
namespace {

struct AdamScalars {
  float b1, omb1, b2, omb2, c1, c2, eps, lr_grid, lr_mlp;
  long long mlp_off;
};

__device__ __forceinline__ void adam1(float& p, float& g, float& m, float& v, float lr, const AdamScalars& k) {
  const float gg = g;
  m = __fadd_rn(__fmul_rn(k.b1, m), __fmul_rn(k.omb1, gg));
  v = __fadd_rn(__fmul_rn(k.b2, v), __fmul_rn(k.omb2, __fmul_rn(gg, gg)));
  const float den = __fadd_rn(__fsqrt_rn(__fmul_rn(v, k.c2)), k.eps);
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(lr, __fmul_rn(m, k.c1)), den));
  g = 0.0f;
}

// acc (deterministic mode, pending hash-grid sums): the first n4_acc float4s of the
// gradient also take acc's fixed-point sums, which are cleared -- the same f32 expression
// as flush_grad_acc (train.cu), so folding here or flushing first gives equal bits.
// guard (optional): the step's loss row; if any entry is non-finite, or *bad is already set
// by an earlier step, the whole step is skipped (parameters, moments and gradients untouched)
// and *bad is set -- the trainer raises NumericError when it next reads the flag, with the
// model still at its last finite state (SPEC.md:494 abort on a non-finite loss).
template <bool Acc>
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ p, float* __restrict__ g,
                                                   float* __restrict__ m, float* __restrict__ v, long long b4,
                                                   long long e4, AdamScalars k, longlong2* __restrict__ acc,
                                                   long long n4_acc, const double* __restrict__ guard,
                                                   int n_guard, int* bad) {
  if (guard) {
    bool nonfinite = false;
    for (int j = 0; j < n_guard; ++j) nonfinite |= !isfinite(guard[j]);
    if (nonfinite && blockIdx.x == 0 && threadIdx.x == 0) atomicExch(bad, 1);
    if (nonfinite || *reinterpret_cast<volatile int*>(bad)) return;
  }
  for (long long i = b4 + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < e4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 P = reinterpret_cast<float4*>(p)[i], G = reinterpret_cast<float4*>(g)[i];
    if (Acc && i < n4_acc) {
      const longlong2 a = acc[2 * i], b = acc[2 * i + 1];
      if ((a.x | a.y | b.x | b.y) != 0) {
        if (a.x) G.x = __fadd_rn(G.x, fix_to_f32(a.x));
        if (a.y) G.y = __fadd_rn(G.y, fix_to_f32(a.y));
        if (b.x) G.z = __fadd_rn(G.z, fix_to_f32(b.x));
        if (b.y) G.w = __fadd_rn(G.w, fix_to_f32(b.y));
        acc[2 * i] = make_longlong2(0, 0);
        acc[2 * i + 1] = make_longlong2(0, 0);
      }
    }
    float4 M = reinterpret_cast<float4*>(m)[i], V = reinterpret_cast<float4*>(v)[i];
    const float lr = (4 * i >= k.mlp_off) ? k.lr_mlp : k.lr_grid;  // mlp_off % 64 == 0
    adam1(P.x, G.x, M.x, V.x, lr, k);
    adam1(P.y, G.y, M.y, V.y, lr, k);
    adam1(P.z, G.z, M.z, V.z, lr, k);
    adam1(P.w, G.w, M.w, V.w, lr, k);
    reinterpret_cast<float4*>(p)[i] = P;
    reinterpret_cast<float4*>(g)[i] = G;
    reinterpret_cast<float4*>(m)[i] = M;
    reinterpret_cast<float4*>(v)[i] = V;
  }
}

}  // namespace

// lr_t = lr0 (f + (1 - f) (1 + cos(pi min(t, T) / T)) / 2), t = step (1-based); T <= 0: constant
double cosine_lr(double lr0, const AdamCfg& c, long long step) {
  if (c.total_steps <= 0) return lr0;
  const double t = static_cast<double>(std::min(step, c.total_steps)) / static_cast<double>(c.total_steps);
  const double f = c.final_lr_factor;
  return lr0 * (f + (1.0 - f) * 0.5 * (1.0 + std::cos(3.14159265358979323846 * t)));
}

void adam_step(ModelImpl& m, const AdamCfg& c, long long step, long long begin, long long end, cudaStream_t s,
               const double* guard, int n_guard, int* bad) {
  const size_t n = m.n_flat;
  if (!m.adam_m.ptr) {
    m.adam_m.alloc(n);
    m.adam_v.alloc(n);
    ARFX_CUDA(cudaMemsetAsync(m.adam_m.ptr, 0, n * sizeof(float), s));
    ARFX_CUDA(cudaMemsetAsync(m.adam_v.ptr, 0, n * sizeof(float), s));
  }
  AdamScalars k;
  k.b1 = static_cast<float>(c.beta1);
  k.omb1 = static_cast<float>(1.0 - c.beta1);
  k.b2 = static_cast<float>(c.beta2);
  k.omb2 = static_cast<float>(1.0 - c.beta2);
  k.c1 = static_cast<float>(1.0 / (1.0 - std::pow(c.beta1, static_cast<double>(step))));
  k.c2 = static_cast<float>(1.0 / (1.0 - std::pow(c.beta2, static_cast<double>(step))));
  k.eps = static_cast<float>(c.eps);
  k.lr_grid = static_cast<float>(cosine_lr(c.lr_grid, c, step));
  k.lr_mlp = static_cast<float>(cosine_lr(c.lr_mlp, c, step));
  k.mlp_off = static_cast<long long>(m.mlp_off);
  const long long b4 = begin / 4, e4 = end / 4;
  if (e4 <= b4) return;
  const long long blocks = resident_grid(adam_kernel<false>, 256, 0, e4 - b4);  // one wave
  m.prof.begin("adam", s);
  if (m.acc_pending && !(begin == 0 && end >= static_cast<long long>(m.grid_acc.n)))
    flush_grad_acc(m, s);  // a shard cannot consume the whole accumulator
  if (m.acc_pending) {
    adam_kernel<true><<<static_cast<unsigned>(blocks), 256, 0, s>>>(
        m.flat_params.ptr, m.flat_grads.ptr, m.adam_m.ptr, m.adam_v.ptr, b4, e4, k,
        reinterpret_cast<longlong2*>(m.grid_acc.ptr), static_cast<long long>(m.grid_acc.n / 4), guard, n_guard,
        bad);
    m.acc_pending = false;
  } else {
    adam_kernel<false><<<static_cast<unsigned>(blocks), 256, 0, s>>>(m.flat_params.ptr, m.flat_grads.ptr, m.adam_m.ptr,
                                                                     m.adam_v.ptr, b4, e4, k, nullptr, 0, guard,
                                                                     n_guard, bad);
  }
  ARFX_CUDA(cudaGetLastError());
  m.prof.end(s);
  stat_add(m, 10, nullptr, static_cast<unsigned long long>(end - begin), s);  // parameters updated
}

}  // namespace arfx
