// field.cuh -- canonical field on sm_100a: multiresolution hash encoding + decoder MLP.
//
// Restates (exact f32 path, same operand order as the reference's -O3
// -ffp-contract=off x86 build):
//   HashGrid::hash_index  R/hash_grid.hpp:87-101 (direct / wrap / XOR-hash levels)
//   HashGrid::gather      R/hash_grid.hpp:114-134 (f64 cell + weights, cast to f32)
//   HashGrid::encode      R/hash_grid.hpp:137-150 (o += w*row in corner order)
//   DecoderMlp::forward   R/mlp.hpp:90-111 (acc = b; acc += W[o][i]*in[i]; ReLU)
//   CanonicalField::query R/field.hpp:75-82 (softplus / logistic, R/math.hpp:264-271)
#pragma once

#include "arfx_internal.h"
#include "exact.cuh"

#ifndef ARFX_PAIR_GATHER
#define ARFX_PAIR_GATHER 1
#endif

namespace arfx {

constexpr int kMlpGenericMaxWidth = 256;

__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }

__device__ __forceinline__ uint32_t hash_index(const FieldView& F, int level, int cx, int cy, int cz) {
  const uint64_t n = static_cast<uint64_t>(F.res[level]);
  const int kind = F.kind[level];
  if (kind == kDirect) {
    const uint64_t corners = n + 1;
    return static_cast<uint32_t>(static_cast<uint64_t>(cx) +
                                 corners * (static_cast<uint64_t>(cy) + corners * static_cast<uint64_t>(cz)));
  }
  if (kind == kWrap) {
    const uint64_t wx = static_cast<uint64_t>(cx) % n, wy = static_cast<uint64_t>(cy) % n,
                   wz = static_cast<uint64_t>(cz) % n;
    return static_cast<uint32_t>(wx + n * (wy + n * wz));
  }
  const uint32_t h = static_cast<uint32_t>(cx) ^ (static_cast<uint32_t>(cy) * 2654435761u) ^
                     (static_cast<uint32_t>(cz) * 805459861u);
  return h & (F.T - 1u);
}

// Aabb::contains (inclusive)  R/math.hpp:226-228
__device__ __forceinline__ bool field_contains(const FieldView& F, d3 p) {
  return p.x >= F.lo[0] && p.x <= F.hi[0] && p.y >= F.lo[1] && p.y <= F.hi[1] && p.z >= F.lo[2] &&
         p.z <= F.hi[2];
}

// Per-level cell corners and trilinear weights (f64, cast to f32).
struct LevelCorners {
  uint32_t idx[8];
  float w[8];
};

__device__ __forceinline__ void level_corners(const FieldView& F, int l, const double u[3],
                                              LevelCorners& lc) {
  const double n = static_cast<double>(F.res[l]);
  int cell[3];
  double f[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double p = dmul(u[a], n);
    double c = floor(p);
    if (c > dsub(n, 1.0)) c = dsub(n, 1.0);
    if (c < 0) c = 0;
    cell[a] = static_cast<int>(c);
    f[a] = dsub(p, c);
  }
  // corner indices (R/hash_grid.hpp:87-101) from per-axis terms in 32-bit arithmetic: the
  // direct and wrap branches only exist when (n+1)^3 resp. n^3 <= 2^T <= 2^30, so the
  // reference's 64-bit products equal the 32-bit ones, and the corner coordinate c + d is in
  // [0, n], so its wrap (c + d) % n is (c + d == n ? 0 : c + d) -- no 64-bit multiplies or
  // modulos (which dominated this function's instruction count and i-cache footprint)
  const uint32_t nu = static_cast<uint32_t>(F.res[l]);
  const int kind = F.kind[l];
  uint32_t tx[2], ty[2], tz[2];
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    const uint32_t cx = static_cast<uint32_t>(cell[0] + d), cy = static_cast<uint32_t>(cell[1] + d),
                   cz = static_cast<uint32_t>(cell[2] + d);
    if (kind == kDirect) {
      const uint32_t c1 = nu + 1u;
      tx[d] = cx;
      ty[d] = c1 * cy;
      tz[d] = c1 * c1 * cz;
    } else if (kind == kWrap) {
      tx[d] = cx == nu ? 0u : cx;
      ty[d] = nu * (cy == nu ? 0u : cy);
      tz[d] = nu * nu * (cz == nu ? 0u : cz);
    } else {
      tx[d] = cx;
      ty[d] = cy * 2654435761u;
      tz[d] = cz * 805459861u;
    }
  }
  const bool hashed = kind != kDirect && kind != kWrap;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
    lc.idx[k] = hashed ? ((tx[dx] ^ ty[dy] ^ tz[dz]) & (F.T - 1u)) : (tx[dx] + ty[dy] + tz[dz]);
    lc.w[k] = static_cast<float>(dmul(dmul(dx ? f[0] : dsub(1.0, f[0]), dy ? f[1] : dsub(1.0, f[1])),
                                      dz ? f[2] : dsub(1.0, f[2])));
  }
}

// normalize_point (caller guarantees in-box)  R/hash_grid.hpp:176-181
__device__ __forceinline__ void normalize_point(const FieldView& F, d3 x, double u[3]) {
  u[0] = ddiv(dsub(x.x, F.lo[0]), F.e[0]);
  u[1] = ddiv(dsub(x.y, F.lo[1]), F.e[1]);
  u[2] = ddiv(dsub(x.z, F.lo[2]), F.e[2]);
}

// HashGrid::encode for F == 2 (float2 rows): feats[2L]
__device__ __forceinline__ void hash_encode_f2(const FieldView& F, d3 x, float* feats) {
  double u[3];
  normalize_point(F, x, u);
  const float2* table = reinterpret_cast<const float2*>(F.grid);
  for (int l = 0; l < F.L; ++l) {
    LevelCorners lc;
    level_corners(F, l, u, lc);
    const float2* t = table + static_cast<size_t>(l) * F.T;
    float2 row[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) row[k] = __ldg(t + lc.idx[k]);
    float o0 = 0.0f, o1 = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      o0 = fadd(o0, fmul(lc.w[k], row[k].x));
      o1 = fadd(o1, fmul(lc.w[k], row[k].y));
    }
    feats[2 * l] = o0;
    feats[2 * l + 1] = o1;
  }
}

// Generic F
__device__ __forceinline__ void hash_encode_generic(const FieldView& F, d3 x, float* feats) {
  double u[3];
  normalize_point(F, x, u);
  for (int l = 0; l < F.L; ++l) {
    LevelCorners lc;
    level_corners(F, l, u, lc);
    const float* t = F.grid + static_cast<size_t>(l) * F.T * F.F;
    float* o = feats + l * F.F;
    for (int f = 0; f < F.F; ++f) o[f] = 0.0f;
    for (int k = 0; k < 8; ++k) {
      const float* row = t + static_cast<size_t>(lc.idx[k]) * F.F;
      for (int f = 0; f < F.F; ++f) o[f] = fadd(o[f], fmul(lc.w[k], __ldg(row + f)));
    }
  }
}

// R/math.hpp:264-271 in f32 (Real = float)
__device__ __forceinline__ float softplus_f(float z) {
  return z > 0 ? fadd(z, log1pf(expf(-z))) : log1pf(expf(z));
}
__device__ __forceinline__ float logistic_f(float z) {
  return z >= 0 ? __fdiv_rn(1.0f, fadd(1.0f, expf(-z))) : __fdiv_rn(expf(z), fadd(1.0f, expf(z)));
}

// Specialised exact MLP: IN -> HID (x NH hidden layers, ReLU) -> OUT, weights in smem
// (same flat layout as the reference). Intermediate activations live in registers;
// the last hidden layer's outputs are streamed straight into the output accumulators
// in the reference's summation order (out[q] = b[q] + sum_o W[q][o] h[o], o ascending).
template <int IN, int HID, int NH, int OUT>
__device__ __forceinline__ void mlp_forward_exact(const float* __restrict__ W, const float* in,
                                                  float* logits) {
  float a[HID], b[HID];
  // layer 0
  {
    const float* w = W;
    const float* bias = W + IN * HID;
#pragma unroll
    for (int o = 0; o < HID; ++o) {
      float acc = bias[o];
      const float4* wr = reinterpret_cast<const float4*>(w + o * IN);
#pragma unroll
      for (int i = 0; i < IN / 4; ++i) {
        const float4 q = wr[i];
        acc = fadd(acc, fmul(q.x, in[4 * i + 0]));
        acc = fadd(acc, fmul(q.y, in[4 * i + 1]));
        acc = fadd(acc, fmul(q.z, in[4 * i + 2]));
        acc = fadd(acc, fmul(q.w, in[4 * i + 3]));
      }
      a[o] = (acc < 0.0f) ? 0.0f : acc;
    }
  }
  int off = IN * HID + HID;
  // middle hidden layers 1..NH-2 (full arrays)
#pragma unroll
  for (int l = 1; l < NH - 1; ++l) {
    const float* w = W + off;
    const float* bias = w + HID * HID;
#pragma unroll
    for (int o = 0; o < HID; ++o) {
      float acc = bias[o];
      const float4* wr = reinterpret_cast<const float4*>(w + o * HID);
#pragma unroll
      for (int i = 0; i < HID / 4; ++i) {
        const float4 q = wr[i];
        acc = fadd(acc, fmul(q.x, a[4 * i + 0]));
        acc = fadd(acc, fmul(q.y, a[4 * i + 1]));
        acc = fadd(acc, fmul(q.z, a[4 * i + 2]));
        acc = fadd(acc, fmul(q.w, a[4 * i + 3]));
      }
      b[o] = (acc < 0.0f) ? 0.0f : acc;
    }
#pragma unroll
    for (int o = 0; o < HID; ++o) a[o] = b[o];
    off += HID * HID + HID;
  }
  // last hidden layer streamed into the output layer
  const float* w = W + off;
  const float* bias = w + HID * HID;
  const float* wo = bias + HID;
  const float* bo = wo + OUT * HID;
  float out[OUT];
#pragma unroll
  for (int q = 0; q < OUT; ++q) out[q] = bo[q];
#pragma unroll
  for (int o = 0; o < HID; ++o) {
    float acc = bias[o];
    const float4* wr = reinterpret_cast<const float4*>(w + o * HID);
#pragma unroll
    for (int i = 0; i < HID / 4; ++i) {
      const float4 q = wr[i];
      acc = fadd(acc, fmul(q.x, a[4 * i + 0]));
      acc = fadd(acc, fmul(q.y, a[4 * i + 1]));
      acc = fadd(acc, fmul(q.z, a[4 * i + 2]));
      acc = fadd(acc, fmul(q.w, a[4 * i + 3]));
    }
    const float h = (acc < 0.0f) ? 0.0f : acc;
#pragma unroll
    for (int q = 0; q < OUT; ++q) out[q] = fadd(out[q], fmul(wo[q * HID + o], h));
  }
#pragma unroll
  for (int q = 0; q < OUT; ++q) logits[q] = out[q];
}

// Generic exact MLP (any layout up to kMlpGenericMaxWidth wide), local-memory activations.
__device__ __forceinline__ void mlp_forward_generic(const FieldView& F, const float* __restrict__ W,
                                                    const float* in, float* logits) {
  float bufA[kMlpGenericMaxWidth], bufB[kMlpGenericMaxWidth];
  for (int i = 0; i < F.in_dim; ++i) bufA[i] = in[i];
  float* cur = bufA;
  float* nxt = bufB;
  for (int l = 0; l < F.n_layers; ++l) {
    const int nin = F.lin[l], non = F.lout[l];
    const float* w = W + F.w_off[l];
    const float* bias = W + F.b_off[l];
    const bool hidden = l + 1 < F.n_layers;
    for (int o = 0; o < non; ++o) {
      float acc = bias[o];
      for (int i = 0; i < nin; ++i) acc = fadd(acc, fmul(w[o * nin + i], cur[i]));
      nxt[o] = (hidden && acc < 0.0f) ? 0.0f : acc;
    }
    float* t = cur;
    cur = nxt;
    nxt = t;
  }
  for (int q = 0; q < F.out_dim; ++q) logits[q] = cur[q];
}

// One level of HashGrid::encode for F == 2 from precomputed normalized coords u (f64).
__device__ __forceinline__ float2 encode_level_f2(const FieldView& F, int l, const double u[3]) {
  LevelCorners lc;
  level_corners(F, l, u, lc);
  const float2* t = reinterpret_cast<const float2*>(F.grid) + static_cast<size_t>(l) * F.T;
  float2 row[8];
#if ARFX_PAIR_GATHER
  // x-neighbour corners (k, k+1) often share one 16-B aligned row pair: always for hashed
  // levels with an even x (idx ^ 1), for direct/wrap levels when idx is even. One 16-B load of
  // the aligned pair holding corner k, plus an 8-B load of corner k+1 only where it lies
  // outside that pair: fewer L1 wavefronts for the same rows (the table base is 256-B aligned)
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const uint32_t a = lc.idx[k], b = lc.idx[k + 1];
    const float4 c = __ldg(reinterpret_cast<const float4*>(t + (a & ~1u)));
    const float2 e0 = make_float2(c.x, c.y), e1 = make_float2(c.z, c.w);
    row[k] = (a & 1u) ? e1 : e0;
    row[k + 1] = ((a ^ b) <= 1u) ? ((b & 1u) ? e1 : e0) : __ldg(t + b);
  }
#else
#pragma unroll
  for (int k = 0; k < 8; ++k) row[k] = __ldg(t + lc.idx[k]);
#endif
  float o0 = 0.0f, o1 = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    o0 = fadd(o0, fmul(lc.w[k], row[k].x));
    o1 = fadd(o1, fmul(lc.w[k], row[k].y));
  }
  return make_float2(o0, o1);
}

// Exact MLP, feature-major first layer: acc[o] accumulates in input order i = 0..IN-1
// exactly as DecoderMlp::forward (R/mlp.hpp:100-104), reading inputs one at a time from
// shared memory and W0 transposed (W0T[i][o]) so 4 consecutive outputs share an LDS.128.
// Wr points at the flat params after W0 (b0, W1, b1, ..., W_out, b_out).
template <int IN, int HID, int NH, int OUT>
__device__ __forceinline__ void mlp_forward_fm(const float* __restrict__ W0T, const float* __restrict__ Wr,
                                               const float* in, float* logits) {
  float a[HID];
  {
    const float* b0 = Wr;
#pragma unroll
    for (int o = 0; o < HID; ++o) a[o] = b0[o];
#pragma unroll 4
    for (int i = 0; i < IN; ++i) {
      const float x = in[i];
      const float4* w4 = reinterpret_cast<const float4*>(W0T + i * HID);
#pragma unroll
      for (int o4 = 0; o4 < HID / 4; ++o4) {
        const float4 q = w4[o4];
        a[4 * o4 + 0] = fadd(a[4 * o4 + 0], fmul(q.x, x));
        a[4 * o4 + 1] = fadd(a[4 * o4 + 1], fmul(q.y, x));
        a[4 * o4 + 2] = fadd(a[4 * o4 + 2], fmul(q.z, x));
        a[4 * o4 + 3] = fadd(a[4 * o4 + 3], fmul(q.w, x));
      }
    }
#pragma unroll
    for (int o = 0; o < HID; ++o) a[o] = (a[o] < 0.0f) ? 0.0f : a[o];
  }
  const float* p = Wr + HID;
#pragma unroll
  for (int l = 1; l < NH - 1; ++l) {  // middle hidden layers (none for NH == 2)
    float b[HID];
    const float* bias = p + HID * HID;
#pragma unroll
    for (int o = 0; o < HID; ++o) {
      float acc = bias[o];
      const float4* wr = reinterpret_cast<const float4*>(p + o * HID);
#pragma unroll
      for (int i = 0; i < HID / 4; ++i) {
        const float4 q = wr[i];
        acc = fadd(acc, fmul(q.x, a[4 * i + 0]));
        acc = fadd(acc, fmul(q.y, a[4 * i + 1]));
        acc = fadd(acc, fmul(q.z, a[4 * i + 2]));
        acc = fadd(acc, fmul(q.w, a[4 * i + 3]));
      }
      b[o] = (acc < 0.0f) ? 0.0f : acc;
    }
#pragma unroll
    for (int o = 0; o < HID; ++o) a[o] = b[o];
    p += HID * HID + HID;
  }
  const float* bias = p + HID * HID;
  const float* wo = bias + HID;
  const float* bo = wo + OUT * HID;
  float out[OUT];
#pragma unroll
  for (int q = 0; q < OUT; ++q) out[q] = bo[q];
#pragma unroll 2
  for (int o = 0; o < HID; ++o) {
    float acc = bias[o];
    const float4* wr = reinterpret_cast<const float4*>(p + o * HID);
#pragma unroll
    for (int i = 0; i < HID / 4; ++i) {
      const float4 q = wr[i];
      acc = fadd(acc, fmul(q.x, a[4 * i + 0]));
      acc = fadd(acc, fmul(q.y, a[4 * i + 1]));
      acc = fadd(acc, fmul(q.z, a[4 * i + 2]));
      acc = fadd(acc, fmul(q.w, a[4 * i + 3]));
    }
    const float h = (acc < 0.0f) ? 0.0f : acc;
#pragma unroll
    for (int q = 0; q < OUT; ++q) out[q] = fadd(out[q], fmul(wo[q * HID + o], h));
  }
#pragma unroll
  for (int q = 0; q < OUT; ++q) logits[q] = out[q];
}

__device__ __forceinline__ bool field_is_standard(const FieldView& F) {
  return F.F == 2 && F.L == 16 && F.in_dim == 32 && F.hidden == 64 && F.n_layers == 3 &&
         F.out_dim == 4;
}

// CanonicalField::query for one in-box point; W = MLP params (smem or global).
// Returns (density, r, g, b).
__device__ __forceinline__ float4 field_query_exact(const FieldView& F, const float* __restrict__ W,
                                                    d3 x) {
  float logits[kMlpGenericMaxWidth > 4 ? 4 : 4];
  if (field_is_standard(F)) {
    float feats[32];
    hash_encode_f2(F, x, feats);
    mlp_forward_exact<32, 64, 2, 4>(W, feats, logits);
  } else {
    float feats[kMaxLevels * 8];
    if (F.F == 2) hash_encode_f2(F, x, feats);
    else hash_encode_generic(F, x, feats);
    float lg[kMlpGenericMaxWidth];
    mlp_forward_generic(F, W, feats, lg);
    for (int q = 0; q < 4; ++q) logits[q] = q < F.out_dim ? lg[q] : 0.0f;
  }
  return make_float4(softplus_f(logits[0]), logistic_f(logits[1]), logistic_f(logits[2]),
                     logistic_f(logits[3]));
}

}  // namespace arfx
