// model.cu -- one-time model construction on the device (build_model, R/model.hpp:68-80).
//
//  * parameter init: HashGrid draws all L*2^T*F params from ONE PCG32 stream
//    (R/hash_grid.hpp:66-73) and DecoderMlp its weights from another
//    (R/mlp.hpp:50-58). Each thread jumps the LCG to its chunk's first draw
//    (pcg_advance, O(log n)) and then steps sequentially, so the 16.7 M-param table
//    of config 1 is initialised in parallel yet bit-identical to the serial stream.
//  * skinning grid: nearest-capsule-axis weights with the 1.5x inverse-distance
//    blend band (R/skinning.hpp:61-111), one thread per lattice node, FP64 exact.
//  * per-cell packed table for the deformer (see SkinView in arfx_internal.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <numeric>

#include "exact.cuh"
#include "model.h"

namespace arfx {

namespace {

__global__ void init_uniform_kernel(float* __restrict__ out, int64_t n, Pcg32 base,
                                    int64_t first_draw, double lo, double hi, int chunk) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t start = t * chunk;
  if (start >= n) return;
  Pcg32 r = base;
  pcg_advance(r, static_cast<uint64_t>(first_draw + start));
  const double span = dsub(hi, lo);
  const int64_t end = start + chunk < n ? start + chunk : n;
  for (int64_t i = start; i < end; ++i) {
    const double u = pcg_double(r);
    out[i] = static_cast<float>(dadd(lo, dmul(span, u)));  // Pcg32::uniform R/rng.hpp:57
  }
}

struct SkelDev {
  int nb;
  double head[kMaxBones][3];
  double tail[kMaxBones][3];
};

__global__ void skinning_grid_kernel(double* __restrict__ w, int rx, int ry, int rz, d3 lo, d3 e,
                                     SkelDev sk, double blend) {
  const int64_t node = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nn = static_cast<int64_t>(rx) * ry * rz;
  if (node >= nn) return;
  const int ix = static_cast<int>(node % rx);
  const int iy = static_cast<int>((node / rx) % ry);
  const int iz = static_cast<int>(node / (static_cast<int64_t>(rx) * ry));
  // p = lo + e * i / (res - 1)   R/skinning.hpp:83-85
  const d3 p = make3(dadd(lo.x, ddiv(dmul(e.x, static_cast<double>(ix)), static_cast<double>(rx - 1))),
                     dadd(lo.y, ddiv(dmul(e.y, static_cast<double>(iy)), static_cast<double>(ry - 1))),
                     dadd(lo.z, ddiv(dmul(e.z, static_cast<double>(iz)), static_cast<double>(rz - 1))));
  double dist[kMaxBones];
  double dmin = 1.7976931348623157e308;
  for (int b = 0; b < sk.nb; ++b) {
    dist[b] = point_segment_distance(p, make3(sk.head[b][0], sk.head[b][1], sk.head[b][2]),
                                     make3(sk.tail[b][0], sk.tail[b][1], sk.tail[b][2]));
    dmin = (dist[b] < dmin) ? dist[b] : dmin;
  }
  double* out = w + node * sk.nb;
  if (dmin < 1e-12) {
    int hits = 0;
    for (int b = 0; b < sk.nb; ++b)
      if (dist[b] < 1e-12) ++hits;
    for (int b = 0; b < sk.nb; ++b) out[b] = dist[b] < 1e-12 ? ddiv(1.0, static_cast<double>(hits)) : 0.0;
    return;
  }
  const double band = dmul(blend, dmin);
  double sum = 0.0;
  for (int b = 0; b < sk.nb; ++b) {
    const double v = dist[b] <= band ? ddiv(1.0, dist[b]) : 0.0;
    out[b] = v;
    sum = dadd(sum, v);
  }
  for (int b = 0; b < sk.nb; ++b) out[b] = ddiv(out[b], sum);
}

__device__ __forceinline__ const double* node_ptr(const double* w, int rx, int ry, int nb, int x,
                                                  int y, int z) {
  return w + ((static_cast<size_t>(z) * ry + y) * rx + x) * nb;
}

__global__ void cell_mask_kernel(const double* __restrict__ w, int rx, int ry, int rz, int nb,
                                 uint32_t* __restrict__ mask, uint32_t* __restrict__ count) {
  const int cx_n = rx - 1, cy_n = ry - 1, cz_n = rz - 1;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= static_cast<int64_t>(cx_n) * cy_n * cz_n) return;
  const int x = static_cast<int>(c % cx_n), y = static_cast<int>((c / cx_n) % cy_n),
            z = static_cast<int>(c / (static_cast<int64_t>(cx_n) * cy_n));
  uint32_t m = 0;
  for (int k = 0; k < 8; ++k) {
    const double* nw = node_ptr(w, rx, ry, nb, x + (k & 1), y + ((k >> 1) & 1), z + ((k >> 2) & 1));
    for (int b = 0; b < nb; ++b)
      if (nw[b] != 0.0) m |= 1u << b;
  }
  mask[c] = m;
  count[c] = static_cast<uint32_t>(__popc(m));
}

__global__ void cell_fill_kernel(const double* __restrict__ w, int rx, int ry, int rz, int nb,
                                 const uint32_t* __restrict__ mask, const uint32_t* __restrict__ off,
                                 double* __restrict__ vals) {
  const int cx_n = rx - 1, cy_n = ry - 1, cz_n = rz - 1;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= static_cast<int64_t>(cx_n) * cy_n * cz_n) return;
  const int x = static_cast<int>(c % cx_n), y = static_cast<int>((c / cx_n) % cy_n),
            z = static_cast<int>(c / (static_cast<int64_t>(cx_n) * cy_n));
  double* o = vals + static_cast<size_t>(off[c]) * 8;
  int j = 0;
  for (uint32_t m = mask[c]; m; m &= m - 1, ++j) {
    const int b = __ffs(m) - 1;
    for (int k = 0; k < 8; ++k)
      o[8 * j + k] = node_ptr(w, rx, ry, nb, x + (k & 1), y + ((k >> 1) & 1), z + ((k >> 2) & 1))[b];
  }
}

int blocks_for(int64_t n, int threads) { return static_cast<int>((n + threads - 1) / threads); }

}  // namespace

void init_params_dev(ModelImpl& m, uint64_t seed) {
  const int chunk = 64;
  {
    const Pcg32 r = keyed_rng(seed, 0x6a1d, 17);
    const int64_t n = static_cast<int64_t>(m.n_grid);
    const int64_t threads = (n + chunk - 1) / chunk;
    init_uniform_kernel<<<blocks_for(threads, 256), 256, 0, m.stream>>>(m.grid_params.ptr, n, r, 0,
                                                                        -1e-4, 1e-4, chunk);
    ARFX_CUDA(cudaGetLastError());
  }
  {
    const Pcg32 r = keyed_rng(seed + 1, 0x3317, 29);
    ARFX_CUDA(cudaMemsetAsync(m.mlp_params.ptr, 0, m.n_mlp * sizeof(float), m.stream));
    int64_t draw = 0;
    for (int l = 0; l < m.mlp.n_layers; ++l) {
      const double s = std::sqrt(6.0 / double(m.mlp.lin[l]));
      const int64_t n = static_cast<int64_t>(m.mlp.lin[l]) * m.mlp.lout[l];
      const int64_t threads = (n + chunk - 1) / chunk;
      init_uniform_kernel<<<blocks_for(threads, 256), 256, 0, m.stream>>>(
          m.mlp_params.ptr + m.mlp.w_off[l], n, r, draw, -s, s, chunk);
      ARFX_CUDA(cudaGetLastError());
      draw += n;
    }
  }
}

void build_skinning_grid_dev(ModelImpl& m, double blend_factor) {
  SkelDev sk{};
  sk.nb = static_cast<int>(m.bones.size());
  for (int b = 0; b < sk.nb; ++b) {
    const HostBone& B = m.bones[static_cast<size_t>(b)];
    sk.head[b][0] = B.head.x;
    sk.head[b][1] = B.head.y;
    sk.head[b][2] = B.head.z;
    sk.tail[b][0] = B.tail.x;
    sk.tail[b][1] = B.tail.y;
    sk.tail[b][2] = B.tail.z;
  }
  const d3 lo = make3(m.skin_box.lo.x, m.skin_box.lo.y, m.skin_box.lo.z);
  const d3 e = make3(m.skin_box.hi.x - m.skin_box.lo.x, m.skin_box.hi.y - m.skin_box.lo.y,
                     m.skin_box.hi.z - m.skin_box.lo.z);
  const int64_t nn = static_cast<int64_t>(m.skin_res[0]) * m.skin_res[1] * m.skin_res[2];
  skinning_grid_kernel<<<blocks_for(nn, 128), 128, 0, m.stream>>>(
      m.skin.ptr, m.skin_res[0], m.skin_res[1], m.skin_res[2], lo, e, sk, blend_factor);
  ARFX_CUDA(cudaGetLastError());
}

__global__ void cell_pack_kernel(const uint32_t* __restrict__ mask, const uint32_t* __restrict__ off, int64_t nc,
                                 uint2* __restrict__ mo) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nc;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    mo[i] = make_uint2(mask[i], off[i]);
}

void build_cell_table(ModelImpl& m) {
  const int rx = m.skin_res[0], ry = m.skin_res[1], rz = m.skin_res[2];
  const int nb = static_cast<int>(m.bones.size());
  const int64_t nc = static_cast<int64_t>(rx - 1) * (ry - 1) * (rz - 1);
  m.cell_mask.alloc(static_cast<size_t>(nc));
  m.cell_off.alloc(static_cast<size_t>(nc));
  DevBuf<uint32_t> cnt;
  cnt.alloc(static_cast<size_t>(nc));
  cell_mask_kernel<<<blocks_for(nc, 128), 128, 0, m.stream>>>(m.skin.ptr, rx, ry, rz, nb,
                                                              m.cell_mask.ptr, cnt.ptr);
  ARFX_CUDA(cudaGetLastError());
  std::vector<uint32_t> h(static_cast<size_t>(nc));
  ARFX_CUDA(cudaMemcpyAsync(h.data(), cnt.ptr, h.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                            m.stream));
  ARFX_CUDA(cudaStreamSynchronize(m.stream));
  std::vector<uint32_t> off(h.size());
  uint64_t acc = 0;
  m.max_union = 1;
  for (size_t i = 0; i < h.size(); ++i) {
    off[i] = static_cast<uint32_t>(acc);
    acc += h[i];
    m.max_union = std::max(m.max_union, static_cast<int>(h[i]));
  }
  m.cell_vals.alloc(static_cast<size_t>(acc) * 8 + 8);
  ARFX_CUDA(cudaMemcpyAsync(m.cell_off.ptr, off.data(), off.size() * sizeof(uint32_t),
                            cudaMemcpyHostToDevice, m.stream));
  cell_fill_kernel<<<blocks_for(nc, 128), 128, 0, m.stream>>>(m.skin.ptr, rx, ry, rz, nb,
                                                              m.cell_mask.ptr, m.cell_off.ptr,
                                                              m.cell_vals.ptr);
  ARFX_CUDA(cudaGetLastError());
  // (union mask, value offset) pairs: one 8-byte load per skinning eval instead of two
  // dependent ones
  m.cell_mo.alloc(static_cast<size_t>(nc));
  cell_pack_kernel<<<blocks_for(nc, 128), 128, 0, m.stream>>>(m.cell_mask.ptr, m.cell_off.ptr, nc, m.cell_mo.ptr);
  ARFX_CUDA(cudaGetLastError());
  ARFX_CUDA(cudaStreamSynchronize(m.stream));
}

}  // namespace arfx
