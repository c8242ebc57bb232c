// render.cu -- the per-frame hot path on sm_100a.
//
//   K1 march_kernel     generate_ray + to_normalized + ray_box + sample_points +
//                       is_occupied (R/camera.hpp:61-70, R/render.hpp:15-37, :67-86,
//                       R/occupancy.hpp:71-85): lane per ray for the ray setup, then warp
//                       ballots over 32 samples at a time with an affine cell-space line
//                       (exact reference arithmetic within 1e-12 of a cell edge); one
//                       block-wide scan + atomic per block; exact recompute of occupied samples.
//   K2 deformer         inverse_lbs_ctx + in-box filter of posed_query_ctx
//                       (R/articulation.hpp:94-145, :163-181), FP64 exact, as the start
//                       pipeline of deform_starts.cuh (prune, sort, Newton, finalize).
//   K3 field            CanonicalField::query over the root pool (R/field.hpp:75-82): exact
//                       field_tile_kernel, or the tcgen05 decoder (field_tc.cu) for renders.
//   K4 composite_kernel max-density root selection (R/articulation.hpp:174) then
//                       composite (R/render.hpp:98-119), one thread per ray.
//   K5 occupancy        build_inference_grid (full or cell-interleaved shard) / update_training_grid /
//                       rebuild_mask / dilated_mask (R/occupancy.hpp:87-171) reuse K2 + K3.
//   L_density           density_points / reduce / flag kernels + K2/K3/K8.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <mutex>
#include <cstdio>

#include "deform.cuh"
#include "deform_starts.cuh"
#include "field.cuh"
#include "ray.cuh"
#include "model.h"

namespace arfx {

namespace {

constexpr int kMarchWarps = 8;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exact cell coordinate of OccupancyGrid::cell_of along one axis (R/occupancy.hpp:73-76):
// returns -1 when the point is outside ([u < 0 || u >= 1]), else int(u * res) clamped.
// The reference divides (u = (x - lo) / e). Only the integer decision matters here, so
// the quotient is first formed with the precomputed reciprocal (|q - u| <= 3 ulp) and the
// correctly rounded division is paid only when q * res lies within 1e-12 of an integer
// (or of the 0 / 1 bounds), where the two could round to different cells.
__device__ __forceinline__ int cell_axis_fast(double x, double lo, double e, double inv_e, int res) {
  const double d = dsub(x, lo);
  const double v = dmul(dmul(d, inv_e), static_cast<double>(res));
  const double fl = floor(v);
  const bool safe = (v - fl) > 1e-12 && (fl + 1.0 - v) > 1e-12 && fabs(d) > 1e-290;
  if (safe) {
    if (v < 0.0 || v >= static_cast<double>(res)) return -1;
    const int c = static_cast<int>(fl);
    return c > res - 1 ? res - 1 : c;
  }
  const double u = ddiv(d, e);
  if (u < 0 || u >= 1) return -1;
  const int c = static_cast<int>(dmul(u, static_cast<double>(res)));
  return (res - 1 < c) ? res - 1 : c;
}

// Cell-space coordinate v ~ (x - lo) / e * res evaluated by a cheaper formula (error
// <= ~1e-13): returns the cell, -1 outside, or -2 when v lies within 1e-12 of an integer
// (cell edge or box bound), where only the reference's own arithmetic may decide.
__device__ __forceinline__ int cell_from_v(double v, int res) {
  const double fl = floor(v);
  const double fr = dsub(v, fl);  // exact
  if (!(fr > 1e-12 && fr < 1.0 - 1e-12)) return -2;
  if (fl < 0.0 || fl >= static_cast<double>(res)) return -1;
  return static_cast<int>(fl);
}

__device__ __forceinline__ bool occupied_fast(const OccView& g, d3 x) {
  const int cx = cell_axis_fast(x.x, g.lo[0], g.e[0], g.inv_e[0], g.rx);
  if (cx < 0) return false;
  const int cy = cell_axis_fast(x.y, g.lo[1], g.e[1], g.inv_e[1], g.ry);
  if (cy < 0) return false;
  const int cz = cell_axis_fast(x.z, g.lo[2], g.e[2], g.inv_e[2], g.rz);
  if (cz < 0) return false;
  return g.mask[(static_cast<size_t>(cz) * g.ry + cy) * g.rx + cx] != 0;
}

// OccupancyGrid::is_occupied  R/occupancy.hpp:71-85 (reference form, kept for reference)
__device__ __forceinline__ bool occupied(const OccView& g, d3 x) {
  const double u0 = ddiv(dsub(x.x, g.lo[0]), g.e[0]);
  const double u1 = ddiv(dsub(x.y, g.lo[1]), g.e[1]);
  const double u2 = ddiv(dsub(x.z, g.lo[2]), g.e[2]);
  if (u0 < 0 || u1 < 0 || u2 < 0 || u0 >= 1 || u1 >= 1 || u2 >= 1) return false;
  int cx = static_cast<int>(dmul(u0, static_cast<double>(g.rx)));
  int cy = static_cast<int>(dmul(u1, static_cast<double>(g.ry)));
  int cz = static_cast<int>(dmul(u2, static_cast<double>(g.rz)));
  cx = (g.rx - 1 < cx) ? g.rx - 1 : cx;
  cy = (g.ry - 1 < cy) ? g.ry - 1 : cy;
  cz = (g.rz - 1 < cz) ? g.rz - 1 : cz;
  return g.mask[(static_cast<size_t>(cz) * g.ry + cy) * g.rx + cx] != 0;
}

struct MarchArgs {
  CameraView cam;
  const PoseCtx* pose;  // world -> normalized rigid read from device memory (graph-replayable)
  double nlo[3], nhi[3];
  OccView occ;
  int has_occ;
  int N, stratified;
  uint64_t seed, frame;
  const int32_t* rows;
  int n_rows, W;
  const int32_t *lpx, *lpy;  // list mode (training rays): ray r = (lpx[r], lpy[r]), ids = r
  long long n_list;
  double *sx, *sy, *sz, *sdelta;
  int32_t* sray;
  int16_t* sidx;
  int32_t *ray_first, *ray_count;
  unsigned long long* counters;
  long long cap;
  int rpw;  // rays per warp (1..32): small ray lists (training) spread over more warps
  const int* occ_box;  // occupied-cell bounding box (-x0, -y0, -z0, x1, y1, z1) or nullptr
  const uint32_t* occ_bits;  // the mask packed to bits (occ_bbox_kernel) or nullptr: u8 mask
  unsigned long long* stats;  // roofline accounting: [11] += samples tested in pass 1
};

// Bounding box of the occupied cells, for the march's empty-space skip: stored as
// (-x0, -y0, -z0, x1, y1, z1) so one atomicMax per entry reduces it; the buffer is preset
// to 0x80808080 (a large negative int) by a memset, so an all-empty mask leaves x1 < x0.
__global__ void __launch_bounds__(256) occ_bbox_kernel(OccView g, int* __restrict__ box, uint32_t* __restrict__ bits) {
  // also packs the mask to bits (one ballot per 32 consecutive cells): march pass 1 tests
  // occupancy in a 32 KB bit array (64^3) that stays L1-resident instead of the 256 KB u8 mask
  int b[6] = {INT_MIN, INT_MIN, INT_MIN, INT_MIN, INT_MIN, INT_MIN};
  const long long n = static_cast<long long>(g.rx) * g.ry * g.rz;
  const int lane = threadIdx.x & 31;
  for (long long base = static_cast<long long>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31); base < n;
       base += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = base + lane;
    const bool m = i < n && g.mask[i] != 0;
    const unsigned word = __ballot_sync(0xffffffffu, m);
    if (lane == 0) bits[base >> 5] = word;
    if (!m) continue;
    const int x = static_cast<int>(i % g.rx), y = static_cast<int>((i / g.rx) % g.ry),
              z = static_cast<int>(i / (static_cast<long long>(g.rx) * g.ry));
    b[0] = max(b[0], -x), b[1] = max(b[1], -y), b[2] = max(b[2], -z);
    b[3] = max(b[3], x), b[4] = max(b[4], y), b[5] = max(b[5], z);
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b[k] = max(b[k], __shfl_xor_sync(0xffffffffu, b[k], o));
  }
  if (lane == 0 && b[3] >= 0)
    for (int k = 0; k < 6; ++k) atomicMax(box + k, b[k]);
}

// Conservative sample-index range [i0, i1] of a ray that can reach an occupied cell: the
// cell-space line v = P + Q t against the occupied box grown by one cell per side, then
// one sample of slack each way (t_i = t_n + (i + j) step, j in [0, 1)). Samples outside
// cannot fall in an occupied cell -- the exact per-sample decision is untouched inside.
__device__ __forceinline__ void occ_index_range(const int* box, d3 P, d3 Q, double tn, double step, int N, int& i0,
                                                int& i1) {
  if (!(step > 0.0)) {  // degenerate segment: every sample at t_n, no skipping
    i0 = 0, i1 = N - 1;
    return;
  }
  double lo_t = -1e300, hi_t = 1e300;
  const double p[3] = {P.x, P.y, P.z}, q[3] = {Q.x, Q.y, Q.z};
  bool empty = box[3] < -box[0];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double lo = static_cast<double>(-box[a] - 1), hi = static_cast<double>(box[3 + a] + 2);
    if (fabs(q[a]) < 1e-300) {
      if (p[a] < lo || p[a] > hi) empty = true;
    } else {
      const double t1 = (lo - p[a]) / q[a], t2 = (hi - p[a]) / q[a];
      lo_t = fmax(lo_t, fmin(t1, t2));
      hi_t = fmin(hi_t, fmax(t1, t2));
    }
  }
  if (empty || !(lo_t <= hi_t)) {
    i0 = 1, i1 = 0;
    return;
  }
  const double a0 = floor((lo_t - tn) / step) - 1.0, a1 = ceil((hi_t - tn) / step) + 1.0;
  i0 = a0 < 0.0 ? 0 : (a0 > static_cast<double>(N) ? N : static_cast<int>(a0));
  i1 = a1 < 0.0 ? -1 : (a1 > static_cast<double>(N - 1) ? N - 1 : static_cast<int>(a1));
}

const int* launch_occ_bbox(Workspace& w, const OccView& g, cudaStream_t s) {
  w.occ_box.ensure(6);
  const long long n = static_cast<long long>(g.rx) * g.ry * g.rz;
  w.occ_bits.ensure(static_cast<size_t>((n + 31) / 32));
  ARFX_CUDA(cudaMemsetAsync(w.occ_box.ptr, 0x80, 6 * sizeof(int), s));
  occ_bbox_kernel<<<static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 1184))), 256, 0,
                    s>>>(g, w.occ_box.ptr, w.occ_bits.ptr);
  ARFX_CUDA(cudaGetLastError());
  return w.occ_box.ptr;
}

#ifndef ARFX_MARCH_BITS
#define ARFX_MARCH_BITS 1
#endif
// occupancy of cell (cx, cy, cz) (in range): the packed bits when present, else the u8 mask
__device__ __forceinline__ bool occ_test(const MarchArgs& A, int cx, int cy, int cz) {
  const size_t i = (static_cast<size_t>(cz) * A.occ.ry + cy) * A.occ.rx + cx;
  return A.occ_bits ? ((__ldg(A.occ_bits + (i >> 5)) >> (i & 31)) & 1u) != 0 : A.occ.mask[i] != 0;
}

__device__ __forceinline__ double jitter_at(const MarchArgs& A, Pcg32 base, int i) {
  if (!A.stratified) return 0.5;
  pcg_advance(base, static_cast<uint64_t>(i));
  return pcg_double(base);
}

__device__ __forceinline__ double shfl_d(double v, int src) {
  return __longlong_as_double(__shfl_sync(0xffffffffu, __double_as_longlong(v), src));
}
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  return static_cast<uint64_t>(__shfl_sync(0xffffffffu, static_cast<long long>(v), src));
}

// K1. Block = 256 rays per iteration. Lane l of warp w sets up ray (w, l) once (make_ray:
// ~100 FP64 incl. 4 divisions and a sqrt); the warp then walks its 32 rays, broadcasting
// each ray's geometry by shuffle and testing its N samples 32 at a time (ballots kept in
// dynamic smem). One block-wide exclusive scan of the 256 ray counts and one atomic place
// the block's samples; the second pass recomputes t / x only for occupied samples.
#ifndef ARFX_MARCH_MIN_BLOCKS
#define ARFX_MARCH_MIN_BLOCKS 2
#endif
__global__ void __launch_bounds__(kMarchWarps * 32, ARFX_MARCH_MIN_BLOCKS) march_kernel(MarchArgs A) {
  extern __shared__ unsigned march_bal[];  // [256 rays][K]
  __shared__ double w2n[12];
  __shared__ int obox[6];
  if (threadIdx.x < 12) w2n[threadIdx.x] = A.pose->w2n[threadIdx.x];
  if (threadIdx.x < 6) obox[threadIdx.x] = A.occ_box ? A.occ_box[threadIdx.x] : 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long n_rays = A.lpx ? A.n_list : static_cast<long long>(A.n_rows) * A.W;
  const int K = (A.N + 31) >> 5;
  const int kRays = kMarchWarps * A.rpw;
  for (long long g0 = static_cast<long long>(blockIdx.x) * kRays; g0 < n_rays;
       g0 += static_cast<long long>(gridDim.x) * kRays) {
    // ---- this lane's ray (lanes >= rpw hold none)
    const long long r = lane < A.rpw ? g0 + warp * A.rpw + lane : n_rays;
    int pix = -1, rid = -1;  // pix keys the RNG stream (R/render.hpp:201); rid indexes outputs
    RayGeom R{};
    double step = 0.0;
    Pcg32 rng{0, 0};
    d3 cP = make3(0.0, 0.0, 0.0), cQ = cP;
    int r_i0 = 0, r_i1 = A.N - 1;  // samples that can reach an occupied cell
    if (r < n_rays) {
      int px, py;
      if (A.lpx) {
        px = A.lpx[r];
        py = A.lpy[r];
      } else {
        py = A.rows[r / A.W];
        px = static_cast<int>(r % A.W);
      }
      pix = py * A.W + px;
      rid = A.lpx ? static_cast<int>(r) : pix;
      R = make_ray(A.cam, w2n, A.nlo, A.nhi, px, py);
      R.valid = R.valid && A.N > 0;
      if (R.valid) {
        step = ddiv(dsub(R.tf, R.tn), static_cast<double>(A.N));
        if (A.stratified) rng = keyed_rng(A.seed, A.frame, static_cast<uint64_t>(pix));
        // cell-space ray: v(t) = P + Q t ~ (G^-1 (o + d t) - lo) / e * res (fast path only)
        const d3 on = rigid_apply(w2n, R.o);
        const d3 dn = matvec(w2n, R.d);
        const double sx = A.occ.inv_e[0] * A.occ.rx, sy = A.occ.inv_e[1] * A.occ.ry, sz = A.occ.inv_e[2] * A.occ.rz;
        cP = make3((on.x - A.occ.lo[0]) * sx, (on.y - A.occ.lo[1]) * sy, (on.z - A.occ.lo[2]) * sz);
        cQ = make3(dn.x * sx, dn.y * sy, dn.z * sz);
        if (A.has_occ && A.occ_box) occ_index_range(obox, cP, cQ, R.tn, step, A.N, r_i0, r_i1);
      }
    }
    int my_count = 0;
    if (A.stats) {  // samples pass 1 tests (the occupied-box range of each valid ray)
      unsigned long long tested = (R.valid && r_i1 >= r_i0) ? static_cast<unsigned long long>(r_i1 - r_i0 + 1) : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tested += __shfl_xor_sync(0xffffffffu, tested, o);
      if (lane == 0 && tested) atomicAdd(A.stats + 11, tested);
    }
    if (A.rpw == 32) {
      // ---- pass 1, thread per ray (full warps): each lane walks its own ray's samples
      // (stratified jitter drawn sequentially from the ray's stream: draw i == jitter_at(i)),
      // only over [r_i0, r_i1], the samples that can reach the occupied box
      if (R.valid) {
        unsigned* bal = march_bal + (warp * 32 + lane) * K;
        for (int k = 0; k < K; ++k) bal[k] = 0u;
        if (!A.has_occ) {
          for (int k = 0; k < K; ++k) bal[k] = (A.N - 32 * k >= 32) ? 0xffffffffu : ((1u << (A.N - 32 * k)) - 1u);
          my_count = A.N;
        } else {
          Pcg32 g = rng;
          if (A.stratified && r_i0 > 0) pcg_advance(g, static_cast<uint64_t>(r_i0));
          unsigned word = 0u;
          int wk = r_i0 >> 5;
          for (int i = r_i0; i <= r_i1; ++i) {
            const double t = sample_t(R.tn, step, i, A.stratified ? pcg_double(g) : 0.5);
            const int cx = cell_from_v(__fma_rn(cQ.x, t, cP.x), A.occ.rx);
            const int cy = cell_from_v(__fma_rn(cQ.y, t, cP.y), A.occ.ry);
            const int cz = cell_from_v(__fma_rn(cQ.z, t, cP.z), A.occ.rz);
            bool f = false;
            if (cx == -2 || cy == -2 || cz == -2)
              f = occupied(A.occ, rigid_apply(w2n, add3(R.o, mul3(R.d, t))));
            else if (cx >= 0 && cy >= 0 && cz >= 0)
              f = occ_test(A, cx, cy, cz);
            if ((i >> 5) != wk) {
              bal[wk] = word;
              word = 0u;
              wk = i >> 5;
            }
            if (f) {
              word |= 1u << (i & 31);
              ++my_count;
            }
          }
          if (r_i0 <= r_i1) bal[wk] = word;
        }
      }
    } else {
      // ---- pass 1, warp per ray (small batches, rays per warp < 32): lanes over samples
      const unsigned vmask = __ballot_sync(0xffffffffu, R.valid);
      for (int j = 0; j < 32; ++j) {
        if (!((vmask >> j) & 1u)) continue;
        const double Px = shfl_d(cP.x, j), Py = shfl_d(cP.y, j), Pz = shfl_d(cP.z, j);
        const double Qx = shfl_d(cQ.x, j), Qy = shfl_d(cQ.y, j), Qz = shfl_d(cQ.z, j);
        const double tn = shfl_d(R.tn, j), st = shfl_d(step, j);
        const Pcg32 rg{shfl_u64(rng.state, j), shfl_u64(rng.inc, j)};
        const int pj = __shfl_sync(0xffffffffu, pix, j);
        const int ri0 = __shfl_sync(0xffffffffu, r_i0, j), ri1 = __shfl_sync(0xffffffffu, r_i1, j);
        unsigned* bal = march_bal + (warp * 32 + j) * K;
        int count = 0;
        for (int k = 0; k < K; ++k) {
          const int i = k * 32 + lane;
          if (k * 32 > ri1 || k * 32 + 31 < ri0) {  // whole chunk outside the occupied box
            if (lane == 0) bal[k] = 0u;
            continue;
          }
          bool f = false;
          if (i < A.N && i >= ri0 && i <= ri1) {
            if (A.has_occ) {
              // t exactly as the reference; the cell decision from v = P + Q t (one FMA per
              // axis), exact reference arithmetic only within 1e-12 of a cell edge
              const double t = sample_t(tn, st, i, jitter_at(A, rg, i));
              const int cx = cell_from_v(__fma_rn(Qx, t, Px), A.occ.rx);
              const int cy = cell_from_v(__fma_rn(Qy, t, Py), A.occ.ry);
              const int cz = cell_from_v(__fma_rn(Qz, t, Pz), A.occ.rz);
              if (cx == -2 || cy == -2 || cz == -2) {
                const RayGeom Rj = make_ray(A.cam, w2n, A.nlo, A.nhi, pj % A.W, pj / A.W);
                f = occupied(A.occ, rigid_apply(w2n, add3(Rj.o, mul3(Rj.d, t))));
              } else if (cx >= 0 && cy >= 0 && cz >= 0) {
                f = occ_test(A, cx, cy, cz);
              }
            } else {
              f = true;
            }
          }
          const unsigned b = __ballot_sync(0xffffffffu, f);
          if (lane == 0) bal[k] = b;
          count += __popc(b);
        }
        if (lane == j) my_count = count;
      }
    }
    // ---- warp exclusive scan of the ray counts, one atomic per warp (no block barrier:
    // a warp whose rays cross few occupied cells does not wait for the block's slowest ray)
    int incl = my_count;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int wtot = __shfl_sync(0xffffffffu, incl, 31);
    long long wbase = 0;
    if (lane == 0 && wtot) wbase = static_cast<long long>(atomicAdd(A.counters, static_cast<unsigned long long>(wtot)));
    wbase = static_cast<long long>(__shfl_sync(0xffffffffu, static_cast<unsigned long long>(wbase), 0));
    const long long first = wbase + (incl - my_count);
    if (r < n_rays) {
      A.ray_first[rid] = static_cast<int32_t>(first < A.cap ? first : A.cap);
      A.ray_count[rid] = (first + my_count <= A.cap) ? my_count : 0;
    }
    // ---- pass 2: write the occupied samples of each ray
    const unsigned cmask = __ballot_sync(0xffffffffu, my_count > 0);
    for (int j = 0; j < 32; ++j) {
      if (!((cmask >> j) & 1u)) continue;
      const d3 o = make3(shfl_d(R.o.x, j), shfl_d(R.o.y, j), shfl_d(R.o.z, j));
      const d3 d = make3(shfl_d(R.d.x, j), shfl_d(R.d.y, j), shfl_d(R.d.z, j));
      const double tn = shfl_d(R.tn, j), tf = shfl_d(R.tf, j), st = shfl_d(step, j);
      const Pcg32 rg{shfl_u64(rng.state, j), shfl_u64(rng.inc, j)};
      const long long f0 = static_cast<long long>(shfl_u64(static_cast<uint64_t>(first), j));
      const int rj = __shfl_sync(0xffffffffu, rid, j);
      const unsigned* bal = march_bal + (warp * 32 + j) * K;
      long long run = f0;
      for (int k = 0; k < K; ++k) {
        const unsigned b = bal[k];
        if ((b >> lane) & 1u) {
          const long long pos = run + __popc(b & lanemask_lt());
          if (pos < A.cap) {
            const int i = k * 32 + lane;
            const double t = sample_t(tn, st, i, jitter_at(A, rg, i));
            double delta;
            if (i + 1 < A.N) delta = dsub(sample_t(tn, st, i + 1, jitter_at(A, rg, i + 1)), t);
            else delta = dsub(tf, t);
            const d3 xn = rigid_apply(w2n, add3(o, mul3(d, t)));
            A.sx[pos] = xn.x;
            A.sy[pos] = xn.y;
            A.sz[pos] = xn.z;
            A.sdelta[pos] = delta;
            A.sray[pos] = rj;
            A.sidx[pos] = static_cast<int16_t>(i);
          }
        }
        run += __popc(b);
      }
    }
    __syncwarp();  // march_bal rows are per warp: the next group's pass 1 reuses them
  }
}

// ---- K2 sources: where the posed targets x' come from ---------------------------

struct ListSrc {  // posed samples from K1 or a user batch
  static constexpr bool kSinglePose = true;
  const double *x, *y, *z;
  const unsigned long long* n_dev;  // device count (K1) or nullptr
  long long n, cap;
  __device__ long long count() const {
    long long c = n_dev ? static_cast<long long>(*n_dev) : n;
    return c < cap ? c : cap;
  }
  __device__ d3 point(long long i, int& pose) const {
    pose = 0;
    return make3(x[i], y[i], z[i]);
  }
};

struct AosSrc {  // user batch of xyz triples (inverse_lbs API / microbench)
  static constexpr bool kSinglePose = true;
  const double* p;
  long long n;
  __device__ long long count() const { return n; }
  __device__ d3 point(long long i, int& pose) const {
    pose = 0;
    return make3(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
  }
};

struct CellSrc {  // cell centres of an occupancy grid  R/occupancy.hpp:53-58, :141-144
  static constexpr bool kSinglePose = true;
  int rx, ry, rz;
  double lo[3], cs[3];
  // multi-GPU shard: cells c = offset + stride * i (cell-interleaved, so every rank gets an
  // equal share of the body's cells whatever its shape); 0 / 1 for the whole grid
  int offset = 0, stride = 1;
  __device__ long long count() const {
    return (static_cast<long long>(rx) * ry * rz - offset + stride - 1) / stride;
  }
  __device__ d3 point(long long i, int& pose) const {
    pose = 0;
    const long long c = offset + static_cast<long long>(stride) * i;
    const int ix = static_cast<int>(c % rx), iy = static_cast<int>((c / rx) % ry),
              iz = static_cast<int>(c / (static_cast<long long>(rx) * ry));
    return make3(dadd(lo[0], dmul(dadd(static_cast<double>(ix), 0.5), cs[0])),
                 dadd(lo[1], dmul(dadd(static_cast<double>(iy), 0.5), cs[1])),
                 dadd(lo[2], dmul(dadd(static_cast<double>(iz), 0.5), cs[2])));
  }
};

struct JitterSrc {  // update_training_grid draws  R/occupancy.hpp:160-166
  static constexpr bool kSinglePose = false;
  int rx, ry, rz, n_poses;
  double lo[3], cs[3];
  uint64_t seed, step;
  __device__ long long count() const { return static_cast<long long>(rx) * ry * rz; }
  __device__ d3 point(long long i, int& pose) const {
    const int ix = static_cast<int>(i % rx), iy = static_cast<int>((i / rx) % ry),
              iz = static_cast<int>(i / (static_cast<long long>(rx) * ry));
    Pcg32 r = keyed_rng(seed, 0x0cc0, static_cast<uint64_t>(i), step);
    pose = static_cast<int>(pcg_below(r, static_cast<uint32_t>(n_poses)));
    const double jx = pcg_double(r);
    const double jy = pcg_double(r);
    const double jz = pcg_double(r);
    return make3(dadd(lo[0], dmul(dadd(static_cast<double>(ix), jx), cs[0])),
                 dadd(lo[1], dmul(dadd(static_cast<double>(iy), jy), cs[1])),
                 dadd(lo[2], dmul(dadd(static_cast<double>(iz), jz), cs[2])));
  }
};

// ---- K3: field over the root pool -----------------------------------------
//
// Standard config (16 levels x 2 features, 32-64-64-4): tiles of 128 pool queries.
//  1. thread q: normalized coords u of query q (3 f64 divisions, once per query);
//  2. thread (q, level): one level of the encode -- 8 independent float2 gathers per
//     thread, 16x more gathers in flight than a thread-per-query encode;
//  3. thread q: exact MLP (feature-major first layer) from the shared-memory features.
constexpr int kFieldTile = 128;

template <int L, int HID>
__global__ void __launch_bounds__(kFieldTile) field_tile_kernel(FieldView F, const double* __restrict__ px,
                                                                const double* __restrict__ py,
                                                                const double* __restrict__ pz,
                                                                const int32_t* __restrict__ owner,
                                                                float4* __restrict__ res,
                                                                const unsigned long long* n_dev, long long cap,
                                                                unsigned long long* stats, long long team_max) {
  constexpr int IN = 2 * L;
  extern __shared__ float4 ft_smem4[];
  float* W0T = reinterpret_cast<float*>(ft_smem4);          // [IN][HID]
  float* Wr = W0T + IN * HID;                                // b0, W1, b1, W2, b2
  const int n_rest = F.n_mlp - IN * HID;
  float* feats = Wr + ((n_rest + 3) / 4) * 4;                // [tile][IN + 1]
  double* U = reinterpret_cast<double*>(feats + kFieldTile * (IN + 1) + (kFieldTile * (IN + 1)) % 2);  // [tile][3]
  int* valid = reinterpret_cast<int*>(U + 3 * kFieldTile);
  long long n = static_cast<long long>(*n_dev);
  n = n < cap ? n : cap;
  if (n <= team_max) return;  // small batch: field_team_kernel has it
  if (static_cast<long long>(blockIdx.x) * kFieldTile >= n) return;
  for (int i = threadIdx.x; i < IN * HID; i += kFieldTile) {  // W0 transposed
    const int o = i / IN, k = i % IN;
    W0T[k * HID + o] = __ldg(F.mlp + i);
  }
  for (int i = threadIdx.x; i < n_rest; i += kFieldTile) Wr[i] = __ldg(F.mlp + IN * HID + i);
  for (long long t0 = static_cast<long long>(blockIdx.x) * kFieldTile; t0 < n;
       t0 += static_cast<long long>(gridDim.x) * kFieldTile) {
    __syncthreads();
    {
      const long long q = t0 + threadIdx.x;
      const bool ok = q < n && owner[q] >= 0;
      valid[threadIdx.x] = ok;
      if (stats) {
        const int c = __syncthreads_count(ok);
        if (threadIdx.x == 0 && c) atomicAdd(stats + 5, static_cast<unsigned long long>(c));
      }
      if (ok) {
        double u[3];
        normalize_point(F, make3(px[q], py[q], pz[q]), u);
        U[3 * threadIdx.x + 0] = u[0];
        U[3 * threadIdx.x + 1] = u[1];
        U[3 * threadIdx.x + 2] = u[2];
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int pass = 0; pass < L; ++pass) {
      // warp-uniform level (no divergence on the direct/wrap/hash kind), 32 queries per warp
      const int l = pass;
      const int ql = threadIdx.x;
      if (valid[ql]) {
        const double u[3] = {U[3 * ql], U[3 * ql + 1], U[3 * ql + 2]};
        const float2 o = encode_level_f2(F, l, u);
        feats[ql * (IN + 1) + 2 * l] = o.x;
        feats[ql * (IN + 1) + 2 * l + 1] = o.y;
      }
    }
    __syncthreads();
    if (valid[threadIdx.x]) {
      float logits[4];
      mlp_forward_fm<IN, HID, 2, 4>(W0T, Wr, feats + threadIdx.x * (IN + 1), logits);
      res[t0 + threadIdx.x] = make_float4(softplus_f(logits[0]), logistic_f(logits[1]), logistic_f(logits[2]),
                                          logistic_f(logits[3]));
    }
  }
}

// Small batches (occupancy grids: ~10^4 queries; training: ~10^4-10^5): the tile kernel's
// thread-per-query MLP is a 13k-op serial chain per thread, so a few thousand queries leave
// the GPU idle. Here a 64-thread team carries 4 queries: thread (query, level) encodes,
// thread o computes hidden unit o of each layer (its sum in the reference's input order, so
// the outputs are bit-identical to field_tile_kernel's), 4 chains per weight load.
constexpr int kFtTeam = 64, kFtTeams = 4, kFtQ = 4;
__global__ void __launch_bounds__(kFtTeam * kFtTeams) field_team_kernel(FieldView F, const double* __restrict__ px,
                                                                        const double* __restrict__ py,
                                                                        const double* __restrict__ pz,
                                                                        const int32_t* __restrict__ owner,
                                                                        float4* __restrict__ res,
                                                                        const unsigned long long* n_dev, long long cap,
                                                                        unsigned long long* stats, long long team_max,
                                                                        float* __restrict__ act) {
  constexpr int IN = 32, HID = 64, W0S = IN + 1, W1S = HID + 1;
  __shared__ float W0p[HID * W0S], W1p[HID * W1S], W2p[4 * W1S], Bs[2 * HID + 4];
  __shared__ float X[kFtTeams][kFtQ][IN], H1[kFtTeams][kFtQ][HID], H2[kFtTeams][kFtQ][HID];
  __shared__ int OK[kFtTeams][kFtQ];
  long long n = static_cast<long long>(*n_dev);
  n = n < cap ? n : cap;
  if (n > team_max) return;  // large batch: field_tile_kernel has it
  const float* W = F.mlp;
  const float* W1g = W + IN * HID + HID;
  const float* W2g = W1g + HID * HID + HID;
  for (int e = threadIdx.x; e < HID * IN; e += blockDim.x) W0p[(e / IN) * W0S + e % IN] = __ldg(W + e);
  for (int e = threadIdx.x; e < HID * HID; e += blockDim.x) W1p[(e / HID) * W1S + e % HID] = __ldg(W1g + e);
  for (int e = threadIdx.x; e < 4 * HID; e += blockDim.x) W2p[(e / HID) * W1S + e % HID] = __ldg(W2g + e);
  for (int e = threadIdx.x; e < HID; e += blockDim.x) {
    Bs[e] = __ldg(W + IN * HID + e);
    Bs[HID + e] = __ldg(W1g + HID * HID + e);
  }
  if (threadIdx.x < 4) Bs[2 * HID + threadIdx.x] = __ldg(W2g + 4 * HID + threadIdx.x);
  __syncthreads();
  const int team = threadIdx.x / kFtTeam, t = threadIdx.x % kFtTeam;
  const int ej = t >> 4, el = t & 15;
  for (long long k0 = (static_cast<long long>(blockIdx.x) * kFtTeams + team) * kFtQ; k0 < n;
       k0 += static_cast<long long>(gridDim.x) * kFtTeams * kFtQ) {
    {
      const long long q = k0 + ej;
      const bool ok = q < n && owner[q] >= 0;
      if (el == 0) OK[team][ej] = ok;
      if (ok) {
        double u[3];
        normalize_point(F, make3(px[q], py[q], pz[q]), u);
        const float2 o = encode_level_f2(F, el, u);
        X[team][ej][2 * el] = o.x;
        X[team][ej][2 * el + 1] = o.y;
      }
      if (stats && el == 0 && ok) atomicAdd(stats + 5, 1ull);
    }
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "n"(kFtTeam) : "memory");
    {
      float a[kFtQ];
#pragma unroll
      for (int j = 0; j < kFtQ; ++j) a[j] = Bs[t];
      for (int i = 0; i < IN; ++i) {
        const float w = W0p[t * W0S + i];
#pragma unroll
        for (int j = 0; j < kFtQ; ++j) a[j] = fadd(a[j], fmul(w, X[team][j][i]));
      }
#pragma unroll
      for (int j = 0; j < kFtQ; ++j) H1[team][j][t] = (a[j] < 0.0f) ? 0.0f : a[j];
    }
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "n"(kFtTeam) : "memory");
    {
      float a[kFtQ];
#pragma unroll
      for (int j = 0; j < kFtQ; ++j) a[j] = Bs[HID + t];
      for (int i = 0; i < HID; ++i) {
        const float w = W1p[t * W1S + i];
#pragma unroll
        for (int j = 0; j < kFtQ; ++j) a[j] = fadd(a[j], fmul(w, H1[team][j][i]));
      }
#pragma unroll
      for (int j = 0; j < kFtQ; ++j) H2[team][j][t] = (a[j] < 0.0f) ? 0.0f : a[j];
    }
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "n"(kFtTeam) : "memory");
    if (t < kFtQ) {  // thread j: the 4 logits of query j (R/field.hpp:78-81)
      const int j = t;
      if (OK[team][j]) {
        float lg[4];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          float a = Bs[2 * HID + o];
          for (int i = 0; i < HID; ++i) a = fadd(a, fmul(W2p[o * W1S + i], H2[team][j][i]));
          lg[o] = a;
        }
        res[k0 + j] = make_float4(softplus_f(lg[0]), logistic_f(lg[1]), logistic_f(lg[2]), logistic_f(lg[3]));
        if (act) {
#pragma unroll
          for (int o = 0; o < 4; ++o) act[(k0 + j) * kActStride + 160 + o] = lg[o];
        }
      }
    }
    if (act) {  // training: keep X | H1 | H2 for the field backward (K8a)
#pragma unroll
      for (int j = 0; j < kFtQ; ++j) {
        if (!OK[team][j]) continue;
        float* A = act + (k0 + j) * kActStride;
        if (t < IN) A[t] = X[team][j][t];
        A[IN + t] = H1[team][j][t];
        A[IN + HID + t] = H2[team][j][t];
      }
    }
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "n"(kFtTeam) : "memory");
  }
}

bool field_is_standard_host(const FieldView& F) {
  return F.F == 2 && F.L == 16 && F.in_dim == 32 && F.hidden == 64 && F.n_layers == 3 && F.out_dim == 4;
}

size_t field_tile_smem(const FieldView& F) {
  const int IN = 32, HID = 64;
  const int n_rest = F.n_mlp - IN * HID;
  size_t b = static_cast<size_t>(IN * HID + (n_rest + 3) / 4 * 4) * 4;
  b += static_cast<size_t>(kFieldTile * (IN + 1) + (kFieldTile * (IN + 1)) % 2) * 4;
  b += static_cast<size_t>(3 * kFieldTile) * 8 + kFieldTile * 4;
  return b;
}

// Generic configs: one thread per query.

__global__ void __launch_bounds__(128) field_pool_kernel(FieldView F, const double* __restrict__ px,
                                                         const double* __restrict__ py,
                                                         const double* __restrict__ pz,
                                                         const int32_t* __restrict__ owner,
                                                         float4* __restrict__ res,
                                                         const unsigned long long* n_dev, long long cap,
                                                         int mlp_in_smem) {
  extern __shared__ float4 wsm4[];
  long long n = static_cast<long long>(*n_dev);
  n = n < cap ? n : cap;
  if (static_cast<long long>(blockIdx.x) * blockDim.x >= n) return;  // no work: skip the weight staging
  const float* W = F.mlp;
  if (mlp_in_smem) {
    const float4* src = reinterpret_cast<const float4*>(F.mlp);
    for (int i = threadIdx.x; i < (F.n_mlp + 3) / 4; i += blockDim.x) wsm4[i] = __ldg(src + i);
    __syncthreads();
    W = reinterpret_cast<const float*>(wsm4);
  }
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (owner[i] < 0) continue;
    res[i] = field_query_exact(F, W, make3(px[i], py[i], pz[i]));
  }
}

// max-density root of a posed sample (R/articulation.hpp:170-179); returns slot or -1
__device__ __forceinline__ int select_root(const uint8_t* snroot, const int32_t* sbase,
                                           const float4* pres, long long s, float4& best) {
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

// ---- K4: selection + composite ----------------------------------------------

struct CompositeArgs {
  const int32_t* rows;
  int n_rows, W;
  const int32_t *ray_first, *ray_count;
  const double* sdelta;
  const uint8_t* snroot;
  const int32_t* sbase;
  const float4* pres;
  int8_t* ssel;
  double eps;
  float *rgb, *alpha;
};

__global__ void composite_kernel(CompositeArgs A) {
  const long long n_rays = static_cast<long long>(A.n_rows) * A.W;
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rays;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int py = A.rows[r / A.W], px = static_cast<int>(r % A.W);
    const int pix = py * A.W + px;
    const int first = A.ray_first[pix], cnt = A.ray_count[pix];
    double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0, acc = 0.0;
    bool done = A.eps > 0 && T <= A.eps;
    // 4 samples at a time: their root selections (dependent snroot -> sbase -> pres loads)
    // and deltas are independent of the compositing chain, so they are fetched together
    // first; the chain then runs over them in order, exactly as the per-sample loop
    for (int j0 = 0; j0 < cnt; j0 += 4) {
      float4 vv[4];
      int ss[4];
      double dd[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ss[u] = -1;
        dd[u] = 0.0;
        vv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j0 + u < cnt) {
          const long long s = first + j0 + u;
          ss[u] = select_root(A.snroot, A.sbase, A.pres, s, vv[u]);
          A.ssel[s] = static_cast<int8_t>(ss[u]);
          if (!done && ss[u] >= 0) dd[u] = A.sdelta[s];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j0 + u >= cnt || done || ss[u] < 0) continue;
        const double sigma = static_cast<double>(vv[u].x);
        if (sigma <= 0.0) continue;
        const double alpha = -expm1(-dmul(sigma, dd[u]));
        const double w = dmul(alpha, T);
        cr = dadd(cr, dmul(static_cast<double>(vv[u].y), w));
        cg = dadd(cg, dmul(static_cast<double>(vv[u].z), w));
        cb = dadd(cb, dmul(static_cast<double>(vv[u].w), w));
        acc = dadd(acc, w);
        T = dmul(T, dsub(1.0, alpha));
        if (A.eps > 0 && T <= A.eps) done = true;
      }
    }
    A.rgb[3 * pix + 0] = static_cast<float>(cr);
    A.rgb[3 * pix + 1] = static_cast<float>(cg);
    A.rgb[3 * pix + 2] = static_cast<float>(cb);
    A.alpha[pix] = static_cast<float>(acc);
  }
}

// ---- occupancy kernels ----------------------------------------------------

__global__ void finalize_counters_kernel(unsigned long long* c, long long cap_posed) {
  if (static_cast<long long>(c[0]) > cap_posed) c[3] += 1;
}

__global__ void occ_values_kernel(long long n, const uint8_t* __restrict__ snroot,
                                  const int32_t* __restrict__ sbase, const float4* __restrict__ pres,
                                  float* __restrict__ values, float decay, int decayed_max) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 v;
    const int sel = select_root(snroot, sbase, pres, i, v);
    const double d = sel >= 0 ? static_cast<double>(v.x) : 0.0;
    const float fresh = static_cast<float>((1.0 < d) ? 1.0 : d);  // float(std::min(d, 1.0))
    if (decayed_max) {
      const float old = __fmul_rn(decay, values[i]);
      values[i] = (old < fresh) ? fresh : old;  // std::max  R/occupancy.hpp:168
    } else {
      values[i] = fresh;
    }
  }
}

// rebuild_mask + dilated_mask (R/occupancy.hpp:87-91, :101-125) in one pass: a cell is
// set iff any cell of its clipped (2r+1)^3 box has values >= thr -- the separable x, y, z
// box dilation of the thresholded mask, evaluated directly (warps walk x-rows, so the
// neighbouring values come from L1)
__global__ void __launch_bounds__(256) occ_rebuild_kernel(int rx, int ry, int rz, int r, const float* __restrict__ values,
                                                          float thr, uint8_t* __restrict__ mask) {
  const long long n = static_cast<long long>(rx) * ry * rz;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int x = static_cast<int>(i % rx), y = static_cast<int>((i / rx) % ry),
              z = static_cast<int>(i / (static_cast<long long>(rx) * ry));
    const int x0 = max(x - r, 0), x1 = min(x + r, rx - 1), y0 = max(y - r, 0), y1 = min(y + r, ry - 1),
              z0 = max(z - r, 0), z1 = min(z + r, rz - 1);
    bool v = false;
    for (int zz = z0; zz <= z1 && !v; ++zz)
      for (int yy = y0; yy <= y1 && !v; ++yy) {
        const float* row = values + (static_cast<long long>(zz) * ry + yy) * rx;
        for (int xx = x0; xx <= x1; ++xx) v = v || (__ldg(row + xx) >= thr);
      }
    mask[i] = v ? 1 : 0;
  }
}

// ---- batch query kernels (API) ----------------------------------------------

__global__ void occ_query_kernel(OccView g, const double* __restrict__ pts, long long n, uint8_t* out) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    out[i] = occupied_fast(g, make3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2])) ? 1 : 0;
}


__global__ void posed_out_kernel(long long n, const uint8_t* __restrict__ snroot,
                                 const int32_t* __restrict__ sbase, const float4* __restrict__ pres,
                                 const double* __restrict__ px, const double* __restrict__ py,
                                 const double* __restrict__ pz, float* dens, float* col,
                                 double* canon, uint8_t* has) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int sel = select_root(snroot, sbase, pres, i, v);
    has[i] = sel >= 0;
    dens[i] = sel >= 0 ? v.x : 0.f;
    col[3 * i + 0] = sel >= 0 ? v.y : 0.f;
    col[3 * i + 1] = sel >= 0 ? v.z : 0.f;
    col[3 * i + 2] = sel >= 0 ? v.w : 0.f;
    const long long p = sel >= 0 ? sbase[i] + sel : -1;
    canon[3 * i + 0] = p >= 0 ? px[p] : 0.0;
    canon[3 * i + 1] = p >= 0 ? py[p] : 0.0;
    canon[3 * i + 2] = p >= 0 ? pz[p] : 0.0;
  }
}

__global__ void field_query_kernel(FieldView F, const double* __restrict__ pts, long long n, float4* out,
                                   int* domain_err) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const d3 x = make3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    if (!field_contains(F, x)) {
      atomicExch(domain_err, 1);
      continue;
    }
    out[i] = field_query_exact(F, F.mlp, x);
  }
}

__global__ void hash_encode_kernel(FieldView F, const double* __restrict__ pts, long long n, float* out,
                                   int* domain_err) {
  const int D = F.L * F.F;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const d3 x = make3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    if (!field_contains(F, x)) {
      atomicExch(domain_err, 1);
      continue;
    }
    if (F.F == 2) hash_encode_f2(F, x, out + i * D);
    else hash_encode_generic(F, x, out + i * D);
  }
}

__global__ void skin_weights_kernel(SkinView S, const double* __restrict__ pts, long long n, double* w) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    skin_weights_dense(S, make3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]), w + i * S.nb);
}

int sm_count() {
  return device_sm_count();
}

int grid_for(long long n, int threads, int per_sm) {
  const long long want = (n + threads - 1) / threads;
  const long long cap = static_cast<long long>(sm_count()) * per_sm;
  return static_cast<int>(std::max(1LL, std::min(want, cap)));
}

template <class Kern>
int persistent_grid(Kern kernel, int threads, size_t smem, long long n_hint) {
  const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kernel), threads, smem);
  const long long want = (n_hint + threads - 1) / threads;
  return static_cast<int>(std::max(1LL, std::min(want, static_cast<long long>(sm_count()) * per_sm)));
}


template <class Src>
void launch_finalize(ModelImpl& m, const Src& src, const PoolSink& K, long long n, cudaStream_t s) {
  Workspace& w = m.ws();
  finalize_pool_kernel<Src><<<resident_grid(finalize_pool_kernel<Src>, 256, 0, n), 256, 0, s>>>(src, w.smask.ptr, w.scount.ptr, w.res4.ptr,
                                                                m.inv.dedup_radius, K,
                                                                static_cast<long long>(w.cap_starts));
  ARFX_CUDA(cudaGetLastError());
}
template <class Src>
void launch_finalize(ModelImpl& m, const Src& src, const RootsSink& K, long long n, cudaStream_t s) {
  Workspace& w = m.ws();
  finalize_roots_kernel<Src><<<grid_for(n, 256, 8), 256, 0, s>>>(src, w.smask.ptr, w.scount.ptr, w.res4.ptr,
                                                                 m.inv.dedup_radius, K,
                                                                 static_cast<long long>(w.cap_starts));
  ARFX_CUDA(cudaGetLastError());
}

// K2 = K2a start masks -> scan -> K2b bone-major scatter -> K2c Newton -> K2d finalize
// (deform_starts.cuh). Counters: [4] item cursor, [6] total starts, [7] items.
// sort-key grid for ~`expect` live targets: the skinning cells coarsened until the key
// count is <= 3x the expected targets (full resolution for frames and occupancy grids)
KeyGrid key_grid(const SkinView& S, long long expect) {
  KeyGrid kg{};
  for (int sh = 0;; ++sh) {
    kg = KeyGrid{sh, ((S.rx - 2) >> sh) + 1, ((S.ry - 2) >> sh) + 1, ((S.rz - 2) >> sh) + 1};
    if (static_cast<long long>(S.nb) * kg.cells() <= 3 * std::max<long long>(expect, 1) || sh >= 5) return kg;
  }
}

template <class Src, class Sink>
void launch_deform_sink(ModelImpl& m, const PoseCtx* d_poses, const Src& src, const Sink& K, long long n_hint,
                        const char* name, cudaStream_t s, long long expect = -1) {
  Workspace& w = m.ws();
  constexpr bool single = Src::kSinglePose;
  const long long n = std::max<long long>(n_hint, 1);
  // items pack (target, bone) as target | bone << kItemBoneShift
  if (n >= (1LL << kItemBoneShift))
    throw std::invalid_argument("deformer: more than 2^26 posed points in one call (split the batch / frame)");
  // the batched inverse_lbs API runs asynchronously and cannot re-run: size its start slots
  // for the worst case (every bone survives pruning); render/occupancy learn from overflow
  const size_t worst = std::is_same<Sink, RootsSink>::value ? static_cast<size_t>(n) * m.sv.nb : 0;
  const KeyGrid kg = key_grid(m.sv, expect >= 0 ? expect : n);
  w.ensure_starts(static_cast<size_t>(n), static_cast<size_t>(m.sv.nb) * kg.cells(), worst);
  const size_t pose_smem = single ? (sizeof(PoseCtx) + 7) / 8 * 8 : 0;
  unsigned long long* C = w.counters.ptr;
  unsigned long long* stats = m.stats_on ? m.stats.ptr : nullptr;
  const long long nkeys = static_cast<long long>(m.sv.nb) * kg.cells();
  const long long cap = static_cast<long long>(w.cap_starts);
  m.prof.begin("prune", s);
  // K2a also resets the call's counters, key histogram and scan status (PruneResets)
  const PruneResets z{C, w.key_hist.ptr, nkeys, w.lb_status.ptr,
                      (n + kLbTile - 1) / kLbTile + (nkeys + kLbTile - 1) / kLbTile + 4};
  start_mask_kernel<Src, single><<<resident_grid(start_mask_kernel<Src, single>, 256, pose_smem, n), 256, pose_smem,
                                   s>>>(d_poses, src, w.smask.ptr, w.scount.ptr, stats, z);
  ARFX_CUDA(cudaGetLastError());
  // start slots: exclusive scan of the per-target start counts (C6 = total starts, C3 += 1
  // when they exceed the slots), single pass
  const long long tiles_t = (n + kLbTile - 1) / kLbTile, tiles_k = (nkeys + kLbTile - 1) / kLbTile;
  unsigned long long* st_t = w.lb_status.ptr;                // [ticket | tiles_t]
  unsigned long long* st_k = w.lb_status.ptr + tiles_t + 2;  // [ticket | tiles_k]
  scan_lookback_kernel<<<persistent_grid(scan_lookback_kernel, kLbThreads, 0, n / kLbItems + 1), kLbThreads, 0, s>>>(
      w.scount.ptr, C + 5, st_t, C + 6, static_cast<unsigned long long>(cap), C + 3);
  // counting sort of the starts by (bone, skinning cell of x0)
  start_key_kernel<Src, single><<<resident_grid(start_key_kernel<Src, single>, 256, pose_smem, n), 256, pose_smem,
                                  s>>>(
      m.sv, kg, d_poses, src, w.smask.ptr, w.scount.ptr, w.keys.ptr, w.unsorted.ptr, w.key_hist.ptr, cap);
  scan_lookback_kernel<<<persistent_grid(scan_lookback_kernel, kLbThreads, 0, nkeys / kLbItems + 1), kLbThreads, 0,
                         s>>>(w.key_hist.ptr, C + 8, st_k, C + 9);
  start_place_kernel<<<grid_for(2 * n, 256, 8), 256, 0, s>>>(C + 6, w.keys.ptr, w.unsorted.ptr, w.key_hist.ptr,
                                                            w.items.ptr, cap);
  ARFX_CUDA(cudaGetLastError());
  m.prof.end(s);
  // per-thread union-bone scratch: the widest cell union (build_cell_table), not n_bones
  const size_t smem = (ARFX_NEWTON_POSE_SMEM ? pose_smem : 0) +
                      static_cast<size_t>(m.max_union) * kDsThreads * sizeof(double);
  auto kern = stats ? start_newton_kernel<Src, single, true> : start_newton_kernel<Src, single, false>;
  const int grid = persistent_grid(kern, kDsThreads, smem, 2 * n);
  m.prof.begin(name, s);
  kern<<<grid, kDsThreads, smem, s>>>(m.sv, d_poses, m.inv, src, w.items.ptr, C + 6, w.smask.ptr, w.scount.ptr,
                                      w.res4.ptr, C + 4, stats,
                                      static_cast<long long>(w.cap_starts), (expect >= 0 ? expect : n) < kBlockQueueMaxTargets);
  ARFX_CUDA(cudaGetLastError());
  m.prof.end(s);
  m.prof.begin("finalize", s);
  launch_finalize(m, src, K, n, s);
  m.prof.end(s);
}

// K2 feeding the root pool.
template <class Src>
void launch_deform(ModelImpl& m, const PoseCtx* d_poses, const Src& src, long long n_hint,
                   cudaStream_t s, long long expect = -1) {
  Workspace& w = m.ws();
  PoolSink K{w.snroot.ptr, w.sbase.ptr, w.px.ptr, w.py.ptr, w.pz.ptr, w.powner.ptr,
             w.counters.ptr, static_cast<long long>(w.cap_pool), m.fv};
  launch_deform_sink(m, d_poses, src, K, n_hint, "deform", s, expect);
}

// allow_tc: the render may use the tcgen05 decoder (arfx_model_set_mlp_mode); occupancy
// grids, training and the query APIs always use the exact f32 MLP so their integer
// decisions (masks, root selection feeding gradients) stay reference-exact.
void launch_field_pool(ModelImpl& m, cudaStream_t s, long long n_hint, bool allow_tc = false,
                       float* act = nullptr) {
  m.wait_params(s);
  if (allow_tc && m.mlp_mode >= 1 && field_tc_supported(m.fv)) {
    launch_field_tc(m, s, n_hint);
    return;
  }
  if (field_is_standard_host(m.fv)) {
    const size_t smem = field_tile_smem(m.fv);
    auto kern = field_tile_kernel<16, 64>;
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), kFieldTile, smem);
    const long long tiles = (n_hint + kFieldTile - 1) / kFieldTile;
    const int grid = static_cast<int>(std::max(1LL, std::min(tiles, static_cast<long long>(sm_count()) *
                                                                        std::max(per_sm, 1))));
    // the query count is only known on the device: both kernels are launched and exactly one
    // of them runs, by the count (teams below kTeamMax queries, tiles above)
    constexpr long long kTeamMax = kTeamMaxQueries;
    m.prof.begin("field", s);
    // persistent: exactly the resident blocks (static smem allows ~6 per SM), so no block
    // waits for a second wave with a full share of the work
    const int team_per_sm = blocks_per_sm(reinterpret_cast<const void*>(field_team_kernel), kFtTeam * kFtTeams, 0);
    field_team_kernel<<<static_cast<unsigned>(sm_count() * team_per_sm), kFtTeam * kFtTeams, 0, s>>>(
        m.fv, m.ws().px.ptr, m.ws().py.ptr, m.ws().pz.ptr, m.ws().powner.ptr, m.ws().pres.ptr, m.ws().counters.ptr + 2,
        static_cast<long long>(m.ws().cap_pool), m.stats_on ? m.stats.ptr : nullptr, kTeamMax, act);
    kern<<<grid, kFieldTile, smem, s>>>(m.fv, m.ws().px.ptr, m.ws().py.ptr, m.ws().pz.ptr, m.ws().powner.ptr,
                                         m.ws().pres.ptr, m.ws().counters.ptr + 2,
                                         static_cast<long long>(m.ws().cap_pool), m.stats_on ? m.stats.ptr : nullptr,
                                         kTeamMax);
    ARFX_CUDA(cudaGetLastError());
    m.prof.end(s);
    return;
  }
  const int threads = 128;
  const size_t wbytes = static_cast<size_t>(m.fv.n_mlp) * sizeof(float);
  const int in_smem = wbytes <= 48 * 1024 ? 1 : 0;
  m.prof.begin("field", s);
  field_pool_kernel<<<grid_for(n_hint, threads, 16), threads, in_smem ? wbytes : 0, s>>>(
      m.fv, m.ws().px.ptr, m.ws().py.ptr, m.ws().pz.ptr, m.ws().powner.ptr, m.ws().pres.ptr,
      m.ws().counters.ptr + 2, static_cast<long long>(m.ws().cap_pool), in_smem);
  ARFX_CUDA(cudaGetLastError());
  m.prof.end(s);
}

}  // namespace

void Workspace::ensure_starts(size_t targets, size_t nkeys, size_t min_starts) {
  if (targets > cap_targets) {
    smask.alloc(targets);
    scount.alloc(targets);
    cap_targets = targets;
  }
  key_hist.ensure(nkeys);
  lb_status.ensure(cap_targets / kLbTile + nkeys / kLbTile + 8);
  // starts per target: mean ~2 on the body, 0 for most occupancy cells; overflow -> regrow
  const size_t want = std::max<size_t>({targets * 5 / 2, static_cast<size_t>(1) << 16, min_starts, learned_starts});
  if (want > cap_starts) {
    items.alloc(want);
    keys.alloc(want);
    unsorted.alloc(want);
    res4.alloc(want + 1);
    cap_starts = want;
  }
}

// Worst-case reservation for a call that must not synchronise with the host: `targets`
// posed points can produce at most kMaxRoots pool entries and n_bones starts each.
void Workspace::reserve_worst(size_t targets, size_t n_bones) {
  ensure(std::max(targets, cap_posed), 0);
  const size_t pool = targets * kMaxRoots + 1024;
  if (pool > cap_pool) {
    px.alloc(pool);
    py.alloc(pool);
    pz.alloc(pool);
    powner.alloc(pool);
    pres.alloc(pool);
    cap_pool = pool;
  }
  learned_starts = std::max(learned_starts, targets * n_bones + 1024);
}

void Workspace::ensure(size_t posed, size_t pix) {
  if (posed > cap_posed) {
    const size_t c = posed;
    sx.alloc(c);
    sy.alloc(c);
    sz.alloc(c);
    sdelta.alloc(c);
    sray.alloc(c);
    sidx.alloc(c);
    snroot.alloc(c);
    sbase.alloc(c);
    ssel.alloc(c);
    cap_posed = c;
    // root pool: in-box roots, ~0.6 per posed sample in practice (<= 8); overflow -> regrow
    const size_t pc = c + c / 2 + 1024;
    px.alloc(pc);
    py.alloc(pc);
    pz.alloc(pc);
    powner.alloc(pc);
    pres.alloc(pc);
    cap_pool = pc;
  }
  if (pix > n_pix) {
    ray_first.alloc(pix);
    ray_count.alloc(pix);
    n_pix = pix;
  }
  if (!counters.ptr) counters.alloc(16);
}

void render_frame(ModelImpl& m, PoseImpl& p, const HostCamera& cam, OccImpl* occ, int N,
                  bool stratified, double eps, uint64_t seed, uint64_t frame, int shard,
                  int nshards, float* d_rgb, float* d_alpha, unsigned long long* d_counters,
                  cudaStream_t s) {
  Workspace& w = m.ws();
  // rows of this shard: interleaved kRowTile-row tiles
  if (w.last_shard != shard || w.last_nshards != nshards || w.last_rows != cam.height ||
      w.last_w != cam.width) {
    std::vector<int32_t> rows;
    for (int y = 0; y < cam.height; ++y)
      if ((y / kRowTile) % nshards == shard) rows.push_back(y);
    w.row_list.alloc(rows.size() + 1);
    if (!rows.empty())
      ARFX_CUDA(cudaMemcpyAsync(w.row_list.ptr, rows.data(), rows.size() * sizeof(int32_t),
                                cudaMemcpyHostToDevice, s));
    ARFX_CUDA(cudaStreamSynchronize(s));
    w.last_shard = shard;
    w.last_nshards = nshards;
    w.last_rows = cam.height;
    w.last_w = cam.width;
    w.n_rows = static_cast<int>(rows.size());
  }
  const int n_rows = w.n_rows;
  const long long n_rays = static_cast<long long>(n_rows) * cam.width;
  // grow-only; overflow beyond this is detected from the counters and the frame re-run
  w.ensure(static_cast<size_t>(std::max<long long>(std::min<long long>(n_rays * std::max(N, 1), 1LL << 22),
                                                   1LL << 16)),
           static_cast<size_t>(cam.width) * cam.height);
  ARFX_CUDA(cudaMemsetAsync(w.counters.ptr, 0, 16 * sizeof(unsigned long long), s));

  MarchArgs A{};
  A.stats = m.stats_on ? m.stats.ptr : nullptr;
  A.cam = CameraView{cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, {}};
  for (int k = 0; k < 12; ++k) A.cam.ext[k] = cam.ext[k];
  A.pose = p.dev.ptr;
  A.nlo[0] = m.norm.lo.x;
  A.nlo[1] = m.norm.lo.y;
  A.nlo[2] = m.norm.lo.z;
  A.nhi[0] = m.norm.hi.x;
  A.nhi[1] = m.norm.hi.y;
  A.nhi[2] = m.norm.hi.z;
  A.has_occ = occ != nullptr;
  if (occ) {
    A.occ = occ->view();
    A.occ_box = launch_occ_bbox(w, A.occ, s);
    A.occ_bits = ARFX_MARCH_BITS ? w.occ_bits.ptr : nullptr;
  }
  A.N = N;
  A.stratified = stratified;
  A.seed = seed;
  A.frame = frame;
  A.rows = w.row_list.ptr;
  A.n_rows = n_rows;
  A.W = cam.width;
  A.sx = w.sx.ptr;
  A.sy = w.sy.ptr;
  A.sz = w.sz.ptr;
  A.sdelta = w.sdelta.ptr;
  A.sray = w.sray.ptr;
  A.sidx = w.sidx.ptr;
  A.ray_first = w.ray_first.ptr;
  A.ray_count = w.ray_count.ptr;
  A.counters = w.counters.ptr;
  A.cap = static_cast<long long>(w.cap_posed);
  if (n_rays > 0) {
    A.rpw = static_cast<int>(std::min<long long>(
        32, std::max<long long>(1, (n_rays + sm_count() * 4LL * kMarchWarps - 1) / (sm_count() * 4LL * kMarchWarps))));
    const long long groups = (n_rays + kMarchWarps * A.rpw - 1) / (kMarchWarps * A.rpw);
    const size_t smem = static_cast<size_t>(kMarchWarps) * 32 * ((A.N + 31) / 32) * sizeof(unsigned);
    // exactly one wave of resident blocks (a second partial wave cost 7 % of the kernel)
    const int grid = static_cast<int>(std::min<long long>(
        groups, static_cast<long long>(sm_count()) *
                    std::max(1, blocks_per_sm(reinterpret_cast<const void*>(march_kernel), kMarchWarps * 32, smem))));
    m.prof.begin("march", s);
    march_kernel<<<grid, kMarchWarps * 32, smem, s>>>(A);
    ARFX_CUDA(cudaGetLastError());
    m.prof.end(s);
  }
  ListSrc src{w.sx.ptr, w.sy.ptr, w.sz.ptr, w.counters.ptr, 0, static_cast<long long>(w.cap_posed)};
  launch_deform(m, p.dev.ptr, src, static_cast<long long>(w.cap_posed), s);
  launch_field_pool(m, s, static_cast<long long>(w.cap_pool), /*allow_tc=*/true);
  CompositeArgs C{w.row_list.ptr, n_rows, cam.width, w.ray_first.ptr, w.ray_count.ptr, w.sdelta.ptr,
                  w.snroot.ptr, w.sbase.ptr, w.pres.ptr, w.ssel.ptr, eps, d_rgb, d_alpha};
  if (n_rays > 0) {
    m.prof.begin("composite", s);
    composite_kernel<<<resident_grid(composite_kernel, 128, 0, n_rays), 128, 0, s>>>(C);
    ARFX_CUDA(cudaGetLastError());
    m.prof.end(s);
  }
  finalize_counters_kernel<<<1, 1, 0, s>>>(w.counters.ptr, static_cast<long long>(w.cap_posed));
  if (d_counters)
    ARFX_CUDA(cudaMemcpyAsync(d_counters, w.counters.ptr, 4 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToDevice, s));
}

// Training forward (K1 in ray-list mode, K2, K3) for n_rays pixels (d_px, d_py on device);
// the composite forward+backward and the field backward follow in train.cu.
void train_forward(ModelImpl& m, PoseImpl& p, const HostCamera& cam, OccImpl* occ, int N, bool stratified,
                   uint64_t seed, uint64_t frame, long long n_rays, const int32_t* d_px, const int32_t* d_py,
                   cudaStream_t s) {
  Workspace& w = m.ws();
  w.ensure(static_cast<size_t>(std::max<long long>(std::min<long long>(n_rays * std::max(N, 1), 1LL << 22), 1LL << 16)),
           static_cast<size_t>(std::max<long long>(n_rays, 1)));
  ARFX_CUDA(cudaMemsetAsync(w.counters.ptr, 0, 16 * sizeof(unsigned long long), s));
  MarchArgs A{};
  A.stats = m.stats_on ? m.stats.ptr : nullptr;
  A.cam = CameraView{cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, {}};
  for (int k = 0; k < 12; ++k) A.cam.ext[k] = cam.ext[k];
  A.pose = p.dev.ptr;
  A.nlo[0] = m.norm.lo.x;
  A.nlo[1] = m.norm.lo.y;
  A.nlo[2] = m.norm.lo.z;
  A.nhi[0] = m.norm.hi.x;
  A.nhi[1] = m.norm.hi.y;
  A.nhi[2] = m.norm.hi.z;
  A.has_occ = occ != nullptr;
  if (occ) {
    A.occ = occ->view();
    // (no occupied-box range here: random training rays gain nothing from it)
  }
  A.N = N;
  A.stratified = stratified;
  A.seed = seed;
  A.frame = frame;
  A.W = cam.width;
  A.lpx = d_px;
  A.lpy = d_py;
  A.n_list = n_rays;
  A.sx = w.sx.ptr;
  A.sy = w.sy.ptr;
  A.sz = w.sz.ptr;
  A.sdelta = w.sdelta.ptr;
  A.sray = w.sray.ptr;
  A.sidx = w.sidx.ptr;
  A.ray_first = w.ray_first.ptr;
  A.ray_count = w.ray_count.ptr;
  A.counters = w.counters.ptr;
  A.cap = static_cast<long long>(w.cap_posed);
  if (n_rays > 0) {
    A.rpw = static_cast<int>(std::min<long long>(
        32, std::max<long long>(1, (n_rays + sm_count() * 4LL * kMarchWarps - 1) / (sm_count() * 4LL * kMarchWarps))));
    const long long groups = (n_rays + kMarchWarps * A.rpw - 1) / (kMarchWarps * A.rpw);
    const size_t smem = static_cast<size_t>(kMarchWarps) * 32 * ((A.N + 31) / 32) * sizeof(unsigned);
    // exactly one wave of resident blocks (a second partial wave cost 7 % of the kernel)
    const int grid = static_cast<int>(std::min<long long>(
        groups, static_cast<long long>(sm_count()) *
                    std::max(1, blocks_per_sm(reinterpret_cast<const void*>(march_kernel), kMarchWarps * 32, smem))));
    m.prof.begin("march", s);
    march_kernel<<<grid, kMarchWarps * 32, smem, s>>>(A);
    ARFX_CUDA(cudaGetLastError());
    m.prof.end(s);
  }
  ListSrc src{w.sx.ptr, w.sy.ptr, w.sz.ptr, w.counters.ptr, 0, static_cast<long long>(w.cap_posed)};
  // training rays: ~13 posed samples per ray size the sort keys
  launch_deform(m, p.dev.ptr, src, static_cast<long long>(w.cap_posed), s, 16LL * n_rays);
  w.fwd_act.ensure(static_cast<size_t>(kTeamMaxQueries) * kActStride);
  launch_field_pool(m, s, static_cast<long long>(w.cap_pool), false, ARFX_SAVE_ACT ? w.fwd_act.ptr : nullptr);
  finalize_counters_kernel<<<1, 1, 0, s>>>(w.counters.ptr, static_cast<long long>(w.cap_posed));
}

void Workspace::ensure_train() {
  if (strans.n < cap_posed) strans.alloc(cap_posed);
  if (pgs.n < cap_pool) {
    pgs.alloc(cap_pool);
    pgc.alloc(3 * cap_pool);
    pflag.alloc(cap_pool);
  }
}

OccView OccImpl::view() const {
  OccView v{};
  v.rx = v.ry = v.rz = res;
  v.lo[0] = box.lo.x;
  v.lo[1] = box.lo.y;
  v.lo[2] = box.lo.z;
  v.hi[0] = box.hi.x;
  v.hi[1] = box.hi.y;
  v.hi[2] = box.hi.z;
  v.e[0] = box.hi.x - box.lo.x;
  v.e[1] = box.hi.y - box.lo.y;
  v.e[2] = box.hi.z - box.lo.z;
  for (int a = 0; a < 3; ++a) v.inv_e[a] = 1.0 / v.e[a];
  v.mask = mask.ptr;
  return v;
}

void occ_query_batch(OccImpl& g, const double* d_pts, int64_t n, uint8_t* d_out, cudaStream_t s) {
  if (n <= 0) return;
  occ_query_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(g.view(), d_pts, n, d_out);
  ARFX_CUDA(cudaGetLastError());
}

void occ_rebuild(OccImpl& g, cudaStream_t s) {
  const long long n = static_cast<long long>(g.res) * g.res * g.res;
  occ_rebuild_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(g.res, g.res, g.res, std::max(g.dilation, 0), g.values.ptr,
                                                        static_cast<float>(g.threshold), g.mask.ptr);
  ARFX_CUDA(cudaGetLastError());
}

static void occ_source_common(OccImpl& g, double lo[3], double cs[3]) {
  lo[0] = g.box.lo.x;
  lo[1] = g.box.lo.y;
  lo[2] = g.box.lo.z;
  // cell_size  R/occupancy.hpp:49-52
  cs[0] = (g.box.hi.x - g.box.lo.x) / g.res;
  cs[1] = (g.box.hi.y - g.box.lo.y) / g.res;
  cs[2] = (g.box.hi.z - g.box.lo.z) / g.res;
}

void inference_grid(ModelImpl& m, PoseImpl& p, OccImpl& g, unsigned long long* d_counters,
                    cudaStream_t s) {
  Workspace& w = m.ws();
  const long long n = static_cast<long long>(g.res) * g.res * g.res;
  w.ensure(static_cast<size_t>(n), 0);
  ARFX_CUDA(cudaMemsetAsync(w.counters.ptr, 0, 16 * sizeof(unsigned long long), s));
  CellSrc src{g.res, g.res, g.res, {}, {}};
  occ_source_common(g, src.lo, src.cs);
  launch_deform(m, p.dev.ptr, src, n, s);
  launch_field_pool(m, s, n);
  m.prof.begin("occ_values+mask", s);
  occ_values_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, w.snroot.ptr, w.sbase.ptr, w.pres.ptr,
                                                       g.values.ptr, 1.0f, 0);
  ARFX_CUDA(cudaGetLastError());
  occ_rebuild(g, s);
  m.prof.end(s);
  if (d_counters)
    ARFX_CUDA(cudaMemcpyAsync(d_counters, w.counters.ptr, 4 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToDevice, s));
}

// Cell-interleaved shard of the inference grid (multi-GPU): shard s of n
// computes the cells c = s + n*j, j < cells/n, into values[s*cells/n + j] (rank-major shard
// blocks, so an in-place all-gather of the blocks assembles the grid); occ_unshard then
// permutes the blocks into cell order before the mask rebuild. Interleaving balances the
// ranks (the body is thin in normalized z: contiguous z-slabs left most ranks idle).
// Bit-identical per cell to the full build.
void inference_grid_shard(ModelImpl& m, PoseImpl& p, OccImpl& g, int shard, int n_shards,
                          unsigned long long* d_counters, cudaStream_t s) {
  Workspace& w = m.ws();
  const long long cells = static_cast<long long>(g.res) * g.res * g.res;
  if (cells % n_shards != 0)
    throw std::invalid_argument("build_inference_grid_shard: the cell count must divide by n_shards");
  const long long n = cells / n_shards;
  w.ensure(static_cast<size_t>(std::max<long long>(n, 1)), 0);
  ARFX_CUDA(cudaMemsetAsync(w.counters.ptr, 0, 16 * sizeof(unsigned long long), s));
  if (n > 0) {
    CellSrc src{g.res, g.res, g.res, {}, {}, shard, n_shards};
    occ_source_common(g, src.lo, src.cs);
    launch_deform(m, p.dev.ptr, src, n, s);
    launch_field_pool(m, s, n);
    m.prof.begin("occ_values+mask", s);
    occ_values_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, w.snroot.ptr, w.sbase.ptr, w.pres.ptr,
                                                         g.values.ptr + n * shard, 1.0f, 0);
    ARFX_CUDA(cudaGetLastError());
    m.prof.end(s);
  }
  if (d_counters)
    ARFX_CUDA(cudaMemcpyAsync(d_counters, w.counters.ptr, 4 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToDevice, s));
}

__global__ void occ_unshard_kernel(const float* __restrict__ blocks, float* __restrict__ out, long long cells,
                                   int n_shards) {
  const long long per = cells / n_shards;
  for (long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; c < cells;
       c += static_cast<long long>(gridDim.x) * blockDim.x)
    out[c] = blocks[(c % n_shards) * per + c / n_shards];
}

// rank-major shard blocks (after the all-gather) -> cell order, in place via the grid's
// scratch buffer
void occ_unshard(OccImpl& g, int n_shards, cudaStream_t s) {
  if (n_shards <= 1) return;
  const long long cells = static_cast<long long>(g.res) * g.res * g.res;
  if (cells % n_shards != 0) throw std::invalid_argument("occ_unshard: the cell count must divide by n_shards");
  g.saved.ensure(static_cast<size_t>(cells));
  occ_unshard_kernel<<<grid_for(cells, 256, 8), 256, 0, s>>>(g.values.ptr, g.saved.ptr, cells, n_shards);
  ARFX_CUDA(cudaGetLastError());
  ARFX_CUDA(cudaMemcpyAsync(g.values.ptr, g.saved.ptr, static_cast<size_t>(cells) * sizeof(float),
                            cudaMemcpyDeviceToDevice, s));
}

void training_grid_update(ModelImpl& m, const std::vector<PoseImpl*>& poses, double decay,
                          uint64_t seed, uint64_t step, OccImpl& g, unsigned long long* d_counters,
                          cudaStream_t s) {
  Workspace& w = m.ws();
  const long long n = static_cast<long long>(g.res) * g.res * g.res;
  w.ensure(static_cast<size_t>(n), 0);
  DevBuf<PoseCtx>& ctxs = m.grid_ctxs;  // persistent: no allocation (device sync) per update
  ctxs.ensure(poses.size());
  for (size_t i = 0; i < poses.size(); ++i)
    ARFX_CUDA(cudaMemcpyAsync(ctxs.ptr + i, poses[i]->dev.ptr, sizeof(PoseCtx), cudaMemcpyDeviceToDevice, s));
  ARFX_CUDA(cudaMemsetAsync(w.counters.ptr, 0, 16 * sizeof(unsigned long long), s));
  JitterSrc src{g.res, g.res, g.res, static_cast<int>(poses.size()), {}, {}, seed, step};
  occ_source_common(g, src.lo, src.cs);
  launch_deform(m, ctxs.ptr, src, n, s);
  launch_field_pool(m, s, n);
  occ_values_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, w.snroot.ptr, w.sbase.ptr, w.pres.ptr,
                                                       g.values.ptr, static_cast<float>(decay), 1);
  ARFX_CUDA(cudaGetLastError());
  occ_rebuild(g, s);
  if (d_counters)
    ARFX_CUDA(cudaMemcpyAsync(d_counters, w.counters.ptr, 4 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToDevice, s));
}

void inverse_lbs_batch(ModelImpl& m, const PoseCtx* d_ctx, const double* d_pts, int64_t n,
                       int32_t* d_counts, double* d_roots, double* d_res, cudaStream_t s) {
  if (n <= 0) return;
  if (!m.ws().counters.ptr) m.ws().counters.alloc(16);
  const AosSrc src{d_pts, n};
  const RootsSink K{d_counts, d_roots, d_res};
  launch_deform_sink(m, d_ctx, src, K, n, "inverse_lbs", s);
}

void posed_query_batch(ModelImpl& m, PoseImpl& p, const double* d_pts, int64_t n, float* d_dens,
                       float* d_col, double* d_canon, uint8_t* d_has, unsigned long long* d_counters,
                       cudaStream_t s) {
  if (n <= 0) return;
  Workspace& w = m.ws();
  w.ensure(static_cast<size_t>(n), 0);
  ARFX_CUDA(cudaMemsetAsync(w.counters.ptr, 0, 16 * sizeof(unsigned long long), s));
  ListSrc src{d_pts, d_pts, d_pts, nullptr, n, n};
  // ListSrc expects SoA; user batches are AoS -> split on device
  DevBuf<double> soa;
  soa.alloc(static_cast<size_t>(3 * n));
  std::vector<double> dummy;
  (void)dummy;
  // transpose AoS -> SoA with three strided 2D copies
  ARFX_CUDA(cudaMemcpy2DAsync(soa.ptr, sizeof(double), d_pts, 3 * sizeof(double), sizeof(double),
                              static_cast<size_t>(n), cudaMemcpyDeviceToDevice, s));
  ARFX_CUDA(cudaMemcpy2DAsync(soa.ptr + n, sizeof(double), d_pts + 1, 3 * sizeof(double), sizeof(double),
                              static_cast<size_t>(n), cudaMemcpyDeviceToDevice, s));
  ARFX_CUDA(cudaMemcpy2DAsync(soa.ptr + 2 * n, sizeof(double), d_pts + 2, 3 * sizeof(double),
                              sizeof(double), static_cast<size_t>(n), cudaMemcpyDeviceToDevice, s));
  src.x = soa.ptr;
  src.y = soa.ptr + n;
  src.z = soa.ptr + 2 * n;
  launch_deform(m, p.dev.ptr, src, n, s);
  launch_field_pool(m, s, n);
  posed_out_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, w.snroot.ptr, w.sbase.ptr, w.pres.ptr, w.px.ptr,
                                                       w.py.ptr, w.pz.ptr, d_dens, d_col, d_canon, d_has);
  ARFX_CUDA(cudaGetLastError());
  if (d_counters)
    ARFX_CUDA(cudaMemcpyAsync(d_counters, w.counters.ptr, 4 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToDevice, s));
  ARFX_CUDA(cudaStreamSynchronize(s));
}

void field_query_batch(ModelImpl& m, const double* d_pts, int64_t n, float4* d_out, int* d_domain_err,
                       cudaStream_t s) {
  if (n <= 0) return;
  field_query_kernel<<<grid_for(n, 128, 16), 128, 0, s>>>(m.fv, d_pts, n, d_out, d_domain_err);
  ARFX_CUDA(cudaGetLastError());
}

void hash_encode_batch(ModelImpl& m, const double* d_pts, int64_t n, float* d_feats, int* d_domain_err,
                       cudaStream_t s) {
  if (n <= 0) return;
  hash_encode_kernel<<<grid_for(n, 128, 16), 128, 0, s>>>(m.fv, d_pts, n, d_feats, d_domain_err);
  ARFX_CUDA(cudaGetLastError());
}

void skin_weights_batch(ModelImpl& m, const double* d_pts, int64_t n, double* d_w, cudaStream_t s) {
  if (n <= 0) return;
  skin_weights_kernel<<<grid_for(n, 128, 16), 128, 0, s>>>(m.sv, d_pts, n, d_w);
  ARFX_CUDA(cudaGetLastError());
}

}  // namespace arfx

namespace arfx {

cudaEvent_t KernelProfiler::take() {
  if (!free_events.empty()) {
    cudaEvent_t e = free_events.back();
    free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  ARFX_CUDA(cudaEventCreate(&e));
  return e;
}

void KernelProfiler::begin(const char* name, cudaStream_t s) {
  if (!on) return;
  Rec r{name, take(), take()};
  ARFX_CUDA(cudaEventRecord(r.a, s));
  pending.push_back(r);
}

void KernelProfiler::end(cudaStream_t s) {
  if (!on || pending.empty()) return;
  ARFX_CUDA(cudaEventRecord(pending.back().b, s));
}

void KernelProfiler::collect() {
  for (Rec& r : pending) {
    ARFX_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    ARFX_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    size_t k = 0;
    while (k < names.size() && names[k] != r.name) ++k;
    if (k == names.size()) {
      names.emplace_back(r.name);
      ms.push_back(0.0);
      launches.push_back(0);
    }
    ms[k] += t;
    launches[k] += 1;
    free_events.push_back(r.a);
    free_events.push_back(r.b);
  }
  pending.clear();
}

KernelProfiler::~KernelProfiler() {
  for (Rec& r : pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : free_events) cudaEventDestroy(e);
}

int blocks_per_sm(const void* kernel, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
  int dev = 0;
  ARFX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(kernel, dev, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  ARFX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  per_sm = per_sm > 0 ? per_sm : 1;
  cache.emplace(key, per_sm);
  return per_sm;
}

int device_sm_count() {
  static int n[64] = {};
  int dev = 0;
  ARFX_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) dev = 0;
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

void ensure_dyn_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  ARFX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = done[{kernel, dev}];
  if (bytes <= cur) return;
  ARFX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  cur = bytes;
}

// Training ray pixels of one step (the trainer's ray_batch on the device): draw 0 of
// keyed_rng(seed, 0x7a11, step, rank) picks the frame (host side); ray i takes draws 1 + 2i
// (px = next_below(W)) and 2 + 2i (py = next_below(H)) -- bit-identical to the host stream.
__global__ void train_rays_kernel(uint64_t seed, uint64_t step, uint64_t rank, long long n, uint32_t W, uint32_t H,
                                  int32_t* __restrict__ px, int32_t* __restrict__ py) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    Pcg32 g = keyed_rng(seed, 0x7a11u, step, rank);
    pcg_advance(g, static_cast<uint64_t>(1 + 2 * i));
    px[i] = static_cast<int32_t>(pcg_below(g, W));
    py[i] = static_cast<int32_t>(pcg_below(g, H));
  }
}

void launch_train_rays(uint64_t seed, uint64_t step, uint64_t rank, long long n, int W, int H, int32_t* px, int32_t* py,
                       cudaStream_t s) {
  if (n <= 0) return;
  train_rays_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(seed, step, rank, n, static_cast<uint32_t>(W),
                                                        static_cast<uint32_t>(H), px, py);
  ARFX_CUDA(cudaGetLastError());
}

// ---- L_density: occupancy-based regulariser (Eq. 12) ----------
// n points uniform in the normalized box, point i from keyed_rng(seed, 0xde45, step, i)
// (x, y, z draws); points in EMPTY cells of the occupancy grid are posed-queried (K2 + exact
// K3) and L_density = mean |sigma| over them (0 when none). Its gradient
// w_density * sign(sigma) / n_empty lands on the selected root's pool entry, and K8 runs
// query_backward there -- the same path as the photometric step.
namespace {
__global__ void density_points_kernel(OccView g, long long n, uint64_t seed, uint64_t step, double* __restrict__ x,
                                      double* __restrict__ y, double* __restrict__ z, uint8_t* __restrict__ empty) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    Pcg32 r = keyed_rng(seed, 0xDE45ull, step, static_cast<uint64_t>(i));
    const double u0 = pcg_double(r), u1 = pcg_double(r), u2 = pcg_double(r);
    const d3 p = make3(dadd(g.lo[0], dmul(g.e[0], u0)), dadd(g.lo[1], dmul(g.e[1], u1)),
                       dadd(g.lo[2], dmul(g.e[2], u2)));
    x[i] = p.x;
    y[i] = p.y;
    z[i] = p.z;
    empty[i] = occupied(g, p) ? 0 : 1;
  }
}

// one block, fixed order: out2 = (mean sigma over empty points with a root... / n_empty, n_empty),
// scale = w / n_empty for the flag pass
__global__ void __launch_bounds__(1024) density_reduce_kernel(long long n, const uint8_t* __restrict__ empty,
                                                             const uint8_t* __restrict__ snroot,
                                                             const int32_t* __restrict__ sbase,
                                                             const float4* __restrict__ pres, double w,
                                                             double* __restrict__ out2, float* __restrict__ scale) {
  __shared__ double ss[1024];
  __shared__ unsigned long long sc[1024];
  double a = 0.0;
  unsigned long long c = 0;
  for (long long i = threadIdx.x; i < n; i += 1024) {
    if (!empty[i]) continue;
    ++c;
    float4 v;
    if (select_root(snroot, sbase, pres, i, v) >= 0) a += fabs(static_cast<double>(v.x));
  }
  ss[threadIdx.x] = a;
  sc[threadIdx.x] = c;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      ss[threadIdx.x] += ss[threadIdx.x + o];
      sc[threadIdx.x] += sc[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double ne = static_cast<double>(sc[0]);
    out2[0] = sc[0] ? ss[0] / ne : 0.0;
    out2[1] = ne;
    *scale = sc[0] ? static_cast<float>(w / ne) : 0.0f;
  }
}

__global__ void density_flag_kernel(long long n, const uint8_t* __restrict__ empty, const uint8_t* __restrict__ snroot,
                                    const int32_t* __restrict__ sbase, const float4* __restrict__ pres,
                                    const float* __restrict__ scale, float* __restrict__ pgs, float* __restrict__ pgc,
                                    uint8_t* __restrict__ pflag) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (!empty[i]) continue;
    float4 v;
    const int sel = select_root(snroot, sbase, pres, i, v);
    if (sel < 0) continue;
    const long long p = sbase[i] + sel;
    // d|sigma|/dsigma = sign(sigma); sigma = softplus > 0 except underflow
    pgs[p] = v.x > 0.0f ? *scale : (v.x < 0.0f ? -*scale : 0.0f);
    pgc[3 * p + 0] = pgc[3 * p + 1] = pgc[3 * p + 2] = 0.0f;
    pflag[p] = 1;
  }
}
}  // namespace

// Forward half: points, occupancy test, posed query into the workspace pool. Returns with
// the counters on the device (the caller checks overflow and re-runs).
void density_forward(ModelImpl& m, PoseImpl& p, OccImpl& g, long long n, uint64_t seed, uint64_t step,
                     cudaStream_t s) {
  Workspace& w = m.ws();
  w.ensure(static_cast<size_t>(n), 0);
  w.dens_pts.ensure(static_cast<size_t>(3 * n));
  w.dens_empty.ensure(static_cast<size_t>(n));
  ARFX_CUDA(cudaMemsetAsync(w.counters.ptr, 0, 16 * sizeof(unsigned long long), s));
  double* x = w.dens_pts.ptr;
  density_points_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(g.view(), n, seed, step, x, x + n, x + 2 * n,
                                                             w.dens_empty.ptr);
  ARFX_CUDA(cudaGetLastError());
  // every point is queried (the occupancy test only decides which ones enter the loss): the
  // empty-cell fraction is ~90 %, and querying all keeps the pipeline branch-free
  ListSrc src{x, x + n, x + 2 * n, nullptr, n, n};
  launch_deform(m, p.dev.ptr, src, n, s);
  w.fwd_act.ensure(static_cast<size_t>(kTeamMaxQueries) * kActStride);
  launch_field_pool(m, s, n, false, ARFX_SAVE_ACT ? w.fwd_act.ptr : nullptr);
}

// Backward half, part 1: loss reduction and gradient flags (reads only the density
// forward's workspace; may run on the forward's stream).
void density_flags(ModelImpl& m, long long n, double w_density, double* d_out2, cudaStream_t s) {
  Workspace& w = m.ws();
  w.ensure_train();
  w.dens_scale.ensure(1);
  ARFX_CUDA(cudaMemsetAsync(w.pflag.ptr, 0, w.cap_pool, s));
  density_reduce_kernel<<<1, 1024, 0, s>>>(n, w.dens_empty.ptr, w.snroot.ptr, w.sbase.ptr, w.pres.ptr, w_density,
                                           d_out2, w.dens_scale.ptr);
  density_flag_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, w.dens_empty.ptr, w.snroot.ptr, w.sbase.ptr,
                                                          w.pres.ptr, w.dens_scale.ptr, w.pgs.ptr, w.pgc.ptr,
                                                          w.pflag.ptr);
  ARFX_CUDA(cudaGetLastError());
}

// Part 2: K8 into the model's gradients (ordered after every other gradient writer).
void density_backward_field(ModelImpl& m, long long n, cudaStream_t s) {
  Workspace& w = m.ws();
  const BwdOwners own{n, nullptr, nullptr, false};  // owner = density point = target
  field_backward_pool(m, w.counters.ptr + 2, static_cast<long long>(w.cap_pool), w.pflag.ptr, w.pgs.ptr, w.pgc.ptr,
                      s, &own, ARFX_SAVE_ACT ? w.fwd_act.ptr : nullptr);
}

void density_backward(ModelImpl& m, long long n, double w_density, double* d_out2, cudaStream_t s) {
  density_flags(m, n, w_density, d_out2, s);
  density_backward_field(m, n, s);
}

}  // namespace arfx
