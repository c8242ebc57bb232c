// deform_starts.cuh -- correspondence search (K2) as independent Newton starts, sm_100a.
//
// inverse_lbs_ctx (R/articulation.hpp:94-145) runs one damped-Newton solve per surviving
// start (bone) of a posed target x', then pushes the converged ones into InverseRoots in
// bone order (R/articulation.hpp:66-81). The solves are independent; only the push order
// couples them. So:
//
//  K2a start_mask_kernel  thread per target: surviving-start mask (f32 bounding-sphere
//                         reject + exact FP64 capsule distance) and start count.
//  (scan)                 exclusive prefix of the start counts -> start slot of each target.
//  K2b start_key/place    counting sort of the (target, bone) items by (bone, skinning cell
//                         of x0 = B_b^-1 x'): a warp's lanes start in the same cell rows, so
//                         the cell-table gathers broadcast in L1.
//  K2c start_newton       persistent warps over the items; per-lane state machine whose
//                         unit of progress is one skinning eval (lanes that converge early
//                         take a new item instead of idling); the Newton step is taken right
//                         after the eval that accepted x; result (root, residual or "no
//                         root") written as one double4 to the start's slot.
//  K2d finalize           thread per target: replays InverseRoots::push over its starts in
//                         bone order (bit-exact dedup / replacement / kMaxRoots), then the
//                         sink: in-box roots to the root pool (render / occupancy) or all
//                         roots to [n][8] (inverse_lbs API).
#pragma once

#include "deform.cuh"
#include "field.cuh"

namespace arfx {

#ifndef ARFX_DS_THREADS
#define ARFX_DS_THREADS 128
#endif
constexpr int kDsThreads = ARFX_DS_THREADS;
#ifndef ARFX_NEWTON_POSE_SMEM
#define ARFX_NEWTON_POSE_SMEM 1
#endif
#ifndef ARFX_DS_MIN_BLOCKS
#define ARFX_DS_MIN_BLOCKS 5
#endif
constexpr int kDsMinBlocks = ARFX_DS_MIN_BLOCKS;  // 5 x 128 threads: <= 102 registers
#ifndef ARFX_DS_ITEM_CHUNK
#define ARFX_DS_ITEM_CHUNK 64
#endif
constexpr int kDsItemChunk = ARFX_DS_ITEM_CHUNK;
constexpr long long kBlockQueueMaxTargets = 262144;  // block-local item queues below this
constexpr int kItemBoneShift = 26;  // item = target | bone << 26 (targets < 2^26)

enum DsState : int { DS_NEED = 0, DS_EVAL_INIT = 2, DS_EVAL_LS = 3, DS_DONE = 4 };

__device__ __forceinline__ unsigned ds_lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <bool kSinglePose>
__device__ __forceinline__ const PoseCtx* ds_stage_pose(const PoseCtx* poses, double* smem) {
  if (!kSinglePose) return poses;
  const int words = static_cast<int>(sizeof(PoseCtx) / 8);
  const double* g = reinterpret_cast<const double*>(poses);
  for (int i = threadIdx.x; i < words; i += blockDim.x) smem[i] = g[i];
  __syncthreads();
  return reinterpret_cast<const PoseCtx*>(smem);
}

// Packed f32x2 add / mul (sm_100 FADD2 / FMUL2) with explicit .rn rounding in PTX.
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
  unsigned long long r;
  asm("{\n\t.reg .b64 ra, rb;\n\tmov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\t"
      "add.rn.f32x2 %0, ra, rb;\n\t}"
      : "=l"(r)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return make_float2(__uint_as_float(static_cast<unsigned>(r)), __uint_as_float(static_cast<unsigned>(r >> 32)));
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  unsigned long long r;
  asm("{\n\t.reg .b64 ra, rb;\n\tmov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\t"
      "mul.rn.f32x2 %0, ra, rb;\n\t}"
      : "=l"(r)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return make_float2(__uint_as_float(static_cast<unsigned>(r)), __uint_as_float(static_cast<unsigned>(r >> 32)));
}

// Surviving starts: bit b set iff cap_dist(x', b) <= cutoff_b (R/articulation.hpp:101-102).
__device__ __forceinline__ uint32_t ds_prune(const PoseCtx* __restrict__ P, d3 xt, int& exact_tests) {
  const float fx = static_cast<float>(xt.x), fy = static_cast<float>(xt.y), fz = static_cast<float>(xt.z);
  // sphere rejects two bones at a time on the packed f32x2 pipe (FADD2 / FMUL2): the same
  // per-lane operations and roundings as the scalar ((dx^2 + dy^2) + dz^2) > r^2 test
  uint32_t cand = 0;
  const int nb = P->nb;
  const float2 fx2 = make_float2(fx, fx), fy2 = make_float2(fy, fy), fz2 = make_float2(fz, fz);
  for (int b = 0; b < nb; b += 2) {
    // PoseCtx::sph rows are 8-byte aligned: two float2 loads per bone
    const float2 a0 = *reinterpret_cast<const float2*>(&P->sph[b][0]), a1 = *reinterpret_cast<const float2*>(&P->sph[b][2]);
    const bool two = b + 1 < nb;
    const float2 c0 = two ? *reinterpret_cast<const float2*>(&P->sph[b + 1][0]) : make_float2(0.f, 0.f);
    const float2 c1 = two ? *reinterpret_cast<const float2*>(&P->sph[b + 1][2]) : make_float2(0.f, -1.f);
    const float2 dx = f2_add(fx2, make_float2(-a0.x, -c0.x));
    const float2 dy = f2_add(fy2, make_float2(-a0.y, -c0.y));
    const float2 dz = f2_add(fz2, make_float2(-a1.x, -c1.x));
    const float2 mx = f2_mul(dx, dx), my = f2_mul(dy, dy), mz = f2_mul(dz, dz);
    // the sums stay scalar add.rn: ptxas fuses a packed mul into a packed add (FFMA2) even
    // with -fmad=false, which would change the rounding; scalar .rn adds are never contracted
    const float2 d2 = make_float2(__fadd_rn(__fadd_rn(mx.x, my.x), mz.x), __fadd_rn(__fadd_rn(mx.y, my.y), mz.y));
    cand |= (d2.x > a1.y ? 0u : 1u) << b;  // else provably pruned (see PoseCtx::sph)
    cand |= (d2.y > c1.y ? 0u : 1u) << (b + 1);
  }
  uint32_t mask = 0;
  for (uint32_t m = cand; m; m &= m - 1) {
    const int b = __ffs(m) - 1;
    ++exact_tests;
    const d3 ca = make3(P->cap_a[b][0], P->cap_a[b][1], P->cap_a[b][2]);
    const d3 cb = make3(P->cap_b[b][0], P->cap_b[b][1], P->cap_b[b][2]);
    if (point_segment_distance(xt, ca, cb) > P->cutoff[b]) continue;
    mask |= 1u << b;
  }
  return mask;
}

// K2a. It also performs the deform call's per-call resets for the kernels after it (formerly a
// 1-thread count kernel and three memsets, i.e. four graph nodes on the critical path):
// C[4] (Newton cursor) = C[6] = C[7] = 0, C[5] = target count, C[8] = key count, the key
// histogram and the look-back scan status words zeroed. Nothing before the scans reads them.
struct PruneResets {
  unsigned long long* C;  // the workspace counters
  uint32_t* key_hist;
  long long nkeys;
  unsigned long long* lb_status;
  long long n_status;
};

template <class Src, bool kSinglePose>
__global__ void __launch_bounds__(256) start_mask_kernel(const PoseCtx* __restrict__ poses, Src src,
                                                         uint32_t* __restrict__ mask_out,
                                                         uint32_t* __restrict__ count_out,
                                                         unsigned long long* stats, PruneResets z) {
  {
    const long long t0 = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long nt = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = t0; i < z.nkeys; i += nt) z.key_hist[i] = 0u;
    for (long long i = t0; i < z.n_status; i += nt) z.lb_status[i] = 0ull;
    if (t0 == 0) {
      z.C[4] = 0ull;
      z.C[5] = static_cast<unsigned long long>(src.count());
      z.C[6] = 0ull;
      z.C[7] = 0ull;
      z.C[8] = static_cast<unsigned long long>(z.nkeys);
    }
  }
  extern __shared__ double sm_smem[];
  const PoseCtx* Pb = ds_stage_pose<kSinglePose>(poses, sm_smem);
  const int lane = threadIdx.x & 31;
  const long long n = src.count();
  int exact = 0;
  for (long long base = (static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
       base < n; base += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long s = base + lane;
    uint32_t mask = 0;
    if (s < n) {
      int pose;
      const d3 xt = src.point(s, pose);
      mask = ds_prune(kSinglePose ? Pb : Pb + pose, xt, exact);
      mask_out[s] = mask;
      count_out[s] = static_cast<uint32_t>(__popc(mask));
    }
  }
  if (stats) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) exact += __shfl_xor_sync(0xffffffffu, exact, o);
    if (lane == 0 && exact) atomicAdd(stats + 4, static_cast<unsigned long long>(exact));
  }
}

// Sort-key cell grid: the skinning cells coarsened by 2^shift per axis (small batches use a
// coarser key space so the key histogram / scan stay proportional to the work).
struct KeyGrid {
  int shift, cx, cy, cz;  // coarse dims
  __host__ __device__ int cells() const { return cx * cy * cz; }
};

// Approximate (f32) skinning cell of a point: only a sort key for locality, never used
// in the arithmetic (skin_eval recomputes the exact cell in FP64). sc = (res - 1) / extent
// per axis, computed once per thread (no division per start).
struct KeyScale {
  float lo[3], sc[3];
};
__device__ __forceinline__ KeyScale key_scale(const SkinView& S) {
  const int res[3] = {S.rx, S.ry, S.rz};
  KeyScale k;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    k.lo[a] = static_cast<float>(S.lo[a]);
    k.sc[a] = static_cast<float>(res[a] - 1) / static_cast<float>(S.e[a]);
  }
  return k;
}
__device__ __forceinline__ int approx_skin_cell(const SkinView& S, const KeyScale& ks, d3 x, const KeyGrid& kg) {
  const float p[3] = {static_cast<float>(x.x), static_cast<float>(x.y), static_cast<float>(x.z)};
  const int res[3] = {S.rx, S.ry, S.rz};
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float u = (p[a] - ks.lo[a]) * ks.sc[a];
    u = fminf(fmaxf(u, 0.0f), static_cast<float>(res[a] - 2));
    c[a] = static_cast<int>(u) >> kg.shift;
  }
  return (c[2] * kg.cy + c[1]) * kg.cx + c[0];
}

// K2b (counting sort by (bone, skinning cell of the start point x0 = B_b^-1 x')):
// pass 1 -- per target, per surviving bone: key, unsorted item, key histogram.
template <class Src, bool kSinglePose>
__global__ void __launch_bounds__(256) start_key_kernel(SkinView S, KeyGrid kg, const PoseCtx* __restrict__ poses,
                                                        Src src,
                                                        const uint32_t* __restrict__ mask_in,
                                                        const uint32_t* __restrict__ slot_base,
                                                        uint32_t* __restrict__ keys, uint32_t* __restrict__ unsorted,
                                                        uint32_t* __restrict__ key_hist, long long cap) {
  extern __shared__ double sk_smem[];
  const PoseCtx* Pb = ds_stage_pose<kSinglePose>(poses, sk_smem);
  const int ncell = kg.cells();
  const KeyScale ks = key_scale(S);
  const long long n = src.count();
  for (long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; s < n;
       s += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint32_t mask = mask_in[s];
    if (!mask) continue;
    int pose;
    const d3 xt = src.point(s, pose);
    const PoseCtx* P = kSinglePose ? Pb : Pb + pose;
    long long slot = slot_base[s];
    for (uint32_t m = mask; m; m &= m - 1, ++slot) {
      const int b = __ffs(m) - 1;
      const uint32_t key = static_cast<uint32_t>(b * ncell + approx_skin_cell(S, ks, rigid_apply(P->bone_inv[b], xt), kg));
      if (slot < cap) {
        keys[slot] = key;
        unsorted[slot] = static_cast<uint32_t>(s) | (static_cast<uint32_t>(b) << kItemBoneShift);
      }
      // warp-aggregated histogram: neighbouring targets' starts often share a key
      const unsigned act = __activemask();
      const unsigned grp = __match_any_sync(act, key);
      if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(grp) - 1)) atomicAdd(key_hist + key, static_cast<uint32_t>(__popc(grp)));
    }
  }
}

// pass 2 -- place each start at its key's next position (order within a key irrelevant)
__global__ void __launch_bounds__(256) start_place_kernel(const unsigned long long* n_starts,
                                                          const uint32_t* __restrict__ keys,
                                                          const uint32_t* __restrict__ unsorted,
                                                          uint32_t* __restrict__ key_cursor,
                                                          StartItem* __restrict__ items, long long cap) {
  long long n = static_cast<long long>(*n_starts);
  n = n < cap ? n : cap;
  const unsigned lane = threadIdx.x & 31;
  for (long long j0 = static_cast<long long>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); j0 < n;
       j0 += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long j = j0 + lane;
    const bool act = j < n;
    const uint32_t key = act ? keys[j] : 0xffffffffu;
    // warp-aggregated: starts of neighbouring targets often share (bone, cell); one atomic
    // per distinct key in the warp, ranks within the group by lane order
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(grp) - 1;
    uint32_t base = 0;
    if (act && static_cast<int>(lane) == leader) base = atomicAdd(key_cursor + key, static_cast<uint32_t>(__popc(grp)));
    base = __shfl_sync(0xffffffffu, base, leader);
    const uint32_t pos = base + __popc(grp & ((1u << lane) - 1u));
    if (act && pos < cap) {
#if ARFX_ITEMS64
      items[pos] = (static_cast<unsigned long long>(j) << 32) | unsorted[j];  // j is the start's slot
#else
      items[pos] = unsorted[j];
#endif
    }
  }
}

// K2c: Newton over the items. Result per start slot: root (x,y,z) and residual, or
// residual = -1 when the start did not converge (singular / stalled / max iterations).
template <class Src, bool kSinglePose, bool kStats>
__global__ void __launch_bounds__(kDsThreads, kDsMinBlocks) start_newton_kernel(SkinView S, const PoseCtx* __restrict__ poses,
                                                                  InverseOpts opt, Src src,
                                                                  const StartItem* __restrict__ items,
                                                                  const unsigned long long* n_items,
                                                                  const uint32_t* __restrict__ mask_in,
                                                                  const uint32_t* __restrict__ slot_base,
                                                                  double4* __restrict__ res,
                                                                  unsigned long long* cursor,
                                                                  unsigned long long* stats, long long cap,
                                                                  bool block_queue) {
  extern __shared__ double ds_smem[];
#if ARFX_NEWTON_POSE_SMEM
  const PoseCtx* Pbase = ds_stage_pose<kSinglePose>(poses, ds_smem);
  double* ws = ds_smem + (kSinglePose ? (sizeof(PoseCtx) + 7) / 8 : 0) + threadIdx.x;
#else
  // the PoseContext is read through L1 (one cached copy per SM) instead of a per-block smem
  // copy: smem per block is only the union-bone scratch, which leaves L1 more room for the
  // skinning cell table gathers
  const PoseCtx* Pbase = poses;
  double* ws = ds_smem + threadIdx.x;
#endif
  const int stride = blockDim.x;
  const int lane = threadIdx.x & 31;
  long long n = static_cast<long long>(*n_items);
  n = n < cap ? n : cap;  // on overflow the host regrows and re-runs the frame
  unsigned long long st_e = 0, st_u = 0, st_i = 0, st_s = 0;

  int state = DS_NEED;
  long long s = 0, slot = 0;
  int pose = 0, it = 0, h = 0;
  // loop-carried per-lane state only: the Newton step is taken eagerly right after the eval
  // that accepted x, so g and J (12 doubles) live within one trip; for DS_EVAL_INIT, x holds
  // the start point x0 until its eval completes
  d3 xt = make3(0, 0, 0), x = xt, step = xt;
  double gn = 0.0, damp = 1.0;
  long long q_next = 0, q_end = 0;  // warp-uniform item queue
  // refill granularity: up to kDsItemChunk items per atomic, smaller when the launch has few
  // items per warp (occupancy grids) so the work spreads over all warps instead of a few
  // block_queue (small launches): block b owns the contiguous slice [q_lo, q_hi) of the
  // sorted items and its warps take chunks from a shared-memory cursor (no global atomics;
  // measured +3 % on the 4,096-ray train step). Large launches keep the global cursor: a
  // static split by slice is unbalanced there (slices of different bones differ in cost;
  // 1.75 -> 2.59 ms on a frame).
  __shared__ unsigned long long bq;
  if (threadIdx.x == 0) bq = 0ull;
  __syncthreads();
  long long q_lo = 0;
  long long n_warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  long long chunk = max(1LL, min(static_cast<long long>(kDsItemChunk), n / (8 * n_warps)));
  if (block_queue) {
    q_lo = n * static_cast<long long>(blockIdx.x) / gridDim.x;
    const long long q_hi = n * (static_cast<long long>(blockIdx.x) + 1) / gridDim.x;
    n_warps = blockDim.x >> 5;
    chunk = max(1LL, min(static_cast<long long>(kDsItemChunk), (q_hi - q_lo) / (8 * n_warps)));
    n = q_hi;
  }

  while (true) {
    // ---- A: refill finished lanes from the warp's item queue ----
    {
      const bool need = state == DS_NEED;
      const unsigned nm = __ballot_sync(0xffffffffu, need);
      if (nm) {
        const int k = __popc(nm);
        const int r = __popc(nm & ds_lanemask_lt());
        const long long avail = q_end - q_next;
        long long id;
        if (avail >= k) {
          id = q_next + r;
          q_next += k;
        } else {
          long long base = 0;
          const long long take = max(chunk, static_cast<long long>(k) - avail);  // >= the lanes still short
          if (lane == 0)
            base = block_queue ? q_lo + static_cast<long long>(atomicAdd(&bq, static_cast<unsigned long long>(take)))
                               : static_cast<long long>(atomicAdd(cursor, static_cast<unsigned long long>(take)));
          base = __shfl_sync(0xffffffffu, base, 0);
          id = r < avail ? q_next + r : base + (r - avail);
          q_next = base + (k - avail);
          q_end = base + take;
        }
        if (need) {
          if (id >= n) {
            state = DS_DONE;
          } else {
            const StartItem it = items[id];
            const uint32_t item = static_cast<uint32_t>(it);
            s = item & ((1u << kItemBoneShift) - 1u);
            const int b = static_cast<int>(item >> kItemBoneShift);
#if ARFX_ITEMS64
            slot = static_cast<long long>(it >> 32);
#else
            slot = static_cast<long long>(slot_base[s]) + __popc(mask_in[s] & ((1u << b) - 1u));
#endif
            if (slot >= cap) slot = cap;  // overflow: scratch slot (result arrays hold cap + 1)
            xt = src.point(s, pose);
            x = rigid_apply((kSinglePose ? Pbase : Pbase + pose)->bone_inv[b], xt);  // x0
            state = DS_EVAL_INIT;
            if (kStats) ++st_s;
          }
        }
      }
    }
    if (__all_sync(0xffffffffu, state == DS_DONE)) break;

    // ---- B: one skinning eval per busy lane ----
    if (state == DS_EVAL_INIT || state == DS_EVAL_LS) {
      const d3 cand = state == DS_EVAL_INIT ? x : sub3(x, mul3(step, damp));
      d3 g;
      double gcn, Jn[9];
      const int nu = skin_eval(S, kSinglePose ? Pbase : Pbase + pose, cand, xt, ws, stride, g, gcn, Jn);
      if (kStats) {
        ++st_e;
        st_u += static_cast<unsigned long long>(nu);
      }
      // ---- C: Newton / line-search bookkeeping (R/articulation.hpp:104-142) ----
      bool iterate = false;
      if (state == DS_EVAL_INIT) {
        gn = gcn;
        if (gn < opt.tolerance) {
          res[slot] = make_double4(x.x, x.y, x.z, gn);
          state = DS_NEED;
        } else {
          it = 0;
          iterate = true;
        }
      } else if (gcn < gn || h == 3) {
        if (gcn >= gn && gn >= opt.tolerance) {
          res[slot] = make_double4(0.0, 0.0, 0.0, -1.0);  // stalled
          state = DS_NEED;
        } else {
          x = cand;
          gn = gcn;
          ++it;
          if (gn < opt.tolerance) {
            res[slot] = make_double4(x.x, x.y, x.z, gn);
            state = DS_NEED;
          } else {
            iterate = true;
          }
        }
      } else {
        damp = dmul(damp, 0.5);
        ++h;
      }
      if (iterate) {  // Newton step with the Jacobian of the accepted eval (R/math.hpp:141-158)
        bool fail = it >= opt.max_iterations;
        if (!fail) {
          const double J0 = Jn[0], J1 = Jn[1], J2 = Jn[2], J3 = Jn[3], J4 = Jn[4], J5 = Jn[5], J6 = Jn[6],
                       J7 = Jn[7], J8 = Jn[8];
          const double c0 = dsub(dmul(J4, J8), dmul(J5, J7));
          const double c1 = dsub(dmul(J3, J8), dmul(J5, J6));
          const double c2 = dsub(dmul(J3, J7), dmul(J4, J6));
          const double det = dadd(dsub(dmul(J0, c0), dmul(J1, c1)), dmul(J2, c2));
          if (fabs(det) < 2.2250738585072014e-308 * 64) {
            fail = true;  // singular: the start fails (R/articulation.hpp:114-118)
          } else {
            if (kStats) ++st_i;
            const double id = ddiv(1.0, det);
            const double i0 = dmul(c0, id);
            const double i1 = dmul(dsub(dmul(J2, J7), dmul(J1, J8)), id);
            const double i2 = dmul(dsub(dmul(J1, J5), dmul(J2, J4)), id);
            const double i3 = dmul(dsub(dmul(J5, J6), dmul(J3, J8)), id);
            const double i4 = dmul(dsub(dmul(J0, J8), dmul(J2, J6)), id);
            const double i5 = dmul(dsub(dmul(J2, J3), dmul(J0, J5)), id);
            const double i6 = dmul(c2, id);
            const double i7 = dmul(dsub(dmul(J1, J6), dmul(J0, J7)), id);
            const double i8 = dmul(dsub(dmul(J0, J4), dmul(J1, J3)), id);
            step = make3(dadd(dadd(dmul(i0, g.x), dmul(i1, g.y)), dmul(i2, g.z)),
                         dadd(dadd(dmul(i3, g.x), dmul(i4, g.y)), dmul(i5, g.z)),
                         dadd(dadd(dmul(i6, g.x), dmul(i7, g.y)), dmul(i8, g.z)));
            damp = 1.0;
            h = 0;
            state = DS_EVAL_LS;
          }
        }
        if (fail) {
          res[slot] = make_double4(0.0, 0.0, 0.0, -1.0);
          state = DS_NEED;
        }
      }
    }
  }
  if (kStats) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      st_e += __shfl_xor_sync(0xffffffffu, st_e, o);
      st_u += __shfl_xor_sync(0xffffffffu, st_u, o);
      st_i += __shfl_xor_sync(0xffffffffu, st_i, o);
      st_s += __shfl_xor_sync(0xffffffffu, st_s, o);
    }
    if (lane == 0) {
      atomicAdd(stats + 0, st_e);
      atomicAdd(stats + 1, st_u);
      atomicAdd(stats + 2, st_i);
      atomicAdd(stats + 3, st_s);
    }
  }
}

// ---- K2d finalize: InverseRoots::push replay + sink -----------------------------

struct PoolSink {  // render / occupancy: in-box roots (posed_query_ctx R/articulation.hpp:170-173)
  uint8_t* snroot;
  int32_t* sbase;
  double *px, *py, *pz;
  int32_t* powner;
  unsigned long long* counters;  // [1] canonical, [2] pool cursor, [3] overflow
  long long cap_pool;
  FieldView F;
};

struct RootsSink {  // batched inverse_lbs API: every root + residual, [n][8]
  int32_t* counts;
  double* roots;
  double* resid;
};

__device__ __forceinline__ void ds_gather_roots(long long s, const uint32_t* mask_in, const uint32_t* slot_base,
                                                const double4* res, double dedup, Roots& R, long long cap) {
  R.count = 0;
  const long long b0 = slot_base[s];
  const int c = static_cast<int>(min(static_cast<long long>(__popc(mask_in[s])), cap - b0));
  // the first four start results are loaded before any push (independent loads in flight;
  // most targets have <= 4 starts), the rest one at a time; pushes stay in bone order
  double4 v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (j < c) v[j] = res[b0 + j];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (j < c && v[j].w >= 0.0) roots_push(R, make3(v[j].x, v[j].y, v[j].z), v[j].w, dedup);
  for (int j = 4; j < c; ++j) {
    const double4 w = res[b0 + j];
    if (w.w < 0.0) continue;
    roots_push(R, make3(w.x, w.y, w.z), w.w, dedup);
  }
}

template <class Src>
__global__ void __launch_bounds__(256) finalize_pool_kernel(Src src, const uint32_t* __restrict__ mask_in,
                                                            const uint32_t* __restrict__ slot_base,
                                                            const double4* __restrict__ res, double dedup,
                                                            PoolSink K, long long cap) {
  const long long n = src.count();
  const int lane = threadIdx.x & 31;
  unsigned canon = 0;
  for (long long base = (static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
       base < n; base += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long s = base + lane;
    Roots R;
    R.count = 0;
    uint32_t inbox = 0;
    if (s < n) {
      ds_gather_roots(s, mask_in, slot_base, res, dedup, R, cap);
      for (int k = 0; k < R.count; ++k)
        if (field_contains(K.F, make3(R.x[k][0], R.x[k][1], R.x[k][2]))) inbox |= 1u << k;
    }
    const int need = __popc(inbox);
    int incl = need;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    long long pbase = 0;
    if (lane == 0 && total) pbase = static_cast<long long>(atomicAdd(K.counters + 2, static_cast<unsigned long long>(total)));
    pbase = __shfl_sync(0xffffffffu, pbase, 0);
    if (s < n) {
      K.snroot[s] = static_cast<uint8_t>(need);
      if (need == 0) {
        K.sbase[s] = -1;
      } else {
        ++canon;
        long long q = pbase + incl - need;
        K.sbase[s] = static_cast<int32_t>(q);
        if (q + need > K.cap_pool) {
          atomicAdd(K.counters + 3, 1ull);
        } else {
          for (uint32_t m = inbox; m; m &= m - 1, ++q) {
            const int k = __ffs(m) - 1;
            K.px[q] = R.x[k][0];
            K.py[q] = R.x[k][1];
            K.pz[q] = R.x[k][2];
            K.powner[q] = static_cast<int32_t>(s);
          }
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) canon += __shfl_xor_sync(0xffffffffu, canon, o);
  if (lane == 0 && canon) atomicAdd(K.counters + 1, static_cast<unsigned long long>(canon));
}

template <class Src>
__global__ void __launch_bounds__(256) finalize_roots_kernel(Src src, const uint32_t* __restrict__ mask_in,
                                                             const uint32_t* __restrict__ slot_base,
                                                             const double4* __restrict__ res, double dedup,
                                                             RootsSink K, long long cap) {
  const long long n = src.count();
  for (long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; s < n;
       s += static_cast<long long>(gridDim.x) * blockDim.x) {
    Roots R;
    ds_gather_roots(s, mask_in, slot_base, res, dedup, R, cap);
    K.counts[s] = R.count;
    // unused slots are zero, as the reference's value-initialised InverseRoots arrays
    for (int k = 0; k < kMaxRoots; ++k) {
      const bool u = k < R.count;
      K.roots[(s * kMaxRoots + k) * 3 + 0] = u ? R.x[k][0] : 0.0;
      K.roots[(s * kMaxRoots + k) * 3 + 1] = u ? R.x[k][1] : 0.0;
      K.roots[(s * kMaxRoots + k) * 3 + 2] = u ? R.x[k][2] : 0.0;
      K.resid[s * kMaxRoots + k] = u ? R.r[k] : 0.0;
    }
  }
}

// ---- block-wide exclusive scan (shared by the single-pass scan below) ------------------

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_sums, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t w = lane < nw ? warp_sums[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < nw) warp_sums[lane] = wi - w;
    if (lane == 31) warp_sums[32] = wi;
  }
  __syncthreads();
  const uint32_t out = warp_sums[warp] + incl - v;
  total = warp_sums[32];
  __syncthreads();
  return out;
}

// ---- single-pass exclusive scan (decoupled look-back) -----------------------------------
// Tiles of 1024 elements are taken in ticket order (so every predecessor is already running);
// a tile publishes its aggregate, warp 0 looks back 32 predecessors at a time until an
// inclusive prefix, then publishes its own (status word = 2-bit flag | 32-bit value, one
// 64-bit store). One launch instead of a 3-kernel (blocks, block sums, add) scan.
constexpr int kLbThreads = 256, kLbItems = 4, kLbTile = kLbThreads * kLbItems;

__device__ __forceinline__ uint32_t lb_exclusive_prefix(unsigned long long* status, long long t, uint32_t tile_total) {
  volatile unsigned long long* st = status;
  const int lane = threadIdx.x & 31;
  constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62;
  if (t == 0) {
    if (lane == 0) st[0] = kInc | tile_total;
    return 0u;
  }
  if (lane == 0) st[t] = kAgg | tile_total;
  uint32_t prefix = 0;
  for (long long p = t - 1;; p -= 32) {
    const long long q = p - lane;  // lane 0 = the closest predecessor
    unsigned long long v = q >= 0 ? st[q] : kInc;
    while (__any_sync(0xffffffffu, (v >> 62) == 0)) {
      if ((v >> 62) == 0) v = st[q];
    }
    const unsigned inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
    const int last = inc ? __ffs(inc) - 1 : 31;
    uint32_t x = lane <= last ? static_cast<uint32_t>(v) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    prefix += x;
    if (inc) break;
  }
  if (lane == 0) st[t] = kInc | static_cast<unsigned long long>(prefix + tile_total);
  return prefix;
}

// In-place exclusive scan of *n_dev u32 (status: [0] ticket, [1..] tile words, zeroed);
// the grand total to *total, and *overflow += 1 when it exceeds cap (if given).
__global__ void __launch_bounds__(kLbThreads) scan_lookback_kernel(uint32_t* __restrict__ a, const unsigned long long* n_dev,
                                                                   unsigned long long* status, unsigned long long* total,
                                                                   unsigned long long cap = 0,
                                                                   unsigned long long* overflow = nullptr) {
  __shared__ uint32_t wsum[33];
  __shared__ long long s_tile;
  __shared__ uint32_t s_prefix;
  const long long n = static_cast<long long>(*n_dev);
  const long long n_tiles = (n + kLbTile - 1) / kLbTile;
  for (;;) {
    if (threadIdx.x == 0) s_tile = static_cast<long long>(atomicAdd(status, 1ull));
    __syncthreads();
    const long long t = s_tile;
    if (t >= (n_tiles > 0 ? n_tiles : 1)) break;
    const long long i0 = t * kLbTile + static_cast<long long>(threadIdx.x) * kLbItems;
    uint32_t v[kLbItems];
    uint32_t mine = 0;
    if (i0 + kLbItems <= n && (reinterpret_cast<uintptr_t>(a + i0) & 15) == 0) {
      const uint4 q = *reinterpret_cast<const uint4*>(a + i0);
      v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
    } else {
#pragma unroll
      for (int k = 0; k < kLbItems; ++k) v[k] = i0 + k < n ? a[i0 + k] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kLbItems; ++k) mine += v[k];
    uint32_t tile_total;
    const uint32_t off = block_exclusive_scan(mine, wsum, tile_total);
    if (threadIdx.x < 32) {
      const uint32_t pre = lb_exclusive_prefix(status + 1, t, tile_total);
      if (threadIdx.x == 0) {
        s_prefix = pre;
        if (t == (n_tiles > 0 ? n_tiles - 1 : 0)) {
          const unsigned long long tot = static_cast<unsigned long long>(pre) + tile_total;
          *total = tot;
          if (overflow && tot > cap) *overflow += 1;
        }
      }
    }
    __syncthreads();
    uint32_t run = s_prefix + off;
    uint32_t o[kLbItems];
#pragma unroll
    for (int k = 0; k < kLbItems; ++k) {
      o[k] = run;
      run += v[k];
    }
    if (i0 + kLbItems <= n && (reinterpret_cast<uintptr_t>(a + i0) & 15) == 0) {
      *reinterpret_cast<uint4*>(a + i0) = make_uint4(o[0], o[1], o[2], o[3]);
    } else {
#pragma unroll
      for (int k = 0; k < kLbItems; ++k)
        if (i0 + k < n) a[i0 + k] = o[k];
    }
    __syncthreads();
  }
}

}  // namespace arfx
