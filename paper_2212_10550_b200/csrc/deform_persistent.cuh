// deform_persistent.cuh -- SIMT-efficient correspondence search (K2) on sm_100a.
//
// Same arithmetic as deform.cuh (bit-exact inverse_lbs_ctx, R/articulation.hpp:94-145),
// re-scheduled for the GPU in two kernels:
//
//  K2a prune_kernel: one thread per target x', all lanes busy. Start pruning
//      (R/articulation.hpp:101-102) rejects bones first with a conservative f32
//      bounding-sphere test and runs the exact FP64 point-segment distance only for
//      bones whose sphere contains x'. Targets with no surviving start are finished
//      here (no roots); the rest are appended, with their start mask, to a compact
//      work list (warp-aggregated atomics).
//
//  K2b deform_persistent_kernel: persistent warps over the work list. Every lane runs
//      the damped-Newton loop as a state machine whose unit of progress is ONE skinning
//      eval (interpolate + lbs + Jacobian); each loop trip every busy lane performs
//      exactly one eval, so a lane whose start converges after one iteration does not
//      idle while a neighbour runs twenty (iteration counts range 0..20, mean 5;
//      SURVEY.md §8a) -- it takes its sample's next start or the next work item.
//      The starts of one sample stay on one lane in bone order, so InverseRoots::push's
//      dedup / replacement order (R/articulation.hpp:66-81) is reproduced exactly.
//      Work items come from a warp-local queue (one global atomic per 64 items); the
//      in-box roots go to warp-local chunks of the root pool (one atomic per chunk),
//      unused chunk slots are marked empty (owner -2) for K3.
#pragma once

#include "deform.cuh"
#include "field.cuh"

namespace arfx {

constexpr int kDfThreads = 128;
constexpr int kDfSampleChunk = 64;
constexpr int kDfPoolChunk = 64;

enum DfState : int { DF_NEED = 0, DF_NEXT = 1, DF_ITER = 2, DF_EVAL_INIT = 3, DF_EVAL_LS = 4, DF_DONE = 5 };

__device__ __forceinline__ unsigned df_lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Surviving starts of inverse_lbs_ctx: bit b set iff cap_dist(x', b) <= cutoff_b (exact).
__device__ __forceinline__ uint32_t df_prune(const PoseCtx* __restrict__ P, d3 xt, int& exact_tests) {
  const float fx = static_cast<float>(xt.x), fy = static_cast<float>(xt.y), fz = static_cast<float>(xt.z);
  uint32_t mask = 0;
  for (int b = 0; b < P->nb; ++b) {
    const float dx = fx - P->sph[b][0], dy = fy - P->sph[b][1], dz = fz - P->sph[b][2];
    const float d2 = dx * dx + dy * dy + dz * dz;
    if (d2 > P->sph[b][3]) continue;  // provably pruned (see PoseCtx::sph)
    ++exact_tests;
    const d3 ca = make3(P->cap_a[b][0], P->cap_a[b][1], P->cap_a[b][2]);
    const d3 cb = make3(P->cap_b[b][0], P->cap_b[b][1], P->cap_b[b][2]);
    if (point_segment_distance(xt, ca, cb) > P->cutoff[b]) continue;
    mask |= 1u << b;
  }
  return mask;
}

// ---- sinks: what happens when a sample's root set is final ----------------------

// Render / occupancy sink (posed_query_ctx R/articulation.hpp:170-173): the in-box roots
// of each sample, in push order, go to consecutive root-pool slots for K3.
struct PoolSink {
  uint8_t* snroot;
  int32_t* sbase;
  double *px, *py, *pz;
  int32_t* powner;
  unsigned long long* counters;  // [1] canonical, [2] pool cursor, [3] overflow
  long long cap_pool;
  FieldView F;
  __device__ void empty(long long s) const {
    snroot[s] = 0;
    sbase[s] = -1;
  }
};

struct RootsSink {  // batched inverse_lbs API: every root + residual, [n][8]
  int32_t* counts;
  double* roots;
  double* resid;
  __device__ void empty(long long s) const { counts[s] = 0; }
};

// Warp-cooperative finish for PoolSink: all 32 lanes call it; `fin` lanes own a finished
// sample `s` with roots R. Pool slots come from the warp's current chunk.
__device__ __forceinline__ void df_finish(const PoolSink& K, bool fin, long long s, const Roots& R,
                                          long long& p_next, long long& p_end, unsigned& canon_count) {
  const int lane = threadIdx.x & 31;
  uint32_t inbox = 0;  // bit k: root k is inside the canonical box
  if (fin)
    for (int k = 0; k < R.count; ++k)
      if (field_contains(K.F, make3(R.x[k][0], R.x[k][1], R.x[k][2]))) inbox |= 1u << k;
  const int need = __popc(inbox);
  int incl = need;  // warp inclusive scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  const int excl = incl - need;
  if (total > 0 && p_end - p_next < total) {
    for (long long q = p_next + lane; q < p_end; q += 32)  // retire the rest of the chunk
      if (q < K.cap_pool) K.powner[q] = -2;
    const long long want = total > kDfPoolChunk ? total : kDfPoolChunk;
    long long base = 0;
    if (lane == 0) base = static_cast<long long>(atomicAdd(K.counters + 2, static_cast<unsigned long long>(want)));
    p_next = __shfl_sync(0xffffffffu, base, 0);
    p_end = p_next + want;
  }
  if (fin) {
    K.snroot[s] = static_cast<uint8_t>(need);
    if (need == 0) {
      K.sbase[s] = -1;
    } else {
      ++canon_count;
      long long q = p_next + excl;
      K.sbase[s] = static_cast<int32_t>(q);
      if (q + need > K.cap_pool) {
        atomicAdd(K.counters + 3, 1ull);  // overflow: the host regrows and re-runs
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
  p_next += total;
}

__device__ __forceinline__ void df_finish(const RootsSink& K, bool fin, long long s, const Roots& R,
                                          long long&, long long&, unsigned&) {
  if (!fin) return;
  K.counts[s] = R.count;
  for (int k = 0; k < R.count; ++k) {
    K.roots[(s * kMaxRoots + k) * 3 + 0] = R.x[k][0];
    K.roots[(s * kMaxRoots + k) * 3 + 1] = R.x[k][1];
    K.roots[(s * kMaxRoots + k) * 3 + 2] = R.x[k][2];
    K.resid[s * kMaxRoots + k] = R.r[k];
  }
}

__device__ __forceinline__ void df_flush_pool(const PoolSink& K, long long p_next, long long p_end) {
  const int lane = threadIdx.x & 31;
  for (long long q = p_next + lane; q < p_end; q += 32)
    if (q < K.cap_pool) K.powner[q] = -2;
}
__device__ __forceinline__ void df_flush_pool(const RootsSink&, long long, long long) {}
__device__ __forceinline__ void df_add_canonical(const PoolSink& K, unsigned c) {
  if (c) atomicAdd(K.counters + 1, static_cast<unsigned long long>(c));
}
__device__ __forceinline__ void df_add_canonical(const RootsSink&, unsigned) {}

template <bool kSinglePose>
__device__ __forceinline__ const PoseCtx* df_stage_pose(const PoseCtx* poses, double* smem) {
  if (!kSinglePose) return poses;
  const int words = static_cast<int>(sizeof(PoseCtx) / 8);
  const double* g = reinterpret_cast<const double*>(poses);
  for (int i = threadIdx.x; i < words; i += blockDim.x) smem[i] = g[i];
  __syncthreads();
  return reinterpret_cast<const PoseCtx*>(smem);
}

// K2a: prune + compaction. One thread per target, grid-stride with warp-uniform trips.
template <class Src, class Sink, bool kSinglePose>
__global__ void __launch_bounds__(256) prune_kernel(const PoseCtx* __restrict__ poses, Src src, Sink sink,
                                                    uint2* __restrict__ work, unsigned long long* work_len,
                                                    unsigned long long* stats) {
  extern __shared__ double pr_smem[];
  const PoseCtx* Pb = df_stage_pose<kSinglePose>(poses, pr_smem);
  const int lane = threadIdx.x & 31;
  const long long n = src.count();
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  int exact = 0;
  for (long long base = (static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
       base < n; base += warps * 32) {
    const long long s = base + lane;
    uint32_t mask = 0;
    if (s < n) {
      int pose;
      const d3 xt = src.point(s, pose);
      mask = df_prune(kSinglePose ? Pb : Pb + pose, xt, exact);
      if (!mask) sink.empty(s);
    }
    const unsigned b = __ballot_sync(0xffffffffu, mask != 0);
    if (!b) continue;
    unsigned long long off = 0;
    if (lane == 0) off = atomicAdd(work_len, static_cast<unsigned long long>(__popc(b)));
    off = __shfl_sync(0xffffffffu, off, 0);
    if (mask) work[off + __popc(b & df_lanemask_lt())] = make_uint2(static_cast<unsigned>(s), mask);
  }
  if (stats) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) exact += __shfl_xor_sync(0xffffffffu, exact, o);
    if (lane == 0 && exact) atomicAdd(stats + 4, static_cast<unsigned long long>(exact));
  }
}

// K2b: the Newton state machine over the work list. kStats: count evals / union bones /
// Newton steps / starts into stats[0..3] (deterministic per frame; used for the roofline).
template <class Src, class Sink, bool kSinglePose, bool kStats>
__global__ void __launch_bounds__(kDfThreads) deform_persistent_kernel(SkinView S, const PoseCtx* __restrict__ poses,
                                                                        InverseOpts opt, Src src, Sink sink,
                                                                        const uint2* __restrict__ work,
                                                                        const unsigned long long* work_len,
                                                                        unsigned long long* cursor,
                                                                        unsigned long long* stats) {
  unsigned long long st_e = 0, st_u = 0, st_i = 0, st_s = 0;
  extern __shared__ double df_smem[];
  const PoseCtx* Pbase = df_stage_pose<kSinglePose>(poses, df_smem);
  double* ws = df_smem + (kSinglePose ? (sizeof(PoseCtx) + 7) / 8 : 0) + threadIdx.x;
  const int stride = blockDim.x;
  const int lane = threadIdx.x & 31;
  const long long n = static_cast<long long>(*work_len);

  int state = DF_NEED;
  long long s = -1;
  uint32_t mask = 0;
  int pose = 0, it = 0, h = 0;
  d3 xt = make3(0, 0, 0), x = xt, g = xt, step = xt, cand = xt;
  double gn = 0.0, gcn = 0.0, damp = 1.0;
  double J0 = 0, J1 = 0, J2 = 0, J3 = 0, J4 = 0, J5 = 0, J6 = 0, J7 = 0, J8 = 0;
  Roots R;
  R.count = 0;
  long long q_next = 0, q_end = 0;  // warp-uniform work queue
  long long p_next = 0, p_end = 0;  // warp-uniform pool chunk
  unsigned canon = 0;

  while (true) {
    // ---- A: bring every lane to an eval (or DONE) ----------------------------------
    while (true) {
      if (state == DF_ITER) {  // Newton step with the frozen Jacobian (R/math.hpp:141-158)
        if (it >= opt.max_iterations) {
          state = DF_NEXT;
        } else {
          const double c0 = dsub(dmul(J4, J8), dmul(J5, J7));
          const double c1 = dsub(dmul(J3, J8), dmul(J5, J6));
          const double c2 = dsub(dmul(J3, J7), dmul(J4, J6));
          const double det = dadd(dsub(dmul(J0, c0), dmul(J1, c1)), dmul(J2, c2));
          if (fabs(det) < 2.2250738585072014e-308 * 64) {
            state = DF_NEXT;  // singular: abandon the start (R/articulation.hpp:114-118)
          } else {
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
            if (kStats) ++st_i;
            step = make3(dadd(dadd(dmul(i0, g.x), dmul(i1, g.y)), dmul(i2, g.z)),
                         dadd(dadd(dmul(i3, g.x), dmul(i4, g.y)), dmul(i5, g.z)),
                         dadd(dadd(dmul(i6, g.x), dmul(i7, g.y)), dmul(i8, g.z)));
            damp = 1.0;
            h = 0;
            cand = sub3(x, mul3(step, damp));
            state = DF_EVAL_LS;
          }
        }
      }
      bool fin = false;
      if (state == DF_NEXT) {
        if (mask) {
          const int b = __ffs(mask) - 1;
          mask &= mask - 1;
          cand = rigid_apply((kSinglePose ? Pbase : Pbase + pose)->bone_inv[b], xt);
          state = DF_EVAL_INIT;
          if (kStats) ++st_s;
        } else {
          fin = true;
          state = DF_NEED;
        }
      }
      if (__any_sync(0xffffffffu, fin)) df_finish(sink, fin, s, R, p_next, p_end, canon);
      const bool need = state == DF_NEED;
      const unsigned nm = __ballot_sync(0xffffffffu, need);
      if (nm) {
        const int k = __popc(nm);
        const int r = __popc(nm & df_lanemask_lt());
        const long long avail = q_end - q_next;
        long long id;
        if (avail >= k) {
          id = q_next + r;
          q_next += k;
        } else {
          long long base = 0;
          if (lane == 0) base = static_cast<long long>(atomicAdd(cursor, static_cast<unsigned long long>(kDfSampleChunk)));
          base = __shfl_sync(0xffffffffu, base, 0);
          id = r < avail ? q_next + r : base + (r - avail);
          q_next = base + (k - avail);
          q_end = base + kDfSampleChunk;
        }
        if (need) {
          if (id >= n) {
            state = DF_DONE;
          } else {
            const uint2 wi = work[id];
            s = wi.x;
            mask = wi.y;
            xt = src.point(s, pose);
            R.count = 0;
            state = DF_NEXT;
          }
        }
      }
      if (!__ballot_sync(0xffffffffu, state == DF_NEXT || state == DF_ITER || state == DF_NEED)) break;
    }
    if (__all_sync(0xffffffffu, state == DF_DONE)) break;

    // ---- B: one skinning eval per busy lane (the hot part) --------------------------
    if (state == DF_EVAL_INIT || state == DF_EVAL_LS) {
      double Jn[9];
      const int nu = skin_eval(S, kSinglePose ? Pbase : Pbase + pose, cand, xt, ws, stride, g, gcn, Jn);
      if (kStats) {
        ++st_e;
        st_u += static_cast<unsigned long long>(nu);
      }
      J0 = Jn[0], J1 = Jn[1], J2 = Jn[2], J3 = Jn[3], J4 = Jn[4], J5 = Jn[5], J6 = Jn[6], J7 = Jn[7], J8 = Jn[8];
    }

    // ---- C: Newton / line-search bookkeeping (R/articulation.hpp:104-142) ------------
    if (state == DF_EVAL_INIT) {
      x = cand;
      gn = gcn;
      if (gn < opt.tolerance) {
        roots_push(R, x, gn, opt.dedup_radius);
        state = DF_NEXT;
      } else {
        it = 0;
        state = DF_ITER;
      }
    } else if (state == DF_EVAL_LS) {
      if (gcn < gn || h == 3) {
        if (gcn >= gn && gn >= opt.tolerance) {
          state = DF_NEXT;  // stalled: drop the start
        } else {
          x = cand;
          gn = gcn;
          ++it;
          if (gn < opt.tolerance) {
            roots_push(R, x, gn, opt.dedup_radius);
            state = DF_NEXT;
          } else {
            state = DF_ITER;
          }
        }
      } else {
        damp = dmul(damp, 0.5);
        ++h;
        cand = sub3(x, mul3(step, damp));
      }
    }
  }
  df_flush_pool(sink, p_next, p_end);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) canon += __shfl_xor_sync(0xffffffffu, canon, o);
  if (lane == 0) df_add_canonical(sink, canon);
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

}  // namespace arfx
