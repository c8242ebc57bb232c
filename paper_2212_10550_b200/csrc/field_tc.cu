// field_tc.cu -- K3 on the 5th-gen tensor cores.
//
// Default (ARFX_TC_FUSED=1): field_fused_kernel, encode and the 32-64-64-4 decoder in one
// persistent warp-specialised kernel (no feature tiles in HBM; see the comment above it).
//
// Two-stage alternative (ARFX_TC_FUSED=0, measured 0.463 vs 0.426 ms/frame for the fused one):
//   encode_tiles_kernel  thread = query, 16 hash-grid levels (warp-uniform level, exact f64
//                        corner weights as field_tile_kernel); the 32 features are split into
//                        bf16 hi / lo planes and written straight into the UMMA K-major,
//                        no-swizzle canonical layout of their 128-query tile in global memory
//                        (coalesced 512-B stores). High occupancy: this stage is the gathers.
//   field_tc_kernel      the decoder: one persistent 512-thread CTA per SM runs 4
//                        independent 128-query pipelines (own TMEM columns, mbarriers, named
//                        barrier) over weights staged once in smem. Per tile:
//     load     one cp.async.bulk of the 16-KB feature tile into the group's A0 buffer (the
//              next tile's copy is issued as soon as layer 0 has consumed A0)
//     layer 0  D[128x64] = A0[128x32] * W0^T    2 K-steps x 3 MMAs, TMEM cols [0, 64)
//     epi 0    tcgen05.ld, + b0, ReLU -> A1 planes
//     layer 1  D[128x64] = A1[128x64] * W1^T    4 x 3 MMAs, TMEM cols [0, 64) (D0 consumed)
//     epi 1    + b1, ReLU -> A1 (in place: the layer-1 MMAs have completed)
//     layer 2  D[128x16] = A1[128x64] * W2p^T   4 x 3 MMAs, W2 padded to N = 16, cols [64, 80)
//     epi 2    + b2, softplus / logistic (R/field.hpp:78-81) -> (density, rgb)
//   One thread issues the MMAs (tcgen05.mma kind::f16); completion is signalled with
//   tcgen05.commit on an mbarrier. The fused kernel runs the same three layers.
//
// Operands are split bf16 pairs (x = hi + lo, hi = bf16(x), lo = bf16(x - hi)) and every
// product is formed as hi*hi + hi*lo + lo*hi (bf16 in, fp32 accumulate in TMEM): ~16
// significant bits, ~1e-5 relative, for the same smem footprint as one fp32 operand.
// Not bit-exact with the reference's sequential f32 sums (stated tolerance);
// the exact SIMT decoder (field_tile_kernel) stays the default (arfx_model_set_mlp_mode).
// ARFX_MLP_TCGEN05_FP16 feeds the encode stage from an fp16 copy of the table.
#include <cuda_runtime.h>

#include <cuda_bf16.h>

#include <algorithm>

#include "field.cuh"
#include "model.h"
#include "umma.cuh"

namespace arfx {
namespace {
using namespace umma;

constexpr int kTcTile = 128;
#ifndef ARFX_TC_FUSED
#define ARFX_TC_FUSED 1
#endif
#ifndef ARFX_TC_REVERSE
#define ARFX_TC_REVERSE 1
#endif
constexpr int kIn = 32, kHid = 64, kOutPad = 16;
constexpr uint32_t kTmemCols = 512;  // 4 groups x 128 columns (whole TMEM: one CTA per SM)

// One CTA per SM runs kGroups independent 128-query pipelines (4 warps each, own TMEM
// columns, own activation tile, own mbarrier, own named barrier) over shared weights, so
// the hash-grid gathers of one group overlap the MMAs/epilogues of the others.
constexpr int kGroups = 4;
constexpr int kTcThreads = kGroups * kTcTile;

struct TcSmem {  // byte offsets inside the dynamic smem; each operand = hi plane, lo plane
  static constexpr int B0P = kHid * kIn * 2, B1P = kHid * kHid * 2, B2P = kOutPad * kHid * 2;
  static constexpr int A0P = kTcTile * kIn * 2, A1P = kTcTile * kHid * 2;
  static constexpr int B0 = 0;                              // W0  64 x 32  (2 x 4 KB)
  static constexpr int B1 = B0 + 2 * B0P;                   // W1  64 x 64  (2 x 8 KB)
  static constexpr int B2 = B1 + 2 * B1P;                   // W2p 16 x 64  (2 x 2 KB)
  static constexpr int BIAS = B2 + 2 * B2P;                 // b0[64] b1[64] b2[4]
  static constexpr int ACT = BIAS + 1024;                   // per group: hidden 128 x 64 (2 x 16 KB);
  static constexpr int ACT_BYTES = 2 * A0P + 2 * A1P;       //   + its own feature tile (2 x 8 KB), so the
                                                            //   next tile's bulk copy overlaps this one
  static constexpr int MBAR = ACT + kGroups * ACT_BYTES;    // u64 [kGroups]: MMA completion
  static constexpr int LBAR = MBAR + 8 * kGroups;           // u64 [kGroups]: feature-tile load
  static constexpr int TADDR = LBAR + 8 * kGroups;          // u32
  static constexpr int TOTAL = TADDR + 16;
};

__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "n"(kTcTile) : "memory");
}

// Encode stage: thread = query, all 16 levels (warp-uniform level), features split into
// bf16 hi/lo and stored straight in the UMMA K-major A0 layout of the query's 128-row tile
// (16 KB per tile in global memory): a warp's 32 consecutive rows are 512 contiguous bytes
// per 16-B chunk, so the stores coalesce. It runs at much higher occupancy than the fused
// encode+MMA kernel could (smem-bound there), which is what hides the hash-table gathers;
// the MMA stage then only streams tiles. (A thread per (query, 4-level chunk) split was
// measured slower: 4x the FP64 normalisation for no extra gather parallelism.)
constexpr int kEncThreads = 256;
#ifndef ARFX_ENC_MIN_BLOCKS
#define ARFX_ENC_MIN_BLOCKS 4
#endif
// fp16 gathers (mode 2): the level's float2 row is read as half2 (4 B instead of 8 B),
// widened to f32, and accumulated exactly like encode_level_f2
__device__ __forceinline__ float2 encode_level_h2(const FieldView& F, const __half2* __restrict__ table, int l,
                                                  const double u[3]) {
  LevelCorners lc;
  level_corners(F, l, u, lc);
  const __half2* t = table + static_cast<size_t>(l) * F.T;
  float2 row[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) row[k] = __half22float2(__ldg(t + lc.idx[k]));
  float o0 = 0.0f, o1 = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    o0 = fadd(o0, fmul(lc.w[k], row[k].x));
    o1 = fadd(o1, fmul(lc.w[k], row[k].y));
  }
  return make_float2(o0, o1);
}

__global__ void to_half2_kernel(const float2* __restrict__ src, __half2* __restrict__ dst, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = __float22half2_rn(src[i]);
}

template <bool kHalf>
__global__ void __launch_bounds__(kEncThreads, ARFX_ENC_MIN_BLOCKS)
    encode_tiles_kernel(FieldView F, const __half2* __restrict__ table_h2, const double* __restrict__ px,
                        const double* __restrict__ py, const double* __restrict__ pz,
                        const int32_t* __restrict__ owner, const unsigned long long* n_dev, long long cap,
                        unsigned char* __restrict__ tiles, unsigned long long* stats) {
  long long n = static_cast<long long>(*n_dev);
  n = n < cap ? n : cap;
  for (long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool ok = owner[q] >= 0;
    if (stats) {
      const unsigned c = __popc(__ballot_sync(__activemask(), ok));
      if ((threadIdx.x & 31) == 0 && c) atomicAdd(stats + 6, static_cast<unsigned long long>(c));
    }
    if (!ok) continue;  // row left as is: rows are independent in the MMAs, its result is dropped
    double u[3];
    normalize_point(F, make3(px[q], py[q], pz[q]), u);
    unsigned char* tile = tiles + (q / kTcTile) * (2 * TcSmem::A0P);
    const int r = static_cast<int>(q % kTcTile);
#pragma unroll 1
    for (int l = 0; l < 16; l += 4) {
      __nv_bfloat16 hi[8], lo[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 o = kHalf ? encode_level_h2(F, table_h2, l + j, u) : encode_level_f2(F, l + j, u);
        split_bf16(o.x, hi[2 * j], lo[2 * j]);
        split_bf16(o.y, hi[2 * j + 1], lo[2 * j + 1]);
      }
      *reinterpret_cast<uint4*>(tile + kmaj_off(r, 2 * l, kTcTile)) = *reinterpret_cast<const uint4*>(hi);
      *reinterpret_cast<uint4*>(tile + TcSmem::A0P + kmaj_off(r, 2 * l, kTcTile)) =
          *reinterpret_cast<const uint4*>(lo);
    }
  }
}

__global__ void __launch_bounds__(kTcThreads, 1) field_tc_kernel(FieldView F, const unsigned char* __restrict__ tiles,
                                                                 const int32_t* __restrict__ owner,
                                                                 float4* __restrict__ res,
                                                                 const unsigned long long* n_dev, long long cap) {
  extern __shared__ __align__(1024) unsigned char tc_smem[];
  const int g = threadIdx.x / kTcTile;  // pipeline group
  const int tid = threadIdx.x % kTcTile, warp = tid >> 5;
  long long n = static_cast<long long>(*n_dev);
  n = n < cap ? n : cap;
  if (static_cast<long long>(blockIdx.x) * kTcTile * kGroups >= n) return;

  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(tc_smem));
  float* bias = reinterpret_cast<float*>(tc_smem + TcSmem::BIAS);
  const uint32_t mbar = sbase + TcSmem::MBAR + 8 * g;
  const uint32_t lbar = sbase + TcSmem::LBAR + 8 * g;
  uint32_t* taddr_smem = reinterpret_cast<uint32_t*>(tc_smem + TcSmem::TADDR);
  const int A0 = TcSmem::ACT + g * TcSmem::ACT_BYTES, A1 = A0 + 2 * TcSmem::A0P;  // this group's tiles

  // ---- stage the weights in the K-major operand layouts (W[o][i] is N x K, K-major) ----
  const float* W0 = F.mlp;
  const float* b0 = W0 + kIn * kHid;
  const float* W1 = b0 + kHid;
  const float* b1 = W1 + kHid * kHid;
  const float* W2 = b1 + kHid;
  const float* b2 = W2 + 4 * kHid;
  auto put = [&](int off, int plane, float x) {
    __nv_bfloat16 hi, lo;
    split_bf16(x, hi, lo);
    *reinterpret_cast<__nv_bfloat16*>(tc_smem + off) = hi;
    *reinterpret_cast<__nv_bfloat16*>(tc_smem + off + plane) = lo;
  };
  const int ctid = threadIdx.x;
  for (int i = ctid; i < kHid * kIn; i += kTcThreads) {
    const int o = i / kIn, k = i % kIn;
    put(TcSmem::B0 + kmaj_off(o, k, kHid), TcSmem::B0P, __ldg(W0 + i));
  }
  for (int i = ctid; i < kHid * kHid; i += kTcThreads) {
    const int o = i / kHid, k = i % kHid;
    put(TcSmem::B1 + kmaj_off(o, k, kHid), TcSmem::B1P, __ldg(W1 + i));
  }
  for (int i = ctid; i < kOutPad * kHid; i += kTcThreads) {
    const int o = i / kHid, k = i % kHid;
    put(TcSmem::B2 + kmaj_off(o, k, kOutPad), TcSmem::B2P, o < 4 ? __ldg(W2 + o * kHid + k) : 0.0f);
  }
  for (int i = ctid; i < kHid; i += kTcThreads) {
    bias[i] = __ldg(b0 + i);
    bias[64 + i] = __ldg(b1 + i);
  }
  if (ctid < 4) bias[128 + ctid] = __ldg(b2 + ctid);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(lbar) : "memory");
  }
  if (ctid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sbase + TcSmem::TADDR),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *taddr_smem + static_cast<uint32_t>(g * 128);        // this group's columns
  const uint32_t tmem_row = tmem + (static_cast<uint32_t>(warp * 32) << 16);  // this warp's 32 lanes
  uint32_t phase = 0, lphase = 0;
  constexpr uint32_t ID64 = idesc_bf16(128, 64);
  constexpr uint32_t ID16 = idesc_bf16(128, 16);
  // writes row `tid`, columns [c, c+8) of a split operand (hi plane, lo plane)
  auto put8 = [&](int base, int plane, int c, const float* x) {
    __nv_bfloat16 hi[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) split_bf16(x[j], hi[j], lo[j]);
    *reinterpret_cast<uint4*>(tc_smem + base + kmaj_off(tid, c, kTcTile)) = *reinterpret_cast<const uint4*>(hi);
    *reinterpret_cast<uint4*>(tc_smem + base + plane + kmaj_off(tid, c, kTcTile)) = *reinterpret_cast<const uint4*>(lo);
  };

  constexpr uint32_t kTileBytes = 2 * TcSmem::A0P;
  auto load_tile = [&](long long t) {  // one bulk copy of a 16-KB feature tile into A0
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lbar), "n"(kTileBytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sbase + A0),
        "l"(tiles + (t / kTcTile) * kTileBytes), "n"(kTileBytes), "r"(lbar)
        : "memory");
  };
  const long long stride = static_cast<long long>(gridDim.x) * kGroups * kTcTile;
  // tiles are consumed in reverse order of production: the encode pass writes ~150 MB of
  // tiles through a 126 MB L2, so the last-written tiles are the ones still resident
  const long long n_tiles = (n + kTcTile - 1) / kTcTile;
  auto phys = [&](long long lt) { return ARFX_TC_REVERSE ? (n_tiles - 1 - lt / kTcTile) * kTcTile : lt; };
  const long long first = (static_cast<long long>(blockIdx.x) * kGroups + g) * kTcTile;
  if (tid == 0 && first < n) load_tile(phys(first));
  for (long long lt0 = first; lt0 < n; lt0 += stride) {
    const long long t0 = phys(lt0);
    const long long q = t0 + tid;
    const bool ok = q < n && owner[q] >= 0;
    mbar_wait(lbar, lphase);  // this tile's features have landed in A0
    lphase ^= 1;
    // ---- layer 0 ----
    if (tid == 0) {
      tc_fence_after();
      mma_split(tmem, sbase + A0, TcSmem::A0P, kTcTile, sbase + TcSmem::B0, TcSmem::B0P, kHid, kIn, ID64);
      mma_commit(mbar);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    tc_fence_after();
    // A0 is free again: the next tile's copy overlaps the rest of this one
    if (tid == 0 && lt0 + stride < n) load_tile(phys(lt0 + stride));
    // ---- epilogue 0: + b0, ReLU -> A1 ----
#pragma unroll
    for (int c = 0; c < kHid; c += 16) {
      float v[16];
      tmem_ld16(tmem_row + c, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j] + bias[c + j], 0.f);
      put8(A1, TcSmem::A1P, c, v);
      put8(A1, TcSmem::A1P, c + 8, v + 8);
    }
    tc_fence_before();
    fence_async_smem();
    group_sync(g);
    // ---- layer 1 ----
    if (tid == 0) {
      tc_fence_after();
      mma_split(tmem, sbase + A1, TcSmem::A1P, kTcTile, sbase + TcSmem::B1, TcSmem::B1P, kHid, kHid, ID64);
      mma_commit(mbar);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- epilogue 1: + b1, ReLU -> A1 (in place) ----
#pragma unroll
    for (int c = 0; c < kHid; c += 16) {
      float v[16];
      tmem_ld16(tmem_row + c, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j] + bias[64 + c + j], 0.f);
      put8(A1, TcSmem::A1P, c, v);
      put8(A1, TcSmem::A1P, c + 8, v + 8);
    }
    tc_fence_before();
    fence_async_smem();
    group_sync(g);
    // ---- layer 2 (N padded to 16) ----
    if (tid == 0) {
      tc_fence_after();
      mma_split(tmem + 64, sbase + A1, TcSmem::A1P, kTcTile, sbase + TcSmem::B2, TcSmem::B2P, kOutPad, kHid,
                ID16);
      mma_commit(mbar);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    tc_fence_after();
    {
      float v[16];
      tmem_ld16(tmem_row + 64, v);
      if (ok) {
        const float l0 = v[0] + bias[128], l1 = v[1] + bias[129], l2 = v[2] + bias[130], l3 = v[3] + bias[131];
        res[t0 + tid] = make_float4(softplus_f(l0), logistic_f(l1), logistic_f(l2), logistic_f(l3));
      }
    }
    tc_fence_before();
    group_sync(g);
  }
  __syncthreads();
  if (ctid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*taddr_smem), "n"(kTmemCols)
                 : "memory");
}

// ---------------------------------------------------------------------------------------------
// Fused encode -> MLP (K3-TC fused, warp-specialised): no feature tiles in HBM. One persistent
// CTA per SM:
//   gather groups  kWG groups of kWS x 4 warps; a group owns kWB A0 buffers (split-bf16
//                  K-major, 2 x 8 KB) and loops over its 128-query tiles: wait until the
//                  buffer is free, thread (row r, level slice s) gathers levels
//                  s, s + kWS, s + 2 kWS, ... of query r (coarse, L1-resident and fine, L2
//                  levels mixed, so a group's slices finish together) straight into it in a
//                  permuted K order (ws_feature_of_k; W0 is staged to match), then one arrive
//                  on the buffer's `full` barrier. These warps never wait on the tensor core
//                  beyond the buffer hand-back, so they keep the L1 gather pipe busy.
//   MMA team       4 warps (TMEM lane quarters 0-3): takes the filled buffers in a fixed
//                  round-robin order, issues layer 0 (whose completion, committed to the
//                  buffer's `empty` barrier, hands the buffer back), then layer 1, and writes
//                  (density, rgb). The hidden activations never leave TMEM: epilogue 0 reads
//                  the fp32 accumulator (tcgen05.ld), adds the bias, applies ReLU, splits into
//                  bf16 hi / lo and stores them back (tcgen05.st) as layer 1's A operand
//                  (`.kind::f16 [d], [a_tmem], b_desc`); epilogue 1 computes the 64 -> 4
//                  output layer as f32 FMAs from the layer-1 accumulator (a third MMA round
//                  trip per tile cost more than the 256 FMAs per row: 0.428 vs 0.402 ms).
// The smem footprint (weights 29 KB + 16 KB per A0 buffer = 78 KB) stays small so the
// unified L1 keeps most of its capacity for the hash-table gathers.
#ifndef ARFX_WS_GROUPS
#define ARFX_WS_GROUPS 3
#endif
#ifndef ARFX_WS_SPLIT
#define ARFX_WS_SPLIT 2
#endif
#ifndef ARFX_WS_BUFS
#define ARFX_WS_BUFS 1
#endif
#ifndef ARFX_WS_LV_UNROLL  // 2: a thread's 8 levels gathered in one unrolled pass
#define ARFX_WS_LV_UNROLL 2
#endif
#ifndef ARFX_WS_L2_SIMT  // layer 2 (64 -> 4) as f32 FMAs in the layer-1 epilogue
#define ARFX_WS_L2_SIMT 1
#endif
constexpr int kWG = ARFX_WS_GROUPS, kWS = ARFX_WS_SPLIT, kWB = ARFX_WS_BUFS;
constexpr int kWGroupThreads = kTcTile * kWS, kWMma = 128;
constexpr int kWThreads = kWMma + kWG * kWGroupThreads;
constexpr int kWTmemCols = 256;
constexpr int kWBarMma = 15;  // named barrier of the MMA team (gather groups use 1..kWG)
static_assert(kWThreads <= 1024 && kWG < kWBarMma && (kWS == 1 || kWS == 2 || kWS == 4), "fused layout");

// K order of the fused kernel's A0 tile: K chunk c (8 bf16 = 4 levels x 2 features) holds
// the levels of gather slice c % kWS, group c / kWS; returns the feature index (2 level + f)
// stored at K position k (W0's columns are staged in the same order)
__device__ __forceinline__ int ws_feature_of_k(int k) {
  const int c = k >> 3, t = (k & 7) >> 1, f = k & 1;
  const int level = (c % kWS) + kWS * (4 * (c / kWS) + t);
  return 2 * level + f;
}

struct WsSmem {
  static constexpr int B0 = TcSmem::B0, B1 = TcSmem::B1, B2 = TcSmem::B2, BIAS = TcSmem::BIAS;
  static constexpr int A0P = TcSmem::A0P, A1P = TcSmem::A1P;
  static constexpr int A0 = TcSmem::ACT;                  // [kWG][kWB] feature tiles (2 x 8 KB)
  static constexpr int FULL = A0 + kWG * kWB * 2 * A0P;   // u64 [kWG * kWB]
  static constexpr int EMPTY = FULL + 8 * kWG * kWB;      // u64 [kWG * kWB]
  static constexpr int MMA = EMPTY + 8 * kWG * kWB;       // u64
  static constexpr int TADDR = MMA + 8;
  static constexpr int W2T = (TADDR + 16 + 15) / 16 * 16;  // f32 [64][4]: W2 transposed (SIMT layer 2)
  static constexpr int TOTAL = W2T + 4 * kHid * 4;
};

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

template <bool kHalf>
__global__ void __launch_bounds__(kWThreads, 1)
    field_fused_kernel(FieldView F, const __half2* __restrict__ table_h2, const double* __restrict__ px,
                       const double* __restrict__ py, const double* __restrict__ pz,
                       const int32_t* __restrict__ owner, float4* __restrict__ res, const unsigned long long* n_dev,
                       long long cap, unsigned long long* stats) {
  extern __shared__ __align__(1024) unsigned char tc_smem[];
  long long n = static_cast<long long>(*n_dev);
  n = n < cap ? n : cap;
  if (static_cast<long long>(blockIdx.x) * kTcTile * kWG >= n) return;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(tc_smem));
  float* bias = reinterpret_cast<float*>(tc_smem + WsSmem::BIAS);
  uint32_t* taddr_smem = reinterpret_cast<uint32_t*>(tc_smem + WsSmem::TADDR);
  const int ctid = threadIdx.x;
  auto full_bar = [&](int g, int b) { return sbase + WsSmem::FULL + 8 * (g * kWB + b); };
  auto empty_bar = [&](int g, int b) { return sbase + WsSmem::EMPTY + 8 * (g * kWB + b); };
  auto a0_off = [&](int g, int b) { return WsSmem::A0 + (g * kWB + b) * 2 * WsSmem::A0P; };
  const uint32_t mma_bar = sbase + WsSmem::MMA;
  // tile of group g in round r (static round-robin over the grid's groups)
  auto tile_q0 = [&](int g, int r) {
    return ((static_cast<long long>(r) * gridDim.x + blockIdx.x) * kWG + g) * kTcTile;
  };

  // ---- stage the weights (W[o][i] is N x K, K-major), barriers, TMEM ----
  const float* W0 = F.mlp;
  const float* b0 = W0 + kIn * kHid;
  const float* W1 = b0 + kHid;
  const float* b1 = W1 + kHid * kHid;
  const float* W2 = b1 + kHid;
  const float* b2 = W2 + 4 * kHid;
  auto put = [&](int off, int plane, float x) {
    __nv_bfloat16 hi, lo;
    split_bf16(x, hi, lo);
    *reinterpret_cast<__nv_bfloat16*>(tc_smem + off) = hi;
    *reinterpret_cast<__nv_bfloat16*>(tc_smem + off + plane) = lo;
  };
  for (int i = ctid; i < kHid * kIn; i += kWThreads) {  // W0's columns in the A0 tile's K order
    const int o = i / kIn, k = i % kIn;
    put(WsSmem::B0 + kmaj_off(o, k, kHid), TcSmem::B0P, __ldg(W0 + o * kIn + ws_feature_of_k(k)));
  }
  for (int i = ctid; i < kHid * kHid; i += kWThreads) {
    const int o = i / kHid, k = i % kHid;
    put(WsSmem::B1 + kmaj_off(o, k, kHid), TcSmem::B1P, __ldg(W1 + i));
  }
  for (int i = ctid; i < kOutPad * kHid; i += kWThreads) {
    const int o = i / kHid, k = i % kHid;
    put(WsSmem::B2 + kmaj_off(o, k, kOutPad), TcSmem::B2P, o < 4 ? __ldg(W2 + o * kHid + k) : 0.0f);
  }
  for (int i = ctid; i < kHid; i += kWThreads) {
    bias[i] = __ldg(b0 + i);
    bias[64 + i] = __ldg(b1 + i);
  }
  if (ctid < 4) bias[128 + ctid] = __ldg(b2 + ctid);
  for (int i = ctid; i < 4 * kHid; i += kWThreads)
    reinterpret_cast<float*>(tc_smem + WsSmem::W2T)[i] = __ldg(W2 + (i % 4) * kHid + i / 4);
  if (ctid < kWG * kWB) {
    const int g = ctid / kWB, b = ctid % kWB;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full_bar(g, b)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty_bar(g, b)) : "memory");
  }
  if (ctid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mma_bar) : "memory");
  if (ctid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sbase + WsSmem::TADDR),
                 "n"(kWTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (ctid >= kWMma) {
    // ================= gather group =================
    const int g = (ctid - kWMma) / kWGroupThreads;
    const int gt = (ctid - kWMma) % kWGroupThreads;
    const int wg = gt >> 5;
    const int row = (wg & 3) * 32 + (gt & 31);
    const int slice = wg >> 2;
    constexpr int kLv = 16 / kWS;
    for (int r = 0;; ++r) {
      const long long q0 = tile_q0(g, r);
      if (q0 >= n) break;
      const int b = r % kWB;
      const long long q = q0 + row;
      const bool ok = q < n && owner[q] >= 0;
      if (stats && slice == 0) {
        const unsigned c = __popc(__ballot_sync(0xffffffffu, ok));
        if ((gt & 31) == 0 && c) atomicAdd(stats + 6, static_cast<unsigned long long>(c));
      }
      double u[3];
      if (ok) normalize_point(F, make3(px[q], py[q], pz[q]), u);
      mbar_wait(empty_bar(g, b), ((r / kWB) & 1) ^ 1);  // layer 0 has consumed this buffer
      if (ok) {
        const int A = a0_off(g, b);
        // slice s gathers levels s, s + kWS, s + 2 kWS, ... (coarse and fine levels mixed, so
        // the group's slices finish together); four of them fill one 16-B K chunk
#if ARFX_WS_LV_UNROLL > 1
#pragma unroll
#else
#pragma unroll 1
#endif
        for (int m0 = 0; m0 < kLv; m0 += 4) {
          __nv_bfloat16 hi[8], lo[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int l = slice + kWS * (m0 + j);
            const float2 o = kHalf ? encode_level_h2(F, table_h2, l, u) : encode_level_f2(F, l, u);
            split_bf16(o.x, hi[2 * j], lo[2 * j]);
            split_bf16(o.y, hi[2 * j + 1], lo[2 * j + 1]);
          }
          const int k = 8 * ((m0 / 4) * kWS + slice);
          *reinterpret_cast<uint4*>(tc_smem + A + kmaj_off(row, k, kTcTile)) = *reinterpret_cast<const uint4*>(hi);
          *reinterpret_cast<uint4*>(tc_smem + A + WsSmem::A0P + kmaj_off(row, k, kTcTile)) =
              *reinterpret_cast<const uint4*>(lo);
        }
      }
      fence_async_smem();  // generic-proxy stores -> visible to the tensor core
      named_sync(1 + g, kWGroupThreads);
      if (gt == 0) mbar_arrive(full_bar(g, b));
    }
  } else {
    // ================= MMA team =================
    const int row = ctid;  // TMEM lane = warp quarter * 32 + lane
    const uint32_t lane_off = static_cast<uint32_t>((ctid >> 5) * 32) << 16;
    const uint32_t t_hid = *taddr_smem, t_out = *taddr_smem + 64;
    // TMEM columns: hidden accumulator [0, 64), layer-2 output [64, 80), A operand hi plane
    // [96, 128) and lo plane [128, 160) (two bf16 per column)
    const uint32_t t_ahi = *taddr_smem + 96, t_alo = *taddr_smem + 128;
    constexpr uint32_t ID64 = idesc_bf16(128, 64);
    constexpr uint32_t ID16 = idesc_bf16(128, 16);
    uint32_t mphase = 0;
    auto hidden_epilogue = [&](int boff) {
#pragma unroll
      for (int c = 0; c < kHid; c += 16) {
        float v[16];
        tmem_ld16(t_hid + lane_off + c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j] + bias[boff + c + j], 0.f);
        uint32_t ph[8], pl[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          __nv_bfloat16 h0, l0, h1, l1;
          split_bf16(v[2 * j], h0, l0);
          split_bf16(v[2 * j + 1], h1, l1);
          ph[j] = static_cast<uint32_t>(__bfloat16_as_ushort(h0)) |
                  (static_cast<uint32_t>(__bfloat16_as_ushort(h1)) << 16);
          pl[j] = static_cast<uint32_t>(__bfloat16_as_ushort(l0)) |
                  (static_cast<uint32_t>(__bfloat16_as_ushort(l1)) << 16);
        }
        tmem_st8(t_ahi + lane_off + c / 2, ph);
        tmem_st8(t_alo + lane_off + c / 2, pl);
      }
      tmem_st_wait();
    };
    auto wait_mma = [&]() {
      mbar_wait(mma_bar, mphase);
      mphase ^= 1;
      tc_fence_after();
    };
    for (int r = 0;; ++r) {
      if (tile_q0(0, r) >= n) break;
      for (int g = 0; g < kWG; ++g) {
        const long long q0 = tile_q0(g, r);
        if (q0 >= n) break;
        const int b = r % kWB;
        mbar_wait(full_bar(g, b), (r / kWB) & 1);
        tc_fence_after();
        // ---- layer 0: its completion also hands the feature buffer back ----
        if (row == 0) {
          mma_split(t_hid, sbase + a0_off(g, b), WsSmem::A0P, kTcTile, sbase + WsSmem::B0, TcSmem::B0P, kHid, kIn,
                    ID64);
          mma_commit(empty_bar(g, b));
          mma_commit(mma_bar);
        }
        wait_mma();
        hidden_epilogue(0);  // + b0, ReLU -> TMEM A operand
        tc_fence_before();
        named_sync(kWBarMma, kWMma);
        // ---- layer 1 ----
        if (row == 0) {
          tc_fence_after();
          mma_split_ts(t_hid, t_ahi, t_alo, sbase + WsSmem::B1, TcSmem::B1P, kHid, kHid, ID64);
          mma_commit(mma_bar);
        }
        wait_mma();
#if ARFX_WS_L2_SIMT
        {  // ---- layer 2 (64 -> 4) on the CUDA cores, straight from the layer-1 accumulator ----
          const float4* w2t = reinterpret_cast<const float4*>(tc_smem + WsSmem::W2T);
          float o0 = bias[128], o1 = bias[129], o2 = bias[130], o3 = bias[131];
#pragma unroll
          for (int c = 0; c < kHid; c += 16) {
            float v[16];
            tmem_ld16(t_hid + lane_off + c, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float h = fmaxf(v[j] + bias[64 + c + j], 0.f);
              const float4 w = w2t[c + j];
              o0 = fmaf(w.x, h, o0);
              o1 = fmaf(w.y, h, o1);
              o2 = fmaf(w.z, h, o2);
              o3 = fmaf(w.w, h, o3);
            }
          }
          const long long q = q0 + row;
          if (q < n && owner[q] >= 0) res[q] = make_float4(softplus_f(o0), logistic_f(o1), logistic_f(o2), logistic_f(o3));
        }
#else
        hidden_epilogue(64);  // + b1, ReLU -> TMEM A operand, in place (layer 1 has completed)
        tc_fence_before();
        named_sync(kWBarMma, kWMma);
        // ---- layer 2 (N padded to 16) ----
        if (row == 0) {
          tc_fence_after();
          mma_split_ts(t_out, t_ahi, t_alo, sbase + WsSmem::B2, TcSmem::B2P, kOutPad, kHid, ID16);
          mma_commit(mma_bar);
        }
        wait_mma();
        {
          float v[16];
          tmem_ld16(t_out + lane_off, v);
          const long long q = q0 + row;
          if (q < n && owner[q] >= 0) {
            const float l0 = v[0] + bias[128], l1 = v[1] + bias[129], l2 = v[2] + bias[130], l3 = v[3] + bias[131];
            res[q] = make_float4(softplus_f(l0), logistic_f(l1), logistic_f(l2), logistic_f(l3));
          }
        }
#endif
        tc_fence_before();
        // every team thread has seen this tile's last completion before the next commit
        named_sync(kWBarMma, kWMma);
      }
    }
  }
  __syncthreads();
  if (ctid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*taddr_smem), "n"(kWTmemCols) : "memory");
}

}  // namespace

bool field_tc_supported(const FieldView& F) {
  return F.F == 2 && F.L == 16 && F.in_dim == kIn && F.hidden == kHid && F.n_layers == 3 && F.out_dim == 4;
}

void launch_field_tc(ModelImpl& m, cudaStream_t s, long long n_hint) {
  const size_t smem = TcSmem::TOTAL + 1024;  // + alignment slack
  ensure_dyn_smem(reinterpret_cast<const void*>(field_tc_kernel), smem);
  const int sms = device_sm_count();
  // persistent: one CTA per SM (it owns all 512 TMEM columns)
  const long long tiles = (n_hint + kTcTile * kGroups - 1) / (kTcTile * kGroups);
  const int grid = static_cast<int>(std::max(1LL, std::min(tiles, static_cast<long long>(sms))));
  const bool half = m.mlp_mode == 2;
  if (half) {  // refresh the fp16 copy of the table (params may have changed since the last render)
    const long long nrow = static_cast<long long>(m.n_grid / 2);
    m.grid_h2.ensure(static_cast<size_t>(nrow));
    m.prof.begin("table_fp16", s);
    to_half2_kernel<<<static_cast<unsigned>(std::min<long long>((nrow + 255) / 256, static_cast<long long>(sms) * 8)), 256,
                      0, s>>>(reinterpret_cast<const float2*>(m.grid_params.ptr), m.grid_h2.ptr, nrow);
    ARFX_CUDA(cudaGetLastError());
    m.prof.end(s);
  }
#if ARFX_TC_FUSED
  {
    const size_t fsmem = WsSmem::TOTAL + 1024;
    auto fk = half ? field_fused_kernel<true> : field_fused_kernel<false>;
    ensure_dyn_smem(reinterpret_cast<const void*>(fk), fsmem);
    const long long ft = (n_hint + kTcTile * kWG - 1) / (kTcTile * kWG);
    const int fgrid = static_cast<int>(std::max(1LL, std::min(ft, static_cast<long long>(sms))));
    m.prof.begin("field_tc", s);
    fk<<<fgrid, kWThreads, fsmem, s>>>(m.fv, m.grid_h2.ptr, m.ws().px.ptr, m.ws().py.ptr, m.ws().pz.ptr,
                                       m.ws().powner.ptr, m.ws().pres.ptr, m.ws().counters.ptr + 2,
                                       static_cast<long long>(m.ws().cap_pool), m.stats_on ? m.stats.ptr : nullptr);
    ARFX_CUDA(cudaGetLastError());
    m.prof.end(s);
    return;
  }
#endif
  const size_t tile_bytes = static_cast<size_t>(2 * TcSmem::A0P);
  m.ws().tc_tiles.ensure(static_cast<size_t>((m.ws().cap_pool + kTcTile - 1) / kTcTile + 1) * tile_bytes);
  m.prof.begin("encode_tc", s);
  auto enc = half ? encode_tiles_kernel<true> : encode_tiles_kernel<false>;
  enc<<<resident_grid(enc, kEncThreads, 0, n_hint), kEncThreads, 0, s>>>(m.fv, m.grid_h2.ptr, m.ws().px.ptr, m.ws().py.ptr, m.ws().pz.ptr, m.ws().powner.ptr,
                                     m.ws().counters.ptr + 2, static_cast<long long>(m.ws().cap_pool), m.ws().tc_tiles.ptr,
                                     m.stats_on ? m.stats.ptr : nullptr);
  ARFX_CUDA(cudaGetLastError());
  m.prof.end(s);
  m.prof.begin("field_tc", s);
  field_tc_kernel<<<grid, kTcThreads, smem, s>>>(m.fv, m.ws().tc_tiles.ptr, m.ws().powner.ptr, m.ws().pres.ptr,
                                              m.ws().counters.ptr + 2, static_cast<long long>(m.ws().cap_pool));
  ARFX_CUDA(cudaGetLastError());
  m.prof.end(s);
}

}  // namespace arfx
