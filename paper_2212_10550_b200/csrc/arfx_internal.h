// arfx_internal.h -- plain structs shared by the host runtime (host.cpp, abi.cu)
// and the sm_100a kernels. Layouts follow the reference's containers so the
// C-ABI can upload/download them without reshaping (SURVEY.md §8b "Ownership"):
//   hash grid  [L][2^T][F] f32          R/hash_grid.hpp:62
//   MLP        per layer W[out][in], b  R/mlp.hpp:40-48
//   skinning   [z][y][x][bone] f64      R/skinning.hpp:16
//   occupancy  [z][y][x] f32 + u8       R/occupancy.hpp:42-48
#pragma once

#include <cstddef>
#include <cstdint>

#include <vector_types.h>  // uint2 (host compilers too)

namespace arfx {

constexpr int kMaxBones = 32;   // R/articulation.hpp:10
constexpr int kMaxRoots = 8;    // R/articulation.hpp:11
// multi-GPU ray shards: interleaved tiles of kRowTile image rows (tile % n_shards == shard);
// 4-row tiles keep the per-rank ray counts within one tile (<1 % at 540 rows / 8 ranks)
constexpr int kRowTile = 4;
constexpr int kMaxLevels = 32;
constexpr int kMaxMlpLayers = 9;  // hidden_layers <= 8 (R/mlp.hpp:17) + output layer

enum LevelKind : int { kDirect = 0, kWrap = 1, kHashed = 2 };  // R/hash_grid.hpp:87-101

// Canonical field (HashGrid + DecoderMlp), device pointers.
struct FieldView {
  int L, F, log2T;
  uint32_t T;
  int res[kMaxLevels];
  int kind[kMaxLevels];
  double lo[3], hi[3], e[3];  // bounding box, e = hi - lo (Aabb::extent)
  const float* grid;          // [L][T][F]
  int n_layers;               // hidden_layers + 1
  int lin[kMaxMlpLayers], lout[kMaxMlpLayers];
  int w_off[kMaxMlpLayers], b_off[kMaxMlpLayers];
  int in_dim, hidden, out_dim, n_mlp;
  const float* mlp;
};

// SkinningGrid (R/skinning.hpp:12-56) plus the per-cell packed table the deformer
// reads: for cell c, the bones with a nonzero node weight at any of its 8 corners
// (bitmask, ascending bone order) and, per such bone, the 8 corner node weights in
// corner order k = 0..7 (k bit0 = x, bit1 = y, bit2 = z).
struct SkinView {
  int rx, ry, rz, nb;
  double lo[3], hi[3], e[3];
  const double* weights;     // [z][y][x][bone]
  const uint32_t* cell_mask; // [(rz-1)(ry-1)(rx-1)]
  const uint32_t* cell_off;  // offset into cell_vals in units of 8 doubles
  const double* cell_vals;
  const uint2* cell_mo;      // (cell_mask, cell_off) pairs: one load per eval
};

// PoseContext (R/articulation.hpp:17-42) + world->normalized rigid (R/model.hpp:85-98).
// Rigid = R row-major (9) then t (3).
// A sorted Newton start: target | bone << 26, and (ARFX_ITEMS64) its result slot in the high
// word, so the Newton refill needs no slot-base / mask loads
#ifndef ARFX_ITEMS64
#define ARFX_ITEMS64 1
#endif
#if ARFX_ITEMS64
using StartItem = unsigned long long;
#else
using StartItem = uint32_t;
#endif

struct PoseCtx {
  int nb;
  int pad_;
  double bone[kMaxBones][12];
  double bone_inv[kMaxBones][12];
  double cap_a[kMaxBones][3];
  double cap_b[kMaxBones][3];
  double cutoff[kMaxBones];
  double w2n[12];
  // Conservative f32 bounding sphere of each posed capsule's start region: centre and
  // (half length + cutoff + 1e-4 m)^2. A target outside it is provably farther than the
  // cutoff from the segment (triangle inequality), so the exact FP64 distance test of
  // R/articulation.hpp:101-102 is only run for bones whose sphere contains the target.
  float sph[kMaxBones][4];
};

struct InverseOpts {  // R/articulation.hpp:84-88
  int max_iterations;
  double tolerance;
  double dedup_radius;
};

struct OccView {
  int rx, ry, rz;
  double lo[3], hi[3], e[3];
  double inv_e[3];  // RN(1/e): fast path of the cell decision (render.cu cell_axis_fast)
  const uint8_t* mask;
};

struct CameraView {  // R/camera.hpp:9-13
  double fx, fy, cx, cy;
  int width, height;
  double ext[12];
};

// arf::CapsuleFigure (R/scene.hpp:13-27) posed by PosedFigure (R/scene.hpp:56-75): per bone
// the (posed or canonical) segment, radius, color, amplitude; the analytic ground truth.
struct FigureView {
  int nb;
  int pad_;
  double a[kMaxBones][3], b[kMaxBones][3];
  double radius[kMaxBones], amp[kMaxBones];
  double col[kMaxBones][3];
  double soft;
};

}  // namespace arfx
