/*
 * arfx.h -- C-ABI of the B200-native InstantAvatar render/train hot path
 * (libarfx.so, paper_2212_10550_b200/lib/). Plain pointers and sizes only.
 *
 * Each entry point replaces one model-bound operation of the reference C++
 * library `arf` (/root/reference/proj/include/arf, cited as R/...):
 *
 *   arfx_build_model            <- arf::build_model<float>            R/model.hpp:68-80
 *   arfx_model_create           <- an existing arf::Model<float> (upload of its members:
 *                                  HashGrid::params R/hash_grid.hpp:62, DecoderMlp::params
 *                                  R/mlp.hpp:31, SkinningGrid::weights R/skinning.hpp:16)
 *   arfx_pose_from_joint_rotations <- arf::pose_from_joint_rotations  R/skeleton.hpp:93-110
 *   arfx_pose_create            <- arf::PosedModelView ctor / PoseContext::make
 *                                  R/model.hpp:92-96, R/articulation.hpp:24-41
 *   arfx_render_model           <- arf::render_model                  R/model.hpp:118-135
 *   arfx_build_inference_grid   <- arf::build_model_inference_grid    R/model.hpp:138-148
 *   arfx_update_training_grid   <- arf::update_training_grid bound to
 *                                  PosedModelView::density_normalized R/occupancy.hpp:155-171
 *   arfx_inverse_lbs            <- arf::inverse_lbs_ctx (batched)     R/articulation.hpp:94-145
 *   arfx_posed_query            <- PosedModelView::query_normalized   R/model.hpp:100-107
 *   arfx_field_query            <- CanonicalField::query (batched)    R/field.hpp:75-82
 *   arfx_hash_encode            <- HashGrid::encode (batched)         R/hash_grid.hpp:137-150
 *   arfx_skinning_weights       <- SkinningGrid::interpolate          R/skinning.hpp:25-55
 *   arfx_composite(_backward)   <- arf::composite / composite_backward R/render.hpp:98-157
 *   arfx_field_query_backward   <- CanonicalField::query_backward     R/field.hpp:91-103
 *   arfx_train_fwd_bwd          <- composed training step
 *   arfx_losses / arfx_train_step(_device)  <- SPEC.md:454-489 losses fused into the step
 *   arfx_density_step(_device)  <- SPEC.md:478-484 L_density occupancy regulariser
 *   arfx_adam_step              <- SPEC.md:508-509 optimizer (flat vector, shardable)
 *   arfx_figure_*               <- R/scene.hpp analytic ground truth (SPEC.md scenegen)
 *   arfx_checkpoint_save/load   <- SPEC.md checkpoint file (versioned, bitwise round trip)
 *
 * Error convention (the reference throws; R/math.hpp:12-18): every function
 * returns an int status, 0 = ok, and sets a thread-local message readable via
 * arfx_last_error():
 *   1 std::invalid_argument, 2 arf::DataError, 3 arf::NumericError,
 *   4 std::domain_error, 5 CUDA / runtime failure, 6 no CUDA device.
 * There is NO CPU fallback: compute entry points return 6 without a GPU.
 *
 * Streams: `stream` is a cudaStream_t passed as void*; NULL means the library's
 * per-device non-blocking stream. Host-pointer variants synchronise before they
 * return (same blocking contract as the reference's value-returning API).
 */
#ifndef ARFX_H
#define ARFX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ARFX_MAX_BONES 32 /* arf::kMaxBones  R/articulation.hpp:10 */
#define ARFX_MAX_ROOTS 8  /* arf::kMaxRoots  R/articulation.hpp:11 */
#define ARFX_MAX_LEVELS 32

enum {
  ARFX_OK = 0,
  ARFX_ERR_INVALID_ARGUMENT = 1,
  ARFX_ERR_DATA = 2,
  ARFX_ERR_NUMERIC = 3,
  ARFX_ERR_DOMAIN = 4,
  ARFX_ERR_RUNTIME = 5,
  ARFX_ERR_NO_DEVICE = 6
};

/* ---- plain-data mirrors of the reference's value types ---------------- */

typedef struct { /* arf::Skeleton  R/skeleton.hpp:9-32 (bones in tree order) */
  int n_bones;
  int parent[ARFX_MAX_BONES];
  double head[ARFX_MAX_BONES][3];
  double tail[ARFX_MAX_BONES][3];
  double radius[ARFX_MAX_BONES];
} arfx_skeleton;

typedef struct { /* arf::HashGridConfig  R/hash_grid.hpp:12-32 */
  int levels, features_per_level, table_size_log2, base_resolution, max_resolution;
  double box_lo[3], box_hi[3];
} arfx_grid_config;

typedef struct { /* arf::MlpConfig  R/mlp.hpp:11-23 */
  int input_dim, hidden_dim, hidden_layers, output_dim;
} arfx_mlp_config;

/* arf::Rigidd (R/math.hpp:186-213) is passed as double[12]: rotation row-major
 * (9) followed by translation (3). A SkeletonPose (R/skeleton.hpp:69-88) is
 * bone_transforms double[n_bones][12] plus global_transform double[12]. */

typedef struct { /* arf::Camera  R/camera.hpp:9-49 */
  double fx, fy, cx, cy;
  int width, height;
  double extrinsic[12]; /* world -> camera */
} arfx_camera;

typedef struct { /* arf::OccupancyConfig  R/occupancy.hpp:13-28 */
  int resolution;
  double alpha_threshold;
  int dilation;
  double decay;
  int update_interval;
} arfx_occ_config;

typedef struct { /* arf::RenderOptions  R/render.hpp:159-165 */
  int samples_per_ray;
  int stratified;
  double epsilon_terminate;
  uint64_t seed;
  uint64_t frame_id;
} arfx_render_options;

typedef struct { /* arf::InverseLbsOptions  R/articulation.hpp:84-88 */
  int max_iterations;
  double tolerance;
  double dedup_radius;
} arfx_inverse_options;

typedef struct { /* arf::QueryCounters  R/model.hpp:11-23 */
  uint64_t posed_queries;
  uint64_t canonical_queries;
} arfx_counters;

typedef struct { /* everything arf::Model<float> holds besides the big arrays */
  arfx_skeleton skeleton;
  arfx_grid_config grid;  /* bounding box == canonical box */
  arfx_mlp_config mlp;
  int skin_res[3];
  double skin_lo[3], skin_hi[3];
  double canonical_lo[3], canonical_hi[3];
  double normalized_lo[3], normalized_hi[3];
  arfx_inverse_options inverse;
  size_t n_grid_params, n_mlp_params, n_skin_weights;
} arfx_model_desc;

typedef struct arfx_model_s* arfx_model;      /* device-resident arf::Model<float> */
typedef struct arfx_pose_s* arfx_pose;        /* device-resident PosedModelView   */
typedef struct arfx_occ_s* arfx_occ_grid;     /* device-resident OccupancyGrid    */
typedef struct arfx_frame_graph_s* arfx_frame_graph; /* a captured frame (CUDA graph)   */

/* ---- library / errors ------------------------------------------------ */
const char* arfx_last_error(void);
const char* arfx_version(void);
int arfx_device_count(int* n);
int arfx_set_device(int device);

/* ---- host-side value helpers (no GPU needed) ------------------------- */
int arfx_level_resolutions(const arfx_grid_config* g, int* out_levels);
int arfx_model_sizes(const arfx_skeleton* s, const arfx_grid_config* g, const arfx_mlp_config* m,
                     const int skin_res[3], size_t* n_grid, size_t* n_mlp, size_t* n_skin);
int arfx_pose_from_joint_rotations(const arfx_skeleton* s, const double* joint_rot9,
                                   const double* global12, double* bone_transforms12);
int arfx_camera_look_at(const double eye[3], const double target[3], const double up[3],
                        double focal, int width, int height, arfx_camera* out);
int arfx_pose_context(const arfx_skeleton* s, const double* bone_transforms12, const double* pre12,
                      double cutoff_factor, double* out_bone12, double* out_bone_inv12,
                      double* out_cap_a3, double* out_cap_b3, double* out_cutoff);

/* ---- model ----------------------------------------------------------- */
int arfx_build_model(const arfx_skeleton* s, const arfx_grid_config* g, const arfx_mlp_config* m,
                     const int skin_res[3], uint64_t seed, arfx_model* out);
int arfx_model_create(const arfx_model_desc* desc, const float* grid_params,
                      const float* mlp_params, const double* skin_weights, arfx_model* out);
int arfx_model_destroy(arfx_model m);
int arfx_model_describe(arfx_model m, arfx_model_desc* out);
int arfx_model_get_params(arfx_model m, float* grid_params, float* mlp_params,
                          double* skin_weights);
int arfx_model_set_params(arfx_model m, const float* grid_params, const float* mlp_params);
/* Decoder used by arfx_render_model*: ARFX_MLP_EXACT (default) = f32 SIMT with the
 * reference's summation order; ARFX_MLP_TCGEN05 = hash encode fused with the MLP's hidden
 * layers on tcgen05.mma (kind::f16 on split-bf16 operands, f32 accumulate in TMEM) and the
 * 64 -> 4 head in f32; ARFX_MLP_TCGEN05_FP16 = the same decoder fed by fp16 hash-table
 * gathers (an fp16 copy of the table is refreshed at every render: half the gather bytes).
 * The tensor-core modes are stated to 1e-3 relative on rendered RGB;
 * occupancy grids, training and the query APIs always use the exact decoder. */
enum { ARFX_MLP_EXACT = 0, ARFX_MLP_TCGEN05 = 1, ARFX_MLP_TCGEN05_FP16 = 2 };
int arfx_model_set_mlp_mode(arfx_model m, int mode);
/* MLP part of the training backward (query_backward R/field.hpp:91-103, R/mlp.hpp:116-154):
 * ARFX_BWD_TCGEN05 (default) = dX = delta . W and dW = sum delta^T . [inputs | 1] as split-bf16
 * tcgen05.mma with f32 accumulation in TMEM (gradients within 1e-4 relative of the reference,
 * DESIGN.md §5); ARFX_BWD_SIMT = f32 SIMT in the reference's summation order. The tcgen05
 * path needs the forward's saved activations (batches of <= 65,536 field queries); larger
 * batches use the SIMT path. Deterministic either way under arfx_model_set_deterministic. */
enum { ARFX_BWD_SIMT = 0, ARFX_BWD_TCGEN05 = 1 };
int arfx_model_set_backward_mode(arfx_model m, int mode);
/* Deterministic gradients (default off): the field backward visits the flagged queries in
 * owner order (rays front to back / points) instead of atomic-compaction order, so the f32
 * MLP weight-gradient sums are fixed, and the hash-grid scatter sums fixed-point int64
 * contributions (each rounded to a multiple of 2^-46) instead of f32 atomics. Repeated
 * train/density steps on the same inputs then give bit-identical gradients, Adam states
 * and parameters. The grid sums stay in an accumulator until consumed: arfx_adam_step over
 * the whole flat vector folds them in during its sweep, arfx_model_get_grads flushes them;
 * code that reads the gradient arrays directly (arfx_model_device_arrays / arfx_model_flat,
 * e.g. a data-parallel reduce-scatter) calls arfx_model_flush_grads first (async on
 * `stream`). arfx_model_zero_grad discards pending sums. */
int arfx_model_set_deterministic(arfx_model m, int on);
int arfx_model_flush_grads(arfx_model m, void* stream);
/* Optimizer on its own stream: every kernel of this model that reads the parameters or
 * writes the gradients (field forward / backward, gradient flush) first waits on `event`
 * (a cudaEvent_t the caller records after each optimizer step; NULL clears). The trainer
 * uses it to run Adam of step t concurrently with the march and deformer of step t+1,
 * which read neither. Host-buffer APIs do not wait on it: synchronise the optimizer's
 * stream before them. */
int arfx_model_set_param_fence(arfx_model m, void* event);
int arfx_model_zero_grad(arfx_model m, void* stream);
int arfx_model_get_grads(arfx_model m, float* grid_grad, float* mlp_grad);
/* device pointers of the parameter / gradient arrays (for NCCL / optimizers) */
int arfx_model_device_arrays(arfx_model m, float** grid_params, float** mlp_params,
                             float** grid_grad, float** mlp_grad);

/* ---- pose (PosedModelView: normalized-space PoseContext) --------------- */
int arfx_pose_create(arfx_model m, const double* bone_transforms12, const double* global12,
                     arfx_pose* out);
int arfx_pose_update(arfx_pose p, const double* bone_transforms12, const double* global12,
                     void* stream);
/* arfx_pose_update without the stream synchronisation: the PoseContext is staged in a
 * pinned ring and copied on `stream` (kernels enqueued earlier still see the old pose);
 * the host arrays may be reused on return. */
int arfx_pose_update_async(arfx_pose p, const double* bones12, const double* global12, void* stream);
int arfx_pose_destroy(arfx_pose p);

/* ---- occupancy grid ---------------------------------------------------- */
int arfx_occ_create(const double box_lo[3], const double box_hi[3], const arfx_occ_config* cfg,
                    arfx_occ_grid* out); /* OccupancyGrid::empty  R/occupancy.hpp:59-69 */
int arfx_occ_destroy(arfx_occ_grid g);
/* an OccupancyGrid from its stored members (density threshold, not alpha; checkpoint restore) */
int arfx_occ_create_raw(const double box_lo[3], const double box_hi[3], int resolution, double density_threshold,
                        int dilation, arfx_occ_grid* out);
int arfx_occ_info(arfx_occ_grid g, int res[3], double box_lo[3], double box_hi[3],
                  double* density_threshold, int* dilation);
int arfx_occ_download(arfx_occ_grid g, float* values, uint8_t* mask);
int arfx_occ_upload(arfx_occ_grid g, const float* values, const uint8_t* mask);
int arfx_occ_rebuild_mask(arfx_occ_grid g, void* stream); /* R/occupancy.hpp:87-91 */
/* OccupancyGrid::is_occupied (R/occupancy.hpp:81-85) over a batch of normalized points */
int arfx_occ_is_occupied(arfx_occ_grid g, const double* pts, int64_t n, uint8_t* out);
/* build_model_inference_grid (R/model.hpp:138-148). With c != NULL it synchronises and
 * reports the query counters; with c == NULL it reserves worst-case workspace and returns
 * without a host round trip (the grid is complete for later work on the same stream; the
 * host-buffer accessors arfx_occ_download / arfx_render_model synchronise). */
int arfx_build_inference_grid(arfx_model m, arfx_pose p, arfx_occ_grid g, arfx_counters* c,
                              void* stream);
/* asynchronous variant: counters (u64 x4: posed, canonical, pool, overflow) to device memory */
int arfx_build_inference_grid_device(arfx_model m, arfx_pose p, arfx_occ_grid g,
                                     uint64_t* d_counters, void* stream);
/* Multi-GPU: the inference grid's cell values for shard `shard` of
 * `n_shards` only -- the cell-interleaved cells c = shard + n_shards*j (j < cells/n_shards;
 * res^3 must divide by n_shards), written as the rank-major block values[shard*cells/n + j].
 * All-gather the blocks in place across ranks (arfx_occ_device_arrays), then
 * arfx_occ_rebuild_mask_shards_async permutes them into cell order and rebuilds the mask.
 * Per-cell values are bit-identical to the full build. */
int arfx_build_inference_grid_shard_device(arfx_model m, arfx_pose p, arfx_occ_grid g, int shard, int n_shards,
                                           uint64_t* d_counters, void* stream);
/* device pointers of the occupancy values [z][y][x] f32 and mask u8 */
int arfx_occ_device_arrays(arfx_occ_grid g, float** values, uint8_t** mask);
/* threshold + dilation of the current values, asynchronous on stream */
int arfx_occ_rebuild_mask_async(arfx_occ_grid g, void* stream);
/* values hold n_shards rank-major shard blocks (arfx_build_inference_grid_shard_device, then
 * an all-gather): permute them into [z][y][x] cell order, then threshold + dilation. */
int arfx_occ_rebuild_mask_shards_async(arfx_occ_grid g, int n_shards, void* stream);
/* Asynchronous variant (no host round trip): the workspace is reserved for the worst case
 * (every bone a start, kMaxRoots roots per cell), so it cannot overflow; counters (u64 x4)
 * to device memory when d_counters != NULL. */
int arfx_update_training_grid_device(arfx_model m, const arfx_pose* poses, int n_poses, double decay,
                                     uint64_t seed, uint64_t step, arfx_occ_grid g, uint64_t* d_counters,
                                     void* stream);
int arfx_update_training_grid(arfx_model m, const arfx_pose* poses, int n_poses, double decay,
                              uint64_t seed, uint64_t step, arfx_occ_grid g, arfx_counters* c,
                              void* stream);

/* ---- render ------------------------------------------------------------- */
/* Host buffers: rgb[H*W*3], alpha[H*W] (arf::RenderImages layout R/render.hpp:167-171).
 * occ may be NULL (no skipping). row_shard/n_shards select interleaved 4-row tiles
 * (tile % n_shards == row_shard) for multi-GPU sharding; use 0/1 for a full frame --
 * rows of other shards are left untouched. */
int arfx_render_model(arfx_model m, arfx_pose p, const arfx_camera* cam, arfx_occ_grid occ,
                      const arfx_render_options* opt, int row_shard, int n_shards, float* rgb,
                      float* alpha, arfx_counters* c, void* stream);
/* Device buffers, asynchronous on `stream`; counters (2 x u64) written to device memory. */
int arfx_render_model_device(arfx_model m, arfx_pose p, const arfx_camera* cam,
                             arfx_occ_grid occ, const arfx_render_options* opt, int row_shard,
                             int n_shards, float* d_rgb, float* d_alpha, uint64_t* d_counters,
                             void* stream);
/* arfx_render_model with host buffers but no host round trip (pipelines frames): the frame
 * renders on `stream` into one of two library-owned device image slots and this shard's
 * rows, plus counters4 = (posed, canonical, pool, overflow), are copied to the host buffers
 * on a library copy stream while the next frame renders. The host buffers (pinned for
 * overlap) are valid after arfx_render_wait. counters4[3] != 0: the workspace overflowed,
 * re-render that frame with arfx_render_model (which grows it). */
int arfx_render_model_async(arfx_model m, arfx_pose p, const arfx_camera* cam, arfx_occ_grid occ,
                            const arfx_render_options* opt, int shard, int n_shards, float* rgb, float* alpha,
                            uint64_t* counters4, void* stream);
/* Pipelined animation through host buffers: builds the inference grid of the NEXT pose
 * (p_next -> occ_next, side stream + side workspace) while the CURRENT pose renders with its
 * already-built grid (p_cur, occ_cur) into host buffers exactly as arfx_render_model_async;
 * later work on `stream` waits for the new grid. Alternate the two (pose, grid) pairs frame
 * by frame; results are identical to arfx_build_inference_grid + arfx_render_model.
 * Internally each (handles, camera, options, shard, image slot, stream) combination is
 * captured once as a CUDA graph and replayed (up to 8 are cached per model; the first call of
 * a combination renders the frame twice, and a capture is renewed after workspace growth). */
int arfx_render_model_pipelined_async(arfx_model m, arfx_pose p_cur, arfx_occ_grid occ_cur, arfx_pose p_next,
                                      arfx_occ_grid occ_next, const arfx_camera* cam,
                                      const arfx_render_options* opt, int row_shard, int n_shards, float* rgb,
                                      float* alpha, uint64_t* counters4, void* stream);
int arfx_render_wait(arfx_model m);
/* Trace of the last render on this model (posed-sample list), for parity tests:
 * per posed sample: pixel, sample index, has_root, density, rgb, canonical root. */
int arfx_render_trace(arfx_model m, int64_t capacity, int64_t* n_samples, int32_t* s_ray,
                      int32_t* s_index, uint8_t* s_has_root, float* s_density, float* s_color,
                      double* s_canonical, double* s_delta);

/* ---- per-kernel timing (CUDA events on the launching stream; for bench/roofline) */
int arfx_profile_enable(arfx_model m, int on);
/* collects (synchronising on the recorded events), returns and resets the totals:
 * names[max][32], total ms and launch count per kernel name; *n = entries written */
int arfx_profile_read(arfx_model m, int max, char* names, double* ms, int64_t* launches, int* n);

/* deterministic work counters for roofline accounting (off by default):
 * out[0] skinning evals, [1] union-bone visits, [2] Newton steps, [3] starts,
 * [4] exact prune distance tests, [5] field queries (exact SIMT decoder), [6] field queries (tcgen05 decoder). arfx_stats_read resets them. */
int arfx_stats_enable(arfx_model m, int on);
int arfx_stats_read(arfx_model m, uint64_t* out16);
/* measured FP64 / FP32 add+mul issue roofs of this GPU (TFLOP/s, 1 flop per add or mul) */
int arfx_pipe_peaks(double* fp64_tflops, double* fp32_tflops);

/* ---- batched lower-level operations (host arrays in/out) ---------------- */
int arfx_skinning_weights(arfx_model m, const double* pts, int64_t n, double* w /*n*n_bones*/);
/* pose context built with `pre` and cutoff factor exactly as PoseContext::make;
 * roots[n][8][3], residuals[n][8], counts[n] */
int arfx_inverse_lbs(arfx_model m, const double* bone_transforms12, const double* pre12,
                     double cutoff_factor, const double* pts, int64_t n, int32_t* counts,
                     double* roots, double* residuals);
/* device-pointer variant for the correspondence microbench (pts/counts/roots/residuals on device) */
int arfx_inverse_lbs_device(arfx_model m, arfx_pose ctx_pose, const double* d_pts, int64_t n,
                            int32_t* d_counts, double* d_roots, double* d_residuals,
                            void* stream);
int arfx_pose_create_context(arfx_model m, const double* bone_transforms12, const double* pre12,
                             double cutoff_factor, arfx_pose* out);
int arfx_hash_encode(arfx_model m, const double* pts, int64_t n, float* feats);
int arfx_field_query(arfx_model m, const double* pts, int64_t n, float* density, float* color);
int arfx_posed_query(arfx_model m, arfx_pose p, const double* pts_norm, int64_t n,
                     float* density, float* color, double* canonical, uint8_t* has_root,
                     arfx_counters* c);
int arfx_composite(int n_rays, const int32_t* ray_len, const double* t, const double* delta,
                   const uint8_t* skipped, const float* density, const float* color,
                   double epsilon, double* out_color3, double* out_alpha, int32_t* terminated_at);
int arfx_composite_backward(int n_rays, const int32_t* ray_len, const double* t,
                            const double* delta, const uint8_t* skipped, const float* density,
                            const float* color, double epsilon, const double* d_color3,
                            const double* d_alpha, double* d_sigma, double* d_c3);
/* accumulates into the model's device gradient buffers (FieldGrads  R/field.hpp:19-36) */
int arfx_field_query_backward(arfx_model m, const double* pts, int64_t n, const float* d_density,
                              const float* d_color);
/* training forward+backward over n rays given by pixel coordinates; accumulates into
 * the model's gradient buffers; rgb/alpha per ray to host (may be NULL). */
int arfx_train_fwd_bwd(arfx_model m, arfx_pose p, const arfx_camera* cam, arfx_occ_grid occ,
                       const arfx_render_options* opt, int64_t n_rays, const int32_t* px,
                       const int32_t* py, const float* d_color, const float* d_alpha, float* rgb,
                       float* alpha, arfx_counters* c, void* stream);

/* ---- training: losses, fused step, optimizer -- */

typedef struct arfx_loss_config { /* LossWeights SPEC.md:446-449; defaults :510 */
  double w_rgb, w_alpha, w_hard, w_density; /* 1, 0.1, 0.1, 0.1 */
  double huber_delta;                       /* 0.1 */
  /* 0 (default): gt_rgb / gt_alpha hold one target per ray. > 0 (device train steps only):
   * they hold whole ground-truth frames [gt_height][gt_width] (row-major, rgb interleaved)
   * and ray r reads the target at its pixel (py[r], px[r]) inside the composite kernel
   * (a pixel outside the frame reads target 0). */
  int64_t gt_width, gt_height;
} arfx_loss_config;

typedef struct arfx_adam_config {
  double lr_grid, lr_mlp; /* 1e-2, 1e-3 */
  double beta1, beta2;    /* 0.9, 0.99 */
  double eps;             /* 1e-15 */
  int64_t total_steps;    /* cosine decay horizon T (<= 0: constant lr) */
  double final_lr_factor; /* lr(T) / lr(0) */
} arfx_adam_config;

/* Per-ray losses on rendered (rgb, alpha) vs targets: loss4 = (L_rgb, L_alpha, L_hard,
 * weighted total) as batch means, and the f32 upstream gradients dL/dC [n][3], dL/dA [n]
 * (any output may be NULL). Host buffers. */
int arfx_losses(int64_t n, const float* rgb, const float* alpha, const float* gt_rgb, const float* gt_alpha,
                const arfx_loss_config* cfg, double* loss4, float* d_rgb, float* d_alpha);
/* Fused training step over n rays: forward (as arfx_train_fwd_bwd), the losses evaluated
 * per ray inside the composite kernel against gt_rgb/gt_alpha, their gradient fed straight
 * into the composite reverse pass, field backward -> accumulated into the model's
 * gradients. loss4 as arfx_losses. Host buffers (synchronous). */
int arfx_train_step(arfx_model m, arfx_pose p, const arfx_camera* cam, arfx_occ_grid occ,
                    const arfx_render_options* opt, int64_t n_rays, const int32_t* px, const int32_t* py,
                    const float* gt_rgb, const float* gt_alpha, const arfx_loss_config* cfg, double* loss4,
                    float* rgb, float* alpha, arfx_counters* c, void* stream);
/* The same on device arrays (d_loss4: 4 doubles on the device; d_rgb/d_alpha may be NULL).
 * Fully asynchronous on `stream` (n_rays * samples_per_ray <= 2^22): workspace capacity is
 * reserved for the worst case instead of checked on the host; pixel coordinates are not
 * range-checked (an out-of-image pixel yields its ray, no out-of-bounds access). */
int arfx_train_step_device(arfx_model m, arfx_pose p, const arfx_camera* cam, arfx_occ_grid occ,
                           const arfx_render_options* opt, int64_t n_rays, const int32_t* d_px,
                           const int32_t* d_py, const float* d_gt_rgb, const float* d_gt_alpha,
                           const arfx_loss_config* cfg, double* d_loss4, float* d_rgb, float* d_alpha,
                           void* stream);
/* L_density (Eq. 12): n points uniform in the normalized box, point i
 * drawn from keyed_rng(seed, 0xde45, step, i) (x, y, z); those in EMPTY cells of `occ`
 * are posed-queried (R/articulation.hpp:163-181); loss2 = (L_density = mean |sigma| over
 * them, n_empty); w_density * dL/dtheta accumulated into the model's gradients. */
int arfx_density_step(arfx_model m, arfx_pose p, arfx_occ_grid occ, int64_t n_points, uint64_t seed,
                      uint64_t step, const arfx_loss_config* cfg, double* loss2, void* stream);
int arfx_density_step_device(arfx_model m, arfx_pose p, arfx_occ_grid occ, int64_t n_points, uint64_t seed,
                             uint64_t step, const arfx_loss_config* cfg, double* d_loss2, void* stream);
/* arfx_train_step_device + arfx_density_step_device in one call (same results): the
 * L_density forward runs on a library-owned side stream with its own workspace,
 * concurrently with the train step; its backward joins on `stream` after the train
 * backward. n_points <= 0 skips the density step. */
int arfx_train_density_step_device(arfx_model m, arfx_pose pose, const arfx_camera* cam, arfx_occ_grid occ,
                                   const arfx_render_options* opt, int64_t n_rays, const int32_t* d_px,
                                   const int32_t* d_py, const float* d_gt_rgb, const float* d_gt_alpha,
                                   const arfx_loss_config* cfg, double* d_loss4, int64_t n_points,
                                   uint64_t seed, uint64_t step, double* d_loss2, void* stream);
/* The same step split in two, for pipelining across steps: arfx_train_forward_device runs
 * the march, deformer and field forward of n rays into train slot 0 or 1 (its field kernels
 * wait on the parameter fence, nothing else reads parameters or gradients);
 * arfx_train_backward_device then runs that slot's composite + fused losses + field
 * backward (+ the L_density step when n_points > 0), accumulating into the gradients. The
 * caller orders them (events): backward(slot) after forward(slot), and a slot's next
 * forward after its previous backward. Capacities are reserved for the worst case. */
/* The trainer's ray batch of one step on the device: ray i's pixel from draws 1 + 2i, 2 + 2i
 * of keyed_rng(seed, 0x7a11, step, rank) (draw 0, the frame index, is the caller's). */
int arfx_train_rays_device(uint64_t seed, uint64_t step, uint64_t rank, int64_t n, int width, int height,
                           int32_t* d_px, int32_t* d_py, void* stream);
int arfx_train_forward_device(arfx_model m, arfx_pose pose, const arfx_camera* cam, arfx_occ_grid occ,
                              const arfx_render_options* opt, int64_t n_rays, const int32_t* d_px,
                              const int32_t* d_py, int slot, void* stream);
int arfx_train_backward_device(arfx_model m, arfx_pose pose, arfx_occ_grid occ, const arfx_render_options* opt,
                               int64_t n_rays, const int32_t* d_px, const int32_t* d_py, const float* d_gt_rgb,
                               const float* d_gt_alpha, const arfx_loss_config* cfg, double* d_loss4, int slot,
                               int64_t n_points, uint64_t seed, uint64_t step, double* d_loss2, void* stream);
/* Adam over flat parameter indices [begin, end) (multiples of 4; end = -1: all), step >= 1,
 * gradients zeroed in the same pass. Asynchronous on stream. */
int arfx_adam_step(arfx_model m, const arfx_adam_config* cfg, int64_t step, int64_t begin, int64_t end,
                   void* stream);
/* arfx_adam_step behind a non-finite-loss guard: d_loss = the step's n_loss
 * loss values (device); if any is non-finite, or *d_bad (device int, sticky) is already set,
 * the step changes nothing and *d_bad = 1. The caller reads *d_bad when convenient and aborts
 * with the model still at its last finite state. */
int arfx_adam_step_guarded(arfx_model m, const arfx_adam_config* cfg, int64_t step, int64_t begin, int64_t end,
                           const double* d_loss, int n_loss, int* d_bad, void* stream);
/* Flat device vectors [grid | pad | mlp | pad] of n_flat floats: params, grads, Adam m, v
 * (allocated on first use); mlp_offset = index of the first MLP parameter. */
int arfx_model_flat(arfx_model m, float** params, float** grads, float** adam_m, float** adam_v,
                    int64_t* n_flat, int64_t* mlp_offset);
/* Host copies of the flat Adam moments (n_flat floats each; checkpoint / resume). */
int arfx_model_get_adam(arfx_model m, float* adam_m, float* adam_v);
int arfx_model_set_adam(arfx_model m, const float* adam_m, const float* adam_v);

/* ---- CUDA-graph frames ---------------------------------------------------------------- */

enum {
  ARFX_GRAPH_GRID = 1,
  ARFX_GRAPH_GRID_SHARD = 2,
  ARFX_GRAPH_MASK = 4,
  ARFX_GRAPH_RENDER = 8,
  ARFX_GRAPH_MASK_SHARDS = 16, /* as arfx_occ_rebuild_mask_shards_async(occ, nshards) */
  ARFX_GRAPH_SIDE_WORKSPACE = 64 /* capture on the side workspace: may run beside a main-workspace graph */
};
/* Captures the chosen parts of one frame for pose handle p as a CUDA graph: the inference
 * grid (GRID) or its z-slab shard (GRID_SHARD), the mask rebuild (MASK), the render into
 * device buffers (RENDER). d_counters [2][4] (grid, render: posed, canonical, pool, overflow)
 * is required for the GRID / GRID_SHARD / RENDER parts: a replay cannot grow the workspace,
 * so a frame that overflowed it sets d_counters[3] / d_counters[4 + 3] != 0 and must be
 * re-rendered through the synchronous API. Every kernel reads the pose from its device
 * PoseContext, so after updating the handle in place (arfx_pose_update, arfx_pose_copy) a
 * replay renders the new pose. `stream` must be non-NULL (capture). The graph holds raw
 * pointers into the model's workspace: any later workspace growth (a larger render, another
 * camera or shard, an overflow regrow) invalidates it, and arfx_frame_graph_launch then
 * returns 1 (invalid_argument) instead of replaying -- destroy and re-create the graph. */
int arfx_frame_graph_create(arfx_model m, arfx_pose p, const arfx_camera* cam, arfx_occ_grid occ,
                            const arfx_render_options* opt, int shard, int n_shards, int parts, float* d_rgb,
                            float* d_alpha, uint64_t* d_counters, void* stream, arfx_frame_graph* out);
/* Pipelined animation frame: one graph with two concurrent branches -- the inference grid of
 * the NEXT pose (p_next -> occ_next, side stream and workspace) and the render of the
 * CURRENT pose with its already-built grid (p_cur, occ_cur). Alternate two such graphs with
 * the (pose, grid) roles swapped: each frame's grid build overlaps the previous frame's
 * render, every frame bit-identical to a direct grid + render. d_counters [2][4] required
 * (next grid, render). Same invalidation rule as arfx_frame_graph_create. */
int arfx_frame_graph_create_pipelined(arfx_model m, arfx_pose p_cur, arfx_occ_grid occ_cur, arfx_pose p_next,
                                      arfx_occ_grid occ_next, const arfx_camera* cam,
                                      const arfx_render_options* opt, int shard, int nshards, float* d_rgb,
                                      float* d_alpha, uint64_t* d_counters, void* stream,
                                      arfx_frame_graph* out);
int arfx_frame_graph_launch(arfx_frame_graph g, void* stream);
int arfx_frame_graph_destroy(arfx_frame_graph g);
/* dst <- src (same model): host and device PoseContext, asynchronous on stream */
int arfx_pose_copy(arfx_pose dst, arfx_pose src, void* stream);

/* ---- checkpoint / wire format --- */

/* Versioned little-endian binary: magic "ARFXCKPT", u32 version (1), then the model
 * description (skeleton, grid / MLP configs, skinning resolution + boxes, canonical and
 * normalized boxes, inverse-LBS options), the parameter arrays in the reference layouts
 * (grid [L][2^T][F] f32, MLP W/b f32, skinning [z][y][x][bone] f64), optionally the
 * occupancy grid (resolution, box, density threshold, dilation, values f32, mask u8) and
 * the optimizer state (step, Adam m / v over the flat vector), then an FNV-1a 64 checksum
 * of everything before it. Round trips are bitwise. */
int arfx_checkpoint_save(const char* path, arfx_model m, arfx_occ_grid occ /* may be NULL */, int64_t step,
                         int with_optimizer);
/* Creates a model (and the occupancy grid when present and occ_out != NULL); restores the
 * Adam moments when present. Errors: 2 (DataError) for a malformed / corrupt file. */
int arfx_checkpoint_load(const char* path, arfx_model* m_out, arfx_occ_grid* occ_out, int64_t* step_out);

/* ---- analytic ground truth (SPEC.md scenegen; R/scene.hpp) -------------------------- */

typedef struct arfx_figure { /* arf::CapsuleFigure  R/scene.hpp:13-27 */
  arfx_skeleton skeleton;
  double color[ARFX_MAX_BONES][3];
  double amplitude[ARFX_MAX_BONES];
  double softness;
} arfx_figure;

/* bones12 == NULL: analytic_query in canonical space (R/scene.hpp:31-50); else the posed
 * field PosedFigure(fig, pose).query (R/scene.hpp:56-97). density[n], color[n][3]. */
int arfx_figure_query(const arfx_figure* fig, const double* bones12, const double* pts, int64_t n,
                      double* density, double* color);
/* Ground-truth frame: render_image (R/render.hpp:178-218) of PosedFigure::query (matter iff
 * density > 0), to_norm = global^-1, box = the model's normalized box, no occupancy; plus
 * the exact silhouette PosedFigure::ray_hits (R/scene.hpp:123-130) per pixel. Host buffers
 * rgb[H][W][3], alpha[H][W], mask[H][W] (any may be NULL). */
int arfx_figure_render(const arfx_figure* fig, const double* bones12, const double* global12,
                       const double box_lo[3], const double box_hi[3], const arfx_camera* cam,
                       const arfx_render_options* opt, float* rgb, float* alpha, uint8_t* mask, void* stream);
/* The same for n rays given by device pixel lists; device outputs; asynchronous on stream. */
int arfx_figure_render_rays_device(const arfx_figure* fig, const double* bones12, const double* global12,
                                   const double box_lo[3], const double box_hi[3], const arfx_camera* cam,
                                   const arfx_render_options* opt, int64_t n, const int32_t* d_px,
                                   const int32_t* d_py, float* d_rgb, float* d_alpha, uint8_t* d_mask,
                                   void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ARFX_H */
