/*
 * oracle_api.h -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * One plain-C API, implemented twice:
 *   arfo_*  : oracle/arf_oracle.c, a from-scratch C restatement of the
 *             reference's per-ray render/train path (each function cites the
 *             reference file:line it follows);
 *   arfr_*  : oracle/ref_driver.cpp, a thin extern "C" shim over the UNMODIFIED
 *             reference headers (/root/reference/proj/include/arf), compiled in
 *             place into oracle/_ref/libarf_ref.so.
 * The parity tests load both and the product (libarfx.so) and compare them.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
 * this. All structs are plain data, layouts identical to include/arfx.h's.
 */
#ifndef ARF_ORACLE_API_H
#define ARF_ORACLE_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AO_MAX_BONES 32 /* arf::kMaxBones, R/articulation.hpp:10 */
#define AO_MAX_ROOTS 8  /* arf::kMaxRoots, R/articulation.hpp:11 */

/* Status codes (same as arfx.h): 0 ok, 1 invalid_argument, 2 DataError,
 * 3 NumericError, 4 domain_error, 5 runtime/other. */

typedef struct { /* arf::Skeleton, R/skeleton.hpp:9-32 */
  int n_bones;
  int parent[AO_MAX_BONES];
  double head[AO_MAX_BONES][3];
  double tail[AO_MAX_BONES][3];
  double radius[AO_MAX_BONES];
} ao_skeleton;

typedef struct { /* arf::HashGridConfig, R/hash_grid.hpp:12-32 */
  int levels, features_per_level, table_size_log2, base_resolution, max_resolution;
  double box_lo[3], box_hi[3];
} ao_grid_cfg;

typedef struct { /* arf::MlpConfig, R/mlp.hpp:11-23 */
  int input_dim, hidden_dim, hidden_layers, output_dim;
} ao_mlp_cfg;

typedef struct { /* arf::Camera, R/camera.hpp:9-49; extrinsic = R(9, row-major) t(3) */
  double fx, fy, cx, cy;
  int width, height;
  double extrinsic[12];
} ao_camera;

typedef struct { /* arf::OccupancyConfig, R/occupancy.hpp:13-28 */
  int resolution;
  double alpha_threshold;
  int dilation;
  double decay;
  int update_interval;
} ao_occ_cfg;

typedef struct { /* arf::RenderOptions, R/render.hpp:159-165 */
  int samples_per_ray;
  int stratified;
  double epsilon_terminate;
  uint64_t seed;
  uint64_t frame_id;
} ao_render_opts;

typedef struct { /* arf::Model<float>, R/model.hpp:28-57 (arrays caller-owned) */
  ao_skeleton skel;
  ao_grid_cfg grid;   /* bounding box == canonical box after build_model */
  ao_mlp_cfg mlp;     /* input_dim == levels * features_per_level */
  int skin_res[3];
  double skin_lo[3], skin_hi[3];
  double canon_lo[3], canon_hi[3];
  double norm_lo[3], norm_hi[3];
  int max_iterations;           /* arf::InverseLbsOptions, R/articulation.hpp:84-88 */
  double tolerance, dedup_radius;
  float* grid_params; size_t n_grid;    /* [L][2^T][F] */
  float* mlp_params; size_t n_mlp;      /* per layer W[out][in] then b[out] */
  double* skin_weights; size_t n_skin;  /* [z][y][x][bone] */
} ao_model;

typedef struct { /* arf::OccupancyGrid, R/occupancy.hpp:37-126 (arrays caller-owned) */
  int res[3];
  double box_lo[3], box_hi[3];
  double density_threshold;
  int dilation;
  float* values;    /* [z][y][x] */
  uint8_t* mask;    /* [z][y][x] */
} ao_occ_grid;

/* Per-sample trace of a render (render_image's loop, R/render.hpp:188-216). */
typedef struct {
  int64_t capacity;   /* in: sample capacity */
  int64_t n_samples;  /* out: number of non-skipped (occupancy-passing) samples */
  int32_t* ray_first; /* [W*H] first sample index (or -1) */
  int32_t* ray_count; /* [W*H] */
  uint8_t* ray_hit;   /* [W*H] */
  double* t_near;     /* [W*H] */
  double* t_far;      /* [W*H] */
  int32_t* terminated_at; /* [W*H] */
  int32_t* s_ray;     /* [cap] pixel index */
  int32_t* s_index;   /* [cap] sample index i in [0,N) */
  uint8_t* s_has_root;/* [cap] */
  float* s_density;   /* [cap] */
  float* s_color;     /* [cap*3] */
  double* s_canonical;/* [cap*3] */
  double* s_t;        /* [cap] */
  double* s_delta;    /* [cap] */
} ao_render_trace;

typedef struct { /* arf::CapsuleFigure, R/scene.hpp:13-27 */
  ao_skeleton skel;
  double color[AO_MAX_BONES][3];
  double amplitude[AO_MAX_BONES];
  double softness;
} ao_figure;

#define AO_API_DECLARE(P)                                                                        \
  const char* P##last_error(void);                                                               \
  int P##model_sizes(const ao_skeleton* s, const ao_grid_cfg* g, const ao_mlp_cfg* m,            \
                     const int skin_res[3], size_t* n_grid, size_t* n_mlp, size_t* n_skin);      \
  int P##build_model(const ao_skeleton* s, const ao_grid_cfg* g, const ao_mlp_cfg* m,            \
                     const int skin_res[3], uint64_t seed, ao_model* out);                       \
  int P##level_resolutions(const ao_grid_cfg* g, int* out);                                      \
  uint32_t P##hash_index(const ao_grid_cfg* g, int level, int cx, int cy, int cz);               \
  int P##pose_from_joint_rotations(const ao_skeleton* s, const double* rot9, const double* g12,  \
                                   double* bones12);                                             \
  int P##look_at(const double eye[3], const double target[3], const double up[3], double focal,  \
                 int w, int h, ao_camera* cam);                                                  \
  int P##skinning_weights(const ao_model* m, const double* pts, int64_t n, double* w);           \
  int P##inverse_lbs(const ao_model* m, const double* bones12, const double* pre12,              \
                     double cutoff_factor, const double* pts, int64_t n, int32_t* counts,        \
                     double* roots, double* residuals);                                          \
  int P##hash_encode(const ao_model* m, const double* pts, int64_t n, float* feats);              \
  int P##field_query(const ao_model* m, const double* pts, int64_t n, float* dens, float* col);  \
  int P##posed_query(const ao_model* m, const double* bones12, const double* global12,           \
                     const double* pts_norm, int64_t n, float* dens, float* col, double* canon,  \
                     uint8_t* has_root);                                                         \
  int P##occ_empty(const double lo[3], const double hi[3], const ao_occ_cfg* c, ao_occ_grid* g); \
  int P##occ_rebuild_mask(ao_occ_grid* g);                                                       \
  int P##build_inference_grid(const ao_model* m, const double* bones12, const double* global12,  \
                              const ao_occ_cfg* c, ao_occ_grid* g, uint64_t* counters);          \
  int P##update_training_grid(const ao_model* m, int n_poses, const double* bones12,             \
                              const double* global12, double decay, uint64_t seed,               \
                              uint64_t step, ao_occ_grid* g, uint64_t* counters);                \
  int P##render(const ao_model* m, const double* bones12, const double* global12,                \
                const ao_camera* cam, const ao_occ_grid* occ, const ao_render_opts* o,           \
                float* rgb, float* alpha, uint64_t* counters);                                   \
  int P##render_trace(const ao_model* m, const double* bones12, const double* global12,          \
                      const ao_camera* cam, const ao_occ_grid* occ, const ao_render_opts* o,     \
                      float* rgb, float* alpha, uint64_t* counters, ao_render_trace* tr);        \
  int P##composite(int n, const double* t, const double* delta, const uint8_t* skipped,          \
                   const float* dens, const float* col, double eps, double* color3,              \
                   double* alpha, int* terminated_at);                                           \
  int P##composite_backward(int n, const double* t, const double* delta, const uint8_t* skipped, \
                            const float* dens, const float* col, double eps,                     \
                            const double* d_color3, double d_alpha, double* d_sigma,             \
                            double* d_c3);                                                       \
  int P##field_query_backward(const ao_model* m, const double* pts, int64_t n,                   \
                              const float* d_dens, const float* d_col, float* grid_grad,         \
                              float* mlp_grad);                                                  \
  int P##train_fwd_bwd(const ao_model* m, const double* bones12, const double* global12,         \
                       const ao_camera* cam, const ao_occ_grid* occ, const ao_render_opts* o,    \
                       int64_t n_rays, const int32_t* px, const int32_t* py,                     \
                       const float* d_color, const float* d_alpha, float* rgb, float* alpha,     \
                       float* grid_grad, float* mlp_grad, uint64_t* counters);                   \
  int P##figure_query(const ao_figure* f, const double* bones12, const double* pts, int64_t n,   \
                      double* dens, double* col);                                                \
  int P##figure_render(const ao_figure* f, const double* bones12, const double* global12,        \
                       const double lo[3], const double hi[3], const ao_camera* cam,             \
                       const ao_render_opts* o, float* rgb, float* alpha, uint8_t* mask);

AO_API_DECLARE(arfo_)
AO_API_DECLARE(arfr_)

/* Training pieces with no reference implementation (SPEC.md:454-530 only; SURVEY.md §8f
 * row 1): restated here from the SPEC text, oracle-only (no arfr_ counterpart). */
typedef struct {
  double w_rgb, w_alpha, w_hard, w_density, huber_delta;
} ao_loss_cfg;
typedef struct {
  double lr_grid, lr_mlp, beta1, beta2, eps;
  int64_t total_steps;
  double final_lr_factor;
} ao_adam_cfg;
int arfo_losses(int64_t n, const float* rgb, const float* alpha, const float* gt_rgb, const float* gt_alpha,
                const ao_loss_cfg* c, double* loss4, float* d_rgb, float* d_alpha);
/* one Adam step over a flat vector; lr_of(i) = i >= mlp_offset ? lr_mlp_t : lr_grid_t */
int arfo_adam(int64_t n, float* p, float* g, float* m, float* v, const ao_adam_cfg* c, int64_t step,
              int64_t mlp_offset);

#ifdef __cplusplus
}
#endif

#endif /* ARF_ORACLE_API_H */
