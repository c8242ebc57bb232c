// host.h -- host-side runtime of libarfx: per-pose / per-model setup that is O(bones)
// or O(levels) and runs once per call (SURVEY.md §2 "Skeleton / FK: host-side").
// Compiled by g++ with -ffp-contract=off so every double matches the reference.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "arfx_internal.h"

struct arfx_skeleton_fwd;

namespace arfx {

// Error types mirrored from the reference (R/math.hpp:12-18) for status mapping.
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoDevice : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct HV {  // host Vec3d
  double x = 0, y = 0, z = 0;
};

struct HostBone {
  int parent;
  HV head, tail;
  double radius;
};

struct HostBox {
  HV lo, hi;
};

void validate_skeleton(const std::vector<HostBone>& bones);               // R/skeleton.hpp:22-31
HostBox rest_bounds(const std::vector<HostBone>& bones, double margin);   // R/skeleton.hpp:53-63
double max_reach(const std::vector<HostBone>& bones);                     // R/skeleton.hpp:39-50
HostBox normalized_reach_box(const std::vector<HostBone>& bones, double margin = 1.05);  // R/model.hpp:59-66

struct GridCfg {
  int levels, F, log2T, nmin, nmax;
  HostBox box;
};
void validate_grid_cfg(const GridCfg& g);                 // R/hash_grid.hpp:20-29
std::vector<int> level_resolutions(const GridCfg& g);     // R/hash_grid.hpp:35-53

struct MlpLayout {
  int n_layers;
  int lin[kMaxMlpLayers], lout[kMaxMlpLayers], w_off[kMaxMlpLayers], b_off[kMaxMlpLayers];
  int n_params;
};
MlpLayout mlp_layout(int input_dim, int hidden_dim, int hidden_layers, int output_dim);  // R/mlp.hpp:37-48

// Rigids as double[12] (R row-major, t)
void rigid_compose(const double* a, const double* b, double* out);  // a after b  R/math.hpp:202-204
void rigid_inverse(const double* a, double* out);                     // R/math.hpp:197-200
HV rigid_apply(const double* a, const HV& v);
bool rigid_is_rotation(const double* a, double tol);                  // R/math.hpp:205-208

void pose_from_joint_rotations(const std::vector<HostBone>& bones, const double* rot9,
                               const double* global12, double* out12);  // R/skeleton.hpp:93-110
void make_pose_ctx(const std::vector<HostBone>& bones, const double* bones12, const double* pre12,
                   double cutoff_factor, PoseCtx& ctx);                 // R/articulation.hpp:24-41
void validate_pose(int n_bones, const double* bones12, const double* global12);  // R/skeleton.hpp:80-87

struct HostCamera {
  double fx, fy, cx, cy;
  int width, height;
  double ext[12];
};
HostCamera look_at(const HV& eye, const HV& target, const HV& up, double focal, int w, int h);  // R/camera.hpp:31-48
void validate_camera(const HostCamera& c);  // R/camera.hpp:15-22

// OccupancyGrid::empty threshold  R/occupancy.hpp:65
double occupancy_threshold(const HostBox& box, int res, double alpha_threshold);
void validate_occ_cfg(int resolution, double alpha_threshold, int dilation, double decay, int interval);

void set_error_message(const std::string& m);  // abi.cu: the thread-local arfx_last_error()

}  // namespace arfx
