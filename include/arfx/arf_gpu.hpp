// arf_gpu.hpp -- header-only C++17 drop-in for the model-bound render path of the
// reference library `arf` (/root/reference/proj/include/arf), over the C-ABI in arfx.h.
//
// The adapter is duck-typed on the caller's own arf types (it does not include the
// reference headers), so a reference user swaps
//
//     arf::OccupancyGrid occ = arf::build_model_inference_grid(model, pose, occ_cfg);
//     arf::RenderImages img  = arf::render_model(model, pose, camera, &occ, opt);
//
// for
//
//     arfx::DeviceModel dm = arfx::DeviceModel::upload(model);        // once
//     arfx::DeviceOccupancyGrid docc(dm, occ_cfg);                     // once
//     arfx::build_model_inference_grid(dm, pose, docc);                // per pose
//     arf::RenderImages img = arfx::render_model<arf::RenderImages>(dm, pose, camera, &docc, opt);
//
// with identical arguments and result layout (R/model.hpp:118-148, R/render.hpp:167-171).
// Errors are rethrown as the reference's exception types: std::invalid_argument,
// std::domain_error, and std::runtime_error for numeric / data / CUDA failures
// (define ARFX_THROW to map codes 2 / 3 onto arf::DataError / arf::NumericError).
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../arfx.h"

namespace arfx {

#ifndef ARFX_THROW
#define ARFX_THROW(code, msg)                                                       \
  do {                                                                              \
    if ((code) == ARFX_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);      \
    if ((code) == ARFX_ERR_DOMAIN) throw std::domain_error(msg);                     \
    throw std::runtime_error(msg);                                                  \
  } while (0)
#endif

inline void check(int code) {
  if (code != ARFX_OK) {
    const std::string msg = arfx_last_error();
    ARFX_THROW(code, msg);
  }
}

template <class V>
inline void put3(double* o, const V& v) {
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.z;
}

template <class Rigid>
inline void put_rigid(double* o, const Rigid& r) {
  for (int i = 0; i < 9; ++i) o[i] = r.rotation.m[static_cast<std::size_t>(i)];
  put3(o + 9, r.translation);
}

template <class Skeleton>
inline arfx_skeleton to_c_skeleton(const Skeleton& s) {
  arfx_skeleton out;
  std::memset(&out, 0, sizeof(out));
  out.n_bones = static_cast<int>(s.bones.size());
  if (out.n_bones > ARFX_MAX_BONES) throw std::invalid_argument("pose context: too many bones");
  for (int i = 0; i < out.n_bones; ++i) {
    const auto& b = s.bones[static_cast<std::size_t>(i)];
    out.parent[i] = b.parent;
    put3(out.head[i], b.head);
    put3(out.tail[i], b.tail);
    out.radius[i] = b.radius;
  }
  return out;
}

// Device-resident arf::Model<float> (R/model.hpp:28-57).
class DeviceModel {
 public:
  DeviceModel() = default;
  explicit DeviceModel(arfx_model h) : h_(h) {}
  DeviceModel(const DeviceModel&) = delete;
  DeviceModel& operator=(const DeviceModel&) = delete;
  DeviceModel(DeviceModel&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  DeviceModel& operator=(DeviceModel&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  ~DeviceModel() {
    if (h_) arfx_model_destroy(h_);
  }
  arfx_model get() const { return h_; }

  // Mirror of an existing arf::Model<float> built by the reference (upload its members).
  template <class ArfModel>
  static DeviceModel upload(const ArfModel& m) {
    arfx_model_desc d;
    std::memset(&d, 0, sizeof(d));
    d.skeleton = to_c_skeleton(m.skeleton);
    const auto& gc = m.field.grid.config;
    d.grid.levels = gc.levels;
    d.grid.features_per_level = gc.features_per_level;
    d.grid.table_size_log2 = gc.table_size_log2;
    d.grid.base_resolution = gc.base_resolution;
    d.grid.max_resolution = gc.max_resolution;
    put3(d.grid.box_lo, gc.bounding_box.lo);
    put3(d.grid.box_hi, gc.bounding_box.hi);
    const auto& mc = m.field.mlp.config;
    d.mlp.input_dim = mc.input_dim;
    d.mlp.hidden_dim = mc.hidden_dim;
    d.mlp.hidden_layers = mc.hidden_layers;
    d.mlp.output_dim = mc.output_dim;
    d.skin_res[0] = m.skinning.resolution.x;
    d.skin_res[1] = m.skinning.resolution.y;
    d.skin_res[2] = m.skinning.resolution.z;
    put3(d.skin_lo, m.skinning.box.lo);
    put3(d.skin_hi, m.skinning.box.hi);
    put3(d.canonical_lo, m.canonical_box.lo);
    put3(d.canonical_hi, m.canonical_box.hi);
    put3(d.normalized_lo, m.normalized_box.lo);
    put3(d.normalized_hi, m.normalized_box.hi);
    d.inverse.max_iterations = m.inverse_options.max_iterations;
    d.inverse.tolerance = m.inverse_options.tolerance;
    d.inverse.dedup_radius = m.inverse_options.dedup_radius;
    d.n_grid_params = m.field.grid.params.size();
    d.n_mlp_params = m.field.mlp.params.size();
    d.n_skin_weights = m.skinning.weights.size();
    arfx_model h = nullptr;
    check(arfx_model_create(&d, m.field.grid.params.data(), m.field.mlp.params.data(), m.skinning.weights.data(), &h));
    return DeviceModel(h);
  }

  // Push host-side parameter edits (optimizer step / checkpoint load) to the device.
  template <class ArfModel>
  void sync_params(const ArfModel& m) {
    check(arfx_model_set_params(h_, m.field.grid.params.data(), m.field.mlp.params.data()));
  }

 private:
  arfx_model h_ = nullptr;
};

// PosedModelView (R/model.hpp:85-114) on the device.
class DevicePose {
 public:
  template <class SkeletonPose>
  DevicePose(const DeviceModel& m, const SkeletonPose& pose) {
    std::vector<double> b(pose.bone_transforms.size() * 12);
    for (std::size_t i = 0; i < pose.bone_transforms.size(); ++i) put_rigid(b.data() + 12 * i, pose.bone_transforms[i]);
    double g[12];
    put_rigid(g, pose.global_transform);
    check(arfx_pose_create(m.get(), b.data(), g, &h_));
  }
  DevicePose(const DevicePose&) = delete;
  DevicePose& operator=(const DevicePose&) = delete;
  ~DevicePose() {
    if (h_) arfx_pose_destroy(h_);
  }
  arfx_pose get() const { return h_; }

 private:
  arfx_pose h_ = nullptr;
};

// OccupancyGrid (R/occupancy.hpp:37-126) on the device, over the model's normalized box.
class DeviceOccupancyGrid {
 public:
  template <class OccupancyConfig>
  DeviceOccupancyGrid(const DeviceModel& m, const OccupancyConfig& cfg) {
    arfx_model_desc d;
    check(arfx_model_describe(m.get(), &d));
    const arfx_occ_config c{cfg.resolution, cfg.alpha_threshold, cfg.dilation, cfg.decay, cfg.update_interval};
    check(arfx_occ_create(d.normalized_lo, d.normalized_hi, &c, &h_));
  }
  DeviceOccupancyGrid(const DeviceOccupancyGrid&) = delete;
  DeviceOccupancyGrid& operator=(const DeviceOccupancyGrid&) = delete;
  ~DeviceOccupancyGrid() {
    if (h_) arfx_occ_destroy(h_);
  }
  arfx_occ_grid get() const { return h_; }
  // copy into an arf::OccupancyGrid (values + mask), e.g. for caching or checkpoints
  template <class ArfGrid>
  void download(ArfGrid& g) const {
    check(arfx_occ_download(h_, g.values.data(), g.mask.data()));
  }

 private:
  arfx_occ_grid h_ = nullptr;
};

template <class SkeletonPose>
inline arfx_counters build_model_inference_grid(const DeviceModel& m, const SkeletonPose& pose,
                                                DeviceOccupancyGrid& g) {
  DevicePose p(m, pose);
  arfx_counters c{0, 0};
  check(arfx_build_inference_grid(m.get(), p.get(), g.get(), &c, nullptr));
  return c;
}

template <class Camera>
inline arfx_camera to_c_camera(const Camera& cam) {
  arfx_camera c;
  c.fx = cam.fx;
  c.fy = cam.fy;
  c.cx = cam.cx;
  c.cy = cam.cy;
  c.width = cam.width;
  c.height = cam.height;
  put_rigid(c.extrinsic, cam.extrinsic);
  return c;
}

// render_model (R/model.hpp:118-135) -> Images (arf::RenderImages layout: width, height,
// rgb[H*W*3], alpha[H*W]).
template <class Images, class SkeletonPose, class Camera, class RenderOptions>
inline Images render_model(const DeviceModel& m, const SkeletonPose& pose, const Camera& cam,
                           const DeviceOccupancyGrid* occ, const RenderOptions& opt,
                           arfx_counters* counters = nullptr) {
  DevicePose p(m, pose);
  const arfx_camera c = to_c_camera(cam);
  const arfx_render_options o{opt.samples_per_ray, opt.stratified ? 1 : 0, opt.epsilon_terminate, opt.seed,
                              opt.frame_id};
  Images out;
  out.width = cam.width;
  out.height = cam.height;
  out.rgb.assign(static_cast<std::size_t>(cam.width) * cam.height * 3, 0.0f);
  out.alpha.assign(static_cast<std::size_t>(cam.width) * cam.height, 0.0f);
  arfx_counters cnt{0, 0};
  check(arfx_render_model(m.get(), p.get(), &c, occ ? occ->get() : nullptr, &o, 0, 1, out.rgb.data(),
                          out.alpha.data(), &cnt, nullptr));
  if (counters) *counters = cnt;
  return out;
}

}  // namespace arfx
