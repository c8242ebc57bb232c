// adapter_parity.cpp -- TEST: the C++ drop-in (include/arfx/arf_gpu.hpp) used exactly as
// a reference user would, next to the UNMODIFIED reference (compiled with
// -include oracle/ref_fix.h -I/root/reference/proj/include). Builds an arf::Model<float>
// with the reference's build_model, uploads it, and compares the reference's
// build_model_inference_grid + render_model with the GPU path. Exit 0 = parity.
#include "arf/scene.hpp"

#include <cmath>
#include <cstdio>

#include "arfx/arf_gpu.hpp"

int main() {
  const arf::CapsuleFigure fig = arf::default_figure();
  arf::HashGridConfig g;
  g.levels = 8;
  g.table_size_log2 = 14;
  g.base_resolution = 4;
  g.max_resolution = 96;
  const arf::Model<float> model = arf::build_model<float>(fig.skeleton, g, arf::MlpConfig{}, {16, 16, 16}, 21);
  const arf::SkeletonPose pose = arf::bend_pose(fig.skeleton, 0.5, 0.3, arf::yaw_about(fig.skeleton.bones[0].head, 0.4));
  const arf::Camera cam = arf::default_camera(fig.skeleton, 64, 48);
  arf::RenderOptions opt;
  opt.samples_per_ray = 96;
  opt.stratified = true;
  opt.seed = 5;
  arf::OccupancyConfig occ_cfg;
  occ_cfg.resolution = 32;

  // reference
  const arf::OccupancyGrid occ = arf::build_model_inference_grid(model, pose, occ_cfg);
  model.counters.reset();
  const arf::RenderImages ref = arf::render_model(model, pose, cam, &occ, opt);

  // drop-in
  try {
    arfx::DeviceModel dm = arfx::DeviceModel::upload(model);
    arfx::DeviceOccupancyGrid docc(dm, occ_cfg);
    arfx::build_model_inference_grid(dm, pose, docc);
    arf::OccupancyGrid gpu_occ = arf::OccupancyGrid::empty(model.normalized_box, occ_cfg);
    docc.download(gpu_occ);
    arfx_counters cnt{};
    const arf::RenderImages img = arfx::render_model<arf::RenderImages>(dm, pose, cam, &docc, opt, &cnt);
    if (gpu_occ.mask != occ.mask) {
      std::printf("FAIL: occupancy mask differs\n");
      return 1;
    }
    double max_d = 0.0;
    for (std::size_t i = 0; i < img.rgb.size(); ++i) max_d = std::max(max_d, double(std::fabs(img.rgb[i] - ref.rgb[i])));
    for (std::size_t i = 0; i < img.alpha.size(); ++i)
      max_d = std::max(max_d, double(std::fabs(img.alpha[i] - ref.alpha[i])));
    const bool counts_ok = cnt.posed_queries == model.counters.posed_queries.load() &&
                           cnt.canonical_queries == model.counters.canonical_queries.load();
    std::printf("adapter parity: max |d| = %.3g, posed %llu/%llu canonical %llu/%llu\n", max_d,
                (unsigned long long)cnt.posed_queries, (unsigned long long)model.counters.posed_queries.load(),
                (unsigned long long)cnt.canonical_queries, (unsigned long long)model.counters.canonical_queries.load());
    if (max_d > 1e-5 || !counts_ok) {
      std::printf("FAIL\n");
      return 1;
    }
    // the reference's exception types survive the C-ABI
    try {
      arfx::DeviceOccupancyGrid bad(dm, arf::OccupancyConfig{1, 0.01, 1, 0.95, 16});
      std::printf("FAIL: invalid config accepted\n");
      return 1;
    } catch (const std::invalid_argument&) {
    }
  } catch (const std::exception& e) {
    std::printf("FAIL: %s\n", e.what());
    return 2;
  }
  std::printf("PASS\n");
  return 0;
}
