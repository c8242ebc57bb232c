// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim (arfr_* in oracle_api.h) over the UNMODIFIED reference library
// at /root/reference/proj/include/arf, compiled in place with -include ref_fix.h
// (see that file for the two compile fixes). Every entry point calls the
// reference's own functions; where a debug trace is needed (arfr_render_trace,
// arfr_train_fwd_bwd) the driver composes reference functions exactly as
// render_image (R/render.hpp:178-218) and render_model (R/model.hpp:118-135) do,
// and tests assert the traced pixels are bit-identical to arf::render_model's.
//
// Built by oracle/Makefile into oracle/_ref/libarf_ref.so. Never shipped in the
// product; used by tests/ and by bench.py's cpu_baseline / --impl reference leg.

#include "arf/scene.hpp"  // pulls in model.hpp -> articulation/render/occupancy/...

#include <chrono>
#include <cstdio>
#include <string>

#include "oracle_api.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(1, e.what());
  } catch (const arf::DataError& e) {
    return fail(2, e.what());
  } catch (const arf::NumericError& e) {
    return fail(3, e.what());
  } catch (const std::domain_error& e) {
    return fail(4, e.what());
  } catch (const std::exception& e) {
    return fail(5, e.what());
  }
}

arf::Vec3d v3(const double* p) { return {p[0], p[1], p[2]}; }
void put3(double* o, const arf::Vec3d& v) {
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.z;
}

arf::Rigidd rigid(const double* p) {
  arf::Rigidd r;
  for (int i = 0; i < 9; ++i) r.rotation.m[static_cast<std::size_t>(i)] = p[i];
  r.translation = {p[9], p[10], p[11]};
  return r;
}
void put_rigid(double* o, const arf::Rigidd& r) {
  for (int i = 0; i < 9; ++i) o[i] = r.rotation.m[static_cast<std::size_t>(i)];
  put3(o + 9, r.translation);
}

arf::Aabbd box(const double* lo, const double* hi) {
  arf::Aabbd b;
  b.lo = v3(lo);
  b.hi = v3(hi);
  return b;
}

arf::Skeleton skeleton(const ao_skeleton* s) {
  arf::Skeleton sk;
  for (int i = 0; i < s->n_bones; ++i) {
    arf::Bone b;
    b.parent = s->parent[i];
    b.head = v3(s->head[i]);
    b.tail = v3(s->tail[i]);
    b.radius = s->radius[i];
    sk.bones.push_back(b);
  }
  return sk;
}

arf::HashGridConfig grid_cfg(const ao_grid_cfg* g) {
  arf::HashGridConfig c;
  c.levels = g->levels;
  c.features_per_level = g->features_per_level;
  c.table_size_log2 = g->table_size_log2;
  c.base_resolution = g->base_resolution;
  c.max_resolution = g->max_resolution;
  c.bounding_box = box(g->box_lo, g->box_hi);
  return c;
}

arf::MlpConfig mlp_cfg(const ao_mlp_cfg* m) {
  arf::MlpConfig c;
  c.input_dim = m->input_dim;
  c.hidden_dim = m->hidden_dim;
  c.hidden_layers = m->hidden_layers;
  c.output_dim = m->output_dim;
  return c;
}

// ao_model -> arf::Model<float>, fields set directly (no re-initialisation).
arf::Model<float> to_model(const ao_model* m) {
  arf::Model<float> M;
  M.skeleton = skeleton(&m->skel);
  M.canonical_box = box(m->canon_lo, m->canon_hi);
  M.normalized_box = box(m->norm_lo, m->norm_hi);
  auto& G = M.field.grid;
  G.config = grid_cfg(&m->grid);
  G.resolutions = arf::level_resolutions(G.config);
  G.table_rows = uint32_t(1) << G.config.table_size_log2;
  G.params.assign(m->grid_params, m->grid_params + m->n_grid);
  M.field.mlp = arf::DecoderMlp<float>(mlp_cfg(&m->mlp), 0);
  if (M.field.mlp.params.size() != m->n_mlp) throw std::invalid_argument("mlp size mismatch");
  std::copy(m->mlp_params, m->mlp_params + m->n_mlp, M.field.mlp.params.begin());
  M.skinning.resolution = {m->skin_res[0], m->skin_res[1], m->skin_res[2]};
  M.skinning.box = box(m->skin_lo, m->skin_hi);
  M.skinning.n_bones = m->skel.n_bones;
  M.skinning.weights.assign(m->skin_weights, m->skin_weights + m->n_skin);
  M.inverse_options.max_iterations = m->max_iterations;
  M.inverse_options.tolerance = m->tolerance;
  M.inverse_options.dedup_radius = m->dedup_radius;
  return M;
}

arf::SkeletonPose pose_of(int n_bones, const double* bones12, const double* global12) {
  arf::SkeletonPose p;
  for (int i = 0; i < n_bones; ++i) p.bone_transforms.push_back(rigid(bones12 + 12 * i));
  p.global_transform = rigid(global12);
  return p;
}

arf::Camera camera(const ao_camera* c) {
  arf::Camera cam;
  cam.fx = c->fx;
  cam.fy = c->fy;
  cam.cx = c->cx;
  cam.cy = c->cy;
  cam.width = c->width;
  cam.height = c->height;
  cam.extrinsic = rigid(c->extrinsic);
  return cam;
}

arf::RenderOptions render_opts(const ao_render_opts* o) {
  arf::RenderOptions r;
  r.samples_per_ray = o->samples_per_ray;
  r.stratified = o->stratified != 0;
  r.epsilon_terminate = o->epsilon_terminate;
  r.seed = o->seed;
  r.frame_id = o->frame_id;
  return r;
}

arf::OccupancyConfig occ_cfg(const ao_occ_cfg* c) {
  arf::OccupancyConfig o;
  o.resolution = c->resolution;
  o.alpha_threshold = c->alpha_threshold;
  o.dilation = c->dilation;
  o.decay = c->decay;
  o.update_interval = c->update_interval;
  return o;
}

arf::OccupancyGrid occ_in(const ao_occ_grid* g) {
  arf::OccupancyGrid o;
  o.resolution = {g->res[0], g->res[1], g->res[2]};
  o.box = box(g->box_lo, g->box_hi);
  o.density_threshold = g->density_threshold;
  o.dilation = g->dilation;
  const std::size_t n = o.cell_count();
  o.values.assign(g->values, g->values + n);
  o.mask.assign(g->mask, g->mask + n);
  return o;
}

void occ_out(const arf::OccupancyGrid& o, ao_occ_grid* g) {
  g->res[0] = o.resolution.x;
  g->res[1] = o.resolution.y;
  g->res[2] = o.resolution.z;
  put3(g->box_lo, o.box.lo);
  put3(g->box_hi, o.box.hi);
  g->density_threshold = o.density_threshold;
  g->dilation = o.dilation;
  if (g->values) std::copy(o.values.begin(), o.values.end(), g->values);
  if (g->mask) std::copy(o.mask.begin(), o.mask.end(), g->mask);
}

void counters_out(const arf::Model<float>& M, uint64_t* c) {
  if (!c) return;
  c[0] = M.counters.posed_queries.load();
  c[1] = M.counters.canonical_queries.load();
}

}  // namespace

extern "C" {

const char* arfr_last_error(void) { return g_err.c_str(); }

int arfr_model_sizes(const ao_skeleton* s, const ao_grid_cfg* g, const ao_mlp_cfg* m,
                     const int skin_res[3], size_t* n_grid, size_t* n_mlp, size_t* n_skin) {
  return guard([&] {
    arf::HashGridConfig gc = grid_cfg(g);
    gc.validate();
    *n_grid = static_cast<std::size_t>(gc.levels) * (static_cast<std::size_t>(1) << gc.table_size_log2) *
              static_cast<std::size_t>(gc.features_per_level);
    arf::MlpConfig mc = mlp_cfg(m);
    mc.input_dim = gc.feature_dim();
    *n_mlp = arf::DecoderMlp<float>(mc, 0).param_count();
    *n_skin = static_cast<std::size_t>(skin_res[0]) * static_cast<std::size_t>(skin_res[1]) *
              static_cast<std::size_t>(skin_res[2]) * static_cast<std::size_t>(s->n_bones);
  });
}

int arfr_build_model(const ao_skeleton* s, const ao_grid_cfg* g, const ao_mlp_cfg* m,
                     const int skin_res[3], uint64_t seed, ao_model* out) {
  return guard([&] {
    const arf::Model<float> M = arf::build_model<float>(
        skeleton(s), grid_cfg(g), mlp_cfg(m), {skin_res[0], skin_res[1], skin_res[2]}, seed);
    out->skel = *s;
    const auto& gc = M.field.grid.config;
    out->grid = *g;
    put3(out->grid.box_lo, gc.bounding_box.lo);
    put3(out->grid.box_hi, gc.bounding_box.hi);
    out->mlp = *m;
    out->mlp.input_dim = M.field.mlp.config.input_dim;
    for (int a = 0; a < 3; ++a) out->skin_res[a] = skin_res[a];
    put3(out->skin_lo, M.skinning.box.lo);
    put3(out->skin_hi, M.skinning.box.hi);
    put3(out->canon_lo, M.canonical_box.lo);
    put3(out->canon_hi, M.canonical_box.hi);
    put3(out->norm_lo, M.normalized_box.lo);
    put3(out->norm_hi, M.normalized_box.hi);
    out->max_iterations = M.inverse_options.max_iterations;
    out->tolerance = M.inverse_options.tolerance;
    out->dedup_radius = M.inverse_options.dedup_radius;
    if (out->n_grid != M.field.grid.params.size() || out->n_mlp != M.field.mlp.params.size() ||
        out->n_skin != M.skinning.weights.size())
      throw std::invalid_argument("build_model: output array sizes do not match model_sizes");
    std::copy(M.field.grid.params.begin(), M.field.grid.params.end(), out->grid_params);
    std::copy(M.field.mlp.params.begin(), M.field.mlp.params.end(), out->mlp_params);
    std::copy(M.skinning.weights.begin(), M.skinning.weights.end(), out->skin_weights);
  });
}

int arfr_level_resolutions(const ao_grid_cfg* g, int* out) {
  return guard([&] {
    const auto r = arf::level_resolutions(grid_cfg(g));
    std::copy(r.begin(), r.end(), out);
  });
}

uint32_t arfr_hash_index(const ao_grid_cfg* g, int level, int cx, int cy, int cz) {
  arf::HashGrid<float> G;
  G.config = grid_cfg(g);
  G.resolutions = arf::level_resolutions(G.config);
  G.table_rows = uint32_t(1) << G.config.table_size_log2;
  return G.hash_index(level, {cx, cy, cz});
}

int arfr_pose_from_joint_rotations(const ao_skeleton* s, const double* rot9, const double* g12,
                                   double* bones12) {
  return guard([&] {
    std::vector<arf::Mat3d> rots(static_cast<std::size_t>(s->n_bones));
    for (int i = 0; i < s->n_bones; ++i)
      for (int k = 0; k < 9; ++k) rots[static_cast<std::size_t>(i)].m[static_cast<std::size_t>(k)] = rot9[9 * i + k];
    const arf::SkeletonPose p = arf::pose_from_joint_rotations(skeleton(s), rots, rigid(g12));
    for (int i = 0; i < s->n_bones; ++i) put_rigid(bones12 + 12 * i, p.bone_transforms[static_cast<std::size_t>(i)]);
  });
}

int arfr_look_at(const double eye[3], const double target[3], const double up[3], double focal,
                 int w, int h, ao_camera* cam) {
  return guard([&] {
    const arf::Camera c = arf::Camera::look_at(v3(eye), v3(target), v3(up), focal, w, h);
    cam->fx = c.fx;
    cam->fy = c.fy;
    cam->cx = c.cx;
    cam->cy = c.cy;
    cam->width = c.width;
    cam->height = c.height;
    put_rigid(cam->extrinsic, c.extrinsic);
  });
}

int arfr_skinning_weights(const ao_model* m, const double* pts, int64_t n, double* w) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    const int nb = M.skinning.n_bones;
    for (int64_t i = 0; i < n; ++i)
      M.skinning.interpolate(v3(pts + 3 * i), std::span<double>(w + i * nb, static_cast<std::size_t>(nb)));
  });
}

int arfr_inverse_lbs(const ao_model* m, const double* bones12, const double* pre12,
                     double cutoff_factor, const double* pts, int64_t n, int32_t* counts,
                     double* roots, double* residuals) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    const arf::SkeletonPose pose = pose_of(m->skel.n_bones, bones12, pre12);  // global unused
    const arf::PoseContext ctx =
        arf::PoseContext::make(M.skeleton, pose, rigid(pre12), cutoff_factor);
    arf::parallel_for(n, [&](int64_t i) {
      const arf::InverseRoots r = arf::inverse_lbs_ctx(v3(pts + 3 * i), ctx, M.skinning, M.inverse_options);
      counts[i] = r.count;
      for (int k = 0; k < r.count; ++k) {
        put3(roots + (i * AO_MAX_ROOTS + k) * 3, r.x[static_cast<std::size_t>(k)]);
        residuals[i * AO_MAX_ROOTS + k] = r.residual[static_cast<std::size_t>(k)];
      }
    });
  });
}

int arfr_hash_encode(const ao_model* m, const double* pts, int64_t n, float* feats) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    const int D = M.field.grid.config.feature_dim();
    for (int64_t i = 0; i < n; ++i)
      M.field.grid.encode(v3(pts + 3 * i), std::span<float>(feats + i * D, static_cast<std::size_t>(D)));
  });
}

int arfr_field_query(const ao_model* m, const double* pts, int64_t n, float* dens, float* col) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    auto s = M.field.make_scratch();
    for (int64_t i = 0; i < n; ++i) {
      const arf::RadianceSample<float> r = M.field.query(v3(pts + 3 * i), s);
      dens[i] = r.density;
      col[3 * i + 0] = r.color.x;
      col[3 * i + 1] = r.color.y;
      col[3 * i + 2] = r.color.z;
    }
  });
}

int arfr_posed_query(const ao_model* m, const double* bones12, const double* global12,
                     const double* pts_norm, int64_t n, float* dens, float* col, double* canon,
                     uint8_t* has_root) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    const arf::PosedModelView<float> view(M, pose_of(m->skel.n_bones, bones12, global12));
    auto s = M.field.make_scratch();
    for (int64_t i = 0; i < n; ++i) {
      const arf::PosedSample<float> p = view.query_normalized(v3(pts_norm + 3 * i), s);
      has_root[i] = p.has_root ? 1 : 0;
      dens[i] = p.has_root ? p.radiance.density : 0.0f;
      col[3 * i + 0] = p.has_root ? p.radiance.color.x : 0.0f;
      col[3 * i + 1] = p.has_root ? p.radiance.color.y : 0.0f;
      col[3 * i + 2] = p.has_root ? p.radiance.color.z : 0.0f;
      put3(canon + 3 * i, p.has_root ? p.canonical : arf::Vec3d{0, 0, 0});
    }
  });
}

int arfr_occ_empty(const double lo[3], const double hi[3], const ao_occ_cfg* c, ao_occ_grid* g) {
  return guard([&] { occ_out(arf::OccupancyGrid::empty(box(lo, hi), occ_cfg(c)), g); });
}

int arfr_occ_rebuild_mask(ao_occ_grid* g) {
  return guard([&] {
    arf::OccupancyGrid o = occ_in(g);
    o.rebuild_mask();
    occ_out(o, g);
  });
}

int arfr_build_inference_grid(const ao_model* m, const double* bones12, const double* global12,
                              const ao_occ_cfg* c, ao_occ_grid* g, uint64_t* counters) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    const arf::OccupancyGrid o = arf::build_model_inference_grid(
        M, pose_of(m->skel.n_bones, bones12, global12), occ_cfg(c));
    occ_out(o, g);
    counters_out(M, counters);
  });
}

int arfr_update_training_grid(const ao_model* m, int n_poses, const double* bones12,
                              const double* global12, double decay, uint64_t seed, uint64_t step,
                              ao_occ_grid* g, uint64_t* counters) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    const int nb = m->skel.n_bones;
    std::vector<arf::PosedModelView<float>> views;
    for (int p = 0; p < n_poses; ++p)
      views.emplace_back(M, pose_of(nb, bones12 + static_cast<std::ptrdiff_t>(p) * nb * 12, global12 + 12 * p));
    arf::OccupancyGrid o = occ_in(g);
    arf::update_training_grid(o, n_poses, decay, seed, step, [&](int p, const arf::Vec3d& x) {
      thread_local arf::CanonicalField<float>::Scratch tl;
      if (tl.features.size() != static_cast<std::size_t>(M.field.grid.config.feature_dim()))
        tl = M.field.make_scratch();
      return views[static_cast<std::size_t>(p)].density_normalized(x, tl);
    });
    occ_out(o, g);
    counters_out(M, counters);
  });
}

int arfr_render(const ao_model* m, const double* bones12, const double* global12,
                const ao_camera* cam, const ao_occ_grid* occ, const ao_render_opts* o, float* rgb,
                float* alpha, uint64_t* counters) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    arf::OccupancyGrid og;
    if (occ) og = occ_in(occ);
    const arf::RenderImages img = arf::render_model(M, pose_of(m->skel.n_bones, bones12, global12),
                                                    camera(cam), occ ? &og : nullptr, render_opts(o));
    std::copy(img.rgb.begin(), img.rgb.end(), rgb);
    std::copy(img.alpha.begin(), img.alpha.end(), alpha);
    counters_out(M, counters);
  });
}

// Single-threaded restatement of render_image's per-pixel loop (R/render.hpp:188-216)
// bound to PosedModelView like render_model (R/model.hpp:125-133), recording the trace.
int arfr_render_trace(const ao_model* m, const double* bones12, const double* global12,
                      const ao_camera* cam, const ao_occ_grid* occ, const ao_render_opts* o,
                      float* rgb, float* alpha, uint64_t* counters, ao_render_trace* tr) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    arf::OccupancyGrid og;
    if (occ) og = occ_in(occ);
    const arf::OccupancyGrid* occp = occ ? &og : nullptr;
    const arf::PosedModelView<float> view(M, pose_of(m->skel.n_bones, bones12, global12));
    const arf::Camera C = camera(cam);
    const arf::RenderOptions opt = render_opts(o);
    auto scratch = M.field.make_scratch();
    const auto to_norm = [&](const arf::Vec3d& xw) { return view.to_normalized(xw); };
    arf::RaySampleSet<float> samples;
    int64_t ns = 0;
    for (int py = 0; py < C.height; ++py)
      for (int px = 0; px < C.width; ++px) {
        const std::size_t pix = static_cast<std::size_t>(py) * C.width + px;
        rgb[pix * 3 + 0] = rgb[pix * 3 + 1] = rgb[pix * 3 + 2] = 0.0f;
        alpha[pix] = 0.0f;
        tr->ray_first[pix] = -1;
        tr->ray_count[pix] = 0;
        tr->ray_hit[pix] = 0;
        tr->t_near[pix] = tr->t_far[pix] = 0.0;
        tr->terminated_at[pix] = 0;
        arf::Ray ray = arf::generate_ray(C, px, py);
        const arf::Vec3d on = to_norm(ray.origin);
        const arf::Vec3d dn = to_norm(ray.at(1.0)) - on;
        const auto hit = arf::ray_box(on, dn, M.normalized_box);
        if (!hit) continue;
        tr->ray_hit[pix] = 1;
        ray.t_near = hit->first;
        ray.t_far = hit->second;
        tr->t_near[pix] = ray.t_near;
        tr->t_far[pix] = ray.t_far;
        arf::Pcg32 rng = arf::keyed_rng(opt.seed, opt.frame_id, pix);
        arf::sample_points<float>(ray, opt.samples_per_ray, opt.stratified, &rng, occp, to_norm, samples);
        tr->ray_first[pix] = static_cast<int32_t>(ns);
        for (int i = 0; i < samples.size(); ++i) {
          const std::size_t si = static_cast<std::size_t>(i);
          if (samples.skipped[si]) continue;
          const arf::PosedSample<float> ps =
              view.query_normalized(view.to_normalized(ray.at(samples.t[si])), scratch);
          if (!ps.has_root) samples.skipped[si] = 1;
          else samples.radiance[si] = ps.radiance;
          if (ns < tr->capacity) {
            tr->s_ray[ns] = static_cast<int32_t>(pix);
            tr->s_index[ns] = i;
            tr->s_has_root[ns] = ps.has_root ? 1 : 0;
            tr->s_density[ns] = ps.has_root ? ps.radiance.density : 0.0f;
            tr->s_color[3 * ns + 0] = ps.has_root ? ps.radiance.color.x : 0.0f;
            tr->s_color[3 * ns + 1] = ps.has_root ? ps.radiance.color.y : 0.0f;
            tr->s_color[3 * ns + 2] = ps.has_root ? ps.radiance.color.z : 0.0f;
            put3(tr->s_canonical + 3 * ns, ps.has_root ? ps.canonical : arf::Vec3d{0, 0, 0});
            tr->s_t[ns] = samples.t[si];
            tr->s_delta[ns] = samples.delta[si];
          }
          ++ns;
          ++tr->ray_count[pix];
        }
        const arf::CompositeResult<float> res = arf::composite(samples, opt.epsilon_terminate);
        tr->terminated_at[pix] = res.terminated_at;
        rgb[pix * 3 + 0] = float(res.color.x);
        rgb[pix * 3 + 1] = float(res.color.y);
        rgb[pix * 3 + 2] = float(res.color.z);
        alpha[pix] = float(res.alpha);
      }
    tr->n_samples = ns;
    counters_out(M, counters);
  });
}

static void fill_samples(arf::RaySampleSet<float>& s, int n, const double* t, const double* delta,
                         const uint8_t* skipped, const float* dens, const float* col) {
  s.resize(n);
  for (int i = 0; i < n; ++i) {
    const std::size_t k = static_cast<std::size_t>(i);
    s.t[k] = t[i];
    s.delta[k] = delta[i];
    s.skipped[k] = skipped[i];
    s.radiance[k].density = dens[i];
    s.radiance[k].color = {col[3 * i], col[3 * i + 1], col[3 * i + 2]};
  }
}

int arfr_composite(int n, const double* t, const double* delta, const uint8_t* skipped,
                   const float* dens, const float* col, double eps, double* color3, double* alpha,
                   int* terminated_at) {
  return guard([&] {
    arf::RaySampleSet<float> s;
    fill_samples(s, n, t, delta, skipped, dens, col);
    const arf::CompositeResult<float> r = arf::composite(s, eps);
    put3(color3, r.color);
    *alpha = r.alpha;
    *terminated_at = r.terminated_at;
  });
}

int arfr_composite_backward(int n, const double* t, const double* delta, const uint8_t* skipped,
                            const float* dens, const float* col, double eps, const double* d_color3,
                            double d_alpha, double* d_sigma, double* d_c3) {
  return guard([&] {
    arf::RaySampleSet<float> s;
    fill_samples(s, n, t, delta, skipped, dens, col);
    const arf::CompositeResult<float> r = arf::composite(s, eps);
    std::vector<double> ds;
    std::vector<arf::Vec3d> dc;
    arf::composite_backward(s, r, v3(d_color3), d_alpha, ds, dc);
    for (int i = 0; i < n; ++i) {
      d_sigma[i] = ds[static_cast<std::size_t>(i)];
      put3(d_c3 + 3 * i, dc[static_cast<std::size_t>(i)]);
    }
  });
}

int arfr_field_query_backward(const ao_model* m, const double* pts, int64_t n, const float* d_dens,
                              const float* d_col, float* grid_grad, float* mlp_grad) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    arf::FieldGrads<float> grads;
    grads.grid.assign(grid_grad, grid_grad + m->n_grid);
    grads.mlp.assign(mlp_grad, mlp_grad + m->n_mlp);
    auto s = M.field.make_scratch();
    for (int64_t i = 0; i < n; ++i)
      M.field.query_backward(v3(pts + 3 * i), d_dens[i],
                             {d_col[3 * i], d_col[3 * i + 1], d_col[3 * i + 2]}, grads, s);
    std::copy(grads.grid.begin(), grads.grid.end(), grid_grad);
    std::copy(grads.mlp.begin(), grads.mlp.end(), mlp_grad);
  });
}

// Training forward+backward composed from reference pieces per SPEC.md:490-494 (no
// reference function exists): per ray forward as render_image, then
// composite_backward (R/render.hpp:125-157), then query_backward (R/field.hpp:91-103) at
// each accumulated non-skipped sample's canonical root. Serial, ray order.
int arfr_train_fwd_bwd(const ao_model* m, const double* bones12, const double* global12,
                       const ao_camera* cam, const ao_occ_grid* occ, const ao_render_opts* o,
                       int64_t n_rays, const int32_t* px, const int32_t* py, const float* d_color,
                       const float* d_alpha, float* rgb, float* alpha, float* grid_grad,
                       float* mlp_grad, uint64_t* counters) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    arf::OccupancyGrid og;
    if (occ) og = occ_in(occ);
    const arf::OccupancyGrid* occp = occ ? &og : nullptr;
    const arf::PosedModelView<float> view(M, pose_of(m->skel.n_bones, bones12, global12));
    const arf::Camera C = camera(cam);
    const arf::RenderOptions opt = render_opts(o);
    auto scratch = M.field.make_scratch();
    arf::FieldGrads<float> grads;
    grads.grid.assign(grid_grad, grid_grad + m->n_grid);
    grads.mlp.assign(mlp_grad, mlp_grad + m->n_mlp);
    const auto to_norm = [&](const arf::Vec3d& xw) { return view.to_normalized(xw); };
    arf::RaySampleSet<float> samples;
    std::vector<arf::Vec3d> canon;
    std::vector<double> ds;
    std::vector<arf::Vec3d> dc;
    for (int64_t r = 0; r < n_rays; ++r) {
      rgb[3 * r + 0] = rgb[3 * r + 1] = rgb[3 * r + 2] = 0.0f;
      alpha[r] = 0.0f;
      const std::size_t pix = static_cast<std::size_t>(py[r]) * C.width + px[r];
      arf::Ray ray = arf::generate_ray(C, px[r], py[r]);
      const arf::Vec3d on = to_norm(ray.origin);
      const arf::Vec3d dn = to_norm(ray.at(1.0)) - on;
      const auto hit = arf::ray_box(on, dn, M.normalized_box);
      if (!hit) continue;
      ray.t_near = hit->first;
      ray.t_far = hit->second;
      arf::Pcg32 rng = arf::keyed_rng(opt.seed, opt.frame_id, pix);
      arf::sample_points<float>(ray, opt.samples_per_ray, opt.stratified, &rng, occp, to_norm, samples);
      canon.assign(static_cast<std::size_t>(samples.size()), arf::Vec3d{0, 0, 0});
      for (int i = 0; i < samples.size(); ++i) {
        const std::size_t si = static_cast<std::size_t>(i);
        if (samples.skipped[si]) continue;
        const arf::PosedSample<float> ps =
            view.query_normalized(view.to_normalized(ray.at(samples.t[si])), scratch);
        if (!ps.has_root) {
          samples.skipped[si] = 1;
          continue;
        }
        samples.radiance[si] = ps.radiance;
        canon[si] = ps.canonical;
      }
      const arf::CompositeResult<float> res = arf::composite(samples, opt.epsilon_terminate);
      rgb[3 * r + 0] = float(res.color.x);
      rgb[3 * r + 1] = float(res.color.y);
      rgb[3 * r + 2] = float(res.color.z);
      alpha[r] = float(res.alpha);
      arf::composite_backward(samples, res, {d_color[3 * r], d_color[3 * r + 1], d_color[3 * r + 2]},
                              d_alpha[r], ds, dc);
      for (int i = 0; i < res.terminated_at; ++i) {
        const std::size_t si = static_cast<std::size_t>(i);
        if (samples.skipped[si]) continue;
        M.field.query_backward(canon[si], float(ds[si]),
                               {float(dc[si].x), float(dc[si].y), float(dc[si].z)}, grads, scratch);
      }
    }
    std::copy(grads.grid.begin(), grads.grid.end(), grid_grad);
    std::copy(grads.mlp.begin(), grads.mlp.end(), mlp_grad);
    counters_out(M, counters);
  });
}

// CPU-baseline timing helper (bench.py --impl reference / cpu_baseline): converts the
// model once, then times `n_frames` x (build_model_inference_grid + render_model) with the
// reference's own thread pool (ARF_THREADS or hardware concurrency). Times in seconds.
int arfr_bench_frames(const ao_model* m, int n_frames, const double* bones12,
                      const double* global12, const ao_camera* cam, const ao_occ_cfg* oc,
                      const ao_render_opts* o, double* seconds, uint64_t* posed_per_frame,
                      float* rgb_last, float* alpha_last, uint8_t* mask_last) {
  return guard([&] {
    const arf::Model<float> M = to_model(m);
    const int nb = m->skel.n_bones;
    for (int f = 0; f < n_frames; ++f) {
      const arf::SkeletonPose pose =
          pose_of(nb, bones12 + static_cast<std::ptrdiff_t>(f) * nb * 12, global12 + 12 * f);
      M.counters.reset();
      const auto t0 = std::chrono::steady_clock::now();
      const arf::OccupancyGrid occ = arf::build_model_inference_grid(M, pose, occ_cfg(oc));
      M.counters.reset();
      const arf::RenderImages img = arf::render_model(M, pose, camera(cam), &occ, render_opts(o));
      const auto t1 = std::chrono::steady_clock::now();
      seconds[f] = std::chrono::duration<double>(t1 - t0).count();
      posed_per_frame[f] = M.counters.posed_queries.load();
      if (f == n_frames - 1 && rgb_last) {
        std::copy(img.rgb.begin(), img.rgb.end(), rgb_last);
        std::copy(img.alpha.begin(), img.alpha.end(), alpha_last);
        if (mask_last) std::copy(occ.mask.begin(), occ.mask.end(), mask_last);
      }
    }
  });
}

int arfr_thread_count(void) { return arf::thread_count(); }

// bench.py --impl reference builds its workload through the reference alone (no product
// code on that arm). random_pose: keyed_rng(seed, stream) (R/rng.hpp:61-63); per non-root
// joint draw axis x, y, z ~ U(-1,1), then angle ~ U(-a,a) (one statement per draw, SURVEY.md
// §8d), axis normalised, Mat3d::axis_angle (R/math.hpp:170-178); global yaw_about the root
// head (R/scene.hpp:169-171); pose_from_joint_rotations (R/skeleton.hpp:93-110).
int arfr_random_pose(const ao_skeleton* s, uint64_t seed, uint64_t stream, double max_angle, double yaw,
                     double* bones12, double* global12) {
  return guard([&] {
    const arf::Skeleton sk = skeleton(s);
    arf::Pcg32 rng = arf::keyed_rng(seed, stream);
    std::vector<arf::Mat3d> rots(static_cast<std::size_t>(s->n_bones), arf::Mat3d::identity());
    for (int i = 1; i < s->n_bones; ++i) {
      const double ax = rng.uniform(-1.0, 1.0);
      const double ay = rng.uniform(-1.0, 1.0);
      const double az = rng.uniform(-1.0, 1.0);
      const double ang = rng.uniform(-max_angle, max_angle);
      const double n = std::sqrt(ax * ax + ay * ay + az * az);
      rots[static_cast<std::size_t>(i)] = arf::Mat3d::axis_angle({ax / n, ay / n, az / n}, ang);
    }
    const arf::Rigidd g = arf::yaw_about(sk.bones[0].head, yaw);
    const arf::SkeletonPose p = arf::pose_from_joint_rotations(sk, rots, g);
    for (int i = 0; i < s->n_bones; ++i) put_rigid(bones12 + 12 * i, p.bone_transforms[static_cast<std::size_t>(i)]);
    put_rigid(global12, p.global_transform);
  });
}

// arf::default_camera (R/scene.hpp:190-197)
int arfr_default_camera(const ao_skeleton* s, int w, int h, ao_camera* cam) {
  return guard([&] {
    const arf::Camera c = arf::default_camera(skeleton(s), w, h);
    cam->fx = c.fx;
    cam->fy = c.fy;
    cam->cx = c.cx;
    cam->cy = c.cy;
    cam->width = c.width;
    cam->height = c.height;
    put_rigid(cam->extrinsic, c.extrinsic);
  });
}

}  // extern "C"

namespace {
arf::CapsuleFigure figure_of(const ao_figure* f) {
  arf::CapsuleFigure fig;
  fig.skeleton = skeleton(&f->skel);
  for (int i = 0; i < f->skel.n_bones; ++i) {
    fig.colors.push_back(v3(f->color[i]));
    fig.amplitudes.push_back(f->amplitude[i]);
  }
  fig.softness = f->softness;
  return fig;
}
}  // namespace

extern "C" {

// analytic_query (R/scene.hpp:31-50) / PosedFigure::query (:79-97)
int arfr_figure_query(const ao_figure* f, const double* bones12, const double* pts, int64_t n, double* dens,
                      double* col) {
  return guard([&] {
    const arf::CapsuleFigure fig = figure_of(f);
    fig.validate();
    if (bones12) {
      const arf::PosedFigure pf(fig, pose_of(f->skel.n_bones, bones12, bones12));
      for (int64_t i = 0; i < n; ++i) {
        const auto r = pf.query(v3(pts + 3 * i));
        dens[i] = r.density;
        put3(col + 3 * i, r.color);
      }
    } else {
      for (int64_t i = 0; i < n; ++i) {
        const auto r = arf::analytic_query(v3(pts + 3 * i), fig);
        dens[i] = r.density;
        put3(col + 3 * i, r.color);
      }
    }
  });
}

// The dataset frame: render_image (R/render.hpp:178-218) of PosedFigure::query through
// G^-1 into the given normalized box, no occupancy; mask = PosedFigure::ray_hits.
int arfr_figure_render(const ao_figure* f, const double* bones12, const double* global12, const double lo[3],
                       const double hi[3], const ao_camera* cam, const ao_render_opts* o, float* rgb, float* alpha,
                       uint8_t* mask) {
  return guard([&] {
    const arf::CapsuleFigure fig = figure_of(f);
    const arf::SkeletonPose pose = pose_of(f->skel.n_bones, bones12, global12);
    const arf::PosedFigure pf(fig, pose);
    const arf::Rigidd ginv = pose.global_transform.inverse();
    const arf::Camera C = camera(cam);
    const arf::RenderImages img = arf::render_image<double>(
        C, box(lo, hi),
        [&](const arf::Vec3d& x, arf::RadianceSample<double>& out) {
          out = pf.query(x);
          return out.density > 0.0;
        },
        [&](const arf::Vec3d& x) { return ginv.apply(x); }, nullptr, render_opts(o));
    if (rgb) std::copy(img.rgb.begin(), img.rgb.end(), rgb);
    if (alpha) std::copy(img.alpha.begin(), img.alpha.end(), alpha);
    if (mask)
      for (int py = 0; py < C.height; ++py)
        for (int px = 0; px < C.width; ++px)
          mask[static_cast<size_t>(py) * C.width + px] = pf.ray_hits(arf::generate_ray(C, px, py)) ? 1 : 0;
  });
}

}  // extern "C"
