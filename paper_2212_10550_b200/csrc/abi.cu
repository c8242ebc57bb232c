// abi.cu -- extern "C" entry points of libarfx.so (declared in include/arfx.h).
// Handles own device memory; errors become status codes + a thread-local message
// (the reference throws: R/math.hpp:12-18, std::invalid_argument / domain_error).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/arfx.h"
#include "host.h"
#include "model.h"

struct arfx_model_s {
  arfx::ModelImpl impl;
};
struct arfx_pose_s {
  arfx::PoseImpl impl;
};
struct arfx_occ_s {
  arfx::OccImpl impl;
};
struct arfx_frame_graph_s {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int device = 0;
  const arfx::Workspace* ws = nullptr;  // the workspace the kernels were captured on
  unsigned long long ws_gen = 0;        // its generation at capture
  const arfx::Workspace* ws2 = nullptr;  // pipelined graphs: the side branch's workspace
  unsigned long long ws2_gen = 0;
  ~arfx_frame_graph_s() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};

namespace arfx {

namespace {
thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename F>
int guard(F&& f) {
  try {
    f();
    return ARFX_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ARFX_ERR_INVALID_ARGUMENT;
  } catch (const DataError& e) {
    g_err = e.what();
    return ARFX_ERR_DATA;
  } catch (const NumericError& e) {
    g_err = e.what();
    return ARFX_ERR_NUMERIC;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return ARFX_ERR_DOMAIN;
  } catch (const NoDevice& e) {
    g_err = e.what();
    return ARFX_ERR_NO_DEVICE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ARFX_ERR_RUNTIME;
  }
}

}  // namespace
// lets host-only translation units (checkpoint.cpp) report through arfx_last_error()
void set_error_message(const std::string& m) { g_err = m; }
namespace {

void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw NoDevice("libarfx: no CUDA device available (there is no CPU fallback)");
  }
}

std::vector<HostBone> bones_of(const arfx_skeleton* s) {
  require(s != nullptr, "skeleton: null");
  require(s->n_bones >= 1, "skeleton: needs at least one bone");
  require(s->n_bones <= ARFX_MAX_BONES, "pose context: too many bones");
  std::vector<HostBone> b(static_cast<size_t>(s->n_bones));
  for (int i = 0; i < s->n_bones; ++i) {
    b[static_cast<size_t>(i)] = HostBone{s->parent[i], {s->head[i][0], s->head[i][1], s->head[i][2]},
                                         {s->tail[i][0], s->tail[i][1], s->tail[i][2]}, s->radius[i]};
  }
  return b;
}

GridCfg grid_of(const arfx_grid_config* g) {
  require(g != nullptr, "grid config: null");
  return GridCfg{g->levels, g->features_per_level, g->table_size_log2, g->base_resolution,
                 g->max_resolution,
                 HostBox{{g->box_lo[0], g->box_lo[1], g->box_lo[2]}, {g->box_hi[0], g->box_hi[1], g->box_hi[2]}}};
}

HostCamera camera_of(const arfx_camera* c) {
  require(c != nullptr, "camera: null");
  HostCamera h{c->fx, c->fy, c->cx, c->cy, c->width, c->height, {}};
  std::memcpy(h.ext, c->extrinsic, sizeof(h.ext));
  return h;
}

cudaStream_t stream_of(ModelImpl& m, void* s) {
  return s ? static_cast<cudaStream_t>(s) : m.stream;
}

template <typename T>
void h2d(T* d, const T* h, size_t n, cudaStream_t s) {
  if (n) ARFX_CUDA(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <typename T>
void d2h(T* h, const T* d, size_t n, cudaStream_t s) {
  if (n) ARFX_CUDA(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}

// Hash-grid level kinds  R/hash_grid.hpp:87-101
void fill_field_view(ModelImpl& m) {
  FieldView& f = m.fv;
  f = FieldView{};
  f.L = m.grid.levels;
  f.F = m.grid.F;
  f.log2T = m.grid.log2T;
  f.T = 1u << m.grid.log2T;
  for (int l = 0; l < f.L; ++l) {
    const uint64_t n = static_cast<uint64_t>(m.res[static_cast<size_t>(l)]);
    const uint64_t c = n + 1;
    f.res[l] = static_cast<int>(n);
    f.kind[l] = (c * c * c <= f.T) ? kDirect : ((n * n * n <= f.T) ? kWrap : kHashed);
  }
  const HostBox& b = m.grid.box;
  f.lo[0] = b.lo.x;
  f.lo[1] = b.lo.y;
  f.lo[2] = b.lo.z;
  f.hi[0] = b.hi.x;
  f.hi[1] = b.hi.y;
  f.hi[2] = b.hi.z;
  f.e[0] = b.hi.x - b.lo.x;
  f.e[1] = b.hi.y - b.lo.y;
  f.e[2] = b.hi.z - b.lo.z;
  f.grid = m.grid_params.ptr;
  f.n_layers = m.mlp.n_layers;
  for (int l = 0; l < m.mlp.n_layers; ++l) {
    f.lin[l] = m.mlp.lin[l];
    f.lout[l] = m.mlp.lout[l];
    f.w_off[l] = m.mlp.w_off[l];
    f.b_off[l] = m.mlp.b_off[l];
  }
  f.in_dim = m.mlp_in;
  f.hidden = m.mlp_hidden;
  f.out_dim = m.mlp_out;
  f.n_mlp = m.mlp.n_params;
  f.mlp = m.mlp_params.ptr;
  SkinView& s = m.sv;
  s.rx = m.skin_res[0];
  s.ry = m.skin_res[1];
  s.rz = m.skin_res[2];
  s.nb = static_cast<int>(m.bones.size());
  s.lo[0] = m.skin_box.lo.x;
  s.lo[1] = m.skin_box.lo.y;
  s.lo[2] = m.skin_box.lo.z;
  s.hi[0] = m.skin_box.hi.x;
  s.hi[1] = m.skin_box.hi.y;
  s.hi[2] = m.skin_box.hi.z;
  s.e[0] = m.skin_box.hi.x - m.skin_box.lo.x;
  s.e[1] = m.skin_box.hi.y - m.skin_box.lo.y;
  s.e[2] = m.skin_box.hi.z - m.skin_box.lo.z;
  s.weights = m.skin.ptr;
  s.cell_mask = m.cell_mask.ptr;
  s.cell_off = m.cell_off.ptr;
  s.cell_mo = m.cell_mo.ptr;
  s.cell_vals = m.cell_vals.ptr;
}

// common model skeleton/config setup (shared by build_model and model_create)
void setup_model(ModelImpl& m, const std::vector<HostBone>& bones, GridCfg grid, int mlp_hidden,
                 int mlp_hl, int mlp_out, const int skin_res[3]) {
  validate_skeleton(bones);
  m.bones = bones;
  m.grid = grid;
  m.res = level_resolutions(grid);  // validates the grid config
  m.mlp_in = grid.levels * grid.F;
  m.mlp_hidden = mlp_hidden;
  m.mlp_hl = mlp_hl;
  m.mlp_out = mlp_out;
  m.mlp = mlp_layout(m.mlp_in, mlp_hidden, mlp_hl, mlp_out);
  require(mlp_out >= 4, "mlp: output_dim must be >= 4 (density + 3 colour logits, R/field.hpp:78-81)");
  require(m.mlp_in <= 256 && mlp_hidden <= 256 && mlp_out <= 256,
          "mlp: libarfx supports layer widths <= 256");
  require(skin_res[0] >= 2 && skin_res[1] >= 2 && skin_res[2] >= 2,
          "skinning grid: resolution must be >= 2 per axis");
  for (int a = 0; a < 3; ++a) m.skin_res[a] = skin_res[a];
  m.n_grid = static_cast<size_t>(grid.levels) * (static_cast<size_t>(1) << grid.log2T) *
             static_cast<size_t>(grid.F);
  m.n_mlp = static_cast<size_t>(m.mlp.n_params);
  m.n_skin = static_cast<size_t>(skin_res[0]) * skin_res[1] * skin_res[2] * bones.size();
}

void alloc_model(ModelImpl& m) {
  ARFX_CUDA(cudaGetDevice(&m.device));
  if (!m.stream) ARFX_CUDA(cudaStreamCreateWithFlags(&m.stream, cudaStreamNonBlocking));
  // [grid | pad to 256 B | mlp (float4-padded for the smem staging) | pad to 1024 floats]
  m.mlp_off = (m.n_grid + 63) / 64 * 64;
  m.n_flat = (m.mlp_off + (m.n_mlp + 3) / 4 * 4 + 1023) / 1024 * 1024;
  m.flat_params.alloc(m.n_flat);
  ARFX_CUDA(cudaMemset(m.flat_params.ptr, 0, m.n_flat * sizeof(float)));
  m.grid_params.view(m.flat_params.ptr, m.n_grid);
  m.mlp_params.view(m.flat_params.ptr + m.mlp_off, (m.n_mlp + 3) / 4 * 4);
  m.skin.alloc(m.n_skin);
}

// FieldGrads (R/field.hpp:19-36) as one flat zeroed vector laid out like the parameters
void ensure_grad_store(ModelImpl& m, cudaStream_t s) {
  if (m.flat_grads.ptr) return;
  m.flat_grads.alloc(m.n_flat);
  ARFX_CUDA(cudaMemsetAsync(m.flat_grads.ptr, 0, m.n_flat * sizeof(float), s));
  ARFX_CUDA(cudaStreamSynchronize(s));
  m.grid_grad.view(m.flat_grads.ptr, m.n_grid);
  m.mlp_grad.view(m.flat_grads.ptr + m.mlp_off, m.n_mlp);
}

void make_pose_host(ModelImpl& m, const double* bones12, const double* global12, PoseCtx& ctx) {
  require(bones12 != nullptr && global12 != nullptr, "pose: null transforms");
  double ginv[12];
  rigid_inverse(global12, ginv);
  make_pose_ctx(m.bones, bones12, ginv, 3.0, ctx);  // PosedModelView ctor R/model.hpp:92-96
}

OccImpl& occ_ref(arfx_occ_grid g) {
  require(g != nullptr, "occupancy grid: null");
  return g->impl;
}

void check_overflow_and_grow(ModelImpl& m, const unsigned long long* c, bool& rerun) {
  rerun = false;
  Workspace& w = m.ws();
  if (c[6] > w.cap_starts) w.learned_starts = static_cast<size_t>(c[6] + c[6] / 4 + 1024);
  if (c[0] > w.cap_posed || c[3] > 0 || c[2] > w.cap_pool) {
    const size_t need = static_cast<size_t>(std::max<unsigned long long>(c[0], w.cap_posed));
    w.cap_posed = 0;  // force reallocation
    w.cap_pool = 0;
    w.ensure(need + need / 4 + 4096, 0);
    rerun = true;
  }
}

}  // namespace

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
      throw NoDevice(std::string("CUDA: ") + cudaGetErrorString(e) + " in " + what);
    throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e) + " in " + what);
  }
}

ModelImpl::~ModelImpl() {
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
  if (side) {
    cudaStreamSynchronize(side);
    cudaStreamDestroy(side);
  }
  for (auto& e : pipe_graphs) delete static_cast<arfx_frame_graph_s*>(e.graph);
  pipe_graphs.clear();
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (ev_pipe_fork) cudaEventDestroy(ev_pipe_fork);
  if (ev_pipe_join) cudaEventDestroy(ev_pipe_join);
  if (aux) {
    cudaStreamSynchronize(aux);
    cudaStreamDestroy(aux);
  }
  if (ev_aux_fork) cudaEventDestroy(ev_aux_fork);
  if (ev_aux_join) cudaEventDestroy(ev_aux_join);
  if (copy_stream) {
    cudaStreamSynchronize(copy_stream);
    cudaStreamDestroy(copy_stream);
  }
  for (auto& a : async_slot) {
    if (a.rendered) cudaEventDestroy(a.rendered);
    if (a.copied) cudaEventDestroy(a.copied);
  }
}

void ModelImpl::refresh_views() { fill_field_view(*this); }

PoseImpl::~PoseImpl() {
  for (auto& e : ring_ev)
    if (e) {
      cudaEventSynchronize(e);
      cudaEventDestroy(e);
    }
  if (ring) cudaFreeHost(ring);
}

}  // namespace arfx

namespace arfx {
namespace {
struct RenderBuffers {
  DevBuf<float> rgb, alpha;
  DevBuf<unsigned long long> counters;
};
// the synchronous render's device staging, per (host thread, device): a thread may drive
// models on several GPUs
thread_local std::unique_ptr<RenderBuffers> t_rb_dev[64];
RenderBuffers& render_buffers(int device) {
  require(device >= 0 && device < 64, "render: device ordinal out of range");
  auto& rb = t_rb_dev[device];
  if (!rb) rb = std::make_unique<RenderBuffers>();
  return *rb;
}

void validate_render(const HostCamera& cam, const arfx_render_options* opt, int shard, int nshards) {
  validate_camera(cam);
  require(opt != nullptr, "render: null options");
  require(opt->samples_per_ray <= 1024, "render: libarfx supports samples_per_ray <= 1024");
  require(nshards >= 1 && shard >= 0 && shard < nshards, "render: bad shard");
}
}  // namespace
namespace {
template <typename T>
struct Staged {
  DevBuf<T> d;
  void up(const T* h, size_t n, cudaStream_t s) {
    d.alloc(n);
    h2d(d.ptr, h, n, s);
  }
};
}  // namespace
namespace {
void ray_offsets(int n_rays, const int32_t* ray_len, std::vector<int64_t>& off) {
  off.assign(static_cast<size_t>(n_rays) + 1, 0);
  for (int r = 0; r < n_rays; ++r) {
    require(ray_len[r] >= 0, "composite: negative ray length");
    off[static_cast<size_t>(r) + 1] = off[static_cast<size_t>(r)] + ray_len[r];
  }
}
}  // namespace
}  // namespace arfx

namespace arfx {
namespace {
// CapsuleFigure::validate (R/scene.hpp:19-26) + PosedFigure ctor (:61-75)
FigureView figure_view_of(const arfx_figure* fig, const double* bones12) {
  require(fig != nullptr, "figure: null");
  const std::vector<HostBone> bones = bones_of(&fig->skeleton);
  validate_skeleton(bones);
  for (int i = 0; i < fig->skeleton.n_bones; ++i)
    if (!(fig->amplitude[i] > 0)) throw std::invalid_argument("figure: amplitudes must be positive");
  if (!(fig->softness > 0)) throw std::invalid_argument("figure: softness must be positive");
  FigureView F{};
  F.nb = fig->skeleton.n_bones;
  F.soft = fig->softness;
  for (int i = 0; i < F.nb; ++i) {
    const HostBone& b = bones[static_cast<size_t>(i)];
    HV a = b.head, t = b.tail;
    if (bones12) {
      a = rigid_apply(bones12 + 12 * i, b.head);
      t = rigid_apply(bones12 + 12 * i, b.tail);
    }
    F.a[i][0] = a.x, F.a[i][1] = a.y, F.a[i][2] = a.z;
    F.b[i][0] = t.x, F.b[i][1] = t.y, F.b[i][2] = t.z;
    F.radius[i] = b.radius;
    F.amp[i] = fig->amplitude[i];
    for (int c = 0; c < 3; ++c) F.col[i][c] = fig->color[i][c];
  }
  return F;
}

struct FigureFrame {
  FigureView F;
  HostCamera cam;
  double w2n[12];
};

FigureFrame figure_frame(const arfx_figure* fig, const double* bones12, const double* global12,
                         const double* lo, const double* hi, const arfx_camera* cam, const arfx_render_options* opt) {
  require(bones12 && global12 && lo && hi && opt, "figure_render: null argument");
  FigureFrame f;
  f.F = figure_view_of(fig, bones12);
  f.cam = camera_of(cam);
  validate_camera(f.cam);
  require(opt->samples_per_ray >= 0, "figure_render: negative samples_per_ray");
  rigid_inverse(global12, f.w2n);
  return f;
}
}  // namespace
}  // namespace arfx

using namespace arfx;

extern "C" {

const char* arfx_last_error(void) { return g_err.c_str(); }
const char* arfx_version(void) { return "arfx 0.1 (sm_100a)"; }

int arfx_device_count(int* n) {
  return guard([&] {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *n = c;
  });
}

int arfx_set_device(int device) { return guard([&] { ARFX_CUDA(cudaSetDevice(device)); }); }

int arfx_level_resolutions(const arfx_grid_config* g, int* out) {
  return guard([&] {
    const auto r = level_resolutions(grid_of(g));
    std::copy(r.begin(), r.end(), out);
  });
}

int arfx_model_sizes(const arfx_skeleton* s, const arfx_grid_config* g, const arfx_mlp_config* mc,
                     const int skin_res[3], size_t* n_grid, size_t* n_mlp, size_t* n_skin) {
  return guard([&] {
    const GridCfg gc = grid_of(g);
    validate_grid_cfg(gc);
    *n_grid = static_cast<size_t>(gc.levels) * (static_cast<size_t>(1) << gc.log2T) * static_cast<size_t>(gc.F);
    *n_mlp = static_cast<size_t>(mlp_layout(gc.levels * gc.F, mc->hidden_dim, mc->hidden_layers, mc->output_dim).n_params);
    *n_skin = static_cast<size_t>(skin_res[0]) * skin_res[1] * skin_res[2] * static_cast<size_t>(s->n_bones);
  });
}

int arfx_pose_from_joint_rotations(const arfx_skeleton* s, const double* rot9, const double* g12,
                                   double* out12) {
  return guard([&] {
    const auto b = bones_of(s);
    pose_from_joint_rotations(b, rot9, g12, out12);
  });
}

int arfx_camera_look_at(const double eye[3], const double target[3], const double up[3], double focal,
                        int width, int height, arfx_camera* out) {
  return guard([&] {
    const HostCamera c = look_at({eye[0], eye[1], eye[2]}, {target[0], target[1], target[2]},
                                 {up[0], up[1], up[2]}, focal, width, height);
    out->fx = c.fx;
    out->fy = c.fy;
    out->cx = c.cx;
    out->cy = c.cy;
    out->width = c.width;
    out->height = c.height;
    std::memcpy(out->extrinsic, c.ext, sizeof(c.ext));
  });
}

int arfx_pose_context(const arfx_skeleton* s, const double* bones12, const double* pre12, double cutoff,
                      double* ob, double* obi, double* ca, double* cb, double* co) {
  return guard([&] {
    const auto b = bones_of(s);
    PoseCtx ctx;
    make_pose_ctx(b, bones12, pre12, cutoff, ctx);
    for (int i = 0; i < ctx.nb; ++i) {
      std::memcpy(ob + 12 * i, ctx.bone[i], 12 * sizeof(double));
      std::memcpy(obi + 12 * i, ctx.bone_inv[i], 12 * sizeof(double));
      std::memcpy(ca + 3 * i, ctx.cap_a[i], 3 * sizeof(double));
      std::memcpy(cb + 3 * i, ctx.cap_b[i], 3 * sizeof(double));
      co[i] = ctx.cutoff[i];
    }
  });
}

// build_model<float>  R/model.hpp:68-80
int arfx_build_model(const arfx_skeleton* s, const arfx_grid_config* g, const arfx_mlp_config* mc,
                     const int skin_res[3], uint64_t seed, arfx_model* out) {
  return guard([&] {
    require(out != nullptr && mc != nullptr && skin_res != nullptr, "build_model: null argument");
    const auto bones = bones_of(s);
    validate_skeleton(bones);
    require_device();
    auto h = std::make_unique<arfx_model_s>();
    ModelImpl& m = h->impl;
    m.canon = rest_bounds(bones, 0.10);
    GridCfg gc = grid_of(g);
    gc.box = m.canon;
    setup_model(m, bones, gc, mc->hidden_dim, mc->hidden_layers, mc->output_dim, skin_res);
    for (const HostBone& b : bones) {  // R/skinning.hpp:67-69
      const double dx = b.tail.x - b.head.x, dy = b.tail.y - b.head.y, dz = b.tail.z - b.head.z;
      require(std::sqrt(dx * dx + dy * dy + dz * dz) > 0, "skinning grid: degenerate zero-length bone");
    }
    m.skin_box = m.canon;
    m.norm = normalized_reach_box(bones, 1.05);
    alloc_model(m);
    init_params_dev(m, seed);
    build_skinning_grid_dev(m, 1.5);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
    build_cell_table(m);
    fill_field_view(m);
    *out = h.release();
  });
}

int arfx_model_create(const arfx_model_desc* d, const float* grid_params, const float* mlp_params,
                      const double* skin_weights, arfx_model* out) {
  return guard([&] {
    require(d != nullptr && out != nullptr && grid_params && mlp_params && skin_weights,
            "model_create: null argument");
    require_device();
    auto h = std::make_unique<arfx_model_s>();
    ModelImpl& m = h->impl;
    const auto bones = bones_of(&d->skeleton);
    setup_model(m, bones, grid_of(&d->grid), d->mlp.hidden_dim, d->mlp.hidden_layers, d->mlp.output_dim,
                d->skin_res);
    require(d->mlp.input_dim == m.mlp_in, "model_create: mlp input_dim must equal levels*features");
    require(d->n_grid_params == m.n_grid && d->n_mlp_params == m.n_mlp && d->n_skin_weights == m.n_skin,
            "model_create: array sizes do not match the configs");
    m.skin_box = HostBox{{d->skin_lo[0], d->skin_lo[1], d->skin_lo[2]}, {d->skin_hi[0], d->skin_hi[1], d->skin_hi[2]}};
    m.canon = HostBox{{d->canonical_lo[0], d->canonical_lo[1], d->canonical_lo[2]},
                      {d->canonical_hi[0], d->canonical_hi[1], d->canonical_hi[2]}};
    m.norm = HostBox{{d->normalized_lo[0], d->normalized_lo[1], d->normalized_lo[2]},
                     {d->normalized_hi[0], d->normalized_hi[1], d->normalized_hi[2]}};
    m.inv = InverseOpts{d->inverse.max_iterations, d->inverse.tolerance, d->inverse.dedup_radius};
    alloc_model(m);
    h2d(m.grid_params.ptr, grid_params, m.n_grid, m.stream);
    h2d(m.mlp_params.ptr, mlp_params, m.n_mlp, m.stream);
    h2d(m.skin.ptr, skin_weights, m.n_skin, m.stream);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
    build_cell_table(m);
    fill_field_view(m);
    *out = h.release();
  });
}

int arfx_model_destroy(arfx_model m) {
  return guard([&] { delete m; });
}

int arfx_model_describe(arfx_model mh, arfx_model_desc* d) {
  return guard([&] {
    require(mh && d, "describe: null");
    ModelImpl& m = mh->impl;
    std::memset(d, 0, sizeof(*d));
    d->skeleton.n_bones = static_cast<int>(m.bones.size());
    for (size_t i = 0; i < m.bones.size(); ++i) {
      const HostBone& b = m.bones[i];
      d->skeleton.parent[i] = b.parent;
      d->skeleton.head[i][0] = b.head.x;
      d->skeleton.head[i][1] = b.head.y;
      d->skeleton.head[i][2] = b.head.z;
      d->skeleton.tail[i][0] = b.tail.x;
      d->skeleton.tail[i][1] = b.tail.y;
      d->skeleton.tail[i][2] = b.tail.z;
      d->skeleton.radius[i] = b.radius;
    }
    d->grid = arfx_grid_config{m.grid.levels, m.grid.F, m.grid.log2T, m.grid.nmin, m.grid.nmax,
                               {m.grid.box.lo.x, m.grid.box.lo.y, m.grid.box.lo.z},
                               {m.grid.box.hi.x, m.grid.box.hi.y, m.grid.box.hi.z}};
    d->mlp = arfx_mlp_config{m.mlp_in, m.mlp_hidden, m.mlp_hl, m.mlp_out};
    for (int a = 0; a < 3; ++a) d->skin_res[a] = m.skin_res[a];
    const HostBox* boxes[3] = {&m.skin_box, &m.canon, &m.norm};
    double* los[3] = {d->skin_lo, d->canonical_lo, d->normalized_lo};
    double* his[3] = {d->skin_hi, d->canonical_hi, d->normalized_hi};
    for (int k = 0; k < 3; ++k) {
      los[k][0] = boxes[k]->lo.x;
      los[k][1] = boxes[k]->lo.y;
      los[k][2] = boxes[k]->lo.z;
      his[k][0] = boxes[k]->hi.x;
      his[k][1] = boxes[k]->hi.y;
      his[k][2] = boxes[k]->hi.z;
    }
    d->inverse = arfx_inverse_options{m.inv.max_iterations, m.inv.tolerance, m.inv.dedup_radius};
    d->n_grid_params = m.n_grid;
    d->n_mlp_params = m.n_mlp;
    d->n_skin_weights = m.n_skin;
  });
}

int arfx_model_get_params(arfx_model mh, float* gp, float* mp, double* sw) {
  return guard([&] {
    require(mh != nullptr, "null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (gp) d2h(gp, m.grid_params.ptr, m.n_grid, m.stream);
    if (mp) d2h(mp, m.mlp_params.ptr, m.n_mlp, m.stream);
    if (sw) d2h(sw, m.skin.ptr, m.n_skin, m.stream);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
  });
}

int arfx_model_set_params(arfx_model mh, const float* gp, const float* mp) {
  return guard([&] {
    require(mh != nullptr, "null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (gp) h2d(m.grid_params.ptr, gp, m.n_grid, m.stream);
    if (mp) h2d(m.mlp_params.ptr, mp, m.n_mlp, m.stream);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
  });
}

int arfx_model_set_mlp_mode(arfx_model mh, int mode) {
  return guard([&] {
    require(mh != nullptr, "set_mlp_mode: null model");
    require(mode == ARFX_MLP_EXACT || mode == ARFX_MLP_TCGEN05 || mode == ARFX_MLP_TCGEN05_FP16,
            "set_mlp_mode: unknown mode");
    mh->impl.mlp_mode = mode;
  });
}

int arfx_model_set_backward_mode(arfx_model mh, int mode) {
  return guard([&] {
    require(mh != nullptr, "set_backward_mode: null model");
    require(mode == ARFX_BWD_SIMT || mode == ARFX_BWD_TCGEN05, "set_backward_mode: unknown mode");
    mh->impl.bwd_tc = mode == ARFX_BWD_TCGEN05;
  });
}

int arfx_model_set_deterministic(arfx_model mh, int on) {
  return guard([&] {
    require(mh != nullptr, "set_deterministic: null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (!on && m.acc_pending) {
      ARFX_CUDA(cudaDeviceSynchronize());
      flush_grad_acc(m, m.stream);
      ARFX_CUDA(cudaStreamSynchronize(m.stream));
    }
    m.det = on != 0;
  });
}

int arfx_model_zero_grad(arfx_model mh, void* stream) {
  return guard([&] {
    require(mh != nullptr, "null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    ensure_grad_store(m, m.stream);
    const cudaStream_t s = stream_of(m, stream);
    ARFX_CUDA(cudaMemsetAsync(m.flat_grads.ptr, 0, m.n_flat * sizeof(float), s));
    if (m.acc_pending) {  // pending deterministic-mode sums are discarded too
      ARFX_CUDA(cudaMemsetAsync(m.grid_acc.ptr, 0, m.grid_acc.n * sizeof(long long), s));
      m.acc_pending = false;
    }
  });
}

int arfx_model_set_param_fence(arfx_model mh, void* event) {
  return guard([&] {
    require(mh != nullptr, "set_param_fence: null model");
    mh->impl.param_fence = static_cast<cudaEvent_t>(event);
  });
}

int arfx_model_flush_grads(arfx_model mh, void* stream) {
  return guard([&] {
    require(mh != nullptr, "flush_grads: null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    flush_grad_acc(m, stream_of(m, stream));
  });
}

int arfx_model_get_grads(arfx_model mh, float* gg, float* mg) {
  return guard([&] {
    require(mh != nullptr, "null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    require(m.grid_grad.ptr != nullptr, "no gradients accumulated yet (call arfx_model_zero_grad)");
    if (m.acc_pending) {
      ARFX_CUDA(cudaDeviceSynchronize());  // the backward may have run on a caller stream
      flush_grad_acc(m, m.stream);
    }
    if (gg) d2h(gg, m.grid_grad.ptr, m.n_grid, m.stream);
    if (mg) d2h(mg, m.mlp_grad.ptr, m.n_mlp, m.stream);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
  });
}

int arfx_model_device_arrays(arfx_model mh, float** gp, float** mp, float** gg, float** mg) {
  return guard([&] {
    require(mh != nullptr, "null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    ensure_grad_store(m, m.stream);
    if (gp) *gp = m.grid_params.ptr;
    if (mp) *mp = m.mlp_params.ptr;
    if (gg) *gg = m.grid_grad.ptr;
    if (mg) *mg = m.mlp_grad.ptr;
  });
}

int arfx_pose_create(arfx_model mh, const double* bones12, const double* global12, arfx_pose* out) {
  return guard([&] {
    require(mh != nullptr && out != nullptr, "pose_create: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    auto p = std::make_unique<arfx_pose_s>();
    p->impl.model = &m;
    make_pose_host(m, bones12, global12, p->impl.host);
    p->impl.dev.alloc(1);
    ARFX_CUDA(cudaMemcpyAsync(p->impl.dev.ptr, &p->impl.host, sizeof(PoseCtx), cudaMemcpyHostToDevice, m.stream));
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
    *out = p.release();
  });
}

int arfx_pose_create_context(arfx_model mh, const double* bones12, const double* pre12, double cutoff,
                             arfx_pose* out) {
  return guard([&] {
    require(mh != nullptr && out != nullptr, "pose_create_context: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    auto p = std::make_unique<arfx_pose_s>();
    p->impl.model = &m;
    make_pose_ctx(m.bones, bones12, pre12, cutoff, p->impl.host);
    p->impl.dev.alloc(1);
    ARFX_CUDA(cudaMemcpyAsync(p->impl.dev.ptr, &p->impl.host, sizeof(PoseCtx), cudaMemcpyHostToDevice, m.stream));
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
    *out = p.release();
  });
}

int arfx_pose_update(arfx_pose ph, const double* bones12, const double* global12, void* stream) {
  return guard([&] {
    require(ph != nullptr, "pose_update: null pose");
    PoseImpl& p = ph->impl;
    ModelImpl& m = *p.model;
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    make_pose_host(m, bones12, global12, p.host);
    ARFX_CUDA(cudaMemcpyAsync(p.dev.ptr, &p.host, sizeof(PoseCtx), cudaMemcpyHostToDevice, s));
    ARFX_CUDA(cudaStreamSynchronize(s));
  });
}

int arfx_pose_update_async(arfx_pose ph, const double* bones12, const double* global12, void* stream) {
  return guard([&] {
    require(ph != nullptr, "pose_update: null pose");
    PoseImpl& p = ph->impl;
    ModelImpl& m = *p.model;
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    make_pose_host(m, bones12, global12, p.host);
    if (!p.ring) {
      ARFX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p.ring), PoseImpl::kRing * sizeof(PoseCtx),
                              cudaHostAllocDefault));
      for (auto& e : p.ring_ev) ARFX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int k = p.ring_next;
    p.ring_next = (k + 1) % PoseImpl::kRing;
    ARFX_CUDA(cudaEventSynchronize(p.ring_ev[k]));  // this staging slot's last copy has run
    p.ring[k] = p.host;
    ARFX_CUDA(cudaMemcpyAsync(p.dev.ptr, p.ring + k, sizeof(PoseCtx), cudaMemcpyHostToDevice, s));
    ARFX_CUDA(cudaEventRecord(p.ring_ev[k], s));
  });
}

int arfx_pose_destroy(arfx_pose p) {
  return guard([&] { delete p; });
}

// OccupancyGrid::empty  R/occupancy.hpp:59-69
int arfx_occ_create(const double lo[3], const double hi[3], const arfx_occ_config* cfg, arfx_occ_grid* out) {
  return guard([&] {
    require(cfg && out && lo && hi, "occ_create: null argument");
    validate_occ_cfg(cfg->resolution, cfg->alpha_threshold, cfg->dilation, cfg->decay, cfg->update_interval);
    require_device();
    auto g = std::make_unique<arfx_occ_s>();
    OccImpl& o = g->impl;
    ARFX_CUDA(cudaGetDevice(&o.device));
    o.res = cfg->resolution;
    o.box = HostBox{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
    o.dilation = cfg->dilation;
    o.threshold = occupancy_threshold(o.box, o.res, cfg->alpha_threshold);
    const size_t n = static_cast<size_t>(o.res) * o.res * o.res;
    o.values.alloc(n);
    o.mask.alloc(n);
    ARFX_CUDA(cudaMemset(o.values.ptr, 0, n * sizeof(float)));
    ARFX_CUDA(cudaMemset(o.mask.ptr, 0, n));
    *out = g.release();
  });
}

// arf::OccupancyGrid members as stored (R/occupancy.hpp:37-48): checkpoint restore
int arfx_occ_create_raw(const double lo[3], const double hi[3], int resolution, double density_threshold,
                        int dilation, arfx_occ_grid* out) {
  return guard([&] {
    require(lo && hi && out, "occ_create_raw: null argument");
    require(resolution >= 1 && resolution <= 1024, "occupancy: resolution out of range");
    require(dilation >= 0, "occupancy: negative dilation");
    require(std::isfinite(density_threshold), "occupancy: non-finite threshold");
    require_device();
    auto g = std::make_unique<arfx_occ_s>();
    OccImpl& o = g->impl;
    ARFX_CUDA(cudaGetDevice(&o.device));
    o.res = resolution;
    o.box = HostBox{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
    o.dilation = dilation;
    o.threshold = density_threshold;
    const size_t n = static_cast<size_t>(o.res) * o.res * o.res;
    o.values.alloc(n);
    o.mask.alloc(n);
    ARFX_CUDA(cudaMemset(o.values.ptr, 0, n * sizeof(float)));
    ARFX_CUDA(cudaMemset(o.mask.ptr, 0, n));
    *out = g.release();
  });
}

int arfx_occ_destroy(arfx_occ_grid g) {
  return guard([&] { delete g; });
}

int arfx_occ_info(arfx_occ_grid gh, int res[3], double lo[3], double hi[3], double* thr, int* dil) {
  return guard([&] {
    OccImpl& g = occ_ref(gh);
    if (res) res[0] = res[1] = res[2] = g.res;
    if (lo) {
      lo[0] = g.box.lo.x;
      lo[1] = g.box.lo.y;
      lo[2] = g.box.lo.z;
    }
    if (hi) {
      hi[0] = g.box.hi.x;
      hi[1] = g.box.hi.y;
      hi[2] = g.box.hi.z;
    }
    if (thr) *thr = g.threshold;
    if (dil) *dil = g.dilation;
  });
}

int arfx_occ_download(arfx_occ_grid gh, float* values, uint8_t* mask) {
  return guard([&] {
    OccImpl& g = occ_ref(gh);
    ARFX_CUDA(cudaSetDevice(g.device));
    ARFX_CUDA(cudaDeviceSynchronize());
    const size_t n = static_cast<size_t>(g.res) * g.res * g.res;
    if (values) ARFX_CUDA(cudaMemcpy(values, g.values.ptr, n * sizeof(float), cudaMemcpyDeviceToHost));
    if (mask) ARFX_CUDA(cudaMemcpy(mask, g.mask.ptr, n, cudaMemcpyDeviceToHost));
  });
}

int arfx_occ_upload(arfx_occ_grid gh, const float* values, const uint8_t* mask) {
  return guard([&] {
    OccImpl& g = occ_ref(gh);
    ARFX_CUDA(cudaSetDevice(g.device));
    ARFX_CUDA(cudaDeviceSynchronize());  // order after asynchronous builds on model streams
    const size_t n = static_cast<size_t>(g.res) * g.res * g.res;
    if (values) ARFX_CUDA(cudaMemcpy(g.values.ptr, values, n * sizeof(float), cudaMemcpyHostToDevice));
    if (mask) ARFX_CUDA(cudaMemcpy(g.mask.ptr, mask, n, cudaMemcpyHostToDevice));
  });
}

int arfx_occ_rebuild_mask(arfx_occ_grid gh, void* stream) {
  return guard([&] {
    OccImpl& g = occ_ref(gh);
    ARFX_CUDA(cudaSetDevice(g.device));
    if (!stream) ARFX_CUDA(cudaDeviceSynchronize());  // legacy stream: order after model streams
    occ_rebuild(g, static_cast<cudaStream_t>(stream));
    ARFX_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  });
}

int arfx_build_inference_grid(arfx_model mh, arfx_pose ph, arfx_occ_grid gh, arfx_counters* c, void* stream) {
  return guard([&] {
    require(mh && ph, "build_inference_grid: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    if (!c) {
      // no counters requested: reserve the worst case (every cell keeps 8 roots / starts on
      // every bone) so nothing can overflow, and return without a host round trip; the grid
      // is complete for any later work on the same stream
      const OccImpl& g = occ_ref(gh);
      m.ws().reserve_worst(static_cast<size_t>(g.res) * g.res * g.res, static_cast<size_t>(m.sv.nb));
      inference_grid(m, ph->impl, occ_ref(gh), nullptr, s);
      return;
    }
    for (int attempt = 0; attempt < 3; ++attempt) {
      inference_grid(m, ph->impl, occ_ref(gh), nullptr, s);
      unsigned long long hc[8];
      d2h(hc, m.ws().counters.ptr, 8, s);
      ARFX_CUDA(cudaStreamSynchronize(s));
      bool rerun;
      check_overflow_and_grow(m, hc, rerun);
      if (rerun) continue;
      if (c) {
        c->posed_queries = hc[0] ? hc[0] : static_cast<uint64_t>(occ_ref(gh).res) * occ_ref(gh).res * occ_ref(gh).res;
        c->canonical_queries = hc[1];
      }
      return;
    }
    throw std::runtime_error("build_inference_grid: workspace overflow persisted");
  });
}

int arfx_build_inference_grid_device(arfx_model mh, arfx_pose ph, arfx_occ_grid gh, uint64_t* d_counters,
                                     void* stream) {
  return guard([&] {
    require(mh && ph, "build_inference_grid_device: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    inference_grid(m, ph->impl, occ_ref(gh), reinterpret_cast<unsigned long long*>(d_counters),
                   stream_of(m, stream));
  });
}

int arfx_build_inference_grid_shard_device(arfx_model mh, arfx_pose ph, arfx_occ_grid gh, int shard,
                                           int n_shards, uint64_t* d_counters, void* stream) {
  return guard([&] {
    require(mh && ph, "build_inference_grid_shard: null argument");
    require(n_shards >= 1 && shard >= 0 && shard < n_shards, "build_inference_grid_shard: bad shard");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    inference_grid_shard(m, ph->impl, occ_ref(gh), shard, n_shards, reinterpret_cast<unsigned long long*>(d_counters),
                         stream_of(m, stream));
  });
}

int arfx_occ_device_arrays(arfx_occ_grid gh, float** values, uint8_t** mask) {
  return guard([&] {
    OccImpl& g = occ_ref(gh);
    if (values) *values = g.values.ptr;
    if (mask) *mask = g.mask.ptr;
  });
}

int arfx_occ_rebuild_mask_async(arfx_occ_grid gh, void* stream) {
  return guard([&] {
    OccImpl& g = occ_ref(gh);
    ARFX_CUDA(cudaSetDevice(g.device));
    occ_rebuild(g, static_cast<cudaStream_t>(stream));
  });
}

int arfx_occ_rebuild_mask_shards_async(arfx_occ_grid gh, int n_shards, void* stream) {
  return guard([&] {
    require(n_shards >= 1, "occ_rebuild_mask_shards: n_shards >= 1");
    OccImpl& g = occ_ref(gh);
    ARFX_CUDA(cudaSetDevice(g.device));
    occ_unshard(g, n_shards, static_cast<cudaStream_t>(stream));
    occ_rebuild(g, static_cast<cudaStream_t>(stream));
  });
}

int arfx_update_training_grid(arfx_model mh, const arfx_pose* poses, int n_poses, double decay,
                              uint64_t seed, uint64_t step, arfx_occ_grid gh, arfx_counters* c, void* stream) {
  return guard([&] {
    require(mh && poses && n_poses >= 1, "update_training_grid: need >= 1 pose");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    std::vector<PoseImpl*> ps;
    for (int i = 0; i < n_poses; ++i) {
      require(poses[i] != nullptr, "update_training_grid: null pose");
      ps.push_back(&poses[i]->impl);
    }
    OccImpl& g = occ_ref(gh);
    const size_t n = static_cast<size_t>(g.res) * g.res * g.res;
    DevBuf<float>& saved = g.saved;  // values are updated in place: keep a copy for overflow reruns
    saved.ensure(n);
    ARFX_CUDA(cudaMemcpyAsync(saved.ptr, g.values.ptr, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
    for (int attempt = 0; attempt < 3; ++attempt) {
      if (attempt)
        ARFX_CUDA(cudaMemcpyAsync(g.values.ptr, saved.ptr, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
      training_grid_update(m, ps, decay, seed, step, g, nullptr, s);
      unsigned long long hc[8];
      d2h(hc, m.ws().counters.ptr, 8, s);
      ARFX_CUDA(cudaStreamSynchronize(s));
      bool rerun;
      check_overflow_and_grow(m, hc, rerun);
      if (rerun) continue;
      if (c) {
        c->posed_queries = n;
        c->canonical_queries = hc[1];
      }
      return;
    }
    throw std::runtime_error("update_training_grid: workspace overflow persisted");
  });
}

int arfx_update_training_grid_device(arfx_model mh, const arfx_pose* poses, int n_poses, double decay,
                                     uint64_t seed, uint64_t step, arfx_occ_grid gh, uint64_t* d_counters,
                                     void* stream) {
  return guard([&] {
    require(mh && poses && n_poses >= 1, "update_training_grid: need >= 1 pose");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    std::vector<PoseImpl*> ps;
    for (int i = 0; i < n_poses; ++i) {
      require(poses[i] != nullptr, "update_training_grid: null pose");
      ps.push_back(&poses[i]->impl);
    }
    OccImpl& g = occ_ref(gh);
    const size_t n = static_cast<size_t>(g.res) * g.res * g.res;
    // no host round trip, so no overflow re-run: the workspace is sized for the worst case
    // (every bone a start, kMaxRoots roots per cell), which cannot overflow
    m.ws().reserve_worst(n, static_cast<size_t>(m.sv.nb));
    training_grid_update(m, ps, decay, seed, step, g, reinterpret_cast<unsigned long long*>(d_counters), s);
  });
}

int arfx_render_model_device(arfx_model mh, arfx_pose ph, const arfx_camera* cam, arfx_occ_grid occ,
                             const arfx_render_options* opt, int shard, int nshards, float* d_rgb,
                             float* d_alpha, uint64_t* d_counters, void* stream) {
  return guard([&] {
    require(mh && ph && d_rgb && d_alpha, "render_model_device: null argument");
    ModelImpl& m = mh->impl;
    const HostCamera hc = camera_of(cam);
    validate_render(hc, opt, shard, nshards);
    ARFX_CUDA(cudaSetDevice(m.device));
    render_frame(m, ph->impl, hc, occ ? &occ->impl : nullptr, opt->samples_per_ray, opt->stratified != 0,
                 opt->epsilon_terminate, opt->seed, opt->frame_id, shard, nshards, d_rgb, d_alpha,
                 reinterpret_cast<unsigned long long*>(d_counters), stream_of(m, stream));
  });
}

// ---- CUDA-graph frames -------------------------------------------------------------------
// The pose is read by every kernel from its device PoseContext, so a graph captured for a
// pose handle replays correctly after the handle is updated in place (arfx_pose_update /
// arfx_pose_copy). The workspace is sized by an uncaptured warm-up run of the same parts.

int arfx_pose_copy(arfx_pose dst, arfx_pose src, void* stream) {
  return guard([&] {
    require(dst && src, "pose_copy: null pose");
    require(dst->impl.model == src->impl.model, "pose_copy: poses of different models");
    ModelImpl& m = *dst->impl.model;
    ARFX_CUDA(cudaSetDevice(m.device));
    dst->impl.host = src->impl.host;
    ARFX_CUDA(cudaMemcpyAsync(dst->impl.dev.ptr, src->impl.dev.ptr, sizeof(PoseCtx), cudaMemcpyDeviceToDevice,
                              stream_of(m, stream)));
  });
}

int arfx_frame_graph_create(arfx_model mh, arfx_pose ph, const arfx_camera* cam, arfx_occ_grid occ,
                            const arfx_render_options* opt, int shard, int nshards, int parts, float* d_rgb,
                            float* d_alpha, uint64_t* d_counters, void* stream, arfx_frame_graph* out) {
  return guard([&] {
    require(mh && ph && out, "frame_graph_create: null argument");
    require(parts > 0 && (parts & ~(ARFX_GRAPH_GRID | ARFX_GRAPH_GRID_SHARD | ARFX_GRAPH_MASK | ARFX_GRAPH_RENDER |
                                    ARFX_GRAPH_MASK_SHARDS | ARFX_GRAPH_SIDE_WORKSPACE)) == 0,
            "frame_graph_create: bad parts");
    require(!((parts & ARFX_GRAPH_MASK) && (parts & ARFX_GRAPH_MASK_SHARDS)), "frame_graph_create: mask or shard mask");
    require(!((parts & ARFX_GRAPH_GRID) && (parts & ARFX_GRAPH_GRID_SHARD)), "frame_graph_create: grid or shard");
    require(!(parts & (ARFX_GRAPH_GRID | ARFX_GRAPH_GRID_SHARD | ARFX_GRAPH_MASK | ARFX_GRAPH_MASK_SHARDS)) || occ,
            "frame_graph_create: the grid parts need an occupancy grid");
    require(!(parts & ARFX_GRAPH_RENDER) || (d_rgb && d_alpha && opt), "frame_graph_create: render outputs");
    require(d_counters != nullptr || !(parts & (ARFX_GRAPH_GRID | ARFX_GRAPH_GRID_SHARD | ARFX_GRAPH_RENDER)),
            "frame_graph_create: d_counters is required (a replay reports workspace overflow in d_counters[4 + 3])");
    ModelImpl& m = mh->impl;
    HostCamera hc{};
    if (parts & ARFX_GRAPH_RENDER) {
      hc = camera_of(cam);
      validate_render(hc, opt, shard, nshards);
    }
    require(nshards >= 1 && shard >= 0 && shard < nshards, "frame_graph_create: bad shard");
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    require(s != nullptr, "frame_graph_create: needs a non-NULL stream");
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(d_counters);
    // SIDE_WORKSPACE: capture on the model's side workspace, so this graph may run
    // concurrently with one captured on the main workspace (e.g. the next frame's grid shard
    // beside the current frame's render)
    WorkspaceScope scope(m, (parts & ARFX_GRAPH_SIDE_WORKSPACE) ? m.ws_side : m.ws());
    auto enqueue = [&] {
      if (parts & ARFX_GRAPH_GRID) inference_grid(m, ph->impl, occ->impl, cnt, s);
      if (parts & ARFX_GRAPH_GRID_SHARD) inference_grid_shard(m, ph->impl, occ->impl, shard, nshards, cnt, s);
      if (parts & ARFX_GRAPH_MASK) occ_rebuild(occ->impl, s);
      if (parts & ARFX_GRAPH_MASK_SHARDS) {
        occ_unshard(occ->impl, nshards, s);
        occ_rebuild(occ->impl, s);
      }
      if (parts & ARFX_GRAPH_RENDER)
        render_frame(m, ph->impl, hc, occ ? &occ->impl : nullptr, opt->samples_per_ray, opt->stratified != 0,
                     opt->epsilon_terminate, opt->seed, opt->frame_id, shard, nshards, d_rgb, d_alpha,
                     cnt ? cnt + 4 : nullptr, s);
    };
    // warm-up (uncaptured): sizes the workspace for the worst case of the grid parts and
    // sets kernel attributes; the render workspace grows from its counters if needed
    if (occ && (parts & (ARFX_GRAPH_GRID | ARFX_GRAPH_GRID_SHARD)))
      m.ws().reserve_worst(static_cast<size_t>(occ->impl.res) * occ->impl.res * occ->impl.res,
                         static_cast<size_t>(m.sv.nb));
    for (int attempt = 0; attempt < 3; ++attempt) {
      enqueue();
      unsigned long long hcnt[8];
      d2h(hcnt, m.ws().counters.ptr, 8, s);
      ARFX_CUDA(cudaStreamSynchronize(s));
      bool rerun;
      check_overflow_and_grow(m, hcnt, rerun);
      if (!rerun) break;
    }
    const bool prof = m.prof.on;
    m.prof.on = false;  // no event records inside the graph
    auto g = std::make_unique<arfx_frame_graph_s>();
    g->device = m.device;
    ARFX_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    try {
      enqueue();
    } catch (...) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(s, &junk);
      if (junk) cudaGraphDestroy(junk);
      m.prof.on = prof;
      throw;
    }
    ARFX_CUDA(cudaStreamEndCapture(s, &g->graph));
    m.prof.on = prof;
    ARFX_CUDA(cudaGraphInstantiate(&g->exec, g->graph, 0));
    g->ws = &m.ws();
    g->ws_gen = m.ws().gen;
    *out = g.release();
  });
}

// Pipelined animation frame: one graph with two concurrent branches -- the inference grid of
// the NEXT pose (pose handle p_next -> occ_next, on the model's side stream and side
// workspace) and the render of the CURRENT pose with its already-built grid (p_cur, occ_cur,
// main workspace). Alternating two such graphs with the roles of (p, occ) swapped renders an
// animation with each frame's grid build overlapping the previous frame's render; every frame
// is bit-identical to a direct grid + render (test_pipelined_frame_graphs_match_direct).
// d_counters [2][4]: the next grid's counters, then the render's.
namespace {
// Captures one pipelined frame (the next pose's inference grid on the side stream / side
// workspace beside the current pose's render) as a graph; shared by
// arfx_frame_graph_create_pipelined and the graph cache of arfx_render_model_pipelined_async.
arfx_frame_graph_s* make_pipelined_graph(ModelImpl& m, PoseImpl& pc, OccImpl& oc, PoseImpl& pn, OccImpl& on,
                                         const HostCamera& hc, const arfx_render_options* opt, int shard,
                                         int nshards, float* d_rgb, float* d_alpha, uint64_t* d_counters,
                                         cudaStream_t s) {
  if (!m.side) ARFX_CUDA(cudaStreamCreateWithFlags(&m.side, cudaStreamNonBlocking));
  cudaEvent_t fork = nullptr, join = nullptr;
  ARFX_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  ARFX_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t a, b;
    ~EvGuard() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  } evg{fork, join};
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(d_counters);
  OccImpl& gn = on;
  auto enqueue = [&] {
    ARFX_CUDA(cudaEventRecord(fork, s));
    ARFX_CUDA(cudaStreamWaitEvent(m.side, fork, 0));
    {
      WorkspaceScope side(m, m.ws_side);
      inference_grid(m, pn, gn, cnt, m.side);
    }
    render_frame(m, pc, hc, &oc, opt->samples_per_ray, opt->stratified != 0,
                 opt->epsilon_terminate, opt->seed, opt->frame_id, shard, nshards, d_rgb, d_alpha, cnt + 4, s);
    ARFX_CUDA(cudaEventRecord(join, m.side));
    ARFX_CUDA(cudaStreamWaitEvent(s, join, 0));
  };
  // warm-up (uncaptured): the side workspace for the worst case of a grid build, the main
  // one from the render's counters
  {
    WorkspaceScope side(m, m.ws_side);
    m.ws().reserve_worst(static_cast<size_t>(gn.res) * gn.res * gn.res, static_cast<size_t>(m.sv.nb));
  }
  for (int attempt = 0; attempt < 3; ++attempt) {
    enqueue();
    unsigned long long hcnt[8];
    d2h(hcnt, m.ws().counters.ptr, 8, s);
    ARFX_CUDA(cudaStreamSynchronize(s));
    bool rerun;
    check_overflow_and_grow(m, hcnt, rerun);
    if (!rerun) break;
  }
  const bool prof = m.prof.on;
  m.prof.on = false;
  auto g = std::make_unique<arfx_frame_graph_s>();
  g->device = m.device;
  ARFX_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
  try {
    enqueue();
  } catch (...) {
    cudaGraph_t junk = nullptr;
    cudaStreamEndCapture(s, &junk);
    if (junk) cudaGraphDestroy(junk);
    m.prof.on = prof;
    throw;
  }
  ARFX_CUDA(cudaStreamEndCapture(s, &g->graph));
  m.prof.on = prof;
  ARFX_CUDA(cudaGraphInstantiate(&g->exec, g->graph, 0));
  g->ws = &m.ws_main;
  g->ws_gen = m.ws_main.gen;
  g->ws2 = &m.ws_side;
  g->ws2_gen = m.ws_side.gen;
  return g.release();
}
}  // namespace

int arfx_frame_graph_create_pipelined(arfx_model mh, arfx_pose p_cur, arfx_occ_grid occ_cur, arfx_pose p_next,
                                      arfx_occ_grid occ_next, const arfx_camera* cam, const arfx_render_options* opt,
                                      int shard, int nshards, float* d_rgb, float* d_alpha, uint64_t* d_counters,
                                      void* stream, arfx_frame_graph* out) {
  return guard([&] {
    require(mh && p_cur && occ_cur && p_next && occ_next && out, "frame_graph_create_pipelined: null argument");
    require(occ_cur != occ_next, "frame_graph_create_pipelined: the two grids must differ");
    require(d_rgb && d_alpha && opt && d_counters, "frame_graph_create_pipelined: render outputs and counters");
    ModelImpl& m = mh->impl;
    const HostCamera hc = camera_of(cam);
    validate_render(hc, opt, shard, nshards);
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    require(s != nullptr, "frame_graph_create_pipelined: needs a non-NULL stream");
    *out = make_pipelined_graph(m, p_cur->impl, occ_cur->impl, p_next->impl, occ_next->impl, hc, opt, shard, nshards,
                                d_rgb, d_alpha, d_counters, s);
  });
}

int arfx_frame_graph_launch(arfx_frame_graph g, void* stream) {
  return guard([&] {
    require(g && g->exec, "frame_graph_launch: null graph");
    if (g->ws->gen != g->ws_gen || (g->ws2 && g->ws2->gen != g->ws2_gen))
      throw std::invalid_argument(
          "frame_graph_launch: the model workspace was reallocated since this graph was captured (a larger "
          "render, a camera / shard change or an overflow regrow); destroy the graph and create it again");
    ARFX_CUDA(cudaSetDevice(g->device));
    ARFX_CUDA(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream)));
  });
}

int arfx_frame_graph_destroy(arfx_frame_graph g) {
  return guard([&] { delete g; });
}

int arfx_render_model(arfx_model mh, arfx_pose ph, const arfx_camera* cam, arfx_occ_grid occ,
                      const arfx_render_options* opt, int shard, int nshards, float* rgb, float* alpha,
                      arfx_counters* c, void* stream) {
  return guard([&] {
    require(mh && ph && rgb && alpha, "render_model: null argument");
    ModelImpl& m = mh->impl;
    const HostCamera hc = camera_of(cam);
    validate_render(hc, opt, shard, nshards);
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    RenderBuffers* t_rb = &render_buffers(m.device);
    const size_t npix = static_cast<size_t>(hc.width) * hc.height;
    t_rb->rgb.ensure(npix * 3);
    t_rb->alpha.ensure(npix);
    for (int attempt = 0; attempt < 3; ++attempt) {
      render_frame(m, ph->impl, hc, occ ? &occ->impl : nullptr, opt->samples_per_ray, opt->stratified != 0,
                   opt->epsilon_terminate, opt->seed, opt->frame_id, shard, nshards, t_rb->rgb.ptr,
                   t_rb->alpha.ptr, nullptr, s);
      unsigned long long hcnt[8];
      d2h(hcnt, m.ws().counters.ptr, 8, s);
      // this shard's row tiles (other shards' rows are left untouched), enqueued behind the
      // counters so one synchronisation covers both; on overflow the frame re-runs and
      // copies again. Full tiles of a shard are one strided 2-D copy per image.
      const int W = hc.width, H = hc.height, T = kRowTile;
      const int full_tiles = H / T;  // tiles 0..full_tiles-1 have T rows
      const int first = shard;        // tiles of this shard: first, first + nshards, ...
      const int n_full = first < full_tiles ? (full_tiles - 1 - first) / nshards + 1 : 0;
      if (n_full > 0) {
        const size_t off = static_cast<size_t>(first) * T * W;
        const size_t pitch3 = static_cast<size_t>(nshards) * T * W * 3 * sizeof(float);
        const size_t pitch1 = static_cast<size_t>(nshards) * T * W * sizeof(float);
        ARFX_CUDA(cudaMemcpy2DAsync(rgb + off * 3, pitch3, t_rb->rgb.ptr + off * 3, pitch3,
                                    static_cast<size_t>(T) * W * 3 * sizeof(float), static_cast<size_t>(n_full),
                                    cudaMemcpyDeviceToHost, s));
        ARFX_CUDA(cudaMemcpy2DAsync(alpha + off, pitch1, t_rb->alpha.ptr + off, pitch1,
                                    static_cast<size_t>(T) * W * sizeof(float), static_cast<size_t>(n_full),
                                    cudaMemcpyDeviceToHost, s));
      }
      if (H % T && full_tiles % nshards == shard) {  // the partial last tile
        const size_t off = static_cast<size_t>(full_tiles) * T * W;
        const size_t rows = static_cast<size_t>(H % T);
        d2h(rgb + off * 3, t_rb->rgb.ptr + off * 3, rows * W * 3, s);
        d2h(alpha + off, t_rb->alpha.ptr + off, rows * W, s);
      }
      ARFX_CUDA(cudaStreamSynchronize(s));
      bool rerun;
      check_overflow_and_grow(m, hcnt, rerun);
      if (rerun) continue;
      if (c) {
        c->posed_queries = hcnt[0];
        c->canonical_queries = hcnt[1];
      }
      return;
    }
    throw std::runtime_error("render_model: workspace overflow persisted");
  });
}

// Host-buffer render without a host round trip: the frame renders into one of two device
// image slots on `stream`; the slot's D2H copies (this shard's row tiles, counters) run on
// the model's copy stream while the next frame renders. A slot is re-used only after its
// previous copies completed (device-side wait).
namespace {
// arfx_render_model_async's device side: render into one of two device image slots on `s`,
// then copy this shard's rows to the host buffers on the model's copy stream
// the next async image slot, sized for the camera; the stream waits until its previous
// copies are done
ModelImpl::AsyncSlot& async_slot_acquire(ModelImpl& m, const HostCamera& hc, cudaStream_t s, int& index) {
  if (!m.copy_stream) {
    ARFX_CUDA(cudaStreamCreateWithFlags(&m.copy_stream, cudaStreamNonBlocking));
    for (auto& a : m.async_slot) {
      ARFX_CUDA(cudaEventCreateWithFlags(&a.rendered, cudaEventDisableTiming));
      ARFX_CUDA(cudaEventCreateWithFlags(&a.copied, cudaEventDisableTiming));
    }
  }
  index = m.async_next;
  ModelImpl::AsyncSlot& a = m.async_slot[m.async_next];
  m.async_next ^= 1;
  const size_t npix = static_cast<size_t>(hc.width) * hc.height;
  if (a.rgb.n < npix * 3 || a.counters.n < 8) {
    ARFX_CUDA(cudaDeviceSynchronize());  // growing a slot: nothing in flight may use it
    a.rgb.ensure(npix * 3);
    a.alpha.ensure(npix);
    a.counters.ensure(8);
  }
  ARFX_CUDA(cudaStreamWaitEvent(s, a.copied, 0));  // the slot's previous copies are done
  return a;
}

// after the frame was rendered into slot a on s: its rows (of this shard) and the render
// counters (dev_counters4) to the host buffers on the copy stream
void async_slot_d2h(ModelImpl& m, ModelImpl::AsyncSlot& a, const HostCamera& hc, int shard, int nshards, float* rgb,
                    float* alpha, const unsigned long long* dev_counters4, uint64_t* counters4, cudaStream_t s) {
  ARFX_CUDA(cudaEventRecord(a.rendered, s));
  const cudaStream_t c = m.copy_stream;
  ARFX_CUDA(cudaStreamWaitEvent(c, a.rendered, 0));
  const int W = hc.width, H = hc.height, T = kRowTile;
  const int full_tiles = H / T;
  const int n_full = shard < full_tiles ? (full_tiles - 1 - shard) / nshards + 1 : 0;
  if (n_full > 0) {
    const size_t off = static_cast<size_t>(shard) * T * W;
    const size_t pitch3 = static_cast<size_t>(nshards) * T * W * 3 * sizeof(float);
    const size_t pitch1 = static_cast<size_t>(nshards) * T * W * sizeof(float);
    ARFX_CUDA(cudaMemcpy2DAsync(rgb + off * 3, pitch3, a.rgb.ptr + off * 3, pitch3,
                                static_cast<size_t>(T) * W * 3 * sizeof(float), static_cast<size_t>(n_full),
                                cudaMemcpyDeviceToHost, c));
    ARFX_CUDA(cudaMemcpy2DAsync(alpha + off, pitch1, a.alpha.ptr + off, pitch1,
                                static_cast<size_t>(T) * W * sizeof(float), static_cast<size_t>(n_full),
                                cudaMemcpyDeviceToHost, c));
  }
  if (H % T && full_tiles % nshards == shard) {
    const size_t off = static_cast<size_t>(full_tiles) * T * W;
    const size_t rows = static_cast<size_t>(H % T);
    ARFX_CUDA(cudaMemcpyAsync(rgb + off * 3, a.rgb.ptr + off * 3, rows * W * 3 * sizeof(float),
                              cudaMemcpyDeviceToHost, c));
    ARFX_CUDA(cudaMemcpyAsync(alpha + off, a.alpha.ptr + off, rows * W * sizeof(float), cudaMemcpyDeviceToHost, c));
  }
  if (counters4)
    ARFX_CUDA(cudaMemcpyAsync(counters4, dev_counters4, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost, c));
  ARFX_CUDA(cudaEventRecord(a.copied, c));
}

void render_async_impl(ModelImpl& m, PoseImpl& p, const HostCamera& hc, OccImpl* occ, const arfx_render_options* opt,
                       int shard, int nshards, float* rgb, float* alpha, uint64_t* counters4, cudaStream_t s) {
  int index = 0;
  ModelImpl::AsyncSlot& a = async_slot_acquire(m, hc, s, index);
  render_frame(m, p, hc, occ, opt->samples_per_ray, opt->stratified != 0, opt->epsilon_terminate, opt->seed,
               opt->frame_id, shard, nshards, a.rgb.ptr, a.alpha.ptr, a.counters.ptr, s);
  async_slot_d2h(m, a, hc, shard, nshards, rgb, alpha, a.counters.ptr, counters4, s);
}
}  // namespace

int arfx_render_model_async(arfx_model mh, arfx_pose ph, const arfx_camera* cam, arfx_occ_grid occ,
                            const arfx_render_options* opt, int shard, int nshards, float* rgb, float* alpha,
                            uint64_t* counters4, void* stream) {
  return guard([&] {
    require(mh && ph && rgb && alpha, "render_model_async: null argument");
    ModelImpl& m = mh->impl;
    const HostCamera hc = camera_of(cam);
    validate_render(hc, opt, shard, nshards);
    ARFX_CUDA(cudaSetDevice(m.device));
    render_async_impl(m, ph->impl, hc, occ ? &occ->impl : nullptr, opt, shard, nshards, rgb, alpha, counters4,
                      stream_of(m, stream));
  });
}

// Pipelined animation through host buffers: the inference grid of the NEXT pose (p_next ->
// occ_next) is built on the model's side stream in the side workspace while the CURRENT pose
// renders with its already-built grid (p_cur, occ_cur) into host buffers as
// arfx_render_model_async does; later work on `stream` waits for the grid. Alternate the two
// (pose, grid) pairs frame by frame (the C-ABI twin of arfx_frame_graph_create_pipelined).
#ifndef ARFX_PIPE_ASYNC_GRAPH
#define ARFX_PIPE_ASYNC_GRAPH 1
#endif
int arfx_render_model_pipelined_async(arfx_model mh, arfx_pose p_cur, arfx_occ_grid occ_cur, arfx_pose p_next,
                                      arfx_occ_grid occ_next, const arfx_camera* cam, const arfx_render_options* opt,
                                      int shard, int nshards, float* rgb, float* alpha, uint64_t* counters4,
                                      void* stream) {
  return guard([&] {
    require(mh && p_cur && occ_cur && p_next && occ_next && rgb && alpha, "render_model_pipelined_async: null argument");
    require(occ_cur != occ_next, "render_model_pipelined_async: the two grids must differ");
    ModelImpl& m = mh->impl;
    const HostCamera hc = camera_of(cam);
    validate_render(hc, opt, shard, nshards);
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    if (!m.side) ARFX_CUDA(cudaStreamCreateWithFlags(&m.side, cudaStreamNonBlocking));
    if (!m.ev_pipe_fork) {
      ARFX_CUDA(cudaEventCreateWithFlags(&m.ev_pipe_fork, cudaEventDisableTiming));
      ARFX_CUDA(cudaEventCreateWithFlags(&m.ev_pipe_join, cudaEventDisableTiming));
    }
    OccImpl& gn = occ_next->impl;
    const size_t cells = static_cast<size_t>(gn.res) * gn.res * gn.res;
    {
      WorkspaceScope side(m, m.ws_side);
      if (m.ws().cap_pool < cells * kMaxRoots + 1024) {  // worst case once (no overflow re-run possible)
        ARFX_CUDA(cudaDeviceSynchronize());
        m.ws().reserve_worst(cells, static_cast<size_t>(m.sv.nb));
      }
    }
#if ARFX_PIPE_ASYNC_GRAPH
    // graph-backed: the frame (next pose's grid beside the current pose's render into the
    // async slot) is captured once per (handles, camera, options, shard, slot, stream) and
    // replayed; a capture whose workspace has since grown is re-captured (the capture's
    // warm-up renders the same frame, so a miss costs one extra frame, never a wrong one)
    if (s != nullptr) {
      int slot = 0;
      ModelImpl::AsyncSlot& a = async_slot_acquire(m, hc, s, slot);
      std::string key;
      auto add = [&key](const void* p, size_t n) { key.append(static_cast<const char*>(p), n); };
      // handles and every device pointer / by-value parameter the capture bakes in (a freed
      // and re-allocated handle, grid or image slot can never hit a stale capture)
      const OccImpl& oc = occ_cur->impl;
      const void* ptrs[13] = {p_cur, occ_cur, p_next, occ_next, s, p_cur->impl.dev.ptr, p_next->impl.dev.ptr,
                              oc.values.ptr, oc.mask.ptr, gn.values.ptr, gn.mask.ptr, a.rgb.ptr, a.counters.ptr};
      add(ptrs, sizeof(ptrs));
      const void* ptrs2[1] = {a.alpha.ptr};
      add(ptrs2, sizeof(ptrs2));
      const double occ_par[4] = {static_cast<double>(oc.res), oc.threshold, static_cast<double>(gn.res), gn.threshold};
      add(occ_par, sizeof(occ_par));
      const int occ_dil[2] = {oc.dilation, gn.dilation};
      add(occ_dil, sizeof(occ_dil));
      add(&oc.box, sizeof(oc.box));
      add(&gn.box, sizeof(gn.box));
      add(cam, sizeof(*cam));
      add(opt, sizeof(*opt));
      const int ints[3] = {shard, nshards, slot};
      add(ints, sizeof(ints));
      arfx_frame_graph_s* g = nullptr;
      for (auto it = m.pipe_graphs.begin(); it != m.pipe_graphs.end(); ++it) {
        if (it->key != key) continue;
        auto* c = static_cast<arfx_frame_graph_s*>(it->graph);
        if (c->ws->gen == c->ws_gen && c->ws2->gen == c->ws2_gen) {
          g = c;
        } else {
          delete c;
          m.pipe_graphs.erase(it);
        }
        break;
      }
      if (!g) {
        if (m.pipe_graphs.size() >= 8) {
          delete static_cast<arfx_frame_graph_s*>(m.pipe_graphs.front().graph);
          m.pipe_graphs.erase(m.pipe_graphs.begin());
        }
        g = make_pipelined_graph(m, p_cur->impl, occ_cur->impl, p_next->impl, gn, hc, opt, shard, nshards, a.rgb.ptr,
                                 a.alpha.ptr, reinterpret_cast<uint64_t*>(a.counters.ptr), s);
        m.pipe_graphs.push_back({key, g});
      }
      ARFX_CUDA(cudaGraphLaunch(g->exec, s));
      async_slot_d2h(m, a, hc, shard, nshards, rgb, alpha, a.counters.ptr + 4, counters4, s);
      return;
    }
#endif
    {
      WorkspaceScope side(m, m.ws_side);
      ARFX_CUDA(cudaEventRecord(m.ev_pipe_fork, s));
      ARFX_CUDA(cudaStreamWaitEvent(m.side, m.ev_pipe_fork, 0));
      inference_grid(m, p_next->impl, gn, nullptr, m.side);
      ARFX_CUDA(cudaEventRecord(m.ev_pipe_join, m.side));
    }
    render_async_impl(m, p_cur->impl, hc, &occ_cur->impl, opt, shard, nshards, rgb, alpha, counters4, s);
    ARFX_CUDA(cudaStreamWaitEvent(s, m.ev_pipe_join, 0));
  });
}

int arfx_render_wait(arfx_model mh) {
  return guard([&] {
    require(mh != nullptr, "render_wait: null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (m.copy_stream) ARFX_CUDA(cudaStreamSynchronize(m.copy_stream));
  });
}

int arfx_render_trace(arfx_model mh, int64_t capacity, int64_t* n_samples, int32_t* s_ray, int32_t* s_index,
                      uint8_t* s_has_root, float* s_density, float* s_color, double* s_canonical,
                      double* s_delta) {
  return guard([&] {
    require(mh && n_samples, "render_trace: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    Workspace& w = m.ws();
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
    ARFX_CUDA(cudaDeviceSynchronize());
    unsigned long long hc[4];
    ARFX_CUDA(cudaMemcpy(hc, w.counters.ptr, sizeof(hc), cudaMemcpyDeviceToHost));
    const int64_t n = static_cast<int64_t>(std::min<unsigned long long>(hc[0], w.cap_posed));
    *n_samples = n;
    if (capacity < n) return;
    std::vector<int16_t> idx(static_cast<size_t>(n));
    std::vector<uint8_t> nroot(static_cast<size_t>(n));
    std::vector<int32_t> base(static_cast<size_t>(n));
    std::vector<int8_t> sel(static_cast<size_t>(n));
    const size_t np = static_cast<size_t>(std::min<unsigned long long>(hc[2], w.cap_pool));
    std::vector<float4> pres(np);
    std::vector<double> px(np), py(np), pz(np);
    ARFX_CUDA(cudaMemcpy(s_ray, w.sray.ptr, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost));
    ARFX_CUDA(cudaMemcpy(idx.data(), w.sidx.ptr, static_cast<size_t>(n) * 2, cudaMemcpyDeviceToHost));
    ARFX_CUDA(cudaMemcpy(nroot.data(), w.snroot.ptr, static_cast<size_t>(n), cudaMemcpyDeviceToHost));
    ARFX_CUDA(cudaMemcpy(base.data(), w.sbase.ptr, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost));
    ARFX_CUDA(cudaMemcpy(sel.data(), w.ssel.ptr, static_cast<size_t>(n), cudaMemcpyDeviceToHost));
    ARFX_CUDA(cudaMemcpy(s_delta, w.sdelta.ptr, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
    ARFX_CUDA(cudaMemcpy(pres.data(), w.pres.ptr, np * sizeof(float4), cudaMemcpyDeviceToHost));
    ARFX_CUDA(cudaMemcpy(px.data(), w.px.ptr, np * 8, cudaMemcpyDeviceToHost));
    ARFX_CUDA(cudaMemcpy(py.data(), w.py.ptr, np * 8, cudaMemcpyDeviceToHost));
    ARFX_CUDA(cudaMemcpy(pz.data(), w.pz.ptr, np * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) {
      s_index[i] = idx[static_cast<size_t>(i)];
      const int k = sel[static_cast<size_t>(i)];
      const bool has = nroot[static_cast<size_t>(i)] > 0 && k >= 0;
      s_has_root[i] = has ? 1 : 0;
      const size_t p = has ? static_cast<size_t>(base[static_cast<size_t>(i)] + k) : 0;
      s_density[i] = has ? pres[p].x : 0.f;
      s_color[3 * i + 0] = has ? pres[p].y : 0.f;
      s_color[3 * i + 1] = has ? pres[p].z : 0.f;
      s_color[3 * i + 2] = has ? pres[p].w : 0.f;
      s_canonical[3 * i + 0] = has ? px[p] : 0.0;
      s_canonical[3 * i + 1] = has ? py[p] : 0.0;
      s_canonical[3 * i + 2] = has ? pz[p] : 0.0;
    }
  });
}

int arfx_profile_enable(arfx_model mh, int on) {
  return guard([&] {
    require(mh != nullptr, "profile_enable: null model");
    mh->impl.prof.on = on != 0;
  });
}

int arfx_profile_read(arfx_model mh, int max, char* names, double* ms, int64_t* launches, int* n) {
  return guard([&] {
    require(mh != nullptr && n != nullptr, "profile_read: null argument");
    KernelProfiler& p = mh->impl.prof;
    ARFX_CUDA(cudaSetDevice(mh->impl.device));
    p.collect();
    int k = 0;
    for (; k < static_cast<int>(p.names.size()) && k < max; ++k) {
      std::strncpy(names + 32 * k, p.names[static_cast<size_t>(k)].c_str(), 31);
      names[32 * k + 31] = 0;
      ms[k] = p.ms[static_cast<size_t>(k)];
      launches[k] = p.launches[static_cast<size_t>(k)];
    }
    *n = k;
    p.names.clear();
    p.ms.clear();
    p.launches.clear();
  });
}

int arfx_occ_is_occupied(arfx_occ_grid gh, const double* pts, int64_t n, uint8_t* out) {
  return guard([&] {
    OccImpl& g = occ_ref(gh);
    require(n == 0 || (pts && out), "occ_is_occupied: null argument");
    ARFX_CUDA(cudaSetDevice(g.device));
    if (n <= 0) return;
    ARFX_CUDA(cudaDeviceSynchronize());  // a grid built asynchronously on a model stream
    Staged<double> P;
    P.up(pts, static_cast<size_t>(3 * n), nullptr);
    DevBuf<uint8_t> o;
    o.alloc(static_cast<size_t>(n));
    occ_query_batch(g, P.d.ptr, n, o.ptr, nullptr);
    d2h(out, o.ptr, static_cast<size_t>(n), nullptr);
    ARFX_CUDA(cudaStreamSynchronize(nullptr));
  });
}

int arfx_stats_enable(arfx_model mh, int on) {
  return guard([&] {
    require(mh != nullptr, "stats_enable: null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (!m.stats.ptr) m.stats.alloc(16);
    ARFX_CUDA(cudaMemset(m.stats.ptr, 0, 16 * sizeof(unsigned long long)));
    m.stats_on = on != 0;
  });
}

int arfx_stats_read(arfx_model mh, uint64_t* out16) {
  return guard([&] {
    require(mh != nullptr && out16 != nullptr, "stats_read: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    ARFX_CUDA(cudaDeviceSynchronize());
    if (!m.stats.ptr) {
      std::memset(out16, 0, 16 * sizeof(uint64_t));
      return;
    }
    ARFX_CUDA(cudaMemcpy(out16, m.stats.ptr, 16 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    ARFX_CUDA(cudaMemset(m.stats.ptr, 0, 16 * sizeof(unsigned long long)));
  });
}

int arfx_pipe_peaks(double* fp64, double* fp32) {
  return guard([&] {
    require(fp64 && fp32, "pipe_peaks: null argument");
    require_device();
    measure_pipe_peaks(fp64, fp32);
  });
}

// ---- batched helpers ------------------------------------------------------


int arfx_skinning_weights(arfx_model mh, const double* pts, int64_t n, double* w) {
  return guard([&] {
    require(mh && (n == 0 || (pts && w)), "skinning_weights: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n <= 0) return;
    Staged<double> P, Wd;
    P.up(pts, static_cast<size_t>(3 * n), m.stream);
    Wd.d.alloc(static_cast<size_t>(n) * m.bones.size());
    skin_weights_batch(m, P.d.ptr, n, Wd.d.ptr, m.stream);
    d2h(w, Wd.d.ptr, static_cast<size_t>(n) * m.bones.size(), m.stream);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
  });
}

int arfx_inverse_lbs_device(arfx_model mh, arfx_pose ph, const double* d_pts, int64_t n, int32_t* d_counts,
                            double* d_roots, double* d_res, void* stream) {
  return guard([&] {
    require(mh && ph, "inverse_lbs_device: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    inverse_lbs_batch(m, ph->impl.dev.ptr, d_pts, n, d_counts, d_roots, d_res, stream_of(m, stream));
  });
}

int arfx_inverse_lbs(arfx_model mh, const double* bones12, const double* pre12, double cutoff,
                     const double* pts, int64_t n, int32_t* counts, double* roots, double* residuals) {
  return guard([&] {
    require(mh && bones12 && pre12 && (n == 0 || (pts && counts && roots && residuals)),
            "inverse_lbs: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n <= 0) return;
    PoseCtx ctx;
    make_pose_ctx(m.bones, bones12, pre12, cutoff, ctx);
    DevBuf<PoseCtx> dctx;
    dctx.alloc(1);
    h2d(dctx.ptr, &ctx, 1, m.stream);
    Staged<double> P;
    P.up(pts, static_cast<size_t>(3 * n), m.stream);
    DevBuf<int32_t> dc;
    DevBuf<double> dr, ds;
    dc.alloc(static_cast<size_t>(n));
    dr.alloc(static_cast<size_t>(n) * kMaxRoots * 3);
    ds.alloc(static_cast<size_t>(n) * kMaxRoots);
    inverse_lbs_batch(m, dctx.ptr, P.d.ptr, n, dc.ptr, dr.ptr, ds.ptr, m.stream);
    d2h(counts, dc.ptr, static_cast<size_t>(n), m.stream);
    d2h(roots, dr.ptr, static_cast<size_t>(n) * kMaxRoots * 3, m.stream);
    d2h(residuals, ds.ptr, static_cast<size_t>(n) * kMaxRoots, m.stream);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
  });
}

int arfx_hash_encode(arfx_model mh, const double* pts, int64_t n, float* feats) {
  return guard([&] {
    require(mh && (n == 0 || (pts && feats)), "hash_encode: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n <= 0) return;
    const size_t D = static_cast<size_t>(m.grid.levels) * m.grid.F;
    Staged<double> P;
    P.up(pts, static_cast<size_t>(3 * n), m.stream);
    DevBuf<float> f;
    f.alloc(static_cast<size_t>(n) * D);
    DevBuf<int> err;
    err.alloc(1);
    ARFX_CUDA(cudaMemsetAsync(err.ptr, 0, sizeof(int), m.stream));
    hash_encode_batch(m, P.d.ptr, n, f.ptr, err.ptr, m.stream);
    int herr = 0;
    d2h(&herr, err.ptr, 1, m.stream);
    d2h(feats, f.ptr, static_cast<size_t>(n) * D, m.stream);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
    if (herr) throw std::domain_error("hash grid: point outside bounding box");
  });
}

int arfx_field_query(arfx_model mh, const double* pts, int64_t n, float* dens, float* col) {
  return guard([&] {
    require(mh && (n == 0 || (pts && dens && col)), "field_query: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n <= 0) return;
    Staged<double> P;
    P.up(pts, static_cast<size_t>(3 * n), m.stream);
    DevBuf<float4> o;
    o.alloc(static_cast<size_t>(n));
    DevBuf<int> err;
    err.alloc(1);
    ARFX_CUDA(cudaMemsetAsync(err.ptr, 0, sizeof(int), m.stream));
    field_query_batch(m, P.d.ptr, n, o.ptr, err.ptr, m.stream);
    std::vector<float4> h(static_cast<size_t>(n));
    int herr = 0;
    d2h(&herr, err.ptr, 1, m.stream);
    d2h(h.data(), o.ptr, static_cast<size_t>(n), m.stream);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
    if (herr) throw std::domain_error("hash grid: point outside bounding box");
    for (int64_t i = 0; i < n; ++i) {
      dens[i] = h[static_cast<size_t>(i)].x;
      col[3 * i + 0] = h[static_cast<size_t>(i)].y;
      col[3 * i + 1] = h[static_cast<size_t>(i)].z;
      col[3 * i + 2] = h[static_cast<size_t>(i)].w;
    }
  });
}

int arfx_posed_query(arfx_model mh, arfx_pose ph, const double* pts, int64_t n, float* dens, float* col,
                     double* canon, uint8_t* has, arfx_counters* c) {
  return guard([&] {
    require(mh && ph && (n == 0 || (pts && dens && col && canon && has)), "posed_query: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n <= 0) return;
    Staged<double> P;
    P.up(pts, static_cast<size_t>(3 * n), m.stream);
    DevBuf<float> dd, dcl;
    DevBuf<double> dcan;
    DevBuf<uint8_t> dh;
    dd.alloc(static_cast<size_t>(n));
    dcl.alloc(static_cast<size_t>(3 * n));
    dcan.alloc(static_cast<size_t>(3 * n));
    dh.alloc(static_cast<size_t>(n));
    for (int attempt = 0; attempt < 3; ++attempt) {
      posed_query_batch(m, ph->impl, P.d.ptr, n, dd.ptr, dcl.ptr, dcan.ptr, dh.ptr, nullptr, m.stream);
      unsigned long long hc[8];
      d2h(hc, m.ws().counters.ptr, 8, m.stream);
      ARFX_CUDA(cudaStreamSynchronize(m.stream));
      bool rerun;
      check_overflow_and_grow(m, hc, rerun);
      if (rerun) continue;
      d2h(dens, dd.ptr, static_cast<size_t>(n), m.stream);
      d2h(col, dcl.ptr, static_cast<size_t>(3 * n), m.stream);
      d2h(canon, dcan.ptr, static_cast<size_t>(3 * n), m.stream);
      d2h(has, dh.ptr, static_cast<size_t>(n), m.stream);
      ARFX_CUDA(cudaStreamSynchronize(m.stream));
      if (c) {
        c->posed_queries = static_cast<uint64_t>(n);
        c->canonical_queries = hc[1];
      }
      return;
    }
    throw std::runtime_error("posed_query: workspace overflow persisted");
  });
}


int arfx_composite(int n_rays, const int32_t* ray_len, const double* t, const double* delta,
                   const uint8_t* skipped, const float* density, const float* color, double eps,
                   double* out_c3, double* out_a, int32_t* term) {
  return guard([&] {
    require(n_rays >= 0, "composite: negative ray count");
    if (n_rays == 0) return;
    require_device();
    (void)t;
    std::vector<int64_t> off;
    ray_offsets(n_rays, ray_len, off);
    const size_t ns = static_cast<size_t>(off.back());
    cudaStream_t s = nullptr;
    Staged<int64_t> O;
    O.up(off.data(), off.size(), s);
    Staged<double> D;
    Staged<uint8_t> K;
    Staged<float> De, Co;
    D.up(delta, ns, s);
    K.up(skipped, ns, s);
    De.up(density, ns, s);
    Co.up(color, 3 * ns, s);
    DevBuf<double> c3, a;
    DevBuf<int32_t> tm;
    c3.alloc(3 * static_cast<size_t>(n_rays));
    a.alloc(static_cast<size_t>(n_rays));
    tm.alloc(static_cast<size_t>(n_rays));
    composite_explicit(n_rays, O.d.ptr, D.d.ptr, K.d.ptr, De.d.ptr, Co.d.ptr, eps, c3.ptr, a.ptr, tm.ptr, s);
    d2h(out_c3, c3.ptr, 3 * static_cast<size_t>(n_rays), s);
    d2h(out_a, a.ptr, static_cast<size_t>(n_rays), s);
    d2h(term, tm.ptr, static_cast<size_t>(n_rays), s);
    ARFX_CUDA(cudaStreamSynchronize(s));
  });
}

int arfx_composite_backward(int n_rays, const int32_t* ray_len, const double* t, const double* delta,
                            const uint8_t* skipped, const float* density, const float* color, double eps,
                            const double* dC3, const double* dA, double* d_sigma, double* d_c3) {
  return guard([&] {
    require(n_rays >= 0, "composite_backward: negative ray count");
    if (n_rays == 0) return;
    require_device();
    (void)t;
    std::vector<int64_t> off;
    ray_offsets(n_rays, ray_len, off);
    const size_t ns = static_cast<size_t>(off.back());
    cudaStream_t s = nullptr;
    Staged<int64_t> O;
    O.up(off.data(), off.size(), s);
    Staged<double> D, DC, DA;
    Staged<uint8_t> K;
    Staged<float> De, Co;
    D.up(delta, ns, s);
    K.up(skipped, ns, s);
    De.up(density, ns, s);
    Co.up(color, 3 * ns, s);
    DC.up(dC3, 3 * static_cast<size_t>(n_rays), s);
    DA.up(dA, static_cast<size_t>(n_rays), s);
    DevBuf<double> tr, ds, dc;
    tr.alloc(ns + 1);
    ds.alloc(ns + 1);
    dc.alloc(3 * ns + 3);
    composite_backward_explicit(n_rays, O.d.ptr, D.d.ptr, K.d.ptr, De.d.ptr, Co.d.ptr, eps, DC.d.ptr, DA.d.ptr,
                                tr.ptr, ds.ptr, dc.ptr, s);
    d2h(d_sigma, ds.ptr, ns, s);
    d2h(d_c3, dc.ptr, 3 * ns, s);
    ARFX_CUDA(cudaStreamSynchronize(s));
  });
}

namespace {
void ensure_grads(ModelImpl& m, cudaStream_t s) { ensure_grad_store(m, s); }
}  // namespace

// CanonicalField::query_backward (R/field.hpp:91-103) over a batch; accumulates into the
// model's gradient buffers (zero them with arfx_model_zero_grad).
int arfx_field_query_backward(arfx_model mh, const double* pts, int64_t n, const float* d_density,
                              const float* d_color) {
  return guard([&] {
    require(mh && (n == 0 || (pts && d_density && d_color)), "field_query_backward: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n <= 0) return;
    const cudaStream_t s = m.stream;
    ensure_grads(m, s);
    Workspace& w = m.ws();
    w.ensure(static_cast<size_t>(n), 0);
    w.ensure_train();
    std::vector<double> sx(static_cast<size_t>(n)), sy(sx.size()), sz(sx.size());
    for (int64_t i = 0; i < n; ++i) {
      sx[static_cast<size_t>(i)] = pts[3 * i];
      sy[static_cast<size_t>(i)] = pts[3 * i + 1];
      sz[static_cast<size_t>(i)] = pts[3 * i + 2];
      const double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
      if (!(x >= m.grid.box.lo.x && x <= m.grid.box.hi.x && y >= m.grid.box.lo.y && y <= m.grid.box.hi.y &&
            z >= m.grid.box.lo.z && z <= m.grid.box.hi.z))
        throw std::domain_error("hash grid: point outside bounding box");
    }
    h2d(w.px.ptr, sx.data(), sx.size(), s);
    h2d(w.py.ptr, sy.data(), sy.size(), s);
    h2d(w.pz.ptr, sz.data(), sz.size(), s);
    h2d(w.pgs.ptr, d_density, static_cast<size_t>(n), s);
    h2d(w.pgc.ptr, d_color, static_cast<size_t>(3 * n), s);
    ARFX_CUDA(cudaMemsetAsync(w.pflag.ptr, 1, static_cast<size_t>(n), s));
    const unsigned long long cnt = static_cast<unsigned long long>(n);
    h2d(w.counters.ptr + 2, &cnt, 1, s);
    const BwdOwners own{static_cast<long long>(n), nullptr, nullptr, true};
    field_backward_pool(m, w.counters.ptr + 2, static_cast<long long>(n), w.pflag.ptr, w.pgs.ptr, w.pgc.ptr, s, &own);
    ARFX_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"

namespace arfx {
namespace {
__global__ void pixel_check_kernel(long long n, const int32_t* px, const int32_t* py, int W, int H,
                                   unsigned long long* bad) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    if (px[i] < 0 || py[i] < 0 || px[i] >= W || py[i] >= H) atomicAdd(bad, 1ull);
}

void validate_train(arfx_model mh, arfx_pose ph, const arfx_render_options* opt, const HostCamera& hc) {
  require(mh && ph && opt, "train: null argument");
  validate_camera(hc);
  require(opt->samples_per_ray <= 1024, "render: libarfx supports samples_per_ray <= 1024");
}

// One training forward + backward over n rays on device arrays (train.cu): ray-list march,
// deformer, field forward (re-run on workspace overflow), composite + reverse pass with
// given upstream gradients (d_dC/d_dA) or the fused losses (lt), field backward into the
// model's flat gradient vector. Returns the posed/canonical counters.
void run_train(ModelImpl& m, PoseImpl& p, const HostCamera& hc, OccImpl* occ, const arfx_render_options* opt,
               long long n_rays, const int32_t* d_px, const int32_t* d_py, const float* d_dC, const float* d_dA,
               const LossTargets* lt, float* d_rgb, float* d_alpha, cudaStream_t s, unsigned long long* hcnt,
               bool host_sync = true) {
  ensure_grad_store(m, s);
  const long long posed_max = n_rays * std::max(opt->samples_per_ray, 1);
  if (!host_sync && posed_max <= (1LL << 22)) {
    // no host round trip: capacities for the worst case (every sample occupied, every root
    // and start kept), so nothing can overflow; pixels are not range-checked here (an
    // out-of-image pixel only yields a ray through it, no out-of-bounds access)
    m.ws().reserve_worst(static_cast<size_t>(posed_max), static_cast<size_t>(m.sv.nb));
    train_forward(m, p, hc, occ, opt->samples_per_ray, opt->stratified != 0, opt->seed, opt->frame_id, n_rays, d_px,
                  d_py, s);
    Workspace& w = m.ws();
    w.ensure_train();
    ARFX_CUDA(cudaMemsetAsync(w.pflag.ptr, 0, w.cap_pool, s));
    train_composite(m, n_rays, opt->samples_per_ray, opt->epsilon_terminate, d_dC, d_dA, d_rgb, d_alpha, s, lt);
    const BwdOwners own{n_rays, w.ray_first.ptr, w.ray_count.ptr, false};
    field_backward_pool(m, w.counters.ptr + 2, static_cast<long long>(w.cap_pool), w.pflag.ptr, w.pgs.ptr,
                        w.pgc.ptr, s, &own, ARFX_SAVE_ACT ? w.fwd_act.ptr : nullptr);
    return;
  }
  DevBuf<unsigned long long> bad;
  bad.alloc(1);
  ARFX_CUDA(cudaMemsetAsync(bad.ptr, 0, sizeof(unsigned long long), s));
  pixel_check_kernel<<<static_cast<unsigned>(std::min<long long>((n_rays + 255) / 256, 1024)), 256, 0, s>>>(
      n_rays, d_px, d_py, hc.width, hc.height, bad.ptr);
  ARFX_CUDA(cudaGetLastError());
  for (int attempt = 0;; ++attempt) {
    train_forward(m, p, hc, occ, opt->samples_per_ray, opt->stratified != 0, opt->seed, opt->frame_id, n_rays, d_px,
                  d_py, s);
    unsigned long long nbad = 0;
    d2h(hcnt, m.ws().counters.ptr, 8, s);
    d2h(&nbad, bad.ptr, 1, s);
    ARFX_CUDA(cudaStreamSynchronize(s));
    if (nbad) throw std::invalid_argument("generate_ray: pixel outside image");
    bool rerun;
    check_overflow_and_grow(m, hcnt, rerun);
    if (!rerun) break;
    if (attempt == 2) throw std::runtime_error("train: workspace overflow persisted");
  }
  Workspace& w = m.ws();
  w.ensure_train();
  ARFX_CUDA(cudaMemsetAsync(w.pflag.ptr, 0, w.cap_pool, s));
  train_composite(m, n_rays, opt->samples_per_ray, opt->epsilon_terminate, d_dC, d_dA, d_rgb, d_alpha, s, lt);
  const BwdOwners own{n_rays, w.ray_first.ptr, w.ray_count.ptr, false};
  field_backward_pool(m, w.counters.ptr + 2, static_cast<long long>(w.cap_pool), w.pflag.ptr, w.pgs.ptr, w.pgc.ptr,
                      s, &own, ARFX_SAVE_ACT ? w.fwd_act.ptr : nullptr);
}

LossTargets loss_targets(const arfx_loss_config* cfg, const float* gt_rgb, const float* gt_alpha, double* terms) {
  require(cfg != nullptr, "loss: null config");
  require(cfg->w_rgb >= 0 && cfg->w_alpha >= 0 && cfg->w_hard >= 0 && cfg->w_density >= 0,
          "loss: weights must be non-negative");
  require(cfg->huber_delta > 0, "loss: huber_delta must be positive");
  require(cfg->gt_width >= 0 && cfg->gt_height >= 0, "loss: negative ground-truth frame size");
  LossTargets lt{gt_rgb, gt_alpha, cfg->w_rgb, cfg->w_alpha, cfg->w_hard, cfg->w_density, cfg->huber_delta, terms};
  lt.gt_w = cfg->gt_width;
  lt.gt_h = cfg->gt_height;
  return lt;
}

AdamCfg adam_of(const arfx_adam_config* c) {
  require(c != nullptr, "adam: null config");
  require(c->lr_grid >= 0 && c->lr_mlp >= 0, "adam: learning rates must be non-negative");
  require(c->beta1 >= 0 && c->beta1 < 1 && c->beta2 >= 0 && c->beta2 < 1, "adam: betas must be in [0, 1)");
  require(c->eps > 0, "adam: eps must be positive");
  return AdamCfg{c->lr_grid, c->lr_mlp, c->beta1, c->beta2, c->eps, static_cast<long long>(c->total_steps),
                 c->final_lr_factor};
}
}  // namespace
}  // namespace arfx

extern "C" {

// Training forward + backward over n rays (composed per SPEC.md:490-494; see train.cu).
int arfx_train_fwd_bwd(arfx_model mh, arfx_pose ph, const arfx_camera* cam, arfx_occ_grid occ,
                       const arfx_render_options* opt, int64_t n_rays, const int32_t* px, const int32_t* py,
                       const float* d_color, const float* d_alpha, float* rgb, float* alpha, arfx_counters* c,
                       void* stream) {
  return guard([&] {
    const HostCamera hc = camera_of(cam);
    validate_train(mh, ph, opt, hc);
    require(n_rays == 0 || (px && py && d_color && d_alpha), "train_fwd_bwd: null argument");
    for (int64_t r = 0; r < n_rays; ++r)
      if (px[r] < 0 || py[r] < 0 || px[r] >= hc.width || py[r] >= hc.height)
        throw std::invalid_argument("generate_ray: pixel outside image");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n_rays <= 0) return;
    const cudaStream_t s = stream_of(m, stream);
    Staged<int32_t> PX, PY;
    Staged<float> DC, DA;
    PX.up(px, static_cast<size_t>(n_rays), s);
    PY.up(py, static_cast<size_t>(n_rays), s);
    DC.up(d_color, static_cast<size_t>(3 * n_rays), s);
    DA.up(d_alpha, static_cast<size_t>(n_rays), s);
    DevBuf<float> orgb, oalpha;
    orgb.alloc(static_cast<size_t>(3 * n_rays));
    oalpha.alloc(static_cast<size_t>(n_rays));
    unsigned long long hcnt[8];
    run_train(m, ph->impl, hc, occ ? &occ->impl : nullptr, opt, n_rays, PX.d.ptr, PY.d.ptr, DC.d.ptr, DA.d.ptr,
              nullptr, orgb.ptr, oalpha.ptr, s, hcnt);
    if (rgb) d2h(rgb, orgb.ptr, static_cast<size_t>(3 * n_rays), s);
    if (alpha) d2h(alpha, oalpha.ptr, static_cast<size_t>(n_rays), s);
    ARFX_CUDA(cudaStreamSynchronize(s));
    if (c) {
      c->posed_queries = hcnt[0];
      c->canonical_queries = hcnt[1];
    }
  });
}

int arfx_losses(int64_t n, const float* rgb, const float* alpha, const float* gt_rgb, const float* gt_alpha,
                const arfx_loss_config* cfg, double* loss4, float* d_rgb, float* d_alpha) {
  return guard([&] {
    require(n == 0 || (rgb && alpha && gt_rgb && gt_alpha), "losses: null argument");
    LossTargets lt = loss_targets(cfg, nullptr, nullptr, nullptr);
    require(lt.gt_w == 0, "loss: frame targets (gt_width > 0) are for the device train steps only");
    require_device();
    const cudaStream_t s = cudaStreamPerThread;
    DevBuf<double> T, L4;
    L4.alloc(4);
    if (n <= 0) {
      if (loss4) std::fill(loss4, loss4 + 4, 0.0);
      return;
    }
    Staged<float> R, A, GR, GA;
    R.up(rgb, static_cast<size_t>(3 * n), s);
    A.up(alpha, static_cast<size_t>(n), s);
    GR.up(gt_rgb, static_cast<size_t>(3 * n), s);
    GA.up(gt_alpha, static_cast<size_t>(n), s);
    T.alloc(static_cast<size_t>(3 * n));
    DevBuf<float> dR, dA;
    dR.alloc(static_cast<size_t>(3 * n));
    dA.alloc(static_cast<size_t>(n));
    lt.gt_rgb = GR.d.ptr;
    lt.gt_alpha = GA.d.ptr;
    lt.ray_terms = T.ptr;
    ray_losses(n, R.d.ptr, A.d.ptr, lt, dR.ptr, dA.ptr, s);
    loss_reduce(T.ptr, n, lt, L4.ptr, s);
    if (loss4) d2h(loss4, L4.ptr, 4, s);
    if (d_rgb) d2h(d_rgb, dR.ptr, static_cast<size_t>(3 * n), s);
    if (d_alpha) d2h(d_alpha, dA.ptr, static_cast<size_t>(n), s);
    ARFX_CUDA(cudaStreamSynchronize(s));
  });
}

int arfx_train_step(arfx_model mh, arfx_pose ph, const arfx_camera* cam, arfx_occ_grid occ,
                    const arfx_render_options* opt, int64_t n_rays, const int32_t* px, const int32_t* py,
                    const float* gt_rgb, const float* gt_alpha, const arfx_loss_config* cfg, double* loss4,
                    float* rgb, float* alpha, arfx_counters* c, void* stream) {
  return guard([&] {
    const HostCamera hc = camera_of(cam);
    validate_train(mh, ph, opt, hc);
    require(n_rays == 0 || (px && py && gt_rgb && gt_alpha), "train_step: null argument");
    LossTargets lt = loss_targets(cfg, nullptr, nullptr, nullptr);
    require(lt.gt_w == 0, "loss: frame targets (gt_width > 0) are for the device train steps only");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n_rays <= 0) return;
    const cudaStream_t s = stream_of(m, stream);
    Staged<int32_t> PX, PY;
    Staged<float> GR, GA;
    PX.up(px, static_cast<size_t>(n_rays), s);
    PY.up(py, static_cast<size_t>(n_rays), s);
    GR.up(gt_rgb, static_cast<size_t>(3 * n_rays), s);
    GA.up(gt_alpha, static_cast<size_t>(n_rays), s);
    DevBuf<float> orgb, oalpha;
    DevBuf<double> T, L4;
    orgb.alloc(static_cast<size_t>(3 * n_rays));
    oalpha.alloc(static_cast<size_t>(n_rays));
    T.alloc(static_cast<size_t>(3 * n_rays));
    L4.alloc(4);
    lt.gt_rgb = GR.d.ptr;
    lt.gt_alpha = GA.d.ptr;
    lt.ray_terms = T.ptr;
    unsigned long long hcnt[8];
    run_train(m, ph->impl, hc, occ ? &occ->impl : nullptr, opt, n_rays, PX.d.ptr, PY.d.ptr, nullptr, nullptr, &lt,
              orgb.ptr, oalpha.ptr, s, hcnt);
    loss_reduce(T.ptr, n_rays, lt, L4.ptr, s);
    if (loss4) d2h(loss4, L4.ptr, 4, s);
    if (rgb) d2h(rgb, orgb.ptr, static_cast<size_t>(3 * n_rays), s);
    if (alpha) d2h(alpha, oalpha.ptr, static_cast<size_t>(n_rays), s);
    ARFX_CUDA(cudaStreamSynchronize(s));
    if (c) {
      c->posed_queries = hcnt[0];
      c->canonical_queries = hcnt[1];
    }
  });
}

int arfx_train_step_device(arfx_model mh, arfx_pose ph, const arfx_camera* cam, arfx_occ_grid occ,
                           const arfx_render_options* opt, int64_t n_rays, const int32_t* d_px,
                           const int32_t* d_py, const float* d_gt_rgb, const float* d_gt_alpha,
                           const arfx_loss_config* cfg, double* d_loss4, float* d_rgb, float* d_alpha,
                           void* stream) {
  return guard([&] {
    const HostCamera hc = camera_of(cam);
    validate_train(mh, ph, opt, hc);
    require(n_rays == 0 || (d_px && d_py && d_gt_rgb && d_gt_alpha && d_loss4), "train_step: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n_rays <= 0) return;
    const cudaStream_t s = stream_of(m, stream);
    Workspace& w = m.ws();
    w.train_terms.ensure(static_cast<size_t>(3 * n_rays));
    w.train_rgb.ensure(static_cast<size_t>(3 * n_rays));
    w.train_alpha.ensure(static_cast<size_t>(n_rays));
    LossTargets lt = loss_targets(cfg, d_gt_rgb, d_gt_alpha, w.train_terms.ptr);
    lt.px = d_px;
    lt.py = d_py;
    unsigned long long hcnt[8];
    run_train(m, ph->impl, hc, occ ? &occ->impl : nullptr, opt, n_rays, d_px, d_py, nullptr, nullptr, &lt,
              d_rgb ? d_rgb : w.train_rgb.ptr, d_alpha ? d_alpha : w.train_alpha.ptr, s, hcnt, /*host_sync=*/false);
    loss_reduce(w.train_terms.ptr, n_rays, lt, d_loss4, s);
  });
}

namespace {
void run_density(ModelImpl& m, PoseImpl& p, OccImpl& g, long long n, uint64_t seed, uint64_t step, double w,
                 double* d_out2, cudaStream_t s, bool host_sync = true) {
  ensure_grad_store(m, s);
  if (!host_sync && n <= (1LL << 22)) {  // worst-case capacities: no overflow check needed
    m.ws().reserve_worst(static_cast<size_t>(n), static_cast<size_t>(m.sv.nb));
    density_forward(m, p, g, n, seed, step, s);
    density_backward(m, n, w, d_out2, s);
    return;
  }
  for (int attempt = 0;; ++attempt) {
    density_forward(m, p, g, n, seed, step, s);
    unsigned long long hc[8];
    d2h(hc, m.ws().counters.ptr, 8, s);
    ARFX_CUDA(cudaStreamSynchronize(s));
    bool rerun;
    check_overflow_and_grow(m, hc, rerun);
    if (!rerun) break;
    if (attempt == 2) throw std::runtime_error("density_step: workspace overflow persisted");
  }
  density_backward(m, n, w, d_out2, s);
}
}  // namespace

int arfx_density_step(arfx_model mh, arfx_pose ph, arfx_occ_grid occ, int64_t n_points, uint64_t seed,
                      uint64_t step, const arfx_loss_config* cfg, double* loss2, void* stream) {
  return guard([&] {
    require(mh && ph && occ, "density_step: null argument");
    const LossTargets lt = loss_targets(cfg, nullptr, nullptr, nullptr);
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n_points <= 0) {
      if (loss2) loss2[0] = loss2[1] = 0.0;
      return;
    }
    const cudaStream_t s = stream_of(m, stream);
    DevBuf<double> out;
    out.alloc(2);
    run_density(m, ph->impl, occ->impl, n_points, seed, step, lt.w_density, out.ptr, s);
    double h[2];
    d2h(h, out.ptr, 2, s);
    ARFX_CUDA(cudaStreamSynchronize(s));
    if (loss2) loss2[0] = h[0], loss2[1] = h[1];
  });
}

int arfx_density_step_device(arfx_model mh, arfx_pose ph, arfx_occ_grid occ, int64_t n_points, uint64_t seed,
                             uint64_t step, const arfx_loss_config* cfg, double* d_loss2, void* stream) {
  return guard([&] {
    require(mh && ph && occ && d_loss2, "density_step: null argument");
    const LossTargets lt = loss_targets(cfg, nullptr, nullptr, nullptr);
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (n_points <= 0) return;
    run_density(m, ph->impl, occ->impl, n_points, seed, step, lt.w_density, d_loss2, stream_of(m, stream),
                /*host_sync=*/false);
  });
}

// Train step + L_density step in one call: the density forward (points, deformer, field
// on the side workspace) runs on the model's side stream concurrently with the train
// step's forward and backward, and its backward joins after the train backward on
// `stream` (gradient accumulation stays ordered). Same results as arfx_train_step_device
// followed by arfx_density_step_device.
int arfx_train_density_step_device(arfx_model mh, arfx_pose ph, const arfx_camera* cam, arfx_occ_grid occ,
                                   const arfx_render_options* opt, int64_t n_rays, const int32_t* d_px,
                                   const int32_t* d_py, const float* d_gt_rgb, const float* d_gt_alpha,
                                   const arfx_loss_config* cfg, double* d_loss4, int64_t n_points, uint64_t dseed,
                                   uint64_t dstep, double* d_loss2, void* stream) {
  return guard([&] {
    const HostCamera hc = camera_of(cam);
    validate_train(mh, ph, opt, hc);
    require(n_rays == 0 || (d_px && d_py && d_gt_rgb && d_gt_alpha && d_loss4), "train_step: null argument");
    require(n_points <= 0 || (occ && d_loss2), "density_step: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    const LossTargets dl = loss_targets(cfg, nullptr, nullptr, nullptr);
    ensure_grad_store(m, s);
    const bool dens = n_points > 0;
    if (dens) {
      require(n_points <= (1LL << 22), "density_step: at most 2^22 points per call");
      if (!m.side) {
        ARFX_CUDA(cudaStreamCreateWithFlags(&m.side, cudaStreamNonBlocking));
        ARFX_CUDA(cudaEventCreateWithFlags(&m.ev_fork, cudaEventDisableTiming));
        ARFX_CUDA(cudaEventCreateWithFlags(&m.ev_join, cudaEventDisableTiming));
      }
      WorkspaceScope side(m, m.ws_side);
      m.ws().reserve_worst(static_cast<size_t>(n_points), static_cast<size_t>(m.sv.nb));
      ARFX_CUDA(cudaEventRecord(m.ev_fork, s));
      ARFX_CUDA(cudaStreamWaitEvent(m.side, m.ev_fork, 0));
      density_forward(m, ph->impl, occ->impl, n_points, dseed, dstep, m.side);
      density_flags(m, n_points, dl.w_density, d_loss2, m.side);
      ARFX_CUDA(cudaEventRecord(m.ev_join, m.side));
    }
    if (n_rays > 0) {
      Workspace& w = m.ws();
      w.train_terms.ensure(static_cast<size_t>(3 * n_rays));
      w.train_rgb.ensure(static_cast<size_t>(3 * n_rays));
      w.train_alpha.ensure(static_cast<size_t>(n_rays));
      LossTargets lt = loss_targets(cfg, d_gt_rgb, d_gt_alpha, w.train_terms.ptr);
      lt.px = d_px;
      lt.py = d_py;
      unsigned long long hcnt[8];
      run_train(m, ph->impl, hc, occ ? &occ->impl : nullptr, opt, n_rays, d_px, d_py, nullptr, nullptr, &lt,
                w.train_rgb.ptr, w.train_alpha.ptr, s, hcnt, /*host_sync=*/false);
      loss_reduce(w.train_terms.ptr, n_rays, lt, d_loss4, s);
    }
    if (dens) {
      ARFX_CUDA(cudaStreamWaitEvent(s, m.ev_join, 0));
      WorkspaceScope side(m, m.ws_side);
      density_backward_field(m, n_points, s);
    }
  });
}

// Split train step for software pipelining across steps (the trainer runs the forward of
// step t+1 -- march, deformer, field -- while step t's backward runs): slot 0 / 1 selects
// one of two train workspaces. The forward needs no gradients; its field kernels wait on
// the parameter fence (arfx_model_set_param_fence). The backward = composite + fused losses
// + field backward of that slot (+ the L_density step as in arfx_train_density_step_device).
namespace {
Workspace& train_slot(ModelImpl& m, int slot) { return slot ? m.ws_alt : m.ws_t0; }
}  // namespace

int arfx_train_rays_device(uint64_t seed, uint64_t step, uint64_t rank, int64_t n, int width, int height,
                           int32_t* d_px, int32_t* d_py, void* stream) {
  return guard([&] {
    require(n <= 0 || (d_px && d_py), "train_rays: null argument");
    require(width > 0 && height > 0, "train_rays: empty image");
    launch_train_rays(seed, step, rank, n, width, height, d_px, d_py, static_cast<cudaStream_t>(stream));
  });
}

int arfx_train_forward_device(arfx_model mh, arfx_pose ph, const arfx_camera* cam, arfx_occ_grid occ,
                              const arfx_render_options* opt, int64_t n_rays, const int32_t* d_px,
                              const int32_t* d_py, int slot, void* stream) {
  return guard([&] {
    const HostCamera hc = camera_of(cam);
    validate_train(mh, ph, opt, hc);
    require(slot == 0 || slot == 1, "train_forward: slot must be 0 or 1");
    require(n_rays == 0 || (d_px && d_py), "train_forward: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    const long long posed_max = n_rays * std::max(opt->samples_per_ray, 1);
    require(posed_max <= (1LL << 22), "train_forward: at most 2^22 ray samples per step");
    if (n_rays <= 0) return;
    WorkspaceScope scope(m, train_slot(m, slot));
    m.ws().reserve_worst(static_cast<size_t>(posed_max), static_cast<size_t>(m.sv.nb));
    train_forward(m, ph->impl, hc, occ ? &occ->impl : nullptr, opt->samples_per_ray, opt->stratified != 0, opt->seed,
                  opt->frame_id, n_rays, d_px, d_py, stream_of(m, stream));
  });
}

int arfx_train_backward_device(arfx_model mh, arfx_pose ph, arfx_occ_grid occ, const arfx_render_options* opt,
                               int64_t n_rays, const int32_t* d_px, const int32_t* d_py, const float* d_gt_rgb,
                               const float* d_gt_alpha, const arfx_loss_config* cfg, double* d_loss4, int slot,
                               int64_t n_points, uint64_t dseed, uint64_t dstep, double* d_loss2, void* stream) {
  return guard([&] {
    require(mh && ph && opt, "train_backward: null argument");
    require(slot == 0 || slot == 1, "train_backward: slot must be 0 or 1");
    require(n_rays == 0 || (d_px && d_py && d_gt_rgb && d_gt_alpha && d_loss4), "train_backward: null argument");
    require(n_points <= 0 || (occ && d_loss2), "density_step: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    const cudaStream_t s = stream_of(m, stream);
    const LossTargets dl = loss_targets(cfg, nullptr, nullptr, nullptr);
    ensure_grad_store(m, s);
    const bool dens = n_points > 0;
    if (dens) {
      require(n_points <= (1LL << 22), "density_step: at most 2^22 points per call");
      if (!m.side) {
        ARFX_CUDA(cudaStreamCreateWithFlags(&m.side, cudaStreamNonBlocking));
        ARFX_CUDA(cudaEventCreateWithFlags(&m.ev_fork, cudaEventDisableTiming));
        ARFX_CUDA(cudaEventCreateWithFlags(&m.ev_join, cudaEventDisableTiming));
      }
      WorkspaceScope side(m, m.ws_side);
      m.ws().reserve_worst(static_cast<size_t>(n_points), static_cast<size_t>(m.sv.nb));
      ARFX_CUDA(cudaEventRecord(m.ev_fork, s));
      ARFX_CUDA(cudaStreamWaitEvent(m.side, m.ev_fork, 0));
      density_forward(m, ph->impl, occ->impl, n_points, dseed, dstep, m.side);
      density_flags(m, n_points, dl.w_density, d_loss2, m.side);
      ARFX_CUDA(cudaEventRecord(m.ev_join, m.side));
    }
    if (n_rays > 0) {
      WorkspaceScope scope(m, train_slot(m, slot));
      Workspace& w = m.ws();
      w.ensure_train();
      w.train_terms.ensure(static_cast<size_t>(3 * n_rays));
      w.train_rgb.ensure(static_cast<size_t>(3 * n_rays));
      w.train_alpha.ensure(static_cast<size_t>(n_rays));
      LossTargets lt = loss_targets(cfg, d_gt_rgb, d_gt_alpha, w.train_terms.ptr);
      lt.px = d_px;
      lt.py = d_py;
      ARFX_CUDA(cudaMemsetAsync(w.pflag.ptr, 0, w.cap_pool, s));
      train_composite(m, n_rays, opt->samples_per_ray, opt->epsilon_terminate, nullptr, nullptr, w.train_rgb.ptr,
                      w.train_alpha.ptr, s, &lt);
      const BwdOwners own{n_rays, w.ray_first.ptr, w.ray_count.ptr, false};
      field_backward_pool(m, w.counters.ptr + 2, static_cast<long long>(w.cap_pool), w.pflag.ptr, w.pgs.ptr,
                          w.pgc.ptr, s, &own, ARFX_SAVE_ACT ? w.fwd_act.ptr : nullptr);
      loss_reduce(w.train_terms.ptr, n_rays, lt, d_loss4, s);
    }
    if (dens) {
      ARFX_CUDA(cudaStreamWaitEvent(s, m.ev_join, 0));
      WorkspaceScope side(m, m.ws_side);
      density_backward_field(m, n_points, s);
    }
  });
}

int arfx_adam_step(arfx_model mh, const arfx_adam_config* cfg, int64_t step, int64_t begin, int64_t end,
                   void* stream) {
  return guard([&] {
    require(mh != nullptr, "adam: null model");
    const AdamCfg c = adam_of(cfg);
    require(step >= 1, "adam: step must be >= 1");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (end < 0) end = static_cast<int64_t>(m.n_flat);
    require(begin >= 0 && begin <= end && end <= static_cast<int64_t>(m.n_flat) && begin % 4 == 0 && end % 4 == 0,
            "adam: range must be a multiple-of-4 slice of the flat vector");
    const cudaStream_t s = stream_of(m, stream);
    ensure_grad_store(m, s);
    adam_step(m, c, step, begin, end, s);
  });
}

int arfx_adam_step_guarded(arfx_model mh, const arfx_adam_config* cfg, int64_t step, int64_t begin, int64_t end,
                           const double* d_loss, int n_loss, int* d_bad, void* stream) {
  return guard([&] {
    require(mh != nullptr, "adam: null model");
    require(d_loss && d_bad && n_loss > 0 && n_loss <= 64, "adam_guarded: loss row (1..64 doubles) and flag required");
    const AdamCfg c = adam_of(cfg);
    require(step >= 1, "adam: step must be >= 1");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (end < 0) end = static_cast<int64_t>(m.n_flat);
    require(begin >= 0 && begin <= end && end <= static_cast<int64_t>(m.n_flat) && begin % 4 == 0 && end % 4 == 0,
            "adam: range must be a multiple-of-4 slice of the flat vector");
    const cudaStream_t s = stream_of(m, stream);
    ensure_grad_store(m, s);
    adam_step(m, c, step, begin, end, s, d_loss, n_loss, d_bad);
  });
}

int arfx_model_flat(arfx_model mh, float** params, float** grads, float** am, float** av, int64_t* n_flat,
                    int64_t* mlp_offset) {
  return guard([&] {
    require(mh != nullptr, "null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    ensure_grad_store(m, m.stream);
    if ((am || av) && !m.adam_m.ptr) {
      m.adam_m.alloc(m.n_flat);
      m.adam_v.alloc(m.n_flat);
      ARFX_CUDA(cudaMemsetAsync(m.adam_m.ptr, 0, m.n_flat * sizeof(float), m.stream));
      ARFX_CUDA(cudaMemsetAsync(m.adam_v.ptr, 0, m.n_flat * sizeof(float), m.stream));
      ARFX_CUDA(cudaStreamSynchronize(m.stream));
    }
    if (params) *params = m.flat_params.ptr;
    if (grads) *grads = m.flat_grads.ptr;
    if (am) *am = m.adam_m.ptr;
    if (av) *av = m.adam_v.ptr;
    if (n_flat) *n_flat = static_cast<int64_t>(m.n_flat);
    if (mlp_offset) *mlp_offset = static_cast<int64_t>(m.mlp_off);
  });
}

int arfx_model_get_adam(arfx_model mh, float* am, float* av) {
  return guard([&] {
    require(mh != nullptr, "null model");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (!m.adam_m.ptr) {
      if (am) std::fill(am, am + m.n_flat, 0.0f);
      if (av) std::fill(av, av + m.n_flat, 0.0f);
      return;
    }
    if (am) d2h(am, m.adam_m.ptr, m.n_flat, m.stream);
    if (av) d2h(av, m.adam_v.ptr, m.n_flat, m.stream);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
  });
}

int arfx_model_set_adam(arfx_model mh, const float* am, const float* av) {
  return guard([&] {
    require(mh && am && av, "set_adam: null argument");
    ModelImpl& m = mh->impl;
    ARFX_CUDA(cudaSetDevice(m.device));
    if (!m.adam_m.ptr) {
      m.adam_m.alloc(m.n_flat);
      m.adam_v.alloc(m.n_flat);
    }
    h2d(m.adam_m.ptr, am, m.n_flat, m.stream);
    h2d(m.adam_v.ptr, av, m.n_flat, m.stream);
    ARFX_CUDA(cudaStreamSynchronize(m.stream));
  });
}

int arfx_figure_query(const arfx_figure* fig, const double* bones12, const double* pts, int64_t n,
                      double* density, double* color) {
  return guard([&] {
    const FigureView F = figure_view_of(fig, bones12);
    require(n == 0 || (pts && density && color), "figure_query: null argument");
    require_device();
    if (n <= 0) return;
    const cudaStream_t s = cudaStreamPerThread;
    Staged<double> P;
    P.up(pts, static_cast<size_t>(3 * n), s);
    DevBuf<double> D, Cc;
    D.alloc(static_cast<size_t>(n));
    Cc.alloc(static_cast<size_t>(3 * n));
    figure_query_batch(F, P.d.ptr, n, D.ptr, Cc.ptr, s);
    d2h(density, D.ptr, static_cast<size_t>(n), s);
    d2h(color, Cc.ptr, static_cast<size_t>(3 * n), s);
    ARFX_CUDA(cudaStreamSynchronize(s));
  });
}

int arfx_figure_render(const arfx_figure* fig, const double* bones12, const double* global12,
                       const double box_lo[3], const double box_hi[3], const arfx_camera* cam,
                       const arfx_render_options* opt, float* rgb, float* alpha, uint8_t* mask, void* stream) {
  return guard([&] {
    const FigureFrame f = figure_frame(fig, bones12, global12, box_lo, box_hi, cam, opt);
    require_device();
    const cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
    const long long n = static_cast<long long>(f.cam.width) * f.cam.height;
    DevBuf<float> R, A;
    DevBuf<uint8_t> M;
    R.alloc(static_cast<size_t>(3 * n));
    A.alloc(static_cast<size_t>(n));
    M.alloc(static_cast<size_t>(n));
    figure_render(f.F, f.cam, f.w2n, box_lo, box_hi, opt->samples_per_ray, opt->stratified != 0,
                  opt->epsilon_terminate, opt->seed, opt->frame_id, n, nullptr, nullptr, R.ptr, A.ptr, M.ptr, s);
    if (rgb) d2h(rgb, R.ptr, static_cast<size_t>(3 * n), s);
    if (alpha) d2h(alpha, A.ptr, static_cast<size_t>(n), s);
    if (mask) d2h(mask, M.ptr, static_cast<size_t>(n), s);
    ARFX_CUDA(cudaStreamSynchronize(s));
  });
}

int arfx_figure_render_rays_device(const arfx_figure* fig, const double* bones12, const double* global12,
                                   const double box_lo[3], const double box_hi[3], const arfx_camera* cam,
                                   const arfx_render_options* opt, int64_t n, const int32_t* d_px,
                                   const int32_t* d_py, float* d_rgb, float* d_alpha, uint8_t* d_mask,
                                   void* stream) {
  return guard([&] {
    const FigureFrame f = figure_frame(fig, bones12, global12, box_lo, box_hi, cam, opt);
    require(n == 0 || (d_px && d_py && d_rgb && d_alpha), "figure_render_rays: null argument");
    require_device();
    const cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
    figure_render(f.F, f.cam, f.w2n, box_lo, box_hi, opt->samples_per_ray, opt->stratified != 0,
                  opt->epsilon_terminate, opt->seed, opt->frame_id, n, d_px, d_py, d_rgb, d_alpha, d_mask, s);
  });
}

}  // extern "C"
