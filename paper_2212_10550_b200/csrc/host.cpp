// host.cpp -- host-side setup of libarfx (skeleton, pose, camera, configs).
// Every expression keeps the reference's operand order; compiled with
// -ffp-contract=off (x86-64 SSE2 doubles), so results are bit-identical to the
// reference's host code. Citations are into /root/reference/proj/include/arf (R/).
#include "host.h"

#include <cmath>
#include <limits>

namespace arfx {
namespace {

HV operator+(const HV& a, const HV& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
HV operator-(const HV& a, const HV& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
HV operator-(const HV& a) { return {-a.x, -a.y, -a.z}; }
HV operator*(const HV& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
double dot(const HV& a, const HV& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
double norm(const HV& a) { return std::sqrt(dot(a, a)); }
HV normalized(const HV& a) {
  const double n = norm(a);
  return {a.x / n, a.y / n, a.z / n};
}
HV cross(const HV& a, const HV& o) {
  return {a.y * o.z - a.z * o.y, a.z * o.x - a.x * o.z, a.x * o.y - a.y * o.x};
}
bool finite(const HV& a) { return std::isfinite(a.x) && std::isfinite(a.y) && std::isfinite(a.z); }
HV cmin(const HV& a, const HV& b) {
  return {b.x < a.x ? b.x : a.x, b.y < a.y ? b.y : a.y, b.z < a.z ? b.z : a.z};
}
HV cmax(const HV& a, const HV& b) {
  return {a.x < b.x ? b.x : a.x, a.y < b.y ? b.y : a.y, a.z < b.z ? b.z : a.z};
}
double dmax(double a, double b) { return a < b ? b : a; }

// Mat3 row-major helpers (R/math.hpp:93-158)
HV matvec(const double* m, const HV& v) {
  return {m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
          m[6] * v.x + m[7] * v.y + m[8] * v.z};
}
void matmul(const double* a, const double* b, double* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += a[i * 3 + k] * b[k * 3 + j];
      r[i * 3 + j] = s;
    }
}
void transpose(const double* a, double* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i * 3 + j] = a[j * 3 + i];
}
double det(const double* m) {
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
         m[2] * (m[3] * m[7] - m[4] * m[6]);
}

void expand(HostBox& b, const HV& p) {
  b.lo = cmin(b.lo, p);
  b.hi = cmax(b.hi, p);
}
HostBox empty_box() {
  const double mx = std::numeric_limits<double>::max();
  const double lw = std::numeric_limits<double>::lowest();
  return {{mx, mx, mx}, {lw, lw, lw}};
}

}  // namespace

void validate_skeleton(const std::vector<HostBone>& bones) {
  if (bones.empty()) throw std::invalid_argument("skeleton: needs at least one bone");
  if (static_cast<int>(bones.size()) > kMaxBones)
    throw std::invalid_argument("pose context: too many bones");
  if (bones[0].parent != -1) throw std::invalid_argument("skeleton: bone 0 must be the root");
  for (size_t i = 0; i < bones.size(); ++i) {
    const HostBone& b = bones[i];
    if (i > 0 && (b.parent < 0 || static_cast<size_t>(b.parent) >= i))
      throw std::invalid_argument("skeleton: parents must form a tree rooted at bone 0");
    if (!(b.radius > 0)) throw std::invalid_argument("skeleton: radii must be positive");
    if (!finite(b.head) || !finite(b.tail)) throw std::invalid_argument("skeleton: non-finite joint");
  }
}

// R/skeleton.hpp:53-63 (extra_pad = 0), Aabb::inflated_relative R/math.hpp:235-241
HostBox rest_bounds(const std::vector<HostBone>& bones, double margin) {
  HostBox box = empty_box();
  for (const HostBone& b : bones) {
    const HV r{b.radius, b.radius, b.radius};
    expand(box, b.head - r);
    expand(box, b.head + r);
    expand(box, b.tail - r);
    expand(box, b.tail + r);
  }
  const HV z{0.0, 0.0, 0.0};
  box.lo = box.lo - z;
  box.hi = box.hi + z;
  const HV m = (box.hi - box.lo) * margin;
  box.lo = box.lo - m;
  box.hi = box.hi + m;
  return box;
}

// R/skeleton.hpp:39-50
double max_reach(const std::vector<HostBone>& bones) {
  std::vector<double> head_reach(bones.size(), 0.0);
  double reach = 0.0;
  for (size_t i = 0; i < bones.size(); ++i) {
    const HostBone& b = bones[i];
    head_reach[i] = (b.parent < 0) ? 0.0
                                   : head_reach[static_cast<size_t>(b.parent)] +
                                         norm(b.head - bones[static_cast<size_t>(b.parent)].head);
    reach = dmax(reach, head_reach[i] + norm(b.tail - b.head) + b.radius);
  }
  return reach;
}

// R/model.hpp:59-66
HostBox normalized_reach_box(const std::vector<HostBone>& bones, double margin) {
  const double reach = max_reach(bones) * margin;
  const HV root = bones[0].head;
  HostBox box = empty_box();
  const HV r{reach, reach, reach};
  expand(box, root - r);
  expand(box, root + r);
  return box;
}

void validate_grid_cfg(const GridCfg& g) {
  if (g.levels < 1) throw std::invalid_argument("hash grid: levels must be >= 1");
  if (g.levels > kMaxLevels) throw std::invalid_argument("hash grid: too many levels for libarfx");
  if (g.F < 1) throw std::invalid_argument("hash grid: features_per_level must be >= 1");
  if (g.log2T < 1 || g.log2T > 30) throw std::invalid_argument("hash grid: table_size_log2 out of range");
  if (g.nmin < 2) throw std::invalid_argument("hash grid: base_resolution must be >= 2");
  if (g.nmax < g.nmin)
    throw std::invalid_argument("hash grid: max_resolution must be >= base_resolution");
  if (!(g.box.lo.x <= g.box.hi.x && g.box.lo.y <= g.box.hi.y && g.box.lo.z <= g.box.hi.z))
    throw std::invalid_argument("hash grid: invalid bounding box");
}

// R/hash_grid.hpp:35-53
std::vector<int> level_resolutions(const GridCfg& g) {
  validate_grid_cfg(g);
  std::vector<int> res(static_cast<size_t>(g.levels));
  if (g.levels == 1) {
    res[0] = g.nmin;
    return res;
  }
  const double growth = std::exp((std::log(double(g.nmax)) - std::log(double(g.nmin))) /
                                 double(g.levels - 1));
  for (int l = 0; l < g.levels; ++l) {
    const double v = g.nmin * std::pow(growth, double(l));
    int r = static_cast<int>(std::floor(v + 1e-6));
    if (g.nmax < r) r = g.nmax;
    if (l > 0 && r < res[static_cast<size_t>(l - 1)]) r = res[static_cast<size_t>(l - 1)];
    res[static_cast<size_t>(l)] = r;
  }
  res.back() = g.nmax;
  return res;
}

// R/mlp.hpp:37-48
MlpLayout mlp_layout(int input_dim, int hidden_dim, int hidden_layers, int output_dim) {
  if (input_dim < 1 || hidden_dim < 1 || output_dim < 1)
    throw std::invalid_argument("mlp: dimensions must be >= 1");
  if (hidden_layers < 1 || hidden_layers > 8)
    throw std::invalid_argument("mlp: hidden_layers out of range");
  MlpLayout L{};
  L.n_layers = hidden_layers + 1;
  int in = input_dim, off = 0;
  for (int l = 0; l < L.n_layers; ++l) {
    const int out = (l == hidden_layers) ? output_dim : hidden_dim;
    L.lin[l] = in;
    L.lout[l] = out;
    L.w_off[l] = off;
    L.b_off[l] = off + in * out;
    off += in * out + out;
    in = out;
  }
  L.n_params = off;
  return L;
}

void rigid_compose(const double* a, const double* b, double* out) {
  double r[9];
  matmul(a, b, r);
  const HV t = matvec(a, {b[9], b[10], b[11]}) + HV{a[9], a[10], a[11]};
  for (int i = 0; i < 9; ++i) out[i] = r[i];
  out[9] = t.x;
  out[10] = t.y;
  out[11] = t.z;
}

void rigid_inverse(const double* a, double* out) {
  double rt[9];
  transpose(a, rt);
  const HV t = -matvec(rt, {a[9], a[10], a[11]});
  for (int i = 0; i < 9; ++i) out[i] = rt[i];
  out[9] = t.x;
  out[10] = t.y;
  out[11] = t.z;
}

HV rigid_apply(const double* a, const HV& v) { return matvec(a, v) + HV{a[9], a[10], a[11]}; }

bool rigid_is_rotation(const double* a, double tol) {
  double rt[9], g[9];
  transpose(a, rt);
  matmul(a, rt, g);
  double e = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) e = dmax(e, std::abs(g[i * 3 + j] - (i == j ? 1.0 : 0.0)));
  return e <= tol && det(a) > 0 && std::isfinite(a[9]) && std::isfinite(a[10]) &&
         std::isfinite(a[11]);
}

void validate_pose(int n_bones, const double* bones12, const double* global12) {
  if (n_bones < 1) throw std::invalid_argument("pose: no bone transforms");
  for (int i = 0; i < n_bones; ++i)
    if (!rigid_is_rotation(bones12 + 12 * i, 1e-6))
      throw std::invalid_argument("pose: bone transform is not rigid");
  if (!rigid_is_rotation(global12, 1e-6))
    throw std::invalid_argument("pose: global transform is not rigid");
}

// R/skeleton.hpp:93-110 with Rigid::about_point R/math.hpp:210-212
void pose_from_joint_rotations(const std::vector<HostBone>& bones, const double* rot9,
                               const double* global12, double* out12) {
  validate_skeleton(bones);
  std::vector<double> chain(bones.size() * 12);
  for (size_t i = 0; i < bones.size(); ++i) {
    const HostBone& b = bones[i];
    double local[12];
    for (int k = 0; k < 9; ++k) local[k] = rot9[9 * i + static_cast<size_t>(k)];
    const HV t = b.head - matvec(local, b.head);
    local[9] = t.x;
    local[10] = t.y;
    local[11] = t.z;
    double* ci = chain.data() + 12 * i;
    if (b.parent < 0) {
      for (int k = 0; k < 12; ++k) ci[k] = local[k];
    } else {
      rigid_compose(chain.data() + 12 * static_cast<size_t>(b.parent), local, ci);
    }
    rigid_compose(global12, ci, out12 + 12 * i);
  }
}

// R/articulation.hpp:24-41
void make_pose_ctx(const std::vector<HostBone>& bones, const double* bones12, const double* pre12,
                   double cutoff_factor, PoseCtx& ctx) {
  const int nb = static_cast<int>(bones.size());
  if (nb > kMaxBones) throw std::invalid_argument("pose context: too many bones");
  ctx = PoseCtx{};
  ctx.nb = nb;
  for (int i = 0; i < nb; ++i) {
    rigid_compose(pre12, bones12 + 12 * i, ctx.bone[i]);
    rigid_inverse(ctx.bone[i], ctx.bone_inv[i]);
    const HV a = rigid_apply(ctx.bone[i], bones[static_cast<size_t>(i)].head);
    const HV b = rigid_apply(ctx.bone[i], bones[static_cast<size_t>(i)].tail);
    ctx.cap_a[i][0] = a.x;
    ctx.cap_a[i][1] = a.y;
    ctx.cap_a[i][2] = a.z;
    ctx.cap_b[i][0] = b.x;
    ctx.cap_b[i][1] = b.y;
    ctx.cap_b[i][2] = b.z;
    ctx.cutoff[i] = cutoff_factor * bones[static_cast<size_t>(i)].radius;
    const HV c = (a + b) * 0.5;
    const double R = 0.5 * norm(b - a) + ctx.cutoff[i] + 1e-4;
    const double R2 = R * R;
    ctx.sph[i][0] = static_cast<float>(c.x);
    ctx.sph[i][1] = static_cast<float>(c.y);
    ctx.sph[i][2] = static_cast<float>(c.z);
    ctx.sph[i][3] = R2 < 3.0e38 ? static_cast<float>(R2) : 3.0e38f;
  }
  for (int k = 0; k < 12; ++k) ctx.w2n[k] = pre12[k];
}

// R/camera.hpp:31-48
HostCamera look_at(const HV& eye, const HV& target, const HV& up, double focal, int w, int h) {
  HostCamera cam{};
  cam.width = w;
  cam.height = h;
  cam.fx = cam.fy = focal;
  cam.cx = w * 0.5;
  cam.cy = h * 0.5;
  const HV fwd = normalized(target - eye);
  HV down = -up + fwd * dot(up, fwd);
  down = normalized(down);
  const HV right = cross(down, fwd);
  const double r[9] = {right.x, right.y, right.z, down.x, down.y, down.z, fwd.x, fwd.y, fwd.z};
  for (int i = 0; i < 9; ++i) cam.ext[i] = r[i];
  const HV t = -matvec(r, eye);
  cam.ext[9] = t.x;
  cam.ext[10] = t.y;
  cam.ext[11] = t.z;
  return cam;
}

// R/camera.hpp:15-22
void validate_camera(const HostCamera& c) {
  if (!(c.fx > 0) || !(c.fy > 0)) throw std::invalid_argument("camera: focal must be positive");
  if (c.width < 1 || c.height < 1) throw std::invalid_argument("camera: empty image");
  if (c.cx < 0 || c.cx > c.width || c.cy < 0 || c.cy > c.height)
    throw std::invalid_argument("camera: principal point outside image");
  if (!rigid_is_rotation(c.ext, 1e-6)) throw std::invalid_argument("camera: extrinsic not rigid");
}

// R/occupancy.hpp:49-52, :65
double occupancy_threshold(const HostBox& box, int res, double alpha_threshold) {
  const HV e = box.hi - box.lo;
  const HV cs{e.x / res, e.y / res, e.z / res};
  return -std::log1p(-alpha_threshold) / norm(cs);
}

// R/occupancy.hpp:20-27
void validate_occ_cfg(int resolution, double alpha_threshold, int dilation, double decay,
                      int interval) {
  if (resolution < 2) throw std::invalid_argument("occupancy: resolution must be >= 2");
  if (!(alpha_threshold > 0 && alpha_threshold < 1))
    throw std::invalid_argument("occupancy: alpha_threshold must be in (0,1)");
  if (dilation < 0) throw std::invalid_argument("occupancy: dilation must be >= 0");
  if (!(decay >= 0 && decay <= 1)) throw std::invalid_argument("occupancy: decay in [0,1]");
  if (interval < 1) throw std::invalid_argument("occupancy: update_interval must be >= 1");
}

}  // namespace arfx
