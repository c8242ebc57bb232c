/*
 * arf_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference's per-ray render/train path
 * (/root/reference/proj/include/arf, cited R/file:line), exposed through the
 * arfo_* entry points of oracle_api.h. Single-threaded, IEEE double / float with
 * -ffp-contract=off, operand order copied from the reference so results are
 * bit-identical to it (pinned by tests/test_oracle_cpu.py against oracle/_ref and
 * the committed golden vectors in tests/golden/).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_api.h"

static char g_err[512];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* arfo_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- math  R/math.hpp */

typedef struct {
  double x, y, z;
} v3;

static v3 V(double x, double y, double z) {
  v3 r = {x, y, z};
  return r;
}
static v3 vadd(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 vsub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 vmul(v3 a, double s) { return V(a.x * s, a.y * s, a.z * s); }
static v3 vneg(v3 a) { return V(-a.x, -a.y, -a.z); }
static double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; } /* :59 */
static double vnorm(v3 a) { return sqrt(vdot(a, a)); }                           /* :62-63 */
static v3 vnormalized(v3 a) {                                                     /* :64 */
  const double n = vnorm(a);
  return V(a.x / n, a.y / n, a.z / n);
}
static v3 vcross(v3 a, v3 o) { return V(a.y * o.z - a.z * o.y, a.z * o.x - a.x * o.z, a.x * o.y - a.y * o.x); }
static v3 vload(const double* p) { return V(p[0], p[1], p[2]); }
static void vstore(double* p, v3 a) {
  p[0] = a.x;
  p[1] = a.y;
  p[2] = a.z;
}
static double vget(v3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
static double dmin_(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double dmax_(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* Mat3 row-major  R/math.hpp:93-158 */
static v3 mv(const double* m, v3 v) {
  return V(m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
           m[6] * v.x + m[7] * v.y + m[8] * v.z);
}
static void mm(const double* a, const double* b, double* r) { /* :111-120 */
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += a[i * 3 + k] * b[k * 3 + j];
      r[i * 3 + j] = s;
    }
}
static void mt(const double* a, double* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i * 3 + j] = a[j * 3 + i];
}
static double mdet(const double* m) { /* :137-140 */
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
         m[2] * (m[3] * m[7] - m[4] * m[6]);
}
static int minverse(const double* m, double* r) { /* :141-158; returns 0 if singular */
  const double d = mdet(m);
  if (fabs(d) < DBL_MIN * 64) return 0;
  const double id = 1.0 / d;
  r[0] = (m[4] * m[8] - m[5] * m[7]) * id;
  r[1] = (m[2] * m[7] - m[1] * m[8]) * id;
  r[2] = (m[1] * m[5] - m[2] * m[4]) * id;
  r[3] = (m[5] * m[6] - m[3] * m[8]) * id;
  r[4] = (m[0] * m[8] - m[2] * m[6]) * id;
  r[5] = (m[2] * m[3] - m[0] * m[5]) * id;
  r[6] = (m[3] * m[7] - m[4] * m[6]) * id;
  r[7] = (m[1] * m[6] - m[0] * m[7]) * id;
  r[8] = (m[0] * m[4] - m[1] * m[3]) * id;
  return 1;
}

/* Rigid = R(9) t(3)  R/math.hpp:186-213 */
static v3 rapply(const double* T, v3 x) { return vadd(mv(T, x), V(T[9], T[10], T[11])); }
static void rinverse(const double* a, double* o) {
  double rt[9];
  mt(a, rt);
  const v3 t = vneg(mv(rt, V(a[9], a[10], a[11])));
  memcpy(o, rt, sizeof rt);
  vstore(o + 9, t);
}
static void rcompose(const double* a, const double* b, double* o) { /* a after b, :202-204 */
  double r[9];
  mm(a, b, r);
  const v3 t = vadd(mv(a, V(b[9], b[10], b[11])), V(a[9], a[10], a[11]));
  memcpy(o, r, sizeof r);
  vstore(o + 9, t);
}

static double point_segment_distance(v3 p, v3 a, v3 b) { /* R/math.hpp:254-261 */
  const v3 ab = vsub(b, a);
  const double len2 = vdot(ab, ab);
  if (len2 <= DBL_MIN) return vnorm(vsub(p, a));
  double t = vdot(vsub(p, a), ab) / len2;
  t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t); /* std::clamp */
  return vnorm(vsub(p, vadd(a, vmul(ab, t))));
}

static float softplusf(float z) { return z > 0 ? z + log1pf(expf(-z)) : log1pf(expf(z)); } /* :264-267 */
static float logisticf(float z) {                                                          /* :268-271 */
  return z >= 0 ? 1.0f / (1.0f + expf(-z)) : expf(z) / (1.0f + expf(z));
}

/* ---------------------------------------------------------------- rng  R/rng.hpp */

static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
static uint64_t mix_key4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  uint64_t h = splitmix64(a);
  h = splitmix64(h ^ b);
  h = splitmix64(h ^ c);
  h = splitmix64(h ^ d);
  return h;
}
typedef struct {
  uint64_t state, inc;
} pcg;
static uint32_t pcg_u32(pcg* r) {
  const uint64_t old = r->state;
  r->state = old * 6364136223846793005ULL + r->inc;
  const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
  const uint32_t rot = (uint32_t)(old >> 59u);
  return (xs >> rot) | (xs << ((32u - rot) & 31u));
}
static pcg pcg_make(uint64_t seed, uint64_t seq) {
  pcg r;
  r.state = 0;
  r.inc = (seq << 1u) | 1u;
  pcg_u32(&r);
  r.state += seed;
  pcg_u32(&r);
  return r;
}
static pcg keyed_rng(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return pcg_make(mix_key4(seed, a, b, 0), mix_key4(c, a ^ 0x5851f42d4c957f2dULL, seed, 0));
}
static double pcg_double(pcg* r) { return pcg_u32(r) * 0x1p-32; }
static uint32_t pcg_below(pcg* r, uint32_t n) { return (uint32_t)(((uint64_t)pcg_u32(r) * n) >> 32); }
static double pcg_uniform(pcg* r, double lo, double hi) { return lo + (hi - lo) * pcg_double(r); }

/* ---------------------------------------------------------------- skeleton */

static int validate_skeleton(const ao_skeleton* s) { /* R/skeleton.hpp:22-31 */
  if (s->n_bones < 1) return fail(1, "skeleton: needs at least one bone");
  if (s->n_bones > AO_MAX_BONES) return fail(1, "pose context: too many bones");
  if (s->parent[0] != -1) return fail(1, "skeleton: bone 0 must be the root");
  for (int i = 0; i < s->n_bones; ++i) {
    if (i > 0 && (s->parent[i] < 0 || s->parent[i] >= i))
      return fail(1, "skeleton: parents must form a tree rooted at bone 0");
    if (!(s->radius[i] > 0)) return fail(1, "skeleton: radii must be positive");
    for (int a = 0; a < 3; ++a)
      if (!isfinite(s->head[i][a]) || !isfinite(s->tail[i][a])) return fail(1, "skeleton: non-finite joint");
  }
  return 0;
}

typedef struct {
  v3 lo, hi;
} box3;

static box3 box_empty(void) {
  box3 b;
  b.lo = V(DBL_MAX, DBL_MAX, DBL_MAX);
  b.hi = V(-DBL_MAX, -DBL_MAX, -DBL_MAX);
  return b;
}
static void box_expand(box3* b, v3 p) { /* R/math.hpp:229-232 */
  b->lo = V(dmin_(b->lo.x, p.x), dmin_(b->lo.y, p.y), dmin_(b->lo.z, p.z));
  b->hi = V(dmax_(b->hi.x, p.x), dmax_(b->hi.y, p.y), dmax_(b->hi.z, p.z));
}
static int box_contains(const double* lo, const double* hi, v3 p) { /* :226-228 */
  return p.x >= lo[0] && p.x <= hi[0] && p.y >= lo[1] && p.y <= hi[1] && p.z >= lo[2] && p.z <= hi[2];
}

static box3 rest_bounds(const ao_skeleton* s, double margin) { /* R/skeleton.hpp:53-63 */
  box3 b = box_empty();
  for (int i = 0; i < s->n_bones; ++i) {
    const v3 r = V(s->radius[i], s->radius[i], s->radius[i]);
    const v3 h = vload(s->head[i]), t = vload(s->tail[i]);
    box_expand(&b, vsub(h, r));
    box_expand(&b, vadd(h, r));
    box_expand(&b, vsub(t, r));
    box_expand(&b, vadd(t, r));
  }
  b.lo = vsub(b.lo, V(0, 0, 0)); /* pad(0) */
  b.hi = vadd(b.hi, V(0, 0, 0));
  const v3 m = vmul(vsub(b.hi, b.lo), margin); /* inflated_relative  R/math.hpp:235-241 */
  b.lo = vsub(b.lo, m);
  b.hi = vadd(b.hi, m);
  return b;
}

static double max_reach(const ao_skeleton* s) { /* R/skeleton.hpp:39-50 */
  double head_reach[AO_MAX_BONES];
  double reach = 0.0;
  for (int i = 0; i < s->n_bones; ++i) {
    const int p = s->parent[i];
    head_reach[i] = p < 0 ? 0.0 : head_reach[p] + vnorm(vsub(vload(s->head[i]), vload(s->head[p])));
    reach = dmax_(reach, head_reach[i] + vnorm(vsub(vload(s->tail[i]), vload(s->head[i]))) + s->radius[i]);
  }
  return reach;
}

/* ---------------------------------------------------------------- hash grid  R/hash_grid.hpp */

static int grid_validate(const ao_grid_cfg* g) { /* :20-29 */
  if (g->levels < 1) return fail(1, "hash grid: levels must be >= 1");
  if (g->features_per_level < 1) return fail(1, "hash grid: features_per_level must be >= 1");
  if (g->table_size_log2 < 1 || g->table_size_log2 > 30) return fail(1, "hash grid: table_size_log2 out of range");
  if (g->base_resolution < 2) return fail(1, "hash grid: base_resolution must be >= 2");
  if (g->max_resolution < g->base_resolution)
    return fail(1, "hash grid: max_resolution must be >= base_resolution");
  if (!(g->box_lo[0] <= g->box_hi[0] && g->box_lo[1] <= g->box_hi[1] && g->box_lo[2] <= g->box_hi[2]))
    return fail(1, "hash grid: invalid bounding box");
  return 0;
}

int arfo_level_resolutions(const ao_grid_cfg* g, int* res) { /* :35-53 */
  const int e = grid_validate(g);
  if (e) return e;
  if (g->levels == 1) {
    res[0] = g->base_resolution;
    return 0;
  }
  const double growth =
      exp((log((double)g->max_resolution) - log((double)g->base_resolution)) / (double)(g->levels - 1));
  for (int l = 0; l < g->levels; ++l) {
    const double v = g->base_resolution * pow(growth, (double)l);
    int r = (int)floor(v + 1e-6);
    if (g->max_resolution < r) r = g->max_resolution;
    if (l > 0 && r < res[l - 1]) r = res[l - 1];
    res[l] = r;
  }
  res[g->levels - 1] = g->max_resolution;
  return 0;
}

static uint32_t hidx(const int* res, uint32_t rows, int level, int cx, int cy, int cz) { /* :87-101 */
  const uint64_t n = (uint64_t)res[level];
  const uint64_t corners = n + 1;
  if (corners * corners * corners <= rows)
    return (uint32_t)((uint64_t)cx + corners * ((uint64_t)cy + corners * (uint64_t)cz));
  if (n * n * n <= rows) {
    const uint64_t wx = (uint64_t)cx % n, wy = (uint64_t)cy % n, wz = (uint64_t)cz % n;
    return (uint32_t)(wx + n * (wy + n * wz));
  }
  const uint32_t h = (uint32_t)cx ^ ((uint32_t)cy * 2654435761u) ^ ((uint32_t)cz * 805459861u);
  return h & (rows - 1);
}

uint32_t arfo_hash_index(const ao_grid_cfg* g, int level, int cx, int cy, int cz) {
  int res[64];
  if (g->levels > 64 || arfo_level_resolutions(g, res)) return 0xffffffffu;
  return hidx(res, 1u << g->table_size_log2, level, cx, cy, cz);
}

typedef struct { /* a prepared field: resolutions + layout, pointers into ao_model */
  const ao_model* m;
  int res[64];
  uint32_t rows;
  int L, F, D;
  int nl, lin[9], lout[9], woff[9], boff[9], act_total, width;
} field_t;

static int field_prepare(const ao_model* m, field_t* f) {
  f->m = m;
  f->L = m->grid.levels;
  f->F = m->grid.features_per_level;
  f->D = f->L * f->F;
  if (f->L > 64) return fail(1, "oracle: too many levels");
  int e = arfo_level_resolutions(&m->grid, f->res);
  if (e) return e;
  f->rows = 1u << m->grid.table_size_log2;
  /* DecoderMlp layout R/mlp.hpp:37-48 */
  const ao_mlp_cfg* c = &m->mlp;
  if (c->hidden_layers < 1 || c->hidden_layers > 8) return fail(1, "mlp: hidden_layers out of range");
  f->nl = c->hidden_layers + 1;
  int in = f->D, off = 0;
  f->act_total = f->D;
  f->width = f->D;
  for (int l = 0; l < f->nl; ++l) {
    const int out = (l == c->hidden_layers) ? c->output_dim : c->hidden_dim;
    f->lin[l] = in;
    f->lout[l] = out;
    f->woff[l] = off;
    f->boff[l] = off + in * out;
    off += in * out + out;
    f->act_total += out;
    if (out > f->width) f->width = out;
    in = out;
  }
  return 0;
}

typedef struct {
  uint32_t index[8];
  double weight[8];
} corners_t;

static void gather(const field_t* f, int level, v3 x, corners_t* cs) { /* :114-134 */
  const ao_model* m = f->m;
  const double u[3] = {(x.x - m->grid.box_lo[0]) / (m->grid.box_hi[0] - m->grid.box_lo[0]),
                       (x.y - m->grid.box_lo[1]) / (m->grid.box_hi[1] - m->grid.box_lo[1]),
                       (x.z - m->grid.box_lo[2]) / (m->grid.box_hi[2] - m->grid.box_lo[2])};
  const double n = (double)f->res[level];
  int cell[3];
  double fr[3];
  for (int a = 0; a < 3; ++a) {
    const double p = u[a] * n;
    double c = floor(p);
    if (c > n - 1) c = n - 1;
    if (c < 0) c = 0;
    cell[a] = (int)c;
    fr[a] = p - c;
  }
  for (int k = 0; k < 8; ++k) {
    const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
    cs->index[k] = hidx(f->res, f->rows, level, cell[0] + dx, cell[1] + dy, cell[2] + dz);
    cs->weight[k] = (dx ? fr[0] : 1.0 - fr[0]) * (dy ? fr[1] : 1.0 - fr[1]) * (dz ? fr[2] : 1.0 - fr[2]);
  }
}

static int grid_contains(const ao_model* m, v3 x) { return box_contains(m->grid.box_lo, m->grid.box_hi, x); }

static void encode(const field_t* f, v3 x, float* out) { /* :137-150 */
  const int F = f->F;
  for (int l = 0; l < f->L; ++l) {
    corners_t cs;
    gather(f, l, x, &cs);
    const float* table = f->m->grid_params + (size_t)l * f->rows * F;
    float* o = out + l * F;
    for (int q = 0; q < F; ++q) o[q] = 0.0f;
    for (int k = 0; k < 8; ++k) {
      const float w = (float)cs.weight[k];
      const float* row = table + (size_t)cs.index[k] * F;
      for (int q = 0; q < F; ++q) o[q] += w * row[q];
    }
  }
}

static void encode_backward(const field_t* f, v3 x, const float* up, float* grad) { /* :155-169 */
  const int F = f->F;
  for (int l = 0; l < f->L; ++l) {
    corners_t cs;
    gather(f, l, x, &cs);
    float* gt = grad + (size_t)l * f->rows * F;
    const float* u = up + l * F;
    for (int k = 0; k < 8; ++k) {
      const float w = (float)cs.weight[k];
      if (w == 0.0f) continue;
      float* row = gt + (size_t)cs.index[k] * F;
      for (int q = 0; q < F; ++q) row[q] += w * u[q];
    }
  }
}

/* DecoderMlp::forward R/mlp.hpp:90-111; act = [input | layer outputs] */
static void mlp_forward(const field_t* f, const float* input, float* act) {
  const float* P = f->m->mlp_params;
  for (int i = 0; i < f->D; ++i) act[i] = input[i];
  const float* cur = act;
  int pos = f->D;
  for (int l = 0; l < f->nl; ++l) {
    const int in = f->lin[l], on = f->lout[l];
    const float* w = P + f->woff[l];
    const float* b = P + f->boff[l];
    float* next = act + pos;
    const int hidden = l + 1 < f->nl;
    for (int o = 0; o < on; ++o) {
      float acc = b[o];
      const float* wrow = w + (size_t)o * in;
      for (int i = 0; i < in; ++i) acc += wrow[i] * cur[i];
      next[o] = (hidden && acc < 0.0f) ? 0.0f : acc;
    }
    cur = next;
    pos += on;
  }
}

static const float* mlp_logits(const field_t* f, const float* act) {
  return act + f->act_total - f->lout[f->nl - 1];
}

/* DecoderMlp::backward R/mlp.hpp:116-154 */
static void mlp_backward(const field_t* f, const float* upstream, const float* act, float* grad, float* d_input,
                         float* dcur, float* dprev) {
  const float* P = f->m->mlp_params;
  int off[10];
  off[0] = 0;
  for (int l = 0; l < f->nl; ++l) off[l + 1] = off[l] + (l == 0 ? f->D : f->lout[l - 1]);
  for (int i = 0; i < f->m->mlp.output_dim; ++i) dcur[i] = upstream[i];
  for (int l = f->nl - 1; l >= 0; --l) {
    const int in = f->lin[l], on = f->lout[l];
    const float* ia = act + off[l];
    if (l + 1 < f->nl) {
      const float* post = act + off[l + 1];
      for (int o = 0; o < on; ++o)
        if (post[o] == 0.0f) dcur[o] = 0.0f;
    }
    float* gw = grad + f->woff[l];
    float* gb = grad + f->boff[l];
    for (int i = 0; i < in; ++i) dprev[i] = 0.0f;
    const float* w = P + f->woff[l];
    for (int o = 0; o < on; ++o) {
      const float u = dcur[o];
      gb[o] += u;
      float* gwrow = gw + (size_t)o * in;
      const float* wrow = w + (size_t)o * in;
      if (u != 0.0f) {
        for (int i = 0; i < in; ++i) {
          gwrow[i] += u * ia[i];
          dprev[i] += u * wrow[i];
        }
      }
    }
    float* t = dcur;
    dcur = dprev;
    dprev = t;
  }
  for (int i = 0; i < f->D; ++i) d_input[i] = dcur[i];
}

typedef struct {
  float* feat;
  float* act;
  float* dlog;
  float* dfeat;
  float* b1;
  float* b2;
} scratch_t;

static int scratch_alloc(const field_t* f, scratch_t* s) {
  s->feat = (float*)malloc(sizeof(float) * (size_t)f->D);
  s->act = (float*)malloc(sizeof(float) * (size_t)f->act_total);
  s->dlog = (float*)malloc(sizeof(float) * (size_t)(f->m->mlp.output_dim + 4));
  s->dfeat = (float*)malloc(sizeof(float) * (size_t)f->D);
  s->b1 = (float*)malloc(sizeof(float) * (size_t)f->width);
  s->b2 = (float*)malloc(sizeof(float) * (size_t)f->width);
  return (s->feat && s->act && s->dlog && s->dfeat && s->b1 && s->b2) ? 0 : fail(5, "oracle: out of memory");
}
static void scratch_free(scratch_t* s) {
  free(s->feat);
  free(s->act);
  free(s->dlog);
  free(s->dfeat);
  free(s->b1);
  free(s->b2);
}

/* CanonicalField::query R/field.hpp:75-82 */
static void field_query(const field_t* f, v3 x, scratch_t* s, float* dens, float* col) {
  encode(f, x, s->feat);
  mlp_forward(f, s->feat, s->act);
  const float* lg = mlp_logits(f, s->act);
  *dens = softplusf(lg[0]);
  col[0] = logisticf(lg[1]);
  col[1] = logisticf(lg[2]);
  col[2] = logisticf(lg[3]);
}

/* CanonicalField::query_backward R/field.hpp:91-103 */
static void field_query_backward(const field_t* f, v3 x, float dd, const float* dc, scratch_t* s, float* gg,
                                 float* mg) {
  encode(f, x, s->feat);
  mlp_forward(f, s->feat, s->act);
  const float* lg = mlp_logits(f, s->act);
  s->dlog[0] = dd * logisticf(lg[0]);
  for (int c = 0; c < 3; ++c) {
    const float v = logisticf(lg[1 + c]);
    s->dlog[1 + c] = dc[c] * v * (1.0f - v);
  }
  for (int c = 4; c < f->m->mlp.output_dim; ++c) s->dlog[c] = 0.0f;
  mlp_backward(f, s->dlog, s->act, mg, s->dfeat, s->b1, s->b2);
  encode_backward(f, x, s->dfeat, gg);
}

/* ---------------------------------------------------------------- skinning  R/skinning.hpp */

static void skin_interp(const ao_model* m, v3 x, double* w) { /* :25-55 */
  const double lo[3] = {m->skin_lo[0], m->skin_lo[1], m->skin_lo[2]};
  const double hi[3] = {m->skin_hi[0], m->skin_hi[1], m->skin_hi[2]};
  const int nb = m->skel.n_bones;
  int c[3];
  double fr[3];
  for (int a = 0; a < 3; ++a) {
    const double e = hi[a] - lo[a];
    double p = vget(x, a);
    p = dmax_(lo[a], dmin_(hi[a], p)); /* clamp_inside */
    const double u = (p - lo[a]) / e * (m->skin_res[a] - 1);
    const int rmax = m->skin_res[a] - 1;
    double fl = floor(u);
    if (fl > rmax - 1) fl = rmax - 1;
    if (fl < 0) fl = 0;
    c[a] = (int)fl;
    fr[a] = u - fl;
  }
  for (int i = 0; i < nb; ++i) w[i] = 0.0;
  for (int k = 0; k < 8; ++k) {
    const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
    const double wt = (dx ? fr[0] : 1 - fr[0]) * (dy ? fr[1] : 1 - fr[1]) * (dz ? fr[2] : 1 - fr[2]);
    if (wt == 0.0) continue;
    const double* nw =
        m->skin_weights +
        (((size_t)(c[2] + dz) * m->skin_res[1] + (size_t)(c[1] + dy)) * m->skin_res[0] + (size_t)(c[0] + dx)) * nb;
    for (int i = 0; i < nb; ++i) w[i] += wt * nw[i];
  }
  double sum = 0.0;
  for (int i = 0; i < nb; ++i) sum += w[i];
  if (sum > 0) {
    const double inv = 1.0 / sum;
    for (int i = 0; i < nb; ++i) w[i] *= inv;
  }
}

static int build_skinning(const ao_skeleton* s, const double* lo, const double* hi, const int* res,
                          double blend, double* W) { /* :61-111 */
  int e = validate_skeleton(s);
  if (e) return e;
  if (res[0] < 2 || res[1] < 2 || res[2] < 2) return fail(1, "skinning grid: resolution must be >= 2 per axis");
  for (int i = 0; i < s->n_bones; ++i)
    if (vnorm(vsub(vload(s->tail[i]), vload(s->head[i]))) <= 0)
      return fail(1, "skinning grid: degenerate zero-length bone");
  const int nb = s->n_bones;
  const v3 ex = V(hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]);
  double dist[AO_MAX_BONES];
  for (int iz = 0; iz < res[2]; ++iz)
    for (int iy = 0; iy < res[1]; ++iy)
      for (int ix = 0; ix < res[0]; ++ix) {
        const v3 p = V(lo[0] + ex.x * ix / (res[0] - 1), lo[1] + ex.y * iy / (res[1] - 1),
                       lo[2] + ex.z * iz / (res[2] - 1));
        double dmn = DBL_MAX;
        for (int b = 0; b < nb; ++b) {
          dist[b] = point_segment_distance(p, vload(s->head[b]), vload(s->tail[b]));
          dmn = dmin_(dmn, dist[b]);
        }
        double* w = W + (((size_t)iz * res[1] + iy) * res[0] + ix) * nb;
        if (dmn < 1e-12) {
          int hits = 0;
          for (int b = 0; b < nb; ++b)
            if (dist[b] < 1e-12) ++hits;
          for (int b = 0; b < nb; ++b) w[b] = dist[b] < 1e-12 ? 1.0 / hits : 0.0;
          continue;
        }
        const double band = blend * dmn;
        double sum = 0.0;
        for (int b = 0; b < nb; ++b) {
          const double v = dist[b] <= band ? 1.0 / dist[b] : 0.0;
          w[b] = v;
          sum += v;
        }
        for (int b = 0; b < nb; ++b) w[b] /= sum;
      }
  return 0;
}

/* ---------------------------------------------------------------- articulation  R/articulation.hpp */

typedef struct { /* PoseContext :17-42 */
  int nb;
  double bone[AO_MAX_BONES][12], inv[AO_MAX_BONES][12];
  v3 cap_a[AO_MAX_BONES], cap_b[AO_MAX_BONES];
  double cutoff[AO_MAX_BONES];
} ctx_t;

static void ctx_make(const ao_skeleton* s, const double* bones12, const double* pre12, double cutoff_factor,
                     ctx_t* c) {
  c->nb = s->n_bones;
  for (int i = 0; i < s->n_bones; ++i) {
    rcompose(pre12, bones12 + 12 * i, c->bone[i]);
    rinverse(c->bone[i], c->inv[i]);
    c->cap_a[i] = rapply(c->bone[i], vload(s->head[i]));
    c->cap_b[i] = rapply(c->bone[i], vload(s->tail[i]));
    c->cutoff[i] = cutoff_factor * s->radius[i];
  }
}

static v3 lbs(const ctx_t* c, v3 x, const double* w) { /* :45-50 */
  v3 out = V(0, 0, 0);
  for (int i = 0; i < c->nb; ++i)
    if (w[i] != 0.0) out = vadd(out, vmul(rapply(c->bone[i], x), w[i]));
  return out;
}

typedef struct {
  int count;
  v3 x[AO_MAX_ROOTS];
  double r[AO_MAX_ROOTS];
} roots_t;

static void roots_push(roots_t* R, v3 p, double r, double dedup) { /* :66-81 */
  for (int i = 0; i < R->count; ++i) {
    if (vnorm(vsub(R->x[i], p)) < dedup) {
      if (r < R->r[i]) {
        R->x[i] = p;
        R->r[i] = r;
      }
      return;
    }
  }
  if (R->count < AO_MAX_ROOTS) {
    R->x[R->count] = p;
    R->r[R->count] = r;
    ++R->count;
  }
}

static roots_t inverse_lbs(const ao_model* m, const ctx_t* c, v3 xt) { /* :94-145 */
  roots_t R;
  R.count = 0;
  double w[AO_MAX_BONES];
  for (int b = 0; b < c->nb; ++b) {
    if (point_segment_distance(xt, c->cap_a[b], c->cap_b[b]) > c->cutoff[b]) continue;
    v3 x = rapply(c->inv[b], xt);
    skin_interp(m, x, w);
    v3 g = vsub(lbs(c, x, w), xt);
    double gn = vnorm(g);
    int converged = gn < m->tolerance;
    for (int it = 0; it < m->max_iterations && !converged; ++it) {
      double jac[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int i = 0; i < c->nb; ++i)
        if (w[i] != 0.0)
          for (int e = 0; e < 9; ++e) jac[e] = jac[e] + c->bone[i][e] * w[i];
      double ji[9];
      if (!minverse(jac, ji)) break;
      const v3 step = mv(ji, g);
      double damp = 1.0;
      v3 xn = x, gx = g;
      double gnn = gn;
      for (int h = 0; h < 4; ++h) {
        const v3 cand = vsub(x, vmul(step, damp));
        skin_interp(m, cand, w);
        const v3 gc = vsub(lbs(c, cand, w), xt);
        const double gcn = vnorm(gc);
        if (gcn < gn || h == 3) {
          xn = cand;
          gx = gc;
          gnn = gcn;
          break;
        }
        damp *= 0.5;
      }
      if (gnn >= gn && gn >= m->tolerance) break;
      x = xn;
      g = gx;
      gn = gnn;
      converged = gn < m->tolerance;
    }
    if (converged) roots_push(&R, x, gn, m->dedup_radius);
  }
  return R;
}

typedef struct {
  int has_root;
  float density, color[3];
  v3 canonical;
} posed_t;

static posed_t posed_query(const field_t* f, const ctx_t* c, v3 xt, scratch_t* s) { /* :163-181 */
  posed_t best;
  memset(&best, 0, sizeof best);
  const roots_t R = inverse_lbs(f->m, c, xt);
  for (int i = 0; i < R.count; ++i) {
    if (!grid_contains(f->m, R.x[i])) continue;
    float d, col[3];
    field_query(f, R.x[i], s, &d, col);
    if (!best.has_root || d > best.density) {
      best.density = d;
      memcpy(best.color, col, sizeof col);
      best.canonical = R.x[i];
      best.has_root = 1;
    }
  }
  return best;
}

/* PosedModelView R/model.hpp:85-114: normalized-space context, counters */
typedef struct {
  ctx_t ctx;
  double w2n[12];
  uint64_t posed, canonical;
} view_t;

static void view_make(const ao_model* m, const double* bones12, const double* global12, view_t* v) {
  rinverse(global12, v->w2n);
  ctx_make(&m->skel, bones12, v->w2n, 3.0, &v->ctx);
  v->posed = v->canonical = 0;
}
static posed_t view_query(const field_t* f, view_t* v, v3 xn, scratch_t* s) {
  v->posed++;
  posed_t p = posed_query(f, &v->ctx, xn, s);
  if (p.has_root) v->canonical++;
  return p;
}

/* ---------------------------------------------------------------- public: model */

static int model_sizes_(const ao_skeleton* s, const ao_grid_cfg* g, const ao_mlp_cfg* mc, const int* skin_res,
                        size_t* n_grid, size_t* n_mlp, size_t* n_skin) {
  int e = grid_validate(g);
  if (e) return e;
  if (mc->input_dim < 1 || mc->hidden_dim < 1 || mc->output_dim < 1) return fail(1, "mlp: dimensions must be >= 1");
  if (mc->hidden_layers < 1 || mc->hidden_layers > 8) return fail(1, "mlp: hidden_layers out of range");
  *n_grid = (size_t)g->levels * ((size_t)1 << g->table_size_log2) * (size_t)g->features_per_level;
  size_t n = 0;
  int in = g->levels * g->features_per_level;
  for (int l = 0; l < mc->hidden_layers + 1; ++l) {
    const int out = (l == mc->hidden_layers) ? mc->output_dim : mc->hidden_dim;
    n += (size_t)in * out + out;
    in = out;
  }
  *n_mlp = n;
  *n_skin = (size_t)skin_res[0] * skin_res[1] * skin_res[2] * (size_t)s->n_bones;
  return 0;
}

int arfo_model_sizes(const ao_skeleton* s, const ao_grid_cfg* g, const ao_mlp_cfg* m, const int skin_res[3],
                     size_t* n_grid, size_t* n_mlp, size_t* n_skin) {
  return model_sizes_(s, g, m, skin_res, n_grid, n_mlp, n_skin);
}

int arfo_build_model(const ao_skeleton* s, const ao_grid_cfg* g, const ao_mlp_cfg* mc, const int skin_res[3],
                     uint64_t seed, ao_model* out) { /* build_model R/model.hpp:68-80 */
  int e = validate_skeleton(s);
  if (e) return e;
  const box3 canon = rest_bounds(s, 0.10);
  ao_grid_cfg gc = *g;
  vstore(gc.box_lo, canon.lo);
  vstore(gc.box_hi, canon.hi);
  size_t ng, nm, ns;
  e = model_sizes_(s, &gc, mc, skin_res, &ng, &nm, &ns);
  if (e) return e;
  if (out->n_grid != ng || out->n_mlp != nm || out->n_skin != ns)
    return fail(1, "build_model: output array sizes do not match model_sizes");
  out->skel = *s;
  out->grid = gc;
  out->mlp = *mc;
  out->mlp.input_dim = gc.levels * gc.features_per_level;
  /* HashGrid ctor R/hash_grid.hpp:66-73 */
  pcg r = keyed_rng(seed, 0x6a1d, 17, 0);
  for (size_t i = 0; i < ng; ++i) out->grid_params[i] = (float)pcg_uniform(&r, -1e-4, 1e-4);
  /* DecoderMlp ctor R/mlp.hpp:50-58 (CanonicalField passes seed + 1, R/field.hpp:50) */
  field_t f;
  e = field_prepare(out, &f);
  if (e) return e;
  pcg rm = keyed_rng(seed + 1, 0x3317, 29, 0);
  for (int l = 0; l < f.nl; ++l) {
    const double sc = sqrt(6.0 / (double)f.lin[l]);
    float* w = out->mlp_params + f.woff[l];
    for (size_t i = 0; i < (size_t)f.lin[l] * (size_t)f.lout[l]; ++i) w[i] = (float)pcg_uniform(&rm, -sc, sc);
    float* b = out->mlp_params + f.boff[l];
    for (int i = 0; i < f.lout[l]; ++i) b[i] = 0.0f;
  }
  for (int a = 0; a < 3; ++a) out->skin_res[a] = skin_res[a];
  vstore(out->skin_lo, canon.lo);
  vstore(out->skin_hi, canon.hi);
  vstore(out->canon_lo, canon.lo);
  vstore(out->canon_hi, canon.hi);
  e = build_skinning(s, out->skin_lo, out->skin_hi, skin_res, 1.5, out->skin_weights);
  if (e) return e;
  /* normalized_reach_box R/model.hpp:59-66 */
  const double reach = max_reach(s) * 1.05;
  const v3 root = vload(s->head[0]);
  box3 nb = box_empty();
  box_expand(&nb, vsub(root, V(reach, reach, reach)));
  box_expand(&nb, vadd(root, V(reach, reach, reach)));
  vstore(out->norm_lo, nb.lo);
  vstore(out->norm_hi, nb.hi);
  out->max_iterations = 20; /* InverseLbsOptions R/articulation.hpp:84-88 */
  out->tolerance = 1e-5;
  out->dedup_radius = 1e-3;
  return 0;
}

int arfo_pose_from_joint_rotations(const ao_skeleton* s, const double* rot9, const double* g12,
                                   double* bones12) { /* R/skeleton.hpp:93-110 */
  int e = validate_skeleton(s);
  if (e) return e;
  double chain[AO_MAX_BONES][12];
  for (int i = 0; i < s->n_bones; ++i) {
    double local[12];
    memcpy(local, rot9 + 9 * i, 9 * sizeof(double));
    const v3 h = vload(s->head[i]);
    vstore(local + 9, vsub(h, mv(local, h))); /* Rigid::about_point R/math.hpp:210-212 */
    if (s->parent[i] < 0) memcpy(chain[i], local, sizeof local);
    else rcompose(chain[s->parent[i]], local, chain[i]);
    rcompose(g12, chain[i], bones12 + 12 * i);
  }
  return 0;
}

int arfo_look_at(const double eye[3], const double target[3], const double up[3], double focal, int w, int h,
                 ao_camera* cam) { /* Camera::look_at R/camera.hpp:31-48 */
  cam->width = w;
  cam->height = h;
  cam->fx = cam->fy = focal;
  cam->cx = w * 0.5;
  cam->cy = h * 0.5;
  const v3 fwd = vnormalized(vsub(vload(target), vload(eye)));
  v3 down = vadd(vneg(vload(up)), vmul(fwd, vdot(vload(up), fwd)));
  down = vnormalized(down);
  const v3 right = vcross(down, fwd);
  const double r[9] = {right.x, right.y, right.z, down.x, down.y, down.z, fwd.x, fwd.y, fwd.z};
  memcpy(cam->extrinsic, r, sizeof r);
  vstore(cam->extrinsic + 9, vneg(mv(r, vload(eye))));
  return 0;
}

int arfo_skinning_weights(const ao_model* m, const double* pts, int64_t n, double* w) {
  for (int64_t i = 0; i < n; ++i) skin_interp(m, vload(pts + 3 * i), w + i * m->skel.n_bones);
  return 0;
}

int arfo_inverse_lbs(const ao_model* m, const double* bones12, const double* pre12, double cutoff_factor,
                     const double* pts, int64_t n, int32_t* counts, double* roots, double* residuals) {
  ctx_t c;
  ctx_make(&m->skel, bones12, pre12, cutoff_factor, &c);
  for (int64_t i = 0; i < n; ++i) {
    const roots_t R = inverse_lbs(m, &c, vload(pts + 3 * i));
    counts[i] = R.count;
    for (int k = 0; k < R.count; ++k) {
      vstore(roots + (i * AO_MAX_ROOTS + k) * 3, R.x[k]);
      residuals[i * AO_MAX_ROOTS + k] = R.r[k];
    }
  }
  return 0;
}

int arfo_hash_encode(const ao_model* m, const double* pts, int64_t n, float* feats) {
  field_t f;
  int e = field_prepare(m, &f);
  if (e) return e;
  for (int64_t i = 0; i < n; ++i) {
    const v3 x = vload(pts + 3 * i);
    if (!grid_contains(m, x)) return fail(4, "hash grid: point outside bounding box"); /* :178 */
    encode(&f, x, feats + i * f.D);
  }
  return 0;
}

int arfo_field_query(const ao_model* m, const double* pts, int64_t n, float* dens, float* col) {
  field_t f;
  scratch_t s;
  int e = field_prepare(m, &f);
  if (e || (e = scratch_alloc(&f, &s))) return e;
  for (int64_t i = 0; i < n; ++i) {
    const v3 x = vload(pts + 3 * i);
    if (!grid_contains(m, x)) {
      scratch_free(&s);
      return fail(4, "hash grid: point outside bounding box");
    }
    field_query(&f, x, &s, dens + i, col + 3 * i);
  }
  scratch_free(&s);
  return 0;
}

int arfo_posed_query(const ao_model* m, const double* bones12, const double* global12, const double* pts,
                     int64_t n, float* dens, float* col, double* canon, uint8_t* has_root) {
  field_t f;
  scratch_t s;
  int e = field_prepare(m, &f);
  if (e || (e = scratch_alloc(&f, &s))) return e;
  view_t v;
  view_make(m, bones12, global12, &v);
  for (int64_t i = 0; i < n; ++i) {
    const posed_t p = view_query(&f, &v, vload(pts + 3 * i), &s);
    has_root[i] = (uint8_t)p.has_root;
    dens[i] = p.has_root ? p.density : 0.0f;
    for (int c = 0; c < 3; ++c) col[3 * i + c] = p.has_root ? p.color[c] : 0.0f;
    vstore(canon + 3 * i, p.has_root ? p.canonical : V(0, 0, 0));
  }
  scratch_free(&s);
  return 0;
}

/* ---------------------------------------------------------------- occupancy  R/occupancy.hpp */

int arfo_occ_empty(const double lo[3], const double hi[3], const ao_occ_cfg* c, ao_occ_grid* g) { /* :59-69 */
  if (c->resolution < 2) return fail(1, "occupancy: resolution must be >= 2");
  if (!(c->alpha_threshold > 0 && c->alpha_threshold < 1))
    return fail(1, "occupancy: alpha_threshold must be in (0,1)");
  if (c->dilation < 0) return fail(1, "occupancy: dilation must be >= 0");
  if (!(c->decay >= 0 && c->decay <= 1)) return fail(1, "occupancy: decay in [0,1]");
  if (c->update_interval < 1) return fail(1, "occupancy: update_interval must be >= 1");
  for (int a = 0; a < 3; ++a) {
    g->res[a] = c->resolution;
    g->box_lo[a] = lo[a];
    g->box_hi[a] = hi[a];
  }
  g->dilation = c->dilation;
  const v3 cs = V((hi[0] - lo[0]) / c->resolution, (hi[1] - lo[1]) / c->resolution, (hi[2] - lo[2]) / c->resolution);
  g->density_threshold = -log1p(-c->alpha_threshold) / vnorm(cs);
  const size_t n = (size_t)c->resolution * c->resolution * c->resolution;
  if (g->values) memset(g->values, 0, n * sizeof(float));
  if (g->mask) memset(g->mask, 0, n);
  return 0;
}

static size_t occ_cells(const ao_occ_grid* g) { return (size_t)g->res[0] * g->res[1] * g->res[2]; }

static void dilate_pass(const ao_occ_grid* g, const uint8_t* src, uint8_t* dst, int axis, int r) { /* :103-119 */
  const int n[3] = {g->res[0], g->res[1], g->res[2]};
  const size_t stride[3] = {1, (size_t)n[0], (size_t)n[0] * n[1]};
  for (int iz = 0; iz < n[2]; ++iz)
    for (int iy = 0; iy < n[1]; ++iy)
      for (int ix = 0; ix < n[0]; ++ix) {
        const int idx[3] = {ix, iy, iz};
        const size_t base = ix * stride[0] + iy * stride[1] + iz * stride[2];
        uint8_t v = 0;
        for (int d = -r; d <= r && !v; ++d) {
          const int j = idx[axis] + d;
          if (j < 0 || j >= n[axis]) continue;
          v = src[(ptrdiff_t)base + (ptrdiff_t)(j - idx[axis]) * (ptrdiff_t)stride[axis]];
        }
        dst[base] = v;
      }
}

int arfo_occ_rebuild_mask(ao_occ_grid* g) { /* :87-91, dilated_mask :101-125 */
  const size_t n = occ_cells(g);
  const float thr = (float)g->density_threshold;
  for (size_t i = 0; i < n; ++i) g->mask[i] = g->values[i] >= thr ? 1 : 0;
  if (g->dilation > 0) {
    uint8_t* b = (uint8_t*)malloc(n);
    if (!b) return fail(5, "oracle: out of memory");
    dilate_pass(g, g->mask, b, 0, g->dilation);
    dilate_pass(g, b, g->mask, 1, g->dilation);
    dilate_pass(g, g->mask, b, 2, g->dilation);
    memcpy(g->mask, b, n);
    free(b);
  }
  return 0;
}

static v3 cell_size(const ao_occ_grid* g) { /* :49-52 */
  return V((g->box_hi[0] - g->box_lo[0]) / g->res[0], (g->box_hi[1] - g->box_lo[1]) / g->res[1],
           (g->box_hi[2] - g->box_lo[2]) / g->res[2]);
}

int arfo_build_inference_grid(const ao_model* m, const double* bones12, const double* global12, const ao_occ_cfg* c,
                              ao_occ_grid* g, uint64_t* counters) { /* :137-149 via R/model.hpp:138-148 */
  int e = arfo_occ_empty(m->norm_lo, m->norm_hi, c, g);
  if (e) return e;
  field_t f;
  scratch_t s;
  if ((e = field_prepare(m, &f)) || (e = scratch_alloc(&f, &s))) return e;
  view_t v;
  view_make(m, bones12, global12, &v);
  const v3 cs = cell_size(g);
  const int rx = g->res[0], ry = g->res[1];
  const size_t n = occ_cells(g);
  for (size_t i = 0; i < n; ++i) {
    const int ix = (int)(i % (size_t)rx), iy = (int)((i / (size_t)rx) % (size_t)ry),
              iz = (int)(i / ((size_t)rx * ry));
    const v3 x = V(g->box_lo[0] + (ix + 0.5) * cs.x, g->box_lo[1] + (iy + 0.5) * cs.y,
                   g->box_lo[2] + (iz + 0.5) * cs.z); /* cell_center :53-58 */
    const posed_t p = view_query(&f, &v, x, &s);
    const double d = p.has_root ? (double)p.density : 0.0; /* density_normalized R/model.hpp:109-113 */
    g->values[i] = (float)dmin_(d, 1.0);
  }
  scratch_free(&s);
  if (counters) {
    counters[0] = v.posed;
    counters[1] = v.canonical;
  }
  return arfo_occ_rebuild_mask(g);
}

int arfo_update_training_grid(const ao_model* m, int n_poses, const double* bones12, const double* global12,
                              double decay, uint64_t seed, uint64_t step, ao_occ_grid* g,
                              uint64_t* counters) { /* R/occupancy.hpp:155-171 */
  field_t f;
  scratch_t s;
  int e;
  if (n_poses < 1) return fail(1, "update_training_grid: need >= 1 pose");
  if ((e = field_prepare(m, &f)) || (e = scratch_alloc(&f, &s))) return e;
  view_t* views = (view_t*)malloc(sizeof(view_t) * (size_t)n_poses);
  if (!views) return fail(5, "oracle: out of memory");
  const int nb = m->skel.n_bones;
  for (int p = 0; p < n_poses; ++p) view_make(m, bones12 + (size_t)p * nb * 12, global12 + 12 * p, &views[p]);
  const v3 cs = cell_size(g);
  const int rx = g->res[0], ry = g->res[1];
  const size_t n = occ_cells(g);
  for (size_t i = 0; i < n; ++i) {
    const int ix = (int)(i % (size_t)rx), iy = (int)((i / (size_t)rx) % (size_t)ry),
              iz = (int)(i / ((size_t)rx * ry));
    pcg r = keyed_rng(seed, 0x0cc0, (uint64_t)i, step);
    const int pose = (int)pcg_below(&r, (uint32_t)n_poses);
    const double jx = pcg_double(&r); /* braced init list: evaluated x, y, z in order */
    const double jy = pcg_double(&r);
    const double jz = pcg_double(&r);
    const v3 x = V(g->box_lo[0] + (ix + jx) * cs.x, g->box_lo[1] + (iy + jy) * cs.y, g->box_lo[2] + (iz + jz) * cs.z);
    const posed_t p = view_query(&f, &views[pose], x, &s);
    const float fresh = (float)dmin_(p.has_root ? (double)p.density : 0.0, 1.0);
    const float old = (float)decay * g->values[i];
    g->values[i] = (old < fresh) ? fresh : old;
  }
  if (counters) {
    counters[0] = counters[1] = 0;
    for (int p = 0; p < n_poses; ++p) {
      counters[0] += views[p].posed;
      counters[1] += views[p].canonical;
    }
  }
  free(views);
  scratch_free(&s);
  return arfo_occ_rebuild_mask(g);
}

static int occ_is_occupied(const ao_occ_grid* g, v3 x) { /* :71-85 */
  const double u[3] = {(x.x - g->box_lo[0]) / (g->box_hi[0] - g->box_lo[0]),
                       (x.y - g->box_lo[1]) / (g->box_hi[1] - g->box_lo[1]),
                       (x.z - g->box_lo[2]) / (g->box_hi[2] - g->box_lo[2])};
  if (u[0] < 0 || u[1] < 0 || u[2] < 0 || u[0] >= 1 || u[1] >= 1 || u[2] >= 1) return 0;
  int c[3];
  for (int a = 0; a < 3; ++a) {
    c[a] = (int)(u[a] * g->res[a]);
    if (g->res[a] - 1 < c[a]) c[a] = g->res[a] - 1;
  }
  return g->mask[((size_t)c[2] * g->res[1] + c[1]) * g->res[0] + c[0]] != 0;
}

/* ---------------------------------------------------------------- renderer  R/render.hpp, R/camera.hpp */

typedef struct {
  v3 o, d;
  double tn, tf;
} ray_t;

static ray_t generate_ray(const ao_camera* cam, int px, int py) { /* R/camera.hpp:61-70 */
  const v3 dc = V((px + 0.5 - cam->cx) / cam->fx, (py + 0.5 - cam->cy) / cam->fy, 1.0);
  double rt[9];
  mt(cam->extrinsic, rt);
  ray_t r;
  r.o = vneg(mv(rt, V(cam->extrinsic[9], cam->extrinsic[10], cam->extrinsic[11])));
  r.d = vnormalized(mv(rt, dc));
  r.tn = r.tf = 0.0;
  return r;
}

static int ray_box(v3 o3, v3 d3, const double* lo, const double* hi, double* tn, double* tf) { /* :15-37 */
  double t0 = 0.0, t1 = DBL_MAX;
  for (int a = 0; a < 3; ++a) {
    const double o = vget(o3, a), d = vget(d3, a);
    if (fabs(d) < 1e-300) {
      if (o < lo[a] || o > hi[a]) return 0;
      continue;
    }
    double ta = (lo[a] - o) / d, tb = (hi[a] - o) / d;
    if (ta > tb) {
      const double t = ta;
      ta = tb;
      tb = t;
    }
    t0 = dmax_(t0, ta);
    t1 = dmin_(t1, tb);
    if (t0 > t1) return 0;
  }
  *tn = t0;
  *tf = t1;
  return 1;
}

typedef struct { /* RaySampleSet<float> :41-61 */
  int n;
  double* t;
  double* delta;
  uint8_t* skipped;
  float* dens;
  float* col;
  v3* canon;
} samples_t;

static int samples_alloc(samples_t* s, int n) {
  s->n = 0;
  s->t = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  s->delta = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  s->skipped = (uint8_t*)malloc((size_t)n + 1);
  s->dens = (float*)malloc(sizeof(float) * (size_t)(n + 1));
  s->col = (float*)malloc(sizeof(float) * 3 * (size_t)(n + 1));
  s->canon = (v3*)malloc(sizeof(v3) * (size_t)(n + 1));
  return (s->t && s->delta && s->skipped && s->dens && s->col && s->canon) ? 0 : fail(5, "oracle: out of memory");
}
static void samples_free(samples_t* s) {
  free(s->t);
  free(s->delta);
  free(s->skipped);
  free(s->dens);
  free(s->col);
  free(s->canon);
}

static v3 ray_at(const ray_t* r, double t) { return vadd(r->o, vmul(r->d, t)); }

/* sample_points :67-86 with to_norm = PosedModelView::to_normalized */
static void sample_points(const ray_t* ray, int n, int stratified, pcg* rng, const ao_occ_grid* occ,
                          const double* w2n, samples_t* out) {
  out->n = 0;
  if (!(ray->tn < ray->tf) || n <= 0) return;
  out->n = n;
  const double step = (ray->tf - ray->tn) / n;
  for (int i = 0; i < n; ++i) {
    const double jitter = stratified && rng ? pcg_double(rng) : 0.5;
    out->t[i] = ray->tn + (i + jitter) * step;
    out->skipped[i] = 0;
    out->dens[i] = 0.0f;
    out->col[3 * i] = out->col[3 * i + 1] = out->col[3 * i + 2] = 0.0f;
  }
  for (int i = 0; i + 1 < n; ++i) out->delta[i] = out->t[i + 1] - out->t[i];
  out->delta[n - 1] = ray->tf - out->t[n - 1];
  if (occ)
    for (int i = 0; i < n; ++i) out->skipped[i] = occ_is_occupied(occ, rapply(w2n, ray_at(ray, out->t[i]))) ? 0 : 1;
}

/* composite :98-119 */
static int composite(const samples_t* s, double eps, double* c3, double* alpha) {
  double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0, a = 0.0;
  int i = 0;
  for (; i < s->n; ++i) {
    if (eps > 0 && T <= eps) break;
    const double sigma = s->skipped[i] ? 0.0 : (double)s->dens[i];
    if (sigma <= 0.0) continue;
    const double al = -expm1(-sigma * s->delta[i]);
    const double w = al * T;
    cr += (double)s->col[3 * i] * w;
    cg += (double)s->col[3 * i + 1] * w;
    cb += (double)s->col[3 * i + 2] * w;
    a += w;
    T *= 1.0 - al;
  }
  c3[0] = cr;
  c3[1] = cg;
  c3[2] = cb;
  *alpha = a;
  return i;
}

/* composite_backward :125-157 */
static int composite_backward(const samples_t* s, int m, const double* dC, double dA, double* ds, double* dc) {
  double* trans = (double*)malloc(sizeof(double) * (size_t)(m + 1));
  if (!trans) return fail(5, "oracle: out of memory");
  for (int i = 0; i < s->n; ++i) {
    ds[i] = 0.0;
    dc[3 * i] = dc[3 * i + 1] = dc[3 * i + 2] = 0.0;
  }
  trans[0] = 1.0;
  for (int i = 0; i < m; ++i) {
    const double sigma = s->skipped[i] ? 0.0 : (double)s->dens[i];
    const double al = sigma <= 0.0 ? 0.0 : -expm1(-sigma * s->delta[i]);
    trans[i + 1] = trans[i] * (1.0 - al);
  }
  v3 chat = V(0, 0, 0);
  double ahat = 0.0;
  for (int i = m - 1; i >= 0; --i) {
    if (s->skipped[i]) continue;
    const double sigma = (double)s->dens[i];
    const double al = sigma <= 0.0 ? 0.0 : -expm1(-sigma * s->delta[i]);
    const v3 c = V((double)s->col[3 * i], (double)s->col[3 * i + 1], (double)s->col[3 * i + 2]);
    const double dC_dalpha = vdot(V(dC[0], dC[1], dC[2]), vsub(c, chat));
    const double dA_dalpha = 1.0 - ahat;
    const double dat = trans[i] * (dC_dalpha + dA * dA_dalpha);
    ds[i] = dat * s->delta[i] * (1.0 - al);
    const double at = al * trans[i];
    dc[3 * i] = dC[0] * at;
    dc[3 * i + 1] = dC[1] * at;
    dc[3 * i + 2] = dC[2] * at;
    chat = vadd(vmul(c, al), vmul(chat, 1.0 - al));
    ahat = al + ahat * (1.0 - al);
  }
  free(trans);
  return 0;
}

/* render_image R/render.hpp:178-218 bound to the model like render_model R/model.hpp:118-135 */
static int render_impl(const ao_model* m, const double* bones12, const double* global12, const ao_camera* cam,
                       const ao_occ_grid* occ, const ao_render_opts* o, float* rgb, float* alpha, uint64_t* counters,
                       ao_render_trace* tr) {
  field_t f;
  scratch_t s;
  samples_t S;
  int e;
  if ((e = field_prepare(m, &f)) || (e = scratch_alloc(&f, &s))) return e;
  if ((e = samples_alloc(&S, o->samples_per_ray > 0 ? o->samples_per_ray : 1))) return e;
  view_t v;
  view_make(m, bones12, global12, &v);
  int64_t ns = 0;
  for (int py = 0; py < cam->height; ++py)
    for (int px = 0; px < cam->width; ++px) {
      const size_t pix = (size_t)py * cam->width + px;
      rgb[3 * pix] = rgb[3 * pix + 1] = rgb[3 * pix + 2] = 0.0f;
      alpha[pix] = 0.0f;
      if (tr) {
        tr->ray_first[pix] = -1;
        tr->ray_count[pix] = 0;
        tr->ray_hit[pix] = 0;
        tr->t_near[pix] = tr->t_far[pix] = 0.0;
        tr->terminated_at[pix] = 0;
      }
      ray_t ray = generate_ray(cam, px, py);
      const v3 on = rapply(v.w2n, ray.o);
      const v3 dn = vsub(rapply(v.w2n, ray_at(&ray, 1.0)), on);
      double tn, tf;
      if (!ray_box(on, dn, m->norm_lo, m->norm_hi, &tn, &tf)) continue;
      ray.tn = tn;
      ray.tf = tf;
      pcg rng = keyed_rng(o->seed, o->frame_id, (uint64_t)pix, 0);
      sample_points(&ray, o->samples_per_ray, o->stratified, &rng, occ, v.w2n, &S);
      if (tr) {
        tr->ray_hit[pix] = 1;
        tr->t_near[pix] = tn;
        tr->t_far[pix] = tf;
        tr->ray_first[pix] = (int32_t)ns;
      }
      for (int i = 0; i < S.n; ++i) {
        if (S.skipped[i]) continue;
        const posed_t p = view_query(&f, &v, rapply(v.w2n, ray_at(&ray, S.t[i])), &s);
        if (!p.has_root) S.skipped[i] = 1;
        else {
          S.dens[i] = p.density;
          memcpy(S.col + 3 * i, p.color, 3 * sizeof(float));
        }
        if (tr) {
          if (ns < tr->capacity) {
            tr->s_ray[ns] = (int32_t)pix;
            tr->s_index[ns] = i;
            tr->s_has_root[ns] = (uint8_t)p.has_root;
            tr->s_density[ns] = p.has_root ? p.density : 0.0f;
            for (int c = 0; c < 3; ++c) tr->s_color[3 * ns + c] = p.has_root ? p.color[c] : 0.0f;
            vstore(tr->s_canonical + 3 * ns, p.has_root ? p.canonical : V(0, 0, 0));
            tr->s_t[ns] = S.t[i];
            tr->s_delta[ns] = S.delta[i];
          }
          ++tr->ray_count[pix];
        }
        ++ns;
      }
      double c3[3], a;
      const int term = composite(&S, o->epsilon_terminate, c3, &a);
      if (tr) tr->terminated_at[pix] = term;
      rgb[3 * pix] = (float)c3[0];
      rgb[3 * pix + 1] = (float)c3[1];
      rgb[3 * pix + 2] = (float)c3[2];
      alpha[pix] = (float)a;
    }
  if (tr) tr->n_samples = ns;
  if (counters) {
    counters[0] = v.posed;
    counters[1] = v.canonical;
  }
  samples_free(&S);
  scratch_free(&s);
  return 0;
}

int arfo_render(const ao_model* m, const double* bones12, const double* global12, const ao_camera* cam,
                const ao_occ_grid* occ, const ao_render_opts* o, float* rgb, float* alpha, uint64_t* counters) {
  return render_impl(m, bones12, global12, cam, occ, o, rgb, alpha, counters, NULL);
}

int arfo_render_trace(const ao_model* m, const double* bones12, const double* global12, const ao_camera* cam,
                      const ao_occ_grid* occ, const ao_render_opts* o, float* rgb, float* alpha, uint64_t* counters,
                      ao_render_trace* tr) {
  return render_impl(m, bones12, global12, cam, occ, o, rgb, alpha, counters, tr);
}

static void samples_view(samples_t* S, int n, const double* t, const double* delta, const uint8_t* skipped,
                         const float* dens, const float* col) {
  S->n = n;
  S->t = (double*)t;
  S->delta = (double*)delta;
  S->skipped = (uint8_t*)skipped;
  S->dens = (float*)dens;
  S->col = (float*)col;
  S->canon = NULL;
}

int arfo_composite(int n, const double* t, const double* delta, const uint8_t* skipped, const float* dens,
                   const float* col, double eps, double* color3, double* alpha, int* terminated_at) {
  samples_t S;
  samples_view(&S, n, t, delta, skipped, dens, col);
  *terminated_at = composite(&S, eps, color3, alpha);
  return 0;
}

int arfo_composite_backward(int n, const double* t, const double* delta, const uint8_t* skipped, const float* dens,
                            const float* col, double eps, const double* d_color3, double d_alpha, double* d_sigma,
                            double* d_c3) {
  samples_t S;
  samples_view(&S, n, t, delta, skipped, dens, col);
  double c3[3], a;
  const int m = composite(&S, eps, c3, &a);
  return composite_backward(&S, m, d_color3, d_alpha, d_sigma, d_c3);
}

int arfo_field_query_backward(const ao_model* m, const double* pts, int64_t n, const float* d_dens,
                              const float* d_col, float* grid_grad, float* mlp_grad) {
  field_t f;
  scratch_t s;
  int e;
  if ((e = field_prepare(m, &f)) || (e = scratch_alloc(&f, &s))) return e;
  for (int64_t i = 0; i < n; ++i) {
    const v3 x = vload(pts + 3 * i);
    if (!grid_contains(m, x)) {
      scratch_free(&s);
      return fail(4, "hash grid: point outside bounding box");
    }
    field_query_backward(&f, x, d_dens[i], d_col + 3 * i, &s, grid_grad, mlp_grad);
  }
  scratch_free(&s);
  return 0;
}

/* training forward+backward composed per SPEC.md:490-494 (see ref_driver.cpp arfr_train_fwd_bwd) */
int arfo_train_fwd_bwd(const ao_model* m, const double* bones12, const double* global12, const ao_camera* cam,
                       const ao_occ_grid* occ, const ao_render_opts* o, int64_t n_rays, const int32_t* px,
                       const int32_t* py, const float* d_color, const float* d_alpha, float* rgb, float* alpha,
                       float* grid_grad, float* mlp_grad, uint64_t* counters) {
  field_t f;
  scratch_t s;
  samples_t S;
  int e;
  if ((e = field_prepare(m, &f)) || (e = scratch_alloc(&f, &s))) return e;
  const int N = o->samples_per_ray > 0 ? o->samples_per_ray : 1;
  if ((e = samples_alloc(&S, N))) return e;
  double* ds = (double*)malloc(sizeof(double) * (size_t)N);
  double* dc = (double*)malloc(sizeof(double) * 3 * (size_t)N);
  if (!ds || !dc) return fail(5, "oracle: out of memory");
  view_t v;
  view_make(m, bones12, global12, &v);
  for (int64_t r = 0; r < n_rays; ++r) {
    rgb[3 * r] = rgb[3 * r + 1] = rgb[3 * r + 2] = 0.0f;
    alpha[r] = 0.0f;
    const size_t pix = (size_t)py[r] * cam->width + px[r];
    ray_t ray = generate_ray(cam, px[r], py[r]);
    const v3 on = rapply(v.w2n, ray.o);
    const v3 dn = vsub(rapply(v.w2n, ray_at(&ray, 1.0)), on);
    double tn, tf;
    if (!ray_box(on, dn, m->norm_lo, m->norm_hi, &tn, &tf)) continue;
    ray.tn = tn;
    ray.tf = tf;
    pcg rng = keyed_rng(o->seed, o->frame_id, (uint64_t)pix, 0);
    sample_points(&ray, o->samples_per_ray, o->stratified, &rng, occ, v.w2n, &S);
    for (int i = 0; i < S.n; ++i) {
      if (S.skipped[i]) continue;
      const posed_t p = view_query(&f, &v, rapply(v.w2n, ray_at(&ray, S.t[i])), &s);
      if (!p.has_root) {
        S.skipped[i] = 1;
        continue;
      }
      S.dens[i] = p.density;
      memcpy(S.col + 3 * i, p.color, 3 * sizeof(float));
      S.canon[i] = p.canonical;
    }
    double c3[3], a;
    const int term = composite(&S, o->epsilon_terminate, c3, &a);
    rgb[3 * r] = (float)c3[0];
    rgb[3 * r + 1] = (float)c3[1];
    rgb[3 * r + 2] = (float)c3[2];
    alpha[r] = (float)a;
    const double dC[3] = {d_color[3 * r], d_color[3 * r + 1], d_color[3 * r + 2]};
    if ((e = composite_backward(&S, term, dC, d_alpha[r], ds, dc))) return e;
    for (int i = 0; i < term; ++i) {
      if (S.skipped[i]) continue;
      const float dcf[3] = {(float)dc[3 * i], (float)dc[3 * i + 1], (float)dc[3 * i + 2]};
      field_query_backward(&f, S.canon[i], (float)ds[i], dcf, &s, grid_grad, mlp_grad);
    }
  }
  if (counters) {
    counters[0] = v.posed;
    counters[1] = v.canonical;
  }
  free(ds);
  free(dc);
  samples_free(&S);
  scratch_free(&s);
  return 0;
}

/* ---- analytic ground truth: CapsuleFigure / PosedFigure (R/scene.hpp:10-130) ---------- */

typedef struct {
  int nb;
  v3 a[AO_MAX_BONES], b[AO_MAX_BONES];
} figpose_t;

static int figure_prepare(const ao_figure* f, const double* bones12, figpose_t* P) { /* :19-26, :61-75 */
  int e;
  if ((e = validate_skeleton(&f->skel))) return e;
  for (int i = 0; i < f->skel.n_bones; ++i)
    if (!(f->amplitude[i] > 0)) return fail(1, "figure: amplitudes must be positive");
  if (!(f->softness > 0)) return fail(1, "figure: softness must be positive");
  P->nb = f->skel.n_bones;
  for (int i = 0; i < P->nb; ++i) {
    const v3 h = vload(f->skel.head[i]), t = vload(f->skel.tail[i]);
    P->a[i] = bones12 ? rapply(bones12 + 12 * i, h) : h;
    P->b[i] = bones12 ? rapply(bones12 + 12 * i, t) : t;
  }
  return 0;
}

static double smoothstep01(double t) { /* R/math.hpp:25-35 */
  t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);
  return t * t * (3.0 - 2.0 * t);
}

/* PosedFigure::query :79-97 (analytic_query :31-50 with rest segments) */
static double figure_query(const ao_figure* f, const figpose_t* P, v3 x, v3* color) {
  double total = 0.0;
  v3 acc = V(0, 0, 0);
  *color = V(0, 0, 0);
  for (int i = 0; i < P->nb; ++i) {
    const double d = point_segment_distance(x, P->a[i], P->b[i]);
    if (d >= f->skel.radius[i]) continue;
    const double s = smoothstep01((f->skel.radius[i] - d) / f->softness);
    if (s <= 0.0) continue;
    const double dens = f->amplitude[i] * s;
    total += dens;
    acc = vadd(acc, vmul(vload(f->color[i]), dens));
  }
  if (total > 0.0) {
    *color = V(acc.x / total, acc.y / total, acc.z / total);
    return total;
  }
  return 0.0;
}

static double ray_segment_distance(v3 o, v3 d, v3 a, v3 b) { /* :103-117 */
  const v3 ab = vsub(b, a);
  double best = 1.7976931348623157e308;
  for (int i = 0; i <= 64; ++i) {
    const double u = (double)i / 64;
    const v3 p = vadd(a, vmul(ab, u));
    const double t = dmax_(0.0, vdot(vsub(p, o), d));
    best = dmin_(best, vnorm(vsub(p, vadd(o, vmul(d, t)))));
  }
  return best;
}

int arfo_figure_query(const ao_figure* f, const double* bones12, const double* pts, int64_t n, double* dens,
                      double* col) {
  figpose_t P;
  int e;
  if ((e = figure_prepare(f, bones12, &P))) return e;
  for (int64_t i = 0; i < n; ++i) {
    v3 c;
    dens[i] = figure_query(f, &P, vload(pts + 3 * i), &c);
    vstore(col + 3 * i, c);
  }
  return 0;
}

/* render_image :178-218 over PosedFigure::query (matter iff density > 0), to_norm = G^-1,
 * no occupancy; mask = PosedFigure::ray_hits :123-130 (the dataset's exact alpha) */
int arfo_figure_render(const ao_figure* f, const double* bones12, const double* global12, const double lo[3],
                       const double hi[3], const ao_camera* cam, const ao_render_opts* o, float* rgb, float* alpha,
                       uint8_t* mask) {
  figpose_t P;
  int e;
  if ((e = figure_prepare(f, bones12, &P))) return e;
  double w2n[12];
  rinverse(global12, w2n);
  const int N = o->samples_per_ray;
  double* t = (double*)malloc(sizeof(double) * (size_t)(N + 1));
  if (!t) return fail(5, "oracle: out of memory");
  for (int py = 0; py < cam->height; ++py)
    for (int px = 0; px < cam->width; ++px) {
      const size_t pix = (size_t)py * cam->width + px;
      ray_t ray = generate_ray(cam, px, py);
      if (mask) {
        int hit = 0;
        for (int i = 0; i < P.nb && !hit; ++i)
          hit = ray_segment_distance(ray.o, ray.d, P.a[i], P.b[i]) < f->skel.radius[i];
        mask[pix] = (uint8_t)hit;
      }
      double cr = 0, cg = 0, cb = 0, a = 0;
      const v3 on = rapply(w2n, ray.o);
      const v3 dn = vsub(rapply(w2n, ray_at(&ray, 1.0)), on);
      double tn, tf;
      if (ray_box(on, dn, lo, hi, &tn, &tf) && tn < tf && N > 0) {
        pcg rng = keyed_rng(o->seed, o->frame_id, (uint64_t)pix, 0);
        const double step = (tf - tn) / N;
        for (int i = 0; i < N; ++i) t[i] = tn + (i + (o->stratified ? pcg_double(&rng) : 0.5)) * step;
        double T = 1.0;
        for (int i = 0; i < N; ++i) {
          if (o->epsilon_terminate > 0 && T <= o->epsilon_terminate) break;
          v3 c;
          const double sigma = figure_query(f, &P, ray_at(&ray, t[i]), &c);
          if (sigma <= 0.0) continue;
          const double delta = (i + 1 < N) ? t[i + 1] - t[i] : tf - t[i];
          const double al = -expm1(-sigma * delta);
          const double w = al * T;
          cr += c.x * w;
          cg += c.y * w;
          cb += c.z * w;
          a += w;
          T *= 1.0 - al;
        }
      }
      if (rgb) {
        rgb[3 * pix] = (float)cr;
        rgb[3 * pix + 1] = (float)cg;
        rgb[3 * pix + 2] = (float)cb;
      }
      if (alpha) alpha[pix] = (float)a;
    }
  free(t);
  return 0;
}

/* ---- training losses + optimizer (no reference code exists) ---------- */

/* Eq. 9-11 per ray on the f32 rendered values, in double; gradients of the weighted batch
 * mean rounded to f32 (hard subgradient at 0/1 = one-sided limit inside). */
int arfo_losses(int64_t n, const float* rgb, const float* alpha, const float* gt_rgb, const float* gt_alpha,
                const ao_loss_cfg* c, double* loss4, float* d_rgb, float* d_alpha) {
  if (!(c->huber_delta > 0)) return fail(1, "loss: huber_delta must be positive");
  const double inv_n = n > 0 ? 1.0 / (double)n : 0.0;
  double sr = 0, sa = 0, sh = 0;
  for (int64_t r = 0; r < n; ++r) {
    const double ex = (double)rgb[3 * r] - (double)gt_rgb[3 * r];
    const double ey = (double)rgb[3 * r + 1] - (double)gt_rgb[3 * r + 1];
    const double ez = (double)rgb[3 * r + 2] - (double)gt_rgb[3 * r + 2];
    const double rn = sqrt(ex * ex + ey * ey + ez * ez);
    const double d = c->huber_delta;
    double lr, gs;
    if (rn <= d) {
      lr = 0.5 * (rn * rn);
      gs = 1.0;
    } else {
      lr = d * (rn - 0.5 * d);
      gs = d / rn;
    }
    const double crgb = c->w_rgb * inv_n;
    if (d_rgb) {
      d_rgb[3 * r] = (float)(crgb * (ex * gs));
      d_rgb[3 * r + 1] = (float)(crgb * (ey * gs));
      d_rgb[3 * r + 2] = (float)(crgb * (ez * gs));
    }
    const double A = (double)alpha[r];
    const double ea = A - (double)gt_alpha[r];
    const double la = fabs(ea);
    const double s1 = ea > 0.0 ? 1.0 : (ea < 0.0 ? -1.0 : 0.0);
    const double p = exp(-fabs(A)), q = exp(-fabs(A - 1.0));
    const double sum = p + q;
    const double lh = -log(sum) + log1p(exp(-1.0));
    const double sp = A < 0.0 ? -1.0 : 1.0, sq = A > 1.0 ? 1.0 : -1.0;
    const double dh = (sp * p + sq * q) / sum;
    if (d_alpha) d_alpha[r] = (float)((c->w_alpha * s1 + c->w_hard * dh) * inv_n);
    sr += lr;
    sa += la;
    sh += lh;
  }
  if (loss4) {
    loss4[0] = sr * inv_n;
    loss4[1] = sa * inv_n;
    loss4[2] = sh * inv_n;
    loss4[3] = c->w_rgb * loss4[0] + c->w_alpha * loss4[1] + c->w_hard * loss4[2];
  }
  return 0;
}

static double cosine_lr(double lr0, const ao_adam_cfg* c, int64_t step) {
  if (c->total_steps <= 0) return lr0;
  const double t = (double)(step < c->total_steps ? step : c->total_steps) / (double)c->total_steps;
  const double f = c->final_lr_factor;
  return lr0 * (f + (1.0 - f) * 0.5 * (1.0 + cos(3.14159265358979323846 * t)));
}

int arfo_adam(int64_t n, float* p, float* g, float* m, float* v, const ao_adam_cfg* c, int64_t step,
              int64_t mlp_offset) {
  if (step < 1) return fail(1, "adam: step must be >= 1");
  const float b1 = (float)c->beta1, omb1 = (float)(1.0 - c->beta1);
  const float b2 = (float)c->beta2, omb2 = (float)(1.0 - c->beta2);
  const float c1 = (float)(1.0 / (1.0 - pow(c->beta1, (double)step)));
  const float c2 = (float)(1.0 / (1.0 - pow(c->beta2, (double)step)));
  const float eps = (float)c->eps;
  const float lrg = (float)cosine_lr(c->lr_grid, c, step), lrm = (float)cosine_lr(c->lr_mlp, c, step);
  for (int64_t i = 0; i < n; ++i) {
    const float gg = g[i];
    const float lr = i >= mlp_offset ? lrm : lrg;
    m[i] = b1 * m[i] + omb1 * gg;
    v[i] = b2 * v[i] + omb2 * (gg * gg);
    const float den = sqrtf(v[i] * c2) + eps;
    p[i] = p[i] - (lr * (m[i] * c1)) / den;
    g[i] = 0.0f;
  }
  return 0;
}
