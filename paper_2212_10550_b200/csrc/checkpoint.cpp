// checkpoint.cpp -- the SPEC's checkpoint file (
// SURVEY.md §8f row 3): versioned binary of configs, grid, MLP, skinning, occupancy and
// optimizer state, written / read through the public C-ABI (host code, g++). Every field
// is serialised explicitly in little-endian order (no struct memcpy), and the file ends
// with an FNV-1a 64 checksum of all preceding bytes. Layout (version 1):
//   "ARFXCKPT" u32 version u32 flags(bit0 occupancy, bit1 optimizer)
//   skeleton: i32 n, n x (i32 parent, f64 head[3], f64 tail[3], f64 radius)
//   grid cfg: i32 levels, F, log2T, nmin, nmax, f64 box_lo[3], box_hi[3]
//   mlp cfg: i32 in, hidden, layers, out
//   i32 skin_res[3], f64 skin_lo[3], skin_hi[3], canonical_lo[3], canonical_hi[3],
//   normalized_lo[3], normalized_hi[3]; i32 max_iterations, f64 tolerance, dedup_radius
//   u64 n_grid, f32[n_grid]; u64 n_mlp, f32[n_mlp]; u64 n_skin, f64[n_skin]
//   [occupancy] i32 res, f64 lo[3], hi[3], f64 threshold, i32 dilation, f32[res^3], u8[res^3]
//   [optimizer] i64 step, u64 n_flat, f32[n_flat] m, f32[n_flat] v
//   u64 fnv1a64
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/arfx.h"
#include "host.h"

namespace {

constexpr char kMagic[8] = {'A', 'R', 'F', 'X', 'C', 'K', 'P', 'T'};
constexpr uint32_t kVersion = 1;

uint64_t fnv1a(const uint8_t* p, size_t n) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

struct Writer {
  std::vector<uint8_t> b;
  void raw(const void* p, size_t n) {
    const uint8_t* c = static_cast<const uint8_t*>(p);
    b.insert(b.end(), c, c + n);
  }
  template <typename T>
  void put(T v) {
    raw(&v, sizeof(T));  // x86-64 / aarch64: little-endian
  }
  template <typename T>
  void arr(const T* p, size_t n) {
    put<uint64_t>(n);
    raw(p, n * sizeof(T));
  }
};

struct Reader {
  const std::vector<uint8_t>& b;
  size_t o = 0;
  void raw(void* p, size_t n) {
    if (n > b.size() - o) throw arfx::DataError("checkpoint: truncated file");
    std::memcpy(p, b.data() + o, n);
    o += n;
  }
  template <typename T>
  T get() {
    T v;
    raw(&v, sizeof(T));
    return v;
  }
  template <typename T>
  std::vector<T> arr(size_t expect) {
    const uint64_t n = get<uint64_t>();
    if (n != expect) throw arfx::DataError("checkpoint: array length does not match the configuration");
    std::vector<T> v(n);
    raw(v.data(), n * sizeof(T));
    return v;
  }
};

struct Status {
  int code;
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return ARFX_OK;
  } catch (const arfx::DataError& e) {
    arfx::set_error_message(e.what());
    return ARFX_ERR_DATA;
  } catch (const std::invalid_argument& e) {
    arfx::set_error_message(e.what());
    return ARFX_ERR_INVALID_ARGUMENT;
  } catch (const Status& s) {
    return s.code;
  } catch (const std::exception& e) {
    arfx::set_error_message(e.what());
    return ARFX_ERR_RUNTIME;
  }
}

void pass(int code) {
  if (code != ARFX_OK) throw Status{code};  // keep the callee's status and message
}

void put3(Writer& w, const double* v) {
  for (int a = 0; a < 3; ++a) w.put<double>(v[a]);
}
void get3(Reader& r, double* v) {
  for (int a = 0; a < 3; ++a) v[a] = r.get<double>();
}

}  // namespace

extern "C" {

int arfx_checkpoint_save(const char* path, arfx_model m, arfx_occ_grid occ, int64_t step, int with_optimizer) {
  return guarded([&] {
    if (!path || !m) throw std::invalid_argument("checkpoint_save: null argument");
    arfx_model_desc d;
    pass(arfx_model_describe(m, &d));
    std::vector<float> gp(d.n_grid_params), mp(d.n_mlp_params);
    std::vector<double> sw(d.n_skin_weights);
    pass(arfx_model_get_params(m, gp.data(), mp.data(), sw.data()));
    Writer w;
    w.raw(kMagic, 8);
    w.put<uint32_t>(kVersion);
    w.put<uint32_t>((occ ? 1u : 0u) | (with_optimizer ? 2u : 0u));
    w.put<int32_t>(d.skeleton.n_bones);
    for (int i = 0; i < d.skeleton.n_bones; ++i) {
      w.put<int32_t>(d.skeleton.parent[i]);
      put3(w, d.skeleton.head[i]);
      put3(w, d.skeleton.tail[i]);
      w.put<double>(d.skeleton.radius[i]);
    }
    const arfx_grid_config& g = d.grid;
    for (int v : {g.levels, g.features_per_level, g.table_size_log2, g.base_resolution, g.max_resolution})
      w.put<int32_t>(v);
    put3(w, g.box_lo);
    put3(w, g.box_hi);
    for (int v : {d.mlp.input_dim, d.mlp.hidden_dim, d.mlp.hidden_layers, d.mlp.output_dim}) w.put<int32_t>(v);
    for (int a = 0; a < 3; ++a) w.put<int32_t>(d.skin_res[a]);
    put3(w, d.skin_lo);
    put3(w, d.skin_hi);
    put3(w, d.canonical_lo);
    put3(w, d.canonical_hi);
    put3(w, d.normalized_lo);
    put3(w, d.normalized_hi);
    w.put<int32_t>(d.inverse.max_iterations);
    w.put<double>(d.inverse.tolerance);
    w.put<double>(d.inverse.dedup_radius);
    w.arr(gp.data(), gp.size());
    w.arr(mp.data(), mp.size());
    w.arr(sw.data(), sw.size());
    if (occ) {
      int res[3];
      double lo[3], hi[3], thr;
      int dil;
      pass(arfx_occ_info(occ, res, lo, hi, &thr, &dil));
      const size_t n = static_cast<size_t>(res[0]) * res[1] * res[2];
      std::vector<float> v(n);
      std::vector<uint8_t> mk(n);
      pass(arfx_occ_download(occ, v.data(), mk.data()));
      w.put<int32_t>(res[0]);
      put3(w, lo);
      put3(w, hi);
      w.put<double>(thr);
      w.put<int32_t>(dil);
      w.raw(v.data(), n * sizeof(float));
      w.raw(mk.data(), n);
    }
    if (with_optimizer) {
      int64_t n_flat = 0, off = 0;
      pass(arfx_model_flat(m, nullptr, nullptr, nullptr, nullptr, &n_flat, &off));
      std::vector<float> am(static_cast<size_t>(n_flat)), av(static_cast<size_t>(n_flat));
      pass(arfx_model_get_adam(m, am.data(), av.data()));
      w.put<int64_t>(step);
      w.arr(am.data(), am.size());
      w.raw(av.data(), av.size() * sizeof(float));
    }
    w.put<uint64_t>(fnv1a(w.b.data(), w.b.size()));
    FILE* f = std::fopen(path, "wb");
    if (!f) throw std::invalid_argument(std::string("checkpoint_save: cannot open ") + path);
    const size_t wr = std::fwrite(w.b.data(), 1, w.b.size(), f);
    const int cl = std::fclose(f);
    if (wr != w.b.size() || cl != 0) throw std::runtime_error("checkpoint_save: write failed");
  });
}

int arfx_checkpoint_load(const char* path, arfx_model* m_out, arfx_occ_grid* occ_out, int64_t* step_out) {
  return guarded([&] {
    if (!path || !m_out) throw std::invalid_argument("checkpoint_load: null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::invalid_argument(std::string("checkpoint_load: cannot open ") + path);
    std::vector<uint8_t> b;
    uint8_t buf[1 << 16];
    size_t k;
    while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) b.insert(b.end(), buf, buf + k);
    std::fclose(f);
    if (b.size() < 8 + 8 + 8) throw arfx::DataError("checkpoint: truncated file");
    if (std::memcmp(b.data(), kMagic, 8) != 0) throw arfx::DataError("checkpoint: bad magic");
    uint64_t stored;
    std::memcpy(&stored, b.data() + b.size() - 8, 8);
    if (fnv1a(b.data(), b.size() - 8) != stored) throw arfx::DataError("checkpoint: checksum mismatch");
    const std::vector<uint8_t> body(b.begin(), b.end() - 8);
    Reader r{body};
    char magic[8];
    r.raw(magic, 8);
    const uint32_t ver = r.get<uint32_t>();
    if (ver != kVersion) throw arfx::DataError("checkpoint: unsupported version " + std::to_string(ver));
    const uint32_t flags = r.get<uint32_t>();
    arfx_model_desc d;
    std::memset(&d, 0, sizeof d);
    d.skeleton.n_bones = r.get<int32_t>();
    if (d.skeleton.n_bones < 1 || d.skeleton.n_bones > ARFX_MAX_BONES)
      throw arfx::DataError("checkpoint: bad bone count");
    for (int i = 0; i < d.skeleton.n_bones; ++i) {
      d.skeleton.parent[i] = r.get<int32_t>();
      get3(r, d.skeleton.head[i]);
      get3(r, d.skeleton.tail[i]);
      d.skeleton.radius[i] = r.get<double>();
    }
    arfx_grid_config& g = d.grid;
    g.levels = r.get<int32_t>();
    g.features_per_level = r.get<int32_t>();
    g.table_size_log2 = r.get<int32_t>();
    g.base_resolution = r.get<int32_t>();
    g.max_resolution = r.get<int32_t>();
    get3(r, g.box_lo);
    get3(r, g.box_hi);
    d.mlp.input_dim = r.get<int32_t>();
    d.mlp.hidden_dim = r.get<int32_t>();
    d.mlp.hidden_layers = r.get<int32_t>();
    d.mlp.output_dim = r.get<int32_t>();
    for (int a = 0; a < 3; ++a) d.skin_res[a] = r.get<int32_t>();
    get3(r, d.skin_lo);
    get3(r, d.skin_hi);
    get3(r, d.canonical_lo);
    get3(r, d.canonical_hi);
    get3(r, d.normalized_lo);
    get3(r, d.normalized_hi);
    d.inverse.max_iterations = r.get<int32_t>();
    d.inverse.tolerance = r.get<double>();
    d.inverse.dedup_radius = r.get<double>();
    size_t ng = 0, nm = 0, ns = 0;
    pass(arfx_model_sizes(&d.skeleton, &d.grid, &d.mlp, d.skin_res, &ng, &nm, &ns));
    d.n_grid_params = ng;
    d.n_mlp_params = nm;
    d.n_skin_weights = ns;
    const std::vector<float> gp = r.arr<float>(ng);
    const std::vector<float> mp = r.arr<float>(nm);
    const std::vector<double> sw = r.arr<double>(ns);
    arfx_model m = nullptr;
    pass(arfx_model_create(&d, gp.data(), mp.data(), sw.data(), &m));
    arfx_occ_grid og = nullptr;
    try {
      if (flags & 1u) {
        const int res = r.get<int32_t>();
        double lo[3], hi[3];
        get3(r, lo);
        get3(r, hi);
        const double thr = r.get<double>();
        const int dil = r.get<int32_t>();
        if (res < 1 || res > 1024) throw arfx::DataError("checkpoint: bad occupancy resolution");
        const size_t n = static_cast<size_t>(res) * res * res;
        std::vector<float> v(n);
        std::vector<uint8_t> mk(n);
        r.raw(v.data(), n * sizeof(float));
        r.raw(mk.data(), n);
        if (occ_out) {
          pass(arfx_occ_create_raw(lo, hi, res, thr, dil, &og));
          pass(arfx_occ_upload(og, v.data(), mk.data()));
        }
      }
      int64_t step = 0;
      if (flags & 2u) {
        step = r.get<int64_t>();
        int64_t n_flat = 0, off = 0;
        pass(arfx_model_flat(m, nullptr, nullptr, nullptr, nullptr, &n_flat, &off));
        const std::vector<float> am = r.arr<float>(static_cast<size_t>(n_flat));
        std::vector<float> av(static_cast<size_t>(n_flat));
        r.raw(av.data(), av.size() * sizeof(float));
        pass(arfx_model_set_adam(m, am.data(), av.data()));
      }
      if (r.o != body.size()) throw arfx::DataError("checkpoint: trailing bytes");
      *m_out = m;
      if (occ_out) *occ_out = og;
      if (step_out) *step_out = step;
    } catch (...) {
      if (og) arfx_occ_destroy(og);
      arfx_model_destroy(m);
      throw;
    }
  });
}

}  // extern "C"
