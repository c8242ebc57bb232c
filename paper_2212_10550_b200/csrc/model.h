// model.h -- device-resident model / pose / occupancy objects behind the C-ABI handles.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <string>
#include <vector>

#include "arfx_internal.h"
#include "host.h"

namespace arfx {

void cuda_check(cudaError_t e, const char* what);
#define ARFX_CUDA(call) ::arfx::cuda_check((call), #call)

template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  bool owned = true;
  unsigned long long* gen = nullptr;  // bumped on every (re)allocation (Workspace::gen)
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (ptr && owned) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
    owned = true;
  }
  void view(T* p, size_t count) {  // non-owning window into another buffer
    release();
    ptr = p;
    n = count;
    owned = false;
  }
  void ensure(size_t count) {  // grow-only, contents not preserved
    if (count <= n) return;
    release();
    if (gen) ++*gen;
    if (count == 0) return;
    ARFX_CUDA(cudaMalloc(&ptr, count * sizeof(T)));
    n = count;
  }
  void alloc(size_t count) {
    release();
    if (gen) ++*gen;
    if (count) ARFX_CUDA(cudaMalloc(&ptr, count * sizeof(T)));
    n = count;
  }
};

// Render / query workspace: compacted posed-sample list, root pool, per-ray ranges.
struct Workspace {
  size_t cap_posed = 0, cap_pool = 0, n_pix = 0;
  DevBuf<double> sx, sy, sz, sdelta;  // posed samples: normalized position, delta
  DevBuf<int32_t> sray;               // pixel index
  DevBuf<int16_t> sidx;               // sample index along the ray
  DevBuf<uint8_t> snroot;             // in-box roots (<= 8)
  DevBuf<int32_t> sbase;              // first pool entry of the sample
  DevBuf<int8_t> ssel;                // selected root slot (-1 none)
  DevBuf<double> px, py, pz;          // root pool (canonical positions)
  DevBuf<int32_t> powner;             // owning sample (-1: value precomputed by deformer)
  DevBuf<float4> pres;                // (density, r, g, b) per pool entry
  DevBuf<int32_t> ray_first, ray_count, row_list;
  DevBuf<double> train_terms;          // fused-loss per-ray terms
  DevBuf<unsigned char> tc_tiles;      // tcgen05 decoder: split-bf16 feature tiles (16 KB / 128 queries)
  DevBuf<double> dens_pts;             // L_density points (SoA)
  DevBuf<uint8_t> dens_empty;          // point lies in an empty occupancy cell
  DevBuf<float> dens_scale;            // w_density / n_empty
  DevBuf<float> train_rgb, train_alpha;  // training outputs when the caller passes none
  DevBuf<unsigned long long> counters;  // [0] posed [1] canonical [2] pool [3] overflow
  DevBuf<int> occ_box;                  // occupied-cell bounding box (march empty-space skip)
  DevBuf<uint32_t> occ_bits;            // occupancy mask packed to bits (march pass 1 reads, L1-resident)
  DevBuf<float> fwd_act;  // training forwards: per pool entry X | H1 | H2 | logits (K8a reuses them)
  // K2 start pipeline (deform_starts.cuh)
  size_t cap_targets = 0, cap_starts = 0;
  DevBuf<uint32_t> smask, scount;  // per target: start mask, start count -> slot base
  DevBuf<StartItem> items;                    // sorted by (bone, cell): target | bone << 26 [| slot << 32]
  DevBuf<uint32_t> keys, unsorted, key_hist;  // counting-sort scratch
  DevBuf<unsigned long long> lb_status;        // single-pass scans: tickets + tile status words
  DevBuf<double4> res4;                        // per start slot: root xyz, residual (-1: no root)
  // training scratch (train.cu)
  DevBuf<double> strans;   // transmittance before each posed sample
  DevBuf<float> pgs, pgc;  // per pool entry: dsigma, dcolor[3]
  DevBuf<uint8_t> pflag;   // per pool entry: query_backward needed
  DevBuf<float> bwd_rec;   // K8a -> K8b: per flagged query, MLP layer inputs and deltas
  DevBuf<int32_t> bwd_list;  // flagged pool entries, compacted
  DevBuf<float> bwd_partial;  // K8b per-block MLP gradient rows
  DevBuf<uint32_t> bwd_own;   // deterministic mode: per-owner flagged count -> list offset
  DevBuf<unsigned long long> bwd_n;
  int last_rows = -1, last_shard = -1, last_nshards = -1, last_w = -1, n_rows = 0;
  // Generation: bumped whenever any buffer above is (re)allocated (or the row list is
  // rewritten). A captured frame graph holds raw pointers into this workspace and refuses to
  // replay once the generation moved (arfx_frame_graph_launch).
  unsigned long long gen = 0;
  Workspace() {
    bind(sx, sy, sz, sdelta, sray, sidx, snroot, sbase, ssel, px, py, pz, powner, pres, ray_first, ray_count,
         row_list, train_terms, tc_tiles, dens_pts, dens_empty, dens_scale, train_rgb, train_alpha, counters,
         occ_box, occ_bits, fwd_act, smask, scount, items, keys, unsorted, key_hist, lb_status, res4, strans, pgs, pgc,
         pflag, bwd_rec, bwd_list, bwd_partial, bwd_own, bwd_n);
  }
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  template <typename... B>
  void bind(B&... b) {
    ((b.gen = &gen), ...);
  }
  void ensure(size_t posed, size_t pix);
  void reserve_worst(size_t targets, size_t n_bones);
  size_t learned_starts = 0;  // raised when a frame overflowed the start slots
  void ensure_starts(size_t targets, size_t nkeys, size_t min_starts = 0);
  void ensure_train();
};

// Optional per-kernel CUDA-event timing on the launching stream (bench / roofline).
struct KernelProfiler {
  bool on = false;
  struct Rec {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> free_events;
  std::vector<std::string> names;
  std::vector<double> ms;
  std::vector<long long> launches;
  cudaEvent_t take();
  void begin(const char* name, cudaStream_t s);
  void end(cudaStream_t s);
  void collect();  // synchronises the recorded events and accumulates
  ~KernelProfiler();
};

struct ModelImpl {
  int device = 0;
  KernelProfiler prof;
  // deterministic work counters (roofline accounting): [0] evals [1] union bones
  // [2] Newton steps [3] starts [4] exact prune tests [5] field queries
  bool stats_on = false;
  DevBuf<unsigned long long> stats;
  bool bwd_tc = true;  // training MLP backward on tcgen05 (arfx_model_set_backward_mode)
  int mlp_mode = 0;  // render decoder: 0 exact f32 SIMT (bit-faithful sums), 1 tcgen05 split-bf16 (3-term,
                     // f32 accumulate), 2 = 1 with fp16 hash-table gathers
  DevBuf<__half2> grid_h2;  // fp16 copy of the hash table (mode 2), refreshed per render
  // deterministic gradients (arfx_model_set_deterministic): K8b/K8c sum fixed-point int64
  // contributions (exact, order-independent); grid_acc is the hash-grid accumulator, kept
  // all-zero between steps (the drain pass takes and clears every touched row)
  bool det = false;
  DevBuf<long long> grid_acc;  // fixed-point hash-grid gradient, one per grid_grad element
  bool acc_pending = false;    // grid_acc holds sums not yet folded into grid_grad
  cudaStream_t stream = nullptr;
  std::vector<HostBone> bones;
  GridCfg grid{};
  std::vector<int> res;
  int mlp_in = 0, mlp_hidden = 0, mlp_hl = 0, mlp_out = 0;
  MlpLayout mlp{};
  int skin_res[3] = {0, 0, 0};
  HostBox skin_box{}, canon{}, norm{};
  InverseOpts inv{20, 1e-5, 1e-3};
  size_t n_grid = 0, n_mlp = 0, n_skin = 0;
  // Flat parameter / gradient / Adam-moment vectors [grid | pad | mlp | pad] (n_flat floats):
  // one buffer each so data-parallel training reduce-scatters / all-gathers them in one call;
  // grid_* and mlp_* are non-owning views into them.
  DevBuf<float> flat_params, flat_grads, adam_m, adam_v;
  size_t n_flat = 0, mlp_off = 0;
  DevBuf<float> grid_params, mlp_params, grid_grad, mlp_grad;
  DevBuf<double> skin;
  DevBuf<uint32_t> cell_mask, cell_off;
  DevBuf<uint2> cell_mo;  // (cell_mask, cell_off) interleaved for the Newton kernel
  DevBuf<PoseCtx> grid_ctxs;  // update_training_grid: the pose list on the device
  DevBuf<double> cell_vals;
  int max_union = 1;  // widest per-cell bone union (sizes the Newton kernel's scratch)
  FieldView fv{};
  SkinView sv{};
  // Workspaces: ws() is the one the launch helpers use; a second one lets the L_density
  // forward run on the side stream concurrently with the train step (WorkspaceScope).
  // ws_t0 / ws_alt: the two train slots of the pipelined trainer (a slot's forward state lives
  // across calls, so nothing else may use them); ws_main serves every other call.
  Workspace ws_main, ws_side, ws_t0, ws_alt;
  Workspace* ws_cur = &ws_main;
  Workspace& ws() { return *ws_cur; }
  cudaStream_t side = nullptr;  // lazily created non-blocking stream
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_pipe_fork = nullptr, ev_pipe_join = nullptr;  // arfx_render_model_pipelined_async
  cudaStream_t aux = nullptr;   // K8b/K8d next to K8c (field_backward_pool)
  // arfx_render_model_async: two device image slots; their D2H copies run on copy_stream
  // while the next frame renders
  struct AsyncSlot {
    DevBuf<float> rgb, alpha;
    DevBuf<unsigned long long> counters;
    cudaEvent_t rendered = nullptr, copied = nullptr;
  } async_slot[2];
  int async_next = 0;
  // arfx_render_model_pipelined_async: captured pipelined frames (grid of the next pose beside
  // the render into an async slot), keyed by (handles, camera, options, shard, slot, stream)
  struct PipeGraphEntry {
    std::string key;
    void* graph = nullptr;  // arfx_frame_graph_s
  };
  std::vector<PipeGraphEntry> pipe_graphs;
  cudaStream_t copy_stream = nullptr;
  // arfx_model_set_param_fence: kernels that read the parameters or write the gradients
  // wait for this event first (an optimizer running on another stream)
  cudaEvent_t param_fence = nullptr;
  void wait_params(cudaStream_t s) const {
    if (param_fence) ARFX_CUDA(cudaStreamWaitEvent(s, param_fence, 0));
  }
  cudaEvent_t ev_aux_fork = nullptr, ev_aux_join = nullptr;
  std::vector<uint8_t> overflow_note;
  ~ModelImpl();
  void refresh_views();
};

struct PoseImpl {
  ModelImpl* model = nullptr;
  PoseCtx host{};
  DevBuf<PoseCtx> dev;
  // arfx_pose_update_async: pinned staging ring (the H2D copy never waits on the stream)
  static constexpr int kRing = 4;
  PoseCtx* ring = nullptr;
  cudaEvent_t ring_ev[kRing] = {};
  int ring_next = 0;
  ~PoseImpl();
};

struct OccImpl {
  int device = 0;
  DevBuf<float> saved;  // update_training_grid: values before the update (overflow rerun)
  int res = 64;
  HostBox box{};
  double threshold = 0.0;
  int dilation = 1;
  DevBuf<float> values;
  DevBuf<uint8_t> mask;
  OccView view() const;
};

// model.cu
void build_skinning_grid_dev(ModelImpl& m, double blend_factor);  // R/skinning.hpp:61-111
void build_cell_table(ModelImpl& m);
void init_params_dev(ModelImpl& m, uint64_t seed);  // R/hash_grid.hpp:66-73, R/mlp.hpp:50-58

// render.cu
void render_frame(ModelImpl& m, PoseImpl& p, const HostCamera& cam, OccImpl* occ, int N,
                  bool stratified, double eps, uint64_t seed, uint64_t frame, int shard,
                  int nshards, float* d_rgb, float* d_alpha, unsigned long long* d_counters,
                  cudaStream_t s);
void inference_grid(ModelImpl& m, PoseImpl& p, OccImpl& g, unsigned long long* d_counters,
                    cudaStream_t s);
void inference_grid_shard(ModelImpl& m, PoseImpl& p, OccImpl& g, int shard, int n_shards,
                          unsigned long long* d_counters, cudaStream_t s);
void occ_unshard(OccImpl& g, int n_shards, cudaStream_t s);
void training_grid_update(ModelImpl& m, const std::vector<PoseImpl*>& poses, double decay,
                          uint64_t seed, uint64_t step, OccImpl& g, unsigned long long* d_counters,
                          cudaStream_t s);
void occ_rebuild(OccImpl& g, cudaStream_t s);
void occ_query_batch(OccImpl& g, const double* d_pts, int64_t n, uint8_t* d_out, cudaStream_t s);
void inverse_lbs_batch(ModelImpl& m, const PoseCtx* d_ctx, const double* d_pts, int64_t n,
                       int32_t* d_counts, double* d_roots, double* d_res, cudaStream_t s);
void posed_query_batch(ModelImpl& m, PoseImpl& p, const double* d_pts, int64_t n, float* d_dens,
                       float* d_col, double* d_canon, uint8_t* d_has, unsigned long long* d_counters,
                       cudaStream_t s);
void field_query_batch(ModelImpl& m, const double* d_pts, int64_t n, float4* d_out, int* d_domain_err,
                       cudaStream_t s);
void hash_encode_batch(ModelImpl& m, const double* d_pts, int64_t n, float* d_feats,
                       int* d_domain_err, cudaStream_t s);
void skin_weights_batch(ModelImpl& m, const double* d_pts, int64_t n, double* d_w, cudaStream_t s);

void train_forward(ModelImpl& m, PoseImpl& p, const HostCamera& cam, OccImpl* occ, int N, bool stratified,
                   uint64_t seed, uint64_t frame, long long n_rays, const int32_t* d_px, const int32_t* d_py,
                   cudaStream_t s);

// train.cu
// fused-loss targets for train_composite (losses.cuh); device arrays
struct LossTargets {
  const float* gt_rgb;    // [n][3], or a [gt_h][gt_w][3] frame when gt_w > 0
  const float* gt_alpha;  // [n], or [gt_h][gt_w]
  double w_rgb, w_alpha, w_hard, w_density, huber_delta;
  double* ray_terms;      // [n][3] out
  long long gt_w = 0, gt_h = 0;
  const int32_t *px = nullptr, *py = nullptr;  // ray pixels (frame targets)
};
void loss_reduce(const double* d_terms, long long n, const LossTargets& lt, double* d_out4, cudaStream_t s);
void ray_losses(long long n, const float* d_rgb, const float* d_alpha, const LossTargets& lt, float* d_grad_rgb,
                float* d_grad_alpha, cudaStream_t s);
// Raises `kernel`'s dynamic shared-memory limit on the current device to at least `bytes`
// (per device and kernel, thread-safe; a no-op when already high enough).
void ensure_dyn_smem(const void* kernel, size_t bytes);

// L_density (render.cu): forward (points + posed query), backward (loss + K8)
void density_forward(ModelImpl& m, PoseImpl& p, OccImpl& g, long long n, uint64_t seed, uint64_t step,
                     cudaStream_t s);
void density_backward(ModelImpl& m, long long n, double w_density, double* d_out2, cudaStream_t s);
void density_flags(ModelImpl& m, long long n, double w_density, double* d_out2, cudaStream_t s);
void density_backward_field(ModelImpl& m, long long n, cudaStream_t s);
void launch_train_rays(uint64_t seed, uint64_t step, uint64_t rank, long long n, int W, int H, int32_t* px, int32_t* py,
                       cudaStream_t s);
// optim.cu: Adam over the flat parameter vector
struct AdamCfg {
  double lr_grid, lr_mlp, beta1, beta2, eps;
  long long total_steps;
  double final_lr_factor;
};
double cosine_lr(double lr0, const AdamCfg& c, long long step);
void adam_step(ModelImpl& m, const AdamCfg& c, long long step, long long begin, long long end, cudaStream_t s,
               const double* guard = nullptr, int n_guard = 0, int* bad = nullptr);
void train_composite(ModelImpl& m, long long n_rays, int N, double eps, const float* d_dC, const float* d_dA,
                     float* d_rgb, float* d_alpha, cudaStream_t s, const LossTargets* lt = nullptr);
// Points the launch helpers at another workspace for a scope (host-side; the kernels
// enqueued inside capture that workspace's buffers).
struct WorkspaceScope {
  ModelImpl& m;
  Workspace* prev;
  WorkspaceScope(ModelImpl& mm, Workspace& w) : m(mm), prev(mm.ws_cur) { m.ws_cur = &w; }
  ~WorkspaceScope() { m.ws_cur = prev; }
  WorkspaceScope(const WorkspaceScope&) = delete;
  WorkspaceScope& operator=(const WorkspaceScope&) = delete;
};

// Owner order of the flagged pool entries (deterministic mode): targets [first[o],
// first[o]+count[o]) per owner o (nullptr: target o), or the pool entries themselves.
struct BwdOwners {
  long long n_owner;
  const int32_t *first, *count;
  bool pool_is_target;
};
// Saved decoder activations (training forwards through the team decoder, pool <= 65536
// queries): per pool entry X[32] | H1[64] | H2[64] | logits[4], bit-identical to a recompute.
constexpr int kActStride = 164;
#ifndef ARFX_SAVE_ACT
#define ARFX_SAVE_ACT 1  // 0: K8a always recomputes the forward (reference build for tests)
#endif
constexpr long long kTeamMaxQueries = 65536;
void field_backward_pool(ModelImpl& m, const unsigned long long* d_n, long long cap, const uint8_t* flag,
                         const float* gs, const float* gc, cudaStream_t s, const BwdOwners* own,
                         const float* act = nullptr);
void flush_grad_acc(ModelImpl& m, cudaStream_t s);
// roofline accounting: m.stats[i] += *d_src + add (when arfx_stats_enable is on)
void stat_add(ModelImpl& m, int i, const unsigned long long* d_src, unsigned long long add, cudaStream_t s);  // deterministic mode: grid_acc -> grid_grad

// field_tc.cu
bool field_tc_supported(const FieldView& F);
void launch_field_tc(ModelImpl& m, cudaStream_t s, long long n_hint);

// peaks.cu
void measure_pipe_peaks(double* fp64_tflops, double* fp32_tflops);

// composite.cu
void composite_explicit(int n_rays, const int64_t* d_off, const double* d_delta, const uint8_t* d_skip,
                        const float* d_dens, const float* d_col, double eps, double* d_c3, double* d_a,
                        int32_t* d_term, cudaStream_t s);
void composite_backward_explicit(int n_rays, const int64_t* d_off, const double* d_delta,
                                 const uint8_t* d_skip, const float* d_dens, const float* d_col,
                                 double eps, const double* d_dC3, const double* d_dA, double* d_trans,
                                 double* d_sigma, double* d_c3, cudaStream_t s);

// scene.cu: analytic ground truth (R/scene.hpp)
void figure_query_batch(const FigureView& F, const double* d_pts, long long n, double* d_dens, double* d_col,
                        cudaStream_t s);
void figure_render(const FigureView& F, const HostCamera& cam, const double* w2n12, const double* nlo,
                   const double* nhi, int N, bool stratified, double eps, uint64_t seed, uint64_t frame, long long n,
                   const int32_t* d_px, const int32_t* d_py, float* d_rgb, float* d_alpha, uint8_t* d_mask,
                   cudaStream_t s);


// Resident blocks per SM of a kernel at a launch shape (cudaOccupancy..., cached per device:
// the launch helpers run on every step, the occupancy calculation is host work).
int blocks_per_sm(const void* kernel, int threads, size_t smem);
int device_sm_count();

// Grid of a grid-stride kernel: at most one wave of resident blocks, so the static partition
// of the items never leaves a fractional last wave running alone.
template <class Kern>
int resident_grid(Kern kernel, int threads, size_t smem, long long n_items) {
  const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kernel), threads, smem);
  const long long want = (n_items + threads - 1) / threads;
  const long long cap = static_cast<long long>(device_sm_count()) * per_sm;
  return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace arfx
