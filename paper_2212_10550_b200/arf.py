"""Python mirror of the reference library's model-bound API (namespace `arf`,
/root/reference/proj/include/arf, cited R/...), backed by libarfx.so on the GPU.

Same names, argument meanings and error behaviour as the reference:
  build_model                  R/model.hpp:68-80
  render_model                 R/model.hpp:118-135     -> RenderImages
  build_model_inference_grid   R/model.hpp:138-148     -> OccupancyGrid
  update_training_grid         R/occupancy.hpp:155-171 (bound to PosedModelView)
  pose_from_joint_rotations    R/skeleton.hpp:93-110
  Camera.look_at               R/camera.hpp:31-48
  inverse_lbs / posed_query / CanonicalField.query / HashGrid.encode / skinning_weights
Exceptions: ValueError subclasses for std::invalid_argument / std::domain_error,
NumericError, DataError; NoDevice when there is no GPU (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib as L
from ._lib import call, ptr

# ----------------------------------------------------------------------------- values


@dataclass
class Bone:  # R/skeleton.hpp:9-14
    parent: int
    head: tuple
    tail: tuple
    radius: float = 0.05


@dataclass
class Skeleton:  # R/skeleton.hpp:16-64
    bones: list

    def bone_count(self) -> int:
        return len(self.bones)

    def to_c(self) -> L.ArfxSkeleton:
        s = L.ArfxSkeleton()
        if len(self.bones) > L.MAX_BONES:
            raise L.InvalidArgument(1, "pose context: too many bones")
        s.n_bones = len(self.bones)
        for i, b in enumerate(self.bones):
            s.parent[i] = b.parent
            for a in range(3):
                s.head[i][a] = float(b.head[a])
                s.tail[i][a] = float(b.tail[a])
            s.radius[i] = float(b.radius)
        return s


@dataclass
class Aabb:
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)


@dataclass
class HashGridConfig:  # R/hash_grid.hpp:12-32
    levels: int = 8
    features_per_level: int = 2
    table_size_log2: int = 16
    base_resolution: int = 16
    max_resolution: int = 256
    bounding_box: Aabb = field(default_factory=Aabb)

    def feature_dim(self) -> int:
        return self.levels * self.features_per_level

    def to_c(self) -> L.ArfxGridConfig:
        g = L.ArfxGridConfig()
        g.levels, g.features_per_level, g.table_size_log2 = self.levels, self.features_per_level, self.table_size_log2
        g.base_resolution, g.max_resolution = self.base_resolution, self.max_resolution
        for a in range(3):
            g.box_lo[a] = self.bounding_box.lo[a]
            g.box_hi[a] = self.bounding_box.hi[a]
        return g


@dataclass
class MlpConfig:  # R/mlp.hpp:11-23
    input_dim: int = 16
    hidden_dim: int = 64
    hidden_layers: int = 2
    output_dim: int = 4

    def to_c(self) -> L.ArfxMlpConfig:
        return L.ArfxMlpConfig(self.input_dim, self.hidden_dim, self.hidden_layers, self.output_dim)


@dataclass
class OccupancyConfig:  # R/occupancy.hpp:13-28
    resolution: int = 64
    alpha_threshold: float = 0.01
    dilation: int = 1
    decay: float = 0.95
    update_interval: int = 16

    def to_c(self) -> L.ArfxOccConfig:
        return L.ArfxOccConfig(self.resolution, self.alpha_threshold, self.dilation, self.decay, self.update_interval)


@dataclass
class RenderOptions:  # R/render.hpp:159-165
    samples_per_ray: int = 128
    stratified: bool = False
    epsilon_terminate: float = 1e-3
    seed: int = 0
    frame_id: int = 0

    def to_c(self) -> L.ArfxRenderOptions:
        return L.ArfxRenderOptions(self.samples_per_ray, int(bool(self.stratified)), self.epsilon_terminate,
                                   self.seed & (2**64 - 1), self.frame_id & (2**64 - 1))


@dataclass
class InverseLbsOptions:  # R/articulation.hpp:84-88
    max_iterations: int = 20
    tolerance: float = 1e-5
    dedup_radius: float = 1e-3


def rigid(R=None, t=None) -> np.ndarray:
    """Rigidd as 12 doubles: rotation row-major then translation."""
    out = np.zeros(12, np.float64)
    out[:9] = np.eye(3).ravel() if R is None else np.asarray(R, np.float64).ravel()
    if t is not None:
        out[9:] = np.asarray(t, np.float64)
    return out


@dataclass
class SkeletonPose:  # R/skeleton.hpp:69-88
    bone_transforms: np.ndarray  # (n_bones, 12)
    global_transform: np.ndarray = field(default_factory=rigid)

    def __post_init__(self):
        self.bone_transforms = np.ascontiguousarray(self.bone_transforms, np.float64).reshape(-1, 12)
        self.global_transform = np.ascontiguousarray(self.global_transform, np.float64).reshape(12)

    @staticmethod
    def identity(n_bones: int) -> "SkeletonPose":
        return SkeletonPose(np.tile(rigid(), (n_bones, 1)))

    def bone_count(self) -> int:
        return int(self.bone_transforms.shape[0])


@dataclass
class Camera:  # R/camera.hpp:9-49
    fx: float = 128.0
    fy: float = 128.0
    cx: float = 64.0
    cy: float = 64.0
    width: int = 128
    height: int = 128
    extrinsic: np.ndarray = field(default_factory=rigid)

    def to_c(self) -> L.ArfxCamera:
        c = L.ArfxCamera()
        c.fx, c.fy, c.cx, c.cy, c.width, c.height = self.fx, self.fy, self.cx, self.cy, self.width, self.height
        for k in range(12):
            c.extrinsic[k] = float(self.extrinsic[k])
        return c

    @staticmethod
    def look_at(eye, target, up, focal: float, width: int, height: int) -> "Camera":
        out = L.ArfxCamera()
        e = np.asarray(eye, np.float64)
        t = np.asarray(target, np.float64)
        u = np.asarray(up, np.float64)
        call("arfx_camera_look_at", ptr(e, C.c_double), ptr(t, C.c_double), ptr(u, C.c_double), focal, width,
             height, C.byref(out))
        return Camera(out.fx, out.fy, out.cx, out.cy, out.width, out.height, np.array(out.extrinsic[:], np.float64))


def pose_from_joint_rotations(skel: Skeleton, joint_rotations, global_transform=None) -> SkeletonPose:
    rot = np.ascontiguousarray(np.asarray(joint_rotations, np.float64).reshape(-1, 9))
    g = rigid() if global_transform is None else np.ascontiguousarray(global_transform, np.float64).reshape(12)
    if rot.shape[0] != skel.bone_count():
        raise L.InvalidArgument(1, "pose_from_joint_rotations: rotation count mismatch")
    out = np.zeros((skel.bone_count(), 12), np.float64)
    call("arfx_pose_from_joint_rotations", C.byref(skel.to_c()), ptr(rot, C.c_double), ptr(g, C.c_double),
         ptr(out, C.c_double))
    return SkeletonPose(out, g.copy())


def level_resolutions(cfg: HashGridConfig) -> list:
    out = np.zeros(max(cfg.levels, 1), np.int32)
    call("arfx_level_resolutions", C.byref(cfg.to_c()), ptr(out, C.c_int32))
    return out.tolist()


@dataclass
class RenderImages:  # R/render.hpp:167-171
    width: int
    height: int
    rgb: np.ndarray    # (H, W, 3) f32
    alpha: np.ndarray  # (H, W) f32


@dataclass
class QueryCounters:  # R/model.hpp:11-23
    posed_queries: int = 0
    canonical_queries: int = 0


# ----------------------------------------------------------------------------- device objects


class Model:
    """Device-resident arf::Model<float> (R/model.hpp:28-57)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        d = L.ArfxModelDesc()
        call("arfx_model_describe", self._h, C.byref(d))
        self.desc = d
        self.counters = QueryCounters()

    # -- reference-layout accessors
    @property
    def n_bones(self) -> int:
        return self.desc.skeleton.n_bones

    @property
    def canonical_box(self) -> Aabb:
        return Aabb(tuple(self.desc.canonical_lo), tuple(self.desc.canonical_hi))

    @property
    def normalized_box(self) -> Aabb:
        return Aabb(tuple(self.desc.normalized_lo), tuple(self.desc.normalized_hi))

    def params(self):
        g = np.empty(self.desc.n_grid_params, np.float32)
        m = np.empty(self.desc.n_mlp_params, np.float32)
        s = np.empty(self.desc.n_skin_weights, np.float64)
        call("arfx_model_get_params", self._h, ptr(g, C.c_float), ptr(m, C.c_float), ptr(s, C.c_double))
        return g, m, s

    def set_params(self, grid=None, mlp=None):
        g = None if grid is None else np.ascontiguousarray(grid, np.float32)
        m = None if mlp is None else np.ascontiguousarray(mlp, np.float32)
        call("arfx_model_set_params", self._h, ptr(g, C.c_float), ptr(m, C.c_float))

    def set_mlp_mode(self, mode: str) -> None:
        """'exact' (f32 SIMT, the reference's summation order; default) or 'tcgen05'
        (tensor cores, split-bf16 operands with f32 accumulation; stated tolerance 1e-3
        relative on rendered RGB); 'tcgen05_fp16' additionally gathers the hash table in fp16.
        Render only."""
        call("arfx_model_set_mlp_mode", self._h, {"exact": 0, "tcgen05": 1, "tcgen05_fp16": 2}[mode])

    def set_backward_mode(self, mode: str) -> None:
        """Training MLP backward: 'tcgen05' (default; split-bf16 tensor-core dX / dW with f32
        accumulation) or 'simt' (f32, the reference's summation order)."""
        call("arfx_model_set_backward_mode", self._h, {"simt": 0, "tcgen05": 1}[mode])

    def set_deterministic(self, on: bool = True) -> None:
        """Bit-reproducible gradients (arfx_model_set_deterministic): owner-ordered backward
        lists and fixed-point int64 hash-grid sums, so repeated train / density steps on the
        same inputs give identical gradients, Adam states and parameters."""
        call("arfx_model_set_deterministic", self._h, 1 if on else 0)

    def flush_grads(self, stream=None) -> None:
        """Deterministic mode: fold pending hash-grid sums into the gradient array (needed
        before reading it through device pointers, e.g. a data-parallel reduce-scatter)."""
        call("arfx_model_flush_grads", self._h, stream)

    def set_param_fence(self, event) -> None:
        """cudaEvent_t handle (e.g. torch.cuda.Event().cuda_event) that parameter-reading /
        gradient-writing kernels wait on; None clears (arfx_model_set_param_fence)."""
        call("arfx_model_set_param_fence", self._h, event)

    def zero_grad(self):
        call("arfx_model_zero_grad", self._h, None)

    def grads(self):
        g = np.empty(self.desc.n_grid_params, np.float32)
        m = np.empty(self.desc.n_mlp_params, np.float32)
        call("arfx_model_get_grads", self._h, ptr(g, C.c_float), ptr(m, C.c_float))
        return g, m

    def device_arrays(self):
        ps = [C.c_void_p() for _ in range(4)]
        call("arfx_model_device_arrays", self._h, *[C.byref(p) for p in ps])
        return [p.value for p in ps]

    def flat(self) -> dict:
        """Flat device vectors [grid | pad | mlp | pad]: pointers to params, grads, Adam m, v,
        their length n_flat and the MLP offset (arfx_model_flat)."""
        ps = [C.c_void_p() for _ in range(4)]
        n, off = C.c_int64(), C.c_int64()
        call("arfx_model_flat", self._h, *[C.byref(p) for p in ps], C.byref(n), C.byref(off))
        return {"params": ps[0].value, "grads": ps[1].value, "adam_m": ps[2].value, "adam_v": ps[3].value,
                "n_flat": n.value, "mlp_offset": off.value}

    def adam_step(self, cfg: "AdamConfig", step: int, begin: int = 0, end: int = -1, stream=None,
                  guard=None) -> None:
        """One Adam step (zero-grad fused) over flat indices [begin, end) (arfx_adam_step).
        guard = (loss row device pointer, n values, device int flag pointer): the step is
        skipped on the device if the loss is non-finite (arfx_adam_step_guarded)."""
        if guard is None:
            call("arfx_adam_step", self._h, C.byref(cfg.to_c()), step, begin, end, stream)
        else:
            d_loss, n, d_bad = guard
            call("arfx_adam_step_guarded", self._h, C.byref(cfg.to_c()), step, begin, end, d_loss, n, d_bad,
                 stream)

    def adam_state(self):
        n = self.flat()["n_flat"]
        m = np.zeros(n, np.float32)
        v = np.zeros(n, np.float32)
        call("arfx_model_get_adam", self._h, ptr(m, C.c_float), ptr(v, C.c_float))
        return m, v

    def set_adam_state(self, m, v) -> None:
        m = np.ascontiguousarray(m, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        call("arfx_model_set_adam", self._h, ptr(m, C.c_float), ptr(v, C.c_float))

    def close(self):
        if self._h:
            L.lib().arfx_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- batched queries
    def skinning_weights(self, pts) -> np.ndarray:
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        w = np.empty((p.shape[0], self.n_bones), np.float64)
        call("arfx_skinning_weights", self._h, ptr(p, C.c_double), p.shape[0], ptr(w, C.c_double))
        return w

    def encode(self, pts) -> np.ndarray:
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        D = self.desc.grid.levels * self.desc.grid.features_per_level
        f = np.empty((p.shape[0], D), np.float32)
        call("arfx_hash_encode", self._h, ptr(p, C.c_double), p.shape[0], ptr(f, C.c_float))
        return f

    def field_query(self, pts):
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        d = np.empty(p.shape[0], np.float32)
        c = np.empty((p.shape[0], 3), np.float32)
        call("arfx_field_query", self._h, ptr(p, C.c_double), p.shape[0], ptr(d, C.c_float), ptr(c, C.c_float))
        return d, c

    def inverse_lbs(self, pose: SkeletonPose, pts, pre=None, cutoff_factor: float = 3.0):
        """inverse_lbs_ctx over a batch with PoseContext::make(skel, pose, pre, cutoff)."""
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        pre = rigid() if pre is None else np.ascontiguousarray(pre, np.float64)
        n = p.shape[0]
        counts = np.zeros(n, np.int32)
        roots = np.zeros((n, L.MAX_ROOTS, 3), np.float64)
        res = np.zeros((n, L.MAX_ROOTS), np.float64)
        call("arfx_inverse_lbs", self._h, ptr(pose.bone_transforms, C.c_double), ptr(pre, C.c_double),
             cutoff_factor, ptr(p, C.c_double), n, ptr(counts, C.c_int32), ptr(roots, C.c_double),
             ptr(res, C.c_double))
        return counts, roots, res

    def posed_query(self, pose: "PosedModelView | SkeletonPose", pts_norm):
        view = pose if isinstance(pose, PosedModelView) else PosedModelView(self, pose)
        p = np.ascontiguousarray(pts_norm, np.float64).reshape(-1, 3)
        n = p.shape[0]
        d = np.zeros(n, np.float32)
        c = np.zeros((n, 3), np.float32)
        x = np.zeros((n, 3), np.float64)
        h = np.zeros(n, np.uint8)
        cnt = L.ArfxCounters()
        call("arfx_posed_query", self._h, view._h, ptr(p, C.c_double), n, ptr(d, C.c_float), ptr(c, C.c_float),
             ptr(x, C.c_double), ptr(h, C.c_uint8), C.byref(cnt))
        self.counters.posed_queries += cnt.posed_queries
        self.counters.canonical_queries += cnt.canonical_queries
        return d, c, x, h.astype(bool)


class PosedModelView:
    """R/model.hpp:85-114: normalized-space PoseContext of one pose, on the device."""

    def __init__(self, model: Model, pose: SkeletonPose):
        if pose.bone_count() != model.n_bones:
            raise L.InvalidArgument(1, "pose context: bone count mismatch")
        self.model = model
        self.pose = pose
        h = C.c_void_p()
        call("arfx_pose_create", model._h, ptr(pose.bone_transforms, C.c_double),
             ptr(pose.global_transform, C.c_double), C.byref(h))
        self._h = h

    def update(self, pose: SkeletonPose, stream=None, sync: bool = True):
        """sync=False: arfx_pose_update_async (staged copy on `stream`, no synchronisation)."""
        self.pose = pose
        call("arfx_pose_update" if sync else "arfx_pose_update_async", self._h,
             ptr(pose.bone_transforms, C.c_double), ptr(pose.global_transform, C.c_double), stream)

    def close(self):
        if self._h:
            L.lib().arfx_pose_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class OccupancyGrid:
    """R/occupancy.hpp:37-126, device-resident."""

    def __init__(self, box: Aabb, cfg: OccupancyConfig):
        lo = np.asarray(box.lo, np.float64)
        hi = np.asarray(box.hi, np.float64)
        h = C.c_void_p()
        call("arfx_occ_create", ptr(lo, C.c_double), ptr(hi, C.c_double), C.byref(cfg.to_c()), C.byref(h))
        self._h = h
        self._describe()

    def _describe(self):
        res = np.zeros(3, np.int32)
        lo = np.zeros(3, np.float64)
        hi = np.zeros(3, np.float64)
        thr = C.c_double()
        dil = C.c_int32()
        call("arfx_occ_info", self._h, ptr(res, C.c_int32), ptr(lo, C.c_double), ptr(hi, C.c_double), C.byref(thr),
             C.byref(dil))
        self.resolution = tuple(int(r) for r in res)
        self.box = Aabb(tuple(lo.tolist()), tuple(hi.tolist()))
        self.density_threshold = thr.value
        self.dilation = dil.value

    def device_arrays(self):
        """(values f32 [z][y][x], mask u8) device pointers."""
        v, m = C.c_void_p(), C.c_void_p()
        call("arfx_occ_device_arrays", self._h, C.byref(v), C.byref(m))
        return v.value, m.value

    @staticmethod
    def _from_handle(h) -> "OccupancyGrid":
        g = OccupancyGrid.__new__(OccupancyGrid)
        g._h = h if isinstance(h, C.c_void_p) else C.c_void_p(h)
        g._describe()
        return g

    @staticmethod
    def empty(box: Aabb, cfg: OccupancyConfig) -> "OccupancyGrid":
        return OccupancyGrid(box, cfg)

    def cell_count(self) -> int:
        return int(np.prod(self.resolution))

    def download(self):
        v = np.empty(self.cell_count(), np.float32)
        m = np.empty(self.cell_count(), np.uint8)
        call("arfx_occ_download", self._h, ptr(v, C.c_float), ptr(m, C.c_uint8))
        return v, m

    @property
    def values(self):
        return self.download()[0]

    @property
    def mask(self):
        return self.download()[1]

    def upload(self, values=None, mask=None):
        v = None if values is None else np.ascontiguousarray(values, np.float32)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        call("arfx_occ_upload", self._h, ptr(v, C.c_float), ptr(m, C.c_uint8))

    def rebuild_mask(self):
        call("arfx_occ_rebuild_mask", self._h, None)

    def is_occupied(self, pts_normalized) -> np.ndarray:
        """OccupancyGrid::is_occupied (R/occupancy.hpp:81-85), batched on the GPU."""
        p = np.ascontiguousarray(pts_normalized, np.float64).reshape(-1, 3)
        out = np.zeros(p.shape[0], np.uint8)
        call("arfx_occ_is_occupied", self._h, ptr(p, C.c_double), p.shape[0], ptr(out, C.c_uint8))
        return out.astype(bool)

    def occupied_fraction(self) -> float:
        m = self.mask
        return float(m.sum()) / float(m.size)

    def close(self):
        if self._h:
            L.lib().arfx_occ_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------- operations


def build_model(skeleton: Skeleton, grid_cfg: HashGridConfig, mlp_cfg: MlpConfig,
                skinning_resolution=(32, 32, 32), seed: int = 0) -> Model:
    h = C.c_void_p()
    res = np.asarray(skinning_resolution, np.int32)
    call("arfx_build_model", C.byref(skeleton.to_c()), C.byref(grid_cfg.to_c()), C.byref(mlp_cfg.to_c()),
         ptr(res, C.c_int32), seed & (2**64 - 1), C.byref(h))
    return Model(h)


def model_from_arrays(desc: L.ArfxModelDesc, grid_params, mlp_params, skin_weights) -> Model:
    g = np.ascontiguousarray(grid_params, np.float32)
    m = np.ascontiguousarray(mlp_params, np.float32)
    s = np.ascontiguousarray(skin_weights, np.float64)
    h = C.c_void_p()
    call("arfx_model_create", C.byref(desc), ptr(g, C.c_float), ptr(m, C.c_float), ptr(s, C.c_double), C.byref(h))
    return Model(h)


def build_model_inference_grid(model: Model, pose: SkeletonPose, cfg: OccupancyConfig,
                               view: PosedModelView | None = None) -> OccupancyGrid:
    view = view or PosedModelView(model, pose)
    g = OccupancyGrid(model.normalized_box, cfg)
    cnt = L.ArfxCounters()
    call("arfx_build_inference_grid", model._h, view._h, g._h, C.byref(cnt), None)
    model.counters.posed_queries += cnt.posed_queries
    model.counters.canonical_queries += cnt.canonical_queries
    return g


def build_inference_grid_shard(model: Model, view: "PosedModelView", grid: OccupancyGrid, shard: int,
                               n_shards: int, stream=None) -> None:
    """Cell values of shard `shard` of `n_shards` (cells c = shard + n_shards * j, written as the
    rank-major block values[shard * cells / n_shards + j]); multi-GPU: all-gather the blocks,
    then occ_rebuild_mask_shards(). Asynchronous on `stream` (NULL: the library stream)."""
    call("arfx_build_inference_grid_shard_device", model._h, view._h, grid._h, shard, n_shards, None, stream)


def occ_rebuild_mask_shards(grid: OccupancyGrid, n_shards: int, stream=None) -> None:
    """Rank-major shard blocks -> cell order, then threshold + dilation (asynchronous)."""
    call("arfx_occ_rebuild_mask_shards_async", grid._h, n_shards, stream)


def update_training_grid(model: Model, grid: OccupancyGrid, poses: Sequence[SkeletonPose], decay: float,
                         seed: int, step: int) -> None:
    views = [PosedModelView(model, p) for p in poses]
    arr = (C.c_void_p * len(views))(*[v._h.value for v in views])
    cnt = L.ArfxCounters()
    call("arfx_update_training_grid", model._h, C.cast(arr, C.POINTER(C.c_void_p)), len(views), decay,
         seed & (2**64 - 1), step & (2**64 - 1), grid._h, C.byref(cnt), None)
    model.counters.posed_queries += cnt.posed_queries
    model.counters.canonical_queries += cnt.canonical_queries


def render_model(model: Model, pose: "SkeletonPose | PosedModelView", camera: Camera,
                 occupancy: OccupancyGrid | None, opt: RenderOptions, shard: int = 0, n_shards: int = 1,
                 out: RenderImages | None = None) -> RenderImages:
    view = pose if isinstance(pose, PosedModelView) else PosedModelView(model, pose)
    W, Hh = camera.width, camera.height
    if out is None:
        out = RenderImages(W, Hh, np.zeros((Hh, W, 3), np.float32), np.zeros((Hh, W), np.float32))
    cnt = L.ArfxCounters()
    call("arfx_render_model", model._h, view._h, C.byref(camera.to_c()),
         occupancy._h if occupancy is not None else None, C.byref(opt.to_c()), shard, n_shards,
         ptr(out.rgb, C.c_float), ptr(out.alpha, C.c_float), C.byref(cnt), None)
    model.counters.posed_queries += cnt.posed_queries
    model.counters.canonical_queries += cnt.canonical_queries
    return out


def render_model_async(model: Model, pose: "PosedModelView", camera: Camera, occupancy: "OccupancyGrid | None",
                       opt: RenderOptions, out: RenderImages, counters: np.ndarray, shard: int = 0,
                       n_shards: int = 1, stream=None) -> None:
    """arfx_render_model_async: enqueue the frame; `out` (pinned numpy arrays for overlap) and
    `counters` (uint64[4]: posed, canonical, pool, overflow) are filled once render_wait
    returns. A frame with counters[3] != 0 overflowed the workspace: re-render it with
    render_model."""
    assert counters.dtype == np.uint64 and counters.size >= 4 and counters.flags.c_contiguous
    call("arfx_render_model_async", model._h, pose._h, C.byref(camera.to_c()),
         occupancy._h if occupancy is not None else None, C.byref(opt.to_c()), shard, n_shards,
         ptr(out.rgb, C.c_float), ptr(out.alpha, C.c_float),
         counters.ctypes.data_as(C.POINTER(C.c_uint64)), stream)


def render_wait(model: Model) -> None:
    """Wait for every render_model_async copy of this model (host buffers valid after)."""
    call("arfx_render_wait", model._h)


@dataclass
class RenderTrace:
    ray: np.ndarray
    index: np.ndarray
    has_root: np.ndarray
    density: np.ndarray
    color: np.ndarray
    canonical: np.ndarray
    delta: np.ndarray


def render_trace(model: Model) -> RenderTrace:
    n = C.c_int64()
    call("arfx_render_trace", model._h, 0, C.byref(n), None, None, None, None, None, None, None)
    k = n.value
    t = RenderTrace(np.zeros(k, np.int32), np.zeros(k, np.int32), np.zeros(k, np.uint8), np.zeros(k, np.float32),
                    np.zeros((k, 3), np.float32), np.zeros((k, 3), np.float64), np.zeros(k, np.float64))
    call("arfx_render_trace", model._h, k, C.byref(n), ptr(t.ray, C.c_int32), ptr(t.index, C.c_int32),
         ptr(t.has_root, C.c_uint8), ptr(t.density, C.c_float), ptr(t.color, C.c_float),
         ptr(t.canonical, C.c_double), ptr(t.delta, C.c_double))
    return t


def composite(ray_lengths, delta, skipped, density, color, epsilon: float):
    """Batched composite (R/render.hpp:98-119) over concatenated per-ray sample sets."""
    rl = np.ascontiguousarray(ray_lengths, np.int32)
    n = rl.shape[0]
    d = np.ascontiguousarray(delta, np.float64)
    s = np.ascontiguousarray(skipped, np.uint8)
    de = np.ascontiguousarray(density, np.float32)
    co = np.ascontiguousarray(color, np.float32)
    c3 = np.zeros((n, 3), np.float64)
    a = np.zeros(n, np.float64)
    term = np.zeros(n, np.int32)
    call("arfx_composite", n, ptr(rl, C.c_int32), None, ptr(d, C.c_double), ptr(s, C.c_uint8),
         ptr(de, C.c_float), ptr(co, C.c_float), epsilon, ptr(c3, C.c_double), ptr(a, C.c_double),
         ptr(term, C.c_int32))
    return c3, a, term


def composite_backward(ray_lengths, delta, skipped, density, color, epsilon: float, d_color, d_alpha):
    """Batched composite_backward (R/render.hpp:125-157)."""
    rl = np.ascontiguousarray(ray_lengths, np.int32)
    n = rl.shape[0]
    ns = int(rl.sum())
    d = np.ascontiguousarray(delta, np.float64)
    s = np.ascontiguousarray(skipped, np.uint8)
    de = np.ascontiguousarray(density, np.float32)
    co = np.ascontiguousarray(color, np.float32)
    dc = np.ascontiguousarray(d_color, np.float64).reshape(n, 3)
    da = np.ascontiguousarray(d_alpha, np.float64).reshape(n)
    ds = np.zeros(ns, np.float64)
    dcs = np.zeros((ns, 3), np.float64)
    call("arfx_composite_backward", n, ptr(rl, C.c_int32), None, ptr(d, C.c_double), ptr(s, C.c_uint8),
         ptr(de, C.c_float), ptr(co, C.c_float), epsilon, ptr(dc, C.c_double), ptr(da, C.c_double),
         ptr(ds, C.c_double), ptr(dcs, C.c_double))
    return ds, dcs


def field_query_backward(model: Model, pts, d_density, d_color) -> None:
    """CanonicalField::query_backward (R/field.hpp:91-103) over a batch; accumulates into
    the model's gradient buffers (Model.zero_grad / Model.grads)."""
    p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    dd = np.ascontiguousarray(d_density, np.float32).reshape(-1)
    dc = np.ascontiguousarray(d_color, np.float32).reshape(-1, 3)
    call("arfx_field_query_backward", model._h, ptr(p, C.c_double), p.shape[0], ptr(dd, C.c_float),
         ptr(dc, C.c_float))


def train_fwd_bwd(model: Model, pose: "SkeletonPose | PosedModelView", camera: Camera,
                  occupancy: OccupancyGrid | None, opt: RenderOptions, px, py, d_color, d_alpha):
    """Training forward + backward for rays through pixels (px, py) with upstream dL/dC, dL/dA
    (composed per SPEC.md:490-494); accumulates FieldGrads into the model. Returns rgb, alpha."""
    view = pose if isinstance(pose, PosedModelView) else PosedModelView(model, pose)
    pxa = np.ascontiguousarray(px, np.int32)
    pya = np.ascontiguousarray(py, np.int32)
    n = pxa.shape[0]
    dc = np.ascontiguousarray(d_color, np.float32).reshape(n, 3)
    da = np.ascontiguousarray(d_alpha, np.float32).reshape(n)
    rgb = np.zeros((n, 3), np.float32)
    alpha = np.zeros(n, np.float32)
    cnt = L.ArfxCounters()
    call("arfx_train_fwd_bwd", model._h, view._h, C.byref(camera.to_c()),
         occupancy._h if occupancy is not None else None, C.byref(opt.to_c()), n, ptr(pxa, C.c_int32),
         ptr(pya, C.c_int32), ptr(dc, C.c_float), ptr(da, C.c_float), ptr(rgb, C.c_float), ptr(alpha, C.c_float),
         C.byref(cnt), None)
    model.counters.posed_queries += cnt.posed_queries
    model.counters.canonical_queries += cnt.canonical_queries
    return rgb, alpha


# ----------------------------------------------------------------------------- training


@dataclass
class LossConfig:  # LossWeights SPEC.md:446-449, defaults
    w_rgb: float = 1.0
    w_alpha: float = 0.1
    w_hard: float = 0.1
    w_density: float = 0.1
    huber_delta: float = 0.1

    def to_c(self, gt_frame: "tuple[int, int] | None" = None) -> L.ArfxLossConfig:
        """gt_frame = (width, height): the device train steps read targets from whole frames
        at each ray's pixel (arfx_loss_config.gt_width / gt_height)."""
        w, h = gt_frame if gt_frame is not None else (0, 0)
        return L.ArfxLossConfig(self.w_rgb, self.w_alpha, self.w_hard, self.w_density, self.huber_delta, w, h)


@dataclass
class AdamConfig:  # SPEC.md:508-509 (betas / eps: the encoding system's practice)
    lr_grid: float = 1e-2
    lr_mlp: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.99
    eps: float = 1e-15
    total_steps: int = 0        # cosine horizon; <= 0: constant lr
    final_lr_factor: float = 0.0

    def to_c(self) -> L.ArfxAdamConfig:
        return L.ArfxAdamConfig(self.lr_grid, self.lr_mlp, self.beta1, self.beta2, self.eps, int(self.total_steps),
                                self.final_lr_factor)


def losses(rgb, alpha, gt_rgb, gt_alpha, cfg: LossConfig):
    """SPEC.md:454-477 losses on rendered values: returns (loss4, d_rgb, d_alpha) with
    loss4 = (L_rgb, L_alpha, L_hard, weighted total) and f32 gradients of the total."""
    r = np.ascontiguousarray(rgb, np.float32).reshape(-1, 3)
    n = r.shape[0]
    a = np.ascontiguousarray(alpha, np.float32).reshape(n)
    gr = np.ascontiguousarray(gt_rgb, np.float32).reshape(n, 3)
    ga = np.ascontiguousarray(gt_alpha, np.float32).reshape(n)
    l4 = np.zeros(4, np.float64)
    dr = np.zeros((n, 3), np.float32)
    da = np.zeros(n, np.float32)
    call("arfx_losses", n, ptr(r, C.c_float), ptr(a, C.c_float), ptr(gr, C.c_float), ptr(ga, C.c_float),
         C.byref(cfg.to_c()), ptr(l4, C.c_double), ptr(dr, C.c_float), ptr(da, C.c_float))
    return l4, dr, da


def train_step(model: Model, pose: "SkeletonPose | PosedModelView", camera: Camera, occupancy: "OccupancyGrid | None",
               opt: RenderOptions, px, py, gt_rgb, gt_alpha, cfg: LossConfig):
    """Fused training forward + losses + backward (arfx_train_step): accumulates gradients
    into the model; returns (loss4, rgb, alpha)."""
    view = pose if isinstance(pose, PosedModelView) else PosedModelView(model, pose)
    pxa = np.ascontiguousarray(px, np.int32)
    pya = np.ascontiguousarray(py, np.int32)
    n = pxa.shape[0]
    gr = np.ascontiguousarray(gt_rgb, np.float32).reshape(n, 3)
    ga = np.ascontiguousarray(gt_alpha, np.float32).reshape(n)
    l4 = np.zeros(4, np.float64)
    rgb = np.zeros((n, 3), np.float32)
    alpha = np.zeros(n, np.float32)
    cnt = L.ArfxCounters()
    call("arfx_train_step", model._h, view._h, C.byref(camera.to_c()),
         occupancy._h if occupancy is not None else None, C.byref(opt.to_c()), n, ptr(pxa, C.c_int32),
         ptr(pya, C.c_int32), ptr(gr, C.c_float), ptr(ga, C.c_float), C.byref(cfg.to_c()), ptr(l4, C.c_double),
         ptr(rgb, C.c_float), ptr(alpha, C.c_float), C.byref(cnt), None)
    model.counters.posed_queries += cnt.posed_queries
    model.counters.canonical_queries += cnt.canonical_queries
    return l4, rgb, alpha


def density_step(model: Model, pose: "SkeletonPose | PosedModelView", occupancy: "OccupancyGrid", n_points: int,
                 seed: int, step: int, cfg: LossConfig):
    """L_density: returns (L_density, n_empty); w_density * gradient is
    accumulated into the model (arfx_density_step)."""
    view = pose if isinstance(pose, PosedModelView) else PosedModelView(model, pose)
    out = np.zeros(2, np.float64)
    call("arfx_density_step", model._h, view._h, occupancy._h, n_points, seed & (2**64 - 1), step & (2**64 - 1),
         C.byref(cfg.to_c()), ptr(out, C.c_double), None)
    return float(out[0]), int(out[1])


def density_points(occupancy_box: Aabb, n: int, seed: int, step: int) -> np.ndarray:
    """The L_density sample points (host restatement of density_points_kernel, for tests):
    point i = lo + e * (u0, u1, u2), u from keyed_rng(seed, 0xde45, step, i)."""
    from .fixtures import keyed_rng
    lo = np.asarray(occupancy_box.lo, np.float64)
    e = np.asarray(occupancy_box.hi, np.float64) - lo
    out = np.empty((n, 3), np.float64)
    for i in range(n):
        r = keyed_rng(seed, 0xDE45, step, i)
        u = (r.next_double(), r.next_double(), r.next_double())
        for a in range(3):
            out[i, a] = lo[a] + e[a] * u[a]
    return out


# ----------------------------------------------------------------------------- checkpoint


def save_checkpoint(path, model: Model, occupancy: "OccupancyGrid | None" = None, step: int = 0,
                    with_optimizer: bool = False) -> None:
    """SPEC checkpoint file (arfx_checkpoint_save): configs, grid, MLP, skinning, optional
    occupancy grid and Adam state; bitwise round trip."""
    call("arfx_checkpoint_save", str(path).encode(), model._h, occupancy._h if occupancy is not None else None,
         int(step), 1 if with_optimizer else 0)


def load_checkpoint(path):
    """-> (Model, OccupancyGrid | None, step)."""
    mh, oh, st = C.c_void_p(), C.c_void_p(), C.c_int64()
    call("arfx_checkpoint_load", str(path).encode(), C.byref(mh), C.byref(oh), C.byref(st))
    model = Model(mh)
    occ = OccupancyGrid._from_handle(oh) if oh.value else None
    return model, occ, st.value


# ----------------------------------------------------------------------------- analytic ground truth


@dataclass
class CapsuleFigure:  # R/scene.hpp:13-27
    skeleton: Skeleton
    colors: np.ndarray       # (n_bones, 3)
    amplitudes: np.ndarray   # (n_bones,)
    softness: float = 0.01

    def to_c(self) -> L.ArfxFigure:
        f = L.ArfxFigure()
        f.skeleton = self.skeleton.to_c()
        col = np.asarray(self.colors, np.float64).reshape(-1, 3)
        amp = np.asarray(self.amplitudes, np.float64).reshape(-1)
        if col.shape[0] != self.skeleton.bone_count() or amp.shape[0] != self.skeleton.bone_count():
            raise L.InvalidArgument(1, "figure: per-bone color/amplitude required")
        for i in range(col.shape[0]):
            for c in range(3):
                f.color[i][c] = float(col[i, c])
            f.amplitude[i] = float(amp[i])
        f.softness = float(self.softness)
        return f


def figure_query(fig: CapsuleFigure, pts, pose: SkeletonPose | None = None):
    """analytic_query (R/scene.hpp:31-50) or, with a pose, PosedFigure::query (:79-97)."""
    p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    n = p.shape[0]
    dens = np.zeros(n, np.float64)
    col = np.zeros((n, 3), np.float64)
    bt = None if pose is None else np.ascontiguousarray(pose.bone_transforms, np.float64)
    call("arfx_figure_query", C.byref(fig.to_c()), ptr(bt, C.c_double), ptr(p, C.c_double), n,
         ptr(dens, C.c_double), ptr(col, C.c_double))
    return dens, col


def figure_render(fig: CapsuleFigure, pose: SkeletonPose, normalized_box: Aabb, camera: Camera,
                  opt: RenderOptions):
    """Ground-truth frame of the posed analytic figure: render_image (R/render.hpp:178-218)
    through normalized space (G^-1) into `normalized_box`, no occupancy; plus the exact
    silhouette mask PosedFigure::ray_hits (R/scene.hpp:123-130). Returns (RenderImages, mask)."""
    W, Hh = camera.width, camera.height
    out = RenderImages(W, Hh, np.zeros((Hh, W, 3), np.float32), np.zeros((Hh, W), np.float32))
    mask = np.zeros((Hh, W), np.uint8)
    lo = np.asarray(normalized_box.lo, np.float64)
    hi = np.asarray(normalized_box.hi, np.float64)
    call("arfx_figure_render", C.byref(fig.to_c()), ptr(pose.bone_transforms, C.c_double),
         ptr(pose.global_transform, C.c_double), ptr(lo, C.c_double), ptr(hi, C.c_double), C.byref(camera.to_c()),
         C.byref(opt.to_c()), ptr(out.rgb, C.c_float), ptr(out.alpha, C.c_float), ptr(mask, C.c_uint8), None)
    return out, mask


ROW_TILE = 4  # kRowTile (arfx_internal.h)


def shard_rows(height: int, rank: int, world: int, tile: int = ROW_TILE) -> list:
    """Rows rendered by `rank` of `world`: interleaved `tile`-row tiles (tile % world == rank),
    the same partition libarfx applies for arfx_render_model(..., rank, world, ...)."""
    return [y for y in range(height) if (y // tile) % world == rank]


def shard_cells(n_cells: int, rank: int, world: int) -> np.ndarray:
    """Occupancy cells computed by `rank` of `world` (arfx_build_inference_grid_shard_device):
    c = rank + world * j, stored as the rank-major block [rank * n_cells / world + j]."""
    if n_cells % world:
        raise L.InvalidArgument(1, "build_inference_grid_shard: the cell count must divide by n_shards")
    return np.arange(rank, n_cells, world, dtype=np.int64)


def unshard_cells(blocks: np.ndarray, world: int) -> np.ndarray:
    """Rank-major shard blocks (after the all-gather) -> cell order (occ_unshard_kernel)."""
    b = np.asarray(blocks).reshape(world, -1)
    return b.T.reshape(-1).copy()


def device_count() -> int:
    n = C.c_int()
    call("arfx_device_count", C.byref(n))
    return n.value
