"""Training loop host side (SPEC.md:440-530 train_step).

The reference code base stops at the differentiable pieces (composite_backward,
query_backward); the SPEC's trainer is built here over the libarfx training ABI:

  per step t (all enqueued on the device without host synchronisation; the occupancy update
  every k steps is the sync point, where the losses are also checked for finiteness):
    rays     B / world rays per rank: frame f and pixels from keyed_rng(seed, 0x7a11, t, rank)
             (draw order: frame, then px, py per ray), ground truth gathered from the
             device-resident dataset frames (analytic figure, arfx_figure_render)
    step     arfx_train_step_device: forward, losses fused into the composite kernel,
             backward -> the model's flat gradient vector
    density  arfx_density_step_device: L_density over 4096 uniform points (w_density > 0)
    sync     world > 1: reduce-scatter(AVG) of the flat gradients over NCCL, Adam on this
             rank's shard, all-gather of the parameter shards (FlatDataParallel)
    optim    arfx_adam_step (zero-grad fused), cosine lr
    occ      every k steps: update_training_grid over the dataset poses (R/occupancy.hpp:155-171),
             identical on every rank (same keys, same parameters)

torch is plumbing only: device tensors for the dataset / ray lists and torch.distributed
for the collectives. Every compute step is a libarfx kernel.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from . import arf
from . import fixtures as fx


def device_view(ptr: int, n: int, dtype="float32"):
    """Zero-copy torch view of n elements of libarfx device memory (__cuda_array_interface__)."""
    import torch

    class _CAI:
        pass

    o = _CAI()
    o.__cuda_array_interface__ = {"shape": (int(n),), "typestr": np.dtype(dtype).str, "data": (int(ptr), False),
                                  "version": 3, "strides": None}
    return torch.as_tensor(o, device="cuda")


@dataclass
class TrainConfig:  # TrainConfig SPEC.md:450-453
    iterations: int = 200
    rays_per_batch: int = 4096           # global batch (split over ranks)
    samples_per_ray: int = 128
    occupancy_interval: int = 16         # k
    seed: int = 1234
    loss: arf.LossConfig = field(default_factory=arf.LossConfig)
    adam: arf.AdamConfig = field(default_factory=arf.AdamConfig)
    occupancy: arf.OccupancyConfig = field(default_factory=arf.OccupancyConfig)
    gt_oversample: int = 4               # SPEC scenegen: ground truth at 4x the training N
    density_points: int = 4096           # L_density point budget per step
    deterministic: bool = False          # bit-reproducible gradients (Model.set_deterministic)


class FlatDataParallel:
    """Gradient / parameter synchronisation of the flat [grid | mlp] vectors over a process
    group: reduce-scatter(AVG) grads -> `optimizer(begin, end)` on this rank's shard ->
    all-gather params, then the other shards' gradients are cleared (the optimizer zeroes
    its own). With world == 1 it is just optimizer(0, n). Backends without reduce-scatter
    (gloo, used by the CPU tests) fall back to all-reduce + slicing, same result."""

    def __init__(self, params, grads, n_flat: int, rank: int = 0, world: int = 1, group=None,
                 force_collectives: bool = False):
        self.params, self.grads, self.n = params, grads, int(n_flat)
        self.rank, self.world, self.group = rank, world, group
        # run the collectives even at world == 1 (exercises the multi-GPU path on one GPU)
        self.collect = world > 1 or force_collectives
        if self.n % (4 * world):
            raise ValueError("flat vector length must split into multiple-of-4 shards")
        self.chunk = self.n // world

    def shard(self, rank: int | None = None):
        r = self.rank if rank is None else rank
        return r * self.chunk, (r + 1) * self.chunk

    def step(self, optimizer) -> None:
        b, e = self.shard()
        if self.collect:
            import torch.distributed as dist
            backend = dist.get_backend(self.group)
            if backend == "nccl":
                dist.reduce_scatter_tensor(self.grads[b:e], self.grads, op=dist.ReduceOp.AVG, group=self.group)
            else:
                dist.all_reduce(self.grads, op=dist.ReduceOp.SUM, group=self.group)
                self.grads.div_(self.world)
        optimizer(b, e)
        if self.collect:
            import torch.distributed as dist
            if dist.get_backend(self.group) == "nccl":
                dist.all_gather_into_tensor(self.params, self.params[b:e], group=self.group)
            else:
                parts = [self.params[r * self.chunk:(r + 1) * self.chunk].clone() for r in range(self.world)]
                dist.all_gather(parts, self.params[b:e].clone(), group=self.group)
                for r, p in enumerate(parts):
                    self.params[r * self.chunk:(r + 1) * self.chunk].copy_(p)
            if b > 0:
                self.grads[:b].zero_()
            if e < self.n:
                self.grads[e:].zero_()


def ray_batch(seed: int, step: int, rank: int, n: int, n_frames: int, width: int, height: int):
    """This rank's rays of step `step`: (frame, px[n], py[n]); keyed_rng(seed, 0x7a11, step, rank),
    draws: frame = next_below(n_frames), then per ray px = next_below(W), py = next_below(H)."""
    rng = fx.keyed_rng(seed, 0x7A11, step, rank)
    f = rng.next_below(n_frames)
    u = fx.pcg_stream_u32(rng, 2 * n).reshape(n, 2)
    px = ((u[:, 0] * np.uint64(width)) >> np.uint64(32)).astype(np.int32)
    py = ((u[:, 1] * np.uint64(height)) >> np.uint64(32)).astype(np.int32)
    return f, px, py


class Trainer:
    """SPEC train_step loop on one GPU per rank (world from torch.distributed when initialised)."""

    def __init__(self, model: arf.Model, figure: arf.CapsuleFigure, poses, camera: arf.Camera, cfg: TrainConfig,
                 rank: int = 0, world: int = 1, group=None, force_collectives: bool = False):
        import torch
        self.torch = torch
        self.model, self.figure, self.poses, self.camera, self.cfg = model, figure, list(poses), camera, cfg
        self.rank, self.world = rank, world
        if cfg.rays_per_batch % world:
            raise ValueError("rays_per_batch must divide by the number of ranks")
        self.n_local = cfg.rays_per_batch // world
        self.views = [arf.PosedModelView(model, p) for p in self.poses]
        model.set_deterministic(cfg.deterministic)
        # ---- dataset: ground-truth frames of the analytic figure (device resident)
        W, H = camera.width, camera.height
        gt_opt = arf.RenderOptions(samples_per_ray=cfg.gt_oversample * cfg.samples_per_ray)
        rgbs, masks = [], []
        for p in self.poses:
            img, mask = arf.figure_render(figure, p, model.normalized_box, camera, gt_opt)
            rgbs.append(img.rgb)
            masks.append(mask.astype(np.float32))
        self.gt_rgb = torch.from_numpy(np.stack(rgbs)).cuda().reshape(len(self.poses), H * W, 3)
        self.gt_alpha = torch.from_numpy(np.stack(masks)).cuda().reshape(len(self.poses), H * W)
        # ---- optimizer state + data-parallel sync over the flat vectors
        fl = model.flat()
        self.n_flat = fl["n_flat"]
        self.params = device_view(fl["params"], self.n_flat)
        self.grads = device_view(fl["grads"], self.n_flat)
        self.dp = FlatDataParallel(self.params, self.grads, self.n_flat, rank, world, group, force_collectives)
        # one non-default stream carries every step: libarfx launches, torch copies/gathers and
        # the NCCL collectives are then ordered without host synchronisation
        self.stream = torch.cuda.Stream()
        self.stream.wait_stream(torch.cuda.current_stream())
        self.loss4 = torch.zeros(4, dtype=torch.float64, device="cuda")
        self.loss_d = torch.zeros(2, dtype=torch.float64, device="cuda")
        self.px = torch.zeros(self.n_local, dtype=torch.int32, device="cuda")
        self.py = torch.zeros(self.n_local, dtype=torch.int32, device="cuda")
        # ---- occupancy: built from the untrained model at step 0
        self.grid = arf.OccupancyGrid(model.normalized_box, cfg.occupancy)
        arf.update_training_grid(model, self.grid, self.poses, cfg.occupancy.decay, cfg.seed, 0)
        self.step_id = 0
        self.fused_density = True  # arfx_train_density_step_device (False: the two calls in sequence)
        # Adam on its own stream behind a parameter fence (overlaps the next step); with several
        # ranks the gradient reduce-scatter / parameter all-gather run on that stream too
        self.adam_stream = torch.cuda.Stream()
        self.ev_params = torch.cuda.Event()
        self._fence_set = False
        # step t+1's forward (march, deformer, field) is enqueued on fstream into the other
        # train slot right after step t's backward (and, with several ranks, beside step t's
        # collectives), so they overlap on the GPU
        self.pipelined = True
        self.fstream = torch.cuda.Stream()
        self.pxs = [torch.zeros(self.n_local, dtype=torch.int32, device="cuda") for _ in range(2)]
        self.pys = [torch.zeros(self.n_local, dtype=torch.int32, device="cuda") for _ in range(2)]
        self.ev_fwd = [torch.cuda.Event(), torch.cuda.Event()]
        self.ev_bwd = [torch.cuda.Event(), torch.cuda.Event()]
        self._pending = [None, None]  # per slot: (step, frame) of the enqueued forward
        # per-step host work kept small: ctypes structs built once, ray pixels drawn on the
        # device, losses written by the library straight into preallocated history rows
        self._cam_c = camera.to_c()
        self._opt_c = self._opt(0, 0).to_c()
        self._lc = cfg.loss.to_c((camera.width, camera.height))
        self._adam_c = cfg.adam.to_c()
        self._hrows = None
        self._hrow_next = 0
        self._hist = []       # per step: device tensor (L_rgb, L_alpha, L_hard, L_density, total)
        self._checked = 0     # steps whose loss has been checked for finiteness
        # set on the device by the guarded Adam when a step's loss is non-finite: that step and
        # every later one leave the model untouched, _check raises
        self.bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._bad_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        self._bad_ev = torch.cuda.Event()
        self._bad_pending = False
        self.ev_grid = torch.cuda.Event()
        self._pose_arr = (C.c_void_p * len(self.views))(*[v._h.value for v in self.views])
        # two pinned host staging slots for the ray pixels (the host runs ahead of the GPU)
        self._h_pix = [torch.zeros((2, self.n_local), dtype=torch.int32).pin_memory() for _ in range(2)]
        self._h_evt = [torch.cuda.Event(), torch.cuda.Event()]

    def _opt(self, frame: int, step: int | None = None) -> arf.RenderOptions:
        st = self.step_id if step is None else step
        return arf.RenderOptions(samples_per_ray=self.cfg.samples_per_ray, stratified=True, seed=self.cfg.seed,
                                 frame_id=st * 1024 + frame)

    def step(self):
        """One SPEC train step, enqueued without host synchronisation (except the occupancy
        update every k steps, which is also where the loss is checked for finiteness).
        Returns the step's loss row as a device tensor (L_rgb, L_alpha, L_hard, their weighted
        sum, L_density, n_empty); `history` gives (L_rgb, L_alpha, L_hard, L_density, total)."""
        if self.pipelined and self.fused_density:
            return self._step_pipelined()  # launches only on its own streams
        with self.torch.cuda.stream(self.stream):
            return self._step()

    def _forward(self, step: int):
        """Enqueue step `step`'s forward on fstream into train slot step & 1."""
        cfg = self.cfg
        k = step & 1
        fs = self.fstream
        fs.wait_event(self.ev_bwd[k])  # the previous backward that used this slot has run
        f = fx.keyed_rng(cfg.seed, 0x7A11, step, self.rank).next_below(len(self.poses))  # ray_batch draw 0
        fsp = C.c_void_p(fs.cuda_stream)
        L.call("arfx_train_rays_device", cfg.seed, step, self.rank, self.n_local, self.camera.width,
               self.camera.height, C.c_void_p(self.pxs[k].data_ptr()), C.c_void_p(self.pys[k].data_ptr()), fsp)
        self._opt_c.frame_id = step * 1024 + f
        L.call("arfx_train_forward_device", self.model._h, self.views[f]._h, C.byref(self._cam_c), self.grid._h,
               C.byref(self._opt_c), self.n_local, C.c_void_p(self.pxs[k].data_ptr()),
               C.c_void_p(self.pys[k].data_ptr()), k, fsp)
        self.ev_fwd[k].record(fs)
        self._pending[k] = (step, f)

    def _history_row(self):
        """A zeroed device row (L_rgb, L_alpha, L_hard, total_without_density, L_density,
        n_empty) for this step's losses; blocks of 1024 rows, never moved (views stay valid)."""
        torch = self.torch
        if self._hrows is None or self._hrow_next == self._hrows.shape[0]:
            with torch.cuda.stream(self.stream):  # zeroed in order before the library writes rows
                self._hrows = torch.zeros((1024, 6), dtype=torch.float64, device="cuda")
            self._hrow_next = 0
        r = self._hrows[self._hrow_next]
        self._hrow_next += 1
        return r

    def _step_pipelined(self):
        cfg = self.cfg
        t = self.step_id
        k = t & 1
        if self._pending[k] is None or self._pending[k][0] != t:
            self._forward(t)  # first step (or after restore / an occupancy update)
        f = self._pending[k][1]
        self._pending[k] = None
        self.stream.wait_event(self.ev_fwd[k])
        dens = cfg.loss.w_density > 0 and cfg.density_points > 0
        row = self._history_row()
        sp = C.c_void_p(self.stream.cuda_stream)
        self._opt_c.frame_id = t * 1024 + f
        L.call("arfx_train_backward_device", self.model._h, self.views[f]._h, self.grid._h, C.byref(self._opt_c),
               self.n_local, C.c_void_p(self.pxs[k].data_ptr()), C.c_void_p(self.pys[k].data_ptr()),
               C.c_void_p(self.gt_rgb[f].data_ptr()), C.c_void_p(self.gt_alpha[f].data_ptr()), C.byref(self._lc),
               C.c_void_p(row.data_ptr()), k, cfg.density_points if dens else 0,
               (cfg.seed * 4 + self.rank) & (2**64 - 1), t, C.c_void_p(row.data_ptr() + 4 * 8), sp)
        self.ev_bwd[k].record(self.stream)
        t1 = t + 1
        self.adam_stream.wait_event(self.ev_bwd[k])  # this step's gradients are complete
        asp = C.c_void_p(self.adam_stream.cuda_stream)
        if self.dp.collect:
            # reduce-scatter(AVG) grads -> guarded Adam on this rank's shard -> all-gather params,
            # on the Adam stream (torch orders the NCCL work after it); the guard is the sum of
            # the ranks' loss rows, so every rank skips a non-finite step together
            import torch.distributed as dist
            with self.torch.cuda.stream(self.adam_stream):
                guard = row.clone()
                dist.all_reduce(guard, op=dist.ReduceOp.SUM, group=self.dp.group)
                if self.cfg.deterministic:
                    self.model.flush_grads(asp)  # the reduce-scatter reads the gradient array directly
                gd = (C.c_void_p(guard.data_ptr()), 6, C.c_void_p(self.bad.data_ptr()))
                self.dp.step(lambda b, e: self.model.adam_step(self.cfg.adam, t1, b, e, asp, gd))
        else:
            L.call("arfx_adam_step_guarded", self.model._h, C.byref(self._adam_c), t1, 0, self.n_flat,
                   C.c_void_p(row.data_ptr()), 6, C.c_void_p(self.bad.data_ptr()), asp)
        self.ev_params.record(self.adam_stream)
        if not self._fence_set:
            self.model.set_param_fence(self.ev_params.cuda_event)
            self._fence_set = True
        self._hist.append(row)
        self.step_id = t1
        if cfg.occupancy_interval > 0 and t1 % cfg.occupancy_interval == 0:
            # the training-grid update (R/occupancy.hpp:155-171) reads the parameters after this
            # step's Adam: enqueued on the Adam stream with no host round trip; the next
            # forward and backward wait for it (the pipeline does not drain)
            L.call("arfx_update_training_grid_device", self.model._h, self._pose_arr, len(self.views),
                   cfg.occupancy.decay, cfg.seed & (2**64 - 1), t1, self.grid._h, None, asp)
            self.ev_grid.record(self.adam_stream)
            self.fstream.wait_event(self.ev_grid)
            self.stream.wait_event(self.ev_grid)
            self._check_async()
        self._forward(t1)  # overlaps this step's backward (its field waits for this Adam)
        return row

    def _check_async(self):
        """Non-blocking finiteness check: the device flag of the guarded Adam is copied to pinned
        memory at every occupancy boundary and read at the next one once the copy has landed
        (a poisoned step has already been skipped on the device, so late detection is safe)."""
        if self._bad_pending and self._bad_ev.query():
            self._bad_pending = False
            if int(self._bad_host[0]):
                self._sync()
                self._check()
        if not self._bad_pending:
            with self.torch.cuda.stream(self.adam_stream):
                self._bad_host.copy_(self.bad, non_blocking=True)
            self._bad_ev.record(self.adam_stream)
            self._bad_pending = True

    def _step(self):
        torch = self.torch
        cfg, W = self.cfg, self.camera.width
        f, px, py = ray_batch(cfg.seed, self.step_id, self.rank, self.n_local, len(self.poses), W, self.camera.height)
        slot = self.step_id & 1
        self._h_evt[slot].synchronize()  # the copy that last used this staging slot has run
        hp = self._h_pix[slot]
        hp[0].numpy()[:] = px
        hp[1].numpy()[:] = py
        self.px.copy_(hp[0], non_blocking=True)
        self.py.copy_(hp[1], non_blocking=True)
        self._h_evt[slot].record(self.stream)
        # targets: the composite kernel reads frame f's ground truth at each ray's pixel
        g_rgb = C.c_void_p(self.gt_rgb[f].data_ptr())
        g_alpha = C.c_void_p(self.gt_alpha[f].data_ptr())
        lc = cfg.loss.to_c((W, self.camera.height))
        sp = C.c_void_p(self.stream.cuda_stream)
        dens = cfg.loss.w_density > 0 and cfg.density_points > 0  # L_density
        if dens and self.fused_density:
            # one call: the density forward overlaps the train step on a side stream
            L.call("arfx_train_density_step_device", self.model._h, self.views[f]._h, C.byref(self.camera.to_c()),
                   self.grid._h, C.byref(self._opt(f).to_c()), self.n_local, C.c_void_p(self.px.data_ptr()),
                   C.c_void_p(self.py.data_ptr()), g_rgb, g_alpha, C.byref(lc), C.c_void_p(self.loss4.data_ptr()),
                   cfg.density_points, (cfg.seed * 4 + self.rank) & (2**64 - 1), self.step_id,
                   C.c_void_p(self.loss_d.data_ptr()), sp)
        else:
            L.call("arfx_train_step_device", self.model._h, self.views[f]._h, C.byref(self.camera.to_c()),
                   self.grid._h, C.byref(self._opt(f).to_c()), self.n_local, C.c_void_p(self.px.data_ptr()),
                   C.c_void_p(self.py.data_ptr()), g_rgb, g_alpha, C.byref(lc), C.c_void_p(self.loss4.data_ptr()),
                   None, None, sp)
            if dens:
                L.call("arfx_density_step_device", self.model._h, self.views[f]._h, self.grid._h, cfg.density_points,
                       (cfg.seed * 4 + self.rank) & (2**64 - 1), self.step_id, C.byref(cfg.loss.to_c()),
                       C.c_void_p(self.loss_d.data_ptr()), sp)
        if not dens:
            self.loss_d.zero_()
        t = self.step_id + 1
        loss = self._history_row()
        loss[0:4].copy_(self.loss4)
        loss[4:6].copy_(self.loss_d)
        self._hist.append(loss)
        guard = loss
        if self.dp.collect:
            # every rank must skip together: the guard is the sum of the ranks' loss rows
            import torch.distributed as dist
            guard = loss.clone()
            dist.all_reduce(guard, op=dist.ReduceOp.SUM, group=self.dp.group)
        gd = (C.c_void_p(guard.data_ptr()), 6, C.c_void_p(self.bad.data_ptr()))
        if cfg.deterministic and self.dp.collect:
            self.model.flush_grads(sp)  # the reduce-scatter reads the gradient array directly
        if not self.dp.collect:
            # Adam of step t on its own stream, fenced: the next step's march and deformer
            # (which read neither parameters nor gradients) run beside it, its field kernels
            # wait on ev_params (arfx_model_set_param_fence)
            self.adam_stream.wait_stream(self.stream)
            self.model.adam_step(cfg.adam, t, 0, self.n_flat, C.c_void_p(self.adam_stream.cuda_stream), gd)
            self.ev_params.record(self.adam_stream)
            if not self._fence_set:
                self.model.set_param_fence(self.ev_params.cuda_event)
                self._fence_set = True
        else:
            self.dp.step(lambda b, e: self.model.adam_step(cfg.adam, t, b, e, sp, gd))
        self.step_id = t
        if cfg.occupancy_interval > 0 and t % cfg.occupancy_interval == 0:
            self._sync()  # the host-buffer API below runs on the library's stream
            arf.update_training_grid(self.model, self.grid, self.poses, cfg.occupancy.decay, cfg.seed, t)
            self._check()
        return loss

    def _sync(self):
        self.stream.synchronize()
        self.fstream.synchronize()
        if self.adam_stream is not None:
            self.adam_stream.synchronize()

    def close(self):
        """Detach the parameter fence (the model outlives the trainer)."""
        self._sync()
        if self._fence_set:
            self.model.set_param_fence(None)
            self._fence_set = False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self):
        if int(self.bad.item()):
            h = self._rows_cpu(self._hist[self._checked:]) if self._checked < len(self._hist) else np.zeros((0, 5))
            bad = ~np.all(np.isfinite(h), axis=1)
            k = self._checked + int(np.argmax(bad)) + 1 if bad.any() else self._checked
            raise L.NumericError(3, f"train_step: non-finite loss at step {k}; the optimizer skipped that step and "
                                    "every later one, so the model holds its last finite state")
        if self._checked < len(self._hist):
            h = self._rows_cpu(self._hist[self._checked:])
            bad = ~np.all(np.isfinite(h), axis=1)
            if bad.any():
                k = self._checked + int(np.argmax(bad)) + 1
                raise L.NumericError(3, f"train_step: non-finite loss at step {k}: {h[np.argmax(bad)].tolist()}")
            self._checked = len(self._hist)

    @property
    def history(self) -> np.ndarray:
        """Per-step losses (synchronises): rows (L_rgb, L_alpha, L_hard, L_density, total)."""
        self._sync()
        self._check()
        return self._rows_cpu(self._hist) if self._hist else np.zeros((0, 5))

    def _rows_cpu(self, rows) -> np.ndarray:
        """Stored rows (L_rgb, L_alpha, L_hard, weighted sum of those, L_density, n_empty) ->
        (L_rgb, L_alpha, L_hard, L_density, total)."""
        r = torch_stack_cpu(self.torch, rows)
        return np.stack([r[:, 0], r[:, 1], r[:, 2], r[:, 4], r[:, 3] + self.cfg.loss.w_density * r[:, 4]], axis=1)

    def save(self, path) -> None:
        """Checkpoint (model, Adam moments, occupancy grid, step) for an exact resume."""
        self._sync()
        arf.save_checkpoint(path, self.model, self.grid, step=self.step_id, with_optimizer=True)

    def restore(self, path) -> None:
        """Resume from `save`: parameters, Adam moments, occupancy grid and step counter are
        replaced, so the following steps draw the same ray batches (keyed by step) as an
        uninterrupted run -- with TrainConfig.deterministic the continuation is bit-identical."""
        self._sync()
        m2, occ, step = arf.load_checkpoint(path)
        if occ is None:
            raise ValueError("restore: checkpoint has no occupancy grid")
        g, w, _ = m2.params()
        self.model.set_params(g, w)
        self.model.set_adam_state(*m2.adam_state())
        m2.close()
        self.grid = occ
        self.step_id = int(step)
        self._pending = [None, None]  # forwards enqueued for the old state are discarded

    def train(self, iterations: int | None = None):
        for _ in range(iterations or self.cfg.iterations):
            self.step()
        return self.history


def torch_stack_cpu(torch, ts) -> np.ndarray:
    return torch.stack(ts).cpu().numpy()


def psnr(img, ref) -> float:
    """PSNR = 10 log10(1 / MSE) for [0,1] images, capped at 99 dB."""
    mse = float(np.mean((np.asarray(img, np.float64) - np.asarray(ref, np.float64)) ** 2))
    return 99.0 if mse == 0 else min(99.0, 10.0 * np.log10(1.0 / mse))
