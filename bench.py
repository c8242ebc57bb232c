#!/usr/bin/env python
"""bench.py -- 540x540 avatar render FPS / posed samples per second (BASELINE.json metric).

Workload (config.workload): BASELINE.json configs[3], the 100-frame novel-pose animation
at 540x540 with a per-frame occupancy refresh, on the config-1 avatar (24-bone smpl24
capsule skeleton, 16-level hash grid 2^19 x 2 f32, 32-64-64-4 MLP, 32^3 skinning grid,
64^3 occupancy, N=128 midpoint samples, random init seed 1234). One step = one frame:
build_model_inference_grid + render_model. With N GPUs each frame's rays are sharded
over ranks in interleaved 4-row tiles (no data-path collective).

  value : frames/s with inputs resident in HBM (per-pose contexts pre-uploaded), device
          outputs; timed with CUDA events per frame, L2 flushed between frames.
  e2e   : the same metric through the public host-buffer API (pose from host, pinned
          RGB/alpha read back every frame), wall clock around the K frames.
  --impl reference : the reference's own CPU implementation (oracle/_ref, compiled
          from /root/reference) on this host's cores, same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "render_fps_540x540"
UNIT = "frames/s"
WORKLOAD = ("100-frame novel-pose animation at 540x540, per-frame 64^3 occupancy refresh; 24-bone smpl24 "
            "avatar, 16-level 2^19 hash grid, 32-64-64-4 MLP, N=128 (BASELINE configs[3] on configs[0]'s avatar)")
W_IMG = H_IMG = 540
N_FRAMES = 100
ROW_TILE = 4  # libarfx kRowTile: ray shards = interleaved 4-row tiles


def shard_rows(world: int, rank: int) -> int:
    return sum(1 for y in range(H_IMG) if (y // ROW_TILE) % world == rank)


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:  # nvidia-smi's own sampling loop (every 50 ms) for the whole timed region
            self._p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "50"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._p = None
        time.sleep(0.3)  # first sample lands before the timed region starts

    def stop(self):
        time.sleep(0.1)
        if getattr(self, "_p", None) is not None:
            self._p.terminate()
            try:
                out, _ = self._p.communicate(timeout=5)
            except Exception:
                out = ""
            self.rows = [[s.strip() for s in ln.split(",")] for ln in out.splitlines() if ln.strip()]
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


DTYPE_EXACT = "f64 march/deformer (bit-exact, no FMA) + f32 hash encode + exact f32 SIMT MLP"
DTYPE = ("f64 march/deformer (bit-exact, no FMA) + f32 hash encode + MLP as split-bf16 tcgen05 "
         "(hi/lo bf16 operands, 3 MMAs per product, f32 accumulate)")


def bench_config(world: int) -> dict:
    """The `config` both arms print (identical by construction)."""
    return {"workload": WORKLOAD, "image": [W_IMG, H_IMG], "frames": N_FRAMES, "samples_per_ray": 128,
            "occupancy": "64^3, rebuilt per frame", "l2": "flushed between timed frames (256 MB write)",
            "parallelism": f"rays sharded over {world} GPU(s) in interleaved {ROW_TILE}-row tiles"}


# ----------------------------------------------------------------------------- reference arm

def reference_frames(n_frames: int, frame0: int = 0, keep_last: bool = False):
    """Time n full frames (inference grid + render) of the reference on all host threads. The
    workload is built by the reference itself (oracle/workload.py: no product code on this arm)."""
    from oracle import workload as wl
    from oracle.oracle_ctypes import Checker
    ref = Checker("ref")
    sk, rm, poses, cam, occ_cfg, opt = wl.build(ref, W_IMG, H_IMG)
    sel = [poses[(frame0 + i) % N_FRAMES] for i in range(n_frames)]
    out = ref.bench_frames(rm, sel, cam, occ_cfg, opt, keep_last=keep_last)
    return (*out, ref.thread_count())


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    t0 = time.time()
    # untimed warm-up frames (the contract's W >= 3; a reference frame is ~1 s), the last one
    # calibrates the step count so the run stays within budget
    n_warm = max(3, min(args.warmup, 5))
    w_secs, _, threads = reference_frames(n_warm)
    per = float(w_secs[-1])
    budget = float(os.environ.get("ARF_REF_BUDGET_S", "150"))
    k = max(1, min(args.steps, int(budget / max(per, 1e-3))))
    secs, posed, threads = reference_frames(k, frame0=1)
    total = float(secs.sum())
    fps = k / total
    line = {"metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": world, "steps": k, "warmup": n_warm,
            "ms_per_step": 1000.0 * total / k, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": DTYPE, "data": "synthetic (random-init avatar, synthetic poses)",
            "config": bench_config(world), "impl": "reference", "frames_timed": k,
            "posed_samples_per_s": float(posed.sum()) / total,
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{k} full frames (inference grid + render) of the animation, "
                                       f"ARF_THREADS={threads}; workload built by the reference "
                                       "(oracle/workload.py, ref_driver.cpp)"},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.time() - t0}
    if k < args.steps:
        line["note"] = f"reference arm ran {k} of {args.steps} requested steps to stay within {budget:.0f} s"
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1 or args.force_dist_paths:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2212_10550_b200 import arf, fixtures as fx
    from paper_2212_10550_b200._lib import InvalidArgument, call, check, lib

    call("arfx_set_device", local)
    sk = fx.smpl24()
    model = arf.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    poses = fx.animation_poses(sk, N_FRAMES)
    cam = fx.default_camera(sk, W_IMG, H_IMG)
    ccam = cam.to_c()
    opt = fx.config1_render_options()
    copt = opt.to_c()
    occ_cfg = fx.config1_occupancy()
    occ = arf.OccupancyGrid(model.normalized_box, occ_cfg)
    views = [arf.PosedModelView(model, p) for p in poses]
    stream = torch.cuda.Stream()  # a real (non-NULL) stream shared by torch events and libarfx
    torch.cuda.set_stream(stream)
    sp = C.c_void_p(stream.cuda_stream)
    npix = W_IMG * H_IMG
    d_rgb = torch.zeros(npix * 3, dtype=torch.float32, device="cuda")
    d_alpha = torch.zeros(npix, dtype=torch.float32, device="cuda")
    K, Wm = args.steps, args.warmup
    d_cnt = torch.zeros((Wm + K + 2, 2, 4), dtype=torch.int64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2
    L = lib()

    # size the workspace through the synchronous API once (overflow-checked)
    model.set_mlp_mode(args.mlp)
    arf.render_model(model, views[0], cam, occ, opt, rank, world)

    # multi-GPU: each rank builds one cell-interleaved shard of the per-pose occupancy grid,
    # the rank-major blocks are all-gathered over NCCL (1 MiB of f32 values) and every rank
    # permutes them into cell order and re-thresholds / dilates
    shard_grid = (world > 1 or args.force_dist_paths) and not args.no_shard_grid and occ_cfg.resolution ** 3 % world == 0
    if shard_grid:
        from paper_2212_10550_b200.trainer import device_view
        occ_vals = device_view(occ.device_arrays()[0], occ.cell_count())
        slab = occ.cell_count() // world
        my_slab = occ_vals[rank * slab:(rank + 1) * slab]

    def frame_direct(i, slot):
        pstate["next"] = None  # the pipelined graphs' grid A may be overwritten below
        v = views[i % N_FRAMES]
        if shard_grid:
            check(L.arfx_build_inference_grid_shard_device(model._h, v._h, occ._h, rank, world,
                                                           C.c_void_p(d_cnt[slot, 0].data_ptr()), sp))
            dist.all_gather_into_tensor(occ_vals, my_slab)
            check(L.arfx_occ_rebuild_mask_shards_async(occ._h, world, sp))
        else:
            check(L.arfx_build_inference_grid_device(model._h, v._h, occ._h,
                                                     C.c_void_p(d_cnt[slot, 0].data_ptr()), sp))
        check(L.arfx_render_model_device(model._h, v._h, C.byref(ccam), occ._h, C.byref(copt), rank, world,
                                         C.c_void_p(d_rgb.data_ptr()), C.c_void_p(d_alpha.data_ptr()),
                                         C.c_void_p(d_cnt[slot, 1].data_ptr()), sp))

    # CUDA-graph frames: the frame's ~40 launches captured once for one pose handle; each frame
    # copies its (device-resident) pose context into that handle and replays (kernels read the
    # pose from device memory). With grid shards the NCCL all-gather sits between two graphs.
    gview = arf.PosedModelView(model, poses[0])
    g_cnt = torch.zeros((2, 4), dtype=torch.int64, device="cuda")
    # 1 GPU: pipelined frame graphs -- each replay renders frame i with its (already built)
    # grid while building frame i+1's grid on a concurrent branch; two graphs alternate the
    # roles of (pose handle, occupancy grid) A/B. Every frame is still one grid build + one
    # render; only their overlap across consecutive frames changes.
    pipelined = world == 1 and not shard_grid and not args.no_graph and not args.no_pipeline
    # N > 1 (grid shards): the same overlap with the exchange -- frame i+1's grid shard, the
    # all-gather of its blocks and the unshard + mask run on a side stream (side workspace)
    # while frame i renders on the main stream
    pipe_dist = shard_grid and not args.no_graph and not args.no_pipeline
    pv = [gview, arf.PosedModelView(model, poses[0])]
    pocc = [occ, arf.OccupancyGrid(model.normalized_box, occ_cfg)] if (pipelined or pipe_dist) else [occ]
    if pipe_dist:
        side = torch.cuda.Stream()
        ssp = C.c_void_p(side.cuda_stream)
        dvals = [device_view(o.device_arrays()[0], o.cell_count()) for o in pocc]
        dslab = [v[rank * slab:(rank + 1) * slab] for v in dvals]
        s_cnt = torch.zeros((2, 4), dtype=torch.int64, device="cuda")
    pstate = {"phase": 0, "next": None}  # next: the frame whose grid the current handle holds

    def make_graphs():
        hs = []
        if args.no_graph:
            return hs
        if pipelined:
            for ph in range(2):
                h = C.c_void_p()
                check(L.arfx_frame_graph_create_pipelined(
                    model._h, pv[ph]._h, pocc[ph]._h, pv[1 - ph]._h, pocc[1 - ph]._h, C.byref(ccam), C.byref(copt),
                    rank, world, C.c_void_p(d_rgb.data_ptr()), C.c_void_p(d_alpha.data_ptr()),
                    C.c_void_p(g_cnt.data_ptr()), sp, C.byref(h)))
                hs.append(h)
            pstate["next"] = None  # the handles' contents are unknown after a capture's warm-up
            return hs
        if pipe_dist:  # per grid X: shard (side workspace), unshard + mask, render
            for x in range(2):
                for pmask, stream_p, cnt_p in ((2 | 64, ssp, s_cnt), (16, ssp, s_cnt), (8, sp, g_cnt)):
                    h = C.c_void_p()
                    check(L.arfx_frame_graph_create(model._h, pv[x]._h, C.byref(ccam), pocc[x]._h, C.byref(copt), rank,
                                                    world, pmask, C.c_void_p(d_rgb.data_ptr()),
                                                    C.c_void_p(d_alpha.data_ptr()), C.c_void_p(cnt_p.data_ptr()),
                                                    stream_p, C.byref(h)))
                    hs.append(h)
            pstate["next"] = None
            torch.cuda.synchronize()
            return hs
        for pmask in ([2, 16 | 8] if shard_grid else [1 | 8]):
            h = C.c_void_p()
            check(L.arfx_frame_graph_create(model._h, gview._h, C.byref(ccam), occ._h, C.byref(copt), rank, world,
                                            pmask, C.c_void_p(d_rgb.data_ptr()), C.c_void_p(d_alpha.data_ptr()),
                                            C.c_void_p(g_cnt.data_ptr()), sp, C.byref(h)))
            hs.append(h)
        return hs

    graphs = make_graphs()

    recaptures = [0]

    def launch_graph_on(k, stream_p):
        # a graph whose workspace grew since capture is refused by the library (stale pointers):
        # re-capture it (never inside the timed region: the warm-up frames size the workspace)
        nonlocal graphs
        try:
            check(L.arfx_frame_graph_launch(graphs[k], stream_p))
        except InvalidArgument:
            for h in graphs:
                check(L.arfx_frame_graph_destroy(h))
            graphs = make_graphs()
            recaptures[0] += 1
            check(L.arfx_frame_graph_launch(graphs[k], stream_p))

    def launch_graph(k):
        launch_graph_on(k, sp)

    def frame_pipelined(i, slot):
        ph = pstate["phase"]
        if pstate["next"] != i:  # out of sequence (or first frame): build frame i's grid directly
            check(L.arfx_pose_copy(pv[ph]._h, views[i % N_FRAMES]._h, sp))
            check(L.arfx_build_inference_grid_device(model._h, pv[ph]._h, pocc[ph]._h, None, sp))
        check(L.arfx_pose_copy(pv[1 - ph]._h, views[(i + 1) % N_FRAMES]._h, sp))
        launch_graph(ph)  # render i from (pv[ph], pocc[ph]); build i + 1 into (pv[1-ph], pocc[1-ph])
        d_cnt[slot, 1].copy_(g_cnt[1])
        pstate["phase"], pstate["next"] = 1 - ph, i + 1

    def grid_dist(x, i, stream_obj, stream_p, launch):
        """frame i's grid into pocc[x] through graphs: shard, all-gather of the blocks, mask."""
        check(L.arfx_pose_copy(pv[x]._h, views[i % N_FRAMES]._h, stream_p))
        launch(3 * x + 0, stream_p)
        with torch.cuda.stream(stream_obj):
            dist.all_gather_into_tensor(dvals[x], dslab[x])
        launch(3 * x + 1, stream_p)

    def frame_dist_pipelined(i, slot):
        ph = pstate["phase"]
        nx = 1 - ph
        if pstate["next"] != i:  # prime: frame i's grid on the main stream
            grid_dist(ph, i, torch.cuda.current_stream(), sp, launch_graph_on)
        side.wait_stream(torch.cuda.current_stream())  # render i-1 (grid nx) is done with it
        grid_dist(nx, i + 1, side, ssp, launch_graph_on)
        launch_graph_on(3 * ph + 2, sp)  # render frame i with pocc[ph]
        torch.cuda.current_stream().wait_stream(side)
        d_cnt[slot, 1].copy_(g_cnt[1])
        pstate["phase"], pstate["next"] = nx, i + 1

    def frame_graph(i, slot):
        if pipelined:
            return frame_pipelined(i, slot)
        if pipe_dist:
            return frame_dist_pipelined(i, slot)
        # `graphs` is looked up at call time (re-captured for the other decoder below)
        check(L.arfx_pose_copy(gview._h, views[i % N_FRAMES]._h, sp))
        launch_graph(0)
        if shard_grid:
            dist.all_gather_into_tensor(occ_vals, my_slab)
            launch_graph(1)
        d_cnt[slot].copy_(g_cnt)

    def frame(i, slot):
        return frame_graph(i, slot) if graphs else frame_direct(i, slot)

    def timed_frames(k0, n):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        torch.cuda.synchronize()
        for k in range(n):
            flush.zero_()
            evs[k][0].record(stream)
            frame(k0 + k, k0 + k)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        return float(sum(a.elapsed_time(b) for a, b in evs))

    for i in range(Wm):
        frame(i, i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    clocks = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[0])
                          if os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[0].isdigit() else local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for k in range(K):
        flush.zero_()
        ev[k][0].record(stream)
        frame(Wm + k, Wm + k)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    # per-kernel device times (libarfx events around each launch) on an untimed direct pass
    # over the same frames
    check(L.arfx_profile_enable(model._h, 1))
    _ = read_profile(model, L)  # reset
    for k in range(K):
        flush.zero_()
        frame_direct(Wm + k, Wm + K + 1)
    torch.cuda.synchronize()
    prof = read_profile(model, L)
    check(L.arfx_profile_enable(model._h, 0))
    # deterministic work counts of the same K frames (re-run untimed with counters on)
    check(L.arfx_stats_enable(model._h, 1))
    for k in range(K):
        frame_direct(Wm + k, Wm + K)
    torch.cuda.synchronize()
    stats = np.zeros(16, np.uint64)
    check(L.arfx_stats_read(model._h, stats.ctypes.data_as(C.POINTER(C.c_uint64))))
    check(L.arfx_stats_enable(model._h, 0))
    p64, p32 = C.c_double(), C.c_double()
    check(L.arfx_pipe_peaks(C.byref(p64), C.byref(p32)))
    ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(ms))
    cnt = d_cnt.cpu().numpy()
    posed = int(cnt[Wm:Wm + K, 1, 0].sum())
    overflow = int(cnt[:Wm + K, :, 3].sum())
    if overflow:
        raise RuntimeError("workspace overflow during the timed frames")
    t = torch.tensor([total_ms, float(posed)], dtype=torch.float64, device="cuda")
    if world > 1:
        tt = t.clone()
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
        t[1] = tt[1]
    total_ms, posed_all = float(t[0]), float(t[1])
    fps = K / (total_ms / 1000.0)

    # kernel launches per frame, counted by the CUDA profiler (kineto) on 2 untimed frames
    frame(Wm + K + 2, Wm + K)  # (pipelined graphs: prime the sequence outside the count)
    launches_per_frame = count_launches(lambda i: frame(Wm + K + 3 + i, Wm + K), 2)

    # e2e through the host-buffer public API
    e2e = run_e2e(args, model, poses, cam, opt, occ, rank, world, views)

    # CPU baseline (rank 0, N = 1): the reference on the host cores, median of 3 frames after a
    # warm-up; its last frame is compared with the same pose through the timed graph path
    cpu, ref_last, parity = None, None, {}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, ref_last = cpu_baseline()

    def frame_parity(decoder):
        """parity_540: the reference's last CPU-baseline frame vs this arm's frame of the same
        pose through the timed path (graph replay), mask bit-exact + pixel error."""
        if ref_last is None:
            return
        j, (rrgb, ralpha, rmask), rposed = ref_last
        frame(j, Wm + K + 1)
        torch.cuda.synchronize()
        rgb = d_rgb.cpu().numpy().reshape(H_IMG, W_IMG, 3)
        alpha = d_alpha.cpu().numpy().reshape(H_IMG, W_IMG)
        mask = pocc[1 - pstate["phase"]].mask if (pipelined or pipe_dist) else occ.mask  # frame j's grid
        d = np.concatenate([np.abs(rgb - rrgb).ravel(), np.abs(alpha - ralpha).ravel()])
        r = np.concatenate([np.abs(rrgb).ravel(), np.abs(ralpha).ravel()])
        parity[decoder] = {"frame": j, "mask_equal": bool(np.array_equal(mask, rmask)),
                           "mask_cells_differing": int((mask != rmask).sum()),
                           "max_abs": float(d.max()), "max_rel": float((d / np.maximum(r, 1e-6)).max()),
                           "max_rel_where_ref_gt_1e-3": float((d[r > 1e-3] / r[r > 1e-3]).max()),
                           "within_1e-3_rel_plus_1e-5": bool(np.all(d <= 1e-3 * r + 1e-5)),
                           "posed_samples_equal": int(d_cnt[Wm + K + 1, 1, 0]) == rposed}

    frame_parity(args.mlp)

    # the same frames with the other render decoder (exact f32 SIMT MLP vs tcgen05); the
    # decoder is part of the captured graph, so the graphs are re-captured for it
    other = "exact" if args.mlp != "exact" else "tcgen05"
    model.set_mlp_mode(other)
    main_graphs = graphs
    graphs = make_graphs()
    for i in range(2):
        frame(i, i)
    ms_other = timed_frames(Wm, K)
    frame_parity(other)
    for h in graphs:
        check(L.arfx_frame_graph_destroy(h))
    graphs = main_graphs
    if world > 1:
        t2 = torch.tensor([ms_other], dtype=torch.float64, device="cuda")
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        ms_other = float(t2[0])
    model.set_mlp_mode(args.mlp)

    line = None
    if rank == 0:
        peaks, peak_kind = measured_peaks()
        line = {"metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": Wm,
                "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": DTYPE if args.mlp != "exact" else DTYPE_EXACT,
                "data": "synthetic (random-init avatar, synthetic animation poses)",
                "config": bench_config(world),
                "multi_gpu": ("occupancy grid cell-interleaved shards + NCCL all-gather of the rank-major blocks"
                              if shard_grid else
                              ("occupancy grid built redundantly per rank" if world > 1 else "n/a (1 GPU)")),
                "posed_samples_per_s": posed_all / (total_ms / 1000.0),
                "rays_per_s": npix * K / (total_ms / 1000.0),
                "kernels_ms_per_frame": {k: v[0] / K for k, v in prof.items()},
                "clocks": clk, "e2e": e2e,
                "gpu_launches": launches_per_frame * K if launches_per_frame else int(sum(v[1] for v in prof.values())),
                "gpu_launches_per_frame": launches_per_frame,
                "peaks_kind": peak_kind,
                "render_decoder": args.mlp,
                "frame_launch": ("cuda_graph, pipelined: frame i's render || frame i+1's grid build (two graphs "
                                 "alternating pose handles and occupancy grids)" if pipelined else
                                 "cuda_graphs, pipelined: frame i's render || frame i+1's grid shard + NCCL all-gather "
                                 "+ mask on a side stream" if pipe_dist else
                                 "cuda_graph (pose copied into the captured handle per frame)") if graphs else "direct",
                "graph_recaptures_outside_timed_region": recaptures[0],
                "other_decoder": {"mlp": other, "value": K / (ms_other / 1000.0), "ms_per_step": ms_other / K}}
        rays_rank = shard_rows(world, rank) * W_IMG
        dom, per_kernel = roofline(prof, stats, K, rays_rank, opt.samples_per_ray, posed, peaks, peak_kind,
                                   (p64.value, p32.value))
        line["roofline"] = dom
        line["roofline_kernels"] = per_kernel
        if os.environ.get("ARFX_ROOFLINE_MD"):
            Path(os.environ["ARFX_ROOFLINE_MD"]).write_text(roofline_table(per_kernel))
        line["work_counts"] = {"evals": int(stats[0]), "union_bone_visits": int(stats[1]),
                               "newton_steps": int(stats[2]), "starts": int(stats[3]),
                               "exact_prune_tests": int(stats[4]), "field_queries": int(stats[5]),
                               "field_queries_tcgen05": int(stats[6]), "march_samples_tested": int(stats[11]),
                               "frames": K}
        line["pipe_peaks_tflops"] = {"fp64_addmul": p64.value, "fp32_addmul": p32.value}
        if cpu is not None:
            line["cpu_baseline"] = cpu
            line["parity_540"] = dict(parity, tolerance="|d| <= 1e-3 |ref| + 1e-5 per pixel (north_star)",
                                      reference="oracle/_ref arf::build_model_inference_grid + render_model")
        if world == 1 and not args.no_extra:
            line["extra_configs"] = {"correspondence_microbench": bench_microbench(5, not args.no_cpu_baseline),
                                     "train_step_4096": bench_train(model, 50, not args.no_cpu_baseline),
                                     "train_step_full": bench_train_full(200)}
            rk, seq_ms, counts = bench_train_roofline(48, peaks, peak_kind, (p64.value, p32.value))
            tsf = line["extra_configs"]["train_step_full"]
            tsf["roofline_kernels"] = rk
            tsf["roofline_run"] = {"ms_per_step_sequential": seq_ms, "work_counts": counts,
                                   "note": "kernels timed one stream, no cross-step overlap; ms_per_iter above "
                                           "is the pipelined step"}
            if os.environ.get("ARFX_ROOFLINE_MD"):
                with open(os.environ["ARFX_ROOFLINE_MD"], "a") as fh:
                    fh.write("\n## SPEC train step (config 3), sequential\n\n" + roofline_table(rk))
    if (world > 1 or args.force_dist_paths) and not args.no_dp_train:
        # config 5: data-parallel SPEC training over NCCL (reduce-scatter grads, sharded Adam,
        # all-gather params); also run at N = 1 under torchrun with --force-dist-paths
        dp = bench_train_full(50, rank, world, None, args.force_dist_paths)
        if rank == 0:
            line["extra_configs"] = {"train_step_dp": dp}
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def count_launches(fn, n):
    """Kernel launches per call of fn(i), counted with torch.profiler (CUPTI activity) over n calls;
    only libarfx kernels run inside fn. None when the profiler is unavailable."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for i in range(n):
                fn(i)
            torch.cuda.synchronize()
        k = sum(1 for e in prof.events() if getattr(e, "device_type", None) is not None
                and str(e.device_type).endswith("CUDA") and "memset" not in e.name.lower()
                and "memcpy" not in e.name.lower())
        return int(round(k / n))
    except Exception:
        return None


def read_profile(model, L):
    from paper_2212_10550_b200._lib import check
    names = C.create_string_buffer(32 * 32)
    ms = np.zeros(32)
    la = np.zeros(32, np.int64)
    n = C.c_int()
    check(L.arfx_profile_read(model._h, 32, names, ms.ctypes.data_as(C.POINTER(C.c_double)),
                              la.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(n)))
    out = {}
    for k in range(n.value):
        nm = names.raw[32 * k:32 * k + 32].split(b"\0")[0].decode()
        out[nm] = (float(ms[k]), int(la[k]))
    return out


def ncu_traffic():
    """dram bytes per launch from the committed ncu --set full summaries (profiles/)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    return json.loads(p.read_text()) if p.exists() else {}


def roofline(prof, stats, K, rays, N, posed, peaks, peak_kind, pipe):
    """Per-kernel achieved vs bound, algorithmic work per DESIGN.md §4 (Roofline accounting).

    stats (deterministic, summed over the same K frames): evals E, union-bone visits U,
    Newton steps I, starts S, exact prune tests P, field queries Q.
    """
    E, U, I, S, P, Q, QT = (float(x) for x in stats[:7])
    tested = float(stats[11])  # samples march pass 1 tested (occupied-box range)
    fp64_peak, fp32_peak = pipe
    traffic = ncu_traffic()
    out = {}

    def entry(name, bound, work, unit, peak, peak_src, note):
        if name not in prof:
            return
        ms, n = prof[name]
        ach = work / (ms * 1e-3) / (1e12 if unit == "TFLOP/s" else 1e9)
        out[name] = {"kernel": name, "bound": bound, "achieved": ach, "peak": peak, "unit": unit,
                     "frac": ach / peak if peak else None, "ms_per_launch": ms / max(n, 1), "launches": n,
                     "work_per_launch": work / max(n, 1),
                     "traffic": traffic.get(name), "peak_source": peak_src, "work": note}

    f64src = "fp64 add/mul issue roof measured by bench.py (arfx_pipe_peaks; not in MEASURED_PEAKS.json)"
    hbm = peaks.get("hbm_gbs")
    f32src = "fp32 add/mul issue roof measured by bench.py (arfx_pipe_peaks)"
    # K2b deformer: 41/eval + 60/union bone + 66/Newton step + 18/start + 7/rejected line-search candidate
    entry("deform", "fp64", 41 * E + 60 * U + 66 * I + 18 * S + 7 * max(E - S - I, 0.0), "TFLOP/s", fp64_peak,
          f64src, "FP64 add/mul/div/sqrt of inverse_lbs_ctx as written (no FMA)")
    # K3 field: exact MLP 6400 mul + 6400 add + 512 encode accumulations (f32) per query
    entry("field", "fp32", Q * 13312, "TFLOP/s", fp32_peak, f32src, "f32 mul+add of encode+MLP, 13312/query")
    # K3 field on tcgen05: 2*(32*64 + 64*64 + 64*4) = 12800 algorithmic MLP flops per query
    # (the split-bf16 scheme issues 3 MMAs per product and pads the head to N=16: not counted)
    if "encode_tc" in prof:  # two-stage build (ARFX_TC_FUSED=0): the MMA stage streams tiles
        entry("field_tc", "tensor", QT * 12800, "TFLOP/s", peaks.get("bf16_tflops"),
              f"MEASURED_PEAKS.json bf16_tflops ({peak_kind})", "12800 MLP flops/query (algorithmic)")
    else:  # fused encode -> tcgen05 MLP: the hash-table gathers bind, the tensor pipe idles
        entry("field_tc", "l2/l1 gathers", QT * (1024 + 16), "GB/s", hbm,
              f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}); gathers are L2-resident, so frac is vs HBM for scale only",
              "1024 B gathered + 16 B (density, rgb) written per query; + 12800 MLP flops/query (layers 0-1 on tcgen05, the 64->4 head as f32 FMAs)")
        if "field_tc" in out and peaks.get("bf16_tflops"):
            e = out["field_tc"]
            e["tensor_tflops"] = QT * 12800 / (prof["field_tc"][0] * 1e-3) / 1e12
            e["tensor_frac"] = e["tensor_tflops"] / peaks["bf16_tflops"]
    # K3 encode stage of the tcgen05 decoder: 16 levels x 8 corners x 8 B gathered (f32 table)
    # + 128 B of split-bf16 features written per query; the table is L2-resident (64 MiB)
    entry("encode_tc", "l2/l1 gathers", QT * (1024 + 128), "GB/s", hbm,
          f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}); gathers are L2-resident, so frac is vs HBM for scale only",
          "1024 B gathered + 128 B written per query")
    # K1 march: ~80 FP64 per ray + 36 per sample it tests (ray.at, to_normalized, t, cell_of):
    # pass 1 tests only the samples that can reach the occupied box (device counter)
    entry("march", "fp64", rays * K * 80 + 36 * tested, "TFLOP/s", fp64_peak, f64src,
          "80/ray + 36/tested sample FP64 (samples outside the occupied box's range are not tested)")
    # K2a/K2b prune + counting sort: HBM/L2 bytes -- per target x' read (24 B), mask + count
    # written (8 B); per start key + item written, read back, sorted item written (20 B)
    n_targets = posed + 64 ** 3 * K  # render samples + occupancy cells
    entry("prune", "hbm", 32.0 * n_targets + 20.0 * S, "GB/s", hbm, f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
          "32 B/target + 20 B/start (mask/count, sort keys, items); 5 launches incl. 2 single-pass look-back scans (K2a does the resets)")
    # K4 composite: 30 B per posed sample + 24 B per ray (HBM)
    entry("composite", "hbm", 30.0 * posed + 24.0 * rays * K, "GB/s", hbm,
          f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})", "30 B/posed sample + 24 B/ray")
    # K2d finalize: per start its 32-B result read, per pool entry its 36-B canonical root +
    # owner + result slot written, per target 9 B of mask / count / base (HBM)
    entry("finalize", "hbm", 32.0 * S + 36.0 * (Q + QT) + 9.0 * n_targets, "GB/s", hbm,
          f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})", "32 B/start + 36 B/pool entry + 9 B/target")
    dom = max(out.values(), key=lambda e: e["ms_per_launch"] * e["launches"]) if out else None
    return dom, out


def roofline_table(per_kernel) -> str:
    """Markdown table of every kernel group's roofline fraction (profiles/roofline_r1.md)."""
    rows = ["| kernel | bound | achieved | peak | unit | frac | ms/launch | launches | DRAM bytes/launch (ncu) |",
            "|---|---|---|---|---|---|---|---|---|"]
    for k, e in sorted(per_kernel.items(), key=lambda kv: -kv[1]["ms_per_launch"] * kv[1]["launches"]):
        tr = e.get("traffic")
        rows.append(f"| {k} | {e['bound']} | {e['achieved']:.3g} | {e['peak']:.4g} | {e['unit']} | "
                    f"{(e['frac'] or 0):.3f} | {e['ms_per_launch']:.4f} | {e['launches']} | "
                    f"{'-' if tr is None else f'{tr / 1e6:.1f} MB'} |")
    return "\n".join(rows) + "\n"


def run_e2e(args, model, poses, cam, opt, occ, rank, world, views):
    import torch
    from paper_2212_10550_b200 import arf
    from paper_2212_10550_b200._lib import ArfxCounters, check, lib
    L = lib()
    npix = W_IMG * H_IMG
    h_rgb = torch.zeros((H_IMG, W_IMG, 3), dtype=torch.float32).pin_memory().numpy()
    h_alpha = torch.zeros((H_IMG, W_IMG), dtype=torch.float32).pin_memory().numpy()
    out = arf.RenderImages(W_IMG, H_IMG, h_rgb, h_alpha)
    view = arf.PosedModelView(model, poses[0])
    K = max(3, args.steps // 2)
    for i in range(2):
        view.update(poses[i])
        check(L.arfx_build_inference_grid(model._h, view._h, occ._h, None, None))
        arf.render_model(model, view, cam, occ, opt, rank, world, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        view.update(poses[(args.warmup + k) % N_FRAMES])  # host -> device pose
        check(L.arfx_build_inference_grid(model._h, view._h, occ._h, None, None))
        arf.render_model(model, view, cam, occ, opt, rank, world, out=out)  # -> pinned host rgb/alpha
    dt_sync = time.perf_counter() - t0
    # pipelined through the async host-buffer API: per frame the pose H2D (pinned staging),
    # the grid + render on the model stream and the image / counter D2H on the library's copy
    # stream, which overlaps the next frame's kernels; one wait at the end
    outs = [out, arf.RenderImages(W_IMG, H_IMG, torch.zeros((H_IMG, W_IMG, 3), dtype=torch.float32).pin_memory().numpy(),
                                  torch.zeros((H_IMG, W_IMG), dtype=torch.float32).pin_memory().numpy())]
    cnts = torch.zeros((K, 4), dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    for i in range(2):
        view.update(poses[i], sync=False)
        check(L.arfx_build_inference_grid(model._h, view._h, occ._h, None, None))
        arf.render_model_async(model, view, cam, occ, opt, outs[i], cnts[i], rank, world)
    arf.render_wait(model)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        view.update(poses[(args.warmup + k) % N_FRAMES], sync=False)
        check(L.arfx_build_inference_grid(model._h, view._h, occ._h, None, None))
        arf.render_model_async(model, view, cam, occ, opt, outs[k % 2], cnts[k], rank, world)
    arf.render_wait(model)
    dt = time.perf_counter() - t0
    if int(cnts[:, 3].sum()):
        raise RuntimeError("e2e: workspace overflow in the pipelined frames")
    # pipelined through the C-ABI host-buffer call: frame k renders (pose handle k % 2, grid
    # k % 2) into host buffers while frame k+1's grid is built on the side stream
    pvs = [arf.PosedModelView(model, poses[0]), arf.PosedModelView(model, poses[0])]
    from paper_2212_10550_b200 import fixtures as fx
    poccs = [arf.OccupancyGrid(model.normalized_box, fx.config1_occupancy()) for _ in range(2)]
    ccam_p, copt_p = cam.to_c(), opt.to_c()
    cnts_p = torch.zeros((K + 2, 4), dtype=torch.int64).pin_memory().numpy().view(np.uint64)

    def pipe_frames(k0, n, first_pose):
        pvs[k0 & 1].update(poses[first_pose % N_FRAMES], sync=False)
        check(L.arfx_build_inference_grid(model._h, pvs[k0 & 1]._h, poccs[k0 & 1]._h, None, None))
        for k in range(k0, k0 + n):
            cur, nxt = k & 1, (k + 1) & 1
            pvs[nxt].update(poses[(first_pose + k - k0 + 1) % N_FRAMES], sync=False)  # host -> device pose
            check(L.arfx_render_model_pipelined_async(
                model._h, pvs[cur]._h, poccs[cur]._h, pvs[nxt]._h, poccs[nxt]._h, C.byref(ccam_p), C.byref(copt_p),
                rank, world, arf.ptr(outs[k % 2].rgb, C.c_float), arf.ptr(outs[k % 2].alpha, C.c_float),
                cnts_p[k - k0].ctypes.data_as(C.POINTER(C.c_uint64)), None))
        arf.render_wait(model)

    pipe_frames(0, 2, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe_frames(0, K, args.warmup)
    dt_pipe = time.perf_counter() - t0
    if int(cnts_p[:K, 3].sum()):
        raise RuntimeError("e2e: workspace overflow in the pipelined frames")
    # the same loop through the public frame-graph API: two captured frames (grid + render)
    # with their own pose handles and device outputs, replayed alternately after an async
    # pose upload; each replay's RGB/alpha/counters go to pinned host memory on a copy
    # stream while the other graph replays
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    gviews = [arf.PosedModelView(model, poses[0]), arf.PosedModelView(model, poses[1])]
    d_out = [(torch.zeros(W_IMG * H_IMG * 3, dtype=torch.float32, device="cuda"),
              torch.zeros(W_IMG * H_IMG, dtype=torch.float32, device="cuda"),
              torch.zeros(4, dtype=torch.int64, device="cuda")) for _ in range(2)]
    h_out = [(torch.zeros(W_IMG * H_IMG * 3, dtype=torch.float32).pin_memory(),
              torch.zeros(W_IMG * H_IMG, dtype=torch.float32).pin_memory(),
              torch.zeros(4, dtype=torch.int64).pin_memory()) for _ in range(2)]
    h_cnt = torch.zeros((K, 4), dtype=torch.int64).pin_memory()
    ccam, copt = cam.to_c(), opt.to_c()
    graphs = []
    for i in range(2):
        h = C.c_void_p()
        check(L.arfx_frame_graph_create(model._h, gviews[i]._h, C.byref(ccam), occ._h, C.byref(copt), rank, world, 1 | 8,
                                        C.c_void_p(d_out[i][0].data_ptr()), C.c_void_p(d_out[i][1].data_ptr()),
                                        C.c_void_p(d_out[i][2].data_ptr()), sp, C.byref(h)))
        graphs.append(h)
    cs = torch.cuda.Stream()
    ev_done = [torch.cuda.Event(), torch.cuda.Event()]
    ev_copied = [torch.cuda.Event(), torch.cuda.Event()]
    cur = torch.cuda.current_stream()

    def graph_frame(k, pose, cnt_row):
        i = k & 1
        cur.wait_event(ev_copied[i])  # this slot's previous outputs have reached the host
        gviews[i].update(pose, stream=sp, sync=False)
        check(L.arfx_frame_graph_launch(graphs[i], sp))
        ev_done[i].record(cur)
        cs.wait_event(ev_done[i])
        with torch.cuda.stream(cs):
            h_out[i][0].copy_(d_out[i][0], non_blocking=True)
            h_out[i][1].copy_(d_out[i][1], non_blocking=True)
            cnt_row.copy_(d_out[i][2], non_blocking=True)
        ev_copied[i].record(cs)

    for k in range(2):
        graph_frame(k, poses[k], h_cnt[k])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        graph_frame(k, poses[(args.warmup + k) % N_FRAMES], h_cnt[k])
    cs.synchronize()
    torch.cuda.synchronize()
    dt_graph = time.perf_counter() - t0
    for h in graphs:
        check(L.arfx_frame_graph_destroy(h))
    if int(h_cnt[:, 3].sum()):
        raise RuntimeError("e2e: workspace overflow in the graph frames")
    rows = shard_rows(world, rank)
    pose_ctx_bytes = 8 + 32 * (12 + 12 + 3 + 3 + 1) * 8 + 12 * 8 + 32 * 16  # sizeof(PoseCtx), kMaxBones 32
    async_value = K / dt
    graph_value = K / dt_graph
    pipe_value = K / dt_pipe
    # the headline is the reference-facing plugin call with HOST buffers (C-ABI); the
    # frame-graph and synchronous variants are reported beside it
    return {"value": pipe_value, "unit": UNIT, "h2d_bytes_per_step": pose_ctx_bytes,
            "d2h_bytes_per_step": rows * W_IMG * 16 + 32, "steps": K,
            "api": "C-ABI host buffers, pipelined: arfx_pose_update_async + arfx_render_model_pipelined_async "
                   "(frame k renders into pinned host RGB/alpha while frame k+1's inference grid is built on the "
                   "side stream; D2H overlaps the next frame), one arfx_render_wait",
            "pipelined_api_value": pipe_value,
            "async_api_value": async_value,
            "async_api": "arfx_pose_update_async + arfx_build_inference_grid + arfx_render_model_async per frame",
            "sync_api_value": K / dt_sync, "graph_api_value": graph_value,
            "graph_api": "arfx_pose_update_async + arfx_frame_graph_launch (two captured grid + render frames, "
                         "alternating) + D2H of RGB/alpha/counters to pinned host on a copy stream"}


def bench_microbench(steps: int, with_cpu: bool):
    """BASELINE configs[1]: Fast-SNARF correspondence search, 1 M posed points x 9 starts
    (9-bone default figure, 32^3 skinning grid, PoseContext with cutoff_factor 1e30)."""
    import torch
    from paper_2212_10550_b200 import arf, fixtures as fx
    from paper_2212_10550_b200._lib import check, lib
    L = lib()
    sk9 = fx.default_figure_skeleton(9)
    tiny = arf.HashGridConfig(levels=2, features_per_level=2, table_size_log2=10, base_resolution=4, max_resolution=8)
    model = arf.build_model(sk9, tiny, arf.MlpConfig(4, 16, 1, 4), (32, 32, 32), 1)
    pose = fx.microbench_pose(sk9)
    n = 1_000_000
    pts = fx.microbench_points(sk9, pose, n)
    h = C.c_void_p()
    pre = arf.rigid()
    check(L.arfx_pose_create_context(model._h, arf.ptr(pose.bone_transforms, C.c_double), arf.ptr(pre, C.c_double),
                                     1e30, C.byref(h)))
    stream = torch.cuda.current_stream()
    d_pts = torch.from_numpy(pts).cuda()
    d_cnt = torch.zeros(n, dtype=torch.int32, device="cuda")
    d_roots = torch.zeros(n * 8 * 3, dtype=torch.float64, device="cuda")
    d_res = torch.zeros(n * 8, dtype=torch.float64, device="cuda")
    sp = C.c_void_p(stream.cuda_stream)

    def run():
        check(L.arfx_inverse_lbs_device(model._h, h, C.c_void_p(d_pts.data_ptr()), n, C.c_void_p(d_cnt.data_ptr()),
                                        C.c_void_p(d_roots.data_ptr()), C.c_void_p(d_res.data_ptr()), sp))
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    roots = d_cnt.cpu().numpy()
    out = {"workload": "BASELINE configs[1]: 1M posed points x 9 starts, 32^3 skinning grid (9-bone figure)",
           "points_per_s": n / (ms * 1e-3), "starts_per_s": 9 * n / (ms * 1e-3), "ms_per_call": ms,
           "mean_roots_per_point": float(roots.mean())}
    if with_cpu:
        try:
            from oracle.oracle_ctypes import Checker
            ref = Checker("ref")
            rm = ref.build_model(sk9, tiny, arf.MlpConfig(4, 16, 1, 4), (32, 32, 32), 1)
            k = n
            t0 = time.perf_counter()
            rc, _, _ = ref.inverse_lbs(rm, pose.bone_transforms, pre, 1e30, pts[:k])
            dt = time.perf_counter() - t0
            out["cpu_baseline"] = {"points_per_s": k / dt, "cores": ref.thread_count(), "kind": "reference",
                                   "sample": f"all {k} points, arf::inverse_lbs_ctx via parallel_for"}
            out["roots_match_reference"] = bool(np.array_equal(rc, roots[:k]))
        except Exception as e:
            out["cpu_baseline"] = {"unavailable": str(e)}
    L.arfx_pose_destroy(h)
    return out


def bench_train(model, steps: int, with_cpu: bool):
    """BASELINE configs[2]: one training step = 4096 rays fwd+bwd through deformer / hash grid /
    MLP / compositing (stratified, training grid after one update over 8 poses), through the
    public host API (pixels + upstream gradients in, rgb/alpha out, grads on the device)."""
    import torch
    from paper_2212_10550_b200 import arf, fixtures as fx
    sk = fx.smpl24()
    cam = fx.default_camera(sk, W_IMG, H_IMG)
    poses = [fx.random_pose(sk, 100 + i) for i in range(8)]
    grid = arf.OccupancyGrid(model.normalized_box, fx.config1_occupancy())
    arf.update_training_grid(model, grid, poses, 0.95, 7, 0)
    rng = fx.keyed_rng(9, 1)
    n = 4096
    px = np.empty(n, np.int32)
    py = np.empty(n, np.int32)
    for k in range(n):
        px[k] = rng.next_below(W_IMG)
        py[k] = rng.next_below(H_IMG)
    opt = arf.RenderOptions(samples_per_ray=128, stratified=True, seed=3, frame_id=0)
    dC = np.ones((n, 3), np.float32)
    dA = np.ones(n, np.float32)
    view = arf.PosedModelView(model, poses[0])
    for i in range(2):
        model.zero_grad()
        arf.train_fwd_bwd(model, view, cam, grid, opt, px, py, dC, dA)
    torch.cuda.synchronize()
    c0 = model.counters.posed_queries
    t0 = time.perf_counter()
    for i in range(steps):
        view.update(poses[i % 8])
        model.zero_grad()
        arf.train_fwd_bwd(model, view, cam, grid, opt, px, py, dC, dA)
    dt = time.perf_counter() - t0
    posed = model.counters.posed_queries - c0
    out = {"workload": "BASELINE configs[2]: 4096-ray training step (fwd+bwd, zero-grad included; no optimizer, "
                       "as in the reference composition)", "iters_per_s": steps / dt, "ms_per_iter": 1000 * dt / steps,
           "posed_samples_per_iter": posed / steps}
    if with_cpu:
        try:
            from oracle.oracle_ctypes import Checker
            ref = Checker("ref")
            rm = ref.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
            rg = ref.occ_empty(rm.norm_lo[:], rm.norm_hi[:], fx.config1_occupancy())
            ref.update_training_grid(rm, [p.bone_transforms for p in poses], [p.global_transform for p in poses],
                                     0.95, 7, 0, rg)
            t0 = time.perf_counter()
            ref.train_fwd_bwd(rm, poses[0].bone_transforms, poses[0].global_transform, cam, rg, opt, px, py, dC, dA)
            dt = time.perf_counter() - t0
            out["cpu_baseline"] = {"iters_per_s": 1.0 / dt, "cores": 1, "kind": "reference",
                                   "sample": "1 step of the reference pieces composed serially (oracle/ref_driver.cpp)"}
        except Exception as e:
            out["cpu_baseline"] = {"unavailable": str(e)}
    return out


def bench_train_full(steps: int, rank: int = 0, world: int = 1, group=None, force_collectives: bool = False):
    """SPEC train_step at config 3 (config 5 when world > 1: 4096 rays per rank, weak scaling):
    rays + ground truth gathered on the device, forward + fused losses + backward
    (arfx_train_step_device), reduce-scatter / sharded Adam / all-gather of the flat vectors over
    NCCL (world > 1), Adam with fused zero-grad, occupancy update every 16 steps. Ground truth:
    8 frames of the analytic smpl24 figure rendered at 4x N by arfx_figure_render. Device-timed
    with CUDA events on the step stream; max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2212_10550_b200 import arf, fixtures as fx
    from paper_2212_10550_b200.trainer import Trainer, TrainConfig
    sk = fx.smpl24()
    model = arf.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    cam = fx.default_camera(sk, W_IMG, H_IMG)
    poses = [fx.random_pose(sk, 100 + i) for i in range(8)]
    cfg = TrainConfig(iterations=steps, rays_per_batch=4096 * world, samples_per_ray=128, occupancy_interval=16,
                      seed=9, adam=arf.AdamConfig(total_steps=1000))
    tr = Trainer(model, fx.figure_for(sk), poses, cam, cfg, rank, world, group, force_collectives)
    # warm-up through the first occupancy update too (its one-time workspace sizing is not
    # a per-step cost)
    for _ in range(cfg.occupancy_interval + 3):
        tr.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(group)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0 = model.counters.posed_queries
    e0.record(tr.stream)  # the trainer's stream carries every step
    for _ in range(steps):
        tr.step()
    e1.record(tr.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        ms = float(t[0])
    h = np.array(tr.history)
    return {"workload": f"SPEC train_step, config {'5' if world > 1 else '3'}: 4096 rays/rank x {world} rank(s), "
                        "fwd + fused losses + bwd + Adam (+ occupancy update every 16 steps)"
                        + (", grads reduce-scatter + params all-gather over NCCL on the Adam stream (pipelined)"
                           if world > 1 or force_collectives else ""),
            "iters_per_s": steps / (ms / 1000.0), "ms_per_iter": ms / steps, "rays_per_s": 4096 * world * steps /
            (ms / 1000.0), "n_flat_params": tr.n_flat, "loss_first": h[0].tolist(), "loss_last": h[-1].tolist(),
            "posed_samples_per_iter_rank0": (model.counters.posed_queries - c0) / steps}


def bench_train_roofline(steps: int, peaks, peak_kind, pipe):
    """Per-kernel roofline of the SPEC train step (config 3): the step run sequentially on one
    stream (no cross-step pipelining, density step unfused) so each kernel group's CUDA-event
    time is its own; algorithmic work from the deterministic device counters of the same steps
    (DESIGN.md §4). Returns {kernel: roofline entry} and the sequential ms/step."""
    import torch
    from paper_2212_10550_b200 import arf, fixtures as fx
    from paper_2212_10550_b200._lib import check, lib
    from paper_2212_10550_b200.trainer import Trainer, TrainConfig
    L = lib()
    sk = fx.smpl24()
    model = arf.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    cam = fx.default_camera(sk, W_IMG, H_IMG)
    poses = [fx.random_pose(sk, 100 + i) for i in range(8)]
    cfg = TrainConfig(iterations=steps, rays_per_batch=4096, samples_per_ray=128, occupancy_interval=16,
                      seed=9, adam=arf.AdamConfig(total_steps=1000))
    tr = Trainer(model, fx.figure_for(sk), poses, cam, cfg)
    tr.pipelined = False
    tr.fused_density = False
    for _ in range(cfg.occupancy_interval + 3):
        tr.step()
    torch.cuda.synchronize()
    check(L.arfx_profile_enable(model._h, 1))
    _ = read_profile(model, L)
    check(L.arfx_stats_enable(model._h, 1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(tr.stream)
    for _ in range(steps):
        tr.step()
    e1.record(tr.stream)
    torch.cuda.synchronize()
    prof = read_profile(model, L)
    stats = np.zeros(16, np.uint64)
    check(L.arfx_stats_read(model._h, stats.ctypes.data_as(C.POINTER(C.c_uint64))))
    check(L.arfx_stats_enable(model._h, 0))
    check(L.arfx_profile_enable(model._h, 0))
    tr.close()
    E, U, I, S, P, Q, _, B, PS, R, NP = (float(x) for x in stats[:11])
    fp64_peak, fp32_peak = pipe
    hbm = peaks.get("hbm_gbs")
    f64src = "fp64 add/mul issue roof measured by bench.py (arfx_pipe_peaks; not in MEASURED_PEAKS.json)"
    f32src = "fp32 add/mul issue roof measured by bench.py (arfx_pipe_peaks)"
    hsrc = f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"
    n_upd = sum(1 for t in range(cfg.occupancy_interval + 3, cfg.occupancy_interval + 3 + steps)
                if (t + 1) % cfg.occupancy_interval == 0)
    targets = PS + steps * cfg.density_points + n_upd * 64 ** 3
    out = {}

    def entry(name, bound, work, unit, peak, src, note):
        if name not in prof:
            return
        ms, n = prof[name]
        ach = work / (ms * 1e-3) / (1e12 if unit == "TFLOP/s" else 1e9)
        out[name] = {"kernel": name, "bound": bound, "achieved": ach, "peak": peak, "unit": unit,
                     "frac": ach / peak if peak else None, "ms_per_launch": ms / max(n, 1), "launches": n,
                     "ms_per_step": ms / steps, "work_per_launch": work / max(n, 1), "peak_source": src, "work": note}

    TS = float(stats[11])
    entry("march", "fp64", R * 80 + 36 * TS, "TFLOP/s", fp64_peak, f64src, "80/ray + 36/tested sample FP64")
    entry("prune", "hbm", 32.0 * targets + 20.0 * S, "GB/s", hbm, hsrc, "32 B/target + 20 B/start")
    entry("deform", "fp64", 41 * E + 60 * U + 66 * I + 18 * S + 7 * max(E - S - I, 0.0), "TFLOP/s", fp64_peak, f64src,
          "FP64 add/mul/div/sqrt of inverse_lbs_ctx as written (no FMA)")
    entry("finalize", "hbm", 32.0 * S + 36.0 * Q + 9.0 * targets, "GB/s", hbm, hsrc,
          "32 B/start + 36 B/pool entry + 9 B/target")
    entry("field", "fp32", 13312.0 * Q, "TFLOP/s", fp32_peak, f32src, "exact f32 encode + MLP, 13312 flops/query")
    entry("train_composite", "hbm", 56.0 * PS + 40.0 * R, "GB/s", hbm, hsrc,
          "56 B/posed sample (field result, delta, index, root slot, transmittance, dsigma/dcolor) + 40 B/ray")
    entry("bwd_list", "hbm", 5.0 * Q + 4.0 * B, "GB/s", hbm, hsrc, "1 B flag + 4 B per pool entry, 4 B per list entry")
    entry("bwd_field", "fp32", 13056.0 * B, "TFLOP/s", fp32_peak, f32src,
          "MLP dX chain 12800 + encode-backward weights 256 f32 flops per backward query")
    entry("bwd_weights", "fp32", 13064.0 * B, "TFLOP/s", fp32_peak, f32src, "dW + db: 2 x 6532 f32 flops per query")
    entry("bwd_scatter", "l2 atomics", 1024.0 * B, "GB/s", hbm, hsrc + "; L2 atomics, vs HBM for scale",
          "16 levels x 8 corners x float2 atomic (8 B) per query")
    entry("adam", "hbm", 32.0 * NP, "GB/s", hbm, hsrc, "p, g, m, v read + p, m, v, g written: 32 B/param")
    return out, e0.elapsed_time(e1) / steps, {"evals": int(E), "starts": int(S), "field_queries": int(Q),
                                              "backward_queries": int(B), "posed_samples": int(PS), "rays": int(R),
                                              "adam_params": int(NP), "steps": steps}


def cpu_baseline():
    """The reference on this host's cores: 1 warm-up frame then the median of 3 (BASELINE.md §3,
    SURVEY.md §8d); returns (cpu_baseline dict, (pose index, last frame's rgb/alpha/mask), posed)."""
    try:
        secs, posed, last, threads = reference_frames(4, keep_last=True)
        med = float(np.median(secs[1:]))
        return ({"value": 1.0 / med, "unit": UNIT, "cores": threads, "kind": "reference",
                 "sample": "median of 3 full frames (inference grid + render; poses 1-3) after 1 warm-up frame, "
                           "reference compiled from /root/reference with -O3 -ffp-contract=off, "
                           f"ARF_THREADS={threads}", "frame_seconds": [float(x) for x in secs[1:]],
                 "posed_samples_per_s": float(np.median(posed[1:] / secs[1:]))}, (3, last, int(posed[3])))
    except Exception as e:  # the checker is test infrastructure; report, do not fail the bench
        return {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": f"unavailable: {e}"}, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100, help="timed frames (default: the 100-frame animation)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mlp", default="tcgen05", choices=["tcgen05", "tcgen05_fp16", "exact"],
                    help="render decoder for `value` (the other one is reported as other_decoder)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-dist-paths", action="store_true",
                    help="exercise the multi-GPU code paths (grid all-gather, DP train) at N = 1 under torchrun")
    ap.add_argument("--no-graph", action="store_true", help="launch each frame's kernels directly (no CUDA graph)")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="1 GPU: one grid + render graph per frame instead of overlapping frame i+1's grid build "
                         "with frame i's render")
    ap.add_argument("--no-shard-grid", action="store_true",
                    help="N > 1: build the occupancy grid redundantly on every rank instead of cell-interleaved shards")
    ap.add_argument("--no-dp-train", action="store_true",
                    help="N > 1: skip the data-parallel SPEC train step side measurement (config 5)")
    ap.add_argument("--no-extra", action="store_true", help="skip the config-2/3 side measurements")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun (127.0.0.1 rendezvous)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
        return subprocess.call(cmd)
    if world_env is not None and int(world_env) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
