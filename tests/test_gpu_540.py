"""Headline-configuration parity (BASELINE configs[0]/[3], north_star target): 540x540
novel-pose frames of the config-1 avatar rendered through exactly the path bench.py times
-- one CUDA-graph replay per frame (inference grid + render, pose copied into the captured
handle), the thread-per-ray march pass 1 with the occupied-box sample range (full-warp
launch at 291,600 rays), the K2 start pipeline and both render decoders -- against the
UNMODIFIED reference's build_model_inference_grid + render_model (R/model.hpp:118-148,
compiled in place as oracle/_ref).

Bars: occupancy mask bit-exact; posed-sample set (pixel, sample index),
deltas and has_root bit-exact vs the reference's traced render loop (which reproduces
arf::render_model bit for bit, asserted below); pixels |d| <= 1e-3 |ref| + 1e-5 for the
tcgen05 split-bf16 decoder and |d| <= 1e-6 |ref| + 1e-6 for the exact f32 decoder."""
import ctypes as C

import numpy as np
import pytest

from paper_2212_10550_b200 import arf, fixtures as fx

pytestmark = pytest.mark.gpu

W = H = 540
FRAMES = (0, 41, 83)          # three of the 100 animation poses (bench.py's workload)
TC_RTOL, TC_ATOL = 1e-3, 1e-5  # north_star: 1e-3 relative on rendered RGB
EX_RTOL, EX_ATOL = 1e-6, 1e-6  # exact f32 decoder: expf/log1pf ulps only


@pytest.fixture(scope="module")
def headline(gpu, ref):
    import torch
    from paper_2212_10550_b200._lib import call
    sk = fx.smpl24()
    dm = gpu.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    rm = ref.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    poses = fx.animation_poses(sk, 100)
    cam = fx.default_camera(sk, W, H)
    opt = fx.config1_render_options()
    occ_cfg = fx.config1_occupancy()
    # the reference frames (parallel render_model; the mask from build_model_inference_grid)
    want = {}
    for f in FRAMES:
        p = poses[f]
        rocc, _ = ref.build_inference_grid(rm, p.bone_transforms, p.global_transform, occ_cfg)
        rgb, alpha, cnt = ref.render(rm, p.bone_transforms, p.global_transform, cam, rocc, opt)
        want[f] = (rocc, ref.occ_arrays(rocc)[1].copy(), rgb, alpha, cnt)
    # the bench's graph frame
    occ = arf.OccupancyGrid(dm.normalized_box, occ_cfg)
    views = {f: arf.PosedModelView(dm, poses[f]) for f in FRAMES}
    gview = arf.PosedModelView(dm, poses[0])
    st = torch.cuda.Stream()
    sp = C.c_void_p(st.cuda_stream)
    d_rgb = torch.zeros(W * H * 3, device="cuda")
    d_alpha = torch.zeros(W * H, device="cuda")
    d_cnt = torch.zeros((2, 4), dtype=torch.int64, device="cuda")
    ccam, copt = cam.to_c(), opt.to_c()
    # size the workspace once through the synchronous (overflow-checked) API, as bench.py does
    arf.render_model(dm, views[FRAMES[0]], cam, arf.build_model_inference_grid(dm, poses[FRAMES[0]], occ_cfg), opt)

    def frames(mode):
        dm.set_mlp_mode(mode)
        g = C.c_void_p()
        call("arfx_frame_graph_create", dm._h, gview._h, C.byref(ccam), occ._h, C.byref(copt), 0, 1, 1 | 8,
             C.c_void_p(d_rgb.data_ptr()), C.c_void_p(d_alpha.data_ptr()), C.c_void_p(d_cnt.data_ptr()), sp,
             C.byref(g))
        out = {}
        try:
            for f in FRAMES:
                call("arfx_pose_copy", gview._h, views[f]._h, sp)
                call("arfx_frame_graph_launch", g, sp)
                st.synchronize()
                cnt = d_cnt.cpu().numpy()
                assert cnt[:, 3].sum() == 0, "workspace overflow in a replayed frame"
                tr = arf.render_trace(dm) if mode == "exact" or f == FRAMES[0] else None
                out[f] = (occ.mask.copy(), d_rgb.cpu().numpy().reshape(H, W, 3),
                          d_alpha.cpu().numpy().reshape(H, W), cnt.copy(), tr)
        finally:
            call("arfx_frame_graph_destroy", g)
            dm.set_mlp_mode("exact")
        return out

    got = {"tcgen05": frames("tcgen05"), "exact": frames("exact")}
    return dict(sk=sk, dm=dm, rm=rm, poses=poses, cam=cam, opt=opt, want=want, got=got)


@pytest.mark.parametrize("frame", FRAMES)
def test_540_inference_mask_bit_exact(headline, frame):
    rocc, rmask, _, _, _ = headline["want"][frame]
    for mode in ("tcgen05", "exact"):
        mask = headline["got"][mode][frame][0]
        assert np.array_equal(mask, rmask), (mode, int((mask != rmask).sum()))
    assert 0.01 < rmask.mean() < 0.2


@pytest.mark.parametrize("mode", ["tcgen05", "exact"])
@pytest.mark.parametrize("frame", FRAMES)
def test_540_pixels(headline, frame, mode):
    _, _, rrgb, ralpha, rcnt = headline["want"][frame]
    _, rgb, alpha, cnt, _ = headline["got"][mode][frame]
    rtol, atol = (TC_RTOL, TC_ATOL) if mode == "tcgen05" else (EX_RTOL, EX_ATOL)
    assert (ralpha > 0).sum() > 50_000  # a real 540^2 frame, not an empty one
    np.testing.assert_allclose(rgb, rrgb, rtol=rtol, atol=atol)
    np.testing.assert_allclose(alpha, ralpha, rtol=rtol, atol=atol)
    # QueryCounters::posed_queries (R/model.hpp:102) == occupied samples: exact
    assert int(cnt[1, 0]) == int(rcnt[0])


@pytest.mark.parametrize("frame", FRAMES)
def test_540_sample_set_bit_exact(headline, ref, frame):
    """The traced reference loop at 540^2 (serial, ~13 s/frame): the posed-sample set the
    thread-per-ray march emits, with its deltas and has_root, is bit-exact; the selected
    canonical root follows the near-tie rule of test_gpu_parity.test_render_trace_parity."""
    h = headline
    p = h["poses"][frame]
    rocc, _, rrgb, ralpha, _ = h["want"][frame]
    rrgb2, ralpha2, _, rtr = ref.render_trace(h["rm"], p.bone_transforms, p.global_transform, h["cam"], rocc,
                                              h["opt"], capacity=4_000_000)
    assert np.array_equal(rrgb2, rrgb) and np.array_equal(ralpha2, ralpha)  # trace == arf::render_model
    tr = h["got"]["exact"][frame][4]
    n = rtr["n_samples"]
    assert n > 1_000_000 and len(tr.ray) == n
    order = np.lexsort((tr.index, tr.ray))
    assert np.array_equal(tr.ray[order], rtr["s_ray"])
    assert np.array_equal(tr.index[order], rtr["s_index"])
    assert np.array_equal(tr.delta[order].view(np.uint64), rtr["s_delta"].view(np.uint64))
    assert np.array_equal(tr.has_root[order], rtr["s_has_root"])
    can, rcan = tr.canonical[order], rtr["s_canonical"]
    flip = np.any(can.view(np.uint64) != rcan.view(np.uint64), axis=1)
    assert flip.sum() <= max(1, 1e-4 * n), flip.sum()
    d_o, d_r = tr.density[order][flip], rtr["s_density"][flip]
    assert np.all(np.abs(d_o - d_r) <= 4 * np.spacing(np.maximum(np.abs(d_o), np.abs(d_r))))
    np.testing.assert_allclose(tr.density[order], rtr["s_density"], rtol=2e-6, atol=1e-7)
    if frame == FRAMES[0]:
        # the tcgen05 frame emits the same sample set (the decoder only changes field values)
        ttr = h["got"]["tcgen05"][frame][4]
        o2 = np.lexsort((ttr.index, ttr.ray))
        assert np.array_equal(ttr.ray[o2], rtr["s_ray"]) and np.array_equal(ttr.index[o2], rtr["s_index"])
        np.testing.assert_allclose(ttr.density[o2], rtr["s_density"], rtol=1e-3, atol=1e-4)


@pytest.mark.parametrize("mode", ["tcgen05", "exact"])
def test_stratified_thread_per_ray_frame(gpu, ref, mode):
    """Stratified sampling through the thread-per-ray march (400x400 = 160,000 rays >= the
    full-warp threshold, so each lane walks its own ray's keyed PCG jitter stream,
    R/render.hpp:201) on a pose outside the benched set, both decoders, against the
    reference's render_model with the same seed / frame id."""
    sk = fx.smpl24()
    dm = gpu.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    rm = ref.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    pose = fx.random_pose(sk, 4242)
    cam = fx.default_camera(sk, 400, 400)
    opt = arf.RenderOptions(samples_per_ray=128, stratified=True, seed=11, frame_id=3)
    occ_cfg = fx.config1_occupancy()
    rocc, _ = ref.build_inference_grid(rm, pose.bone_transforms, pose.global_transform, occ_cfg)
    rrgb, ralpha, rcnt = ref.render(rm, pose.bone_transforms, pose.global_transform, cam, rocc, opt)
    dm.set_mlp_mode(mode)
    try:
        occ = arf.build_model_inference_grid(dm, pose, occ_cfg)
        assert np.array_equal(occ.mask, ref.occ_arrays(rocc)[1])
        c0 = dm.counters.posed_queries
        img = arf.render_model(dm, arf.PosedModelView(dm, pose), cam, occ, opt)
        posed = dm.counters.posed_queries - c0
    finally:
        dm.set_mlp_mode("exact")
    rtol, atol = (TC_RTOL, TC_ATOL) if mode == "tcgen05" else (EX_RTOL, EX_ATOL)
    assert (ralpha > 0).sum() > 20_000
    np.testing.assert_allclose(img.rgb, rrgb, rtol=rtol, atol=atol)
    np.testing.assert_allclose(img.alpha, ralpha, rtol=rtol, atol=atol)
    assert posed == int(rcnt[0])
