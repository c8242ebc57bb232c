"""GPU edge cases against the reference (oracle/_ref): empty and degenerate inputs, the
maximum sizes libarfx accepts, skeleton extremes, no early termination."""
import math

import numpy as np
import pytest

from paper_2212_10550_b200 import arf, fixtures as fx

pytestmark = pytest.mark.gpu

PIX = dict(rtol=1e-3, atol=1e-5)


def small_grid(levels=16, T=14):
    return arf.HashGridConfig(levels=levels, features_per_level=2, table_size_log2=T, base_resolution=4,
                              max_resolution=96)


def pair(gpu, ref, sk, seed=3, skin=(12, 12, 12), levels=16):
    g, m = small_grid(levels), arf.MlpConfig(2 * levels, 64, 2, 4)
    return gpu.build_model(sk, g, m, skin, seed), ref.build_model(sk, g, m, skin, seed)


def render_both(ref, dm, rm, pose, cam, occ_cfg, opt):
    if occ_cfg is not None:
        occ = arf.build_model_inference_grid(dm, pose, occ_cfg)
        rocc, _ = ref.build_inference_grid(rm, pose.bone_transforms, pose.global_transform, occ_cfg)
    else:
        occ, rocc = None, None
    before = dm.counters.posed_queries
    img = arf.render_model(dm, pose, cam, occ, opt)
    rrgb, ralpha, rcnt = ref.render(rm, pose.bone_transforms, pose.global_transform, cam, rocc, opt)
    img.posed_queries = dm.counters.posed_queries - before  # this render only
    return img, rrgb, ralpha, rcnt


def test_camera_missing_the_box(gpu, ref):
    sk = fx.default_figure_skeleton()
    dm, rm = pair(gpu, ref, sk)
    pose = arf.pose_from_joint_rotations(sk, fx.bend_pose_rotations(10, 0.2, 0.1))
    # looking away from the figure: every ray misses the normalized box
    cam = arf.Camera.look_at((0.0, 1.0, -3.2), (0.0, 1.0, -10.0), (0.0, 1.0, 0.0), 40.0, 24, 20)
    img, rrgb, ralpha, rcnt = render_both(ref, dm, rm, pose, cam, arf.OccupancyConfig(), arf.RenderOptions())
    assert np.all(img.rgb == 0) and np.all(img.alpha == 0)
    assert np.all(rrgb == 0) and np.all(ralpha == 0) and int(rcnt[0]) == 0


@pytest.mark.parametrize("n", [1, 2, 1024])
def test_samples_per_ray_extremes(gpu, ref, n):
    sk = fx.default_figure_skeleton()
    dm, rm = pair(gpu, ref, sk)
    pose = arf.pose_from_joint_rotations(sk, fx.bend_pose_rotations(10, 0.3, 0.2), fx.yaw_about(sk.bones[0].head, 0.4))
    cam = fx.default_camera(sk, 20, 18)
    opt = arf.RenderOptions(samples_per_ray=n, stratified=n != 1, seed=7)
    img, rrgb, ralpha, rcnt = render_both(ref, dm, rm, pose, cam, arf.OccupancyConfig(), opt)
    np.testing.assert_allclose(img.rgb, rrgb, **PIX)
    np.testing.assert_allclose(img.alpha, ralpha, **PIX)


def test_samples_per_ray_over_limit_is_invalid(gpu):
    sk = fx.default_figure_skeleton()
    dm = gpu.build_model(sk, small_grid(), arf.MlpConfig(32, 64, 2, 4), (8, 8, 8), 1)
    pose = arf.SkeletonPose.identity(10)
    with pytest.raises(ValueError):
        arf.render_model(dm, pose, fx.default_camera(sk, 8, 8), None, arf.RenderOptions(samples_per_ray=1025))


def test_no_early_termination(gpu, ref):
    sk = fx.default_figure_skeleton()
    dm, rm = pair(gpu, ref, sk)
    gp, mp, _ = ref.arrays(rm)
    rng = np.random.default_rng(0)
    gp[:] = rng.uniform(-1, 1, gp.size).astype(np.float32)
    mp[:] = rng.uniform(-0.5, 0.5, mp.size).astype(np.float32) + 0.05
    dm.set_params(gp, mp)
    pose = arf.pose_from_joint_rotations(sk, fx.bend_pose_rotations(10, 0.3, 0.2))
    cam = fx.default_camera(sk, 24, 24)
    for eps in (0.0, 0.5):
        opt = arf.RenderOptions(samples_per_ray=64, epsilon_terminate=eps)
        img, rrgb, ralpha, _ = render_both(ref, dm, rm, pose, cam, None, opt)
        np.testing.assert_allclose(img.rgb, rrgb, **PIX)
        np.testing.assert_allclose(img.alpha, ralpha, **PIX)


def test_single_bone_skeleton(gpu, ref):
    sk = arf.Skeleton([arf.Bone(-1, (0.0, 0.5, 0.0), (0.0, 1.3, 0.0), 0.15)])
    dm, rm = pair(gpu, ref, sk, skin=(8, 8, 8))
    assert np.array_equal(dm.params()[2].view(np.uint64), ref.arrays(rm)[2].view(np.uint64))
    pose = arf.pose_from_joint_rotations(sk, [fx.IDENTITY9], fx.yaw_about((0.0, 0.5, 0.0), 0.7))
    cam = fx.default_camera(sk, 24, 24)
    img, rrgb, ralpha, rcnt = render_both(ref, dm, rm, pose, cam, arf.OccupancyConfig(), arf.RenderOptions())
    np.testing.assert_allclose(img.rgb, rrgb, **PIX)
    assert img.posed_queries == int(rcnt[0]) > 0


def test_max_bones_chain(gpu, ref):
    """32 bones (kMaxBones), a zig-zag chain: start masks use all 32 bits."""
    bones = []
    y = 0.2
    for i in range(32):
        x = 0.04 * (1 if i % 2 else -1)
        bones.append(arf.Bone(i - 1, (x, y, 0.0), (-x, y + 0.05, 0.0), 0.03))
        y += 0.05
    sk = arf.Skeleton(bones)
    dm, rm = pair(gpu, ref, sk, skin=(10, 10, 10), levels=16)
    assert np.array_equal(dm.params()[2].view(np.uint64), ref.arrays(rm)[2].view(np.uint64))
    rots = np.tile(fx.IDENTITY9, (32, 1))
    for i in range(1, 32, 3):
        rots[i] = fx.rot_z(0.05 * (i % 5 - 2))
    pose = arf.pose_from_joint_rotations(sk, rots)
    rng = np.random.default_rng(3)
    pts = np.column_stack([rng.uniform(-0.15, 0.15, 3000), rng.uniform(0.2, 1.9, 3000), rng.uniform(-0.05, 0.05, 3000)])
    c, r, res = dm.inverse_lbs(pose, pts)
    rc, rr, rres = ref.inverse_lbs(rm, pose.bone_transforms, fx.IDENTITY9.tolist() + [0, 0, 0], 3.0, pts)
    assert np.array_equal(c, rc)
    assert np.array_equal(r.view(np.uint64), rr.view(np.uint64))
    with pytest.raises(ValueError):
        arf.Skeleton(bones + [arf.Bone(31, (0, 2.0, 0), (0, 2.1, 0), 0.03)]).to_c()


def test_empty_batches(gpu):
    sk = fx.default_figure_skeleton()
    dm = gpu.build_model(sk, small_grid(), arf.MlpConfig(32, 64, 2, 4), (8, 8, 8), 2)
    pose = arf.SkeletonPose.identity(10)
    z = np.zeros((0, 3))
    c, r, res = dm.inverse_lbs(pose, z)
    assert c.shape == (0,)
    d, col = dm.field_query(z)
    assert d.shape == (0,)
    dm.zero_grad()
    rgb, a = arf.train_fwd_bwd(dm, pose, fx.default_camera(sk, 8, 8), None, arf.RenderOptions(),
                               np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 3)), np.zeros(0))
    assert rgb.shape == (0, 3)
    gg, gm = dm.grads()
    assert not gg.any() and not gm.any()
    l4, dr, da = arf.losses(np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)), np.zeros(0), arf.LossConfig())
    assert np.all(l4 == 0)


def test_all_empty_occupancy_renders_black(gpu):
    sk = fx.default_figure_skeleton()
    dm = gpu.build_model(sk, small_grid(), arf.MlpConfig(32, 64, 2, 4), (8, 8, 8), 4)
    occ = arf.OccupancyGrid(dm.normalized_box, arf.OccupancyConfig())  # empty grid: nothing occupied
    before = dm.counters.posed_queries
    img = arf.render_model(dm, arf.SkeletonPose.identity(10), fx.default_camera(sk, 32, 32), occ, arf.RenderOptions())
    assert np.all(img.rgb == 0) and np.all(img.alpha == 0)
    assert dm.counters.posed_queries == before
