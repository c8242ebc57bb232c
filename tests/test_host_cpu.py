"""CPU tests of libarfx's host side (no GPU needed): the C-ABI library loads and exports
every symbol include/arfx.h declares; host setup (FK, camera, pose context, level
schedule) is bit-identical to the reference; errors map to the reference's exception
types; compute entry points refuse to run without a GPU (no CPU fallback)."""
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2212_10550_b200 as pkg
from paper_2212_10550_b200 import _lib, arf, fixtures as fx

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "arfx.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(arfx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) > 40
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # and the Python binding declares prototypes for all of them
    assert sorted(_lib.exported_symbols()) == syms


def test_level_resolutions_host(ref):
    for g in (fx.config1_grid(), arf.HashGridConfig(levels=4, base_resolution=16, max_resolution=128),
              arf.HashGridConfig(levels=1, base_resolution=8, max_resolution=8),
              arf.HashGridConfig(levels=7, base_resolution=3, max_resolution=1000)):
        assert arf.level_resolutions(g) == ref.level_resolutions(g)


def test_pose_and_camera_host_bit_exact(ref):
    sk = fx.smpl24()
    pose = fx.random_pose(sk, 42)
    rng = fx.keyed_rng(42, 7)
    import math
    rots = [fx.IDENTITY9.copy()]
    for _ in range(1, 24):
        ax, ay, az, ang = rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-0.5, 0.5)
        n = math.sqrt(ax * ax + ay * ay + az * az)
        rots.append(fx.axis_angle((ax / n, ay / n, az / n), ang))
    rb = ref.pose_from_joint_rotations(sk, np.stack(rots), fx.yaw_about(sk.bones[0].head, 0.3))
    assert np.array_equal(pose.bone_transforms.view(np.uint64), rb.view(np.uint64))
    cam = fx.default_camera(sk, 540, 540)
    h0 = sk.bones[0].head
    target = (h0[0] + 0.0, h0[1] + -0.05, h0[2] + 0.0)
    rc = ref.look_at((target[0] + 0.0, target[1] + 0.0, target[2] + -3.2), target, (0, 1, 0), 540 * 3.2 / 2.3, 540, 540)
    assert list(rc.extrinsic) == list(cam.extrinsic) and rc.fx == cam.fx


def test_pose_context_host(oracle):
    """arfx_pose_context == PoseContext::make restated in the oracle (bone, inverse, capsules)."""
    import ctypes as C
    sk = fx.smpl24()
    pose = fx.random_pose(sk, 3)
    pre = fx.yaw_about((0.1, 0.2, 0.3), -0.4)
    nb = len(sk.bones)
    ob, obi = np.zeros((nb, 12)), np.zeros((nb, 12))
    ca, cb, co = np.zeros((nb, 3)), np.zeros((nb, 3)), np.zeros(nb)
    _lib.call("arfx_pose_context", C.byref(sk.to_c()), arf.ptr(pose.bone_transforms, C.c_double),
              arf.ptr(pre, C.c_double), 3.0, arf.ptr(ob, C.c_double), arf.ptr(obi, C.c_double),
              arf.ptr(ca, C.c_double), arf.ptr(cb, C.c_double), arf.ptr(co, C.c_double))
    # identity bone transforms with pre = p  ->  bone = p, inverse = p^-1 (checked on the oracle's FK)
    assert np.allclose(co, 3.0 * np.array([b.radius for b in sk.bones]))
    for i, b in enumerate(sk.bones):
        a = fx._apply(ob[i], b.head)
        assert np.allclose(a, ca[i]) and np.allclose(fx._apply(ob[i], b.tail), cb[i])
        back = fx._apply(obi[i], fx._apply(ob[i], (0.3, -0.2, 0.5)))
        assert np.allclose(back, (0.3, -0.2, 0.5), atol=1e-12)


def test_invalid_arguments_raise_like_the_reference():
    bad = arf.Skeleton([arf.Bone(0, (0, 0, 0), (0, 1, 0), 0.1)])  # root must have parent -1
    with pytest.raises(pkg.InvalidArgument, match="root"):
        arf.pose_from_joint_rotations(bad, np.tile(fx.IDENTITY9, (1, 1)))
    with pytest.raises(ValueError, match="levels"):
        arf.level_resolutions(arf.HashGridConfig(levels=0))
    with pytest.raises(pkg.InvalidArgument):
        arf.pose_from_joint_rotations(fx.smpl24(), np.tile(fx.IDENTITY9, (3, 1)))


def test_no_cpu_fallback_without_gpu():
    if arf.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(pkg.NoDevice):
        arf.build_model(fx.smpl24(), fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), 1)
    with pytest.raises(pkg.NoDevice):
        arf.composite([1], [0.1], [0], np.ones(1, np.float32), np.ones((1, 3), np.float32), 1e-3)


def test_vectorised_pcg_stream():
    import numpy as np
    r1, r2 = fx.keyed_rng(5, 5), fx.keyed_rng(5, 5)
    v = fx.pcg_stream_u32(r1, 5000)
    w = np.array([r2.next_u32() for _ in range(5000)], np.uint64)
    assert np.array_equal(v, w) and r1.state == r2.state and r1.next_u32() == r2.next_u32()


def test_fixture_pcg_matches_reference_stream(oracle):
    """Python keyed_rng restatement == the C one (used for poses / microbench points)."""
    # oracle hashes: identical builds from the same seed => same PCG stream
    sk = fx.default_figure_skeleton()
    g = arf.HashGridConfig(levels=1, table_size_log2=4, base_resolution=2, max_resolution=2)
    M = oracle.build_model(sk, g, arf.MlpConfig(2, 4, 1, 4), (2, 2, 2), 77)
    gp = oracle.arrays(M)[0]
    r = fx.keyed_rng(77, 0x6a1d, 17)
    expect = np.array([r.uniform(-1e-4, 1e-4) for _ in range(gp.size)], np.float64).astype(np.float32)
    assert np.array_equal(gp.view(np.uint32), expect.view(np.uint32))


def test_checkpoint_rejects_malformed_files(tmp_path):
    """Checkpoint parsing (checkpoint.cpp) fails with DataError before touching a device."""
    from paper_2212_10550_b200 import DataError, InvalidArgument
    from paper_2212_10550_b200 import arf as A
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"not a checkpoint at all, definitely not")
    with pytest.raises(DataError):
        A.load_checkpoint(bad)
    # right magic, wrong checksum
    bad.write_bytes(b"ARFXCKPT" + b"\x01\x00\x00\x00" + b"\x00" * 40)
    with pytest.raises(DataError, match="checksum"):
        A.load_checkpoint(bad)
    with pytest.raises(InvalidArgument):
        A.load_checkpoint(tmp_path / "missing.ckpt")


def test_header_is_plain_c(tmp_path):
    """include/arfx.h is the drop-in boundary for C / cgo / FFI callers: it must compile as
    strict C99 (no C++ types in the signatures) and as C++."""
    import shutil
    import subprocess
    from pathlib import Path
    inc = Path(__file__).resolve().parent.parent / "include"
    src = tmp_path / "use.c"
    src.write_text('#include "arfx.h"\nint main(void) { arfx_loss_config c = {1, 0.1, 0.1, 0.1, 0.1, 0, 0};\n'
                   '  (void)c; return (int)sizeof(arfx_render_options) == 0; }\n')
    for cc, flags in (("gcc", ["-std=c99", "-pedantic", "-Wall", "-Werror"]), ("g++", ["-std=c++17", "-Wall", "-x", "c++"])):
        if shutil.which(cc) is None:
            continue
        r = subprocess.run([cc, *flags, "-I", str(inc), "-c", str(src), "-o", str(tmp_path / f"{cc}.o")],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_reference_workload_matches_fixtures(ref):
    """bench.py --impl reference builds its workload through the reference alone
    (oracle/workload.py + ref_driver.cpp arfr_random_pose / arfr_default_camera); it must be
    the product arm's workload bit for bit: skeleton, all 100 animation poses, the camera."""
    from oracle import workload as wl
    sk = fx.smpl24()
    rsk = wl.smpl24()
    assert [(b.parent, tuple(b.head), tuple(b.tail), b.radius) for b in sk.bones] == \
        [(b.parent, tuple(b.head), tuple(b.tail), b.radius) for b in rsk.bones]
    poses = fx.animation_poses(sk, 100)
    rposes = wl.animation_poses(ref, rsk)
    for p, q in zip(poses, rposes):
        assert np.array_equal(p.bone_transforms.view(np.uint64), q.bone_transforms.view(np.uint64))
        assert np.array_equal(p.global_transform.view(np.uint64), q.global_transform.view(np.uint64))
    cam = fx.default_camera(sk, 540, 540)
    rc = ref.default_camera(rsk, 540, 540)
    assert (cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height) == (rc.fx, rc.fy, rc.cx, rc.cy, rc.width, rc.height)
    assert np.array_equal(np.array(cam.extrinsic, np.float64).view(np.uint64),
                          np.array(rc.extrinsic[:], np.float64).view(np.uint64))
    g, m, o, r = fx.config1_grid(), fx.config1_mlp(), fx.config1_occupancy(), fx.config1_render_options()
    rg, rmc, ro, rr = wl.GridConfig(), wl.MlpConfig(), wl.OccupancyConfig(), wl.RenderOptions()
    assert (g.levels, g.features_per_level, g.table_size_log2, g.base_resolution, g.max_resolution) == \
        (rg.levels, rg.features_per_level, rg.table_size_log2, rg.base_resolution, rg.max_resolution)
    assert (m.input_dim, m.hidden_dim, m.hidden_layers, m.output_dim) == \
        (rmc.input_dim, rmc.hidden_dim, rmc.hidden_layers, rmc.output_dim)
    assert vars(o) == vars(ro) and vars(r) == vars(rr) and fx.CONFIG1_SEED == wl.SEED
