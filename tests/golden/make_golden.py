"""Generate tests/golden/golden_small.npz from the UNMODIFIED reference compiled in place
(oracle/_ref/libarf_ref.so). Run here, where /root/reference exists:
    python tests/golden/make_golden.py
The fixture inputs are regenerated deterministically by golden_inputs() (also used by
tests/test_golden.py); only reference OUTPUTS are stored.
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2212_10550_b200 import arf, fixtures as fx  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden_small.npz"


def golden_inputs():
    sk = fx.default_figure_skeleton()
    g = arf.HashGridConfig(levels=4, features_per_level=2, table_size_log2=12, base_resolution=4, max_resolution=48)
    m = arf.MlpConfig(8, 16, 2, 4)
    pose = arf.pose_from_joint_rotations(sk, fx.bend_pose_rotations(10, 0.45, 0.35), fx.yaw_about(sk.bones[0].head, 0.8))
    cam = fx.default_camera(sk, 28, 24)
    rng = np.random.default_rng(2024)
    return dict(sk=sk, g=g, m=m, skin_res=(12, 12, 12), seed=5, pose=pose, cam=cam,
                occ=arf.OccupancyConfig(resolution=24),
                opt=arf.RenderOptions(samples_per_ray=48, stratified=True, seed=3, frame_id=9),
                unit=rng.uniform(0, 1, (200, 3)), skin_unit=rng.uniform(-0.1, 1.1, (100, 3)),
                norm_unit=rng.uniform(0.3, 0.7, (300, 3)), px=rng.integers(0, 28, 48), py=rng.integers(0, 24, 48),
                hash_cells=rng.integers(0, 300, (64, 3)))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def compute(chk):
    I = golden_inputs()
    M = chk.build_model(I["sk"], I["g"], I["m"], I["skin_res"], I["seed"])
    gp, mp, sw = chk.arrays(M)
    lo, hi = np.array(M.canon_lo[:]), np.array(M.canon_hi[:])
    nlo, nhi = np.array(M.norm_lo[:]), np.array(M.norm_hi[:])
    pts = lo + (hi - lo) * I["unit"]
    P = I["pose"]
    out = {}
    out["grid_sha"] = np.array(sha(gp))
    out["mlp"] = mp.copy()
    out["skin_sha"] = np.array(sha(sw))
    out["boxes"] = np.array([M.canon_lo[:], M.canon_hi[:], M.norm_lo[:], M.norm_hi[:]])
    g216 = arf.HashGridConfig(levels=2, table_size_log2=16, base_resolution=16, max_resolution=256)
    out["hash_idx"] = np.array([[chk.hash_index(g216, l, *c) for c in I["hash_cells"]] for l in range(2)], np.uint32)
    out["res_config1"] = np.array(chk.level_resolutions(fx.config1_grid()), np.int32)
    out["skin_w"] = chk.skinning_weights(M, lo + (hi - lo) * I["skin_unit"])
    out["feats"] = chk.hash_encode(M, pts)
    out["dens"], out["col"] = chk.field_query(M, pts)
    bp = []
    for i, b in enumerate(I["sk"].bones):
        a_, e_ = fx._apply(P.bone_transforms[i], b.head), fx._apply(P.bone_transforms[i], b.tail)
        for u in np.linspace(0.05, 0.95, 10):
            bp.append([a_[k] + (e_[k] - a_[k]) * u for k in range(3)])
    bp = np.array(bp) + 0.03 * (I["unit"][:len(bp)] - 0.5)
    out["root_pts"] = bp
    out["root_cnt"], out["roots"], out["root_res"] = chk.inverse_lbs(M, P.bone_transforms, arf.rigid(), 3.0, bp)
    q = nlo + (nhi - nlo) * I["norm_unit"]
    out["pq_dens"], out["pq_col"], out["pq_canon"], out["pq_has"] = chk.posed_query(
        M, P.bone_transforms, P.global_transform, q)
    og, cnt = chk.build_inference_grid(M, P.bone_transforms, P.global_transform, I["occ"])
    out["occ_values"], out["occ_mask"] = [a.copy() for a in chk.occ_arrays(og)]
    out["occ_counters"] = cnt
    rgb, alpha, rc, tr = chk.render_trace(M, P.bone_transforms, P.global_transform, I["cam"], og, I["opt"])
    out["rgb"], out["alpha"], out["render_counters"] = rgb, alpha, rc
    for k in ("s_ray", "s_index", "s_has_root", "s_t", "s_delta", "terminated_at"):
        out["trace_" + k] = tr[k]
    dC = np.ones((len(I["px"]), 3), np.float32)
    dA = np.ones(len(I["px"]), np.float32)
    trgb, talpha, gg, mg, tc = chk.train_fwd_bwd(M, P.bone_transforms, P.global_transform, I["cam"], og, I["opt"],
                                                 I["px"], I["py"], dC, dA)
    nz = np.nonzero(gg)[0]
    out["train_rgb"], out["train_grid_idx"], out["train_grid_val"], out["train_mlp"] = trgb, nz, gg[nz], mg
    return out


if __name__ == "__main__":
    from oracle.oracle_ctypes import Checker, build
    build("ref")
    out = compute(Checker("ref"))
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(out)} arrays)")
