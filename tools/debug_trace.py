import sys, numpy as np
sys.path.insert(0, '.')
from paper_2212_10550_b200 import arf, fixtures as fx
from oracle.oracle_ctypes import Checker
ref = Checker("ref")
sk = fx.smpl24(); g, m = fx.config1_grid(), fx.config1_mlp()
dm = arf.build_model(sk, g, m, (32,32,32), fx.CONFIG1_SEED)
rm = ref.build_model(sk, g, m, (32,32,32), fx.CONFIG1_SEED)
pose = fx.random_pose(sk, fx.CONFIG1_POSE_SEED)
cam = fx.default_camera(sk, 96, 96)
cfg = arf.OccupancyConfig()
occ = arf.build_model_inference_grid(dm, pose, cfg)
rocc, _ = ref.build_inference_grid(rm, pose.bone_transforms, pose.global_transform, cfg)
opt = arf.RenderOptions(samples_per_ray=128, stratified=False, seed=11, frame_id=3)
img = arf.render_model(dm, pose, cam, occ, opt)
tr = arf.render_trace(dm)
rrgb, ralpha, rcnt, rtr = ref.render_trace(rm, pose.bone_transforms, pose.global_transform, cam, rocc, opt)
order = np.lexsort((tr.index, tr.ray))
can = tr.canonical[order]; rcan = rtr["s_canonical"]
bad = np.where(np.any(can != rcan, axis=1))[0]
print("n", len(order), "bad", len(bad))
for i in bad[:10]:
    print(i, tr.ray[order][i], tr.index[order][i], "ours", can[i], tr.density[order][i], "ref", rcan[i], rtr["s_density"][i], "hasroot", tr.has_root[order][i], rtr["s_has_root"][i])
print("max |rgb diff|", np.abs(img.rgb - rrgb).max(), "alpha", np.abs(img.alpha - ralpha).max())
