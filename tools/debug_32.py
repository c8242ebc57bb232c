import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2212_10550_b200 import arf, fixtures as fx
from oracle.oracle_ctypes import Checker
ref = Checker("ref")
bones = []
y = 0.2
for i in range(32):
    x = 0.04 * (1 if i % 2 else -1)
    bones.append(arf.Bone(i - 1, (x, y, 0.0), (-x, y + 0.05, 0.0), 0.03))
    y += 0.05
sk = arf.Skeleton(bones)
g, m = arf.HashGridConfig(levels=16, features_per_level=2, table_size_log2=14, base_resolution=4, max_resolution=96), arf.MlpConfig(32, 64, 2, 4)
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sk = arf.Skeleton(bones[:nb])
dm = arf.build_model(sk, g, m, (10, 10, 10), 3)
rm = ref.build_model(sk, g, m, (10, 10, 10), 3)
rots = np.tile(fx.IDENTITY9, (nb, 1))
for i in range(1, nb, 3):
    rots[i] = fx.rot_z(0.05 * (i % 5 - 2))
pose = arf.pose_from_joint_rotations(sk, rots)
rng = np.random.default_rng(3)
pts = np.column_stack([rng.uniform(-0.15, 0.15, 3000), rng.uniform(0.2, 1.9, 3000), rng.uniform(-0.05, 0.05, 3000)])
c, r, res = dm.inverse_lbs(pose, pts)
rc, rr, rres = ref.inverse_lbs(rm, pose.bone_transforms, fx.IDENTITY9.tolist() + [0, 0, 0], 3.0, pts)
bad = np.where(np.any(r.reshape(3000, -1).view(np.uint64) != rr.reshape(3000, -1).view(np.uint64), axis=1))[0]
print("nb", nb, "count equal", np.array_equal(c, rc), "bad points", len(bad))
for i in bad[:3]:
    print(i, c[i], rc[i])
    print(" gpu", r[i, :c[i]].tolist(), res[i, :c[i]].tolist())
    print(" ref", rr[i, :rc[i]].tolist(), rres[i, :rc[i]].tolist())
