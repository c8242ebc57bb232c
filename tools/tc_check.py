"""tcgen05 decoder vs the exact decoder on the same render (quick numerics check)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2212_10550_b200 import arf, fixtures as fx

sk = fx.smpl24()
m = arf.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
pose = fx.random_pose(sk, 42)
cam = fx.default_camera(sk, 160, 160)
occ = arf.build_model_inference_grid(m, pose, arf.OccupancyConfig())
opt = arf.RenderOptions()
for label, scale in [("random-init", None), ("structured", 0.5)]:
    if scale:
        g, w, _ = m.params()
        rng = np.random.default_rng(0)
        m.set_params(rng.uniform(-scale, scale, g.size).astype(np.float32), (w * 2).astype(np.float32))
    m.set_mlp_mode("exact")
    a = arf.render_model(m, pose, cam, occ, opt)
    m.set_mlp_mode("tcgen05")
    b = arf.render_model(m, pose, cam, occ, opt)
    d = np.abs(a.rgb - b.rgb)
    rel = d / np.maximum(np.abs(a.rgb), 1e-6)
    print(label, "max|d|", d.max(), "max rel (px>1e-3)", rel[np.abs(a.rgb) > 1e-3].max() if (np.abs(a.rgb) > 1e-3).any() else 0,
          "alpha max|d|", np.abs(a.alpha - b.alpha).max(), "mean rgb", a.rgb.mean())
