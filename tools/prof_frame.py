"""Small driver for ncu: config-1 avatar, F frames of (inference grid + render) at 540x540
through the device API on one stream. Usage: python tools/prof_frame.py [frames] [exact|tcgen05] [stats]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_2212_10550_b200 import arf, fixtures as fx  # noqa: E402
from paper_2212_10550_b200._lib import check, lib  # noqa: E402


def main(frames: int = 3, mlp: str = "exact"):
    L = lib()
    sk = fx.smpl24()
    model = arf.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    model.set_mlp_mode(mlp)
    poses = fx.animation_poses(sk, 4)
    cam = fx.default_camera(sk, 540, 540)
    opt = fx.config1_render_options()
    occ = arf.OccupancyGrid(model.normalized_box, fx.config1_occupancy())
    views = [arf.PosedModelView(model, p) for p in poses]
    out = arf.RenderImages(540, 540, np.zeros((540, 540, 3), np.float32), np.zeros((540, 540), np.float32))
    stats = np.zeros(16, np.uint64)
    with_stats = len(sys.argv) > 3 and sys.argv[3] == "stats"
    check(L.arfx_stats_enable(model._h, 1 if with_stats else 0))
    for f in range(frames):
        v = views[f % len(views)]
        check(L.arfx_build_inference_grid(model._h, v._h, occ._h, None, None))
        arf.render_model(model, v, cam, occ, opt, out=out)
    if with_stats:
        check(L.arfx_stats_read(model._h, stats.ctypes.data_as(C.POINTER(C.c_uint64))))
        print("per-frame stats E U I S P Q QT:", (stats[:7] / frames).astype(np.int64).tolist())
    print("frames", frames, "posed", model.counters.posed_queries, "alpha sum", float(out.alpha.sum()))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3, sys.argv[2] if len(sys.argv) > 2 else "exact")
