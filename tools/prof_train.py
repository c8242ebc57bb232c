"""Small driver for ncu: SPEC train steps at config 3 (smpl24 avatar, 540x540 camera,
4096 rays, analytic ground truth, L_density on). Usage: python tools/prof_train.py [steps]
(ARFX_DET=1: TrainConfig.deterministic)"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2212_10550_b200 import arf, fixtures as fx  # noqa: E402
from paper_2212_10550_b200.trainer import Trainer, TrainConfig  # noqa: E402


def main(steps: int = 4):
    sk = fx.smpl24()
    model = arf.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    poses = [fx.random_pose(sk, 100 + i) for i in range(4)]
    cam = fx.default_camera(sk, 540, 540)
    tr = Trainer(model, fx.figure_for(sk), poses, cam, TrainConfig(iterations=steps, seed=9,
                                                                               deterministic=os.environ.get("ARFX_DET") == "1"))
    h = tr.train()
    print("loss", h[-1].tolist())


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
