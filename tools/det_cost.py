"""Deterministic-gradient cost: SPEC train steps (config 3: smpl24 avatar, 540x540, 4096
rays, L_density on) timed with CUDA events on the trainer's stream, default vs
TrainConfig.deterministic. Usage: python tools/det_cost.py [steps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2212_10550_b200 import arf, fixtures as fx  # noqa: E402
from paper_2212_10550_b200.trainer import Trainer, TrainConfig  # noqa: E402


def run(det: bool, steps: int, pipelined: bool = True, interval: int = 0) -> float:
    sk = fx.smpl24()
    model = arf.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    poses = [fx.random_pose(sk, 100 + i) for i in range(4)]
    cam = fx.default_camera(sk, 540, 540)
    tr = Trainer(model, fx.figure_for(sk), poses, cam,
                 TrainConfig(iterations=steps, seed=9, occupancy_interval=interval, deterministic=det))
    tr.pipelined = pipelined
    tr.train(5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tr.stream.synchronize()
    e0.record(tr.stream)
    tr.train(steps)
    e1.record(tr.stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


if __name__ == "__main__":
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    if len(sys.argv) > 2 and sys.argv[2] == "pipe":
        for interval in (0, 16):
            for pipe in (False, True, False, True):
                print(f"interval={interval} pipelined={pipe}: {run(False, k, pipe, interval):.3f} ms/step")
    else:
        for det in (False, True, False, True):
            print(f"deterministic={det}: {run(det, k):.3f} ms/step")
