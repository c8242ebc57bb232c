"""Host enqueue time vs device time of the pipelined SPEC train step (config 3): if the
host needs as long to enqueue a step as the GPU needs to run it, the step is host-bound.
Usage: python tools/train_host_time.py [steps]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main(steps=300):
    import torch
    from paper_2212_10550_b200 import arf, fixtures as fx
    from paper_2212_10550_b200.trainer import Trainer, TrainConfig
    sk = fx.smpl24()
    model = arf.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    cam = fx.default_camera(sk, 540, 540)
    poses = [fx.random_pose(sk, 100 + i) for i in range(8)]
    cfg = TrainConfig(iterations=steps, rays_per_batch=4096, samples_per_ray=128, occupancy_interval=16, seed=9,
                      adam=arf.AdamConfig(total_steps=1000))
    tr = Trainer(model, fx.figure_for(sk), poses, cam, cfg)
    for _ in range(40):
        tr.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(tr.stream)
    t0 = time.perf_counter()
    host = []
    for _ in range(steps):
        a = time.perf_counter()
        tr.step()
        host.append(time.perf_counter() - a)
    t1 = time.perf_counter()
    e1.record(tr.stream)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    host.sort()
    print(f"device {e0.elapsed_time(e1) / steps * 1e3:.1f} us/step, host enqueue {(t1 - t0) / steps * 1e6:.1f} us/step "
          f"(median {host[len(host) // 2] * 1e6:.1f}), wall {(t2 - t0) / steps * 1e6:.1f} us/step")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 300)
