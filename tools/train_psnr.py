"""End-to-end training check: train on the analytic figure's turntable
frames, then render a held-out pose and report PSNR against its ground truth.
Usage: python tools/train_psnr.py [steps] [res]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2212_10550_b200 import arf, fixtures as fx  # noqa: E402
from paper_2212_10550_b200.trainer import Trainer, TrainConfig, psnr  # noqa: E402


def turntable(sk, n, yaw0=0.0):
    return [arf.pose_from_joint_rotations(sk, fx.bend_pose_rotations(sk.bone_count(), 0.0, 0.0),
                                          fx.yaw_about(sk.bones[0].head, yaw0 + 2 * np.pi * i / n)) for i in range(n)]


def main(steps=1500, res=128):
    fig = fx.default_figure()
    sk = fig.skeleton
    g = arf.HashGridConfig(levels=16, features_per_level=2, table_size_log2=19, base_resolution=16,
                           max_resolution=2048)
    m = arf.build_model(sk, g, fx.config1_mlp(), (32, 32, 32), 7)
    poses = turntable(sk, 12)
    cam = fx.default_camera(sk, res, res)
    cfg = TrainConfig(iterations=steps, rays_per_batch=4096, samples_per_ray=128, seed=11,
                      adam=arf.AdamConfig(total_steps=steps, final_lr_factor=0.05))
    tr = Trainer(m, fig, poses, cam, cfg)
    t0 = time.perf_counter()
    h = tr.train()
    dt = time.perf_counter() - t0
    held = turntable(sk, 12, yaw0=np.pi / 12)[3]  # between two training views
    gt, mask = arf.figure_render(fig, held, m.normalized_box, cam, arf.RenderOptions(samples_per_ray=512))
    occ = arf.build_model_inference_grid(m, held, arf.OccupancyConfig())
    img = arf.render_model(m, held, cam, occ, arf.RenderOptions(samples_per_ray=128))
    p = psnr(img.rgb, gt.rgb)
    print(f"steps {steps} in {dt:.1f}s ({steps / dt:.0f} it/s); loss {h[0, 4]:.4f} -> {h[-20:, 4].mean():.4f}; "
          f"held-out PSNR {p:.2f} dB")
    return p


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1500, int(sys.argv[2]) if len(sys.argv) > 2 else 128)
