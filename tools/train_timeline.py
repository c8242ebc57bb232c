"""Kernel timeline of the pipelined SPEC train step (config 3) via the CUDA profiler
(torch.profiler / CUPTI): per stream, the kernels of a few steady-state steps with start
offsets and durations, plus per-stream busy time. Usage: python tools/train_timeline.py [steps]"""
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main(steps=4):
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2212_10550_b200 import arf, fixtures as fx
    from paper_2212_10550_b200.trainer import Trainer, TrainConfig
    sk = fx.smpl24()
    model = arf.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
    cam = fx.default_camera(sk, 540, 540)
    poses = [fx.random_pose(sk, 100 + i) for i in range(8)]
    cfg = TrainConfig(iterations=100, rays_per_batch=4096, samples_per_ray=128, occupancy_interval=16, seed=9,
                      adam=arf.AdamConfig(total_steps=1000))
    tr = Trainer(model, fx.figure_for(sk), poses, cam, cfg)
    for _ in range(20):
        tr.step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            tr.step()
        torch.cuda.synchronize()
    path = Path(tempfile.mkdtemp()) / "trace.json"
    prof.export_chrome_trace(str(path))
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    t0 = min(e["ts"] for e in ev)
    t1 = max(e["ts"] + e["dur"] for e in ev)
    streams = {}
    for e in sorted(ev, key=lambda e: e["ts"]):
        streams.setdefault(e["args"].get("stream", e.get("tid")), []).append(e)
    print(f"{steps} steps, span {t1 - t0:.1f} us ({(t1 - t0) / steps:.1f} us/step)")
    for s, es in streams.items():
        busy = sum(e["dur"] for e in es)
        print(f"\n== stream {s}: {len(es)} kernels, busy {busy / steps:.1f} us/step")
        agg = {}
        for e in es:
            nm = e["name"].replace("(anonymous namespace)::", "").replace("void ", "").replace("arfx::", "")
            nm = nm.split("(")[0]
            a = agg.setdefault(nm[:60], [0, 0.0])
            a[0] += 1
            a[1] += e["dur"]
        for nm, (c, d) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
            print(f"   {nm:60s} {c / steps:5.1f}/step {d / steps:8.1f} us/step")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
