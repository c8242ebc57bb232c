"""Per-kernel device time of the SPEC train step (libarfx profiler), config 3."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2212_10550_b200 import arf, fixtures as fx  # noqa: E402
from paper_2212_10550_b200._lib import check, lib  # noqa: E402
from paper_2212_10550_b200.trainer import Trainer, TrainConfig  # noqa: E402

sk = fx.smpl24()
model = arf.build_model(sk, fx.config1_grid(), fx.config1_mlp(), (32, 32, 32), fx.CONFIG1_SEED)
poses = [fx.random_pose(sk, 100 + i) for i in range(8)]
cam = fx.default_camera(sk, 540, 540)
tr = Trainer(model, fx.figure_for(sk), poses, cam, TrainConfig(iterations=40, seed=9))
for _ in range(5):
    tr.step()
torch.cuda.synchronize()
L = lib()
check(L.arfx_profile_enable(model._h, 1))
names = C.create_string_buffer(32 * 32)
ms = np.zeros(32)
la = np.zeros(32, np.int64)
n = C.c_int()
check(L.arfx_profile_read(model._h, 32, names, ms.ctypes.data_as(C.POINTER(C.c_double)),
                          la.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(n)))
K = 32
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(tr.stream)
for _ in range(K):
    tr.step()
e1.record(tr.stream)
torch.cuda.synchronize()
check(L.arfx_profile_read(model._h, 32, names, ms.ctypes.data_as(C.POINTER(C.c_double)),
                          la.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(n)))
tot = e0.elapsed_time(e1) / K
print(f"step {tot:.3f} ms")
acc = 0
for k in range(n.value):
    nm = names.raw[32 * k:32 * k + 32].split(b"\\0")[0].decode()
    print(f"  {nm:20s} {ms[k] / K:.3f} ms  x{la[k] // K}")
    acc += ms[k] / K
print(f"  {'(kernels)':20s} {acc:.3f} ms; host/other {tot - acc:.3f} ms")
