"""NCCL collectives on libarfx device memory wrapped via __cuda_array_interface__ (world 1):
all_gather_into_tensor (in place) and reduce_scatter_tensor (in place) as the bench / trainer
use them. Run: torchrun --nproc-per-node 1 --master-addr 127.0.0.1 tools/nccl_cai_check.py"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2212_10550_b200 import arf, fixtures as fx  # noqa: E402
from paper_2212_10550_b200.trainer import device_view  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
sk = fx.default_figure_skeleton()
m = arf.build_model(sk, arf.HashGridConfig(levels=16, table_size_log2=12), arf.MlpConfig(32, 64, 2, 4), (8, 8, 8), 1)
occ = arf.OccupancyGrid(m.normalized_box, arf.OccupancyConfig())
vals = device_view(occ.device_arrays()[0], occ.cell_count())
slab = occ.cell_count() // world
vals[rank * slab:(rank + 1) * slab].fill_(float(rank + 1))
dist.all_gather_into_tensor(vals, vals[rank * slab:(rank + 1) * slab])
torch.cuda.synchronize()
assert float(vals.sum()) == sum((r + 1) * slab for r in range(world))
fl = m.flat()
g = device_view(fl["grads"], fl["n_flat"])
g.fill_(2.0)
chunk = fl["n_flat"] // world
dist.reduce_scatter_tensor(g[rank * chunk:(rank + 1) * chunk], g, op=dist.ReduceOp.AVG)
torch.cuda.synchronize()
assert float(g[rank * chunk]) == 2.0
dist.barrier()
dist.destroy_process_group()
print("nccl on libarfx memory ok, world", world)
