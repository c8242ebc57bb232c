"""N>1 host logic on CPU with torch.distributed (gloo, world_size 2): the interleaved
row-tile partition covers every pixel row exactly once, ranks agree on the frame
schedule, and the bench's timing reduction is the max over ranks while posed-sample
counts are summed -- the same collectives bench.py runs over NCCL."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import numpy as np

from paper_2212_10550_b200.arf import shard_cells, shard_rows, unshard_cells


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, heights, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for H in heights:
            rows = torch.tensor(shard_rows(H, rank, world), dtype=torch.int64)
            n = torch.tensor([rows.numel()])
            sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(sizes, n)
            mx = int(max(s.item() for s in sizes))
            padded = torch.full((mx,), -1, dtype=torch.int64)
            padded[: rows.numel()] = rows
            allr = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(allr, padded)
            cat = torch.cat([a[a >= 0] for a in allr])
            assert sorted(cat.tolist()) == list(range(H)), H
            assert len(set(cat.tolist())) == H
        # occupancy grid shards: each rank computes its cell-interleaved cells into its block,
        # the blocks are all-gathered, every rank permutes them into cell order
        cells = 64 ** 3 if 64 ** 3 % world == 0 else 60 ** 3
        mine = shard_cells(cells, rank, world)
        block = torch.from_numpy(np.sin(mine.astype(np.float64)).astype(np.float32))
        parts = [torch.zeros_like(block) for _ in range(world)]
        dist.all_gather(parts, block)
        grid = unshard_cells(torch.cat(parts).numpy(), world)
        assert np.array_equal(grid, np.sin(np.arange(cells, dtype=np.float64)).astype(np.float32))
        # bench.py reduction: max of per-rank device time, sum of per-rank posed samples
        t = torch.tensor([10.0 + rank, 100.0 * (rank + 1)], dtype=torch.float64)
        tt = t.clone()
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
        assert t[0].item() == 10.0 + world - 1
        assert tt[1].item() == sum(100.0 * (r + 1) for r in range(world))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharding_and_reductions_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, [540, 96, 17, 1], q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(msg == "ok" for _, msg in res), res


def test_partitions_are_balanced():
    """4-row ray tiles: at 540 rows every rank of 2/4/8 renders within one tile of the mean;
    cell-interleaved grid shards: equal cell counts."""
    for world in (2, 4, 8):
        rows = [len(shard_rows(540, r, world)) for r in range(world)]
        assert sum(rows) == 540 and max(rows) - min(rows) <= 4, rows
        cells = [len(shard_cells(64 ** 3, r, world)) for r in range(world)]
        assert len(set(cells)) == 1 and sum(cells) == 64 ** 3
