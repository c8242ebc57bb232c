"""CPU tests of the training pieces the reference lacks:
the C restatement of the losses and Adam against SPEC known answers and finite differences,
and the data-parallel flat-vector synchronisation (gloo, world 2) against one process."""
import math
import os

import numpy as np
import pytest

from paper_2212_10550_b200 import arf


def _one(oracle, rgb, alpha, gt_rgb, gt_alpha, cfg=None):
    cfg = cfg or arf.LossConfig(w_rgb=1.0, w_alpha=1.0, w_hard=1.0)
    return oracle.losses(np.array([rgb], np.float32), np.array([alpha], np.float32), np.array([gt_rgb], np.float32),
                         np.array([gt_alpha], np.float32), cfg)


def test_loss_kats(oracle):
    # SPEC.md:459-463 Huber: C = C* -> 0; r = 2 delta, delta = 0.1 -> delta (r - delta/2) = 0.015
    l4, _, _ = _one(oracle, (0.3, 0.3, 0.3), 0.5, (0.3, 0.3, 0.3), 0.5)
    assert l4[0] == 0.0
    l4, _, _ = _one(oracle, (0.2, 0.0, 0.0), 1.0, (0.0, 0.0, 0.0), 1.0)
    assert abs(l4[0] - 0.015) < 1e-8
    # quadratic branch r << delta -> r^2/2
    l4, _, _ = _one(oracle, (0.01, 0.0, 0.0), 1.0, (0.0, 0.0, 0.0), 1.0)
    assert abs(l4[0] - 0.5 * float(np.float32(0.01)) ** 2) < 1e-15
    # SPEC.md:466-470 L1 alpha: A = A* -> 0; (1, 0) -> 1; (0.25, 0.75) -> 0.5
    assert _one(oracle, (0, 0, 0), 0.3, (0, 0, 0), 0.3)[0][1] == 0.0
    assert _one(oracle, (0, 0, 0), 1.0, (0, 0, 0), 0.0)[0][1] == 1.0
    assert _one(oracle, (0, 0, 0), 0.25, (0, 0, 0), 0.75)[0][1] == 0.5
    # SPEC.md:473-477 hard surface: 0 at A in {0, 1}; A = 0.5 -> 0.12011
    assert abs(_one(oracle, (0, 0, 0), 0.0, (0, 0, 0), 0.0)[0][2]) < 1e-15
    assert abs(_one(oracle, (0, 0, 0), 1.0, (0, 0, 0), 1.0)[0][2]) < 1e-15
    assert abs(_one(oracle, (0, 0, 0), 0.5, (0, 0, 0), 0.5)[0][2] - 0.12011) < 1e-5
    # non-negative on [0, 1] (SPEC invariant)
    a = np.linspace(0, 1, 101, dtype=np.float32)
    l4, _, _ = oracle.losses(np.zeros((101, 3), np.float32), a, np.zeros((101, 3), np.float32), a,
                             arf.LossConfig(w_rgb=0, w_alpha=0, w_hard=1))
    assert l4[2] >= 0.0


def test_loss_gradients_match_fd(oracle):
    """Each loss gradient vs central differences of its double-precision value."""
    rng = np.random.default_rng(0)
    n = 64
    rgb = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    alpha = rng.uniform(0.02, 0.98, n).astype(np.float32)
    gt = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    gta = (rng.uniform(0, 1, n) > 0.5).astype(np.float32)
    cfg = arf.LossConfig()
    _, dr, da = oracle.losses(rgb, alpha, gt, gta, cfg)

    def total(r, a):  # double-precision restatement of the weighted batch mean
        e = r.astype(np.float64) - gt
        rn = np.sqrt((e * e).sum(1))
        d = cfg.huber_delta
        hub = np.where(rn <= d, 0.5 * rn * rn, d * (rn - 0.5 * d))
        A = a.astype(np.float64)
        hard = -np.log(np.exp(-np.abs(A)) + np.exp(-np.abs(A - 1))) + math.log1p(math.exp(-1))
        return (cfg.w_rgb * hub.mean() + cfg.w_alpha * np.abs(A - gta).mean() + cfg.w_hard * hard.mean())

    h = 1e-4
    for k in range(8):
        for c in range(3):
            rp, rm = rgb.astype(np.float64).copy(), rgb.astype(np.float64).copy()
            rp[k, c] += h
            rm[k, c] -= h
            fd = (total(rp, alpha) - total(rm, alpha)) / (2 * h)
            assert abs(fd - dr[k, c]) <= 1e-4 * max(abs(fd), 1e-3), (k, c, fd, dr[k, c])
        ap, am = alpha.astype(np.float64).copy(), alpha.astype(np.float64).copy()
        ap[k] += h
        am[k] -= h
        fd = (total(rgb, ap) - total(rgb, am)) / (2 * h)
        assert abs(fd - da[k]) <= 1e-4 * max(abs(fd), 1e-3), (k, fd, da[k])


def test_adam_restatement(oracle):
    n = 1024
    rng = np.random.default_rng(1)
    p = rng.normal(size=n).astype(np.float32)
    g = rng.normal(size=n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    cfg = arf.AdamConfig()
    p0, g0 = p.copy(), g.copy()
    oracle.adam(p, g, m, v, cfg, 1, 512)
    assert np.all(g == 0)
    # first step from zero moments: p -= lr * g / (|g| + eps) = lr * sign(g)
    lr = np.where(np.arange(n) >= 512, cfg.lr_mlp, cfg.lr_grid)
    assert np.allclose(p0 - p, lr * np.sign(g0), rtol=1e-4)
    # zero learning rate leaves the parameters unchanged
    q = p.copy()
    oracle.adam(q, rng.normal(size=n).astype(np.float32), m, v, arf.AdamConfig(lr_grid=0, lr_mlp=0), 2, 512)
    assert np.array_equal(q, p)


def _dp_worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist
    from oracle.oracle_ctypes import Checker
    from paper_2212_10550_b200.trainer import FlatDataParallel
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    n = 4096
    rng = np.random.default_rng(7)
    p = torch.from_numpy(rng.normal(size=n).astype(np.float32))
    grads_all = [np.random.default_rng(100 + r).normal(size=n).astype(np.float32) for r in range(world)]
    g = torch.from_numpy(grads_all[rank].copy())
    m = torch.zeros(n)
    v = torch.zeros(n)
    ora = Checker("oracle")
    cfg = arf.AdamConfig()

    def opt(b, e):  # the sharded optimizer: oracle Adam on this rank's slice
        ps, gs, ms, vs = (t[b:e].numpy() for t in (p, g, m, v))
        ps, gs, ms, vs = (np.ascontiguousarray(x) for x in (ps, gs, ms, vs))
        ora.adam(ps, gs, ms, vs, cfg, 1, 2048 - b)
        p[b:e] = torch.from_numpy(ps)
        g[b:e] = torch.from_numpy(gs)
        m[b:e] = torch.from_numpy(ms)
        v[b:e] = torch.from_numpy(vs)

    FlatDataParallel(p, g, n, rank, world).step(opt)
    out_q.put((rank, p.numpy().copy(), g.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_flat_data_parallel_matches_single_process(world, oracle):
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dp_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict((r, (p, g)) for r, p, g in (q.get(timeout=120) for _ in range(world)))
    for pr in procs:
        pr.join(timeout=60)
    # single process: mean gradient, full-vector Adam
    n = 4096
    p = np.random.default_rng(7).normal(size=n).astype(np.float32)
    g = np.mean([np.random.default_rng(100 + r).normal(size=n).astype(np.float32) for r in range(world)],
                axis=0).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    oracle.adam(p, g, m, v, arf.AdamConfig(), 1, 2048)
    for r in range(world):
        assert np.array_equal(res[r][0], p), r
        assert np.all(res[r][1] == 0)
