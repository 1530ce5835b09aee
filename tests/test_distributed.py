"""Multi-process (world_size 2, gloo, CPU) tests of the view-batch data-parallel logic:
view partitioning, the gradient all-reduce of the flat buffer, identical Adam updates on
every rank after the exchange, and max-over-ranks timing."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import REPO


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from oracle import pipeline as orc
    from paper_2501_18630_b200 import distributed as dd
    from paper_2501_18630_b200.primitive import group_layout

    r, w, _ = dd.init(backend="gloo")
    assert (r, w) == (rank, world)
    views = list(dd.partition_views(32, w, r))
    # every rank contributes a per-view gradient (a deterministic function of the view id)
    n, k = 50, 16
    layout, total = group_layout(n, k)
    flat = torch.zeros(total, dtype=torch.float32)
    for v in views:
        g = torch.from_numpy(np.random.default_rng(1000 + v).standard_normal(total).astype(np.float32))
        flat += g
    dd.allreduce_grads(flat)
    # identical Adam on every rank after the exchange (oracle Adam, training.py:258-273)
    params = {"p": np.zeros(total)}
    m = {"p": np.zeros(total)}
    v2 = {"p": np.zeros(total)}
    orc.adam_step(params, {"p": flat.double().numpy()}, m, v2, 1, {"p": 5e-3})
    tmax = dd.max_over_ranks(1.0 + r)
    tsum = dd.sum_over_ranks(1.0)
    np.savez(os.path.join(out_dir, f"rank{r}.npz"), views=np.array(views), flat=flat.numpy(),
             params=params["p"], tmax=tmax, tsum=tsum)
    torch.distributed.destroy_process_group()


def test_partition_views_covers_batch():
    from paper_2501_18630_b200.distributed import partition_views

    for world in (1, 2, 4, 8, 3):
        seen = []
        for r in range(world):
            seen += list(partition_views(32, world, r))
        assert seen == list(range(32))
    assert list(partition_views(32, 8, 3)) == [12, 13, 14, 15]
    with pytest.raises(ValueError):
        partition_views(32, 2, 2)


def test_two_rank_gradient_allreduce_and_adam(tmp_path):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    a = np.load(tmp_path / "rank0.npz")
    b = np.load(tmp_path / "rank1.npz")
    assert list(a["views"]) == list(range(16)) and list(b["views"]) == list(range(16, 32))
    # the reduced gradient is the sum over all 32 views, identical on both ranks
    from paper_2501_18630_b200.primitive import group_layout

    _, total = group_layout(50, 16)
    expect = np.zeros(total, np.float32)
    for v in range(32):
        expect += np.random.default_rng(1000 + v).standard_normal(total).astype(np.float32)
    np.testing.assert_allclose(a["flat"], expect, rtol=1e-5, atol=1e-4)
    np.testing.assert_array_equal(a["flat"], b["flat"])
    np.testing.assert_array_equal(a["params"], b["params"])
    assert float(a["tmax"]) == 2.0 and float(b["tmax"]) == 2.0
    assert float(a["tsum"]) == 2.0


def _shard_worker(rank, world, port, out_dir):
    """ShardedOptimizer on CPU tensors (gloo): each rank contributes gradients, the
    reduce-scatter gives its shard of the sum, an Adam update (oracle arithmetic, per-group
    lrs from the shifted group ends) on the shard only, all-gather -> full parameters."""
    import sys

    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2501_18630_b200 import distributed as dd
    from paper_2501_18630_b200.primitive import GradientBuffer, PrimitiveSet

    dd.init(backend="gloo")
    n, k = 37, 4
    rng = np.random.default_rng(5)
    prims = PrimitiveSet(rng.standard_normal((n, 3)), rng.standard_normal((n, 4)), rng.standard_normal((n, 3)),
                         rng.standard_normal(n), rng.standard_normal(n), rng.standard_normal((n, k, 3)),
                         device="cpu")
    flat0 = prims.flat.clone()
    sh = dd.ShardedOptimizer(prims, GradientBuffer)
    assert prims.flat.data_ptr() == sh.pbuf.data_ptr() and torch.equal(prims.flat, flat0)
    assert sh.padded % (4 * world) == 0 and sh.lo % 4 == 0
    g = torch.from_numpy(np.random.default_rng(100 + rank).standard_normal(sh.total).astype(np.float32))
    sh.grads.flat.copy_(g)
    sh.reduce_scatter()
    # Adam (first step, bias-corrected) on the shard with per-group lrs from the shifted ends
    lrs = {name: 1e-3 * (i + 1) for i, name in enumerate(prims.groups)}
    ends = sh.shard_group_ends()
    lr = torch.empty(sh.shard)
    prev = 0
    for name, e in zip(prims.groups, ends):
        lr[prev:e] = lrs[name]
        prev = max(prev, e)
    lr[prev:] = lrs[prims.groups[-1]]
    gs = sh.gshard.double()
    m, v = 0.1 * gs, 0.001 * gs * gs
    upd = lr.double() * (m / 0.1) / (torch.sqrt(v / 0.001) + 1e-15)
    mine = sh.pbuf[sh.lo: sh.lo + sh.shard]
    mine.copy_((mine.double() - upd).float())
    sh.all_gather()
    np.savez(os.path.join(out_dir, f"shard{rank}.npz"), flat=prims.flat.numpy(), flat0=flat0.numpy(),
             lo=sh.lo, shard=sh.shard)
    torch.distributed.destroy_process_group()


def test_sharded_optimizer_equals_allreduce_adam_world2(tmp_path):
    """Reduce-scatter -> sharded Adam -> all-gather == all-reduce -> replicated Adam, with the
    global per-group learning rates (distributed.ShardedOptimizer, gloo world 2)."""
    world = 2
    mp.spawn(_shard_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(os.path.join(tmp_path, f"shard{r}.npz")) for r in range(world)]
    np.testing.assert_array_equal(res[0]["flat"], res[1]["flat"])
    # reference: summed gradient, replicated Adam over the full buffer
    from paper_2501_18630_b200.primitive import group_layout

    flat0 = res[0]["flat0"].astype(np.float64)
    total = flat0.size
    g = sum(np.random.default_rng(100 + r).standard_normal(total).astype(np.float32) for r in range(world))
    g = g.astype(np.float32).astype(np.float64)
    layout, _ = group_layout(37, 4)
    lr = np.zeros(total)
    prev = 0
    for i, (name, a, b, _) in enumerate(layout):  # a group owns [previous end, its end) (adam.cu group_lr)
        lr[prev:b] = 1e-3 * (i + 1)
        prev = b
    lr[prev:] = 1e-3 * len(layout)
    upd = lr * g / (np.abs(g) + 1e-15)
    ref = (flat0 - upd).astype(np.float32)
    np.testing.assert_allclose(res[0]["flat"], ref, rtol=0, atol=1e-6)
