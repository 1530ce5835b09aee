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
