"""View-batch data parallelism on the GPU box: TrainStep(process_group=...) with two ranks
(processes) sharing the one GPU over a gloo group (CUDA tensors through the host), views
{0, 1} and {2, 3}, against one process stepping all four views.  The gradient sum equals
the single-process one up to fp32 summation order; after Adam (all-reduce + replicated, and
reduce-scatter -> sharded Adam -> all-gather) the parameters agree the same way and the two
ranks are bit-identical.  (NCCL needs one GPU per rank; the driver's scaling run covers it.)"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_view_batch_equals_single_process(cuda, tmp_path):
    worker = os.path.join(HERE, "dist_train_worker.py")
    steps = 3
    port = _port()
    procs = [subprocess.Popen([sys.executable, worker, str(r), "2", str(port), str(tmp_path), "4", str(steps)])
             for r in range(2)]
    ref = subprocess.run([sys.executable, worker, "0", "1", "0", str(tmp_path), "4", str(steps)], timeout=600)
    rcs = [p.wait(timeout=600) for p in procs]
    assert ref.returncode == 0 and rcs == [0, 0]
    r0, r1 = (np.load(os.path.join(tmp_path, f"rank{r}_w2.npz")) for r in range(2))
    one = np.load(os.path.join(tmp_path, "rank0_w1.npz"))
    # the summed gradient: identical on both ranks, equal to the single process's
    np.testing.assert_array_equal(r0["grad"], r1["grad"])
    scale = np.abs(one["grad"]).max()
    np.testing.assert_allclose(r0["grad"], one["grad"], rtol=1e-5, atol=1e-6 * scale)
    for mode in ("allreduce", "sharded"):
        np.testing.assert_array_equal(r0[mode], r1[mode])  # replicas stay bit-identical
        d = np.abs(r0[mode] - one[mode])
        # Adam normalises each gradient: elements whose gradient is at fp32 noise level may
        # move differently (at most 2 lr per step); everything else agrees to fp32 noise
        assert np.mean(d > 1e-5) < 1e-3 and d.max() <= 2 * 5e-3 * steps + 1e-6, (mode, d.max(), np.mean(d > 1e-5))
    np.testing.assert_allclose(r0["sharded"], r0["allreduce"], rtol=0, atol=1e-6)
