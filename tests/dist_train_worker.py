"""Worker of tests/test_gpu_distributed.py: one rank of a view-batch DP TrainStep on the
single GPU (gloo process group, CUDA tensors staged through the host), or the single-process
reference over all views.  Writes its result to OUT/rank{r}.npz."""

import os
import sys

import numpy as np
import torch


def run(rank, world, port, out_dir, n_views, steps):
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, repo)
    from paper_2501_18630_b200 import PrimitiveSet
    from paper_2501_18630_b200 import distributed as dd
    from paper_2501_18630_b200.scenes import make_workload, target_scene
    from paper_2501_18630_b200.training import TrainStep, render_targets

    pg = None
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                          LOCAL_RANK="0")
        torch.cuda.set_device(0)
        torch.distributed.init_process_group("gloo")
        pg = torch.distributed.group.WORLD
    wl = make_workload("c3", seed=0, n=20_000, views=n_views, width=128, height=96)
    cams = wl.cameras
    tgt = render_targets(PrimitiveSet.from_scene(target_scene("c3", 1, 20_000)), cams, wl.background)
    mine = list(dd.partition_views(n_views, world, rank)) if world > 1 else list(range(n_views))
    res = {}
    for mode in ("allreduce", "sharded"):
        prims = PrimitiveSet.from_scene(wl.scene)
        st = TrainStep(prims, [cams[v] for v in mine], [tgt[v] for v in mine], wl.background, process_group=pg,
                       shard_optimizer=(mode == "sharded"), deterministic=True)
        st.step(check=True, adam=False)  # gradients only (summed over all views)
        torch.cuda.synchronize()
        if mode == "allreduce":
            res["grad"] = st.grads.flat.cpu().numpy().copy()
        st.grads.flat.zero_()
        for _ in range(steps):
            st.step()
        torch.cuda.synchronize()
        res[mode] = prims.flat.cpu().numpy().copy()
    np.savez(os.path.join(out_dir, f"rank{rank}_w{world}.npz"), **res)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    r, w, port, out, nv, steps = sys.argv[1:7]
    run(int(r), int(w), int(port), out, int(nv), int(steps))
