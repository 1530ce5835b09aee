"""Golden vectors for the training-loop neighbours, produced by running
the REFERENCE package itself (this container only):

    python tests/golden/make_golden_train.py      # needs /root/reference and `make -C oracle ref`

Covers mcmc.find_dead / plan_relocation / apply_relocation / grow (mcmc.py:32-146),
training.inject_noise (training.py:276-292), the loss regularisers (training.py:98-131)
and exponential_lr (training.py:134-145).  Every random draw the reference makes is
replayed from a cloned numpy Generator and stored, so the device path can be fed the
identical uniforms / normals.  Output: tests/golden/train_aux.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import OUT, REPO, import_reference  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    import_reference()
    sys.path.insert(0, REPO)
    from betasplat import mcmc, training
    from betasplat.primitive import PrimitiveSet

    save = {}
    # ---- MCMC: many dead primitives (o < 0.005 <=> raw < -5.29), two SB lobes
    rng = np.random.default_rng(17)
    n, lobes = 3000, 2
    params = dict(positions=f32(rng.normal(0, 1, (n, 3))), opacity_raw=f32(rng.normal(-3.5, 2.5, n)),
                  rotations=f32(rng.normal(0, 1, (n, 4))), log_scales=f32(rng.normal(-3, 0.5, (n, 3))),
                  shapes=f32(rng.normal(0, 0.5, n)), base_colors=f32(rng.normal(0, 0.5, (n, 3))),
                  lobe_axes=f32(rng.normal(0, 1, (n, lobes, 3))), lobe_colors=f32(rng.normal(0, 0.3, (n, lobes, 3))))
    for k, v in params.items():
        save["in_" + k] = v
    prims = PrimitiveSet(**{k: v.copy() for k, v in params.items()})
    state = training.AdamState.zeros_for(prims)
    for buf in (state.exp_avg, state.exp_avg_sq):
        for k in buf:
            buf[k][...] = f32(rng.uniform(0.1, 1.0, buf[k].shape))
    for k in state.exp_avg:
        save["in_m_" + k] = state.exp_avg[k].copy()
        save["in_v_" + k] = state.exp_avg_sq[k].copy()

    seed = 23
    mrng = np.random.default_rng(seed)
    dead = mcmc.find_dead(prims)
    plan = mcmc.plan_relocation(prims, dead, mrng)
    mcmc.apply_relocation(prims, plan, state)
    for k, v in prims.parameters().items():  # snapshot: grow() adjusts its sources in place
        save["reloc_" + k] = v.copy()
    budget = n + 100
    grown = mcmc.grow(prims, budget, mrng, state)
    # replay the draws: plan_relocation draws len(dead) uniforms, grow draws n_add
    replay = np.random.default_rng(seed)
    n_add = min(int(mcmc.GROWTH_RATE * n), budget - n)
    save["u_plan"] = replay.random(dead.size)
    save["u_grow"] = replay.random(n_add)
    save["dead"] = dead
    save["targets"] = plan.targets
    save["budget"] = np.array(budget)
    for k, v in grown.parameters().items():
        save["grow_" + k] = v
    for k in state.exp_avg:
        save["grow_m_" + k] = state.exp_avg[k]
        save["grow_v_" + k] = state.exp_avg_sq[k]

    # ---- inject_noise (positions only), defaults of TrainConfig
    cfg = training.TrainConfig()
    nrng = np.random.default_rng(29)
    p2 = PrimitiveSet(**{k: v.copy() for k, v in params.items()})
    p2.opacity_raw[...] = f32(np.random.default_rng(30).normal(-2.0, 1.5, n))  # gate (1-o)^100 spread
    save["noise_opacity_raw"] = p2.opacity_raw.copy()
    lr = cfg.position_lr(1234, 2.5)
    save["noise_lr"] = np.array([cfg.noise_lr, lr])
    training.inject_noise(p2, cfg, lr, nrng)
    save["noise_eta"] = np.random.default_rng(29).standard_normal((n, 3))
    save["noise_positions"] = p2.positions

    # ---- regularisers through training.loss (lambda_opacity = lambda_scale = 0.01)
    rng = np.random.default_rng(31)
    a = f32(rng.uniform(0.0, 1.0, (24, 30, 3)))
    b = f32(np.clip(a + rng.normal(0, 0.1, a.shape), 0, 1))
    p3 = PrimitiveSet(**{k: v.copy() for k, v in params.items()})
    value, d_image, direct, parts = training.loss(a, b, p3, cfg, return_parts=True)
    save.update(reg_a=a, reg_b=b, reg_value=np.array(value), reg_d_image=d_image,
                reg_d_opacity_raw=direct["opacity_raw"], reg_d_log_scales=direct["log_scales"],
                reg_l1=np.array(parts["l1"]), reg_ssim_term=np.array(parts["ssim_term"]))

    # ---- exponential_lr table (with and without the delay ramp)
    steps = np.array([0, 1, 7, 100, 2999, 15000, 29999, 30000, 45000])
    save["lr_steps"] = steps
    save["lr_plain"] = np.array([training.exponential_lr(s, 1.6e-4, 1.6e-6, 30000) for s in steps])
    save["lr_delay"] = np.array([training.exponential_lr(s, 1.6e-4, 1.6e-6, 30000, 5000, 0.01) for s in steps])
    np.savez_compressed(os.path.join(OUT, "train_aux.npz"), **save)
    print("wrote", os.path.join(OUT, "train_aux.npz"), "dead", dead.size, "n_add", n_add)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def checkpoints():
    """Reference-written checkpoints (sceneio.save_checkpoint) of fp32-valued parameters."""
    import_reference()
    from betasplat import sceneio
    from betasplat.primitive import PrimitiveSet

    for name, n, lobes, seed in (("ckpt_l2.ply", 37, 2, 41), ("ckpt_l0.ply", 5, 0, 42)):
        rng = np.random.default_rng(seed)
        prims = PrimitiveSet(positions=f32(rng.normal(0, 1, (n, 3))), opacity_raw=f32(rng.normal(0, 1, n)),
                             rotations=f32(rng.normal(0, 1, (n, 4))), log_scales=f32(rng.normal(-3, 1, (n, 3))),
                             shapes=f32(rng.normal(0, 1, n)), base_colors=f32(rng.normal(0, 1, (n, 3))),
                             lobe_axes=f32(rng.normal(0, 1, (n, lobes, 3))),
                             lobe_colors=f32(rng.normal(0, 1, (n, lobes, 3))))
        sceneio.save_checkpoint(os.path.join(OUT, name), prims)
    print("wrote checkpoints")


def codec():
    """Reference-written archives (compression.pack, compression.py:141-187) plus the keys,
    permutation and unpacked values (compression.py:45-66, 190-250) they imply."""
    import shutil

    import_reference()
    from betasplat import compression
    from betasplat.primitive import PrimitiveSet

    save = {}
    cases = (("codec_l2", 777, 2, 51, True), ("codec_l0_keep", 50, 0, 52, False))
    for name, n, lobes, seed, sort in cases:
        rng = np.random.default_rng(seed)
        pos = f32(rng.normal(0, 2, (n, 3)))
        pos[n // 3] = pos[n // 5]  # a tie: the sort must stay stable
        prims = PrimitiveSet(positions=pos, opacity_raw=f32(rng.normal(0, 1, n)),
                             rotations=f32(rng.normal(0, 1, (n, 4))), log_scales=f32(rng.normal(-3, 1, (n, 3))),
                             shapes=np.zeros(n) if lobes == 0 else f32(rng.normal(0, 1, n)),  # constant channel
                             base_colors=f32(rng.normal(0, 1, (n, 3))),
                             lobe_axes=f32(rng.normal(0, 1, (n, lobes, 3))),
                             lobe_colors=f32(rng.normal(0, 1, (n, lobes, 3))))
        for k, v in prims.parameters().items():
            save[f"{name}_in_{k}"] = np.asarray(v, np.float64).copy()
        save[f"{name}_keys"] = compression.morton_keys(prims.positions)
        save[f"{name}_perm"] = compression.sort_primitives(prims)
        out = os.path.join(OUT, name)
        shutil.rmtree(out, ignore_errors=True)
        compression.pack(prims, out, sort=sort)
        back = compression.unpack(out)
        for k, v in back.parameters().items():
            save[f"{name}_out_{k}"] = np.asarray(v, np.float64).copy()
    np.savez_compressed(os.path.join(OUT, "codec.npz"), **save)
    print("wrote codec archives")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "checkpoints":
    checkpoints()
if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "codec":
    codec()
