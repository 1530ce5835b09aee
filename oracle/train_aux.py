"""ORACLE -- test infrastructure only (never imported by the product package).

fp64 numpy restatement of the training-loop neighbours of the hot path (SURVEY 8(f)
rank 2), with every random draw passed in explicitly so the device kernels can be fed the
same numbers.  Paths relative to /root/reference/pkg/src/betasplat/:

  find_dead            mcmc.py:32-36
  sample_live          mcmc.py:49-70 / 108-128 (+ numpy Generator.choice with p: cdf =
                       cumsum(p) / cdf[-1], idx = searchsorted(cdf, u, side="right"))
  apply_relocation     mcmc.py:86-106
  grow                 mcmc.py:108-146
  inject_noise         training.py:276-292 (kernel.beta_eval kernel.py:47-57,
                       primitive.covariance_many primitive.py:75-80)
  regularizers         training.py:112-124
  exponential_lr       training.py:134-145

Pinned against golden vectors produced by the reference package itself
(tests/golden/make_golden_train.py -> tests/golden/train_aux.npz) in tests/test_oracle.py.
Parameters are dicts of fp64 arrays keyed like PrimitiveSet.parameters().
"""

from __future__ import annotations

import numpy as np

from .pipeline import covariance_many, sigmoid

DEAD_THRESHOLD = 0.005
NOISE_EXPONENT = 4.0 * 25.0  # beta_eval(o, ln 25): (1 - o)^(4 e^{ln 25})


def logit(p):
    p = np.clip(np.asarray(p, dtype=np.float64), 1e-12, 1.0 - 1e-12)
    return np.log(p) - np.log1p(-p)


def find_dead(opacity_raw, threshold=DEAD_THRESHOLD):
    return np.flatnonzero(sigmoid(opacity_raw) < threshold)


def sample_live(opacity_raw, uniforms, threshold=DEAD_THRESHOLD, exclude=None):
    """Indices drawn with odds o / sum(o) over live = {o >= threshold} minus ``exclude``."""
    o = sigmoid(opacity_raw)
    live_mask = o >= threshold
    if exclude is not None and len(exclude):
        live_mask[np.asarray(exclude)] = False
    live = np.flatnonzero(live_mask)
    if live.size == 0:
        raise RuntimeError("no live primitives")
    p = o[live] / o[live].sum()
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    return live[np.searchsorted(cdf, np.asarray(uniforms), side="right")]


def adjusted_logit(o, mult, floor):
    """logit(max(new_opacity(o, mult), floor))  (mcmc.py:73-83, 100-102)."""
    p = o if mult == 1 else 1.0 - (1.0 - o) ** (1.0 / mult)
    return logit(max(p, floor))


def apply_relocation(params, moments, dead, targets, floor=DEAD_THRESHOLD):
    """In place on ``params`` (dict of arrays) and ``moments`` (list of such dicts)."""
    dead, targets = np.asarray(dead), np.asarray(targets)
    if dead.size == 0:
        return params
    o = sigmoid(params["opacity_raw"])
    uniq, cnt = np.unique(targets, return_counts=True)
    for t, c in zip(uniq, cnt):
        copies = dead[targets == t]
        for name, arr in params.items():
            if name != "opacity_raw":
                arr[copies] = arr[t]
        adj = adjusted_logit(float(o[t]), int(c) + 1, floor)
        params["opacity_raw"][copies] = adj
        params["opacity_raw"][t] = adj
    touched = np.concatenate([dead, uniq])
    for mom in moments:
        for arr in mom.values():
            arr[touched] = 0.0
    return params


def grow(params, moments, sources, floor=DEAD_THRESHOLD):
    """Returns (grown params, grown moments) for the drawn ``sources``."""
    sources = np.asarray(sources)
    o = sigmoid(params["opacity_raw"])
    new_rows = {k: v[sources].copy() for k, v in params.items()}
    uniq, cnt = np.unique(sources, return_counts=True)
    params = {k: v.copy() for k, v in params.items()}
    for t, c in zip(uniq, cnt):
        adj = adjusted_logit(float(o[t]), int(c) + 1, floor)
        params["opacity_raw"][t] = adj
        new_rows["opacity_raw"][sources == t] = adj
    grown = {k: np.concatenate([v, new_rows[k]], axis=0) for k, v in params.items()}
    out_m = []
    for mom in moments:
        m = {k: v.copy() for k, v in mom.items()}
        for arr in m.values():
            arr[uniq] = 0.0
        out_m.append({k: np.concatenate([v, np.zeros((sources.size,) + v.shape[1:])], axis=0)
                      for k, v in m.items()})
    return grown, out_m


def inject_noise(params, noise_lr, position_lr, eta):
    o = sigmoid(params["opacity_raw"])
    gate = (1.0 - np.clip(o, 0.0, 1.0)) ** NOISE_EXPONENT
    cov = covariance_many(params["rotations"], np.exp(params["log_scales"]))
    return params["positions"] + noise_lr * position_lr * gate[:, None] * np.einsum("nij,nj->ni", cov, eta)


def regularizers(opacity_raw, log_scales, lambda_opacity, lambda_scale):
    """(value term, d opacity_raw, d log_scales)."""
    o = sigmoid(opacity_raw)
    s = np.exp(log_scales)
    value = lambda_opacity * float(o.sum()) + lambda_scale * float(s.sum())
    return value, lambda_opacity * o * (1.0 - o), lambda_scale * s


def exponential_lr(step, lr_init, lr_final, max_steps, delay_steps=0, delay_mult=0.01):
    t = np.clip(step / max_steps, 0.0, 1.0)
    lr = float(np.exp((1.0 - t) * np.log(lr_init) + t * np.log(lr_final)))
    if delay_steps > 0:
        u = np.clip(step / delay_steps, 0.0, 1.0)
        lr *= delay_mult + (1.0 - delay_mult) * np.sin(0.5 * np.pi * u)
    return lr
