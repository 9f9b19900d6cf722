"""Float64 restatement of reference fusion.py (task vectors, normalise, dropout, erase, fuse).

Operates on flat float64 arrays (one tensor = the reference's ParamTable.reshape(1, 1, -1)).
Test-only: see oracle/__init__.py.
"""
from __future__ import annotations

import numpy as np

from . import rng as R

MEAN = "mean_of_inputs"


def norm(delta: np.ndarray) -> float:
    """fusion.py:44: float(np.linalg.norm(delta))."""
    return float(np.linalg.norm(delta))


def normalize(deltas, norms, target_norm):
    """fusion.py:86-102.  Returns (new deltas, new norms, scale factors (1.0 where untouched))."""
    if target_norm is None:
        return list(deltas), list(norms), [1.0] * len(deltas)
    nonzero = [n for n in norms if n > 0.0]
    if isinstance(target_norm, str):
        if not nonzero:
            raise ValueError("cannot take mean norm of all-zero task vectors")
        target = sum(nonzero) / len(nonzero)
    else:
        target = float(target_norm)
    out, out_norms, scales = [], [], []
    for d, n in zip(deltas, norms):
        if n == 0.0:
            out.append(d)
            out_norms.append(n)
            scales.append(1.0)
        else:
            s = target / n
            nd = d * s
            out.append(nd)
            out_norms.append(norm(nd))
            scales.append(s)
    return out, out_norms, scales


def dropout(delta: np.ndarray, p: float, counter0: int) -> np.ndarray:
    """fusion.py:105-115 with draw j keyed by the flat index j."""
    if p == 0.0:
        return delta
    kept = R.keep_mask(counter0, 0, delta.size, p)
    return np.where(kept, delta / (1.0 - p), 0.0)


def erase(deltas, weighting="sum"):
    """fusion.py:118-142."""
    stack = np.stack(deltas)
    if weighting == "sum":
        vote = stack.sum(axis=0)
    else:
        vote = (np.sign(stack) * stack ** 2).sum(axis=0)
    majority = np.sign(vote)
    return [np.where((majority != 0) & (np.sign(d) == -majority), 0.0, d) for d in deltas]


def fuse(base: np.ndarray, experts, *, dropout_p=0.0, target_norm=MEAN, merge_weights=None, erase_mode=True,
         erase_weighting="sum", seed=0):
    """fusion.py:154-188 on flat f64 arrays.  Returns (fused, stats dict)."""
    base = np.asarray(base, dtype=np.float64).ravel()
    deltas = [np.asarray(e, dtype=np.float64).ravel() - base for e in experts]
    n = len(deltas)
    weights = merge_weights or tuple(1.0 / n for _ in range(n))
    norms_before = [norm(d) for d in deltas]
    cur, norms_after, scales = normalize(deltas, norms_before, target_norm)
    if dropout_p > 0.0:
        cur = [dropout(d, dropout_p, R.fusion_child_seed(seed, i)) for i, d in enumerate(cur)]
    kept = [float(np.count_nonzero(d)) / d.size for d in cur]
    pre = cur
    if erase_mode and n >= 2:
        cur = erase(cur, erase_weighting)
    erased = [int(np.count_nonzero(a) - np.count_nonzero(b)) for a, b in zip(pre, cur)]
    fused = base.copy()
    for w, d in zip(weights, cur):
        fused = fused + w * d
    stats = dict(norms_before=norms_before, norms_after=norms_after, kept=kept, erased=erased,
                 weights=list(weights), scales=scales)
    return fused, stats


def erase_decisions(base, experts, scales, *, dropout_p=0.0, seed=0, erase_weighting="sum", j0=0):
    """Zero pattern after erase for flat slices [j0, j0+len) given the per-expert scales (the closed
    form used for sampled parity at full size): returns (kept_after_dropout[n, L], erased[n, L])."""
    base = np.asarray(base, dtype=np.float64)
    ks = []
    keeps = []
    for i, e in enumerate(experts):
        d = np.asarray(e, dtype=np.float64) - base
        k = d * scales[i]
        if dropout_p > 0.0:
            keep = R.keep_mask(R.fusion_child_seed(seed, i), j0, d.size, dropout_p)
            k = np.where(keep, k / (1.0 - dropout_p), 0.0)
        ks.append(k)
        keeps.append(k != 0)
    after = erase(ks, erase_weighting) if len(ks) >= 2 else ks
    erased = [(a != 0) & (b == 0) for a, b in zip(ks, after)]
    return np.array(keeps), np.array(erased), ks, after
