"""Float64 restatement of reference objective.py / toy_env.log_token_dist over packed rows.

Test-only: see oracle/__init__.py.
"""
from __future__ import annotations

import math

import numpy as np


def log_token_dist(z: np.ndarray, temperature: float = 1.0) -> np.ndarray:
    """toy_env.py:157-175 for one row (TrainEngine)."""
    z = np.asarray(z, dtype=np.float64)
    if temperature != 1.0:
        z = z / temperature
    m = float(np.max(z))
    lse = m + float(np.log(np.sum(np.exp(z - m))))
    return z - lse


def triplet_value_slope(r, adv, eps_neg_low=0.2, eps_pos_high=0.2, eps_neg_high=3.0, guard_positive=True):
    """objective.py:133-150."""
    clipped = min(max(r, 1.0 - eps_neg_low), 1.0 + eps_pos_high)
    clip_slope = 1.0 if (1.0 - eps_neg_low) <= r <= (1.0 + eps_pos_high) else 0.0
    raw = r * adv
    capped = clipped * adv
    if raw <= capped:
        inner, inner_slope = raw, adv
    else:
        inner, inner_slope = capped, adv * clip_slope
    if guard_positive and adv > 0.0:
        return inner, inner_slope
    floor = eps_neg_high * adv
    if inner >= floor:
        return inner, inner_slope
    return floor, 0.0


def tis_weight(lt, li, cap):
    """objective.py:161-165."""
    return min(math.exp(lt - li), cap)


def token_terms(logits2d, rows, tokens, lt, li, sample_of_row, adv, use, temps, clip, norm=1.0):
    """Per-token (logp, term, coef) following objective.py:243-248 and 271-279 (coef = norm*w*slope*r/tau)."""
    n = len(tokens)
    logp = np.zeros(n)
    term = np.zeros(n)
    coefn = np.zeros(n)
    for k in range(n):
        s = int(sample_of_row[k])
        if not use[s]:
            continue
        z = logits2d[int(rows[k]) if rows is not None else k]
        lv = log_token_dist(z, temps[s])
        lp = float(lv[int(tokens[k])])
        r = math.exp(lp - lt[k])
        w = tis_weight(lt[k], li[k], clip["tis_cap"])
        v, sl = triplet_value_slope(r, adv[s], clip["eps_neg_low"], clip["eps_pos_high"], clip["eps_neg_high"],
                                    clip["guard_positive"])
        logp[k] = lp
        term[k] = w * v
        coefn[k] = norm * w * sl * r / temps[s]
    return logp, term, coefn


def objective(term, group_rows, G, t_max):
    """objective.py:237-250: per group sum / (G * T_max), mean over groups."""
    total = 0.0
    ng = len(group_rows) - 1
    for g in range(ng):
        g_sum = 0.0
        for k in range(group_rows[g], group_rows[g + 1]):
            g_sum += term[k]
        total += g_sum / (G * t_max)
    return total / ng if ng else 0.0


def gradient_rows(logits2d, rows, tokens, coef, temps_tok, out_rows_shape):
    """objective.py:271-282: grad[row] -= coef * p; grad[row][tok] += coef, tokens in order."""
    grad = np.zeros(out_rows_shape)
    for k in range(len(tokens)):
        c = coef[k]
        if c == 0.0:
            continue
        row = int(rows[k]) if rows is not None else k
        p = np.exp(log_token_dist(logits2d[row], temps_tok[k]))
        grad[row] -= c * p
        grad[row][int(tokens[k])] += c
    return grad
