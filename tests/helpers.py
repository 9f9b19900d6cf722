"""Shared helpers for the parity tests (bf16 rounding oracle-side, synthetic state dicts)."""
import numpy as np


def rne_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float64 values to bf16 with ONE rounding (RNE); returns uint16 bit patterns."""
    x = np.asarray(x, dtype=np.float64)
    # exact: decompose via float32 round-to-odd then RNE to bf16
    f = x.astype(np.float32)  # RN to f32
    back = f.astype(np.float64)
    u = f.view(np.uint32).copy()
    # convert RN-f32 to round-to-odd-f32: if inexact and rounded away, step toward x and set sticky
    inexact = back != x
    away = np.abs(back) > np.abs(x)
    u[inexact & away] -= 1  # truncate (toward zero) then set sticky bit
    u[inexact] |= 1
    u64 = u.astype(np.uint64)
    r = ((u64 + 0x7FFF + ((u64 >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    r[nan] = 0x7FC0
    return r


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def bf16_round(x):
    return bf16_bits_to_f64(rne_bf16_bits(x))


def mlp_dict_shapes(scale=1):
    """Config-1 toy MLP dict: 9,966,592 params at scale 1."""
    return {"embed": (1536 // scale, 1024), "fc1.w": (4096 // scale, 1024), "fc1.b": (4096 // scale,),
            "fc2.w": (1024, 4096 // scale), "fc2.b": (1024,)}


def synth_state_dicts(shapes, n_experts=3, seed=0, dtype_round=None):
    """base ~ N(0, 0.02^2); expert_i = base + N(0, (sigma_i 1e-3)^2), sigma_i = 1, 2, 3."""
    base, experts = {}, [dict() for _ in range(n_experts)]
    for t, (name, shp) in enumerate(shapes.items()):
        g = np.random.default_rng([seed, t])
        b = g.normal(0.0, 0.02, shp)
        if dtype_round:
            b = dtype_round(b)
        base[name] = b
        for i in range(n_experts):
            e = b + g.normal(0.0, (i + 1) * 1e-3, shp)
            experts[i][name] = dtype_round(e) if dtype_round else e
    return base, experts


def grad_rows_error(got, z, tokens, coef, temps, rtol, floor=1e-30):
    """Per-element parity of gradient rows with the reference (objective.py:271-282).

    got[k] is the kernel's row for token k (logits z[k], f64), coef[k] the kernel's own dJ/dlogit scale.
    The reference row is coef * (onehot(token) - softmax(z / T)) in float64; every entry must satisfy
    |got - ref| <= rtol * |coef| * (p + onehot) + floor, i.e. a RELATIVE bound on each softmax entry
    (entries down to ~1e-11 of the row are checked, not only the few above an absolute tolerance).
    Returns (max of |got - ref| / bound, index of that entry); the row passes iff the max <= 1."""
    worst, where = 0.0, None
    for k in range(len(tokens)):
        zz = np.asarray(z[k], dtype=np.float64) / temps[k]
        m = zz.max()
        e = np.exp(zz - m)
        p = e / e.sum()
        ref = -coef[k] * p
        ref[int(tokens[k])] += coef[k]
        onehot = np.zeros_like(p)
        onehot[int(tokens[k])] = 1.0
        bound = rtol * abs(coef[k]) * (p + onehot) + floor
        r = np.abs(np.asarray(got[k], dtype=np.float64) - ref) / bound
        j = int(np.argmax(r))
        if r[j] > worst:
            worst, where = float(r[j]), (k, j)
    return worst, where


def assert_grad_rows(got, z, tokens, coef, temps, rtol, floor=1e-30):
    worst, where = grad_rows_error(got, z, tokens, coef, temps, rtol, floor)
    assert worst <= 1.0, f"gradient entry {where} off by {worst:.3g}x the per-element bound (rtol {rtol})"
    # the check has teeth: the same rows with every non-target entry zeroed must fail it
    bad = np.array(got, dtype=np.float64, copy=True)
    for k in range(len(tokens)):
        if coef[k] != 0.0:
            keep = bad[k][int(tokens[k])]
            bad[k][:] = 0.0
            bad[k][int(tokens[k])] = keep
    if any(c != 0.0 for c in coef):
        assert grad_rows_error(bad, z, tokens, coef, temps, rtol, floor)[0] > 1.0
    return worst
