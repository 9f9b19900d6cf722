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
