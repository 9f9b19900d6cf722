"""SPEC.md worked examples written against the reference's own API (`rolloutlab.*`), run unchanged
against whichever implementation `rolloutlab` resolves to: the reference itself, or this package
installed under that name by `swap_in()` (the import swap a user would make).

Every result is converted with `to_np` (reference: numpy / float; this package: CUDA tensors)."""
from __future__ import annotations

import importlib
import math
import sys
import types
from contextlib import contextmanager

import numpy as np

MODULES = ("core", "toy_env", "fusion", "objective")


@contextmanager
def swap_in():
    """Install paper_2509_18883_b200.{core,toy_env,fusion,objective} as rolloutlab.* for the duration."""
    saved = {k: v for k, v in sys.modules.items() if k == "rolloutlab" or k.startswith("rolloutlab.")}
    for k in saved:
        del sys.modules[k]
    pkg = types.ModuleType("rolloutlab")
    pkg.__path__ = []
    sys.modules["rolloutlab"] = pkg
    for m in MODULES:
        mod = importlib.import_module(f"paper_2509_18883_b200.{m}")
        sys.modules[f"rolloutlab.{m}"] = mod
        setattr(pkg, m, mod)
    try:
        yield
    finally:
        for k in [k for k in sys.modules if k == "rolloutlab" or k.startswith("rolloutlab.")]:
            del sys.modules[k]
        sys.modules.update(saved)


def to_np(x):
    if hasattr(x, "logits"):  # ParamTable
        x = x.logits
    if hasattr(x, "delta") and not isinstance(x, np.ndarray):  # TaskVector
        x = x.delta
    if hasattr(x, "detach"):  # torch
        return x.detach().double().cpu().numpy()
    if isinstance(x, (list, tuple)):
        return np.array([float(v) for v in x])
    return np.asarray(x, dtype=np.float64)


def run_examples() -> dict:
    from rolloutlab import core, fusion, objective, toy_env
    PT = lambda a: toy_env.ParamTable(np.asarray(a, dtype=np.float64).reshape(1, 1, -1))
    out = {}
    # ---- group_advantages (SPEC.md: [1,0,0,1] MeanStd -> [1,-1,-1,1]; identical -> 0; [1,0] MeanOnly)
    A = objective.AdvantageConfig
    out["adv/meanstd"] = to_np(objective.group_advantages([1.0, 0.0, 0.0, 1.0], A()))
    out["adv/identical"] = to_np(objective.group_advantages([1.0, 1.0, 1.0, 1.0], A()))
    out["adv/meanonly"] = to_np(objective.group_advantages([1.0, 0.0], A(norm_mode=objective.NormMode.MEAN_ONLY)))
    # ---- triplet clip and TIS weight
    cfg = objective.ClipConfig(eps_neg_low=0.2, eps_pos_high=0.2, eps_neg_high=2.0)
    out["clip/on_policy"] = objective.triplet_clip_term(1.0, 1.0, objective.ClipConfig())
    out["clip/pos"] = objective.triplet_clip_term(1.5, 2.0, cfg)
    out["clip/neg"] = objective.triplet_clip_term(3.0, -1.0, cfg)
    out["tis/equal"] = objective.tis_weight(-1.0, -1.0, 2.0)
    out["tis/capped"] = objective.tis_weight(math.log(1.8), 0.0, 1.5)
    out["tis/free"] = objective.tis_weight(math.log(0.9), 0.0, 1.5)
    # ---- task vectors and the fusion stages
    base = PT([0.5, -1.0, 2.0, 0.0])
    out["tv/zero_norm"] = fusion.task_vector(base, base).norm
    out["tv/one_entry"] = to_np(fusion.task_vector(PT([0.5, -0.5, 2.0, 0.0]), base))
    t2, t4 = (fusion.task_vector(PT(np.array([0.5, -1.0, 2.0, 0.0]) + np.array(v)), base)
              for v in ([2.0, 0.0, 0.0, 0.0], [0.0, 4.0, 0.0, 0.0]))
    nm = fusion.normalize_magnitudes([t2, t4], fusion.FusionConfig())
    out["norm/mean"] = np.array([t.norm for t in nm])
    rng = core.make_rng(3, "spec-dropout")
    out["dropout/p0"] = to_np(fusion.dropout_prune(t2, 0.0, rng))
    tvd = fusion.task_vector(PT([0.9] * 64), PT([0.5] * 64))
    out["dropout/p05"] = to_np(fusion.dropout_prune(tvd, 0.5, core.make_rng(11, "spec-dropout")))
    e = lambda v: fusion.task_vector(PT(np.array([0.5, -1.0, 2.0, 0.0]) + np.array(v)), base)
    out["erase/majority"] = np.stack([to_np(t) for t in fusion.erase_minority(
        [e([0.3, 0, 0, 0]), e([0.1, 0, 0, 0]), e([-0.2, 0, 0, 0])])])
    out["erase/tie"] = np.stack([to_np(t) for t in fusion.erase_minority([e([0.1, 0, 0, 0]), e([-0.1, 0, 0, 0])])])
    rl = PT([0.25, 3.0, -1.5, 7.0])
    ident = fusion.FusionConfig(dropout_p=0.0, target_norm=None, merge_weights=(1.0,), erase_mode=False)
    out["merge/round_trip"] = to_np(fusion.merge(base, [fusion.task_vector(rl, base)], ident))
    two = fusion.FusionConfig(target_norm=None, merge_weights=(0.5, 0.5), erase_mode=False)
    out["merge/identical"] = to_np(fusion.merge(base, [fusion.task_vector(rl, base)] * 2, two))
    opp = fusion.FusionConfig(target_norm=None)
    out["merge/opposite_tie"] = to_np(fusion.merge(base, [e([1.0, 0, 0, 0]), e([-1.0, 0, 0, 0])], opp))
    # ---- a full fuse with statistics (seeded dropout, mean-norm, erase)
    g = np.random.default_rng(7)
    b = g.normal(0, 0.02, 3001)
    xs = [b + g.normal(0, 1e-3 * (i + 1), 3001) for i in range(3)]
    fused, st = fusion.fuse(PT(b), [fusion.task_vector(PT(x), PT(b)) for x in xs],
                            fusion.FusionConfig(dropout_p=0.3, seed=5))
    out["fuse/values"] = to_np(fused).reshape(-1)
    out["fuse/norms_before"] = to_np(st.norms_before)
    out["fuse/kept"] = to_np(st.dropout_kept_fraction)
    out["fuse/erased"] = to_np(st.erased_counts)
    # ---- objective value / gradient / ascent on the tabular policy (SPEC on-policy example)
    C, T, V, G = 2, 4, 9, 2
    params = toy_env.ParamTable(g.normal(0, 1.0, (C, T, V)))
    eng = toy_env.TrainEngine()
    samples = []
    for si in range(G):
        toks = tuple(int(t) for t in g.integers(0, V, T - si))  # unequal lengths: J = sum_i A_i L_i / (G T_max)
        lt = tuple(float(toy_env.log_token_dist(params, eng, 0, t, 1.0)[tok]) for t, tok in enumerate(toks))
        rw = core.RewardOutcome.passed() if si == 0 else core.RewardOutcome.failed()
        samples.append(core.Sample(prompt_id=0, context_id=0, version_id=0, tokens=toks, infer_logps=lt,
                                   status=core.SampleStatus.COMPLETE, t_start=0, train_logps=lt, reward=rw,
                                   gen_temperature=1.0))
    batch = objective.apply_masks([core.Group(0, tuple(samples))], T)
    clip = objective.ClipConfig()
    out["obj/advantages"] = to_np(batch.groups[0].advantages)
    out["obj/value"] = float(objective.objective_value(batch, params, clip))
    grad = objective.objective_gradient(batch, params, clip)
    out["obj/gradient"] = to_np(grad)
    out["obj/ascent"] = to_np(objective.ascent_step(params, to_np(grad), 0.1))
    return out


# values SPEC.md states outright (the rest are compared implementation against implementation)
SPEC_EXPECTED = {
    "adv/meanstd": [1.0, -1.0, -1.0, 1.0], "adv/identical": [0.0] * 4, "adv/meanonly": [0.5, -0.5],
    "clip/on_policy": 1.0, "clip/neg": -2.0, "tis/equal": 1.0, "tis/capped": 1.5, "tis/free": 0.9,
    "tv/zero_norm": 0.0, "tv/one_entry": [0.0, 0.5, 0.0, 0.0], "norm/mean": [3.0, 3.0],
    "dropout/p0": [2.0, 0.0, 0.0, 0.0], "erase/tie": [[0.1, 0, 0, 0], [-0.1, 0, 0, 0]],
    "erase/majority": [[0.3, 0, 0, 0], [0.1, 0, 0, 0], [0.0, 0, 0, 0]],
    "merge/round_trip": [0.25, 3.0, -1.5, 7.0], "merge/identical": [0.25, 3.0, -1.5, 7.0],
    "merge/opposite_tie": [0.5, -1.0, 2.0, 0.0],
}
