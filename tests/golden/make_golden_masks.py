"""Golden vectors for the host-side GRPO masking branches and the configs' error messages, generated from
the UNMODIFIED reference (build container only; the tests read the committed fixtures):

    OPENBLAS_NUM_THREADS=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_masks.py

Writes tests/golden/objective_masks.npz (batches with TRUNCATED samples with and without a tail repetition
loop, groups with fewer than two usable samples, GRADE_ERROR samples, MEAN_ONLY advantages; apply_masks'
masks / advantages and objective_value / objective_gradient on them) and tests/golden/errors.json (the
exception type and message of every validation branch of FusionConfig, ClipConfig, AdvantageConfig,
MaskedGroup, MaskedBatch, group_advantages, detect_repetition, apply_masks and tis_weight).
Reference lines: objective.py:40-203, fusion.py:54-76, toy_env.py:315-327.
"""
from __future__ import annotations

import json
import math
import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from rolloutlab import core, fusion, objective, toy_env  # noqa: E402

OUT = Path(__file__).resolve().parent


def _err(fn):
    try:
        fn()
    except Exception as exc:  # noqa: BLE001 - recording the reference's behaviour
        return type(exc).__name__, str(exc)
    return None, None


def _sample(pid, ctx, toks, status, reward, lt=None, li=None, tau=1.0):
    li = tuple(li) if li is not None else tuple(-1.0 for _ in toks)
    return core.Sample(prompt_id=pid, context_id=ctx, version_id=0, tokens=tuple(toks), infer_logps=li,
                       status=status, t_start=0, train_logps=None if lt is None else tuple(lt), reward=reward,
                       gen_temperature=tau)


def error_cases() -> list[dict]:
    """(constructor, JSON kwargs) -> (exception type, message) for every validation branch."""
    C = core.SampleStatus
    ok = _sample(0, 0, [1, 2], C.COMPLETE, core.RewardOutcome.passed())
    grp = core.Group(0, (ok, ok))
    cases = [
        ("FusionConfig", dict(dropout_p=1.0)), ("FusionConfig", dict(dropout_p=-0.1)),
        ("FusionConfig", dict(target_norm="median")), ("FusionConfig", dict(target_norm=0.0)),
        ("FusionConfig", dict(target_norm=-2)), ("FusionConfig", dict(merge_weights=[0.5, -0.1, 0.6])),
        ("FusionConfig", dict(merge_weights=[0.5, 0.3, 0.3])), ("FusionConfig", dict(erase_weighting="max")),
        ("FusionConfig", dict(dropout_p=0.3, target_norm=None, merge_weights=[0.2, 0.8])),
        ("ClipConfig", dict(eps_neg_low=0.0)), ("ClipConfig", dict(eps_neg_low=1.0)),
        ("ClipConfig", dict(eps_pos_high=0.0)), ("ClipConfig", dict(eps_neg_high=1.0)),
        ("ClipConfig", dict(eps_neg_high=1.1, eps_pos_high=0.2)), ("ClipConfig", dict(tis_cap=0.5)),
        ("ClipConfig", dict(eps_neg_low=0.1, eps_pos_high=0.3, eps_neg_high=1.3, tis_cap=1.0)),
        ("AdvantageConfig", dict(std_floor=0.0)), ("AdvantageConfig", dict(std_floor=-1.0)),
        ("group_advantages", dict(rewards=[1.0])), ("group_advantages", dict(rewards=[1.0, float("nan")])),
        ("group_advantages", dict(rewards=[1.0, float("inf"), 0.0])),
        ("detect_repetition", dict(tokens=[1, 2, 1, 2], ngram=0, min_repeats=3)),
        ("detect_repetition", dict(tokens=[1, 2, 1, 2], ngram=2, min_repeats=1)),
        ("tis_weight", dict(lt=float("nan"), li=-1.0, cap=2.0)),
        ("tis_weight", dict(lt=-1.0, li=float("-inf"), cap=2.0)),
        ("MaskedGroup", dict(advantages=[0.0], masks=2)), ("MaskedGroup", dict(advantages=[0.0, 0.0], masks=1)),
        ("MaskedBatch", dict(t_max=0)), ("MaskedBatch", dict(t_max=1)),
        ("MaskedBatch", dict(t_max=4, mixed_sizes=True)),
        ("apply_masks", dict(ungraded=True)),
        ("Group", dict(n=1)), ("Group", dict(n=2, mixed_prompts=True)),
    ]
    out = []
    for ctor, kw in cases:
        def call(ctor=ctor, kw=kw):
            if ctor == "FusionConfig":
                k = dict(kw)
                if "merge_weights" in k:
                    k["merge_weights"] = tuple(k["merge_weights"])
                return fusion.FusionConfig(**k)
            if ctor == "ClipConfig":
                return objective.ClipConfig(**kw)
            if ctor == "AdvantageConfig":
                return objective.AdvantageConfig(**kw)
            if ctor == "group_advantages":
                return objective.group_advantages(kw["rewards"], objective.AdvantageConfig())
            if ctor == "detect_repetition":
                return toy_env.detect_repetition(kw["tokens"], kw["ngram"], kw["min_repeats"])
            if ctor == "tis_weight":
                return objective.tis_weight(kw["lt"], kw["li"], kw["cap"])
            if ctor == "MaskedGroup":
                return objective.MaskedGroup(grp, tuple(kw["advantages"]), tuple([objective.Mask.USE] * kw["masks"]))
            if ctor == "MaskedBatch":
                mg = objective.MaskedGroup(grp, (0.0, 0.0), (objective.Mask.USE,) * 2)
                groups = (mg,)
                if kw.get("mixed_sizes"):
                    g3 = core.Group(1, tuple(_sample(1, 0, [1], C.COMPLETE, core.RewardOutcome.passed())
                                             for _ in range(3)))
                    groups = (mg, objective.MaskedGroup(g3, (0.0,) * 3, (objective.Mask.USE,) * 3))
                return objective.MaskedBatch(groups, kw["t_max"])
            if ctor == "apply_masks":
                bad = _sample(0, 0, [1], C.COMPLETE, None)
                return objective.apply_masks([core.Group(0, (ok, bad))], 4)
            if ctor == "Group":
                if kw.get("mixed_prompts"):
                    return core.Group(0, (ok, _sample(1, 0, [1], C.COMPLETE, core.RewardOutcome.passed())))
                return core.Group(0, (ok,) * kw["n"])
            raise AssertionError(ctor)
        et, msg = _err(call)
        # et None: a boundary value the reference accepts (recorded so the mirror must accept it too)
        out.append(dict(ctor=ctor, kwargs={k: (v if not (isinstance(v, float) and not math.isfinite(v)) else repr(v))
                                            for k, v in kw.items()}, exc=et, msg=msg))
    return out


def mask_cases() -> dict:
    """Batches exercising every apply_masks branch, with the reference's objective and gradient."""
    out = {}
    g = np.random.default_rng(17)
    C = core.SampleStatus
    C_ctx, T, V, G = 3, 12, 61, 4
    for cname, (rep, adv_cfg, tau) in {
        "rep_default": (objective.RepetitionConfig(), objective.AdvantageConfig(), 1.0),
        "rep_ngram3": (objective.RepetitionConfig(ngram=3, min_repeats=2), objective.AdvantageConfig(), 0.8),
        "mean_only": (objective.RepetitionConfig(ngram=1, min_repeats=4),
                      objective.AdvantageConfig(norm_mode=objective.NormMode.MEAN_ONLY), 1.0),
    }.items():
        logits = g.normal(0, 1.5, (C_ctx, T, V))
        params = toy_env.ParamTable(logits)
        n = rep.ngram * rep.min_repeats
        groups = []
        # per group: a list of (status, reward kind, tail-loop?) recipes
        recipes = [
            # truncated with a tail loop (kept, keeps its Fail), truncated without (masked), complete ones
            [(C.TRUNCATED, "fail", True), (C.TRUNCATED, "pass", False), (C.COMPLETE, "pass", False),
             (C.COMPLETE, "fail", False)],
            # fewer than two usable samples: one USE, the rest masked -> every advantage 0
            [(C.TRUNCATED, "pass", False), (C.COMPLETE, "pass", False), (C.COMPLETE, "grade_error", False),
             (C.TRUNCATED, "fail", False)],
            # no usable sample at all
            [(C.COMPLETE, "grade_error", False), (C.TRUNCATED, "fail", False), (C.TRUNCATED, "pass", False),
             (C.COMPLETE, "grade_error", False)],
            # a loop that is NOT at the tail (masked), a loop exactly at the tail, truncated too short for
            # the span (masked), complete with a loop (USE regardless)
            [(C.TRUNCATED, "fail", "mid"), (C.TRUNCATED, "fail", True), (C.TRUNCATED, "pass", "short"),
             (C.COMPLETE, "pass", True)],
        ]
        for gi, rec in enumerate(recipes):
            ctx = gi % C_ctx
            samples = []
            for status, kind, loop in rec:
                if loop == "short":
                    toks = [int(x) for x in g.integers(0, V, max(1, n - 1))]
                else:
                    L = int(g.integers(n + 2, T + 1))
                    toks = [int(x) for x in g.integers(0, V, L)]
                    unit = [int(x) for x in g.integers(0, V, rep.ngram)]
                    if loop is True:
                        toks[-n:] = unit * rep.min_repeats
                    elif loop == "mid":
                        toks[:n] = unit * rep.min_repeats
                        toks[-1] = (unit[-1] + 1) % V  # break any tail loop
                lt = [float(toy_env.log_token_dist(params, toy_env.TrainEngine(), ctx, t, tau)[tok]
                            + g.normal(0, 0.3)) for t, tok in enumerate(toks)]
                li = [x + float(g.normal(0, 0.05)) for x in lt]
                rw = {"pass": core.RewardOutcome.passed(), "fail": core.RewardOutcome.failed(),
                      "grade_error": core.RewardOutcome.grade_error()}[kind]
                samples.append(_sample(gi, ctx, toks, status, rw, lt, li, tau))
            groups.append(core.Group(gi, tuple(samples)))
        batch = objective.apply_masks(groups, T, rep, adv_cfg)
        clip = objective.ClipConfig()
        out[f"{cname}/logits"] = logits
        out[f"{cname}/value"] = np.array([objective.objective_value(batch, params, clip)])
        out[f"{cname}/grad"] = objective.objective_gradient(batch, params, clip)
        meta = []
        for mg in batch.groups:
            for s, a, mk in zip(mg.group.samples, mg.advantages, mg.masks):
                meta.append(dict(ctx=s.context_id, tokens=list(s.tokens), lt=list(s.train_logps),
                                 li=list(s.infer_logps), adv=a, mask=mk.value, tau=s.gen_temperature,
                                 status=s.status.value, reward=s.reward.raw_score, kind=s.reward.kind.value))
        out[f"{cname}/meta"] = np.array(json.dumps(dict(
            samples=meta, G=G, n_groups=len(groups), t_max=T, ngram=rep.ngram, min_repeats=rep.min_repeats,
            norm_mode=adv_cfg.norm_mode.value)))
    return out


if __name__ == "__main__":
    (OUT / "errors.json").write_text(json.dumps(error_cases(), indent=1))
    np.savez_compressed(OUT / "objective_masks.npz", **mask_cases())
    print("mask / error golden vectors written to", OUT)
