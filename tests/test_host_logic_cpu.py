"""CPU parity of the host-side logic the kernels rely on, against fixtures generated from the unmodified
reference (tests/golden/make_golden_masks.py): every validation branch raises the reference's exception
type and message, and apply_masks reproduces the reference's masks and advantages on batches with
TRUNCATED samples with and without a tail repetition loop and groups with fewer than two usable samples
(objective.py:40-203, fusion.py:54-76, toy_env.py:315-327)."""
import json
import math

import numpy as np
import pytest

from tests.conftest import GOLDEN

ERRORS = json.loads((GOLDEN / "errors.json").read_text())


def _f(v):
    return float(v) if isinstance(v, str) else v


def _call(ctor, kw):
    from paper_2509_18883_b200 import core, fusion, objective, toy_env
    C = core.SampleStatus

    def sample(pid, toks, reward):
        return core.Sample(prompt_id=pid, context_id=0, version_id=0, tokens=tuple(toks),
                           infer_logps=tuple(-1.0 for _ in toks), status=C.COMPLETE, t_start=0, reward=reward)
    ok = sample(0, [1, 2], core.RewardOutcome.passed())
    grp = core.Group(0, (ok, ok))
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
        return objective.group_advantages([_f(x) for x in kw["rewards"]], objective.AdvantageConfig())
    if ctor == "detect_repetition":
        return toy_env.detect_repetition(kw["tokens"], kw["ngram"], kw["min_repeats"])
    if ctor == "tis_weight":
        return objective.tis_weight(_f(kw["lt"]), _f(kw["li"]), kw["cap"])
    if ctor == "MaskedGroup":
        return objective.MaskedGroup(grp, tuple(kw["advantages"]), tuple([objective.Mask.USE] * kw["masks"]))
    if ctor == "MaskedBatch":
        mg = objective.MaskedGroup(grp, (0.0, 0.0), (objective.Mask.USE,) * 2)
        groups = (mg,)
        if kw.get("mixed_sizes"):
            g3 = core.Group(1, tuple(sample(1, [1], core.RewardOutcome.passed()) for _ in range(3)))
            groups = (mg, objective.MaskedGroup(g3, (0.0,) * 3, (objective.Mask.USE,) * 3))
        return objective.MaskedBatch(groups, kw["t_max"])
    if ctor == "apply_masks":
        return objective.apply_masks([core.Group(0, (ok, sample(0, [1], None)))], 4)
    if ctor == "Group":
        if kw.get("mixed_prompts"):
            return core.Group(0, (ok, sample(1, [1], core.RewardOutcome.passed())))
        return core.Group(0, (ok,) * kw["n"])
    raise AssertionError(ctor)


@pytest.mark.parametrize("case", ERRORS, ids=lambda c: f"{c['ctor']}-{c['kwargs']}")
def test_validation_messages_match_reference(case):
    if case["exc"] is None:
        _call(case["ctor"], case["kwargs"])  # the reference accepts this boundary value
        return
    with pytest.raises(Exception) as ei:
        _call(case["ctor"], case["kwargs"])
    assert type(ei.value).__name__ == case["exc"]
    assert str(ei.value) == case["msg"]


def rebuild_mask_batch(z, cname, apply=True):
    """Samples of a golden mask case as this package's records; apply_masks with the case's configs."""
    from paper_2509_18883_b200 import core, objective as O
    meta = json.loads(str(z[f"{cname}/meta"]))
    G = meta["G"]
    groups = []
    for gi in range(meta["n_groups"]):
        samples = []
        for s in meta["samples"][gi * G:(gi + 1) * G]:
            rw = core.RewardOutcome(core.RewardKind(s["kind"]), s["reward"])
            samples.append(core.Sample(prompt_id=gi, context_id=s["ctx"], version_id=0, tokens=tuple(s["tokens"]),
                                       infer_logps=tuple(s["li"]), status=core.SampleStatus(s["status"]), t_start=0,
                                       train_logps=tuple(s["lt"]), reward=rw, gen_temperature=s["tau"]))
        groups.append(core.Group(gi, tuple(samples)))
    rep = O.RepetitionConfig(ngram=meta["ngram"], min_repeats=meta["min_repeats"])
    adv = O.AdvantageConfig(norm_mode=O.NormMode(meta["norm_mode"]))
    return O.apply_masks(groups, meta["t_max"], rep, adv), meta


@pytest.mark.parametrize("cname", ["rep_default", "rep_ngram3", "mean_only"])
def test_apply_masks_branches_match_reference(cname):
    z = np.load(GOLDEN / "objective_masks.npz")
    batch, meta = rebuild_mask_batch(z, cname)
    got = [(m.value, a) for mg in batch.groups for m, a in zip(mg.masks, mg.advantages)]
    want = [(s["mask"], s["adv"]) for s in meta["samples"]]
    assert got == want  # exact: same host float64 arithmetic
    # the fixture covers every branch: kept truncation (tail loop), masked truncation, grade error,
    # a group with exactly one usable sample and a group with none (all advantages 0)
    statuses = {(s["status"], s["mask"]) for s in meta["samples"]}
    assert {("truncated", "use"), ("truncated", "mask_truncated"), ("complete", "mask_grade_error")} <= statuses
    G = meta["G"]
    usable = [sum(s["mask"] == "use" for s in meta["samples"][g * G:(g + 1) * G]) for g in range(meta["n_groups"])]
    assert 0 in usable and 1 in usable
    for g, u in enumerate(usable):
        if u < 2:
            assert all(s["adv"] == 0.0 for s in meta["samples"][g * G:(g + 1) * G])


def test_grpo_batch_shard_and_select_cpu():
    """GRPOBatch.shard: contiguous sample ranges balanced by rows, covering every sample once, with the
    global normalisation and sample slots kept (the all-reduce of per-sample sums relies on it)."""
    import numpy as np
    import torch
    from paper_2509_18883_b200 import objective as O
    lens = [7, 0, 3, 12, 1, 9, 4, 4]
    cu = np.concatenate([[0], np.cumsum(lens)])
    R = int(cu[-1])
    b = O.GRPOBatch.pack(np.arange(R), np.zeros(R), np.zeros(R), cu, np.arange(8.0), np.ones(8, np.uint8), 4, 12,
                         device=torch.device("cpu"))
    for world in (1, 2, 3, 4, 8, 11):
        bounds = b.shard_bounds(world)
        assert bounds[0] == 0 and bounds[-1] == 8 and bounds == sorted(bounds) and len(bounds) == world + 1
        rows = []
        for r in range(world):
            s = b.shard(world, r)
            assert s.sample_base == bounds[r] and s.n_samples == 8 and s.n_groups == 2
            assert s.n_local_samples == bounds[r + 1] - bounds[r]
            assert torch.equal(s.adv, b.adv[bounds[r]:bounds[r + 1]])
            assert torch.equal(s.norm, b.norm[bounds[r]:bounds[r + 1]])
            assert s.sample_rows_host[0] == 0 and s.sample_rows_host[-1] == s.n_rows
            if s.n_rows:
                assert int(s.sample_of_row.min()) >= 0 and int(s.sample_of_row.max()) < s.n_local_samples
            rows.extend(s.tokens.tolist())
        assert rows == list(range(R))
    with pytest.raises(IndexError):
        b.select(3, 9)
