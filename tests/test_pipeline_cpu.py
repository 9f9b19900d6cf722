"""Sample-intake pipeline vs fixtures generated from the unmodified reference (tests/golden/pipeline_kat.json,
made by tests/golden/make_golden_pipeline.py from rolloutlab/pipeline.py).  Every offer's decision, emitted
batch order, stale drops, reuse count, pending list and buffer contents, and the rng state afterwards,
must match exactly."""
import json
from pathlib import Path

import pytest

from paper_2509_18883_b200 import core as C
from paper_2509_18883_b200 import pipeline as P

KAT = json.loads((Path(__file__).resolve().parent / "golden" / "pipeline_kat.json").read_text())
KINDS = {"pass": C.RewardOutcome.passed, "fail": C.RewardOutcome.failed,
         "grade_error": C.RewardOutcome.grade_error, "none": lambda: None}


def make_group(spec):
    pid, versions, kinds = spec
    return C.Group(pid, tuple(C.Sample(prompt_id=pid, context_id=0, version_id=v, tokens=(1, 2),
                                       infer_logps=(-1.0, -1.0), status=C.SampleStatus.COMPLETE, t_start=0,
                                       reward=KINDS[k]()) for v, k in zip(versions, kinds)))


def ids(groups):
    return None if groups is None else [g.prompt_id for g in groups]


@pytest.mark.parametrize("sc", KAT["assembler"], ids=[s["name"] for s in KAT["assembler"]])
def test_assembler_stream_vs_reference(sc):
    buf = None if sc["capacity"] is None else P.ReplayBuffer(sc["capacity"], sc["reuse_ratio"])
    asm = P.BatchAssembler(sc["batch_groups"], P.StalenessPolicy(sc["max_staleness"]), buf, C.Rng(sc["seed"]))
    version = sc["start_version"]
    side = iter(sc["side"])
    for i, (item, want) in enumerate(zip(sc["stream"], sc["trace"], strict=True)):
        if buf is not None and sc["side_every"] and i % sc["side_every"] == 0:
            extra = next(side)
            buf.insert(make_group((extra["pid"], [max(0, version - l) for l in extra["lags"]], extra["kinds"])))
        res = asm.offer(make_group((item["pid"], [max(0, version - l) for l in item["lags"]], item["kinds"])), version)
        got = {"version": version, "decision": res.decision.value, "batch": ids(res.batch),
               "dropped": ids(res.dropped_stale), "reused": res.reused_count, "pending": ids(asm.pending),
               "buffer": None if buf is None else ids(buf.entries)}
        assert got == want, f"offer {i}"
        if res.batch is not None:
            version += 1
            # SPEC invariants: no all-pass / all-fail group, nothing past the staleness bound
            for g in res.batch:
                assert P.online_filter(g) is P.FilterDecision.KEEP
                assert P.staleness_check(g, got["version"], asm.policy) is P.StalenessDecision.REUSE
        if buf is not None:
            assert len(buf.entries) <= buf.capacity
    assert hex(asm.rng.next_u64()) == sc["rng_after"]


@pytest.mark.parametrize("k", range(len(KAT["mix"])))
def test_buffer_mix_vs_reference(k):
    m = KAT["mix"][k]
    buf = P.ReplayBuffer(m["capacity"], m["reuse_ratio"])
    for s in m["buffer_specs"]:
        buf.insert(make_group(s))
    assert ids(buf.entries) == m["buffer_before"]
    policy = P.StalenessPolicy(m["max_staleness"])
    assert buf.valid_count(m["version"], policy) == m["valid_before"]
    fresh = [make_group(s) for s in m["fresh_specs"]]
    rng = C.Rng(m["seed"])
    batch = P.buffer_mix(buf, fresh, m["batch_groups"], m["version"], policy, rng)
    assert ids(batch) == m["batch"]
    assert ids(buf.entries) == m["buffer_after"]
    assert ids(fresh) == m["fresh_after"]  # the caller's list is never modified
    assert hex(rng.next_u64()) == m["rng_after"]


def test_assemble_batch_generator_vs_reference():
    gcase = KAT["generator"]
    v = gcase["version"]
    groups = [make_group((s["pid"], [max(0, v - l) for l in s["lags"]], s["kinds"])) for s in gcase["stream"]]
    buf = P.ReplayBuffer(gcase["capacity"], gcase["reuse_ratio"])
    got = [ids(b) for b in P.assemble_batch(iter(groups), gcase["batch_groups"],
                                            P.StalenessPolicy(gcase["max_staleness"]), v, buf, C.Rng(gcase["seed"]))]
    assert got == gcase["batches"]
    assert ids(buf.entries) == gcase["buffer_after"]


def _catch(fn):
    try:
        r = fn()
    except Exception as e:  # noqa: BLE001
        return [type(e).__name__, str(e)]
    return ["ok", r.value if hasattr(r, "value") else repr(r)]


SPEC_CASES = {
    "filter_all_pass": lambda: P.online_filter(make_group((1, [0] * 4, ["pass"] * 4))),
    "filter_mixed": lambda: P.online_filter(make_group((1, [0] * 4, ["pass", "fail", "fail", "pass"]))),
    "filter_all_error": lambda: P.online_filter(make_group((1, [0] * 4, ["grade_error"] * 4))),
    "filter_all_fail": lambda: P.online_filter(make_group((1, [0] * 3, ["fail"] * 3))),
    "filter_pass_error": lambda: P.online_filter(make_group((1, [0] * 3, ["pass", "grade_error", "pass"]))),
    "filter_ungraded": lambda: P.online_filter(make_group((7, [0] * 3, ["pass", "none", "fail"]))),
    "filter_ungraded_first_error": lambda: P.online_filter(make_group((8, [0] * 2, ["grade_error", "none"]))),
    "stale_5_7_2": lambda: P.staleness_check(make_group((1, [5, 5], ["pass", "fail"])), 7, P.StalenessPolicy(2)),
    "stale_5_8_2": lambda: P.staleness_check(make_group((1, [5, 5], ["pass", "fail"])), 8, P.StalenessPolicy(2)),
    "stale_5_5_0": lambda: P.staleness_check(make_group((1, [5, 5], ["pass", "fail"])), 5, P.StalenessPolicy(0)),
    "stale_mixed_birth": lambda: P.staleness_check(make_group((1, [2, 6], ["pass", "fail"])), 8,
                                                   P.StalenessPolicy(2)),
    "stale_future": lambda: P.staleness_check(make_group((1, [9, 3], ["pass", "fail"])), 8, P.StalenessPolicy(2)),
    "policy_negative": lambda: P.StalenessPolicy(-1),
    "buffer_capacity0": lambda: P.ReplayBuffer(0, 0.5),
    "buffer_ratio1": lambda: P.ReplayBuffer(4, 1.0),
    "buffer_ratio_neg": lambda: P.ReplayBuffer(4, -0.1),
    "mix_batch0": lambda: P.buffer_mix(P.ReplayBuffer(2, 0.5), [], 0, 0, P.StalenessPolicy(2), C.Rng(1)),
    "assembler_batch0": lambda: P.BatchAssembler(0, P.StalenessPolicy(2)),
    "assembler_ungraded": lambda: P.BatchAssembler(2, P.StalenessPolicy(2)).offer(
        make_group((5, [0, 0], ["none", "pass"])), 0),
    "assembler_future": lambda: P.BatchAssembler(2, P.StalenessPolicy(2)).offer(
        make_group((5, [4, 0], ["fail", "pass"])), 1),
}


@pytest.mark.parametrize("name", sorted(KAT["spec"]))
def test_spec_examples_and_errors_vs_reference(name):
    assert _catch(SPEC_CASES[name]) == KAT["spec"][name]


def test_spec_buffer_mix_examples():
    """reuse 0 -> fresh only; 0.25 x 8 with 10 valid -> 2 + 6; all expired -> fresh only."""
    fresh = [make_group((100 + i, [3, 3], ["pass", "fail"])) for i in range(8)]
    buf = P.ReplayBuffer(10, 0.0)
    for i in range(10):
        buf.insert(make_group((200 + i, [3, 3], ["pass", "fail"])))
    assert sorted(ids(P.buffer_mix(buf, fresh, 8, 3, P.StalenessPolicy(2), C.Rng(0)))) == list(range(100, 108))
    buf = P.ReplayBuffer(10, 0.25)
    for i in range(10):
        buf.insert(make_group((200 + i, [3, 3], ["pass", "fail"])))
    out = ids(P.buffer_mix(buf, fresh, 8, 3, P.StalenessPolicy(2), C.Rng(0)))
    assert sum(i >= 200 for i in out) == 2 and sum(i < 200 for i in out) == 6 and len(buf.entries) == 10  # 8 left + 2 overflow fresh
    buf = P.ReplayBuffer(10, 0.5)
    for i in range(4):
        buf.insert(make_group((200 + i, [0, 0], ["pass", "fail"])))
    out = ids(P.buffer_mix(buf, fresh, 8, 5, P.StalenessPolicy(2), C.Rng(0)))
    assert sorted(out) == list(range(100, 108)) and buf.entries == []


def test_pack_batch_host_layout():
    """pack_batch on the CPU: every sample packed in batch order, `use` = apply_masks' USE, one row per token."""
    import torch
    from paper_2509_18883_b200.objective import Mask
    groups = []
    for pid, kinds in enumerate((["pass", "fail", "grade_error"], ["fail", "fail", "pass"])):
        samples = []
        for i, k in enumerate(kinds):
            toks = tuple(range(i + 2))
            samples.append(C.Sample(prompt_id=pid, context_id=0, version_id=0, tokens=toks,
                                    infer_logps=tuple(-1.0 for _ in toks), status=C.SampleStatus.COMPLETE, t_start=0,
                                    train_logps=tuple(-1.5 for _ in toks) + (9.0,), reward=KINDS[k](),
                                    gen_temperature=0.5 + i))
        groups.append(C.Group(pid, tuple(samples)))
    masked, b = P.pack_batch(groups, 6, device=torch.device("cpu"))
    assert b.n_groups == 2 and b.group_size == 3 and b.n_samples == 6
    assert list(b.sample_rows_host) == [0, 2, 5, 9, 11, 14, 18]
    assert b.use.tolist() == [int(m is Mask.USE) for mg in masked.groups for m in mg.masks] == [1, 1, 0, 1, 1, 1]
    assert b.adv.tolist() == [a for mg in masked.groups for a in mg.advantages]
    assert b.temperature.tolist() == [0.5, 1.5, 2.5] * 2
    assert b.logp_train.tolist()[:2] == [-1.5, -1.5] and b.logp_train.tolist()[5:9] == [0.0] * 4  # masked: zeros
    assert b.row_index is None and b.n_rows == 18
