"""Golden vectors for the sample-intake pipeline, from the UNMODIFIED reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_pipeline.py

Writes tests/golden/pipeline_kat.json: seeded completion streams (each group as prompt id, sample
versions and reward kinds) driven through the reference's BatchAssembler / buffer_mix /
assemble_batch, with every decision, emitted batch (prompt ids in shuffled order), stale drop,
reuse count and buffer state recorded, plus the SPEC examples and error messages
(rolloutlab/pipeline.py:1-248).  tests/test_pipeline_cpu.py replays the same
drivers through paper_2509_18883_b200.pipeline and compares.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from rolloutlab import core, pipeline  # noqa: E402

OUT = Path(__file__).resolve().parent
KINDS = {"pass": core.RewardOutcome.passed, "fail": core.RewardOutcome.failed,
         "grade_error": core.RewardOutcome.grade_error, "none": lambda: None}


def make_group(spec):
    pid, versions, kinds = spec
    samples = tuple(core.Sample(prompt_id=pid, context_id=0, version_id=v, tokens=(1, 2), infer_logps=(-1.0, -1.0),
                                status=core.SampleStatus.COMPLETE, t_start=0, reward=KINDS[k]())
                    for v, k in zip(versions, kinds))
    return core.Group(pid, samples)


def ids(groups):
    return None if groups is None else [g.prompt_id for g in groups]


def random_stream(g, n, G, max_lag):
    """n group specs; kinds drawn so that all four filter outcomes occur; versions filled in by the driver
    as (current version at arrival) - lag."""
    out = []
    for pid in range(n):
        u = g.random()
        if u < 0.12:
            kinds = ["pass"] * G
        elif u < 0.24:
            kinds = ["fail"] * G
        elif u < 0.30:
            kinds = ["grade_error"] * G
        else:
            kinds = [str(x) for x in g.choice(["pass", "fail", "grade_error"], size=G, p=[0.45, 0.45, 0.10])]
        lags = [int(x) for x in g.integers(0, max_lag + 1, size=G)]
        out.append({"pid": 1000 + pid, "kinds": kinds, "lags": lags})
    return out


def drive_assembler(sc):
    """Offer the stream; the policy version advances by one after every emitted batch (a training step).
    Oversampled groups (`side`) go straight into the buffer every `side_every` offers, the way a rollout
    manager stores extra kept groups; the assembler itself only feeds the buffer its overflow."""
    buf = None if sc["capacity"] is None else pipeline.ReplayBuffer(sc["capacity"], sc["reuse_ratio"])
    asm = pipeline.BatchAssembler(sc["batch_groups"], pipeline.StalenessPolicy(sc["max_staleness"]), buf,
                                  core.Rng(sc["seed"]))
    version = sc["start_version"]
    trace = []
    side = iter(sc["side"])
    for i, item in enumerate(sc["stream"]):
        if buf is not None and sc["side_every"] and i % sc["side_every"] == 0:
            extra = next(side)
            buf.insert(make_group((extra["pid"], [max(0, version - lag) for lag in extra["lags"]], extra["kinds"])))
        versions = [max(0, version - lag) for lag in item["lags"]]
        res = asm.offer(make_group((item["pid"], versions, item["kinds"])), version)
        trace.append({"version": version, "decision": res.decision.value, "batch": ids(res.batch),
                      "dropped": ids(res.dropped_stale), "reused": res.reused_count,
                      "pending": ids(asm.pending), "buffer": None if buf is None else ids(buf.entries)})
        if res.batch is not None:
            version += 1
    return trace, asm.rng.next_u64()


def assembler_scenarios():
    g = np.random.default_rng(2509)
    out = []
    for name, bg, cap, ratio, mst, lag, n, v0 in [
        ("no_buffer_b4", 4, None, 0.0, 2, 3, 60, 3),
        ("buffer_r025_b8", 8, 6, 0.25, 2, 3, 120, 4),
        ("buffer_r05_b4_cap3_strict", 4, 3, 0.5, 0, 1, 80, 2),
        ("buffer_r0_b3", 3, 5, 0.0, 1, 2, 50, 1),
        ("buffer_r09_b5_cap20", 5, 20, 0.9, 3, 4, 150, 5),
        ("no_buffer_b1", 1, None, 0.0, 2, 2, 30, 0),
        ("no_buffer_b3_strict", 3, None, 0.0, 0, 2, 60, 4),
        ("buffer_r04_b5_strict", 5, 4, 0.4, 0, 2, 90, 6),
    ]:
        sc = {"name": name, "batch_groups": bg, "capacity": cap, "reuse_ratio": ratio, "max_staleness": mst,
              "seed": int(g.integers(0, 2 ** 63)), "start_version": v0,
              "stream": random_stream(g, n, G := int(g.integers(2, 6)), lag), "side_every": 0 if cap is None else 3}
        sc["side"] = [dict(x, pid=x["pid"] + 5000, kinds=["pass", "fail"] + x["kinds"][2:])
                      for x in random_stream(g, n // 3 + 1, G, lag + 1)]
        sc["trace"], sc["rng_after"] = drive_assembler(sc)
        sc["rng_after"] = hex(sc["rng_after"])
        out.append(sc)
    return out


def mix_cases():
    """Direct buffer_mix calls: buffer contents, fresh list, batch size, version -> batch, buffer after."""
    g = np.random.default_rng(18883)
    out = []
    for k in range(40):
        G = 2
        cap = int(g.integers(1, 9))
        ratio = float(g.choice([0.0, 0.1, 0.25, 0.5, 0.75, 0.99]))
        version = int(g.integers(0, 6))
        mst = int(g.integers(0, 3))
        n_buf = int(g.integers(0, 12))
        n_fresh = int(g.integers(0, 10))
        bg = int(g.integers(1, 9))
        buf_specs = [[2000 + 100 * k + i, [max(0, version - int(g.integers(0, 4)))] * G, ["pass", "fail"]]
                     for i in range(n_buf)]
        fresh_specs = [[3000 + 100 * k + i, [version] * G, ["fail", "pass"]] for i in range(n_fresh)]
        buf = pipeline.ReplayBuffer(cap, ratio)
        for s in buf_specs:
            buf.insert(make_group(s))
        seed = int(g.integers(0, 2 ** 63))
        rng = core.Rng(seed)
        before = ids(buf.entries)
        valid = buf.valid_count(version, pipeline.StalenessPolicy(mst))
        fresh = [make_group(s) for s in fresh_specs]
        batch = pipeline.buffer_mix(buf, fresh, bg, version, pipeline.StalenessPolicy(mst), rng)
        out.append({"capacity": cap, "reuse_ratio": ratio, "version": version, "max_staleness": mst,
                    "batch_groups": bg, "seed": seed, "buffer_specs": buf_specs, "fresh_specs": fresh_specs,
                    "buffer_before": before, "valid_before": valid, "batch": ids(batch),
                    "buffer_after": ids(buf.entries), "fresh_after": ids(fresh), "rng_after": hex(rng.next_u64())})
    return out


def generator_cases():
    """assemble_batch over a finite stream (one version, a buffer)."""
    g = np.random.default_rng(7)
    stream = random_stream(g, 70, 4, 2)
    version = 3
    groups = [make_group((s["pid"], [max(0, version - l) for l in s["lags"]], s["kinds"])) for s in stream]
    buf = pipeline.ReplayBuffer(4, 0.3)
    batches = [ids(b) for b in pipeline.assemble_batch(iter(groups), 5, pipeline.StalenessPolicy(1), version, buf,
                                                        core.Rng(99))]
    return {"stream": stream, "version": version, "batch_groups": 5, "capacity": 4, "reuse_ratio": 0.3,
            "max_staleness": 1, "seed": 99, "batches": batches, "buffer_after": ids(buf.entries)}


def catch(fn):
    try:
        r = fn()
    except Exception as e:  # noqa: BLE001 - record the reference's exception type and message
        return [type(e).__name__, str(e)]
    return ["ok", r.value if hasattr(r, "value") else repr(r)]


def spec_and_errors():
    P = pipeline
    cases = {
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
        "mix_batch0": lambda: P.buffer_mix(P.ReplayBuffer(2, 0.5), [], 0, 0, P.StalenessPolicy(2), core.Rng(1)),
        "assembler_batch0": lambda: P.BatchAssembler(0, P.StalenessPolicy(2)),
        "assembler_ungraded": lambda: P.BatchAssembler(2, P.StalenessPolicy(2)).offer(
            make_group((5, [0, 0], ["none", "pass"])), 0),
        "assembler_future": lambda: P.BatchAssembler(2, P.StalenessPolicy(2)).offer(
            make_group((5, [4, 0], ["fail", "pass"])), 1),
    }
    return {k: catch(f) for k, f in cases.items()}


if __name__ == "__main__":
    data = {"assembler": assembler_scenarios(), "mix": mix_cases(), "generator": generator_cases(),
            "spec": spec_and_errors()}
    (OUT / "pipeline_kat.json").write_text(json.dumps(data, separators=(",", ":")))
    n = sum(len(s["trace"]) for s in data["assembler"])
    print(f"pipeline_kat.json: {len(data['assembler'])} assembler streams ({n} offers), {len(data['mix'])} mixes, "
          f"{len(data['generator']['batches'])} generator batches, {len(data['spec'])} spec/error cases")
