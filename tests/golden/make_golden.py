"""Generate golden vectors from the UNMODIFIED reference (run in the build container only).

    OPENBLAS_NUM_THREADS=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/rng.json, fusion_kat.npz, objective_kat.npz.  The reference tree is not needed
at test time; these fixtures pin oracle/ (tests/test_oracle_golden.py) and the GPU parity tests.
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from rolloutlab import core, fusion, objective, toy_env  # noqa: E402

OUT = Path(__file__).resolve().parent


def rng_vectors():
    out = {"label_hash": {}, "streams": []}
    for lab in ["fusion-dropout", "perturb", "payloads", 0, 1, 2, 7]:
        out["label_hash"][repr(lab)] = hex(core._label_hash(lab))
    for seed in [0, 7, 42, 123456789, 2 ** 64 - 1]:
        parent = core.make_rng(seed, "fusion-dropout")
        for i in range(4):
            child = parent.split(i)
            r = core.Rng(child.seed)
            draws = [r.next_u64() for _ in range(256)]
            keeps = {}
            for p in [0.3, 0.5, 0.9]:
                rr = core.Rng(child.seed)
                keeps[str(p)] = "".join("1" if rr.uniform() >= p else "0" for _ in range(1024))
            out["streams"].append({"seed": seed, "parent": hex(parent.seed), "i": i, "child": hex(child.seed),
                                   "draws": [hex(d) for d in draws], "keep": keeps})
    (OUT / "rng.json").write_text(json.dumps(out, indent=1))


def PT(a):
    return toy_env.ParamTable(np.asarray(a, dtype=np.float64).reshape(1, 1, -1))


def bf16_round(x):
    """Round float64 values to bf16-representable values (RNE), returned as float64."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def fusion_cases():
    cases = {}
    n = 4096
    i = np.arange(n)
    base = 0.5 * np.sin(i)
    experts = [base + 0.01 * (k + 1) * np.cos(i * (k + 1) + k) for k in range(3)]
    cfgs = {
        "default": fusion.FusionConfig(),
        "p05_s42": fusion.FusionConfig(dropout_p=0.5, seed=42),
        "p05_s42_sq": fusion.FusionConfig(dropout_p=0.5, seed=42, erase_weighting="squared"),
        "p03_s7_t1_w": fusion.FusionConfig(dropout_p=0.3, seed=7, target_norm=1.0, merge_weights=(0.5, 0.3, 0.2)),
        "none_noerase": fusion.FusionConfig(target_norm=None, erase_mode=False),
        "p09_s3_none": fusion.FusionConfig(dropout_p=0.9, seed=3, target_norm=None),
    }
    # bf16-representable case: 70001 elements (crosses a 65536 item boundary, odd tail)
    g = np.random.default_rng([0, 1])
    m = 70001
    bb = bf16_round(g.normal(0, 0.02, m))
    eb = [bf16_round(bb + g.normal(0, (k + 1) * 1e-3, m)) for k in range(3)]
    eb[0][:50] = bb[:50]  # some exact-zero deltas
    data = {"kat": (base, experts), "bf16": (bb, eb)}
    for dname, (b, es) in data.items():
        cases[f"{dname}/base"] = b
        for k, e in enumerate(es):
            cases[f"{dname}/expert{k}"] = e
        for cname, cfg in cfgs.items():
            taus = [fusion.task_vector(PT(e), PT(b)) for e in es]
            fused, st = fusion.fuse(PT(b), taus, cfg)
            key = f"{dname}/{cname}"
            cases[key + "/fused"] = fused.logits.ravel()
            cases[key + "/norms_before"] = np.array(st.norms_before)
            cases[key + "/norms_after"] = np.array(st.norms_after_normalize)
            cases[key + "/kept"] = np.array(st.dropout_kept_fraction)
            cases[key + "/erased"] = np.array(st.erased_counts)
            cases[key + "/weights"] = np.array(st.weights)
    # staged functions on the KAT inputs
    taus = [fusion.task_vector(PT(e), PT(base)) for e in experts]
    nm = fusion.normalize_magnitudes(taus, fusion.FusionConfig())
    for k, t in enumerate(nm):
        cases[f"stage/normalized{k}"] = t.delta.ravel()
    r = core.make_rng(11, "stage")
    dp = fusion.dropout_prune(taus[0], 0.4, r)
    cases["stage/dropout0"] = dp.delta.ravel()
    cases["stage/dropout_rng_after"] = np.array([r.next_u64()], dtype=np.uint64)
    for w in ("sum", "squared"):
        er = fusion.erase_minority(taus, w)
        for k, t in enumerate(er):
            cases[f"stage/erase_{w}{k}"] = t.delta.ravel()
    # SPEC worked examples
    e3 = fusion.erase_minority([fusion.TaskVector(np.array([[[v]]])) for v in (0.3, 0.1, -0.2)])
    cases["spec/erase3"] = np.array([t.delta.item() for t in e3])
    np.savez_compressed(OUT / "fusion_kat.npz", **cases)


def objective_cases():
    out = {}
    g = np.random.default_rng(5)
    for cname, (C, T, V, G, ngroups, tau, guard) in {
        "small": (2, 5, 7, 4, 2, 0.7, True),
        "mid": (3, 8, 257, 4, 3, 1.0, True),
        "mid_literal": (3, 8, 257, 4, 3, 0.9, False),
    }.items():
        logits = g.normal(0, 2.0, (C, T, V))
        params = toy_env.ParamTable(logits)
        groups = []
        for gi in range(ngroups):
            ctx = gi % C
            samples = []
            for si in range(G):
                L = int(g.integers(1, T + 1))
                toks = tuple(int(x) for x in g.integers(0, V, L))
                lt = tuple(float(toy_env.log_token_dist(params, toy_env.TrainEngine(), ctx, t, tau)[tok]
                                 + g.normal(0, 0.3)) for t, tok in enumerate(toks))
                li = tuple(float(x + g.normal(0, 0.05)) for x in lt)
                st = core.SampleStatus.COMPLETE
                rw = core.RewardOutcome.passed() if g.random() < 0.5 else core.RewardOutcome.failed()
                if si == 1 and gi == 0:
                    rw = core.RewardOutcome.grade_error()
                s = core.Sample(prompt_id=gi, context_id=ctx, version_id=0, tokens=toks, infer_logps=li,
                                status=st, t_start=0, train_logps=lt, reward=rw, gen_temperature=tau)
                samples.append(s)
            groups.append(core.Group(gi, tuple(samples)))
        batch = objective.apply_masks(groups, T)
        clip = objective.ClipConfig(guard_positive=guard)
        out[f"{cname}/logits"] = logits
        out[f"{cname}/value"] = np.array([objective.objective_value(batch, params, clip)])
        out[f"{cname}/grad"] = objective.objective_gradient(batch, params, clip)
        # flatten the batch for the tests
        meta = []
        for mg in batch.groups:
            for s, a, mk in zip(mg.group.samples, mg.advantages, mg.masks):
                meta.append(dict(ctx=s.context_id, tokens=list(s.tokens), lt=list(s.train_logps),
                                 li=list(s.infer_logps), adv=a, mask=mk.value, tau=s.gen_temperature,
                                 reward=None if s.reward.raw_score is None else s.reward.raw_score,
                                 kind=s.reward.kind.value))
        out[f"{cname}/meta"] = np.array(json.dumps(dict(samples=meta, G=G, n_groups=ngroups, t_max=T,
                                                        guard=guard)))
    np.savez_compressed(OUT / "objective_kat.npz", **out)


if __name__ == "__main__":
    rng_vectors()
    fusion_cases()
    objective_cases()
    print("golden vectors written to", OUT)
