"""Pin the CPU oracle (oracle/) to golden vectors produced by the unmodified reference."""
import json

import numpy as np
import pytest

from oracle import fusion as OF
from oracle import objective as OO
from oracle import rng as OR

FUSION_CFGS = {
    "default": dict(),
    "p05_s42": dict(dropout_p=0.5, seed=42),
    "p05_s42_sq": dict(dropout_p=0.5, seed=42, erase_weighting="squared"),
    "p03_s7_t1_w": dict(dropout_p=0.3, seed=7, target_norm=1.0, merge_weights=(0.5, 0.3, 0.2)),
    "none_noerase": dict(target_norm=None, erase_mode=False),
    "p09_s3_none": dict(dropout_p=0.9, seed=3, target_norm=None),
}


def test_label_hash(golden_rng):
    for lab, h in golden_rng["label_hash"].items():
        assert hex(OR.label_hash(eval(lab))) == h
    # SURVEY Appendix A pins
    assert OR.label_hash("fusion-dropout") == 0xBE1693CB125BD7AD


def test_streams_and_keeps(golden_rng):
    for st in golden_rng["streams"]:
        child = OR.fusion_child_seed(st["seed"], st["i"])
        assert hex(child) == st["child"]
        assert hex(OR.split(st["seed"], "fusion-dropout")) == st["parent"]
        d = OR.draws(child, 0, 256)
        assert [hex(int(x)) for x in d] == st["draws"]
        for p, bits in st["keep"].items():
            k = OR.keep_mask(child, 0, 1024, float(p))
            assert "".join("1" if b else "0" for b in k) == bits


def test_appendix_a_far_draw():
    # draw[2^32 + 5] of child (seed 0, i 0) from SURVEY Appendix A
    child = OR.fusion_child_seed(0, 0)
    assert child == 0xAB5C8D087CC10FEC
    assert int(OR.draws(child, 2 ** 32 + 5, 1)[0]) == 0x4AF712A1124C0995


@pytest.mark.parametrize("dname", ["kat", "bf16"])
@pytest.mark.parametrize("cname", list(FUSION_CFGS))
def test_fuse_oracle_matches_reference(golden_fusion, dname, cname):
    key = f"{dname}/{cname}"
    if key + "/fused" not in golden_fusion:
        pytest.skip("case not generated")
    base = golden_fusion[f"{dname}/base"]
    experts = [golden_fusion[f"{dname}/expert{k}"] for k in range(3)]
    fused, st = OF.fuse(base, experts, **FUSION_CFGS[cname])
    np.testing.assert_array_equal(fused, golden_fusion[key + "/fused"])
    np.testing.assert_array_equal(st["norms_before"], golden_fusion[key + "/norms_before"])
    np.testing.assert_allclose(st["norms_after"], golden_fusion[key + "/norms_after"], rtol=1e-15)
    np.testing.assert_array_equal(st["kept"], golden_fusion[key + "/kept"])
    np.testing.assert_array_equal(st["erased"], golden_fusion[key + "/erased"])


def test_appendix_a_stats(golden_fusion):
    # erased counts of the default and p=0.5/seed 42 KATs
    assert list(golden_fusion["kat/default/erased"]) == [1051, 1367, 1069]
    assert list(golden_fusion["kat/p05_s42/erased"]) == [377, 414, 412]
    assert list(golden_fusion["kat/p05_s42_sq/erased"]) == [389, 432, 434]


def test_staged_oracle(golden_fusion):
    base = golden_fusion["kat/base"]
    deltas = [golden_fusion[f"kat/expert{k}"] - base for k in range(3)]
    norms = [OF.norm(d) for d in deltas]
    nd, _, _ = OF.normalize(deltas, norms, "mean_of_inputs")
    for k in range(3):
        np.testing.assert_array_equal(nd[k], golden_fusion[f"stage/normalized{k}"])
    child = OR.split(11, "stage")
    np.testing.assert_array_equal(OF.dropout(deltas[0], 0.4, child), golden_fusion["stage/dropout0"])
    for w in ("sum", "squared"):
        er = OF.erase(deltas, w)
        for k in range(3):
            np.testing.assert_array_equal(er[k], golden_fusion[f"stage/erase_{w}{k}"])
    e3 = OF.erase([np.array([0.3]), np.array([0.1]), np.array([-0.2])])
    assert [float(x[0]) for x in e3] == [0.3, 0.1, 0.0]


def _flatten_objective(g, cname):
    meta = json.loads(str(g[f"{cname}/meta"]))
    logits = g[f"{cname}/logits"]
    C, T, V = logits.shape
    toks, lt, li, rows, sor, adv, use, temps, group_rows = [], [], [], [], [], [], [], [], [0]
    G = meta["G"]
    for si, s in enumerate(meta["samples"]):
        adv.append(s["adv"])
        use.append(s["mask"] == "use")
        temps.append(s["tau"])
        for t, tok in enumerate(s["tokens"]):
            toks.append(tok)
            lt.append(s["lt"][t])
            li.append(s["li"][t])
            rows.append(s["ctx"] * T + t)
            sor.append(si)
        if (si + 1) % G == 0:
            group_rows.append(len(toks))
    return meta, logits, dict(tokens=toks, lt=lt, li=li, rows=rows, sor=sor, adv=adv, use=use, temps=temps,
                              group_rows=group_rows)


@pytest.mark.parametrize("cname", ["small", "mid", "mid_literal"])
def test_objective_oracle(golden_objective, cname):
    meta, logits, b = _flatten_objective(golden_objective, cname)
    C, T, V = logits.shape
    l2 = logits.reshape(-1, V)
    clip = dict(eps_neg_low=0.2, eps_pos_high=0.2, eps_neg_high=3.0, tis_cap=2.0, guard_positive=meta["guard"])
    norm = 1.0 / (meta["n_groups"] * meta["G"] * meta["t_max"])
    logp, term, coef = OO.token_terms(l2, b["rows"], b["tokens"], b["lt"], b["li"], b["sor"], b["adv"], b["use"],
                                      b["temps"], clip, norm=norm)
    J = OO.objective(term, b["group_rows"], meta["G"], meta["t_max"])
    ref = float(golden_objective[f"{cname}/value"][0])
    assert J == pytest.approx(ref, rel=1e-12, abs=1e-15)
    temps_tok = [b["temps"][s] for s in b["sor"]]
    grad = OO.gradient_rows(l2, b["rows"], b["tokens"], coef, temps_tok, l2.shape)
    np.testing.assert_allclose(grad.reshape(C, T, V), golden_objective[f"{cname}/grad"], rtol=1e-10, atol=1e-15)
