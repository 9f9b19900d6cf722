"""Property tests transcribed from the reference SPEC's "Invariants & Properties" (SPEC.md:576-580
fusion, :287-294 objective), run through the CUDA path with hypothesis-generated inputs
(test plan item 3)."""
import math

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu

SETTINGS = dict(max_examples=25, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])


def _pt(x, dev, dtype=torch.float64):
    from paper_2509_18883_b200.toy_env import ParamTable
    return ParamTable(torch.from_numpy(np.asarray(x, dtype=np.float64).reshape(1, 1, -1)).to(dev, dtype))


vec = st.integers(min_value=1, max_value=3000).flatmap(
    lambda n: st.tuples(st.just(n), st.integers(min_value=0, max_value=2**31 - 1)))


@settings(**SETTINGS)
@given(vec, st.integers(min_value=2, max_value=5), st.sampled_from(["sum", "squared"]))
def test_erase_never_flips_or_grows(cuda, nv, n_exp, weighting):
    """erase_minority never changes the sign of a surviving element and never increases |element|."""
    from paper_2509_18883_b200 import fusion as F
    n, seed = nv
    g = np.random.default_rng(seed)
    base = _pt(np.zeros(n), cuda)
    taus = [F.task_vector(_pt(g.normal(0, 1, n) * (g.random(n) < 0.8), cuda), base) for _ in range(n_exp)]
    out = F.erase_minority(taus, weighting)
    for t, o in zip(taus, out):
        a, b = t.delta.reshape(-1).cpu().numpy(), o.delta.reshape(-1).cpu().numpy()
        kept = b != 0
        assert np.all(np.sign(b[kept]) == np.sign(a[kept]))
        assert np.all(np.abs(b) <= np.abs(a))
        assert np.all((b == a) | (b == 0))


@settings(**SETTINGS)
@given(vec, st.floats(min_value=0.05, max_value=0.9), st.integers(min_value=0, max_value=2**40))
def test_dropout_survivors_rescaled_exactly(cuda, nv, p, cfg_seed):
    """dropout_prune: every entry is either 0 or value / (1 - p), bit-exactly as in f64."""
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.core import make_rng
    n, seed = nv
    x = np.random.default_rng(seed).normal(0, 1, n)
    tv = F.task_vector(_pt(x, cuda), _pt(np.zeros(n), cuda))
    d = F.dropout_prune(tv, p, make_rng(cfg_seed, "fusion-dropout").split(0)).delta.reshape(-1).cpu().numpy()
    assert np.all((d == 0) | (d == x / (1.0 - p)))


def test_dropout_unbiased(cuda):
    """dropout_prune is unbiased per element: the mean over many seeds approaches the input."""
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.core import make_rng
    n, p, trials = 512, 0.4, 600
    x = np.random.default_rng(1).normal(0, 1, n)
    tv = F.task_vector(_pt(x, cuda), _pt(np.zeros(n), cuda))
    acc = torch.zeros(n, dtype=torch.float64, device=cuda)
    for s in range(trials):
        acc += F.dropout_prune(tv, p, make_rng(s, "fusion-dropout").split(0)).delta.reshape(-1)
    mean = (acc / trials).cpu().numpy()
    # per-element std of the estimator: |x| sqrt(p / (1 - p)) / sqrt(trials); 5 sigma
    tol = 5 * np.abs(x) * math.sqrt(p / (1 - p)) / math.sqrt(trials) + 1e-12
    assert np.all(np.abs(mean - x) <= tol)


@settings(**SETTINGS)
@given(vec, st.sampled_from([torch.bfloat16, torch.float32, torch.float64]), st.floats(min_value=0.0, max_value=0.8))
def test_fuse_deterministic(cuda, nv, dtype, p):
    """Identical (inputs, cfg, seed) give an identical fused table and stats."""
    from paper_2509_18883_b200 import fusion as F
    n, seed = nv
    g = np.random.default_rng(seed)
    b = _pt(g.normal(0, 0.02, n), cuda, dtype)
    es = [_pt(b.logits.double().cpu().numpy().reshape(-1) + g.normal(0, 1e-3 * (i + 1), n), cuda, dtype)
          for i in range(3)]
    cfg = F.FusionConfig(dropout_p=p, seed=seed)
    r1 = F.fuse(b, [F.task_vector(e, b) for e in es], cfg)
    r2 = F.fuse(b, [F.task_vector(e, b) for e in es], cfg)
    assert torch.equal(r1[0].logits, r2[0].logits)
    assert r1[1] == r2[1]


@settings(**SETTINGS)
@given(vec)
def test_identical_experts_convexity(cuda, nv):
    """Two identical experts, w = (0.5, 0.5), no pruning -> that expert."""
    from paper_2509_18883_b200 import fusion as F
    n, seed = nv
    g = np.random.default_rng(seed)
    b = _pt(g.normal(0, 1, n), cuda)
    e = _pt(b.logits.cpu().numpy().reshape(-1) + g.normal(0, 0.1, n), cuda)
    cfg = F.FusionConfig(target_norm=None, merge_weights=(0.5, 0.5))
    fused, _ = F.fuse(b, [F.task_vector(e, b), F.task_vector(e, b)], cfg)
    np.testing.assert_allclose(fused.logits.cpu().numpy(), e.logits.cpu().numpy(), rtol=0, atol=1e-15)


r_st = st.floats(min_value=1e-3, max_value=20.0)
adv_st = st.floats(min_value=-5.0, max_value=5.0).filter(lambda a: abs(a) > 1e-6)


@settings(max_examples=300, deadline=None)
@given(r_st, adv_st)
def test_triplet_bounds(r, adv):
    """adv < 0: term >= eps_neg_high * adv for all r > 0; adv > 0: term <= (1 + eps_pos_high) * adv."""
    from paper_2509_18883_b200.objective import ClipConfig, triplet_clip_term
    c = ClipConfig()
    v = triplet_clip_term(r, adv, c)
    if adv < 0:
        assert v >= c.eps_neg_high * adv - 1e-12
    else:
        assert v <= (1 + c.eps_pos_high) * adv + 1e-12


@settings(max_examples=300, deadline=None)
@given(st.floats(min_value=-30, max_value=0), st.floats(min_value=-30, max_value=0),
       st.floats(min_value=1.0, max_value=10.0))
def test_tis_weight_capped(lt, li, cap):
    """tis_weight <= C always; 1 when the engines coincide."""
    from paper_2509_18883_b200.objective import tis_weight
    assert tis_weight(lt, li, cap) <= cap
    assert tis_weight(lt, lt, cap) == 1.0


def test_grpo_terms_respect_bounds_on_device(cuda):
    """The device token terms obey the same triplet bounds (randomized off-policy batch)."""
    from paper_2509_18883_b200 import objective as O
    V, R = 4096, 2048
    g = np.random.default_rng(3)
    logits = torch.from_numpy(g.normal(0, 2.0, (R, V))).to(cuda, torch.float32)
    lt = g.normal(-8, 2.0, R)
    adv = np.array([1.3, -0.7, 2.0, -1.5])
    b = O.GRPOBatch.pack(g.integers(0, V, R), lt, lt + g.normal(0, 0.1, R), np.arange(5) * (R // 4), adv,
                         [1, 1, 1, 1], 2, R // 4, device=cuda)
    fwd = O.grpo_forward(logits, b)
    c = O.ClipConfig()
    term = fwd.term.cpu().numpy()
    a_row = np.repeat(adv, R // 4)
    neg = a_row < 0
    # term = w * value, 0 <= w <= C; value >= eps_nh * adv for adv < 0, value <= (1 + eps_h) * adv for adv > 0
    assert np.all(term[neg] >= c.tis_cap * c.eps_neg_high * a_row[neg] - 1e-9)
    assert np.all(term[~neg] <= c.tis_cap * (1 + c.eps_pos_high) * a_row[~neg] + 1e-9)


def test_denominator_is_constant(cuda):
    """Length-bias control: J = sum of terms / (G * T_max) with T_max fixed, whatever the lengths."""
    from paper_2509_18883_b200 import objective as O
    V = 512
    g = np.random.default_rng(4)
    lens = [5, 9, 2, 7]
    R = sum(lens)
    logits = torch.from_numpy(g.normal(0, 1.0, (R, V))).to(cuda, torch.float64)
    lt = g.normal(-6, 0.5, R)
    cu = np.concatenate([[0], np.cumsum(lens)])
    adv = np.array([1.0, -1.0, 0.5, -0.5])
    for t_max in (9, 32):
        b = O.GRPOBatch.pack(g.integers(0, V, R), lt, lt, cu, adv, [1, 1, 1, 1], 4, t_max, device=cuda)
        fwd = O.grpo_forward(logits, b)
        assert float(fwd.objective) == pytest.approx(float(fwd.term.sum()) / (4 * t_max), rel=1e-12, abs=1e-15)
