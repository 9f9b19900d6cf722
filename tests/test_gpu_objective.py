"""GPU parity: the GRPO kernels (K4/K5) vs the reference's golden vectors and the CPU oracle."""
import json
import math

import numpy as np
import pytest
import torch

from oracle import objective as OO
from tests.helpers import assert_grad_rows, bf16_round

pytestmark = pytest.mark.gpu


def _rebuild_batch(g, cname):
    from paper_2509_18883_b200 import core, objective as O
    meta = json.loads(str(g[f"{cname}/meta"]))
    G = meta["G"]
    groups = []
    for gi in range(meta["n_groups"]):
        samples = []
        for s in meta["samples"][gi * G:(gi + 1) * G]:
            rw = core.RewardOutcome(core.RewardKind(s["kind"]), s["reward"])
            samples.append(core.Sample(prompt_id=gi, context_id=s["ctx"], version_id=0, tokens=tuple(s["tokens"]),
                                       infer_logps=tuple(s["li"]), status=core.SampleStatus.COMPLETE, t_start=0,
                                       train_logps=tuple(s["lt"]), reward=rw, gen_temperature=s["tau"]))
        groups.append(core.Group(gi, tuple(samples)))
    batch = O.apply_masks(groups, meta["t_max"])
    for mg, gi in zip(batch.groups, range(meta["n_groups"])):
        for a, m, s in zip(mg.advantages, mg.masks, meta["samples"][gi * G:(gi + 1) * G]):
            assert a == s["adv"] and m.value == s["mask"]
    return batch, O.ClipConfig(guard_positive=meta["guard"])


@pytest.mark.parametrize("cname", ["small", "mid", "mid_literal"])
def test_objective_kat(cuda, golden_objective, cname):
    from paper_2509_18883_b200 import objective as O
    from paper_2509_18883_b200.toy_env import ParamTable
    batch, clip = _rebuild_batch(golden_objective, cname)
    params = ParamTable(golden_objective[f"{cname}/logits"])
    J = O.objective_value(batch, params, clip)
    assert J == pytest.approx(float(golden_objective[f"{cname}/value"][0]), rel=1e-12, abs=1e-16)
    grad = O.objective_gradient(batch, params, clip).cpu().numpy()
    np.testing.assert_allclose(grad, golden_objective[f"{cname}/grad"], rtol=1e-10, atol=1e-16)
    # ascent_step
    p2 = O.ascent_step(params, grad, 0.5)
    np.testing.assert_array_equal(p2.numpy(), params.numpy() + 0.5 * grad)


def _synthetic_rows(R_per_sample, S, V, G, seed=0, tau=1.0, masked=()):
    """SURVEY 8(d) config-5 style rows: logits N(0, 2^2) + a peaked column, tokens ~ softmax."""
    g = np.random.default_rng(seed)
    R = R_per_sample * S
    logits = g.normal(0, 2.0, (R, V)).astype(np.float32)
    peak = g.integers(0, V, R)
    logits[np.arange(R), peak] += 8.0
    logits = bf16_round(logits)
    toks = np.empty(R, dtype=np.int64)
    lt = np.empty(R)
    for r in range(R):
        lp = OO.log_token_dist(logits[r], tau)
        p = np.exp(lp)
        toks[r] = g.choice(V, p=p / p.sum())
        lt[r] = lp[toks[r]] + g.normal(0, 0.3)
    li = lt + g.normal(0, 0.05, R)
    rewards = g.integers(0, 2, S).astype(float)
    adv = np.zeros(S)
    for k in range(S // G):
        r = rewards[k * G:(k + 1) * G]
        adv[k * G:(k + 1) * G] = (r - r.mean()) / max(r.std(), 1e-8)
    use = np.ones(S, dtype=np.uint8)
    for m in masked:
        use[m] = 0
    cu = np.arange(S + 1) * R_per_sample
    return logits, toks, lt, li, adv, use, cu


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("tau", [1.0, 0.7])
def test_tensor_api_vs_oracle(cuda, dtype, tau):
    from paper_2509_18883_b200 import objective as O
    V, G, S, Rps, T_max = 131072, 4, 8, 12, 16
    logits, toks, lt, li, adv, use, cu = _synthetic_rows(Rps, S, V, G, seed=1, tau=tau, masked=(3,))
    b = O.GRPOBatch.pack(toks, lt, li, cu, adv, use, G, T_max, temperature=tau, device=cuda)
    lg = torch.from_numpy(logits).to(cuda, dtype)
    fwd = O.grpo_forward(lg, b)
    clip = dict(eps_neg_low=0.2, eps_pos_high=0.2, eps_neg_high=3.0, tis_cap=2.0, guard_positive=True)
    sor = np.repeat(np.arange(S), Rps)
    norm = 1.0 / ((S // G) * G * T_max)
    logp, term, coef = OO.token_terms(logits, None, toks, lt, li, sor, adv, use, [tau] * S, clip, norm=norm)
    J = OO.objective(term, list(cu[::G]), G, T_max)
    got_logp = fwd.logp.cpu().numpy()
    act = use[sor].astype(bool)
    np.testing.assert_allclose(got_logp[act], logp[act], rtol=0, atol=2e-5)
    np.testing.assert_allclose(fwd.term.cpu().numpy(), term, rtol=1e-4, atol=1e-6)
    assert float(fwd.objective) == pytest.approx(J, rel=1e-3)  # north-star tolerance
    assert int(fwd.flags.item()) == 0
    # masked sample rows contribute nothing and are not read
    assert np.all(fwd.coef.cpu().numpy()[~act] == 0)
    # the kernel's per-token coefficient vs the oracle's (objective.py:278): relative, except tokens whose
    # clip slope flips at a branch boundary between f32-row and f64 arithmetic (Appendix B of SURVEY)
    cg = fwd.coef.cpu().numpy()
    flip = (cg == 0) != (coef == 0)
    assert flip.sum() <= 1
    np.testing.assert_allclose(cg[~flip], coef[~flip], rtol=1e-5, atol=0)
    # backward, EVERY entry of every row vs coef * (onehot - softmax) in f64 (per-element relative bound):
    # f32 grad: ex2.approx + f32 argument rounding + the f32 row log-sum-exp -> rtol 5e-6 (measured <= 2.3e-6);
    # bf16 grad: plus one bf16 rounding (unit roundoff 2^-8)
    temps = [tau] * len(toks)
    for gdt, rtol in ((torch.float32, 5e-6), (torch.bfloat16, 2.0 ** -8 + 5e-6)):
        grad = O.grpo_backward(lg, b, fwd, grad_dtype=gdt).double().cpu().numpy()
        worst = assert_grad_rows(grad, logits, toks, cg, temps, rtol)
        print(f"grad {gdt} {dtype} tau={tau}: worst per-element error = {worst:.3f} of the bound")


def test_autograd_and_bf16_grad(cuda):
    from paper_2509_18883_b200 import objective as O
    V, G, S, Rps, T_max = 4096, 2, 4, 6, 8
    logits, toks, lt, li, adv, use, cu = _synthetic_rows(Rps, S, V, G, seed=2)
    b = O.GRPOBatch.pack(toks, lt, li, cu, adv, use, G, T_max, device=cuda)
    lg = torch.from_numpy(logits).to(cuda, torch.bfloat16).requires_grad_(True)
    J = O.grpo_token_objective(lg, b)
    (-2.0 * J).backward()
    fwd = O.grpo_forward(lg.detach(), b)
    ref = O.grpo_backward(lg.detach(), b, fwd, grad_dtype=torch.float32) * -2.0
    np.testing.assert_allclose(lg.grad.float().cpu().numpy(), ref.cpu().numpy(), rtol=1e-2, atol=1e-9)
    # fused mode: loss = -J with fused_scale = -1 returns the one-read gradient; a different grad_out
    # falls back to K5
    scale = float(np.abs(ref.cpu().numpy()).max())
    for mult, fused in ((-1.0, -1.0), (3.0, -1.0)):
        lg2 = torch.from_numpy(logits).to(cuda, torch.bfloat16).requires_grad_(True)
        (mult * O.grpo_token_objective(lg2, b, fused_scale=fused)).backward()
        ref2 = O.grpo_backward(lg.detach(), b, fwd, grad_dtype=torch.float32) * mult
        np.testing.assert_allclose(lg2.grad.float().cpu().numpy(), ref2.cpu().numpy(), rtol=0,
                                   atol=1e-2 * scale * abs(mult) / 2 + 1e-12)


def test_f64_finite_difference(cuda):
    """objective_gradient matches central finite differences of objective_value."""
    from paper_2509_18883_b200 import core, objective as O
    from paper_2509_18883_b200.toy_env import ParamTable
    g = np.random.default_rng(4)
    C, T, V, G = 1, 4, 6, 3
    logits = g.normal(0, 1.0, (C, T, V))
    samples = []
    for si in range(G):
        toks = tuple(int(x) for x in g.integers(0, V, T))
        lt = tuple(float(g.normal(-1.5, 0.3)) for _ in toks)
        li = tuple(x + float(g.normal(0, 0.05)) for x in lt)
        rw = core.RewardOutcome.passed() if si % 2 else core.RewardOutcome.failed()
        samples.append(core.Sample(0, 0, 0, toks, li, core.SampleStatus.COMPLETE, 0, train_logps=lt, reward=rw,
                                   gen_temperature=0.8))
    batch = O.apply_masks([core.Group(0, tuple(samples))], T)
    clip = O.ClipConfig()
    grad = O.objective_gradient(batch, ParamTable(logits), clip).cpu().numpy()
    h = 1e-6
    for idx in [(0, 0, 1), (0, 1, 3), (0, 3, 5), (0, 2, 0)]:
        lp, lm = logits.copy(), logits.copy()
        lp[idx] += h
        lm[idx] -= h
        fd = (O.objective_value(batch, ParamTable(lp), clip) - O.objective_value(batch, ParamTable(lm), clip)) / (2 * h)
        assert fd == pytest.approx(grad[idx], rel=1e-5, abs=1e-9)


def test_log_token_dist_and_trace(cuda):
    from paper_2509_18883_b200 import core
    from paper_2509_18883_b200.toy_env import ParamTable, TrainEngine, log_token_dist, logprob_trace
    g = np.random.default_rng(6)
    logits = g.normal(0, 1.5, (2, 3, 50))
    pt = ParamTable(logits)
    for tau in (1.0, 0.6):
        got = log_token_dist(pt, TrainEngine(), 1, 2, tau).cpu().numpy()
        np.testing.assert_allclose(got, OO.log_token_dist(logits[1, 2], tau), rtol=1e-13, atol=1e-14)
    s = core.Sample(0, 1, 0, (3, 7, 9), (0.0, 0.0, 0.0), core.SampleStatus.COMPLETE, 0, gen_temperature=0.9)
    tr = logprob_trace(pt, TrainEngine(), s)
    ref = [OO.log_token_dist(logits[1, t], 0.9)[tok] for t, tok in enumerate(s.tokens)]
    np.testing.assert_allclose(tr, ref, rtol=1e-13)
    with pytest.raises(IndexError):
        log_token_dist(pt, TrainEngine(), 2, 0)
    # the reference's per-call memo (objective.py:206-220): same rows, computed once per key
    from paper_2509_18883_b200 import objective as O
    cache = O._LogDistCache(pt)
    a = cache.get(1, 2, 0.6)
    assert cache.get(1, 2, 0.6) is a and len(cache._cache) == 1
    np.testing.assert_allclose(a.cpu().numpy(), OO.log_token_dist(logits[1, 2], 0.6), rtol=1e-13, atol=1e-14)


def test_bad_token_flag(cuda):
    from paper_2509_18883_b200 import objective as O
    V = 256
    b = O.GRPOBatch.pack([5, V + 3], [-1.0, -1.0], [-1.0, -1.0], [0, 1, 2], [1.0, -1.0], [1, 1], 2, 4, device=cuda)
    fwd = O.grpo_forward(torch.zeros((2, V), device=cuda, dtype=torch.bfloat16), b)
    assert int(fwd.flags.item()) & 2


@pytest.mark.parametrize("V", [131072, 4096])
def test_fused_forward_backward(cuda, V):
    """Single-pass cluster kernel == K4 + K5 (loss, per-token outputs, bf16 gradient)."""
    from paper_2509_18883_b200 import objective as O
    G, S, Rps, T_max = 4, 8, 9, 16
    logits, toks, lt, li, adv, use, cu = _synthetic_rows(Rps, S, V, G, seed=3, tau=0.8, masked=(2, 5))
    b = O.GRPOBatch.pack(toks, lt, li, cu, adv, use, G, T_max, temperature=0.8, device=cuda)
    lg = torch.from_numpy(logits).to(cuda, torch.bfloat16)
    _fused_vs_k4k5(O, lg, b, logits, toks, use, S, Rps, V, 2.0 ** -8 + 1e-5, "bf16")


@pytest.mark.parametrize("V", [131072, 4096, 204800])
def test_fused_forward_backward_f32(cuda, V):
    """f32 logits: the 4-CTA-cluster one-read kernel == K4 + K5, f32 gradient pinned per element."""
    from paper_2509_18883_b200 import objective as O
    G, S, Rps, T_max = 4, 8, 9, 16
    logits, toks, lt, li, adv, use, cu = _synthetic_rows(Rps, S, V, G, seed=4, tau=0.8, masked=(1, 6))
    g = np.random.default_rng(9)
    logits = (logits + g.normal(0, 1e-3, logits.shape)).astype(np.float32).astype(np.float64)  # not bf16-valued
    b = O.GRPOBatch.pack(toks, lt, li, cu, adv, use, G, T_max, temperature=0.8, device=cuda)
    lg = torch.from_numpy(logits).to(cuda, torch.float32)
    _fused_vs_k4k5(O, lg, b, logits, toks, use, S, Rps, V, 5e-6, "f32")


def _fused_vs_k4k5(O, lg, b, logits, toks, use, S, Rps, V, rtol, tag):
    fwd, grad = O.grpo_forward_backward(lg, b, grad_scale=-1.0)
    ref = O.grpo_forward(lg, b)
    gref = O.grpo_backward(lg, b, ref, -1.0, grad_dtype=torch.float32)
    # the fused kernel's epilogue is float64 like K4's; the row sums differ only in f32 summation order
    assert float(fwd.objective) == pytest.approx(float(ref.objective), rel=2e-6, abs=1e-12)
    np.testing.assert_allclose(fwd.logp.cpu().numpy(), ref.logp.cpu().numpy(), rtol=0, atol=2e-6)
    np.testing.assert_allclose(fwd.coef.cpu().numpy(), ref.coef.cpu().numpy(), rtol=2e-6, atol=1e-12)
    # every entry of the one-read gradient vs grad_scale * coef * (onehot - softmax) in f64
    assert grad.dtype == lg.dtype
    cf = -fwd.coef.cpu().numpy()
    worst = assert_grad_rows(grad.double().cpu().numpy(), logits, toks, cf, [0.8] * len(toks), rtol)
    print(f"fused {tag} grad V={V}: worst per-element error = {worst:.3f} of the bound")
    # and against K5's f32 gradient: both within bf16 rounding of each other
    g32 = gref.cpu().numpy()
    assert_grad_rows(g32, logits, toks, cf, [0.8] * len(toks), 1e-5)
    sor = np.repeat(np.arange(S), Rps)
    assert not grad[torch.from_numpy(~use[sor].astype(bool)).to(lg.device)].any()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_extreme_logits_vs_oracle(cuda, dtype):
    """Rows with very large spreads (a +60 spike over -1e4 tails, temperature 0.3 and 3.0): the online
    log-sum-exp (K4), the fused loss+gradient and the oracle agree; no overflow or flag."""
    from paper_2509_18883_b200 import objective as O
    V, R = 4096, 64
    g = np.random.default_rng(8)
    logits = g.normal(0, 3.0, (R, V))
    logits[:, ::7] = -1.0e4
    logits[np.arange(R), g.integers(0, V, R)] = 60.0
    logits = bf16_round(logits) if dtype == torch.bfloat16 else logits.astype(np.float32).astype(np.float64)
    toks = g.integers(0, V, R)
    toks[::5] = np.argmax(logits[::5], axis=1)
    for tau in (0.3, 3.0):
        lt = np.array([OO.log_token_dist(logits[r], tau)[toks[r]] for r in range(R)]) + g.normal(0, 0.2, R)
        li = lt + g.normal(0, 0.05, R)
        b = O.GRPOBatch.pack(toks, lt, li, [0, R // 2, R], [1.0, -1.0], [1, 1], 2, R, temperature=tau, device=cuda)
        lg = torch.from_numpy(logits).to(cuda, dtype)
        fwd = O.grpo_forward(lg, b)
        assert int(fwd.flags.item()) == 0
        clip = dict(eps_neg_low=0.2, eps_pos_high=0.2, eps_neg_high=3.0, tis_cap=2.0, guard_positive=True)
        logp, term, coef = OO.token_terms(logits, None, toks, lt, li, (np.arange(R) >= R // 2).astype(np.int64),
                                          [1.0, -1.0], [1, 1], [tau, tau], clip, norm=1.0 / (2 * R))
        np.testing.assert_allclose(fwd.logp.cpu().numpy(), logp, rtol=1e-6, atol=1e-5)
        np.testing.assert_allclose(fwd.term.cpu().numpy(), term, rtol=1e-4, atol=1e-9)
        if True:  # the one-read kernel for both dtypes (2- and 4-CTA clusters)
            fused, grad = O.grpo_forward_backward(lg, b)
            assert int(fused.flags.item()) == 0
            assert float(fused.objective) == pytest.approx(float(fwd.objective), rel=1e-4, abs=1e-9)
            assert bool(torch.isfinite(grad.float()).all())


@pytest.mark.parametrize("gdt", [torch.float64, torch.float32])
def test_backward_row_index_shared_and_unused_rows(cuda, gdt):
    """Tokens that read the same logits row accumulate into it (CSR, reference order) and rows no token
    reads get a zero gradient -- through grpo_backward, the fused entry point's fallback and autograd
    (objective.py:271-282: grad[c, t] -= coef p; grad[c, t][tok] += coef)."""
    from paper_2509_18883_b200 import objective as O
    g = np.random.default_rng(21)
    V, Rl = 2048, 10
    logits = g.normal(0, 1.5, (Rl, V))
    rows = np.array([3, 3, 7, 0, 3, 7, 9, 0])  # rows 1, 2, 4, 5, 6, 8 are never read
    R = len(rows)
    toks = g.integers(0, V, R)
    toks[1] = toks[0]  # two tokens with the same id on the same row
    lt = np.array([OO.log_token_dist(logits[r], 0.9)[t] for r, t in zip(rows, toks)]) + g.normal(0, 0.2, R)
    li = lt + g.normal(0, 0.05, R)
    b = O.GRPOBatch.pack(toks, lt, li, [0, 4, R], [1.0, -1.0], [1, 1], 2, 4, temperature=0.9, device=cuda,
                         row_index=rows)
    lg = torch.from_numpy(logits).to(cuda)
    fwd = O.grpo_forward(lg, b)
    coef = fwd.coef.cpu().numpy()
    assert (coef != 0).sum() >= 4
    ref = OO.gradient_rows(logits, rows, toks, coef, [0.9] * R, logits.shape)
    outs = [O.grpo_backward(lg, b, fwd, grad_dtype=gdt)]
    if gdt == torch.float64:
        outs.append(O.grpo_forward_backward(lg, b)[1])  # f64 logits: the K4 + K5 fallback
        lga = lg.clone().requires_grad_(True)
        O.grpo_token_objective(lga, b).backward()
        outs.append(lga.grad)
    for got in outs:
        got = got.double().cpu().numpy()
        assert got.shape == logits.shape
        unused = sorted(set(range(Rl)) - set(rows.tolist()))
        assert not got[unused].any()
        if gdt == torch.float64:
            np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-18)
        else:
            # per element: sum over the row's tokens of |coef| (p + onehot) bounds the f32 error
            bound = np.zeros_like(ref)
            for k in range(R):
                p = np.exp(OO.log_token_dist(logits[rows[k]], 0.9))
                p[toks[k]] += 1.0
                bound[rows[k]] += abs(coef[k]) * p
            assert np.all(np.abs(got - ref) <= 2e-5 * bound + 1e-30)


def test_backward_rejects_short_logits(cuda):
    from paper_2509_18883_b200 import objective as O
    b = O.GRPOBatch.pack([1, 2, 3], [-1.0] * 3, [-1.0] * 3, [0, 3], [1.0], [1], 1, 4, device=cuda)
    lg = torch.zeros((4, 16), device=cuda)
    fwd = O.grpo_forward(lg, b)
    g = O.grpo_backward(lg, b, fwd)  # extra logits rows: zero gradient there
    assert g.shape == (4, 16) and not g[3].any()
    with pytest.raises(ValueError):
        O.grpo_backward(lg[:2], b, fwd)


def test_train_logps_length_semantics(cuda, golden_objective):
    """The reference reads train_logps[t] for t < len(tokens) only (objective.py:243-247): extra entries
    change nothing, a short list raises IndexError."""
    import dataclasses
    from paper_2509_18883_b200 import core, objective as O
    from paper_2509_18883_b200.toy_env import ParamTable
    batch, clip = _rebuild_batch(golden_objective, "mid")
    params = ParamTable(golden_objective["mid/logits"])
    J0 = O.objective_value(batch, params, clip)
    G0 = O.objective_gradient(batch, params, clip).cpu().numpy()

    def edit(fn):
        groups = []
        for mg in batch.groups:
            samples = tuple(fn(s) for s in mg.group.samples)
            groups.append(O.MaskedGroup(core.Group(mg.group.prompt_id, samples), mg.advantages, mg.masks))
        return O.MaskedBatch(tuple(groups), batch.t_max)

    longer = edit(lambda s: dataclasses.replace(s, train_logps=tuple(s.train_logps) + (123.0, -7.0)))
    assert O.objective_value(longer, params, clip) == J0
    np.testing.assert_array_equal(O.objective_gradient(longer, params, clip).cpu().numpy(), G0)
    shorter = edit(lambda s: dataclasses.replace(s, train_logps=tuple(s.train_logps)[:-1]))
    with pytest.raises(IndexError):
        O.objective_value(shorter, params, clip)


@pytest.mark.parametrize("cname", ["rep_default", "rep_ngram3", "mean_only"])
def test_objective_mask_branches_vs_reference(cuda, cname):
    """objective_value / objective_gradient on batches with kept and masked truncations, grade errors and
    groups with fewer than two usable samples, against the unmodified reference's numbers
    (tests/golden/make_golden_masks.py; objective.py:168-203, 230-283)."""
    from paper_2509_18883_b200 import objective as O
    from paper_2509_18883_b200.toy_env import ParamTable
    from tests.conftest import GOLDEN
    from tests.test_host_logic_cpu import rebuild_mask_batch
    z = np.load(GOLDEN / "objective_masks.npz")
    batch, _ = rebuild_mask_batch(z, cname)
    params = ParamTable(z[f"{cname}/logits"])
    clip = O.ClipConfig()
    J = O.objective_value(batch, params, clip)
    assert J == pytest.approx(float(z[f"{cname}/value"][0]), rel=1e-12, abs=1e-16)
    grad = O.objective_gradient(batch, params, clip).cpu().numpy()
    np.testing.assert_allclose(grad, z[f"{cname}/grad"], rtol=1e-10, atol=1e-16)


@pytest.mark.parametrize("V", [1000, 250000])
def test_forward_backward_fallback_shapes(cuda, V):
    """Vocabularies the cluster kernel does not take (V % 16 != 0, V > 204,800) go through K4 + K5 with the
    same results: J and every gradient entry against the f64 oracle."""
    from paper_2509_18883_b200 import objective as O
    G, S, Rps, T_max = 4, 4, 5, 8
    logits, toks, lt, li, adv, use, cu = _synthetic_rows(Rps, S, V, G, seed=6, tau=1.0, masked=(1,))
    b = O.GRPOBatch.pack(toks, lt, li, cu, adv, use, G, T_max, device=cuda)
    lg = torch.from_numpy(logits).to(cuda, torch.bfloat16)
    fwd, grad = O.grpo_forward_backward(lg, b)
    clip = dict(eps_neg_low=0.2, eps_pos_high=0.2, eps_neg_high=3.0, tis_cap=2.0, guard_positive=True)
    sor = np.repeat(np.arange(S), Rps)
    norm = 1.0 / ((S // G) * G * T_max)
    logp, term, coef = OO.token_terms(logits, None, toks, lt, li, sor, adv, use, [1.0] * S, clip, norm=norm)
    J = OO.objective(term, list(cu[::G]), G, T_max)
    assert float(fwd.objective) == pytest.approx(J, rel=1e-3)
    cg = fwd.coef.cpu().numpy()
    rtol = 5e-6 if grad.dtype == torch.float32 else 2.0 ** -8 + 5e-6
    assert_grad_rows(grad.double().cpu().numpy(), logits, toks, cg, [1.0] * len(toks), rtol)
