"""Wider GPU parity matrix for fusion: expert counts 1..8, every dtype pair, fixed targets and weights,
delta-mode task vectors, ragged / tiny / empty-delta tensors.  Reference = oracle (pinned to the
unmodified reference by tests/test_oracle_golden.py)."""
import numpy as np
import pytest
import torch

from oracle import fusion as OF
from tests.helpers import bf16_round, rne_bf16_bits, synth_state_dicts

pytestmark = pytest.mark.gpu

SHAPES = {"a": (257, 129), "b": (65536 + 9,), "c": (3,), "d": (64, 64)}


def _round_for(dtype):
    if dtype == torch.bfloat16:
        return bf16_round
    if dtype == torch.float32:
        return lambda x: np.asarray(x, np.float32).astype(np.float64)
    return lambda x: np.asarray(x, np.float64)


def _check(out, ref, dtype, name):
    if dtype == torch.bfloat16:
        g = out.reshape(-1).view(torch.int16).cpu().numpy().view(np.uint16)
        assert (g != rne_bf16_bits(ref)).sum() == 0, name
    elif dtype == torch.float32:
        np.testing.assert_array_equal(out.reshape(-1).cpu().numpy(), ref.astype(np.float32), err_msg=name)
    else:
        # scale factors differ from numpy's by <= 1 ulp; cancellation can amplify that in relative terms
        np.testing.assert_allclose(out.reshape(-1).cpu().numpy(), ref, rtol=1e-12, atol=1e-14 * np.abs(ref).max(),
                                   err_msg=name)


@pytest.mark.parametrize("n_exp", [1, 2, 4, 5, 8])
@pytest.mark.parametrize("cfgkw", [dict(), dict(dropout_p=0.3, seed=5, erase_weighting="squared")])
def test_expert_counts(cuda, n_exp, cfgkw):
    from paper_2509_18883_b200 import fusion as F
    base, experts = synth_state_dicts(SHAPES, n_exp, seed=11, dtype_round=bf16_round)
    to = lambda d: {k: torch.from_numpy(v).to(cuda, torch.bfloat16) for k, v in d.items()}
    outs, rep = F.fuse_state_dict(to(base), [to(e) for e in experts], F.FusionConfig(**cfgkw))
    for name in base:
        ref, st = OF.fuse(base[name], [e[name] for e in experts], **cfgkw)
        _check(outs[name], ref, torch.bfloat16, name)
        s = rep.stats(name)
        assert list(s.erased_counts) == st["erased"] and list(s.dropout_kept_fraction) == st["kept"], name


@pytest.mark.parametrize("din", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("dout", [torch.bfloat16, torch.float32, torch.float64])
def test_dtype_pairs(cuda, din, dout):
    from paper_2509_18883_b200 import fusion as F
    cfgkw = dict(dropout_p=0.5, seed=9, target_norm=0.5, merge_weights=(0.2, 0.3, 0.5))
    base, experts = synth_state_dicts(SHAPES, 3, seed=12, dtype_round=_round_for(din))
    to = lambda d: {k: torch.from_numpy(v).to(cuda, din) for k, v in d.items()}
    outs, rep = F.fuse_state_dict(to(base), [to(e) for e in experts], F.FusionConfig(**cfgkw), out_dtype=dout)
    for name in base:
        ref, st = OF.fuse(base[name], [e[name] for e in experts], **cfgkw)
        _check(outs[name], ref, dout, name)
        assert list(rep.stats(name).erased_counts) == st["erased"], name


def test_delta_mode_and_unchanged_tensor(cuda):
    """TaskVectors given as explicit deltas (delta-mode kernels) and a tensor no expert changed."""
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.toy_env import ParamTable
    g = np.random.default_rng(3)
    b = g.normal(0, 1, 1000)
    ds = [g.normal(0, 0.1, 1000) for _ in range(3)]
    base = ParamTable(b.reshape(1, 1, -1))
    taus = [F.TaskVector(d.reshape(1, 1, -1)) for d in ds]
    for cfgkw in (dict(), dict(dropout_p=0.4, seed=2), dict(erase_weighting="squared", target_norm=None)):
        fused, st = F.fuse(base, taus, F.FusionConfig(**cfgkw))
        ref, rst = OF.fuse(b, [b + d for d in ds], **cfgkw)
        # reference deltas are (b + d) - b; ours are d exactly -> compare against the oracle on exact deltas
        np.testing.assert_allclose(fused.numpy().ravel(), ref, rtol=1e-9, atol=1e-12)
    # fuse_state_dict passes an unchanged tensor through (documented deviation)
    t = torch.randn(300, device=cuda, dtype=torch.bfloat16)
    outs, rep = F.fuse_state_dict({"w": t, "x": t + 0}, [{"w": t, "x": t * 2} for _ in range(2)], F.FusionConfig())
    assert torch.equal(outs["w"], t)
    assert rep.passthrough() == ["w"]


def test_ragged_tails_and_item_boundaries(cuda):
    from paper_2509_18883_b200 import fusion as F
    for n in (1, 7, 8, 9, 4095, 4096, 4097, 65535, 65536, 65537, 131071 + 65536):
        base, experts = synth_state_dicts({"t": (n,)}, 3, seed=n, dtype_round=bf16_round)
        to = lambda d: {k: torch.from_numpy(v).to(cuda, torch.bfloat16) for k, v in d.items()}
        cfgkw = dict(dropout_p=0.5, seed=1)
        outs, rep = F.fuse_state_dict(to(base), [to(e) for e in experts], F.FusionConfig(**cfgkw))
        ref, st = OF.fuse(base["t"], [e["t"] for e in experts], **cfgkw)
        _check(outs["t"], ref, torch.bfloat16, f"n={n}")
        assert list(rep.stats("t").erased_counts) == st["erased"], n


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_generic_path_extreme_magnitudes(cuda, dtype):
    """The reference-order f64 merge on f32 / f64 data spanning 1e-30..1e30, signed zeros and
    opposite-sign experts: f32 output = RN_f32(reference), f64 output within 1e-12."""
    from paper_2509_18883_b200 import fusion as F
    g = np.random.default_rng(31)
    n = 40000
    base = 10.0 ** g.uniform(-30, 30, n) * g.choice([-1.0, 1.0], n)
    base[g.random(n) < 0.05] = 0.0
    experts = []
    for i in range(3):
        e = base * (1 + g.normal(0, 0.01 * (i + 1), n))
        flip = g.random(n) < 0.1
        e[flip] = -base[flip] * 0.5
        experts.append(e)
    rnd = _round_for(dtype)
    base, experts = rnd(base), [rnd(e) for e in experts]
    to = lambda a: {"w": torch.from_numpy(a).to(cuda, dtype)}
    for cfgkw in (dict(dropout_p=0.5, seed=2), dict(erase_weighting="squared", target_norm=None)):
        outs, rep = F.fuse_state_dict(to(base), [to(e) for e in experts], F.FusionConfig(**cfgkw))
        ref, st = OF.fuse(base, experts, **cfgkw)
        _check(outs["w"], ref, dtype, str(cfgkw))
        assert list(rep.stats("w").erased_counts) == st["erased"]
