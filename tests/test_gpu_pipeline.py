"""Pipeline -> GPU loss: a batch emitted by the BatchAssembler, packed by `pipeline.pack_batch`, through
the GRPO kernels (K4 forward, fused forward+backward) against the oracle on the same rows."""
import numpy as np
import pytest
import torch

from oracle import objective as OO
from paper_2509_18883_b200 import core as C
from paper_2509_18883_b200 import objective as O
from paper_2509_18883_b200 import pipeline as P
from tests.helpers import assert_grad_rows

pytestmark = pytest.mark.gpu


def _stream(g, n_groups, G, V, t_max, pid0=0):
    """Graded groups with mixed outcomes, grade errors and truncations (some ending in a repetition loop)."""
    out = []
    for pid in range(pid0, pid0 + n_groups):
        samples = []
        for i in range(G):
            L = int(g.integers(1, t_max + 1))
            toks = [int(x) for x in g.integers(0, V, L)]
            status = C.SampleStatus.COMPLETE
            if g.random() < 0.25:
                status = C.SampleStatus.TRUNCATED
                if g.random() < 0.5 and L >= 8:  # tail loop of a 2-gram
                    toks[-8:] = toks[-2:] * 4
            u = g.random()
            reward = C.RewardOutcome.grade_error() if u < 0.1 else (
                C.RewardOutcome.passed() if u < 0.55 else C.RewardOutcome.failed())
            lt = tuple(float(-np.log(V) + g.normal(0, 0.3)) for _ in toks)
            li = tuple(x + float(g.normal(0, 0.05)) for x in lt)
            samples.append(C.Sample(prompt_id=pid, context_id=0, version_id=0, tokens=tuple(toks), infer_logps=li,
                                    status=status, t_start=0, train_logps=lt, reward=reward,
                                    gen_temperature=float(g.choice([1.0, 0.8]))))
        out.append(C.Group(pid, tuple(samples)))
    return out


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_assembled_batch_through_grpo_kernels(cuda, dtype):
    g = np.random.default_rng(31)
    V, G, t_max = 8192, 4, 24
    asm = P.BatchAssembler(6, P.StalenessPolicy(2), P.ReplayBuffer(8, 0.25), C.Rng(5))
    for grp in _stream(g, 4, G, V, t_max):  # oversampled groups already in the buffer
        asm.buffer.insert(grp)
    batch = None
    for grp in _stream(g, 40, G, V, t_max, pid0=100):
        res = asm.offer(grp, 0)
        if res.batch is not None:
            batch = res.batch
            assert res.reused_count == 1
            break
    assert batch is not None
    masked, b = P.pack_batch(batch, t_max, device=cuda)
    R = b.n_rows
    logits = g.normal(0, 2.0, (R, V)).astype(np.float32)
    lg = torch.from_numpy(logits).to(cuda, dtype)
    z = lg.double().cpu().numpy()
    # oracle on the same packed rows (apply_masks is pinned against the reference separately)
    toks = b.tokens.cpu().numpy()
    lt, li = b.logp_train.cpu().numpy(), b.logp_infer.cpu().numpy()
    sor = b.sample_of_row.cpu().numpy()
    adv, use, temps = b.adv.cpu().numpy(), b.use.cpu().numpy(), b.temperature.cpu().numpy()
    assert use.sum() < len(use)  # the stream produced masked samples
    clip = dict(eps_neg_low=0.2, eps_pos_high=0.2, eps_neg_high=3.0, tis_cap=2.0, guard_positive=True)
    norm = 1.0 / (b.n_groups * G * t_max)
    logp, term, coef = OO.token_terms(z, None, toks, lt, li, sor, adv, use, temps, clip, norm=norm)
    cu = list(b.sample_rows_host)
    J = OO.objective(term, cu[::G], G, t_max)
    fwd = O.grpo_forward(lg, b)
    assert float(fwd.objective) == pytest.approx(J, rel=1e-3, abs=1e-9)  # north-star tolerance
    act = use[sor].astype(bool)
    np.testing.assert_allclose(fwd.logp.cpu().numpy()[act], logp[act], rtol=0, atol=2e-5)
    # fused forward+backward on the same batch: same J, every gradient entry per element
    ff, grad = O.grpo_forward_backward(lg, b)
    assert float(ff.objective) == pytest.approx(J, rel=1e-3, abs=1e-9)  # north-star tolerance
    assert grad.dtype == dtype
    rtol = 5e-6 if dtype == torch.float32 else 2.0 ** -8 + 5e-6
    assert_grad_rows(grad.double().cpu().numpy(), z, toks, ff.coef.cpu().numpy(), temps[sor], rtol)
