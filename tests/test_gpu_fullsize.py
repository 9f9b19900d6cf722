"""Parity at BASELINE.json's full config-3 size (Llama-3-8B-shaped, 8.03e9 params, 291 tensors, 3 experts,
FusionConfig(dropout_p=0.5, seed=42), the bench workload), through size-independent checks:

* the certified f32x2 merge and the reference-order float64 merge give bit-identical outputs and
  FusionStats counters over every tensor (64-bit checksums of each output tensor);
* whole full-size tensors against the oracle: a 4096x4096 q_proj (16.8M) and a 1024x4096 k_proj
  (every element, bit-exact RNE_bf16 of the reference, exact FusionStats);
* the K1 norms of the 525M-element embedding against numpy's float64 norm of the same data.
Needs ~100 GB of HBM; skipped on smaller devices."""
import numpy as np
import pytest
import torch

from oracle import fusion as OF
from tests.helpers import assert_grad_rows, rne_bf16_bits

pytestmark = pytest.mark.gpu


def _checksums(tensors, stream=None):
    from paper_2509_18883_b200 import _lib as L
    sums = torch.zeros(len(tensors), dtype=torch.int64, device=tensors[0].device)
    for k, t in enumerate(tensors):
        flat = t.view(torch.uint8)
        n = flat.numel() // 8
        L.call("rlk_checksum64", L.ptr(flat), n, 0, L.ptr(sums[k:k + 1]), L.stream_handle(stream))
    return sums.cpu()


@pytest.fixture(scope="module")
def config3(cuda):
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.layouts import LAYOUTS, fill_synthetic, numel
    torch.cuda.empty_cache()
    free, total = torch.cuda.mem_get_info()
    if free < 100 << 30:
        pytest.skip("needs ~100 GB of free HBM")
    shapes = LAYOUTS["llama8b"]()
    names = list(shapes)
    pieces = []
    for t, k in enumerate(names):
        n = numel(shapes[k])
        b = torch.empty(n, dtype=torch.bfloat16, device=cuda)
        es = [torch.empty(n, dtype=torch.bfloat16, device=cuda) for _ in range(3)]
        fill_synthetic(b, es, t, seed=0)
        pieces.append(F.Piece(t, 0, b, es, torch.empty(n, dtype=torch.bfloat16, device=cuda)))
    layout = F.FusionLayout([p.numel for p in pieces])
    cfg = F.FusionConfig(dropout_p=0.5, seed=42)
    call = F.FusionCall(pieces, layout, 3, cfg)
    call.run((1 / 3,) * 3)
    torch.cuda.synchronize()
    yield names, pieces, call
    del pieces, call
    torch.cuda.empty_cache()


def test_fullsize_fast_equals_reference_order(config3):
    names, pieces, call = config3
    fast = _checksums([p.out for p in pieces])
    counters = call.counters.clone()
    call.counters[:, 3:].zero_()  # the erased counts are K3's; the non-zero counts stay from K1
    call.exact_merge = True
    try:
        call.merge((1 / 3,) * 3)
    finally:
        call.exact_merge = False
    torch.cuda.synchronize()
    exact = _checksums([p.out for p in pieces])
    assert torch.equal(fast, exact)
    assert torch.equal(counters, call.counters)


@pytest.mark.parametrize("name", ["model.layers.0.self_attn.q_proj.weight", "model.layers.31.self_attn.k_proj.weight"])
def test_fullsize_tensor_vs_oracle(config3, name):
    names, pieces, call = config3
    t = names.index(name)
    p = pieces[t]
    f64 = lambda x: x.float().double().cpu().numpy()
    ref, st = OF.fuse(f64(p.base), [f64(e) for e in p.experts], dropout_p=0.5, seed=42)
    got = p.out.view(torch.int16).cpu().numpy().view(np.uint16)
    assert int((got != rne_bf16_bits(ref)).sum()) == 0
    mine = call.stats(t, (1 / 3,) * 3)
    assert list(mine.erased_counts) == st["erased"]
    assert list(mine.dropout_kept_fraction) == st["kept"]
    np.testing.assert_allclose(mine.norms_before, st["norms_before"], rtol=1e-13)


def test_fullsize_embedding_norms(config3):
    names, pieces, call = config3
    t = names.index("model.embed_tokens.weight")
    p = pieces[t]
    b = p.base.float().double()
    for i, e in enumerate(p.experts):
        d = (e.float().double() - b).cpu().numpy()
        ref = float(np.sqrt(np.dot(d, d)))
        got = float(np.sqrt(call.sumsq[t, i].item()))
        assert got == pytest.approx(ref, rel=1e-13)


def test_fullsize_grpo_config5_chunk(cuda):
    """Config 5 at its launch size (2 responses x 32,768 tokens, V = 131,072 bf16 = 16 GiB of logits,
    off-policy, tau = 0.7): the fused loss+gradient kernel agrees with the K4 forward on J and every
    row's coefficient; sampled rows (incl. the first and last) match the oracle's logp / term / coef
    and gradient rows; every gradient row sums to ~0 (softmax sums to one)."""
    from paper_2509_18883_b200 import _lib as L
    from paper_2509_18883_b200 import objective as O
    from oracle import objective as OO
    torch.cuda.empty_cache()
    if torch.cuda.mem_get_info()[0] < 40 << 30:
        pytest.skip("needs ~40 GB of free HBM")
    V, T = 131072, 32768
    R = 2 * T
    lg = torch.empty((R, V), dtype=torch.bfloat16, device=cuda)
    L.call("rlk_synth_normal", L.ptr(lg), L.RLK_BF16, lg.numel(), 0, 99, 2.0, None, L.stream_handle())
    g = np.random.default_rng(5)
    toks = g.integers(0, V, R)
    lt = g.normal(-12.0, 0.3, R)
    li = lt + g.normal(0, 0.05, R)
    adv = np.array([1.0, -1.0])
    b = O.GRPOBatch.pack(toks, lt, li, [0, T, R], adv, [1, 1], 2, T, temperature=0.7, device=cuda)
    fwd = O.grpo_forward(lg, b)
    fused, grad = O.grpo_forward_backward(lg, b)
    assert float(fused.objective) == pytest.approx(float(fwd.objective), rel=2e-6)
    np.testing.assert_allclose(fused.coef.cpu().numpy(), fwd.coef.cpu().numpy(), rtol=2e-6, atol=1e-14)
    rows = np.unique(np.concatenate([[0, T - 1, T, R - 1], g.integers(0, R, 28)]))
    z = lg[torch.from_numpy(rows).to(cuda)].float().double().cpu().numpy()
    clip = dict(eps_neg_low=0.2, eps_pos_high=0.2, eps_neg_high=3.0, tis_cap=2.0, guard_positive=True)
    sample = (rows >= T).astype(np.int64)
    logp, term, coef = OO.token_terms(z, None, toks[rows], lt[rows], li[rows], sample, adv, [1, 1], [0.7, 0.7],
                                      clip, norm=1.0 / (1 * 2 * T))
    # K4 sums 2^x in f32 per thread over the 131,072-wide row (f64 combine): logp to ~1e-7 absolute
    np.testing.assert_allclose(fwd.logp.cpu().numpy()[rows], logp, rtol=0, atol=2e-6)
    np.testing.assert_allclose(fwd.term.cpu().numpy()[rows], term, rtol=1e-5, atol=1e-15)
    np.testing.assert_allclose(fwd.coef.cpu().numpy()[rows], coef, rtol=1e-5, atol=1e-18)
    # every entry of the sampled bf16 gradient rows (131,072 each) vs coef * (onehot - softmax) in f64,
    # relative per element (bf16 unit roundoff 2^-8 + the f32 row arithmetic)
    gg = grad[torch.from_numpy(rows).to(cuda)].double().cpu().numpy()
    cf = fused.coef.cpu().numpy()[rows]
    worst = assert_grad_rows(gg, z, toks[rows], cf, [0.7] * len(rows), 2.0 ** -8 + 1e-5)
    print(f"config-5 chunk: worst per-element gradient error = {worst:.3f} of the bound")
    sums = grad.float().sum(dim=1).double().cpu().numpy()
    cmax = np.abs(fused.coef.cpu().numpy())
    assert np.all(np.abs(sums) <= 1e-2 * cmax + 1e-12)
    del lg, grad
    torch.cuda.empty_cache()
