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
from tests.helpers import rne_bf16_bits

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


def test_fullsize_fast_equals_reference_order(config3, monkeypatch):
    names, pieces, call = config3
    fast = _checksums([p.out for p in pieces])
    counters = call.counters.clone()
    monkeypatch.setenv("RLK_MERGE_FAST", "0")
    call.counters[:, 3:].zero_()  # the erased counts are K3's; the non-zero counts stay from K1
    call.merge((1 / 3,) * 3)
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
