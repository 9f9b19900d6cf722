"""GPU parity: the sm_100a fusion kernels vs the reference's golden vectors and the CPU oracle."""
import os

import numpy as np
import pytest
import torch

from oracle import fusion as OF
from oracle import rng as OR
from tests.helpers import bf16_bits_to_f64, bf16_round, mlp_dict_shapes, rne_bf16_bits, synth_state_dicts

pytestmark = pytest.mark.gpu

CFGS = {
    "default": dict(),
    "p05_s42": dict(dropout_p=0.5, seed=42),
    "p05_s42_sq": dict(dropout_p=0.5, seed=42, erase_weighting="squared"),
    "p03_s7_t1_w": dict(dropout_p=0.3, seed=7, target_norm=1.0, merge_weights=(0.5, 0.3, 0.2)),
    "none_noerase": dict(target_norm=None, erase_mode=False),
    "p09_s3_none": dict(dropout_p=0.9, seed=3, target_norm=None),
}


def _pt(x, dtype, dev):
    from paper_2509_18883_b200.toy_env import ParamTable
    return ParamTable(torch.from_numpy(np.asarray(x, dtype=np.float64).reshape(1, 1, -1)).to(dev, dtype))


def _fuse(base, experts, cfgkw, dtype, dev, out_dtype=None, exact_merge=False):
    from paper_2509_18883_b200 import fusion as F
    b = _pt(base, dtype, dev)
    taus = [F.task_vector(_pt(e, dtype, dev), b) for e in experts]
    return F.fuse(b, taus, F.FusionConfig(**cfgkw), out_dtype=out_dtype, exact_merge=exact_merge)


@pytest.mark.parametrize("cname", list(CFGS))
def test_fuse_kat_f64(cuda, golden_fusion, cname):
    base = golden_fusion["kat/base"]
    experts = [golden_fusion[f"kat/expert{k}"] for k in range(3)]
    fused, st = _fuse(base, experts, CFGS[cname], torch.float64, cuda)
    ref = golden_fusion[f"kat/{cname}/fused"]
    got = fused.numpy().ravel()
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-15)
    assert list(st.erased_counts) == list(golden_fusion[f"kat/{cname}/erased"])
    assert list(st.dropout_kept_fraction) == list(golden_fusion[f"kat/{cname}/kept"])
    np.testing.assert_allclose(st.norms_before, golden_fusion[f"kat/{cname}/norms_before"], rtol=1e-13)
    np.testing.assert_allclose(st.norms_after_normalize, golden_fusion[f"kat/{cname}/norms_after"], rtol=1e-13)
    # erase decisions bit-exact: zero pattern of the fused-minus-base contribution
    assert (got == base).sum() == (ref == base).sum()


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("cname", ["default", "p05_s42", "p05_s42_sq", "p03_s7_t1_w", "p09_s3_none", "none_noerase"])
def test_fuse_bf16_exact(cuda, golden_fusion, cname, exact):
    """bf16 in / bf16 out must equal RNE_bf16(reference f64 output) bit for bit (fast and exact K3)."""
    base = golden_fusion["bf16/base"]
    experts = [golden_fusion[f"bf16/expert{k}"] for k in range(3)]
    fused, st = _fuse(base, experts, CFGS[cname], torch.bfloat16, cuda, exact_merge=exact)
    got = fused.logits.reshape(-1).view(torch.int16).cpu().numpy().view(np.uint16)
    ref = rne_bf16_bits(golden_fusion[f"bf16/{cname}/fused"])
    mism = np.flatnonzero(got != ref)
    assert mism.size == 0, (mism[:10], got[mism[:10]], ref[mism[:10]])
    assert list(st.erased_counts) == list(golden_fusion[f"bf16/{cname}/erased"])
    assert list(st.dropout_kept_fraction) == list(golden_fusion[f"bf16/{cname}/kept"])
    # f64 output from bf16 inputs: same numbers as the f64 reference
    fused64, _ = _fuse(base, experts, CFGS[cname], torch.bfloat16, cuda, out_dtype=torch.float64)
    np.testing.assert_allclose(fused64.numpy().ravel(), golden_fusion[f"bf16/{cname}/fused"], rtol=1e-12,
                               atol=1e-16)


def test_staged_functions(cuda, golden_fusion):
    from paper_2509_18883_b200 import core, fusion as F
    base = golden_fusion["kat/base"]
    experts = [golden_fusion[f"kat/expert{k}"] for k in range(3)]
    b = _pt(base, torch.float64, cuda)
    taus = [F.task_vector(_pt(e, torch.float64, cuda), b) for e in experts]
    nm = F.normalize_magnitudes(taus, F.FusionConfig())
    for k in range(3):
        np.testing.assert_allclose(nm[k].delta.cpu().numpy().ravel(), golden_fusion[f"stage/normalized{k}"],
                                   rtol=1e-12, atol=1e-17)
    r = core.make_rng(11, "stage")
    dp = F.dropout_prune(taus[0], 0.4, r)
    got = dp.delta.cpu().numpy().ravel()
    ref = golden_fusion["stage/dropout0"]
    np.testing.assert_array_equal(got == 0, ref == 0)  # bit-exact mask
    np.testing.assert_array_equal(got, ref)  # (d / 0.6 exact division)
    assert r.next_u64() == int(golden_fusion["stage/dropout_rng_after"][0])  # rng advanced like the loop
    for w in ("sum", "squared"):
        er = F.erase_minority(taus, w)
        for k in range(3):
            np.testing.assert_array_equal(er[k].delta.cpu().numpy().ravel(), golden_fusion[f"stage/erase_{w}{k}"])
    tv = [F.TaskVector(np.array([[[v]]])) for v in (0.3, 0.1, -0.2)]
    assert [float(t.delta.item()) for t in F.erase_minority(tv)] == [0.3, 0.1, 0.0]


def test_fuse_validation_messages(cuda):
    from paper_2509_18883_b200 import fusion as F
    b = _pt(np.zeros(8), torch.float64, cuda)
    e = _pt(np.ones(8), torch.float64, cuda)
    with pytest.raises(ValueError, match="need at least one task vector"):
        F.fuse(b, [], F.FusionConfig())
    with pytest.raises(ValueError, match="merge_weights length"):
        F.fuse(b, [F.task_vector(e, b)], F.FusionConfig(merge_weights=(0.5, 0.5)))
    with pytest.raises(ValueError, match="cannot take mean norm of all-zero task vectors"):
        F.fuse(b, [F.task_vector(b, b)], F.FusionConfig())
    with pytest.raises(ValueError, match="logits must be finite"):
        F.ParamTable(torch.tensor([[[1.0, float("nan")]]], device=cuda))
    # an empty table, as the reference: no non-zero norm for the mean target; else 0 / 0 in the stats
    z = _pt(np.zeros(0), torch.float64, cuda)
    tz = F.task_vector(z, z)
    assert tz.norm == 0.0
    with pytest.raises(ValueError, match="cannot take mean norm of all-zero task vectors"):
        F.fuse(z, [tz, tz], F.FusionConfig())
    with pytest.raises(ZeroDivisionError):
        F.fuse(z, [tz, tz], F.FusionConfig(target_norm=None, dropout_p=0.5))
    # identity round trip: 1 expert, w=1, p=0, erase off
    fused, _ = F.fuse(b, [F.task_vector(e, b)], F.FusionConfig(target_norm=None, erase_mode=False))
    assert torch.equal(fused.logits, e.logits)
    # opposite deltas cancel back to the base
    e2 = _pt(-np.ones(8), torch.float64, cuda)
    fused, st = F.fuse(b, [F.task_vector(e, b), F.task_vector(e2, b)], F.FusionConfig())
    assert torch.equal(fused.logits, b.logits)


def _oracle_dict(base, experts, cfgkw):
    out, stats = {}, {}
    for name in base:
        f, s = OF.fuse(base[name], [e[name] for e in experts], **cfgkw)
        out[name], stats[name] = f, s
    return out, stats


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("cfgkw", [dict(), dict(dropout_p=0.5, seed=42), dict(dropout_p=0.3, seed=0,
                                                                             erase_weighting="squared")])
def test_state_dict_vs_oracle(cuda, dtype, cfgkw):
    """Config-1 shaped MLP dict (scaled 1/4): every tensor equals the per-tensor reference fuse."""
    from paper_2509_18883_b200 import fusion as F
    rnd = bf16_round if dtype == torch.bfloat16 else (lambda x: np.asarray(x, np.float32).astype(np.float64))
    base, experts = synth_state_dicts(mlp_dict_shapes(4), 3, seed=1, dtype_round=rnd)
    to = lambda d: {k: torch.from_numpy(v).to(cuda, dtype) for k, v in d.items()}
    outs, rep = F.fuse_state_dict(to(base), [to(e) for e in experts], F.FusionConfig(**cfgkw))
    ref, rstats = _oracle_dict(base, experts, cfgkw)
    for name in base:
        got = outs[name].reshape(-1)
        if dtype == torch.bfloat16:
            g = got.view(torch.int16).cpu().numpy().view(np.uint16)
            r = rne_bf16_bits(ref[name])
            assert (g != r).sum() == 0, name
        else:
            np.testing.assert_array_equal(got.cpu().numpy(), ref[name].astype(np.float32), err_msg=name)
        st = rep.stats(name)
        assert list(st.erased_counts) == rstats[name]["erased"], name
        assert list(st.dropout_kept_fraction) == rstats[name]["kept"], name
        np.testing.assert_allclose(st.norms_before, rstats[name]["norms_before"], rtol=1e-13)


def test_dropout_bitmap_equals_inline(cuda):
    from paper_2509_18883_b200 import fusion as F
    base, experts = synth_state_dicts(mlp_dict_shapes(4), 3, seed=2, dtype_round=bf16_round)
    to = lambda d: {k: torch.from_numpy(v).to(cuda, torch.bfloat16) for k, v in d.items()}
    cfg = F.FusionConfig(dropout_p=0.5, seed=9)
    res = []
    for mode in (1, 2):
        outs, rep = F.fuse_state_dict(to(base), [to(e) for e in experts], cfg, dropout_mode=mode)
        assert rep.call.dropout_mode == mode
        res.append((outs, rep.call.counters.cpu()))
    for k in res[0][0]:
        assert torch.equal(res[0][0][k], res[1][0][k])
    assert torch.equal(res[0][1], res[1][1])


def test_mask_bitmap_bit_exact(cuda):
    """K2 keep bits == the reference's `uniform >= p` draws, incl. a far index window."""
    from paper_2509_18883_b200 import _lib as L
    from paper_2509_18883_b200.core import fusion_child_seeds, keep_threshold
    # 0.3 / 0.9: full 64-bit compare; 1288490189 / 2^32: high-word compare with an odd threshold;
    # 0.5 / 0.75: even high-word threshold (K2's three modes)
    for p in (0.3, 0.5, 0.9, 1288490189 / 2**32, 0.75):
        seeds = fusion_child_seeds(42, 3)
        n_bits = 1 << 20
        wpr = n_bits // 32
        bm = torch.empty(3 * wpr, dtype=torch.int32, device=cuda)
        L.call("rlk_fusion_mask_bitmap", (L.C.c_uint64 * 3)(*seeds), 3, keep_threshold(p), n_bits, L.ptr(bm), wpr,
               L.stream_handle())
        bits = np.unpackbits(bm.cpu().numpy().view(np.uint8), bitorder="little").reshape(3, n_bits)
        for i in range(3):
            ref = OR.keep_mask(OR.fusion_child_seed(42, i), 0, n_bits, p)
            assert np.array_equal(bits[i].astype(bool), ref)
        # the sharded form: 3 'ranks' each draw one slice of every row (rlk_fusion_mask_bitmap_range)
        part = torch.full_like(bm, -1)
        cuts = [0, 11 * 32 * 1024, 23 * 32 * 1024, n_bits]
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            L.call("rlk_fusion_mask_bitmap_range", (L.C.c_uint64 * 3)(*seeds), 3, keep_threshold(p), lo, hi,
                   L.ptr(part), wpr, L.stream_handle())
        assert torch.equal(part, bm)


def test_fast_path_equals_exact_path_random(cuda, monkeypatch):
    """f32 fast path with certified guards == pure reference-order f64 path, on 24M bf16 elements
    including crafted near-ties and midpoint cases."""
    from paper_2509_18883_b200 import fusion as F
    g = torch.Generator(device=cuda).manual_seed(0)
    n = 24 * 1024 * 1024 + 7
    base = (torch.randn(n, device=cuda, generator=g) * 0.02).to(torch.bfloat16)
    experts = [(base.float() + torch.randn(n, device=cuda, generator=g) * 1e-3 * (i + 1)).to(torch.bfloat16)
               for i in range(3)]
    # near-ties: expert 2 = base - (d0 + d1) rounded
    idx = torch.arange(0, n, 97, device=cuda)
    d0 = experts[0].float()[idx] - base.float()[idx]
    d1 = experts[1].float()[idx] - base.float()[idx]
    experts[2][idx] = (base.float()[idx] - d0 - d1).to(torch.bfloat16)
    for cfg in (F.FusionConfig(), F.FusionConfig(dropout_p=0.5, seed=1), F.FusionConfig(erase_weighting="squared"),
                F.FusionConfig(target_norm=None), F.FusionConfig(target_norm=None, dropout_p=0.5, seed=2),
                F.FusionConfig(target_norm=None, dropout_p=0.75, seed=3, merge_weights=(0.5, 0.25, 0.25))):
        outs = []
        for exact in (False, True):
            o, rep = F.fuse_state_dict({"w": base}, [{"w": e} for e in experts], cfg, exact_merge=exact)
            outs.append((o["w"], rep.call.counters.clone()))
        assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16)), cfg
        assert torch.equal(outs[0][1], outs[1][1]), cfg


@pytest.mark.parametrize("striped", [False, True])
def test_sharded_items_identical(cuda, striped, monkeypatch):
    """Pieces split over 2/4 'ranks' (item-aligned) give bit-identical norms, outputs and counters.
    Striped: each rank's FusionCall takes the sharded keep-bitmap path (draws only the index ranges
    its pieces read, `needed_bit_ranges`), with the world size reported by a stand-in group."""
    from paper_2509_18883_b200 import fusion as F
    base, experts = synth_state_dicts({"a": (3000, 517), "b": (70001,), "c": (1024, 1024)}, 3, seed=3,
                                      dtype_round=bf16_round)
    names = list(base)
    to = lambda a: torch.from_numpy(a.reshape(-1)).to(cuda, torch.bfloat16)
    B = [to(base[k]) for k in names]
    E = [[to(e[k]) for k in names] for e in experts]
    layout = F.FusionLayout([b.numel() for b in B])
    cfg = F.FusionConfig(dropout_p=0.5, seed=5)
    w = (1 / 3, 1 / 3, 1 / 3)
    results = []
    for world in (1, 2, 4):
        outs = [torch.empty_like(b) for b in B]
        partials = torch.zeros(layout.n_items * 3, dtype=torch.float64, device=cuda)
        calls = []
        for rank in range(world):
            pieces = [F.Piece(t, lo, B[t][lo:hi], [E[i][t][lo:hi] for i in range(3)], outs[t][lo:hi])
                      for t, lo, hi in (layout.partition_striped if striped else layout.partition)(world, rank)]
            c = F.FusionCall(pieces, layout, 3, cfg)
            c.partials = partials
            from paper_2509_18883_b200 import _lib as L
            if striped and world > 1:
                import torch.distributed as dist
                monkeypatch.setattr(dist, "get_world_size", lambda group=None, w=world: w)
                c.group = "stand-in"
                c._bitmap(L.stream_handle())
                c.group = None
                monkeypatch.undo()
            else:
                c._bitmap(L.stream_handle())
            L.call("rlk_fusion_sumsq", L.C.byref(c.plan.c), 3, L.RLK_BF16, 0, L.ptr(partials), L.ptr(c.counters),
                   c.dropout_mode, (L.C.c_uint64 * 3)(*c.seeds), c.thresh, L.ptr(c.bitmap), c.words_per_row,
                   L.stream_handle())
            calls.append(c)
        counters = torch.zeros((3, 6), dtype=torch.int64, device=cuda)
        for c in calls:
            counters += c.counters  # K1's non-zero counts
            c.counters.zero_()
            L.call("rlk_fusion_finalize", L.ptr(partials), L.ptr(layout.tensor_items_device(cuda)), 3, 3, 1, 0.0,
                   L.ptr(c.sumsq), L.ptr(c.scale), L.ptr(c.status), L.stream_handle())
            c.merge(w)
            counters += c.counters
        results.append((calls[0].sumsq.clone(), [o.clone() for o in outs], counters))
    for r in results[1:]:
        assert torch.equal(r[0], results[0][0])
        for a, b in zip(r[1], results[0][1]):
            assert torch.equal(a.view(torch.int16), b.view(torch.int16))
        assert torch.equal(r[2], results[0][2])


def test_graph_capture_replays_the_step(cuda):
    """FusionCall.capture: the replayed graph gives the eager step's outputs and counters."""
    from paper_2509_18883_b200 import fusion as F
    base, experts = synth_state_dicts(mlp_dict_shapes(8), 3, seed=13, dtype_round=bf16_round)
    names = list(base)
    B = [torch.from_numpy(base[k].reshape(-1)).to(cuda, torch.bfloat16) for k in names]
    E = [[torch.from_numpy(e[k].reshape(-1)).to(cuda, torch.bfloat16) for k in names] for e in experts]
    pieces = [F.Piece(t, 0, B[t], [E[i][t] for i in range(3)], torch.empty_like(B[t])) for t in range(len(names))]
    call = F.FusionCall(pieces, F.FusionLayout([b.numel() for b in B]), 3, F.FusionConfig(dropout_p=0.5, seed=3),
                        stream=torch.cuda.Stream())
    w = (1 / 3,) * 3
    call.run(w)
    torch.cuda.synchronize()
    eager = [p.out.clone() for p in pieces]
    cnt = call.counters.clone()
    g = call.capture(w)
    for p in pieces:
        p.out.zero_()
    torch.cuda.synchronize()
    with torch.cuda.stream(call.stream):
        g.replay()
    torch.cuda.synchronize()
    for a, p in zip(eager, pieces):
        assert torch.equal(a.view(torch.int16), p.out.view(torch.int16))
    assert torch.equal(cnt, call.counters)


def test_fast_path_adversarial_values(cuda, monkeypatch):
    """The certified f32x2 merge against the reference-order f64 merge (bit-identical) and the oracle on
    bf16 data built to stress the guards: magnitudes from 1e-30 to 1e30 in one tensor, exact zeros of
    both signs, bf16 subnormals, experts of opposite sign to the base, exact vote ties and deltas that
    cancel across experts."""
    from paper_2509_18883_b200 import fusion as F
    g = np.random.default_rng(21)
    n = 1 << 18
    mag = 10.0 ** g.uniform(-30, 30, n)
    base = bf16_round(mag * g.choice([-1.0, 1.0], n))
    base[g.random(n) < 0.05] = 0.0
    base[g.random(n) < 0.02] = -0.0
    base[g.random(n) < 0.01] = bf16_round(np.full(1, 1e-39))[0]  # subnormal
    experts = []
    for i in range(3):
        e = bf16_round(base * (1 + g.normal(0, 0.01 * (i + 1), n)))
        flip = g.random(n) < 0.1
        e[flip] = bf16_round(-base[flip] * 0.5)  # opposite sign to the base
        same = g.random(n) < 0.1
        e[same] = base[same]  # zero deltas
        experts.append(e)
    # exact ties: expert 2's delta cancels expert 0's and expert 1 has none
    tie = g.random(n) < 0.05
    experts[1][tie] = base[tie]
    experts[2][tie] = bf16_round(2 * base[tie] - experts[0][tie])
    bt = torch.from_numpy(base).to(cuda, torch.bfloat16)
    ets = [torch.from_numpy(e).to(cuda, torch.bfloat16) for e in experts]
    for cfgkw in (dict(dropout_p=0.5, seed=4), dict(target_norm=None, dropout_p=0.5, seed=4),
                  dict(erase_weighting="squared", merge_weights=(0.5, 0.3, 0.2))):
        outs = []
        for exact in (False, True):
            o, rep = F.fuse_state_dict({"w": bt}, [{"w": e} for e in ets], F.FusionConfig(**cfgkw),
                                       exact_merge=exact)
            outs.append((o["w"].clone(), rep.call.counters.clone()))
        assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16)), cfgkw
        assert torch.equal(outs[0][1], outs[1][1]), cfgkw
        b64 = bt.float().double().cpu().numpy()
        ref, st = OF.fuse(b64, [e.float().double().cpu().numpy() for e in ets], **cfgkw)
        got = outs[0][0].view(torch.int16).cpu().numpy().view(np.uint16)
        assert int((got != rne_bf16_bits(ref)).sum()) == 0, cfgkw
        assert list(rep.stats("w").erased_counts) == st["erased"], cfgkw


def test_fast_path_power_of_two_boundaries(cuda):
    """Results just below / above a power of two under heavy cancellation (S ~ 2^11..2^12 |y|): the
    bf16 rounding boundary below 2^E sits at 2^E - 2^(E-9), a quarter of the upper ulp away, so a
    guard that only measures the distance to the upper midpoint would accept an f32 value above 2^E
    whose reference value rounds down.  The certified fast path (bracket [y - 2^-20 S, y + 2^-20 S]
    must round to one word) must equal the reference-order f64 path and RNE_bf16(oracle)."""
    from paper_2509_18883_b200 import fusion as F
    g = np.random.default_rng(5)
    n = 1 << 22
    # four experts: two huge cancelling deltas, then two finer ones steering the result onto the
    # boundary below 2^E (the last expert's granularity puts y within ~2^(E-10) of the target)
    w = np.array([0.4, 0.3, 0.2, 0.1])
    E = g.integers(-12, 12, n).astype(np.float64)
    p2 = 2.0 ** E
    base = bf16_round(p2 * (1 + g.integers(-4, 5, n) * 2.0 ** -8))
    target = p2 * (1 - 2.0 ** -9 * (1 + g.uniform(-2.0 ** -6, 2.0 ** -6, n)))  # the boundary below 2^E
    A = p2 * 2.0 ** g.uniform(10.5, 12.0, n)
    experts, acc = [], base.copy()
    e0 = bf16_round(base + A)
    experts.append(e0)
    acc += w[0] * (e0 - base)
    experts.append(bf16_round(base - w[0] * (e0 - base) / w[1]))
    acc += w[1] * (experts[1] - base)
    for i in (2, 3):
        experts.append(bf16_round(base + (target - acc) / w[i]))
        acc += w[i] * (experts[i] - base)
    bt = torch.from_numpy(base).to(cuda, torch.bfloat16)
    ets = [torch.from_numpy(e).to(cuda, torch.bfloat16) for e in experts]
    cfgkw = dict(target_norm=None, erase_mode=False, merge_weights=tuple(w))
    outs = []
    for exact in (False, True):
        o, _ = F.fuse_state_dict({"w": bt}, [{"w": e} for e in ets], F.FusionConfig(**cfgkw), exact_merge=exact)
        outs.append(o["w"].clone())
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    ref, _ = OF.fuse(base, experts, **cfgkw)
    got = outs[0].view(torch.int16).cpu().numpy().view(np.uint16)
    assert int((got != rne_bf16_bits(ref)).sum()) == 0
    near = np.abs(ref - p2 * (1 - 2.0 ** -9)) < 2.0 ** -14 * p2
    assert near.sum() > n // 4  # the construction really lands on the boundary


def test_fast_path_overflow_falls_back(cuda):
    """Deltas beyond the f32 range (|e - b| > 3.4e38) make the f32 merge produce inf, or NaN through a
    zero weight times an infinite delta, and finite deltas can still overflow the weighted sums; with
    or without the erase vote the fast path must send those elements to the exact f64 path (the
    reference never overflows in float64)."""
    from paper_2509_18883_b200 import fusion as F
    g = np.random.default_rng(8)
    n = 1 << 18
    # magnitudes from 1e29 (finite f32 deltas whose weighted sums overflow in the scaled fast path)
    # to 2.5e38 (deltas beyond the f32 range)
    base = bf16_round(g.choice([-1.0, 1.0], n) * 10.0 ** g.uniform(29.0, 38.4, n))
    experts = [bf16_round(-base * g.uniform(0.5, 1.0, n)), bf16_round(-base * 0.9), bf16_round(base * 0.5)]
    small = g.random(n) < 0.5  # half the columns stay in range
    for e in experts:
        e[small] = bf16_round(base[small] * 1.01)
    bt = torch.from_numpy(base).to(cuda, torch.bfloat16)
    ets = [torch.from_numpy(e).to(cuda, torch.bfloat16) for e in experts]
    for cfgkw in (dict(target_norm=None, erase_mode=False, merge_weights=(1.0, 0.0, 0.0)),
                  dict(target_norm=None, erase_mode=False, merge_weights=(0.5, 0.3, 0.2)),
                  dict(target_norm=None), dict(target_norm=None, merge_weights=(0.5, 0.3, 0.2)),
                  dict(target_norm=None, erase_weighting="squared"), dict(dropout_p=0.5, seed=3)):
        outs = []
        for exact in (False, True):
            o, _ = F.fuse_state_dict({"w": bt}, [{"w": e} for e in ets], F.FusionConfig(**cfgkw),
                                     exact_merge=exact)
            outs.append(o["w"].clone())
        assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16)), cfgkw
        ref, _ = OF.fuse(base, experts, **cfgkw)
        got = outs[0].view(torch.int16).cpu().numpy().view(np.uint16)
        assert int((got != rne_bf16_bits(ref)).sum()) == 0, cfgkw


F32_CASES = [
    (2, dict()), (4, dict()), (2, dict(dropout_p=0.5, seed=1)), (4, dict(dropout_p=0.75, seed=9)),
    (3, dict(dropout_p=0.75, seed=5, erase_weighting="squared")), (4, dict(dropout_p=0.2, seed=3, erase_mode=False)),
    (2, dict(dropout_p=0.5, seed=8, target_norm=None, erase_mode=False)),
    (4, dict(dropout_p=0.5, seed=2, target_norm=2.0, merge_weights=(0.4, 0.3, 0.2, 0.1))),
    (3, dict(dropout_p=0.6, seed=4, erase_weighting="squared", merge_weights=(0.5, 0.375, 0.125))),
]


@pytest.mark.parametrize("n,cfgkw", F32_CASES)
def test_f32_specialised_merge_vs_oracle(cuda, n, cfgkw):
    """f32 checkpoints run the compile-time-mode K3 (k_merge<f32, f32, N, SPEC>; with keep_prob a power of
    two the dropout rescale is folded into the scale): bit-identical to the reference-order f64 result
    rounded to f32, and to the generic kernel (exact_merge), for 2-4 experts and every mode."""
    from paper_2509_18883_b200 import fusion as F
    rnd = lambda x: np.asarray(x, np.float32).astype(np.float64)
    base, experts = synth_state_dicts(mlp_dict_shapes(8), n, seed=11 + n, dtype_round=rnd)
    # adversarial columns: exact zero deltas, vote ties, a huge and a subnormal-scale delta
    for name in base:
        b = base[name].reshape(-1)
        for i, e in enumerate(experts):
            v = e[name].reshape(-1)
            v[:64] = b[:64]
            v[64:96] = rnd(b[64:96] + (1e-3 if i % 2 == 0 else -1e-3))
            v[96] = rnd(b[96] + 3e4 * (i + 1))
            v[97] = rnd(b[97] + 1e-40)
    to = lambda d: {k: torch.from_numpy(v).to(cuda, torch.float32) for k, v in d.items()}
    cfg = F.FusionConfig(**cfgkw)
    outs, rep = F.fuse_state_dict(to(base), [to(e) for e in experts], cfg)
    outs_x, rep_x = F.fuse_state_dict(to(base), [to(e) for e in experts], cfg, exact_merge=True)
    ref, rstats = _oracle_dict(base, experts, cfgkw)
    for name in base:
        got = outs[name].reshape(-1).cpu().numpy()
        np.testing.assert_array_equal(got, ref[name].astype(np.float32), err_msg=name)
        np.testing.assert_array_equal(got.view(np.uint32), outs_x[name].reshape(-1).cpu().numpy().view(np.uint32))
        st = rep.stats(name)
        assert list(st.erased_counts) == rstats[name]["erased"] == list(rep_x.stats(name).erased_counts), name
        assert list(st.dropout_kept_fraction) == rstats[name]["kept"], name


def test_empty_tables_match_reference(cuda):
    """Zero-size tables behave like the reference (checked against rolloutlab here): the task vector's
    norm is 0, mean normalisation raises its ValueError, and without normalisation the kept fraction
    0/0 raises ZeroDivisionError; in a state dict, empty tensors pass through beside fused ones."""
    from paper_2509_18883_b200 import fusion as F
    b = _pt(np.zeros(0), torch.float64, cuda)
    t = F.task_vector(_pt(np.zeros(0), torch.float64, cuda), b)
    assert t.norm == 0.0
    with pytest.raises(ValueError, match="cannot take mean norm of all-zero task vectors"):
        F.fuse(b, [t, t], F.FusionConfig())
    for cfg in (F.FusionConfig(target_norm=None), F.FusionConfig(dropout_p=0.5, target_norm=1.0)):
        with pytest.raises(ZeroDivisionError):
            F.fuse(b, [t, t], cfg)
    g = np.random.default_rng(4)
    base = {"e0": np.zeros(0), "w": bf16_round(g.normal(0, 0.02, 4096)), "e1": np.zeros((3, 0))}
    experts = [{k: (bf16_round(v + g.normal(0, 1e-3, v.shape)) if v.size else v) for k, v in base.items()}
               for _ in range(3)]
    to = lambda d: {k: torch.from_numpy(np.asarray(v)).to(cuda, torch.bfloat16) for k, v in d.items()}
    outs, rep = F.fuse_state_dict(to(base), [to(e) for e in experts], F.FusionConfig(dropout_p=0.5, seed=1))
    assert outs["e0"].shape == (0,) and outs["e1"].shape == (3, 0)
    ref, _ = OF.fuse(base["w"], [e["w"] for e in experts], dropout_p=0.5, seed=1)
    assert (outs["w"].view(torch.int16).cpu().numpy().view(np.uint16) != rne_bf16_bits(ref)).sum() == 0
