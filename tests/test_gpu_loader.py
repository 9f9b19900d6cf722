"""GPU tests of the K7 streaming loader: host checkpoints fused group-by-group through pinned slots
must equal the all-in-HBM fuse_state_dict bit for bit (and the per-tensor oracle)."""
import numpy as np
import pytest
import torch

from oracle import fusion as OF
from tests.helpers import bf16_round, rne_bf16_bits, synth_state_dicts

pytestmark = pytest.mark.gpu

SHAPES = {"emb": (2000, 333), "w1": (512, 1024), "b1": (1024,), "w2": (1024, 512), "tiny": (7,), "w3": (300, 300)}


def _host_bf16(d):
    return {k: torch.from_numpy(v.astype(np.float32)).to(torch.bfloat16) for k, v in d.items()}


@pytest.mark.parametrize("budget", [16 << 20, 256 << 20])
def test_streaming_equals_in_hbm(cuda, budget):
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.loader import ArraySink, ArraySource, HostLoader, fuse_streaming
    base, experts = synth_state_dicts(SHAPES, 3, seed=7, dtype_round=bf16_round)
    hb, he = _host_bf16(base), [_host_bf16(e) for e in experts]
    cfg = F.FusionConfig(dropout_p=0.5, seed=3)
    out = {k: torch.empty(v.shape, dtype=torch.bfloat16) for k, v in hb.items()}
    names = list(hb)
    ld = HostLoader(slot_bytes=1 << 20, n_slots=3, n_threads=4)
    rep = fuse_streaming(names, [hb[k].numel() for k in names], 3, ArraySource(hb, he), ArraySink(out), cfg,
                         device_budget_bytes=budget, loader=ld)
    ld.close()
    assert rep.groups >= (2 if budget < (32 << 20) else 1)
    dev_out, drep = F.fuse_state_dict({k: v.to(cuda) for k, v in hb.items()},
                                      [{k: v.to(cuda) for k, v in e.items()} for e in he], cfg)
    for k in names:
        assert torch.equal(out[k].view(torch.int16), dev_out[k].cpu().view(torch.int16)), k
        ref, st = OF.fuse(base[k], [e[k] for e in experts], dropout_p=0.5, seed=3)
        assert (out[k].reshape(-1).view(torch.int16).numpy().view(np.uint16) != rne_bf16_bits(ref)).sum() == 0
        assert list(rep.stats[k].erased_counts) == st["erased"]
        assert list(rep.stats[k].dropout_kept_fraction) == st["kept"]


@pytest.mark.parametrize("pinned,budget", [(False, 32 << 20), (True, 32 << 20), (True, 2 << 20)])
def test_streaming_ring_of_workspaces(cuda, pinned, budget):
    """Many small groups through the device ring buffer, pageable or pinned host buffers (the pinned
    path DMAs directly); a 2 MiB ring forces every group to wait for its predecessor's D2H.  Identical
    to the all-in-HBM fuse."""
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.loader import ArraySink, ArraySource, fuse_streaming
    shapes = {f"t{i}": (257 + 64 * i, 129) for i in range(20)}
    base, experts = synth_state_dicts(shapes, 3, seed=17, dtype_round=bf16_round)
    pin = (lambda t: t.pin_memory()) if pinned else (lambda t: t)
    hb = {k: pin(v) for k, v in _host_bf16(base).items()}
    he = [{k: pin(v) for k, v in _host_bf16(e).items()} for e in experts]
    out = {k: pin(torch.empty(v.shape, dtype=torch.bfloat16)) for k, v in hb.items()}
    names = list(hb)
    cfg = F.FusionConfig(dropout_p=0.3, seed=1)
    rep = fuse_streaming(names, [hb[k].numel() for k in names], 3, ArraySource(hb, he), ArraySink(out), cfg,
                         device_budget_bytes=budget, group_bytes=2 << 20)
    assert rep.groups >= 8
    dev_out, drep = F.fuse_state_dict({k: v.to(cuda) for k, v in hb.items()},
                                      [{k: v.to(cuda) for k, v in e.items()} for e in he], cfg)
    for k in names:
        assert torch.equal(out[k].view(torch.int16), dev_out[k].cpu().view(torch.int16)), k
        assert rep.stats[k].erased_counts == drep.stats(k).erased_counts, k


def test_loader_roundtrip_and_checksum(cuda):
    from paper_2509_18883_b200.loader import HostLoader
    ld = HostLoader(slot_bytes=1 << 20, n_slots=4, n_threads=3)
    s = torch.cuda.Stream()
    src = np.random.default_rng(0).integers(0, 2 ** 16, 5_000_003, dtype=np.uint16)
    dst = torch.empty(src.size, dtype=torch.int16, device=cuda)
    ld.h2d(dst, src, s)
    back = np.empty_like(src)
    ld.d2h(back, dst, s)
    assert np.array_equal(back, src)
    # page-locked host buffers take the direct DMA path
    src_p = torch.from_numpy(src.view(np.int16)).pin_memory()
    dst2 = torch.empty_like(dst)
    ld.h2d(dst2, src_p, s)
    back_p = torch.empty_like(src_p).pin_memory()
    ld.d2h(back_p, dst2, s)
    s.synchronize()
    assert np.array_equal(back_p.numpy().view(np.uint16), src)
    x = torch.arange(1 << 20, dtype=torch.int64, device=cuda)
    torch.cuda.synchronize()  # produced on the default stream, read on s
    assert ld.d2h_checksum(x.view(torch.uint8), s) == sum(range(1 << 20))
    # synthesis: deterministic and base-consistent
    a = torch.empty(1 << 20, dtype=torch.bfloat16, device=cuda)
    b = torch.empty_like(a)
    ld.synth_h2d(a, 0, 11, 0.02, 0, 0.0, s)
    ld.synth_h2d(b, 0, 11, 0.02, 0, 0.0, s)
    s.synchronize()
    assert torch.equal(a, b) and 0.015 < float(a.float().std()) < 0.025
    ld.close()


def test_streaming_validates_inputs(cuda, tmp_path):
    """fuse_streaming / cmd_fuse check finalize's per-tensor status after the last group: a non-finite
    input raises the reference's ValueError (and cmd_fuse leaves no output file); a tensor no expert
    changed is written as the base and reported (or raises the reference's mean-norm error on request)."""
    from paper_2509_18883_b200 import checkpoint as CK
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.loader import ArraySink, ArraySource, fuse_streaming
    shapes = {"a": (64, 33), "same": (100,), "c": (50, 7)}
    base, experts = synth_state_dicts(shapes, 3, seed=5, dtype_round=bf16_round)
    for e in experts:
        e["same"] = base["same"].copy()
    hb, he = _host_bf16(base), [_host_bf16(e) for e in experts]
    names = list(hb)
    numels = [hb[k].numel() for k in names]
    out = {k: torch.empty(v.shape, dtype=torch.bfloat16) for k, v in hb.items()}
    rep = fuse_streaming(names, numels, 3, ArraySource(hb, he), ArraySink(out), F.FusionConfig())
    assert rep.passthrough == ["same"]
    assert torch.equal(out["same"].view(torch.int16), hb["same"].view(torch.int16))
    with pytest.raises(ValueError, match="cannot take mean norm of all-zero task vectors"):
        fuse_streaming(names, numels, 3, ArraySource(hb, he), ArraySink(out), F.FusionConfig(), on_unchanged="raise")
    he[1]["c"][3, 4] = float("nan")
    with pytest.raises(ValueError, match="logits must be finite"):
        fuse_streaming(names, numels, 3, ArraySource(hb, he), ArraySink(out), F.FusionConfig())
    # cmd_fuse: same checks before the rename, so no partial output exists
    paths = []
    for i, d in enumerate([hb] + he):
        p = tmp_path / f"in{i}.rlk"
        CK.save(p, d)
        paths.append(p)
    dst = tmp_path / "fused.rlk"
    with pytest.raises(ValueError, match="logits must be finite"):
        CK.cmd_fuse(paths[0], paths[1:], dst, F.FusionConfig())
    assert not dst.exists() and not (tmp_path / "fused.rlk.tmp").exists()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_partitioned_stream_equals_in_hbm(cuda, world):
    """Config-4 sharding: every rank streams its whole-tensor share (`partition_tensors`); the union of
    the ranks' outputs and statistics equals the all-in-HBM fuse bit for bit (norms are per tensor, so
    no collective is involved).  Ranks run one after another on this GPU."""
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.loader import ArraySink, ArraySource, fuse_streaming, partition_tensors
    base, experts = synth_state_dicts(SHAPES, 3, seed=9, dtype_round=bf16_round)
    hb, he = _host_bf16(base), [_host_bf16(e) for e in experts]
    names = list(hb)
    numels = [hb[k].numel() for k in names]
    cfg = F.FusionConfig(dropout_p=0.5, seed=11)
    out = {k: torch.zeros(v.shape, dtype=torch.bfloat16) for k, v in hb.items()}
    stats, seen = {}, []
    for r in range(world):
        rep = fuse_streaming(names, numels, 3, ArraySource(hb, he), ArraySink(out), cfg, device_budget_bytes=16 << 20,
                             world=world, rank=r)
        mine = [names[t] for t in partition_tensors(numels, world, r)]
        assert sorted(rep.stats) == sorted(mine) and rep.tensors == len(mine)
        stats.update(rep.stats)
        seen += mine
    assert sorted(seen) == sorted(names)
    dev_out, drep = F.fuse_state_dict({k: v.to(cuda) for k, v in hb.items()},
                                      [{k: v.to(cuda) for k, v in e.items()} for e in he], cfg)
    for k in names:
        assert torch.equal(out[k].view(torch.int16), dev_out[k].cpu().view(torch.int16)), k
        assert stats[k] == drep.stats(k)
