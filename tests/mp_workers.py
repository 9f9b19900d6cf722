"""Worker bodies for the multi-rank tests (importable by spawned processes).

Every rank of a real process group runs the product's sharded path -- `dist.shard_state_dicts` ->
`ShardedFusion.build(..., group).run().stats()`, `GRPOBatch.shard` -> `grpo_forward(..., group)` /
`grpo_forward_backward(..., group)` -- and checks its share against the world-1 result that it
computes itself (same seeded inputs): outputs, norms, scales, FusionStats and J bit for bit.  On a
one-GPU box all ranks share cuda:0 and talk over gloo (it reduces CUDA tensors; NCCL refuses two
ranks on one device).  The same functions run one rank per GPU over NCCL."""
from __future__ import annotations

import os
import sys
import traceback
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def _init(rank: int, world: int, port: int, backend: str):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0 if backend == "gloo" else rank)
    torch.cuda.set_device(dev)
    kw = dict(device_id=dev) if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    return dev, dist.group.WORLD


def fusion_inputs():
    import torch
    from tests.helpers import bf16_round, synth_state_dicts
    from paper_2509_18883_b200.fusion import ITEM
    # a striped embedding-sized tensor, tensors straddling rank boundaries, a short tail tensor
    shapes = {"embed": (64, 5 * ITEM // 64 + 3), "q": (3 * ITEM + 17,), "b": (70001,), "k": (ITEM,), "n": (5,)}
    base, experts = synth_state_dicts(shapes, 3, seed=11, dtype_round=bf16_round)
    to = lambda d: {k: torch.from_numpy(v).to(torch.bfloat16) for k, v in d.items()}
    return to(base), [to(e) for e in experts]


def fusion_worker(rank: int, world: int, port: int, backend: str, cfgkw: dict):
    import torch
    import torch.distributed as dist
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.dist import ShardedFusion, shard_state_dicts
    dev, group = _init(rank, world, port, backend)
    try:
        base, experts = fusion_inputs()
        cfg = F.FusionConfig(**cfgkw)
        names, layout, pieces = shard_state_dicts(base, experts, world, rank)
        sf = ShardedFusion.build(names, layout, pieces, 3, cfg, group=group).run()
        stats = sf.stats()
        torch.cuda.synchronize()
        ref, rep = F.fuse_state_dict({k: v.to(dev) for k, v in base.items()},
                                     [{k: v.to(dev) for k, v in e.items()} for e in experts], cfg)
        n_mine = 0
        for p in pieces:
            want = ref[names[p.tensor]].reshape(-1)[p.j0:p.j0 + p.numel]
            assert torch.equal(p.out.view(torch.int16), want.view(torch.int16)), (rank, names[p.tensor], p.j0)
            n_mine += p.numel
        held = sf.call.held  # norms of every tensor this rank holds (others are never normalised here)
        assert torch.equal(sf.call.sumsq[held], rep.call.sumsq[held])
        assert torch.equal(sf.call.scale[held], rep.call.scale[held])
        for name in names:
            assert stats[name] == rep.stats(name), (rank, name)
        # every element is owned by exactly one rank
        tot = torch.tensor([n_mine], dtype=torch.int64, device=dev)
        dist.all_reduce(tot, group=group)
        assert int(tot) == sum(v.numel() for v in base.values())
    except Exception:
        traceback.print_exc()
        raise
    finally:
        dist.destroy_process_group()


def grpo_inputs(dev):
    import numpy as np
    import torch
    from paper_2509_18883_b200 import objective as O
    V, G, n_groups = 4096, 4, 3
    g = np.random.default_rng(17)
    lens = g.integers(5, 40, G * n_groups)
    lens[5] = 0  # an empty response
    cu = np.concatenate([[0], np.cumsum(lens)])
    R = int(cu[-1])
    logits = (torch.from_numpy(g.normal(0, 2.0, (R, V))).to(dev)).to(torch.bfloat16)
    toks = g.integers(0, V, R)
    lt = g.normal(-8.0, 0.3, R)
    li = lt + g.normal(0, 0.05, R)
    adv = g.normal(0, 1, G * n_groups)
    use = (g.random(G * n_groups) > 0.15).astype(np.uint8)
    b = O.GRPOBatch.pack(toks, lt, li, cu, adv, use, G, int(lens.max()), temperature=0.8, device=dev)
    return logits, b


def grpo_worker(rank: int, world: int, port: int, backend: str):
    import torch
    import torch.distributed as dist
    from paper_2509_18883_b200 import objective as O
    dev, group = _init(rank, world, port, backend)
    try:
        logits, full = grpo_inputs(dev)
        ref = O.grpo_forward(logits, full)
        ref_fb, ref_grad = O.grpo_forward_backward(logits, full)
        local = full.shard(world, rank)
        r0 = full.sample_rows_host[full.shard_bounds(world)[rank]]
        rows = slice(r0, r0 + local.n_rows)
        lg = logits[rows].contiguous()
        got = O.grpo_forward(lg, local, group=group)
        got_fb, grad = O.grpo_forward_backward(lg, local, group=group)
        torch.cuda.synchronize()
        assert torch.equal(got.objective, ref.objective), (rank, float(got.objective), float(ref.objective))
        assert torch.equal(got_fb.objective, ref_fb.objective), rank
        assert torch.equal(got.group_sums, ref.group_sums)
        for k in ("logp", "lse", "term", "coef"):
            assert torch.equal(getattr(got, k), getattr(ref, k)[rows]), (rank, k)
        assert torch.equal(grad.view(torch.int16), ref_grad[rows].view(torch.int16)), rank
    except Exception:
        traceback.print_exc()
        raise
    finally:
        dist.destroy_process_group()


def stream_worker(rank: int, world: int, port: int, backend: str):
    """fuse_streaming(group=...): each rank streams its tensors; the gathered statistics on every rank
    equal the all-in-HBM fuse's, and each rank's outputs match it bit for bit."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.loader import ArraySink, ArraySource, fuse_streaming, partition_tensors
    from tests.helpers import bf16_round, synth_state_dicts
    dev, group = _init(rank, world, port, backend)
    try:
        shapes = {f"t{i}": (100 + 37 * i, 65) for i in range(9)}
        base, experts = synth_state_dicts(shapes, 3, seed=5, dtype_round=bf16_round)
        hb = {k: torch.from_numpy(v.astype(np.float32)).to(torch.bfloat16) for k, v in base.items()}
        he = [{k: torch.from_numpy(v.astype(np.float32)).to(torch.bfloat16) for k, v in e.items()} for e in experts]
        names = list(hb)
        out = {k: torch.zeros(v.shape, dtype=torch.bfloat16) for k, v in hb.items()}
        cfg = F.FusionConfig(dropout_p=0.5, seed=2)
        rep = fuse_streaming(names, [hb[k].numel() for k in names], 3, ArraySource(hb, he), ArraySink(out), cfg,
                             device_budget_bytes=4 << 20, group=group)
        ref, rrep = F.fuse_state_dict({k: v.to(dev) for k, v in hb.items()},
                                      [{k: v.to(dev) for k, v in e.items()} for e in he], cfg)
        assert sorted(rep.stats) == sorted(names)
        for k in names:
            assert rep.stats[k] == rrep.stats(k), (rank, k)
        for t in partition_tensors([hb[k].numel() for k in names], world, rank):
            k = names[t]
            assert torch.equal(out[k].view(torch.int16), ref[k].cpu().view(torch.int16)), (rank, k)
    except Exception:
        traceback.print_exc()
        raise
    finally:
        dist.destroy_process_group()
