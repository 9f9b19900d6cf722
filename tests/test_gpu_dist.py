"""The sharded fusion path through a real NCCL process group (world size 1 on a one-GPU box; the
multi-rank host logic is covered by tests/test_dist_cpu.py over gloo)."""
import os
import socket

import numpy as np
import pytest
import torch

from tests.helpers import bf16_round, synth_state_dicts

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_fusion_over_nccl(cuda):
    import torch.distributed as dist
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.dist import ShardedFusion, shard_state_dicts
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        base, experts = synth_state_dicts({"a": (300, 700), "b": (70001,)}, 3, seed=5, dtype_round=bf16_round)
        to = lambda d: {k: torch.from_numpy(v).to(torch.bfloat16) for k, v in d.items()}
        cfg = F.FusionConfig(dropout_p=0.5, seed=8)
        names, layout, pieces = shard_state_dicts(to(base), [to(e) for e in experts], 1, 0)
        sf = ShardedFusion.build(names, layout, pieces, 3, cfg, group=dist.group.WORLD).run()
        stats = sf.stats()
        ref, rep = F.fuse_state_dict({k: v.cuda() for k, v in to(base).items()},
                                     [{k: v.cuda() for k, v in to(e).items()} for e in experts], cfg)
        for t, name in enumerate(names):
            got = torch.cat([p.out for p in pieces if p.tensor == t])
            assert torch.equal(got.view(torch.int16), ref[name].reshape(-1).view(torch.int16))
            assert stats[name] == rep.stats(name)
    finally:
        dist.destroy_process_group()
