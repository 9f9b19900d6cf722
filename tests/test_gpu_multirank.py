"""The sharded product path through REAL multi-rank process groups.

2 and 4 processes share cuda:0 and talk over gloo, which reduces CUDA tensors (NCCL refuses two
ranks on one GPU).  Each rank runs `ShardedFusion` / `grpo_forward(group=...)` on its own share
and checks it bit for bit against the world-1 result (tests/mp_workers.py)."""
import socket

import pytest
import torch.multiprocessing as mp

from tests import mp_workers as W

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("cfgkw", [dict(dropout_p=0.5, seed=8), dict(erase_weighting="squared", target_norm=0.5)],
                         ids=["p05", "sq_t05"])
def test_sharded_fusion_multirank(cuda, world, cfgkw):
    mp.spawn(W.fusion_worker, args=(world, _port(), "gloo", cfgkw), nprocs=world, join=True)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_grpo_multirank(cuda, world):
    mp.spawn(W.grpo_worker, args=(world, _port(), "gloo"), nprocs=world, join=True)


def test_streamed_fusion_multirank(cuda):
    mp.spawn(W.stream_worker, args=(2, _port(), "gloo"), nprocs=2, join=True)
