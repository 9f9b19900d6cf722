"""Profiling driver for the fused GRPO kernel (8192 rows, V = 131072)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2509_18883_b200 import _lib as L
from paper_2509_18883_b200 import objective as O
V, R = 131072, 8192
dev = torch.device("cuda", 0)
lg = torch.empty((R, V), dtype=torch.bfloat16, device=dev)
L.call("rlk_synth_normal", L.ptr(lg), 0, lg.numel(), 0, 7, 2.0, None, L.stream_handle())
g = np.random.default_rng(0)
b = O.GRPOBatch.pack(g.integers(0, V, R), g.normal(-12, .3, R), g.normal(-12, .3, R), [0, R // 2, R], [1., -1.],
                     [1, 1], 2, R, device=dev)
for _ in range(3):
    O.grpo_forward(lg, b)
    O.grpo_forward_backward(lg, b)
torch.cuda.synchronize()
print("ok")
