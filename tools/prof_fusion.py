"""Profiling driver: one warm fuse of a layout's state dict (for ncu -k regex:k_merge -s <warm> -c 1)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2509_18883_b200 import fusion as F  # noqa: E402
from paper_2509_18883_b200.layouts import LAYOUTS, fill_synthetic, numel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layout", default="gpt1p3b")
ap.add_argument("--dropout", type=float, default=0.5)
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--grpo", action="store_true")
ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
a = ap.parse_args()
dev = torch.device("cuda", 0)
if a.grpo:
    from paper_2509_18883_b200 import objective as O
    import numpy as np
    V, R = 131072, 8192
    lg = torch.empty((R, V), dtype=torch.bfloat16, device=dev)
    from paper_2509_18883_b200 import _lib as L
    L.call("rlk_synth_normal", L.ptr(lg), 0, lg.numel(), 0, 7, 2.0, None, L.stream_handle())
    g = np.random.default_rng(0)
    b = O.GRPOBatch.pack(g.integers(0, V, R), g.normal(-12, .3, R), g.normal(-12, .3, R), [0, R // 2, R], [1., -1.],
                         [1, 1], 2, R, device=dev)
    for _ in range(a.runs):
        f = O.grpo_forward(lg, b)
        O.grpo_backward(lg, b, f)
    torch.cuda.synchronize()
    sys.exit(0)
shapes = LAYOUTS[a.layout]()
base, experts = {}, [dict() for _ in range(3)]
dt = {"bf16": torch.bfloat16, "f32": torch.float32}[a.dtype]
for t, (k, s) in enumerate(shapes.items()):
    base[k] = torch.empty(s, dtype=dt, device=dev)
    for e in experts:
        e[k] = torch.empty(s, dtype=dt, device=dev)
    fill_synthetic(base[k].view(-1), [e[k].view(-1) for e in experts], t)
cfg = F.FusionConfig(dropout_p=a.dropout, seed=42)
for _ in range(a.runs):
    F.fuse_state_dict(base, experts, cfg)
torch.cuda.synchronize()
print("ok")
