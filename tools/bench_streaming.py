"""Config 4 (BASELINE.json configs[3]): LongCat-Flash-560B-MoE-shaped random-init experts, fused by
streaming layer slices through pinned host buffers (K7).  Host threads synthesise base + 3 experts
per slice (counter hash, loader.cpp) straight into pinned slots; the fused output is checksummed on
the host (outputs larger than RAM).  On one GPU this runs a bounded number of layers and reports
rates; the full model is sharded by parameter range over 8 GPUs (dist.py), i.e. 1/8 per GPU.

    python tools/bench_streaming.py --layers 1 [--source synth|replay]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2509_18883_b200 import fusion as F
from paper_2509_18883_b200.layouts import longcat_560b, numel
from paper_2509_18883_b200.loader import ArraySource, ChecksumSink, HostLoader, SyntheticSource, fuse_streaming


class ReplaySource:
    """Pageable host memory (like a checkpoint in the page cache): slices of one 4 GiB random pool."""

    def __init__(self, n_streams=4, pool_elems=1 << 31, pinned=False):
        g = np.random.default_rng(0)
        self.pool = (g.standard_normal(pool_elems // 8, dtype=np.float32) * 0.02).astype(np.float32)
        self.pool = np.tile(self.pool.view(np.uint32) >> 16, 8).astype(np.uint16)
        if pinned:  # page-locked: the loader DMAs straight from it
            self._pinned = torch.from_numpy(self.pool.view(np.int16)).pin_memory()
            self.pool = self._pinned.numpy().view(np.uint16)
        self.n = pool_elems

    def fill(self, loader, name, si, dst, stream):
        n = dst.numel()
        off = (hash((name, si)) % (self.n - n)) & ~7
        loader.h2d(dst, self.pool[off:off + n], stream)


ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=1)
ap.add_argument("--source", choices=["synth", "replay", "pinned"], default="replay")
ap.add_argument("--budget-gb", type=float, default=48)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--group-gb", type=float, default=2.0)
ap.add_argument("--json-out", default=None)
a = ap.parse_args()
shapes = longcat_560b(n_layers=a.layers)
names = list(shapes)
numels = [numel(s) for s in shapes.values()]
total = sum(numels)
full = sum(numel(s) for s in longcat_560b().values())
src = SyntheticSource() if a.source == "synth" else ReplaySource(pinned=a.source == "pinned")
sink = ChecksumSink()
ld = HostLoader(slot_bytes=64 << 20, n_slots=6, n_threads=a.threads)
cfg = F.FusionConfig(dropout_p=0.5, seed=42)
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = fuse_streaming(names, numels, 3, src, sink, cfg, device_budget_bytes=int(a.budget_gb * (1 << 30)), stats=False,
                     loader=ld, group_bytes=int(a.group_gb * (1 << 30)))
dt = time.perf_counter() - t0
ld.close()
res = {"workload": f"config4 slice: longcat560b layout, {a.layers} layer(s) + embeddings/head, 3 experts + base, "
                   f"bf16, FusionConfig(dropout_p=0.5, seed=42), source={a.source}",
       "params": total, "full_model_params": full, "seconds": dt, "params_per_s": total / dt,
       "h2d_gbs": rep.h2d_bytes / dt / 1e9, "d2h_gbs": rep.d2h_bytes / dt / 1e9, "groups": rep.groups, "group_gb": a.group_gb,
       "projected_full_model_8gpu_s": full / 8 / (total / dt)}
print(json.dumps(res))
if a.json_out:
    Path(a.json_out).write_text(json.dumps(res, indent=1))
