"""Small launches of every async kernel for compute-sanitizer (tools/sanitize.sh, tests/test_gpu_sanitizer.py).

Covers the mbarrier/TMA rings and the cross-CTA exchange: K1 (bf16 fast kernel and the generic f32
kernel), K2 (whole rows and sharded index ranges), finalize, K3 (certified bf16 fast path incl. its
phase-2 recompute, and the reference-order f64 path), K4a/K4b (split forward), K4 (single kernel),
K5 (bf16 / f32 / f64 gradients, CSR rows) and the 2-CTA-cluster fused GRPO kernel.  Sizes are a few
items so racecheck finishes in seconds."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_18883_b200 import _lib as L  # noqa: E402
from paper_2509_18883_b200 import fusion as F  # noqa: E402
from paper_2509_18883_b200 import objective as O  # noqa: E402
from paper_2509_18883_b200.core import fusion_child_seeds, keep_threshold  # noqa: E402
from paper_2509_18883_b200.fusion import ITEM  # noqa: E402


def fusion_cases(dev):
    g = torch.Generator(device=dev).manual_seed(3)
    shapes = {"a": (2 * ITEM + 4099,), "b": (777,), "c": (ITEM,)}
    for dt in (torch.bfloat16, torch.float32):
        base = {k: (torch.randn(s, device=dev, generator=g) * 0.02).to(dt) for k, s in shapes.items()}
        exps = [{k: (v.float() + torch.randn(v.shape, device=dev, generator=g) * 1e-3 * (i + 1)).to(dt)
                 for k, v in base.items()} for i in range(3)]
        # near-ties so the fast path's phase 2 runs
        for k in base:
            d0 = exps[0][k].float() - base[k].float()
            exps[2][k][::5] = (base[k].float() - d0)[::5].to(dt)
        for cfg in (F.FusionConfig(dropout_p=0.5, seed=1), F.FusionConfig(erase_weighting="squared"),
                    F.FusionConfig(target_norm=None, erase_mode=False)):
            for exact in (False, True):
                F.fuse_state_dict(base, exps, cfg, exact_merge=exact)
    # sharded K2 ranges (FusionCall with an explicit partition of two 'ranks' on this device)
    names = list(shapes)
    layout = F.FusionLayout([int(np.prod(shapes[k])) for k in names])
    seeds = (L.C.c_uint64 * 3)(*fusion_child_seeds(5, 3))
    words = ((max(layout.numels) + 8191) // 8192) * 8192 // 32
    bm = torch.zeros(3 * words, dtype=torch.int32, device=dev)
    L.call("rlk_fusion_mask_bitmap_range", seeds, 3, keep_threshold(0.5), ITEM // 2, ITEM + 8192 * 3, L.ptr(bm),
           words, L.stream_handle())
    torch.cuda.synchronize()


def grpo_cases(dev):
    V, R = 16384, 6
    g = np.random.default_rng(0)
    for dt in (torch.bfloat16, torch.float32, torch.float64):
        logits = (torch.randn((R, V), device=dev) * 2).to(dt)
        b = O.GRPOBatch.pack(g.integers(0, V, R), g.normal(-9, .3, R), g.normal(-9, .3, R), [0, 2, 4, 6],
                             [1.0, -1.0, 0.5], [1, 1, 1], 3, 2, device=dev)
        fwd = O.grpo_forward(logits, b)  # K4a/K4b (bf16/f32), K4 (f64)
        for gd in (torch.bfloat16, torch.float32, torch.float64):
            O.grpo_backward(logits, b, fwd, grad_dtype=gd)  # K5
        if dt == torch.bfloat16:
            O.grpo_forward_backward(logits, b)  # fused 2-CTA cluster kernel
            # K4 single-kernel path (no workspace)
            f64 = dict(dtype=torch.float64, device=dev)
            logp, lse, term, coef = (torch.empty(R, **f64) for _ in range(4))
            flags = torch.zeros(1, dtype=torch.int32, device=dev)
            c = O.ClipConfig().c_struct()
            L.call("rlk_grpo_fwd", L.ptr(logits), L.dtype_code(dt), R, V, V, None, L.ptr(b.tokens),
                   L.ptr(b.logp_train), L.ptr(b.logp_infer), L.ptr(b.sample_of_row), L.ptr(b.adv), L.ptr(b.use),
                   L.ptr(b.temperature), L.ptr(b.norm), L.C.byref(c), L.ptr(logp), L.ptr(lse), L.ptr(term),
                   L.ptr(coef), L.ptr(flags), None, 0, L.stream_handle())
    # tabular policy rows (row_index, CSR gradient with shared rows)
    logits = torch.randn((8, V), device=dev, dtype=torch.float64)
    b = O.GRPOBatch.pack([1, 2, 3, 4], [-9.0] * 4, [-9.0] * 4, [0, 2, 4], [1.0, -1.0], [1, 1], 2, 2, device=dev,
                         row_index=[0, 3, 3, 5])
    fwd = O.grpo_forward(logits, b)
    O.grpo_backward(logits, b, fwd)
    torch.cuda.synchronize()


if __name__ == "__main__":
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "fusion"):
        fusion_cases(dev)
    if which in ("all", "grpo"):
        grpo_cases(dev)
    print("sanitize driver ok")
