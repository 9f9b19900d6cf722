"""Per-kernel times of one FusionConfig on a layout (CUDA events around each launch):
    python tools/prof_variant.py --layout llama8b --cfg '{"dropout_p": 0.5, "seed": 42, "target_norm": null}'"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2509_18883_b200 import fusion as F  # noqa: E402
from paper_2509_18883_b200.layouts import LAYOUTS, fill_synthetic, numel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layout", default="llama8b")
ap.add_argument("--cfg", action="append", default=[])
ap.add_argument("--runs", type=int, default=5)
ap.add_argument("--no-fixup", action="store_true", help="exact path inside the merge (no fix-up queue)")
a = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = LAYOUTS[a.layout]()
layout = F.FusionLayout([numel(s) for s in shapes.values()])
pieces = []
for t, n in enumerate(layout.numels):
    b = torch.empty(n, dtype=torch.bfloat16, device=dev)
    es = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(3)]
    fill_synthetic(b, es, t)
    pieces.append(F.Piece(t, 0, b, es, torch.empty(n, dtype=torch.bfloat16, device=dev)))
for cj in a.cfg or ['{"dropout_p": 0.5, "seed": 42}']:
    kw = json.loads(cj)
    cfg = F.FusionConfig(**kw)
    call = F.FusionCall(pieces, layout, 3, cfg, fixup=not a.no_fixup)
    w = cfg.merge_weights or (1 / 3, 1 / 3, 1 / 3)
    call.run(w)
    call.timers = {}
    for _ in range(a.runs):
        call.run(w)
    torch.cuda.synchronize()
    ws = getattr(call, "_ws", None)
    queued = int(ws[:4096].view(torch.int32).sum()) if ws is not None else None  # fix-up queue lengths
    print(kw, {k.replace("rlk_fusion_", ""): round(statistics.mean(x.elapsed_time(y) for x, y in v), 3)
               for k, v in call.timers.items()}, "fix-up queued", queued)
