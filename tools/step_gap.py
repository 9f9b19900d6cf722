"""Where the fusion step's time goes between kernels: interleaved rounds of (a) a CUDA-graph replay of
the step, (b) the same step launched eagerly with CUDA events around every C-ABI call and around the
whole step.  (b)'s per-call sum vs its own step time is the host/launch gap of eager launches; (a) vs
(b) in the same round is what the graph saves; the spread over rounds is the clock drift between
measurement passes (bench.py times the headline and the per-kernel split in separate passes)."""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2509_18883_b200 import fusion as F  # noqa: E402
from paper_2509_18883_b200.layouts import LAYOUTS, fill_synthetic, numel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layout", default="llama8b")
ap.add_argument("--rounds", type=int, default=6)
ap.add_argument("--steps", type=int, default=4)
a = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = LAYOUTS[a.layout]()
layout = F.FusionLayout([numel(s) for s in shapes.values()])
stream = torch.cuda.Stream(dev)
pieces = []
with torch.cuda.stream(stream):
    for t, lo, hi in layout.partition_striped(1, 0):
        b = torch.empty(hi - lo, dtype=torch.bfloat16, device=dev)
        es = [torch.empty_like(b) for _ in range(3)]
        fill_synthetic(b, es, t, j0=lo, stream=stream)
        pieces.append(F.Piece(t, lo, b, es, torch.empty_like(b)))
stream.synchronize()
call = F.FusionCall(pieces, layout, 3, F.FusionConfig(dropout_p=0.5, seed=42), stream=stream)
w = (1 / 3,) * 3
for _ in range(2):
    call.run(w)
graph = call.capture(w)


def ev():
    return torch.cuda.Event(enable_timing=True)


rows = []
for r in range(a.rounds):
    # (a) graph replays
    e0, e1 = ev(), ev()
    torch.cuda.synchronize()
    e0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(a.steps):
            graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    g_ms = e0.elapsed_time(e1) / a.steps
    # (b) eager with per-call events
    call.timers = {}
    s0, s1 = ev(), ev()
    s0.record(stream)
    for _ in range(a.steps):
        call.run(w)
    s1.record(stream)
    torch.cuda.synchronize()
    eager_ms = s0.elapsed_time(s1) / a.steps
    kern = {k: sum(x.elapsed_time(y) for x, y in v) / a.steps for k, v in call.timers.items()}
    call.timers = None
    rows.append((g_ms, eager_ms, sum(kern.values()), kern))
    print(f"round {r}: graph {g_ms:7.3f} ms | eager step {eager_ms:7.3f} ms, sum of calls {sum(kern.values()):7.3f} ms "
          + " ".join(f"{k.replace('rlk_fusion_', '')}={v:.3f}" for k, v in kern.items()))
g = [x[0] for x in rows]
e = [x[1] for x in rows]
k = [x[2] for x in rows]
print(f"median: graph {statistics.median(g):.3f} ms, eager {statistics.median(e):.3f} ms, "
      f"sum of calls {statistics.median(k):.3f} ms; graph - calls = {statistics.median(g) - statistics.median(k):+.3f} ms, "
      f"eager - calls = {statistics.median(e) - statistics.median(k):+.3f} ms")
