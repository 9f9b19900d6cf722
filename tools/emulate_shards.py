"""Per-rank work of the sharded config-3 fusion, run one rank at a time on ONE GPU (no collectives):
for world = 1, 2, 4, 8 and every rank, the rank's pieces (FusionLayout.partition_striped, or
partition with --contiguous) go through K2 (only the keep-bit ranges the rank reads), K1, finalize
and K3; the partials all-reduce is not timed here.  Prints the slowest rank per world size and the
implied strong-scaling efficiency of the compute."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2509_18883_b200 import _lib as L  # noqa: E402
from paper_2509_18883_b200 import fusion as F  # noqa: E402
from paper_2509_18883_b200.layouts import LAYOUTS, fill_synthetic, numel  # noqa: E402

layout_name = sys.argv[1] if len(sys.argv) > 1 else "llama8b"
STRIPED = "--contiguous" not in sys.argv
shapes = LAYOUTS[layout_name]()
numels = [numel(s) for s in shapes.values()]
layout = F.FusionLayout(numels)
dev = torch.device("cuda", 0)
cfg = F.FusionConfig(dropout_p=0.5, seed=42)
w = (1 / 3,) * 3
s = torch.cuda.Stream()
n_bits = ((max(numels) + 8191) // 8192) * 8192


def time_rank(world, rank, reps=5):
    pieces = []
    with torch.cuda.stream(s):
        for t, lo, hi in (layout.partition_striped if STRIPED else layout.partition)(world, rank):
            n = hi - lo
            b = torch.empty(n, dtype=torch.bfloat16, device=dev)
            es = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(3)]
            fill_synthetic(b, es, t, j0=lo, stream=s)
            pieces.append(F.Piece(t, lo, b, es, torch.empty(n, dtype=torch.bfloat16, device=dev)))
    call = F.FusionCall(pieces, layout, 3, cfg, stream=s)
    call.words_per_row = n_bits // 32
    call._alloc_bitmap()
    seeds = (L.C.c_uint64 * 3)(*call.seeds)
    ranges = F.needed_bit_ranges([(p.j0, p.j0 + p.numel) for p in pieces])  # what the sharded K2 draws
    call._bitmap = lambda *_a, **_k: None  # K2 is the explicit range launches below

    def step():
        with torch.cuda.stream(s):
            call.counters.zero_()
        for lo_b, hi_b in ranges:
            L.call("rlk_fusion_mask_bitmap_range", seeds, 3, call.thresh, lo_b, min(hi_b, n_bits), L.ptr(call.bitmap),
                   call.words_per_row, L.stream_handle(s))
        call.norms().merge(w)  # K1 + finalize + K3 (outputs not checked: timing only)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    params = sum(p.numel for p in pieces)
    del pieces, call
    torch.cuda.empty_cache()
    return ms, params


res = {}
for world in (1, 2, 4, 8):
    per = [time_rank(world, r) for r in range(world)]
    worst = max(m for m, _ in per)
    res[world] = {"rank_ms": [round(m, 3) for m, _ in per], "rank_params": [p for _, p in per],
                  "max_ms": worst}
    base = res[1]["max_ms"]
    print(f"world {world}: per-rank ms {res[world]['rank_ms']}  max {worst:.3f}  "
          f"compute scaling efficiency {base / (world * worst) * 100:.1f}%", flush=True)
print(json.dumps({"layout": layout_name, "results": res}))
