"""Host-side timeline of one fuse_streaming call on the config-3 layout from pinned host memory
(where the e2e step spends its wall time)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2509_18883_b200 import fusion as F  # noqa: E402
from paper_2509_18883_b200 import loader as LD  # noqa: E402
from paper_2509_18883_b200.layouts import LAYOUTS, numel  # noqa: E402

shapes = LAYOUTS[sys.argv[1] if len(sys.argv) > 1 else "llama8b"]()
names = list(shapes)
numels = [numel(s) for s in shapes.values()]
total = sum(numels)
hb_flat = [torch.empty(total, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
ho_flat = torch.empty(total, dtype=torch.bfloat16, pin_memory=True)
for h in hb_flat:
    h.view(torch.int16).random_(-1000, 1000)
views, off = {}, 0
hb, he, ho = {}, [{}, {}, {}], {}
for n, k in zip(numels, names):
    hb[k] = hb_flat[0][off:off + n]
    for i in range(3):
        he[i][k] = hb_flat[i + 1][off:off + n]
    ho[k] = ho_flat[off:off + n]
    off += n
cfg = F.FusionConfig(dropout_p=0.5, seed=42)

T = {}
orig = {"fill": LD.ArraySource.fill, "drain": LD.ArraySink.drain, "run": F.FusionCall.run,
        "host_tables": F.FusionCall.host_tables, "init": F.FusionCall.__init__}


def wrap(name, cls, attr):
    f = orig[name]

    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return r
    setattr(cls, attr, g)


wrap("fill", LD.ArraySource, "fill")
wrap("drain", LD.ArraySink, "drain")
wrap("run", F.FusionCall, "run")
wrap("host_tables", F.FusionCall, "host_tables")
wrap("init", F.FusionCall, "__init__")
sync0 = torch.cuda.synchronize


def sync(*a):
    t0 = time.perf_counter()
    sync0(*a)
    T["sync"] = T.get("sync", 0.0) + time.perf_counter() - t0


for it in range(3):
    T.clear()
    torch.cuda.synchronize = sync
    t0 = time.perf_counter()
    rep = LD.fuse_streaming(names, numels, 3, LD.ArraySource(hb, he), LD.ArraySink(ho), cfg,
                            device_budget_bytes=16 << 30, group_bytes=2 << 30)
    wall = time.perf_counter() - t0
    torch.cuda.synchronize = sync0
    print(f"iter {it}: wall {wall * 1e3:.1f} ms, groups {rep.groups}, " +
          ", ".join(f"{k} {v * 1e3:.1f}" for k, v in T.items()), flush=True)
