"""A/B timing of library builds for the GRPO kernels (config-5 rows, V = 131072, 65,536 rows per launch).
Usage: python tools/ab_grpo.py [--rounds R] lib_a.so lib_b.so ..."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2509_18883_b200 import _lib as L
from paper_2509_18883_b200 import objective as O
V, R = 131072, 65536
dev = torch.device("cuda", 0)
lg = torch.empty((R, V), dtype=torch.bfloat16, device=dev)
L.call("rlk_synth_normal", L.ptr(lg), 0, lg.numel(), 0, 7, 2.0, None, L.stream_handle())
g = np.random.default_rng(0)
b = O.GRPOBatch.pack(g.integers(0, V, R), g.normal(-12, .3, R), g.normal(-12, .3, R), [0, R // 2, R], [1., -1.],
                     [1, 1], 2, R, device=dev)
res = []
for fn in (O.grpo_forward, O.grpo_forward_backward):
    for _ in range(3):
        fn(lg, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn(lg, b)
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 10)
print("RESULT", *res)
'''


def main():
    argv = sys.argv[1:]
    rounds = 3
    if argv and argv[0] == "--rounds":
        rounds, argv = int(argv[1]), argv[2:]
    out = {lib: [] for lib in argv}
    for r in range(rounds):
        for lib in argv:
            env = dict(os.environ, RLK_LIB_PATH=str(Path(lib).resolve()))
            p = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=env, capture_output=True, text=True)
            line = [x for x in p.stdout.splitlines() if x.startswith("RESULT")]
            if not line:
                print(lib, "FAILED", p.stderr[-1500:], flush=True)
                continue
            fwd, fb = map(float, line[0].split()[1:])
            out[lib].append((fwd, fb))
            print(f"r{r} {Path(lib).name:24s} fwd {fwd:.3f} ms  fwd+bwd {fb:.3f} ms", flush=True)
    for lib, v in out.items():
        if v:
            print(f"{Path(lib).name:24s} fwd min {min(x[0] for x in v):.3f}  fwd+bwd min {min(x[1] for x in v):.3f}")


if __name__ == "__main__":
    main()
