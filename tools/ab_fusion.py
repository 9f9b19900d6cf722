"""A/B timing of library builds on one box: runs the quick fusion bench once per (round, library),
interleaved, and prints ms/step and per-kernel times.  Usage:
  python tools/ab_fusion.py --rounds 3 lib_a.so lib_b.so [-- extra bench.py args]
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    argv = sys.argv[1:]
    extra = []
    if "--" in argv:
        i = argv.index("--")
        argv, extra = argv[:i], argv[i + 1:]
    rounds = 3
    if argv and argv[0] == "--rounds":
        rounds, argv = int(argv[1]), argv[2:]
    libs = argv
    res = {lib: [] for lib in libs}
    for r in range(rounds):
        for lib in libs:
            env = dict(os.environ, RLK_LIB_PATH=str(Path(lib).resolve()))
            out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--quick", "--no-e2e", "--no-grpo", "--no-cpu",
                                  "--steps", "20", "--warmup", "3", *extra], env=env, capture_output=True, text=True,
                                 cwd=ROOT)
            line = [x for x in out.stdout.splitlines() if x.startswith("{")]
            if not line:
                print(lib, "FAILED", out.stderr[-2000:], flush=True)
                continue
            d = json.loads(line[-1])
            k = d["roofline"]["kernels_ms"]
            res[lib].append(d["ms_per_step"])
            print(f"r{r} {Path(lib).name:28s} step {d['ms_per_step']:.3f} " +
                  " ".join(f"{n.replace('rlk_fusion_', '')} {v:.3f}" for n, v in k.items()) +
                  f" sm {d['clocks'].get('sm_mhz')}", flush=True)
    for lib, v in res.items():
        if v:
            print(f"{Path(lib).name:28s} min {min(v):.3f} mean {sum(v) / len(v):.3f}")


if __name__ == "__main__":
    main()
