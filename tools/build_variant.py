"""Build an experimental variant of the library with extra nvcc flags into tools/var/ (A/B timing with
tools/ab_fusion.py).  Usage: python tools/build_variant.py NAME [-DFOO=1 ...]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2509_18883_b200 import _build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
B.NVCC_FLAGS = B.NVCC_FLAGS + flags
B.BUILD = ROOT / "build" / ("var_" + name)
B.LIB = ROOT / "tools" / "var" / f"_rlk_{name}.so"
B.LIB.parent.mkdir(parents=True, exist_ok=True)
print(B.build(force=True, checked=False))
