"""Build the sm_100a C-ABI library (`_rlk.so`) and the host streaming loader in-tree with nvcc/g++.

Each translation unit is compiled in parallel (`-gencode arch=compute_100a,code=sm_100a -lineinfo`);
the CUDA runtime is linked statically so the library does not depend on the runtime torch ships.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "_rlk.so"
BUILD = PKG.parent / "build"

CU_SOURCES = ["capi.cu", "fusion.cu", "grpo.cu", "grpo_fused.cu"]
CPP_SOURCES = ["loader.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills", "-diag-suppress", "177",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the rolloutlab B200 kernels cannot be built")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


LIB_CHECKED = PKG / "_rlk_checked.so"


def build(force: bool = False, verbose: bool = False, checked: bool = True) -> Path:
    """Compile every kernel TU and link `_rlk.so` (and the RLK_CHECKED assert build `_rlk_checked.so`
    that tests/test_gpu_checked.py runs the GPU suite against); returns the release library's path.
    Incremental unless force."""
    lib = _build_one(LIB, BUILD, [], force, verbose)
    if checked:
        _build_one(LIB_CHECKED, BUILD / "checked", ["-DRLK_CHECKED"], force, verbose)
    return lib


def _build_one(LIB: Path, BUILD: Path, extra: list, force: bool, verbose: bool) -> Path:
    nvcc = _nvcc()
    BUILD.mkdir(parents=True, exist_ok=True)
    headers = sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [INCLUDE / "rlk.h"]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        obj = BUILD / (src + ".o")
        objs.append(obj)
        if force or _stale(obj, [CSRC / src] + headers):
            jobs.append([nvcc, *NVCC_FLAGS, *extra, "-I", str(INCLUDE), "-c", str(CSRC / src), "-o", str(obj)])
    for src in CPP_SOURCES:
        if not (CSRC / src).exists():
            continue
        obj = BUILD / (src + ".o")
        objs.append(obj)
        if force or _stale(obj, [CSRC / src] + headers):
            jobs.append([nvcc, "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-pthread", "-I", str(INCLUDE),
                         "-c", str(CSRC / src), "-o", str(obj)])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr)
        return r

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIB, objs):
        tmp = LIB.with_suffix(".so.tmp")
        run([nvcc, "-shared", "-Wno-deprecated-gpu-targets", "-cudart", "static", "-Xcompiler", "-pthread", *map(str, objs), "-o", str(tmp)])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose=True))
