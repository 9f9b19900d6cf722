"""The C-ABI library loads without a GPU and exports every entry point include/rlk.h declares."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    syms = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        syms |= set(re.findall(r"\b(rlk_[a-z0-9_]+)\s*\(", text))
    return sorted(syms)


def test_header_declares_hot_path():
    syms = declared_symbols()
    for s in ["rlk_fusion_sumsq", "rlk_fusion_finalize", "rlk_fusion_mask_bitmap", "rlk_fusion_mask_bitmap_range", "rlk_fusion_merge",
              "rlk_grpo_fwd", "rlk_grpo_bwd", "rlk_last_error"]:
        assert s in syms


def test_library_exports_all_declared_symbols():
    from paper_2509_18883_b200 import _lib
    if not _lib.LIB_PATH.exists():
        from paper_2509_18883_b200._build import build
        build()
    handle = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(handle, s)]
    assert not missing, missing
    assert handle.rlk_abi_version() == 2
    # every declared symbol has a ctypes signature in the binding
    assert not [s for s in declared_symbols() if s not in _lib.SIGNATURES]


def test_invalid_arguments_map_to_value_error():
    from paper_2509_18883_b200 import _lib as L
    L.lib()
    with pytest.raises(ValueError, match="expert count"):
        L.call("rlk_fusion_sumsq", ctypes.byref(L.FusionPlanC(0, 0, 0, 1)), 9, 0, 0, 8, None, 0, None, 0, None, 0, None)
    with pytest.raises(ValueError, match="bad dtype"):
        L.call("rlk_nonfinite_count", 8, 7, 1, 8, None)


def test_more_argument_checks_before_any_device_work():
    """Validation happens on the host before any CUDA call, with the reference-style message."""
    from paper_2509_18883_b200 import _lib as L
    L.lib()
    seeds = (ctypes.c_uint64 * 3)(1, 2, 3)
    with pytest.raises(ValueError, match="bad bit range"):
        L.call("rlk_fusion_mask_bitmap_range", seeds, 3, 0, 33, 64, 8, 4, None)
    with pytest.raises(ValueError, match="row too short"):
        L.call("rlk_fusion_mask_bitmap_range", seeds, 3, 0, 0, 1 << 20, 8, 4, None)
    plan = ctypes.byref(L.FusionPlanC(8, 8, 1, 1))
    w = (ctypes.c_double * 3)(1 / 3, 1 / 3, 1 / 3)
    with pytest.raises(ValueError, match="bad erase mode"):
        L.call("rlk_fusion_merge", plan, 3, 0, 0, 0, 8, w, 0, None, 0, 1.0, None, 0, 5, 8, 0, None)
    with pytest.raises(ValueError, match="bad dropout mode"):
        L.call("rlk_fusion_merge", plan, 3, 0, 0, 0, 8, w, 7, seeds, 0, 1.0, None, 0, 1, 8, 0, None)
    clip = L.ClipC(0.2, 0.2, 3.0, 2.0, 1)
    with pytest.raises(ValueError, match="bad dtype"):
        L.call("rlk_grpo_fwd", 8, 9, 4, 16, 16, None, 8, 8, 8, 8, 8, 8, 8, 8, ctypes.byref(clip), None, None, 8, 8, 8,
               None, 0, None)
    with pytest.raises(ValueError, match="multiple of 16"):
        L.call("rlk_grpo_fused_bf16", 16, 4, 100, 100, None, 16, 8, 8, 8, 8, 8, 8, 8, ctypes.byref(clip), 1.0, None,
               None, 8, 8, 8, 16, 100, None)


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: with the sm_100a library absent, the first kernel call raises RlkError."""
    import os
    import subprocess
    import sys
    code = ("from paper_2509_18883_b200 import _lib as L\n"
            "try:\n    L.lib()\nexcept L.RlkError as e:\n    print('RAISED', e)\n")
    env = dict(os.environ, RLK_LIB_PATH=str(tmp_path / "absent.so"), RLK_AUTOBUILD="0")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, env=env, timeout=300)
    assert "RAISED" in out.stdout and "no CPU fallback" in out.stdout, out.stdout + out.stderr


def test_integration_ctypes_stub_binds():
    """The ctypes stub INTEGRATION.md shows a maintainer binds every symbol it names (no GPU calls)."""
    import re
    from paper_2509_18883_b200 import _lib
    if not _lib.LIB_PATH.exists():
        from paper_2509_18883_b200._build import build
        build()
    text = (ROOT / "INTEGRATION.md").read_text()
    stub = next(b for b in re.findall(r"```python\n(.*?)```", text, re.S) if "C.CDLL" in b)
    stub = stub.replace('"paper_2509_18883_b200/_rlk.so"', repr(str(_lib.LIB_PATH)))
    exec(compile(stub, "INTEGRATION.md", "exec"), {})
