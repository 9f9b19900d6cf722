"""rolloutlab-b200: B200-native (sm_100a) hot path of arXiv 2509.18883 (LongCat-Flash-Thinking).

Drop-in replacements for the reference's `rolloutlab.fusion` and `rolloutlab.objective` (plus the
`ParamTable` / `log_token_dist` pieces of `rolloutlab.toy_env` and the RNG of `rolloutlab.core`),
computing on the GPU through the C ABI in include/rlk.h (`_rlk.so`).  There is no CPU fallback.
"""
from . import core, fusion, objective, toy_env  # noqa: F401
from ._lib import LIB_PATH, lib  # noqa: F401

__all__ = ["core", "fusion", "objective", "toy_env", "lib", "LIB_PATH"]
