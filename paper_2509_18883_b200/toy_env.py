"""GPU-resident parameter tables and the per-slot log-softmax (the pieces of the reference
`rolloutlab.toy_env` that sit on the fusion / objective hot path).

* `ParamTable` (reference toy_env.py:61-102): an immutable 3-d table, now a CUDA tensor (bf16, f32 or
  f64; numpy input becomes f64 like the reference).  Construction runs the finite check on the GPU
  (`rlk_nonfinite_count`) and raises ``ValueError("logits must be finite")`` as the reference does.
* `log_token_dist` / `token_dist` (toy_env.py:157-179) and `logprob_trace` (toy_env.py:287-297) on the
  train engine, computed by the sm_100a kernels (`rlk_logsoftmax_rows`, `rlk_grpo_fwd`).
* `detect_repetition` (toy_env.py:315-327): host logic feeding `objective.apply_masks`.

The toy task family, rollout sampling, grading and sequence enumeration are outside the hot path.
`InferEngine` is accepted for API compatibility; its seeded Gaussian perturbation (toy_env.py:144-147)
is host-side simulation of engine drift and is only supported with ``perturb_scale == 0``.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence, Union

import numpy as np
import torch

from . import _lib as L
from .core import Sample, SampleStatus

_FLOAT_DTYPES = (torch.bfloat16, torch.float32, torch.float64)


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("rolloutlab-b200 needs a CUDA device (sm_100a); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def as_device_tensor(x, device: torch.device | None = None) -> torch.Tensor:
    """numpy / sequences -> f64 CUDA tensor (reference semantics); torch tensors keep bf16/f32/f64."""
    dev = device or default_device()
    if isinstance(x, torch.Tensor):
        t = x if x.dtype in _FLOAT_DTYPES else x.to(torch.float64)
        return t.to(dev).contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to(dev)


def nonfinite_count(t: torch.Tensor) -> int:
    """Number of non-finite elements, counted by `rlk_nonfinite_count` (synchronises)."""
    t = t.contiguous()
    cnt = torch.zeros(1, dtype=torch.int64, device=t.device)
    L.call("rlk_nonfinite_count", L.ptr(t), L.dtype_code(t.dtype), t.numel(), L.ptr(cnt), L.stream_handle())
    return int(cnt.item())


class ParamTable:
    """Immutable logit table of shape (context_count, max_len, vocab_size) held on the GPU."""

    __slots__ = ("_t",)

    def __init__(self, logits, *, copy: bool = True, check_finite: bool = True):
        t = as_device_tensor(logits)
        if t.ndim != 3:
            raise ValueError(f"logits must be 3-d, got shape {tuple(t.shape)}")
        if check_finite and t.numel() and nonfinite_count(t):
            raise ValueError("logits must be finite")
        if copy and isinstance(logits, torch.Tensor) and t.data_ptr() == logits.data_ptr():
            t = t.clone()
        self._t = t

    @staticmethod
    def zeros(context_count: int, max_len: int, vocab_size: int, dtype=torch.float64) -> "ParamTable":
        return ParamTable(torch.zeros((context_count, max_len, vocab_size), dtype=dtype, device=default_device()),
                          copy=False, check_finite=False)

    @property
    def logits(self) -> torch.Tensor:
        return self._t

    def numpy(self) -> np.ndarray:
        return self._t.detach().to(torch.float64).cpu().numpy()

    @property
    def context_count(self) -> int:
        return self._t.shape[0]

    @property
    def max_len(self) -> int:
        return self._t.shape[1]

    @property
    def vocab_size(self) -> int:
        return self._t.shape[2]

    @property
    def shape(self) -> tuple[int, int, int]:
        return tuple(self._t.shape)

    @property
    def dtype(self) -> torch.dtype:
        return self._t.dtype

    def equals(self, other: "ParamTable") -> bool:
        return self.shape == other.shape and bool(torch.equal(self._t, other._t))


@dataclass(frozen=True)
class TrainEngine:
    """Exact softmax over the stored logits."""


@dataclass(frozen=True)
class InferEngine:
    perturb_scale: float
    perturb_seed: int = 0

    def __post_init__(self):
        if self.perturb_scale < 0:
            raise ValueError("perturb_scale must be >= 0")


Engine = Union[TrainEngine, InferEngine]


def _check_engine(engine: Engine) -> None:
    if isinstance(engine, InferEngine) and engine.perturb_scale != 0.0:
        raise NotImplementedError("InferEngine perturbation is a host-side simulation outside the B200 hot path")


def _check_indices(params: ParamTable, context_id: int, position: int) -> None:
    if not 0 <= context_id < params.context_count:
        raise IndexError(f"context_id {context_id} out of range [0, {params.context_count})")
    if not 0 <= position < params.max_len:
        raise IndexError(f"position {position} out of range [0, {params.max_len})")


def log_token_dists(params: ParamTable, rows: torch.Tensor, temperatures: torch.Tensor,
                    out_dtype=torch.float64) -> torch.Tensor:
    """Batched log_token_dist: rows[k] = context * max_len + position; returns [len(rows), V]."""
    t = params.logits
    V = params.vocab_size
    n = int(rows.numel())
    out = torch.empty((n, V), dtype=out_dtype, device=t.device)
    L.call("rlk_logsoftmax_rows", L.ptr(t), L.dtype_code(t.dtype), n, V, V, L.ptr(rows), L.ptr(temperatures),
           L.ptr(out), L.dtype_code(out_dtype), L.stream_handle())
    return out


def log_token_dist(params: ParamTable, engine: Engine, context_id: int, position: int,
                   temperature: float = 1.0) -> torch.Tensor:
    """Log-probabilities over the vocabulary at one (context, position) slot (toy_env.py:157-175)."""
    _check_indices(params, context_id, position)
    _check_engine(engine)
    if temperature != 1.0 and temperature <= 0:
        raise ValueError("temperature must be > 0")
    dev = params.logits.device
    rows = torch.tensor([context_id * params.max_len + position], dtype=torch.int64, device=dev)
    temps = torch.tensor([float(temperature)], dtype=torch.float64, device=dev)
    return log_token_dists(params, rows, temps)[0]


def token_dist(params: ParamTable, engine: Engine, context_id: int, position: int) -> torch.Tensor:
    return torch.exp(log_token_dist(params, engine, context_id, position))


def logprob_trace(params: ParamTable, engine: Engine, sample: Sample) -> tuple[float, ...]:
    """Token log-probs of a finished sample at its recorded temperature (toy_env.py:287-297), via the
    K4 forward kernel with a log-prob-only epilogue."""
    if sample.status is SampleStatus.IN_FLIGHT:
        raise ValueError("cannot recompute log-probs for an in-flight sample")
    _check_engine(engine)
    if not sample.tokens:
        return ()
    for t in range(len(sample.tokens)):
        _check_indices(params, sample.context_id, t)
    from .objective import token_logprobs
    rows = [sample.context_id * params.max_len + t for t in range(len(sample.tokens))]
    lp = token_logprobs(params.logits.reshape(-1, params.vocab_size), list(sample.tokens),
                        temperature=sample.gen_temperature, rows=rows)
    return tuple(float(x) for x in lp.cpu().tolist())


def detect_repetition(tokens: Sequence[int], ngram: int, min_repeats: int) -> bool:
    """True iff the tail is one n-gram repeated >= min_repeats times back to back (toy_env.py:315-327)."""
    if ngram < 1:
        raise ValueError("ngram must be >= 1")
    if min_repeats < 2:
        raise ValueError("min_repeats must be >= 2")
    span = ngram * min_repeats
    if len(tokens) < span:
        return False
    tail = list(tokens[-span:])
    unit = tail[-ngram:]
    return all(tail[k * ngram:(k + 1) * ngram] == unit for k in range(min_repeats))
