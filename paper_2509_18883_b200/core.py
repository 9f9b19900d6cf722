"""Host-side RNG and domain records feeding the B200 hot path.

Mirrors the reference `rolloutlab.core` surface that the fusion and objective paths use:

* SplitMix64 counter RNG (`Rng`, `make_rng`, `split`) -- reference core.py:26-103.  Only the host needs
  it: it derives the per-expert child seeds whose draw j is computed on the GPU as
  ``mix64(child + (j + 1) * GAMMA)`` (core.py:69-71) inside the fusion kernels.
* `Sample`, `Group`, `RewardOutcome`, `RewardKind`, `SampleStatus` -- reference core.py:106-232, the
  records `objective.apply_masks` / `objective_value` consume.

The orchestration types (`Prompt`, `PolicyVersion`, `VersionRegistry`, `validate_sample`) are outside
the hot path and are not provided.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace
from enum import Enum
from fractions import Fraction
from typing import Iterable, Sequence, Union

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3

Tick = Union[int, Fraction]
RngLabel = Union[int, str]


def mix64(z: int) -> int:
    """SplitMix64 finaliser (core.py:42-49): xor-shift 30/27/31 with the two odd multipliers."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    return z ^ (z >> 31)


def label_hash(label: RngLabel) -> int:
    """64-bit FNV-1a over the UTF-8 bytes of ``repr(label)`` (core.py:52-57)."""
    h = FNV_OFFSET
    for byte in repr(label).encode("utf-8"):
        h = ((h ^ byte) * FNV_PRIME) & MASK64
    return h


# the reference's private names (core.py:42, 52), for callers that import them
_mix64 = mix64
_label_hash = label_hash


class Rng:
    """Counter-based SplitMix64 stream (core.py:60-97); `split` derives children from the seed only."""

    __slots__ = ("seed", "_counter")

    def __init__(self, seed: int):
        self.seed = seed & MASK64
        self._counter = self.seed

    @property
    def counter(self) -> int:
        return self._counter

    def advance(self, n_draws: int) -> None:
        """Skip n draws (what the reference's per-element loop would consume)."""
        self._counter = (self._counter + n_draws * GAMMA) & MASK64

    def next_u64(self) -> int:
        self._counter = (self._counter + GAMMA) & MASK64
        return mix64(self._counter)

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def normal(self) -> float:
        u1 = 1.0 - self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)

    def randrange(self, n: int) -> int:
        if n <= 0:
            raise ValueError(f"randrange needs n >= 1, got {n}")
        return self.next_u64() % n

    def shuffle(self, items: list) -> None:
        for i in range(len(items) - 1, 0, -1):
            j = self.randrange(i + 1)
            items[i], items[j] = items[j], items[i]

    def split(self, label: RngLabel) -> "Rng":
        return Rng(mix64(self.seed ^ label_hash(label)))


def make_rng(seed: int, label: RngLabel | None = None) -> Rng:
    rng = Rng(seed)
    return rng if label is None else rng.split(label)


def keep_threshold(p: float) -> int:
    """Integer form of the dropout test: ``uniform >= p``  <=>  ``(u64 >> 11) >= ceil(p * 2**53)``.

    ``p * 2**53`` is exact in binary64 (power-of-two scaling), so the ceiling is exact too.
    """
    if not 0.0 <= p < 1.0:
        raise ValueError("p must be in [0, 1)")
    return math.ceil(p * 2.0 ** 53)


def fusion_child_seeds(seed: int, n_experts: int) -> list[int]:
    """Child stream seeds used by `fuse` for expert i: make_rng(seed, "fusion-dropout").split(i)
    (fusion.py:170-171)."""
    parent = make_rng(seed, "fusion-dropout")
    return [parent.split(i).seed for i in range(n_experts)]


class SampleStatus(Enum):
    IN_FLIGHT = "in_flight"
    COMPLETE = "complete"
    TRUNCATED = "truncated"


class RewardKind(Enum):
    PASS = "pass"
    FAIL = "fail"
    GRADE_ERROR = "grade_error"


@dataclass(frozen=True)
class RewardOutcome:
    """Grading verdict; a GRADE_ERROR carries no score and is masked downstream (core.py:118-140)."""

    kind: RewardKind
    raw_score: float | None = None

    @staticmethod
    def passed() -> "RewardOutcome":
        return RewardOutcome(RewardKind.PASS, 1.0)

    @staticmethod
    def failed() -> "RewardOutcome":
        return RewardOutcome(RewardKind.FAIL, 0.0)

    @staticmethod
    def grade_error() -> "RewardOutcome":
        return RewardOutcome(RewardKind.GRADE_ERROR, None)

    @property
    def graded(self) -> bool:
        return self.kind is not RewardKind.GRADE_ERROR


@dataclass(frozen=True)
class Sample:
    """One rollout (core.py:157-183): tokens, behaviour log-probs on both engines, grading state."""

    prompt_id: int
    context_id: int
    version_id: int
    tokens: tuple[int, ...]
    infer_logps: tuple[float, ...]
    status: SampleStatus
    t_start: Tick
    t_end: Tick | None = None
    train_logps: tuple[float, ...] | None = None
    reward: RewardOutcome | None = None
    gen_temperature: float = 1.0

    def with_train_logps(self, logps: Sequence[float]) -> "Sample":
        return replace(self, train_logps=tuple(logps))

    def with_reward(self, reward: RewardOutcome) -> "Sample":
        return replace(self, reward=reward)


@dataclass(frozen=True)
class Group:
    """The G samples of one prompt (core.py:210-232)."""

    prompt_id: int
    samples: tuple[Sample, ...]

    def __post_init__(self):
        if len(self.samples) < 2:
            raise ValueError("a group needs G >= 2 samples")
        if any(s.prompt_id != self.prompt_id for s in self.samples):
            raise ValueError("all samples in a group must share prompt_id")

    @property
    def size(self) -> int:
        return len(self.samples)

    @property
    def birth_version(self) -> int:
        return max(s.version_id for s in self.samples)

    def with_samples(self, samples: Iterable[Sample]) -> "Group":
        return Group(self.prompt_id, tuple(samples))
