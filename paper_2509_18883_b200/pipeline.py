"""Sample intake in front of the GRPO loss: online filter, staleness gate, replay mix, batch assembly.

SURVEY.md §8(f) row 4 -- the host-side composition of the batch that `apply_masks` and the GRPO
kernels consume.  The reference's module (`rolloutlab/pipeline.py:1-260`) is per-arrival control flow
over a few dozen `Group` objects per batch: microseconds of host work per training step, with nothing
to move to the GPU.  It stays host logic here with the reference's names, argument meanings, seeded
draw order and error messages (pinned against fixtures generated from the reference,
tests/golden/pipeline_kat.json), and gains one bridge the reference does not need: `pack_batch`
turns an emitted batch into the device-side `GRPOBatch` in one host->device copy per field, so the
batch goes straight from the assembler into `grpo_forward` / `grpo_forward_backward`.

Draw order matters for bit-exact replay: `buffer_mix` takes `rng.randrange(len(entries))` once per
reused group, in order, popping from the current FIFO, then one `rng.shuffle` of the whole batch;
`BatchAssembler` without a buffer only shuffles.  Both match the reference draw for draw.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Iterable, Iterator, Sequence

from .core import Group, RewardKind, Rng

__all__ = [
    "FilterDecision", "StalenessDecision", "StalenessPolicy", "online_filter", "staleness_check",
    "ReplayBuffer", "buffer_mix", "AssemblyResult", "BatchAssembler", "assemble_batch", "pack_batch",
]


class FilterDecision(Enum):
    """pipeline.py:23-27."""
    KEEP = "keep"
    DISCARD_ALL_CORRECT = "discard_all_correct"
    DISCARD_ALL_WRONG = "discard_all_wrong"
    DISCARD_UNGRADABLE = "discard_ungradable"


class StalenessDecision(Enum):
    """pipeline.py:30-32."""
    REUSE = "reuse"
    REGENERATE = "regenerate"


@dataclass(frozen=True)
class StalenessPolicy:
    """pipeline.py:35-41: a group may be trained on while current - birth <= max_staleness."""
    max_staleness: int = 2

    def __post_init__(self):
        if self.max_staleness < 0:
            raise ValueError("max_staleness must be >= 0")


def online_filter(group: Group) -> FilterDecision:
    """pipeline.py:44-56: keep a group only if its graded samples hold both a PASS and a FAIL.

    Every sample must carry a reward (ValueError otherwise, checked before any decision); GRADE_ERROR
    samples are ignored, and a group with no graded sample is DISCARD_UNGRADABLE."""
    ungraded = next((s for s in group.samples if s.reward is None), None)
    if ungraded is not None:
        raise ValueError(f"ungraded sample in group for prompt {group.prompt_id}")
    seen_pass = seen_fail = False
    for s in group.samples:
        kind = s.reward.kind
        seen_pass |= kind is RewardKind.PASS
        seen_fail |= kind is RewardKind.FAIL
    if seen_pass and seen_fail:
        return FilterDecision.KEEP
    if seen_pass:
        return FilterDecision.DISCARD_ALL_CORRECT
    if seen_fail:
        return FilterDecision.DISCARD_ALL_WRONG
    return FilterDecision.DISCARD_UNGRADABLE


def staleness_check(group: Group, current_version: int, policy: StalenessPolicy) -> StalenessDecision:
    """pipeline.py:59-66 (birth version = newest sample version, core.py:230)."""
    birth = group.birth_version
    if birth > current_version:
        raise ValueError(f"group born at version {birth} is ahead of current {current_version}")
    lag = current_version - birth
    return StalenessDecision.REUSE if lag <= policy.max_staleness else StalenessDecision.REGENERATE


def _fresh_enough(group: Group, current_version: int, policy: StalenessPolicy) -> bool:
    return staleness_check(group, current_version, policy) is StalenessDecision.REUSE


def _split_stale(groups: Sequence[Group], current_version: int, policy: StalenessPolicy):
    """(kept, stale) in arrival order; every group is checked (a future version raises)."""
    verdict = [_fresh_enough(g, current_version, policy) for g in groups]
    kept = [g for g, ok in zip(groups, verdict) if ok]
    stale = [g for g, ok in zip(groups, verdict) if not ok]
    return kept, stale


@dataclass
class ReplayBuffer:
    """pipeline.py:69-106: FIFO store (oldest first) of kept groups for later batches.

    `insert` appends and evicts from the front beyond `capacity`; staleness is re-evaluated against
    the caller's version whenever entries are read."""

    capacity: int
    reuse_ratio: float
    entries: list[Group] = field(default_factory=list)

    def __post_init__(self):
        if self.capacity < 1:
            raise ValueError("capacity must be >= 1")
        if not 0.0 <= self.reuse_ratio < 1.0:
            raise ValueError("reuse_ratio must be in [0, 1)")

    def insert(self, group: Group) -> None:
        self.entries.append(group)
        excess = len(self.entries) - self.capacity
        if excess > 0:
            del self.entries[:excess]

    def drop_expired(self, current_version: int, policy: StalenessPolicy) -> list[Group]:
        """Remove and return the entries past the staleness bound (oldest first)."""
        self.entries, expired = _split_stale(self.entries, current_version, policy)
        return expired

    def valid_count(self, current_version: int, policy: StalenessPolicy) -> int:
        return sum(_fresh_enough(g, current_version, policy) for g in self.entries)

    def reuse_quota(self, batch_groups: int) -> int:
        """floor(reuse_ratio * batch_groups) capped by what the buffer holds (pipeline.py:128-129)."""
        return min(math.floor(self.reuse_ratio * batch_groups), len(self.entries))


def buffer_mix(buffer: ReplayBuffer, fresh: list[Group], batch_groups: int, current_version: int,
               policy: StalenessPolicy, rng: Rng) -> list[Group] | None:
    """pipeline.py:109-145: floor(reuse_ratio * batch_groups) staleness-valid buffer groups plus fresh
    ones, shuffled with `rng`.

    Expired buffer entries are dropped first.  With too few fresh groups it returns None and leaves
    `fresh` and the remaining buffer entries as they are; otherwise the drawn entries leave the buffer
    and the fresh groups the batch does not need are inserted into it (FIFO eviction)."""
    if batch_groups < 1:
        raise ValueError("batch_groups must be >= 1")
    buffer.drop_expired(current_version, policy)
    n_reuse = buffer.reuse_quota(batch_groups)
    n_fresh = batch_groups - n_reuse
    if len(fresh) < n_fresh:
        return None
    batch = [buffer.entries.pop(rng.randrange(len(buffer.entries))) for _ in range(n_reuse)]
    batch.extend(fresh[:n_fresh])
    for g in fresh[n_fresh:]:
        buffer.insert(g)
    rng.shuffle(batch)
    return batch


@dataclass(frozen=True)
class AssemblyResult:
    """pipeline.py:148-155: what offering one graded group produced."""

    decision: FilterDecision
    batch: list[Group] | None
    dropped_stale: tuple[Group, ...]
    reused_count: int = 0


class BatchAssembler:
    """pipeline.py:158-230: filter arrivals, emit a batch the moment enough kept groups are pending.

    The staleness gate runs on every kept arrival: pending groups that fell behind are dropped and
    returned to the caller for regeneration.  Without a buffer a batch is the first `batch_groups`
    pending groups, shuffled; with one, `buffer_mix` composes it and the leftover pending groups move
    into the buffer."""

    def __init__(self, batch_groups: int, policy: StalenessPolicy, buffer: ReplayBuffer | None = None,
                 rng: Rng | None = None):
        if batch_groups < 1:
            raise ValueError("batch_groups must be >= 1")
        self.batch_groups = batch_groups
        self.policy = policy
        self.buffer = buffer
        self.rng = rng if rng is not None else Rng(0)
        self.pending: list[Group] = []

    def _emit(self, current_version: int) -> tuple[list[Group] | None, int]:
        buf = self.buffer
        if buf is None:
            if len(self.pending) < self.batch_groups:
                return None, 0
            batch, self.pending = self.pending[:self.batch_groups], self.pending[self.batch_groups:]
            self.rng.shuffle(batch)
            return batch, 0
        buf.drop_expired(current_version, self.policy)
        n_reuse = buf.reuse_quota(self.batch_groups)
        if len(self.pending) + n_reuse < self.batch_groups:
            return None, 0
        batch = buffer_mix(buf, self.pending, self.batch_groups, current_version, self.policy, self.rng)
        if batch is None:  # unreachable: sized above with the same quota
            raise RuntimeError("buffer_mix returned no batch after sizing")
        self.pending = []
        return batch, n_reuse

    def offer(self, group: Group, current_version: int) -> AssemblyResult:
        decision = online_filter(group)
        if decision is not FilterDecision.KEEP:
            return AssemblyResult(decision, None, ())
        self.pending.append(group)
        self.pending, stale = _split_stale(self.pending, current_version, self.policy)
        batch, reused = self._emit(current_version)
        return AssemblyResult(decision, batch, tuple(stale), reused)


def assemble_batch(completion_stream: Iterable[Group], batch_size_groups: int, policy: StalenessPolicy,
                   current_version: int = 0, buffer: ReplayBuffer | None = None,
                   rng: Rng | None = None) -> Iterator[list[Group]]:
    """pipeline.py:233-248: yield each batch a `BatchAssembler` emits over a completion-ordered stream."""
    asm = BatchAssembler(batch_size_groups, policy, buffer, rng)
    for group in completion_stream:
        out = asm.offer(group, current_version)
        if out.batch is not None:
            yield out.batch


def pack_batch(groups: Sequence[Group], t_max: int, *, rep_cfg=None, adv_cfg=None, device=None):
    """An emitted batch -> (`MaskedBatch`, device `GRPOBatch`) for the LM-head GRPO kernels.

    `apply_masks` (objective.py:168-203) decides masks and advantages; every sample of every group is
    packed in batch order (one logits row per response token, `use` = 0 for masked samples), so the
    caller's forward over the batch's responses produces the logits rows in the same order.  The
    packed arrays are built on the host and copied once per field."""
    import torch

    from .objective import AdvantageConfig, Mask, RepetitionConfig, GRPOBatch, apply_masks

    masked = apply_masks(groups, t_max, rep_cfg or RepetitionConfig(), adv_cfg or AdvantageConfig())
    if not masked.groups:
        raise ValueError("cannot pack an empty batch")
    toks, lt, li, cu, adv, use, temps = [], [], [], [0], [], [], []
    for mg in masked.groups:
        for s, a, m in zip(mg.group.samples, mg.advantages, mg.masks):
            n = len(s.tokens)
            live = m is Mask.USE
            if live and (s.train_logps is None or len(s.train_logps) < n):
                raise ValueError(f"sample of prompt {s.prompt_id} has no train_logps for all its tokens")
            if len(s.infer_logps) < n:
                raise ValueError(f"sample of prompt {s.prompt_id} has fewer infer_logps than tokens")
            toks.extend(int(t) for t in s.tokens)
            # masked samples' rows are never read by the kernels; their train log-probs may be absent
            lt.extend([float(x) for x in s.train_logps[:n]] if live else [0.0] * n)
            li.extend(float(x) for x in s.infer_logps[:n])
            cu.append(len(toks))
            adv.append(float(a))
            use.append(1 if live else 0)
            temps.append(float(s.gen_temperature))
    batch = GRPOBatch.pack(toks, lt, li, cu, adv, use, masked.groups[0].group.size, t_max,
                           temperature=torch.tensor(temps, dtype=torch.float64), device=device)
    return masked, batch
