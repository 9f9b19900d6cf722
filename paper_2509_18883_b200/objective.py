"""GRPO token-level objective on B200 (drop-in for `rolloutlab.objective`).

Reference: pkg/src/rolloutlab/objective.py.  The per-token term is

    min(exp(logp_train - logp_infer), cap) * triplet_clip(exp(logp - logp_train), A)

summed over the USE samples of each group, divided by G * T_max, averaged over groups
(objective.py:230-250).  The vocab-wide work -- log-softmax of z / T, the gather of the token's
log-prob, the ratio / TIS / clip epilogue and the gradient coef * (onehot - softmax) -- runs in the
sm_100a kernels of csrc/grpo.cu (K4 `rlk_grpo_fwd`, K5 `rlk_grpo_bwd`).  Advantages, masks and the
batch packing are host logic, as in the reference.

Two entry points:
* the reference's object API (`objective_value`, `objective_gradient` over `MaskedBatch` +
  `ParamTable`), packed into the tensor form;
* the tensor API `grpo_token_objective` / `GRPOTokenLoss` over packed logits rows [R, V] (the LLM
  layout: one row per response token) -- the hot path benchmarked in bench.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np
import torch

from . import _lib as L
from .core import Group, RewardKind, Sample, SampleStatus
from .toy_env import ParamTable, detect_repetition


# ----------------------------------------------------------------------------- configs / records
@dataclass(frozen=True)
class ClipConfig:
    """Triplet clip + TIS cap, validated like objective.py:40-58."""

    eps_neg_low: float = 0.2
    eps_pos_high: float = 0.2
    eps_neg_high: float = 3.0
    tis_cap: float = 2.0
    guard_positive: bool = True

    def __post_init__(self):
        if not 0.0 < self.eps_neg_low < 1.0:
            raise ValueError("eps_neg_low must be in (0, 1)")
        if self.eps_pos_high <= 0.0:
            raise ValueError("eps_pos_high must be > 0")
        if self.eps_neg_high <= 1.0:
            raise ValueError("eps_neg_high must be > 1")
        if self.eps_neg_high < 1.0 + self.eps_pos_high:
            raise ValueError("eps_neg_high must be >= 1 + eps_pos_high")
        if self.tis_cap < 1.0:
            raise ValueError("tis_cap must be >= 1")

    def c_struct(self) -> L.ClipC:
        return L.ClipC(self.eps_neg_low, self.eps_pos_high, self.eps_neg_high, self.tis_cap,
                       1 if self.guard_positive else 0)


class NormMode(Enum):
    MEAN_STD = "mean_std"
    MEAN_ONLY = "mean_only"


@dataclass(frozen=True)
class AdvantageConfig:
    norm_mode: NormMode = NormMode.MEAN_STD
    std_floor: float = 1e-8

    def __post_init__(self):
        if self.std_floor <= 0.0:
            raise ValueError("std_floor must be > 0")


class Mask(Enum):
    USE = "use"
    MASK_GRADE_ERROR = "mask_grade_error"
    MASK_TRUNCATED = "mask_truncated"


@dataclass(frozen=True)
class RepetitionConfig:
    ngram: int = 2
    min_repeats: int = 3


@dataclass(frozen=True)
class MaskedGroup:
    group: Group
    advantages: tuple[float, ...]
    masks: tuple[Mask, ...]

    def __post_init__(self):
        if not (len(self.advantages) == len(self.masks) == self.group.size):
            raise ValueError("advantages/masks must align with the group's samples")


@dataclass(frozen=True)
class MaskedBatch:
    groups: tuple[MaskedGroup, ...]
    t_max: int

    def __post_init__(self):
        if self.t_max < 1:
            raise ValueError("t_max must be >= 1")
        longest = max((len(s.tokens) for mg in self.groups for s in mg.group.samples), default=0)
        if self.t_max < longest:
            raise ValueError(f"t_max {self.t_max} below max token length {longest}")
        if len({mg.group.size for mg in self.groups}) > 1:
            raise ValueError("all groups in a batch must share the same G")


# ----------------------------------------------------------------------------- host scalar math
def group_advantages(rewards: Sequence[float], cfg: AdvantageConfig) -> list[float]:
    """(r - mean) / max(population std, floor), or r - mean (objective.py:119-130)."""
    if len(rewards) < 2:
        raise ValueError("advantage normalization needs G >= 2 rewards")
    r = np.asarray(rewards, dtype=np.float64)
    if not np.isfinite(r).all():
        raise ValueError("rewards must be finite")
    centred = r - r.mean()
    if cfg.norm_mode is NormMode.MEAN_ONLY:
        return [float(x) for x in centred]
    denom = max(float(r.std()), cfg.std_floor)
    return [float(x / denom) for x in centred]


def _triplet_value_slope(r_theta: float, adv: float, cfg: ClipConfig) -> tuple[float, float]:
    """Host copy of the kernel's triplet epilogue (objective.py:133-150); ties take the unclipped branch."""
    lo, hi = 1.0 - cfg.eps_neg_low, 1.0 + cfg.eps_pos_high
    clipped = min(max(r_theta, lo), hi)
    in_band = 1.0 if lo <= r_theta <= hi else 0.0
    raw, capped = r_theta * adv, clipped * adv
    inner, slope = (raw, adv) if raw <= capped else (capped, adv * in_band)
    if cfg.guard_positive and adv > 0.0:
        return inner, slope
    floor = cfg.eps_neg_high * adv
    return (inner, slope) if inner >= floor else (floor, 0.0)


def triplet_clip_term(r_theta: float, adv: float, cfg: ClipConfig) -> float:
    if r_theta <= 0.0:
        raise ValueError("probability ratio must be > 0")
    return _triplet_value_slope(r_theta, adv, cfg)[0]


def tis_weight(logp_mu_train: float, logp_mu_infer: float, cap: float) -> float:
    """min(exp(logp_train - logp_infer), cap) (objective.py:161-165)."""
    if not (math.isfinite(logp_mu_train) and math.isfinite(logp_mu_infer)):
        raise ValueError("log-probs must be finite")
    return min(math.exp(logp_mu_train - logp_mu_infer), cap)


def apply_masks(groups: Sequence[Group], t_max: int, rep_cfg: RepetitionConfig = RepetitionConfig(),
                adv_cfg: AdvantageConfig = AdvantageConfig()) -> MaskedBatch:
    """Mask GradeErrors and non-repetitive truncations; advantages over usable samples (objective.py:168-203)."""
    out = []
    for group in groups:
        masks = []
        for s in group.samples:
            if s.reward is None:
                raise ValueError(f"ungraded sample for prompt {s.prompt_id}")
            if s.reward.kind is RewardKind.GRADE_ERROR:
                masks.append(Mask.MASK_GRADE_ERROR)
            elif s.status is SampleStatus.TRUNCATED and not detect_repetition(s.tokens, rep_cfg.ngram,
                                                                                rep_cfg.min_repeats):
                masks.append(Mask.MASK_TRUNCATED)
            else:
                masks.append(Mask.USE)
        usable = [i for i, m in enumerate(masks) if m is Mask.USE]
        adv = [0.0] * group.size
        if len(usable) >= 2:
            for i, a in zip(usable, group_advantages([group.samples[i].reward.raw_score for i in usable], adv_cfg)):
                adv[i] = a
        out.append(MaskedGroup(group, tuple(adv), tuple(masks)))
    return MaskedBatch(tuple(out), t_max)


# ----------------------------------------------------------------------------- tensor API
GRPO_WS_FLOATS_PER_ROW = 32  # K4a partials: (max, sum) per consumer warp (include/rlk.h)

@dataclass
class GRPOBatch:
    """Packed device-side description of a token batch (rows grouped by sample, samples by group).

    Per row: tokens i32, logp_train / logp_infer f64, sample_of_row i32 (local sample index),
    row_index i64 or None.  Per local sample: adv, use (u8), temperature, norm = 1/(n_groups*G*T_max),
    and sample_rows[S_local + 1] (row offsets).  A batch may hold a contiguous slice of the global
    sample list (`select`, `shard`): `sample_base` is its first global sample and `group_samples`
    [n_groups + 1] the global sample offsets of the groups, so per-sample token sums land at fixed
    global slots and the objective is reduced in the same order at every world size."""

    tokens: torch.Tensor
    logp_train: torch.Tensor
    logp_infer: torch.Tensor
    sample_of_row: torch.Tensor
    adv: torch.Tensor
    use: torch.Tensor
    temperature: torch.Tensor
    norm: torch.Tensor
    sample_rows: torch.Tensor
    group_samples: torch.Tensor
    n_groups: int
    group_size: int
    t_max: int
    n_samples: int
    sample_base: int = 0
    row_index: torch.Tensor | None = None
    sample_rows_host: tuple[int, ...] = ()

    @property
    def n_rows(self) -> int:
        return int(self.tokens.numel())

    @property
    def n_local_samples(self) -> int:
        return int(self.adv.numel())

    def all_groups_seg(self) -> torch.Tensor:
        seg = getattr(self, "_all_seg", None)
        if seg is None:
            seg = torch.tensor([0, self.n_groups], dtype=torch.int64, device=self.tokens.device)
            self._all_seg = seg
        return seg

    @staticmethod
    def pack(tokens, logp_train, logp_infer, cu_seqlens, adv, use, group_size: int, t_max: int,
             temperature=1.0, device=None, row_index=None) -> "GRPOBatch":
        """Build from per-row arrays and per-sample cu_seqlens (samples of one group contiguous)."""
        dev = device or torch.device("cuda", torch.cuda.current_device())
        cu = torch.as_tensor(cu_seqlens, dtype=torch.int64).cpu()
        S = cu.numel() - 1
        if S % group_size:
            raise ValueError("sample count must be a multiple of the group size")
        n_groups = S // group_size
        lens = (cu[1:] - cu[:-1])
        if lens.numel() and int(lens.max()) > t_max:
            raise ValueError(f"t_max {t_max} below max token length {int(lens.max())}")
        sample_of_row = torch.repeat_interleave(torch.arange(S, dtype=torch.int32), lens).to(dev)
        temp = torch.as_tensor(temperature, dtype=torch.float64)
        temp = (temp.expand(S) if temp.ndim == 0 else temp).contiguous().to(dev)
        if bool((temp <= 0).any()):
            raise ValueError("temperature must be > 0")
        norm = torch.full((S,), 1.0 / (n_groups * group_size * t_max), dtype=torch.float64, device=dev)
        f64 = lambda x: torch.as_tensor(x, dtype=torch.float64).to(dev).contiguous()
        return GRPOBatch(
            tokens=torch.as_tensor(tokens, dtype=torch.int32).to(dev).contiguous(),
            logp_train=f64(logp_train), logp_infer=f64(logp_infer), sample_of_row=sample_of_row,
            adv=f64(adv), use=torch.as_tensor(use, dtype=torch.uint8).to(dev).contiguous(), temperature=temp,
            norm=norm, sample_rows=cu.to(dev).contiguous(),
            group_samples=torch.arange(0, S + 1, group_size, dtype=torch.int64).to(dev), n_groups=n_groups,
            group_size=group_size, t_max=t_max, n_samples=S, sample_rows_host=tuple(int(x) for x in cu),
            row_index=None if row_index is None else torch.as_tensor(row_index, dtype=torch.int64).to(dev))

    def select(self, s0: int, s1: int) -> "GRPOBatch":
        """The sub-batch of local samples [s0, s1) (their rows, same global normalisation): a response
        shard of a rank, or a chunk streamed through one logits buffer."""
        S = self.n_local_samples
        if not 0 <= s0 <= s1 <= S:
            raise IndexError(f"sample range [{s0}, {s1}) outside [0, {S})")
        cu = self.sample_rows_host
        r0, r1 = cu[s0], cu[s1]
        rows = slice(r0, r1)
        sub_cu = tuple(c - r0 for c in cu[s0:s1 + 1])
        return GRPOBatch(
            tokens=self.tokens[rows], logp_train=self.logp_train[rows], logp_infer=self.logp_infer[rows],
            sample_of_row=(self.sample_of_row[rows] - s0).contiguous(), adv=self.adv[s0:s1],
            use=self.use[s0:s1], temperature=self.temperature[s0:s1], norm=self.norm[s0:s1],
            sample_rows=torch.tensor(sub_cu, dtype=torch.int64, device=self.tokens.device),
            group_samples=self.group_samples, n_groups=self.n_groups, group_size=self.group_size,
            t_max=self.t_max, n_samples=self.n_samples, sample_base=self.sample_base + s0,
            row_index=None if self.row_index is None else self.row_index[rows], sample_rows_host=sub_cu)

    def shard_bounds(self, world: int) -> list[int]:
        """Sample boundaries of `world` contiguous shards balanced by row count (the loss
        shards by response; a rank may get none)."""
        cu = self.sample_rows_host
        R = cu[-1]
        bounds = [0]
        for r in range(1, world):
            target = R * r / world
            # first sample boundary at or after the target row count, never moving backwards
            k = bounds[-1]
            while k < len(cu) - 1 and cu[k] < target:
                k += 1
            bounds.append(k)
        bounds.append(len(cu) - 1)
        return bounds

    def shard(self, world: int, rank: int) -> "GRPOBatch":
        """This rank's contiguous share of the samples (`shard_bounds`)."""
        b = self.shard_bounds(world)
        return self.select(b[rank], b[rank + 1])


@dataclass
class GRPOForward:
    objective: torch.Tensor  # 0-d f64 (J, to maximise)
    group_sums: torch.Tensor  # [n_groups] f64: sum of token terms per group
    logp: torch.Tensor
    lse: torch.Tensor
    term: torch.Tensor
    coef: torch.Tensor
    flags: torch.Tensor
    sample_sums: torch.Tensor | None = None  # [n_local_samples] f64: this batch's per-sample sums


def grpo_objective(sample_sums: torch.Tensor, batch: GRPOBatch, group=None, *, stream=None) -> tuple:
    """J from per-sample token sums: the sums go to their global slots of an [n_samples] vector (zero
    elsewhere), which is all-reduced over `group` -- every slot has exactly one non-zero contributor,
    so the sum is exact -- then summed per group in a fixed order, / (G T_max), averaged over groups
    (objective.py:237-250).  J is therefore bit-identical at every world size.  Returns (J, group sums)."""
    dev = sample_sums.device
    f64 = dict(dtype=torch.float64, device=dev)
    s = L.stream_handle(stream)
    if batch.sample_base == 0 and sample_sums.numel() == batch.n_samples and group is None:
        full = sample_sums
    else:
        full = torch.zeros(batch.n_samples, **f64)
        full[batch.sample_base:batch.sample_base + sample_sums.numel()] = sample_sums
    if group is not None:
        import torch.distributed as dist
        dist.all_reduce(full, group=group)
    gs = torch.empty(batch.n_groups, **f64)
    L.call("rlk_segment_sum_f64", L.ptr(full), L.ptr(batch.group_samples), batch.n_groups, L.ptr(gs), s)
    scaled = gs / float(batch.group_size * batch.t_max)
    tot = torch.empty(1, **f64)
    L.call("rlk_segment_sum_f64", L.ptr(scaled), L.ptr(batch.all_groups_seg()), 1, L.ptr(tot), s)
    return tot[0] / batch.n_groups, gs


def _finish(term: torch.Tensor, batch: GRPOBatch, group, s) -> tuple:
    ss = torch.empty(batch.n_local_samples, dtype=torch.float64, device=term.device)
    L.call("rlk_segment_sum_f64", L.ptr(term), L.ptr(batch.sample_rows), batch.n_local_samples, L.ptr(ss), s)
    J, gs = grpo_objective(ss, batch, group)
    return J, gs, ss


def grpo_forward(logits: torch.Tensor, batch: GRPOBatch, clip: ClipConfig = ClipConfig(), *, stream=None,
                 group=None) -> GRPOForward:
    """K4 over every row + fixed-order per-sample then per-group sums; J = sum_g (S_g / (G T_max)) / n_groups.

    `logits` is [rows, V] (row_stride = V) in bf16/f32/f64.  With a process group, `batch` is this
    rank's share of the samples (`GRPOBatch.shard`) and the per-sample sums are all-reduced (one f64
    vector of n_samples entries); without one, a partial batch gives its own samples' share of J."""
    if logits.ndim != 2:
        raise ValueError("logits must be [rows, vocab]")
    if stream is not None:
        with torch.cuda.stream(stream):
            return grpo_forward(logits, batch, clip, group=group)
    logits = logits.contiguous()
    R, V = batch.n_rows, logits.shape[1]
    dev = logits.device
    f64 = dict(dtype=torch.float64, device=dev)
    logp, lse, term, coef = (torch.empty(R, **f64) for _ in range(4))
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    s = L.stream_handle(stream)
    c = clip.c_struct()
    ws = torch.empty(R * GRPO_WS_FLOATS_PER_ROW, dtype=torch.float32, device=dev)
    L.call("rlk_grpo_fwd", L.ptr(logits), L.dtype_code(logits.dtype), R, V, V, L.ptr(batch.row_index),
           L.ptr(batch.tokens), L.ptr(batch.logp_train), L.ptr(batch.logp_infer), L.ptr(batch.sample_of_row),
           L.ptr(batch.adv), L.ptr(batch.use), L.ptr(batch.temperature), L.ptr(batch.norm), L.C.byref(c),
           L.ptr(logp), L.ptr(lse), L.ptr(term), L.ptr(coef), L.ptr(flags), L.ptr(ws), ws.numel(), s)
    J, gs, ss = _finish(term, batch, group, s)
    return GRPOForward(J, gs, logp, lse, term, coef, flags, ss)


def _row_csr(row_index: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Tokens grouped by the logits row they read: (distinct rows ascending, CSR pointers, token ids in
    stable order) -- tokens sharing a row accumulate in the reference's order (objective.py:278-282)."""
    order = torch.sort(row_index, stable=True).indices
    rows, counts = torch.unique_consecutive(row_index[order], return_counts=True)
    ptr = torch.zeros(rows.numel() + 1, dtype=torch.int64, device=row_index.device)
    torch.cumsum(counts, 0, out=ptr[1:])
    return rows.contiguous(), ptr, order.contiguous()


def grpo_backward(logits: torch.Tensor, batch: GRPOBatch, fwd: GRPOForward, grad_scale: torch.Tensor | float = 1.0,
                  grad_dtype: torch.dtype | None = None, *, stream=None, group=None) -> torch.Tensor:
    """K5: grad_scale * dJ/dlogits, same shape as `logits` (the autograd grad_out is `grad_scale`).

    Without `row_index`, token r reads logits row r (the batch's rows must not exceed the logits'; rows
    past the batch get a zero gradient) and a sharded batch needs no communication.  With `row_index`,
    every distinct row read is written once as the sum over the tokens that read it (CSR), and rows no
    token reads are zero (objective.py:253-283); with a process group the shared table's gradient is
    then summed over the ranks (all_reduce)."""
    if stream is not None:
        with torch.cuda.stream(stream):
            return grpo_backward(logits, batch, fwd, grad_scale, grad_dtype, group=group)
    if logits.ndim != 2:
        raise ValueError("logits must be [rows, vocab]")
    logits = logits.contiguous()
    R, V = logits.shape
    nb = batch.n_rows
    coef = fwd.coef if (isinstance(grad_scale, float) and grad_scale == 1.0) else fwd.coef * grad_scale
    coef = coef.contiguous()
    temp_tok = batch.temperature[batch.sample_of_row.long()].contiguous()
    gdt = grad_dtype or logits.dtype
    s = L.stream_handle(stream)
    if batch.row_index is None:
        if nb > R:
            raise ValueError(f"batch has {nb} token rows but logits only {R}")
        grad = torch.empty((R, V), dtype=gdt, device=logits.device)
        if nb < R:
            grad[nb:].zero_()
        L.call("rlk_grpo_bwd", L.ptr(logits), L.dtype_code(logits.dtype), nb, V, V, None, None, None,
               L.ptr(batch.tokens), L.ptr(temp_tok), L.ptr(fwd.lse), L.ptr(coef), L.ptr(grad),
               L.dtype_code(grad.dtype), V, s)
        return grad
    ri = batch.row_index
    if nb and (int(ri.min()) < 0 or int(ri.max()) >= R):
        raise IndexError(f"row_index out of range [0, {R})")
    grad = torch.zeros((R, V), dtype=gdt, device=logits.device)
    if nb:
        rows, ptr_, order = _row_csr(ri)
        L.call("rlk_grpo_bwd", L.ptr(logits), L.dtype_code(logits.dtype), rows.numel(), V, V, L.ptr(rows),
               L.ptr(ptr_), L.ptr(order), L.ptr(batch.tokens), L.ptr(temp_tok), L.ptr(fwd.lse), L.ptr(coef),
               L.ptr(grad), L.dtype_code(grad.dtype), V, s)
    if group is not None:
        import torch.distributed as dist
        dist.all_reduce(grad, group=group)
    return grad


def grpo_forward_backward(logits: torch.Tensor, batch: GRPOBatch, clip: ClipConfig = ClipConfig(),
                          grad_scale: float = 1.0, *, stream=None, group=None) -> tuple[GRPOForward, torch.Tensor]:
    """J and grad_scale * dJ/dlogits in ONE read of the logits (bf16 or f32, one row per token): the
    fused cluster kernel `rlk_grpo_fused` (2-CTA clusters for bf16, 4 for f32); the gradient has the
    logits' dtype.  f64 logits and `row_index` layouts fall back to K4 + K5."""
    if stream is not None:
        with torch.cuda.stream(stream):
            return grpo_forward_backward(logits, batch, clip, grad_scale, group=group)
    logits = logits.contiguous()
    R, V = logits.shape
    cl = 2 if logits.dtype == torch.bfloat16 else 4
    if logits.dtype not in (torch.bfloat16, torch.float32) or batch.row_index is not None or V % (8 * cl) \
            or V > 204800:
        fwd = grpo_forward(logits, batch, clip, group=group)
        return fwd, grpo_backward(logits, batch, fwd, grad_scale, group=group)
    nb = batch.n_rows  # token r reads logits row r; rows past the batch get a zero gradient
    if nb > R:
        raise ValueError(f"batch has {nb} token rows but logits only {R}")
    dev = logits.device
    f64 = dict(dtype=torch.float64, device=dev)
    logp, lse, term, coef = (torch.empty(nb, **f64) for _ in range(4))
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    grad = torch.empty_like(logits)
    if nb < R:
        grad[nb:].zero_()
    c = clip.c_struct()
    s = L.stream_handle()
    L.call("rlk_grpo_fused", L.ptr(logits), L.dtype_code(logits.dtype), nb, V, V, None, L.ptr(batch.tokens),
           L.ptr(batch.logp_train),
           L.ptr(batch.logp_infer), L.ptr(batch.sample_of_row), L.ptr(batch.adv), L.ptr(batch.use),
           L.ptr(batch.temperature), L.ptr(batch.norm), L.C.byref(c), float(grad_scale), L.ptr(logp), L.ptr(lse),
           L.ptr(term), L.ptr(coef), L.ptr(flags), L.ptr(grad), V, s)
    J, gs, ss = _finish(term, batch, group, s)
    return GRPOForward(J, gs, logp, lse, term, coef, flags, ss), grad


class GRPOTokenLoss(torch.autograd.Function):
    """Autograd wrapper: forward returns J (maximised objective); backward runs K5.

    With `fused_scale` set (the d(loss)/dJ the caller will back-propagate, e.g. -1.0 for
    loss = -J), the forward runs the fused loss+gradient kernel -- one read of the logits instead of
    K4 now and K5 later -- and keeps `fused_scale * dJ/dlogits`; backward returns it when grad_out
    equals fused_scale (one scalar read), and otherwise recomputes with K5."""

    @staticmethod
    def forward(ctx, logits, batch: GRPOBatch, clip: ClipConfig, fused_scale=None):
        ctx.saved_grad = None
        if fused_scale is not None and logits.requires_grad:
            fwd, g = grpo_forward_backward(logits, batch, clip, grad_scale=float(fused_scale))
            ctx.saved_grad, ctx.fused_scale = g, float(fused_scale)
        else:
            fwd = grpo_forward(logits, batch, clip)
        ctx.save_for_backward(logits)
        ctx.batch, ctx.fwd = batch, fwd
        return fwd.objective

    @staticmethod
    def backward(ctx, grad_out):
        (logits,) = ctx.saved_tensors
        if ctx.saved_grad is not None and float(grad_out) == ctx.fused_scale:
            g, ctx.saved_grad = ctx.saved_grad, None
            return g.to(logits.dtype), None, None, None
        g = grpo_backward(logits, ctx.batch, ctx.fwd, grad_out.to(torch.float64))
        return g, None, None, None


def grpo_token_objective(logits: torch.Tensor, batch: GRPOBatch, clip: ClipConfig = ClipConfig(),
                         fused_scale: float | None = None) -> torch.Tensor:
    """J with autograd support; see GRPOTokenLoss for `fused_scale` (one-read loss + gradient)."""
    return GRPOTokenLoss.apply(logits, batch, clip, fused_scale)


def token_logprobs(logits2d: torch.Tensor, tokens: Sequence[int], temperature: float = 1.0,
                   rows: Sequence[int] | None = None) -> torch.Tensor:
    """log p(token) under z / T for the given rows (K4 with a log-prob-only epilogue)."""
    n = len(tokens)
    dev = logits2d.device
    zeros = np.zeros(n)
    b = GRPOBatch.pack(tokens, zeros, zeros, [0, n], [0.0], [1], 1, max(n, 1), temperature=[temperature],
                       device=dev, row_index=rows)
    return grpo_forward(logits2d, b).logp


# ----------------------------------------------------------------------------- object API (reference)
class _LogDistCache:
    """Memoizes per-(context, position, temperature) log-dists for one call (objective.py:206-220).

    The batched paths (objective_value / objective_gradient) compute every row's log-sum-exp in one
    K4 launch instead; this mirror serves callers of the reference's per-token interface, each miss
    being one device row (`toy_env.log_token_dist`, the fused log-softmax kernel)."""

    def __init__(self, params: ParamTable):
        from .toy_env import TrainEngine
        self.params = params
        self.engine = TrainEngine()
        self._cache: dict[tuple[int, int, float], torch.Tensor] = {}

    def get(self, context_id: int, position: int, temperature: float) -> torch.Tensor:
        from .toy_env import log_token_dist
        key = (context_id, position, temperature)
        if key not in self._cache:
            self._cache[key] = log_token_dist(self.params, self.engine, context_id, position, temperature)
        return self._cache[key]


def _require_logps(sample: Sample) -> None:
    if sample.train_logps is None:
        raise ValueError(f"sample for prompt {sample.prompt_id} is missing train log-probs")
    if len(sample.infer_logps) != len(sample.tokens):
        raise ValueError("infer log-probs do not align with tokens")


def _pack_masked_batch(batch: MaskedBatch, params: ParamTable) -> tuple[GRPOBatch, list]:
    """USE samples' tokens -> packed rows reading logits row context_id * max_len + t."""
    V, T = params.vocab_size, params.max_len
    toks, lt, li, rows, cu, adv, temps = [], [], [], [], [0], [], []
    group_samples = [0]
    for mg in batch.groups:
        for sample, a, mask in zip(mg.group.samples, mg.advantages, mg.masks):
            if mask is not Mask.USE:
                continue
            _require_logps(sample)
            tau = sample.gen_temperature
            if tau != 1.0 and tau <= 0:
                raise ValueError("temperature must be > 0")
            if not 0 <= sample.context_id < params.context_count:
                raise IndexError(f"context_id {sample.context_id} out of range [0, {params.context_count})")
            for t, tok in enumerate(sample.tokens):
                if not 0 <= t < T:
                    raise IndexError(f"position {t} out of range [0, {T})")
                tok = int(tok)
                if not -V <= tok < V:
                    raise IndexError(f"index {tok} is out of bounds for axis 0 with size {V}")
                toks.append(tok % V)  # numpy indexing wraps negative ids (objective.py:244)
                rows.append(sample.context_id * T + t)
            # the reference reads train_logps[t] for t < len(tokens) only (objective.py:243-247): extra
            # entries are ignored, a short list raises IndexError at the first missing position
            n_tok = len(sample.tokens)
            if len(sample.train_logps) < n_tok:
                raise IndexError("tuple index out of range")
            lt.extend(float(x) for x in sample.train_logps[:n_tok])
            li.extend(float(x) for x in sample.infer_logps)
            cu.append(len(toks))
            adv.append(float(a))
            temps.append(float(tau))
        group_samples.append(len(cu) - 1)
    lt_a, li_a = np.asarray(lt, dtype=np.float64), np.asarray(li, dtype=np.float64)
    if not (np.isfinite(lt_a).all() and np.isfinite(li_a).all()):
        raise ValueError("log-probs must be finite")
    S = len(adv)
    dev = params.logits.device
    cu_t = torch.tensor(cu, dtype=torch.int64)
    lens = cu_t[1:] - cu_t[:-1]
    G, n_groups = batch.groups[0].group.size, len(batch.groups)
    b = GRPOBatch(
        tokens=torch.tensor(toks, dtype=torch.int32, device=dev),
        logp_train=torch.from_numpy(lt_a).to(dev), logp_infer=torch.from_numpy(li_a).to(dev),
        sample_of_row=torch.repeat_interleave(torch.arange(S, dtype=torch.int32), lens).to(dev),
        adv=torch.tensor(adv, dtype=torch.float64, device=dev),
        use=torch.ones(S, dtype=torch.uint8, device=dev),
        temperature=torch.tensor(temps, dtype=torch.float64, device=dev),
        norm=torch.full((S,), 1.0 / (n_groups * G * batch.t_max), dtype=torch.float64, device=dev),
        sample_rows=cu_t.to(dev), group_samples=torch.tensor(group_samples, dtype=torch.int64, device=dev),
        n_groups=n_groups, group_size=G, t_max=batch.t_max, n_samples=S, sample_rows_host=tuple(cu),
        row_index=torch.tensor(rows, dtype=torch.int64, device=dev))
    return b, rows


def objective_value(batch: MaskedBatch, params: ParamTable, clip: ClipConfig) -> float:
    """Per group sum token terms / (G * T_max), averaged over groups (objective.py:230-250)."""
    if not batch.groups:
        return 0.0
    b, _ = _pack_masked_batch(batch, params)
    if b.n_rows == 0:
        return 0.0
    fwd = grpo_forward(params.logits.reshape(-1, params.vocab_size), b, clip)
    if int(fwd.flags.item()) & 1:
        raise ValueError("log-probs must be finite")
    gs = fwd.group_sums.cpu().tolist()
    G = batch.groups[0].group.size
    total = 0.0
    for g_sum in gs:
        total += g_sum / (G * batch.t_max)
    return total / len(batch.groups)


def objective_gradient(batch: MaskedBatch, params: ParamTable, clip: ClipConfig) -> torch.Tensor:
    """Exact gradient of objective_value w.r.t. the logit table (objective.py:253-283), f64, same shape.

    Tokens that share a (context, position) row accumulate in the reference's order (K5, CSR rows)."""
    grad = torch.zeros(params.shape, dtype=torch.float64, device=params.logits.device)
    if not batch.groups:
        return grad
    b, rows = _pack_masked_batch(batch, params)
    if b.n_rows == 0:
        return grad
    logits2d = params.logits.reshape(-1, params.vocab_size)
    fwd = grpo_forward(logits2d, b, clip)
    # K5 over the distinct (context, position) rows; tokens sharing a row accumulate (CSR)
    return grpo_backward(logits2d, b, fwd, grad_dtype=torch.float64).view(params.shape)


def ascent_step(params: ParamTable, gradient, lr: float) -> ParamTable:
    """New snapshot params + lr * gradient (objective.py:286-293), via rlk_scaled_add."""
    if lr < 0:
        raise ValueError("lr must be >= 0")
    g = torch.as_tensor(np.asarray(gradient, dtype=np.float64)) if not isinstance(gradient, torch.Tensor) else gradient
    if tuple(g.shape) != params.shape:
        raise ValueError(f"gradient shape {tuple(g.shape)} != params shape {params.shape}")
    p = params.logits.to(torch.float64).contiguous()
    g = g.to(device=p.device, dtype=torch.float64).contiguous()
    out = torch.empty_like(p)
    L.call("rlk_scaled_add", L.ptr(p), L.ptr(g), float(lr), L.ptr(out), L.RLK_F64, p.numel(), L.stream_handle())
    return ParamTable(out, copy=False)
