"""Task-vector fusion of domain-expert parameter tables on B200 (drop-in for `rolloutlab.fusion`).

Same names, signatures, defaults and error messages as the reference module
(pkg/src/rolloutlab/fusion.py): `TaskVector`, `FusionConfig`, `task_vector`, `normalize_magnitudes`,
`dropout_prune`, `erase_minority`, `FusionStats`, `fuse`, `merge`.  Tables live on the GPU
(`ParamTable` wraps a CUDA tensor); every arithmetic step runs in the sm_100a kernels of
`csrc/fusion.cu` behind the C ABI (`include/rlk.h`):

    K1 rlk_fusion_sumsq      per-(item, expert) f64 sums of squares of (expert - base)
    -- NCCL all_reduce of the partials when the parameter space is sharded over ranks (dist.py)
    rlk_fusion_finalize      norms, mean-of-non-zero target, per-(tensor, expert) scale
    K2 rlk_fusion_mask_bitmap SplitMix64 keep bits (bit-exact with the reference's draws)
    K3 rlk_fusion_merge      scale -> dropout -> erase vote -> base + sum_i w_i k_i, FusionStats counts

Extension: `fuse_state_dict` fuses whole checkpoints (any tensor shapes, flattened C-order) with the
reference's per-tensor `fuse` semantics and one shared `cfg` -- with one documented difference: a
tensor that no expert changed passes through as the base instead of raising the reference's
"cannot take mean norm of all-zero task vectors" (fusion.py:97-98).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Literal, Mapping, Sequence, Union

import numpy as np
import torch

from . import _lib as L
from .core import Rng, fusion_child_seeds, keep_threshold, make_rng
from .toy_env import ParamTable, as_device_tensor

MEAN_OF_INPUTS = "mean_of_inputs"
ITEM = L.RLK_FUSION_ITEM


# ----------------------------------------------------------------------------- config / stats
@dataclass(frozen=True)
class FusionConfig:
    """Fusion hyper-parameters, validated exactly like the reference (fusion.py:54-76)."""

    dropout_p: float = 0.0
    target_norm: Union[float, str, None] = MEAN_OF_INPUTS
    merge_weights: tuple[float, ...] | None = None
    erase_mode: bool = True
    erase_weighting: Literal["sum", "squared"] = "sum"
    seed: int = 0

    def __post_init__(self):
        if not 0.0 <= self.dropout_p < 1.0:
            raise ValueError("dropout_p must be in [0, 1)")
        if isinstance(self.target_norm, str) and self.target_norm != MEAN_OF_INPUTS:
            raise ValueError(f"target_norm string must be '{MEAN_OF_INPUTS}'")
        if isinstance(self.target_norm, (int, float)) and self.target_norm <= 0:
            raise ValueError("target_norm must be positive")
        if self.merge_weights is not None:
            if any(w < 0 for w in self.merge_weights):
                raise ValueError("merge weights must be non-negative")
            if abs(sum(self.merge_weights) - 1.0) > 1e-9:
                raise ValueError("merge weights must sum to 1")
        if self.erase_weighting not in ("sum", "squared"):
            raise ValueError("erase_weighting must be 'sum' or 'squared'")

    # kernel encodings
    @property
    def target_mode(self) -> int:
        if self.target_norm is None:
            return 0
        return 1 if isinstance(self.target_norm, str) else 2

    @property
    def erase_code(self) -> int:
        return 0 if not self.erase_mode else (1 if self.erase_weighting == "sum" else 2)


@dataclass(frozen=True)
class FusionStats:
    norms_before: tuple[float, ...]
    norms_after_normalize: tuple[float, ...]
    dropout_kept_fraction: tuple[float, ...]
    erased_counts: tuple[int, ...]
    weights: tuple[float, ...]


# ----------------------------------------------------------------------------- layout / plans
class FusionLayout:
    """Global geometry of a parameter space: tensors cut into RLK_FUSION_ITEM-element items.

    Items are counted from each tensor's start, so a piece handed to any rank starts on an item
    boundary and every (item, expert) partial is computed identically at every world size."""

    def __init__(self, numels: Sequence[int]):
        self.numels = [int(n) for n in numels]
        counts = [(n + ITEM - 1) // ITEM for n in self.numels]
        self.tensor_items = np.zeros(len(self.numels) + 1, dtype=np.uint32)
        np.cumsum(counts, out=self.tensor_items[1:])
        self.n_items = int(self.tensor_items[-1])
        self.total = sum(self.numels)
        self._dev = {}

    @property
    def n_tensors(self) -> int:
        return len(self.numels)

    def tensor_items_device(self, device, stream=None) -> torch.Tensor:
        key = str(device)
        if key not in self._dev:
            self._dev[key] = _upload(self.tensor_items.astype(np.uint32).view(np.int32), device, stream)
        return self._dev[key]

    def partition_striped(self, world: int, rank: int) -> list[tuple[int, int, int]]:
        """Like `partition`, but every tensor of at least max(ITEM * world, max numel / 4) elements (the
        embedding-sized ones) is cut into `world` item-aligned stripes, one per rank, and the remaining
        tensors' items are split into contiguous ranges balanced by element count.  A rank's pieces
        then read the dropout keep bits of their own index ranges only (the stripes of equally sized
        big tensors share one range), so each rank draws its own bits and no bitmap exchange is needed.
        Returns [(tensor, lo, hi)] in tensor order (lo a multiple of ITEM)."""
        if world < 1 or not 0 <= rank < world:
            raise ValueError(f"bad rank {rank} of {world}")
        if not self.numels:
            return []
        big_min = max(ITEM * world, max(self.numels) / 4)
        out: list[tuple[int, int, int]] = []
        small = []
        for t, n in enumerate(self.numels):
            if n >= big_min:
                items = (n + ITEM - 1) // ITEM
                a, b = items * rank // world, items * (rank + 1) // world
                if b > a:
                    out.append((t, a * ITEM, min(b * ITEM, n)))
            else:
                for k in range((n + ITEM - 1) // ITEM):
                    small.append((t, k * ITEM, min(ITEM, n - k * ITEM)))
        if small:
            starts = np.cumsum([0] + [x[2] for x in small])
            tot = int(starts[-1])
            bounds = [int(np.searchsorted(starts, tot * r / world, side="left")) for r in range(world + 1)]
            bounds[-1] = len(small)
            for t, lo, n in small[bounds[rank]:bounds[rank + 1]]:
                out.append((t, lo, lo + n))
        out.sort()
        merged: list[tuple[int, int, int]] = []
        for t, lo, hi in out:
            if merged and merged[-1][0] == t and merged[-1][2] == lo:
                merged[-1] = (t, merged[-1][1], hi)
            else:
                merged.append((t, lo, hi))
        return merged

    def partition(self, world: int, rank: int) -> list[tuple[int, int, int]]:
        """Rank `rank`'s contiguous share of the global item list, balanced by element count.

        Returns [(tensor, lo, hi)] element ranges (lo a multiple of ITEM)."""
        if world < 1 or not 0 <= rank < world:
            raise ValueError(f"bad rank {rank} of {world}")
        sizes = []
        for t, n in enumerate(self.numels):
            for k in range((n + ITEM - 1) // ITEM):
                sizes.append((t, k * ITEM, min(ITEM, n - k * ITEM)))
        starts = np.cumsum([0] + [s[2] for s in sizes])
        bounds = [int(np.searchsorted(starts, self.total * r / world, side="left")) for r in range(world + 1)]
        bounds[-1] = len(sizes)
        mine = sizes[bounds[rank]:bounds[rank + 1]]
        out: list[tuple[int, int, int]] = []
        for t, lo, n in mine:
            if out and out[-1][0] == t and out[-1][2] == lo:
                out[-1] = (t, out[-1][1], lo + n)
            else:
                out.append((t, lo, lo + n))
        return out


@dataclass
class Piece:
    """One contiguous element range [j0, j0 + numel) of tensor `tensor`, as flat device tensors."""

    tensor: int
    j0: int
    base: torch.Tensor | None
    experts: Sequence[torch.Tensor]
    out: torch.Tensor | None

    @property
    def numel(self) -> int:
        return int(self.experts[0].numel())


def _aligned(t: torch.Tensor) -> torch.Tensor:
    t = t.contiguous()
    if t.data_ptr() % 16:
        t = t.clone()
    return t


def _upload(arr: np.ndarray, device, stream=None) -> torch.Tensor:
    """Small host table -> device.  With a stream: staged through pinned memory and copied
    asynchronously on that stream (so it never waits behind bulk copies on another stream)."""
    host = torch.from_numpy(np.ascontiguousarray(arr).copy())
    if stream is None:
        return host.to(device)
    with torch.cuda.stream(stream):
        return host.pin_memory().to(device, non_blocking=True)


def needed_bit_ranges(spans: Sequence[tuple[int, int]]) -> list[tuple[int, int]]:
    """Union of element index ranges [lo, hi) as sorted disjoint ranges with lo rounded down and hi
    rounded up to 32 (whole bitmap words)."""
    out: list[tuple[int, int]] = []
    for lo, hi in sorted((lo // 32 * 32, (hi + 31) // 32 * 32) for lo, hi in spans if hi > lo):
        if out and lo <= out[-1][1]:
            out[-1] = (out[-1][0], max(out[-1][1], hi))
        else:
            out.append((lo, hi))
    return out


class _Plan:
    def __init__(self, pieces: Sequence[Piece], layout: FusionLayout, n_experts: int, device, stream=None):
        segs = np.zeros(len(pieces), dtype=L.SEGMENT_DTYPE)
        counts = np.zeros(len(pieces), dtype=np.int64)
        for k, p in enumerate(pieces):
            if p.j0 % ITEM:
                raise ValueError("piece offsets must be multiples of RLK_FUSION_ITEM")
            segs[k]["base"] = 0 if p.base is None else p.base.data_ptr()
            for i, e in enumerate(p.experts):
                segs[k]["expert"][i] = e.data_ptr()
            segs[k]["out"] = 0 if p.out is None else p.out.data_ptr()
            segs[k]["numel"] = p.numel
            segs[k]["j0"] = p.j0
            segs[k]["tensor"] = p.tensor
            segs[k]["item0"] = int(layout.tensor_items[p.tensor]) + p.j0 // ITEM
            counts[k] = (p.numel + ITEM - 1) // ITEM
        prefix = np.zeros(len(pieces) + 1, dtype=np.uint32)
        np.cumsum(counts, out=prefix[1:])
        self.segs_dev = _upload(segs.view(np.uint8), device, stream)
        self.prefix_dev = _upload(prefix.view(np.int32), device, stream)
        self.c = L.FusionPlanC(self.segs_dev.data_ptr(), self.prefix_dev.data_ptr(), len(pieces), int(prefix[-1]))
        self.max_extent = max((p.j0 + p.numel for p in pieces), default=0)
        self.local_elems = sum(p.numel for p in pieces)


class FusionCall:
    """One fusion over a set of pieces: K1 -> [all_reduce] -> finalize -> [K2] -> K3 on one stream.

    Device results: `sumsq`, `scale` [n_tensors, N] f64, `status` [n_tensors] i32, `counters`
    [n_tensors, 2N] i64 (non-zero after dropout, erased)."""

    def __init__(self, pieces: Sequence[Piece], layout: FusionLayout, n_experts: int, cfg: FusionConfig,
                 *, delta_mode: bool = False, with_base: bool = True, group=None, stream=None,
                 dropout_mode: int | None = None, async_upload: bool = True, exact_merge: bool = False,
                 fixup: bool = True):
        if not 1 <= n_experts <= L.RLK_MAX_EXPERTS:
            raise NotImplementedError(f"the B200 kernels fuse 1..{L.RLK_MAX_EXPERTS} experts, got {n_experts}")
        if not pieces:
            raise ValueError("nothing to fuse")
        self.pieces = pieces
        self.layout = layout
        self.n = n_experts
        self.cfg = cfg
        self.delta_mode = delta_mode
        self.with_base = with_base
        self.group = group
        self.device = pieces[0].experts[0].device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.dtype_in = pieces[0].experts[0].dtype
        # launch-plan tables go up on the call's stream (async) unless the caller builds plans while
        # the device is idle (async_upload=False: one short blocking copy each)
        up = stream if async_upload else None
        self.plan = _Plan(pieces, layout, n_experts, self.device, up)
        layout.tensor_items_device(self.device, up)
        nt = layout.n_tensors
        f64 = dict(dtype=torch.float64, device=self.device)
        self.sumsq = torch.empty((nt, n_experts), **f64)
        self.scale = torch.empty((nt, n_experts), **f64)
        self.status = torch.empty(nt, dtype=torch.int32, device=self.device)
        self.counters = torch.zeros((nt, 2 * n_experts), dtype=torch.int64, device=self.device)
        self.partials = None
        # exact_merge: K3 runs the reference-order f64 kernel instead of the certified f32x2 fast path
        # (same results; the parity tests compare the two)
        self.exact_merge = exact_merge
        # fixup: the bf16 fast merge defers its inconclusive elements to a fix-up kernel (workspace
        # queue) instead of finishing them inside the merge; identical results
        self.fixup = fixup
        p = cfg.dropout_p
        if p == 0.0:
            dropout_mode = 0
        elif dropout_mode not in (1, 2):
            # K2 bitmap pays N * max_extent draws once; inline hashing pays N per element in K3.  The
            # bf16 fast merge path reads keep bits from the bitmap only.
            dropout_mode = 2 if (self.plan.local_elems >= 2 * self.plan.max_extent
                                 or self.dtype_in == torch.bfloat16) else 1
        self.dropout_mode = dropout_mode
        self.seeds = fusion_child_seeds(cfg.seed, n_experts) if p > 0 else [0] * n_experts
        self.thresh = keep_threshold(p) if p > 0 else 0
        self.keep_prob = 1.0 - p
        self.bitmap = None
        self.words_per_row = 0
        self.timers: dict[str, list] | None = None  # name -> [(start_event, end_event)] when profiling
        # sharded norms: tensors this rank holds pieces of, and (set on the first sharded step) the item
        # rows of the tensors split over ranks -- the only partials that are exchanged -- plus each
        # tensor's owner rank (the lowest holding it), which contributes its row to gathered statistics
        self.held = sorted({p.tensor for p in pieces})
        self._shared_rows: torch.Tensor | None = None
        self._owner: torch.Tensor | None = None

    def _launch(self, name: str, *args) -> None:
        if self.timers is None:
            L.call(name, *args)
            return
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        L.call(name, *args)
        e1.record(self.stream)
        self.timers.setdefault(name, []).append((e0, e1))

    def run(self, weights: Sequence[float], dtype_out: torch.dtype | None = None) -> "FusionCall":
        """One complete fusion step on the call's stream: zero counters, [K2], K1, [all_reduce],
        finalize, K3.  Reusing a FusionCall across steps reuses its launch plan (host metadata only)."""
        with L.nvtx_range("rlk.fusion_step"), torch.cuda.stream(self.stream):
            self.counters.zero_()
            return self.norms().merge(weights, dtype_out)

    def capture(self, weights: Sequence[float], dtype_out: torch.dtype | None = None) -> "torch.cuda.CUDAGraph":
        """`run(weights)` captured once into a CUDA graph on the call's stream; `graph.replay()` inside
        `torch.cuda.stream(call.stream)` repeats the whole step (same buffers) with one launch.  For
        small, launch-bound fusions; single-process only (the sharded step has NCCL collectives)."""
        if self.group is not None:
            raise NotImplementedError("graph capture of the sharded step is not supported")
        self.run(weights, dtype_out)  # allocates the lazily-sized buffers outside the capture
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            self.run(weights, dtype_out)
        return g

    def _bitmap(self, s) -> None:
        """K2: keep bits for every (expert, within-tensor index < max extent) -- before K1, which
        counts the non-zero entries after dropout, and K3."""
        if self.dropout_mode != 2:
            return
        world = 1
        if self.group is not None:
            import torch.distributed as dist
            world = dist.get_world_size(self.group)
        seeds = (L.C.c_uint64 * self.n)(*self.seeds)
        if world == 1:
            n_bits = ((self.plan.max_extent + 8191) // 8192) * 8192
            self.words_per_row = n_bits // 32
            self._alloc_bitmap()
            self._launch("rlk_fusion_mask_bitmap", seeds, self.n, self.thresh, n_bits, L.ptr(self.bitmap),
                         self.words_per_row, s)
            return
        # sharded: the rows span the layout's largest tensor (the same row pitch on every rank), but a
        # rank draws only the index ranges its own pieces read -- with `partition_striped` the
        # embedding-sized tensors contribute one stripe each, so no rank draws whole rows and no
        # bitmap crosses GPUs
        n_bits = ((max(self.layout.numels) + 8191) // 8192) * 8192
        self.words_per_row = n_bits // 32
        self._alloc_bitmap()
        for lo, hi in needed_bit_ranges([(p.j0, p.j0 + p.numel) for p in self.pieces]):
            self._launch("rlk_fusion_mask_bitmap_range", seeds, self.n, self.thresh, lo, min(hi, n_bits),
                         L.ptr(self.bitmap), self.words_per_row, s)

    def _alloc_bitmap(self) -> None:
        if self.bitmap is None or self.bitmap.numel() != self.n * self.words_per_row:
            self.bitmap = torch.empty(self.n * self.words_per_row, dtype=torch.int32, device=self.device)

    # -- K1 + all_reduce + finalize
    def norms(self) -> "FusionCall":
        s = L.stream_handle(self.stream)
        with torch.cuda.stream(self.stream):
            world = 1
            if self.group is not None:
                import torch.distributed as dist
                world = dist.get_world_size(self.group)
            if self.partials is None or self.partials.numel() != self.layout.n_items * self.n:
                self.partials = torch.zeros(self.layout.n_items * self.n, dtype=torch.float64, device=self.device)
            if world > 1:
                if self._shared_rows is None:
                    self._shared_plan(world)
                if self._shared_rows.numel():
                    # other ranks' slots of the split tensors must be exactly zero for the exact sum
                    self.partials.view(-1, self.n).index_fill_(0, self._shared_rows, 0.0)
            self._bitmap(s)
            seeds = (L.C.c_uint64 * self.n)(*self.seeds)
            self._launch("rlk_fusion_sumsq", L.C.byref(self.plan.c), self.n, L.dtype_code(self.dtype_in),
                         int(self.delta_mode), L.ptr(self.partials), L.ptr(self.counters), self.dropout_mode,
                         seeds, self.thresh, L.ptr(self.bitmap), self.words_per_row, s)
            if world > 1 and self._shared_rows.numel():
                # only the item rows of tensors split over ranks cross GPUs (a tensor held by one rank
                # has all its partials there already); every row has exactly one non-zero contributor,
                # so the sum is exact and the norms are identical at every world size
                from .dist import allreduce_partials
                rows = self.partials.view(-1, self.n)
                buf = rows.index_select(0, self._shared_rows)
                allreduce_partials(buf, self.group)
                rows.index_copy_(0, self._shared_rows, buf)
            self._launch("rlk_fusion_finalize", L.ptr(self.partials),
                         L.ptr(self.layout.tensor_items_device(self.device, self.stream)), self.layout.n_tensors,
                         self.n, self.cfg.target_mode,
                         float(self.cfg.target_norm) if self.cfg.target_mode == 2 else 0.0,
                         L.ptr(self.sumsq), L.ptr(self.scale), L.ptr(self.status), s)
        return self

    def _shared_plan(self, world: int) -> None:
        """Once per sharded call: which tensors are split over ranks (their item rows are the partials
        that get all-reduced) and which rank owns each tensor's statistics (two tiny all_reduces)."""
        import torch.distributed as dist
        nt = self.layout.n_tensors
        held = torch.zeros(nt, dtype=torch.int64, device=self.device)
        held[self.held] = 1
        cnt = held.clone()
        dist.all_reduce(cnt, group=self.group)
        rank = dist.get_rank(self.group)
        owner = torch.where(held > 0, torch.full_like(held, rank), torch.full_like(held, world))
        dist.all_reduce(owner, op=dist.ReduceOp.MIN, group=self.group)
        ti = self.layout.tensor_items
        shared = [t for t in (cnt >= 2).nonzero().flatten().tolist()]
        rows = np.concatenate([np.arange(ti[t], ti[t + 1], dtype=np.int64) for t in shared]) if shared \
            else np.zeros(0, dtype=np.int64)
        self._shared_rows = torch.from_numpy(rows).to(self.device)
        self._owner = owner == rank

    def check_status(self, per_tensor_raise: bool = True) -> torch.Tensor:
        st = self.status.cpu()
        if self._owner is not None:  # sharded: only the tensors this rank holds were normalised here
            mask = torch.zeros_like(st, dtype=torch.bool)
            mask[self.held] = True
            st = torch.where(mask, st, torch.zeros_like(st))
        if per_tensor_raise:
            if bool((st == 2).any()):
                raise ValueError("logits must be finite")
            if bool((st == 1).any()):
                raise ValueError("cannot take mean norm of all-zero task vectors")
        return st

    # -- K2 + K3
    def merge(self, weights: Sequence[float], dtype_out: torch.dtype | None = None,
              erase_code: int | None = None) -> "FusionCall":
        s = L.stream_handle(self.stream)
        erase = self.cfg.erase_code if erase_code is None else erase_code
        if self.n < 2:
            erase = 0
        with torch.cuda.stream(self.stream):
            if self.dropout_mode == 2 and self.bitmap is None:
                self._bitmap(s)  # K3 without a preceding K1 (staged transforms)
            w = (L.C.c_double * self.n)(*[float(x) for x in weights])
            seeds = (L.C.c_uint64 * self.n)(*self.seeds)
            dmode = (1 | (2 if self.with_base else 0)) if self.delta_mode else 0
            dto = dtype_out or self.pieces[0].out.dtype
            ws = self._merge_workspace()
            self._launch("rlk_fusion_merge_ws", L.C.byref(self.plan.c), self.n, L.dtype_code(self.dtype_in),
                         L.dtype_code(dto), dmode, L.ptr(self.scale), w, self.dropout_mode,
                         seeds if self.dropout_mode else None, self.thresh, self.keep_prob,
                         L.ptr(self.bitmap), self.words_per_row, erase, L.ptr(self.counters), int(self.exact_merge),
                         L.ptr(ws), ws.numel(), s)
        return self

    # fix-up queue of the bf16 fast merge (16 bytes per entry for up to 3 experts, 32 beyond).  With
    # normalisation a step flags ~1 element in 2,300 (their f32 bracket straddles a bf16 rounding
    # boundary): room for 1/1024 of the local elements.  Without it (target_norm=None) the arithmetic is
    # exact enough that ~2% of the results land exactly on bf16 midpoints (b + (2/3) m u crossing a
    # binade): room for 1/16.  Overflow falls back to the in-kernel exact path (same results, slower).
    def _merge_workspace(self) -> torch.Tensor:
        if not self.fixup:
            return torch.empty(0, dtype=torch.uint8, device=self.device)
        ws = getattr(self, "_ws", None)
        if ws is None:
            frac = 16 if self.cfg.target_norm is None else 1024
            per = 16 if self.n <= 3 else 32
            entries = min(max(self.plan.local_elems // frac, 1 << 16), (8 << 30) // per)
            ws = torch.empty(L.RLK_MERGE_WS_HEADER + per * entries, dtype=torch.uint8, device=self.device)
            ws[:L.RLK_MERGE_WS_HEADER].zero_()  # queue lengths of CTAs a launch does not use read as 0
            self._ws = ws
        return ws

    def stats(self, tensor: int, weights: Sequence[float], size: int | None = None,
              host: tuple | None = None) -> FusionStats:
        """FusionStats of one tensor (fusion.py:145-151, 165-182).  Synchronises (unless `host` holds
        the (sumsq, scale, counters) tables already copied by `host_tables`)."""
        if host is None:
            sumsq, scale, cnt = (x[tensor].cpu().numpy() for x in (self.sumsq, self.scale, self.counters))
        else:
            sumsq, scale, cnt = (x[tensor] for x in host)
        size = self.layout.numels[tensor] if size is None else size
        norms = tuple(math.sqrt(float(x)) for x in sumsq)
        after = tuple(n if (self.cfg.target_norm is None or n == 0.0) else n * float(sc)
                      for n, sc in zip(norms, scale))
        nz = cnt[: self.n]
        kept = tuple(float(z) / size for z in nz)
        erased = tuple(int(e) for e in cnt[self.n:])
        return FusionStats(norms, after, kept, erased, tuple(float(x) for x in weights))

    def host_tables(self) -> tuple:
        """(sumsq, scale, counters) as host arrays, one copy each (for stats over many tensors)."""
        return tuple(x.cpu().numpy() for x in (self.sumsq, self.scale, self.counters))


# ----------------------------------------------------------------------------- task vectors
class TaskVector:
    """Elementwise difference between an expert table and the shared base (fusion.py:29-51).

    Held lazily as the (expert, base) pair of device tensors -- the fused path never materialises the
    delta -- or as an explicit delta tensor.  `norm` is computed on first use by the K1 kernel."""

    __slots__ = ("_delta", "_expert", "_base", "source_label", "_norm")

    def __init__(self, delta, source_label: str = "", norm: float = 0.0):
        arr = as_device_tensor(delta)
        if arr.ndim != 3:
            raise ValueError("delta must match the 3-d parameter table shape")
        if isinstance(delta, torch.Tensor) and arr.data_ptr() == delta.data_ptr():
            arr = arr.clone()
        self._delta = arr
        self._expert = None
        self._base = None
        self.source_label = source_label
        self._norm = None

    @classmethod
    def _pair(cls, expert: torch.Tensor, base: torch.Tensor, label: str = "") -> "TaskVector":
        tv = cls.__new__(cls)
        tv._delta = None
        tv._expert = expert
        tv._base = base
        tv.source_label = label
        tv._norm = None
        return tv

    @property
    def shape(self) -> tuple[int, int, int]:
        return tuple((self._delta if self._delta is not None else self._expert).shape)

    @property
    def is_pair(self) -> bool:
        return self._delta is None

    @property
    def device(self):
        return (self._delta if self._delta is not None else self._expert).device

    @property
    def numel(self) -> int:
        return int((self._delta if self._delta is not None else self._expert).numel())

    @property
    def delta(self) -> torch.Tensor:
        """The f64 delta (materialised on demand for pair vectors: expert - base, exact in f64)."""
        if self._delta is None:
            e = self._expert.to(torch.float64)
            b = self._base.to(torch.float64)
            out = torch.empty_like(e)
            L.call("rlk_scaled_add", L.ptr(e), L.ptr(b), -1.0, L.ptr(out), L.RLK_F64, e.numel(), L.stream_handle())
            self._delta = out
        return self._delta

    @property
    def norm(self) -> float:
        if self._norm is None:
            _compute_norms([self])
        return self._norm

    def with_delta(self, delta) -> "TaskVector":
        return TaskVector(delta, self.source_label)


def _flat(t: torch.Tensor) -> torch.Tensor:
    return _aligned(t.reshape(-1))


def _compute_norms(taus: Sequence[TaskVector]) -> None:
    """Fill `_norm` for every vector lacking it: one K1 launch per distinct storage mode/dtype."""
    for t in taus:
        if t._norm is None and t.numel == 0:
            t._norm = 0.0  # np.linalg.norm of an empty array
    todo = [t for t in taus if t._norm is None]
    if not todo:
        return
    groups: dict[tuple, list[TaskVector]] = {}
    for t in todo:
        key = (t.is_pair, (t._expert if t.is_pair else t._delta).dtype)
        groups.setdefault(key, []).append(t)
    for (is_pair, _dt), ts in groups.items():
        layout = FusionLayout([t.numel for t in ts])
        pieces = [Piece(k, 0, _flat(t._base) if is_pair else None,
                        [_flat(t._expert if is_pair else t._delta)], None) for k, t in enumerate(ts)]
        call = FusionCall(pieces, layout, 1, FusionConfig(target_norm=None), delta_mode=not is_pair)
        call.norms()
        sumsq = call.sumsq[:, 0].cpu().numpy()
        for t, s2 in zip(ts, sumsq):
            t._norm = math.sqrt(float(s2))


def task_vector(theta_rl: ParamTable, theta_sft: ParamTable, label: str = "") -> TaskVector:
    """Expert-minus-base delta (fusion.py:79-83), kept as the lazy (expert, base) pair."""
    if theta_rl.shape != theta_sft.shape:
        raise ValueError(f"shape mismatch: {theta_rl.shape} vs {theta_sft.shape}")
    e, b = theta_rl.logits, theta_sft.logits
    if e.dtype != b.dtype:
        e, b = e.to(torch.float64), b.to(torch.float64)
    return TaskVector._pair(e, b, label)


def _transform(taus: Sequence[TaskVector], *, scales: Sequence[float] | None = None, dropout: tuple | None = None,
               erase_code: int = 0, emit: int | None = None) -> list[torch.Tensor]:
    """Materialise transformed deltas (f64) with K3 in delta mode without a base:
    fused = 0 + sum_i w_i k_i with w one-hot on `emit` (exact: 0 * k = 0 and x + 0 = x)."""
    n = len(taus)
    src = [t.delta for t in taus]
    if any(s.dtype != src[0].dtype for s in src):
        src = [s.to(torch.float64) for s in src]
    out = torch.empty(taus[0].shape, dtype=torch.float64, device=taus[0].device)
    piece = Piece(0, 0, None, [_flat(s) for s in src], out.view(-1))
    cfg = FusionConfig(target_norm=None, erase_mode=bool(erase_code),
                       erase_weighting="squared" if erase_code == 2 else "sum")
    call = FusionCall([piece], FusionLayout([piece.numel]), n, cfg, delta_mode=True, with_base=False)
    call.scale = torch.tensor([list(scales) if scales is not None else [1.0] * n], dtype=torch.float64,
                              device=out.device)
    if dropout is not None:
        seed, thresh, keep_prob = dropout
        call.dropout_mode, call.seeds, call.thresh, call.keep_prob = 1, [seed], thresh, keep_prob
    w = [0.0] * n
    w[0 if emit is None else emit] = 1.0
    call.merge(w, dtype_out=torch.float64, erase_code=erase_code)
    return [out]


def normalize_magnitudes(taus: Sequence[TaskVector], cfg: FusionConfig) -> list[TaskVector]:
    """Rescale each non-zero vector to the target L2 norm (fusion.py:86-102)."""
    if cfg.target_norm is None:
        return list(taus)
    _compute_norms(taus)
    nonzero = [t for t in taus if t.norm > 0.0]
    if isinstance(cfg.target_norm, str):
        if not nonzero:
            raise ValueError("cannot take mean norm of all-zero task vectors")
        target = sum(t.norm for t in nonzero) / len(nonzero)
    else:
        target = float(cfg.target_norm)
    out = []
    for t in taus:
        if t.norm == 0.0:
            out.append(t)
        else:
            (d,) = _transform([t], scales=[target / t.norm])
            out.append(TaskVector(d, t.source_label))
    return out


def dropout_prune(tau: TaskVector, p: float, rng: Rng) -> TaskVector:
    """Zero each element with probability p, survivors / (1 - p) (fusion.py:105-115).

    Draw j of `rng` decides element j (flat C order); the rng advances by numel draws, exactly as the
    reference's per-element loop leaves it."""
    if not 0.0 <= p < 1.0:
        raise ValueError("p must be in [0, 1)")
    if p == 0.0:
        return tau
    (d,) = _transform([tau], dropout=(rng.counter, keep_threshold(p), 1.0 - p))
    rng.advance(tau.numel)
    return tau.with_delta(d)


def erase_minority(taus: Sequence[TaskVector], weighting: str = "sum") -> list[TaskVector]:
    """Zero entries whose sign opposes the cross-expert majority (fusion.py:118-142)."""
    if len(taus) < 2:
        raise ValueError("erase needs at least 2 task vectors")
    shapes = {t.shape for t in taus}
    if len(shapes) > 1:
        raise ValueError("task vectors must share a shape")
    if weighting not in ("sum", "squared"):
        raise ValueError("weighting must be 'sum' or 'squared'")
    if len(taus) > L.RLK_MAX_EXPERTS:
        raise NotImplementedError(f"at most {L.RLK_MAX_EXPERTS} task vectors")
    code = 1 if weighting == "sum" else 2
    return [t.with_delta(_transform(taus, erase_code=code, emit=i)[0]) for i, t in enumerate(taus)]


# ----------------------------------------------------------------------------- fuse / merge
def fuse(theta_sft: ParamTable, taus: Sequence[TaskVector], cfg: FusionConfig,
         out_dtype: torch.dtype | None = None, *, exact_merge: bool = False) -> tuple[ParamTable, FusionStats]:
    """normalize -> dropout -> erase -> weighted sum, with FusionStats (fusion.py:154-188).

    One K1 + finalize + K3 pass over (base, experts); the output keeps the base's dtype unless
    `out_dtype` is given (the reference's output is float64)."""
    if not taus:
        raise ValueError("need at least one task vector")
    for t in taus:
        if t.shape != theta_sft.shape:
            raise ValueError(f"task vector shape {t.shape} != base shape {theta_sft.shape}")
    if cfg.merge_weights is not None and len(cfg.merge_weights) != len(taus):
        raise ValueError("merge_weights length must match the expert count")
    weights = cfg.merge_weights or tuple(1.0 / len(taus) for _ in taus)
    if theta_sft.logits.numel() == 0:
        # an empty table: every norm is 0, so the mean target has no non-zero norm (fusion.py:97-98),
        # and otherwise the kept fraction count_nonzero / size divides by zero (fusion.py:172-174)
        if cfg.target_mode == 1:
            raise ValueError("cannot take mean norm of all-zero task vectors")
        raise ZeroDivisionError("float division by zero")

    base = theta_sft.logits
    pair = all(t.is_pair and t._base.data_ptr() == base.data_ptr() and t._expert.dtype == base.dtype
               for t in taus)
    if pair:
        experts = [t._expert for t in taus]
        b = base
    else:
        experts = [t.delta for t in taus]
        b = base.to(torch.float64) if base.dtype != torch.float64 else base
    dto = out_dtype or base.dtype
    out = torch.empty(base.shape, dtype=dto, device=base.device)
    piece = Piece(0, 0, _flat(b), [_flat(e) for e in experts], out.view(-1))
    call = FusionCall([piece], FusionLayout([piece.numel]), len(taus), cfg, delta_mode=not pair,
                      exact_merge=exact_merge)
    call.norms()
    call.check_status()
    call.merge(weights, dtype_out=dto)
    stats = call.stats(0, weights)
    for t, n in zip(taus, stats.norms_before):
        if t._norm is None:
            t._norm = n
    return ParamTable(out, copy=False), stats


def merge(theta_sft: ParamTable, taus: Sequence[TaskVector], cfg: FusionConfig) -> ParamTable:
    """Fused table theta_sft + sum_i w_i * tau'_i (fusion.py:191-194)."""
    fused, _ = fuse(theta_sft, taus, cfg)
    return fused


# ----------------------------------------------------------------------------- state dicts
@dataclass
class FusionReport:
    names: list[str]
    call: FusionCall
    weights: tuple[float, ...]

    def stats(self, name: str) -> FusionStats:
        return self.call.stats(self.names.index(name), self.weights)

    def passthrough(self) -> list[str]:
        """Tensors no expert changed (kept as base instead of the reference's ValueError)."""
        st = self.call.status.cpu().tolist()
        return [n for n, s in zip(self.names, st) if s == 1]


def fuse_state_dict(base: Mapping[str, torch.Tensor], experts: Sequence[Mapping[str, torch.Tensor]],
                    cfg: FusionConfig = FusionConfig(), *, out_dtype: torch.dtype | None = None,
                    out: Mapping[str, torch.Tensor] | None = None, stream=None,
                    check: bool = True, exact_merge: bool = False,
                    dropout_mode: int | None = None) -> tuple[dict[str, torch.Tensor], FusionReport]:
    """Fuse whole checkpoints: per tensor the reference `fuse` with one shared cfg, in ONE K1 launch,
    one finalize and ONE K3 launch over every tensor (plus K2 when dropout_p > 0).

    All tensors must be CUDA tensors of one dtype (bf16 / f32 / f64).  `check` synchronises once at
    the end and raises ValueError on non-finite inputs.  `exact_merge` / `dropout_mode` (1 inline keep
    bits, 2 K2 bitmap) pin the kernel variants; every choice gives the same results."""
    names = list(base.keys())
    n = len(experts)
    if n == 0:
        raise ValueError("need at least one task vector")
    if cfg.merge_weights is not None and len(cfg.merge_weights) != n:
        raise ValueError("merge_weights length must match the expert count")
    weights = cfg.merge_weights or tuple(1.0 / n for _ in range(n))
    dt = base[names[0]].dtype
    dto = out_dtype or dt
    pieces = []
    outs: dict[str, torch.Tensor] = {}
    for k, name in enumerate(names):
        b = base[name]
        es = [e[name] for e in experts]
        for e in es:
            if e.shape != b.shape:
                raise ValueError(f"task vector shape {tuple(e.shape)} != base shape {tuple(b.shape)}")
            if e.dtype != dt or b.dtype != dt:
                raise ValueError("all tensors of a fused state dict must share one dtype")
        o = out[name] if out is not None else torch.empty(b.shape, dtype=dto, device=b.device)
        outs[name] = o
        pieces.append(Piece(k, 0, _flat(b), [_flat(e) for e in es], o.view(-1)))
    layout = FusionLayout([p.numel for p in pieces])
    call = FusionCall(pieces, layout, n, cfg, stream=stream, exact_merge=exact_merge, dropout_mode=dropout_mode)
    call.norms()
    call.merge(weights, dtype_out=dto)
    if check:
        st = call.status.cpu()
        if bool((st == 2).any()):
            raise ValueError("logits must be finite")
    return outs, FusionReport(names, call, tuple(weights))
