"""Streaming fusion of checkpoints larger than HBM (BASELINE configs[3]).

Host state dicts (numpy arrays, CPU torch tensors, memory maps) are fused tensor-group by tensor-group:
each group's base + N experts are copied host -> device through the C++ loader (`rlk_loader_*`:
pinned slot ring + worker threads, csrc/loader.cpp) on a copy stream, fused on a compute stream
(K2 -> K1 -> finalize -> K3, exactly `fuse_state_dict` on the group), and the fused group is copied
back device -> host while the next group streams in.  Device workspaces are double-buffered, so
H2D of group g+1 overlaps the kernels and the D2H of group g.

Per-tensor semantics are those of the reference `fuse` (fusion.py:154-188) with one shared cfg; a
tensor must fit in half the device budget (large MoE checkpoints store experts per matrix).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _lib as L
from .fusion import FusionCall, FusionConfig, FusionLayout, FusionStats, Piece


class HostLoader:
    """RAII wrapper over the C++ pinned-slot loader."""

    def __init__(self, slot_bytes: int = 64 << 20, n_slots: int = 4, n_threads: int = 0):
        self._h = L.lib().rlk_loader_create(slot_bytes, n_slots, n_threads)
        if not self._h:
            raise L.RlkError("rlk_loader_create failed (slot_bytes must be > 0 and n_slots >= 2)")

    def _check(self, st: int, what: str) -> None:
        if st != 0:
            raise L.RlkError(f"{what}: {L.lib().rlk_loader_last_error().decode()} (status {st})")

    def h2d(self, dst: torch.Tensor, src, stream) -> None:
        arr = src if isinstance(src, np.ndarray) else src.numpy()
        arr = np.ascontiguousarray(arr)
        nbytes = dst.numel() * dst.element_size()
        if arr.nbytes != nbytes:
            raise ValueError(f"host/device size mismatch {arr.nbytes} != {nbytes}")
        self._check(L.lib().rlk_loader_h2d(self._h, dst.data_ptr(), arr.ctypes.data, nbytes,
                                           L.stream_handle(stream)), "rlk_loader_h2d")

    def d2h(self, dst, src: torch.Tensor, stream) -> None:
        arr = dst if isinstance(dst, np.ndarray) else dst.numpy()
        nbytes = src.numel() * src.element_size()
        if arr.nbytes != nbytes or not arr.flags.c_contiguous:
            raise ValueError("host output must be a contiguous buffer of the device tensor's size")
        self._check(L.lib().rlk_loader_d2h(self._h, arr.ctypes.data, src.data_ptr(), nbytes,
                                           L.stream_handle(stream)), "rlk_loader_d2h")

    def synth_h2d(self, dst: torch.Tensor, j0: int, base_seed: int, base_std: float, noise_seed: int,
                  noise_std: float, stream) -> None:
        self._check(L.lib().rlk_loader_synth_h2d(self._h, dst.data_ptr(), L.dtype_code(dst.dtype), dst.numel(), j0,
                                                 base_seed, base_std, noise_seed, noise_std,
                                                 L.stream_handle(stream)), "rlk_loader_synth_h2d")

    def d2h_checksum(self, src: torch.Tensor, stream) -> int:
        c = C.c_uint64(0)
        self._check(L.lib().rlk_loader_d2h_checksum(self._h, src.data_ptr(), src.numel() * src.element_size(),
                                                    C.byref(c), L.stream_handle(stream)), "rlk_loader_d2h_checksum")
        return c.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            L.lib().rlk_loader_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


# ----------------------------------------------------------------------------- sources / sinks
class ArraySource:
    """Host arrays: base[name] and experts[i][name] (bf16 as torch CPU tensors or uint16 numpy)."""

    def __init__(self, base: Mapping, experts: Sequence[Mapping]):
        self.base, self.experts = base, experts

    def fill(self, loader: HostLoader, name: str, stream_idx: int, dst: torch.Tensor, stream) -> None:
        src = self.base[name] if stream_idx == 0 else self.experts[stream_idx - 1][name]
        if isinstance(src, torch.Tensor):
            src = src.contiguous().view(torch.int16).numpy() if src.dtype == torch.bfloat16 else src.numpy()
        loader.h2d(dst, np.ascontiguousarray(src).reshape(-1), stream)


class SyntheticSource:
    """Random-init parameters synthesised on the host workers (counter hash; see loader.cpp)."""

    def __init__(self, seed: int = 0, base_std: float = 0.02, expert_std: float = 1e-3):
        self.seed, self.base_std, self.expert_std = seed, base_std, expert_std

    def fill(self, loader: HostLoader, name: str, stream_idx: int, dst: torch.Tensor, stream) -> None:
        from .core import mix64, label_hash
        t = label_hash(name)
        bs = mix64(self.seed ^ t)
        ns = 0 if stream_idx == 0 else mix64(bs + stream_idx)
        loader.synth_h2d(dst, 0, bs, self.base_std, ns, self.expert_std * stream_idx, stream)


class ArraySink:
    def __init__(self, out: Mapping):
        self.out = out
        # page-locked outputs are written by direct async DMA; anything else is staged synchronously
        self.blocking = not all(isinstance(v, torch.Tensor) and v.is_pinned() for v in out.values())

    def drain(self, loader: HostLoader, name: str, src: torch.Tensor, stream) -> None:
        dst = self.out[name]
        if isinstance(dst, torch.Tensor):
            dst = dst.view(torch.int16).numpy() if dst.dtype == torch.bfloat16 else dst.numpy()
        loader.d2h(dst.reshape(-1), src, stream)


class ChecksumSink:
    """Keeps a 64-bit checksum per tensor instead of the fused values (for outputs larger than RAM)."""

    blocking = True  # host pass over every chunk

    def __init__(self):
        self.sums: dict[str, int] = {}

    def drain(self, loader: HostLoader, name: str, src: torch.Tensor, stream) -> None:
        nb = src.numel() * src.element_size()
        main = nb - nb % 8
        flat = src.view(torch.uint8)[:main] if main else None
        s = loader.d2h_checksum(flat, stream) if main else 0
        self.sums[name] = s


# ----------------------------------------------------------------------------- driver
@dataclass
class StreamingReport:
    stats: dict[str, FusionStats] = field(default_factory=dict)
    groups: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    passthrough: list = field(default_factory=list)  # tensors no expert changed (written as the base)
    tensors: int = 0  # tensors this rank streamed
    params: int = 0
    error: str | None = None  # a sharded rank's validation failure, raised after the gather


def plan_groups(numels: Sequence[int], n_experts: int, esize: int, budget_bytes: int) -> list[list[int]]:
    """Consecutive tensor groups whose (N+1 inputs + output) bytes fit `budget_bytes` each."""
    groups, cur, cur_b = [], [], 0
    for t, n in enumerate(numels):
        b = _footprint(n, n_experts, esize)
        if b > budget_bytes:
            raise ValueError(f"tensor {t} ({n} elements) does not fit the workspace; raise the budget")
        if cur and cur_b + b > budget_bytes:
            groups.append(cur)
            cur, cur_b = [], 0
        cur.append(t)
        cur_b += b
    if cur:
        groups.append(cur)
    return groups


def ring_placement(sizes: Sequence[int], cap: int) -> tuple[list[int], list[list[int]]]:
    """Place groups of `sizes` elements one after another in a ring of `cap` (wrapping to 0 when a
    group does not fit before the end).  Returns each group's offset and, per group, the earlier groups
    whose space it overwrites (its H2D must wait for their D2H); a group is evicted by the first later
    group that overlaps it."""
    place, waits, live, head = [], [], [], 0
    for gi, size in enumerate(sizes):
        if size > cap:
            raise ValueError(f"group {gi} ({size} elements) exceeds the ring ({cap})")
        if head + size > cap:
            head = 0
        lo, hi = head, head + size
        waits.append([j for j, a, b in live if a < hi and lo < b])
        live = [(j, a, b) for j, a, b in live if not (a < hi and lo < b)] + [(gi, lo, hi)]
        place.append(lo)
        head = hi
    return place, waits


def _footprint(n: int, n_experts: int, esize: int) -> int:
    return (n + 63) // 64 * 64 * esize * (n_experts + 2)


def partition_tensors(numels: Sequence[int], world: int, rank: int) -> list[int]:
    """Rank `rank`'s tensors for streamed fusion: contiguous runs of whole tensors balanced by element
    count (a cut falls at the first tensor boundary at or after k/world of the elements).  Norms are
    per tensor, so whole-tensor shards need no collective at all (config 4)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    total = sum(numels)
    cuts, acc, t = [0], 0, 0
    for r in range(1, world):
        target = total * r / world
        while t < len(numels) and acc + numels[t] / 2 < target:  # cut nearest the target
            acc += numels[t]
            t += 1
        cuts.append(max(t, cuts[-1]))
    cuts.append(len(numels))
    return list(range(cuts[rank], cuts[rank + 1]))


def fuse_streaming(names: Sequence[str], numels: Sequence[int], n_experts: int, source, sink,
                   cfg: FusionConfig = FusionConfig(), dtype: torch.dtype = torch.bfloat16,
                   device_budget_bytes: int = 64 << 30, stats: bool = True,
                   loader: HostLoader | None = None, group_bytes: int = 2 << 30,
                   on_unchanged: str = "passthrough", world: int = 1, rank: int = 0,
                   group=None, _defer_errors: bool = False) -> StreamingReport:
    """Fuse a host-resident (or synthesised) checkpoint through the device in pipelined groups.

    Consecutive tensors are grouped up to min(`group_bytes`, half the budget) of device footprint
    ((N+1) inputs + output; a larger tensor is a group of its own) and placed one after another in a ring buffer of
    `device_budget_bytes`.  Three streams: H2D of group g + 1, the fusion kernels of group g and the
    D2H of group g - 1 run concurrently (PCIe is full duplex); a group's H2D waits (on events, not on
    the host) for the D2H of every earlier group whose ring space it reuses.  Pinned host
    sources/sinks are DMA'd directly; pageable ones go through the loader's pinned slots.  Blocking
    sinks (pageable outputs, checksums) run on a worker thread with their own loader, overlapping the
    main thread's H2D staging.

    After the last group: non-finite inputs raise ValueError("logits must be finite"); tensors no
    expert changed are listed in `report.passthrough` (written as the base), or raise the reference's
    "cannot take mean norm of all-zero task vectors" with on_unchanged="raise".

    Multi-GPU (one process per GPU): with `world` > 1 this rank streams only its whole-tensor share
    (`partition_tensors`) -- every rank reads its own slice of the checkpoint over its own PCIe link and
    no parameter data or norm crosses GPUs.  With a process group the per-tensor statistics (and the
    validation outcome) are gathered so every rank returns the full report."""
    if on_unchanged not in ("passthrough", "raise"):
        raise ValueError("on_unchanged must be 'passthrough' or 'raise'")
    if group is not None:
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world > 1:
        mine = partition_tensors(numels, world, rank)
        rep = fuse_streaming([names[t] for t in mine], [numels[t] for t in mine], n_experts, source, sink, cfg,
                             dtype, device_budget_bytes, stats, loader, group_bytes, "passthrough",
                             _defer_errors=True) if mine else StreamingReport()
        rep.tensors = len(mine)
        rep.params = sum(numels[t] for t in mine)
        if group is not None:
            import torch.distributed as dist
            parts = [None] * world
            dist.all_gather_object(parts, (rep.stats, rep.passthrough, rep.error), group=group)
            errs = [e for _, _, e in parts if e]
            if errs:
                raise ValueError(errs[0])
            rep.stats = {k: v for st, _, _ in parts for k, v in st.items()}
            rep.passthrough = [n for _, pt, _ in parts for n in pt]
        elif rep.error:
            raise ValueError(rep.error)
        if rep.passthrough and on_unchanged == "raise":
            raise ValueError("cannot take mean norm of all-zero task vectors")
        return rep
    dev = torch.device("cuda", torch.cuda.current_device())
    esize = torch.tensor([], dtype=dtype).element_size()
    cap = device_budget_bytes // esize // 64 * 64  # ring capacity in elements
    biggest = max(_footprint(n, n_experts, esize) for n in numels) // esize
    if biggest > cap:
        raise ValueError("the largest tensor does not fit the device budget; raise the budget")
    # groups of at most half the ring, so that one can stream in while the previous one computes
    groups = plan_groups(numels, n_experts, esize, max(min(group_bytes, device_budget_bytes // 2), biggest * esize))
    sizes = [sum(_footprint(numels[t], n_experts, esize) for t in g) // esize for g in groups]
    place, waits = ring_placement(sizes, cap)
    ring = torch.empty(min(cap, max(p + z for p, z in zip(place, sizes))), dtype=dtype, device=dev)
    own_loader = loader is None
    loader = loader or HostLoader()
    h2d_s, comp_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    weights = cfg.merge_weights or tuple(1.0 / n_experts for _ in range(n_experts))
    rep = StreamingReport(groups=len(groups))

    def build(gi, group):
        off = place[gi]
        pieces, views_all = [], []
        for k, t in enumerate(group):
            n = numels[t]
            views = []
            for _ in range(n_experts + 2):
                views.append(ring[off:off + n])
                off += (n + 63) // 64 * 64  # keep 128-byte alignment
            pieces.append(Piece(k, 0, views[0], views[1:n_experts + 1], views[-1]))
            views_all.append(views)
        layout = FusionLayout([numels[t] for t in group])
        return group, views_all, FusionCall(pieces, layout, n_experts, cfg, stream=comp_s, async_upload=False)

    # every launch plan is built before the first bulk copy: its small blocking uploads must not queue
    # behind gigabytes of H2D traffic (and pinned staging for them would not recycle in time)
    plans = [build(gi, group) for gi, group in enumerate(groups)]
    # Sinks run on a worker thread with a loader of their own: a pageable sink's staged D2H (and a
    # checksum sink's host pass) then overlaps the main thread's staging of the next groups' H2D,
    # instead of leaving PCIe idle in between (ctypes releases the GIL inside the C calls).
    # Sinks that block the host (pageable outputs, checksums) do not need the host thread that stages
    # H2D: with a non-blocking sink (page-locked outputs, direct DMA) everything stays on this thread.
    import concurrent.futures as cf
    blocking = getattr(sink, "blocking", True)
    drain_pool = cf.ThreadPoolExecutor(max_workers=1) if blocking else None
    drain_loader = HostLoader() if blocking else loader
    freed: dict[int, cf.Future] = {}  # group -> future of the event marking its D2H complete
    pending = None  # (group index, out views, compute-done event)

    def drain_on_worker(pend):
        with torch.cuda.device(dev):  # the worker thread's current device is not inherited
            return _drain(pend, drain_loader, sink, d2h_s, names, rep, groups)

    def drain_async(pend):
        if drain_pool is None:
            f = cf.Future()
            f.set_result(_drain(pend, loader, sink, d2h_s, names, rep, groups))
            return f
        return drain_pool.submit(drain_on_worker, pend)

    try:
        for gi, (group, views_all, call) in enumerate(plans):
            for j in waits[gi]:
                if pending is not None and pending[0] == j:  # ring too small to overlap: drain now
                    freed[j] = drain_async(pending)
                    pending = None
                h2d_s.wait_event(freed.pop(j).result())
            for t, views in zip(group, views_all):
                for si in range(n_experts + 1):
                    source.fill(loader, names[t], si, views[si], h2d_s)
                    rep.h2d_bytes += numels[t] * esize
            ready = torch.cuda.Event()
            ready.record(h2d_s)
            comp_s.wait_event(ready)
            with L.nvtx_range(f"rlk.stream_group.{gi}"):
                call.run(weights)
            done = torch.cuda.Event()
            done.record(comp_s)
            # drain the previous group while this one computes
            if pending is not None:
                freed[pending[0]] = drain_async(pending)
            pending = (gi, [v[-1] for v in views_all], done)
        if pending is not None:
            freed[pending[0]] = drain_async(pending)
        for f in freed.values():
            f.result()  # re-raises a sink error
        torch.cuda.synchronize(dev)
        # finalize's per-tensor status (fusion.cu k_finalize): 2 = non-finite input (the reference's
        # ParamTable rejects it, toy_env.py:71-72), 1 = no expert changed the tensor (the reference's
        # per-tensor fuse raises, fusion.py:97-98; the state-dict path writes the base unchanged)
        bad, unchanged = [], []
        for group, _, call in plans:
            for t, st in zip(group, call.status.cpu().tolist()):
                if st == 2:
                    bad.append(names[t])
                elif st == 1:
                    unchanged.append(names[t])
        if bad:
            msg = (f"logits must be finite (non-finite values in {bad[:8]}"
                   f"{' ...' if len(bad) > 8 else ''})")
            if _defer_errors:  # a sharded caller reports it after every rank is done (no rank left hanging)
                rep.error = msg
            else:
                raise ValueError(msg)
        if unchanged and on_unchanged == "raise":
            raise ValueError("cannot take mean norm of all-zero task vectors")
        rep.passthrough = unchanged
        if stats:
            for group, _, call in plans:
                host = call.host_tables()
                for k, t in enumerate(group):
                    rep.stats[names[t]] = call.stats(k, weights, host=host)
    finally:
        if drain_pool is not None:
            drain_pool.shutdown(wait=True)
            drain_loader.close()
        if own_loader:
            loader.close()
    return rep


def _drain(pending, loader, sink, d2h_s, names, rep, groups) -> torch.cuda.Event:
    gi, outs, done = pending
    d2h_s.wait_event(done)
    for t, o in zip(groups[gi], outs):
        sink.drain(loader, names[t], o, d2h_s)
        rep.d2h_bytes += o.numel() * o.element_size()
    ev = torch.cuda.Event()
    ev.record(d2h_s)
    return ev
