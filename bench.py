#!/usr/bin/env python
"""Benchmark of the B200 fusion + GRPO-loss hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

Headline workload (BASELINE.json configs[2], the 1/2/4/8-GPU config; it fits one GPU): 3 domain experts +
base, Llama-3-8B-shaped bf16 state dict (291 tensors, 8.03e9 params), FusionConfig(dropout_p=0.5,
seed=42) -- normalise + DARE dropout + sign erase + weighted merge -- sharded by parameter range
(strong scaling); the only cross-GPU traffic is the NCCL all_reduce of the norm partials.

A step = one complete fusion (K1 norm partials -> all_reduce -> finalize -> K2 dropout bitmap -> K3
merge) over inputs resident in HBM (80 GB >> 126 MB L2, so no L2 flush is needed).  `e2e` repeats it
through the public API with HOST (pinned) buffers: H2D of base + experts and D2H of the fused output
inside the timed region.  GRPO token loss (config 5: V=131072, one group of 16 x 32768-token
responses) is reported under "grpo".  The CPU baseline is the oracle port (oracle/) on a bounded
sample, rank 0 at N=1 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fusion params/s & HBM GB/s (%roofline) at 1/2/4/8 B200; GRPO loss tokens/s"
N_EXPERTS = 3
# K3 is launched through rlk_fusion_merge_ws (merge + fix-up queue); its per-call CUDA-event time
# includes the fix-up kernel.  profiles/traffic.json keys the ncu traffic by the kernel family.
MERGE_CALL = "rlk_fusion_merge_ws"
TRAFFIC_KEY = {MERGE_CALL: "rlk_fusion_merge"}


def measured_peak_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during a timed region."""

    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        rows = [r for r in self.samples if len(r) == len(self.FIELDS)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in rows:
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][2]),
                "reasons": sorted(reasons), "samples": len(rows)}


# ----------------------------------------------------------------------------------- distributed
def _backend_name(group) -> str:
    import torch.distributed as dist
    return str(dist.get_backend(group)).upper()


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return rank, world, local, None
    # RLK_BENCH_BACKEND=gloo runs the N > 1 code path with every rank on the visible GPUs round-robin
    # (a functional check of the sharded bench on a one-GPU box; NCCL refuses two ranks per GPU).
    backend = os.environ.get("RLK_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
    return rank, world, local, group


def max_over_ranks(values, group):
    import torch
    t = torch.tensor(values, dtype=torch.float64, device="cuda")
    if group is not None:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()


def sum_over_ranks(values, group):
    import torch
    t = torch.tensor(values, dtype=torch.float64, device="cuda")
    if group is not None:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.tolist()


def barrier(group):
    if group is not None:
        import torch.distributed as dist
        dist.barrier(group=group)


# ----------------------------------------------------------------------------------- fusion
def local_params_of(pieces) -> int:
    return sum(p.numel for p in pieces)


def fusion_bench(args, rank, world, local, group):
    import torch
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.layouts import LAYOUTS, fill_synthetic, numel

    shapes = LAYOUTS[args.layout]()
    numels = [numel(s) for s in shapes.values()]
    layout = F.FusionLayout(numels)
    dev = torch.device("cuda", local)
    dt = {"bf16": torch.bfloat16, "f32": torch.float32}[args.dtype]
    stream = torch.cuda.Stream(dev)
    pieces = []
    with torch.cuda.stream(stream):
        for t, lo, hi in layout.partition_striped(world, rank):
            n = hi - lo
            b = torch.empty(n, dtype=dt, device=dev)
            es = [torch.empty(n, dtype=dt, device=dev) for _ in range(N_EXPERTS)]
            fill_synthetic(b, es, t, j0=lo, seed=0, stream=stream)
            pieces.append(F.Piece(t, lo, b, es, torch.empty(n, dtype=dt, device=dev)))
    stream.synchronize()
    local_params = sum(p.numel for p in pieces)
    cfg = F.FusionConfig(dropout_p=args.dropout, seed=42)
    weights = tuple(1.0 / N_EXPERTS for _ in range(N_EXPERTS))
    call = F.FusionCall(pieces, layout, N_EXPERTS, cfg, group=group, stream=stream)

    # inputs smaller than ~2x L2 (config 1): flush L2 between timed steps (a 512 MiB write, outside
    # the per-step events); larger inputs stream through L2 on their own
    in_bytes = local_params_of(pieces) * dt.itemsize * (N_EXPERTS + 1)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if in_bytes < (256 << 20) else None

    graph = None

    def step(profile):
        if graph is not None and not profile:
            with torch.cuda.stream(stream):
                graph.replay()
        else:
            call.run(weights)

    def timed(steps, profile):
        call.timers = {} if profile else None
        barrier(group)
        torch.cuda.synchronize(dev)
        if flush is None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                step(profile)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            barrier(group)
            return e0.elapsed_time(e1) / steps
        evs = []
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(profile)
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize(dev)
        barrier(group)
        return sum(a.elapsed_time(b) for a, b in evs) / steps

    for _ in range(args.warmup):
        call.run(weights)
    if group is None and not args.no_graph:
        # one CUDA graph per step (K2, K1, finalize, K3 and the counter reset): the timed loop replays it
        graph = call.capture(weights)
        for _ in range(2):
            step(False)
    with ClockSampler(local) as clk:
        ms = timed(args.steps, profile=False)
    clocks = clk.summary()
    # per-kernel durations on the launching stream (separate pass so the headline has no extra events)
    timed(max(3, min(args.steps, 10)), profile=True)  # nprof steps
    nprof = max(3, min(args.steps, 10))
    # per-step kernel time (a sharded K2 may be several range launches per step)
    kern = {name: sum(a.elapsed_time(b) for a, b in evs) / nprof for name, evs in call.timers.items()}
    launches = sum(len(evs) for evs in call.timers.values()) // nprof
    launches += 1 if getattr(call, "_ws", None) is not None else 0  # rlk_fusion_merge_ws: merge + fix-up kernel
    call.timers = None
    ms_max, = max_over_ranks([ms], group)
    kmax = dict(zip(kern.keys(), max_over_ranks(list(kern.values()), group)))
    st = call.check_status(per_tensor_raise=False)
    nonfinite = int((st == 2).sum())
    res = dict(ms=ms_max, ms_local=ms, kern_local=kern, kern_max=kmax, local_params=local_params,
               launch=("one CUDA-graph replay per step (FusionCall.capture)" if graph is not None else "eager launches"),
               l2=("L2 flushed (512 MiB write) before every timed step; inputs "
                   f"{in_bytes / 2**20:.0f} MiB" if flush is not None else
                   f"inputs {in_bytes / 1e9:.0f} GB >> 126 MB L2; no flush needed"),
               total_params=layout.total, n_tensors=layout.n_tensors, clocks=clocks, nonfinite=nonfinite,
               dropout_mode=call.dropout_mode, launches_per_step=launches)

    # SURVEY 8(d) variants on the same buffers: p = 0 (the reference default config), squared-vote
    # erasure, seed 0, and no normalisation (target_norm=None; K1 still runs: FusionStats.norms_before)
    if not args.quick:
        res["variants"] = {}
        for vname, vcfg in (("p0_default_cfg", F.FusionConfig()),
                            ("p05_squared_erase", F.FusionConfig(dropout_p=0.5, seed=42, erase_weighting="squared")),
                            ("p05_seed0", F.FusionConfig(dropout_p=0.5, seed=0)),
                            ("p05_no_normalize", F.FusionConfig(dropout_p=0.5, seed=42, target_norm=None))):
            call0 = F.FusionCall(pieces, layout, N_EXPERTS, vcfg, group=group, stream=stream)
            for _ in range(2):
                call0.run(weights)
            barrier(group)
            torch.cuda.synchronize(dev)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(args.steps):
                call0.run(weights)
            a1.record(stream)
            torch.cuda.synchronize(dev)
            ms0, = max_over_ranks([a0.elapsed_time(a1) / args.steps], group)
            res["variants"][vname] = ms0
            del call0

    cfg_run = call.cfg
    del call, pieces
    torch.cuda.empty_cache()
    # e2e through the public API with pinned host buffers
    if not args.no_e2e:
        res.update(fusion_e2e(args, layout, cfg_run, stream, dev, rank, world, group))
        torch.cuda.empty_cache()
    return res


def fusion_e2e(args, layout, cfg, stream, dev, rank, world, group):
    """End to end through the public API (loader.fuse_streaming) from pinned host memory, every step:
    H2D of base + experts, fusion, D2H of the fused output, in tensor groups on three streams -- H2D of
    group g+1, K2/K1/finalize/K3 of group g and D2H of group g-1 overlap (per-tensor norms only need the
    tensor's own data).  Under torchrun every rank streams its whole-tensor share
    (`loader.partition_tensors`) over its own link: no parameter data or norm crosses GPUs."""
    import torch
    from paper_2509_18883_b200.layouts import fill_synthetic
    from paper_2509_18883_b200.loader import ArraySink, ArraySource, fuse_streaming, partition_tensors
    dt = {"bf16": torch.bfloat16, "f32": torch.float32}[args.dtype]
    numels = list(layout.numels)
    names = [str(t) for t in range(len(numels))]
    mine = partition_tensors(numels, world, rank)
    hb, he, ho = {}, [dict() for _ in range(N_EXPERTS)], {}
    with torch.cuda.stream(stream):
        for t in mine:  # the same synthetic values as the in-HBM step, generated on the device, pinned on the host
            n = numels[t]
            b = torch.empty(n, dtype=dt, device=dev)
            es = [torch.empty(n, dtype=dt, device=dev) for _ in range(N_EXPERTS)]
            fill_synthetic(b, es, t, j0=0, seed=0, stream=stream)
            hb[names[t]] = torch.empty(n, dtype=dt, pin_memory=True)
            hb[names[t]].copy_(b, non_blocking=True)
            for i in range(N_EXPERTS):
                he[i][names[t]] = torch.empty(n, dtype=dt, pin_memory=True)
                he[i][names[t]].copy_(es[i], non_blocking=True)
            ho[names[t]] = torch.empty(n, dtype=dt, pin_memory=True)
            stream.synchronize()
            del b, es
    mine_params = sum(numels[t] for t in mine)

    def step():
        with torch.cuda.stream(stream):
            fuse_streaming(names, numels, N_EXPERTS, ArraySource(hb, he), ArraySink(ho), cfg, dtype=dt,
                           device_budget_bytes=int(args.e2e_budget_gb * (1 << 30)), group_bytes=2 << 30,
                           world=world, rank=rank)

    steps, warm = max(1, min(args.steps, args.e2e_steps)), 1
    for _ in range(warm):
        step()
    barrier(group)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier(group)
    ms, = max_over_ranks([e0.elapsed_time(e1) / steps], group)
    es_ = dt.itemsize
    h2d, d2h = sum_over_ranks([float(mine_params * es_ * (N_EXPERTS + 1)), float(mine_params * es_)], group)
    del hb, he, ho
    return dict(e2e_ms=ms, e2e_steps=steps, e2e_warmup=warm, h2d=int(h2d), d2h=int(d2h),
                e2e_path=("loader.fuse_streaming (public API): pinned host dicts, 2 GiB tensor groups, "
                          "H2D | fuse | D2H on 3 streams, FusionStats returned"
                          + (f"; whole-tensor shards x{world}, one PCIe link per rank" if world > 1 else "")))


# ----------------------------------------------------------------------------------- GRPO
def grpo_bench(args, rank, world, local, group):
    """Config 5: V = 131072, one group of G = 16 responses x T = 32768 tokens, responses split over ranks."""
    import numpy as np
    import torch
    from paper_2509_18883_b200 import _lib as L
    from paper_2509_18883_b200 import objective as O

    V, G, T = 131072, 16, args.grpo_tokens
    mine = [r for r in range(G) if r % world == rank]
    chunk = min(2, len(mine))
    rows = chunk * T
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    logits = torch.empty((rows, V), dtype=torch.bfloat16, device=dev)
    L.call("rlk_synth_normal", L.ptr(logits), L.RLK_BF16, logits.numel(), 0, 1234 + rank, 2.0, None,
           L.stream_handle(stream))
    g = np.random.default_rng(rank)
    toks = g.integers(0, V, rows)
    lt = g.normal(-12.0, 0.3, rows)
    li = lt + g.normal(0, 0.05, rows)
    adv = np.where(np.arange(chunk) % 2 == 0, 1.0, -1.0)
    batch = O.GRPOBatch.pack(toks, lt, li, np.arange(chunk + 1) * T, adv, np.ones(chunk, np.uint8), chunk, T,
                             device=dev)
    n_chunks = (len(mine) + chunk - 1) // chunk
    torch.cuda.synchronize(dev)

    def run(bwd: bool, events=None):
        for _ in range(n_chunks):
            a = b = None
            if events is not None:
                a = torch.cuda.Event(enable_timing=True)
                a.record(stream)
            if bwd:  # loss + gradient in one read of the logits (rlk_grpo_fused_bf16, 2-CTA clusters)
                O.grpo_forward_backward(logits, batch, stream=stream)
            else:
                O.grpo_forward(logits, batch, stream=stream)
            if events is not None:
                b = torch.cuda.Event(enable_timing=True)
                b.record(stream)
                events.setdefault("rlk_grpo_fused_bf16" if bwd else "rlk_grpo_fwd", []).append((a, b))

    out = {}
    for bwd in (False, True):
        for _ in range(args.warmup):
            run(bwd)
        barrier(group)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            run(bwd)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier(group)
        ms, = max_over_ranks([e0.elapsed_time(e1) / args.steps], group)
        out["fwdbwd_ms" if bwd else "fwd_ms"] = ms
    ev = {}
    run(False, ev)
    run(True, ev)
    torch.cuda.synchronize(dev)
    kern = {k: statistics.mean(a.elapsed_time(b) for a, b in v) for k, v in ev.items()}
    kmax = dict(zip(kern, max_over_ranks(list(kern.values()), group)))
    out.update(kern=kmax, rows_per_launch=rows, tokens=G * T, V=V)

    # SURVEY 8(d) variants (not in the headline): temperature 0.7; 2 of 16 samples masked (12.5 %);
    # ragged lengths ~ U[T/2, T] (seeded).  Tokens counted = unmasked tokens actually read.
    if not args.quick:
        lens_rng = np.random.default_rng(100 + rank)

        def variant(tau=1.0, masked=(), ragged=False):
            plans, counted = [], 0
            for k in range(n_chunks):
                samples = mine[k * chunk:(k + 1) * chunk]
                lens = (lens_rng.integers(T // 2, T + 1, len(samples)) if ragged else np.full(len(samples), T))
                use = np.array([0 if sidx in masked else 1 for sidx in samples], np.uint8)
                counted += int(sum(n for n, u in zip(lens, use) if u))
                n_rows = int(lens.sum())
                bt = O.GRPOBatch.pack(toks[:n_rows], lt[:n_rows], li[:n_rows], np.concatenate([[0], np.cumsum(lens)]),
                                      adv[:len(samples)], use, len(samples), T, temperature=tau, device=dev)
                plans.append((logits[:n_rows], bt))
            res = {}
            for bwd in (False, True):
                def once():
                    for lg, bt in plans:
                        (O.grpo_forward_backward if bwd else O.grpo_forward)(lg, bt, stream=stream)
                for _ in range(args.warmup):
                    once()
                barrier(group)
                torch.cuda.synchronize(dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(args.steps):
                    once()
                e1.record(stream)
                torch.cuda.synchronize(dev)
                ms, = max_over_ranks([e0.elapsed_time(e1) / args.steps], group)
                res["fwd_bwd_ms" if bwd else "fwd_ms"] = ms
            tot, = sum_over_ranks([counted], group)
            res.update(tokens_counted=tot, tokens_per_s=tot / (res["fwd_ms"] / 1e3),
                       fwd_bwd_tokens_per_s=tot / (res["fwd_bwd_ms"] / 1e3))
            return res

        out["variants"] = {"tau_0.7": variant(tau=0.7), "masked_12.5pct": variant(masked=(3, 11)),
                           "ragged_lengths": variant(ragged=True)}
    del logits
    torch.cuda.empty_cache()
    if not args.quick:
        out["variants"]["f32_logits"] = grpo_f32_variant(args, batch, rows, V, n_chunks, G * T, stream, dev, group)
    return out


def grpo_f32_variant(args, batch, rows, V, n_chunks, tokens, stream, dev, group) -> dict:
    """Config 5 with f32 logits (as trainers that upcast the LM head produce): the one-read fused loss +
    gradient on 4-CTA clusters (8 B/logit: f32 read + f32 grad write) against K4 + K5 (12 B/logit)."""
    import torch
    from paper_2509_18883_b200 import _lib as L
    from paper_2509_18883_b200 import objective as O
    lg = torch.empty((rows, V), dtype=torch.float32, device=dev)
    L.call("rlk_synth_normal", L.ptr(lg), L.RLK_F32, lg.numel(), 0, 4321, 2.0, None, L.stream_handle(stream))
    res = {}
    for name, fn in (("fused", lambda: O.grpo_forward_backward(lg, batch, stream=stream)),
                     ("k4_k5", lambda: O.grpo_backward(lg, batch, O.grpo_forward(lg, batch, stream=stream),
                                                       stream=stream))):
        for _ in range(args.warmup):
            fn()
        barrier(group)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            for _ in range(n_chunks):
                fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms, = max_over_ranks([e0.elapsed_time(e1) / args.steps], group)
        res[f"{name}_ms"] = ms
        res[f"{name}_tokens_per_s"] = tokens / (ms / 1e3)
    peak, _ = measured_peak_gbs()
    per_launch = res["fused_ms"] / n_chunks
    res["fused_roofline"] = {"bytes_per_token": V * 8, "achieved": rows * V * 8 / (per_launch / 1e3) / 1e9,
                             "peak": peak, "unit": "GB/s",
                             "frac": rows * V * 8 / (per_launch / 1e3) / 1e9 / peak}
    del lg
    torch.cuda.empty_cache()
    return res


# ----------------------------------------------------------------------------------- CPU baseline
# ----------------------------------------------------------------------------- config 4 (streamed)
def pcie_h2d_peak_gbs(dev, nbytes: int = 1 << 30, reps: int = 5) -> float:
    """Bare pinned host -> device copy bandwidth on this rank's link (the streaming bound)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize(dev)
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


class PinnedPoolSource:
    """A checkpoint already resident in page-locked host memory: every (tensor, stream) is a slice of
    one pinned pool of synthetic bf16 values at a hashed offset, DMA'd directly (the loader's pinned
    path).  Host-side synthesis (loader.SyntheticSource) runs at ~1 GB/s on this host, far below the
    link, so it would measure the CPU, not the streaming path."""

    def __init__(self, pool_elems: int = 1 << 31, seed: int = 0):
        import numpy as np
        import torch
        g = np.random.default_rng(seed)
        vals = (g.standard_normal(pool_elems // 16, dtype=np.float32) * 0.02).view(np.uint32) >> 16
        self.pool = torch.from_numpy(np.tile(vals.astype(np.uint16).view(np.int16), 16)).pin_memory()
        self.n = pool_elems

    def fill(self, loader, name, si, dst, stream):
        import zlib
        n = dst.numel()
        off = (zlib.crc32(f"{name}/{si}".encode()) * 4099) % max(1, self.n - n) & ~63
        loader.h2d(dst, self.pool[off:off + n].numpy(), stream)


def stream_bench(args, rank, world, local, group, peak, peak_src) -> dict | None:
    """BASELINE.json configs[3]: LongCat-Flash-560B-MoE-shaped random-init experts (layouts.longcat_560b,
    `--stream-layers` of its 28 layers + embeddings/head), fused by streaming tensor groups through
    pinned host buffers (K7).  Host workers synthesise base + 3 experts (counter hash) straight into
    pinned slots; outputs are checksummed on the way back (larger than RAM).  Under torchrun every
    rank streams its whole-tensor share (`loader.partition_tensors`) over its own PCIe link: no
    parameter data or norm crosses GPUs.  A step = one complete streamed fusion of the slice."""
    import torch
    from paper_2509_18883_b200 import fusion as F
    from paper_2509_18883_b200.layouts import longcat_560b, numel
    from paper_2509_18883_b200.loader import (ChecksumSink, HostLoader, SyntheticSource, fuse_streaming,
                                              partition_tensors)
    dev = torch.device("cuda", local)
    shapes = longcat_560b(n_layers=args.stream_layers)
    names = list(shapes)
    numels = [numel(s) for s in shapes.values()]
    total = sum(numels)
    full = sum(numel(s) for s in longcat_560b().values())
    mine = sum(numels[t] for t in partition_tensors(numels, world, rank))
    pcie = pcie_h2d_peak_gbs(dev)
    cfg = F.FusionConfig(dropout_p=args.dropout, seed=42)
    ld = HostLoader(slot_bytes=64 << 20, n_slots=6)
    src = SyntheticSource() if args.stream_source == "synth" else PinnedPoolSource()
    sink = ChecksumSink()

    def step():
        return fuse_streaming(names, numels, N_EXPERTS, src, sink, cfg, device_budget_bytes=48 << 30, stats=False,
                              loader=ld, world=world, rank=rank)

    for _ in range(args.warmup):
        step()
    times, reps = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            barrier(group)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            reps.append(step())  # returns after its final device synchronize
            times.append(time.perf_counter() - t0)
    ld.close()
    sec = statistics.mean(times)
    h2d = reps[-1].h2d_bytes
    h2d_gbs = h2d / sec / 1e9
    sec_max, = max_over_ranks([sec], group)
    per_rank = [0.0] * world
    vals = torch.zeros(world, 3, dtype=torch.float64, device=dev)
    vals[rank] = torch.tensor([h2d_gbs, pcie, mine], dtype=torch.float64)
    if group is not None:
        import torch.distributed as dist
        dist.all_reduce(vals, group=group)
    per_rank = vals.cpu().tolist()
    if rank != 0:
        return None
    alg = total * (2 * (N_EXPERTS + 1) * 2 + 2)  # 18 B/param of HBM traffic
    return {
        "metric": METRIC, "value": total / sec_max, "unit": "params/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec_max * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init bf16 values in host memory)",
        "config": {"workload": f"config4: LongCat-Flash-560B-MoE-shaped bf16 (layouts.longcat_560b, "
                               f"{args.stream_layers} of 28 layers + embeddings/head: {total} params, {len(numels)} "
                               f"tensors; full model {full}), 3 experts + base, FusionConfig(dropout_p={args.dropout}, "
                               f"seed=42), streamed from host ({'host-synthesised' if args.stream_source == 'synth' else 'pinned pool'} "
                               f"source, checksum sink), whole-tensor shards x{world}",
                   "timing": "wall clock around each complete streamed step (host synthesis, H2D, kernels, D2H "
                             "and the final device synchronize), max over ranks"},
        "stream": {"h2d_bytes_per_step_rank0": h2d, "h2d_gbs_per_rank": [r[0] for r in per_rank],
                   "pcie_h2d_peak_gbs_per_rank": [r[1] for r in per_rank],
                   "h2d_frac_of_pcie_peak": [r[0] / r[1] for r in per_rank],
                   "params_per_rank": [int(r[2]) for r in per_rank],
                   "hbm_gbs": alg / sec_max / 1e9, "hbm_frac": alg / sec_max / 1e9 / peak,
                   "hbm_peak": peak, "hbm_peak_source": peak_src,
                   "projected_full_model_s": full / (total / sec_max)},
        "clocks": clk.summary(),
        "e2e": {"value": total / sec_max, "unit": "params/s", "h2d_bytes_per_step": int(total * 2 * (N_EXPERTS + 1)),
                "d2h_bytes_per_step": int(total * 2)},
    }


def _cpu_job(args):
    """One oracle fuse over a slice of a synthetic bf16-valued tensor (f64 math, like the reference)."""
    import numpy as np
    from oracle import fusion as OF
    t, n, p, seed = args
    g = np.random.default_rng([seed, t])
    b = g.normal(0, 0.02, n).astype(np.float32).astype(np.float64)
    es = [b + g.normal(0, 1e-3 * (i + 1), n) for i in range(N_EXPERTS)]
    t0 = time.perf_counter()
    OF.fuse(b, es, dropout_p=p, seed=42)
    return time.perf_counter() - t0, n


def cpu_baseline(layout_name: str, p: float, cores: int | None = None, slice_elems: int = 4 << 20,
                 max_params: int = 112 << 20) -> dict:
    """Oracle port on one transformer layer of the layout (4M-element slices), one process per core."""
    import concurrent.futures as cf
    from paper_2509_18883_b200.layouts import LAYOUTS, numel
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    shapes = LAYOUTS[layout_name]()
    layer = [(k, numel(s)) for k, s in shapes.items() if ".0." in k or k.startswith("h.0.")] or list(
        (k, numel(s)) for k, s in shapes.items())
    jobs = []
    for t, (name, n) in enumerate(layer):
        for lo in range(0, n, slice_elems):
            if sum(j[1] for j in jobs) >= max_params:
                break
            jobs.append((t, min(slice_elems, n - lo), p, lo))
    cores = cores or os.cpu_count() or 1
    t0 = time.perf_counter()
    with cf.ProcessPoolExecutor(max_workers=cores) as ex:
        res = list(ex.map(_cpu_job, jobs))
    wall = time.perf_counter() - t0
    cpu_s = sum(r[0] for r in res)
    params = sum(r[1] for r in res)
    per_core = params / cpu_s
    return {"value": per_core * cores, "unit": "params/s", "cores": cores, "kind": "port",
            "per_core": per_core, "cpu_seconds": cpu_s, "wall_s_incl_datagen": wall,
            "sample": f"oracle fuse (numpy f64, FusionConfig(dropout_p={p}, seed=42)) on layer 0 of {layout_name}: "
                      f"{params / 1e6:.1f}M params (first slices) in {len(jobs)} slices of <=4M elements, one process per core; "
                      f"value = per-core rate (sum params / sum compute seconds) x cores (extrapolated, ideal scaling)"}


def _cpu_grpo_job(args):
    """Oracle token terms (numpy f64 log-softmax over V per token, objective.py:243-248) for a few rows."""
    import numpy as np
    from oracle import objective as OO
    seed, rows, V = args
    g = np.random.default_rng(seed)
    z = g.normal(0, 2.0, (rows, V)).astype(np.float32).astype(np.float64)
    toks = g.integers(0, V, rows)
    lt = g.normal(-12, 0.3, rows)
    clip = dict(eps_neg_low=0.2, eps_pos_high=0.2, eps_neg_high=3.0, tis_cap=2.0, guard_positive=True)
    t0 = time.perf_counter()
    OO.token_terms(z, None, toks, lt, lt + 0.01, np.zeros(rows, np.int64), [1.0], [1], [1.0], clip)
    return time.perf_counter() - t0, rows


def grpo_cpu_baseline(V: int = 131072, rows_per_job: int = 64, cores: int | None = None) -> dict:
    """Config-5 GRPO loss on the host: the oracle's per-token log-softmax + triplet/TIS terms, one
    process per core on a bounded sample of rows."""
    import concurrent.futures as cf
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    cores = cores or os.cpu_count() or 1
    jobs = [(k, rows_per_job, V) for k in range(cores)]
    with cf.ProcessPoolExecutor(max_workers=cores) as ex:
        res = list(ex.map(_cpu_grpo_job, jobs))
    cpu_s = sum(r[0] for r in res)
    toks = sum(r[1] for r in res)
    per_core = toks / cpu_s
    return {"value": per_core * cores, "unit": "tokens/s", "cores": cores, "kind": "port", "per_core": per_core,
            "sample": f"oracle token terms (numpy f64, V={V}) on {toks} synthetic rows, {rows_per_job} per process, "
                      "one process per core; value = per-core rate x cores (extrapolated, ideal scaling)"}


# ------------------------------------------------------------- the unmodified reference (rolloutlab)
REF_DIR = ROOT / "baseline" / "_ref"  # `pip install --target baseline/_ref` of /root/reference/pkg (DESIGN 8)


def _import_reference():
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    from rolloutlab import core, fusion, objective, toy_env  # noqa: F401
    return core, fusion, objective, toy_env


def _ref_fuse_job(args):
    """rolloutlab.fusion.fuse, unmodified (its per-element Python dropout loop, fusion.py:105-115), on
    one slice of a synthetic bf16-valued tensor."""
    import numpy as np
    _, fusion, _, toy_env = _import_reference()
    t, n, p = args
    g = np.random.default_rng([7, t])
    b = g.normal(0, 0.02, n).astype(np.float32).astype(np.float64)
    pt = lambda a: toy_env.ParamTable(a.reshape(1, 1, -1))
    base = pt(b)
    es = [pt(b + g.normal(0, 1e-3 * (i + 1), n)) for i in range(N_EXPERTS)]
    t0 = time.perf_counter()
    taus = [fusion.task_vector(e, base) for e in es]
    fusion.fuse(base, taus, fusion.FusionConfig(dropout_p=p, seed=42))
    return time.perf_counter() - t0, n


def _ref_grpo_job(args):
    """rolloutlab.objective.objective_value, unmodified, on one group of G responses over a V-wide
    tabular policy (its per-token numpy log-softmax, toy_env.py:157-175)."""
    import numpy as np
    core, _, objective, toy_env = _import_reference()
    seed, G, T, V = args
    g = np.random.default_rng(seed)
    # one context per response: every token reads its own logits row, as in config 5 (no cache reuse)
    params = toy_env.ParamTable(g.normal(0, 2.0, (G, T, V)))
    samples = []
    for si in range(G):
        toks = tuple(int(x) for x in g.integers(0, V, T))
        lt = tuple(float(x) for x in g.normal(-12.0, 0.3, T))
        li = tuple(x + 0.01 for x in lt)
        rw = core.RewardOutcome.passed() if si % 2 == 0 else core.RewardOutcome.failed()
        samples.append(core.Sample(prompt_id=0, context_id=si, version_id=0, tokens=toks, infer_logps=li,
                                   status=core.SampleStatus.COMPLETE, t_start=0, train_logps=lt, reward=rw,
                                   gen_temperature=1.0))
    batch = objective.apply_masks([core.Group(0, tuple(samples))], T)
    t0 = time.perf_counter()
    objective.objective_value(batch, params, objective.ClipConfig())
    return time.perf_counter() - t0, G * T


def reference_cpu(p: float, cores: int | None = None, fuse_elems: int = 1 << 17, fuse_jobs_per_core: int = 2,
                  grpo_g: int = 4, grpo_t: int = 32) -> dict:
    """Times the UNMODIFIED reference (baseline/_ref) on a bounded sample, one process per core:
    fusion = `fuse` on 131,072-element slices (3 experts, FusionConfig(dropout_p=p, seed=42));
    GRPO = `objective_value` on one group of 4 x 32 tokens at V = 131,072.  Values are per-core rates x
    cores (extrapolated to all cores, ideal scaling)."""
    import concurrent.futures as cf
    try:
        _import_reference()
    except Exception as e:  # not installed on this box
        return {"unavailable": f"rolloutlab not importable from {REF_DIR}: {type(e).__name__}"}
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    cores = cores or os.cpu_count() or 1
    with cf.ProcessPoolExecutor(max_workers=cores) as ex:
        fz = list(ex.map(_ref_fuse_job, [(k, fuse_elems, p) for k in range(cores * fuse_jobs_per_core)]))
        gr = list(ex.map(_ref_grpo_job, [(k, grpo_g, grpo_t, 131072) for k in range(cores)]))
    f_rate = sum(r[1] for r in fz) / sum(r[0] for r in fz)
    g_rate = sum(r[1] for r in gr) / sum(r[0] for r in gr)
    return {
        "kind": "reference", "cores": cores,
        "fusion": {"value": f_rate * cores, "unit": "params/s", "per_core": f_rate,
                   "sample": f"rolloutlab.fusion.fuse unmodified, {len(fz)} slices x {fuse_elems} elements, 3 experts, "
                             f"FusionConfig(dropout_p={p}, seed=42); value = per-core rate x {cores} cores (extrapolated)"},
        "grpo": {"value": g_rate * cores, "unit": "tokens/s", "per_core": g_rate,
                 "sample": f"rolloutlab.objective.objective_value unmodified, {len(gr)} groups of {grpo_g} x {grpo_t} "
                           f"tokens, V=131072; value = per-core rate x {cores} cores (extrapolated)"},
    }


# ----------------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--layout", default="llama8b")
    ap.add_argument("--dtype", choices=["bf16", "f32"], default="bf16", help="parameter dtype (config 1 is f32)")
    ap.add_argument("--dropout", type=float, default=0.5)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-budget-gb", type=float, default=40.0, help="device ring for the streamed e2e step")
    ap.add_argument("--grpo-tokens", type=int, default=32768)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-grpo", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the timed fusion steps eagerly")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--stream", action="store_true",
                    help="config 4: stream --layout longcat560b from host memory (K7) instead of the in-HBM step")
    ap.add_argument("--stream-layers", type=int, default=1, help="layers of the 28-layer longcat560b layout")
    ap.add_argument("--stream-source", choices=["pinned", "synth"], default="pinned")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local, group = dist_setup(args)
    peak, peak_src = measured_peak_gbs()
    cname = {"mlp10m": "config1: toy-MLP-shaped", "gpt1p3b": "config2: GPT-1.3B-shaped",
             "llama8b": "config3: Llama-3-8B-shaped", "longcat560b": "config4: LongCat-560B-shaped"}[args.layout]
    workload = (f"{cname} {args.dtype} state dict ({args.layout}), {N_EXPERTS} experts + base, "
                f"FusionConfig(dropout_p={args.dropout}, seed=42, erase sum, mean-norm), sharded by param range")

    if args.impl == "reference":
        if rank != 0:
            return
        vals = []
        for i in range(args.warmup + args.steps):
            r = cpu_baseline(args.layout, args.dropout)
            if i >= args.warmup:
                vals.append(r)
        v = statistics.mean(r["value"] for r in vals)
        sec_per_step = statistics.mean(r["cpu_seconds"] / r["cores"] for r in vals)
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "params/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec_per_step * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": workload, "sample": vals[0]["sample"]},
                "cpu_baseline": {k: vals[0][k] for k in ("unit", "cores", "kind", "sample")} | {"value": v},
                "e2e": {"value": v, "unit": "params/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        if not args.no_grpo:
            gc = grpo_cpu_baseline()
            line["grpo"] = {"workload": "config5 token terms, V=131072", "tokens_per_s": gc["value"],
                            "cpu_baseline": gc}
        # the unmodified reference beside the port (the port is the line's value: it is ~15x faster
        # than the reference's per-element Python dropout loop, so the ratio against it is conservative)
        line["reference_unmodified"] = reference_cpu(args.dropout)
        print(json.dumps(line))
        return

    import torch
    if args.stream:
        line = stream_bench(args, rank, world, local, group, peak, peak_src)
        if line is not None:
            print(json.dumps(line))
            if args.json_out:
                Path(args.json_out).write_text(json.dumps(line, indent=1))
        if group is not None:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    fz = fusion_bench(args, rank, world, local, group)
    gr = None if args.no_grpo else grpo_bench(args, rank, world, local, group)
    # BASELINE.json configs 2 and 1 (parity cases, reported beside the headline): the same step on the
    # GPT-1.3B-shaped bf16 dict and on the 10M-param f32 MLP dict (L2 flushed between its steps)
    others = {}
    if world == 1 and not args.quick and args.layout == "llama8b":
        for key, lay, dt in (("config2", "gpt1p3b", "bf16"), ("config1", "mlp10m", "f32")):
            sub = argparse.Namespace(**{**vars(args), "layout": lay, "dtype": dt, "quick": True, "no_e2e": True})
            r = fusion_bench(sub, rank, world, local, group)
            es_ = {"bf16": 2, "f32": 4}[dt]
            kb_ = {"rlk_fusion_sumsq": (N_EXPERTS + 1) * es_, MERGE_CALL: (N_EXPERTS + 1) * es_ + es_}
            kern_ = {k: v for k, v in r["kern_local"].items() if k in kb_}
            dom_ = max(kern_, key=kern_.get)
            ach_ = r["local_params"] * kb_[dom_] / (kern_[dom_] / 1e3) / 1e9
            step_b = r["total_params"] * es_ * ((N_EXPERTS + 1) * 2 + 1)
            others[key] = {"workload": f"{lay} {dt}, {r['total_params']} params, {r['n_tensors']} tensors, "
                                       f"FusionConfig(dropout_p={args.dropout}, seed=42)",
                           "value": r["total_params"] / (r["ms"] / 1e3), "unit": "params/s",
                           "ms_per_step": r["ms"], "hbm_frac_step": step_b / (r["ms"] / 1e3) / 1e9 / peak,
                           "roofline": {"bound": "hbm", "kernel": dom_, "achieved": ach_, "peak": peak,
                                        "unit": "GB/s", "frac": ach_ / peak, "bytes_per_param": kb_[dom_],
                                        "kernels_ms": r["kern_local"]},
                           "l2": r["l2"], "launch": r["launch"], "clocks": r["clocks"]}
    cpu = gcpu = None
    ref_cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.layout, args.dropout)
        if gr is not None:
            gcpu = grpo_cpu_baseline()
        ref_cpu = reference_cpu(args.dropout)
    if rank != 0:
        if group is not None:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    total = fz["total_params"]
    ms = fz["ms"]
    value = total / (ms / 1e3)
    # dominant kernel roofline (rank 0's launches; algorithmic bytes = SURVEY 8(d) per-param figures)
    es = {"bf16": 2, "f32": 4}[args.dtype]
    kb = {"rlk_fusion_sumsq": (N_EXPERTS + 1) * es, MERGE_CALL: (N_EXPERTS + 1) * es + es}
    kern = {k: v for k, v in fz["kern_local"].items() if k in kb}
    dom = max(kern, key=kern.get)
    achieved = fz["local_params"] * kb[dom] / (kern[dom] / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        try:
            tj = json.loads(tfile.read_text())
            traffic = tj.get(args.layout, {}).get(f"{world}", {}).get(TRAFFIC_KEY.get(dom, dom))
        except Exception:
            traffic = None
    step_gbs = (total * es * (N_EXPERTS + 1) * 2 + total * es) / (ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "params/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (counter-hash normal, SURVEY 8(d))",
        "config": {"workload": workload, "params": total, "tensors": fz["n_tensors"], "experts": N_EXPERTS,
                   "parallelism": f"param-range shards x{world} (embedding-sized tensors striped), "
                                  + (f"{_backend_name(group)} all_reduce of the split tensors' norm partials"
                                     if group is not None else "no collective at one rank"),
                   "l2": fz["l2"], "launch": fz["launch"],
                   "dropout_mode": {1: "inline", 2: "bitmap"}.get(fz["dropout_mode"], "none")},
        "hbm_gbs_step": step_gbs, "hbm_frac_step": step_gbs / peak,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "frac_of_8tbs_spec": achieved / 8000.0, "traffic": traffic,
                     "peak_source": peak_src,
                     "bytes_per_param": kb[dom], "kernels_ms": fz["kern_local"]},
        "clocks": fz["clocks"],
        "gpu_launches": fz["launches_per_step"] * args.steps,
    }
    if "variants" in fz:
        line["variants"] = {k: {"value": total / (ms / 1e3), "ms_per_step": ms} for k, ms in fz["variants"].items()}
    if "e2e_ms" in fz:
        line["e2e"] = {"value": total / (fz["e2e_ms"] / 1e3), "unit": "params/s",
                       "h2d_bytes_per_step": fz["h2d"], "d2h_bytes_per_step": fz["d2h"],
                       "ms_per_step": fz["e2e_ms"], "steps": fz["e2e_steps"], "warmup": fz["e2e_warmup"],
                       "h2d_gbs": fz["h2d"] / (fz["e2e_ms"] / 1e3) / 1e9,
                       "path": fz["e2e_path"]}
    if gr is not None:
        tok = gr["tokens"]
        fwd_b = gr["kern"]["rlk_grpo_fwd"]
        ach = gr["rows_per_launch"] * (gr["V"] * 2 + 12) / (fwd_b / 1e3) / 1e9
        line["grpo"] = {"workload": f"config5: V={gr['V']}, G=16 x T={tok // 16} tokens (one group), bf16 logits",
                        "tokens_per_s": tok / (gr["fwd_ms"] / 1e3), "fwd_ms": gr["fwd_ms"],
                        "fwd_bwd_tokens_per_s": tok / (gr["fwdbwd_ms"] / 1e3), "fwd_bwd_ms": gr["fwdbwd_ms"],
                        "fwd_bwd_path": "rlk_grpo_fused_bf16 (one read of the logits, bf16 grad written)",
                        "fwd_bwd_roofline": {"achieved": gr["rows_per_launch"] * gr["V"] * 4 / (gr["kern"]["rlk_grpo_fused_bf16"] / 1e3) / 1e9,
                                             "peak": peak, "unit": "GB/s", "bytes_per_token": gr["V"] * 4,
                                             "frac": gr["rows_per_launch"] * gr["V"] * 4 / (gr["kern"]["rlk_grpo_fused_bf16"] / 1e3) / 1e9 / peak},
                        "roofline": {"bound": "hbm", "kernel": "rlk_grpo_fwd", "achieved": ach, "peak": peak,
                                     "unit": "GB/s", "frac": ach / peak, "bytes_per_token": gr["V"] * 2 + 12},
                        "kernels_ms": gr["kern"]}
        if "variants" in gr:
            line["grpo"]["variants"] = gr["variants"]
        if gcpu is not None:
            line["grpo"]["cpu_baseline"] = gcpu
    if others:
        line["other_configs"] = others
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if ref_cpu is not None:
        line["cpu_baseline_reference_unmodified"] = ref_cpu
    print(json.dumps(line))
    if args.json_out:
        Path(args.json_out).write_text(json.dumps(line, indent=1))
    if group is not None:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
