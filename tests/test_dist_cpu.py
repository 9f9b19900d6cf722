"""Multi-process (gloo, world_size 2) tests of the sharded host logic: partitioning, the exact
all_reduce of norm partials, counter sums and the GRPO group-sum reduction.  The per-item partials
are produced here by the test itself (numpy) as stand-ins for K1's output."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_18883_b200.fusion import ITEM, FusionLayout

NUMELS = [3 * ITEM + 17, 5, ITEM, 2 * ITEM - 1, 70001, 1]


def test_partition_covers_every_item_once():
    layout = FusionLayout(NUMELS)
    for world in (1, 2, 3, 4, 8):
        seen = {}
        sizes = []
        for r in range(world):
            parts = layout.partition(world, r)
            sizes.append(sum(hi - lo for _, lo, hi in parts))
            for t, lo, hi in parts:
                assert lo % ITEM == 0 and 0 <= lo < hi <= NUMELS[t]
                for k in range(lo // ITEM, (hi + ITEM - 1) // ITEM):
                    assert (t, k) not in seen
                    seen[(t, k)] = r
        assert len(seen) == layout.n_items
        assert sum(sizes) == layout.total
        # contiguous ranks: item ownership is non-decreasing along the global item order
        order = [seen[(t, k)] for t in range(len(NUMELS)) for k in range((NUMELS[t] + ITEM - 1) // ITEM)]
        assert order == sorted(order)


def test_striped_partition_covers_every_item_once_and_balances():
    from paper_2509_18883_b200.layouts import LAYOUTS, numel
    for numels in (NUMELS, [numel(s) for s in LAYOUTS["llama8b"]().values()],
                   [numel(s) for s in LAYOUTS["gpt1p3b"]().values()]):
        layout = FusionLayout(numels)
        for world in (1, 2, 3, 4, 8):
            seen = set()
            sizes = []
            for r in range(world):
                parts = layout.partition_striped(world, r)
                sizes.append(sum(hi - lo for _, lo, hi in parts))
                for t, lo, hi in parts:
                    assert lo % ITEM == 0 and 0 <= lo < hi <= numels[t]
                    for k in range(lo // ITEM, (hi + ITEM - 1) // ITEM):
                        assert (t, k) not in seen
                        seen.add((t, k))
            assert len(seen) == layout.n_items and sum(sizes) == layout.total
            if layout.total > 10 ** 8:
                assert max(sizes) <= 1.01 * layout.total / world + 2 * ITEM


def test_striped_partition_shrinks_each_ranks_keep_bits():
    """With the embedding-sized tensors striped, no rank of an 8-way config-3 job reads keep bits beyond
    the layer tensors' extent plus one 1/8 stripe (vs the whole 525M-bit rows with contiguous ranges)."""
    from paper_2509_18883_b200.fusion import needed_bit_ranges
    from paper_2509_18883_b200.layouts import LAYOUTS, numel
    numels = [numel(s) for s in LAYOUTS["llama8b"]().values()]
    layout = FusionLayout(numels)
    big = max(numels)
    small_max = max(n for n in numels if n < big)
    for r in range(8):
        bits = sum(hi - lo for lo, hi in needed_bit_ranges(
            [(lo, hi) for _, lo, hi in layout.partition_striped(8, r)]))
        assert bits <= small_max + big // 8 + 2 * ITEM
    contiguous = sum(hi - lo for lo, hi in needed_bit_ranges([(lo, hi) for _, lo, hi in layout.partition(8, 0)]))
    assert contiguous >= big


def test_needed_bit_ranges_union():
    from paper_2509_18883_b200.fusion import needed_bit_ranges
    assert needed_bit_ranges([(0, 10), (5, 70), (96, 100), (200, 200)]) == [(0, 128)]
    assert needed_bit_ranges([(64, 65), (0, 1)]) == [(0, 32), (64, 96)]
    assert needed_bit_ranges([]) == []


def _item_partials(values, layout, parts, n_exp):
    """Per-item f64 sums of squares for this rank's pieces (what K1 writes)."""
    out = np.zeros(layout.n_items * n_exp)
    for t, lo, hi in parts:
        for k in range(lo // ITEM, (hi + ITEM - 1) // ITEM):
            a, b = k * ITEM, min((k + 1) * ITEM, NUMELS[t])
            for i in range(n_exp):
                d = values[i][t][a:b]
                out[(layout.tensor_items[t] + k) * n_exp + i] = float(np.dot(d, d))
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_18883_b200.dist import allreduce_counts, allreduce_partials
        layout = FusionLayout(NUMELS)
        g = np.random.default_rng(0)
        values = [[g.normal(0, 1e-3, n) for n in NUMELS] for _ in range(3)]
        mine = _item_partials(values, layout, layout.partition(world, rank), 3)
        p = torch.from_numpy(mine.copy())
        allreduce_partials(p, dist.group.WORLD)
        full = _item_partials(values, layout, layout.partition(1, 0), 3)
        exact = bool(np.array_equal(p.numpy(), full))
        c = torch.tensor([rank + 1, 10 * (rank + 1)], dtype=torch.int64)
        allreduce_counts(c, dist.group.WORLD)
        gs = torch.tensor([0.25 * (rank + 1), -1.0], dtype=torch.float64)
        dist.all_reduce(gs)
        q.put((rank, exact, c.tolist(), gs.tolist()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_world2_exact_partials_and_counts():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, exact, counts, gs in res:
        assert exact, f"rank {rank}: sharded partials differ from the world-1 table"
        assert counts == [3, 30]
        assert gs == [0.75, -2.0]
