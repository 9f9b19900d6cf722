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
        # keep bitmap: each rank draws its column slice of every expert row, then the rows are gathered
        from oracle import rng as ORNG
        from paper_2509_18883_b200.dist import allgather_bitmap_rows
        n_bits = 40960
        wc = ((n_bits // 32 + world - 1) // world + 3) // 4 * 4
        rows = [np.packbits(ORNG.keep_mask(ORNG.fusion_child_seed(42, i), 0, n_bits, 0.5), bitorder="little")
                .view(np.int32) for i in range(3)]
        bm = torch.full((3, wc * world), -7, dtype=torch.int32)
        lo, hi = rank * wc, min((rank + 1) * wc, n_bits // 32)
        for i in range(3):
            bm[i, lo:hi] = torch.from_numpy(rows[i][lo:hi].copy())
        allgather_bitmap_rows(bm, wc, dist.group.WORLD)
        bm_ok = all(np.array_equal(bm[i, :n_bits // 32].numpy(), rows[i]) for i in range(3))
        q.put((rank, exact, c.tolist(), gs.tolist(), bm_ok))
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
    for rank, exact, counts, gs, bm_ok in res:
        assert exact, f"rank {rank}: sharded partials differ from the world-1 table"
        assert bm_ok, f"rank {rank}: gathered keep bitmap differs from the full rows"
        assert counts == [3, 30]
        assert gs == [0.75, -2.0]
