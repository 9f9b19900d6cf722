"""Host logic of the streaming loader (no GPU): tensor grouping and the device ring placement."""
import numpy as np
import pytest

from paper_2509_18883_b200.loader import _footprint, plan_groups, ring_placement


def test_plan_groups_consecutive_and_bounded():
    g = np.random.default_rng(0)
    numels = list(g.integers(1, 5000, 200))
    budget = 40_000 * 2 * 5
    groups = plan_groups(numels, 3, 2, budget)
    assert [t for grp in groups for t in grp] == list(range(len(numels)))
    for grp in groups:
        assert sum(_footprint(numels[t], 3, 2) for t in grp) <= budget
    with pytest.raises(ValueError, match="does not fit"):
        plan_groups([10**9], 3, 2, budget)


@pytest.mark.parametrize("seed", range(20))
def test_ring_placement_never_overwrites_live_data(seed):
    """Replay the placement: every earlier group whose data group g overwrites must have been waited on
    by g or by an earlier group (the H2D stream is in order, so an earlier wait covers g too)."""
    g = np.random.default_rng(seed)
    cap = int(g.integers(100, 1000))
    sizes = [int(x) for x in g.integers(1, cap + 1, 60)]
    place, waits = ring_placement(sizes, cap)
    owner = [-1] * cap  # which group's data occupies each slot
    waited = set()
    for gi, (lo, size) in enumerate(zip(place, sizes)):
        assert 0 <= lo and lo + size <= cap
        waited |= set(waits[gi])
        overwritten = {owner[x] for x in range(lo, lo + size) if owner[x] >= 0}
        assert overwritten <= waited, (gi, overwritten, waited)
        assert all(j < gi for j in waits[gi])
        for x in range(lo, lo + size):
            owner[x] = gi
    # every group is waited on at most once
    flat = [j for w in waits for j in w]
    assert len(flat) == len(set(flat))
    with pytest.raises(ValueError, match="exceeds the ring"):
        ring_placement([cap + 1], cap)
