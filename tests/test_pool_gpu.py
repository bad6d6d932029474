"""Device pool under fragmentation: page moves must never corrupt live data.

A second context with its own small budget (not the allocator of the test
session) is fragmented until an allocation that fits the budget only by
moving physical pages; every live block keeps its contents, the moved-to
block is fully writable, and trimming the stale aliases keeps it so.  This is
the pool's version of the reference's residency model (sim.py:116-124,
:193-211): bytes stay with their owner until it frees them.
"""

import pytest
import torch

from paper_1807_02037_b200 import runtime as rt

pytestmark = pytest.mark.gpu

MIB = 1 << 20


def _view(ptr, nbytes):
    return torch.as_tensor(rt.DeviceBuffer(ptr, nbytes), device="cuda")


def test_page_moves_keep_live_blocks_intact(lms_ctx):
    ctx = rt.Context(device=0, device_reserve=1 << 30, timing=False)   # 16 pages of 64 MiB
    try:
        blocks = []
        for i in range(12):   # 12 one-page blocks, then 4 free pages at the end
            p = ctx.dev_alloc(64 * MIB)
            v = _view(p, 64 * MIB)
            v.fill_(i + 1)
            blocks.append((p, i + 1))
        torch.cuda.synchronize()
        # free every other block: plenty of free bytes, no contiguous run big enough
        for p, _ in blocks[1:11:2]:   # 1,3,5,7,9: one-page holes; 11 stays, so the free tail is 4 pages
            ctx.dev_free(p)
        keep = blocks[0::2] + [blocks[11]]
        torch.cuda.synchronize()
        before = ctx.stats()
        big = ctx.dev_alloc(320 * MIB)     # 5 pages: fits only with pages moved (aliased) under fresh VA
        after = ctx.stats()
        vb = _view(big, 320 * MIB)
        vb.fill_(0xAB)
        torch.cuda.synchronize()
        for p, val in keep:
            assert bool((_view(p, 64 * MIB) == val).all()), "a live block changed after a page move"
        assert bool((vb == 0xAB).all())
        assert after["n_reclaims"] > before["n_reclaims"]
        # trimming the stale VA aliases must not touch live data either
        torch.cuda.synchronize()
        ctx.trim()
        for p, val in keep:
            assert bool((_view(p, 64 * MIB) == val).all())
        assert bool((vb == 0xAB).all())
        ctx.dev_free(big)
        for p, _ in keep:
            ctx.dev_free(p)
        # the whole budget is usable again after the moves
        p = ctx.dev_alloc(900 * MIB)
        _view(p, 900 * MIB).fill_(7)
        torch.cuda.synchronize()
        ctx.dev_free(p)
    finally:
        torch.cuda.synchronize()
        ctx.close()


def test_budget_is_physical(lms_ctx):
    ctx = rt.Context(device=0, device_reserve=256 * MIB, timing=False)
    try:
        p = ctx.dev_alloc(200 * MIB)
        with pytest.raises(rt.LmsOutOfMemoryError):
            ctx.dev_alloc(100 * MIB)
        ctx.dev_free(p)
        q = ctx.dev_alloc(250 * MIB)
        ctx.dev_free(q)
    finally:
        ctx.close()


def test_record_stream_holds_reuse(lms_ctx):
    """Tensor.record_stream(s) through the pluggable allocator: a block freed on the
    compute stream is not handed out again before the work queued on `s` ran."""
    side = torch.cuda.Stream()
    t = torch.empty(64 * MIB, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(200_000_000)     # keep `side` busy (~0.1 s)
        t.fill_(3)
    t.record_stream(side)
    before = lms_ctx.stats()["n_deferred_frees"]
    del t
    st = lms_ctx.stats()
    assert st["n_deferred_frees"] == before + 1    # held for `side`, not reusable yet
    torch.cuda.synchronize()
    lms_ctx.synchronize()
    assert lms_ctx.stats()["device_deferred_bytes"] == 0


def test_plan_record_replay_refine_keeps_data(lms_ctx):
    """A synthetic 'step' (fixed sequence of allocations and frees, some blocks held
    by in-flight side-stream work like swap-out copies) run dynamically, recorded,
    refined and replayed: every live block keeps its own bytes in every mode."""
    import random
    ctx = rt.Context(device=0, device_reserve=768 * MIB, timing=False)
    side = torch.cuda.Stream()
    rng = random.Random(7)
    seq = []                  # ("a", slot, size) / ("f", slot, hold)
    live = []
    for i in range(160):
        if live and (rng.random() < 0.45 or len(live) > 12):
            k = live.pop(rng.randrange(len(live)))
            seq.append(("f", k, rng.random() < 0.3))
        else:
            seq.append(("a", i, rng.choice([1, 3, 8, 24, 40]) * MIB + rng.randrange(0, 4096, 512)))
            live.append(i)
    for k in live:
        seq.append(("f", k, False))
    try:
        modes = [None, rt.PLAN_RECORD, rt.PLAN_REFINE, rt.PLAN_REPLAY, rt.PLAN_REPLAY]
        for step, mode in enumerate(modes):
            if mode is not None:
                ctx.plan_begin(mode)
            blocks = {}
            for op, k, x in seq:
                if op == "a":
                    p = ctx.dev_alloc(x)
                    _view(p, x).fill_((k * 7 + step) % 251)
                    blocks[k] = (p, x)
                else:
                    p, n = blocks.pop(k)
                    assert bool((_view(p, n) == (k * 7 + step) % 251).all()), (step, mode, k)
                    if x:   # a copy still reading it: the block is held until `side` passes
                        side.wait_stream(torch.cuda.current_stream())
                        with torch.cuda.stream(side):
                            torch.cuda._sleep(2_000_000)
                        ctx.hold_until(_view(p, n), side)
                    ctx.dev_free(p)
            torch.cuda.synchronize()
            if mode is not None:
                ctx.plan_end()
            if mode == rt.PLAN_RECORD:
                assert ctx.plan_info()["ready"]
        info = ctx.plan_info()
        assert info["hits"] > 0 and info["diverged_steps"] == 0
        ctx.plan_reset()
    finally:
        torch.cuda.synchronize()
        ctx.close()


def test_plan_replay_tolerates_extra_and_skipped_allocations(lms_ctx):
    """A replayed step that makes one allocation the recording did not (e.g. DDP's
    buffer-broadcast staging tensor) and skips two it did: the extra one is served
    by the dynamic pool, the skipped ones are stepped over, the rest still replay
    from their planned offsets (no divergence), and every block keeps its bytes."""
    ctx = rt.Context(device=0, device_reserve=512 * MIB, timing=False)
    sizes = [8 * MIB, 24 * MIB, 3 * MIB, 40 * MIB, 8 * MIB, 1 * MIB, 16 * MIB]

    def run(step, extra_at=None, skip=()):
        blocks = []
        for i, n in enumerate(sizes):
            if i == extra_at:
                e = ctx.dev_alloc(64 * 1024)
                _view(e, 64 * 1024).fill_(99)
                blocks.append((e, 64 * 1024, 99))
            if i in skip:
                continue
            p = ctx.dev_alloc(n)
            _view(p, n).fill_((i * 13 + step) % 251)
            blocks.append((p, n, (i * 13 + step) % 251))
        for p, n, v in blocks:
            assert bool((_view(p, n) == v).all()), (step, p)
        for p, _, _ in reversed(blocks):
            ctx.dev_free(p)
        torch.cuda.synchronize()

    try:
        run(0)
        ctx.plan_begin(rt.PLAN_RECORD)
        run(1)
        ctx.plan_end()
        ctx.plan_begin(rt.PLAN_REPLAY)
        run(2)
        ctx.plan_end()
        base = ctx.plan_info()
        ctx.plan_begin(rt.PLAN_REPLAY)
        run(3, extra_at=2, skip=(4, 5))
        ctx.plan_end()
        info = ctx.plan_info()
        assert info["diverged_steps"] == base["diverged_steps"] == 0
        assert info["hits"] - base["hits"] == len(sizes) - 2       # all but the skipped ones planned
        assert info["dynamic"] - base["dynamic"] == 1              # the extra one
        ctx.plan_reset()
    finally:
        torch.cuda.synchronize()
        ctx.close()
