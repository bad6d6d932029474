"""Swap engine round trips, budget enforcement and free-after-transfer semantics.

Reference behaviour being realised: swap nodes are identities on values
(interp.py:168-170); a swapped-out block is freed only after its outbound
transfer completes (sim.py:205-211); exceeding device capacity is an OOM
(sim.py:471).
"""

import pytest
import torch

from paper_1807_02037_b200 import runtime as rt

pytestmark = pytest.mark.gpu


def _cases():
    g = torch.Generator(device="cuda").manual_seed(0)
    yield "contig_f32", torch.randn(1024, 1031, device="cuda", generator=g)
    yield "relu_sparse", torch.relu(torch.randn(64, 256, 56, 56, device="cuda", generator=g))
    yield "channels_last", torch.randn(8, 64, 28, 28, device="cuda", generator=g).contiguous(
        memory_format=torch.channels_last)
    yield "strided_slice", torch.randn(300, 500, device="cuda", generator=g)[:, 100:400]
    yield "transposed_slice", torch.randn(300, 500, device="cuda", generator=g).t()[10:300]
    yield "expand", torch.randn(1, 512, device="cuda", generator=g).expand(64, 512)
    yield "bf16", torch.randn(333, 777, device="cuda", generator=g).bfloat16()
    yield "odd_bytes", torch.randint(0, 255, (1001,), device="cuda", dtype=torch.uint8)
    yield "empty", torch.empty(0, 16, device="cuda")


@pytest.mark.parametrize("codec", ["ce", "sm", "zvc"])
def test_roundtrip_bit_exact(lms_ctx, codec):
    for name, t in _cases():
        want = t.clone()
        h = lms_ctx.swap_out(t, codec)
        out = lms_ctx.swap_in(h)
        lms_ctx.wait(h)
        lms_ctx.release(h)
        torch.cuda.synchronize()
        assert out.shape == want.shape, name
        assert torch.equal(out, want), (name, codec)


def test_zvc_shrinks_sparse_and_not_dense(lms_ctx):
    sparse = torch.relu(torch.randn(1 << 22, device="cuda"))
    dense = torch.randn(1 << 22, device="cuda")
    hs = lms_ctx.swap_out(sparse, "zvc")
    hd = lms_ctx.swap_out(dense, "zvc")
    torch.cuda.synchronize()
    lms_ctx.synchronize()
    assert lms_ctx.wire_bytes(hs) < 0.6 * sparse.numel() * 4
    # raw tiles: never bigger than the words plus the header and the tile table
    assert lms_ctx.wire_bytes(hd) <= dense.numel() * 4 + 64 + 8 * (dense.numel() // 4096)
    for h in (hs, hd):
        out = lms_ctx.swap_in(h)
        lms_ctx.wait(h)
        lms_ctx.release(h)
    torch.cuda.synchronize()


def test_free_waits_for_swap_out(lms_ctx):
    """Freeing a tensor right after swap_out must not let the block be recycled
    before the D2H has read it."""
    s = torch.cuda.current_stream()
    for _ in range(3):
        t = torch.randn(64 << 20, device="cuda")  # 256 MiB: the copy takes milliseconds
        want = t[:1024].clone(), t[-1024:].clone()
        h = lms_ctx.swap_out(t, "ce")
        del t                                       # free immediately (stream-ordered)
        junk = torch.full((64 << 20,), 3.0, device="cuda")  # would reuse the block if not held
        out = lms_ctx.swap_in(h, trigger_stream=s)
        lms_ctx.wait(h)
        torch.cuda.synchronize()
        assert torch.equal(out[:1024], want[0]) and torch.equal(out[-1024:], want[1])
        lms_ctx.release(h)
        del junk, out


def test_budget_is_enforced(lms_ctx):
    st = lms_ctx.stats()
    lms_ctx.set_limit(st["device_in_use"] + (64 << 20))
    try:
        a = torch.empty(32 << 20, dtype=torch.uint8, device="cuda")
        with pytest.raises(RuntimeError, match="LMS_OOM"):
            torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
        del a
    finally:
        lms_ctx.set_limit(0)
    assert lms_ctx.stats()["n_oom"] >= 1


def test_stats_count_bytes_and_kernels(lms_ctx):
    lms_ctx.trace_clear()
    t = torch.relu(torch.randn(1 << 20, device="cuda"))
    h = lms_ctx.swap_out(t, "zvc")
    out = lms_ctx.swap_in(h)
    lms_ctx.wait(h)
    lms_ctx.release(h)
    torch.cuda.synchronize()
    lms_ctx.synchronize()
    st = lms_ctx.stats()
    assert st["d2h_logical_bytes"] == 4 << 20 and st["h2d_logical_bytes"] == 4 << 20
    assert st["kernel_launches"] >= 2  # one-pass encode, decode
    assert 0 < st["d2h_wire_bytes"] < 4 << 20
    tr = lms_ctx.trace()
    assert {r["direction"] for r in tr} == {0, 1}
    assert all(r["end_ms"] >= r["start_ms"] for r in tr)


@pytest.mark.parametrize("bulk,ctas", [(1, 0), (0, 0), (1, 3), (0, 5), (1, 1000)])
def test_zvc_zero_copy_paths(lms_ctx, bulk, ctas):
    """Encode into / decode out of pinned memory with bulk (TMA) and per-thread
    copies, few and many CTAs: bit-exact, including ragged last tiles."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    lms_ctx.set_tuning(ctas or sms, bulk)
    try:
        g = torch.Generator(device="cuda").manual_seed(ctas + bulk)
        for n in (1, 4095, 4096, 4097, 3 * 4096 + 5, (1 << 21) + 17):
            x = torch.relu(torch.randn(n, device="cuda", generator=g))
            x[: min(n, 7)] = torch.tensor([-0.0, float("nan"), 1.0, 0.0, -1.0, 0.0, 2.0], device="cuda")[: min(n, 7)]
            h = lms_ctx.swap_out(x, "zvc")
            outs = [lms_ctx.swap_in(h) for _ in range(2)]  # two swap-ins of one handle
            lms_ctx.wait(h)
            torch.cuda.synchronize()
            lms_ctx.synchronize()
            for o in outs:
                assert torch.equal(o.view(torch.int32), x.view(torch.int32)), n
            lms_ctx.release(h)
    finally:
        lms_ctx.set_tuning(sms, 1)


def test_strided_swap_goes_through_staging(lms_ctx):
    """A non-dense view (channel slice, > one 32 MiB staging slab) is packed in HBM
    by the TMA kernels into the D2H channel's staging block and moved by the copy
    engine; restoring into another strided view unpacks through the H2D block."""
    g = torch.Generator(device="cuda").manual_seed(11)
    base = torch.randn(48, 96, 56, 56, device="cuda", generator=g)
    v = base[:, 16:80]                       # 48 x 64 x 56 x 56 fp32 = 37.6 MiB, not dense
    want = v.contiguous()
    lms_ctx.trace_clear()
    h = lms_ctx.swap_out(v, "ce")
    assert lms_ctx.handle_codec(h) == rt.CODEC_RAW_CE
    out = lms_ctx.swap_in(h)                  # natural (contiguous) restore: copy engine
    lms_ctx.wait(h)
    big = torch.zeros(48, 128, 56, 56, device="cuda")
    dst = big[:, 32:96]                       # strided destination: staged H2D + TMA unpack
    lms_ctx.swap_in(h, dst=dst)
    lms_ctx.wait(h)
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    assert torch.equal(dst, want)
    assert float(big[:, :32].abs().sum()) == 0.0 and float(big[:, 96:].abs().sum()) == 0.0
    lms_ctx.release(h)
    st = lms_ctx.stats()
    assert st["kernel_launches"] >= 4        # >= 2 pack slabs + 2 unpack slabs
