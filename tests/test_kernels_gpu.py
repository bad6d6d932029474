"""sm_100a staging kernels vs PyTorch reference ops, bit-exact.

pack  == tensor.contiguous()          (rows / transpose / generic paths)
unpack== strided_view.copy_(contig)
ZVC   == identity on the 32-bit words  (encode -> decode round trip)
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

DTYPES = [torch.float32, torch.float16, torch.bfloat16, torch.float64, torch.int8, torch.int64]


def _views(dtype):
    dev = "cuda"
    base = torch.randn(6, 40, 66, device=dev).to(dtype) if dtype.is_floating_point else \
        torch.randint(-100, 100, (6, 40, 66), device=dev, dtype=dtype)
    yield "contiguous", base
    yield "slice_rows", base[:, 3:37, :]
    yield "slice_cols", base[:, :, 2:50]
    yield "transpose_last", base.transpose(1, 2)
    yield "permute", base.permute(2, 0, 1)
    yield "step", base[::2, ::3, ::5]
    yield "expand", base[:, :1, :].expand(6, 40, 66)
    yield "channels_last", torch.randn(4, 8, 9, 10, device=dev).to(dtype).contiguous(
        memory_format=torch.channels_last) if dtype.is_floating_point else base
    yield "empty", base[:, :0, :]
    yield "scalar", base[0, 0, 0]
    yield "big_rows", (torch.randn(257, 1030, device=dev).to(dtype) if dtype.is_floating_point
                       else torch.randint(0, 5, (257, 1030), device=dev, dtype=dtype))[:, 7:1007]
    # 16 B-aligned row strides: these take the tensor-map (TMA) path when enabled
    big = (torch.randn(4, 64, 24, 64, device=dev).to(dtype) if dtype.is_floating_point
           else torch.randint(-9, 9, (4, 64, 24, 64), device=dev, dtype=dtype))
    yield "tma_channel_slice", big[:, 8:40]
    yield "tma_inner_slice", big[:, :, 3:21, 16:48]
    yield "tma_ragged_box", big[1:, 5:61, :, :48]
    yield "tma_6d", big.view(4, 8, 8, 24, 8, 8)[:, 1:7, :, 2:22, :, :]
    wide = (torch.randn(3, 40, 56, 56, device=dev).to(dtype) if dtype.is_floating_point
            else torch.randint(-9, 9, (3, 40, 56, 56), device=dev, dtype=dtype))
    yield "tma_odd_box_bytes", wide[:, :, :, 4:52]   # 192 B rows: boxes not a multiple of 128 B
    # channels-last views of NCHW tensors: the TMA transpose path (128 B-swizzled tiles)
    yield "tma_nhwc", big.permute(0, 2, 3, 1)
    yield "tma_nhwc_batch_slice", big[1:, :, 2:22, :].permute(0, 2, 3, 1)
    odd = (torch.randn(2, 40, 12, 48, device=dev).to(dtype) if dtype.is_floating_point
           else torch.randint(-9, 9, (2, 40, 12, 48), device=dev, dtype=dtype))
    yield "tma_nhwc_partial_tiles", odd.permute(0, 2, 3, 1)


@pytest.mark.parametrize("tma", [1, 0])
@pytest.mark.parametrize("dtype", DTYPES)
def test_pack_matches_contiguous(lms_ctx, dtype, tma):
    lms_ctx.set_tuning(0, -1, tma)
    try:
        for name, v in _views(dtype):
            got = lms_ctx.pack(v)
            torch.cuda.synchronize()
            want = v.contiguous()
            assert torch.equal(got, want), name
    finally:
        lms_ctx.set_tuning(0, -1, 1)


@pytest.mark.parametrize("tma", [1, 0])
@pytest.mark.parametrize("dtype", DTYPES)
def test_unpack_matches_copy(lms_ctx, dtype, tma):
    lms_ctx.set_tuning(0, -1, tma)
    for name, v in _views(dtype):
        if name == "expand":
            continue  # overlapping destination: ill-defined scatter
        src = (torch.arange(v.numel(), device="cuda") % 97).to(dtype).reshape(v.shape).contiguous()
        dst = v.clone() if v.dim() == 0 else torch.empty_strided(v.shape, v.stride(), dtype=dtype, device="cuda")
        want_base = dst.clone()
        want_base.copy_(src)
        lms_ctx.unpack(src, dst)
        torch.cuda.synchronize()
        assert torch.equal(dst, src), name
    lms_ctx.set_tuning(0, -1, 1)


@pytest.mark.parametrize("exponents", [0, 1])
@pytest.mark.parametrize("bulk", [1, 0])
@pytest.mark.parametrize("nwords,density", [(0, 0.5), (1, 1.0), (3, 0.0), (4095, 0.5), (4096, 0.5),
                                            (4097, 0.3), (1 << 20, 0.5), (1 << 20, 0.0),
                                            (1 << 20, 1.0), ((1 << 22) + 13, 0.47)])
def test_zvc_roundtrip(lms_ctx, nwords, density, bulk, exponents):
    lms_ctx.set_tuning(0, bulk)
    torch.manual_seed(nwords)
    x = torch.randn(nwords, device="cuda")
    x = torch.where(torch.rand(nwords, device="cuda") < density, x, torch.zeros_like(x))
    if nwords > 8:
        x[5] = -0.0           # sign-only word is nonzero as bits: must survive
        x[7] = float("nan")
    bound = lms_ctx.zvc_bound(nwords)
    enc = torch.empty(max(bound, 16), dtype=torch.uint8, device="cuda")
    lms_ctx.zvc_encode(x, enc, exponents=bool(exponents))
    out = torch.full_like(x, 7.0)
    lms_ctx.zvc_decode(enc, out)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int32), x.view(torch.int32))
    if nwords:
        host = enc.cpu()
        hdr = host[:64].view(torch.int64)
        assert int(hdr[1]) == nwords and int(hdr[2]) == (nwords + 4095) // 4096
        wire = lms_ctx.zvc_encoded_size(host)
        assert wire <= bound
        if density == 0.0:
            # all-zero tiles are a bare mask (tile 0 also holds the -0.0 and NaN words)
            assert wire <= 64 + 8 * int(hdr[2]) + 512 * int(hdr[2]) + 16
    lms_ctx.set_tuning(0, 1)


def _special_words(n, g):
    """fp32 bit patterns the exponent planes must carry exactly."""
    x = torch.randn(n, device="cuda", generator=g)
    specials = torch.tensor([0.0, -0.0, float("inf"), float("-inf"), float("nan"), 1e-45, -1e-45, 1e-38,
                             3.4e38, -3.4e38, 1.0, -1.0], device="cuda")
    idx = torch.randint(0, n, (min(n, 64),), device="cuda", generator=g)
    x[idx] = specials[torch.arange(idx.numel(), device="cuda") % specials.numel()]
    return x


@pytest.mark.parametrize("n", [5, 4096, 4096 * 7 + 11, 1 << 22])
def test_zx_exponent_planes_roundtrip(lms_ctx, n):
    """ZX tiles (exponent planes over all words or over the nonzero ones): bit-exact
    on normal activations, all-positive ReLU outputs (no sign plane), scaled
    ranges (wide exponent bands) and special values."""
    g = torch.Generator(device="cuda").manual_seed(n)
    cases = {
        "normal": torch.randn(n, device="cuda", generator=g),
        "relu": torch.relu(torch.randn(n, device="cuda", generator=g)),
        "wide": torch.randn(n, device="cuda", generator=g) * torch.exp(8 * torch.randn(n, device="cuda", generator=g)),
        "special": _special_words(n, g),
        "ints": torch.randint(-2**31, 2**31 - 1, (n,), device="cuda", dtype=torch.int32, generator=g).view(torch.float32),
    }
    for name, x in cases.items():
        enc = torch.empty(lms_ctx.zvc_bound(n), dtype=torch.uint8, device="cuda")
        lms_ctx.zvc_encode(x, enc, exponents=True)
        out = torch.empty_like(x)
        lms_ctx.zvc_decode(enc, out)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int32), x.view(torch.int32)), name
        if n >= 4096 and name in ("normal", "relu"):
            wire = lms_ctx.zvc_encoded_size(enc.cpu())
            # normal: sign + ~3-4 exponent bits + 24 low bits per word; relu: mask + no sign
            assert wire < (0.92 if name == "normal" else 0.5) * 4 * n, (name, wire / (4 * n))


def test_zx_swap_roundtrip_and_wire(lms_ctx):
    """ZX round trips of a dense and a ReLU tensor issued after the swap-out landed."""
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(64, 256, 28, 28, device="cuda", generator=g)
    lms_ctx.synchronize()
    lms_ctx.trace_clear()
    for codec in ("zx", "zvc"):
        h = lms_ctx.swap_out(x, codec)
        torch.cuda.synchronize()
        lms_ctx.synchronize()      # the stream's tile table is readable: the exact wire size is known
        out = lms_ctx.swap_in(h)
        lms_ctx.wait(h)
        torch.cuda.synchronize()
        lms_ctx.synchronize()
        wire = lms_ctx.wire_bytes(h)
        lms_ctx.release(h)
        assert torch.equal(out, x), codec
        if codec == "zx":
            assert wire < 0.92 * x.numel() * 4
        else:
            assert wire >= x.numel() * 4   # dense: ZVC keeps raw tiles
    r = torch.relu(x)
    h = lms_ctx.swap_out(r, "zx")
    torch.cuda.synchronize()
    lms_ctx.synchronize()
    out = lms_ctx.swap_in(h)
    lms_ctx.wait(h)
    torch.cuda.synchronize()
    assert torch.equal(out, r)
    lms_ctx.release(h)
