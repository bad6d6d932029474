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


@pytest.mark.parametrize("bulk", [1, 0])
@pytest.mark.parametrize("nwords,density", [(0, 0.5), (1, 1.0), (3, 0.0), (4095, 0.5), (4096, 0.5),
                                            (4097, 0.3), (1 << 20, 0.5), (1 << 20, 0.0),
                                            (1 << 20, 1.0), ((1 << 22) + 13, 0.47)])
def test_zvc_roundtrip(lms_ctx, nwords, density, bulk):
    lms_ctx.set_tuning(0, bulk)
    torch.manual_seed(nwords)
    x = torch.randn(nwords, device="cuda")
    x = torch.where(torch.rand(nwords, device="cuda") < density, x, torch.zeros_like(x))
    if nwords > 8:
        x[5] = -0.0           # sign-only word is nonzero as bits: must survive
        x[7] = float("nan")
    bound = lms_ctx.zvc_bound(nwords)
    enc = torch.empty(max(bound, 16), dtype=torch.uint8, device="cuda")
    lms_ctx.zvc_encode(x, enc)
    out = torch.full_like(x, 7.0)
    lms_ctx.zvc_decode(enc, out)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int32), x.view(torch.int32))
    hdr = enc[:64].cpu().view(torch.int64)
    nnz = int((x.view(torch.int32) != 0).sum())
    if nwords:
        assert int(hdr[3]) == nnz  # total_nnz field
    lms_ctx.set_tuning(0, 1)
