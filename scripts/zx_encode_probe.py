"""One ZX encode + decode of a ReLU-like 256 MiB tensor in HBM, a few times (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1807_02037_b200 import runtime as rt
    ctx = rt.Context(device=0, device_reserve=4 << 30, timing=False)
    rt.install_allocator(ctx)
    n = (256 << 20) // 4
    kind = sys.argv[1] if len(sys.argv) > 1 else "relu"
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, device="cuda", generator=g)
    if kind == "relu":
        x = torch.relu(x)
    enc = torch.empty(ctx.zvc_bound(n), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(x)
    for _ in range(3):
        ctx.zvc_encode(x, enc, exponents=True)
        ctx.zvc_decode(enc, out)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int32), x.view(torch.int32))
    print("ok", ctx.zvc_encoded_size(enc.cpu()) / (4 * n))


if __name__ == "__main__":
    main()
