"""Every liblms kernel once, at small sizes, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python scripts/sanitize_kernels.py
    compute-sanitizer --tool racecheck python scripts/sanitize_kernels.py
    compute-sanitizer --tool synccheck python scripts/sanitize_kernels.py

Covers: the ZVC v3 encode (ZVC and ZX forms, tiles raw / mask / exponent
planes, ragged last tiles) and decode, to HBM and to pinned memory; TMA rows
and transpose pack/unpack and the SIMT fallbacks; the SM zero-copy copy; the
staged strided swap (TMA + copy engine); the measured-simulate op kernel.
Each result is checked, so a clean sanitizer run is also a correct one.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1807_02037_b200 import SimConfig, RewriteConfig, chain, rewrite, simulate, topo_order
    from paper_1807_02037_b200 import runtime as rt

    ctx = rt.Context(device=0, device_reserve=1 << 30, host_chunk=256 << 20, timing=True)
    rt.install_allocator(ctx)
    g = torch.Generator(device="cuda").manual_seed(0)
    n = 3 * 4096 + 77
    cases = {
        "dense": torch.randn(n, device="cuda", generator=g),
        "relu": torch.relu(torch.randn(n, device="cuda", generator=g)),
        "zeros": torch.zeros(n, device="cuda"),
    }
    cases["mixed"] = torch.cat([cases["relu"][:4096], cases["dense"][:4096], cases["zeros"][:4096 + 77]])
    for name, x in cases.items():
        for exps in (False, True):
            for bulk in (1, 0):
                ctx.set_tuning(0, bulk)
                enc = torch.empty(ctx.zvc_bound(n), dtype=torch.uint8, device="cuda")
                ctx.zvc_encode(x, enc, exponents=exps)
                out = torch.empty_like(x)
                ctx.zvc_decode(enc, out)
                torch.cuda.synchronize()
                assert torch.equal(out.view(torch.int32), x.view(torch.int32)), (name, exps, bulk)
        for codec in ("zvc", "zx", "sm", "ce"):
            h = ctx.swap_out(x, codec)
            y = ctx.swap_in(h)
            ctx.wait(h)
            torch.cuda.synchronize()
            assert torch.equal(y.view(torch.int32), x.view(torch.int32)), (name, codec)
            ctx.release(h)
    ctx.set_tuning(0, 1)
    base = torch.randn(4, 48, 20, 36, device="cuda", generator=g)
    for view in (base.permute(0, 2, 3, 1), base[:, 8:40], base[:, :, :, 4:30], base.transpose(1, 3)):
        for tma in (1, 0):
            ctx.set_tuning(0, -1, tma)
            assert torch.equal(ctx.pack(view), view.contiguous())
            dst = torch.zeros_like(base)
            dv = dst.permute(0, 2, 3, 1) if view.shape == base.permute(0, 2, 3, 1).shape else None
            if dv is not None:
                ctx.unpack(view.contiguous(), dv)
                torch.cuda.synchronize()
                assert torch.equal(dv, view)
        ctx.set_tuning(0, -1, 1)
        h = ctx.swap_out(view, "ce")              # strided: staged (TMA pack + copy engine)
        y = ctx.swap_in(h)
        ctx.wait(h)
        torch.cuda.synchronize()
        assert torch.equal(y, view.contiguous())
        ctx.release(h)
    gr = chain(4, tensor_bytes=1 << 16)
    g2, _ = rewrite(gr, RewriteConfig())
    simulate(g2, topo_order(g2), SimConfig())     # lms_sim_op: verifies every input word
    torch.cuda.synchronize()
    print("sanitize_kernels ok")


if __name__ == "__main__":
    main()
