"""Zero-copy kernel tuning sweep: CTAs per launch x bulk (TMA) on/off for the ZVC and SM
swap paths, 512 MiB tensors, wire GB/s per direction (CUDA events on the copy channels)."""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1807_02037_b200 import runtime as rt

    ctx = rt.Context(device=0, device_reserve=12 << 30, host_chunk=4 << 30, timing=True)
    rt.install_allocator(ctx)
    n = (512 << 20) // 4
    relu = torch.relu(torch.randn(n, device="cuda"))
    dense = torch.randn(n, device="cuda")
    s = torch.cuda.current_stream()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = []
    for codec, t in (("zvc", relu), ("sm", dense)):
        for bulk in (1, 0):
            if codec == "sm" and bulk == 0:
                continue
            for ctas in (16, 32, 64, 148, 296, 592):
                ctx.set_tuning(ctas, bulk)
                dst = torch.empty_like(t)
                ctx.synchronize()
                ctx.trace_clear()
                hs = []
                for _ in range(4):
                    h = ctx.swap_out(t, codec, s)
                    ctx.swap_in(h, dst, trigger_stream=s)
                    ctx.wait(h, s)
                    hs.append(h)
                torch.cuda.synchronize()
                ctx.synchronize()
                tr = ctx.trace()
                row = {"codec": codec, "bulk": bulk, "ctas": ctas, "ok": bool(torch.equal(dst, t))}
                for dirn, name in ((0, "d2h"), (1, "h2d")):
                    rec = [r for r in tr if r["direction"] == dirn][1:]
                    ms = sum(r["end_ms"] - r["start_ms"] for r in rec)
                    row[name + "_wire_gbs"] = round(sum(r["wire_bytes"] for r in rec) / ms / 1e6, 2)
                for h in hs:
                    ctx.release(h)
                out.append(row)
                print(json.dumps(row), flush=True)
    ctx.set_tuning(sms, 1)


if __name__ == "__main__":
    main()
