"""Staging/transfer kernel microbenchmark on one B200 (CUDA events on the launching stream).

Every number is bytes the operation must move ÷ its device time:
  pack / unpack      HBM read + write of the tensor (2 x bytes) vs MEASURED_PEAKS hbm_gbs
  swap D2H / H2D     tensor bytes on the host link vs the copy-engine peak measured here
  zvc encode/decode  logical tensor bytes and wire (compressed) bytes per second

Usage: python scripts/kernel_bench.py [--mib 512] [--iters 5] [--out gpurun_out/kernel_bench.json]
Under ncu, pass --iters 1 --quick so each kernel launches a handful of times.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=512)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "kernel_bench.json"))
    args = ap.parse_args()

    import torch
    from paper_1807_02037_b200 import runtime as rt

    ctx = rt.Context(device=0, device_reserve=(16 * args.mib << 20) + (4 << 30), host_chunk=4 << 30, timing=True)
    rt.install_allocator(ctx)
    dev = torch.device("cuda", 0)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    nbytes = args.mib << 20
    n = nbytes // 4
    res = {"tensor_mib": args.mib, "hbm_peak_gbs": hbm_peak,
           "hbm_peak_source": "MEASURED_PEAKS.json" if peaks else "fallback (B200_PROFILING.md)"}
    s = torch.cuda.current_stream()

    def timed(fn, iters=args.iters, warm=2):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(iters):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters * 1e-3

    want = set(args.only.split(",")) if args.only else None

    def on(name):
        return want is None or name in want

    # NCHW activation -> channels-last view (the transpose path) and a sliced view (rows path)
    C = 64
    HW = 56 * 56
    B = max(1, n // (C * HW))
    x = torch.randn(B, C, 56, 56, device=dev)
    tb = x.numel() * 4
    if on("pack"):
        v = x.permute(0, 2, 3, 1)            # strided: unit stride on W (not last)
        out = torch.empty(v.shape, device=dev)
        t = timed(lambda: ctx.pack(v, out))
        assert torch.equal(out, v.contiguous())
        res["pack_transpose_tma"] = {"gbs": 2 * tb / t / 1e9, "frac_hbm": 2 * tb / t / 1e9 / hbm_peak,
                                     "ms": t * 1e3}
        ctx.set_tuning(0, -1, 0)
        t = timed(lambda: ctx.pack(v, out))
        res["pack_transpose_simt"] = {"gbs": 2 * tb / t / 1e9, "frac_hbm": 2 * tb / t / 1e9 / hbm_peak,
                                      "ms": t * 1e3}
        ctx.set_tuning(0, -1, 1)
        vs = x[:, :, :, 4:52]                # rows path (unit-stride last dim, 192 B rows)
        outs = torch.empty(vs.shape, device=dev)
        b2 = vs.numel() * 4
        t = timed(lambda: ctx.pack(vs, outs))
        res["pack_rows_tma"] = {"gbs": 2 * b2 / t / 1e9, "frac_hbm": 2 * b2 / t / 1e9 / hbm_peak, "ms": t * 1e3}
        assert torch.equal(outs, vs.contiguous())
        vc = x[:, 8:40]                      # channel slice: 16 B-aligned strides, long contiguous runs
        outc = torch.empty(vc.shape, device=dev)
        b3 = vc.numel() * 4
        t = timed(lambda: ctx.pack(vc, outc))
        res["pack_channel_slice_tma"] = {"gbs": 2 * b3 / t / 1e9, "frac_hbm": 2 * b3 / t / 1e9 / hbm_peak,
                                         "ms": t * 1e3}
        assert torch.equal(outc, vc.contiguous())
        ctx.set_tuning(0, -1, 0)             # the SIMT rows kernel on the same views
        t = timed(lambda: ctx.pack(vs, outs))
        res["pack_rows_simt"] = {"gbs": 2 * b2 / t / 1e9, "frac_hbm": 2 * b2 / t / 1e9 / hbm_peak, "ms": t * 1e3}
        t = timed(lambda: ctx.pack(vc, outc))
        res["pack_channel_slice_simt"] = {"gbs": 2 * b3 / t / 1e9, "frac_hbm": 2 * b3 / t / 1e9 / hbm_peak,
                                          "ms": t * 1e3}
        ctx.set_tuning(0, -1, 1)
        refc = torch.empty_like(outc)
        t = timed(lambda: refc.copy_(vc))
        res["torch_contiguous_channel_slice"] = {"gbs": 2 * b3 / t / 1e9, "ms": t * 1e3}
        ref = torch.empty_like(out)
        t = timed(lambda: ref.copy_(v))
        res["torch_contiguous_same_view"] = {"gbs": 2 * tb / t / 1e9, "ms": t * 1e3}
    if on("unpack"):
        v = torch.empty(B, 56, 56, C, device=dev).permute(0, 3, 1, 2)  # channels-last destination
        src = x.contiguous()
        t = timed(lambda: ctx.unpack(src, v))
        assert torch.equal(v, src)
        res["unpack_transpose_tma"] = {"gbs": 2 * tb / t / 1e9, "frac_hbm": 2 * tb / t / 1e9 / hbm_peak,
                                       "ms": t * 1e3}
        big = torch.empty(B, 2 * C, 56, 56, device=dev)
        vd = big[:, 16:16 + C]                # unpack into a channel slice (TMA store path)
        t = timed(lambda: ctx.unpack(src, vd))
        assert torch.equal(vd, src)
        res["unpack_channel_slice_tma"] = {"gbs": 2 * tb / t / 1e9, "frac_hbm": 2 * tb / t / 1e9 / hbm_peak,
                                           "ms": t * 1e3}

    # host-link transfers through the swap engine (per-transfer CUDA events on the copy streams)
    def swap_rates(codec, t_in, settled=False):
        ctx.synchronize()
        ctx.trace_clear()
        hs = []
        ok = True
        dst = torch.empty_like(t_in)
        for _ in range(max(2, args.iters)):
            h = ctx.swap_out(t_in, codec, s)
            if settled:   # the swap-out landed before the swap-in is issued, as in a training step
                torch.cuda.synchronize()
                ctx.synchronize()
            ctx.swap_in(h, dst, trigger_stream=s)
            ctx.wait(h, s)
            hs.append(h)
        torch.cuda.synchronize()
        ctx.synchronize()
        ok = torch.equal(dst, t_in)
        tr = ctx.trace()
        st = ctx.stats()
        for h in hs:
            ctx.release(h)
        out = {"ok": ok}
        for dirn, name in ((0, "d2h"), (1, "h2d")):
            recs = [r for r in tr if r["direction"] == dirn][1:]  # first one is a warm-up
            if not recs:
                continue
            busy = sum(r["end_ms"] - r["start_ms"] for r in recs) * 1e-3
            logical = sum(r["logical_bytes"] for r in recs)
            wire = sum(r["wire_bytes"] for r in recs)
            out[name] = {"logical_gbs": logical / busy / 1e9, "wire_gbs": wire / busy / 1e9,
                         "wire_frac": wire / max(logical, 1), "ms_each": busy / len(recs) * 1e3}
        out["kernel_launches"] = st["kernel_launches"]
        return out

    if on("swap"):
        dense = torch.randn(n, device=dev)
        relu = torch.relu(torch.randn(n, device=dev))   # ~50% zero words, like a ReLU output
        res["swap_ce_dense"] = swap_rates("ce", dense)
        res["swap_sm_dense"] = swap_rates("sm", dense)
        res["swap_zvc_relu"] = swap_rates("zvc", relu)
        res["swap_zvc_dense"] = swap_rates("zvc", dense)
        res["swap_zx_relu"] = swap_rates("zx", relu)
        res["swap_zx_dense"] = swap_rates("zx", dense)
        # swap-ins issued after their swap-out landed (as in a training step)
        res["swap_zx_dense_settled"] = swap_rates("zx", dense, settled=True)
        res["swap_zx_relu_settled"] = swap_rates("zx", relu, settled=True)
        res["swap_ce_relu"] = swap_rates("ce", relu)
        # strided views (not dense in memory): channels-last view of NCHW and a channel slice
        xv = torch.randn(max(1, n // (64 * 56 * 56)), 64, 56, 56, device=dev)
        res["swap_ce_channels_last_view"] = swap_rates("ce", xv.permute(0, 2, 3, 1))
        res["swap_ce_channel_slice"] = swap_rates("ce", xv[:, 8:40])

    if on("zvc"):
        # HBM-side codec rates: one pass reads the tensor and writes the encoded
        # stream (decode: the reverse); algorithmic HBM bytes = tensor + wire bytes
        relu = torch.relu(torch.randn(n, device=dev))
        dense = torch.randn(n, device=dev)
        for name, src, exps in (("zvc", relu, False), ("zx", relu, True), ("zx_dense", dense, True)):
            enc = torch.empty(ctx.zvc_bound(n), dtype=torch.uint8, device=dev)
            t = timed(lambda: ctx.zvc_encode(src, enc, exponents=exps))
            torch.cuda.synchronize()
            wire = ctx.zvc_encoded_size(enc.cpu())
            res[f"{name}_encode_hbm"] = {"logical_gbs": nbytes / t / 1e9, "hbm_gbs": (nbytes + wire) / t / 1e9,
                                         "frac_hbm": (nbytes + wire) / t / 1e9 / hbm_peak,
                                         "wire_frac": wire / nbytes, "ms": t * 1e3}
            outd = torch.empty_like(src)
            t = timed(lambda: ctx.zvc_decode(enc, outd))
            assert torch.equal(outd.view(torch.int32), src.view(torch.int32))
            res[f"{name}_decode_hbm"] = {"logical_gbs": nbytes / t / 1e9, "hbm_gbs": (nbytes + wire) / t / 1e9,
                                         "frac_hbm": (nbytes + wire) / t / 1e9 / hbm_peak, "ms": t * 1e3}

    print(json.dumps(res, indent=1))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
