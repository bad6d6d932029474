"""OOM inside a swapped backward: memory must come back."""
import sys, gc, time, traceback, faulthandler
faulthandler.dump_traceback_later(50, repeat=True)
sys.path.insert(0, '.')
import torch, torchvision
from paper_1807_02037_b200 import runtime as rt, RewriteConfig
from paper_1807_02037_b200.torch_lms import LMS
ctx = rt.Context(device=0, device_reserve=8 << 30, timing=True)
rt.install_allocator(ctx)
torch.backends.cudnn.benchmark = False
m = torchvision.models.resnet50().cuda()
opt = torch.optim.SGD(m.parameters(), lr=0.1, momentum=0.9)
lf = torch.nn.functional.cross_entropy
def live():
    torch.cuda.synchronize(); ctx.synchronize(); return round(ctx.stats()["device_in_use"] / 2**30, 3)
lms = LMS(m, lf, opt, RewriteConfig(fuse_swapins=True), ctx, codec="ce", min_swap_bytes=1 << 14)
x = torch.randn(4, 3, 224, 224, device="cuda"); y = torch.randint(0, 1000, (4,), device="cuda")
lms.capture(x, y); opt.zero_grad(set_to_none=True); gc.collect()
for B in [int(a) for a in sys.argv[1:]]:
    x = torch.randn(B, 3, 224, 224, device="cuda"); y = torch.randint(0, 1000, (B,), device="cuda")
    t0 = time.time()
    try:
        for i in range(int(__import__("os").environ.get("STEPS", "2"))):
            s0 = ctx.stats(); t1 = time.time()
            lms.step(x, y); torch.cuda.synchronize()
            s1 = ctx.stats()
            d = {k: round(s1[k] - s0[k], 1) for k in ("n_map", "n_unmap", "n_reclaims", "n_device_syncs",
                 "pool_driver_ms", "d2h_busy_ms", "h2d_busy_ms", "swap_wait_ms", "n_deferred_frees")}
            d["GB_d2h"] = round((s1["d2h_wire_bytes"] - s0["d2h_wire_bytes"]) / 1e9, 2)
            d["GB_h2d"] = round((s1["h2d_wire_bytes"] - s0["h2d_wire_bytes"]) / 1e9, 2)
            print(B, "step", i, round(time.time() - t1, 3), "s", d, flush=True)
        print(B, "ok", round(time.time() - t0, 2), "s; peak", round(ctx.stats()["device_peak"] / 2**30, 2), flush=True)
    except RuntimeError as e:
        print(B, "OOM", "".join(traceback.format_exception_only(e))[:150].strip(), flush=True)
        print("   in", [f.name for f in traceback.extract_tb(e.__traceback__)][-4:], flush=True)
    x = y = None
    opt.zero_grad(set_to_none=True); gc.collect()
    n, sizes = ctx.live_blocks(6)
    print("  live after", live(), n, [round(s / 2**20) for s in sizes], flush=True)
    ctx.reset_peaks()
