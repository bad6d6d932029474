"""After an OOM inside a swapped step, is device memory released?"""
import sys, gc, json, faulthandler
faulthandler.dump_traceback_later(45, repeat=True)
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
import time
def pstats(tag):
    s = ctx.stats()
    print(tag, {k: (round(s[k], 1) if isinstance(s[k], float) else s[k]) for k in
                ("n_map", "n_unmap", "n_reclaims", "n_device_syncs", "n_oom", "pool_driver_ms")}, flush=True)
def live():
    torch.cuda.synchronize(); ctx.synchronize(); s = ctx.stats(); return round(s["device_in_use"] / 2**30, 3)
lms = LMS(m, lf, opt, RewriteConfig(fuse_swapins=True), ctx, codec="ce", min_swap_bytes=1 << 14)
x = torch.randn(4, 3, 224, 224, device="cuda"); y = torch.randint(0, 1000, (4,), device="cuda")
t0 = time.time(); lms.capture(x, y); opt.zero_grad(set_to_none=True); gc.collect(); print("capture s", time.time() - t0)
pstats("after capture")
print("after capture", live())
for B in (int(a) for a in (sys.argv[1:] or ["400", "96", "400", "96"])):
    x = torch.randn(B, 3, 224, 224, device="cuda"); y = torch.randint(0, 1000, (B,), device="cuda")
    t0 = time.time()
    try:
        for _ in range(2):
            lms.step(x, y)
        print(B, "ok", round(time.time() - t0, 1), "s peak", round(ctx.stats()["device_peak"] / 2**30, 2))
    except RuntimeError as e:
        print(B, "OOM", str(e)[:120])
    x = y = None
    opt.zero_grad(set_to_none=True)
    gc.collect()
    print("  live after", live(), ctx.live_blocks(8)[0], [round(s / 2**20) for s in ctx.live_blocks(8)[1]])
    pstats("  pool")
    ctx.reset_peaks()
