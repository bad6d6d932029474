"""OOM inside a swapped backward: memory must come back."""
import sys, gc, time, traceback
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
        for _ in range(2):
            lms.step(x, y)
        print(B, "ok", round(time.time() - t0, 2), "s; peak", round(ctx.stats()["device_peak"] / 2**30, 2), flush=True)
    except RuntimeError as e:
        print(B, "OOM", "".join(traceback.format_exception_only(e))[:150].strip(), flush=True)
        print("   in", [f.name for f in traceback.extract_tb(e.__traceback__)][-4:], flush=True)
    x = y = None
    opt.zero_grad(set_to_none=True); gc.collect()
    n, sizes = ctx.live_blocks(6)
    print("  live after", live(), n, [round(s / 2**20) for s in sizes], flush=True)
    ctx.reset_peaks()
