"""Where does device memory go in a swapped ResNet-50 step? (pool live bytes after forward / peak)."""
import sys, gc, json
sys.path.insert(0, '.')
import torch, torchvision
from paper_1807_02037_b200 import runtime as rt, RewriteConfig
from paper_1807_02037_b200.torch_lms import LMS
ctx = rt.Context(device=0, device_reserve=40 << 30, timing=True)
rt.install_allocator(ctx)
torch.backends.cudnn.benchmark = False
torch.backends.cudnn.allow_tf32 = False
m = torchvision.models.resnet50().cuda()
opt = torch.optim.SGD(m.parameters(), lr=0.1, momentum=0.9)
lf = torch.nn.functional.cross_entropy
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
x = torch.randn(B, 3, 224, 224, device="cuda"); y = torch.randint(0, 1000, (B,), device="cuda")
def live(): torch.cuda.synchronize(); ctx.synchronize(); s = ctx.stats(); return round(s["device_in_use"] / 2**30, 3)
print("base", live())
opt.zero_grad(set_to_none=True)
loss = lf(m(x), y)
print("no-swap after fwd", live())
ctx.reset_peaks(); loss.backward(); print("no-swap bwd peak", round(ctx.stats()["device_peak"] / 2**30, 3)); del loss
opt.zero_grad(set_to_none=True); gc.collect(); print("after", live())
lms = LMS(m, lf, opt, RewriteConfig(fuse_swapins=True), ctx, codec="ce", min_swap_bytes=1 << 14)
lms.capture(x[:4], y[:4]); opt.zero_grad(set_to_none=True); gc.collect()
print("plan", json.dumps(lms.plan.summary()))
print("after capture", live())
ex = lms._exec
# replicate SwapExecutor.run forward half to measure
import paper_1807_02037_b200.torch_lms as T
loss_holder = {}
orig = ex.run
def fwd_only():
    l = lf(m(x), y); loss_holder["l"] = l; print("swap after fwd (pre-backward)", live()); return l
ctx.reset_peaks()
opt.zero_grad(set_to_none=True)
ex.run(fwd_only)
print("swap step peak", round(ctx.stats()["device_peak"] / 2**30, 3), "live after", live())
n, sizes = ctx.live_blocks(12)
print("live blocks", n, [round(s / 2**20) for s in sizes])
