"""Device live bytes across one swapped ResNet-50 step (forward packs, backward swap-ins).

Usage: python scripts/mem_timeline_probe.py B [reserve_gib]
Prints no-swap peak, swapped peak, and the live-bytes timeline at every swap call.
"""
import sys, gc, json
sys.path.insert(0, '.')
import torch, torchvision
from paper_1807_02037_b200 import runtime as rt, RewriteConfig
from paper_1807_02037_b200.torch_lms import LMS
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ctx = rt.Context(device=0, device_reserve=int(float(sys.argv[2]) if len(sys.argv) > 2 else 40) << 30, timing=True)
rt.install_allocator(ctx)
torch.backends.cudnn.benchmark = False
m = torchvision.models.resnet50().cuda()
opt = torch.optim.SGD(m.parameters(), lr=0.1, momentum=0.9)
lf = torch.nn.functional.cross_entropy
x = torch.randn(B, 3, 224, 224, device="cuda"); y = torch.randint(0, 1000, (B,), device="cuda")
G = 2 ** 30
def st(): return ctx.stats()
def plain():
    opt.zero_grad(set_to_none=True); l = lf(m(x), y); l.backward(); opt.step()
plain(); torch.cuda.synchronize(); ctx.synchronize()
ctx.reset_peaks(); base = st()["device_in_use"]
plain(); torch.cuda.synchronize(); ctx.synchronize()
print("no-swap: base %.2f GiB peak %.2f GiB" % (base / G, st()["device_peak"] / G), flush=True)
lms = LMS(m, lf, opt, RewriteConfig(fuse_swapins=True, swapin_fuse_distance=1), ctx, codec="ce",
          min_swap_bytes=(256 << 10) // 4)
lms.capture(x[:4], y[:4]); opt.zero_grad(set_to_none=True); gc.collect()
print("plan", json.dumps(lms.plan.summary()), flush=True)
tl = []
so, si, wt = ctx.swap_out, ctx.swap_in, ctx.wait
def rec(tag, n):
    s = st(); tl.append((tag, n, round(s["device_in_use"] / G, 3), round(s["device_deferred_bytes"] / G, 3)))
def swap_out(t, codec="ce", stream=None):
    h = so(t, codec, stream); rec("out", t.numel() * t.element_size()); return h
def swap_in(h, dst=None, trigger_stream=None):
    r = si(h, dst, trigger_stream); rec("in", h.logical_bytes); return r
def wait(h, stream=None):
    wt(h, stream); rec("wait", h.logical_bytes)
ctx.swap_out, ctx.swap_in, ctx.wait = swap_out, swap_in, wait
for step in range(2):
    tl.clear(); torch.cuda.synchronize(); ctx.synchronize(); ctx.reset_peaks()
    try:
        lms.step(x, y); torch.cuda.synchronize(); ctx.synchronize()
        print("swap step %d: peak %.2f GiB" % (step, st()["device_peak"] / G), flush=True)
    except RuntimeError as e:
        print("swap step OOM:", str(e)[:200], flush=True)
    mx = max(tl, key=lambda r: r[2]) if tl else None
    print("  max live at", mx, "events", len(tl), flush=True)
for r in tl[::max(1, len(tl) // 60)]:
    print("  ", r)
