"""After an OOM inside a swapped step: who holds the device memory? (Python-visible tensors vs pool)."""
import sys, gc, traceback
sys.path.insert(0, '.')
import torch, torchvision
from paper_1807_02037_b200 import runtime as rt, RewriteConfig
from paper_1807_02037_b200.torch_lms import LMS
G = 2 ** 30
ctx = rt.Context(device=0, device_reserve=4 << 30, timing=True)
rt.install_allocator(ctx)
torch.backends.cudnn.benchmark = False
m = torchvision.models.resnet50().cuda()
opt = torch.optim.SGD(m.parameters(), lr=0.1, momentum=0.9)
lf = torch.nn.functional.cross_entropy
lms = LMS(m, lf, opt, RewriteConfig(fuse_swapins=True), ctx, codec="ce", min_swap_bytes=1 << 16)
x = torch.randn(4, 3, 224, 224, device="cuda"); y = torch.randint(0, 1000, (4,), device="cuda")
lms.capture(x, y); opt.zero_grad(set_to_none=True); x = y = None; gc.collect()
def live():
    torch.cuda.synchronize(); ctx.synchronize(); return ctx.stats()["device_in_use"] / G
def pyvisible():
    tot, n, big = 0, 0, []
    seen = set()
    for o in gc.get_objects():
        try:
            if isinstance(o, torch.Tensor) and o.is_cuda:
                k = o.untyped_storage().data_ptr()
                if k in seen: continue
                seen.add(k); nb = o.untyped_storage().nbytes(); tot += nb; n += 1; big.append((nb, o))
        except Exception:
            pass
    big.sort(key=lambda t: -t[0])
    return tot / G, n, big[:3]
print("base live %.3f py %.3f" % (live(), pyvisible()[0]), flush=True)
for B, nt in ((300, 20), (300, -1), (40, -1)):
    lms.replan(RewriteConfig(fuse_swapins=True, n_tensors=nt))
    x = torch.randn(B, 3, 224, 224, device="cuda"); y = torch.randint(0, 1000, (B,), device="cuda")
    try:
        lms.step(x, y); torch.cuda.synchronize(); print(B, nt, "ok", flush=True)
    except RuntimeError as e:
        print(B, nt, "OOM in", [f.name for f in traceback.extract_tb(e.__traceback__)][-5:], flush=True)
        traceback.clear_frames(e.__traceback__)
    x = y = None
    opt.zero_grad(set_to_none=True); gc.collect()
    lv = live(); pv, n, big = pyvisible()
    print("  live %.3f GiB, python-visible cuda tensors %.3f GiB in %d storages" % (lv, pv, n), flush=True)
    for nb, t in big[:2]:
        refs = gc.get_referrers(t)
        print("   ", nb >> 20, "MiB", tuple(t.shape), "grad_fn", type(t.grad_fn).__name__ if t.grad_fn else None,
              "referrers:", [type(r).__name__ for r in refs][:6], flush=True)
        for r in refs[:3]:
            if isinstance(r, (dict, list, tuple)):
                print("      <-", [type(rr).__name__ + (":" + getattr(rr, "__name__", getattr(getattr(rr, "f_code", None), "co_name", ""))) for rr in gc.get_referrers(r)][:6], flush=True)
    st = ctx.stats()
    print("  handles live", st["n_handles_live"], "deferred GiB %.3f" % (st["device_deferred_bytes"] / G), flush=True)
